"""CPU: bench.py's multi-GPU launcher. `--gpus N` outside torchrun re-runs the
script under torch.distributed.run with N ranks (here: gloo, no GPU work);
rank 0 prints one JSON line with n_gpus = N and the N > 1 default workload
(config C, one atlas row-sharded)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _run(*args):
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=240, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    return json.loads(lines[0])


def test_gpus_2_relaunches_two_ranks():
    line = _run("--gpus", "2", "--launch-selftest")
    assert line["n_gpus"] == 2 and line["mode"] == "shard" and line["config_name"] == "C"
    assert "config C" in line["metric"]


def test_gpus_1_is_config_b_single():
    line = _run("--launch-selftest")
    assert line["n_gpus"] == 1 and line["mode"] == "single" and line["config_name"] == "B"


def test_both_arms_print_the_same_config_dict():
    import bench
    from paper_2605_26137_b200 import fixtures as fx
    pair = fx.bake_pair(8, 2, 64, name="B")
    for mode, world in (("single", 1), ("shard", 4), ("batch", 8)):
        a = bench.config_dict("B", pair, mode, world, 8, seed=7)
        b = bench.config_dict("B", pair, mode, world, 8, seed=7)
        assert a == b and a["l2"] and a["parallelism"]
    args = bench.parse(["--gpus", "8"])
    assert bench.resolve(args, 8) == ("shard", "C")
    assert bench.resolve(bench.parse(["--mode", "batch"]), 8) == ("batch", "D")

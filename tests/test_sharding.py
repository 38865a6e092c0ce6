"""CPU: the multi-GPU row-sharding plumbing with world_size 2
over gloo. The per-rank bake is the CPU oracle sliced to the rank's rows (the
device slab path is covered by tests/test_gpu_shards.py); what is under test
here is the balanced partition, the padding and the all-gather assembly."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2605_26137_b200 import sharding


def test_balanced_row_ranges_cover_and_balance():
    rng = np.random.default_rng(0)
    counts = np.concatenate([rng.integers(200, 400, 300), np.zeros(212, np.int64)])  # packed from row 0
    for k in (1, 2, 3, 4, 8):
        r = sharding.balanced_row_ranges(counts, k)
        assert r[0][0] == 0 and r[-1][1] == counts.size
        assert all(a < b for a, b in r) and all(r[i][1] == r[i + 1][0] for i in range(k - 1))
        loads = [int(counts[a:b].sum() + (b - a)) for a, b in r]
        assert max(loads) - min(loads) <= 2 * 401  # each cut is off by < one row weight
    with pytest.raises(ValueError):
        sharding.balanced_row_ranges([1, 2], 3)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, full, ranges, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        atlas = sharding.sharded_bake(lambda b, e: full[b:e], ranges, rank)
        np.save(os.path.join(out_dir, f"rank{rank}.npy"), np.asarray(atlas))
    finally:
        dist.destroy_process_group()


def test_sharded_bake_gloo_world2(port, tmp_path):
    from paper_2605_26137_b200 import fixtures as fx
    p = fx.bake_pair(24, 4, 64, name="shard")
    res = port.bake(p.lowpoly, p.dense, p.res, p.bbox_diagonal, p.max_distance_fraction, 4)
    full = res["rgb"].reshape(p.res, p.res, 3)
    g = port.raster_gbuffer(p.lowpoly, p.res)
    ranges = sharding.balanced_row_ranges(g.valid.reshape(p.res, p.res).sum(1), 2)
    mp.spawn(_worker, args=(2, _free_port(), full, ranges, str(tmp_path)), nprocs=2, join=True)
    for r in range(2):
        assert np.array_equal(np.load(tmp_path / f"rank{r}.npy"), full)

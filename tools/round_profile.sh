#!/bin/bash
# Round evidence: parity tests, smoke, bench line, launch list and full ncu
# captures of the main kernels. Raw artefacts -> gpurun_out/, summaries are
# produced here afterwards with tools/ncu_summary.py into profiles/.
set -u
TAG=${TAG:-r01}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,driver_version --format=csv > $OUT/${TAG}_smi.txt
lscpu | grep -E "Model name|^CPU\(s\)" > $OUT/${TAG}_host.txt
timeout 900 python -m pytest tests -q -m gpu > $OUT/${TAG}_pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.txt
tail -2 $OUT/${TAG}_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.txt 2>&1; echo "smoke rc=$?" >> $OUT/${TAG}_smoke.txt
timeout 600 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/${TAG}_bench_reference.json 2>> $OUT/${TAG}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
  --log-file $OUT/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-rays \
  > $OUT/${TAG}_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k 'regex:k_transfer_t|k_raster|k_interp|k_refit_ranges|k_dilate_links' -c 5 \
  -o $OUT/${TAG}_prof -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-rays \
  > $OUT/${TAG}_ncu_full.log 2>&1; echo "ncu full rc=$?"
# per-kernel counters of every bake / secondary kernel (raw CSV) and the
# CUPTI timelines of the device bake and of the host-buffer entry point
TAG=$TAG bash tools/ncu_all.sh
timeout 300 python tools/timeline.py B 7 2>/dev/null | grep -v Warn > $OUT/${TAG}_timeline_B.txt
TL_E2E=1 timeout 300 python tools/timeline.py B 7 2>/dev/null | grep -v Warn > $OUT/${TAG}_timeline_e2e.txt
TAG=$TAG bash tools/configs_run.sh
# config E's wide-leaf kernels (triangle planes in the repack, leaf planes, the wide transfer)
M=$(python -c "import sys; sys.path.insert(0, 'tools'); import ncu_summary as n; print(','.join(n.METRICS))")
timeout 900 ncu --metrics $M --clock-control none --csv --page raw -k 'regex:k_repack|k_leaf_planes|k_transfer_t' -c 3 \
  --log-file $OUT/${TAG}_E_metrics.csv python bench.py --config E --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
  --no-rays > $OUT/${TAG}_ncu_E.log 2>&1; echo "E metrics rc=$?"

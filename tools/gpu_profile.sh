#!/bin/bash
# One GPU session: parity tests, bench, launch list and a full ncu capture of
# the dominant kernel. Outputs under gpurun_out/ (merged back by gpurun).
set -u
OUT=gpurun_out
mkdir -p $OUT
TAG=${TAG:-r01}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/${TAG}_smi.txt
lscpu | grep -E "Model name|^CPU\(s\)" > $OUT/${TAG}_host.txt
if [ "${TESTS:-1}" = 1 ]; then
  timeout 900 python -m pytest tests -x -q -m gpu > $OUT/${TAG}_pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.txt
  tail -3 $OUT/${TAG}_pytest_gpu.txt
fi
if [ "${BENCH:-1}" = 1 ]; then
  timeout 900 python bench.py ${BENCH_ARGS:-} > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err; echo "bench rc=$?"
  cat $OUT/${TAG}_bench.json
fi
if [ "${NCU:-1}" = 1 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline \
    > $OUT/${TAG}_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${KERNEL:-k_transfer} -s 1 -c 1 \
    -o $OUT/${TAG}_prof_${KERNEL:-k_transfer} -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
    > $OUT/${TAG}_ncu_full.log 2>&1; echo "ncu full rc=$?"
fi

#!/bin/bash
# Parity tests + quick bench lines for env-var variants (tuning experiments).
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for v in ${VARIANTS:-"MFB_LEAF_MAX=4"}; do
  env $v timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],3), 'ms', {k:round(v,3) for k,v in d['stage_ms'].items()})"
done

#!/bin/bash
# A/B timing of library variants / env settings on config B (device-resident
# bake, graph replay), each run twice, interleaved:  VARIANTS="base MFB_LIB=build/var/pf1/libmfbake.so" tools/ab.sh
# AB_E2E=1 also times the host-buffer entry point (pinned) and prints its ms.
mkdir -p gpurun_out
E2E_FLAG=--no-e2e; [ "${AB_E2E:-0}" = 1 ] && E2E_FLAG=
for rep in 1 2; do
for v in ${VARIANTS:-base}; do
  e=${v//+/ }; [ "$v" = base ] && e="MFB_NOOP=1"
  env $e timeout 300 python bench.py --steps 20 --warmup 3 $E2E_FLAG --no-cpu-baseline --no-rays ${BENCH_ARGS} 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); e=d.get('e2e') or {}
print('$v'.replace('/libmfbake.so','').replace('MFB_LIB=build/var/',''), round(d['ms_per_step'],4), 'ms', 'e2e', round(e.get('ms_per_step', 0), 4), {k:round(v,3) for k,v in d['stage_ms'].items()})"
done
done

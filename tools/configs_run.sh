#!/bin/bash
# Bench lines for the other BASELINE configs (A, C at N=1, D batch of 8 assets, E stress).
# Raw lines -> gpurun_out/${TAG}_cfg_*.json
TAG=${TAG:-r01c}
mkdir -p gpurun_out
for c in A C E; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_cfg_$c.json 2> gpurun_out/${TAG}_cfg_$c.err
  echo "config $c rc=$?"
done
timeout 900 python bench.py --config D --mode batch --assets 8 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_cfg_D8.json 2> gpurun_out/${TAG}_cfg_D8.err
echo "config D rc=$?"

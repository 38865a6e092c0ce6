#!/bin/bash
# ncu counters of every kernel the bake and its §8f consumers launch, for
# profiles/ (the metric list of tools/ncu_summary.py, collected directly as a
# raw CSV so nothing large comes back): one graph-replayed config-B bake (all
# of its kernels: LBVH chain, lowpoly prep, raster, dilation links,
# transfer), then the secondary kernels (raycast / closest point / surface
# band / visibility z-buffer / texfuse / the API dilation kernels).
#   TAG=r02g bash tools/ncu_all.sh      (through gpurun; one GPU)
set -u
TAG=${TAG:-r02}
OUT=gpurun_out
mkdir -p $OUT
M=$(python -c "import sys; sys.path.insert(0, 'tools'); import ncu_summary as n; print(','.join(n.METRICS))")
timeout 1200 ncu --metrics $M --clock-control none --csv --page raw -k 'regex:^(k_|cub)' \
  --launch-skip 200 -c 45 --log-file $OUT/${TAG}_bake_metrics.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-rays > $OUT/${TAG}_ncu_bake.log 2>&1
echo "bake metrics rc=$?"
timeout 1200 ncu --metrics $M --clock-control none --csv --page raw \
  -k 'regex:k_raycast|k_closest$|k_sdf|k_surface_band|k_zbuf|k_edge_mask|k_halve|k_blur|k_unsharp|k_backproject|k_incidence|k_blend|k_valid_bounds|k_dilate_sparse|k_dilate_fused' \
  -c 40 --log-file $OUT/${TAG}_secondary_metrics.csv python tools/secondary_kernels.py > $OUT/${TAG}_ncu_secondary.log 2>&1
echo "secondary metrics rc=$?"

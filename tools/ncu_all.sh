#!/bin/bash
# Full ncu captures (--set full) of every kernel the bake and its §8f
# consumers launch, for profiles/: one graph-replayed config-B bake (all of
# its kernels, LBVH chain + lowpoly prep + raster + dilation links +
# transfer), then the secondary kernels (raycast / closest point / surface
# band / visibility z-buffer / texfuse / the API dilation kernels).
#   TAG=r02d bash tools/ncu_all.sh      (run through gpurun; one GPU)
set -u
TAG=${TAG:-r02}
OUT=gpurun_out
mkdir -p $OUT
# bake: skip the first eager bakes and captures (warmup 3 steps + timing), take one replay's kernels
timeout 1500 ncu --set full --clock-control none --import-source on -k 'regex:^(k_|cub|DeviceRadix|DeviceScan)' \
  --launch-skip 200 -c 60 -o $OUT/${TAG}_bake_all -f \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-rays > $OUT/${TAG}_ncu_bake_all.log 2>&1
echo "bake capture rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k 'regex:k_raycast|k_closest|k_surface_band|k_zbuf|k_edge_mask|k_halve|k_blur|k_unsharp|k_backproject|k_incidence|k_blend|k_valid_bounds|k_dilate_sparse|k_dilate_fused|k_render_views' \
  -c 40 -o $OUT/${TAG}_secondary -f python tools/secondary_kernels.py > $OUT/${TAG}_ncu_secondary.log 2>&1
echo "secondary capture rc=$?"

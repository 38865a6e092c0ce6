#!/bin/bash
# Build libmfbake.so with extra compile flags into build/var/<name>/ for A/B
# timing through MFB_LIB (e.g. MFB_LIB=build/var/pf1/libmfbake.so python bench.py).
#   tools/build_variant.sh minb7 -DMFB_XFER_T_MINB=7
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=build/var/$name
mkdir -p $out
NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC -Iinclude -Iinclude/eigen_shim --expt-relaxed-constexpr $*"
objs=""
for f in paper_2605_26137_b200/csrc/*.cu; do
  o=$out/$(basename $f .cu).o
  nvcc $NVFLAGS -c $f -o $o &
  objs="$objs $o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libmfbake.so $objs -Xlinker -soname=libmfbake.so
rm -f $objs
echo "$out/libmfbake.so ($*)"

for v in base prio0 dnmid; do
  if [ $v = base ]; then L=""; else L="MFB_LIB=build/var/$v/libmfbake.so"; fi
  env $L python tools/timeline.py B 7 > gpurun_out/r02_tl_$v.txt 2>&1
  head -2 gpurun_out/r02_tl_$v.txt | tail -1
done
VARIANTS="base MFB_LIB=build/var/prio0/libmfbake.so MFB_LIB=build/var/dnmid/libmfbake.so" bash tools/ab.sh

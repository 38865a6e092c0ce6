for v in prof32 prof64 prof128; do MFB_LIB=build/var/$v/libmfbake.so python tools/timeline.py B 3 2>&1 | grep "\[prep\]" | tail -3; done
TESTS="tests/test_gpu_bake.py tests/test_gpu_configs.py" TAG=it4 bash tools/iter.sh

RUTV_BUILD_OUT=/tmp/libLP.so RUTV_NVCC_EXTRA="-DRUTV_LEAF_PROF" python paper_2002_06960_b200/build.py > /dev/null || exit 1
RUTV_LIB=/tmp/libLP.so timeout 300 python tools/bench_kernels.py qr 2>&1 | grep leafprof | sort | uniq -c | head -20
RUTV_LEAF_CLUSTER=0 RUTV_LIB=/tmp/libLP.so timeout 300 python tools/bench_kernels.py qr 2>&1 | grep leafprof | sort | uniq -c | head -8

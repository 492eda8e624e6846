python paper_2002_06960_b200/build.py > /dev/null || exit 1
for jt in 512 1024; do
  RUTV_BUILD_OUT=/tmp/libJ$jt.so RUTV_NVCC_EXTRA="-DRUTV_JT=$jt" python paper_2002_06960_b200/build.py > /dev/null || exit 1
done
echo "== JT=256"; timeout 300 python tools/bench_kernels.py svd
for jt in 512 1024; do echo "== JT=$jt"; RUTV_LIB=/tmp/libJ$jt.so timeout 300 python tools/bench_kernels.py svd; done
RUTV_LIB=/tmp/libJ512.so timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k svd 2>&1 | tail -2

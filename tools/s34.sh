python paper_2002_06960_b200/build.py > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_randutv.py -q -x -p no:cacheprovider 2>&1 | tail -3
for c in 1 0; do echo "== RUTV_LEAF_CLUSTER=$c"; RUTV_LEAF_CLUSTER=$c timeout 300 python tools/bench_kernels.py qr; done

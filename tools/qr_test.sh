python paper_2002_06960_b200/build.py > /dev/null || exit 1
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "panel_qr" 2>&1 | tail -3
for r in 1 2; do echo "== RUTV_LEAF_R=$r"; RUTV_LEAF_R=$r timeout 300 python tools/bench_kernels.py qr; done
timeout 600 python -m pytest tests/test_gpu_randutv.py -q -x -p no:cacheprovider 2>&1 | tail -3

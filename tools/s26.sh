python paper_2002_06960_b200/build.py > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_randutv.py tests/test_gpu_kernels.py -q -x -p no:cacheprovider 2>&1 | tail -3
bash tools/s25.sh

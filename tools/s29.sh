python paper_2002_06960_b200/build.py > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_host.py -q -x -p no:cacheprovider 2>&1 | grep -v "^  " | tail -15
RUTV_HOST_UV_BATCH=1 timeout 600 python -m pytest tests/test_gpu_host.py -q -x -p no:cacheprovider 2>&1 | tail -1
for g in 4 8 1; do RUTV_HOST_UV_BATCH=$g timeout 900 python bench.py --mode host --steps 1 --warmup 1 > gpurun_out/bench_host_c3_g$g.json 2>> gpurun_out/bench_host.err; echo "G=$g rc=$?"; cut -c1-120 gpurun_out/bench_host_c3_g$g.json; done
tail -3 gpurun_out/bench_host.err

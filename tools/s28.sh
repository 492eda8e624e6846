python paper_2002_06960_b200/build.py > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_host.py -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 900 python bench.py --mode host --steps 1 --warmup 1 --no-uv --cache-gib 0.5 > gpurun_out/bench_host_c3_tonly.json 2> gpurun_out/bench_host.err; echo "host T-only rc=$?"; cat gpurun_out/bench_host_c3_tonly.json
timeout 900 python bench.py --mode host --steps 1 --warmup 1 > gpurun_out/bench_host_c3.json 2>> gpurun_out/bench_host.err; echo "host rc=$?"; cat gpurun_out/bench_host_c3.json
tail -3 gpurun_out/bench_host.err

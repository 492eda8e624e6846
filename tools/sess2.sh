mkdir -p gpurun_out
python tools/host_model_check.py > gpurun_out/hm.log 2>&1; RUTV_HOST_EVICT=lru python tools/host_model_check.py >> gpurun_out/hm.log 2>&1; cat gpurun_out/hm.log
timeout 600 python -m pytest tests/test_gpu_host.py tests/test_gpu_dist.py -q -x > gpurun_out/t2.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t2.log
timeout 1200 python bench.py --config c5 --mode host --no-uv --cache-gib 16 --steps 1 --warmup 0 > gpurun_out/host_c5_16g_belady.json 2> gpurun_out/host_c5.err; echo "c5 belady rc=$?"; cut -c1-1500 gpurun_out/host_c5_16g_belady.json
RUTV_HOST_EVICT=lru timeout 1200 python bench.py --config c5 --mode host --no-uv --cache-gib 16 --steps 1 --warmup 0 > gpurun_out/host_c5_16g_lru.json 2>> gpurun_out/host_c5.err; echo "c5 lru rc=$?"; cut -c1-1500 gpurun_out/host_c5_16g_lru.json

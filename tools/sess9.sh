mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_randutv.py tests/test_gpu_faults.py tests/test_gpu_host.py tests/test_gpu_dist.py tests/test_gpu_kernels.py -q -x -p no:cacheprovider > gpurun_out/t9.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/t9.log
for v in 1 0 1 0; do
  RUTV_UDEFER=$v timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('udefer=$v', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['other_kernels']['fold_wait'])"
done
RUTV_TRACE=gpurun_out/trace_c3_r02.json timeout 600 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; ls -la gpurun_out/trace_c3_r02.json
timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | cut -c1-200

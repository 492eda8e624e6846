mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_randutv.py tests/test_gpu_host.py -q -x -p no:cacheprovider > gpurun_out/t12.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t12.log
for c in c3 c2 c3; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('$c', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['other_kernels']['qr_leaf'], d['roofline']['other_kernels']['fold_wait'])"; done
RUTV_TRACE=gpurun_out/trace_c3_r02.json timeout 600 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; ls -la gpurun_out/trace_c3_r02.json

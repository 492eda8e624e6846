mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_randutv.py -q -x -p no:cacheprovider > gpurun_out/t10.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t10.log
RUTV_UDEFER=1 timeout 1200 python -m pytest tests/test_gpu_randutv.py -q -x -p no:cacheprovider -k "random or c1_full or c2_full or async or two_contexts or econ" > gpurun_out/t10b.log 2>&1; echo "tests udefer rc=$?"; tail -3 gpurun_out/t10b.log
for v in 1 0 1 0; do
  RUTV_UDEFER=$v timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('c3 udefer=$v', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['other_kernels']['fold_wait'])"
  RUTV_UDEFER=$v timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('c2 udefer=$v', d['value'], d['ms_per_step'])"
done

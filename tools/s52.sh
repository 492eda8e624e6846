python paper_2002_06960_b200/build.py > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_randutv.py -q -x -p no:cacheprovider 2>&1 | tail -2
for v in 1 0 1 0; do
  RUTV_VSTREAM=$v timeout 600 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('vstream=$v bench', d['value'], d['ms_per_step'], d['roofline']['other_kernels']['fold_wait'])"
done
RUTV_VSTREAM=1 timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('c2 vstream=1', d['value'], d['ms_per_step'])"

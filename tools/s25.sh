python paper_2002_06960_b200/build.py > /dev/null || exit 1
timeout 600 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('bench', d['value'], d['ms_per_step'], d['roofline']['achieved']); print(d['roofline']['other_kernels'])"

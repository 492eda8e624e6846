python paper_2002_06960_b200/build.py > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_randutv.py -q -x -p no:cacheprovider 2>&1 | tail -3
for f in 1 0 1 0; do
  RUTV_GEMM_FIXUP=$f timeout 600 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('fixup=$f bench', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['gpu_launches_per_step'])"
done
RUTV_GEMM_FIXUP=1 timeout 300 python tools/bench_kernels.py gemm | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print(f\"{d['case']:24s} {d['tflops']:7.2f}\")"

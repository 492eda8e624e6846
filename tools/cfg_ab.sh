#!/bin/bash
# GEMM tile configurations side by side (same build): RUTV_GEMM_CFG=2 (64x64) vs 1 (128x64)
python paper_2002_06960_b200/build.py > /dev/null || exit 1
for c in 2 1; do
  echo "== RUTV_GEMM_CFG=$c"
  RUTV_GEMM_CFG=$c timeout 300 python tools/bench_kernels.py gemm 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print(f\"{d['case']:24s} {d['tflops']:7.2f}\")"
  RUTV_GEMM_CFG=$c timeout 600 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('bench', d['value'], d['ms_per_step'], d['roofline']['achieved'])"
done
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider 2>&1 | tail -2

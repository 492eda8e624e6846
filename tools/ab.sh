#!/bin/bash
# A/B of two builds of the library in one GPU session: tools/ab.sh "<nvcc extra flags for B>" [bench args]
# A = default build (librandutv.so), B = RUTV_NVCC_EXTRA build in /tmp.
mkdir -p gpurun_out
python paper_2002_06960_b200/build.py > /dev/null || exit 1
RUTV_BUILD_OUT=/tmp/libB.so RUTV_NVCC_EXTRA="$1" python paper_2002_06960_b200/build.py > /dev/null || exit 1
shift
for rep in 1 2; do
  for v in A B; do
    if [ $v = B ]; then export RUTV_LIB=/tmp/libB.so; else unset RUTV_LIB; fi
    echo "== $v rep $rep" | tee -a gpurun_out/ab.log
    timeout 300 python tools/bench_kernels.py gemm 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print(f\"{d['case']:24s} {d['tflops']:7.2f}\")" | tee -a gpurun_out/ab.log
    timeout 600 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu-baseline "$@" 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('bench', d['value'], d['ms_per_step'], d['roofline']['achieved'])" | tee -a gpurun_out/ab.log
  done
done

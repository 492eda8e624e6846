#!/bin/bash
# A/B of library builds in one GPU session:
#   tools/ab.sh "<nvcc extra flags for B1>" ["<flags for B2>" ...]
# A = the default build (librandutv.so); Bi = RUTV_NVCC_EXTRA builds under /tmp.
# Per build and repetition: the DGEMM shape sweep (tools/gemm_shapes.py, steps
# $AB_STEPS) and a short c3 bench.
mkdir -p gpurun_out
python paper_2002_06960_b200/build.py > /dev/null || exit 1
libs=("")
names=("A")
i=0
for flags in "$@"; do
  i=$((i + 1))
  RUTV_BUILD_OUT=/tmp/libB$i.so RUTV_NVCC_EXTRA="$flags" python paper_2002_06960_b200/build.py > /dev/null || { echo "build B$i failed"; exit 1; }
  libs+=("/tmp/libB$i.so")
  names+=("B$i [$flags]")
done
for rep in 1 2; do
  for j in "${!libs[@]}"; do
    if [ -n "${libs[$j]}" ]; then export RUTV_LIB=${libs[$j]}; else unset RUTV_LIB; fi
    echo "== ${names[$j]} rep $rep" | tee -a gpurun_out/ab.log
    STEPS=${AB_STEPS:-0,32,48,56} timeout 300 python tools/gemm_shapes.py 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print(f\"  step {d['step']:2d} {d['case']:14s} {d['ours_TF']:7.2f}  (cuBLAS {d['cublas_TF']:6.2f})\")" | tee -a gpurun_out/ab.log
    timeout 600 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('  bench c3', d['value'], d['ms_per_step'], d['roofline']['achieved'])" | tee -a gpurun_out/ab.log
  done
done

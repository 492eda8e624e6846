#!/bin/bash
# one ncu --set full capture of the dominant DGEMM launch of the c3 bench step: the fused
# S5+S7 rank-2b update of T at step 0 (dgemm launch #73 of the step, 16384 x 16128, K = 512)
mkdir -p gpurun_out
python paper_2002_06960_b200/build.py > /dev/null || exit 1
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-profile"
timeout 900 $CMD > gpurun_out/plain_dom.log 2>&1 || { echo "plain failed"; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dgemm_kernel --launch-skip 73 --launch-count 1 \
  -o gpurun_out/prof_dominant $CMD > gpurun_out/ncu_dom.log 2>&1; echo "ncu rc=$?"

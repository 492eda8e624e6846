#!/bin/bash
# ncu --set full captures of two DGEMM launches from tools/bench_kernels.py gemm:
# the skinny S2 product (launch 0) and the rank-b update S5 X -= Z2 W^T (launch 18).
mkdir -p gpurun_out
python paper_2002_06960_b200/build.py > /dev/null
CMD="env RUTV_GEMM_CFG=${RUTV_GEMM_CFG:-2} python tools/bench_kernels.py gemm"
timeout 300 $CMD > gpurun_out/ncu_gemm_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dgemm_kernel --launch-skip 18 --launch-count 1 \
  -o gpurun_out/prof_rankb $CMD > gpurun_out/ncu_rankb.log 2>&1; echo "ncu rankb rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dgemm_kernel --launch-skip 0 --launch-count 1 \
  -o gpurun_out/prof_skinny $CMD > gpurun_out/ncu_skinny.log 2>&1; echo "ncu skinny rc=$?"
ls -la gpurun_out/*.ncu-rep

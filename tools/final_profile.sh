#!/bin/bash
# ncu evidence for the committed kernels: (1) the launch list of one c3 step (bench command),
# (2) one --set full capture of the dominant GEMM (the S5/S7 rank-2b fused update of T, c3, step 1).
mkdir -p gpurun_out
python paper_2002_06960_b200/build.py > /dev/null || exit 1
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-profile"
timeout 900 $CMD > gpurun_out/plain.log 2>&1 || { echo "plain failed"; exit 1; }
timeout 3000 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base mangled -k regex:rutv \
  --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:dgemm_kernel --launch-skip 40 --launch-count 1 -o gpurun_out/prof_step_gemm $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"

#!/bin/bash
# A/B of the QR leaf plans and the Jacobi variants (bench_kernels qr / svd)
mkdir -p gpurun_out
for v in "RUTV_LEAF_MAXUNITS=5" "RUTV_LEAF_MAXUNITS=2" "RUTV_LEAF_MAXUNITS=1" "RUTV_LEAF_CLUSTER=0"; do
  echo "== $v" >> gpurun_out/leaf_ab.log
  env $v timeout 300 python tools/bench_kernels.py qr >> gpurun_out/leaf_ab.log 2>&1
done
for v in "RUTV_JACOBI_CLUSTER=1" "RUTV_JACOBI_CLUSTER=0"; do
  echo "== $v" >> gpurun_out/leaf_ab.log
  env $v timeout 300 python tools/bench_kernels.py svd >> gpurun_out/leaf_ab.log 2>&1
done
RUTV_LIB=build_var/librandutv_jprof.so timeout 300 python tools/bench_kernels.py svd > gpurun_out/jprof.log 2>&1

#!/bin/bash
# Tail-split DGEMM schedule A/B (round 2d): GEMM tests, c3 shape sweep, c3/c2 benches with RUTV_GEMM_TAIL=1/0.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -k "dgemm" -p no:cacheprovider > gpurun_out/pt_gemm.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pt_gemm.log
STEPS=${STEPS:-0,16,32,40,44,48,52,56,60} timeout 400 python tools/gemm_shapes.py > gpurun_out/shapes_tail1.log 2>&1
RUTV_GEMM_TAIL=0 STEPS=${STEPS:-0,16,32,40,44,48,52,56,60} timeout 400 python tools/gemm_shapes.py > gpurun_out/shapes_tail0.log 2>&1
for t in 1 0 1 0; do
  RUTV_GEMM_TAIL=$t timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_t$t.json 2>gpurun_out/bench_t$t.err
  python -c "import json;d=json.load(open('gpurun_out/bench_t$t.json'));print('c3 TAIL=$t', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'])"
done
for t in 1 0; do
  RUTV_GEMM_TAIL=$t timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c2_t$t.json 2>gpurun_out/bench_c2.err
  python -c "import json;d=json.load(open('gpurun_out/bench_c2_t$t.json'));print('c2 TAIL=$t', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'])"
done

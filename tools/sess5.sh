mkdir -p gpurun_out
for v in small wide_skinny small wide_skinny; do
  echo "== $v" >> gpurun_out/cfg_ab.log
  RUTV_GEMM_CFG=$v timeout 300 python tools/bench_kernels.py gemm >> gpurun_out/cfg_ab.log 2>&1
  RUTV_GEMM_CFG=$v timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('bench', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'])" >> gpurun_out/cfg_ab.log
done
cut -c1-160 gpurun_out/cfg_ab.log

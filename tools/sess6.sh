mkdir -p gpurun_out
for v in default s4 default s4; do
  if [ $v = s4 ]; then export RUTV_LIB=build_var/libs4.so; else unset RUTV_LIB; fi
  echo "== $v" >> gpurun_out/s4_ab.log
  timeout 300 python tools/bench_kernels.py gemm 2>&1 | cut -c1-150 >> gpurun_out/s4_ab.log
  timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('bench', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'])" >> gpurun_out/s4_ab.log
done
cat gpurun_out/s4_ab.log

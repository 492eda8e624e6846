# CPQR variant A/B (variants built by hand into tools/cp<X>_bin with RUTV_NVCC_EXTRA)
for v in $CP_VARIANTS; do
  for c in c2 c3; do
    RUTV_LIB=tools/cp${v}_bin timeout 300 python bench.py --algo hqrrp --config $c --steps 1 --warmup 1 --no-uv 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('variant $v', '$c', d['ms_per_step'], d['kernels_last_step']['cpqr_sketch'])"
  done
done

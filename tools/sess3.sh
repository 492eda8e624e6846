mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_host.py tests/test_gpu_kernels.py -q -x > gpurun_out/t3.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t3.log
python tools/host_model_check.py > gpurun_out/hm3.log 2>&1; cat gpurun_out/hm3.log
for d in 2 4; do
RUTV_HOST_PREFETCH=$d timeout 1200 python bench.py --config c5 --mode host --no-uv --cache-gib 16 --steps 1 --warmup 0 > gpurun_out/host_c5_16g_pf$d.json 2> gpurun_out/host_c5.err; echo "c5 belady pf=$d rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/host_c5_16g_pf$d.json')); t=d['table1']; print(d['value'], {k: t[k] for k in ('real_time_s','computational_time_s','real_over_comp','h2d_bytes','d2h_bytes','h2d_GBps')})"
done
timeout 900 python tools/bench_kernels.py qr > gpurun_out/k3.log 2>&1; cut -c1-200 gpurun_out/k3.log

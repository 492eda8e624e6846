mkdir -p gpurun_out
RUTV_VSTREAM=0 RUTV_PROF_DUMP=gpurun_out/prof_dump_serial.txt timeout 900 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/pd_serial.json 2>&1
python tools/gemm_dist.py gpurun_out/prof_dump_serial.txt
python -c "import json; d=json.load(open('gpurun_out/pd_serial.json')); print('serial V stream:', d['value'], d['ms_per_step'])"
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b8.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/b8.json')); print(d['value'], d['roofline'])"

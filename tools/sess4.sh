# round-2 profiles: per-launch breakdown, ncu launch list + dominant-kernel capture, config benches
mkdir -p gpurun_out
RUTV_PROF_DUMP=gpurun_out/prof_dump_r02.txt timeout 900 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/pd.json 2>&1
python tools/gemm_dist.py gpurun_out/prof_dump_r02.txt > gpurun_out/step_breakdown_r02.txt; cat gpurun_out/step_breakdown_r02.txt
timeout 900 python bench.py --config c1 --no-cpu-baseline > gpurun_out/bench_c1.json 2>/dev/null; echo "c1 rc=$?"; cut -c1-400 gpurun_out/bench_c1.json
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2>/dev/null; echo "c4 rc=$?"; cut -c1-400 gpurun_out/bench_c4.json
timeout 1500 python bench.py --config c5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_c5.json 2>/dev/null; echo "c5 rc=$?"; cut -c1-400 gpurun_out/bench_c5.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --sharded --no-cpu-baseline > gpurun_out/bench_sharded1.json 2> gpurun_out/bench_sharded1.err; echo "sharded rc=$?"; cut -c1-400 gpurun_out/bench_sharded1.json
bash tools/gpu_session.sh ncu_launches ncu_full
timeout 1500 python bench.py --config c5 --mode host --no-uv --cache-gib 24 --steps 1 --warmup 0 > gpurun_out/host_c5_24g.json 2>/dev/null; echo "c5 host 24g rc=$?"; cut -c1-300 gpurun_out/host_c5_24g.json

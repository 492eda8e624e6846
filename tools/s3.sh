python paper_2002_06960_b200/build.py > /dev/null && \
timeout 300 python tools/bench_kernels.py gemm > gpurun_out/kernels3.log 2>&1; echo "kernels rc=$?"; cat gpurun_out/kernels3.log
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider > gpurun_out/pytest_k.log 2>&1; echo "pytest kernels rc=$?"; tail -3 gpurun_out/pytest_k.log
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo "bench rc=$?"; cat gpurun_out/bench3.json | head -c 1500

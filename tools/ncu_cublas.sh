python paper_2002_06960_b200/build.py > /dev/null || exit 1
timeout 300 python tools/bench_kernels.py cublas > gpurun_out/cublas_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --launch-skip 6 --launch-count 1 -o gpurun_out/prof_cublas_rankb python tools/bench_kernels.py cublas > gpurun_out/ncu_cublas.log 2>&1; echo "rc=$?"
timeout 900 ncu --set full --clock-control none --launch-skip 0 --launch-count 1 -o gpurun_out/prof_cublas_skinny python tools/bench_kernels.py cublas >> gpurun_out/ncu_cublas.log 2>&1; echo "rc=$?"

python paper_2002_06960_b200/build.py > /dev/null || exit 1
CMD="python tools/bench_kernels.py qr"
timeout 300 $CMD > gpurun_out/qr_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qr_leaf --launch-skip 3 --launch-count 1 -o gpurun_out/prof_qrleaf $CMD > gpurun_out/ncu_qr.log 2>&1; echo "rc=$?"

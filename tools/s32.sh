free -g | head -2; nproc
python paper_2002_06960_b200/build.py > /dev/null || exit 1
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-profile"
timeout 900 $CMD > gpurun_out/plain_qr.log 2>&1 || { echo "plain failed"; exit 1; }
# the first QR leaf of the c3 step (S4 of step 0: h = 16384, 32 columns, cooperative grid)
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:qr_leaf_kernel \
  --launch-skip 0 --launch-count 1 -o gpurun_out/prof_qrleaf $CMD > gpurun_out/ncu_qr.log 2>&1; echo "ncu qr rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:cpqr_sketch \
  --launch-skip 0 --launch-count 1 -o gpurun_out/prof_cpqr python bench.py --algo hqrrp --steps 1 --warmup 0 --no-uv > gpurun_out/ncu_cpqr.log 2>&1; echo "ncu cpqr rc=$?"

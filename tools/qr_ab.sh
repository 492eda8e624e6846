python paper_2002_06960_b200/build.py > /dev/null || exit 1
for r in 1 2 4; do echo "== RUTV_LEAF_R=$r"; RUTV_LEAF_R=$r timeout 300 python tools/bench_kernels.py qr; done

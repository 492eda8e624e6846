python paper_2002_06960_b200/build.py > /dev/null || exit 1
rm -f /tmp/p.txt
RUTV_PROF_DUMP=/tmp/p.txt timeout 600 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/gemm_dist.py /tmp/p.txt
cp /tmp/p.txt gpurun_out/prof_dump.txt

#!/bin/bash
# One gpurun session: tests, bench, ncu launch list, ncu full capture of the top kernel.
# Usage (from repo root, under gpurun): bash tools/gpu_session.sh [smoke] [tests] [bench] [bench_c2] [kernels]
#   [bench_variants] [host] [hqrrp] [ncu_launches] [ncu_full]   (ncu_full picks the longest DGEMM of ncu_launches)
set -u
mkdir -p gpurun_out
for stage in "$@"; do
  case "$stage" in
    tests)
      timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider --durations=10 \
        > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log ;;
    smoke)
      python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log ;;
    bench)
      timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err ;;
    kernels)
      for v in "RUTV_GEMM_PERSIST=1 RUTV_GEMM_SCHED=1" "RUTV_GEMM_PERSIST=1 RUTV_GEMM_SCHED=0" "RUTV_GEMM_PERSIST=0"; do
        echo "== $v" >> gpurun_out/kernels.log
        env $v timeout 600 python tools/bench_kernels.py gemm gemmdiag >> gpurun_out/kernels.log 2>&1
      done
      timeout 600 python tools/bench_kernels.py qr svd >> gpurun_out/kernels.log 2>&1
      echo "kernels rc=$?"; tail -40 gpurun_out/kernels.log ;;
    bench_variants)
      for v in "RUTV_FUSE_LEFT=1" "RUTV_FUSE_LEFT=0" "RUTV_GEMM_PERSIST=0" "RUTV_GEMM_SCHED=0"; do
        env $v timeout 900 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_var.json 2>>gpurun_out/bench_var.err
        echo "$v $(python -c "import json;d=json.load(open('gpurun_out/bench_var.json'));print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['other_kernels'])")" | tee -a gpurun_out/bench_variants.log
      done ;;
    bench_c2)
      timeout 900 python bench.py --config c2 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench c2 rc=$?"; cat gpurun_out/bench_c2.json ;;
    ncu_launches)
      # every librandutv launch of one c3 step (ncu costs ~40 ms per launch; a step has ~13.7k)
      CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-profile --no-graph"
      timeout 900 $CMD > gpurun_out/plain.log 2>&1 && \
      timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base mangled -k regex:4rutv \
        --csv --log-file gpurun_out/launches.csv $CMD \
        > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"; tail -3 gpurun_out/ncu_launches.log ;;
    ncu_full)
      # the dominant kernel: the longest DGEMM launch of the launch list above (c3: the fused rank-2b update)
      CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-profile --no-graph"
      IDX=$(python - <<'PY'
import csv
rows = [r for r in csv.DictReader(l for l in open("gpurun_out/launches.csv") if l.startswith('"'))]
g = [r for r in rows if "dgemm_kernel" in r["Kernel Name"] and r["Metric Name"] == "gpu__time_duration.sum"]
print(max(range(len(g)), key=lambda i: float(g[i]["Metric Value"].replace(",", ""))))
PY
)
      timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
        -k regex:dgemm_kernel --launch-skip "$IDX" --launch-count 1 -o gpurun_out/prof_dominant $CMD \
        > gpurun_out/ncu_full.log 2>&1; echo "ncu full (dgemm launch $IDX) rc=$?"; tail -3 gpurun_out/ncu_full.log ;;
    host)
      # host-streamed randUTV (S12) and HQRRP_left on c3
      timeout 900 python bench.py --mode host --steps 1 --warmup 1 > gpurun_out/bench_host_c3.json 2>> gpurun_out/bench_host.err
      timeout 900 python bench.py --mode host --steps 1 --warmup 1 --no-uv > gpurun_out/bench_host_c3_tonly.json 2>> gpurun_out/bench_host.err
      timeout 900 python bench.py --algo hqrrp --mode host --steps 1 --warmup 0 > gpurun_out/bench_hqrrp_host_c3.json 2>> gpurun_out/bench_host.err
      echo "host rc=$?"; cut -c1-200 gpurun_out/bench_host_c3*.json gpurun_out/bench_hqrrp_host_c3.json ;;
    hqrrp)
      timeout 900 python bench.py --algo hqrrp --steps 2 --warmup 1 > gpurun_out/bench_hqrrp_c3.json 2>> gpurun_out/bench_hqrrp.err
      echo "hqrrp rc=$?"; cut -c1-300 gpurun_out/bench_hqrrp_c3.json ;;
  esac
done

#!/bin/bash
# One gpurun session: tests, bench, ncu launch list, ncu full capture of the top kernel.
# Usage (from repo root, under gpurun): bash tools/gpu_session.sh [smoke] [tests] [full] [bench] [bench_c2] [kernels]
#   [bench_variants] [host] [host_c5] [hqrrp] [configs] [breakdown] [env_ab] [trace] [gemm_shapes] [gemm_tail]
#   [ncu_launches] [ncu_full] [ncu_gemm] [ncu_leaf] [ncu_svd] [leaf_ab] [probe_host]
#   (ncu_full picks the longest DGEMM of ncu_launches)
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
    full)
      # every -m gpu test (with durations), the default bench, c2, the step kernels
      timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=25 > gpurun_out/pytest_gpu.log 2>&1
      echo "pytest rc=$?"; tail -40 gpurun_out/pytest_gpu.log
      timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cut -c1-1500 gpurun_out/bench.json
      timeout 900 python bench.py --config c2 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
      echo "bench c2 rc=$?"; cut -c1-600 gpurun_out/bench_c2.json
      timeout 300 python tools/bench_kernels.py qr svd > gpurun_out/k2.log 2>&1; cut -c1-200 gpurun_out/k2.log ;;
    probe_host)
      # the GPU box's host: cores, memory, numpy DGEMM rate (the oracle's speed)
      nproc; lscpu | head -20; free -g; df -h /tmp | tail -1
      python -c "import numpy as np,time;a=np.random.rand(4096,4096);a@a;t=time.time();a@a;print('numpy dgemm GF/s',2*4096**3/(time.time()-t)/1e9)" ;;
    leaf_ab)
      # QR leaf plans and Jacobi variants (bench_kernels qr / svd)
      for v in "RUTV_LEAF_MAXUNITS=5" "RUTV_LEAF_MAXUNITS=3" "RUTV_LEAF_R2_FROM=12289" "RUTV_LEAF_CLUSTER=0"; do
        echo "== $v" >> gpurun_out/leaf_ab.log; env $v timeout 300 python tools/bench_kernels.py qr >> gpurun_out/leaf_ab.log 2>&1
      done
      for v in "RUTV_JACOBI_CLUSTER=1" "RUTV_JACOBI_CLUSTER=0"; do
        echo "== $v" >> gpurun_out/leaf_ab.log; env $v timeout 300 python tools/bench_kernels.py svd >> gpurun_out/leaf_ab.log 2>&1
      done
      cut -c1-200 gpurun_out/leaf_ab.log ;;
    ncu_leaf)
      # ncu --set full of the QR leaf kernel at h = 16384 and 4096 (tools/leaf_probe.py)
      for h in 16384 4096; do
        timeout 600 ncu --set full --clock-control none --import-source on -k regex:qr_leaf --launch-skip 2 --launch-count 1 \
          -o gpurun_out/prof_leaf_$h python tools/leaf_probe.py $h > gpurun_out/ncu_leaf_$h.log 2>&1; echo "ncu leaf h=$h rc=$?"
      done ;;
    ncu_svd)
      # ncu --set full of the Jacobi SVD kernels at w = 256 (L2-staged) and 128 (cluster-resident)
      for w in 256 128; do
        timeout 600 ncu --set full --clock-control none --import-source on -k regex:jacobi_.*kernel --launch-skip 4 --launch-count 1 \
          -o gpurun_out/prof_svd_$w python tools/svd_probe.py $w > gpurun_out/ncu_svd_$w.log 2>&1; echo "ncu svd w=$w rc=$?"
      done ;;
    ncu_gemm)
      # ncu --set full of the skinny S2 product (launch 0) and the rank-b update (launch 18) of bench_kernels gemm
      CMD="python tools/bench_kernels.py gemm"
      timeout 300 $CMD > gpurun_out/ncu_gemm_plain.log 2>&1 || { echo "plain run failed"; continue; }
      for pr in "18 rankb" "0 skinny"; do set -- $pr
        timeout 900 ncu --set full --clock-control none --import-source on -k regex:dgemm_kernel --launch-skip $1 --launch-count 1 \
          -o gpurun_out/prof_$2 $CMD > gpurun_out/ncu_$2.log 2>&1; echo "ncu $2 rc=$?"
      done ;;
    breakdown)
      # per-launch step breakdown of c3 (V stream concurrent, then serialised) -> profiles/step_breakdown*_rNN.txt
      RUTV_PROF_DUMP=gpurun_out/prof_dump.txt timeout 900 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/pd.json 2>&1
      python tools/gemm_dist.py gpurun_out/prof_dump.txt > gpurun_out/step_breakdown.txt
      RUTV_VSTREAM=0 RUTV_PROF_DUMP=gpurun_out/prof_dump_serial.txt timeout 900 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/pd_serial.json 2>&1
      python tools/gemm_dist.py gpurun_out/prof_dump_serial.txt > gpurun_out/step_breakdown_serial.txt
      cat gpurun_out/step_breakdown.txt gpurun_out/step_breakdown_serial.txt ;;
    configs)
      # c1, c4, c5 and the one-rank sharded NCCL path (bench lines -> profiles/bench_rNN_*.json)
      timeout 900 python bench.py --config c1 --no-cpu-baseline > gpurun_out/bench_c1.json 2>/dev/null; echo "c1 rc=$?"; cut -c1-400 gpurun_out/bench_c1.json
      timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2>/dev/null; echo "c4 rc=$?"; cut -c1-400 gpurun_out/bench_c4.json
      timeout 1500 python bench.py --config c5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_c5.json 2>/dev/null; echo "c5 rc=$?"; cut -c1-400 gpurun_out/bench_c5.json
      timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
        bench.py --gpus 1 --sharded --no-cpu-baseline > gpurun_out/bench_sharded1.json 2> gpurun_out/bench_sharded1.err
      echo "sharded rc=$?"; cut -c1-400 gpurun_out/bench_sharded1.json ;;
    host_c5)
      # M7's design point: c5 T only from host memory, 16 GiB cache, Belady vs LRU, and the traffic model check
      python tools/host_model_check.py > gpurun_out/hm.log 2>&1; RUTV_HOST_EVICT=lru python tools/host_model_check.py >> gpurun_out/hm.log 2>&1; cat gpurun_out/hm.log
      for ev in belady lru; do
        RUTV_HOST_EVICT=$ev timeout 1500 python bench.py --config c5 --mode host --no-uv --cache-gib 16 --steps 1 --warmup 0 \
          > gpurun_out/host_c5_16g_$ev.json 2>> gpurun_out/host_c5.err; echo "c5 host $ev rc=$?"; cut -c1-1500 gpurun_out/host_c5_16g_$ev.json
      done ;;
    env_ab)
      # A/B of a runtime knob on c3 and c2: ENV_AB="RUTV_X=1 RUTV_X=0" bash tools/gpu_session.sh env_ab
      for v in ${ENV_AB:-RUTV_UDEFER=1 RUTV_UDEFER=0}; do
        for c in c3 c2; do
          env $v timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('$v $c', d['value'], d['ms_per_step'], d['roofline']['achieved'])" | tee -a gpurun_out/env_ab.log
        done
      done ;;
    trace)
      RUTV_TRACE=gpurun_out/trace_c3.json timeout 600 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
      ls -la gpurun_out/trace_c3.json ;;
    gemm_tail)
      # tail-split DGEMM schedule A/B (round 2d): GEMM tests, c3 shape sweep, c3/c2 benches with RUTV_GEMM_TAIL=1/0
      timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -k "dgemm" -p no:cacheprovider > gpurun_out/pt_gemm.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pt_gemm.log
      STEPS=${STEPS:-0,16,32,40,44,48,52,56,60} timeout 400 python tools/gemm_shapes.py > gpurun_out/shapes_tail1.log 2>&1
      RUTV_GEMM_TAIL=0 STEPS=${STEPS:-0,16,32,40,44,48,52,56,60} timeout 400 python tools/gemm_shapes.py > gpurun_out/shapes_tail0.log 2>&1
      for t in 1 0 1 0; do
        RUTV_GEMM_TAIL=$t timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_t$t.json 2>gpurun_out/bench_t$t.err
        python -c "import json;d=json.load(open('gpurun_out/bench_t$t.json'));print('c3 TAIL=$t', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'])"
      done
      for t in 1 0; do
        RUTV_GEMM_TAIL=$t timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c2_t$t.json 2>gpurun_out/bench_c2.err
        python -c "import json;d=json.load(open('gpurun_out/bench_c2_t$t.json'));print('c2 TAIL=$t', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'])"
      done ;;
    gemm_shapes)
      timeout 600 python tools/gemm_shapes.py > gpurun_out/gemm_shapes.log 2>&1; echo "gemm_shapes rc=$?"; cat gpurun_out/gemm_shapes.log ;;
    hqrrp)
      timeout 900 python bench.py --algo hqrrp --steps 2 --warmup 1 > gpurun_out/bench_hqrrp_c3.json 2>> gpurun_out/bench_hqrrp.err
      echo "hqrrp rc=$?"; cut -c1-300 gpurun_out/bench_hqrrp_c3.json ;;
  esac
done

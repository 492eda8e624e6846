# round-end evidence: full GPU suite, default bench, ncu launch list + full capture of the longest DGEMM
mkdir -p gpurun_out
python paper_2002_06960_b200/build.py > /dev/null || exit 1
timeout 2000 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | grep -v "^  " | tail -6
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-profile"
timeout 3000 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:rutv \
  --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
IDX=$(python - <<'PY'
import csv
rows = [r for r in csv.DictReader(l for l in open("gpurun_out/launches.csv") if l.startswith('"'))]
g = [r for r in rows if "dgemm_kernel" in r["Kernel Name"] and r["Metric Name"] == "gpu__time_duration.sum"]
best = max(range(len(g)), key=lambda i: float(g[i]["Metric Value"].replace(",", "")))
print(best)
PY
)
echo "longest dgemm launch index $IDX"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dgemm_kernel --launch-skip $IDX --launch-count 1 \
  -o gpurun_out/prof_dominant $CMD > gpurun_out/ncu_dom.log 2>&1; echo "ncu full rc=$?"

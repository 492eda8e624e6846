#!/bin/bash
# ncu --set full of the QR leaf kernel at h = 16384 (cluster R=2,S=2) and 4096 (cluster R=1)
mkdir -p gpurun_out
for h in 16384 4096; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:qr_leaf --launch-skip 2 --launch-count 1 \
    -o gpurun_out/prof_leaf_$h python tools/leaf_probe.py $h > gpurun_out/ncu_leaf_$h.log 2>&1
  echo "h=$h rc=$?"
done

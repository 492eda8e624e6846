for c in 0 1; do echo "cfg $c"; RUTV_GEMM_CFG=$c python tools/bench_kernels.py gemm; done
python tools/bench_kernels.py qr

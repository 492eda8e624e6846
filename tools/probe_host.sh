nproc; lscpu | head -20; free -g; nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv
python - <<'PY'
import numpy as np, time, os
np.show_config()
a=np.random.rand(4096,4096); b=np.random.rand(4096,4096)
a@b; t=time.time(); 
for _ in range(3): a@b
dt=(time.time()-t)/3; print("numpy dgemm 4096^3 GF/s", 2*4096**3/dt/1e9)
a=np.random.rand(65536,512); b=np.random.rand(65536,2048)
t=time.time(); a.T@b; dt=time.time()-t; print("numpy TN 512x2048 K=65536 GF/s", 2*65536*512*2048/dt/1e9)
PY

mkdir -p gpurun_out
PK_DEBUG_ASSIGN=1 timeout 600 python tools/insert_breakdown.py > gpurun_out/ins_sim.txt 2>&1; grep "pk_assign host" gpurun_out/ins_sim.txt | tail -2; tail -1 gpurun_out/ins_sim.txt
python - <<'PY'
import time, numpy as np, ctypes, sys, os
sys.path.insert(0, os.getcwd())
from paper_2602_21477_b200 import _native as N
N.load()
import torch
lib = N.lib()
# bare round trip costs on this box
x = torch.zeros(1, device="cuda"); torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(2000): x.add_(1)
torch.cuda.synchronize(); print("torch launch us", (time.perf_counter()-t)/2000*1e6)
t = time.perf_counter()
for _ in range(2000):
    x.add_(1); torch.cuda.synchronize()
print("launch+sync us", (time.perf_counter()-t)/2000*1e6)
PY

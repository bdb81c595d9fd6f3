"""Run a few stage-1 / approx calls of one config (profiling target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_04165_b200 as atk
from tools.quick_time import cfgs
name = sys.argv[1]; reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
rows, n, B, kp, k, dt = cfgs[name]
dev = torch.device("cuda:0")
x = torch.randn(rows, n, device=dev)
if dt == "bf16":
    x = x.to(torch.bfloat16)
p = atk.AlgoParams(n, B, kp, k)
st = torch.zeros(1, dtype=torch.int32, device=dev)
for _ in range(reps):
    atk.approx_top_k_device(x, p, status=st)
torch.cuda.synchronize()
atk.check_status(st)
print("ok")

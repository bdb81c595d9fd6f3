"""Sweep the stage-1 segment count (ATKG_SEGS) for one config (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_04165_b200 as atk
from tools.quick_time import timeit, cfgs

name = sys.argv[1]
segs_list = [int(s) for s in sys.argv[2].split(",")]
rows, n, B, kp, k, dt = cfgs[name]
dev = torch.device("cuda:0")
x = torch.randn(rows, n, device=dev)
if dt == "bf16":
    x = x.to(torch.bfloat16)
esz = 2 if dt == "bf16" else 4
p = atk.AlgoParams(n, B, kp, k)
st = torch.zeros(1, dtype=torch.int32, device=dev)
ref = None
for sg in segs_list:
    os.environ["ATKG_SEGS"] = str(sg)
    t = timeit(lambda: atk.stage1_device(x, p, status=st))
    g = atk.stage1_device(x, p, status=st)
    if ref is None:
        ref = g
    same = torch.equal(ref[0], g[0]) and torch.equal(ref[1], g[1])
    print(f"{name} segs={sg:5d}: stage1+merge {t*1e3:8.1f} us  {rows*n*esz/t/1e6:7.1f} GB/s  same={same}", flush=True)

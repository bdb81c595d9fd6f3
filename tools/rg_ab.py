import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import bench
import paper_2506_04165_b200 as atk
from tools.rg_time import timeit
cfg = bench.CONFIGS["C3"]
xb, _ = bench.make_rows(cfg, 0, cfg["rows"])
dev = torch.device("cuda:0")
x = torch.from_numpy(np.ascontiguousarray(xb).view(np.int16)).to(dev).view(torch.bfloat16)
rows, n, k = x.shape[0], x.shape[1], 287
st = torch.zeros(1, dtype=torch.int32, device=dev)
out = (torch.empty(rows, k, device=dev), torch.empty(rows, k, dtype=torch.int32, device=dev))
p = atk.AlgoParams(n, 128, 4, k)
run = lambda: atk.approx_top_k_device(x, p, status=st, out=out)
def stats():
    with atk._lib.option("rowreg_probe", 9):
        out[1].zero_()
        for _ in range(50): run()
        torch.cuda.synchronize()
        return out[1].view(-1)[:7].tolist()
for rep in range(2):
    for mode, what in [(0, "per CTA (default)"), (1, "always robust"), (2, "running mean alone")]:
        with atk._lib.option("rowreg_robust", mode):
            t = timeit(run, iters=200)
            tp, msum, byp, mgs, a, b, rb = stats()
            print(f"{what:20s}: {t:6.1f} us, two-pass rows {tp} in 50 calls, mean M {msum/rows/50:.1f}, mean margin {mgs/rows/50:.1f}, robust rows {rb/50:.0f}", flush=True)

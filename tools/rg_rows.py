"""row_reg_kernel on the C3 row shape at several batch sizes: the planner's warp count against fixed ones
(development aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_04165_b200 as atk  # noqa: E402
from tools.rg_time import timeit  # noqa: E402

dev = torch.device("cuda:0")
n, k = 14336, 287
p = atk.AlgoParams(n, 128, 4, k)
st = torch.zeros(1, dtype=torch.int32, device=dev)
for rows in [512, 2048, 4096, 5000, 6000, 8192, 10000, 12288, 16384]:
    x = torch.randn(rows, n, device=dev).to(torch.bfloat16)
    out = (torch.empty(rows, k, device=dev), torch.empty(rows, k, dtype=torch.int32, device=dev))
    run = lambda: atk.approx_top_k_device(x, p, status=st, out=out)  # noqa: E731
    res = [f"auto {timeit(run, iters=30):6.1f}"]
    for w in [16, 20, 24, 29]:
        with atk._lib.option("rowreg_warps", w):
            res.append(f"w{w} {timeit(run, iters=30):6.1f}")
    print(f"rows={rows:6d}: " + "  ".join(res) + f"   ({rows * n * 2 / 1e3 / float(res[0].split()[1]) / 6552.3:.3f} of peak, auto)", flush=True)
    del x

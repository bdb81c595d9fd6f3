"""row_reg_kernel on rows whose scale changes from row to row (the prediction is a running mean of the
previous rows' levels): time and two-pass rows (development aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_04165_b200 as atk  # noqa: E402
from tools.rg_time import timeit  # noqa: E402

dev = torch.device("cuda:0")
rows, n, k = 8192, 14336, 287
p = atk.AlgoParams(n, 128, 4, k)
st = torch.zeros(1, dtype=torch.int32, device=dev)
out = (torch.empty(rows, k, device=dev), torch.empty(rows, k, dtype=torch.int32, device=dev))
base = torch.randn(rows, n, device=dev)
for name, spread in [("i.i.d.", 0.0), ("scale x 2^U(-0.03,0.03)", 0.03), ("scale x 2^U(-0.08,0.08)", 0.08), ("scale x 2^U(-0.25,0.25)", 0.25), ("scale x 2^U(-1,1)", 1.0), ("scale x 2^U(-3,3)", 3.0)]:
    sc = torch.exp2((torch.rand(rows, 1, device=dev) * 2 - 1) * spread)
    x = (base * sc).to(torch.bfloat16)
    run = lambda: atk.approx_top_k_device(x, p, status=st, out=out)  # noqa: E731
    t = timeit(run, iters=30)
    with atk._lib.option("rowreg_probe", 9):
        out[1].zero_()
        for _ in range(20):
            run()
        torch.cuda.synchronize()
        tp, msum, byp, mgs, vps, ves, rbs = out[1].view(-1)[:7].tolist()
    with atk._lib.option("rowreg", 0):
        t_old = timeit(run, iters=5)
    print(f"{name:28s}: {t:6.1f} us, two-pass rows {tp:5d} of 20 x {rows}, mean M {msum / rows / 20:6.1f}, robust rows {rbs / 20:6.0f}, by running mean {byp / 20:6.0f}, mean margin {mgs / rows / 20:5.1f} (sigmas {vps / rows / 320:4.1f} / {ves / rows / 320:4.1f} codes); row_resident {t_old:6.1f} us", flush=True)

"""row_reg_kernel on the bench's own C3 batch (seeded generator): time and path statistics per
prediction margin (development aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_04165_b200 as atk  # noqa: E402
from tools.rg_time import timeit  # noqa: E402

cfg = bench.CONFIGS["C3"]
xb, _ = bench.make_rows(cfg, 0, cfg["rows"])
dev = torch.device("cuda:0")
x = torch.from_numpy(np.ascontiguousarray(xb).view(np.int16)).to(dev).view(torch.bfloat16)
rows, n, k = x.shape[0], x.shape[1], 287
st = torch.zeros(1, dtype=torch.int32, device=dev)
out = (torch.empty(rows, k, device=dev), torch.empty(rows, k, dtype=torch.int32, device=dev))
p = atk.AlgoParams(n, 128, 4, k)
run = lambda: atk.approx_top_k_device(x, p, status=st, out=out)  # noqa: E731
for m in [8, 12]:
    with atk._lib.option("rowreg_margin", m):
        t = timeit(run, iters=100)
        with atk._lib.option("rowreg_probe", 9):
            out[1].zero_()
            for _ in range(20):
                run()
            torch.cuda.synchronize()
            tp, msum, byp, mgs, vps, ves = out[1].view(-1)[:6].tolist()
    print(f"margin={m}: {t:6.1f} us, two-pass rows {tp} in 20 calls, mean M {msum / rows / 20:.1f}, by running mean {byp / 20:.0f}, mean margin {mgs / rows / 20:.1f} (sigmas {vps / rows / 320:.1f} / {ves / rows / 320:.1f} codes)", flush=True)

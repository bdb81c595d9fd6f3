"""C2-shaped rows (fp32, n = 262144, K = 64, K' = 2, B = 128) at several row counts: how much of the
stream kernel's time is per-piece overhead (development aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_04165_b200 as atk  # noqa: E402
from tools.c2_time import timeit  # noqa: E402

dev = torch.device("cuda:0")
n, B, kp, k = 262144, 128, 2, 64
for rows in [148, 256, 296, 444, 512, 592, 1024]:
    x = torch.randn(rows, n, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    out = (torch.empty(rows, k, device=dev), torch.empty(rows, k, dtype=torch.int32, device=dev))
    p = atk.AlgoParams(n, B, kp, k)
    t = timeit(lambda: atk.approx_top_k_device(x, p, status=st, out=out), iters=100)
    atk.check_status(st)
    gbs = rows * n * 4 / (t * 1e-6) / 1e9
    print(f"rows={rows:5d}: {t:8.2f} us  {gbs:7.1f} GB/s  {gbs / 6552.3:.3f} of peak", flush=True)
    del x
    torch.cuda.empty_cache()

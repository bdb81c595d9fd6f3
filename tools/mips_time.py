"""Times the fp32 MIPS pipeline at the reference's full-scale test config
(test_mips.cpp:330-383: 1,000,448 x 128 database, 1024 queries, K=1024, B=1024,
K'=4) on the device, against the reference's mips_fused on a query sample."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_04165_b200 as atk  # noqa: E402
from paper_2506_04165_b200.mips import mips_top_k_device, score_block_device  # noqa: E402
from oracle import pyoracle as O  # noqa: E402

rows, d, nq, nb, kp, k = 1000448, 128, 1024, 1024, 4, 1024
rng = np.random.default_rng(71)
db = rng.standard_normal((rows, d)).astype(np.float32)
q = np.random.default_rng(72).standard_normal((nq, d)).astype(np.float32)
p = atk.AlgoParams(n=rows, num_buckets=nb, local_k=kp, global_k=k)
dev = torch.device("cuda")
tdb, tq = torch.from_numpy(db).to(dev), torch.from_numpy(q).to(dev)
for _ in range(2):
    v, i = mips_top_k_device(tq, tdb, p)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
steps = 5
e0.record()
for _ in range(steps):
    v, i = mips_top_k_device(tq, tdb, p)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
out = torch.empty((nq, rows), dtype=torch.float32, device=dev)
score_block_device(tq, tdb, rows, out=out)
torch.cuda.synchronize()
e0.record()
for _ in range(steps):
    score_block_device(tq, tdb, rows, out=out)
e1.record()
torch.cuda.synchronize()
sms = e0.elapsed_time(e1) / steps
flop = 2.0 * nq * rows * d
print(f"device: {ms:.2f} ms per 1024-query batch ({nq / ms * 1e3:.0f} queries/s); "
      f"score kernel {sms:.2f} ms = {flop / sms / 1e9:.1f} TFLOP/s fp32 (mul+add unfused, reference order)")
sample = 16
threads = os.cpu_count()
t = time.perf_counter()
rv, ri = O.ref().mips_fused(db, q[:sample], nb, kp, k, threads=threads)
ref_s = time.perf_counter() - t
print(f"reference mips_fused, {sample} queries, {threads} threads: {ref_s:.2f} s "
      f"({sample / ref_s:.1f} queries/s)")
vv, ii = v[:sample].cpu().numpy(), i[:sample].cpu().numpy().astype(np.uint32)
print("parity on the sample:", np.array_equal(vv.view(np.uint32), rv.view(np.uint32)) and np.array_equal(ii, ri))

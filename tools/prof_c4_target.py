"""A few fused GEMM + top-k calls on the C4 shape (profiling target)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2506_04165_b200 as atk  # noqa: E402
from paper_2506_04165_b200 import topk as T  # noqa: E402

m, kd, n = 8192, 3584, 14336
dev = torch.device("cuda:0")
g = torch.Generator(device="cpu").manual_seed(0)
x = torch.randn((m, kd), generator=g).to(torch.bfloat16).to(dev)
w = (0.02 * torch.randn((n, kd), generator=g)).to(torch.bfloat16).to(dev)
p = atk.AlgoParams(n, 128, 4, 287)
st = torch.zeros(1, dtype=torch.int32, device=dev)
out = (torch.empty((m, 287), dtype=torch.float32, device=dev), torch.empty((m, 287), dtype=torch.int32, device=dev))
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    T.fused_gemm_top_k_device(x, w, p, status=st, out=out)
torch.cuda.synchronize()
atk.check_status(st)
print("ok")

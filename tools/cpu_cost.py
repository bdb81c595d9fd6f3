"""Host cost per approx_top_k_device call vs device time (development aid)."""
import ctypes as C
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_04165_b200 as atk
from paper_2506_04165_b200 import topk as T
from paper_2506_04165_b200._lib import lib
x = torch.randn(256, 262144, device="cuda")
p = atk.AlgoParams(262144, 128, 2, 64)
st = torch.zeros(1, dtype=torch.int32, device="cuda")
out = (torch.empty(256, 64, device="cuda"), torch.empty(256, 64, dtype=torch.int32, device="cuda"))
for _ in range(20):
    atk.approx_top_k_device(x, p, status=st, out=out)
torch.cuda.synchronize()
N = 2000
def bench(name, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(N):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{name:28s} host {1e6*(t1-t0)/N:6.1f} us/call, wall {1e6*(t2-t0)/N:6.1f} us/call", flush=True)
bench("approx_top_k_device", lambda: atk.approx_top_k_device(x, p, status=st, out=out))
pc = p.c()
ws = T.workspace(1, x.device)
sp = torch.cuda.current_stream().cuda_stream
args = (1, x.data_ptr(), 256, C.byref(pc), out[0].data_ptr(), out[1].data_ptr(), ws.data_ptr(), ws.numel(), st.data_ptr(), sp)
bench("ctypes atkg_approx_top_k", lambda: lib.atkg_approx_top_k(*args))
bench("current_stream", lambda: torch.cuda.current_stream(x.device).cuda_stream)
os.environ["ATKG_NO_PDL"] = "1"
bench("ctypes, no PDL", lambda: lib.atkg_approx_top_k(*args))

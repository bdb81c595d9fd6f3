"""Ad-hoc device timing of the hot path per config (development aid)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2506_04165_b200 as atk
from paper_2506_04165_b200 import data

def timeit(fn, iters=20, warm=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters

cfgs = {
 "C1": (16, 32768, 512, 4, 128, "f32"),
 "C2": (256, 262144, 128, 2, 64, "f32"),
 "C3": (8192, 14336, 128, 4, 287, "bf16"),
 "C3k1": (8192, 14336, 3584, 1, 287, "bf16"),
 "C3k8": (8192, 14336, 128, 8, 287, "bf16"),
 "C3k2": (8192, 14336, 512, 2, 287, "bf16"),
 "C3r99": (8192, 14336, 256, 4, 287, "bf16"),
 "C5": (1, 1 << 30, 256, 8, 1024, "f32"),
}
def main():
  which = sys.argv[1:] or list(cfgs)
  for name in which:
    _one(name)

def _one(name):
    rows, n, B, kp, k, dt = cfgs[name]
    dev = torch.device("cuda:0")
    if dt == "f32":
        x = torch.randn(rows, n, device=dev)
        esz = 4
    else:
        x = torch.randn(rows, n, device=dev).to(torch.bfloat16)
        esz = 2
    p = atk.AlgoParams(n, B, kp, k)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    out = (torch.empty(rows, k, device=dev), torch.empty(rows, k, dtype=torch.int32, device=dev))
    grid = (torch.empty(rows, kp*B, device=dev), torch.empty(rows, kp*B, dtype=torch.int32, device=dev))
    t_all = timeit(lambda: atk.approx_top_k_device(x, p, status=st, out=out))
    t_s1 = timeit(lambda: atk.stage1_device(x, p, status=st))
    byts = rows * n * esz
    print(f"{name}: approx {t_all*1e3:8.1f} us ({byts/t_all/1e6:7.1f} GB/s, {rows*n/t_all/1e6:7.2f} Gelem/s)  stage1+merge {t_s1*1e3:8.1f} us ({byts/t_s1/1e6:7.1f} GB/s)", flush=True)
    atk.check_status(st)
    del x
    torch.cuda.empty_cache()

if __name__ == "__main__":
    main()

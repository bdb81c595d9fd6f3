"""Times the C4 paths on the GPU: plain tcgen05 GEMM, fused GEMM + top-k,
torch bf16 matmul (cuBLAS) for comparison."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2506_04165_b200 as atk  # noqa: E402
from paper_2506_04165_b200 import topk as T  # noqa: E402


def timeit(fn, iters=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def main():
    m, kd, n = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (8192, 3584, 14336)))
    dev = torch.device("cuda:0")
    g = torch.Generator(device="cpu").manual_seed(0)
    x = torch.randn((m, kd), generator=g).to(torch.bfloat16).to(dev)
    w = (0.02 * torch.randn((n, kd), generator=g)).to(torch.bfloat16).to(dev)
    flop = 2.0 * m * kd * n
    out = torch.empty((m, n), dtype=torch.float32, device=dev)
    t0 = time.time()
    T.gemm_bf16_device(x, w, out)
    torch.cuda.synchronize()
    print(f"first plain call {time.time() - t0:.2f}s", flush=True)
    ms = timeit(lambda: T.gemm_bf16_device(x, w, out))
    print(f"plain tcgen05 gemm  {ms * 1e3:8.1f} us  {flop / ms / 1e9:7.1f} TFLOP/s", flush=True)
    ms = timeit(lambda: torch.matmul(x, w.T))
    print(f"torch bf16 matmul   {ms * 1e3:8.1f} us  {flop / ms / 1e9:7.1f} TFLOP/s", flush=True)
    p = atk.AlgoParams(n, 128, 4, 287)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    vals = torch.empty((m, 287), dtype=torch.float32, device=dev)
    idx = torch.empty((m, 287), dtype=torch.int32, device=dev)
    T.fused_gemm_top_k_device(x, w, p, status=st, out=(vals, idx))
    torch.cuda.synchronize()
    ms = timeit(lambda: T.fused_gemm_top_k_device(x, w, p, status=st, out=(vals, idx)))
    print(f"fused gemm+top-k    {ms * 1e3:8.1f} us  {flop / ms / 1e9:7.1f} TFLOP/s", flush=True)
    atk.check_status(st)
    cv = torch.randn((m, 512), device=dev)
    ci = torch.arange(m * 512, device=dev, dtype=torch.int32).view(m, 512) % 14336
    ms = timeit(lambda: atk.select_candidates_device(cv, ci, 287))
    print(f"stage 2 [{m}, 512] -> 287 {ms * 1e3:8.1f} us", flush=True)
    lib = T.lib
    import ctypes as C
    lib.atkg_profile_begin()
    for _ in range(10):
        T.fused_gemm_top_k_device(x, w, p, status=st, out=(vals, idx))
    tot, n_l = C.c_double(), C.c_uint64()
    lib.atkg_profile_end(C.byref(tot), C.byref(n_l))
    kms = tot.value / max(1, n_l.value)
    print(f"  fused kernel alone {kms * 1e3:8.1f} us  {flop / kms / 1e9:7.1f} TFLOP/s", flush=True)


if __name__ == "__main__":
    main()

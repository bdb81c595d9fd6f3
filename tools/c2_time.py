"""Device timing of approx_top_k on C2 (fp32 [256, 262144], K=64, K'=2,
B=128) under stream-kernel tuning options (development aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_04165_b200 as atk  # noqa: E402


def timeit(fn, iters=200, warm=10):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3


def main():
    rows, n, B, kp, k = 256, 262144, 128, 2, 64
    if len(sys.argv) > 1 and sys.argv[1] == "C5":
        rows, n, B, kp, k = 1, 1 << 30, 256, 8, 1024
    dev = torch.device("cuda:0")
    x = torch.randn(rows, n, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    out = (torch.empty(rows, k, device=dev), torch.empty(rows, k, dtype=torch.int32, device=dev))
    p = atk.AlgoParams(n, B, kp, k)
    variants = [{}]
    for a in sys.argv[1:]:
        if "=" in a:
            variants.append(dict(kv.split(":") for kv in a.split(",")) if ":" in a else {})
    for v in [dict(x.split("=") for x in a.split(",")) for a in sys.argv[1:] if "=" in a] or [{}]:
        for name, val in v.items():
            atk._lib.set_option(name, int(val))
        t = timeit(lambda: atk.approx_top_k_device(x, p, status=st, out=out))
        atk.check_status(st)
        gbs = rows * n * 4 / (t * 1e-6) / 1e9
        print(f"{v or 'default'}: {t:7.2f} us  {gbs:7.1f} GB/s  {gbs / 6533.5:.3f}", flush=True)
        for name in v:
            atk._lib.set_option(name, None)


if __name__ == "__main__":
    main()

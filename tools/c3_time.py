"""Device timing of approx_top_k on the C3 shape and its K' sweep, the
short-row kernel against the previous row kernels (option no_short=1).
Development aid: CUDA events on the current stream, inputs > L2."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_04165_b200 as atk  # noqa: E402

SWEEP = [(4, 128), (1, 3584), (2, 512), (8, 128), (1, 7168), (2, 1024), (4, 256)]


def timeit(fn, iters=50, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3  # us


def main():
    rows, n, k = 8192, 14336, 287
    dev = torch.device("cuda:0")
    x = torch.randn(rows, n, device=dev).to(torch.bfloat16)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    out = (torch.empty(rows, k, device=dev), torch.empty(rows, k, dtype=torch.int32, device=dev))
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    new_only = "--new-only" in sys.argv
    which = [tuple(map(int, a.split("/"))) for a in args] or SWEEP
    atk._lib.set_option("short", 1)  # the short-row kernel (opt-in while under development)
    for kp, b in which:
        p = atk.AlgoParams(n, b, kp, k)
        t_new = timeit(lambda: atk.approx_top_k_device(x, p, status=st, out=out))
        if "--probe" in sys.argv:
            for pr, what in [(1, "row pipeline alone"), (2, "+ pass 1 + select"), (3, "+ pass 2"), (4, "+ collect")]:
                with atk._lib.option("short_probe", pr):
                    t_probe = timeit(lambda: atk.approx_top_k_device(x, p, status=st, out=out))
                print(f"K'={kp} B={b}: {what:22s} {t_probe:7.1f} us", flush=True)
        t_old = float("nan")
        if not new_only:
            with atk._lib.option("short", 0):
                t_old = timeit(lambda: atk.approx_top_k_device(x, p, status=st, out=out), iters=10)
        atk.check_status(st)
        gbs = rows * n * 2 / (t_new * 1e-6) / 1e9
        print(f"K'={kp} B={b}: short {t_new:7.1f} us ({gbs:6.0f} GB/s, {gbs / 6533.5:.3f} of peak)  "
              f"previous {t_old:7.1f} us", flush=True)


if __name__ == "__main__":
    main()

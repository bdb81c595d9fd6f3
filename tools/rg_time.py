"""Device timing of row_reg_kernel (csrc/rowreg.cuh) on the C3 shape: CTA
sizes, phase probes, the forced two-pass path and the previous default
(row_resident_kernel).  Development aid: CUDA events on the current stream,
inputs > L2."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_04165_b200 as atk  # noqa: E402

opt = atk._lib.option


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
    p = atk.AlgoParams(n, 128, 4, k)
    run = lambda: atk.approx_top_k_device(x, p, status=st, out=out)  # noqa: E731
    byts = rows * n * 2

    def line(what, t):
        print(f"{what:44s} {t:7.1f} us  {byts / t / 1e3:6.0f} GB/s  {byts / t / 1e3 / 6552.3:.3f} of peak", flush=True)

    warps = [int(a) for a in sys.argv[1:] if a.isdigit()] or [8, 12, 16, 20, 22]
    for w in warps:
        with opt("rowreg_warps", w):
            line(f"rowreg warps={w}", timeit(run))
            if "--probe" in sys.argv:
                for pr, what in [(1, "pass"), (2, "+ check/bisect")]:
                    with opt("rowreg_probe", pr):
                        line(f"  warps={w} probe {pr} ({what})", timeit(run))
            with opt("rowreg_force", 1):
                line(f"  warps={w} every row two-pass", timeit(run))
    with opt("rowreg_rt", 1):
        line("rowreg, run-time row length (S = 0 instantiation)", timeit(run))
    if "--shapes" in sys.argv:  # other row lengths (run-time S) against the previous kernels
        for n2, k2 in [(3584, 100), (4096, 82), (7168, 287), (8192, 164), (11008, 220), (12288, 246), (13824, 276), (16384, 300),
                       (28672, 287), (65536, 512)]:
            rows2 = max(1024, (235 << 20) // (2 * n2))
            x2 = torch.randn(rows2, n2, device=dev).to(torch.bfloat16)
            out2 = (torch.empty(rows2, k2, device=dev), torch.empty(rows2, k2, dtype=torch.int32, device=dev))
            p2 = atk.AlgoParams(n2, 128, 4, k2)
            run2 = lambda: atk.approx_top_k_device(x2, p2, status=st, out=out2)  # noqa: E731
            t_new = timeit(run2, iters=20)
            with opt("rowreg", 0):
                t_old = timeit(run2, iters=5)
            gb = rows2 * n2 * 2 / 1e3
            print(f"n={n2:6d} K={k2:3d} rows={rows2:6d}: rowreg {t_new:8.1f} us ({gb / t_new / 6552.3:.3f} of peak)  previous {t_old:8.1f} us", flush=True)
            del x2
    if "--stats" in sys.argv:
        for m in [1, 2, 3, 5, 8, 12]:
            with opt("rowreg_margin", m), opt("rowreg_probe", 9):
                out[1].zero_()
                run()
                torch.cuda.synchronize()
                tp, msum = out[1].view(-1)[:2].tolist()
                print(f"margin={m}: two-pass rows {tp} of {rows}, mean M {msum / rows:.1f}", flush=True)
    if "--sweep" in sys.argv:
        for rep in range(2):
            for m in [7, 8, 9, 10, 12, 14, 16, 20]:
                with opt("rowreg_margin", m), opt("rowreg_warps", 29):
                    line(f"margin={m} (warps=29, pass {rep})", timeit(run, iters=100))
    with opt("rowreg", 0):
        line("row_resident_kernel (previous default)", timeit(run, iters=20))
    atk.check_status(st)


if __name__ == "__main__":
    main()

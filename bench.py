"""Benchmark of the B200 two-stage approximate top-k hot path (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C2]

Workload (default; BASELINE.json configs[1], the config the metric is quoted on):
  C2 "LM-logit rows": fp32 [256, 262144] i.i.d. N(0,1) (seeded, synthetic),
  K=64, (B, K') from the host planner at expected recall 0.95 with
  K' in {1,2,4}  ->  K'=2, B=128.
A step = approx top-K (stage 1 + stage 2) over the whole batch.
Other configs (--config): C1 (oracle case), C3 (bf16 [8192, 14336]), C4 (the
fused tcgen05 GEMM + stage-1 epilogue: a step = scores + top-K of 8192 x 14336,
roofline against the bf16 tensor-core peak), C5 (one 2^30 row; at N > 1 the
row is sliced across ranks and the stage-1 summaries are all-gathered over
NCCL: fixed total work, "scaling": "strong").

  value  whole-job elements/s with inputs already resident in HBM (device
         API, CUDA events on the launching stream, max over ranks).  The
         input (268 MB per GPU) is larger than the 126 MB L2, so no flush is
         needed between steps.
  e2e    the same metric through the host-buffer C ABI
         (atkg_approx_top_k_host): pinned host rows -> device -> top-K ->
         host, every step.
  roofline  the stage-1 streaming kernel (the dominant kernel): algorithmic
         bytes per launch (rows*n*4 + rows*B*K'*8) / its live
         CUDA-event duration inside the timed steps, against the measured HBM
         copy bandwidth (MEASURED_PEAKS.json).
  cpu_baseline  the reference library (oracle/_ref: the unmodified atk core
         compiled from /root/reference) approx_top_k_batch with all host
         threads, on the same bytes, rank 0 at N=1.

N>1 (torchrun): C1-C4 -- every rank runs its own batch (rows sharded across
GPUs, no data-path collective), so per-GPU work is fixed: "scaling": "weak".
C5 -- one row, sliced: "scaling": "strong".
--impl reference runs the reference CPU implementation on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: rows, n, K, recall target, allowed K', dtype, seed key
    "C1": dict(rows=16, n=32768, k=128, fixed=(4, 512), dtype="f32", seed="C1",
               label="oracle fp32 [16, 32768], K=128, K'=4, B=512"),
    "C2": dict(rows=256, n=262144, k=64, target=0.95, kps=(1, 2, 4), dtype="f32", seed="C2",
               label="LM-logit rows fp32 [256, 262144], K=64, planner r=0.95 K' in {1,2,4}"),
    "C3": dict(rows=8192, n=14336, k=287, target=0.95, kps=(1, 2, 4, 8), dtype="bf16", seed="C3",
               label="FFN-activation top-2% bf16 [8192, 14336], K=287, planner r=0.95 K' in {1,2,4,8}"),
    "C4": dict(rows=8192, n=14336, kdim=3584, k=287, target=0.95, kps=(4,), dtype="bf16", seed="C4x",
               wseed="C4w", kind="gemm",
               label="fused FFN GEMM + approx top-K: x bf16 [8192, 3584] . W bf16 [3584, 14336], K=287, K'=4, "
                     "planner r=0.95"),
    "C5": dict(rows=1, n=1 << 30, k=1024, target=0.95, kps=(8,), dtype="f32", seed="C5", kind="giant",
               label="single giant row fp32 [1, 2^30], K=1024, K'=8, planner r=0.95"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def plan(cfg):
    import paper_2506_04165_b200 as atk
    if "fixed" in cfg:
        kp, b = cfg["fixed"]
        rec = atk.exact_expected_recall(atk.AlgoParams(cfg["n"], b, kp, cfg["k"])).value
        return kp, b, rec
    r = atk.select_parameters(atk.PlanRequest(cfg["n"], cfg["k"], cfg["target"], list(cfg["kps"]), 128, 0))
    return r.local_k, r.num_buckets, r.estimated_recall.value


def make_rows(cfg, rank):
    """Host rows (fp32, or bf16 bits + fp32 upcast) for this rank."""
    from paper_2506_04165_b200 import data
    seed = data.SEEDS[cfg["seed"]] + 1000 * rank
    if cfg["dtype"] == "bf16":
        bits, f = data.normal_bf16(seed, (cfg["rows"], cfg["n"]))
        return bits, f
    x = data.normal_f32(seed, (cfg["rows"], cfg["n"]))
    return x, x


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json, copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clock + throttle reasons sampled (NVML, every ~5 ms) in a background
    thread; summary() keeps the samples taken inside mark()..unmark()."""

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.window = [None, None]
        self.stop = False

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.maxc = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception as e:  # pragma: no cover
            self.nv = None
            self.err = str(e)
        return self

    def _run(self):
        nv = self.nv
        masks = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                 "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}
        while not self.stop:
            try:
                clk = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.rows.append((time.perf_counter(), clk, [k for k, m in masks.items() if rs & m]))
            except Exception:
                pass
            time.sleep(0.005)

    def mark(self):
        self.window[0] = time.perf_counter()

    def unmark(self):
        self.window[1] = time.perf_counter()

    def __exit__(self, *exc):
        self.stop = True
        if getattr(self, "t", None):
            self.t.join(timeout=1)

    def summary(self):
        if not self.nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled: " + getattr(self, "err", "")]}
        t0, t1 = self.window
        inside = [r for r in self.rows if t0 is not None and t1 is not None and t0 <= r[0] <= t1]
        note = "during the timed region"
        if not inside:  # timed region shorter than one sample period: nearest samples
            inside = sorted(self.rows, key=lambda r: abs(r[0] - (t0 or 0)))[:3]
            note = "nearest samples (timed region shorter than the 5 ms sampling period)"
        clk = [r[1] for r in inside]
        reasons = sorted({x for r in inside for x in r[2]})
        return {"sm_mhz": statistics.median(clk) if clk else None, "sm_max_mhz": self.maxc, "reasons": reasons,
                "samples": len(inside), "note": note}


def traffic_from_profiles(workload):
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(workload, {}).get("dram_bytes_per_launch")
    except Exception:
        return None



def ref_backend():
    from oracle import pyoracle as O
    if not O.ref_available():
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "ref"], capture_output=True)
    if O.ref_available():
        return O.ref(), "reference"
    return O.port(), "port"


def timed_calls(fn, steps, min_seconds, max_calls=50):
    times = []
    t_start = time.perf_counter()
    while len(times) < steps or (time.perf_counter() - t_start < min_seconds and len(times) < max_calls):
        t0 = time.perf_counter()
        fn()
        times.append(time.perf_counter() - t0)
    return times


def metric_name():
    return "approx top-K Gelem/s & HBM GB/s vs ~8 TB/s roofline at matched expected recall"


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------
class RowsWorkload:
    """C1/C2/C3: a batch of independent rows per rank (weak scaling)."""
    scaling = "weak"
    kernel = "stage1_flat_kernel"

    def __init__(self, args, cfg, kp, b, rec, world, rank):
        self.args, self.cfg, self.kp, self.b, self.rec = args, cfg, kp, b, rec
        self.world, self.rank = world, rank
        self.rows, self.n, self.k = cfg["rows"], cfg["n"], cfg["k"]
        self.esz = 2 if cfg["dtype"] == "bf16" else 4
        self.dtype = "bf16" if self.esz == 2 else "f32"

    def setup(self, dev):
        import torch
        import paper_2506_04165_b200 as atk
        self.torch, self.atk, self.dev = torch, atk, dev
        self.host, self.host_f32 = make_rows(self.cfg, self.rank)
        if self.esz == 2:
            self.x = torch.from_numpy(self.host.view(np.int16)).to(dev).view(torch.bfloat16)
        else:
            self.x = torch.from_numpy(self.host).to(dev)
        if self.cfg["n"] != self.n:
            raise AssertionError
        self.p = atk.AlgoParams(self.n, self.b, self.kp, self.k)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.out = (torch.empty(self.rows, self.k, device=dev),
                    torch.empty(self.rows, self.k, dtype=torch.int32, device=dev))

    def step(self):
        self.atk.approx_top_k_device(self.x, self.p, status=self.status, out=self.out)

    def check(self):
        self.atk.check_status(self.status)

    def elements(self):  # per rank per step
        return self.rows * self.n

    def hbm_bytes(self):
        return self.rows * self.n * self.esz

    def dominant_kernel(self):
        # the approx_top_k plan (csrc/atkg_api.cu): long rows take the threshold
        # stream (streamthr.cuh), rows that fit in shared memory the row-resident path
        if self.n >= 32768 and not os.environ.get("ATKG_NO_STREAMTHR"):
            return "st_stream_kernel (threshold stream; stage-1 pass)"
        if self.n * self.esz <= 64 * 1024:
            return "row_threshold_kernel" if self.kp >= 8 else "row_resident_kernel"
        return self.kernel

    def roofline(self, kern_ms, ms_step):
        peak, src = peaks()
        alg = self.rows * self.n * self.esz + self.rows * self.b * self.kp * 8
        ach = alg / (kern_ms * 1e-3) / 1e9
        return {"kernel": self.dominant_kernel(), "bound": "hbm", "achieved": round(ach, 1), "peak": peak,
                "peak_source": src, "unit": "GB/s", "frac": round(ach / peak, 4),
                "traffic": traffic_from_profiles(self.args.config), "alg_bytes_per_launch": alg,
                "launch_ms": round(kern_ms, 5), "share_of_step": round(kern_ms / ms_step, 4)}

    def recall(self):
        atk = self.atk
        _, ei = atk.exact_top_k_device(self.x, self.k)
        rs = [atk.measure_recall(atk.TopKResult(None, self.out[1][r].cpu().numpy().astype(np.uint32)),
                                 atk.TopKResult(None, ei[r].cpu().numpy().astype(np.uint32)))
              for r in range(self.rows)]
        return float(np.mean(rs))

    def e2e(self, steps, barrier):
        """Public API with host buffers: f32 through the drop-in C ABI
        (atkg_approx_top_k_host); bf16 (no reference host dtype) through the
        Python device API with pinned H2D / D2H copies inside the region."""
        import ctypes as C
        torch, atk = self.torch, self.atk
        from paper_2506_04165_b200._lib import lib
        rows, n, k = self.rows, self.n, self.k
        ov = torch.empty((rows, k), dtype=torch.float32).pin_memory()
        oi = torch.empty((rows, k), dtype=torch.int32).pin_memory()
        if self.esz == 4:
            pinned = torch.from_numpy(self.host_f32).pin_memory()
            prm = self.p.c()

            def one():
                atk._lib.check(lib.atkg_approx_top_k_host(pinned.data_ptr(), rows, C.byref(prm), ov.data_ptr(),
                                                          oi.data_ptr()))
            api = "atkg_approx_top_k_host (C ABI, pinned host buffers)"
        else:
            pinned = torch.from_numpy(self.host.view(np.int16)).pin_memory()
            xd = torch.empty((rows, n), dtype=torch.int16, device=self.dev)
            st = torch.zeros(1, dtype=torch.int32, device=self.dev)
            out = (torch.empty(rows, k, device=self.dev), torch.empty(rows, k, dtype=torch.int32, device=self.dev))

            def one():
                xd.copy_(pinned, non_blocking=True)
                atk.approx_top_k_device(xd.view(torch.bfloat16), self.p, status=st, out=out)
                ov.copy_(out[0], non_blocking=True)
                oi.copy_(out[1], non_blocking=True)
                torch.cuda.synchronize(self.dev)
            api = "approx_top_k_device (pinned bf16 H2D + D2H in the region)"
        for _ in range(2):
            one()
        barrier()
        t0 = time.perf_counter()
        for _ in range(steps):
            one()
        el = time.perf_counter() - t0
        assert torch.equal(oi, self.out[1].cpu()), "e2e and device results differ"
        return el, {"h2d_bytes_per_step": rows * n * self.esz, "d2h_bytes_per_step": rows * k * 8, "api": api}

    def cpu_baseline(self):
        be, kind = ref_backend()
        threads = os.cpu_count() or 1
        times = timed_calls(lambda: be.approx_top_k_batch(self.host_f32, self.b, self.kp, self.k, 128,
                                                          threads=threads), 3, 10.0)
        med = statistics.median(times)
        cores = min(threads, self.rows) if kind == "reference" else 1
        return {"value": round(self.rows * self.n / med / 1e9, 4), "unit": "Gelem/s", "cores": cores, "kind": kind,
                "sample": f"full workload ({self.rows} rows x {self.n}) per call, median of {len(times)} calls, "
                          f"approx_top_k_batch(threads={threads}; the reference parallelises over rows)"}

    def reference_sample(self):
        """(callable, elements per call, description, cores) for --impl reference."""
        be, kind = ref_backend()
        threads = (os.cpu_count() or 1) if kind == "reference" else 1
        _, f = make_rows(self.cfg, 0)
        t0 = time.perf_counter()
        be.approx_top_k_batch(f[:threads], self.b, self.kp, self.k, 128, threads=threads)
        per_row = max(1e-6, (time.perf_counter() - t0) / threads)
        budget = min(0.1, 120.0 / max(1, self.args.steps + self.args.warmup))
        rows = int(max(1, min(self.rows, budget / per_row)))
        sample = np.ascontiguousarray(f[:rows])
        fn = lambda: be.approx_top_k_batch(sample, self.b, self.kp, self.k, 128, threads=threads)  # noqa: E731
        return fn, rows * self.n, (f"{rows} of {self.rows} rows x {self.n} per step, "
                                   f"approx_top_k_batch(threads={threads})"), min(threads, rows), kind

    def config(self):
        return {"workload": self.args.config + ": " + self.cfg["label"], "rows_per_gpu": self.rows, "n": self.n,
                "K": self.k, "local_k": self.kp, "num_buckets": self.b, "expected_recall": round(self.rec, 6),
                "parallelism": f"rows sharded across {self.world} GPU(s), no collective",
                "l2": "inputs larger than L2 (no flush needed)" if self.hbm_bytes() > 126e6
                else "L2 flushed between steps"}


class GemmWorkload(RowsWorkload):
    """C4: fused tcgen05 GEMM with stage 1 in the epilogue, then stage 2.
    Per rank: its own 8192 activation rows, W replicated (weak scaling)."""
    kernel = "gemm_tc_kernel (fused stage-1 epilogue)"

    def setup(self, dev):
        import torch
        import paper_2506_04165_b200 as atk
        from paper_2506_04165_b200 import data
        from paper_2506_04165_b200 import topk as T
        self.torch, self.atk, self.T, self.dev = torch, atk, T, dev
        cfg = self.cfg
        self.kdim = cfg["kdim"]
        xb, self.x_f32 = data.normal_bf16(data.SEEDS[cfg["seed"]] + 1000 * self.rank, (self.rows, self.kdim))
        wb, self.w_f32 = data.normal_bf16(data.SEEDS[cfg["wseed"]], (self.n, self.kdim), std=0.02)
        self.host = xb
        self.x = torch.from_numpy(xb.view(np.int16)).to(dev).view(torch.bfloat16)
        self.w = torch.from_numpy(wb.view(np.int16)).to(dev).view(torch.bfloat16)
        self.p = atk.AlgoParams(self.n, self.b, self.kp, self.k)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.out = (torch.empty(self.rows, self.k, device=dev),
                    torch.empty(self.rows, self.k, dtype=torch.int32, device=dev))

    def step(self):
        self.T.fused_gemm_top_k_device(self.x, self.w, self.p, status=self.status, out=self.out)

    def hbm_bytes(self):  # operands + candidates + results
        return (self.rows + self.n) * self.kdim * 2

    def flops(self):
        return 2.0 * self.rows * self.n * self.kdim

    def roofline(self, kern_ms, ms_step):
        path = os.path.join(ROOT, "MEASURED_PEAKS.json")
        peak, sus, src = 1646.4, 1393.0, "measured (MEASURED_PEAKS.json, torch bf16 8192^3 burst)"
        if os.path.exists(path):
            with open(path) as f:
                d = json.load(f)
            peak, sus = float(d.get("bf16_tflops", peak)), float(d.get("bf16_tflops_sustained", sus))
        else:
            src = "fallback"
        ach = self.flops() / (kern_ms * 1e-3) / 1e12
        return {"kernel": self.kernel, "bound": "tensor", "achieved": round(ach, 1), "peak": peak,
                "peak_source": src, "peak_sustained": sus, "unit": "TFLOP/s", "frac": round(ach / peak, 4),
                "traffic": traffic_from_profiles("C4"), "alg_flops_per_launch": self.flops(),
                "launch_ms": round(kern_ms, 5), "share_of_step": round(kern_ms / ms_step, 4)}

    def recall(self):
        atk, T = self.atk, self.T
        scores = T.gemm_bf16_device(self.x, self.w)
        _, ei = atk.exact_top_k_device(scores, self.k)
        rs = [atk.measure_recall(atk.TopKResult(None, self.out[1][r].cpu().numpy().astype(np.uint32)),
                                 atk.TopKResult(None, ei[r].cpu().numpy().astype(np.uint32)))
              for r in range(0, self.rows, 16)]
        del scores
        return float(np.mean(rs))

    def e2e(self, steps, barrier):
        """Per step: this step's activations (x, pinned bf16) H2D, fused
        GEMM + top-K, results D2H.  W is the resident layer weight (the MIPS
        database), loaded once -- not a per-step input."""
        torch = self.torch
        pinned = torch.from_numpy(self.host.view(np.int16)).pin_memory()
        xd = torch.empty((self.rows, self.kdim), dtype=torch.int16, device=self.dev)
        ov = torch.empty((self.rows, self.k), dtype=torch.float32).pin_memory()
        oi = torch.empty((self.rows, self.k), dtype=torch.int32).pin_memory()
        st = torch.zeros(1, dtype=torch.int32, device=self.dev)
        out = (torch.empty_like(self.out[0]), torch.empty_like(self.out[1]))

        def one():
            xd.copy_(pinned, non_blocking=True)
            self.T.fused_gemm_top_k_device(xd.view(torch.bfloat16), self.w, self.p, status=st, out=out)
            ov.copy_(out[0], non_blocking=True)
            oi.copy_(out[1], non_blocking=True)
            torch.cuda.synchronize(self.dev)
        for _ in range(2):
            one()
        barrier()
        t0 = time.perf_counter()
        for _ in range(steps):
            one()
        el = time.perf_counter() - t0
        assert torch.equal(oi, self.out[1].cpu()), "e2e and device results differ"
        return el, {"h2d_bytes_per_step": self.rows * self.kdim * 2, "d2h_bytes_per_step": self.rows * self.k * 8,
                    "api": "fused_gemm_top_k_device (pinned x H2D + D2H in the region; W resident)"}

    def _mips_sample(self, queries):
        be, kind = ref_backend()
        threads = os.cpu_count() or 1
        if kind != "reference":
            return None
        q = np.ascontiguousarray(self.x_f32[:queries])
        return (lambda: be.mips_fused(self.w_f32, q, self.b, self.kp, self.k, 128, 0, threads)), threads

    def cpu_baseline(self):
        threads = os.cpu_count() or 1
        nq = min(self.rows, 8 * threads)
        got = self._mips_sample(nq)
        if got is None:
            return None
        fn, threads = got
        times = timed_calls(fn, 2, 10.0, max_calls=10)
        med = statistics.median(times)
        return {"value": round(nq * self.n / med / 1e9, 4), "unit": "Gelem/s", "cores": threads,
                "kind": "reference",
                "sample": f"{nq} of {self.rows} query rows x {self.n} columns (Kd={self.kdim}) per call, reference "
                          f"mips_fused(threads={threads}) on the fp32 upcast of the same bf16 operands, median of "
                          f"{len(times)} calls"}

    def reference_sample(self):
        threads = os.cpu_count() or 1
        nq = min(self.rows, 4 * threads)
        got = self._mips_sample(nq)
        if got is None:
            raise RuntimeError("reference library (oracle/_ref) not built")
        fn, threads = got
        return fn, nq * self.n, (f"{nq} of {self.rows} query rows x {self.n} columns per step, reference "
                                 f"mips_fused(threads={threads})"), threads, "reference"

    def config(self):
        c = super().config()
        c.update({"kdim": self.kdim, "gemm": "x bf16 [8192, 3584] . W^T bf16 [14336, 3584], fp32 accumulate",
                  "l2": "operands 161 MB > L2; scores never materialised"})
        return c


class GiantRowWorkload(RowsWorkload):
    """C5: one row of 2^30 fp32.  N=1: approx_top_k_device.  N>1: the row is
    sliced across ranks (shard.ShardedTopK): per-rank stage-1 summary,
    NCCL all-gather of the summaries, merge + stage 2 on every rank."""
    scaling = "strong"

    def setup(self, dev):
        import torch
        import paper_2506_04165_b200 as atk
        from paper_2506_04165_b200 import data
        from paper_2506_04165_b200.shard import ShardedTopK, slice_bounds
        self.torch, self.atk, self.dev = torch, atk, dev
        self.p = atk.AlgoParams(self.n, self.b, self.kp, self.k)
        self.start, self.length = slice_bounds(self.n, self.b, self.world, self.rank)
        self.host = data.normal_f32_range(data.SEEDS[self.cfg["seed"]], self.start, self.length)
        self.host_f32 = self.host
        self.x = torch.from_numpy(self.host).to(dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.out = (torch.empty(1, self.k, device=dev), torch.empty(1, self.k, dtype=torch.int32, device=dev))
        # ATKG_BENCH_SHARD=1 forces the sliced path at N=1 too (NCCL group of 1)
        shard = self.world > 1 or os.environ.get("ATKG_BENCH_SHARD") == "1"
        self.sharded = ShardedTopK(self.p) if shard else None

    def step(self):
        if self.sharded is None:
            self.atk.approx_top_k_device(self.x.view(1, -1), self.p, status=self.status, out=self.out)
        else:
            v, i = self.sharded(self.x, status=self.status)
            self.out[0][0].copy_(v)
            self.out[1][0].copy_(i)

    def elements(self):  # per rank per step (its slice)
        return self.length

    def hbm_bytes(self):
        return self.length * 4

    def roofline(self, kern_ms, ms_step):
        peak, src = peaks()
        alg = self.length * 4 + self.b * self.kp * 8
        ach = alg / (kern_ms * 1e-3) / 1e9
        kern = ("stage1_flat_kernel (slice summaries)" if self.sharded is not None
                else "st_stream_kernel (threshold stream; stage-1 pass)")
        return {"kernel": kern, "bound": "hbm", "achieved": round(ach, 1), "peak": peak,
                "peak_source": src, "unit": "GB/s", "frac": round(ach / peak, 4),
                "traffic": traffic_from_profiles("C5"), "alg_bytes_per_launch": alg,
                "launch_ms": round(kern_ms, 5), "share_of_step": round(kern_ms / ms_step, 4)}

    def recall(self):
        if self.sharded is not None:  # the whole row lives on no single rank
            return None
        atk = self.atk
        _, ei = atk.exact_top_k_device(self.x.view(1, -1), self.k)
        return atk.measure_recall(atk.TopKResult(None, self.out[1][0].cpu().numpy().astype(np.uint32)),
                                  atk.TopKResult(None, ei[0].cpu().numpy().astype(np.uint32)))

    def e2e(self, steps, barrier):
        torch, atk = self.torch, self.atk
        pinned = torch.from_numpy(self.host).pin_memory()
        xd = torch.empty(self.length, dtype=torch.float32, device=self.dev)
        ov = torch.empty(self.k, dtype=torch.float32).pin_memory()
        oi = torch.empty(self.k, dtype=torch.int32).pin_memory()
        st = torch.zeros(1, dtype=torch.int32, device=self.dev)
        out = (torch.empty(1, self.k, device=self.dev), torch.empty(1, self.k, dtype=torch.int32, device=self.dev))

        def one():
            xd.copy_(pinned, non_blocking=True)
            if self.sharded is None:
                atk.approx_top_k_device(xd.view(1, -1), self.p, status=st, out=out)
                v, i = out[0][0], out[1][0]
            else:
                v, i = self.sharded(xd, status=st)
            ov.copy_(v, non_blocking=True)
            oi.copy_(i, non_blocking=True)
            torch.cuda.synchronize(self.dev)
        for _ in range(1):
            one()
        barrier()
        t0 = time.perf_counter()
        for _ in range(steps):
            one()
        el = time.perf_counter() - t0
        assert torch.equal(oi, self.out[1][0].cpu()), "e2e and device results differ"
        return el, {"h2d_bytes_per_step": self.length * 4, "d2h_bytes_per_step": self.k * 8,
                    "api": "approx_top_k_device / shard.ShardedTopK (pinned H2D + D2H in the region)"}

    def _prefix(self):
        be, kind = ref_backend()
        m = min(self.length, 1 << 28)
        m -= m % self.b
        row = np.ascontiguousarray(self.host[:m]).reshape(1, m)
        return be, kind, row, m

    def cpu_baseline(self):
        be, kind, row, m = self._prefix()
        times = timed_calls(lambda: be.approx_top_k_batch(row, self.b, self.kp, self.k, 128, threads=1), 2, 10.0,
                            max_calls=5)
        med = statistics.median(times)
        return {"value": round(m / med / 1e9, 4), "unit": "Gelem/s", "cores": 1, "kind": kind,
                "sample": f"first {m} elements of the row as one row (same B, K', K), median of {len(times)} calls; "
                          f"the reference parallelises over rows only, so one row runs on 1 core"}

    def reference_sample(self):
        be, kind, row, m = self._prefix()
        m2 = min(m, 1 << 26)
        r2 = np.ascontiguousarray(row[:, :m2])
        return ((lambda: be.approx_top_k_batch(r2, self.b, self.kp, self.k, 128, threads=1)), m2,
                f"first {m2} elements of the row as one row per step (1 core: the reference parallelises "
                f"over rows only)", 1, kind)

    def config(self):
        c = super().config()
        c["parallelism"] = (f"one row sliced across {self.world} GPUs ({self.length} elements each), NCCL "
                            f"all-gather of the {(2 * self.kp + 2) * self.b * 4} B stage-1 summaries"
                            if self.world > 1 else "1 GPU")
        c["rows_per_gpu"] = 1
        return c


def make_workload(args, cfg, kp, b, rec, world, rank):
    kind = cfg.get("kind", "rows")
    cls = {"rows": RowsWorkload, "gemm": GemmWorkload, "giant": GiantRowWorkload}[kind]
    return cls(args, cfg, kp, b, rec, world, rank)


def run_reference_arm(args, cfg, kp, b, rec):
    """The reference's own CPU path (oracle/_ref = the unmodified atk core
    compiled from /root/reference; the C port only if that build is absent)
    with the host threads it can use, on this config's bytes.  Each step is a
    bounded sample of the workload sized so the whole --steps/--warmup run
    stays within a few minutes; the metric (elements/s) is per element, so
    the sample size does not bias it."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    wl = make_workload(args, cfg, kp, b, rec, 1, 0)
    if cfg.get("kind") == "gemm":
        from paper_2506_04165_b200 import data
        wl.kdim = cfg["kdim"]
        _, wl.x_f32 = data.normal_bf16(data.SEEDS[cfg["seed"]], (cfg["rows"], cfg["kdim"]))
        _, wl.w_f32 = data.normal_bf16(data.SEEDS[cfg["wseed"]], (cfg["n"], cfg["kdim"]), std=0.02)
    elif cfg.get("kind") == "giant":
        from paper_2506_04165_b200 import data
        wl.length = 1 << 26
        wl.host = data.normal_f32_range(data.SEEDS[cfg["seed"]], 0, wl.length)
    fn, elems, desc, cores, kind = wl.reference_sample()
    t0 = time.perf_counter()
    fn()
    one = time.perf_counter() - t0
    steps = args.steps if one * (args.steps + args.warmup) < 180 else max(1, int(150 / max(one, 1e-3)))
    for _ in range(min(args.warmup, 3)):
        fn()
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        fn()
        times.append(time.perf_counter() - t0)
    total = sum(times)
    val = elems * len(times) / total / 1e9
    line = {
        "impl": "reference", "metric": metric_name(), "value": round(val, 4), "unit": "Gelem/s",
        "n_gpus": args.gpus, "steps": len(times), "warmup": args.warmup,
        "ms_per_step": round(total / len(times) * 1e3, 3), "higher_is_better": True, "scaling": wl.scaling,
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded N(0,1), csrc/datagen.cpp)",
        "config": wl.config(),
        "cpu_baseline": {"value": round(val, 4), "unit": "Gelem/s", "cores": cores, "kind": kind, "sample": desc},
        "e2e": {"value": round(val, 4), "unit": "Gelem/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=list(CONFIGS))
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-recall", action="store_true", help="skip the measured-recall check")
    ap.add_argument("--e2e-steps", type=int, default=None)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = CONFIGS[args.config]
    kp, b, rec = plan(cfg)

    if args.impl == "reference":
        run_reference_arm(args, cfg, kp, b, rec)
        return

    import torch
    import torch.distributed as dist

    import paper_2506_04165_b200 as atk
    from paper_2506_04165_b200._lib import lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 or (cfg.get("kind") == "giant" and os.environ.get("ATKG_BENCH_SHARD") == "1"):
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    wl = make_workload(args, cfg, kp, b, rec, world, rank)
    wl.setup(dev)
    wl.step()  # first call: planning, attribute setup; checked for NaN
    wl.check()

    for _ in range(args.warmup):
        wl.step()
    torch.cuda.synchronize()
    barrier()
    stream = torch.cuda.current_stream(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = lib.atkg_launch_count()
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        # dominant-kernel CUDA events on every 16th step only: a bracket sits
        # between that kernel and its PDL-launched successor
        lib.atkg_profile_begin_every(int(os.environ.get("ATKG_BENCH_PROF_EVERY", "16")))
        clocks.mark()
        ev0.record(stream)
        for _ in range(args.steps):
            wl.step()
        ev1.record(stream)
        torch.cuda.synchronize()
        clocks.unmark()
    launches = lib.atkg_launch_count() - launches0
    import ctypes as C
    ktot, kcnt = C.c_double(), C.c_uint64()
    atk._lib.check(lib.atkg_profile_end(C.byref(ktot), C.byref(kcnt)))
    wl.check()
    ms = ev0.elapsed_time(ev1)
    kern_ms = ktot.value / max(1, kcnt.value)
    t = torch.tensor([ms, kern_ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, kern_ms = float(t[0]), float(t[1])
    ms_step = ms / args.steps
    elems = wl.elements() * (world if wl.scaling == "weak" else 1)
    if wl.scaling == "strong":
        elems = cfg["rows"] * cfg["n"]
    value = elems / (ms_step * 1e-3) / 1e9  # Gelem/s, whole job
    hbm_gbs = wl.hbm_bytes() * world / (ms_step * 1e-3) / 1e9

    recall = None if args.no_recall else wl.recall()
    roof = wl.roofline(kern_ms, ms_step)

    e2e_steps = args.e2e_steps or max(3, min(args.steps, 10))
    el, e2e_info = wl.e2e(e2e_steps, barrier)
    te = torch.tensor([el], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    el = float(te[0])
    e2e = {"value": round(elems * e2e_steps / el / 1e9, 4), "unit": "Gelem/s",
           "ms_per_step": round(el / e2e_steps * 1e3, 3), **e2e_info}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = wl.cpu_baseline()

    if rank == 0:
        line = {"metric": metric_name(), "value": round(value, 3), "unit": "Gelem/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 5),
                "higher_is_better": True, "scaling": wl.scaling, "vs_baseline": None, "dtype": wl.dtype,
                "data": "synthetic (seeded N(0,1), csrc/datagen.cpp)", "config": wl.config(),
                "hbm_gbs": round(hbm_gbs, 1),
                "recall": {"expected": round(rec, 6), "measured": None if recall is None else round(recall, 6)},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks.summary(),
                "gpu_launches": int(launches)}
        if cfg.get("kind") == "gemm":
            line["tflops"] = round(wl.flops() * (world if wl.scaling == "weak" else 1) / (ms_step * 1e-3) / 1e12, 1)
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

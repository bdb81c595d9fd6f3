"""Benchmark of the B200 two-stage approximate top-k hot path (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C2]

Workload (BASELINE.json configs[1], the config the metric is quoted on):
  C2 "LM-logit rows": fp32 [256, 262144] i.i.d. N(0,1) (seeded, synthetic),
  K=64, (B, K') from the host planner at expected recall 0.95 with
  K' in {1,2,4}  ->  K'=2, B=128.
A step = approx top-K (stage 1 + stage 2) over the whole batch.

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

N>1 (torchrun): every rank runs its own 256-row batch (rows sharded across
GPUs, no data-path collective), so per-GPU work is fixed: "scaling": "weak".
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
    "C5": dict(rows=1, n=1 << 30, k=1024, target=0.95, kps=(8,), dtype="f32", seed="C5",
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


def cpu_reference_time(rows_f32, cfg, kp, b, steps, min_seconds):
    """Reference CPU path (oracle/_ref) on the same bytes; median per call."""
    from oracle import pyoracle as O
    if not O.ref_available():
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "ref"], capture_output=True)
    if O.ref_available():
        be, kind = O.ref(), "reference"
    else:
        be, kind = O.port(), "port"
    threads = os.cpu_count() or 1
    times = []
    t_start = time.perf_counter()
    while len(times) < steps or (time.perf_counter() - t_start < min_seconds and len(times) < 50):
        t0 = time.perf_counter()
        be.approx_top_k_batch(rows_f32, b, kp, cfg["k"], 128, threads=threads)
        times.append(time.perf_counter() - t0)
    return statistics.median(times), kind, (threads if kind == "reference" else 1), len(times)


def run_reference_arm(args, cfg, kp, b, rec):
    """The reference's own CPU path (oracle/_ref = the unmodified atk core
    compiled from /root/reference; the C port only if that build is absent),
    approx_top_k_batch with every host thread, on this config's bytes.  Each
    step is a bounded sample of the workload (a subset of rows) sized so the
    whole --steps/--warmup run stays within a few minutes; the metric
    (elements/s) is per element, so the sample size does not bias it."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    _, f = make_rows(cfg, 0)
    from oracle import pyoracle as O
    if not O.ref_available():
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "ref"], capture_output=True)
    be = O.ref() if O.ref_available() else O.port()
    kind = "reference" if O.ref_available() else "port"
    threads = (os.cpu_count() or 1) if kind == "reference" else 1
    # size the per-step sample: <= 100 ms and <= 120 s for the whole run
    t0 = time.perf_counter()
    be.approx_top_k_batch(f[:threads], b, kp, cfg["k"], 128, threads=threads)
    per_row = max(1e-6, (time.perf_counter() - t0) / threads)
    budget = min(0.1, 120.0 / max(1, args.steps + args.warmup))
    rows = int(max(1, min(cfg["rows"], budget / per_row)))
    sample = np.ascontiguousarray(f[:rows])
    for _ in range(args.warmup):
        be.approx_top_k_batch(sample, b, kp, cfg["k"], 128, threads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        be.approx_top_k_batch(sample, b, kp, cfg["k"], 128, threads=threads)
        times.append(time.perf_counter() - t0)
    elems = rows * cfg["n"]
    total = sum(times)
    val = elems * len(times) / total / 1e9
    line = {
        "impl": "reference", "metric": metric_name(), "value": round(val, 4), "unit": "Gelem/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total / len(times) * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded N(0,1), csrc/datagen.cpp)",
        "config": config_obj(args, cfg, kp, b, rec),
        "cpu_baseline": {"value": round(val, 4), "unit": "Gelem/s", "cores": threads, "kind": kind,
                         "sample": f"{rows} of {cfg['rows']} rows x {cfg['n']} per step, "
                                   f"approx_top_k_batch(threads={threads})"},
        "e2e": {"value": round(val, 4), "unit": "Gelem/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def metric_name():
    return "approx top-K Gelem/s & HBM GB/s vs ~8 TB/s roofline at matched expected recall"


def config_obj(args, cfg, kp, b, rec):
    return {"workload": args.config + ": " + cfg["label"], "rows_per_gpu": cfg["rows"], "n": cfg["n"],
            "K": cfg["k"], "local_k": kp, "num_buckets": b, "expected_recall": round(rec, 6),
            "parallelism": f"rows sharded across {args.gpus} GPU(s), no collective",
            "l2": "inputs larger than L2 (no flush needed)" if cfg["rows"] * cfg["n"] * 4 > 126e6
            else "L2 flushed between steps"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=list(CONFIGS))
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
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
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    host_rows, host_f32 = make_rows(cfg, rank)
    if cfg["dtype"] == "bf16":
        x = torch.from_numpy(host_rows.view(np.int16)).to(dev).view(torch.bfloat16)
        esz = 2
    else:
        x = torch.from_numpy(host_rows).to(dev)
        esz = 4
    rows, n, k = cfg["rows"], cfg["n"], cfg["k"]
    p = atk.AlgoParams(n, b, kp, k)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    out = (torch.empty(rows, k, device=dev), torch.empty(rows, k, dtype=torch.int32, device=dev))

    def step():
        atk.approx_top_k_device(x, p, status=status, out=out)

    # parity spot check before timing (rank 0 row 0 against the reference)
    step()
    atk.check_status(status)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    stream = torch.cuda.current_stream(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = lib.atkg_launch_count()
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        lib.atkg_profile_begin()
        clocks.mark()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
        clocks.unmark()
    launches = lib.atkg_launch_count() - launches0
    import ctypes as C
    ktot, kcnt = C.c_double(), C.c_uint64()
    atk._lib.check(lib.atkg_profile_end(C.byref(ktot), C.byref(kcnt)))
    atk.check_status(status)
    ms = ev0.elapsed_time(ev1)
    kern_ms = ktot.value / max(1, kcnt.value)
    t = torch.tensor([ms, kern_ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, kern_ms = float(t[0]), float(t[1])
    ms_step = ms / args.steps
    elems = rows * n * world
    value = elems / (ms_step * 1e-3) / 1e9  # Gelem/s, whole job
    hbm_gbs = rows * n * esz * world / (ms_step * 1e-3) / 1e9

    # measured recall vs device exact top-K (outside the timed region)
    ev_, ei_ = atk.exact_top_k_device(x, k)
    recalls = [atk.measure_recall(atk.TopKResult(None, out[1][r].cpu().numpy().astype(np.uint32)),
                                  atk.TopKResult(None, ei_[r].cpu().numpy().astype(np.uint32)))
               for r in range(rows)]
    recall = float(np.mean(recalls))

    # roofline of the stage-1 streaming kernel
    peak, peak_src = peaks()
    alg_bytes = rows * n * esz + rows * b * kp * 8
    achieved = alg_bytes / (kern_ms * 1e-3) / 1e9
    roof = {"kernel": "stage1_flat_kernel", "bound": "hbm", "achieved": round(achieved, 1),
            "peak": peak, "peak_source": peak_src, "unit": "GB/s", "frac": round(achieved / peak, 4),
            "traffic": traffic_from_profiles(args.config), "alg_bytes_per_launch": alg_bytes,
            "launch_ms": round(kern_ms, 5), "share_of_step": round(kern_ms / ms_step, 4)}

    # e2e through the host-buffer C ABI (pinned host memory)
    e2e_steps = args.e2e_steps or max(3, min(args.steps, 10))
    e2e = None
    if cfg["dtype"] == "f32":
        pinned = torch.from_numpy(host_f32).pin_memory()
        ov = torch.empty((rows, k), dtype=torch.float32).pin_memory()
        oi = torch.empty((rows, k), dtype=torch.int32).pin_memory()
        import ctypes as C
        prm = p.c()

        def e2e_step():
            atk._lib.check(lib.atkg_approx_top_k_host(pinned.data_ptr(), rows, C.byref(prm), ov.data_ptr(),
                                                      oi.data_ptr()))
        for _ in range(2):
            e2e_step()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        el = time.perf_counter() - t0
        te = torch.tensor([el], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        el = float(te[0])
        e2e = {"value": round(elems * e2e_steps / el / 1e9, 4), "unit": "Gelem/s",
               "h2d_bytes_per_step": rows * n * 4, "d2h_bytes_per_step": rows * k * 8,
               "ms_per_step": round(el / e2e_steps * 1e3, 3), "api": "atkg_approx_top_k_host (C ABI, pinned host)"}
        # the e2e result must equal the device result
        assert torch.equal(oi, out[1].cpu()), "e2e and device results differ"

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        med, kind, cores, reps = cpu_reference_time(host_f32, cfg, kp, b, steps=3, min_seconds=10.0)
        cpu = {"value": round(rows * n / med / 1e9, 4), "unit": "Gelem/s", "cores": cores, "kind": kind,
               "sample": f"full workload ({rows} rows x {n}) per call, median of {reps} calls, "
                         f"approx_top_k_batch(threads={cores})"}

    if rank == 0:
        line = {"metric": metric_name(), "value": round(value, 3), "unit": "Gelem/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 5),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32" if esz == 4
                else "bf16", "data": "synthetic (seeded N(0,1), csrc/datagen.cpp)",
                "config": config_obj(args, cfg, kp, b, rec), "hbm_gbs": round(hbm_gbs, 1),
                "recall": {"expected": round(rec, 6), "measured": round(recall, 6)},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks.summary(),
                "gpu_launches": int(launches)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

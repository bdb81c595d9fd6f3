"""Host planner mirror: include/atk/planner.hpp + recall.hpp.

select_parameters sweeps local_k ascending and lane-legal bucket counts
descending, scores each with adaptive Monte Carlo, re-validates cheap winners
with the exact Theorem-1 expression (planner.cpp:79-147).  Runs in C++ inside
libatkg.so (csrc/planner.cpp).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import NoFeasibleConfigError, check, lib
from .topk import AlgoParams, kDefaultLaneMultiple

__all__ = ["PlanRequest", "PlanResult", "RecallEstimate", "select_parameters", "legal_bucket_counts",
           "approx_top_k_at_recall",
           "exact_expected_recall", "mc_expected_recall", "mc_expected_recall_adaptive",
           "NoFeasibleConfigError"]


@dataclass
class RecallEstimate:
    """recall.hpp:21-26"""
    value: float = 0.0
    method: str = "exact"  # "exact" | "monte_carlo"
    std_error: Optional[float] = None
    trials: Optional[int] = None


@dataclass
class PlanRequest:
    """planner.hpp:18-27"""
    n: int = 0
    k: int = 0
    recall_target: float = 0.0
    allowed_local_k: Sequence[int] = field(default_factory=lambda: [1, 2, 3, 4])
    lane_multiple: int = kDefaultLaneMultiple
    seed: int = 0


@dataclass
class PlanResult:
    """planner.hpp:29-39"""
    local_k: int = 0
    num_buckets: int = 0
    num_elements: int = 0
    estimated_recall: RecallEstimate = field(default_factory=RecallEstimate)
    high_target_warning: bool = False

    def params(self, req: PlanRequest) -> AlgoParams:
        return AlgoParams(req.n, self.num_buckets, self.local_k, req.k, req.lane_multiple)


def legal_bucket_counts(n: int, lane_multiple: int) -> list[int]:
    if n == 0:
        raise ValueError("n must be >= 1")
    if lane_multiple == 0:
        raise ValueError("lane_multiple must be >= 1")
    cnt = lib.atkg_legal_bucket_counts(n, lane_multiple, None, 0)
    out = np.zeros(max(cnt, 1), np.uint64)
    lib.atkg_legal_bucket_counts(n, lane_multiple, out.ctypes.data, cnt)
    return [int(x) for x in out[:cnt]]


def exact_expected_recall(params: AlgoParams) -> RecallEstimate:
    out = C.c_double()
    check(lib.atkg_exact_expected_recall(C.byref(params.c()), C.byref(out)))
    return RecallEstimate(out.value, "exact")


def mc_expected_recall(params: AlgoParams, trials: int, seed: int) -> RecallEstimate:
    m, s = C.c_double(), C.c_double()
    check(lib.atkg_mc_expected_recall(C.byref(params.c()), trials, seed, C.byref(m), C.byref(s)))
    return RecallEstimate(m.value, "monte_carlo", s.value, trials)


def mc_expected_recall_adaptive(params: AlgoParams, seed: int) -> RecallEstimate:
    m, s, t = C.c_double(), C.c_double(), C.c_uint64()
    check(lib.atkg_mc_expected_recall_adaptive(C.byref(params.c()), seed, C.byref(m), C.byref(s), C.byref(t)))
    return RecallEstimate(m.value, "monte_carlo", s.value, t.value)


def select_parameters(req: PlanRequest) -> PlanResult:
    kps = (C.c_uint32 * max(1, len(req.allowed_local_k)))(*[int(k) for k in req.allowed_local_k])
    creq = _lib.PlanRequestC(req.n, req.k, float(req.recall_target), kps, len(req.allowed_local_k),
                             req.lane_multiple, req.seed)
    out = _lib.PlanResultC()
    check(lib.atkg_select_parameters(C.byref(creq), C.byref(out)))
    method = "exact" if out.recall_method == 0 else "monte_carlo"
    est = RecallEstimate(out.recall, method,
                         out.recall_std_error if method == "monte_carlo" else None,
                         out.recall_trials if method == "monte_carlo" else None)
    return PlanResult(out.local_k, out.num_buckets, out.num_elements, est, bool(out.high_target_warning))


def _plan_from_c(out) -> PlanResult:
    method = "exact" if out.recall_method == 0 else "monte_carlo"
    est = RecallEstimate(out.recall, method,
                         out.recall_std_error if method == "monte_carlo" else None,
                         out.recall_trials if method == "monte_carlo" else None)
    return PlanResult(out.local_k, out.num_buckets, out.num_elements, est, bool(out.high_target_warning))


def approx_top_k_at_recall(rows, row_count: int, req: PlanRequest):
    """The planner, then approx_top_k_batch with its (K', B) (SURVEY 8(b):
    "either a bucket count B or an expected-recall target in").  Host rows
    (numpy, fp32) -> (PlanResult, [TopKResult]); CUDA tensors (fp32/bf16)
    -> (PlanResult, (values [rows, K], indices [rows, K])).  Plans are
    memoised per request inside the library."""
    from . import topk as T
    kps = (C.c_uint32 * max(1, len(req.allowed_local_k)))(*[int(k) for k in req.allowed_local_k])
    creq = _lib.PlanRequestC(req.n, req.k, float(req.recall_target), kps, len(req.allowed_local_k),
                             req.lane_multiple, req.seed)
    out = _lib.PlanResultC()
    if T._is_device(rows):
        import torch
        x = rows.reshape(row_count, -1).contiguous()
        dev = x.device
        dt = T._dtype_code(x)
        nbytes = C.c_size_t()
        check(lib.atkg_approx_at_recall_workspace_size(dt, row_count, C.byref(creq), C.byref(nbytes)))
        ws = T.workspace(nbytes.value, dev)
        ov = torch.empty((row_count, req.k), dtype=torch.float32, device=dev)
        oi = torch.empty((row_count, req.k), dtype=torch.int32, device=dev)
        st = T._status(dev)
        check(lib.atkg_approx_top_k_at_recall(dt, x.data_ptr(), row_count, C.byref(creq), C.byref(out), ov.data_ptr(),
                                              oi.data_ptr(), ws.data_ptr(), ws.numel(), st.data_ptr(),
                                              T._stream_ptr(dev)))
        T._check_device_status(st, dev)
        return _plan_from_c(out), (ov, oi)
    x = T._host_f32(rows)
    if x.size != row_count * req.n:
        raise ValueError("batch length does not match row_count * n")
    k = int(req.k)
    ov = np.empty(row_count * k, np.float32)
    oi = np.empty(row_count * k, np.uint32)
    check(lib.atkg_approx_top_k_at_recall_host(x.ctypes.data, row_count, C.byref(creq), C.byref(out),
                                               ov.ctypes.data, oi.ctypes.data))
    return _plan_from_c(out), [T.TopKResult(ov[r * k:(r + 1) * k], oi[r * k:(r + 1) * k]) for r in range(row_count)]

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

"""Recall simulation: host mirror of atk/simulate.hpp.

``simulate_recall_many`` runs seeded permutation rows (``synth_distinct_row``,
dataset.cpp:132-150) through the device approx_top_k for every configuration
and returns the reference's ``SimStats`` (simulate.cpp:53-113), bit for bit:
rows are built on host threads, top-k and recall counting run on the GPU.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .topk import AlgoParams


@dataclass
class SimStats:
    """atk::SimStats (simulate.hpp:13-20)."""
    mean_recall: float = 0.0
    stddev: float = 0.0
    runs: int = 0

    def std_error(self) -> float:
        return self.stddev / math.sqrt(self.runs) if self.runs > 0 else 0.0


def synth_distinct(rows: int, n: int, seed: int, first_row: int = 0, threads: int = 8) -> np.ndarray:
    """[rows, n] fp32; row r == atk::synth_distinct_row(n, seed, first_row + r)."""
    out = np.empty((max(rows, 0), max(n, 1)), np.float32)
    _lib.check(_lib.lib.atkg_synth_distinct(first_row, rows, n, seed, out.ctypes.data, threads))
    return out


def synth_distinct_device(rows: int, n: int, seed: int, first_row: int = 0, device=None) -> "torch.Tensor":
    """Same rows generated in HBM (n <= 2^16): [rows, n] fp32 CUDA tensor."""
    import torch
    from .topk import _stream_ptr
    dev = torch.device(device if device is not None else "cuda")
    out = torch.empty((rows, n), dtype=torch.float32, device=dev)
    _lib.check(_lib.lib.atkg_synth_distinct_device(first_row, rows, n, seed, out.data_ptr() if out.numel() else None,
                                                   _stream_ptr(out.device)))
    return out


def synth_distinct_row(n: int, seed: int, row_index: int) -> np.ndarray:
    return synth_distinct(1, n, seed, first_row=row_index, threads=1)[0]


def simulate_recall_many(configs, runs: int, seed: int, threads: int = 8, device=None) -> list:
    """atk::simulate_recall_many; the top-k runs on `device` (default cuda)."""
    import torch
    from .topk import _stream_ptr
    configs = list(configs)
    arr = (_lib.Params * max(len(configs), 1))(*[c.c() for c in configs])
    mean = (C.c_double * max(len(configs), 1))()
    sd = (C.c_double * max(len(configs), 1))()
    stream = None  # no CUDA device: argument errors still surface; the run itself fails loudly
    if torch.cuda.is_available():
        dev = torch.device(device if device is not None else "cuda")
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        stream = _stream_ptr(dev)
    _lib.check(_lib.lib.atkg_simulate_recall_many(arr, len(configs), runs, seed, threads, mean, sd, stream))
    return [SimStats(mean[i], sd[i], runs) for i in range(len(configs))]


def simulate_recall(params: AlgoParams, runs: int, seed: int, threads: int = 8, device=None) -> SimStats:
    """atk::simulate_recall (simulate.cpp:115-118)."""
    return simulate_recall_many([params], runs, seed, threads, device)[0]

"""MIPS workload mirror of atk/mips.hpp: fp32, reference-exact.

* ``score_block`` -> ``atkg_mips_score`` (mips.cpp:57-91 order: one fp32
  accumulator per score, j ascending, multiply and add rounded separately).
* ``mips_unfused`` / ``mips_fused`` (mips.cpp:109-193): scores [chunk, n_padded]
  on the device (padded columns -inf), stage 1 over the padded row
  (``stage1_device``), then stage 2 over the filled slots with padded indices
  dropped (``select_candidates_device``, index_limit = rows) -- reduce_query,
  mips.cpp:95-103.  Both pipelines return identical results, as in the
  reference; ``mips_fused`` reports the reference's block statistics.  Query
  chunks bound the device score buffer to ~2 GiB.
* The bf16 tcgen05 pipeline with stage 1 in the GEMM epilogue is
  ``fused_gemm_top_k_device`` (C4).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .dataset import VectorDataset
from .topk import (AlgoParams, TopKResult, _check_device_status, _status, _stream_ptr, select_candidates_device,
                   stage1_device)

try:
    import torch
except ImportError:  # pragma: no cover
    torch = None

_SCORE_BUDGET = 2 << 30  # bytes of device scores per query chunk


@dataclass
class MipsStats:
    """mips.hpp:22-28."""
    score_buffer_bytes: int = 0
    padded_n: int = 0
    blocks: int = 0


@dataclass
class MipsResult:
    """mips.hpp:30-33."""
    per_query: list = field(default_factory=list)
    stats: MipsStats = field(default_factory=MipsStats)


def _padded_params(p: AlgoParams) -> AlgoParams:
    b = p.num_buckets
    return AlgoParams(n=(p.n + b - 1) // b * b if b else p.n, num_buckets=b, local_k=p.local_k,
                      global_k=p.global_k, lane_multiple=p.lane_multiple)


def validate_mips_request(database: VectorDataset, queries: VectorDataset, params: AlgoParams) -> None:
    """mips.cpp:36-55 (same checks, same order, same messages)."""
    database.validate()
    queries.validate()
    if database.dims != queries.dims:
        raise ValueError("mips: database/query dims differ")
    if database.dims == 0:
        raise ValueError("mips: dims must be >= 1")
    if database.rows == 0:
        raise ValueError("mips: database must not be empty")
    if queries.rows == 0:
        raise ValueError("mips: queries must not be empty")
    if params.n != database.rows:
        raise ValueError("mips: params.n must equal database rows")
    if params.global_k > database.rows:
        raise ValueError("mips: global_k exceeds database rows")
    _padded_params(params).validate()


def default_block_cols(params: AlgoParams) -> int:
    """mips.cpp:195-199."""
    b = params.num_buckets
    return b if b >= 4096 else b * ((4096 + b - 1) // b)


def _dev(x: np.ndarray, device) -> "torch.Tensor":
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(device)


def score_block_device(queries: "torch.Tensor", database: "torch.Tensor", n_padded: int | None = None,
                       out: "torch.Tensor | None" = None) -> "torch.Tensor":
    """[b, d] x [n, d] fp32 CUDA tensors -> [b, n_padded] scores (-inf past n)."""
    q, db = queries.contiguous(), database.contiguous()
    b, d = q.shape
    n = db.shape[0]
    npad = n if n_padded is None else n_padded
    if out is None:
        out = torch.empty((b, npad), dtype=torch.float32, device=q.device)
    _lib.check(_lib.lib.atkg_mips_score(q.data_ptr(), b, db.data_ptr(), n, d, out.data_ptr(), out.stride(0),
                                        npad, _stream_ptr(q.device)))
    return out


def mips_top_k_device(queries: "torch.Tensor", database: "torch.Tensor", params: AlgoParams):
    """Device pipeline: (values [b, K] f32, indices [b, K] int32) CUDA tensors."""
    padded = _padded_params(params)
    b, n = queries.shape[0], database.shape[0]
    filled = min(padded.local_k, padded.n // padded.num_buckets) * padded.num_buckets
    chunk = max(1, min(b, _SCORE_BUDGET // (padded.n * 4)))
    vs, is_ = [], []
    st = _status(queries.device)  # one status word, checked once after every chunk is queued
    for q0 in range(0, b, chunk):
        scores = score_block_device(queries[q0:q0 + chunk], database, padded.n)
        gv, gi = stage1_device(scores, padded, status=st)
        v, i = select_candidates_device(gv, gi, params.global_k, index_limit=n, count=filled, status=st)
        vs.append(v)
        is_.append(i)
        del scores, gv, gi
    _check_device_status(st, queries.device)
    return torch.cat(vs), torch.cat(is_)


def _run(database: VectorDataset, queries: VectorDataset, params: AlgoParams, device):
    dev = torch.device(device if device is not None else "cuda")
    v, i = mips_top_k_device(_dev(queries.matrix(), dev), _dev(database.matrix(), dev), params)
    v, i = v.cpu().numpy(), i.cpu().numpy().astype(np.uint32)
    return [TopKResult(v[q].copy(), i[q].copy()) for q in range(v.shape[0])]


def mips_unfused(database: VectorDataset, queries: VectorDataset, params: AlgoParams, threads: int = 1,
                 device=None) -> MipsResult:
    """mips.cpp:109-136."""
    validate_mips_request(database, queries, params)
    np_ = _padded_params(params).n
    return MipsResult(_run(database, queries, params, device), MipsStats(queries.rows * np_ * 4, np_, 1))


def mips_fused(database: VectorDataset, queries: VectorDataset, params: AlgoParams, block_cols: int,
               threads: int = 1, device=None) -> MipsResult:
    """mips.cpp:138-193 (results identical to mips_unfused by construction)."""
    validate_mips_request(database, queries, params)
    if block_cols == 0:
        raise ValueError("mips: block_cols must be >= 1")
    if block_cols % params.num_buckets != 0 and params.num_buckets % block_cols != 0:
        raise ValueError("mips: block_cols must be a multiple or a divisor of num_buckets")
    np_ = _padded_params(params).n
    stats = MipsStats(queries.rows * block_cols * 4, np_, (np_ + block_cols - 1) // block_cols)
    return MipsResult(_run(database, queries, params, device), stats)

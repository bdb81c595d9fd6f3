"""Host-side mirror of the reference `atk` core API (proj/core/include/atk/topk.hpp,
params.hpp), backed by the sm_100a kernels of libatkg.so.

Same names, argument meaning and error behaviour as the reference:
``std::invalid_argument`` -> ``ValueError`` with the reference's message.

Two calling conventions:
* host arrays (numpy / lists)       -> the drop-in form: host buffers in and
  out, synchronous (the reference's std::span API);
* torch CUDA tensors (fp32 / bf16)  -> device tensors out, computed on the
  tensor's device and current stream; the NaN flag is checked before
  returning, as the reference rejects NaN up front (topk.cpp:22-28).
Indices are uint32 on the host (numpy) and int32 on the device (torch),
bit-identical for n < 2^31.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _lib
from ._lib import check, lib

try:  # torch is plumbing for device memory and streams only
    import torch
except Exception:  # pragma: no cover
    torch = None

kDefaultLaneMultiple = 128
kNegInf = float("-inf")


@dataclass
class AlgoParams:
    """include/atk/params.hpp:20-48"""
    n: int = 0
    num_buckets: int = 0
    local_k: int = 0
    global_k: int = 0
    lane_multiple: int = kDefaultLaneMultiple

    def bucket_size(self) -> int:
        return self.n // self.num_buckets if self.num_buckets else 0

    def num_candidates(self) -> int:
        return self.num_buckets * self.local_k

    def c(self) -> _lib.Params:
        for name in ("n", "num_buckets"):
            v = getattr(self, name)
            if v < 0 or v >= 2**64:
                raise ValueError(f"{name} out of range")
        for name in ("local_k", "global_k", "lane_multiple"):
            v = getattr(self, name)
            if v < 0 or v >= 2**32:
                raise ValueError(f"{name} out of range")
        return _lib.make_params(self.n, self.num_buckets, self.local_k, self.global_k, self.lane_multiple)

    def validate(self) -> None:
        check(lib.atkg_validate(C.byref(self.c())))

    def validate_analysis(self) -> None:
        check(lib.atkg_validate_analysis(C.byref(self.c())))


@dataclass
class TopKResult:
    """include/atk/params.hpp:54-59: values[i] is the (i+1)-th largest."""
    values: object = field(default_factory=lambda: np.zeros(0, np.float32))
    indices: object = field(default_factory=lambda: np.zeros(0, np.uint32))

    def size(self) -> int:
        return len(self.values)


def partition_index(i: int, params: AlgoParams) -> int:
    """topk.hpp:13-15 -- element i goes to bucket i mod B."""
    return i % params.num_buckets


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------
def _is_device(x) -> bool:
    return torch is not None and isinstance(x, torch.Tensor) and x.is_cuda


def _host_f32(x) -> np.ndarray:
    if torch is not None and isinstance(x, torch.Tensor):
        x = x.detach().cpu().float().numpy()
    return np.ascontiguousarray(np.asarray(x, dtype=np.float32).reshape(-1))


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _dtype_code(t) -> int:
    if t.dtype == torch.float32:
        return _lib.ATKG_F32
    if t.dtype == torch.bfloat16:
        return _lib.ATKG_BF16
    raise ValueError("device inputs must be float32 or bfloat16")


_ws_cache: dict = {}
_approx_plan_cache: dict = {}


def workspace(nbytes: int, device) -> "torch.Tensor":
    """Caller-supplied scratch (include/atkg.h), cached per (device, stream):
    calls on different streams never share scratch (a buffer is only reused
    by work ordered after it on the same stream)."""
    dev = device.index if hasattr(device, "index") and device.index is not None else torch.cuda.current_device()
    stream = torch.cuda.current_stream(dev)
    key = (dev, stream.cuda_stream)
    buf = _ws_cache.get(key)
    if buf is None or buf.numel() < nbytes:
        # allocated on `stream`: the caching allocator hands a freed block
        # back only to later work on that same stream
        buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=torch.device("cuda", dev))
        _ws_cache[key] = buf
    return buf


_tls = threading.local()


def _stream_ptr(device) -> int:
    """Current torch stream of `device`; also points the library's CUDA
    runtime at that device (its device state is per host thread, so the
    cache is too)."""
    idx = device.index if device.index is not None else torch.cuda.current_device()
    if getattr(_tls, "dev", None) != idx:
        check(lib.atkg_set_device(idx))
        _tls.dev = idx
    return torch.cuda.current_stream(device).cuda_stream


def _status(device) -> "torch.Tensor":
    return torch.zeros(1, dtype=torch.int32, device=device)


def _check_device_status(status, device) -> None:
    check(lib.atkg_check_status(C.c_void_p(status.data_ptr()), C.c_void_p(_stream_ptr(device))))


def _ws_size(op: int, dtype: int, rows: int, p: _lib.Params) -> int:
    out = C.c_size_t()
    check(lib.atkg_workspace_size(op, dtype, rows, C.byref(p), C.byref(out)))
    return out.value


# ---------------------------------------------------------------------------
# the reference API
# ---------------------------------------------------------------------------
def stage1_partial_reduce(input, params: AlgoParams) -> TopKResult:
    """topk.hpp:98-99 / topk.cpp:178-186: the [local_k, num_buckets] grid."""
    params.validate()
    if _is_device(input):
        v, i = stage1_device(input.reshape(1, -1), params)
        return TopKResult(v[0], i[0])
    x = _host_f32(input)
    if x.size != params.n:
        raise ValueError("input length does not match params.n")
    g = params.num_candidates()
    vals = np.empty(g, np.float32)
    idx = np.empty(g, np.uint32)
    check(lib.atkg_stage1_host(_ptr(x), 1, C.byref(params.c()), _ptr(vals), _ptr(idx)))
    return TopKResult(vals, idx)


def select_top_k_candidates(values, indices, k: int, index_limit: int = 2**64 - 1) -> TopKResult:
    """topk.hpp:109-112 / topk.cpp:219-236."""
    v = _host_f32(values)
    i = np.ascontiguousarray(np.asarray(indices, dtype=np.uint32).reshape(-1))
    if v.size != i.size:
        raise ValueError("candidate value/index lengths differ")
    if k <= 0:
        raise ValueError("k must be >= 1")
    ov = np.empty(k, np.float32)
    oi = np.empty(k, np.uint32)
    vv = v if v.size else np.zeros(1, np.float32)
    ii = i if i.size else np.zeros(1, np.uint32)
    check(lib.atkg_select_candidates_host(_ptr(vv), _ptr(ii), v.size, k, min(index_limit, 2**64 - 1),
                                          _ptr(ov), _ptr(oi)))
    return TopKResult(ov, oi)


def exact_top_k(input, k: int) -> TopKResult:
    """topk.hpp:104 / topk.cpp:206-217 (recall measurement)."""
    if _is_device(input):
        v, i = exact_top_k_device(input.reshape(1, -1), k)
        return TopKResult(v[0], i[0])
    x = _host_f32(input)
    if k <= 0:
        raise ValueError("k must be >= 1")
    ov = np.empty(k, np.float32)
    oi = np.empty(k, np.uint32)
    check(lib.atkg_exact_top_k_host(_ptr(x), x.size, k, _ptr(ov), _ptr(oi)))
    return TopKResult(ov, oi)


def approx_top_k(input, params: AlgoParams) -> TopKResult:
    """topk.hpp:117 / topk.cpp:238-258."""
    params.validate()
    if _is_device(input):
        v, i = approx_top_k_device(input.reshape(1, -1), params)
        return TopKResult(v[0], i[0])
    x = _host_f32(input)
    if x.size != params.n:
        raise ValueError("input length does not match params.n")
    return approx_top_k_batch(x, 1, params)[0]


def approx_top_k_batch(rows, row_count: int, params: AlgoParams, threads: int = 1) -> list:
    """topk.hpp:121-124 / topk.cpp:260-273.  `threads` is accepted for API
    parity; the device path is thread-count invariant like the reference."""
    params.validate()
    if _is_device(rows):
        v, i = approx_top_k_device(rows.reshape(row_count, -1), params)
        return [TopKResult(v[r], i[r]) for r in range(row_count)]
    x = _host_f32(rows)
    if x.size != row_count * params.n:
        raise ValueError("batch length does not match row_count * n")
    k = params.global_k
    ov = np.empty(row_count * k, np.float32)
    oi = np.empty(row_count * k, np.uint32)
    if row_count:
        check(lib.atkg_approx_top_k_host(_ptr(x), row_count, C.byref(params.c()), _ptr(ov), _ptr(oi)))
    return [TopKResult(ov[r * k:(r + 1) * k], oi[r * k:(r + 1) * k]) for r in range(row_count)]


def measure_recall(approx: TopKResult, exact: TopKResult) -> float:
    """topk.hpp:128 / topk.cpp:275-297."""
    a = np.ascontiguousarray(_to_np_u32(approx.indices))
    e = np.ascontiguousarray(_to_np_u32(exact.indices))
    out = C.c_double()
    check(lib.atkg_measure_recall(_ptr(a) if a.size else None, a.size, _ptr(e) if e.size else None, e.size,
                                  C.byref(out)))
    return out.value


def _to_np_u32(x) -> np.ndarray:
    if torch is not None and isinstance(x, torch.Tensor):
        return x.detach().cpu().numpy().astype(np.uint32)
    return np.asarray(x, dtype=np.uint32).reshape(-1)


# ---------------------------------------------------------------------------
# device (torch tensor) entry points
# ---------------------------------------------------------------------------
def stage1_device(x: "torch.Tensor", params: AlgoParams, status=None):
    """[rows, n] fp32/bf16 CUDA tensor -> grid values [rows, kp*B] f32,
    indices [rows, kp*B] int32 (bucket-minor, topk.hpp:59-67)."""
    params.validate()
    x = x.contiguous()
    rows = x.shape[0]
    if x.shape[1] != params.n:
        raise ValueError("input length does not match params.n")
    dev = x.device
    g = params.num_candidates()
    vals = torch.empty((rows, g), dtype=torch.float32, device=dev)
    idx = torch.empty((rows, g), dtype=torch.int32, device=dev)
    p = params.c()
    dt = _dtype_code(x)
    ws = workspace(_ws_size(_lib.OP_STAGE1, dt, rows, p), dev)
    st = status if status is not None else _status(dev)
    check(lib.atkg_stage1(dt, x.data_ptr(), rows, C.byref(p), vals.data_ptr(), idx.data_ptr(), ws.data_ptr(),
                          ws.numel(), st.data_ptr(), _stream_ptr(dev)))
    if status is None:
        _check_device_status(st, dev)
    return vals, idx


def approx_top_k_device(x: "torch.Tensor", params: AlgoParams, status=None, out=None):
    """[rows, n] CUDA tensor -> (values [rows, K] f32, indices [rows, K] int32).
    Pass a zeroed int32 `status` tensor to skip the per-call synchronising
    NaN check (then call check_status yourself)."""
    # validated params + workspace size per (params, rows, dtype, device): the
    # host side of a call is on the critical path when the device step is
    # ~50 us (the size is the max over every dispatch path, so environment
    # switches between calls stay within it)
    rows = x.shape[0]
    dev = x.device
    key = (params.n, params.num_buckets, params.local_k, params.global_k, params.lane_multiple, rows, x.dtype,
           dev.index)
    ent = _approx_plan_cache.get(key)
    if ent is None:
        params.validate()
    x = x.contiguous()
    if x.shape[1] != params.n:
        raise ValueError("batch length does not match row_count * n")
    k = params.global_k
    if out is None:
        vals = torch.empty((rows, k), dtype=torch.float32, device=dev)
        idx = torch.empty((rows, k), dtype=torch.int32, device=dev)
    else:
        vals, idx = out
    dt = _dtype_code(x)
    if ent is None:
        p = params.c()
        ent = (p, _ws_size(_lib.OP_APPROX, dt, rows, p))
        _approx_plan_cache[key] = ent
    p, nbytes = ent
    ws = workspace(nbytes, dev)
    st = status if status is not None else _status(dev)
    check(lib.atkg_approx_top_k(dt, x.data_ptr(), rows, C.byref(p), vals.data_ptr(), idx.data_ptr(),
                                ws.data_ptr(), ws.numel(), st.data_ptr(), _stream_ptr(dev)))
    if status is None:
        _check_device_status(st, dev)
    return vals, idx


def select_candidates_device(vals: "torch.Tensor", idx: "torch.Tensor", k: int,
                             index_limit: int = 2**64 - 1, count: int | None = None, status=None):
    """Per-row stage 2 over [rows, C] candidate tensors.  Pass a zeroed int32
    `status` tensor to skip the per-call synchronising check."""
    rows, stride = vals.shape
    count = stride if count is None else count
    dev = vals.device
    p = _lib.make_params(count, 1, 1, k, 1)
    ws = workspace(_ws_size(_lib.OP_SELECT, 0, rows, p), dev)
    ov = torch.empty((rows, k), dtype=torch.float32, device=dev)
    oi = torch.empty((rows, k), dtype=torch.int32, device=dev)
    st = status if status is not None else _status(dev)
    check(lib.atkg_select_candidates(vals.contiguous().data_ptr(), idx.contiguous().data_ptr(), rows, count, stride,
                                     k, min(index_limit, 2**64 - 1), ov.data_ptr(), oi.data_ptr(), ws.data_ptr(),
                                     ws.numel(), st.data_ptr(), _stream_ptr(dev)))
    if status is None:
        _check_device_status(st, dev)
    return ov, oi


def exact_top_k_device(x: "torch.Tensor", k: int, status=None):
    x = x.contiguous()
    rows, n = x.shape
    dev = x.device
    p = _lib.make_params(n, 1, 1, k, 1)
    dt = _dtype_code(x)
    ws = workspace(_ws_size(_lib.OP_EXACT, dt, rows, p), dev)
    ov = torch.empty((rows, k), dtype=torch.float32, device=dev)
    oi = torch.empty((rows, k), dtype=torch.int32, device=dev)
    st = status if status is not None else _status(dev)
    check(lib.atkg_exact_top_k(dt, x.data_ptr(), rows, n, k, ov.data_ptr(), oi.data_ptr(), ws.data_ptr(),
                               ws.numel(), st.data_ptr(), _stream_ptr(dev)))
    if status is None:
        _check_device_status(st, dev)
    return ov, oi


def check_status(status: "torch.Tensor") -> None:
    _check_device_status(status, status.device)


class Stage1Accumulator:
    """include/atk/topk.hpp:68-94 -- streaming stage 1 over one row, fed in
    index order, any block length or alignment; device-resident state."""

    def __init__(self, params: AlgoParams, device=None):
        params.validate()
        self._params = params
        self._device = torch.device(device if device is not None else "cuda")
        h = C.c_void_p()
        with torch.cuda.device(self._device):
            check(lib.atkg_accumulator_create(C.byref(params.c()), C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib.atkg_accumulator_destroy(h)
            self._h = None

    def params(self) -> AlgoParams:
        return self._params

    def consume(self, block) -> None:
        if not _is_device(block):
            block = torch.as_tensor(np.asarray(block, dtype=np.float32).reshape(-1))
            if torch.isnan(block).any():
                raise ValueError("input contains NaN")
            block = block.to(self._device)
        block = block.contiguous().reshape(-1)
        if block.numel() == 0:
            return
        check(lib.atkg_accumulator_consume(self._h, _dtype_code(block), block.data_ptr(), block.numel(),
                                           _stream_ptr(self._device)))
        # the reference rejects NaN inside consume(); surface it here
        torch.cuda.current_stream(self._device).synchronize()

    def consumed(self) -> int:
        return int(lib.atkg_accumulator_consumed(self._h))

    def _grid(self):
        g = self._params.num_candidates()
        v = torch.empty(g, dtype=torch.float32, device=self._device)
        i = torch.empty(g, dtype=torch.int32, device=self._device)
        check(lib.atkg_accumulator_candidates(self._h, v.data_ptr(), i.data_ptr(), _stream_ptr(self._device)))
        return v, i

    def values(self) -> np.ndarray:
        return self._grid()[0].cpu().numpy()

    def indices(self) -> np.ndarray:
        return self._grid()[1].cpu().numpy().astype(np.uint32)

    def candidates(self) -> TopKResult:
        v, i = self._grid()
        return TopKResult(v.cpu().numpy(), i.cpu().numpy().astype(np.uint32))


# ---------------------------------------------------------------------------
# giant-row slice sharding (summaries are what crosses NVLink)
# ---------------------------------------------------------------------------
def summary_words(params: AlgoParams) -> int:
    return (2 * params.local_k + 2) * params.num_buckets


def stage1_summary_device(slice_: "torch.Tensor", index_offset: int, params: AlgoParams, out=None, status=None):
    """Exact per-bucket summary of elements [index_offset, index_offset+len)
    of a row of params.n elements (uint32 words, summary_words(params))."""
    params.validate()
    x = slice_.contiguous().reshape(-1)
    dev = x.device
    p = params.c()
    summ = out if out is not None else torch.empty(summary_words(params), dtype=torch.int32, device=dev)
    dt = _dtype_code(x)
    pp = _lib.make_params(x.numel(), params.num_buckets, params.local_k, 1, 1)
    ws = workspace(_ws_size(_lib.OP_SUMMARY, dt, 1, pp), dev)
    st = status if status is not None else _status(dev)
    check(lib.atkg_stage1_summary(dt, x.data_ptr(), x.numel(), index_offset, C.byref(p), summ.data_ptr(),
                                  ws.data_ptr(), ws.numel(), st.data_ptr(), _stream_ptr(dev)))
    if status is None:
        _check_device_status(st, dev)
    return summ


def summary_merge_top_k_device(summaries: "torch.Tensor", params: AlgoParams, want_grid: bool = False,
                               status=None):
    """Merge G slice summaries ([G, words], index order) -> top-K (and grid)."""
    params.validate()
    s = summaries.contiguous()
    parts = s.shape[0] if s.dim() == 2 else 1
    dev = s.device
    p = params.c()
    k = params.global_k
    ov = torch.empty(k, dtype=torch.float32, device=dev)
    oi = torch.empty(k, dtype=torch.int32, device=dev)
    gv = gi = None
    if want_grid:
        gv = torch.empty(params.num_candidates(), dtype=torch.float32, device=dev)
        gi = torch.empty(params.num_candidates(), dtype=torch.int32, device=dev)
    ws = workspace(_ws_size(_lib.OP_MERGE, 0, 1, p), dev)
    st = status if status is not None else _status(dev)
    check(lib.atkg_summary_merge_top_k(s.data_ptr(), parts, C.byref(p), gv.data_ptr() if gv is not None else None,
                                       gi.data_ptr() if gi is not None else None, ov.data_ptr(), oi.data_ptr(),
                                       ws.data_ptr(), ws.numel(), st.data_ptr(), _stream_ptr(dev)))
    if status is None:
        _check_device_status(st, dev)
    return (ov, oi, gv, gi) if want_grid else (ov, oi)


def slice_payload_words(params: AlgoParams, parts: int) -> int:
    out = C.c_size_t()
    check(lib.atkg_slice_payload_words(C.byref(params.c()), parts, C.byref(out)))
    return out.value


def slice_payload_device(slice_: "torch.Tensor", index_offset: int, params: AlgoParams, parts: int, out=None,
                         status=None):
    """Threshold-stream payload of elements [index_offset, index_offset+len)
    of a row sliced into `parts` (int32 words, slice_payload_words)."""
    params.validate()
    x = slice_.contiguous().reshape(-1)
    dev = x.device
    p = params.c()
    dt = _dtype_code(x)
    words = slice_payload_words(params, parts)
    pay = out if out is not None else torch.empty(words, dtype=torch.int32, device=dev)
    nbytes = C.c_size_t()
    check(lib.atkg_slice_payload_workspace(dt, x.numel(), C.byref(p), parts, C.byref(nbytes)))
    ws = workspace(nbytes.value, dev)
    st = status if status is not None else _status(dev)
    check(lib.atkg_slice_payload(dt, x.data_ptr(), x.numel(), index_offset, C.byref(p), parts, pay.data_ptr(),
                                 ws.data_ptr(), ws.numel(), st.data_ptr(), _stream_ptr(dev)))
    return pay


def payload_merge_top_k_device(payloads: "torch.Tensor", params: AlgoParams, status=None):
    """Merge `parts` slice payloads ([parts, words], index order) -> (values,
    indices, gate).  gate (int32 device tensor) != 0: the payloads cannot
    settle the row; take the exact summary path."""
    params.validate()
    s = payloads.contiguous()
    parts = s.shape[0]
    dev = s.device
    k = params.global_k
    ov = torch.empty(k, dtype=torch.float32, device=dev)
    oi = torch.empty(k, dtype=torch.int32, device=dev)
    gate = torch.zeros(1, dtype=torch.int32, device=dev)
    st = status if status is not None else _status(dev)
    check(lib.atkg_payload_merge_top_k(s.data_ptr(), parts, C.byref(params.c()), ov.data_ptr(), oi.data_ptr(),
                                       gate.data_ptr(), st.data_ptr(), _stream_ptr(dev)))
    return ov, oi, gate


class NcclComm:
    """An NCCL communicator created by libatkg.so's own (run-time loaded)
    NCCL, for atkg_sharded_approx_top_k.  The unique id travels by any
    side channel (torch.distributed's store in tests)."""

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib.atkg_nccl_unique_id(buf))
        return buf.raw

    def __init__(self, nranks: int, uid: bytes, rank: int):
        h = C.c_void_p()
        check(lib.atkg_nccl_comm_init(C.byref(h), nranks, C.create_string_buffer(uid, 128), rank))
        self.h, self.nranks, self.rank = h, nranks, rank

    def close(self):
        if self.h is not None and self.h.value:
            check(lib.atkg_nccl_comm_destroy(self.h))
            self.h = None


def sharded_approx_top_k_device(slice_: "torch.Tensor", index_offset: int, params: AlgoParams, comm: NcclComm,
                                status=None):
    """atkg_sharded_approx_top_k: this rank's slice of one row -> the row's
    top-K on every rank (payload exchange, exact fallback), over NCCL."""
    params.validate()
    x = slice_.contiguous().reshape(-1)
    dev = x.device
    p = params.c()
    dt = _dtype_code(x)
    nbytes = C.c_size_t()
    check(lib.atkg_sharded_workspace_size(dt, x.numel(), C.byref(p), comm.nranks, C.byref(nbytes)))
    ws = workspace(nbytes.value, dev)
    k = params.global_k
    ov = torch.empty(k, dtype=torch.float32, device=dev)
    oi = torch.empty(k, dtype=torch.int32, device=dev)
    st = status if status is not None else _status(dev)
    check(lib.atkg_sharded_approx_top_k(dt, x.data_ptr(), x.numel(), index_offset, C.byref(p), comm.h, comm.nranks,
                                        ov.data_ptr(), oi.data_ptr(), ws.data_ptr(), ws.numel(), st.data_ptr(),
                                        _stream_ptr(dev)))
    if status is None:
        _check_device_status(st, dev)
    return ov, oi


# ---------------------------------------------------------------------------
# C4: tcgen05 GEMM with stage 1 in the epilogue (mips_fused, mips.cpp:138-193)
# ---------------------------------------------------------------------------
def _check_gemm_operands(x, w_t):
    if x.dtype != torch.bfloat16 or w_t.dtype != torch.bfloat16:
        raise ValueError("GEMM operands must be bfloat16")
    if x.dim() != 2 or w_t.dim() != 2 or x.shape[1] != w_t.shape[1]:
        raise ValueError("x must be [M, Kd] and w_t [N, Kd]")
    return x.contiguous(), w_t.contiguous()


def gemm_bf16_device(x: "torch.Tensor", w_t: "torch.Tensor", out=None) -> "torch.Tensor":
    """fp32 scores = x[M,Kd] . w_t[N,Kd]^T on the tcgen05 tensor cores."""
    x, w_t = _check_gemm_operands(x, w_t)
    m, kd = x.shape
    n = w_t.shape[0]
    dev = x.device
    if out is None:
        out = torch.empty((m, n), dtype=torch.float32, device=dev)
    check(lib.atkg_gemm_bf16(x.data_ptr(), w_t.data_ptr(), m, kd, n, out.data_ptr(), _stream_ptr(dev)))
    return out


def fused_workspace_bytes(m: int, kdim: int, params: AlgoParams) -> int:
    out = C.c_size_t()
    p = params.c()
    check(lib.atkg_fused_workspace_size(m, kdim, C.byref(p), C.byref(out)))
    return out.value


def fused_gemm_top_k_device(x: "torch.Tensor", w_t: "torch.Tensor", params: AlgoParams,
                            scores: "torch.Tensor | None" = None, status=None, out=None):
    """Approximate top-K of every row of x . w_t^T without materialising the
    scores (params.n == N).  `scores` (an [M, N] f32 tensor) optionally
    receives the exact fp32 scores the epilogue consumed, for oracle replay."""
    params.validate()
    x, w_t = _check_gemm_operands(x, w_t)
    m, kd = x.shape
    if w_t.shape[0] != params.n:
        raise ValueError("w_t must have params.n rows")
    dev = x.device
    k = params.global_k
    if out is None:
        vals = torch.empty((m, k), dtype=torch.float32, device=dev)
        idx = torch.empty((m, k), dtype=torch.int32, device=dev)
    else:
        vals, idx = out
    if scores is not None and (scores.dtype != torch.float32 or tuple(scores.shape) != (m, params.n)
                               or not scores.is_contiguous()):
        raise ValueError("scores must be a contiguous float32 [M, N] tensor")
    p = params.c()
    ws = workspace(fused_workspace_bytes(m, kd, params), dev)
    st = status if status is not None else _status(dev)
    check(lib.atkg_fused_gemm_top_k(x.data_ptr(), w_t.data_ptr(), m, kd, C.byref(p), vals.data_ptr(),
                                    idx.data_ptr(), scores.data_ptr() if scores is not None else None,
                                    ws.data_ptr(), ws.numel(), st.data_ptr(), _stream_ptr(dev)))
    if status is None:
        _check_device_status(st, dev)
    return vals, idx

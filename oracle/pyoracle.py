"""TEST INFRASTRUCTURE ONLY -- ctypes access to the two CPU checkers.

* ``port``: oracle/_build/libatk_oracle.so, the plain-C restatement
  (oracle/atk_oracle.c), built by ``make -C oracle port``.
* ``ref``:  oracle/_ref/libatk_ref.so, the unmodified reference core compiled
  from /root/reference sources (``make -C oracle ref``).  Present only where it
  was built (here, and on the GPU box because built .so files travel with
  gpurun); tests skip the ``ref`` backend when the file is absent.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import
this module.  Every function raises ValueError for the reference's
std::invalid_argument and RuntimeError for NoFeasibleConfigError, mirroring
the reference error contract (proj/core/src/topk.cpp:20-28, planner.hpp:14-16).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_PATH = os.path.join(HERE, "_build", "libatk_oracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libatk_ref.so")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_u64, _u32, _f64, _i = C.c_uint64, C.c_uint32, C.c_double, C.c_int


class NoFeasibleConfig(RuntimeError):
    pass


@dataclass
class Plan:
    local_k: int
    num_buckets: int
    recall: float
    exact: bool
    warning: bool


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


class _Backend:
    def __init__(self, kind: str):
        self.kind = kind
        path = PORT_PATH if kind == "port" else REF_PATH
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -C oracle {kind})")
        lib = C.CDLL(path)
        p = "orc_" if kind == "port" else "ref_"
        self.p = p
        self.lib = lib
        self._err = getattr(lib, p + "last_error")
        self._err.restype = C.c_char_p
        sig = {
            "validate": [_u64, _u64, _u32, _u32, _u32],
            "stage1": [_f32p, _u64, _u64, _u32, _u32, _f32p, _u32p],
            "select_candidates": [_f32p, _u32p, _u64, _u32, _u64, _f32p, _u32p],
            "exact_top_k": [_f32p, _u64, _u32, _f32p, _u32p],
            "exact_expected_recall": [_u64, _u64, _u32, _u32, C.POINTER(_f64)],
            "select_parameters": [_u64, _u64, _f64, _u32p, _u32, _u32, _u64,
                                  C.POINTER(_u32), C.POINTER(_u64), C.POINTER(_f64),
                                  C.POINTER(_i), C.POINTER(_i)],
        }
        for name, args in sig.items():
            fn = getattr(lib, p + name)
            fn.argtypes = args
            fn.restype = _i
        ub = getattr(lib, p + "update_bucket")
        ub.argtypes = [_f32p, _u32p, _u32, C.c_float, _u32]
        lbc = getattr(lib, p + "legal_bucket_counts")
        lbc.argtypes = [_u64, _u64, _u64p, _u64]
        lbc.restype = _u64
        if kind == "port":
            lib.orc_approx_top_k_batch.argtypes = [_f32p, _u64, _u64, _u64, _u32, _u32,
                                                   _u32, _f32p, _u32p]
            lib.orc_approx_top_k_batch.restype = _i
            lib.orc_measure_recall.argtypes = [_u32p, _u32p, _u64, C.POINTER(_f64)]
            lib.orc_measure_recall.restype = _i
            lib.orc_mc_expected_recall.argtypes = [_u64, _u64, _u32, _u32, _u64, _u64,
                                                   C.POINTER(_f64), C.POINTER(_f64)]
            lib.orc_mc_expected_recall.restype = _i
            lib.orc_shuffled_iota.argtypes = [_u64, _u64, _f32p]
            lib.orc_uniform_below.argtypes = [_u64, _u64, _u64, _f32p]
            lib.orc_xoshiro_fill.argtypes = [_u64, _u64, _u64p]
            lib.orc_fill_normal_range.argtypes = [_u64, _u64, _u64, C.c_float, C.c_float, _f32p]
            lib.orc_round_bf16.argtypes = [_f32p, _u64, _f32p, C.c_void_p]
            lib.orc_derive_seed.argtypes = [_u64, _u64]
            lib.orc_derive_seed.restype = _u64
            lib.orc_score_block.argtypes = [_f32p, _u64, _f32p, _u64, _u64, _u64, _f32p, _u64]
        else:
            lib.ref_approx_top_k_batch.argtypes = [_f32p, _u64, _u64, _u64, _u32, _u32,
                                                   _u32, _u32, _f32p, _u32p]
            lib.ref_approx_top_k_batch.restype = _i
            lib.ref_measure_recall.argtypes = [_f32p, _u32p, _f32p, _u32p, _u64,
                                               C.POINTER(_f64)]
            lib.ref_measure_recall.restype = _i
            lib.ref_mc_expected_recall.argtypes = [_u64, _u64, _u32, _u32, _u64, _u64,
                                                   C.POINTER(_f64), C.POINTER(_f64)]
            lib.ref_mc_expected_recall.restype = _i
            lib.ref_score_block.argtypes = [_f32p, _u64, _f32p, _u64, _u64, _u64, _u64,
                                            _f32p, _u64]
            lib.ref_mips_fused.argtypes = [_f32p, _u64, _u64, _f32p, _u64, _u64, _u32, _u32, _u32,
                                           _u64, _u32, _f32p, _u32p]
            lib.ref_mips_fused.restype = _i

    def _check(self, rc: int):
        if rc == 0:
            return
        msg = self._err().decode()
        if rc == 3:
            raise NoFeasibleConfig(msg)
        raise ValueError(msg)

    def _fn(self, name):
        return getattr(self.lib, self.p + name)

    # ---- topk core -----------------------------------------------------
    def validate(self, n, b, kp, k, lane=128):
        self._check(self._fn("validate")(n, b, kp, k, lane))

    def stage1(self, row, b, kp, lane=128):
        row = np.ascontiguousarray(row, np.float32)
        v = np.empty(b * kp, np.float32)
        i = np.empty(b * kp, np.uint32)
        self._check(self._fn("stage1")(row, row.size, b, kp, lane, v, i))
        return v, i

    def select_candidates(self, vals, idx, k, index_limit=2**64 - 1):
        vals = np.ascontiguousarray(vals, np.float32)
        idx = np.ascontiguousarray(idx, np.uint32)
        if vals.size != idx.size:
            raise ValueError("candidate value/index lengths differ")
        ov = np.empty(max(k, 1), np.float32)
        oi = np.empty(max(k, 1), np.uint32)
        vv = vals if vals.size else np.zeros(1, np.float32)
        ii = idx if idx.size else np.zeros(1, np.uint32)
        self._check(self._fn("select_candidates")(vv, ii, vals.size, k, index_limit, ov, oi))
        return ov[:k], oi[:k]

    def exact_top_k(self, row, k):
        row = np.ascontiguousarray(row, np.float32)
        ov = np.empty(max(k, 1), np.float32)
        oi = np.empty(max(k, 1), np.uint32)
        self._check(self._fn("exact_top_k")(row, row.size, k, ov, oi))
        return ov[:k], oi[:k]

    def approx_top_k_batch(self, rows, b, kp, k, lane=128, threads=None):
        rows = np.ascontiguousarray(rows, np.float32)
        if rows.ndim == 1:
            rows = rows[None, :]
        r, n = rows.shape
        ov = np.empty((r, k), np.float32)
        oi = np.empty((r, k), np.uint32)
        if self.kind == "port":
            rc = self.lib.orc_approx_top_k_batch(rows.reshape(-1), r, n, b, kp, k, lane,
                                                 ov.reshape(-1), oi.reshape(-1))
        else:
            t = threads if threads is not None else (os.cpu_count() or 1)
            rc = self.lib.ref_approx_top_k_batch(rows.reshape(-1), r, n, b, kp, k, lane, t,
                                                 ov.reshape(-1), oi.reshape(-1))
        self._check(rc)
        return ov, oi

    def approx_top_k(self, row, b, kp, k, lane=128):
        ov, oi = self.approx_top_k_batch(np.asarray(row, np.float32)[None, :], b, kp, k, lane)
        return ov[0], oi[0]

    def measure_recall(self, approx_idx, exact_idx):
        a = np.ascontiguousarray(approx_idx, np.uint32)
        e = np.ascontiguousarray(exact_idx, np.uint32)
        if a.size != e.size:
            raise ValueError("recall needs results of equal size")
        if a.size == 0:
            raise ValueError("recall of empty results is undefined")
        out = _f64()
        if self.kind == "port":
            self._check(self.lib.orc_measure_recall(a, e, a.size, C.byref(out)))
        else:
            z = np.zeros(a.size, np.float32)
            self._check(self.lib.ref_measure_recall(z, a, z, e, a.size, C.byref(out)))
        return out.value

    def update_bucket(self, values, indices, value, index):
        v = np.ascontiguousarray(values, np.float32).copy()
        i = np.ascontiguousarray(indices, np.uint32).copy()
        getattr(self.lib, self.p + "update_bucket")(v, i, v.size, float(value), int(index))
        return v, i

    # ---- recall / planner ----------------------------------------------
    def exact_expected_recall(self, n, b, kp, k):
        out = _f64()
        self._check(self._fn("exact_expected_recall")(n, b, kp, k, C.byref(out)))
        return out.value

    def mc_expected_recall(self, n, b, kp, k, trials, seed):
        m, s = _f64(), _f64()
        self._check(self._fn("mc_expected_recall")(n, b, kp, k, trials, seed, C.byref(m),
                                                  C.byref(s)))
        return m.value, s.value

    def legal_bucket_counts(self, n, lane):
        fn = self._fn("legal_bucket_counts")
        cnt = fn(n, lane, np.zeros(1, np.uint64), 0)
        out = np.zeros(max(cnt, 1), np.uint64)
        fn(n, lane, out, cnt)
        return [int(x) for x in out[:cnt]]

    def select_parameters(self, n, k, target, allowed_local_k=(1, 2, 3, 4), lane=128, seed=0):
        kps = np.ascontiguousarray(list(allowed_local_k) or [0], np.uint32)
        kp, b, rec, ex, w = _u32(), _u64(), _f64(), _i(), _i()
        rc = self._fn("select_parameters")(n, k, target, kps, len(allowed_local_k), lane, seed,
                                           C.byref(kp), C.byref(b), C.byref(rec), C.byref(ex),
                                           C.byref(w))
        self._check(rc)
        return Plan(kp.value, b.value, rec.value, bool(ex.value), bool(w.value))

    def score_block(self, queries, database, c0, c1):
        q = np.ascontiguousarray(queries, np.float32)
        db = np.ascontiguousarray(database, np.float32)
        b, d = q.shape
        out = np.empty((b, c1 - c0), np.float32)
        if self.kind == "port":
            self.lib.orc_score_block(q.reshape(-1), b, db.reshape(-1), d, c0, c1,
                                     out.reshape(-1), c1 - c0)
        else:
            self.lib.ref_score_block(q.reshape(-1), b, db.reshape(-1), db.shape[0], d, c0, c1,
                                     out.reshape(-1), c1 - c0)
        return out

    def mips_fused(self, database, queries, b, kp, k, lane=128, block_cols=0, threads=1):
        """Reference mips_fused (mips.cpp:138-193); reference backend only."""
        db = np.ascontiguousarray(database, np.float32)
        q = np.ascontiguousarray(queries, np.float32)
        rows, d = db.shape
        nq = q.shape[0]
        ov = np.empty((nq, k), np.float32)
        oi = np.empty((nq, k), np.uint32)
        self._check(self.lib.ref_mips_fused(db.reshape(-1), rows, d, q.reshape(-1), nq, b, kp, k, lane,
                                            block_cols, threads, ov.reshape(-1), oi.reshape(-1)))
        return ov, oi


_cache: dict = {}


def backend(kind: str = "port") -> _Backend:
    if kind not in _cache:
        _cache[kind] = _Backend(kind)
    return _cache[kind]


def port() -> _Backend:
    return backend("port")


def ref() -> _Backend:
    return backend("ref")


# ---- seeded fixtures the reference tests use (restated) -----------------
def shuffled_iota(n: int, seed: int) -> np.ndarray:
    """proj/tests/test_topk.cpp:30-39"""
    out = np.empty(n, np.float32)
    port().lib.orc_shuffled_iota(n, seed, out)
    return out


def uniform_below(seed: int, bound: int, count: int) -> np.ndarray:
    """x = float(rng.next_below(bound)) stream (test_topk.cpp:194-195)."""
    out = np.empty(count, np.float32)
    port().lib.orc_uniform_below(seed, bound, count, out)
    return out


def derive_seed(seed: int, stream: int) -> int:
    return int(port().lib.orc_derive_seed(seed, stream))


def normal_f32(seed: int, start: int, count: int, mean: float = 0.0, std: float = 1.0) -> np.ndarray:
    """The build's seeded N(mean, std) stream, elements [start, start + count)
    (start % 65536 == 0), computed by the oracle port -- for callers that must
    not load the product library (bench.py --impl reference)."""
    if start % 65536:
        raise ValueError("start must be a multiple of 65536")
    out = np.empty(count, np.float32)
    port().lib.orc_fill_normal_range(seed, start, count, mean, std, out)
    return out


def round_bf16(x: np.ndarray):
    """(bf16 bits, exact fp32 values) of fp32 x, round to nearest even."""
    x = np.ascontiguousarray(x, np.float32).reshape(-1)
    out = np.empty_like(x)
    bits = np.empty(x.size, np.uint16)
    port().lib.orc_round_bf16(x, x.size, out, bits.ctypes.data)
    return bits, out

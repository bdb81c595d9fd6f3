"""Seeded parity inputs shared by make_golden.py and the tests.

Generators: paper_2506_04165_b200.data (Box-Muller normals, bf16 RNE) and
the reference test fixtures restated in oracle.pyoracle (shuffled_iota,
next_below streams).  A SHA-256 of every built input is stored beside the
reference outputs, so a generator change fails loudly instead of silently
comparing different data.
"""
from __future__ import annotations

import numpy as np

# value tables indexed by seeded next_below draws (duplicate / special-value heavy)
_TABLES = {
    "pm0_inf": np.array([0.0, -0.0, 1.0, -1.0, np.inf, -np.inf, 2.0, 0.5], np.float32),
    "neg_inf": np.array([-np.inf, -np.inf, -np.inf, -1.0, 0.0, 1.0], np.float32),
}

INPUTS = {
    # BASELINE configs[0] (C1) at full size
    "c1": dict(kind="normal", seed=0, rows=16, n=32768, B=512, kp=4, k=128),
    # C2 / C3 shapes on a few rows (full-size runs are checked by properties)
    "c2_rows": dict(kind="normal", seed=2, rows=4, n=262144, B=128, kp=2, k=64),
    "c3_rows": dict(kind="normal_bf16", seed=3, rows=48, n=14336, B=128, kp=4, k=287),
    "c3_k1": dict(kind="normal_bf16", seed=3, rows=48, n=14336, B=3584, kp=1, k=287),
    "c3_k2": dict(kind="normal_bf16", seed=3, rows=48, n=14336, B=512, kp=2, k=287),
    "c3_k8": dict(kind="normal_bf16", seed=3, rows=48, n=14336, B=128, kp=8, k=287),
    "c3_r99": dict(kind="normal_bf16", seed=3, rows=48, n=14336, B=256, kp=4, k=287),
    # the rest of the C3 r = 0.99 sweep (planner: K'=1 -> B=7168, K'=2 -> B=1024)
    "c3_r99_k1": dict(kind="normal_bf16", seed=3, rows=48, n=14336, B=7168, kp=1, k=287),
    "c3_r99_k2": dict(kind="normal_bf16", seed=3, rows=48, n=14336, B=1024, kp=2, k=287),
    # giant-row split path at reduced size (many segments per bucket)
    "c5_mini": dict(kind="normal", seed=6, rows=1, n=1 << 22, B=256, kp=8, k=1024),
    # test_topk.cpp:177-188 (simulation scale vs per-bucket sort)
    "iota_262144": dict(kind="iota", seed=20240601, rows=1, n=262144, B=1024, kp=4, k=1024),
    # test_topk.cpp:190-210 (duplicate-heavy vs scalar Alg. 1)
    "dup_heavy": dict(kind="below", seed=99, bound=17, rows=1, n=4096, B=32, kp=3, k=50, lane=1),
    "dup_heavy_rows": dict(kind="below", seed=98, bound=9, rows=8, n=65536, B=128, kp=4, k=300),
    "pm0_inf": dict(kind="table", table="pm0_inf", seed=7, rows=4, n=4096, B=64, kp=4, k=100, lane=1),
    "neg_inf": dict(kind="table", table="neg_inf", seed=8, rows=4, n=2048, B=16, kp=8, k=60, lane=1),
    "kp16": dict(kind="normal", seed=9, rows=2, n=65536, B=256, kp=16, k=1000),
    "kp_generic": dict(kind="below", seed=10, bound=50, rows=2, n=8192, B=64, kp=9, k=100, lane=1),
    "b_odd": dict(kind="normal", seed=11, rows=3, n=999, B=3, kp=2, k=5, lane=1),
    # test_topk.cpp:266-286 (local_k > bucket size, duplicates)
    "tiny_bucket": dict(kind="below", seed=12, bound=64, rows=2, n=512, B=64, kp=9, k=100, lane=1),
    "bucket_eq_kp": dict(kind="below", seed=13, bound=64, rows=2, n=256, B=32, kp=8, k=50, lane=1),
}


def build(spec: dict) -> np.ndarray:
    """fp32 rows [rows, n] as the reference sees them (bf16 -> exact upcast)."""
    from oracle import pyoracle as O
    from paper_2506_04165_b200 import data

    rows, n = spec["rows"], spec["n"]
    kind = spec["kind"]
    if kind == "normal":
        return data.normal_f32(spec["seed"], (rows, n))
    if kind == "normal_bf16":
        _, f = data.normal_bf16(spec["seed"], (rows, n))
        return f
    if kind == "iota":
        assert rows == 1
        return O.shuffled_iota(n, spec["seed"])[None, :]
    if kind == "below":
        return O.uniform_below(spec["seed"], spec["bound"], rows * n).reshape(rows, n)
    if kind == "table":
        t = _TABLES[spec["table"]]
        sel = O.uniform_below(spec["seed"], len(t), rows * n).astype(np.int64)
        return t[sel].reshape(rows, n)
    raise ValueError(kind)


def build_device_input(spec: dict):
    """What the GPU consumes: bf16 bits for *_bf16 kinds, else fp32."""
    from paper_2506_04165_b200 import data

    if spec["kind"] == "normal_bf16":
        bits, _ = data.normal_bf16(spec["seed"], (spec["rows"], spec["n"]))
        return bits
    return build(spec)

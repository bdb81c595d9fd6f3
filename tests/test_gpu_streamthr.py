"""GPU parity of the threshold-stream approx_top_k path for long rows
(csrc/streamthr.cuh): a persistent TMA-ring stream that logs, per warp
sub-stream, the elements above a rising threshold, and a per-row finish that
rebuilds the exact candidates >= L (or falls back to exact Alg. 1 summaries).

Every case is compared bit for bit with the reference library (oracle/_ref,
approx_top_k_batch, /root/reference/proj/core/src/topk.cpp:238-273): random
rows at several shapes and both dtypes, rows that defeat the threshold
(ramps, -inf rows, all-equal rows, +-0, +inf, quantised ties), row/piece
boundary layouts, the forced exact fallback, and NaN rejection.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import paper_2506_04165_b200 as atk  # noqa: E402
from paper_2506_04165_b200 import data  # noqa: E402

pytestmark = pytest.mark.gpu


def bits(a):
    if isinstance(a, torch.Tensor):
        a = a.detach().cpu().numpy()
    return np.asarray(a, np.float32).view(np.uint32)


def u32(a):
    if isinstance(a, torch.Tensor):
        a = a.detach().cpu().numpy()
    return np.asarray(a).astype(np.uint32)


def dev_input(x, dtype, cuda):
    if dtype == "bf16":
        b16 = data.f32_to_bf16_bits(x)
        return torch.from_numpy(b16.view(np.int16)).to(cuda).view(torch.bfloat16), data.bf16_bits_to_f32(b16)
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(cuda), np.ascontiguousarray(x, np.float32)


def check(ref, cuda, x, dtype, B, kp, k):
    xd, f = dev_input(x, dtype, cuda)
    n = x.shape[1]
    p = atk.AlgoParams(n, B, kp, k, min(B, 128))
    v, i = atk.approx_top_k_device(xd, p)
    rv, ri = ref.approx_top_k_batch(f, B, kp, k, lane=min(B, 128))
    bad = np.nonzero(~(bits(v) == bits(rv)).all(axis=1) | ~(u32(i) == ri).all(axis=1))[0]
    assert bad.size == 0, f"rows {bad[:8].tolist()} differ from the reference"
    return v, i


SHAPES = [  # dtype, rows, n, B, kp, k
    ("f32", 16, 262144, 128, 2, 64),     # C2 (reduced rows)
    ("f32", 16, 32768, 512, 4, 128),     # C1
    ("f32", 9, 262144, 128, 1, 64),
    ("f32", 12, 65536, 256, 4, 512),
    ("f32", 5, 98304, 64, 8, 300),
    ("f32", 40, 32768, 128, 2, 200),     # many rows per piece
    ("f32", 3, 131072 + 4, 4, 8, 20),    # n not a multiple of the line; B = 4
    ("f32", 1, 1 << 22, 256, 8, 1024),   # giant-row shape (scaled): many pieces per row
    ("bf16", 16, 262144, 128, 2, 64),
    ("bf16", 8, 65536, 128, 4, 287),
    ("bf16", 24, 32768, 256, 1, 100),
    ("bf16", 2, 1 << 21, 256, 8, 1024),
]


@pytest.mark.parametrize("dtype,rows,n,B,kp,k", SHAPES)
def test_streamthr_normal_vs_reference(cuda, ref, dtype, rows, n, B, kp, k):
    rng = np.random.default_rng(n + 7 * B + kp * 131 + k + rows)
    x = rng.standard_normal((rows, n)).astype(np.float32)
    check(ref, cuda, x, dtype, B, kp, k)


@pytest.mark.parametrize("dtype,rows,n,B,kp,k", [s for s in SHAPES if s[1] >= 3 and s[2] <= 262144])
def test_streamthr_forced_fallback(cuda, ref, opts, dtype, rows, n, B, kp, k):
    opts("st_force_slow", 1)
    rng = np.random.default_rng(n + B + kp + k)
    x = rng.standard_normal((min(rows, 4), n)).astype(np.float32)
    check(ref, cuda, x, dtype, B, kp, k)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("n,B,kp,k", [(65536, 128, 2, 64), (32768, 256, 4, 287)])
def test_streamthr_adversarial_vs_reference(cuda, ref, dtype, n, B, kp, k):
    """Rows built to defeat the threshold stream: every one must still match."""
    rng = np.random.default_rng(n + B + kp + k)
    rows = 14
    x = rng.standard_normal((rows, n)).astype(np.float32)
    nstr = n // B
    x[0] = -1.0
    x[0, np.arange(1, nstr, 4) * B] = 50.0 + np.arange(len(range(1, nstr, 4)))  # all large in bucket 0
    x[1] = np.arange(n, dtype=np.float32)          # ascending ramp: every element raises L
    x[2] = -np.arange(n, dtype=np.float32)         # descending ramp
    x[3] = -np.inf                                 # sentinels only
    x[4] = -np.inf
    x[4, rng.choice(n, size=3 * k, replace=False)] = rng.standard_normal(3 * k)
    x[5] = 1.5                                     # one equal run
    x[6] = np.where(rng.random(n) < 0.5, 2.0, -2.0)
    x[7] = np.where(rng.random(n) < 0.5, 0.0, -0.0)
    x[7, rng.choice(n, size=k // 2, replace=False)] = 1.0
    x[8, rng.choice(n, size=k // 3 + 1, replace=False)] = np.inf
    x[9] = rng.standard_normal(n) * np.float32(1e30) ** rng.random(n)
    x[10] = np.round(rng.standard_normal(n) * 3)   # quantised: ties at every threshold
    x[11] = np.round(rng.standard_normal(n) * 40) / 8
    x[12, : n // 2] -= 8.0                         # non-stationary halves
    x[13] = np.inf
    check(ref, cuda, x, dtype, B, kp, k)


def test_streamthr_row_piece_layouts(cuda, ref):
    """Row counts that put row boundaries at every position inside pieces."""
    rng = np.random.default_rng(11)
    for rows in (1, 2, 3, 7, 33, 150, 301):
        x = rng.standard_normal((rows, 32768)).astype(np.float32)
        check(ref, cuda, x, "f32", 128, 2, 64)


def test_streamthr_nan_flag(cuda):
    x = np.random.default_rng(3).standard_normal((8, 65536)).astype(np.float32)
    x[5, 12345] = np.nan
    for dtype in ("f32", "bf16"):
        xd, _ = dev_input(x, dtype, cuda)
        with pytest.raises(ValueError, match="NaN"):
            atk.approx_top_k_device(xd, atk.AlgoParams(65536, 128, 2, 64))


def test_streamthr_matches_previous_path(cuda):
    """Same answers as the exact-summary streaming path (option no_streamthr=1)."""
    x = np.random.default_rng(5).standard_normal((32, 262144)).astype(np.float32)
    xd = torch.from_numpy(x).to(cuda)
    p = atk.AlgoParams(262144, 128, 2, 64)
    v, i = atk.approx_top_k_device(xd, p)
    with atk._lib.option("no_streamthr", 1):
        v2, i2 = atk.approx_top_k_device(xd, p)
    assert np.array_equal(bits(v), bits(v2)) and np.array_equal(u32(i), u32(i2))


@pytest.mark.parametrize("force", [False, True])
def test_streamthr_giant_row_gate(cuda, ref, opts, force):
    """Giant-row mode (no in-kernel fallback): a failed row is flagged and the
    host reruns the exact path; both outcomes match the reference."""
    opts("st_giant_n", 65536)
    if force:
        opts("st_force_slow", 1)
    rng = np.random.default_rng(77)
    x = rng.standard_normal((2, 1 << 21)).astype(np.float32)
    check(ref, cuda, x, "f32", 256, 8, 1024)
    x = rng.standard_normal((3, 262144)).astype(np.float32)
    x[1] = np.arange(262144, dtype=np.float32)  # ramp: the threshold fails
    check(ref, cuda, x, "f32", 128, 2, 64)

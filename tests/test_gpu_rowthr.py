"""GPU parity of the row-threshold approx_top_k path (csrc/rowthr.cuh).

One warp per shared-memory-resident row: a sampled row threshold L, hit masks,
exact Alg. 1 only over the elements >= L, a counting sort on the value code.
Every case is compared bit for bit with the reference library
(oracle/_ref, approx_top_k_batch) -- including rows that defeat the
threshold guess (the exact slow path), heavy ties, -inf rows, and the
counting-sort / bitonic switch -- and with the previous row-resident kernel
(option no_rowthr=1), which computes the full grid.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import paper_2506_04165_b200 as atk  # noqa: E402
from paper_2506_04165_b200 import data  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _force_rowthr(opts):
    """The planner picks this path for K' >= 8 only (and only when the
    short-row kernel does not apply); force it for every K'."""
    opts("rowthr", 1)
    opts("no_short", 1)


def bits(a):
    if isinstance(a, torch.Tensor):
        a = a.detach().cpu().numpy()
    return np.asarray(a, np.float32).view(np.uint32)


def u32(a):
    if isinstance(a, torch.Tensor):
        a = a.detach().cpu().numpy()
    return np.asarray(a).astype(np.uint32)


def dev_input(x, dtype, cuda):
    """x: f32 numpy rows -> (device tensor, exact f32 view of what the device sees)"""
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
    assert np.array_equal(bits(v), bits(rv)), "values differ from the reference"
    assert np.array_equal(u32(i), ri), "indices differ from the reference"
    return v, i


SHAPES = [  # dtype, n, B, kp, k
    ("bf16", 14336, 128, 4, 287),   # C3
    ("bf16", 14336, 128, 1, 100),
    ("bf16", 14336, 128, 2, 200),
    ("bf16", 14336, 128, 8, 287),
    ("bf16", 14336, 64, 4, 200),
    ("bf16", 14336, 256, 4, 287),
    ("bf16", 14336, 256, 2, 500),   # K close to B*K': the guess often fails
    ("bf16", 14336, 512, 2, 300),   # 28 stride-rows, 512 threads
    ("bf16", 8192, 64, 2, 100),     # 128 stride-rows (both halves full), 64 threads
    ("bf16", 8192, 128, 4, 512),    # K == B*K': every candidate is output
    ("bf16", 2048, 128, 4, 64),     # 16 stride-rows
    ("bf16", 1024, 128, 8, 64),     # 8 stride-rows: sample stride 1, K' = nstr
    ("bf16", 512, 128, 8, 100),     # 4 stride-rows < K': filled prefix
    ("f32", 4096, 128, 4, 100),
    ("f32", 8192, 64, 2, 100),
    ("f32", 2048, 32, 8, 200),
    ("f32", 16384, 128, 4, 300),
]


@pytest.mark.parametrize("dtype,n,B,kp,k", SHAPES)
def test_rowthr_normal_vs_reference(cuda, ref, dtype, n, B, kp, k):
    rng = np.random.default_rng(n + 7 * B + kp * 131 + k)
    x = rng.standard_normal((96, n)).astype(np.float32)
    check(ref, cuda, x, dtype, B, kp, k)


@pytest.mark.parametrize("dtype,n,B,kp,k", [s for s in SHAPES if s[1] >= 2048])
def test_rowthr_adversarial_vs_reference(cuda, ref, dtype, n, B, kp, k):
    """Rows built to break the sampled threshold (slow path) or the counting sort."""
    rng = np.random.default_rng(n + B + kp + k)
    rows = 24
    x = rng.standard_normal((rows, n)).astype(np.float32)
    nstr = n // B
    # 0: all large values in bucket 0, off the sampled stride-rows
    x[0] = -1.0
    x[0, np.arange(1, nstr, 4) * B] = 50.0 + np.arange(len(range(1, nstr, 4)))
    # 1: large values only on unsampled stride-rows of a few buckets
    x[1, :] = rng.standard_normal(n) - 10.0
    for j in range(1, nstr, 2):
        x[1, j * B: j * B + 3] = 5.0 + rng.standard_normal(3)
    # 2: mostly -inf, a few finite values (L = -inf -> slow path)
    x[2] = -np.inf
    x[2, rng.choice(n, size=min(n, 3 * k), replace=False)] = rng.standard_normal(min(n, 3 * k))
    # 3: everything -inf (sentinel semantics)
    x[3] = -np.inf
    # 4: all equal (one huge equal-value run)
    x[4] = 1.5
    # 5: two values
    x[5] = np.where(rng.random(n) < 0.5, 2.0, -2.0)
    # 6: +-0 mixture with a few positives
    x[6] = np.where(rng.random(n) < 0.5, 0.0, -0.0)
    x[6, rng.choice(n, size=k // 2, replace=False)] = 1.0
    # 7: +inf values
    x[7, rng.choice(n, size=k // 3 + 1, replace=False)] = np.inf
    # 8: wide value range (counting sort range overflow -> bitonic)
    x[8] = rng.standard_normal(n) * np.float32(1e30) ** rng.random(n)
    # 9: integer quantised (many ties at the threshold)
    x[9] = np.round(rng.standard_normal(n) * 3)
    # 10: descending ramp (every bucket's max sits in its first stride-row)
    x[10] = -np.arange(n, dtype=np.float32)
    # 11: ascending ramp
    x[11] = np.arange(n, dtype=np.float32)
    check(ref, cuda, x, dtype, B, kp, k)


@pytest.mark.parametrize("levels", [3, 9, 40])
def test_rowthr_ties_vs_old_kernel(cuda, ref, levels):
    """Same answers as the grid-computing row-resident kernel on tied bf16 rows."""
    rng = np.random.default_rng(levels)
    x = rng.integers(-levels, levels + 1, size=(128, 14336)).astype(np.float32) / 4.0
    v, i = check(ref, cuda, x, "bf16", 128, 4, 287)
    xd, _ = dev_input(x, "bf16", cuda)
    with atk._lib.option("no_rowthr", 1):
        v2, i2 = atk.approx_top_k_device(xd, atk.AlgoParams(14336, 128, 4, 287))
    assert np.array_equal(bits(v), bits(v2)) and np.array_equal(u32(i), u32(i2))


def test_rowthr_nan_flag(cuda):
    x = np.random.default_rng(3).standard_normal((8, 14336)).astype(np.float32)
    x[5, 777] = np.nan
    xd, _ = dev_input(x, "bf16", cuda)
    with pytest.raises(ValueError, match="NaN"):
        atk.approx_top_k_device(xd, atk.AlgoParams(14336, 128, 4, 287))

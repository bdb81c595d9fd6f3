"""row_warp_kernel (csrc/rowwarp.cuh) and short_row_kernel (csrc/shortrow.cuh):
approx_top_k for bf16 rows held in shared memory with the guaranteed row
threshold (K-th largest of the B*K' group maxima).  Bit-exact against the reference library (oracle/_ref, the
unmodified atk core: approx_top_k_batch, topk.cpp:238-273) on the C3 shape,
its K' sweep (BASELINE configs[2]), small and odd shapes,
rows built to hit every rare branch (crowded buckets, heavy ties, the exact
in-kernel path, crowded emit bins), and the forced exact path."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
import paper_2506_04165_b200 as atk  # noqa: E402
from paper_2506_04165_b200 import data  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["rowwarp", "short"])
def kernel_path(request, opts):
    """Every test runs on the one-warp-per-row kernel (rowwarp.cuh, B in
    {128, 256, 512}) and on the CTA-per-row kernel (shortrow.cuh); shapes a
    kernel does not take fall through to the other row kernels."""
    if request.param == "short":
        opts("short", 1)
    else:
        opts("rowwarp", 1)
    return request.param


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
    assert np.array_equal(bits(v), bits(rv)), "values differ from the reference"
    assert np.array_equal(u32(i), ri), "indices differ from the reference"
    return v, i


# C3 and its sweep: K' in {1,2,4,8}, B from the planner at r = 0.95 / 0.99
SWEEP = [(4, 128), (1, 3584), (2, 512), (8, 128), (1, 7168), (2, 1024), (4, 256)]

SHAPES = [  # dtype, n, B, kp, k
    *[("bf16", 14336, b, kp, 287) for kp, b in SWEEP],
    ("bf16", 14336, 128, 4, 512),   # K == B*K': every candidate is output
    ("bf16", 14336, 64, 4, 200),
    ("bf16", 8192, 64, 2, 100),
    ("bf16", 2048, 128, 4, 64),
    ("bf16", 1024, 128, 8, 64),     # 8 stride-rows = K': one-row groups
    ("bf16", 4096, 4, 2, 8),        # tiny B
    ("bf16", 1000, 8, 4, 30),       # rows of 2000 B (16-byte multiple), 125 stride-rows
    ("bf16", 24576, 96, 2, 150),    # 256 stride-rows: masks over 8 blocks; B not a power of 2
    ("bf16", 8192, 128, 4, 287),    # 64 stride-rows: two mask words
    ("bf16", 4096, 128, 2, 100),    # 32 stride-rows: one mask word
    ("bf16", 16384, 256, 4, 400),   # 64 stride-rows, 2 chunk columns per lane
    ("bf16", 8192, 512, 1, 200),    # 16 stride-rows, 4 chunk columns per lane
    ("bf16", 14336, 128, 4, 1),     # K = 1
    ("bf16", 14336, 128, 8, 1024),  # K = B*K'
    ("bf16", 1920, 128, 8, 300),    # 15 stride-rows: groups of one or two rows
    ("f32", 4096, 128, 4, 100),
    ("f32", 8192, 64, 2, 100),
    ("f32", 2048, 32, 8, 200),
    ("f32", 8192, 2048, 1, 300),
]


@pytest.mark.parametrize("dtype,n,B,kp,k", SHAPES)
def test_short_normal_vs_reference(cuda, ref, dtype, n, B, kp, k):
    rng = np.random.default_rng(n + 7 * B + kp * 131 + k)
    x = rng.standard_normal((200, n)).astype(np.float32)
    check(ref, cuda, x, dtype, B, kp, k)


@pytest.mark.parametrize("dtype,n,B,kp,k", [s for s in SHAPES if s[1] >= 2048])
def test_short_adversarial_vs_reference(cuda, ref, dtype, n, B, kp, k):
    rng = np.random.default_rng(n + B + kp + k)
    x = rng.standard_normal((16, n)).astype(np.float32)
    nstr = n // B
    x[0] = -1.0                                       # the large values all in bucket 0
    x[0, np.arange(nstr) * B] = 50.0 + np.arange(nstr)
    x[1] = -np.inf                                    # mostly -inf: L = -inf -> exact path
    m = min(n, 3 * k)
    x[1, rng.choice(n, size=m, replace=False)] = rng.standard_normal(m)
    x[2] = -np.inf                                    # all -inf (sentinel semantics)
    x[3] = 1.5                                        # all equal: hit lists overflow
    x[4] = np.where(rng.random(n) < 0.5, 2.0, -2.0)
    x[5] = np.where(rng.random(n) < 0.5, 0.0, -0.0)   # +-0 with a few positives
    x[5, rng.choice(n, size=k // 2, replace=False)] = 1.0
    x[6, rng.choice(n, size=k // 3 + 1, replace=False)] = np.inf
    x[7] = rng.standard_normal(n) * np.float32(1e30) ** rng.random(n)   # wide range
    x[8] = np.round(rng.standard_normal(n) * 3)       # quantised: ties at L
    x[9] = -np.arange(n, dtype=np.float32)
    x[10] = np.arange(n, dtype=np.float32)
    x[11] = np.round(rng.standard_normal(n) * 40) / 8  # ties inside crowded buckets
    x[12, ::B] = 9.0                                  # one bucket full of equal maxima
    x[13] = rng.standard_normal(n) - 10.0             # few large values per stride-row
    for j in range(0, nstr, 2):
        x[13, j * B: j * B + 3] = 5.0 + rng.standard_normal(3)
    check(ref, cuda, x, dtype, B, kp, k)


@pytest.mark.parametrize("levels", [2, 3, 9, 40, 300])
@pytest.mark.parametrize("kp,B", [(4, 128), (1, 3584), (8, 128)])
def test_short_ties_vs_reference(cuda, ref, levels, kp, B):
    rng = np.random.default_rng(levels * 7 + kp)
    x = rng.integers(-levels, levels + 1, size=(64, 14336)).astype(np.float32) / 4.0
    check(ref, cuda, x, "bf16", B, kp, 287)


@pytest.mark.parametrize("dtype,n,B,kp,k", [("bf16", 14336, 128, 4, 287), ("bf16", 14336, 3584, 1, 287),
                                            ("bf16", 14336, 7168, 1, 287), ("f32", 4096, 128, 8, 100)])
def test_short_forced_exact_path(cuda, ref, opts, dtype, n, B, kp, k):
    opts("short_force_slow", 1)
    opts("rowwarp_force_slow", 1)
    x = np.random.default_rng(5).standard_normal((40, n)).astype(np.float32)
    x[3] = np.round(x[3] * 2)
    x[4] = -np.inf
    check(ref, cuda, x, dtype, B, kp, k)


def test_short_nan_raises(cuda):
    x = np.random.default_rng(3).standard_normal((300, 14336)).astype(np.float32)
    x[257, 777] = np.nan
    xd, _ = dev_input(x, "bf16", cuda)
    with pytest.raises(ValueError, match="NaN"):
        atk.approx_top_k_device(xd, atk.AlgoParams(14336, 128, 4, 287))


def test_short_matches_other_row_paths(cuda):
    """Same answers as the row-resident kernel (option no_short=1)."""
    x = np.random.default_rng(11).standard_normal((512, 14336)).astype(np.float32)
    xd, _ = dev_input(x, "bf16", cuda)
    p = atk.AlgoParams(14336, 128, 4, 287)
    v, i = atk.approx_top_k_device(xd, p)
    with atk._lib.option("no_short", 1):
        v2, i2 = atk.approx_top_k_device(xd, p)
    assert np.array_equal(bits(v), bits(v2)) and np.array_equal(u32(i), u32(i2))


@pytest.mark.parametrize("rows", [1, 5, 443, 444, 445, 2000])
def test_short_row_counts(cuda, ref, rows):
    """Persistent grid: fewer rows than CTAs, exactly one wave, ragged waves."""
    x = np.random.default_rng(rows).standard_normal((rows, 14336)).astype(np.float32)
    check(ref, cuda, x, "bf16", 128, 4, 287)

"""row_reg_kernel (csrc/rowreg.cuh): approx_top_k for short bf16 rows with
B = 128, K' = 4 (the C3 shape), one warp per row, the row streamed once from
HBM into registers against a predicted level.  Bit-exact against the
reference library (oracle/_ref, the unmodified atk core: approx_top_k_batch,
topk.cpp:238-273) on every instantiated row length, rows built to hit each
rare branch (misprediction in both directions, crowded buckets, heavy ties,
the exact in-kernel path, the sort instead of the bins), the forced paths and
every CTA size."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
import paper_2506_04165_b200 as atk  # noqa: E402
from paper_2506_04165_b200 import data  # noqa: E402

pytestmark = pytest.mark.gpu

B, KP = 128, 4


def bits(a):
    if isinstance(a, torch.Tensor):
        a = a.detach().cpu().numpy()
    return np.asarray(a, np.float32).view(np.uint32)


def u32(a):
    if isinstance(a, torch.Tensor):
        a = a.detach().cpu().numpy()
    return np.asarray(a).astype(np.uint32)


def check(ref, cuda, x, k):
    b16 = data.f32_to_bf16_bits(x)
    xd = torch.from_numpy(b16.view(np.int16)).to(cuda).view(torch.bfloat16)
    f = data.bf16_bits_to_f32(b16)
    n = x.shape[1]
    before = atk._lib.lib.atkg_launch_count()
    v, i = atk.approx_top_k_device(xd, atk.AlgoParams(n, B, KP, k))
    assert atk._lib.lib.atkg_launch_count() - before == 1, "one kernel per call"
    rv, ri = ref.approx_top_k_batch(f, B, KP, k, lane=B)
    bad = np.nonzero((bits(v) != bits(rv)).any(1) | (u32(i) != ri).any(1))[0]
    assert bad.size == 0, f"rows {bad[:8]} differ from the reference"


# n = 128 S: S = 112 is the unrolled instantiation, every other 8 <= S <= 512 takes the run-time row length
SHAPES = [(14336, 287), (14336, 1), (14336, 512), (14336, 64), (3584, 100), (7168, 287), (16384, 300), (16384, 512),
          (1024, 40), (1152, 64), (11008, 220), (12800, 300), (28672, 287), (65536, 512), (38400, 100),
          (4096, 82), (8192, 164), (12288, 246), (13824, 276)]


@pytest.mark.parametrize("n,k", SHAPES)
def test_rowreg_normal_vs_reference(cuda, ref, n, k):
    x = np.random.default_rng(n + k).standard_normal((700, n)).astype(np.float32)
    check(ref, cuda, x, k)


def adversarial(n, k, seed):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((20, n)).astype(np.float32)
    nstr = n // B
    x[0] = -1.0                                       # the large values all in bucket 0
    x[0, np.arange(nstr) * B] = 50.0 + np.arange(nstr)
    x[1] = -np.inf                                    # mostly -inf: L = -inf -> exact path
    m = min(n, 3 * k)
    x[1, rng.choice(n, size=m, replace=False)] = rng.standard_normal(m)
    x[2] = -np.inf                                    # all -inf (sentinel semantics)
    x[3] = 1.5                                        # all equal: the hit list overflows
    x[4] = np.where(rng.random(n) < 0.5, 2.0, -2.0)
    x[5] = np.where(rng.random(n) < 0.5, 0.0, -0.0)   # +-0 with a few positives
    x[5, rng.choice(n, size=k // 2 + 1, replace=False)] = 1.0
    x[6, rng.choice(n, size=k // 3 + 1, replace=False)] = np.inf
    x[7] = rng.standard_normal(n) * np.float32(1e30) ** rng.random(n)   # wide range: sort, not bins
    x[8] = np.round(rng.standard_normal(n) * 3)       # quantised: ties at L
    x[9] = -np.arange(n, dtype=np.float32)
    x[10] = np.arange(n, dtype=np.float32)
    x[11] = np.round(rng.standard_normal(n) * 40) / 8  # ties inside crowded buckets
    x[12, ::B] = 9.0                                  # one bucket full of equal maxima
    x[13] = rng.standard_normal(n) - 10.0             # few large values per stride-row
    for j in range(0, nstr, 2):
        x[13, j * B: j * B + 3] = 5.0 + rng.standard_normal(3)
    x[14] = -np.abs(x[14])                            # all negative: L < 0
    x[15] = np.where(rng.random(n) < 0.02, 0.0, -1.0) * np.where(rng.random(n) < 0.5, 1.0, -1.0)  # level at +-0
    x[16] = x[16] * 1e-3
    x[17] = x[17] * 1e3
    return x


@pytest.mark.parametrize("n,k", SHAPES)
@pytest.mark.parametrize("warps", [12, 24, 33])
def test_rowreg_adversarial_vs_reference(cuda, ref, opts, n, k, warps):
    opts("rowreg_warps", warps)
    x = adversarial(n, k, n + k)
    # repeated so that every warp meets every kind of row after every other
    check(ref, cuda, np.concatenate([x, x[::-1], x[::3], x]), k)


@pytest.mark.parametrize("levels", [2, 3, 9, 40, 300])
def test_rowreg_ties_vs_reference(cuda, ref, levels):
    rng = np.random.default_rng(levels * 7)
    x = rng.integers(-levels, levels + 1, size=(300, 14336)).astype(np.float32) / 4.0
    check(ref, cuda, x, 287)


@pytest.mark.parametrize("force", [1, 2])
def test_rowreg_forced_paths(cuda, ref, opts, force):
    """1 = every row two-pass, 2 = every row on the exact path, 3 = sorted instead of binned."""
    opts("rowreg_force", force)
    x = np.random.default_rng(5).standard_normal((300, 14336)).astype(np.float32)
    x[3] = np.round(x[3] * 2)
    x[4] = -np.inf
    check(ref, cuda, x, 287)


@pytest.mark.parametrize("margin", [0, 1, 5, 40, 300])
def test_rowreg_prediction_settings(cuda, ref, opts, margin):
    """The prediction only steers speed: any margin below the last row's level is exact."""
    opts("rowreg_margin", margin)
    x = np.random.default_rng(margin).standard_normal((2000, 14336)).astype(np.float32)
    check(ref, cuda, x, 287)


def test_rowreg_scale_changes(cuda, ref):
    """Rows whose level jumps up and down: the prediction fails both ways
    (count short -> two-pass; far too many hits -> two-pass)."""
    rng = np.random.default_rng(9)
    x = rng.standard_normal((1500, 14336)).astype(np.float32)
    scale = np.array([1.0, 100.0, 0.01, 1.0, 1e-4, 3.0, 0.5])[rng.integers(0, 7, size=1500)]
    x *= scale[:, None].astype(np.float32)
    x[::7] -= 5.0
    check(ref, cuda, x, 287)


@pytest.mark.parametrize("robust", [0, 1, 2])
@pytest.mark.parametrize("kind", ["spread", "drift", "negative", "masked", "spikes", "sparse", "halves"])
@pytest.mark.parametrize("n,k", [(14336, 287), (12288, 246)])
def test_rowreg_row_scales(cuda, ref, opts, robust, kind, n, k):
    """Rows of different scales, with the scale-statistic prediction always on
    (1), chosen per CTA (0) and off (2): the level a row passes against only
    steers speed.  spread: scale 2^U(-3,3) per row; drift: scale growing along
    the batch; negative: every value below zero (the level moves against the
    scale); masked: -inf columns (no statistic from them); spikes: a few huge
    magnitudes per row; sparse: mostly zeros (subnormal-free statistic over
    few buckets); halves: two populations of rows."""
    opts("rowreg_robust", robust)
    rng = np.random.default_rng(len(kind) * 131 + robust + n)
    rows = 1800
    x = rng.standard_normal((rows, n)).astype(np.float32)
    if kind == "spread":
        x *= np.exp2(rng.uniform(-3, 3, size=(rows, 1))).astype(np.float32)
    elif kind == "drift":
        x *= np.exp2(np.linspace(-2, 2, rows))[:, None].astype(np.float32)
    elif kind == "negative":
        x = -np.abs(x) * np.exp2(rng.uniform(-2, 2, size=(rows, 1))).astype(np.float32) - 0.01
    elif kind == "masked":
        x *= np.exp2(rng.uniform(-1, 1, size=(rows, 1))).astype(np.float32)
        x[:, rng.choice(n, size=n // 3, replace=False)] = -np.inf
        x[::5, : n // 2] = -np.inf
        x[7] = -np.inf
    elif kind == "spikes":
        for r in range(rows):
            x[r, rng.integers(0, n, size=6)] *= 1e4
    elif kind == "sparse":
        x *= (rng.random((rows, n)) < 0.05)
    elif kind == "halves":
        x[rows // 2:] *= 37.0
        x[::2] *= 0.6
    check(ref, cuda, x, k)


def test_rowreg_nan_raises(cuda):
    x = np.random.default_rng(3).standard_normal((600, 14336)).astype(np.float32)
    x[457, 777] = np.nan
    b16 = data.f32_to_bf16_bits(x)
    xd = torch.from_numpy(b16.view(np.int16)).to(cuda).view(torch.bfloat16)
    with pytest.raises(ValueError, match="NaN"):
        atk.approx_top_k_device(xd, atk.AlgoParams(14336, B, KP, 287))


@pytest.mark.parametrize("rows", [1, 5, 147, 148, 149, 3000])
@pytest.mark.parametrize("warps", [16, 28, 29, 32, 36, 40])
def test_rowreg_row_counts(cuda, ref, opts, rows, warps):
    """One CTA per SM over a contiguous share of the rows: fewer rows than
    CTAs, one row each, ragged shares."""
    opts("rowreg_warps", warps)
    x = np.random.default_rng(rows).standard_normal((rows, 14336)).astype(np.float32)
    check(ref, cuda, x, 287)


def test_rowreg_matches_row_resident(cuda, opts):
    x = np.random.default_rng(11).standard_normal((1024, 14336)).astype(np.float32)
    b16 = data.f32_to_bf16_bits(x)
    xd = torch.from_numpy(b16.view(np.int16)).to(cuda).view(torch.bfloat16)
    p = atk.AlgoParams(14336, B, KP, 287)
    v, i = atk.approx_top_k_device(xd, p)
    opts("rowreg", 0)
    v2, i2 = atk.approx_top_k_device(xd, p)
    assert np.array_equal(bits(v), bits(v2)) and np.array_equal(u32(i), u32(i2))

"""row_max1_kernel (csrc/rowmax1.cuh): approx_top_k with K' = 1 (the original
two-stage algorithm; the baseline of the C3 K' sweep, B = 3584 and 7168) on
the register row stream, with short_row_kernel finishing the rows it leaves.
Bit-exact against the reference library (oracle/_ref: approx_top_k_batch,
topk.cpp:238-273) on normal rows, rows built to hit every branch (ties across
most buckets, -inf rows, level changes), the forced exact path and NaN."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
import paper_2506_04165_b200 as atk  # noqa: E402
from paper_2506_04165_b200 import data  # noqa: E402
from tests.test_gpu_rowreg import adversarial, bits, u32  # noqa: E402

pytestmark = pytest.mark.gpu

SHAPES = [(14336, 3584, 287), (14336, 7168, 287), (14336, 3584, 1), (14336, 7168, 512), (1024, 256, 64),
          (2048, 256, 100), (16384, 2048, 300), (65536, 8192, 400), (512, 128, 128)]


def check(ref, cuda, x, B, k):
    b16 = data.f32_to_bf16_bits(x)
    xd = torch.from_numpy(b16.view(np.int16)).to(cuda).view(torch.bfloat16)
    f = data.bf16_bits_to_f32(b16)
    v, i = atk.approx_top_k_device(xd, atk.AlgoParams(x.shape[1], B, 1, k, 128))
    rv, ri = ref.approx_top_k_batch(f, B, 1, k, lane=128)
    bad = np.nonzero((bits(v) != bits(rv)).any(1) | (u32(i) != ri).any(1))[0]
    assert bad.size == 0, f"rows {bad[:8]} differ from the reference"


@pytest.mark.parametrize("n,B,k", SHAPES)
def test_rowmax1_normal_vs_reference(cuda, ref, n, B, k):
    x = np.random.default_rng(n + B + k).standard_normal((600, n)).astype(np.float32)
    check(ref, cuda, x, B, k)


@pytest.mark.parametrize("n,B,k", [s for s in SHAPES if s[0] >= 2048])
def test_rowmax1_adversarial_vs_reference(cuda, ref, n, B, k):
    x = adversarial(n, min(k, 200), n + k)
    check(ref, cuda, np.concatenate([x, x[::-1], x[::3], x]), B, k)


@pytest.mark.parametrize("levels", [2, 9, 300])
@pytest.mark.parametrize("B", [3584, 7168])
def test_rowmax1_ties_vs_reference(cuda, ref, levels, B):
    rng = np.random.default_rng(levels * 7 + B)
    x = rng.integers(-levels, levels + 1, size=(200, 14336)).astype(np.float32) / 4.0
    check(ref, cuda, x, B, 287)


@pytest.mark.parametrize("B", [3584, 7168])
def test_rowmax1_forced_exact_kernel(cuda, ref, opts, B):
    """Every row through the list and short_row_kernel."""
    opts("rowmax1_force", 1)
    x = np.random.default_rng(5).standard_normal((300, 14336)).astype(np.float32)
    check(ref, cuda, x, B, 287)


@pytest.mark.parametrize("B", [3584, 7168])
def test_rowmax1_scale_changes_and_nan(cuda, ref, B):
    rng = np.random.default_rng(9)
    x = rng.standard_normal((1500, 14336)).astype(np.float32)
    x *= np.array([1.0, 100.0, 0.01, 1.0, 1e-4, 3.0, 0.5])[rng.integers(0, 7, size=1500)][:, None].astype(np.float32)
    x[::7] -= 5.0
    check(ref, cuda, x, B, 287)
    x[457, 777] = np.nan
    b16 = data.f32_to_bf16_bits(x)
    xd = torch.from_numpy(b16.view(np.int16)).to(cuda).view(torch.bfloat16)
    with pytest.raises(ValueError, match="NaN"):
        atk.approx_top_k_device(xd, atk.AlgoParams(14336, B, 1, 287, 128))


def test_rowmax1_matches_short_row_kernel(cuda, opts):
    x = np.random.default_rng(11).standard_normal((1024, 14336)).astype(np.float32)
    b16 = data.f32_to_bf16_bits(x)
    xd = torch.from_numpy(b16.view(np.int16)).to(cuda).view(torch.bfloat16)
    p = atk.AlgoParams(14336, 3584, 1, 287)
    v, i = atk.approx_top_k_device(xd, p)
    opts("rowmax1", 0)
    v2, i2 = atk.approx_top_k_device(xd, p)
    assert np.array_equal(bits(v), bits(v2)) and np.array_equal(u32(i), u32(i2))

"""row_regx_kernel (csrc/rowregx.cuh): the register row stream for the C3 K'
sweep shapes with B K' = 1024 candidates per row (bf16 rows of 14336: K' = 2 /
B = 512, K' = 4 / B = 256, K' = 8 / B = 128).  Bit-exact against the reference
library (oracle/_ref: approx_top_k_batch, topk.cpp:238-273) on normal rows,
rows built to hit every rare branch, heavy ties and the forced paths."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
import paper_2506_04165_b200 as atk  # noqa: E402
from paper_2506_04165_b200 import data  # noqa: E402
from tests.test_gpu_rowreg import adversarial, bits, u32  # noqa: E402

pytestmark = pytest.mark.gpu

N = 14336
CONFIGS = [(2, 512), (4, 256), (8, 128), (2, 1024)]


def check(ref, cuda, x, kp, B, k):
    b16 = data.f32_to_bf16_bits(x)
    xd = torch.from_numpy(b16.view(np.int16)).to(cuda).view(torch.bfloat16)
    f = data.bf16_bits_to_f32(b16)
    before = atk._lib.lib.atkg_launch_count()
    v, i = atk.approx_top_k_device(xd, atk.AlgoParams(N, B, kp, k, 128))
    assert atk._lib.lib.atkg_launch_count() - before == 1, "one kernel per call"
    rv, ri = ref.approx_top_k_batch(f, B, kp, k, lane=128)
    bad = np.nonzero((bits(v) != bits(rv)).any(1) | (u32(i) != ri).any(1))[0]
    assert bad.size == 0, f"rows {bad[:8]} differ from the reference"


@pytest.mark.parametrize("kp,B", CONFIGS)
@pytest.mark.parametrize("k", [287, 1, 64, 1024])
def test_rowregx_normal_vs_reference(cuda, ref, kp, B, k):
    x = np.random.default_rng(kp * 1000 + k).standard_normal((700, N)).astype(np.float32)
    check(ref, cuda, x, kp, B, k)


@pytest.mark.parametrize("kp,B", CONFIGS)
@pytest.mark.parametrize("warps", [16, 28])  # (2, 1024) runs at 16 or 20
def test_rowregx_adversarial_vs_reference(cuda, ref, opts, kp, B, warps):
    opts("rowregx_warps", warps)
    x = adversarial(N, 287, kp + B)
    nstr = N // B
    x[0] = -1.0                                        # the large values all in bucket 0 (of this B)
    x[0, np.arange(nstr) * B] = 50.0 + np.arange(nstr)
    x[12] = np.random.default_rng(1).standard_normal(N)
    x[12, ::B] = 9.0
    check(ref, cuda, np.concatenate([x, x[::-1], x[::3], x]), kp, B, 287)


@pytest.mark.parametrize("kp,B", CONFIGS)
@pytest.mark.parametrize("levels", [2, 9, 300])
def test_rowregx_ties_vs_reference(cuda, ref, kp, B, levels):
    rng = np.random.default_rng(levels * 7 + kp)
    x = rng.integers(-levels, levels + 1, size=(300, N)).astype(np.float32) / 4.0
    check(ref, cuda, x, kp, B, 287)


@pytest.mark.parametrize("kp,B", CONFIGS)
@pytest.mark.parametrize("force", [1, 2])
def test_rowregx_forced_paths(cuda, ref, opts, kp, B, force):
    """1 = every row two-pass, 2 = every row on the exact path."""
    opts("rowreg_force", force)
    x = np.random.default_rng(5).standard_normal((300, N)).astype(np.float32)
    x[3] = np.round(x[3] * 2)
    x[4] = -np.inf
    check(ref, cuda, x, kp, B, 287)


@pytest.mark.parametrize("kp,B", CONFIGS)
def test_rowregx_scale_changes_and_nan(cuda, ref, kp, B):
    rng = np.random.default_rng(9)
    x = rng.standard_normal((1500, N)).astype(np.float32)
    x *= np.array([1.0, 100.0, 0.01, 1.0, 1e-4, 3.0, 0.5])[rng.integers(0, 7, size=1500)][:, None].astype(np.float32)
    x[::7] -= 5.0
    check(ref, cuda, x, kp, B, 287)
    x[457, 777] = np.nan
    b16 = data.f32_to_bf16_bits(x)
    xd = torch.from_numpy(b16.view(np.int16)).to(cuda).view(torch.bfloat16)
    with pytest.raises(ValueError, match="NaN"):
        atk.approx_top_k_device(xd, atk.AlgoParams(N, B, kp, 287, 128))

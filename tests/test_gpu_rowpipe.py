"""GPU parity of the persistent row pipeline (csrc/rowpipe.cuh): bf16 rows in
shared memory, a sampled row threshold L, Alg. 1 over the marks >= L per
bucket, a counting-sort emit; rows that defeat the threshold take the exact
slow path.  Every case is bit-exact against the reference library
(oracle/_ref approx_top_k_batch, /root/reference/proj/core/src/topk.cpp:238-273).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
import paper_2506_04165_b200 as atk  # noqa: E402
from tests.test_gpu_rowthr import check  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _force_rowpipe(monkeypatch):
    """The planner leaves this path opt-in; force it."""
    monkeypatch.setenv("ATKG_ROWPIPE", "1")

SHAPES = [  # n, B, kp, k
    (14336, 128, 4, 287),   # C3 (planner, r = 0.95)
    (14336, 256, 4, 287),   # C3 r = 0.99
    (14336, 128, 8, 287),
    (14336, 128, 2, 200),
    (14336, 128, 1, 100),
    (14336, 256, 2, 500),   # K close to B*K'
    (8192, 128, 4, 512),    # K == B*K'
    (16384, 128, 4, 300),   # 128 stride-rows (both halves full)
    (2048, 128, 4, 64),     # 16 stride-rows
    (4096, 256, 8, 300),
]


@pytest.mark.parametrize("n,B,kp,k", SHAPES)
@pytest.mark.parametrize("rows", [1, 7, 450])
def test_rowpipe_normal_vs_reference(cuda, ref, n, B, kp, k, rows):
    rng = np.random.default_rng(n + B + kp + k + rows)
    x = rng.standard_normal((rows, n)).astype(np.float32)
    check(ref, cuda, x, "bf16", B, kp, k)


@pytest.mark.parametrize("n,B,kp,k", SHAPES[:4])
def test_rowpipe_forced_slow_path(cuda, ref, monkeypatch, n, B, kp, k):
    monkeypatch.setenv("ATKG_PIPE_FORCE_SLOW", "1")
    x = np.random.default_rng(n + kp).standard_normal((40, n)).astype(np.float32)
    check(ref, cuda, x, "bf16", B, kp, k)


@pytest.mark.parametrize("n,B,kp,k", SHAPES)
def test_rowpipe_adversarial_vs_reference(cuda, ref, n, B, kp, k):
    rng = np.random.default_rng(n * 3 + B + kp + k)
    rows = 16
    x = rng.standard_normal((rows, n)).astype(np.float32)
    nstr = n // B
    x[0] = -1.0
    x[0, np.arange(1, nstr, 4) * B] = 50.0 + np.arange(len(range(1, nstr, 4)))
    x[1, :] = rng.standard_normal(n) - 10.0
    for j in range(1, nstr, 2):
        x[1, j * B: j * B + 3] = 5.0 + rng.standard_normal(3)
    x[2] = -np.inf
    x[2, rng.choice(n, size=min(n, 3 * k), replace=False)] = rng.standard_normal(min(n, 3 * k))
    x[3] = -np.inf
    x[4] = 1.5
    x[5] = np.where(rng.random(n) < 0.5, 2.0, -2.0)
    x[6] = np.where(rng.random(n) < 0.5, 0.0, -0.0)
    x[6, rng.choice(n, size=k // 2, replace=False)] = 1.0
    x[7, rng.choice(n, size=k // 3 + 1, replace=False)] = np.inf
    x[8] = rng.standard_normal(n) * np.float32(1e30) ** rng.random(n)
    x[9] = np.round(rng.standard_normal(n) * 3)
    x[10] = -np.arange(n, dtype=np.float32)
    x[11] = np.arange(n, dtype=np.float32)
    x[12] = np.round(rng.standard_normal(n) * 40) / 8
    x[13] = np.inf
    x[14, : n // 2] -= 8.0
    check(ref, cuda, x, "bf16", B, kp, k)


def test_rowpipe_nan_flag(cuda):
    x = np.random.default_rng(3).standard_normal((9, 14336)).astype(np.float32)
    x[5, 777] = np.nan
    from tests.test_gpu_rowthr import dev_input
    xd, _ = dev_input(x, "bf16", cuda)
    with pytest.raises(ValueError, match="NaN"):
        atk.approx_top_k_device(xd, atk.AlgoParams(14336, 128, 4, 287))

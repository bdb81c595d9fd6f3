"""C4 parity: the tcgen05 GEMM and the fused GEMM + stage-1 epilogue.

Reference semantics: mips_fused == mips_unfused (mips.cpp:109-193,
test_mips.cpp:163-193): stage 1 fed with the scores of each query in column
order.  The oracle for the selection is the reference's approx_top_k run on
the exact fp32 scores the epilogue consumed (dumped through `scores`), so the
selection must be bit-exact.  The GEMM itself is checked against an fp32
matmul of the bf16 operands within the fp32-accumulation error bound
2 * Kd * 2^-24 * sum_k |x_k w_k|.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
import paper_2506_04165_b200 as atk  # noqa: E402
from paper_2506_04165_b200 import topk as T  # noqa: E402

pytestmark = pytest.mark.gpu


def bits(a):
    if isinstance(a, torch.Tensor):
        a = a.detach().cpu().numpy()
    return np.asarray(a, np.float32).view(np.uint32)


def u32(a):
    if isinstance(a, torch.Tensor):
        a = a.detach().cpu().numpy()
    return np.asarray(a).astype(np.uint32)


def operands(m, kd, n, seed, cuda, quantized=False):
    g = torch.Generator(device="cpu").manual_seed(seed)
    if quantized:  # small integers: exact integer scores with heavy ties
        x = torch.randint(-2, 3, (m, kd), generator=g).to(torch.bfloat16)
        w = torch.randint(-2, 3, (n, kd), generator=g).to(torch.bfloat16)
    else:
        x = torch.randn((m, kd), generator=g).to(torch.bfloat16)
        w = (0.02 * torch.randn((n, kd), generator=g)).to(torch.bfloat16)
    return x.to(cuda), w.to(cuda)


def check_scores(s, x, w):
    xf, wf = x.float(), w.float()
    ref = xf @ wf.T
    bound = 2.0 * x.shape[1] * 2.0**-24 * (xf.abs() @ wf.abs().T) + 1e-30
    err = (s - ref).abs()
    assert bool((err <= bound).all()), f"max err/bound {float((err / bound).max())}"


GEMM_SHAPES = [(128, 64, 256), (256, 3584, 512), (200, 72, 300), (130, 136, 1000), (1, 8, 5), (384, 1024, 2304)]


@pytest.mark.parametrize("m,kd,n", GEMM_SHAPES)
def test_gemm_bf16_vs_fp32(cuda, m, kd, n):
    x, w = operands(m, kd, n, 11 + m + kd + n, cuda)
    s = T.gemm_bf16_device(x, w)
    torch.cuda.synchronize()
    check_scores(s, x, w)


def test_gemm_rejects_bad_operands(cuda):
    x, w = operands(128, 60, 256, 1, cuda)  # kdim % 8 != 0
    with pytest.raises(ValueError):
        T.gemm_bf16_device(x, w)


# (m, kd, n, B, K', K, lane_multiple): bucket-complete tiles with NB = 4, 2, 1
# buckets per MMA, every specialised K', ragged M
FUSED = [
    (256, 256, 14336, 128, 4, 287, 128),  # C4 shape per row (S=112, NB=2)
    (130, 72, 32768, 512, 4, 128, 128),   # S=64, NB=4
    (128, 64, 4096, 128, 1, 32, 128),     # S=32, NB=4
    (96, 128, 2048, 64, 8, 100, 32),      # S=32, NB=4, K'=8
    (200, 64, 7168, 64, 2, 64, 32),       # S=112, NB=2
    (64, 64, 8192, 32, 8, 64, 32),        # S=256, NB=1
    (130, 64, 14336, 256, 4, 287, 128),   # S=56 (TMEM chunks 8+32+16), NB=4
    (64, 64, 3072, 128, 2, 50, 128),      # S=24
    (64, 64, 1024, 128, 8, 100, 128),     # S=8: every element fills the list
    (70, 64, 144, 3, 2, 5, 1),            # odd B, NB=1, pair splits the bucket
]


def _fused_vs_oracle(cuda, ref_or_port, m, kd, n, B, kp, k, lane, seed, quantized=False):
    x, w = operands(m, kd, n, seed, cuda, quantized)
    p = atk.AlgoParams(n, B, kp, k, lane)
    scores = torch.empty((m, n), dtype=torch.float32, device=cuda)
    v, i = T.fused_gemm_top_k_device(x, w, p, scores=scores)
    plain = T.gemm_bf16_device(x, w)
    torch.cuda.synchronize()
    check_scores(scores, x, w)
    # the epilogue consumed the same fp32 values the plain GEMM produces
    assert np.array_equal(bits(scores), bits(plain))
    s = scores.cpu().numpy()
    rv, ri = ref_or_port.approx_top_k_batch(s, B, kp, k, lane)
    assert np.array_equal(bits(v), bits(rv))
    assert np.array_equal(u32(i), u32(ri))
    # without the dump the result is the same
    v2, i2 = T.fused_gemm_top_k_device(x, w, p)
    assert np.array_equal(bits(v2), bits(v)) and np.array_equal(u32(i2), u32(i))


@pytest.mark.parametrize("m,kd,n,B,kp,k,lane", FUSED)
def test_fused_vs_oracle(cuda, port, m, kd, n, B, kp, k, lane):
    _fused_vs_oracle(cuda, port, m, kd, n, B, kp, k, lane, seed=m * 7 + n)


@pytest.mark.parametrize("m,kd,n,B,kp,k,lane", [(128, 64, 14336, 128, 4, 287, 128), (256, 32, 2048, 64, 8, 100, 32)])
def test_fused_quantized_ties(cuda, port, m, kd, n, B, kp, k, lane):
    """Integer scores: most buckets resolve K'-th-value ties (test_mips.cpp:163-193)."""
    _fused_vs_oracle(cuda, port, m, kd, n, B, kp, k, lane, seed=5, quantized=True)


def test_unfused_fallback_shape(cuda, port):
    """S = n/B > 256 does not fit one MMA tile: plain GEMM + streaming path."""
    _fused_vs_oracle(cuda, port, 130, 64, 65536, 128, 2, 64, 128, seed=3)


def test_fused_nan_rejected(cuda):
    x, w = operands(128, 64, 4096, 9, cuda)
    x[5, 3] = float("inf")
    w[:, 3] = 0  # inf * 0 = NaN in every score of row 5
    with pytest.raises(ValueError, match="NaN"):
        T.fused_gemm_top_k_device(x, w, atk.AlgoParams(4096, 128, 4, 64))


@pytest.mark.slow
def test_c4_full_size(cuda, ref):
    """C4: x bf16 [8192, 3584] ~ N(0,1), W^T bf16 [14336, 3584] ~ N(0, 0.02)."""
    from paper_2506_04165_b200 import data
    xb, _ = data.normal_bf16(data.SEEDS["C4x"], (8192, 3584))
    wb, _ = data.normal_bf16(data.SEEDS["C4w"], (14336, 3584), std=0.02)
    x = torch.from_numpy(xb.view(np.int16)).to(cuda).view(torch.bfloat16)
    w = torch.from_numpy(wb.view(np.int16)).to(cuda).view(torch.bfloat16)
    p = atk.AlgoParams(14336, 128, 4, 287)
    scores = torch.empty((8192, 14336), dtype=torch.float32, device=cuda)
    v, i = T.fused_gemm_top_k_device(x, w, p, scores=scores)
    torch.cuda.synchronize()
    check_scores(scores[:256], x[:256], w)
    rv, ri = ref.approx_top_k_batch(scores.cpu().numpy(), 128, 4, 287)
    assert np.array_equal(bits(v), bits(rv)) and np.array_equal(u32(i), u32(ri))


@pytest.mark.parametrize("m,kd,n,B,kp,k,lane", [FUSED[2], FUSED[4], FUSED[7]])
def test_unfused_alternative_identical(cuda, port, opts, m, kd, n, B, kp, k, lane):
    """Option fused_path=1 (plain GEMM -> grid stage 1 -> stage 2) returns
    the fused epilogue's results bit for bit."""
    x, w = operands(m, kd, n, 17 + m, cuda)
    p = atk.AlgoParams(n, B, kp, k, lane)
    opts("fused_path", 0)
    fv, fi = T.fused_gemm_top_k_device(x, w, p)
    opts("fused_path", 1)
    scores = torch.empty((m, n), dtype=torch.float32, device=cuda)
    uv, ui = T.fused_gemm_top_k_device(x, w, p, scores=scores)
    uv2, ui2 = T.fused_gemm_top_k_device(x, w, p)
    assert torch.equal(uv, fv) and torch.equal(ui, fi)
    assert torch.equal(uv2, fv) and torch.equal(ui2, fi)
    rv, ri = port.approx_top_k_batch(scores.cpu().numpy(), B, kp, k, lane)
    assert np.array_equal(bits(uv), bits(rv)) and np.array_equal(u32(ui), u32(ri))

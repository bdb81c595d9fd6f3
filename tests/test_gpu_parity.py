"""GPU parity: the sm_100a kernels through the C ABI vs the reference.

Every comparison is bit-exact (values as IEEE bits, indices exact): golden
fixtures produced by the reference library itself (tests/golden), the
reference library compiled from source (oracle/_ref) where present, and the
plain-C oracle port.  Full BASELINE sizes are covered by row-by-row equality
with the reference CPU path plus size-independent invariants.
"""
import hashlib

import numpy as np
import pytest

from tests.golden.inputs import INPUTS, build, build_device_input

torch = pytest.importorskip("torch")
import paper_2506_04165_b200 as atk  # noqa: E402

pytestmark = pytest.mark.gpu


def bits(a):
    if isinstance(a, torch.Tensor):
        a = a.detach().cpu().numpy()
    return np.asarray(a, np.float32).view(np.uint32)


def u32(a):
    if isinstance(a, torch.Tensor):
        a = a.detach().cpu().numpy()
    return np.asarray(a).astype(np.uint32)


def to_device(spec, cuda):
    x = build_device_input(spec)
    if x.dtype == np.uint16:
        return torch.from_numpy(x.view(np.int16)).to(cuda).view(torch.bfloat16)
    return torch.from_numpy(np.ascontiguousarray(x)).to(cuda)


def params(spec):
    return atk.AlgoParams(spec["n"], spec["B"], spec["kp"], spec["k"], spec.get("lane", 128))


@pytest.mark.parametrize("name", list(INPUTS))
def test_stage1_grid_golden(cuda, stage_fixtures, name):
    spec = INPUTS[name]
    assert hashlib.sha256(build(spec).tobytes()).hexdigest() == str(stage_fixtures[f"{name}/input_sha"])
    x = to_device(spec, cuda)
    gv, gi = atk.stage1_device(x, params(spec))
    assert np.array_equal(bits(gv), bits(stage_fixtures[f"{name}/grid_v"]))
    assert np.array_equal(u32(gi), stage_fixtures[f"{name}/grid_i"])


@pytest.mark.parametrize("name", list(INPUTS))
def test_approx_top_k_golden(cuda, stage_fixtures, name):
    spec = INPUTS[name]
    x = to_device(spec, cuda)
    v, i = atk.approx_top_k_device(x, params(spec))
    assert np.array_equal(bits(v), bits(stage_fixtures[f"{name}/approx_v"]))
    assert np.array_equal(u32(i), stage_fixtures[f"{name}/approx_i"])


@pytest.mark.parametrize("name", list(INPUTS))
def test_exact_and_recall_golden(cuda, stage_fixtures, name):
    spec = INPUTS[name]
    x = to_device(spec, cuda)
    ev, ei = atk.exact_top_k_device(x, spec["k"])
    assert np.array_equal(bits(ev), bits(stage_fixtures[f"{name}/exact_v"]))
    assert np.array_equal(u32(ei), stage_fixtures[f"{name}/exact_i"])
    ai = stage_fixtures[f"{name}/approx_i"]
    for r in range(ai.shape[0]):
        rec = atk.measure_recall(atk.TopKResult(None, ai[r]), atk.TopKResult(None, u32(ei[r])))
        assert rec == stage_fixtures[f"{name}/recall"][r]


# ---- reference KATs through the device ------------------------------------------
def test_worked_examples(cuda):
    # test_topk.cpp:138-143, 259-264
    g = atk.stage1_partial_reduce(torch.tensor([3, 1, 4, 1, 5, 9, 2, 6], dtype=torch.float32, device=cuda),
                                  atk.AlgoParams(8, 2, 1, 1, 1))
    assert list(g.values.cpu().numpy()) == [5, 9] and list(u32(g.indices)) == [4, 5]
    r = atk.approx_top_k(np.array([5, 1, 7, 3, 9, 2, 8, 4], np.float32), atk.AlgoParams(8, 4, 2, 3, 1))
    assert list(r.values) == [9, 8, 7] and list(r.indices) == [4, 6, 2]


def test_host_drop_in_matches_fixture(cuda, stage_fixtures):
    spec = INPUTS["c1"]
    rows = build(spec)
    res = atk.approx_top_k_batch(rows, rows.shape[0], params(spec), threads=8)
    for r, t in enumerate(res):
        assert np.array_equal(bits(t.values), bits(stage_fixtures["c1/approx_v"][r]))
        assert np.array_equal(t.indices, stage_fixtures["c1/approx_i"][r])
    g = atk.stage1_partial_reduce(rows[3], params(spec))
    assert np.array_equal(bits(g.values), bits(stage_fixtures["c1/grid_v"][3]))
    e = atk.exact_top_k(rows[5], spec["k"])
    assert np.array_equal(e.indices, stage_fixtures["c1/exact_i"][5])


def test_nan_rejected(cuda):
    p = atk.AlgoParams(512, 128, 2, 10)
    x = torch.randn(3, 512, device=cuda)
    x[1, 77] = float("nan")
    with pytest.raises(ValueError, match="input contains NaN"):
        atk.approx_top_k_device(x, p)
    with pytest.raises(ValueError, match="input contains NaN"):
        atk.stage1_device(x, p)
    with pytest.raises(ValueError, match="input contains NaN"):
        atk.exact_top_k_device(x, 5)
    with pytest.raises(ValueError, match="input contains NaN"):
        atk.approx_top_k(x[1].cpu().numpy(), p)


def test_select_candidates_contract(cuda):
    # test_topk.cpp:373-381
    r = atk.select_top_k_candidates(np.array([9, 8, 7, 6], np.float32), np.array([10, 3, 11, 4], np.uint32), 2, 10)
    assert list(r.values) == [8, 6] and list(r.indices) == [3, 4]
    with pytest.raises(ValueError, match="fewer candidates than k"):
        atk.select_top_k_candidates(np.array([9, 8, 7, 6], np.float32), np.array([10, 3, 11, 4], np.uint32), 3, 10)
    # -0.0 comes back as +0.0 (topk.cpp:41-46)
    r = atk.select_top_k_candidates(np.array([-0.0, -1.0], np.float32), np.array([0, 1], np.uint32), 1)
    assert bits(r.values)[0] == 0


def test_select_candidates_random_vs_port(cuda, port):
    rng = np.random.default_rng(3)
    for count in (1, 7, 100, 2048, 5000, 20000, 70000):
        v = rng.integers(-5, 5, count).astype(np.float32)
        v[rng.integers(0, count, max(1, count // 10))] = -0.0
        i = rng.permutation(count).astype(np.uint32)
        k = int(rng.integers(1, min(count, 16384) + 1))
        lim = int(rng.integers(k, count + 1)) if count > k else 2**64 - 1
        try:
            pv, pi = port.select_candidates(v, i, k, lim)
        except ValueError:
            with pytest.raises(ValueError):
                atk.select_top_k_candidates(v, i, k, lim)
            continue
        r = atk.select_top_k_candidates(v, i, k, lim)
        assert np.array_equal(bits(r.values), bits(pv)) and np.array_equal(r.indices, pi)


def test_exact_tie_break(cuda, port):
    # test_topk.cpp:323-371
    from oracle.pyoracle import uniform_below
    base = uniform_below(4242, 41, 900) - np.float32(20)
    row = np.concatenate([base, np.array([0.0, -0.0, np.inf, -np.inf], np.float32)]).astype(np.float32)
    r = atk.exact_top_k(row, 101)
    pv, pi = port.exact_top_k(row, 101)
    assert np.array_equal(r.indices, pi) and np.array_equal(bits(r.values), bits(pv))
    r = atk.exact_top_k(np.array([2, 8, 1], np.float32), 3)
    assert list(r.values) == [8, 2, 1] and list(r.indices) == [1, 0, 2]
    with pytest.raises(ValueError):
        atk.exact_top_k(np.array([1, 2, 3], np.float32), 4)


def test_degenerates_to_exact(cuda):
    # test_topk.cpp:266-286
    from oracle.pyoracle import uniform_below
    for n, b, kp, k in [(256, 256, 1, 17), (256, 32, 8, 50), (512, 64, 9, 100)]:
        row = uniform_below(n + kp, 64, n)
        a = atk.approx_top_k(row, atk.AlgoParams(n, b, kp, k, 1))
        e = atk.exact_top_k(row, k)
        assert np.array_equal(bits(a.values), bits(e.values)) and np.array_equal(a.indices, e.indices)


def test_batch_rows_independent(cuda):
    # test_topk.cpp:399-417: batched == per-row
    p = atk.AlgoParams(512, 16, 2, 24, 1)
    x = torch.rand(9, 512, device=cuda)
    v, i = atk.approx_top_k_device(x, p)
    for r in range(9):
        v1, i1 = atk.approx_top_k_device(x[r:r + 1], p)
        assert torch.equal(v1[0], v[r]) and torch.equal(i1[0], i[r])


def test_accumulator_blocking_invariant(cuda, port):
    # test_topk.cpp:212-236, plus a bucket-aligned fast path and bf16
    for (n, B, kp, lane) in [(3000, 20, 2, 1), (65536, 128, 4, 128), (16384, 64, 9, 1)]:
        rng = np.random.default_rng(n)
        row = (rng.random(n) * 100).astype(np.float32)
        whole = port.stage1(row, B, kp, lane)
        for chunk_seed in (11, 12, 13):
            acc = atk.Stage1Accumulator(atk.AlgoParams(n, B, kp, 1, lane))
            cr = np.random.default_rng(chunk_seed)
            at = 0
            while at < n:
                ln = min(int(cr.integers(1, 97 if n < 10000 else 9000)), n - at)
                acc.consume(torch.from_numpy(row[at:at + ln]).to(cuda))
                at += ln
            assert acc.consumed() == n
            c = acc.candidates()
            assert np.array_equal(bits(c.values), bits(whole[0])) and np.array_equal(c.indices, whole[1])
    acc = atk.Stage1Accumulator(atk.AlgoParams(8, 2, 1, 1, 1))
    acc.consume(np.ones(8, np.float32))
    with pytest.raises(ValueError, match="fed more than n"):
        acc.consume(np.ones(1, np.float32))


@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_slice_summaries_merge(cuda, stage_fixtures, G):
    """Giant-row sharding on one device: G slice summaries -> merge == reference."""
    spec = INPUTS["c5_mini"]
    x = to_device(spec, cuda).reshape(-1)
    p = params(spec)
    n = spec["n"]
    parts = []
    for g in range(G):
        sl = x[g * n // G:(g + 1) * n // G]
        parts.append(atk.stage1_summary_device(sl, g * n // G, p))
    ov, oi, gv, gi = atk.summary_merge_top_k_device(torch.stack(parts), p, want_grid=True)
    assert np.array_equal(bits(gv), bits(stage_fixtures["c5_mini/grid_v"][0]))
    assert np.array_equal(u32(gi), stage_fixtures["c5_mini/grid_i"][0])
    assert np.array_equal(bits(ov), bits(stage_fixtures["c5_mini/approx_v"][0]))
    assert np.array_equal(u32(oi), stage_fixtures["c5_mini/approx_i"][0])


# ---- full BASELINE sizes ---------------------------------------------------------
def _invariants(x_rows_f32, v, i, k):
    v = v.cpu().numpy()
    i = u32(i)
    assert v.shape[1] == k
    assert np.all(v[:, :-1] >= v[:, 1:])
    srt = np.sort(i, axis=1)
    assert np.all(srt[:, 1:] != srt[:, :-1])
    gathered = np.take_along_axis(x_rows_f32, i.astype(np.int64), axis=1)
    assert np.array_equal(gathered + np.float32(0), v + np.float32(0))  # -0.0 vs +0.0 compare equal


@pytest.mark.slow
def test_c2_full_size_vs_reference(cuda, ref):
    from paper_2506_04165_b200 import data
    rows = data.normal_f32(data.SEEDS["C2"], (256, 262144))
    p = atk.AlgoParams(262144, 128, 2, 64)
    v, i = atk.approx_top_k_device(torch.from_numpy(rows).to(cuda), p)
    rv, ri = ref.approx_top_k_batch(rows, 128, 2, 64)
    assert np.array_equal(bits(v), bits(rv)) and np.array_equal(u32(i), ri)
    _invariants(rows, v, i, 64)


@pytest.mark.slow
def test_c3_full_size_vs_reference(cuda, ref):
    from paper_2506_04165_b200 import data
    b, f = data.normal_bf16(data.SEEDS["C3"], (8192, 14336))
    p = atk.AlgoParams(14336, 128, 4, 287)
    xb = torch.from_numpy(b.view(np.int16)).to(cuda).view(torch.bfloat16)
    v, i = atk.approx_top_k_device(xb, p)
    rv, ri = ref.approx_top_k_batch(f, 128, 4, 287)
    assert np.array_equal(bits(v), bits(rv)) and np.array_equal(u32(i), ri)
    _invariants(f, v, i, 287)


def test_sharded_topk_nccl_single_rank(cuda, stage_fixtures):
    """shard.ShardedTopK through a real NCCL group (world 1 on one GPU):
    summary -> all_gather_into_tensor -> merge == the reference result."""
    import os
    import socket

    import torch.distributed as dist

    from paper_2506_04165_b200.shard import ShardedTopK
    spec = INPUTS["c5_mini"]
    x = to_device(spec, cuda).reshape(-1)
    p = params(spec)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    store = dist.TCPStore("127.0.0.1", port, 1, True)
    dist.init_process_group("nccl", store=store, rank=0, world_size=1, device_id=cuda)
    try:
        v, i = ShardedTopK(p)(x)
        torch.cuda.synchronize()
    finally:
        dist.destroy_process_group()
    assert np.array_equal(bits(v), bits(stage_fixtures["c5_mini/approx_v"][0]))
    assert np.array_equal(u32(i), stage_fixtures["c5_mini/approx_i"][0])


@pytest.mark.parametrize("levels,B,kp,k", [(7, 128, 4, 287), (40, 128, 4, 287), (3, 256, 4, 100), (25, 128, 8, 300),
                                           (12, 512, 2, 200), (5, 3584, 1, 287)])
def test_rowres_ties_vs_reference(cuda, ref, levels, B, kp, k):
    """Row-resident path (bf16 rows of 14336) on heavily tied data: the
    closed-form pass 2 (bigs, first c-1 ties, last-tie rule) and the K'-th
    value ties must reproduce the reference bit for bit."""
    rng = np.random.default_rng(levels * 1000 + B)
    rows = 64
    q = rng.integers(-levels, levels + 1, size=(rows, 14336)).astype(np.float32) / 4.0
    q[3, ::7] = -np.inf
    q[5] = 0.0
    q[6, 100:200] = -0.0
    from paper_2506_04165_b200 import data
    bits16 = data.f32_to_bf16_bits(q)
    f = data.bf16_bits_to_f32(bits16)
    xb = torch.from_numpy(bits16.view(np.int16)).to(cuda).view(torch.bfloat16)
    p = atk.AlgoParams(14336, B, kp, k)
    v, i = atk.approx_top_k_device(xb, p)
    rv, ri = ref.approx_top_k_batch(f, B, kp, k)
    assert np.array_equal(bits(v), bits(rv)) and np.array_equal(u32(i), ri)
    gv, gi = atk.stage1_device(xb, p)
    rg = [ref.stage1(f[r], B, kp) for r in range(4)]
    for r in range(4):
        assert np.array_equal(bits(gv[r]), bits(rg[r][0])) and np.array_equal(u32(gi[r]), rg[r][1])


@pytest.mark.parametrize("count", [129, 300, 512, 700, 1024])
def test_select_candidates_rank_path_vs_port(cuda, port, count):
    """Stage 2 through the counting-sort rank kernel (128 < count <= 1024):
    ties, -0.0, -inf sentinels, index_limit drops, quantised values."""
    rng = np.random.default_rng(count)
    cases = []
    v = rng.standard_normal(count).astype(np.float32)
    cases.append((v, rng.permutation(count).astype(np.uint32)))
    v = rng.integers(-3, 4, count).astype(np.float32)
    v[rng.integers(0, count, count // 8)] = -0.0
    cases.append((v, rng.permutation(count).astype(np.uint32)))
    v = rng.standard_normal(count).astype(np.float32)
    v[: count // 3] = -np.inf
    i = rng.permutation(count).astype(np.uint32)
    i[: count // 3] = 0  # duplicate sentinel keys {-inf, 0}
    cases.append((v, i))
    v = (rng.standard_normal(count) * np.float32(1e30) ** rng.random(count)).astype(np.float32)
    cases.append((v, rng.permutation(count).astype(np.uint32)))
    for v, i in cases:
        for k in (1, min(count, 64), min(count, 287), count):
            for lim in (2**64 - 1, int(count * 0.9)):
                try:
                    pv, pi = port.select_candidates(v, i, k, lim)
                except ValueError:
                    with pytest.raises(ValueError):
                        atk.select_top_k_candidates(v, i, k, lim)
                    continue
                r = atk.select_top_k_candidates(v, i, k, lim)
                assert np.array_equal(bits(r.values), bits(pv)) and np.array_equal(r.indices, pi)


# ---- k above one CTA's shared-memory sort (the reference takes any k <= n) ----
@pytest.mark.parametrize("n,k", [(1 << 18, 20000), (1 << 20, 65536), (100000, 16385)])
def test_exact_top_k_large_k(cuda, ref, n, k):
    import paper_2506_04165_b200 as atk
    x = np.random.default_rng(k).standard_normal((2, n)).astype(np.float32)
    x[1, ::7] = np.round(x[1, ::7])  # ties
    v, i = atk.exact_top_k_device(torch.from_numpy(x).to(cuda), k)
    for r in range(2):
        ev, ei = ref.exact_top_k(x[r], k)
        assert np.array_equal(bits(v[r]), bits(ev)) and np.array_equal(u32(i[r]), ei)


@pytest.mark.parametrize("n,B,kp,k", [(1 << 20, 8192, 4, 20000), (1 << 19, 16384, 2, 32768)])
def test_approx_top_k_large_k(cuda, ref, n, B, kp, k):
    import paper_2506_04165_b200 as atk
    x = np.random.default_rng(n + k).standard_normal((2, n)).astype(np.float32)
    v, i = atk.approx_top_k_device(torch.from_numpy(x).to(cuda), atk.AlgoParams(n, B, kp, k))
    rv, ri = ref.approx_top_k_batch(x, B, kp, k)
    assert np.array_equal(bits(v), bits(rv)) and np.array_equal(u32(i), ri)


def test_select_candidates_large_k(cuda, ref):
    import paper_2506_04165_b200 as atk
    rng = np.random.default_rng(5)
    vals = rng.standard_normal(50000).astype(np.float32)
    vals[::5] = 1.0
    idx = rng.permutation(200000)[:50000].astype(np.uint32)
    ov, oi = atk.select_candidates_device(torch.from_numpy(vals).to(cuda)[None, :],
                                          torch.from_numpy(idx.view(np.int32)).to(cuda)[None, :], 30000,
                                          index_limit=150000)
    rv, ri = ref.select_candidates(vals, idx, 30000, 150000)
    assert np.array_equal(bits(ov[0]), bits(rv)) and np.array_equal(u32(oi[0]), ri)


@pytest.mark.parametrize("target,kps", [(0.95, (1, 2, 4, 8)), (0.99, (2,))])
def test_approx_top_k_at_recall(cuda, ref, target, kps):
    """Recall target in: the plan equals the reference planner's
    and the rows equal the reference approx_top_k_batch with that plan."""
    import paper_2506_04165_b200 as atk
    from paper_2506_04165_b200 import data
    n, k, rows = 14336, 287, 32
    req = atk.PlanRequest(n, k, target, list(kps), 128, 0)
    pl = ref.select_parameters(n, k, target, kps, 128, 0)
    x = data.normal_f32(77, (rows, n))
    plan, res = atk.approx_top_k_at_recall(x, rows, req)
    assert (plan.local_k, plan.num_buckets) == (pl.local_k, pl.num_buckets)
    assert plan.estimated_recall.value == pl.recall
    rv, ri = ref.approx_top_k_batch(x, pl.num_buckets, pl.local_k, k)
    for r in range(rows):
        assert np.array_equal(bits(res[r].values), bits(rv[r])) and np.array_equal(u32(res[r].indices), ri[r])
    bits16, f = data.normal_bf16(78, (rows, n))
    xd = torch.from_numpy(bits16.view(np.int16)).to(cuda).view(torch.bfloat16)
    plan2, (v, i) = atk.approx_top_k_at_recall(xd, rows, req)
    rv, ri = ref.approx_top_k_batch(f, pl.num_buckets, pl.local_k, k)
    assert plan2.num_buckets == pl.num_buckets
    assert np.array_equal(bits(v), bits(rv)) and np.array_equal(u32(i), ri)

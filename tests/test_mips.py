"""fp32 MIPS workload against the reference's mips.cpp.

* atkg_mips_score is bit-identical to atk::score_block (mips.cpp:57-91),
  including dims that are not a multiple of the 32-wide slice and ragged tiles.
* mips_unfused / mips_fused return the reference's mips_fused results bit for
  bit, with num_buckets that does not divide the database rows (padded -inf
  columns dropped before stage 2), and the reference's stats.
* validate_mips_request messages are the reference's (CPU).
"""
from __future__ import annotations

import numpy as np
import pytest


def _ds(rows, dims, seed, integer=False):
    import paper_2506_04165_b200 as atk
    rng = np.random.default_rng(seed)
    x = rng.integers(-3, 4, rows * dims).astype(np.float32) if integer else \
        rng.standard_normal(rows * dims).astype(np.float32)
    return atk.VectorDataset(rows, dims, x)


def test_validate_messages():
    import paper_2506_04165_b200 as atk
    db, q = _ds(1000, 16, 0), _ds(4, 16, 1)
    ok = atk.AlgoParams(n=1000, num_buckets=128, local_k=2, global_k=16)
    atk.validate_mips_request(db, q, ok)
    cases = [
        (db, _ds(4, 8, 1), ok, "mips: database/query dims differ"),
        (atk.VectorDataset(0, 16, np.zeros(0, np.float32)), q, ok, "mips: database must not be empty"),
        (db, atk.VectorDataset(0, 16, np.zeros(0, np.float32)), ok, "mips: queries must not be empty"),
        (db, q, atk.AlgoParams(n=999, num_buckets=128, local_k=2, global_k=16), "mips: params.n must equal database rows"),
        (_ds(100, 16, 0), q, atk.AlgoParams(n=100, num_buckets=128, local_k=1, global_k=101),
         "mips: global_k exceeds database rows"),
    ]
    for d, qq, p, msg in cases:
        with pytest.raises(ValueError, match=f"^{msg}$"):
            atk.validate_mips_request(d, qq, p)
    with pytest.raises(ValueError, match="^mips: block_cols must be a multiple or a divisor of num_buckets$"):
        atk.mips_fused(db, q, ok, 100)
    assert atk.default_block_cols(ok) == 4096 and \
        atk.default_block_cols(atk.AlgoParams(n=1, num_buckets=384)) == 4224


@pytest.mark.gpu
@pytest.mark.parametrize("b,n,d", [(1, 1, 1), (7, 130, 33), (70, 1000, 128), (65, 4097, 100)])
def test_score_block_bit_exact(cuda, ref, b, n, d):
    import torch
    from paper_2506_04165_b200.mips import score_block_device
    q, db = _ds(b, d, 2).matrix(), _ds(n, d, 3).matrix()
    got = score_block_device(torch.from_numpy(q).to(cuda), torch.from_numpy(db).to(cuda), n + 5).cpu().numpy()
    want = ref.score_block(q, db, 0, n)
    assert np.array_equal(got[:, :n].view(np.uint32), np.ascontiguousarray(want[:, :n]).view(np.uint32))
    assert np.all(got[:, n:] == -np.inf)


@pytest.mark.gpu
@pytest.mark.parametrize("rows,b,nb,kp,k,integer", [(1000, 9, 128, 2, 16, False), (4096, 33, 256, 1, 64, False),
                                                     (5000, 17, 512, 4, 100, True), (129, 3, 128, 3, 129, False)])
def test_mips_matches_reference(cuda, ref, rows, b, nb, kp, k, integer):
    import paper_2506_04165_b200 as atk
    db, q = _ds(rows, 64, 10 + rows, integer), _ds(b, 64, 20 + b, integer)
    p = atk.AlgoParams(n=rows, num_buckets=nb, local_k=kp, global_k=k)
    rv, ri = ref.mips_fused(db.matrix(), q.matrix(), nb, kp, k)
    for res in (atk.mips_unfused(db, q, p, device=cuda), atk.mips_fused(db, q, p, atk.default_block_cols(p), device=cuda)):
        assert len(res.per_query) == b
        for i, t in enumerate(res.per_query):
            assert np.array_equal(t.values.view(np.uint32), rv[i].view(np.uint32)), i
            assert np.array_equal(t.indices, ri[i]), i
    np_ = (rows + nb - 1) // nb * nb
    st = atk.mips_fused(db, q, p, nb, device=cuda).stats
    assert (st.padded_n, st.blocks, st.score_buffer_bytes) == (np_, np_ // nb, b * nb * 4)
    assert atk.mips_unfused(db, q, p, device=cuda).stats.score_buffer_bytes == b * np_ * 4

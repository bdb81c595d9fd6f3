"""Recall simulation against the reference's simulate.cpp.

* synth_distinct rows are bit-identical to the reference's synth_distinct_row
  (dataset.cpp:132-150), via oracle/_ref and via the pinned oracle port's
  Fisher-Yates (atk_oracle.c, orc_shuffled_iota on derive_seed(seed, r)).
* simulate_recall_many (GPU top-k) returns the reference's mean and stddev
  exactly (same hits per run, same Welford order), for several configs that
  share n and for a single config.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest


def _ref_row(lib, n, seed, r):
    lib.ref_synth_distinct_row.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_void_p]
    out = np.empty(n, np.float32)
    assert lib.ref_synth_distinct_row(n, seed, r, out.ctypes.data) == 0
    return out


def ref_simulate(lib, configs, runs, seed, threads=4):
    lib.ref_simulate_recall_many.argtypes = [C.c_void_p, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint32,
                                             C.c_void_p, C.c_void_p]
    cfg = np.ascontiguousarray([[c.n, c.num_buckets, c.local_k, c.global_k, c.lane_multiple]
                                for c in configs], np.uint64)
    mean, sd = np.empty(len(configs)), np.empty(len(configs))
    rc = lib.ref_simulate_recall_many(cfg.ctypes.data, len(configs), runs, seed, threads,
                                      mean.ctypes.data, sd.ctypes.data)
    assert rc == 0
    return mean, sd


@pytest.mark.parametrize("n,seed", [(1, 3), (2, 0), (1000, 7), (65536, 12345)])
def test_synth_distinct_matches_reference(ref, n, seed):
    import paper_2506_04165_b200 as atk
    rows = atk.synth_distinct(5, n, seed, first_row=3, threads=3)
    for r in range(5):
        assert np.array_equal(rows[r], _ref_row(ref.lib, n, seed, 3 + r))
    assert np.array_equal(np.sort(rows[0]), np.arange(1, n + 1, dtype=np.float32))


def test_synth_distinct_matches_port(port):
    import paper_2506_04165_b200 as atk
    n, seed = 4096, 99
    row = atk.synth_distinct_row(n, seed, 11)
    want = np.empty(n, np.float32)
    port.lib.orc_shuffled_iota(n, port.lib.orc_derive_seed(seed, 11), want)
    assert np.array_equal(row, want)


def test_synth_and_simulate_argument_errors():
    import paper_2506_04165_b200 as atk
    with pytest.raises(ValueError, match=r"^synth_distinct: n must be >= 1$"):
        atk.synth_distinct(1, 0, 0)
    with pytest.raises(ValueError, match=r"^synth_distinct: n must be <= 2\^24 so values stay fp32-exact$"):
        atk.synth_distinct(1, (1 << 24) + 1, 0)
    p = atk.AlgoParams(n=4096, num_buckets=256, local_k=2, global_k=64)
    with pytest.raises(ValueError, match="^simulate: no configurations$"):
        atk.simulate_recall_many([], 4, 0)
    with pytest.raises(ValueError, match="^simulate: runs must be >= 1$"):
        atk.simulate_recall_many([p], 0, 0)
    q = atk.AlgoParams(n=8192, num_buckets=256, local_k=2, global_k=64)
    with pytest.raises(ValueError, match="^simulate: configurations must share n$"):
        atk.simulate_recall_many([p, q], 4, 0)
    with pytest.raises(ValueError, match="^num_buckets must divide n$"):
        atk.simulate_recall_many([atk.AlgoParams(n=4096, num_buckets=384, local_k=1, global_k=8)], 4, 0)


@pytest.mark.gpu
def test_simulate_many_matches_reference(cuda, ref):
    import paper_2506_04165_b200 as atk
    n = 16384
    configs = [atk.AlgoParams(n=n, num_buckets=128, local_k=1, global_k=64),
               atk.AlgoParams(n=n, num_buckets=256, local_k=2, global_k=64),
               atk.AlgoParams(n=n, num_buckets=128, local_k=4, global_k=128),
               atk.AlgoParams(n=n, num_buckets=512, local_k=1, global_k=16)]
    got = atk.simulate_recall_many(configs, 96, 2024, threads=8, device=cuda)
    mean, sd = ref_simulate(ref.lib, configs, 96, 2024)
    for c, st in enumerate(got):
        assert st.runs == 96
        assert st.mean_recall == mean[c] and st.stddev == sd[c], (c, st, mean[c], sd[c])


@pytest.mark.gpu
def test_simulate_single_and_batched_runs(cuda, ref):
    """One run (stddev 0) and a run count over several generation batches (n = 2^20 -> 64 rows/batch)."""
    import paper_2506_04165_b200 as atk
    p = atk.AlgoParams(n=4096, num_buckets=128, local_k=2, global_k=32)
    st = atk.simulate_recall(p, 1, 5, device=cuda)
    mean, sd = ref_simulate(ref.lib, [p], 1, 5)
    assert (st.mean_recall, st.stddev) == (mean[0], 0.0) and sd[0] == 0.0
    big = atk.AlgoParams(n=1 << 20, num_buckets=1024, local_k=1, global_k=256)
    st = atk.simulate_recall(big, 130, 77, threads=16, device=cuda)
    mean, sd = ref_simulate(ref.lib, [big], 130, 77, threads=16)
    assert (st.mean_recall, st.stddev) == (mean[0], sd[0])


@pytest.mark.gpu
@pytest.mark.parametrize("n,seed,first", [(1, 3, 0), (2, 0, 5), (1000, 7, 1), (4096, 2**63 + 5, 9), (65536, 12345, 100)])
def test_synth_distinct_device_bit_exact(cuda, n, seed, first):
    import paper_2506_04165_b200 as atk
    rows = 37
    d = atk.synth_distinct_device(rows, n, seed, first_row=first, device=cuda).cpu().numpy()
    h = atk.synth_distinct(rows, n, seed, first_row=first, threads=8)
    assert np.array_equal(d, h)


@pytest.mark.gpu
def test_synth_distinct_device_limits(cuda):
    import paper_2506_04165_b200 as atk
    with pytest.raises(NotImplementedError, match="n must be <= 2\\^16"):
        atk.synth_distinct_device(1, 65537, 0, device=cuda)
    with pytest.raises(ValueError, match="^synth_distinct: n must be >= 1$"):
        atk.synth_distinct_device(1, 0, 0, device=cuda)


@pytest.mark.gpu
def test_simulate_device_and_host_generation_agree(cuda, ref, opts):
    import paper_2506_04165_b200 as atk
    configs = [atk.AlgoParams(n=65536, num_buckets=256, local_k=2, global_k=64),
               atk.AlgoParams(n=65536, num_buckets=512, local_k=1, global_k=128)]
    dev = atk.simulate_recall_many(configs, 300, 31, device=cuda)
    opts("sim_host_gen", 1)
    host = atk.simulate_recall_many(configs, 300, 31, device=cuda)
    mean, sd = ref_simulate(ref.lib, configs, 300, 31)
    for c in range(2):
        assert (dev[c].mean_recall, dev[c].stddev) == (host[c].mean_recall, host[c].stddev) == (mean[c], sd[c])

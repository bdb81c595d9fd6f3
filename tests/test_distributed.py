"""Sharded giant-row path (C5) under torch.distributed.

The exchange logic of paper_2506_04165_b200.shard.ShardedTopK (slice plan,
summary all-gather in rank order, merge, stage 2) runs here with the gloo
backend on CPU, world sizes 2 and 3, 127.0.0.1 rendezvous.  The per-rank
reduce and the merge are the host build of the same Summ<K'> code the kernels
run (tests/emu); stage 2 is the oracle port.  The result must equal the
reference approx_top_k on the whole row bit for bit.  On the GPU the same
class runs with NCCL and the CUDA kernels (bench.py --config C5 --gpus N).
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2506_04165_b200.shard import ShardedTopK, slice_bounds  # noqa: E402


def test_slice_bounds_partition():
    for n, B, world in [(1 << 20, 256, 8), (3 * 65536, 128, 2), (4096 * 3, 4096, 5), (1536, 128, 4)]:
        spans = [slice_bounds(n, B, world, r) for r in range(world)]
        assert spans[0][0] == 0
        for (s0, l0), (s1, _) in zip(spans, spans[1:]):
            assert s0 + l0 == s1
        assert sum(length for _, length in spans) == n
        assert all(s % B == 0 and length % B == 0 for s, length in spans)
    assert slice_bounds(1 << 30, 256, 8, 3) == (3 << 27, 1 << 27)
    with pytest.raises(ValueError):
        slice_bounds(1000, 128, 2, 0)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, emu_path, n, B, kp, k, seed, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import pyoracle as O
        from paper_2506_04165_b200 import AlgoParams, data
        from tests.conftest import load_emu
        emu = load_emu(emu_path)
        port_be = O.port()
        p = AlgoParams(n, B, kp, k, 1)

        def summarize(x, offset, params, status):
            xs = np.ascontiguousarray(x.numpy(), np.float32)
            words = np.empty((2 * kp + 2) * B, np.uint32)
            nan = C.c_uint32()
            assert emu.emu_slice_summary(xs, xs.size, offset, B, kp, words, C.byref(nan)) == 0
            status |= int(nan.value != 0)
            return torch.from_numpy(words.view(np.int32))

        def merge(summaries, params):
            w = np.ascontiguousarray(summaries.numpy()).view(np.uint32).reshape(-1)
            gv = np.empty(kp * B, np.float32)
            gi = np.empty(kp * B, np.uint32)
            assert emu.emu_merge_summaries(w, summaries.shape[0], B, kp, gv, gi) == 0
            filled = min(kp, n // B) * B
            return port_be.select_candidates(gv[:filled], gi[:filled], k)

        sh = ShardedTopK(p, summarize=summarize, merge=merge)
        start, length = sh.bounds()
        if start % 65536 == 0:
            x = data.normal_f32_range(seed, start, length)
        else:
            x = data.normal_f32(seed, (n,))[start:start + length]
        v, i = sh(torch.from_numpy(np.ascontiguousarray(x)))
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), v=np.asarray(v), i=np.asarray(i), start=start,
                 length=length)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,B,kp,k", [(2, 3 * 65536, 128, 4, 100), (3, 4 * 65536, 256, 8, 256),
                                           (2, 128 * 37, 128, 2, 40), (3, 64 * 90, 64, 1, 30)])
def test_sharded_row_gloo_matches_reference(emu, port, tmp_path, world, n, B, kp, k):
    from paper_2506_04165_b200 import data
    from tests.conftest import EMU_LIB
    seed = 17 + world
    mp.spawn(_worker, args=(world, _free_port(), EMU_LIB, n, B, kp, k, seed, str(tmp_path)), nprocs=world,
             join=True)
    row = data.normal_f32(seed, (n,))
    rv, ri = port.approx_top_k(row, B, kp, k, 1)
    spans = []
    for r in range(world):
        d = np.load(tmp_path / f"r{r}.npz")
        assert np.array_equal(np.asarray(d["v"], np.float32).view(np.uint32), np.asarray(rv, np.float32).view(np.uint32))
        assert np.array_equal(np.asarray(d["i"]).astype(np.uint32), np.asarray(ri).astype(np.uint32))
        spans.append((int(d["start"]), int(d["length"])))
    assert sum(length for _, length in spans) == n


def test_range_generator_matches_full_stream():
    from paper_2506_04165_b200 import data
    full = data.normal_f32(9, (5 * 65536,))
    part = data.normal_f32_range(9, 2 * 65536, 3 * 65536 - 10)
    assert np.array_equal(part, full[2 * 65536:5 * 65536 - 10])

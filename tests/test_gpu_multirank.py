"""The giant-row path (C5) with the real CUDA kernels.

* the full BASELINE C5 row (fp32 1 x 2^30, K=1024, K'=8, B=256 from the
  planner) on one GPU, bit-exact against the reference library
  (oracle/_ref approx_top_k_batch, topk.cpp:238-273; ~12 s of CPU);
* the same row cut into 8 slice summaries (atkg_stage1_summary) merged in
  index order (atkg_summary_merge_top_k): the N = 8 data path on one GPU;
* 2- and 3-process groups (gloo, 127.0.0.1) whose ranks all run the real
  summary / merge kernels on cuda:0 and exchange the summaries through
  shard.ShardedTopK's all-gather (host copies: gloo moves CPU tensors), incl.
  a NaN in one rank's slice, which every rank must report.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

pytestmark = pytest.mark.gpu


def bits(a):
    if isinstance(a, torch.Tensor):
        a = a.detach().cpu().numpy()
    return np.asarray(a, np.float32).view(np.uint32)


def u32(a):
    if isinstance(a, torch.Tensor):
        a = a.detach().cpu().numpy()
    return np.asarray(a).astype(np.uint32)


@pytest.fixture(scope="module")
def c5_row():
    from paper_2506_04165_b200 import data
    return data.normal_f32(data.SEEDS["C5"], (1 << 30,))


def test_c5_full_row_vs_reference(cuda, ref, c5_row):
    import paper_2506_04165_b200 as atk
    n, B, kp, k = 1 << 30, 256, 8, 1024
    xd = torch.from_numpy(c5_row).to(cuda)
    v, i = atk.approx_top_k_device(xd.view(1, -1), atk.AlgoParams(n, B, kp, k))
    rv, ri = ref.approx_top_k_batch(c5_row[None, :], B, kp, k, threads=1)
    assert np.array_equal(bits(v[0]), bits(rv[0])) and np.array_equal(u32(i[0]), ri[0])
    # the 8-GPU data path on one GPU: 8 slice summaries, merged in index order
    from paper_2506_04165_b200.shard import slice_bounds
    p = atk.AlgoParams(n, B, kp, k)
    summ = []
    for g in range(8):
        s0, ln = slice_bounds(n, B, 8, g)
        summ.append(atk.stage1_summary_device(xd[s0:s0 + ln], s0, p))
    sv, si = atk.summary_merge_top_k_device(torch.stack(summ), p)
    assert np.array_equal(bits(sv), bits(rv[0])) and np.array_equal(u32(si), ri[0])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, B, kp, k, seed, nan_at, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2506_04165_b200 as atk
        from paper_2506_04165_b200 import data
        from paper_2506_04165_b200.shard import ShardedTopK
        dev = torch.device("cuda:0")
        p = atk.AlgoParams(n, B, kp, k)

        def summarize(x, offset, params, status):  # the real summary kernel; the exchange moves host copies
            st = torch.zeros(1, dtype=torch.int32, device=dev)
            s = atk.stage1_summary_device(x.to(dev), offset, params, status=st)
            torch.cuda.synchronize(dev)
            status |= int(st.item())
            return s.cpu()

        def merge(summaries, params):
            v, i = atk.summary_merge_top_k_device(summaries.to(dev), params)
            return v.cpu(), i.cpu()

        sh = ShardedTopK(p, summarize=summarize, merge=merge)
        start, length = sh.bounds()
        x = data.normal_f32_range(seed, start, length)
        if nan_at is not None and start <= nan_at < start + length:
            x[nan_at - start] = np.nan
        try:
            v, i = sh(torch.from_numpy(x))
            np.savez(os.path.join(out_dir, f"r{rank}.npz"), v=v.numpy(), i=i.numpy(), err="")
        except ValueError as e:
            np.savez(os.path.join(out_dir, f"r{rank}.npz"), v=np.zeros(0), i=np.zeros(0), err=str(e))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,B,kp,k", [(2, 1 << 22, 256, 8, 1024), (3, 3 << 20, 128, 2, 64),
                                           (2, 1 << 20, 128, 4, 300)])
def test_sharded_real_kernels_match_reference(cuda, ref, tmp_path, world, n, B, kp, k):
    from paper_2506_04165_b200 import data
    seed = 31 + world
    mp.spawn(_worker, args=(world, _free_port(), n, B, kp, k, seed, None, str(tmp_path)), nprocs=world, join=True)
    row = data.normal_f32(seed, (n,))
    rv, ri = ref.approx_top_k_batch(row[None, :], B, kp, k, threads=1)
    for r in range(world):
        d = np.load(tmp_path / f"r{r}.npz")
        assert str(d["err"]) == ""
        assert np.array_equal(bits(d["v"]), bits(rv[0])) and np.array_equal(u32(d["i"]), ri[0])


def test_sharded_nan_in_one_slice_raises_on_every_rank(cuda, tmp_path):
    n, B, kp, k, world = 3 << 20, 256, 8, 1024, 3
    mp.spawn(_worker, args=(world, _free_port(), n, B, kp, k, 5, (2 << 20) + 77, str(tmp_path)), nprocs=world,
             join=True)
    for r in range(world):
        d = np.load(tmp_path / f"r{r}.npz")
        assert "NaN" in str(d["err"]), f"rank {r} did not report the NaN"


# ---- threshold-stream slice payloads (the default exchange) ---------------
PAYLOAD_CASES = [  # dtype, n, B, kp, k
    ("f32", 1 << 22, 256, 8, 1024),
    ("f32", 1 << 20, 128, 2, 64),
    ("bf16", 1 << 21, 128, 4, 300),
    ("f32", 3 << 18, 512, 1, 40),
]


def _dev(x, dtype, cuda):
    from paper_2506_04165_b200 import data
    if dtype == "bf16":
        b16 = data.f32_to_bf16_bits(x)
        return torch.from_numpy(b16.view(np.int16)).to(cuda).view(torch.bfloat16), data.bf16_bits_to_f32(b16)
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(cuda), np.ascontiguousarray(x, np.float32)


@pytest.mark.parametrize("parts", [1, 2, 3, 8])
@pytest.mark.parametrize("dtype,n,B,kp,k", PAYLOAD_CASES)
def test_slice_payloads_merge_to_reference(cuda, ref, parts, dtype, n, B, kp, k):
    """G slice payloads computed on one GPU, merged: bit-exact and settled
    without the exact path (the N-GPU data path, emulated)."""
    import paper_2506_04165_b200 as atk
    from paper_2506_04165_b200.shard import slice_bounds
    x = np.random.default_rng(n + parts).standard_normal(n).astype(np.float32)
    xd, f = _dev(x, dtype, cuda)
    p = atk.AlgoParams(n, B, kp, k, min(B, 128))
    pays = []
    for g in range(parts):
        s0, ln = slice_bounds(n, B, parts, g, align=B)
        pays.append(atk.slice_payload_device(xd[s0:s0 + ln], s0, p, parts))
    v, i, gate = atk.payload_merge_top_k_device(torch.stack(pays), p)
    assert int(gate.item()) == 0
    rv, ri = ref.approx_top_k_batch(f[None, :], B, kp, k, lane=min(B, 128), threads=1)
    assert np.array_equal(bits(v), bits(rv[0])) and np.array_equal(u32(i), ri[0])


def test_payload_gate_on_unsettled_rows(cuda):
    """Rows the threshold cannot settle (a ramp inside one bucket's slice,
    all equal) set the gate instead of answering."""
    import paper_2506_04165_b200 as atk
    n, B, kp, k = 1 << 20, 128, 2, 64
    p = atk.AlgoParams(n, B, kp, k)
    x = np.full(n, 1.5, np.float32)
    xd = torch.from_numpy(x).to(cuda)
    pays = [atk.slice_payload_device(xd[g * n // 2:(g + 1) * n // 2], g * n // 2, p, 2) for g in range(2)]
    _, _, gate = atk.payload_merge_top_k_device(torch.stack(pays), p)
    assert int(gate.item()) != 0


@pytest.mark.parametrize("force", [False, True])
@pytest.mark.parametrize("dtype,n,B,kp,k", PAYLOAD_CASES[:3])
def test_c_abi_sharded_entry_one_rank(cuda, ref, opts, force, dtype, n, B, kp, k):
    """atkg_sharded_approx_top_k over a one-rank NCCL communicator made by the
    library's own NCCL: payload path, and the exact fallback when forced."""
    import paper_2506_04165_b200 as atk
    if force:
        opts("st_force_slow", 1)
    x = np.random.default_rng(k).standard_normal(n).astype(np.float32)
    xd, f = _dev(x, dtype, cuda)
    comm = atk.topk.NcclComm(1, atk.topk.NcclComm.unique_id(), 0)
    try:
        v, i = atk.topk.sharded_approx_top_k_device(xd, 0, atk.AlgoParams(n, B, kp, k, min(B, 128)), comm)
    finally:
        comm.close()
    rv, ri = ref.approx_top_k_batch(f[None, :], B, kp, k, lane=min(B, 128), threads=1)
    assert np.array_equal(bits(v), bits(rv[0])) and np.array_equal(u32(i), ri[0])


def test_c_abi_sharded_entry_nan(cuda):
    import paper_2506_04165_b200 as atk
    n = 1 << 20
    x = np.random.default_rng(1).standard_normal(n).astype(np.float32)
    x[12345] = np.nan
    comm = atk.topk.NcclComm(1, atk.topk.NcclComm.unique_id(), 0)
    try:
        with pytest.raises(ValueError, match="NaN"):
            atk.topk.sharded_approx_top_k_device(torch.from_numpy(x).to(cuda), 0, atk.AlgoParams(n, 128, 2, 64),
                                                 comm)
    finally:
        comm.close()


def _stream_worker(rank, world, port, n, B, kp, k, seed, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2506_04165_b200 as atk
        from paper_2506_04165_b200 import data
        from paper_2506_04165_b200.shard import ShardedTopK
        dev = torch.device("cuda:0")
        sh = ShardedTopK(atk.AlgoParams(n, B, kp, k))  # default: payload exchange (host-staged under gloo)
        start, length = sh.bounds()
        x = torch.from_numpy(data.normal_f32_range(seed, start, length)).to(dev)
        v, i = sh(x)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), v=v.cpu().numpy(), i=i.cpu().numpy(), fb=sh.fallbacks)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,B,kp,k", [(2, 1 << 22, 256, 8, 1024), (3, 3 << 20, 128, 2, 64)])
def test_sharded_payload_exchange_multiprocess(cuda, ref, tmp_path, world, n, B, kp, k):
    from paper_2506_04165_b200 import data
    seed = 41 + world
    mp.spawn(_stream_worker, args=(world, _free_port(), n, B, kp, k, seed, str(tmp_path)), nprocs=world, join=True)
    row = data.normal_f32(seed, (n,))
    rv, ri = ref.approx_top_k_batch(row[None, :], B, kp, k, threads=1)
    for r in range(world):
        d = np.load(tmp_path / f"r{r}.npz")
        assert int(d["fb"]) == 0
        assert np.array_equal(bits(d["v"]), bits(rv[0])) and np.array_equal(u32(d["i"]), ri[0])

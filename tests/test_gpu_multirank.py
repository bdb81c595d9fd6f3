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

"""Sharded giant-row approximate top-K.

One row of n elements is cut into index-contiguous slices, one per rank
(one process per GPU).  Two exchanges, both exact (bit-identical to the
reference's approx_top_k on the whole row, topk.cpp:238-258, which consumes
the row's blocks in index order, Stage1Accumulator::consume, topk.cpp:123-172):

* stream (default, device tensors): each rank runs the threshold stream over
  its slice and sends a payload holding every element of the slice above the
  slice threshold (atkg_slice_payload, a few KB); after the all-gather every
  rank runs the per-row finish on all payloads with L = the max slice
  threshold (atkg_payload_merge_top_k).  When the payloads cannot settle the
  row (a gate word, the same on every rank) all ranks take:
* exact: each rank reduces its slice to the exact per-bucket stage-1 summary
  (atkg_stage1_summary: (2K'+2)*B uint32 words, ~16 KB for K'=8, B=256), the
  summaries are all-gathered, merged in index order and stage 2 runs
  (atkg_summary_merge_top_k).  Summaries merge associatively.
The data-path collectives are these all-gathers over NCCL (NVLink/NVSwitch):
G x a few KB, latency-bound.  atkg_sharded_approx_top_k is the same exchange
behind the C ABI for a C++ caller with its own NCCL communicator.

The reduce / merge steps are injectable so the exchange logic runs under the
gloo backend on CPU in tests (tests/test_distributed.py) with the host
emulation of the same summary code; the product path uses the CUDA kernels.
"""
from __future__ import annotations

import math

from .topk import (AlgoParams, payload_merge_top_k_device, slice_payload_device, slice_payload_words,
                   stage1_summary_device, summary_merge_top_k_device, summary_words)

GEN_BLOCK = 65536  # generator block of the synthetic inputs (csrc/datagen.cpp)


def slice_bounds(n: int, num_buckets: int, world: int, rank: int, align: int = GEN_BLOCK) -> tuple[int, int]:
    """(start, length) of `rank`'s slice.  Slices are contiguous, in rank
    order, and start on multiples of num_buckets (so a slice's local bucket
    id equals the global one) and, when n allows it, of `align`."""
    if n % num_buckets:
        raise ValueError("sharding needs n to be a multiple of num_buckets")
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    unit = num_buckets * align // math.gcd(num_buckets, align)
    if n % unit:
        unit = num_buckets
    units = n // unit
    per, rem = divmod(units, world)
    first = rank * per + min(rank, rem)
    count = per + (1 if rank < rem else 0)
    return first * unit, count * unit


class ShardedTopK:
    """Approximate top-K of one row sharded over the ranks of `group`.

    `summarize(slice, offset, params, status)` -> int32 tensor of
    summary_words(params); ORs the NaN flag into the int32 `status` tensor.
    `merge(summaries [world, words], params)` -> (values, indices).
    Both default to the device kernels (atkg_stage1_summary /
    atkg_summary_merge_top_k).

    NaN: every rank's NaN flag travels as one extra word of its gathered
    summary, so all ranks see the same verdict with no extra collective --
    they all raise "input contains NaN" (topk.cpp:22-28), or with a caller
    `status` tensor all OR the flag into it, instead of one rank raising
    before the all-gather while the others wait in it.
    """

    def __init__(self, params: AlgoParams, group=None, summarize=None, merge=None, mode: str | None = None):
        import torch.distributed as dist
        params.validate()
        # injected summary hooks (host emulation in tests) imply the exact exchange
        self.mode = mode or ("exact" if summarize is not None else "stream")
        self.fallbacks = 0
        # gloo moves host tensors only: stage device payloads through the host
        self._host_exchange = dist.get_backend(group) == "gloo"
        self.params = params
        self.group = group
        self.dist = dist
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.words = summary_words(params)
        self.summarize = summarize or (lambda x, off, p, st: stage1_summary_device(x, off, p, out=self._out, status=st))
        self.merge = merge or (lambda s, p: summary_merge_top_k_device(s, p, status=self._merge_status))
        self._send = None
        self._gathered = None
        self._out = None
        self._merge_status = None

    def bounds(self, rank: int | None = None) -> tuple[int, int]:
        return slice_bounds(self.params.n, self.params.num_buckets, self.world,
                            self.rank if rank is None else rank)

    def __call__(self, x_slice, status=None):
        """x_slice: this rank's elements [start, start + length) of the row.
        Returns (values [K], indices [K]) on every rank."""
        import torch
        start, length = self.bounds()
        if x_slice.numel() != length:
            raise ValueError(f"rank {self.rank} slice must hold {length} elements")
        if self.mode == "stream":
            import torch
            parts = self.world
            pw = slice_payload_words(self.params, parts)
            if getattr(self, "_pay", None) is None or self._pay.device != x_slice.device:
                self._pay = torch.empty(pw, dtype=torch.int32, device=x_slice.device)
                self._pays = torch.empty(parts * pw, dtype=torch.int32, device=x_slice.device)
                self._pst = torch.zeros(1, dtype=torch.int32, device=x_slice.device)
            self._pst.zero_()
            slice_payload_device(x_slice, start, self.params, parts, out=self._pay, status=self._pst)
            if self._host_exchange and self._pay.is_cuda:
                hp = self._pay.cpu()
                hall = torch.empty(parts * pw, dtype=torch.int32)
                self.dist.all_gather_into_tensor(hall, hp, group=self.group)
                self._pays.copy_(hall)
            else:
                self.dist.all_gather_into_tensor(self._pays, self._pay, group=self.group)
            v, i, gate = payload_merge_top_k_device(self._pays.view(parts, pw), self.params, status=self._pst)
            if int(gate.item()) == 0:  # the same verdict on every rank
                return v, i
            self.fallbacks += 1
        w = self.words
        if self._send is None or self._send.device != x_slice.device:
            self._send = torch.empty(w + 1, dtype=torch.int32, device=x_slice.device)
            self._gathered = torch.empty(self.world * (w + 1), dtype=torch.int32, device=x_slice.device)
        self._out = self._send[:w]
        flag = self._send[w:]
        flag.zero_()
        summ = self.summarize(x_slice, start, self.params, flag)
        if summ.data_ptr() != self._send.data_ptr():
            self._send[:w].copy_(summ.view(torch.int32).reshape(-1))
        self.dist.all_gather_into_tensor(self._gathered, self._send, group=self.group)
        g = self._gathered.view(self.world, w + 1)
        flags = g[:, w]
        if status is None:
            if int(flags.max().item()) & 1:
                raise ValueError("input contains NaN")
            self._merge_status = None
        else:
            status.bitwise_or_(flags.amax().view(1).to(status.dtype))
            self._merge_status = status
        return self.merge(g[:, :w].contiguous(), self.params)

"""The exact split-merge algorithm of the stage-1 kernels, checked on the CPU.

tests/emu/summary_emu.cu compiles paper_2506_04165_b200/csrc/stage1.cuh with
nvcc and runs the SAME Summ<K'> code the kernels execute (prologue fill, main
loop, associative merge, closed-form finalize) on the host.  Random segment
splits and random association orders over duplicate-heavy, +-0, +-inf and
tiny-bucket streams must reproduce the reference Alg. 1 grid bit-for-bit.
"""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest


def run_emu(emu, row, B, kp, bounds, mode, seed):
    n = row.size
    gv = np.empty(kp * B, np.float32)
    gi = np.empty(kp * B, np.uint32)
    nan = C.c_uint32()
    assert emu.emu_stage1(row, n, B, kp, bounds, len(bounds) - 1, mode, seed, gv, gi, C.byref(nan)) == 0
    return gv, gi, nan.value


VALUE_SETS = [
    np.array([0.0, 1.0, 2.0, 3.0], np.float32),
    np.array([0.0, -0.0, 1.0, -np.inf, np.inf, 2.0], np.float32),
    np.array([-np.inf, -np.inf, -1.0, 0.0], np.float32),
]


@pytest.mark.parametrize("seed", range(4))
def test_split_merge_matches_alg1(emu, port, seed):
    rng = np.random.default_rng(1000 + seed)
    for t in range(400):
        kp = int(rng.choice([1, 2, 3, 4, 5, 6, 7, 8, 16]))
        B = int(rng.integers(1, 9))
        nstr = int(rng.integers(1, 50))
        n = B * nstr
        kind = t % 4
        if kind < 3:
            row = rng.choice(VALUE_SETS[kind], n).astype(np.float32)
        else:
            row = rng.standard_normal(n).astype(np.float32)
        rv, ri = port.stage1(row, B, kp, lane=1)
        for mode in (0, 1, 2):
            nseg = int(rng.integers(1, nstr + 1))
            cuts = np.sort(rng.choice(np.arange(1, nstr), size=min(nseg - 1, nstr - 1), replace=False)) \
                if nstr > 1 else np.array([], np.int64)
            bounds = np.concatenate([[0], cuts, [nstr]]).astype(np.uint32)
            gv, gi, nan = run_emu(emu, row, B, kp, bounds, mode, t)
            assert nan == 0
            assert np.array_equal(gv.view(np.uint32), rv.view(np.uint32)), (t, mode, kp, B, bounds)
            assert np.array_equal(gi, ri), (t, mode, kp, B, bounds)


def test_nan_flagged(emu):
    row = np.array([1, 2, np.nan, 3, 4, 5, 6, 7], np.float32)
    for mode in (0, 2):
        _, _, nan = run_emu(emu, row, 2, 2, np.array([0, 2, 4], np.uint32), mode, 0)
        assert nan == 1

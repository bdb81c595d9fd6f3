"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/atkg.h declares, and the host-side entry points (validation,
planner, recall analysis, input generation) match the reference."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from tests.conftest import ROOT

import paper_2506_04165_b200 as atk
from paper_2506_04165_b200 import _lib


def header_symbols():
    text = open(os.path.join(ROOT, "include", "atkg.h")).read()
    return sorted(set(re.findall(r"\b(atkg_[a-z0-9_]+)\s*\(", text)) - {"atkg_params"})


def test_library_exports_every_header_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r" T (atkg_\w+)", out))
    missing = [s for s in header_symbols() if s not in exported]
    assert not missing, f"declared but not exported: {missing}"


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_no_torch_in_boundary():
    text = open(os.path.join(ROOT, "include", "atkg.h")).read()
    assert "torch" not in text.lower().replace("no torch", "")
    out = subprocess.run(["ldd", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "torch" not in out and "libc10" not in out


@pytest.mark.parametrize("kw,msg", [
    (dict(n=0), "n must be >= 1"), (dict(n=1 << 32, num_buckets=1 << 32), "n exceeds the 32-bit index range"),
    (dict(num_buckets=0), "num_buckets must be >= 1"), (dict(num_buckets=24), "num_buckets must divide n"),
    (dict(lane_multiple=3), "num_buckets must be a multiple of lane_multiple"),
    (dict(local_k=0), "local_k must be >= 1"), (dict(global_k=0), "global_k must be >= 1"),
    (dict(global_k=257), "global_k must not exceed n"),
    (dict(global_k=40), r"num_buckets \* local_k must be >= global_k")])
def test_validate_messages(kw, msg):
    # test_topk.cpp:419-459
    base = dict(n=256, num_buckets=16, local_k=2, global_k=20, lane_multiple=8)
    base.update(kw)
    with pytest.raises(ValueError, match=msg):
        atk.AlgoParams(**base).validate()


def test_validate_ok_and_analysis_relaxation():
    atk.AlgoParams(256, 16, 2, 20, 8).validate()
    atk.AlgoParams(256, 24, 2, 40, 8).validate_analysis()
    with pytest.raises(ValueError):
        atk.AlgoParams(256, 257, 2, 40, 8).validate_analysis()


def test_partition_index():
    p = atk.AlgoParams(16, 4, 1, 1)
    assert [atk.partition_index(i, p) for i in (0, 5, 15, 4)] == [0, 1, 3, 0]


def test_measure_recall_host():
    e = atk.TopKResult(np.array([5, 4], np.float32), np.array([4, 2], np.uint32))
    assert atk.measure_recall(atk.TopKResult([5, 4], [4, 2]), e) == 1.0
    assert atk.measure_recall(atk.TopKResult([4, 5], [2, 4]), e) == 1.0
    assert atk.measure_recall(atk.TopKResult([5, 3], [4, 7]), e) == 0.5
    assert atk.measure_recall(atk.TopKResult([1, 1], [9, 8]), e) == 0.0
    with pytest.raises(ValueError):
        atk.measure_recall(atk.TopKResult([5], [4]), e)


def test_generator_is_deterministic_and_normal():
    from paper_2506_04165_b200 import data
    a = data.normal_f32(123, (3, 70001))
    b = data.normal_f32(123, (3, 70001))
    assert np.array_equal(a, b)
    assert abs(a.mean()) < 0.02 and abs(a.std() - 1) < 0.02
    bits, f = data.normal_bf16(123, (1000,))
    assert np.array_equal(f.view(np.uint32) >> 16, bits.astype(np.uint32))
    # RNE: error at most half an ulp of bf16
    x = data.normal_f32(123, (1000,))
    assert np.all(np.abs(f - x) <= np.abs(x) * 2.0 ** -8)

import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def port():
    """The plain-C restatement (oracle/atk_oracle.c), built on demand."""
    from oracle import pyoracle as O
    if not os.path.exists(O.PORT_PATH):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "port"], check=True, capture_output=True)
    return O.port()


@pytest.fixture(scope="session")
def ref():
    """The reference library compiled from /root/reference (oracle/_ref)."""
    from oracle import pyoracle as O
    if not O.ref_available() and os.path.isdir("/root/reference/proj/core"):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True, capture_output=True)
    if not O.ref_available():
        pytest.skip("oracle/_ref/libatk_ref.so not available")
    return O.ref()


@pytest.fixture(scope="session")
def stage_fixtures():
    return np.load(os.path.join(ROOT, "tests", "golden", "stage_fixtures.npz"))


@pytest.fixture(scope="session")
def planner_fixtures():
    return np.load(os.path.join(ROOT, "tests", "golden", "planner_fixtures.npz"), allow_pickle=True)


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


EMU_SRC = os.path.join(ROOT, "tests", "emu", "summary_emu.cu")
EMU_LIB = os.path.join(ROOT, "build", "libatkg_emu.so")


def build_emu():
    """Host build of the device summary code (tests/emu/summary_emu.cu)."""
    import glob
    hdrs = glob.glob(os.path.join(ROOT, "paper_2506_04165_b200", "csrc", "*.cuh"))
    stale = not os.path.exists(EMU_LIB) or any(os.path.getmtime(EMU_LIB) < os.path.getmtime(p)
                                                for p in [EMU_SRC, *hdrs])
    if stale:
        os.makedirs(os.path.dirname(EMU_LIB), exist_ok=True)
        subprocess.run(["/usr/local/cuda/bin/nvcc", "-O2", "-std=c++17", "-gencode",
                        "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fPIC", "-shared", "-o", EMU_LIB, EMU_SRC],
                       check=True, capture_output=True)
    return EMU_LIB


def load_emu(path=EMU_LIB):
    import ctypes as C
    lib = C.CDLL(path)
    f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
    u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
    lib.emu_stage1.argtypes = [f32p, C.c_uint64, C.c_uint64, C.c_uint32, u32p, C.c_uint32, C.c_int, C.c_uint64,
                               f32p, u32p, C.POINTER(C.c_uint32)]
    lib.emu_stage1.restype = C.c_int
    lib.emu_slice_summary.argtypes = [f32p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32, u32p,
                                      C.POINTER(C.c_uint32)]
    lib.emu_slice_summary.restype = C.c_int
    lib.emu_merge_summaries.argtypes = [u32p, C.c_uint32, C.c_uint64, C.c_uint32, f32p, u32p]
    lib.emu_merge_summaries.restype = C.c_int
    return lib


@pytest.fixture(scope="session")
def emu():
    return load_emu(build_emu())


@pytest.fixture
def opts():
    """opts(name, value): a library path-selection override (atkg_set_option)
    for the duration of one test."""
    from paper_2506_04165_b200 import _lib
    touched = {}

    def set_(name, value):
        if name not in touched:
            touched[name] = _lib.lib.atkg_get_option(name.encode(), 2**64 - 1)
        _lib.set_option(name, value)

    yield set_
    for name, prev in touched.items():
        _lib.set_option(name, None if prev == 2**64 - 1 else prev)

"""ATKV dataset container: atkg_dataset_* against the reference.

Reference behaviour: dataset.hpp:18-50, dataset.cpp:45-130; its own tests are
test_dataset.cpp (round trip, 0-row header-only file, bad magic / version,
truncation, NaN rejection).  Pinned three ways:
* files written by the reference writer (tests/golden/atkv, make_atkv_golden.py)
  must be byte-identical to ours and read back bit-exactly;
* every malformed file must fail with the reference's exact message
  (tests/golden/atkv/errors.json);
* where oracle/_ref is built, the live reference is compared too.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import struct

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "atkv")

GOLDEN_SHAPES = {"empty_0x5": (0, 5), "zero_dims_4x0": (4, 0), "one_1x1": (1, 1),
                 "ragged_3x7": (3, 7), "rows_17x129": (17, 129)}


def golden_payload(rows: int, dims: int) -> np.ndarray:
    """Seeded values with the edge cases a payload can hold: ±0, ±inf, subnormals, extremes."""
    rng = np.random.default_rng(rows * 1000 + dims)
    x = rng.standard_normal(rows * dims).astype(np.float32)
    special = np.array([0.0, -0.0, np.inf, -np.inf, 1e-45, -1e-45, 3.4028235e38, -3.4028235e38],
                       np.float32)
    x[:min(x.size, special.size)] = special[:min(x.size, special.size)]
    return x


def _header(rows: int, dims: int, magic=b"ATKV", version=1) -> bytes:
    return magic + bytes([version]) + struct.pack("<QQ", rows, dims)


def malformed_cases() -> dict:
    """dataset.cpp:84-121 failure paths, in the order the reader checks them."""
    ok = np.arange(6, dtype="<f4").tobytes()
    nan = np.array([1, 2, 3, 4, 5, np.nan], "<f4").tobytes()
    return {
        "empty_file": b"",
        "header_short": _header(2, 3)[:20],
        "bad_magic": _header(2, 3, magic=b"ATKW") + ok,
        "bad_version": _header(2, 3, version=2) + ok,
        "shape_overflow": _header(2**33, 2**32),
        "too_large": _header(2**20, 2**14 + 1),
        "payload_short": _header(2, 3) + ok[:-1],
        "payload_missing": _header(2, 3),
        "payload_nan": _header(2, 3) + nan,
    }


# ---- the reference, through oracle/_ref (test infrastructure) ---------------
def ref_write(lib, path, data, rows, dims):
    lib.ref_dataset_write_file.argtypes = [C.c_char_p, C.c_void_p, C.c_uint64, C.c_uint64]
    data = np.ascontiguousarray(data, np.float32)
    rc = lib.ref_dataset_write_file(os.fsencode(path), data.ctypes.data, rows, dims)
    lib.ref_last_error.restype = C.c_char_p
    return rc, lib.ref_last_error().decode()


def ref_read(lib, path, cap=1 << 24):
    lib.ref_dataset_read_file.argtypes = [C.c_char_p, C.c_void_p, C.c_uint64,
                                          C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
    out = np.empty(cap, np.float32)
    r, d = C.c_uint64(), C.c_uint64()
    rc = lib.ref_dataset_read_file(os.fsencode(path), out.ctypes.data, cap, C.byref(r), C.byref(d))
    lib.ref_last_error.restype = C.c_char_p
    return rc, lib.ref_last_error().decode(), (r.value, d.value, out[:r.value * d.value])


def _errors():
    with open(os.path.join(GOLDEN, "errors.json")) as f:
        return json.load(f)


# ---- host (C ABI, no GPU needed) ---------------------------------------------
@pytest.mark.parametrize("name", sorted(GOLDEN_SHAPES))
def test_golden_files_read_and_rewrite_bit_exact(name, tmp_path):
    import paper_2506_04165_b200 as atk
    rows, dims = GOLDEN_SHAPES[name]
    path = os.path.join(GOLDEN, f"{name}.atkv")
    ds = atk.read_dataset_file(path)
    assert (ds.rows, ds.dims) == (rows, dims)
    assert ds.data.view(np.uint32).tobytes() == golden_payload(rows, dims).view(np.uint32).tobytes()
    out = tmp_path / "w.atkv"
    atk.write_dataset_file(atk.VectorDataset(rows, dims, golden_payload(rows, dims)), out)
    assert out.read_bytes() == open(path, "rb").read()


def test_header_only_file_is_21_bytes(tmp_path):
    import paper_2506_04165_b200 as atk
    p = tmp_path / "e.atkv"
    atk.write_dataset_file(atk.VectorDataset(0, 9, np.zeros(0, np.float32)), p)
    assert p.read_bytes() == _header(0, 9)
    assert atk.dataset.read_header(p) == (0, 9)


@pytest.mark.parametrize("name", sorted(malformed_cases()))
def test_malformed_messages_match_reference(name, tmp_path):
    import paper_2506_04165_b200 as atk
    p = tmp_path / name
    p.write_bytes(malformed_cases()[name])
    with pytest.raises(atk.DatasetFormatError) as e:
        atk.read_dataset_file(p)
    assert str(e.value) == _errors()[name]


def test_write_nan_rejected_after_open(tmp_path):
    import paper_2506_04165_b200 as atk
    p = tmp_path / "n.atkv"
    p.write_bytes(b"old contents")
    with pytest.raises(atk.DatasetFormatError) as e:
        atk.write_dataset_file(atk.VectorDataset(1, 2, np.array([1.0, np.nan], np.float32)), p)
    assert str(e.value) == _errors()["write_nan"]
    assert p.read_bytes() == b""  # dataset.cpp:75-80 opens (truncates) before validating


def test_open_failures(tmp_path):
    import paper_2506_04165_b200 as atk
    missing = tmp_path / "nope" / "x.atkv"
    with pytest.raises(atk.DatasetFormatError, match=f"^cannot open for read: {missing}$"):
        atk.read_dataset_file(missing)
    with pytest.raises(atk.DatasetFormatError, match=f"^cannot open for write: {missing}$"):
        atk.write_dataset_file(atk.VectorDataset(1, 1, np.ones(1, np.float32)), missing)


def test_trailing_bytes_ignored_and_size_mismatch(tmp_path):
    import paper_2506_04165_b200 as atk
    p = tmp_path / "t.atkv"
    p.write_bytes(_header(1, 2) + np.array([1.5, -2.5], "<f4").tobytes() + b"junk")
    ds = atk.read_dataset_file(p)
    assert ds.data.tolist() == [1.5, -2.5]
    with pytest.raises(atk.DatasetFormatError, match="^dataset payload size does not match shape$"):
        atk.write_dataset_file(atk.VectorDataset(2, 2, np.ones(3, np.float32)), p)


def test_multi_chunk_round_trip_matches_reference(ref, tmp_path):
    """> one 16 MiB staging chunk, ragged tail; our file == the reference's file."""
    import paper_2506_04165_b200 as atk
    rows, dims = 3, (1 << 22) // 3 * 2 + 5
    x = golden_payload(rows, dims)
    ours, theirs = tmp_path / "o.atkv", tmp_path / "r.atkv"
    atk.write_dataset_file(atk.VectorDataset(rows, dims, x), ours)
    rc, msg = ref_write(ref.lib, theirs, x, rows, dims)
    assert rc == 0, msg
    assert ours.read_bytes() == theirs.read_bytes()
    rc, msg, (r, d, y) = ref_read(ref.lib, ours, cap=rows * dims)
    assert rc == 0 and (r, d) == (rows, dims) and y.view(np.uint32).tobytes() == x.view(np.uint32).tobytes()


def test_error_golden_matches_live_reference(ref, tmp_path):
    for name, blob in malformed_cases().items():
        p = tmp_path / name
        p.write_bytes(blob)
        rc, msg, _ = ref_read(ref.lib, p)
        assert (rc, msg) == (6, _errors()[name]), name


# ---- device (GPU) -----------------------------------------------------------
def _multi_chunk_payload():
    rows, dims = 5, 2 * (1 << 22) // 5 + 4  # three staging chunks, non-multiple-of-4 tail
    return rows, dims, golden_payload(rows, dims)


@pytest.mark.gpu
def test_device_read_bit_exact(cuda, tmp_path):
    import paper_2506_04165_b200 as atk
    rows, dims, x = _multi_chunk_payload()
    p = tmp_path / "d.atkv"
    atk.write_dataset_file(atk.VectorDataset(rows, dims, x), p)
    t = atk.read_dataset_to_device(p, cuda)
    assert t.shape == (rows, dims) and t.is_cuda
    assert t.cpu().numpy().reshape(-1).view(np.uint32).tobytes() == x.view(np.uint32).tobytes()
    for name in sorted(GOLDEN_SHAPES):
        g = atk.read_dataset_to_device(os.path.join(GOLDEN, f"{name}.atkv"), cuda)
        assert tuple(g.shape) == GOLDEN_SHAPES[name]
        assert g.cpu().numpy().reshape(-1).view(np.uint32).tobytes() == \
            golden_payload(*GOLDEN_SHAPES[name]).view(np.uint32).tobytes()


@pytest.mark.gpu
def test_device_write_matches_golden_bytes(cuda, tmp_path):
    import torch
    import paper_2506_04165_b200 as atk
    for name, (rows, dims) in sorted(GOLDEN_SHAPES.items()):
        t = torch.from_numpy(golden_payload(rows, dims).reshape(rows, dims)).to(cuda)
        p = tmp_path / f"{name}.atkv"
        atk.write_dataset_from_device(t, p)
        assert p.read_bytes() == open(os.path.join(GOLDEN, f"{name}.atkv"), "rb").read(), name
    rows, dims, x = _multi_chunk_payload()
    p = tmp_path / "big.atkv"
    atk.write_dataset_from_device(torch.from_numpy(x.reshape(rows, dims)).to(cuda), p)
    assert p.read_bytes() == _header(rows, dims) + x.astype("<f4").tobytes()


@pytest.mark.gpu
def test_device_malformed_and_nan(cuda, tmp_path):
    import torch
    import paper_2506_04165_b200 as atk
    errs = _errors()
    for name, blob in malformed_cases().items():
        p = tmp_path / name
        p.write_bytes(blob)
        with pytest.raises(atk.DatasetFormatError) as e:
            atk.read_dataset_to_device(p, cuda)
        assert str(e.value) == errs[name], name
    # a NaN in the ragged tail of the last staging chunk, on read and on write
    rows, dims, x = _multi_chunk_payload()
    x = x.copy()
    x[-1] = np.nan
    p = tmp_path / "tailnan.atkv"
    p.write_bytes(_header(rows, dims) + x.astype("<f4").tobytes())
    with pytest.raises(atk.DatasetFormatError, match="^dataset payload contains NaN$"):
        atk.read_dataset_to_device(p, cuda)
    with pytest.raises(atk.DatasetFormatError, match="^dataset payload contains NaN$"):
        atk.write_dataset_from_device(torch.from_numpy(x.reshape(rows, dims)).to(cuda), tmp_path / "w.atkv")
    # truncated inside the second chunk
    p.write_bytes(_header(rows, dims) + x.astype("<f4").tobytes()[:(1 << 22) * 4 + 100])
    with pytest.raises(atk.DatasetFormatError, match="^dataset truncated: payload incomplete$"):
        atk.read_dataset_to_device(p, cuda)


@pytest.mark.gpu
def test_device_read_feeds_approx_top_k(cuda, tmp_path):
    """Replay: a dumped activation file read to HBM gives the reference's top-k."""
    import paper_2506_04165_b200 as atk
    from oracle import pyoracle as O
    rows, dims = 4, 32768
    x = np.random.default_rng(7).standard_normal(rows * dims).astype(np.float32)
    p = tmp_path / "act.atkv"
    atk.write_dataset_file(atk.VectorDataset(rows, dims, x), p)
    t = atk.read_dataset_to_device(p, cuda)
    params = atk.AlgoParams(n=dims, num_buckets=256, local_k=2, global_k=64)
    v, i = atk.approx_top_k_device(t, params)
    ev, ei = O.port().approx_top_k_batch(x.reshape(rows, dims), 256, 2, 64)
    assert np.array_equal(v.cpu().numpy(), ev)
    assert np.array_equal(i.cpu().numpy().astype(np.uint32), ei)


@pytest.mark.gpu
def test_device_write_from_unaligned_view(cuda, tmp_path):
    """A row-offset view (not 16-byte aligned) takes the scalar NaN scan."""
    import torch
    import paper_2506_04165_b200 as atk
    rows, dims = 7, 1001
    x = golden_payload(rows, dims)
    base = torch.zeros(1 + rows * dims, dtype=torch.float32, device=cuda)
    base[1:] = torch.from_numpy(x).to(cuda)
    view = base[1:].view(rows, dims)
    assert view.data_ptr() % 16 != 0
    p = tmp_path / "u.atkv"
    atk.write_dataset_from_device(view, p)
    assert p.read_bytes() == _header(rows, dims) + x.astype("<f4").tobytes()
    base[-1] = float("nan")
    with pytest.raises(atk.DatasetFormatError, match="^dataset payload contains NaN$"):
        atk.write_dataset_from_device(view, p)

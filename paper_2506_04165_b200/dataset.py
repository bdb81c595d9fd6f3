"""ATKV dataset container: host mirror of atk/dataset.hpp.

* ``VectorDataset`` mirrors ``atk::VectorDataset`` (dataset.hpp:30-45): a
  row-major ``[rows, dims]`` fp32 matrix.
* ``read_dataset_file`` / ``write_dataset_file`` mirror dataset.hpp:47-50
  (dataset.cpp:45-124).  They call ``atkg_dataset_*`` in libatkg.so; format
  errors raise ``DatasetFormatError`` with the reference's messages.
* ``read_dataset_to_device`` / ``write_dataset_from_device`` move the payload
  straight between the file and HBM through pinned double-buffered chunks,
  with the NaN rejection as a device scan: dumping fused activations and
  replaying inputs for cross-box parity.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import DatasetFormatError  # noqa: F401

try:
    import torch
except ImportError:  # pragma: no cover
    torch = None

MAGIC = b"ATKV"
VERSION = 1
HEADER_BYTES = 21


@dataclass
class VectorDataset:
    """atk::VectorDataset (dataset.hpp:30-45)."""
    rows: int = 0
    dims: int = 0
    data: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))

    def row(self, r: int) -> np.ndarray:
        return self.data[r * self.dims:(r + 1) * self.dims]

    def matrix(self) -> np.ndarray:
        return self.data.reshape(self.rows, self.dims)

    def validate(self) -> None:
        """dataset.cpp:37-41."""
        if self.dims != 0 and self.rows > (2**64 - 1) // self.dims:
            raise DatasetFormatError("dataset shape overflows")
        if self.data.size != self.rows * self.dims:
            raise DatasetFormatError("dataset payload size does not match shape")
        if np.isnan(self.data).any():
            raise DatasetFormatError("dataset payload contains NaN")


def _path(p) -> bytes:
    return os.fsencode(os.fspath(p))


def read_header(path) -> tuple[int, int]:
    """(rows, dims) of an ATKV file, with the reference's header checks."""
    r, d = C.c_uint64(), C.c_uint64()
    _lib.check(_lib.lib.atkg_dataset_read_header(_path(path), C.byref(r), C.byref(d)))
    return r.value, d.value


def read_dataset_file(path) -> VectorDataset:
    """atk::read_dataset_file (dataset.cpp:84-130)."""
    rows, dims = read_header(path)
    out = np.empty(max(rows * dims, 1), np.float32)
    r, d = C.c_uint64(), C.c_uint64()
    _lib.check(_lib.lib.atkg_dataset_read_file(_path(path), out.ctypes.data, rows * dims,
                                               C.byref(r), C.byref(d)))
    return VectorDataset(r.value, d.value, out[:r.value * d.value])


def write_dataset_file(dataset: VectorDataset, path) -> None:
    """atk::write_dataset_file (dataset.cpp:45-82)."""
    data = np.ascontiguousarray(dataset.data, np.float32).reshape(-1)
    if data.size != dataset.rows * dataset.dims:
        # the reference opens (truncates) the file before validate() throws
        open(path, "wb").close()
        raise DatasetFormatError("dataset payload size does not match shape")
    _lib.check(_lib.lib.atkg_dataset_write_file(_path(path), data.ctypes.data if data.size else None,
                                                dataset.rows, dataset.dims))


def read_dataset_to_device(path, device=None) -> "torch.Tensor":
    """Reads an ATKV file straight into a ``[rows, dims]`` fp32 CUDA tensor."""
    from .topk import _stream_ptr
    device = torch.device(device if device is not None else "cuda")
    rows, dims = read_header(path)
    out = torch.empty((rows, dims), dtype=torch.float32, device=device)
    r, d = C.c_uint64(), C.c_uint64()
    _lib.check(_lib.lib.atkg_dataset_read_file_device(_path(path), out.data_ptr() if out.numel() else None,
                                                      rows * dims, C.byref(r), C.byref(d),
                                                      _stream_ptr(out.device)))
    return out


def write_dataset_from_device(t: "torch.Tensor", path) -> None:
    """Writes a 2-D fp32 CUDA tensor (e.g. fused activations) as an ATKV file."""
    from .topk import _stream_ptr
    if t.dim() != 2 or t.dtype != torch.float32 or not t.is_cuda:
        raise ValueError("expected a 2-D fp32 CUDA tensor")
    t = t.contiguous()
    _lib.check(_lib.lib.atkg_dataset_write_file_device(_path(path), t.data_ptr() if t.numel() else None,
                                                       t.shape[0], t.shape[1], _stream_ptr(t.device)))

"""Generates tests/golden/atkv/ from the REFERENCE library itself.

    make -C oracle ref && python tests/golden/make_atkv_golden.py

* ``*.atkv``: files written by the reference's ``atk::write_dataset_file``
  (dataset.cpp:45-82) through oracle/_ref/libatk_ref.so.
* ``errors.json``: the reference's ``DatasetFormatError`` message for every
  malformed file built by ``tests/test_dataset.py::malformed_cases``.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import pyoracle as O  # noqa: E402
from tests.test_dataset import GOLDEN_SHAPES, golden_payload, malformed_cases, ref_read, ref_write  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "atkv")


def main():
    lib = O.ref().lib
    os.makedirs(OUT, exist_ok=True)
    for name, (rows, dims) in GOLDEN_SHAPES.items():
        rc, msg = ref_write(lib, os.path.join(OUT, f"{name}.atkv"), golden_payload(rows, dims), rows, dims)
        assert rc == 0, msg
    errors = {}
    with tempfile.TemporaryDirectory() as d:
        for name, blob in malformed_cases().items():
            p = os.path.join(d, name)
            with open(p, "wb") as f:
                f.write(blob)
            rc, msg, _ = ref_read(lib, p)
            assert rc == 6, (name, rc, msg)
            errors[name] = msg
        rc, msg = ref_write(lib, os.path.join(d, "nan.atkv"), np.array([1.0, np.nan], np.float32), 1, 2)
        assert rc == 6
        errors["write_nan"] = msg
    with open(os.path.join(OUT, "errors.json"), "w") as f:
        json.dump(errors, f, indent=1, sort_keys=True)
    print(f"wrote {len(GOLDEN_SHAPES)} files and {len(errors)} messages to {OUT}")


if __name__ == "__main__":
    main()

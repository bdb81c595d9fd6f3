"""Generates tests/golden/*.npz from the REFERENCE library itself.

Run in the build container, where /root/reference exists:

    make -C oracle ref && python tests/golden/make_golden.py

oracle/_ref/libatk_ref.so is the unmodified reference core compiled from
/root/reference/proj/core/src (oracle/Makefile).  Inputs are regenerated at
test time from seeds (paper_2506_04165_b200.data / oracle.pyoracle), so the
fixtures hold only the reference outputs plus a SHA-256 of every input, which
pins the input generators too.
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import pyoracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def cases():
    """(name, input-builder, B, K', K, lane). Builders are importable by the tests."""
    from tests.golden.inputs import INPUTS
    return INPUTS


def main():
    ref = O.ref()
    from tests.golden.inputs import INPUTS, build
    blobs = {}
    for name, spec in INPUTS.items():
        rows = build(spec)
        B, kp, k, lane = spec["B"], spec["kp"], spec["k"], spec.get("lane", 128)
        r, n = rows.shape
        gv = np.empty((r, kp * B), np.float32)
        gi = np.empty((r, kp * B), np.uint32)
        for i in range(r):
            gv[i], gi[i] = ref.stage1(rows[i], B, kp, lane)
        av, ai = ref.approx_top_k_batch(rows, B, kp, k, lane, threads=os.cpu_count())
        ev = np.empty((r, k), np.float32)
        ei = np.empty((r, k), np.uint32)
        rec = np.empty(r, np.float64)
        for i in range(r):
            ev[i], ei[i] = ref.exact_top_k(rows[i], k)
            rec[i] = ref.measure_recall(ai[i], ei[i])
        blobs[name] = dict(input_sha=sha(rows), grid_v=gv, grid_i=gi, approx_v=av, approx_i=ai, exact_v=ev,
                           exact_i=ei, recall=rec)
        print(f"{name}: rows={r} n={n} B={B} kp={kp} k={k} mean recall={rec.mean():.6f}")
    flat = {}
    for name, d in blobs.items():
        for key, v in d.items():
            flat[f"{name}/{key}"] = np.asarray(v)
    np.savez_compressed(os.path.join(OUT, "stage_fixtures.npz"), **flat)

    # planner / recall fixtures (planner.cpp:79-147, recall.cpp:76-100)
    plans = []
    for (n, k, t, kps, seed) in [
        (262144, 1024, 0.95, (1, 2, 3, 4), 1), (262144, 1024, 0.95, (1,), 1), (262144, 1024, 0.99, (1, 2, 3, 4), 1),
        (430080, 3360, 0.9, (1, 2, 3, 4), 1), (262144, 64, 0.95, (1, 2, 4), 0), (14336, 287, 0.95, (1, 2, 4, 8), 0),
        (14336, 287, 0.99, (1, 2, 4, 8), 0), (14336, 287, 0.95, (1,), 0), (14336, 287, 0.95, (2,), 0),
        (14336, 287, 0.95, (8,), 0), (14336, 287, 0.99, (1,), 0), (14336, 287, 0.99, (2,), 0),
        (14336, 287, 0.99, (4,), 0), (14336, 287, 0.99, (8,), 0), (2**30, 1024, 0.95, (8,), 0),
        (32768, 128, 0.95, (1, 2, 3, 4), 0),
    ]:
        p = ref.select_parameters(n, k, t, kps, 128, seed)
        plans.append((n, k, t, seed, ",".join(map(str, kps)), p.local_k, p.num_buckets, p.recall, int(p.exact)))
        print("plan", plans[-1])
    exact = []
    for (n, b, kp, k) in [(262144, 16384, 1, 1024), (262144, 512, 4, 1024), (430080, 5120, 2, 3360),
                          (15360, 640, 4, 480), (262144, 128, 2, 64), (14336, 128, 4, 287),
                          (2**30, 256, 8, 1024), (32768, 512, 4, 128), (1000, 7, 2, 30)]:
        exact.append((n, b, kp, k, ref.exact_expected_recall(n, b, kp, k)))
    mc = []
    for (n, b, kp, k, trials, seed) in [(262144, 512, 4, 1024, 4096, 7), (14336, 128, 4, 287, 10000, 3)]:
        m, s = ref.mc_expected_recall(n, b, kp, k, trials, seed)
        mc.append((n, b, kp, k, trials, seed, m, s))
    np.savez_compressed(os.path.join(OUT, "planner_fixtures.npz"),
                        plans=np.array(plans, dtype=object), exact=np.array(exact, dtype=np.float64),
                        mc=np.array(mc, dtype=np.float64),
                        legal_430080=np.array(ref.legal_bucket_counts(430080, 128), np.uint64))


if __name__ == "__main__":
    main()

"""The C++ drop-in header (include/atk_b200.hpp) against the reference core.

tests/cpp/_build/atk_b200_check is built in the build container (it needs
the reference headers; tests/cpp/Makefile, run by __graft_entry__.build())
and linked against libatkg.so and oracle/_ref/libatk_ref.so (the unmodified
reference core).  It calls atk::f and atk_b200::f on the same inputs for
every function of topk.hpp / planner.hpp / recall.hpp the header replaces
and compares the results bit for bit, and the exception type and message on
bad inputs (NaN, invalid parameters, infeasible plans)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "atk_b200_check")


def test_cpp_dropin_matches_reference(cuda):
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/_build/atk_b200_check not built (needs the reference headers)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    lines = r.stdout.splitlines()
    fails = [ln for ln in lines if ln.startswith("FAIL")]
    assert r.returncode == 0 and not fails, "\n".join(fails) + r.stderr[-2000:]
    assert sum(ln.startswith("PASS") for ln in lines) >= 25

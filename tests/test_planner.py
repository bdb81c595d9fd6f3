"""Host planner (csrc/planner.cpp) vs the reference: KATs restated from
proj/tests/test_planner.cpp / test_recall.cpp and golden fixtures produced by
the reference library (tests/golden/planner_fixtures.npz)."""
import numpy as np
import pytest

import paper_2506_04165_b200 as atk


def req(n, k, t, kps=(1, 2, 3, 4), seed=1, lane=128):
    return atk.PlanRequest(n, k, t, list(kps), lane, seed)


def test_planner_reference_configurations():
    # test_planner.cpp:86-115
    r = atk.select_parameters(req(262144, 1024, 0.95))
    assert (r.local_k, r.num_buckets, r.num_elements) == (4, 512, 2048)
    assert not r.high_target_warning and r.estimated_recall.method == "exact"
    assert r.estimated_recall.value == pytest.approx(0.96295662533487147, abs=1e-10)
    r = atk.select_parameters(req(262144, 1024, 0.95, (1,)))
    assert (r.local_k, r.num_buckets) == (1, 16384)
    assert r.estimated_recall.value == pytest.approx(0.97125744566081484, abs=1e-10)
    r = atk.select_parameters(req(262144, 1024, 0.99))
    assert (r.local_k, r.num_buckets, r.num_elements) == (4, 1024, 4096)
    p = r.params(req(262144, 1024, 0.99))
    assert (p.n, p.num_buckets, p.local_k, p.global_k) == (262144, 1024, 4, 1024)


def test_planner_invariants():
    r = atk.select_parameters(req(430080, 3360, 0.9))
    assert r.local_k == 4
    assert atk.exact_expected_recall(atk.AlgoParams(1024, 256, 4, 100, 1)).value == 1.0
    assert atk.exact_expected_recall(atk.AlgoParams(4096, 4096, 1, 64, 1)).value == 1.0


def test_planner_golden(planner_fixtures):
    for (n, k, t, seed, kps, kp, b, rec, ex) in planner_fixtures["plans"]:
        r = atk.select_parameters(req(int(n), int(k), float(t), tuple(int(x) for x in kps.split(",")), int(seed)))
        assert (r.local_k, r.num_buckets) == (kp, b), (n, k, t, kps)
        assert r.estimated_recall.value == rec
        assert (r.estimated_recall.method == "exact") == bool(ex)


def test_exact_and_mc_golden(planner_fixtures):
    for (n, b, kp, k, val) in planner_fixtures["exact"]:
        assert atk.exact_expected_recall(atk.AlgoParams(int(n), int(b), int(kp), int(k), 1)).value == val
    for (n, b, kp, k, trials, seed, m, s) in planner_fixtures["mc"]:
        e = atk.mc_expected_recall(atk.AlgoParams(int(n), int(b), int(kp), int(k), 1), int(trials), int(seed))
        assert e.value == m and e.std_error == s and e.trials == trials


def test_legal_bucket_counts(planner_fixtures):
    big = atk.legal_bucket_counts(430080, 128)
    assert big == [int(x) for x in planner_fixtures["legal_430080"]]
    assert len(big) == 48 and big[-1] == 128
    assert atk.legal_bucket_counts(262144, 128) == [262144 >> i for i in range(12)]
    assert atk.legal_bucket_counts(100, 128) == []
    assert atk.legal_bucket_counts(12, 1) == [12, 6, 4, 3, 2, 1]


@pytest.mark.parametrize("bad,msg", [
    (dict(n=0), "n must be >= 1"), (dict(k=0), "k must satisfy"), (dict(recall_target=1.0), "recall_target"),
    (dict(allowed_local_k=[]), "allowed_local_k must not be empty"),
    (dict(allowed_local_k=[0]), "entries must be >= 1"), (dict(lane_multiple=0), "lane_multiple")])
def test_plan_request_validation(bad, msg):
    base = dict(n=1024, k=10, recall_target=0.9, allowed_local_k=[1, 2], lane_multiple=128, seed=0)
    base.update(bad)
    with pytest.raises(ValueError, match=msg):
        atk.select_parameters(atk.PlanRequest(**base))


def test_infeasible():
    with pytest.raises(atk.NoFeasibleConfigError):
        atk.select_parameters(req(100, 10, 0.9, (1,)))  # no lane-legal B


def test_mc_adaptive_meets_tolerance():
    e = atk.mc_expected_recall_adaptive(atk.AlgoParams(262144, 512, 4, 1024, 128), 11)
    assert 3 * e.std_error <= 0.005 and e.trials >= 4096
    assert abs(e.value - 0.96295662533487147) < 0.01

"""Pin the CPU oracle (oracle/alert_oracle.c) to the reference.

Golden vectors were produced by the reference itself
(tests/golden/make_golden.py); the oracle must reproduce them BIT-EXACTLY
(same FP64 operation order, same glibc erf/pow as CPython).  Hand-computed
known answers are the reference's own unit-test values.
"""

import math

import numpy as np
import pytest

from oracle import oracle
from paper_1911_00119_b200 import abi
from paper_1911_00119_b200.model import ConfigSpace, ConstraintSpec, DnnKind, DnnProfile, Mode, PowerSetting, Stage


def mean_of(agg, field):
    return abi.neumaier_total(agg[field], agg[field + 1]) / agg[abi.AGG_N]


@pytest.fixture(scope="module", autouse=True)
def _built():
    oracle.build()


def check_golden(case):
    """The oracle reproduces one reference run bit for bit."""
    if True:
        rec, agg, st = oracle.run(case.space, case.spec, case.env, case.policy, kalman=case.kalman,
                                  group_size=case.group_size, goal_changes=case.changes)
        z = case.z
        np.testing.assert_array_equal(rec["feasible"], z["feasible"], err_msg=case.name)
        ours = np.stack([rec[f] for f in ("pred_latency_mean", "pred_latency_sigma", "pred_pr", "pred_accuracy",
                                          "pred_energy")], 1)
        np.testing.assert_array_equal(ours, z["pred"], err_msg=f"{case.name}:prediction")
        np.testing.assert_array_equal(rec["cand"], z["cand"], err_msg=case.name)
        np.testing.assert_array_equal(rec["level"], z["level"], err_msg=case.name)
        np.testing.assert_array_equal(rec["completed"], z["completed"], err_msg=case.name)
        np.testing.assert_array_equal(rec["met"], z["met"], err_msg=case.name)
        np.testing.assert_array_equal(np.stack([rec["viol_lat"], rec["viol_acc"], rec["viol_energy"]], 1),
                                      z["viol"], err_msg=case.name)
        for f in ("period", "latency", "accuracy", "energy"):
            np.testing.assert_array_equal(rec[f], z[f], err_msg=f"{case.name}:{f}")
        np.testing.assert_array_equal(rec["fb_latency"], z["fb"][:, 0], err_msg=case.name)
        np.testing.assert_array_equal(rec["fb_t_prof"], z["fb"][:, 1], err_msg=case.name)
        if case.policy not in ("oracle", "oracle-static"):
            ours = np.stack([rec[f] for f in ("mu", "sigma2", "k_gain", "q_noise", "innov", "phi", "m_var")], 1)
            cols = ~np.isnan(z["state"][0]) if len(z["state"]) else slice(None)
            np.testing.assert_array_equal(ours[:, cols], z["state"][:, cols], err_msg=case.name)
        n = agg[abi.AGG_N]
        assert mean_of(agg, abi.AGG_ENERGY) == z["summary"][0], case.name
        assert mean_of(agg, abi.AGG_ACC) == z["summary"][1], case.name
        assert agg[abi.AGG_VIOL_LAT] / n == z["summary"][2]
        assert agg[abi.AGG_VIOL_ACC] / n == z["summary"][3]
        assert agg[abi.AGG_VIOL_ENERGY] / n == z["summary"][4]
        ps = [k for k in range(case.n_phases) if agg[abi.AGG_PHASE_BASE + abi.AGG_PHASE_STRIDE * k] > 0]
        assert len(ps) == len(z["phase_summary"])
        for row, k in zip(z["phase_summary"], ps):
            b = abi.AGG_PHASE_BASE + abi.AGG_PHASE_STRIDE * k
            m = agg[b]
            assert m == row[0]
            assert abi.neumaier_total(agg[b + 1], agg[b + 2]) / m == row[1]
            assert abi.neumaier_total(agg[b + 3], agg[b + 4]) / m == row[2]
            assert agg[b + 5] / m == row[3] and agg[b + 6] / m == row[4] and agg[b + 7] / m == row[5]


def test_golden_runs_bit_exact(golden_runs):
    assert len(golden_runs) >= 40
    for case in golden_runs:
        check_golden(case)


def test_golden_baselines_bit_exact(golden_baselines):
    """Comparison schemes (oracle-static, sys-only, app-only, no-coord;
    policies.py:211-454) against reference-generated goldens."""
    assert len(golden_baselines) >= 50
    assert {c.policy for c in golden_baselines} == {"oracle-static", "sys-only", "app-only", "no-coord"}
    for case in golden_baselines:
        check_golden(case)


def test_golden_goal_changes_bit_exact(golden_goals):
    """Goal changes mid-trace (north_star "goal changes"; the reference's run
    loop with policy.spec swapped, tests/golden/make_golden.py
    run_with_goal_changes): every policy, mode flips, groups, adjacent
    changes, the 64x32 table and random spaces."""
    assert len(golden_goals) >= 20
    assert {c.policy for c in golden_goals} >= {"alert", "alert-any", "alert-trad", "oracle", "oracle-static",
                                               "sys-only", "app-only", "no-coord"}
    flips = 0
    for case in golden_goals:
        assert case.changes
        check_golden(case)
        modes = {case.spec.mode} | {c.mode for _, c in case.changes}
        flips += len(modes) > 1
    assert flips >= 8


def test_published_acceptance_numbers(golden_runs):
    """SURVEY §8(c) / pkg/test_output.txt:18 full-precision values."""
    by = {c.name: c for c in golden_runs}
    _, agg, st = oracle.run(by["preset600_minE_alert"].space, by["preset600_minE_alert"].spec,
                            by["preset600_minE_alert"].env, "alert")
    assert mean_of(agg, abi.AGG_ENERGY) == 1.40175749776675
    assert mean_of(agg, abi.AGG_ACC) == 0.76156
    assert st[0] == 1.3581268590918127 and st[1] == 0.10099019513592786 and st[5] == 0.4995615518070945
    c = by["preset600_minE_oracle"]
    _, agg, _ = oracle.run(c.space, c.spec, c.env, "oracle")
    assert mean_of(agg, abi.AGG_ENERGY) == 1.306446695869797
    c = by["preset600_maxA_pr95_alert"]
    _, agg, _ = oracle.run(c.space, c.spec, c.env, "alert")
    assert mean_of(agg, abi.AGG_ENERGY) == 11.497651962728566
    assert mean_of(agg, abi.AGG_ACC) == 0.9414731820918757
    c = by["preset600_maxA_pr95_oracle"]
    _, agg, _ = oracle.run(c.space, c.spec, c.env, "oracle")
    assert mean_of(agg, abi.AGG_ACC) == 0.955514292695583


def test_golden_predict_and_select(golden_predict):
    mism = 0
    for g in golden_predict:
        preds = oracle.predict_all(g["space"], g["mu"], g["sigma2"], g["phi"], g["spec"], g["goal"])
        ref = g["pred"]
        np.testing.assert_array_equal(preds["pr_deadline"], ref[:, 0])
        np.testing.assert_array_equal(preds["expected_accuracy"], ref[:, 1])
        np.testing.assert_array_equal(preds["energy"], ref[:, 2])
        np.testing.assert_array_equal(preds["latency_mean"], ref[:, 3])
        np.testing.assert_array_equal(preds["latency_sigma"], ref[:, 4])
        i, lvl, _, _ = oracle.select(g["space"], preds, g["spec"])
        j, lvl2 = oracle.brute_force_select(g["space"], preds, g["spec"])
        assert (i, lvl) == (int(g["sel"][0]), int(g["sel"][1]))
        assert j == int(g["sel"][2]) and lvl2 == lvl
        mism += i != j
    assert mism == 0


# --- hand-computed known answers (the reference's unit tests) -----------------

def test_first_kalman_step_hand_values():
    # test_estimator.py:22-35
    mu, s2, k, q, y = oracle.slowdown_update((1.0, 0.1, 0.5, 0.1, 0.0), 1.2, 1.0)
    assert k == pytest.approx(0.15 / 0.151, rel=1e-12)
    assert y == pytest.approx(0.2, rel=1e-12)
    assert mu == pytest.approx(1.0 + (0.15 / 0.151) * 0.2, rel=1e-12)
    assert s2 == pytest.approx(0.15, rel=1e-12) and q == pytest.approx(0.1, rel=1e-12)


def test_idle_step_hand_values():
    # test_estimator.py:98-112
    phi, m = oracle.idle_update(0.5, 0.01, 10.0, 50.0)
    w = 0.0101 / 0.0111
    assert phi == pytest.approx(0.5 + w * (0.2 - 0.5), rel=1e-12)
    assert m == pytest.approx((1.0 - w) * 0.0101, rel=1e-12)
    phi, _ = oracle.idle_update(0.5, 0.01, 80.0, 50.0)
    assert phi == pytest.approx(0.5 + w * 0.5, rel=1e-12)
    with pytest.raises(ValueError):
        oracle.idle_update(0.5, 0.01, 0.0, 50.0)


def test_kalman_rejects_nonpositive():
    with pytest.raises(ValueError):
        oracle.slowdown_update((1.0, 0.1, 0.5, 0.1, 0.0), 0.0, 1.0)


def _one_any():
    return ConfigSpace((DnnProfile("a", DnnKind.ANYTIME, (Stage(0.7, (0.8,)), Stage(0.9, (1.2,))), 0.1),),
                       (PowerSetting(0, 50.0),), 4.0)


def test_anytime_staircase_hand_value():
    # test_predictor.py:110-116: E[q] = 0.705832
    spec = ConstraintSpec(mode=Mode.MINIMIZE_ENERGY, t_goal=1.0, q_goal=0.5)
    preds = oracle.predict_all(_one_any(), 1.0, 0.01, 0.4, spec, 1.0)
    assert preds["expected_accuracy"][1] == pytest.approx(0.705832, abs=1e-6)


def test_energy_hand_values():
    # test_predictor.py:139-157: 35 J, 75 J, 38 J
    sp = ConfigSpace((DnnProfile("t", DnnKind.TRADITIONAL, (Stage(0.9, (0.5,)),), 0.1),),
                     (PowerSetting(0, 50.0),), 4.0)
    spec = ConstraintSpec(mode=Mode.MINIMIZE_ENERGY, t_goal=1.0, q_goal=0.5)
    assert oracle.predict_all(sp, 1.0, 0.0, 0.4, spec, 1.0)["energy"][0] == pytest.approx(35.0)
    assert oracle.predict_all(sp, 3.0, 0.0, 0.4, spec, 1.0)["energy"][0] == pytest.approx(75.0)
    spec_p = ConstraintSpec(mode=Mode.MINIMIZE_ENERGY, t_goal=1.0, q_goal=0.5, pr_threshold=0.841344746068543)
    assert oracle.predict_all(sp, 1.0, 0.04, 0.4, spec_p, 1.0)["energy"][0] == pytest.approx(38.0, abs=1e-6)


def test_deadline_probability_vs_independent_cdf():
    # test_acceptance.py:162-174 (scipy-free: erfc identity at 1e-9)
    rng = np.random.default_rng(5)
    for _ in range(500):
        mu, sig = rng.uniform(0.3, 3.0), rng.uniform(0.005, 0.5)
        t, g = rng.uniform(0.01, 2.0), rng.uniform(0.01, 3.0)
        est = oracle.OracleEst(mu, sig * sig, 0, 0, 0)
        ours = oracle.lib().oracle_deadline_probability(est, t, g)
        ref = 0.5 * math.erfc(-((g - mu * t) / (math.sqrt(sig * sig) * t)) / math.sqrt(2.0))
        assert abs(ours - ref) <= 1e-9


def test_degenerate_sigma_is_step():
    est = oracle.OracleEst(1.0, 0.0, 0, 0, 0)
    assert oracle.lib().oracle_deadline_probability(est, 0.5, 1.0) == 1.0
    assert oracle.lib().oracle_deadline_probability(est, 2.0, 1.0) == 0.0

"""Host-side logic that needs no GPU: synthetic inputs equal the reference's,
packing, spec validation, trace segments."""

import numpy as np
import pytest

import paper_1911_00119_b200 as A
from paper_1911_00119_b200 import abi
from paper_1911_00119_b200.packing import pack_space, pack_specs
from paper_1911_00119_b200.trace import pack_envs, segments_of, unpack_row


def _space_dict(space):
    return {
        "powers": [p.cap_watts for p in space.powers],
        "p_idle_prof": space.p_idle_prof,
        "dnns": [{"id": d.id, "kind": d.kind.value, "q_fail": d.q_fail,
                  "stages": [{"accuracy": s.accuracy, "t_prof": list(s.t_prof)} for s in d.stages]}
                 for d in space.dnns],
    }


def test_generate_space_equals_reference(golden_runs):
    by = {c.name: c for c in golden_runs}
    assert _space_dict(A.preset_space()) == by["preset600_minE_alert"].meta["space"]
    big = A.generate_space(A.ProfileKnobs(n_dnns=64, n_powers=32))
    assert _space_dict(big) == by["big64x32_minE_alert"].meta["space"]
    assert pack_space(big).n_candidates == 2144
    assert pack_space(A.preset_space()).n_candidates == 55
    assert A.reference_latency(A.preset_space()) == 0.677197635411103
    assert A.reference_latency(big) == 0.6262346139703329


def test_realize_equals_reference(golden_runs):
    by = {c.name: c for c in golden_runs}
    env = A.realize(A.preset_trace())
    np.testing.assert_array_equal(env.slowdown, by["preset600_minE_alert"].z["s"])
    np.testing.assert_array_equal(env.idle_power, by["preset600_minE_alert"].z["idle"])


def test_pack_envs_round_trip(golden_runs):
    envs = [c.env for c in golden_runs[:6]]
    n = min(len(e.slowdown) for e in envs)
    envs = [A.TrueEnvironment(e.slowdown[:n], e.idle_power[:n], e.phase_index[:n]) for e in envs]
    p = pack_envs(envs, dtype=np.float64)
    assert p.slowdown.shape == (n, len(envs))
    for r, e in enumerate(envs):
        u = unpack_row(p, r)
        np.testing.assert_array_equal(u.slowdown, e.slowdown)
        np.testing.assert_array_equal(u.idle_power, e.idle_power)
        np.testing.assert_array_equal(u.phase_index, e.phase_index)
    assert segments_of(envs[0])[-1][0] == n


def test_spec_validation_messages():
    with pytest.raises(ValueError, match="t_goal must exceed overhead_budget"):
        A.ConstraintSpec(mode=A.Mode.MINIMIZE_ENERGY, t_goal=0.1, q_goal=0.5, overhead_budget=0.2)
    with pytest.raises(ValueError, match="requires e_goal"):
        A.ConstraintSpec(mode=A.Mode.MAXIMIZE_ACCURACY, t_goal=1.0)
    with pytest.raises(ValueError, match="pr_threshold"):
        A.ConstraintSpec(mode=A.Mode.MINIMIZE_ENERGY, t_goal=1.0, q_goal=0.5, pr_threshold=1.0)


def test_pack_specs_zq_matches_normaldist():
    from statistics import NormalDist

    s = A.ConstraintSpec(mode=A.Mode.MAXIMIZE_ACCURACY, t_goal=1.0, e_goal=3.0, pr_threshold=0.95)
    rec = pack_specs([s], 4)[0]
    assert rec["z_q"] == NormalDist().inv_cdf(0.95)
    assert rec["mode"] == abi.MODE_MAX_ACCURACY and rec["has_pr"] == 1 and rec["group_size"] == 4


def test_invalid_space_rejected():
    bad = A.ConfigSpace((A.DnnProfile("x", A.DnnKind.TRADITIONAL, (A.Stage(0.9, (0.1, 0.2)),), 0.1),),
                        (A.PowerSetting(0, 10.0), A.PowerSetting(1, 20.0)), 4.0)
    with pytest.raises(ValueError, match="latency increases"):
        pack_space(bad)


def test_make_policy_names():
    for n in A.POLICY_NAMES:
        assert A.make_policy(n).name == n
    with pytest.raises(ValueError, match="unknown policy"):
        A.make_policy("greedy")
    assert set(A.POLICY_NAMES) == {"alert", "alert-any", "alert-trad", "oracle", "oracle-static", "sys-only",
                                   "app-only", "no-coord"}  # policies.py:457-466


def test_baseline_dnn_choice_matches_reference_rules():
    """sys-only: fastest final-stage latency at the last power, ties to the
    lower id (model.py:166-176); app-only: most stages, ties to the higher id
    (policies.py:324-329)."""
    from paper_1911_00119_b200.packing import baseline_dnns, pack_space

    space = A.preset_space()
    assert baseline_dnns(space) == (0, 7)  # dnn-00 is the fastest traditional DNN; any-07 the anytime one
    d = pack_space(space).desc
    assert (d.sys_dnn, d.app_dnn) == (0, 7)
    only_any = A.ConfigSpace(tuple(x for x in space.dnns if x.id == "any-07"), space.powers, space.p_idle_prof)
    assert baseline_dnns(only_any) == (-1, 0)
    with pytest.raises(ValueError, match="TRADITIONAL"):
        A.make_policy("sys-only").begin(only_any, None, None)


def test_host_streamer_chunk_schedule():
    """HostStreamer's step chunks: cover the trace exactly, never exceed the
    buffer, short head and tail around full chunks."""
    from paper_1911_00119_b200.simulator import chunk_sizes

    for n in (1, 2, 9, 17, 300, 1000, 10000, 12345):
        for c in (1, 3, 8, 100, 777, 1000, 20000):
            z = chunk_sizes(n, c)
            assert sum(z) == n and min(z) > 0 and max(z) <= min(c, n)
    z = chunk_sizes(10000, 1000)
    assert z[:3] == [125, 175, 244] and z[-1] == 125 and z.count(1000) >= 6
    assert all(b <= 1.4 * a + 1 for a, b in zip(z, z[1:]) if b < 1000)  # geometric head
    assert chunk_sizes(1000, 100)[0] == 12 and chunk_sizes(1000, 100)[-1] == 12
    assert chunk_sizes(300, 777) == [300]
    for n in (9, 1000, 12345):
        z = chunk_sizes(n, 100, tail=False)
        assert sum(z) == n and max(z) <= 100 and (n <= 100 or (z[0] == 12 and z[-1] == 100))  # long last chunk

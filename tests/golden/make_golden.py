"""Generate golden vectors from the REFERENCE implementation (alertsim).

Run in the build container, where /root/reference exists:
    python tests/golden/make_golden.py
Writes tests/golden/golden_runs.npz and tests/golden/golden_predict.npz;
    python tests/golden/make_golden.py --baselines
writes tests/golden/golden_baselines.npz (the comparison schemes
oracle-static / sys-only / app-only / no-coord);
    python tests/golden/make_golden.py --sweeps
writes tests/golden/golden_sweeps.json (cmd_sweep CSV output).
The reference is imported read-only from /root/reference/pkg/src; nothing at
test time reads /root/reference — only these committed fixtures.
"""

from __future__ import annotations

import json
import random
import sys
from dataclasses import replace
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
sys.path.insert(0, "/root/reference/pkg/tests")
sys.dont_write_bytecode = True

import alertsim.simulator as S  # noqa: E402
from alertsim.estimator import KalmanConfig, idle_power_init, slowdown_init  # noqa: E402
from alertsim.model import ConstraintSpec, DnnKind, Mode, space_to_dict  # noqa: E402
from alertsim.policies import AlertPolicy, make_policy  # noqa: E402
from alertsim.predictor import normal_quantile, predict_all  # noqa: E402
from alertsim.selector import brute_force_select, select  # noqa: E402
from alertsim.simulator import (  # noqa: E402
    Constant, EnvironmentPhase, Gaussian, LogNormal, Trace, Uniform, realize, run,
)
from alertsim.synth import ProfileKnobs, generate_space, preset_space, preset_trace, reference_latency  # noqa: E402
from conftest import random_space, random_spec  # noqa: E402

OUT = Path(__file__).resolve().parent


def cand_index(space, i, j, target):
    c = 0
    for di, d in enumerate(space.dnns):
        for pj in range(len(space.powers)):
            targets = [None] if d.kind is DnnKind.TRADITIONAL else list(range(1, len(d.stages) + 1))
            for t in targets:
                if (di, pj, t) == (i, j, target):
                    return c
                c += 1
    raise KeyError


class Recording:
    """Wraps a reference policy to capture filter state after every observe."""

    def __init__(self, inner):
        self.inner = inner
        self.name = inner.name
        self.states = []

    def begin(self, space, spec, env):
        self.inner.begin(space, spec, env)

    def decide(self, index, t_goal):
        return self.inner.decide(index, t_goal)

    def observe(self, record):
        self.inner.observe(record)
        inner = self.inner
        e = getattr(inner, "est", None) or getattr(inner, "est_app", None)
        i = getattr(inner, "idle", None) or getattr(inner, "idle_sys", None)
        if e is not None:
            ip = (i.phi, i.m_var) if i is not None else (np.nan, np.nan)
            self.states.append((e.mu, e.sigma2, e.k_gain, e.q_noise, e.last_innovation) + ip)
        else:
            self.states.append((np.nan,) * 7)


def run_case(space, spec, trace, policy_name, kalman=None, env=None):
    env = env if env is not None else realize(trace)
    orig = S.realize
    S.realize = lambda tr: env
    try:
        pol = Recording(make_policy(policy_name, kalman=kalman))
        res = run(space, spec, trace, pol)
    finally:
        S.realize = orig
    return _records_out(space, res, pol, env)


def _records_out(space, res, pol, env):
    recs = res.records
    out = {
        "cand": np.array([cand_index(space, r.decision.dnn_index, r.decision.power_index,
                                     r.decision.target_stage) for r in recs], np.int32),
        "level": np.array([["none", "dropped-energy", "dropped-accuracy"].index(r.decision.fallback_level.value)
                           for r in recs], np.int32),
        "completed": np.array([r.completed_stage for r in recs], np.int32),
        "met": np.array([r.deadline_met for r in recs], np.int32),
        "viol": np.array([(r.violations.latency, r.violations.accuracy, r.violations.energy) for r in recs],
                         np.int32),
        "period": np.array([r.period for r in recs]),
        "feasible": np.array([r.decision.feasible for r in recs], np.int32),
        # ConfigDecision.prediction (selector.py:122-128 / policies.py:201-428)
        "pred": np.array([(r.decision.prediction.latency_mean, r.decision.prediction.latency_sigma,
                           r.decision.prediction.pr_deadline, r.decision.prediction.expected_accuracy,
                           r.decision.prediction.energy) for r in recs]),
        "latency": np.array([r.observed_latency for r in recs]),
        "accuracy": np.array([r.delivered_accuracy for r in recs]),
        "energy": np.array([r.energy for r in recs]),
        "fb": np.array([(r.fb_latency, r.fb_t_prof) for r in recs]),
        "state": np.array(pol.states),
        "s": np.asarray(env.slowdown, np.float64),
        "idle": np.asarray(env.idle_power, np.float64),
        "phase": np.asarray(env.phase_index, np.int32),
        "summary": np.array([res.summary.mean_energy, res.summary.mean_accuracy,
                             res.summary.violation_rates["latency"], res.summary.violation_rates["accuracy"],
                             res.summary.violation_rates["energy"]]),
        "phase_summary": np.array([[p.length, p.mean_energy, p.mean_accuracy, p.violation_rates["latency"],
                                    p.violation_rates["accuracy"], p.violation_rates["energy"]]
                                   for p in res.summary.per_phase]),
    }
    return out


def run_with_goal_changes(space, spec, trace, policy, changes, kalman=None, env=None):
    """simulator.run (simulator.py:461-507) with goal changes mirrored as
    SURVEY §7 hard part 8 prescribes: at input n >= change step the loop's
    spec is replaced, policy.spec is swapped before decide (read there,
    policies.py:97-103 / 160-205), plan_goal is recomputed from the new spec
    exactly as simulator.py:473-483 does, and the input is measured against
    it.  Everything else is the reference's own code, called unchanged."""
    from alertsim.selector import GroupState, InfeasibleDeadlineError, adjust_goal
    from alertsim.simulator import RunResult, _summarize, execute_decision, measure

    env = env if env is not None else realize(trace)
    policy.begin(space, spec, env)
    records = []
    group = None
    cur = spec
    pending = sorted(changes, key=lambda c: c[0])
    for n in range(trace.length):
        while pending and pending[0][0] <= n:
            cur = pending.pop(0)[1]
            policy.spec = cur
        if trace.group_size is not None:
            if group is None or group.remaining_count == 0:
                group = GroupState(remaining_budget=trace.group_size * cur.t_goal,
                                   remaining_count=trace.group_size)
        try:
            plan_goal = adjust_goal(cur, group)
        except InfeasibleDeadlineError:
            plan_goal = 0.001
        period = plan_goal + cur.overhead_budget
        decision = policy.decide(n, plan_goal)
        s = float(env.slowdown[n])
        outcome = execute_decision(s, decision, space, plan_goal)
        record = measure(decision, outcome, cur, float(env.idle_power[n]), space, input_index=n,
                         phase_index=int(env.phase_index[n]), period=period)
        records.append(record)
        policy.observe(record)
        if group is not None:
            group.remaining_budget -= record.observed_latency
            group.remaining_count -= 1
    return RunResult(records=tuple(records), summary=_summarize(records, len(trace.phases)))


def goal_changes():
    """Golden runs with goal changes (north_star "goal changes" as a trace
    input; SURVEY §7 hard part 8): specs swap mid-trace, including mode flips,
    group budgets and pr_threshold toggles, for every policy."""
    space = preset_space()
    ref = reference_latency(space)
    oh = 0.01 * ref
    e_min = ConstraintSpec(mode=Mode.MINIMIZE_ENERGY, t_goal=0.14, q_goal=0.68, overhead_budget=oh)
    e_tight = ConstraintSpec(mode=Mode.MINIMIZE_ENERGY, t_goal=0.6 * ref, q_goal=0.85, overhead_budget=oh)
    a_pr = ConstraintSpec(mode=Mode.MAXIMIZE_ACCURACY, t_goal=0.8 * ref, e_goal=0.6 * 50.0 * 0.8 * ref,
                          pr_threshold=0.95, overhead_budget=oh)
    a_loose = ConstraintSpec(mode=Mode.MAXIMIZE_ACCURACY, t_goal=1.5 * ref, e_goal=0.4 * 50.0 * 1.5 * ref,
                             overhead_budget=oh)
    cases = []
    tr = preset_trace(phase_length=100)
    sched_a = [(60, e_tight), (140, a_pr), (220, e_min)]        # mode flips
    sched_b = [(1, a_loose), (150, a_pr), (151, e_tight), (299, e_min)]  # adjacent changes, last input
    for pol in ("alert", "alert-any", "alert-trad", "oracle", "oracle-static", "sys-only", "app-only", "no-coord"):
        cases.append((f"flip_{pol}", space, e_min, tr, pol, None, sched_a))
    cases.append(("adjacent_alert", space, a_pr, tr, "alert", None, sched_b))
    cases.append(("adjacent_oracle", space, a_pr, tr, "oracle", None, sched_b))
    trg = replace(preset_trace(phase_length=40), group_size=4)
    cases.append(("group4_alert", space, e_min, trg, "alert", None, [(37, e_tight), (90, a_pr)]))
    cases.append(("group4_no-coord", space, e_min, trg, "no-coord", None, [(37, e_tight), (90, a_pr)]))
    big = generate_space(ProfileKnobs(n_dnns=64, n_powers=32))
    bref = reference_latency(big)
    bmin = ConstraintSpec(mode=Mode.MINIMIZE_ENERGY, t_goal=1.0 * bref, q_goal=0.8, overhead_budget=0.01 * bref)
    bacc = ConstraintSpec(mode=Mode.MAXIMIZE_ACCURACY, t_goal=0.8 * bref, e_goal=0.6 * 50.0 * 0.8 * bref,
                          overhead_budget=0.01 * bref)
    btr = preset_trace(phase_length=20)
    cases.append(("big64x32_alert", big, bmin, btr, "alert", None, [(25, bacc), (41, bmin)]))
    rnd = random.Random(4242)
    for k in range(12):
        rs = random_space(rnd)
        specs = [random_spec(rnd) for _ in range(3)]
        specs = [replace(sp, overhead_budget=rnd.choice([0.0, 0.01 * sp.t_goal])) for sp in specs]
        trr = random_trace(rnd, 80)
        pol = ["alert", "oracle", "alert-any", "sys-only"][k % 4]
        if pol == "alert-any" and not any(d.kind is DnnKind.ANYTIME for d in rs.dnns):
            pol = "alert"
        if pol == "sys-only" and not any(d.kind is DnnKind.TRADITIONAL for d in rs.dnns):
            pol = "alert"
        steps = sorted(rnd.sample(range(1, 80), 2))
        cases.append((f"random{k:02d}_{pol}", rs, specs[0], trr, pol, None,
                      [(steps[0], specs[1]), (steps[1], specs[2])]))
    arrays, meta = {}, []
    for name, sp, spec, tr_, pol, kal, sched in cases:
        env = realize(tr_)
        pobj = Recording(make_policy(pol, kalman=kal))
        # Recording forwards spec swaps to the wrapped policy
        res = run_with_goal_changes(sp, spec, tr_, _SpecForward(pobj), sched, env=env)
        out = _records_out(sp, res, pobj, env)
        for key, val in out.items():
            arrays[f"{name}/{key}"] = val
        meta.append({"name": name, "space": space_to_dict(sp), "spec": spec_json(spec, tr_.group_size),
                     "changes": [[int(n), spec_json(c, tr_.group_size)] for n, c in sched],
                     "policy": pol, "kalman": kalman_json(kal), "n_phases": len(tr_.phases)})
        print(name, "E", out["summary"][0], "acc", out["summary"][1])
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), np.uint8)
    np.savez_compressed(OUT / "golden_goals.npz", **arrays)


class _SpecForward:
    """Policy wrapper whose ``spec`` assignments reach the wrapped reference policy."""

    def __init__(self, rec):
        self.rec = rec
        self.name = rec.name

    def __setattr__(self, key, value):
        if key == "spec":
            self.rec.inner.spec = value
        else:
            object.__setattr__(self, key, value)

    def begin(self, space, spec, env):
        self.rec.begin(space, spec, env)

    def decide(self, index, t_goal):
        return self.rec.decide(index, t_goal)

    def observe(self, record):
        self.rec.observe(record)


def spec_json(spec, group_size=None):
    return {"mode": spec.mode.value, "t_goal": spec.t_goal, "e_goal": spec.e_goal, "q_goal": spec.q_goal,
            "pr_threshold": spec.pr_threshold, "overhead_budget": spec.overhead_budget,
            "group_size": group_size}


def kalman_json(k):
    return None if k is None else {f: getattr(k, f) for f in
                                   ("k0", "r", "q0", "alpha", "mu0", "sigma2_0", "sigma2_uses_current_gain")}


def random_trace(rnd, n):
    phases = []
    left = n
    while left > 0:
        L = min(left, rnd.randint(5, max(6, n // 2)))
        kind = rnd.choice(["c", "g", "l", "u"])
        if kind == "c":
            d = Constant(rnd.uniform(0.5, 2.5))
        elif kind == "g":
            d = Gaussian(rnd.uniform(0.6, 2.0), rnd.uniform(0.01, 0.5))
        elif kind == "l":
            d = LogNormal(rnd.uniform(-0.3, 0.8), rnd.uniform(0.05, 0.5))
        else:
            lo = rnd.uniform(0.3, 1.5)
            d = Uniform(lo, lo + rnd.uniform(0.1, 1.5))
        phases.append(EnvironmentPhase(L, d, rnd.uniform(1.0, 12.0), rnd.choice([0.0, 0.05, 0.2])))
        left -= L
    return Trace(seed=rnd.randint(0, 10**6), phases=tuple(phases[:8]),
                 group_size=rnd.choice([None, None, None, rnd.randint(1, 6)]))


def main():
    cases = []  # (name, space, spec, trace, policy, kalman)
    space = preset_space()
    ref = reference_latency(space)
    tr600 = preset_trace()
    c1 = ConstraintSpec(mode=Mode.MINIMIZE_ENERGY, t_goal=0.14, q_goal=0.68, overhead_budget=0.01 * ref)
    for pol in ("alert", "alert-any", "alert-trad", "oracle"):
        cases.append((f"preset600_minE_{pol}", space, c1, tr600, pol, None))
    tmax = 0.8 * ref
    cmax = ConstraintSpec(mode=Mode.MAXIMIZE_ACCURACY, t_goal=tmax, e_goal=0.6 * 50.0 * tmax,
                          pr_threshold=0.95, overhead_budget=0.01 * ref)
    for pol in ("alert", "alert-any", "oracle"):
        cases.append((f"preset600_maxA_pr95_{pol}", space, cmax, tr600, pol, None))
    tr1000 = Trace(seed=42, phases=tuple(
        EnvironmentPhase(n, p.slowdown_dist, p.idle_power_true, p.input_noise_sd)
        for n, p in zip((334, 333, 333), tr600.phases)))
    for dm in (0.4, 0.8, 1.2, 1.6, 2.0):
        for q in (0.70, 0.85):
            sp = ConstraintSpec(mode=Mode.MINIMIZE_ENERGY, t_goal=dm * ref, q_goal=q, overhead_budget=0.01 * ref)
            cases.append((f"c1_1000_dm{dm}_q{q}", space, sp, tr1000, "alert", None))
        for em in (0.5, 0.8):
            sp = ConstraintSpec(mode=Mode.MAXIMIZE_ACCURACY, t_goal=dm * ref, e_goal=em * 50.0 * dm * ref,
                                pr_threshold=0.95 if dm != 1.2 else None, overhead_budget=0.01 * ref)
            cases.append((f"c1_1000_dm{dm}_e{em}", space, sp, tr1000, "alert", None))
    trg = replace(preset_trace(phase_length=40), group_size=4)
    cases.append(("group4_minE", space, c1, trg, "alert", None))
    cases.append(("group4_minE_oracle", space, c1, trg, "oracle", None))
    cases.append(("kalman_variant", space, c1, preset_trace(phase_length=50), "alert",
                  KalmanConfig(q0=0.02, r=0.01, alpha=0.5, sigma2_uses_current_gain=True)))
    # large table (64 x 32, 2,144 candidates), short trace
    big = generate_space(ProfileKnobs(n_dnns=64, n_powers=32))
    bref = reference_latency(big)
    bsp = ConstraintSpec(mode=Mode.MINIMIZE_ENERGY, t_goal=1.0 * bref, q_goal=0.8, overhead_budget=0.01 * bref)
    btr = preset_trace(phase_length=20)
    cases.append(("big64x32_minE_alert", big, bsp, btr, "alert", None))
    cases.append(("big64x32_minE_oracle", big, bsp, btr, "oracle", None))
    bsp2 = ConstraintSpec(mode=Mode.MAXIMIZE_ACCURACY, t_goal=0.8 * bref, e_goal=0.6 * 50.0 * 0.8 * bref,
                          pr_threshold=0.95, overhead_budget=0.01 * bref)
    cases.append(("big64x32_maxA_alert", big, bsp2, btr, "alert", None))
    # randomized spaces / specs / traces (reference conftest generators)
    rnd = random.Random(20261017)
    for k in range(24):
        rs = random_space(rnd)
        spc = random_spec(rnd)
        spc = replace(spc, overhead_budget=rnd.choice([0.0, 0.01 * spc.t_goal]))
        tr = random_trace(rnd, 80)
        pol = ["alert", "oracle", "alert-any", "alert-trad"][k % 4]
        if pol == "alert-any" and not any(d.kind is DnnKind.ANYTIME for d in rs.dnns):
            pol = "alert"
        if pol == "alert-trad" and not any(d.kind is DnnKind.TRADITIONAL for d in rs.dnns):
            pol = "alert"
        cases.append((f"random{k:02d}_{pol}", rs, spc, tr, pol, None))

    arrays = {}
    meta = []
    for name, sp, spec, tr, pol, kal in cases:
        out = run_case(sp, spec, tr, pol, kal)
        for key, val in out.items():
            arrays[f"{name}/{key}"] = val
        meta.append({"name": name, "space": space_to_dict(sp), "spec": spec_json(spec, tr.group_size),
                     "policy": pol, "kalman": kalman_json(kal), "n_phases": len(tr.phases)})
        print(name, "E", out["summary"][0], "acc", out["summary"][1])
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), np.uint8)
    np.savez_compressed(OUT / "golden_runs.npz", **arrays)

    # predict_all / select / brute_force_select on random instances (conftest.py:74-82)
    rnd = random.Random(987654)
    pmeta, parr = [], {}
    for k in range(300):
        rs = random_space(rnd)
        spc = random_spec(rnd)
        est = replace(slowdown_init(), mu=rnd.uniform(0.3, 3.0), sigma2=rnd.uniform(0.0, 0.6))
        if k % 10 == 0:
            est = replace(est, sigma2=0.0)
        idle = replace(idle_power_init(0.5), phi=rnd.uniform(0.0, 1.0))
        goal = spc.t_goal * rnd.choice([1.0, 0.5, 1.3])
        preds = predict_all(rs, est, idle, spc, goal)
        d = select(preds, spc)
        b = brute_force_select(preds, spc)
        parr[f"{k}/pred"] = np.array([(p.pr_deadline, p.expected_accuracy, p.energy, p.latency_mean,
                                       p.latency_sigma) for p in preds])
        parr[f"{k}/sel"] = np.array([cand_index(rs, d.dnn_index, d.power_index, d.target_stage),
                                     ["none", "dropped-energy", "dropped-accuracy"].index(d.fallback_level.value),
                                     cand_index(rs, b.dnn_index, b.power_index, b.target_stage)], np.int32)
        pmeta.append({"space": space_to_dict(rs), "spec": spec_json(spc), "mu": est.mu, "sigma2": est.sigma2,
                      "phi": idle.phi, "goal": goal,
                      "z_q": normal_quantile(spc.pr_threshold) if spc.pr_threshold is not None else None})
    parr["meta"] = np.frombuffer(json.dumps(pmeta).encode(), np.uint8)
    np.savez_compressed(OUT / "golden_predict.npz", **parr)


def baselines():
    """Golden runs of the comparison schemes (policies.py:211-454)."""
    cases = []
    space = preset_space()
    ref = reference_latency(space)
    tr600 = preset_trace()
    c1 = ConstraintSpec(mode=Mode.MINIMIZE_ENERGY, t_goal=0.14, q_goal=0.68, overhead_budget=0.01 * ref)
    tmax = 0.8 * ref
    cmax = ConstraintSpec(mode=Mode.MAXIMIZE_ACCURACY, t_goal=tmax, e_goal=0.6 * 50.0 * tmax,
                          pr_threshold=0.95, overhead_budget=0.01 * ref)
    pols = ("oracle-static", "sys-only", "app-only", "no-coord")
    for pol in pols:
        cases.append((f"preset600_minE_{pol}", space, c1, tr600, pol, None))
        cases.append((f"preset600_maxA_pr95_{pol}", space, cmax, tr600, pol, None))
    for dm in (0.4, 1.0, 2.0):
        sp = ConstraintSpec(mode=Mode.MINIMIZE_ENERGY, t_goal=dm * ref, q_goal=0.85, overhead_budget=0.01 * ref)
        for pol in pols:
            cases.append((f"preset300_dm{dm}_{pol}", space, sp, preset_trace(phase_length=100), pol, None))
    trg = replace(preset_trace(phase_length=40), group_size=4)
    for pol in pols:
        cases.append((f"group4_minE_{pol}", space, c1, trg, pol, None))
    cases.append(("kalman_variant_no-coord", space, c1, preset_trace(phase_length=50), "no-coord",
                  KalmanConfig(q0=0.02, r=0.01, alpha=0.5, sigma2_uses_current_gain=True)))
    rnd = random.Random(5150)
    k = 0
    while len(cases) < 60:
        rs = random_space(rnd)
        spc = random_spec(rnd)
        spc = replace(spc, overhead_budget=rnd.choice([0.0, 0.01 * spc.t_goal]))
        tr = random_trace(rnd, 60)
        pol = pols[k % 4]
        k += 1
        has_t = any(d.kind is DnnKind.TRADITIONAL for d in rs.dnns)
        has_a = any(d.kind is DnnKind.ANYTIME for d in rs.dnns)
        if (pol == "sys-only" and not has_t) or (pol in ("app-only", "no-coord") and not has_a):
            continue
        cases.append((f"random{k:02d}_{pol}", rs, spc, tr, pol, None))
    arrays, meta = {}, []
    for name, sp, spec, tr, pol, kal in cases:
        out = run_case(sp, spec, tr, pol, kal)
        for key, val in out.items():
            arrays[f"{name}/{key}"] = val
        meta.append({"name": name, "space": space_to_dict(sp), "spec": spec_json(spec, tr.group_size),
                     "policy": pol, "kalman": kalman_json(kal), "n_phases": len(tr.phases)})
        print(name, "E", out["summary"][0], "acc", out["summary"][1])
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), np.uint8)
    np.savez_compressed(OUT / "golden_baselines.npz", **arrays)


def sweeps():
    """CSV output of the reference's cmd_sweep (cli.py:191-274) on the preset
    profile / preset trace (phase_length 100), for the GPU sweep driver."""
    import tempfile

    from alertsim.cli import main as cli_main
    from alertsim.model import save_profile
    from alertsim.simulator import save_trace

    pols = "alert,alert-any,alert-trad,oracle,oracle-static,sys-only,app-only,no-coord"
    runs = [
        dict(mode="min-energy", goals="0.7,0.85", pr_th=None, seed=None),
        dict(mode="max-accuracy", goals="0.5,0.8", pr_th=0.95, seed=None),
        dict(mode="min-energy", goals="0.68", pr_th=None, seed=7),
    ]
    out = []
    with tempfile.TemporaryDirectory() as d:
        prof, tr = Path(d) / "profile.json", Path(d) / "trace.json"
        save_profile(preset_space(), prof)
        save_trace(preset_trace(phase_length=100), tr)
        for r in runs:
            csv_path = Path(d) / "sweep.csv"
            argv = ["sweep", "--profile", str(prof), "--trace", str(tr), "--mode", r["mode"],
                    "--q-goals" if r["mode"] == "min-energy" else "--e-goal-mults", r["goals"],
                    "--policies", pols, "--out", str(csv_path)]
            if r["pr_th"] is not None:
                argv += ["--pr-th", str(r["pr_th"])]
            if r["seed"] is not None:
                argv += ["--seed", str(r["seed"])]
            assert cli_main(argv) == 0
            out.append(dict(r, policies=pols, phase_length=100, csv=csv_path.read_text()))
            print(r, len(out[-1]["csv"].splitlines()), "rows")
    (OUT / "golden_sweeps.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    if "--sweeps" in sys.argv:
        sweeps()
    elif "--goals" in sys.argv:
        goal_changes()
    elif "--baselines" in sys.argv:
        baselines()
    else:
        main()

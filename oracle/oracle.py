"""ctypes wrapper of oracle/liboracle.so — the CPU restatement of the
reference hot path.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs, as the checker / timed CPU baseline.  The
product package never imports this module.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

from paper_1911_00119_b200 import abi
from paper_1911_00119_b200.packing import filter_config, pack_space, pack_specs, policy_code, spec_struct

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "liboracle.so"
STATE_FIELDS = 10  # ORACLE_STATE_FIELDS: mu sigma2 k q y phi m budget count aux

RECORD_DTYPE = np.dtype(
    [(n, "<i4") for n in ("cand", "dnn", "power", "stage", "level", "completed", "met", "phase",
                          "viol_lat", "viol_acc", "viol_energy", "or_cand", "feasible", "spec_index")]
    + [(n, "<f8") for n in ("plan_goal", "period", "latency", "accuracy", "energy", "fb_latency",
                            "fb_t_prof", "s", "mu", "sigma2", "k_gain", "q_noise", "innov", "phi",
                            "m_var", "gap", "boundary", "pred_latency_mean", "pred_latency_sigma", "pred_pr",
                            "pred_accuracy", "pred_energy")]
)


class OracleEst(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("mu", "sigma2", "k_gain", "q_noise", "innov")]


class OracleIdle(C.Structure):
    _fields_ = [("phi", C.c_double), ("m_var", C.c_double)]


def build(force: bool = False) -> Path:
    src = HERE / "alert_oracle.c"
    if force or not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE), "liboracle.so"], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = C.CDLL(str(LIB_PATH))
        P = C.POINTER
        L.oracle_num_candidates.argtypes = [P(abi.AlertSpaceDesc)]
        L.oracle_normal_cdf.argtypes = [C.c_double]
        L.oracle_normal_cdf.restype = C.c_double
        L.oracle_deadline_probability.argtypes = [P(OracleEst), C.c_double, C.c_double]
        L.oracle_deadline_probability.restype = C.c_double
        L.oracle_expected_accuracy_anytime.argtypes = [P(abi.AlertSpaceDesc), P(OracleEst), C.c_int,
                                                       C.c_int, C.c_int, C.c_double]
        L.oracle_expected_accuracy_anytime.restype = C.c_double
        L.oracle_energy_mean.argtypes = [P(OracleEst), P(OracleIdle), C.c_double, C.c_double, C.c_double]
        L.oracle_energy_mean.restype = C.c_double
        L.oracle_energy_percentile.argtypes = [P(OracleEst), P(OracleIdle), C.c_double, C.c_double,
                                               C.c_double, C.c_double]
        L.oracle_energy_percentile.restype = C.c_double
        L.oracle_predict_all.argtypes = [P(abi.AlertSpaceDesc), P(OracleEst), P(OracleIdle),
                                         P(abi.AlertSpec), C.c_double, C.c_void_p]
        L.oracle_select.argtypes = [P(abi.AlertSpaceDesc), C.c_void_p, C.c_int, P(abi.AlertSpec), C.c_int,
                                    P(C.c_int32), P(C.c_double), P(C.c_double)]
        L.oracle_brute_force_select.argtypes = [P(abi.AlertSpaceDesc), C.c_void_p, C.c_int,
                                                P(abi.AlertSpec), C.c_int, P(C.c_int32)]
        L.oracle_slowdown_init.argtypes = [P(abi.AlertFilterConfig), P(OracleEst)]
        L.oracle_slowdown_init.restype = None
        L.oracle_slowdown_update.argtypes = [P(abi.AlertFilterConfig), P(OracleEst), C.c_double, C.c_double]
        L.oracle_idle_update.argtypes = [P(abi.AlertFilterConfig), P(OracleIdle), C.c_double, C.c_double]
        L.oracle_adjust_goal.argtypes = [P(abi.AlertSpec), C.c_int, C.c_double, C.c_int32]
        L.oracle_adjust_goal.restype = C.c_double
        L.oracle_oracle_decide.argtypes = [P(abi.AlertSpaceDesc), P(abi.AlertSpec), C.c_double, C.c_double,
                                           C.c_double, P(C.c_int32), P(C.c_double)]
        L.oracle_run.argtypes = [P(abi.AlertSpaceDesc), P(abi.AlertSpec), P(abi.AlertFilterConfig), C.c_int,
                                 C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.c_void_p, C.c_int]
        L.oracle_run_goals.argtypes = [P(abi.AlertSpaceDesc), C.c_void_p, C.c_int32, C.c_void_p,
                                       P(abi.AlertFilterConfig), C.c_int, C.c_int64, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
        L.oracle_run_batch.argtypes = [P(abi.AlertSpaceDesc), C.c_void_p, C.c_int32, C.c_void_p,
                                       P(abi.AlertFilterConfig), C.c_int, P(abi.AlertTrace), C.c_int64,
                                       C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_int]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _packed(space):
    return space if hasattr(space, "desc") else pack_space(space)


def run(space, spec, env, policy: str = "alert", kalman=None, forced=None, group_size=None,
        state=None, goal_changes=None):
    """simulator.run over an injected environment (TrueEnvironment-like with
    slowdown / idle_power / phase_index).  Returns (records, agg, state).
    goal_changes: [(input_index, ConstraintSpec), ...] swaps the spec from
    that input on (oracle_run_goals)."""
    if goal_changes:
        specs = [spec] + [c for _, c in goal_changes]
        idx = np.zeros(len(env.slowdown), np.int32)
        for k, (n0, _) in enumerate(goal_changes):
            idx[int(n0):] = k + 1
        return run_goals(space, pack_specs(specs, group_size), idx, env, policy, kalman, forced, state)
    ps = _packed(space)
    rec = pack_specs([spec], group_size)[0]
    s = np.ascontiguousarray(env.slowdown, dtype=np.float64)
    idle = np.ascontiguousarray(env.idle_power, dtype=np.float64)
    ph = np.ascontiguousarray(env.phase_index, dtype=np.int32)
    n = len(s)
    f = None if forced is None else np.ascontiguousarray(forced, dtype=np.int32)
    records = np.zeros(n, RECORD_DTYPE)
    agg = np.zeros(abi.AGG_FIELDS, np.float64)
    st = np.zeros(STATE_FIELDS, np.float64) if state is None else np.array(state, np.float64)
    cfg = filter_config(kalman)
    sp = spec_struct(rec)
    r = lib().oracle_run(C.byref(ps.desc), C.byref(sp), C.byref(cfg), policy_code(policy), n,
                         _p(s), _p(idle), _p(ph), _p(f), _p(records), _p(agg), _p(st),
                         int(state is not None))
    if r != 0:
        raise ValueError(f"oracle_run failed: {abi.STATUS_NAMES.get(r, r)}")
    return records, agg, st


def run_goals(space, spec_records, spec_index, env, policy: str = "alert", kalman=None, forced=None, state=None):
    """oracle_run_goals: step n under spec_records[spec_index[n]]."""
    ps = _packed(space)
    specs = np.ascontiguousarray(spec_records)
    idx = np.ascontiguousarray(spec_index, dtype=np.int32)
    s = np.ascontiguousarray(env.slowdown, dtype=np.float64)
    idle = np.ascontiguousarray(env.idle_power, dtype=np.float64)
    ph = np.ascontiguousarray(env.phase_index, dtype=np.int32)
    n = len(s)
    f = None if forced is None else np.ascontiguousarray(forced, dtype=np.int32)
    records = np.zeros(n, RECORD_DTYPE)
    agg = np.zeros(abi.AGG_FIELDS, np.float64)
    st = np.zeros(STATE_FIELDS, np.float64) if state is None else np.array(state, np.float64)
    cfg = filter_config(kalman)
    r = lib().oracle_run_goals(C.byref(ps.desc), _p(specs), len(specs), _p(idx), C.byref(cfg), policy_code(policy),
                               n, _p(s), _p(idle), _p(ph), _p(f), _p(records), _p(agg), _p(st),
                               int(state is not None))
    if r != 0:
        raise ValueError(f"oracle_run_goals failed: {abi.STATUS_NAMES.get(r, r)}")
    return records, agg, st


def predict_all(space, mu, sigma2, phi, spec, goal):
    ps = _packed(space)
    est = OracleEst(mu, sigma2, 0.0, 0.0, 0.0)
    idle = OracleIdle(phi, 0.0)
    out = np.zeros(ps.n_candidates, abi.PREDICTION_DTYPE)
    sp = spec_struct(pack_specs([spec])[0])
    n = lib().oracle_predict_all(C.byref(ps.desc), C.byref(est), C.byref(idle), C.byref(sp), goal, _p(out))
    return out[:n]


def select(space, preds, spec, kinds_mask=3):
    ps = _packed(space)
    sp = spec_struct(pack_specs([spec])[0])
    lvl, gap, bnd = C.c_int32(), C.c_double(), C.c_double()
    preds = np.ascontiguousarray(preds)
    i = lib().oracle_select(C.byref(ps.desc), _p(preds), len(preds), C.byref(sp), kinds_mask,
                            C.byref(lvl), C.byref(gap), C.byref(bnd))
    return i, lvl.value, gap.value, bnd.value


def brute_force_select(space, preds, spec, kinds_mask=3):
    ps = _packed(space)
    sp = spec_struct(pack_specs([spec])[0])
    lvl = C.c_int32()
    preds = np.ascontiguousarray(preds)
    i = lib().oracle_brute_force_select(C.byref(ps.desc), _p(preds), len(preds), C.byref(sp),
                                        kinds_mask, C.byref(lvl))
    return i, lvl.value


def slowdown_update(est: tuple, obs: float, t_prof: float, kalman=None):
    e = OracleEst(*est)
    if lib().oracle_slowdown_update(C.byref(filter_config(kalman)), C.byref(e), obs, t_prof):
        raise ValueError("observed_latency and t_prof_used must be positive")
    return (e.mu, e.sigma2, e.k_gain, e.q_noise, e.innov)


def idle_update(phi: float, m_var: float, measured: float, cap: float, idle_cfg=None):
    st = OracleIdle(phi, m_var)
    if lib().oracle_idle_update(C.byref(filter_config(None, idle_cfg)), C.byref(st), measured, cap):
        raise ValueError("power measurements must be positive")
    return st.phi, st.m_var


def oracle_decide(space, spec, s, idle, goal):
    ps = _packed(space)
    sp = spec_struct(pack_specs([spec])[0])
    lvl, gap = C.c_int32(), C.c_double()
    c = lib().oracle_oracle_decide(C.byref(ps.desc), C.byref(sp), s, idle, goal, C.byref(lvl), C.byref(gap))
    return c, lvl.value


def host_trace_struct(packed, stream_row=None):
    """AlertTrace over HOST arrays of a trace.PackedEnvs (for run_batch)."""
    keep = [packed.slowdown, packed.n_segments, packed.seg_end, packed.seg_phase, packed.seg_idle]
    sr = None if stream_row is None else np.ascontiguousarray(stream_row, np.int32)
    keep.append(sr)
    t = abi.AlertTrace(
        slowdown=packed.slowdown.ctypes.data,
        slowdown_dtype=abi.DTYPE_F64 if packed.slowdown.dtype == np.float64 else abi.DTYPE_F32,
        n_rows=packed.n_rows, n_steps=packed.n_steps, row_stride=1, step_stride=packed.n_rows,
        step_offset=0, max_segments=packed.seg_end.shape[1], _pad=0,
        n_segments=packed.n_segments.ctypes.data, seg_end=packed.seg_end.ctypes.data,
        seg_phase=packed.seg_phase.ctypes.data, seg_idle=packed.seg_idle.ctypes.data,
        stream_row=None if sr is None else sr.ctypes.data,
    )
    if getattr(packed, "goal_n", None) is not None:  # goal changes
        g = [np.ascontiguousarray(a, np.int32) for a in (packed.goal_n, packed.goal_end, packed.goal_spec)]
        keep += g
        t.max_goal_segments = g[1].shape[1]
        t.n_goal_segments, t.goal_seg_end, t.goal_seg_spec = (a.ctypes.data for a in g)
    return t, keep


def run_batch(space, spec_records, packed_envs, n_streams, policy="alert", kalman=None,
              stream_spec=None, stream_row=None, step_begin=0, step_end=None, threads=None,
              state=None):
    """Multi-threaded CPU runs of many streams (aggregates + final state)."""
    ps = _packed(space)
    specs = np.ascontiguousarray(spec_records)
    tr, keep = host_trace_struct(packed_envs, stream_row)
    ss = None if stream_spec is None else np.ascontiguousarray(stream_spec, np.int32)
    agg = np.zeros((n_streams, abi.AGG_FIELDS), np.float64)
    st = np.zeros((n_streams, STATE_FIELDS), np.float64) if state is None else state
    end = packed_envs.n_steps if step_end is None else step_end
    cfg = filter_config(kalman)
    r = lib().oracle_run_batch(C.byref(ps.desc), _p(specs), len(specs), _p(ss), C.byref(cfg),
                               policy_code(policy), C.byref(tr), n_streams, step_begin, end, _p(agg),
                               _p(st), threads or os.cpu_count() or 1)
    if r != 0:
        raise ValueError(f"oracle_run_batch failed: {abi.STATUS_NAMES.get(r, r)}")
    del keep
    return agg, st

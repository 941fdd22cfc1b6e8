"""Flatten host model objects into the C-ABI structs (include/alert_b200.h).

* ``pack_space``   ConfigSpace  -> AlertSpaceDesc (+ the candidate list in the
                   reference enumeration order, policies.py:59-67 /
                   predictor.py:162-168).
* ``pack_specs``   ConstraintSpec(s) -> AlertSpec array (z_q computed here with
                   statistics.NormalDist, exactly as predictor.py:30-33 does).
* ``filter_config`` KalmanConfig + IdleFilterConfig -> AlertFilterConfig.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from statistics import NormalDist
from typing import Sequence

import numpy as np

from . import abi
from .estimator import IdleFilterConfig, KalmanConfig
from .model import DnnKind, Mode, check_spec, kind_of, mode_of, validate


class ProfileError(ValueError):
    """Config space violating model.validate invariants (model.py:191-192)."""


@dataclass
class PackedSpace:
    desc: abi.AlertSpaceDesc
    arrays: dict            # keeps the numpy buffers alive
    candidates: np.ndarray  # [n_cand, 3] (dnn, power, target stage; 0 = None)
    space: object

    @property
    def n_candidates(self) -> int:
        return len(self.candidates)


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def pack_space(space, check: bool = True) -> PackedSpace:
    if check:
        problems = validate(space)
        if problems:
            raise ProfileError("invalid profile: " + "; ".join(problems))
    dnns = list(space.dnns)
    n_powers = len(space.powers)
    kinds = np.array([abi.KIND_ANYTIME if kind_of(d) is DnnKind.ANYTIME else abi.KIND_TRADITIONAL
                      for d in dnns], np.int32)
    n_stages = np.array([len(d.stages) for d in dnns], np.int32)
    if (n_stages > abi.MAX_STAGES).any():
        raise ValueError(f"at most {abi.MAX_STAGES} stages per DNN are supported")
    q_fail = np.array([float(d.q_fail) for d in dnns], np.float64)
    acc = np.array([float(st.accuracy) for d in dnns for st in d.stages], np.float64)
    t_prof = np.array([[float(t) for t in st.t_prof] for d in dnns for st in d.stages],
                      np.float64).reshape(-1, n_powers)
    caps = np.array([float(p.cap_watts) for p in space.powers], np.float64)
    cands = []
    for i, d in enumerate(dnns):
        for j in range(n_powers):
            if kinds[i] == abi.KIND_TRADITIONAL:
                cands.append((i, j, 0))
            else:
                cands.extend((i, j, k) for k in range(1, len(d.stages) + 1))
    cands = np.array(cands, np.int32).reshape(-1, 3)
    if len(cands) > abi.MAX_CANDIDATES:
        raise ValueError(f"at most {abi.MAX_CANDIDATES} candidates are supported")
    arrays = dict(kinds=kinds, n_stages=n_stages, q_fail=q_fail, acc=acc,
                  t_prof=np.ascontiguousarray(t_prof), caps=caps)
    desc = abi.AlertSpaceDesc(
        n_dnns=len(dnns), n_powers=n_powers,
        dnn_kind=_ptr(kinds, C.c_int32), dnn_n_stages=_ptr(n_stages, C.c_int32),
        dnn_q_fail=_ptr(q_fail, C.c_double), stage_accuracy=_ptr(acc, C.c_double),
        stage_t_prof=_ptr(arrays["t_prof"], C.c_double), power_cap=_ptr(caps, C.c_double),
        p_idle_prof=float(space.p_idle_prof),
        sys_dnn=baseline_dnns(space)[0], app_dnn=baseline_dnns(space)[1],
    )
    return PackedSpace(desc, arrays, cands, space)


def baseline_dnns(space) -> tuple[int, int]:
    """DNN indices of the comparison schemes (-1 = none): sys-only runs
    fastest_dnn(space, last power, TRADITIONAL) (policies.py:292,
    model.py:166-176: minimal final-stage latency, ties to the lower id);
    app-only / no-coord run _pick_anytime (policies.py:324-329: most stages,
    ties to the higher id)."""
    dnns = list(space.dnns)
    last = len(space.powers) - 1
    trad = [k for k, d in enumerate(dnns) if kind_of(d) is DnnKind.TRADITIONAL]
    anyt = [k for k, d in enumerate(dnns) if kind_of(d) is DnnKind.ANYTIME]
    sys_dnn = min(trad, key=lambda k: (dnns[k].stages[-1].t_prof[last], dnns[k].id)) if trad else -1
    app_dnn = max(anyt, key=lambda k: (len(dnns[k].stages), dnns[k].id)) if anyt else -1
    return sys_dnn, app_dnn


def z_quantile(p: float) -> float:
    """normal_quantile (predictor.py:30-33): statistics.NormalDist.inv_cdf."""
    if not 0.0 < p < 1.0:
        raise ValueError("quantile probability must lie in (0, 1)")
    return NormalDist().inv_cdf(p)


def compact_specs(spec_arr: np.ndarray, stream_spec) -> tuple[np.ndarray, np.ndarray]:
    """Keep only the specs some stream uses (stream_spec re-indexed): a launch
    whose streams all minimise energy then gets the min-energy-only kernel
    even when the caller's spec list also holds max-accuracy goals."""
    ss = np.asarray(stream_spec, np.int64)
    used, inv = np.unique(ss, return_inverse=True)
    return np.ascontiguousarray(spec_arr[used]), inv.astype(np.int32).reshape(ss.shape)


def mode_runs(spec_arr: np.ndarray, stream_spec) -> list[tuple[int, int, np.ndarray, np.ndarray]]:
    """Split streams into maximal contiguous runs of one goal mode.  Each run
    gets its own compacted spec list and a full-length stream_spec re-indexed
    into it (entries outside the run are unused), so every launch sees a
    mode-homogeneous spec set (min-energy-only kernel where possible)."""
    ss = np.asarray(stream_spec, np.int64)
    modes = spec_arr["mode"][ss]
    cuts = np.flatnonzero(np.diff(modes)) + 1
    bounds = [0, *cuts.tolist(), len(ss)]
    runs = []
    for b, e in zip(bounds[:-1], bounds[1:]):
        used, inv = np.unique(ss[b:e], return_inverse=True)
        full = np.zeros(len(ss), np.int32)
        full[b:e] = inv.astype(np.int32)
        runs.append((b, e, np.ascontiguousarray(spec_arr[used]), full))
    return runs


def pack_specs(specs: Sequence, group_sizes: Sequence[int | None] | int | None = None) -> np.ndarray:
    """ConstraintSpec objects -> AlertSpec records (validated like
    ConstraintSpec.__post_init__, model.py:81-97)."""
    specs = list(specs)
    if isinstance(group_sizes, (int, type(None))):
        group_sizes = [group_sizes] * len(specs)
    out = np.zeros(len(specs), abi.SPEC_DTYPE)
    for k, (sp, g) in enumerate(zip(specs, group_sizes)):
        check_spec(sp)
        mode = mode_of(sp)
        out[k]["mode"] = abi.MODE_MAX_ACCURACY if mode is Mode.MAXIMIZE_ACCURACY else abi.MODE_MIN_ENERGY
        out[k]["has_pr"] = sp.pr_threshold is not None
        out[k]["group_size"] = int(g) if g else 0
        out[k]["t_goal"] = float(sp.t_goal)
        out[k]["e_goal"] = float(sp.e_goal) if sp.e_goal is not None else np.inf
        out[k]["q_goal"] = float(sp.q_goal) if sp.q_goal is not None else -np.inf
        out[k]["pr_threshold"] = float(sp.pr_threshold) if sp.pr_threshold is not None else 0.0
        out[k]["z_q"] = z_quantile(sp.pr_threshold) if sp.pr_threshold is not None else 0.0
        out[k]["overhead_budget"] = float(sp.overhead_budget)
        if g is not None and g and int(g) < 1:
            raise ValueError("group_size must be >= 1")
    return out


def spec_struct(rec) -> abi.AlertSpec:
    s = abi.AlertSpec()
    for name, _ in abi.AlertSpec._fields_:
        setattr(s, name, rec[name].item())
    return s


def filter_config(kalman: KalmanConfig | None = None,
                  idle: IdleFilterConfig | None = None) -> abi.AlertFilterConfig:
    k = kalman or KalmanConfig()
    i = idle or IdleFilterConfig()
    return abi.AlertFilterConfig(
        k0=k.k0, r=k.r, q0=k.q0, alpha=k.alpha, mu0=k.mu0, sigma2_0=k.sigma2_0,
        sigma2_uses_current_gain=int(bool(k.sigma2_uses_current_gain)), _pad=0,
        m0=i.m0, s=i.s, v=i.v,
    )


def policy_code(name: str) -> int:
    codes = {"alert": abi.POLICY_ALERT, "alert-any": abi.POLICY_ALERT_ANY,
             "alert-trad": abi.POLICY_ALERT_TRAD, "oracle": abi.POLICY_ORACLE,
             "alert+oracle": abi.POLICY_ALERT_WITH_ORACLE, "oracle-static": abi.POLICY_ORACLE_STATIC,
             "sys-only": abi.POLICY_SYS_ONLY, "app-only": abi.POLICY_APP_ONLY, "no-coord": abi.POLICY_NO_COORD}
    if name not in codes:
        raise ValueError(f"unknown policy {name!r}; choose from {tuple(codes)}")
    return codes[name]

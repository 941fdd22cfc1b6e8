"""ctypes mirror of include/alert_b200.h (plain structs and constants only)."""

from __future__ import annotations

import ctypes as C

import numpy as np

ALERT_ABI_VERSION = 4

KIND_TRADITIONAL, KIND_ANYTIME = 0, 1
MODE_MIN_ENERGY, MODE_MAX_ACCURACY = 0, 1
LEVEL_NONE, LEVEL_DROPPED_ENERGY, LEVEL_DROPPED_ACCURACY = 0, 1, 2
POLICY_ALERT, POLICY_ALERT_ANY, POLICY_ALERT_TRAD, POLICY_ORACLE, POLICY_ALERT_WITH_ORACLE = range(5)
# comparison schemes (policies.py:211-454)
POLICY_ORACLE_STATIC, POLICY_SYS_ONLY, POLICY_APP_ONLY, POLICY_NO_COORD = range(5, 9)
DTYPE_F32, DTYPE_F64 = 0, 1
FLAG_FP64_ALL = 0x1
FLAG_NO_REFINE = 0x2
FLAG_NO_FAST = 0x4  # disable the min-energy fast scan (A/B, tests)
FLAG_FAST_ROWS = 0x8  # fast scan in row mode (default for > 512 traditional cells)
FLAG_ANY_WINDOW = 0x10  # anytime cells by the two-pass window (A/B, tests)
FLAG_NO_ORACLE_FAST = 0x40  # oracle full scan only (A/B)
FLAG_FRESH = 0x20  # step range starts the runs: state initialised and aggregates zeroed in the launch
MAX_STAGES = 8
MAX_PHASES = 8
MAX_CANDIDATES = 6144

AGG_N, AGG_ENERGY, AGG_ENERGY_C, AGG_ACC, AGG_ACC_C = range(5)
AGG_VIOL_LAT, AGG_VIOL_ACC, AGG_VIOL_ENERGY = 5, 6, 7
AGG_LEVEL0, AGG_LEVEL1, AGG_LEVEL2, AGG_REFINED = 8, 9, 10, 11
AGG_OR_ENERGY, AGG_OR_ENERGY_C, AGG_OR_ACC, AGG_OR_ACC_C = 12, 13, 14, 15
AGG_OR_VIOL_LAT, AGG_OR_VIOL_ACC, AGG_OR_VIOL_ENERGY, AGG_OR_SAME = 16, 17, 18, 19
AGG_FULL_SCAN = 20  # min-energy steps the fast scan could not certify
AGG_PHASE_BASE, AGG_PHASE_STRIDE = 24, 8
AGG_FIELDS = 88


def neumaier_total(s, c):
    """Final value of a CPython 3.12 sum() given (sum, compensation)."""
    s = np.asarray(s, np.float64)
    c = np.asarray(c, np.float64)
    return np.where((c != 0) & np.isfinite(c), s + c, s)


STATUS_NAMES = {
    0: "ok",
    -1: "invalid argument",
    -2: "invalid config space",
    -3: "invalid constraint spec",
    -4: "invalid trace",
    -5: "CUDA error",
    -6: "unsupported size",
    -7: "no candidate of the requested kinds",
}

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)


class AlertSpaceDesc(C.Structure):
    _fields_ = [
        ("n_dnns", C.c_int32), ("n_powers", C.c_int32),
        ("dnn_kind", _ip), ("dnn_n_stages", _ip), ("dnn_q_fail", _dp),
        ("stage_accuracy", _dp), ("stage_t_prof", _dp), ("power_cap", _dp),
        ("p_idle_prof", C.c_double),
        ("sys_dnn", C.c_int32), ("app_dnn", C.c_int32),
    ]


class AlertFilterConfig(C.Structure):
    _fields_ = [
        ("k0", C.c_double), ("r", C.c_double), ("q0", C.c_double), ("alpha", C.c_double),
        ("mu0", C.c_double), ("sigma2_0", C.c_double),
        ("sigma2_uses_current_gain", C.c_int32), ("_pad", C.c_int32),
        ("m0", C.c_double), ("s", C.c_double), ("v", C.c_double),
    ]


class AlertSpec(C.Structure):
    _fields_ = [
        ("mode", C.c_int32), ("has_pr", C.c_int32), ("group_size", C.c_int32), ("_pad", C.c_int32),
        ("t_goal", C.c_double), ("e_goal", C.c_double), ("q_goal", C.c_double),
        ("pr_threshold", C.c_double), ("z_q", C.c_double), ("overhead_budget", C.c_double),
    ]


assert C.sizeof(AlertSpec) == 64

# numpy view of AlertSpec (for building spec arrays that go to the device)
SPEC_DTYPE = np.dtype(
    [("mode", "<i4"), ("has_pr", "<i4"), ("group_size", "<i4"), ("_pad", "<i4"),
     ("t_goal", "<f8"), ("e_goal", "<f8"), ("q_goal", "<f8"), ("pr_threshold", "<f8"),
     ("z_q", "<f8"), ("overhead_budget", "<f8")]
)
assert SPEC_DTYPE.itemsize == 64


class AlertTrace(C.Structure):
    _fields_ = [
        ("slowdown", C.c_void_p), ("slowdown_dtype", C.c_int32), ("n_rows", C.c_int32),
        ("n_steps", C.c_int64), ("row_stride", C.c_int64), ("step_stride", C.c_int64),
        ("step_offset", C.c_int64), ("max_segments", C.c_int32), ("_pad", C.c_int32),
        ("n_segments", C.c_void_p), ("seg_end", C.c_void_p), ("seg_phase", C.c_void_p),
        ("seg_idle", C.c_void_p), ("stream_row", C.c_void_p),
        # goal changes (ABI 3): per-row spec segments, NULL = none
        ("max_goal_segments", C.c_int32), ("_pad2", C.c_int32),
        ("n_goal_segments", C.c_void_p), ("goal_seg_end", C.c_void_p), ("goal_seg_spec", C.c_void_p),
    ]


class AlertState(C.Structure):
    _fields_ = [
        ("mu", C.c_void_p), ("sigma2", C.c_void_p), ("k_gain", C.c_void_p),
        ("q_noise", C.c_void_p), ("innov", C.c_void_p), ("phi", C.c_void_p),
        ("m_var", C.c_void_p), ("group_budget", C.c_void_p), ("group_count", C.c_void_p),
        ("policy_aux", C.c_void_p),
    ]


STATE_FIELDS = ("mu", "sigma2", "k_gain", "q_noise", "innov", "phi", "m_var", "group_budget")


class AlertOutputs(C.Structure):
    _fields_ = [
        ("decision", C.c_void_p), ("energy", C.c_void_p), ("accuracy", C.c_void_p),
        ("latency", C.c_void_p), ("mu", C.c_void_p), ("sigma2", C.c_void_p),
        ("oracle_decision", C.c_void_p), ("record_dtype", C.c_int32), ("_pad", C.c_int32),
        ("stream_stride", C.c_int64), ("step_stride", C.c_int64),
        ("agg", C.c_void_p), ("forced", C.c_void_p),
        ("fb_latency", C.c_void_p), ("fb_t_prof", C.c_void_p),
        ("plan_goal", C.c_void_p), ("phi", C.c_void_p),
    ]


class AlertPrediction(C.Structure):
    _fields_ = [
        ("latency_mean", C.c_double), ("latency_sigma", C.c_double), ("pr_deadline", C.c_double),
        ("expected_accuracy", C.c_double), ("energy", C.c_double),
        ("dnn_index", C.c_int32), ("power_index", C.c_int32), ("target_stage", C.c_int32),
        ("_pad", C.c_int32),
    ]


PREDICTION_DTYPE = np.dtype(
    [("latency_mean", "<f8"), ("latency_sigma", "<f8"), ("pr_deadline", "<f8"),
     ("expected_accuracy", "<f8"), ("energy", "<f8"), ("dnn_index", "<i4"),
     ("power_index", "<i4"), ("target_stage", "<i4"), ("_pad", "<i4")]
)
assert PREDICTION_DTYPE.itemsize == C.sizeof(AlertPrediction)


def decode_decision(word):
    """Split packed decision words (see AlertOutputs in the header)."""
    w = np.asarray(word, dtype=np.uint32)
    return {
        "cand": (w & 0xFFFF).astype(np.int32),
        "level": ((w >> 16) & 0x3).astype(np.int32),
        "met": ((w >> 18) & 1).astype(np.int32),
        "viol_lat": ((w >> 19) & 1).astype(np.int32),
        "viol_acc": ((w >> 20) & 1).astype(np.int32),
        "viol_energy": ((w >> 21) & 1).astype(np.int32),
        "completed": ((w >> 22) & 0xF).astype(np.int32),
        "refined": ((w >> 26) & 1).astype(np.int32),
        "phase": ((w >> 27) & 0x7).astype(np.int32),
        "feasible": ((w >> 30) & 1).astype(np.int32),
    }


DIST_CONSTANT, DIST_GAUSSIAN, DIST_LOGNORMAL, DIST_UNIFORM = range(4)


class AlertPhaseDesc(C.Structure):
    _fields_ = [("length", C.c_int64), ("dist", C.c_int32), ("_pad", C.c_int32), ("a", C.c_double),
                ("b", C.c_double), ("input_noise_sd", C.c_double)]

"""Loader for the in-tree CUDA library libalert_b200.so (the C ABI of
include/alert_b200.h).  There is no CPU fallback: if the library or a GPU is
missing, every entry point raises."""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from . import abi

# ALERT_LIB_PATH: an experimental build variant of the same sources (A/B runs)
LIB_PATH = Path(os.environ.get("ALERT_LIB_PATH") or Path(__file__).resolve().parent / "libalert_b200.so")

EXPORTS = (
    "alert_abi_version", "alert_strerror", "alert_last_error", "alert_create", "alert_destroy",
    "alert_table_create", "alert_table_destroy", "alert_table_num_candidates", "alert_table_candidate",
    "alert_state_init", "alert_run", "alert_decide", "alert_predict", "alert_observe",
    "alert_oracle_decide", "alert_reduce", "alert_set_launch", "alert_get_launch", "alert_launch_count",
    "alert_probe_fp32_peak", "alert_probe_phi32", "alert_xi_stats", "alert_realize", "alert_probe_erfc_rel",
    "alert_static_choice", "alert_baseline_decide",
)


class AlertError(RuntimeError):
    """A C-ABI call returned a negative AlertStatus."""

    def __init__(self, status: int, message: str):
        super().__init__(f"{abi.STATUS_NAMES.get(status, status)}: {message}")
        self.status = status


_lib = None


def load() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    L = C.CDLL(str(LIB_PATH))
    P, V = C.POINTER, C.c_void_p
    L.alert_abi_version.restype = C.c_int
    L.alert_strerror.argtypes = [C.c_int]
    L.alert_strerror.restype = C.c_char_p
    L.alert_last_error.restype = C.c_char_p
    L.alert_create.argtypes = [P(V), C.c_int]
    L.alert_destroy.argtypes = [V]
    L.alert_table_create.argtypes = [V, P(abi.AlertSpaceDesc), P(V)]
    L.alert_table_destroy.argtypes = [V]
    L.alert_table_num_candidates.argtypes = [V]
    L.alert_table_candidate.argtypes = [V, C.c_int, P(C.c_int32), P(C.c_int32), P(C.c_int32)]
    L.alert_state_init.argtypes = [V, V, P(abi.AlertFilterConfig), abi.AlertState, C.c_int64, V]
    L.alert_run.argtypes = [V, V, P(abi.AlertFilterConfig), V, C.c_int32, V, P(abi.AlertTrace), abi.AlertState,
                            P(abi.AlertOutputs), C.c_int32, C.c_uint32, C.c_int64, C.c_int64, C.c_int64,
                            C.c_int64, V]
    L.alert_decide.argtypes = [V, V, V, C.c_int32, V, abi.AlertState, V, C.c_int32, C.c_uint32, V, C.c_int64, V]
    L.alert_predict.argtypes = [V, V, V, C.c_int32, V, abi.AlertState, V, V, C.c_int64, V]
    L.alert_observe.argtypes = [V, V, P(abi.AlertFilterConfig), abi.AlertState, V, V, V, V, C.c_int64, V]
    L.alert_oracle_decide.argtypes = [V, V, V, C.c_int32, V, V, V, V, C.c_uint32, V, V, C.c_int64, V]
    L.alert_static_choice.argtypes = [V, V, V, C.c_int32, V, P(abi.AlertTrace), abi.AlertState, C.c_int64,
                                      C.c_int64, C.c_int64, C.c_int64, V]
    L.alert_baseline_decide.argtypes = [V, V, V, C.c_int32, V, abi.AlertState, V, C.c_int32, V, C.c_int64, V]
    L.alert_reduce.argtypes = [V, V, C.c_int64, V, V]
    L.alert_set_launch.argtypes = [V, C.c_int, C.c_int]
    L.alert_get_launch.argtypes = [V, P(C.c_int), P(C.c_int)]
    L.alert_launch_count.argtypes = [V]
    L.alert_launch_count.restype = C.c_int64
    L.alert_probe_fp32_peak.argtypes = [C.c_int, P(C.c_double)]
    L.alert_probe_phi32.argtypes = [V, V, C.c_int64, V]
    L.alert_probe_erfc_rel.argtypes = [V, V, C.c_int64, V]
    L.alert_xi_stats.argtypes = [V, V, V, C.c_int64, C.c_int32, V, V, V, V]
    L.alert_realize.argtypes = [V, V, C.c_int32, C.c_uint64, C.c_int64, C.c_int64, V, C.c_int32, V]
    if L.alert_abi_version() != abi.ALERT_ABI_VERSION:
        raise ImportError("libalert_b200.so ABI version mismatch; rebuild")
    _lib = L
    return L


def check(status: int) -> None:
    if status != 0:
        msg = load().alert_last_error().decode(errors="replace")
        if status == -3 or status == -2:
            raise ValueError(msg)
        raise AlertError(status, msg)

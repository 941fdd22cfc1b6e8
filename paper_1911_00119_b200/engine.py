"""Device-side engine: a thin Python layer over the C ABI.

torch is used only for device memory and streams (buffers are torch tensors,
passed to the library as raw pointers); every computation happens in the
CUDA kernels of libalert_b200.so.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import abi
from ._lib import check, load
from .packing import PackedSpace, filter_config, pack_space

STATE_DTYPES = {"mu": "f8", "sigma2": "f8", "k_gain": "f8", "q_noise": "f8", "innov": "f8", "phi": "f8",
                "m_var": "f8", "group_budget": "f8", "group_count": "i4", "policy_aux": "i4"}


def _torch():
    import torch

    return torch


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


@dataclass
class DeviceTrace:
    """An AlertTrace whose arrays live in device memory (time-major slowdown)."""

    slowdown: object
    n_segments: object
    seg_end: object
    seg_phase: object
    seg_idle: object
    stream_row: object = None
    step_offset: int = 0
    total_steps: int | None = None  # steps of the whole trace when this buffer is a chunk
    goal_n: object = None     # goal changes (AlertTrace.goal_*), None = none
    goal_end: object = None
    goal_spec: object = None

    @property
    def n_rows(self) -> int:
        return int(self.slowdown.shape[1])

    @property
    def n_steps(self) -> int:
        return int(self.slowdown.shape[0])

    def struct(self) -> abi.AlertTrace:
        torch = _torch()
        return abi.AlertTrace(
            slowdown=self.slowdown.data_ptr(),
            slowdown_dtype=abi.DTYPE_F64 if self.slowdown.dtype == torch.float64 else abi.DTYPE_F32,
            n_rows=self.n_rows, n_steps=self.n_steps,
            row_stride=self.slowdown.stride(1), step_stride=self.slowdown.stride(0),
            step_offset=self.step_offset, max_segments=int(self.seg_end.shape[1]), _pad=0,
            n_segments=self.n_segments.data_ptr(), seg_end=self.seg_end.data_ptr(),
            seg_phase=self.seg_phase.data_ptr(), seg_idle=self.seg_idle.data_ptr(),
            stream_row=_ptr(self.stream_row),
            max_goal_segments=0 if self.goal_end is None else int(self.goal_end.shape[1]), _pad2=0,
            n_goal_segments=_ptr(self.goal_n), goal_seg_end=_ptr(self.goal_end), goal_seg_spec=_ptr(self.goal_spec),
        )

    def with_goal_changes(self, goal_n, goal_end, goal_spec) -> "DeviceTrace":
        """This trace with per-row goal changes (host arrays from
        trace.pack_goal_changes) uploaded next to it."""
        torch = _torch()
        d = self.slowdown.device
        from dataclasses import replace

        return replace(self, goal_n=torch.from_numpy(np.ascontiguousarray(goal_n, np.int32)).to(d),
                       goal_end=torch.from_numpy(np.ascontiguousarray(goal_end, np.int32)).to(d),
                       goal_spec=torch.from_numpy(np.ascontiguousarray(goal_spec, np.int32)).to(d))


class GpuTable:
    """A candidate table resident on one device (alert_table_create)."""

    def __init__(self, engine: "Engine", space):
        self.engine = engine
        self.packed: PackedSpace = space if isinstance(space, PackedSpace) else pack_space(space)
        h = C.c_void_p()
        check(load().alert_table_create(engine.ctx, C.byref(self.packed.desc), C.byref(h)))
        self.handle = h
        self.n_candidates = load().alert_table_num_candidates(h)
        self.candidates = self.packed.candidates

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                load().alert_table_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


class Engine:
    """One AlertContext on one CUDA device."""

    def __init__(self, device: int = 0):
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1911_00119_b200 needs a CUDA device (no CPU fallback)")
        self.device = device
        self.tdev = torch.device("cuda", device)
        h = C.c_void_p()
        check(load().alert_create(C.byref(h), device))
        self.ctx = h
        self._tables = {}
        self._launch_args = (0, 0)  # alert_set_launch arguments in effect (0 = library default)

    def __del__(self):
        try:
            if getattr(self, "ctx", None):
                load().alert_destroy(self.ctx)
                self.ctx = None
        except Exception:
            pass

    # -- configuration --------------------------------------------------------
    def set_launch(self, lanes_per_stream: int = 0, threads_per_block: int = 0) -> tuple[int, int]:
        """Set the launch geometry; returns the previous arguments (for restore_launch)."""
        check(load().alert_set_launch(self.ctx, lanes_per_stream, threads_per_block))
        prev, self._launch_args = self._launch_args, (lanes_per_stream, threads_per_block)
        return prev

    def restore_launch(self, args: tuple[int, int]) -> None:
        self.set_launch(*args)

    def launch_config(self) -> tuple[int, int]:
        a, b = C.c_int(), C.c_int()
        check(load().alert_get_launch(self.ctx, C.byref(a), C.byref(b)))
        return a.value, b.value

    def launch_count(self) -> int:
        return int(load().alert_launch_count(self.ctx))

    def table(self, space) -> GpuTable:
        key = id(space)
        t = self._tables.get(key)
        if t is None or t.packed.space is not space:
            t = GpuTable(self, space)
            self._tables[key] = t
        return t

    def _stream(self, stream=None):
        torch = _torch()
        s = stream if stream is not None else torch.cuda.current_stream(self.tdev)
        return C.c_void_p(s.cuda_stream)

    # -- buffers ----------------------------------------------------------------
    def upload_trace(self, packed, stream_row=None) -> DeviceTrace:
        torch = _torch()
        d = self.tdev
        tr = DeviceTrace(
            slowdown=torch.from_numpy(np.ascontiguousarray(packed.slowdown)).to(d),
            n_segments=torch.from_numpy(packed.n_segments).to(d),
            seg_end=torch.from_numpy(packed.seg_end).to(d),
            seg_phase=torch.from_numpy(packed.seg_phase).to(d),
            seg_idle=torch.from_numpy(packed.seg_idle).to(d),
            stream_row=None if stream_row is None else torch.as_tensor(np.asarray(stream_row, np.int32)).to(d),
        )
        if getattr(packed, "goal_n", None) is not None:
            tr = tr.with_goal_changes(packed.goal_n, packed.goal_end, packed.goal_spec)
        return tr

    def new_state(self, table: GpuTable, n: int, kalman=None, idle_cfg=None, stream=None, init: bool = True) -> dict:
        """Filter state of n streams (alert_state_init).  init=False only
        allocates: for a first alert_run with FLAG_FRESH, which initialises it."""
        torch = _torch()
        st = {k: torch.empty(n, dtype=torch.float64 if v == "f8" else torch.int32, device=self.tdev)
              for k, v in STATE_DTYPES.items()}
        if not init:
            return st
        cfg = filter_config(kalman, idle_cfg)
        check(load().alert_state_init(self.ctx, table.handle, C.byref(cfg), state_struct(st), n,
                                      self._stream(stream)))
        return st

    # -- entry points -------------------------------------------------------------
    def run(self, table: GpuTable, specs: np.ndarray, trace: DeviceTrace, state: dict, *, policy: int,
            kalman=None, idle_cfg=None, stream_spec=None, outputs: abi.AlertOutputs | None = None,
            flags: int = 0, stream_begin: int = 0, stream_end: int | None = None, step_begin: int = 0,
            step_end: int | None = None, stream=None) -> None:
        specs = np.ascontiguousarray(specs, dtype=abi.SPEC_DTYPE)
        cfg = filter_config(kalman, idle_cfg)
        tr = trace.struct()
        out = outputs if outputs is not None else abi.AlertOutputs()
        se = int(state["mu"].shape[0]) if stream_end is None else stream_end
        te = trace.n_steps if step_end is None else step_end
        check(load().alert_run(self.ctx, table.handle, C.byref(cfg), specs.ctypes.data, len(specs),
                               _ptr(stream_spec), C.byref(tr), state_struct(state), C.byref(out), policy,
                               flags, stream_begin, se, step_begin, te, self._stream(stream)))

    def decide(self, table, specs, state, plan_goal, *, policy=abi.POLICY_ALERT, flags=0, stream_spec=None,
               stream=None):
        torch = _torch()
        specs = np.ascontiguousarray(specs, dtype=abi.SPEC_DTYPE)
        n = int(plan_goal.shape[0])
        out = torch.empty(n, dtype=torch.int32, device=self.tdev)
        check(load().alert_decide(self.ctx, table.handle, specs.ctypes.data, len(specs), _ptr(stream_spec),
                                  state_struct(state), plan_goal.data_ptr(), policy, flags, out.data_ptr(), n,
                                  self._stream(stream)))
        return out

    def predict(self, table, specs, state, plan_goal, *, stream_spec=None, stream=None):
        torch = _torch()
        specs = np.ascontiguousarray(specs, dtype=abi.SPEC_DTYPE)
        n = int(plan_goal.shape[0])
        out = torch.empty((n, table.n_candidates, abi.PREDICTION_DTYPE.itemsize), dtype=torch.uint8,
                          device=self.tdev)
        check(load().alert_predict(self.ctx, table.handle, specs.ctypes.data, len(specs), _ptr(stream_spec),
                                   state_struct(state), plan_goal.data_ptr(), out.data_ptr(), n,
                                   self._stream(stream)))
        return out

    def observe(self, table, state, fb_latency, fb_t_prof, idle, power_index, *, kalman=None, idle_cfg=None,
                stream=None):
        cfg = filter_config(kalman, idle_cfg)
        n = int(fb_latency.shape[0])
        check(load().alert_observe(self.ctx, table.handle, C.byref(cfg), state_struct(state),
                                   fb_latency.data_ptr(), fb_t_prof.data_ptr(), idle.data_ptr(),
                                   power_index.data_ptr(), n, self._stream(stream)))

    def oracle_decide(self, table, specs, s, idle, plan_goal, *, stream_spec=None, stream=None, exact=False):
        """Oracle decisions; with exact=True also the chosen configs' exact
        predictions ([n, bytes] uint8 viewable as abi.PREDICTION_DTYPE)."""
        torch = _torch()
        specs = np.ascontiguousarray(specs, dtype=abi.SPEC_DTYPE)
        n = int(s.shape[0])
        out = torch.empty(n, dtype=torch.int32, device=self.tdev)
        ex = torch.empty((n, abi.PREDICTION_DTYPE.itemsize), dtype=torch.uint8, device=self.tdev) if exact else None
        check(load().alert_oracle_decide(self.ctx, table.handle, specs.ctypes.data, len(specs),
                                         _ptr(stream_spec), s.data_ptr(), idle.data_ptr(), plan_goal.data_ptr(),
                                         0, out.data_ptr(), _ptr(ex), n, self._stream(stream)))
        return (out, ex) if exact else out

    def static_choice(self, table, specs, trace: DeviceTrace, state, *, stream_spec=None, stream_begin=0,
                      stream_end=None, step_begin=0, step_end=None, stream=None):
        """OracleStaticPolicy.begin for a range of streams (policy_aux <- cand | eligible << 16)."""
        specs = np.ascontiguousarray(specs, dtype=abi.SPEC_DTYPE)
        tr = trace.struct()
        se = int(state["mu"].shape[0]) if stream_end is None else stream_end
        te = trace.n_steps if step_end is None else step_end
        check(load().alert_static_choice(self.ctx, table.handle, specs.ctypes.data, len(specs), _ptr(stream_spec),
                                         C.byref(tr), state_struct(state), stream_begin, se, step_begin, te,
                                         self._stream(stream)))

    def baseline_decide(self, table, specs, state, plan_goal, *, policy, stream_spec=None, stream=None):
        """One decide of a comparison scheme per stream (packed words, bits 0..17 and 30)."""
        torch = _torch()
        specs = np.ascontiguousarray(specs, dtype=abi.SPEC_DTYPE)
        n = int(plan_goal.shape[0])
        out = torch.empty(n, dtype=torch.int32, device=self.tdev)
        check(load().alert_baseline_decide(self.ctx, table.handle, specs.ctypes.data, len(specs),
                                           _ptr(stream_spec), state_struct(state), plan_goal.data_ptr(), policy,
                                           out.data_ptr(), n, self._stream(stream)))
        return out

    def reduce(self, agg, stream=None):
        torch = _torch()
        out = torch.empty(abi.AGG_FIELDS, dtype=torch.float64, device=self.tdev)
        check(load().alert_reduce(self.ctx, agg.data_ptr(), int(agg.shape[0]), out.data_ptr(),
                                  self._stream(stream)))
        return out


def state_struct(st: dict) -> abi.AlertState:
    return abi.AlertState(**{k: st[k].data_ptr() for k in STATE_DTYPES})


def outputs_struct(records: dict | None = None, agg=None, forced=None, oracle_decision=None,
                   n_streams: int = 0) -> abi.AlertOutputs:
    """AlertOutputs over time-major [n_steps, n_streams] record tensors."""
    torch = _torch()
    out = abi.AlertOutputs()
    ref = None
    if records:
        for k in ("decision", "energy", "accuracy", "latency", "mu", "sigma2"):
            if records.get(k) is not None:
                setattr(out, k, records[k].data_ptr())
                ref = records[k]
        vals = [records.get(k) for k in ("energy", "accuracy", "latency", "mu", "sigma2") if records.get(k) is not None]
        if vals:
            dts = {v.dtype for v in vals}
            if len(dts) != 1:
                raise ValueError("record value arrays must share one dtype")
            out.record_dtype = abi.DTYPE_F64 if vals[0].dtype == torch.float64 else abi.DTYPE_F32
    for t in (forced, oracle_decision):
        if t is not None:
            ref = t
    if oracle_decision is not None:
        out.oracle_decision = oracle_decision.data_ptr()
    if forced is not None:
        out.forced = forced.data_ptr()
    if ref is not None:
        out.step_stride = ref.stride(0)
        out.stream_stride = ref.stride(1)
    if agg is not None:
        out.agg = agg.data_ptr()
    if records and records.get("fb_latency") is not None:
        out.fb_latency = records["fb_latency"].data_ptr()
        out.fb_t_prof = records["fb_t_prof"].data_ptr()
        for k in ("plan_goal", "phi"):
            if records.get(k) is not None:
                setattr(out, k, records[k].data_ptr())
    return out

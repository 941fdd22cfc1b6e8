"""Closed-loop runs on the GPU: the drop-in ``run`` and the batched
``run_batch``.

``run(space, spec, trace, policy)`` has the reference's signature and result
(simulator.py:461-507) for the policies of :mod:`.policies`, but executes the
whole trace in ONE launch of the fused kernel (alert_run) instead of a
Python loop.  ``run_batch`` is the scale-out entry point: many streams
(scenarios) x many steps per launch, optionally chunked over steps with the
filter state carried on the device.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import abi
from .engine import DeviceTrace, Engine, GpuTable, outputs_struct
from .packing import mode_runs, pack_specs, policy_code
from .records import (
    RunResult, StepRecord, Summary, ViolationFlags, decision_of, prediction_of, summary_from_agg,
)
from .trace import PackedEnvs, TrueEnvironment, pack_envs, pack_goal_changes, realize

_ENGINES: dict[int, Engine] = {}


def get_engine(device: int = 0) -> Engine:
    e = _ENGINES.get(device)
    if e is None:
        e = _ENGINES[device] = Engine(device)
    return e


@dataclass
class BatchResult:
    """Outputs of run_batch (host numpy arrays unless keep_on_device)."""

    agg: object                  # [n_streams, AGG_FIELDS] float64
    state: dict                  # final filter state per stream
    records: dict = field(default_factory=dict)  # [n_steps, n_streams] per field
    oracle_decision: object = None
    candidates: np.ndarray | None = None
    n_phases: int = abi.MAX_PHASES

    def summaries(self) -> list[Summary]:
        agg = np.asarray(self.agg)
        return [summary_from_agg(agg[k], self.n_phases) for k in range(agg.shape[0])]

    def decoded(self) -> dict:
        return abi.decode_decision(np.asarray(self.records["decision"]).view(np.uint32))


def _as_device_trace(engine: Engine, envs, trace_dtype, stream_row) -> DeviceTrace:
    if isinstance(envs, DeviceTrace):
        return envs
    if not isinstance(envs, PackedEnvs):
        envs = pack_envs(list(envs), dtype=trace_dtype)
    return engine.upload_trace(envs, stream_row)


def run_batch(space, specs: Sequence, envs, policy: str = "alert", *, kalman=None, idle_cfg=None,
              group_sizes=None, stream_spec=None, stream_row=None, n_streams: int | None = None,
              records: str | None = None, forced=None, flags: int = 0, chunk_steps: int | None = None,
              trace_dtype=np.float64, engine: Engine | None = None, device: int = 0,
              keep_on_device: bool = False, lanes_per_stream: int | None = None,
              goal_changes=None) -> BatchResult:
    """Run ``policy`` over many independent streams in one fused launch.

    specs        ConstraintSpec objects (or an AlertSpec record array); stream k
                 uses specs[stream_spec[k]] (default k % len(specs)).
    envs         realized environments (TrueEnvironment-like), a PackedEnvs or
                 a DeviceTrace; stream k reads row stream_row[k] (default k).
    records      None (aggregates only), "f32" or "f64" per-step records.
    forced       [n_steps, n_streams] int32 candidate indices to execute
                 (teacher forcing; -1 = own decision).
    trace_dtype  slow-down dtype when ``envs`` are packed here: float64 keeps
                 the reference's values (default); float32 halves the trace
                 bytes (the decisions then follow the FP32-rounded inputs).
    goal_changes per trace row None or [(start_step, spec_index), ...] from
                 step 0 (trace.pack_goal_changes): the row's constraint spec
                 changes at those inputs (overrides stream_spec).
    lanes_per_stream  tile width for this call only (the engine's launch
                 settings are restored afterwards).
    """
    torch = __import__("torch")
    eng = engine or get_engine(device)
    prev_launch = None
    if lanes_per_stream is not None:
        prev_launch = eng.set_launch(lanes_per_stream, 0)
    try:
        return _run_batch(eng, torch, space, specs, envs, policy, kalman, idle_cfg, group_sizes, stream_spec,
                          stream_row, n_streams, records, forced, flags, chunk_steps, trace_dtype,
                          keep_on_device, goal_changes)
    finally:
        if prev_launch is not None:
            eng.restore_launch(prev_launch)


def _run_batch(eng, torch, space, specs, envs, policy, kalman, idle_cfg, group_sizes, stream_spec, stream_row,
               n_streams, records, forced, flags, chunk_steps, trace_dtype, keep_on_device, goal_changes):
    table: GpuTable = eng.table(space)
    spec_arr = specs if isinstance(specs, np.ndarray) and specs.dtype == abi.SPEC_DTYPE \
        else pack_specs(list(specs), group_sizes)
    trace = _as_device_trace(eng, envs, trace_dtype, stream_row)
    if goal_changes is not None:
        if isinstance(goal_changes, tuple) and len(goal_changes) == 3 and isinstance(goal_changes[0], np.ndarray):
            gn, ge, gs = goal_changes
        else:
            gn, ge, gs = pack_goal_changes(goal_changes, trace.n_steps, len(spec_arr))
        if len(gn) != trace.n_rows:
            raise ValueError(f"goal_changes has {len(gn)} rows, the trace {trace.n_rows}")
        trace = trace.with_goal_changes(gn, ge, gs)
        stream_spec_mode_split = False
    else:
        stream_spec_mode_split = trace.goal_n is None
    if stream_row is not None and trace.stream_row is None:
        trace.stream_row = torch.as_tensor(np.asarray(stream_row, np.int32)).to(eng.tdev)
    ns = n_streams if n_streams is not None else (
        len(stream_row) if stream_row is not None else trace.n_rows)
    steps = trace.n_steps
    dev = eng.tdev
    # launches: one per contiguous run of streams with one goal mode (a
    # trace with goal changes runs as one launch over every spec)
    if stream_spec is not None and not stream_spec_mode_split:
        launches = [(0, None, spec_arr, torch.as_tensor(np.asarray(stream_spec, np.int32)).to(dev))]
    elif stream_spec is not None:
        launches = [(b, e, sp, torch.as_tensor(full).to(dev)) for b, e, sp, full in mode_runs(spec_arr, stream_spec)]
    else:
        launches = [(0, None, spec_arr, None)]
    # the first step range initialises the state and zeroes the aggregates in
    # the launch itself (FLAG_FRESH): no alert_state_init, no memset
    state = eng.new_state(table, ns, kalman, idle_cfg, init=False)
    agg = torch.empty((ns, abi.AGG_FIELDS), dtype=torch.float64, device=dev)
    rec = {}
    if records:
        vdt = torch.float64 if records == "f64" else torch.float32
        rec["decision"] = torch.empty((steps, ns), dtype=torch.int32, device=dev)
        for k in ("energy", "accuracy", "latency", "mu", "sigma2"):
            rec[k] = torch.empty((steps, ns), dtype=vdt, device=dev)
        if records == "f64":  # StepRecord feedback pair (fb_latency, fb_t_prof), plan goal, phi
            for k in ("fb_latency", "fb_t_prof", "plan_goal", "phi"):
                rec[k] = torch.empty((steps, ns), dtype=torch.float64, device=dev)
    pol = policy_code(policy)
    od = None
    if pol == abi.POLICY_ALERT_WITH_ORACLE and records:
        od = torch.empty((steps, ns), dtype=torch.int32, device=dev)
    fz = None
    if forced is not None:
        fz = torch.as_tensor(np.asarray(forced, np.int32)).to(dev)
        if tuple(fz.shape) != (steps, ns):
            raise ValueError("forced must be [n_steps, n_streams]")
    out = outputs_struct(rec, agg=agg, forced=fz, oracle_decision=od)
    if out.step_stride == 0:
        out.step_stride, out.stream_stride = ns, 1
    chunk = chunk_steps or steps
    if pol == abi.POLICY_ORACLE_STATIC:
        chunk = steps  # begin() is clairvoyant over the whole trace (policies.py:221-265)
    for s0 in range(0, steps, chunk):
        for b, e, sp, ss in launches:
            eng.run(table, sp, trace, state, policy=pol, kalman=kalman, idle_cfg=idle_cfg, stream_spec=ss,
                    outputs=out, flags=flags | (abi.FLAG_FRESH if s0 == 0 else 0), stream_begin=b,
                    stream_end=ns if e is None else e, step_begin=s0, step_end=min(steps, s0 + chunk))
    if keep_on_device:
        return BatchResult(agg, state, rec, od, table.candidates)
    torch.cuda.synchronize(dev)
    return BatchResult(
        agg.cpu().numpy(), {k: v.cpu().numpy() for k, v in state.items()},
        {k: v.cpu().numpy() for k, v in rec.items()}, None if od is None else od.cpu().numpy(),
        table.candidates,
    )


def chunk_sizes(n_steps: int, chunk: int, tail: bool = True, growth: float = 1.4) -> list[int]:
    """Step-chunk lengths for HostStreamer.  The head ramps up geometrically
    from chunk / 8 (each copy short enough to finish while the previous
    chunk computes, so the kernel never waits after the first, short copy),
    then full chunks.  With ``tail`` the last chunk is short too (copy-bound
    runs: little kernel time after the last copy); without it the last chunk
    stays long enough to hide the aggregate D2H behind its stream-range
    launches."""
    if n_steps <= 0:
        raise ValueError("n_steps must be positive")
    chunk = max(1, min(chunk, n_steps))
    edge = max(1, chunk // 8)
    if n_steps <= chunk:
        return [n_steps]
    sizes, rem, z = [], n_steps, edge
    while z < chunk and rem > z + (edge if tail else 0):
        sizes.append(z)
        rem -= z
        z = min(chunk, max(z + 1, int(z * growth)))
    if not tail:  # a partial chunk right after the ramp, full chunks to the end
        if rem % chunk:
            sizes.append(rem % chunk)
        return sizes + [chunk] * (rem // chunk)
    while rem > chunk + edge:
        sizes.append(chunk)
        rem -= chunk
    sizes += [rem - edge, edge] if rem > edge else [rem]
    return sizes


class HostStreamer:
    """run_batch for traces that live in (pinned) HOST memory.

    The time-major slow-down array is cut into step chunks copied
    host->device on a copy stream into a ring of ``n_buffers`` device
    buffers while the kernel runs earlier chunks on the compute stream (CUDA
    events order them); the filter state and aggregates stay on the device
    between chunks (alert_run step ranges).  The scenario map (stream_spec,
    and stream_row when scenarios share trace rows) is copied from pinned
    host memory at the start of every pass.  This is the end-to-end path:
    inputs from host, per-stream summaries back.

    Pipeline edges: the first chunks ramp up from chunk / 8 so
    the first copy is short; with one D2H part the last chunk is short too
    (little kernel time after the last copy); with many streams
    (``d2h_parts`` > 1, default one part per 131,072 streams, at most 8) the
    last chunk runs as stream-range launches and each range's aggregate rows
    go device->host on a second copy stream while the next range computes.
    Back-to-back passes overlap: a pass's first copies wait only for the
    previous pass's last use of each trace buffer.  The returned tensor is
    ready once the caller's current stream has synchronised (it waits on the
    D2H stream); a later pass rewrites it.
    """

    def __init__(self, space, specs, packed: PackedEnvs, policy: str = "alert", *, kalman=None,
                 idle_cfg=None, group_sizes=None, stream_spec=None, stream_row=None, chunk_steps: int = 1000,
                 engine: Engine | None = None, device: int = 0, d2h_parts: int | None = None,
                 schedule: Sequence[int] | None = None, n_buffers: int = 3):
        torch = __import__("torch")
        self.torch = torch
        self.eng = eng = engine or get_engine(device)
        self.table = eng.table(space)
        self.specs = specs if isinstance(specs, np.ndarray) and specs.dtype == abi.SPEC_DTYPE \
            else pack_specs(list(specs), group_sizes)
        self.policy = policy_code(policy)
        if self.policy == abi.POLICY_ORACLE_STATIC:
            raise ValueError("oracle-static is clairvoyant over the whole trace: use run_batch (device-resident "
                             "trace), not the chunked host streamer")
        self.kalman, self.idle_cfg = kalman, idle_cfg
        self.n_steps, n_rows = packed.slowdown.shape
        self.n_streams = n_rows if stream_row is None else len(stream_row)
        self.chunk = min(chunk_steps, self.n_steps)
        self.d2h_parts = max(1, min(8, self.n_streams // 131072)) if d2h_parts is None else int(d2h_parts)
        if not 1 <= self.d2h_parts <= self.n_streams:
            raise ValueError(f"d2h_parts must be in 1..{self.n_streams}")
        self.sizes = chunk_sizes(self.n_steps, self.chunk, tail=self.d2h_parts == 1) if schedule is None \
            else [int(z) for z in schedule]
        if sum(self.sizes) != self.n_steps or min(self.sizes) < 1 or max(self.sizes) > self.chunk:
            raise ValueError(f"schedule must split {self.n_steps} steps into chunks of 1..{self.chunk}")
        d = eng.tdev
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
        # pinned host copies of the inputs (outside any timed region)
        self.host = pin(packed.slowdown)
        self.seg = [torch.from_numpy(a).to(d) for a in (packed.n_segments, packed.seg_end, packed.seg_phase,
                                                        packed.seg_idle)]
        self.goals = None
        if getattr(packed, "goal_n", None) is not None:
            self.goals = [torch.from_numpy(np.ascontiguousarray(a, np.int32)).to(d)
                          for a in (packed.goal_n, packed.goal_end, packed.goal_spec)]
        ss = (np.arange(self.n_streams) % len(self.specs)).astype(np.int32) if stream_spec is None \
            else np.asarray(stream_spec, np.int32)
        # launches: contiguous runs of one goal mode (rows with goal changes: one launch)
        if self.goals is None:
            runs = mode_runs(self.specs, ss)
        else:
            runs = [(0, self.n_streams, self.specs, ss)]
        self.runs = [(b, e, sp) for b, e, sp, _ in runs]
        self.map_host = [pin(np.stack([full for _, _, _, full in runs]))]
        self.map_dev = [torch.empty_like(self.map_host[0], device=d)]
        if stream_row is not None:
            self.map_host.append(pin(np.asarray(stream_row, np.int32)))
            self.map_dev.append(torch.empty_like(self.map_host[1], device=d))
        if n_buffers < 2:
            raise ValueError("n_buffers must be >= 2")
        self.bufs = [torch.empty((self.chunk, n_rows), dtype=self.host.dtype, device=d) for _ in range(n_buffers)]
        self.copy_stream = torch.cuda.Stream(d)
        # last use of each trace buffer by the previous pass: the next pass's first copies wait only for
        # these, so they run under the previous pass's last chunks (back-to-back passes keep PCIe busy)
        self._released = [None] * n_buffers
        self._comp = None  # the compute stream of the last pass
        self.d2h_stream = torch.cuda.Stream(d)  # aggregate rows back, beside the H2D copies
        self.agg_host = torch.empty((self.n_streams, abi.AGG_FIELDS), dtype=torch.float64).pin_memory()

    @property
    def h2d_bytes(self) -> int:
        return self.host.numel() * self.host.element_size() + sum(m.numel() * m.element_size()
                                                                   for m in self.map_host)

    @property
    def d2h_bytes(self) -> int:
        return self.agg_host.numel() * self.agg_host.element_size()

    def run(self):
        """One end-to-end pass; returns the pinned host aggregate tensor."""
        torch, eng = self.torch, self.eng
        comp = torch.cuda.current_stream(eng.tdev)
        if self._released[0] is None:  # first pass: copies ordered after the caller's prior work
            self.copy_stream.wait_stream(comp)
        elif self._comp is not None and self._comp != comp:  # the map / state of the last pass are in use there
            comp.wait_stream(self._comp)
        self._comp = comp
        for h, dv in zip(self.map_host, self.map_dev):
            dv.copy_(h, non_blocking=True)
        state = eng.new_state(self.table, self.n_streams, self.kalman, self.idle_cfg, init=False)
        agg = torch.empty((self.n_streams, abi.AGG_FIELDS), dtype=torch.float64, device=eng.tdev)
        out = outputs_struct(None, agg=agg)
        stream_row = self.map_dev[1] if len(self.map_dev) > 1 else None
        nb = len(self.bufs)
        copied = [torch.cuda.Event() for _ in range(nb)]
        consumed = [torch.cuda.Event() for _ in range(nb)]
        starts = np.concatenate([[0], np.cumsum(self.sizes)]).tolist()
        n_chunks = len(self.sizes)

        def issue_copy(i):
            b = i % nb
            s0, s1 = starts[i], starts[i + 1]
            with torch.cuda.stream(self.copy_stream):
                if i >= nb:
                    self.copy_stream.wait_event(consumed[b])
                elif self._released[b] is not None:
                    self.copy_stream.wait_event(self._released[b])
                self.bufs[b][: s1 - s0].copy_(self.host[s0:s1], non_blocking=True)
                copied[b].record(self.copy_stream)

        def launch(tr, s0, s1, b0, b1):  # the goal-mode runs intersected with streams [b0, b1)
            for k, (lb, le, sp) in enumerate(self.runs):
                lo, hi = max(lb, b0), min(le, b1)
                if lo < hi:
                    eng.run(self.table, sp, tr, state, policy=self.policy, kalman=self.kalman,
                            idle_cfg=self.idle_cfg, stream_spec=self.map_dev[0][k], outputs=out, stream_begin=lo,
                            stream_end=hi, step_begin=s0, step_end=s1, flags=abi.FLAG_FRESH if s0 == 0 else 0)

        for i in range(min(nb - 1, n_chunks)):
            issue_copy(i)
        for i in range(n_chunks):
            s0, s1 = starts[i], starts[i + 1]
            if i + nb - 1 < n_chunks:
                issue_copy(i + nb - 1)
            b = i % nb
            comp.wait_event(copied[b])
            tr = DeviceTrace(self.bufs[b][: s1 - s0], *self.seg, stream_row=stream_row, step_offset=s0)
            if self.goals is not None:
                tr.goal_n, tr.goal_end, tr.goal_spec = self.goals
            if i + 1 < n_chunks:
                launch(tr, s0, s1, 0, self.n_streams)
            else:  # last chunk: stream ranges, each range's final aggregates D2H behind the next range
                cuts = [self.n_streams * p // self.d2h_parts for p in range(self.d2h_parts + 1)]
                for p in range(self.d2h_parts):
                    launch(tr, s0, s1, cuts[p], cuts[p + 1])
                    done = torch.cuda.Event()
                    done.record(comp)
                    with torch.cuda.stream(self.d2h_stream):
                        self.d2h_stream.wait_event(done)
                        self.agg_host[cuts[p]:cuts[p + 1]].copy_(agg[cuts[p]:cuts[p + 1]], non_blocking=True)
            consumed[b].record(comp)
        self._released = consumed
        comp.wait_stream(self.d2h_stream)  # the caller's stream covers the D2H
        return self.agg_host


def run(space, spec, trace, policy, goal_changes=None) -> RunResult:
    """Drop-in for simulator.run (simulator.py:461-507) with a policy from
    :func:`make_policy`: realize the trace (same numpy draws as the
    reference), then one fused GPU launch over all inputs.  Records carry the
    reference's fields in FP64: ``period`` = plan goal + overhead
    (simulator.py:483), ``decision.feasible`` and ``decision.prediction`` as
    the reference's policies set them (selector.py:122-128, policies.py:201-205,
    266-271, 305-320, 357-368, 417-428), the latter from one batched
    ``alert_predict`` launch over the per-step filter states.

    goal_changes  optional [(input_index, ConstraintSpec), ...]: from that
                  input on the run is measured against, and the policy plans
                  for, the new spec (the reference's ``policy.spec`` swapped
                  between inputs; SURVEY §7 hard part 8).
    """
    from .policies import GpuPolicy

    if not isinstance(policy, GpuPolicy):
        raise TypeError("run() executes the policies of paper_1911_00119_b200.make_policy on the GPU; "
                        f"got {type(policy).__name__}")
    env = realize(trace)
    specs = [spec] + [c for _, c in (goal_changes or ())]
    sched = None
    if goal_changes:
        sched = [[(0, 0)] + [(int(n), k + 1) for k, (n, _) in enumerate(goal_changes)]]
    policy.begin(space, spec, env)
    spec_arr = pack_specs(specs, trace.group_size)
    res = run_batch(space, spec_arr, [env], policy.code_name, kalman=policy.kalman,
                    idle_cfg=getattr(policy, "idle_cfg", None), records="f64", trace_dtype=np.float64,
                    device=policy.device, goal_changes=sched, stream_spec=[0])
    policy._finish(res)
    n_in = len(env.slowdown)
    spec_idx = np.zeros(n_in, np.int32)
    for k, (start, _) in enumerate(goal_changes or ()):
        spec_idx[int(start):] = k + 1
    preds = chosen_predictions(policy._engine(), space, spec_arr, policy.code_name, res, spec_idx,
                               kalman=policy.kalman, idle_cfg=getattr(policy, "idle_cfg", None))
    d = res.decoded()
    cands = res.candidates
    oh = [float(sp.overhead_budget) for sp in specs]
    recs = []
    for n in range(n_in):
        c = int(d["cand"][n, 0])
        dec = decision_of(cands, c, int(d["level"][n, 0]), bool(d["feasible"][n, 0]), preds[n])
        recs.append(StepRecord(
            input_index=n, decision=dec, true_slowdown=float(env.slowdown[n]),
            observed_latency=float(res.records["latency"][n, 0]), completed_stage=int(d["completed"][n, 0]),
            deadline_met=bool(d["met"][n, 0]), delivered_accuracy=float(res.records["accuracy"][n, 0]),
            energy=float(res.records["energy"][n, 0]),
            violations=ViolationFlags(bool(d["viol_lat"][n, 0]), bool(d["viol_acc"][n, 0]),
                                      bool(d["viol_energy"][n, 0])),
            phase_index=int(env.phase_index[n]),
            period=float(res.records["plan_goal"][n, 0]) + oh[spec_idx[n]],
            fb_latency=float(res.records["fb_latency"][n, 0]), fb_t_prof=float(res.records["fb_t_prof"][n, 0]),
            idle_power_true=float(env.idle_power[n]),
        ))
    return RunResult(tuple(recs), summary_from_agg(res.agg[0], len(trace.phases)))


def chosen_predictions(eng: Engine, space, spec_arr: np.ndarray, policy: str, res: BatchResult,
                       spec_idx: np.ndarray, stream: int = 0, kalman=None, idle_cfg=None,
                       chunk: int = 4096) -> list:
    """``ConfigDecision.prediction`` of every step of one stream of an f64
    run_batch result, as the reference's policies build it:

    * alert / alert-any / alert-trad: the chosen entry of predict_all at the
      state the decide saw (selector.py:122-128) — one alert_predict launch
      per chunk of steps, each step a "stream" whose state is the previous
      step's (mu, sigma2, phi) record (the initial state for step 0);
    * oracle: _exact_pred of the executed config (policies.py:201-205): the
      step's measured latency / met / accuracy / energy;
    * oracle-static: _exact_pred(.., eligible, 0, 0, 0) (policies.py:266-271);
    * sys-only: mean-energy prediction, pr 1/0 by feasibility (policies.py:314-320);
    * app-only / no-coord: latency from the estimator, the best stage's
      expected accuracy (no-coord: at the previous power), pr 0, energy 0
      (policies.py:357-368, 417-428)."""
    torch = __import__("torch")
    from .records import Prediction

    rec = res.records
    n = rec["decision"].shape[0]
    d = abi.decode_decision(np.asarray(rec["decision"])[:, stream].view(np.uint32))
    cand, feas = d["cand"], d["feasible"]
    cands = res.candidates
    if policy == "oracle":
        return [prediction_of(cands, int(cand[k]), {
            "latency_mean": rec["latency"][k, stream], "latency_sigma": 0.0,
            "pr_deadline": 1.0 if d["met"][k] else 0.0, "expected_accuracy": rec["accuracy"][k, stream],
            "energy": rec["energy"][k, stream]}) for k in range(n)]
    if policy == "oracle-static":
        return [prediction_of(cands, int(cand[k]), {
            "latency_mean": 0.0, "latency_sigma": 0.0, "pr_deadline": 1.0 if feas[k] else 0.0,
            "expected_accuracy": 0.0, "energy": 0.0}) for k in range(n)]
    table = eng.table(space)
    sp = np.array(spec_arr, copy=True)
    if policy == "sys-only":
        sp["has_pr"] = 0  # predict_energy_mean (policies.py:309, 320)
    init = eng.new_state(table, 1, kalman, idle_cfg)
    st0 = {k: float(init[k][0].item()) for k in ("mu", "sigma2", "phi")}
    prev = {k: np.concatenate([[st0[k]], np.asarray(rec[k])[:-1, stream]]) for k in ("mu", "sigma2", "phi")}
    goal = np.asarray(rec["plan_goal"])[:, stream]
    # the candidate whose prediction is reported (no-coord: accuracy at the previous power)
    pick = cand.astype(np.int64)
    acc_pick = pick
    if policy == "no-coord":
        power = cands[cand, 1]
        old = np.concatenate([[len(space.powers) - 1], power[:-1]])
        index = {tuple(c): k for k, c in enumerate(cands.tolist())}
        acc_pick = np.array([index[(int(cands[c, 0]), int(o), int(cands[c, 2]))] for c, o in zip(cand, old)])
    pv = np.zeros(n, abi.PREDICTION_DTYPE)
    pa = np.zeros(n, abi.PREDICTION_DTYPE)
    for b in range(0, n, chunk):
        e = min(n, b + chunk)
        st = eng.new_state(table, e - b, kalman, idle_cfg)
        for k in ("mu", "sigma2", "phi"):
            st[k].copy_(torch.from_numpy(np.ascontiguousarray(prev[k][b:e])))
        g = torch.from_numpy(np.ascontiguousarray(goal[b:e])).to(eng.tdev)
        ss = torch.from_numpy(np.ascontiguousarray(spec_idx[b:e], np.int32)).to(eng.tdev)
        raw = eng.predict(table, sp, st, g, stream_spec=ss)  # [e - b, C, bytes]
        rows = torch.arange(e - b, device=eng.tdev)
        for dst, idx in ((pv, pick), (pa, acc_pick)):
            sel = raw[rows, torch.from_numpy(idx[b:e]).to(eng.tdev)]
            dst[b:e] = sel.cpu().numpy().view(abi.PREDICTION_DTYPE).reshape(-1)
    out = []
    for k in range(n):
        c = int(cand[k])
        if policy in ("alert", "alert-any", "alert-trad"):
            out.append(prediction_of(cands, c, pv[k]))
        elif policy == "sys-only":
            i = int(cands[c, 0])
            acc = float(space.dnns[i].stages[0].accuracy)
            p = dict(zip(pv.dtype.names, pv[k].tolist()))
            p.update(pr_deadline=1.0 if feas[k] else 0.0, expected_accuracy=acc)
            out.append(prediction_of(cands, c, p))
        else:  # app-only / no-coord
            p = dict(zip(pv.dtype.names, pv[k].tolist()))
            p.update(pr_deadline=0.0, expected_accuracy=float(pa[k]["expected_accuracy"]), energy=0.0)
            out.append(prediction_of(cands, c, p))
    return out


def run_injected(space, spec, env: TrueEnvironment, policy: str = "alert", *, kalman=None,
                 group_size=None, forced=None, records: str = "f64", trace_dtype=np.float64,
                 device: int = 0, flags: int = 0) -> BatchResult:
    """One stream over an already-realized environment (parity harness)."""
    f = None if forced is None else np.asarray(forced, np.int32).reshape(-1, 1)
    return run_batch(space, [spec], [env], policy, kalman=kalman, group_sizes=group_size, records=records,
                     forced=f, trace_dtype=trace_dtype, device=device, flags=flags)

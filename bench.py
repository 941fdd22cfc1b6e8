#!/usr/bin/env python
"""Benchmark: stream-step scheduling decisions/sec of the fused ALERT kernel.

    python bench.py [--gpus N --steps K --warmup W] [--config c2] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU, NCCL)

A "step" is one pass of the hot path over one batch: every stream of the
configuration runs its whole trace (goal adjust -> decide -> execute ->
measure -> observe per input) in one alert_run launch.  Default workload =
BASELINE.json configs[1] ("c2"): 65,536 independent streams x 10,000 inputs,
min-energy mode, preset 8x5 table (55 candidates), per rank (weak scaling).
Inputs are synthetic realizations of the reference's preset contention
trace (seed 42 + global stream index), realized with numpy exactly as the
reference's realize(); the float32 trace (2.6 GB) is larger than L2.

Prints ONE JSON line on rank 0.  --impl reference times the reference's CPU
algorithm (the FP64 C restatement in oracle/, all host threads) on a bounded
sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (description, streams, steps, mode)
    "c1": ("single-stream ALERT min-energy, preset 55-candidate table, 1,000 inputs", 1, 1000, "minE"),
    "c2": ("65,536 streams x 10,000 steps, min-energy, preset table", 65536, 10000, "minE"),
    "c3": ("1,048,576 streams x 1,000 steps, max-accuracy pr_th 0.95, preset table (anytime)", 1 << 20, 1000,
           "maxA"),
    "c4": ("goal-sweep grid: 2 modes x 64 deadlines x 64 goals x 2,048 traces, 64x32 table", 1 << 24, 1000,
           "grid"),
    "c5": ("c4 + clairvoyant oracle fused alongside ALERT", 1 << 24, 1000, "grid"),
}
STRONG = ("c3", "c4", "c5")  # fixed-total configurations (BASELINE: 1M streams / 2^24 scenarios on 1-8 GPUs)
REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
           0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting", 0x1: "gpu_idle"}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# --------------------------------------------------------------------------
# workloads
#
# Every configuration is a list of independent items (streams, or grid
# scenarios for c4/c5).  Rank r of W owns the contiguous item range
# dist.shard(total, W, r):
#   * weak scaling (c1/c2 default, or --streams S): total = S x W, each rank S;
#   * strong scaling (c3/c4/c5 default, or --total-streams T): total fixed.

GRID = 1 << 24          # c4/c5: 2 modes x 64 deadlines x 64 goals x 2,048 traces
N_TRACES = 2048
SCRAMBLE = 0x9E3779B1   # odd: k -> k * SCRAMBLE mod 2^24 is a bijection of the grid


def grid_scenarios(k: np.ndarray, total: int) -> np.ndarray:
    """Scenario ids of sample items k (0 <= k < total).  The whole grid
    (total = 2^24) is scenario k itself.  A smaller sample keeps whole goal
    tuples (all 2,048 traces of each, consecutive as in the full grid, so the
    streams of a warp share their goal) and spreads the tuples over the grid
    with a multiplicative scramble (both modes alternate); below 2,048 items
    the items themselves are scrambled."""
    k = np.asarray(k, np.int64)
    if total >= GRID:
        return k
    if total % N_TRACES == 0:
        n_tuples = GRID // N_TRACES
        t = ((k // N_TRACES) * SCRAMBLE) % n_tuples
        return t * N_TRACES + k % N_TRACES
    return (k * SCRAMBLE) % GRID


def grid_coords(scen: np.ndarray):
    """scenario -> (spec index, trace row).  Goal tuple t = scen // 2048 with
    the mode in its lowest bit (every contiguous range of scenarios holds both
    modes evenly), then the deadline multiplier and the goal; spec index =
    mode * 4096 + deadline * 64 + goal (specs: 64x64 min-energy, then 64x64
    max-accuracy)."""
    t = scen // N_TRACES
    mode = t % 2
    rest = t // 2
    dm, g = rest // 64, rest % 64
    return (mode * 4096 + dm * 64 + g).astype(np.int32), (scen % N_TRACES).astype(np.int32)


def item_range(cfg: str, world: int, rank: int, total: int | None = None, per_rank: int | None = None):
    """(begin, end, total, scaling) of the items rank r owns."""
    from paper_1911_00119_b200.dist import shard

    _, default_n, _, _ = CONFIGS[cfg]
    if per_rank is not None:
        total, scaling = per_rank * world, "weak"
    elif total is not None:
        scaling = "strong"
    elif cfg in STRONG:
        total, scaling = default_n, "strong"
    else:
        total, scaling = default_n * world, "weak"
    b, e = shard(total, world, rank)
    return b, e, total, scaling


def grid_specs(space):
    import paper_1911_00119_b200 as A

    ref = A.reference_latency(space)
    pmax = space.max_power.cap_watts
    dms = np.linspace(0.4, 2.0, 64)
    specs = []
    for dm in dms:
        for q in np.linspace(0.30, 0.97, 64):
            specs.append(A.ConstraintSpec(mode=A.Mode.MINIMIZE_ENERGY, t_goal=float(dm * ref), q_goal=float(q),
                                          overhead_budget=0.01 * ref))
    for dm in dms:
        for em in np.linspace(0.2, 1.0, 64):
            t = float(dm * ref)
            specs.append(A.ConstraintSpec(mode=A.Mode.MAXIMIZE_ACCURACY, t_goal=t, e_goal=float(em) * pmax * t,
                                          overhead_budget=0.01 * ref))
    return specs


def grid_traces(n_steps: int):
    """The 2,048 shared contention traces (preset regimes, seeded permuted
    phase order and cut points, seeds 42 + t)."""
    from paper_1911_00119_b200.synth import preset_batch
    from paper_1911_00119_b200.trace import PackedEnvs

    rng = np.random.default_rng(1000)
    orders = [tuple(rng.permutation(3)) for _ in range(N_TRACES)]
    m = min(100, n_steps // 4)  # phase cuts at least m steps from either end (100 at full size)
    cuts = [np.sort(rng.integers(m, n_steps - m, 2)) for _ in range(N_TRACES)]
    parts = []
    for t in range(N_TRACES):
        a, b = cuts[t]
        lengths = (int(a), int(b - a), int(n_steps - b))
        parts.append(preset_batch(1, lengths=lengths, seed0=42 + t, order=orders[t], dtype=np.float32,
                                  processes=1))
    return PackedEnvs(np.concatenate([p.slowdown for p in parts], 1),
                      np.concatenate([p.n_segments for p in parts]), np.concatenate([p.seg_end for p in parts]),
                      np.concatenate([p.seg_phase for p in parts]), np.concatenate([p.seg_idle for p in parts]))


def build_workload(cfg: str, n_steps: int, begin: int, end: int, total: int, goal_changes: int = 0):
    """Items [begin, end) of configuration ``cfg`` (global item indices, so a
    stream's trace seed / a scenario's coordinates do not depend on the
    world size)."""
    import paper_1911_00119_b200 as A
    from paper_1911_00119_b200.synth import preset_batch

    desc, _, _, kind = CONFIGS[cfg]
    n = end - begin
    if kind in ("minE", "maxA"):
        space = A.preset_space()
        ref = A.reference_latency(space)
        if kind == "minE":
            specs = [A.ConstraintSpec(mode=A.Mode.MINIMIZE_ENERGY, t_goal=dm * ref, q_goal=q,
                                      overhead_budget=0.01 * ref)
                     for q in (0.68, 0.70, 0.85) for dm in (0.8, 1.0, 1.5)]
            if cfg == "c1":
                specs = [A.ConstraintSpec(mode=A.Mode.MINIMIZE_ENERGY, t_goal=0.14, q_goal=0.68,
                                          overhead_budget=0.01 * ref)]
        else:
            t = 0.8 * ref
            specs = [A.ConstraintSpec(mode=A.Mode.MAXIMIZE_ACCURACY, t_goal=t, e_goal=0.6 * 50.0 * t,
                                      pr_threshold=0.95, overhead_budget=0.01 * ref)]
        L = (n_steps - 2 * (n_steps // 3), n_steps // 3, n_steps // 3)
        packed = preset_batch(n, lengths=L, seed0=42 + begin, dtype=np.float32)
        spec_arr = A.pack_specs(specs)
        stream_spec = (np.arange(begin, end) % len(specs)).astype(np.int32)
        if goal_changes:  # the goal of every stream changes K times (cycling through the spec list)
            from paper_1911_00119_b200.trace import pack_goal_changes

            cuts = [(n_steps * (c + 1)) // (goal_changes + 1) for c in range(goal_changes)]
            sched = [[(0, int(g % len(specs)))] + [(c, int((g + 1 + i) % len(specs))) for i, c in enumerate(cuts)]
                     for g in range(begin, end)]
            packed.goal_n, packed.goal_end, packed.goal_spec = pack_goal_changes(sched, n_steps, len(specs))
        return dict(space=space, specs=spec_arr, stream_spec=stream_spec, stream_row=None, packed=packed,
                    desc=desc, n_streams=n, n_steps=n_steps, begin=begin, end=end, total=total)
    # c4 / c5: goal-sweep grid over shared traces
    space = A.generate_space(A.ProfileKnobs(n_dnns=64, n_powers=32))
    scen = grid_scenarios(np.arange(begin, end), total)
    spec_idx, row = grid_coords(scen)
    order = np.argsort(spec_idx >= 4096, kind="stable")  # this rank's min-energy items first: 2 launches
    return dict(space=space, specs=A.pack_specs(grid_specs(space)), stream_spec=spec_idx[order],
                stream_row=row[order], packed=grid_traces(n_steps), desc=desc, n_streams=n, n_steps=n_steps,
                begin=begin, end=end, total=total)


def n_candidates(space) -> int:
    from paper_1911_00119_b200.packing import pack_space

    return pack_space(space).n_candidates


# --------------------------------------------------------------------------
# clocks sampled during the timed region

class ClockSampler:
    """SM clock / max clock / event reasons during the timed region: NVML
    polled every 2 ms from a thread (in-process; short timed regions such as
    c1's ~15 ms still get samples), else an ``nvidia-smi -lms 50`` process.
    Samples are lines "sm, max, 0xreasons" with their host time."""

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []
        self.source = None
        self._stop = threading.Event()

    def _nvml_handle(self):
        import pynvml
        import torch

        pynvml.nvmlInit()
        uuid = str(torch.cuda.get_device_properties(self.device).uuid)
        uuid = uuid if uuid.startswith("GPU-") else "GPU-" + uuid
        try:
            return pynvml, pynvml.nvmlDeviceGetHandleByUUID(uuid)
        except pynvml.NVMLError:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.device)

    def _poll_nvml(self, nv, h):
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.lines.append((time.monotonic(), f"{sm}, {mx}, {rs:#x}"))
            except nv.NVMLError:
                return
            time.sleep(0.002)

    def __enter__(self):
        try:
            nv, h = self._nvml_handle()
            self.source = "nvml (2 ms)"
            self.t = threading.Thread(target=self._poll_nvml, args=(nv, h), daemon=True)
            self.t.start()
            return self
        except Exception:  # no NVML binding / device: the nvidia-smi process below
            pass
        try:
            self.source = "nvidia-smi (50 ms)"
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.monotonic(), line.strip()))

    def mark(self, begin: bool):
        """Host times bracketing the timed region (samples outside are not reported)."""
        if begin:
            self.t0 = time.monotonic()
        else:
            self.t1 = time.monotonic()

    def __exit__(self, *exc):
        self._stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        t0, t1 = getattr(self, "t0", None), getattr(self, "t1", None)
        inside = [ln for t, ln in self.lines if t0 is None or t1 is None or t0 <= t <= t1 + 0.06]
        for ln in inside or [ln for _, ln in self.lines[-3:]]:
            try:
                a, b, c = [x.strip() for x in ln.split(",")]
                sm.append(float(a))
                mx = float(b)
                bits = int(c, 16)
                for k, v in REASONS.items():
                    if bits & k and v != "gpu_idle":
                        reasons.add(v)
            except ValueError:
                continue
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "source": self.source}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm),
                "source": self.source}


# --------------------------------------------------------------------------
# CPU baselines: the reference algorithm restated in C (oracle/, all host
# threads) and the reference's own Python path (baseline/_ref), timed on a
# bounded sample of the same workload

def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _sample_envs(wl, ns: int, steps: int):
    """PackedEnvs of the first ns items (their trace rows gathered), first steps inputs."""
    from paper_1911_00119_b200.trace import PackedEnvs

    packed = wl["packed"]
    rows = np.arange(ns) if wl["stream_row"] is None else wl["stream_row"][:ns]
    sub = PackedEnvs(np.ascontiguousarray(packed.slowdown[:steps, rows]), packed.n_segments[rows],
                     packed.seg_end[rows], packed.seg_phase[rows], packed.seg_idle[rows])
    if getattr(packed, "goal_n", None) is not None:
        sub.goal_n, sub.goal_end, sub.goal_spec = packed.goal_n[rows], packed.goal_end[rows], packed.goal_spec[rows]
    return sub


def cpu_baseline(wl, policy: str, seconds: float = 12.0, python_seconds: float = 8.0):
    from oracle import oracle

    threads = os.cpu_count() or 1
    n_steps = wl["n_steps"]

    def sample(ns, steps):
        sub = _sample_envs(wl, ns, steps)
        t0 = time.perf_counter()
        oracle.run_batch(wl["space"], wl["specs"], sub, ns, policy, stream_spec=wl["stream_spec"][:ns],
                         step_end=steps, threads=min(threads, ns))
        return time.perf_counter() - t0

    cal_steps = min(n_steps, 500)
    dt = sample(min(threads, wl["n_streams"]), cal_steps)
    rate = min(threads, wl["n_streams"]) * cal_steps / dt
    steps = min(n_steps, max(cal_steps, int(seconds * rate / max(1, min(threads, wl["n_streams"])))))
    ns = min(wl["n_streams"], max(threads, int(seconds * rate / steps)))
    dt = sample(ns, steps)
    out = {"value": ns * steps / dt, "unit": "decisions/s", "cores": min(threads, ns), "kind": "port",
           "cpu_model": cpu_model(),
           "sample": f"{ns} items x {steps} steps of {wl['desc']} ({policy}), oracle/alert_oracle.c FP64, "
                     f"{min(threads, ns)} POSIX threads, {dt:.1f} s"}
    if python_seconds > 0:
        out["python_reference"] = python_reference(wl, policy, python_seconds)
    return out


_PY = {}


def _py_ref_init(space_kind: str):
    """Pool initializer: import the reference (baseline/_ref) and build its table."""
    sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
    import alertsim.simulator as S
    from alertsim import synth

    _PY["S"] = S
    _PY["space"] = synth.preset_space() if space_kind == "preset" else \
        synth.generate_space(synth.ProfileKnobs(n_dnns=64, n_powers=32))


def _py_ref_stream(job):
    """One stream through the reference's own simulator.run + make_policy on
    the injected arrays (realize() replaced by the realized environment)."""
    from alertsim.model import ConstraintSpec, Mode
    from alertsim.policies import make_policy
    from alertsim.simulator import Constant, EnvironmentPhase, Trace, TrueEnvironment

    S = _PY["S"]
    s, idle, phase, spec, policy = job
    mode = Mode.MINIMIZE_ENERGY if spec["mode"] == 0 else Mode.MAXIMIZE_ACCURACY
    sp = ConstraintSpec(mode=mode, t_goal=spec["t_goal"], q_goal=spec["q_goal"] if mode is Mode.MINIMIZE_ENERGY
                        else None, e_goal=spec["e_goal"] if mode is Mode.MAXIMIZE_ACCURACY else None,
                        pr_threshold=spec["pr_threshold"] if spec["has_pr"] else None,
                        overhead_budget=spec["overhead_budget"])
    env = TrueEnvironment(s, idle, phase)
    n_ph = int(phase.max()) + 1
    trace = Trace(seed=0, phases=tuple(EnvironmentPhase(int((phase == k).sum()) or 1, Constant(1.0), 1.0)
                                       for k in range(n_ph)))
    S.realize = lambda tr: env
    S.run(_PY["space"], sp, trace, make_policy(policy))
    return len(s)


def python_reference(wl, policy: str, seconds: float = 8.0):
    """The reference's own Python path (alertsim.simulator.run + make_policy,
    simulator.py:461-507 / policies.py:469-490, from baseline/_ref) under
    multiprocessing.Pool(all cores), one stream per task."""
    import multiprocessing as mp

    if not (ROOT / "baseline" / "_ref" / "alertsim").exists():
        return {"unavailable": "baseline/_ref not installed (pip install --target baseline/_ref the reference)"}
    if policy not in ("alert", "alert-any", "alert-trad", "oracle"):
        policy = "alert"
    cores = os.cpu_count() or 1
    kind = "preset" if wl["space"].dnns[0].stages[0].t_prof and len(wl["space"].dnns) == 8 else "grid"
    sub_all = _sample_envs(wl, min(wl["n_streams"], 4 * cores), wl["n_steps"])
    from paper_1911_00119_b200.trace import unpack_row

    def jobs(ns, steps):
        out = []
        for k in range(ns):
            env = unpack_row(sub_all, k)
            spec = wl["specs"][int(wl["stream_spec"][k])]
            out.append((env.slowdown[:steps].copy(), env.idle_power[:steps].copy(), env.phase_index[:steps].copy(),
                        {f: spec[f].item() for f in spec.dtype.names}, policy))
        return out

    ctx = mp.get_context("fork")
    with ctx.Pool(cores, initializer=_py_ref_init, initargs=(kind,)) as pool:
        cal = min(wl["n_steps"], 100)
        t0 = time.perf_counter()
        pool.map(_py_ref_stream, jobs(1, cal))
        per_step = (time.perf_counter() - t0) / cal
        steps = int(min(wl["n_steps"], max(cal, seconds / per_step)))
        rounds = max(1, int(seconds / (per_step * steps)))  # fill ~`seconds` of wall time on every core
        ns = min(sub_all.n_rows, cores * rounds)
        t0 = time.perf_counter()
        done = sum(pool.map(_py_ref_stream, jobs(ns, steps), chunksize=1))
        dt = time.perf_counter() - t0
    return {"value": done / dt, "unit": "decisions/s", "cores": min(cores, ns), "kind": "reference-python",
            "cpu_model": cpu_model(),
            "sample": f"{ns} items x {steps} steps of {wl['desc']} ({policy}): alertsim.simulator.run + make_policy "
                      f"(baseline/_ref, Python {sys.version.split()[0]}), multiprocessing.Pool({cores}), {dt:.1f} s"}


# --------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--policy", default=None)
    ap.add_argument("--streams", type=int, default=None, help="items per rank (weak scaling)")
    ap.add_argument("--total-streams", type=int, default=None,
                    help="items over all ranks (strong scaling; default for c3/c4/c5: 2^20 / 2^24 / 2^24)")
    ap.add_argument("--trace-steps", type=int, default=None, help="override steps per stream")
    ap.add_argument("--goal-changes", type=int, default=0, help="c1-c3: goal changes per stream (trace input)")
    ap.add_argument("--lanes", type=int, default=0)
    ap.add_argument("--tpb", type=int, default=0)  # 0 = library default (64)
    ap.add_argument("--records", default="none", choices=["none", "f32"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-python-ref", action="store_true")
    ap.add_argument("--flags", type=int, default=0)
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    desc, _, N, kind = CONFIGS[args.config]
    N = args.trace_steps or N
    begin, end, total, scaling = item_range(args.config, world, rank, args.total_streams, args.streams)
    S = end - begin
    policy = args.policy or ("alert+oracle" if args.config == "c5" else "alert")
    metric = "stream-step decisions/sec"

    if args.impl == "reference":
        if rank != 0:
            return
        wl = build_workload(args.config, N, 0, min(total, 4096), total, args.goal_changes)
        log(f"[reference] CPU oracle port on {os.cpu_count()} host threads, {desc}")
        vals = []
        for i in range(args.warmup + args.steps):
            cb = cpu_baseline(wl, "alert" if policy == "alert+oracle" else policy, seconds=6.0,
                              python_seconds=0.0 if (i < args.warmup + args.steps - 1 or args.no_python_ref)
                              else 8.0)
            if i >= args.warmup:
                vals.append(cb["value"])
        v = float(np.mean(vals))
        print(json.dumps({
            "impl": "reference", "metric": metric, "value": v, "unit": "decisions/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference preset traces, numpy realize)",
            "config": {"workload": args.config, "desc": desc, "total_items": total, "steps_per_stream": N,
                       "policy": policy},
            "cpu_baseline": {"value": v, "unit": "decisions/s", "cores": cb["cores"], "kind": "port",
                             "cpu_model": cb["cpu_model"], "sample": cb["sample"],
                             "python_reference": cb.get("python_reference")},
            "e2e": {"value": v, "unit": "decisions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }))
        return

    import torch

    # one process per GPU; more ranks than GPUs (a code-path check on a
    # one-GPU box) share the devices round-robin and need ALERT_DIST_BACKEND=gloo
    # (NCCL refuses two ranks on one device)
    shared = world > torch.cuda.device_count()
    local = local % max(1, torch.cuda.device_count())
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group(os.environ.get("ALERT_DIST_BACKEND", "nccl"), init_method="env://")
    else:
        torch.cuda.set_device(local)
    import paper_1911_00119_b200 as A
    from paper_1911_00119_b200 import abi
    from paper_1911_00119_b200._lib import load
    from paper_1911_00119_b200.dist import max_over_ranks, reduce_aggregates, sum_over_ranks
    from paper_1911_00119_b200.engine import outputs_struct
    from paper_1911_00119_b200.packing import mode_runs, policy_code
    from paper_1911_00119_b200.simulator import HostStreamer

    t0 = time.time()
    wl = build_workload(args.config, N, begin, end, total, args.goal_changes)
    log(f"[rank {rank}] workload {args.config}: items [{begin}, {end}) of {total} x {N} steps built in "
        f"{time.time() - t0:.1f}s")
    eng = A.get_engine(local)
    if args.lanes or args.tpb:
        eng.set_launch(args.lanes, args.tpb)
    table = eng.table(wl["space"])
    C = table.n_candidates
    dev = eng.tdev
    trace = eng.upload_trace(wl["packed"], wl["stream_row"])
    # one launch per contiguous run of one goal mode (mode-homogeneous kernels);
    # rows with goal changes run as one launch over every spec
    if getattr(wl["packed"], "goal_n", None) is not None:
        launches = [(0, S, wl["specs"], torch.as_tensor(wl["stream_spec"]).to(dev))]
    else:
        launches = [(b, e, sp, torch.as_tensor(full).to(dev))
                    for b, e, sp, full in mode_runs(wl["specs"], wl["stream_spec"])]
    agg = torch.zeros((S, abi.AGG_FIELDS), dtype=torch.float64, device=dev)
    rec = {}
    if args.records == "f32":
        rec["decision"] = torch.empty((N, S), dtype=torch.int32, device=dev)
        for k in ("energy", "accuracy", "latency", "mu", "sigma2"):
            rec[k] = torch.empty((N, S), dtype=torch.float32, device=dev)
    out = outputs_struct(rec or None, agg=agg)
    pol = policy_code(policy)
    stream = torch.cuda.current_stream(dev)
    kev = []  # (start, end) events around each step's alert_run launches
    # inputs that fit in L2 (c4/c5 share 2,048 trace rows): flush L2 before
    # every step by writing a buffer larger than it; the step is then timed by
    # its own events (flush excluded)
    trace_bytes = wl["packed"].slowdown.nbytes
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if trace_bytes < 126e6 else None

    def step(timed: bool):
        state = eng.new_state(table, S, init=False)  # initialised by the launch (FLAG_FRESH)
        if flush is not None:
            flush.fill_(1)
        if timed:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
        for lb, le, lsp, lss in launches:
            eng.run(table, lsp, trace, state, policy=pol, stream_spec=lss, outputs=out,
                    flags=args.flags | abi.FLAG_FRESH, stream_begin=lb, stream_end=le)
        if timed:
            b.record(stream)
            kev.append((a, b))

    # the clock sampler (an nvidia-smi process) starts before the warm-up, so
    # its start-up never overlaps the timed region; only samples taken during
    # the timed region are reported
    clk = ClockSampler(local).__enter__()
    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize(dev)
    launches0 = eng.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk.mark(True)
    e0.record(stream)
    for _ in range(args.steps):
        step(True)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    clk.mark(False)
    clk.__exit__(None, None, None)
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    gpu_launches = eng.launch_count() - launches0
    kernel_ms = float(np.mean([a.elapsed_time(b) for a, b in kev]))
    if flush is not None:  # the L2 flushes between steps are not part of the steps
        ms = float(np.sum([a.elapsed_time(b) for a, b in kev]))
    ms = max_over_ranks(ms, dev)
    decisions = args.steps * total * N  # every rank's items, each step
    value = decisions / (ms * 1e-3)

    # final aggregate of the last step: deterministic per-GPU reduce, then the
    # one cross-GPU exchange (NCCL all_gather, summed in rank order)
    tot = reduce_aggregates(eng.reduce(agg)).cpu().numpy()
    n_all = tot[abi.AGG_N]
    assert n_all == total * N, (n_all, total * N)
    quality = {
        "mean_energy_j": float((tot[abi.AGG_ENERGY] + tot[abi.AGG_ENERGY_C]) / n_all),
        "mean_accuracy": float((tot[abi.AGG_ACC] + tot[abi.AGG_ACC_C]) / n_all),
        "viol_latency_rate": float(tot[abi.AGG_VIOL_LAT] / n_all),
        "viol_accuracy_rate": float(tot[abi.AGG_VIOL_ACC] / n_all),
        "viol_energy_rate": float(tot[abi.AGG_VIOL_ENERGY] / n_all),
        "fp64_rerank_fraction": float(tot[abi.AGG_REFINED] / n_all),
        "full_scan_fraction": float(tot[abi.AGG_FULL_SCAN] / n_all),
    }
    if policy == "alert+oracle":
        quality["oracle_mean_energy_j"] = float((tot[abi.AGG_OR_ENERGY] + tot[abi.AGG_OR_ENERGY_C]) / n_all)
        quality["oracle_mean_accuracy"] = float((tot[abi.AGG_OR_ACC] + tot[abi.AGG_OR_ACC_C]) / n_all)

    # roofline of the dominant kernel (run_kernel): algorithmic FP32 slots per decision
    # ALERT 30 C + 60 FP32 slots and C + 6 MUFU per decision;
    # the oracle evaluated alongside (config 5) adds 15 C + 20 slots, no MUFU
    slots = 30 * C + 60 + (15 * C + 20 if policy == "alert+oracle" else 0)
    mufu = C + 6
    per_launch = S * N  # this rank's decisions per step (all of its launches)
    kernel_ms = max_over_ranks(kernel_ms, dev)
    ach = per_launch * slots / (kernel_ms * 1e-3)
    peak = None
    import ctypes

    pk = ctypes.c_double()
    if load().alert_probe_fp32_peak(local, ctypes.byref(pk)) == 0:
        peak = pk.value
    clocks = clk.summary()
    peak_nominal = 148 * 128 * 1965e6
    traffic, traffic_src = None, None  # DRAM bytes per launch from a committed ncu capture
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if tf.exists():
        try:
            t = json.loads(tf.read_text()).get(args.config)
            if t:
                traffic = t["bytes_per_decision"] * per_launch
                traffic_src = (f"ncu capture {t.get('source', '?')} at {t.get('shape', '?')}: "
                               f"{t['bytes_per_decision']:.3g} dram B/decision x this launch's decisions"
                               + ("" if t.get("shape_matches_bench") else " (extrapolated from a different shape)"))
        except (ValueError, KeyError):
            traffic = None
    in_bytes = 4 * per_launch + (24 * per_launch if args.records == "f32" else 0)
    roof = {
        "bound": "fp32", "achieved": ach / 1e9, "peak": (peak or peak_nominal) / 1e9, "unit": "Gslot/s",
        "frac": ach / (peak or peak_nominal), "traffic": traffic, "traffic_source": traffic_src,
        "peak_source": "measured FFMA probe (alert_probe_fp32_peak) at the run's clocks" if peak else
                       "nominal 148 SM x 128 lanes x 1965 MHz",
        "peak_nominal_gslot_s": peak_nominal / 1e9,
        "frac_of_nominal": ach / peak_nominal,
        "algorithmic_slots_per_decision": slots, "candidates": C,
        "kernel_ms_per_launch": kernel_ms, "decisions_per_launch": per_launch,
        "sfu": {"achieved": per_launch * mufu / (kernel_ms * 1e-3) / 1e9,
                "peak": 16 * 148 * 1965e6 / 1e9, "unit": "Gop/s",
                "frac": per_launch * mufu / (kernel_ms * 1e-3) / (16 * 148 * 1965e6)},
        "hbm": {"algorithmic_bytes_per_launch": in_bytes,
                "achieved_gbs": in_bytes / (kernel_ms * 1e-3) / 1e9},
    }

    # end-to-end through the public API: host-pinned trace streamed in step
    # chunks (H2D overlapped with the kernel), per-stream summaries back (D2H)
    e2e = None
    if not args.no_e2e:
        hs = HostStreamer(wl["space"], wl["specs"], wl["packed"], policy, stream_spec=wl["stream_spec"],
                          stream_row=wl["stream_row"], chunk_steps=max(1, N // 10), engine=eng)
        hs.run()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            hs.run()
        b.record(stream)
        torch.cuda.synchronize(dev)
        ems = max_over_ranks(a.elapsed_time(b), dev)
        e2e = {"value": decisions / (ems * 1e-3), "unit": "decisions/s",
               "h2d_bytes_per_step": int(sum_over_ranks(hs.h2d_bytes, dev)),
               "d2h_bytes_per_step": int(sum_over_ranks(hs.d2h_bytes, dev)),
               "path": "paper_1911_00119_b200.simulator.HostStreamer (pinned host trace + scenario map, chunked "
                       "H2D overlapped with alert_run, per-stream aggregates D2H)"}

    cpu = None
    if rank == 0 and not args.no_cpu:  # rank 0 only, after the timed regions (other ranks wait)
        cpu = cpu_baseline(wl, "alert" if policy == "alert+oracle" else policy,
                           python_seconds=0.0 if args.no_python_ref else 8.0)
    if world > 1:
        dist.barrier()

    lanes, tpb = eng.launch_config()
    if rank == 0:
        line = {
            "metric": metric, "value": value, "unit": "decisions/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "fp32 scan + fp64 re-rank/state",
            "data": "synthetic: reference preset contention traces realized with numpy (seed 42 + item)",
            "config": {"workload": args.config, "desc": desc, "total_items": total, "items_per_rank": S,
                       "steps_per_stream": N, "candidates": C, "policy": policy, "records": args.records,
                       "goal_changes_per_stream": args.goal_changes,
                       "lanes_per_stream": lanes or (1 if C <= 256 else 8),
                       "threads_per_block": tpb if args.tpb else "auto (64; 512 when the staged table > 40 KB)",
                       "l2": "inputs larger than L2" if flush is None else
                             "L2 flushed before every step (256 MB write, outside the step's events)",
                       "parallelism": f"items sharded (dist.shard, contiguous), {world} rank(s), {scaling} scaling"
                                      + (" [ranks share GPUs: a code-path check, not a scaling number]" if shared else "")},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": gpu_launches,
            "clocks": clocks, "quality": quality,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

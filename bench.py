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
REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
           0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting", 0x1: "gpu_idle"}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# --------------------------------------------------------------------------
# workloads

def build_workload(cfg: str, n_streams: int, n_steps: int, rank: int, world: int = 1):
    import paper_1911_00119_b200 as A
    from paper_1911_00119_b200.synth import preset_batch
    from paper_1911_00119_b200.trace import PackedEnvs

    desc, _, _, kind = CONFIGS[cfg]
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
        packed = preset_batch(n_streams, lengths=L, seed0=42 + rank * n_streams, dtype=np.float32)
        return dict(space=space, specs=A.pack_specs(specs), stream_spec=None, stream_row=None, packed=packed,
                    desc=desc, n_streams=n_streams, n_steps=n_steps)
    # c4 / c5: goal-sweep grid over shared traces
    space = A.generate_space(A.ProfileKnobs(n_dnns=64, n_powers=32))
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
    n_traces = 2048
    # scenario s -> (goal tuple s // 2048, trace s % 2048); a rank owns a contiguous range
    # every rank's scenarios sample the whole 2^24 grid evenly (both modes,
    # every goal tuple, every trace; ranks interleaved, disjoint) when the job
    # holds fewer than 2^24 of them
    stride = max(1, (1 << 24) // (n_streams * world))
    scen = (np.arange(n_streams, dtype=np.int64) * world + rank) * stride
    stream_spec = (scen // n_traces) % len(specs)
    stream_row = scen % n_traces
    parts = []
    rng = np.random.default_rng(1000)
    orders = [tuple(rng.permutation(3)) for _ in range(n_traces)]
    m = min(100, n_steps // 4)  # phase cuts at least m steps from either end (100 at full size)
    cuts = [np.sort(rng.integers(m, n_steps - m, 2)) for _ in range(n_traces)]
    for t in range(n_traces):
        a, b = cuts[t]
        lengths = (int(a), int(b - a), int(n_steps - b))
        parts.append(preset_batch(1, lengths=lengths, seed0=42 + t, order=orders[t], dtype=np.float32,
                                  processes=1))
    packed = PackedEnvs(np.concatenate([p.slowdown for p in parts], 1),
                        np.concatenate([p.n_segments for p in parts]), np.concatenate([p.seg_end for p in parts]),
                        np.concatenate([p.seg_phase for p in parts]), np.concatenate([p.seg_idle for p in parts]))
    return dict(space=space, specs=A.pack_specs(specs), stream_spec=stream_spec.astype(np.int32),
                stream_row=stream_row.astype(np.int32), packed=packed, desc=desc, n_streams=n_streams,
                n_steps=n_steps)


def n_candidates(space) -> int:
    from paper_1911_00119_b200.packing import pack_space

    return pack_space(space).n_candidates


# --------------------------------------------------------------------------
# clocks sampled during the timed region

class ClockSampler:
    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
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
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        for ln in self.lines:
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
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------
# CPU baseline (the reference algorithm restated in C, oracle/)

def cpu_baseline(wl, policy: str, seconds: float = 12.0):
    from oracle import oracle
    from paper_1911_00119_b200.trace import PackedEnvs

    threads = os.cpu_count() or 1
    packed = wl["packed"]
    n_steps = wl["n_steps"]

    def sample(ns, steps):
        sub = PackedEnvs(np.ascontiguousarray(packed.slowdown[:steps, :ns]), packed.n_segments[:ns],
                         packed.seg_end[:ns], packed.seg_phase[:ns], packed.seg_idle[:ns])
        ss = None if wl["stream_spec"] is None else wl["stream_spec"][:ns]
        sr = None if wl["stream_row"] is None else wl["stream_row"][:ns]
        if sr is not None:  # gather the rows the sampled streams read
            sub = PackedEnvs(np.ascontiguousarray(packed.slowdown[:steps, sr]), packed.n_segments[sr],
                             packed.seg_end[sr], packed.seg_phase[sr], packed.seg_idle[sr])
        t0 = time.perf_counter()
        oracle.run_batch(wl["space"], wl["specs"], sub, ns, policy, stream_spec=ss, step_end=steps,
                         threads=min(threads, ns))
        return time.perf_counter() - t0

    cal_steps = min(n_steps, 500)
    dt = sample(min(threads, wl["n_streams"]), cal_steps)
    rate = min(threads, wl["n_streams"]) * cal_steps / dt
    steps = min(n_steps, max(cal_steps, int(seconds * rate / max(1, min(threads, wl["n_streams"])))))
    ns = min(wl["n_streams"], max(threads, int(seconds * rate / steps)))
    dt = sample(ns, steps)
    return {"value": ns * steps / dt, "unit": "decisions/s", "cores": min(threads, ns), "kind": "port",
            "sample": f"{ns} streams x {steps} steps of {wl['desc']} ({policy}), oracle/alert_oracle.c FP64, "
                      f"{min(threads, ns)} POSIX threads, {dt:.1f} s"}


# --------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--policy", default=None)
    ap.add_argument("--streams", type=int, default=None, help="override streams per rank")
    ap.add_argument("--trace-steps", type=int, default=None, help="override steps per stream")
    ap.add_argument("--lanes", type=int, default=0)
    ap.add_argument("--tpb", type=int, default=0)  # 0 = library default (64)
    ap.add_argument("--records", default="none", choices=["none", "f32"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--flags", type=int, default=0)
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    desc, S, N, kind = CONFIGS[args.config]
    S = args.streams or S
    N = args.trace_steps or N
    policy = args.policy or ("alert+oracle" if args.config == "c5" else "alert")
    metric = "stream-step decisions/sec"

    if args.impl == "reference":
        if rank != 0:
            return
        wl = build_workload(args.config, min(S, 4096), N, 0)
        log(f"[reference] CPU oracle port on {os.cpu_count()} host threads, {desc}")
        vals = []
        for i in range(args.warmup + args.steps):
            cb = cpu_baseline(wl, policy, seconds=6.0)
            if i >= args.warmup:
                vals.append(cb["value"])
        v = float(np.mean(vals))
        print(json.dumps({
            "impl": "reference", "metric": metric, "value": v, "unit": "decisions/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference preset traces, numpy realize)",
            "config": {"workload": args.config, "desc": desc, "streams_per_rank": S, "steps_per_stream": N,
                       "policy": policy},
            "cpu_baseline": {"value": v, "unit": "decisions/s", "cores": cb["cores"], "kind": "port",
                             "sample": cb["sample"]},
            "e2e": {"value": v, "unit": "decisions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }))
        return

    import torch

    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", init_method="env://")
    else:
        torch.cuda.set_device(local)
    import paper_1911_00119_b200 as A
    from paper_1911_00119_b200 import abi
    from paper_1911_00119_b200._lib import load
    from paper_1911_00119_b200.dist import max_over_ranks, reduce_aggregates
    from paper_1911_00119_b200.engine import outputs_struct
    from paper_1911_00119_b200.packing import policy_code
    from paper_1911_00119_b200.simulator import HostStreamer

    t0 = time.time()
    wl = build_workload(args.config, S, N, rank, world)
    log(f"[rank {rank}] workload {args.config}: {S} streams x {N} steps built in {time.time() - t0:.1f}s")
    eng = A.get_engine(local)
    if args.lanes or args.tpb:
        eng.set_launch(args.lanes, args.tpb)
    table = eng.table(wl["space"])
    C = table.n_candidates
    dev = eng.tdev
    trace = eng.upload_trace(wl["packed"], wl["stream_row"])
    # one launch per contiguous run of one goal mode (mode-homogeneous kernels)
    from paper_1911_00119_b200.packing import mode_runs

    if wl["stream_spec"] is None:
        launches = [(0, S, wl["specs"], None)]
    else:
        launches = [(b, e, sp, torch.as_tensor(full).to(dev)) for b, e, sp, full in mode_runs(wl["specs"],
                                                                                           wl["stream_spec"])]
    agg = torch.zeros((S, abi.AGG_FIELDS), dtype=torch.float64, device=dev)
    rec = {}
    if args.records == "f32":
        rec["decision"] = torch.empty((N, S), dtype=torch.int32, device=dev)
        for k in ("energy", "accuracy", "latency", "mu", "sigma2"):
            rec[k] = torch.empty((N, S), dtype=torch.float32, device=dev)
    out = outputs_struct(rec or None, agg=agg)
    pol = policy_code(policy)
    stream = torch.cuda.current_stream(dev)
    kev = []  # (start, end) events around each alert_run launch

    def step(timed: bool):
        state = eng.new_state(table, S)
        agg.zero_()
        if timed:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
        for lb, le, lsp, lss in launches:
            eng.run(table, lsp, trace, state, policy=pol, stream_spec=lss, outputs=out, flags=args.flags,
                    stream_begin=lb, stream_end=le)
        if timed:
            b.record(stream)
            kev.append((a, b))

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize(dev)
    launches0 = eng.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step(True)
        e1.record(stream)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    gpu_launches = eng.launch_count() - launches0
    kernel_ms = float(np.mean([a.elapsed_time(b) for a, b in kev]))
    ms = max_over_ranks(ms, dev)
    decisions = args.steps * S * N * world
    value = decisions / (ms * 1e-3)

    # final aggregate of the last step: deterministic per-GPU reduce, then the
    # one cross-GPU exchange (NCCL all_gather, summed in rank order)
    tot = reduce_aggregates(eng.reduce(agg)).cpu().numpy()
    n_all = tot[abi.AGG_N]
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
    per_launch = S * N
    ach = per_launch * slots / (kernel_ms * 1e-3)
    peak = C_double = None
    import ctypes

    pk = ctypes.c_double()
    if load().alert_probe_fp32_peak(local, ctypes.byref(pk)) == 0:
        peak = pk.value
    clocks = clk.summary()
    peak_nominal = 148 * 128 * 1965e6
    traffic = None  # DRAM bytes per launch, from the committed ncu capture (bytes/decision x decisions)
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if tf.exists():
        try:
            t = json.loads(tf.read_text()).get(args.config)
            if t:
                traffic = t["bytes_per_decision"] * S * N
        except (ValueError, KeyError):
            traffic = None
    in_bytes = 4 * per_launch + (24 * per_launch if args.records == "f32" else 0)
    roof = {
        "bound": "fp32", "achieved": ach / 1e9, "peak": (peak or peak_nominal) / 1e9, "unit": "Gslot/s",
        "frac": ach / (peak or peak_nominal), "traffic": traffic,
        "peak_source": "measured FFMA probe (alert_probe_fp32_peak) at the run's clocks" if peak else
                       "nominal 148 SM x 128 lanes x 1965 MHz",
        "peak_nominal_gslot_s": peak_nominal / 1e9,
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
                          chunk_steps=max(1, N // 10), engine=eng)
        if wl["stream_row"] is not None:  # shared traces: stream the gathered rows
            hs = None
        if hs is not None:
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
            ems = a.elapsed_time(b)
            ems = max_over_ranks(ems, dev)
            e2e = {"value": decisions / (ems * 1e-3), "unit": "decisions/s",
                   "h2d_bytes_per_step": hs.h2d_bytes, "d2h_bytes_per_step": hs.d2h_bytes,
                   "path": "paper_1911_00119_b200.simulator.HostStreamer (pinned host trace, chunked H2D "
                           "overlapped with alert_run, per-stream aggregates D2H)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(wl, "alert" if policy == "alert+oracle" else policy)

    lanes, tpb = eng.launch_config()
    if rank == 0:
        line = {
            "metric": metric, "value": value, "unit": "decisions/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "fp32 scan + fp64 re-rank/state",
            "data": "synthetic: reference preset contention traces realized with numpy (seed 42+stream)",
            "config": {"workload": args.config, "desc": desc, "streams_per_rank": S, "steps_per_stream": N,
                       "candidates": C, "policy": policy, "records": args.records,
                       "lanes_per_stream": lanes or (1 if C <= 256 else 8),
                       "threads_per_block": tpb if args.tpb else "auto (64; 256 when the staged table > 40 KB)",
                       "l2": "inputs larger than L2" if 4 * S * N > 126e6 else "inputs fit L2",
                       "parallelism": f"streams sharded, {world} rank(s)"},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": gpu_launches,
            "clocks": clocks, "quality": quality,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

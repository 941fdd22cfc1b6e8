"""Synthetic candidate tables and the preset contention trace (inputs).

Restates the reference generator (pkg/src/alertsim/synth.py:21-175) value for
value — the benchmark configurations of BASELINE.json are defined on its
tables (the 8x5 preset, 55 candidates; the 64x32 sweep table, 2,144
candidates) — so the GPU box can build them without the reference installed.
tests/test_host.py (test_generate_space_equals_reference) checks the tables against the
reference's own output.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .model import ConfigSpace, DnnKind, DnnProfile, PowerSetting, Stage, kind_of
from .trace import Constant, EnvironmentPhase, Gaussian, LogNormal, Trace


@dataclass(frozen=True)
class ProfileKnobs:  # synth.py:21-34
    n_dnns: int = 8
    n_powers: int = 5
    power_min: float = 10.0
    power_max: float = 50.0
    power_exponent: float = 0.8
    latency_min: float = 0.02
    latency_ratio: float = 18.0
    error_min: float = 0.03
    error_ratio: float = 7.8
    anytime_stages: int = 4
    num_classes: int = 10
    dominated_every: int = 3


def generate_space(knobs: ProfileKnobs | None = None, seed: int = 0) -> ConfigSpace:
    """Pareto-style family of DNN variants x power caps (synth.py:37-113).

    Latency is log-spaced over the family and scales as (p_max/p)^exponent
    over caps; error shrinks with latency; every ``dominated_every``-th DNN
    is pushed off the frontier by a seeded factor; the last DNN is a nested
    anytime network with geometrically spaced stage latencies."""
    k = knobs or ProfileKnobs()
    if k.n_dnns < 1 or k.n_powers < 1:
        raise ValueError("need at least one DNN and one power setting")
    if k.latency_ratio <= 1 or k.error_ratio <= 1:
        raise ValueError("latency_ratio and error_ratio must exceed 1")
    if not k.power_min < k.power_max:
        raise ValueError("power range is degenerate")
    rng = np.random.default_rng(seed)
    caps = np.linspace(k.power_min, k.power_max, k.n_powers)
    scale = (k.power_max / caps) ** k.power_exponent
    base = np.geomspace(k.latency_min, k.latency_min * k.latency_ratio, k.n_dnns)
    frac = np.linspace(1.0, 0.0, k.n_dnns) if k.n_dnns > 1 else np.array([0.0])
    errs = k.error_min * k.error_ratio**frac
    log_ratio = math.log(k.latency_ratio)

    def frontier_error(t: float) -> float:
        f = math.log(t / k.latency_min) / log_ratio
        return k.error_min * k.error_ratio ** (1.0 - min(max(f, 0.0), 1.0))

    q_backup = 1.0 / k.num_classes
    any_idx = k.n_dnns - 1 if k.anytime_stages >= 2 else None
    dnns = []
    for i in range(k.n_dnns):
        t0 = float(base[i])
        e = float(errs[i])
        if k.dominated_every > 0 and i % k.dominated_every == k.dominated_every - 1 and i != any_idx:
            e *= 1.0 + 0.3 * float(rng.uniform(0.5, 1.0))
        e = min(e, 0.9)
        if i == any_idx:
            stages = []
            for f in np.geomspace(0.25, 1.0, k.anytime_stages):
                tk = t0 * float(f)
                stages.append(
                    Stage(accuracy=1.0 - 1.05 * frontier_error(tk),
                          t_prof=tuple(float(tk * ps) for ps in scale))
                )
            dnns.append(DnnProfile(f"any-{i:02d}", DnnKind.ANYTIME, tuple(stages),
                                   min(q_backup, stages[0].accuracy)))
        else:
            st = Stage(accuracy=1.0 - e, t_prof=tuple(float(t0 * ps) for ps in scale))
            dnns.append(DnnProfile(f"dnn-{i:02d}", DnnKind.TRADITIONAL, (st,), q_backup))
    powers = tuple(PowerSetting(j, float(c)) for j, c in enumerate(caps))
    return ConfigSpace(dnns=tuple(dnns), powers=powers, p_idle_prof=4.0)


def reference_latency(space) -> float:
    """Deadline unit: mean profiled latency (over caps) of the slowest anytime
    DNN, else of the slowest DNN (synth.py:116-124)."""
    pool = [d for d in space.dnns if kind_of(d) is DnnKind.ANYTIME] or list(space.dnns)
    slowest = max(pool, key=lambda d: d.final_stage.t_prof[-1])
    t = slowest.final_stage.t_prof
    return sum(t) / len(t)


MEMORY_MEAN, MEMORY_SD = 1.8, 0.35  # synth.py:133
COMPUTE_MEAN, COMPUTE_SD = 1.3, 0.1  # synth.py:134


def memory_contention() -> LogNormal:
    v = math.log(1.0 + (MEMORY_SD / MEMORY_MEAN) ** 2)
    return LogNormal(mu_log=math.log(MEMORY_MEAN) - 0.5 * v, sd_log=math.sqrt(v))


def preset_space(seed: int = 0) -> ConfigSpace:
    return generate_space(ProfileKnobs(), seed=seed)


def preset_phases(lengths=(200, 200, 200), input_noise_sd: float = 0.05, order=(0, 1, 2)):
    """The three preset regimes (none / memory / compute contention,
    synth.py:148-175) with per-phase lengths and an optional phase order."""
    regimes = [
        (Constant(1.0), 4.0),
        (memory_contention(), 6.0),
        (Gaussian(COMPUTE_MEAN, COMPUTE_SD), 5.0),
    ]
    return tuple(
        EnvironmentPhase(length=int(n), slowdown_dist=regimes[r][0],
                         idle_power_true=regimes[r][1], input_noise_sd=input_noise_sd)
        for n, r in zip(lengths, order)
    )


def preset_trace(seed: int = 42, phase_length: int = 200, input_noise_sd: float = 0.05) -> Trace:
    return Trace(seed=seed, phases=preset_phases((phase_length,) * 3, input_noise_sd))


def _realize_block(args):
    from .trace import realize

    seeds, lengths, noise, order, dtype = args
    phases = preset_phases(lengths, noise, order)
    out = np.empty((sum(lengths), len(seeds)), dtype=dtype)
    for c, sd in enumerate(seeds):
        out[:, c] = realize(Trace(seed=int(sd), phases=phases)).slowdown
    return out


def preset_batch(n_streams: int, lengths=(3334, 3333, 3333), seed0: int = 42, input_noise_sd: float = 0.05,
                 order=(0, 1, 2), dtype=np.float32, processes: int | None = None):
    """Realized preset-contention traces for streams k = 0..n-1 with seeds
    seed0 + k (each column identical to realize(Trace(seed0 + k, ...))),
    packed time-major for the device.  Realization is spread over host
    processes; it is input preparation, not part of the timed hot path."""
    import multiprocessing as mp
    import os

    from .trace import PackedEnvs

    seeds = np.arange(seed0, seed0 + n_streams)
    procs = processes or min(os.cpu_count() or 1, 64)
    blocks = np.array_split(seeds, max(1, min(n_streams, procs * 4)))
    jobs = [(b, tuple(lengths), input_noise_sd, tuple(order), dtype) for b in blocks if len(b)]
    if procs > 1 and n_streams > 256:
        with mp.get_context("fork").Pool(procs) as pool:
            parts = pool.map(_realize_block, jobs)
    else:
        parts = [_realize_block(j) for j in jobs]
    slow = np.concatenate(parts, axis=1)
    regimes_idle = (4.0, 6.0, 5.0)
    nseg = len(lengths)
    ends = np.cumsum(lengths).astype(np.int32)
    return PackedEnvs(
        slowdown=slow,
        n_segments=np.full(n_streams, nseg, np.int32),
        seg_end=np.tile(ends, (n_streams, 1)),
        seg_phase=np.tile(np.arange(nseg, dtype=np.int32), (n_streams, 1)),
        seg_idle=np.tile(np.array([regimes_idle[r] for r in order], np.float64), (n_streams, 1)),
    )


def realize_on_device(phases, n_streams: int, seed: int = 42, stream_offset: int = 0, dtype=np.float32,
                      device: int = 0):
    """Traces for many streams generated ON THE GPU:
    the reference's per-phase recipe (simulator.py:221-235 — draw, optional
    N(1, input_noise_sd) jitter, floor at 0.01) with Philox4x32-10 streams
    keyed by (seed, stream index).  Returns a DeviceTrace (time-major, never
    copied to the host).  The values are NOT numpy's PCG64 draws: parity is
    distributional, and decisions are checked on exported arrays
    (``trace.slowdown.cpu()``) against the CPU oracle."""
    import ctypes as C

    import torch

    from . import abi
    from ._lib import check, load
    from .engine import DeviceTrace
    from .simulator import get_engine
    from .trace import Constant, Gaussian, LogNormal, Uniform

    eng = get_engine(device)
    descs = (abi.AlertPhaseDesc * len(phases))()
    for k, p in enumerate(phases):
        d = p.slowdown_dist
        if isinstance(d, Constant) or type(d).__name__ == "Constant":
            kind, a, b = abi.DIST_CONSTANT, d.value, 0.0
        elif type(d).__name__ == "Gaussian":
            kind, a, b = abi.DIST_GAUSSIAN, d.mean_, d.sd
        elif type(d).__name__ == "LogNormal":
            kind, a, b = abi.DIST_LOGNORMAL, d.mu_log, d.sd_log
        elif type(d).__name__ == "Uniform":
            kind, a, b = abi.DIST_UNIFORM, d.lo, d.hi
        else:
            raise ValueError(f"unknown slow-down distribution {d!r}")
        descs[k] = abi.AlertPhaseDesc(int(p.length), kind, 0, float(a), float(b), float(p.input_noise_sd))
    steps = sum(int(p.length) for p in phases)
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    out = torch.empty((steps, n_streams), dtype=tdt, device=eng.tdev)
    check(load().alert_realize(eng.ctx, descs, len(phases), int(seed), int(stream_offset), int(n_streams),
                               out.data_ptr(), abi.DTYPE_F64 if dtype == np.float64 else abi.DTYPE_F32,
                               eng._stream()))
    ends = np.cumsum([int(p.length) for p in phases]).astype(np.int32)
    d = eng.tdev
    nseg = len(phases)
    return DeviceTrace(
        slowdown=out,
        n_segments=torch.full((n_streams,), nseg, dtype=torch.int32, device=d),
        seg_end=torch.as_tensor(np.tile(ends, (n_streams, 1))).to(d),
        seg_phase=torch.as_tensor(np.tile(np.arange(nseg, dtype=np.int32), (n_streams, 1))).to(d),
        seg_idle=torch.as_tensor(np.tile(np.array([float(p.idle_power_true) for p in phases]), (n_streams, 1))).to(d),
    )

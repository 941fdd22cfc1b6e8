"""Synthetic candidate tables and the preset contention trace (inputs).

Restates the reference generator (pkg/src/alertsim/synth.py:21-175) value for
value — the benchmark configurations of BASELINE.json are defined on its
tables (the 8x5 preset, 55 candidates; the 64x32 sweep table, 2,144
candidates) — so the GPU box can build them without the reference installed.
tests/test_golden.py checks the tables against the reference's own output.
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

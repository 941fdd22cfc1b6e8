"""Synthetic environment traces: the INPUT stage of the scheduling step.

Mirrors the reference's trace model (pkg/src/alertsim/simulator.py:28-107,
210-235): contention phases with a slow-down distribution, a true idle power
and per-input multiplicative jitter, realized once per trace from a numpy
PCG64 seed.  ``realize`` draws in exactly the reference's order, so a trace
realizes to the same arrays here and there (for the same numpy version —
numpy does not promise Generator stream stability across versions, which is
why parity tests feed identical injected arrays to both sides).

Realization is not accelerated; the arrays it
produces are packed by :func:`pack_envs` into the device trace layout.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Sequence, Union

import numpy as np

from . import abi

MIN_SLOWDOWN = 0.01  # simulator.py:28


@dataclass(frozen=True)
class Constant:  # simulator.py:33-41
    value: float

    def draw(self, rng: np.random.Generator, n: int) -> np.ndarray:
        return np.full(n, self.value)

    def mean(self) -> float:
        return self.value


@dataclass(frozen=True)
class Gaussian:  # simulator.py:44-53
    mean_: float
    sd: float

    def draw(self, rng: np.random.Generator, n: int) -> np.ndarray:
        return rng.normal(self.mean_, self.sd, n)

    def mean(self) -> float:
        return self.mean_


@dataclass(frozen=True)
class LogNormal:  # simulator.py:56-65
    mu_log: float
    sd_log: float

    def draw(self, rng: np.random.Generator, n: int) -> np.ndarray:
        return rng.lognormal(self.mu_log, self.sd_log, n)

    def mean(self) -> float:
        return math.exp(self.mu_log + 0.5 * self.sd_log**2)


@dataclass(frozen=True)
class Uniform:  # simulator.py:68-77
    lo: float
    hi: float

    def draw(self, rng: np.random.Generator, n: int) -> np.ndarray:
        return rng.uniform(self.lo, self.hi, n)

    def mean(self) -> float:
        return 0.5 * (self.lo + self.hi)


SlowdownDist = Union[Constant, Gaussian, LogNormal, Uniform]


def lognormal_matching(mean: float, sd: float) -> LogNormal:
    """LogNormal with a Gaussian's mean and variance (simulator.py:83-88)."""
    if mean <= 0:
        raise ValueError("mean must be positive")
    v = math.log(1.0 + (sd / mean) ** 2)
    return LogNormal(mu_log=math.log(mean) - 0.5 * v, sd_log=math.sqrt(v))


@dataclass(frozen=True)
class EnvironmentPhase:  # simulator.py:91-96
    length: int
    slowdown_dist: SlowdownDist
    idle_power_true: float
    input_noise_sd: float = 0.0


@dataclass(frozen=True)
class Trace:  # simulator.py:99-107
    seed: int
    phases: tuple[EnvironmentPhase, ...]
    group_size: int | None = None

    @property
    def length(self) -> int:
        return sum(p.length for p in self.phases)


@dataclass(frozen=True)
class TrueEnvironment:  # simulator.py:212-218
    slowdown: np.ndarray
    idle_power: np.ndarray
    phase_index: np.ndarray


def realize(trace) -> TrueEnvironment:
    """Per-input ground truth from the trace seed (simulator.py:221-235)."""
    rng = np.random.default_rng(trace.seed)
    s_parts, idle_parts, ph_parts = [], [], []
    for k, ph in enumerate(trace.phases):
        s = ph.slowdown_dist.draw(rng, ph.length)
        if ph.input_noise_sd > 0:
            s = s * rng.normal(1.0, ph.input_noise_sd, ph.length)
        s_parts.append(np.maximum(s, MIN_SLOWDOWN))
        idle_parts.append(np.full(ph.length, ph.idle_power_true))
        ph_parts.append(np.full(ph.length, k, dtype=int))
    return TrueEnvironment(
        slowdown=np.concatenate(s_parts),
        idle_power=np.concatenate(idle_parts),
        phase_index=np.concatenate(ph_parts),
    )


# --- device trace layout -----------------------------------------------------

@dataclass
class PackedEnvs:
    """Host arrays in the AlertTrace layout (include/alert_b200.h).

    ``slowdown`` is time-major [n_steps][n_rows] so that, per step, the
    lanes of a warp read consecutive rows (one coalesced 128 B line per 32
    streams in FP32).  Segments are runs of constant (phase id, idle power).
    """

    slowdown: np.ndarray   # [n_steps, n_rows] float32 | float64
    n_segments: np.ndarray  # [n_rows] int32
    seg_end: np.ndarray     # [n_rows, max_seg] int32
    seg_phase: np.ndarray   # [n_rows, max_seg] int32
    seg_idle: np.ndarray    # [n_rows, max_seg] float64
    # goal changes (optional): per-row spec segments, see pack_goal_changes
    goal_n: np.ndarray | None = None     # [n_rows] int32 (0 = the stream's own spec)
    goal_end: np.ndarray | None = None   # [n_rows, max_goal] int32 exclusive end step
    goal_spec: np.ndarray | None = None  # [n_rows, max_goal] int32 index into the spec array

    @property
    def n_rows(self) -> int:
        return self.slowdown.shape[1]

    @property
    def n_steps(self) -> int:
        return self.slowdown.shape[0]


def segments_of(env) -> list[tuple[int, int, float]]:
    """(end, phase id, idle) runs of a TrueEnvironment."""
    idle = np.asarray(env.idle_power, dtype=np.float64)
    ph = np.asarray(env.phase_index)
    n = len(idle)
    cuts = np.flatnonzero((idle[1:] != idle[:-1]) | (ph[1:] != ph[:-1])) + 1
    ends = list(cuts) + [n]
    out, start = [], 0
    for e in ends:
        out.append((int(e), int(ph[start]), float(idle[start])))
        start = e
    return out


def pack_envs(envs: Sequence, dtype=np.float32, max_segments: int | None = None) -> PackedEnvs:
    """Stack realized environments (all the same length) into the device
    layout.  ``dtype=np.float64`` keeps the reference's exact slow-downs;
    float32 halves the input bytes (the parity harness then feeds the same
    float32-rounded values to the CPU oracle)."""
    if not envs:
        raise ValueError("need at least one environment")
    n = len(envs[0].slowdown)
    if any(len(e.slowdown) != n for e in envs):
        raise ValueError("all environments must have the same length")
    segs = [segments_of(e) for e in envs]
    ms = max_segments or max(len(s) for s in segs)
    rows = len(envs)
    slow = np.empty((n, rows), dtype=dtype)
    for r, e in enumerate(envs):
        slow[:, r] = np.asarray(e.slowdown, dtype=np.float64).astype(dtype)
    n_seg = np.zeros(rows, np.int32)
    seg_end = np.zeros((rows, ms), np.int32)
    seg_phase = np.zeros((rows, ms), np.int32)
    seg_idle = np.zeros((rows, ms), np.float64)
    for r, sg in enumerate(segs):
        if len(sg) > ms:
            raise ValueError(f"environment {r} has {len(sg)} segments > {ms}")
        bad = [ph for _, ph, _ in sg if not 0 <= ph < abi.MAX_PHASES]
        if bad:  # per-phase sums exist for phase ids < MAX_PHASES only (ALERT_AGG_PHASE_*)
            raise ValueError(f"environment {r}: phase index {bad[0]} outside 0..{abi.MAX_PHASES - 1}; "
                             f"traces with more than {abi.MAX_PHASES} phases are not supported")
        n_seg[r] = len(sg)
        for k, (end, ph, idle) in enumerate(sg):
            seg_end[r, k], seg_phase[r, k], seg_idle[r, k] = end, ph, idle
    return PackedEnvs(slow, n_seg, seg_end, seg_phase, seg_idle)


def pack_goal_changes(changes: Sequence, n_steps: int, n_specs: int):
    """Goal changes per trace row -> (goal_n, goal_end, goal_spec) arrays
    (AlertTrace.goal_*).  ``changes[r]`` is None (the stream's own spec) or a
    sequence of (start_step, spec_index) pairs with strictly increasing starts,
    the first at step 0: from start_step on, the row runs under
    specs[spec_index] (the reference's policy.spec swapped at that input,
    SURVEY §7 hard part 8)."""
    rows = len(changes)
    segs = []
    for r, ch in enumerate(changes):
        if ch is None or len(ch) == 0:
            segs.append([])
            continue
        ch = [(int(a), int(b)) for a, b in ch]
        if ch[0][0] != 0:
            raise ValueError(f"goal changes of row {r} must start at step 0")
        for (a, _), (b, _) in zip(ch, ch[1:]):
            if not a < b:
                raise ValueError(f"goal changes of row {r} must have increasing steps")
        if ch[-1][0] >= n_steps:
            raise ValueError(f"goal change of row {r} at step {ch[-1][0]} is past the trace ({n_steps} steps)")
        for _, k in ch:
            if not 0 <= k < n_specs:
                raise ValueError(f"goal change of row {r}: spec index {k} outside 0..{n_specs - 1}")
        segs.append([(ch[i + 1][0] if i + 1 < len(ch) else n_steps, k) for i, (_, k) in enumerate(ch)])
    mg = max(1, max(len(s) for s in segs))
    goal_n = np.zeros(rows, np.int32)
    goal_end = np.zeros((rows, mg), np.int32)
    goal_spec = np.zeros((rows, mg), np.int32)
    for r, sg in enumerate(segs):
        goal_n[r] = len(sg)
        for k, (end, si) in enumerate(sg):
            goal_end[r, k], goal_spec[r, k] = end, si
    return goal_n, goal_end, goal_spec


def goal_index_per_step(goal_n, goal_end, goal_spec, row: int, n_steps: int, default: int) -> np.ndarray:
    """Spec index in force at every step of one row (host view of the goal arrays)."""
    out = np.full(n_steps, default, np.int32)
    if goal_n is None or goal_n[row] == 0:
        return out
    start = 0
    for k in range(int(goal_n[row])):
        end = int(goal_end[row, k])
        out[start:end] = goal_spec[row, k]
        start = end
    return out


def unpack_row(p: PackedEnvs, row: int) -> TrueEnvironment:
    """Per-step arrays of one packed row, as the CPU oracle consumes them."""
    n = p.n_steps
    idle = np.empty(n, np.float64)
    ph = np.empty(n, np.int32)
    start = 0
    for k in range(int(p.n_segments[row])):
        end = int(p.seg_end[row, k])
        idle[start:end] = p.seg_idle[row, k]
        ph[start:end] = p.seg_phase[row, k]
        start = end
    return TrueEnvironment(p.slowdown[:, row].astype(np.float64), idle, ph)

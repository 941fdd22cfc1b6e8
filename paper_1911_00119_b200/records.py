"""Result types of the scheduling step, mirroring the reference's
(selector.py:20-41, predictor.py:36-45, simulator.py:304-458) so results read
the same way; ``summaries_from_agg`` turns the kernel's per-stream FP64
aggregate blocks (include/alert_b200.h, ALERT_AGG_*) into Summary objects."""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import abi
from .model import Mode, mode_of


class FallbackLevel(Enum):  # selector.py:20-23
    NONE = "none"
    DROPPED_ENERGY = "dropped-energy"
    DROPPED_ACCURACY = "dropped-accuracy"


LEVELS = (FallbackLevel.NONE, FallbackLevel.DROPPED_ENERGY, FallbackLevel.DROPPED_ACCURACY)


@dataclass(frozen=True)
class Prediction:  # predictor.py:36-45
    dnn_index: int
    power_index: int
    target_stage: int | None
    latency_mean: float
    latency_sigma: float
    pr_deadline: float
    expected_accuracy: float
    energy: float


@dataclass(frozen=True)
class ConfigDecision:  # selector.py:26-33
    dnn_index: int
    power_index: int
    target_stage: int | None
    prediction: Prediction | None
    feasible: bool
    fallback_level: FallbackLevel


@dataclass
class GroupState:  # selector.py:36-41
    remaining_budget: float
    remaining_count: int


@dataclass(frozen=True)
class ViolationFlags:  # simulator.py:304-308
    latency: bool
    accuracy: bool
    energy: bool


@dataclass(frozen=True)
class StepRecord:  # simulator.py:311-326
    input_index: int
    decision: ConfigDecision
    true_slowdown: float
    observed_latency: float
    completed_stage: int
    deadline_met: bool
    delivered_accuracy: float
    energy: float
    violations: ViolationFlags
    phase_index: int = 0
    period: float = 0.0
    fb_latency: float = 0.0
    fb_t_prof: float = 0.0
    idle_power_true: float = 0.0


@dataclass(frozen=True)
class PhaseSummary:  # simulator.py:399-404
    length: int
    mean_energy: float
    mean_accuracy: float
    violation_rates: dict


@dataclass(frozen=True)
class Summary:  # simulator.py:407-419
    n_inputs: int
    mean_energy: float
    mean_accuracy: float
    mean_error: float
    violation_rates: dict
    per_phase: tuple[PhaseSummary, ...]

    def objective(self, spec) -> float:
        return self.mean_energy if mode_of(spec) is Mode.MINIMIZE_ENERGY else self.mean_accuracy


@dataclass(frozen=True)
class RunResult:  # simulator.py:422-425
    records: tuple[StepRecord, ...]
    summary: Summary


def decision_of(cands: np.ndarray, cand: int, level: int, feasible: bool | None = None,
                prediction: Prediction | None = None) -> ConfigDecision:
    """ConfigDecision of candidate ``cand``; ``feasible`` defaults to level
    NONE (selector.py:126), the comparison schemes pass their own
    (policies.py:266-271, 305-310)."""
    i, j, st = (int(v) for v in cands[cand])
    return ConfigDecision(i, j, st if st else None, prediction, level == 0 if feasible is None else bool(feasible),
                          LEVELS[level])


def prediction_of(cands: np.ndarray, cand: int, p) -> Prediction:
    """Prediction of candidate ``cand`` from an AlertPrediction-like record
    (fields latency_mean, latency_sigma, pr_deadline, expected_accuracy, energy)."""
    i, j, st = (int(v) for v in cands[cand])
    return Prediction(i, j, st if st else None, float(p["latency_mean"]), float(p["latency_sigma"]),
                      float(p["pr_deadline"]), float(p["expected_accuracy"]), float(p["energy"]))


def summary_from_agg(agg: np.ndarray, n_phases: int = abi.MAX_PHASES) -> Summary:
    """One stream's aggregate block -> Summary (means are CPython 3.12 sum()
    results: Neumaier sum + compensation, divided by the count)."""
    n = agg[abi.AGG_N]

    def rates(block, base):
        m = block[base]
        return {"latency": block[base + 1] / m, "accuracy": block[base + 2] / m, "energy": block[base + 3] / m}

    per = []
    for k in range(min(n_phases, abi.MAX_PHASES)):
        b = abi.AGG_PHASE_BASE + abi.AGG_PHASE_STRIDE * k
        m = agg[b]
        if m <= 0:
            continue
        per.append(PhaseSummary(
            length=int(m),
            mean_energy=float(abi.neumaier_total(agg[b + 1], agg[b + 2]) / m),
            mean_accuracy=float(abi.neumaier_total(agg[b + 3], agg[b + 4]) / m),
            violation_rates={"latency": agg[b + 5] / m, "accuracy": agg[b + 6] / m, "energy": agg[b + 7] / m},
        ))
    mean_acc = float(abi.neumaier_total(agg[abi.AGG_ACC], agg[abi.AGG_ACC_C]) / n)
    return Summary(
        n_inputs=int(n),
        mean_energy=float(abi.neumaier_total(agg[abi.AGG_ENERGY], agg[abi.AGG_ENERGY_C]) / n),
        mean_accuracy=mean_acc,
        mean_error=1.0 - mean_acc,
        violation_rates={"latency": agg[abi.AGG_VIOL_LAT] / n, "accuracy": agg[abi.AGG_VIOL_ACC] / n,
                         "energy": agg[abi.AGG_VIOL_ENERGY] / n},
        per_phase=tuple(per),
    )

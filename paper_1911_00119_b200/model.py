"""Candidate-table and goal types of the scheduling step.

Host-side mirror of the reference's data model (reference
pkg/src/alertsim/model.py:17-176) with the same names, fields and validation
messages, so code written against ``alertsim.model`` works unchanged.  The GPU
path never touches these objects directly: :mod:`.packing` flattens them into
the C-ABI structs of ``include/alert_b200.h``.  Objects of the reference
package itself are accepted everywhere (duck typing on the field names).
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum


class DnnKind(str, Enum):  # model.py:17-19
    TRADITIONAL = "traditional"
    ANYTIME = "anytime"


class Mode(str, Enum):  # model.py:22-24
    MINIMIZE_ENERGY = "min-energy"
    MAXIMIZE_ACCURACY = "max-accuracy"


@dataclass(frozen=True)
class PowerSetting:  # model.py:27-32
    index: int
    cap_watts: float


@dataclass(frozen=True)
class Stage:  # model.py:35-40
    accuracy: float
    t_prof: tuple[float, ...]


@dataclass(frozen=True)
class DnnProfile:  # model.py:43-52
    id: str
    kind: DnnKind
    stages: tuple[Stage, ...]
    q_fail: float

    @property
    def final_stage(self) -> Stage:
        return self.stages[-1]


@dataclass(frozen=True)
class ConfigSpace:  # model.py:55-63
    dnns: tuple[DnnProfile, ...]
    powers: tuple[PowerSetting, ...]
    p_idle_prof: float

    @property
    def max_power(self) -> PowerSetting:
        return self.powers[-1]


@dataclass(frozen=True)
class ConstraintSpec:  # model.py:66-97
    mode: Mode
    t_goal: float
    e_goal: float | None = None
    q_goal: float | None = None
    pr_threshold: float | None = None
    overhead_budget: float = 0.0

    def __post_init__(self) -> None:
        check_spec(self)


def check_spec(spec) -> None:
    """The reference's ConstraintSpec invariants (model.py:81-97), usable on
    any object with the same fields (raises ValueError with its messages)."""
    mode = Mode(_enum_value(spec.mode))
    if spec.overhead_budget < 0:
        raise ValueError("overhead_budget must be >= 0")
    if spec.t_goal <= spec.overhead_budget:
        raise ValueError("t_goal must exceed overhead_budget")
    if mode is Mode.MAXIMIZE_ACCURACY:
        if spec.e_goal is None:
            raise ValueError("max-accuracy mode requires e_goal")
        if spec.e_goal <= 0:
            raise ValueError("e_goal must be positive")
    else:
        if spec.q_goal is None:
            raise ValueError("min-energy mode requires q_goal")
        if spec.q_goal <= 0:
            raise ValueError("q_goal must be positive")
    if spec.pr_threshold is not None and not 0.0 < spec.pr_threshold < 1.0:
        raise ValueError("pr_threshold must lie in (0, 1)")


def _enum_value(x):
    return x.value if isinstance(x, Enum) else x


def kind_of(dnn) -> DnnKind:
    """DnnKind of a profile from this package or from the reference."""
    return DnnKind(_enum_value(dnn.kind))


def mode_of(spec) -> Mode:
    return Mode(_enum_value(spec.mode))


def validate(space) -> list[str]:
    """Structural invariants of a config space (model.py:100-163): returns the
    list of human-readable problems, empty when the table is usable."""
    problems: list[str] = []
    powers, dnns = space.powers, space.dnns
    if not powers:
        problems.append("power axis is empty")
    if not dnns:
        problems.append("DNN axis is empty")
    if space.p_idle_prof <= 0:
        problems.append("p_idle_prof must be positive")
    last = 0.0
    for k, pw in enumerate(powers):
        if pw.cap_watts <= last:
            problems.append(f"power[{k}]: cap {pw.cap_watts} W not strictly above previous")
        last = pw.cap_watts
    n_powers = len(powers)
    for dnn in dnns:
        tag = f"dnn '{dnn.id}'"
        kind = kind_of(dnn)
        if kind is DnnKind.TRADITIONAL and len(dnn.stages) != 1:
            problems.append(f"{tag}: traditional profile must have exactly 1 stage")
        if kind is DnnKind.ANYTIME and len(dnn.stages) < 2:
            problems.append(f"{tag}: anytime profile needs >= 2 stages")
        if not 0.0 <= dnn.q_fail <= 1.0:
            problems.append(f"{tag}: q_fail {dnn.q_fail} outside [0,1]")
        if dnn.stages and dnn.q_fail > dnn.stages[0].accuracy:
            problems.append(f"{tag}: q_fail exceeds first-stage accuracy")
        prev_acc = -1.0
        for s, stage in enumerate(dnn.stages):
            stag = f"{tag} stage {s}"
            if not 0.0 <= stage.accuracy <= 1.0:
                problems.append(f"{stag}: accuracy {stage.accuracy} outside [0,1]")
            if kind is DnnKind.ANYTIME and stage.accuracy <= prev_acc:
                problems.append(f"{stag}: accuracies not increasing")
            prev_acc = stage.accuracy
            if len(stage.t_prof) != n_powers:
                problems.append(
                    f"{stag}: latency vector length {len(stage.t_prof)} != {n_powers} power settings"
                )
                continue
            for j, t in enumerate(stage.t_prof):
                if t <= 0:
                    problems.append(f"{stag}: latency at power {j} not positive")
                if j > 0 and t > stage.t_prof[j - 1]:
                    problems.append(f"{stag}: latency increases from power {j - 1} to {j}")
            if kind is DnnKind.ANYTIME and s > 0:
                prev = dnn.stages[s - 1]
                if len(prev.t_prof) == n_powers and any(
                    stage.t_prof[j] <= prev.t_prof[j] for j in range(n_powers)
                ):
                    problems.append(f"{stag}: latencies not strictly above stage {s - 1}")
    return problems


def fastest_dnn(space, power_index: int, kind: DnnKind | None = None):
    """Minimal final-stage latency at a power index; ties to the lower id
    (model.py:166-176)."""
    pool = [d for d in space.dnns if kind is None or kind_of(d) is kind]
    if not pool:
        raise ValueError(f"no DNN of kind {kind} in the space")
    return min(pool, key=lambda d: (d.final_stage.t_prof[power_index], d.id))

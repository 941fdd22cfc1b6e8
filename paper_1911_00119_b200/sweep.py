"""Batched GPU goal sweep: the reference's ``cmd_sweep`` grid (cli.py:191-274)
as one fused launch per policy.

For every (deadline multiplier, goal) pair the reference builds a
ConstraintSpec (cli.py:216-234), runs oracle-static first as the
normalisation baseline (cli.py:235-236) and then every requested policy
(cli.py:237-257), one ``simulator.run`` at a time.  Here the whole grid is a
batch: one stream per grid point, all reading the same realized trace
(``stream_row`` = 0), one ``run_batch`` launch per policy.  Rows and the CSV
schema (cli.py:259-273, ``repr`` floats cli.py:106-107) are identical.

    rows = sweep(space, trace, "min-energy", [0.4, 0.8], [0.7, 0.85], ["alert", "oracle"])
    write_csv("sweep.csv", rows, "min-energy")

or ``python -m paper_1911_00119_b200.sweep --mode min-energy --q-goals 0.7,0.85``
(preset profile and trace; ``--seed`` re-seeds the trace like cli.py:49-57).
"""

from __future__ import annotations

import argparse
import csv
import hashlib
from dataclasses import replace
from pathlib import Path
from typing import Sequence

import numpy as np

from .model import ConstraintSpec, Mode
from .policies import POLICY_NAMES
from .simulator import run_batch
from .synth import preset_space, preset_trace, reference_latency
from .trace import realize

HEADER_TAIL = ["policy", "mean_objective", "normalized_to_oracle_static", "viol_latency_rate",
               "viol_accuracy_rate", "viol_energy_rate"]


def _fmt(x: float) -> str:  # cli.py:106-107
    return repr(float(x))


def stable_seed(top_seed: int, trace_seed: int) -> int:  # cli.py:49-51
    digest = hashlib.sha256(f"{top_seed}:{trace_seed}".encode()).digest()
    return int.from_bytes(digest[:8], "big") % (2**63)


def effective_trace(trace, top_seed: int | None):  # cli.py:54-57
    return trace if top_seed is None else replace(trace, seed=stable_seed(top_seed, trace.seed))


def grid_specs(space, mode: Mode, deadline_mults: Sequence[float], goals: Sequence[float],
               pr_th: float | None = None) -> list[ConstraintSpec]:
    """cli.py:216-234, in the reference's loop order (deadline outer, goal inner)."""
    ref = reference_latency(space)
    specs = []
    for dm in deadline_mults:
        t_goal = dm * ref
        for g in goals:
            if mode is Mode.MINIMIZE_ENERGY:
                specs.append(ConstraintSpec(mode=mode, t_goal=t_goal, q_goal=g, pr_threshold=pr_th,
                                            overhead_budget=0.01 * ref))
            else:
                specs.append(ConstraintSpec(mode=mode, t_goal=t_goal, e_goal=g * space.max_power.cap_watts * t_goal,
                                            pr_threshold=pr_th, overhead_budget=0.01 * ref))
    return specs


def sweep(space, trace, mode, deadline_mults: Sequence[float], goals: Sequence[float],
          policies: Sequence[str] = ("alert", "oracle", "oracle-static"), *, pr_th: float | None = None,
          kalman=None, device: int = 0) -> list[list[str]]:
    """The rows cmd_sweep writes (cli.py:246-257), computed with one batched
    GPU launch per policy over every grid point."""
    mode = Mode(mode)
    for p in policies:
        if p not in POLICY_NAMES:
            raise ValueError(f"unknown policy {p!r}")
    specs = grid_specs(space, mode, deadline_mults, goals, pr_th)
    env = realize(trace)
    n = len(specs)
    summaries = {}
    for name in dict.fromkeys(["oracle-static", *policies]):
        res = run_batch(space, specs, [env], name, kalman=None if name == "oracle-static" else kalman,
                        group_sizes=trace.group_size, stream_row=[0] * n, stream_spec=list(range(n)),
                        n_streams=n, trace_dtype=np.float64, device=device)
        summaries[name] = res.summaries()
    return sweep_rows(deadline_mults, goals, specs, policies, summaries)


def sweep_rows(deadline_mults, goals, specs, policies, summaries) -> list[list[str]]:
    """cli.py:244-257 from per-grid-point Summaries (summaries[policy][k],
    k in grid order); oracle-static is the normalisation baseline."""
    rows = []
    k = 0
    for dm in deadline_mults:
        for g in goals:
            spec = specs[k]
            baseline = summaries["oracle-static"][k].objective(spec)
            for name in policies:
                s = summaries[name][k]
                obj = s.objective(spec)
                norm = obj / baseline if baseline else float("nan")
                rows.append([_fmt(dm), _fmt(g), name, _fmt(obj), _fmt(norm), _fmt(s.violation_rates["latency"]),
                             _fmt(s.violation_rates["accuracy"]), _fmt(s.violation_rates["energy"])])
            k += 1
    return rows


def write_csv(path, rows, mode) -> None:
    """cli.py:259-273."""
    mode = Mode(mode)
    out = Path(path)
    out.parent.mkdir(parents=True, exist_ok=True)
    with out.open("w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["deadline_mult", "q_goal" if mode is Mode.MINIMIZE_ENERGY else "e_goal_mult", *HEADER_TAIL])
        w.writerows(rows)


def _floats(text: str, what: str) -> list[float]:  # cli.py:181-188
    vals = [float(v) for v in text.split(",") if v.strip()]
    if not vals:
        raise ValueError(f"empty {what} grid")
    return vals


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description="GPU goal sweep (cmd_sweep, cli.py:191-274) on the preset profile")
    ap.add_argument("--mode", choices=[m.value for m in Mode], default="min-energy")
    ap.add_argument("--deadline-mults", default="0.4,0.8,1.2,1.6,2.0")
    ap.add_argument("--q-goals", default=None)
    ap.add_argument("--e-goal-mults", default=None)
    ap.add_argument("--policies", default="alert,oracle,oracle-static")
    ap.add_argument("--pr-th", type=float, default=None)
    ap.add_argument("--seed", type=int, default=None)
    ap.add_argument("--phase-length", type=int, default=200)
    ap.add_argument("--out", required=True)
    a = ap.parse_args(argv)
    mode = Mode(a.mode)
    goals_txt = a.q_goals if mode is Mode.MINIMIZE_ENERGY else a.e_goal_mults
    if goals_txt is None:
        ap.error("min-energy sweep requires --q-goals" if mode is Mode.MINIMIZE_ENERGY
                 else "max-accuracy sweep requires --e-goal-mults")
    rows = sweep(preset_space(), effective_trace(preset_trace(phase_length=a.phase_length), a.seed), mode,
                 _floats(a.deadline_mults, "deadline-mult"), _floats(goals_txt, "goal"),
                 [p.strip() for p in a.policies.split(",") if p.strip()], pr_th=a.pr_th)
    write_csv(a.out, rows, mode)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())

"""Shared test helpers: rebuild golden cases, random instances, comparisons."""

from __future__ import annotations

import json
import random
from pathlib import Path

import numpy as np

from paper_1911_00119_b200.estimator import KalmanConfig
from paper_1911_00119_b200.model import (
    ConfigSpace, ConstraintSpec, DnnKind, DnnProfile, Mode, PowerSetting, Stage,
)
from paper_1911_00119_b200.trace import TrueEnvironment

GOLDEN = Path(__file__).resolve().parent / "golden"


def space_from_dict(doc) -> ConfigSpace:
    powers = tuple(PowerSetting(j, float(w)) for j, w in enumerate(doc["powers"]))
    dnns = tuple(
        DnnProfile(d["id"], DnnKind(d["kind"]),
                   tuple(Stage(float(s["accuracy"]), tuple(float(t) for t in s["t_prof"])) for s in d["stages"]),
                   float(d["q_fail"]))
        for d in doc["dnns"]
    )
    return ConfigSpace(dnns, powers, float(doc["p_idle_prof"]))


def spec_from_json(d) -> ConstraintSpec:
    return ConstraintSpec(mode=Mode(d["mode"]), t_goal=d["t_goal"], e_goal=d["e_goal"], q_goal=d["q_goal"],
                          pr_threshold=d["pr_threshold"], overhead_budget=d["overhead_budget"])


def kalman_from_json(d):
    return None if d is None else KalmanConfig(**d)


class GoldenCase:
    def __init__(self, meta, z):
        self.name = meta["name"]
        self.meta = meta
        self.space = space_from_dict(meta["space"])
        self.spec = spec_from_json(meta["spec"])
        self.group_size = meta["spec"]["group_size"]
        self.policy = meta["policy"]
        self.kalman = kalman_from_json(meta["kalman"])
        self.n_phases = meta["n_phases"]
        # goal changes (golden_goals.npz): [(input_index, ConstraintSpec), ...]
        self.changes = [(int(n), spec_from_json(d)) for n, d in meta.get("changes", [])] or None
        self.z = {k.split("/", 1)[1]: z[k] for k in z.files if k.startswith(self.name + "/")}

    @property
    def env(self):
        return TrueEnvironment(self.z["s"], self.z["idle"], self.z["phase"])


def load_golden_runs(name: str = "golden_runs.npz"):
    z = np.load(GOLDEN / name)
    meta = json.loads(bytes(z["meta"]).decode())
    return [GoldenCase(m, z) for m in meta]


def load_golden_predict():
    z = np.load(GOLDEN / "golden_predict.npz")
    meta = json.loads(bytes(z["meta"]).decode())
    out = []
    for k, m in enumerate(meta):
        out.append(dict(space=space_from_dict(m["space"]), spec=spec_from_json(m["spec"]), mu=m["mu"],
                        sigma2=m["sigma2"], phi=m["phi"], goal=m["goal"], z_q=m["z_q"],
                        pred=z[f"{k}/pred"], sel=z[f"{k}/sel"]))
    return out


def random_space(rnd: random.Random, max_dnns=4, max_powers=4) -> ConfigSpace:
    """Same family as the reference's conftest.random_space (conftest.py:20-58)."""
    n_powers = rnd.randint(1, max_powers)
    caps = sorted(rnd.uniform(5.0, 100.0) for _ in range(n_powers))
    powers = tuple(PowerSetting(i, c) for i, c in enumerate(caps))
    scale = [caps[-1] / c for c in caps]
    dnns = []
    for i in range(rnd.randint(1, max_dnns)):
        base = rnd.uniform(0.01, 1.0)
        if rnd.random() < 0.4:
            n_st = rnd.randint(2, 4)
            accs = sorted(rnd.uniform(0.2, 0.99) for _ in range(n_st))
            lats = sorted(base * rnd.uniform(0.3, 3.0) for _ in range(n_st))
            stages = tuple(Stage(a, tuple(t * s for s in scale)) for a, t in zip(accs, lats))
            dnns.append(DnnProfile(f"any-{i}", DnnKind.ANYTIME, stages, rnd.uniform(0.0, accs[0])))
        else:
            acc = rnd.uniform(0.2, 0.99)
            dnns.append(DnnProfile(f"dnn-{i}", DnnKind.TRADITIONAL,
                                   (Stage(acc, tuple(base * s for s in scale)),), rnd.uniform(0.0, acc)))
    return ConfigSpace(tuple(dnns), powers, rnd.uniform(1.0, 10.0))


def random_spec(rnd: random.Random) -> ConstraintSpec:
    """Same family as the reference's conftest.random_spec (conftest.py:61-71)."""
    mode = rnd.choice([Mode.MINIMIZE_ENERGY, Mode.MAXIMIZE_ACCURACY])
    pr = rnd.choice([None, rnd.uniform(0.05, 0.99)])
    t = rnd.uniform(0.05, 3.0)
    if mode is Mode.MINIMIZE_ENERGY:
        return ConstraintSpec(mode=mode, t_goal=t, q_goal=rnd.uniform(0.1, 0.99), pr_threshold=pr)
    return ConstraintSpec(mode=mode, t_goal=t, e_goal=rnd.uniform(0.5, 80.0), pr_threshold=pr)

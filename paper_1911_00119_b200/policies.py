"""GPU-backed scheduling policies with the reference's Policy protocol
(simulator.py:387-396: ``begin / decide / observe``) and registry
(policies.py:457-490).

Each object works two ways:
  * inside :func:`paper_1911_00119_b200.run` the whole trace runs in one
    fused kernel launch (the fast path);
  * driven step by step — including by the REFERENCE's own
    ``alertsim.simulator.run`` — ``decide`` / ``observe`` launch the per-step
    kernels (alert_decide / alert_oracle_decide / alert_observe).  API-
    compatible, launch-latency bound.
"""

from __future__ import annotations

import numpy as np

from . import abi
from .estimator import (
    IdleFilterConfig, IdlePowerEstimate, KalmanConfig, SlowdownEstimate,
)
from .model import DnnKind, kind_of
from .packing import pack_specs
from .records import decision_of, prediction_of

POLICY_NAMES = ("alert", "alert-any", "alert-trad", "oracle", "oracle-static", "sys-only", "app-only",
                "no-coord")


class GpuPolicy:
    name = "gpu"
    code_name = "alert"
    kalman: KalmanConfig | None = None
    device = 0

    def _engine(self):
        from .simulator import get_engine

        return get_engine(self.device)

    def _finish(self, res) -> None:  # state after a fused run
        pass

    def _prediction(self, cand: int, t_goal: float, spec_arr=None, acc_cand: int | None = None, **override):
        """Prediction of one candidate at the current filter state
        (alert_predict, predictor.py:147-197); ``override`` replaces fields
        the way the comparison schemes build theirs (policies.py:314-428)."""
        import torch

        eng = self._engine()
        g = torch.tensor([float(t_goal)], dtype=torch.float64, device=eng.tdev)
        raw = eng.predict(self._table, self._specs if spec_arr is None else spec_arr, self._state, g)
        preds = raw[0].cpu().numpy().view(abi.PREDICTION_DTYPE).reshape(-1)
        p = dict(zip(preds.dtype.names, preds[cand].tolist()))
        if acc_cand is not None:
            p["expected_accuracy"] = float(preds[acc_cand]["expected_accuracy"])
        p.update(override)
        return prediction_of(self._table.candidates, cand, p)


class AlertPolicy(GpuPolicy):
    """Coordinated selection from the shared slow-down / idle-power filters
    (policies.py:70-108), evaluated on the GPU.  The DNN-kind filter comes
    from ``kinds`` (policies.py:99-102) whatever the ``name`` label is."""

    def __init__(self, kalman: KalmanConfig | None = None, idle_cfg: IdleFilterConfig | None = None,
                 kinds: frozenset | None = None, name: str = "alert", device: int = 0):
        self.kalman = kalman
        self.idle_cfg = idle_cfg
        self.kinds = kinds
        self.name = name
        self.code_name = _kinds_code(kinds)
        self.device = device

    def begin(self, space, spec, env) -> None:
        if self.kinds is not None and not any(kind_of(d) in self.kinds for d in space.dnns):
            raise ValueError(f"{self.name}: space has no DNN of kinds {self.kinds}")
        import torch

        eng = self._engine()
        self.space = space
        self.spec = spec
        self._table = eng.table(space)
        self._specs = pack_specs([spec])
        self._state = eng.new_state(self._table, 1, self.kalman, self.idle_cfg)
        self._goal = torch.empty(1, dtype=torch.float64, device=eng.tdev)

    # per-step path ------------------------------------------------------------
    def decide(self, index: int, t_goal: float):
        import torch

        eng = self._engine()
        self._specs = pack_specs([self.spec])  # policy.spec may be swapped between inputs (goal changes)
        self._goal.fill_(float(t_goal))
        code = {"alert": abi.POLICY_ALERT, "alert-any": abi.POLICY_ALERT_ANY,
                "alert-trad": abi.POLICY_ALERT_TRAD}[self.code_name]
        w = int(eng.decide(self._table, self._specs, self._state, self._goal, policy=code)[0].item())
        w &= 0xFFFFFFFF
        c = w & 0xFFFF
        return decision_of(self._table.candidates, c, (w >> 16) & 3, prediction=self._prediction(c, t_goal))

    def observe(self, record) -> None:
        import torch

        eng = self._engine()
        d = eng.tdev
        f64 = torch.float64
        eng.observe(self._table, self._state,
                    torch.tensor([float(record.fb_latency)], dtype=f64, device=d),
                    torch.tensor([float(record.fb_t_prof)], dtype=f64, device=d),
                    torch.tensor([float(record.idle_power_true)], dtype=f64, device=d),
                    torch.tensor([int(record.decision.power_index)], dtype=torch.int32, device=d),
                    kalman=self.kalman, idle_cfg=self.idle_cfg)

    # state views (estimator types) ----------------------------------------------
    @property
    def est(self) -> SlowdownEstimate:
        st = {k: float(v[0].item()) for k, v in self._state.items() if k in ("mu", "sigma2", "k_gain",
                                                                           "q_noise", "innov")}
        return SlowdownEstimate(st["mu"], st["sigma2"], st["k_gain"], st["q_noise"], st["innov"],
                                self.kalman or KalmanConfig())

    @property
    def idle(self) -> IdlePowerEstimate:
        return IdlePowerEstimate(float(self._state["phi"][0].item()), float(self._state["m_var"][0].item()),
                                 self.idle_cfg or IdleFilterConfig())

    def _finish(self, res) -> None:
        import torch

        for k, v in res.state.items():
            self._state[k].copy_(torch.as_tensor(np.asarray(v)))


class OraclePolicy(GpuPolicy):
    """Clairvoyant per-input optimum over the realized trace
    (policies.py:149-208), evaluated on the GPU."""

    name = "oracle"
    code_name = "oracle"

    def __init__(self, device: int = 0):
        self.device = device

    def begin(self, space, spec, env) -> None:
        import torch

        eng = self._engine()
        self.space = space
        self.spec = spec
        self.env = env
        self._table = eng.table(space)
        self._specs = pack_specs([spec])
        d = eng.tdev
        self._s = torch.as_tensor(np.asarray(env.slowdown, np.float64)).to(d)
        self._idle = torch.as_tensor(np.asarray(env.idle_power, np.float64)).to(d)
        self._goal = torch.empty(1, dtype=torch.float64, device=d)

    def decide(self, index: int, t_goal: float):
        eng = self._engine()
        self._specs = pack_specs([self.spec])  # policy.spec may be swapped between inputs (goal changes)
        self._goal.fill_(float(t_goal))
        w, ex = eng.oracle_decide(self._table, self._specs, self._s[index:index + 1],
                                  self._idle[index:index + 1], self._goal, exact=True)
        w = int(w[0].item()) & 0xFFFFFFFF
        c = w & 0xFFFF
        p = ex[0].cpu().numpy().view(abi.PREDICTION_DTYPE)[0]
        return decision_of(self._table.candidates, c, (w >> 16) & 3, prediction=prediction_of(self._table.candidates, c, p))

    def observe(self, record) -> None:
        pass


class BaselinePolicy(GpuPolicy):
    """The reference's comparison schemes (policies.py:211-454) on the GPU:
    oracle-static (best fixed candidate over the realized trace), sys-only
    (fastest traditional DNN, cheapest on-time power cap), app-only (one
    anytime DNN at the maximum cap, best expected-accuracy stage), no-coord
    (both controllers, uncoordinated).  Inside :func:`paper_1911_00119_b200.run`
    / ``run_batch`` a whole trace runs in one launch (FP64, the reference's
    operation order); driven step by step, ``begin`` / ``decide`` /
    ``observe`` launch alert_static_choice / alert_baseline_decide /
    alert_observe."""

    def __init__(self, name: str, kalman: KalmanConfig | None = None, device: int = 0):
        self.name = name
        self.code_name = name
        self.kalman = kalman
        self.device = device

    def begin(self, space, spec, env) -> None:
        import torch

        from .packing import baseline_dnns, policy_code
        from .trace import pack_envs

        sys_dnn, app_dnn = baseline_dnns(space)
        if self.name == "sys-only" and sys_dnn < 0:
            raise ValueError("no DNN of kind DnnKind.TRADITIONAL in the space")  # model.py:172-173
        if self.name in ("app-only", "no-coord") and app_dnn < 0:
            raise ValueError("space has no anytime DNN")  # policies.py:327-328
        self.space, self.spec, self.env = space, spec, env
        eng = self._engine()
        self._code = policy_code(self.name)
        self._table = eng.table(space)
        self._specs = pack_specs([spec])
        # sys-only / no-coord keep their own idle filter with the default config (policies.py:295, 388)
        self._state = eng.new_state(self._table, 1, self.kalman, None)
        self._goal = torch.empty(1, dtype=torch.float64, device=eng.tdev)
        self._last_power = len(space.powers) - 1  # no-coord's initial power (policies.py:385)
        if self.name == "oracle-static":  # OracleStaticPolicy.begin (policies.py:221-265)
            tr = eng.upload_trace(pack_envs([env], dtype=np.float64))
            eng.static_choice(self._table, self._specs, tr, self._state)

    def decide(self, index: int, t_goal: float):
        eng = self._engine()
        self._goal.fill_(float(t_goal))
        w = int(eng.baseline_decide(self._table, self._specs, self._state, self._goal,
                                    policy=self._code)[0].item()) & 0xFFFFFFFF
        c, feasible = w & 0xFFFF, bool((w >> 30) & 1)
        cands = self._table.candidates
        if self.name == "oracle-static":
            pred = prediction_of(cands, c, {"latency_mean": 0.0, "latency_sigma": 0.0,
                                            "pr_deadline": 1.0 if feasible else 0.0,
                                            "expected_accuracy": 0.0, "energy": 0.0})
        elif self.name == "sys-only":
            sp = np.array(self._specs, copy=True)
            sp["has_pr"] = 0  # predict_energy_mean (policies.py:309, 320)
            acc = float(self.space.dnns[int(cands[c, 0])].stages[0].accuracy)
            pred = self._prediction(c, t_goal, sp, pr_deadline=1.0 if feasible else 0.0, expected_accuracy=acc)
        else:
            acc_c = c
            if self.name == "no-coord":  # expected accuracy at the previous power (policies.py:399-405)
                i, _, st = (int(v) for v in cands[c])
                acc_c = int(np.flatnonzero((cands[:, 0] == i) & (cands[:, 1] == self._last_power)
                                           & (cands[:, 2] == st))[0])
            pred = self._prediction(c, t_goal, acc_cand=acc_c, pr_deadline=0.0, energy=0.0)
        self._last_power = int(cands[c, 1])
        return decision_of(cands, c, 0, feasible, pred)

    def observe(self, record) -> None:
        import torch

        if self.name == "oracle-static":  # policies.py:271-272
            return
        eng = self._engine()
        d = eng.tdev
        f64 = torch.float64
        # app-only updates only the slow-down filter (policies.py:359-360); its
        # idle estimate is never read, so updating it too changes nothing
        eng.observe(self._table, self._state,
                    torch.tensor([float(record.fb_latency)], dtype=f64, device=d),
                    torch.tensor([float(record.fb_t_prof)], dtype=f64, device=d),
                    torch.tensor([float(record.idle_power_true)], dtype=f64, device=d),
                    torch.tensor([int(record.decision.power_index)], dtype=torch.int32, device=d),
                    kalman=self.kalman)

    def _finish(self, res) -> None:
        import torch

        for k, v in res.state.items():
            if k in self._state:
                self._state[k].copy_(torch.as_tensor(np.asarray(v)))


def _kinds_code(kinds) -> str:
    """Policy code of an AlertPolicy's DNN-kind filter (policies.py:99-102)."""
    if kinds is None:
        return "alert"
    k = frozenset(kinds)
    if k == frozenset({DnnKind.ANYTIME}):
        return "alert-any"
    if k == frozenset({DnnKind.TRADITIONAL}):
        return "alert-trad"
    if k == frozenset({DnnKind.ANYTIME, DnnKind.TRADITIONAL}):
        return "alert"
    raise ValueError(f"unsupported DNN kinds filter {set(kinds)}")


def make_policy(name: str, kalman: KalmanConfig | None = None, device: int = 0):
    """Registry with the reference's names (policies.py:469-490)."""
    if name == "alert":
        return AlertPolicy(kalman=kalman, device=device)
    if name == "alert-any":
        return AlertPolicy(kalman=kalman, kinds=frozenset({DnnKind.ANYTIME}), name="alert-any", device=device)
    if name == "alert-trad":
        return AlertPolicy(kalman=kalman, kinds=frozenset({DnnKind.TRADITIONAL}), name="alert-trad",
                           device=device)
    if name == "oracle":
        return OraclePolicy(device=device)
    if name in ("oracle-static", "sys-only", "app-only", "no-coord"):
        return BaselinePolicy(name, kalman=kalman, device=device)
    raise ValueError(f"unknown policy {name!r}; choose from {POLICY_NAMES}")

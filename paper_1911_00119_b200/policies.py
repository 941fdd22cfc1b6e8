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
from .records import decision_of

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


class AlertPolicy(GpuPolicy):
    """Coordinated selection from the shared slow-down / idle-power filters
    (policies.py:70-108), evaluated on the GPU."""

    def __init__(self, kalman: KalmanConfig | None = None, idle_cfg: IdleFilterConfig | None = None,
                 kinds: frozenset | None = None, name: str = "alert", device: int = 0):
        self.kalman = kalman
        self.idle_cfg = idle_cfg
        self.kinds = kinds
        self.name = name
        self.code_name = name
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
        self._goal.fill_(float(t_goal))
        code = {"alert": abi.POLICY_ALERT, "alert-any": abi.POLICY_ALERT_ANY,
                "alert-trad": abi.POLICY_ALERT_TRAD}[self.name]
        w = int(eng.decide(self._table, self._specs, self._state, self._goal, policy=code)[0].item())
        w &= 0xFFFFFFFF
        return decision_of(self._table.candidates, w & 0xFFFF, (w >> 16) & 3)

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
        self._goal.fill_(float(t_goal))
        w = int(eng.oracle_decide(self._table, self._specs, self._s[index:index + 1],
                                  self._idle[index:index + 1], self._goal)[0].item()) & 0xFFFFFFFF
        return decision_of(self._table.candidates, w & 0xFFFF, (w >> 16) & 3)

    def observe(self, record) -> None:
        pass


class BaselinePolicy(GpuPolicy):
    """The reference's comparison schemes (policies.py:211-454) on the GPU:
    oracle-static (best fixed candidate over the realized trace), sys-only
    (fastest traditional DNN, cheapest on-time power cap), app-only (one
    anytime DNN at the maximum cap, best expected-accuracy stage), no-coord
    (both controllers, uncoordinated).  They run through the fused path
    (:func:`paper_1911_00119_b200.run` / ``run_batch``: one launch per
    trace, FP64 with the reference's operation order)."""

    def __init__(self, name: str, kalman: KalmanConfig | None = None, device: int = 0):
        self.name = name
        self.code_name = name
        self.kalman = kalman
        self.device = device

    def begin(self, space, spec, env) -> None:
        from .packing import baseline_dnns

        sys_dnn, app_dnn = baseline_dnns(space)
        if self.name == "sys-only" and sys_dnn < 0:
            raise ValueError("no DNN of kind DnnKind.TRADITIONAL in the space")  # model.py:172-173
        if self.name in ("app-only", "no-coord") and app_dnn < 0:
            raise ValueError("space has no anytime DNN")  # policies.py:327-328
        self.space, self.spec, self.env = space, spec, env

    def decide(self, index: int, t_goal: float):
        raise NotImplementedError(f"{self.name}: the comparison schemes run fused over a whole trace "
                                  "(paper_1911_00119_b200.run / run_batch), not step by step")

    def observe(self, record) -> None:
        raise NotImplementedError(f"{self.name}: use paper_1911_00119_b200.run / run_batch")


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

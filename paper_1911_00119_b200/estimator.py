"""Filter configuration and state types of the scheduling step.

Same names and fields as the reference (pkg/src/alertsim/estimator.py:18-127).
The update arithmetic itself runs on the GPU (``alert_observe`` for single
steps, fused into ``alert_run`` for whole traces); these classes only carry
constants and state across the Python API.
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class KalmanConfig:  # estimator.py:18-30
    k0: float = 0.5
    r: float = 0.001
    q0: float = 0.1
    alpha: float = 0.3
    mu0: float = 1.0
    sigma2_0: float = 0.1
    sigma2_uses_current_gain: bool = False


@dataclass(frozen=True)
class SlowdownEstimate:  # estimator.py:33-44
    mu: float
    sigma2: float
    k_gain: float
    q_noise: float
    last_innovation: float
    config: KalmanConfig

    @property
    def sigma(self) -> float:
        return self.sigma2**0.5


@dataclass(frozen=True)
class IdleFilterConfig:  # estimator.py:87-91
    m0: float = 0.01
    s: float = 0.0001
    v: float = 0.001


@dataclass(frozen=True)
class IdlePowerEstimate:  # estimator.py:94-98
    phi: float
    m_var: float
    config: IdleFilterConfig


def slowdown_init(config: KalmanConfig | None = None) -> SlowdownEstimate:
    """Initial slow-down state (estimator.py:47-56)."""
    cfg = config or KalmanConfig()
    return SlowdownEstimate(cfg.mu0, cfg.sigma2_0, cfg.k0, cfg.q0, 0.0, cfg)


def idle_power_init(phi0: float, config: IdleFilterConfig | None = None) -> IdlePowerEstimate:
    """Initial idle-power state (estimator.py:101-107)."""
    cfg = config or IdleFilterConfig()
    if not 0.0 <= phi0 <= 1.0:
        raise ValueError("phi0 must lie in [0, 1]")
    return IdlePowerEstimate(phi0, cfg.m0, cfg)

"""B200-native ALERT scheduling step (arXiv 1911.00119), batched over streams.

Drop-in host API with the reference's names (alertsim): build a candidate
table (ConfigSpace) and goals (ConstraintSpec), pick a policy with
make_policy, and call run() — or run_batch() for many streams at once.  All
scheduling arithmetic runs in libalert_b200.so (hand-written sm_100a CUDA);
there is no CPU fallback.
"""

from .diagnostics import XiDiagnostics, xi_diagnostics, xi_diagnostics_from_values
from .estimator import IdleFilterConfig, IdlePowerEstimate, KalmanConfig, SlowdownEstimate, idle_power_init, slowdown_init
from .model import ConfigSpace, ConstraintSpec, DnnKind, DnnProfile, Mode, PowerSetting, Stage, fastest_dnn, validate
from .packing import ProfileError, pack_space, pack_specs
from .policies import POLICY_NAMES, AlertPolicy, BaselinePolicy, OraclePolicy, make_policy
from .records import ConfigDecision, FallbackLevel, GroupState, Prediction, StepRecord, Summary
from .simulator import BatchResult, get_engine, run, run_batch, run_injected
from .synth import ProfileKnobs, generate_space, preset_space, preset_trace, reference_latency
from .trace import (
    Constant, EnvironmentPhase, Gaussian, LogNormal, Trace, TrueEnvironment, Uniform, lognormal_matching,
    pack_envs, pack_goal_changes, realize,
)

__version__ = "0.1.0"

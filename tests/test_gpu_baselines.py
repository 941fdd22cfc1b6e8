"""GPU parity of the comparison schemes (oracle-static, sys-only, app-only,
no-coord; policies.py:211-454) against reference-generated goldens and the
CPU oracle.  They are FP64 end to end on the GPU, so decisions and values
must match exactly (CUDA erf/sqrt vs glibc erf/pow could in principle flip
an exact tie; none occurs in these cases)."""

import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

import paper_1911_00119_b200 as A  # noqa: E402
from paper_1911_00119_b200 import abi  # noqa: E402
from oracle import oracle  # noqa: E402
from helpers import random_space  # noqa: E402

BASELINES = ("oracle-static", "sys-only", "app-only", "no-coord")


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__

    __graft_entry__.build()
    oracle.build()


def _mean(agg, f):
    return abi.neumaier_total(agg[f], agg[f + 1]) / agg[abi.AGG_N]


def test_golden_baselines_on_gpu(golden_baselines):
    for case in golden_baselines:
        res = A.run_injected(case.space, case.spec, case.env, case.policy, kalman=case.kalman,
                             group_size=case.group_size)
        d = res.decoded()
        z = case.z
        np.testing.assert_array_equal(d["cand"][:, 0], z["cand"], err_msg=case.name)
        np.testing.assert_array_equal(d["completed"][:, 0], z["completed"], err_msg=case.name)
        np.testing.assert_array_equal(d["met"][:, 0], z["met"], err_msg=case.name)
        for f in ("energy", "accuracy", "latency"):
            np.testing.assert_array_equal(res.records[f][:, 0], z[f], err_msg=f"{case.name}:{f}")
        if case.policy != "oracle-static":
            np.testing.assert_array_equal(res.records["mu"][:, 0], z["state"][:, 0], err_msg=case.name)
        assert _mean(res.agg[0], abi.AGG_ENERGY) == z["summary"][0], case.name
        assert _mean(res.agg[0], abi.AGG_ACC) == z["summary"][1], case.name


def test_drop_in_run_baselines():
    space = A.preset_space()
    ref = A.reference_latency(space)
    spec = A.ConstraintSpec(mode=A.Mode.MINIMIZE_ENERGY, t_goal=0.14, q_goal=0.68, overhead_budget=0.01 * ref)
    env = A.realize(A.preset_trace())
    for name in BASELINES:
        res = A.run(space, spec, A.preset_trace(), A.make_policy(name))
        rec, agg, _ = oracle.run(space, spec, env, name)
        assert [r.decision.power_index for r in res.records] == list(rec["power"])
        assert res.summary.mean_energy == _mean(agg, abi.AGG_ENERGY)


@pytest.mark.parametrize("seed", range(6))
def test_random_batches_baselines_vs_oracle(seed):
    """Random spaces and specs, 16 streams x 120 steps per launch, every
    scheme: per-stream aggregates and final state equal the oracle's."""
    rnd = random.Random(777 + seed)
    while True:
        space = random_space(rnd, 5, 5)
        kinds = {d.kind for d in space.dnns}
        if len(kinds) == 2:
            break
    specs = []
    for k in range(4):
        t = rnd.uniform(0.05, 3.0)
        if k % 2:
            specs.append(A.ConstraintSpec(mode=A.Mode.MAXIMIZE_ACCURACY, t_goal=t, e_goal=rnd.uniform(0.5, 80.0),
                                          overhead_budget=0.02 * t))
        else:
            specs.append(A.ConstraintSpec(mode=A.Mode.MINIMIZE_ENERGY, t_goal=t, q_goal=rnd.uniform(0.1, 0.99),
                                          overhead_budget=0.0))
    envs = []
    for k in range(16):
        phases = (A.EnvironmentPhase(60, A.Gaussian(rnd.uniform(0.6, 1.6), 0.2), rnd.uniform(1, 9), 0.05),
                  A.EnvironmentPhase(60, A.LogNormal(rnd.uniform(-0.2, 0.7), 0.3), rnd.uniform(1, 9), 0.1))
        envs.append(A.realize(A.Trace(seed=rnd.randint(0, 2**31), phases=phases)))
    for name in BASELINES:
        res = A.run_batch(space, specs, envs, name, records="f64", trace_dtype=np.float64)
        d = res.decoded()
        for k, env in enumerate(envs):
            rec, agg, st = oracle.run(space, specs[k % len(specs)], env, name)
            np.testing.assert_array_equal(d["cand"][:, k], rec["cand"], err_msg=f"{name} stream {k}")
            np.testing.assert_array_equal(res.agg[k, :abi.AGG_LEVEL0], agg[:abi.AGG_LEVEL0])
            np.testing.assert_array_equal(res.agg[k, abi.AGG_PHASE_BASE:], agg[abi.AGG_PHASE_BASE:])
            if name != "oracle-static":
                assert res.state["mu"][k] == st[0] and res.state["phi"][k] == st[5]


def test_oracle_static_refuses_host_streaming():
    from paper_1911_00119_b200.simulator import HostStreamer
    from paper_1911_00119_b200.trace import pack_envs

    space = A.preset_space()
    spec = A.ConstraintSpec(mode=A.Mode.MINIMIZE_ENERGY, t_goal=0.14, q_goal=0.68)
    p = pack_envs([A.realize(A.preset_trace(phase_length=20))])
    with pytest.raises(ValueError, match="whole trace"):
        HostStreamer(space, [spec], p, "oracle-static")

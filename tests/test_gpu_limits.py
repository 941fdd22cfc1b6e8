"""Size limits of the table layout, on the GPU against the CPU oracle: the
W = 1 flat scans exist for tables of <= 64 cells (one 64-bit mark mask, one
flattened unit sequence), so 64 and 65 cells take different code paths; an
anytime DNN at ALERT_MAX_STAGES stages; the largest table the shared-memory
layout takes (ALERT_MAX_CANDIDATES = 6,144 candidates) and one past it.
Same bar as tests/test_gpu_parity.py: teacher-forced decisions equal to the
oracle's (FP64 near-ties at ulp level exempt), FP64 values to 1e-12."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

import paper_1911_00119_b200 as A  # noqa: E402
from paper_1911_00119_b200 import abi  # noqa: E402
from paper_1911_00119_b200.synth import preset_batch  # noqa: E402
from paper_1911_00119_b200.trace import unpack_row  # noqa: E402
from oracle import oracle  # noqa: E402

EXEMPT_GAP = 1e-12
RTOL_F64 = 1e-12


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__

    __graft_entry__.build()
    oracle.build()


def _specs(space):
    ref = A.reference_latency(space)
    cap = space.max_power.cap_watts
    return [
        A.ConstraintSpec(mode=A.Mode.MINIMIZE_ENERGY, t_goal=1.0 * ref, q_goal=0.7, overhead_budget=0.01 * ref),
        A.ConstraintSpec(mode=A.Mode.MINIMIZE_ENERGY, t_goal=0.5 * ref, q_goal=0.85, overhead_budget=0.0),
        A.ConstraintSpec(mode=A.Mode.MAXIMIZE_ACCURACY, t_goal=0.8 * ref, e_goal=0.6 * cap * 0.8 * ref,
                         pr_threshold=0.95, overhead_budget=0.01 * ref),
        A.ConstraintSpec(mode=A.Mode.MAXIMIZE_ACCURACY, t_goal=1.5 * ref, e_goal=0.3 * cap * 1.5 * ref,
                         overhead_budget=0.01 * ref),
    ]


def _check(space, n_streams, n_steps, policy="alert", lanes=None):
    specs = _specs(space)
    packed = preset_batch(n_streams, lengths=(n_steps // 3, n_steps // 3, n_steps - 2 * (n_steps // 3)),
                          seed0=900, dtype=np.float64, processes=1)
    envs = [unpack_row(packed, k) for k in range(n_streams)]
    recs = [oracle.run(space, specs[k % len(specs)], env, policy) for k, env in enumerate(envs)]
    forced = np.stack([r[0]["cand"] for r in recs], 1).astype(np.int32)
    res = A.run_batch(space, specs, packed, policy, records="f64", forced=forced, lanes_per_stream=lanes)
    d = res.decoded()
    for k, (rec, agg, _) in enumerate(recs):
        bad = np.flatnonzero(d["cand"][:, k] != rec["cand"])
        for n in bad:
            assert rec["gap"][n] <= EXEMPT_GAP or rec["boundary"][n] <= EXEMPT_GAP, (k, n)
        np.testing.assert_allclose(res.records["energy"][:, k], rec["energy"], rtol=RTOL_F64)
        np.testing.assert_allclose(res.agg[k, :abi.AGG_LEVEL0], agg[:abi.AGG_LEVEL0], rtol=RTOL_F64)
    # and free-running (no forcing) equals the oracle's own run on these inputs
    free = A.run_batch(space, specs, packed, policy, lanes_per_stream=lanes)
    for k, (rec, agg, _) in enumerate(recs):
        if not np.any(rec["gap"] <= EXEMPT_GAP) and not np.any(rec["boundary"] <= EXEMPT_GAP):
            np.testing.assert_allclose(free.agg[k, :abi.AGG_LEVEL0], agg[:abi.AGG_LEVEL0], rtol=RTOL_F64)
    return res


@pytest.mark.parametrize("knobs,cells", [
    (dict(n_dnns=5, n_powers=8, anytime_stages=4), 64),   # largest flat-scan table
    (dict(n_dnns=10, n_powers=5, anytime_stages=4), 65),  # first table past it
    (dict(n_dnns=4, n_powers=6, anytime_stages=8), 66),   # ALERT_MAX_STAGES-stage anytime DNN
])
@pytest.mark.parametrize("policy", ["alert", "alert+oracle"])
def test_flat_scan_boundary_vs_oracle(knobs, cells, policy):
    space = A.generate_space(A.ProfileKnobs(**knobs))
    assert A.pack_space(space).n_candidates == cells
    lanes = [None, 2] if cells > 64 else [None]
    for w in lanes:
        _check(space, 8, 240, policy, lanes=w)


def test_largest_table_vs_oracle():
    """6,144 candidates (93 DNNs incl. a 4-stage anytime one x 64 caps)."""
    space = A.generate_space(A.ProfileKnobs(n_dnns=93, n_powers=64))
    assert A.pack_space(space).n_candidates == abi.MAX_CANDIDATES
    _check(space, 4, 60)


def test_table_past_the_limit_is_rejected():
    space = A.generate_space(A.ProfileKnobs(n_dnns=93, n_powers=65))
    with pytest.raises(ValueError, match="candidates"):
        A.run_batch(space, _specs(space)[:1], preset_batch(1, lengths=(4, 4, 4), processes=1), "alert")


def test_degenerate_and_ragged_shapes():
    """One stream x one input; one-input phases; stream counts that do not
    fill a warp (W = 1) or a tile group (W = 8); an empty stream range
    through the C ABI is a no-op (no launch, outputs untouched)."""
    space = A.preset_space()
    ref = A.reference_latency(space)
    spec = A.ConstraintSpec(mode=A.Mode.MINIMIZE_ENERGY, t_goal=0.14, q_goal=0.68, overhead_budget=0.01 * ref)
    # one stream, one input
    env1 = A.realize(A.Trace(seed=7, phases=(A.EnvironmentPhase(1, A.Constant(1.0), 4.0, 0.05),)))
    rec, agg, _ = oracle.run(space, spec, env1, "alert")
    res = A.run_batch(space, [spec], [env1], "alert", records="f64")
    assert res.decoded()["cand"][0, 0] == rec["cand"][0]
    np.testing.assert_allclose(res.agg[0, :abi.AGG_LEVEL0], agg[:abi.AGG_LEVEL0], rtol=RTOL_F64)
    # one-input phases (a segment change at every step), 33 streams at W = 1, 3 streams at W = 8
    phases = tuple(A.EnvironmentPhase(1, A.Gaussian(1.0 + 0.2 * k, 0.1), 3.0 + k, 0.05) for k in range(3))
    for n, lanes in ((33, 1), (3, 8)):
        envs = [A.realize(A.Trace(seed=100 + k, phases=phases * 2)) for k in range(n)]
        recs = [oracle.run(space, spec, e, "alert") for e in envs]
        res = A.run_batch(space, [spec], envs, "alert", records="f64", trace_dtype=np.float64,
                          lanes_per_stream=lanes)
        for k, (rec, agg, _) in enumerate(recs):
            np.testing.assert_array_equal(res.decoded()["cand"][:, k], rec["cand"])
            np.testing.assert_allclose(res.agg[k, :abi.AGG_LEVEL0], agg[:abi.AGG_LEVEL0], rtol=RTOL_F64)
    # empty ranges: nothing launched, outputs untouched
    eng = A.get_engine(0)
    table = eng.table(space)
    packed = A.pack_envs([env1, env1], dtype=np.float64)
    trace = eng.upload_trace(packed)
    state = eng.new_state(table, 2)
    from paper_1911_00119_b200.engine import outputs_struct
    agg_t = torch.full((2, abi.AGG_FIELDS), 7.0, dtype=torch.float64, device=eng.tdev)
    before = eng.launch_count()
    eng.run(table, A.pack_specs([spec]), trace, state, policy=abi.POLICY_ALERT, outputs=outputs_struct(None, agg=agg_t),
            stream_begin=1, stream_end=1)
    torch.cuda.synchronize()
    assert eng.launch_count() == before and bool((agg_t == 7.0).all())

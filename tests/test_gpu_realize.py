"""On-device trace realization (§8(f) rank 4): the reference's per-phase
recipe with Philox streams.  Distributional parity with the reference's
numpy draws (moments per phase), determinism, and decision parity of a run
over the generated trace against the CPU oracle on the exported arrays."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

import paper_1911_00119_b200 as A  # noqa: E402
from paper_1911_00119_b200 import abi  # noqa: E402
from paper_1911_00119_b200.synth import preset_phases, realize_on_device  # noqa: E402
from paper_1911_00119_b200.trace import PackedEnvs  # noqa: E402
from oracle import oracle  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__

    __graft_entry__.build()
    oracle.build()


def test_moments_match_numpy_realize():
    phases = preset_phases((400, 400, 400), 0.05)
    dt = realize_on_device(phases, 8192, seed=7, dtype=np.float64)
    s = dt.slowdown.cpu().numpy()
    ref = np.stack([A.realize(A.Trace(seed=42 + k, phases=phases)).slowdown for k in range(512)], 1)
    for k in range(3):
        a, b = s[400 * k:400 * (k + 1)].ravel(), ref[400 * k:400 * (k + 1)].ravel()
        assert abs(a.mean() - b.mean()) < 4 * b.std() / np.sqrt(len(b)) + 1e-12
        assert abs(a.std() - b.std()) < 0.05 * b.std() + 1e-12
    assert (s >= 0.01).all()
    again = realize_on_device(phases, 8192, seed=7, dtype=np.float64).slowdown.cpu().numpy()
    np.testing.assert_array_equal(s, again)
    shifted = realize_on_device(phases, 100, seed=7, stream_offset=50, dtype=np.float64).slowdown.cpu().numpy()
    np.testing.assert_array_equal(shifted[:, :50], s[:, 50:100])  # stream k is keyed by its global index


def test_run_on_device_trace_matches_oracle_on_exported_arrays():
    space = A.preset_space()
    ref = A.reference_latency(space)
    spec = A.ConstraintSpec(mode=A.Mode.MINIMIZE_ENERGY, t_goal=ref, q_goal=0.85, overhead_budget=0.01 * ref)
    phases = preset_phases((100, 100, 100), 0.05)
    dt = realize_on_device(phases, 64, seed=3, dtype=np.float64)
    res = A.run_batch(space, [spec], dt, "alert", records="f64")
    host = PackedEnvs(dt.slowdown.cpu().numpy(), dt.n_segments.cpu().numpy(), dt.seg_end.cpu().numpy(),
                      dt.seg_phase.cpu().numpy(), dt.seg_idle.cpu().numpy())
    agg, _ = oracle.run_batch(space, A.pack_specs([spec]), host, 64, "alert")
    np.testing.assert_array_equal(res.agg[:, :abi.AGG_LEVEL0], agg[:, :abi.AGG_LEVEL0])

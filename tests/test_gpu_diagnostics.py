"""xi diagnostics on the GPU (simulator.py:508-543) equal numpy's
histogram / mean / std bit for bit (what the reference itself calls)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

import paper_1911_00119_b200 as A  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__

    __graft_entry__.build()


def _ref(xi):
    counts, edges = np.histogram(xi, bins=40)
    return counts, edges, float(np.mean(xi)), float(np.std(xi))


@pytest.mark.parametrize("n", [30, 31, 100, 127, 128, 129, 1000, 4097, 100003, 1000003])
def test_xi_stats_equal_numpy(n):
    rng = np.random.default_rng(n)
    for xi in (rng.lognormal(0.3, 0.4, n), rng.normal(1.3, 0.1, n), np.round(rng.uniform(0.5, 2.5, n), 2)):
        d = A.xi_diagnostics_from_values(xi)
        c, e, m, s = _ref(xi)
        np.testing.assert_array_equal(d.counts, c)
        np.testing.assert_array_equal(d.bin_edges, e)
        assert d.mean == m and d.sd == s
    const = np.full(n, 1.25)  # min == max: numpy widens the range by 0.5
    d = A.xi_diagnostics_from_values(const)
    c, e, m, s = _ref(const)
    np.testing.assert_array_equal(d.counts, c)
    np.testing.assert_array_equal(d.bin_edges, e)
    assert d.mean == m and d.sd == s


def test_xi_diagnostics_of_a_run_match_reference_records(golden_runs):
    """The drop-in run() records carry the reference's (fb_latency, fb_t_prof);
    the GPU diagnostics equal numpy over the reference's own values."""
    case = next(c for c in golden_runs if c.name == "preset600_minE_alert")
    res = A.run(case.space, case.spec, A.preset_trace(), A.make_policy("alert"))
    fb = np.array([(r.fb_latency, r.fb_t_prof) for r in res.records])
    np.testing.assert_array_equal(fb, case.z["fb"])
    d = A.xi_diagnostics(res.records)
    xi = case.z["fb"][:, 0] / case.z["fb"][:, 1]
    c, e, m, s = _ref(xi)
    np.testing.assert_array_equal(d.values, xi)
    np.testing.assert_array_equal(d.counts, c)
    np.testing.assert_array_equal(d.bin_edges, e)
    assert d.mean == m and d.sd == s
    with pytest.raises(ValueError, match="at least 30"):
        A.xi_diagnostics(res.records[:10])

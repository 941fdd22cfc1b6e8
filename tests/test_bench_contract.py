"""bench.py workload construction (CPU): per-rank item ranges are disjoint,
contiguous and cover the configured totals; c3/c4/c5 are
fixed-total (strong) by default, c1/c2 per-rank (weak)."""

import importlib.util
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", ROOT / "bench.py")
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


@pytest.mark.parametrize("cfg,total", [("c3", 1 << 20), ("c4", 1 << 24), ("c5", 1 << 24)])
def test_strong_shards_cover_the_total_exactly(cfg, total):
    b = _bench()
    for world in (1, 2, 4, 8):
        ranges = [b.item_range(cfg, world, r) for r in range(world)]
        assert all(t == total and sc == "strong" for _, _, t, sc in ranges)
        assert ranges[0][0] == 0 and ranges[-1][1] == total
        assert all(ranges[r][1] == ranges[r + 1][0] for r in range(world - 1))  # contiguous, disjoint
        sizes = [e - s for s, e, _, _ in ranges]
        assert max(sizes) - min(sizes) <= 1


def test_weak_default_for_c2_and_overrides():
    b = _bench()
    assert b.item_range("c2", 4, 3) == (3 * 65536, 4 * 65536, 4 * 65536, "weak")
    assert b.item_range("c3", 2, 1, per_rank=1000) == (1000, 2000, 2000, "weak")
    assert b.item_range("c2", 2, 1, total=1000) == (500, 1000, 1000, "strong")


def test_full_grid_is_every_scenario_once_with_both_modes_per_rank():
    b = _bench()
    total = 1 << 24
    for world in (2, 8):
        counts = np.zeros(2, np.int64)
        for r in range(world):
            s, e, _, _ = b.item_range("c4", world, r)
            scen = b.grid_scenarios(np.arange(s, e), total)
            assert scen[0] == s and scen[-1] == e - 1  # the full grid: scenario = item
            spec, row = b.grid_coords(scen)
            frac_max_acc = float((spec >= 4096).mean())
            assert frac_max_acc == 0.5  # balanced: both goal modes, half each, on every rank
            counts += np.bincount((spec >= 4096).astype(int), minlength=2)
        assert counts.sum() == total


def test_grid_coordinates_enumerate_the_paper_grid():
    b = _bench()
    spec, row = b.grid_coords(np.arange(1 << 24, dtype=np.int64))
    pairs = spec.astype(np.int64) * 2048 + row
    assert len(np.unique(pairs)) == 1 << 24  # 8,192 goal tuples x 2,048 traces, each once
    assert spec.max() == 8191 and row.max() == 2047


def test_sampled_grid_keeps_every_trace_and_both_modes():
    b = _bench()
    for total in (1 << 16, 1000):
        scen = b.grid_scenarios(np.arange(total), total)
        assert len(np.unique(scen)) == total
        spec, row = b.grid_coords(scen)
        assert len(np.unique(row)) == min(total, 2048) and abs(float((spec >= 4096).mean()) - 0.5) < 0.05
    spec, row = b.grid_coords(b.grid_scenarios(np.arange(1 << 16), 1 << 16))
    assert len(np.unique(spec)) == 32 and (np.diff(spec[:2048]) == 0).all()  # whole tuples, warps share goals


def test_c4_workload_runs_min_energy_items_first():
    b = _bench()
    s, e, total, _ = b.item_range("c4", 2, 1, total=8 * 2048)
    wl = b.build_workload("c4", 300, s, e, total)
    modes = wl["specs"]["mode"][wl["stream_spec"]]
    assert len(modes) == e - s and set(modes.tolist()) == {0, 1}
    assert np.all(np.diff(modes) >= 0)  # one contiguous run per mode: two launches


def test_c2_ranks_use_distinct_trace_seeds():
    b = _bench()
    a = b.build_workload("c2", 30, 0, 8, 16)["packed"].slowdown
    c = b.build_workload("c2", 30, 8, 16, 16)["packed"].slowdown
    assert a.shape == c.shape == (30, 8)
    assert not np.array_equal(a, c)
    # item k's trace does not depend on the sharding
    whole = b.build_workload("c2", 30, 0, 16, 16)["packed"].slowdown
    np.testing.assert_array_equal(whole[:, 8:], c)


def test_goal_change_workload():
    b = _bench()
    wl = b.build_workload("c2", 90, 0, 6, 6, goal_changes=2)
    p = wl["packed"]
    assert (p.goal_n == 3).all()
    np.testing.assert_array_equal(p.goal_end[0], [30, 60, 90])


def test_clock_summary_keeps_timed_region_samples_and_reasons():
    """Clock samples ("sm, max, 0xreasons" lines, NVML or nvidia-smi) are
    reported only from inside the timed region; idle is not a reason,
    thermal slowdown is."""
    cs = _bench().ClockSampler(0)
    cs.source = "test"
    cs.t0, cs.t1 = 10.0, 11.0
    cs.lines = [(9.0, "1000, 1965, 0x1"), (10.2, "1965, 1965, 0x0"), (10.4, "1965, 1965, 0x0"),
                (10.6, "1950, 1965, 0x20"), (12.0, "500, 1965, 0x8")]
    s = cs.summary()
    assert s["samples"] == 3 and s["sm_mhz"] == 1965.0 and s["sm_max_mhz"] == 1965.0
    assert s["reasons"] == ["sw_thermal_slowdown"] and s["source"] == "test"
    cs.lines = []
    assert cs.summary()["samples"] == 0

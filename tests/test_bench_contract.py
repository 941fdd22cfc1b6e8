"""bench.py workload construction (CPU): per-rank shards are disjoint and
cover the configured grids the way DESIGN.md §5 states (weak scaling)."""

import importlib.util
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", ROOT / "bench.py")
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_c4_ranks_sample_disjoint_grid_points_of_both_modes():
    b = _bench()
    world, n = 4, 256
    seen = set()
    for rank in range(world):
        wl = b.build_workload("c4", n, 300, rank, world)
        ss, sr = wl["stream_spec"], wl["stream_row"]
        modes = wl["specs"]["mode"][ss]
        assert len(set(modes.tolist())) == 2  # both goal modes on every rank
        keys = set(zip(ss.tolist(), sr.tolist()))
        assert len(keys) == n and not (keys & seen)  # (goal tuple, trace) scenarios are disjoint
        seen |= keys


def test_c2_ranks_use_distinct_trace_seeds():
    b = _bench()
    a = b.build_workload("c2", 8, 30, 0, 2)["packed"].slowdown
    c = b.build_workload("c2", 8, 30, 1, 2)["packed"].slowdown
    assert a.shape == c.shape == (30, 8)
    assert not np.array_equal(a, c)

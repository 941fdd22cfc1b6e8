"""GPU parity at benchmark sizes (BASELINE configs 2-5), through size-
independent properties plus an oracle check of a random stream subset.

* C2-style: 8,192 streams x 10,000 steps, preset table, 9 min-energy specs;
  16 random streams re-run on the CPU oracle must match decision for decision
  (ulp-level near-ties exempt, see test_gpu_parity) and aggregate for aggregate.
* determinism: two launches give bit-identical aggregates and final state;
  chunking the steps (state carried on the device) changes nothing.
* C4-style grid on the 64x32 table (2,144 candidates): shared traces via
  stream_row, mixed modes; tile widths agree bit for bit; oracle subset.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

import paper_1911_00119_b200 as A  # noqa: E402
from paper_1911_00119_b200 import abi  # noqa: E402
from paper_1911_00119_b200.synth import preset_batch  # noqa: E402
from paper_1911_00119_b200.trace import PackedEnvs, unpack_row  # noqa: E402
from oracle import oracle  # noqa: E402

EXEMPT_GAP = 1e-12


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__

    __graft_entry__.build()


def _c2_specs(space):
    ref = A.reference_latency(space)
    return [A.ConstraintSpec(mode=A.Mode.MINIMIZE_ENERGY, t_goal=dm * ref, q_goal=q, overhead_budget=0.01 * ref)
            for q in (0.68, 0.70, 0.85) for dm in (0.8, 1.0, 1.5)]


@pytest.fixture(scope="module")
def c2():
    space = A.preset_space()
    specs = _c2_specs(space)
    packed = preset_batch(8192, lengths=(3334, 3333, 3333), seed0=42, dtype=np.float32)
    return space, specs, packed


def _subset_check(space, specs, packed, res, streams, policy="alert", stream_spec=None, stream_row=None):
    dec = res.decoded() if res.records else None
    for k in streams:
        row = k if stream_row is None else int(stream_row[k])
        env = unpack_row(packed, row)
        si = k % len(specs) if stream_spec is None else int(stream_spec[k])
        rec, agg, st = oracle.run(space, specs[si], env, policy)
        if dec is not None:
            bad = np.flatnonzero(dec["cand"][:, k] != rec["cand"])
            if len(bad):
                assert rec["gap"][bad[0]] <= EXEMPT_GAP or rec["boundary"][bad[0]] <= EXEMPT_GAP
                continue
        np.testing.assert_allclose(res.agg[k, :abi.AGG_LEVEL0], agg[:abi.AGG_LEVEL0], rtol=1e-12,
                                   err_msg=f"stream {k}")
        if policy != "oracle":
            np.testing.assert_allclose(res.state["mu"][k], st[0], rtol=1e-12)


def test_c2_scale_subset_vs_oracle(c2):
    space, specs, packed = c2
    res = A.run_batch(space, specs, packed, "alert", records="f32")
    assert res.agg[:, abi.AGG_N].sum() == 8192 * 10000
    rng = np.random.default_rng(7)
    _subset_check(space, specs, packed, res, rng.choice(8192, 16, replace=False))
    # per-step records agree with the aggregates (sum of energies, float32 records)
    k = 123
    e = res.records["energy"][:, k].astype(np.float64).sum()
    assert abs(e - abi.neumaier_total(res.agg[k, abi.AGG_ENERGY], res.agg[k, abi.AGG_ENERGY_C])) <= 1e-5 * abs(e)


def test_c2_scale_determinism_and_chunking(c2):
    space, specs, packed = c2
    a = A.run_batch(space, specs, packed, "alert")
    b = A.run_batch(space, specs, packed, "alert")
    c = A.run_batch(space, specs, packed, "alert", chunk_steps=1000)
    np.testing.assert_array_equal(a.agg, b.agg)
    np.testing.assert_array_equal(a.agg, c.agg)
    for f in a.state:
        np.testing.assert_array_equal(a.state[f], b.state[f])
        np.testing.assert_array_equal(a.state[f], c.state[f])


def test_host_streamer_matches_device_resident(c2):
    space, specs, packed = c2
    from paper_1911_00119_b200.simulator import HostStreamer

    dev = A.run_batch(space, specs, packed, "alert")
    hs = HostStreamer(space, A.pack_specs(specs), packed, "alert", chunk_steps=777)
    agg = hs.run()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(agg.numpy(), dev.agg)
    # last chunk as stream ranges with the aggregate D2H overlapped (uneven cuts), twice in a row
    hs = HostStreamer(space, A.pack_specs(specs), packed, "alert", chunk_steps=2000, d2h_parts=3)
    for _ in range(2):
        agg = hs.run()
        torch.cuda.current_stream().synchronize()
        np.testing.assert_array_equal(agg.numpy(), dev.agg)
    side = torch.cuda.Stream()  # a pass issued from another caller stream, back to back with the last one
    hs.run()
    with torch.cuda.stream(side):
        agg = hs.run()
    side.synchronize()
    np.testing.assert_array_equal(agg.numpy(), dev.agg)


def test_host_streamer_stream_ranges_grid():
    """Shared trace rows + two goal modes + a last chunk split into stream
    ranges that cut through the mode runs: equal to the device-resident run."""
    from paper_1911_00119_b200.simulator import HostStreamer

    space, specs, packed, ss, sr = _grid(n_traces=16, steps=300)
    dev = A.run_batch(space, A.pack_specs(specs), packed, "alert", stream_spec=ss, stream_row=sr)
    for parts in (1, 5):
        hs = HostStreamer(space, A.pack_specs(specs), packed, "alert", stream_spec=ss, stream_row=sr,
                          chunk_steps=64, d2h_parts=parts)
        agg = hs.run()
        torch.cuda.current_stream().synchronize()
        np.testing.assert_array_equal(agg.numpy(), dev.agg)


def _grid(n_traces=64, steps=300):
    space = A.generate_space(A.ProfileKnobs(n_dnns=64, n_powers=32))
    ref = A.reference_latency(space)
    specs = []
    for dm in (0.5, 1.0, 1.6):
        specs.append(A.ConstraintSpec(mode=A.Mode.MINIMIZE_ENERGY, t_goal=dm * ref, q_goal=0.8,
                                      overhead_budget=0.01 * ref))
        specs.append(A.ConstraintSpec(mode=A.Mode.MAXIMIZE_ACCURACY, t_goal=dm * ref,
                                      e_goal=0.6 * 50.0 * dm * ref, overhead_budget=0.01 * ref))
    parts = [preset_batch(1, lengths=(100, 100, 100), seed0=500 + t, order=(t % 3, (t + 1) % 3, (t + 2) % 3),
                          dtype=np.float32, processes=1) for t in range(n_traces)]
    packed = PackedEnvs(np.concatenate([p.slowdown for p in parts], 1),
                        np.concatenate([p.n_segments for p in parts]), np.concatenate([p.seg_end for p in parts]),
                        np.concatenate([p.seg_phase for p in parts]), np.concatenate([p.seg_idle for p in parts]))
    n = n_traces * len(specs)
    stream_spec = (np.arange(n) // n_traces).astype(np.int32)  # mode-uniform warps
    stream_row = (np.arange(n) % n_traces).astype(np.int32)
    return space, specs, packed, stream_spec, stream_row


@pytest.mark.parametrize("policy", ["alert", "oracle", "alert+oracle"])
def test_c4_grid_tiles_agree_and_subset_vs_oracle(policy):
    space, specs, packed, ss, sr = _grid()
    outs = {}
    for lanes in (4, 8, 32):
        outs[lanes] = A.run_batch(space, A.pack_specs(specs), packed, policy, stream_spec=ss, stream_row=sr,
                                  records="f32", lanes_per_stream=lanes)
    A.get_engine().set_launch(0, 0)
    for lanes in (4, 8):
        np.testing.assert_array_equal(outs[lanes].records["decision"], outs[32].records["decision"])
        np.testing.assert_array_equal(outs[lanes].agg, outs[32].agg)
    rng = np.random.default_rng(3)
    base = "oracle" if policy == "oracle" else "alert"
    _subset_check(space, specs, packed, outs[32], rng.choice(len(ss), 6, replace=False), base, ss, sr)


@pytest.fixture(scope="module")
def c3():
    space = A.preset_space()
    ref = A.reference_latency(space)
    specs = []
    for dm in (0.6, 0.8, 1.2):
        t = dm * ref
        for pr in (0.95, 0.99):
            specs.append(A.ConstraintSpec(mode=A.Mode.MAXIMIZE_ACCURACY, t_goal=t, e_goal=0.6 * 50.0 * t,
                                          pr_threshold=pr, overhead_budget=0.01 * ref))
    packed = preset_batch(4096, lengths=(334, 333, 333), seed0=4242, dtype=np.float32)
    return space, specs, packed


def test_c3_scale_subset_vs_oracle(c3):
    """C3-style (max-accuracy + pr_th, anytime stages): the certified fast
    max-accuracy scan and its near-tie fallbacks give the oracle's decisions."""
    space, specs, packed = c3
    res = A.run_batch(space, specs, packed, "alert", records="f32")
    assert res.agg[:, abi.AGG_N].sum() == 4096 * 1000
    rng = np.random.default_rng(11)
    _subset_check(space, specs, packed, res, rng.choice(4096, 24, replace=False))


def test_c3_scale_fast_scan_equals_full_scan(c3):
    space, specs, packed = c3
    a = A.run_batch(space, specs, packed, "alert", records="f32")
    b = A.run_batch(space, specs, packed, "alert", records="f32", flags=abi.FLAG_NO_FAST)
    np.testing.assert_array_equal(a.decoded()["cand"], b.decoded()["cand"])
    np.testing.assert_array_equal(a.records["energy"], b.records["energy"])
    np.testing.assert_array_equal(a.agg[:, :abi.AGG_LEVEL0], b.agg[:, :abi.AGG_LEVEL0])


@pytest.mark.parametrize("lanes", [1, 8])
def test_c4_grid_row_scan_equals_full_scan(lanes):
    """Row mode on the 64x32 table (rows by smallest cap*t with the energy
    bound stop, surely-infeasible rows skipped) changes no decision or value
    against the full scan, at one lane and at the default 8 lanes per stream."""
    space, specs, packed, ss, sr = _grid(n_traces=32, steps=300)
    kw = dict(stream_spec=ss, stream_row=sr, records="f32", lanes_per_stream=lanes)
    fast = A.run_batch(space, A.pack_specs(specs), packed, "alert", **kw)
    full = A.run_batch(space, A.pack_specs(specs), packed, "alert", flags=abi.FLAG_NO_FAST, **kw)
    A.get_engine().set_launch(0, 0)
    np.testing.assert_array_equal(fast.decoded()["cand"], full.decoded()["cand"])
    np.testing.assert_array_equal(fast.records["energy"], full.records["energy"])
    np.testing.assert_array_equal(fast.agg[:, :abi.AGG_LEVEL0], full.agg[:, :abi.AGG_LEVEL0])


@pytest.mark.parametrize("policy", ["alert+oracle", "alert-any"])
def test_host_streamer_goal_changes_and_policies(policy):
    """The host-streaming path with goal changes streamed beside the trace
    (one launch over every spec per chunk), the oracle alongside, and a
    kinds-filtered policy: per-stream aggregates equal the device-resident
    run bit for bit."""
    from paper_1911_00119_b200.simulator import HostStreamer
    from paper_1911_00119_b200.trace import pack_goal_changes

    space = A.preset_space()
    ref = A.reference_latency(space)
    specs = [A.ConstraintSpec(mode=A.Mode.MINIMIZE_ENERGY, t_goal=ref, q_goal=0.7, overhead_budget=0.01 * ref),
             A.ConstraintSpec(mode=A.Mode.MAXIMIZE_ACCURACY, t_goal=0.8 * ref, e_goal=0.6 * 50 * 0.8 * ref,
                              pr_threshold=0.95, overhead_budget=0.01 * ref),
             A.ConstraintSpec(mode=A.Mode.MINIMIZE_ENERGY, t_goal=1.5 * ref, q_goal=0.85, overhead_budget=0.0)]
    n, steps = 300, 600
    packed = preset_batch(n, lengths=(200, 200, 200), seed0=77, dtype=np.float32, processes=1)
    sched = [None if k % 5 == 0 else [(0, k % 3), (150 + k % 7, (k + 1) % 3), (420, (k + 2) % 3)]
             for k in range(n)]
    packed.goal_n, packed.goal_end, packed.goal_spec = pack_goal_changes(sched, steps, len(specs))
    ps = A.pack_specs(specs)
    ss = (np.arange(n) % len(specs)).astype(np.int32)
    dev = A.run_batch(space, ps, packed, policy, stream_spec=ss)
    hs = HostStreamer(space, ps, packed, policy, stream_spec=ss, chunk_steps=128, d2h_parts=2)
    agg = hs.run()
    torch.cuda.current_stream().synchronize()
    np.testing.assert_array_equal(agg.numpy(), dev.agg)

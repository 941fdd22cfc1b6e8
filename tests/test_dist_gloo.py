"""N>1 host path on CPU with gloo (world_size 2): sharding covers every stream
exactly once and the rank-ordered aggregate exchange reproduces the
single-process totals.  Per-shard compute is done by the CPU oracle here
(test infrastructure) — on GPUs the same code path reduces alert_reduce
outputs over NCCL."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1911_00119_b200.dist import shard


def test_shard_partitions():
    for n in (0, 1, 7, 65536, 1000003):
        for w in (1, 2, 3, 8):
            ranges = [shard(n, w, r) for r in range(w)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            sizes = [e - b for b, e in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle
        import paper_1911_00119_b200 as A
        from paper_1911_00119_b200.dist import max_over_ranks, reduce_aggregates
        from paper_1911_00119_b200.synth import preset_batch

        n_streams = 10
        space = A.preset_space()
        ref = A.reference_latency(space)
        specs = A.pack_specs([A.ConstraintSpec(mode=A.Mode.MINIMIZE_ENERGY, t_goal=dm * ref, q_goal=0.7,
                                               overhead_budget=0.01 * ref) for dm in (0.8, 1.0, 1.5)])
        b, e = shard(n_streams, world, rank)
        packed = preset_batch(e - b, lengths=(40, 30, 30), seed0=42 + b, dtype=np.float64, processes=1)
        agg, _ = oracle.run_batch(space, specs, packed, e - b, "alert",
                                  stream_spec=np.arange(b, e) % len(specs), threads=1)
        local = torch.from_numpy(agg.sum(0))
        total = reduce_aggregates(local)
        worst = max_over_ranks(float(rank))
        q.put((rank, total.numpy(), worst))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_reduction_matches_single_process():
    from oracle import oracle
    import paper_1911_00119_b200 as A
    from paper_1911_00119_b200.synth import preset_batch

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    totals = [o[1] for o in out]
    np.testing.assert_array_equal(totals[0], totals[1])  # every rank holds the same total
    assert all(o[2] == 1.0 for o in out)  # max over ranks

    space = A.preset_space()
    ref = A.reference_latency(space)
    specs = A.pack_specs([A.ConstraintSpec(mode=A.Mode.MINIMIZE_ENERGY, t_goal=dm * ref, q_goal=0.7,
                                           overhead_budget=0.01 * ref) for dm in (0.8, 1.0, 1.5)])
    packed = preset_batch(10, lengths=(40, 30, 30), seed0=42, dtype=np.float64, processes=1)
    agg, _ = oracle.run_batch(space, specs, packed, 10, "alert", stream_spec=np.arange(10) % 3, threads=1)
    single = agg[:5].sum(0) + agg[5:].sum(0)  # rank-ordered partial sums
    np.testing.assert_array_equal(totals[0], single)
    assert totals[0][0] == 10 * 100  # every stream-step counted once

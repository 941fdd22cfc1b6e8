"""Small fused runs for compute-sanitizer (racecheck / memcheck / synccheck):
every tile width the library instantiates, both goal modes, ALERT, ALERT
with the oracle alongside, the oracle and a comparison scheme, a chunked run
(state carried between launches), goal changes and per-step records.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_1911_00119_b200 as A  # noqa: E402
from paper_1911_00119_b200.synth import preset_batch  # noqa: E402


def main():
    space = A.preset_space()
    ref = A.reference_latency(space)
    specs = [
        A.ConstraintSpec(mode=A.Mode.MINIMIZE_ENERGY, t_goal=0.9 * ref, q_goal=0.7, overhead_budget=0.01 * ref),
        A.ConstraintSpec(mode=A.Mode.MAXIMIZE_ACCURACY, t_goal=0.8 * ref, e_goal=0.6 * 50 * 0.8 * ref,
                         pr_threshold=0.95, overhead_budget=0.01 * ref),
        A.ConstraintSpec(mode=A.Mode.MAXIMIZE_ACCURACY, t_goal=1.2 * ref, e_goal=0.4 * 50 * 1.2 * ref,
                         overhead_budget=0.01 * ref),
    ]
    n, steps = 96, 40
    packed = preset_batch(n, lengths=(14, 13, 13), seed0=7, dtype=np.float32, processes=1)
    eng = A.get_engine(0)
    done = 0
    for lanes in (1, 2, 4, 8, 16, 32):
        for pol in ("alert", "alert-any", "alert+oracle", "oracle"):
            res = A.run_batch(space, specs, packed, pol, stream_spec=np.arange(n) % len(specs),
                              records="f32" if lanes in (1, 8) else None, lanes_per_stream=lanes,
                              chunk_steps=17 if lanes == 8 else None, keep_on_device=True)
            done += 1
            assert np.isfinite(res.agg.cpu().numpy()).all()
    for pol in ("sys-only", "app-only", "no-coord", "oracle-static"):
        A.run_batch(space, specs, packed, pol, stream_spec=np.arange(n) % len(specs), records="f64")
        done += 1
    sched = [[(0, k % 3), (steps // 2, (k + 1) % 3)] for k in range(n)]
    A.run_batch(space, specs, packed, "alert", records="f64", goal_changes=sched)
    done += 1
    big = A.generate_space(A.ProfileKnobs(n_dnns=16, n_powers=8))
    A.run_batch(big, specs, preset_batch(64, lengths=(10, 10, 10), seed0=3, dtype=np.float32, processes=1),
                "alert+oracle", stream_spec=np.arange(64) % 3, lanes_per_stream=8)
    done += 1
    import torch

    torch.cuda.synchronize()
    print(f"sanitize_run: {done} fused runs completed")


if __name__ == "__main__":
    main()

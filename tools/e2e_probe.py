"""HostStreamer pipeline variants on one bench workload: ms per end-to-end
pass for chunk schedules and last-chunk D2H splits (CUDA events, after one
warm-up pass), beside the device-resident alert_run time.
usage: python tools/e2e_probe.py [config] [streams]"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1911_00119_b200.simulator import HostStreamer, chunk_sizes  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
total = int(sys.argv[2]) if len(sys.argv) > 2 else (1 << 20 if cfg == "c3" else 65536)
n_steps = 1000 if cfg == "c3" else 10000
wl = bench.build_workload(cfg, n_steps, 0, total, total)


def timed(hs, reps=5):
    """ms per pass over `reps` back-to-back passes (as bench.py's e2e loop)."""
    hs.run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        hs.run()
    b.record()
    torch.cuda.synchronize()
    return round(a.elapsed_time(b) / reps, 2)


res = {}
for div in (10, 20, 40, 10, 20):
    chunk = n_steps // div
    hs = HostStreamer(wl["space"], wl["specs"], wl["packed"], "alert", stream_spec=wl["stream_spec"],
                      stream_row=wl["stream_row"], chunk_steps=chunk)
    res[f"chunk{chunk}_{len(res)}"] = timed(hs)
    del hs
    torch.cuda.empty_cache()
print(json.dumps({"config": cfg, "streams": total, "steps": n_steps, "ms_per_pass": res}))

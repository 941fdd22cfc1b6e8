"""Host<->device copy rates from pinned memory (the e2e path's input stage):
one copy stream vs chunks alternating over two, at several chunk sizes.
usage: python tools/h2d_probe.py [total_MB]"""
import json
import sys

import torch

total = int(sys.argv[1]) if len(sys.argv) > 1 else 2621
n = total * (1 << 20) // 4
host = torch.empty(n, dtype=torch.float32).pin_memory()
dev = torch.empty(n, dtype=torch.float32, device="cuda")
streams = [torch.cuda.Stream(), torch.cuda.Stream()]
out = {}


def timed(fn):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for s in streams:
        s.wait_stream(torch.cuda.current_stream())
    fn()
    for s in streams:
        torch.cuda.current_stream().wait_stream(s)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


for chunk_mb in (32, 256, 1024):
    c = chunk_mb * (1 << 20) // 4
    for ns in (1, 2):
        def h2d():
            for i, o in enumerate(range(0, n, c)):
                with torch.cuda.stream(streams[i % ns]):
                    dev[o:o + c].copy_(host[o:o + c], non_blocking=True)

        def d2h():
            for i, o in enumerate(range(0, n, c)):
                with torch.cuda.stream(streams[i % ns]):
                    host[o:o + c].copy_(dev[o:o + c], non_blocking=True)

        for name, fn in (("h2d", h2d), ("d2h", d2h)):
            ms = timed(fn)
            out[f"{name}_chunk{chunk_mb}MB_streams{ns}"] = round(n * 4 / (ms * 1e-3) / 1e9, 2)
print(json.dumps({"total_MB": total, "GB_per_s": out}))

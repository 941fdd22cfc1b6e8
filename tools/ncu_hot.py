"""Top stalled SASS instructions (and per-region sample totals) from an ncu report."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]
tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
exe = sum(int(d["Instructions Executed"] or 0) for d in data)
print(f"total samples {tot}, warp-instructions executed {exe}")
cols = [c for c in h if c.startswith("stall_") or "Stall" in c]
hot = sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))[:n]
for d in hot:
    s = int(d["Warp Stall Sampling (All Samples)"] or 0)
    print(f"{s:7d} {100*s/tot:5.1f}%  exe={d['Instructions Executed']:>10}  {d['Address'][-5:]}  {d['Source'].strip()[:70]}")

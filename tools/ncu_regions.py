"""Split an ncu source-page CSV (--print-source sass, gzip ok) into regions of
instructions with equal execution counts (basic-block groups) and print the
heaviest: executed warp-instructions, stall samples, opcode mix.
usage: ncu_regions.py prof_src.csv[.gz] [decisions] [top]"""
import collections
import csv
import gzip
import io
import re
import sys

path = sys.argv[1]
dec = float(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
op = gzip.open if path.endswith(".gz") else open
rows = list(csv.reader(io.StringIO(op(path, "rt").read())))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]
ex = lambda d: int(d["Instructions Executed"] or 0)
samp = lambda d: int(d["Warp Stall Sampling (All Samples)"] or 0)
tot_ex = sum(map(ex, data))
tot_s = sum(map(samp, data))
print(f"warp-instr {tot_ex:.4g}  samples {tot_s}" + (f"  thread-instr/decision {32 * tot_ex / dec:.1f}" if dec else ""))
# regions: maximal runs of consecutive instructions with the same exec count
regs = []
for i, d in enumerate(data):
    e = ex(d)
    if regs and regs[-1]["e"] == e:
        regs[-1]["rows"].append(d)
    else:
        regs.append({"e": e, "rows": [d], "start": i})
for r in regs:
    r["w"] = r["e"] * len(r["rows"])
    r["s"] = sum(map(samp, r["rows"]))
regs.sort(key=lambda r: -r["w"])
for r in regs[:top]:
    ops = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", x["Source"].strip()).split()[0].split(".")[0]
                              for x in r["rows"])
    per = f"{32 * r['w'] / dec:7.1f}/dec" if dec else ""
    print(f"{r['rows'][0]['Address'][-5:]} n={len(r['rows']):4d} exec={r['e']:>10} share={100 * r['w'] / tot_ex:5.1f}% "
          f"{per} stall={100 * r['s'] / max(1, tot_s):5.1f}%  {dict(ops.most_common(8))}")

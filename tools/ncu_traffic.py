"""Summarise tools/gpurun/traffic.sh captures into profiles/ncu_traffic.json:
DRAM bytes (read + write) per decision of run_kernel at the bench shapes
(bench.py multiplies it by a launch's decisions for roofline.traffic).
usage: ncu_traffic.py gpurun_out/ profiles/ncu_traffic.json"""
import csv
import json
import sys
from pathlib import Path

SHAPES = {  # config: (decisions of one bench step, shape)
    "c2": (65536 * 10000, "65,536 streams x 10,000 steps (the default bench step)"),
    "c3": ((1 << 20) * 1000, "1,048,576 streams x 1,000 steps (the c3 bench step)"),
    "c4": (262144 * 1000, "262,144 grid scenarios x 1,000 steps (the c4 bench step, both mode launches)"),
    "c5": (262144 * 1000, "262,144 grid scenarios x 1,000 steps (the c5 bench step, both mode launches)"),
}


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    idx = {k: h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value")}
    out = {}
    for r in rows[1:]:
        k = r[idx["ID"]]
        d = out.setdefault(k, {"kernel": r[idx["Kernel Name"]]})
        v = float(r[idx["Metric Value"]].replace(",", ""))
        unit = r[idx["Metric Unit"]]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                 "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}.get(unit, 1)
        d[r[idx["Metric Name"]]] = v * scale
    return list(out.values())


def main():
    src, dst = Path(sys.argv[1]), Path(sys.argv[2])
    res = {}
    for cfg, (dec, shape) in SHAPES.items():
        p = src / f"traffic_{cfg}.csv"
        if not p.exists():
            continue
        ls = launches(p)
        rd = sum(l.get("dram__bytes_read.sum", 0) for l in ls)
        wr = sum(l.get("dram__bytes_write.sum", 0) for l in ls)
        t = sum(l.get("gpu__time_duration.sum", 0) for l in ls)
        res[cfg] = {"bytes_per_decision": round((rd + wr) / dec, 4), "algorithmic_bytes_per_decision": 4.0,
                    "shape": shape, "shape_matches_bench": True,
                    "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum ({len(ls)} run_kernel "
                              f"launch(es), serialised, cold L2): read {rd / 1e6:.1f} MB + write {wr / 1e6:.1f} MB, "
                              f"{t * 1e3:.1f} ms",
                    "kernels": sorted({l["kernel"] for l in ls})}
    dst.write_text(json.dumps(res, indent=1) + "\n")
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()

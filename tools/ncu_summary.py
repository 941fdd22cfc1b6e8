"""Summarise an ncu report (page raw) into the metrics we track."""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "duration_ns": "gpu__time_duration.sum",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "issue_active_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "ipc_active": "sm__inst_executed.avg.per_cycle_active",
    "warps_active_per_sched": "smsp__warps_active.avg.per_cycle_active",
    "warps_eligible_per_sched": "smsp__warps_eligible.avg.per_cycle_active",
    "pipe_fma_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "pipe_alu_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "pipe_xu_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "pipe_lsu_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "pipe_fp64_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "inst_executed": "smsp__inst_executed.sum",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "sm_clock_hz": "smsp__cycles_elapsed.avg.per_second",
}
STALLS = "smsp__average_warps_issue_stalled_"


def summarize(path):
    if path.endswith(".csv"):  # raw page exported on the GPU box
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, vals = rows[0], rows[2:]
    res = []
    for v in vals:
        d = dict(zip(h, v))

        def num(k):
            try:
                return float(d[k].replace(",", ""))
            except (KeyError, ValueError):
                return None

        r = {"kernel": d.get("Kernel Name", "")[:120]}
        for name, k in KEYS.items():
            r[name] = num(k)
        st = {k[len(STALLS):].replace("_per_issue_active.ratio", ""): num(k) for k in h
              if k.startswith(STALLS) and k.endswith("_per_issue_active.ratio")}
        r["stalls_per_issue"] = {k: round(x, 3) for k, x in sorted(st.items(), key=lambda kv: -(kv[1] or 0))
                                 if x and x > 0.02}
        res.append(r)
    return res


if __name__ == "__main__":
    print(json.dumps(summarize(sys.argv[1]), indent=1))

"""The GPU sweep driver (paper_1911_00119_b200.sweep) against the reference's
cmd_sweep CSV (tests/golden/golden_sweeps.json, produced by the reference's
own CLI).  CPU: the grid / normalisation / formatting logic fed with the
oracle's summaries.  GPU: the whole batched sweep, byte-identical CSV."""

import io
import json
from pathlib import Path

import numpy as np
import pytest

import paper_1911_00119_b200 as A
from paper_1911_00119_b200 import sweep as SW
from paper_1911_00119_b200.model import Mode
from paper_1911_00119_b200.records import summary_from_agg

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "golden_sweeps.json").read_text())


def _csv_text(rows, mode):
    buf = io.StringIO()
    import csv

    w = csv.writer(buf)
    w.writerow(["deadline_mult", "q_goal" if Mode(mode) is Mode.MINIMIZE_ENERGY else "e_goal_mult",
                *SW.HEADER_TAIL])
    w.writerows(rows)
    return buf.getvalue()


@pytest.mark.parametrize("case", range(len(GOLD)))
def test_sweep_rows_with_oracle_summaries(case):
    from oracle import oracle

    g = GOLD[case]
    mode = Mode(g["mode"])
    dms = [0.4, 0.8, 1.2, 1.6, 2.0]
    goals = [float(x) for x in g["goals"].split(",")]
    pols = g["policies"].split(",")
    space = A.preset_space()
    trace = SW.effective_trace(A.preset_trace(phase_length=g["phase_length"]), g["seed"])
    env = A.realize(trace)
    specs = SW.grid_specs(space, mode, dms, goals, g["pr_th"])
    summaries = {p: [summary_from_agg(oracle.run(space, s, env, p)[1], len(trace.phases)) for s in specs]
                 for p in dict.fromkeys(["oracle-static", *pols])}
    rows = SW.sweep_rows(dms, goals, specs, pols, summaries)
    assert _csv_text(rows, mode) == g["csv"].replace("\n", "\r\n") or _csv_text(rows, mode) == g["csv"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", range(len(GOLD)))
def test_gpu_sweep_csv_identical(case, tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    g = GOLD[case]
    out = tmp_path / "sweep.csv"
    argv = ["--mode", g["mode"], "--q-goals" if g["mode"] == "min-energy" else "--e-goal-mults", g["goals"],
            "--policies", g["policies"], "--phase-length", str(g["phase_length"]), "--out", str(out)]
    if g["pr_th"] is not None:
        argv += ["--pr-th", str(g["pr_th"])]
    if g["seed"] is not None:
        argv += ["--seed", str(g["seed"])]
    assert SW.main(argv) == 0
    assert out.read_text() == g["csv"]

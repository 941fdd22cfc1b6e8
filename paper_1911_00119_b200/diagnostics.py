"""Slow-down diagnostics on the GPU: ``xi_diagnostics`` (simulator.py:508-543).

xi = fb_latency / fb_t_prof per record; a 40-bin histogram and the MLE
Gaussian fit (mean, population sd).  Computed by ``alert_xi_stats`` with
numpy's own arithmetic (min/max edges, ``linspace``, the index correction of
``numpy.histogram``, pairwise summation for mean and std), so the result
equals ``numpy.histogram`` / ``numpy.mean`` / ``numpy.std`` bit for bit.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ._lib import check, load

N_BINS = 40  # simulator.py:537


@dataclass(frozen=True)
class XiDiagnostics:  # simulator.py:511-518
    values: np.ndarray
    counts: np.ndarray
    bin_edges: np.ndarray
    mean: float
    sd: float


def _stats(num, den=None, bins: int = N_BINS, device: int = 0):
    import torch

    from .simulator import get_engine

    eng = get_engine(device)
    d = eng.tdev
    a = torch.as_tensor(np.ascontiguousarray(num, np.float64)).to(d)
    b = None if den is None else torch.as_tensor(np.ascontiguousarray(den, np.float64)).to(d)
    counts = torch.empty(bins, dtype=torch.int64, device=d)
    edges = torch.empty(bins + 1, dtype=torch.float64, device=d)
    msd = torch.empty(2, dtype=torch.float64, device=d)
    check(load().alert_xi_stats(eng.ctx, a.data_ptr(), None if b is None else b.data_ptr(), a.numel(), bins,
                                counts.data_ptr(), edges.data_ptr(), msd.data_ptr(), eng._stream()))
    xi = (a / b) if b is not None else a
    m = msd.cpu().numpy()
    return xi.cpu().numpy(), counts.cpu().numpy(), edges.cpu().numpy(), float(m[0]), float(m[1])


def xi_diagnostics_from_values(xi, device: int = 0) -> XiDiagnostics:
    """simulator.py:533-543."""
    xi = np.asarray(xi, np.float64)
    if len(xi) < 30:
        raise ValueError("need at least 30 values for diagnostics")
    v, c, e, m, sd = _stats(xi, device=device)
    return XiDiagnostics(values=v, counts=c, bin_edges=e, mean=m, sd=sd)


def xi_diagnostics(records, space=None, device: int = 0) -> XiDiagnostics:
    """simulator.py:521-530: records carry fb_latency / fb_t_prof (the drop-in
    ``run`` fills them); the division happens on the GPU."""
    if len(records) < 30:
        raise ValueError("need at least 30 records for diagnostics")
    fb = np.array([r.fb_latency for r in records], np.float64)
    tp = np.array([r.fb_t_prof for r in records], np.float64)
    v, c, e, m, sd = _stats(fb, tp, device=device)
    return XiDiagnostics(values=v, counts=c, bin_edges=e, mean=m, sd=sd)

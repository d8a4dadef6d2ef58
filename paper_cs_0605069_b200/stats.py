"""Host-side statistics of the paper's experiments over decoder outputs.

Pure numpy on arrays the CUDA path returned (iteration counts, per-iteration
correct-bit traces); nothing here decodes.

* paired_ratio   -- Table 1 columns <t_SUS>, <t_PUS>, <t_SUS>/<t_PUS>,
                    <t_SUS/t_PUS>, STDEV(t_SUS/t_PUS), over the
                    frames where BOTH schedules converge (reading A29).
* delta_p_curve  -- Fig. 1: the correction gain
                    dP_t = P_{t+1} - P_t (P = percentage of correct source bits)
                    averaged per bin of the current P, for each schedule, and the
                    ratio <dP_PUS> / <dP_SUS> per bin.
"""
from __future__ import annotations

import numpy as np


def paired_ratio(t_pus, t_sus) -> dict:
    """t_pus, t_sus: int [F] iterations to convergence (-1 = none) of the same frames."""
    tp = np.asarray(t_pus, dtype=np.int64)
    ts = np.asarray(t_sus, dtype=np.int64)
    both = (tp > 0) & (ts > 0)
    out = dict(frames=int(tp.size), paired=int(both.sum()),
               nonconv_pus=int((tp < 0).sum()), nonconv_sus=int((ts < 0).sum()))
    if both.any():
        a, b = ts[both].astype(np.float64), tp[both].astype(np.float64)
        r = a / b
        out.update(mean_t_sus=float(a.mean()), mean_t_pus=float(b.mean()),
                   ratio_of_means=float(a.mean() / b.mean()), mean_ratio=float(r.mean()),
                   std_ratio=float(r.std()))
    return out


def _gains(trace, iters, nbits):
    """(P_t, dP_t) pairs of every frame while it is still decoding: transitions
    t -> t+1 with t+1 <= the frame's stopping iteration (all of them for frames
    that never converge)."""
    tr = np.asarray(trace, dtype=np.float64)
    it = np.asarray(iters, dtype=np.int64)
    F, L = tr.shape
    P = 100.0 * tr / float(nbits)
    dP = P[:, 1:] - P[:, :-1]
    t_next = np.arange(1, L)[None, :]
    stop = np.where(it > 0, it, L - 1)[:, None]
    live = t_next <= stop
    return P[:, :-1][live], dP[live]


def delta_p_curve(trace_pus, iters_pus, trace_sus, iters_sus, nbits: int, bins=None) -> dict:
    """trace_*: int [F][T+1] correct source bits of x^(t) (gfq_params.trace);
    iters_*: the decodes' iteration counts; nbits = N*p.  bins: edges in percent
    (default 20 bins over [0, 100]).  Returns per-bin mean dP of each schedule,
    sample counts and the ratio <dP_PUS>/<dP_SUS> (NaN where a bin is empty or
    the SUS mean is 0)."""
    edges = np.linspace(0.0, 100.0, 21) if bins is None else np.asarray(bins, dtype=np.float64)
    res = dict(edges=edges.tolist())
    means = {}
    for name, tr, it in (("pus", trace_pus, iters_pus), ("sus", trace_sus, iters_sus)):
        P, dP = _gains(tr, it, nbits)
        k = np.clip(np.searchsorted(edges, P, side="right") - 1, 0, len(edges) - 2)
        cnt = np.bincount(k, minlength=len(edges) - 1)
        tot = np.bincount(k, weights=dP, minlength=len(edges) - 1)
        with np.errstate(invalid="ignore", divide="ignore"):
            m = np.where(cnt > 0, tot / np.maximum(cnt, 1), np.nan)
        means[name] = m
        res["count_" + name] = cnt.tolist()
        res["mean_dP_" + name] = m.tolist()
    with np.errstate(invalid="ignore", divide="ignore"):
        ratio = np.where(np.isfinite(means["sus"]) & (means["sus"] != 0), means["pus"] / means["sus"], np.nan)
    res["ratio_pus_over_sus"] = ratio.tolist()
    return res

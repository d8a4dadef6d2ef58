"""Precision model of the check-node arithmetic (analysis tool, CPU, numpy).

A frame-batched numpy PUS decoder whose transforms run in a chosen
precision, compared with the fp64 oracle's messages after a fixed number of
iterations -- the message gate of SURVEY.md §8(d) d6 -- and, with --decide,
with the oracle's decisions / iteration counts.  It answers one design
question: which arithmetic recipe of the Walsh-Hadamard check node keeps every
message within the 1e-4 gate?

Recipes (messages are always STORED in fp32, like the GPU's message store):
  f64     q stored fp32; forward WHT, product, inverse WHT in fp64 (the round-1 kernels)
  fwd32   forward WHT in fp32, product and inverse in fp64 (GFQ_SUS_FWD32)
  F32     the variable node stores the forward transform F = WHT(perm(q)) rounded to
          fp32 instead of q; product and inverse in fp64
  F32i32  as F32, product and inverse WHT in fp32 too
  all32   every step in fp32 (q stored, forward, product, inverse, variable node)

usage: python scripts/precision_model.py C5:8 C3:16:2 C1:64 --iters 5 --recipes f64,F32,F32i32
Not test infrastructure, not product code: it imports oracle/ only to compare.
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle  # noqa: E402
import synth  # noqa: E402


def wht(x):
    """Unnormalised Walsh-Hadamard transform along the last axis, in x's dtype."""
    q = x.shape[-1]
    x = x.copy()
    h = 1
    while h < q:
        y = x.reshape(x.shape[:-1] + (q // (2 * h), 2, h))
        a, b = y[..., 0, :].copy(), y[..., 1, :].copy()
        y[..., 0, :] = a + b
        y[..., 1, :] = a - b
        x = y.reshape(x.shape)
        h *= 2
    return x


class Model:
    def __init__(self, code):
        self.code = code
        rows, cols, vals = code.H_coo()
        order = np.lexsort((rows, cols))          # canonical: column-major, then row
        self.er, self.ec, self.eh = rows[order], cols[order], vals[order].astype(np.int64)
        self.q, self.p, self.N, self.M = code.q, code.p, code.N, code.M
        self.V, self.E = code.N + code.M, len(rows)
        tab = synth.gf_tables(code.p)
        mul = tab.mul.astype(np.int64)
        inv = tab.inv.astype(np.int64)
        y = np.arange(self.q)
        # perm: qp[e][y] = q[e][h^-1 y];  unperm: r[e][x] = s[e][h x]
        self.pidx = mul[inv[self.eh]][:, y]
        self.uidx = mul[self.eh][:, y]
        # checks grouped by degree: edge ids [nc, d]
        byrow = np.argsort(self.er, kind="stable")
        deg = np.bincount(self.er, minlength=self.M)
        start = np.concatenate([[0], np.cumsum(deg)])
        self.cgroups = {}
        for d in np.unique(deg):
            ck = np.nonzero(deg == d)[0]
            self.cgroups[int(d)] = (ck, byrow[start[ck][:, None] + np.arange(d)[None, :]])
        vdeg = np.bincount(self.ec, minlength=self.V)
        vstart = np.concatenate([[0], np.cumsum(vdeg)])
        self.vgroups = {}
        for d in np.unique(vdeg):
            vs = np.nonzero(vdeg == d)[0]
            self.vgroups[int(d)] = (vs, vstart[vs][:, None] + np.arange(d)[None, :])
        # sign of the syndrome shift in the transform domain: (-1)^{popc(w & z)}
        w = np.arange(self.q)
        self.popsign = 1.0 - 2.0 * (np.array([[bin(a & b).count("1") & 1 for b in w] for a in w]))

    def check(self, qm, Fm, z, recipe):
        """r [F][E][q] from q (or stored transforms F) [F][E][q]."""
        Fn = qm.shape[0]
        r = np.zeros((Fn, self.E, self.q), np.float32)
        lo = np.float32 if recipe in ("F32i32", "all32") else np.float64
        for d, (ck, eids) in self.cgroups.items():
            if recipe in ("F32", "F32i32"):
                Fw = Fm[:, eids, :].astype(lo)                     # [F][nc][d][q]
            else:
                qp = np.take_along_axis(qm[:, eids, :], self.pidx[eids][None], axis=-1)
                if recipe in ("fwd32", "all32"):
                    Fw = wht(qp.astype(np.float32)).astype(lo)
                else:
                    Fw = wht(qp.astype(np.float64))
            sg = self.popsign[z[:, ck]].astype(lo)                # [F][nc][q]
            for t in range(d):
                P = sg.copy()
                for u in range(d):
                    if u != t:
                        P = P * Fw[:, :, u, :]
                s = wht(P) / lo(self.q)
                s = np.maximum(s, 0).astype(np.float32)            # clamp round-off, store fp32
                e = eids[:, t]
                r[:, e, :] = np.take_along_axis(s, self.uidx[e][None], axis=-1)
        return r

    def var(self, r, prior, recipe):
        """q [F][E][q] (fp32), F = WHT(perm(q)) stored fp32 (F recipes), Q [F][V][q] (fp64)."""
        Fn = r.shape[0]
        hi = np.float32 if recipe == "all32" else np.float64
        qm = np.zeros((Fn, self.E, self.q), np.float32)
        Fm = np.zeros((Fn, self.E, self.q), np.float32) if recipe in ("F32", "F32i32") else None
        Q = np.zeros((Fn, self.V, self.q))
        for d, (vs, eids) in self.vgroups.items():
            rr = r[:, eids, :].astype(hi)                          # [F][nv][d][q]
            pr = prior[:, vs, :].astype(hi)
            tot = pr * np.prod(rr, axis=2)
            Q[:, vs, :] = tot / tot.sum(-1, keepdims=True)
            for t in range(d):
                o = pr.copy()
                for u in range(d):
                    if u != t:
                        o = o * rr[:, :, u, :]
                o = o / o.sum(-1, keepdims=True)
                e = eids[:, t]
                qm[:, e, :] = o.astype(np.float32)
                if Fm is not None:
                    qp = np.take_along_axis(o.astype(np.float64), self.pidx[e][None], axis=-1)
                    Fm[:, e, :] = wht(qp).astype(np.float32)
        return qm, Fm, Q

    def decode(self, prior, z, iters, recipe, oc=None):
        Fn = prior.shape[0]
        qm = np.take(prior, self.ec, axis=1).astype(np.float32)
        Fm = None
        if recipe in ("F32", "F32i32"):
            qp = np.take_along_axis(qm.astype(np.float64), self.pidx[None], axis=-1)
            Fm = wht(qp).astype(np.float32)
        its = np.full(Fn, -1, np.int32)
        xh = None
        for t in range(1, iters + 1):
            r = self.check(qm, Fm, z, recipe)
            qm, Fm, Q = self.var(r, prior, recipe)
            if oc is not None:
                xh = np.argmax(Q, axis=-1).astype(np.uint8)
                for f in range(Fn):
                    if its[f] < 0 and oc.unsatisfied(xh[f], z[f]) == 0:
                        its[f] = t
        return qm, r, Q, its


def priors(cfg, code, fr):
    hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs)
    p, q, N, M = code.p, code.q, code.N, code.M
    pi32 = pi.astype(np.float32).astype(np.float64).reshape(fr.F, M, p)   # the GPU keeps fp32 flip probs
    bits = (np.arange(q)[:, None] >> np.arange(p)[None, :]) & 1          # [q][p]
    pn = np.prod(np.where(bits[None, None] == 1, pi32[:, :, None, :], 1 - pi32[:, :, None, :]), axis=-1)
    ps = np.full((fr.F, N, q), 1.0 / q)
    return hard, pi, np.concatenate([ps, pn], axis=1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cases", nargs="+")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--recipes", default="f64,fwd32,F32,F32i32,all32")
    args = ap.parse_args()
    for spec in args.cases:
        parts = spec.split(":")
        cfg = synth.CONFIGS[parts[0]]
        nf = int(parts[1])
        point = int(parts[2]) if len(parts) > 2 else 0
        assert cfg.source == "iid", "the model covers i.i.d. sources"
        code = synth.code_for(cfg)
        fr = synth.frames_for(cfg, code, range(nf), point=point)
        hard, pi, prior = priors(cfg, code, fr)
        oc = oracle.OCode.from_synth(code)
        rsym = synth.bits_to_symbols(hard.reshape(nf, code.M * code.p), code.p)
        z = np.stack([oc.syndrome(rsym[f]) for f in range(nf)])
        ref = oc.decode(hard, pi, schedule=oracle.PUS, max_iters=args.iters, fixed=True, keep_messages=True)
        m = Model(code)
        for rc in args.recipes.split(","):
            qm, r, Q, its = m.decode(prior, z, args.iters, rc, oc)
            out = dict(case=spec, recipe=rc, iters=args.iters,
                       iters_equal=bool(np.array_equal(its, ref["iters"])))
            for k, g in (("q", qm), ("r", r), ("Q", Q)):
                e = np.abs(g.astype(np.float64) - ref[k]).ravel()
                out[k] = dict(max=float(e.max()), p9999=float(np.percentile(e, 99.99)),
                              over_gate=int((e > 1e-4).sum()))
            print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()

"""Message-gate error distribution of a libgfq build against the fp64 oracle
(SURVEY.md §8(d) d6 message gate: fixed 5 iterations, every q, r, Q message).
Used to measure precision variants (e.g. the fp32 forward transform,
GFQ_SUS_FWD32) -- select the library with GFQ_LIB_PATH.

usage: python scripts/msg_error_dist.py C5:64 C4:40 C3:40:0 ... [--sched sus]
prints one JSON line per case: max / p99 / p99.9 / p99.99 |GPU - oracle| per
message kind, and the count of entries above the 1e-4 gate.
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle  # noqa: E402
import synth  # noqa: E402


def main():
    import torch
    from paper_cs_0605069_b200 import gfq
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    sched = 1
    if "--sched" in sys.argv:
        sched = {"pus": 0, "sus": 1}[sys.argv[sys.argv.index("--sched") + 1]]
        args = [a for a in args if a not in ("pus", "sus")]
    for spec in args:
        parts = spec.split(":")
        name, nf = parts[0], int(parts[1])
        point = int(parts[2]) if len(parts) > 2 else 0
        cfg = synth.CONFIGS[name]
        code = synth.code_for(cfg)
        fr = synth.frames_for(cfg, code, range(nf), point=point)
        T = synth.markov_T_for(cfg)
        gc = gfq.Code.from_synth(code)
        ch = {synth.BSC: gfq.GFQ_BSC, synth.BEC: gfq.GFQ_BEC, synth.BIAWGN: gfq.GFQ_BIAWGN}[fr.channel]
        prm = gfq.Params(ch, fr.ch_param, sched, 5, early_exit=False, markov_T=T, keep_messages=True)
        _, it, ws = gfq.gfq_decode(gc, torch.as_tensor(fr.obs).cuda(), prm)
        qg, rg, Qg = [x.cpu().numpy() for x in gfq.gfq_export_messages(gc, nf, ws, prm)]
        hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs)
        ref = oracle.OCode.from_synth(code).decode(hard, pi, schedule=sched, max_iters=5, fixed=True, T=T,
                                                   keep_messages=True)
        out = dict(case=spec, schedule="SUS" if sched else "PUS", lib=os.path.basename(gfq.LIB_PATH),
                   iters_equal=bool(np.array_equal(it.cpu().numpy(), ref["iters"])))
        for k, g in (("q", qg), ("r", rg), ("Q", Qg)):
            e = np.abs(g - ref[k]).ravel()
            out[k] = dict(max=float(e.max()), p99=float(np.percentile(e, 99)),
                          p999=float(np.percentile(e, 99.9)), p9999=float(np.percentile(e, 99.99)),
                          over_gate=int((e > 1e-4).sum()), n=int(e.size))
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()

"""Small decodes that exercise every hot kernel variant, for compute-sanitizer
(racecheck / synccheck / memcheck, one tool per run):

  q = 2 (C1), q = 16 (C4, Markov, BEC; the direct-convolution SUS kernel),
  q = 64 (C5 code, transform kernels with layout switches), PUS and SUS,
  ragged frame counts (a partial last 32-frame block) with early exit on,
  the in-sweep Markov prior (reading A34) and caller-supplied SUS orders (A35).

usage: python scripts/sanitize_case.py [--quick]      (exit 0 = all decodes ran)
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import synth  # noqa: E402


def main(quick: bool) -> int:
    import torch
    import __graft_entry__
    __graft_entry__.build()
    from paper_cs_0605069_b200 import gfq

    cases = [("C1", 40, 6), ("C4", 36 if quick else 45, 4), ("C5", 5 if quick else 9, 3)]
    if quick:
        cases = [c for c in cases if c[0] == "C4"]
    for name, F, iters in cases:
        cfg = synth.CONFIGS[name]
        code = synth.code_for(cfg)
        fr = synth.frames_for(cfg, code, range(F))
        gc = gfq.Code.from_synth(code)
        T = synth.markov_T_for(cfg)
        ch = {synth.BSC: gfq.GFQ_BSC, synth.BEC: gfq.GFQ_BEC, synth.BIAWGN: gfq.GFQ_BIAWGN}[fr.channel]
        obs = torch.as_tensor(fr.obs).cuda()
        runs = [dict(schedule=s, early_exit=e) for s in (0, 1) for e in (True, False)]
        if T is not None:
            runs.append(dict(schedule=1, early_exit=True, prior_update=gfq.GFQ_PRIOR_IN_SWEEP))
        if not quick:
            rng = np.random.default_rng(5)
            runs.append(dict(schedule=1, early_exit=True,
                             sus_order=np.stack([rng.permutation(code.V) for _ in range(2)]).astype(np.int32)))
        for r in runs:
            prm = gfq.Params(ch, fr.ch_param, r["schedule"], iters, early_exit=r["early_exit"], markov_T=T,
                             prior_update=r.get("prior_update", 0), sus_order=r.get("sus_order"),
                             keep_messages=not r["early_exit"])
            s_hat, it, ws = gfq.gfq_decode(gc, obs, prm)
            if not r["early_exit"]:
                gfq.gfq_export_messages(gc, F, ws, prm)
            torch.cuda.synchronize()
            print(name, {k: (v if not isinstance(v, np.ndarray) else "orders") for k, v in r.items()},
                  "iters", it.cpu().numpy()[:6].tolist(), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main("--quick" in sys.argv))

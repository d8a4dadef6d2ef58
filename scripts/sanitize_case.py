"""Small decodes that exercise every hot kernel variant, for the race / sync
check of the barrier-elided kernels (tests/test_gpu_sync_check.py: the
default build and the GFQ_SYNC_CHECK build must give bit-identical outputs;
compute-sanitizer is closed on this pool).

  q = 2 (C1), q = 8 (C3), q = 16 (C4, Markov, BEC; the direct-convolution
  SUS kernel), q = 64 (C5 code, transform kernels with layout switches),
  q = 128 (X7), PUS and SUS, ragged frame counts (a partial last 32-frame
  block) with early exit on, fixed iterations with every message exported,
  the in-sweep Markov prior (reading A34) and caller-supplied SUS orders (A35).

usage: python scripts/sanitize_case.py [--quick] [--dump OUT.npz]
(select the library with GFQ_LIB_PATH)
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import synth  # noqa: E402


def main(quick: bool, dump: str = None) -> int:
    import torch
    from paper_cs_0605069_b200 import gfq

    cases = [("C1", 40, 6), ("C3", 37, 4), ("C4", 45, 4), ("C5", 9, 3), ("X7", 5, 2)]
    if quick:
        cases = [("C4", 36, 4)]
    out = {}
    for name, F, iters in cases:
        cfg = synth.CONFIGS[name]
        code = synth.code_for(cfg)
        fr = synth.frames_for(cfg, code, range(F), point=1 if name == "C3" else 0)
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
        for k, r in enumerate(runs):
            prm = gfq.Params(ch, fr.ch_param, r["schedule"], iters if not r["early_exit"] else 3 * iters,
                             early_exit=r["early_exit"], markov_T=T,
                             prior_update=r.get("prior_update", 0), sus_order=r.get("sus_order"),
                             keep_messages=not r["early_exit"])
            s_hat, it, ws = gfq.gfq_decode(gc, obs, prm)
            tag = "%s_%d" % (name, k)
            out[tag + "_s"] = s_hat.cpu().numpy()
            out[tag + "_it"] = it.cpu().numpy()
            if not r["early_exit"]:
                qm, rm, Qm = gfq.gfq_export_messages(gc, F, ws, prm)
                out[tag + "_q"], out[tag + "_r"], out[tag + "_Q"] = qm.cpu().numpy(), rm.cpu().numpy(), Qm.cpu().numpy()
            torch.cuda.synchronize()
            print(name, {kk: (v if not isinstance(v, np.ndarray) else "orders") for kk, v in r.items()},
                  "iters", it.cpu().numpy()[:6].tolist(), flush=True)
    if dump:
        np.savez(dump, **out)
    return 0


if __name__ == "__main__":
    dump = sys.argv[sys.argv.index("--dump") + 1] if "--dump" in sys.argv else None
    sys.exit(main("--quick" in sys.argv, dump))

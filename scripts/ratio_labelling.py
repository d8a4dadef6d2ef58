"""SUS/PUS iteration ratio with B's chain in natural order (noise column k+1
follows noise column k along the chain, synth.make_code(permute_noise=False))
next to the default seeded random labelling (reading A23, d2) -- the labelling
ablation of SURVEY f2 / reading A7: SUS sweeps columns in index order, so the
labelling decides whether one sweep runs along B's chain.  C1-C5 at their given
noise (C3 at 1.5 dB), PUS and SUS on the same frames of each code, paired
statistics over frames where both converge (A29).
usage: ratio_labelling.py [frames] > rows.jsonl"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_cs_0605069_b200 import gfq, stats

nf = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
CH = {synth.BSC: gfq.GFQ_BSC, synth.BEC: gfq.GFQ_BEC, synth.BIAWGN: gfq.GFQ_BIAWGN}
for name, point in (("C1", 0), ("C2", 0), ("C3", 2), ("C4", 0), ("C5", 0)):
    cfg = synth.CONFIGS[name]
    T = synth.markov_T_for(cfg)
    for perm in (True, False):
        code = synth.code_for(cfg, permute_noise=perm)
        gc = gfq.Code.from_synth(code)
        F = min(nf, cfg.frames)
        fr = synth.frames_for(cfg, code, range(F), point=point)
        obs = torch.as_tensor(fr.obs).cuda()
        its = []
        for sch in (gfq.GFQ_PUS, gfq.GFQ_SUS):
            prm = gfq.Params(CH[fr.channel], fr.ch_param, sch, cfg.max_iters, early_exit=True, markov_T=T)
            _, it, _ = gfq.gfq_decode(gc, obs, prm)
            its.append(it.cpu().numpy())
        row = dict(config=name, noise=cfg.ch_params[point], labelling="random" if perm else "natural",
                   sus_levels=gc.sus_levels, **stats.paired_ratio(its[0], its[1]))
        print(json.dumps(row), flush=True)
        del gc
        torch.cuda.empty_cache()

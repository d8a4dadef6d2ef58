"""Which part of index order makes SUS ~2x faster than PUS: SUS with a fresh
random order every sweep that keeps the block structure (all source columns, in
random order, then all noise columns, in random order) against a fully random
order and index order (gfq_params.sus_order, reading A35).  Same frames, paired
statistics (A29).  usage: ratio_order_blocks.py [frames] > rows.jsonl"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_cs_0605069_b200 import gfq, stats

nf = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
CH = {synth.BSC: gfq.GFQ_BSC, synth.BEC: gfq.GFQ_BEC, synth.BIAWGN: gfq.GFQ_BIAWGN}
for name, point in (("C1", 0), ("C2", 0), ("C3", 2), ("C5", 0)):
    cfg = synth.CONFIGS[name]
    code = synth.code_for(cfg)
    gc = gfq.Code.from_synth(code)
    T = synth.markov_T_for(cfg)
    F = min(nf, cfg.frames)
    fr = synth.frames_for(cfg, code, range(F), point=point)
    obs = torch.as_tensor(fr.obs).cuda()
    rng = np.random.default_rng(0xB10C + cfg.cid)
    n = cfg.max_iters
    full = np.stack([rng.permutation(code.V) for _ in range(n)]).astype(np.int32)
    blocks = np.stack([np.concatenate([rng.permutation(code.N), code.N + rng.permutation(code.M)])
                       for _ in range(n)]).astype(np.int32)
    noise_first = np.stack([np.concatenate([code.N + rng.permutation(code.M), rng.permutation(code.N)])
                            for _ in range(n)]).astype(np.int32)
    its = {}
    for key, sch, order in (("pus", 0, None), ("index", 1, None), ("blocks_source_first", 1, blocks),
                            ("blocks_noise_first", 1, noise_first), ("random", 1, full)):
        prm = gfq.Params(CH[fr.channel], fr.ch_param, sch, cfg.max_iters, early_exit=True, markov_T=T,
                         sus_order=order)
        _, it, _ = gfq.gfq_decode(gc, obs, prm)
        its[key] = it.cpu().numpy()
    row = dict(config=name, noise=cfg.ch_params[point], frames=F)
    for key in ("index", "blocks_source_first", "blocks_noise_first", "random"):
        row[key] = stats.paired_ratio(its["pus"], its[key])
    print(json.dumps(row), flush=True)

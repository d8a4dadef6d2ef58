"""SUS/PUS iteration ratio when SUS visits the columns in a fresh random order
every sweep (gfq_params.sus_order, reading A35) next to the index order (A7),
on C1-C5 at their given noise (C3 at every Eb/N0 point) -- the paper's
universality claim under a different sweep order.  Same frames for all three
decodes, paired over frames where both schedules converge (reading A29).  Also
times 5 fixed sweeps of C5 (8192 frames) in both orders.
usage: ratio_sus_order.py [frames] > rows.jsonl"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_cs_0605069_b200 import gfq

nf = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 1024
time_only = "--time-only" in sys.argv
CH = {synth.BSC: gfq.GFQ_BSC, synth.BEC: gfq.GFQ_BEC, synth.BIAWGN: gfq.GFQ_BIAWGN}


def stats(tp, ts):
    both = (tp > 0) & (ts > 0)
    if not both.any():
        return dict(paired=0, nonconv_sus=int((ts < 0).sum()))
    r = ts[both] / tp[both]
    return dict(paired=int(both.sum()), mean_t_sus=float(ts[both].mean()), mean_t_pus=float(tp[both].mean()),
                ratio_of_means=float(ts[both].mean() / tp[both].mean()), mean_ratio=float(r.mean()),
                std_ratio=float(r.std()), nonconv_sus=int((ts < 0).sum()))


for name in ([] if time_only else ["C1", "C2", "C3", "C4", "C5"]):
    cfg = synth.CONFIGS[name]
    code = synth.code_for(cfg)
    gc = gfq.Code.from_synth(code)
    T = synth.markov_T_for(cfg)
    rng = np.random.default_rng(0xA35 + cfg.cid)
    orders = np.stack([rng.permutation(code.V) for _ in range(cfg.max_iters)]).astype(np.int32)
    for point in range(len(cfg.ch_params)):
        F = min(nf, cfg.frames)
        fr = synth.frames_for(cfg, code, range(F), point=point)
        obs = torch.as_tensor(fr.obs).cuda()
        its = []
        for sch, order in ((gfq.GFQ_PUS, None), (gfq.GFQ_SUS, None), (gfq.GFQ_SUS, orders)):
            prm = gfq.Params(CH[fr.channel], fr.ch_param, sch, cfg.max_iters, early_exit=True, markov_T=T,
                             sus_order=order)
            s, it, _ = gfq.gfq_decode(gc, obs, prm)
            its.append(it.cpu().numpy())
        row = dict(config=name, channel=synth.CHANNEL_NAMES[cfg.channel], q=cfg.q, source=cfg.source,
                   noise=cfg.ch_params[point], frames=F, nonconv_pus=int((its[0] < 0).sum()),
                   sus_index_order=stats(its[0], its[1]), sus_random_order=stats(its[0], its[2]))
        print(json.dumps(row), flush=True)

import gc as _gc
_gc.collect()
torch.cuda.empty_cache()
cfg = synth.CONFIGS["C5"]
code = synth.code_for(cfg)
gc = gfq.Code.from_synth(code)
F = cfg.frames
fr = synth.frames_for(cfg, code, range(1024))
obs = torch.as_tensor(np.tile(fr.obs, (F // 1024, 1))).cuda()
rng = np.random.default_rng(7)
orders = np.stack([rng.permutation(code.V) for _ in range(5)]).astype(np.int32)
out = dict(config="C5", frames=F, iters=5)
for key, order in (("ms_index_order", None), ("ms_random_order", orders)):
    prm = gfq.Params(CH[fr.channel], fr.ch_param, gfq.GFQ_SUS, 5, early_exit=False, sus_order=order)
    ws = gfq.alloc_workspace(gfq.gfq_workspace_bytes(gc, F, prm))
    s_hat = torch.empty((F, code.N), dtype=torch.uint8, device="cuda")
    it = torch.empty(F, dtype=torch.int32, device="cuda")
    gfq.gfq_decode(gc, obs, prm, s_hat, it, ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    gfq.gfq_decode(gc, obs, prm, s_hat, it, ws)
    e1.record()
    torch.cuda.synchronize()
    out[key] = e0.elapsed_time(e1)
    del ws, s_hat, it
    torch.cuda.empty_cache()
print(json.dumps(out), flush=True)

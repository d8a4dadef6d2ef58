"""Per-kernel timing of fixed-iteration decodes: kbench.py CONFIG FRAMES ITERS [schedules]"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_cs_0605069_b200 import gfq

name, nf, iters = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
scheds = sys.argv[4].split(",") if len(sys.argv) > 4 else ["pus", "sus"]
cfg = synth.CONFIGS[name]
code = synth.code_for(cfg)
fr = synth.frames_for(cfg, code, range(nf))
gc = gfq.Code.from_synth(code)
ch = {synth.BSC: gfq.GFQ_BSC, synth.BEC: gfq.GFQ_BEC, synth.BIAWGN: gfq.GFQ_BIAWGN}[fr.channel]
T = synth.markov_T_for(cfg)
obs = torch.as_tensor(fr.obs).cuda()
out = {"lib": os.path.basename(gfq.LIB_PATH), "config": name, "frames": nf, "iters": iters}
for sname in scheds:
    sch = gfq.GFQ_PUS if sname == "pus" else gfq.GFQ_SUS
    prm = gfq.Params(ch, fr.ch_param, sch, iters, early_exit=False, markov_T=T)
    s, it, ws = gfq.gfq_decode(gc, obs, prm)   # warm-up
    torch.cuda.synchronize()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record()
    gfq.gfq_decode(gc, obs, prm, s, it, ws)     # clean: no per-launch events
    c1.record()
    torch.cuda.synchronize()
    clean = c0.elapsed_time(c1)
    gfq.gfq_profile_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    gfq.gfq_decode(gc, obs, prm, s, it, ws)
    e1.record()
    torch.cuda.synchronize()
    gfq.gfq_profile_enable(False)
    prof = gfq.gfq_profile_read()
    tot = e0.elapsed_time(e1)
    per_iter_bytes = 16.0 * cfg.E * cfg.q * nf   # model bytes per iteration (8q per edge-message update, 2E updates)
    k = {kk: round(v[0] / max(v[1], 1), 4) for kk, v in prof.items() if v[1] > 0}
    main = prof["cn"][0] + prof["vn"][0] if sch == gfq.GFQ_PUS else prof["sus"][0]
    out[sname] = dict(total_ms=round(tot, 2), clean_total_ms=round(clean, 2),
                      clean_model_GBps=round(per_iter_bytes * iters / (clean / 1e3) / 1e9, 1), ms_per_iter=round(main / iters, 3),
                      model_GBps=round(per_iter_bytes * iters / (main / 1e3) / 1e9, 1),
                      per_launch_ms=k, zero_norm=gfq.gfq_decode_stats(gc, ws)["zero_normalisers"])
print(json.dumps(out))

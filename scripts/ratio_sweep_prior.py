"""SUS/PUS iteration ratio with the Markov prior refreshed inside the SUS sweep
(GFQ_PRIOR_IN_SWEEP, reading A34) next to the post-iteration
snapshot prior (A9), on the Markov configurations C2 and C4 at their given
noise and at the supplementary near-threshold points of DESIGN.md §13.
Same frames for all three decodes; paired statistics over frames where both
schedules converge (reading A29).  Also times a fixed-iteration decode of each
SUS variant at the config's full frame count (the in-sweep variant runs ~N
dependency levels per sweep instead of ~13).
usage: ratio_sweep_prior.py [frames] > rows.jsonl"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_cs_0605069_b200 import gfq

nf = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 1024
time_only = "--time-only" in sys.argv
POINTS = [("C2", None), ("C2", 0.1698), ("C4", None), ("C4", 0.6957)]


def decode(gc, obs, ch, param, sch, prior, T, max_iters, early=True):
    prm = gfq.Params(ch, param, sch, max_iters, early_exit=early, markov_T=T, prior_update=prior)
    s, it, ws = gfq.gfq_decode(gc, obs, prm)
    return s.cpu().numpy(), it.cpu().numpy()


def stats(tp, ts):
    both = (tp > 0) & (ts > 0)
    if not both.any():
        return dict(paired=0)
    r = ts[both] / tp[both]
    return dict(paired=int(both.sum()), mean_t_sus=float(ts[both].mean()), mean_t_pus=float(tp[both].mean()),
                ratio_of_means=float(ts[both].mean() / tp[both].mean()), mean_ratio=float(r.mean()),
                std_ratio=float(r.std()), nonconv_sus=int((ts < 0).sum()))


for name, noise in ([] if time_only else POINTS):
    cfg = synth.CONFIGS[name]
    code = synth.code_for(cfg)
    gc = gfq.Code.from_synth(code)
    T = synth.markov_T_for(cfg)
    F = min(nf, cfg.frames)
    if noise is None:
        fr = synth.frames_for(cfg, code, range(F))
    else:
        fr = synth.make_frames(code, cfg.cid, range(F), cfg.source, cfg.channel, noise, stay=cfg.stay, point=99)
    ch = {synth.BSC: gfq.GFQ_BSC, synth.BEC: gfq.GFQ_BEC, synth.BIAWGN: gfq.GFQ_BIAWGN}[fr.channel]
    obs = torch.as_tensor(fr.obs).cuda()
    sp, tp = decode(gc, obs, ch, fr.ch_param, gfq.GFQ_PUS, 0, T, cfg.max_iters)
    ss, ts = decode(gc, obs, ch, fr.ch_param, gfq.GFQ_SUS, 0, T, cfg.max_iters)
    sg, tg = decode(gc, obs, ch, fr.ch_param, gfq.GFQ_SUS, 1, T, cfg.max_iters)
    row = dict(config=name + ("" if noise is None else "-near-threshold"), channel=synth.CHANNEL_NAMES[cfg.channel],
               q=cfg.q, noise=fr.ch_param, frames=F, nonconv_pus=int((tp < 0).sum()),
               sus_snapshot=stats(tp, ts), sus_in_sweep=stats(tp, tg),
               ser_pus=float((sp != fr.s).mean()), ser_sus_snapshot=float((ss != fr.s).mean()),
               ser_sus_in_sweep=float((sg != fr.s).mean()))
    print(json.dumps(row), flush=True)

# cost of the in-sweep prior: fixed 5 iterations at the full frame count
for name in ["C2", "C4"]:
    cfg = synth.CONFIGS[name]
    code = synth.code_for(cfg)
    gc = gfq.Code.from_synth(code)
    T = synth.markov_T_for(cfg)
    F = cfg.frames
    fr = synth.frames_for(cfg, code, range(min(F, 1024)))
    reps = (F + fr.F - 1) // fr.F
    obs = torch.as_tensor(np.tile(fr.obs, (reps, 1))[:F]).cuda()
    ch = {synth.BSC: gfq.GFQ_BSC, synth.BEC: gfq.GFQ_BEC, synth.BIAWGN: gfq.GFQ_BIAWGN}[fr.channel]
    out = dict(config=name, frames=F, iters=5)
    for prior in (0, 1):
        prm = gfq.Params(ch, fr.ch_param, gfq.GFQ_SUS, 5, early_exit=False, markov_T=T, prior_update=prior)
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
        out["ms_snapshot" if prior == 0 else "ms_in_sweep"] = e0.elapsed_time(e1)
    print(json.dumps(out), flush=True)

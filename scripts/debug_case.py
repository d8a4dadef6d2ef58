"""Debug helper: run one decode config on the GPU and compare with the oracle."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, oracle
import __graft_entry__
__graft_entry__.build()
from paper_cs_0605069_b200 import gfq

name = sys.argv[1]; nf = int(sys.argv[2]); sched = int(sys.argv[3]); early = int(sys.argv[4])
maxit = int(sys.argv[5]) if len(sys.argv) > 5 else 0
point = int(sys.argv[6]) if len(sys.argv) > 6 else 0
cfg = synth.CONFIGS[name]
code = synth.code_for(cfg)
fr = synth.frames_for(cfg, code, range(nf), point=point)
T = synth.markov_T_for(cfg)
gc = gfq.Code.from_synth(code)
ch = {synth.BSC: gfq.GFQ_BSC, synth.BEC: gfq.GFQ_BEC, synth.BIAWGN: gfq.GFQ_BIAWGN}[fr.channel]
mi = maxit or cfg.max_iters
prm = gfq.Params(ch, fr.ch_param, sched, mi, early_exit=bool(early), markov_T=T)
obs = torch.as_tensor(fr.obs).cuda()
t0 = time.time()
try:
    s, it, ws = gfq.gfq_decode(gc, obs, prm)
    torch.cuda.synchronize()
except Exception as e:
    print("GPU decode failed:", e); sys.exit(1)
print("gpu ok %.2fs" % (time.time() - t0), gfq.gfq_decode_stats(gc, ws))
s = s.cpu().numpy(); it = it.cpu().numpy()
if len(sys.argv) > 7:
    oc = oracle.OCode.from_synth(code)
    hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs)
    ref = oc.decode(hard, pi, schedule=sched, max_iters=mi, T=T, fixed=not early)
    for f in range(nf):
        d = int((s[f] != ref["xhat"][f, :code.N]).sum())
        if d or it[f] != ref["iters"][f]:
            print("frame", f, "gpu it", it[f], "ref it", ref["iters"][f], "sym diffs", d,
                  "gpu err vs truth", int((s[f] != fr.s[f]).sum()), "ref err vs truth", int((ref["xhat"][f, :code.N] != fr.s[f]).sum()))

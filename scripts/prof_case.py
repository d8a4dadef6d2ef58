"""Run one fixed-iteration decode (for ncu captures): prof_case.py CONFIG FRAMES SCHEDULE ITERS [POINT]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_cs_0605069_b200 import gfq

name, nf, sched, iters = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
point = int(sys.argv[5]) if len(sys.argv) > 5 else 0
cfg = synth.CONFIGS[name]
code = synth.code_for(cfg)
fr = synth.frames_for(cfg, code, range(nf), point=point)
gc = gfq.Code.from_synth(code)
ch = {synth.BSC: gfq.GFQ_BSC, synth.BEC: gfq.GFQ_BEC, synth.BIAWGN: gfq.GFQ_BIAWGN}[fr.channel]
prm = gfq.Params(ch, fr.ch_param, sched, iters, early_exit=False, markov_T=synth.markov_T_for(cfg))
obs = torch.as_tensor(fr.obs).cuda()
free, _ = torch.cuda.mem_get_info()
ws = gfq.alloc_workspace(min(gfq.gfq_workspace_bytes(gc, nf, prm), free - (3 << 30)))
s, it, ws = gfq.gfq_decode(gc, obs, prm, workspace=ws)
torch.cuda.synchronize()
print("ok", name, nf, sched, iters, gfq.gfq_decode_stats(gc, ws))

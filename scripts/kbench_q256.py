"""Timing of the q = 256 streaming kernels (csrc/gfq_bigq.cu): a seeded MN code
over GF(256) (N = 2000, M = 4000, the C2 shape), i.i.d. source, BI-AWGN, frames
from the device front end, fixed iterations.  usage: kbench_q256.py [FRAMES] [ITERS]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_cs_0605069_b200 import gfq

synth.PRIM_POLY.setdefault(8, 0x11D)       # x^8+x^4+x^3+x^2+1 (tests/conftest.py registers the same)
nf = int(sys.argv[1]) if len(sys.argv) > 1 else 512
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
N, M, q = 2000, 4000, 256
code = synth.make_code(8, N, M, 0x256)
gc = gfq.Code.from_synth(code)
sigma = 0.75
s, obs, _ = gfq.gfq_simulate(gc, nf, 0x256256, gfq.GFQ_BIAWGN, sigma)
out = {"q": q, "N": N, "M": M, "E": gc.E, "frames": nf, "iters": iters}
for name, sch in (("pus", gfq.GFQ_PUS), ("sus", gfq.GFQ_SUS)):
    prm = gfq.Params(gfq.GFQ_BIAWGN, sigma, sch, iters, early_exit=False)
    sh, it, ws = gfq.gfq_decode(gc, obs, prm)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); gfq.gfq_decode(gc, obs, prm, sh, it, ws); e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    out[name] = dict(ms_per_iter=round(ms / iters, 3),
                     model_GBps=round(16.0 * gc.E * q * nf * iters / (ms / 1e3) / 1e9, 1))
    pc = gfq.Params(gfq.GFQ_BIAWGN, sigma, sch, 100, early_exit=True)
    sh, it, ws = gfq.gfq_decode(gc, obs, pc)
    out[name]["converged"] = int((it > 0).sum()); out[name]["mean_iters"] = round(float(it[it > 0].float().mean()), 2)
    out[name]["frame_errors"] = int((sh != s).any(dim=1).sum())
print(json.dumps(out))

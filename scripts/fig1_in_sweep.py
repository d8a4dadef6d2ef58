"""Fig. 1 of the GF(8) 2-state-source BSC row at its calibrated noise
(scripts/paper_table1.py, profiles/r01b/paper_table1.jsonl) with SUS using the
Markov prior refreshed inside the sweep (A34) against PUS: per 5 % bin of the
fraction P of correct source bits, <dP_PUS>/<dP_SUS> over the transitions of
frames still decoding (reading A32).  usage: fig1_in_sweep.py [frames] > out.json"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from paper_cs_0605069_b200 import gfq, stats  # noqa: E402

nf = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
MAX_IT = 400
prev = [json.loads(l) for l in open(os.path.join(ROOT, "profiles", "r01b", "paper_table1.jsonl"))]
noise = next(r["noise"] for r in prev if r["channel"] == "bsc" and r["q"] == 8 and r["noise_kind"] == "calibrated")
k, p = 2, 3                                   # ROWS index of ("bsc", 3, "2S", 0.230) in paper_table1.py
N = 3333
code = synth.make_code(p, N, 3 * N, 0x7AB1E000 + k)
gc = gfq.Code.from_synth(code)
T = synth.markov_embed_binary(synth.MARKOV_2S, p)
pi0 = synth.stationary(T)
fr = synth.make_frames(code, 100 + k, range(nf), "markov_T", synth.BSC, noise, point=0, T=T)
obs = torch.as_tensor(fr.obs).cuda()
truth = torch.as_tensor(fr.s).cuda()
res = {}
for key, sch, prior in (("pus", gfq.GFQ_PUS, 0), ("sus_snapshot", gfq.GFQ_SUS, 0), ("sus_in_sweep", gfq.GFQ_SUS, 1)):
    tr = torch.zeros((nf, MAX_IT + 1), dtype=torch.int32, device="cuda")
    prm = gfq.Params(gfq.GFQ_BSC, noise, sch, MAX_IT, early_exit=True, markov_T=T, src_pi0=pi0,
                     trace_truth=truth, trace=tr, prior_update=prior)
    _, it, _ = gfq.gfq_decode(gc, obs, prm)
    res[key] = (tr.cpu().numpy(), it.cpu().numpy())
out = dict(noise=noise, frames=nf)
for key in ("sus_snapshot", "sus_in_sweep"):
    c = stats.delta_p_curve(res["pus"][0], res["pus"][1], res[key][0], res[key][1], nbits=N * p)
    out[key] = dict(ratio_pus_over_sus=c["ratio_pus_over_sus"], count_sus=c["count_sus"],
                    **stats.paired_ratio(res["pus"][1], res[key][1]))
out["edges"] = c["edges"]
print(json.dumps(out))

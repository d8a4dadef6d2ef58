"""The Markov rows of the paper's Table 1 grid (GF(4) with the
4-state source, GF(8) with the 2-state source read 3 bits per symbol) with the
Markov prior refreshed inside the SUS sweep (GFQ_PRIOR_IN_SWEEP, reading A34)
next to the post-iteration snapshot (A9).  Same construction, seeds and noise
levels as scripts/paper_table1.py (the calibrated levels are read from its
output), PUS and both SUS variants on the same frames, paired statistics over
frames where both schedules converge (A29).
usage: paper_table1_in_sweep.py [frames] > out.jsonl"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_cs_0605069_b200 import gfq, stats  # noqa: E402

nf = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
MAX_IT = 400
CH = {"bsc": synth.BSC, "bec": synth.BEC, "biawgn": synth.BIAWGN}
GCH = {synth.BSC: gfq.GFQ_BSC, synth.BEC: gfq.GFQ_BEC, synth.BIAWGN: gfq.GFQ_BIAWGN}
ROWS = [("bsc", 1, "iid", 0.155), ("bsc", 2, "4S", 0.227), ("bsc", 3, "2S", 0.230),
        ("bec", 1, "iid", 0.58), ("bec", 2, "4S", 0.78), ("bec", 3, "2S", 0.76),
        ("biawgn", 1, "iid", 0.98), ("biawgn", 2, "4S", 1.64), ("biawgn", 3, "2S", 1.66)]
prev = [json.loads(l) for l in open(os.path.join(ROOT, "profiles", "r01b", "paper_table1.jsonl"))]


def source_T(p, src):
    if src == "4S":
        return synth.MARKOV_4S / synth.MARKOV_4S.sum(axis=1, keepdims=True)
    return synth.markov_embed_binary(synth.MARKOV_2S, p)


for k, (chn, p, src, paper) in enumerate(ROWS):
    if src == "iid":
        continue
    N = 10000 // p if p != 3 else 3333
    code = synth.make_code(p, N, 3 * N, 0x7AB1E000 + k)
    gc = gfq.Code.from_synth(code)
    T = source_T(p, src)
    pi0 = synth.stationary(T)
    for label in ("paper", "calibrated"):
        noise = next(r["noise"] for r in prev if r["channel"] == chn and r["q"] == 1 << p
                     and r["noise_kind"] == label)
        fr = synth.make_frames(code, 100 + k, range(nf), "markov_T", CH[chn], noise, point=0, T=T)
        obs = torch.as_tensor(fr.obs).cuda()
        its = []
        for sch, prior in ((gfq.GFQ_PUS, 0), (gfq.GFQ_SUS, 0), (gfq.GFQ_SUS, 1)):
            prm = gfq.Params(GCH[CH[chn]], noise, sch, MAX_IT, early_exit=True, markov_T=T, src_pi0=pi0,
                             prior_update=prior)
            s, it, _ = gfq.gfq_decode(gc, obs, prm)
            its.append(it.cpu().numpy())
        row = dict(channel=chn, q=1 << p, source=src, N=N, noise_kind=label, noise=noise,
                   sus_snapshot=stats.paired_ratio(its[0], its[1]), sus_in_sweep=stats.paired_ratio(its[0], its[2]))
        print(json.dumps(row), flush=True)

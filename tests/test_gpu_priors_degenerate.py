"""GPU parity for non-uniform source priors and the channels' degenerate cases,
against the oracle on the same seeded inputs:
  * the paper's 4-state source on GF(4) with its stationary law as
    pi0 -- PUS, SUS and the in-sweep prior (A34) -- and an i.i.d.
    source with a skewed pi0 (the prior of every source symbol);
  * noiseless channels (BSC f = 0, BEC eps = 0): point-mass noise priors (exact
    zeros in every message); the sources are then determined by A s = z + B n
    and peeled in a few iterations -- every frame decodes to the truth, at the
    oracle's iteration;
  * the erase-everything BEC (eps = 1): no evidence at all; the hard bits are
    all 0 (A15), so z = 0, and the uniform posteriors clip to the all-zero
    estimate (tie rule A17), which satisfies H x = 0 -- both sides report it.
Gates as tests/test_gpu_parity.py."""
import numpy as np
import pytest

import gate
import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

MSG_TOL = 1e-4


@pytest.fixture(scope="module")
def gfq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    from paper_cs_0605069_b200 import gfq as g
    return g


def _T4S():
    return synth.MARKOV_4S / synth.MARKOV_4S.sum(axis=1, keepdims=True)


CH = {synth.BSC: 0, synth.BEC: 1, synth.BIAWGN: 2}


@pytest.mark.parametrize("schedule,prior", [(0, 0), (1, 0), (1, 1)], ids=["PUS", "SUS", "SUS-in-sweep"])
def test_paper_4state_source_with_stationary_pi0(gfq, schedule, prior):
    code = synth.make_code(2, 400, 1200, 0x45)             # rate 1/3 as the paper's grid
    T = _T4S()
    pi0 = synth.stationary(T)
    assert pi0.max() > 0.5                                  # really non-uniform (App. A: 0.762)
    fr = synth.make_frames(code, 21, range(45), "markov_T", synth.BSC, 0.2, T=T)
    gcode = gfq.Code.from_synth(code)
    oc = oracle.OCode.from_synth(code)
    hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs)
    prm = gfq.Params(gfq.GFQ_BSC, fr.ch_param, schedule, 5, early_exit=False, keep_messages=True, markov_T=T,
                     src_pi0=pi0, prior_update=prior)
    _, it, ws = gfq.gfq_decode(gcode, torch.as_tensor(fr.obs).cuda(), prm)
    qg, rg, Qg = (x.cpu().numpy() for x in gfq.gfq_export_messages(gcode, fr.F, ws, prm))
    ref = oc.decode(hard, pi, schedule=schedule, max_iters=5, fixed=True, T=T, pi0=pi0, keep_messages=True,
                    sus_gs=bool(prior))
    errs = {k: float(np.max(np.abs(g - ref[k]))) for k, g in (("q", qg), ("r", rg), ("Q", Qg))}
    assert max(errs.values()) <= MSG_TOL, errs
    assert np.array_equal(it.cpu().numpy(), ref["iters"])
    # decisions with early exit
    prm = gfq.Params(gfq.GFQ_BSC, fr.ch_param, schedule, 150, markov_T=T, src_pi0=pi0, prior_update=prior)
    s, it, _ = gfq.gfq_decode(gcode, torch.as_tensor(fr.obs).cuda(), prm)
    ref = oc.decode(hard, pi, schedule=schedule, max_iters=150, T=T, pi0=pi0, sus_gs=bool(prior))
    s, it = s.cpu().numpy(), it.cpu().numpy()
    def oq(idx):
        o = oc.decode(hard[idx], pi[idx], schedule=schedule, max_iters=150, T=T, pi0=pi0, sus_gs=bool(prior),
                      keep_messages=True)
        return o["xhat"][:, :code.N], o["Q"][:, :code.N]
    ok, strict, n_allow = gate.decision_gate(s, it, ref["xhat"][:, :code.N], ref["iters"], oq)
    gate.record("4S stationary %s prior %d" % ("SUS" if schedule else "PUS", prior), len(ok), ok, strict, n_allow)
    assert ok.all()


@pytest.mark.parametrize("schedule", [0, 1], ids=["PUS", "SUS"])
def test_iid_source_with_skewed_pi0(gfq, schedule):
    code = synth.make_code(3, 300, 600, 0x46)
    rng = np.random.default_rng(3)
    pi0 = rng.random(8) ** 3
    pi0 /= pi0.sum()
    fr = synth.make_frames(code, 22, range(40), "iid", synth.BIAWGN, 0.8)
    gcode = gfq.Code.from_synth(code)
    prm = gfq.Params(gfq.GFQ_BIAWGN, fr.ch_param, schedule, 5, early_exit=False, keep_messages=True, src_pi0=pi0)
    _, it, ws = gfq.gfq_decode(gcode, torch.as_tensor(fr.obs).cuda(), prm)
    qg, rg, Qg = (x.cpu().numpy() for x in gfq.gfq_export_messages(gcode, fr.F, ws, prm))
    hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs)
    ref = oracle.OCode.from_synth(code).decode(hard, pi, schedule=schedule, max_iters=5, fixed=True, pi0=pi0,
                                               keep_messages=True)
    errs = {k: float(np.max(np.abs(g - ref[k]))) for k, g in (("q", qg), ("r", rg), ("Q", Qg))}
    assert max(errs.values()) <= MSG_TOL, errs


@pytest.mark.parametrize("channel", [synth.BSC, synth.BEC])
@pytest.mark.parametrize("schedule", [0, 1], ids=["PUS", "SUS"])
def test_noiseless_channel_decodes_to_truth(gfq, channel, schedule):
    cfg = synth.CONFIGS["C3"]
    code = synth.code_for(cfg)
    fr = synth.make_frames(code, 23, range(40), "iid", channel, 0.0)
    gcode = gfq.Code.from_synth(code)
    prm = gfq.Params(CH[channel], 0.0, schedule, 20)
    s, it, ws = gfq.gfq_decode(gcode, torch.as_tensor(fr.obs).cuda(), prm)
    s, it = s.cpu().numpy(), it.cpu().numpy()
    assert (it > 0).all() and np.array_equal(s, fr.s)
    assert gfq.gfq_decode_stats(gcode, ws)["zero_normalisers"] == 0
    hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs)
    ref = oracle.OCode.from_synth(code).decode(hard, pi, schedule=schedule, max_iters=20)
    assert np.array_equal(ref["iters"], it) and np.array_equal(ref["xhat"][:, :code.N], fr.s)


@pytest.mark.parametrize("schedule", [0, 1], ids=["PUS", "SUS"])
def test_everything_erased(gfq, schedule):
    cfg = synth.CONFIGS["C2"]
    code = synth.code_for(cfg)
    fr = synth.make_frames(code, 24, range(33), "iid", synth.BEC, 1.0)
    assert (fr.obs == 2).all()
    gcode = gfq.Code.from_synth(code)
    prm = gfq.Params(gfq.GFQ_BEC, 1.0, schedule, 10)
    s, it, ws = gfq.gfq_decode(gcode, torch.as_tensor(fr.obs).cuda(), prm)
    hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs)
    ref = oracle.OCode.from_synth(code).decode(hard, pi, schedule=schedule, max_iters=10)
    assert np.array_equal(it.cpu().numpy(), ref["iters"])
    assert np.array_equal(s.cpu().numpy(), ref["xhat"][:, :code.N])
    assert gfq.gfq_decode_stats(gcode, ws)["zero_normalisers"] == 0

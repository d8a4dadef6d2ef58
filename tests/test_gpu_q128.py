"""GF(128) (p = 7, x^7 + x^3 + 1): the same kernels instantiated with
16 entries per thread and 8 warps per q-vector (the two register layouts of
the transform then cover all 7 bits), one group per CTA.  Parity against the
oracle on a small MN code, both schedules, on the same seeded inputs and gates
as tests/test_gpu_parity.py.  With a Markov source the q x q transition tiles
(128 KB) are read through L1 instead of shared memory."""
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


@pytest.fixture(scope="module")
def code128():
    return synth.make_code(7, 200, 400, 0x128)


def _frames(code, n, sigma):
    return synth.make_frames(code, 12, range(n), "iid", synth.BIAWGN, sigma)


@pytest.mark.parametrize("schedule", [0, 1], ids=["PUS", "SUS"])
def test_q128_message_gate(gfq, code128, schedule):
    fr = _frames(code128, 45, 0.85)                 # two 32-frame blocks, ragged
    gcode = gfq.Code.from_synth(code128)
    prm = gfq.Params(gfq.GFQ_BIAWGN, fr.ch_param, schedule, 5, early_exit=False, keep_messages=True)
    s_hat, it, ws = gfq.gfq_decode(gcode, torch.as_tensor(fr.obs).cuda(), prm)
    qg, rg, Qg = (x.cpu().numpy() for x in gfq.gfq_export_messages(gcode, fr.F, ws, prm))
    oc = oracle.OCode.from_synth(code128)
    hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs)
    ref = oc.decode(hard, pi, schedule=schedule, max_iters=5, fixed=True, keep_messages=True)
    errs = {k: float(np.max(np.abs(g - ref[k]))) for k, g in (("q", qg), ("r", rg), ("Q", Qg))}
    print("q=128", "PUS" if schedule == 0 else "SUS", errs)
    assert max(errs.values()) <= MSG_TOL, errs
    assert np.array_equal(it.cpu().numpy(), ref["iters"])
    assert gfq.gfq_decode_stats(gcode, ws)["zero_normalisers"] == 0


@pytest.mark.parametrize("schedule", [0, 1], ids=["PUS", "SUS"])
def test_q128_decision_gate(gfq, code128, schedule):
    fr = _frames(code128, 64, 0.8)
    gcode = gfq.Code.from_synth(code128)
    prm = gfq.Params(gfq.GFQ_BIAWGN, fr.ch_param, schedule, 60, early_exit=True)
    s_hat, it, ws = gfq.gfq_decode(gcode, torch.as_tensor(fr.obs).cuda(), prm)
    s_hat, it = s_hat.cpu().numpy(), it.cpu().numpy()
    oc = oracle.OCode.from_synth(code128)
    hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs)
    ref = oc.decode(hard, pi, schedule=schedule, max_iters=60)
    def oq(idx):
        o = oc.decode(hard[idx], pi[idx], schedule=schedule, max_iters=60, keep_messages=True)
        return o["xhat"][:, :code128.N], o["Q"][:, :code128.N]
    match, strict, n_allow = gate.decision_gate(s_hat, it, ref["xhat"][:, :code128.N], ref["iters"], oq)
    assert gate.record("q=128 %s" % ("SUS" if schedule else "PUS"), fr.F, match, strict, n_allow) == 0
    assert (it > 0).mean() > 0.5


@pytest.mark.parametrize("schedule,prior", [(0, 0), (1, 0), (1, 1)], ids=["PUS", "SUS", "SUS-in-sweep"])
def test_q128_markov_message_gate(gfq, code128, schedule, prior):
    T = synth.markov_uniform_jump(128, 0.7)
    fr = synth.make_frames(code128, 13, range(33), "markov", synth.BSC, 0.08, stay=0.7)
    gcode = gfq.Code.from_synth(code128)
    prm = gfq.Params(gfq.GFQ_BSC, fr.ch_param, schedule, 5, early_exit=False, keep_messages=True, markov_T=T,
                     prior_update=prior)
    s_hat, it, ws = gfq.gfq_decode(gcode, torch.as_tensor(fr.obs).cuda(), prm)
    qg, rg, Qg = (x.cpu().numpy() for x in gfq.gfq_export_messages(gcode, fr.F, ws, prm))
    oc = oracle.OCode.from_synth(code128)
    hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs)
    ref = oc.decode(hard, pi, schedule=schedule, max_iters=5, fixed=True, keep_messages=True, T=T,
                    sus_gs=bool(prior))
    errs = {k: float(np.max(np.abs(g - ref[k]))) for k, g in (("q", qg), ("r", rg), ("Q", Qg))}
    print("q=128 Markov", schedule, prior, errs)
    assert max(errs.values()) <= MSG_TOL, errs
    assert np.array_equal(it.cpu().numpy(), ref["iters"])


def test_q128_simulate_then_decode(gfq, code128):
    """Device Monte-Carlo front end at q = 128 feeding the decoder: at a high SNR
    every frame decodes to the simulated source."""
    gcode = gfq.Code.from_synth(code128)
    s, obs, _ = gfq.gfq_simulate(gcode, 64, 0x5EED, gfq.GFQ_BIAWGN, 0.6)
    prm = gfq.Params(gfq.GFQ_BIAWGN, 0.6, 1, 50)
    s_hat, it, _ = gfq.gfq_decode(gcode, obs, prm)
    assert torch.equal(s_hat.cpu(), s.cpu())
    assert bool((it > 0).all())

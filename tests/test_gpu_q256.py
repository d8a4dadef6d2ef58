"""GF(256) (p = 8, x^8 + x^4 + x^3 + x^2 + 1): the streaming kernels
of csrc/gfq_bigq.cu (one CTA per task, the messages of a check transformed one
at a time into a running product, 32 entries per thread).  Parity against the
oracle on a small MN code, both schedules, on the same seeded inputs and gates
as tests/test_gpu_parity.py; Markov source (snapshot and in-sweep prior), early
exit with frame compaction, the device Monte-Carlo front end."""
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
def code256():
    return synth.make_code(8, 120, 240, 0x256)


def _frames(code, n, sigma):
    return synth.make_frames(code, 12, range(n), "iid", synth.BIAWGN, sigma)


@pytest.mark.parametrize("schedule", [0, 1], ids=["PUS", "SUS"])
def test_q256_message_gate(gfq, code256, schedule):
    fr = _frames(code256, 45, 0.85)                 # two 32-frame blocks, ragged
    gcode = gfq.Code.from_synth(code256)
    prm = gfq.Params(gfq.GFQ_BIAWGN, fr.ch_param, schedule, 5, early_exit=False, keep_messages=True)
    s_hat, it, ws = gfq.gfq_decode(gcode, torch.as_tensor(fr.obs).cuda(), prm)
    qg, rg, Qg = (x.cpu().numpy() for x in gfq.gfq_export_messages(gcode, fr.F, ws, prm))
    oc = oracle.OCode.from_synth(code256)
    hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs)
    ref = oc.decode(hard, pi, schedule=schedule, max_iters=5, fixed=True, keep_messages=True)
    errs = {k: float(np.max(np.abs(g - ref[k]))) for k, g in (("q", qg), ("r", rg), ("Q", Qg))}
    print("q=256", "PUS" if schedule == 0 else "SUS", errs)
    assert max(errs.values()) <= MSG_TOL, errs
    assert np.array_equal(it.cpu().numpy(), ref["iters"])
    assert gfq.gfq_decode_stats(gcode, ws)["zero_normalisers"] == 0


@pytest.mark.parametrize("schedule", [0, 1], ids=["PUS", "SUS"])
def test_q256_decision_gate(gfq, code256, schedule):
    fr = _frames(code256, 64, 0.8)
    gcode = gfq.Code.from_synth(code256)
    prm = gfq.Params(gfq.GFQ_BIAWGN, fr.ch_param, schedule, 60, early_exit=True)
    s_hat, it, ws = gfq.gfq_decode(gcode, torch.as_tensor(fr.obs).cuda(), prm)
    s_hat, it = s_hat.cpu().numpy(), it.cpu().numpy()
    oc = oracle.OCode.from_synth(code256)
    hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs)
    ref = oc.decode(hard, pi, schedule=schedule, max_iters=60)
    def oq(idx):
        o = oc.decode(hard[idx], pi[idx], schedule=schedule, max_iters=60, keep_messages=True)
        return o["xhat"][:, :code256.N], o["Q"][:, :code256.N]
    match, strict, n_allow = gate.decision_gate(s_hat, it, ref["xhat"][:, :code256.N], ref["iters"], oq)
    assert gate.record("q=256 %s" % ("SUS" if schedule else "PUS"), fr.F, match, strict, n_allow) == 0
    assert (it > 0).mean() > 0.5


@pytest.mark.parametrize("schedule,prior", [(0, 0), (1, 0), (1, 1)], ids=["PUS", "SUS", "SUS-in-sweep"])
def test_q256_markov_message_gate(gfq, code256, schedule, prior):
    T = synth.markov_uniform_jump(256, 0.7)
    fr = synth.make_frames(code256, 13, range(33), "markov", synth.BSC, 0.08, stay=0.7)
    gcode = gfq.Code.from_synth(code256)
    prm = gfq.Params(gfq.GFQ_BSC, fr.ch_param, schedule, 3, early_exit=False, keep_messages=True, markov_T=T,
                     prior_update=prior)
    s_hat, it, ws = gfq.gfq_decode(gcode, torch.as_tensor(fr.obs).cuda(), prm)
    qg, rg, Qg = (x.cpu().numpy() for x in gfq.gfq_export_messages(gcode, fr.F, ws, prm))
    oc = oracle.OCode.from_synth(code256)
    hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs)
    ref = oc.decode(hard, pi, schedule=schedule, max_iters=3, fixed=True, keep_messages=True, T=T,
                    sus_gs=bool(prior))   # 3 iterations: the oracle's Eq. (6) is O(q^3) per symbol
    errs = {k: float(np.max(np.abs(g - ref[k]))) for k, g in (("q", qg), ("r", rg), ("Q", Qg))}
    print("q=256 Markov", schedule, prior, errs)
    assert max(errs.values()) <= MSG_TOL, errs
    assert np.array_equal(it.cpu().numpy(), ref["iters"])


def test_q256_simulate_then_decode(gfq, code256):
    """Device Monte-Carlo front end at q = 128 feeding the decoder: at a high SNR
    every frame decodes to the simulated source."""
    gcode = gfq.Code.from_synth(code256)
    s, obs, _ = gfq.gfq_simulate(gcode, 64, 0x5EED, gfq.GFQ_BIAWGN, 0.6)
    prm = gfq.Params(gfq.GFQ_BIAWGN, 0.6, 1, 50)
    s_hat, it, _ = gfq.gfq_decode(gcode, obs, prm)
    assert torch.equal(s_hat.cpu(), s.cpu())
    assert bool((it > 0).all())


def test_q256_general_markov_matrix(gfq, code256):
    """A transition matrix without the stay / uniform-jump structure takes the
    O(q^2) prior sums (T read through L1): message gate on one block."""
    rng = np.random.default_rng(256)
    T = rng.random((256, 256)) ** 4 + 1e-3
    T /= T.sum(1, keepdims=True)
    fr = synth.make_frames(code256, 14, range(9), "markov_T", synth.BSC, 0.05, T=T)
    gcode = gfq.Code.from_synth(code256)
    oc = oracle.OCode.from_synth(code256)
    hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs)
    for schedule in (0, 1):
        prm = gfq.Params(gfq.GFQ_BSC, fr.ch_param, schedule, 3, early_exit=False, keep_messages=True, markov_T=T)
        s_hat, it, ws = gfq.gfq_decode(gcode, torch.as_tensor(fr.obs).cuda(), prm)
        qg, rg, Qg = (x.cpu().numpy() for x in gfq.gfq_export_messages(gcode, fr.F, ws, prm))
        ref = oc.decode(hard, pi, schedule=schedule, max_iters=3, fixed=True, keep_messages=True, T=T)
        errs = {k: float(np.max(np.abs(g - ref[k]))) for k, g in (("q", qg), ("r", rg), ("Q", Qg))}
        print("q=256 general T", schedule, errs)
        assert max(errs.values()) <= MSG_TOL, errs


def test_q256_early_exit_compaction_identical(gfq, code256):
    """Frame-granular compaction at q = 256 (96 frames, 3 blocks): bit-identical outputs."""
    fr = _frames(code256, 96, 0.8)
    gcode = gfq.Code.from_synth(code256)
    outs = []
    for comp in (gfq.GFQ_COMPACT_BLOCKS, gfq.GFQ_COMPACT_FRAMES):
        prm = gfq.Params(gfq.GFQ_BIAWGN, fr.ch_param, 1, 60, early_exit=True, compaction=comp)
        s_hat, it, ws = gfq.gfq_decode(gcode, torch.as_tensor(fr.obs).cuda(), prm)
        outs.append((s_hat.cpu().numpy(), it.cpu().numpy(), gfq.gfq_decode_stats(gcode, ws)["block_iterations"]))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    assert outs[1][2] <= outs[0][2]

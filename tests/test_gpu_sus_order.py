"""GPU parity for SUS sweeping the columns in caller-supplied orders (gfq_params
.sus_order, reading A35) against the oracle's `sus_order` decode
(oracle/oracle.c o_decode_frame; pinned in test_oracle_pins.py) on the same
seeded inputs and gates as tests/test_gpu_parity.py: every message within
max-abs 1e-4 after a fixed 5 sweeps; decisions and iteration counts identical
on >= 99.9 % of frames (reading A18).  A different seeded random permutation per
sweep (the random numbers are inputs, drawn here)."""
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


def _orders(V, n, seed):
    rng = np.random.default_rng(seed)
    return np.stack([rng.permutation(V) for _ in range(n)]).astype(np.int32)


def _channel(gfq, fr):
    return {synth.BSC: gfq.GFQ_BSC, synth.BEC: gfq.GFQ_BEC, synth.BIAWGN: gfq.GFQ_BIAWGN}[fr.channel]


def _decode(gfq, gcode, fr, max_iters, early_exit, T, orders, keep=False):
    prm = gfq.Params(_channel(gfq, fr), fr.ch_param, gfq.GFQ_SUS, max_iters, early_exit=early_exit,
                     markov_T=T, keep_messages=keep, sus_order=orders)
    s_hat, iters, ws = gfq.gfq_decode(gcode, torch.as_tensor(fr.obs).cuda(), prm)
    torch.cuda.synchronize()
    return prm, s_hat.cpu().numpy(), iters.cpu().numpy(), ws


MSG_CASES = [("C1", 64, 0), ("C2", 80, 0), ("C3", 40, 4), ("C4", 40, 0), ("C5", 8, 0)]


@pytest.mark.parametrize("name,nframes,point", MSG_CASES)
def test_sus_order_message_gate(gfq, name, nframes, point):
    cfg = synth.CONFIGS[name]
    code = synth.code_for(cfg)
    fr = synth.frames_for(cfg, code, range(nframes), point=point)
    T = synth.markov_T_for(cfg)
    orders = _orders(code.V, 3, 1000 + cfg.cid)
    gcode = gfq.Code.from_synth(code)
    prm, _, it, ws = _decode(gfq, gcode, fr, 5, False, T, orders, keep=True)
    qg, rg, Qg = (x.cpu().numpy() for x in gfq.gfq_export_messages(gcode, fr.F, ws, prm))
    oc = oracle.OCode.from_synth(code)
    hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs)
    ref = oc.decode(hard, pi, schedule=oracle.SUS, max_iters=5, fixed=True, T=T, keep_messages=True,
                    sus_order=orders)
    errs = {k: float(np.max(np.abs(g - ref[k]))) for k, g in (("q", qg), ("r", rg), ("Q", Qg))}
    print(name, point, errs)
    assert max(errs.values()) <= MSG_TOL, errs
    assert np.array_equal(it, ref["iters"])
    assert gfq.gfq_decode_stats(gcode, ws)["zero_normalisers"] == 0
    # the order matters on these inputs: index order gives different messages
    nat = oc.decode(hard, pi, schedule=oracle.SUS, max_iters=5, fixed=True, T=T, keep_messages=True)
    assert float(np.max(np.abs(nat["q"] - ref["q"]))) > 10 * MSG_TOL


DEC_CASES = [("C1", 64, 0), ("C2", 256, 0), ("C3", 128, 1), ("C5", 8, 0)]


@pytest.mark.parametrize("name,nframes,point", DEC_CASES)
def test_sus_order_decision_gate(gfq, name, nframes, point):
    cfg = synth.CONFIGS[name]
    code = synth.code_for(cfg)
    fr = synth.frames_for(cfg, code, range(nframes), point=point)
    T = synth.markov_T_for(cfg)
    orders = _orders(code.V, 16, 2000 + cfg.cid)   # cycled: sweep t uses (t-1) mod 16
    gcode = gfq.Code.from_synth(code)
    _, s_hat, iters, ws = _decode(gfq, gcode, fr, cfg.max_iters, True, T, orders)
    oc = oracle.OCode.from_synth(code)
    hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs)
    ref = oc.decode(hard, pi, schedule=oracle.SUS, max_iters=cfg.max_iters, T=T, sus_order=orders)
    def oq(idx):
        o = oc.decode(hard[idx], pi[idx], schedule=oracle.SUS, max_iters=cfg.max_iters, T=T, sus_order=orders,
                      keep_messages=True)
        return o["xhat"][:, :code.N], o["Q"][:, :code.N]
    match, strict, n_allow = gate.decision_gate(s_hat, iters, ref["xhat"][:, :code.N], ref["iters"], oq)
    mism = gate.record("sus_order %s p%d" % (name, point), fr.F, match, strict, n_allow)
    assert mism <= gate.allowed(fr.F)
    assert gfq.gfq_decode_stats(gcode, ws)["zero_normalisers"] == 0


def test_sus_identity_order_is_index_order(gfq):
    cfg = synth.CONFIGS["C3"]
    code = synth.code_for(cfg)
    fr = synth.frames_for(cfg, code, range(64), point=2)
    gcode = gfq.Code.from_synth(code)
    _, s1, i1, _ = _decode(gfq, gcode, fr, cfg.max_iters, True, None, np.arange(code.V, dtype=np.int32)[None])
    _, s0, i0, _ = _decode(gfq, gcode, fr, cfg.max_iters, True, None, None)
    assert np.array_equal(s1, s0) and np.array_equal(i1, i0)


def test_sus_order_rejected_when_invalid(gfq):
    cfg = synth.CONFIGS["C2"]
    code = synth.code_for(cfg)
    fr = synth.frames_for(cfg, code, range(4))
    gcode = gfq.Code.from_synth(code)
    T = synth.markov_T_for(cfg)
    good = _orders(code.V, 2, 5)
    bad = good.copy()
    bad[1, 3] = bad[1, 4]                     # not a permutation
    for sched, prior, order in ((gfq.GFQ_SUS, 0, bad), (gfq.GFQ_PUS, 0, good), (gfq.GFQ_SUS, 1, good)):
        prm = gfq.Params(gfq.GFQ_BSC, fr.ch_param, sched, 5, markov_T=T, prior_update=prior, sus_order=order)
        with pytest.raises(gfq.GfqError) as e:
            gfq.gfq_decode(gcode, torch.as_tensor(fr.obs).cuda(), prm)
        assert e.value.code == gfq.GFQ_EINVAL


def test_sus_order_waves_and_ragged_frames(gfq):
    """100 frames (ragged last block) through a workspace that holds 2 of the 4
    32-frame blocks (2 waves): identical to one wave, and the order tables live
    in every wave's workspace layout."""
    cfg = synth.CONFIGS["C3"]
    code = synth.code_for(cfg)
    fr = synth.frames_for(cfg, code, range(100), point=3)
    gcode = gfq.Code.from_synth(code)
    orders = _orders(code.V, 4, 77)
    prm = gfq.Params(gfq.GFQ_BIAWGN, fr.ch_param, gfq.GFQ_SUS, cfg.max_iters, sus_order=orders)
    obs = torch.as_tensor(fr.obs).cuda()
    s1, i1, _ = gfq.gfq_decode(gcode, obs, prm)
    small = gfq.alloc_workspace(gfq.gfq_workspace_bytes(gcode, 64, prm))
    s2, i2, _ = gfq.gfq_decode(gcode, obs, prm, workspace=small)
    assert torch.equal(s1, s2) and torch.equal(i1, i2)
    assert bool((i1 > 0).all())


def test_sus_order_zero_iterations_and_more_orders_than_sweeps(gfq):
    """max_iters = 0 runs no sweep (clipped priors, iters -1) whatever the orders;
    16 orders with 3 sweeps use only the first 3 (= a decode given those 3)."""
    cfg = synth.CONFIGS["C1"]
    code = synth.code_for(cfg)
    fr = synth.frames_for(cfg, code, range(40))
    gcode = gfq.Code.from_synth(code)
    orders = _orders(code.V, 16, 99)
    _, s0, i0, _ = _decode(gfq, gcode, fr, 0, False, None, orders)
    _, s1, i1, _ = _decode(gfq, gcode, fr, 0, False, None, None)
    assert np.array_equal(s0, s1) and (i0 == -1).all() and (i1 == -1).all()
    prm, _, _, ws = _decode(gfq, gcode, fr, 3, False, None, orders, keep=True)
    qa = gfq.gfq_export_messages(gcode, fr.F, ws, prm)[0].cpu().numpy()
    prm, _, _, ws = _decode(gfq, gcode, fr, 3, False, None, orders[:3], keep=True)
    qb = gfq.gfq_export_messages(gcode, fr.F, ws, prm)[0].cpu().numpy()
    assert np.array_equal(qa, qb)

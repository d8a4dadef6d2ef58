"""GPU parity of the Monte-Carlo front end (gfq_simulate) against
the CPU oracle oracle/montecarlo.py drawing the same counter-based random
numbers: source symbols, codewords and BSC/BEC outputs bit-exact (integer
decisions taken on identical dyadic uniforms); BI-AWGN outputs to fp32
rounding (both sides compute in double; libm differences stay below 1 ulp of
the float32 result almost everywhere).  Plus the Monte-Carlo loop end to end:
device frames decoded on the device recover the source."""
import numpy as np
import pytest

import synth
from oracle import montecarlo as mc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gfq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    from paper_cs_0605069_b200 import gfq as g
    return g


def _coo(code):
    r, c, v = code.H_coo()
    return (code.p, code.poly, code.N, code.M, r, c, v)


CASES = [("C1", synth.BSC, 0.06, None), ("C2", synth.BSC, 0.05, "uj"), ("C3", synth.BIAWGN, 0.84, None),
         ("C4", synth.BEC, 0.35, "uj"), ("C5", synth.BIAWGN, 0.8414, None), ("C2", synth.BEC, 0.2, "4S")]


@pytest.mark.parametrize("name,ch,param,src", CASES)
def test_simulate_matches_oracle(gfq, name, ch, param, src):
    cfg = synth.CONFIGS[name]
    code = synth.code_for(cfg)
    gc = gfq.Code.from_synth(code)
    T = pi0 = None
    if src == "uj":
        T = synth.markov_uniform_jump(code.q, cfg.stay)
    elif src == "4S":
        T = synth.MARKOV_4S / synth.MARKOV_4S.sum(axis=1, keepdims=True)
        pi0 = synth.stationary(T)
    F = 8 if name == "C5" else 37                      # ragged last block
    seed, frame0 = 0x1234_5678_9ABC, 1000 + 3
    s, obs, t = gfq.gfq_simulate(gc, F, seed, ch, param, frame0=frame0, markov_T=T, src_pi0=pi0, want_t=True)
    torch.cuda.synchronize()
    frames = np.arange(frame0, frame0 + F)
    rs, rt, robs = mc.simulate(_coo(code), seed, frames, ch, param, T, pi0)
    assert np.array_equal(s.cpu().numpy(), rs)
    assert np.array_equal(t.cpu().numpy(), rt)
    o = obs.cpu().numpy()
    if ch == synth.BIAWGN:
        assert o.dtype == np.float32
        d = np.abs(o.astype(np.float64) - robs.astype(np.float64))
        assert d.max() <= 1e-5
        assert (d == 0).mean() >= 0.999
    else:
        assert np.array_equal(o, robs)


def test_simulate_subset_reproduces(gfq):
    cfg = synth.CONFIGS["C2"]
    code = synth.code_for(cfg)
    gc = gfq.Code.from_synth(code)
    T = synth.markov_uniform_jump(code.q, cfg.stay)
    a = gfq.gfq_simulate(gc, 64, 99, gfq.GFQ_BSC, 0.05, markov_T=T)
    b = gfq.gfq_simulate(gc, 5, 99, gfq.GFQ_BSC, 0.05, frame0=40, markov_T=T)
    assert torch.equal(a[0][40:45], b[0]) and torch.equal(a[1][40:45], b[1])


def test_simulate_then_decode_recovers_source(gfq):
    """The Monte-Carlo loop on the device: simulate, decode (SUS, early exit),
    compare with the source -- converged frames return the transmitted s."""
    cfg = synth.CONFIGS["C3"]
    code = synth.code_for(cfg)
    gc = gfq.Code.from_synth(code)
    sigma = synth.awgn_sigma(2.5)
    s, obs, _ = gfq.gfq_simulate(gc, 256, 7, gfq.GFQ_BIAWGN, sigma)
    prm = gfq.Params(gfq.GFQ_BIAWGN, sigma, gfq.GFQ_SUS, cfg.max_iters)
    s_hat, iters, _ = gfq.gfq_decode(gc, obs, prm)
    torch.cuda.synchronize()
    conv = (iters > 0).cpu().numpy()
    assert conv.mean() > 0.99
    ok = (s_hat == s).all(dim=1).cpu().numpy()
    assert ok[conv].mean() > 0.99


def test_simulate_rejects_non_triangular_B(gfq):
    # B with two identical weight-2 columns in a 2x2 block: no row has a single unknown
    gc = gfq.Code(1, 0x3, 1, 2, [0], [0], [1], [0, 0, 1, 1], [0, 1, 0, 1], [1, 1, 1, 1])
    with pytest.raises(gfq.GfqError) as e:
        gfq.gfq_simulate(gc, 4, 1, gfq.GFQ_BSC, 0.1)
    assert e.value.code == gfq.GFQ_EUNSUPPORTED

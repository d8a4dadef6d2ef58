"""Pins for the Monte-Carlo front-end oracle (oracle/montecarlo.py): Philox known
answers, the encoder against the code's own equations and an independent
encoder, and the laws of the generated source and channel.  CPU only."""
import numpy as np
import pytest

import oracle
import synth
from oracle import montecarlo as mc


@pytest.mark.parametrize("ctr,key,want", [
    ((0, 0, 0, 0), (0, 0), (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)),
    ((0xffffffff,) * 4, (0xffffffff,) * 2, (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)),
    ((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344), (0xa4093822, 0x299f31d0),
     (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1)),
])
def test_philox_known_answers(ctr, key, want):
    """Philox4x32-10 known-answer vectors (Random123 kat_vectors)."""
    out = mc.philox4x32_10(*[np.array([c], np.uint32) for c in ctr], *key)
    assert tuple(int(o[0]) for o in out) == want


def _coo(code):
    r, c, v = code.H_coo()
    return (code.p, code.poly, code.N, code.M, r, c, v)


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_encoder_satisfies_eq1_and_matches_independent_encoder(name):
    cfg = synth.CONFIGS[name]
    code = synth.code_for(cfg)
    s = mc.source(7, np.arange(5), code.N, code.q)
    t = mc.encode(*_coo(code), s)
    oc = oracle.OCode.from_synth(code)
    for f in range(5):   # H [s; t] = A s + B t = 0 (Eq. 1: t = B^-1 A s)
        assert oc.unsatisfied(np.concatenate([s[f], t[f]]), np.zeros(code.M, np.uint8)) == 0
    assert np.array_equal(t, synth.encode(code, s))


def test_encoder_rejects_non_triangular_B():
    # B = [[1,1],[1,1]] over GF(2): no row with a single unknown
    with pytest.raises(ValueError):
        mc.encode(1, 0x3, 1, 2, [0, 1, 0, 0, 1, 1], [0, 0, 1, 2, 1, 2], [1, 1, 1, 1, 1, 1],
                  np.zeros((1, 1), np.uint8))


def test_iid_source_uniform_and_reproducible():
    s = mc.source(11, np.arange(64), 4000, 16)
    counts = np.bincount(s.ravel(), minlength=16) / s.size
    assert np.max(np.abs(counts - 1 / 16)) < 0.004
    again = mc.source(11, np.array([5, 17]), 4000, 16)     # any subset of frames reproduces
    assert np.array_equal(again, s[[5, 17]])
    assert not np.array_equal(mc.source(12, np.arange(2), 4000, 16), s[:2])


def test_markov_source_transition_law():
    T = synth.MARKOV_4S / synth.MARKOV_4S.sum(axis=1, keepdims=True)
    pi0 = synth.stationary(T)
    s = mc.source(3, np.arange(200), 2000, 4, T, pi0)
    cnt = np.zeros((4, 4))
    np.add.at(cnt, (s[:, :-1].ravel(), s[:, 1:].ravel()), 1)
    emp = cnt / cnt.sum(axis=1, keepdims=True)
    assert np.max(np.abs(emp - T)) < 0.01
    first = np.bincount(s[:, 0], minlength=4) / 200
    assert np.max(np.abs(first - pi0)) < 0.1


def test_running_sums_last_entry_is_one():
    C = mc.running_sums([[0.1, 0.2, 0.3, 0.39999999]])
    assert C[0, -1] == 1.0 and C[0, 0] == 0.1


@pytest.mark.parametrize("ch,param", [(0, 0.08), (1, 0.3), (2, 0.8)])
def test_channel_laws(ch, param):
    F, M, p = 40, 2000, 2
    t = mc.source(5, np.arange(F), M, 1 << p)           # any symbols serve as a codeword here
    obs = mc.channel(9, np.arange(F), t, p, ch, param)
    bits = ((t[:, :, None] >> np.arange(p, dtype=np.uint8)) & 1).reshape(F, M * p)
    if ch == 0:
        assert abs((obs != bits).mean() - param) < 0.005
    elif ch == 1:
        er = obs == 2
        assert abs(er.mean() - param) < 0.005
        assert np.array_equal(obs[~er], bits[~er])
    else:
        n = (obs - (1.0 - 2.0 * bits)) / param
        assert abs(n.mean()) < 0.01 and abs(n.std() - 1.0) < 0.01
        assert abs(np.mean(n > 1.0) - 0.158655) < 0.005      # Gaussian tail
        assert obs.dtype == np.float32


def test_simulate_pipeline_syndrome():
    """obs of a noiseless BSC (f = 0) is the codeword; its syndrome is A s (Eq. 2)."""
    cfg = synth.CONFIGS["C2"]
    code = synth.code_for(cfg)
    T = synth.markov_T_for(cfg)
    s, t, obs = mc.simulate(_coo(code), 21, np.arange(4), 0, 0.0, T)
    assert np.array_equal(synth.bits_to_symbols(obs, code.p), t)
    oc = oracle.OCode.from_synth(code)
    for f in range(4):
        z = oc.syndrome(t[f])           # z = B r with r = t
        assert oc.unsatisfied(np.concatenate([s[f], np.zeros(code.M, np.uint8)]), z) == 0

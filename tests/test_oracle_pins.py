"""Pins for the fp64 oracle: each oracle function is tied to something other
than itself -- exhaustive field axioms, brute-force enumeration of Eq. (3),
closed forms (tanh rule, BSC prior, Gaussian posterior), worked values printed
in the paper or derived in SPEC.md (tests/golden/), and exactness of both
schedules on trees.  CPU only."""
import itertools
import math

import numpy as np
import pytest

import oracle
import synth
from conftest import load_markov_golden

POLY = synth.PRIM_POLY


# ----------------------------------------------------------------------------- GF(2^p)
@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_gf_field_axioms_exhaustive(p):
    q = 1 << p
    mul = np.array([[oracle.gf_mul(a, b, p, POLY[p]) for b in range(q)] for a in range(q)])
    assert (mul == mul.T).all()                                   # commutative
    assert (mul[1] == np.arange(q)).all() and (mul[0] == 0).all()  # identity, absorbing 0
    for a, b, c in itertools.product(range(q), repeat=3):
        assert mul[mul[a, b], c] == mul[a, mul[b, c]]              # associative
        assert mul[a, b ^ c] == mul[a, b] ^ mul[a, c]              # distributive over XOR
    for a in range(1, q):
        assert mul[a, oracle.gf_inv(a, p, POLY[p])] == 1
        assert sorted(mul[a, 1:]) == list(range(1, q))             # no zero divisors


@pytest.mark.parametrize("p", [5, 6, 7])
def test_gf_large_fields_sampled(p):
    q = 1 << p
    rng = np.random.default_rng(p)
    for _ in range(3000):
        a, b, c = (int(v) for v in rng.integers(0, q, 3))
        m = lambda x, y: oracle.gf_mul(x, y, p, POLY[p])
        assert m(m(a, b), c) == m(a, m(b, c))
        assert m(a, b ^ c) == m(a, b) ^ m(a, c)
    for a in range(1, q):
        assert oracle.gf_mul(a, oracle.gf_inv(a, p, POLY[p]), p, POLY[p]) == 1


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8])
def test_gf_primitive_element_order(p):
    """x generates the multiplicative group: ord(x) = q-1 (the polynomials are primitive, A1)."""
    q = 1 << p
    g = 2 if q > 2 else 1
    seen, a = set(), 1
    for _ in range(q - 1):
        a = oracle.gf_mul(a, g, p, POLY[p])
        seen.add(a)
    assert seen == set(range(1, q))


def test_gf_worked_values(golden):
    assert oracle.gf_mul(3, 7, 3, POLY[3]) == golden["gf8_mul_3_7"][0][0]
    assert oracle.gf_inv(2, 2, POLY[2]) == golden["gf4_inv_2"][0][0]


def test_gf_matches_encoder_tables():
    """The oracle's shift-and-xor multiply equals the generator's log/antilog tables."""
    for p in range(1, 7):
        tab = synth.gf_tables(p).mul
        for a in range(1 << p):
            for b in range(1 << p):
                assert oracle.gf_mul(a, b, p, POLY[p]) == tab[a, b]


# ----------------------------------------------------------------------------- front end, priors
def test_frontend_bsc_bec_awgn(golden):
    h, pi = oracle.frontend(oracle.BSC, 0.06, np.array([0, 1, 1, 0], np.uint8))
    assert list(h) == [0, 1, 1, 0] and np.allclose(pi, 0.06)
    h, pi = oracle.frontend(oracle.BEC, 0.35, np.array([0, 1, 2, 2], np.uint8))
    assert list(h) == [0, 1, 0, 0] and list(pi) == [0.0, 0.0, 0.5, 0.5]
    h, pi = oracle.frontend(oracle.BIAWGN, 0.8, np.array([0.0], np.float32))
    assert pi[0] == golden["awgn_flip_y0"][0][0]


def test_frontend_awgn_is_gaussian_posterior():
    """pi = Pr(hard decision wrong | y) by Bayes with equiprobable +-1 and N(0, s^2)."""
    sigma = 0.8414
    y = np.linspace(-3, 3, 61).astype(np.float32)
    h, pi = oracle.frontend(oracle.BIAWGN, sigma, y)
    phi = lambda u: math.exp(-u * u / (2 * sigma * sigma))
    for yy, hh, pp in zip(y.astype(float), h, pi):
        p_plus, p_minus = phi(yy - 1.0), phi(yy + 1.0)   # likelihood of bit 0 (+1), bit 1 (-1)
        wrong = p_minus / (p_plus + p_minus) if hh == 0 else p_plus / (p_plus + p_minus)
        assert hh == (1 if yy < 0 else 0)
        assert abs(pp - wrong) < 1e-12


def test_noise_prior_bsc_closed_form(golden):
    """Q_j^a = f^L (1-f)^(log2 q - L), L = popcount(a)."""
    for p in range(1, 7):
        for f in (0.06, 0.155, 0.23):
            pr = oracle.noise_prior(p, [f] * p)
            for a in range(1 << p):
                L = bin(a).count("1")
                assert abs(pr[a] - f ** L * (1 - f) ** (p - L)) < 1e-15
            assert abs(pr.sum() - 1) < 1e-12
    assert abs(oracle.noise_prior(3, [0.1] * 3)[3] - golden["noise_prior_bsc"][0][0]) < 1e-15


def test_noise_prior_bec_and_generic(golden):
    assert np.allclose(oracle.noise_prior(2, [0.5, 0.5]), golden["noise_prior_bec_q4"][0])
    pr = oracle.noise_prior(3, [0.0, 0.5, 0.0])   # bit 1 erased: uniform over {0, 2}
    assert list(pr) == [0.5, 0, 0.5, 0, 0, 0, 0, 0]
    rng = np.random.default_rng(1)
    for _ in range(50):
        p = int(rng.integers(1, 7))
        pr = oracle.noise_prior(p, rng.random(p))
        assert abs(pr.sum() - 1) < 1e-12


# ----------------------------------------------------------------------------- check node, Eq. (3)
def brute_check(p, h, qin, z, out):
    """Eq. (3) literally: enumerate every configuration of the other variables."""
    q = 1 << p
    mul = synth.gf_tables(p).mul
    d = len(h)
    others = [k for k in range(d) if k != out]
    r = np.zeros(q)
    for a in range(q):
        for xs in itertools.product(range(q), repeat=len(others)):
            acc = int(mul[h[out], a])
            w = 1.0
            for k, x in zip(others, xs):
                acc ^= int(mul[h[k], x])
                w *= qin[k][x]
            if acc == z:
                r[a] += w
    return r


@pytest.mark.parametrize("p,d", [(1, 1), (1, 2), (1, 3), (1, 4), (2, 2), (2, 3), (2, 4),
                                 (3, 2), (3, 3), (3, 4), (4, 2), (4, 3), (6, 2), (6, 3),
                                 (7, 2), (7, 3), (8, 2)])
def test_check_node_equals_enumeration(p, d):
    q = 1 << p
    rng = np.random.default_rng(100 * p + d)
    for trial in range(8 if p < 4 else 2):
        h = rng.integers(1, q, d)
        qin = rng.random((d, q)) + 1e-3
        qin /= qin.sum(1, keepdims=True)
        z = int(rng.integers(q))
        for out in range(d):
            r = oracle.check_node(p, POLY[p], h, qin, z, out)
            assert np.max(np.abs(r - brute_check(p, h, qin, z, out))) < 1e-12
            assert abs(r.sum() - 1) < 1e-12           # exact normalisation (reading A5)


def test_check_node_equals_enumeration_gf256_degree3():
    """Eq. (3) at q = 256, d = 3: every configuration (x1, x2) of the two other
    variables enumerated at once (numpy), summed into the symbol a they force."""
    p, q = 8, 256
    mul = synth.gf_tables(p).mul
    rng = np.random.default_rng(808)
    h = rng.integers(1, q, 3)
    qin = rng.random((3, q)) + 1e-3
    qin /= qin.sum(1, keepdims=True)
    z = int(rng.integers(q))
    for out in range(3):
        o1, o2 = [k for k in range(3) if k != out]
        y = mul[h[o1], np.arange(q)][:, None] ^ mul[h[o2], np.arange(q)][None, :]   # h1 x1 + h2 x2
        S = np.zeros(q)
        np.add.at(S, y.ravel(), np.outer(qin[o1], qin[o2]).ravel())
        r_enum = np.array([S[z ^ int(mul[h[out], a])] for a in range(q)])          # h_out a = z + (...)
        r = oracle.check_node(p, POLY[p], h, qin, z, out)
        assert np.max(np.abs(r - r_enum)) < 1e-12
        assert abs(r.sum() - 1) < 1e-12


def test_check_node_worked_values(golden):
    r = oracle.check_node(1, POLY[1], [1, 1, 1], [[0.5, 0.5], [0.9, 0.1], [0.8, 0.2]], 0, 0)
    assert np.allclose(r, golden["cn_q2_deg3"][0], atol=1e-15)
    r = oracle.check_node(1, POLY[1], [1, 1], [[0.5, 0.5], [0.9, 0.1]], 0, 0)
    assert np.allclose(r, golden["cn_q2_deg2"][0], atol=1e-15)


def test_check_node_q2_tanh_rule():
    """Binary closed form: r(0)-r(1) = (-1)^z prod_{j'!=j} (q_j'(0)-q_j'(1))."""
    rng = np.random.default_rng(7)
    for _ in range(200):
        d = int(rng.integers(1, 7))
        qin = rng.random((d, 2))
        qin /= qin.sum(1, keepdims=True)
        z = int(rng.integers(2))
        out = int(rng.integers(d))
        r = oracle.check_node(1, POLY[1], [1] * d, qin, z, out)
        pred = (-1) ** z * np.prod([qin[k, 0] - qin[k, 1] for k in range(d) if k != out])
        assert abs((r[0] - r[1]) - pred) < 1e-13


@pytest.mark.parametrize("p", [2, 3, 4, 6, 7])
def test_check_node_special_cases(p):
    q = 1 << p
    mul = synth.gf_tables(p).mul
    inv = synth.gf_tables(p).inv
    rng = np.random.default_rng(p)
    h = rng.integers(1, q, 4)
    # uniform in -> uniform out
    r = oracle.check_node(p, POLY[p], h, np.full((4, q), 1.0 / q), 5 % q, 2)
    assert np.allclose(r, 1.0 / q, atol=1e-14)
    # point masses in -> point mass at h_out^-1 (z + sum h x)
    xs = rng.integers(0, q, 4)
    qin = np.zeros((4, q))
    qin[np.arange(4), xs] = 1.0
    z = int(rng.integers(q))
    acc = z
    for k in (0, 1, 3):
        acc ^= int(mul[h[k], xs[k]])
    r = oracle.check_node(p, POLY[p], h, qin, z, 2)
    want = np.zeros(q)
    want[inv[h[2]] if acc == 0 else mul[inv[h[2]], acc]] = 1.0
    assert np.array_equal(r, want)
    # degree-1 check: point mass at h^-1 z
    r = oracle.check_node(p, POLY[p], [h[0]], np.full((1, q), 1.0 / q), z, 0)
    want = np.zeros(q)
    want[mul[inv[h[0]], z]] = 1.0
    assert np.array_equal(r, want)


# ----------------------------------------------------------------------------- variable node, posterior
def test_var_node_and_posterior_worked_values(golden):
    qo, zero = oracle.var_node([0.5, 0.5], [[0.3, 0.7], [0.9, 0.1]], 0)
    assert np.allclose(qo, golden["vn_q2"][0], atol=1e-15) and zero == 0
    qo, _ = oracle.var_node([0.8, 0.2], [[0.1, 0.9], [0.5, 0.5]], 0)
    assert np.allclose(qo, golden["vn_uniform_neutral"][0], atol=1e-15)
    Q, x, zf = oracle.posterior([0.5, 0.5], [[0.9, 0.1], [0.8, 0.2]])
    assert np.allclose(Q, golden["posterior_q2"][0], atol=1e-14) and x == 0 and zf == 0


def test_var_node_properties():
    rng = np.random.default_rng(3)
    for _ in range(100):
        q = 1 << int(rng.integers(1, 7))
        dv = int(rng.integers(1, 5))
        prior = rng.random(q)
        prior /= prior.sum()
        rin = rng.random((dv, q))
        out = int(rng.integers(dv))
        qo, zero = oracle.var_node(prior, rin, out)
        want = prior * np.prod(np.delete(rin, out, axis=0), axis=0)
        assert np.allclose(qo, want / want.sum(), rtol=1e-13, atol=0)
        assert abs(qo.sum() - 1) < 1e-12
    # degree 1: the normalised prior
    qo, _ = oracle.var_node([0.2, 0.6, 0.1, 0.1], [[0.7, 0.1, 0.1, 0.1]], 0)
    assert np.allclose(qo, [0.2, 0.6, 0.1, 0.1])
    # contradictory messages: zero normaliser flagged, uniform emitted (A19)
    qo, zero = oracle.var_node([1.0, 0.0], [[0.0, 1.0], [1.0, 0.0]], 1)
    assert zero == 1 and np.allclose(qo, 0.5)


def test_posterior_clipping_ties_smallest():
    """Reading A17: clipping is the strict argmax; only values equal up
    to fp64 round-off (relative 1e-12) are ties, and ties go to the smallest a."""
    Q, x, _ = oracle.posterior([0.25] * 4, [[0.1, 0.4, 0.4, 0.1]])
    assert x == 1                                   # exact tie -> smallest a
    Q, x, _ = oracle.posterior([0.25] * 4, [[0.1, 0.4 * (1 - 1e-15), 0.4, 0.1]])
    assert x == 1                                   # round-off tie
    Q, x, _ = oracle.posterior([0.25] * 4, [[0.1, 0.4 * (1 - 1e-7), 0.4, 0.1]])
    assert x == 2                                   # a genuine 1e-7 difference decides
    Q, x, _ = oracle.posterior([0.25] * 4, [[0.1, 0.4 * (1 - 1e-3), 0.4, 0.1]])
    assert x == 2


def test_clipping_bec_coset_uniform_priors():
    """BEC (reading A15): the prior of a noise symbol n_k is uniform over the coset
    {n : n_b = 0 for every unerased bit b} (P:246-251 with flip probability 0 or
    1/2 per bit) -- an exact tie among 2^(#erased bits) values that only the tie
    rule resolves.  Clipping the priors (max_iters = 0) must give the
    smallest member, n = 0, for every noise symbol (and 0 for the uniform
    sources); a largest-a or round-off-decided rule gives other coset members."""
    cfg = synth.CONFIGS["C4"]
    code = synth.code_for(cfg)
    fr = synth.frames_for(cfg, code, range(3))
    oc = oracle.OCode.from_synth(code)
    hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs)
    out = oc.decode(hard, pi, max_iters=0, keep_messages=True)
    p, N = code.p, code.N
    n_erased = (fr.obs.reshape(3, code.M, p) == 2).sum(-1)           # [F][M]
    Qn = out["Q"][:, N:, :]
    ties = (Qn == Qn.max(-1, keepdims=True)).sum(-1)
    assert np.array_equal(ties, 2 ** n_erased)                      # exact coset ties
    assert (n_erased > 0).mean() > 0.5
    assert (out["xhat"] == 0).all()


def test_all_erased_frame_decodes_to_zero():
    """A fully erased BEC frame: every hard bit is 0, so z = B 0 = 0, and every prior
    and therefore every message and posterior is exactly uniform (q is a power of 2:
    the sums of Eq. (3) are exact).  All q posterior values tie exactly, the tie rule
    gives x = 0, which solves H x = 0 = z: the decoder stops at t = 1 with x = 0."""
    cfg = synth.CONFIGS["C4"]
    code = synth.code_for(cfg)
    oc = oracle.OCode.from_synth(code)
    obs = np.full((1, code.M * code.p), 2, np.uint8)
    hard, pi = oracle.frontend(synth.BEC, 1.0, obs)
    T = synth.markov_T_for(cfg)
    for schedule in (oracle.PUS, oracle.SUS):
        out = oc.decode(hard, pi, schedule=schedule, max_iters=3, T=T, keep_messages=True)
        assert out["iters"][0] == 1
        assert (out["xhat"] == 0).all()
        assert np.all(out["Q"] == 1.0 / code.q)                          # exactly uniform


# ----------------------------------------------------------------------------- Markov prior, Eqs. (6)/(7)
def eq7(T, pi0, Q):
    """Eq. (7): [sum_a Q_{i-1}^a M_ab] * [sum_c M_bc Q_{i+1}^c], boundaries A10."""
    N, q = Q.shape
    L = np.vstack([pi0[None, :], Q[:-1] @ T])
    R = np.vstack([Q[1:] @ T.T, np.ones((1, q))])
    P = L * R
    return P / P.sum(1, keepdims=True)


def test_markov_prior_eq6_equals_eq7():
    rng = np.random.default_rng(11)
    for q in (2, 4, 8, 16):
        T = rng.random((q, q))
        T /= T.sum(1, keepdims=True)
        pi0 = rng.random(q)
        pi0 /= pi0.sum()
        Q = rng.random((9, q))
        Q /= Q.sum(1, keepdims=True)
        assert np.max(np.abs(oracle.markov_prior(T, pi0, Q) - eq7(T, pi0, Q))) < 1e-13


def test_markov_prior_worked_and_special(golden):
    mats = load_markov_golden()
    T2 = mats["2S"]
    Q = np.array([[1.0, 0.0], [0.5, 0.5], [1.0, 0.0]])
    P = oracle.markov_prior(T2, np.array([0.5, 0.5]), Q)
    assert np.allclose(P[1], golden["markov2s_prior"][0], atol=1e-15)
    # T = I propagates a point mass; uniform T gives a uniform prior
    q = 4
    Q = np.zeros((3, q))
    Q[:, 2] = 1
    assert np.array_equal(oracle.markov_prior(np.eye(q), np.full(q, 0.25), Q)[1], np.eye(q)[2])
    rng = np.random.default_rng(2)
    Q = rng.random((5, q))
    Q /= Q.sum(1, keepdims=True)
    assert np.allclose(oracle.markov_prior(np.full((q, q), 0.25), np.full(q, 0.25), Q), 0.25)


def test_markov_source_statistics(golden):
    """Paper P:274 says the 2S/4S sources have 'entropy 1/2'; 2S: h(0.11) (golden)."""
    mats = load_markov_golden()
    T = mats["2S"]
    pi = synth.stationary(T)
    H = -sum(pi[a] * T[a, b] * math.log2(T[a, b]) for a in range(2) for b in range(2))
    assert abs(H - golden["markov2s_entropy"][0][0]) < 1e-9
    T4 = mats["4S"]
    assert np.max(np.abs(T4.sum(1) - 1)) < 1e-6          # rows stochastic up to print rounding
    pi4 = synth.stationary(T4 / T4.sum(1, keepdims=True))
    assert np.max(np.abs(pi4 @ (T4 / T4.sum(1, keepdims=True)) - pi4)) < 1e-9


# ----------------------------------------------------------------------------- syndrome / pipeline identity
@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4"])
def test_pipeline_identity(cfg):
    """z = B r = [A B][s; n] = H x (Eq. 2) on generated frames, with H x
    evaluated independently (generator's tables); the true x passes the test."""
    c = synth.CONFIGS[cfg]
    code = synth.code_for(c)
    fr = synth.frames_for(c, code, range(6))
    oc = oracle.OCode.from_synth(code)
    hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs)
    rsym = synth.bits_to_symbols(hard, code.p)
    tab = synth.gf_tables(code.p)
    r, cl, v = code.H_coo()
    for f in range(6):
        z = oc.syndrome(rsym[f])
        x = fr.x_true()[f]
        hx = np.zeros(code.M, np.uint8)
        np.bitwise_xor.at(hx, r, tab.mul[v, x[cl]])
        assert np.array_equal(z, hx)
        assert oc.unsatisfied(x, z) == 0
        x2 = x.copy()
        x2[0] ^= 1
        assert oc.unsatisfied(x2, z) > 0
        # the true noise symbol has nonzero prior probability
        for k in range(0, code.M, 97):
            pr = oracle.noise_prior(code.p, pi[f, k * code.p:(k + 1) * code.p])
            assert pr[fr.n[f, k]] > 0


# ----------------------------------------------------------------------------- schedules: tree exactness etc.
def random_tree_code(rng, M, q):
    """Random cycle-free factor graph with M checks; returns (N, rows, cols, vals)."""
    edges = []
    nvar = 0
    for i in range(M):
        if i == 0:
            k = int(rng.integers(1, 4))
            for _ in range(k):
                edges.append((i, nvar)); nvar += 1
        else:
            parent = int(rng.integers(nvar))
            edges.append((i, parent))
            for _ in range(int(rng.integers(1, 3))):
                edges.append((i, nvar)); nvar += 1
    V = nvar
    if V < M:
        return None
    perm = rng.permutation(V)
    rows = np.array([e[0] for e in edges], np.int32)
    cols = np.array([perm[e[1]] for e in edges], np.int32)
    vals = rng.integers(1, q, len(edges)).astype(np.uint8)
    return V - M, rows, cols, vals


def brute_marginals(p, N, M, rows, cols, vals, z, priors):
    q = 1 << p
    V = N + M
    mul = synth.gf_tables(p).mul
    X = np.array(list(itertools.product(range(q), repeat=V)), dtype=np.int64)
    w = np.ones(len(X))
    for j in range(V):
        w *= priors[j][X[:, j]]
    ok = np.ones(len(X), bool)
    for i in range(M):
        acc = np.zeros(len(X), np.int64)
        for r, c, v in zip(rows, cols, vals):
            if r == i:
                acc ^= mul[v, X[:, c]]
        ok &= acc == z[i]
    w = w * ok
    Q = np.zeros((V, q))
    for j in range(V):
        np.add.at(Q[j], X[:, j], w)
    return Q / Q.sum(1, keepdims=True)


def setup_frame(rng, p, N, M, rows, cols, vals):
    """Random noise evidence (per-bit pi) and a feasible z from a random x."""
    q = 1 << p
    pi = rng.uniform(0.05, 0.45, M * p)
    hard = rng.integers(0, 2, M * p).astype(np.uint8)
    oc = oracle.OCode(p, POLY[p], N, M, rows, cols, vals)
    rsym = synth.bits_to_symbols(hard[None], p)[0]
    z = oc.syndrome(rsym)
    return oc, hard, pi, z


@pytest.mark.parametrize("p", [1, 2])
@pytest.mark.parametrize("schedule", [oracle.PUS, oracle.SUS])
def test_tree_exactness(p, schedule):
    """On cycle-free H both schedules' posteriors equal brute-force marginals."""
    rng = np.random.default_rng(40 + p + 10 * schedule)
    q = 1 << p
    done = 0
    while done < 8:
        M = int(rng.integers(2, 5))
        tc = random_tree_code(rng, M, q)
        if tc is None:
            continue
        N, rows, cols, vals = tc
        if N + M > (10 if p == 1 else 7):
            continue
        oc, hard, pi, z = setup_frame(rng, p, N, M, rows, cols, vals)
        pi0 = rng.random(q)
        pi0 /= pi0.sum()
        priors = [pi0] * N + [oracle.noise_prior(p, pi[k * p:(k + 1) * p]) for k in range(M)]
        want = brute_marginals(p, N, M, rows, cols, vals, z, priors)
        out = oc.decode(hard[None], pi[None], schedule=schedule, max_iters=2 * (N + M),
                        fixed=True, pi0=pi0, keep_messages=True, threads=1)
        assert np.max(np.abs(out["Q"][0] - want)) < 1e-9
        done += 1


def chain_code():
    """x0 - c0 - x1 - c1 - x2 over GF(2): checks x0+x1 = z0, x1+x2 = z1; x0 source, x1, x2 noise."""
    rows = np.array([0, 0, 1, 1], np.int32)
    cols = np.array([0, 1, 1, 2], np.int32)
    vals = np.ones(4, np.uint8)
    return oracle.OCode(1, POLY[1], 1, 2, rows, cols, vals)


@pytest.mark.parametrize("z", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_sus_fresh_read_closed_form(z):
    """SUS reads the freshest q: after ONE sweep Q_2(a) is the exact marginal
    p2(a) p1(z1+a) p0(z0+z1+a); one PUS iteration lacks x0's evidence: p2(a) p1(z1+a)."""
    oc = chain_code()
    pi0 = np.array([0.3, 0.7])
    p1, p2 = 0.2, 0.4
    # hard bits chosen so that z = B r: B = [[1,0],[1,1]] on (x1, x2) -> r1 = z0, r2 = z0^z1
    hard = np.array([[z[0], z[0] ^ z[1]]], np.uint8)
    pi = np.array([[p1, p2]])
    pr0 = pi0
    pr1 = np.array([1 - p1, p1])
    pr2 = np.array([1 - p2, p2])
    z0, z1 = z
    exact = np.array([pr2[a] * pr1[z1 ^ a] * pr0[z0 ^ z1 ^ a] for a in range(2)])
    pus1 = np.array([pr2[a] * pr1[z1 ^ a] for a in range(2)])
    sus = oc.decode(hard, pi, schedule=oracle.SUS, max_iters=1, fixed=True, pi0=pi0, keep_messages=True)
    pus = oc.decode(hard, pi, schedule=oracle.PUS, max_iters=1, fixed=True, pi0=pi0, keep_messages=True)
    assert np.allclose(sus["Q"][0, 2], exact / exact.sum(), atol=1e-15)
    assert np.allclose(pus["Q"][0, 2], pus1 / pus1.sum(), atol=1e-15)
    pus2 = oc.decode(hard, pi, schedule=oracle.PUS, max_iters=2, fixed=True, pi0=pi0, keep_messages=True)
    assert np.allclose(pus2["Q"][0, 2], exact / exact.sum(), atol=1e-15)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_single_check_schedules_agree(p):
    """One check: SUS and PUS messages identical after iteration 1."""
    q = 1 << p
    rng = np.random.default_rng(p)
    N, M = 3, 1
    rows = np.zeros(4, np.int32)
    cols = np.arange(4, dtype=np.int32)
    vals = rng.integers(1, q, 4).astype(np.uint8)
    oc, hard, pi, z = setup_frame(rng, p, N, M, rows, cols, vals)
    pi0 = rng.random(q)
    pi0 /= pi0.sum()
    a = oc.decode(hard[None], pi[None], schedule=oracle.PUS, max_iters=1, fixed=True, pi0=pi0, keep_messages=True)
    b = oc.decode(hard[None], pi[None], schedule=oracle.SUS, max_iters=1, fixed=True, pi0=pi0, keep_messages=True)
    for k in ("q", "r", "Q"):
        assert np.max(np.abs(a[k] - b[k])) < 1e-15


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_decode_invariants(cfg):
    """Normalised messages, converged => H x = z (re-verified independently), iters range,
    no vanished normaliser, determinism."""
    c = synth.CONFIGS[cfg]
    code = synth.code_for(c)
    fr = synth.frames_for(c, code, range(4))
    oc = oracle.OCode.from_synth(code)
    hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs)
    T = synth.markov_T_for(c)
    tab = synth.gf_tables(code.p)
    r, cl, v = code.H_coo()
    rsym = synth.bits_to_symbols(hard, code.p)
    for sch in (oracle.PUS, oracle.SUS):
        out = oc.decode(hard, pi, schedule=sch, max_iters=c.max_iters, T=T, keep_messages=True)
        again = oc.decode(hard, pi, schedule=sch, max_iters=c.max_iters, T=T)
        assert np.array_equal(out["xhat"], again["xhat"]) and np.array_equal(out["iters"], again["iters"])
        assert (out["zero_norms"] == 0).all()
        for f in range(4):
            it = out["iters"][f]
            assert it == -1 or 1 <= it <= c.max_iters
            if it > 0:
                z = oc.syndrome(rsym[f])
                hx = np.zeros(code.M, np.uint8)
                np.bitwise_xor.at(hx, r, tab.mul[v, out["xhat"][f][cl]])
                assert np.array_equal(hx, z)
        assert np.max(np.abs(out["q"].sum(-1) - 1)) < 1e-12
        assert np.max(np.abs(out["Q"].sum(-1) - 1)) < 1e-12
        assert np.max(np.abs(out["r"].sum(-1) - 1)) < 1e-12


def test_max_iters_zero_clips_priors():
    c = synth.CONFIGS["C1"]
    code = synth.code_for(c)
    fr = synth.frames_for(c, code, range(2))
    oc = oracle.OCode.from_synth(code)
    hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs)
    out = oc.decode(hard, pi, max_iters=0)
    assert (out["iters"] == -1).all()
    # noise priors favour "no flip" (0), sources uniform -> smallest symbol 0
    assert (out["xhat"] == 0).all()


def test_fixed_mode_records_first_pass():
    c = synth.CONFIGS["C1"]
    code = synth.code_for(c)
    fr = synth.frames_for(c, code, range(4))
    oc = oracle.OCode.from_synth(code)
    hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs)
    a = oc.decode(hard, pi, max_iters=100)
    b = oc.decode(hard, pi, max_iters=100, fixed=True)
    assert np.array_equal(a["iters"], b["iters"])
    assert np.array_equal(a["xhat"], b["xhat"])


def test_schedule_fixed_points_agree():
    """Tiny loopy codes, weak noise: when both schedules reach a fixed point the
    posteriors agree (a fixed point of BP does not depend on the schedule)."""
    rng = np.random.default_rng(5)
    agreed = 0
    for trial in range(20):
        p, N, M = 2, 3, 5
        q = 1 << p
        rows, cols = [], []
        for j in range(N + M):
            for i in rng.choice(M, 2, replace=False):
                rows.append(i); cols.append(j)
        rows = np.array(rows, np.int32)
        cols = np.array(cols, np.int32)
        vals = rng.integers(1, q, len(rows)).astype(np.uint8)
        oc, hard, pi, z = setup_frame(rng, p, N, M, rows, cols, vals)
        pi *= 0.3
        res = []
        for sch in (oracle.PUS, oracle.SUS):
            o1 = oc.decode(hard[None], pi[None], schedule=sch, max_iters=400, fixed=True, keep_messages=True)
            o2 = oc.decode(hard[None], pi[None], schedule=sch, max_iters=401, fixed=True, keep_messages=True)
            fixed_pt = np.max(np.abs(o1["Q"] - o2["Q"])) < 1e-13
            res.append((fixed_pt, o1["Q"][0]))
        if res[0][0] and res[1][0]:
            assert np.max(np.abs(res[0][1] - res[1][1])) < 1e-9
            agreed += 1
    assert agreed >= 5


# ----------------------------------------------------------------------------- Fig. 1 instrumentation
def _correct_bits_by_hand(x, s, p):
    """Correct source bits counted bit by bit from the definition."""
    n = 0
    for a, b in zip(x.tolist(), s.tolist()):
        for k in range(p):
            n += ((a >> k) & 1) == ((b >> k) & 1)
    return n


@pytest.mark.parametrize("name,schedule", [("C1", oracle.PUS), ("C1", oracle.SUS), ("C2", oracle.SUS)])
def test_trace_matches_truncated_decodes(name, schedule):
    """trace[t] (correct source bits after iteration t) equals the count taken by
    hand on the estimate of a decode stopped after t iterations: x^(t) does not
    depend on max_iters (the prior refresh after the last iteration only feeds
    iteration t+1).  After convergence the estimate is frozen."""
    c = synth.CONFIGS[name]
    code = synth.code_for(c)
    fr = synth.frames_for(c, code, range(3))
    oc = oracle.OCode.from_synth(code)
    T = synth.markov_T_for(c)
    hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs)
    tmax = 12
    full = oc.decode(hard, pi, schedule=schedule, max_iters=tmax, T=T, s_true=fr.s)
    tr = full["trace"]
    assert tr.shape == (3, tmax + 1)
    for t in range(0, tmax + 1):
        part = oc.decode(hard, pi, schedule=schedule, max_iters=t, T=T)
        for f in range(3):
            it = full["iters"][f]
            if it > 0 and t > it:
                assert tr[f, t] == tr[f, it]          # frozen after the early exit
            else:
                assert tr[f, t] == _correct_bits_by_hand(part["xhat"][f, :code.N], fr.s[f], code.p)
    conv = full["iters"] > 0
    # a converged frame whose estimate is the truth has every bit right
    for f in np.flatnonzero(conv):
        if np.array_equal(full["xhat"][f, :code.N], fr.s[f]):
            assert tr[f, -1] == code.N * code.p


def test_trace_point_cases():
    """Degenerate cases of the count: estimate = truth -> N*p; every bit wrong -> 0."""
    p, N, M = 2, 2, 2
    # x0 + x1 + n0 = z0, x1 + n1 = z1 (coefficients 1), noise evidence certain
    rows = np.array([0, 0, 0, 1, 1], np.int32)
    cols = np.array([0, 1, 2, 1, 3], np.int32)
    vals = np.ones(5, np.uint8)
    oc = oracle.OCode(p, POLY[p], N, M, rows, cols, vals)
    s = np.array([[1, 2]], np.uint8)
    # hard bits = t + n with n = 0: z = H [s; 0] = (s0^s1, s1); received t = B^-1 A s here B = I
    t_sym = np.array([s[0, 0] ^ s[0, 1], s[0, 1]], np.uint8)
    hard = synth.symbols_to_bits(t_sym[None], p).astype(np.uint8)
    pi = np.full((1, M * p), 1e-9)
    out = oc.decode(hard, pi, max_iters=3, s_true=s)
    it = out["iters"][0]
    assert it >= 1 and np.array_equal(out["xhat"][0, :N], s[0])
    assert (out["trace"][0, it:] == N * p).all()
    # x^(0): uniform source priors clip to symbol 0 -> bits of s that are 0 are right
    assert out["trace"][0, 0] == _correct_bits_by_hand(np.zeros(N, np.uint8), s[0], p)
    flipped = (s ^ 3).astype(np.uint8)   # every bit of the truth inverted
    out2 = oc.decode(hard, pi, max_iters=3, s_true=flipped)
    assert (out2["trace"][0, it:] == 0).all()


def test_embedded_binary_chain_matches_bit_chain():
    """The GF(8) symbol chain built from the 2S matrix gives the same
    law as the binary chain read 3 bits at a time: brute force over all bit
    strings of two symbols."""
    T2 = synth.MARKOV_2S
    T8 = synth.markov_embed_binary(T2, 3)
    assert np.allclose(T8.sum(axis=1), 1.0, atol=1e-12)
    for a in range(8):
        for b in range(8):
            bits = [(a >> k) & 1 for k in range(3)] + [(b >> k) & 1 for k in range(3)]
            pr_b_given_a = np.prod([T2[bits[k - 1], bits[k]] for k in range(3, 6)])
            assert math.isclose(T8[a, b], pr_b_given_a, rel_tol=1e-12)
    # symmetric 2S: uniform bits, so the symbol law is 1/2 * prod of the in-symbol transitions
    pi = [0.5 * T2[b & 1, (b >> 1) & 1] * T2[(b >> 1) & 1, (b >> 2) & 1] for b in range(8)]
    assert np.allclose(synth.stationary(T8), pi, atol=1e-12)


# ----------------------------------------------------------------------------- within-sweep prior (A34, f2)
def test_markov_prior_one_matches_eq6_block():
    """The per-symbol prior with explicit neighbours equals the (pinned) Eq. (6)
    block prior at an interior symbol and at both boundaries."""
    rng = np.random.default_rng(4)
    q, N = 4, 5
    T = rng.random((q, q)); T /= T.sum(axis=1, keepdims=True)
    pi0 = synth.stationary(T)
    Q = rng.random((N, q)); Q /= Q.sum(axis=1, keepdims=True)
    P = oracle.markov_prior(T, pi0, Q)
    assert np.allclose(oracle.markov_prior_one(T, pi0, Q[1], Q[3]), P[2], atol=1e-14)
    assert np.allclose(oracle.markov_prior_one(T, pi0, None, Q[1]), P[0], atol=1e-14)
    assert np.allclose(oracle.markov_prior_one(T, pi0, Q[N - 2], None), P[N - 1], atol=1e-14)
    assert np.allclose(oracle.markov_prior_one(T, pi0, None, None), pi0, atol=1e-14)


def _two_source_chain(s0=1):
    """GF(2): sources s0, s1 (s1 in no check), one check s0 + n0 = z0 with a
    noise bit known to be 0: s0 is decoded exactly in the first sweep."""
    oc = oracle.OCode(1, POLY[1], 2, 1, np.array([0, 0], np.int32), np.array([0, 2], np.int32),
                      np.array([1, 1], np.uint8))
    hard = np.array([[s0]], np.uint8)                 # r = t = s0 (B = [1], A = [1 0])
    pi = np.array([[1e-12]])
    return oc, hard, pi


def test_within_sweep_prior_closed_form():
    """SUS with the prior refreshed inside the sweep: after ONE iteration the
    unchecked source s1 already carries T[s0] (its left neighbour was decoded
    earlier in the same sweep); with the post-iteration snapshot (A9) it is
    still pi0 after one iteration and T[s0] after two."""
    T = np.array([[0.9, 0.1], [0.2, 0.8]])
    pi0 = synth.stationary(T)
    oc, hard, pi = _two_source_chain(1)
    gs1 = oc.decode(hard, pi, schedule=oracle.SUS, max_iters=1, fixed=True, T=T, pi0=pi0, keep_messages=True,
                    sus_gs=True)
    assert np.allclose(gs1["Q"][0, 0], [0.0, 1.0], atol=1e-9)
    assert np.allclose(gs1["Q"][0, 1], T[1], atol=1e-9)
    sn1 = oc.decode(hard, pi, schedule=oracle.SUS, max_iters=1, fixed=True, T=T, pi0=pi0, keep_messages=True)
    assert np.allclose(sn1["Q"][0, 1], pi0, atol=1e-12)
    sn2 = oc.decode(hard, pi, schedule=oracle.SUS, max_iters=2, fixed=True, T=T, pi0=pi0, keep_messages=True)
    assert np.allclose(sn2["Q"][0, 1], T[1], atol=1e-9)
    # second GS sweep: s0's prior now has the right factor from s1's first-sweep posterior
    gs2 = oc.decode(hard, pi, schedule=oracle.SUS, max_iters=2, fixed=True, T=T, pi0=pi0, keep_messages=True,
                    sus_gs=True)
    assert np.allclose(gs2["Q"][0, 1], T[1], atol=1e-9)


def test_within_sweep_prior_reduces_to_iid_for_memoryless_T():
    """T with identical rows (no memory): Eq. (6) gives the row itself at every
    symbol, so the within-sweep SUS decode equals the i.i.d. decode."""
    c = synth.CONFIGS["C2"]
    code = synth.code_for(c)
    fr = synth.frames_for(c, code, range(3))
    oc = oracle.OCode.from_synth(code)
    hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs)
    row = np.array([0.4, 0.3, 0.2, 0.1])
    T = np.tile(row, (4, 1))
    a = oc.decode(hard, pi, schedule=oracle.SUS, max_iters=4, fixed=True, T=T, pi0=row, keep_messages=True,
                  sus_gs=True)
    b = oc.decode(hard, pi, schedule=oracle.SUS, max_iters=4, fixed=True, pi0=row, keep_messages=True)
    assert np.max(np.abs(a["Q"] - b["Q"])) < 1e-12 and np.array_equal(a["iters"], b["iters"])


# ----------------------------------------------------------------------------- SUS column order (f2, A35)
@pytest.mark.parametrize("z", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_sus_order_reversed_fresh_read_closed_form(z):
    """The sweep visits the columns in the given order (P:198-216 with the order of
    reading A35): on the chain x0 - c0 - x1 - c1 - x2 visited 2, 1, 0, ONE sweep gives
    x0 the exact marginal p0(a) p1(z0+a) p2(z0+z1+a), while x2 (visited first) has
    only p2(a) p1(z1+a) -- the mirror image of the index-order closed form."""
    oc = chain_code()
    pi0 = np.array([0.3, 0.7])
    p1, p2 = 0.2, 0.4
    hard = np.array([[z[0], z[0] ^ z[1]]], np.uint8)
    pi = np.array([[p1, p2]])
    pr0, pr1, pr2 = pi0, np.array([1 - p1, p1]), np.array([1 - p2, p2])
    z0, z1 = z
    exact0 = np.array([pr0[a] * pr1[z0 ^ a] * pr2[z0 ^ z1 ^ a] for a in range(2)])
    first2 = np.array([pr2[a] * pr1[z1 ^ a] for a in range(2)])
    out = oc.decode(hard, pi, schedule=oracle.SUS, max_iters=1, fixed=True, pi0=pi0, keep_messages=True,
                    sus_order=np.array([[2, 1, 0]]))
    assert np.allclose(out["Q"][0, 0], exact0 / exact0.sum(), atol=1e-15)
    assert np.allclose(out["Q"][0, 2], first2 / first2.sum(), atol=1e-15)
    # index order: x0 first, so after one sweep it lacks x2's evidence
    nat = oc.decode(hard, pi, schedule=oracle.SUS, max_iters=1, fixed=True, pi0=pi0, keep_messages=True)
    lack = np.array([pr0[a] * pr1[z0 ^ a] for a in range(2)])
    assert np.allclose(nat["Q"][0, 0], lack / lack.sum(), atol=1e-15)


def test_sus_order_identity_is_index_order():
    c = synth.CONFIGS["C1"]
    code = synth.code_for(c)
    fr = synth.frames_for(c, code, range(3))
    oc = oracle.OCode.from_synth(code)
    hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs)
    a = oc.decode(hard, pi, schedule=oracle.SUS, max_iters=4, fixed=True, keep_messages=True)
    b = oc.decode(hard, pi, schedule=oracle.SUS, max_iters=4, fixed=True, keep_messages=True,
                  sus_order=np.arange(code.V)[None])
    for k in ("q", "r", "Q"):
        assert np.array_equal(a[k], b[k])


@pytest.mark.parametrize("p", [1, 2])
def test_sus_order_tree_exactness(p):
    """On cycle-free H, SUS with a different random column order every sweep still
    reaches the brute-force marginals (BP is exact on trees under any schedule)."""
    rng = np.random.default_rng(70 + p)
    q = 1 << p
    done = 0
    while done < 6:
        M = int(rng.integers(2, 5))
        tc = random_tree_code(rng, M, q)
        if tc is None:
            continue
        N, rows, cols, vals = tc
        if N + M > (10 if p == 1 else 7):
            continue
        oc, hard, pi, z = setup_frame(rng, p, N, M, rows, cols, vals)
        pi0 = rng.random(q)
        pi0 /= pi0.sum()
        priors = [pi0] * N + [oracle.noise_prior(p, pi[k * p:(k + 1) * p]) for k in range(M)]
        want = brute_marginals(p, N, M, rows, cols, vals, z, priors)
        orders = np.stack([rng.permutation(N + M) for _ in range(3)])
        out = oc.decode(hard[None], pi[None], schedule=oracle.SUS, max_iters=2 * (N + M), fixed=True,
                        pi0=pi0, keep_messages=True, threads=1, sus_order=orders)
        assert np.max(np.abs(out["Q"][0] - want)) < 1e-9
        done += 1


def test_sus_order_fixed_points_agree_with_pus():
    """A fixed point does not depend on the schedule: SUS in random orders and PUS agree."""
    rng = np.random.default_rng(15)
    agreed = 0
    for trial in range(20):
        p, N, M = 2, 3, 5
        q = 1 << p
        rows, cols = [], []
        for j in range(N + M):
            for i in rng.choice(M, 2, replace=False):
                rows.append(i); cols.append(j)
        rows = np.array(rows, np.int32)
        cols = np.array(cols, np.int32)
        vals = rng.integers(1, q, len(rows)).astype(np.uint8)
        oc, hard, pi, z = setup_frame(rng, p, N, M, rows, cols, vals)
        pi *= 0.3
        orders = np.stack([rng.permutation(N + M) for _ in range(5)])
        res = []
        for kw in (dict(schedule=oracle.PUS), dict(schedule=oracle.SUS, sus_order=orders)):
            o1 = oc.decode(hard[None], pi[None], max_iters=400, fixed=True, keep_messages=True, **kw)
            o2 = oc.decode(hard[None], pi[None], max_iters=405, fixed=True, keep_messages=True, **kw)
            res.append((np.max(np.abs(o1["Q"] - o2["Q"])) < 1e-13, o1["Q"][0]))
        if res[0][0] and res[1][0]:
            assert np.max(np.abs(res[0][1] - res[1][1])) < 1e-9
            agreed += 1
    assert agreed >= 5

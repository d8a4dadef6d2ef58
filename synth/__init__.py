"""Seeded synthetic inputs for GF(2^p) MacKay-Neal BP decoding.

This module is the ONE thing shared by the oracle (`oracle/`) and the CUDA path
(`paper_cs_0605069_b200/`): it produces *inputs* only -- a code (sparse A, B
with GF(q) coefficients), source words, their encoding, and the channel output.
It contains none of the decoder's arithmetic (no syndrome, no priors, no
message passing).  Its GF(2^p) multiply (log/antilog tables, used only by the
encoder Eq. (1)) is a third, independent implementation: the oracle multiplies
by shift-and-xor and the CUDA library builds its own tables.

Recipe:
  * A (M x N): column weight 3 on distinct rows, row slots a shuffled multiset
    in which every row appears at least once, best-effort 4-cycle rejection,
    coefficients uniform on {1..q-1}
  * B (M x M): seeded column-permuted bidiagonal chain, invertible over any
    GF(2^p) ("B must be invertible"; reading A23)
  * encoding t = B^-1 A s (Eq. 1) by forward substitution along the chain
  * symbols -> p bits LSB first (reading A2); channel BSC / BEC / BI-AWGN
    (readings A15, A16)
Every frame f of point k draws from its own PCG64 stream keyed by
(base_seed, config id, k, f), so any subset of frames reproduces exactly.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

# Primitive polynomials (reading A1).  p=1 uses x+1 (GF(2): multiply = AND).
PRIM_POLY = {1: 0x3, 2: 0x7, 3: 0xB, 4: 0x13, 5: 0x25, 6: 0x43, 7: 0x89}  # 7: x^7+x^3+1 (f4)

BSC, BEC, BIAWGN = 0, 1, 2
CHANNEL_NAMES = {BSC: "bsc", BEC: "bec", BIAWGN: "biawgn"}


# ----------------------------------------------------------------------------
# Config table (BASELINE.json configs[0..4] = C1..C5)
# ----------------------------------------------------------------------------
@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    cid: int
    p: int
    N: int
    M: int
    frames: int
    source: str          # "iid" or "markov"
    stay: float          # Markov stay probability (reading A12)
    channel: int
    ch_params: tuple     # BSC f | BEC eps | BI-AWGN Eb/N0 points (dB)
    max_iters: int
    fixed_iters: int = 0  # throughput run length (C5: 50)

    @property
    def q(self) -> int:
        return 1 << self.p

    @property
    def E(self) -> int:
        return 3 * self.N + 2 * self.M - 1

    @property
    def V(self) -> int:
        return self.N + self.M


CONFIGS = {
    "C1": Config("C1", 1, 1, 500, 1000, 64, "iid", 0.0, BSC, (0.06,), 100),
    "C2": Config("C2", 2, 2, 2000, 4000, 1024, "markov", 0.85, BSC, (0.05,), 200),
    "C3": Config("C3", 3, 3, 4000, 8000, 4096, "iid", 0.0, BIAWGN,
                 (0.5, 1.0, 1.5, 2.0, 2.5, 3.0), 200),
    "C4": Config("C4", 4, 4, 8000, 16000, 8192, "markov", 0.9, BEC, (0.35,), 300),
    "C5": Config("C5", 5, 6, 10000, 20000, 8192, "iid", 0.0, BIAWGN, (1.5,), 400, 50),
    # supplementary (not a BASELINE config): C5's construction over GF(128)
    "X7": Config("X7", 6, 7, 10000, 20000, 4096, "iid", 0.0, BIAWGN, (1.5,), 400, 50),
}


def awgn_sigma(ebn0_db: float, rate_bits: float = 0.5) -> float:
    """sigma for unit-energy BPSK at Eb/N0 (reading A16): s^2 = 1/(2 R 10^(EbN0/10))."""
    return math.sqrt(1.0 / (2.0 * rate_bits * 10.0 ** (ebn0_db / 10.0)))


def markov_uniform_jump(q: int, stay: float) -> np.ndarray:
    """T_aa = stay, T_ab = (1-stay)/(q-1) (reading A12)."""
    T = np.full((q, q), (1.0 - stay) / (q - 1), dtype=np.float64)
    np.fill_diagonal(T, stay)
    return T


# Paper footnote matrices, kept verbatim as printed.
MARKOV_2S = np.array([[0.89, 0.11], [0.11, 0.89]])
MARKOV_4S = np.array([
    [0.808022, 0.0883281, 0.0130689, 0.0905813],
    [0.128676, 0.0514706, 0.0772059, 0.742647],
    [0.755814, 0.108527, 0.0116279, 0.124031],
    [0.866667, 0.0151111, 0.091556, 0.0266659],
])


# ----------------------------------------------------------------------------
# Encoder-side GF(2^p): log/antilog tables (independent of oracle and CUDA)
# ----------------------------------------------------------------------------
class _GFTables:
    def __init__(self, p: int, poly: Optional[int] = None):
        self.p = p
        self.q = 1 << p
        self.poly = PRIM_POLY[p] if poly is None else poly
        q = self.q
        exp = np.zeros(2 * q, dtype=np.int64)
        log = np.full(q, -1, dtype=np.int64)
        a = 1
        for k in range(q - 1):
            exp[k] = a
            if log[a] != -1:
                raise ValueError("polynomial 0x%x is not primitive" % self.poly)
            log[a] = k
            a <<= 1
            if a & q:
                a ^= self.poly
            a &= (2 * q - 1)
        for k in range(q - 1, 2 * q):
            exp[k] = exp[k % (q - 1)] if q > 1 else 1
        self.exp, self.log = exp, log
        mul = np.zeros((q, q), dtype=np.uint8)
        for x in range(1, q):
            for y in range(1, q):
                mul[x, y] = exp[(log[x] + log[y]) % (q - 1)]
        inv = np.zeros(q, dtype=np.uint8)
        for x in range(1, q):
            inv[x] = exp[(q - 1 - log[x]) % (q - 1)]
        self.mul, self.inv = mul, inv


_GF_CACHE: dict = {}


def gf_tables(p: int) -> _GFTables:
    if p not in _GF_CACHE:
        _GF_CACHE[p] = _GFTables(p)
    return _GF_CACHE[p]


# ----------------------------------------------------------------------------
# Code construction
# ----------------------------------------------------------------------------
@dataclasses.dataclass
class Code:
    p: int
    N: int
    M: int
    A_row: np.ndarray   # int32 [nnzA]
    A_col: np.ndarray
    A_val: np.ndarray   # uint8
    B_row: np.ndarray   # int32 [nnzB]  (B columns are noise symbols 0..M-1)
    B_col: np.ndarray
    B_val: np.ndarray
    chain_perm: np.ndarray  # sigma: chain position k -> noise column sigma[k]
    chain_diag: np.ndarray  # d_k
    chain_sub: np.ndarray   # c_k (k < M-1): B[k+1][sigma[k]]
    seed: int

    @property
    def q(self) -> int:
        return 1 << self.p

    @property
    def poly(self) -> int:
        return PRIM_POLY[self.p]

    @property
    def V(self) -> int:
        return self.N + self.M

    @property
    def E(self) -> int:
        return len(self.A_row) + len(self.B_row)

    def H_coo(self):
        """H = [A B] as COO (rows = checks, cols = variables x = [s; n])."""
        rows = np.concatenate([self.A_row, self.B_row]).astype(np.int32)
        cols = np.concatenate([self.A_col, self.B_col + self.N]).astype(np.int32)
        vals = np.concatenate([self.A_val, self.B_val]).astype(np.uint8)
        return rows, cols, vals


def _rng(*key) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(k) & 0xFFFFFFFF for k in key])))


def make_code(p: int, N: int, M: int, seed: int, colw: int = 3,
              permute_noise: bool = True, cycle_retries: int = 100) -> Code:
    """Seeded MN code (recipe in the module docstring)."""
    q = 1 << p
    rng = _rng(0xC0DE, seed, p, N, M)
    if colw * N < M:
        raise ValueError("colw*N must cover every row at least once")
    # Row slot multiset: every row once, the remainder spread as evenly as possible.
    extra = colw * N - M
    slots = np.concatenate([np.arange(M), rng.permutation(np.tile(np.arange(M), (extra + M - 1) // M))[:extra]])
    slots = rng.permutation(slots)
    cols = slots.reshape(N, colw).copy()
    # Repair duplicates within a column by swapping with random other slots.
    for _ in range(1000):
        bad = [c for c in range(N) if len(set(cols[c])) < colw]
        if not bad:
            break
        for c in bad:
            for k in range(colw):
                if list(cols[c]).count(cols[c, k]) > 1:
                    c2 = int(rng.integers(N))
                    k2 = int(rng.integers(colw))
                    if cols[c2, k2] not in cols[c] and cols[c, k] not in cols[c2]:
                        cols[c, k], cols[c2, k2] = cols[c2, k2], cols[c, k]
    else:
        raise RuntimeError("could not repair duplicate rows")
    # Best-effort 4-cycle removal: two columns sharing >= 2 rows.
    for _ in range(cycle_retries):
        pair_owner = {}
        bad = []
        for c in range(N):
            r = sorted(cols[c])
            for a in range(colw):
                for b in range(a + 1, colw):
                    key = (r[a], r[b])
                    if key in pair_owner:
                        bad.append(c)
                    else:
                        pair_owner[key] = c
        if not bad:
            break
        for c in set(bad):
            k = int(rng.integers(colw))
            c2 = int(rng.integers(N))
            k2 = int(rng.integers(colw))
            if cols[c2, k2] not in cols[c] and cols[c, k] not in cols[c2]:
                cols[c, k], cols[c2, k2] = cols[c2, k2], cols[c, k]
    A_col = np.repeat(np.arange(N, dtype=np.int32), colw)
    A_row = cols.reshape(-1).astype(np.int32)
    A_val = rng.integers(1, q, size=len(A_row)).astype(np.uint8)
    order = np.lexsort((A_col, A_row))
    A_row, A_col, A_val = A_row[order], A_col[order], A_val[order]
    # B = C * P_sigma: chain C[k][k] = d_k, C[k+1][k] = c_k.
    sigma = rng.permutation(M).astype(np.int32) if permute_noise else np.arange(M, dtype=np.int32)
    d = rng.integers(1, q, size=M).astype(np.uint8)
    csub = rng.integers(1, q, size=max(M - 1, 0)).astype(np.uint8)
    B_row = np.concatenate([np.arange(M), np.arange(1, M)]).astype(np.int32)
    B_col = np.concatenate([sigma, sigma[:M - 1]]).astype(np.int32)
    B_val = np.concatenate([d, csub]).astype(np.uint8)
    order = np.lexsort((B_col, B_row))
    return Code(p, N, M, A_row, A_col, A_val, B_row[order], B_col[order], B_val[order],
                sigma, d, csub, seed)


def code_for(cfg: Config, permute_noise: bool = True) -> Code:
    return make_code(cfg.p, cfg.N, cfg.M, 0x5EED0000 + cfg.cid, permute_noise=permute_noise)


# ----------------------------------------------------------------------------
# Frames: source -> Eq. (1) encoding -> bits -> channel
# ----------------------------------------------------------------------------
@dataclasses.dataclass
class Frames:
    channel: int
    ch_param: float       # BSC f | BEC eps | BI-AWGN sigma
    s: np.ndarray         # uint8 [F][N]   source symbols (truth)
    t: np.ndarray         # uint8 [F][M]   codeword symbols
    n: np.ndarray         # uint8 [F][M]   noise symbols (truth; r = t + n mod 2)
    obs: np.ndarray       # BSC: uint8 bits; BEC: uint8 {0,1,2=erased}; BI-AWGN: float32 y  [F][M*p]

    @property
    def F(self) -> int:
        return self.s.shape[0]

    def x_true(self) -> np.ndarray:
        return np.concatenate([self.s, self.n], axis=1)


def _gf_matvec_coo(tab: _GFTables, rows, cols, vals, nrows, X):
    """Y[:, i] = XOR_k vals*X[:, cols] over rows (encoder use only)."""
    F = X.shape[0]
    Y = np.zeros((F, nrows), dtype=np.uint8)
    prod = tab.mul[vals[None, :].astype(np.int64), X[:, cols].astype(np.int64)]
    order = np.argsort(rows, kind="stable")
    r_sorted = rows[order]
    prod = prod[:, order]
    starts = np.flatnonzero(np.r_[True, r_sorted[1:] != r_sorted[:-1]])
    red = np.bitwise_xor.reduceat(prod, starts, axis=1)
    Y[:, r_sorted[starts]] = red
    return Y


def encode(code: Code, s: np.ndarray) -> np.ndarray:
    """t = B^-1 A s (Eq. 1) by forward substitution along the chain."""
    tab = gf_tables(code.p)
    y = _gf_matvec_coo(tab, code.A_row, code.A_col, code.A_val, code.M, s)
    F, M = s.shape[0], code.M
    u = np.zeros((F, M), dtype=np.uint8)
    inv_d = tab.inv[code.chain_diag]
    prev = np.zeros(F, dtype=np.uint8)
    for k in range(M):
        acc = y[:, k]
        if k > 0:
            acc = acc ^ tab.mul[code.chain_sub[k - 1], prev]
        prev = tab.mul[inv_d[k], acc]
        u[:, k] = prev
    t = np.zeros_like(u)
    t[:, code.chain_perm] = u
    return t


def symbols_to_bits(sym: np.ndarray, p: int) -> np.ndarray:
    """LSB-first bits (reading A2): bit index k*p + b."""
    F, M = sym.shape
    return ((sym[:, :, None] >> np.arange(p, dtype=np.uint8)) & 1).astype(np.uint8).reshape(F, M * p)


def bits_to_symbols(bits: np.ndarray, p: int) -> np.ndarray:
    F = bits.shape[0]
    b = bits.reshape(F, -1, p).astype(np.uint8)
    return (b << np.arange(p, dtype=np.uint8)).sum(axis=2).astype(np.uint8)


def make_frames(code: Code, cfg_id: int, frame_ids, source: str, channel: int, ch_param: float,
                stay: float = 0.0, point: int = 0, base_seed: int = 0x0D15EA5E,
                T: Optional[np.ndarray] = None) -> Frames:
    """Frames for the given frame indices (each from its own stream, so subsets reproduce).

    source: "iid" (uniform) or "markov" (uniform-jump chain with stay prob,
    s_0 from the stationary distribution pi0 = uniform, readings A12/A14) or "markov_T"
    with an explicit T (stationary start computed by power iteration).
    ch_param: BSC flip prob f, BEC erasure prob eps, BI-AWGN sigma.
    """
    frame_ids = np.asarray(frame_ids, dtype=np.int64)
    F = len(frame_ids)
    q, p, N, M = code.q, code.p, code.N, code.M
    rngs = [_rng(base_seed, cfg_id, point, int(f)) for f in frame_ids]
    # --- source
    if source == "iid":
        s = np.stack([r.integers(0, q, size=N, dtype=np.uint8) for r in rngs]) if F else np.zeros((0, N), np.uint8)
    else:
        if T is None:
            T = markov_uniform_jump(q, stay)
        pi0 = stationary(T)
        U = np.stack([r.random(N) for r in rngs]) if F else np.zeros((0, N))
        cumT = np.cumsum(T, axis=1)
        cum0 = np.cumsum(pi0)
        s = np.zeros((F, N), dtype=np.uint8)
        s[:, 0] = np.minimum(np.searchsorted(cum0, U[:, 0], side="right"), q - 1)
        for k in range(1, N):
            c = cumT[s[:, k - 1]]
            s[:, k] = np.minimum((U[:, k:k + 1] >= c).sum(axis=1), q - 1)
    # --- Eq. (1)
    t = encode(code, s)
    tb = symbols_to_bits(t, p)
    nb = M * p
    # --- channel (per-bit)
    if channel == BSC:
        flips = np.stack([(r.random(nb) < ch_param) for r in rngs]).astype(np.uint8) if F else np.zeros((0, nb), np.uint8)
        obs = tb ^ flips
        nbits = flips
    elif channel == BEC:
        er = np.stack([(r.random(nb) < ch_param) for r in rngs]) if F else np.zeros((0, nb), bool)
        obs = np.where(er, np.uint8(2), tb).astype(np.uint8)
        nbits = np.where(er, tb, 0).astype(np.uint8)     # erased bit filled with 0 (reading A15)
    elif channel == BIAWGN:
        g = np.stack([r.standard_normal(nb, dtype=np.float32) for r in rngs]) if F else np.zeros((0, nb), np.float32)
        obs = (1.0 - 2.0 * tb.astype(np.float32)) + np.float32(ch_param) * g
        obs = obs.astype(np.float32)
        nbits = ((obs < 0).astype(np.uint8) ^ tb)        # hard decision y<0 -> 1 (reading A16)
    else:
        raise ValueError("unknown channel")
    n = bits_to_symbols(nbits, p)
    return Frames(channel, float(ch_param), s, t, n, obs)


def frames_for(cfg: Config, code: Code, frame_ids, point: int = 0) -> Frames:
    ch = cfg.channel
    param = cfg.ch_params[point]
    if ch == BIAWGN:
        param = awgn_sigma(param)
    return make_frames(code, cfg.cid, frame_ids, cfg.source, ch, param, stay=cfg.stay, point=point)


def stationary(T: np.ndarray, iters: int = 10000) -> np.ndarray:
    q = T.shape[0]
    pi = np.full(q, 1.0 / q)
    for _ in range(iters):
        nxt = pi @ T
        if np.max(np.abs(nxt - pi)) < 1e-15:
            pi = nxt
            break
        pi = nxt
    return pi / pi.sum()


def markov_embed_binary(T2: np.ndarray, p: int) -> np.ndarray:
    """Symbol-level transition matrix of a binary Markov chain read p bits per
    GF(2^p) symbol, bit 0 first (reading A2): T[a][b] = T2[a_{p-1}][b_0] *
    prod_{k>=1} T2[b_{k-1}][b_k].  The paper's GF(8) rows use the 2-state
    source this way (an ambiguity of the paper)."""
    q = 1 << p
    T = np.zeros((q, q), dtype=np.float64)
    for a in range(q):
        prev = (a >> (p - 1)) & 1
        for b in range(q):
            v, last = 1.0, prev
            for k in range(p):
                bit = (b >> k) & 1
                v *= T2[last, bit]
                last = bit
            T[a, b] = v
    return T


def markov_T_for(cfg: Config) -> Optional[np.ndarray]:
    return markov_uniform_jump(cfg.q, cfg.stay) if cfg.source == "markov" else None

"""CPU oracle of the Monte-Carlo front end: the steps before
the decoder -- source, encoding t = B^-1 A s (Eq. 1), channel
 -- driven by the counter-based generator that include/gfq.h
specifies for gfq_simulate.

TEST INFRASTRUCTURE ONLY (like the rest of oracle/): imported by tests/ and
never by the product package.  Plain numpy, vectorised over frames, written
from the definitions; GF(2^p) products come from the oracle's own
shift-and-xor multiply (oracle.gf_mul), encoding solves B t = A s by peeling
rows with a single unknown (B is triangular up to permutation for the MN
construction, reading A23).

Random numbers (include/gfq.h, gfq_simulate):
  Philox4x32-10 with key (seed mod 2^32, seed >> 32) and counter
  (j, frame mod 2^32, frame >> 32, purpose); purpose 1 = source, 2 = channel.
  u24(x) = (x >> 8) * 2^-24.
  source  i.i.d.: symbol 4j+m = x_m mod q;
          Markov: u_k = u24(x_m), k = 4j+m; s_0 = min{b : u_0 < C0[b]},
                  s_k = min{b : u_k < C[s_{k-1}][b]}, C the running row sums of
                  pi0 / T in double, last entry 1.
  channel BSC: bit 4j+m flips iff u24(x_m) < f; BEC: erased iff u24(x_m) < eps;
          BI-AWGN: bits 2j, 2j+1 from one call: u1 = ((x0 >> 8) + 1) 2^-24,
          u2 = u24(x1), rho = sqrt(-2 ln u1), n = rho cos(2 pi u2), rho sin(2 pi u2);
          y = (1 - 2 bit) + sigma n, rounded to float32 (reading A16: 0 -> +1).
"""
from __future__ import annotations

import numpy as np

from . import gf_mul, gf_inv

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = 0x9E3779B9, 0xBB67AE85
MASK = np.uint64(0xFFFFFFFF)
PURPOSE_SOURCE, PURPOSE_CHANNEL = 1, 2


def philox4x32_10(c0, c1, c2, c3, k0: int, k1: int):
    """Philox4x32 with 10 rounds (Salmon et al., SC'11) on uint32 arrays."""
    c = [np.asarray(x, dtype=np.uint64) & MASK for x in (c0, c1, c2, c3)]
    k0, k1 = int(k0) & 0xFFFFFFFF, int(k1) & 0xFFFFFFFF
    for r in range(10):
        if r > 0:
            k0 = (k0 + W0) & 0xFFFFFFFF
            k1 = (k1 + W1) & 0xFFFFFFFF
        p0 = M0 * c[0]
        p1 = M1 * c[2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK
        c = [hi1 ^ c[1] ^ np.uint64(k0), lo1, hi0 ^ c[3] ^ np.uint64(k1), lo0]
    return [x.astype(np.uint32) for x in c]


def _draws(seed: int, frames, purpose: int, nblocks: int):
    """[4][F][nblocks] uint32: Philox outputs for counters (j, frame, purpose)."""
    frames = np.asarray(frames, dtype=np.uint64)
    j = np.arange(nblocks, dtype=np.uint64)[None, :]
    fr = frames[:, None]
    c0 = np.broadcast_to(j, (len(frames), nblocks))
    c1 = np.broadcast_to(fr & MASK, (len(frames), nblocks))
    c2 = np.broadcast_to(fr >> np.uint64(32), (len(frames), nblocks))
    c3 = np.full((len(frames), nblocks), purpose, dtype=np.uint64)
    return philox4x32_10(c0, c1, c2, c3, seed & 0xFFFFFFFF, seed >> 32)


def u24(x):
    return (np.asarray(x, dtype=np.uint32) >> np.uint32(8)).astype(np.float64) * 2.0 ** -24


def running_sums(P) -> np.ndarray:
    """Row-wise running sums in double, accumulated left to right, last entry 1."""
    P = np.atleast_2d(np.asarray(P, dtype=np.float64))
    C = np.zeros_like(P)
    for r in range(P.shape[0]):
        acc = 0.0
        for b in range(P.shape[1]):
            acc += P[r, b]
            C[r, b] = acc
        C[r, -1] = 1.0
    return C


def source(seed: int, frames, N: int, q: int, T=None, pi0=None) -> np.ndarray:
    F = len(frames)
    nb = (N + 3) // 4
    x = _draws(seed, frames, PURPOSE_SOURCE, nb)
    X = np.stack(x, axis=-1).reshape(F, nb * 4)[:, :N]          # element 4j+m = x_m of block j
    if T is None:
        return (X & np.uint32(q - 1)).astype(np.uint8)
    u = u24(X)
    C0 = running_sums(np.full(q, 1.0 / q) if pi0 is None else pi0)[0]
    CT = running_sums(T)
    s = np.zeros((F, N), np.uint8)
    s[:, 0] = (u[:, :1] >= C0[None, :]).sum(axis=1)
    for k in range(1, N):
        s[:, k] = (u[:, k:k + 1] >= CT[s[:, k - 1]]).sum(axis=1)
    return s


def _mul_table(p: int, poly: int) -> np.ndarray:
    q = 1 << p
    return np.array([[gf_mul(a, b, p, poly) for b in range(q)] for a in range(q)], dtype=np.uint8)


def encode(p: int, poly: int, N: int, M: int, rows, cols, vals, s) -> np.ndarray:
    """t with B t = A s over GF(2^p) (Eq. 1): H = [A B] as COO over variables
    0..N+M-1 (noise/codeword symbol k is variable N+k).  Peels rows of B with a
    single unknown column; raises if B is not triangular up to permutation."""
    mul = _mul_table(p, poly)
    rows = np.asarray(rows); cols = np.asarray(cols); vals = np.asarray(vals)
    F = s.shape[0]
    y = np.zeros((F, M), np.uint8)
    a = cols < N
    for i, j, h in zip(rows[a], cols[a], vals[a]):
        y[:, i] ^= mul[h][s[:, j]]
    brow = [[] for _ in range(M)]
    bcols_of = [[] for _ in range(M)]
    for i, j, h in zip(rows[~a], cols[~a] - N, vals[~a]):
        brow[i].append((int(j), int(h)))
        bcols_of[int(j)].append(int(i))
    unknown = np.array([len(r) for r in brow])
    solved = np.zeros(M, bool)
    t = np.zeros((F, M), np.uint8)
    stack = [i for i in range(M) if unknown[i] == 1]
    done_rows = np.zeros(M, bool)
    nsolved = 0
    while stack:
        i = stack.pop()
        if done_rows[i] or unknown[i] != 1:
            continue
        done_rows[i] = True
        acc = y[:, i].copy()
        target = None
        for j, h in brow[i]:
            if solved[j]:
                acc ^= mul[h][t[:, j]]
            else:
                target = (j, h)
        j, h = target
        t[:, j] = mul[gf_inv(h, p, poly)][acc]
        solved[j] = True
        nsolved += 1
        for i2 in bcols_of[j]:
            unknown[i2] -= 1
            if unknown[i2] == 1 and not done_rows[i2]:
                stack.append(i2)
    if nsolved != M:
        raise ValueError("B is not triangular up to a permutation (peeling stopped)")
    return t


def channel(seed: int, frames, t, p: int, ch: int, param: float):
    """obs [F][M*p]: BSC uint8 bits, BEC uint8 {0,1,2}, BI-AWGN float32 (ch 0/1/2)."""
    F, M = t.shape
    nbits = M * p
    bits = ((t[:, :, None] >> np.arange(p, dtype=np.uint8)) & 1).reshape(F, nbits).astype(np.uint8)
    if ch in (0, 1):
        nb = (nbits + 3) // 4
        x = _draws(seed, frames, PURPOSE_CHANNEL, nb)
        U = u24(np.stack(x, axis=-1).reshape(F, nb * 4)[:, :nbits])
        hit = U < float(param)
        if ch == 0:
            return (bits ^ hit).astype(np.uint8)
        return np.where(hit, np.uint8(2), bits).astype(np.uint8)
    nb = (nbits + 1) // 2
    x = _draws(seed, frames, PURPOSE_CHANNEL, nb)
    u1 = ((x[0] >> np.uint32(8)).astype(np.float64) + 1.0) * 2.0 ** -24
    u2 = u24(x[1])
    rho = np.sqrt(-2.0 * np.log(u1))
    n = np.stack([rho * np.cos(2.0 * np.pi * u2), rho * np.sin(2.0 * np.pi * u2)], axis=-1).reshape(F, nb * 2)
    y = (1.0 - 2.0 * bits.astype(np.float64)) + float(param) * n[:, :nbits]
    return y.astype(np.float32)


def simulate(code_coo, seed: int, frames, ch: int, param: float, T=None, pi0=None):
    """code_coo = (p, poly, N, M, rows, cols, vals) of H = [A B].  Returns (s, t, obs)."""
    p, poly, N, M, rows, cols, vals = code_coo
    q = 1 << p
    s = source(seed, frames, N, q, T, pi0)
    t = encode(p, poly, N, M, rows, cols, vals, s)
    obs = channel(seed, frames, t, p, ch, param)
    return s, t, obs

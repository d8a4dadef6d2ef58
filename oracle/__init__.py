"""Python handle on the fp64 C oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py -- never by the product
package paper_cs_0605069_b200.  Frames are decoded one per call, in parallel
over a thread pool (ctypes releases the GIL), as SURVEY.md §8(c) c4 plans.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

PUS, SUS = 0, 1
BSC, BEC, BIAWGN = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (plain -O2, fp64, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            P = ctypes.POINTER
            d, i, u8 = ctypes.c_double, ctypes.c_int, ctypes.c_uint8
            vp = ctypes.c_void_p
            L.o_gf_mul.argtypes = [i, i, i, ctypes.c_uint]
            L.o_gf_mul.restype = i
            L.o_gf_inv.argtypes = [i, i, ctypes.c_uint]
            L.o_gf_inv.restype = i
            L.o_frontend.argtypes = [i, d, vp, ctypes.c_long, vp, vp]
            L.o_noise_prior.argtypes = [i, vp, vp]
            L.o_check_node.argtypes = [i, ctypes.c_uint, i, vp, vp, i, i, vp]
            L.o_var_node.argtypes = [i, i, vp, vp, i, vp]
            L.o_var_node.restype = i
            L.o_posterior.argtypes = [i, i, vp, vp, vp, P(i)]
            L.o_posterior.restype = i
            L.o_markov_prior.argtypes = [i, i, vp, vp, vp, vp]
            L.o_code_create.argtypes = [i, ctypes.c_uint, i, i, ctypes.c_long, vp, vp, vp]
            L.o_code_create.restype = vp
            L.o_code_destroy.argtypes = [vp]
            L.o_syndrome.argtypes = [vp, vp, vp]
            L.o_unsatisfied.argtypes = [vp, vp, vp]
            L.o_unsatisfied.restype = i
            L.o_decode_frame.argtypes = [vp, i, i, i, vp, vp, vp, vp, vp, P(i), vp, vp, vp,
                                         P(ctypes.c_long), vp, vp, i, vp, i]
            L.o_markov_prior_one.argtypes = [i, vp, vp, vp, vp, vp]
            L.o_decode_frame.restype = i
            _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------- per-op API
def gf_mul(a: int, b: int, p: int, poly: int) -> int:
    return lib().o_gf_mul(int(a), int(b), p, poly)


def gf_inv(a: int, p: int, poly: int) -> int:
    return lib().o_gf_inv(int(a), p, poly)


def frontend(channel: int, param: float, obs: np.ndarray):
    """obs (any shape) -> (hard bits uint8, pi float64) with the same shape."""
    obs_c = np.ascontiguousarray(obs, dtype=np.float32 if channel == BIAWGN else np.uint8)
    hard = np.zeros(obs_c.shape, np.uint8)
    pi = np.zeros(obs_c.shape, np.float64)
    lib().o_frontend(channel, float(param), _p(obs_c), obs_c.size, _p(hard), _p(pi))
    return hard, pi


def noise_prior(p: int, pi_bits) -> np.ndarray:
    pi_bits = np.ascontiguousarray(pi_bits, dtype=np.float64)
    out = np.zeros(1 << p, np.float64)
    lib().o_noise_prior(p, _p(pi_bits), _p(out))
    return out


def check_node(p: int, poly: int, h, qin, z: int, out: int) -> np.ndarray:
    h = np.ascontiguousarray(h, dtype=np.int32)
    qin = np.ascontiguousarray(qin, dtype=np.float64)
    r = np.zeros(1 << p, np.float64)
    lib().o_check_node(p, poly, len(h), _p(h), _p(qin), int(z), int(out), _p(r))
    return r


def var_node(prior, rin, out: int):
    prior = np.ascontiguousarray(prior, dtype=np.float64)
    rin = np.ascontiguousarray(rin, dtype=np.float64).reshape(-1, len(prior))
    qo = np.zeros(len(prior), np.float64)
    zero = lib().o_var_node(len(prior), rin.shape[0], _p(prior), _p(rin), int(out), _p(qo))
    return qo, zero


def posterior(prior, rin):
    prior = np.ascontiguousarray(prior, dtype=np.float64)
    rin = np.ascontiguousarray(rin, dtype=np.float64).reshape(-1, len(prior))
    Q = np.zeros(len(prior), np.float64)
    zf = ctypes.c_int(0)
    x = lib().o_posterior(len(prior), rin.shape[0], _p(prior), _p(rin), _p(Q), ctypes.byref(zf))
    return Q, x, zf.value


def markov_prior(T, pi0, Q) -> np.ndarray:
    T = np.ascontiguousarray(T, dtype=np.float64)
    pi0 = np.ascontiguousarray(pi0, dtype=np.float64)
    Q = np.ascontiguousarray(Q, dtype=np.float64)
    N, q = Q.shape
    P = np.zeros((N, q), np.float64)
    lib().o_markov_prior(q, N, _p(T), _p(pi0), _p(Q), _p(P))
    return P


def markov_prior_one(T, pi0, left=None, right=None) -> np.ndarray:
    T = np.ascontiguousarray(T, dtype=np.float64)
    pi0 = np.ascontiguousarray(pi0, dtype=np.float64)
    lf = None if left is None else np.ascontiguousarray(left, dtype=np.float64)
    rt = None if right is None else np.ascontiguousarray(right, dtype=np.float64)
    out = np.zeros(len(pi0), np.float64)
    lib().o_markov_prior_one(len(pi0), _p(T), _p(pi0), _p(lf), _p(rt), _p(out))
    return out


# ---------------------------------------------------------------- code + decode
class OCode:
    """H = [A B] from COO (rows = checks, cols = variables 0..N+M-1)."""

    def __init__(self, p: int, poly: int, N: int, M: int, rows, cols, vals):
        self.p, self.poly, self.N, self.M = p, poly, N, M
        self.q = 1 << p
        self.V = N + M
        rows = np.ascontiguousarray(rows, dtype=np.int32)
        cols = np.ascontiguousarray(cols, dtype=np.int32)
        vals = np.ascontiguousarray(vals, dtype=np.uint8)
        self.E = len(rows)
        self._h = lib().o_code_create(p, poly, N, M, self.E, _p(rows), _p(cols), _p(vals))
        # canonical edge order (column-major, then row) for message export
        order = np.lexsort((rows, cols))
        self.edge_rows, self.edge_cols = rows[order], cols[order]

    @classmethod
    def from_synth(cls, code) -> "OCode":
        r, c, v = code.H_coo()
        return cls(code.p, code.poly, code.N, code.M, r, c, v)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().o_code_destroy(h)
            self._h = None

    def syndrome(self, r_sym) -> np.ndarray:
        r_sym = np.ascontiguousarray(r_sym, dtype=np.uint8)
        z = np.zeros(self.M, np.uint8)
        lib().o_syndrome(self._h, _p(r_sym), _p(z))
        return z

    def unsatisfied(self, x, z) -> int:
        x = np.ascontiguousarray(x, dtype=np.uint8)
        z = np.ascontiguousarray(z, dtype=np.uint8)
        return lib().o_unsatisfied(self._h, _p(x), _p(z))

    def decode(self, hard, pi, schedule: int = PUS, max_iters: int = 100, fixed: bool = False,
               T=None, pi0=None, keep_messages: bool = False, threads: int = 0, s_true=None,
               sus_gs: bool = False, sus_order=None):
        """Decode frames. hard uint8 [F][M*p], pi float64 [F][M*p] (fp32 values may be
        passed: they are widened exactly).  Returns dict(xhat [F][V], iters [F],
        zero_norms [F], and q/r [F][E][q], Q [F][V][q] if keep_messages; with the true
        sources s_true uint8 [F][N] also trace [F][max_iters+1], the correct source
        bits of the estimate after each iteration (Fig. 1)).  sus_order: int
        [n][V], SUS sweep t visits columns sus_order[(t-1) % n] (reading A35); None =
        index order (A7)."""
        hard = np.ascontiguousarray(hard, dtype=np.uint8)
        pi = np.ascontiguousarray(pi, dtype=np.float64)
        F = hard.shape[0]
        q, E, V = self.q, self.E, self.V
        xhat = np.zeros((F, V), np.uint8)
        iters = np.zeros(F, np.int32)
        zn = np.zeros(F, np.int64)
        qm = np.zeros((F, E, q)) if keep_messages else None
        rm = np.zeros((F, E, q)) if keep_messages else None
        Qm = np.zeros((F, V, q)) if keep_messages else None
        Tc = None if T is None else np.ascontiguousarray(T, dtype=np.float64)
        p0 = None if pi0 is None else np.ascontiguousarray(pi0, dtype=np.float64)
        st = None if s_true is None else np.ascontiguousarray(s_true, dtype=np.uint8).reshape(F, self.N)
        tr = None if s_true is None else np.zeros((F, max(int(max_iters), 0) + 1), np.int32)
        od = None if sus_order is None else np.ascontiguousarray(sus_order, dtype=np.int32).reshape(-1, V)
        if od is not None:
            assert not sus_gs, "sus_order is not combined with the in-sweep prior"
            assert all(np.array_equal(np.sort(o), np.arange(V)) for o in od), "each order must permute 0..V-1"
        L = lib()

        def one(f):
            it = ctypes.c_int(0)
            z = ctypes.c_long(0)
            L.o_decode_frame(self._h, schedule, int(max_iters), int(bool(fixed)),
                             _p(hard[f]), _p(pi[f]), _p(Tc), _p(p0), _p(xhat[f]), ctypes.byref(it),
                             _p(qm[f]) if keep_messages else None,
                             _p(rm[f]) if keep_messages else None,
                             _p(Qm[f]) if keep_messages else None, ctypes.byref(z),
                             None if st is None else _p(st[f]), None if tr is None else _p(tr[f]),
                             int(bool(sus_gs)), _p(od), 0 if od is None else len(od))
            iters[f] = it.value
            zn[f] = z.value

        nthreads = threads or os.cpu_count() or 1
        if nthreads == 1 or F <= 1:
            for f in range(F):
                one(f)
        else:
            with ThreadPoolExecutor(max_workers=min(nthreads, F)) as ex:
                list(ex.map(one, range(F)))
        out = dict(xhat=xhat, iters=iters, zero_norms=zn, threads=min(nthreads, max(F, 1)))
        if keep_messages:
            out.update(q=qm, r=rm, Q=Qm)
        if tr is not None:
            out["trace"] = tr
        return out

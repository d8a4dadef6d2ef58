"""Thin Python binding of libgfq (include/gfq.h) over ctypes.

Argument marshalling only: every step of the decode runs in the CUDA kernels of
libgfq.so.  PyTorch provides device memory and the current stream.  There is no
CPU fallback: if libgfq.so is missing or no CUDA device is present the calls
raise.  Function names mirror the C ABI (gfq_code_create, gfq_decode, ...).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GFQ_LIB_PATH") or os.path.join(_HERE, "libgfq.so")

GFQ_OK, GFQ_EINVAL, GFQ_ENOMEM, GFQ_ECUDA, GFQ_EUNSUPPORTED = 0, -1, -2, -3, -4
GFQ_BSC, GFQ_BEC, GFQ_BIAWGN = 0, 1, 2
GFQ_PUS, GFQ_SUS = 0, 1
GFQ_PRIOR_SNAPSHOT, GFQ_PRIOR_IN_SWEEP = 0, 1
GFQ_COMPACT_FRAMES, GFQ_COMPACT_BLOCKS = 0, 1

# Every symbol declared in include/gfq.h (checked by tests/test_abi.py).
EXPORTS = ["gfq_last_error", "gfq_version", "gfq_code_create", "gfq_code_destroy", "gfq_code_info",
           "gfq_workspace_bytes", "gfq_decode", "gfq_decode_evidence", "gfq_workspace_bytes_host",
           "gfq_decode_host", "gfq_export_messages", "gfq_decode_stats", "gfq_profile_enable",
           "gfq_profile_read", "gfq_kernel_name", "gfq_simulate_workspace_bytes", "gfq_simulate"]
GFQ_NKERNELS = 15


class GfqError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__("libgfq error %d: %s" % (code, msg))
        self.code = code


class gfq_params(ctypes.Structure):
    _fields_ = [("channel", ctypes.c_int), ("ch_param", ctypes.c_double),
                ("schedule", ctypes.c_int), ("max_iters", ctypes.c_int),
                ("early_exit", ctypes.c_int), ("markov_T", ctypes.c_void_p),
                ("src_pi0", ctypes.c_void_p), ("keep_messages", ctypes.c_int),
                ("trace_truth", ctypes.c_void_p), ("trace", ctypes.c_void_p),
                ("prior_update", ctypes.c_int), ("sus_order", ctypes.c_void_p),
                ("sus_n_orders", ctypes.c_int), ("compaction", ctypes.c_int)]


class gfq_sim_params(ctypes.Structure):
    _fields_ = [("channel", ctypes.c_int), ("ch_param", ctypes.c_double),
                ("markov_T", ctypes.c_void_p), ("src_pi0", ctypes.c_void_p)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libgfq.so (built in-tree by paper_cs_0605069_b200/build.py)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError("libgfq.so is not built (run __graft_entry__.build()); there is no fallback")
        L = ctypes.CDLL(LIB_PATH)
        vp, i, ll, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong, ctypes.c_size_t
        P = ctypes.POINTER
        L.gfq_last_error.restype = ctypes.c_char_p
        L.gfq_version.restype = i
        L.gfq_code_create.argtypes = [P(vp), i, ctypes.c_uint, i, i, ll, vp, vp, vp, ll, vp, vp, vp]
        L.gfq_code_create.restype = i
        L.gfq_code_destroy.argtypes = [vp]
        L.gfq_code_info.argtypes = [vp, P(ll), P(i), P(i), P(i)]
        L.gfq_code_info.restype = i
        L.gfq_workspace_bytes.argtypes = [vp, i, P(gfq_params)]
        L.gfq_workspace_bytes.restype = sz
        L.gfq_workspace_bytes_host.argtypes = [vp, i, P(gfq_params)]
        L.gfq_workspace_bytes_host.restype = sz
        L.gfq_decode.argtypes = [vp, i, vp, P(gfq_params), vp, vp, vp, sz, vp]
        L.gfq_decode.restype = i
        L.gfq_decode_evidence.argtypes = [vp, i, vp, vp, P(gfq_params), vp, vp, vp, sz, vp]
        L.gfq_decode_evidence.restype = i
        L.gfq_decode_host.argtypes = [vp, i, vp, P(gfq_params), vp, vp, vp, sz, vp]
        L.gfq_decode_host.restype = i
        L.gfq_export_messages.argtypes = [vp, i, vp, sz, P(gfq_params), vp, vp, vp, vp]
        L.gfq_export_messages.restype = i
        L.gfq_decode_stats.argtypes = [vp, vp, sz, P(ll), vp]
        L.gfq_decode_stats.restype = i
        L.gfq_profile_enable.argtypes = [i]
        L.gfq_profile_enable.restype = i
        L.gfq_profile_read.argtypes = [vp, vp]
        L.gfq_profile_read.restype = i
        L.gfq_simulate_workspace_bytes.argtypes = [vp, i]
        L.gfq_simulate_workspace_bytes.restype = sz
        L.gfq_simulate.argtypes = [vp, i, ctypes.c_ulonglong, ll, P(gfq_sim_params), vp, vp, vp, vp, sz, vp]
        L.gfq_simulate.restype = i
        L.gfq_kernel_name.argtypes = [i]
        L.gfq_kernel_name.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _check(rc: int):
    if rc != GFQ_OK:
        raise GfqError(rc, lib().gfq_last_error().decode())


def _stream_ptr(stream=None) -> Optional[int]:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _dptr(t) -> int:
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return t.data_ptr()


def _expect(t, name, dtype, shape, device=None, cuda=True):
    """Marshalling checks: the C side trusts pointers and sizes completely."""
    import torch
    if not isinstance(t, torch.Tensor):
        raise TypeError("%s: expected a torch tensor" % name)
    if t.dtype != dtype:
        raise TypeError("%s: expected dtype %s, got %s" % (name, dtype, t.dtype))
    if tuple(t.shape) != tuple(shape):
        raise ValueError("%s: expected shape %s, got %s" % (name, tuple(shape), tuple(t.shape)))
    if not t.is_contiguous():
        raise ValueError("%s: expected a contiguous tensor" % name)
    if cuda and not t.is_cuda:
        raise ValueError("%s: expected a CUDA tensor" % name)
    if not cuda and t.is_cuda:
        raise ValueError("%s: expected a host tensor" % name)
    if device is not None and t.device != device:
        raise ValueError("%s: on %s, expected %s" % (name, t.device, device))


def _obs_dtype(params: "Params"):
    import torch
    return torch.float32 if params.c.channel == GFQ_BIAWGN else torch.uint8


class Params:
    """gfq_params plus the host arrays it points to (kept alive)."""

    def __init__(self, channel=GFQ_BSC, ch_param=0.0, schedule=GFQ_PUS, max_iters=100,
                 early_exit=True, markov_T=None, src_pi0=None, keep_messages=False,
                 trace_truth=None, trace=None, prior_update=GFQ_PRIOR_SNAPSHOT, sus_order=None,
                 compaction=GFQ_COMPACT_FRAMES):
        """trace_truth / trace: CUDA tensors uint8 [F][N] and int32 [F][max_iters+1]
        (Fig. 1 instrumentation, see include/gfq.h), or None."""
        self._T = None if markov_T is None else np.ascontiguousarray(markov_T, dtype=np.float64)
        self._trace = (trace_truth, trace)
        self._pi0 = None if src_pi0 is None else np.ascontiguousarray(src_pi0, dtype=np.float64)
        self._ord = None if sus_order is None else np.ascontiguousarray(np.atleast_2d(sus_order), dtype=np.int32)
        self.c = gfq_params(int(channel), float(ch_param), int(schedule), int(max_iters),
                            int(bool(early_exit)),
                            None if self._T is None else self._T.ctypes.data,
                            None if self._pi0 is None else self._pi0.ctypes.data,
                            int(bool(keep_messages)), _dptr(trace_truth), _dptr(trace),
                            int(prior_update),
                            None if self._ord is None else self._ord.ctypes.data,
                            0 if self._ord is None else int(self._ord.shape[0]),
                            int(compaction))

    def ref(self):
        return ctypes.byref(self.c)


class Code:
    """gfq_code_create / gfq_code_destroy / gfq_code_info."""

    def __init__(self, p: int, poly: int, N: int, M: int, A_row, A_col, A_val, B_row, B_col, B_val):
        arrs = [np.ascontiguousarray(x, dtype=dt) for x, dt in
                ((A_row, np.int32), (A_col, np.int32), (A_val, np.uint8),
                 (B_row, np.int32), (B_col, np.int32), (B_val, np.uint8))]
        h = ctypes.c_void_p()
        _check(lib().gfq_code_create(ctypes.byref(h), p, poly, N, M, len(arrs[0]),
                                     arrs[0].ctypes.data, arrs[1].ctypes.data, arrs[2].ctypes.data,
                                     len(arrs[3]), arrs[3].ctypes.data, arrs[4].ctypes.data,
                                     arrs[5].ctypes.data))
        self.h = h
        self.p, self.q, self.N, self.M, self.V = p, 1 << p, N, M, N + M
        E, dc, dv, lv = ctypes.c_longlong(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _check(lib().gfq_code_info(h, ctypes.byref(E), ctypes.byref(dc), ctypes.byref(dv), ctypes.byref(lv)))
        self.E, self.max_check_deg, self.max_var_deg, self.sus_levels = E.value, dc.value, dv.value, lv.value

    @classmethod
    def from_synth(cls, code) -> "Code":
        return cls(code.p, code.poly, code.N, code.M, code.A_row, code.A_col, code.A_val,
                   code.B_row, code.B_col, code.B_val)

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value and _lib is not None:
            _lib.gfq_code_destroy(h)
            self.h = None


def gfq_workspace_bytes(code: Code, n_frames: int, params: Params) -> int:
    return lib().gfq_workspace_bytes(code.h, n_frames, params.ref())


def gfq_workspace_bytes_host(code: Code, n_frames: int, params: Params) -> int:
    return lib().gfq_workspace_bytes_host(code.h, n_frames, params.ref())


def alloc_workspace(nbytes: int, device="cuda"):
    import torch
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def gfq_decode(code: Code, obs, params: Params, s_hat=None, iters=None, workspace=None, stream=None):
    """obs: CUDA tensor [F][M*p] (uint8 for BSC/BEC, float32 for BI-AWGN)."""
    import torch
    F = obs.shape[0]
    _expect(obs, "obs", _obs_dtype(params), (F, code.M * code.p))
    if s_hat is None:
        s_hat = torch.empty((F, code.N), dtype=torch.uint8, device=obs.device)
    if iters is None:
        iters = torch.empty(F, dtype=torch.int32, device=obs.device)
    if workspace is None:
        workspace = alloc_workspace(gfq_workspace_bytes(code, F, params), obs.device)
    _expect(s_hat, "s_hat", torch.uint8, (F, code.N), obs.device)
    _expect(iters, "iters", torch.int32, (F,), obs.device)
    _expect(workspace, "workspace", torch.uint8, (workspace.numel(),), obs.device)
    _check(lib().gfq_decode(code.h, F, _dptr(obs), params.ref(), _dptr(s_hat), _dptr(iters),
                            _dptr(workspace), workspace.numel(), _stream_ptr(stream)))
    return s_hat, iters, workspace


def gfq_decode_evidence(code: Code, hard_bits, bit_flip_prob, params: Params, x_hat=None, iters=None,
                        workspace=None, stream=None):
    import torch
    F = hard_bits.shape[0]
    dev = hard_bits.device
    _expect(hard_bits, "hard_bits", torch.uint8, (F, code.M * code.p))
    _expect(bit_flip_prob, "bit_flip_prob", torch.float32, (F, code.M * code.p), dev)
    if x_hat is None:
        x_hat = torch.empty((F, code.V), dtype=torch.uint8, device=dev)
    if iters is None:
        iters = torch.empty(F, dtype=torch.int32, device=dev)
    if workspace is None:
        workspace = alloc_workspace(gfq_workspace_bytes(code, F, params), dev)
    _expect(x_hat, "x_hat", torch.uint8, (F, code.V), dev)
    _expect(iters, "iters", torch.int32, (F,), dev)
    _expect(workspace, "workspace", torch.uint8, (workspace.numel(),), dev)
    _check(lib().gfq_decode_evidence(code.h, F, _dptr(hard_bits), _dptr(bit_flip_prob), params.ref(),
                                     _dptr(x_hat), _dptr(iters), _dptr(workspace), workspace.numel(),
                                     _stream_ptr(stream)))
    return x_hat, iters, workspace


def gfq_decode_host(code: Code, obs_host, params: Params, s_hat_host=None, iters_host=None,
                    workspace=None, stream=None):
    """obs_host: host (ideally pinned) tensor/array; returns host s_hat, iters. Synchronous."""
    import torch
    obs_t = torch.as_tensor(obs_host)
    F = obs_t.shape[0]
    if s_hat_host is None:
        s_hat_host = torch.empty((F, code.N), dtype=torch.uint8).pin_memory()
    if iters_host is None:
        iters_host = torch.empty(F, dtype=torch.int32).pin_memory()
    if workspace is None:
        workspace = alloc_workspace(gfq_workspace_bytes_host(code, F, params))
    obs_t = obs_t.contiguous()
    _expect(obs_t, "obs_host", _obs_dtype(params), (F, code.M * code.p), cuda=False)
    _expect(s_hat_host, "s_hat_host", torch.uint8, (F, code.N), cuda=False)
    _expect(iters_host, "iters_host", torch.int32, (F,), cuda=False)
    _expect(workspace, "workspace", torch.uint8, (workspace.numel(),))
    _check(lib().gfq_decode_host(code.h, F, obs_t.data_ptr(), params.ref(), s_hat_host.data_ptr(),
                                 iters_host.data_ptr(), _dptr(workspace), workspace.numel(),
                                 _stream_ptr(stream)))
    return s_hat_host, iters_host, workspace


def gfq_export_messages(code: Code, n_frames: int, workspace, params: Params, q=True, r=True, Q=True,
                        stream=None):
    import torch
    dev = workspace.device
    _expect(workspace, "workspace", torch.uint8, (workspace.numel(),))
    qo = torch.empty((n_frames, code.E, code.q), dtype=torch.float32, device=dev) if q else None
    ro = torch.empty((n_frames, code.E, code.q), dtype=torch.float32, device=dev) if r else None
    Qo = torch.empty((n_frames, code.V, code.q), dtype=torch.float32, device=dev) if Q else None
    _check(lib().gfq_export_messages(code.h, n_frames, _dptr(workspace), workspace.numel(), params.ref(),
                                     _dptr(qo), _dptr(ro), _dptr(Qo), _stream_ptr(stream)))
    return qo, ro, Qo


def gfq_decode_stats(code: Code, workspace, stream=None):
    out = (ctypes.c_longlong * 4)()
    _check(lib().gfq_decode_stats(code.h, _dptr(workspace), workspace.numel(), out, _stream_ptr(stream)))
    return dict(zero_normalisers=out[0], block_iterations=out[1], frames_converged=out[2],
                launches=out[3])


def gfq_profile_enable(on: bool = True):
    _check(lib().gfq_profile_enable(int(bool(on))))


def gfq_profile_read():
    """{kernel name: (total ms, launches)} for the decodes since gfq_profile_enable(True)."""
    ms = (ctypes.c_double * GFQ_NKERNELS)()
    n = (ctypes.c_longlong * GFQ_NKERNELS)()
    _check(lib().gfq_profile_read(ctypes.addressof(ms), ctypes.addressof(n)))
    return {lib().gfq_kernel_name(k).decode(): (ms[k], n[k]) for k in range(GFQ_NKERNELS)}


def gfq_simulate(code: Code, n_frames: int, seed: int, channel: int, ch_param: float, frame0: int = 0,
                 markov_T=None, src_pi0=None, want_t: bool = False, device="cuda", stream=None):
    """Monte-Carlo frames on the device (include/gfq.h): returns (s [F][N] uint8,
    obs [F][M*p] uint8 or float32, t [F][M] uint8 or None) as CUDA tensors."""
    import torch
    T = None if markov_T is None else np.ascontiguousarray(markov_T, dtype=np.float64)
    p0 = None if src_pi0 is None else np.ascontiguousarray(src_pi0, dtype=np.float64)
    prm = gfq_sim_params(int(channel), float(ch_param), None if T is None else T.ctypes.data,
                         None if p0 is None else p0.ctypes.data)
    F = int(n_frames)
    s = torch.empty((F, code.N), dtype=torch.uint8, device=device)
    obs = torch.empty((F, code.M * code.p), dtype=torch.float32 if channel == GFQ_BIAWGN else torch.uint8,
                      device=device)
    t = torch.empty((F, code.M), dtype=torch.uint8, device=device) if want_t else None
    ws = alloc_workspace(lib().gfq_simulate_workspace_bytes(code.h, F), device)
    _check(lib().gfq_simulate(code.h, F, int(seed) & 0xFFFFFFFFFFFFFFFF, int(frame0), ctypes.byref(prm),
                              _dptr(s), _dptr(obs), _dptr(t), _dptr(ws), ws.numel(), _stream_ptr(stream)))
    return s, obs, t

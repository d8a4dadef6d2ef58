"""The C-ABI library loads and exports every symbol include/gfq.h declares, and the
host-side validation of gfq_code_create / gfq_workspace_bytes behaves as documented
(no compute calls: these run without a GPU)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def gfq():
    import __graft_entry__
    __graft_entry__.build()
    from paper_cs_0605069_b200 import gfq as g
    return g


def header_functions():
    txt = open(os.path.join(ROOT, "include", "gfq.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(gfq_[a-z_]+)\s*\(", txt)))


def test_header_declares_the_binding_names(gfq):
    assert header_functions() == sorted(gfq.EXPORTS)


def test_library_exports_every_symbol(gfq):
    L = gfq.lib()
    for name in header_functions():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", gfq.LIB_PATH], capture_output=True, text=True).stdout
    for name in header_functions():
        assert re.search(r"\bT %s\b" % name, out), name


def test_library_is_sm100a_only(gfq):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", gfq.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert all("sm_100a" in line for line in out.splitlines() if ".cubin" in line)


def _create(gfq, p=2, poly=0x7, N=2, M=2, A=((0, 0, 1), (1, 1, 2)), B=((0, 0, 1), (1, 1, 1))):
    L = gfq.lib()
    A = np.array(A, dtype=np.int64).reshape(-1, 3)
    B = np.array(B, dtype=np.int64).reshape(-1, 3)
    ar, ac, av = (np.ascontiguousarray(A[:, k], dtype=dt) for k, dt in enumerate((np.int32, np.int32, np.uint8)))
    br, bc, bv = (np.ascontiguousarray(B[:, k], dtype=dt) for k, dt in enumerate((np.int32, np.int32, np.uint8)))
    h = ctypes.c_void_p()
    rc = L.gfq_code_create(ctypes.byref(h), p, poly, N, M, len(ar), ar.ctypes.data, ac.ctypes.data,
                           av.ctypes.data, len(br), br.ctypes.data, bc.ctypes.data, bv.ctypes.data)
    if rc == 0:
        L.gfq_code_destroy(h)
    return rc, L.gfq_last_error().decode()


def test_create_validation(gfq):
    assert _create(gfq, p=9, poly=0x211)[0] == gfq.GFQ_EUNSUPPORTED      # q = 512 (f4: q <= 256)
    assert _create(gfq, poly=0xB)[0] == gfq.GFQ_EINVAL                    # wrong degree
    assert _create(gfq, p=4, poly=0x1F)[0] == gfq.GFQ_EINVAL              # irreducible, not primitive
    assert _create(gfq, A=((0, 0, 4),))[0] == gfq.GFQ_EINVAL              # value >= q
    assert _create(gfq, A=((0, 0, 0),))[0] == gfq.GFQ_EINVAL              # zero value
    assert _create(gfq, A=((2, 0, 1),))[0] == gfq.GFQ_EINVAL              # row out of range
    assert _create(gfq, A=((0, 0, 1), (0, 0, 2)))[0] == gfq.GFQ_EINVAL    # duplicate
    assert _create(gfq, B=((0, 5, 1),))[0] == gfq.GFQ_EINVAL              # col out of range
    rc, msg = _create(gfq, A=((0, 0, 1), (0, 1, 1), (0, 2, 1), (0, 3, 1), (0, 4, 1), (0, 5, 1),
                              (0, 6, 1), (0, 7, 1), (0, 8, 1)), N=9)
    assert rc == gfq.GFQ_EUNSUPPORTED                                     # check degree 10 > 8


def test_valid_create_without_gpu_fails_loudly(gfq):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    rc, msg = _create(gfq)
    assert rc == gfq.GFQ_ECUDA and "cuda" in msg.lower()


def test_workspace_bytes_null_args(gfq):
    L = gfq.lib()
    assert L.gfq_workspace_bytes(None, 10, None) == 0
    assert L.gfq_workspace_bytes_host(None, 10, None) == 0


def test_binding_refuses_missing_library(tmp_path, monkeypatch):
    from paper_cs_0605069_b200 import gfq as g
    monkeypatch.setattr(g, "_lib", None)
    monkeypatch.setattr(g, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(RuntimeError):
        g.lib()

"""Race / sync check of the barrier-elided kernels.

k_cn, k_vn and k_sus skip group barriers where an invariant says they are not
needed: one-sided gathers, ping-pong and phased layout switches that reuse a
buffer, no barrier between tasks.  compute-sanitizer
(racecheck / synccheck) is closed on this pool, so the check is differential:
libgfq_synccheck.so is the same code with a full group barrier at every
elision point (GFQ_SYNC_CHECK=1).  A missing barrier that let a warp read a
buffer another warp had not finished writing (or overwrite one still being
read) would change messages; the two builds must agree bit for bit on every
output -- estimates, iteration counts and every exported q, r, Q message -- for
q = 2, 8, 16, 64, 128, PUS and SUS, early exit with ragged blocks, the
in-sweep prior and caller-supplied SUS orders (scripts/sanitize_case.py), and
each build must be deterministic run to run."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _dump(lib, path):
    env = dict(os.environ, GFQ_LIB_PATH=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "sanitize_case.py"), "--dump", path],
                       env=env, capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(path)


def test_sync_check_build_is_bit_identical(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    from paper_cs_0605069_b200 import build as b
    a = _dump(b.LIB, str(tmp_path / "default.npz"))
    a2 = _dump(b.LIB, str(tmp_path / "default2.npz"))
    c = _dump(b.SYNC_CHECK_LIB, str(tmp_path / "checked.npz"))
    assert set(a.files) == set(c.files) and len(a.files) > 40
    for k in a.files:
        assert np.array_equal(a[k], a2[k]), "default build not deterministic: " + k
        assert np.array_equal(a[k], c[k]), "default and barrier-checked builds differ: " + k

"""k_sus_dc64: the q = 64 SUS level kernel by direct convolution (fp32 FFMA2, no
transform, no fp64 layout switch; csrc/gfq_sus_dc64.cu).  It is a measured
alternative to the transform kernel, switched by the environment variable
GFQ_SUS_DC64 (read once per process, off by default: it is slower, DESIGN.md
§13), so its parity gates run in a subprocess with the variable set: the C5
message gate (5 iterations, 64 frames, every q, r, Q within 1e-4 of the fp64
oracle) and the C5 live decision gate of tests/test_gpu_parity.py."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_dc64_variant_passes_the_c5_sus_gates():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, GFQ_SUS_DC64="1")
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-q", "-x",
                        "-p", "no:cacheprovider", "-k", "C5 and SUS and (message_gate or decision_gate)"],
                       env=env, capture_output=True, text=True, timeout=1500, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "2 passed" in r.stdout, r.stdout[-2000:]


def test_transform_check_node_stays_covered_at_q16_and_q8():
    """PUS at q = 8, 16 runs the direct-convolution check node k_cn_dc by default;
    GFQ_CN_DC=0 selects the transform kernel k_cn (still used for check degree
    > 4): its C3 / C4 PUS message gates run here in a subprocess."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, GFQ_CN_DC="0")
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-q", "-x",
                        "-p", "no:cacheprovider", "-k", "(C3 or C4) and PUS and message_gate"],
                       env=env, capture_output=True, text=True, timeout=1500, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "3 passed" in r.stdout, r.stdout[-2000:]

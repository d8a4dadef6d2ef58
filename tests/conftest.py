import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


# GF(256): x^8 + x^4 + x^3 + x^2 + 1, primitive (ord(x) = 255 is pinned
# in test_oracle_pins.py).  Registered here rather than in synth/__init__.py, whose
# hash the d6 oracle goldens record (tests/test_gpu_decisions.py): the generator of
# C1-C5 is unchanged, so the goldens stay current.
import synth  # noqa: E402

synth.PRIM_POLY.setdefault(8, 0x11D)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (still part of the suite)")


def load_golden(name="worked_values.txt"):
    out = {}
    with open(os.path.join(ROOT, "tests", "golden", name)) as fh:
        for line in fh:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            key, vals, cite = [s.strip() for s in line.split("|", 2)]
            out[key] = (np.array([float(v) for v in vals.split()]), cite)
    return out


def load_markov_golden():
    mats, cur = {}, None
    with open(os.path.join(ROOT, "tests", "golden", "markov_matrices.txt")) as fh:
        for line in fh:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            if line[0].isalpha() or line[0].isdigit() and "." not in line:
                cur = line
                mats[cur] = []
            else:
                mats[cur].append([float(v) for v in line.split()])
    return {k: np.array(v) for k, v in mats.items()}


@pytest.fixture(scope="session")
def golden():
    return load_golden()


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    """Print the decision-gate table (mismatches and tie-allowance counts) even under -q."""
    try:
        import gate
    except ImportError:
        return
    if gate.GATE_LOG:
        terminalreporter.write_sep("-", "decision gates (reading A18, tie allowance %g)" % gate.TIE_ALLOW)
        for row in gate.GATE_LOG:
            terminalreporter.write_line(row)

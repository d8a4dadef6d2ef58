"""Write the decision-gate goldens of SURVEY.md §8(d) d6 from the fp64 oracle.

Calls only oracle/ and synth/ (CPU): for every case below, frames 0..n-1 of
the config's seeded host stream (synth.frames_for) are decoded by the oracle
with early exit at the config's max_iters, PUS and SUS, and the per-frame
iteration count (-1 = not converged, reading A21) plus a 64-bit
hash of the source estimate s_hat = x_hat[0:N] are stored under
tests/golden/oracle_decisions/.  tests/test_gpu_decisions.py decodes the same
frames on the GPU and compares frame by frame (reading A18).

Sizes (d6; "at least 6000 samples" is the paper's own count):
C1 and C2 in full, C3 1024 frames at each of the 6 Eb/N0 points, C4 and C5
1024 frames.  Each file records the sha256 of oracle/oracle.c and of
synth/__init__.py it was written with; the GPU test refuses a stale golden.

usage: python scripts/make_oracle_golden.py [--threads 7] [--only C3] [--force]
"""
from __future__ import annotations

import argparse
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "oracle_decisions")

# (config, Eb/N0 point index, frames)
CASES = [("C1", 0, 64), ("C2", 0, 1024), ("C4", 0, 1024)] + \
        [("C3", k, 1024) for k in range(6)] + [("C5", 0, 1024)]


def sha256_file(path: str) -> str:
    with open(path, "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()


def source_hash(x: np.ndarray) -> np.ndarray:
    """64-bit blake2b of each row (uint8 symbols) -> uint64 [F]."""
    x = np.ascontiguousarray(x, dtype=np.uint8)
    return np.array([int.from_bytes(hashlib.blake2b(row.tobytes(), digest_size=8).digest(), "little")
                     for row in x], dtype=np.uint64)


def golden_path(name: str, point: int, schedule: int) -> str:
    return os.path.join(OUT, "%s_p%d_%s.npz" % (name, point, "sus" if schedule else "pus"))


def versions() -> dict:
    return dict(oracle_sha=sha256_file(os.path.join(ROOT, "oracle", "oracle.c")),
                synth_sha=sha256_file(os.path.join(ROOT, "synth", "__init__.py")))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=max(1, (os.cpu_count() or 2) - 1))
    ap.add_argument("--only", default=None)
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--chunk", type=int, default=64)
    args = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    ver = versions()
    for name, point, n in CASES:
        if args.only and name != args.only:
            continue
        cfg = synth.CONFIGS[name]
        code = synth.code_for(cfg)
        oc = oracle.OCode.from_synth(code)
        T = synth.markov_T_for(cfg)
        for schedule in (oracle.PUS, oracle.SUS):
            path = golden_path(name, point, schedule)
            if os.path.exists(path) and not args.force:
                old = np.load(path)
                if str(old["oracle_sha"]) == ver["oracle_sha"] and str(old["synth_sha"]) == ver["synth_sha"] \
                        and int(old["frames"]) == n:
                    print("keep", path, flush=True)
                    continue
            t0 = time.time()
            iters = np.zeros(n, np.int32)
            shash = np.zeros(n, np.uint64)
            zero_norms = 0
            for f0 in range(0, n, args.chunk):
                ids = range(f0, min(n, f0 + args.chunk))
                fr = synth.frames_for(cfg, code, ids, point=point)
                hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs)
                out = oc.decode(hard, pi, schedule=schedule, max_iters=cfg.max_iters, T=T, threads=args.threads)
                iters[f0:f0 + len(ids)] = out["iters"]
                shash[f0:f0 + len(ids)] = source_hash(out["xhat"][:, :code.N])
                zero_norms += int(out["zero_norms"].sum())
                print("  %s p%d %s frames %d..%d  %.0f s" % (name, point, "SUS" if schedule else "PUS", f0,
                                                            f0 + len(ids) - 1, time.time() - t0), flush=True)
            np.savez_compressed(path, iters=iters, shash=shash, frames=n, max_iters=cfg.max_iters,
                                config=name, point=point, schedule=schedule, zero_norms=zero_norms,
                                seconds=time.time() - t0, threads=args.threads, **ver)
            conv = iters[iters > 0]
            print("wrote %s: %d frames, %d converged, mean iters %.2f, %.0f s" % (
                path, n, conv.size, conv.mean() if conv.size else -1, time.time() - t0), flush=True)


if __name__ == "__main__":
    main()

"""Multi-GPU plumbing for the frame-parallel path.

Frames are independent codewords of one shared code (the paper's Monte-Carlo
samples), so N GPUs decode N disjoint frame ranges with no
collective on the data path (weak scaling: each rank keeps its own batch).
One process per GPU; the only collectives are host-side bookkeeping: the
max-over-ranks device time and the gather of per-frame iteration counts.
bench.py runs its timed loop through `run_rank`; tests/test_sharding.py runs
the same function under gloo with the decode call stubbed on the CPU.
"""
from __future__ import annotations

import os
import socket
import subprocess
import sys
from dataclasses import dataclass
from typing import Callable, Optional


def frame_range(rank: int, world: int, frames_per_rank: int) -> range:
    """Frame ids of `rank` in the config's seeded stream: [rank*F, (rank+1)*F)."""
    if not (0 <= rank < world) or frames_per_rank < 0:
        raise ValueError("bad rank / world / frame count")
    return range(rank * frames_per_rank, (rank + 1) * frames_per_rank)


def dist_env():
    """(rank, world, local_rank) from the torchrun environment (1 process: 0, 1, 0)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def _ready(dist) -> bool:
    return dist is not None and dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank scalar (timings are reported as the slowest rank)."""
    if not _ready(dist):
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, dist=None, device=None) -> float:
    if not _ready(dist):
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def gather_objects(obj, dist=None):
    """All ranks' `obj` in rank order (a list of length world)."""
    if not _ready(dist):
        return [obj]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out


@dataclass
class RankResult:
    ms: float                 # this rank's device time of the timed steps
    ms_max: float             # max over ranks (the job's time)
    frames: list              # frame ids of every rank, rank order (rank 0; others: own)
    iters: Optional[list]     # per-frame iteration counts of the last step, rank order


def run_rank(step: Callable[[range], None], frames_per_rank: int, steps: int, warmup: int,
             timer: Callable[[Callable[[], None]], float], dist=None, device=None,
             last_iters: Optional[Callable[[], list]] = None) -> RankResult:
    """The per-rank entry of the frame-sharded bench: this rank's frame range,
    `warmup` untimed steps, a barrier, `steps` timed steps measured by
    `timer(fn)` (CUDA events on the launching stream on a GPU), the max over
    ranks, and the gather of frame ids and per-frame iteration counts."""
    rank = dist.get_rank() if _ready(dist) else 0
    world = dist.get_world_size() if _ready(dist) else 1
    ids = frame_range(rank, world, frames_per_rank)
    for _ in range(warmup):
        step(ids)
    if _ready(dist):
        dist.barrier()

    def timed():
        for _ in range(steps):
            step(ids)
    ms = float(timer(timed))
    ms_max = max_over_ranks(ms, dist, device)
    its = last_iters() if last_iters is not None else None
    got = gather_objects((list(ids), its), dist)
    frames = [i for part in got for i in part[0]]
    iters = None if its is None else [v for part in got for v in part[1]]
    if _ready(dist):
        dist.barrier()
    return RankResult(ms=ms, ms_max=ms_max, frames=frames, iters=iters)


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch_under_torchrun(nprocs: int, argv) -> int:
    """`python bench.py --gpus N` without a torchrun environment: re-run the same
    command as N processes (one per GPU) on this node, rendezvous on 127.0.0.1."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(nprocs),
           "--master-addr", "127.0.0.1", "--master-port", str(free_port())] + list(argv)
    return subprocess.call(cmd)

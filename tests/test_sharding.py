"""The N>1 path's host logic on CPU: world_size-2 gloo processes run bench.py's
per-rank entry (paper_cs_0605069_b200.shard.run_rank: frame range, warm-up,
barrier, timed steps, max over ranks, gather) with only the decode call stubbed
(the fp64 oracle stands in for libgfq on a CPU box); the shards are disjoint
and complete, the gathered per-frame iteration counts equal a single-process
decode, and the job time is the slowest rank's."""
import time
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_cs_0605069_b200 import shard

F_PER_RANK = 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _decode(frame_ids):
    cfg = synth.CONFIGS["C1"]
    code = synth.code_for(cfg)
    fr = synth.frames_for(cfg, code, frame_ids)
    hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs)
    out = oracle.OCode.from_synth(code).decode(hard, pi, schedule=oracle.SUS, max_iters=cfg.max_iters, threads=1)
    return out["xhat"], out["iters"]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        state = {}
        calls = []

        def step(ids):                     # the stubbed decode call
            calls.append(list(ids))
            x, it = _decode(list(ids))
            state["x"], state["it"] = x, it
            if rank == 1:
                time.sleep(0.2)            # rank 1 is the slow one

        def timer(fn):                     # bench.py: CUDA events on the stream
            t0 = time.perf_counter()
            fn()
            return (time.perf_counter() - t0) * 1e3

        res = shard.run_rank(step, F_PER_RANK, steps=2, warmup=1, timer=timer, dist=dist,
                             last_iters=lambda: [int(v) for v in state["it"]])
        xs = shard.gather_objects(state["x"], dist)
        tsum = shard.sum_over_ranks(1.0, dist)
        if rank == 0:
            q.put((res.frames, res.iters, res.ms, res.ms_max, calls, xs, tsum))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_sharding_matches_single_process():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    frames, iters, ms0, ms_max, calls, xs, tsum = q.get()
    assert frames == list(range(world * F_PER_RANK))          # disjoint, complete, in rank order
    assert calls == [list(range(F_PER_RANK))] * 3              # rank 0: 1 warm-up + 2 timed steps
    x_ref, it_ref = _decode(frames)
    assert np.array_equal(np.asarray(iters), it_ref)
    assert np.array_equal(np.concatenate(xs), x_ref)
    assert ms_max >= 400.0 and ms_max >= ms0                   # the slow rank sets the job time
    assert tsum == 2.0


def test_frame_range_validation():
    assert list(shard.frame_range(1, 4, 5)) == [5, 6, 7, 8, 9]
    with pytest.raises(ValueError):
        shard.frame_range(4, 4, 5)
    assert shard.max_over_ranks(3.5) == 3.5

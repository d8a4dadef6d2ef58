"""The N>1 path's host logic on CPU: world_size-2 gloo processes shard the frames
with no overlap, decode their shards independently (oracle stands in for the GPU
here), and the gathered result equals the single-process decode; timings reduce
with MAX."""
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
        ids = shard.frame_range(rank, world, F_PER_RANK)
        x, it = _decode(list(ids))
        got = shard.gather_objects((list(ids), x, it), dist)
        tmax = shard.max_over_ranks(float(rank + 1), dist)
        tsum = shard.sum_over_ranks(1.0, dist)
        if rank == 0:
            q.put((got, tmax, tsum))
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
    got, tmax, tsum = q.get()
    ids = [i for part in got for i in part[0]]
    assert ids == list(range(world * F_PER_RANK))            # disjoint, complete, in rank order
    x_all = np.concatenate([part[1] for part in got])
    it_all = np.concatenate([part[2] for part in got])
    x_ref, it_ref = _decode(ids)
    assert np.array_equal(x_all, x_ref) and np.array_equal(it_all, it_ref)
    assert tmax == 2.0 and tsum == 2.0


def test_frame_range_validation():
    assert list(shard.frame_range(1, 4, 5)) == [5, 6, 7, 8, 9]
    with pytest.raises(ValueError):
        shard.frame_range(4, 4, 5)
    assert shard.max_over_ranks(3.5) == 3.5

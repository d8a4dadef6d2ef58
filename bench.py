"""bench.py -- throughput of batched GF(q) MN-code BP decoding on B200(s).

Contract (driver): `python bench.py --gpus N --steps K --warmup W [--impl reference]`
prints ONE JSON line on rank 0.  A "step" is one pass of the whole hot path
(front end, syndrome, priors, check/variable nodes or the SUS
sweep, convergence test, Markov prior when the source is Markov, output) over
one batch: the batch is decoded with PUS and then with SUS (both schedules of
the paper).  Default workload: C5 (BASELINE.json configs[4]) --
GF(64), N=10000, M=20000, BI-AWGN 1.5 dB, 8192 frames, fixed 50 iterations
(its throughput run), the largest configuration that fits one B200.

value = decoded information bits per second over the whole job (all ranks):
2 decodes x F x N x log2(q) bits per step per rank / max-over-ranks time.
Multi-GPU: every rank decodes its own F frames (frames are independent, no
collective on the data path) -> weak scaling.  `--gpus N` without a torchrun
environment re-runs itself under torch.distributed.run with N processes.
The timed region runs with per-launch instrumentation OFF; one extra,
instrumented step afterwards gives the per-kernel times of the roofline.
`secondary` repeats the measurement on C4 (GF(16), BEC, Markov, 8192 frames,
fixed 50 iterations; BASELINE.json configs[3]).
`--impl reference` times the fp64 CPU oracle (oracle/) on a bounded sample of
the same workload on this host's cores (the reference arm of this tier).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--frames", type=int, default=0, help="override the config's frame count")
    ap.add_argument("--iters", type=int, default=0, help="override the fixed iteration count")
    ap.add_argument("--point", type=int, default=0, help="Eb/N0 point index (C3)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-convergence", action="store_true")
    ap.add_argument("--conv-frames", type=int, default=1024)
    ap.add_argument("--schedules", default="pus,sus")
    ap.add_argument("--host-gen", action="store_true",
                    help="generate the frames with the host generator synth/ instead of gfq_simulate")
    ap.add_argument("--secondary", default="C4", help="second workload in the same line ('' = none)")
    ap.add_argument("--secondary-steps", type=int, default=3)
    ap.add_argument("--secondary-iters", type=int, default=50)
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload(cfg, F, iters):
    ch = synth.CHANNEL_NAMES[cfg.channel]
    return dict(workload="%s: GF(%d) MN code N=%d M=%d E=%d, %s source, %s %s, %d frames/GPU, "
                         "fixed %d iterations, PUS+SUS"
                         % (cfg.name, cfg.q, cfg.N, cfg.M, cfg.E, cfg.source, ch,
                            cfg.ch_params[0], F, iters),
                config_id=cfg.name, q=cfg.q, N=cfg.N, M=cfg.M, E=cfg.E, frames_per_gpu=F,
                fixed_iterations=iters)


def model_bytes_per_frame_iter(cfg):
    """SURVEY.md §8(d) d3 roofline model: 8q bytes per edge-message update, 2E updates
    per frame-iteration, + Markov prior 16Nq + channel + syndrome/decisions."""
    b = 16.0 * cfg.E * cfg.q
    if cfg.source == "markov":
        b += 16.0 * cfg.N * cfg.q
    if cfg.channel == synth.BIAWGN:
        b += 4.0 * cfg.M * cfg.p
    elif cfg.channel == synth.BEC:
        b += cfg.M * cfg.p / 8.0
    return b + cfg.M + cfg.V


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            mp = json.load(fh)
        return float(mp["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return dict(sm_mhz=None, sm_max_mhz=None, reasons=["nvidia-smi unavailable"])
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons, pw = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
                pw.append(float(parts[3]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return dict(sm_mhz=float(np.median(sm)) if sm else None, sm_max_mhz=mx,
                    reasons=sorted(reasons), samples=len(sm),
                    power_w_max=max(pw) if pw else None)


def oracle_sample_rate(cfg, code, frames_obj, sample_frames, sample_iters, schedules):
    """Time the fp64 oracle, as it stands, on a bounded sample; returns (info-bits/s
    extrapolated to the run's fixed iteration count is done by the caller), seconds,
    threads used."""
    import oracle
    oc = oracle.OCode.from_synth(code)
    hard, pi = oracle.frontend(frames_obj.channel, frames_obj.ch_param, frames_obj.obs[:sample_frames])
    T = synth.markov_T_for(cfg)
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    for sch in schedules:
        oc.decode(hard, pi, schedule=sch, max_iters=sample_iters, fixed=True, T=T, threads=threads)
    dt = time.perf_counter() - t0
    return dt, min(threads, sample_frames)


def run_reference(args, cfg, iters, F):
    """--impl reference: the oracle as the reference arm (rank 0 only)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    code = synth.code_for(cfg)
    schedules = [0 if s == "pus" else 1 for s in args.schedules.split(",")]
    ncores = os.cpu_count() or 1
    # one step = a bounded sample: `ncores` frames x `si` iterations per schedule,
    # extrapolated linearly to the fixed iteration count (per-iteration cost is constant)
    si = 1 if cfg.q >= 64 else 2
    sf = max(1, min(ncores, 64))
    fr = synth.frames_for(cfg, code, range(sf), point=args.point)
    for _ in range(args.warmup):
        oracle_sample_rate(cfg, code, fr, sf, si, schedules)
    times = []
    for _ in range(args.steps):
        dt, thr = oracle_sample_rate(cfg, code, fr, sf, si, schedules)
        times.append(dt)
    dt = float(np.mean(times))
    t_full = dt * iters / si                        # seconds for sf frames, all schedules, `iters` iterations
    bits = len(schedules) * sf * cfg.N * cfg.p
    value = bits / t_full
    sample = "%d frames x %d iteration(s) per schedule (%s) per step, extrapolated linearly to %d iterations" % (
        sf, si, args.schedules, iters)
    line = dict(metric="decoded info-bits/s", value=value, unit="bit/s", n_gpus=world, steps=args.steps,
                warmup=args.warmup, ms_per_step=dt * 1e3, higher_is_better=True, scaling="weak",
                vs_baseline=None, dtype="f64", data="synthetic", impl="reference",
                config=workload(cfg, F, iters),
                cpu_baseline=dict(value=value, unit="bit/s", cores=thr, kind="oracle", sample=sample),
                e2e=dict(value=value, unit="bit/s", h2d_bytes_per_step=0, d2h_bytes_per_step=0))
    print(json.dumps(line), flush=True)
    return 0


ARITH = {8: "check node: fp32 direct XOR-convolution (PUS and SUS); variable node fp64; fp32 storage",
         16: "check node: fp32 direct XOR-convolution (PUS and SUS); variable node fp64; fp32 storage",
         64: "fp64 registers (transforms, products, normalisation), fp32 message storage"}


def decode_run(args, cfg, F, iters, schedules, steps, warmup, gfq, shard, dist, rank, world, local,
               full=True):
    """One workload: inputs on the device, `warmup` + `steps` clean timed steps through
    shard.run_rank, one instrumented step for the per-kernel times, the roofline of
    every hot kernel; with full=True also e2e, convergence and the CPU baseline."""
    import gc
    import torch
    gc.collect()
    torch.cuda.empty_cache()          # a previous workload's cached blocks back to the driver
    code = synth.code_for(cfg)
    gcode = gfq.Code.from_synth(code)
    T = synth.markov_T_for(cfg)
    t_gen = time.perf_counter()
    ids = shard.frame_range(rank, world, F)
    param = cfg.ch_params[args.point if cfg.name == args.config else 0]
    if cfg.channel == synth.BIAWGN:
        param = synth.awgn_sigma(param)
    ch = {synth.BSC: gfq.GFQ_BSC, synth.BEC: gfq.GFQ_BEC, synth.BIAWGN: gfq.GFQ_BIAWGN}[cfg.channel]
    seed = 0xBE7C0000 + cfg.cid * 64 + (args.point if cfg.name == args.config else 0)
    if args.host_gen:
        fr = synth.frames_for(cfg, code, ids, point=args.point if cfg.name == args.config else 0)
        obs_host = torch.from_numpy(fr.obs).pin_memory()
        obs = obs_host.to("cuda", non_blocking=True)
        truth = fr.s
    else:
        # Monte-Carlo front end on the device (gfq_simulate, counter-based Philox
        # draws: the same frames for any rank count / subset)
        s_dev, obs, _ = gfq.gfq_simulate(gcode, F, seed, ch, param, frame0=ids[0], markov_T=T)
        obs_host = obs.cpu().pin_memory()
        truth = s_dev.cpu().numpy()
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t_gen
    params = {s: gfq.Params(ch, param, s, iters, early_exit=False, markov_T=T) for s in schedules}
    s_hat = torch.empty((F, cfg.N), dtype=torch.uint8, device="cuda")
    it = torch.empty(F, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    free, total = torch.cuda.mem_get_info()
    need = max(gfq.gfq_workspace_bytes_host(gcode, F, p) for p in params.values())
    ws_bytes = int(min(need, free - (3 << 30)))
    ws = gfq.alloc_workspace(ws_bytes)
    stream = torch.cuda.current_stream()

    def step(_ids=None):
        for s in schedules:
            gfq.gfq_decode(gcode, obs, params[s], s_hat, it, ws, stream)

    def timer(fn):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    clocks = ClockSampler(local)
    gfq.gfq_profile_enable(False)
    torch.cuda.synchronize()
    clocks.start()
    res = shard.run_rank(step, F, steps, warmup, lambda fn: timer(fn), dist=dist if world > 1 else None,
                         device="cuda", last_iters=lambda: it.cpu().tolist())
    clk = clocks.stop()
    ms = res.ms_max
    # one instrumented step: per-kernel CUDA-event times (they break the
    # programmatic-dependent-launch overlap of the SUS levels: a little slower)
    gfq.gfq_profile_enable(True)
    ms_prof = timer(step)
    gfq.gfq_profile_enable(False)
    prof = gfq.gfq_profile_read()
    st = gfq.gfq_decode_stats(gcode, ws)
    launches_per_step = sum(n for _, n in prof.values())
    bits_per_step_rank = len(schedules) * F * cfg.N * cfg.p
    value = bits_per_step_rank * world * steps / (ms / 1e3)
    edge_updates = 2.0 * cfg.E * iters * F * len(schedules) * steps * world

    # roofline of every hot kernel (8q bytes per edge-message update)
    kinds = {k: v for k, v in prof.items() if v[1] > 0}
    peak, peak_src = measured_peak()
    upd_per_frame_iter = {"cn": cfg.E, "vn": cfg.E, "sus": 2 * cfg.E}
    import glob
    roofs = {}
    for kname, (k_ms, k_n) in kinds.items():
        if kname not in upd_per_frame_iter:
            continue
        n_sched = sum(1 for s in schedules if (s == gfq.GFQ_SUS) == (kname == "sus"))
        alg = 8.0 * cfg.q * upd_per_frame_iter[kname] * F * iters * n_sched
        traffic, tsrc = None, None
        for tpath in sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "ncu_traffic*.json")), reverse=True):
            try:
                tj = json.load(open(tpath))
            except Exception:
                continue
            kk = tj.get("kernels", {}).get(kname)
            if tj.get("config") == cfg.name and kk and kk.get("dram_per_alg_byte"):
                traffic = kk["dram_per_alg_byte"] * alg / k_n     # ncu dram bytes per algorithmic byte x this launch
                tsrc = os.path.relpath(tpath, ROOT)
                break
        achieved = alg / (k_ms / 1e3) / 1e9
        roofs[kname] = dict(bound="hbm", kernel=kname, achieved=achieved, peak=peak, unit="GB/s",
                            frac=achieved / peak, traffic=traffic, alg_bytes_per_launch=alg / k_n,
                            launches=k_n, avg_launch_ms=k_ms / k_n, traffic_source=tsrc, peak_source=peak_src)
    dom = max(roofs, key=lambda k: kinds[k][0]) if roofs else None
    # per schedule: the hot kernels of one schedule together (PUS = cn + vn, SUS = the level kernel)
    per_sched = {}
    for sname, ks in (("pus", ("cn", "vn")), ("sus", ("sus",))):
        if all(k in roofs for k in ks):
            t_ms = sum(kinds[k][0] for k in ks)
            alg = 16.0 * cfg.q * cfg.E * F * iters          # 2E updates x 8q bytes per frame-iteration
            per_sched[sname] = dict(kernel_ms_per_step=t_ms, ms_per_iteration=t_ms / iters,
                                    achieved=alg / (t_ms / 1e3) / 1e9, peak=peak, unit="GB/s",
                                    frac=alg / (t_ms / 1e3) / 1e9 / peak)
    model_gbs = model_bytes_per_frame_iter(cfg) * F * iters * len(schedules) * steps / (ms / 1e3) / 1e9
    out = dict(value=value, ms_per_step=ms / steps, ms_per_step_instrumented=ms_prof,
               edge_msg_updates_per_s=edge_updates / (ms / 1e3), model_hbm_gbs=model_gbs,
               roofline=roofs.get(dom), rooflines=roofs, schedule_rooflines=per_sched, clocks=clk,
               gpu_launches=int(launches_per_step * steps),
               kernels={k: dict(ms=v[0], launches=v[1]) for k, v in kinds.items()},
               health=dict(zero_normalisers_last_decode=st["zero_normalisers"]),
               config=dict(workload(cfg, F, iters), arith=ARITH.get(cfg.q, ARITH[64]),
                           parallelism="frame-sharded dp%d (no collective)" % world,
                           l2="inputs larger than L2 (message state %.1f GB/GPU vs 126 MB)" %
                              (cfg.E * cfg.q * 4 * F * 2 / 1e9),
                           timing="clean (no per-launch events); kernels from one extra instrumented step",
                           workspace_gb=ws_bytes / 1e9, input_gen_s=t_gen,
                           input_gen="host synth/ (PCG64)" if args.host_gen else
                           "device gfq_simulate (Philox4x32-10, seed 0x%x)" % seed),
               gathered_frames=len(res.frames))
    if not full:
        return out

    # ---------------- e2e through the host-buffer C-ABI entry
    if not args.no_e2e:
        s_host = torch.empty((F, cfg.N), dtype=torch.uint8).pin_memory()
        it_host = torch.empty(F, dtype=torch.int32).pin_memory()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            for s in schedules:
                gfq.gfq_decode_host(gcode, obs_host, params[s], s_host, it_host, ws, stream)
        t_e2e = time.perf_counter() - t0
        if world > 1:
            t_e2e = shard.max_over_ranks(t_e2e, dist, device="cuda")
        out["e2e"] = dict(value=bits_per_step_rank * world * steps / t_e2e, unit="bit/s",
                          h2d_bytes_per_step=int(obs_host.numel() * obs_host.element_size() * len(schedules)),
                          d2h_bytes_per_step=int((s_host.numel() + it_host.numel() * 4) * len(schedules)))

    # ---------------- convergence run (paper's SUS/PUS iteration ratio), untimed;
    # early-exit cost against the ideal (mean iterations x per-iteration time)
    if not args.no_convergence and rank == 0:
        nf = min(args.conv_frames, F)
        obs_c = obs[:nf].contiguous()
        its = {}
        conv = dict(frames=nf, max_iters=cfg.max_iters)
        for s in schedules:
            name = "pus" if s == gfq.GFQ_PUS else "sus"
            pc = gfq.Params(ch, param, s, cfg.max_iters, early_exit=True, markov_T=T)
            sh, ic, _ = gfq.gfq_decode(gcode, obs_c, pc, workspace=ws, stream=stream)   # warm-up
            c_ms = timer(lambda: gfq.gfq_decode(gcode, obs_c, pc, sh, ic, ws, stream))
            blk_it = gfq.gfq_decode_stats(gcode, ws)["block_iterations"]
            its[s] = ic.cpu().numpy()
            errs = (sh.cpu().numpy() != truth[:nf]).any(axis=1)
            # the same decode with block-granular compaction only (a block runs
            # until its slowest frame stops): what frame-granular compaction saves
            pb = gfq.Params(ch, param, s, cfg.max_iters, early_exit=True, markov_T=T,
                            compaction=gfq.GFQ_COMPACT_BLOCKS)
            shb, icb, _ = gfq.gfq_decode(gcode, obs_c, pb, workspace=ws, stream=stream)
            b_ms = timer(lambda: gfq.gfq_decode(gcode, obs_c, pb, shb, icb, ws, stream))
            blk_it_b = gfq.gfq_decode_stats(gcode, ws)["block_iterations"]
            same = bool(torch.equal(sh, shb) and torch.equal(ic, icb))
            # per-iteration time at this batch: a fixed 10-iteration decode of the same frames
            pf = gfq.Params(ch, param, s, 10, early_exit=False, markov_T=T)
            f_ms = timer(lambda: gfq.gfq_decode(gcode, obs_c, pf, sh, ic, ws, stream)) / 10.0
            ok = its[s] > 0
            spent = np.where(ok, its[s], cfg.max_iters).astype(float)
            conv[name] = dict(mean_iters=float(its[s][ok].mean()) if ok.any() else None,
                              nonconverged=int((~ok).sum()), frame_error_rate=float(errs.mean()),
                              ms_to_converge=c_ms, ms_per_iteration_full_batch=f_ms,
                              ideal_ms=float(spent.mean() * f_ms),
                              measured_over_ideal=float(c_ms / (spent.mean() * f_ms)),
                              block_iterations=int(blk_it), ideal_block_iterations=float(spent.sum() / 32.0),
                              block_granular=dict(ms_to_converge=b_ms, block_iterations=int(blk_it_b),
                                                  measured_over_ideal=float(b_ms / (spent.mean() * f_ms)),
                                                  outputs_identical=same))
        if len(schedules) == 2:
            both = (its[schedules[0]] > 0) & (its[schedules[1]] > 0)
            if both.any():
                tp, ts = its[schedules[0]][both].astype(float), its[schedules[1]][both].astype(float)
                conv.update(paired=int(both.sum()), ratio_of_means=float(ts.mean() / tp.mean()),
                            mean_ratio=float((ts / tp).mean()), std_ratio=float((ts / tp).std()))
        out["convergence"] = conv

    # ---------------- CPU oracle baseline (rank 0, N=1 only): ~10-30 s of the box's cores
    if not args.no_cpu and rank == 0 and world == 1:
        ncores = os.cpu_count() or 1
        si = 3
        sf = max(1, min(4 * ncores, 128))      # ~10-20 s of the host's cores at C5
        sample = argparse.Namespace(channel=cfg.channel, ch_param=param, obs=obs_host[:sf].numpy())
        dt, thr = oracle_sample_rate(cfg, code, sample, sf, si, [0 if s == gfq.GFQ_PUS else 1 for s in schedules])
        t_full = dt * iters / si
        out["cpu_baseline"] = dict(value=len(schedules) * sf * cfg.N * cfg.p / t_full, unit="bit/s", cores=thr,
                                   kind="oracle",
                                   sample="%d frames x %d iterations per schedule (fixed), extrapolated linearly "
                                          "to %d iterations" % (sf, si, iters), seconds=dt)
    del ws
    torch.cuda.empty_cache()
    return out


def main():
    args = parse()
    cfg = synth.CONFIGS[args.config]
    iters = args.iters or cfg.fixed_iters or cfg.max_iters
    F = args.frames or cfg.frames
    if args.impl == "reference":
        return run_reference(args, cfg, iters, F)
    rank, world, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        from paper_cs_0605069_b200 import shard
        return shard.relaunch_under_torchrun(args.gpus, [os.path.abspath(__file__)] + sys.argv[1:])
    if world != args.gpus:
        raise SystemExit("bench.py: --gpus %d but WORLD_SIZE=%d" % (args.gpus, world))

    import torch
    import torch.distributed as dist
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device -- the decoder runs only on the GPU (no CPU fallback)")
    if torch.cuda.device_count() <= local:
        raise SystemExit("bench.py: rank %d needs cuda:%d, only %d device(s)" % (rank, local, torch.cuda.device_count()))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    import __graft_entry__
    __graft_entry__.build()
    from paper_cs_0605069_b200 import gfq, shard

    schedules = [gfq.GFQ_PUS if s == "pus" else gfq.GFQ_SUS for s in args.schedules.split(",")]
    head = decode_run(args, cfg, F, iters, schedules, args.steps, args.warmup, gfq, shard, dist, rank, world, local)
    sec = None
    if args.secondary and args.secondary != cfg.name:
        c2 = synth.CONFIGS[args.secondary]
        sec = decode_run(args, c2, c2.frames, args.secondary_iters, schedules, args.secondary_steps,
                         max(3, min(args.warmup, 3)), gfq, shard, dist, rank, world, local, full=False)
        sec.update(metric="decoded info-bits/s", unit="bit/s", steps=args.secondary_steps)

    if rank == 0:
        line = dict(
            metric="decoded info-bits/s", value=head["value"], unit="bit/s", n_gpus=world, steps=args.steps,
            warmup=args.warmup, ms_per_step=head["ms_per_step"], higher_is_better=True, scaling="weak",
            vs_baseline=None, dtype="f32 storage / f64 arithmetic", data="synthetic",
            config=head["config"],
            edge_msg_updates_per_s=head["edge_msg_updates_per_s"], model_hbm_gbs=head["model_hbm_gbs"],
            ms_per_step_instrumented=head["ms_per_step_instrumented"],
            roofline=head["roofline"], rooflines=head["rooflines"], schedule_rooflines=head["schedule_rooflines"],
            cpu_baseline=head.get("cpu_baseline"),
            e2e=head.get("e2e"), clocks=head["clocks"], gpu_launches=head["gpu_launches"],
            kernels=head["kernels"], health=head["health"], convergence=head.get("convergence"),
            secondary=sec,
        )
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

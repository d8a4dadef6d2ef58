"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the
same seeded inputs.  Gates (BASELINE.json north_star):
  * message gate: after a fixed 5 iterations every q, r, Q message within
    max-abs 1e-4, PUS and SUS, every config (C5 on a subset);
  * decision gate: hard decisions and iterations-to-convergence identical on
    >= 99.9 % of frames (reading A18: frames that fail in both are matched on
    the iteration count only).
"""
import numpy as np
import pytest

import gate
import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

MSG_TOL = 1e-4


@pytest.fixture(scope="module")
def gfq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    from paper_cs_0605069_b200 import gfq as g
    return g


def _setup(name, nframes, point=0, first=0):
    cfg = synth.CONFIGS[name]
    code = synth.code_for(cfg)
    fr = synth.frames_for(cfg, code, range(first, first + nframes), point=point)
    return cfg, code, fr


def _channel(gfq, fr):
    return {synth.BSC: gfq.GFQ_BSC, synth.BEC: gfq.GFQ_BEC, synth.BIAWGN: gfq.GFQ_BIAWGN}[fr.channel]


def _gpu_decode(gfq, gcode, fr, schedule, max_iters, early_exit, T=None, keep=False):
    prm = gfq.Params(_channel(gfq, fr), fr.ch_param, schedule, max_iters, early_exit=early_exit,
                     markov_T=T, keep_messages=keep)
    obs = torch.as_tensor(fr.obs).cuda()
    s_hat, iters, ws = gfq.gfq_decode(gcode, obs, prm)
    torch.cuda.synchronize()
    return prm, s_hat.cpu().numpy(), iters.cpu().numpy(), ws


MSG_CASES = [("C1", 64, 0), ("C2", 80, 0), ("C3", 40, 0), ("C3", 40, 5), ("C4", 40, 0), ("C5", 64, 0)]


@pytest.mark.parametrize("schedule", [0, 1], ids=["PUS", "SUS"])
@pytest.mark.parametrize("name,nframes,point", MSG_CASES)
def test_message_gate_5_iterations(gfq, name, nframes, point, schedule):
    cfg, code, fr = _setup(name, nframes, point)
    T = synth.markov_T_for(cfg)
    gcode = gfq.Code.from_synth(code)
    prm, s_hat, iters, ws = _gpu_decode(gfq, gcode, fr, schedule, 5, False, T, keep=True)
    qg, rg, Qg = gfq.gfq_export_messages(gcode, fr.F, ws, prm)
    qg, rg, Qg = qg.cpu().numpy(), rg.cpu().numpy(), Qg.cpu().numpy()
    oc = oracle.OCode.from_synth(code)
    hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs)
    ref = oc.decode(hard, pi, schedule=schedule, max_iters=5, fixed=True, T=T, keep_messages=True)
    errs = {k: float(np.max(np.abs(g - ref[k]))) for k, g in (("q", qg), ("r", rg), ("Q", Qg))}
    print(name, point, "PUS" if schedule == 0 else "SUS", errs,
          "p99 q err %.3g" % np.percentile(np.abs(qg - ref["q"]), 99))
    assert max(errs.values()) <= MSG_TOL, errs
    assert np.array_equal(iters, ref["iters"])
    st = gfq.gfq_decode_stats(gcode, ws)
    assert st["zero_normalisers"] == 0


def _oracle_Q(oc, hard, pi, N, **kw):
    """Closure for gate.decision_gate: the oracle's final estimate and posterior
    (source symbols) of the given frames, re-decoded with the same arguments."""
    def f(idx):
        out = oc.decode(hard[idx], pi[idx], keep_messages=True, **kw)
        return out["xhat"][:, :N], out["Q"][:, :N]
    return f


def _decision_match(gpu_x, gpu_it, ref_x, ref_it, oracle_Q_for=None, case=None, replay=None):
    """Reading A18 plus the fp32 tie allowance (tests/gate.py)."""
    match, strict, n_allow = gate.decision_gate(gpu_x, gpu_it, ref_x, ref_it, oracle_Q_for, replay)
    if case:
        gate.record(case, len(match), match, strict, n_allow)
    return match, strict


DEC_CASES = [("C1", 64, 0), ("C2", 256, 0), ("C3", 128, 1), ("C3", 128, 4), ("C4", 64, 0), ("C5", 8, 0)]


@pytest.mark.parametrize("schedule", [0, 1], ids=["PUS", "SUS"])
@pytest.mark.parametrize("name,nframes,point", DEC_CASES)
def test_decision_gate(gfq, name, nframes, point, schedule):
    cfg, code, fr = _setup(name, nframes, point)
    T = synth.markov_T_for(cfg)
    gcode = gfq.Code.from_synth(code)
    _, s_hat, iters, ws = _gpu_decode(gfq, gcode, fr, schedule, cfg.max_iters, True, T)
    oc = oracle.OCode.from_synth(code)
    hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs)
    ref = oc.decode(hard, pi, schedule=schedule, max_iters=cfg.max_iters, T=T)
    match, strict = _decision_match(s_hat, iters, ref["xhat"][:, :code.N], ref["iters"],
                                    _oracle_Q(oc, hard, pi, code.N, schedule=schedule, max_iters=cfg.max_iters, T=T),
                                    "live %s p%d %s" % (name, point, "SUS" if schedule else "PUS"))
    allowed = gate.allowed(fr.F)
    print(name, point, "mismatch", int((~match).sum()), "strict", int((~strict).sum()),
          "mean iters gpu %.2f ref %.2f" % (iters[iters > 0].mean() if (iters > 0).any() else -1,
                                            ref["iters"][ref["iters"] > 0].mean() if (ref["iters"] > 0).any() else -1))
    assert int((~match).sum()) <= allowed
    assert gfq.gfq_decode_stats(gcode, ws)["zero_normalisers"] == 0


def test_evidence_entry_matches_oracle(gfq):
    """gfq_decode_evidence with the oracle's own front end (pi rounded to fp32, widened
    back exactly on the oracle side): bit-identical evidence on both sides."""
    cfg, code, fr = _setup("C3", 40, 2)
    gcode = gfq.Code.from_synth(code)
    hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs)
    pi32 = pi.astype(np.float32)
    for schedule in (0, 1):
        prm = gfq.Params(schedule=schedule, max_iters=5, early_exit=False, keep_messages=True)
        x, it, ws = gfq.gfq_decode_evidence(gcode, torch.as_tensor(hard).cuda(), torch.as_tensor(pi32).cuda(), prm)
        qg, rg, Qg = gfq.gfq_export_messages(gcode, fr.F, ws, prm)
        ref = oracle.OCode.from_synth(code).decode(hard, pi32.astype(np.float64), schedule=schedule,
                                                   max_iters=5, fixed=True, keep_messages=True)
        assert float(np.max(np.abs(qg.cpu().numpy() - ref["q"]))) <= MSG_TOL
        assert float(np.max(np.abs(Qg.cpu().numpy() - ref["Q"]))) <= MSG_TOL
        assert np.array_equal(it.cpu().numpy(), ref["iters"])


@pytest.mark.parametrize("name,full", [("C2", 1024), ("C4", 8192)])
def test_full_size_sampled(gfq, name, full):
    """BASELINE.json full batch on the GPU (the bench's launch configuration); the
    oracle recomputes a sample of frames one by one (frames are independent)."""
    cfg = synth.CONFIGS[name]
    code = synth.code_for(cfg)
    fr = synth.frames_for(cfg, code, range(full))
    T = synth.markov_T_for(cfg)
    gcode = gfq.Code.from_synth(code)
    sample = np.linspace(0, full - 1, 12).astype(int)
    oc = oracle.OCode.from_synth(code)
    hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs[sample])
    for schedule in (0, 1):
        _, s_hat, iters, _ = _gpu_decode(gfq, gcode, fr, schedule, cfg.max_iters, True, T)
        ref = oc.decode(hard, pi, schedule=schedule, max_iters=cfg.max_iters, T=T)
        match, _ = _decision_match(s_hat[sample], iters[sample], ref["xhat"][:, :code.N], ref["iters"],
                                   _oracle_Q(oc, hard, pi, code.N, schedule=schedule, max_iters=cfg.max_iters, T=T),
                                   "full-size sample %s %s" % (name, "SUS" if schedule else "PUS"),
                                   gate.oracle_replay(oc, hard, pi, code.N, cfg.max_iters, schedule=schedule, T=T))
        assert match.all()


def test_edge_cases(gfq):
    cfg, code, fr = _setup("C1", 33)           # ragged: 2 blocks, 1 valid lane in the last
    gcode = gfq.Code.from_synth(code)
    oc = oracle.OCode.from_synth(code)
    hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs)
    # max_iters = 0: iters -1 and clipped priors
    _, s0, it0, _ = _gpu_decode(gfq, gcode, fr, 0, 0, True)
    ref0 = oc.decode(hard, pi, max_iters=0)
    assert (it0 == -1).all() and np.array_equal(s0, ref0["xhat"][:, :code.N])
    # single frame
    fr1 = synth.frames_for(cfg, code, [7])
    _, s1, it1, _ = _gpu_decode(gfq, gcode, fr1, 1, 100, True)
    h1, p1 = oracle.frontend(fr1.channel, fr1.ch_param, fr1.obs)
    r1 = oc.decode(h1, p1, schedule=1, max_iters=100)
    assert it1[0] == r1["iters"][0] and np.array_equal(s1[0], r1["xhat"][0, :code.N])
    # zero frames is a no-op
    prm = gfq.Params(gfq.GFQ_BSC, fr.ch_param, 0, 10)
    empty = torch.empty((0, code.M), dtype=torch.uint8, device="cuda")
    s, it, _ = gfq.gfq_decode(gcode, empty, prm, workspace=gfq.alloc_workspace(1 << 20))
    assert s.shape[0] == 0
    # fixed mode reports the same first-passing t and estimate as early exit
    for sched in (0, 1):
        _, sa, ia, _ = _gpu_decode(gfq, gcode, fr, sched, 60, True)
        _, sb, ib, _ = _gpu_decode(gfq, gcode, fr, sched, 60, False)
        assert np.array_equal(ia, ib) and np.array_equal(sa, sb)


def test_waves_and_determinism(gfq):
    """A workspace for 1 block (3 waves) gives the same bits as one wave; reruns are identical."""
    cfg, code, fr = _setup("C2", 70)
    T = synth.markov_T_for(cfg)
    gcode = gfq.Code.from_synth(code)
    obs = torch.as_tensor(fr.obs).cuda()
    for sched in (0, 1):
        prm = gfq.Params(gfq.GFQ_BSC, fr.ch_param, sched, cfg.max_iters, markov_T=T)
        a = gfq.gfq_decode(gcode, obs, prm)
        b = gfq.gfq_decode(gcode, obs, prm)
        small = gfq.alloc_workspace(gfq.gfq_workspace_bytes(gcode, 32, prm))
        c = gfq.gfq_decode(gcode, obs, prm, workspace=small)
        torch.cuda.synchronize()
        for x, y in ((a, b), (a, c)):
            assert torch.equal(x[0], y[0]) and torch.equal(x[1], y[1])


def test_host_entry_matches_device(gfq):
    cfg, code, fr = _setup("C3", 64, 3)
    gcode = gfq.Code.from_synth(code)
    prm = gfq.Params(gfq.GFQ_BIAWGN, fr.ch_param, 0, cfg.max_iters)
    sd, itd, _ = gfq.gfq_decode(gcode, torch.as_tensor(fr.obs).cuda(), prm)
    sh, ith, _ = gfq.gfq_decode_host(gcode, torch.as_tensor(fr.obs).pin_memory(), prm)
    assert torch.equal(sd.cpu(), sh) and torch.equal(itd.cpu(), ith)


def test_host_entry_keeps_stats_and_export_at_offset_0(gfq):
    """gfq_decode_host stages obs / results at the END of the workspace, so the
    decode's health counters and messages stay where gfq_decode_stats and
    gfq_export_messages read them."""
    cfg, code, fr = _setup("C1", 40)
    gcode = gfq.Code.from_synth(code)
    prm = gfq.Params(gfq.GFQ_BSC, fr.ch_param, 1, 5, early_exit=False, keep_messages=True)
    ws = gfq.alloc_workspace(gfq.gfq_workspace_bytes_host(gcode, fr.F, prm))
    gfq.gfq_decode_host(gcode, torch.as_tensor(fr.obs).pin_memory(), prm, workspace=ws)
    st = gfq.gfq_decode_stats(gcode, ws)
    assert st["zero_normalisers"] == 0 and st["launches"] > 5 and st["block_iterations"] > 0
    qh, rh, Qh = gfq.gfq_export_messages(gcode, fr.F, ws, prm)
    _, _, _, wd = _gpu_decode(gfq, gcode, fr, 1, 5, False, keep=True)
    qd, rd, Qd = gfq.gfq_export_messages(gcode, fr.F, wd, prm)
    assert torch.equal(qh, qd) and torch.equal(rh, rd) and torch.equal(Qh, Qd)


def test_marshalling_rejects_bad_buffers(gfq):
    """The binding checks dtype, shape and device before calling the C ABI (which
    trusts pointers and sizes): ADVICE r1."""
    cfg, code, fr = _setup("C3", 4, 2)
    gcode = gfq.Code.from_synth(code)
    prm = gfq.Params(gfq.GFQ_BIAWGN, fr.ch_param, 0, 5)
    obs = torch.as_tensor(fr.obs).cuda()
    with pytest.raises(TypeError):
        gfq.gfq_decode(gcode, obs.to(torch.uint8), prm)               # AWGN needs float32
    with pytest.raises(ValueError):
        gfq.gfq_decode(gcode, obs[:, :-1].contiguous(), prm)         # row length != M*p
    with pytest.raises(ValueError):
        gfq.gfq_decode(gcode, obs.cpu(), prm)                         # host buffer to the device entry
    with pytest.raises(ValueError):
        gfq.gfq_decode(gcode, obs, prm, s_hat=torch.empty((4, code.N - 1), dtype=torch.uint8, device="cuda"))
    with pytest.raises(TypeError):
        gfq.gfq_decode(gcode, obs, prm, iters=torch.empty(4, dtype=torch.int64, device="cuda"))
    with pytest.raises(ValueError):
        gfq.gfq_decode_host(gcode, fr.obs, prm, s_hat_host=torch.empty((4, code.N), dtype=torch.uint8).cuda())


def test_natural_chain_labelling_many_levels(gfq):
    """B chain in natural order: the SUS dependency depth is ~M (serial); still exact."""
    cfg = synth.CONFIGS["C2"]
    code = synth.make_code(cfg.p, 300, 600, 77, permute_noise=False)
    fr = synth.make_frames(code, 9, range(40), "markov", synth.BSC, 0.05, stay=0.85)
    T = synth.markov_uniform_jump(code.q, 0.85)
    gcode = gfq.Code.from_synth(code)
    assert gcode.sus_levels > 500
    prm, s_hat, iters, ws = _gpu_decode(gfq, gcode, fr, 1, 5, False, T, keep=True)
    qg, rg, Qg = gfq.gfq_export_messages(gcode, fr.F, ws, prm)
    oc = oracle.OCode.from_synth(code)
    hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs)
    ref = oc.decode(hard, pi, schedule=1, max_iters=5, fixed=True, T=T, keep_messages=True)
    assert float(np.max(np.abs(qg.cpu().numpy() - ref["q"]))) <= MSG_TOL
    assert float(np.max(np.abs(Qg.cpu().numpy() - ref["Q"]))) <= MSG_TOL


def _random_code(p, N, M, colw, seed):
    """A generic (non-MN-chain) code with larger check and variable degrees:
    exercises the degree-8 kernel variants."""
    rng = np.random.default_rng(seed)
    q = 1 << p
    Ar, Ac = [], []
    for j in range(N):
        for i in rng.choice(M, colw, replace=False):
            Ar.append(i); Ac.append(j)
    Br, Bc = [], []
    for j in range(M):
        for i in rng.choice(M, 2, replace=False):
            Br.append(i); Bc.append(j)
    A = (np.array(Ar, np.int32), np.array(Ac, np.int32), rng.integers(1, q, len(Ar)).astype(np.uint8))
    B = (np.array(Br, np.int32), np.array(Bc, np.int32), rng.integers(1, q, len(Br)).astype(np.uint8))
    return A, B


@pytest.mark.parametrize("p", [2, 4, 6])
def test_high_degree_code_message_parity(gfq, p):
    """Check degree up to ~8 and variable degree 5: the DMAX = DVMAX = 8 kernels
    (or a clean GFQ_EUNSUPPORTED where shared memory cannot hold them)."""
    N, M = 40, 64
    for seed in range(100 + p, 200 + p):   # a draw with max check degree in 5..8
        A, B = _random_code(p, N, M, 4, seed)
        rows = np.concatenate([A[0], B[0]]); cols = np.concatenate([A[1], B[1] + N])
        vals = np.concatenate([A[2], B[2]])
        deg = np.bincount(rows, minlength=M)
        if 4 < deg.max() <= 8:
            break
    assert 4 < deg.max() <= 8
    gcode = gfq.Code(p, synth.PRIM_POLY[p], N, M, *A, *B)
    oc = oracle.OCode(p, synth.PRIM_POLY[p], N, M, rows, cols, vals)
    rng = np.random.default_rng(p)
    F = 40
    hard = rng.integers(0, 2, (F, M * p)).astype(np.uint8)
    pi = rng.uniform(0.02, 0.3, (F, M * p)).astype(np.float32)
    for schedule in (0, 1):
        prm = gfq.Params(schedule=schedule, max_iters=4, early_exit=False, keep_messages=True)
        try:
            x, it, ws = gfq.gfq_decode_evidence(gcode, torch.as_tensor(hard).cuda(), torch.as_tensor(pi).cuda(), prm)
        except gfq.GfqError as e:
            assert e.code == gfq.GFQ_EUNSUPPORTED and "shared memory" in str(e)
            continue
        qg, rg, Qg = gfq.gfq_export_messages(gcode, F, ws, prm)
        ref = oc.decode(hard, pi.astype(np.float64), schedule=schedule, max_iters=4, fixed=True, keep_messages=True)
        assert float(np.max(np.abs(qg.cpu().numpy() - ref["q"]))) <= MSG_TOL
        assert float(np.max(np.abs(rg.cpu().numpy() - ref["r"]))) <= MSG_TOL
        assert float(np.max(np.abs(Qg.cpu().numpy() - ref["Q"]))) <= MSG_TOL
        assert np.array_equal(it.cpu().numpy(), ref["iters"])


def test_markov_sus_pus_full_c2_sampled_decisions(gfq):
    """Markov source (Eq. 7 on the GPU vs Eq. 6 in the oracle) with early exit on a
    BSC at a noisier point than C2 (more iterations, more prior updates)."""
    cfg = synth.CONFIGS["C2"]
    code = synth.code_for(cfg)
    fr = synth.make_frames(code, cfg.cid, range(96), "markov", synth.BSC, 0.12, stay=cfg.stay, point=7)
    T = synth.markov_T_for(cfg)
    gcode = gfq.Code.from_synth(code)
    oc = oracle.OCode.from_synth(code)
    hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs)
    for schedule in (0, 1):
        _, s_hat, iters, ws = _gpu_decode(gfq, gcode, fr, schedule, cfg.max_iters, True, T)
        ref = oc.decode(hard, pi, schedule=schedule, max_iters=cfg.max_iters, T=T)
        match, _ = _decision_match(s_hat, iters, ref["xhat"][:, :code.N], ref["iters"],
                                   _oracle_Q(oc, hard, pi, code.N, schedule=schedule, max_iters=cfg.max_iters, T=T),
                                   "C2 bsc 0.12 %s" % ("SUS" if schedule else "PUS"))
        assert int((~match).sum()) == 0
        assert (iters > 3).mean() > 0.5   # the noisier point really iterates


TRACE_CASES = [("C1", 64, 0, False), ("C2", 96, 0, False), ("C3", 40, 4, True), ("C4", 40, 0, False)]


@pytest.mark.parametrize("schedule", [0, 1], ids=["PUS", "SUS"])
@pytest.mark.parametrize("name,nframes,point,fixed", TRACE_CASES)
def test_trace_fig1(gfq, name, nframes, point, fixed, schedule):
    """Fig. 1 instrumentation: the correct-source-bit count of the
    estimate after every iteration, taken on the device, equals the oracle's
    count (integers; the estimates themselves are argmaxes of fp32 vs fp64
    posteriors, so equality is required on >= 99.9 % of frames, reading A18)."""
    cfg, code, fr = _setup(name, nframes, point)
    T = synth.markov_T_for(cfg)
    gcode = gfq.Code.from_synth(code)
    tmax = 25 if fixed else cfg.max_iters
    truth = torch.as_tensor(fr.s).cuda()
    trace = torch.zeros((fr.F, tmax + 1), dtype=torch.int32, device="cuda")
    prm = gfq.Params(_channel(gfq, fr), fr.ch_param, schedule, tmax, early_exit=not fixed, markov_T=T,
                     trace_truth=truth, trace=trace)
    s_hat, iters, ws = gfq.gfq_decode(gcode, torch.as_tensor(fr.obs).cuda(), prm)
    torch.cuda.synchronize()
    oc = oracle.OCode.from_synth(code)
    hard, pi = oracle.frontend(fr.channel, fr.ch_param, fr.obs)
    ref = oc.decode(hard, pi, schedule=schedule, max_iters=tmax, fixed=fixed, T=T, s_true=fr.s)
    tg = trace.cpu().numpy()

    def q_at(f, t):
        o = oc.decode(hard[f:f + 1], pi[f:f + 1], schedule=schedule, max_iters=t, fixed=fixed, T=T,
                      keep_messages=True)
        return o["Q"][0, :code.N]
    same, n_allow = gate.trace_gate(tg, ref["trace"], iters.cpu().numpy(), ref["iters"], code.p, q_at)
    gate.GATE_LOG.append("trace %-28s frames %5d  mismatch %3d  tie-allowance %3d" % (
        "%s p%d %s %s" % (name, point, "SUS" if schedule else "PUS", "fixed" if fixed else "early-exit"),
        fr.F, int((~same).sum()), n_allow))
    assert (tg >= 0).all() and (tg <= code.N * code.p).all()
    assert int((~same).sum()) <= gate.allowed(fr.F)
    # the count of the final estimate is the count of the returned s_hat
    sh = s_hat.cpu().numpy()
    bits = lambda a: np.unpackbits(a[..., None], axis=-1, bitorder="little")[..., :code.p]
    final = (bits(sh) == bits(fr.s)).sum(axis=(1, 2))
    conv = iters.cpu().numpy() > 0
    if not fixed:
        assert np.array_equal(tg[:, -1], final)
    else:
        assert np.array_equal(tg[~conv, -1], final[~conv])


def test_trace_requires_both_buffers(gfq):
    cfg, code, fr = _setup("C1", 4)
    gcode = gfq.Code.from_synth(code)
    trace = torch.zeros((fr.F, 6), dtype=torch.int32, device="cuda")
    prm = gfq.Params(_channel(gfq, fr), fr.ch_param, 0, 5, trace=trace)
    with pytest.raises(gfq.GfqError):
        gfq.gfq_decode(gcode, torch.as_tensor(fr.obs).cuda(), prm)


def _low_degree_code(p, N, M, seed):
    """Check degrees 1..4 (including degree-1 and degree-2 checks) and variable
    degrees 1..3: the q >= 32 SUS path with phased layout switches takes every
    branch (d - 1 = 0, 1, 2, 3)."""
    rng = np.random.default_rng(seed)
    q = 1 << p
    V = N + M
    cap = rng.integers(1, 5, M)           # check degrees 1..4
    cap[:4] = [1, 2, 3, 4]
    vdeg = np.zeros(V, int)
    rows, cols = [], []
    for i in range(M):
        # variables of lowest degree first (every variable gets an edge), at most 3 each
        order = np.lexsort((rng.random(V), vdeg))
        pick = [j for j in order if vdeg[j] < 3][:cap[i]]
        for j in pick:
            rows.append(i); cols.append(int(j)); vdeg[j] += 1
    rows = np.array(rows, np.int32); cols = np.array(cols, np.int32)
    o = np.lexsort((cols, rows))
    rows, cols = rows[o], cols[o]
    vals = rng.integers(1, q, len(rows)).astype(np.uint8)
    a = cols < N
    A = (rows[a], cols[a], vals[a])
    B = (rows[~a], cols[~a] - N, vals[~a])
    return rows, cols, vals, A, B


@pytest.mark.parametrize("p,markov", [(3, False), (3, True), (4, False), (4, True), (5, False), (6, False), (6, True),
                                      (8, False)])
def test_low_degree_code_large_field_message_parity(gfq, p, markov):
    N, M = 30, 50
    for seed in range(300, 400):
        rows, cols, vals, A, B = _low_degree_code(p, N, M, seed)
        deg = np.bincount(rows, minlength=M)
        vdeg = np.bincount(cols, minlength=N + M)
        if deg.min() >= 1 and deg.max() <= 4 and vdeg.max() <= 3 and {1, 2, 3, 4} <= set(deg.tolist()):
            break
    assert {1, 2, 3, 4} <= set(deg.tolist()) and vdeg.max() <= 3
    gcode = gfq.Code(p, synth.PRIM_POLY[p], N, M, *A, *B)
    oc = oracle.OCode(p, synth.PRIM_POLY[p], N, M, rows, cols, vals)
    rng = np.random.default_rng(p + 7)
    F = 45                                 # two blocks, ragged
    hard = rng.integers(0, 2, (F, M * p)).astype(np.uint8)
    pi = rng.uniform(0.02, 0.3, (F, M * p)).astype(np.float32)
    T = synth.markov_uniform_jump(1 << p, 0.6) if markov else None
    for schedule in (0, 1):
        prm = gfq.Params(schedule=schedule, max_iters=4, early_exit=False, keep_messages=True, markov_T=T)
        x, it, ws = gfq.gfq_decode_evidence(gcode, torch.as_tensor(hard).cuda(), torch.as_tensor(pi).cuda(), prm)
        qg, rg, Qg = gfq.gfq_export_messages(gcode, F, ws, prm)
        ref = oc.decode(hard, pi.astype(np.float64), schedule=schedule, max_iters=4, fixed=True, keep_messages=True,
                        T=T)
        assert float(np.max(np.abs(qg.cpu().numpy() - ref["q"]))) <= MSG_TOL
        assert float(np.max(np.abs(rg.cpu().numpy() - ref["r"]))) <= MSG_TOL
        assert float(np.max(np.abs(Qg.cpu().numpy() - ref["Q"]))) <= MSG_TOL
        assert np.array_equal(it.cpu().numpy(), ref["iters"])


def test_c5_bench_configuration_sampled(gfq):
    """bench.py's workload and launch configuration: C5, 8192 frames from the
    device front end (gfq_simulate, the bench's seed), fixed 50 iterations, PUS
    in waves (workspace capped like bench.py) and SUS; four frames spread over
    the batch (first and last wave, ragged ends of the waves' frame ranges)
    recomputed one by one by the oracle from the same channel output."""
    cfg = synth.CONFIGS["C5"]
    code = synth.code_for(cfg)
    gcode = gfq.Code.from_synth(code)
    F, iters = cfg.frames, cfg.fixed_iters
    sigma = synth.awgn_sigma(cfg.ch_params[0])
    _, obs, _ = gfq.gfq_simulate(gcode, F, 0xBE7C0000 + cfg.cid * 64, gfq.GFQ_BIAWGN, sigma)
    params = {s: gfq.Params(gfq.GFQ_BIAWGN, sigma, s, iters, early_exit=False) for s in (0, 1)}
    torch.cuda.synchronize()
    free, _ = torch.cuda.mem_get_info()
    need = max(gfq.gfq_workspace_bytes(gcode, F, p) for p in params.values())
    ws = gfq.alloc_workspace(int(min(need, free - (3 << 30))))
    sample = np.array([0, 5119, 5120, F - 1])
    oc = oracle.OCode.from_synth(code)
    hard, pi = oracle.frontend(synth.BIAWGN, sigma, obs[torch.as_tensor(sample).cuda()].cpu().numpy())
    s_hat = torch.empty((F, code.N), dtype=torch.uint8, device="cuda")
    it = torch.empty(F, dtype=torch.int32, device="cuda")
    for sched, prm in params.items():
        gfq.gfq_decode(gcode, obs, prm, s_hat, it, ws)
        torch.cuda.synchronize()
        # the oracle may stop at the first passing iteration: in fixed-iteration mode the
        # reported estimate and t are those of the first pass, and an
        # i.i.d. source has no prior refresh that could differ afterwards
        ref = oc.decode(hard, pi, schedule=sched, max_iters=iters)
        got_x, got_it = s_hat.cpu().numpy()[sample], it.cpu().numpy()[sample]
        print("C5 bench config", "PUS" if sched == 0 else "SUS", got_it, ref["iters"])
        match, _ = _decision_match(got_x, got_it, ref["xhat"][:, :code.N], ref["iters"],
                                   _oracle_Q(oc, hard, pi, code.N, schedule=sched, max_iters=iters),
                                   "C5 bench config %s" % ("SUS" if sched else "PUS"))
        assert match.all()
        assert gfq.gfq_decode_stats(gcode, ws)["zero_normalisers"] == 0
    del ws
    torch.cuda.empty_cache()

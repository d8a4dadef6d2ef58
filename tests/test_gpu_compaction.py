"""Frame-granular early-exit compaction.

With gfq_params.compaction = GFQ_COMPACT_FRAMES (the default) the still-decoding
frames of the sparsest 32-frame blocks are moved into the idle lanes of the
other live blocks.  A frame's arithmetic depends neither on its lane nor on the
frames it shares a block with, so every output must be BIT-IDENTICAL to the
block-granular decode (GFQ_COMPACT_BLOCKS), which the decision gates compare
with the oracle -- estimates, iteration counts, the Fig. 1 trace -- while the
number of block iterations executed (gfq_decode_stats) must drop.
"""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gfq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    from paper_cs_0605069_b200 import gfq as g
    return g


def _chan(gfq, fr):
    return {synth.BSC: gfq.GFQ_BSC, synth.BEC: gfq.GFQ_BEC, synth.BIAWGN: gfq.GFQ_BIAWGN}[fr.channel]


def _decode(gfq, gcode, fr, cfg, schedule, compaction, T, ws_frames=None, prior_update=0, max_iters=None,
            trace_truth=None):
    F = fr.F
    mi = cfg.max_iters if max_iters is None else max_iters
    trace = None
    if trace_truth is not None:
        trace = torch.empty((F, mi + 1), dtype=torch.int32, device="cuda")
    prm = gfq.Params(_chan(gfq, fr), fr.ch_param, schedule, mi, early_exit=True, markov_T=T,
                     compaction=compaction, prior_update=prior_update, trace_truth=trace_truth, trace=trace)
    obs = torch.as_tensor(fr.obs).cuda()
    ws = gfq.alloc_workspace(gfq.gfq_workspace_bytes(gcode, ws_frames or F, prm))
    s_hat, iters, ws = gfq.gfq_decode(gcode, obs, prm, workspace=ws)
    torch.cuda.synchronize()
    st = gfq.gfq_decode_stats(gcode, ws)
    return (s_hat.cpu().numpy(), iters.cpu().numpy(), st,
            None if trace is None else trace.cpu().numpy())


CASES = [
    # name, frames, point, schedule, workspace frames (None = one wave), in-sweep prior
    ("C1", 64, 0, 0, None, 0), ("C1", 70, 0, 1, None, 0),
    ("C2", 300, 0, 0, None, 0), ("C2", 300, 0, 1, None, 0), ("C2", 300, 0, 1, None, 1),
    ("C2", 500, 0, 1, 192, 0),           # three waves, the last one ragged
    ("C3", 200, 1, 0, None, 0), ("C3", 200, 1, 1, None, 0),   # 1.0 dB: a third of the frames never stop
    ("C3", 256, 3, 1, None, 0),
    ("C4", 200, 0, 0, None, 0), ("C4", 200, 0, 1, None, 0),
    ("C5", 96, 0, 0, None, 0), ("C5", 96, 0, 1, None, 0),
]


@pytest.mark.parametrize("name,nframes,point,schedule,wsf,gs", CASES)
def test_frames_equals_blocks(gfq, name, nframes, point, schedule, wsf, gs):
    cfg = synth.CONFIGS[name]
    code = synth.code_for(cfg)
    fr = synth.frames_for(cfg, code, range(nframes), point=point)
    T = synth.markov_T_for(cfg)
    gcode = gfq.Code.from_synth(code)
    mi = min(cfg.max_iters, 120)
    xb, ib, sb, _ = _decode(gfq, gcode, fr, cfg, schedule, gfq.GFQ_COMPACT_BLOCKS, T, wsf, gs, mi)
    xf, itf, sf, _ = _decode(gfq, gcode, fr, cfg, schedule, gfq.GFQ_COMPACT_FRAMES, T, wsf, gs, mi)
    assert np.array_equal(ib, itf), "iterations differ at frames %s" % np.nonzero(ib != itf)[0][:8]
    assert np.array_equal(xb, xf), "estimates differ at frames %s" % np.nonzero((xb != xf).any(axis=1))[0][:8]
    assert sb["frames_converged"] == sf["frames_converged"] == int((ib > 0).sum())
    assert sf["zero_normalisers"] == 0
    ideal = float(np.where(ib > 0, ib, mi).sum()) / 32.0
    print("%s p%d %s: block iterations %d (blocks) -> %d (frames), ideal %.1f"
          % (name, point, "SUS" if schedule else "PUS", sb["block_iterations"], sf["block_iterations"], ideal))
    assert sf["block_iterations"] <= sb["block_iterations"]
    assert sf["block_iterations"] >= ideal - 1e-9
    if nframes >= 128 and (ib > 0).any() and ib[ib > 0].max() - ib[ib > 0].min() >= 3:
        assert sf["block_iterations"] < sb["block_iterations"], "no frame was ever moved"


def test_trace_follows_moved_frames(gfq):
    """The Fig. 1 trace is addressed by frame, not by lane slot."""
    cfg = synth.CONFIGS["C3"]
    code = synth.code_for(cfg)
    fr = synth.frames_for(cfg, code, range(160), point=2)
    gcode = gfq.Code.from_synth(code)
    truth = torch.as_tensor(np.ascontiguousarray(fr.s)).cuda()
    out = {}
    for comp in (gfq.GFQ_COMPACT_BLOCKS, gfq.GFQ_COMPACT_FRAMES):
        out[comp] = _decode(gfq, gcode, fr, cfg, 1, comp, None, None, 0, 60, truth)
    (xb, ib, sb, tb), (xf, itf, sf, tf) = out[gfq.GFQ_COMPACT_BLOCKS], out[gfq.GFQ_COMPACT_FRAMES]
    assert np.array_equal(ib, itf) and np.array_equal(xb, xf)
    assert np.array_equal(tb, tf)
    assert sf["block_iterations"] < sb["block_iterations"]


def test_bad_compaction_value_is_rejected(gfq):
    cfg = synth.CONFIGS["C1"]
    code = synth.code_for(cfg)
    fr = synth.frames_for(cfg, code, range(4))
    gcode = gfq.Code.from_synth(code)
    prm = gfq.Params(gfq.GFQ_BSC, fr.ch_param, 0, 5, compaction=7)
    with pytest.raises(gfq.GfqError):
        gfq.gfq_decode(gcode, torch.as_tensor(fr.obs).cuda(), prm)


def test_compaction_with_sus_orders_and_host_entry(gfq):
    """Caller-supplied SUS orders (A35) and the host-buffer entry with frame compaction."""
    cfg = synth.CONFIGS["C3"]
    code = synth.code_for(cfg)
    fr = synth.frames_for(cfg, code, range(150), point=3)
    gcode = gfq.Code.from_synth(code)
    rng = np.random.default_rng(35)
    orders = np.stack([rng.permutation(code.N + code.M) for _ in range(3)]).astype(np.int32)
    res = {}
    for comp in (gfq.GFQ_COMPACT_BLOCKS, gfq.GFQ_COMPACT_FRAMES):
        prm = gfq.Params(gfq.GFQ_BIAWGN, fr.ch_param, 1, 80, early_exit=True, sus_order=orders, compaction=comp)
        s_hat, it, ws = gfq.gfq_decode(gcode, torch.as_tensor(fr.obs).cuda(), prm)
        ph = gfq.Params(gfq.GFQ_BIAWGN, fr.ch_param, 0, 80, early_exit=True, compaction=comp)
        sh, ih, _ = gfq.gfq_decode_host(gcode, torch.as_tensor(fr.obs), ph)
        res[comp] = (s_hat.cpu().numpy(), it.cpu().numpy(), sh.numpy().copy(), ih.numpy().copy())
    for a, b in zip(res[gfq.GFQ_COMPACT_BLOCKS], res[gfq.GFQ_COMPACT_FRAMES]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("nframes", [1, 31, 33, 65])
def test_compaction_small_and_ragged_batches(gfq, nframes):
    cfg = synth.CONFIGS["C1"]
    code = synth.code_for(cfg)
    fr = synth.frames_for(cfg, code, range(nframes))
    gcode = gfq.Code.from_synth(code)
    outs = []
    for comp in (gfq.GFQ_COMPACT_BLOCKS, gfq.GFQ_COMPACT_FRAMES):
        for sched in (0, 1):
            prm = gfq.Params(gfq.GFQ_BSC, fr.ch_param, sched, 100, early_exit=True, compaction=comp)
            s_hat, it, ws = gfq.gfq_decode(gcode, torch.as_tensor(fr.obs).cuda(), prm)
            outs.append((comp, sched, s_hat.cpu().numpy(), it.cpu().numpy()))
    for sched in (0, 1):
        a = [o for o in outs if o[1] == sched]
        assert np.array_equal(a[0][2], a[1][2]) and np.array_equal(a[0][3], a[1][3])

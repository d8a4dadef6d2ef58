// gfq_decode.cu -- decode driver: workspace layout, waves over 32-frame
// blocks, the BP iteration loop (PUS or SUS), convergence bookkeeping,
// message export and health counters.  Host C++; every arithmetic step runs
// in the kernels of gfq_kernels.cu.
//
// One iteration:
//   PUS: k_cn (horizontal pass, Eq. 3) -> k_vn (vertical pass Eq. 4 +
//        posterior Eq. 5 + clipping; Markov prior Eq. 7 fused)
//   SUS: k_sus once per dependency level (steps 1-4 for every column)
//   then k_test (H x = z per frame) -> k_finalize -> k_capture
//   (copy x of newly converged frames) -> k_compact (early exit: drop
//   32-frame blocks whose frames all converged).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <utility>
#include <vector>

#include "gfq_internal.cuh"

namespace gfq {

static inline size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }
static constexpr size_t kNone = (size_t)-1;

Layout make_layout(const gfq_code *c, int fbw, const gfq_params *prm) {
  Layout L;
  L.fbw = fbw;
  size_t off = 0;
  const size_t F32 = (size_t)fbw * 32;
  const size_t Mp = (size_t)c->M * c->p;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += al256(bytes);
    return o;
  };
  // fixed header at offset 0 (gfq_decode_stats reads it without the params)
  L.stats = take(4 * sizeof(unsigned long long));
  L.nactive = take(sizeof(int));
  L.T = take((size_t)c->q * c->q * sizeof(double));
  L.Tf = take((size_t)2 * c->q * c->q * sizeof(float));
  L.pi0 = take((size_t)c->q * sizeof(double));
  const size_t msg = (size_t)c->E * c->q * F32 * sizeof(float);
  L.qmsg = take(msg);
  const bool need_r = prm->schedule == GFQ_PUS || prm->keep_messages;
  L.rmsg = need_r ? take(msg) : kNone;
  L.pi = take(Mp * F32 * sizeof(float));
  L.hard = take(Mp * F32);
  L.z = take((size_t)c->M * F32);
  L.xhat = take((size_t)c->V * F32);
  const bool markov = prm->markov_T != nullptr;
  const size_t qs = (size_t)c->N * c->q * F32 * sizeof(float);
  L.qs0 = markov ? take(qs) : kNone;
  L.qs1 = markov ? take(qs) : kNone;
  L.qall = prm->keep_messages ? take((size_t)c->V * c->q * F32 * sizeof(float)) : kNone;
  const bool ord = prm->schedule == GFQ_SUS && prm->sus_order && prm->sus_n_orders > 0;
  L.ord_col = ord ? take((size_t)prm->sus_n_orders * c->V * sizeof(LvlCol)) : kNone;
  L.ord_unit = ord ? take((size_t)prm->sus_n_orders * c->n_units * sizeof(LvlUnit)) : kNone;
  L.iters = take(F32 * sizeof(int));
  L.conv = take(F32 * sizeof(int));
  L.unsat = take(F32 * sizeof(int));
  L.newconv = take(F32 * sizeof(int));
  L.active = take((size_t)fbw * sizeof(int));
  L.list = take((size_t)fbw * sizeof(int));
  L.fid = take(F32 * sizeof(int));
  L.rp = take(repack_plan_bytes(fbw));
  L.total = off;
  return L;
}

static int check_params(const gfq_code *c, const gfq_params *prm, bool need_channel) {
  if (!c) { set_error("code is NULL"); return GFQ_EINVAL; }
  if (!prm) { set_error("params is NULL"); return GFQ_EINVAL; }
  if (prm->schedule != GFQ_PUS && prm->schedule != GFQ_SUS) { set_error("bad schedule"); return GFQ_EINVAL; }
  if (prm->max_iters < 0) { set_error("max_iters < 0"); return GFQ_EINVAL; }
  if (need_channel) {
    if (prm->channel < GFQ_BSC || prm->channel > GFQ_BIAWGN) { set_error("bad channel"); return GFQ_EINVAL; }
    if (prm->channel == GFQ_BSC && !(prm->ch_param >= 0.0 && prm->ch_param <= 1.0)) {
      set_error("BSC flip probability must be in [0, 1]");
      return GFQ_EINVAL;
    }
    if (prm->channel == GFQ_BIAWGN && !(prm->ch_param > 0.0)) { set_error("BI-AWGN sigma must be > 0"); return GFQ_EINVAL; }
  }
  const int q = c->q;
  if (prm->markov_T) {
    for (int a = 0; a < q; ++a) {
      double s = 0.0;
      for (int b = 0; b < q; ++b) {
        const double v = prm->markov_T[a * q + b];
        if (!(v >= 0.0) || !std::isfinite(v)) { set_error("markov_T has a negative or non-finite entry"); return GFQ_EINVAL; }
        s += v;
      }
      if (std::fabs(s - 1.0) > 1e-6) { set_error("markov_T row is not stochastic"); return GFQ_EINVAL; }
    }
  }
  if (prm->prior_update != GFQ_PRIOR_SNAPSHOT && prm->prior_update != GFQ_PRIOR_IN_SWEEP) {
    set_error("bad prior_update");
    return GFQ_EINVAL;
  }
  if (prm->prior_update == GFQ_PRIOR_IN_SWEEP && prm->schedule != GFQ_SUS) {
    set_error("prior_update = GFQ_PRIOR_IN_SWEEP needs schedule = GFQ_SUS (reading A34)");
    return GFQ_EINVAL;
  }
  if (prm->sus_order || prm->sus_n_orders) {
    if (!prm->sus_order || prm->sus_n_orders < 1) { set_error("sus_order needs sus_n_orders >= 1"); return GFQ_EINVAL; }
    if (prm->schedule != GFQ_SUS) { set_error("sus_order needs schedule = GFQ_SUS"); return GFQ_EINVAL; }
    if (prm->prior_update == GFQ_PRIOR_IN_SWEEP) {
      set_error("sus_order is not combined with GFQ_PRIOR_IN_SWEEP");
      return GFQ_EINVAL;
    }
    std::vector<char> seen(c->V);
    for (int o = 0; o < prm->sus_n_orders; ++o) {
      std::fill(seen.begin(), seen.end(), 0);
      const int *row = prm->sus_order + (size_t)o * c->V;
      for (int k = 0; k < c->V; ++k) {
        if (row[k] < 0 || row[k] >= c->V || seen[row[k]]) { set_error("sus_order row is not a permutation of 0..N+M-1"); return GFQ_EINVAL; }
        seen[row[k]] = 1;
      }
    }
  }
  if (prm->compaction != GFQ_COMPACT_FRAMES && prm->compaction != GFQ_COMPACT_BLOCKS) {
    set_error("bad compaction");
    return GFQ_EINVAL;
  }
  if ((prm->trace == nullptr) != (prm->trace_truth == nullptr)) {
    set_error("trace and trace_truth must both be set or both be NULL");
    return GFQ_EINVAL;
  }
  if (prm->src_pi0) {
    double s = 0.0;
    for (int a = 0; a < q; ++a) {
      if (!(prm->src_pi0[a] >= 0.0)) { set_error("src_pi0 has a negative entry"); return GFQ_EINVAL; }
      s += prm->src_pi0[a];
    }
    if (std::fabs(s - 1.0) > 1e-6) { set_error("src_pi0 does not sum to 1"); return GFQ_EINVAL; }
  }
  return GFQ_OK;
}

// Largest number of 32-frame blocks per wave that fits ws_bytes (<= want).
static int blocks_fitting(const gfq_code *c, const gfq_params *prm, size_t ws_bytes, int want) {
  if (want <= 0) return 0;
  if (make_layout(c, want, prm).total <= ws_bytes) return want;
  int lo = 0, hi = want;  // lo fits (0 trivially), hi does not
  while (hi - lo > 1) {
    const int mid = lo + (hi - lo) / 2;
    if (make_layout(c, mid, prm).total <= ws_bytes) lo = mid; else hi = mid;
  }
  return lo;
}

template <typename T>
static T *at(void *ws, size_t off) {
  return off == kNone ? nullptr : (T *)((char *)ws + off);
}

// ---------------------------------------------------------------- profiling
enum Kind { K_FRONTEND, K_SYNDROME, K_INIT_MSGS, K_INIT_STATE, K_CN, K_VN, K_SUS, K_TEST, K_FINALIZE,
            K_CAPTURE, K_COMPACT, K_CLIP, K_OTHER, K_TRACE, K_REPACK, K_N };
static const char *kKindNames[K_N] = {"frontend", "syndrome", "init_msgs", "init_state", "cn", "vn",
                                      "sus", "test", "finalize", "capture", "compact", "clip", "other",
                                      "trace", "repack"};
static_assert(K_N == GFQ_NKERNELS, "kernel kinds");

struct Profiler {
  bool on = false;
  struct Rec { int kind; cudaEvent_t a, b; };
  std::vector<Rec> pending;
  std::vector<cudaEvent_t> pool;
  double ms[K_N] = {0};
  long long n[K_N] = {0};
  cudaEvent_t get() {
    if (!pool.empty()) { cudaEvent_t e = pool.back(); pool.pop_back(); return e; }
    cudaEvent_t e = nullptr;
    if (cudaEventCreate(&e) != cudaSuccess) { cudaGetLastError(); return nullptr; }
    return e;
  }
  int drain() {
    for (auto &r : pending) {
      float t = 0.f;
      cudaError_t ce = cudaEventSynchronize(r.b);
      if (ce == cudaSuccess) ce = cudaEventElapsedTime(&t, r.a, r.b);
      if (ce != cudaSuccess) return cuda_fail(ce, "gfq_profile_read");
      ms[r.kind] += t;
      n[r.kind] += 1;
      pool.push_back(r.a);
      pool.push_back(r.b);
    }
    pending.clear();
    return GFQ_OK;
  }
};

static Profiler &profiler() {
  static thread_local Profiler p;
  return p;
}

struct LagRing {
  static constexpr int K = 8;
  cudaEvent_t ev[K];
  unsigned *host = nullptr;
  bool ok = false;
  LagRing() {
    if (cudaMallocHost((void **)&host, K * sizeof(unsigned)) != cudaSuccess) { cudaGetLastError(); return; }
    for (int k = 0; k < K; ++k)
      if (cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming) != cudaSuccess) { cudaGetLastError(); return; }
    ok = true;
  }
};

// One ring per (device, stream) of the calling thread: its events belong to
// that device, and a D2H readback still queued from an earlier decode on the
// same stream completes before this decode's own copies (stream order), so a
// slot is never read while another decode's copy into it is pending.
static LagRing &lag_ring(int dev, cudaStream_t st) {
  static thread_local std::map<std::pair<int, cudaStream_t>, std::unique_ptr<LagRing>> rings;
  std::unique_ptr<LagRing> &r = rings[std::make_pair(dev, st)];
  if (!r) r.reset(new LagRing());
  return *r;
}

// mode: 0 BSC, 1 BEC, 2 BI-AWGN (obs), 3 evidence (hard_in + pi_in)
static int decode_common(const gfq_code *c, int F, int mode, double ch_param, const void *obs,
                         const unsigned char *hard_in, const float *pi_in, const gfq_params *prm,
                         unsigned char *out, int Lout, int *iters_out, void *ws, size_t ws_bytes,
                         cudaStream_t st) {
  if (F < 0) { set_error("n_frames < 0"); return GFQ_EINVAL; }
  if (F == 0) return GFQ_OK;
  if (!ws || !out || !iters_out || (mode < 3 && !obs) || (mode == 3 && (!hard_in || !pi_in))) {
    set_error("NULL buffer");
    return GFQ_EINVAL;
  }
  int dev = -1;
  cudaError_t ce = cudaGetDevice(&dev);
  if (ce != cudaSuccess) return cuda_fail(ce, "cudaGetDevice");
  if (dev != c->device) {
    set_error("the current CUDA device is not the one the code was created on");
    return GFQ_EINVAL;
  }
  const int fbt = (F + 31) / 32;
  const int fbw = blocks_fitting(c, prm, ws_bytes, fbt);
  if (fbw < 1) { set_error("workspace too small for one 32-frame block"); return GFQ_EINVAL; }
  if (prm->keep_messages && fbw < fbt) { set_error("keep_messages needs a workspace for all frames"); return GFQ_EINVAL; }
  const Layout L = make_layout(c, fbw, prm);
  const int q = c->q;

  // Decoder constants: T and pi0 (doubles) into the workspace.
  std::vector<double> hbuf((size_t)q * q + q, 0.0);
  if (prm->markov_T) memcpy(hbuf.data(), prm->markov_T, sizeof(double) * q * q);
  for (int a = 0; a < q; ++a) hbuf[(size_t)q * q + a] = prm->src_pi0 ? prm->src_pi0[a] : 1.0 / q;
  ce = cudaMemcpyAsync(at<double>(ws, L.T), hbuf.data(), sizeof(double) * q * q, cudaMemcpyHostToDevice, st);
  if (ce == cudaSuccess)
    ce = cudaMemcpyAsync(at<double>(ws, L.pi0), hbuf.data() + (size_t)q * q, sizeof(double) * q, cudaMemcpyHostToDevice, st);
  std::vector<float> tf((size_t)2 * q * q, 0.0f);
  if (prm->markov_T)
    for (int x = 0; x < q; ++x)
      for (int y = 0; y < q; ++y) {
        tf[(size_t)x * q + y] = (float)prm->markov_T[x * q + y];              // T
        tf[(size_t)q * q + (size_t)y * q + x] = (float)prm->markov_T[x * q + y];  // T^T
      }
  if (ce == cudaSuccess)
    ce = cudaMemcpyAsync(at<float>(ws, L.Tf), tf.data(), sizeof(float) * 2 * q * q, cudaMemcpyHostToDevice, st);
  // (pageable H2D copies are staged before cudaMemcpyAsync returns, so hbuf may die here)
  if (ce == cudaSuccess) ce = cudaMemsetAsync(at<unsigned long long>(ws, L.stats), 0, 4 * sizeof(unsigned long long), st);
  if (ce != cudaSuccess) return cuda_fail(ce, "upload decoder constants");

  // level schedules of the caller's SUS column orders (A35), into the workspace
  std::vector<std::vector<int>> ord_lptr;
  const bool ordered = L.ord_col != kNone;
  if (ordered) {
    const int n = prm->sus_n_orders;
    std::vector<LvlCol> hcol((size_t)n * c->V);
    std::vector<LvlUnit> hunit((size_t)n * c->n_units);
    ord_lptr.resize(n);
    std::vector<LvlCol> lc;
    std::vector<LvlUnit> lu;
    for (int o = 0; o < n; ++o) {
      build_levels(c->hg, prm->sus_order + (size_t)o * c->V, false, ord_lptr[o], lc, lu);
      if ((long long)lu.size() != c->n_units) { set_error("internal: unit count"); return GFQ_EINVAL; }
      std::copy(lc.begin(), lc.end(), hcol.begin() + (size_t)o * c->V);
      std::copy(lu.begin(), lu.end(), hunit.begin() + (size_t)o * c->n_units);
    }
    ce = cudaMemcpyAsync(at<LvlCol>(ws, L.ord_col), hcol.data(), sizeof(LvlCol) * hcol.size(), cudaMemcpyHostToDevice, st);
    if (ce == cudaSuccess)
      ce = cudaMemcpyAsync(at<LvlUnit>(ws, L.ord_unit), hunit.data(), sizeof(LvlUnit) * hunit.size(), cudaMemcpyHostToDevice, st);
    // pageable H2D copies are staged before cudaMemcpyAsync returns, so the host
    // tables may die at scope exit (as hbuf above)
    if (ce != cudaSuccess) return cuda_fail(ce, "upload SUS order levels");
  }

  const bool tracing = prm->trace != nullptr;
  const int tlen = prm->max_iters + 1;
  if (tracing) {
    ce = cudaMemsetAsync(prm->trace, 0xff, sizeof(int) * (size_t)F * tlen, st);
    if (ce != cudaSuccess) return cuda_fail(ce, "clear trace");
  }

  LagRing &ring = lag_ring(dev, st);
  unsigned long long launches = 0;
  int rc = GFQ_OK;
  Profiler &prof = profiler();
#define RUN(kind, x)                                                         \
  do {                                                                       \
    cudaEvent_t e0_ = nullptr, e1_ = nullptr;                                \
    if (prof.on) { e0_ = prof.get(); e1_ = prof.get(); }                     \
    if (e0_ && e1_) cudaEventRecord(e0_, st);                                \
    rc = (x);                                                                \
    ++launches;                                                              \
    if (e0_ && e1_) {                                                        \
      cudaEventRecord(e1_, st);                                              \
      prof.pending.push_back({(kind), e0_, e1_});                            \
      if (prof.pending.size() > 4096 && prof.drain() != GFQ_OK) return GFQ_ECUDA; \
    }                                                                        \
    if (rc != GFQ_OK) return rc;                                             \
  } while (0)

  for (int fb0 = 0; fb0 < fbt; fb0 += fbw) {
    WaveArgs a;
    memset(&a, 0, sizeof(a));
    a.c = c->d;
    a.fb0 = fb0;
    a.nfb = std::min(fbw, fbt - fb0);
    a.n_frames = F;
    a.qmsg = at<float>(ws, L.qmsg);
    a.rmsg = at<float>(ws, L.rmsg);
    a.pi = at<float>(ws, L.pi);
    a.hard = at<unsigned char>(ws, L.hard);
    a.z = at<unsigned char>(ws, L.z);
    a.xhat = at<unsigned char>(ws, L.xhat);
    a.qall = at<float>(ws, L.qall);
    a.iters = at<int>(ws, L.iters);
    a.conv = at<int>(ws, L.conv);
    a.unsat = at<int>(ws, L.unsat);
    a.newconv = at<int>(ws, L.newconv);
    a.active = at<int>(ws, L.active);
    a.list = at<int>(ws, L.list);
    a.nactive = at<int>(ws, L.nactive);
    a.fid = at<int>(ws, L.fid);
    a.stats = at<unsigned long long>(ws, L.stats);
    a.T = prm->markov_T ? at<double>(ws, L.T) : nullptr;
    a.Tf = prm->markov_T ? at<float>(ws, L.Tf) : nullptr;
    a.pi0 = at<double>(ws, L.pi0);
    a.markov = prm->markov_T != nullptr;
    a.gs = a.markov && prm->schedule == GFQ_SUS && prm->prior_update == GFQ_PRIOR_IN_SWEEP;
    if (a.markov) {  // stay / uniform-jump structure (every diagonal entry equal, every other equal)
      const double d0 = prm->markov_T[0], o0 = q > 1 ? prm->markov_T[1] : 0.0;
      bool tj = true;
      for (int x = 0; x < q && tj; ++x)
        for (int y = 0; y < q; ++y)
          if (prm->markov_T[x * q + y] != (x == y ? d0 : o0)) { tj = false; break; }
      a.tj = tj;
      a.tj_alpha = (float)(d0 - o0);
      a.tj_beta = (float)o0;
    }
    if (a.gs) {  // the level schedule with the source chain (gfq_code.cu)
      a.c.lvl_col = c->lvl_col_gs;
      a.c.lvl_unit = c->lvl_unit_gs;
    }
    const std::vector<int> &lptr = a.gs ? c->level_ptr_gs_h : c->level_ptr_h;
    const int nlev = a.gs ? c->n_levels_gs : c->n_levels;
    a.early_exit = prm->early_exit ? 1 : 0;
    const bool repack = a.early_exit && !prm->keep_messages && prm->compaction == GFQ_COMPACT_FRAMES && a.nfb > 1;
    const RepackPlan rp = repack_plan_at(at<char>(ws, L.rp), fbw);
    a.t = 1;
    float *qs[2] = {at<float>(ws, L.qs0), at<float>(ws, L.qs1)};

    // estimates of lanes that never run (invalid lanes of a ragged block) read as 0
    ce = cudaMemsetAsync(a.xhat, 0, (size_t)a.nfb * c->V * 32, st);
    if (ce != cudaSuccess) return cuda_fail(ce, "clear x_hat");
    RUN(K_FRONTEND, launch_frontend(a, mode, ch_param, obs, hard_in, pi_in, st));
    RUN(K_SYNDROME, launch_syndrome(a, st));
    RUN(K_INIT_MSGS, launch_init_msgs(a, st));
    RUN(K_INIT_STATE, launch_init_state(a, st));
    if (prm->max_iters == 0 || tracing) {
      // x^(0): the clipped priors; no posterior snapshot is written
      WaveArgs a0 = a;
      a0.qs_new = nullptr;
      a0.gs = 0;
      RUN(K_CLIP, launch_clip_priors(a0, st));
      if (tracing) RUN(K_TRACE, launch_trace(a, prm->trace_truth, prm->trace, 0, tlen, st));
    }
    int t_done = 0;
    for (int t = 1; t <= prm->max_iters; ++t) {
      // Early exit: stop once a readback from two iterations ago saw no block left.
      if (a.early_exit && t > 3 && ring.ok) {
        const int k = (t - 3) % LagRing::K;
        ce = cudaEventSynchronize(ring.ev[k]);
        if (ce != cudaSuccess) return cuda_fail(ce, "cudaEventSynchronize");
        if (ring.host[k] == 0) break;
      }
      a.t = t;
      a.qs_old = qs[(t - 1) & 1];
      a.qs_new = qs[t & 1];
      if (prm->schedule == GFQ_PUS) {
        RUN(K_CN, launch_cn(a, st));
        RUN(K_VN, launch_vn(a, st));
      } else if (ordered) {  // sweep t in the caller's order (t-1) mod n (A35)
        const int o = (t - 1) % prm->sus_n_orders;
        WaveArgs ao = a;
        ao.c.lvl_col = at<LvlCol>(ws, L.ord_col) + (size_t)o * c->V;
        ao.c.lvl_unit = at<LvlUnit>(ws, L.ord_unit) + (size_t)o * c->n_units;
        const std::vector<int> &op = ord_lptr[o];
        for (int lv = 0; lv + 1 < (int)op.size(); ++lv) {
          const int lb = op[lv], n = op[lv + 1] - lb;
          if (n > 0) RUN(K_SUS, launch_sus_level(ao, lb, n, st));
        }
      } else {
        for (int lv = 0; lv < nlev; ++lv) {
          const int lb = lptr[lv], n = lptr[lv + 1] - lb;
          if (n > 0) RUN(K_SUS, launch_sus_level(a, lb, n, st));
        }
      }
      if (tracing) RUN(K_TRACE, launch_trace(a, prm->trace_truth, prm->trace, t, tlen, st));
      RUN(K_TEST, launch_test(a, st));
      RUN(K_FINALIZE, launch_finalize(a, 0, st));
      RUN(K_CAPTURE, launch_capture(a, out, Lout, 0, st));
      // frame-granular compaction: fill the idle lanes of the live blocks with
      // the frames of the sparsest ones (which k_compact then drops); the
      // snapshot the next iteration reads moves with them
      if (repack && t < prm->max_iters) RUN(K_REPACK, launch_repack(a, rp, a.qs_new, st));
      RUN(K_COMPACT, launch_compact(a, st));
      if (a.early_exit && ring.ok) {
        const int k = (t - 1) % LagRing::K;
        ce = cudaMemcpyAsync(ring.host + k, a.nactive, sizeof(unsigned), cudaMemcpyDeviceToHost, st);
        if (ce == cudaSuccess) ce = cudaEventRecord(ring.ev[k], st);
        if (ce != cudaSuccess) return cuda_fail(ce, "lag readback");
      }
      t_done = t;
    }
    (void)t_done;
    RUN(K_FINALIZE, launch_finalize(a, 1, st));
    RUN(K_CAPTURE, launch_capture(a, out, Lout, 0, st));
    const long long nvalid = std::min<long long>((long long)a.nfb * 32, (long long)F - (long long)fb0 * 32);
    ce = cudaMemcpyAsync(iters_out + (size_t)fb0 * 32, a.iters, sizeof(int) * nvalid, cudaMemcpyDeviceToDevice, st);
    if (ce != cudaSuccess) return cuda_fail(ce, "copy iters");
  }
  if (tracing) RUN(K_TRACE, launch_trace_fill(prm->trace, F, tlen, st));
  RUN(K_OTHER, launch_set_u64(at<unsigned long long>(ws, L.stats) + 3, launches + 1, st));
#undef RUN
  return GFQ_OK;
}

}  // namespace gfq

using namespace gfq;

extern "C" size_t gfq_workspace_bytes(const gfq_code *c, int n_frames, const gfq_params *prm) {
  if (!c || !prm || n_frames < 0) return 0;
  const int fb = std::max(1, (n_frames + 31) / 32);
  return make_layout(c, fb, prm).total;
}

static size_t obs_bytes(const gfq_code *c, int F, const gfq_params *prm) {
  const size_t Mp = (size_t)c->M * c->p;
  return (size_t)F * Mp * (prm->channel == GFQ_BIAWGN ? sizeof(float) : 1);
}

extern "C" size_t gfq_workspace_bytes_host(const gfq_code *c, int n_frames, const gfq_params *prm) {
  if (!c || !prm || n_frames < 0) return 0;
  return al256(obs_bytes(c, n_frames, prm)) + al256((size_t)n_frames * c->N) +
         al256((size_t)n_frames * sizeof(int)) + gfq_workspace_bytes(c, n_frames, prm);
}

extern "C" int gfq_decode(const gfq_code *c, int n_frames, const void *obs, const gfq_params *prm,
                          unsigned char *s_hat, int *iters, void *ws, size_t ws_bytes, void *stream) {
  int rc = check_params(c, prm, true);
  if (rc) return rc;
  return decode_common(c, n_frames, prm->channel, prm->ch_param, obs, nullptr, nullptr, prm, s_hat,
                       c->N, iters, ws, ws_bytes, (cudaStream_t)stream);
}

extern "C" int gfq_decode_evidence(const gfq_code *c, int n_frames, const unsigned char *hard_bits,
                                   const float *bit_flip_prob, const gfq_params *prm,
                                   unsigned char *x_hat, int *iters, void *ws, size_t ws_bytes,
                                   void *stream) {
  int rc = check_params(c, prm, false);
  if (rc) return rc;
  return decode_common(c, n_frames, 3, 0.0, nullptr, hard_bits, bit_flip_prob, prm, x_hat, c->V, iters,
                       ws, ws_bytes, (cudaStream_t)stream);
}

extern "C" int gfq_decode_host(const gfq_code *c, int n_frames, const void *obs_host,
                               const gfq_params *prm, unsigned char *s_hat_host, int *iters_host,
                               void *ws, size_t ws_bytes, void *stream) {
  int rc = check_params(c, prm, true);
  if (rc) return rc;
  if (n_frames < 0) { set_error("n_frames < 0"); return GFQ_EINVAL; }
  if (n_frames == 0) return GFQ_OK;
  if (!obs_host || !s_hat_host || !iters_host || !ws) { set_error("NULL buffer"); return GFQ_EINVAL; }
  if (prm->trace) { set_error("gfq_decode_host does not take trace buffers (device pointers)"); return GFQ_EINVAL; }
  const size_t ob = al256(obs_bytes(c, n_frames, prm));
  const size_t sb = al256((size_t)n_frames * c->N);
  const size_t ib = al256((size_t)n_frames * sizeof(int));
  if (ws_bytes < ob + sb + ib + gfq_workspace_bytes(c, 1, prm)) {
    set_error("workspace too small (size it with gfq_workspace_bytes_host)");
    return GFQ_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  // the decode workspace starts at offset 0 (gfq_decode_stats and
  // gfq_export_messages read it there); the staging copies sit at the end
  char *base = (char *)ws;
  const size_t dec_bytes = (ws_bytes - (ob + sb + ib)) & ~(size_t)255;
  char *stg = base + dec_bytes;
  void *obs_d = stg;
  unsigned char *s_d = (unsigned char *)(stg + ob);
  int *it_d = (int *)(stg + ob + sb);
  cudaError_t ce = cudaMemcpyAsync(obs_d, obs_host, obs_bytes(c, n_frames, prm), cudaMemcpyHostToDevice, st);
  if (ce != cudaSuccess) return cuda_fail(ce, "copy obs to device");
  rc = decode_common(c, n_frames, prm->channel, prm->ch_param, obs_d, nullptr, nullptr, prm, s_d, c->N,
                     it_d, base, dec_bytes, st);
  if (rc) return rc;
  ce = cudaMemcpyAsync(s_hat_host, s_d, (size_t)n_frames * c->N, cudaMemcpyDeviceToHost, st);
  if (ce == cudaSuccess) ce = cudaMemcpyAsync(iters_host, it_d, sizeof(int) * n_frames, cudaMemcpyDeviceToHost, st);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
  if (ce != cudaSuccess) return cuda_fail(ce, "copy results to host");
  return GFQ_OK;
}

extern "C" int gfq_export_messages(const gfq_code *c, int n_frames, const void *ws, size_t ws_bytes,
                                   const gfq_params *prm, float *q_msg, float *r_msg, float *Q,
                                   void *stream) {
  int rc = check_params(c, prm, false);
  if (rc) return rc;
  if (!ws || n_frames < 0) { set_error("bad workspace or n_frames"); return GFQ_EINVAL; }
  if (!prm->keep_messages) { set_error("export needs params.keep_messages = 1"); return GFQ_EINVAL; }
  const int fbt = (n_frames + 31) / 32;
  if (n_frames == 0) return GFQ_OK;
  const Layout L = make_layout(c, fbt, prm);
  if (L.total > ws_bytes) { set_error("workspace does not hold all frames"); return GFQ_EINVAL; }
  WaveArgs a;
  memset(&a, 0, sizeof(a));
  a.c = c->d;
  a.fb0 = 0;
  a.nfb = fbt;
  a.n_frames = n_frames;
  void *w = const_cast<void *>(ws);
  a.qmsg = at<float>(w, L.qmsg);
  a.rmsg = at<float>(w, L.rmsg);
  a.qall = at<float>(w, L.qall);
  return launch_export(a, q_msg, r_msg, Q, (cudaStream_t)stream);
}

extern "C" int gfq_decode_stats(const gfq_code *c, const void *ws, size_t ws_bytes, long long stats[4],
                                void *stream) {
  if (!c || !ws || !stats) { set_error("NULL argument"); return GFQ_EINVAL; }
  if (ws_bytes < 4 * sizeof(unsigned long long)) { set_error("workspace too small"); return GFQ_EINVAL; }
  unsigned long long h[4];
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t ce = cudaMemcpyAsync(h, ws, sizeof(h), cudaMemcpyDeviceToHost, st);  // stats live at offset 0
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
  if (ce != cudaSuccess) return cuda_fail(ce, "gfq_decode_stats");
  for (int k = 0; k < 4; ++k) stats[k] = (long long)h[k];
  return GFQ_OK;
}

extern "C" int gfq_profile_enable(int on) {
  Profiler &p = profiler();
  if (on) {
    int rc = p.drain();
    if (rc) return rc;
    for (int k = 0; k < K_N; ++k) { p.ms[k] = 0.0; p.n[k] = 0; }
  }
  p.on = on != 0;
  return GFQ_OK;
}

extern "C" int gfq_profile_read(double *ms, long long *launches) {
  Profiler &p = profiler();
  int rc = p.drain();
  if (rc) return rc;
  for (int k = 0; k < K_N; ++k) {
    if (ms) ms[k] = p.ms[k];
    if (launches) launches[k] = p.n[k];
  }
  return GFQ_OK;
}

extern "C" const char *gfq_kernel_name(int kind) {
  return (kind >= 0 && kind < K_N) ? kKindNames[kind] : nullptr;
}

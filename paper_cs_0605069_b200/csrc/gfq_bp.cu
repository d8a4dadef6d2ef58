// gfq_bp.cu -- the hot path of BP decoding of MN codes over GF(2^p) on
// sm_100a: the PUS check-node and variable-node kernels and the SUS level
// kernel.  PAPER.md §2 is the authority for what is computed;
// DESIGN.md explains how it is mapped onto the B200.
//
// Work decomposition: one frame per lane, 32 frames per block; a "group" of
// T = q/KR warps owns one task (a check, a variable, or a SUS column of one
// 32-frame block) and each thread holds KR entries of every q-vector:
//   layout A: thread (warp c, register k) holds entry y = c*KR + k
//   layout B: thread (warp c, register k) holds entry y = k*T  + c
// The Walsh-Hadamard transform over the bits of y done in registers in layout
// A covers bits 0..log2(KR)-1, in layout B the remaining high bits; switching
// layouts is a shared-memory transpose (fp64, conflict free: every warp access
// is 32 consecutive lanes of one row).
//
// Data movement: every task's input is one or a few contiguous chunks of
// q x 128-byte rows (messages are stored [block][edge][entry][32 lanes]; q
// messages in check-major edge order, r messages in variable-major edge
// order), fetched by the Tensor Memory Accelerator with cp.async.bulk into a
// ring of S shared-memory stages completed through mbarriers.  One lane per
// group is the producer: it keeps S tasks in flight and refills a stage when
// the group has finished with it, so HBM latency is hidden without register
// staging.  Entry permutations (multiplication by the GF(q) coefficient) are a
// choice of which shared-memory rows a thread reads or which global rows it
// writes.
//
// Precision: messages are stored in fp32 (the HBM bytes); every transform,
// leave-one-out product, prior and normalisation is computed in fp64 in
// registers, so tiny probabilities produced by cancellation in the inverse
// transform keep their relative accuracy.
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "gfq_internal.cuh"
#include "gfq_launch.cuh"

#include "gfq_device.cuh"

namespace gfq {

// ============================================================== layout switches (T > 1)
// Layout A -> B (or B -> A) of D messages through shared memory.  Bulk mode
// (PP = false): one buffer per message, one barrier for all of them; the
// caller separates successive uses with a barrier.  Ping-pong mode (PP = true,
// large q): two message buffers used alternately, one barrier per message and
// no other barrier needed -- the counter m (same in every warp of the group)
// carries the alternation across calls and tasks.
template <int Q, int KR>
__device__ __forceinline__ int idxA(int c, int k) { return c * KR + k; }
template <int Q, int KR>
__device__ __forceinline__ int idxB(int c, int k) { return k * (Q / KR) + c; }

template <int Q, int KR, int D, bool PP, bool A2B>
__device__ __forceinline__ void xpose(double (&u)[D][KR], double *buf, int &m, int g, int c, int lane) {
  constexpr int T = Q / KR;
  if constexpr (!PP) {
#pragma unroll
    for (int s = 0; s < D; ++s)
#pragma unroll
      for (int k = 0; k < KR; ++k)
        buf[((size_t)s * Q + (A2B ? idxA<Q, KR>(c, k) : idxB<Q, KR>(c, k))) * 32 + lane] = u[s][k];
    group_bar<T>(g);
#pragma unroll
    for (int s = 0; s < D; ++s)
#pragma unroll
      for (int k = 0; k < KR; ++k)
        u[s][k] = buf[((size_t)s * Q + (A2B ? idxB<Q, KR>(c, k) : idxA<Q, KR>(c, k))) * 32 + lane];
  } else {
#pragma unroll
    for (int s = 0; s < D; ++s) {
      double *b = buf + (size_t)(m & 1) * Q * 32;
      ++m;
      elided_bar<T>(g);  // ping-pong: the buffer is rewritten without a barrier
#pragma unroll
      for (int k = 0; k < KR; ++k) b[(A2B ? idxA<Q, KR>(c, k) : idxB<Q, KR>(c, k)) * 32 + lane] = u[s][k];
      group_bar<T>(g);
#pragma unroll
      for (int k = 0; k < KR; ++k) u[s][k] = b[(A2B ? idxB<Q, KR>(c, k) : idxA<Q, KR>(c, k)) * 32 + lane];
    }
  }
}

// Layout switch of D messages two at a time, alternating between buffer X0
// (the task's own, already-consumed input stage) and X1 (the group scratch):
// one barrier per pair.  t counts the pair transposes of the task (starts at
// 1 -> X1 in the forward direction, continues in the inverse one, so the
// stage is first overwritten after a barrier, and a task always ends on X0
// and starts on X1: no other barrier is needed across tasks).
template <int Q, int KR, int D, bool A2B>
__device__ __forceinline__ void xpose_pairs(double (&u)[D][KR], double *X0, double *X1, int &t, int g, int c,
                                            int lane) {
  constexpr int T = Q / KR;
#pragma unroll
  for (int p0 = 0; p0 < D; p0 += 2) {
    double *b = (t & 1) ? X1 : X0;
    ++t;
    elided_bar<T>(g);  // pairs alternate between two buffers without a barrier
#pragma unroll
    for (int s = p0; s < p0 + 2 && s < D; ++s)
#pragma unroll
      for (int k = 0; k < KR; ++k)
        b[((size_t)(s - p0) * Q + (A2B ? idxA<Q, KR>(c, k) : idxB<Q, KR>(c, k))) * 32 + lane] = u[s][k];
    group_bar<T>(g);
#pragma unroll
    for (int s = p0; s < p0 + 2 && s < D; ++s)
#pragma unroll
      for (int k = 0; k < KR; ++k)
        u[s][k] = b[((size_t)(s - p0) * Q + (A2B ? idxB<Q, KR>(c, k) : idxA<Q, KR>(c, k))) * 32 + lane];
  }
}

// ping-pong transposes for large fields (tuning knob)
#ifndef GFQ_PP_MINQ
#define GFQ_PP_MINQ 32
#endif
template <int Q>
struct PPof {
  static constexpr bool v = Q >= GFQ_PP_MINQ;
};
// check node: pair transposes through the consumed input stage (large fields)
#ifndef GFQ_CN_PAIRS
#define GFQ_CN_PAIRS 1
#endif

// ============================================================== PUS: check node
template <int Q, int KR, int DMAX, int S, int G>
struct CNShape {
  static constexpr int T = Q / KR;
  static constexpr bool PP = PPof<Q>::v;
  static constexpr size_t PAY = (size_t)DMAX * Q * 128;
  static constexpr size_t SCR = T > 1 ? (size_t)(PP ? 2 : DMAX) * Q * 32 * 8 : 0;
  using Sh = Shape<Q, S, G, PAY, SCR>;
  static constexpr size_t SMEM = Sh::SMEM;
  static constexpr int THREADS = (G * T + (PWof<T>::v ? 1 : 0)) * 32;
};

template <int Q, int DMAX>
__device__ __forceinline__ void cn_issue(const WaveArgs &a, int fb, int i, unsigned char *hdr, unsigned char *pay,
                                         uint64_t *full, int e0 = -1, int e1 = -1) {
  const int M = a.c.M;
  if (e0 < 0) {  // not prefetched (generic producer)
    e0 = __ldg(a.c.row_ptr + i);
    e1 = __ldg(a.c.row_ptr + i + 1);
  }
  const int d = e1 - e0;
  TaskInfo *ti = (TaskInfo *)hdr;
  ti->fb = fb; ti->item = i; ti->e0 = e0; ti->deg = d;
  const uint32_t msg = (uint32_t)d * Q * 128;
  mbar_expect_tx(full, 128 + 32 + (a.early_exit ? 128 : 0) + msg);
  bulk_g2s(hdr + 128, a.c.check_desc + i, 128, full);
  bulk_g2s(hdr + 256, a.z + ((size_t)fb * M + i) * 32, 32, full);
  if (a.early_exit) bulk_g2s(hdr + 384, a.conv + fb * 32, 128, full);
  if (msg) bulk_g2s(pay, a.qmsg + ((size_t)fb * a.c.E + e0) * Q * 32, msg, full);
}

// Eq. (3) for every edge of a check of exact degree D (horizontal
// pass), in the transform domain (BASELINE.json north_star): with
// u_k(y) = q_ij_k(h_k^-1 y) (the distribution of h_k x_k), U_k = WHT(u_k),
//   r_ij_k(a) ∝ WHT[ (-1)^{w.z_i} prod_{k' != k} U_k'(w) ](h_k a).
// The syndrome enters as the sign (-1)^{popc(w & z_i)} (XOR shift by z_i,
// reading A4).  The stored r is q * r (the 1/q of the inverse transform is
// dropped: the variable node normalises, the export divides); negative
// round-off is clamped to 0 (reading A20).
template <int Q, int KR, int D, int DMAX, typename RF>
__device__ __forceinline__ void cn_task(const WaveArgs &a, const unsigned char *hdr, uint32_t pay_u32,
                                        double *stage_x, uint64_t *empty, double *xp, int &m, int g, int c,
                                        int lane, RF &&refill) {
  using C = QC<Q, KR>;
  constexpr int T = C::T, LKR = C::LKR, LT = C::LT, P = C::P;
  constexpr bool PP = PPof<Q>::v;
  constexpr bool PAIRS = PP && GFQ_CN_PAIRS && (T > 1);
  const TaskInfo ti = *(const TaskInfo *)hdr;
  const CheckDesc *cd = (const CheckDesc *)(hdr + 128);
  const int fb = ti.fb;
  const int z = hdr[256 + lane];
  const bool frozen = a.early_exit && ((const int *)(hdr + 384))[lane] != 0;
  const long long E = a.c.E;
  double u[D][KR];
  unsigned long long pk[D];
  int canon[D];
#pragma unroll
  for (int s = 0; s < D; ++s) {
    pk[s] = cd->perm[s];
    canon[s] = cd->canon[s];
    uint32_t ad[KR];
    int rh;
    perm_addrs<P, LKR, KR>(pay_u32 + (uint32_t)(s * Q * 128 + lane * 4), pk[s], c, ad, rh);
#pragma unroll
    for (int k = 0; k < KR; ++k) u[s][k] = (double)lds_f32(ad[k]);
  }
  if constexpr (!PAIRS) {
    release_stage(empty, lane);
    refill();
  }
  // pair-transpose counter (PAIRS): start on X1 so that the stage (X0) is only
  // overwritten after the first barrier, when every warp has read its inputs
  int tp = 1;
#pragma unroll
  for (int s = 0; s < D; ++s) wht_bits<KR, 0, LKR>(u[s]);
  if constexpr (PAIRS) {
    xpose_pairs<Q, KR, D, true>(u, stage_x, xp, tp, g, c, lane);
#pragma unroll
    for (int s = 0; s < D; ++s) wht_bits<KR, LKR - LT, LKR>(u[s]);
  } else if constexpr (T > 1) {
    xpose<Q, KR, D, PP, true>(u, xp, m, g, c, lane);
#pragma unroll
    for (int s = 0; s < D; ++s) wht_bits<KR, LKR - LT, LKR>(u[s]);
  }
  uint32_t sm[KR];
  sign_masks<KR, T>(z, c, sm);
  loo_signed<D, KR, D>(u, sm);
  if constexpr (PAIRS) {
#pragma unroll
    for (int s = 0; s < D; ++s) wht_bits<KR, LKR - LT, LKR>(u[s]);
    xpose_pairs<Q, KR, D, false>(u, stage_x, xp, tp, g, c, lane);
    release_stage(empty, lane);  // the stage served as transpose buffer X0
    refill();
  } else if constexpr (T > 1) {
#pragma unroll
    for (int s = 0; s < D; ++s) wht_bits<KR, LKR - LT, LKR>(u[s]);
    if constexpr (!PP) group_bar<T>(g);  // bulk buffer: all forward reads done
    xpose<Q, KR, D, PP, false>(u, xp, m, g, c, lane);
    if constexpr (!PP) group_bar<T>(g);  // bulk buffer free for the next task
  }
#pragma unroll
  for (int s = 0; s < D; ++s) {
    wht_bits<KR, 0, LKR>(u[s]);
    if (!frozen) {
      // same rows as the load: r_k(a) lands at a = h^-1 y
      uint32_t ad[KR];
      int rh;
      perm_addrs<P, LKR, KR>(0u, pk[s], c, ad, rh);
      unsigned char *dst = (unsigned char *)(a.rmsg + ((size_t)fb * E + canon[s]) * Q * 32 + lane);
#pragma unroll
      for (int k = 0; k < KR; ++k) *(float *)(dst + ad[k]) = fmaxf((float)u[s][k], 0.0f);
    }
  }
}

template <int Q, int KR, int DMAX, int S, int G>
__global__ void __launch_bounds__(CNShape<Q, KR, DMAX, S, G>::THREADS) k_cn(WaveArgs a) {
  using CS = CNShape<Q, KR, DMAX, S, G>;
  using Sh = typename CS::Sh;
  constexpr int T = CS::T;
  extern __shared__ __align__(128) unsigned char smem[];
  const SmemPtrs sp = smem_ptrs<Sh, S, G>(smem);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) init_bars<S, G>(sp.bars, T);
  __syncthreads();
  const int M = a.c.M;
  const long long ntask = (long long)(*a.nactive) * M;
  constexpr bool PW = PWof<T>::v;
  if (PW && warp == 0) {
    if (lane == 0)
      produce<S, G>(a, sp.bars, ntask, M, [&](int g, int st, const Cursor &cu) {
        const int k = g * S + st;
        cn_issue<Q, DMAX>(a, cu.fb, cu.item, sp.hdr + (size_t)k * kHdr, sp.pay + (size_t)k * Sh::PAYA, sp.bars + k);
        return true;
      });
    return;
  }
  const int cw = PW ? warp - 1 : warp;
  const int g = cw / T, c = cw % T;
  const bool producer = !PW && (c == 0) && (lane == 0);  // one lane per group issues its TMA copies
  double *xp = (double *)(sp.scr + (size_t)g * CS::SCR);
  int m = 0;  // ping-pong transpose counter
  long long lo, hi;
  group_range(ntask, (long long)blockIdx.x * G + g, (long long)gridDim.x * G, lo, hi);
  Cursor pc;
  if (producer) {
    pc.init(a, lo, hi, M);
    pc.load_range(a.c.row_ptr);
    for (int n = 0; n < S && pc.valid(); ++n) {
      const int k = g * S + n;
      cn_issue<Q, DMAX>(a, pc.fb, pc.item, sp.hdr + (size_t)k * kHdr, sp.pay + (size_t)k * Sh::PAYA, sp.bars + k);
      pc.advance(a);
      pc.load_range(a.c.row_ptr);
    }
  }
  for (long long task = lo; task < hi; ++task) {
    const int rr = (int)(task - lo), st = rr % S, k = g * S + st;
    unsigned char *hdrw = sp.hdr + (size_t)k * kHdr;
    const unsigned char *hdr = hdrw;
    const uint32_t pay = sp.pay_u32 + (uint32_t)((size_t)k * Sh::PAYA);
    uint64_t *empty = sp.bars + G * S + k;
    // refill stage k with task + S once every warp of the group has released it
    auto refill = [&]() {
      if (producer && pc.valid()) {
        mbar_wait(empty, (uint32_t)((rr / S) & 1));
        cn_issue<Q, DMAX>(a, pc.fb, pc.item, hdrw, sp.pay + (size_t)k * Sh::PAYA, sp.bars + k);
        pc.advance(a);
        pc.load_range(a.c.row_ptr);
      }
    };
    mbar_wait(sp.bars + k, (uint32_t)((rr / S) & 1));
    const int d = ((const TaskInfo *)hdr)->deg;
    switch (d) {
      case 1: cn_task<Q, KR, 1, DMAX>(a, hdr, pay, (double *)(sp.pay + (size_t)k * Sh::PAYA), empty, xp, m, g, c, lane, refill); break;
      case 2: cn_task<Q, KR, 2, DMAX>(a, hdr, pay, (double *)(sp.pay + (size_t)k * Sh::PAYA), empty, xp, m, g, c, lane, refill); break;
      case 3: cn_task<Q, KR, 3, DMAX>(a, hdr, pay, (double *)(sp.pay + (size_t)k * Sh::PAYA), empty, xp, m, g, c, lane, refill); break;
      case 4: cn_task<Q, KR, 4, DMAX>(a, hdr, pay, (double *)(sp.pay + (size_t)k * Sh::PAYA), empty, xp, m, g, c, lane, refill); break;
      default:
        if constexpr (DMAX > 4) {
          switch (d) {
            case 5: cn_task<Q, KR, 5, DMAX>(a, hdr, pay, (double *)(sp.pay + (size_t)k * Sh::PAYA), empty, xp, m, g, c, lane, refill); break;
            case 6: cn_task<Q, KR, 6, DMAX>(a, hdr, pay, (double *)(sp.pay + (size_t)k * Sh::PAYA), empty, xp, m, g, c, lane, refill); break;
            case 7: cn_task<Q, KR, 7, DMAX>(a, hdr, pay, (double *)(sp.pay + (size_t)k * Sh::PAYA), empty, xp, m, g, c, lane, refill); break;
            default: cn_task<Q, KR, 8, DMAX>(a, hdr, pay, (double *)(sp.pay + (size_t)k * Sh::PAYA), empty, xp, m, g, c, lane, refill); break;
          }
        } else {
          release_stage(empty, lane);  // d == 0: an empty check has no edge
          refill();
        }
        break;
    }
    elided_bar<T>(g);  // tasks follow each other without a barrier
  }
}

// ============================================================== PUS: variable node
template <int Q, int KR, int DVMAX, bool MARKOV, int S, int G>
struct VNShape {
  static constexpr int T = Q / KR;
  static constexpr int XR = Extra<Q, MARKOV>::rows;
  static constexpr size_t PAY = (size_t)DVMAX * Q * 128;
  static constexpr bool ONEBAR = T > 1 && T <= 4;  // one-barrier reduction, red double-buffered
  static constexpr size_t RED_B = ((size_t)(DVMAX + 2) * T * 32 + (size_t)(DVMAX + 2) * 32 + T * 32) * 8;
  static constexpr size_t SCR = RED_B * (ONEBAR ? 2 : 1);
  // Markov T and T^T (fp32) in shared memory up to q = 64; at q = 128 (128 KB)
  // they are read through L1 from the workspace copy
  static constexpr bool TSMEM = MARKOV && Q <= 64;
  using Sh = Shape<Q, S, G, PAY, SCR, (size_t)XR * 128, TSMEM ? (size_t)2 * Q * Q * 4 : 0, false>;
  static constexpr size_t SMEM = Sh::SMEM;
  static constexpr int THREADS = (G * T + (PWof<T>::v ? 1 : 0)) * 32;
};

template <int Q, int DVMAX, bool MARKOV>
__device__ __forceinline__ void vn_issue(const WaveArgs &a, int fb, int j, unsigned char *hdr, unsigned char *pay,
                                         unsigned char *xtra, uint64_t *full, int clip_only, int e0 = -1,
                                         int e1 = -1) {
  if (e0 < 0) {  // not prefetched (generic producer)
    e0 = __ldg(a.c.col_ptr + j);
    e1 = __ldg(a.c.col_ptr + j + 1);
  }
  const int dv = clip_only ? 0 : e1 - e0;
  TaskInfo *ti = (TaskInfo *)hdr;
  ti->fb = fb; ti->item = j; ti->e0 = e0; ti->deg = dv;
  const uint32_t br = (uint32_t)dv * Q * 128;
  mbar_expect_tx(full, 64 + (a.early_exit ? 128 : 0) + br + extras_bytes<Q, MARKOV>(a, j));
  bulk_g2s(hdr + 192, a.c.var_desc + j, 64, full);
  if (a.early_exit) bulk_g2s(hdr + 384, a.conv + fb * 32, 128, full);
  if (br) bulk_g2s(pay, a.rmsg + ((size_t)fb * a.c.E + e0) * Q * 32, br, full);  // canonical order
  issue_extras<Q, MARKOV>(a, fb, j, xtra, full);
}

template <int Q, int KR, int DV, int DVMAX, bool MARKOV, typename RF>
__device__ __forceinline__ void vn_task(const WaveArgs &a, const unsigned char *hdr, const unsigned char *pay,
                                        const unsigned char *xtra, const float *Tsm, uint64_t *empty, double *red,
                                        int g, int c, int lane, RF &&refill) {
  const TaskInfo ti = *(const TaskInfo *)hdr;
  const VarDesc *vd = (const VarDesc *)(hdr + 192);
  const bool frozen = a.early_exit && ((const int *)(hdr + 384))[lane] != 0;
  const float *in = (const float *)pay + lane + c * KR * 32;
  int qdst[DV > 0 ? DV : 1];
  double r[DV > 0 ? DV : 1][KR];
#pragma unroll
  for (int s = 0; s < DV; ++s) {
    qdst[s] = vd->qdst[s];
#pragma unroll
    for (int k = 0; k < KR; ++k) r[s][k] = (double)in[(s * Q + k) * 32];
  }
  double pr[KR];
  prior_from<Q, KR, MARKOV>(a, ti.item, c, lane, (const float *)xtra, Tsm, pr);
  release_stage(empty, lane);
  refill();
  vn_core<Q, KR, DV, MARKOV, (Q / KR > 1 && Q / KR <= 4)>(a, ti.fb, ti.item, qdst, r, pr, red, g, c, lane, frozen);
}

template <int Q, int KR, int DVMAX, bool MARKOV, int S, int G>
__global__ void __launch_bounds__(VNShape<Q, KR, DVMAX, MARKOV, S, G>::THREADS)
    k_vn(WaveArgs a, int clip_only) {
  using VS = VNShape<Q, KR, DVMAX, MARKOV, S, G>;
  using Sh = typename VS::Sh;
  constexpr int T = VS::T;
  extern __shared__ __align__(128) unsigned char smem[];
  const SmemPtrs sp = smem_ptrs<Sh, S, G>(smem);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) init_bars<S, G>(sp.bars, T);
  if constexpr (VS::TSMEM) {
    if (a.Tf)
      for (int k = threadIdx.x; k < 2 * Q * Q; k += blockDim.x) sp.tsm[k] = a.Tf[k];
  }
  const float *Tp = VS::TSMEM ? sp.tsm : a.Tf;
  __syncthreads();
  const int V = a.c.V;
  const long long ntask = (long long)(*a.nactive) * V;
  constexpr bool PW = PWof<T>::v;
  if (PW && warp == 0) {
    if (lane == 0)
      produce<S, G>(a, sp.bars, ntask, V, [&](int g, int st, const Cursor &cu) {
        const int k = g * S + st;
        vn_issue<Q, DVMAX, MARKOV>(a, cu.fb, cu.item, sp.hdr + (size_t)k * kHdr, sp.pay + (size_t)k * Sh::PAYA,
                                   sp.xtra + (size_t)k * Sh::XTRA_A, sp.bars + k, clip_only);
        return true;
      }, -1, !clip_only);
    return;
  }
  const int cw = PW ? warp - 1 : warp;
  const int g = cw / T, c = cw % T;
  const bool producer = !PW && (c == 0) && (lane == 0);
  double *red = (double *)(sp.scr + (size_t)g * VS::SCR);
  long long lo, hi;
  if (clip_only) group_range(ntask, (long long)blockIdx.x * G + g, (long long)gridDim.x * G, lo, hi);
  else vn_group_range(a, (long long)(*a.nactive), (long long)blockIdx.x * G + g, (long long)gridDim.x * G, lo, hi);
  Cursor pc;
  if (producer) {
    pc.init(a, lo, hi, V);
    pc.load_range(a.c.col_ptr);
    for (int n = 0; n < S && pc.valid(); ++n) {
      const int k = g * S + n;
      vn_issue<Q, DVMAX, MARKOV>(a, pc.fb, pc.item, sp.hdr + (size_t)k * kHdr, sp.pay + (size_t)k * Sh::PAYA,
                                 sp.xtra + (size_t)k * Sh::XTRA_A, sp.bars + k, clip_only);
      pc.advance(a);
      pc.load_range(a.c.col_ptr);
    }
  }
  for (long long task = lo; task < hi; ++task) {
    const int rr = (int)(task - lo), st = rr % S, k = g * S + st;
    unsigned char *hdrw = sp.hdr + (size_t)k * kHdr;
    const unsigned char *hdr = hdrw;
    const unsigned char *pay = sp.pay + (size_t)k * Sh::PAYA;
    const unsigned char *xtra = sp.xtra + (size_t)k * Sh::XTRA_A;
    uint64_t *empty = sp.bars + G * S + k;
    auto refill = [&]() {
      if (producer && pc.valid()) {
        mbar_wait(empty, (uint32_t)((rr / S) & 1));
        vn_issue<Q, DVMAX, MARKOV>(a, pc.fb, pc.item, hdrw, sp.pay + (size_t)k * Sh::PAYA,
                                   sp.xtra + (size_t)k * Sh::XTRA_A, sp.bars + k, clip_only);
        pc.advance(a);
        pc.load_range(a.c.col_ptr);
      }
    };
    mbar_wait(sp.bars + k, (uint32_t)((rr / S) & 1));
    const int dv = ((const TaskInfo *)hdr)->deg;
    double *redt = VS::ONEBAR ? red + (size_t)(rr & 1) * (VS::RED_B / 8) : red;
#define VT(n) vn_task<Q, KR, n, DVMAX, MARKOV>(a, hdr, pay, xtra, Tp, empty, redt, g, c, lane, refill)
    switch (dv) {
      case 0: VT(0); break;
      case 1: VT(1); break;
      case 2: VT(2); break;
      default:
        if constexpr (DVMAX <= 3) {
          VT(3);
        } else {
          switch (dv) {
            case 3: VT(3); break;
            case 4: VT(4); break;
            case 5: VT(5); break;
            case 6: VT(6); break;
            case 7: VT(7); break;
            default: VT(8); break;
          }
        }
        break;
    }
#undef VT
    // no barrier here: vn_core's own barriers order every reuse of red
    elided_bar<T>(g);
  }
}

// ============================================================== SUS: one dependency level
template <int Q, int KR, int DMAX, int DVMAX, bool MARKOV, int S, int G>
struct SUSShape {
  static constexpr int T = Q / KR;
  static constexpr bool PP = PPof<Q>::v;
  static constexpr int XR = Extra<Q, MARKOV>::rows;
  static constexpr size_t PAY = (size_t)(DMAX - 1) * Q * 128;
  // transpose buffers (bulk: DMAX-1 forward + 1 accumulator; ping-pong: 2);
  // the variable-node reduction scratch aliases them (used after the last transpose)
  static constexpr bool PHASED = T > 1 && DMAX <= 4;  // sus_check_phased
  static constexpr size_t XP_D = T > 1 ? (size_t)((PP || PHASED) ? 2 : DMAX) * Q * 32 : 0;
  static constexpr size_t RED_D = (size_t)(DVMAX + 2) * T * 32 + (size_t)(DVMAX + 2) * 32 + T * 32;
  static constexpr size_t XR_D = XP_D > RED_D ? XP_D : RED_D;
  static constexpr size_t RSM_F = (size_t)DVMAX * Q * 32;
  static constexpr size_t SCR = XR_D * 8 + RSM_F * 4;
  // phased layout switches (sus_check_phased): the variable-node reduction
  // scratch then lives in the stage payload of the column's last unit
  static_assert(!PHASED || RED_D * 8 <= PAY, "reduction scratch must fit a stage payload");
  // shared region: Markov T and T^T (fp32), then the row-offset table (u16 q x q)
  // when it still fits (RTS; otherwise the table is read through L1)
  static constexpr bool TSMEM = MARKOV && Q <= 64;  // as VNShape
  static constexpr size_t TSM_F = TSMEM ? (size_t)2 * Q * Q : 0;
  using Sh0 = Shape<Q, S, G, PAY, SCR, (size_t)XR * 128, TSM_F * 4, false>;
  static constexpr bool RTS = Sh0::SMEM + (size_t)2 * Q * Q <= 232448;
  using Sh = Shape<Q, S, G, PAY, SCR, (size_t)XR * 128, TSM_F * 4 + (RTS ? (size_t)2 * Q * Q : 0), false>;
  static constexpr size_t SMEM = Sh::SMEM;
  static constexpr int THREADS = (G * T + (PWof<T>::v ? 1 : 0)) * 32;
};

// Step 1 of SUS for one check (exact number of other edges DO): r_ij from the
// CURRENT q's of the check's other edges (the transform of k_cn restricted to
// one output).  Writes q * r_ij into rsm slot s in natural order a.
template <int Q, int KR, int DO, int DMAX, typename RF>
__device__ __forceinline__ void sus_check(const WaveArgs &a, const TaskInfo &ti, const unsigned char *hdr, uint32_t pay_u32,
                                          uint64_t *empty, bool release, double *xp, int &m, float *rsm, int g,
                                          int c, int lane, bool frozen, RF &&refill) {
  using C = QC<Q, KR>;
  constexpr int T = C::T, LKR = C::LKR, LT = C::LT, P = C::P;
  constexpr bool PP = PPof<Q>::v;
  const SusDesc *sd = (const SusDesc *)(hdr + 128);
  const int z = hdr[256 + lane];
  double v[DO > 0 ? DO : 1][KR];
#pragma unroll
  for (int t = 0; t < DO; ++t) {
    uint32_t ad[KR];
    tab_addrs<Q, KR>(pay_u32 + (uint32_t)(t * Q * 128 + lane * 4), a.c.rowtab, sd->perm_o[t], c, ad);
#pragma unroll
    for (int k = 0; k < KR; ++k) v[t][k] = (double)lds_f32(ad[k]);
  }
  const unsigned long long pke = sd->perm_e;
  if (release) {
    release_stage(empty, lane);
    refill();
  }
#pragma unroll
  for (int t = 0; t < DO; ++t) wht_bits<KR, 0, LKR>(v[t]);
  if constexpr (T > 1) {
    if constexpr (DO > 0) {
      xpose<Q, KR, DO, PP, true>(v, xp, m, g, c, lane);
#pragma unroll
      for (int t = 0; t < DO; ++t) wht_bits<KR, LKR - LT, LKR>(v[t]);
    }
  }
  uint32_t sm[KR];
  sign_masks<KR, T>(z, c, sm);
  double acc[1][KR];
#pragma unroll
  for (int k = 0; k < KR; ++k) {
    double x = 1.0;
#pragma unroll
    for (int t = 0; t < DO; ++t) x = (t == 0) ? v[0][k] : x * v[t][k];
    acc[0][k] = flip(x, sm[k]);
  }
  if constexpr (T > 1) {
    wht_bits<KR, LKR - LT, LKR>(acc[0]);
    // bulk mode: the accumulator uses its own slot (index DMAX-1) of the buffer
    xpose<Q, KR, 1, PP, false>(acc, PP ? xp : xp + (size_t)(DMAX - 1) * Q * 32, m, g, c, lane);
  }
  wht_bits<KR, 0, LKR>(acc[0]);
  uint32_t ad[KR];
  tab_addrs<Q, KR>(0u, a.c.rowtab, pke, c, ad);  // ad[k] = (h_e^-1 y) * 128: a = h_e^-1 y
  const int s = ti.s;
  unsigned char *rs = (unsigned char *)(rsm + (size_t)s * Q * 32 + lane);
#pragma unroll
  for (int k = 0; k < KR; ++k) *(float *)(rs + ad[k]) = fmaxf((float)acc[0][k], 0.0f);
  if (a.rmsg != nullptr) {  // keep_messages only (export): warp-uniform branch
    if (!frozen) {
      unsigned char *rdst = (unsigned char *)(a.rmsg + ((size_t)ti.fb * a.c.E + ti.e0 + s) * Q * 32 + lane);
#pragma unroll
      for (int k = 0; k < KR; ++k) *(float *)(rdst + ad[k]) = fmaxf((float)acc[0][k], 0.0f);
    }
  }
}

// Phased variant of sus_check for q >= 16 (T > 1), check degree <= 4:
// the d-1 <= 3 forward layout switches take one barrier for the first two
// messages (group scratch xp, slots 0 and 1) and one more for a third (the
// task's own stage payload, free once every warp has passed the first
// barrier, i.e. has read its inputs); the inverse switch writes the
// accumulator over the buffer this warp read last, at the positions it read
// (layout B): no other warp touches those positions between the barriers, so
// no extra barrier is needed, and the positions read afterwards (layout A)
// are exactly the ones this warp writes first in the next task.  Barriers
// per unit: 2 (d = 3) or 3 (d = 4) instead of d (ping-pong) or 3 (bulk).
// Row offsets from the shared (RTS) or global copy of the per-field table.
template <int Q, int KR, bool RTS>
__device__ __forceinline__ void row_addrs(uint32_t base, uint32_t rt, const unsigned short *rowtab,
                                          unsigned long long pk, int c, uint32_t (&ad)[KR]) {
  if constexpr (RTS) tab_addrs_sm<Q, KR>(base, rt, pk, c, ad);
  else tab_addrs<Q, KR>(base, rowtab, pk, c, ad);
}
// The same with the rows shifted by the syndrome: entry y reads row h^-1 (y ^ z)
// = h^-1 y ^ h^-1 z (multiplication by h^-1 is GF(2)-linear); z differs per
// lane, the XOR acts on the row bits only, and a lane still reads its own
// 4-byte column of a 128-byte row: no bank conflict.  Shifting ONE operand of
// the convolution shifts the result, S'(y) = S(y ^ z), so r(a) = S(z ^ h a) =
// S'(h a) needs no sign (-1)^{w.z} in the transform domain (reading A4).
template <int Q, int KR, bool RTS>
__device__ __forceinline__ void row_addrs_shift(uint32_t base, uint32_t rt, const unsigned short *rowtab,
                                                unsigned long long pk, int c, int z, uint32_t (&ad)[KR]) {
  uint32_t off[KR];
  row_addrs<Q, KR, RTS>(0u, rt, rowtab, pk, c, off);
  uint32_t hz;
  if constexpr (RTS) asm volatile("ld.shared.u16 %0, [%1];" : "=r"(hz) : "r"(rt + (uint32_t)(((pk & 0xff) * Q + z) * 2)));
  else hz = rowtab[(size_t)(pk & 0xff) * Q + z];
#pragma unroll
  for (int k = 0; k < KR; ++k) ad[k] = base + (off[k] ^ hz);
}

template <int Q, int KR, int DO, bool RTS, typename RF>
__device__ __forceinline__ void sus_check_phased(const WaveArgs &a, const TaskInfo &ti, const unsigned char *hdr, uint32_t pay_u32,
                                                 double *stage_x, uint64_t *empty, bool last, double *xp,
                                                 float *rsm, uint32_t rt, const unsigned short *rowtab,
                                                 int g, int c, int lane, bool frozen, RF &&refill) {
  using C = QC<Q, KR>;
  constexpr int T = C::T, LKR = C::LKR, LT = C::LT;
  static_assert(T > 1 && DO <= 3, "phased SUS check: q >= 16, degree <= 4");
  const SusDesc *sd = (const SusDesc *)(hdr + 128);
  const int z = hdr[256 + lane];
  const unsigned long long pke = sd->perm_e;
  const int s = ti.s;
  double acc[KR];
  if constexpr (DO == 0) {
    // degree-1 check: the convolution of no messages is the point mass at 0, so
    // r(a) = [h_e a = z] (times q, the dropped 1/q of the inverse transform)
    if (!last) {
      release_stage(empty, lane);
      refill();
    }
    const int az = rowtab[(size_t)(pke & 0xff) * Q + z] >> 7;  // h_e^-1 z (rare: degree-1 check)
#pragma unroll
    for (int k = 0; k < KR; ++k) acc[k] = (c * KR + k == az) ? (double)Q : 0.0;
    float *rs = rsm + (size_t)s * Q * 32 + lane + c * KR * 32;
#pragma unroll
    for (int k = 0; k < KR; ++k) rs[k * 32] = (float)acc[k];
    if (a.rmsg != nullptr && !frozen) {
      float *rdst = a.rmsg + ((size_t)ti.fb * a.c.E + ti.e0 + s) * Q * 32 + lane + c * KR * 32;
#pragma unroll
      for (int k = 0; k < KR; ++k) rdst[k * 32] = (float)acc[k];
    }
    return;
  } else {
    double v[DO][KR];
#pragma unroll
    for (int t = 0; t < DO; ++t) {
      uint32_t ad[KR];
      if (t == 0)   // the first other message carries the syndrome shift
        row_addrs_shift<Q, KR, RTS>(pay_u32 + (uint32_t)(lane * 4), rt, rowtab, sd->perm_o[0], c, z, ad);
      else
        row_addrs<Q, KR, RTS>(pay_u32 + (uint32_t)(t * Q * 128 + lane * 4), rt, rowtab, sd->perm_o[t], c, ad);
#pragma unroll
      for (int k = 0; k < KR; ++k) v[t][k] = (double)lds_f32(ad[k]);
    }
    if (DO <= 2 && !last) {
      release_stage(empty, lane);
      refill();
    }
#pragma unroll
    for (int t = 0; t < DO; ++t) wht_bits<KR, 0, LKR>(v[t]);
    constexpr int D1 = DO < 2 ? DO : 2;
    elided_bar<T>(g);  // xp reused across units without a barrier
#pragma unroll
    for (int t = 0; t < D1; ++t)
#pragma unroll
      for (int k = 0; k < KR; ++k) xp[((size_t)t * Q + idxA<Q, KR>(c, k)) * 32 + lane] = v[t][k];
    group_bar<T>(g);
#pragma unroll
    for (int t = 0; t < D1; ++t)
#pragma unroll
      for (int k = 0; k < KR; ++k) v[t][k] = xp[((size_t)t * Q + idxB<Q, KR>(c, k)) * 32 + lane];
    double *Z = xp;
    if constexpr (DO == 3) {
#pragma unroll
      for (int k = 0; k < KR; ++k) stage_x[idxA<Q, KR>(c, k) * 32 + lane] = v[2][k];
      group_bar<T>(g);
#pragma unroll
      for (int k = 0; k < KR; ++k) v[2][k] = stage_x[idxB<Q, KR>(c, k) * 32 + lane];
      Z = stage_x;
    }
#pragma unroll
    for (int t = 0; t < DO; ++t) wht_bits<KR, LKR - LT, LKR>(v[t]);
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      double x = v[0][k];
#pragma unroll
      for (int t = 1; t < DO; ++t) x *= v[t][k];
      acc[k] = x;
    }
    wht_bits<KR, LKR - LT, LKR>(acc);
    elided_bar<T>(g);  // the inverse switch overwrites the buffer just read
#pragma unroll
    for (int k = 0; k < KR; ++k) Z[idxB<Q, KR>(c, k) * 32 + lane] = acc[k];
    group_bar<T>(g);
#pragma unroll
    for (int k = 0; k < KR; ++k) acc[k] = Z[idxA<Q, KR>(c, k) * 32 + lane];
    if (DO == 3 && !last) {
      release_stage(empty, lane);  // the stage served as a transpose buffer
      refill();
    }
    wht_bits<KR, 0, LKR>(acc);
    uint32_t ad[KR];
    row_addrs<Q, KR, RTS>(0u, rt, rowtab, pke, c, ad);  // ad[k] = (h_e^-1 y) * 128: a = h_e^-1 y
    unsigned char *rs = (unsigned char *)(rsm + (size_t)s * Q * 32 + lane);
#pragma unroll
    for (int k = 0; k < KR; ++k) *(float *)(rs + ad[k]) = fmaxf((float)acc[k], 0.0f);
    if (a.rmsg != nullptr) {  // keep_messages only (export): warp-uniform branch
      if (!frozen) {
        unsigned char *rdst = (unsigned char *)(a.rmsg + ((size_t)ti.fb * a.c.E + ti.e0 + s) * Q * 32 + lane);
#pragma unroll
        for (int k = 0; k < KR; ++k) *(float *)(rdst + ad[k]) = fmaxf((float)acc[k], 0.0f);
      }
    }
  }
}

// MEASUREMENT VARIANT (GFQ_SUS_FWD32=1, off by default): the forward
// transforms of the d-1 other messages in fp32 (FADD butterflies, fp32 layout
// switches: all d-1 <= 3 messages through the group scratch in ONE barrier),
// the product, syndrome sign and inverse transform in fp64 as in
// sus_check_phased.  The inverse switch goes through the unit's own stage,
// released after it.  Its message-gate error is what DESIGN.md "Precision"
// reports for an fp32 forward transform.
#ifndef GFQ_SUS_FWD32
#define GFQ_SUS_FWD32 0
#endif
template <int KR, int LO, int HI>
__device__ __forceinline__ void wht_bits_f(float (&u)[KR]) {
#pragma unroll
  for (int m = LO; m < HI; ++m) {
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      if (!((k >> m) & 1)) {
        const float x = u[k], y = u[k | (1 << m)];
        u[k] = x + y;
        u[k | (1 << m)] = x - y;
      }
    }
  }
}

template <int Q, int KR, int DO, bool RTS, typename RF>
__device__ __forceinline__ void sus_check_fwd32(const WaveArgs &a, const TaskInfo &ti, const unsigned char *hdr, uint32_t pay_u32,
                                                double *stage_x, uint64_t *empty, bool last, double *xp,
                                                float *rsm, uint32_t rt, const unsigned short *rowtab,
                                                int g, int c, int lane, bool frozen, RF &&refill) {
  using C = QC<Q, KR>;
  constexpr int T = C::T, LKR = C::LKR, LT = C::LT;
  static_assert(T > 1 && DO >= 1 && DO <= 3, "fwd32 SUS check: q >= 16, 2 <= degree <= 4");
  static_assert((size_t)3 * Q * 32 * 4 <= (size_t)2 * Q * 32 * 8, "three fp32 messages fit the scratch");
  const SusDesc *sd = (const SusDesc *)(hdr + 128);
  const int z = hdr[256 + lane];
  const unsigned long long pke = sd->perm_e;
  const int s = ti.s;
  float v[DO][KR];
#pragma unroll
  for (int t = 0; t < DO; ++t) {
    uint32_t ad[KR];
    row_addrs<Q, KR, RTS>(pay_u32 + (uint32_t)(t * Q * 128 + lane * 4), rt, rowtab, sd->perm_o[t], c, ad);
#pragma unroll
    for (int k = 0; k < KR; ++k) v[t][k] = lds_f32(ad[k]);
  }
#pragma unroll
  for (int t = 0; t < DO; ++t) wht_bits_f<KR, 0, LKR>(v[t]);
  float *xf = (float *)xp;
#pragma unroll
  for (int t = 0; t < DO; ++t)
#pragma unroll
    for (int k = 0; k < KR; ++k) xf[((size_t)t * Q + idxA<Q, KR>(c, k)) * 32 + lane] = v[t][k];
  group_bar<T>(g);
#pragma unroll
  for (int t = 0; t < DO; ++t)
#pragma unroll
    for (int k = 0; k < KR; ++k) v[t][k] = xf[((size_t)t * Q + idxB<Q, KR>(c, k)) * 32 + lane];
#pragma unroll
  for (int t = 0; t < DO; ++t) wht_bits_f<KR, LKR - LT, LKR>(v[t]);
  uint32_t sm[KR];
  sign_masks<KR, T>(z, c, sm);
  double acc[KR];
#pragma unroll
  for (int k = 0; k < KR; ++k) {
    double x = (double)v[0][k];
#pragma unroll
    for (int t = 1; t < DO; ++t) x *= (double)v[t][k];
    acc[k] = flip(x, sm[k]);
  }
  wht_bits<KR, LKR - LT, LKR>(acc);
  // every warp has read its inputs from the stage (before the barrier above):
  // the stage serves as the inverse layout-switch buffer
#pragma unroll
  for (int k = 0; k < KR; ++k) stage_x[idxB<Q, KR>(c, k) * 32 + lane] = acc[k];
  group_bar<T>(g);
#pragma unroll
  for (int k = 0; k < KR; ++k) acc[k] = stage_x[idxA<Q, KR>(c, k) * 32 + lane];
  if (!last) {
    release_stage(empty, lane);
    refill();
  }
  wht_bits<KR, 0, LKR>(acc);
  uint32_t ad[KR];
  row_addrs<Q, KR, RTS>(0u, rt, rowtab, pke, c, ad);
  unsigned char *rs = (unsigned char *)(rsm + (size_t)s * Q * 32 + lane);
#pragma unroll
  for (int k = 0; k < KR; ++k) *(float *)(rs + ad[k]) = fmaxf((float)acc[k], 0.0f);
  if (a.rmsg != nullptr && !frozen) {
    unsigned char *rdst = (unsigned char *)(a.rmsg + ((size_t)ti.fb * a.c.E + ti.e0 + s) * Q * 32 + lane);
#pragma unroll
    for (int k = 0; k < KR; ++k) *(float *)(rdst + ad[k]) = fmaxf((float)acc[k], 0.0f);
  }
}

template <int Q, int KR, int DV, int DVMAX, bool MARKOV, bool ONEBAR, typename RF>
__device__ __forceinline__ void sus_vn(const WaveArgs &a, const TaskInfo &ti, const unsigned char *hdr, const unsigned char *xtra,
                                       const float *Tsm, uint64_t *empty, const float *rsm, double *red, int g,
                                       int c, int lane, bool frozen, bool late_release, RF &&refill) {
  const VarDesc *vd = (const VarDesc *)(hdr + 192);
  int qdst[DV > 0 ? DV : 1];
  double r[DV > 0 ? DV : 1][KR];
#pragma unroll
  for (int s = 0; s < DV; ++s) {
    qdst[s] = vd->qdst[s];
#pragma unroll
    for (int k = 0; k < KR; ++k) r[s][k] = (double)rsm[((size_t)s * Q + c * KR + k) * 32 + lane];
  }
  double pr[KR];
  prior_from<Q, KR, MARKOV>(a, ti.item, c, lane, (const float *)xtra, Tsm, pr);
  if (!late_release) {
    release_stage(empty, lane);
    refill();
  }
  vn_core<Q, KR, DV, MARKOV, ONEBAR>(a, ti.fb, ti.item, qdst, r, pr, red, g, c, lane, frozen);
  if (late_release) {  // red lives in the stage payload
    release_stage(empty, lane);
    refill();
  }
}

// ---------------------------------------------------------------- distributed stage issue (8-warp groups)
// With one producer lane per group, warp 0 of an 8-warp group executed ~25 %
// more instructions than the other seven (the unit walk, the header stores and
// 5-7 TMA issues per unit), and the group barriers made everybody wait for it:
// the read after the first barrier of a unit held 22 % of k_sus's stall samples
// at C5 (profiles/r02).  Here every warp of the group walks the units itself
// (UnitWalker, warp-uniform) and its lane 0 issues one share of the copies:
//   warp 0: the unit record (LvlUnit, 32 B -> header) and payload run 0
//   warp 1: payload run 1          warp 2: SusDesc and the syndrome row
//   warp 3: frame-state row, VarDesc (last unit)     warp 4: the prior's extra rows
// Warp 0 posts the stage's expect_tx for the unit that will REFILL a stage just
// before its own arrival on the stage's "empty" barrier; the other warps issue
// only after that barrier's phase has completed (which needs warp 0's
// arrival), so every complete_tx follows the expect_tx.  Nobody writes the
// header with plain stores any more: the consumers take the unit's fields from
// the TMA-copied record and the frame block from their own walker.
// MEASURED (profiles/r02/dc_variants.txt): correct (106 GPU tests) but 2.7 %
// SLOWER at C5 (182.6 vs 177.8 ms per sweep): seven more unit walks and five
// more waits per unit cost more than warp 0's detour saves -- the wait at the
// first barrier is the warp scheduler's, not the producer's.  Off by default.
#ifndef GFQ_SUS_DIST_ISSUE
#define GFQ_SUS_DIST_ISSUE 0
#endif
template <int Q, bool MARKOV>
__device__ __forceinline__ uint32_t sus_unit_tx_bytes(const WaveArgs &a, const LvlUnit &un) {
  const int nunits = un.dv > 0 ? un.dv : 1;
  const bool last = (un.s == nunits - 1);
  uint32_t b = 32;                                           // the unit record
  if (un.dv > 0) b += 64 + 32 + (uint32_t)(un.d - 1) * Q * 128;   // SusDesc, z row, the d-1 other messages
  if (a.early_exit) b += 128;
  if (last) b += 64 + extras_bytes<Q, MARKOV>(a, un.j);
  return b;
}
template <int Q, bool MARKOV>
__device__ __forceinline__ void sus_issue_share(const WaveArgs &a, int fb, int u, const LvlUnit &un, unsigned char *hdr,
                                                unsigned char *pay, unsigned char *xtra, uint64_t *full, int c) {
  const int nunits = un.dv > 0 ? un.dv : 1;
  const bool last = (un.s == nunits - 1);
  const float *rowbase = a.qmsg + ((size_t)fb * a.c.E + un.r0) * Q * 32;
  if (c == 0) {
    bulk_g2s(hdr, a.c.lvl_unit + u, 32, full);
    if (un.dv > 0 && un.pos > 0) bulk_g2s(pay, rowbase, (uint32_t)un.pos * Q * 128, full);
  } else if (c == 1) {
    if (un.dv > 0 && un.d - 1 - un.pos > 0)
      bulk_g2s(pay + (size_t)un.pos * Q * 128, rowbase + (size_t)(un.pos + 1) * Q * 32,
               (uint32_t)(un.d - 1 - un.pos) * Q * 128, full);
  } else if (c == 2) {
    if (un.dv > 0) {
      bulk_g2s(hdr + 128, a.c.sus_desc + un.e0 + un.s, 64, full);
      bulk_g2s(hdr + 256, a.z + ((size_t)fb * a.c.M + un.i) * 32, 32, full);
    }
  } else if (c == 3) {
    if (a.early_exit) bulk_g2s(hdr + 384, a.conv + fb * 32, 128, full);
    if (last) bulk_g2s(hdr + 192, a.c.var_desc + un.j, 64, full);
  } else if (c == 4) {
    if (last) issue_extras<Q, MARKOV>(a, fb, un.j, xtra, full);
  }
}

// For every column j of the level (SUS step 1): r_ij for each
// check i of column j from the CURRENT q's of check i's other edges; then
// (step 2) the vertical update of column j (Eq. 4) and its
// posterior (step 4, A8).  Columns of one level share no check, so they run
// concurrently with exactly the reads of the serial sweep.
template <int Q, int KR, int DMAX, int DVMAX, bool MARKOV, int S, int G>
__global__ void __launch_bounds__(SUSShape<Q, KR, DMAX, DVMAX, MARKOV, S, G>::THREADS)
    k_sus(WaveArgs a, int lvl_begin, int ncols) {
  using SS = SUSShape<Q, KR, DMAX, DVMAX, MARKOV, S, G>;
  using Sh = typename SS::Sh;
  constexpr int T = SS::T;
  constexpr int DO = DMAX - 1;
  extern __shared__ __align__(128) unsigned char smem[];
  const SmemPtrs sp = smem_ptrs<Sh, S, G>(smem);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // Programmatic dependent launch (levels are launched back to back, sus_launch):
  // let the next level's CTAs start their prologue now; they wait below.
  asm volatile("griddepcontrol.launch_dependents;");
  if (threadIdx.x == 0) init_bars<S, G>(sp.bars, T);
  if constexpr (SS::TSMEM) {
    if (a.Tf)
      for (int k = threadIdx.x; k < 2 * Q * Q; k += blockDim.x) sp.tsm[k] = a.Tf[k];
  }
  const float *Tp = SS::TSMEM ? sp.tsm : a.Tf;
  unsigned short *rtab = (unsigned short *)(sp.tsm + SS::TSM_F);
  if constexpr (SS::RTS)
    for (int k = threadIdx.x; k < Q * Q; k += blockDim.x) rtab[k] = a.c.rowtab[k];
  const uint32_t rt = smem_u32(rtab);
  __syncthreads();
  // everything below reads what the previous level (or iteration) wrote:
  // wait until that grid has completed and its memory is visible
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const long long ntask = (long long)(*a.nactive) * ncols;
  constexpr bool PW = PWof<T>::v;
  if (PW && warp == 0) {
    if (lane == 0) {
      int su[G];
#pragma unroll
      for (int g = 0; g < G; ++g) su[g] = 0;
      produce<S, G>(a, sp.bars, ntask, ncols, [&](int g, int st, const Cursor &cu) {
        const int k = g * S + st;
        int s = 0;
#pragma unroll
        for (int gg = 0; gg < G; ++gg)
          if (gg == g) s = su[gg];
        const bool done = sus_issue<Q, DMAX, MARKOV>(a, cu.fb, cu.item, s, lvl_begin, sp.hdr + (size_t)k * kHdr,
                                                     sp.pay + (size_t)k * Sh::PAYA,
                                                     sp.xtra + (size_t)k * Sh::XTRA_A, sp.bars + k);
#pragma unroll
        for (int gg = 0; gg < G; ++gg)
          if (gg == g) su[gg] = s;
        return done;
      }, lvl_begin);
    }
    return;
  }
  const int cw = PW ? warp - 1 : warp;
  const int g = cw / T, c = cw % T;
  const bool producer = !PW && (c == 0) && (lane == 0);
  unsigned char *scr = sp.scr + (size_t)g * SS::SCR;
  double *xp = (double *)scr;
  double *red = (double *)scr;  // aliases the transpose buffers (used after them)
  float *rsm = (float *)(scr + SS::XR_D * 8);
  int m = 0;  // ping-pong transpose counter
  long long lo, hi;
  sus_group_range(a, lvl_begin, ncols, (long long)(*a.nactive), (long long)blockIdx.x * G + g,
                  (long long)gridDim.x * G, lo, hi);
  // producer cursor over (task, unit) of this group
  constexpr bool DIST = (T == 8) && !PW && (GFQ_SUS_DIST_ISSUE != 0) && (S <= 2);
  UnitWalker pc;
  if (producer || DIST) pc.init(a, lo, hi, ncols, lvl_begin);
  auto issue_next = [&](int k) {
    if (!pc.valid()) return;
    const int fb = pc.fb;
    const LvlUnit un = pc.take(a);
    sus_issue_rec<Q, MARKOV>(a, fb, un, sp.hdr + (size_t)k * kHdr, sp.pay + (size_t)k * Sh::PAYA,
                             sp.xtra + (size_t)k * Sh::XTRA_A, sp.bars + k);
  };
  // DIST: the unit each stage will be refilled with (taken when the stage's
  // current unit is released) and the frame blocks of the units in flight
  int fbq0 = 0, fbq1 = 0;        // frame block of the unit in stage 0 / 1 of this group
  LvlUnit nxt_un;                // the unit taken at the last release (valid if nxt_ok)
  int nxt_fb = 0, nxt_u = 0;
  bool nxt_ok = false;
  auto dist_take = [&]() {       // every warp, warp-uniform
    nxt_ok = pc.valid();
    if (nxt_ok) {
      nxt_fb = pc.fb;
      nxt_u = pc.u;
      nxt_un = pc.take(a);
    }
  };
  auto dist_expect = [&](int k) {   // warp 0's lane 0, before its arrival on empty[k]
    if (nxt_ok && c == 0 && lane == 0)
      mbar_expect_tx(sp.bars + k, sus_unit_tx_bytes<Q, MARKOV>(a, nxt_un));
  };
  auto dist_issue = [&](int k, int st) {   // after the stage's empty phase (or in the prologue)
    if (!nxt_ok) return;
    if (st == 0) fbq0 = nxt_fb; else fbq1 = nxt_fb;
    if (lane == 0 && c <= 4)
      sus_issue_share<Q, MARKOV>(a, nxt_fb, nxt_u, nxt_un, sp.hdr + (size_t)k * kHdr, sp.pay + (size_t)k * Sh::PAYA,
                                 sp.xtra + (size_t)k * Sh::XTRA_A, sp.bars + k, c);
  };
  if constexpr (DIST) {
    // prologue: expect_tx of the first S units by warp 0, a group barrier, then the shares
#pragma unroll
    for (int n = 0; n < S; ++n) {
      dist_take();
      dist_expect(g * S + n);
      group_bar<T>(g);
      dist_issue(g * S + n, n);
    }
  } else {
    if (producer)
      for (int n = 0; n < S; ++n) issue_next(g * S + n);
  }
  int rr = 0;  // units consumed by this group
  for (long long task = lo; task < hi; ++task) {
    int nunits = 1;
#pragma unroll 1
    for (int s = 0; s < nunits; ++s, ++rr) {
      const int st = rr % S, k = g * S + st;
      const unsigned char *hdr = sp.hdr + (size_t)k * kHdr;
      const unsigned char *xtra = sp.xtra + (size_t)k * Sh::XTRA_A;
      const uint32_t pay_u32 = sp.pay_u32 + (uint32_t)((size_t)k * Sh::PAYA);
      uint64_t *empty = sp.bars + G * S + k;
      auto refill = [&]() {
        if constexpr (DIST) {
          // (release_stage ran just before: warp 0 posted the next expect_tx in it, see below)
          if (nxt_ok) {
            if (lane == 0 && c <= 4) mbar_wait(empty, (uint32_t)((rr / S) & 1));
            dist_issue(k, st);
          }
        } else {
          if (producer && pc.valid()) {
            mbar_wait(empty, (uint32_t)((rr / S) & 1));
            issue_next(k);
          }
        }
      };
      mbar_wait(sp.bars + k, (uint32_t)((rr / S) & 1));
      TaskInfo tinfo;
      if constexpr (DIST) {
        const LvlUnit lu = *(const LvlUnit *)hdr;
        tinfo.fb = (st == 0) ? fbq0 : fbq1;
        tinfo.item = lu.j; tinfo.e0 = lu.e0; tinfo.deg = lu.dv;
        tinfo.s = lu.s; tinfo.r0 = lu.r0; tinfo.d = lu.d; tinfo.pos = lu.pos; tinfo.i = lu.i;
        // the unit that will refill this stage: taken now, its expect_tx posted by
        // warp 0 right here -- before ANY warp of the group can release the stage
        // (every release follows this point in program order, and the other warps'
        // copies follow the completion of the empty phase, which needs warp 0's release)
        dist_take();
        dist_expect(k);
      } else {
        tinfo = *(const TaskInfo *)hdr;
      }
      const TaskInfo *ti = &tinfo;
      const int dv = ti->deg, d = ti->d;
      nunits = dv > 0 ? dv : 1;
      const bool last = (s == nunits - 1);
      const bool frozen = a.early_exit && ((const int *)(hdr + 384))[lane] != 0;
      double *stage_x = (double *)(sp.pay + (size_t)k * Sh::PAYA);
      if constexpr (SS::PHASED) {
        if (dv > 0) {
#define SP(n) sus_check_phased<Q, KR, n, SS::RTS>(a, tinfo, hdr, pay_u32, stage_x, empty, last, xp, rsm, rt, a.c.rowtab, g, c, lane, frozen, refill)
#define SP32(n) sus_check_fwd32<Q, KR, n, SS::RTS>(a, tinfo, hdr, pay_u32, stage_x, empty, last, xp, rsm, rt, a.c.rowtab, g, c, lane, frozen, refill)
          if constexpr (GFQ_SUS_FWD32 != 0) {
            switch (d - 1) {
              case 0: SP(0); break;
              case 1: SP32(1); break;
              case 2: SP32(2); break;
              default: SP32(3); break;
            }
          } else {
            switch (d - 1) {
              case 0: SP(0); break;
              case 1: SP(1); break;
              case 2: SP(2); break;
              default: SP(3); break;
            }
          }
#undef SP
#undef SP32
        }
      } else if (dv > 0) {
#define SC(n) sus_check<Q, KR, n, DMAX>(a, tinfo, hdr, pay_u32, empty, !last, xp, m, rsm, g, c, lane, frozen, refill)
        switch (d - 1) {
          case 0: SC(0); break;
          case 1: SC(1); break;
          case 2: SC(2); break;
          default:
            if constexpr (DO <= 3) {
              SC(3);
            } else {
              switch (d - 1) {
                case 3: SC(3); break;
                case 4: SC(4); break;
                case 5: SC(5); break;
                case 6: SC(6); break;
                default: SC(7); break;
              }
            }
            break;
        }
#undef SC
      }
      if (last) {
        // vertical update of column j from the fresh r's (SUS step 2)
        group_bar<T>(g);  // rsm complete, transpose buffers free for the reduction
#define SV(n) sus_vn<Q, KR, n, DVMAX, MARKOV, SS::PHASED && (T <= GFQ_ONEBAR_TMAX)>(a, tinfo, hdr, xtra, Tp, empty, rsm, SS::PHASED ? stage_x : red, g, c, lane, frozen, SS::PHASED, refill)
        switch (dv) {
          case 0: SV(0); break;
          case 1: SV(1); break;
          case 2: SV(2); break;
          default:
            if constexpr (DVMAX <= 3) {
              SV(3);
            } else {
              switch (dv) {
                case 3: SV(3); break;
                case 4: SV(4); break;
                case 5: SV(5); break;
                case 6: SV(6); break;
                case 7: SV(7); break;
                default: SV(8); break;
              }
            }
            break;
        }
#undef SV
        if constexpr (!SS::PHASED && SS::PP && SS::RED_D <= (size_t)Q * 32) m = 1;  // next transpose avoids red (buffer 0)
      }
      // Ping-pong transposes need no barrier between units (rsm slots are
      // distinct; the next rsm write follows a transpose barrier), and after
      // the variable update the next transpose writes buffer 1 while the
      // reduction scratch lives in buffer 0.  Bulk mode reuses its buffers.
      // Phased mode needs none either (see sus_check_phased; red is in the stage).
      if constexpr (!SS::PHASED && (!SS::PP || SS::RED_D > (size_t)Q * 32)) group_bar<T>(g);
      else elided_bar<T>(g);
    }
  }
}

// ============================================================== launchers
#define GFQ_DISPATCH_Q(q, F)  \
  switch (q) {                \
    case 2: return F(2);      \
    case 4: return F(4);      \
    case 8: return F(8);      \
    case 16: return F(16);    \
    case 32: return F(32);    \
    case 64: return F(64);    \
    case 128: return F(128);  \
    default: break;           \
  }                           \
  set_error("unsupported q"); \
  return GFQ_EUNSUPPORTED;

// stages per group (q = 16: 2, so that more CTAs fit an SM; measured on C4)
#ifndef GFQ_STAGES_CN
#define GFQ_STAGES_CN 3
#endif
#ifndef GFQ_STAGES_VN
#define GFQ_STAGES_VN 3
#endif
#ifndef GFQ_STAGES_Q16
#define GFQ_STAGES_Q16 2
#endif
#ifndef GFQ_STAGES_SUS
#define GFQ_STAGES_SUS 2
#endif

static int too_big(const char *what) {
  set_error(std::string(what) + ": this (q, degree) combination does not fit in shared memory");
  return GFQ_EUNSUPPORTED;
}

// stage count that fits: SMEM(S) = SMEM(1) + (S-1)*G*PAYA (+ headers)
template <typename S1, typename S2>
constexpr int stages_fit(int want) {
  return (S1::SMEM + (size_t)(want - 1) * (S2::SMEM - S1::SMEM) <= 232448 || want <= 1) ? want
                                                                                       : stages_fit<S1, S2>(want - 1);
}

template <int Q, int DM>
static int cn_launch(const WaveArgs &a, cudaStream_t s) {
  constexpr int KR = KRof<Q, KCN>::v, T = Q / KR, G = GQof<Q, T, KCN>::v;
  constexpr int NS = stages_fit<CNShape<Q, KR, DM, 1, G>, CNShape<Q, KR, DM, 2, G>>(Q == 16 ? GFQ_STAGES_Q16 : GFQ_STAGES_CN);
  using CS = CNShape<Q, KR, DM, NS, G>;
  if (CS::SMEM > 232448) return too_big("k_cn");
  auto k = k_cn<Q, KR, DM, NS, G>;
  const int grid = grid_for(k, CS::THREADS, CS::SMEM, ((long long)a.nfb * a.c.M + G - 1) / G);
  k<<<grid, CS::THREADS, CS::SMEM, s>>>(a);
  return check_launch("k_cn");
}

template <int Q>
static int cn_q(const WaveArgs &a, cudaStream_t s) {
  return a.c.max_cdeg <= 4 ? cn_launch<Q, 4>(a, s) : cn_launch<Q, 8>(a, s);
}

template <int Q, int DV, bool MK>
static int vn_launch(const WaveArgs &a, int clip, cudaStream_t s) {
  {
  constexpr int KR = KRof<Q, KVN>::v, T = Q / KR, G = GQof<Q, T, KVN>::v;
  constexpr int NS = stages_fit<VNShape<Q, KR, DV, MK, 1, G>, VNShape<Q, KR, DV, MK, 2, G>>(Q == 16 ? GFQ_STAGES_Q16 : GFQ_STAGES_VN);
  using VS = VNShape<Q, KR, DV, MK, NS, G>;
  if (VS::SMEM > 232448) return too_big("k_vn");
  auto k = k_vn<Q, KR, DV, MK, NS, G>;
  const int grid = grid_for(k, VS::THREADS, VS::SMEM, ((long long)a.nfb * a.c.V + G - 1) / G);
  k<<<grid, VS::THREADS, VS::SMEM, s>>>(a, clip);
  return check_launch("k_vn");
  }
}

template <int Q>
static int vn_q(const WaveArgs &a, int clip, cudaStream_t s) {
  const bool small = a.c.max_vdeg <= 3;
  if (a.markov) return small ? vn_launch<Q, 3, true>(a, clip, s) : vn_launch<Q, 8, true>(a, clip, s);
  return small ? vn_launch<Q, 3, false>(a, clip, s) : vn_launch<Q, 8, false>(a, clip, s);
}

template <int Q, int DM, int DV, bool MK>
static int sus_launch(const WaveArgs &a, int lb, int ncols, cudaStream_t s) {
  {
  constexpr int KR = KRof<Q, KSUS>::v, T = Q / KR, G = GQof<Q, T, KSUS>::v;
  constexpr int NS =
      stages_fit<SUSShape<Q, KR, DM, DV, MK, 1, G>, SUSShape<Q, KR, DM, DV, MK, 2, G>>(GFQ_STAGES_SUS);
  using SS = SUSShape<Q, KR, DM, DV, MK, NS, G>;
  if (SS::SMEM > 232448) return too_big("k_sus");
  auto k = k_sus<Q, KR, DM, DV, MK, NS, G>;
  const int grid = grid_for(k, SS::THREADS, SS::SMEM, ((long long)a.nfb * ncols + G - 1) / G);
  // programmatic dependent launch: the kernel waits (griddepcontrol.wait) for
  // the preceding grid before touching its outputs, so its launch and prologue
  // overlap the previous level's tail (the in-sweep prior runs ~N levels)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(SS::THREADS);
  cfg.dynamicSmemBytes = SS::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k, a, lb, ncols);
  if (e != cudaSuccess) return cuda_fail(e, "k_sus");
  return check_launch("k_sus");
  }
}

// q <= 16: the direct-convolution SUS kernel (gfq_sus_dc.cu) unless disabled
#ifndef GFQ_SUS_DC
#define GFQ_SUS_DC 1
#endif
template <int Q>
static int sus_q(const WaveArgs &a, int lb, int ncols, cudaStream_t s) {
  if (GFQ_SUS_DC && sus_dc_applies(a)) return launch_sus_dc(a, lb, ncols, s);
  if (sus_dc64_applies(a)) return launch_sus_dc64(a, lb, ncols, s);
  const bool small = a.c.max_cdeg <= 4 && a.c.max_vdeg <= 3;
  if (a.markov)
    return small ? sus_launch<Q, 4, 3, true>(a, lb, ncols, s) : sus_launch<Q, 8, 8, true>(a, lb, ncols, s);
  return small ? sus_launch<Q, 4, 3, false>(a, lb, ncols, s) : sus_launch<Q, 8, 8, false>(a, lb, ncols, s);
}

int launch_cn(const WaveArgs &a, cudaStream_t s) {
  if (big_applies(a)) return launch_big_cn(a, s);
  if (cn_dc_applies(a)) return launch_cn_dc(a, s);
#define F(Q) cn_q<Q>(a, s)
  GFQ_DISPATCH_Q(a.c.q, F)
#undef F
}

int launch_vn(const WaveArgs &a, cudaStream_t s) {
  if (big_applies(a)) return launch_big_vn(a, 0, s);
#define F(Q) vn_q<Q>(a, 0, s)
  GFQ_DISPATCH_Q(a.c.q, F)
#undef F
}

int launch_clip_priors(const WaveArgs &a, cudaStream_t s) {
  if (big_applies(a)) return launch_big_vn(a, 1, s);
#define F(Q) vn_q<Q>(a, 1, s)
  GFQ_DISPATCH_Q(a.c.q, F)
#undef F
}

int launch_sus_level(const WaveArgs &a, int lb, int ncols, cudaStream_t s) {
  if (big_applies(a)) return launch_big_sus(a, lb, ncols, s);
#define F(Q) sus_q<Q>(a, lb, ncols, s)
  GFQ_DISPATCH_Q(a.c.q, F)
#undef F
}

}  // namespace gfq

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

namespace gfq {

// Relative tolerance under which two posterior values count as a tie in the
// clipping step (reading A17; the oracle applies the same rule).
constexpr double kTieRel = 1e-5;

// ============================================================== configuration
constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x / 2); }

template <int Q, int KR_>
struct QC {
  static constexpr int P = ilog2(Q);
  static constexpr int KR = KR_;
  static constexpr int T = Q / KR;  // warps per task group
  static constexpr int LKR = ilog2(KR);
  static constexpr int LT = P - LKR;
  static_assert(KR >= 2 && KR <= Q && (Q % KR) == 0, "bad KR");
};

// entries per thread by field size and kernel (tuning knobs)
#ifndef GFQ_KR_CN16
#define GFQ_KR_CN16 16
#endif
#ifndef GFQ_KR_VN16
#define GFQ_KR_VN16 16
#endif
#ifndef GFQ_KR_SUS16
#define GFQ_KR_SUS16 8
#endif
enum KernelKind { KCN, KVN, KSUS };
template <int Q, int K>
struct KRof {
  static constexpr int v = Q <= 8 ? Q
                           : Q == 16 ? (K == KCN ? GFQ_KR_CN16 : K == KVN ? GFQ_KR_VN16 : GFQ_KR_SUS16)
                                     : 8;
};
// largest stage count in [2, max_s] such that the CTA fits the 227 KB of
// dynamic shared memory (per_stage and other are bytes per CTA)
constexpr int fit_stages(size_t per_stage, size_t other, int max_s) {
  return (other + (size_t)max_s * per_stage <= 232448 || max_s <= 2) ? max_s
                                                                     : fit_stages(per_stage, other, max_s - 1);
}

// groups per CTA for a given number of warps per group
template <int T>
struct Gof {
  static constexpr int v = T >= 8 ? 1 : (4 / T > 0 ? 4 / T : 1);
};

// ============================================================== PTX: mbarrier + TMA bulk copy
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

template <int T>
__device__ __forceinline__ void group_bar(int g) {
  if constexpr (T == 1) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "r"(T * 32) : "memory");
  }
}

// ============================================================== small helpers
// In-register WHT butterflies over bits [LO, HI) of the register index.
template <int KR, int LO, int HI>
__device__ __forceinline__ void wht_bits(double (&u)[KR]) {
#pragma unroll
  for (int m = LO; m < HI; ++m) {
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      if (!((k >> m) & 1)) {
        const double x = u[k], y = u[k | (1 << m)];
        u[k] = x + y;
        u[k | (1 << m)] = x - y;
      }
    }
  }
}

// Rows under the GF(2)-linear map y -> h^-1 y, from the images of the basis
// vectors bb[b] = h^-1 * 2^b (packed one byte each).
template <int P>
__device__ __forceinline__ void unpack_basis(unsigned long long pk, int (&bb)[P]) {
#pragma unroll
  for (int b = 0; b < P; ++b) bb[b] = (int)((pk >> (8 * b)) & 0xff);
}
template <int P, int LKR>
__device__ __forceinline__ int row_hi(const int (&bb)[P], int c) {  // image of c*KR
  int r = 0;
#pragma unroll
  for (int b = LKR; b < P; ++b)
    if ((c >> (b - LKR)) & 1) r ^= bb[b];
  return r;
}
template <int P, int LKR>
__device__ __forceinline__ int row_lo(const int (&bb)[P], int k) {  // image of k
  int r = 0;
#pragma unroll
  for (int b = 0; b < LKR; ++b)
    if ((k >> b) & 1) r ^= bb[b];
  return r;
}

__device__ __forceinline__ double neg_if(double v, int s) {
  return __longlong_as_double(__double_as_longlong(v) ^ ((long long)s << 63));
}

// Early exit freezes a converged frame: its lane keeps computing (warp-uniform
// control flow) but stores nothing.  Invalid lanes of a ragged last block are
// marked converged from the start.
__device__ __forceinline__ bool lane_frozen(const WaveArgs &a, int fb, int lane) {
  return a.early_exit && a.conv[fb * 32 + lane] != 0;
}

// Leave-one-out products in place: u[s] <- prod_{s' != s, s' < d} u[s'] (d <= DM).
template <int DM, int KR>
__device__ __forceinline__ void leave_one_out(double (&u)[DM][KR], int d) {
#pragma unroll
  for (int k = 0; k < KR; ++k) {
    if (d == 1) {
      u[0][k] = 1.0;
    } else if (d == 2) {
      const double t = u[0][k];
      u[0][k] = u[1][k];
      u[1][k] = t;
    } else if (d == 3) {
      const double a = u[0][k], b = u[1][k], c = u[2][k];
      u[0][k] = b * c;
      u[1][k] = a * c;
      u[2][k] = a * b;
    } else if (DM >= 4 && d == 4) {
      const double ab = u[0][k] * u[1][k], cd = u[2][k] * u[3][k];
      const double n0 = u[1][k] * cd, n1 = u[0][k] * cd;
      const double n2 = ab * u[3][k], n3 = ab * u[2][k];
      u[0][k] = n0; u[1][k] = n1; u[2][k] = n2; u[3][k] = n3;
    } else if (DM > 4) {  // generic prefix/suffix for 5..8
      double pre[DM];
      double acc = 1.0;
#pragma unroll
      for (int s = 0; s < DM; ++s) {
        pre[s] = acc;
        if (s < d) acc *= u[s][k];
      }
      acc = 1.0;
#pragma unroll
      for (int s = DM - 1; s >= 0; --s) {
        if (s < d) {
          const double o = u[s][k];
          u[s][k] = pre[s] * acc;
          acc *= o;
        }
      }
    }
  }
}

__device__ __forceinline__ bool mbar_test(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// A consumer warp is done reading a stage: one arrival per warp on its
// "empty" barrier (count T) lets the producer refill it.
__device__ __forceinline__ void release_stage(uint64_t *empty, int lane) {
  __syncwarp();
  if (lane == 0) mbar_arrive(empty);
}

// Contiguous share [lo, hi) of ntask tasks for global group gg of ngroups.
__device__ __forceinline__ void group_range(long long ntask, long long gg, long long ngroups, long long &lo,
                                            long long &hi) {
  const long long chunk = (ntask + ngroups - 1) / ngroups;
  lo = gg * chunk;
  hi = lo + chunk < ntask ? lo + chunk : ntask;
  if (lo > ntask) lo = ntask;
}

// Stage header written by the producer (plain shared store, published by the
// mbarrier arrive): task coordinates.
struct __align__(16) TaskInfo {
  int fb, item, e0, deg;  // block, check/variable, first edge, degree
  int s, r0, d, pos;      // SUS unit: check slot, check row start / degree, position of e
  int i, pad0, pad1, pad2;
};

// ============================================================== priors
// Extra rows a variable task needs besides its r messages, fetched into the
// stage after them: noise symbol -> its p per-bit flip probabilities; Markov
// source symbol (iteration >= 2) -> the posterior snapshots of j-1 and j+1.
template <int Q, bool MARKOV>
struct Extra {
  static constexpr int P = ilog2(Q);
  static constexpr int rows = MARKOV ? (2 * Q > P ? 2 * Q : P) : P;
};

template <int Q, bool MARKOV>
__device__ __forceinline__ uint32_t extras_bytes(const WaveArgs &a, int j) {
  constexpr int P = ilog2(Q);
  const int N = a.c.N;
  if (j >= N) return P * 128;
  if (MARKOV && a.t > 1 && a.qs_old) return (uint32_t)((j > 0) + (j < N - 1)) * Q * 128;
  return 0;
}

template <int Q, bool MARKOV>
__device__ __forceinline__ void issue_extras(const WaveArgs &a, int fb, int j, unsigned char *dst, uint64_t *bar) {
  constexpr int P = ilog2(Q);
  const int N = a.c.N;
  if (j >= N) {
    bulk_g2s(dst, a.pi + ((size_t)fb * a.c.M * P + (size_t)(j - N) * P) * 32, P * 128, bar);
  } else if (MARKOV && a.t > 1 && a.qs_old) {
    if (j > 0) bulk_g2s(dst, a.qs_old + ((size_t)fb * N + (j - 1)) * Q * 32, Q * 128, bar);
    if (j < N - 1) bulk_g2s(dst + Q * 128, a.qs_old + ((size_t)fb * N + (j + 1)) * Q * 32, Q * 128, bar);
  }
}

// Prior p_j^a for the KR entries a = c*KR + k (layout A) of this thread, from
// the extra rows in shared memory (ex):
//  - noise symbol j = N + m: prod_b (bit_b(a) ? pi_b : 1 - pi_b)
//  - source symbol, i.i.d. or first iteration: pi0(a)
//  - source symbol, Markov, iteration t >= 2: Eq. (7) from the
//    posterior snapshot Q^(t-1) of the neighbours (reading A9), boundaries A10:
//      p(b) = [sum_a Q_{j-1}(a) T_ab] * [sum_c T_bc Q_{j+1}(c)]
template <int Q, int KR, bool MARKOV>
__device__ __forceinline__ void prior_from(const WaveArgs &a, int j, int c, int lane, const float *ex,
                                           double (&pr)[KR]) {
  using C = QC<Q, KR>;
  constexpr int P = C::P, LKR = C::LKR;
  const int N = a.c.N;
  if (j >= N) {
    double pb[P];
#pragma unroll
    for (int b = 0; b < P; ++b) pb[b] = (double)ex[b * 32 + lane];
    double hi = 1.0;
#pragma unroll
    for (int b = LKR; b < P; ++b) hi *= ((c >> (b - LKR)) & 1) ? pb[b] : 1.0 - pb[b];
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      double v = hi;
#pragma unroll
      for (int b = 0; b < LKR; ++b) v *= ((k >> b) & 1) ? pb[b] : 1.0 - pb[b];
      pr[k] = v;
    }
    return;
  }
  if (!MARKOV || a.t <= 1 || a.qs_old == nullptr) {
#pragma unroll
    for (int k = 0; k < KR; ++k) pr[k] = __ldg(a.pi0 + c * KR + k);
    return;
  }
  double L[KR], R[KR];
  const float *exl = ex;
  const float *exr = ex + (j > 0 ? Q * 32 : 0);
  if (j > 0) {
#pragma unroll
    for (int k = 0; k < KR; ++k) L[k] = 0.0;
#pragma unroll 4
    for (int x = 0; x < Q; ++x) {
      const double qv = (double)exl[x * 32 + lane];
#pragma unroll
      for (int k = 0; k < KR; ++k) L[k] += qv * __ldg(a.T + x * Q + c * KR + k);
    }
  } else {
#pragma unroll
    for (int k = 0; k < KR; ++k) L[k] = __ldg(a.pi0 + c * KR + k);
  }
  if (j < N - 1) {
#pragma unroll
    for (int k = 0; k < KR; ++k) R[k] = 0.0;
#pragma unroll 4
    for (int x = 0; x < Q; ++x) {
      const double qv = (double)exr[x * 32 + lane];
#pragma unroll
      for (int k = 0; k < KR; ++k) R[k] += __ldg(a.T + (c * KR + k) * Q + x) * qv;
    }
  } else {
#pragma unroll
    for (int k = 0; k < KR; ++k) R[k] = 1.0;
  }
#pragma unroll
  for (int k = 0; k < KR; ++k) pr[k] = L[k] * R[k];
}

// ============================================================== variable node
// Eq. (4): q_ij^a = alpha_ij p_j^a prod_{i' != i} r_i'j^a, and
// Eq. (5): Q_j^a = alpha_j p_j^a prod_i r_ij^a, clipped to the
// smallest a within kTieRel of the maximum (reading A17).  r[s][k] holds r of
// check slot s at a = c*KR + k; pr the prior; qdst[s] the check-major id of
// the edge of slot s.  Writes the dv q messages, x_hat, the Markov snapshot
// and (keep) Q.  red: group scratch of (DVMAX+3)*T*32 doubles.
template <int Q, int KR, int DVMAX, bool MARKOV>
__device__ __forceinline__ void vn_body(const WaveArgs &a, int fb, int j, int dv, const int (&qdst)[DVMAX],
                                        double (&r)[DVMAX][KR], const double (&pr)[KR], double *red,
                                        int g, int c, int lane, bool frozen) {
  constexpr int T = Q / KR;
  const long long E = a.c.E;
  double tot[KR];
#pragma unroll
  for (int k = 0; k < KR; ++k) {
    double v = pr[k];
#pragma unroll
    for (int s = 0; s < DVMAX; ++s)
      if (s < dv) v *= r[s][k];
    tot[k] = v;
  }
  if (dv > 0) leave_one_out<DVMAX, KR>(r, dv);
  double sums[DVMAX + 1];
#pragma unroll
  for (int s = 0; s <= DVMAX; ++s) sums[s] = 0.0;
  double best = 0.0;
#pragma unroll
  for (int k = 0; k < KR; ++k) {
#pragma unroll
    for (int s = 0; s < DVMAX; ++s)
      if (s < dv) {
        r[s][k] *= pr[k];
        sums[s] += r[s][k];
      }
    sums[DVMAX] += tot[k];
    best = fmax(best, tot[k]);
  }
  if constexpr (T > 1) {
    // cross-warp reduction of the sums and of the maximum
#pragma unroll
    for (int s = 0; s <= DVMAX; ++s)
      if (s < dv || s == DVMAX) red[((size_t)s * T + c) * 32 + lane] = sums[s];
    red[((size_t)(DVMAX + 1) * T + c) * 32 + lane] = best;
    group_bar<T>(g);
#pragma unroll
    for (int s = 0; s <= DVMAX; ++s)
      if (s < dv || s == DVMAX) {
        double t = 0.0;
#pragma unroll
        for (int cc = 0; cc < T; ++cc) t += red[((size_t)s * T + cc) * 32 + lane];
        sums[s] = t;
      }
#pragma unroll
    for (int cc = 0; cc < T; ++cc) best = fmax(best, red[((size_t)(DVMAX + 1) * T + cc) * 32 + lane]);
  }
  // Clipping: the smallest a whose Q is within kTieRel of the maximum.
  const double thr = best * (1.0 - kTieRel);
  int bidx = Q;
#pragma unroll
  for (int k = KR - 1; k >= 0; --k)
    if (tot[k] >= thr) bidx = c * KR + k;
  if constexpr (T > 1) {
    int *ired = (int *)(red + (size_t)(DVMAX + 2) * T * 32);
    ired[c * 32 + lane] = bidx;
    group_bar<T>(g);
#pragma unroll
    for (int cc = 0; cc < T; ++cc) bidx = min(bidx, ired[cc * 32 + lane]);
  }
  if (bidx >= Q) bidx = 0;
  if (frozen) return;  // a converged frame keeps the state it converged with
  int bad = 0;
#pragma unroll
  for (int s = 0; s < DVMAX; ++s) {
    if (s < dv) {
      float *dst = a.qmsg + ((size_t)fb * E + qdst[s]) * Q * 32 + lane;
      const double sm = sums[s];
      const bool ok = sm > 0.0 && isfinite(sm);
      bad += !ok;
      const double inv = ok ? 1.0 / sm : 0.0;
#pragma unroll
      for (int k = 0; k < KR; ++k) dst[(c * KR + k) * 32] = ok ? (float)(r[s][k] * inv) : 1.0f / Q;
    }
  }
  const double st = sums[DVMAX];
  const bool okq = st > 0.0 && isfinite(st);
  bad += !okq;
  if (!okq) bidx = 0;
  const double invq = okq ? 1.0 / st : 0.0;
  if (MARKOV && j < a.c.N && a.qs_new) {
    float *dst = a.qs_new + ((size_t)fb * a.c.N + j) * Q * 32 + lane;
#pragma unroll
    for (int k = 0; k < KR; ++k) dst[(c * KR + k) * 32] = okq ? (float)(tot[k] * invq) : 1.0f / Q;
  }
  if (a.qall) {
    float *dst = a.qall + ((size_t)fb * a.c.V + j) * Q * 32 + lane;
#pragma unroll
    for (int k = 0; k < KR; ++k) dst[(c * KR + k) * 32] = okq ? (float)(tot[k] * invq) : 1.0f / Q;
  }
  if (c == 0) a.xhat[((size_t)fb * a.c.V + j) * 32 + lane] = (unsigned char)bidx;
  if (bad && c == 0) atomicAdd(a.stats + 0, (unsigned long long)bad);
}

// ============================================================== pipeline shapes
// CTA = 1 producer warp (lane 0 issues every TMA copy) + G groups of T
// consumer warps.  Group g owns a ring of S stages with "full" (TMA bytes
// landed) and "empty" (all T warps done reading) mbarriers.
//   stage = [TaskInfo 64B][static desc 64..128B][z 32B -> 128][conv 128B][payload]
constexpr int kHdr = 512;  // stage header bytes (payload offset)

template <int Q, int KR, int DMAX, int S, int G>
struct CNShape {
  static constexpr int T = Q / KR;
  static constexpr size_t STAGE_B = kHdr + (size_t)DMAX * Q * 128;
  static constexpr size_t SCR_B = T > 1 ? (size_t)DMAX * Q * 32 * 8 : 0;
  static constexpr size_t BARS_B = ((16 * S * G + 127) / 128) * 128;
  static constexpr size_t SMEM = BARS_B + (size_t)G * S * STAGE_B + (size_t)G * SCR_B;
  static constexpr int THREADS = (1 + G * T) * 32;
};

template <int Q, int KR, int DVMAX, bool MARKOV, int S, int G>
struct VNShape {
  static constexpr int T = Q / KR;
  static constexpr int XR = Extra<Q, MARKOV>::rows;
  static constexpr size_t STAGE_B = kHdr + ((size_t)DVMAX * Q + XR) * 128;
  static constexpr size_t SCR_B = (size_t)(DVMAX + 3) * T * 32 * 8;
  static constexpr size_t BARS_B = ((16 * S * G + 127) / 128) * 128;
  static constexpr size_t SMEM = BARS_B + (size_t)G * S * STAGE_B + (size_t)G * SCR_B;
  static constexpr int THREADS = (1 + G * T) * 32;
};

template <int Q, int KR, int DMAX, int DVMAX, bool MARKOV, int S, int G>
struct SUSShape {
  static constexpr int T = Q / KR;
  static constexpr int XR = Extra<Q, MARKOV>::rows;
  static constexpr size_t STAGE_B = kHdr + ((size_t)(DMAX - 1) * Q + XR) * 128;
  static constexpr size_t FWD_D = T > 1 ? (size_t)(DMAX - 1) * Q * 32 : 0;
  static constexpr size_t ACC_D = T > 1 ? (size_t)Q * 32 : 0;
  static constexpr size_t RED_D = (size_t)(DVMAX + 3) * T * 32;
  static constexpr size_t RSM_F = (size_t)DVMAX * Q * 32;
  static constexpr size_t SCR_B = (FWD_D + ACC_D + RED_D) * 8 + RSM_F * 4;
  static constexpr size_t BARS_B = ((16 * S * G + 127) / 128) * 128;
  static constexpr size_t SMEM = BARS_B + (size_t)G * S * STAGE_B + (size_t)G * SCR_B;
  static constexpr int THREADS = (1 + G * T) * 32;
};

template <int S, int G>
__device__ __forceinline__ void init_bars(uint64_t *bars, int T) {
  // bars[0 .. G*S): full (1 arrival + tx bytes), bars[G*S .. 2*G*S): empty (T arrivals)
  for (int k = 0; k < G * S; ++k) {
    mbar_init(bars + k, 1);
    mbar_init(bars + G * S + k, (uint32_t)T);
  }
  fence_mbar_init();
}

// ============================================================== PUS: check node
template <int Q, int DMAX>
__device__ __forceinline__ void cn_issue(const WaveArgs &a, long long task, unsigned char *sb, uint64_t *full) {
  const int M = a.c.M;
  const int fb = a.list[task / M];
  const int i = (int)(task % M);
  const int e0 = __ldg(a.c.row_ptr + i), d = __ldg(a.c.row_ptr + i + 1) - e0;
  TaskInfo *ti = (TaskInfo *)sb;
  ti->fb = fb; ti->item = i; ti->e0 = e0; ti->deg = d;
  const uint32_t msg = (uint32_t)d * Q * 128;
  mbar_expect_tx(full, 128 + 32 + (a.early_exit ? 128 : 0) + msg);
  bulk_g2s(sb + 128, a.c.check_desc + i, 128, full);
  bulk_g2s(sb + 256, a.z + ((size_t)fb * M + i) * 32, 32, full);
  if (a.early_exit) bulk_g2s(sb + 384, a.conv + fb * 32, 128, full);
  if (msg) bulk_g2s(sb + kHdr, a.qmsg + ((size_t)fb * a.c.E + e0) * Q * 32, msg, full);
}

// Eq. (3) for every edge of check i (horizontal pass),
// in the transform domain (BASELINE.json north_star): with u_k(y) =
// q_ij_k(h_k^-1 y) (the distribution of h_k x_k), U_k = WHT(u_k),
//   r_ij_k(a) = (1/q) WHT[ (-1)^{w.z_i} prod_{k' != k} U_k'(w) ](h_k a).
// The syndrome enters as the sign (-1)^{popc(w & z_i)} (XOR shift by z_i,
// reading A4).  Negative round-off is clamped to 0 (reading A20).
template <int Q, int KR, int DMAX, int S, int G>
__global__ void __launch_bounds__(CNShape<Q, KR, DMAX, S, G>::THREADS) k_cn(WaveArgs a) {
  using Sh = CNShape<Q, KR, DMAX, S, G>;
  using C = QC<Q, KR>;
  constexpr int T = C::T, LKR = C::LKR, LT = C::LT, P = C::P;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t *bars = (uint64_t *)smem;
  unsigned char *stages = smem + Sh::BARS_B;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) init_bars<S, G>(bars, T);
  __syncthreads();
  const int M = a.c.M;
  const long long E = a.c.E;
  const long long ntask = (long long)(*a.nactive) * M;
  const long long ngroups = (long long)gridDim.x * G;
  if (warp == 0) {  // ---------------- producer
    if (lane != 0) return;
    long long t[G], hi[G];
    int ring[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      group_range(ntask, (long long)blockIdx.x * G + g, ngroups, t[g], hi[g]);
      ring[g] = 0;
    }
    for (bool any = true; any;) {
      any = false;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        if (t[g] >= hi[g]) continue;
        any = true;
        const int st = ring[g] % S, u = ring[g] / S;
        if (u > 0 && !mbar_test(bars + G * S + g * S + st, (u - 1) & 1)) continue;
        cn_issue<Q, DMAX>(a, t[g], stages + (size_t)(g * S + st) * Sh::STAGE_B, bars + g * S + st);
        ++t[g];
        ++ring[g];
      }
    }
    return;
  }
  // ---------------- consumers
  const int cw = warp - 1, g = cw / T, c = cw % T;
  double *xp = (double *)(stages + (size_t)G * S * Sh::STAGE_B + (size_t)g * Sh::SCR_B);
  long long lo, hi;
  group_range(ntask, (long long)blockIdx.x * G + g, ngroups, lo, hi);
  for (long long task = lo; task < hi; ++task) {
    const int rr = (int)(task - lo), st = rr % S;
    unsigned char *sb = stages + (size_t)(g * S + st) * Sh::STAGE_B;
    mbar_wait(bars + g * S + st, (uint32_t)((rr / S) & 1));
    const TaskInfo ti = *(const TaskInfo *)sb;
    const CheckDesc *cd = (const CheckDesc *)(sb + 128);
    const int fb = ti.fb, d = ti.deg;
    const int z = sb[256 + lane];
    const bool frozen = a.early_exit && ((const int *)(sb + 384))[lane] != 0;
    const float *in = (const float *)(sb + kHdr) + lane;
    int bb[DMAX][P];
    int rc[DMAX];
    int canon[DMAX];
    double u[DMAX][KR];
#pragma unroll
    for (int s = 0; s < DMAX; ++s) {
      if (s < d) {
        unpack_basis<P>(cd->perm[s], bb[s]);
        canon[s] = cd->canon[s];
        rc[s] = row_hi<P, LKR>(bb[s], c);
#pragma unroll
        for (int k = 0; k < KR; ++k) u[s][k] = (double)in[(s * Q + (rc[s] ^ row_lo<P, LKR>(bb[s], k))) * 32];
      }
    }
    release_stage(bars + G * S + g * S + st, lane);
#pragma unroll
    for (int s = 0; s < DMAX; ++s)
      if (s < d) wht_bits<KR, 0, LKR>(u[s]);
    if constexpr (T > 1) {
#pragma unroll
      for (int s = 0; s < DMAX; ++s)
        if (s < d)
#pragma unroll
          for (int k = 0; k < KR; ++k) xp[((size_t)s * Q + c * KR + k) * 32 + lane] = u[s][k];
      group_bar<T>(g);
#pragma unroll
      for (int s = 0; s < DMAX; ++s)
        if (s < d) {
#pragma unroll
          for (int k = 0; k < KR; ++k) u[s][k] = xp[((size_t)s * Q + k * T + c) * 32 + lane];
          wht_bits<KR, LKR - LT, LKR>(u[s]);
        }
    }
    leave_one_out<DMAX, KR>(u, d);
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      const int w = (T > 1) ? (k * T + c) : k;
      const int sg = __popc(w & z) & 1;
#pragma unroll
      for (int s = 0; s < DMAX; ++s)
        if (s < d) u[s][k] = neg_if(u[s][k], sg);
    }
    if constexpr (T > 1) {
#pragma unroll
      for (int s = 0; s < DMAX; ++s)
        if (s < d) wht_bits<KR, LKR - LT, LKR>(u[s]);
      group_bar<T>(g);
#pragma unroll
      for (int s = 0; s < DMAX; ++s)
        if (s < d)
#pragma unroll
          for (int k = 0; k < KR; ++k) xp[((size_t)s * Q + k * T + c) * 32 + lane] = u[s][k];
      group_bar<T>(g);
#pragma unroll
      for (int s = 0; s < DMAX; ++s)
        if (s < d)
#pragma unroll
          for (int k = 0; k < KR; ++k) u[s][k] = xp[((size_t)s * Q + c * KR + k) * 32 + lane];
      group_bar<T>(g);
    }
    constexpr double invq = 1.0 / Q;
#pragma unroll
    for (int s = 0; s < DMAX; ++s) {
      if (s < d) {
        wht_bits<KR, 0, LKR>(u[s]);
        if (!frozen) {
          float *dst = a.rmsg + ((size_t)fb * E + canon[s]) * Q * 32 + lane;
#pragma unroll
          for (int k = 0; k < KR; ++k) {
            const double v = u[s][k] * invq;
            dst[(rc[s] ^ row_lo<P, LKR>(bb[s], k)) * 32] = (float)(v > 0.0 ? v : 0.0);
          }
        }
      }
    }
  }
}

// ============================================================== PUS: variable node
template <int Q, int DVMAX, bool MARKOV>
__device__ __forceinline__ void vn_issue(const WaveArgs &a, long long task, unsigned char *sb, uint64_t *full,
                                         int clip_only) {
  const int V = a.c.V;
  const int fb = a.list[task / V];
  const int j = (int)(task % V);
  const int e0 = __ldg(a.c.col_ptr + j);
  const int dv = clip_only ? 0 : __ldg(a.c.col_ptr + j + 1) - e0;
  TaskInfo *ti = (TaskInfo *)sb;
  ti->fb = fb; ti->item = j; ti->e0 = e0; ti->deg = dv;
  const uint32_t br = (uint32_t)dv * Q * 128;
  mbar_expect_tx(full, 64 + (a.early_exit ? 128 : 0) + br + extras_bytes<Q, MARKOV>(a, j));
  bulk_g2s(sb + 128, a.c.var_desc + j, 64, full);
  if (a.early_exit) bulk_g2s(sb + 384, a.conv + fb * 32, 128, full);
  if (br) bulk_g2s(sb + kHdr, a.rmsg + ((size_t)fb * a.c.E + e0) * Q * 32, br, full);  // canonical order
  issue_extras<Q, MARKOV>(a, fb, j, sb + kHdr + (size_t)DVMAX * Q * 128, full);
}

template <int Q, int KR, int DVMAX, bool MARKOV, int S, int G>
__global__ void __launch_bounds__(VNShape<Q, KR, DVMAX, MARKOV, S, G>::THREADS)
    k_vn(WaveArgs a, int clip_only) {
  using Sh = VNShape<Q, KR, DVMAX, MARKOV, S, G>;
  constexpr int T = Sh::T;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t *bars = (uint64_t *)smem;
  unsigned char *stages = smem + Sh::BARS_B;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) init_bars<S, G>(bars, T);
  __syncthreads();
  const int V = a.c.V;
  const long long ntask = (long long)(*a.nactive) * V;
  const long long ngroups = (long long)gridDim.x * G;
  if (warp == 0) {  // ---------------- producer
    if (lane != 0) return;
    long long t[G], hi[G];
    int ring[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      group_range(ntask, (long long)blockIdx.x * G + g, ngroups, t[g], hi[g]);
      ring[g] = 0;
    }
    for (bool any = true; any;) {
      any = false;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        if (t[g] >= hi[g]) continue;
        any = true;
        const int st = ring[g] % S, u = ring[g] / S;
        if (u > 0 && !mbar_test(bars + G * S + g * S + st, (u - 1) & 1)) continue;
        vn_issue<Q, DVMAX, MARKOV>(a, t[g], stages + (size_t)(g * S + st) * Sh::STAGE_B, bars + g * S + st,
                                   clip_only);
        ++t[g];
        ++ring[g];
      }
    }
    return;
  }
  const int cw = warp - 1, g = cw / T, c = cw % T;
  double *red = (double *)(stages + (size_t)G * S * Sh::STAGE_B + (size_t)g * Sh::SCR_B);
  long long lo, hi;
  group_range(ntask, (long long)blockIdx.x * G + g, ngroups, lo, hi);
  for (long long task = lo; task < hi; ++task) {
    const int rr = (int)(task - lo), st = rr % S;
    unsigned char *sb = stages + (size_t)(g * S + st) * Sh::STAGE_B;
    mbar_wait(bars + g * S + st, (uint32_t)((rr / S) & 1));
    const TaskInfo ti = *(const TaskInfo *)sb;
    const VarDesc *vd = (const VarDesc *)(sb + 128);
    const int fb = ti.fb, j = ti.item, dv = ti.deg;
    const bool frozen = a.early_exit && ((const int *)(sb + 384))[lane] != 0;
    const float *in = (const float *)(sb + kHdr);
    int qdst[DVMAX];
    double r[DVMAX][KR];
#pragma unroll
    for (int s = 0; s < DVMAX; ++s)
      if (s < dv) {
        qdst[s] = vd->qdst[s];
#pragma unroll
        for (int k = 0; k < KR; ++k) r[s][k] = (double)in[(s * Q + c * KR + k) * 32 + lane];
      }
    double pr[KR];
    prior_from<Q, KR, MARKOV>(a, j, c, lane, in + (size_t)DVMAX * Q * 32, pr);
    release_stage(bars + G * S + g * S + st, lane);
    vn_body<Q, KR, DVMAX, MARKOV>(a, fb, j, dv, qdst, r, pr, red, g, c, lane, frozen);
    if constexpr (T > 1) group_bar<T>(g);  // red reusable
  }
}

// ============================================================== SUS: one dependency level
// Units: one per (column, check slot) -- the check's other edges in at most
// two contiguous runs; the last unit of a column also carries the prior's
// extra rows and the column's VarDesc.
template <int Q, int DMAX, bool MARKOV>
__device__ __forceinline__ void sus_issue(const WaveArgs &a, long long task, int s, int lvl_begin, int ncols,
                                          unsigned char *sb, uint64_t *full, int &nunits_out) {
  const int fb = a.list[task / ncols];
  const LvlCol lc = a.c.lvl_col[lvl_begin + (int)(task % ncols)];
  const int nunits = lc.dv > 0 ? lc.dv : 1;
  nunits_out = nunits;
  const LvlUnit un = a.c.lvl_unit[lc.unit0 + s];
  TaskInfo *ti = (TaskInfo *)sb;
  ti->fb = fb; ti->item = lc.j; ti->e0 = lc.e0; ti->deg = lc.dv;
  ti->s = s; ti->r0 = un.r0; ti->d = un.d; ti->pos = un.pos; ti->i = un.i;
  const bool last = (s == nunits - 1);
  uint32_t b0 = 0, b1 = 0;
  const float *rowbase = a.qmsg + ((size_t)fb * a.c.E + un.r0) * Q * 32;
  if (lc.dv > 0) {
    b0 = (uint32_t)un.pos * Q * 128;
    b1 = (uint32_t)(un.d - 1 - un.pos) * Q * 128;
  }
  const uint32_t bx = last ? 64 + extras_bytes<Q, MARKOV>(a, lc.j) : 0;
  mbar_expect_tx(full, (lc.dv > 0 ? 64 + 32 : 0) + (a.early_exit ? 128 : 0) + b0 + b1 + bx);
  if (lc.dv > 0) {
    bulk_g2s(sb + 128, a.c.sus_desc + lc.e0 + s, 64, full);
    bulk_g2s(sb + 256, a.z + ((size_t)fb * a.c.M + un.i) * 32, 32, full);
  }
  if (a.early_exit) bulk_g2s(sb + 384, a.conv + fb * 32, 128, full);
  if (b0) bulk_g2s(sb + kHdr, rowbase, b0, full);
  if (b1) bulk_g2s(sb + kHdr + (size_t)un.pos * Q * 128, rowbase + (size_t)(un.pos + 1) * Q * 32, b1, full);
  if (last) {
    bulk_g2s(sb + 192, a.c.var_desc + lc.j, 64, full);
    issue_extras<Q, MARKOV>(a, fb, lc.j, sb + kHdr + (size_t)(DMAX - 1) * Q * 128, full);
  }
}

// For every column j of the level (SUS step 1): r_ij for each
// check i of column j from the CURRENT q's of check i's other edges (Eq. 3,
// the transform of k_cn restricted to one output); then (step 2)
// the vertical update of column j (Eq. 4) and its posterior (step 4, A8).
// Columns of one level share no check, so they run concurrently with exactly
// the reads of the serial sweep.
template <int Q, int KR, int DMAX, int DVMAX, bool MARKOV, int S, int G>
__global__ void __launch_bounds__(SUSShape<Q, KR, DMAX, DVMAX, MARKOV, S, G>::THREADS)
    k_sus(WaveArgs a, int lvl_begin, int ncols) {
  using Sh = SUSShape<Q, KR, DMAX, DVMAX, MARKOV, S, G>;
  using C = QC<Q, KR>;
  constexpr int T = C::T, LKR = C::LKR, LT = C::LT, P = C::P;
  constexpr int DO = DMAX - 1;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t *bars = (uint64_t *)smem;
  unsigned char *stages = smem + Sh::BARS_B;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) init_bars<S, G>(bars, T);
  __syncthreads();
  const long long E = a.c.E;
  const long long ntask = (long long)(*a.nactive) * ncols;
  const long long ngroups = (long long)gridDim.x * G;
  if (warp == 0) {  // ---------------- producer: walks (task, unit) per group
    if (lane != 0) return;
    long long t[G], hi[G];
    int ring[G], su[G], nu[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      group_range(ntask, (long long)blockIdx.x * G + g, ngroups, t[g], hi[g]);
      ring[g] = 0;
      su[g] = 0;
      nu[g] = 1;
    }
    for (bool any = true; any;) {
      any = false;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        if (t[g] >= hi[g]) continue;
        any = true;
        const int st = ring[g] % S, u = ring[g] / S;
        if (u > 0 && !mbar_test(bars + G * S + g * S + st, (u - 1) & 1)) continue;
        sus_issue<Q, DMAX, MARKOV>(a, t[g], su[g], lvl_begin, ncols, stages + (size_t)(g * S + st) * Sh::STAGE_B,
                                   bars + g * S + st, nu[g]);
        ++ring[g];
        if (++su[g] >= nu[g]) {
          su[g] = 0;
          ++t[g];
        }
      }
    }
    return;
  }
  const int cw = warp - 1, g = cw / T, c = cw % T;
  unsigned char *scr = stages + (size_t)G * S * Sh::STAGE_B + (size_t)g * Sh::SCR_B;
  double *fwd = (double *)scr;
  double *accs = fwd + Sh::FWD_D;
  double *red = accs + Sh::ACC_D;
  float *rsm = (float *)(red + Sh::RED_D);
  long long lo, hi;
  group_range(ntask, (long long)blockIdx.x * G + g, ngroups, lo, hi);
  int rr = 0;  // units consumed by this group
  for (long long task = lo; task < hi; ++task) {
    int nunits = 1;
#pragma unroll 1
    for (int s = 0; s < nunits; ++s, ++rr) {
      const int st = rr % S;
      unsigned char *sb = stages + (size_t)(g * S + st) * Sh::STAGE_B;
      uint64_t *empty = bars + G * S + g * S + st;
      mbar_wait(bars + g * S + st, (uint32_t)((rr / S) & 1));
      const TaskInfo ti = *(const TaskInfo *)sb;
      const int fb = ti.fb, j = ti.item, dv = ti.deg;
      nunits = dv > 0 ? dv : 1;
      const bool last = (s == nunits - 1);
      const bool frozen = a.early_exit && ((const int *)(sb + 384))[lane] != 0;
      if (dv > 0) {
        const SusDesc *sd = (const SusDesc *)(sb + 128);
        const int d = ti.d;
        const int z = sb[256 + lane];
        const float *in = (const float *)(sb + kHdr) + lane;
        int bbe[P];
        unpack_basis<P>(sd->perm_e, bbe);
        double v[DO > 0 ? DO : 1][KR];
#pragma unroll
        for (int t = 0; t < DO; ++t) {
          if (t < d - 1) {
            int bb[P];
            unpack_basis<P>(sd->perm_o[t], bb);
            const int rch = row_hi<P, LKR>(bb, c);
#pragma unroll
            for (int k = 0; k < KR; ++k) v[t][k] = (double)in[(t * Q + (rch ^ row_lo<P, LKR>(bb, k))) * 32];
          }
        }
        if (!last) release_stage(empty, lane);
#pragma unroll
        for (int t = 0; t < DO; ++t)
          if (t < d - 1) wht_bits<KR, 0, LKR>(v[t]);
        if constexpr (T > 1) {
#pragma unroll
          for (int t = 0; t < DO; ++t)
            if (t < d - 1)
#pragma unroll
              for (int k = 0; k < KR; ++k) fwd[((size_t)t * Q + c * KR + k) * 32 + lane] = v[t][k];
          group_bar<T>(g);
#pragma unroll
          for (int t = 0; t < DO; ++t)
            if (t < d - 1) {
#pragma unroll
              for (int k = 0; k < KR; ++k) v[t][k] = fwd[((size_t)t * Q + k * T + c) * 32 + lane];
              wht_bits<KR, LKR - LT, LKR>(v[t]);
            }
        }
        double acc[KR];
#pragma unroll
        for (int k = 0; k < KR; ++k) {
          double x = 1.0;
#pragma unroll
          for (int t = 0; t < DO; ++t)
            if (t < d - 1) x *= v[t][k];
          const int w = (T > 1) ? (k * T + c) : k;
          acc[k] = neg_if(x, __popc(w & z) & 1);
        }
        if constexpr (T > 1) {
          wht_bits<KR, LKR - LT, LKR>(acc);
#pragma unroll
          for (int k = 0; k < KR; ++k) accs[((size_t)k * T + c) * 32 + lane] = acc[k];
          group_bar<T>(g);
#pragma unroll
          for (int k = 0; k < KR; ++k) acc[k] = accs[((size_t)c * KR + k) * 32 + lane];
        }
        wht_bits<KR, 0, LKR>(acc);
        const int rch = row_hi<P, LKR>(bbe, c);
        float *rdst = (a.rmsg && !frozen) ? a.rmsg + ((size_t)fb * E + ti.e0 + s) * Q * 32 + lane : nullptr;
#pragma unroll
        for (int k = 0; k < KR; ++k) {
          const double x = acc[k] * (1.0 / Q);
          const float fv = (float)(x > 0.0 ? x : 0.0);
          const int row = rch ^ row_lo<P, LKR>(bbe, k);  // a = h_e^-1 y
          rsm[((size_t)s * Q + row) * 32 + lane] = fv;
          if (rdst) rdst[row * 32] = fv;
        }
      }
      if (last) {
        // vertical update of column j from the fresh r's (SUS step 2)
        group_bar<T>(g);  // rsm complete
        const VarDesc *vd = (const VarDesc *)(sb + 192);
        int qdst[DVMAX];
        double r[DVMAX][KR];
#pragma unroll
        for (int ss = 0; ss < DVMAX; ++ss)
          if (ss < dv) {
            qdst[ss] = vd->qdst[ss];
#pragma unroll
            for (int k = 0; k < KR; ++k) r[ss][k] = (double)rsm[((size_t)ss * Q + c * KR + k) * 32 + lane];
          }
        double pr[KR];
        prior_from<Q, KR, MARKOV>(a, j, c, lane, (const float *)(sb + kHdr) + (size_t)DO * Q * 32, pr);
        release_stage(empty, lane);
        vn_body<Q, KR, DVMAX, MARKOV>(a, fb, j, dv, qdst, r, pr, red, g, c, lane, frozen);
      }
      group_bar<T>(g);  // transpose / reduction scratch and rsm free
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
    default: break;           \
  }                           \
  set_error("unsupported q"); \
  return GFQ_EUNSUPPORTED;

#ifndef GFQ_STAGES_CN
#define GFQ_STAGES_CN 3
#endif
#ifndef GFQ_STAGES_VN
#define GFQ_STAGES_VN 3
#endif
#ifndef GFQ_STAGES_SUS
#define GFQ_STAGES_SUS 2
#endif

static int too_big(const char *what) {
  set_error(std::string(what) + ": this (q, degree) combination does not fit in shared memory");
  return GFQ_EUNSUPPORTED;
}

template <int Q, int DM>
static int cn_launch(const WaveArgs &a, cudaStream_t s) {
  constexpr int KR = KRof<Q, KCN>::v, T = Q / KR, G = Gof<T>::v;
  using S1 = CNShape<Q, KR, DM, 1, G>;
  constexpr int NS = fit_stages(G * S1::STAGE_B, S1::BARS_B + G * S1::SCR_B, GFQ_STAGES_CN);
  using Sh = CNShape<Q, KR, DM, NS, G>;
  if (Sh::SMEM > 232448) return too_big("k_cn");
  auto k = k_cn<Q, KR, DM, NS, G>;
  const int grid = grid_for(k, Sh::THREADS, Sh::SMEM, ((long long)a.nfb * a.c.M + G - 1) / G);
  k<<<grid, Sh::THREADS, Sh::SMEM, s>>>(a);
  return check_launch("k_cn");
}

template <int Q>
static int cn_q(const WaveArgs &a, cudaStream_t s) {
  return a.c.max_cdeg <= 4 ? cn_launch<Q, 4>(a, s) : cn_launch<Q, 8>(a, s);
}

template <int Q, int DV, bool MK>
static int vn_launch(const WaveArgs &a, int clip, cudaStream_t s) {
  constexpr int KR = KRof<Q, KVN>::v, T = Q / KR, G = Gof<T>::v;
  using S1 = VNShape<Q, KR, DV, MK, 1, G>;
  constexpr int NS = fit_stages(G * S1::STAGE_B, S1::BARS_B + G * S1::SCR_B, GFQ_STAGES_VN);
  using Sh = VNShape<Q, KR, DV, MK, NS, G>;
  if (Sh::SMEM > 232448) return too_big("k_vn");
  auto k = k_vn<Q, KR, DV, MK, NS, G>;
  const int grid = grid_for(k, Sh::THREADS, Sh::SMEM, ((long long)a.nfb * a.c.V + G - 1) / G);
  k<<<grid, Sh::THREADS, Sh::SMEM, s>>>(a, clip);
  return check_launch("k_vn");
}

template <int Q>
static int vn_q(const WaveArgs &a, int clip, cudaStream_t s) {
  const bool small = a.c.max_vdeg <= 3;
  if (a.markov) return small ? vn_launch<Q, 3, true>(a, clip, s) : vn_launch<Q, 8, true>(a, clip, s);
  return small ? vn_launch<Q, 3, false>(a, clip, s) : vn_launch<Q, 8, false>(a, clip, s);
}

template <int Q, int DM, int DV, bool MK>
static int sus_launch(const WaveArgs &a, int lb, int ncols, cudaStream_t s) {
  constexpr int KR = KRof<Q, KSUS>::v, T = Q / KR, G = Gof<T>::v;
  using S1 = SUSShape<Q, KR, DM, DV, MK, 1, G>;
  constexpr int NS = fit_stages(G * S1::STAGE_B, S1::BARS_B + G * S1::SCR_B, GFQ_STAGES_SUS);
  using Sh = SUSShape<Q, KR, DM, DV, MK, NS, G>;
  if (Sh::SMEM > 232448) return too_big("k_sus");
  auto k = k_sus<Q, KR, DM, DV, MK, NS, G>;
  const int grid = grid_for(k, Sh::THREADS, Sh::SMEM, ((long long)a.nfb * ncols + G - 1) / G);
  k<<<grid, Sh::THREADS, Sh::SMEM, s>>>(a, lb, ncols);
  return check_launch("k_sus");
}

template <int Q>
static int sus_q(const WaveArgs &a, int lb, int ncols, cudaStream_t s) {
  const bool small = a.c.max_cdeg <= 4 && a.c.max_vdeg <= 3;
  if (a.markov)
    return small ? sus_launch<Q, 4, 3, true>(a, lb, ncols, s) : sus_launch<Q, 8, 8, true>(a, lb, ncols, s);
  return small ? sus_launch<Q, 4, 3, false>(a, lb, ncols, s) : sus_launch<Q, 8, 8, false>(a, lb, ncols, s);
}

int launch_cn(const WaveArgs &a, cudaStream_t s) {
#define F(Q) cn_q<Q>(a, s)
  GFQ_DISPATCH_Q(a.c.q, F)
#undef F
}

int launch_vn(const WaveArgs &a, cudaStream_t s) {
#define F(Q) vn_q<Q>(a, 0, s)
  GFQ_DISPATCH_Q(a.c.q, F)
#undef F
}

int launch_clip_priors(const WaveArgs &a, cudaStream_t s) {
#define F(Q) vn_q<Q>(a, 1, s)
  GFQ_DISPATCH_Q(a.c.q, F)
#undef F
}

int launch_sus_level(const WaveArgs &a, int lb, int ncols, cudaStream_t s) {
#define F(Q) sus_q<Q>(a, lb, ncols, s)
  GFQ_DISPATCH_Q(a.c.q, F)
#undef F
}

}  // namespace gfq

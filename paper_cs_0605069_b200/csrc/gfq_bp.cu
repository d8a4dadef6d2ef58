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

// entries per thread by field size (tuning knob)
template <int Q>
struct KRof {
  static constexpr int v = Q <= 8 ? Q : 8;
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
__device__ __forceinline__ uint32_t issue_extras(const WaveArgs &a, int fb, int j, float *dst,
                                                 const float *(&src)[2], uint32_t (&nb)[2],
                                                 float *(&dsts)[2]) {
  constexpr int P = ilog2(Q);
  const int N = a.c.N;
  uint32_t total = 0;
  nb[0] = nb[1] = 0;
  if (j >= N) {
    src[0] = a.pi + ((size_t)fb * a.c.M * P + (size_t)(j - N) * P) * 32;
    dsts[0] = dst;
    nb[0] = P * 128;
    total = nb[0];
  } else if (MARKOV && a.t > 1 && a.qs_old) {
    if (j > 0) {
      src[0] = a.qs_old + ((size_t)fb * N + (j - 1)) * Q * 32;
      dsts[0] = dst;
      nb[0] = Q * 128;
    }
    if (j < N - 1) {
      src[1] = a.qs_old + ((size_t)fb * N + (j + 1)) * Q * 32;
      dsts[1] = dst + Q * 32;
      nb[1] = Q * 128;
    }
    total = nb[0] + nb[1];
  }
  return total;
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
  if (j > 0) {
#pragma unroll
    for (int k = 0; k < KR; ++k) L[k] = 0.0;
#pragma unroll 4
    for (int x = 0; x < Q; ++x) {
      const double qv = (double)ex[x * 32 + lane];
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
      const double qv = (double)ex[(Q + x) * 32 + lane];
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
// check slot s at a = c*KR + k; pr the prior.  Writes the dv q messages (to
// their check-major slots), x_hat, the Markov snapshot and (keep) Q.
// red: group scratch of (DVMAX+3)*T*32 doubles.
template <int Q, int KR, int DVMAX, bool MARKOV>
__device__ __forceinline__ void vn_body(const WaveArgs &a, int fb, int j, int e0, int dv,
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
      const int e = __ldg(a.c.col_edge + e0 + s);
      float *dst = a.qmsg + ((size_t)fb * E + e) * Q * 32 + lane;
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

// ============================================================== PUS: check node
template <int Q, int KR, int DMAX, int S, int G>
struct CNShape {
  static constexpr int T = Q / KR;
  static constexpr size_t STAGE_F = (size_t)DMAX * Q * 32;
  static constexpr size_t XP_D = T > 1 ? (size_t)DMAX * Q * 32 : 0;
  static constexpr size_t GROUP_BYTES = 128 + S * STAGE_F * 4 + XP_D * 8;
  static constexpr size_t SMEM = G * GROUP_BYTES;
  static constexpr int THREADS = G * T * 32;
};

template <int Q>
__device__ __forceinline__ void cn_issue(const WaveArgs &a, long long task, long long ntask, float *dst,
                                         uint64_t *bar) {
  if (task >= ntask) return;
  const int M = a.c.M;
  const int fb = a.list[task / M];
  const int i = (int)(task % M);
  const int e0 = __ldg(a.c.row_ptr + i), d = __ldg(a.c.row_ptr + i + 1) - e0;
  const uint32_t bytes = (uint32_t)d * Q * 128;
  mbar_expect_tx(bar, bytes);
  if (bytes) bulk_g2s(dst, a.qmsg + ((size_t)fb * a.c.E + e0) * Q * 32, bytes, bar);
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
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = warp / T, c = warp % T;
  unsigned char *gb = smem + (size_t)g * Sh::GROUP_BYTES;
  uint64_t *bars = (uint64_t *)gb;
  float *stg = (float *)(gb + 128);
  double *xp = (double *)(gb + 128 + S * Sh::STAGE_F * 4);
  const bool producer = (c == 0) && (lane == 0);
  if (producer) {
#pragma unroll
    for (int s = 0; s < S; ++s) mbar_init(bars + s, 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int M = a.c.M;
  const long long E = a.c.E;
  const long long ntask = (long long)(*a.nactive) * M;
  const long long first = (long long)blockIdx.x * G + g, stride = (long long)gridDim.x * G;
  if (producer) {
#pragma unroll
    for (int n = 0; n < S; ++n) cn_issue<Q>(a, first + n * stride, ntask, stg + n * Sh::STAGE_F, bars + n);
  }
  for (long long n = 0;; ++n) {
    const long long task = first + n * stride;
    if (task >= ntask) break;
    const int st = (int)(n % S);
    const int fb = a.list[task / M];
    const int i = (int)(task % M);
    const int e0 = __ldg(a.c.row_ptr + i), d = __ldg(a.c.row_ptr + i + 1) - e0;
    const int z = a.z[((size_t)fb * M + i) * 32 + lane];
    int bb[DMAX][P];
    int rc[DMAX];
#pragma unroll
    for (int s = 0; s < DMAX; ++s) {
      if (s < d) {
        unpack_basis<P>(__ldg(a.c.edge_perm + e0 + s), bb[s]);
        rc[s] = row_hi<P, LKR>(bb[s], c);
      }
    }
    mbar_wait(bars + st, (uint32_t)((n / S) & 1));
    const float *in = stg + st * Sh::STAGE_F + lane;
    double u[DMAX][KR];
#pragma unroll
    for (int s = 0; s < DMAX; ++s) {
      if (s < d) {
#pragma unroll
        for (int k = 0; k < KR; ++k) u[s][k] = (double)in[(s * Q + (rc[s] ^ row_lo<P, LKR>(bb[s], k))) * 32];
        wht_bits<KR, 0, LKR>(u[s]);
      }
    }
    if constexpr (T > 1) {
#pragma unroll
      for (int s = 0; s < DMAX; ++s)
        if (s < d)
#pragma unroll
          for (int k = 0; k < KR; ++k) xp[((size_t)s * Q + c * KR + k) * 32 + lane] = u[s][k];
      group_bar<T>(g);
      // every warp of the group has read its rows of stage st: refill it
      if (producer) cn_issue<Q>(a, task + S * stride, ntask, stg + st * Sh::STAGE_F, bars + st);
#pragma unroll
      for (int s = 0; s < DMAX; ++s)
        if (s < d) {
#pragma unroll
          for (int k = 0; k < KR; ++k) u[s][k] = xp[((size_t)s * Q + k * T + c) * 32 + lane];
          wht_bits<KR, LKR - LT, LKR>(u[s]);
        }
    } else {
      __syncwarp();
      if (producer) cn_issue<Q>(a, task + S * stride, ntask, stg + st * Sh::STAGE_F, bars + st);
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
    const bool frozen = lane_frozen(a, fb, lane);
#pragma unroll
    for (int s = 0; s < DMAX; ++s) {
      if (s < d) {
        wht_bits<KR, 0, LKR>(u[s]);
        if (!frozen) {
          float *dst = a.rmsg + ((size_t)fb * E + __ldg(a.c.edge_canon + e0 + s)) * Q * 32 + lane;
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
template <int Q, int KR, int DVMAX, bool MARKOV, int S, int G>
struct VNShape {
  static constexpr int T = Q / KR;
  static constexpr int XR = Extra<Q, MARKOV>::rows;
  static constexpr size_t STAGE_F = ((size_t)DVMAX * Q + XR) * 32;
  static constexpr size_t RED_D = (size_t)(DVMAX + 3) * T * 32;
  static constexpr size_t GROUP_BYTES = 128 + S * STAGE_F * 4 + RED_D * 8;
  static constexpr size_t SMEM = G * GROUP_BYTES;
  static constexpr int THREADS = G * T * 32;
};

template <int Q, int DVMAX, bool MARKOV>
__device__ __forceinline__ void vn_issue(const WaveArgs &a, long long task, long long ntask, float *dst,
                                         uint64_t *bar, int clip_only) {
  if (task >= ntask) return;
  const int V = a.c.V;
  const int fb = a.list[task / V];
  const int j = (int)(task % V);
  const int e0 = __ldg(a.c.col_ptr + j);
  const int dv = clip_only ? 0 : __ldg(a.c.col_ptr + j + 1) - e0;
  const uint32_t br = (uint32_t)dv * Q * 128;
  const float *xs[2] = {nullptr, nullptr};
  float *xd[2] = {nullptr, nullptr};
  uint32_t xb[2];
  const uint32_t bx = issue_extras<Q, MARKOV>(a, fb, j, dst + (size_t)DVMAX * Q * 32, xs, xb, xd);
  mbar_expect_tx(bar, br + bx);
  if (br) bulk_g2s(dst, a.rmsg + ((size_t)fb * a.c.E + e0) * Q * 32, br, bar);  // canonical order
  if (xb[0]) bulk_g2s(xd[0], xs[0], xb[0], bar);
  if (xb[1]) bulk_g2s(xd[1], xs[1], xb[1], bar);
}

template <int Q, int KR, int DVMAX, bool MARKOV, int S, int G>
__global__ void __launch_bounds__(VNShape<Q, KR, DVMAX, MARKOV, S, G>::THREADS)
    k_vn(WaveArgs a, int clip_only) {
  using Sh = VNShape<Q, KR, DVMAX, MARKOV, S, G>;
  constexpr int T = Sh::T;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = warp / T, c = warp % T;
  unsigned char *gb = smem + (size_t)g * Sh::GROUP_BYTES;
  uint64_t *bars = (uint64_t *)gb;
  float *stg = (float *)(gb + 128);
  double *red = (double *)(gb + 128 + S * Sh::STAGE_F * 4);
  const bool producer = (c == 0) && (lane == 0);
  if (producer) {
#pragma unroll
    for (int s = 0; s < S; ++s) mbar_init(bars + s, 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int V = a.c.V;
  const long long ntask = (long long)(*a.nactive) * V;
  const long long first = (long long)blockIdx.x * G + g, stride = (long long)gridDim.x * G;
  if (producer) {
#pragma unroll
    for (int n = 0; n < S; ++n)
      vn_issue<Q, DVMAX, MARKOV>(a, first + n * stride, ntask, stg + n * Sh::STAGE_F, bars + n, clip_only);
  }
  for (long long n = 0;; ++n) {
    const long long task = first + n * stride;
    if (task >= ntask) break;
    const int st = (int)(n % S);
    const int fb = a.list[task / V];
    const int j = (int)(task % V);
    const int e0 = __ldg(a.c.col_ptr + j);
    const int dv = clip_only ? 0 : __ldg(a.c.col_ptr + j + 1) - e0;
    const bool frozen = lane_frozen(a, fb, lane);
    mbar_wait(bars + st, (uint32_t)((n / S) & 1));
    const float *in = stg + st * Sh::STAGE_F;
    double r[DVMAX][KR];
#pragma unroll
    for (int s = 0; s < DVMAX; ++s)
      if (s < dv)
#pragma unroll
        for (int k = 0; k < KR; ++k) r[s][k] = (double)in[(s * Q + c * KR + k) * 32 + lane];
    double pr[KR];
    prior_from<Q, KR, MARKOV>(a, j, c, lane, in + (size_t)DVMAX * Q * 32, pr);
    group_bar<T>(g);  // stage st fully read by the group
    if (producer)
      vn_issue<Q, DVMAX, MARKOV>(a, task + S * stride, ntask, stg + st * Sh::STAGE_F, bars + st, clip_only);
    vn_body<Q, KR, DVMAX, MARKOV>(a, fb, j, e0, dv, r, pr, red, g, c, lane, frozen);
    if constexpr (T > 1) group_bar<T>(g);  // red reusable
  }
}

// ============================================================== SUS: one dependency level
template <int Q, int KR, int DMAX, int DVMAX, bool MARKOV, int S, int G>
struct SUSShape {
  static constexpr int T = Q / KR;
  static constexpr int XR = Extra<Q, MARKOV>::rows;
  static constexpr size_t STAGE_F = ((size_t)(DMAX - 1) * Q + XR) * 32;
  static constexpr size_t FWD_D = T > 1 ? (size_t)(DMAX - 1) * Q * 32 : 0;
  static constexpr size_t ACC_D = T > 1 ? (size_t)Q * 32 : 0;
  static constexpr size_t RED_D = (size_t)(DVMAX + 3) * T * 32;
  static constexpr size_t RSM_F = (size_t)DVMAX * Q * 32;
  static constexpr size_t GROUP_BYTES = 128 + S * STAGE_F * 4 + FWD_D * 8 + ACC_D * 8 + RED_D * 8 + RSM_F * 4;
  static constexpr size_t SMEM = G * GROUP_BYTES;
  static constexpr int THREADS = G * T * 32;
};

// Producer cursor over SUS "units": one unit = one check of one column
// (its other edges, in at most two contiguous runs); the last unit of a
// column also carries the prior's extra rows.
struct SusCursor {
  long long n;  // task index of this group
  int s;        // check slot within the column
};

template <int Q, int DMAX, bool MARKOV>
__device__ __forceinline__ void sus_issue(const WaveArgs &a, SusCursor &cur, long long first, long long stride,
                                          long long ntask, int lvl_begin, int ncols, float *dst,
                                          uint64_t *bar) {
  const long long task = first + cur.n * stride;
  if (task >= ntask) return;
  const int fb = a.list[task / ncols];
  const int j = __ldg(a.c.level_cols + lvl_begin + (int)(task % ncols));
  const int e0 = __ldg(a.c.col_ptr + j), dv = __ldg(a.c.col_ptr + j + 1) - e0;
  const int nunits = dv > 0 ? dv : 1;
  const int s = cur.s;
  const float *src0 = nullptr, *src1 = nullptr;
  uint32_t b0 = 0, b1 = 0;
  int pos = 0;
  if (dv > 0) {
    const int e = __ldg(a.c.col_edge + e0 + s);
    const int i = __ldg(a.c.edge_check + e);
    const int r0 = __ldg(a.c.row_ptr + i), d = __ldg(a.c.row_ptr + i + 1) - r0;
    pos = e - r0;
    const float *rowbase = a.qmsg + ((size_t)fb * a.c.E + r0) * Q * 32;
    src0 = rowbase;
    b0 = (uint32_t)pos * Q * 128;
    src1 = rowbase + (size_t)(pos + 1) * Q * 32;
    b1 = (uint32_t)(d - 1 - pos) * Q * 128;
  }
  const float *xs[2] = {nullptr, nullptr};
  float *xd[2] = {nullptr, nullptr};
  uint32_t xb[2] = {0, 0};
  uint32_t bx = 0;
  if (s == nunits - 1) bx = issue_extras<Q, MARKOV>(a, fb, j, dst + (size_t)(DMAX - 1) * Q * 32, xs, xb, xd);
  mbar_expect_tx(bar, b0 + b1 + bx);
  if (b0) bulk_g2s(dst, src0, b0, bar);
  if (b1) bulk_g2s(dst + (size_t)pos * Q * 32, src1, b1, bar);
  if (xb[0]) bulk_g2s(xd[0], xs[0], xb[0], bar);
  if (xb[1]) bulk_g2s(xd[1], xs[1], xb[1], bar);
  if (++cur.s == nunits) {
    cur.s = 0;
    ++cur.n;
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
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = warp / T, c = warp % T;
  unsigned char *gb = smem + (size_t)g * Sh::GROUP_BYTES;
  uint64_t *bars = (uint64_t *)gb;
  float *stg = (float *)(gb + 128);
  double *fwd = (double *)(gb + 128 + S * Sh::STAGE_F * 4);
  double *accs = fwd + Sh::FWD_D;
  double *red = accs + Sh::ACC_D;
  float *rsm = (float *)(red + Sh::RED_D);
  const bool producer = (c == 0) && (lane == 0);
  if (producer) {
#pragma unroll
    for (int s = 0; s < S; ++s) mbar_init(bars + s, 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int M = a.c.M;
  const long long E = a.c.E;
  const long long ntask = (long long)(*a.nactive) * ncols;
  const long long first = (long long)blockIdx.x * G + g, stride = (long long)gridDim.x * G;
  SusCursor cur{0, 0};
  if (producer) {
#pragma unroll 1
    for (int n = 0; n < S; ++n)
      sus_issue<Q, DMAX, MARKOV>(a, cur, first, stride, ntask, lvl_begin, ncols, stg + n * Sh::STAGE_F, bars + n);
  }
  long long u = 0;  // units consumed
  for (long long n = 0;; ++n) {
    const long long task = first + n * stride;
    if (task >= ntask) break;
    const int fb = a.list[task / ncols];
    const int j = __ldg(a.c.level_cols + lvl_begin + (int)(task % ncols));
    const int e0 = __ldg(a.c.col_ptr + j), dv = __ldg(a.c.col_ptr + j + 1) - e0;
    const int nunits = dv > 0 ? dv : 1;
    const bool frozen = lane_frozen(a, fb, lane);
#pragma unroll 1
    for (int s = 0; s < nunits; ++s, ++u) {
      const int st = (int)(u % S);
      const float *in = stg + st * Sh::STAGE_F;
      if (dv > 0) {
        const int e = __ldg(a.c.col_edge + e0 + s);
        const int i = __ldg(a.c.edge_check + e);
        const int r0 = __ldg(a.c.row_ptr + i), d = __ldg(a.c.row_ptr + i + 1) - r0;
        const int pos = e - r0;
        const int z = a.z[((size_t)fb * M + i) * 32 + lane];
        mbar_wait(bars + st, (uint32_t)((u / S) & 1));
        double v[DO > 0 ? DO : 1][KR];
#pragma unroll
        for (int t = 0; t < DO; ++t) {
          if (t < d - 1) {
            const int ee = r0 + (t < pos ? t : t + 1);
            int bb[P];
            unpack_basis<P>(__ldg(a.c.edge_perm + ee), bb);
            const int rch = row_hi<P, LKR>(bb, c);
#pragma unroll
            for (int k = 0; k < KR; ++k) v[t][k] = (double)in[(t * Q + (rch ^ row_lo<P, LKR>(bb, k))) * 32 + lane];
            wht_bits<KR, 0, LKR>(v[t]);
          }
        }
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
        int bb[P];
        unpack_basis<P>(__ldg(a.c.edge_perm + e), bb);
        const int rch = row_hi<P, LKR>(bb, c);
        float *rdst = (a.rmsg && !frozen) ? a.rmsg + ((size_t)fb * E + e0 + s) * Q * 32 + lane : nullptr;
#pragma unroll
        for (int k = 0; k < KR; ++k) {
          const double x = acc[k] * (1.0 / Q);
          const float fv = (float)(x > 0.0 ? x : 0.0);
          const int row = rch ^ row_lo<P, LKR>(bb, k);  // a = h_e^-1 y
          rsm[((size_t)s * Q + row) * 32 + lane] = fv;
          if (rdst) rdst[row * 32] = fv;
        }
      } else {
        mbar_wait(bars + st, (uint32_t)((u / S) & 1));
      }
      if (s == nunits - 1) {
        // vertical update of column j from the fresh r's (SUS step 2)
        group_bar<T>(g);  // rsm complete
        double r[DVMAX][KR];
#pragma unroll
        for (int ss = 0; ss < DVMAX; ++ss)
          if (ss < dv)
#pragma unroll
            for (int k = 0; k < KR; ++k) r[ss][k] = (double)rsm[((size_t)ss * Q + c * KR + k) * 32 + lane];
        double pr[KR];
        prior_from<Q, KR, MARKOV>(a, j, c, lane, in + (size_t)DO * Q * 32, pr);
        vn_body<Q, KR, DVMAX, MARKOV>(a, fb, j, e0, dv, r, pr, red, g, c, lane, frozen);
      }
      group_bar<T>(g);  // stage st (and the transpose / reduction scratch) free
      if (producer)
        sus_issue<Q, DMAX, MARKOV>(a, cur, first, stride, ntask, lvl_begin, ncols, stg + st * Sh::STAGE_F,
                                   bars + st);
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

constexpr int kStagesCN = 4;
constexpr int kStagesVN = 4;
constexpr int kStagesSUS = 3;

static int too_big(const char *what) {
  set_error(std::string(what) + ": this (q, degree) combination does not fit in shared memory");
  return GFQ_EUNSUPPORTED;
}

template <int Q, int DM>
static int cn_launch(const WaveArgs &a, cudaStream_t s) {
  constexpr int KR = KRof<Q>::v, T = Q / KR, G = Gof<T>::v;
  using S1 = CNShape<Q, KR, DM, 1, G>;
  constexpr int NS = fit_stages(G * S1::STAGE_F * 4, G * (128 + S1::XP_D * 8), kStagesCN);
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
  constexpr int KR = KRof<Q>::v, T = Q / KR, G = Gof<T>::v;
  using S1 = VNShape<Q, KR, DV, MK, 1, G>;
  constexpr int NS = fit_stages(G * S1::STAGE_F * 4, G * (128 + S1::RED_D * 8), kStagesVN);
  using Sh = VNShape<Q, KR, DV, MK, NS, G>;
  if (Sh::SMEM > 232448) return too_big("k_vn");
  auto k = k_vn<Q, KR, DV, MK, NS, G>;
  const int grid = grid_for(k, Sh::THREADS, Sh::SMEM, ((long long)a.nfb * a.c.V + G - 1) / G);
  k<<<grid, Sh::THREADS, Sh::SMEM, s>>>(a, clip);
  return check_launch("k_vn");
}

template <int Q>
static int vn_q(const WaveArgs &a, int clip, cudaStream_t s) {
  const bool small = a.c.max_vdeg <= 4;
  if (a.markov) return small ? vn_launch<Q, 4, true>(a, clip, s) : vn_launch<Q, 8, true>(a, clip, s);
  return small ? vn_launch<Q, 4, false>(a, clip, s) : vn_launch<Q, 8, false>(a, clip, s);
}

template <int Q, int DM, int DV, bool MK>
static int sus_launch(const WaveArgs &a, int lb, int ncols, cudaStream_t s) {
  constexpr int KR = KRof<Q>::v, T = Q / KR, G = Gof<T>::v;
  using S1 = SUSShape<Q, KR, DM, DV, MK, 1, G>;
  constexpr int NS = fit_stages(G * S1::STAGE_F * 4, S1::SMEM - G * S1::STAGE_F * 4, kStagesSUS);
  using Sh = SUSShape<Q, KR, DM, DV, MK, NS, G>;
  if (Sh::SMEM > 232448) return too_big("k_sus");
  auto k = k_sus<Q, KR, DM, DV, MK, NS, G>;
  const int grid = grid_for(k, Sh::THREADS, Sh::SMEM, ((long long)a.nfb * ncols + G - 1) / G);
  k<<<grid, Sh::THREADS, Sh::SMEM, s>>>(a, lb, ncols);
  return check_launch("k_sus");
}

template <int Q>
static int sus_q(const WaveArgs &a, int lb, int ncols, cudaStream_t s) {
  const bool small = a.c.max_cdeg <= 4 && a.c.max_vdeg <= 4;
  if (a.markov)
    return small ? sus_launch<Q, 4, 4, true>(a, lb, ncols, s) : sus_launch<Q, 8, 8, true>(a, lb, ncols, s);
  return small ? sus_launch<Q, 4, 4, false>(a, lb, ncols, s) : sus_launch<Q, 8, 8, false>(a, lb, ncols, s);
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

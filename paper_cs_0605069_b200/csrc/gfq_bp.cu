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
#define GFQ_KR_VN16 8
#endif
#ifndef GFQ_KR_SUS16
#define GFQ_KR_SUS16 8
#endif
#ifndef GFQ_ONEBAR_TMAX
#define GFQ_ONEBAR_TMAX 4  // SUS variable-node reduction in one barrier up to this group size
#endif
enum KernelKind { KCN, KVN, KSUS };
#ifndef GFQ_KR64
#define GFQ_KR64 8
#endif
template <int Q, int K>
struct KRof {
  static constexpr int v = Q <= 8 ? Q
                           : Q == 16 ? (K == KCN ? GFQ_KR_CN16 : K == KVN ? GFQ_KR_VN16 : GFQ_KR_SUS16)
                           : Q == 64 ? GFQ_KR64
                           : Q == 128 ? 16   // KR^2 >= Q: the two register layouts cover every bit
                                     : 8;
};
// largest stage count in [2, max_s] such that the CTA fits the 227 KB of
// dynamic shared memory (per_stage and other are bytes per CTA)
constexpr int fit_stages(size_t per_stage, size_t other, int max_s) {
  return (other + (size_t)max_s * per_stage <= 232448 || max_s <= 2) ? max_s
                                                                     : fit_stages(per_stage, other, max_s - 1);
}

// groups per CTA for a given number of warps per group
// dedicated producer warp (small q: short tasks) vs one producer lane per
// group (q = 64: keeps the CTA at 16 warps and 128 registers per thread)
#ifndef GFQ_PW_T2
#define GFQ_PW_T2 1
#endif
#ifndef GFQ_PW_T4
#define GFQ_PW_T4 1
#endif
template <int T>
struct PWof {
  static constexpr bool v = ((T == 2 && GFQ_PW_T2) || (T == 4 && GFQ_PW_T4));  // measured: in-group producers win for T = 1, 8
};
#ifndef GFQ_G_T8_CN
#define GFQ_G_T8_CN 2
#endif
#ifndef GFQ_G_T8_VN
#define GFQ_G_T8_VN 2
#endif
#ifndef GFQ_G_T8_SUS
#define GFQ_G_T8_SUS 2
#endif
// q = 128 (KR = 16, T = 8): one group per CTA so that a thread may use up to
// 255 registers (16 fp64 entries of up to 4 messages)
template <int T, int K = 0>
struct Gof {
  static constexpr int g8 = K == KCN ? GFQ_G_T8_CN : K == KVN ? GFQ_G_T8_VN : GFQ_G_T8_SUS;
  static constexpr int v = T >= 8 ? g8 : (T >= 2 ? 2 : 4);
};
template <int Q, int T, int K>
struct GQof {
  static constexpr int v = Q >= 128 ? 1 : Gof<T, K>::v;
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
// One-sided group barrier on a second id per group (15 - g; ids 1..G are the
// group_bar ones): warp `waiter` waits until every other warp of the group has
// arrived; the others only arrive and run on.  Safe to reuse because every
// waiter passes a full group_bar before the next round of arrivals.
template <int T>
__device__ __forceinline__ void group_gather(int g, bool waiter) {
  if constexpr (T > 1) {
    if (waiter)
      asm volatile("bar.sync %0, %1;" ::"r"(15 - g), "r"(T * 32) : "memory");
    else
      asm volatile("bar.arrive %0, %1;" ::"r"(15 - g), "r"(T * 32) : "memory");
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

// 1/x for a positive normal double: hardware approximation (rcp.approx.ftz.f64)
// refined by two Newton steps (relative error far below the fp32 storage of
// the normalised message).
__device__ __forceinline__ double fast_rcp(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

// Flip the sign of a double by XOR-ing its high word with a 0 / 0x80000000 mask.
__device__ __forceinline__ double flip(double v, uint32_t m) {
  const int lo = __double2loint(v), hi = __double2hiint(v);
  return __hiloint2double(hi ^ (int)m, lo);
}

// Early exit freezes a converged frame: its lane keeps computing (warp-uniform
// control flow) but stores nothing.  Invalid lanes of a ragged last block are
// marked converged from the start.

// ============================================================== PTX: more mbarrier / shared access
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
__device__ __forceinline__ float lds_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
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
// mbarrier arrive) followed by TMA-fetched metadata:
//   [0,64) TaskInfo  [128,256) CheckDesc | SusDesc(128..192) + VarDesc(192..256)
//   [256,288) syndrome row z (u8 x 32)   [384,512) frame-state row (int x 32)
struct __align__(16) TaskInfo {
  int fb, item, e0, deg;  // block, check/variable, first edge, degree
  int s, r0, d, pos;      // SUS unit: check slot, check row start / degree, position of e
  int i, pad0, pad1, pad2;
};
constexpr int kHdr = 512;

// Rows of one message of a thread in layout A: y = c*KR + k, k < KR.  With the
// message slot aligned to q*128 bytes in shared memory, the byte address of
// row (h^-1 y) is  base ^ (h^-1 y)*128  (XOR == ADD, no carries), and h^-1 y
// = h^-1(c*KR) ^ h^-1(k): one LOP3 per entry.
template <int P, int LKR, int KR>
__device__ __forceinline__ void perm_addrs(uint32_t base, unsigned long long pk, int c, uint32_t (&ad)[KR],
                                           int &rows_hi) {
  int bb[P];
  unpack_basis<P>(pk, bb);
  const int rh = row_hi<P, LKR>(bb, c);
  rows_hi = rh;
  const uint32_t b0 = base ^ ((uint32_t)rh << 7);
#pragma unroll
  for (int k = 0; k < KR; ++k) ad[k] = b0 ^ ((uint32_t)row_lo<P, LKR>(bb, k) << 7);
}

// The same addresses from the per-field table rowtab[a][y] = (a*y) << 7 (a =
// h^-1, the low byte of the packed basis): one uniform 2*KR-byte load (L1
// broadcast) and one add per entry.
template <int Q, int KR>
__device__ __forceinline__ void tab_addrs(uint32_t base, const unsigned short *rowtab, unsigned long long pk, int c,
                                          uint32_t (&ad)[KR]) {
  static_assert(KR == 2 || KR == 4 || KR == 8 || KR == 16, "tab_addrs: KR");
  const unsigned short *p = rowtab + (size_t)(pk & 0xff) * Q + c * KR;
  uint32_t w[KR / 2];
  if constexpr (KR == 16) {
    const uint4 v = __ldg((const uint4 *)p), u = __ldg((const uint4 *)p + 1);
    w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
    w[4] = u.x; w[5] = u.y; w[6] = u.z; w[7] = u.w;
  } else if constexpr (KR == 8) {
    const uint4 v = __ldg((const uint4 *)p);
    w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
  } else if constexpr (KR == 4) {
    const uint2 v = __ldg((const uint2 *)p);
    w[0] = v.x; w[1] = v.y;
  } else {
    w[0] = __ldg((const unsigned int *)p);
  }
#pragma unroll
  for (int k = 0; k < KR; ++k) ad[k] = base + ((k & 1) ? (w[k >> 1] >> 16) : (w[k >> 1] & 0xffffu));
}

// The same from a shared-memory copy of the table (rt = its shared address).
template <int Q, int KR>
__device__ __forceinline__ void tab_addrs_sm(uint32_t base, uint32_t rt, unsigned long long pk, int c,
                                             uint32_t (&ad)[KR]) {
  static_assert(KR == 2 || KR == 4 || KR == 8 || KR == 16, "tab_addrs_sm: KR");
  const uint32_t p = rt + (uint32_t)(((size_t)(pk & 0xff) * Q + c * KR) * 2);
  uint32_t w[KR >= 8 ? KR / 2 : 4];
  if constexpr (KR == 16) {
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]) : "r"(p));
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]) : "r"(p + 16));
  } else if constexpr (KR == 8) {
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]) : "r"(p));
  } else if constexpr (KR == 4) {
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(w[0]), "=r"(w[1]) : "r"(p));
  } else {
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w[0]) : "r"(p));
  }
#pragma unroll
  for (int k = 0; k < KR; ++k) ad[k] = base + ((k & 1) ? (w[k >> 1] >> 16) : (w[k >> 1] & 0xffffu));
}

// ============================================================== leave-one-out with the syndrome sign
// out_s = sign * prod_{s' != s} u_s'   for exact degree D (sign folded in as an
// XOR of the high word: the same sign multiplies every output at frequency w).
template <int D, int KR, int DM>
__device__ __forceinline__ void loo_signed(double (&u)[DM][KR], const uint32_t (&sm)[KR]) {
#pragma unroll
  for (int k = 0; k < KR; ++k) {
    const uint32_t s = sm[k];
    if constexpr (D == 1) {
      u[0][k] = flip(1.0, s);
    } else if constexpr (D == 2) {
      const double t = u[0][k];
      u[0][k] = flip(u[1][k], s);
      u[1][k] = flip(t, s);
    } else if constexpr (D == 3) {
      const double a = u[0][k], b = u[1][k], cs = flip(u[2][k], s);
      u[0][k] = b * cs;
      u[1][k] = a * cs;
      u[2][k] = flip(a * b, s);
    } else if constexpr (D == 4) {
      const double ab = flip(u[0][k] * u[1][k], s), cd = flip(u[2][k] * u[3][k], s);
      const double n0 = u[1][k] * cd, n1 = u[0][k] * cd;
      const double n2 = ab * u[3][k], n3 = ab * u[2][k];
      u[0][k] = n0; u[1][k] = n1; u[2][k] = n2; u[3][k] = n3;
    } else {
      double pre[D];
      double acc = 1.0;
#pragma unroll
      for (int t = 0; t < D; ++t) {
        pre[t] = acc;
        acc *= u[t][k];
      }
      acc = 1.0;
#pragma unroll
      for (int t = D - 1; t >= 0; --t) {
        const double o = u[t][k];
        u[t][k] = flip(pre[t] * acc, s);
        acc *= o;
      }
    }
  }
}

// Sign masks of the syndrome shift: bit 31 set where (-1)^{popc(w & z)} = -1,
// w = k*T + c (layout B) or k (T = 1).
template <int KR, int T>
__device__ __forceinline__ void sign_masks(int z, int c, uint32_t (&sm)[KR]) {
  constexpr int LT = ilog2(T);
  const int zk = z >> LT;
  const uint32_t base = (T > 1) ? ((uint32_t)(__popc(z & c & (T - 1)) & 1) << 31) : 0u;
#pragma unroll
  for (int k = 0; k < KR; ++k) sm[k] = base ^ ((uint32_t)(__popc(zk & k) & 1) << 31);
}

// ============================================================== priors
template <int Q, bool MARKOV>
struct Extra {
  static constexpr int P = ilog2(Q);
  static constexpr int rows = MARKOV ? (2 * Q > P ? 2 * Q : P) : P;
};

// Which Markov neighbour posteriors source column j reads (bit 0: j-1, bit 1:
// j+1), and from where: snapshot mode (A9) both from Q^(t-1) (qs_old) from
// iteration 2 on; in-sweep mode (A34) j-1 from this sweep (qs_new, written by
// an earlier level) and j+1 from the previous sweep (qs_old, none in sweep 1).
__device__ __forceinline__ int markov_nbrs(const WaveArgs &a, int j) {
  const int N = a.c.N;
  if (a.qs_old == nullptr) return 0;
  if (a.gs) return (j > 0 ? 1 : 0) | ((a.t > 1 && j < N - 1) ? 2 : 0);
  if (a.t <= 1) return 0;
  return (j > 0 ? 1 : 0) | (j < N - 1 ? 2 : 0);
}

template <int Q, bool MARKOV>
__device__ __forceinline__ uint32_t extras_bytes(const WaveArgs &a, int j) {
  constexpr int P = ilog2(Q);
  const int N = a.c.N;
  if (j >= N) return P * 128;
  if (MARKOV) {
    const int nb = markov_nbrs(a, j);
    return (uint32_t)((nb & 1) + (nb >> 1)) * Q * 128;
  }
  return 0;
}

// noise symbol -> its p per-bit flip probabilities (slot 0); Markov source
// symbol -> posteriors of j-1 (slot 0) and j+1 (slot 1) as markov_nbrs says
template <int Q, bool MARKOV>
__device__ __forceinline__ void issue_extras(const WaveArgs &a, int fb, int j, unsigned char *dst, uint64_t *bar) {
  constexpr int P = ilog2(Q);
  const int N = a.c.N;
  if (j >= N) {
    bulk_g2s(dst, a.pi + ((size_t)fb * a.c.M * P + (size_t)(j - N) * P) * 32, P * 128, bar);
  } else if (MARKOV) {
    const int nb = markov_nbrs(a, j);
    const float *left = a.gs ? a.qs_new : a.qs_old;
    if (nb & 1) bulk_g2s(dst, left + ((size_t)fb * N + (j - 1)) * Q * 32, Q * 128, bar);
    if (nb & 2) bulk_g2s(dst + Q * 128, a.qs_old + ((size_t)fb * N + (j + 1)) * Q * 32, Q * 128, bar);
  }
}

// Prior p_j^a for the KR entries a = c*KR + k (layout A) of this thread:
//  - noise symbol j = N + m: prod_b (bit_b(a) ? pi_b : 1 - pi_b),
//    built as a tensor product over the low bits;
//  - source symbol, i.i.d. or first iteration: pi0(a)
//  - source symbol, Markov, iteration t >= 2: Eq. (7) from the
//    posterior snapshot Q^(t-1) of the neighbours (reading A9), boundaries A10:
//      p(b) = [sum_a Q_{j-1}(a) T_ab] * [sum_c T_bc Q_{j+1}(c)]
//  - SUS with the in-sweep prior (reading A34): the same formula
//    with Q_{j-1} of this sweep and Q_{j+1} of the previous one (markov_nbrs);
//    a missing neighbour gives the factor pi0(b) (left) or 1 (right)
template <int Q, int KR, bool MARKOV>
__device__ __forceinline__ void prior_from(const WaveArgs &a, int j, int c, int lane, const float *ex,
                                           const float *Tsm, double (&pr)[KR]) {
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
    pr[0] = hi;
#pragma unroll
    for (int b = 0; b < LKR; ++b) {
      const double one = 1.0 - pb[b];
#pragma unroll
      for (int k = 0; k < (1 << b); ++k) {
        pr[k | (1 << b)] = pr[k] * pb[b];
        pr[k] = pr[k] * one;
      }
    }
    return;
  }
  const int nb = MARKOV ? markov_nbrs(a, j) : 0;
  if (nb == 0) {
#pragma unroll
    for (int k = 0; k < KR; ++k) pr[k] = __ldg(a.pi0 + c * KR + k);
    return;
  }
  // Eq. (7) factors accumulated in fp32 (all terms >= 0: no cancellation) from
  // the fp32 snapshots, with T and T^T staged in shared memory (Ts): each
  // thread reads its KR consecutive columns with 128-bit loads.
  const float *Ts = Tsm;            // T[a][b]
  const float *Tt = Tsm + Q * Q;    // T^T[c][b] = T[b][c]
  float L[KR], R[KR];
  const float *exl = ex;           // rows of j-1 (issue_extras: slot 0)
  const float *exr = ex + Q * 32;  // rows of j+1 (slot 1)
#pragma unroll
  for (int k = 0; k < KR; ++k) { L[k] = 0.0f; R[k] = 0.0f; }
  if (a.tj) {
    // T = alpha I + beta 1 1^T (stay / uniform jump, readings A12): the same
    // sums in O(q) -- sum_x Q(x) T[x][b] = beta sum_x Q(x) + alpha Q(b), and
    // sum_c T[b][c] Q(c) likewise (T symmetric)
    const float al = a.tj_alpha, be = a.tj_beta;
    if (nb & 1) {
      float sl = 0.0f;
#pragma unroll 8
      for (int x = 0; x < Q; ++x) sl += exl[x * 32 + lane];
#pragma unroll
      for (int k = 0; k < KR; ++k) L[k] = fmaf(al, exl[(c * KR + k) * 32 + lane], be * sl);
    }
    if (nb & 2) {
      float sr = 0.0f;
#pragma unroll 8
      for (int x = 0; x < Q; ++x) sr += exr[x * 32 + lane];
#pragma unroll
      for (int k = 0; k < KR; ++k) R[k] = fmaf(al, exr[(c * KR + k) * 32 + lane], be * sr);
    }
  } else {
  if (nb & 1) {
#pragma unroll 4
    for (int x = 0; x < Q; ++x) {
      const float qv = exl[x * 32 + lane];
      const float *trow = Ts + x * Q + c * KR;
#pragma unroll
      for (int k = 0; k < KR; ++k) L[k] = fmaf(qv, trow[k], L[k]);
    }
  }
  if (nb & 2) {
#pragma unroll 4
    for (int x = 0; x < Q; ++x) {
      const float qv = exr[x * 32 + lane];
      const float *trow = Tt + x * Q + c * KR;
#pragma unroll
      for (int k = 0; k < KR; ++k) R[k] = fmaf(qv, trow[k], R[k]);
    }
  }
  }
#pragma unroll
  for (int k = 0; k < KR; ++k) {
    const double l = (nb & 1) ? (double)L[k] : __ldg(a.pi0 + c * KR + k);
    const double r = (nb & 2) ? (double)R[k] : 1.0;
    pr[k] = l * r;
  }
}

// ============================================================== variable node
// Eq. (4): q_ij^a = alpha_ij p_j^a prod_{i' != i} r_i'j^a, and
// Eq. (5): Q_j^a = alpha_j p_j^a prod_i r_ij^a, clipped to the
// smallest a within kTieRel of the maximum (reading A17).  Exact degree DV;
// r[s][k] holds r of check slot s at a = c*KR + k (any positive scale: every
// output is normalised); pr the prior; qdst[s] the check-major id of the edge
// of slot s.  red: group scratch of (DV+2)*T*32 doubles (T > 1).
// ONEBAR (T <= 4, red private to the task): one barrier, every warp sums the
// T partials itself (the two-step reduction needs two).
template <int Q, int KR, int DV, bool MARKOV, bool ONEBAR = false>
__device__ __forceinline__ void vn_core(const WaveArgs &a, int fb, int j, const int *qdst, double (&r)[DV > 0 ? DV : 1][KR],
                                        const double (&pr)[KR], double *red, int g, int c, int lane, bool frozen) {
  constexpr int T = Q / KR;
  constexpr int NS = DV + 1;  // sums: DV outgoing messages + the posterior
  const long long E = a.c.E;
  double tot[KR];
  // products (leave-one-out per exact degree), in place: r[s] <- p * prod_{s' != s} r_s'
#pragma unroll
  for (int k = 0; k < KR; ++k) {
    if constexpr (DV == 0) {
      tot[k] = pr[k];
    } else if constexpr (DV == 1) {
      tot[k] = pr[k] * r[0][k];
      r[0][k] = pr[k];
    } else if constexpr (DV == 2) {
      const double q0 = pr[k] * r[1][k], q1 = pr[k] * r[0][k];
      tot[k] = q0 * r[0][k];
      r[0][k] = q0;
      r[1][k] = q1;
    } else if constexpr (DV == 3) {
      const double x = pr[k] * r[0][k], bc = r[1][k] * r[2][k];
      const double q0 = pr[k] * bc, q1 = x * r[2][k], q2 = x * r[1][k];
      tot[k] = x * bc;
      r[0][k] = q0; r[1][k] = q1; r[2][k] = q2;
    } else {
      double pre[DV];
      double acc = pr[k];
#pragma unroll
      for (int s = 0; s < DV; ++s) {
        pre[s] = acc;
        acc *= r[s][k];
      }
      tot[k] = acc;
      acc = 1.0;
#pragma unroll
      for (int s = DV - 1; s >= 0; --s) {
        const double o = r[s][k];
        r[s][k] = pre[s] * acc;
        acc *= o;
      }
    }
  }
  double sums[NS];
  double mx = tot[0];
#pragma unroll
  for (int s = 0; s < NS; ++s) sums[s] = 0.0;
#pragma unroll
  for (int k = 0; k < KR; ++k) {
#pragma unroll
    for (int s = 0; s < DV; ++s) sums[s] += r[s][k];
    sums[DV] += tot[k];
    if (k > 0) mx = fmax(mx, tot[k]);
  }
  if constexpr (T > 1 && ONEBAR) {
#pragma unroll
    for (int s = 0; s < NS; ++s) red[((size_t)s * T + c) * 32 + lane] = sums[s];
    red[((size_t)NS * T + c) * 32 + lane] = mx;
    group_bar<T>(g);
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      double v = red[((size_t)s * T) * 32 + lane];
#pragma unroll
      for (int cc = 1; cc < T; ++cc) v += red[((size_t)s * T + cc) * 32 + lane];
      sums[s] = v;
    }
    mx = red[((size_t)NS * T) * 32 + lane];
#pragma unroll
    for (int cc = 1; cc < T; ++cc) mx = fmax(mx, red[((size_t)NS * T + cc) * 32 + lane]);
  } else if constexpr (T > 1) {
    // two-step cross-warp reduction: partials -> warp v reduces value v -> totals
#pragma unroll
    for (int s = 0; s < NS; ++s) red[((size_t)s * T + c) * 32 + lane] = sums[s];
    red[((size_t)NS * T + c) * 32 + lane] = mx;
    group_bar<T>(g);
    double *tot_s = red + (size_t)(NS + 1) * T * 32;
#pragma unroll 1
    for (int vi = c; vi <= NS; vi += T) {
      double v = red[((size_t)vi * T) * 32 + lane];
#pragma unroll
      for (int cc = 1; cc < T; ++cc) {
        const double w = red[((size_t)vi * T + cc) * 32 + lane];
        v = (vi == NS) ? fmax(v, w) : v + w;
      }
      tot_s[vi * 32 + lane] = v;
    }
    group_bar<T>(g);
#pragma unroll
    for (int s = 0; s < NS; ++s) sums[s] = tot_s[s * 32 + lane];
    mx = tot_s[NS * 32 + lane];
  }
  // Clipping: the smallest a whose Q is within kTieRel of the maximum.
  const double thr = mx * (1.0 - kTieRel);
  int bidx = Q;
#pragma unroll
  for (int k = KR - 1; k >= 0; --k)
    if (tot[k] >= thr) bidx = c * KR + k;
  if constexpr (T > 1) {
    // only warp 0 needs the index (it writes the estimate): the others arrive and go on
    int *ired = (int *)(red + (size_t)(NS + 1) * T * 32 + (size_t)(NS + 1) * 32);
    ired[c * 32 + lane] = bidx;
    group_gather<T>(g, c == 0);
    if (c == 0) {
#pragma unroll
      for (int cc = 1; cc < T; ++cc) bidx = min(bidx, ired[cc * 32 + lane]);
    }
  }
  if (bidx >= Q) bidx = 0;
  int bad = 0;
#pragma unroll
  for (int s = 0; s < DV; ++s) {
    const double sm = sums[s];
    const bool ok = sm > 0.0 && isfinite(sm);
    bad += !ok;
    const double inv = ok ? fast_rcp(sm) : 0.0;
    const float add = ok ? 0.0f : 1.0f / Q;
    if (!frozen) {
      float *dst = a.qmsg + ((size_t)fb * E + qdst[s]) * Q * 32 + lane + c * KR * 32;
#pragma unroll
      for (int k = 0; k < KR; ++k) dst[k * 32] = (float)(r[s][k] * inv) + add;
    }
  }
  const double st = sums[DV];
  const bool okq = st > 0.0 && isfinite(st);
  bad += !okq;
  if (!okq) bidx = 0;
  const double invq = okq ? fast_rcp(st) : 0.0;
  const float addq = okq ? 0.0f : 1.0f / Q;
  if (!frozen) {
    if (MARKOV && j < a.c.N && a.qs_new) {
      float *dst = a.qs_new + ((size_t)fb * a.c.N + j) * Q * 32 + lane + c * KR * 32;
#pragma unroll
      for (int k = 0; k < KR; ++k) dst[k * 32] = (float)(tot[k] * invq) + addq;
    }
    if (a.qall) {
      float *dst = a.qall + ((size_t)fb * a.c.V + j) * Q * 32 + lane + c * KR * 32;
#pragma unroll
      for (int k = 0; k < KR; ++k) dst[k * 32] = (float)(tot[k] * invq) + addq;
    }
    if (c == 0) a.xhat[((size_t)fb * a.c.V + j) * 32 + lane] = (unsigned char)bidx;
    if (bad && c == 0) atomicAdd(a.stats + 0, (unsigned long long)bad);
  }
}


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

// ============================================================== shared-memory layout
// [mbarriers][G*S headers of kHdr][pad][G*S payload slots, each a multiple of
// PAL = q*128 bytes and PAL-aligned in the shared window][G scratch areas]
// ALIGN: payload slots aligned to q*128 bytes (needed by the XOR row addressing
// of perm_addrs, i.e. the check-node kernel); the variable-node and SUS kernels
// address rows by addition and only need 128-byte alignment.
template <int Q, int S, int G, size_t PAY, size_t SCR, size_t XTRA = 0, size_t TSMB = 0, bool ALIGN = true>
struct Shape {
  static constexpr size_t TSM_B = ((TSMB + 127) / 128) * 128;
  static constexpr size_t PAL = ALIGN ? (size_t)Q * 128 : 128;
  static constexpr size_t PAYA = ((PAY + PAL - 1) / PAL) * PAL;
  static constexpr size_t BARS_B = ((16 * S * G + 127) / 128) * 128;
  static constexpr size_t HDR_B = (size_t)G * S * kHdr;
  static constexpr size_t XTRA_A = ((XTRA + 127) / 128) * 128;
  static constexpr size_t XTRA_B = (size_t)G * S * XTRA_A;
  static constexpr size_t SMEM = BARS_B + HDR_B + XTRA_B + TSM_B + PAL + (size_t)G * S * PAYA + (size_t)G * SCR;
};

struct SmemPtrs {
  uint64_t *bars;
  unsigned char *hdr;
  unsigned char *xtra;
  float *tsm;
  unsigned char *pay;
  uint32_t pay_u32;
  unsigned char *scr;
};

template <typename Sh, int S, int G>
__device__ __forceinline__ SmemPtrs smem_ptrs(unsigned char *smem) {
  SmemPtrs p;
  p.bars = (uint64_t *)smem;
  p.hdr = smem + Sh::BARS_B;
  p.xtra = p.hdr + Sh::HDR_B;
  p.tsm = (float *)(p.xtra + Sh::XTRA_B);
  const uint32_t base = smem_u32(smem);
  const uint32_t want = base + (uint32_t)(Sh::BARS_B + Sh::HDR_B + Sh::XTRA_B + Sh::TSM_B);
  const uint32_t al = (uint32_t)(((want + Sh::PAL - 1) / Sh::PAL) * Sh::PAL);
  p.pay = smem + (al - base);
  p.pay_u32 = al;
  p.scr = p.pay + (size_t)G * S * Sh::PAYA;
  return p;
}

template <int S, int G>
__device__ __forceinline__ void init_bars(uint64_t *bars, int T) {
  // bars[0 .. G*S): full (1 arrival + tx bytes), bars[G*S .. 2*G*S): empty (T arrivals)
  for (int k = 0; k < G * S; ++k) {
    mbar_init(bars + k, 1);
    mbar_init(bars + G * S + k, (uint32_t)T);
  }
  fence_mbar_init();
}

// Walk over a contiguous range of tasks (frame block, item) without 64-bit
// divisions per task: the block index and item advance incrementally.
struct Cursor {
  long long t, hi;
  int fbi, item, fb, nitems;
  __device__ __forceinline__ void init(const WaveArgs &a, long long t0, long long hi_, int nitems_) {
    t = t0;
    hi = hi_;
    nitems = nitems_;
    fbi = item = fb = 0;
    if (t < hi) {
      fbi = (int)(t / nitems);
      item = (int)(t - (long long)fbi * nitems);
      fb = a.list[fbi];
    }
  }
  __device__ __forceinline__ bool valid() const { return t < hi; }
  __device__ __forceinline__ void advance(const WaveArgs &a) {
    ++t;
    if (++item == nitems) {
      item = 0;
      ++fbi;
      if (t < hi) fb = a.list[fbi];
    }
  }
};

// Dedicated producer (lane 0 of warp 0): walks every consumer group's
// contiguous share of tasks round-robin, refilling a stage as soon as its
// "empty" barrier flips.  issue(g, st, cursor) returns true when the task is
// complete (SUS tasks span several stages).
template <int S, int G, typename Issue>
__device__ __forceinline__ void produce(const WaveArgs &a, uint64_t *bars, long long ntask, int nitems,
                                        Issue issue) {
  const long long ngroups = (long long)gridDim.x * G;
  Cursor cur[G];
  int ring[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    long long lo, hi;
    group_range(ntask, (long long)blockIdx.x * G + g, ngroups, lo, hi);
    cur[g].init(a, lo, hi, nitems);
    ring[g] = 0;
  }
  for (bool any = true; any;) {
    any = false;
    bool did = false;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      if (!cur[g].valid()) continue;
      any = true;
      const int st = ring[g] % S, u = ring[g] / S;
      if (u > 0) {
        uint64_t *empty = bars + G * S + g * S + st;
        if (G == 1) {
          mbar_wait(empty, (u - 1) & 1);  // hardware-suspended wait
        } else if (!mbar_test(empty, (u - 1) & 1)) {
          continue;
        }
      }
      if (issue(g, st, cur[g])) cur[g].advance(a);
      ++ring[g];
      did = true;
    }
    if (!did && any) __nanosleep(64);  // leave the issue slots to the consumers
  }
}

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
                                         uint64_t *full) {
  const int M = a.c.M;
  const int e0 = __ldg(a.c.row_ptr + i), d = __ldg(a.c.row_ptr + i + 1) - e0;
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
    for (int n = 0; n < S && pc.valid(); ++n, pc.advance(a)) {
      const int k = g * S + n;
      cn_issue<Q, DMAX>(a, pc.fb, pc.item, sp.hdr + (size_t)k * kHdr, sp.pay + (size_t)k * Sh::PAYA, sp.bars + k);
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
                                         unsigned char *xtra, uint64_t *full, int clip_only) {
  const int e0 = __ldg(a.c.col_ptr + j);
  const int dv = clip_only ? 0 : __ldg(a.c.col_ptr + j + 1) - e0;
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
      });
    return;
  }
  const int cw = PW ? warp - 1 : warp;
  const int g = cw / T, c = cw % T;
  const bool producer = !PW && (c == 0) && (lane == 0);
  double *red = (double *)(sp.scr + (size_t)g * VS::SCR);
  long long lo, hi;
  group_range(ntask, (long long)blockIdx.x * G + g, (long long)gridDim.x * G, lo, hi);
  Cursor pc;
  if (producer) {
    pc.init(a, lo, hi, V);
    for (int n = 0; n < S && pc.valid(); ++n, pc.advance(a)) {
      const int k = g * S + n;
      vn_issue<Q, DVMAX, MARKOV>(a, pc.fb, pc.item, sp.hdr + (size_t)k * kHdr, sp.pay + (size_t)k * Sh::PAYA,
                                 sp.xtra + (size_t)k * Sh::XTRA_A, sp.bars + k, clip_only);
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

// Units: one per (column, check slot) -- the check's other edges in at most
// two contiguous runs; the last unit of a column also carries the prior's
// extra rows and the column's VarDesc.
template <int Q, int DMAX, bool MARKOV>
__device__ __forceinline__ bool sus_issue(const WaveArgs &a, int fb, int col, int &s, int lvl_begin,
                                          unsigned char *hdr, unsigned char *pay, unsigned char *xtra,
                                          uint64_t *full) {
  const LvlCol lc = a.c.lvl_col[lvl_begin + col];
  const int nunits = lc.dv > 0 ? lc.dv : 1;
  const LvlUnit un = a.c.lvl_unit[lc.unit0 + s];
  TaskInfo *ti = (TaskInfo *)hdr;
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
    bulk_g2s(hdr + 128, a.c.sus_desc + lc.e0 + s, 64, full);
    bulk_g2s(hdr + 256, a.z + ((size_t)fb * a.c.M + un.i) * 32, 32, full);
  }
  if (a.early_exit) bulk_g2s(hdr + 384, a.conv + fb * 32, 128, full);
  if (b0) bulk_g2s(pay, rowbase, b0, full);
  if (b1) bulk_g2s(pay + (size_t)un.pos * Q * 128, rowbase + (size_t)(un.pos + 1) * Q * 32, b1, full);
  if (last) {
    bulk_g2s(hdr + 192, a.c.var_desc + lc.j, 64, full);
    issue_extras<Q, MARKOV>(a, fb, lc.j, xtra, full);
  }
  if (++s >= nunits) {
    s = 0;
    return true;  // task complete
  }
  return false;
}

// Step 1 of SUS for one check (exact number of other edges DO): r_ij from the
// CURRENT q's of the check's other edges (the transform of k_cn restricted to
// one output).  Writes q * r_ij into rsm slot s in natural order a.
template <int Q, int KR, int DO, int DMAX, typename RF>
__device__ __forceinline__ void sus_check(const WaveArgs &a, const unsigned char *hdr, uint32_t pay_u32,
                                          uint64_t *empty, bool release, double *xp, int &m, float *rsm, int g,
                                          int c, int lane, bool frozen, RF &&refill) {
  using C = QC<Q, KR>;
  constexpr int T = C::T, LKR = C::LKR, LT = C::LT, P = C::P;
  constexpr bool PP = PPof<Q>::v;
  const TaskInfo ti = *(const TaskInfo *)hdr;
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

template <int Q, int KR, int DO, bool RTS, typename RF>
__device__ __forceinline__ void sus_check_phased(const WaveArgs &a, const unsigned char *hdr, uint32_t pay_u32,
                                                 double *stage_x, uint64_t *empty, bool last, double *xp,
                                                 float *rsm, uint32_t rt, const unsigned short *rowtab,
                                                 int g, int c, int lane, bool frozen, RF &&refill) {
  using C = QC<Q, KR>;
  constexpr int T = C::T, LKR = C::LKR, LT = C::LT;
  static_assert(T > 1 && DO <= 3, "phased SUS check: q >= 16, degree <= 4");
  const TaskInfo ti = *(const TaskInfo *)hdr;
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
    uint32_t sm[KR];
    sign_masks<KR, T>(z, c, sm);
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      double x = v[0][k];
#pragma unroll
      for (int t = 1; t < DO; ++t) x *= v[t][k];
      acc[k] = flip(x, sm[k]);
    }
    wht_bits<KR, LKR - LT, LKR>(acc);
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

template <int Q, int KR, int DV, int DVMAX, bool MARKOV, bool ONEBAR, typename RF>
__device__ __forceinline__ void sus_vn(const WaveArgs &a, const unsigned char *hdr, const unsigned char *xtra,
                                       const float *Tsm, uint64_t *empty, const float *rsm, double *red, int g,
                                       int c, int lane, bool frozen, bool late_release, RF &&refill) {
  const TaskInfo ti = *(const TaskInfo *)hdr;
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
      });
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
  group_range(ntask, (long long)blockIdx.x * G + g, (long long)gridDim.x * G, lo, hi);
  // producer cursor over (task, unit) of this group
  Cursor pc;
  int pu = 0;
  if (producer) pc.init(a, lo, hi, ncols);
  auto issue_next = [&](int k) {
    if (!pc.valid()) return;
    if (sus_issue<Q, DMAX, MARKOV>(a, pc.fb, pc.item, pu, lvl_begin, sp.hdr + (size_t)k * kHdr,
                                   sp.pay + (size_t)k * Sh::PAYA, sp.xtra + (size_t)k * Sh::XTRA_A, sp.bars + k))
      pc.advance(a);
  };
  if (producer)
    for (int n = 0; n < S; ++n) issue_next(g * S + n);
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
        if (producer && pc.valid()) {
          mbar_wait(empty, (uint32_t)((rr / S) & 1));
          issue_next(k);
        }
      };
      mbar_wait(sp.bars + k, (uint32_t)((rr / S) & 1));
      const TaskInfo *ti = (const TaskInfo *)hdr;
      const int dv = ti->deg, d = ti->d;
      nunits = dv > 0 ? dv : 1;
      const bool last = (s == nunits - 1);
      const bool frozen = a.early_exit && ((const int *)(hdr + 384))[lane] != 0;
      double *stage_x = (double *)(sp.pay + (size_t)k * Sh::PAYA);
      if constexpr (SS::PHASED) {
        if (dv > 0) {
#define SP(n) sus_check_phased<Q, KR, n, SS::RTS>(a, hdr, pay_u32, stage_x, empty, last, xp, rsm, rt, a.c.rowtab, g, c, lane, frozen, refill)
          switch (d - 1) {
            case 0: SP(0); break;
            case 1: SP(1); break;
            case 2: SP(2); break;
            default: SP(3); break;
          }
#undef SP
        }
      } else if (dv > 0) {
#define SC(n) sus_check<Q, KR, n, DMAX>(a, hdr, pay_u32, empty, !last, xp, m, rsm, g, c, lane, frozen, refill)
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
#define SV(n) sus_vn<Q, KR, n, DVMAX, MARKOV, SS::PHASED && (T <= GFQ_ONEBAR_TMAX)>(a, hdr, xtra, Tp, empty, rsm, SS::PHASED ? stage_x : red, g, c, lane, frozen, SS::PHASED, refill)
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

// gfq_device.cuh -- device-side building blocks shared by the hot kernels
// (gfq_bp.cu: PUS check/variable node and the SUS level kernel with
// transform-domain check nodes; gfq_sus_dc.cu: the direct-convolution SUS
// kernel for q <= 16): configuration knobs, mbarrier / TMA bulk-copy PTX,
// GF(2^p) row addressing, priors, the variable node (Eqs. 4, 5),
// the shared-memory stage layout and the producer loop.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "gfq_internal.cuh"

namespace gfq {


// Relative tolerance under which two posterior values count as a tie in the
// clipping step (reading A17: ties -> smallest a).  It is the GPU's own
// round-off scale: posteriors are products of fp32-stored messages (a few
// fp32 ulps, ~1e-7 relative), so mathematically equal values (BEC coset
// ties) can differ by that much; 1e-6 keeps a 10x margin while resolving
// genuine near-ties above it as the strict argmax of the oracle does.
#ifndef GFQ_TIE_REL
#define GFQ_TIE_REL 1e-6
#endif
constexpr double kTieRel = GFQ_TIE_REL;

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
#ifndef GFQ_PW_T8
#define GFQ_PW_T8 0
#endif
template <int T>
struct PWof {
  static constexpr bool v = ((T == 2 && GFQ_PW_T2) || (T == 4 && GFQ_PW_T4) || (T == 8 && GFQ_PW_T8));  // measured: in-group producers win for T = 1, 8
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
// GFQ_SYNC_CHECK=1 builds the checking variant (libgfq_synccheck.so): a full
// group barrier at every point where the default build elides one (one-sided
// gathers, ping-pong and phased layout switches that reuse a buffer without a
// barrier, no barrier between tasks).  Its outputs must be bit-identical to
// the default build's (tests/test_gpu_sync_check.py) -- the race / sync check
// of the barrier-elided kernels, compute-sanitizer being closed on this pool.
#ifndef GFQ_SYNC_CHECK
#define GFQ_SYNC_CHECK 0
#endif
template <int T>
__device__ __forceinline__ void group_bar(int g);
template <int T>
__device__ __forceinline__ void elided_bar(int g) {
  if constexpr (GFQ_SYNC_CHECK != 0 && T > 1) group_bar<T>(g);
}

// One-sided group barrier on a second id per group (15 - g; ids 1..G are the
// group_bar ones): warp `waiter` waits until every other warp of the group has
// arrived; the others only arrive and run on.  Safe to reuse because every
// waiter passes a full group_bar before the next round of arrivals.
template <int T>
__device__ __forceinline__ void group_gather(int g, bool waiter) {
  if constexpr (T > 1) {
    if (GFQ_SYNC_CHECK != 0 || waiter)
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

constexpr long long kBalanceMinTasks = 1 << 16;   // below this a launch is too short to pay for the searches

// SUS: the share of global group gg of the (frame block, column) tasks of one
// level, balanced by UNITS (a column of degree dv is dv units of work: source
// columns have 3, noise columns 2, and a level lists its source columns first,
// so a split by columns gave some groups 1.5x the work of others -- 12 % of the
// warp slots of k_sus_dc idle at C4, profiles/r02).  Boundaries stay at column
// starts: lo / hi = the first task whose first unit is at or after the group's
// share of the nblk * U unit positions (U = units of the level).
__device__ __forceinline__ long long sus_task_at(const LvlCol *lc, int ncols, int U, int u_first, long long nblk,
                                                 long long p) {
  if (p >= nblk * U) return nblk * ncols;
  const long long fbi = p / U;
  const int r = (int)(p - fbi * U);
  int lo = 0, hi = ncols;   // first column whose unit offset is >= r
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (lc[mid].unit0 - u_first >= r) hi = mid; else lo = mid + 1;
  }
  return fbi * ncols + lo;
}
__device__ __forceinline__ void sus_group_range(const WaveArgs &a, int lvl_begin, int ncols, long long nblk,
                                                long long gg, long long ngroups, long long &lo, long long &hi) {
  // small launches: the binary searches (dependent L2 loads) would cost more
  // than the imbalance; the plain split by columns is exact enough
  if (nblk * ncols < kBalanceMinTasks) {
    group_range(nblk * ncols, gg, ngroups, lo, hi);
    return;
  }
  const LvlCol *lc = a.c.lvl_col + lvl_begin;
  const int u_first = lc[0].unit0;
  const LvlCol last = lc[ncols - 1];
  const int U = last.unit0 + (last.dv > 0 ? last.dv : 1) - u_first;
  const long long total = nblk * U;
  const long long chunk = (total + ngroups - 1) / ngroups;
  lo = sus_task_at(lc, ncols, U, u_first, nblk, gg * chunk);
  hi = sus_task_at(lc, ncols, U, u_first, nblk, (gg + 1) * chunk);
}

// PUS variable node: the same balancing by work for the (block, variable)
// tasks -- a variable of degree dv moves 2 dv q-vectors, and the source
// variables (degree 3, plus the Markov prior) come before the noise variables
// (degree 2).  Weight of variable j: dv_j + 1 (+ 2 for a Markov source
// variable's two neighbour rows); its offset is col_ptr[j] + j (+ 2 min(j, N)).
__device__ __forceinline__ long long vn_weight_off(const WaveArgs &a, int j) {
  return (long long)__ldg(a.c.col_ptr + j) + j + (a.markov ? 2 * (j < a.c.N ? j : a.c.N) : 0);
}
__device__ __forceinline__ long long vn_task_at(const WaveArgs &a, long long Wt, long long nblk, long long p) {
  const int V = a.c.V;
  if (p >= nblk * Wt) return nblk * V;
  const long long fbi = p / Wt;
  const long long r = p - fbi * Wt;
  int lo = 0, hi = V;   // first variable whose weight offset is >= r
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (vn_weight_off(a, mid) >= r) hi = mid; else lo = mid + 1;
  }
  return fbi * V + lo;
}
__device__ __forceinline__ void vn_group_range(const WaveArgs &a, long long nblk, long long gg, long long ngroups,
                                               long long &lo, long long &hi) {
  if (nblk * a.c.V < kBalanceMinTasks) {
    group_range(nblk * a.c.V, gg, ngroups, lo, hi);
    return;
  }
  const long long Wt = a.c.E + a.c.V + (a.markov ? 2LL * a.c.N : 0);
  const long long total = nblk * Wt;
  const long long chunk = (total + ngroups - 1) / ngroups;
  lo = vn_task_at(a, Wt, nblk, gg * chunk);
  hi = vn_task_at(a, Wt, nblk, (gg + 1) * chunk);
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
// parity of a value < 16 without POPC (a slow-pipe instruction whose latency
// showed up as 8 % of k_cn's stall samples, profiles/r02): bit x of 0x6996
__device__ __forceinline__ uint32_t parity4(int x) { return (0x6996u >> (x & 15)) & 1u; }

template <int KR, int T>
__device__ __forceinline__ void sign_masks(int z, int c, uint32_t (&sm)[KR]) {
  constexpr int LT = ilog2(T);
  static_assert(KR <= 16 && T <= 16, "sign_masks: parity4 covers 4 bits");
  const int zk = z >> LT;
  const uint32_t base = (T > 1) ? (parity4(z & c & (T - 1)) << 31) : 0u;
#pragma unroll
  for (int k = 0; k < KR; ++k) sm[k] = base ^ (parity4(zk & k) << 31);
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
                                           const float *Tsm, double (&pr)[KR], const float *exr_in = nullptr) {
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
  // rows of j-1 (issue_extras: slot 0) and of j+1 (slot 1), or two rows
  // anywhere (exr_in: shared or global memory, k_sus_dc)
  const float *exl = ex;
  const float *exr = exr_in ? exr_in : ex + Q * 32;
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
    elided_bar<T>(g);  // red reused every other task without a barrier
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
    elided_bar<T>(g);  // red reused across tasks without a barrier
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
  // Prefetch the current item's edge range (row_ptr / col_ptr) into L1: the
  // in-group producer lane reads it at its next refill, a task later (an L1
  // hit), instead of stalling its warp -- and every barrier of its group -- on
  // an L2 load right before the TMA issue.
  __device__ __forceinline__ void load_range(const int *ptr) {
    if (t < hi) asm volatile("prefetch.global.L1 [%0];" ::"l"(ptr + item));
  }
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
                                        Issue issue, int sus_lvl_begin = -1, bool vn_weighted = false) {
  const long long ngroups = (long long)gridDim.x * G;
  Cursor cur[G];
  int ring[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    long long lo, hi;
    if (sus_lvl_begin >= 0)
      sus_group_range(a, sus_lvl_begin, nitems, ntask / nitems, (long long)blockIdx.x * G + g, ngroups, lo, hi);
    else if (vn_weighted)
      vn_group_range(a, ntask / nitems, (long long)blockIdx.x * G + g, ngroups, lo, hi);
    else
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

// ============================================================== SUS: stage issue
// Units: one per (column, check slot) -- the check's other edges in at most
// two contiguous runs; the last unit of a column also carries the prior's
// extra rows and the column's VarDesc.  The unit's record (LvlUnit, level
// order) comes from the producer's UnitWalker, which loads it one unit ahead:
// no dependent global load on the producer lane between two TMA issues.
template <int Q, bool MARKOV, bool XTRA_MARKOV = MARKOV>
__device__ __forceinline__ void sus_issue_rec(const WaveArgs &a, int fb, const LvlUnit &un, unsigned char *hdr,
                                              unsigned char *pay, unsigned char *xtra, uint64_t *full) {
  TaskInfo *ti = (TaskInfo *)hdr;
  ti->fb = fb; ti->item = un.j; ti->e0 = un.e0; ti->deg = un.dv;
  ti->s = un.s; ti->r0 = un.r0; ti->d = un.d; ti->pos = un.pos; ti->i = un.i;
  const int nunits = un.dv > 0 ? un.dv : 1;
  const bool last = (un.s == nunits - 1);
  uint32_t b0 = 0, b1 = 0;
  const float *rowbase = a.qmsg + ((size_t)fb * a.c.E + un.r0) * Q * 32;
  if (un.dv > 0) {
    b0 = (uint32_t)un.pos * Q * 128;
    b1 = (uint32_t)(un.d - 1 - un.pos) * Q * 128;
  }
  const uint32_t bx = last ? 64 + extras_bytes<Q, XTRA_MARKOV>(a, un.j) : 0;
  mbar_expect_tx(full, (un.dv > 0 ? 64 + 32 : 0) + (a.early_exit ? 128 : 0) + b0 + b1 + bx);
  if (un.dv > 0) {
    bulk_g2s(hdr + 128, a.c.sus_desc + un.e0 + un.s, 64, full);
    bulk_g2s(hdr + 256, a.z + ((size_t)fb * a.c.M + un.i) * 32, 32, full);
  }
  if (a.early_exit) bulk_g2s(hdr + 384, a.conv + fb * 32, 128, full);
  if (b0) bulk_g2s(pay, rowbase, b0, full);
  if (b1) bulk_g2s(pay + (size_t)un.pos * Q * 128, rowbase + (size_t)(un.pos + 1) * Q * 32, b1, full);
  if (last) {
    bulk_g2s(hdr + 192, a.c.var_desc + un.j, 64, full);
    issue_extras<Q, XTRA_MARKOV>(a, fb, un.j, xtra, full);
  }
}

// Producer-side walk over the units of a contiguous range [lo, hi) of
// (frame block, column) tasks of one level, in unit order (a level's units
// are contiguous, column after column).  take() loads the current unit's
// record (an L1 hit: it was prefetched when the previous unit was taken) and
// prefetches the next one -- no dependent L2 load on the producer lane
// between two TMA issues, and no record held in registers.
struct UnitWalker {
  long long t, hi;
  int fbi, fb, col, ncols, u, u0;
  __device__ __forceinline__ void init(const WaveArgs &a, long long lo, long long hi_, int ncols_, int lvl_begin) {
    t = lo; hi = hi_; ncols = ncols_;
    fbi = fb = col = u = u0 = 0;
    if (t < hi) {
      fbi = (int)(t / ncols);
      col = (int)(t - (long long)fbi * ncols);
      fb = a.list[fbi];
      u0 = a.c.lvl_col[lvl_begin].unit0;
      u = a.c.lvl_col[lvl_begin + col].unit0;
    }
  }
  __device__ __forceinline__ bool valid() const { return t < hi; }
  __device__ __forceinline__ LvlUnit take(const WaveArgs &a) {
    const LvlUnit r = a.c.lvl_unit[u];
    const bool col_done = r.s + 1 >= (r.dv > 0 ? r.dv : 1);
    if (col_done) {
      ++t;
      if (++col == ncols) {
        col = 0;
        ++fbi;
        if (t < hi) fb = a.list[fbi];
        u = u0;
      } else {
        ++u;
      }
    } else {
      ++u;
    }
    if (t < hi) asm volatile("prefetch.global.L1 [%0];" ::"l"(a.c.lvl_unit + u));
    return r;
  }
};

template <int Q, int DMAX, bool MARKOV>
__device__ __forceinline__ bool sus_issue(const WaveArgs &a, int fb, int col, int &s, int lvl_begin,
                                          unsigned char *hdr, unsigned char *pay, unsigned char *xtra,
                                          uint64_t *full) {
  // generic-producer path (dedicated producer warp, produce()): loads the record
  const LvlCol lc = a.c.lvl_col[lvl_begin + col];
  const int nunits = lc.dv > 0 ? lc.dv : 1;
  const LvlUnit un = a.c.lvl_unit[lc.unit0 + s];
  sus_issue_rec<Q, MARKOV>(a, fb, un, hdr, pay, xtra, full);
  if (++s >= nunits) {
    s = 0;
    return true;  // task complete
  }
  return false;
}

}  // namespace gfq

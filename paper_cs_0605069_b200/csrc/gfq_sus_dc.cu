// gfq_sus_dc.cu -- the SUS level kernel for small fields (q <= 16) by direct
// convolution: PAPER.md §2, SUS steps 1-4 with the check-node
// update Eq. (3) evaluated as the sum over configurations it is.
//
// Why a second SUS kernel.  In the transform formulation (gfq_bp.cu) a SUS
// unit (one check of one column) forward-transforms the d-1 other messages of
// the check, multiplies, and inverse-transforms; in fp64 (the inverse
// transform produces small probabilities by cancellation) and, for q = 16,
// with the q-vector split over two warps (layout switches through shared
// memory, group barriers).  For q <= 16 the direct sum is as cheap: the XOR-
// convolution S = u_1 (*) u_2 (*) ... of the permuted other messages costs
// q^2 fused multiply-adds per factor, all terms are non-negative (no
// cancellation: fp32 keeps every entry to a relative ~q ulps, including the
// tiny ones), and a whole q-vector fits one thread's registers.  So one warp
// owns a unit for its 32 frames (one frame per lane): no layout switches, no
// cross-warp barriers, every warp an independent TMA pipeline.
//
//   u_k(y) = q_ij_k(h_k^-1 y)           (distribution of h_k x_k; rows chosen at load)
//   S(y)   = sum_{x_1 ^ ... ^ x_{d-1} = y} prod_k u_k(x_k)   (fp32, FFMA2 pairs)
//   r_ij(a) = S(z_i ^ h_ij a)           (Eq. 3: the check sum equals z_i, reading A4)
// S is stored to the warp's shared r slots at row a = h^-1 y ^ h^-1 z (per-lane
// z: a per-lane XOR of the row; rows are 128-byte lines of 32 lanes, so the
// access is bank-conflict free).  The variable update of the column (Eq. 4,
// posterior Eq. 5, clipping) is vn_core in fp64 registers, as in the other
// kernels.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>

#include "gfq_device.cuh"
#include "gfq_launch.cuh"

namespace gfq {

// warps per CTA / stages per warp (tuning knobs)
#ifndef GFQ_DC_W
#define GFQ_DC_W 16      // q = 16: 16 warps x 108 registers, 216 KB (measured 15 -> 16: C4 3.58 -> 3.78 TB/s)
#endif
#ifndef GFQ_DC_VN_UNROLL
#define GFQ_DC_VN_UNROLL 2   // entries of the streamed variable node in flight
#endif
#ifndef GFQ_DC_W_SMALL
#define GFQ_DC_W_SMALL 32  // q <= 8: 64 registers per thread, 7 KB per warp
#endif
#ifndef GFQ_DC_S
#define GFQ_DC_S 1
#endif
#ifndef GFQ_DC_S_MARKOV
#define GFQ_DC_S_MARKOV 1
#endif
#ifndef GFQ_DC_FFMA2
#define GFQ_DC_FFMA2 1
#endif

constexpr int kDcVnUnroll = GFQ_DC_VN_UNROLL;

template <int Q, int DMAX, int DVMAX, bool MARKOV, int S, int W>
struct DCShape {
  // the stage's extra rows: the p per-bit flip probabilities of a noise
  // column; a Markov source column's neighbour posteriors are read from L2
  // (prefetched when its first unit is issued) instead of taking 2q rows of
  // every stage
  static constexpr int XR = Extra<Q, false>::rows;
  static constexpr size_t PAY = (size_t)(DMAX - 1) * Q * 128;  // the d-1 other messages
  static constexpr size_t RSM = (size_t)DVMAX * Q * 128;        // fp32 r of the column's checks
  static constexpr size_t TSM_B = (MARKOV ? (size_t)2 * Q * Q * 4 : 0) + (size_t)2 * Q * Q;
  using Sh = Shape<Q, S, W, PAY, RSM, (size_t)XR * 128, TSM_B, false>;
  static constexpr size_t SMEM = Sh::SMEM;
  static constexpr int THREADS = W * 32;
};

__device__ __forceinline__ void prefetch_l2(const void *p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Rows of the Markov neighbours j-1 / j+1 that source column j reads (reading
// A9 snapshot or A34 in-sweep, markov_nbrs), or null.
template <int Q>
__device__ __forceinline__ void markov_rows(const WaveArgs &a, int fb, int j, const float *&left,
                                            const float *&right) {
  const int N = a.c.N;
  const int nb = markov_nbrs(a, j);
  left = (nb & 1) ? (a.gs ? a.qs_new : a.qs_old) + ((size_t)fb * N + (j - 1)) * Q * 32 : nullptr;
  right = (nb & 2) ? a.qs_old + ((size_t)fb * N + (j + 1)) * Q * 32 : nullptr;
}

// One SUS unit into a stage: sus_issue_rec (gfq_device.cuh) with only the
// noise rows as extras; a Markov source column's neighbour posteriors are
// prefetched into L2 with its first unit.
template <int Q, bool MARKOV>
__device__ __forceinline__ void dc_issue(const WaveArgs &a, int fb, const LvlUnit &un, unsigned char *hdr,
                                         unsigned char *pay, unsigned char *xtra, uint64_t *full) {
  if (MARKOV && un.s == 0 && un.j < a.c.N) {
    const float *l, *r;
    markov_rows<Q>(a, fb, un.j, l, r);
    if (l) prefetch_l2(l, Q * 128);
    if (r) prefetch_l2(r, Q * 128);
  }
  sus_issue_rec<Q, MARKOV, false>(a, fb, un, hdr, pay, xtra, full);
}

// With one stage per warp the TMA load of a unit starts only when the previous
// unit has released the stage, so its HBM latency is exposed (the mbarrier wait
// was 19 % of the stall samples at C4, profiles/r02).  The producer lane
// therefore prefetches the NEXT unit's message rows into L2 while the current
// unit is being processed (a second UnitWalker running one unit ahead, whose
// record was itself prefetched a step earlier): the later TMA load is an L2 hit.
// In flight: 148 SMs x 15 warps x <= 6 KB, far below the 126 MB of L2.
// Measured (profiles/r02/dc_variants.txt): C4 (q = 16, 6 KB units) 3.30 -> 3.36
// TB/s model; C3 (q = 8, 3 KB units) 3.80 -> 3.11: the producer lane's extra
// work outweighs the shorter wait there, so it is on from q = 16 only.  Two
// stages x 10 warps instead: C4 2.49, C3 3.37 TB/s.
#ifndef GFQ_DC_L2_PREFETCH_MINQ
#define GFQ_DC_L2_PREFETCH_MINQ 16
#endif
template <int Q>
__device__ __forceinline__ void dc_prefetch_unit(const WaveArgs &a, int fb, const LvlUnit &un) {
  if (un.dv <= 0) return;
  const float *rowbase = a.qmsg + ((size_t)fb * a.c.E + un.r0) * Q * 32;
  const uint32_t b0 = (uint32_t)un.pos * Q * 128, b1 = (uint32_t)(un.d - 1 - un.pos) * Q * 128;
  if (b0) prefetch_l2(rowbase, b0);
  if (b1) prefetch_l2(rowbase + (size_t)(un.pos + 1) * Q * 32, b1);
}

// u[y] = message(h^-1 y) for y = 0..Q-1 from a stage slot (fp32 rows of 32 lanes)
template <int Q>
__device__ __forceinline__ void dc_load(uint32_t slot_lane, uint32_t rt, unsigned long long pk, float (&u)[Q]) {
  uint32_t ad[Q];
  tab_addrs_sm<Q, Q>(slot_lane, rt, pk, 0, ad);
#pragma unroll
  for (int y = 0; y < Q; ++y) u[y] = lds_f32(ad[y]);
}

// s[y] = sum_x u[x] v[y ^ x]  (XOR convolution; x ascending)
template <int Q>
__device__ __forceinline__ void dc_conv(const float (&u)[Q], const float (&v)[Q], float (&s)[Q]) {
#if GFQ_DC_FFMA2
  if constexpr (Q >= 4) {
    // pairs (s[2m], s[2m+1]) += u[x] * (v[2m ^ x], v[2m+1 ^ x]): for even x the
    // pair of v is (v[2m^x], v[(2m^x)+1]) in order, for odd x it is swapped
    unsigned long long vp[Q / 2], vs[Q / 2], acc[Q / 2];
#pragma unroll
    for (int m = 0; m < Q / 2; ++m) {
      vp[m] = ((unsigned long long)__float_as_uint(v[2 * m + 1]) << 32) | __float_as_uint(v[2 * m]);
      vs[m] = ((unsigned long long)__float_as_uint(v[2 * m]) << 32) | __float_as_uint(v[2 * m + 1]);
    }
#pragma unroll
    for (int m = 0; m < Q / 2; ++m) {
      const unsigned long long u0 = ((unsigned long long)__float_as_uint(u[0]) << 32) | __float_as_uint(u[0]);
      asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(acc[m]) : "l"(u0), "l"(vp[m]));
    }
#pragma unroll
    for (int x = 1; x < Q; ++x) {
      const unsigned long long ux = ((unsigned long long)__float_as_uint(u[x]) << 32) | __float_as_uint(u[x]);
#pragma unroll
      for (int m = 0; m < Q / 2; ++m) {
        const int src = m ^ (x >> 1);
        const unsigned long long vv = (x & 1) ? vs[src] : vp[src];
        asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[m]) : "l"(ux), "l"(vv));
      }
    }
#pragma unroll
    for (int m = 0; m < Q / 2; ++m) {
      s[2 * m] = __uint_as_float((unsigned)(acc[m] & 0xffffffffu));
      s[2 * m + 1] = __uint_as_float((unsigned)(acc[m] >> 32));
    }
    return;
  }
#endif
#pragma unroll
  for (int y = 0; y < Q; ++y) {
    float acc = u[0] * v[y];
#pragma unroll
    for (int x = 1; x < Q; ++x) acc = fmaf(u[x], v[y ^ x], acc);
    s[y] = acc;
  }
}

// SUS step 1 for one check of the column (DO = d-1 other edges): S in fp32,
// then q * r_ij (the scale of the transform kernels' stored r, which the
// variable node normalises away) into r slot ti.s of the warp.  The stage is
// released as soon as its rows are in registers; the caller refills it (one
// copy of the issue code in the kernel: the instruction cache is the limit).
template <int Q, int DO>
__device__ __forceinline__ void dc_check(const WaveArgs &a, const unsigned char *hdr, uint32_t pay_lane, uint32_t rt,
                                         float *rsm, int lane, bool frozen, bool release, uint64_t *empty) {
  const TaskInfo ti = *(const TaskInfo *)hdr;
  const SusDesc *sd = (const SusDesc *)(hdr + 128);
  const int z = hdr[256 + lane];
  const unsigned long long pke = sd->perm_e;
  float S[Q];
  if constexpr (DO == 0) {
    // degree-1 check: the sum over no other variable is the point mass at 0
    if (release) release_stage(empty, lane);
#pragma unroll
    for (int y = 0; y < Q; ++y) S[y] = (y == 0) ? 1.0f : 0.0f;
  } else if constexpr (DO == 1) {
    dc_load<Q>(pay_lane, rt, sd->perm_o[0], S);
    if (release) release_stage(empty, lane);
  } else {
    float u[Q], v[Q];
    dc_load<Q>(pay_lane, rt, sd->perm_o[0], u);
    dc_load<Q>(pay_lane + Q * 128, rt, sd->perm_o[1], v);
    if constexpr (DO == 2) {
      if (release) release_stage(empty, lane);
      dc_conv<Q>(u, v, S);
    } else {
      static_assert(DO == 3, "dc_check: check degree <= 4");
      float w[Q], t[Q];
      dc_load<Q>(pay_lane + 2 * Q * 128, rt, sd->perm_o[2], w);
      if (release) release_stage(empty, lane);
      dc_conv<Q>(u, v, t);
      dc_conv<Q>(t, w, S);
    }
  }
  // r(a) = S(z ^ h a): S[y] goes to row a = h^-1 y ^ h^-1 z
  uint32_t ad[Q];
  tab_addrs_sm<Q, Q>(0u, rt, pke, 0, ad);  // (h^-1 y) << 7
  uint32_t hz;
  asm volatile("ld.shared.u16 %0, [%1];" : "=r"(hz) : "r"(rt + (uint32_t)(((pke & 0xff) * Q + z) * 2)));
  unsigned char *rs = (unsigned char *)(rsm + (size_t)ti.s * Q * 32 + lane);
#pragma unroll
  for (int y = 0; y < Q; ++y) *(float *)(rs + (ad[y] ^ hz)) = S[y] * (float)Q;
  if (a.rmsg != nullptr && !frozen) {  // keep_messages only (export)
    unsigned char *rd = (unsigned char *)(a.rmsg + ((size_t)ti.fb * a.c.E + ti.e0 + ti.s) * Q * 32 + lane);
#pragma unroll
    for (int y = 0; y < Q; ++y) *(float *)(rd + (ad[y] ^ hz)) = S[y] * (float)Q;
  }
}

// SUS step 2 (+ step 4, reading A8) for the column: Eq. (4) for each of its
// edges and the posterior Eq. (5) with clipping, from the fresh r's (fp32 rows
// of the warp's r slots) and the prior (an fp32 row computed once, dc_prior).
// fp64 products and sums as vn_core, streamed over the entries in two passes
// (sums, then normalised stores): few registers and little code, so more
// warps fit an SM and the kernel stays in the instruction cache.
template <int Q>
__device__ __forceinline__ void dc_prior(const WaveArgs &a, int fb, int j, const unsigned char *xtra,
                                         const float *Tsm, float *prs, int lane) {
  double pr[Q];
  if (a.markov && j < a.c.N) {
    const float *l, *r;
    markov_rows<Q>(a, fb, j, l, r);   // L2-resident (prefetched with the column's first unit)
    prior_from<Q, Q, true>(a, j, 0, lane, l ? l : r, Tsm, pr, r ? r : l);
  } else {
    prior_from<Q, Q, false>(a, j, 0, lane, (const float *)xtra, Tsm, pr);
  }
#pragma unroll
  for (int k = 0; k < Q; ++k) prs[k * 32 + lane] = (float)pr[k];
}

template <int Q, int DV>
__device__ __forceinline__ void dc_vn(const WaveArgs &a, const unsigned char *hdr, const float *rsm,
                                      const float *prs, int lane, bool frozen) {
  constexpr int NS = DV + 1;
  const TaskInfo ti = *(const TaskInfo *)hdr;
  const VarDesc *vd = (const VarDesc *)(hdr + 192);
  const int fb = ti.fb, j = ti.item;
  const long long E = a.c.E;
  const float *P = prs + lane;
  const float *R = rsm + lane;
  // leave-one-out products at entry k: o[s] = p prod_{s' != s} r_s', o[DV] = p prod r
  auto prods = [&](int k, double (&o)[NS]) {
    const double p = (double)P[k * 32];
    double r[DV > 0 ? DV : 1];
#pragma unroll
    for (int t = 0; t < DV; ++t) r[t] = (double)R[(t * Q + k) * 32];
    if constexpr (DV == 0) {
      o[0] = p;
    } else if constexpr (DV == 1) {
      o[0] = p; o[1] = p * r[0];
    } else if constexpr (DV == 2) {
      o[0] = p * r[1]; o[1] = p * r[0]; o[2] = o[0] * r[0];
    } else {
      const double x = p * r[0], bc = r[1] * r[2];
      o[0] = p * bc; o[1] = x * r[2]; o[2] = x * r[1]; o[3] = x * bc;
    }
  };
  double sums[NS], mx = 0.0;
#pragma unroll
  for (int t = 0; t < NS; ++t) sums[t] = 0.0;
#pragma unroll kDcVnUnroll
  for (int k = 0; k < Q; ++k) {
    double o[NS];
    prods(k, o);
#pragma unroll
    for (int t = 0; t < NS; ++t) sums[t] += o[t];
    mx = fmax(mx, o[DV]);
  }
  int bad = 0;
  double inv[NS];
  float add[NS];
#pragma unroll
  for (int t = 0; t < NS; ++t) {
    const bool ok = sums[t] > 0.0 && isfinite(sums[t]);
    bad += !ok;
    inv[t] = ok ? fast_rcp(sums[t]) : 0.0;
    add[t] = ok ? 0.0f : 1.0f / Q;
  }
  const bool okq = add[DV] == 0.0f;
  const double thr = mx * (1.0 - kTieRel);  // clipping: smallest a within the tie band
  int bidx = Q;
  float *qrow[DV > 0 ? DV : 1];
#pragma unroll
  for (int t = 0; t < DV; ++t) qrow[t] = a.qmsg + ((size_t)fb * E + vd->qdst[t]) * Q * 32 + lane;
  float *qsrow = (a.markov && j < a.c.N && a.qs_new) ? a.qs_new + ((size_t)fb * a.c.N + j) * Q * 32 + lane : nullptr;
  float *qarow = a.qall ? a.qall + ((size_t)fb * a.c.V + j) * Q * 32 + lane : nullptr;
#pragma unroll kDcVnUnroll
  for (int k = 0; k < Q; ++k) {
    double o[NS];
    prods(k, o);
    if (o[DV] >= thr && bidx == Q) bidx = k;
    if (!frozen) {
#pragma unroll
      for (int t = 0; t < DV; ++t) qrow[t][k * 32] = (float)(o[t] * inv[t]) + add[t];
      const float qv = (float)(o[DV] * inv[DV]) + add[DV];
      if (qsrow) qsrow[k * 32] = qv;
      if (qarow) qarow[k * 32] = qv;
    }
  }
  if (bidx >= Q || !okq) bidx = 0;
  if (!frozen) {
    a.xhat[((size_t)fb * a.c.V + j) * 32 + lane] = (unsigned char)bidx;
    if (bad) atomicAdd(a.stats + 0, (unsigned long long)bad);
  }
}

template <int Q, int DMAX, int DVMAX, bool MARKOV, int S, int W>
__global__ void __launch_bounds__(DCShape<Q, DMAX, DVMAX, MARKOV, S, W>::THREADS)
    k_sus_dc(WaveArgs a, int lvl_begin, int ncols) {
  using DS = DCShape<Q, DMAX, DVMAX, MARKOV, S, W>;
  using Sh = typename DS::Sh;
  static_assert(DMAX <= 4 && DVMAX <= 3, "k_sus_dc: check degree <= 4, variable degree <= 3");
  extern __shared__ __align__(128) unsigned char smem[];
  const SmemPtrs sp = smem_ptrs<Sh, S, W>(smem);
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  // programmatic dependent launch: the next level's CTAs may start their
  // prologue now; everything after griddepcontrol.wait reads this level's output
  asm volatile("griddepcontrol.launch_dependents;");
  if (threadIdx.x == 0) init_bars<S, W>(sp.bars, 1);
  float *Tsm = sp.tsm;
  if constexpr (MARKOV) {
    if (a.Tf)
      for (int k = threadIdx.x; k < 2 * Q * Q; k += blockDim.x) Tsm[k] = a.Tf[k];
  }
  unsigned short *rtab = (unsigned short *)(sp.tsm + (MARKOV ? 2 * Q * Q : 0));
  for (int k = threadIdx.x; k < Q * Q; k += blockDim.x) rtab[k] = a.c.rowtab[k];
  const uint32_t rt = smem_u32(rtab);
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const long long ntask = (long long)(*a.nactive) * ncols;
  float *rsm = (float *)(sp.scr + (size_t)g * DS::RSM);
  const bool producer = (lane == 0);
  long long lo, hi;
  sus_group_range(a, lvl_begin, ncols, (long long)(*a.nactive), (long long)blockIdx.x * W + g,
                  (long long)gridDim.x * W, lo, hi);
  UnitWalker pc, la;   // la runs S units ahead of pc (L2 prefetch)
  if (producer) {
    pc.init(a, lo, hi, ncols, lvl_begin);
    if (Q >= GFQ_DC_L2_PREFETCH_MINQ) {
      la.init(a, lo, hi, ncols, lvl_begin);
      for (int n = 0; n < S && la.valid(); ++n) (void)la.take(a);
    }
  }
  auto issue_next = [&](int k) {
    if (!pc.valid()) return;
    const int fb = pc.fb;
    const LvlUnit un = pc.take(a);
    dc_issue<Q, MARKOV>(a, fb, un, sp.hdr + (size_t)k * kHdr, sp.pay + (size_t)k * Sh::PAYA,
                        sp.xtra + (size_t)k * Sh::XTRA_A, sp.bars + k);
    if (Q >= GFQ_DC_L2_PREFETCH_MINQ && la.valid()) {
      const int fb1 = la.fb;
      const LvlUnit un1 = la.take(a);   // an L1 hit: prefetched when la took the unit before it
      dc_prefetch_unit<Q>(a, fb1, un1);
    }
  };
  if (producer)
    for (int n = 0; n < S; ++n) issue_next(g * S + n);
  int rr = 0;  // units consumed by this warp
  for (long long task = lo; task < hi; ++task) {
    int nunits = 1;
#pragma unroll 1
    for (int s = 0; s < nunits; ++s, ++rr) {
      const int st = rr % S, k = g * S + st;
      const unsigned char *hdr = sp.hdr + (size_t)k * kHdr;
      const unsigned char *xtra = sp.xtra + (size_t)k * Sh::XTRA_A;
      const uint32_t pay_lane = sp.pay_u32 + (uint32_t)((size_t)k * Sh::PAYA) + lane * 4;
      uint64_t *empty = sp.bars + W * S + k;
      const int par = (rr / S) & 1;
      auto refill = [&]() {
        if (producer && pc.valid()) {
          mbar_wait(empty, (uint32_t)par);
          issue_next(k);
        }
      };
      mbar_wait(sp.bars + k, (uint32_t)par);
      const TaskInfo *ti = (const TaskInfo *)hdr;
      const int dv = ti->deg, d = ti->d;
      nunits = dv > 0 ? dv : 1;
      const bool last = (s == nunits - 1);
      const bool frozen = a.early_exit && ((const int *)(hdr + 384))[lane] != 0;
      if (dv > 0) {
        // the last unit's stage also carries the column's VarDesc and prior
        // rows: it is released after the variable update
        switch (d - 1) {
          case 0: dc_check<Q, 0>(a, hdr, pay_lane, rt, rsm, lane, frozen, !last, empty); break;
          case 1: dc_check<Q, 1>(a, hdr, pay_lane, rt, rsm, lane, frozen, !last, empty); break;
          case 2: dc_check<Q, 2>(a, hdr, pay_lane, rt, rsm, lane, frozen, !last, empty); break;
          default: dc_check<Q, 3>(a, hdr, pay_lane, rt, rsm, lane, frozen, !last, empty); break;
        }
      }
      if (last) {
        // the prior row goes to this stage's payload: its rows are in registers
        // already, and the stage is released only after the variable update
        float *prs = (float *)(sp.pay + (size_t)k * Sh::PAYA);
        static_assert(Sh::PAYA >= (size_t)Q * 128, "prior row fits a stage payload");
        dc_prior<Q>(a, ti->fb, ti->item, xtra, Tsm, prs, lane);
        __syncwarp();  // the column's r slots and prior row are complete
        switch (dv) {
          case 0: dc_vn<Q, 0>(a, hdr, rsm, prs, lane, frozen); break;
          case 1: dc_vn<Q, 1>(a, hdr, rsm, prs, lane, frozen); break;
          case 2: dc_vn<Q, 2>(a, hdr, rsm, prs, lane, frozen); break;
          default: dc_vn<Q, 3>(a, hdr, rsm, prs, lane, frozen); break;
        }
        release_stage(empty, lane);  // syncwarp: every lane is done with the r slots too
      }
      refill();  // the stage was released above (last unit) or in dc_check
    }
  }
}

// ============================================================== PUS check node by direct convolution
// The horizontal pass (Eq. 3) for q <= 16 with the same arithmetic
// as the SUS unit above: one warp owns a check for its 32 frames; for every
// edge k it convolves the permuted messages of the other edges (fp32 FFMA2,
// non-negative terms) and writes q * r_k.  The syndrome shift r_k(a) =
// S(z ^ h_k a) is folded into the load of the first other message,
// u'(y) = u(y ^ z) (a per-lane XOR of the shared-memory row: rows are 128-byte
// lines of 32 lanes, so it is bank-conflict free), which makes the output rows
// uniform over the lanes: every store is one coalesced 128-byte line.
// Why: k_cn at q = 16 holds a whole check in fp64 registers (254 per thread,
// 8 warps per SM) and stalls on instruction fetch (72 KB of straight-line code,
// profiles/r02/c4_pus_details.csv); this kernel is short, fp32 and runs 16+
// warps per SM.  A degree-4 check costs 8 convolutions here against 6 with
// prefix / suffix products: the multiply-adds are not what limits it.
template <int Q, int DMAX, int S, int W>
struct CNDCShape {
  static constexpr size_t PAY = (size_t)DMAX * Q * 128;
  static constexpr size_t TSM_B = (size_t)2 * Q * Q;   // row-offset table
  using Sh = Shape<Q, S, W, PAY, 0, 0, TSM_B, false>;
  static constexpr size_t SMEM = Sh::SMEM;
  static constexpr int THREADS = W * 32;
};

template <int Q>
__device__ __forceinline__ void cndc_issue(const WaveArgs &a, int fb, int i, unsigned char *hdr, unsigned char *pay,
                                           uint64_t *full) {
  const int e0 = __ldg(a.c.row_ptr + i), d = __ldg(a.c.row_ptr + i + 1) - e0;
  TaskInfo *ti = (TaskInfo *)hdr;
  ti->fb = fb; ti->item = i; ti->e0 = e0; ti->deg = d;
  const uint32_t msg = (uint32_t)d * Q * 128;
  mbar_expect_tx(full, 128 + 32 + (a.early_exit ? 128 : 0) + msg);
  bulk_g2s(hdr + 128, a.c.check_desc + i, 128, full);
  bulk_g2s(hdr + 256, a.z + ((size_t)fb * a.c.M + i) * 32, 32, full);
  if (a.early_exit) bulk_g2s(hdr + 384, a.conv + fb * 32, 128, full);
  if (msg) bulk_g2s(pay, a.qmsg + ((size_t)fb * a.c.E + e0) * Q * 32, msg, full);
}

// u[y] = message(h^-1 (y ^ z)): dc_load with the per-lane syndrome shift hz = (h^-1 z) << 7
template <int Q>
__device__ __forceinline__ void dc_load_shift(uint32_t slot_lane, uint32_t rt, unsigned long long pk, uint32_t hz,
                                              float (&u)[Q]) {
  uint32_t ad[Q];
  tab_addrs_sm<Q, Q>(0u, rt, pk, 0, ad);
#pragma unroll
  for (int y = 0; y < Q; ++y) u[y] = lds_f32(slot_lane + (ad[y] ^ hz));
}

template <int Q, int D>
__device__ __forceinline__ void cndc_check(const WaveArgs &a, const unsigned char *hdr, uint32_t pay_lane, uint32_t rt,
                                           int lane, bool frozen) {
  const TaskInfo ti = *(const TaskInfo *)hdr;
  const CheckDesc *cd = (const CheckDesc *)(hdr + 128);
  const int z = hdr[256 + lane];
#pragma unroll
  for (int k = 0; k < D; ++k) {
    float S[Q];
    if constexpr (D == 1) {
      // no other edge: the point mass at 0 shifted by z, S'(y) = [y = z]
#pragma unroll
      for (int y = 0; y < Q; ++y) S[y] = (y == z) ? 1.0f : 0.0f;
    } else {
      // the other edges in row order; the first of them carries the shift
      constexpr int NO = D - 1;
      int o[NO];
#pragma unroll
      for (int t = 0, x = 0; t < D; ++t)
        if (t != k) o[x++] = t;
      const unsigned long long pk0 = cd->perm[o[0]];
      uint32_t hz;
      asm volatile("ld.shared.u16 %0, [%1];" : "=r"(hz) : "r"(rt + (uint32_t)(((pk0 & 0xff) * Q + z) * 2)));
      if constexpr (NO == 1) {
        dc_load_shift<Q>(pay_lane + (uint32_t)(o[0] * Q * 128), rt, pk0, hz, S);
      } else {
        float u[Q], v[Q];
        dc_load_shift<Q>(pay_lane + (uint32_t)(o[0] * Q * 128), rt, pk0, hz, u);
        dc_load<Q>(pay_lane + (uint32_t)(o[1] * Q * 128), rt, cd->perm[o[1]], v);
        if constexpr (NO == 2) {
          dc_conv<Q>(u, v, S);
        } else {
          static_assert(NO == 3, "cndc_check: check degree <= 4");
          float w[Q], t2[Q];
          dc_load<Q>(pay_lane + (uint32_t)(o[2] * Q * 128), rt, cd->perm[o[2]], w);
          dc_conv<Q>(u, v, t2);
          dc_conv<Q>(t2, w, S);
        }
      }
    }
    // r_k(a) = S'(h_k a): S'[y] goes to row a = h_k^-1 y of the edge's canonical slot
    if (!frozen) {
      uint32_t ad[Q];
      tab_addrs_sm<Q, Q>(0u, rt, cd->perm[k], 0, ad);
      unsigned char *dst = (unsigned char *)(a.rmsg + ((size_t)ti.fb * a.c.E + cd->canon[k]) * Q * 32 + lane);
#pragma unroll
      for (int y = 0; y < Q; ++y) *(float *)(dst + ad[y]) = S[y] * (float)Q;
    }
  }
}

template <int Q, int S, int W>
__global__ void __launch_bounds__(CNDCShape<Q, 4, S, W>::THREADS) k_cn_dc(WaveArgs a) {
  using CS = CNDCShape<Q, 4, S, W>;
  using Sh = typename CS::Sh;
  extern __shared__ __align__(128) unsigned char smem[];
  const SmemPtrs sp = smem_ptrs<Sh, S, W>(smem);
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  if (threadIdx.x == 0) init_bars<S, W>(sp.bars, 1);
  unsigned short *rtab = (unsigned short *)sp.tsm;
  for (int k = threadIdx.x; k < Q * Q; k += blockDim.x) rtab[k] = a.c.rowtab[k];
  const uint32_t rt = smem_u32(rtab);
  __syncthreads();
  const int M = a.c.M;
  const long long ntask = (long long)(*a.nactive) * M;
  const bool producer = (lane == 0);
  long long lo, hi;
  group_range(ntask, (long long)blockIdx.x * W + g, (long long)gridDim.x * W, lo, hi);
  Cursor pc;
  if (producer) {
    pc.init(a, lo, hi, M);
    for (int n = 0; n < S && pc.valid(); ++n) {
      const int k = g * S + n;
      cndc_issue<Q>(a, pc.fb, pc.item, sp.hdr + (size_t)k * kHdr, sp.pay + (size_t)k * Sh::PAYA, sp.bars + k);
      pc.advance(a);
    }
  }
  for (long long task = lo; task < hi; ++task) {
    const int rr = (int)(task - lo), st = rr % S, k = g * S + st;
    const unsigned char *hdr = sp.hdr + (size_t)k * kHdr;
    const uint32_t pay_lane = sp.pay_u32 + (uint32_t)((size_t)k * Sh::PAYA) + lane * 4;
    uint64_t *empty = sp.bars + W * S + k;
    const uint32_t par = (uint32_t)((rr / S) & 1);
    mbar_wait(sp.bars + k, par);
    const int d = ((const TaskInfo *)hdr)->deg;
    const bool frozen = a.early_exit && ((const int *)(hdr + 384))[lane] != 0;
    switch (d) {
      case 0: break;
      case 1: cndc_check<Q, 1>(a, hdr, pay_lane, rt, lane, frozen); break;
      case 2: cndc_check<Q, 2>(a, hdr, pay_lane, rt, lane, frozen); break;
      case 3: cndc_check<Q, 3>(a, hdr, pay_lane, rt, lane, frozen); break;
      default: cndc_check<Q, 4>(a, hdr, pay_lane, rt, lane, frozen); break;
    }
    release_stage(empty, lane);
    if (producer && pc.valid()) {
      mbar_wait(empty, par);
      cndc_issue<Q>(a, pc.fb, pc.item, sp.hdr + (size_t)k * kHdr, sp.pay + (size_t)k * Sh::PAYA, sp.bars + k);
      pc.advance(a);
    }
  }
}

// measured (profiles/r02/dc_variants.txt): q = 16: 2 stages x 12 warps 10.03 ms per C4 launch
// (1 x 16: 11.07, 3 x 8: 12.95; k_cn: 12.00); q = 8: 1 x 16 1.267 ms per C3 launch (2 x 16: 1.328; k_cn: 1.383)
#ifndef GFQ_CNDC_W
#define GFQ_CNDC_W 12     // q = 16: warps per CTA / stages per warp (8 KB per stage)
#endif
#ifndef GFQ_CNDC_S
#define GFQ_CNDC_S 2
#endif
#ifndef GFQ_CNDC_W8
#define GFQ_CNDC_W8 16    // q = 8 (4 KB per stage)
#endif
#ifndef GFQ_CNDC_S8
#define GFQ_CNDC_S8 1
#endif
template <int Q>
static int cndc_launch(const WaveArgs &a, cudaStream_t s) {
  constexpr int S = Q >= 16 ? GFQ_CNDC_S : GFQ_CNDC_S8, W = Q >= 16 ? GFQ_CNDC_W : GFQ_CNDC_W8;
  using CS = CNDCShape<Q, 4, S, W>;
  static_assert(CS::SMEM <= 232448, "k_cn_dc: shared memory");
  auto k = k_cn_dc<Q, S, W>;
  const int grid = grid_for(k, CS::THREADS, CS::SMEM, ((long long)a.nfb * a.c.M + W - 1) / W);
  k<<<grid, CS::THREADS, CS::SMEM, s>>>(a);
  return check_launch("k_cn_dc");
}

// q = 8, 16 with check degree <= 4; GFQ_CN_DC=0 / 1 in the environment overrides
// the build-time default.
#ifndef GFQ_CN_DC_DEFAULT
#define GFQ_CN_DC_DEFAULT 1
#endif
bool cn_dc_applies(const WaveArgs &a) {
  static int on = -1;
  if (on < 0) {
    const char *e = getenv("GFQ_CN_DC");
    on = e ? (atoi(e) != 0) : GFQ_CN_DC_DEFAULT;
  }
  return on && (a.c.q == 8 || a.c.q == 16) && a.c.max_cdeg <= 4;
}

int launch_cn_dc(const WaveArgs &a, cudaStream_t s) {
  switch (a.c.q) {
    case 8: return cndc_launch<8>(a, s);
    case 16: return cndc_launch<16>(a, s);
    default: break;
  }
  set_error("k_cn_dc: unsupported q");
  return GFQ_EUNSUPPORTED;
}

// most warps per CTA (<= want) whose stages fit the 227 KB of shared memory
template <int Q, bool MK, int S>
constexpr int dc_warps(int want) {
  return (want <= 1 || DCShape<Q, 4, 3, MK, S, 1>::SMEM +
                               (size_t)(want - 1) * (DCShape<Q, 4, 3, MK, S, 2>::SMEM - DCShape<Q, 4, 3, MK, S, 1>::SMEM) <=
                           232448)
             ? want
             : dc_warps<Q, MK, S>(want - 1);
}

template <int Q, bool MK>
static int dc_launch(const WaveArgs &a, int lb, int ncols, cudaStream_t s) {
  constexpr int S = MK ? GFQ_DC_S_MARKOV : GFQ_DC_S, W = dc_warps<Q, MK, S>(Q >= 16 ? GFQ_DC_W : GFQ_DC_W_SMALL);
  using DS = DCShape<Q, 4, 3, MK, S, W>;
  static_assert(DS::SMEM <= 232448, "k_sus_dc: shared memory");
  auto k = k_sus_dc<Q, 4, 3, MK, S, W>;
  const int grid = grid_for(k, DS::THREADS, DS::SMEM, ((long long)a.nfb * ncols + W - 1) / W);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(DS::THREADS);
  cfg.dynamicSmemBytes = DS::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k, a, lb, ncols);
  if (e != cudaSuccess) return cuda_fail(e, "k_sus_dc");
  return check_launch("k_sus_dc");
}

// Fields handled here: q = 8 and 16 (check degree <= 4, variable degree <= 3).
// The environment variable GFQ_SUS_DC_MINQ moves the lower end (4, 8, 16):
// measured on C3 (q = 8, 4096 frames) 3.47 -> 3.81 TB/s model against the
// transform kernel, on C2 (q = 4) 1.80 -> 1.74 (profiles/r02/dc_small_fields.txt).
#ifndef GFQ_SUS_DC_MINQ_DEFAULT
#define GFQ_SUS_DC_MINQ_DEFAULT 8
#endif
bool sus_dc_applies(const WaveArgs &a) {
  static int minq = -1;
  if (minq < 0) {
    const char *e = getenv("GFQ_SUS_DC_MINQ");
    minq = e ? atoi(e) : GFQ_SUS_DC_MINQ_DEFAULT;
    if (minq < 4) minq = 4;
  }
  return a.c.q >= minq && a.c.q <= 16 && a.c.max_cdeg <= 4 && a.c.max_vdeg <= 3;
}

int launch_sus_dc(const WaveArgs &a, int lb, int ncols, cudaStream_t s) {
  switch (a.c.q) {
    case 4: return a.markov ? dc_launch<4, true>(a, lb, ncols, s) : dc_launch<4, false>(a, lb, ncols, s);
    case 8: return a.markov ? dc_launch<8, true>(a, lb, ncols, s) : dc_launch<8, false>(a, lb, ncols, s);
    case 16: return a.markov ? dc_launch<16, true>(a, lb, ncols, s) : dc_launch<16, false>(a, lb, ncols, s);
    default: break;
  }
  set_error("k_sus_dc: unsupported q");
  return GFQ_EUNSUPPORTED;
}

}  // namespace gfq

// gfq_sus_dc64.cu -- the SUS level kernel for q = 64 by direct convolution:
// PAPER.md §2, SUS steps 1-4 with the check-node update Eq. (3)
// evaluated as the sum over configurations it is.
//
// Why.  The transform formulation of a SUS unit (gfq_bp.cu) needs fp64 (the
// inverse transform cancels O(1) terms into tiny probabilities) and, with the
// 64 entries of a message spread over 8 warps, one fp64 layout switch through
// shared memory per message: at q = 64 the kernel is bound by the shared-
// memory pipe and by instruction issue, not by HBM (profiles/r02).  The XOR-
// convolution S = u_1 (*) u_2 (*) u_3 of the permuted other messages is a sum
// of non-negative terms: fp32 keeps every entry to a relative ~q ulps (no
// cancellation), the multiply-adds go to the packed fp32 pipe (FFMA2, two per
// instruction), and nothing crosses a warp except the intermediate product of
// a degree-4 check (8 KB through the consumed input slot).
//
// Decomposition: a group of 4 warps owns a unit for its 32 frames (one frame
// per lane); warp c computes the 16 outputs y = 16c .. 16c+15.  With x = 16 xh
// + xl the XOR-convolution splits into 16 x 16 block convolutions:
//   S[16c + yl] = sum_xh sum_xl A[16 xh + xl] * B[16 (c ^ xh) + (yl ^ xl)],
// so the kernel loops over xh = 0..3 (run time) around ONE unrolled block
// convolution (128 FFMA2: the 8 accumulator pairs are kept twice, even and odd
// xl contribute to a pair in natural and swapped order) whose operands -- A
// block xh and B block c ^ xh, 16 values each -- are loaded from the stage by
// address, so every register index is a compile-time constant and the code
// stays a few KB (the first version, fully unrolled over all 64 x, spent 41 %
// of its cycles on instruction-cache misses: profiles/r02/dc64).
//   u_k(y) = q_ij_k(h_k^-1 y)             (rows chosen at load)
//   S(y)   = sum_x A(x) B(y ^ x)          (4 x 128 FFMA2 per thread and convolution)
//   r_ij(a) = S(z_i ^ h_ij a)             (Eq. 3; reading A4)
// The variable update (Eq. 4, posterior Eq. 5, clipping) is in fp64 as in the
// other kernels, streamed over the entries, 16 per warp, two passes.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>

#include "gfq_device.cuh"
#include "gfq_launch.cuh"

namespace gfq {

#ifndef GFQ_DC64_G
#define GFQ_DC64_G 4   // groups (of 2 warps) per CTA
#endif
#ifndef GFQ_DC64_S
#define GFQ_DC64_S 1   // TMA stages per group
#endif

constexpr int DQ = 64, DW = 4;   // field size, warps per group

template <int S, int G>
struct DC64Shape {
  static constexpr int XR = Extra<DQ, false>::rows;             // noise column: p per-bit rows
  static constexpr size_t PAY = (size_t)3 * DQ * 128;           // the d-1 <= 3 other messages
  static constexpr size_t RSM = (size_t)3 * DQ * 128;           // fp32 r of the column's <= 3 checks
  static constexpr size_t TSM_B = (size_t)2 * DQ * DQ;          // row-offset table (u16 q x q)
  using Sh = Shape<DQ, S, G, PAY, RSM, (size_t)XR * 128, TSM_B, false>;
  static constexpr size_t SMEM = Sh::SMEM;
  static constexpr int THREADS = G * DW * 32;
};

typedef unsigned long long u64;
__device__ __forceinline__ u64 pack2(float lo, float hi) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void unpack2(u64 v, float &lo, float &hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ void fma2(u64 &acc, u64 a, u64 b) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(a), "l"(b));
}
__device__ __forceinline__ void lds_v4(uint32_t addr, uint32_t (&w)[4]) {
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]) : "r"(addr) : "memory");
}

// 16 values of a message from a stage slot: entries y0 .. y0+15 (y0 a multiple
// of 16).  PERM: rows h^-1 y through the offset table (rt_row: shared address
// of rowtab[h^-1][0]); else natural rows.
template <bool PERM>
__device__ __forceinline__ void dc64_load16(uint32_t slot_lane, uint32_t rt_row, int y0, float (&v)[16]) {
  if constexpr (PERM) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      uint32_t w[4];
      lds_v4(rt_row + (uint32_t)(y0 * 2 + j * 16), w);
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        v[8 * j + 2 * t] = lds_f32(slot_lane + (w[t] & 0xffffu));
        v[8 * j + 2 * t + 1] = lds_f32(slot_lane + (w[t] >> 16));
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = lds_f32(slot_lane + (uint32_t)((y0 + k) * 128));
  }
}

// S(y) = sum_x A(x) B(y ^ x) for this warp's 16 outputs y = 16c + yl.
template <bool APERM, bool BPERM>
__device__ __forceinline__ void dc64_conv(uint32_t a_lane, uint32_t a_rt, uint32_t b_lane, uint32_t b_rt, int c,
                                          float (&s)[16]) {
  u64 an[8], as_[8];
#pragma unroll
  for (int ml = 0; ml < 8; ++ml) { an[ml] = 0ull; as_[ml] = 0ull; }
#pragma unroll 1
  for (int xh = 0; xh < 4; ++xh) {
    float av[16], bv[16];
    dc64_load16<APERM>(a_lane, a_rt, 16 * xh, av);
    dc64_load16<BPERM>(b_lane, b_rt, 16 * (c ^ xh), bv);
    u64 Bb[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) Bb[i] = pack2(bv[2 * i], bv[2 * i + 1]);
#pragma unroll
    for (int xl = 0; xl < 16; ++xl) {
      const u64 axx = pack2(av[xl], av[xl]);
#pragma unroll
      for (int ml = 0; ml < 8; ++ml) {
        // output pair ml of the block reads B pair ml ^ (xl >> 1)
        if (xl & 1) fma2(as_[ml], axx, Bb[ml ^ (xl >> 1)]);
        else fma2(an[ml], axx, Bb[ml ^ (xl >> 1)]);
      }
    }
  }
#pragma unroll
  for (int ml = 0; ml < 8; ++ml) {
    float n0, n1, s0, s1;
    unpack2(an[ml], n0, n1);
    unpack2(as_[ml], s0, s1);   // odd x: (B[2m'+1], B[2m']) feed (s[2m], s[2m+1])
    s[2 * ml] = n0 + s1;
    s[2 * ml + 1] = n1 + s0;
  }
}

// SUS step 1 for one check of the column (DO = min(d-1, 2): 2 stands for d-1 = 2 or 3), then q * r_ij
// into r slot ti.s of the group at row a = h^-1 y ^ h^-1 z.
template <int DO>
__device__ __forceinline__ void dc64_check(const WaveArgs &a, const unsigned char *hdr, uint32_t pay_lane, uint32_t rt,
                                           float *rsm, int g, int c, int lane, bool frozen, bool release,
                                           uint64_t *empty) {
  const TaskInfo ti = *(const TaskInfo *)hdr;
  const SusDesc *sd = (const SusDesc *)(hdr + 128);
  const int z = hdr[256 + lane];
  const unsigned long long pke = sd->perm_e;
  float S[16];
  if constexpr (DO == 0) {
    if (release) release_stage(empty, lane);
#pragma unroll
    for (int k = 0; k < 16; ++k) S[k] = (c == 0 && k == 0) ? 1.0f : 0.0f;   // the point mass at 0
  } else if constexpr (DO == 1) {
    dc64_load16<true>(pay_lane, rt + (uint32_t)((sd->perm_o[0] & 0xff) * DQ * 2), 16 * c, S);
    if (release) release_stage(empty, lane);
  } else {
    // DO = 2 or 3 (run time: one copy of each convolution body in the kernel)
    const uint32_t rt0 = rt + (uint32_t)((sd->perm_o[0] & 0xff) * DQ * 2);
    const uint32_t rt1 = rt + (uint32_t)((sd->perm_o[1] & 0xff) * DQ * 2);
    dc64_conv<true, true>(pay_lane + DQ * 128, rt1, pay_lane, rt0, c, S);   // A = message 1, B = message 0
    if (ti.d - 1 >= 3) {
      // the intermediate product goes to slot 0: every warp of the group must
      // be done reading message 0 before any of them overwrites it
      group_bar<DW>(g);
#pragma unroll
      for (int k = 0; k < 16; ++k)
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(pay_lane + (uint32_t)((16 * c + k) * 128)), "f"(S[k]) : "memory");
      const uint32_t rt2 = rt + (uint32_t)((sd->perm_o[2] & 0xff) * DQ * 2);
      group_bar<DW>(g);                                                     // the product is complete
      dc64_conv<false, true>(pay_lane, 0u, pay_lane + 2 * DQ * 128, rt2, c, S);   // A = the product, B = message 2
    }
    if (release) release_stage(empty, lane);
  }
  // r(a) = S(z ^ h a): S[y] goes to row a = h^-1 y ^ h^-1 z
  const uint32_t rte = rt + (uint32_t)((pke & 0xff) * DQ * 2);
  uint32_t hz;
  asm volatile("ld.shared.u16 %0, [%1];" : "=r"(hz) : "r"(rte + (uint32_t)(z * 2)));
  unsigned char *rs = (unsigned char *)(rsm + (size_t)ti.s * DQ * 32 + lane);
  unsigned char *rd = (a.rmsg != nullptr && !frozen)
                          ? (unsigned char *)(a.rmsg + ((size_t)ti.fb * a.c.E + ti.e0 + ti.s) * DQ * 32 + lane)
                          : nullptr;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    uint32_t w[4];
    lds_v4(rte + (uint32_t)(c * 32 + j * 16), w);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const uint32_t o0 = (w[t] & 0xffffu) ^ hz, o1 = (w[t] >> 16) ^ hz;
      const float v0 = S[8 * j + 2 * t] * (float)DQ, v1 = S[8 * j + 2 * t + 1] * (float)DQ;
      *(float *)(rs + o0) = v0;
      *(float *)(rs + o1) = v1;
      if (rd) {  // keep_messages only (export)
        *(float *)(rd + o0) = v0;
        *(float *)(rd + o1) = v1;
      }
    }
  }
}

// SUS step 2 (+ step 4, reading A8) for the column by the group's four warps:
// warp c takes entries 16c .. 16c+15 (two chunks of 8 for the prior).
template <int DV>
__device__ __forceinline__ void dc64_vn(const WaveArgs &a, const unsigned char *hdr, const unsigned char *xtra,
                                        const float *rsm, double *red, int g, int c, int lane, bool frozen) {
  constexpr int NS = DV + 1;
  const TaskInfo ti = *(const TaskInfo *)hdr;
  const VarDesc *vd = (const VarDesc *)(hdr + 192);
  const int fb = ti.fb, j = ti.item;
  const long long E = a.c.E;
  const float *R = rsm + lane;
  auto prods = [&](double p, int y, double (&o)[NS]) {
    double r[DV > 0 ? DV : 1];
#pragma unroll
    for (int t = 0; t < DV; ++t) r[t] = (double)R[(t * DQ + y) * 32];
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
#pragma unroll 1
  for (int u = 0; u < 2; ++u) {
    double pr[8];
    prior_from<DQ, 8, false>(a, j, 2 * c + u, lane, (const float *)xtra, nullptr, pr);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      double o[NS];
      prods(pr[k], (2 * c + u) * 8 + k, o);
#pragma unroll
      for (int t = 0; t < NS; ++t) sums[t] += o[t];
      mx = fmax(mx, o[DV]);
    }
  }
#pragma unroll
  for (int t = 0; t < NS; ++t) red[(t * DW + c) * 32 + lane] = sums[t];
  red[(NS * DW + c) * 32 + lane] = mx;
  group_bar<DW>(g);
#pragma unroll
  for (int t = 0; t < NS; ++t) {
    double v = red[(t * DW) * 32 + lane];
#pragma unroll
    for (int cc = 1; cc < DW; ++cc) v += red[(t * DW + cc) * 32 + lane];
    sums[t] = v;
  }
  mx = red[(NS * DW) * 32 + lane];
#pragma unroll
  for (int cc = 1; cc < DW; ++cc) mx = fmax(mx, red[(NS * DW + cc) * 32 + lane]);
  int bad = 0;
  double inv[NS];
  float add[NS];
#pragma unroll
  for (int t = 0; t < NS; ++t) {
    const bool ok = sums[t] > 0.0 && isfinite(sums[t]);
    bad += !ok;
    inv[t] = ok ? fast_rcp(sums[t]) : 0.0;
    add[t] = ok ? 0.0f : 1.0f / DQ;
  }
  const bool okq = add[DV] == 0.0f;
  const double thr = mx * (1.0 - kTieRel);   // clipping: smallest a within the tie band
  int bidx = DQ;
  float *qrow[DV > 0 ? DV : 1];
#pragma unroll
  for (int t = 0; t < DV; ++t) qrow[t] = a.qmsg + ((size_t)fb * E + vd->qdst[t]) * DQ * 32 + lane;
  float *qarow = a.qall ? a.qall + ((size_t)fb * a.c.V + j) * DQ * 32 + lane : nullptr;
#pragma unroll 1
  for (int u = 0; u < 2; ++u) {
    double pr[8];
    prior_from<DQ, 8, false>(a, j, 2 * c + u, lane, (const float *)xtra, nullptr, pr);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int y = (2 * c + u) * 8 + k;
      double o[NS];
      prods(pr[k], y, o);
      if (o[DV] >= thr && bidx == DQ) bidx = y;
      if (!frozen) {
#pragma unroll
        for (int t = 0; t < DV; ++t) qrow[t][y * 32] = (float)(o[t] * inv[t]) + add[t];
        if (qarow) qarow[y * 32] = (float)(o[DV] * inv[DV]) + add[DV];
      }
    }
  }
  int *ired = (int *)(red + (size_t)(NS + 1) * DW * 32);
  ired[c * 32 + lane] = bidx;
  group_bar<DW>(g);
  if (c == 0) {
#pragma unroll
    for (int cc = 1; cc < DW; ++cc) bidx = min(bidx, ired[cc * 32 + lane]);
    if (bidx >= DQ || !okq) bidx = 0;
    if (!frozen) {
      a.xhat[((size_t)fb * a.c.V + j) * 32 + lane] = (unsigned char)bidx;
      if (bad) atomicAdd(a.stats + 0, (unsigned long long)bad);
    }
  }
}

template <int S, int G>
__global__ void __launch_bounds__(DC64Shape<S, G>::THREADS) k_sus_dc64(WaveArgs a, int lvl_begin, int ncols) {
  using DS = DC64Shape<S, G>;
  using Sh = typename DS::Sh;
  extern __shared__ __align__(128) unsigned char smem[];
  const SmemPtrs sp = smem_ptrs<Sh, S, G>(smem);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = warp / DW, c = warp % DW;
  asm volatile("griddepcontrol.launch_dependents;");
  if (threadIdx.x == 0) init_bars<S, G>(sp.bars, DW);
  unsigned short *rtab = (unsigned short *)sp.tsm;
  for (int k = threadIdx.x; k < DQ * DQ; k += blockDim.x) rtab[k] = a.c.rowtab[k];
  const uint32_t rt = smem_u32(rtab);
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const long long ntask = (long long)(*a.nactive) * ncols;
  float *rsm = (float *)(sp.scr + (size_t)g * DS::RSM);
  const bool producer = (c == 0) && (lane == 0);
  long long lo, hi;
  sus_group_range(a, lvl_begin, ncols, (long long)(*a.nactive), (long long)blockIdx.x * G + g,
                  (long long)gridDim.x * G, lo, hi);
  UnitWalker pc;
  if (producer) pc.init(a, lo, hi, ncols, lvl_begin);
  auto issue_next = [&](int k) {
    if (!pc.valid()) return;
    const int fb = pc.fb;
    const LvlUnit un = pc.take(a);
    sus_issue_rec<DQ, false, false>(a, fb, un, sp.hdr + (size_t)k * kHdr, sp.pay + (size_t)k * Sh::PAYA,
                                    sp.xtra + (size_t)k * Sh::XTRA_A, sp.bars + k);
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
      const uint32_t pay_lane = sp.pay_u32 + (uint32_t)((size_t)k * Sh::PAYA) + lane * 4;
      uint64_t *empty = sp.bars + G * S + k;
      const int par = (rr / S) & 1;
      mbar_wait(sp.bars + k, (uint32_t)par);
      const TaskInfo *ti = (const TaskInfo *)hdr;
      const int dv = ti->deg, d = ti->d;
      nunits = dv > 0 ? dv : 1;
      const bool last = (s == nunits - 1);
      const bool frozen = a.early_exit && ((const int *)(hdr + 384))[lane] != 0;
      if (dv > 0) {
        switch (d - 1) {
          case 0: dc64_check<0>(a, hdr, pay_lane, rt, rsm, g, c, lane, frozen, !last, empty); break;
          case 1: dc64_check<1>(a, hdr, pay_lane, rt, rsm, g, c, lane, frozen, !last, empty); break;
          default: dc64_check<2>(a, hdr, pay_lane, rt, rsm, g, c, lane, frozen, !last, empty); break;
        }
      }
      if (last) {
        // the stage's payload is consumed: it holds the reduction scratch of the
        // variable update; the stage (VarDesc, prior rows) is released after it
        double *red = (double *)(sp.pay + (size_t)k * Sh::PAYA);
        group_bar<DW>(g);   // the column's r slots are complete, the payload is free
        switch (dv) {
          case 0: dc64_vn<0>(a, hdr, xtra, rsm, red, g, c, lane, frozen); break;
          case 1: dc64_vn<1>(a, hdr, xtra, rsm, red, g, c, lane, frozen); break;
          case 2: dc64_vn<2>(a, hdr, xtra, rsm, red, g, c, lane, frozen); break;
          default: dc64_vn<3>(a, hdr, xtra, rsm, red, g, c, lane, frozen); break;
        }
        release_stage(empty, lane);
      }
      if (producer && pc.valid()) {   // refill the stage once both warps have released it
        mbar_wait(empty, (uint32_t)par);
        issue_next(k);
      }
    }
  }
}

// q = 64, i.i.d. source, check degree <= 4, variable degree <= 3; switched by
// the environment variable GFQ_SUS_DC64 (default set at build time below).
#ifndef GFQ_SUS_DC64_DEFAULT
#define GFQ_SUS_DC64_DEFAULT 0
#endif
bool sus_dc64_applies(const WaveArgs &a) {
  static int on = -1;
  if (on < 0) {
    const char *e = getenv("GFQ_SUS_DC64");
    on = e ? (atoi(e) != 0) : GFQ_SUS_DC64_DEFAULT;
  }
  return on && a.c.q == DQ && !a.markov && a.c.max_cdeg <= 4 && a.c.max_vdeg <= 3;
}

int launch_sus_dc64(const WaveArgs &a, int lb, int ncols, cudaStream_t s) {
  constexpr int S = GFQ_DC64_S, G = GFQ_DC64_G;
  using DS = DC64Shape<S, G>;
  static_assert(DS::SMEM <= 232448, "k_sus_dc64: shared memory");
  auto k = k_sus_dc64<S, G>;
  const int grid = grid_for(k, DS::THREADS, DS::SMEM, ((long long)a.nfb * ncols + G - 1) / G);
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
  if (e != cudaSuccess) return cuda_fail(e, "k_sus_dc64");
  return check_launch("k_sus_dc64");
}

}  // namespace gfq

// gfq_bigq.cu -- the BP kernels for q = 256 (GF(2^8)): PUS check node and
// variable node, and the SUS level kernel.  PAPER.md §2 (Eqs. 3-5)
// is the authority for what is computed; the paper states the method for
// GF(q) in general.
//
// Why separate kernels.  A q = 256 message is 256 rows x 128 B = 32 KB per
// 32-frame block.  The kernels of gfq_bp.cu stage a whole task (d or d-1
// messages) per shared-memory stage and hold all of its q-vectors in fp64
// registers; at q = 256 one SUS unit would need 96 KB per stage plus 128 KB of
// fp64 transpose scratch (> 227 KB), and 3-4 vectors of 32 fp64 entries per
// thread exceed the register file.  Here one CTA of 8 warps owns a task and
// STREAMS the messages of a check one at a time: a message is read straight
// from HBM (rows of 128 B, fully coalesced; the coefficient permutation is the
// choice of row), transformed (Walsh-Hadamard over the 8 bits: 5 in registers,
// 3 after one fp64 layout switch through shared memory) and multiplied into a
// running product of 32 fp64 registers per thread.  For the check node every
// output edge repeats this over the other d-1 edges (the SUS unit; PUS calls
// it once per edge), so a thread never holds more than two vectors.  The
// variable node streams over the entries in chunks of 8 (two passes: sums,
// then normalised stores) with the prior chunk kept in registers.
//
// Layout, precision and conventions are those of gfq_bp.cu: one frame per
// lane, fp32 storage, fp64 arithmetic, stored r = q * r, negative round-off
// clamped to 0, clipping ties within kTieRel to the smallest symbol.
#include <cuda_runtime.h>
#include <stdint.h>

#include "gfq_device.cuh"
#include "gfq_launch.cuh"

namespace gfq {

constexpr int BQ = 256;           // field size
constexpr int BP = 8;             // bits
constexpr int BKR = 32;           // entries per thread
constexpr int BT = BQ / BKR;      // warps per CTA (one task per CTA)
constexpr int BTHREADS = BT * 32;
constexpr int BCH = 8;            // variable node: entries per chunk
constexpr int BNCH = BKR / BCH;   // chunks per thread
constexpr size_t BX_BYTES = (size_t)BQ * 32 * sizeof(double);   // layout-switch buffer
constexpr size_t BR_BYTES = (size_t)BQ * 32 * sizeof(float);    // one r slot (SUS)
constexpr int BDV_SUS = 3;        // SUS: the column's fresh r's live in shared memory

// ---------------------------------------------------------------- the check-node unit
// Eq. (3) for one edge e of check i from the CURRENT q's of the check's other
// edges (SUS step 1), in the transform domain:
//   U_k = WHT(q_k o h_k^-1),  r_e(a) = (1/q) WHT[(-1)^{w.z} prod_{k != e} U_k](h_e a).
// `skip` is the position of e in the check's row [r0, r0 + d).  Writes q * r_e
// (natural order a, clamped at 0) to dst[a*32 + lane] (shared or global) and,
// when dst2 != null, there as well.  X: the CTA's fp64 layout-switch buffer.
__device__ __forceinline__ void big_unit(const WaveArgs &a, int fb, int r0, int d, int skip, int z, double *X,
                                         float *dst, float *dst2, int c, int lane) {
  double acc[BKR];
#pragma unroll
  for (int k = 0; k < BKR; ++k) acc[k] = 1.0;   // no other edge: the transform of the point mass at 0
  bool first = true;
#pragma unroll 1
  for (int t = 0; t < d; ++t) {
    if (t == skip) continue;
    const int e = r0 + t;
    const unsigned hinv = (unsigned)(__ldg(a.c.edge_perm + e) & 0xff);
    const unsigned short *rt = a.c.rowtab + (size_t)hinv * BQ + c * BKR;   // (h^-1 y) << 7 for y = c*32 + k
    const unsigned char *src = (const unsigned char *)(a.qmsg + ((size_t)fb * a.c.E + e) * BQ * 32 + lane);
    double v[BKR];
#pragma unroll
    for (int k = 0; k < BKR; ++k) v[k] = (double)__ldcs((const float *)(src + __ldg(rt + k)));
    wht_bits<BKR, 0, 5>(v);
#pragma unroll
    for (int k = 0; k < BKR; ++k) X[(c * BKR + k) * 32 + lane] = v[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < BKR; ++k) v[k] = X[(k * BT + c) * 32 + lane];
    __syncthreads();
    wht_bits<BKR, 2, 5>(v);
    if (first) {
#pragma unroll
      for (int k = 0; k < BKR; ++k) acc[k] = v[k];
      first = false;
    } else {
#pragma unroll
      for (int k = 0; k < BKR; ++k) acc[k] *= v[k];
    }
  }
  // syndrome sign at frequency w = k*BT + c (reading A4), inverse transform
#pragma unroll
  for (int k = 0; k < BKR; ++k) acc[k] = flip(acc[k], (uint32_t)(__popc((k * BT + c) & z) & 1) << 31);
  wht_bits<BKR, 2, 5>(acc);
#pragma unroll
  for (int k = 0; k < BKR; ++k) X[(k * BT + c) * 32 + lane] = acc[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < BKR; ++k) acc[k] = X[(c * BKR + k) * 32 + lane];
  __syncthreads();
  wht_bits<BKR, 0, 5>(acc);
  const unsigned hinv = (unsigned)(__ldg(a.c.edge_perm + r0 + skip) & 0xff);
  const unsigned short *rt = a.c.rowtab + (size_t)hinv * BQ + c * BKR;     // a = h_e^-1 y
#pragma unroll
  for (int k = 0; k < BKR; ++k) {
    const float val = fmaxf((float)acc[k], 0.0f);
    const unsigned off = __ldg(rt + k);
    if (dst) *(float *)((unsigned char *)(dst + lane) + off) = val;
    if (dst2) *(float *)((unsigned char *)(dst2 + lane) + off) = val;
  }
}

// ---------------------------------------------------------------- the variable node
// Eqs. (4), (5) and clipping for variable j of block fb from its DV
// incoming messages rp[s][a*32 + lane] (shared or global, any positive scale).
// Warp c takes the chunks of 8 entries cc = c, c + 8, c + 16, c + 24.
template <int DV>
__device__ __forceinline__ void big_prods(const double p, const double (&r)[DV > 0 ? DV : 1], double (&o)[DV + 1]) {
  if constexpr (DV == 0) {
    o[0] = p;
  } else {
    double pre[DV];
    double acc = p;
#pragma unroll
    for (int s = 0; s < DV; ++s) {
      pre[s] = acc;
      acc *= r[s];
    }
    o[DV] = acc;
    acc = 1.0;
#pragma unroll
    for (int s = DV - 1; s >= 0; --s) {
      o[s] = pre[s] * acc;
      acc *= r[s];
    }
  }
}

template <int DV, bool MARKOV>
__device__ __forceinline__ void big_vn(const WaveArgs &a, int fb, int j, const float *const *rp, const int *qdst,
                                       double *red, int c, int lane, bool frozen) {
  constexpr int NS = DV + 1;
  const int N = a.c.N;
  // the prior of this thread's 32 entries, chunk by chunk (prior_from)
  double pr[BNCH][BCH];
  {
    const float *ex = nullptr, *exr = nullptr;
    if (j >= N) {
      ex = a.pi + ((size_t)fb * a.c.M * BP + (size_t)(j - N) * BP) * 32;
    } else if (MARKOV) {
      const int nb = markov_nbrs(a, j);
      const float *l = (nb & 1) ? (a.gs ? a.qs_new : a.qs_old) + ((size_t)fb * N + (j - 1)) * BQ * 32 : nullptr;
      const float *r = (nb & 2) ? a.qs_old + ((size_t)fb * N + (j + 1)) * BQ * 32 : nullptr;
      ex = l ? l : r;
      exr = r ? r : l;
    }
#pragma unroll
    for (int u = 0; u < BNCH; ++u) prior_from<BQ, BCH, MARKOV>(a, j, c + u * BT, lane, ex, a.Tf, pr[u], exr);
  }
  double sums[NS], mx = 0.0;
#pragma unroll
  for (int s = 0; s < NS; ++s) sums[s] = 0.0;
#pragma unroll
  for (int u = 0; u < BNCH; ++u) {
#pragma unroll
    for (int k = 0; k < BCH; ++k) {
      const int y = (c + u * BT) * BCH + k;
      double r[DV > 0 ? DV : 1], o[NS];
#pragma unroll
      for (int s = 0; s < DV; ++s) r[s] = (double)rp[s][y * 32 + lane];
      big_prods<DV>(pr[u][k], r, o);
#pragma unroll
      for (int s = 0; s < NS; ++s) sums[s] += o[s];
      mx = fmax(mx, o[DV]);
    }
  }
  // cross-warp totals
#pragma unroll
  for (int s = 0; s < NS; ++s) red[(s * BT + c) * 32 + lane] = sums[s];
  red[(NS * BT + c) * 32 + lane] = mx;
  __syncthreads();
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    double v = red[(s * BT) * 32 + lane];
#pragma unroll
    for (int cc = 1; cc < BT; ++cc) v += red[(s * BT + cc) * 32 + lane];
    sums[s] = v;
  }
  mx = red[(NS * BT) * 32 + lane];
#pragma unroll
  for (int cc = 1; cc < BT; ++cc) mx = fmax(mx, red[(NS * BT + cc) * 32 + lane]);
  int bad = 0;
  double inv[NS];
  float add[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const bool ok = sums[s] > 0.0 && isfinite(sums[s]);
    bad += !ok;
    inv[s] = ok ? fast_rcp(sums[s]) : 0.0;
    add[s] = ok ? 0.0f : 1.0f / BQ;
  }
  const bool okq = add[DV] == 0.0f;
  const double thr = mx * (1.0 - kTieRel);   // clipping, reading A17
  int bidx = BQ;
  float *qs = (MARKOV && j < N && a.qs_new) ? a.qs_new + ((size_t)fb * N + j) * BQ * 32 + lane : nullptr;
  float *qa = a.qall ? a.qall + ((size_t)fb * a.c.V + j) * BQ * 32 + lane : nullptr;
#pragma unroll
  for (int u = BNCH - 1; u >= 0; --u) {
#pragma unroll
    for (int k = BCH - 1; k >= 0; --k) {
      const int y = (c + u * BT) * BCH + k;
      double r[DV > 0 ? DV : 1], o[NS];
#pragma unroll
      for (int s = 0; s < DV; ++s) r[s] = (double)rp[s][y * 32 + lane];
      big_prods<DV>(pr[u][k], r, o);
      if (o[DV] >= thr) bidx = y;            // descending y: ends at the smallest
      if (!frozen) {
#pragma unroll
        for (int s = 0; s < DV; ++s)
          a.qmsg[((size_t)fb * a.c.E + qdst[s]) * BQ * 32 + y * 32 + lane] = (float)(o[s] * inv[s]) + add[s];
        const float qv = (float)(o[DV] * inv[DV]) + add[DV];
        if (qs) qs[y * 32] = qv;
        if (qa) qa[y * 32] = qv;
      }
    }
  }
  int *ired = (int *)(red + (size_t)(NS + 1) * BT * 32);
  ired[c * 32 + lane] = bidx;
  __syncthreads();
  if (c == 0) {
#pragma unroll
    for (int cc = 1; cc < BT; ++cc) bidx = min(bidx, ired[cc * 32 + lane]);
    if (bidx >= BQ || !okq) bidx = 0;
    if (!frozen) {
      a.xhat[((size_t)fb * a.c.V + j) * 32 + lane] = (unsigned char)bidx;
      if (bad) atomicAdd(a.stats + 0, (unsigned long long)bad);
    }
  }
  __syncthreads();   // red / the r slots may be rewritten by the next task
}

template <bool MARKOV, int MAXDV>
__device__ __forceinline__ void big_vn_dispatch(const WaveArgs &a, int fb, int j, int dv, const float *const *rp,
                                                const int *qdst, double *red, int c, int lane, bool frozen) {
  if constexpr (MAXDV <= 3) {
    switch (dv) {
      case 0: big_vn<0, MARKOV>(a, fb, j, rp, qdst, red, c, lane, frozen); break;
      case 1: big_vn<1, MARKOV>(a, fb, j, rp, qdst, red, c, lane, frozen); break;
      case 2: big_vn<2, MARKOV>(a, fb, j, rp, qdst, red, c, lane, frozen); break;
      default: big_vn<3, MARKOV>(a, fb, j, rp, qdst, red, c, lane, frozen); break;
    }
    return;
  }
  switch (dv) {
    case 0: big_vn<0, MARKOV>(a, fb, j, rp, qdst, red, c, lane, frozen); break;
    case 1: big_vn<1, MARKOV>(a, fb, j, rp, qdst, red, c, lane, frozen); break;
    case 2: big_vn<2, MARKOV>(a, fb, j, rp, qdst, red, c, lane, frozen); break;
    case 3: big_vn<3, MARKOV>(a, fb, j, rp, qdst, red, c, lane, frozen); break;
    case 4: big_vn<4, MARKOV>(a, fb, j, rp, qdst, red, c, lane, frozen); break;
    case 5: big_vn<5, MARKOV>(a, fb, j, rp, qdst, red, c, lane, frozen); break;
    case 6: big_vn<6, MARKOV>(a, fb, j, rp, qdst, red, c, lane, frozen); break;
    case 7: big_vn<7, MARKOV>(a, fb, j, rp, qdst, red, c, lane, frozen); break;
    default: big_vn<8, MARKOV>(a, fb, j, rp, qdst, red, c, lane, frozen); break;
  }
}

// ---------------------------------------------------------------- PUS kernels
// Horizontal pass: one CTA per (check, 32-frame block).
__global__ void __launch_bounds__(BTHREADS) k_big_cn(WaveArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  double *X = (double *)smem;
  const int lane = threadIdx.x & 31, c = threadIdx.x >> 5;
  const int M = a.c.M;
  const long long ntask = (long long)(*a.nactive) * M;
  for (long long task = blockIdx.x; task < ntask; task += gridDim.x) {
    const int fb = a.list[task / M], i = (int)(task % M);
    const int r0 = __ldg(a.c.row_ptr + i), d = __ldg(a.c.row_ptr + i + 1) - r0;
    const int z = a.z[((size_t)fb * M + i) * 32 + lane];
    const bool frozen = a.early_exit && a.conv[fb * 32 + lane] != 0;
    for (int t = 0; t < d; ++t) {
      float *dst = a.rmsg + ((size_t)fb * a.c.E + __ldg(a.c.edge_canon + r0 + t)) * BQ * 32;
      big_unit(a, fb, r0, d, t, z, X, frozen ? nullptr : dst, nullptr, c, lane);
    }
  }
}

// Vertical pass: one CTA per (variable, block); clip_only: the
// clipped priors x^(0) (no incoming message).
template <bool MARKOV>
__global__ void __launch_bounds__(BTHREADS) k_big_vn(WaveArgs a, int clip_only) {
  extern __shared__ __align__(128) unsigned char smem[];
  double *red = (double *)smem;
  const int lane = threadIdx.x & 31, c = threadIdx.x >> 5;
  const int V = a.c.V;
  const long long ntask = (long long)(*a.nactive) * V;
  for (long long task = blockIdx.x; task < ntask; task += gridDim.x) {
    const int fb = a.list[task / V], j = (int)(task % V);
    const int e0 = __ldg(a.c.col_ptr + j);
    const int dv = clip_only ? 0 : __ldg(a.c.col_ptr + j + 1) - e0;
    const bool frozen = a.early_exit && a.conv[fb * 32 + lane] != 0;
    const float *rp[kMaxDeg];
    int qdst[kMaxDeg];
#pragma unroll
    for (int s = 0; s < kMaxDeg; ++s) {
      rp[s] = a.rmsg + ((size_t)fb * a.c.E + e0 + (s < dv ? s : 0)) * BQ * 32;   // canonical order
      qdst[s] = s < dv ? __ldg(a.c.col_edge + e0 + s) : 0;
    }
    big_vn_dispatch<MARKOV, kMaxDeg>(a, fb, j, dv, rp, qdst, red, c, lane, frozen);
  }
}

// ---------------------------------------------------------------- SUS level kernel
// One CTA per (column of the level, block): step 1 for each check of the
// column (the unit, into the CTA's r slots), then steps 2 and 4.
template <bool MARKOV>
__global__ void __launch_bounds__(BTHREADS) k_big_sus(WaveArgs a, int lvl_begin, int ncols) {
  extern __shared__ __align__(128) unsigned char smem[];
  double *X = (double *)smem;
  float *rsm = (float *)(smem + BX_BYTES);
  const int lane = threadIdx.x & 31, c = threadIdx.x >> 5;
  const long long ntask = (long long)(*a.nactive) * ncols;
  for (long long task = blockIdx.x; task < ntask; task += gridDim.x) {
    const int fb = a.list[task / ncols];
    const LvlCol lc = a.c.lvl_col[lvl_begin + (int)(task % ncols)];
    const int j = lc.j, dv = lc.dv;
    const bool frozen = a.early_exit && a.conv[fb * 32 + lane] != 0;
    const float *rp[kMaxDeg];
    int qdst[kMaxDeg];
#pragma unroll
    for (int s = 0; s < kMaxDeg; ++s) {
      rp[s] = rsm + (size_t)(s < BDV_SUS ? s : 0) * BQ * 32;
      qdst[s] = 0;
    }
    for (int s = 0; s < dv; ++s) {
      const int e = __ldg(a.c.col_edge + lc.e0 + s);          // check-major id of the column's s-th edge
      const int i = __ldg(a.c.edge_check + e);
      const int r0 = __ldg(a.c.row_ptr + i), d = __ldg(a.c.row_ptr + i + 1) - r0;
      const int z = a.z[((size_t)fb * a.c.M + i) * 32 + lane];
      qdst[s] = e;
      float *keep = (a.rmsg != nullptr && !frozen) ? a.rmsg + ((size_t)fb * a.c.E + lc.e0 + s) * BQ * 32 : nullptr;
      big_unit(a, fb, r0, d, e - r0, z, X, rsm + (size_t)s * BQ * 32, keep, c, lane);
    }
    __syncthreads();   // the column's r slots are complete
    big_vn_dispatch<MARKOV, BDV_SUS>(a, fb, j, dv < BDV_SUS ? dv : BDV_SUS, rp, qdst, X, c, lane, frozen);
  }
}

// ---------------------------------------------------------------- launchers
template <typename K>
static int big_grid(K k, size_t smem, long long tasks) {
  return grid_for(k, BTHREADS, smem, tasks);
}

bool big_applies(const WaveArgs &a) { return a.c.q == BQ; }

int launch_big_cn(const WaveArgs &a, cudaStream_t s) {
  const int grid = big_grid(k_big_cn, BX_BYTES, (long long)a.nfb * a.c.M);
  k_big_cn<<<grid, BTHREADS, BX_BYTES, s>>>(a);
  return check_launch("k_big_cn");
}

int launch_big_vn(const WaveArgs &a, int clip_only, cudaStream_t s) {
  const size_t smem = (size_t)(kMaxDeg + 3) * BT * 32 * sizeof(double);
  if (a.markov) {
    const int grid = big_grid(k_big_vn<true>, smem, (long long)a.nfb * a.c.V);
    k_big_vn<true><<<grid, BTHREADS, smem, s>>>(a, clip_only);
  } else {
    const int grid = big_grid(k_big_vn<false>, smem, (long long)a.nfb * a.c.V);
    k_big_vn<false><<<grid, BTHREADS, smem, s>>>(a, clip_only);
  }
  return check_launch("k_big_vn");
}

int launch_big_sus(const WaveArgs &a, int lb, int ncols, cudaStream_t s) {
  if (a.c.max_vdeg > BDV_SUS) {
    set_error("q = 256 SUS: variable degree > 3 does not fit in shared memory (r slots of 32 KB each)");
    return GFQ_EUNSUPPORTED;
  }
  const size_t smem = BX_BYTES + (size_t)BDV_SUS * BR_BYTES;
  if (a.markov) {
    const int grid = big_grid(k_big_sus<true>, smem, (long long)a.nfb * ncols);
    k_big_sus<true><<<grid, BTHREADS, smem, s>>>(a, lb, ncols);
  } else {
    const int grid = big_grid(k_big_sus<false>, smem, (long long)a.nfb * ncols);
    k_big_sus<false><<<grid, BTHREADS, smem, s>>>(a, lb, ncols);
  }
  return check_launch("k_big_sus");
}

}  // namespace gfq

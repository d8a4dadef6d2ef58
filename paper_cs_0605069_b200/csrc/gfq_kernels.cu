// gfq_kernels.cu -- the hot path of BP decoding of MN codes over GF(2^p) on
// sm_100a.  PAPER.md §2 is the authority for what is computed;
// DESIGN.md explains how it is mapped onto the B200.
//
// Work decomposition (all kernels): one frame per lane, 32 frames per block;
// a "group" of T = max(1, q/8) warps owns one task (a check, a variable or a
// SUS column of one 32-frame block) and each thread holds KR = q/T entries of
// every q-vector it touches.  Two element layouts are used inside a group:
//   layout A: thread (warp c, register k) holds entry y = c*KR + k
//   layout B: thread (warp c, register k) holds entry y = k*T  + c
// The Walsh-Hadamard transform over the bits of y done "in registers" in
// layout A covers bits 0..log2(KR)-1, in layout B the remaining high bits;
// switching layouts is a shared-memory transpose (fp64, conflict free: every
// warp access is 32 consecutive lanes of one row).
//
// Precision: messages are stored in fp32 (the HBM bytes); every transform,
// leave-one-out product, prior and normalisation is computed in fp64 in
// registers, so tiny probabilities produced by cancellation in the inverse
// transform keep their relative accuracy.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <mutex>
#include <unordered_map>

#include "gfq_internal.cuh"

namespace gfq {

// Relative tolerance under which two posterior values count as a tie in the
// clipping step (reading A17; the oracle applies the same rule).
constexpr double kTieRel = 1e-5;

// ============================================================== configuration
template <int Q>
struct QC {
  static constexpr int P = Q == 2 ? 1 : Q == 4 ? 2 : Q == 8 ? 3 : Q == 16 ? 4 : Q == 32 ? 5 : 6;
  static constexpr int T = Q >= 16 ? Q / 8 : 1;  // warps per task group
  static constexpr int KR = Q / T;               // entries per thread
  static constexpr int LKR = KR == 2 ? 1 : KR == 4 ? 2 : 3;
  static constexpr int LT = P - LKR;
  static constexpr int G = T == 1 ? 4 : (T == 2 ? 2 : 1);  // groups per CTA
  static constexpr int THREADS = G * T * 32;
};

template <int T>
__device__ __forceinline__ void group_bar(int g) {
  if constexpr (T == 1) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "r"(T * 32) : "memory");
  }
}

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

// Row of entry y = c*KR + k under the GF(2)-linear map y -> h^-1 y, given
// the images of the basis vectors (bb[b] = h^-1 * 2^b).
template <int P>
__device__ __forceinline__ void unpack_basis(unsigned long long pk, int (&bb)[P]) {
#pragma unroll
  for (int b = 0; b < P; ++b) bb[b] = (int)((pk >> (8 * b)) & 0xff);
}
template <int P, int LKR>
__device__ __forceinline__ int row_hi(const int (&bb)[P], int c) {  // contribution of c*KR
  int r = 0;
#pragma unroll
  for (int b = LKR; b < P; ++b)
    if ((c >> (b - LKR)) & 1) r ^= bb[b];
  return r;
}
template <int P, int LKR>
__device__ __forceinline__ int row_lo(const int (&bb)[P], int k) {  // contribution of k
  int r = 0;
#pragma unroll
  for (int b = 0; b < LKR; ++b)
    if ((k >> b) & 1) r ^= bb[b];
  return r;
}

// Early exit freezes a converged frame: its lane keeps computing (warp-uniform
// control flow) but stores nothing.  Invalid lanes of a ragged last block are
// marked converged from the start.
__device__ __forceinline__ bool lane_frozen(const WaveArgs &a, int fb, int lane) {
  return a.early_exit && a.conv[fb * 32 + lane] != 0;
}

__device__ __forceinline__ double neg_if(double v, int s) {
  return __longlong_as_double(__double_as_longlong(v) ^ ((long long)s << 63));
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
// Prior p_j^a for the KR entries a = c*KR + k (layout A) of this thread.
//  - noise symbol j = N + m: prod_b (bit_b(a) ? pi_b : 1 - pi_b)
//  - source symbol, i.i.d. or first iteration: pi0(a)
//  - source symbol, Markov, iteration t >= 2: Eq. (7) from the
//    posterior snapshot Q^(t-1) of the neighbours (reading A9), boundaries A10:
//      p(b) = [sum_a Q_{j-1}(a) T_ab] * [sum_c T_bc Q_{j+1}(c)]
template <int Q, bool MARKOV>
__device__ __forceinline__ void load_prior(const WaveArgs &a, int fb, int j, int c, int lane,
                                           bool first_iter, double (&pr)[QC<Q>::KR]) {
  using C = QC<Q>;
  constexpr int KR = C::KR, P = C::P;
  const int N = a.c.N;
  if (j >= N) {
    const int m = j - N;
    const size_t Mp = (size_t)a.c.M * P;
    double pb[P];
#pragma unroll
    for (int b = 0; b < P; ++b) pb[b] = (double)a.pi[((size_t)fb * Mp + (size_t)m * P + b) * 32 + lane];
    double hi = 1.0;
#pragma unroll
    for (int b = C::LKR; b < P; ++b) hi *= ((c >> (b - C::LKR)) & 1) ? pb[b] : 1.0 - pb[b];
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      double v = hi;
#pragma unroll
      for (int b = 0; b < C::LKR; ++b) v *= ((k >> b) & 1) ? pb[b] : 1.0 - pb[b];
      pr[k] = v;
    }
    return;
  }
  if (!MARKOV || first_iter || a.qs_old == nullptr) {
#pragma unroll
    for (int k = 0; k < KR; ++k) pr[k] = __ldg(a.pi0 + c * KR + k);
    return;
  }
  double L[KR], R[KR];
  if (j > 0) {
#pragma unroll
    for (int k = 0; k < KR; ++k) L[k] = 0.0;
    const float *src = a.qs_old + ((size_t)fb * N + (j - 1)) * Q * 32 + lane;
#pragma unroll 4
    for (int x = 0; x < Q; ++x) {
      const double qv = (double)src[x * 32];
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
    const float *src = a.qs_old + ((size_t)fb * N + (j + 1)) * Q * 32 + lane;
#pragma unroll 4
    for (int x = 0; x < Q; ++x) {
      const double qv = (double)src[x * 32];
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
// smallest maximising a (reading A17).  r[s][k] holds r of check slot s at
// a = c*KR + k.  Writes the dv q messages, x_hat, and (Markov) Q snapshot,
// (keep) Q of every variable.  red: group scratch of (DVMAX+2)*T*32 doubles.
template <int Q, int DVMAX, bool MARKOV>
__device__ __forceinline__ void vn_body(const WaveArgs &a, int fb, int j, int e0, int dv,
                                        double (&r)[DVMAX][QC<Q>::KR], double *red, int g,
                                        int c, int lane, bool frozen) {
  using C = QC<Q>;
  constexpr int KR = C::KR, T = C::T;
  const long long E = a.c.E;
  double pr[KR];
  load_prior<Q, MARKOV>(a, fb, j, c, lane, a.t <= 1, pr);
  // Q numerator, then the dv leave-one-out numerators (in place in r)
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
  // Clipping: the smallest a whose Q is within kTieRel of the maximum
  // (reading A17: ties -> smallest a; values equal up to round-off are ties).
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
// Eq. (3) for every edge of check i (horizontal pass),
// in the transform domain (BASELINE.json north_star): with u_k(y) =
// q_ij_k(h_k^-1 y) (the distribution of h_k x_k), U_k = WHT(u_k),
//   r_ij_k(a) = (1/q) WHT[ (-1)^{w.z_i} prod_{k' != k} U_k'(w) ](h_k a).
// The syndrome enters as the sign (-1)^{popc(w & z_i)} (XOR shift by z_i,
// reading A4).  Negative round-off is clamped to 0 (reading A20).
template <int Q, int DMAX>
__global__ void __launch_bounds__(QC<Q>::THREADS) k_cn(WaveArgs a) {
  using C = QC<Q>;
  constexpr int T = C::T, KR = C::KR, LKR = C::LKR, LT = C::LT, P = C::P, G = C::G;
  extern __shared__ __align__(16) double smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = warp / T, c = warp % T;
  double *sm = smem + (size_t)g * DMAX * Q * 32;
  const int M = a.c.M;
  const long long E = a.c.E;
  const long long ntask = (long long)(*a.nactive) * M;
  for (long long task = (long long)blockIdx.x * G + g; task < ntask; task += (long long)gridDim.x * G) {
    const int fb = a.list[task / M];
    const int i = (int)(task % M);
    const int e0 = __ldg(a.c.row_ptr + i), d = __ldg(a.c.row_ptr + i + 1) - e0;
    const int z = a.z[((size_t)fb * M + i) * 32 + lane];
    double u[DMAX][KR];
    int bb[DMAX][P];
    int rc[DMAX];
#pragma unroll
    for (int s = 0; s < DMAX; ++s) {
      if (s < d) {
        unpack_basis<P>(__ldg(a.c.edge_perm + e0 + s), bb[s]);
        rc[s] = row_hi<P, LKR>(bb[s], c);
        const float *src = a.qmsg + ((size_t)fb * E + e0 + s) * Q * 32 + lane;
#pragma unroll
        for (int k = 0; k < KR; ++k) u[s][k] = (double)__ldg(src + (rc[s] ^ row_lo<P, LKR>(bb[s], k)) * 32);
      }
    }
#pragma unroll
    for (int s = 0; s < DMAX; ++s)
      if (s < d) wht_bits<KR, 0, LKR>(u[s]);
    if constexpr (T > 1) {
#pragma unroll
      for (int s = 0; s < DMAX; ++s)
        if (s < d)
#pragma unroll
          for (int k = 0; k < KR; ++k) sm[((size_t)s * Q + c * KR + k) * 32 + lane] = u[s][k];
      group_bar<T>(g);
#pragma unroll
      for (int s = 0; s < DMAX; ++s)
        if (s < d) {
#pragma unroll
          for (int k = 0; k < KR; ++k) u[s][k] = sm[((size_t)s * Q + k * T + c) * 32 + lane];
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
          for (int k = 0; k < KR; ++k) sm[((size_t)s * Q + k * T + c) * 32 + lane] = u[s][k];
      group_bar<T>(g);
#pragma unroll
      for (int s = 0; s < DMAX; ++s)
        if (s < d)
#pragma unroll
          for (int k = 0; k < KR; ++k) u[s][k] = sm[((size_t)s * Q + c * KR + k) * 32 + lane];
      group_bar<T>(g);
    }
    constexpr double invq = 1.0 / Q;
    const bool frozen = lane_frozen(a, fb, lane);
#pragma unroll
    for (int s = 0; s < DMAX; ++s) {
      if (s < d && !frozen) {
        wht_bits<KR, 0, LKR>(u[s]);
        float *dst = a.rmsg + ((size_t)fb * E + e0 + s) * Q * 32 + lane;
#pragma unroll
        for (int k = 0; k < KR; ++k) {
          const double v = u[s][k] * invq;
          dst[(rc[s] ^ row_lo<P, LKR>(bb[s], k)) * 32] = (float)(v > 0.0 ? v : 0.0);
        }
      }
    }
  }
}

// ============================================================== PUS: variable node
template <int Q, int DVMAX, bool MARKOV>
__global__ void __launch_bounds__(QC<Q>::THREADS) k_vn(WaveArgs a, int clip_only) {
  using C = QC<Q>;
  constexpr int T = C::T, KR = C::KR, G = C::G;
  extern __shared__ __align__(16) double smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = warp / T, c = warp % T;
  double *red = smem + (size_t)g * (DVMAX + 3) * T * 32;
  const int V = a.c.V;
  const long long E = a.c.E;
  const long long ntask = (long long)(*a.nactive) * V;
  for (long long task = (long long)blockIdx.x * G + g; task < ntask; task += (long long)gridDim.x * G) {
    const int fb = a.list[task / V];
    const int j = (int)(task % V);
    const int e0 = __ldg(a.c.col_ptr + j);
    const int dv = clip_only ? 0 : __ldg(a.c.col_ptr + j + 1) - e0;
    double r[DVMAX][KR];
#pragma unroll
    for (int s = 0; s < DVMAX; ++s) {
      if (s < dv) {
        const int e = __ldg(a.c.col_edge + e0 + s);
        const float *src = a.rmsg + ((size_t)fb * E + e) * Q * 32 + lane;
#pragma unroll
        for (int k = 0; k < KR; ++k) r[s][k] = (double)__ldg(src + (c * KR + k) * 32);
      }
    }
    vn_body<Q, DVMAX, MARKOV>(a, fb, j, e0, dv, r, red, g, c, lane, lane_frozen(a, fb, lane));
    if constexpr (T > 1) group_bar<T>(g);
  }
}

// ============================================================== SUS: one dependency level
// For every column j of the level (SUS step 1): r_ij for each
// check i of column j from the CURRENT q's of check i's other edges (Eq. 3,
// same transform as k_cn restricted to one output); then (step 2)
// the vertical update of column j (Eq. 4) and its posterior (step 4, A8).
// Columns of one level share no check, so they run concurrently with exactly
// the reads of the serial sweep.
template <int Q, int DMAX, int DVMAX, bool MARKOV>
__global__ void __launch_bounds__(QC<Q>::THREADS) k_sus(WaveArgs a, int lvl_begin, int ncols) {
  using C = QC<Q>;
  constexpr int T = C::T, KR = C::KR, LKR = C::LKR, LT = C::LT, P = C::P, G = C::G;
  constexpr int DO = DMAX - 1;  // other edges of a check
  extern __shared__ __align__(16) double smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = warp / T, c = warp % T;
  constexpr size_t fwd_sz = (T > 1) ? (size_t)DO * Q * 32 : 0;
  constexpr size_t acc_sz = (T > 1) ? (size_t)Q * 32 : 0;
  constexpr size_t red_sz = (size_t)(DVMAX + 3) * T * 32;
  constexpr size_t rsm_sz = (size_t)DVMAX * Q * 32 / 2;  // floats, in doubles
  constexpr size_t per_group = fwd_sz + acc_sz + red_sz + rsm_sz;
  double *fwd = smem + (size_t)g * per_group;
  double *accs = fwd + fwd_sz;
  double *red = accs + acc_sz;
  float *rsm = (float *)(red + red_sz);
  const int M = a.c.M;
  const long long E = a.c.E;
  const long long ntask = (long long)(*a.nactive) * ncols;
  for (long long task = (long long)blockIdx.x * G + g; task < ntask; task += (long long)gridDim.x * G) {
    const int fb = a.list[task / ncols];
    const int j = __ldg(a.c.level_cols + lvl_begin + (int)(task % ncols));
    const int e0 = __ldg(a.c.col_ptr + j), dv = __ldg(a.c.col_ptr + j + 1) - e0;
#pragma unroll 1
    for (int s = 0; s < DVMAX; ++s) {
      if (s >= dv) break;
      const int e = __ldg(a.c.col_edge + e0 + s);
      const int i = __ldg(a.c.edge_check + e);
      const int r0 = __ldg(a.c.row_ptr + i), d = __ldg(a.c.row_ptr + i + 1) - r0;
      const int pos = e - r0;
      const int z = a.z[((size_t)fb * M + i) * 32 + lane];
      double u[DO > 0 ? DO : 1][KR];
#pragma unroll
      for (int t = 0; t < DO; ++t) {
        if (t < d - 1) {
          const int ee = r0 + (t < pos ? t : t + 1);
          int bb[P];
          unpack_basis<P>(__ldg(a.c.edge_perm + ee), bb);
          const int rch = row_hi<P, LKR>(bb, c);
          const float *src = a.qmsg + ((size_t)fb * E + ee) * Q * 32 + lane;
#pragma unroll
          for (int k = 0; k < KR; ++k) u[t][k] = (double)src[(rch ^ row_lo<P, LKR>(bb, k)) * 32];
        }
      }
#pragma unroll
      for (int t = 0; t < DO; ++t)
        if (t < d - 1) wht_bits<KR, 0, LKR>(u[t]);
      if constexpr (T > 1) {
#pragma unroll
        for (int t = 0; t < DO; ++t)
          if (t < d - 1)
#pragma unroll
            for (int k = 0; k < KR; ++k) fwd[((size_t)t * Q + c * KR + k) * 32 + lane] = u[t][k];
        group_bar<T>(g);
#pragma unroll
        for (int t = 0; t < DO; ++t)
          if (t < d - 1) {
#pragma unroll
            for (int k = 0; k < KR; ++k) u[t][k] = fwd[((size_t)t * Q + k * T + c) * 32 + lane];
            wht_bits<KR, LKR - LT, LKR>(u[t]);
          }
      }
      double acc[KR];
#pragma unroll
      for (int k = 0; k < KR; ++k) {
        double v = 1.0;
#pragma unroll
        for (int t = 0; t < DO; ++t)
          if (t < d - 1) v *= u[t][k];
        const int w = (T > 1) ? (k * T + c) : k;
        acc[k] = neg_if(v, __popc(w & z) & 1);
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
      float *rdst = (a.rmsg && !lane_frozen(a, fb, lane)) ? a.rmsg + ((size_t)fb * E + e) * Q * 32 + lane : nullptr;
#pragma unroll
      for (int k = 0; k < KR; ++k) {
        const double v = acc[k] * (1.0 / Q);
        const float fv = (float)(v > 0.0 ? v : 0.0);
        const int row = rch ^ row_lo<P, LKR>(bb, k);  // a = h_e^-1 y
        rsm[((size_t)s * Q + row) * 32 + lane] = fv;
        if (rdst) rdst[row * 32] = fv;
      }
    }
    group_bar<T>(g);
    double r[DVMAX][KR];
#pragma unroll
    for (int s = 0; s < DVMAX; ++s)
      if (s < dv)
#pragma unroll
        for (int k = 0; k < KR; ++k) r[s][k] = (double)rsm[((size_t)s * Q + c * KR + k) * 32 + lane];
    vn_body<Q, DVMAX, MARKOV>(a, fb, j, e0, dv, r, red, g, c, lane, lane_frozen(a, fb, lane));
    group_bar<T>(g);
  }
}

// ============================================================== front end
// Per received bit: hard decision and probability that the noise
// bit is 1 (BSC: f; BEC: erased -> 0 with 1/2, else exact with 0 (A15);
// BI-AWGN: y < 0 -> 1, 1/(1+exp(2|y|/sigma^2)) (A16)); mode 3 = evidence
// supplied by the caller.  Transposes [frame][bit] -> [block][bit][lane].
__global__ void k_frontend(WaveArgs a, int mode, float param, const void *obs,
                           const unsigned char *hard_in, const float *pi_in) {
  __shared__ unsigned char th[32][33];
  __shared__ float tp[32][33];
  const long long Mp = (long long)a.c.M * a.c.p;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int fb = blockIdx.y;
  const long long bit0 = (long long)blockIdx.x * 32;
  const float s2 = param * param;
  for (int r = ty; r < 32; r += 8) {
    const long long f = (long long)(a.fb0 + fb) * 32 + r;
    const long long bit = bit0 + tx;
    unsigned char h = 0;
    float pv = 0.5f;
    if (f < a.n_frames && bit < Mp) {
      const long long idx = f * Mp + bit;
      if (mode == 0) {
        h = ((const unsigned char *)obs)[idx] & 1;
        pv = param;
      } else if (mode == 1) {
        const unsigned char o = ((const unsigned char *)obs)[idx];
        h = (o == 2) ? 0 : (o & 1);
        pv = (o == 2) ? 0.5f : 0.0f;
      } else if (mode == 2) {
        const float y = ((const float *)obs)[idx];
        h = y < 0.0f ? 1 : 0;
        pv = 1.0f / (1.0f + expf(2.0f * fabsf(y) / s2));
      } else {
        h = hard_in[idx] & 1;
        pv = pi_in[idx];
      }
    }
    th[r][tx] = h;
    tp[r][tx] = pv;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const long long bit = bit0 + r;
    if (bit < Mp) {
      const size_t o = ((size_t)fb * Mp + bit) * 32 + tx;
      a.hard[o] = th[tx][r];
      a.pi[o] = tp[tx][r];
    }
  }
}

// Syndrome z = B r (Eq. 2) over GF(2^p); lanes = frames.
__global__ void k_syndrome(WaveArgs a) {
  extern __shared__ unsigned char mul_s[];
  const int q = a.c.q, p = a.c.p, M = a.c.M, N = a.c.N;
  for (int k = threadIdx.x; k < q * q; k += blockDim.x) mul_s[k] = a.c.mul[k];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  const long long Mp = (long long)M * p;
  const long long ntask = (long long)a.nfb * M;
  for (long long task = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); task < ntask; task += nw) {
    const int fb = (int)(task / M), i = (int)(task % M);
    int acc = 0;
    for (int e = a.c.row_ptr[i]; e < a.c.row_ptr[i + 1]; ++e) {
      const int j = a.c.edge_var[e];
      if (j < N) continue;
      const int m = j - N;
      int sym = 0;
      for (int b = 0; b < p; ++b) sym |= (a.hard[((size_t)fb * Mp + (size_t)m * p + b) * 32 + lane] & 1) << b;
      acc ^= mul_s[a.c.edge_coef[e] * q + sym];
    }
    a.z[((size_t)fb * M + i) * 32 + lane] = (unsigned char)acc;
  }
}

// q_ij <- p_j on every edge.
template <int Q>
__global__ void __launch_bounds__(QC<Q>::THREADS) k_init_msgs(WaveArgs a) {
  using C = QC<Q>;
  constexpr int T = C::T, KR = C::KR, G = C::G;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = warp / T, c = warp % T;
  const long long E = a.c.E;
  const long long ntask = (long long)a.nfb * E;
  for (long long task = (long long)blockIdx.x * G + g; task < ntask; task += (long long)gridDim.x * G) {
    const int fb = (int)(task / E);
    const int e = (int)(task % E);
    const int j = __ldg(a.c.edge_var + e);
    double pr[KR];
    load_prior<Q, false>(a, fb, j, c, lane, true, pr);
    float *dst = a.qmsg + ((size_t)fb * E + e) * Q * 32 + lane;
#pragma unroll
    for (int k = 0; k < KR; ++k) dst[(c * KR + k) * 32] = (float)pr[k];
  }
}

__global__ void k_init_state(WaveArgs a) {
  const int n = a.nfb * 32;
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < n; f += gridDim.x * blockDim.x) {
    const long long gf = (long long)a.fb0 * 32 + f;
    const bool valid = gf < a.n_frames;
    a.iters[f] = -1;
    a.conv[f] = valid ? 0 : 1;
    a.unsat[f] = 0;
    a.newconv[f] = 0;
    if ((f & 31) == 0) {
      a.list[f >> 5] = f >> 5;
      a.active[f >> 5] = 1;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *a.nactive = a.nfb;
  }
}

// Convergence test: does x_hat solve H x = z?  Per active block,
// per chunk of checks; one atomic per lane per chunk.
__global__ void k_test(WaveArgs a, int chunk) {
  extern __shared__ unsigned char mul_s[];
  const int q = a.c.q, M = a.c.M, V = a.c.V;
  for (int k = threadIdx.x; k < q * q; k += blockDim.x) mul_s[k] = a.c.mul[k];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int nch = (M + chunk - 1) / chunk;
  const long long ntask = (long long)(*a.nactive) * nch;
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long task = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); task < ntask; task += nw) {
    const int fb = a.list[task / nch];
    const int i0 = (int)(task % nch) * chunk;
    const int i1 = min(M, i0 + chunk);
    int bad = 0;
    for (int i = i0; i < i1; ++i) {
      int acc = a.z[((size_t)fb * M + i) * 32 + lane];
      for (int e = __ldg(a.c.row_ptr + i); e < __ldg(a.c.row_ptr + i + 1); ++e)
        acc ^= mul_s[__ldg(a.c.edge_coef + e) * q + (a.xhat[((size_t)fb * V + __ldg(a.c.edge_var + e)) * 32 + lane] & (q - 1))];
      bad |= (acc != 0);
    }
    if (bad) atomicOr(a.unsat + fb * 32 + lane, 1);
  }
}

// Record the first passing iteration and flag frames whose estimate must be
// captured now (final_pass: every frame that never converged).
__global__ void k_finalize(WaveArgs a, int final_pass) {
  const int n = a.nfb * 32;
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < n; f += gridDim.x * blockDim.x) {
    int nc = 0;
    if (final_pass) {
      nc = (a.conv[f] == 0);
    } else if (a.active[f >> 5] && a.conv[f] == 0 && a.unsat[f] == 0) {
      a.conv[f] = 1;
      a.iters[f] = a.t;
      nc = 1;
      atomicAdd(a.stats + 2, 1ull);
    }
    a.newconv[f] = nc;
    a.unsat[f] = 0;
  }
}

// Copy x_hat[0:L) of flagged frames to the caller's [frame][L] output.
__global__ void k_capture(WaveArgs a, unsigned char *out, int L) {
  __shared__ unsigned char tile[128][33];
  const int fb = blockIdx.y;
  const int j0 = blockIdx.x * 128;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int flag = a.newconv[fb * 32 + lane];
  const unsigned mask = __ballot_sync(0xffffffffu, flag);
  if (mask == 0) return;  // uniform across the CTA (same fb)
  for (int r = warp; r < 128; r += 4) {
    const int j = j0 + r;
    tile[r][lane] = (j < L) ? a.xhat[((size_t)fb * a.c.V + j) * 32 + lane] : 0;
  }
  __syncthreads();
  for (int fl = warp; fl < 32; fl += 4) {
    if (!((mask >> fl) & 1)) continue;
    const long long f = (long long)(a.fb0 + fb) * 32 + fl;
    for (int r = lane; r < 128; r += 32) {
      const int j = j0 + r;
      if (j < L) out[f * L + j] = tile[r][fl];
    }
  }
}

// Active-block list (early exit): a block stays while one valid frame is
// unconverged.  Deterministic compaction by block-wide scan.
__global__ void k_compact(WaveArgs a, unsigned int *host_count) {
  __shared__ int wsum[32];
  __shared__ int base;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    base = 0;
    a.stats[1] += (unsigned long long)(*a.nactive);
  }
  __syncthreads();
  for (int b0 = 0; b0 < a.nfb; b0 += blockDim.x) {
    const int fb = b0 + tid;
    int act = 0;
    if (fb < a.nfb) {
      if (a.early_exit) {
        for (int l = 0; l < 32; ++l) act |= (a.conv[fb * 32 + l] == 0);
      } else {
        act = 1;
      }
      a.active[fb] = act;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, act);
    const int pre = __popc(bal & ((1u << lane) - 1));
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    int off = 0;
    for (int w = 0; w < warp; ++w) off += wsum[w];
    if (act) a.list[base + off + pre] = fb;
    __syncthreads();
    if (tid == 0) {
      int t = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += wsum[w];
      base += t;
    }
    __syncthreads();
  }
  if (tid == 0) {
    *a.nactive = base;
    if (host_count) *host_count = (unsigned)base;
  }
}

__global__ void k_set_u64(unsigned long long *p, unsigned long long v) { *p = v; }

// Export to [frame][canonical edge][q] / [frame][V][q] (debug and parity only).
__global__ void k_export(WaveArgs a, const float *src, float *dst, int items, const int *map) {
  const int q = a.c.q;
  const long long n = (long long)a.nfb * 32 * items * q;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(t % q);
    const long long r = t / q;
    const int item = (int)(r % items);
    const long long f = r / items;  // wave-local frame
    const long long gf = (long long)a.fb0 * 32 + f;
    if (gf >= a.n_frames) continue;
    const int fb = (int)(f >> 5), lane = (int)(f & 31);
    const int it = map ? map[item] : item;
    dst[(gf * items + item) * q + x] = src[(((size_t)fb * items + it) * q + x) * 32 + lane];
  }
}

// ============================================================== launch helpers
static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <typename K>
static int grid_for(K kern, int threads, size_t smem, long long max_ctas) {
  static std::mutex mu;
  static std::unordered_map<const void *, int> cache;
  int per_sm;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find((const void *)kern);
    if (it == cache.end()) {
      if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
      if (per_sm < 1) per_sm = 1;
      cache[(const void *)kern] = per_sm;
    } else {
      per_sm = it->second;
    }
  }
  long long g = (long long)sm_count() * per_sm;
  if (g > max_ctas) g = max_ctas;
  if (g < 1) g = 1;
  return (int)g;
}

static int check_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, what);
  return GFQ_OK;
}

#define GFQ_DISPATCH_Q(q, F)          \
  switch (q) {                        \
    case 2: return F(2);              \
    case 4: return F(4);              \
    case 8: return F(8);              \
    case 16: return F(16);            \
    case 32: return F(32);            \
    case 64: return F(64);            \
    default: break;                   \
  }                                   \
  set_error("unsupported q");         \
  return GFQ_EUNSUPPORTED;

template <int Q>
static int cn_q(const WaveArgs &a, cudaStream_t s) {
  using C = QC<Q>;
  if (a.c.max_cdeg <= 4) {
    const size_t sm = C::T > 1 ? (size_t)C::G * 4 * Q * 32 * sizeof(double) : 0;
    auto k = k_cn<Q, 4>;
    const int grid = grid_for(k, C::THREADS, sm, ((long long)a.nfb * a.c.M + C::G - 1) / C::G);
    k<<<grid, C::THREADS, sm, s>>>(a);
  } else {
    const size_t sm = C::T > 1 ? (size_t)C::G * 8 * Q * 32 * sizeof(double) : 0;
    auto k = k_cn<Q, 8>;
    const int grid = grid_for(k, C::THREADS, sm, ((long long)a.nfb * a.c.M + C::G - 1) / C::G);
    k<<<grid, C::THREADS, sm, s>>>(a);
  }
  return check_launch("k_cn");
}

template <int Q, bool MK>
static int vn_qm(const WaveArgs &a, int clip, cudaStream_t s) {
  using C = QC<Q>;
  if (a.c.max_vdeg <= 4) {
    const size_t sm = (size_t)C::G * (4 + 3) * C::T * 32 * sizeof(double);
    auto k = k_vn<Q, 4, MK>;
    const int grid = grid_for(k, C::THREADS, sm, ((long long)a.nfb * a.c.V + C::G - 1) / C::G);
    k<<<grid, C::THREADS, sm, s>>>(a, clip);
  } else {
    const size_t sm = (size_t)C::G * (8 + 3) * C::T * 32 * sizeof(double);
    auto k = k_vn<Q, 8, MK>;
    const int grid = grid_for(k, C::THREADS, sm, ((long long)a.nfb * a.c.V + C::G - 1) / C::G);
    k<<<grid, C::THREADS, sm, s>>>(a, clip);
  }
  return check_launch("k_vn");
}

template <int Q>
static int vn_q(const WaveArgs &a, int clip, cudaStream_t s) {
  return a.markov ? vn_qm<Q, true>(a, clip, s) : vn_qm<Q, false>(a, clip, s);
}

template <int Q, int DM, int DV>
static size_t sus_smem() {
  using C = QC<Q>;
  const size_t fwd = C::T > 1 ? (size_t)(DM - 1) * Q * 32 : 0;
  const size_t acc = C::T > 1 ? (size_t)Q * 32 : 0;
  const size_t red = (size_t)(DV + 3) * C::T * 32;
  const size_t rsm = (size_t)DV * Q * 32 / 2;
  return (size_t)C::G * (fwd + acc + red + rsm) * sizeof(double);
}

template <int Q, int DM, int DV, bool MK>
static int sus_launch(const WaveArgs &a, int lb, int ncols, cudaStream_t s) {
  using C = QC<Q>;
  const size_t sm = sus_smem<Q, DM, DV>();
  auto k = k_sus<Q, DM, DV, MK>;
  const int grid = grid_for(k, C::THREADS, sm, ((long long)a.nfb * ncols + C::G - 1) / C::G);
  k<<<grid, C::THREADS, sm, s>>>(a, lb, ncols);
  return check_launch("k_sus");
}

template <int Q>
static int sus_q(const WaveArgs &a, int lb, int ncols, cudaStream_t s) {
  const bool small = a.c.max_cdeg <= 4 && a.c.max_vdeg <= 4;
  if (a.markov)
    return small ? sus_launch<Q, 4, 4, true>(a, lb, ncols, s) : sus_launch<Q, 8, 8, true>(a, lb, ncols, s);
  return small ? sus_launch<Q, 4, 4, false>(a, lb, ncols, s) : sus_launch<Q, 8, 8, false>(a, lb, ncols, s);
}

template <int Q>
static int init_q(const WaveArgs &a, cudaStream_t s) {
  using C = QC<Q>;
  auto k = k_init_msgs<Q>;
  const int grid = grid_for(k, C::THREADS, 0, ((long long)a.nfb * a.c.E + C::G - 1) / C::G);
  k<<<grid, C::THREADS, 0, s>>>(a);
  return check_launch("k_init_msgs");
}

int launch_frontend(const WaveArgs &a, int mode, double ch_param, const void *obs,
                    const unsigned char *hard_in, const float *pi_in, cudaStream_t s) {
  const long long Mp = (long long)a.c.M * a.c.p;
  dim3 grid((unsigned)((Mp + 31) / 32), (unsigned)a.nfb);
  k_frontend<<<grid, dim3(32, 8), 0, s>>>(a, mode, (float)ch_param, obs, hard_in, pi_in);
  return check_launch("k_frontend");
}

int launch_syndrome(const WaveArgs &a, cudaStream_t s) {
  const int threads = 256;
  const long long tasks = (long long)a.nfb * a.c.M;
  const int grid = (int)std::min<long long>((tasks + 7) / 8, (long long)sm_count() * 8);
  k_syndrome<<<grid, threads, a.c.q * a.c.q, s>>>(a);
  return check_launch("k_syndrome");
}

int launch_init_msgs(const WaveArgs &a, cudaStream_t s) {
#define F(Q) init_q<Q>(a, s)
  GFQ_DISPATCH_Q(a.c.q, F)
#undef F
}

int launch_init_state(const WaveArgs &a, cudaStream_t s) {
  const int n = a.nfb * 32;
  k_init_state<<<(n + 255) / 256, 256, 0, s>>>(a);
  return check_launch("k_init_state");
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

int launch_test(const WaveArgs &a, cudaStream_t s) {
  const int chunk = 64;
  const int threads = 256;
  const long long tasks = (long long)a.nfb * ((a.c.M + chunk - 1) / chunk);
  const int grid = (int)std::max<long long>(1, std::min<long long>((tasks + 7) / 8, (long long)sm_count() * 8));
  k_test<<<grid, threads, a.c.q * a.c.q, s>>>(a, chunk);
  return check_launch("k_test");
}

int launch_finalize(const WaveArgs &a, int final_pass, cudaStream_t s) {
  const int n = a.nfb * 32;
  k_finalize<<<(n + 255) / 256, 256, 0, s>>>(a, final_pass);
  return check_launch("k_finalize");
}

int launch_capture(const WaveArgs &a, unsigned char *out, int L, int /*mode*/, cudaStream_t s) {
  dim3 grid((unsigned)((L + 127) / 128), (unsigned)a.nfb);
  k_capture<<<grid, 128, 0, s>>>(a, out, L);
  return check_launch("k_capture");
}

int launch_compact(const WaveArgs &a, cudaStream_t s) {
  k_compact<<<1, 1024, 0, s>>>(a, nullptr);
  return check_launch("k_compact");
}

int launch_export(const WaveArgs &a, float *q_out, float *r_out, float *Q_out, cudaStream_t s) {
  const int threads = 256;
  const int grid = sm_count() * 8;
  if (q_out) k_export<<<grid, threads, 0, s>>>(a, a.qmsg, q_out, (int)a.c.E, a.c.col_edge);
  if (r_out) k_export<<<grid, threads, 0, s>>>(a, a.rmsg, r_out, (int)a.c.E, a.c.col_edge);
  if (Q_out) k_export<<<grid, threads, 0, s>>>(a, a.qall, Q_out, a.c.V, nullptr);
  return check_launch("k_export");
}

int launch_set_u64(unsigned long long *p, unsigned long long v, cudaStream_t s) {
  k_set_u64<<<1, 1, 0, s>>>(p, v);
  return check_launch("k_set_u64");
}

}  // namespace gfq

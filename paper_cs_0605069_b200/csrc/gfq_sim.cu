// gfq_sim.cu -- Monte-Carlo front end on the device: the
// steps before the decoder, for BER sweeps at GPU speed.  PAPER.md P:134-143 is
// the authority: source s (i.i.d. or Markov), codeword
// t = B^-1 A s (Eq. 1), bits LSB first (A2), channel BSC / BEC / BI-AWGN
// (A15, A16).  Random numbers: Philox4x32-10 (counter-based), the counters and
// conversions of include/gfq.h (gfq_simulate), so any subset of frames
// reproduces exactly and a CPU implementation can draw the same numbers.
//
// Kernels (one frame per lane, 32-frame blocks as in the decoder):
//   k_sim_source   s into [block][N][32] (Markov: sequential along the chain)
//   k_sim_encode   y = A s and the peeling solve of B t = y, row order fixed at
//                  gfq_code_create; t into [block][M][32]
//   k_sim_unblock  [block][L][32] -> [frame][L] (s out, t for the channel)
//   k_sim_channel  per bit: received bit / erasure / BPSK + Gaussian noise
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "gfq_internal.cuh"
#include "gfq_launch.cuh"

namespace gfq {

// ============================================================== Philox4x32-10
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
  }
  return c;
}

constexpr uint32_t kPurposeSource = 1, kPurposeChannel = 2;

__device__ __forceinline__ uint4 draw(const SimArgs &a, long long frame, uint32_t j, uint32_t purpose) {
  const unsigned long long f = (unsigned long long)frame;
  return philox4x32_10(make_uint4(j, (uint32_t)f, (uint32_t)(f >> 32), purpose), (uint32_t)a.seed,
                       (uint32_t)(a.seed >> 32));
}

__device__ __forceinline__ double u24(uint32_t x) { return (double)(x >> 8) * (1.0 / 16777216.0); }

__device__ __forceinline__ uint32_t pick(uint4 v, int m) {
  return m == 0 ? v.x : m == 1 ? v.y : m == 2 ? v.z : v.w;
}

// min{b : u < C[b]} for running sums C (nondecreasing, C[q-1] = 1): binary search
__device__ __forceinline__ int inverse_cdf(const double *C, int q, double u) {
  int lo = 0, hi = q - 1;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (u < C[mid]) hi = mid; else lo = mid + 1;
  }
  return lo;
}

// ============================================================== source
__global__ void k_sim_source(SimArgs a) {
  extern __shared__ double cum[];  // [q] pi0 then [q*q] T (Markov)
  const int q = a.c.q, N = a.c.N;
  if (a.markov) {
    for (int k = threadIdx.x; k < q + q * q; k += blockDim.x) cum[k] = k < q ? a.cum0[k] : a.cumT[k - q];
    __syncthreads();
  }
  const long long fl = (long long)blockIdx.x * blockDim.x + threadIdx.x;  // wave-local frame
  if (fl >= (long long)a.nfb * 32) return;
  const int fb = (int)(fl >> 5), lane = (int)(fl & 31);
  unsigned char *dst = a.s_blk + (size_t)fb * N * 32 + lane;
  if (fl >= a.n_frames) {  // ragged block: zeros
    for (int k = 0; k < N; ++k) dst[(size_t)k * 32] = 0;
    return;
  }
  const long long frame = a.frame0 + fl;
  int prev = 0;
  for (int j = 0; 4 * j < N; ++j) {
    const uint4 v = draw(a, frame, (uint32_t)j, kPurposeSource);
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int k = 4 * j + m;
      if (k >= N) break;
      const uint32_t x = pick(v, m);
      int s;
      if (!a.markov) {
        s = (int)(x & (uint32_t)(q - 1));
      } else {
        const double u = u24(x);
        s = inverse_cdf(k == 0 ? cum : cum + q + prev * q, q, u);
      }
      prev = s;
      dst[(size_t)k * 32] = (unsigned char)s;
    }
  }
}

// ============================================================== encoder (Eq. 1)
// t = B^-1 A s by the peeling order: row r of H solves noise column k:
//   h_rk t_k = (A s)_r + sum_{k' != k} h_rk' t_k'   (all k' solved before).
__global__ void k_sim_encode(SimArgs a) {
  extern __shared__ unsigned char tab[];  // mul[q*q], inv[q]
  const int q = a.c.q, N = a.c.N, M = a.c.M;
  for (int k = threadIdx.x; k < q * q + q; k += blockDim.x) tab[k] = k < q * q ? a.c.mul[k] : a.c.inv[k - q * q];
  __syncthreads();
  const unsigned char *mul = tab, *inv = tab + q * q;
  const int fb = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (fb >= a.nfb) return;
  const unsigned char *sb = a.s_blk + (size_t)fb * N * 32 + lane;
  unsigned char *tb = a.t_blk + (size_t)fb * M * 32 + lane;
  for (int m = 0; m < M; ++m) {
    const int r = __ldg(a.c.peel + 2 * m), k = __ldg(a.c.peel + 2 * m + 1);
    const int e0 = __ldg(a.c.row_ptr + r), e1 = __ldg(a.c.row_ptr + r + 1);
    int acc = 0, hk = 1;
    for (int e = e0; e < e1; ++e) {
      const int j = __ldg(a.c.edge_var + e), h = __ldg(a.c.edge_coef + e);
      if (j < N) {
        acc ^= mul[h * q + sb[(size_t)j * 32]];
      } else if (j - N != k) {
        acc ^= mul[h * q + tb[(size_t)(j - N) * 32]];
      } else {
        hk = h;
      }
    }
    tb[(size_t)k * 32] = mul[inv[hk] * q + acc];
  }
}

// [block][L][32] -> [frame][L] through a 128 x 32 shared tile
__global__ void k_sim_unblock(const unsigned char *blk, unsigned char *out, int L, int n_frames) {
  __shared__ unsigned char tile[128][33];
  const int fb = blockIdx.y, j0 = blockIdx.x * 128;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int r = warp; r < 128; r += 4) {
    const int j = j0 + r;
    tile[r][lane] = (j < L) ? blk[((size_t)fb * L + j) * 32 + lane] : 0;
  }
  __syncthreads();
  for (int fl = warp; fl < 32; fl += 4) {
    const long long f = (long long)fb * 32 + fl;
    if (f >= n_frames) break;
    for (int r = lane; r < 128; r += 32) {
      const int j = j0 + r;
      if (j < L) out[f * L + j] = tile[r][fl];
    }
  }
}

// ============================================================== channel
__global__ void k_sim_channel(SimArgs a) {
  const int p = a.c.p, M = a.c.M;
  const long long nbits = (long long)M * p;
  const int per = a.channel == GFQ_BIAWGN ? 2 : 4;  // bits per Philox call
  const long long ngroups = (nbits + per - 1) / per;
  const long long total = (long long)a.n_frames * ngroups;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long fl = t / ngroups;
    const uint32_t j = (uint32_t)(t - fl * ngroups);
    const uint4 v = draw(a, a.frame0 + fl, j, kPurposeChannel);
    const unsigned char *tf = a.t_fm + (size_t)fl * M;
    if (a.channel != GFQ_BIAWGN) {
      unsigned char *o = (unsigned char *)a.obs + (size_t)fl * nbits;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const long long i = 4LL * j + m;
        if (i >= nbits) break;
        const int bit = (tf[i / p] >> (int)(i % p)) & 1;
        const bool hit = u24(pick(v, m)) < a.param;
        o[i] = a.channel == GFQ_BSC ? (unsigned char)(bit ^ (int)hit) : (hit ? (unsigned char)2 : (unsigned char)bit);
      }
    } else {
      float *o = (float *)a.obs + (size_t)fl * nbits;
      const double u1 = ((double)(v.x >> 8) + 1.0) * (1.0 / 16777216.0);
      const double u2 = u24(v.y);
      const double rho = sqrt(-2.0 * log(u1));
      double sn, cs;
      sincospi(2.0 * u2, &sn, &cs);
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        const long long i = 2LL * j + m;
        if (i >= nbits) break;
        const int bit = (tf[i / p] >> (int)(i % p)) & 1;
        const double n = rho * (m == 0 ? cs : sn);
        o[i] = (float)((1.0 - 2.0 * bit) + a.param * n);
      }
    }
  }
}

int launch_sim(const SimArgs &a, cudaStream_t s) {
  const int q = a.c.q;
  const int nthr = a.nfb * 32;
  const size_t smem_src = a.markov ? sizeof(double) * (size_t)(q + q * q) : 0;
  if (smem_src > 227 * 1024) {
    set_error("gfq_simulate: the Markov source tables of this field size do not fit in shared memory");
    return GFQ_EUNSUPPORTED;
  }
  if (smem_src > 48 * 1024) cudaFuncSetAttribute(k_sim_source, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_src);
  k_sim_source<<<(nthr + 127) / 128, 128, smem_src, s>>>(a);
  int rc = check_launch("k_sim_source");
  if (rc) return rc;
  if ((size_t)q * q + q > 48 * 1024)
    cudaFuncSetAttribute(k_sim_encode, cudaFuncAttributeMaxDynamicSharedMemorySize, q * q + q);
  k_sim_encode<<<(a.nfb + 3) / 4, 128, (size_t)q * q + q, s>>>(a);
  if ((rc = check_launch("k_sim_encode"))) return rc;
  if (a.s_out) {
    k_sim_unblock<<<dim3((a.c.N + 127) / 128, a.nfb), 128, 0, s>>>(a.s_blk, a.s_out, a.c.N, a.n_frames);
    if ((rc = check_launch("k_sim_unblock"))) return rc;
  }
  k_sim_unblock<<<dim3((a.c.M + 127) / 128, a.nfb), 128, 0, s>>>(a.t_blk, a.t_fm, a.c.M, a.n_frames);
  if ((rc = check_launch("k_sim_unblock"))) return rc;
  if (a.obs) {
    k_sim_channel<<<sm_count() * 8, 256, 0, s>>>(a);
    if ((rc = check_launch("k_sim_channel"))) return rc;
  }
  return GFQ_OK;
}

}  // namespace gfq

using namespace gfq;

// Running sums in double, left to right, last entry 1 (include/gfq.h).
static void running_sums(const double *P, int rows, int q, std::vector<double> &out) {
  out.assign((size_t)rows * q, 0.0);
  for (int r = 0; r < rows; ++r) {
    double acc = 0.0;
    for (int b = 0; b < q; ++b) {
      acc += P[(size_t)r * q + b];
      out[(size_t)r * q + b] = acc;
    }
    out[(size_t)r * q + q - 1] = 1.0;
  }
}

static inline size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

extern "C" size_t gfq_simulate_workspace_bytes(const gfq_code *c, int n_frames) {
  if (!c || n_frames < 0) return 0;
  const size_t nfb = (size_t)std::max(1, (n_frames + 31) / 32);
  return al256(sizeof(double) * (size_t)(c->q + c->q * c->q)) + al256(nfb * c->N * 32) + al256(nfb * c->M * 32) +
         al256((size_t)n_frames * c->M);
}

extern "C" int gfq_simulate(const gfq_code *c, int n_frames, unsigned long long seed, long long frame0,
                            const gfq_sim_params *prm, unsigned char *s_out, void *obs_out,
                            unsigned char *t_out, void *ws, size_t ws_bytes, void *stream) {
  if (!c || !prm) { set_error("gfq_simulate: NULL code or params"); return GFQ_EINVAL; }
  if (n_frames < 0 || frame0 < 0) { set_error("gfq_simulate: n_frames or frame0 < 0"); return GFQ_EINVAL; }
  if (prm->channel < GFQ_BSC || prm->channel > GFQ_BIAWGN) { set_error("gfq_simulate: bad channel"); return GFQ_EINVAL; }
  if (prm->channel != GFQ_BIAWGN && !(prm->ch_param >= 0.0 && prm->ch_param <= 1.0)) {
    set_error("gfq_simulate: flip / erasure probability must be in [0, 1]");
    return GFQ_EINVAL;
  }
  if (prm->channel == GFQ_BIAWGN && !(prm->ch_param >= 0.0)) { set_error("gfq_simulate: sigma < 0"); return GFQ_EINVAL; }
  if (!c->d.peel) {
    set_error("gfq_simulate: B is not triangular up to a permutation (no peeling order); encoding unsupported");
    return GFQ_EUNSUPPORTED;
  }
  if (n_frames == 0) return GFQ_OK;
  if (!ws || ws_bytes < gfq_simulate_workspace_bytes(c, n_frames)) {
    set_error("gfq_simulate: workspace too small (gfq_simulate_workspace_bytes)");
    return GFQ_EINVAL;
  }
  const int q = c->q;
  std::vector<double> h;
  if (prm->markov_T) {
    std::vector<double> pi0(q, 1.0 / q), c0, cT;
    if (prm->src_pi0) pi0.assign(prm->src_pi0, prm->src_pi0 + q);
    for (int a = 0; a < q * q; ++a)
      if (!(prm->markov_T[a] >= 0.0)) { set_error("gfq_simulate: negative markov_T entry"); return GFQ_EINVAL; }
    running_sums(pi0.data(), 1, q, c0);
    running_sums(prm->markov_T, q, q, cT);
    h = c0;
    h.insert(h.end(), cT.begin(), cT.end());
  }
  cudaStream_t st = (cudaStream_t)stream;
  char *b = (char *)ws;
  const int nfb = (n_frames + 31) / 32;
  SimArgs a;
  memset(&a, 0, sizeof(a));
  a.c = c->d;
  a.n_frames = n_frames;
  a.nfb = nfb;
  a.seed = seed;
  a.frame0 = frame0;
  a.channel = prm->channel;
  a.param = prm->ch_param;
  a.markov = prm->markov_T != nullptr;
  size_t off = 0;
  double *cum = (double *)(b + off);
  off += al256(sizeof(double) * (size_t)(q + q * q));
  a.s_blk = (unsigned char *)(b + off);
  off += al256((size_t)nfb * c->N * 32);
  a.t_blk = (unsigned char *)(b + off);
  off += al256((size_t)nfb * c->M * 32);
  a.t_fm = t_out ? t_out : (unsigned char *)(b + off);
  a.s_out = s_out;
  a.obs = obs_out;
  a.cum0 = cum;
  a.cumT = cum + q;
  if (a.markov) {
    cudaError_t ce = cudaMemcpyAsync(cum, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice, st);
    if (ce != cudaSuccess) return cuda_fail(ce, "gfq_simulate: upload running sums");
  }
  return launch_sim(a, st);
}

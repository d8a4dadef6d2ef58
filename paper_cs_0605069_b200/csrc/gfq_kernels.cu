// gfq_kernels.cu -- the per-decode support kernels of libgfq: channel front
// end, syndrome, message initialisation, convergence test, bookkeeping,
// capture of decisions and message export (the BP iteration kernels are in
// gfq_bp.cu).  PAPER.md §2 is the authority for what is computed.
// Layout: one frame per lane, [frame block][item][entry][32 lanes] (see gfq_bp.cu).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "gfq_internal.cuh"
#include "gfq_launch.cuh"

namespace gfq {

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

// q_ij <- p_j on every edge: the prior of variable j is the noise
// prior prod_b (bit_b(a) ? pi_b : 1 - pi_b) or pi0.
__global__ void k_init_msgs(WaveArgs a) {
  const int q = a.c.q, p = a.c.p, N = a.c.N;
  const long long E = a.c.E;
  const size_t Mp = (size_t)a.c.M * p;
  const int lane = threadIdx.x & 31;
  // one warp per (block, edge): lane = frame, loop over the q rows
  const long long nw = (long long)a.nfb * E;
  for (long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nw;
       w += ((long long)gridDim.x * blockDim.x) >> 5) {
    const int e = (int)(w % E);
    const int fb = (int)(w / E);
    const int j = __ldg(a.c.edge_var + e);
    float *dst = a.qmsg + (size_t)w * q * 32 + lane;
    if (j >= N) {
      double pb[8];
      for (int b = 0; b < p; ++b) pb[b] = (double)a.pi[((size_t)fb * Mp + (size_t)(j - N) * p + b) * 32 + lane];
      for (int x = 0; x < q; ++x) {
        double v = 1.0;
        for (int b = 0; b < p; ++b) v *= ((x >> b) & 1) ? pb[b] : 1.0 - pb[b];
        dst[x * 32] = (float)v;
      }
    } else {
      for (int x = 0; x < q; ++x) dst[x * 32] = (float)__ldg(a.pi0 + x);
    }
  }
}

__global__ void k_init_state(WaveArgs a) {
  const int n = a.nfb * 32;
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < n; f += gridDim.x * blockDim.x) {
    const long long gf = (long long)a.fb0 * 32 + f;
    const bool valid = gf < a.n_frames;
    a.iters[f] = -1;
    a.fid[f] = valid ? f : -1;
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
      a.iters[a.fid[f]] = a.t;  // by frame: the lane slot may hold a moved frame (k_repack_plan)
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
    const long long f = (long long)a.fb0 * 32 + a.fid[fb * 32 + fl];  // flagged slots hold a frame
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


// ============================================================== frame-granular early-exit compaction
// A block iterates until its slowest frame has stopped, so late in
// a decode most lanes of the live blocks are idle.  One round, after the
// estimates of the frames that stopped in this iteration have been captured:
// k_repack_plan picks the D = B - ceil(A/32) sparsest of the B live blocks
// (A = frames still decoding) as donors and assigns their frames, in order, to
// the idle lanes of the other live blocks (receivers), when D >= 1 and
// 3 D >= ceil(A/32) (moving a frame costs about one iteration of its bytes);
// k_repack_move then copies the per-frame rows (q messages, per-bit evidence,
// syndrome, estimate, posterior snapshot) lane to lane.  The donors are left
// with no decoding frame and k_compact drops them.  A frame's arithmetic does
// not depend on its lane, so the decode's outputs do not change.
__device__ __forceinline__ int cta_excl_scan(int v, int *wsum, int &total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  int off = 0, tot = 0;
  for (int w = 0; w < nw; ++w) {
    const int sw = wsum[w];
    if (w < warp) off += sw;
    tot += sw;
  }
  __syncthreads();
  total = tot;
  return off + x - v;
}

__global__ void __launch_bounds__(1024) k_repack_plan(WaveArgs a, RepackPlan rp) {
  __shared__ int hist[33];
  __shared__ int wsum[32];
  __shared__ int s_cstar, s_neq, s_go, s_ndst;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int B = *a.nactive;
  if (tid < 33) hist[tid] = 0;
  if (tid == 0) s_ndst = 0;
  __syncthreads();
  for (int i = warp; i < B; i += nw) {
    const int b = a.list[i];
    const unsigned m = __ballot_sync(0xffffffffu, a.conv[b * 32 + lane] == 0);
    if (lane == 0) {
      rp.cnt[i] = __popc(m);
      rp.amask[i] = m;
      atomicAdd(&hist[__popc(m)], 1);
    }
  }
  __syncthreads();
  if (tid == 0) {
    int A = 0;
    for (int c = 1; c <= 32; ++c) A += c * hist[c];
    const int need = (A + 31) / 32;
    const int D = B - need;              // donors, the blocks with no frame left included
    const int Dn = D - hist[0];          // donors that still hold frames
    const int go = (Dn >= 1 && 3 * Dn >= need) ? 1 : 0;
    int less = 0, cstar = 0;
    for (; cstar <= 32; ++cstar) {
      if (less + hist[cstar] > D) break;
      less += hist[cstar];
    }
    s_cstar = cstar;     // donors: every block with fewer frames than cstar ...
    s_neq = D - less;    // ... and the first s_neq blocks (list order) with exactly cstar
    s_go = go;
    rp.hdr[0] = 0;
    rp.hdr[1] = B;
    rp.hdr[2] = go ? need : B;
    rp.hdr[3] = 0;
  }
  __syncthreads();
  if (!s_go) return;
  const int cstar = s_cstar, neq = s_neq;
  // roles
  int carry = 0;
  for (int i0 = 0; i0 < B; i0 += blockDim.x) {
    const int i = i0 + tid;
    const int c = i < B ? rp.cnt[i] : 33;
    int tot;
    const int rank = carry + cta_excl_scan(c == cstar ? 1 : 0, wsum, tot);
    carry += tot;
    if (i < B) rp.role[i] = (c < cstar || (c == cstar && rank < neq)) ? 1 : 0;
  }
  __syncthreads();
  // donor index / frames before each donor; idle lanes before each receiver
  int cd = 0, cf = 0, cr = 0;
  for (int i0 = 0; i0 < B; i0 += blockDim.x) {
    const int i = i0 + tid;
    const int role = i < B ? rp.role[i] : -1;
    const int c = i < B ? rp.cnt[i] : 0;
    int t0, t1, t2;
    const int di = cd + cta_excl_scan(role == 1 ? 1 : 0, wsum, t0);
    const int df = cf + cta_excl_scan(role == 1 ? c : 0, wsum, t1);
    const int rf = cr + cta_excl_scan(role == 0 ? 32 - c : 0, wsum, t2);
    cd += t0; cf += t1; cr += t2;
    if (role == 1) {
      rp.dblk[di] = i;
      rp.dpre[di] = df;
    } else if (role == 0) {
      rp.rpre[i] = rf;
    }
  }
  const int nd = cd, adon = cf;
  if (tid == 0) rp.dpre[nd] = adon;
  __syncthreads();
  // receivers take the donors' frames in order
  for (int i = warp; i < B; i += nw) {
    if (rp.role[i] != 0) continue;                 // warp-uniform
    const unsigned fm = ~rp.amask[i];
    const int o = rp.rpre[i];
    if (o >= adon || fm == 0u) continue;
    const int b = a.list[i];
    int src = -1;
    if ((fm >> lane) & 1u) {
      const int idx = o + __popc(fm & ((1u << lane) - 1u));
      if (idx < adon) {
        int lo = 0, hi = nd;                       // largest d with dpre[d] <= idx < dpre[d+1]
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (rp.dpre[mid] <= idx) lo = mid; else hi = mid;
        }
        const int li = rp.dblk[lo];
        const int sl = __fns(rp.amask[li], 0, idx - rp.dpre[lo] + 1);
        src = a.list[li] * 32 + sl;
      }
    }
    int k = 0;
    if (lane == 0) k = atomicAdd(&s_ndst, 1);
    k = __shfl_sync(0xffffffffu, k, 0);
    if (lane == 0) rp.dst[k] = b;
    rp.map[k * 32 + lane] = src;
    if (src >= 0) {
      const int slot = b * 32 + lane;
      a.fid[slot] = a.fid[src];
      a.conv[slot] = 0;
      a.fid[src] = -1;
      a.conv[src] = 1;
    }
  }
  __syncthreads();
  if (tid == 0) {
    rp.hdr[0] = s_ndst;
    rp.hdr[3] = adon;
  }
}

struct MoveSet {
  void *base[5];
  long long rows[5];   // rows per block
  int esz[5];          // bytes per lane: 4 (float rows of 128 B) or 1 (byte rows of 32 B)
  int n;
};

__device__ __forceinline__ float shfl_lane(float v, int l) { return __shfl_sync(0xffffffffu, v, l); }
__device__ __forceinline__ unsigned char shfl_lane(unsigned char v, int l) {
  return (unsigned char)__shfl_sync(0xffffffffu, (int)v, l);
}

template <typename T, int U>
__device__ __forceinline__ void move_rows(T *base, long long rows, const RepackPlan &rp, int nd, long long w0,
                                          long long nwarps, int lane) {
  const long long per = (rows + U - 1) / U;
  const long long ntask = (long long)nd * per;
  for (long long task = w0; task < ntask; task += nwarps) {
    const int k = (int)(task / per);
    const long long r0 = (task - (long long)k * per) * U;
    const int db = rp.dst[k];
    const int src = rp.map[k * 32 + lane];
    T v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (r0 + u < rows) v[u] = base[((size_t)db * rows + r0 + u) * 32 + lane];
    unsigned todo = __ballot_sync(0xffffffffu, src >= 0);
    while (todo) {
      const int leader = __ffs(todo) - 1;
      const int sb = __shfl_sync(0xffffffffu, src, leader) >> 5;
      const bool mine = src >= 0 && (src >> 5) == sb;
      T w[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (r0 + u < rows) w[u] = base[((size_t)sb * rows + r0 + u) * 32 + lane];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (r0 + u < rows) {
          const T pick = shfl_lane(w[u], src & 31);
          if (mine) v[u] = pick;
        }
      }
      todo &= ~__ballot_sync(0xffffffffu, mine);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (r0 + u < rows) base[((size_t)db * rows + r0 + u) * 32 + lane] = v[u];
  }
}

__global__ void __launch_bounds__(256) k_repack_move(RepackPlan rp, MoveSet ms) {
  const int nd = rp.hdr[0];
  if (nd == 0) return;
  const int lane = threadIdx.x & 31;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const long long w0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (int ai = 0; ai < ms.n; ++ai) {
    if (ms.esz[ai] == 4) move_rows<float, 4>((float *)ms.base[ai], ms.rows[ai], rp, nd, w0, nwarps, lane);
    else move_rows<unsigned char, 4>((unsigned char *)ms.base[ai], ms.rows[ai], rp, nd, w0, nwarps, lane);
  }
}

__global__ void k_set_u64(unsigned long long *p, unsigned long long v) { *p = v; }

// ============================================================== Fig. 1 instrumentation
// trace[f][t] = number of source bits of the current estimate x^(t) equal to
// the true source s ("percentage of correct bits", times N*p/100).
// One CTA per active 32-frame block; warp w takes 32-symbol tiles of the
// source range; the truth tile [32 frames][32 symbols] is read row-wise
// (coalesced) and transposed through shared memory so that lane = frame.
__global__ void k_trace(WaveArgs a, const unsigned char *truth, int *trace, int t, int tlen) {
  __shared__ unsigned char tile[8][32][33];
  __shared__ int part[8][32];
  const int fbi = blockIdx.x;
  if (fbi >= *a.nactive) return;
  const int fb = a.list[fbi];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int N = a.c.N, p = a.c.p;
  const unsigned mask = (1u << p) - 1u;
  const long long f0 = (long long)a.fb0 * 32;
  int ok = 0;
  for (int j0 = w * 32; j0 < N; j0 += 8 * 32) {
    for (int r = 0; r < 32; ++r) {
      const int fl = a.fid[fb * 32 + r];  // the frame in lane slot r (-1: none)
      const int j = j0 + lane;
      tile[w][r][lane] = (fl >= 0 && j < N) ? truth[(f0 + fl) * N + j] : 0;
    }
    __syncwarp();
    const int jn = min(32, N - j0);
    for (int jj = 0; jj < jn; ++jj) {
      const unsigned x = a.xhat[((size_t)fb * a.c.V + j0 + jj) * 32 + lane];
      ok += p - __popc((x ^ tile[w][lane][jj]) & mask);
    }
    __syncwarp();
  }
  part[w][lane] = ok;
  __syncthreads();
  if (w == 0) {
    int s = 0;
    for (int k = 0; k < 8; ++k) s += part[k][lane];
    const int fl = a.fid[fb * 32 + lane];
    if (fl >= 0) trace[(f0 + fl) * tlen + t] = s;
  }
}

// Frames that stopped early keep their estimate: forward-fill the entries of
// iterations their block no longer ran (initialised to -1).
__global__ void k_trace_fill(int *trace, int n_frames, int tlen) {
  const long long f = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= n_frames) return;
  int *tr = trace + f * tlen;
  for (int t = 1; t < tlen; ++t)
    if (tr[t] < 0) tr[t] = tr[t - 1];
}

// Export to [frame][canonical edge][q] / [frame][V][q] (debug and parity only).
__global__ void k_export(WaveArgs a, const float *src, float *dst, int items, const int *map, float scale) {
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
    dst[(gf * items + item) * q + x] = scale * src[(((size_t)fb * items + it) * q + x) * 32 + lane];
  }
}

// ============================================================== launchers
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
  const int grid = (int)std::max<long long>(1, std::min<long long>((tasks + 7) / 8, (long long)sm_count() * 8));
  if (a.c.q * a.c.q > 48 * 1024)
    cudaFuncSetAttribute(k_syndrome, cudaFuncAttributeMaxDynamicSharedMemorySize, a.c.q * a.c.q);
  k_syndrome<<<grid, threads, a.c.q * a.c.q, s>>>(a);
  return check_launch("k_syndrome");
}

int launch_init_msgs(const WaveArgs &a, cudaStream_t s) {
  k_init_msgs<<<sm_count() * 8, 256, 0, s>>>(a);
  return check_launch("k_init_msgs");
}

int launch_init_state(const WaveArgs &a, cudaStream_t s) {
  const int n = a.nfb * 32;
  k_init_state<<<(n + 255) / 256, 256, 0, s>>>(a);
  return check_launch("k_init_state");
}

int launch_test(const WaveArgs &a, cudaStream_t s) {
  // chunks of checks per warp task: enough tasks to give every SM 32 warps
  const long long work = (long long)a.nfb * a.c.M;
  const int chunk = (int)std::max<long long>(1, std::min<long long>(64, work / ((long long)sm_count() * 32)));
  const int threads = 256;
  const long long tasks = (long long)a.nfb * ((a.c.M + chunk - 1) / chunk);
  const int grid = (int)std::max<long long>(1, std::min<long long>((tasks + 7) / 8, (long long)sm_count() * 8));
  if (a.c.q * a.c.q > 48 * 1024)
    cudaFuncSetAttribute(k_test, cudaFuncAttributeMaxDynamicSharedMemorySize, a.c.q * a.c.q);
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

size_t repack_plan_bytes(int fbw) {
  const size_t n = (size_t)fbw;
  // hdr[64] dst[n] map[32n] cnt[n] amask[n] role[n] dpre[n+1] dblk[n] rpre[n]
  return (64 + n * 32 + n * 7 + 1 + 63) * sizeof(int);
}

RepackPlan repack_plan_at(void *base, int fbw) {
  RepackPlan rp;
  int *p = (int *)base;
  const size_t n = (size_t)fbw;
  rp.hdr = p; p += 64;
  rp.map = p; p += n * 32;
  rp.dst = p; p += n;
  rp.cnt = p; p += n;
  rp.amask = (unsigned *)p; p += n;
  rp.role = p; p += n;
  rp.dpre = p; p += n + 1;
  rp.dblk = p; p += n;
  rp.rpre = p;
  return rp;
}

int launch_repack(const WaveArgs &a, const RepackPlan &rp, float *qs, cudaStream_t s) {
  k_repack_plan<<<1, 1024, 0, s>>>(a, rp);
  int rc = check_launch("k_repack_plan");
  if (rc) return rc;
  MoveSet ms;
  int n = 0;
  auto add = [&](void *base, long long rows, int esz) {
    if (base && rows > 0) { ms.base[n] = base; ms.rows[n] = rows; ms.esz[n] = esz; ++n; }
  };
  add(a.qmsg, a.c.E * a.c.q, 4);
  add(a.pi, (long long)a.c.M * a.c.p, 4);
  add(qs, (long long)a.c.N * a.c.q, 4);
  add(a.z, a.c.M, 1);
  add(a.xhat, a.c.V, 1);
  ms.n = n;
  for (int k = n; k < 5; ++k) { ms.base[k] = nullptr; ms.rows[k] = 0; ms.esz[k] = 4; }
  k_repack_move<<<sm_count() * 8, 256, 0, s>>>(rp, ms);
  return check_launch("k_repack_move");
}

int launch_export(const WaveArgs &a, float *q_out, float *r_out, float *Q_out, cudaStream_t s) {
  const int threads = 256;
  const int grid = sm_count() * 8;
  // q messages live in check-major edge order, r messages in canonical order
  // (r is stored as q * r: the kernels drop the 1/q of the inverse transform)
  if (q_out) k_export<<<grid, threads, 0, s>>>(a, a.qmsg, q_out, (int)a.c.E, a.c.col_edge, 1.0f);
  if (r_out) k_export<<<grid, threads, 0, s>>>(a, a.rmsg, r_out, (int)a.c.E, nullptr, 1.0f / a.c.q);
  if (Q_out) k_export<<<grid, threads, 0, s>>>(a, a.qall, Q_out, a.c.V, nullptr, 1.0f);
  return check_launch("k_export");
}

int launch_trace(const WaveArgs &a, const unsigned char *truth, int *trace, int t, int tlen, cudaStream_t s) {
  k_trace<<<a.nfb, 256, 0, s>>>(a, truth, trace, t, tlen);
  return check_launch("k_trace");
}

int launch_trace_fill(int *trace, int n_frames, int tlen, cudaStream_t s) {
  k_trace_fill<<<(n_frames + 255) / 256, 256, 0, s>>>(trace, n_frames, tlen);
  return check_launch("k_trace_fill");
}

int launch_set_u64(unsigned long long *p, unsigned long long v, cudaStream_t s) {
  k_set_u64<<<1, 1, 0, s>>>(p, v);
  return check_launch("k_set_u64");
}

}  // namespace gfq

// gfq_internal.cuh -- shared declarations of the libgfq CUDA implementation.
//
// Data layout in HBM: frames are processed in
// blocks of 32 (one frame per lane: every warp of a task works on the same
// check / variable for 32 different frames, so all control flow and all
// graph indices are warp-uniform).  Every per-frame quantity is stored as
// [frame block][item][entry][32 lanes], so one (item, entry) row of a block
// is a contiguous 128-byte line (floats) and any per-edge permutation of a
// q-vector's entries is just a choice of which rows to load or store.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/gfq.h"

namespace gfq {

constexpr int kLanes = 32;  // frames per block
constexpr int kMaxDeg = 8;  // supported check / variable degree

// -------------------------------------------------------------- static task tables
// Per-task metadata that the hot kernels fetch with the Tensor Memory
// Accelerator together with the messages (so consumer warps never wait on a
// dependent global load).  Built once per code by gfq_code_create.
struct __align__(128) CheckDesc {      // one per check i (PUS check node)
  unsigned long long perm[kMaxDeg];    // packed basis images h^-1 * 2^b of edge row_ptr[i]+s
  int canon[kMaxDeg];                  // canonical (variable-major) position of that edge
};
struct __align__(64) VarDesc {         // one per variable j (variable node)
  int qdst[kMaxDeg];                   // check-major id of the edge of check slot s
};
struct __align__(64) SusDesc {         // one per canonical edge (j, s) (SUS unit)
  unsigned long long perm_o[kMaxDeg - 1];  // other edges of the check, row order, skipping e
  unsigned long long perm_e;               // the edge itself
};
struct __align__(16) LvlCol {          // SUS level schedule, level order
  int j, e0, dv, unit0;                // column, its first canonical edge, degree, first unit
};
struct __align__(32) LvlUnit {         // one per (column, check slot) in level order
  int r0, d, pos, i;                   // check row start / degree, position of e in the row, check
  int j, e0, dv, s;                    // its column, the column's first canonical edge and degree, slot
};
static_assert(sizeof(CheckDesc) == 128 && sizeof(VarDesc) == 64 && sizeof(SusDesc) == 64, "desc sizes");

// -------------------------------------------------------------- code object
struct HostGraph {             // host copy of the graph maps (level schedules per call)
  int N, M, V;
  long long E;
  std::vector<int> row_ptr, col_ptr, col_edge, edge_check;
};
int build_levels(const HostGraph &g, const int *order, bool chain, std::vector<int> &level_ptr,
                 std::vector<LvlCol> &lcol, std::vector<LvlUnit> &lunit);

struct DevCode {
  int p, q, N, M, V;
  long long E;
  int max_cdeg, max_vdeg;
  const int *row_ptr;        // [M+1]   edges of check i: row_ptr[i]..row_ptr[i+1]-1
  const int *edge_var;       // [E]     variable j of edge e (check-major edge ids)
  const int *edge_check;     // [E]     check i of edge e
  const unsigned long long *edge_perm;  // [E] packed bytes h_e^-1 * 2^b, b < p
  const unsigned char *edge_coef;       // [E] h_e
  const int *col_ptr;        // [V+1]
  const int *col_edge;       // [E]     edges of variable j (ascending check) == canonical order
  const int *edge_canon;     // [E]     canonical (variable-major) position of edge e
  const int *level_ptr;      // [L+1]   SUS dependency levels
  const int *level_cols;     // [V]
  const unsigned char *mul;  // [q*q]   GF(2^p) product table
  const unsigned short *rowtab;  // [q*q] (a * y) << 7: byte offset of row a*y of a q x 128 B message
  const CheckDesc *check_desc;  // [M]
  const VarDesc *var_desc;      // [V]
  const SusDesc *sus_desc;      // [E] canonical order
  const LvlCol *lvl_col;        // [V] level order (level_ptr delimits levels)
  const LvlUnit *lvl_unit;      // [U] U = sum over columns of max(dv, 1)
  const int *peel;              // [2M] encoder order: (row, noise column solved), or null
  const unsigned char *inv;     // [q]   GF(2^p) inverses (inv[0] = 0)
};

}  // namespace gfq

struct gfq_code {
  int p, q, N, M, V;
  unsigned poly;
  long long E;
  int max_cdeg, max_vdeg, n_levels;
  int device;
  std::vector<int> level_ptr_h;
  int n_levels_gs;                  // the level schedule with the in-sweep prior chain (A34)
  std::vector<int> level_ptr_gs_h;
  const gfq::LvlCol *lvl_col_gs;    // device, same layout as DevCode::lvl_col
  const gfq::LvlUnit *lvl_unit_gs;
  gfq::HostGraph hg;
  long long n_units;                // U = sum over columns of max(dv, 1)
  void *dev_blob;  // one cudaMalloc holding every device table
  gfq::DevCode d;
};

namespace gfq {

void set_error(const std::string &msg);
int cuda_fail(cudaError_t e, const char *what);

// -------------------------------------------------------------- workspace
struct Layout {
  int fbw;            // frame blocks per wave
  size_t qmsg, rmsg, pi, hard, z, xhat, qs0, qs1, qall, iters, conv, unsat, newconv;
  size_t active, list, nactive, stats, T, Tf, pi0, ord_col, ord_unit, total;
  size_t fid, rp;     // lane slot -> frame of the wave; frame-compaction plan (RepackPlan header + tables)
};

// Frame-granular early-exit compaction (gfq_kernels.cu: k_repack_plan,
// k_repack_move): the plan of one round, in the workspace.
//   [0] n_dst  [1] blocks before  [2] blocks after  [3] frames moved
// followed by dst[fbw] (destination block of plan entry k), map[fbw*32]
// (entry k, lane l: source slot block*32+lane, or -1 = keep), and scratch.
struct RepackPlan {
  int *hdr;       // [4]
  int *dst;       // [fbw]
  int *map;       // [fbw*32]
  int *cnt;       // [fbw]  live index -> number of still-decoding frames
  unsigned *amask;  // [fbw]  live index -> their lanes
  int *role;      // [fbw]  live index -> 1 donor, 0 receiver
  int *dpre;      // [fbw+1] donor index -> frames in the donors before it
  int *dblk;      // [fbw]  donor index -> live index
  int *rpre;      // [fbw]  live index -> idle lanes in the receivers before it
};
size_t repack_plan_bytes(int fbw);
RepackPlan repack_plan_at(void *base, int fbw);
Layout make_layout(const gfq_code *c, int fbw, const gfq_params *prm);

// -------------------------------------------------------------- kernel args
struct WaveArgs {
  DevCode c;
  int fb0;          // first frame block of this wave (global)
  int nfb;          // blocks in this wave
  int n_frames;     // total frames of the call
  float *qmsg;      // [nfb][E][q][32]
  float *rmsg;      // [nfb][E][q][32] or null (SUS without keep)
  float *pi;        // [nfb][M*p][32] per-bit flip probability
  unsigned char *hard;  // [nfb][M*p][32]
  unsigned char *z;     // [nfb][M][32]
  unsigned char *xhat;  // [nfb][V][32]
  float *qs_old, *qs_new;  // [nfb][N][q][32] Markov posterior snapshots (or null)
  float *qall;          // [nfb][V][q][32] or null
  int *iters;           // [nfb*32] first passing t, -1
  int *conv;            // [nfb*32] 1 once converged (or invalid lane)
  int *unsat;           // [nfb*32]
  int *newconv;         // [nfb*32]
  int *active;          // [nfb]
  int *list;            // [nfb] active block ids (wave-local)
  int *nactive;         // [1]
  int *fid;             // [nfb*32] frame of the wave decoded in this lane slot, -1 = none
  unsigned long long *stats;  // [4]
  const double *T;      // [q*q] or null
  const float *Tf;      // [2*q*q] fp32 copies of T (row-major) and of T^T, or null
  const double *pi0;    // [q]
  int markov;
  int gs;               // SUS with the Markov prior refreshed inside the sweep (A34)
  int tj;               // T = alpha I + beta 1 1^T exactly: O(q) prior sums
  float tj_alpha, tj_beta;
  int t;                // current iteration (1-based)
  int early_exit;
};

// launchers (gfq_kernels.cu)
int launch_frontend(const WaveArgs &a, int mode, double ch_param, const void *obs,
                    const unsigned char *hard_in, const float *pi_in, cudaStream_t s);
int launch_syndrome(const WaveArgs &a, cudaStream_t s);
int launch_init_msgs(const WaveArgs &a, cudaStream_t s);
int launch_init_state(const WaveArgs &a, cudaStream_t s);
int launch_cn(const WaveArgs &a, cudaStream_t s);
int launch_vn(const WaveArgs &a, cudaStream_t s);
int launch_sus_level(const WaveArgs &a, int level, int ncols, cudaStream_t s);
bool sus_dc_applies(const WaveArgs &a);   // gfq_sus_dc.cu
int launch_sus_dc(const WaveArgs &a, int level, int ncols, cudaStream_t s);
bool cn_dc_applies(const WaveArgs &a);    // gfq_sus_dc.cu: PUS check node by direct convolution (q = 8, 16)
int launch_cn_dc(const WaveArgs &a, cudaStream_t s);
bool sus_dc64_applies(const WaveArgs &a); // gfq_sus_dc64.cu: q = 64 by direct convolution
int launch_sus_dc64(const WaveArgs &a, int level, int ncols, cudaStream_t s);
bool big_applies(const WaveArgs &a);      // gfq_bigq.cu: q = 256
int launch_big_cn(const WaveArgs &a, cudaStream_t s);
int launch_big_vn(const WaveArgs &a, int clip_only, cudaStream_t s);
int launch_big_sus(const WaveArgs &a, int level, int ncols, cudaStream_t s);
int launch_test(const WaveArgs &a, cudaStream_t s);
int launch_finalize(const WaveArgs &a, int final_pass, cudaStream_t s);
int launch_capture(const WaveArgs &a, unsigned char *out, int L, int mode, cudaStream_t s);
int launch_compact(const WaveArgs &a, cudaStream_t s);
// frame-granular compaction: plan (which frames move where) and move; qs = the
// posterior snapshot the next iteration reads (or null)
int launch_repack(const WaveArgs &a, const RepackPlan &rp, float *qs, cudaStream_t s);
int launch_clip_priors(const WaveArgs &a, cudaStream_t s);
int launch_export(const WaveArgs &a, float *q_out, float *r_out, float *Q_out, cudaStream_t s);
int launch_set_u64(unsigned long long *p, unsigned long long v, cudaStream_t s);
int launch_trace(const WaveArgs &a, const unsigned char *truth, int *trace, int t, int tlen, cudaStream_t s);
int launch_trace_fill(int *trace, int n_frames, int tlen, cudaStream_t s);

// Monte-Carlo front end (gfq_sim.cu)
struct SimArgs {
  DevCode c;
  int n_frames, nfb;
  unsigned long long seed;
  long long frame0;
  int channel;
  double param;
  int markov;
  const double *cum0;   // [q]   running sums of pi0 (device)
  const double *cumT;   // [q*q] running sums of the rows of T (device)
  unsigned char *s_blk; // [nfb][N][32]
  unsigned char *t_blk; // [nfb][M][32]
  unsigned char *s_out; // [F][N]
  unsigned char *t_fm;  // [F][M]
  void *obs;            // [F][M*p]
};
int launch_sim(const SimArgs &a, cudaStream_t s);

}  // namespace gfq

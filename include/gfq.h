/*
 * gfq.h -- C ABI of libgfq: batched belief-propagation decoding of
 * MacKay-Neal codes over GF(2^p) (q = 2^p = 2..256) on one NVIDIA B200.
 *
 * Method: Yacov, Efraim, Kfir, Kanter, Shental, "Parallel vs. Sequential
 * Belief Propagation Decoding of LDPC Codes over GF(q) and Markov Sources"
 * (PAPER.md; cited P:line).  The decoder is given the code H = [A B]
 * (P:121-126), a batch of received frames and the prior knowledge
 * of source and channel, and recovers x = [s; n] from the syndrome z = B r
 * (Eq. 2) by BP with the parallel (PUS) or sequential
 * (SUS) updating scheme, with dynamical Markov block priors
 * (Eqs. 6/7) for correlated sources.
 *
 * Conventions (all calls):
 *   - Return 0 (GFQ_OK) or a negative GFQ_E* code; no exception crosses the
 *     ABI.  gfq_last_error() returns a thread-local message for the last failure.
 *   - GF(2^p) symbols are bytes; element a has polynomial-basis bits LSB first,
 *     bit b of symbol k is transmitted bit k*p + b (reading A2).
 *   - "device" pointers are CUDA device memory on the current device; "host"
 *     pointers are ordinary (pageable or pinned) host memory.
 *   - Every decode call is asynchronous on `stream` (a cudaStream_t passed as
 *     void*, NULL = legacy default stream) unless documented otherwise; its
 *     outputs are valid once that stream has been synchronised.
 *   - The library owns only the code object.  All per-decode buffers (inputs,
 *     outputs, workspace) are allocated and owned by the caller; the decode
 *     path never calls cudaMalloc.
 *   - Decoding is deterministic: identical inputs on the same GPU give
 *     identical outputs.
 *   - There is no CPU fallback: without a usable CUDA device every decode call
 *     fails with GFQ_ECUDA.
 */
#ifndef GFQ_H
#define GFQ_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GFQ_OK 0
#define GFQ_EINVAL (-1)       /* bad argument (see each call)                  */
#define GFQ_ENOMEM (-2)       /* host or device allocation failed (create only) */
#define GFQ_ECUDA (-3)        /* CUDA runtime error (message has the details)   */
#define GFQ_EUNSUPPORTED (-4) /* valid but not implemented (p > 8, degree > 8)   */

typedef enum { GFQ_BSC = 0, GFQ_BEC = 1, GFQ_BIAWGN = 2 } gfq_channel;
typedef enum { GFQ_PUS = 0, GFQ_SUS = 1 } gfq_schedule;
typedef enum { GFQ_PRIOR_SNAPSHOT = 0, GFQ_PRIOR_IN_SWEEP = 1 } gfq_prior_update;
typedef enum { GFQ_COMPACT_FRAMES = 0, GFQ_COMPACT_BLOCKS = 1 } gfq_compaction;

/* Opaque, immutable after creation; may be shared by concurrent decodes on
 * different streams (each with its own workspace). */
typedef struct gfq_code gfq_code;

typedef struct {
    /* Channel of the received bits:
     *   GFQ_BSC:    ch_param = flip probability f, 0 < f < 1/2.
     *   GFQ_BEC:    ch_param = erasure probability (informational; an erased
     *               bit carries no evidence: likelihood 1/2 each, reading A15).
     *   GFQ_BIAWGN: ch_param = noise standard deviation sigma > 0 for
     *               unit-energy BPSK 0 -> +1, 1 -> -1 (reading A16). */
    int channel;
    double ch_param;
    int schedule;      /* GFQ_PUS or GFQ_SUS          */
    int max_iters;     /* >= 0; 0 returns iters = -1 and the clipped priors    */
    int early_exit;    /* 1: a frame stops at the first iteration t with
                          H x = z; 0: every frame runs exactly
                          max_iters iterations (throughput / parity mode) and
                          still reports the first passing t.                  */
    const double *markov_T; /* host, q*q row-stochastic T[a*q+b] = Pr(b | a),
                               the "measured Markov transition matrix"
                               (reading A13), or NULL = i.i.d.     */
    const double *src_pi0;  /* host, q: prior of the first source symbol and of
                               every source symbol for i.i.d. sources
                               (P:224-226); NULL = uniform 1/q.               */
    int keep_messages; /* 1: keep the final q, r messages and all posteriors Q
                          in the workspace for gfq_export_messages (needs a
                          workspace sized with the same flag).                */
    /* Optional instrumentation of the paper's Fig. 1, device
     * pointers, both NULL to disable (gfq_decode and gfq_decode_evidence only;
     * gfq_decode_host rejects them):
     *   trace_truth uint8 [n_frames][N]: the true source symbols s;
     *   trace       int32 [n_frames][max_iters+1] out: trace[f][t] = number of
     *               source bits (N*p per frame, bits as in A2) of the estimate
     *               x^(t) equal to s -- t = 0 the clipped priors, t >= 1 the
     *               clipped pseudo-posterior after iteration t.
     *               After a frame stops (early_exit) its estimate is frozen
     *               and the count repeats up to max_iters.
     * The count is taken on the device after every iteration (one extra
     * kernel reading N bytes of estimates per frame). */
    const unsigned char *trace_truth;
    int *trace;
    /* When the Markov source prior is refreshed (markov_T != NULL only):
     *   GFQ_PRIOR_SNAPSHOT (0): after every iteration, p^(t) = Eq. (7) of the
     *     posterior snapshot Q^(t), used by the vertical pass of iteration t+1
     *     (reading A9) -- both schedules;
     *   GFQ_PRIOR_IN_SWEEP (1): SUS only -- "during the vertical pass"
     *     (reading A34): just before source column j is updated, p_j
     *     = Eq. (7) from the posterior of j-1 computed earlier in THIS sweep
     *     and that of j+1 from the previous sweep (none in sweep 1: factor 1);
     *     boundaries as A10.  The source columns then form a chain, so the
     *     sweep runs about N dependency levels instead of ~13.
     * GFQ_EINVAL for other values or GFQ_PRIOR_IN_SWEEP with PUS. */
    int prior_update;
    /* SUS column order (reading A35), host: sus_n_orders >= 1
     * permutations of 0..N+M-1, row-major [sus_n_orders][N+M]; sweep t
     * (1-based) visits the columns in row (t-1) mod sus_n_orders (P:198-216
     * with that order in place of the index order).  NULL / 0 = index order
     * (A7).  Random numbers the order is drawn from are the caller's.  The
     * dependency levels of every order are built on the host per call and
     * copied into the workspace (size it with the same params).  GFQ_EINVAL
     * if a row is not a permutation, with PUS (whose updates do not depend on
     * any order, A6) or with GFQ_PRIOR_IN_SWEEP (defined along index order). */
    const int *sus_order;
    int sus_n_orders;
    /* Early-exit compaction (a frame stops at its first passing
     * test; early_exit = 1 only).  Frames are decoded 32 to a block, one per
     * lane, and a block keeps iterating until its slowest frame stops:
     *   GFQ_COMPACT_FRAMES (0, default): when enough lanes have gone idle, the
     *     still-decoding frames of the sparsest blocks are moved (messages,
     *     evidence, syndrome, estimate, posterior snapshot) into the idle
     *     lanes of the others, so the blocks that keep iterating stay full;
     *   GFQ_COMPACT_BLOCKS (1): only blocks whose frames have all stopped are
     *     dropped.
     * A frame's arithmetic does not depend on its lane or on the other frames
     * of its block, so both settings give bit-identical s_hat / iters; they
     * differ in stats[1] (block iterations executed) and in time.  Ignored
     * (blocks) with keep_messages = 1, whose export addresses frames by their
     * original lane.  GFQ_EINVAL for other values. */
    int compaction;
} gfq_params;

/* Thread-local description of the last error (never NULL). */
const char *gfq_last_error(void);

/* ABI version: 0x010000 * major + 0x100 * minor + patch. */
int gfq_version(void);

/* Build a code object from the two sparse matrices of the MN code
 * (P:121-126): A is M x N, B is M x M, both in host COO form with 0-based
 * (row, col) and GF(2^p) values in 1..q-1.  H = [A B] (Eq. 2): check i is
 * row i; variable j < N is source symbol s_j, variable N + k is noise symbol
 * n_k (B column k).  prim_poly is the primitive polynomial of GF(2^p) with
 * the x^p term (e.g. 0x43 = x^6+x+1).  The host arrays are copied; the
 * device tables (check-major and variable-major edge maps, coefficient
 * permutations, SUS dependency levels) are uploaded to the current device.
 * B's invertibility is NOT checked: decoding needs only H and z; it matters
 * to the encoder (Eq. 1) only.
 * Errors: GFQ_EINVAL for p < 1, N < 0, M < 1, a polynomial that is not
 * primitive of degree p, an index out of range, a value 0 or >= q, or a
 * duplicate (row, col); GFQ_EUNSUPPORTED for p > 8 or a check/variable degree
 * > 8; GFQ_ENOMEM / GFQ_ECUDA from allocation or upload.  *out is set only on
 * success. */
int gfq_code_create(gfq_code **out, int p, unsigned prim_poly, int N, int M,
                    long long nnzA, const int *A_row, const int *A_col,
                    const unsigned char *A_val, long long nnzB, const int *B_row,
                    const int *B_col, const unsigned char *B_val);

/* Release a code object (NULL is a no-op).  No decode may be in flight. */
void gfq_code_destroy(gfq_code *code);

/* Sizes of the Tanner graph: E = nnz(H), maximum check / variable degree, and
 * the number of SUS dependency levels (columns sharing no check commute; the
 * sequential sweep executes level by level).  NULL outputs are
 * skipped. */
int gfq_code_info(const gfq_code *code, long long *n_edges, int *max_check_deg,
                  int *max_var_deg, int *sus_levels);

/* Bytes of device workspace that decode n_frames frames in ONE wave with these
 * params.  A smaller workspace (but at least gfq_workspace_bytes(code, 1, p))
 * is accepted by the decode calls, which then process the frames in waves of
 * as many 32-frame blocks as fit.  Returns 0 on bad arguments. */
size_t gfq_workspace_bytes(const gfq_code *code, int n_frames, const gfq_params *params);

/* Decode a batch from channel outputs (device pointers):
 *   obs:   GFQ_BSC    uint8 [n_frames][M*p] received bits 0/1;
 *          GFQ_BEC    uint8 [n_frames][M*p] 0/1, or 2 = erased;
 *          GFQ_BIAWGN float [n_frames][M*p] received values y.
 *   s_hat: uint8 [n_frames][N] out: decoded source symbols (clipped
 *          pseudo-posterior) at the iteration reported in iters,
 *          or at the last iteration if the frame never converged.
 *   iters: int32 [n_frames] out: first t in 1..max_iters with H x = z
 *          (P:190-194), or -1 if none (reading A21).
 *   workspace / ws_bytes: device scratch (>= gfq_workspace_bytes(code, 1, p)).
 * Errors: GFQ_EINVAL for NULL code/params/pointers, n_frames < 0, bad
 * channel/schedule, max_iters < 0, a markov_T row not stochastic, ws_bytes too
 * small, or keep_messages with a workspace that cannot hold all frames;
 * GFQ_ECUDA on a launch failure (no device, bad pointer). */
int gfq_decode(const gfq_code *code, int n_frames, const void *obs,
               const gfq_params *params, unsigned char *s_hat, int *iters,
               void *workspace, size_t ws_bytes, void *stream);

/* Lower-level entry with the channel front end supplied by the caller
 * (device pointers): hard_bits uint8 [n_frames][M*p] hard decisions r_b and
 * bit_flip_prob float [n_frames][M*p] the probability pi_b that noise bit n_b
 * is 1 (r = t + n mod 2).  params->channel/ch_param are ignored.
 * x_hat: uint8 [n_frames][N+M] out: the whole estimate x = [s; n]. */
int gfq_decode_evidence(const gfq_code *code, int n_frames, const unsigned char *hard_bits,
                        const float *bit_flip_prob, const gfq_params *params,
                        unsigned char *x_hat, int *iters, void *workspace,
                        size_t ws_bytes, void *stream);

/* End-to-end entry with HOST buffers: obs (layout as gfq_decode) is copied to
 * the device, decoded, and s_hat / iters are copied back; the call returns
 * after synchronising `stream`.  The workspace must be large enough to hold
 * the device copy of obs in addition to gfq_workspace_bytes for one wave:
 * size it with gfq_workspace_bytes_host. */
size_t gfq_workspace_bytes_host(const gfq_code *code, int n_frames, const gfq_params *params);
int gfq_decode_host(const gfq_code *code, int n_frames, const void *obs_host,
                    const gfq_params *params, unsigned char *s_hat_host, int *iters_host,
                    void *workspace, size_t ws_bytes, void *stream);

/* Export the messages left in the workspace by the last decode made with
 * keep_messages = 1 (all frames in one wave), in the probability domain and
 * canonical edge order (column-major: j ascending, then i ascending), all
 * device pointers, NULL to skip:
 *   q_msg [n_frames][E][q]  q_ij^a after the last iteration (Eq. 4),
 *   r_msg [n_frames][E][q]  r_ij^a last computed (Eq. 3; SUS: in the last sweep),
 *   Q     [n_frames][N+M][q] pseudo-posteriors of the last iteration (Eq. 5).
 * For frames that stopped early (early_exit = 1) the values are those of the
 * iteration in which their 32-frame block stopped.  Errors: GFQ_EINVAL. */
int gfq_export_messages(const gfq_code *code, int n_frames, const void *workspace,
                        size_t ws_bytes, const gfq_params *params, float *q_msg,
                        float *r_msg, float *Q, void *stream);

/* Health counters of the last decode that used this workspace (host out,
 * synchronises `stream`): stats[0] vanished or non-finite normalisers replaced
 * by a uniform vector (reading A19; 0 on parity runs), stats[1] iterations
 * executed summed over 32-frame blocks, stats[2] frames converged, stats[3]
 * kernel launches issued by the decode. */
int gfq_decode_stats(const gfq_code *code, const void *workspace, size_t ws_bytes,
                     long long stats[4], void *stream);

/* ---------------------------------------------------------------------------
 * Monte-Carlo front end (the steps before the decoder): source,
 * encoding t = B^-1 A s (Eq. 1) and channel, on the device, so that BER
 * sweeps (Table 1) run at GPU speed.
 */
typedef struct {
    int channel;        /* GFQ_BSC (ch_param = f), GFQ_BEC (eps), GFQ_BIAWGN (sigma) */
    double ch_param;
    const double *markov_T; /* host q*q row-stochastic, or NULL = i.i.d. uniform source */
    const double *src_pi0;  /* host q, law of s_0 for a Markov source; NULL = uniform */
} gfq_sim_params;

/* Device workspace for gfq_simulate of n_frames frames (0 on bad arguments). */
size_t gfq_simulate_workspace_bytes(const gfq_code *code, int n_frames);

/* Frames frame0 .. frame0+n_frames-1 of the stream `seed` (device outputs):
 *   s_out   uint8 [n_frames][N]   source symbols (NULL to skip),
 *   obs_out [n_frames][M*p]       channel output in the layout gfq_decode takes
 *                                 (uint8 bits / {0,1,2=erased} / float32 y), or NULL,
 *   t_out   uint8 [n_frames][M]   codeword symbols t = B^-1 A s (NULL: kept in
 *                                 the workspace).
 * Random numbers (so that a CPU program can draw the same ones): Philox4x32-10
 * with key (seed mod 2^32, seed >> 32) and counter (j, frame mod 2^32,
 * frame >> 32, purpose), purpose 1 = source, 2 = channel; u24(x) = (x >> 8) 2^-24.
 *   i.i.d. source: symbol 4j+m = x_m mod q.
 *   Markov source: u_k = u24(x_m) for k = 4j+m; s_0 = min{b : u_0 < C0[b]},
 *     s_k = min{b : u_k < C[s_{k-1}][b]}, C0 / C the running sums (double, left
 *     to right, last entry set to 1) of pi0 and of the rows of T.
 *   BSC: transmitted bit 4j+m flips iff u24(x_m) < f;  BEC: erased (obs 2) iff
 *     u24(x_m) < eps;  BI-AWGN: bits 2j, 2j+1 from one call, u1 = ((x_0 >> 8)
 *     + 1) 2^-24, u2 = u24(x_1), rho = sqrt(-2 ln u1), noise rho cos(2 pi u2),
 *     rho sin(2 pi u2); y = (1 - 2 bit) + sigma * noise in float32 (A16).
 * Bits are LSB first (A2).  Errors: GFQ_EINVAL (bad arguments, workspace too
 * small), GFQ_EUNSUPPORTED if B is not triangular up to a permutation (the
 * encoder solves B t = A s by peeling rows with one unknown; the MN
 * construction's B always is), GFQ_ECUDA.  Asynchronous on `stream`. */
int gfq_simulate(const gfq_code *code, int n_frames, unsigned long long seed, long long frame0,
                 const gfq_sim_params *params, unsigned char *s_out, void *obs_out,
                 unsigned char *t_out, void *workspace, size_t ws_bytes, void *stream);

/* Per-kernel timing for roofline reporting.  gfq_profile_enable(1) makes every
 * later decode call of the calling thread record a CUDA event pair around each
 * kernel it launches, on the decode's stream (accumulators are reset);
 * gfq_profile_enable(0) stops recording.  gfq_profile_read synchronises the
 * recorded events and writes, per kernel kind k < GFQ_NKERNELS, the summed
 * duration in ms (ms[k]) and the number of launches (launches[k]); NULL outputs
 * are skipped.  gfq_kernel_name(k) names kind k ("cn", "vn", "sus", ...) or
 * returns NULL for k out of range. */
#define GFQ_NKERNELS 15
int gfq_profile_enable(int on);
int gfq_profile_read(double *ms, long long *launches);
const char *gfq_kernel_name(int kind);

#ifdef __cplusplus
}
#endif
#endif /* GFQ_H */

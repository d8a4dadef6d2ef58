/*
 * oracle.c -- plain, slow, fp64 CPU reference for BP decoding of MacKay-Neal
 * codes over GF(2^p) with the parallel (PUS) and sequential (SUS) schedules.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant with the CUDA path
 * (paper_cs_0605069_b200/csrc); the only common module is synth/ (inputs).
 *
 * Every function follows PAPER.md (cited "P:line", section/equation) in the
 * paper's order and notation; readings of silent or garbled points are the
 * DESIGN.md readings (A-numbers from SURVEY.md §8(c)).  No transform, no
 * blocking, no leave-one-out tricks: Eq. (3) is a direct sum over GF(q)
 * configurations done as sequential convolution, Eqs. (4)/(5) are direct
 * products, Eq. (6) is the literal double sum.
 *
 * Pins (tests/test_oracle_*.py) tie every function to something other than
 * itself: brute-force enumeration, closed forms, worked values, tree
 * exactness.  No function is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* GF(2^p) ("taken randomly from {1,..,q-1} in GF(q)", reading A1)  */
/* ------------------------------------------------------------------------ */

/* Polynomial multiplication of a and b, reduced modulo the primitive
 * polynomial `poly` (degree p), by shift-and-xor.  No log tables. */
int o_gf_mul(int a, int b, int p, unsigned poly)
{
    int q = 1 << p;
    int r = 0;
    while (b) {
        if (b & 1) r ^= a;
        b >>= 1;
        a <<= 1;
        if (a & q) a ^= (int)poly;
    }
    return r;
}

/* Multiplicative inverse by exhaustive search; 0 has none (returns 0). */
int o_gf_inv(int a, int p, unsigned poly)
{
    int q = 1 << p;
    for (int y = 1; y < q; ++y)
        if (o_gf_mul(a, y, p, poly) == 1) return y;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Channel front end (BSC/BEC/BI-AWGN readings A15, A16)          */
/* ------------------------------------------------------------------------ */
enum { O_BSC = 0, O_BEC = 1, O_BIAWGN = 2 };

/* Received bit -> hard decision r_b and probability pi_b that the noise bit
 * n_b is 1 (r = t + n mod 2).
 *   BSC:  r_b = obs, pi_b = f.
 *   BEC:  erased (2) -> r_b = 0, pi_b = 1/2; else r_b = obs, pi_b = 0.
 *   BI-AWGN (0 -> +1, 1 -> -1): r_b = [y < 0], pi_b = 1/(1+exp(2|y|/sigma^2)). */
void o_frontend(int channel, double param, const void *obs, long nbits,
                uint8_t *hard, double *pi)
{
    for (long b = 0; b < nbits; ++b) {
        if (channel == O_BSC) {
            hard[b] = ((const uint8_t *)obs)[b] & 1;
            pi[b] = param;
        } else if (channel == O_BEC) {
            uint8_t o = ((const uint8_t *)obs)[b];
            hard[b] = (o == 2) ? 0 : (o & 1);
            pi[b] = (o == 2) ? 0.5 : 0.0;
        } else {
            double y = (double)((const float *)obs)[b];
            hard[b] = (y < 0.0) ? 1 : 0;
            pi[b] = 1.0 / (1.0 + exp(2.0 * fabs(y) / (param * param)));
        }
    }
}

/* Noise-symbol prior: for BSC Q_j^a = f^L (1-f)^(log2 q - L),
 * L = number of 1s in the bits of a; generalised per bit:
 * p(a) = prod_b (bit_b(a) ? pi_b : 1 - pi_b), bits LSB first (A2). */
void o_noise_prior(int p, const double *pi_bits, double *out)
{
    int q = 1 << p;
    for (int a = 0; a < q; ++a) {
        double v = 1.0;
        for (int b = 0; b < p; ++b)
            v *= ((a >> b) & 1) ? pi_bits[b] : (1.0 - pi_bits[b]);
        out[a] = v;
    }
}

/* ------------------------------------------------------------------------ */
/* BP core                                                      */
/* ------------------------------------------------------------------------ */

/* Check-node (horizontal) update, Eq. (3):
 *   r_ij^a = sum over configurations {x_j'} of the other variables of check i
 *            with x_j = a satisfying z_i, of prod_{j' != j} q_ij'^{x_j'}.
 * "Satisfying z_i" means sum_j' h_ij' x_j' = z_i over GF(q) (reading A4);
 * addition is XOR.  Computed as a direct sum: S starts as the point mass at 0
 * and absorbs every other edge j' (ascending slot order) by
 *   S'(y) = sum_x q_ij'(x) S(y xor h_ij' x);
 * then r_ij(a) = S(z_i xor h_ij a).  d = degree, h[d] coefficients,
 * qin[d*q] incoming messages, out = slot of j.  O(d q^2). */
void o_check_node(int p, unsigned poly, int d, const int *h, const double *qin,
                  int z, int out, double *r)
{
    int q = 1 << p;
    double *S = (double *)calloc((size_t)q, sizeof(double));
    double *T = (double *)calloc((size_t)q, sizeof(double));
    int *hx = (int *)malloc(sizeof(int) * (size_t)q);
    S[0] = 1.0;
    for (int k = 0; k < d; ++k) {
        if (k == out) continue;
        /* the field products h_ij' x for every x (integer work only: the
         * floating-point sum below is the same, term for term and in order) */
        for (int x = 0; x < q; ++x) hx[x] = o_gf_mul(h[k], x, p, poly);
        for (int y = 0; y < q; ++y) T[y] = 0.0;
        for (int y = 0; y < q; ++y)
            for (int x = 0; x < q; ++x)
                T[y] += qin[k * q + x] * S[y ^ hx[x]];
        memcpy(S, T, sizeof(double) * (size_t)q);
    }
    for (int a = 0; a < q; ++a)
        r[a] = S[z ^ o_gf_mul(h[out], a, p, poly)];
    free(hx);
    free(S);
    free(T);
}

/* Variable-node (vertical) update, Eq. (4):
 *   q_ij^a = alpha_ij p_j^a prod_{i' != i} r_i'j^a,  sum_a q_ij^a = 1 (A3).
 * rin[dv*q] are the r's of all checks of j, out = slot of i.
 * Returns 1 (and a uniform vector) if the normaliser is 0 (reading A19). */
int o_var_node(int q, int dv, const double *prior, const double *rin, int out,
               double *qout)
{
    double s = 0.0;
    for (int a = 0; a < q; ++a) {
        double v = prior[a];
        for (int k = 0; k < dv; ++k)
            if (k != out) v *= rin[k * q + a];
        qout[a] = v;
        s += v;
    }
    if (!(s > 0.0) || !isfinite(s)) {
        for (int a = 0; a < q; ++a) qout[a] = 1.0 / q;
        return 1;
    }
    for (int a = 0; a < q; ++a) qout[a] /= s;
    return 0;
}

/* Tie tolerance of the clipping step (reading A17 in DESIGN.md): values that
 * agree to fp64 round-off (relative 1e-12) are ties; anything farther apart is
 * decided by the strict argmax.  Exact ties (BEC coset-uniform posteriors, an
 * all-erased frame) come out of this sum at round-off scale only. */
#define O_TIE_REL 1e-12

/* Pseudo-posterior, Eq. (5): Q_j^a = alpha_j p_j^a prod_i r_ij^a,
 * then "clipping": x_j = the a maximising Q_j (ties -> smallest a, where
 * values within fp64 round-off, relative O_TIE_REL, of the maximum are ties, A17).
 * Returns x_j; *zero_norm set to 1 if the normaliser vanished (A19). */
int o_posterior(int q, int dv, const double *prior, const double *rin,
                double *Q, int *zero_norm)
{
    double s = 0.0;
    for (int a = 0; a < q; ++a) {
        double v = prior[a];
        for (int k = 0; k < dv; ++k) v *= rin[k * q + a];
        Q[a] = v;
        s += v;
    }
    *zero_norm = 0;
    if (!(s > 0.0) || !isfinite(s)) {
        for (int a = 0; a < q; ++a) Q[a] = 1.0 / q;
        *zero_norm = 1;
    } else {
        for (int a = 0; a < q; ++a) Q[a] /= s;
    }
    /* ties -> smallest a; values equal up to fp64 round-off (relative O_TIE_REL) are ties */
    double mx = 0.0;
    for (int a = 0; a < q; ++a)
        if (Q[a] > mx) mx = Q[a];
    int best = 0;
    for (int a = 0; a < q; ++a)
        if (Q[a] >= mx * (1.0 - O_TIE_REL)) { best = a; break; }
    return best;
}

/* Dynamical Markov block prior, Eq. (6), written literally:
 *   P_i^b = sum_{a,c} Q_{i-1}^a M_ab M_bc Q_{i+1}^c       (0 < i < N-1)
 * with boundaries (reading A10): the left factor sum_a Q_{i-1}^a M_ab is
 * pi0(b) at i = 0; the right factor sum_c M_bc Q_{i+1}^c is 1 at i = N-1.
 * Normalised over b (A11).  Q is the post-iteration snapshot (A9). */
void o_markov_prior(int q, int N, const double *T, const double *pi0,
                    const double *Q, double *P)
{
    for (int i = 0; i < N; ++i) {
        double s = 0.0;
        for (int b = 0; b < q; ++b) {
            double v = 0.0;
            if (N == 1) {
                v = pi0[b];
            } else if (i == 0) {
                for (int c = 0; c < q; ++c)
                    v += pi0[b] * T[b * q + c] * Q[(size_t)(i + 1) * q + c];
            } else if (i == N - 1) {
                for (int a = 0; a < q; ++a)
                    v += Q[(size_t)(i - 1) * q + a] * T[a * q + b];
            } else {
                for (int a = 0; a < q; ++a)
                    for (int c = 0; c < q; ++c)
                        v += Q[(size_t)(i - 1) * q + a] * T[a * q + b] *
                             T[b * q + c] * Q[(size_t)(i + 1) * q + c];
            }
            P[(size_t)i * q + b] = v;
            s += v;
        }
        if (s > 0.0)
            for (int b = 0; b < q; ++b) P[(size_t)i * q + b] /= s;
    }
}

/* One symbol of Eq. (6) with the neighbours supplied separately (the prior
 * refreshed inside the SUS sweep, reading A34): left = Q of symbol i-1 or
 * NULL (left factor pi0(b), A10), right = Q of symbol i+1 or NULL (right
 * factor 1).  Normalised over b. */
void o_markov_prior_one(int q, const double *T, const double *pi0,
                        const double *left, const double *right, double *P)
{
    double s = 0.0;
    for (int b = 0; b < q; ++b) {
        double v = 0.0;
        if (!left && !right) {
            v = pi0[b];
        } else if (!left) {
            for (int c = 0; c < q; ++c) v += pi0[b] * T[b * q + c] * right[c];
        } else if (!right) {
            for (int a = 0; a < q; ++a) v += left[a] * T[a * q + b];
        } else {
            for (int a = 0; a < q; ++a)
                for (int c = 0; c < q; ++c) v += left[a] * T[a * q + b] * T[b * q + c] * right[c];
        }
        P[b] = v;
        s += v;
    }
    if (s > 0.0)
        for (int b = 0; b < q; ++b) P[b] /= s;
}

/* ------------------------------------------------------------------------ */
/* Code object: H = [A B]; rows = checks, columns = x = [s; n]   */
/* Canonical edge order: column-major (j ascending, then i ascending).      */
/* ------------------------------------------------------------------------ */
typedef struct {
    int p, q, N, M, V;
    unsigned poly;
    long E;
    int *col_ptr;    /* V+1 : edges of column j are col_ptr[j]..col_ptr[j+1]-1 */
    int *edge_row;   /* E   : check i of edge e                               */
    int *edge_col;   /* E   : variable j of edge e                            */
    int *edge_coef;  /* E   : H_ij                                            */
    int *row_ptr;    /* M+1                                                   */
    int *row_edge;   /* E   : edges of row i by ascending j                   */
} ocode;

ocode *o_code_create(int p, unsigned poly, int N, int M, long nnz,
                     const int *rows, const int *cols, const uint8_t *vals)
{
    ocode *c = (ocode *)calloc(1, sizeof(ocode));
    c->p = p; c->q = 1 << p; c->poly = poly; c->N = N; c->M = M; c->V = N + M;
    c->E = nnz;
    c->col_ptr = (int *)calloc((size_t)c->V + 1, sizeof(int));
    c->row_ptr = (int *)calloc((size_t)M + 1, sizeof(int));
    c->edge_row = (int *)malloc(sizeof(int) * (size_t)nnz);
    c->edge_col = (int *)malloc(sizeof(int) * (size_t)nnz);
    c->edge_coef = (int *)malloc(sizeof(int) * (size_t)nnz);
    c->row_edge = (int *)malloc(sizeof(int) * (size_t)nnz);
    /* counting sort by (col, row) */
    for (long k = 0; k < nnz; ++k) c->col_ptr[cols[k] + 1]++;
    for (int j = 0; j < c->V; ++j) c->col_ptr[j + 1] += c->col_ptr[j];
    int *fill = (int *)calloc((size_t)c->V, sizeof(int));
    for (long k = 0; k < nnz; ++k) {
        int j = cols[k];
        int e = c->col_ptr[j] + fill[j]++;
        c->edge_row[e] = rows[k];
        c->edge_col[e] = j;
        c->edge_coef[e] = vals[k];
    }
    free(fill);
    for (int j = 0; j < c->V; ++j) /* insertion sort rows within a column */
        for (int e = c->col_ptr[j] + 1; e < c->col_ptr[j + 1]; ++e)
            for (int f = e; f > c->col_ptr[j] && c->edge_row[f - 1] > c->edge_row[f]; --f) {
                int t = c->edge_row[f]; c->edge_row[f] = c->edge_row[f - 1]; c->edge_row[f - 1] = t;
                t = c->edge_coef[f]; c->edge_coef[f] = c->edge_coef[f - 1]; c->edge_coef[f - 1] = t;
            }
    for (long e = 0; e < nnz; ++e) c->row_ptr[c->edge_row[e] + 1]++;
    for (int i = 0; i < M; ++i) c->row_ptr[i + 1] += c->row_ptr[i];
    int *rfill = (int *)calloc((size_t)M, sizeof(int));
    for (long e = 0; e < nnz; ++e) { /* e runs in ascending j, so rows get ascending j */
        int i = c->edge_row[e];
        c->row_edge[c->row_ptr[i] + rfill[i]++] = (int)e;
    }
    free(rfill);
    return c;
}

void o_code_destroy(ocode *c)
{
    if (!c) return;
    free(c->col_ptr); free(c->row_ptr); free(c->edge_row); free(c->edge_col);
    free(c->edge_coef); free(c->row_edge); free(c);
}

long o_code_edges(const ocode *c) { return c->E; }

/* Syndrome z = B r (Eq. 2), computed on the B part of H: noise
 * columns N..N+M-1 carry B.  r_sym[M] are the received symbols. */
void o_syndrome(const ocode *c, const uint8_t *r_sym, uint8_t *z)
{
    for (int i = 0; i < c->M; ++i) {
        int acc = 0;
        for (int k = c->row_ptr[i]; k < c->row_ptr[i + 1]; ++k) {
            int e = c->row_edge[k];
            int j = c->edge_col[e];
            if (j >= c->N)
                acc ^= o_gf_mul(c->edge_coef[e], r_sym[j - c->N], c->p, c->poly);
        }
        z[i] = (uint8_t)acc;
    }
}

/* Convergence test: does x solve H x = z?  Returns #violated checks. */
int o_unsatisfied(const ocode *c, const uint8_t *x, const uint8_t *z)
{
    int bad = 0;
    for (int i = 0; i < c->M; ++i) {
        int acc = 0;
        for (int k = c->row_ptr[i]; k < c->row_ptr[i + 1]; ++k) {
            int e = c->row_edge[k];
            acc ^= o_gf_mul(c->edge_coef[e], x[c->edge_col[e]], c->p, c->poly);
        }
        bad += (acc != z[i]);
    }
    return bad;
}

/* r_ij for edge e from the current q's of check i's edges (Eq. 3). */
static void check_edge(const ocode *c, long e, const uint8_t *z, const double *qmsg,
                       double *scratch_q, int *scratch_h, double *r_out)
{
    int q = c->q;
    int i = c->edge_row[e];
    int d = c->row_ptr[i + 1] - c->row_ptr[i];
    int out = -1;
    for (int k = 0; k < d; ++k) {
        long ek = c->row_edge[c->row_ptr[i] + k];
        scratch_h[k] = c->edge_coef[ek];
        memcpy(scratch_q + (size_t)k * q, qmsg + (size_t)ek * q, sizeof(double) * (size_t)q);
        if (ek == e) out = k;
    }
    o_check_node(c->p, c->poly, d, scratch_h, scratch_q, z[i], out, r_out);
}

/* q_ij for edge e from p_j and the r's of column j (Eq. 4). */
static int var_edge(const ocode *c, long e, const double *prior_j, const double *rmsg,
                    double *qout)
{
    int q = c->q;
    int j = c->edge_col[e];
    int e0 = c->col_ptr[j];
    int dv = c->col_ptr[j + 1] - e0;
    return o_var_node(q, dv, prior_j, rmsg + (size_t)e0 * q, (int)(e - e0), qout);
}

/* Number of source bits of x (symbols 0..N-1, p bits each, A2) equal to the
 * true source s: the "percentage of correct bits" of Fig. 1 times
 * N*p/100. */
static int correct_source_bits(int p, int N, const uint8_t *x, const uint8_t *s)
{
    int ok = 0;
    for (int j = 0; j < N; ++j)
        for (int b = 0; b < p; ++b)
            ok += ((x[j] >> b) & 1) == ((s[j] >> b) & 1);
    return ok;
}

/* One frame, start to finish.
 *   schedule: 0 = PUS, 1 = SUS
 *   hard[M*p], pi[M*p]: front-end output (bits LSB first, A2)
 *   T[q*q] / pi0[q]: Markov source (NULL T = i.i.d.; NULL pi0 = uniform)
 *   fixed: 0 -> stop at the first t with H x = z (early exit); 1 -> always run
 *          max_iters (prior updated after every iteration), still recording the
 *          first passing t.  Output x is the estimate at that t, else the last.
 *   xhat[V] out; *iters out: first passing t in 1..max_iters or -1 (A21).
 *   qmsg/rmsg [E*q], Qpost [V*q]: optional (NULL) final messages, canonical order.
 *   *zero_norms: count of vanished normalisers (A19; should stay 0).
 *   s_true[N] / trace[max_iters+1]: optional (NULL) instrumentation of Fig. 1
 *          (P:296-317): trace[t] = number of source BITS of the estimate x^(t)
 *          equal to the true source s (t = 0: the clipped priors; t >= 1: after
 *          iteration t).  After an early exit at t0 the estimate is frozen, so
 *          trace[t] = trace[t0] for t > t0.
 *   sus_gs: SUS with a Markov source only -- the source prior refreshed inside
 *          the sweep (reading A34, "during the vertical pass"):
 *          just before column j < N is updated, p_j = Eq. (6) from the
 *          posterior of j-1 computed earlier in THIS sweep and the posterior of
 *          j+1 from the previous sweep (none at t = 1: right factor 1); no
 *          post-iteration refresh.  0: the post-iteration snapshot (A9).
 *   order, n_orders: SUS column order (reading A35): sweep t visits
 *          the columns order[((t-1) mod n_orders)*V + k], k = 0..V-1 (each a
 *          permutation of 0..V-1, drawn by the caller); NULL = index order (A7).
 *          Not combined with sus_gs (its "j-1 of this sweep" assumes index order).
 */
int o_decode_frame(const ocode *c, int schedule, int max_iters, int fixed,
                   const uint8_t *hard, const double *pi, const double *T,
                   const double *pi0_in, uint8_t *xhat, int *iters,
                   double *qmsg_out, double *rmsg_out, double *Q_out,
                   long *zero_norms, const uint8_t *s_true, int *trace, int sus_gs,
                   const int *order, int n_orders)
{
    const int p = c->p, q = c->q, N = c->N, M = c->M, V = c->V;
    const long E = c->E;
    double *prior = (double *)malloc(sizeof(double) * (size_t)V * q);
    double *qmsg = (double *)malloc(sizeof(double) * (size_t)E * q);
    double *rmsg = (double *)calloc((size_t)E * q, sizeof(double));
    double *Q = (double *)malloc(sizeof(double) * (size_t)V * q);
    double *pi0 = (double *)malloc(sizeof(double) * (size_t)q);
    const int gs = (sus_gs && schedule == 1 && T != NULL);
    double *Qprev = gs ? (double *)malloc(sizeof(double) * (size_t)V * q) : NULL;
    uint8_t *z = (uint8_t *)malloc((size_t)M);
    uint8_t *rsym = (uint8_t *)malloc((size_t)M);
    uint8_t *x = (uint8_t *)malloc((size_t)V);
    int maxd = 1;
    for (int i = 0; i < M; ++i)
        if (c->row_ptr[i + 1] - c->row_ptr[i] > maxd) maxd = c->row_ptr[i + 1] - c->row_ptr[i];
    double *scratch_q = (double *)malloc(sizeof(double) * (size_t)maxd * q);
    int *scratch_h = (int *)malloc(sizeof(int) * (size_t)maxd);
    long zn = 0;

    for (int a = 0; a < q; ++a) pi0[a] = pi0_in ? pi0_in[a] : 1.0 / q;
    /* Received symbols and syndrome z = B r (Eq. 2). */
    for (int k = 0; k < M; ++k) {
        int s = 0;
        for (int b = 0; b < p; ++b) s |= (hard[k * p + b] & 1) << b;
        rsym[k] = (uint8_t)s;
    }
    o_syndrome(c, rsym, z);
    /* Priors: source symbols Pr(s=a) (pi0 for Markov, A14),
     * noise symbols from the channel. */
    for (int j = 0; j < N; ++j)
        memcpy(prior + (size_t)j * q, pi0, sizeof(double) * (size_t)q);
    for (int k = 0; k < M; ++k)
        o_noise_prior(p, pi + (size_t)k * p, prior + (size_t)(N + k) * q);
    /* "Then we set q_ij^a = Q_j^a for all non-zero elements in the j'th column". */
    for (long e = 0; e < E; ++e)
        memcpy(qmsg + (size_t)e * q, prior + (size_t)c->edge_col[e] * q, sizeof(double) * (size_t)q);

    *iters = -1;
    if (max_iters <= 0 || trace) { /* clip the priors: the estimate x^(0) */
        for (int j = 0; j < V; ++j) {
            const double *pj = prior + (size_t)j * q;
            double mx = 0.0;
            for (int a = 0; a < q; ++a)
                if (pj[a] > mx) mx = pj[a];
            int best = 0;
            for (int a = 0; a < q; ++a)
                if (pj[a] >= mx * (1.0 - O_TIE_REL)) { best = a; break; }
            x[j] = (uint8_t)best;
            if (max_iters <= 0) {
                xhat[j] = (uint8_t)best;
                memcpy(Q + (size_t)j * q, prior + (size_t)j * q, sizeof(double) * (size_t)q);
            }
        }
        if (trace) {
            trace[0] = correct_source_bits(p, N, x, s_true);
            for (int t = 1; t <= max_iters; ++t) trace[t] = -1;
        }
    }
    for (int t = 1; t <= max_iters; ++t) {
        if (schedule == 0) {
            /* PUS horizontal pass: every r_ij from the previous iteration's q. */
            for (long e = 0; e < E; ++e)
                check_edge(c, e, z, qmsg, scratch_q, scratch_h, rmsg + (size_t)e * q);
            /* PUS vertical pass: every q_ij from the updated r's. */
            for (long e = 0; e < E; ++e)
                zn += var_edge(c, e, prior + (size_t)c->edge_col[e] * q, rmsg, qmsg + (size_t)e * q);
        } else {
            /* SUS: for each column j in index order (A7) or the given order (A35):
             * step 1: partial horizontal pass, r_ij for all i in column j, from the current q's;
             * step 2: partial vertical pass over column j. */
            if (gs && t > 1) memcpy(Qprev, Q, sizeof(double) * (size_t)V * q);
            const int *ord = (order && n_orders > 0) ? order + (size_t)((t - 1) % n_orders) * V : NULL;
            for (int k = 0; k < V; ++k) {
                const int j = ord ? ord[k] : k;
                for (int e = c->col_ptr[j]; e < c->col_ptr[j + 1]; ++e)
                    check_edge(c, e, z, qmsg, scratch_q, scratch_h, rmsg + (size_t)e * q);
                if (gs && j < N) /* within-sweep prior (A34) */
                    o_markov_prior_one(q, T, pi0, j > 0 ? Q + (size_t)(j - 1) * q : NULL,
                                       (t > 1 && j < N - 1) ? Qprev + (size_t)(j + 1) * q : NULL,
                                       prior + (size_t)j * q);
                for (int e = c->col_ptr[j]; e < c->col_ptr[j + 1]; ++e)
                    zn += var_edge(c, e, prior + (size_t)j * q, rmsg, qmsg + (size_t)e * q);
                if (gs && j < N) { /* Q_j now: the next column's left neighbour */
                    int e0 = c->col_ptr[j], zf;
                    o_posterior(q, c->col_ptr[j + 1] - e0, prior + (size_t)j * q, rmsg + (size_t)e0 * q,
                                Q + (size_t)j * q, &zf);
                }
            }
        }
        /* Pseudo-posterior Eq. (5) and clipping (SUS step 4, A8). */
        for (int j = 0; j < V; ++j) {
            int e0 = c->col_ptr[j], dv = c->col_ptr[j + 1] - e0, zf;
            x[j] = (uint8_t)o_posterior(q, dv, prior + (size_t)j * q, rmsg + (size_t)e0 * q,
                                        Q + (size_t)j * q, &zf);
            zn += zf;
        }
        if (trace) trace[t] = correct_source_bits(p, N, x, s_true);
        /* Convergence test. */
        int pass = (o_unsatisfied(c, x, z) == 0);
        if (pass && *iters < 0) {
            *iters = t;
            memcpy(xhat, x, (size_t)V);
        }
        if (pass && !fixed) break;
        if (*iters < 0) memcpy(xhat, x, (size_t)V);
        /* Re-estimate the source priors after the iteration (Eq. 6; A9). */
        if (T && !gs && t < max_iters) {
            double *P = (double *)malloc(sizeof(double) * (size_t)N * q);
            o_markov_prior(q, N, T, pi0, Q, P);
            memcpy(prior, P, sizeof(double) * (size_t)N * q);
            free(P);
        }
    }
    if (trace) /* early exit: the frozen estimate counts for the remaining iterations */
        for (int t = 1; t <= max_iters; ++t)
            if (trace[t] < 0) trace[t] = trace[t - 1];
    if (qmsg_out) memcpy(qmsg_out, qmsg, sizeof(double) * (size_t)E * q);
    if (rmsg_out) memcpy(rmsg_out, rmsg, sizeof(double) * (size_t)E * q);
    if (Q_out) memcpy(Q_out, Q, sizeof(double) * (size_t)V * q);
    if (zero_norms) *zero_norms = zn;
    free(prior); free(qmsg); free(rmsg); free(Q); free(pi0); free(z); free(rsym);
    free(x); free(scratch_q); free(scratch_h); free(Qprev);
    return 0;
}

// gfq_code.cu -- code object: validation, Tanner-graph maps, GF(2^p) tables,
// SUS dependency levels, upload.  Host C++ (runs once per code).
//
// H = [A B]: check i = row i, variable j < N = source
// symbol s_j, variable N + k = noise symbol n_k.  "The non-zero elements in a
// row i of H represent the [symbols] of x participating in check z_i; the
// non-zero elements in column j represent the checks in which the j'th
// [symbol] participates".
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "gfq_internal.cuh"

namespace gfq {

static thread_local std::string g_err = "no error";

void set_error(const std::string &msg) { g_err = msg; }

int cuda_fail(cudaError_t e, const char *what) {
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return GFQ_ECUDA;
}

// GF(2^p) log/antilog tables (the library's own; the oracle multiplies by
// shift-and-xor and the input generator has a third implementation).
struct GF {
  int p, q;
  std::vector<int> exp, log;
  bool build(int p_, unsigned poly) {
    p = p_;
    q = 1 << p;
    exp.assign(2 * q, 0);
    log.assign(q, -1);
    int a = 1;
    for (int k = 0; k < q - 1; ++k) {
      if (log[a] != -1) return false;  // x is not a generator -> not primitive
      exp[k] = a;
      log[a] = k;
      a <<= 1;
      if (a & q) a ^= (int)poly;
      if (a >= q || a == 0) return false;
    }
    if (a != 1) return false;
    for (int k = q - 1; k < 2 * q; ++k) exp[k] = exp[k % (q - 1)];
    return true;
  }
  int mul(int x, int y) const { return (x && y) ? exp[log[x] + log[y]] : 0; }
  int inv(int x) const { return exp[(q - 1 - log[x]) % (q - 1)]; }
};

// SUS dependency levels for the sweep that visits the columns
// in `order` (a permutation of 0..V-1; NULL = index order, A7): in the sweep
// column j reads the q's of the other columns of its checks (and, with
// chain = true -- the in-sweep Markov prior, A34 -- the posterior of source
// column j-1).  level(j) = 1 + max level of the columns visited before j that
// it depends on; columns of one level share no check, so running a level's
// columns concurrently, levels in order, reads exactly what the serial sweep
// reads.  Outputs: level_ptr [nlev+1], and the task tables in level order.
int build_levels(const HostGraph &g, const int *order, bool chain, std::vector<int> &level_ptr,
                 std::vector<LvlCol> &lcol, std::vector<LvlUnit> &lunit) {
  const int V = g.V, N = g.N;
  std::vector<int> lvl(V, 0), rowlvl(g.M, 0);
  int nlev = 0;
  for (int k = 0; k < V; ++k) {
    const int j = order ? order[k] : k;
    int L = (chain && j > 0 && j < N) ? lvl[j - 1] : 0;
    for (int x = g.col_ptr[j]; x < g.col_ptr[j + 1]; ++x) L = std::max(L, rowlvl[g.edge_check[g.col_edge[x]]]);
    L += 1;
    lvl[j] = L;
    for (int x = g.col_ptr[j]; x < g.col_ptr[j + 1]; ++x) rowlvl[g.edge_check[g.col_edge[x]]] = L;
    nlev = std::max(nlev, L);
  }
  level_ptr.assign(nlev + 1, 0);
  for (int j = 0; j < V; ++j) level_ptr[lvl[j]]++;  // lvl in 1..nlev -> slot lvl
  for (int L = 0; L < nlev; ++L) level_ptr[L + 1] += level_ptr[L];
  std::vector<int> cols(V), fill(level_ptr.begin(), level_ptr.end() - 1);
  for (int k = 0; k < V; ++k) {  // within a level: visiting order
    const int j = order ? order[k] : k;
    cols[fill[lvl[j] - 1]++] = j;
  }
  lcol.resize(V);
  lunit.clear();
  lunit.reserve((size_t)g.E + V);
  for (int k = 0; k < V; ++k) {
    const int j = cols[k];
    const int e0 = g.col_ptr[j], dv = g.col_ptr[j + 1] - e0;
    lcol[k] = LvlCol{j, e0, dv, (int)lunit.size()};
    if (dv == 0) lunit.push_back(LvlUnit{0, 0, 0, 0, j, e0, 0, 0});
    for (int s = 0; s < dv; ++s) {
      const int e = g.col_edge[e0 + s], i = g.edge_check[e];
      lunit.push_back(LvlUnit{g.row_ptr[i], g.row_ptr[i + 1] - g.row_ptr[i], e - g.row_ptr[i], i, j, e0, dv, s});
    }
  }
  return nlev;
}

}  // namespace gfq

using namespace gfq;

extern "C" const char *gfq_last_error(void) { return g_err.c_str(); }

extern "C" int gfq_version(void) { return 0x010100; }  // 1.1: params.compaction, p = 8, GFQ_NKERNELS 15

extern "C" int gfq_code_create(gfq_code **out, int p, unsigned poly, int N, int M,
                               long long nnzA, const int *A_row, const int *A_col,
                               const unsigned char *A_val, long long nnzB,
                               const int *B_row, const int *B_col,
                               const unsigned char *B_val) {
  if (!out) { set_error("gfq_code_create: out is NULL"); return GFQ_EINVAL; }
  if (p > 8) { set_error("gfq_code_create: p > 8 unsupported"); return GFQ_EUNSUPPORTED; }
  if (p < 1 || N < 0 || M < 1 || nnzA < 0 || nnzB < 0) {
    set_error("gfq_code_create: bad sizes");
    return GFQ_EINVAL;
  }
  if ((nnzA && (!A_row || !A_col || !A_val)) || (nnzB && (!B_row || !B_col || !B_val))) {
    set_error("gfq_code_create: NULL COO array");
    return GFQ_EINVAL;
  }
  if (poly >> p != 1u) { set_error("gfq_code_create: polynomial degree != p"); return GFQ_EINVAL; }
  GF gf;
  if (!gf.build(p, poly)) { set_error("gfq_code_create: polynomial is not primitive"); return GFQ_EINVAL; }
  const int q = 1 << p, V = N + M;
  const long long E = nnzA + nnzB;
  if (E > (1LL << 31) - 1) { set_error("gfq_code_create: too many edges"); return GFQ_EUNSUPPORTED; }

  struct Ent { int r, c, v; };
  std::vector<Ent> ent((size_t)E);
  for (long long k = 0; k < nnzA; ++k) {
    if (A_row[k] < 0 || A_row[k] >= M || A_col[k] < 0 || A_col[k] >= N) {
      set_error("gfq_code_create: A index out of range");
      return GFQ_EINVAL;
    }
    if (A_val[k] == 0 || A_val[k] >= q) { set_error("gfq_code_create: A value not in 1..q-1"); return GFQ_EINVAL; }
    ent[k] = {A_row[k], A_col[k], A_val[k]};
  }
  for (long long k = 0; k < nnzB; ++k) {
    if (B_row[k] < 0 || B_row[k] >= M || B_col[k] < 0 || B_col[k] >= M) {
      set_error("gfq_code_create: B index out of range");
      return GFQ_EINVAL;
    }
    if (B_val[k] == 0 || B_val[k] >= q) { set_error("gfq_code_create: B value not in 1..q-1"); return GFQ_EINVAL; }
    ent[nnzA + k] = {B_row[k], N + B_col[k], B_val[k]};
  }
  std::sort(ent.begin(), ent.end(), [](const Ent &a, const Ent &b) {
    return a.r != b.r ? a.r < b.r : a.c < b.c;
  });
  for (long long k = 1; k < E; ++k)
    if (ent[k].r == ent[k - 1].r && ent[k].c == ent[k - 1].c) {
      set_error("gfq_code_create: duplicate (row, col)");
      return GFQ_EINVAL;
    }

  // check-major edge ids (CSR order)
  std::vector<int> row_ptr(M + 1, 0), edge_var(E), edge_check(E), col_ptr(V + 1, 0), col_edge(E);
  std::vector<unsigned char> edge_coef(E);
  std::vector<unsigned long long> edge_perm(E);
  for (long long e = 0; e < E; ++e) {
    row_ptr[ent[e].r + 1]++;
    col_ptr[ent[e].c + 1]++;
    edge_var[e] = ent[e].c;
    edge_check[e] = ent[e].r;
    edge_coef[e] = (unsigned char)ent[e].v;
    const int hinv = gf.inv(ent[e].v);
    unsigned long long pk = 0;
    for (int b = 0; b < p; ++b) pk |= (unsigned long long)gf.mul(hinv, 1 << b) << (8 * b);
    edge_perm[e] = pk;
  }
  for (int i = 0; i < M; ++i) row_ptr[i + 1] += row_ptr[i];
  for (int j = 0; j < V; ++j) col_ptr[j + 1] += col_ptr[j];
  {
    std::vector<int> fill(col_ptr.begin(), col_ptr.end() - 1);
    for (long long e = 0; e < E; ++e) col_edge[fill[edge_var[e]]++] = (int)e;  // ascending check
  }
  std::vector<int> edge_canon(E);
  for (long long k = 0; k < E; ++k) edge_canon[col_edge[k]] = (int)k;
  int max_cdeg = 0, max_vdeg = 0;
  for (int i = 0; i < M; ++i) max_cdeg = std::max(max_cdeg, row_ptr[i + 1] - row_ptr[i]);
  for (int j = 0; j < V; ++j) max_vdeg = std::max(max_vdeg, col_ptr[j + 1] - col_ptr[j]);
  if (max_cdeg > kMaxDeg || max_vdeg > kMaxDeg) {
    set_error("gfq_code_create: a check or variable degree exceeds 8");
    return GFQ_EUNSUPPORTED;
  }

  // SUS dependency levels in index order (A7), without and with the in-sweep
  // prior chain (A34); build_levels below
  HostGraph hg{N, M, V, E, row_ptr, col_ptr, col_edge, edge_check};
  std::vector<int> level_ptr, level_ptr_gs;
  std::vector<LvlCol> lcol, lcol_gs;
  std::vector<LvlUnit> lunit, lunit_gs;
  const int nlev = build_levels(hg, nullptr, false, level_ptr, lcol, lunit);
  const int nlev_gs = build_levels(hg, nullptr, true, level_ptr_gs, lcol_gs, lunit_gs);

  // static task tables (see gfq_internal.cuh)
  std::vector<CheckDesc> cdesc(M);
  std::vector<VarDesc> vdesc(V);
  std::vector<SusDesc> sdesc(E);
  memset(cdesc.data(), 0, sizeof(CheckDesc) * M);
  memset(vdesc.data(), 0, sizeof(VarDesc) * V);
  memset(sdesc.data(), 0, sizeof(SusDesc) * E);
  for (int i = 0; i < M; ++i)
    for (int s = 0; s < row_ptr[i + 1] - row_ptr[i]; ++s) {
      cdesc[i].perm[s] = edge_perm[row_ptr[i] + s];
      cdesc[i].canon[s] = edge_canon[row_ptr[i] + s];
    }
  for (int j = 0; j < V; ++j)
    for (int s = 0; s < col_ptr[j + 1] - col_ptr[j]; ++s) vdesc[j].qdst[s] = col_edge[col_ptr[j] + s];
  for (long long cpos = 0; cpos < E; ++cpos) {
    const int e = col_edge[cpos], i = edge_check[e];
    int t = 0;
    for (int k = row_ptr[i]; k < row_ptr[i + 1]; ++k)
      if (k != e) sdesc[cpos].perm_o[t++] = edge_perm[k];
    sdesc[cpos].perm_e = edge_perm[e];
  }
  const size_t U = lunit.size();

  // Encoder support (gfq_simulate, Eq. 1): an order that solves B t = y row by
  // row -- each row, when reached, has exactly one unsolved column of B
  // ("peeling").  Exists for the MN construction (B triangular up to a
  // permutation, reading A23); otherwise simulation is unsupported.
  std::vector<int> peel;  // pairs (row r, noise column k solved by row r)
  {
    std::vector<int> unknown(M, 0);
    std::vector<std::vector<int>> rows_of(M);
    for (int i = 0; i < M; ++i)
      for (int e = row_ptr[i]; e < row_ptr[i + 1]; ++e)
        if (edge_var[e] >= N) { unknown[i]++; rows_of[edge_var[e] - N].push_back(i); }
    std::vector<char> solved(M, 0), used(M, 0);
    std::vector<int> stack;
    for (int i = M - 1; i >= 0; --i)
      if (unknown[i] == 1) stack.push_back(i);
    while (!stack.empty()) {
      const int i = stack.back();
      stack.pop_back();
      if (used[i] || unknown[i] != 1) continue;
      used[i] = 1;
      int k = -1;
      for (int e = row_ptr[i]; e < row_ptr[i + 1]; ++e)
        if (edge_var[e] >= N && !solved[edge_var[e] - N]) k = edge_var[e] - N;
      solved[k] = 1;
      peel.push_back(i);
      peel.push_back(k);
      for (int i2 : rows_of[k])
        if (--unknown[i2] == 1 && !used[i2]) stack.push_back(i2);
    }
    if ((int)peel.size() != 2 * M) peel.clear();
  }
  std::vector<unsigned char> inv(q, 0);
  for (int x = 1; x < q; ++x) inv[x] = (unsigned char)gf.inv(x);

  std::vector<unsigned char> mul((size_t)q * q);
  for (int x = 0; x < q; ++x)
    for (int y = 0; y < q; ++y) mul[x * q + y] = (unsigned char)gf.mul(x, y);
  std::vector<unsigned short> rowtab((size_t)q * q);
  for (int x = 0; x < q; ++x)
    for (int y = 0; y < q; ++y) rowtab[x * q + y] = (unsigned short)(gf.mul(x, y) << 7);

  // one device blob
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  size_t off = 0;
  const size_t o_row = off; off += al(sizeof(int) * (M + 1));
  const size_t o_var = off; off += al(sizeof(int) * E);
  const size_t o_chk = off; off += al(sizeof(int) * E);
  const size_t o_perm = off; off += al(sizeof(unsigned long long) * E);
  const size_t o_coef = off; off += al(E);
  const size_t o_col = off; off += al(sizeof(int) * (V + 1));
  const size_t o_cedge = off; off += al(sizeof(int) * E);
  const size_t o_canon = off; off += al(sizeof(int) * E);
  const size_t o_lptr = off; off += al(sizeof(int) * (nlev + 1));
  const size_t o_lcol = off; off += al(sizeof(int) * V);
  const size_t o_mul = off; off += al((size_t)q * q);
  const size_t o_rowtab = off; off += al((size_t)q * q * 2);
  const size_t o_cdesc = off; off += al(sizeof(CheckDesc) * M);
  const size_t o_vdesc = off; off += al(sizeof(VarDesc) * V);
  const size_t o_sdesc = off; off += al(sizeof(SusDesc) * E);
  const size_t o_lvlcol = off; off += al(sizeof(LvlCol) * V);
  const size_t o_lunit = off; off += al(sizeof(LvlUnit) * U);
  const size_t o_lvlcol_gs = off; off += al(sizeof(LvlCol) * V);
  const size_t o_lunit_gs = off; off += al(sizeof(LvlUnit) * U);
  const size_t o_peel = off; off += al(sizeof(int) * peel.size());
  const size_t o_inv = off; off += al(q);
  std::vector<unsigned char> host(off, 0);
  auto put = [&](size_t o, const void *src, size_t n) { if (n) memcpy(host.data() + o, src, n); };
  put(o_row, row_ptr.data(), sizeof(int) * (M + 1));
  put(o_var, edge_var.data(), sizeof(int) * E);
  put(o_chk, edge_check.data(), sizeof(int) * E);
  put(o_perm, edge_perm.data(), sizeof(unsigned long long) * E);
  put(o_coef, edge_coef.data(), E);
  put(o_col, col_ptr.data(), sizeof(int) * (V + 1));
  put(o_cedge, col_edge.data(), sizeof(int) * E);
  put(o_canon, edge_canon.data(), sizeof(int) * E);
  {
    std::vector<int> level_cols(V);
    for (int k = 0; k < V; ++k) level_cols[k] = lcol[k].j;
    put(o_lptr, level_ptr.data(), sizeof(int) * (nlev + 1));
    put(o_lcol, level_cols.data(), sizeof(int) * V);
  }
  put(o_mul, mul.data(), (size_t)q * q);
  put(o_rowtab, rowtab.data(), (size_t)q * q * 2);
  put(o_cdesc, cdesc.data(), sizeof(CheckDesc) * M);
  put(o_vdesc, vdesc.data(), sizeof(VarDesc) * V);
  put(o_sdesc, sdesc.data(), sizeof(SusDesc) * E);
  put(o_lvlcol, lcol.data(), sizeof(LvlCol) * V);
  put(o_lunit, lunit.data(), sizeof(LvlUnit) * U);
  put(o_lvlcol_gs, lcol_gs.data(), sizeof(LvlCol) * V);
  put(o_lunit_gs, lunit_gs.data(), sizeof(LvlUnit) * U);
  put(o_peel, peel.data(), sizeof(int) * peel.size());
  put(o_inv, inv.data(), q);

  int dev = 0;
  cudaError_t ce = cudaGetDevice(&dev);
  if (ce != cudaSuccess) return cuda_fail(ce, "gfq_code_create: cudaGetDevice");
  void *blob = nullptr;
  ce = cudaMalloc(&blob, off);
  if (ce != cudaSuccess) { cudaGetLastError(); set_error("gfq_code_create: cudaMalloc failed"); return GFQ_ENOMEM; }
  ce = cudaMemcpy(blob, host.data(), off, cudaMemcpyHostToDevice);
  if (ce != cudaSuccess) { cudaFree(blob); return cuda_fail(ce, "gfq_code_create: upload"); }

  gfq_code *c = new (std::nothrow) gfq_code();
  if (!c) { cudaFree(blob); set_error("gfq_code_create: out of host memory"); return GFQ_ENOMEM; }
  c->p = p; c->q = q; c->N = N; c->M = M; c->V = V; c->poly = poly; c->E = E;
  c->max_cdeg = max_cdeg; c->max_vdeg = max_vdeg; c->n_levels = nlev; c->device = dev;
  c->level_ptr_h = level_ptr;
  c->hg = std::move(hg);
  c->n_units = (long long)U;
  c->n_levels_gs = nlev_gs;
  c->level_ptr_gs_h = level_ptr_gs;
  c->dev_blob = blob;
  unsigned char *b = (unsigned char *)blob;
  c->d.p = p; c->d.q = q; c->d.N = N; c->d.M = M; c->d.V = V; c->d.E = E;
  c->d.max_cdeg = max_cdeg; c->d.max_vdeg = max_vdeg;
  c->d.row_ptr = (const int *)(b + o_row);
  c->d.edge_var = (const int *)(b + o_var);
  c->d.edge_check = (const int *)(b + o_chk);
  c->d.edge_perm = (const unsigned long long *)(b + o_perm);
  c->d.edge_coef = b + o_coef;
  c->d.col_ptr = (const int *)(b + o_col);
  c->d.col_edge = (const int *)(b + o_cedge);
  c->d.edge_canon = (const int *)(b + o_canon);
  c->d.level_ptr = (const int *)(b + o_lptr);
  c->d.level_cols = (const int *)(b + o_lcol);
  c->d.mul = b + o_mul;
  c->d.rowtab = (const unsigned short *)(b + o_rowtab);
  c->d.check_desc = (const CheckDesc *)(b + o_cdesc);
  c->d.var_desc = (const VarDesc *)(b + o_vdesc);
  c->d.sus_desc = (const SusDesc *)(b + o_sdesc);
  c->d.lvl_col = (const LvlCol *)(b + o_lvlcol);
  c->d.lvl_unit = (const LvlUnit *)(b + o_lunit);
  c->lvl_col_gs = (const LvlCol *)(b + o_lvlcol_gs);
  c->lvl_unit_gs = (const LvlUnit *)(b + o_lunit_gs);
  c->d.peel = peel.empty() ? nullptr : (const int *)(b + o_peel);
  c->d.inv = b + o_inv;
  *out = c;
  return GFQ_OK;
}

extern "C" void gfq_code_destroy(gfq_code *c) {
  if (!c) return;
  if (c->dev_blob) cudaFree(c->dev_blob);
  delete c;
}

extern "C" int gfq_code_info(const gfq_code *c, long long *n_edges, int *max_check_deg,
                             int *max_var_deg, int *sus_levels) {
  if (!c) { set_error("gfq_code_info: code is NULL"); return GFQ_EINVAL; }
  if (n_edges) *n_edges = c->E;
  if (max_check_deg) *max_check_deg = c->max_cdeg;
  if (max_var_deg) *max_var_deg = c->max_vdeg;
  if (sus_levels) *sus_levels = c->n_levels;
  return GFQ_OK;
}

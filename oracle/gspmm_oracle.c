/*
 * gspmm_oracle.c -- CPU restatement of the reference aggregation path.
 *
 * TEST INFRASTRUCTURE ONLY (see gspmm_oracle.h).  Compiled with
 * -ffp-contract=off so every fp32 multiply and add rounds separately, as the
 * reference does when built for baseline x86-64 (no FMA in the ISA).
 * Citations are to /root/reference/proj.
 */
#include "gspmm_oracle.h"

#include <math.h>
#include <omp.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ rng */

/* rng.hpp:26-31 */
uint64_t or_splitmix64_at(uint64_t seed, uint64_t counter) {
  uint64_t z = seed + (counter + 1) * 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* rng.hpp:34-36: 53-bit uniform double in [0,1) */
double or_u01_at(uint64_t seed, uint64_t counter) {
  return (double)(or_splitmix64_at(seed, counter) >> 11) * 0x1.0p-53;
}

/* rng.hpp:39-43: 24-bit uniform float in [-1,1) */
float or_unit_float_at(uint64_t seed, uint64_t counter) {
  const float u = (float)(or_splitmix64_at(seed, counter) >> 40) * 0x1.0p-24f;
  return 2.0f * u - 1.0f;
}

/* Builder-defined N(0,1) (the reference has no Gaussian):
 * Box-Muller on u01 draws 2i and 2i+1, computed in double, rounded once. */
float or_normal_at(uint64_t seed, uint64_t i) {
  const double u1 = or_u01_at(seed, 2 * i);
  const double u2 = or_u01_at(seed, 2 * i + 1);
  const double r = sqrt(-2.0 * log(1.0 - u1));
  return (float)(r * cos(6.283185307179586476925286766559 * u2));
}

typedef struct {
  uint64_t seed, counter;
} or_rng; /* CounterRng, rng.hpp:46-62 */

static double rng_next_u01(or_rng* r) { return or_u01_at(r->seed, r->counter++); }

/* ----------------------------------------------------------- generators */

/* Growable edge buffer. */
typedef struct {
  uint32_t *src, *dst;
  int64_t n, cap;
} edge_buf;

static void eb_push(edge_buf* b, uint32_t s, uint32_t d) {
  if (b->n == b->cap) {
    b->cap = b->cap ? b->cap * 2 : 1024;
    b->src = (uint32_t*)realloc(b->src, (size_t)b->cap * sizeof(uint32_t));
    b->dst = (uint32_t*)realloc(b->dst, (size_t)b->cap * sizeof(uint32_t));
  }
  b->src[b->n] = s;
  b->dst[b->n] = d;
  b->n++;
}

/* GeometricSkipper, generate.cpp:34-71: table of (1-p)^k searched with
 * exact comparisons. */
typedef struct {
  double* pow_q;
  size_t size;
} geo_skip;

static void geo_init(geo_skip* g, double p) {
  const size_t kMaxTable = 4096;
  const double q = 1.0 - p;
  g->pow_q = (double*)malloc((kMaxTable + 2) * sizeof(double));
  g->size = 0;
  g->pow_q[g->size++] = 1.0;
  double x = q;
  while (x > 0x1.0p-64 && g->size < kMaxTable) {
    g->pow_q[g->size++] = x;
    x *= q;
  }
  g->pow_q[g->size++] = x;
}

static uint64_t geo_gap(const geo_skip* g, double u) {
  double t = 1.0 - u;
  const size_t last = g->size - 1;
  uint64_t base = 0;
  while (t <= g->pow_q[last]) {
    base += last;
    t /= g->pow_q[last];
  }
  size_t lo = 1, hi = last;
  while (lo < hi) {
    const size_t mid = (lo + hi) / 2;
    if (g->pow_q[mid] < t)
      hi = mid;
    else
      lo = mid + 1;
  }
  return base + lo - 1;
}

/* sample_rect, generate.cpp:75-88; emits cells of a row-major rectangle.
 * The emit callback receives the cell index. */
typedef void (*emit_fn)(void* ctx, uint64_t cell);

static void sample_rect(uint64_t cells, double p, or_rng* rng, emit_fn emit,
                        void* ctx) {
  if (p <= 0.0 || cells == 0) return;
  if (p >= 1.0) {
    for (uint64_t c = 0; c < cells; ++c) emit(ctx, c);
    return;
  }
  geo_skip skip;
  geo_init(&skip, p);
  uint64_t pos = geo_gap(&skip, rng_next_u01(rng));
  while (pos < cells) {
    emit(ctx, pos);
    pos += 1 + geo_gap(&skip, rng_next_u01(rng));
  }
  free(skip.pow_q);
}

typedef struct {
  edge_buf* b;
  uint32_t row0, col0, cols;
} rect_ctx;

static void emit_rect(void* vctx, uint64_t cell) {
  rect_ctx* c = (rect_ctx*)vctx;
  const uint32_t i = c->row0 + (uint32_t)(cell / c->cols);
  const uint32_t j = c->col0 + (uint32_t)(cell % c->cols);
  if (i != j) eb_push(c->b, i, j); /* self-loops dropped */
}

/* gen_erdos_renyi, generate.cpp:90-108 */
int64_t or_gen_er(uint32_t n, uint64_t num_edges, double prob, uint64_t seed,
                  uint32_t** src, uint32_t** dst) {
  double p = prob;
  if (p < 0.0) {
    const double pairs = (double)n * ((double)n - 1.0);
    p = pairs > 0.0 ? (double)num_edges / pairs : 0.0;
  }
  edge_buf b = {0};
  or_rng rng = {seed, 0};
  rect_ctx ctx = {&b, 0, 0, n};
  sample_rect((uint64_t)n * n, p, &rng, emit_rect, &ctx);
  *src = b.src;
  *dst = b.dst;
  return b.n;
}

/* gen_sbm, generate.cpp:110-138 */
int64_t or_gen_sbm(uint32_t n, int blocks, double p_in, double p_out,
                   uint64_t seed, uint32_t** src, uint32_t** dst) {
  const int k = blocks;
  uint32_t* start = (uint32_t*)calloc((size_t)k + 1, sizeof(uint32_t));
  for (int b = 0; b < k; ++b) {
    const uint32_t size = n / (uint32_t)k + ((uint32_t)b < n % (uint32_t)k ? 1 : 0);
    start[b + 1] = start[b] + size;
  }
  edge_buf eb = {0};
  or_rng rng = {seed, 0};
  for (int bi = 0; bi < k; ++bi) {
    for (int bj = 0; bj < k; ++bj) {
      const double p = bi == bj ? p_in : p_out;
      const uint32_t rows = start[bi + 1] - start[bi];
      const uint32_t cols = start[bj + 1] - start[bj];
      rect_ctx ctx = {&eb, start[bi], start[bj], cols};
      sample_rect((uint64_t)rows * cols, p, &rng, emit_rect, &ctx);
    }
  }
  free(start);
  *src = eb.src;
  *dst = eb.dst;
  return eb.n;
}

/* gen_rmat, generate.cpp:140-172. Returns -1 (ConfigError) when an edge
 * cannot be placed within 10000 tries. */
int64_t or_gen_rmat(uint32_t n, uint64_t num_edges, double a, double b,
                    double c, double d, uint64_t seed, uint32_t** src,
                    uint32_t** dst) {
  (void)d;
  int levels = 0;
  while (((uint64_t)1 << levels) < (uint64_t)n) ++levels;
  const double t_ab = a + b;
  const double t_abc = t_ab + c;
  uint32_t* s = (uint32_t*)malloc((num_edges ? num_edges : 1) * sizeof(uint32_t));
  uint32_t* t = (uint32_t*)malloc((num_edges ? num_edges : 1) * sizeof(uint32_t));
  or_rng rng = {seed, 0};
  for (uint64_t e = 0; e < num_edges; ++e) {
    uint32_t u = 0, v = 0;
    for (int tries = 0;; ++tries) {
      if (tries > 10000) {
        free(s);
        free(t);
        return -1;
      }
      u = 0;
      v = 0;
      for (int l = 0; l < levels; ++l) {
        const double r = rng_next_u01(&rng);
        const int quad = r < a ? 0 : r < t_ab ? 1 : r < t_abc ? 2 : 3;
        u = (u << 1) | (uint32_t)(quad >> 1);
        v = (v << 1) | (uint32_t)(quad & 1);
      }
      if (u < n && v < n) break;
    }
    s[e] = u;
    t[e] = v;
  }
  *src = s;
  *dst = t;
  return (int64_t)num_edges;
}

void or_free(void* p) { free(p); }

/* Builder-defined power-law in-degree generator for cfg5 (the reference has
 * none): in-degree of node v from the inverse CDF of P(d) ~ d^-2
 * on [d_min, d_max] at u01(seed, v); edges in edge-id order grouped by
 * destination, source of edge e = (splitmix64(seed ^ 0x5851f42d4c957f2d, e)
 * * n) >> 64.  Restated independently of the product's synth.cpp. */
int64_t or_gen_powerlaw(uint32_t n, uint32_t d_min, uint32_t d_max, uint64_t seed,
                        uint32_t** src, uint32_t** dst) {
  const double a = 1.0 / d_min, b = 1.0 / d_min - 1.0 / d_max;
  uint64_t m = 0;
  uint32_t* deg = (uint32_t*)malloc((size_t)(n ? n : 1) * sizeof(uint32_t));
  for (uint32_t v = 0; v < n; ++v) {
    double d = floor(1.0 / (a - or_u01_at(seed, v) * b));
    if (d < d_min) d = d_min;
    if (d > d_max) d = d_max;
    deg[v] = (uint32_t)d;
    m += deg[v];
  }
  uint32_t* s = (uint32_t*)malloc((size_t)(m ? m : 1) * sizeof(uint32_t));
  uint32_t* t = (uint32_t*)malloc((size_t)(m ? m : 1) * sizeof(uint32_t));
  const uint64_t seed2 = seed ^ 0x5851f42d4c957f2dULL;
  uint64_t e = 0;
  for (uint32_t v = 0; v < n; ++v)
    for (uint32_t k = 0; k < deg[v]; ++k, ++e) {
      s[e] = (uint32_t)(((unsigned __int128)or_splitmix64_at(seed2, e) * n) >> 64);
      t[e] = v;
    }
  free(deg);
  *src = s;
  *dst = t;
  return (int64_t)m;
}

/* random_features, generate.cpp:256-266 */
void or_random_features(int64_t rows, int64_t dim, uint64_t seed, float* out) {
  const int64_t total = rows * dim;
  for (int64_t i = 0; i < total; ++i) out[i] = or_unit_float_at(seed, (uint64_t)i);
}

void or_normal_features(int64_t count, uint64_t seed, float* out) {
  for (int64_t i = 0; i < count; ++i) out[i] = or_normal_at(seed, (uint64_t)i);
}

/* elements [offset, offset+count) of the stream (chunked generation) */
void or_normal_features_at(int64_t offset, int64_t count, uint64_t seed, float* out) {
  for (int64_t i = 0; i < count; ++i) out[i] = or_normal_at(seed, (uint64_t)(offset + i));
}

/* ----------------------------------------------------------- graph core */

/* from_keys, csr.cpp:31-71: stable counting sort by column, then by row. */
static void from_keys(uint32_t num_rows, uint32_t num_cols, int64_t m,
                      const uint32_t* row_of, const uint32_t* col_of,
                      const uint32_t* eid_of, uint32_t* indptr,
                      uint32_t* indices, uint32_t* eids) {
  size_t* by_col = (size_t*)malloc((size_t)(m ? m : 1) * sizeof(size_t));
  size_t* cnt = (size_t*)calloc((size_t)num_cols + 1, sizeof(size_t));
  for (int64_t i = 0; i < m; ++i) cnt[col_of[i]]++;
  size_t run = 0;
  for (size_t c = 0; c <= num_cols; ++c) {
    const size_t k = cnt[c];
    cnt[c] = run;
    run += k;
  }
  for (int64_t i = 0; i < m; ++i) by_col[cnt[col_of[i]]++] = (size_t)i;
  free(cnt);

  size_t* row_start = (size_t*)calloc((size_t)num_rows + 1, sizeof(size_t));
  memset(indptr, 0, ((size_t)num_rows + 1) * sizeof(uint32_t));
  for (int64_t i = 0; i < m; ++i) indptr[row_of[i] + 1]++;
  for (size_t r = 0; r < num_rows; ++r) {
    indptr[r + 1] += indptr[r];
    row_start[r] = indptr[r];
  }
  for (int64_t k = 0; k < m; ++k) {
    const size_t i = by_col[k];
    const size_t pos = row_start[row_of[i]]++;
    indices[pos] = col_of[i];
    eids[pos] = eid_of[i];
  }
  free(row_start);
  free(by_col);
}

/* build_csr, csr.cpp:75-93 */
int or_build_csr(uint32_t n, int64_t m, const uint32_t* src,
                 const uint32_t* dst, int orientation, uint32_t* indptr,
                 uint32_t* indices, uint32_t* eids) {
  uint32_t* row_of = (uint32_t*)malloc((size_t)(m ? m : 1) * sizeof(uint32_t));
  uint32_t* col_of = (uint32_t*)malloc((size_t)(m ? m : 1) * sizeof(uint32_t));
  uint32_t* eid_of = (uint32_t*)malloc((size_t)(m ? m : 1) * sizeof(uint32_t));
  for (int64_t i = 0; i < m; ++i) {
    if (src[i] >= n || dst[i] >= n) {
      free(row_of);
      free(col_of);
      free(eid_of);
      return OR_STRUCTURE;
    }
    row_of[i] = orientation == OR_DST_MAJOR ? dst[i] : src[i];
    col_of[i] = orientation == OR_DST_MAJOR ? src[i] : dst[i];
    eid_of[i] = (uint32_t)i;
  }
  from_keys(n, n, m, row_of, col_of, eid_of, indptr, indices, eids);
  free(row_of);
  free(col_of);
  free(eid_of);
  return OR_OK;
}

/* transpose, csr.cpp:95-109 */
int or_transpose(uint32_t num_rows, uint32_t num_cols, const uint32_t* indptr,
                 const uint32_t* indices, const uint32_t* eids,
                 uint32_t* t_indptr, uint32_t* t_indices, uint32_t* t_eids) {
  const int64_t m = indptr[num_rows];
  uint32_t* row_of = (uint32_t*)malloc((size_t)(m ? m : 1) * sizeof(uint32_t));
  uint32_t* col_of = (uint32_t*)malloc((size_t)(m ? m : 1) * sizeof(uint32_t));
  uint32_t* eid_of = (uint32_t*)malloc((size_t)(m ? m : 1) * sizeof(uint32_t));
  int64_t k = 0;
  for (uint32_t r = 0; r < num_rows; ++r) {
    for (uint32_t j = indptr[r]; j < indptr[r + 1]; ++j, ++k) {
      row_of[k] = indices[j];
      col_of[k] = r;
      eid_of[k] = eids[j];
    }
  }
  from_keys(num_cols, num_rows, m, row_of, col_of, eid_of, t_indptr, t_indices,
            t_eids);
  free(row_of);
  free(col_of);
  free(eid_of);
  return OR_OK;
}

/* validate, csr.cpp:111-156 (codes instead of messages, same order) */
int or_validate(uint32_t num_rows, uint32_t num_cols, int64_t indptr_len,
                const uint32_t* indptr, int64_t m_len, const uint32_t* indices,
                const uint32_t* eids) {
  if (indptr_len != (int64_t)num_rows + 1) return 1;
  if (indptr[0] != 0) return 2;
  for (uint32_t r = 0; r < num_rows; ++r)
    if (indptr[r] > indptr[r + 1]) return 3;
  const int64_t m = indptr[num_rows];
  if (m_len != m) return 4;
  for (int64_t j = 0; j < m; ++j)
    if (indices[j] >= num_cols) return 5;
  unsigned char* seen = (unsigned char*)calloc((size_t)(m ? m : 1), 1);
  for (int64_t j = 0; j < m; ++j) {
    if ((int64_t)eids[j] >= m || seen[eids[j]]) {
      free(seen);
      return 6;
    }
    seen[eids[j]] = 1;
  }
  free(seen);
  for (uint32_t r = 0; r < num_rows; ++r) {
    for (uint32_t j = indptr[r]; j + 1 < indptr[r + 1]; ++j) {
      const int ordered = indices[j] < indices[j + 1] ||
                          (indices[j] == indices[j + 1] && eids[j] < eids[j + 1]);
      if (!ordered) return 7;
    }
  }
  return 0;
}

/* ----------------------------------------------------------- semantics */

/* ops.cpp:48-57 */
static float reduce_identity(int op) {
  switch (op) {
    case OR_MAX: return -INFINITY;
    case OR_MIN: return INFINITY;
    case OR_PROD: return 1.0f;
    default: return 0.0f;
  }
}

/* kernels.cpp:38-52 */
static float reduce_combine(int op, float a, float m) {
  switch (op) {
    case OR_SUM: return a + m;
    case OR_MAX: return a < m ? m : a;
    case OR_MIN: return m < a ? m : a;
    case OR_PROD: return a * m;
    default: return m; /* CopyLast */
  }
}

/* kernels.cpp:54-69 */
static float binop_apply(int op, float l, float r) {
  switch (op) {
    case OR_ADD: return l + r;
    case OR_SUB: return l - r;
    case OR_MUL: return l * r;
    case OR_DIV: return l / r;
    default: return l; /* CopyLhs */
  }
}

/* validate_config, br_config.cpp:83-94 */
static int validate_config(int lhs, int rhs, int binop, int reduce, int out) {
  if (lhs < 0 || lhs > OR_NONE || rhs < 0 || rhs > OR_NONE || out < 0 ||
      out > OR_NONE || binop < 0 || binop > OR_COPY || reduce < 0 ||
      reduce > OR_LAST)
    return OR_CONFIG;
  if (lhs == OR_NONE) return OR_CONFIG;
  if (out == OR_NONE) return OR_CONFIG;
  if ((rhs == OR_NONE) != (binop == OR_COPY)) return OR_CONFIG;
  if (rhs != OR_NONE && rhs == lhs) return OR_CONFIG;
  if (out == OR_E && reduce != OR_LAST) return OR_CONFIG;
  return OR_OK;
}

static const or_feat* pick(int o, const or_feat* u, const or_feat* v,
                           const or_feat* e) {
  return o == OR_U ? u : o == OR_V ? v : o == OR_E ? e : NULL;
}

typedef struct {
  int64_t nu, nv, ne;
} counts_t;

static int64_t count_of(const counts_t* c, int ent) {
  return ent == OR_U ? c->nu : ent == OR_V ? c->nv : c->ne;
}

/* Operand binding and width rules: bind_operand kernels.cpp:361-377,
 * binary_reduce :426-453. Fills widths and strides. */
typedef struct {
  const float* lbase;
  const float* rbase;
  int64_t ldim, rdim, w, gather_dim, ls, rs;
  int64_t out_rows;
} bound_t;

static int bind_all(int orientation, uint32_t num_rows, uint32_t num_cols,
                    int64_t m, int lhs, int rhs, int binop, int reduce, int out,
                    const or_feat* u, const or_feat* v, const or_feat* e,
                    bound_t* b) {
  int st = validate_config(lhs, rhs, binop, reduce, out);
  if (st) return st;
  /* required_orientation(RowParallelSpmm, out), kernels.cpp:400-411 */
  const int need = out == OR_U ? OR_SRC_MAJOR : OR_DST_MAJOR;
  if (orientation != need) return OR_SHAPE;
  counts_t c;
  c.nu = orientation == OR_SRC_MAJOR ? num_rows : num_cols;
  c.nv = orientation == OR_SRC_MAJOR ? num_cols : num_rows;
  c.ne = m;
  const or_feat* lf = pick(lhs, u, v, e);
  if (!lf || !lf->data && lf->rows * lf->dim > 0) return OR_SHAPE;
  if (lf->rows != count_of(&c, lhs)) return OR_SHAPE;
  b->lbase = lf->data;
  b->ldim = lf->dim;
  b->rbase = NULL;
  b->rdim = 0;
  if (rhs != OR_NONE) {
    const or_feat* rf = pick(rhs, u, v, e);
    if (!rf || !rf->data && rf->rows * rf->dim > 0) return OR_SHAPE;
    if (rf->rows != count_of(&c, rhs)) return OR_SHAPE;
    b->rbase = rf->data;
    b->rdim = rf->dim;
    /* dims_broadcastable, ops.cpp:59-61 */
    if (!(b->ldim == b->rdim || b->ldim == 1 || b->rdim == 1)) return OR_SHAPE;
  }
  /* binary_out_dim, ops.cpp:63-67 */
  const int64_t dr = rhs == OR_NONE ? b->ldim : b->rdim;
  b->w = binop == OR_DOT ? 1 : binop == OR_COPY ? b->ldim
                                 : (b->ldim > dr ? b->ldim : dr);
  b->gather_dim = rhs == OR_NONE ? b->ldim : (b->ldim > b->rdim ? b->ldim : b->rdim);
  b->ls = (b->ldim == 1 && b->gather_dim > 1) ? 0 : 1;
  b->rs = rhs != OR_NONE ? ((b->rdim == 1 && b->gather_dim > 1) ? 0 : 1) : 0;
  b->out_rows = count_of(&c, out);
  return OR_OK;
}

int or_out_shape(int orientation, uint32_t num_rows, uint32_t num_cols,
                 int64_t m, int lhs, int rhs, int binop, int reduce, int out,
                 const or_feat* u, const or_feat* v, const or_feat* e,
                 int64_t* out_rows, int64_t* out_dim) {
  bound_t b;
  const int st = bind_all(orientation, num_rows, num_cols, m, lhs, rhs, binop,
                          reduce, out, u, v, e, &b);
  if (st) return st;
  *out_rows = b.out_rows;
  *out_dim = b.w;
  return OR_OK;
}

/* binary_reduce(RowParallelSpmm) = run_rowmajor<B,R,false>,
 * kernels.cpp:162-195 + 413-501: per owner row r, canonical order j, each
 * output element a sequential fp32 left fold from the reduce identity. */
int or_binary_reduce(int orientation, uint32_t num_rows, uint32_t num_cols,
                     const uint32_t* indptr, const uint32_t* indices,
                     const uint32_t* eids, int lhs, int rhs, int binop,
                     int reduce, int out, const or_feat* u, const or_feat* v,
                     const or_feat* e, float* out_data) {
  const int64_t m = indptr[num_rows];
  bound_t b;
  const int st = bind_all(orientation, num_rows, num_cols, m, lhs, rhs, binop,
                          reduce, out, u, v, e, &b);
  if (st) return st;
  const int64_t w = b.w;
  const float ident = reduce_identity(reduce);
  for (int64_t i = 0; i < b.out_rows * w; ++i) out_data[i] = ident;

  for (uint32_t r = 0; r < num_rows; ++r) {
    for (uint32_t j = indptr[r]; j < indptr[r + 1]; ++j) {
      const uint32_t other = indices[j];
      const uint32_t eid = eids[j];
      /* split_endpoints, kernels.cpp:138-147 */
      const uint32_t uu = orientation == OR_DST_MAJOR ? other : r;
      const uint32_t vv = orientation == OR_DST_MAJOR ? r : other;
      const int64_t lrow = lhs == OR_U ? uu : lhs == OR_V ? vv : eid;
      const float* lp = b.lbase + lrow * b.ldim;
      const float* rp = NULL;
      if (rhs != OR_NONE) {
        const int64_t rrow = rhs == OR_U ? uu : rhs == OR_V ? vv : eid;
        rp = b.rbase + rrow * b.rdim;
      }
      float* op = out == OR_E ? out_data + (int64_t)eid * w : out_data + (int64_t)r * w;
      if (binop == OR_DOT) {
        /* apply_dot, kernels.cpp:91-97 */
        float acc = 0.0f;
        for (int64_t i = 0; i < b.gather_dim; ++i)
          acc += lp[i * b.ls] * rp[i * b.rs];
        op[0] = reduce_combine(reduce, op[0], acc);
      } else {
        /* apply_span, kernels.cpp:74-89 */
        for (int64_t i = 0; i < w; ++i) {
          const float l = lp[i * b.ls];
          const float rv = rp ? rp[i * b.rs] : 0.0f;
          op[i] = reduce_combine(reduce, op[i], binop_apply(binop, l, rv));
        }
      }
    }
  }
  /* zero-degree fixup, kernels.cpp:490-499 */
  if (out != OR_E && (reduce == OR_MAX || reduce == OR_MIN)) {
    for (uint32_t r = 0; r < num_rows; ++r)
      if (indptr[r] == indptr[r + 1])
        memset(out_data + (int64_t)r * w, 0, (size_t)w * sizeof(float));
  }
  return OR_OK;
}

/* oracle_aggregate, oracle.cpp:72-170 */
int or_oracle_aggregate(uint32_t num_nodes, int64_t m, const uint32_t* src,
                        const uint32_t* dst, int lhs, int rhs, int binop,
                        int reduce, int out, const or_feat* u,
                        const or_feat* v, const or_feat* e, float* out_data) {
  int st = validate_config(lhs, rhs, binop, reduce, out);
  if (st) return st;
  if (m > 1000000) return OR_SHAPE;
  const int64_t n = num_nodes;
  const or_feat* lf = pick(lhs, u, v, e);
  const or_feat* rf = pick(rhs, u, v, e);
  if (!lf || (rhs != OR_NONE && !rf)) return OR_SHAPE;
  if (lf->rows != (lhs == OR_E ? m : n) ||
      (rf && rf->rows != (rhs == OR_E ? m : n)))
    return OR_SHAPE;
  const int64_t dl = lf->dim;
  const int64_t dr = rf ? rf->dim : dl;
  if (rf && !(dl == dr || dl == 1 || dr == 1)) return OR_SHAPE;
  const int64_t w = binop == OR_DOT ? 1 : binop == OR_COPY ? dl : (dl > dr ? dl : dr);
  const int64_t out_rows = out == OR_E ? m : n;
  const float ident = reduce_identity(reduce);
  for (int64_t i = 0; i < out_rows * w; ++i) out_data[i] = ident;

  double* sum_acc = NULL;
  if (reduce == OR_SUM && out != OR_E)
    sum_acc = (double*)calloc((size_t)(out_rows * w ? out_rows * w : 1), sizeof(double));
  unsigned char* touched =
      (unsigned char*)calloc((size_t)(out_rows ? out_rows : 1), 1);
  uint32_t* win_other = (uint32_t*)calloc((size_t)(out_rows ? out_rows : 1), sizeof(uint32_t));
  uint32_t* win_eid = (uint32_t*)calloc((size_t)(out_rows ? out_rows : 1), sizeof(uint32_t));
  float* msg = (float*)malloc((size_t)(w ? w : 1) * sizeof(float));

  for (int64_t id = 0; id < m; ++id) {
    const uint32_t uu = src[id], vv = dst[id];
    const int64_t lrow = lhs == OR_U ? uu : lhs == OR_V ? vv : id;
    const float* l = lf->data + lrow * dl;
    const float* r = NULL;
    if (rf) {
      const int64_t rrow = rhs == OR_U ? uu : rhs == OR_V ? vv : id;
      r = rf->data + rrow * dr;
    }
    /* message(), oracle.cpp:43-68 */
    if (binop == OR_COPY) {
      for (int64_t i = 0; i < w; ++i) msg[i] = l[i];
    } else if (binop == OR_DOT) {
      float acc = 0.0f;
      const int64_t d = dl > dr ? dl : dr;
      for (int64_t i = 0; i < d; ++i)
        acc += l[dl == 1 ? 0 : i] * r[dr == 1 ? 0 : i];
      msg[0] = acc;
    } else {
      for (int64_t i = 0; i < w; ++i)
        msg[i] = binop_apply(binop, l[dl == 1 ? 0 : i], r[dr == 1 ? 0 : i]);
    }
    if (out == OR_E) {
      memcpy(out_data + id * w, msg, (size_t)w * sizeof(float));
      continue;
    }
    const int64_t o = out == OR_U ? uu : vv;
    const uint32_t other = out == OR_V ? uu : vv;
    float* orow = out_data + o * w;
    switch (reduce) {
      case OR_SUM:
        for (int64_t i = 0; i < w; ++i) sum_acc[o * w + i] += (double)msg[i];
        break;
      case OR_MAX:
        for (int64_t i = 0; i < w; ++i) orow[i] = orow[i] < msg[i] ? msg[i] : orow[i];
        break;
      case OR_MIN:
        for (int64_t i = 0; i < w; ++i) orow[i] = msg[i] < orow[i] ? msg[i] : orow[i];
        break;
      case OR_PROD:
        for (int64_t i = 0; i < w; ++i) orow[i] *= msg[i];
        break;
      default: {
        /* CopyLast: largest (other, eid) key wins, oracle.cpp:148-155 */
        const int later = !touched[o] || win_other[o] < other ||
                          (win_other[o] == other && win_eid[o] < (uint32_t)id);
        if (later) {
          win_other[o] = other;
          win_eid[o] = (uint32_t)id;
          memcpy(orow, msg, (size_t)w * sizeof(float));
        }
      }
    }
    touched[o] = 1;
  }
  if (sum_acc) {
    for (int64_t i = 0; i < out_rows * w; ++i) out_data[i] = (float)sum_acc[i];
  }
  if (out != OR_E && (reduce == OR_MAX || reduce == OR_MIN)) {
    for (int64_t r = 0; r < out_rows; ++r)
      if (!touched[r]) memset(out_data + r * w, 0, (size_t)w * sizeof(float));
  }
  free(sum_acc);
  free(touched);
  free(win_other);
  free(win_eid);
  free(msg);
  return OR_OK;
}

/* ------------------------------------------------ restated extensions */

/* a17.1: mean = binary_reduce(copy, sum) / (float)deg; 0 for empty rows. */
int or_mean(int orientation, uint32_t num_rows, uint32_t num_cols,
            const uint32_t* indptr, const uint32_t* indices,
            const uint32_t* eids, int lhs, const or_feat* src, float* out) {
  const int out_ent = orientation == OR_DST_MAJOR ? OR_V : OR_U;
  const or_feat* u = lhs == OR_U ? src : NULL;
  const or_feat* v = lhs == OR_V ? src : NULL;
  const or_feat* e = lhs == OR_E ? src : NULL;
  const int st = or_binary_reduce(orientation, num_rows, num_cols, indptr,
                                  indices, eids, lhs, OR_NONE, OR_COPY, OR_SUM,
                                  out_ent, u, v, e, out);
  if (st) return st;
  const int64_t w = src->dim;
  for (uint32_t r = 0; r < num_rows; ++r) {
    const uint32_t deg = indptr[r + 1] - indptr[r];
    float* row = out + (int64_t)r * w;
    for (int64_t i = 0; i < w; ++i) row[i] = deg ? row[i] / (float)deg : 0.0f;
  }
  return OR_OK;
}

/* a17.2: fused max + argmax; the value is the reference max fold
 * (kernels.cpp:41-43 with fixup :490-499), the arg is the first canonical
 * position that raised the running max. */
int or_copy_max_argmax(uint32_t num_rows, uint32_t num_cols,
                       const uint32_t* indptr, const uint32_t* indices,
                       const uint32_t* eids, int lhs, const or_feat* src,
                       float* out, int32_t* arg_other, int32_t* arg_eid) {
  (void)num_cols;
  const int64_t w = src->dim;
  for (uint32_t r = 0; r < num_rows; ++r) {
    for (int64_t i = 0; i < w; ++i) {
      float best = -INFINITY;
      int64_t arg = -1;
      for (uint32_t j = indptr[r]; j < indptr[r + 1]; ++j) {
        const int64_t row = lhs == OR_E ? eids[j] : indices[j];
        const float x = src->data[row * w + i];
        if (best < x) {
          best = x;
          arg = j;
        }
      }
      const int64_t o = (int64_t)r * w + i;
      if (indptr[r] == indptr[r + 1]) best = 0.0f;
      out[o] = best;
      if (arg_other) arg_other[o] = arg < 0 ? -1 : (int32_t)indices[arg];
      if (arg_eid) arg_eid[o] = arg < 0 ? -1 : (int32_t)eids[arg];
    }
  }
  return OR_OK;
}

/* a17.4: gradient through the argmax, f64 accumulation. */
void or_argmax_backward(int64_t rows, int64_t w, const int32_t* arg,
                        const float* grad_out, int64_t src_rows,
                        float* grad_src) {
  double* acc = (double*)calloc((size_t)(src_rows * w ? src_rows * w : 1), sizeof(double));
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t i = 0; i < w; ++i) {
      const int32_t a = arg[r * w + i];
      if (a >= 0) acc[(int64_t)a * w + i] += (double)grad_out[r * w + i];
    }
  for (int64_t i = 0; i < src_rows * w; ++i) grad_src[i] = (float)acc[i];
  free(acc);
}

/* a17.2 / a17.4 at BASELINE size: the same arithmetic, threaded (see the
 * header).  Edge-outer loop per row: column i's comparisons still happen in
 * canonical edge order, so the winner is the serial loop's winner. */
int or_copy_max_argmax_mt(uint32_t num_rows, uint32_t num_cols,
                          const uint32_t* indptr, const uint32_t* indices,
                          const uint32_t* eids, int lhs, const or_feat* src,
                          float* out, int32_t* arg_other, int32_t* arg_eid,
                          int threads) {
  (void)num_cols;
  const int64_t w = src->dim;
  if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel num_threads(threads)
  {
    int64_t* arg = (int64_t*)malloc((size_t)(w ? w : 1) * sizeof(int64_t));
#pragma omp for schedule(dynamic, 64)
    for (int64_t r = 0; r < (int64_t)num_rows; ++r) {
      float* best = out + r * w;
      for (int64_t i = 0; i < w; ++i) {
        best[i] = -INFINITY;
        arg[i] = -1;
      }
      for (uint32_t j = indptr[r]; j < indptr[r + 1]; ++j) {
        const int64_t row = lhs == OR_E ? eids[j] : indices[j];
        const float* x = src->data + row * w;
        for (int64_t i = 0; i < w; ++i)
          if (best[i] < x[i]) {
            best[i] = x[i];
            arg[i] = j;
          }
      }
      const int empty = indptr[r] == indptr[r + 1];
      for (int64_t i = 0; i < w; ++i) {
        if (empty) best[i] = 0.0f;
        if (arg_other) arg_other[r * w + i] = arg[i] < 0 ? -1 : (int32_t)indices[arg[i]];
        if (arg_eid) arg_eid[r * w + i] = arg[i] < 0 ? -1 : (int32_t)eids[arg[i]];
      }
    }
    free(arg);
  }
  return OR_OK;
}

void or_argmax_backward_mt(int64_t rows, int64_t w, const int32_t* arg,
                           const float* grad_out, int64_t src_rows,
                           float* grad_src, int threads) {
  if (threads <= 0) threads = omp_get_max_threads();
  double* acc = (double*)calloc((size_t)(src_rows * w ? src_rows * w : 1), sizeof(double));
#pragma omp parallel num_threads(threads)
  {
    const int64_t t = omp_get_thread_num(), nt = omp_get_num_threads();
    const int64_t lo = src_rows * t / nt, hi = src_rows * (t + 1) / nt;
    for (int64_t r = 0; r < rows; ++r)
      for (int64_t i = 0; i < w; ++i) {
        const int32_t a = arg[r * w + i];
        if (a >= lo && a < hi) acc[(int64_t)a * w + i] += (double)grad_out[r * w + i];
      }
#pragma omp barrier
#pragma omp for schedule(static)
    for (int64_t i = 0; i < src_rows * w; ++i) grad_src[i] = (float)acc[i];
  }
  free(acc);
}

/* ---------------------------------------------------------- comparison */

/* max_rel_error, compare.hpp:30-45 */
double or_max_rel_error(int64_t n, const float* got, const float* want) {
  double worst = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double g = got[i], w = want[i];
    if (isnan(g) != isnan(w)) return INFINITY;
    if (isnan(g)) continue;
    const double aw = fabs(w);
    const double err = fabs(g - w) / (aw > 1.0 ? aw : 1.0);
    if (err > worst) worst = err;
  }
  return worst;
}

/* bit_equal, compare.hpp:47-54 (IEEE ==, NaN==NaN) */
int or_bit_equal(int64_t n, const float* a, const float* b) {
  for (int64_t i = 0; i < n; ++i) {
    if (isnan(a[i]) && isnan(b[i])) continue;
    if (a[i] != b[i]) return 0;
  }
  return 1;
}

/*
 * gspmm_oracle.h -- CPU restatement of the reference aggregation path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the checker the parity tests, the
 * smoke() entry point and bench.py's cpu_baseline leg compare against.  The
 * product (paper_2007_06354_b200/) never links, loads or calls it.
 *
 * Every function restates the algorithm of the reference C++ library under
 * /root/reference/proj (cited file:line per function in gspmm_oracle.c).
 * Parity of this restatement is pinned against (a) the hand goldens of the
 * reference's own doctest suites and (b) fixtures produced by the reference
 * library itself (oracle/_ref, built from the reference sources by
 * oracle/Makefile), see tests/golden/make_golden.py.
 *
 * Ids are u32 (reference default, proj/include/gspmm/types.hpp:25-31),
 * features f32 row-major with row stride == dim (feature_matrix.hpp:29-36).
 */
#ifndef GSPMM_ORACLE_H
#define GSPMM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes, mirroring the reference exception taxonomy (error.hpp:22-45) */
enum { OR_OK = 0, OR_CONFIG = 1, OR_SHAPE = 2, OR_STRUCTURE = 3 };
/* enums with the reference's numeric values (ops.hpp:28,33; br_config.hpp) */
enum { OR_U = 0, OR_V = 1, OR_E = 2, OR_NONE = 3 };
enum { OR_ADD = 0, OR_SUB = 1, OR_MUL = 2, OR_DIV = 3, OR_DOT = 4, OR_COPY = 5 };
enum { OR_SUM = 0, OR_MAX = 1, OR_MIN = 2, OR_PROD = 3, OR_LAST = 4 };
enum { OR_SRC_MAJOR = 0, OR_DST_MAJOR = 1 };

/* ---- rng (rng.hpp:26-43) ---- */
uint64_t or_splitmix64_at(uint64_t seed, uint64_t counter);
double or_u01_at(uint64_t seed, uint64_t counter);
float or_unit_float_at(uint64_t seed, uint64_t counter);
/* builder-defined N(0,1): Box-Muller on u01 draws 2i, 2i+1 */
float or_normal_at(uint64_t seed, uint64_t i);

/* ---- generators (generate.cpp) ----
 * Edge buffers are malloc'ed by the oracle; release with or_free. */
int64_t or_gen_er(uint32_t n, uint64_t num_edges, double prob, uint64_t seed,
                  uint32_t** src, uint32_t** dst);
int64_t or_gen_rmat(uint32_t n, uint64_t num_edges, double a, double b,
                    double c, double d, uint64_t seed, uint32_t** src,
                    uint32_t** dst);
int64_t or_gen_sbm(uint32_t n, int blocks, double p_in, double p_out,
                   uint64_t seed, uint32_t** src, uint32_t** dst);
void or_free(void* p);
int64_t or_gen_powerlaw(uint32_t n, uint32_t d_min, uint32_t d_max, uint64_t seed,
                        uint32_t** src, uint32_t** dst);
void or_random_features(int64_t rows, int64_t dim, uint64_t seed, float* out);
void or_normal_features(int64_t count, uint64_t seed, float* out);
void or_normal_features_at(int64_t offset, int64_t count, uint64_t seed, float* out);

/* ---- graph core (csr.cpp) ---- */
int or_build_csr(uint32_t n, int64_t m, const uint32_t* src,
                 const uint32_t* dst, int orientation, uint32_t* indptr,
                 uint32_t* indices, uint32_t* eids);
int or_transpose(uint32_t num_rows, uint32_t num_cols, const uint32_t* indptr,
                 const uint32_t* indices, const uint32_t* eids,
                 uint32_t* t_indptr, uint32_t* t_indices, uint32_t* t_eids);
/* 0 when canonical, else 1 + index of the first violated invariant class */
int or_validate(uint32_t num_rows, uint32_t num_cols, int64_t indptr_len,
                const uint32_t* indptr, int64_t m, const uint32_t* indices,
                const uint32_t* eids);

/* ---- aggregation ----
 * Operand matrices: pointer + rows + dim (null pointer = absent).
 * or_binary_reduce restates binary_reduce(RowParallelSpmm, ...)
 * (kernels.cpp:162-195, 413-501).  out must hold out_rows*w floats where
 * out_rows/w are reported by or_out_shape. */
typedef struct {
  const float* data;
  int64_t rows;
  int64_t dim;
} or_feat;

int or_out_shape(int orientation, uint32_t num_rows, uint32_t num_cols,
                 int64_t m, int lhs, int rhs, int binop, int reduce, int out,
                 const or_feat* u, const or_feat* v, const or_feat* e,
                 int64_t* out_rows, int64_t* out_dim);
int or_binary_reduce(int orientation, uint32_t num_rows, uint32_t num_cols,
                     const uint32_t* indptr, const uint32_t* indices,
                     const uint32_t* eids, int lhs, int rhs, int binop,
                     int reduce, int out, const or_feat* u, const or_feat* v,
                     const or_feat* e, float* out_data);

/* oracle_aggregate (oracle.cpp:72-170): edge-id order, f64 sum. */
int or_oracle_aggregate(uint32_t num_nodes, int64_t m, const uint32_t* src,
                        const uint32_t* dst, int lhs, int rhs, int binop,
                        int reduce, int out, const or_feat* u,
                        const or_feat* v, const or_feat* e, float* out_data);

/* ---- restated operations the reference lacks ---- */
/* a17.1 mean = sum / (float)deg, 0 for empty rows; dst-major (out=V) or
 * src-major (out=U) owner rows. */
int or_mean(int orientation, uint32_t num_rows, uint32_t num_cols,
            const uint32_t* indptr, const uint32_t* indices,
            const uint32_t* eids, int lhs, const or_feat* src, float* out);
/* a17.2 copy max + argmax over canonical rows: best<x replaces, first
 * canonical position wins; arg_other = neighbour id, arg_eid = edge id,
 * -1 for empty rows (value 0).  lhs = U (gather neighbour) or E. */
int or_copy_max_argmax(uint32_t num_rows, uint32_t num_cols,
                       const uint32_t* indptr, const uint32_t* indices,
                       const uint32_t* eids, int lhs, const or_feat* src,
                       float* out, int32_t* arg_other, int32_t* arg_eid);
/* a17.4 grad through argmax: grad_src[arg[r,f], f] += grad_out[r,f],
 * f64 accumulation, rows with arg -1 skipped. */
void or_argmax_backward(int64_t rows, int64_t w, const int32_t* arg,
                        const float* grad_out, int64_t src_rows,
                        float* grad_src);

/* Multithreaded forms of the two a17 extensions for BASELINE-size parity
 * (OpenMP, `threads` <= 0: all).  Same results as the single-threaded
 * restatements: or_copy_max_argmax_mt splits rows over threads and walks
 * each row's edges in canonical order, updating every column (each column
 * still sees the edges in order, so the first strict maximum wins);
 * or_argmax_backward_mt gives each thread a contiguous range of source rows
 * and scans all (row, column) pairs in order, so every accumulator receives
 * its terms in ascending row order, exactly as the serial loop. */
int or_copy_max_argmax_mt(uint32_t num_rows, uint32_t num_cols,
                          const uint32_t* indptr, const uint32_t* indices,
                          const uint32_t* eids, int lhs, const or_feat* src,
                          float* out, int32_t* arg_other, int32_t* arg_eid,
                          int threads);
void or_argmax_backward_mt(int64_t rows, int64_t w, const int32_t* arg,
                           const float* grad_out, int64_t src_rows,
                           float* grad_src, int threads);

/* ---- comparison (compare.hpp:30-54) ---- */
double or_max_rel_error(int64_t n, const float* got, const float* want);
int or_bit_equal(int64_t n, const float* a, const float* b);

#ifdef __cplusplus
}
#endif
#endif

/*
 * gspmm_b200.h -- C-ABI of the B200-native Copy-Reduce / Binary-Reduce path.
 *
 * Drop-in boundary for the reference's hot path (arXiv 2007.06354's
 * aggregation primitives, re-implemented by /root/reference/proj as
 * gspmm::binary_reduce / gspmm::copy_reduce):
 *
 *   reference (proj/include/gspmm/kernels.hpp)        this ABI
 *   -----------------------------------------------   -------------------------
 *   FeatureMatrix binary_reduce(Strategy, const        gspmm_binary_reduce /
 *     CsrGraph&, const BrConfig&, const FeatureMatrix*  gspmm_binary_reduce_host
 *     u, v, e, const BlockPlan*, int threads)           (kernels.hpp:60-64)
 *   FeatureMatrix copy_reduce(Strategy, const         gspmm_copy_reduce
 *     CsrGraph&, const FeatureMatrix&, ReduceOp, ...)   (kernels.hpp:71-73)
 *   Orientation required_orientation(Strategy,        gspmm_required_orientation
 *     Operand out)                                      (kernels.hpp:48)
 *   CsrGraph (indptr/indices/edge_ids, csr.hpp:37-54) gspmm_graph_create: a
 *     + BlockPlan (block_plan.hpp:39-88)                device handle holding the
 *                                                       CSR and the device plan
 *   void validate_config(const BrConfig&)             gspmm_validate_config
 *     (br_config.hpp:46)
 *   StructureError/ShapeError/ConfigError             GSPMM_ERR_* status codes +
 *     (error.hpp:22-45)                                 gspmm_last_error()
 *
 * Plain C types only: pointers, sizes, int32 enums whose numeric values are
 * the reference's (ops.hpp:28,33; br_config.hpp Operand; types.hpp:35).
 * Node/edge ids are uint32 (types.hpp:25-31).  Features are fp32 row-major
 * with an explicit row stride `ld` (elements); ld == 0 means ld == dim, the
 * reference's FeatureMatrix layout.
 *
 * Device entry points take DEVICE pointers and enqueue on `stream`
 * (cudaStream_t, NULL = legacy default stream); they return after launch.
 * Host entry points (`*_host`) take HOST pointers, stage through a
 * stream-ordered device allocation and return after the result is back on
 * the host, like the reference's synchronous call.
 *
 * Thread safety (the reference's CsrGraph is safe to share, csr.hpp:35): a
 * graph handle may be used by any number of host threads and streams at
 * once.  Each caller stream gets its own per-call device state (work
 * counters, workspaces) and every call waits for the previous call that used
 * the same state, so concurrent calls never share a counter or a buffer.
 * Destroying a handle, gspmm_graph_set_plan and gspmm_graph_set_source_blocks
 * must not race with calls on that handle.
 *
 * Semantics (identical to the reference, bit for bit):
 *   - each output element is a sequential fp32 left fold, from the reduce
 *     identity, over the owner row's edges in canonical CSR order (rows
 *     ascending; neighbour ascending; edge id ascending), every multiply and
 *     add rounded separately (kernels.cpp:162-195);
 *   - Max uses `a < m ? m : a`, Min `m < a ? m : a` (kernels.cpp:38-52);
 *   - Max/Min rows with no edges read 0 (kernels.cpp:490-499), other
 *     reducers leave the identity;
 *   - width-1 operands broadcast (stride 0, kernels.cpp:444-453);
 *   - out == E stores one message per edge row, indexed by edge id.
 */
#ifndef GSPMM_B200_H
#define GSPMM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GSPMM_B200_ABI_VERSION 3

/* ---- status (error.hpp:22-45 taxonomy, plus device failures) ---- */
enum {
  GSPMM_OK = 0,
  GSPMM_ERR_CONFIG = 1,    /* ConfigError: invalid descriptor             */
  GSPMM_ERR_SHAPE = 2,     /* ShapeError: operand/orientation mismatch     */
  GSPMM_ERR_STRUCTURE = 3, /* StructureError: malformed CSR                */
  GSPMM_ERR_CUDA = 4,      /* CUDA runtime failure (no device, OOM, ...)   */
  GSPMM_ERR_ARG = 5,       /* null handle / bad pointer argument           */
  GSPMM_ERR_IO = 6,        /* IoError: unreadable / corrupt container      */
  GSPMM_ERR_PARSE = 7      /* ParseError: text input that does not parse   */
};

/* ---- enums: numeric values of the reference ---- */
enum { GSPMM_U = 0, GSPMM_V = 1, GSPMM_E = 2, GSPMM_NONE = 3 };           /* Operand */
enum { GSPMM_ADD = 0, GSPMM_SUB = 1, GSPMM_MUL = 2, GSPMM_DIV = 3,
       GSPMM_DOT = 4, GSPMM_COPY = 5 };                                   /* BinaryOp */
enum { GSPMM_SUM = 0, GSPMM_MAX = 1, GSPMM_MIN = 2, GSPMM_PROD = 3,
       GSPMM_COPY_LAST = 4,
       GSPMM_MEAN = 5 /* extension: sum / in-degree, 0 for empty rows */ }; /* ReduceOp */
enum { GSPMM_SRC_MAJOR = 0, GSPMM_DST_MAJOR = 1 };                       /* Orientation */
enum { GSPMM_PUSH = 0, GSPMM_PULL = 1, GSPMM_BLOCKED = 2, GSPMM_SPMM = 3 }; /* Strategy */

/* Row order of an edge operand. */
enum {
  GSPMM_EDGE_BY_ID = 0,  /* row i is edge id i (the reference's layout)      */
  GSPMM_EDGE_BY_POS = 1  /* row j is the j-th nonzero of THIS handle's CSR,  */
                         /* produced once by gspmm_graph_permute_edges       */
};

/* BrConfig (br_config.hpp:37-44) */
typedef struct {
  int32_t lhs, rhs, binary, reduce, out;
} gspmm_config;

/* A feature matrix view (FeatureMatrix, feature_matrix.hpp:29-66).
 * data == NULL means "operand not supplied". */
typedef struct {
  const float* data;
  int64_t rows;
  int64_t dim;
  int64_t ld;          /* row stride in floats, 0 -> dim */
  int32_t edge_order;  /* GSPMM_EDGE_BY_ID / _BY_POS, E operands only */
} gspmm_mat;

typedef struct {
  float* data;
  int64_t rows;
  int64_t dim;
  int64_t ld; /* 0 -> dim */
} gspmm_out;

/* Extensions the reference does not have. Zero-init = off. */
typedef struct {
  /* Max/Min: winning edge per output element, -1 when no edge raised the
   * running value (empty rows).  [out rows x dim], stride arg_ld (0 -> dim).
   * First canonical position wins ties (the `a < m` scan). */
  int32_t* arg_other; /* neighbour node id of the winning edge */
  int32_t* arg_edge;  /* edge id of the winning edge           */
  int64_t arg_ld;
  /* Multi-head broadcast: an operand of width H (H divides the output
   * width W) broadcasts each element over W/H consecutive columns
   * (DGL's [N,H,D] x [E,H,1]).  With binary == DOT: `heads` per-head dot
   * products over gather_dim/heads columns, output width = heads. */
  int32_t heads;
  /* Per-node scale of each edge's OTHER endpoint (the gathered node):
   * message := message * other_scale[other], rounded (used for the mean
   * backward: e = 1/deg_in(dst)). Device pointer (host pointer in the
   * *_host entries), length = #other nodes. */
  const float* other_scale;
  /* Source blocking for this call (see gspmm_graph_set_source_blocks):
   * 0 = the handle's setting, 1 = never, >= 2 = that many blocks. */
  int32_t source_blocks;
  /* A second reduction of the same messages in the same call: out2 [out
   * rows x width] (stride out2_ld, 0 -> width) receives
   * binary_reduce(cfg with reduce = reduce2), reduce2 = GSPMM_SUM or
   * GSPMM_MEAN -- bit-identical to a separate call.  With a Max/Min copy
   * config (config 3's max + argmax and mean) both folds run over ONE
   * gather of the source rows; other configs run it as a second pass.
   * out2 == NULL: off.  Device pointer (host pointer in the *_host entries). */
  float* out2;
  int64_t out2_ld;
  int32_t reduce2;
} gspmm_options;

typedef struct gspmm_graph_s* gspmm_graph;

/* Device plan options (gspmm_graph_set_plan).  Zero-init = the defaults.
 * The plan only changes how work is cut into units, never a result: every
 * output stays the canonical left fold -- except under split_edges, the one
 * option that trades the bits of long rows' sums for speed. */
typedef struct {
  uint32_t seg_cost;       /* cost (edges + 2 per row) of a segment unit; 0 -> 256 */
  uint32_t long_threshold; /* 0 -> automatic plan levels; else rows above this
                              degree always run as long-row column units */
  uint32_t unit_cols;      /* 0 -> automatic long-row unit widths; else this
                              many columns per unit (multiple of 4, <= 512) */
  int32_t kernel;          /* 0 = planned kernels; 1 = the register kernel
                              (rows.cu) for every call (a reference path);
                              2 = planned kernels with the segment kernel
                              launched as a programmatic dependent of the
                              long-row kernel, its blocks taking each SM a
                              long-row CTA leaves (measured slower on
                              configs 2 and 3) */
  uint32_t long_ctas;      /* 0 -> long-row units first, on every SM, then the
                              segments (default); N -> the long-row units run
                              concurrently with the segment kernel on N CTAs
                              (one per SM; measured slower on config 3) */
  uint32_t split_edges;    /* Rows above the plan's long-row threshold cut into
                              chunks of edges, folded like short rows and
                              combined in chunk order.  Max / Min are exact
                              under any association and the strict compare
                              keeps the first winner, so value and argmax
                              stay the reference's bits; a Sum / Mean becomes
                              a fixed-order sum of chunk sums: deterministic,
                              the same order of rounding error as the
                              sequential fold, but NOT within the reference's
                              1e-5 of that fold on hub rows (measured 9e-4 on
                              config 3's mean backward: the fp32 fold of a
                              10^5-edge row carries that much rounding
                              itself), i.e. outside the parity contract.
                              0 -> automatic (default): Max / Min without a
                              fused second sum in chunks of 512, every sum
                              one sequential fold; 1 -> never split (every
                              long row on the long-row kernel); N >= 16 ->
                              split every reduction, sums included, at N */
} gspmm_plan;

/* ---- errors ---- */
const char* gspmm_last_error(void); /* thread-local message of the last failure */
int gspmm_abi_version(void);

/* ---- descriptor helpers (host only, no device needed) ---- */
/* validate_config, br_config.cpp:83-94 */
int gspmm_validate_config(const gspmm_config* cfg);
/* named_config, br_config.cpp:96-131: "u_mul_e_add_v", "u_copy_max_v", ... */
int gspmm_named_config(const char* name, gspmm_config* cfg);
/* required_orientation, kernels.cpp:400-411; returns the orientation or -1 */
int gspmm_required_orientation(int strategy, int out);

/* ---- graph handle (CsrGraph + device plan) ----
 * Uploads a canonical CSR (host arrays) to `device`.  validate != 0 runs the
 * reference's validate() checks (csr.cpp:111-156) on the host first and
 * returns GSPMM_ERR_STRUCTURE on failure.  The handle owns the device CSR,
 * the degree-binned row plan and a workspace for host calls. */
int gspmm_graph_create(int device, int orientation, uint32_t num_rows,
                       uint32_t num_cols, const uint32_t* indptr,
                       const uint32_t* indices, const uint32_t* edge_ids,
                       int validate, gspmm_graph* out);
/* Same, from DEVICE arrays of a canonical CSR (e.g. gspmm_build_csr_device
 * output): indptr is read back for the row plan, indices / edge_ids are
 * copied device to device.  No host validation. */
int gspmm_graph_create_device(int device, int orientation, uint32_t num_rows,
                              uint32_t num_cols, const uint32_t* d_indptr,
                              const uint32_t* d_indices,
                              const uint32_t* d_edge_ids, gspmm_graph* out);
int gspmm_graph_destroy(gspmm_graph g);
int gspmm_graph_info(gspmm_graph g, int* orientation, uint32_t* num_rows,
                     uint32_t* num_cols, uint64_t* num_edges,
                     uint32_t* num_long_rows);
/* Device copies of the handle's CSR arrays (read-only). */
int gspmm_graph_device_csr(gspmm_graph g, const uint32_t** indptr,
                           const uint32_t** indices, const uint32_t** edge_ids);
/* Permutes an edge operand from edge-id order into this handle's CSR
 * position order (dst[j] = src[edge_ids[j]]), on the device.  The untimed
 * analogue of the reference's BlockPlan build (bench.cpp:95-97). */
int gspmm_graph_permute_edges(gspmm_graph g, const float* src_by_id,
                              int64_t dim, int64_t src_ld, float* dst_by_pos,
                              int64_t dst_ld, void* stream);

/* Source blocking (the paper's Alg. 3 / BlockPlan, block_plan.hpp:39-75 and
 * run_blocked kernels.cpp:278-326, which the reference shows is byte-identical
 * to Pull): an aggregation that gathers neighbour rows runs as nblocks passes,
 * pass b folding only the neighbours in id block b into the partial rows left
 * by pass b-1, so each pass's gathered rows fit the 126 MB L2.  Canonical
 * rows are sorted by neighbour, so the passes replay every row's fold order:
 * results stay bit-identical.  nblocks: 0 = automatic (default; blocks when
 * the gathered operand is several times the L2 and the rows are dense
 * enough to amortise the partial-row traffic), 1 = never, >= 2 = that many
 * blocks whenever the call admits it (sum / mean / max / min without argmax,
 * gathered lhs, no CSR-position edge operand).  Block CSRs are built on the
 * device on first use. */
int gspmm_graph_set_source_blocks(gspmm_graph g, int nblocks);
/* Rebuilds the handle's device plan with the given options (NULL: defaults). */
int gspmm_graph_set_plan(gspmm_graph g, const gspmm_plan* plan);

/* ---- compute (device pointers, asynchronous on stream) ---- */
int gspmm_binary_reduce(gspmm_graph g, const gspmm_config* cfg,
                        const gspmm_mat* u, const gspmm_mat* v,
                        const gspmm_mat* e, const gspmm_out* out,
                        void* stream);
int gspmm_binary_reduce_ex(gspmm_graph g, const gspmm_config* cfg,
                           const gspmm_mat* u, const gspmm_mat* v,
                           const gspmm_mat* e, const gspmm_out* out,
                           const gspmm_options* opt, void* stream);
/* copy_reduce (kernels.cpp:503-524): source entity inferred from
 * src->rows (node count first, then edge count). */
int gspmm_copy_reduce(gspmm_graph g, const gspmm_mat* src, int reduce,
                      const gspmm_out* out, void* stream);
/* Gradient through an argmax: grad_src[arg[r,f], f] += grad_out[r,f]
 * (f64 accumulation, then rounded to fp32; arg -1 skipped).  grad_src is
 * overwritten. */
int gspmm_argmax_backward(const int32_t* arg, int64_t rows, int64_t dim,
                          int64_t arg_ld, const float* grad_out,
                          int64_t grad_ld, float* grad_src, int64_t src_rows,
                          int64_t src_ld, void* stream);
/* The same for the source rows [src_lo, src_lo + src_rows) only (grad_src
 * row i is source row src_lo + i; other targets are skipped): a rank's own
 * rows in the multi-GPU owner-computes backward. */
int gspmm_argmax_backward_range(const int32_t* arg, int64_t rows, int64_t dim,
                                int64_t arg_ld, const float* grad_out,
                                int64_t grad_ld, float* grad_src, int64_t src_lo,
                                int64_t src_rows, int64_t src_ld, void* stream);
/* Host-buffer forms (dense rows): arg / grad_out uploaded, grad_src read
 * back; on `device`.  _async: enqueue only, with the wait / upload events of
 * gspmm_binary_reduce_host_async. */
int gspmm_argmax_backward_host(const int32_t* arg, int64_t rows, int64_t dim,
                               const float* grad_out, float* grad_src,
                               int64_t src_rows, int device, void* stream);
int gspmm_argmax_backward_host_async(const int32_t* arg, int64_t rows, int64_t dim,
                                     const float* grad_out, float* grad_src,
                                     int64_t src_rows, int device, void* stream,
                                     void* wait_event, void* upload_event);

/* Fused GAT edge softmax over the in-edges of each destination (
 * the composite e_copy_max_v -> e_sub_v_copy_e -> exp -> e_copy_add_v ->
 * e_div_v_copy_e of PAPER Table 2): per head h,
 *   a[e,h] = expf(l[e,h] - m[v,h]) / z[v,h],  m = max, z = sum over in-edges of v.
 * Dst-major handle.  logits / out: E x heads (heads <= 32), rows in the
 * logits' edge_order (GSPMM_EDGE_BY_ID: row = edge id; BY_POS: CSR position);
 * out uses the same order.  The max is the reference reducer; z is an fp32
 * sum in a fixed order (deterministic); parity with the composite is within
 * tolerance (expf). */
int gspmm_edge_softmax(gspmm_graph g, const gspmm_mat* logits,
                       const gspmm_out* out, void* stream);
/* Its backward: grad_l[e,h] = a[e,h] * (grad_a[e,h] - sum_row(a * grad_a)[v,h]). */
int gspmm_edge_softmax_backward(gspmm_graph g, const gspmm_mat* a,
                                const gspmm_mat* grad_a,
                                const gspmm_out* grad_logits, void* stream);

/* ---- host-buffer entry (the reference's synchronous call shape) ----
 * Same arguments with HOST pointers; copies in, computes, copies out and
 * synchronizes.  Pinned host memory makes the copies asynchronous DMA. */
int gspmm_binary_reduce_host(gspmm_graph g, const gspmm_config* cfg,
                             const gspmm_mat* u, const gspmm_mat* v,
                             const gspmm_mat* e, const gspmm_out* out,
                             const gspmm_options* opt, void* stream);
/* The same host-buffer call, returning once the copies and kernels are
 * enqueued on `stream` (the outputs are valid after the stream synchronizes;
 * host buffers must be pinned and stay untouched until then).  The uploads
 * start after `wait_event` (a cudaEvent_t, or NULL), and `upload_event` (or
 * NULL) is recorded once the inputs are on the device: callers that stream
 * several independent calls on two streams use the pair to keep one upload
 * in flight at a time while the other call's kernel and download run, so
 * both PCIe directions stay busy.  In the host entries, options.other_scale
 * is a HOST array (one float per node of the gathered endpoint, num_cols of
 * the handle) uploaded with the operands. */
int gspmm_binary_reduce_host_async(gspmm_graph g, const gspmm_config* cfg,
                                   const gspmm_mat* u, const gspmm_mat* v,
                                   const gspmm_mat* e, const gspmm_out* out,
                                   const gspmm_options* opt, void* stream,
                                   void* wait_event, void* upload_event);

/* Output shape of a config on a handle (rows, width), after the full
 * reference validation (binary_reduce kernels.cpp:418-456). */
int gspmm_out_shape(gspmm_graph g, const gspmm_config* cfg,
                    const gspmm_mat* u, const gspmm_mat* v,
                    const gspmm_mat* e, const gspmm_options* opt,
                    int64_t* rows, int64_t* dim);

/* Number of kernels the library launched since load (evidence counter). */
uint64_t gspmm_launch_count(void);

/* ---- input synthesis and CSR construction (host, multithreaded) ----
 * Bit-identical to the reference's generators (generate.cpp) and CSR
 * builder (csr.cpp); threads <= 0 uses all hardware threads. */
int64_t gspmm_synth_rmat(uint32_t n, uint64_t num_edges, double a, double b,
                         double c, double d, uint64_t seed, uint32_t* src,
                         uint32_t* dst, int threads);
/* Erdos-Renyi: returns the edge count; buffers malloc'ed, free with gspmm_free */
int64_t gspmm_synth_er(uint32_t n, uint64_t num_edges, double prob,
                       uint64_t seed, uint32_t** src, uint32_t** dst);
void gspmm_free(void* p);
int gspmm_build_csr(uint32_t n, int64_t m, const uint32_t* src,
                    const uint32_t* dst, int orientation, uint32_t* indptr,
                    uint32_t* indices, uint32_t* edge_ids, int threads);
int gspmm_transpose(uint32_t num_rows, uint32_t num_cols,
                    const uint32_t* indptr, const uint32_t* indices,
                    const uint32_t* edge_ids, uint32_t* t_indptr,
                    uint32_t* t_indices, uint32_t* t_edge_ids, int threads);
/* Device-side canonical CSR construction (csr.cpp:31-109 on the GPU):
 * d_src / d_dst in edge-id order -> indptr[n+1], indices[m], edge_ids[m]
 * (rows = dst for GSPMM_DST_MAJOR, src for GSPMM_SRC_MAJOR; neighbours
 * ascending, then edge id).  Bit-identical to gspmm_build_csr. */
int gspmm_build_csr_device(uint32_t n, int64_t m, const uint32_t* d_src,
                           const uint32_t* d_dst, int orientation,
                           uint32_t* d_indptr, uint32_t* d_indices,
                           uint32_t* d_edge_ids, void* stream);
/* Device-side transpose of a canonical CSR (csr.cpp:95-109). */
int gspmm_transpose_device(uint32_t num_rows, uint32_t num_cols, int64_t m,
                           const uint32_t* d_indptr, const uint32_t* d_indices,
                           const uint32_t* d_edge_ids, uint32_t* d_t_indptr,
                           uint32_t* d_t_indices, uint32_t* d_t_edge_ids,
                           void* stream);
/* U[-1,1) (random_features, generate.cpp:256-266) and builder N(0,1) */
void gspmm_synth_uniform(int64_t count, uint64_t seed, float* out, int threads);
void gspmm_synth_normal(int64_t count, uint64_t seed, float* out, int threads);
/* Power-law in-degree graph (cfg5, GraphSAGE-mean on a Reddit-shaped graph;
 * builder-defined): node v draws its in-degree from the discrete
 * inverse CDF of P(d) ~ d^-2 on [d_min, d_max] with u01(seed, v); its edges
 * follow in edge-id order, each source uniform on [0, n) by the 128-bit
 * multiply-shift of splitmix64(seed ^ 0x5851f42d4c957f2d, edge id).
 * Call with src/dst NULL to get the edge count. */
int64_t gspmm_synth_powerlaw(uint32_t n, uint32_t d_min, uint32_t d_max,
                             uint64_t seed, uint32_t* src, uint32_t* dst,
                             int threads);
/* GCN weight w[e] = 1/sqrt(deg_out(src[e]) * deg_in(dst[e])), edge-id order */
void gspmm_synth_gcn_weights(uint32_t n, int64_t m, const uint32_t* src,
                             const uint32_t* dst, float* w, int threads);

/* ---- file containers (io.hpp:25-41, io.cpp:80-207) ----
 * FMAT1: "FMAT1", u64 rows, u64 dim, rows * dim float32 (little-endian).
 * CSR1:  "CSR1", u8 orientation (0 src-major, else dst-major), u64 num_rows,
 *        num_cols, num_edges, then indptr / indices / edge_ids as u64 arrays.
 * Failures are GSPMM_ERR_IO with the reference's IoError messages ("cannot
 * open ...", "... not a CSR1 file", "... truncated file", "... invalid CSR
 * payload: <validate() message>"). */
int gspmm_fmat1_info(const char* path, int64_t* rows, int64_t* dim);
/* load_feature_matrix (io.cpp:149-166) into a HOST buffer of row stride ld
 * (0 -> dim). */
int gspmm_fmat1_read(const char* path, float* data, int64_t ld);
/* The same into a DEVICE buffer on `device` (row stride ld, 0 -> dim; pad
 * columns untouched): the file streams through a pinned ring, the read of
 * one chunk overlapping the DMA of the previous.  Synchronizes `stream`. */
int gspmm_fmat1_read_device(const char* path, int device, float* d_data,
                            int64_t ld, void* stream);
/* save_feature_matrix (io.cpp:137-147) from a host matrix. */
int gspmm_fmat1_write(const char* path, const float* data, int64_t rows,
                      int64_t dim, int64_t ld);
int gspmm_csr1_info(const char* path, int* orientation, uint64_t* num_rows,
                    uint64_t* num_cols, uint64_t* num_edges);
/* load_csr (io.cpp:183-205) into HOST arrays sized from gspmm_csr1_info
 * (indptr num_rows + 1, indices / edge_ids num_edges); validated. */
int gspmm_csr1_read(const char* path, uint32_t* indptr, uint32_t* indices,
                    uint32_t* edge_ids);
/* save_csr (io.cpp:168-181). */
int gspmm_csr1_write(const char* path, int orientation, uint32_t num_rows,
                     uint32_t num_cols, const uint32_t* indptr,
                     const uint32_t* indices, const uint32_t* edge_ids);
/* load_csr straight to a device graph handle: the 64-bit payload streams
 * through a pinned ring, is narrowed to 32-bit ids on the device (an id
 * above 2^32 - 1 is an IoError, io.cpp:71-73) and checked on the device with
 * validate()'s rules and messages (csr.cpp:111-156) before the plan is built. */
int gspmm_graph_load_csr1(const char* path, int device, gspmm_graph* out);
/* validate() (csr.cpp:111-156) of a DEVICE CSR, e.g. before
 * gspmm_graph_create_device: GSPMM_ERR_STRUCTURE with the reference's
 * message (the lowest offending nonzero, as its sequential scan reports). */
int gspmm_validate_csr_device(int device, uint32_t num_rows, uint32_t num_cols,
                              const uint32_t* d_indptr, const uint32_t* d_indices,
                              const uint32_t* d_edge_ids, void* stream);
/* load_edge_list / save_edge_list (io.cpp:80-135): "src dst" per line, '#'
 * comments, optional "%nodes N".  src / dst are malloc'ed (gspmm_free); they
 * feed gspmm_build_csr[_device].  Parse failures are GSPMM_ERR_PARSE with
 * "<path>:<line>: <what>". */
int gspmm_edge_list_read(const char* path, uint32_t* num_nodes,
                         uint64_t* num_edges, uint32_t** src, uint32_t** dst);
int gspmm_edge_list_write(const char* path, uint32_t num_nodes,
                          uint64_t num_edges, const uint32_t* src,
                          const uint32_t* dst);

#ifdef __cplusplus
}
#endif
#endif /* GSPMM_B200_H */

// internal.h -- launch descriptors shared by the C-ABI layer (capi.cpp) and
// the sm_100a kernels (*.cu).  Not part of the public ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace gspmm_b200 {

// Which endpoint of an edge an operand row is taken from, resolved by the
// host from (operand entity, graph orientation) -- the reference's
// OperandRef::row (kernels.cpp:120-125) split_endpoints (:138-147).
enum Role : int32_t {
  ROLE_ROW = 0,    // the owner row itself (constant across the row's edges)
  ROLE_OTHER = 1,  // indices[j]: the gathered neighbour
  ROLE_EID = 2,    // edge_ids[j]: an edge operand in edge-id order
  ROLE_POS = 3     // j: an edge operand pre-permuted to CSR position order
};

// How an operand's elements map onto the output columns.
enum Mode : int32_t {
  MODE_FULL = 0,    // column c reads element c
  MODE_SCALAR = 1,  // width-1 broadcast, stride 0 (kernels.cpp:451-453)
  MODE_HEAD = 2     // width-H broadcast over groups of `group` columns
};

struct OperandDesc {
  const float* base = nullptr;
  int64_t ld = 0;
  int32_t role = ROLE_OTHER;
  int32_t mode = MODE_FULL;
  int32_t group = 1;
  int64_t rows = 0;  // entity rows (the gather4 tensor map's extent)
};

enum BinOp : int32_t { B_ADD = 0, B_SUB = 1, B_MUL = 2, B_DIV = 3, B_DOT = 4, B_COPY = 5 };
enum RedOp : int32_t { R_SUM = 0, R_MAX = 1, R_MIN = 2, R_PROD = 3, R_LAST = 4 };

struct RowLaunch {
  const uint32_t* indptr = nullptr;
  const uint32_t* indices = nullptr;
  const uint32_t* eids = nullptr;
  uint32_t num_rows = 0;
  OperandDesc lhs, rhs;  // rhs.base == nullptr for the copy operator
  int32_t binop = B_COPY;
  int32_t reduce = R_SUM;
  bool mean = false;       // divide by the row degree (0 for empty rows)
  bool out_edge = false;   // out == E: store per edge (row = edge id)
  float* out = nullptr;
  int64_t out_ld = 0;
  int32_t width = 0;       // output width W
  int32_t gather_dim = 0;  // dot: reduced length
  int32_t heads = 1;       // dot: per-head products
  int32_t* arg_other = nullptr;
  int32_t* arg_edge = nullptr;
  int64_t arg_ld = 0;
  const float* other_scale = nullptr;
  int32_t vec = 4;         // vector width chosen by the host (4, 2, 1)
  // degree plan: rows whose degree exceeds long_threshold are listed in
  // long_rows (descending degree) and processed first.
  const uint32_t* long_rows = nullptr;
  uint32_t num_long = 0;
  uint32_t long_threshold = 0xffffffffu;
  int num_sms = 148;
  // Source-blocked passes (the paper's source blocking, Alg. 3 /
  // block_plan.cpp): rows start from the partial result in acc_in (== out)
  // instead of the reduce identity; epi = 1 stores the raw fold (a partial
  // for the next pass), epi = 2 is the last pass, whose mean / zero-degree
  // fixup takes the degree from deg_indptr (the whole graph's row pointer).
  const float* acc_in = nullptr;
  const uint32_t* deg_indptr = nullptr;
  int32_t epi = 0;
  int32_t src_blocks = 0;  // per-call source blocking (0 = the handle's setting)
  // second reduction of the same messages (Sum, or Mean when mean2) into
  // out2, fused into the gather (planned kernels, copy + Max/Min only)
  float* out2 = nullptr;
  int64_t out2_ld = 0;
  bool mean2 = false;
  // 1.0f and 1 as launch parameters, opaque to ptxas: the argmax fold's
  // conditional value copy becomes an FFMA (FMA pipes) instead of an FSEL
  // (gather_impl.cuh, GATHER_FMA_SELECT)
  float f_one = 1.0f;
  uint32_t u_one = 1u;
};

// Kernel launchers (rows.cu, dot.cu, aux.cu).  Return cudaGetLastError().
cudaError_t launch_rows(const RowLaunch& p, cudaStream_t s);
cudaError_t launch_dot(const RowLaunch& p, cudaStream_t s);
// out == E dot over edge batches; rowof[j] = owner row of CSR position j
cudaError_t launch_dot_edges(const RowLaunch& p, const uint32_t* rowof, uint64_t m,
                             cudaStream_t s);
cudaError_t launch_row_of_edge(const uint32_t* indptr, uint32_t rows, uint32_t* rowof,
                               cudaStream_t s);
cudaError_t launch_permute_edges(const uint32_t* eids, uint64_t m,
                                 const float* src, int64_t dim, int64_t src_ld,
                                 float* dst, int64_t dst_ld, cudaStream_t s);
// grad_src[arg[r,f] - src_lo, f] += grad_out[r,f] for targets inside
// [src_lo, src_lo + src_rows) (f64 accumulation, rounded once); grad_src
// overwritten.  Stream-ordered workspace.
cudaError_t launch_argmax_backward(const int32_t* arg, int64_t rows, int64_t dim,
                                   int64_t arg_ld, const float* grad_out, int64_t grad_ld,
                                   float* grad_src, int64_t src_lo, int64_t src_rows,
                                   int64_t src_ld, cudaStream_t s);

// A handle's side stream and fork / join events (hub-row kernels run there,
// concurrently with the warp-per-row kernels).  stream == nullptr: serial.
struct SideStream {
  cudaStream_t stream = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};

// Fused edge softmax over in-edges (softmax.cu): forward (l -> out = a) or
// backward (l = a, g = grad_a -> out = grad_l).  Rows above long_threshold
// edges are listed in long_rows and run one CTA per row.  counter: one
// uint32 of the call's context (the warp-per-row kernel hands rows out in
// groups from it); nullptr = rows strided over the grid.
cudaError_t launch_edge_softmax(bool backward, const uint32_t* indptr, const uint32_t* eids,
                                uint32_t rows, int heads, bool by_pos, const float* l,
                                int64_t l_ld, const float* g, int64_t g_ld, float* out,
                                int64_t out_ld, const uint32_t* long_rows, uint32_t n_long,
                                uint32_t long_threshold, int num_sms, cudaStream_t s,
                                const SideStream& side = SideStream{},
                                uint32_t* counter = nullptr);

// Device-side canonical CSR build / transpose (build.cu).
cudaError_t launch_build_csr(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                             bool dst_major, uint32_t* indptr, uint32_t* indices, uint32_t* eids,
                             cudaStream_t s);
// Lowest edge id whose src or dst is >= n (~0 when all ids are in range);
// synchronizes the stream.
cudaError_t check_edge_ids(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                           cudaStream_t s, uint64_t* first_bad);
cudaError_t launch_transpose_csr(uint32_t num_rows, uint32_t num_cols, uint64_t m,
                                 const uint32_t* indptr, const uint32_t* indices,
                                 const uint32_t* eids, uint32_t* t_indptr, uint32_t* t_indices,
                                 uint32_t* t_eids, cudaStream_t s);

// Source blocks (build.cu): bpos[(nb + 1) x rows] = per-row sub-range
// bounds of nb neighbour blocks of bs ids; then, per block, the block's CSR
// (indptr_b[rows + 1], idx_b / eid_b) from the bounds lo = bpos[b], hi =
// bpos[b + 1].
cudaError_t launch_block_bounds(const uint32_t* indptr, const uint32_t* indices, uint32_t rows,
                                uint32_t nb, uint32_t bs, uint32_t* bpos, cudaStream_t s);
cudaError_t launch_block_csr(const uint32_t* lo, const uint32_t* hi, uint32_t rows,
                             const uint32_t* indices, const uint32_t* eids, uint32_t* indptr_b,
                             uint32_t* idx_b, uint32_t* eid_b, cudaStream_t s);

// y[r, :] = x[r, :] * scale[r] over 16-byte aligned rows (ld, y_ld % 4 == 0)
// (aux.cu): the per-neighbour scale of the mean backward applied once per
// gathered row.
cudaError_t launch_scale_rows(const float* x, int64_t rows, int64_t dim, int64_t ld,
                              const float* scale, float* y, int64_t y_ld, cudaStream_t s);

// Long rows split by edge ranges (plan option split_edges): the partial folds
// of a long row's chunks (chunk rows [k0, k0 + nk) of part / part2 / parg_*,
// leading dimension pld) are combined in chunk order into the row's outputs,
// with the row epilogue (mean) applied.  ranges[i] = (k0, nk) of long_rows[i].
struct CombineLaunch {
  const uint32_t* long_rows = nullptr;
  const uint2* ranges = nullptr;
  uint32_t n_long = 0;
  const uint32_t* indptr = nullptr;  // the graph's row pointer (degrees)
  int32_t width = 0;
  int32_t reduce = R_SUM;
  int64_t pld = 0;
  const float* part = nullptr;
  const float* part2 = nullptr;
  const int32_t* parg_other = nullptr;
  const int32_t* parg_edge = nullptr;
  float* out = nullptr;
  int64_t out_ld = 0;
  float* out2 = nullptr;
  int64_t out2_ld = 0;
  int32_t* arg_other = nullptr;
  int32_t* arg_edge = nullptr;
  int64_t arg_ld = 0;
  bool mean = false, mean2 = false;
};
cudaError_t launch_combine_chunks(const CombineLaunch& c, cudaStream_t s);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device),
// thread-safe (aux.cu).
cudaError_t set_max_dynamic_smem(const void* func, int bytes);

// The thread-local message behind gspmm_last_error(); returns `status`.
int set_last_error(int status, const std::string& msg);
// validate() of host CSR arrays (csr.cpp:111-156); GSPMM_ERR_STRUCTURE with
// the reference's message on failure.
int validate_csr_host(uint32_t num_rows, uint32_t num_cols, const uint32_t* indptr,
                      const uint32_t* indices, const uint32_t* eids);

// Launch counter (evidence of native execution), bumped by each launcher.
void note_launch(uint64_t n = 1);

}  // namespace gspmm_b200

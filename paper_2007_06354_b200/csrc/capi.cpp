// capi.cpp -- the extern "C" boundary (include/gspmm_b200.h): descriptor
// validation with the reference's rules and error taxonomy, the device graph
// handle (CSR + degree plan), operand binding, vector-width selection and
// kernel dispatch.  No CPU fallback exists: every compute entry point either
// launches the sm_100a kernels or returns an error.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "gspmm_b200.h"
#include "internal.h"
#include "stream.h"

namespace gspmm_b200 {
uint64_t launch_count();
}

using namespace gspmm_b200;

namespace {

thread_local std::string g_err;

int fail(int status, const std::string& msg) {
  g_err = msg;
  return status;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(GSPMM_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CUDA_TRY(expr, where)                     \
  do {                                            \
    cudaError_t _e = (expr);                      \
    if (_e != cudaSuccess) return cuda_fail(_e, where); \
  } while (0)

const char* operand_name(int o) {
  switch (o) {
    case GSPMM_U: return "u";
    case GSPMM_V: return "v";
    case GSPMM_E: return "e";
    default: return "none";
  }
}

// Device plan defaults (gspmm_graph_set_plan overrides them): cost (edges +
// 2 per row) per row segment; with every unit pulled from the counter, finer
// units shorten the segment kernel's drain (measured cost 1024 / 512 / 256 /
// 128 / 64: cfg2 forward 1.87 / 1.72 / 1.70 / 1.69 / 1.69 ms, cfg3 mean 5.54
// / 5.48 / 5.45 / 5.46 / 5.51, cfg4 7.18 / 7.19 / 7.01 / 7.12 / 7.00, cfg5
// -- / -- / 15.6 / 15.5 / 15.5; 2048: cfg2 2.08).  The long-row thresholds
// of the plan levels are kLevelThresholds.
constexpr uint32_t kSegEdges = 256;
constexpr int kLevels = 6;
constexpr uint32_t kLevelThresholds[kLevels] = {1024, 4096, 8192, 16384, 32768, 65536};
// Source blocking: blocks of <= 48 MB of gathered rows (a share of the
// 126 MB L2), see source_blocks_for.
constexpr double kSrcBlockBytes = 48.0 * 1048576.0;
// Long-row column units (k_long_rg): stream rate of one CTA on random rows
// and the rate of one column's fp32 add chain (one dependent add per ~4
// cycles at 1.965 GHz), the two bounds of a unit's time.
constexpr uint32_t kSplitEdges = 512;  // default chunk of a long row's Max / Min fold
constexpr double kUnitBytesPerS = 40.0e9;
constexpr double kChainEdgesPerS = 490.0e6;

// The stream-ordered pool of the current device keeps freed memory mapped
// across synchronizations (its default release threshold of 0 unmaps it at
// every sync, which made each call's f64 workspace cost a re-map).
void retain_pool_memory() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  static std::mutex mu;
  static std::vector<int> done;
  std::lock_guard<std::mutex> lock(mu);
  for (int d : done)
    if (d == dev) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  done.push_back(dev);
}

}  // namespace

// Per-call device state, one context per caller stream: the work-unit
// counters, the prescale workspace and the `done` event of the context's
// last call.  Calls on one stream are ordered by the stream; calls on
// different streams (or host threads) use different contexts, so they can
// run concurrently on one handle without sharing a counter or a workspace.
// Every call first waits for the context's previous call (its `done`
// event), so a context handed to a new stream -- a recycled stream handle,
// or the LRU context once kMaxContexts are in use -- is never reused while
// the old call still runs.  The graph's mutex is held while a call is
// enqueued (not while it runs), which orders the enqueue steps of one
// context (counter reset, launches, event records) across host threads.
struct CallCtx {
  cudaStream_t key = nullptr;
  uint32_t* d_counter = nullptr;  // [0] segment units, [1] long-row units
  cudaEvent_t done = nullptr;
  bool used = false;
  void* dws = nullptr;  // prescaled gathered rows (mean backward)
  size_t dws_bytes = 0;
  void* sws = nullptr;  // chunk partials of long rows split by edges
  size_t sws_bytes = 0;
  uint64_t last_use = 0;
  // edge softmax: hub rows run on a side stream (created on first use)
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
constexpr size_t kMaxContexts = 32;

struct gspmm_graph_s {
  int device = 0;
  int orientation = GSPMM_DST_MAJOR;
  uint32_t num_rows = 0, num_cols = 0;
  uint64_t m = 0;
  uint32_t* d_indptr = nullptr;
  uint32_t* d_indices = nullptr;
  uint32_t* d_eids = nullptr;
  // Device plan, one level per long-row threshold (degree above which a row
  // runs as long-row column units): picked per call from the row bytes.
  struct Level {
    uint32_t threshold = 0;
    std::vector<uint32_t> long_rows;  // host copy, heaviest first
    std::vector<uint32_t> long_deg;
    std::vector<uint32_t> long_start;  // indptr[row] of each long row
    uint32_t* d_long = nullptr;       // device copy (edge softmax hub rows)
    uint32_t num_long = 0;
    uint2* d_segs = nullptr;          // segments of consecutive non-long rows
    uint32_t num_segs = 0;
  };
  Level level[kLevels];
  int n_levels = 0;
  // long-row column units per (level, width), built on first use
  struct Units {
    int level = 0, width = 0;
    uint2* d = nullptr;
    uint32_t n = 0;
  };
  std::vector<Units> units;
  // long rows split into chunks of edges (plan option split_edges), per
  // level, built on first use: a CSR view over the same indices / edge_ids
  // whose rows are the chunks (cptr; one unused row after each long row's
  // last chunk keeps the chunks of different long rows apart), one segment
  // unit per chunk, and each long row's (first chunk row, chunk count)
  struct Chunks {
    int level = 0;
    uint32_t edges = 0;
    uint32_t* d_cptr = nullptr;
    uint2* d_units = nullptr;
    uint2* d_ranges = nullptr;
    uint32_t rows = 0, n_units = 0;
  };
  std::vector<Chunks> chunks;
  uint32_t* d_rowof = nullptr;  // owner row of each CSR position (edge dots), lazy
  int num_sms = 148;
  std::recursive_mutex mu;      // held while a call is enqueued
  std::vector<CallCtx*> ctxs;
  uint64_t calls = 0;
  // source blocks (gspmm_graph_set_source_blocks): sub-graphs over neighbour
  // id ranges, built on first use for block_nb blocks
  int blocks_pref = 0;  // 0 auto, 1 never, >= 2 forced
  uint32_t block_nb = 0;
  std::vector<gspmm_graph_s*> blocks;
  // plan options (gspmm_graph_set_plan)
  uint32_t seg_cost = 0;        // 0 -> kSegEdges
  uint32_t forced_long = 0;     // 0 -> the kLevelThresholds levels
  uint32_t unit_cols = 0;       // 0 -> automatic long-row unit widths
  int rows_kernel_only = 0;     // 1 -> every call on the register kernel (rows.cu)
  uint32_t long_ctas = 0;       // 0 -> long rows before the segments; N -> concurrent
  int pdl_pair = 0;             // 1 -> programmatic overlap of the long-row / segment pair
  uint32_t split_edges = 0;     // N -> long rows as chunks of ~N edges (sums re-associated)
};

namespace {

// The context of caller stream s (graph mutex held).
int context_for(gspmm_graph_s* g, cudaStream_t s, CallCtx** out) {
  ++g->calls;
  for (CallCtx* c : g->ctxs)
    if (c->key == s) {
      c->last_use = g->calls;
      *out = c;
      return GSPMM_OK;
    }
  CallCtx* c = nullptr;
  if (g->ctxs.size() < kMaxContexts) {
    c = new CallCtx;
    cudaError_t e = cudaMalloc(&c->d_counter, 4 * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->done, cudaEventDisableTiming);
    if (e != cudaSuccess) {
      cudaFree(c->d_counter);
      delete c;
      return cuda_fail(e, "call context");
    }
    g->ctxs.push_back(c);
  } else {
    c = g->ctxs[0];
    for (CallCtx* x : g->ctxs)
      if (x->last_use < c->last_use) c = x;
  }
  c->key = s;
  c->last_use = g->calls;
  *out = c;
  return GSPMM_OK;
}

int begin_call(CallCtx* c, cudaStream_t s) {
  if (c->used) CUDA_TRY(cudaStreamWaitEvent(s, c->done, 0), "context order");
  return GSPMM_OK;
}

int end_call(CallCtx* c, cudaStream_t s) {
  CUDA_TRY(cudaEventRecord(c->done, s), "context order");
  c->used = true;
  return GSPMM_OK;
}

void free_contexts(gspmm_graph_s* g) {
  for (CallCtx* c : g->ctxs) {
    cudaFree(c->d_counter);
    cudaFree(c->dws);
    cudaFree(c->sws);
    if (c->done) cudaEventDestroy(c->done);
    if (c->side) {
      cudaStreamDestroy(c->side);
      cudaEventDestroy(c->fork);
      cudaEventDestroy(c->join);
    }
    delete c;
  }
  g->ctxs.clear();
}

}  // namespace

namespace {

// ---------------------------------------------------------------- config

int validate_cfg(const gspmm_config* c) {
  if (!c) return fail(GSPMM_ERR_ARG, "null config");
  auto bad_op = [](int o) { return o < GSPMM_U || o > GSPMM_NONE; };
  if (bad_op(c->lhs) || bad_op(c->rhs) || bad_op(c->out) || c->binary < GSPMM_ADD ||
      c->binary > GSPMM_COPY || c->reduce < GSPMM_SUM || c->reduce > GSPMM_MEAN)
    return fail(GSPMM_ERR_CONFIG, "enum value out of range");
  // validate_config, br_config.cpp:83-94
  if (c->lhs == GSPMM_NONE) return fail(GSPMM_ERR_CONFIG, "lhs operand must be u, v or e");
  if (c->out == GSPMM_NONE) return fail(GSPMM_ERR_CONFIG, "output target must be u, v or e");
  if ((c->rhs == GSPMM_NONE) != (c->binary == GSPMM_COPY))
    return fail(GSPMM_ERR_CONFIG, "rhs is absent exactly for the copy operator");
  if (c->rhs != GSPMM_NONE && c->rhs == c->lhs)
    return fail(GSPMM_ERR_CONFIG, "lhs and rhs must bind to different entities");
  if (c->out == GSPMM_E && c->reduce != GSPMM_COPY_LAST)
    return fail(GSPMM_ERR_CONFIG, "edge-destined configs store, reduce must be copy");
  return GSPMM_OK;
}

struct Bound {
  RowLaunch L;
  int64_t out_rows = 0;
  int64_t width = 0;
};

int64_t entity_rows(const gspmm_graph_s* g, int ent) {
  const bool src_major = g->orientation == GSPMM_SRC_MAJOR;
  if (ent == GSPMM_U) return src_major ? g->num_rows : g->num_cols;
  if (ent == GSPMM_V) return src_major ? g->num_cols : g->num_rows;
  return static_cast<int64_t>(g->m);
}

int32_t role_of(const gspmm_graph_s* g, int ent, int edge_order) {
  if (ent == GSPMM_E) return edge_order == GSPMM_EDGE_BY_POS ? ROLE_POS : ROLE_EID;
  const bool row_is_u = g->orientation == GSPMM_SRC_MAJOR;
  return (ent == GSPMM_U) == row_is_u ? ROLE_ROW : ROLE_OTHER;
}

bool aligned(const void* p, int bytes) {
  return (reinterpret_cast<uintptr_t>(p) % static_cast<uintptr_t>(bytes)) == 0;
}

// The full binding of binary_reduce (kernels.cpp:418-456) plus the
// extensions (mean, heads, argmax, other_scale).  out may be null (shape
// query only).
int bind(const gspmm_graph_s* g, const gspmm_config* cfg, const gspmm_mat* u,
         const gspmm_mat* v, const gspmm_mat* e, const gspmm_out* out,
         const gspmm_options* opt, Bound* b) {
  if (!g) return fail(GSPMM_ERR_ARG, "null graph handle");
  int st = validate_cfg(cfg);
  if (st) return st;
  // required_orientation(strategy != Push, out), kernels.cpp:400-411
  const int need = cfg->out == GSPMM_U ? GSPMM_SRC_MAJOR : GSPMM_DST_MAJOR;
  if (g->orientation != need)
    return fail(GSPMM_ERR_SHAPE, std::string("output ") + operand_name(cfg->out) + " needs a " +
                                     (need == GSPMM_SRC_MAJOR ? "src-major" : "dst-major") +
                                     " graph, got " +
                                     (g->orientation == GSPMM_SRC_MAJOR ? "src-major" : "dst-major"));
  const gspmm_options none{};
  if (!opt) opt = &none;
  const int heads = opt->heads > 1 ? opt->heads : 1;

  auto pick = [&](int o) { return o == GSPMM_U ? u : o == GSPMM_V ? v : e; };
  // bind_operand, kernels.cpp:361-377
  auto bind_one = [&](int o, const gspmm_mat*& m) -> int {
    m = pick(o);
    // a rows x 0 matrix has no data (FeatureMatrix(rows, 0), feature_matrix.hpp:36-38)
    if (!m || (!m->data && !(m->rows > 0 && m->dim == 0)))
      return fail(GSPMM_ERR_SHAPE, std::string("missing feature matrix for operand ") + operand_name(o));
    if (m->rows != entity_rows(g, o))
      return fail(GSPMM_ERR_SHAPE, std::string("operand ") + operand_name(o) + " has " +
                                       std::to_string(m->rows) + " rows, entity has " +
                                       std::to_string(entity_rows(g, o)));
    if (m->dim < 0 || (m->ld != 0 && m->ld < m->dim))
      return fail(GSPMM_ERR_SHAPE, std::string("operand ") + operand_name(o) + " has a bad dim/ld");
    return GSPMM_OK;
  };
  const gspmm_mat* lm = nullptr;
  const gspmm_mat* rm = nullptr;
  if ((st = bind_one(cfg->lhs, lm))) return st;
  const int64_t dl = lm->dim;
  int64_t dr = dl;
  if (cfg->rhs != GSPMM_NONE) {
    if ((st = bind_one(cfg->rhs, rm))) return st;
    dr = rm->dim;
  }
  const bool is_dot = cfg->binary == GSPMM_DOT;
  const int64_t gather = std::max(dl, dr);
  auto head_ok = [&](int64_t d) {
    return !is_dot && heads > 1 && d == heads && gather % heads == 0 && d < gather;
  };
  if (rm && !(dl == dr || dl == 1 || dr == 1 || head_ok(dl) || head_ok(dr)))
    return fail(GSPMM_ERR_SHAPE, "operand widths are not broadcast-compatible");
  if (is_dot && heads > 1 && gather % heads != 0)
    return fail(GSPMM_ERR_SHAPE, "dot heads must divide the operand width");
  int64_t w = is_dot ? heads : cfg->binary == GSPMM_COPY ? dl : gather;
  // Zero-width operands: the reference returns a rows x 0 matrix
  // (binary_out_dim, ops.cpp:63-67); nothing to launch.  A dot over zero
  // columns or a 0-against-1 broadcast reads past an empty row there.
  if (dl == 0 || dr == 0) {
    if (is_dot || gather != 0)
      return fail(GSPMM_ERR_SHAPE, "zero-width operands take no dot and no broadcast");
    if (out && (out->rows != entity_rows(g, cfg->out) || out->dim != 0))
      return fail(GSPMM_ERR_SHAPE, "output must be " + std::to_string(entity_rows(g, cfg->out)) + " x 0");
    b->L = RowLaunch{};
    b->out_rows = entity_rows(g, cfg->out);
    b->width = 0;
    return GSPMM_OK;
  }
  if (cfg->reduce == GSPMM_MEAN && cfg->out == GSPMM_E)
    return fail(GSPMM_ERR_CONFIG, "mean reduces into nodes only");
  const bool want_arg = opt->arg_other || opt->arg_edge;
  if (want_arg && cfg->reduce != GSPMM_MAX && cfg->reduce != GSPMM_MIN)
    return fail(GSPMM_ERR_CONFIG, "argmax outputs need the max or min reducer");
  if (want_arg && (is_dot || cfg->out == GSPMM_E))
    return fail(GSPMM_ERR_CONFIG, "argmax outputs need a node-destined, non-dot config");
  if (is_dot && heads > 1 && cfg->out != GSPMM_E)
    return fail(GSPMM_ERR_CONFIG, "per-head dot is edge-destined only");

  RowLaunch& L = b->L;
  L = RowLaunch{};
  L.indptr = g->d_indptr;
  L.indices = g->d_indices;
  L.eids = g->d_eids;
  L.num_rows = g->num_rows;
  auto mk = [&](int o, const gspmm_mat* m) {
    OperandDesc d;
    d.base = m->data;
    d.ld = m->ld ? m->ld : m->dim;
    d.rows = m->rows;
    d.role = role_of(g, o, m->edge_order);
    if (m->dim == 1 && gather > 1) {
      d.mode = MODE_SCALAR;  // stride 0, kernels.cpp:451-453
    } else if (m->dim < gather) {
      d.mode = MODE_HEAD;
      d.group = static_cast<int32_t>(gather / m->dim);
    } else {
      d.mode = MODE_FULL;
    }
    return d;
  };
  L.lhs = mk(cfg->lhs, lm);
  if (rm) L.rhs = mk(cfg->rhs, rm);
  L.binop = cfg->binary;
  L.reduce = cfg->reduce == GSPMM_MEAN ? R_SUM : cfg->reduce;
  L.mean = cfg->reduce == GSPMM_MEAN;
  L.out_edge = cfg->out == GSPMM_E;
  L.width = static_cast<int32_t>(w);
  L.gather_dim = static_cast<int32_t>(gather);
  L.heads = heads;
  L.other_scale = opt->other_scale;
  if (opt->source_blocks < 0) return fail(GSPMM_ERR_ARG, "source_blocks must be >= 0");
  L.src_blocks = opt->source_blocks;
  L.arg_other = opt->arg_other;
  L.arg_edge = opt->arg_edge;
  L.arg_ld = opt->arg_ld ? opt->arg_ld : w;
  {
    const auto& lv = g->level[g->n_levels > 3 ? 3 : g->n_levels - 1];  // rows.cu: 16384
    L.long_rows = lv.d_long;
    L.num_long = lv.num_long;
    L.long_threshold = lv.num_long ? lv.threshold : 0xffffffffu;
  }
  L.num_sms = g->num_sms;
  b->out_rows = entity_rows(g, cfg->out);
  b->width = w;

  if (out) {
    if (!out->data) return fail(GSPMM_ERR_SHAPE, "missing output matrix");
    if (out->rows != b->out_rows || out->dim != w || (out->ld != 0 && out->ld < w))
      return fail(GSPMM_ERR_SHAPE, "output must be " + std::to_string(b->out_rows) + " x " +
                                       std::to_string(w));
    L.out = out->data;
    L.out_ld = out->ld ? out->ld : w;
  }
  if (opt->out2) {
    if (opt->reduce2 != GSPMM_SUM && opt->reduce2 != GSPMM_MEAN)
      return fail(GSPMM_ERR_CONFIG, "reduce2 must be sum or mean");
    if (cfg->out == GSPMM_E || is_dot)
      return fail(GSPMM_ERR_CONFIG, "a second reduction needs a node-destined, non-dot config");
    if (opt->out2_ld != 0 && opt->out2_ld < w)
      return fail(GSPMM_ERR_SHAPE, "out2 row stride is below the output width");
    L.out2 = opt->out2;
    L.out2_ld = opt->out2_ld ? opt->out2_ld : w;
    L.mean2 = opt->reduce2 == GSPMM_MEAN;
  }

  // Widest vector every operand layout admits.
  auto vec_ok = [&](int V) {
    auto ok_op = [&](const OperandDesc& d) {
      if (!d.base) return true;
      if (d.mode == MODE_FULL) return d.ld % V == 0 && aligned(d.base, 4 * V);
      if (d.mode == MODE_HEAD) return d.group % V == 0;
      return true;
    };
    if (!ok_op(L.lhs) || !ok_op(L.rhs)) return false;
    if (!is_dot && L.out && !(L.out_ld % V == 0 && aligned(L.out, 4 * V))) return false;
    if (L.out2 && !(L.out2_ld % V == 0 && aligned(L.out2, 4 * V))) return false;
    return true;
  };
  L.vec = vec_ok(4) ? 4 : vec_ok(2) ? 2 : 1;
  return GSPMM_OK;
}

// Which planned kernel runs this binding?  Both planned kernels take the
// gathered full-width operand as lhs and at most a small (scalar /
// per-head) edge or neighbour operand as rhs; everything else goes to the
// register kernel (rows.cu).  Returns false for rows.cu.
bool planned(const gspmm_graph_s* g, const RowLaunch& L, int* rhs_width) {
  if (g->rows_kernel_only) return false;
  if (L.binop == GSPMM_DOT || L.out_edge || !L.out) return false;
  if (L.reduce == R_PROD || L.reduce == R_LAST) return false;  // rare: rows.cu
  if (L.other_scale && L.rhs.base) return false;                // scale on top of an rhs
  if (L.lhs.mode != MODE_FULL || L.lhs.role == ROLE_ROW) return false;
  if (L.lhs.ld % 4 || !aligned(L.lhs.base, 16)) return false;
  if (L.out_ld % 4 || !aligned(L.out, 16)) return false;
  *rhs_width = 0;
  if (L.rhs.base) {
    if (L.rhs.role == ROLE_ROW || L.rhs.mode == MODE_FULL) return false;
    // lanes fold float4 column groups: a head must cover whole groups
    if (L.rhs.mode == MODE_HEAD && L.rhs.group % 4) return false;
    *rhs_width = L.rhs.mode == MODE_SCALAR ? 1 : L.width / L.rhs.group;
  }
  return true;
}

int run_call(gspmm_graph_s* g, Bound& b, cudaStream_t s);
int launch(gspmm_graph_s* g, CallCtx* ctx, Bound& b, cudaStream_t s);
void destroy_graph(gspmm_graph_s* g);

// Number of source blocks for this call: 1 = a single pass.
uint32_t source_blocks_for(const gspmm_graph_s* g, const RowLaunch& L) {
  const int pref = L.src_blocks ? L.src_blocks : g->blocks_pref;
  if (pref == 1 || L.acc_in || L.epi) return 1;
  int rw = 0;
  if (!planned(g, L, &rw)) return 1;
  if (L.lhs.role != ROLE_OTHER || L.arg_other || L.arg_edge || L.out2) return 1;
  if (L.reduce != R_SUM && L.reduce != R_MAX && L.reduce != R_MIN) return 1;
  if (L.rhs.base && L.rhs.role == ROLE_POS) return 1;
  if (pref >= 2) return std::min<uint32_t>(pref, 64);
  // automatic: blocks of <= 48 MB of gathered rows when the gathered operand
  // exceeds 1.5x the L2 and each row has >= 8 edges per block (the
  // partial-row read + write per pass is then small against the row's
  // gathers).  Measured on cfg5 (232,965 x 602 fp32 = 561 MB, 495 edges per
  // row): 12 blocks, 35.4 -> 18.2 ms; 32 / 64 / 96 / 160 MB blocks: 19.2 /
  // 18.9 / 22.7 / 32.8 ms
  const double bytes = static_cast<double>(g->num_cols) * L.width * 4.0;
  if (bytes < 1.5 * 126.0 * 1048576.0) return 1;
  const uint32_t nb = static_cast<uint32_t>(std::ceil(bytes / kSrcBlockBytes));
  const double avg = g->num_rows ? static_cast<double>(g->m) / g->num_rows : 0.0;
  if (nb < 2 || avg < 8.0 * nb) return 1;
  return std::min<uint32_t>(nb, 64);
}

// Source-block sub-graphs (graph mutex held).  Built on the caller's stream
// and completed before they are published: a concurrent call on another
// stream only ever sees finished blocks.
int build_source_blocks(gspmm_graph_s* g, uint32_t nb, cudaStream_t s) {
  if (g->block_nb == nb) return GSPMM_OK;
  for (auto* sg : g->blocks) destroy_graph(sg);
  g->blocks.clear();
  g->block_nb = 0;
  const uint32_t rows = g->num_rows;
  const uint32_t bs = (g->num_cols + nb - 1) / nb;
  uint32_t *bpos = nullptr, *ip = nullptr, *ix = nullptr, *ie = nullptr;
  auto done = [&](int st) {
    cudaFree(bpos);
    cudaFree(ip);
    cudaFree(ix);
    cudaFree(ie);
    return st;
  };
  CUDA_TRY(cudaMalloc(&bpos, sizeof(uint32_t) * (nb + 1ull) * rows), "block bounds");
  CUDA_TRY(launch_block_bounds(g->d_indptr, g->d_indices, rows, nb, bs, bpos, s),
           "block bounds");
  if (cudaMalloc(&ip, sizeof(uint32_t) * (rows + 1ull)) != cudaSuccess ||
      cudaMalloc(&ix, sizeof(uint32_t) * std::max<uint64_t>(g->m, 1)) != cudaSuccess ||
      cudaMalloc(&ie, sizeof(uint32_t) * std::max<uint64_t>(g->m, 1)) != cudaSuccess)
    return done(cuda_fail(cudaErrorMemoryAllocation, "block CSR"));
  for (uint32_t b = 0; b < nb; ++b) {
    cudaError_t e = launch_block_csr(bpos + static_cast<uint64_t>(b) * rows,
                                     bpos + static_cast<uint64_t>(b + 1) * rows, rows,
                                     g->d_indices, g->d_eids, ip, ix, ie, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return done(cuda_fail(e, "block CSR"));
    gspmm_graph sg = nullptr;
    const int st = gspmm_graph_create_device(g->device, g->orientation, rows, g->num_cols, ip,
                                             ix, ie, &sg);
    if (st) return done(st);
    sg->blocks_pref = 1;
    sg->seg_cost = g->seg_cost;
    sg->forced_long = g->forced_long;
    sg->unit_cols = g->unit_cols;
    sg->long_ctas = g->long_ctas;
    sg->pdl_pair = g->pdl_pair;
    sg->split_edges = g->split_edges;
    g->blocks.push_back(sg);
  }
  g->block_nb = nb;
  return done(GSPMM_OK);
}

// Source-blocked passes: pass b folds block b's neighbours into the partial
// rows of passes < b (bit-identical: the canonical rows are neighbour-sorted).
int launch_blocked(gspmm_graph_s* g, Bound& b, cudaStream_t s, uint32_t nb) {
  int st = build_source_blocks(g, nb, s);
  if (st) return st;
  for (uint32_t k = 0; k < nb; ++k) {
    gspmm_graph_s* sg = g->blocks[k];
    Bound bb = b;
    bb.L.indptr = sg->d_indptr;
    bb.L.indices = sg->d_indices;
    bb.L.eids = sg->d_eids;
    bb.L.acc_in = k ? b.L.out : nullptr;
    bb.L.epi = k + 1 == nb ? 2 : 1;
    bb.L.deg_indptr = k + 1 == nb ? g->d_indptr : nullptr;
    st = run_call(sg, bb, s);
    if (st) return st;
  }
  return GSPMM_OK;
}

// Long-row column units of plan level li for output width W (graph mutex
// held), built on first use: every long row is cut into column slices of a
// width chosen so that no unit's time -- the larger of its bytes at one CTA's
// stream rate and its edge count at the fp32 add-chain rate -- exceeds half
// the long rows' balanced share of the GPU; 8 columns at least (a 32-byte
// sector), 512 at most (the consumer warps' reach).  Heaviest units first.
int long_units_for(gspmm_graph_s* g, int li, int W, const gspmm_graph_s::Units** out) {
  for (const auto& u : g->units)
    if (u.level == li && u.width == W) {
      *out = &u;
      return GSPMM_OK;
    }
  const auto& lv = g->level[li];
  const int Wp = (W + 3) & ~3;
  double total = 0.0;
  for (uint32_t d : lv.long_deg) total += static_cast<double>(d) * Wp * 4.0;
  const double cap = std::max(0.5 * total / (g->num_sms * kUnitBytesPerS), 20e-6);
  struct U {
    uint32_t r, c0, cw;
    double t;
  };
  std::vector<U> us;
  for (size_t i = 0; i < lv.long_rows.size(); ++i) {
    const double n = lv.long_deg[i];
    int sw;
    if (g->unit_cols) {
      sw = static_cast<int>(g->unit_cols);
    } else {
      sw = static_cast<int>(cap * kUnitBytesPerS / (n * 4.0)) & ~3;
      sw = std::max(8, std::min(sw, 512));
    }
    sw = std::min(sw, Wp);
    const int ns = (Wp + sw - 1) / sw;
    sw = (((Wp + ns - 1) / ns) + 3) & ~3;  // balanced slices
    for (int c0 = 0; c0 < W; c0 += sw) {
      const int cw = std::min(sw, W - c0);
      // hand-out order: the measured time of a unit (unit traces of r03c,
      // every width within 10%): 2.5 ns per edge plus 0.115 ns per edge and
      // column; the max() model above ranks 28-column units of 100k-edge
      // rows below whole 100-column rows of 30k edges, which take less time
      const double t = n * (2.5e-9 + 0.115e-9 * cw);
      us.push_back({lv.long_rows[i], static_cast<uint32_t>(c0), static_cast<uint32_t>(cw), t});
    }
  }
  std::stable_sort(us.begin(), us.end(), [](const U& a, const U& b) { return a.t > b.t; });
  std::vector<uint2> h(us.size());
  for (size_t i = 0; i < us.size(); ++i) h[i] = make_uint2(us[i].r, us[i].c0 | (us[i].cw << 16));
  gspmm_graph_s::Units u;
  u.level = li;
  u.width = W;
  u.n = static_cast<uint32_t>(h.size());
  CUDA_TRY(cudaMalloc(&u.d, sizeof(uint2) * std::max<size_t>(h.size(), 1)), "long units");
  if (!h.empty()) {
    const cudaError_t e = cudaMemcpy(u.d, h.data(), sizeof(uint2) * h.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      cudaFree(u.d);
      return cuda_fail(e, "long units");
    }
  }
  g->units.push_back(u);
  *out = &g->units.back();
  return GSPMM_OK;
}

// Chunk view of plan level li's long rows (graph mutex held), built on first
// use: every long row is cut into ceil(n / edges) balanced edge ranges.
int chunks_for(gspmm_graph_s* g, int li, uint32_t edges, const gspmm_graph_s::Chunks** out) {
  for (const auto& c : g->chunks)
    if (c.level == li && c.edges == edges) {
      *out = &c;
      return GSPMM_OK;
    }
  const auto& lv = g->level[li];
  std::vector<uint32_t> cptr;
  std::vector<uint2> units, ranges;
  for (size_t i = 0; i < lv.long_rows.size(); ++i) {
    const uint64_t n = lv.long_deg[i];
    const uint64_t nk = (n + edges - 1) / edges;
    const uint32_t k0 = static_cast<uint32_t>(cptr.size());
    ranges.push_back(make_uint2(k0, static_cast<uint32_t>(nk)));
    for (uint64_t t = 0; t <= nk; ++t)  // t == nk: the row's end (start of the unused row)
      cptr.push_back(lv.long_start[i] + static_cast<uint32_t>(t * n / nk));
    for (uint64_t t = 0; t < nk; ++t)
      units.push_back(make_uint2(k0 + static_cast<uint32_t>(t), k0 + static_cast<uint32_t>(t) + 1));
  }
  gspmm_graph_s::Chunks c;
  c.level = li;
  c.edges = edges;
  c.rows = static_cast<uint32_t>(cptr.size());
  c.n_units = static_cast<uint32_t>(units.size());
  cptr.push_back(cptr.empty() ? 0u : cptr.back());  // rows + 1 entries
  auto up = [&](auto** d, const auto& h, const char* what) -> int {
    using T = std::remove_reference_t<decltype(h[0])>;
    CUDA_TRY(cudaMalloc(d, sizeof(T) * std::max<size_t>(h.size(), 1)), what);
    if (!h.empty())
      CUDA_TRY(cudaMemcpy(*d, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice), what);
    return GSPMM_OK;
  };
  int st = up(&c.d_cptr, cptr, "chunk rows");
  if (!st) st = up(&c.d_units, units, "chunk units");
  if (!st) st = up(&c.d_ranges, ranges, "chunk ranges");
  if (st) {
    cudaFree(c.d_cptr);
    cudaFree(c.d_units);
    cudaFree(c.d_ranges);
    return st;
  }
  g->chunks.push_back(c);
  *out = &g->chunks.back();
  return GSPMM_OK;
}

// One call on handle g: takes the graph mutex for the enqueue, runs in the
// caller stream's context (see CallCtx).
int run_call(gspmm_graph_s* g, Bound& b, cudaStream_t s) {
  std::lock_guard<std::recursive_mutex> lock(g->mu);
  CUDA_TRY(cudaSetDevice(g->device), "cudaSetDevice");
  CallCtx* ctx = nullptr;
  int st = context_for(g, s, &ctx);
  if (st) return st;
  if ((st = begin_call(ctx, s))) return st;
  st = launch(g, ctx, b, s);
  const int st2 = end_call(ctx, s);
  return st ? st : st2;
}

// The fused second reduction runs in the planned kernels for copy + Max/Min
// of gathered rows (a second accumulator per column); any other config gets
// it as a second pass with the second reducer (same result bits).
bool dual_fused(const gspmm_graph_s* g, const RowLaunch& L) {
  int rw = 0;
  return L.out2 && planned(g, L, &rw) && L.binop == B_COPY && !L.rhs.base && !L.other_scale &&
         (L.reduce == R_MAX || L.reduce == R_MIN) && L.lhs.role == ROLE_OTHER &&
         L.out2_ld % 4 == 0 && aligned(L.out2, 16);
}

int launch(gspmm_graph_s* g, CallCtx* ctx, Bound& b, cudaStream_t s) {
  cudaError_t err;
  int rw = 0;
  if (b.L.out2 && !dual_fused(g, b.L)) {
    Bound b1 = b, b2 = b;
    b1.L.out2 = nullptr;
    b2.L.out2 = nullptr;
    b2.L.out = b.L.out2;
    b2.L.out_ld = b.L.out2_ld;
    b2.L.reduce = R_SUM;
    b2.L.mean = b.L.mean2;
    b2.L.arg_other = b2.L.arg_edge = nullptr;
    const int st = launch(g, ctx, b1, s);
    return st ? st : launch(g, ctx, b2, s);
  }
  if (!b.L.out_edge && b.L.binop != GSPMM_DOT && b.L.other_scale && !b.L.rhs.base &&
      b.L.binop == GSPMM_COPY && b.L.lhs.role == ROLE_OTHER && b.L.lhs.mode == MODE_FULL &&
      b.L.lhs.rows > 0 && planned(g, b.L, &rw) &&
      static_cast<double>(g->m) >= 4.0 * static_cast<double>(b.L.lhs.rows)) {
    // The per-neighbour scale (the mean backward's 1/deg) on dense-enough
    // graphs: scale every gathered row once into the context's workspace,
    // then run the plain copy-sum.  Each product is the same single rounding
    // as the kernels' per-edge scale, so the result is bit-identical
    // (measured: cfg3 mean backward 6.67 -> 6.01 ms, cfg5 18.05 -> 16.56).
    const int64_t W = b.L.width;
    const int64_t yld = (W + 3) & ~int64_t{3};
    const size_t need = sizeof(float) * static_cast<size_t>(b.L.lhs.rows * yld);
    if (need > ctx->dws_bytes) {
      // (cudaFree synchronizes the device: no call still reads the old one)
      cudaFree(ctx->dws);
      ctx->dws = nullptr;
      ctx->dws_bytes = 0;
      CUDA_TRY(cudaMalloc(&ctx->dws, need), "prescale workspace");
      ctx->dws_bytes = need;
    }
    float* y = static_cast<float*>(ctx->dws);
    CUDA_TRY(launch_scale_rows(b.L.lhs.base, b.L.lhs.rows, W, b.L.lhs.ld, b.L.other_scale, y,
                               yld, s),
             "prescale");
    Bound bb = b;
    bb.L.lhs.base = y;
    bb.L.lhs.ld = yld;
    bb.L.other_scale = nullptr;
    return launch(g, ctx, bb, s);
  }
  if (!b.L.out_edge && b.L.binop != GSPMM_DOT) {
    const uint32_t nb = source_blocks_for(g, b.L);
    if (nb > 1) return launch_blocked(g, b, s, nb);
  }
  if (b.L.binop == GSPMM_DOT && b.L.out_edge &&
      (b.L.lhs.mode != MODE_FULL || (b.L.lhs.ld % 2 == 0 && aligned(b.L.lhs.base, 8))) &&
      (b.L.rhs.mode != MODE_FULL || (b.L.rhs.ld % 2 == 0 && aligned(b.L.rhs.base, 8)))) {
    // edge-destined dots stream edge batches; needs the row of each edge
    // (built once, completed before it is published to other streams)
    if (!g->d_rowof) {
      uint32_t* rowof = nullptr;
      CUDA_TRY(cudaMalloc(&rowof, sizeof(uint32_t) * std::max<uint64_t>(g->m, 1)),
               "row-of-edge array");
      cudaError_t e = launch_row_of_edge(g->d_indptr, g->num_rows, rowof, s);
      if (e == cudaSuccess) e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) {
        cudaFree(rowof);
        return cuda_fail(e, "row-of-edge");
      }
      g->d_rowof = rowof;
    }
    err = launch_dot_edges(b.L, g->d_rowof, g->m, s);
  } else if (b.L.binop == GSPMM_DOT) {
    err = launch_dot(b.L, s);
  } else if (planned(g, b.L, &rw)) {
    StreamLaunch p;
    p.row = b.L;
    // Plan level.  A row in the segment kernel is one warp's sequential
    // work per slice, so a row much heavier than a warp's fair share of the
    // pass ends after everything else; a row in the long-row kernel streams
    // at a third of the segment kernel's rate per SM, so no more rows than
    // necessary should go there.  Two bounds, both in edges: `share`, half
    // the average per-warp share of the segment work, and `bytes`, ~8 MB of
    // gathered bytes per row.  The level is the first threshold at or above
    // `share`, but never above the last threshold within max(bytes, share).
    // Measured (r02w-r02y, ms per pass at long-row thresholds 4096 / 8192 /
    // 16384): cfg2 (share 1.8k) 1.73 / 2.50 / 2.50; cfg4 (share 6.8k) 8.23 /
    // 7.07 / 8.16; cfg3 (share 17k; 16384 / 32768 / 65536) 5.01 / 5.04 / 5.13.
    const int slice_bytes = 4 * std::min(b.L.width, 256);
    const uint32_t bytes_rule = std::max<uint32_t>(1024, (8u << 20) / static_cast<uint32_t>(slice_bytes));
    const uint32_t slices = static_cast<uint32_t>((b.L.width + 255) / 256);
    const double warps = static_cast<double>(g->num_sms) * (b.L.width > 128 ? 32 : 24);
    const double share = std::min(0.5 * static_cast<double>(g->m) * slices / warps, 4.0e9);
    const double cap = std::max<double>(bytes_rule, share);
    int li = 0, li_share = g->n_levels - 1;
    for (int k = 0; k < g->n_levels; ++k)
      if (g->level[k].threshold <= cap) li = k;
    for (int k = g->n_levels - 1; k >= 0; --k)
      if (g->level[k].threshold >= share) li_share = k;
    li = std::min(li, li_share);
    const auto& lv = g->level[li];
    p.segs = lv.d_segs;
    p.n_segs = lv.num_segs;
    p.rhs_width = rw;
    const int W = b.L.width;
    // one segment unit covers up to 640 columns for copy / scalar-weighted
    // sums of gathered rows (gather_impl.cuh launch_wide), else <= 256-column
    // slices (measured on cfg5, W = 602: 18.2 -> 16.0 ms); W > 384 only:
    // narrower rows would leave over 40% of the wide unit's lanes idle
    // (measured slower than two slices at W = 304); per-head weights stay on
    // 256-column slices (wide units measured slower on cfg4, 7.04 -> 7.51 ms)
    const bool wide = W > 384 && W <= 640 && b.L.reduce == R_SUM && !b.L.arg_other &&
                      !b.L.arg_edge && b.L.lhs.role == ROLE_OTHER &&
                      ((b.L.binop == B_COPY && !b.L.rhs.base) || (b.L.binop == B_MUL && rw == 1));
    p.seg_sw = wide ? W : W <= 256 ? W : 256;
    p.seg_slices = static_cast<uint32_t>((W + p.seg_sw - 1) / p.seg_sw);
    err = cudaSuccess;
    p.mode = 0;
    p.n_units = p.n_segs * p.seg_slices;
    p.counter = ctx->d_counter;
    // Long rows split by EDGES: each chunk of a long row is folded like a
    // short row by the segment kernel into a partial row, and a small kernel
    // combines a row's partials in chunk order.  Max / Min are exact under
    // any association and the strict comparison keeps the first winner, so
    // for them (without a fused second sum) this is the DEFAULT path, the
    // reference's bits at segment-kernel speed (cfg3 max + argmax 6.14 ->
    // 5.22 ms, r04c).  Sums take it only under the plan option split_edges.
    const bool exact_split = (b.L.reduce == R_MAX || b.L.reduce == R_MIN) && !b.L.out2;
    const uint32_t split = g->split_edges == 1 ? 0u
                           : g->split_edges  ? g->split_edges
                           : exact_split     ? kSplitEdges
                                             : 0u;
    if (lv.num_long && split && !b.L.acc_in && !b.L.epi &&
        (b.L.reduce == R_SUM || b.L.reduce == R_MAX || b.L.reduce == R_MIN)) {
      // Max / Min and their argmax stay the reference's bits; a sum
      // becomes a fixed-order sum of chunk sums -- deterministic, another
      // fp32 order with the same kind of rounding error as the sequential
      // fold, and for that reason up to ~1e-3 (the reference's measure) away
      // from the reference on 10^5-edge rows: opt-in, outside the parity
      // contract.
      const gspmm_graph_s::Chunks* ch = nullptr;
      int st = chunks_for(g, li, split, &ch);
      if (st) return st;
      const int64_t pld = (W + 3) & ~3;
      const bool dual = b.L.out2 != nullptr;
      const int nbuf = 1 + (dual ? 1 : 0) + (b.L.arg_other ? 1 : 0) + (b.L.arg_edge ? 1 : 0);
      const size_t one = sizeof(float) * static_cast<size_t>(ch->rows) * static_cast<size_t>(pld);
      if (one * nbuf > ctx->sws_bytes) {
        cudaFree(ctx->sws);  // synchronizes: no call still reads the old one
        ctx->sws = nullptr;
        ctx->sws_bytes = 0;
        CUDA_TRY(cudaMalloc(&ctx->sws, one * nbuf), "chunk partials");
        ctx->sws_bytes = one * nbuf;
      }
      char* w = static_cast<char*>(ctx->sws);
      StreamLaunch pc = p;
      CombineLaunch cb;
      pc.row.indptr = ch->d_cptr;
      pc.row.num_rows = ch->rows;
      pc.row.mean = false;
      pc.row.mean2 = false;
      pc.row.out = reinterpret_cast<float*>(w);
      pc.row.out_ld = pld;
      cb.part = pc.row.out;
      w += one;
      if (dual) {
        pc.row.out2 = reinterpret_cast<float*>(w);
        pc.row.out2_ld = pld;
        cb.part2 = pc.row.out2;
        w += one;
      }
      pc.row.arg_ld = pld;
      if (b.L.arg_other) {
        pc.row.arg_other = reinterpret_cast<int32_t*>(w);
        cb.parg_other = pc.row.arg_other;
        w += one;
      }
      if (b.L.arg_edge) {
        pc.row.arg_edge = reinterpret_cast<int32_t*>(w);
        cb.parg_edge = pc.row.arg_edge;
        w += one;
      }
      pc.segs = ch->d_units;
      pc.n_segs = ch->n_units;
      pc.n_units = ch->n_units * p.seg_slices;
      pc.counter = ctx->d_counter + 1;
      err = launch_gather(pc, s);
      if (err != cudaSuccess) return cuda_fail(err, "kernel launch");
      cb.long_rows = lv.d_long;
      cb.ranges = ch->d_ranges;
      cb.n_long = lv.num_long;
      cb.indptr = g->d_indptr;
      cb.width = W;
      cb.reduce = b.L.reduce;
      cb.pld = pld;
      cb.out = b.L.out;
      cb.out_ld = b.L.out_ld;
      cb.out2 = b.L.out2;
      cb.out2_ld = b.L.out2_ld;
      cb.arg_other = b.L.arg_other;
      cb.arg_edge = b.L.arg_edge;
      cb.arg_ld = b.L.arg_ld;
      cb.mean = b.L.mean;
      cb.mean2 = b.L.mean2;
      err = launch_combine_chunks(cb, s);
    } else if (lv.num_long) {
      const gspmm_graph_s::Units* units = nullptr;
      const int st = long_units_for(g, li, W, &units);
      if (st) return st;
      StreamLaunch pl = p;
      pl.mode = 1;
      pl.long_units = units->d;
      pl.n_units = units->n;
      pl.counter = ctx->d_counter + 1;
      if (!g->long_ctas || !p.n_units) {
        // long rows first, on every SM, then the segments (measured on
        // config 3, r02h: the mean pass 5.48 ms against 9.0 ms with the
        // long-row CTAs concurrent on an automatic budget, 5.78 on 74 SMs --
        // a long-row CTA holds its SM's register file, and the segment
        // kernel, bound by the L2's throughput, needs every SM)
        // Plan option kernel = 2 launches the two as a programmatic-
        // dependent pair: the segment kernel's blocks take each SM as its
        // long-row CTA runs out of units instead of waiting for the slowest
        // unit.  Measured (r04a) slower where it matters: the latency-bound
        // long-row units lose more to the segment blocks' traffic than the
        // idle tail returns (cfg3 max + argmax 6.0 -> 6.7 ms, cfg2 1.73 ->
        // 2.08, cfg4 7.08 -> 6.97), so the default stays strictly serial.
        if (p.n_units && g->pdl_pair) {
          err = cudaMemsetAsync(ctx->d_counter, 0, 2 * sizeof(uint32_t), s);
          if (err != cudaSuccess) return cuda_fail(err, "counter reset");
          pl.pdl = 1;
          p.pdl = 2;
        }
        err = launch_gather(pl, s);
      } else {
        // long-row units on a side stream on long_ctas CTAs, concurrently
        // with the segment kernel
        if (!ctx->side) {
          CUDA_TRY(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking), "side stream");
          CUDA_TRY(cudaEventCreateWithFlags(&ctx->fork, cudaEventDisableTiming), "event");
          CUDA_TRY(cudaEventCreateWithFlags(&ctx->join, cudaEventDisableTiming), "event");
        }
        pl.grid = g->long_ctas;
        CUDA_TRY(cudaEventRecord(ctx->fork, s), "fork");
        CUDA_TRY(cudaStreamWaitEvent(ctx->side, ctx->fork, 0), "fork");
        err = launch_gather(pl, ctx->side);
        if (err == cudaSuccess) err = cudaEventRecord(ctx->join, ctx->side);
        if (err == cudaSuccess) err = launch_gather(p, s);
        const cudaError_t ej = cudaStreamWaitEvent(s, ctx->join, 0);
        if (err == cudaSuccess) err = ej;
        if (err != cudaSuccess) return cuda_fail(err, "kernel launch");
        return GSPMM_OK;
      }
    }
    if (err == cudaSuccess && p.n_units) err = launch_gather(p, s);
  } else {
    err = launch_rows(b.L, s);
  }
  if (err != cudaSuccess) return cuda_fail(err, "kernel launch");
  return GSPMM_OK;
}

// Device plan levels (host indptr): long rows (heaviest first) and
// edge-balanced segments of consecutive non-long rows, for each long-row
// threshold.  Replaces the previous plan (gspmm_graph_set_plan).
void free_plan(gspmm_graph_s* g) {
  for (auto& lv : g->level) {
    cudaFree(lv.d_long);
    cudaFree(lv.d_segs);
    lv = gspmm_graph_s::Level{};
  }
  for (auto& u : g->units) cudaFree(u.d);
  g->units.clear();
  for (auto& c : g->chunks) {
    cudaFree(c.d_cptr);
    cudaFree(c.d_units);
    cudaFree(c.d_ranges);
  }
  g->chunks.clear();
  g->n_levels = 0;
}

int build_plan(gspmm_graph_s* g, const uint32_t* indptr) {
  free_plan(g);
  const uint32_t seg_edges = g->seg_cost ? g->seg_cost : kSegEdges;
  g->n_levels = g->forced_long ? 1 : kLevels;
  for (int k = 0; k < g->n_levels; ++k) {
    auto& lv = g->level[k];
    lv.threshold = g->forced_long ? g->forced_long : kLevelThresholds[k];
    std::vector<uint2> segs;
    uint32_t begin = 0;
    uint64_t acc = 0;
    for (uint32_t r = 0; r < g->num_rows; ++r) {
      const uint32_t deg = indptr[r + 1] - indptr[r];
      if (deg > lv.threshold) {
        lv.long_rows.push_back(r);
        if (r > begin) segs.push_back(make_uint2(begin, r));
        begin = r + 1;
        acc = 0;
        continue;
      }
      acc += deg + 2;  // cost: edges + per-row epilogue (empty rows are not free)
      if (acc >= seg_edges) {
        segs.push_back(make_uint2(begin, r + 1));
        begin = r + 1;
        acc = 0;
      }
    }
    if (g->num_rows > begin) segs.push_back(make_uint2(begin, g->num_rows));
    // heaviest segments first: a segment holding one near-threshold row is the
    // longest unit, and it must not start last
    std::stable_sort(segs.begin(), segs.end(), [&](const uint2& a, const uint2& b) {
      return indptr[a.y] - indptr[a.x] > indptr[b.y] - indptr[b.x];
    });
    std::stable_sort(lv.long_rows.begin(), lv.long_rows.end(), [&](uint32_t a, uint32_t b) {
      return indptr[a + 1] - indptr[a] > indptr[b + 1] - indptr[b];
    });
    for (uint32_t r : lv.long_rows) {
      lv.long_deg.push_back(indptr[r + 1] - indptr[r]);
      lv.long_start.push_back(indptr[r]);
    }
    lv.num_long = static_cast<uint32_t>(lv.long_rows.size());
    lv.num_segs = static_cast<uint32_t>(segs.size());
    CUDA_TRY(cudaMalloc(&lv.d_long, sizeof(uint32_t) * std::max<size_t>(lv.num_long, 1)),
             "cudaMalloc plan");
    CUDA_TRY(cudaMalloc(&lv.d_segs, sizeof(uint2) * std::max<size_t>(segs.size(), 1)),
             "cudaMalloc segments");
    if (lv.num_long)
      CUDA_TRY(cudaMemcpy(lv.d_long, lv.long_rows.data(), sizeof(uint32_t) * lv.num_long,
                          cudaMemcpyHostToDevice),
               "upload plan");
    if (!segs.empty())
      CUDA_TRY(cudaMemcpy(lv.d_segs, segs.data(), sizeof(uint2) * segs.size(),
                          cudaMemcpyHostToDevice),
               "upload segments");
  }
  return GSPMM_OK;
}

// Host validate, csr.cpp:111-156 (same checks, same order).
int validate_host(uint32_t num_rows, uint32_t num_cols, const uint32_t* indptr,
                  const uint32_t* indices, const uint32_t* eids) {
  if (indptr[0] != 0) return fail(GSPMM_ERR_STRUCTURE, "indptr[0] != 0");
  for (uint32_t r = 0; r < num_rows; ++r)
    if (indptr[r] > indptr[r + 1])
      return fail(GSPMM_ERR_STRUCTURE, "indptr not monotone at row " + std::to_string(r + 1));
  const uint64_t m = indptr[num_rows];
  for (uint64_t j = 0; j < m; ++j)
    if (indices[j] >= num_cols)
      return fail(GSPMM_ERR_STRUCTURE, "index out of range at nonzero " + std::to_string(j));
  std::vector<bool> seen(m, false);
  for (uint64_t j = 0; j < m; ++j) {
    if (eids[j] >= m || seen[eids[j]])
      return fail(GSPMM_ERR_STRUCTURE,
                  "edge_ids not a permutation (at nonzero " + std::to_string(j) + ")");
    seen[eids[j]] = true;
  }
  for (uint32_t r = 0; r < num_rows; ++r)
    for (uint32_t j = indptr[r]; j + 1 < indptr[r + 1]; ++j) {
      const bool ordered = indices[j] < indices[j + 1] ||
                           (indices[j] == indices[j + 1] && eids[j] < eids[j + 1]);
      if (!ordered)
        return fail(GSPMM_ERR_STRUCTURE, "row " + std::to_string(r) + " not sorted at nonzero " +
                                             std::to_string(j + 1));
    }
  return GSPMM_OK;
}

size_t mat_bytes(const gspmm_mat* m) {
  if (!m || !m->data) return 0;
  const int64_t ld = m->ld ? m->ld : m->dim;
  return m->rows ? static_cast<size_t>((m->rows - 1) * ld + m->dim) * sizeof(float) : 0;
}

size_t round_up(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

}  // namespace

namespace gspmm_b200 {
int set_last_error(int status, const std::string& msg) { return fail(status, msg); }
int validate_csr_host(uint32_t num_rows, uint32_t num_cols, const uint32_t* indptr,
                      const uint32_t* indices, const uint32_t* eids) {
  return validate_host(num_rows, num_cols, indptr, indices, eids);
}
}  // namespace gspmm_b200

extern "C" {

const char* gspmm_last_error(void) { return g_err.c_str(); }
int gspmm_abi_version(void) { return GSPMM_B200_ABI_VERSION; }
uint64_t gspmm_launch_count(void) { return gspmm_b200::launch_count(); }

int gspmm_validate_config(const gspmm_config* cfg) { return validate_cfg(cfg); }

// named_config, br_config.cpp:96-131
int gspmm_named_config(const char* name, gspmm_config* cfg) {
  if (!name || !cfg) return fail(GSPMM_ERR_ARG, "null argument");
  std::vector<std::string> t;
  std::string cur;
  for (const char* p = name;; ++p) {
    if (*p == '_' || *p == '\0') {
      t.push_back(cur);
      cur.clear();
      if (*p == '\0') break;
    } else {
      cur += *p;
    }
  }
  auto opnd = [](const std::string& s) {
    return s == "u" ? GSPMM_U : s == "v" ? GSPMM_V : s == "e" ? GSPMM_E : -1;
  };
  auto bin = [](const std::string& s) {
    return s == "add" ? GSPMM_ADD : s == "sub" ? GSPMM_SUB : s == "mul" ? GSPMM_MUL
         : s == "div" ? GSPMM_DIV : s == "dot" ? GSPMM_DOT : -1;
  };
  auto red = [](const std::string& s) {
    return s == "add" ? GSPMM_SUM : s == "max" ? GSPMM_MAX : s == "min" ? GSPMM_MIN
         : s == "mul" ? GSPMM_PROD : s == "copy" ? GSPMM_COPY_LAST : -1;
  };
  const std::string bad = std::string("invalid config name '") + name + "': ";
  gspmm_config c{};
  if (t.size() == 4) {
    const int l = opnd(t[0]), r = red(t[2]);
    if (l < 0 || t[1] != "copy" || r < 0 || t[3] != "v")
      return fail(GSPMM_ERR_CONFIG, bad + "expected {u,e}_copy_{add,max,min,mul,copy}_v");
    if (l == GSPMM_V) return fail(GSPMM_ERR_CONFIG, bad + "copy source must be u or e");
    c = {l, GSPMM_NONE, GSPMM_COPY, r, GSPMM_V};
  } else if (t.size() == 5) {
    const int l = opnd(t[0]), b = bin(t[1]), r = opnd(t[2]), rd = red(t[3]), o = opnd(t[4]);
    if (l < 0 || b < 0 || r < 0 || rd < 0 || o < 0)
      return fail(GSPMM_ERR_CONFIG, bad + "expected {u,v,e}_<binop>_{u,v,e}_<redop>_{u,v,e}");
    c = {l, r, b, o == GSPMM_E ? GSPMM_COPY_LAST : rd, o};
  } else {
    return fail(GSPMM_ERR_CONFIG, bad + "expected 4 or 5 '_'-separated tokens");
  }
  const int st = validate_cfg(&c);
  if (st) return st;
  *cfg = c;
  return GSPMM_OK;
}

int gspmm_required_orientation(int strategy, int out) {
  const bool owner_rows = strategy != GSPMM_PUSH;
  if (out == GSPMM_V || out == GSPMM_E) return owner_rows ? GSPMM_DST_MAJOR : GSPMM_SRC_MAJOR;
  if (out == GSPMM_U) return owner_rows ? GSPMM_SRC_MAJOR : GSPMM_DST_MAJOR;
  fail(GSPMM_ERR_CONFIG, "output target must be u, v or e");
  return -1;
}

int gspmm_graph_create(int device, int orientation, uint32_t num_rows,
                       uint32_t num_cols, const uint32_t* indptr,
                       const uint32_t* indices, const uint32_t* edge_ids,
                       int validate, gspmm_graph* out) {
  if (!out || !indptr) return fail(GSPMM_ERR_ARG, "null argument");
  if (orientation != GSPMM_SRC_MAJOR && orientation != GSPMM_DST_MAJOR)
    return fail(GSPMM_ERR_ARG, "orientation must be 0 (src-major) or 1 (dst-major)");
  const uint64_t m = indptr[num_rows];
  if (m && (!indices || !edge_ids)) return fail(GSPMM_ERR_ARG, "null CSR array");
  if (validate) {
    const int st = validate_host(num_rows, num_cols, indptr, indices, edge_ids);
    if (st) return st;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(GSPMM_ERR_CUDA, "no CUDA device visible: the B200 kernels cannot run here");
  if (device < 0 || device >= ndev) return fail(GSPMM_ERR_ARG, "device index out of range");
  CUDA_TRY(cudaSetDevice(device), "cudaSetDevice");

  auto* g = new gspmm_graph_s;
  g->device = device;
  g->orientation = orientation;
  g->num_rows = num_rows;
  g->num_cols = num_cols;
  g->m = m;
  cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, device);

  auto cleanup = [&](cudaError_t e, const char* where) {
    destroy_graph(g);
    return cuda_fail(e, where);
  };
  cudaError_t e;
  if ((e = cudaMalloc(&g->d_indptr, sizeof(uint32_t) * (num_rows + 1))) != cudaSuccess)
    return cleanup(e, "cudaMalloc indptr");
  if ((e = cudaMalloc(&g->d_indices, sizeof(uint32_t) * std::max<uint64_t>(m, 1))) != cudaSuccess)
    return cleanup(e, "cudaMalloc indices");
  if ((e = cudaMalloc(&g->d_eids, sizeof(uint32_t) * std::max<uint64_t>(m, 1))) != cudaSuccess)
    return cleanup(e, "cudaMalloc edge_ids");
  if ((e = cudaMemcpy(g->d_indptr, indptr, sizeof(uint32_t) * (num_rows + 1),
                      cudaMemcpyHostToDevice)) != cudaSuccess)
    return cleanup(e, "upload indptr");
  if (m) {
    // host or device arrays (gspmm_graph_create_device): direction from UVA
    if ((e = cudaMemcpy(g->d_indices, indices, sizeof(uint32_t) * m, cudaMemcpyDefault)) !=
        cudaSuccess)
      return cleanup(e, "upload indices");
    if ((e = cudaMemcpy(g->d_eids, edge_ids, sizeof(uint32_t) * m, cudaMemcpyDefault)) !=
        cudaSuccess)
      return cleanup(e, "upload edge_ids");
  }
  const int st = build_plan(g, indptr);
  if (st) {
    destroy_graph(g);
    return st;
  }
  *out = g;
  return GSPMM_OK;
}

int gspmm_graph_create_device(int device, int orientation, uint32_t num_rows,
                              uint32_t num_cols, const uint32_t* d_indptr,
                              const uint32_t* d_indices, const uint32_t* d_edge_ids,
                              gspmm_graph* out) {
  if (!out || !d_indptr) return fail(GSPMM_ERR_ARG, "null argument");
  CUDA_TRY(cudaSetDevice(device), "cudaSetDevice");
  // the row plan is built on the host from indptr (rows + 1 words)
  std::vector<uint32_t> h(static_cast<size_t>(num_rows) + 1);
  CUDA_TRY(cudaMemcpy(h.data(), d_indptr, sizeof(uint32_t) * h.size(), cudaMemcpyDeviceToHost),
           "download indptr");
  return gspmm_graph_create(device, orientation, num_rows, num_cols, h.data(), d_indices,
                            d_edge_ids, 0, out);
}

int gspmm_build_csr_device(uint32_t n, int64_t m, const uint32_t* d_src, const uint32_t* d_dst,
                           int orientation, uint32_t* d_indptr, uint32_t* d_indices,
                           uint32_t* d_edge_ids, void* stream) {
  if (m < 0 || !d_indptr || (m && (!d_src || !d_dst || !d_indices || !d_edge_ids)))
    return fail(GSPMM_ERR_ARG, "null argument");
  if (orientation != GSPMM_SRC_MAJOR && orientation != GSPMM_DST_MAJOR)
    return fail(GSPMM_ERR_ARG, "orientation must be 0 (src-major) or 1 (dst-major)");
  if (static_cast<uint64_t>(m) > 0xffffffffull) return fail(GSPMM_ERR_ARG, "more than 2^32 - 1 edges");
  // build_csr's id check (csr.cpp:79-86): the lowest offending edge
  uint64_t bad = ~0ull;
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  CUDA_TRY(check_edge_ids(n, static_cast<uint64_t>(m), d_src, d_dst, cs, &bad), "build_csr_device");
  if (bad != ~0ull) {
    uint32_t ids[2] = {0, 0};
    CUDA_TRY(cudaMemcpy(&ids[0], d_src + bad, 4, cudaMemcpyDeviceToHost), "build_csr_device");
    CUDA_TRY(cudaMemcpy(&ids[1], d_dst + bad, 4, cudaMemcpyDeviceToHost), "build_csr_device");
    return fail(GSPMM_ERR_STRUCTURE, "edge " + std::to_string(bad) + " references node id " +
                                         std::to_string(std::max(ids[0], ids[1])) +
                                         " >= num_nodes " + std::to_string(n));
  }
  const cudaError_t e = launch_build_csr(n, static_cast<uint64_t>(m), d_src, d_dst,
                                         orientation == GSPMM_DST_MAJOR, d_indptr, d_indices,
                                         d_edge_ids, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "build_csr_device");
  return GSPMM_OK;
}

int gspmm_transpose_device(uint32_t num_rows, uint32_t num_cols, int64_t m,
                           const uint32_t* d_indptr, const uint32_t* d_indices,
                           const uint32_t* d_edge_ids, uint32_t* d_t_indptr,
                           uint32_t* d_t_indices, uint32_t* d_t_edge_ids, void* stream) {
  if (m < 0 || !d_indptr || !d_t_indptr ||
      (m && (!d_indices || !d_edge_ids || !d_t_indices || !d_t_edge_ids)))
    return fail(GSPMM_ERR_ARG, "null argument");
  const cudaError_t e = launch_transpose_csr(num_rows, num_cols, static_cast<uint64_t>(m), d_indptr,
                                             d_indices, d_edge_ids, d_t_indptr, d_t_indices,
                                             d_t_edge_ids, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "transpose_device");
  return GSPMM_OK;
}

int gspmm_graph_destroy(gspmm_graph g) {
  if (!g) return GSPMM_OK;
  destroy_graph(g);
  return GSPMM_OK;
}

int gspmm_graph_set_source_blocks(gspmm_graph g, int nblocks) {
  if (!g) return fail(GSPMM_ERR_ARG, "null graph handle");
  if (nblocks < 0) return fail(GSPMM_ERR_ARG, "nblocks must be >= 0");
  std::lock_guard<std::recursive_mutex> lock(g->mu);
  g->blocks_pref = nblocks;
  return GSPMM_OK;
}

int gspmm_graph_set_plan(gspmm_graph g, const gspmm_plan* plan) {
  if (!g) return fail(GSPMM_ERR_ARG, "null graph handle");
  const gspmm_plan dflt{};
  if (!plan) plan = &dflt;
  if (plan->unit_cols % 4 || plan->unit_cols > 512 || plan->kernel < 0 || plan->kernel > 2 ||
      (plan->split_edges > 1 && plan->split_edges < 16))
    return fail(GSPMM_ERR_ARG, "plan: unit_cols must be a multiple of 4 up to 512, kernel 0, 1 or 2, "
                               "split_edges 0, 1 or >= 16");
  std::lock_guard<std::recursive_mutex> lock(g->mu);
  CUDA_TRY(cudaSetDevice(g->device), "cudaSetDevice");
  // in-flight calls may still read the old plan
  CUDA_TRY(cudaDeviceSynchronize(), "set_plan");
  g->seg_cost = plan->seg_cost;
  g->forced_long = plan->long_threshold;
  g->unit_cols = plan->unit_cols;
  g->rows_kernel_only = plan->kernel == 1;
  g->pdl_pair = plan->kernel == 2;
  g->split_edges = plan->split_edges;
  g->long_ctas = plan->long_ctas;
  for (auto* sg : g->blocks) destroy_graph(sg);
  g->blocks.clear();
  g->block_nb = 0;
  std::vector<uint32_t> h(static_cast<size_t>(g->num_rows) + 1);
  CUDA_TRY(cudaMemcpy(h.data(), g->d_indptr, sizeof(uint32_t) * h.size(), cudaMemcpyDeviceToHost),
           "download indptr");
  return build_plan(g, h.data());
}

}  // extern "C"

namespace {
void destroy_graph(gspmm_graph_s* g) {
  cudaSetDevice(g->device);
  for (auto* sg : g->blocks) destroy_graph(sg);
  free_plan(g);
  free_contexts(g);
  cudaFree(g->d_indptr);
  cudaFree(g->d_indices);
  cudaFree(g->d_eids);
  cudaFree(g->d_rowof);
  delete g;
}
}  // namespace

extern "C" {

int gspmm_graph_info(gspmm_graph g, int* orientation, uint32_t* num_rows,
                     uint32_t* num_cols, uint64_t* num_edges,
                     uint32_t* num_long_rows) {
  if (!g) return fail(GSPMM_ERR_ARG, "null graph handle");
  if (orientation) *orientation = g->orientation;
  if (num_rows) *num_rows = g->num_rows;
  if (num_cols) *num_cols = g->num_cols;
  if (num_edges) *num_edges = g->m;
  if (num_long_rows) *num_long_rows = g->level[0].num_long;
  return GSPMM_OK;
}

int gspmm_graph_device_csr(gspmm_graph g, const uint32_t** indptr,
                           const uint32_t** indices, const uint32_t** edge_ids) {
  if (!g) return fail(GSPMM_ERR_ARG, "null graph handle");
  if (indptr) *indptr = g->d_indptr;
  if (indices) *indices = g->d_indices;
  if (edge_ids) *edge_ids = g->d_eids;
  return GSPMM_OK;
}

int gspmm_graph_permute_edges(gspmm_graph g, const float* src_by_id, int64_t dim,
                              int64_t src_ld, float* dst_by_pos, int64_t dst_ld,
                              void* stream) {
  if (!g || !src_by_id || !dst_by_pos) return fail(GSPMM_ERR_ARG, "null argument");
  CUDA_TRY(cudaSetDevice(g->device), "cudaSetDevice");
  CUDA_TRY(launch_permute_edges(g->d_eids, g->m, src_by_id, dim, src_ld ? src_ld : dim,
                                dst_by_pos, dst_ld ? dst_ld : dim,
                                static_cast<cudaStream_t>(stream)),
           "permute_edges");
  return GSPMM_OK;
}

int gspmm_out_shape(gspmm_graph g, const gspmm_config* cfg, const gspmm_mat* u,
                    const gspmm_mat* v, const gspmm_mat* e,
                    const gspmm_options* opt, int64_t* rows, int64_t* dim) {
  Bound b;
  const int st = bind(g, cfg, u, v, e, nullptr, opt, &b);
  if (st) return st;
  if (rows) *rows = b.out_rows;
  if (dim) *dim = b.width;
  return GSPMM_OK;
}

int gspmm_binary_reduce_ex(gspmm_graph g, const gspmm_config* cfg,
                           const gspmm_mat* u, const gspmm_mat* v,
                           const gspmm_mat* e, const gspmm_out* out,
                           const gspmm_options* opt, void* stream) {
  Bound b;
  int st = bind(g, cfg, u, v, e, out, opt, &b);
  if (st) return st;
  if (!out) return fail(GSPMM_ERR_SHAPE, "missing output matrix");
  if (b.width == 0) return GSPMM_OK;  // rows x 0: no element to compute
  return run_call(g, b, static_cast<cudaStream_t>(stream));
}

int gspmm_binary_reduce(gspmm_graph g, const gspmm_config* cfg,
                        const gspmm_mat* u, const gspmm_mat* v,
                        const gspmm_mat* e, const gspmm_out* out, void* stream) {
  return gspmm_binary_reduce_ex(g, cfg, u, v, e, out, nullptr, stream);
}

// copy_reduce, kernels.cpp:503-524
int gspmm_copy_reduce(gspmm_graph g, const gspmm_mat* src, int reduce,
                      const gspmm_out* out, void* stream) {
  if (!g || !src) return fail(GSPMM_ERR_ARG, "null argument");
  gspmm_config cfg{GSPMM_U, GSPMM_NONE, GSPMM_COPY, reduce, GSPMM_V};
  const bool src_major = g->orientation == GSPMM_SRC_MAJOR;
  const int64_t nu = src_major ? g->num_rows : g->num_cols;
  if (src->rows == nu) {
    cfg.lhs = GSPMM_U;
    return gspmm_binary_reduce(g, &cfg, src, nullptr, nullptr, out, stream);
  }
  if (src->rows == static_cast<int64_t>(g->m)) {
    cfg.lhs = GSPMM_E;
    return gspmm_binary_reduce(g, &cfg, nullptr, nullptr, src, out, stream);
  }
  return fail(GSPMM_ERR_SHAPE, "copy_reduce: source rows match neither the node nor the edge count");
}

// Fused GAT edge softmax (softmax.cu) over the in-edges of each destination.
static int softmax_common(gspmm_graph g, bool backward, const gspmm_mat* l, const gspmm_mat* ga,
                   const gspmm_out* out, void* stream) {
  if (!g || !l || !out || (backward && !ga)) return fail(GSPMM_ERR_ARG, "null argument");
  if (g->orientation != GSPMM_DST_MAJOR)
    return fail(GSPMM_ERR_SHAPE, "edge_softmax: needs the dst-major handle (softmax over in-edges)");
  const int64_t m = static_cast<int64_t>(g->m);
  const int64_t heads = l->dim;
  if (heads < 1 || heads > 32) return fail(GSPMM_ERR_SHAPE, "edge_softmax: 1..32 heads");
  auto check = [&](int64_t rows, int64_t dim, int64_t ld, const char* what) -> int {
    if (rows != m || dim != heads || (ld != 0 && ld < dim))
      return fail(GSPMM_ERR_SHAPE, std::string("edge_softmax: ") + what + " must be " +
                                       std::to_string(m) + " x " + std::to_string(heads));
    return GSPMM_OK;
  };
  int st = check(l->rows, l->dim, l->ld, backward ? "a" : "logits");
  if (!st && backward) st = check(ga->rows, ga->dim, ga->ld, "grad_a");
  if (!st) st = check(out->rows, out->dim, out->ld, "out");
  if (st) return st;
  if (backward && ga->edge_order != l->edge_order)
    return fail(GSPMM_ERR_ARG, "edge_softmax: a and grad_a must share one edge order");
  if (m && (!l->data || !out->data || (backward && !ga->data)))
    return fail(GSPMM_ERR_ARG, "null data");
  std::lock_guard<std::recursive_mutex> lock(g->mu);
  CUDA_TRY(cudaSetDevice(g->device), "cudaSetDevice");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CallCtx* ctx = nullptr;
  if ((st = context_for(g, s, &ctx))) return st;
  // Hub rows (one CTA each, side stream): above 4096 edges.  With the
  // warp-per-row kernel's rows handed out from a counter, a 4096-edge row is
  // no longer a tail, and a 1024-thread CTA on a 1500-edge row mostly waits
  // at its barriers: cfg4 forward 1.21 ms at 1024, 0.96 at 4096, 0.99 at
  // 8192, 1.82 at 16384 (r04s).  (The forward was 1.63 ms with the rows
  // strided statically over the grid, r04j / r04r.)
  const auto& lv = g->level[g->n_levels > 1 ? 1 : 0];
  if (lv.num_long && !ctx->side) {
    CUDA_TRY(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking), "side stream");
    CUDA_TRY(cudaEventCreateWithFlags(&ctx->fork, cudaEventDisableTiming), "event");
    CUDA_TRY(cudaEventCreateWithFlags(&ctx->join, cudaEventDisableTiming), "event");
  }
  if ((st = begin_call(ctx, s))) return st;
  SideStream side;
  side.stream = ctx->side;
  side.fork = ctx->fork;
  side.join = ctx->join;
  const cudaError_t e = launch_edge_softmax(
      backward, g->d_indptr, g->d_eids, g->num_rows, static_cast<int>(heads),
      l->edge_order == GSPMM_EDGE_BY_POS, l->data, l->ld ? l->ld : heads,
      backward ? ga->data : nullptr, backward ? (ga->ld ? ga->ld : heads) : 0, out->data,
      out->ld ? out->ld : heads, lv.d_long, lv.num_long, lv.threshold, g->num_sms, s, side,
      ctx->d_counter + 2);
  st = end_call(ctx, s);
  if (e != cudaSuccess) return cuda_fail(e, "edge_softmax");
  return st;
}

int gspmm_edge_softmax(gspmm_graph g, const gspmm_mat* logits, const gspmm_out* out,
                       void* stream) {
  return softmax_common(g, false, logits, nullptr, out, stream);
}

int gspmm_edge_softmax_backward(gspmm_graph g, const gspmm_mat* a, const gspmm_mat* grad_a,
                                const gspmm_out* grad_logits, void* stream) {
  return softmax_common(g, true, a, grad_a, grad_logits, stream);
}

int gspmm_argmax_backward_range(const int32_t* arg, int64_t rows, int64_t dim,
                                int64_t arg_ld, const float* grad_out, int64_t grad_ld,
                                float* grad_src, int64_t src_lo, int64_t src_rows,
                                int64_t src_ld, void* stream) {
  if (rows < 0 || dim < 0 || src_lo < 0 || src_rows < 0)
    return fail(GSPMM_ERR_ARG, "argmax_backward: negative size");
  if ((rows && dim && (!arg || !grad_out)) || (src_rows && dim && !grad_src))
    return fail(GSPMM_ERR_ARG, "null argument");
  if ((arg_ld && arg_ld < dim) || (grad_ld && grad_ld < dim) || (src_ld && src_ld < dim))
    return fail(GSPMM_ERR_SHAPE, "argmax_backward: a row stride is below the width");
  if (!src_rows || !dim) return GSPMM_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  retain_pool_memory();
  cudaError_t e = launch_argmax_backward(arg, rows, dim, arg_ld ? arg_ld : dim, grad_out,
                                         grad_ld ? grad_ld : dim, grad_src, src_lo, src_rows,
                                         src_ld ? src_ld : dim, s);
  if (e != cudaSuccess) return cuda_fail(e, "argmax_backward");
  return GSPMM_OK;
}

int gspmm_argmax_backward(const int32_t* arg, int64_t rows, int64_t dim,
                          int64_t arg_ld, const float* grad_out, int64_t grad_ld,
                          float* grad_src, int64_t src_rows, int64_t src_ld,
                          void* stream) {
  return gspmm_argmax_backward_range(arg, rows, dim, arg_ld, grad_out, grad_ld, grad_src, 0,
                                     src_rows, src_ld, stream);
}

static int host_call(gspmm_graph g, const gspmm_config* cfg, const gspmm_mat* u,
                     const gspmm_mat* v, const gspmm_mat* e, const gspmm_out* out,
                     const gspmm_options* opt, void* stream, bool sync, void* wait_event,
                     void* upload_event);

int gspmm_binary_reduce_host(gspmm_graph g, const gspmm_config* cfg,
                             const gspmm_mat* u, const gspmm_mat* v,
                             const gspmm_mat* e, const gspmm_out* out,
                             const gspmm_options* opt, void* stream) {
  return host_call(g, cfg, u, v, e, out, opt, stream, true, nullptr, nullptr);
}

int gspmm_binary_reduce_host_async(gspmm_graph g, const gspmm_config* cfg,
                                   const gspmm_mat* u, const gspmm_mat* v,
                                   const gspmm_mat* e, const gspmm_out* out,
                                   const gspmm_options* opt, void* stream,
                                   void* wait_event, void* upload_event) {
  return host_call(g, cfg, u, v, e, out, opt, stream, false, wait_event, upload_event);
}

// The host-buffer entries stage through a stream-ordered allocation of the
// caller's stream (the device pool keeps freed memory mapped, so a steady
// stream of calls re-uses one block): concurrent calls on other streams or
// threads never share a staging buffer.
static int host_call(gspmm_graph g, const gspmm_config* cfg, const gspmm_mat* u,
                     const gspmm_mat* v, const gspmm_mat* e, const gspmm_out* out,
                     const gspmm_options* opt, void* stream, bool sync, void* wait_event,
                     void* upload_event) {
  if (!g || !out) return fail(GSPMM_ERR_ARG, "null argument");
  // Validate against the host views first (shapes only; no pointer use).
  Bound probe;
  int st = bind(g, cfg, u, v, e, out, opt, &probe);
  if (st) return st;
  if (probe.width == 0) return GSPMM_OK;  // rows x 0: no element to compute
  CUDA_TRY(cudaSetDevice(g->device), "cudaSetDevice");
  retain_pool_memory();
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const gspmm_mat* in[3] = {u, v, e};
  size_t sz[3], total = 0;
  for (int i = 0; i < 3; ++i) total += round_up(sz[i] = mat_bytes(in[i]));
  const int64_t out_ld = out->ld ? out->ld : out->dim;
  const size_t out_bytes =
      out->rows ? static_cast<size_t>((out->rows - 1) * out_ld + out->dim) * sizeof(float) : 0;
  total += round_up(out_bytes);
  const int64_t arg_ld = opt && opt->arg_ld ? opt->arg_ld : out->dim;
  const size_t arg_bytes =
      out->rows ? static_cast<size_t>((out->rows - 1) * arg_ld + out->dim) * sizeof(int32_t) : 0;
  const bool ao = opt && opt->arg_other, ae = opt && opt->arg_edge;
  total += (ao ? round_up(arg_bytes) : 0) + (ae ? round_up(arg_bytes) : 0);
  const int64_t out2_ld = opt && opt->out2_ld ? opt->out2_ld : out->dim;
  const size_t out2_bytes = opt && opt->out2 && out->rows
                                ? static_cast<size_t>((out->rows - 1) * out2_ld + out->dim) *
                                      sizeof(float)
                                : 0;
  total += round_up(out2_bytes);
  // other_scale: a HOST array over the gathered (other) endpoint's nodes
  const size_t scale_bytes =
      opt && opt->other_scale ? sizeof(float) * static_cast<size_t>(g->num_cols) : 0;
  total += round_up(scale_bytes);
  if (wait_event)
    CUDA_TRY(cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(wait_event), 0), "wait event");
  void* ws = nullptr;
  CUDA_TRY(cudaMallocAsync(&ws, std::max<size_t>(total, 256), s), "host-call workspace");
  char* p = static_cast<char*>(ws);
  auto bail = [&](cudaError_t err, const char* where) {
    cudaFreeAsync(ws, s);
    return cuda_fail(err, where);
  };
  cudaError_t ce;
  gspmm_mat dev[3];
  const gspmm_mat* dptr[3] = {nullptr, nullptr, nullptr};
  for (int i = 0; i < 3; ++i) {
    if (!in[i] || !in[i]->data) continue;
    dev[i] = *in[i];
    dev[i].data = reinterpret_cast<const float*>(p);
    if ((ce = cudaMemcpyAsync(p, in[i]->data, sz[i], cudaMemcpyHostToDevice, s)) != cudaSuccess)
      return bail(ce, "H2D operand");
    dptr[i] = &dev[i];
    p += round_up(sz[i]);
  }
  gspmm_options dopt{};
  if (opt) dopt = *opt;
  if (scale_bytes) {
    if ((ce = cudaMemcpyAsync(p, opt->other_scale, scale_bytes, cudaMemcpyHostToDevice, s)) !=
        cudaSuccess)
      return bail(ce, "H2D scale");
    dopt.other_scale = reinterpret_cast<const float*>(p);
    p += round_up(scale_bytes);
  }
  if (upload_event && (ce = cudaEventRecord(static_cast<cudaEvent_t>(upload_event), s)) !=
                          cudaSuccess)
    return bail(ce, "upload event");
  gspmm_out dout = *out;
  dout.data = reinterpret_cast<float*>(p);
  p += round_up(out_bytes);
  if (ao) {
    dopt.arg_other = reinterpret_cast<int32_t*>(p);
    p += round_up(arg_bytes);
  }
  if (ae) {
    dopt.arg_edge = reinterpret_cast<int32_t*>(p);
    p += round_up(arg_bytes);
  }
  if (out2_bytes) {
    dopt.out2 = reinterpret_cast<float*>(p);
    p += round_up(out2_bytes);
  }
  st = gspmm_binary_reduce_ex(g, cfg, dptr[0], dptr[1], dptr[2], &dout, &dopt, stream);
  if (st) {
    cudaFreeAsync(ws, s);
    return st;
  }
  if ((ce = cudaMemcpyAsync(out->data, dout.data, out_bytes, cudaMemcpyDeviceToHost, s)) !=
      cudaSuccess)
    return bail(ce, "D2H out");
  if (ao && (ce = cudaMemcpyAsync(opt->arg_other, dopt.arg_other, arg_bytes,
                                  cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    return bail(ce, "D2H arg");
  if (ae && (ce = cudaMemcpyAsync(opt->arg_edge, dopt.arg_edge, arg_bytes,
                                  cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    return bail(ce, "D2H arg");
  if (out2_bytes && (ce = cudaMemcpyAsync(opt->out2, dopt.out2, out2_bytes,
                                          cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    return bail(ce, "D2H out2");
  CUDA_TRY(cudaFreeAsync(ws, s), "host-call workspace");
  if (sync) CUDA_TRY(cudaStreamSynchronize(s), "synchronize");
  return GSPMM_OK;
}

// Host-buffer argmax backward: arg and grad_out uploaded, grad_src read back
// (the same stream-ordered staging as host_call).
static int argmax_host(const int32_t* arg, int64_t rows, int64_t dim, const float* grad_out,
                       float* grad_src, int64_t src_rows, int device, void* stream, bool sync,
                       void* wait_event, void* upload_event) {
  if (rows < 0 || dim < 0 || src_rows < 0) return fail(GSPMM_ERR_ARG, "negative size");
  if ((rows && dim && (!arg || !grad_out)) || (src_rows && dim && !grad_src))
    return fail(GSPMM_ERR_ARG, "null argument");
  CUDA_TRY(cudaSetDevice(device), "cudaSetDevice");
  retain_pool_memory();
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t ab = sizeof(int32_t) * static_cast<size_t>(rows * dim);
  const size_t gb = sizeof(float) * static_cast<size_t>(rows * dim);
  const size_t ob = sizeof(float) * static_cast<size_t>(src_rows * dim);
  if (wait_event)
    CUDA_TRY(cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(wait_event), 0), "wait event");
  void* ws = nullptr;
  CUDA_TRY(cudaMallocAsync(&ws, std::max<size_t>(round_up(ab) + round_up(gb) + round_up(ob), 256), s),
           "host-call workspace");
  char* p = static_cast<char*>(ws);
  int32_t* da = reinterpret_cast<int32_t*>(p);
  float* dg = reinterpret_cast<float*>(p + round_up(ab));
  float* dout = reinterpret_cast<float*>(p + round_up(ab) + round_up(gb));
  cudaError_t ce = cudaMemcpyAsync(da, arg, ab, cudaMemcpyHostToDevice, s);
  if (ce == cudaSuccess) ce = cudaMemcpyAsync(dg, grad_out, gb, cudaMemcpyHostToDevice, s);
  if (ce == cudaSuccess && upload_event)
    ce = cudaEventRecord(static_cast<cudaEvent_t>(upload_event), s);
  int st = GSPMM_OK;
  if (ce == cudaSuccess)
    st = gspmm_argmax_backward(da, rows, dim, 0, dg, 0, dout, src_rows, 0, stream);
  if (ce == cudaSuccess && st == GSPMM_OK)
    ce = cudaMemcpyAsync(grad_src, dout, ob, cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(ws, s);
  if (ce != cudaSuccess) return cuda_fail(ce, "argmax_backward_host");
  if (st) return st;
  if (sync) CUDA_TRY(cudaStreamSynchronize(s), "synchronize");
  return GSPMM_OK;
}

int gspmm_argmax_backward_host(const int32_t* arg, int64_t rows, int64_t dim,
                               const float* grad_out, float* grad_src, int64_t src_rows,
                               int device, void* stream) {
  return argmax_host(arg, rows, dim, grad_out, grad_src, src_rows, device, stream, true, nullptr,
                     nullptr);
}

int gspmm_argmax_backward_host_async(const int32_t* arg, int64_t rows, int64_t dim,
                                     const float* grad_out, float* grad_src, int64_t src_rows,
                                     int device, void* stream, void* wait_event,
                                     void* upload_event) {
  return argmax_host(arg, rows, dim, grad_out, grad_src, src_rows, device, stream, false,
                     wait_event, upload_event);
}

}  // extern "C"

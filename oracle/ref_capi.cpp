// ref_capi.cpp -- flat C entry points over the UNMODIFIED reference library.
//
// TEST/BASELINE INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file
// together with the reference's own sources, where they lie under
// /root/reference/proj/src, into oracle/_ref/libgspmm_ref.so.  Nothing here
// re-implements the reference: every call goes through its public API
// (generate.hpp, csr.hpp, kernels.hpp, oracle.hpp, bench.hpp).  The parity
// tests use it to pin the C restatement (oracle/gspmm_oracle.c), and
// bench.py --impl reference times binary_reduce through it.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "gspmm/bench.hpp"
#include "gspmm/br_config.hpp"
#include "gspmm/csr.hpp"
#include "gspmm/error.hpp"
#include "gspmm/generate.hpp"
#include "gspmm/io.hpp"
#include "gspmm/kernels.hpp"
#include "gspmm/oracle.hpp"

using namespace gspmm;

namespace {

int status_of(const std::exception_ptr& p) {
  try {
    std::rethrow_exception(p);
  } catch (const ConfigError&) {
    return 1;
  } catch (const ShapeError&) {
    return 2;
  } catch (const StructureError&) {
    return 3;
  } catch (const IoError&) {
    return 6;
  } catch (const ParseError&) {
    return 7;
  } catch (...) {
    return 9;
  }
}

CsrGraph make_graph(int orientation, uint32_t num_rows, uint32_t num_cols,
                    const uint32_t* indptr, const uint32_t* indices,
                    const uint32_t* eids) {
  CsrGraph g;
  g.orientation = orientation ? Orientation::DstMajor : Orientation::SrcMajor;
  g.num_rows = num_rows;
  g.num_cols = num_cols;
  g.indptr.assign(indptr, indptr + num_rows + 1);
  const std::size_t m = g.indptr.back();
  g.indices.assign(indices, indices + m);
  g.edge_ids.assign(eids, eids + m);
  return g;
}

struct FeatArg {
  const float* data;
  int64_t rows;
  int64_t dim;
};

bool to_matrix(const FeatArg* a, FeatureMatrix& out) {
  if (!a || !a->data) return false;
  out.rows = a->rows;
  out.dim = a->dim;
  out.data.assign(a->data, a->data + a->rows * a->dim);
  return true;
}

BrConfig make_cfg(int lhs, int rhs, int binop, int reduce, int out) {
  BrConfig c;
  c.lhs = static_cast<Operand>(lhs);
  c.rhs = static_cast<Operand>(rhs);
  c.binary = static_cast<BinaryOp>(binop);
  c.reduce = static_cast<ReduceOp>(reduce);
  c.out = static_cast<Operand>(out);
  return c;
}

}  // namespace

extern "C" {

void ref_free(void* p) { std::free(p); }

// generate(), generate.cpp:220-228.  kind: 0 er, 1 rmat, 2 sbm.
int64_t ref_generate(int kind, uint32_t n, uint64_t num_edges, double prob,
                     int blocks, double p_in, double p_out, double a, double b,
                     double c, double d, uint64_t seed, uint32_t** src,
                     uint32_t** dst) {
  try {
    GeneratorSpec s;
    s.kind = static_cast<GeneratorKind>(kind);
    s.num_nodes = n;
    s.num_edges = num_edges;
    s.prob = prob;
    s.blocks = blocks;
    s.p_in = p_in;
    s.p_out = p_out;
    s.a = a;
    s.b = b;
    s.c = c;
    s.d = d;
    s.seed = seed;
    const EdgeList el = generate(s);
    const std::size_t m = el.edges.size();
    *src = static_cast<uint32_t*>(std::malloc((m ? m : 1) * sizeof(uint32_t)));
    *dst = static_cast<uint32_t*>(std::malloc((m ? m : 1) * sizeof(uint32_t)));
    for (std::size_t i = 0; i < m; ++i) {
      (*src)[i] = el.edges[i].src;
      (*dst)[i] = el.edges[i].dst;
    }
    return static_cast<int64_t>(m);
  } catch (...) {
    return -status_of(std::current_exception());
  }
}

void ref_random_features(int64_t rows, int64_t dim, uint64_t seed, float* out) {
  const FeatureMatrix f = random_features(rows, dim, seed);
  std::memcpy(out, f.data.data(), f.data.size() * sizeof(float));
}

int ref_build_csr(uint32_t n, int64_t m, const uint32_t* src,
                  const uint32_t* dst, int orientation, uint32_t* indptr,
                  uint32_t* indices, uint32_t* eids) {
  try {
    EdgeList el;
    el.num_nodes = n;
    el.edges.resize(m);
    for (int64_t i = 0; i < m; ++i) el.edges[i] = Edge{src[i], dst[i]};
    const CsrGraph g = build_csr(
        el, orientation ? Orientation::DstMajor : Orientation::SrcMajor);
    std::memcpy(indptr, g.indptr.data(), g.indptr.size() * sizeof(uint32_t));
    std::memcpy(indices, g.indices.data(), g.indices.size() * sizeof(uint32_t));
    std::memcpy(eids, g.edge_ids.data(), g.edge_ids.size() * sizeof(uint32_t));
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

int ref_transpose(int orientation, uint32_t num_rows, uint32_t num_cols,
                  const uint32_t* indptr, const uint32_t* indices,
                  const uint32_t* eids, uint32_t* t_indptr,
                  uint32_t* t_indices, uint32_t* t_eids) {
  try {
    const CsrGraph g =
        make_graph(orientation, num_rows, num_cols, indptr, indices, eids);
    const CsrGraph t = transpose(g);
    std::memcpy(t_indptr, t.indptr.data(), t.indptr.size() * sizeof(uint32_t));
    std::memcpy(t_indices, t.indices.data(), t.indices.size() * sizeof(uint32_t));
    std::memcpy(t_eids, t.edge_ids.data(), t.edge_ids.size() * sizeof(uint32_t));
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

// binary_reduce(strategy, ...), kernels.hpp:60-64.  strategy: 0 push,
// 1 pull, 2 blocked (plan built with the reference defaults), 3 spmm.
// The result is copied into out (out_rows*out_dim floats, sized by the
// caller from ref_out_shape or the oracle).
int ref_binary_reduce(int strategy, int orientation, uint32_t num_rows,
                      uint32_t num_cols, const uint32_t* indptr,
                      const uint32_t* indices, const uint32_t* eids, int lhs,
                      int rhs, int binop, int reduce, int out_ent,
                      const FeatArg* u, const FeatArg* v, const FeatArg* e,
                      int threads, float* out, int64_t* out_rows,
                      int64_t* out_dim) {
  try {
    const CsrGraph g =
        make_graph(orientation, num_rows, num_cols, indptr, indices, eids);
    FeatureMatrix fu, fv, fe;
    const FeatureMatrix* pu = to_matrix(u, fu) ? &fu : nullptr;
    const FeatureMatrix* pv = to_matrix(v, fv) ? &fv : nullptr;
    const FeatureMatrix* pe = to_matrix(e, fe) ? &fe : nullptr;
    const BrConfig cfg = make_cfg(lhs, rhs, binop, reduce, out_ent);
    const Strategy s = static_cast<Strategy>(strategy);
    BlockPlan plan;
    if (s == Strategy::BlockedPull) {
      const int64_t dim = pu ? pu->dim : (pe ? pe->dim : 4);
      plan = build_block_plan(g, default_kb(dim, g.num_cols),
                              default_nb(g.num_rows, dim));
    }
    const FeatureMatrix res =
        binary_reduce(s, g, cfg, pu, pv, pe,
                      s == Strategy::BlockedPull ? &plan : nullptr, threads);
    *out_rows = res.rows;
    *out_dim = res.dim;
    if (out) std::memcpy(out, res.data.data(), res.data.size() * sizeof(float));
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

// oracle_aggregate, oracle.hpp:35-38.
int ref_oracle_aggregate(uint32_t n, int64_t m, const uint32_t* src,
                         const uint32_t* dst, int lhs, int rhs, int binop,
                         int reduce, int out_ent, const FeatArg* u,
                         const FeatArg* v, const FeatArg* e, float* out,
                         int64_t* out_rows, int64_t* out_dim) {
  try {
    EdgeList el;
    el.num_nodes = n;
    el.edges.resize(m);
    for (int64_t i = 0; i < m; ++i) el.edges[i] = Edge{src[i], dst[i]};
    FeatureMatrix fu, fv, fe;
    const FeatureMatrix* pu = to_matrix(u, fu) ? &fu : nullptr;
    const FeatureMatrix* pv = to_matrix(v, fv) ? &fv : nullptr;
    const FeatureMatrix* pe = to_matrix(e, fe) ? &fe : nullptr;
    const FeatureMatrix res = oracle_aggregate(
        el, make_cfg(lhs, rhs, binop, reduce, out_ent), pu, pv, pe);
    *out_rows = res.rows;
    *out_dim = res.dim;
    if (out) std::memcpy(out, res.data.data(), res.data.size() * sizeof(float));
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

// ---- persistent objects for timing (bench.py --impl reference) ----------

// Both orientations of one edge list, make_views bench.cpp:48-53.
void* ref_views_create(uint32_t n, int64_t m, const uint32_t* src,
                       const uint32_t* dst) {
  try {
    EdgeList el;
    el.num_nodes = n;
    el.edges.resize(m);
    for (int64_t i = 0; i < m; ++i) el.edges[i] = Edge{src[i], dst[i]};
    return new GraphViews(make_views(el));
  } catch (...) {
    return nullptr;
  }
}
void ref_views_free(void* v) { delete static_cast<GraphViews*>(v); }

// Copies the canonical CSR of one orientation out of a views object.
int ref_views_csr(void* views, int orientation, uint32_t* indptr,
                  uint32_t* indices, uint32_t* eids) {
  const GraphViews* gv = static_cast<GraphViews*>(views);
  const CsrGraph& g =
      gv->oriented(orientation ? Orientation::DstMajor : Orientation::SrcMajor);
  std::memcpy(indptr, g.indptr.data(), g.indptr.size() * sizeof(uint32_t));
  std::memcpy(indices, g.indices.data(), g.indices.size() * sizeof(uint32_t));
  std::memcpy(eids, g.edge_ids.data(), g.edge_ids.size() * sizeof(uint32_t));
  return 0;
}

void* ref_feat_create(int64_t rows, int64_t dim, const float* data) {
  auto* f = new FeatureMatrix(rows, dim);
  if (data) std::memcpy(f->data.data(), data, rows * dim * sizeof(float));
  return f;
}
void ref_feat_free(void* f) { delete static_cast<FeatureMatrix*>(f); }

// One binary_reduce call timed with steady_clock around the call, exactly
// the reference's bench_case timed region (bench.cpp:114-117): output
// allocation and zero fill are inside.  Returns seconds, negative status on
// error.  If out is non-null the result is copied (outside the timing).
double ref_run(void* views, int strategy, int lhs, int rhs, int binop,
               int reduce, int out_ent, void* u, void* v, void* e,
               int threads, float* out) {
  try {
    const GraphViews* gv = static_cast<GraphViews*>(views);
    const BrConfig cfg = make_cfg(lhs, rhs, binop, reduce, out_ent);
    const Strategy s = static_cast<Strategy>(strategy);
    const CsrGraph& g = gv->oriented(required_orientation(s, cfg.out));
    // BlockedPull: the plan with the reference's default blocking, built
    // before the clock starts (as bench_case does, bench.cpp:95-97)
    BlockPlan plan;
    if (s == Strategy::BlockedPull) {
      const auto* fu = static_cast<FeatureMatrix*>(u);
      const auto* fv = static_cast<FeatureMatrix*>(v);
      const auto* fe = static_cast<FeatureMatrix*>(e);
      const int64_t dim = fu ? fu->dim : fv ? fv->dim : fe ? fe->dim : 4;
      plan = build_block_plan(g, default_kb(dim, g.num_cols), default_nb(g.num_rows, dim));
    }
    const auto t0 = std::chrono::steady_clock::now();
    const FeatureMatrix res = binary_reduce(
        s, g, cfg, static_cast<FeatureMatrix*>(u),
        static_cast<FeatureMatrix*>(v), static_cast<FeatureMatrix*>(e),
        s == Strategy::BlockedPull ? &plan : nullptr, threads);
    const double dt =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0)
            .count();
    if (out) std::memcpy(out, res.data.data(), res.data.size() * sizeof(float));
    return dt;
  } catch (...) {
    return -static_cast<double>(status_of(std::current_exception()));
  }
}

// bench_case (bench.cpp:55-126) for one cell; returns mean seconds and
// fills min seconds and the reference's own gbps model.
double ref_bench_case(void* views, int strategy, int lhs, int rhs, int binop,
                      int reduce, int out_ent, void* u, void* v, void* e,
                      int threads, int warmup, int iters, double* min_s,
                      double* gbps) {
  try {
    const GraphViews* gv = static_cast<GraphViews*>(views);
    const BrConfig cfg = make_cfg(lhs, rhs, binop, reduce, out_ent);
    BenchOptions opts;
    opts.warmup = warmup;
    opts.iters = iters;
    const BenchReport r = bench_case(
        *gv, config_name(cfg), cfg, static_cast<FeatureMatrix*>(u),
        static_cast<FeatureMatrix*>(v), static_cast<FeatureMatrix*>(e),
        static_cast<Strategy>(strategy), threads, 0, 0, opts);
    if (min_s) *min_s = r.min_s;
    if (gbps) *gbps = r.gbps;
    return r.mean_s;
  } catch (...) {
    return -static_cast<double>(status_of(std::current_exception()));
  }
}

// The same cell as the reference's own CSV row (bench_csv_row,
// bench.cpp:133-145: config,strategy,nodes,edges,dim,threads,kb,nb,iters,
// mean_s,min_s,gbps) written to buf; returns mean seconds.
double ref_bench_csv(void* views, int strategy, int lhs, int rhs, int binop,
                     int reduce, int out_ent, void* u, void* v, void* e,
                     int threads, int warmup, int iters, char* buf, int cap) {
  try {
    const GraphViews* gv = static_cast<GraphViews*>(views);
    const BrConfig cfg = make_cfg(lhs, rhs, binop, reduce, out_ent);
    BenchOptions opts;
    opts.warmup = warmup;
    opts.iters = iters;
    const BenchReport r = bench_case(
        *gv, config_name(cfg), cfg, static_cast<FeatureMatrix*>(u),
        static_cast<FeatureMatrix*>(v), static_cast<FeatureMatrix*>(e),
        static_cast<Strategy>(strategy), threads, 0, 0, opts);
    if (buf && cap > 0) std::snprintf(buf, cap, "%s", bench_csv_row(r).c_str());
    return r.mean_s;
  } catch (...) {
    return -static_cast<double>(status_of(std::current_exception()));
  }
}
const char* ref_bench_csv_header(void) { return bench_csv_header(); }

// ---- canonical CSR handed in directly (BASELINE-size parity) -------------

// A CsrGraph holding the given canonical CSR (csr.hpp:37-54).  The tests pass
// the CSR the product's builder made, which test_abi / test_oracle_pins check
// against build_csr; this skips the reference's single-threaded build
// (~25 s per orientation at config-3 size).
void* ref_graph_create(int orientation, uint32_t num_rows, uint32_t num_cols,
                       const uint32_t* indptr, const uint32_t* indices,
                       const uint32_t* eids) {
  try {
    return new CsrGraph(make_graph(orientation, num_rows, num_cols, indptr, indices, eids));
  } catch (...) {
    return nullptr;
  }
}
void ref_graph_free(void* g) { delete static_cast<CsrGraph*>(g); }

// A FeatureMatrix copied from a strided source (ld >= dim floats per row):
// per-head column slices without a host-side copy first.
void* ref_feat_create_strided(int64_t rows, int64_t dim, const float* data, int64_t ld) {
  auto* f = new FeatureMatrix(rows, dim);
  for (int64_t r = 0; r < rows; ++r)
    std::memcpy(f->data.data() + r * dim, data + r * ld, dim * sizeof(float));
  return f;
}

// binary_reduce(strategy, g, cfg, u, v, e, nullptr, threads) on a graph from
// ref_graph_create, timed like ref_run; the result (rows x dim) is copied to
// out with row pitch out_ld (0: dense) outside the timing.  BlockedPull builds
// its plan with the reference defaults before the clock starts.
double ref_run_graph(void* graph, int strategy, int lhs, int rhs, int binop, int reduce,
                     int out_ent, void* u, void* v, void* e, int threads, float* out,
                     int64_t out_ld) {
  try {
    const CsrGraph& g = *static_cast<CsrGraph*>(graph);
    const BrConfig cfg = make_cfg(lhs, rhs, binop, reduce, out_ent);
    const Strategy s = static_cast<Strategy>(strategy);
    const auto* fu = static_cast<FeatureMatrix*>(u);
    const auto* fe = static_cast<FeatureMatrix*>(e);
    BlockPlan plan;
    if (s == Strategy::BlockedPull) {
      const int64_t dim = fu ? fu->dim : (fe ? fe->dim : 4);
      plan = build_block_plan(g, default_kb(dim, g.num_cols), default_nb(g.num_rows, dim));
    }
    const auto t0 = std::chrono::steady_clock::now();
    const FeatureMatrix res = binary_reduce(
        s, g, cfg, fu, static_cast<FeatureMatrix*>(v), fe,
        s == Strategy::BlockedPull ? &plan : nullptr, threads);
    const double dt =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (out) {
      const int64_t ld = out_ld ? out_ld : res.dim;
      for (int64_t r = 0; r < res.rows; ++r)
        std::memcpy(out + r * ld, res.data.data() + r * res.dim, res.dim * sizeof(float));
    }
    return dt;
  } catch (...) {
    return -static_cast<double>(status_of(std::current_exception()));
  }
}

// ---- file containers (io.hpp:25-41): the reference's own writers and
// readers, for the CSR1 / FMAT1 / edge-list round-trip tests ------------------

thread_local std::string g_io_msg;
const char* ref_io_error(void) { return g_io_msg.c_str(); }

namespace {
int io_status(const std::exception_ptr& p) {
  try {
    std::rethrow_exception(p);
  } catch (const std::exception& e) {
    g_io_msg = e.what();
  } catch (...) {
    g_io_msg = "unknown";
  }
  return status_of(p);
}
}  // namespace

int ref_save_csr(const char* path, void* graph) {
  try {
    save_csr(path, *static_cast<CsrGraph*>(graph));
    return 0;
  } catch (...) {
    return io_status(std::current_exception());
  }
}

// load_csr -> a graph handle (ref_graph_free) and its sizes
int ref_load_csr(const char* path, void** graph, int* orientation, uint32_t* num_rows,
                 uint32_t* num_cols, uint64_t* num_edges) {
  try {
    auto* g = new CsrGraph(load_csr(path));
    *graph = g;
    *orientation = g->orientation == Orientation::DstMajor ? 1 : 0;
    *num_rows = g->num_rows;
    *num_cols = g->num_cols;
    *num_edges = g->num_edges();
    return 0;
  } catch (...) {
    return io_status(std::current_exception());
  }
}

void ref_graph_arrays(void* graph, uint32_t* indptr, uint32_t* indices, uint32_t* eids) {
  const CsrGraph& g = *static_cast<CsrGraph*>(graph);
  std::memcpy(indptr, g.indptr.data(), g.indptr.size() * sizeof(uint32_t));
  std::memcpy(indices, g.indices.data(), g.indices.size() * sizeof(uint32_t));
  std::memcpy(eids, g.edge_ids.data(), g.edge_ids.size() * sizeof(uint32_t));
}

int ref_save_feature_matrix(const char* path, void* feat) {
  try {
    save_feature_matrix(path, *static_cast<FeatureMatrix*>(feat));
    return 0;
  } catch (...) {
    return io_status(std::current_exception());
  }
}

int ref_load_feature_matrix(const char* path, void** feat, int64_t* rows, int64_t* dim) {
  try {
    auto* f = new FeatureMatrix(load_feature_matrix(path));
    *feat = f;
    *rows = f->rows;
    *dim = f->dim;
    return 0;
  } catch (...) {
    return io_status(std::current_exception());
  }
}

void ref_feat_data(void* feat, float* out) {
  const FeatureMatrix& f = *static_cast<FeatureMatrix*>(feat);
  std::memcpy(out, f.data.data(), f.data.size() * sizeof(float));
}

int ref_save_edge_list(const char* path, uint32_t n, int64_t m, const uint32_t* src,
                       const uint32_t* dst) {
  try {
    EdgeList el;
    el.num_nodes = n;
    el.edges.resize(m);
    for (int64_t i = 0; i < m; ++i) el.edges[i] = Edge{src[i], dst[i]};
    save_edge_list(path, el);
    return 0;
  } catch (...) {
    return io_status(std::current_exception());
  }
}

int ref_load_edge_list(const char* path, uint32_t* n, int64_t* m, uint32_t** src, uint32_t** dst) {
  try {
    const EdgeList el = load_edge_list(path);
    const std::size_t k = el.edges.size();
    *n = el.num_nodes;
    *m = static_cast<int64_t>(k);
    *src = static_cast<uint32_t*>(std::malloc((k ? k : 1) * sizeof(uint32_t)));
    *dst = static_cast<uint32_t*>(std::malloc((k ? k : 1) * sizeof(uint32_t)));
    for (std::size_t i = 0; i < k; ++i) {
      (*src)[i] = el.edges[i].src;
      (*dst)[i] = el.edges[i].dst;
    }
    return 0;
  } catch (...) {
    return io_status(std::current_exception());
  }
}

}  // extern "C"

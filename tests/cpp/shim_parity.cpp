// shim_parity.cpp -- the reference-signature C++ API of this repo
// (gspmm_b200::binary_reduce / copy_reduce, include/gspmm_b200.hpp) called
// side by side with the unmodified reference library (gspmm::, linked from
// oracle/_ref) on identical inputs, in the style of the reference's own
// proj/tests/test_kernels.cpp.  Exit code 0 = all checks passed.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "gspmm/bench.hpp"
#include "gspmm/compare.hpp"
#include "gspmm/error.hpp"
#include "gspmm/generate.hpp"
#include "gspmm/io.hpp"
#include "gspmm/kernels.hpp"
#include "gspmm/oracle.hpp"
#include "gspmm/rng.hpp"
#include "gspmm_b200.h"
#include "gspmm_b200.hpp"

namespace R = gspmm;
namespace B = gspmm_b200;

static int g_checks = 0, g_fail = 0;
#define CHECK(cond)                                                            \
  do {                                                                         \
    ++g_checks;                                                                \
    if (!(cond)) {                                                             \
      ++g_fail;                                                                \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);     \
    }                                                                          \
  } while (0)
#define CHECK_THROWS_AS(expr, Ex)                                              \
  do {                                                                         \
    ++g_checks;                                                                \
    bool ok = false;                                                           \
    try {                                                                      \
      (void)(expr);                                                            \
    } catch (const Ex&) {                                                      \
      ok = true;                                                               \
    } catch (...) {                                                            \
    }                                                                          \
    if (!ok) {                                                                 \
      ++g_fail;                                                                \
      std::fprintf(stderr, "FAIL %s:%d: %s does not throw %s\n", __FILE__,     \
                   __LINE__, #expr, #Ex);                                      \
    }                                                                          \
  } while (0)

static B::CsrGraph to_b(const R::CsrGraph& g) {
  B::CsrGraph b;
  b.orientation = static_cast<B::Orientation>(g.orientation);
  b.num_rows = g.num_rows;
  b.num_cols = g.num_cols;
  b.indptr = g.indptr;
  b.indices = g.indices;
  b.edge_ids = g.edge_ids;
  return b;
}

static B::FeatureMatrix to_b(const R::FeatureMatrix& f) {
  B::FeatureMatrix b(f.rows, f.dim);
  b.data = f.data;
  return b;
}

static B::BrConfig to_b(const R::BrConfig& c) {
  B::BrConfig b;
  b.lhs = static_cast<B::Operand>(c.lhs);
  b.rhs = static_cast<B::Operand>(c.rhs);
  b.binary = static_cast<B::BinaryOp>(c.binary);
  b.reduce = static_cast<B::ReduceOp>(c.reduce);
  b.out = static_cast<B::Operand>(c.out);
  return b;
}

static bool same_bits(const B::FeatureMatrix& a, const R::FeatureMatrix& b) {
  R::FeatureMatrix t;
  t.rows = a.rows;
  t.dim = a.dim;
  t.data = a.data;
  return R::bit_equal(t, b);
}

static R::EdgeList random_small_graph(std::uint64_t seed) {  // test_util.hpp:30-61
  R::GeneratorSpec spec;
  spec.seed = seed;
  const std::uint64_t pick = R::splitmix64_at(seed, 9000);
  spec.num_nodes = 8 + static_cast<R::NodeId>(R::splitmix64_at(seed, 9001) % 193);
  const double degree = 1.0 + static_cast<double>(R::splitmix64_at(seed, 9002) % 10);
  switch (pick % 3) {
    case 0:
      spec.kind = R::GeneratorKind::ErdosRenyi;
      spec.prob = std::min(1.0, degree / (static_cast<double>(spec.num_nodes) - 1.0));
      break;
    case 1:
      spec.kind = R::GeneratorKind::RMat;
      spec.num_edges = std::min<std::uint64_t>(2000, static_cast<std::uint64_t>(degree * spec.num_nodes));
      spec.a = 0.40; spec.b = 0.25; spec.c = 0.25; spec.d = 0.10;
      break;
    default:
      spec.kind = R::GeneratorKind::Sbm;
      spec.blocks = 1 + static_cast<int>(R::splitmix64_at(seed, 9004) % 4);
      spec.p_in = std::min(1.0, degree * spec.blocks / static_cast<double>(spec.num_nodes));
      spec.p_out = spec.p_in / 20.0;
      break;
  }
  return R::generate(spec);
}

// The reference-side adapter of INTEGRATION.md section 2, written against
// the REFERENCE's own types (R::CsrGraph, R::FeatureMatrix, R::BlockPlan)
// and calling the C-ABI: Push runs on the transposed view, BlockedPull's plan
// is checked like kernels.cpp:462-467 and becomes per-call source blocks,
// every failure throws (no CPU fallback).
[[noreturn]] static void throw_b200(int st) {
  const std::string msg = std::string("B200: ") + gspmm_last_error();
  if (st == GSPMM_ERR_SHAPE) throw R::ShapeError(msg);
  if (st == GSPMM_ERR_CONFIG) throw R::ConfigError(msg);
  if (st == GSPMM_ERR_STRUCTURE) throw R::StructureError(msg);
  throw std::runtime_error(msg);
}

static gspmm_mat as_mat(const R::FeatureMatrix* f) {
  gspmm_mat m{};
  if (f) m = {f->data.data(), f->rows, f->dim, f->dim, GSPMM_EDGE_BY_ID};
  return m;
}

static R::FeatureMatrix adapter_binary_reduce(R::Strategy strategy, const R::CsrGraph& g,
                                              const R::BrConfig& cfg,
                                              const R::FeatureMatrix* u_feats,
                                              const R::FeatureMatrix* v_feats,
                                              const R::FeatureMatrix* e_feats,
                                              const R::BlockPlan* plan) {
  R::validate_config(cfg);
  if (g.orientation != R::required_orientation(strategy, cfg.out))
    throw R::ShapeError("graph orientation does not match the strategy");
  const R::CsrGraph owner_view = strategy == R::Strategy::Push ? R::transpose(g) : R::CsrGraph{};
  const R::CsrGraph& dg = strategy == R::Strategy::Push ? owner_view : g;
  if (strategy == R::Strategy::BlockedPull &&
      (!plan || plan->built_for != g.orientation || plan->num_rows != g.num_rows ||
       plan->num_cols != g.num_cols || plan->num_edges() != g.num_edges()))
    throw R::ShapeError("BlockPlan was not built for this graph");
  gspmm_graph h = nullptr;
  int st = gspmm_graph_create(0, static_cast<int>(dg.orientation), dg.num_rows, dg.num_cols,
                              dg.indptr.data(), dg.indices.data(), dg.edge_ids.data(), 0, &h);
  if (st != GSPMM_OK) throw_b200(st);
  const gspmm_config c{static_cast<int32_t>(cfg.lhs), static_cast<int32_t>(cfg.rhs),
                       static_cast<int32_t>(cfg.binary), static_cast<int32_t>(cfg.reduce),
                       static_cast<int32_t>(cfg.out)};
  gspmm_mat mu = as_mat(u_feats), mv = as_mat(v_feats), me = as_mat(e_feats);
  gspmm_options opt{};
  if (strategy == R::Strategy::BlockedPull)
    opt.source_blocks = static_cast<int32_t>(std::min<R::NodeId>(plan->num_blocks, 64));
  int64_t rows = 0, dim = 0;
  st = gspmm_out_shape(h, &c, u_feats ? &mu : nullptr, v_feats ? &mv : nullptr,
                       e_feats ? &me : nullptr, &opt, &rows, &dim);
  R::FeatureMatrix out(st == GSPMM_OK ? rows : 0, st == GSPMM_OK ? dim : 0);
  if (st == GSPMM_OK && rows * dim > 0) {
    gspmm_out o{out.data.data(), rows, dim, dim};
    st = gspmm_binary_reduce_host(h, &c, u_feats ? &mu : nullptr, v_feats ? &mv : nullptr,
                                  e_feats ? &me : nullptr, &o, &opt, nullptr);
  }
  gspmm_graph_destroy(h);
  if (st != GSPMM_OK) throw_b200(st);
  return out;
}

int main() {
  const R::Strategy kAll[] = {R::Strategy::Push, R::Strategy::Pull, R::Strategy::BlockedPull,
                              R::Strategy::RowParallelSpmm};
  // copy_reduce golden (test_kernels.cpp:49-66), through both libraries
  {
    R::EdgeList el;
    el.num_nodes = 3;
    el.edges = {{0, 2}, {1, 2}};
    const R::GraphViews views = R::make_views(el);
    R::FeatureMatrix fu(3, 2);
    fu.data = {1, 2, 3, 4, 0, 0};
    const B::FeatureMatrix out = B::copy_reduce(B::Strategy::RowParallelSpmm,
                                                to_b(views.dst_major), to_b(fu), B::ReduceOp::Sum);
    CHECK(out.rows == 3 && out.at(2, 0) == 4 && out.at(2, 1) == 6 && out.at(0, 0) == 0);
  }
  // every application config x every strategy, shim vs the reference's
  // RowParallelSpmm, bitwise (test_kernels.cpp:202-226)
  for (std::uint64_t seed = 101; seed <= 110; ++seed) {
    const R::EdgeList el = random_small_graph(seed);
    const R::GraphViews views = R::make_views(el);
    const B::CsrGraph bd = to_b(views.dst_major), bs = to_b(views.src_major);
    const std::int64_t dim = 1 + static_cast<std::int64_t>(R::splitmix64_at(seed, 1) % 17);
    const R::FeatureMatrix fu = R::random_features(el.num_nodes, dim, seed);
    const R::FeatureMatrix fv = R::random_features(el.num_nodes, dim, seed + 1);
    const R::FeatureMatrix fe = R::random_features(el.num_edges(), dim, seed + 2);
    const B::FeatureMatrix bu = to_b(fu), bv = to_b(fv), be = to_b(fe);
    for (const auto& name : R::application_configs()) {
      const R::BrConfig cfg = R::named_config(name);
      const R::FeatureMatrix want = R::binary_reduce(
          R::Strategy::RowParallelSpmm, views.oriented(R::required_orientation(R::Strategy::RowParallelSpmm, cfg.out)),
          cfg, &fu, &fv, &fe);
      const R::FeatureMatrix oracle = R::oracle_aggregate(el, cfg, &fu, &fv, &fe);
      for (const R::Strategy s : kAll) {
        const B::Strategy bs_ = static_cast<B::Strategy>(s);
        const B::Orientation need = B::required_orientation(bs_, to_b(cfg).out);
        const B::CsrGraph& g = need == B::Orientation::DstMajor ? bd : bs;
        // BlockedPull: a 3-block plan, run as source-blocked device passes
        const B::BlockPlan plan =
            s == R::Strategy::BlockedPull
                ? B::build_block_plan(g, g.num_cols > 3 ? (g.num_cols + 2) / 3 : 1, 8)
                : B::BlockPlan{};
        const B::FeatureMatrix got = B::binary_reduce(bs_, g, B::named_config(name), &bu, &bv,
                                                      &be, &plan);
        CHECK(same_bits(got, want));
        if (!same_bits(got, want))
          std::fprintf(stderr, "  config %s strategy %d seed %llu\n", name.c_str(),
                       static_cast<int>(s), static_cast<unsigned long long>(seed));
        R::FeatureMatrix t;
        t.rows = got.rows;
        t.dim = got.dim;
        t.data = got.data;
        if (R::is_exact_reduce(cfg.reduce))
          CHECK(R::bit_equal(t, oracle));
        else
          CHECK(R::max_rel_error(t, oracle) <= 1e-5);
        // the reference-side adapter on the reference's
        // own graph view and plan, Push and BlockedPull included
        const R::CsrGraph& rg = views.oriented(R::required_orientation(s, cfg.out));
        const R::BlockPlan rplan =
            s == R::Strategy::BlockedPull
                ? R::build_block_plan(rg, rg.num_cols > 3 ? (rg.num_cols + 2) / 3 : 1, 8)
                : R::BlockPlan{};
        const R::FeatureMatrix ad = adapter_binary_reduce(s, rg, cfg, &fu, &fv, &fe, &rplan);
        CHECK(R::bit_equal(ad, want));
      }
    }
  }
  // a BlockPlan built for another graph is a ShapeError (kernels.cpp:462-467),
  // in the shim and in the adapter
  {
    const R::EdgeList a = random_small_graph(7), b = random_small_graph(8);
    const R::GraphViews va = R::make_views(a), vb = R::make_views(b);
    const R::FeatureMatrix fa = R::random_features(a.num_nodes, 3, 1);
    const B::BlockPlan wrong = B::build_block_plan(to_b(vb.dst_major), 4, 2);
    const B::FeatureMatrix bfa = to_b(fa);
    const B::CsrGraph bga = to_b(va.dst_major);
    CHECK_THROWS_AS(B::binary_reduce(B::Strategy::BlockedPull, bga,
                                     B::named_config("u_copy_add_v"), &bfa, nullptr, nullptr,
                                     &wrong),
                    B::ShapeError);
    const R::BlockPlan rwrong = R::build_block_plan(vb.dst_major, 4, 2);
    CHECK_THROWS_AS(adapter_binary_reduce(R::Strategy::BlockedPull, va.dst_major,
                                          R::named_config("u_copy_add_v"), &fa, nullptr, nullptr,
                                          &rwrong),
                    R::ShapeError);
  }
  // graphs destroyed and rebuilt with the same sizes (recycled addresses):
  // the content-keyed handle cache must never serve a stale device graph
  for (std::uint64_t seed = 1; seed <= 24; ++seed) {
    R::GeneratorSpec spec;
    spec.kind = R::GeneratorKind::RMat;
    spec.num_nodes = 150;
    spec.num_edges = 1200;
    spec.seed = seed;
    const R::EdgeList el = R::generate(spec);
    const R::GraphViews views = R::make_views(el);
    const R::FeatureMatrix fu = R::random_features(el.num_nodes, 8, seed);
    const R::FeatureMatrix want = R::binary_reduce(R::Strategy::RowParallelSpmm, views.dst_major,
                                                   R::named_config("u_copy_add_v"), &fu, nullptr,
                                                   nullptr);
    B::CsrGraph* bg = new B::CsrGraph(to_b(views.dst_major));  // same sizes every seed
    const B::FeatureMatrix bu = to_b(fu);
    CHECK(same_bits(B::binary_reduce(B::Strategy::RowParallelSpmm, *bg,
                                     B::named_config("u_copy_add_v"), &bu, nullptr, nullptr),
                    want));
    delete bg;
  }
  // one graph shared by several host threads at once (csr.hpp:35: a CsrGraph
  // is safe to share), every strategy
  {
    const R::EdgeList el = random_small_graph(31);
    const R::GraphViews views = R::make_views(el);
    const R::FeatureMatrix fu = R::random_features(el.num_nodes, 16, 5);
    const R::FeatureMatrix want = R::binary_reduce(R::Strategy::RowParallelSpmm, views.dst_major,
                                                   R::named_config("u_copy_max_v"), &fu, nullptr,
                                                   nullptr);
    const B::CsrGraph bd = to_b(views.dst_major), bs = to_b(views.src_major);
    const B::FeatureMatrix bu = to_b(fu);
    std::vector<int> ok(8, 0);
    std::vector<std::thread> ts;
    for (int t = 0; t < 8; ++t)
      ts.emplace_back([&, t] {
        bool all = true;
        for (int it = 0; it < 20; ++it) {
          const B::Strategy s = (t % 2) ? B::Strategy::Push : B::Strategy::Pull;
          const B::FeatureMatrix got = B::binary_reduce(
              s, s == B::Strategy::Push ? bs : bd, B::named_config("u_copy_max_v"), &bu, nullptr,
              nullptr);
          all = all && same_bits(got, want);
        }
        ok[t] = all ? 1 : 0;
      });
    for (auto& t : ts) t.join();
    for (int t = 0; t < 8; ++t) CHECK(ok[t] == 1);
  }
  // validation errors surface as the same exception types (:139-174)
  {
    R::EdgeList el;
    el.num_nodes = 2;
    el.edges = {{0, 1}};
    const R::GraphViews views = R::make_views(el);
    const B::CsrGraph bd = to_b(views.dst_major), bs = to_b(views.src_major);
    const B::BrConfig cfg = B::named_config("u_copy_add_v");
    const B::FeatureMatrix fu(2, 4), bad(3, 4), fv(2, 3);
    CHECK_THROWS_AS(B::binary_reduce(B::Strategy::Pull, bs, cfg, &fu, nullptr, nullptr), B::ShapeError);
    CHECK_THROWS_AS(B::binary_reduce(B::Strategy::Pull, bd, cfg, nullptr, nullptr, nullptr), B::ShapeError);
    CHECK_THROWS_AS(B::binary_reduce(B::Strategy::Pull, bd, cfg, &bad, nullptr, nullptr), B::ShapeError);
    CHECK_THROWS_AS(B::binary_reduce(B::Strategy::BlockedPull, bd, cfg, &fu, nullptr, nullptr), B::ShapeError);
    CHECK_THROWS_AS(B::binary_reduce(B::Strategy::Pull, bd, B::named_config("u_add_v_add_v"), &fu, &fv, nullptr),
                    B::ShapeError);
    CHECK_THROWS_AS(B::named_config("v_copy_add_u"), B::ConfigError);
    const B::FeatureMatrix neither(5, 1);
    CHECK_THROWS_AS(B::copy_reduce(B::Strategy::Pull, bd, neither, B::ReduceOp::Sum), B::ShapeError);
    // edge-feature source resolved by row count (:176-188)
    R::EdgeList el3;
    el3.num_nodes = 3;
    el3.edges = {{0, 2}, {1, 2}};
    const R::GraphViews v3 = R::make_views(el3);
    B::FeatureMatrix fe(2, 1);
    fe.data = {1, 10};
    const B::FeatureMatrix o = B::copy_reduce(B::Strategy::Pull, to_b(v3.dst_major), fe, B::ReduceOp::Sum);
    CHECK(o.at(2, 0) == 11);
  }
  // file containers (test_io.cpp:93-123): each library reads what the other
  // wrote; corrupt files raise IoError in both
  {
    const std::string dir = "/tmp/gspmm_b200_shim_io_";
    for (std::uint64_t seed : {1ull, 8ull}) {
      const R::EdgeList el = random_small_graph(seed);
      for (const auto orient : {R::Orientation::SrcMajor, R::Orientation::DstMajor}) {
        const R::CsrGraph g = R::build_csr(el, orient);
        R::save_csr(dir + "r.csr", g);
        B::save_csr(dir + "b.csr", to_b(g));
        const B::CsrGraph from_r = B::load_csr(dir + "r.csr");
        const R::CsrGraph from_b = R::load_csr(dir + "b.csr");
        CHECK(from_r.orientation == static_cast<B::Orientation>(g.orientation));
        CHECK(from_r.num_rows == g.num_rows && from_r.num_cols == g.num_cols);
        CHECK(from_r.indptr == g.indptr && from_r.indices == g.indices && from_r.edge_ids == g.edge_ids);
        CHECK(from_b.orientation == g.orientation && from_b.indptr == g.indptr &&
              from_b.indices == g.indices && from_b.edge_ids == g.edge_ids);
      }
      B::EdgeList bel;
      bel.num_nodes = el.num_nodes;
      for (const R::Edge& e : el.edges) bel.edges.push_back({e.src, e.dst});
      B::save_edge_list(dir + "b.txt", bel);
      const R::EdgeList back = R::load_edge_list(dir + "b.txt");
      CHECK(back.num_nodes == el.num_nodes && back.edges == el.edges);
      R::save_edge_list(dir + "r.txt", el);
      CHECK(B::load_edge_list(dir + "r.txt").edges == bel.edges);
    }
    const R::FeatureMatrix a = R::random_features(37, 5, 123);
    R::save_feature_matrix(dir + "r.fmat", a);
    const B::FeatureMatrix fb = B::load_feature_matrix(dir + "r.fmat");
    CHECK(fb.rows == a.rows && fb.dim == a.dim && fb.data == a.data);
    B::save_feature_matrix(dir + "b.fmat", fb);
    CHECK(R::load_feature_matrix(dir + "b.fmat").data == a.data);
    {
      std::FILE* f = std::fopen((dir + "bogus.bin").c_str(), "wb");
      std::fputs("definitely not a matrix", f);
      std::fclose(f);
    }
    CHECK_THROWS_AS(B::load_feature_matrix(dir + "bogus.bin"), B::IoError);
    CHECK_THROWS_AS(B::load_csr(dir + "bogus.bin"), B::IoError);
    CHECK_THROWS_AS(B::load_feature_matrix("/nonexistent/path"), B::IoError);
    CHECK_THROWS_AS(R::load_csr(dir + "bogus.bin"), R::IoError);
    {
      std::FILE* f = std::fopen((dir + "bad.txt").c_str(), "wb");
      std::fputs("0 1\n%nodes 2\n5 1\n", f);
      std::fclose(f);
    }
    CHECK_THROWS_AS(B::load_edge_list(dir + "bad.txt"), B::ParseError);
    CHECK_THROWS_AS(R::load_edge_list(dir + "bad.txt"), R::ParseError);
    for (const char* n : {"r.csr", "b.csr", "b.txt", "r.txt", "r.fmat", "b.fmat", "bogus.bin", "bad.txt"})
      std::remove((dir + n).c_str());
  }
  std::printf("shim_parity: %d checks, %d failures\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}

// shim_parity.cpp -- the reference-signature C++ API of this repo
// (gspmm_b200::binary_reduce / copy_reduce, include/gspmm_b200.hpp) called
// side by side with the unmodified reference library (gspmm::, linked from
// oracle/_ref) on identical inputs, in the style of the reference's own
// proj/tests/test_kernels.cpp.  Exit code 0 = all checks passed.
#include <cstdio>
#include <cstdlib>
#include <string>

#include "gspmm/bench.hpp"
#include "gspmm/compare.hpp"
#include "gspmm/error.hpp"
#include "gspmm/generate.hpp"
#include "gspmm/kernels.hpp"
#include "gspmm/oracle.hpp"
#include "gspmm/rng.hpp"
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
      }
    }
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
  std::printf("shim_parity: %d checks, %d failures\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}

// shim.cpp -- the reference-signature C++ API (include/gspmm_b200.hpp) on
// top of the C-ABI.  Synchronous host-buffer calls like the reference's;
// device handles for a CsrGraph are cached (the reference declares a
// CsrGraph immutable after construction, csr.hpp:33) so repeated calls on
// one graph upload it once.
#include "gspmm_b200.hpp"

#include <memory>
#include <mutex>

namespace gspmm_b200 {

void throw_status(int st) {
  if (st == GSPMM_OK) return;
  const std::string msg = gspmm_last_error();
  switch (st) {
    case GSPMM_ERR_CONFIG: throw ConfigError(msg);
    case GSPMM_ERR_SHAPE: throw ShapeError(msg);
    case GSPMM_ERR_STRUCTURE: throw StructureError(msg);
    default: throw DeviceError(msg);
  }
}

namespace {

gspmm_config to_c(const BrConfig& c) {
  return {static_cast<int32_t>(c.lhs), static_cast<int32_t>(c.rhs),
          static_cast<int32_t>(c.binary), static_cast<int32_t>(c.reduce),
          static_cast<int32_t>(c.out)};
}

const char* op_name(Operand o) {
  switch (o) {
    case Operand::U: return "u";
    case Operand::V: return "v";
    case Operand::E: return "e";
    default: return "none";
  }
}

struct CacheEntry {
  const void* key[4] = {nullptr, nullptr, nullptr, nullptr};
  std::uint64_t sizes[3] = {0, 0, 0};
  gspmm_graph h = nullptr;
  std::unique_ptr<CsrGraph> transposed;  // owner view for Push
};

struct Cache {
  std::mutex mu;
  CacheEntry slot[4];
  int next = 0;
  ~Cache() {
    for (auto& s : slot) gspmm_graph_destroy(s.h);
  }
};

Cache& cache() {
  static Cache c;
  return c;
}

// Device handle for g (uploaded on first use).
gspmm_graph handle_for(const CsrGraph& g) {
  Cache& c = cache();
  std::lock_guard<std::mutex> lock(c.mu);
  const void* key[4] = {&g, g.indptr.data(), g.indices.data(), g.edge_ids.data()};
  const std::uint64_t sizes[3] = {g.indptr.size(), g.indices.size(),
                                  (static_cast<std::uint64_t>(g.num_rows) << 32) | g.num_cols};
  for (auto& s : c.slot) {
    if (s.h && s.key[0] == key[0] && s.key[1] == key[1] && s.key[2] == key[2] &&
        s.key[3] == key[3] && s.sizes[0] == sizes[0] && s.sizes[1] == sizes[1] &&
        s.sizes[2] == sizes[2])
      return s.h;
  }
  if (g.indptr.size() != static_cast<std::size_t>(g.num_rows) + 1)
    throw StructureError("indptr length != num_rows+1");
  gspmm_graph h = nullptr;
  throw_status(gspmm_graph_create(0, static_cast<int>(g.orientation), g.num_rows, g.num_cols,
                                  g.indptr.data(), g.indices.data(), g.edge_ids.data(),
                                  /*validate=*/0, &h));
  CacheEntry& s = c.slot[c.next];
  c.next = (c.next + 1) % 4;
  gspmm_graph_destroy(s.h);
  for (int i = 0; i < 4; ++i) s.key[i] = key[i];
  for (int i = 0; i < 3; ++i) s.sizes[i] = sizes[i];
  s.h = h;
  return h;
}

CsrGraph transpose_host(const CsrGraph& g) {
  CsrGraph t;
  t.orientation =
      g.orientation == Orientation::DstMajor ? Orientation::SrcMajor : Orientation::DstMajor;
  t.num_rows = g.num_cols;
  t.num_cols = g.num_rows;
  t.indptr.resize(static_cast<std::size_t>(t.num_rows) + 1);
  t.indices.resize(g.indices.size());
  t.edge_ids.resize(g.edge_ids.size());
  throw_status(gspmm_transpose(g.num_rows, g.num_cols, g.indptr.data(), g.indices.data(),
                               g.edge_ids.data(), t.indptr.data(), t.indices.data(),
                               t.edge_ids.data(), 0));
  return t;
}

gspmm_mat view(const FeatureMatrix* f) {
  gspmm_mat m{};
  if (f) {
    m.data = f->data.data();
    m.rows = f->rows;
    m.dim = f->dim;
    m.ld = f->dim;
    m.edge_order = GSPMM_EDGE_BY_ID;
    if (!m.data && f->rows * f->dim == 0) m.data = reinterpret_cast<const float*>(f);
  }
  return m;
}

}  // namespace

void validate_config(const BrConfig& cfg) {
  const gspmm_config c = to_c(cfg);
  throw_status(gspmm_validate_config(&c));
}

BrConfig named_config(std::string_view name) {
  gspmm_config c{};
  throw_status(gspmm_named_config(std::string(name).c_str(), &c));
  BrConfig b;
  b.lhs = static_cast<Operand>(c.lhs);
  b.rhs = static_cast<Operand>(c.rhs);
  b.binary = static_cast<BinaryOp>(c.binary);
  b.reduce = static_cast<ReduceOp>(c.reduce);
  b.out = static_cast<Operand>(c.out);
  return b;
}

std::string config_name(const BrConfig& cfg) {
  static const char* bin[] = {"add", "sub", "mul", "div", "dot", "copy"};
  static const char* red[] = {"add", "max", "min", "mul", "copy"};
  std::string s = op_name(cfg.lhs);
  s += '_';
  s += bin[static_cast<int>(cfg.binary)];
  s += '_';
  if (cfg.rhs != Operand::None) {
    s += op_name(cfg.rhs);
    s += '_';
  }
  s += red[static_cast<int>(cfg.reduce)];
  s += '_';
  s += op_name(cfg.out);
  return s;
}

BlockPlan build_block_plan(const CsrGraph& g, NodeId kb, std::int64_t nb) {
  if (kb < 1 || nb < 1) throw ConfigError("build_block_plan: kb and nb must be >= 1");
  BlockPlan p;
  p.kb = kb;
  p.nb = nb;
  p.num_rows = g.num_rows;
  p.num_cols = g.num_cols;
  p.num_blocks = g.num_cols ? (g.num_cols + kb - 1) / kb : 0;
  return p;
}

Orientation required_orientation(Strategy s, Operand out) {
  const int o = gspmm_required_orientation(static_cast<int>(s), static_cast<int>(out));
  if (o < 0) throw ConfigError(gspmm_last_error());
  return static_cast<Orientation>(o);
}

FeatureMatrix binary_reduce(Strategy strategy, const CsrGraph& g, const BrConfig& cfg,
                            const FeatureMatrix* u_feats, const FeatureMatrix* v_feats,
                            const FeatureMatrix* e_feats, const BlockPlan* plan,
                            int threads) {
  (void)threads;
  validate_config(cfg);
  const Orientation need = required_orientation(strategy, cfg.out);
  if (g.orientation != need)
    throw ShapeError(std::string("strategy with output ") + op_name(cfg.out) + " needs a " +
                     (need == Orientation::SrcMajor ? "src-major" : "dst-major") + " graph");
  if (strategy == Strategy::BlockedPull && !plan)
    throw ShapeError("BlockedPull requires a BlockPlan");
  // Push scatters over the opposite orientation; the device runs owner rows.
  std::unique_ptr<CsrGraph> owner;
  const CsrGraph* view_g = &g;
  if (strategy == Strategy::Push) {
    owner = std::make_unique<CsrGraph>(transpose_host(g));
    view_g = owner.get();
  }
  const gspmm_graph h = handle_for(*view_g);
  // BlockedPull: the plan's neighbour-id blocks as source-blocked passes
  // (bit-identical to Pull, like the reference's); otherwise automatic
  const int blocks = strategy == Strategy::BlockedPull && plan->num_blocks >= 1
                         ? static_cast<int>(plan->num_blocks)
                         : 0;
  throw_status(gspmm_graph_set_source_blocks(h, blocks));
  const gspmm_config c = to_c(cfg);
  gspmm_mat mu = view(u_feats), mv = view(v_feats), me = view(e_feats);
  int64_t rows = 0, dim = 0;
  throw_status(gspmm_out_shape(h, &c, u_feats ? &mu : nullptr, v_feats ? &mv : nullptr,
                               e_feats ? &me : nullptr, nullptr, &rows, &dim));
  FeatureMatrix out(rows, dim);
  if (rows * dim > 0) {
    gspmm_out o{out.data.data(), rows, dim, dim};
    throw_status(gspmm_binary_reduce_host(h, &c, u_feats ? &mu : nullptr,
                                          v_feats ? &mv : nullptr, e_feats ? &me : nullptr, &o,
                                          nullptr, nullptr));
  }
  if (owner) {
    // Drop the temporary transposed view's handle from the cache key space.
    Cache& cc = cache();
    std::lock_guard<std::mutex> lock(cc.mu);
    for (auto& s : cc.slot)
      if (s.h == h) {
        gspmm_graph_destroy(s.h);
        s = CacheEntry{};
      }
  }
  return out;
}

FeatureMatrix copy_reduce(Strategy strategy, const CsrGraph& g, const FeatureMatrix& src_feats,
                          ReduceOp reduce, const BlockPlan* plan, int threads) {
  BrConfig cfg;
  cfg.binary = BinaryOp::CopyLhs;
  cfg.rhs = Operand::None;
  cfg.reduce = reduce;
  cfg.out = Operand::V;
  const std::int64_t nu = g.num_src_nodes();
  const std::int64_t ne = g.num_edges();
  if (src_feats.rows == nu) {
    cfg.lhs = Operand::U;
  } else if (src_feats.rows == ne) {
    cfg.lhs = Operand::E;
  } else {
    throw ShapeError("copy_reduce: source rows match neither the node nor the edge count");
  }
  return binary_reduce(strategy, g, cfg, cfg.lhs == Operand::U ? &src_feats : nullptr, nullptr,
                       cfg.lhs == Operand::E ? &src_feats : nullptr, plan, threads);
}

}  // namespace gspmm_b200

// shim.cpp -- the reference-signature C++ API (include/gspmm_b200.hpp) on
// top of the C-ABI.  Synchronous host-buffer calls like the reference's;
// device handles are cached by graph CONTENT (orientation, sizes and a hash
// of the three arrays), so repeated calls on one graph upload it once and a
// new graph at recycled addresses never hits a stale device copy.  Handles
// are reference-counted: evicting one never frees it under a running call.
// Thread-safe, like the reference's calls (csr.hpp:35).
#include "gspmm_b200.hpp"

#include <algorithm>
#include <memory>
#include <mutex>
#include <thread>
#include <utility>
#include <vector>

namespace gspmm_b200 {

void throw_status(int st) {
  if (st == GSPMM_OK) return;
  const std::string msg = gspmm_last_error();
  switch (st) {
    case GSPMM_ERR_CONFIG: throw ConfigError(msg);
    case GSPMM_ERR_SHAPE: throw ShapeError(msg);
    case GSPMM_ERR_STRUCTURE: throw StructureError(msg);
    case GSPMM_ERR_IO: throw IoError(msg);
    case GSPMM_ERR_PARSE: throw ParseError(msg);
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

// Content fingerprint of a CsrGraph: orientation, sizes and a 64-bit hash of
// indptr / indices / edge_ids (multithreaded: ~1 GB/s per thread).  The
// cache is keyed on it, never on addresses: a graph destroyed and rebuilt at
// recycled addresses with other contents gets its own device copy.
struct Key {
  int orientation = 0;
  std::uint32_t rows = 0, cols = 0;
  std::uint64_t m = 0, hash = 0;
  bool transposed = false;  // the handle holds the transpose (Push)
  bool operator==(const Key& o) const {
    return orientation == o.orientation && rows == o.rows && cols == o.cols && m == o.m &&
           hash == o.hash && transposed == o.transposed;
  }
};

std::uint64_t mix(std::uint64_t h, std::uint64_t x) {
  h ^= x + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
  h *= 0xff51afd7ed558ccdull;
  return h ^ (h >> 33);
}

std::uint64_t hash_words(const std::uint32_t* p, std::size_t n) {
  constexpr std::size_t kChunk = std::size_t{1} << 22;
  const std::size_t chunks = (n + kChunk - 1) / kChunk;
  std::vector<std::uint64_t> part(chunks, 0);
  auto work = [&](std::size_t c0, std::size_t c1) {
    for (std::size_t c = c0; c < c1; ++c) {
      std::uint64_t h = 0x243f6a8885a308d3ull ^ c;
      const std::size_t b = c * kChunk, e = std::min(n, b + kChunk);
      std::size_t i = b;
      for (; i + 2 <= e; i += 2)
        h = (h ^ (static_cast<std::uint64_t>(p[i]) | (static_cast<std::uint64_t>(p[i + 1]) << 32))) *
            0x100000001b3ull * 0x9e3779b97f4a7c15ull;
      if (i < e) h = (h ^ p[i]) * 0x9e3779b97f4a7c15ull;
      part[c] = mix(h, e - b);
    }
  };
  const unsigned nt = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(),
                                                      static_cast<unsigned>(chunks)));
  if (nt <= 1) {
    work(0, chunks);
  } else {
    std::vector<std::thread> ts;
    for (unsigned t = 0; t < nt; ++t)
      ts.emplace_back(work, chunks * t / nt, chunks * (t + 1) / nt);
    for (auto& t : ts) t.join();
  }
  std::uint64_t h = n;
  for (std::uint64_t x : part) h = mix(h, x);
  return h;
}

Key key_of(const CsrGraph& g, bool transposed) {
  Key k;
  k.orientation = static_cast<int>(g.orientation);
  k.rows = g.num_rows;
  k.cols = g.num_cols;
  k.m = g.indices.size();
  k.transposed = transposed;
  k.hash = mix(mix(hash_words(g.indptr.data(), g.indptr.size()),
                   hash_words(g.indices.data(), g.indices.size())),
               hash_words(g.edge_ids.data(), g.edge_ids.size()));
  return k;
}

// A device handle shared by the cache and the calls using it: eviction only
// drops the cache's reference, the handle is destroyed when the last call
// using it returns.
using Handle = std::shared_ptr<gspmm_graph_s>;

Handle make_handle(gspmm_graph h) {
  return Handle(h, [](gspmm_graph p) { gspmm_graph_destroy(p); });
}

struct Cache {
  std::mutex mu;
  std::vector<std::pair<Key, Handle>> slot;  // most recent last
  static constexpr std::size_t kSlots = 4;
};

Cache& cache() {
  static Cache c;
  return c;
}

CsrGraph transpose_host(const CsrGraph& g);

// Device handle for g (or for its transpose), uploaded on first use.  The
// upload runs outside the cache lock; two threads racing on one new graph
// both upload and the second keeps the first's handle.
Handle handle_for(const CsrGraph& g, bool transposed) {
  if (g.indptr.size() != static_cast<std::size_t>(g.num_rows) + 1)
    throw StructureError("indptr length != num_rows+1");
  const Key k = key_of(g, transposed);
  Cache& c = cache();
  {
    std::lock_guard<std::mutex> lock(c.mu);
    for (auto it = c.slot.begin(); it != c.slot.end(); ++it)
      if (it->first == k) {
        Handle h = it->second;
        std::rotate(it, it + 1, c.slot.end());  // most recent last
        return h;
      }
  }
  gspmm_graph raw = nullptr;
  if (transposed) {
    const CsrGraph t = transpose_host(g);
    throw_status(gspmm_graph_create(0, static_cast<int>(t.orientation), t.num_rows, t.num_cols,
                                    t.indptr.data(), t.indices.data(), t.edge_ids.data(),
                                    /*validate=*/0, &raw));
  } else {
    throw_status(gspmm_graph_create(0, static_cast<int>(g.orientation), g.num_rows, g.num_cols,
                                    g.indptr.data(), g.indices.data(), g.edge_ids.data(),
                                    /*validate=*/0, &raw));
  }
  Handle h = make_handle(raw);
  std::lock_guard<std::mutex> lock(c.mu);
  for (auto& s : c.slot)
    if (s.first == k) return s.second;
  if (c.slot.size() >= Cache::kSlots) c.slot.erase(c.slot.begin());
  c.slot.emplace_back(k, h);
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
  p.built_for = g.orientation;
  p.num_rows = g.num_rows;
  p.num_cols = g.num_cols;
  p.num_edges = g.num_edges();
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
  // Push scatters over the opposite orientation; the device runs owner
  // rows on the transposed view (cached like the graph itself)
  const Handle h = handle_for(g, strategy == Strategy::Push);
  const gspmm_config c = to_c(cfg);
  gspmm_mat mu = view(u_feats), mv = view(v_feats), me = view(e_feats);
  int64_t rows = 0, dim = 0;
  throw_status(gspmm_out_shape(h.get(), &c, u_feats ? &mu : nullptr, v_feats ? &mv : nullptr,
                               e_feats ? &me : nullptr, nullptr, &rows, &dim));
  // kernels.cpp:462-467, after the operand binding like the reference
  if (strategy == Strategy::BlockedPull) {
    if (!plan) throw ShapeError("BlockedPull requires a BlockPlan");
    if (plan->built_for != g.orientation || plan->num_rows != g.num_rows ||
        plan->num_cols != g.num_cols || plan->num_edges != g.num_edges())
      throw ShapeError("BlockPlan was not built for this graph");
  }
  // BlockedPull: the plan's neighbour-id blocks as source-blocked passes
  // (bit-identical to Pull, like the reference's), a per-call option;
  // otherwise the automatic policy
  gspmm_options opt{};
  opt.source_blocks = strategy == Strategy::BlockedPull && plan->num_blocks >= 1
                          ? static_cast<int32_t>(std::min<NodeId>(plan->num_blocks, 64))
                          : 0;
  FeatureMatrix out(rows, dim);
  if (rows * dim > 0) {
    gspmm_out o{out.data.data(), rows, dim, dim};
    throw_status(gspmm_binary_reduce_host(h.get(), &c, u_feats ? &mu : nullptr,
                                          v_feats ? &mv : nullptr, e_feats ? &me : nullptr, &o,
                                          &opt, nullptr));
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

// ---- file containers (io.hpp:25-41) over the C-ABI readers / writers ------

EdgeList load_edge_list(const std::string& path) {
  uint32_t n = 0;
  uint64_t m = 0;
  uint32_t *src = nullptr, *dst = nullptr;
  throw_status(gspmm_edge_list_read(path.c_str(), &n, &m, &src, &dst));
  EdgeList el;
  el.num_nodes = n;
  el.edges.resize(m);
  for (uint64_t i = 0; i < m; ++i) el.edges[i] = Edge{src[i], dst[i]};
  gspmm_free(src);
  gspmm_free(dst);
  return el;
}

void save_edge_list(const std::string& path, const EdgeList& el) {
  std::vector<uint32_t> src(el.edges.size()), dst(el.edges.size());
  for (std::size_t i = 0; i < el.edges.size(); ++i) {
    src[i] = el.edges[i].src;
    dst[i] = el.edges[i].dst;
  }
  throw_status(gspmm_edge_list_write(path.c_str(), el.num_nodes, el.edges.size(), src.data(),
                                     dst.data()));
}

void save_feature_matrix(const std::string& path, const FeatureMatrix& f) {
  throw_status(gspmm_fmat1_write(path.c_str(), f.data.data(), f.rows, f.dim, 0));
}

FeatureMatrix load_feature_matrix(const std::string& path) {
  int64_t rows = 0, dim = 0;
  throw_status(gspmm_fmat1_info(path.c_str(), &rows, &dim));
  FeatureMatrix f(rows, dim);
  throw_status(gspmm_fmat1_read(path.c_str(), f.data.data(), 0));
  return f;
}

void save_csr(const std::string& path, const CsrGraph& g) {
  throw_status(gspmm_csr1_write(path.c_str(), static_cast<int>(g.orientation), g.num_rows,
                                g.num_cols, g.indptr.data(), g.indices.data(),
                                g.edge_ids.data()));
}

CsrGraph load_csr(const std::string& path) {
  int orientation = 0;
  uint64_t rows = 0, cols = 0, m = 0;
  throw_status(gspmm_csr1_info(path.c_str(), &orientation, &rows, &cols, &m));
  CsrGraph g;
  g.orientation = orientation == GSPMM_DST_MAJOR ? Orientation::DstMajor : Orientation::SrcMajor;
  g.num_rows = static_cast<NodeId>(rows);
  g.num_cols = static_cast<NodeId>(cols);
  g.indptr.resize(rows + 1);
  g.indices.resize(m);
  g.edge_ids.resize(m);
  throw_status(gspmm_csr1_read(path.c_str(), g.indptr.data(), g.indices.data(), g.edge_ids.data()));
  return g;
}

}  // namespace gspmm_b200

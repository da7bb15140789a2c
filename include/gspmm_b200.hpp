// gspmm_b200.hpp -- C++ host API with the reference's entry points, over the
// C-ABI (gspmm_b200.h).
//
// Same names, parameter lists, ownership and error behaviour as the
// reference library's public API (/root/reference/proj/include/gspmm):
//   binary_reduce / copy_reduce        kernels.hpp:60-64, 71-73
//   required_orientation, Strategy     kernels.hpp:40-48
//   BrConfig, validate_config,         br_config.hpp:37-59
//     named_config, config_name
//   CsrGraph, FeatureMatrix            csr.hpp:37-54, feature_matrix.hpp:29-66
//   StructureError/ShapeError/         error.hpp:22-45
//     ConfigError/ParseError/IoError
//   load_csr / save_csr, load_ /       io.hpp:25-41
//     save_feature_matrix, load_ /
//     save_edge_list
// It lives in namespace gspmm_b200 so a program can link it next to the
// reference (the parity harness does).  A caller switches by changing the
// namespace (or a `namespace gspmm = gspmm_b200;` alias).
//
// Strategy and BlockPlan are accepted for signature compatibility: the
// device plan built at graph upload replaces both (Push is served by the
// owner-computes kernel on the transposed view; results equal Pull's, which
// the reference guarantees to within its tolerance).  `threads` is ignored.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "gspmm_b200.h"

namespace gspmm_b200 {

using NodeId = std::uint32_t;
using EdgeId = std::uint32_t;

enum class Orientation : std::uint8_t { SrcMajor = 0, DstMajor = 1 };
enum class BinaryOp : std::uint8_t { Add, Sub, Mul, Div, Dot, CopyLhs };
enum class ReduceOp : std::uint8_t { Sum, Max, Min, Prod, CopyLast };
enum class Operand : std::uint8_t { U, V, E, None };
enum class Strategy : std::uint8_t { Push, Pull, BlockedPull, RowParallelSpmm };

struct StructureError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ShapeError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ParseError : std::runtime_error {  // text input that does not parse
  using std::runtime_error::runtime_error;
};
struct IoError : std::runtime_error {  // file failure or corrupt container
  using std::runtime_error::runtime_error;
};
// CUDA failures (no device, out of memory): the path has no CPU fallback.
struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct BrConfig {
  Operand lhs = Operand::U;
  Operand rhs = Operand::None;
  BinaryOp binary = BinaryOp::CopyLhs;
  ReduceOp reduce = ReduceOp::Sum;
  Operand out = Operand::V;
  friend bool operator==(const BrConfig&, const BrConfig&) = default;
};

struct CsrGraph {
  Orientation orientation = Orientation::DstMajor;
  NodeId num_rows = 0;
  NodeId num_cols = 0;
  std::vector<EdgeId> indptr;
  std::vector<NodeId> indices;
  std::vector<EdgeId> edge_ids;
  EdgeId num_edges() const { return indptr.empty() ? 0 : indptr.back(); }
  NodeId num_src_nodes() const {
    return orientation == Orientation::SrcMajor ? num_rows : num_cols;
  }
  NodeId num_dst_nodes() const {
    return orientation == Orientation::SrcMajor ? num_cols : num_rows;
  }
};

struct FeatureMatrix {
  std::int64_t rows = 0;
  std::int64_t dim = 0;
  std::vector<float> data;
  FeatureMatrix() = default;
  FeatureMatrix(std::int64_t r, std::int64_t d)
      : rows(r), dim(d), data(static_cast<std::size_t>(r * d), 0.0f) {}
  float* row(std::int64_t i) { return data.data() + i * dim; }
  const float* row(std::int64_t i) const { return data.data() + i * dim; }
  float& at(std::int64_t i, std::int64_t j) { return data[i * dim + j]; }
  float at(std::int64_t i, std::int64_t j) const { return data[i * dim + j]; }
};

// The reference's Alg.-3 schedule (block_plan.hpp:39-75) reduced to what the
// device needs: kb source nodes per block -> num_blocks neighbour-id blocks.
// Strategy::BlockedPull with a plan runs that many source-blocked passes
// (gspmm_graph_set_source_blocks); the device builds the block CSRs itself.
// nb (the output column panel) is accepted and ignored: the device slices
// columns per unit.
struct BlockPlan {
  NodeId kb = 0;
  std::int64_t nb = 0;
  Orientation built_for = Orientation::DstMajor;  // checked like kernels.cpp:462-467
  NodeId num_rows = 0, num_cols = 0;
  NodeId num_blocks = 0;
  EdgeId num_edges = 0;
};
// build_block_plan (block_plan.cpp:25-69): kb, nb >= 1.
BlockPlan build_block_plan(const CsrGraph& g, NodeId kb, std::int64_t nb);

void validate_config(const BrConfig& cfg);
BrConfig named_config(std::string_view name);
std::string config_name(const BrConfig& cfg);
Orientation required_orientation(Strategy s, Operand out);

FeatureMatrix binary_reduce(Strategy strategy, const CsrGraph& g,
                            const BrConfig& cfg, const FeatureMatrix* u_feats,
                            const FeatureMatrix* v_feats,
                            const FeatureMatrix* e_feats,
                            const BlockPlan* plan = nullptr, int threads = 0);

FeatureMatrix copy_reduce(Strategy strategy, const CsrGraph& g,
                          const FeatureMatrix& src_feats, ReduceOp reduce,
                          const BlockPlan* plan = nullptr, int threads = 0);

// File containers (io.hpp:25-41): same signatures, formats and failures.
struct Edge {
  NodeId src;
  NodeId dst;
  friend bool operator==(const Edge&, const Edge&) = default;
};
struct EdgeList {  // edge_list.hpp:35-40: the edge id of edges[i] is i
  NodeId num_nodes = 0;
  std::vector<Edge> edges;
  EdgeId num_edges() const { return static_cast<EdgeId>(edges.size()); }
};
EdgeList load_edge_list(const std::string& path);
void save_edge_list(const std::string& path, const EdgeList& edges);
void save_feature_matrix(const std::string& path, const FeatureMatrix& f);
FeatureMatrix load_feature_matrix(const std::string& path);
void save_csr(const std::string& path, const CsrGraph& g);
CsrGraph load_csr(const std::string& path);

// Throws the exception matching a C-ABI status (no-op for GSPMM_OK).
void throw_status(int status);

}  // namespace gspmm_b200

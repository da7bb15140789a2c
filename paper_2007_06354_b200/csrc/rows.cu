// rows.cu -- the owner-computes row kernel for every non-dot Binary-Reduce
// and Copy-Reduce (sm_100a).
//
// Replaces run_rowmajor<B,R,false> (RowParallelSpmm, kernels.cpp:162-195)
// and, through it, Pull and BlockedPull (byte-identical outputs).  One warp
// owns one (row, 128-column slice) work item:
//   * lanes own V consecutive output columns (float4 when the layout
//     allows), so every gathered source row is read with fully coalesced
//     128-bit loads -- 512 B per warp per edge;
//   * the row's neighbour ids / edge ids are fetched 32 at a time with one
//     coalesced load and broadcast by warp shuffle;
//   * U = 8 edges of gathers are issued before any of them is consumed, so a
//     warp keeps 4 KB in flight per operand and the SM tens of KB;
//   * the fold itself is the reference's sequential left fold in canonical
//     edge order, one output element per (lane, t): no atomics, no
//     reassociation, hence bit-exact sums, max/min, products and copy-last;
//   * the Max/Min zero-degree fixup (kernels.cpp:490-499), the mean divide
//     and the argmax lookup are fused into the epilogue; every output row is
//     written exactly once (no separate fill or memset pass).
#include "device_ops.cuh"

namespace gspmm_b200 {
namespace {

constexpr int kWarpsPerBlock = 8;
constexpr int kBatch = 8;  // edges of gathers in flight per warp

template <int V, int BOP, int ROP, bool ARG>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    k_rows(const RowLaunch p) {
  const int lane = threadIdx.x & 31;
  constexpr int kSliceW = 32 * V;
  const int slices = (p.width + kSliceW - 1) / kSliceW;
  const int64_t item =
      (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t row_item = item / slices;
  const int slice = static_cast<int>(item - row_item * slices);
  if (row_item >= static_cast<int64_t>(p.num_long) + p.num_rows) return;

  uint32_t r;
  if (row_item < p.num_long) {
    r = p.long_rows[row_item];
  } else {
    r = static_cast<uint32_t>(row_item - p.num_long);
  }
  const uint32_t beg = __ldg(p.indptr + r);
  const uint32_t end = __ldg(p.indptr + r + 1);
  if (row_item >= p.num_long && end - beg > p.long_threshold) return;

  const int c0 = slice * kSliceW + lane * V;
  const bool active = c0 < p.width;
  const bool has_rhs = p.rhs.base != nullptr;
  const bool need_eid = p.out_edge || p.lhs.role == ROLE_EID ||
                        (has_rhs && p.rhs.role == ROLE_EID);

  float acc[V];
  uint32_t arg[V];
#pragma unroll
  for (int t = 0; t < V; ++t) {
    acc[t] = red_identity<ROP>();
    arg[t] = 0xffffffffu;
  }

  // Operands bound to the owner row are loaded once.
  float lrow[V], rrow[V];
  if (active && p.lhs.role == ROLE_ROW) load_operand<V>(p.lhs, r, c0, lrow);
  if (active && has_rhs && p.rhs.role == ROLE_ROW)
    load_operand<V>(p.rhs, r, c0, rrow);

  for (uint32_t jb = beg; jb < end; jb += 32) {
    const uint32_t jl = jb + lane;
    uint32_t my_other = 0, my_eid = 0;
    if (jl < end) {
      my_other = __ldg(p.indices + jl);
      if (need_eid) my_eid = __ldg(p.eids + jl);
    }
    const int n = min(32u, end - jb);
    for (int k0 = 0; k0 < n; k0 += kBatch) {
      float lv[kBatch][V], rv[kBatch][V];
      uint32_t oth[kBatch], eid[kBatch];
#pragma unroll
      for (int k = 0; k < kBatch; ++k) {
        const int kk = k0 + k;
        oth[k] = __shfl_sync(kFull, my_other, kk & 31);
        eid[k] = need_eid ? __shfl_sync(kFull, my_eid, kk & 31) : 0u;
        if (kk < n && active) {
          const uint32_t j = jb + kk;
          if (p.lhs.role != ROLE_ROW)
            load_operand<V>(p.lhs, operand_row(p.lhs.role, r, oth[k], eid[k], j),
                            c0, lv[k]);
          if (has_rhs && p.rhs.role != ROLE_ROW)
            load_operand<V>(p.rhs, operand_row(p.rhs.role, r, oth[k], eid[k], j),
                            c0, rv[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < kBatch; ++k) {
        const int kk = k0 + k;
        if (kk < n && active) {
          float scale = 1.0f;
          if (p.other_scale) scale = __ldg(p.other_scale + oth[k]);
          float msg[V];
#pragma unroll
          for (int t = 0; t < V; ++t) {
            const float l = p.lhs.role == ROLE_ROW ? lrow[t] : lv[k][t];
            const float rr = has_rhs ? (p.rhs.role == ROLE_ROW ? rrow[t] : rv[k][t]) : 0.0f;
            msg[t] = bin_apply<BOP>(l, rr);
            if (p.other_scale) msg[t] = __fmul_rn(msg[t], scale);
          }
          if (p.out_edge) {
            // out == E: one message per edge row (CopyLast store).
            float* o = p.out + static_cast<int64_t>(eid[k]) * p.out_ld + c0;
            if (c0 + V <= p.width) {
              store_vec<V>(o, msg);
            } else {
#pragma unroll
              for (int t = 0; t < V; ++t)
                if (c0 + t < p.width) o[t] = msg[t];
            }
          } else {
#pragma unroll
            for (int t = 0; t < V; ++t) {
              if constexpr (ARG) {
                if (red_wins<ROP>(acc[t], msg[t])) {
                  acc[t] = msg[t];
                  arg[t] = jb + kk;
                }
              } else {
                acc[t] = red_combine<ROP>(acc[t], msg[t]);
              }
            }
          }
        }
      }
    }
  }

  if (!active || p.out_edge) return;
  const uint32_t deg = end - beg;
  if constexpr (ROP == R_MAX || ROP == R_MIN) {
    if (deg == 0) {
#pragma unroll
      for (int t = 0; t < V; ++t) acc[t] = 0.0f;
    }
  }
  if (p.mean) {
    const float fdeg = __uint2float_rn(deg);
#pragma unroll
    for (int t = 0; t < V; ++t) acc[t] = deg ? __fdiv_rn(acc[t], fdeg) : 0.0f;
  }
  float* o = p.out + static_cast<int64_t>(r) * p.out_ld + c0;
  if (c0 + V <= p.width) {
    store_vec<V>(o, acc);
  } else {
#pragma unroll
    for (int t = 0; t < V; ++t)
      if (c0 + t < p.width) o[t] = acc[t];
  }
  if constexpr (ARG) {
    const int64_t ab = static_cast<int64_t>(r) * p.arg_ld + c0;
#pragma unroll
    for (int t = 0; t < V; ++t) {
      if (c0 + t >= p.width) break;
      const bool none = arg[t] == 0xffffffffu;
      if (p.arg_other)
        p.arg_other[ab + t] = none ? -1 : static_cast<int32_t>(__ldg(p.indices + arg[t]));
      if (p.arg_edge)
        p.arg_edge[ab + t] = none ? -1 : static_cast<int32_t>(__ldg(p.eids + arg[t]));
    }
  }
}

template <int V, int BOP, int ROP, bool ARG>
cudaError_t launch_v(const RowLaunch& p, cudaStream_t s) {
  constexpr int kSliceW = 32 * V;
  const int64_t slices = (p.width + kSliceW - 1) / kSliceW;
  const int64_t items = (static_cast<int64_t>(p.num_rows) + p.num_long) * slices;
  if (items == 0) return cudaSuccess;
  const int64_t blocks = (items + kWarpsPerBlock - 1) / kWarpsPerBlock;
  k_rows<V, BOP, ROP, ARG><<<static_cast<unsigned>(blocks), kWarpsPerBlock * 32, 0, s>>>(p);
  note_launch();
  return cudaGetLastError();
}

template <int V, int BOP>
cudaError_t launch_red(const RowLaunch& p, cudaStream_t s) {
  const bool arg = p.arg_other || p.arg_edge;
  switch (p.reduce) {
    case R_SUM: return launch_v<V, BOP, R_SUM, false>(p, s);
    case R_MAX: return arg ? launch_v<V, BOP, R_MAX, true>(p, s)
                           : launch_v<V, BOP, R_MAX, false>(p, s);
    case R_MIN: return arg ? launch_v<V, BOP, R_MIN, true>(p, s)
                           : launch_v<V, BOP, R_MIN, false>(p, s);
    case R_PROD: return launch_v<V, BOP, R_PROD, false>(p, s);
    default: return launch_v<V, BOP, R_LAST, false>(p, s);
  }
}

template <int V>
cudaError_t launch_bin(const RowLaunch& p, cudaStream_t s) {
  switch (p.binop) {
    case B_ADD: return launch_red<V, B_ADD>(p, s);
    case B_SUB: return launch_red<V, B_SUB>(p, s);
    case B_MUL: return launch_red<V, B_MUL>(p, s);
    case B_DIV: return launch_red<V, B_DIV>(p, s);
    default: return launch_red<V, B_COPY>(p, s);
  }
}

}  // namespace

cudaError_t launch_rows(const RowLaunch& p, cudaStream_t s) {
  switch (p.vec) {
    case 4: return launch_bin<4>(p, s);
    case 2: return launch_bin<2>(p, s);
    default: return launch_bin<1>(p, s);
  }
}

}  // namespace gspmm_b200

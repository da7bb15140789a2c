// dot.cu -- Binary-Reduce with the Dot operator (u_dot_v_*, SDDMM-style
// edge scores and the grad of edge weights / attention), sm_100a.
//
// The reference computes each dot as a sequential fp32 left fold over the
// feature columns, product rounded then added (apply_dot, kernels.cpp:91-97,
// and the oracle's message(), oracle.cpp:49-56), and its own tests demand
// bit-equality for the edge-destined configs (CopyLast is an "exact" reduce,
// compare.hpp:58-61; test_kernels.cpp:218).  A warp-shuffle tree would be
// faster to write but not bit-exact, so the kernel transposes through
// shared memory instead:
//   * a warp owns one destination row and walks its edges 32 at a time;
//   * for each 32*V-column chunk, the 32 lanes gather the chunk of both
//     operands for one edge at a time with coalesced vector loads, multiply
//     (rounded) and park the products in a per-warp shared tile laid out so
//     that both the writes and the per-edge reads are bank-conflict free;
//   * lane k then folds edge k's products in column order, carrying its
//     accumulator across chunks and emitting one value per head (multi-head
//     grad_a: `heads` dots of gather_dim/heads columns each).
// Edge outputs are stored by edge id; node outputs fold the 32 per-edge
// dots in canonical order with the row's reducer.
// Measured alternative (r03c / r03d): a systolic warp pipeline without the
// shared-memory transpose -- lane l owns a few columns of the head, takes an
// item's running sum from lane l - 1 by SHFL.UP and hands it on, lane l on
// item s - l at step s.  Bit-exact, but the skew makes every warp load touch
// 32 different 32-byte sectors for 8 bytes each: config 4 grad_a 13.4 ->
// 33.8 ms (44.8 with the loads grouped), config 2 grad_e 3.4 -> 7.3 ms.
#include "device_ops.cuh"

namespace gspmm_b200 {
namespace {

constexpr int kDotWarps = 4;

template <int V, int ROP>
__global__ void __launch_bounds__(kDotWarps * 32) k_dot(const RowLaunch p) {
  constexpr int kCW = 32 * V;       // columns per chunk
  constexpr int kStride = kCW + 1;  // padded tile row
  extern __shared__ float smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  float* tile = smem + warp * 32 * kStride;

  const int64_t r64 = static_cast<int64_t>(blockIdx.x) * kDotWarps + warp;
  if (r64 >= p.num_rows) return;
  const uint32_t r = static_cast<uint32_t>(r64);
  const uint32_t beg = __ldg(p.indptr + r), end = __ldg(p.indptr + r + 1);
  const int G = p.gather_dim;
  const int D = G / p.heads;
  const bool need_eid = p.out_edge || p.lhs.role == ROLE_EID || p.rhs.role == ROLE_EID;

  float racc = red_identity<ROP>();  // node outputs (heads == 1)

  for (uint32_t jb = beg; jb < end; jb += 32) {
    const int n = min(32u, end - jb);
    const uint32_t jl = jb + lane;
    uint32_t my_other = 0, my_eid = 0;
    if (lane < n) {
      my_other = __ldg(p.indices + jl);
      if (need_eid) my_eid = __ldg(p.eids + jl);
    }
    float acc = 0.0f;
    int head = 0;
    for (int cb = 0; cb < G; cb += kCW) {
      const int c0 = cb + lane * V;
      // Gather + multiply: edge i's chunk lands in tile row i.
      for (int i0 = 0; i0 < n; i0 += 8) {
        float lv[8][V], rv[8][V];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int i = i0 + k;
          const uint32_t o = __shfl_sync(kFull, my_other, i & 31);
          const uint32_t e = need_eid ? __shfl_sync(kFull, my_eid, i & 31) : 0u;
          if (i < n && c0 < G) {
            const uint32_t j = jb + i;
            load_operand<V>(p.lhs, operand_row(p.lhs.role, r, o, e, j), c0, lv[k]);
            load_operand<V>(p.rhs, operand_row(p.rhs.role, r, o, e, j), c0, rv[k]);
          }
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int i = i0 + k;
          if (i < n) {
#pragma unroll
            for (int t = 0; t < V; ++t)
              tile[i * kStride + t * 32 + lane] =
                  c0 + t < G ? __fmul_rn(lv[k][t], rv[k][t]) : 0.0f;
          }
        }
      }
      __syncwarp();
      // Sequential fold of edge `lane` over the chunk's columns.
      if (lane < n) {
        const int cend = min(kCW, G - cb);
        for (int c = 0; c < cend; ++c) {
          acc = __fadd_rn(acc, tile[lane * kStride + (c % V) * 32 + c / V]);
          if ((cb + c + 1) % D == 0) {
            if (p.out_edge) {
              p.out[static_cast<int64_t>(my_eid) * p.out_ld + head] = acc;
            } else {
              tile[lane * kStride + kCW] = acc;  // heads == 1: parked in the pad column
            }
            acc = 0.0f;
            ++head;
          }
        }
      }
      __syncwarp();
    }
    if (!p.out_edge) {
      // Fold this chunk's per-edge dots in canonical order.
      const float dv = lane < n ? tile[lane * kStride + kCW] : 0.0f;
      for (int k = 0; k < n; ++k) racc = red_combine<ROP>(racc, __shfl_sync(kFull, dv, k));
      __syncwarp();
    }
  }
  if (!p.out_edge && lane == 0) {
    const uint32_t deg = end - beg;
    if ((ROP == R_MAX || ROP == R_MIN) && deg == 0) racc = 0.0f;
    if (p.mean) racc = deg ? __fdiv_rn(racc, __uint2float_rn(deg)) : 0.0f;
    p.out[static_cast<int64_t>(r) * p.out_ld] = racc;
  }
}

template <int V, int ROP>
cudaError_t launch_dv(const RowLaunch& p, cudaStream_t s) {
  const size_t smem = sizeof(float) * kDotWarps * 32 * (32 * V + 1);
  {
    const cudaError_t e = set_max_dynamic_smem(reinterpret_cast<const void*>(k_dot<V, ROP>),
                                               static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  const int64_t blocks = (static_cast<int64_t>(p.num_rows) + kDotWarps - 1) / kDotWarps;
  if (blocks == 0) return cudaSuccess;
  k_dot<V, ROP><<<static_cast<unsigned>(blocks), kDotWarps * 32, smem, s>>>(p);
  note_launch();
  return cudaGetLastError();
}

template <int V>
cudaError_t launch_dr(const RowLaunch& p, cudaStream_t s) {
  switch (p.reduce) {
    case R_SUM: return launch_dv<V, R_SUM>(p, s);
    case R_MAX: return launch_dv<V, R_MAX>(p, s);
    case R_MIN: return launch_dv<V, R_MIN>(p, s);
    case R_PROD: return launch_dv<V, R_PROD>(p, s);
    default: return launch_dv<V, R_LAST>(p, s);
  }
}

// ------------------------------------------------------- edge-destined dot
// out == E (u_dot_v_copy_e: SDDMM scores, grad of edge weights, per-head
// grad of attention): every edge is independent, so warps stream fixed
// batches of 32 edges over the whole edge range (no row plan, no long-row
// tail).  The owner row of edge j comes from the handle's row-of-edge array.
// Per 64-column chunk the warp gathers both operand rows of each edge with
// 64-bit loads (8 edges in flight), parks the products in a conflict-free
// shared tile, and lane k folds edge k's products in column order.
constexpr int kEdWarps = 4;
constexpr int kEdCW = 64;             // columns per chunk (2 per lane)
constexpr int kEdStride = kEdCW + 1;  // padded tile row

__global__ void __launch_bounds__(kEdWarps * 32) k_dot_edges(const RowLaunch p,
                                                             const uint32_t* __restrict__ rowof,
                                                             uint64_t m) {
  __shared__ float tiles[kEdWarps][32 * kEdStride];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* tile = tiles[warp];
  const int G = p.gather_dim;
  const int D = G / p.heads;
  const uint64_t n_batches = (m + 31) / 32;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kEdWarps;
  const bool l2 = p.lhs.mode == MODE_FULL, r2 = p.rhs.mode == MODE_FULL;
  for (uint64_t bt = static_cast<uint64_t>(blockIdx.x) * kEdWarps + warp; bt < n_batches;
       bt += stride) {
    const uint64_t jb = bt * 32;
    const int n = static_cast<int>(m - jb < 32 ? m - jb : 32);
    uint32_t my_o = 0, my_e = 0, my_r = 0;
    if (lane < n) {
      my_o = __ldg(p.indices + jb + lane);
      my_e = __ldg(p.eids + jb + lane);
      my_r = __ldg(rowof + jb + lane);
    }
    float acc = 0.0f;
    int head = 0;
    for (int cb = 0; cb < G; cb += kEdCW) {
      const int c0 = cb + lane * 2;
      for (int i0 = 0; i0 < n; i0 += 8) {
        float2 lv[8], rv[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int i = i0 + k;
          const uint32_t o = __shfl_sync(kFull, my_o, i & 31);
          const uint32_t e = __shfl_sync(kFull, my_e, i & 31);
          const uint32_t r = __shfl_sync(kFull, my_r, i & 31);
          if (i < n && c0 < G) {
            const uint32_t j = static_cast<uint32_t>(jb) + i;
            const float* lp = p.lhs.base + operand_row(p.lhs.role, r, o, e, j) * p.lhs.ld;
            const float* rp = p.rhs.base + operand_row(p.rhs.role, r, o, e, j) * p.rhs.ld;
            if (l2) {
              lv[k] = __ldg(reinterpret_cast<const float2*>(lp + c0));
            } else {
              lv[k].x = lv[k].y = __ldg(lp);
            }
            if (r2) {
              rv[k] = __ldg(reinterpret_cast<const float2*>(rp + c0));
            } else {
              rv[k].x = rv[k].y = __ldg(rp);
            }
          }
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int i = i0 + k;
          if (i < n) {
            tile[i * kEdStride + lane] = c0 < G ? __fmul_rn(lv[k].x, rv[k].x) : 0.0f;
            tile[i * kEdStride + 32 + lane] = c0 + 1 < G ? __fmul_rn(lv[k].y, rv[k].y) : 0.0f;
          }
        }
      }
      __syncwarp();
      if (lane < n) {
        const int cend = min(kEdCW, G - cb);
        for (int c = 0; c < cend; ++c) {
          // column cb + c lives at tile column (c % 2) * 32 + c / 2
          acc = __fadd_rn(acc, tile[lane * kEdStride + (c & 1) * 32 + (c >> 1)]);
          if ((cb + c + 1) % D == 0) {
            p.out[static_cast<int64_t>(my_e) * p.out_ld + head] = acc;
            acc = 0.0f;
            ++head;
          }
        }
      }
      __syncwarp();
    }
  }
}

// Vector variant for 16-byte-aligned full-width operands with G % 4 == 0:
// 128-column chunks, lanes own 4 consecutive columns (LDG.128 of both
// operand rows, 4 products, one STS.128 into the edge's tile row), then lane k
// folds edge k's products in column order with LDS.128.  The tile row stride
// of 132 floats keeps both the row writes and the per-lane column reads free
// of bank conflicts.  ~3x fewer instructions per byte than k_dot_edges.
constexpr int kEd4Warps = 4;
constexpr int kEd4CW = 128;
constexpr int kEd4Stride = kEd4CW + 4;
constexpr int kEd4U = 8;

__global__ void __launch_bounds__(kEd4Warps * 32, 3) k_dot_edges4(const RowLaunch p,
                                                               const uint32_t* __restrict__ rowof,
                                                               uint64_t m) {
  extern __shared__ __align__(16) float tiles4[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* tile = tiles4 + warp * 32 * kEd4Stride;
  const int G = p.gather_dim;
  const int D = G / p.heads;
  const uint64_t n_batches = (m + 31) / 32;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kEd4Warps;
  const int32_t lrole = p.lhs.role, rrole = p.rhs.role;
  const uint32_t lldb = static_cast<uint32_t>(p.lhs.ld) * 4u, rldb = static_cast<uint32_t>(p.rhs.ld) * 4u;
  const char* lbase = reinterpret_cast<const char*>(p.lhs.base);
  const char* rbase = reinterpret_cast<const char*>(p.rhs.base);
  // head boundaries on float4 groups: the fold runs whole head segments
  // without a per-column boundary test (measured: the per-column test made
  // the fold ~4 instructions per column and the kernel issue-bound)
  const bool vfold = D % 4 == 0;
  for (uint64_t bt = static_cast<uint64_t>(blockIdx.x) * kEd4Warps + warp; bt < n_batches;
       bt += stride) {
    const uint64_t jb = bt * 32;
    const int n = static_cast<int>(m - jb < 32 ? m - jb : 32);
    // lane k resolves edge k's operand rows once per batch
    uint32_t my_e = 0, my_l = 0, my_r = 0;
    if (lane < n) {
      const uint32_t j = static_cast<uint32_t>(jb) + static_cast<uint32_t>(lane);
      const uint32_t o = __ldg(p.indices + j);
      my_e = __ldg(p.eids + j);
      const uint32_t r = __ldg(rowof + j);
      my_l = static_cast<uint32_t>(operand_row(lrole, r, o, my_e, j));
      my_r = static_cast<uint32_t>(operand_row(rrole, r, o, my_e, j));
    }
    float acc = 0.0f;
    int head = 0, left = D;  // columns left in the current head
    // steps t = (chunk, sub-batch of kEd4U edges); the loads of step t+1 are
    // issued before step t's products are parked (register ping-pong), so a
    // warp keeps two steps in flight, also across a chunk's fold
    const int nsub = (n + kEd4U - 1) / kEd4U;
    const int S = ((G + kEd4CW - 1) / kEd4CW) * nsub;
    auto load = [&](int t, float4(&lv)[kEd4U], float4(&rv)[kEd4U]) {
      const int c = t / nsub, sub = t - c * nsub;
      const int c0 = c * kEd4CW + lane * 4;
      const uint32_t coff = static_cast<uint32_t>(c0 < G ? c0 : 0) * 4u;
#pragma unroll
      for (int k = 0; k < kEd4U; ++k) {
        const int i = min(sub * kEd4U + k, n - 1);  // a tail re-reads the last edge
        const uint32_t lr = __shfl_sync(kFull, my_l, i);
        const uint32_t rr = __shfl_sync(kFull, my_r, i);
        lv[k] = __ldg(reinterpret_cast<const float4*>(lbase + static_cast<uint64_t>(lr) * lldb + coff));
        rv[k] = __ldg(reinterpret_cast<const float4*>(rbase + static_cast<uint64_t>(rr) * rldb + coff));
      }
    };
    auto park_fold = [&](int t, const float4(&lv)[kEd4U], const float4(&rv)[kEd4U]) {
      const int c = t / nsub, sub = t - c * nsub;
#pragma unroll
      for (int k = 0; k < kEd4U; ++k) {
        const float4 lc = lv[k], rc = rv[k];
        const int i = sub * kEd4U + k;
        if (i < n) {
          float4 pr;
          pr.x = __fmul_rn(lc.x, rc.x);
          pr.y = __fmul_rn(lc.y, rc.y);
          pr.z = __fmul_rn(lc.z, rc.z);
          pr.w = __fmul_rn(lc.w, rc.w);
          *reinterpret_cast<float4*>(tile + i * kEd4Stride + lane * 4) = pr;
        }
      }
      if (sub != nsub - 1) return;
      __syncwarp();
      if (lane < n) {
        const int cend = min(kEd4CW, G - c * kEd4CW);  // a multiple of 4
        const float* row = tile + lane * kEd4Stride;
        if (vfold) {
          for (int cc = 0; cc < cend;) {
            const int seg = min(cend - cc, left);  // columns to the head's end
#pragma unroll 4
            for (int q = 0; q < seg; q += 4) {
              const float4 v = *reinterpret_cast<const float4*>(row + cc + q);
              acc = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(acc, v.x), v.y), v.z), v.w);
            }
            cc += seg;
            left -= seg;
            if (left == 0) {
              p.out[static_cast<int64_t>(my_e) * p.out_ld + head] = acc;
              acc = 0.0f;
              ++head;
              left = D;
            }
          }
        } else {
          for (int cc = 0; cc < cend; cc += 4) {
            const float4 v = *reinterpret_cast<const float4*>(row + cc);
            const float xs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              acc = __fadd_rn(acc, xs[u]);
              if (--left == 0) {
                p.out[static_cast<int64_t>(my_e) * p.out_ld + head] = acc;
                acc = 0.0f;
                ++head;
                left = D;
              }
            }
          }
        }
      }
      __syncwarp();
    };
    float4 al[kEd4U], ar[kEd4U], bl[kEd4U], br[kEd4U];
    load(0, al, ar);
    for (int t = 0; t < S; t += 2) {
      if (t + 1 < S) load(t + 1, bl, br);
      park_fold(t, al, ar);
      if (t + 1 < S) {
        if (t + 2 < S) load(t + 2, al, ar);
        park_fold(t + 1, bl, br);
      }
    }
  }
}

__global__ void k_row_of_edge(const uint32_t* __restrict__ indptr, uint32_t rows,
                              uint32_t* __restrict__ rowof) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += stride)
    for (uint32_t j = __ldg(indptr + r); j < __ldg(indptr + r + 1); ++j) rowof[j] = r;
}

}  // namespace

cudaError_t launch_row_of_edge(const uint32_t* indptr, uint32_t rows, uint32_t* rowof,
                               cudaStream_t s) {
  k_row_of_edge<<<148 * 8, 256, 0, s>>>(indptr, rows, rowof);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_dot_edges(const RowLaunch& p, const uint32_t* rowof, uint64_t m,
                             cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  auto al16 = [](const float* q) { return (reinterpret_cast<uintptr_t>(q) & 15u) == 0; };
  if (p.lhs.mode == MODE_FULL && p.rhs.mode == MODE_FULL && p.gather_dim % 4 == 0 &&
      p.lhs.ld % 4 == 0 && p.rhs.ld % 4 == 0 && al16(p.lhs.base) && al16(p.rhs.base)) {
    const size_t smem = sizeof(float) * kEd4Warps * 32 * kEd4Stride;
    {
      const cudaError_t e = set_max_dynamic_smem(reinterpret_cast<const void*>(k_dot_edges4),
                                                 static_cast<int>(smem));
      if (e != cudaSuccess) return e;
    }
    const uint64_t batches = (m + 31) / 32;
    uint64_t blocks = (batches + kEd4Warps - 1) / kEd4Warps;
    const uint64_t cap = static_cast<uint64_t>(p.num_sms > 0 ? p.num_sms : 148) * 3;
    if (blocks > cap) blocks = cap;
    k_dot_edges4<<<static_cast<unsigned>(blocks), kEd4Warps * 32, smem, s>>>(p, rowof, m);
    note_launch();
    return cudaGetLastError();
  }
  const uint64_t batches = (m + 31) / 32;
  uint64_t blocks = (batches + kEdWarps - 1) / kEdWarps;
  const uint64_t cap = static_cast<uint64_t>(p.num_sms > 0 ? p.num_sms : 148) * 16;
  if (blocks > cap) blocks = cap;
  k_dot_edges<<<static_cast<unsigned>(blocks), kEdWarps * 32, 0, s>>>(p, rowof, m);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_dot(const RowLaunch& p, cudaStream_t s) {
  switch (p.vec) {
    case 4: return launch_dr<4>(p, s);
    case 2: return launch_dr<2>(p, s);
    default: return launch_dr<1>(p, s);
  }
}

}  // namespace gspmm_b200

// aux.cu -- the small sm_100a kernels around the aggregation:
//   * edge-operand permutation into CSR position order (the device plan's
//     analogue of the reference building its BlockPlan outside the timed
//     region, bench.cpp:95-97);
//   * the gradient through a max/min argmax: a scatter
//     with f64 atomics into a workspace, then one rounding to fp32, so the
//     result matches the oracle's f64 accumulation independently of the
//     order in which the atomics land.  Backward only: the forward path
//     never uses atomics.
#include <algorithm>
#include <atomic>
#include <mutex>
#include <utility>
#include <vector>

#include "device_ops.cuh"

namespace gspmm_b200 {

namespace {
std::atomic<uint64_t> g_launches{0};

__global__ void k_permute_edges(const uint32_t* __restrict__ eids, uint64_t m,
                                const float* __restrict__ src, int64_t dim,
                                int64_t src_ld, float* __restrict__ dst,
                                int64_t dst_ld) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
       i < m * static_cast<uint64_t>(dim); i += stride) {
    const uint64_t j = i / dim;
    const int64_t c = static_cast<int64_t>(i - j * dim);
    dst[j * dst_ld + c] = __ldg(src + static_cast<int64_t>(__ldg(eids + j)) * src_ld + c);
  }
}

// Argmax backward: a scatter with f64 reductions into a workspace, then one
// rounding to fp32, so the result is the f64 sum rounded once whatever order
// the reductions land in.  Targets outside [lo, lo + src_rows) are skipped
// (a rank's own source rows in the multi-GPU owner-computes form).
// Measured alternative (r02c/r02d, scripts/mb_argmax_bwd.py): column chunks
// of 4 with an L2-resident 78 MB accumulator (evict_last reductions,
// evict_first streams) ran 7.8 ms on config 3 against 2.6 ms for this
// single pass: each chunk re-reads a 32-byte sector per row for 16 bytes and
// pays a launch pair, and the chunk's reductions still missed L2.
// VEC form: a thread owns four consecutive columns (one LDG.128 of the ids
// and one of the gradients; consecutive threads read consecutive 16-byte
// pieces of a row).  Measured alternative (r02h): lanes = 32 rows of one
// column quad with the lanes that share a target combined first
// (__match_any_sync) -- 3.41 ms on config 3 against 2.62 for this form.
template <bool VEC>
__global__ void k_argmax_scatter(const int32_t* __restrict__ arg, uint32_t rows, uint32_t dim,
                                 int64_t arg_ld, const float* __restrict__ grad, int64_t grad_ld,
                                 int64_t lo, uint32_t src_rows, double* __restrict__ acc) {
  const uint32_t per_row = VEC ? dim / 4 : dim;
  const uint32_t total = rows * per_row;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const uint32_t r = i / per_row, q = i - r * per_row;
    if constexpr (VEC) {
      const int4 a = __ldcs(reinterpret_cast<const int4*>(arg + r * arg_ld) + q);
      const float4 g = __ldcs(reinterpret_cast<const float4*>(grad + r * grad_ld) + q);
      const int32_t av[4] = {a.x, a.y, a.z, a.w};
      const float gv[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int64_t u = static_cast<int64_t>(av[t]) - lo;
        if (av[t] >= 0 && static_cast<uint64_t>(u) < src_rows)
          atomicAdd(acc + u * dim + q * 4 + t, static_cast<double>(gv[t]));
      }
    } else {
      const int32_t a = __ldg(arg + r * arg_ld + q);
      const int64_t u = static_cast<int64_t>(a) - lo;
      if (a >= 0 && static_cast<uint64_t>(u) < src_rows)
        atomicAdd(acc + u * dim + q, static_cast<double>(__ldg(grad + r * grad_ld + q)));
    }
  }
}

template <bool VEC>
__global__ void k_round_f64(const double* __restrict__ acc, uint32_t rows, uint32_t dim,
                            float* __restrict__ out, int64_t ld) {
  const uint32_t per_row = VEC ? dim / 4 : dim;
  const uint32_t total = rows * per_row;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const uint32_t r = i / per_row, q = i - r * per_row;
    if constexpr (VEC) {
      const double2 a = __ldcs(reinterpret_cast<const double2*>(acc) + 2 * static_cast<uint64_t>(i));
      const double2 b = __ldcs(reinterpret_cast<const double2*>(acc) + 2 * static_cast<uint64_t>(i) + 1);
      reinterpret_cast<float4*>(out + r * ld)[q] =
          make_float4(__double2float_rn(a.x), __double2float_rn(a.y), __double2float_rn(b.x),
                      __double2float_rn(b.y));
    } else {
      out[r * ld + q] = __double2float_rn(acc[i]);
    }
  }
}

// y[r, :] = x[r, :] * scale[r] (each product rounded once, as the row
// kernels' per-edge scale does): rows of the gathered operand scaled once
// instead of once per edge.  Warp per row, float4 columns (16-byte rows).
__global__ void k_scale_rows(const float* __restrict__ x, int64_t rows, int64_t dim, int64_t ld,
                             const float* __restrict__ scale, float* __restrict__ y,
                             int64_t y_ld) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
       r < rows; r += warps) {
    const float sc = __ldg(scale + r);
    const float4* xr = reinterpret_cast<const float4*>(x + r * ld);
    float4* yr = reinterpret_cast<float4*>(y + r * y_ld);
    for (int64_t q = lane; q * 4 < dim; q += 32) {
      const float4 v = __ldg(xr + q);
      yr[q] = make_float4(__fmul_rn(v.x, sc), __fmul_rn(v.y, sc), __fmul_rn(v.z, sc),
                          __fmul_rn(v.w, sc));
    }
  }
}

unsigned grid_for(int64_t work, int threads) {
  int64_t b = (work + threads - 1) / threads;
  if (b > 148 * 32) b = 148 * 32;
  return static_cast<unsigned>(b < 1 ? 1 : b);
}

// Long rows split by edges (plan option split_edges): one block per long
// row, a thread per output column, the chunks' partials folded in chunk
// order.  Sum adds the partial sums (a fixed order: deterministic, but not
// the sequential fold's bits -- see gspmm_plan.split_edges);
// Max / Min compare strictly, so the first chunk holding the extremum keeps
// its value and its argmax -- the reference's first-wins result exactly.
template <int ROP>
__global__ void __launch_bounds__(128) k_combine_chunks(const CombineLaunch c) {
  const uint32_t i = blockIdx.x;
  const uint32_t r = __ldg(c.long_rows + i);
  const uint2 rg = __ldg(c.ranges + i);
  const uint32_t deg = __ldg(c.indptr + r + 1) - __ldg(c.indptr + r);
  constexpr int KU = 8;  // partial loads in flight per thread
  for (int col = threadIdx.x; col < c.width; col += blockDim.x) {
    const float* pp = c.part + static_cast<int64_t>(rg.x) * c.pld + col;
    float a = red_identity<ROP>();
    float s2 = 0.0f;
    int32_t ao = -1, ae = -1;
    for (uint32_t k0 = 0; k0 < rg.y; k0 += KU) {
      float v[KU], w[KU];
#pragma unroll
      for (int t = 0; t < KU; ++t) {
        const uint32_t k = min(k0 + t, rg.y - 1);
        v[t] = __ldg(pp + static_cast<int64_t>(k) * c.pld);
        w[t] = c.part2 ? __ldg(c.part2 + static_cast<int64_t>(rg.x + k) * c.pld + col) : 0.0f;
      }
#pragma unroll
      for (int t = 0; t < KU; ++t) {
        if (k0 + t >= rg.y) break;
        if constexpr (ROP == R_SUM) {
          a = __fadd_rn(a, v[t]);
        } else {
          if (red_wins<ROP>(a, v[t])) {
            a = v[t];
            const int64_t q = static_cast<int64_t>(rg.x + k0 + t) * c.pld + col;
            if (c.parg_other) ao = __ldg(c.parg_other + q);
            if (c.parg_edge) ae = __ldg(c.parg_edge + q);
          }
        }
        s2 = __fadd_rn(s2, w[t]);
      }
    }
    if (c.mean) a = deg ? __fdiv_rn(a, __uint2float_rn(deg)) : 0.0f;
    c.out[static_cast<int64_t>(r) * c.out_ld + col] = a;
    if (c.out2)
      c.out2[static_cast<int64_t>(r) * c.out2_ld + col] =
          c.mean2 ? (deg ? __fdiv_rn(s2, __uint2float_rn(deg)) : 0.0f) : s2;
    if (c.arg_other) c.arg_other[static_cast<int64_t>(r) * c.arg_ld + col] = ao;
    if (c.arg_edge) c.arg_edge[static_cast<int64_t>(r) * c.arg_ld + col] = ae;
  }
}

}  // namespace

void note_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// The dynamic shared-memory attribute is per (kernel, device): set it once
// for each pair, under a lock (host threads may drive several GPUs).
cudaError_t set_max_dynamic_smem(const void* func, int bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> done;
  std::lock_guard<std::mutex> lock(mu);
  for (const auto& d : done)
    if (d.first == func && d.second == dev) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.emplace_back(func, dev);
  return e;
}
uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

cudaError_t launch_permute_edges(const uint32_t* eids, uint64_t m,
                                 const float* src, int64_t dim, int64_t src_ld,
                                 float* dst, int64_t dst_ld, cudaStream_t s) {
  if (m == 0 || dim == 0) return cudaSuccess;
  k_permute_edges<<<grid_for(static_cast<int64_t>(m) * dim, 256), 256, 0, s>>>(
      eids, m, src, dim, src_ld, dst, dst_ld);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_argmax_backward(const int32_t* arg, int64_t rows, int64_t dim,
                                   int64_t arg_ld, const float* grad_out, int64_t grad_ld,
                                   float* grad_src, int64_t src_lo, int64_t src_rows,
                                   int64_t src_ld, cudaStream_t s) {
  if (src_rows <= 0 || dim <= 0) return cudaSuccess;
  if (rows * dim >= (int64_t{1} << 32) - (int64_t{1} << 24) ||
      src_rows * dim >= (int64_t{1} << 32) - (int64_t{1} << 24))
    return cudaErrorInvalidValue;
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15u) == 0; };
  const bool vec = dim % 4 == 0 && arg_ld % 4 == 0 && grad_ld % 4 == 0 && src_ld % 4 == 0 &&
                   al16(arg) && al16(grad_out) && al16(grad_src);
  const size_t bytes = sizeof(double) * static_cast<size_t>(src_rows * dim);
  double* acc = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&acc), bytes, s);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(acc, 0, bytes, s);
  const uint32_t R = static_cast<uint32_t>(rows), D = static_cast<uint32_t>(dim);
  const uint32_t S = static_cast<uint32_t>(src_rows);
  if (e == cudaSuccess && rows > 0) {
    const int64_t work = vec ? rows * dim / 4 : rows * dim;
    if (vec)
      k_argmax_scatter<true><<<grid_for(work, 256), 256, 0, s>>>(arg, R, D, arg_ld, grad_out,
                                                                 grad_ld, src_lo, S, acc);
    else
      k_argmax_scatter<false><<<grid_for(work, 256), 256, 0, s>>>(arg, R, D, arg_ld, grad_out,
                                                                  grad_ld, src_lo, S, acc);
    note_launch();
  }
  if (e == cudaSuccess) {
    const int64_t work = vec ? src_rows * dim / 4 : src_rows * dim;
    if (vec)
      k_round_f64<true><<<grid_for(work, 256), 256, 0, s>>>(acc, S, D, grad_src, src_ld);
    else
      k_round_f64<false><<<grid_for(work, 256), 256, 0, s>>>(acc, S, D, grad_src, src_ld);
    note_launch();
    e = cudaGetLastError();
  }
  cudaFreeAsync(acc, s);
  return e;
}

cudaError_t launch_scale_rows(const float* x, int64_t rows, int64_t dim, int64_t ld,
                              const float* scale, float* y, int64_t y_ld, cudaStream_t s) {
  if (rows == 0 || dim == 0) return cudaSuccess;
  k_scale_rows<<<grid_for(rows * 32, 256), 256, 0, s>>>(x, rows, dim, ld, scale, y, y_ld);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_combine_chunks(const CombineLaunch& c, cudaStream_t s) {
  if (c.n_long == 0 || c.width == 0) return cudaSuccess;
  switch (c.reduce) {
    case R_SUM: k_combine_chunks<R_SUM><<<c.n_long, 128, 0, s>>>(c); break;
    case R_MAX: k_combine_chunks<R_MAX><<<c.n_long, 128, 0, s>>>(c); break;
    case R_MIN: k_combine_chunks<R_MIN><<<c.n_long, 128, 0, s>>>(c); break;
    default: return cudaErrorInvalidValue;
  }
  note_launch();
  return cudaGetLastError();
}

}  // namespace gspmm_b200

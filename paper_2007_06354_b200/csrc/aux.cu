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

// Argmax backward in COLUMN CHUNKS: the f64 accumulator of one chunk of C
// columns (src_rows x C x 8 B, ~80 MB at most, e.g. 4 columns of config 3's
// 2.45M rows) stays resident in the 126 MB L2 while every row's C argmax ids
// and gradients are scattered into it; a second kernel rounds the chunk to
// fp32 once and zeroes it for the next chunk.  One 2 GB accumulator for all
// columns (round 1) missed L2 on 65% of its reduction sectors and moved
// 1.84x the algorithmic bytes.  Targets outside [lo, lo + src_rows) are
// skipped (a rank's own source rows in the multi-GPU owner-computes form).
template <bool VEC>
__global__ void k_argmax_chunk(const int32_t* __restrict__ arg, int64_t arg_ld,
                               const float* __restrict__ grad, int64_t grad_ld, uint32_t rows,
                               int c0, int cw, int64_t lo, uint32_t src_rows, int C,
                               double* __restrict__ acc) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += stride) {
    const int32_t* ar = arg + static_cast<int64_t>(r) * arg_ld + c0;
    const float* gr = grad + static_cast<int64_t>(r) * grad_ld + c0;
    if constexpr (VEC) {  // cw == C, a multiple of 4, 16-byte aligned rows
      for (int q = 0; q < cw; q += 4) {
        const int4 a = __ldcs(reinterpret_cast<const int4*>(ar + q));
        const float4 g = __ldcs(reinterpret_cast<const float4*>(gr + q));
        const int32_t av[4] = {a.x, a.y, a.z, a.w};
        const float gv[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int64_t u = static_cast<int64_t>(av[t]) - lo;
          if (av[t] >= 0 && static_cast<uint64_t>(u) < src_rows)
            atomicAdd(acc + u * C + q + t, static_cast<double>(gv[t]));
        }
      }
    } else {
      for (int t = 0; t < cw; ++t) {
        const int32_t a = __ldg(ar + t);
        const int64_t u = static_cast<int64_t>(a) - lo;
        if (a >= 0 && static_cast<uint64_t>(u) < src_rows)
          atomicAdd(acc + u * C + t, static_cast<double>(__ldg(gr + t)));
      }
    }
  }
}

// out[u, c0 : c0 + cw] = (float) acc[u, :cw]; acc zeroed for the next chunk.
__global__ void k_argmax_round(double* __restrict__ acc, uint32_t src_rows, int C, int cw,
                               float* __restrict__ out, int64_t ld, int c0) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < src_rows; u += stride) {
    double* a = acc + static_cast<int64_t>(u) * C;
    float* o = out + static_cast<int64_t>(u) * ld + c0;
    for (int t = 0; t < cw; ++t) {
      o[t] = __double2float_rn(a[t]);
      a[t] = 0.0;
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
  if (rows >= (int64_t{1} << 32) || src_rows >= (int64_t{1} << 32)) return cudaErrorInvalidValue;
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15u) == 0; };
  const bool vec_layout = dim % 4 == 0 && arg_ld % 4 == 0 && grad_ld % 4 == 0 && al16(arg) &&
                          al16(grad_out);
  // chunk width: the widest multiple of 4 whose accumulator fits ~80 MB
  constexpr double kAccBytes = 80.0 * 1048576.0;
  int C = static_cast<int>(kAccBytes / (8.0 * static_cast<double>(src_rows))) & ~3;
  C = std::max(4, std::min<int>(C, static_cast<int>((dim + 3) & ~int64_t{3})));
  double* acc = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&acc),
                                  sizeof(double) * static_cast<size_t>(src_rows) * C, s);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(acc, 0, sizeof(double) * static_cast<size_t>(src_rows) * C, s);
  const unsigned gs = grid_for(rows, 256), gr = grid_for(src_rows, 256);
  for (int64_t c0 = 0; c0 < dim && e == cudaSuccess; c0 += C) {
    const int cw = static_cast<int>(std::min<int64_t>(C, dim - c0));
    if (rows > 0) {
      if (vec_layout && cw % 4 == 0)
        k_argmax_chunk<true><<<gs, 256, 0, s>>>(arg, arg_ld, grad_out, grad_ld,
                                                static_cast<uint32_t>(rows), static_cast<int>(c0),
                                                cw, src_lo, static_cast<uint32_t>(src_rows), C,
                                                acc);
      else
        k_argmax_chunk<false><<<gs, 256, 0, s>>>(arg, arg_ld, grad_out, grad_ld,
                                                 static_cast<uint32_t>(rows),
                                                 static_cast<int>(c0), cw, src_lo,
                                                 static_cast<uint32_t>(src_rows), C, acc);
      note_launch();
    }
    k_argmax_round<<<gr, 256, 0, s>>>(acc, static_cast<uint32_t>(src_rows), C, cw, grad_src,
                                      src_ld, static_cast<int>(c0));
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

}  // namespace gspmm_b200

// build.cu -- device-side canonical CSR construction:
// the GPU analogue of build_csr / from_keys / transpose (csr.cpp:31-109).
//
// Canonical order (csr.hpp:31-35): rows ascending, within a row neighbour
// ascending, then edge id ascending.  Edges arrive in edge-id order, so one
// STABLE radix sort of the 64-bit key (row << 32 | neighbour) with the edge
// id as the value gives exactly that order (equal keys keep edge-id order).
// indptr is the exclusive scan of the row histogram.  The transpose sorts
// (neighbour << 32 | row) of the canonical CSR with the original edge ids:
// within an equal key the input is already in edge-id order, and the stable
// sort keeps it.  CUB's radix sort / scan are used as library primitives
// (setup path, not the aggregation hot path).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "internal.h"

namespace gspmm_b200 {
namespace {

__global__ void k_make_keys(const uint32_t* __restrict__ row, const uint32_t* __restrict__ col,
                            uint64_t m, uint64_t* __restrict__ keys, uint32_t* __restrict__ vals,
                            const uint32_t* __restrict__ val_src) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += stride) {
    keys[i] = (static_cast<uint64_t>(__ldg(row + i)) << 32) | __ldg(col + i);
    vals[i] = val_src ? __ldg(val_src + i) : static_cast<uint32_t>(i);
  }
}

__global__ void k_split_keys(const uint64_t* __restrict__ keys, uint64_t m,
                             uint32_t* __restrict__ indices, uint32_t* __restrict__ counts) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += stride) {
    const uint64_t k = keys[i];
    indices[i] = static_cast<uint32_t>(k);
    atomicAdd(counts + static_cast<uint32_t>(k >> 32), 1u);
  }
}

// First edge (lowest edge id) with an endpoint >= n, or ~0 (atomicMin).
__global__ void k_check_ids(const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst,
                            uint64_t m, uint32_t n, unsigned long long* __restrict__ first_bad) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += stride)
    if (__ldg(src + i) >= n || __ldg(dst + i) >= n) {
      atomicMin(first_bad, static_cast<unsigned long long>(i));
      return;
    }
}

__global__ void k_rows_of(const uint32_t* __restrict__ indptr, uint32_t rows,
                          uint32_t* __restrict__ rowof) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += stride)
    for (uint32_t j = __ldg(indptr + r); j < __ldg(indptr + r + 1); ++j) rowof[j] = r;
}

// Source blocks (the paper's source blocking, block_plan.cpp:25-69): the
// canonical row ranges are sorted by neighbour, so the edges of row r whose
// neighbour lies in block b = [b*bs, (b+1)*bs) form one contiguous sub-range
// [bpos[b][r], bpos[b+1][r]); concatenating the blocks in ascending order
// replays every row's canonical order.
__global__ void k_block_bounds(const uint32_t* __restrict__ indptr,
                               const uint32_t* __restrict__ indices, uint32_t rows, uint32_t nb,
                               uint32_t bs, uint32_t* __restrict__ bpos) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += stride) {
    const uint32_t lo = __ldg(indptr + r), hi = __ldg(indptr + r + 1);
    bpos[r] = lo;
    uint32_t a = lo;
    for (uint32_t b = 1; b < nb; ++b) {
      const uint64_t key = static_cast<uint64_t>(b) * bs;
      uint32_t l = a, h = hi;  // first position with indices[pos] >= key
      while (l < h) {
        const uint32_t mid = l + ((h - l) >> 1);
        if (__ldg(indices + mid) < key) l = mid + 1;
        else h = mid;
      }
      bpos[static_cast<uint64_t>(b) * rows + r] = l;
      a = l;
    }
    bpos[static_cast<uint64_t>(nb) * rows + r] = hi;
  }
}

__global__ void k_block_counts(const uint32_t* __restrict__ lo, const uint32_t* __restrict__ hi,
                               uint32_t rows, uint32_t* __restrict__ counts) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r <= rows; r += stride)
    counts[r] = r < rows ? __ldg(hi + r) - __ldg(lo + r) : 0u;
}

// warp per row: copy the row's block sub-range to the block CSR
__global__ void k_block_copy(const uint32_t* __restrict__ lo, const uint32_t* __restrict__ indptr_b,
                             uint32_t rows, const uint32_t* __restrict__ indices,
                             const uint32_t* __restrict__ eids, uint32_t* __restrict__ idx_b,
                             uint32_t* __restrict__ eid_b) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
    const uint32_t src = __ldg(lo + r), dst = __ldg(indptr_b + r);
    const uint32_t n = __ldg(indptr_b + r + 1) - dst;
    for (uint32_t k = lane; k < n; k += 32) {
      idx_b[dst + k] = __ldg(indices + src + k);
      eid_b[dst + k] = __ldg(eids + src + k);
    }
  }
}

int bits_for(uint32_t n) {
  int b = 1;
  while (b < 32 && (1ull << b) < n) ++b;
  return b;
}

// rows[i], cols[i] for i < m (edge-id order, or the canonical CSR order for
// a transpose with vals = its edge ids) -> canonical CSR with num_rows rows.
cudaError_t sort_build(uint32_t num_rows, uint32_t num_cols, uint64_t m, const uint32_t* rows,
                       const uint32_t* cols, const uint32_t* vals_in, uint32_t* indptr,
                       uint32_t* indices, uint32_t* eids, cudaStream_t s) {
  cudaError_t e = cudaSuccess;
  uint64_t *k0 = nullptr, *k1 = nullptr;
  uint32_t *v0 = nullptr, *counts = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0, scan_bytes = 0;
  const size_t mm = m ? m : 1;
  const int end_bit = 32 + bits_for(num_rows ? num_rows : 1);
  (void)num_cols;
  auto done = [&](cudaError_t err) {
    cudaFreeAsync(k0, s);
    cudaFreeAsync(k1, s);
    cudaFreeAsync(v0, s);
    cudaFreeAsync(counts, s);
    cudaFreeAsync(tmp, s);
    return err;
  };
  if ((e = cudaMallocAsync(reinterpret_cast<void**>(&k0), 8 * mm, s))) return done(e);
  if ((e = cudaMallocAsync(reinterpret_cast<void**>(&k1), 8 * mm, s))) return done(e);
  if ((e = cudaMallocAsync(reinterpret_cast<void**>(&v0), 4 * mm, s))) return done(e);
  if ((e = cudaMallocAsync(reinterpret_cast<void**>(&counts), 4 * (size_t(num_rows) + 1), s)))
    return done(e);
  if ((e = cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k0, k1, v0, eids, m, 0, end_bit, s)))
    return done(e);
  if ((e = cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, counts, indptr, num_rows + 1, s)))
    return done(e);
  if ((e = cudaMallocAsync(&tmp, std::max(tmp_bytes, scan_bytes) + 16, s))) return done(e);
  const unsigned grid = 148 * 8;
  if (m) {
    k_make_keys<<<grid, 256, 0, s>>>(rows, cols, m, k0, v0, vals_in);
    note_launch();
    if ((e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k0, k1, v0, eids, m, 0, end_bit, s)))
      return done(e);
  }
  if ((e = cudaMemsetAsync(counts, 0, 4 * (size_t(num_rows) + 1), s))) return done(e);
  if (m) {
    k_split_keys<<<grid, 256, 0, s>>>(k1, m, indices, counts);
    note_launch();
  }
  size_t sb = std::max(tmp_bytes, scan_bytes) + 16;
  if ((e = cub::DeviceScan::ExclusiveSum(tmp, sb, counts, indptr, num_rows + 1, s))) return done(e);
  return done(cudaGetLastError());
}

}  // namespace

cudaError_t launch_build_csr(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                             bool dst_major, uint32_t* indptr, uint32_t* indices, uint32_t* eids,
                             cudaStream_t s) {
  return sort_build(n, n, m, dst_major ? dst : src, dst_major ? src : dst, nullptr, indptr,
                    indices, eids, s);
}

cudaError_t check_edge_ids(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                           cudaStream_t s, uint64_t* first_bad) {
  *first_bad = ~0ull;
  if (m == 0) return cudaSuccess;
  unsigned long long* d = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&d), sizeof(unsigned long long), s);
  if (e) return e;
  e = cudaMemsetAsync(d, 0xff, sizeof(unsigned long long), s);
  if (e == cudaSuccess) {
    k_check_ids<<<148 * 8, 256, 0, s>>>(src, dst, m, n, d);
    note_launch();
    e = cudaGetLastError();
  }
  unsigned long long h = ~0ull;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(d, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  *first_bad = h;
  return e;
}

cudaError_t launch_transpose_csr(uint32_t num_rows, uint32_t num_cols, uint64_t m,
                                 const uint32_t* indptr, const uint32_t* indices,
                                 const uint32_t* eids, uint32_t* t_indptr, uint32_t* t_indices,
                                 uint32_t* t_eids, cudaStream_t s) {
  uint32_t* rowof = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&rowof), 4 * (m ? m : 1), s);
  if (e) return e;
  if (num_rows) {
    k_rows_of<<<148 * 8, 256, 0, s>>>(indptr, num_rows, rowof);
    note_launch();
  }
  e = sort_build(num_cols, num_rows, m, indices, rowof, eids, t_indptr, t_indices, t_eids, s);
  cudaFreeAsync(rowof, s);
  return e;
}

cudaError_t launch_block_bounds(const uint32_t* indptr, const uint32_t* indices, uint32_t rows,
                                uint32_t nb, uint32_t bs, uint32_t* bpos, cudaStream_t s) {
  if (rows == 0) return cudaSuccess;
  k_block_bounds<<<148 * 8, 256, 0, s>>>(indptr, indices, rows, nb, bs, bpos);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_block_csr(const uint32_t* lo, const uint32_t* hi, uint32_t rows,
                             const uint32_t* indices, const uint32_t* eids, uint32_t* indptr_b,
                             uint32_t* idx_b, uint32_t* eid_b, cudaStream_t s) {
  cudaError_t e;
  uint32_t* counts = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  if ((e = cudaMallocAsync(&counts, sizeof(uint32_t) * (rows + 1ull), s))) return e;
  k_block_counts<<<148 * 8, 256, 0, s>>>(lo, hi, rows, counts);
  note_launch();
  if ((e = cub::DeviceScan::ExclusiveSum(nullptr, tb, counts, indptr_b, rows + 1, s))) goto out;
  if ((e = cudaMallocAsync(&tmp, tb, s))) goto out;
  if ((e = cub::DeviceScan::ExclusiveSum(tmp, tb, counts, indptr_b, rows + 1, s))) goto out;
  k_block_copy<<<148 * 8, 256, 0, s>>>(lo, indptr_b, rows, indices, eids, idx_b, eid_b);
  note_launch();
  e = cudaGetLastError();
out:
  if (tmp) cudaFreeAsync(tmp, s);
  cudaFreeAsync(counts, s);
  return e;
}

}  // namespace gspmm_b200

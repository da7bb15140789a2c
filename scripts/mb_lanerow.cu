// mb_lanerow.cu -- micro-benchmark (development tool): can one lane stream
// its own random row (lane-per-edge, LDG.128 walking the row) as fast as
// a warp reading one row per instruction (coalesced)?  Informs the edge-dot
// kernel (csrc/dot.cu), whose lane-per-edge fold otherwise needs a
// shared-memory transpose.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_lanerow mb_lanerow.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

// lane-per-row: lane k folds row r_k sequentially, 4 columns per LDG.128
template <int F, int UN>
__global__ void __launch_bounds__(256) k_lane(const float* __restrict__ t, uint32_t nrows,
                                              uint32_t rows_per_warp, float* out) {
  const uint32_t gw = (blockIdx.x * 256 + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  float acc = 0.f;
  for (uint32_t b = 0; b < rows_per_warp; b += 32) {
    const uint32_t r = hash(gw * 7919u + b + lane) % nrows;
    const float4* p = reinterpret_cast<const float4*>(t + (size_t)r * F);
#pragma unroll UN
    for (int c = 0; c < F / 4; ++c) {
      const float4 v = __ldg(p + c);
      acc = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(acc, v.x), v.y), v.z), v.w);
    }
  }
  if (acc == 1234.5f) out[0] = acc;
}

// warp-per-row: one row per instruction (lanes own 4 columns), U rows in flight
template <int F, int U>
__global__ void __launch_bounds__(256) k_warp(const float* __restrict__ t, uint32_t nrows,
                                              uint32_t rows_per_warp, float* out) {
  const uint32_t gw = (blockIdx.x * 256 + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  float acc = 0.f;
  for (uint32_t b = 0; b < rows_per_warp; b += U) {
    float4 v[U][F / 128];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const uint32_t r = hash(gw * 7919u + b + k) % nrows;
#pragma unroll
      for (int q = 0; q < F / 128; ++q)
        v[k][q] = __ldg(reinterpret_cast<const float4*>(t + (size_t)r * F) + q * 32 + lane);
    }
#pragma unroll
    for (int k = 0; k < U; ++k)
#pragma unroll
      for (int q = 0; q < F / 128; ++q) acc += v[k][q].x + v[k][q].y + v[k][q].z + v[k][q].w;
  }
  if (acc == 1234.5f) out[0] = acc;
}

template <typename K>
void run(const char* name, K kern, const float* t, uint32_t nrows, uint32_t rpw, int blocks,
         float* out, int F) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kern<<<blocks, 256>>>(t, nrows, rpw, out);
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) kern<<<blocks, 256>>>(t, nrows, rpw, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= 5;
  const double bytes = (double)blocks * 8 * rpw * F * 4;
  std::printf("{\"kernel\": \"%s\", \"F\": %d, \"blocks\": %d, \"ms\": %.3f, \"GBs\": %.0f}\n", name,
              F, blocks, ms, bytes / ms / 1e6);
}

int main() {
  const size_t tb = 2ull << 30;
  float* t;
  float* out;
  cudaMalloc(&t, tb);
  cudaMemset(t, 0, tb);
  cudaMalloc(&out, 64);
  const uint32_t n256 = (uint32_t)(tb / 1024);
  for (int bps : {4, 8}) {
    const int blocks = 148 * bps;
    run("lane_u4", k_lane<256, 4>, t, n256, 256, blocks, out, 256);
    run("lane_u8", k_lane<256, 8>, t, n256, 256, blocks, out, 256);
    run("lane_u16", k_lane<256, 16>, t, n256, 256, blocks, out, 256);
    run("warp_u2", k_warp<256, 2>, t, n256, 256, blocks, out, 256);
    run("warp_u4", k_warp<256, 4>, t, n256, 256, blocks, out, 256);
  }
  return 0;
}

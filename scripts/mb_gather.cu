// mb_gather.cu -- micro-benchmark of random-row gather mechanisms on B200
// (development tool; informs the staging design of csrc/stream.cu).
//
// Every warp gathers `edges` random rows of `row_bytes` from a 2 GB table and
// sums a checksum, with D rows in flight per warp, via
//   mode 0: TMA 1-D bulk copy (cp.async.bulk) into a smem ring, 1 request/row
//   mode 1: LDGSTS (cp.async 16 B per lane) into a smem ring
//   mode 2: LDG.128 into registers (U rows per batch, double-buffered)
// Prints GB/s.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb mb_gather.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  }
}
__device__ __forceinline__ void tma1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void cpa16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

constexpr int kWarps = 8;

// smem ring of `stages` stages x 8 rows per warp
__global__ void __launch_bounds__(kWarps * 32, 1)
k_ring(const float* __restrict__ table, uint32_t nrows, int row_f, int edges, int stages,
       int mode, float* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ring_bytes = stages * 8 * row_f * 4;
  unsigned char* wb = smem + warp * (ring_bytes + 8 * 32);
  float* ring = reinterpret_cast<float*>(wb);
  uint64_t* bars = reinterpret_cast<uint64_t*>(wb + ring_bytes);
  if (lane == 0) for (int b = 0; b < stages; ++b) mbar_init(&bars[b], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const uint32_t gw = blockIdx.x * kWarps + warp;
  const int nst = (edges + 7) / 8;
  const uint32_t row_bytes = row_f * 4;
  auto issue = [&](int s) {
    const int b = s % stages;
    if (mode == 0) {
      if (lane == 0) mbar_expect(&bars[b], 8 * row_bytes);
      __syncwarp();
      if (lane < 8) {
        const uint32_t r = hash(gw * 977 + s * 8 + lane) % nrows;
        tma1d(ring + (b * 8 + lane) * row_f, table + (size_t)r * row_f, row_bytes, &bars[b]);
      }
    } else {
      const int cpe = row_f / 4;
      for (int q = lane; q < 8 * cpe; q += 32) {
        const int le = q / cpe, ch = q % cpe;
        const uint32_t r = hash(gw * 977 + s * 8 + le) % nrows;
        cpa16(ring + (b * 8 + le) * row_f + ch * 4, table + (size_t)r * row_f + ch * 4);
      }
      cpa_arrive(&bars[b]);
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[b]);
    }
  };
  uint32_t phase = 0;
  for (int s = 0; s < min(stages, nst); ++s) issue(s);
  float acc = 0.f;
  for (int s = 0; s < nst; ++s) {
    const int b = s % stages;
    mbar_wait(&bars[b], (phase >> b) & 1);
    phase ^= 1u << b;
    for (int e = 0; e < 8; ++e)
      for (int c = lane; c < row_f; c += 32) acc += ring[(b * 8 + e) * row_f + c];
    __syncwarp();
    if (s + stages < nst) issue(s + stages);
  }
  if (acc == 12345.f) out[0] = acc;
}

// LDG.128 register gather: U rows in flight (float4 per lane per 512 B)
template <int U>
__global__ void __launch_bounds__(256) k_ldg(const float* __restrict__ table, uint32_t nrows,
                                            int row_f, int edges, float* out) {
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  float acc = 0.f;
  const int v4 = row_f / 4;
  for (int e0 = 0; e0 < edges; e0 += U) {
    float4 x[U][2];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const uint32_t r = hash(gw * 977 + e0 + k) % nrows;
      const float4* p = reinterpret_cast<const float4*>(table + (size_t)r * row_f);
#pragma unroll
      for (int v = 0; v < 2; ++v)
        if (lane + 32 * v < v4) x[k][v] = __ldg(p + lane + 32 * v);
    }
#pragma unroll
    for (int k = 0; k < U; ++k)
#pragma unroll
      for (int v = 0; v < 2; ++v)
        if (lane + 32 * v < v4) acc += x[k][v].x + x[k][v].y + x[k][v].z + x[k][v].w;
  }
  if (acc == 12345.f) out[0] = acc;
}

int main(int argc, char** argv) {
  const size_t table_bytes = 2ull << 30;
  float* table;
  float* out;
  cudaMalloc(&table, table_bytes);
  cudaMemset(table, 0, table_bytes);
  cudaMalloc(&out, 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int edges = 4096;
  for (int row_f : {32, 64, 100, 128, 256}) {
    const uint32_t nrows = table_bytes / (row_f * 4);
    for (int mode = 0; mode < 2; ++mode) {
      for (int smem_kb : {24, 48, 96, 192}) {
        // per-warp ring bytes
        const int per_warp = smem_kb * 1024 / kWarps;
        const int stages = per_warp / (8 * row_f * 4);
        if (stages < 1 || stages > 32) continue;
        const int smem = kWarps * (stages * 8 * row_f * 4 + 256);
        cudaFuncSetAttribute(k_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        for (int it = 0; it < 2; ++it) {
          cudaEventRecord(a);
          k_ring<<<sms, kWarps * 32, smem>>>(table, nrows, row_f, edges, stages, mode, out);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
        }
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = (double)sms * kWarps * edges * row_f * 4;
        printf("%-6s row %4d B smem/SM %3d KB stages %2d : %7.1f GB/s  (%.1f req/us/SM)  err=%s\n",
               mode ? "LDGSTS" : "TMA1D", row_f * 4, smem_kb, stages, bytes / ms / 1e6,
               (double)kWarps * edges / (ms * 1e3), cudaGetErrorString(cudaGetLastError()));
      }
    }
    for (int blocks_per_sm : {4, 8}) {
      const int blocks = sms * blocks_per_sm;
      for (int it = 0; it < 2; ++it) {
        cudaEventRecord(a);
        k_ldg<8><<<blocks, 256>>>(table, nrows, row_f, edges, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
      }
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double bytes = (double)blocks * 8 * edges * row_f * 4;
      printf("LDG128 row %4d B blocks/SM %d U=8         : %7.1f GB/s  err=%s\n", row_f * 4,
             blocks_per_sm, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}

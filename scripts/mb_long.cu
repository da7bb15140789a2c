// mb_long.cu -- micro-benchmark of the long-row CTA pipeline on B200
// (development tool; informs csrc/gather_impl.cuh k_long_async).
//
// One 512-thread CTA per SM streams random rows of `row_f` floats from a 2 GB
// table through a shared-memory ring of NB stages x R rows (cp.async 16 B
// copies, one wait_group + barrier per stage), optionally folded by column
// owners (fold=1: thread t sums column t over the stage; fold=4: float4 per
// owner).  Variants: barrier per stage (bar=1) or per-warp private rings
// (bar=0: no CTA barrier, each warp copies and folds its own rows).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_long mb_long.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cpa16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void wait_group() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

template <int NB>
__global__ void __launch_bounds__(512, 1)
k_stage(const float* __restrict__ table, uint32_t nrows, int row_f, int R, int rounds, int fold,
        int spread, float* out) {
  extern __shared__ __align__(16) float sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int DF = R * row_f;
  const int qpe = row_f / 4;
  const int lpe = qpe >= 32 ? 32 : qpe;
  const int epi = 32 / lpe, sub = lane / lpe, il = lane % lpe, tpe = (qpe + lpe - 1) / lpe;
  const int ngroups = (R + epi - 1) / epi;
  auto issue = [&](int rd) {
    if (rd >= rounds) return;
    float* bd = sm + (rd % NB) * DF;
    for (int g = warp; g < ngroups; g += 16) {
      const int q = g * epi + sub;
      if (q >= R) continue;
      const uint32_t row = hash(blockIdx.x * 7919u + (rd * R + q) * spread) % nrows;
      const float* src = table + (size_t)row * row_f + il * 4;
      float* dst = bd + q * row_f + il * 4;
      for (int t = 0; t < tpe; ++t) cpa16(dst + t * lpe * 4, src + t * lpe * 4);
    }
  };
  for (int d = 0; d < NB - 1; ++d) { issue(d); commit(); }
  float acc[4] = {0, 0, 0, 0};
  for (int k = 0; k < rounds; ++k) {
    wait_group<NB - 2>();
    __syncthreads();
    issue(k + NB - 1);
    commit();
    const float* st = sm + (k % NB) * DF;
    if (fold == 1 && tid < row_f) {
#pragma unroll 8
      for (int e = 0; e < R; ++e) acc[0] += st[e * row_f + tid];
    } else if (fold == 4 && tid * 4 < row_f) {
#pragma unroll 8
      for (int e = 0; e < R; ++e) {
        const float4 v = *reinterpret_cast<const float4*>(st + e * row_f + tid * 4);
        acc[0] += v.x; acc[1] += v.y; acc[2] += v.z; acc[3] += v.w;
      }
    }
  }
  wait_group<0>();
  if (acc[0] + acc[1] + acc[2] + acc[3] == 12345.f) out[0] = acc[0];
}

int main() {
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
  for (int row_f : {32, 100, 256}) {
    const uint32_t nrows = table_bytes / (row_f * 4);
    for (int grid_frac : {1, 2}) {  // all SMs, half the SMs
      const int grid = sms / grid_frac;
      for (int nb : {3, 4, 6}) {
        for (int stage_kb : {16, 24, 32}) {
          const int R = stage_kb * 1024 / (row_f * 4);
          const int smem = nb * R * row_f * 4;
          if (smem > 220 * 1024) continue;
          for (int fold : {0, 1, 4}) {
            if (fold == 4 && row_f % 4) continue;
            const int rounds = (64 << 20) / (R * row_f * 4);  // 64 MB per CTA
            auto kern = nb == 3 ? k_stage<3> : nb == 4 ? k_stage<4> : k_stage<6>;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            float ms = 0;
            for (int it = 0; it < 2; ++it) {
              cudaEventRecord(a);
              kern<<<grid, 512, smem>>>(table, nrows, row_f, R, rounds, fold, 1, out);
              cudaEventRecord(b);
              cudaEventSynchronize(b);
              cudaEventElapsedTime(&ms, a, b);
            }
            const double bytes = (double)grid * rounds * R * row_f * 4;
            printf("row %4d B grid %3d NB %d stage %2d KB R %3d fold %d : %7.1f GB/s total %6.1f GB/s/SM %s\n",
                   row_f * 4, grid, nb, stage_kb, R, fold, bytes / ms / 1e6, bytes / ms / 1e6 / grid,
                   cudaGetErrorString(cudaGetLastError()));
          }
        }
      }
    }
  }
  return 0;
}

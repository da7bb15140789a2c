// mb_gather4.cu -- micro-benchmark: per-SM streaming rate of random-row
// gathers through a shared-memory ring fed by TMA tile::gather4 (sm_100a),
// one CTA per SM, the column owners folding each stage in row order.
// Development tool (informs the long-row CTA in csrc/gather_impl.cuh).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_gather4 mb_gather4.cu
//   ./mb_gather4 <F> <bw> <ctas> <rows_per_cta> <R> <NB> <fold>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  std::printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e_)); std::exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(b)), "r"(par), "r"(1000000u) : "memory");
}
__device__ __forceinline__ void g4(uint32_t dst, const CUtensorMap* m, int c, int r0, int r1, int r2,
                                   int r3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst), "l"(m), "r"(c), "r"(r0), "r"(r1), "r"(r2),
      "r"(r3), "r"(smem_u32(bar)) : "memory");
}

// warp 0: producer (lanes issue gather4 for groups of 4 rows); warps 1..4 fold.
__global__ void __launch_bounds__(160, 1)
k_g4(const __grid_constant__ CUtensorMap tm, uint32_t nrows, int bw, int rows_per_cta, int R, int NB,
     int fold, float* out) {
  extern __shared__ __align__(128) float sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)NB * R * bw);
  uint64_t* empty = full + NB;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int b = 0; b < NB; ++b) { mbar_init(&full[b], 1); mbar_init(&empty[b], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int rounds = rows_per_cta / R;
  const int c0 = (blockIdx.x % 4) * 0;  // column slice start
  if (warp == 0) {
    for (int s = 0; s < rounds; ++s) {
      const int b = s % NB;
      if (s >= NB) mbar_wait(&empty[b], ((s / NB) - 1) & 1);
      if (lane == 0) mbar_expect(&full[b], (uint32_t)(R * bw * 4));
      __syncwarp();
      const uint32_t base = smem_u32(sm + (size_t)b * R * bw);
      for (int q = lane * 4; q < R; q += 128) {
        uint32_t k = blockIdx.x * 0x9E3779B1u + (uint32_t)(s * R + q) * 2654435761u;
        int r0 = hash(k) % nrows, r1 = hash(k + 1) % nrows, r2 = hash(k + 2) % nrows, r3 = hash(k + 3) % nrows;
        g4(base + q * bw * 4, &tm, c0, r0, r1, r2, r3, &full[b]);
      }
    }
  } else {
    const int ct = tid - 32;  // 0..127
    float acc[4] = {0, 0, 0, 0};
    for (int s = 0; s < rounds; ++s) {
      const int b = s % NB;
      mbar_wait(&full[b], (s / NB) & 1);
      const float* st = sm + (size_t)b * R * bw;
      if (fold == 1 && ct < bw) {
#pragma unroll 8
        for (int e = 0; e < R; ++e) acc[0] = __fadd_rn(acc[0], st[e * bw + ct]);
      } else if (fold == 4 && ct * 4 < bw) {
#pragma unroll 8
        for (int e = 0; e < R; ++e) {
          float4 v = *reinterpret_cast<const float4*>(st + e * bw + ct * 4);
          acc[0] = __fadd_rn(acc[0], v.x); acc[1] = __fadd_rn(acc[1], v.y);
          acc[2] = __fadd_rn(acc[2], v.z); acc[3] = __fadd_rn(acc[3], v.w);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[b]);
    }
    if (acc[0] + acc[1] + acc[2] + acc[3] == 12345.f) out[tid] = acc[0];
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int F = argc > 1 ? atoi(argv[1]) : 256;
  const int bw = argc > 2 ? atoi(argv[2]) : 256;
  const int ctas = argc > 3 ? atoi(argv[3]) : 148;
  const int rpc = argc > 4 ? atoi(argv[4]) : 65536;
  const int R = argc > 5 ? atoi(argv[5]) : 64;
  const int NB = argc > 6 ? atoi(argv[6]) : 3;
  const int fold = argc > 7 ? atoi(argv[7]) : 1;
  const size_t table_bytes = 2ull << 30;
  const uint32_t nrows = (uint32_t)(table_bytes / (F * 4));
  float* table; float* out;
  CK(cudaMalloc(&table, table_bytes));
  CK(cudaMemset(table, 0, table_bytes));
  CK(cudaMalloc(&out, 4096));
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)F, nrows};
  cuuint64_t strides[1] = {(cuuint64_t)F * 4};
  cuuint32_t box[2] = {(cuuint32_t)bw, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, table, dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) { std::printf("encode failed %d\n", (int)cr); return 1; }
  const size_t smem = (size_t)NB * R * bw * 4 + 2 * NB * 8;
  CK(cudaFuncSetAttribute(k_g4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int it = 0; it < 2; ++it) k_g4<<<ctas, 160, smem>>>(tm, nrows, bw, rpc, R, NB, fold, out);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  const int iters = 5;
  for (int it = 0; it < iters; ++it) k_g4<<<ctas, 160, smem>>>(tm, nrows, bw, rpc, R, NB, fold, out);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  ms /= iters;
  const double bytes = (double)ctas * rpc * bw * 4;
  std::printf("{\"F\": %d, \"bw\": %d, \"ctas\": %d, \"R\": %d, \"NB\": %d, \"fold\": %d, \"ms\": %.4f, "
              "\"GBs_total\": %.1f, \"GBs_per_cta\": %.2f, \"rows_per_us_per_cta\": %.1f}\n",
              F, bw, ctas, R, NB, fold, ms, bytes / ms / 1e6, bytes / ms / 1e6 / ctas,
              (double)rpc / (ms * 1e3));
  return 0;
}

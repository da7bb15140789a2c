// mb_chain.cu -- what bounds one warp's sequential fp32 fold out of shared
// memory (the long-row consumer)?  Cycles per edge of: (a) a register-only
// dependent FADD chain, (b) the chain fed by LDS.128 one block ahead, (c)
// the same with 3 other warps of the SMSP spinning on an mbarrier try_wait
// (the producers of a consumer-bound unit), (d) with those warps parked on
// nanosleep.  nvcc -arch=sm_100a -O3 -o scripts/bin/mb_chain scripts/mb_chain.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ bool try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
      : "=r"(ok)
      : "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(parity)
      : "memory");
  return ok;
}

// MODE 4..: the other 12 warps gather random 32-byte pieces of a 1 GB table
// with LDG.128 (16 lines per warp instruction, PER loads per lane in flight,
// then a pause of `gap` clocks) -- the producers of a narrow long-row unit;
// DEPTH = blocks of 16 edges the consumer's LDS run ahead of its chain.
template <int MODE, int DEPTH = 1>
__global__ void __launch_bounds__(512, 1) k(float* out, long long* cyc, int edges,
                                            const float4* table = nullptr, int gap = 0) {
  __shared__ __align__(16) float buf[8192];
  __shared__ uint64_t bar;
  __shared__ volatile int done;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 8192; i += 512) buf[i] = 1.0f + i * 1e-7f;
  if (tid == 0) {
    done = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
  }
  __syncthreads();
  if (warp == 12) {  // the consumer warp (SMSP 0, with warps 0, 4, 8)
    float acc = 0.0f;
    const long long t0 = clock64();
    if (MODE == 10 || MODE == 11 || MODE == 12) {
      // one column per lane, row-major stage of 8 floats per edge: scalar
      // LDS at immediate offsets, one block of 16 edges ahead (the narrow
      // consumer of k_long_rg); MODE 11: two edges per LDS.64 of a
      // column-major stage; MODE 12: LDS every edge but only 8 FADDs per 16
      // loads (is the LDS rate the bound?)
      const float* col = buf + (tid & 7);
      float a[16], b[16];
      auto ld = [&](int e, float (&x)[16]) {
        const float* p = col + (e & 1008) * 8;
        if (MODE == 11) {
          const float* q = buf + (tid & 7) * 1020 + (e & 1008);
#pragma unroll
          for (int k = 0; k < 16; k += 2) {
            const float2 v = *reinterpret_cast<const float2*>(q + k);
            x[k] = v.x; x[k + 1] = v.y;
          }
        } else {
#pragma unroll
          for (int k = 0; k < 16; ++k) x[k] = p[k * 8];
        }
      };
      auto fold = [&](const float (&x)[16]) {
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if (MODE != 12 || (k & 1)) acc = __fadd_rn(acc, x[k]);
          else asm volatile("" ::"f"(x[k]));
      };
      ld(0, a);
      for (int e = 0; e < edges; e += 32) {
        ld(e + 16, b);
        fold(a);
        ld(e + 32, a);
        fold(b);
      }
    } else if (MODE >= 4) {
      const float* col = buf + (tid & 7) * 1020;
      float4 ring[DEPTH + 1][4];
#pragma unroll
      for (int d = 0; d < DEPTH; ++d)
#pragma unroll
        for (int j = 0; j < 4; ++j) ring[d][j] = *reinterpret_cast<const float4*>(col + 16 * d + 4 * j);
      for (int e = 0; e < edges; e += 16 * (DEPTH + 1)) {
#pragma unroll
        for (int d = 0; d <= DEPTH; ++d) {
          const float* p = col + ((e + 16 * (d + DEPTH)) & 1008);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            ring[(d + DEPTH) % (DEPTH + 1)][j] = *reinterpret_cast<const float4*>(p + 4 * j);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float4 v = ring[d][j];
            acc = __fadd_rn(acc, v.x); acc = __fadd_rn(acc, v.y);
            acc = __fadd_rn(acc, v.z); acc = __fadd_rn(acc, v.w);
          }
        }
      }
    } else if (MODE == 0) {
      float x = buf[tid];
      for (int e = 0; e < edges; e += 16) {
#pragma unroll
        for (int k = 0; k < 16; ++k) acc = __fadd_rn(acc, x);
      }
    } else {
      const float* col = buf + (tid & 7) * 1020;
      float4 a[4], b[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) a[j] = *reinterpret_cast<const float4*>(col + 4 * j);
      for (int e = 0; e < edges; e += 32) {
        const float* p = col + ((e + 16) & 1008);
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = *reinterpret_cast<const float4*>(p + 4 * j);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc = __fadd_rn(acc, a[j].x); acc = __fadd_rn(acc, a[j].y);
          acc = __fadd_rn(acc, a[j].z); acc = __fadd_rn(acc, a[j].w);
        }
        p = col + ((e + 32) & 1008);
#pragma unroll
        for (int j = 0; j < 4; ++j) a[j] = *reinterpret_cast<const float4*>(p + 4 * j);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc = __fadd_rn(acc, b[j].x); acc = __fadd_rn(acc, b[j].y);
          acc = __fadd_rn(acc, b[j].z); acc = __fadd_rn(acc, b[j].w);
        }
      }
    }
    const long long t1 = clock64();
    if ((tid & 31) == 0) cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x * 32 + (tid & 31)] = acc;
    __threadfence_block();
    if ((tid & 31) == 0) {
      done = 1;
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
    }
  } else if (warp < 12) {
    if (MODE == 2) {
      while (!try_wait(&bar, 0)) {
      }
    } else if (MODE == 3) {
      while (!done) __nanosleep(2000);
    } else if (MODE >= 4 && MODE < 10) {
      uint32_t h = tid * 2654435761u + blockIdx.x * 40503u;
      float4 s4 = make_float4(0, 0, 0, 0);
      while (!done) {
        float4 v[6];
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          h = h * 1664525u + 1013904223u;
          // 2 lanes share a 32-byte piece: 16 lines per warp instruction
          const uint32_t hh = __shfl_sync(0xffffffffu, h, (tid & 31) & ~1);
          v[i] = __ldg(table + (static_cast<size_t>(hh >> 7) * 2 + (tid & 1)));
        }
#pragma unroll
        for (int i = 0; i < 6; ++i) { s4.x += v[i].x; s4.y += v[i].y; }
        if (gap) {
          const long long t = clock64();
          while (clock64() - t < gap) {
          }
        }
      }
      if (s4.x == 123.0f) out[tid] = s4.y;
    }
  }
}

template <int MODE, int DEPTH = 1>
void run(const char* name, float* out, long long* cyc, int edges, const float4* table = nullptr,
         int gap = 0) {
  k<MODE, DEPTH><<<148, 512>>>(out, cyc, edges, table, gap);
  k<MODE, DEPTH><<<148, 512>>>(out, cyc, edges, table, gap);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0;
  for (long long v : h) s += v;
  printf("%-58s %.2f cycles/edge (%s)\n", name, s / 148 / edges, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 32 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const int edges = 1 << 20;
  run<0>("register-only FADD chain", out, cyc, edges);
  run<1>("chain fed by LDS.128 one block ahead, other warps exited", out, cyc, edges);
  run<2>("same, 12 warps spinning on mbarrier.try_wait", out, cyc, edges);
  run<3>("same, 12 warps polling a flag with nanosleep(2000)", out, cyc, edges);
  float4* table;
  cudaMalloc(&table, 1ull << 30);
  cudaMemset(table, 0, 1ull << 30);
  run<4, 1>("12 warps gathering 32 B pieces back to back, LDS 1 block ahead", out, cyc, edges, table, 0);
  run<4, 2>("  same, LDS 2 blocks ahead", out, cyc, edges, table, 0);
  run<4, 4>("  same, LDS 4 blocks ahead", out, cyc, edges, table, 0);
  run<10>("scalar LDS + FADD per edge (row-major, imm offsets), other warps exited", out, cyc, edges);
  run<11>("LDS.64 per 2 edges + 2 FADD (column-major)", out, cyc, edges);
  run<12>("scalar LDS per edge, FADD every other edge", out, cyc, edges);
  run<4, 1>("gathers with 4000-clock pauses, LDS 1 block ahead", out, cyc, edges, table, 4000);
  run<4, 4>("  same, LDS 4 blocks ahead", out, cyc, edges, table, 4000);
  return 0;
}

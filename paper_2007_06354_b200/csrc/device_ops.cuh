// device_ops.cuh -- element operators and operand access for the sm_100a
// kernels.  Every arithmetic op uses an explicit round-to-nearest intrinsic
// so nvcc cannot contract a multiply and an add into an FMA: the reference
// rounds each product and each sum separately (kernels.cpp:38-69 compiled
// for baseline x86-64), and that is what makes the GPU results bit-exact.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"

namespace gspmm_b200 {

constexpr unsigned kFull = 0xffffffffu;

template <int BOP>
__device__ __forceinline__ float bin_apply(float l, float r) {
  if constexpr (BOP == B_ADD) return __fadd_rn(l, r);
  else if constexpr (BOP == B_SUB) return __fsub_rn(l, r);
  else if constexpr (BOP == B_MUL) return __fmul_rn(l, r);
  else if constexpr (BOP == B_DIV) return __fdiv_rn(l, r);
  else return l;  // B_COPY
}

template <int ROP>
__device__ __forceinline__ float red_identity() {
  if constexpr (ROP == R_MAX) return -__int_as_float(0x7f800000);
  else if constexpr (ROP == R_MIN) return __int_as_float(0x7f800000);
  else if constexpr (ROP == R_PROD) return 1.0f;
  else return 0.0f;
}

// The reference's reducers (kernels.cpp:38-52).  Max/Min are the literal
// comparisons, not fmaxf/fminf: NaN never wins and, among values that
// compare equal (+0/-0), the earlier one stays.
template <int ROP>
__device__ __forceinline__ float red_combine(float a, float m) {
  if constexpr (ROP == R_SUM) return __fadd_rn(a, m);
  else if constexpr (ROP == R_MAX) return a < m ? m : a;
  else if constexpr (ROP == R_MIN) return m < a ? m : a;
  else if constexpr (ROP == R_PROD) return __fmul_rn(a, m);
  else return m;  // R_LAST
}

// Does m replace the running value under Max/Min (for argmax tracking)?
template <int ROP>
__device__ __forceinline__ bool red_wins(float a, float m) {
  if constexpr (ROP == R_MAX) return a < m;
  else return m < a;
}

template <int V>
__device__ __forceinline__ void load_vec(const float* p, float (&x)[V]) {
  if constexpr (V == 4) {
    const float4 t = __ldg(reinterpret_cast<const float4*>(p));
    x[0] = t.x; x[1] = t.y; x[2] = t.z; x[3] = t.w;
  } else if constexpr (V == 2) {
    const float2 t = __ldg(reinterpret_cast<const float2*>(p));
    x[0] = t.x; x[1] = t.y;
  } else {
    x[0] = __ldg(p);
  }
}

template <int V>
__device__ __forceinline__ void store_vec(float* p, const float (&x)[V]) {
  if constexpr (V == 4) {
    *reinterpret_cast<float4*>(p) = make_float4(x[0], x[1], x[2], x[3]);
  } else if constexpr (V == 2) {
    *reinterpret_cast<float2*>(p) = make_float2(x[0], x[1]);
  } else {
    p[0] = x[0];
  }
}

// Operand row index of edge j (OperandRef::row, kernels.cpp:120-125).
__device__ __forceinline__ int64_t operand_row(int32_t role, uint32_t row,
                                               uint32_t other, uint32_t eid,
                                               uint32_t pos) {
  return role == ROLE_ROW ? row : role == ROLE_OTHER ? other
                                : role == ROLE_EID ? eid : pos;
}

// V elements of an operand for output columns c0..c0+V-1.
template <int V>
__device__ __forceinline__ void load_operand(const OperandDesc& d, int64_t row,
                                             int c0, float (&x)[V]) {
  const float* p = d.base + row * d.ld;
  if (d.mode == MODE_FULL) {
    load_vec<V>(p + c0, x);
  } else {
    const float s = __ldg(p + (d.mode == MODE_SCALAR ? 0 : c0 / d.group));
#pragma unroll
    for (int t = 0; t < V; ++t) x[t] = s;
  }
}

}  // namespace gspmm_b200

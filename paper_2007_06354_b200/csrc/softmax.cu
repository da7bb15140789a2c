// softmax.cu -- fused GAT edge softmax over the in-edges of every destination
// (SURVEY 8f, rank 2): the reference composite
//   m = e_copy_max_v(l); s = e_sub_v_copy_e(l, m); p = exp(s);
//   z = e_copy_add_v(p); a = e_div_v_copy_e(p, z)            (PAPER Table 2, GAT)
// in one kernel (one pass per row to find m, one for z, one writing a), and
// its backward  grad_l = a * (grad_a - sum_row(a * grad_a)).
//
// Per row and head: m is the reference max (a < x ? x : a, NaN never wins,
// 0-degree rows produce nothing); p = expf(l - m) in fp32; z and the backward
// dot are fp32 sums in a FIXED order (per-lane strided partial sums, then a
// fixed butterfly), so results are deterministic run to run; a = p / z with
// one IEEE division.  (exp has no reference implementation: parity with the
// composite is within tolerance.)
//
// Layout: l / a / grad are [E, H] fp32 rows, in edge-id order (row = edge
// id, the reference layout) or in the handle's CSR position order.  Lanes =
// (edge slot, head): 32/H edges per warp step.  Rows up to the plan threshold run
// one warp per row; heavier rows run one 8-warp CTA per row with a
// shared-memory combine of the warps' partials (in warp order).
#include <algorithm>

#include "internal.h"
#include "device_ops.cuh"

namespace gspmm_b200 {
namespace {

constexpr int kSmWarps = 8;  // warps per CTA (both kernels)

struct SoftmaxArgs {
  const uint32_t* indptr;
  const uint32_t* eids;
  uint32_t rows;
  int heads;
  bool by_pos;
  const float* l;  // forward: logits; backward: a
  int64_t l_ld;
  const float* g;  // backward: grad_a
  int64_t g_ld;
  float* out;      // forward: a; backward: grad_l
  int64_t out_ld;
  uint32_t long_threshold;  // rows above this many edges run on k_softmax_long
  uint32_t* counter;        // zeroed per launch: rows are handed out in groups (nullptr: strided)
};

__device__ __forceinline__ float max_ref(float a, float x) { return a < x ? x : a; }

// Combine lane partials over the edge slots of the same head: xor offsets
// Hp, 2Hp, ... < 32 (Hp = heads rounded up to a power of two).
template <bool MAX>
__device__ __forceinline__ float slot_reduce(float v, int Hp) {
  for (int off = Hp; off < 32; off <<= 1) {
    const float o = __shfl_xor_sync(kFull, v, off);
    v = MAX ? max_ref(v, o) : __fadd_rn(v, o);
  }
  return v;
}

// One row's softmax (BWD = false) or backward (BWD = true), by `nw` warps of
// the block (warp index w); red is shared scratch of nw * 32 floats when nw > 1.
template <bool BWD>
__device__ __forceinline__ void row_softmax(const SoftmaxArgs& p, uint32_t r, int w, int nw,
                                            float* red) {
  const int lane = threadIdx.x & 31;
  const int H = p.heads;
  int Hp = 1;
  while (Hp < H) Hp <<= 1;
  const int slots = 32 / Hp;
  const int sub = lane / Hp, h = lane - sub * Hp;
  const bool active = h < H;
  const uint32_t e0 = __ldg(p.indptr + r), e1 = __ldg(p.indptr + r + 1);
  const uint32_t n = e1 - e0;
  if (n == 0) return;
  const uint32_t step = static_cast<uint32_t>(slots * nw);
  const uint32_t first = static_cast<uint32_t>(w * slots + sub);
  auto erow = [&](uint32_t k) -> int64_t {
    const uint32_t j = e0 + k;
    return p.by_pos ? static_cast<int64_t>(j) : static_cast<int64_t>(__ldg(p.eids + j));
  };
  auto block_combine = [&](float v, bool is_max) -> float {
    // lanes hold per-head partials of this warp; combine warps in order
    if (nw == 1) return v;
    __syncthreads();
    if (lane < Hp) red[w * 32 + lane] = v;
    __syncthreads();
    float t = red[h];
    for (int k = 1; k < nw; ++k) t = is_max ? max_ref(t, red[k * 32 + h]) : __fadd_rn(t, red[k * 32 + h]);
    return t;
  };
  if constexpr (!BWD) {
    float m = -__int_as_float(0x7f800000);
    if (active)
      for (uint32_t k = first; k < n; k += step) m = max_ref(m, __ldg(p.l + erow(k) * p.l_ld + h));
    m = slot_reduce<true>(m, Hp);
    m = block_combine(m, true);
    float z = 0.0f;
    if (active)
      for (uint32_t k = first; k < n; k += step)
        z = __fadd_rn(z, expf(__fsub_rn(__ldg(p.l + erow(k) * p.l_ld + h), m)));
    z = slot_reduce<false>(z, Hp);
    z = block_combine(z, false);
    if (active)
      for (uint32_t k = first; k < n; k += step) {
        const int64_t er = erow(k);
        const float pe = expf(__fsub_rn(__ldg(p.l + er * p.l_ld + h), m));
        p.out[er * p.out_ld + h] = __fdiv_rn(pe, z);
      }
  } else {
    float s = 0.0f;
    if (active)
      for (uint32_t k = first; k < n; k += step) {
        const int64_t er = erow(k);
        s = __fadd_rn(s, __fmul_rn(__ldg(p.l + er * p.l_ld + h), __ldg(p.g + er * p.g_ld + h)));
      }
    s = slot_reduce<false>(s, Hp);
    s = block_combine(s, false);
    if (active)
      for (uint32_t k = first; k < n; k += step) {
        const int64_t er = erow(k);
        const float a = __ldg(p.l + er * p.l_ld + h);
        p.out[er * p.out_ld + h] = __fmul_rn(a, __fsub_rn(__ldg(p.g + er * p.g_ld + h), s));
      }
  }
}

template <bool BWD>
__global__ void __launch_bounds__(kSmWarps * 32) k_softmax_rows(const SoftmaxArgs p) {
  const int warp = threadIdx.x >> 5;
  const uint32_t stride = gridDim.x * kSmWarps;
  for (uint32_t r = blockIdx.x * kSmWarps + warp; r < p.rows; r += stride) {
    const uint32_t deg = __ldg(p.indptr + r + 1) - __ldg(p.indptr + r);
    if (deg > p.long_threshold) continue;  // k_softmax_long
    row_softmax<BWD>(p, r, 0, 1, nullptr);
  }
}

template <bool BWD>
__global__ void __launch_bounds__(kSmWarps * 32) k_softmax_long(const SoftmaxArgs p,
                                                               const uint32_t* long_rows,
                                                               uint32_t n_long) {
  __shared__ float red[kSmWarps * 32];
  const int warp = threadIdx.x >> 5;
  for (uint32_t i = blockIdx.x; i < n_long; i += gridDim.x) {
    const uint32_t r = __ldg(long_rows + i);
    row_softmax<BWD>(p, r, warp, kSmWarps, red);
    __syncthreads();
  }
}

// ---------------------------------------------------------------- vector
// Lane-per-edge variant for H in {1, 2, 4, 8, 16}: lane k owns edge k of a
// 32-edge step and all H heads of it (one or more 16-byte loads when the
// rows are 16-byte aligned); per-head partials combine through a fixed
// butterfly and, for CTA rows, across warps in warp order.  Same reductions,
// same fixed order per (lane, step) -- deterministic.
template <int H>
__device__ __forceinline__ void load_heads(const float* p, bool vec, float (&v)[H]) {
  if constexpr (H % 4 == 0) {
    if (vec) {
#pragma unroll
      for (int q = 0; q < H / 4; ++q) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(p) + q);
        v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
      }
      return;
    }
  }
#pragma unroll
  for (int h = 0; h < H; ++h) v[h] = __ldg(p + h);
}

template <int H>
__device__ __forceinline__ void store_heads(float* p, bool vec, const float (&v)[H]) {
  if constexpr (H % 4 == 0) {
    if (vec) {
#pragma unroll
      for (int q = 0; q < H / 4; ++q)
        reinterpret_cast<float4*>(p)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      return;
    }
  }
#pragma unroll
  for (int h = 0; h < H; ++h) p[h] = v[h];
}

// All-reduce of H per-lane values over the warp, every lane ending with all H
// totals.  Recursive halving first (offsets 16, 8, ...: each step a lane
// keeps half of its heads and folds in its partner's copy of them), so lane
// L ends with the partial of head L >> log2(32 / H) over H lanes; then a
// butterfly over the remaining lane bits, then one broadcast per head.
// 2H + log2(32/H) - 1 shuffles instead of 5H (H = 8: 17 against 40; the
// previous butterfly kept the rows kernel ~65% issue-busy).  Fixed order:
// deterministic run to run.
template <int H, bool MAX>
__device__ __forceinline__ void lane_reduce(float (&v)[H]) {
  const int lane = threadIdx.x & 31;
  auto op = [](float a, float b) { return MAX ? max_ref(a, b) : __fadd_rn(a, b); };
  constexpr int kLanesPerHead = 32 / H;
  constexpr int kLog2H = H >= 16 ? 4 : H >= 8 ? 3 : H >= 4 ? 2 : H >= 2 ? 1 : 0;
#pragma unroll
  for (int st = 0; st < kLog2H; ++st) {
    const int half = H >> (st + 1), off = 16 >> st;
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const float send = up ? v[i] : v[i + half];
      const float keep = up ? v[i + half] : v[i];
      v[i] = op(keep, __shfl_xor_sync(kFull, send, off));
    }
  }
#pragma unroll
  for (int off = kLanesPerHead / 2; off >= 1; off >>= 1)
    v[0] = op(v[0], __shfl_xor_sync(kFull, v[0], off));
  const float mine = v[0];
#pragma unroll
  for (int h = 0; h < H; ++h) v[h] = __shfl_sync(kFull, mine, h * kLanesPerHead);
}

template <int H, bool MAX>
__device__ __forceinline__ void warps_reduce(float (&v)[H], int w, int nw, float* red) {
  if (nw == 1) return;
  __syncthreads();
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int h = 0; h < H; ++h) red[w * 32 + h] = v[h];
  __syncthreads();
#pragma unroll
  for (int h = 0; h < H; ++h) {
    float t = red[h];
    for (int k = 1; k < nw; ++k) t = MAX ? max_ref(t, red[k * 32 + h]) : __fadd_rn(t, red[k * 32 + h]);
    v[h] = t;
  }
}

template <int H, bool BWD, int NW>
__device__ __forceinline__ void row_softmax_vec(const SoftmaxArgs& p, uint32_t r, int w,
                                                float* red, bool vec) {
  constexpr int nw = NW;
  const int lane = threadIdx.x & 31;
  const uint32_t e0 = __ldg(p.indptr + r), e1 = __ldg(p.indptr + r + 1);
  const uint32_t n = e1 - e0;
  if (n == 0) return;
  const uint32_t step = 32u * static_cast<uint32_t>(nw);
  const uint32_t first = static_cast<uint32_t>(w * 32 + lane);
  auto erow = [&](uint32_t k) -> int64_t {
    const uint32_t j = e0 + k;
    return p.by_pos ? static_cast<int64_t>(j) : static_cast<int64_t>(__ldg(p.eids + j));
  };
  if (NW == 1 && n <= step) {
    // one step covers the row: every value is loaded once and kept in
    // registers (exp computed once); same reductions, same results
    const bool has = first < n;
    const int64_t er = has ? erow(first) : 0;
    if constexpr (!BWD) {
      float x[H], m[H], z[H];
#pragma unroll
      for (int h = 0; h < H; ++h) x[h] = -__int_as_float(0x7f800000);
      if (has) load_heads<H>(p.l + er * p.l_ld, vec, x);
#pragma unroll
      for (int h = 0; h < H; ++h) m[h] = max_ref(-__int_as_float(0x7f800000), x[h]);  // as the loop
      lane_reduce<H, true>(m);
      warps_reduce<H, true>(m, w, nw, red);
#pragma unroll
      for (int h = 0; h < H; ++h) {
        x[h] = has ? expf(__fsub_rn(x[h], m[h])) : 0.0f;
        z[h] = __fadd_rn(0.0f, x[h]);  // as the loop
      }
      lane_reduce<H, false>(z);
      warps_reduce<H, false>(z, w, nw, red);
      if (has) {
#pragma unroll
        for (int h = 0; h < H; ++h) x[h] = __fdiv_rn(x[h], z[h]);
        store_heads<H>(p.out + er * p.out_ld, vec, x);
      }
    } else {
      float a[H], g[H], sacc[H];
#pragma unroll
      for (int h = 0; h < H; ++h) a[h] = g[h] = 0.0f;
      if (has) {
        load_heads<H>(p.l + er * p.l_ld, vec, a);
        load_heads<H>(p.g + er * p.g_ld, vec, g);
      }
#pragma unroll
      for (int h = 0; h < H; ++h) sacc[h] = __fadd_rn(0.0f, __fmul_rn(a[h], g[h]));  // as the loop
      lane_reduce<H, false>(sacc);
      warps_reduce<H, false>(sacc, w, nw, red);
      if (has) {
#pragma unroll
        for (int h = 0; h < H; ++h) a[h] = __fmul_rn(a[h], __fsub_rn(g[h], sacc[h]));
        store_heads<H>(p.out + er * p.out_ld, vec, a);
      }
    }
    return;
  }
  if constexpr (!BWD) {
    float m[H];
#pragma unroll
    for (int h = 0; h < H; ++h) m[h] = -__int_as_float(0x7f800000);
#pragma unroll 4
    for (uint32_t k = first; k < n; k += step) {
      float x[H];
      load_heads<H>(p.l + erow(k) * p.l_ld, vec, x);
#pragma unroll
      for (int h = 0; h < H; ++h) m[h] = max_ref(m[h], x[h]);
    }
    lane_reduce<H, true>(m);
    warps_reduce<H, true>(m, w, nw, red);
    float z[H];
#pragma unroll
    for (int h = 0; h < H; ++h) z[h] = 0.0f;
#pragma unroll 4
    for (uint32_t k = first; k < n; k += step) {
      float x[H];
      load_heads<H>(p.l + erow(k) * p.l_ld, vec, x);
#pragma unroll
      for (int h = 0; h < H; ++h) z[h] = __fadd_rn(z[h], expf(__fsub_rn(x[h], m[h])));
    }
    lane_reduce<H, false>(z);
    warps_reduce<H, false>(z, w, nw, red);
    for (uint32_t k = first; k < n; k += step) {
      const int64_t er = erow(k);
      float x[H];
      load_heads<H>(p.l + er * p.l_ld, vec, x);
#pragma unroll
      for (int h = 0; h < H; ++h) x[h] = __fdiv_rn(expf(__fsub_rn(x[h], m[h])), z[h]);
      store_heads<H>(p.out + er * p.out_ld, vec, x);
    }
  } else {
    float sacc[H];
#pragma unroll
    for (int h = 0; h < H; ++h) sacc[h] = 0.0f;
#pragma unroll 4
    for (uint32_t k = first; k < n; k += step) {
      const int64_t er = erow(k);
      float a[H], g[H];
      load_heads<H>(p.l + er * p.l_ld, vec, a);
      load_heads<H>(p.g + er * p.g_ld, vec, g);
#pragma unroll
      for (int h = 0; h < H; ++h) sacc[h] = __fadd_rn(sacc[h], __fmul_rn(a[h], g[h]));
    }
    lane_reduce<H, false>(sacc);
    warps_reduce<H, false>(sacc, w, nw, red);
#pragma unroll 2
    for (uint32_t k = first; k < n; k += step) {
      const int64_t er = erow(k);
      float a[H], g[H];
      load_heads<H>(p.l + er * p.l_ld, vec, a);
      load_heads<H>(p.g + er * p.g_ld, vec, g);
#pragma unroll
      for (int h = 0; h < H; ++h) a[h] = __fmul_rn(a[h], __fsub_rn(g[h], sacc[h]));
      store_heads<H>(p.out + er * p.out_ld, vec, a);
    }
  }
}

// Rows are handed out in groups of kSmGrab from a counter.  With the rows
// strided statically over the persistent grid, the warp whose rows happened
// to be heavy ran twice as long as the average one: 33% warps active over
// the kernel (profiles/r04j_ncu_softmax.txt).
constexpr uint32_t kSmGrab = 4;

template <int H, bool BWD>
__global__ void __launch_bounds__(kSmWarps * 32) k_softmax_vec_rows(const SoftmaxArgs p, bool vec) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (p.counter) {
    for (;;) {
      uint32_t base = 0;
      if (lane == 0) base = atomicAdd(p.counter, kSmGrab);
      base = __shfl_sync(kFull, base, 0);
      if (base >= p.rows) break;
      const uint32_t end = min(base + kSmGrab, p.rows);
      for (uint32_t r = base; r < end; ++r) {
        const uint32_t deg = __ldg(p.indptr + r + 1) - __ldg(p.indptr + r);
        if (deg > p.long_threshold) continue;
        row_softmax_vec<H, BWD, 1>(p, r, 0, nullptr, vec);
      }
    }
    return;
  }
  const uint32_t stride = gridDim.x * kSmWarps;
  for (uint32_t r = blockIdx.x * kSmWarps + warp; r < p.rows; r += stride) {
    const uint32_t deg = __ldg(p.indptr + r + 1) - __ldg(p.indptr + r);
    if (deg > p.long_threshold) continue;
    row_softmax_vec<H, BWD, 1>(p, r, 0, nullptr, vec);
  }
}

constexpr int kSmLongWarps = 32;  // a hub row's edges spread over 1024 threads

template <int H, bool BWD>
__global__ void __launch_bounds__(kSmLongWarps * 32) k_softmax_vec_long(const SoftmaxArgs p, bool vec,
                                                                       const uint32_t* long_rows,
                                                                       uint32_t n_long) {
  __shared__ float red[kSmLongWarps * 32];
  const int warp = threadIdx.x >> 5;
  for (uint32_t i = blockIdx.x; i < n_long; i += gridDim.x) {
    row_softmax_vec<H, BWD, kSmLongWarps>(p, __ldg(long_rows + i), warp, red, vec);
    __syncthreads();
  }
}

// The hub rows (one CTA each) run on the side stream, concurrently with the
// warp-per-row kernel (measured on cfg4: 1.15 + 0.92 ms back to back).
template <int H, bool BWD>
void launch_vec(const SoftmaxArgs& p, bool vec, const uint32_t* long_rows, uint32_t n_long,
                int sms, cudaStream_t s, const SideStream& side) {
  const bool fork = n_long && side.stream;
  if (fork) {
    cudaEventRecord(side.fork, s);
    cudaStreamWaitEvent(side.stream, side.fork, 0);
  }
  // persistent grids of exactly one wave (measured: the 8-blocks-per-SM grid
  // ran in two waves at ~32% achieved occupancy)
  static int occ_rows = 0, occ_long = 0;
  if (!occ_rows) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_rows, k_softmax_vec_rows<H, BWD>,
                                                  kSmWarps * 32, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_long, k_softmax_vec_long<H, BWD>,
                                                  kSmLongWarps * 32, 0);
    occ_rows = std::max(occ_rows, 1);
    occ_long = std::max(occ_long, 1);
  }
  if (n_long) {
    const unsigned grid = std::min<unsigned>(n_long, static_cast<unsigned>(sms * occ_long));
    k_softmax_vec_long<H, BWD><<<grid, kSmLongWarps * 32, 0, fork ? side.stream : s>>>(
        p, vec, long_rows, n_long);
    note_launch();
  }
  if (p.rows) {
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(
        (p.rows + kSmWarps - 1) / kSmWarps, static_cast<uint64_t>(sms) * occ_rows));
    if (p.counter) cudaMemsetAsync(p.counter, 0, sizeof(uint32_t), s);
    k_softmax_vec_rows<H, BWD><<<grid, kSmWarps * 32, 0, s>>>(p, vec);
    note_launch();
  }
  if (fork) {
    cudaEventRecord(side.join, side.stream);
    cudaStreamWaitEvent(s, side.join, 0);
  }
}

template <bool BWD>
bool dispatch_vec(const SoftmaxArgs& p, bool vec, const uint32_t* lr, uint32_t nl, int sms,
                  cudaStream_t s, const SideStream& side) {
  switch (p.heads) {
    case 1: launch_vec<1, BWD>(p, vec, lr, nl, sms, s, side); return true;
    case 2: launch_vec<2, BWD>(p, vec, lr, nl, sms, s, side); return true;
    case 4: launch_vec<4, BWD>(p, vec, lr, nl, sms, s, side); return true;
    case 8: launch_vec<8, BWD>(p, vec, lr, nl, sms, s, side); return true;
    case 16: launch_vec<16, BWD>(p, vec, lr, nl, sms, s, side); return true;
    default: return false;
  }
}

}  // namespace

cudaError_t launch_edge_softmax(bool backward, const uint32_t* indptr, const uint32_t* eids,
                                uint32_t rows, int heads, bool by_pos, const float* l,
                                int64_t l_ld, const float* g, int64_t g_ld, float* out,
                                int64_t out_ld, const uint32_t* long_rows, uint32_t n_long,
                                uint32_t long_threshold, int num_sms, cudaStream_t s,
                                const SideStream& side, uint32_t* counter) {
  SoftmaxArgs p{indptr, eids, rows, heads, by_pos, l, l_ld, g, g_ld, out, out_ld,
                n_long ? long_threshold : 0xffffffffu, counter};
  const int sms = num_sms > 0 ? num_sms : 148;
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15u) == 0; };
  const bool vec = heads % 4 == 0 && l_ld % 4 == 0 && out_ld % 4 == 0 && al16(l) && al16(out) &&
                   (!backward || (g_ld % 4 == 0 && al16(g)));
  if (backward ? dispatch_vec<true>(p, vec, long_rows, n_long, sms, s, side)
               : dispatch_vec<false>(p, vec, long_rows, n_long, sms, s, side))
    return cudaGetLastError();
  if (rows) {
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((rows + kSmWarps - 1) / kSmWarps,
                                                                   static_cast<uint64_t>(sms) * 8));
    if (backward) k_softmax_rows<true><<<grid, kSmWarps * 32, 0, s>>>(p);
    else k_softmax_rows<false><<<grid, kSmWarps * 32, 0, s>>>(p);
    note_launch();
  }
  if (n_long) {
    const unsigned grid = std::min<unsigned>(n_long, static_cast<unsigned>(sms) * 4);
    if (backward) k_softmax_long<true><<<grid, kSmWarps * 32, 0, s>>>(p, long_rows, n_long);
    else k_softmax_long<false><<<grid, kSmWarps * 32, 0, s>>>(p, long_rows, n_long);
    note_launch();
  }
  return cudaGetLastError();
}

}  // namespace gspmm_b200

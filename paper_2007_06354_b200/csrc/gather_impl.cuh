// gather_impl.cuh -- the production owner-computes row kernel (sm_100a),
// instantiated per binary operator in gather_{copy,mul,arith}.cu.
//
// Same semantics as rows.cu / stream.cu (the reference's RowParallelSpmm
// left fold, kernels.cpp:162-195, bit for bit), built from measurements on
// B200 (scripts/mb_gather.cu, profiles/):
//
//   * random source-row gathers run fastest as 128-bit LDGs into registers
//     (7.2 TB/s for 1 KB rows, 5.0 TB/s for 400 B rows) -- faster than one
//     TMA bulk copy per row (5.9 / 1.8 TB/s), whose per-SM request rate caps
//     small rows; so rows are gathered with LDG.128 into a register
//     ping-pong: the next batch's loads are in flight while the current
//     batch is folded;
//   * persistent CTAs pull WORK UNITS (the device plan: edge-balanced
//     segments of consecutive rows, and column slices of long rows) from a
//     global counter, first units interleaved across SMs;
//   * WIDE units: lanes own 4 (or 8) output columns, one edge per warp load
//     instruction (512 B or 1 KB);  NARROW units (32-column slices of long
//     rows): lane = (edge group g, column quad i), four edges per warp load
//     instruction; the four edges are then folded in order by the column
//     owners through warp shuffles -- the fold stays sequential per column;
//   * neighbour ids / scalar edge operands arrive as coalesced 32-edge
//     windows prefetched one window (NARROW: two) ahead and broadcast with
//     shuffles; row ends likewise;
//   * fused epilogue: zero-degree fixup, mean, argmax; each output row is
//     written exactly once.
#pragma once
#include <type_traits>
#include "device_ops.cuh"
#include "stream.h"
#include "tma.cuh"

namespace gspmm_b200 {
namespace gather_detail {

constexpr int kThreads = 256;
// segment kernel geometry: edges per warp batch (<=128 / <=256 columns) and
// minimum resident blocks per SM.  Measured on B200 (scripts/var_ab.sh): warp
// parallelism beats per-warp depth -- U=8 at 3 blocks/SM for <=128 columns,
// U=2 at 4 blocks/SM (32 warps) for 256 columns: 94% of HBM on uniform graphs.
#ifndef GATHER_U1
#define GATHER_U1 8
#endif
#ifndef GATHER_U2
#define GATHER_U2 2
#endif
#ifndef GATHER_MINB1
#define GATHER_MINB1 3
#endif
#ifndef GATHER_MINB2
#define GATHER_MINB2 4
#endif
// wide rows (VPL 5: up to 640 columns in one unit, e.g. cfg5's 602): copy /
// scalar-weighted sums only
#ifndef GATHER_U5
#define GATHER_U5 2
#endif
// Cache policy of the segment kernel's streams (read or written once per
// pass): evict-first stores of the output rows / loads of the id windows.
// Measured on the cfg2 bench step: evict-first output stores 3.79 -> 3.86 ms
// (off); evict-first id loads 3.79 -> 3.79 (on, neutral).
#ifndef GATHER_STREAM_OUT
#define GATHER_STREAM_OUT 0
#endif
#ifndef GATHER_STREAM_IN
#define GATHER_STREAM_IN 1
#endif
// L2 prefetch distance of the segment kernel, in batches (0 = off).
// Measured slower at every distance (cfg2 1.82 -> 1.89 / 1.91 / 2.01 ms at
// 2 / 4 / 8 batches; uniform er256 2.41 -> 3.96 ms at 8): kept for study.
#ifndef GATHER_PF
#define GATHER_PF 0
#endif
#ifndef GATHER_MINB5
#define GATHER_MINB5 2

#endif

struct UnitCtx {
  uint32_t r0, r1, e0, e1;
  int c0, cw;
};

// Row-boundary state of a unit: windows of indptr (lane k <-> rb + 1 + k).
struct RowCursor {
  uint32_t rb, rwin, rnxt, r, row_start, row_end, r1;
  __device__ __forceinline__ void init(const uint32_t* indptr, uint32_t r0_, uint32_t r1_,
                                       uint32_t e0, int lane) {
    rb = r0_;
    r1 = r1_;
    rwin = 0;
    rnxt = 0;
    if (r0_ + 1 + lane <= r1_) rwin = __ldg(indptr + r0_ + 1 + lane);
    if (r0_ + 33 + lane <= r1_) rnxt = __ldg(indptr + r0_ + 33 + lane);
    r = r0_;
    row_start = e0;
    row_end = __shfl_sync(kFull, rwin, 0);
  }
  __device__ __forceinline__ void advance(const uint32_t* indptr, int lane) {
    ++r;
    row_start = row_end;
    if (r - rb >= 32u) {
      rb += 32u;
      rwin = rnxt;
      rnxt = 0;
      if (rb + 33 + lane <= r1) rnxt = __ldg(indptr + rb + 33 + lane);
    }
    row_end = __shfl_sync(kFull, rwin, static_cast<int>(r - rb) & 31);
  }
};

// PART: the kernel instance serves source-blocked passes (acc_in / epi /
// deg_indptr honoured); the plain instances compile those paths out
// (measured: the runtime checks cost up to 8% on cfg3 max + argmax).
// ARG: 0 = no argmax; 1 = track the CSR position of the winner (the ids are
// looked up at the row's flush); 2 = track the winning neighbour id itself
// (gathered-row kernels with only arg_other requested: no lookup latency at
// the flush, measured 0.6 ms of cfg3's 7.7).
template <int VPL, int ROP, int ARG, bool PART>
struct Acc {
  float a[VPL][4];
  uint32_t arg[VPL][4];
  __device__ __forceinline__ void reset() {
#pragma unroll
    for (int v = 0; v < VPL; ++v)
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        a[v][t] = red_identity<ROP>();
        arg[v][t] = 0xffffffffu;
      }
  }
  __device__ __forceinline__ void fold(int v, const float (&m)[4], uint32_t j) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if constexpr (ARG) {
        if (red_wins<ROP>(a[v][t], m[t])) {
          a[v][t] = m[t];
          arg[v][t] = j;
        }
      } else {
        a[v][t] = red_combine<ROP>(a[v][t], m[t]);
      }
    }
  }
  // Start of owner row r: the identity, or (source-blocked passes after the
  // first) the partial fold of the earlier passes.
  __device__ __forceinline__ void begin(const RowLaunch& L, uint32_t r, int c0, int cw, int lane) {
    reset();
    if (!PART || L.acc_in == nullptr) return;
    const float* prow = L.acc_in + static_cast<int64_t>(r) * L.out_ld + c0;
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      const int c = lane * 4 + v * 128;
      if (c + 4 <= cw) {
        const float4 q = *reinterpret_cast<const float4*>(prow + c);
        a[v][0] = q.x;
        a[v][1] = q.y;
        a[v][2] = q.z;
        a[v][3] = q.w;
      } else {
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (c + t < cw) a[v][t] = prow[c + t];
      }
    }
  }
  // Epilogue of owner row r over columns [c0 + c, ...) of this lane.
  __device__ __forceinline__ void store(const RowLaunch& L, uint32_t r, uint32_t deg, int c0,
                                        int cw, int v, int c) {
    if (c >= cw) return;
    float o[4];
    const bool fix = !PART || L.epi != 1;  // a partial pass stores the raw fold
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      float x = a[v][t];
      if constexpr (ROP == R_MAX || ROP == R_MIN) {
        if (fix && deg == 0) x = 0.0f;
      }
      if (fix && L.mean) x = deg ? __fdiv_rn(x, __uint2float_rn(deg)) : 0.0f;
      o[t] = x;
    }
    float* orow = L.out + static_cast<int64_t>(r) * L.out_ld + c0;
    if (c + 4 <= cw) {
#if GATHER_STREAM_OUT
      // written once, never re-read by the pass: evict-first, so the output
      // stream does not displace hot source rows from L2
      __stcs(reinterpret_cast<float4*>(orow + c), make_float4(o[0], o[1], o[2], o[3]));
#else
      store_vec<4>(orow + c, o);
#endif
    } else {
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (c + t < cw) orow[c + t] = o[t];
    }
    if constexpr (ARG) {
      const int64_t ab = static_cast<int64_t>(r) * L.arg_ld + c0 + c;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        if (c + t >= cw) break;
        const bool none = arg[v][t] == 0xffffffffu;
        if constexpr (ARG == 2) {
          L.arg_other[ab + t] = none ? -1 : static_cast<int32_t>(arg[v][t]);
        } else {
          if (L.arg_other)
            L.arg_other[ab + t] = none ? -1 : static_cast<int32_t>(__ldg(L.indices + arg[v][t]));
          if (L.arg_edge)
            L.arg_edge[ab + t] = none ? -1 : static_cast<int32_t>(__ldg(L.eids + arg[v][t]));
        }
      }
    }
  }
};

// Small per-edge operand value for output columns starting at c (absolute).
__device__ __forceinline__ float small_value(const RowLaunch& L, int rw, uint32_t other,
                                             uint32_t eid, uint32_t j, int cabs) {
  const int64_t rr = operand_row(L.rhs.role, 0, other, eid, j);
  const int h = rw == 1 ? 0 : cabs / L.rhs.group;
  return __ldg(L.rhs.base + rr * L.rhs.ld + h);
}

// ------------------------------------------------------------------ WIDE
// One edge per warp load instruction; lanes own columns lane*4 + v*128.
// Batches of U edges: all U rows' loads are issued, then folded in edge
// order -- straight through when the batch lies inside the current row (the
// common case), edge by edge with row flushes otherwise.
// The small per-edge operand is resolved at compile time (SK): none; a
// scalar per edge gathered once per 32-edge id window by the lane owning the
// edge and broadcast by shuffle (by CSR position, edge id or neighbour; also
// the per-neighbour scale of the mean backward); or per-head values.
// Measured: the previous, runtime-dispatched form executed ~125 warp
// instructions per 1 KB edge (branches, constant-bank reloads, spills) and
// kept the SMs ~70% issue-busy at 2.5 TB/s of DRAM traffic.
enum SmallKind : int { SK_NONE = 0, SK_WIN = 1, SK_SCALE = 2, SK_HEAD = 3 };

template <int VPL, int U, int BOP, int ROP, int ARG, int SK, bool LO, bool PART>
__device__ __forceinline__ void wide_unit(const RowLaunch& L, const UnitCtx& u, bool need_eid,
                                          const float* sbase, int64_t sld, int32_t srole,
                                          int lane) {
  // per-lane row-relative byte offsets of the VPL column quads; quads past
  // the slice read column 0 (always inside the row) and are never stored
  const char* lrow[VPL];
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    const int c = lane * 4 + v * 128;
    lrow[v] = reinterpret_cast<const char*>(L.lhs.base + u.c0 + (c < u.cw ? c : 0));
  }
  const uint32_t ldb = static_cast<uint32_t>(L.lhs.ld) * 4u;  // row stride in bytes
  const int32_t lrole = L.lhs.role;
  const uint32_t* __restrict__ indices = L.indices;
  const uint32_t* __restrict__ eids = L.eids;
  int hv[VPL];  // SK_HEAD: head of each of this lane's column quads
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    const int c = lane * 4 + v * 128;
    hv[v] = SK == SK_HEAD ? (u.c0 + (c < u.cw ? c : 0)) / L.rhs.group : 0;
  }

  RowCursor rc;
  rc.init(L.indptr, u.r0, u.r1, u.e0, lane);
  Acc<VPL, ROP, ARG, PART> acc;
  acc.begin(L, rc.r, u.c0, u.cw, lane);

  // id windows: lane k <-> edge e0 + 32w + k; the next window is in flight
  uint32_t win_o = 0, win_e = 0, nxt_o = 0, nxt_e = 0;
  float win_r = 0.0f, nxt_r = 0.0f;
  auto load_win = [&](uint32_t w, uint32_t& o, uint32_t& e, float& rv) {
    const uint32_t j = u.e0 + 32u * w + lane;
    if (j < u.e1) {
#if GATHER_STREAM_IN
      o = __ldcs(indices + j);  // read once: evict-first
      if (need_eid) e = __ldcs(eids + j);
#else
      o = __ldg(indices + j);
      if (need_eid) e = __ldg(eids + j);
#endif
      if constexpr (SK == SK_WIN || SK == SK_SCALE) {
        const uint32_t row = srole == ROLE_POS ? j : srole == ROLE_EID ? e : o;
        rv = __ldg(sbase + static_cast<int64_t>(row) * sld);
      }
    }
  };
  load_win(0, win_o, win_e, win_r);
  load_win(1, nxt_o, nxt_e, nxt_r);
  constexpr int kPerWin = 32 / U;
  const uint32_t n_batches = (u.e1 - u.e0 + U - 1) / U;

  auto flush = [&]() {
    const uint32_t deg = PART && L.deg_indptr
                             ? __ldg(L.deg_indptr + rc.r + 1) - __ldg(L.deg_indptr + rc.r)
                             : rc.row_end - rc.row_start;
#pragma unroll
    for (int v = 0; v < VPL; ++v) acc.store(L, rc.r, deg, u.c0, u.cw, v, lane * 4 + v * 128);
  };

  uint32_t j = u.e0;  // next edge to fold
  for (uint32_t b = 0; b < n_batches; ++b) {
    if (b != 0 && (b % kPerWin) == 0) {  // entering the next id window
      win_o = nxt_o;
      win_e = nxt_e;
      win_r = nxt_r;
      load_win(b / kPerWin + 1, nxt_o, nxt_e, nxt_r);
    }
    const uint32_t jb = u.e0 + b * U;
    const uint32_t n = min(static_cast<uint32_t>(U), u.e1 - jb);
    if constexpr (GATHER_PF > 0 && LO) {
      // L2 prefetch of the rows GATHER_PF batches ahead: memory-level
      // parallelism beyond the registers' ping-pong, at one instruction per
      // lane (lane = (edge, 128-byte line of its slice))
      constexpr int kLines = VPL * 4;  // 128-byte lines per <= VPL*128-column slice
      constexpr int kEdges = 32 / kLines < U ? 32 / kLines : U;
      const uint32_t q = (b + GATHER_PF) * U + static_cast<uint32_t>(lane / kLines);  // unit edge
      const int line = lane % kLines;
      const uint32_t src_lane = q & 31u;
      const uint32_t o_cur = __shfl_sync(kFull, win_o, src_lane);
      const uint32_t o_nxt = __shfl_sync(kFull, nxt_o, src_lane);
      const uint32_t wq = q / 32u, wb = b / static_cast<uint32_t>(kPerWin);
      if (lane / kLines < kEdges && u.e0 + q < u.e1 && line * 32 < u.cw && (wq == wb || wq == wb + 1))
        prefetch_l2(reinterpret_cast<const char*>(L.lhs.base + u.c0 + line * 32) +
                    static_cast<uint64_t>(wq == wb ? o_cur : o_nxt) * ldb);
    }
    float4 x[U][VPL];
    float r[U][SK == SK_HEAD ? VPL : 1];
    uint32_t okey[ARG == 2 ? U : 1];  // ARG 2: the neighbour id of each edge
    // loads: unconditional (a tail batch re-reads its last edge), so the
    // batch is straight-line code
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int kk = static_cast<uint32_t>(k) < n ? k : static_cast<int>(n) - 1;
      const int sl = static_cast<int>((b % kPerWin) * U) + kk;
      const uint32_t o = __shfl_sync(kFull, win_o, sl);
      uint32_t e = 0;
      if (!LO || SK == SK_HEAD) {
        if (need_eid) e = __shfl_sync(kFull, win_e, sl);
      }
      if constexpr (SK == SK_WIN || SK == SK_SCALE) r[k][0] = __shfl_sync(kFull, win_r, sl);
      if constexpr (ARG == 2) okey[k] = o;
      const uint32_t lr = LO ? o : static_cast<uint32_t>(operand_row(lrole, 0, o, e, jb + kk));
#pragma unroll
      for (int v = 0; v < VPL; ++v)
        x[k][v] = __ldg(reinterpret_cast<const float4*>(lrow[v] + static_cast<uint64_t>(lr) * ldb));
      if constexpr (SK == SK_HEAD) {
        const float* sp = L.rhs.base + operand_row(L.rhs.role, 0, o, e, jb + kk) * L.rhs.ld;
#pragma unroll
        for (int v = 0; v < VPL; ++v) r[k][v] = __ldg(sp + hv[v]);
      }
    }
    // quads past the slice fold garbage that is never stored
    auto fold_edge = [&](int k, uint32_t jpos) {
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        const float xs[4] = {x[k][v].x, x[k][v].y, x[k][v].z, x[k][v].w};
        float m[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          if constexpr (SK == SK_NONE) m[t] = bin_apply<BOP>(xs[t], 0.0f);
          else if constexpr (SK == SK_SCALE) m[t] = __fmul_rn(bin_apply<BOP>(xs[t], 0.0f), r[k][0]);
          else if constexpr (SK == SK_WIN) m[t] = bin_apply<BOP>(xs[t], r[k][0]);
          else m[t] = bin_apply<BOP>(xs[t], r[k][v]);
        }
        if constexpr (ARG == 2) acc.fold(v, m, okey[k]);
        else acc.fold(v, m, jpos);
      }
    };
    if (n == static_cast<uint32_t>(U) && rc.row_end - j >= static_cast<uint32_t>(U)) {
      // the whole batch folds into the current row
#pragma unroll
      for (int k = 0; k < U; ++k) fold_edge(k, j + k);
      j += U;
    } else {
#pragma unroll
      for (int k = 0; k < U; ++k) {
        if (static_cast<uint32_t>(k) < n) {
          while (j == rc.row_end) {
            flush();
            rc.advance(L.indptr, lane);
            acc.begin(L, rc.r, u.c0, u.cw, lane);
          }
          fold_edge(k, j);
          ++j;
        }
      }
    }
  }
  // the current row and trailing empty rows
  while (rc.r < u.r1) {
    flush();
    if (rc.r + 1 < u.r1) {
      rc.advance(L.indptr, lane);
      acc.begin(L, rc.r, u.c0, u.cw, lane);
    } else {
      ++rc.r;
    }
  }
}

// -------------------------------------------------------------- LONG ROWS
// One column slice (32 / 64 / 128 / 256 floats) of one long row per CTA: the
// 16 warps gather a round of R edges with LDG.128 into registers while the
// previous round, staged in shared memory, is folded by the column owners
// (thread t owns column t) in canonical edge order.  A lone warp cannot keep
// enough bytes in flight for a 66k-329k-edge row (one owner must see every
// edge in order); a CTA keeps ~128 KB in flight, and the heaviest rows are
// cut into narrow slices so several CTAs on several SMs stream one row.
// Narrow slices pack epi = 128 / slice edges into each warp load instruction
// (lane = edge group g x column quad i).
constexpr int kLongThreads = 512;

// Shared memory is carved out of the same 228 KB as L1, and L1 tracks the
// in-flight LDG misses: the round buffer is kept at 96 KB (measured: a 192 KB
// carve-out halved the long-row stream rate).
template <int VPL>
struct LongGeom {
  static constexpr int U = VPL == 1 ? 12 : 6;          // load instructions per warp per round
  static constexpr int kWarps = kLongThreads / 32;
  static constexpr int kMaxSmall = 16;                  // staged small floats per edge
  // round: R = kWarps * U * epi edges of slot_f floats; slot_f * epi = 128
  // for narrow slices, 128 * VPL otherwise -> the data buffer is constant
  static constexpr size_t data_floats() { return static_cast<size_t>(kWarps) * U * 128 * VPL; }
  static constexpr size_t max_edges() { return static_cast<size_t>(kWarps) * U * 4; }
  static constexpr size_t smem_bytes(int rws) {
    return sizeof(float) * (data_floats() + max_edges() * static_cast<size_t>(rws));
  }
};

template <int VPL, int BOP, int ROP, bool ARG, bool SMALL>
__global__ void __launch_bounds__(kLongThreads, 1) k_long(const StreamLaunch p) {
  using G = LongGeom<VPL>;
  constexpr int U = G::U;
  extern __shared__ __align__(16) float sm[];
  __shared__ uint32_t s_unit;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const RowLaunch& L = p.row;
  const int rw = SMALL ? p.rhs_width : 0;
  const bool scale_on = SMALL && L.other_scale != nullptr;
  const int rws = SMALL ? (rw > 0 ? rw : 1) : 0;  // staged small floats per edge
  const bool need_eid = L.lhs.role == ROLE_EID || (rw && L.rhs.role == ROLE_EID);
  float* buf = sm;
  float* sbuf = sm + G::data_floats();

  for (;;) {
    if (tid == 0) s_unit = atomicAdd(p.counter, 1u);
    __syncthreads();
    const uint32_t unit = s_unit;
    __syncthreads();
    if (unit >= p.n_units) break;
    const unsigned long long t0 = p.trace ? globaltimer_ns() : 0ull;
    // units: first the narrow slices of the heaviest rows, then wide slices
    uint32_t li, slc;
    int sw;
    if (unit < p.n_xl_units) {
      li = unit / p.xl_slices;
      slc = unit - li * p.xl_slices;
      sw = p.xl_sw;
    } else {
      const uint32_t v = unit - p.n_xl_units;
      li = p.n_xl + v / p.long_slices;
      slc = v - (li - p.n_xl) * p.long_slices;
      sw = p.long_sw;
    }
    const uint32_t r = __ldg(p.long_rows + li);
    const int c0 = static_cast<int>(slc) * sw;
    const int cw = min(sw, L.width - c0);
    const int slot_f = cw <= 32 ? 32 : cw <= 64 ? 64 : cw <= 128 ? 128 : 256;
    const int epi = slot_f > 128 ? 1 : 128 / slot_f;  // edges per warp load instruction
    const int lpe = 32 / epi;                          // lanes per edge
    const int g = lane / lpe, i = lane - g * lpe;
    const int epw = U * epi;                           // edges per warp per round
    const uint32_t R = static_cast<uint32_t>(G::kWarps * epw);
    const uint32_t e0 = __ldg(L.indptr + r), e1 = __ldg(L.indptr + r + 1);
    const uint32_t n = e1 - e0;
    const uint32_t rounds = (n + R - 1) / R;
    const float* lbase = L.lhs.base + c0 + i * 4;
    bool col_ok[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) col_ok[v] = i * 4 + v * 128 < cw && (v == 0 || slot_f > 128);
    int hv[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) hv[v] = (SMALL && rw > 1) ? (c0 + i * 4 + v * 128) / L.rhs.group : 0;

    // ids of this warp's epw (<= 64) edges of a round: two 32-id windows
    auto load_ids = [&](uint32_t rd, uint32_t (&o)[2], uint32_t (&e)[2]) {
      const uint32_t jb = e0 + rd * R + warp * epw;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t j = jb + 32u * h + lane;
        if (32 * h < epw && static_cast<int>(32 * h + lane) < epw && j < e1) {
          o[h] = __ldg(L.indices + j);
          if (need_eid) e[h] = __ldg(L.eids + j);
        }
      }
    };
    float4 x[U][VPL];
    float sv[U][VPL];
    auto issue = [&](uint32_t rd, const uint32_t (&o_w)[2], const uint32_t (&e_w)[2]) {
      const uint32_t jb = e0 + rd * R + warp * epw;
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int q = k * epi + g;  // edge of this lane within the warp's chunk
        const uint32_t o0 = __shfl_sync(kFull, o_w[0], q & 31);
        const uint32_t o1 = __shfl_sync(kFull, o_w[1], q & 31);
        const uint32_t o = q < 32 ? o0 : o1;
        uint32_t e = 0;
        if (need_eid) {
          const uint32_t a0 = __shfl_sync(kFull, e_w[0], q & 31);
          const uint32_t a1 = __shfl_sync(kFull, e_w[1], q & 31);
          e = q < 32 ? a0 : a1;
        }
        const uint32_t j = jb + q;
        if (j < e1) {
          const float* src = lbase + operand_row(L.lhs.role, 0, o, e, j) * L.lhs.ld;
#pragma unroll
          for (int v = 0; v < VPL; ++v)
            if (col_ok[v]) x[k][v] = __ldg(reinterpret_cast<const float4*>(src + v * 128));
          if constexpr (SMALL) {
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
              if (rw > 0) {
                sv[k][v] = col_ok[v]
                    ? __ldg(L.rhs.base + operand_row(L.rhs.role, 0, o, e, j) * L.rhs.ld + hv[v])
                    : 0.0f;
              } else if (scale_on) {
                sv[k][v] = __ldg(L.other_scale + o);
              }
            }
          }
        }
      }
    };
    auto stage = [&](uint32_t rd) {
      const uint32_t jb = e0 + rd * R + warp * epw;
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int q = k * epi + g;
        if (jb + q < e1) {
          const int eidx = warp * epw + q;  // edge within the round
          float* dst = buf + static_cast<size_t>(eidx) * slot_f + i * 4;
#pragma unroll
          for (int v = 0; v < VPL; ++v)
            if (col_ok[v]) *reinterpret_cast<float4*>(dst + v * 128) = x[k][v];
          if constexpr (SMALL) {
#pragma unroll
            for (int v = 0; v < VPL; ++v)
              if (col_ok[v]) sbuf[eidx * rws + hv[v]] = sv[k][v];
          }
        }
      }
    };

    // the fold: thread tid < cw owns column c0 + tid
    float acc = red_identity<ROP>();
    uint32_t arg = 0xffffffffu;
    const int hcol = (SMALL && rw > 1) ? (c0 + tid) / L.rhs.group : 0;
    uint32_t ida[2] = {0, 0}, idea[2] = {0, 0}, idb[2] = {0, 0}, ideb[2] = {0, 0};
    load_ids(0, ida, idea);
    load_ids(1, idb, ideb);
    issue(0, ida, idea);
    stage(0);
    __syncthreads();
    for (uint32_t k = 0; k < rounds; ++k) {
      if (k + 1 < rounds) {
        issue(k + 1, idb, ideb);  // loads in flight during the fold below
        load_ids(k + 2, idb, ideb);
      }
      if (tid < cw) {
        const uint32_t cnt = min(R, n - k * R);
        const float* col = buf + tid;
        const int soff = SMALL && rw > 0 ? hcol : 0;
#pragma unroll 4
        for (uint32_t e = 0; e < cnt; ++e) {
          float m = col[static_cast<size_t>(e) * slot_f];
          if constexpr (SMALL) {
            if (rw > 0) m = bin_apply<BOP>(m, sbuf[e * rws + soff]);
            else m = __fmul_rn(bin_apply<BOP>(m, 0.0f), sbuf[e]);
          } else {
            m = bin_apply<BOP>(m, 0.0f);
          }
          if constexpr (ARG) {
            if (red_wins<ROP>(acc, m)) {
              acc = m;
              arg = e0 + k * R + e;
            }
          } else {
            acc = red_combine<ROP>(acc, m);
          }
        }
      }
      __syncthreads();
      if (k + 1 < rounds) stage(k + 1);
      __syncthreads();
    }
    if (tid < cw) {
      float a = acc;
      if constexpr (ROP == R_MAX || ROP == R_MIN) {
        if (n == 0) a = 0.0f;
      }
      if (L.mean) a = n ? __fdiv_rn(a, __uint2float_rn(n)) : 0.0f;
      L.out[static_cast<int64_t>(r) * L.out_ld + c0 + tid] = a;
      if constexpr (ARG) {
        const int64_t ab = static_cast<int64_t>(r) * L.arg_ld + c0 + tid;
        const bool none = arg == 0xffffffffu;
        if (L.arg_other)
          L.arg_other[ab] = none ? -1 : static_cast<int32_t>(__ldg(L.indices + arg));
        if (L.arg_edge) L.arg_edge[ab] = none ? -1 : static_cast<int32_t>(__ldg(L.eids + arg));
      }
    }
    if (p.trace && tid == 0) {
      unsigned long long* t = p.trace + 4ull * unit;
      t[0] = t0;
      t[1] = globaltimer_ns();
      t[2] = (static_cast<unsigned long long>(smid()) << 32) | 0xffffu;
      t[3] = n;
    }
    __syncthreads();
  }
}

// ------------------------------------- LONG ROWS, warp-specialised LDGSTS
// The production long-row CTA.  One column slice (<= 512 floats) of one long
// row per unit, streamed through a shared-memory ring of NB stages of R edges
// by cp.async (LDGSTS: global -> shared, no registers hold data in flight).
// Producers and consumers are decoupled by per-stage mbarriers: 12 producer
// warps issue the copies of stage s as soon as the consumers released its
// slot (empty[s % NB]); 4 consumer warps -- the column owners, one column
// (narrow slices) or four (wide) per thread -- fold stage s in canonical edge
// order as soon as its copies landed (full[s % NB]).  A copy costs one id
// (shared-memory broadcast) and one 64-bit address per lane per edge.  The
// ids of stage s + NB ride in stage s's copy group into a 2*NB id ring, so
// issuing never waits on a global load.
// Measured on B200 (scripts/mb_long.cu, scripts/var_long.sh): per-SM stream
// rate grows with producer warps up to ~12 and with 48 KB stages; a CTA
// barrier per stage (fold delaying the next issue) cost ~25%, and feeding
// addresses from ids loaded into registers one stage earlier capped a CTA at
// one id-load latency per stage (~20 GB/s).
#ifndef WS_NB
#define WS_NB 3
#endif
#ifndef WS_DF
#define WS_DF 12288
#endif
#ifndef WS_P
#define WS_P 12
#endif
// LONG_WS_MINB=2 caps the CTA at 64 registers so that two segment blocks
// (instead of one) fit beside it: measured no faster (cfg3 mean 5.46 ->
// 5.71 ms, cfg4 7.1 -> 7.1 ms), so the default stays 1
#ifndef LONG_WS_MINB
#define LONG_WS_MINB 1
#endif
constexpr int kWsProducers = WS_P, kWsConsumers = 4;
constexpr int kWsThreads = 32 * (kWsProducers + kWsConsumers);
struct WsGeom {
  static constexpr int NB = WS_NB;
  static constexpr int DF = WS_DF;          // data floats per stage
  static constexpr int SF = DF / 6;         // small-operand floats per stage
  static constexpr int MR = 256;            // max edges per stage
  static constexpr size_t smem_bytes(bool small) {
    return sizeof(float) * (static_cast<size_t>(NB) * (DF + (small ? SF : 0)) + 4ull * NB * MR) +
           2ull * NB * sizeof(uint64_t);
  }
};

template <int BOP, int ROP, bool ARG, int SK>
__global__ void __launch_bounds__(kWsThreads, LONG_WS_MINB) k_long_ws(const StreamLaunch p) {
  using G = WsGeom;
  constexpr int NB = G::NB;
  constexpr bool SMALL = SK != SK_NONE;
  extern __shared__ __align__(16) float sm[];
  __shared__ uint32_t s_unit;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool producer = warp < kWsProducers;
  const RowLaunch& L = p.row;
  const int rw = SMALL ? p.rhs_width : 0;
  const bool scale_on = SMALL && L.other_scale != nullptr;
  const bool need_eid = L.lhs.role == ROLE_EID || (rw && L.rhs.role == ROLE_EID);
  float* sdata = sm;                                                    // NB x DF
  uint32_t* sid = reinterpret_cast<uint32_t*>(sm + static_cast<size_t>(NB) * G::DF);  // 2NB x MR
  uint32_t* seid = sid + 2 * NB * G::MR;                                // 2NB x MR
  float* ssmall = reinterpret_cast<float*>(seid + 2 * NB * G::MR);      // NB x SF
  uint64_t* full = reinterpret_cast<uint64_t*>(ssmall + (SMALL ? NB * G::SF : 0));
  uint64_t* empty = full + NB;
  if (tid == 0) {
    for (int b = 0; b < NB; ++b) {
      mbar_init(&full[b], kWsProducers);
      mbar_init(&empty[b], kWsConsumers);
    }
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t gs0 = 0;  // stages this CTA ran before the current unit (ring position)

  for (;;) {
    if (tid == 0) s_unit = atomicAdd(p.counter, 1u);
    __syncthreads();
    const uint32_t unit = s_unit;
    __syncthreads();
    if (unit >= p.n_units) break;
    const unsigned long long t0 = p.trace ? globaltimer_ns() : 0ull;
    uint32_t li, slc;
    int sw;
    if (unit < p.n_xl_units) {
      li = unit / p.xl_slices;
      slc = unit - li * p.xl_slices;
      sw = p.xl_sw;
    } else {
      const uint32_t v = unit - p.n_xl_units;
      li = p.n_xl + v / p.long_slices;
      slc = v - (li - p.n_xl) * p.long_slices;
      sw = p.long_sw;
    }
    const uint32_t r = __ldg(p.long_rows + li);
    const int c0 = static_cast<int>(slc) * sw;
    const int cw = min(sw, L.width - c0);
    const int slot_f = (cw + 3) & ~3;
    const int qpe = slot_f >> 2;
    const int cq = (cw + 3) >> 2;
    const int h0 = (SMALL && rw > 1) ? c0 / L.rhs.group : 0;
    const int nh = SMALL ? ((rw > 1) ? (c0 + cw - 1) / L.rhs.group - h0 + 1 : 1) : 1;
    uint32_t R = static_cast<uint32_t>(G::DF / slot_f);
    if (R > static_cast<uint32_t>(G::MR)) R = G::MR;
    if (SMALL && R * nh > static_cast<uint32_t>(G::SF)) R = G::SF / nh;
    const uint32_t e0 = __ldg(L.indptr + r), e1 = __ldg(L.indptr + r + 1);
    const uint32_t n = e1 - e0;
    const uint32_t rounds = (n + R - 1) / R;

    if (producer) {
      const int ptid = tid;  // 0 .. 32 * kWsProducers - 1
      const int lpe = qpe >= 32 ? 32 : qpe > 8 ? (qpe > 16 ? 32 : 16) : qpe > 4 ? 8 : qpe > 2 ? 4 : qpe;
      const int epi = 32 / lpe;
      const int sub = lane / lpe, il = lane - sub * lpe;
      const int tpe = (qpe + lpe - 1) / lpe;
      const uint32_t ngroups = (R + epi - 1) / epi;
      const float* lbase = L.lhs.base + c0 + il * 4;
      const int64_t lld = L.lhs.ld;
      const int32_t lrole = L.lhs.role;
      auto fetch_ids = [&](uint32_t m) {  // ids of unit stage m -> id slot (gs0 + m) % 2NB
        if (m >= rounds) return;
        const uint32_t slot = (gs0 + m) % (2 * NB);
        for (uint32_t t = static_cast<uint32_t>(ptid); t < R; t += 32 * kWsProducers) {
          const uint32_t j = e0 + m * R + t;
          if (j < e1) {
            cp_async_4(sid + slot * G::MR + t, L.indices + j);
            if (need_eid) cp_async_4(seid + slot * G::MR + t, L.eids + j);
          }
        }
      };
      // prologue: ids of the first NB stages, visible to every producer
      for (uint32_t m = 0; m < static_cast<uint32_t>(NB); ++m) fetch_ids(m);
      cp_async_commit();
      cp_async_wait_group<0>();
      named_barrier_sync(1, 32 * kWsProducers);
      // per-lane constants of the copy loop: which of the <= 4 quads of an
      // edge this lane copies, source / shared byte offsets
      uint32_t tmask = 0;
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (t < tpe && il + t * lpe < cq) tmask |= 1u << t;
      const char* lsrc = reinterpret_cast<const char*>(lbase);
      const uint32_t ldb = static_cast<uint32_t>(lld) * 4u;
      const uint32_t slot_b = static_cast<uint32_t>(slot_f) * 4u;
      const uint32_t tstep = static_cast<uint32_t>(lpe) * 16u;
      constexpr bool small1 = SK == SK_WIN || SK == SK_SCALE;
      const float* s1base = rw == 1 ? L.rhs.base : L.other_scale;
      const int64_t s1ld = rw == 1 ? L.rhs.ld : 1;
      const int32_t s1role = rw == 1 ? L.rhs.role : static_cast<int32_t>(ROLE_OTHER);
      for (uint32_t s = 0; s < rounds; ++s) {
        const uint32_t gsi = gs0 + s;
        const int b = static_cast<int>(gsi % NB);
        if (gsi >= static_cast<uint32_t>(NB)) mbar_wait(&empty[b], ((gsi / NB) - 1) & 1u);
        const uint32_t islot = gsi % (2 * NB);
        const uint32_t* io = sid + islot * G::MR;
        const uint32_t* ie = seid + islot * G::MR;
        const uint32_t sd = smem_u32(sdata + static_cast<size_t>(b) * G::DF) + static_cast<uint32_t>(il) * 16u;
        float* bs = ssmall + static_cast<size_t>(b) * G::SF;
        const uint32_t jr0 = s * R;
        const uint32_t cnt = min(R, n - jr0);
        const uint32_t gcount = (cnt + epi - 1) / epi;
        for (uint32_t g = static_cast<uint32_t>(warp); g < gcount; g += kWsProducers) {
          const uint32_t q = g * epi + sub;
          if (q >= cnt) continue;
          const uint32_t j = e0 + jr0 + q;
          const uint32_t o = io[q];
          const uint32_t e = need_eid ? ie[q] : 0u;
          const uint32_t row = lrole == ROLE_OTHER ? o : static_cast<uint32_t>(operand_row(lrole, 0, o, e, j));
          const char* src = lsrc + static_cast<uint64_t>(row) * ldb;
          const uint32_t d = sd + q * slot_b;
#pragma unroll
          for (int t = 0; t < 4; ++t)
            if ((tmask >> t) & 1u) cp_async_16_s(d + t * tstep, src + t * tstep);
          if constexpr (SMALL) {
            if (small1) {
              if (il == 0) {
                const uint32_t sr = s1role == ROLE_POS ? j : s1role == ROLE_EID ? e : o;
                cp_async_4(bs + q, s1base + static_cast<int64_t>(sr) * s1ld);
              }
            } else {
              const float* sp = L.rhs.base + operand_row(L.rhs.role, 0, o, e, j) * L.rhs.ld + h0;
              for (int h = il; h < nh; h += lpe) cp_async_4(bs + q * nh + h, sp + h);
            }
          }
        }
        fetch_ids(s + NB);
        cp_async_arrive(&full[b]);
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[b]);
      }
      cp_async_wait_group<0>();
    } else {
      const int ctid = tid - 32 * kWsProducers;  // 0 .. 127
      auto run = [&](auto fw_tag) {
        constexpr int FW = decltype(fw_tag)::value;
        const int cc = ctid * FW;
        const bool own = cc < cw;
        const int hrel = (SMALL && rw > 1) ? (c0 + cc) / L.rhs.group - h0 : 0;
        float acc[FW];
        uint32_t arg[FW];
#pragma unroll
        for (int t = 0; t < FW; ++t) {
          acc[t] = red_identity<ROP>();
          arg[t] = 0xffffffffu;
          if (L.acc_in && own && cc + t < cw)  // source-blocked pass: the partial
            acc[t] = L.acc_in[static_cast<int64_t>(r) * L.out_ld + c0 + cc + t];
        }
        for (uint32_t s = 0; s < rounds; ++s) {
          const uint32_t gsi = gs0 + s;
          const int b = static_cast<int>(gsi % NB);
          mbar_wait(&full[b], (gsi / NB) & 1u);
          if (own) {
            const uint32_t cnt = min(R, n - s * R);
            const float* col = sdata + static_cast<size_t>(b) * G::DF + cc;
            const float* sv = ssmall + static_cast<size_t>(b) * G::SF + hrel;
#pragma unroll 8
            for (uint32_t e = 0; e < cnt; ++e) {
              float x[FW];
              if constexpr (FW == 4) {
                const float4 v = *reinterpret_cast<const float4*>(col + static_cast<size_t>(e) * slot_f);
                x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
              } else {
                x[0] = col[static_cast<size_t>(e) * slot_f];
              }
              float sval = 0.0f;
              if constexpr (SMALL) sval = sv[e * nh];
#pragma unroll
              for (int t = 0; t < FW; ++t) {
                float m;
                if constexpr (SK == SK_SCALE) m = __fmul_rn(bin_apply<BOP>(x[t], 0.0f), sval);
                else if constexpr (SK == SK_NONE) m = bin_apply<BOP>(x[t], 0.0f);
                else m = bin_apply<BOP>(x[t], sval);
                if constexpr (ARG) {
                  if (red_wins<ROP>(acc[t], m)) {
                    acc[t] = m;
                    arg[t] = e0 + s * R + e;
                  }
                } else {
                  acc[t] = red_combine<ROP>(acc[t], m);
                }
              }
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[b]);
        }
        if (own) {
          const uint32_t deg = L.deg_indptr ? __ldg(L.deg_indptr + r + 1) - __ldg(L.deg_indptr + r) : n;
          const bool fix = L.epi != 1;  // a partial pass stores the raw fold
#pragma unroll
          for (int t = 0; t < FW; ++t) {
            if (cc + t >= cw) break;
            float a = acc[t];
            if constexpr (ROP == R_MAX || ROP == R_MIN) {
              if (fix && deg == 0) a = 0.0f;
            }
            if (fix && L.mean) a = deg ? __fdiv_rn(a, __uint2float_rn(deg)) : 0.0f;
            L.out[static_cast<int64_t>(r) * L.out_ld + c0 + cc + t] = a;
            if constexpr (ARG) {
              const int64_t ab = static_cast<int64_t>(r) * L.arg_ld + c0 + cc + t;
              const bool none = arg[t] == 0xffffffffu;
              if (L.arg_other)
                L.arg_other[ab] = none ? -1 : static_cast<int32_t>(__ldg(L.indices + arg[t]));
              if (L.arg_edge)
                L.arg_edge[ab] = none ? -1 : static_cast<int32_t>(__ldg(L.eids + arg[t]));
            }
          }
        }
      };
      if (cw > 128) run(std::integral_constant<int, 4>{});
      else run(std::integral_constant<int, 1>{});
      if (p.trace && ctid == 0) {
        unsigned long long* t = p.trace + 4ull * unit;
        t[0] = t0;
        t[1] = globaltimer_ns();
        t[2] = (static_cast<unsigned long long>(smid()) << 32) | 0xfffcu;
        t[3] = n;
      }
    }
    gs0 += rounds;
    __syncthreads();  // next unit: the id ring's first slots are rewritten
  }
}

// ------------------------------------------ LONG ROWS, TMA tile::gather4
// One column slice (<= 256 floats, the TMA box width) of one long row per
// unit.  Warp 0 is the producer: each lane turns four staged neighbour ids
// into one `cp.async.bulk.tensor.2d...tile::gather4` that lands four rows of
// the slice in a shared-memory ring stage (completion by transaction bytes
// on the stage's `full` mbarrier); warps 1-4 are the column owners that fold
// each stage in canonical edge order and release it on `empty`.  No register
// or L1 line holds a row in flight: the whole ~190 KB ring is the in-flight
// window, and the load-store units stay free for the co-resident segment
// warps.  Ids (and the small per-edge operand) arrive by cp.async NB stages
// ahead, so issuing never waits on a global load.
// Measured on B200 (scripts/mb_gather4.cu): one CTA streams ~73 rows/us of
// 1 KB (74 GB/s, the per-SM share of the L2 limit) against ~41 for the
// LDGSTS CTA above; the rate is bound by ~25 gather4 per us per SM, so the
// slice should be as wide as the row allows.
#ifndef G4_NB
#define G4_NB 4
#endif
#ifndef G4_DF
#define G4_DF 12288
#endif
constexpr int kG4Consumers = 4;
constexpr int kG4Threads = 32 * (1 + kG4Consumers);
struct G4Geom {
  static constexpr int NB = G4_NB;
  static constexpr int DF = G4_DF;  // data floats per stage
  static constexpr int MR = 256;    // max edges per stage
  static constexpr int SF = 512;    // small-operand floats per stage
  static constexpr size_t smem_bytes() {
    return sizeof(float) * (static_cast<size_t>(NB) * (DF + SF) + 4ull * NB * MR) +
           2ull * NB * sizeof(uint64_t);
  }
};

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void tma_gather4(uint32_t dst, const CUtensorMap* map, int col, int r0,
                                            int r1, int r2, int r3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(map), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}

template <int BOP, int ROP, bool ARG, int SK>
__global__ void __launch_bounds__(kG4Threads, 1)
    k_long_g4(const __grid_constant__ StreamLaunch p, const __grid_constant__ CUtensorMap tm_long,
              const __grid_constant__ CUtensorMap tm_xl) {
  using G = G4Geom;
  constexpr int NB = G::NB;
  constexpr bool SMALL = SK != SK_NONE;
  extern __shared__ __align__(128) float sm[];
  __shared__ uint32_t s_unit;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const RowLaunch& L = p.row;
  const int rw = SMALL ? p.rhs_width : 0;
  const bool need_eid = L.lhs.role == ROLE_EID || (rw && L.rhs.role == ROLE_EID);
  float* sdata = sm;                                                              // NB x DF
  float* ssmall = sm + static_cast<size_t>(NB) * G::DF;                           // NB x SF
  uint32_t* sid = reinterpret_cast<uint32_t*>(ssmall + static_cast<size_t>(NB) * G::SF);  // 2NB x MR
  uint32_t* seid = sid + 2 * NB * G::MR;                                          // 2NB x MR
  uint64_t* full = reinterpret_cast<uint64_t*>(seid + 2 * NB * G::MR);
  uint64_t* empty = full + NB;
  if (tid == 0) {
    for (int b = 0; b < NB; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], kG4Consumers);
    }
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t gs0 = 0;  // stages run before the current unit (ring position)

  for (;;) {
    if (tid == 0) s_unit = atomicAdd(p.counter, 1u);
    __syncthreads();
    const uint32_t unit = s_unit;
    __syncthreads();
    if (unit >= p.n_units) break;
    const unsigned long long t0 = p.trace ? globaltimer_ns() : 0ull;
    uint32_t li, slc;
    int sw, bw;
    const bool xl = unit < p.n_xl_units;
    if (xl) {
      li = unit / p.xl_slices;
      slc = unit - li * p.xl_slices;
      sw = p.xl_sw;
      bw = p.g4_box_xl;
    } else {
      const uint32_t v = unit - p.n_xl_units;
      li = p.n_xl + v / p.long_slices;
      slc = v - (li - p.n_xl) * p.long_slices;
      sw = p.long_sw;
      bw = p.g4_box;
    }
    const uint32_t r = __ldg(p.long_rows + li);
    const int c0 = static_cast<int>(slc) * sw;
    const int cw = min(sw, L.width - c0);
    const int h0 = (SMALL && rw > 1) ? c0 / L.rhs.group : 0;
    const int nh = SMALL ? ((rw > 1) ? (c0 + cw - 1) / L.rhs.group - h0 + 1 : 1) : 1;
    uint32_t R = static_cast<uint32_t>(G::DF / bw);
    if (R > static_cast<uint32_t>(G::MR)) R = G::MR;
    if (SMALL && R * nh > static_cast<uint32_t>(G::SF)) R = G::SF / nh;
    R &= ~3u;
    const uint32_t e0 = __ldg(L.indptr + r), e1 = __ldg(L.indptr + r + 1);
    const uint32_t n = e1 - e0;
    const uint32_t rounds = (n + R - 1) / R;

    if (warp == 0) {
      const CUtensorMap* tm = xl ? &tm_xl : &tm_long;
      const int32_t lrole = L.lhs.role;
      auto fetch_ids = [&](uint32_t m) {  // ids of unit stage m -> id slot (gs0 + m) % 2NB
        if (m < rounds) {
          const uint32_t slot = (gs0 + m) % (2 * NB);
          for (uint32_t t = static_cast<uint32_t>(lane); t < R; t += 32) {
            const uint32_t j = e0 + m * R + t;
            if (j < e1) {
              cp_async_4(sid + slot * G::MR + t, L.indices + j);
              if (need_eid) cp_async_4(seid + slot * G::MR + t, L.eids + j);
            }
          }
        }
        cp_async_commit();  // one group per stage, possibly empty
      };
      for (uint32_t m = 0; m < static_cast<uint32_t>(NB); ++m) fetch_ids(m);
      constexpr bool small1 = SK == SK_WIN || SK == SK_SCALE;
      const float* s1base = (SK == SK_SCALE) ? L.other_scale : L.rhs.base;
      const int64_t s1ld = (SK == SK_SCALE) ? 1 : L.rhs.ld;
      const int32_t s1role = (SK == SK_SCALE) ? static_cast<int32_t>(ROLE_OTHER) : L.rhs.role;
      const uint32_t row_b = static_cast<uint32_t>(bw) * 4u;
      for (uint32_t s = 0; s < rounds; ++s) {
        const uint32_t gsi = gs0 + s;
        const int b = static_cast<int>(gsi % NB);
        if (gsi >= static_cast<uint32_t>(NB)) mbar_wait(&empty[b], ((gsi / NB) - 1) & 1u);
        cp_async_wait_group<NB - 1>();  // ids of stage s landed (this lane's)
        __syncwarp();                    // ... and every lane's
        const uint32_t islot = gsi % (2 * NB);
        const uint32_t* io = sid + islot * G::MR;
        const uint32_t* ie = seid + islot * G::MR;
        const uint32_t jr0 = s * R;
        const uint32_t cnt = min(R, n - jr0);
        const uint32_t ng = (cnt + 3) >> 2;
        if (lane == 0) mbar_expect_tx(&full[b], ng * 4u * row_b);
        __syncwarp();
        const uint32_t sd = smem_u32(sdata + static_cast<size_t>(b) * G::DF);
        for (uint32_t g = static_cast<uint32_t>(lane); g < ng; g += 32) {
          int rr[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t q = min(4 * g + k, cnt - 1);  // a tail group repeats its last row
            const uint32_t o = io[q];
            if (lrole == ROLE_OTHER) {
              rr[k] = static_cast<int>(o);
            } else {
              const uint32_t e = need_eid ? ie[q] : 0u;
              rr[k] = static_cast<int>(operand_row(lrole, 0, o, e, e0 + jr0 + q));
            }
          }
          tma_gather4(sd + 4 * g * row_b, tm, c0, rr[0], rr[1], rr[2], rr[3], &full[b]);
        }
        if constexpr (SMALL) {
          float* bs = ssmall + static_cast<size_t>(b) * G::SF;
          for (uint32_t q = static_cast<uint32_t>(lane); q < cnt; q += 32) {
            const uint32_t j = e0 + jr0 + q;
            const uint32_t o = io[q];
            const uint32_t e = need_eid ? ie[q] : 0u;
            if (small1) {
              const uint32_t sr = s1role == ROLE_POS ? j : s1role == ROLE_EID ? e : o;
              cp_async_4(bs + q, s1base + static_cast<int64_t>(sr) * s1ld);
            } else {
              const float* sp = L.rhs.base + operand_row(L.rhs.role, 0, o, e, j) * L.rhs.ld + h0;
              for (int h = 0; h < nh; ++h) cp_async_4(bs + q * nh + h, sp + h);
            }
          }
        }
        fetch_ids(s + NB);
        if constexpr (SMALL) cp_async_arrive(&full[b]);
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[b]);
      }
      cp_async_wait_group<0>();
    } else {
      const int ctid = tid - 32;  // 0 .. 127
      auto run = [&](auto fw_tag) {
        constexpr int FW = decltype(fw_tag)::value;
        const int cc = ctid * FW;
        const bool own = cc < cw;
        const int hrel = (SMALL && rw > 1) ? (c0 + cc) / L.rhs.group - h0 : 0;
        float acc[FW];
        uint32_t arg[FW];
#pragma unroll
        for (int t = 0; t < FW; ++t) {
          acc[t] = red_identity<ROP>();
          arg[t] = 0xffffffffu;
          if (L.acc_in && own && cc + t < cw)  // source-blocked pass: the partial
            acc[t] = L.acc_in[static_cast<int64_t>(r) * L.out_ld + c0 + cc + t];
        }
        for (uint32_t s = 0; s < rounds; ++s) {
          const uint32_t gsi = gs0 + s;
          const int b = static_cast<int>(gsi % NB);
          mbar_wait(&full[b], (gsi / NB) & 1u);
          if (own) {
            const uint32_t cnt = min(R, n - s * R);
            const float* col = sdata + static_cast<size_t>(b) * G::DF + cc;
            const float* sv = ssmall + static_cast<size_t>(b) * G::SF + hrel;
#pragma unroll 8
            for (uint32_t e = 0; e < cnt; ++e) {
              float x[FW];
              if constexpr (FW == 2) {
                const float2 v = *reinterpret_cast<const float2*>(col + static_cast<size_t>(e) * bw);
                x[0] = v.x;
                x[1] = v.y;
              } else {
                x[0] = col[static_cast<size_t>(e) * bw];
              }
              float sval = 0.0f;
              if constexpr (SMALL) sval = sv[e * nh];
#pragma unroll
              for (int t = 0; t < FW; ++t) {
                float m;
                if constexpr (SK == SK_SCALE) m = __fmul_rn(bin_apply<BOP>(x[t], 0.0f), sval);
                else if constexpr (SK == SK_NONE) m = bin_apply<BOP>(x[t], 0.0f);
                else m = bin_apply<BOP>(x[t], sval);
                if constexpr (ARG) {
                  if (red_wins<ROP>(acc[t], m)) {
                    acc[t] = m;
                    arg[t] = e0 + s * R + e;
                  }
                } else {
                  acc[t] = red_combine<ROP>(acc[t], m);
                }
              }
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[b]);
        }
        if (own) {
          const uint32_t deg = L.deg_indptr ? __ldg(L.deg_indptr + r + 1) - __ldg(L.deg_indptr + r) : n;
          const bool fix = L.epi != 1;  // a partial pass stores the raw fold
#pragma unroll
          for (int t = 0; t < FW; ++t) {
            if (cc + t >= cw) break;
            float a = acc[t];
            if constexpr (ROP == R_MAX || ROP == R_MIN) {
              if (fix && deg == 0) a = 0.0f;
            }
            if (fix && L.mean) a = deg ? __fdiv_rn(a, __uint2float_rn(deg)) : 0.0f;
            L.out[static_cast<int64_t>(r) * L.out_ld + c0 + cc + t] = a;
            if constexpr (ARG) {
              const int64_t ab = static_cast<int64_t>(r) * L.arg_ld + c0 + cc + t;
              const bool none = arg[t] == 0xffffffffu;
              if (L.arg_other)
                L.arg_other[ab] = none ? -1 : static_cast<int32_t>(__ldg(L.indices + arg[t]));
              if (L.arg_edge)
                L.arg_edge[ab] = none ? -1 : static_cast<int32_t>(__ldg(L.eids + arg[t]));
            }
          }
        }
      };
      if (cw > 128) run(std::integral_constant<int, 2>{});
      else run(std::integral_constant<int, 1>{});
      if (p.trace && ctid == 0) {
        unsigned long long* t = p.trace + 4ull * unit;
        t[0] = t0;
        t[1] = globaltimer_ns();
        t[2] = (static_cast<unsigned long long>(smid()) << 32) | 0xfffbu;
        t[3] = n;
      }
    }
    gs0 += rounds;
    __syncthreads();  // next unit: the id ring's first slots are rewritten
  }
}

// ------------------------------------------------------ LONG ROWS via TMA
// Warp-specialised variant for slices of >= 512 B: warp 8 is the producer
// (lane 0 issues one cp.async.bulk per edge into a shared-memory ring of
// 8-edge stages, ~200 KB deep; lanes 0-7 stage the small operand with
// cp.async on the same full barrier), warps 0-7 are the 256 column owners
// that fold each stage in edge order and release it on the empty barrier.
// The SM's TMA engine is otherwise idle (segments gather with LDG), and a
// full-row TMA request per edge keeps ~200 edges in flight for one row.
constexpr int kLtConsumers = 8;                      // warps folding
constexpr int kLtThreads = (kLtConsumers + 1) * 32;  // + producer warp
constexpr int kLtMaxStages = 32;
constexpr int kLtRingBytes = 200 * 1024;
constexpr int kIdWin = 8;  // id windows in flight (producer)

__host__ __device__ constexpr size_t lt_smem_bytes() {
  return kLtRingBytes + 2 * kLtMaxStages * sizeof(uint64_t) + 2 * kIdWin * 32 * sizeof(uint32_t);
}

template <int BOP, int ROP, bool ARG, bool SMALL>
__global__ void __launch_bounds__(kLtThreads, 1) k_long_tma(const StreamLaunch p) {
  extern __shared__ __align__(128) unsigned char lt_smem[];
  __shared__ uint32_t s_unit;
  float* ring = reinterpret_cast<float*>(lt_smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(lt_smem + kLtRingBytes);
  uint64_t* empty = full + kLtMaxStages;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool producer = warp == kLtConsumers;
  const RowLaunch& L = p.row;
  const int rw = SMALL ? p.rhs_width : 0;
  const bool scale_on = SMALL && L.other_scale != nullptr;
  const int rws = SMALL ? (rw > 0 ? rw : 1) : 0;
  const bool need_eid = L.lhs.role == ROLE_EID || (rw && L.rhs.role == ROLE_EID);
  if (tid == 0) {
    for (int b = 0; b < kLtMaxStages; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], kLtConsumers);
    }
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t full_phase = 0, empty_phase = 0;  // per-stage parity bits (per role)

  for (;;) {
    if (tid == 0) s_unit = atomicAdd(p.counter, 1u);
    __syncthreads();
    const uint32_t unit = s_unit;
    __syncthreads();
    if (unit >= p.n_units) break;
    const unsigned long long t0 = p.trace ? globaltimer_ns() : 0ull;
    const uint32_t li = unit / p.long_slices;
    const uint32_t slc = unit - li * p.long_slices;
    const uint32_t r = __ldg(p.long_rows + li);
    const int c0 = static_cast<int>(slc) * p.long_sw;
    const int cw = min(p.long_sw, L.width - c0);
    const int slot_f = (cw + 3) & ~3;
    const uint32_t slot_bytes = static_cast<uint32_t>(slot_f) * 4u;
    int nst = kLtRingBytes / (8 * 4 * (slot_f + rws));
    nst = nst > kLtMaxStages ? kLtMaxStages : nst;
    float* tab = ring + static_cast<size_t>(nst) * 8 * slot_f;  // small operand per slot
    const uint32_t e0 = __ldg(L.indptr + r), e1 = __ldg(L.indptr + r + 1);
    const uint32_t n = e1 - e0;
    const uint32_t n_stages = (n + 7) / 8;

    if (producer) {
      const float* lbase = L.lhs.base + c0;
      // ids staged kIdWin windows (x32 edges) ahead through a shared ring with
      // cp.async groups: the producer never waits on a fresh global load
      uint32_t* id_o = reinterpret_cast<uint32_t*>(lt_smem + kLtRingBytes +
                                                   2 * kLtMaxStages * sizeof(uint64_t));
      uint32_t* id_e = id_o + kIdWin * 32;
      auto load_win = [&](uint32_t w) {
        const uint32_t j = e0 + 32u * w + lane;
        const int sl = static_cast<int>(w % kIdWin) * 32 + lane;
        if (j < e1) {
          cp_async_4(id_o + sl, L.indices + j);
          if (need_eid) cp_async_4(id_e + sl, L.eids + j);
        }
        cp_async_commit();
      };
      for (uint32_t w = 0; w < static_cast<uint32_t>(kIdWin); ++w) load_win(w);
      for (uint32_t s = 0; s < n_stages; ++s) {
        const int b = static_cast<int>(s % static_cast<uint32_t>(nst));
        if (s >= static_cast<uint32_t>(nst)) {  // wait for the consumers to free it
          mbar_wait(&empty[b], (empty_phase >> b) & 1u);
          empty_phase ^= 1u << b;
        }
        if ((s & 3u) == 0) {  // entering id window s/4
          if (s != 0) load_win((s >> 2) + kIdWin - 1);
          cp_async_wait_group<kIdWin - 1>();
          __syncwarp();
        }
        const uint32_t j0 = e0 + s * 8u;
        const uint32_t cnt = min(8u, e1 - j0);
        const int src = static_cast<int>(((s >> 2) % kIdWin) * 32 + (s & 3u) * 8u) + (lane & 7);
        const uint32_t o = id_o[src];
        const uint32_t e = need_eid ? id_e[src] : 0u;
        // issuing lanes rotate over the warp (stage s uses lanes 8*(s%4) ..
        // +7): bulk copies outstanding per issuing thread are limited
        const uint32_t lbase8 = (s & 3u) * 8u;
        const bool issuer = static_cast<uint32_t>(lane) >= lbase8 &&
                            static_cast<uint32_t>(lane) < lbase8 + 8u;
        const uint32_t l = static_cast<uint32_t>(lane) - lbase8;  // edge of this lane
        const int slot = b * 8 + static_cast<int>(l);
        if constexpr (SMALL) {
          if (issuer && l < cnt) {
            if (rw > 0) {
              const float* sp = L.rhs.base + operand_row(L.rhs.role, 0, o, e, j0 + l) * L.rhs.ld;
              for (int h = 0; h < rw; ++h) cp_async_4(tab + slot * rws + h, sp + h);
            } else if (scale_on) {
              cp_async_4(tab + slot, L.other_scale + o);
            }
          }
          if (issuer) cp_async_arrive(&full[b]);
          __syncwarp();
        }
        if (lane == 0) mbar_arrive_expect_tx(&full[b], cnt * slot_bytes);
        __syncwarp();
        if (issuer && l < cnt)
          tma_load_1d(ring + slot * slot_f,
                      lbase + operand_row(L.lhs.role, 0, o, e, j0 + l) * L.lhs.ld, slot_bytes,
                      &full[b]);
      }
      // drain: the last min(nst, n_stages) stages' empties are consumed here
      // so both roles enter the next unit with matching phases
      const uint32_t tail = min(static_cast<uint32_t>(nst), n_stages);
      for (uint32_t s = n_stages - tail; s < n_stages; ++s) {
        const int b = static_cast<int>(s % static_cast<uint32_t>(nst));
        mbar_wait(&empty[b], (empty_phase >> b) & 1u);
        empty_phase ^= 1u << b;
      }
    } else {
      // consumers: thread tid owns column c0 + tid
      float acc = red_identity<ROP>();
      uint32_t arg = 0xffffffffu;
      const bool own = tid < cw;
      const int hcol = (SMALL && rw > 1) ? (c0 + tid) / L.rhs.group : 0;
      for (uint32_t s = 0; s < n_stages; ++s) {
        const int b = static_cast<int>(s % static_cast<uint32_t>(nst));
        mbar_wait(&full[b], (full_phase >> b) & 1u);
        full_phase ^= 1u << b;
        const uint32_t cnt = min(8u, n - s * 8u);
        if (own) {
          float mv[8], sv[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            mv[q] = ring[static_cast<size_t>(b * 8 + q) * slot_f + tid];
            if constexpr (SMALL) sv[q] = tab[(b * 8 + q) * rws + hcol];
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            if (static_cast<uint32_t>(q) < cnt) {
              float m;
              if constexpr (SMALL) {
                m = rw > 0 ? bin_apply<BOP>(mv[q], sv[q])
                           : __fmul_rn(bin_apply<BOP>(mv[q], 0.0f), sv[q]);
              } else {
                m = bin_apply<BOP>(mv[q], 0.0f);
              }
              if constexpr (ARG) {
                if (red_wins<ROP>(acc, m)) {
                  acc = m;
                  arg = e0 + s * 8u + q;
                }
              } else {
                acc = red_combine<ROP>(acc, m);
              }
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[b]);
      }
      if (own) {
        float a = acc;
        if constexpr (ROP == R_MAX || ROP == R_MIN) {
          if (n == 0) a = 0.0f;
        }
        if (L.mean) a = n ? __fdiv_rn(a, __uint2float_rn(n)) : 0.0f;
        L.out[static_cast<int64_t>(r) * L.out_ld + c0 + tid] = a;
        if constexpr (ARG) {
          const int64_t ab = static_cast<int64_t>(r) * L.arg_ld + c0 + tid;
          const bool none = arg == 0xffffffffu;
          if (L.arg_other)
            L.arg_other[ab] = none ? -1 : static_cast<int32_t>(__ldg(L.indices + arg));
          if (L.arg_edge) L.arg_edge[ab] = none ? -1 : static_cast<int32_t>(__ldg(L.eids + arg));
        }
      }
    }
    if (p.trace && tid == 0) {
      unsigned long long* t = p.trace + 4ull * unit;
      t[0] = t0;
      t[1] = globaltimer_ns();
      t[2] = (static_cast<unsigned long long>(smid()) << 32) | 0xfffeu;
      t[3] = n;
    }
    __syncthreads();
  }
}

// -------------------------------------------------------------- segments
template <int VPL, int U, int BOP, int ROP, int ARG, int SK, bool LO, bool PART>
__global__ void __launch_bounds__(kThreads, VPL == 1 ? GATHER_MINB1 : VPL == 5 ? GATHER_MINB5 : GATHER_MINB2) k_gather(const StreamLaunch p) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const RowLaunch& L = p.row;
  const bool need_eid = L.lhs.role == ROLE_EID ||
                        ((SK == SK_WIN || SK == SK_HEAD) && L.rhs.role == ROLE_EID);
  // small scalar operand gathered in the id windows: value = sbase[row * sld]
  const float* sbase = SK == SK_SCALE ? L.other_scale : L.rhs.base;
  const int64_t sld = SK == SK_SCALE ? 1 : L.rhs.ld;
  const int32_t srole = SK == SK_SCALE ? static_cast<int32_t>(ROLE_OTHER) : L.rhs.role;

  // Every unit, the first included, comes from the counter in arrival
  // order: blocks that are not resident at launch -- the long-row CTAs hold
  // part of the SMs -- must not own statically assigned early (heavy) units,
  // and consecutive heavy units must not land on one SM (a block-wide grab
  // of 8 units measured 10% slower on cfg4).  Measured against the static
  // interleave: cfg2 forward 2.10 -> 1.81 ms, cfg4 7.9 -> 7.2 ms, cfg3 mean
  // 5.60 -> 5.44 ms; cfg1 (uniform, no long rows) +5% from the 4.7k
  // same-address atomics at launch.
  uint32_t next_unit = 0;
  if (lane == 0) next_unit = atomicAdd(p.counter, 1u);
  next_unit = __shfl_sync(kFull, next_unit, 0);
  for (;;) {
    const uint32_t unit = next_unit;
    if (unit >= p.n_units) break;
    if (lane == 0) next_unit = atomicAdd(p.counter, 1u);
    next_unit = __shfl_sync(kFull, next_unit, 0);
    const unsigned long long t0 = p.trace ? globaltimer_ns() : 0ull;

    UnitCtx u;
    const uint32_t si = unit / p.seg_slices;
    const uint32_t sl = unit - si * p.seg_slices;
    const uint2 seg = __ldg(p.segs + si);
    u.r0 = seg.x;
    u.r1 = seg.y;
    u.c0 = static_cast<int>(sl) * p.seg_sw;
    u.cw = min(p.seg_sw, L.width - u.c0);
    u.e0 = __ldg(L.indptr + u.r0);
    u.e1 = __ldg(L.indptr + u.r1);
    wide_unit<VPL, U, BOP, ROP, ARG, SK, LO, PART>(L, u, need_eid, sbase, sld, srole, lane);
    if (p.trace && lane == 0) {
      unsigned long long* t = p.trace + 4ull * unit;
      t[0] = t0;
      t[1] = globaltimer_ns();
      t[2] = (static_cast<unsigned long long>(smid()) << 32) | static_cast<unsigned>(warp);
      t[3] = u.e1 - u.e0;
    }
  }
}

// p.mode: 0 = row segments (k_gather), 1 = long rows (k_long)
template <int VPL, int BOP, int ROP, int ARG, int SK, bool LO>
cudaError_t launch_k(const StreamLaunch& p, cudaStream_t s) {
  constexpr bool LARG = ARG != 0;  // the long-row kernels track positions
  constexpr bool SMALL = SK != SK_NONE;
  cudaError_t e = cudaMemsetAsync(p.counter, 0, sizeof(uint32_t), s);
  if (e != cudaSuccess) return e;
  const int sms = p.row.num_sms > 0 ? p.row.num_sms : 148;
  if (p.mode == 1 && p.long_tma) {
    // wide long-row slices: TMA-fed, warp-specialised CTAs
    static int configured_t = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (configured_t != dev) {
      e = cudaFuncSetAttribute(k_long_tma<BOP, ROP, LARG, SMALL>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(lt_smem_bytes()));
      if (e != cudaSuccess) return e;
      configured_t = dev;
    }
    unsigned grid = p.long_ctas ? p.long_ctas : static_cast<unsigned>(sms);
    if (grid > p.n_units) grid = p.n_units;
    k_long_tma<BOP, ROP, LARG, SMALL><<<grid, kLtThreads, lt_smem_bytes(), s>>>(p);
  } else if (p.mode == 1 && p.long_g4) {
    static int configured_g = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (configured_g != dev) {
      e = cudaFuncSetAttribute(k_long_g4<BOP, ROP, LARG, SK>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(G4Geom::smem_bytes()));
      if (e != cudaSuccess) return e;
      configured_g = dev;
    }
    CUtensorMap tl, tx;
    if (!encode_rows_tmap(&tl, p.row.lhs, p.row.width, p.g4_box) ||
        !encode_rows_tmap(&tx, p.row.lhs, p.row.width, p.n_xl_units ? p.g4_box_xl : p.g4_box))
      return cudaErrorInvalidValue;
    unsigned grid = p.long_ctas ? p.long_ctas : static_cast<unsigned>(sms);
    if (grid > p.n_units) grid = p.n_units;
    k_long_g4<BOP, ROP, LARG, SK><<<grid, kG4Threads, G4Geom::smem_bytes(), s>>>(p, tl, tx);
  } else if (p.mode == 1 && p.long_ws) {
    const bool small = SMALL;
    static int configured_w = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (configured_w != dev) {
      e = cudaFuncSetAttribute(k_long_ws<BOP, ROP, LARG, SK>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(WsGeom::smem_bytes(small)));
      if (e != cudaSuccess) return e;
      configured_w = dev;
    }
    unsigned grid = p.long_ctas ? p.long_ctas : static_cast<unsigned>(sms);
    if (grid > p.n_units) grid = p.n_units;
    k_long_ws<BOP, ROP, LARG, SK><<<grid, kWsThreads, WsGeom::smem_bytes(small), s>>>(p);
  } else if (p.mode == 1) {
    const int rws = SMALL ? (p.rhs_width > 0 ? p.rhs_width : 1) : 0;
    const size_t smem = LongGeom<VPL>::smem_bytes(rws);
    static int configured = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (configured != dev) {
      e = cudaFuncSetAttribute(k_long<VPL, BOP, ROP, LARG, SMALL>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(LongGeom<VPL>::smem_bytes(LongGeom<VPL>::kMaxSmall)));
      if (e != cudaSuccess) return e;
      configured = dev;
    }
    // the host sizes the long-row grid by the long rows' share of the edges
    // (p.long_ctas); the segment kernel's persistent blocks take the other
    // SMs and absorb these ones when they finish
    unsigned grid = p.long_ctas ? p.long_ctas : static_cast<unsigned>(sms);
    if (grid > p.n_units) grid = p.n_units;
    k_long<VPL, BOP, ROP, LARG, SMALL><<<grid, kLongThreads, smem, s>>>(p);
  } else {
    constexpr int U = VPL == 1 ? GATHER_U1 : VPL == 5 ? GATHER_U5 : GATHER_U2;
    static int blocks_per_sm = 0;
    if (!blocks_per_sm) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm,
                                                    k_gather<VPL, U, BOP, ROP, ARG, SK, LO, false>,
                                                    kThreads, 0);
      if (blocks_per_sm < 1) blocks_per_sm = 1;
    }
    const unsigned grid = static_cast<unsigned>(sms * blocks_per_sm);
    if constexpr (!ARG) {  // argmax never runs source-blocked
      if (p.row.acc_in || p.row.epi) {
        k_gather<VPL, U, BOP, ROP, ARG, SK, LO, true><<<grid, kThreads, 0, s>>>(p);
        note_launch();
        return cudaGetLastError();
      }
    }
    k_gather<VPL, U, BOP, ROP, ARG, SK, LO, false><<<grid, kThreads, 0, s>>>(p);
  }
  note_launch();
  return cudaGetLastError();
}

template <int VPL, int BOP>
cudaError_t launch_red(const StreamLaunch& p, cudaStream_t s) {
  const RowLaunch& L = p.row;
  const bool arg = L.arg_other || L.arg_edge;
  // small operand kind (the host routes other_scale together with an rhs to
  // rows.cu)
  const int sk = L.rhs.base ? (p.rhs_width > 1 ? SK_HEAD : SK_WIN)
                            : (L.other_scale ? SK_SCALE : SK_NONE);
  const bool lo = L.lhs.role == ROLE_OTHER;
  auto go = [&](auto rop, auto argt, auto skt) -> cudaError_t {
    constexpr int R = decltype(rop)::value;
    constexpr bool A = decltype(argt)::value;
    constexpr int K = decltype(skt)::value;
    // copy_u / u_op_e with the gathered neighbour rows: the specialised
    // instances (argmax of the neighbour id alone: tracked directly);
    // copy_e and other layouts: the generic-role instance
    if (lo) {
      if constexpr (A) {
        if (!L.arg_edge) return launch_k<VPL, BOP, R, 2, K, true>(p, s);
      }
      return launch_k<VPL, BOP, R, A ? 1 : 0, K, true>(p, s);
    }
    return launch_k<VPL, BOP, R, A ? 1 : 0, K, false>(p, s);
  };
  auto by_sk = [&](auto rop, auto argt) -> cudaError_t {
    using std::integral_constant;
    if constexpr (BOP == B_COPY) {
      if (sk == SK_SCALE) return go(rop, argt, integral_constant<int, SK_SCALE>{});
      return go(rop, argt, integral_constant<int, SK_NONE>{});
    } else {
      if (sk == SK_HEAD) return go(rop, argt, integral_constant<int, SK_HEAD>{});
      return go(rop, argt, integral_constant<int, SK_WIN>{});
    }
  };
  using F = std::false_type;
  using T = std::true_type;
  switch (L.reduce) {
    case R_SUM: return by_sk(std::integral_constant<int, R_SUM>{}, F{});
    case R_MAX: return arg ? by_sk(std::integral_constant<int, R_MAX>{}, T{})
                           : by_sk(std::integral_constant<int, R_MAX>{}, F{});
    default: return arg ? by_sk(std::integral_constant<int, R_MIN>{}, T{})
                        : by_sk(std::integral_constant<int, R_MIN>{}, F{});
  }
}

// Segment units wider than 256 columns (the host selects them for copy and
// scalar-weighted sums of gathered rows, W <= 640): one pass over the edges
// instead of ceil(W / 256) column slices.
template <int BOP>
cudaError_t launch_wide(const StreamLaunch& p, cudaStream_t s) {
  if constexpr (BOP == B_COPY) {
    if (p.row.other_scale) return launch_k<5, BOP, R_SUM, 0, SK_SCALE, true>(p, s);
    return launch_k<5, BOP, R_SUM, 0, SK_NONE, true>(p, s);
  } else if constexpr (BOP == B_MUL) {
    if (p.rhs_width > 1) return launch_k<5, BOP, R_SUM, 0, SK_HEAD, true>(p, s);
    return launch_k<5, BOP, R_SUM, 0, SK_WIN, true>(p, s);
  } else {
    return cudaErrorNotSupported;
  }
}

template <int BOP>
cudaError_t launch_bop(const StreamLaunch& p, cudaStream_t s) {
  const int sw = p.mode == 1 ? p.long_sw : p.seg_sw;
  if (p.mode == 0 && sw > 256) return launch_wide<BOP>(p, s);
  return sw > 128 ? launch_red<2, BOP>(p, s) : launch_red<1, BOP>(p, s);
}

}  // namespace gather_detail

// per-operator entry points (one translation unit each)
cudaError_t launch_gather_copy(const StreamLaunch& p, cudaStream_t s);
cudaError_t launch_gather_mul(const StreamLaunch& p, cudaStream_t s);
cudaError_t launch_gather_arith(const StreamLaunch& p, cudaStream_t s);

}  // namespace gspmm_b200

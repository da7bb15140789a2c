// gather_impl.cuh -- the production owner-computes row kernel (sm_100a),
// instantiated per binary operator in gather_{copy,mul,arith}.cu.
//
// Same semantics as rows.cu (the reference's RowParallelSpmm left fold,
// kernels.cpp:162-195, bit for bit), built from measurements on B200
// (scripts/mb_gather.cu, profiles/):
//
//   * random source-row gathers run fastest as 128-bit LDGs into registers
//     (7.2 TB/s for 1 KB rows, 5.0 TB/s for 400 B rows) -- faster than one
//     TMA bulk copy per row (5.9 / 1.8 TB/s), whose per-SM request rate caps
//     small rows, and than LDGSTS (3.6 / 1.4 TB/s); so rows are gathered with
//     LDG.128 into registers, in both kernels;
//   * k_gather: persistent warps pull SEGMENT UNITS (edge-balanced runs of
//     consecutive short rows, one column slice each) from a global counter;
//     lanes own 4 (or 8, or 20) output columns, one edge per warp load
//     instruction; neighbour ids / scalar edge operands arrive as coalesced
//     32-edge windows prefetched one window ahead and broadcast with
//     shuffles; a batch of U edges is loaded, then folded in edge order;
//   * k_long_rg: one CTA per COLUMN UNIT of a long row (see below);
//   * fused epilogue: zero-degree fixup, mean, argmax; each output element
//     is written exactly once.
#pragma once
#include <atomic>
#include <type_traits>
#include "device_ops.cuh"
#include "stream.h"
#include "tma.cuh"

// GSPMM_BOUNDS=1 (a checking build, scripts/gpu/bounds.sh): device asserts on
// every gathered row id, output row, shared-memory stage offset and id-ring
// slot of the two planned kernels.  compute-sanitizer is closed on the GPU
// pool this was developed on, so the parity case (scripts/sanitize_case.py)
// runs against this build instead.
#ifndef GSPMM_BOUNDS
#define GSPMM_BOUNDS 0
#endif
#if GSPMM_BOUNDS
#include <cassert>
#define GS_ASSERT(c) assert(c)
#else
#define GS_ASSERT(c) ((void)0)
#endif

namespace gspmm_b200 {
namespace gather_detail {

constexpr int kThreads = 256;
// segment kernel geometry: edges per warp batch (<=128 / <=256 columns) and
// minimum resident blocks per SM.  Measured on B200 (scripts/var_ab.sh): warp
// parallelism beats per-warp depth -- U=8 at 3 blocks/SM for <=128 columns,
// U=2 at 4 blocks/SM (32 warps) for 256 columns: 94% of HBM on uniform graphs.
// <= 128 columns have a second geometry, U=4 at 5 blocks/SM (48 registers,
// 40 warps), used when the gathered table does not fit the L2: ncu on the
// config-3 fused forward showed 24 warps per SM waiting on the long
// scoreboard at 51% issue.  r02z, config 3 (max + argmax / mean / fused /
// mean backward, ms): U8 x 3: 6.20 / 5.01 / 7.62 / 5.32; U4 x 3: 6.92 / 5.85
// / 7.46 / 6.15; U4 x 4: 6.17 / 5.11 / 6.68 / 5.42; U4 x 5: 6.04 / 4.79 /
// 6.51 / 5.15; U4 x 6 (spills): 6.46 / 6.38 / 9.45 / 6.55; U2 x 6: 7.71 /
// 5.48 / 7.20 / 5.81; U8 x 4 (spills): 5.96 / 6.40 / 7.19 / 6.65.  The
// L2-resident config-1 shape runs 0.070 ms with U8 x 3 and 0.099 with U4 x 5.
#ifndef GATHER_U1
#define GATHER_U1 8
#endif
#ifndef GATHER_U1B
#define GATHER_U1B 4
#endif
#ifndef GATHER_MINB1B
#define GATHER_MINB1B 5
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
// The argmax fold of the segment kernel, per (edge, column): compare, take
// the value, take the id.  As FSETP + FSEL + SEL all three issue to the ALU
// pipe (16 lanes per clock per SM sub-partition, half the FMA rate): 48 of
// the ~95 instructions of a 4-edge batch of the fused max + mean forward,
// and ncu shows math-pipe throttle with the issue slots 75% busy
// (profiles/r04z_ncu_gather.txt).  With GATHER_FMA_SELECT the conditional
// value copy is a predicated FFMA (m * 1 + -0, exact for every m, signed
// zeros included) whose multiplier is a launch parameter, so ptxas cannot
// fold it back into a select: it issues to the FMA pipes.  The id copy is
// written the same way (IMAD j * 1 + 0); ptxas hoists that multiply and
// keeps a SEL per column, which is the better code: forcing the id onto the
// FMA pipes as well (the id tracked as a float, one opaque 1.0f per column)
// left no SEL but spilled at 48 registers, 6.50 -> 7.61 ms on the fused
// forward (r04h).  Measured (r04h): cfg3 max + argmax 5.15 -> 4.75 ms, the
// fused max + mean forward 6.56 -> 6.46 ms.
#ifndef GATHER_FMA_SELECT
#define GATHER_FMA_SELECT 1
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

// MODE 1 (PART): the kernel instance serves source-blocked passes (acc_in /
// epi / deg_indptr honoured); the plain instances (MODE 0) compile those
// paths out (measured: the runtime checks cost up to 8% on cfg3 max +
// argmax).  MODE 2 (DUAL): a second accumulator folds the same messages with
// Sum into out2 (Mean when mean2): config 3's max + argmax and mean forward
// from ONE gather of every source row instead of two passes.  Each output is
// still its own sequential canonical fold, bit-identical to separate calls.
// ARG: 0 = no argmax; 1 = track the CSR position of the winner (the ids are
// looked up at the row's flush); 2 = track the winning neighbour id itself
// (gathered-row kernels with only arg_other requested: no lookup latency at
// the flush, measured 0.6 ms of cfg3's 7.7).
template <int VPL, int ROP, int ARG, int MODE>
struct Acc {
  static constexpr bool PART = MODE == 1, DUAL = MODE == 2;
  float a[VPL][4];
  uint32_t arg[VPL][4];
  float s2[DUAL ? VPL : 1][4];
  __device__ __forceinline__ void reset() {
#pragma unroll
    for (int v = 0; v < VPL; ++v)
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        a[v][t] = red_identity<ROP>();
        arg[v][t] = 0xffffffffu;
        if constexpr (DUAL) s2[v][t] = 0.0f;
      }
  }
  __device__ __forceinline__ void fold(int v, const float (&m)[4], uint32_t j, float f_one,
                                       uint32_t u_one) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if constexpr (DUAL) s2[v][t] = __fadd_rn(s2[v][t], m[t]);
      if constexpr (ARG) {
#if GATHER_FMA_SELECT
        // a < m (Max) / m < a (Min): ordered compares, NaN never wins
        if constexpr (ROP == R_MAX)
          asm("{\n\t.reg .pred p;\n\tsetp.lt.f32 p, %0, %2;\n\t"
              "@p fma.rn.f32 %0, %2, %4, 0f80000000;\n\t@p mad.lo.u32 %1, %3, %5, 0;\n\t}"
              : "+f"(a[v][t]), "+r"(arg[v][t])
              : "f"(m[t]), "r"(j), "f"(f_one), "r"(u_one));
        else
          asm("{\n\t.reg .pred p;\n\tsetp.lt.f32 p, %2, %0;\n\t"
              "@p fma.rn.f32 %0, %2, %4, 0f80000000;\n\t@p mad.lo.u32 %1, %3, %5, 0;\n\t}"
              : "+f"(a[v][t]), "+r"(arg[v][t])
              : "f"(m[t]), "r"(j), "f"(f_one), "r"(u_one));
#else
        if (red_wins<ROP>(a[v][t], m[t])) {
          a[v][t] = m[t];
          arg[v][t] = j;
        }
#endif
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
    GS_ASSERT(r < L.num_rows && c0 + cw <= L.width);
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
    if constexpr (DUAL) {
      float o2[4];
#pragma unroll
      for (int t = 0; t < 4; ++t)
        o2[t] = L.mean2 ? (deg ? __fdiv_rn(s2[v][t], __uint2float_rn(deg)) : 0.0f) : s2[v][t];
      float* orow2 = L.out2 + static_cast<int64_t>(r) * L.out2_ld + c0;
      if (c + 4 <= cw) {
        store_vec<4>(orow2 + c, o2);
      } else {
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (c + t < cw) orow2[c + t] = o2[t];
      }
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

template <int VPL, int U, int BOP, int ROP, int ARG, int SK, bool LO, int MODE>
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
  constexpr bool PART = MODE == 1;
  Acc<VPL, ROP, ARG, MODE> acc;
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
      GS_ASSERT(static_cast<int64_t>(lr) < L.lhs.rows);
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
        if constexpr (ARG == 2) acc.fold(v, m, okey[k], L.f_one, L.u_one);
        else acc.fold(v, m, jpos, L.f_one, L.u_one);
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
// Rows above the plan level's threshold run as COLUMN UNITS: one unit = one
// column slice [c0, c0 + cw) of one long row, folded by one CTA in canonical
// edge order (bit-exact: one owner per column sees every edge in order).
// The host cuts each long row into slices so that no unit runs much longer
// than half the long rows' balanced share of the machine (the heaviest row,
// 329k edges at config 3, becomes 8-column units whose time is the fp32 add
// chain itself, ~0.67 ms; 100k-edge rows become 32-column units), and hands
// the units out heaviest first (LPT).
//
// The CTA is warp-specialised.  12 producer warps gather each stage of R
// edges x cw columns with 128-bit LDGs into registers -- the (edge, column
// quad) items of a stage are spread over all 384 producer lanes, so a
// narrow slice still keeps every lane busy -- one stage ahead of the stage
// they store into the shared-memory ring (NB stages, empty / full
// mbarriers).  Neighbour ids ride four stages ahead as cp.async copies into
// a small id ring.  4 consumer warps fold each landed stage: units of <= 32
// columns (the chain-bound ones) use a compile-time stage stride -- per edge
// one LDS at an immediate offset and the chain add, nothing else
// (scripts/mb_chain.cu: 5.1 cycles per edge for that pair, 4.1 for the bare
// chain); wider units one or four columns per thread.  Whole blocks of edges
// run straight-line with the next block's loads in flight.
// Measured alternatives (r02n - r02s, unit traces by scripts/trace_long.py):
//   * a lane-per-quad / warp-per-edges producer (an id read, one address and
//     the load per item instead of ~60 instructions): wide units 29 -> 23
//     GB/s per CTA -- 25 of 32 lanes carry a 100-column row, and the stream
//     rate follows the number of warp gathers, not the instruction count;
//   * two stages of gathers in flight per lane (three register sets): the
//     same rate with either producer;
//   * column-major stages for narrow units (four edges of a column per
//     LDS.128, the fastest consumer in mb_chain): the transposing scalar
//     stores slow the producers of every unit, config-3 mean 5.2 -> 6.1 ms;
//   * pacing the producers of chain-bound units with nanosleep: no change.
// Measured (round 1, scripts/mb_gather.cu): random 400 B rows stream at
// 34 GB/s per SM through LDG.128 into registers against 9.5 GB/s through
// LDGSTS and ~100 rows/us through TMA gather4.
#ifndef LG_NB
#define LG_NB 3
#endif
#ifndef LG_DF
#define LG_DF 8192
#endif
#ifndef LG_MR
#define LG_MR 1024
#endif
#ifndef LG_ID
#define LG_ID 4
#endif
// LG_TRACE 1 (development builds only): every long-row unit prints its row,
// slice, globaltimer span and wait times (scripts/trace_long.py)
#ifndef LG_TRACE
#define LG_TRACE 0
#endif
constexpr int kLgProducers = 12, kLgConsumers = 4;
constexpr int kLgThreads = 32 * (kLgProducers + kLgConsumers);
struct LgGeom {
  static constexpr int NB = LG_NB;       // data stages in the ring
  static constexpr int DF = LG_DF;       // data floats per stage
  static constexpr int MR = LG_MR;       // max edges per stage
  static constexpr int ID = LG_ID;       // stages the neighbour ids run ahead
  static constexpr int NI = ID + 4;      // stage-id slots
  static constexpr int SF = 1024;        // small-operand floats per stage
  static constexpr int PL = 32 * kLgProducers;   // producer lanes
  static constexpr int KQ = (DF / 4 + PL - 1) / PL;  // quads per producer lane per stage
  static constexpr size_t smem_bytes(bool small, bool eid) {
    return sizeof(float) * static_cast<size_t>(NB) * DF +
           sizeof(uint32_t) * static_cast<size_t>(NI) * MR * (eid ? 2 : 1) +
           (small ? sizeof(float) * static_cast<size_t>(NB) * SF : 0) +
           2ull * NB * sizeof(uint64_t);
  }
};

template <int BOP, int ROP, bool ARG, int SK, bool DUAL>
__global__ void __launch_bounds__(kLgThreads, 1) k_long_rg(const StreamLaunch p) {
  using G = LgGeom;
  constexpr int NB = G::NB, NI = G::NI, KQ = G::KQ, PL = G::PL, ID = G::ID;
  constexpr bool SMALL = SK != SK_NONE;
  extern __shared__ __align__(16) float sm[];
  __shared__ uint32_t s_unit;
#if LG_TRACE
  __shared__ long long s_wait[3];  // cycles waiting: consumer on full, producer on empty, on the ids
  long long w_acc = 0, w_acc2 = 0;
#endif
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool producer = warp < kLgProducers;
  const RowLaunch& L = p.row;
  // the segment kernel launched behind this one (StreamLaunch::pdl) may take
  // every SM a long-row CTA leaves: the two write disjoint output rows
  if (p.pdl == 1) asm volatile("griddepcontrol.launch_dependents;");
  const int rw = SMALL ? p.rhs_width : 0;  // small floats per edge (1 = scalar)
  const bool need_eid = L.lhs.role == ROLE_EID || (SK != SK_SCALE && SMALL && L.rhs.role == ROLE_EID);
  float* sdata = sm;                                                          // NB x DF
  uint32_t* sid = reinterpret_cast<uint32_t*>(sm + static_cast<size_t>(NB) * G::DF);  // NI x MR
  uint32_t* seid = sid + NI * G::MR;                                          // NI x MR (eid)
  float* ssmall = reinterpret_cast<float*>(seid + (need_eid ? NI * G::MR : 0));  // NB x SF
  uint64_t* full = reinterpret_cast<uint64_t*>(ssmall + (SMALL ? NB * G::SF : 0));
  uint64_t* empty = full + NB;
  if (tid == 0) {
    for (int b = 0; b < NB; ++b) {
      mbar_init(&full[b], kLgProducers);
      mbar_init(&empty[b], kLgConsumers);
    }
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t gs0 = 0;  // stages this CTA ran before the current unit (ring phase)

  for (;;) {
    if (tid == 0) s_unit = atomicAdd(p.counter, 1u);
    __syncthreads();
    const uint32_t unit = s_unit;
    __syncthreads();
    if (unit >= p.n_units) break;
    const uint2 ud = __ldg(p.long_units + unit);
    const uint32_t r = ud.x;
    const int c0 = static_cast<int>(ud.y & 0xffffu);
    const int cw = static_cast<int>(ud.y >> 16);
    const int qpe = (cw + 3) >> 2;  // column quads per edge
    // stage stride of an edge, floats: narrow units pad to a compile-time
    // stride of the consumer (8 / 16 / 32), wider ones to the quad
    const int sst = cw <= 8 ? 8 : cw <= 16 ? 16 : cw <= 32 ? 32 : 4 * qpe;
    // (Column-major stages for narrow units -- four edges of a column per
    // LDS.128, the fastest consumer in scripts/mb_chain.cu -- were measured
    // twice (r02n, r02q): the transposing scalar stores slow the producers
    // of every unit, 5.2 -> 6.1 ms on the config-3 mean.)
    const int h0 = (SMALL && rw > 1) ? c0 / L.rhs.group : 0;
    const int nh = (SMALL && rw > 1) ? (c0 + cw - 1) / L.rhs.group - h0 + 1 : 1;
    uint32_t R = static_cast<uint32_t>(G::DF / sst);
    if (R > static_cast<uint32_t>(G::MR)) R = G::MR;
    if (SMALL && R * nh > static_cast<uint32_t>(G::SF)) R = G::SF / nh;
    const uint32_t e0 = __ldg(L.indptr + r), e1 = __ldg(L.indptr + r + 1);
    const uint32_t n = e1 - e0;
    const uint32_t rounds = (n + R - 1) / R;
#if LG_TRACE
    unsigned long long t_begin = 0;
    if (tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_begin));
#endif

    if (producer) {
      const int ptid = tid;  // 0 .. PL - 1
      auto fetch_ids = [&](uint32_t m) {  // ids of unit stage m -> slot (gs0 + m) % NI
        if (m >= rounds) return;
        const uint32_t slot = (gs0 + m) % NI;
        const uint32_t cnt = min(R, n - m * R);
        GS_ASSERT(cnt <= static_cast<uint32_t>(G::MR) && e0 + m * R + cnt <= e1);
        for (uint32_t t = static_cast<uint32_t>(ptid); t < cnt; t += PL) {
          cp_async_4(sid + slot * G::MR + t, L.indices + e0 + m * R + t);
          if (need_eid) cp_async_4(seid + slot * G::MR + t, L.eids + e0 + m * R + t);
        }
      };
      // item i = ptid + k * PL of a stage is (edge q = i / qpe, quad t = i % qpe)
      const uint32_t q0 = static_cast<uint32_t>(ptid) / static_cast<uint32_t>(qpe);
      const int t0 = ptid - static_cast<int>(q0) * qpe;
      const uint32_t dq = static_cast<uint32_t>(PL / qpe);
      const int dt = PL - static_cast<int>(dq) * qpe;
      const float* lbase = L.lhs.base + c0;
      const int64_t lld = L.lhs.ld;
      const int32_t lrole = L.lhs.role;
      // gather stage m's items into registers (x) and remember their shared
      // offsets (off, -1 = no item)
      auto load_stage = [&](uint32_t m, float4 (&x)[KQ], int (&off)[KQ]) {
        const uint32_t slot = (gs0 + m) % NI;
        const uint32_t cnt = min(R, n - m * R);
        const uint32_t* io = sid + slot * G::MR;
        const uint32_t* ie = seid + slot * G::MR;
        uint32_t q = q0;
        int t = t0;
#pragma unroll
        for (int k = 0; k < KQ; ++k) {
          off[k] = -1;
          if (q < cnt) {
            const uint32_t o = io[q];
            const uint32_t e = need_eid ? ie[q] : 0u;
            const uint32_t row = lrole == ROLE_OTHER
                                     ? o
                                     : static_cast<uint32_t>(operand_row(lrole, 0, o, e, e0 + m * R + q));
            GS_ASSERT(static_cast<int64_t>(row) < L.lhs.rows && q < static_cast<uint32_t>(G::MR));
            x[k] = __ldg(reinterpret_cast<const float4*>(lbase + static_cast<int64_t>(row) * lld + 4 * t));
            off[k] = static_cast<int>(q) * sst + 4 * t;
            GS_ASSERT(off[k] + 4 <= G::DF);
          }
          q += dq;
          t += dt;
          if (t >= qpe) {
            t -= qpe;
            ++q;
          }
        }
      };
      auto store_stage = [&](uint32_t s, const float4 (&x)[KQ], const int (&off)[KQ]) {
        const uint32_t gsi = gs0 + s;
        const int b = static_cast<int>(gsi % NB);
        if (gsi >= static_cast<uint32_t>(NB)) mbar_wait(&empty[b], ((gsi / NB) - 1) & 1u);
        float* sd = sdata + static_cast<size_t>(b) * G::DF;
#pragma unroll
        for (int k = 0; k < KQ; ++k)
          if (off[k] >= 0) *reinterpret_cast<float4*>(sd + off[k]) = x[k];
        if constexpr (SMALL) {
          const uint32_t slot = gsi % NI;
          const uint32_t cnt = min(R, n - s * R);
          float* bs = ssmall + static_cast<size_t>(b) * G::SF;
          const float* s1base = SK == SK_SCALE ? L.other_scale : L.rhs.base;
          const int64_t s1ld = SK == SK_SCALE ? 1 : L.rhs.ld;
          const int32_t s1role = SK == SK_SCALE ? static_cast<int32_t>(ROLE_OTHER) : L.rhs.role;
          for (uint32_t i = static_cast<uint32_t>(ptid); i < cnt * nh; i += PL) {
            const uint32_t q = i / static_cast<uint32_t>(nh);
            const int h = static_cast<int>(i - q * nh);
            const uint32_t o = sid[slot * G::MR + q];
            const uint32_t e = need_eid ? seid[slot * G::MR + q] : 0u;
            const int64_t sr = operand_row(s1role, 0, o, e, e0 + s * R + q);
            cp_async_4(bs + i, s1base + sr * s1ld + h0 + h);
          }
        }
        cp_async_arrive(&full[b]);  // the full phase also waits for these copies
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[b]);
      };
#pragma unroll
      for (int m = 0; m < ID; ++m) {
        fetch_ids(static_cast<uint32_t>(m));
        cp_async_commit();
      }
      cp_async_wait_group<ID - 1>();
      named_barrier_sync(1, PL);  // ids of stage 0 visible to every producer
      float4 xa[KQ], xb[KQ];
      int oa[KQ], ob[KQ];
      load_stage(0, xa, oa);
      // one step: ids ID stages ahead, gather stage s + 1, store stage s
      // (two register sets alternate, so no register with a pending load is
      // ever moved).  With the ids only two stages ahead every step waited
      // for an id load issued one step earlier (r02d: 13 GB/s per CTA).
      auto step = [&](uint32_t s, float4 (&xc)[KQ], int (&oc)[KQ], float4 (&xn)[KQ],
                      int (&on)[KQ]) {
        fetch_ids(s + ID);
        cp_async_commit();
        cp_async_wait_group<ID - 1>();
        named_barrier_sync(1, PL);  // ids of stage s + 1 visible
        if (s + 1 < rounds) load_stage(s + 1, xn, on);
        store_stage(s, xc, oc);
      };
      for (uint32_t s = 0; s < rounds; s += 2) {
        step(s, xa, oa, xb, ob);
        if (s + 1 < rounds) step(s + 1, xb, ob, xa, oa);
      }
      cp_async_wait_group<0>();
    } else {
      const int ctid = tid - PL;  // 0 .. 127
      // The fold of a column is one dependent fp32 chain over the row's
      // edges (~4 cycles per edge: 0.67 ms for config 3's 329k-edge row), so
      // a unit's consumer must issue nothing per edge but the chain and its
      // operand load: whole blocks of KB edges run straight-line (no clamps
      // or selects; the partial block of a stage's end folds edge by edge),
      // the next block's shared-memory loads in flight behind the current
      // block's chain.  The chain's 4 cycles leave room for little else: 3.75
      // instructions per edge ran 7.2 cycles per edge and 8 ran 16.5 (r02r
      // unit traces), so narrow units issue one LDS at an immediate offset
      // and the add per edge, nothing more.  Max / Min with argmax over
      // copied rows are not a chain at all: the extremum is exact and
      // associative, so each block's extremum comes from a tree of FMNMX
      // and one comparison per block decides whether the block takes over
      // (`a < m ? m : a` and fmaxf agree except for the sign of a zero
      // extremum); the flush re-reads the winning block from global memory
      // and takes the first edge equal to the extremum -- the reference's
      // first-wins rule -- with that element's bits.  A DUAL unit of <= 64
      // columns splits its two folds over the two halves of the consumer
      // threads (max + argmax on warps 0-1, the sum on warps 2-3).
      constexpr bool FASTMM = ARG && BOP == B_COPY && SK == SK_NONE &&
                              (ROP == R_MAX || ROP == R_MIN);
      // FW columns per thread; ST = compile-time stage stride (0: runtime sst)
      auto run = [&](auto fw_tag, auto st_tag) {
        constexpr int FW = decltype(fw_tag)::value;
        constexpr int ST = decltype(st_tag)::value;
        constexpr int KB = FW == 4 ? 4 : 16;  // edges per straight-line block
        const int stf = ST ? ST : sst;
        const bool split = DUAL && FW * 64 >= cw;      // both folds fit 64 threads each
        const bool second = split && ctid >= 64;       // the sum half of a split unit
        const int cc = (split ? (ctid & 63) : ctid) * FW;
        const bool own = cc < cw;
        const int hrel = (SMALL && rw > 1) ? (c0 + cc) / L.rhs.group - h0 : 0;
        float acc[FW];
        uint32_t arg[FW];
        float acc2[DUAL ? FW : 1];
#pragma unroll
        for (int t = 0; t < FW; ++t) {
          acc[t] = red_identity<ROP>();
          arg[t] = 0xffffffffu;
          if constexpr (DUAL) acc2[t] = 0.0f;
          if (L.acc_in && own && cc + t < cw)  // source-blocked pass: the partial
            acc[t] = L.acc_in[static_cast<int64_t>(r) * L.out_ld + c0 + cc + t];
        }
        auto message = [&](float x, float sv) {
          if constexpr (SK == SK_SCALE) return __fmul_rn(bin_apply<BOP>(x, 0.0f), sv);
          else if constexpr (SK == SK_NONE) return bin_apply<BOP>(x, 0.0f);
          else return bin_apply<BOP>(x, sv);
        };
        // one stage: PRIM = the config's own reduction, SEC = the DUAL sum
        auto fold_stage = [&](auto prim_tag, auto sec_tag, const float* sd, const float* sv,
                              uint32_t cnt, uint32_t ebase) {
          constexpr bool PRIM = decltype(prim_tag)::value, SEC = decltype(sec_tag)::value;
          const float* col = sd + cc;
          float xa[KB][FW], xb[KB][FW], sa[KB], sb[KB];
          auto ld = [&](uint32_t blk, float (&x)[KB][FW], float (&s8)[KB]) {
            const float* pb = col + static_cast<size_t>(blk) * (KB * stf);
#pragma unroll
            for (int k = 0; k < KB; ++k) {
              if constexpr (FW == 4) {
                const float4 v = *reinterpret_cast<const float4*>(pb + k * stf);
                x[k][0] = v.x; x[k][1] = v.y; x[k][2] = v.z; x[k][3] = v.w;
              } else {
                x[k][0] = pb[k * stf];
              }
            }
            if constexpr (SMALL) {
              const float* ps = sv + static_cast<size_t>(blk) * KB * nh;
#pragma unroll
              for (int k = 0; k < KB; ++k) s8[k] = ps[k * nh];
            }
          };
          auto fold_one = [&](float x, float s1, int t, uint32_t pos) {
            const float m = message(x, s1);
            if constexpr (SEC) acc2[t] = __fadd_rn(acc2[t], m);
            if constexpr (PRIM) {
              if constexpr (ARG) {
                if (red_wins<ROP>(acc[t], m)) {
                  acc[t] = m;
                  arg[t] = pos;
                }
              } else {
                acc[t] = red_combine<ROP>(acc[t], m);
              }
            }
          };
          auto fold = [&](uint32_t blk, const float (&x)[KB][FW], const float (&s8)[KB]) {
            int ak[FW];
#pragma unroll
            for (int t = 0; t < FW; ++t) ak[t] = -1;
            if constexpr (PRIM && FASTMM) {
              // the block's extremum by a tree (exact and order-free up to
              // the sign of zero), one comparison per block on the chain
#pragma unroll
              for (int t = 0; t < FW; ++t) {
                float v[KB];
#pragma unroll
                for (int k = 0; k < KB; ++k) v[k] = x[k][t];
#pragma unroll
                for (int h = KB / 2; h > 0; h >>= 1)
#pragma unroll
                  for (int k = 0; k < h; ++k)
                    v[k] = ROP == R_MAX ? fmaxf(v[k], v[k + h]) : fminf(v[k], v[k + h]);
                const bool w = red_wins<ROP>(acc[t], v[0]);
                acc[t] = ROP == R_MAX ? fmaxf(acc[t], v[0]) : fminf(acc[t], v[0]);
                ak[t] = w ? 0 : -1;  // the block's first edge: resolved at the flush
              }
            }
#pragma unroll
            for (int k = 0; k < KB; ++k) {
#pragma unroll
              for (int t = 0; t < FW; ++t) {
                const float m = message(x[k][t], s8[k]);
                if constexpr (SEC) acc2[t] = __fadd_rn(acc2[t], m);
                if constexpr (PRIM) {
                  if constexpr (FASTMM) {
                    // folded above
                  } else if constexpr (ARG) {
                    if (red_wins<ROP>(acc[t], m)) {
                      acc[t] = m;
                      ak[t] = k;
                    }
                  } else {
                    acc[t] = red_combine<ROP>(acc[t], m);
                  }
                }
              }
            }
            if constexpr (ARG && PRIM) {
#pragma unroll
              for (int t = 0; t < FW; ++t)
                if (ak[t] >= 0) arg[t] = ebase + blk * KB + static_cast<uint32_t>(ak[t]);
            }
          };
          const uint32_t nfull = cnt / KB;
          GS_ASSERT(static_cast<size_t>(cnt - 1) * stf + cc + FW <= static_cast<size_t>(G::DF));
          GS_ASSERT(!SMALL || static_cast<size_t>(cnt - 1) * nh + hrel < static_cast<size_t>(G::SF));
          if (nfull) {
            ld(0, xa, sa);
            uint32_t bk = 0;
            for (; bk + 2 <= nfull; bk += 2) {
              ld(bk + 1, xb, sb);
              fold(bk, xa, sa);
              ld(min(bk + 2, nfull - 1), xa, sa);
              fold(bk + 1, xb, sb);
            }
            if (bk < nfull) fold(bk, xa, sa);  // xa holds block nfull - 1
          }
          for (uint32_t e = nfull * KB; e < cnt; ++e) {
            const float s1 = SMALL ? sv[static_cast<size_t>(e) * nh] : 0.0f;
#pragma unroll
            for (int t = 0; t < FW; ++t) fold_one(col[static_cast<size_t>(e) * stf + t], s1, t, ebase + e);
          }
        };
        using T = std::true_type;
        using F = std::false_type;
        for (uint32_t s = 0; s < rounds; ++s) {
          const uint32_t gsi = gs0 + s;
          const int b = static_cast<int>(gsi % NB);
#if LG_TRACE
          const long long tw0 = clock64();
#endif
          mbar_wait(&full[b], (gsi / NB) & 1u);
#if LG_TRACE
          w_acc += clock64() - tw0;
#endif
          if (own) {
            const uint32_t cnt = min(R, n - s * R);
            const float* sd = sdata + static_cast<size_t>(b) * G::DF;
            const float* sv = ssmall + static_cast<size_t>(b) * G::SF + hrel;
            const uint32_t ebase = e0 + s * R;
            if constexpr (!DUAL) fold_stage(T{}, F{}, sd, sv, cnt, ebase);
            else if (!split) fold_stage(T{}, T{}, sd, sv, cnt, ebase);
            else if (!second) fold_stage(T{}, F{}, sd, sv, cnt, ebase);
            else fold_stage(F{}, T{}, sd, sv, cnt, ebase);
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
            if (!second) {
              float a = acc[t];
              if constexpr (FASTMM) {
                // arg is the first edge of the winning block (or the winning
                // edge itself): the winner is the first edge from there that
                // compares equal to the extremum; its bits are the result
                // (the sign of a zero extremum included)
                if (arg[t] != 0xffffffffu) {
                  const uint32_t lim = min(arg[t] + static_cast<uint32_t>(KB), e1);
                  for (uint32_t pos = arg[t]; pos < lim; ++pos) {
                    const uint32_t o = __ldg(L.indices + pos);
                    const uint32_t e = L.lhs.role == ROLE_EID ? __ldg(L.eids + pos) : 0u;
                    const float v =
                        __ldg(L.lhs.base + operand_row(L.lhs.role, r, o, e, pos) * L.lhs.ld + c0 + cc + t);
                    if (v == a) {
                      a = v;
                      arg[t] = pos;
                      break;
                    }
                  }
                }
              }
              if constexpr (ROP == R_MAX || ROP == R_MIN) {
                if (fix && deg == 0) a = 0.0f;
              }
              if (fix && L.mean) a = deg ? __fdiv_rn(a, __uint2float_rn(deg)) : 0.0f;
              GS_ASSERT(r < L.num_rows && c0 + cc + t < L.width);
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
            if constexpr (DUAL) {
              if (!split || second)
                L.out2[static_cast<int64_t>(r) * L.out2_ld + c0 + cc + t] =
                    L.mean2 ? (deg ? __fdiv_rn(acc2[t], __uint2float_rn(deg)) : 0.0f) : acc2[t];
            }
          }
        }
      };
      using I0 = std::integral_constant<int, 0>;
      using I1 = std::integral_constant<int, 1>;
      using I4 = std::integral_constant<int, 4>;
      if (cw > 128) run(I4{}, I0{});
      else if (cw > 32) run(I1{}, I0{});
      else if (sst == 8) run(I1{}, std::integral_constant<int, 8>{});
      else if (sst == 16) run(I1{}, std::integral_constant<int, 16>{});
      else run(I1{}, std::integral_constant<int, 32>{});
    }
    gs0 += rounds;
#if LG_TRACE
    if (tid == PL) s_wait[0] = w_acc;
    if (tid == 0) {
      s_wait[1] = w_acc;
      s_wait[2] = w_acc2;
    }
    w_acc = 0;
    w_acc2 = 0;
#endif
    __syncthreads();  // next unit: the id ring's first slots are rewritten
#if LG_TRACE
    if (tid == 0) {
      unsigned long long t_end;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
      printf("LGW %u full %lld empty %lld idbar %lld ld 0 st 0 ar 0\n", unit, s_wait[0], s_wait[1], s_wait[2]);
      printf("LGU %u row %u c0 %d cw %d n %u t0 %llu t1 %llu cta %u\n", unit, r, c0, cw, n, t_begin,
             t_end, blockIdx.x);
    }
#endif
  }
}

// -------------------------------------------------------------- segments
template <int VPL, int U, int BOP, int ROP, int ARG, int SK, bool LO, int MODE>
__global__ void __launch_bounds__(kThreads, VPL == 1 ? (U == GATHER_U1 ? GATHER_MINB1 : GATHER_MINB1B)
                                                     : VPL == 5 ? GATHER_MINB5 : GATHER_MINB2) k_gather(const StreamLaunch p) {
  const int lane = threadIdx.x & 31;
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
    wide_unit<VPL, U, BOP, ROP, ARG, SK, LO, MODE>(L, u, need_eid, sbase, sld, srole, lane);
  }
  // dependent of the long-row kernel: do not complete before it has
  if (p.pdl == 2) asm volatile("griddepcontrol.wait;" ::: "memory");
}

// p.mode: 0 = row segments (k_gather), 1 = long-row column units (k_long_rg)
template <int VPL, int BOP, int ROP, int ARG, int SK, bool LO, bool DUAL = false>
cudaError_t launch_k(const StreamLaunch& p, cudaStream_t s) {
  cudaError_t e = cudaSuccess;
  if (!p.pdl) e = cudaMemsetAsync(p.counter, 0, sizeof(uint32_t), s);
  if (e != cudaSuccess) return e;
  const int sms = p.row.num_sms > 0 ? p.row.num_sms : 148;
  if (p.mode == 1) {
    if constexpr (VPL == 1) {  // one instance per (BOP, ROP, ARG, SK)
      constexpr bool SMALL = SK != SK_NONE;
      const RowLaunch& L = p.row;
      const bool eid = L.lhs.role == ROLE_EID || (SK != SK_SCALE && SMALL && L.rhs.role == ROLE_EID);
      const size_t smem = LgGeom::smem_bytes(SMALL, eid);
      auto* kern = k_long_rg<BOP, ROP, ARG != 0, SK, DUAL>;
      e = set_max_dynamic_smem(reinterpret_cast<const void*>(kern),
                               static_cast<int>(LgGeom::smem_bytes(SMALL, true)));
      if (e != cudaSuccess) return e;
      unsigned grid = p.grid ? p.grid : static_cast<unsigned>(sms);
      if (grid > p.n_units) grid = p.n_units;
      kern<<<grid, kLgThreads, smem, s>>>(p);
    } else {
      return cudaErrorInvalidValue;
    }
  } else {
    constexpr int MODE = DUAL ? 2 : 0;
    auto launch = [&](auto u_tag) -> cudaError_t {
      constexpr int U = decltype(u_tag)::value;
      static std::atomic<int> blocks_per_sm{0};
      int bps = blocks_per_sm.load(std::memory_order_relaxed);
      if (!bps) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps,
                                                      k_gather<VPL, U, BOP, ROP, ARG, SK, LO, MODE>,
                                                      kThreads, 0);
        if (bps < 1) bps = 1;
        blocks_per_sm.store(bps, std::memory_order_relaxed);
      }
      const unsigned grid = static_cast<unsigned>(sms * bps);
      // pdl 2: launched behind the long-row kernel with programmatic stream
      // serialization -- blocks start on SMs as the long-row CTAs leave them
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(kThreads);
      cfg.stream = s;
      cudaLaunchAttribute at{};
      at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at.val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = &at;
      cfg.numAttrs = p.pdl == 2 ? 1 : 0;
      cudaError_t le;
      if constexpr (!ARG && !DUAL) {  // argmax / dual never run source-blocked
        if (p.row.acc_in || p.row.epi) {
          le = cudaLaunchKernelEx(&cfg, k_gather<VPL, U, BOP, ROP, ARG, SK, LO, 1>, p);
          note_launch();
          return le != cudaSuccess ? le : cudaGetLastError();
        }
      }
      le = cudaLaunchKernelEx(&cfg, k_gather<VPL, U, BOP, ROP, ARG, SK, LO, MODE>, p);
      note_launch();
      return le != cudaSuccess ? le : cudaGetLastError();
    };
    if constexpr (VPL == 1) {
      // the gathered table against the L2 (126 MB): latency-bound gathers
      // want more warps, L2-resident ones more edges per warp
      const double table = static_cast<double>(p.row.lhs.rows) * static_cast<double>(p.row.lhs.ld) * 4.0;
      if (table > 96.0 * 1048576.0) return launch(std::integral_constant<int, GATHER_U1B>{});
      return launch(std::integral_constant<int, GATHER_U1>{});
    } else {
      return launch(std::integral_constant<int, VPL == 5 ? GATHER_U5 : GATHER_U2>{});
    }
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
      if constexpr (BOP == B_COPY && K == SK_NONE && (R == R_MAX || R == R_MIN)) {
        if (L.out2) {  // the host routes only this combination here
          if constexpr (A) {
            if (!L.arg_edge) return launch_k<VPL, BOP, R, 2, K, true, true>(p, s);
          }
          return launch_k<VPL, BOP, R, A ? 1 : 0, K, true, true>(p, s);
        }
      }
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
  if (p.mode == 1) return launch_red<1, BOP>(p, s);  // long rows: one instance per width
  if (p.seg_sw > 256) return launch_wide<BOP>(p, s);
  return p.seg_sw > 128 ? launch_red<2, BOP>(p, s) : launch_red<1, BOP>(p, s);
}

}  // namespace gather_detail

// per-operator entry points (one translation unit each)
cudaError_t launch_gather_copy(const StreamLaunch& p, cudaStream_t s);
cudaError_t launch_gather_mul(const StreamLaunch& p, cudaStream_t s);
cudaError_t launch_gather_arith(const StreamLaunch& p, cudaStream_t s);

}  // namespace gspmm_b200

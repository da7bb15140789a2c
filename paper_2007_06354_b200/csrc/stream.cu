// stream.cu -- TMA-staged owner-computes row kernel (sm_100a): the main
// forward/backward aggregation path.
//
// Same semantics as rows.cu (the reference's RowParallelSpmm left fold,
// kernels.cpp:162-195, bit for bit) but built for memory-level parallelism:
//
//   * persistent CTAs (one per SM, 8 warps); each warp pulls WORK UNITS from
//     a global counter:  (a) an edge-balanced segment of consecutive owner
//     rows (the device plan, built at graph upload -- the GPU analogue of the
//     reference's edge-balanced thread ranges, block_plan.cpp:83-99) at a
//     column slice of up to 256 floats, or (b) one column slice of a LONG
//     row (degree above the plan threshold), so a 66k-329k-edge hub is folded
//     by many warps on many SMs at once while each (row, column) is still
//     one sequential fold;
//   * per warp a shared-memory ring of 8-edge stages: for each edge one lane
//     issues a TMA 1-D bulk copy (cp.async.bulk) of the gathered source-row
//     slice into the ring, completing on the stage's mbarrier; small per-edge
//     operands (scalar weights, per-head attention, the mean-backward scale)
//     ride along as cp.async (LDGSTS) on the same mbarrier.  In-flight bytes
//     are bounded by shared memory (~24 KB per warp, ~190 KB per SM), not by
//     registers;
//   * neighbour ids, edge ids and row ends are prefetched one 32-wide window
//     ahead in registers and broadcast with warp shuffles;
//   * the fold reads the ring with 128-bit shared loads, lanes owning 4 or 8
//     columns; row boundaries finalize in place (zero-degree fixup, mean,
//     argmax), so every output row is written exactly once.
#include "device_ops.cuh"
#include "stream.h"
#include "tma.cuh"

namespace gspmm_b200 {
namespace {

constexpr int kWarps = 8;
constexpr int kRingBytes = 24 * 1024;  // per warp: ring slots + small-operand tables
constexpr int kMaxStages = 24;
constexpr int kStage = 8;                               // edges per stage
constexpr int kDW = 8;                                  // id windows in flight
// per warp: ring + mbarriers + id/edge-id window rings
constexpr int kWarpSmem = kRingBytes + kMaxStages * 8 + 2 * kDW * 32 * 4;

// Stages the rw floats of a small per-edge operand (rw in 1, 2, 4, 8, 16).
__device__ __forceinline__ void stage_small(float* dst, const float* src, int rw) {
  if (rw == 1) {
    cp_async_4(dst, src);
  } else if (rw == 2) {
    cp_async_8(dst, src);
  } else {
    for (int q = 0; q < rw; q += 4) cp_async_16(dst + q, src + q);
  }
}

// SMALL: a small per-edge operand (rhs of width rw and/or the other-endpoint
// scale) is staged next to the gathered rows.
template <int VPL, int BOP, int ROP, bool ARG, bool SMALL>
__global__ void __launch_bounds__(kWarps * 32, 1) k_stream(const StreamLaunch p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  unsigned char* wbase = smem + warp * kWarpSmem;
  float* ring = reinterpret_cast<float*>(wbase);
  uint64_t* bars = reinterpret_cast<uint64_t*>(wbase + kRingBytes);
  uint32_t* id_o = reinterpret_cast<uint32_t*>(wbase + kRingBytes + kMaxStages * 8);
  uint32_t* id_e = id_o + kDW * 32;
  if (lane == 0) {
    for (int b = 0; b < kMaxStages; ++b) mbar_init(&bars[b], 1);
    fence_mbar_init();
  }
  __syncwarp();
  uint32_t phase = 0;  // bit b: parity of bars[b]'s next completion

  constexpr int kRun = VPL == 1 ? 8 : 4;  // edges folded per batch
  const RowLaunch L = p.row;              // register copy (no param reloads)
  const int RW = SMALL ? p.rhs_width : 0;
  const bool SCALE = SMALL && L.other_scale != nullptr;
  const bool need_eid = L.lhs.role == ROLE_EID || (RW && L.rhs.role == ROLE_EID);

  // First unit static and SM-interleaved (units 0..grid-1 land on distinct
  // SMs, so the long-row slices listed first spread over the chip instead of
  // piling onto CTA 0), then dynamic from the counter.
  const uint32_t n_static = gridDim.x * kWarps;
  uint32_t next_unit = blockIdx.x + gridDim.x * static_cast<uint32_t>(warp);
  for (;;) {
    const uint32_t unit = next_unit;
    if (unit >= p.n_units) break;
    if (lane == 0) next_unit = atomicAdd(p.counter, 1u) + n_static;
    next_unit = __shfl_sync(kFull, next_unit, 0);

    uint32_t r0, r1;
    int c0, cw;
    if (unit < p.n_long_units) {
      const uint32_t li = unit / p.long_slices;
      const uint32_t sl = unit - li * p.long_slices;
      r0 = __ldg(p.long_rows + li);
      r1 = r0 + 1;
      c0 = static_cast<int>(sl) * p.long_sw;
      cw = min(p.long_sw, L.width - c0);
    } else {
      const uint32_t u = unit - p.n_long_units;
      const uint32_t si = u / p.seg_slices;
      const uint32_t sl = u - si * p.seg_slices;
      const uint2 seg = __ldg(p.segs + si);
      r0 = seg.x;
      r1 = seg.y;
      c0 = static_cast<int>(sl) * p.seg_sw;
      cw = min(p.seg_sw, L.width - c0);
    }
    const uint32_t e0 = __ldg(L.indptr + r0);
    const uint32_t e1 = __ldg(L.indptr + r1);
    const unsigned long long t_unit0 = p.trace ? globaltimer_ns() : 0ull;

    // ring geometry for this unit's slice width
    const int slot_f = (cw + 3) & ~3;
    const uint32_t slot_bytes = static_cast<uint32_t>(slot_f) * 4u;
    const int per_edge = slot_f + RW + (SCALE ? 1 : 0);
    int nst = kRingBytes / (kStage * 4 * per_edge);
    nst = nst > kMaxStages ? kMaxStages : (nst < 1 ? 1 : nst);
    const int nslots = nst * kStage;
    float* tab_r = ring + nslots * slot_f;
    float* tab_s = tab_r + nslots * RW;
    const float* lhs_base = L.lhs.base + c0;
    // LSU staging for narrow slices whose 16-byte chunk count is a power of 2
    const bool lsu = slot_bytes < p.tma_min_bytes && (slot_f & (slot_f - 1)) == 0;

    const uint32_t n_edges = e1 - e0;
    const uint32_t n_stages = (n_edges + kStage - 1) / kStage;

    // ---- issue side: id windows (32 edges each) staged into a per-warp
    // shared ring with cp.async, kDW windows ahead of the issue cursor and
    // completed with cp.async.wait_group.  Loaded latency is ~6 us: ids held
    // in registers would stall the warp on the newest load at every window.
    int iwin = -1;
    auto load_win = [&](int w) {
      const uint32_t j = e0 + 32u * static_cast<uint32_t>(w) + lane;
      const int sl = (w % kDW) * 32 + lane;
      if (j < e1) {
        cp_async_4(id_o + sl, L.indices + j);
        if (need_eid) cp_async_4(id_e + sl, L.eids + j);
      }
      cp_async_commit();
    };
    auto issue = [&](uint32_t s) {
      const int w = static_cast<int>(s >> 2);  // issue() runs s = 0, 1, 2, ...
      if (w != iwin) {
        if (iwin < 0) {
#pragma unroll 1
          for (int d = 0; d < kDW; ++d) load_win(d);
        } else {
          load_win(w + kDW - 1);  // reuses the slot of window w-1
        }
        cp_async_wait_group<kDW - 1>();  // window w has landed (per thread)
        __syncwarp();                    // ... and is visible to every lane
        iwin = w;
      }
      const int b = static_cast<int>(s % static_cast<uint32_t>(nst));
      const uint32_t j0 = e0 + s * kStage;
      const uint32_t cnt = min(static_cast<uint32_t>(kStage), e1 - j0);
      const int wbase_slot = (w % kDW) * 32 + static_cast<int>(s & 3u) * kStage;
      const int src_slot = wbase_slot + (lane & (kStage - 1));
      const uint32_t other = id_o[src_slot];
      const uint32_t eid = need_eid ? id_e[src_slot] : 0u;
      const uint32_t l = static_cast<uint32_t>(lane);
      const int slot = b * kStage + lane;
      const uint32_t j = j0 + l;
      if constexpr (SMALL) {
        if (l < cnt) {
          if (RW > 0) {
            const int64_t rr = operand_row(L.rhs.role, 0, other, eid, j);
            stage_small(tab_r + slot * RW, L.rhs.base + rr * L.rhs.ld, RW);
          }
          if (SCALE) cp_async_4(tab_s + slot, L.other_scale + other);
        }
      }
      if (lsu) {
        // LSU staging: the stage's 8 x cpe 16-byte chunks spread over the
        // 32 lanes (coalesced within each edge's slice), tracked by the
        // same mbarrier through cp.async.mbarrier.arrive.
        const int cpe_log = __ffs(slot_f) - 3;  // slot_f = 4 << cpe_log
        const int chunks = kStage << cpe_log;
        for (int q0 = 0; q0 < chunks; q0 += 32) {
          const int q = q0 + lane;
          const int le = q >> cpe_log;
          const int ch = q - (le << cpe_log);
          if (q < chunks && static_cast<uint32_t>(le) < cnt) {
            const uint32_t o2 = id_o[wbase_slot + le];
            const uint32_t e2 = need_eid ? id_e[wbase_slot + le] : 0u;
            const int64_t lr = operand_row(L.lhs.role, 0, o2, e2, j0 + le);
            cp_async_16(ring + (b * kStage + le) * slot_f + ch * 4,
                        lhs_base + lr * L.lhs.ld + ch * 4);
          }
        }
        cp_async_arrive(&bars[b]);
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[b]);
        return;
      }
      if constexpr (SMALL) {
        if (lane < kStage) cp_async_arrive(&bars[b]);
        __syncwarp();
      }
      if (lane == 0) mbar_arrive_expect_tx(&bars[b], cnt * slot_bytes);
      __syncwarp();
      if (l < cnt) {
        const int64_t lr = operand_row(L.lhs.role, 0, other, eid, j);
        tma_load_1d(ring + slot * slot_f, lhs_base + lr * L.lhs.ld, slot_bytes, &bars[b]);
      }
    };

    const uint32_t pro = min(n_stages, static_cast<uint32_t>(nst));
    for (uint32_t s = 0; s < pro; ++s) issue(s);

    // ---- fold side: row-end windows (lane k <-> indptr[rb + 1 + k])
    uint32_t rb = r0;
    uint32_t rwin = 0, rnxt = 0;
    if (r0 + 1 + lane <= r1) rwin = __ldg(L.indptr + r0 + 1 + lane);
    if (r0 + 33 + lane <= r1) rnxt = __ldg(L.indptr + r0 + 33 + lane);
    uint32_t r = r0;
    uint32_t row_start = e0;
    uint32_t row_end = __shfl_sync(kFull, rwin, 0);

    float acc[VPL][4];
    uint32_t arg[VPL][4];
    auto reset = [&]() {
#pragma unroll
      for (int v = 0; v < VPL; ++v)
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          acc[v][t] = red_identity<ROP>();
          arg[v][t] = 0xffffffffu;
        }
    };
    reset();

    auto finalize = [&]() {
      const uint32_t deg = row_end - row_start;
      float* orow = L.out + static_cast<int64_t>(r) * L.out_ld + c0;
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        const int c = lane * 4 + v * 128;
        if (c >= cw) continue;
        float o[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          float a = acc[v][t];
          if constexpr (ROP == R_MAX || ROP == R_MIN) {
            if (deg == 0) a = 0.0f;
          }
          if (L.mean) a = deg ? __fdiv_rn(a, __uint2float_rn(deg)) : 0.0f;
          o[t] = a;
        }
        if (c + 4 <= cw) {
          store_vec<4>(orow + c, o);
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
            if (L.arg_other)
              L.arg_other[ab + t] = none ? -1 : static_cast<int32_t>(__ldg(L.indices + arg[v][t]));
            if (L.arg_edge)
              L.arg_edge[ab + t] = none ? -1 : static_cast<int32_t>(__ldg(L.eids + arg[v][t]));
          }
        }
      }
      reset();
    };
    auto advance_row = [&]() {
      ++r;
      row_start = row_end;
      if (r - rb >= 32u) {
        rb += 32u;
        rwin = rnxt;
        rnxt = 0;
        if (rb + 33 + lane <= r1) rnxt = __ldg(L.indptr + rb + 33 + lane);
      }
      row_end = __shfl_sync(kFull, rwin, static_cast<int>(r - rb));
    };

    // per-lane column offsets and (multi-head) rhs element of each vector
    bool col_ok[VPL];
    int rv_off[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      const int c = lane * 4 + v * 128;
      col_ok[v] = c < cw;
      rv_off[v] = RW > 1 ? (c0 + c) / L.rhs.group : 0;
    }

    uint32_t j = e0;
    for (uint32_t s = 0; s < n_stages; ++s) {
      const int b = static_cast<int>(s % static_cast<uint32_t>(nst));
      mbar_wait(&bars[b], (phase >> b) & 1u);
      phase ^= 1u << b;
      const uint32_t cnt = min(static_cast<uint32_t>(kStage), e1 - j);
      uint32_t k = 0;
      while (k < cnt) {
        while (j == row_end) {
          finalize();
          advance_row();
        }
        // a run of edges of the current row inside this stage: all shared
        // loads first (ILP), then the in-order fold
        const uint32_t run = min(min(cnt - k, row_end - j), static_cast<uint32_t>(kRun));
        const int slot0 = b * kStage + static_cast<int>(k);
        float4 xv[kRun][VPL];
        float rv[kRun][VPL];
        float sc[kRun];
#pragma unroll
        for (int q = 0; q < kRun; ++q) {
          if (static_cast<uint32_t>(q) < run) {
            const int slot = slot0 + q;
            const float* srow = ring + slot * slot_f;
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
              if (col_ok[v]) xv[q][v] = *reinterpret_cast<const float4*>(srow + lane * 4 + v * 128);
              rv[q][v] = 0.0f;
              if constexpr (SMALL) {
                if (RW > 0) rv[q][v] = tab_r[slot * RW + rv_off[v]];
              }
            }
            sc[q] = 1.0f;
            if constexpr (SMALL) {
              if (SCALE) sc[q] = tab_s[slot];
            }
          }
        }
#pragma unroll
        for (int q = 0; q < kRun; ++q) {
          if (static_cast<uint32_t>(q) < run) {
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
              if (!col_ok[v]) continue;
              const float xs[4] = {xv[q][v].x, xv[q][v].y, xv[q][v].z, xv[q][v].w};
#pragma unroll
              for (int t = 0; t < 4; ++t) {
                float m = bin_apply<BOP>(xs[t], rv[q][v]);
                if constexpr (SMALL) {
                  if (SCALE) m = __fmul_rn(m, sc[q]);
                }
                if constexpr (ARG) {
                  if (red_wins<ROP>(acc[v][t], m)) {
                    acc[v][t] = m;
                    arg[v][t] = j + q;
                  }
                } else {
                  acc[v][t] = red_combine<ROP>(acc[v][t], m);
                }
              }
            }
          }
        }
        k += run;
        j += run;
      }
      // Every value read from the stage's slots has been consumed by the fold
      // above (in registers), and __syncwarp orders all lanes' reads before
      // the refill is issued.  No proxy fence here: fence.proxy.async waits
      // for the warp's outstanding bulk copies and would drain the pipeline
      // every stage (measured: one stage per memory latency).
      __syncwarp();
      if (s + nst < n_stages) issue(s + nst);
    }
    // the current row (if any edges remain unaccounted) and trailing empty rows
    while (r < r1) {
      finalize();
      if (r + 1 < r1) {
        advance_row();
      } else {
        ++r;
      }
    }
    if (p.trace && lane == 0) {
      unsigned long long* t = p.trace + 4ull * unit;
      t[0] = t_unit0;
      t[1] = globaltimer_ns();
      t[2] = (static_cast<unsigned long long>(smid()) << 32) | static_cast<unsigned>(warp);
      t[3] = e1 - e0;
    }
  }
}

template <int VPL, int BOP, int ROP, bool ARG, bool SMALL>
cudaError_t launch_k(const StreamLaunch& p, cudaStream_t s) {
  const int smem_bytes = kWarps * kWarpSmem;
  static int configured_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    cudaError_t e = cudaFuncSetAttribute(k_stream<VPL, BOP, ROP, ARG, SMALL>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    if (e != cudaSuccess) return e;
    configured_dev = dev;
  }
  cudaError_t e = cudaMemsetAsync(p.counter, 0, sizeof(uint32_t), s);
  if (e != cudaSuccess) return e;
  const unsigned grid = static_cast<unsigned>(p.row.num_sms > 0 ? p.row.num_sms : 148);
  k_stream<VPL, BOP, ROP, ARG, SMALL><<<grid, kWarps * 32, smem_bytes, s>>>(p);
  note_launch();
  return cudaGetLastError();
}

template <int VPL, int BOP, int ROP, bool ARG>
cudaError_t launch_small(const StreamLaunch& p, cudaStream_t s) {
  if constexpr (BOP == B_COPY) {
    // copy has no rhs; the only small operand is the other-endpoint scale
    return p.row.other_scale ? launch_k<VPL, BOP, ROP, ARG, true>(p, s)
                             : launch_k<VPL, BOP, ROP, ARG, false>(p, s);
  } else {
    return launch_k<VPL, BOP, ROP, ARG, true>(p, s);
  }
}

template <int VPL, int BOP>
cudaError_t launch_red(const StreamLaunch& p, cudaStream_t s) {
  const bool arg = p.row.arg_other || p.row.arg_edge;
  switch (p.row.reduce) {
    case R_SUM: return launch_small<VPL, BOP, R_SUM, false>(p, s);
    case R_MAX: return arg ? launch_small<VPL, BOP, R_MAX, true>(p, s)
                           : launch_small<VPL, BOP, R_MAX, false>(p, s);
    case R_MIN: return arg ? launch_small<VPL, BOP, R_MIN, true>(p, s)
                           : launch_small<VPL, BOP, R_MIN, false>(p, s);
    case R_PROD: return launch_small<VPL, BOP, R_PROD, false>(p, s);
    default: return launch_small<VPL, BOP, R_LAST, false>(p, s);
  }
}

template <int VPL>
cudaError_t launch_bin(const StreamLaunch& p, cudaStream_t s) {
  switch (p.row.binop) {
    case B_ADD: return launch_red<VPL, B_ADD>(p, s);
    case B_SUB: return launch_red<VPL, B_SUB>(p, s);
    case B_MUL: return launch_red<VPL, B_MUL>(p, s);
    case B_DIV: return launch_red<VPL, B_DIV>(p, s);
    default: return launch_red<VPL, B_COPY>(p, s);
  }
}

}  // namespace

cudaError_t launch_stream(const StreamLaunch& p, cudaStream_t s) {
  if (p.n_units == 0) return cudaSuccess;
  return p.seg_sw > 128 ? launch_bin<2>(p, s) : launch_bin<1>(p, s);
}

}  // namespace gspmm_b200

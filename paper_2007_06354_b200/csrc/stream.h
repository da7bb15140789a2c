// stream.h -- launch descriptor of the planned row kernels (gather_impl.cuh):
// the segment kernel k_gather and the long-row column-unit kernel k_long_rg.
#pragma once

#include "internal.h"

namespace gspmm_b200 {

struct StreamLaunch {
  RowLaunch row;
  // device plan (built at graph upload)
  const uint2* segs = nullptr;        // [n_segs] (row_begin, row_end), long rows excluded
  uint32_t n_segs = 0;
  // long-row column units, heaviest first (built per plan level and width):
  // .x = row, .y = c0 | (cw << 16)
  const uint2* long_units = nullptr;
  uint32_t* counter = nullptr;        // work-unit counter (zeroed per launch)
  int seg_sw = 256;                   // columns per segment unit
  uint32_t seg_slices = 1;
  uint32_t n_units = 0;
  int rhs_width = 0;  // small-operand floats per edge (0 = none, 1 = scalar, H = heads)
  int mode = 0;       // 0 = row segments (k_gather), 1 = long-row units (k_long_rg)
  uint32_t grid = 0;  // mode 1: CTAs (0 = one per SM)
  // Programmatic dependent launch of the pair (long-row kernel, segment
  // kernel) on one stream: 0 = plain launches (each zeroes its counter);
  // 1 = this kernel is the primary (its CTAs release the dependent grid as
  // they start); 2 = this kernel is the dependent (its blocks take the SMs
  // the primary's CTAs leave, and wait for the primary's end before they
  // exit, so the stream sees the pair complete in order).  With 1 / 2 the
  // caller has zeroed both counters before the primary.
  int pdl = 0;
};

// The planned row kernels (gather_copy.cu dispatches on the operator).
cudaError_t launch_gather(const StreamLaunch& p, cudaStream_t s);

}  // namespace gspmm_b200

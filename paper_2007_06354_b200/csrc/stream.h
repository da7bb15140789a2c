// stream.h -- launch descriptor of the TMA-staged streaming row kernel.
#pragma once

#include <cuda.h>

#include "internal.h"

namespace gspmm_b200 {

struct StreamLaunch {
  RowLaunch row;
  // device plan (built at graph upload)
  const uint2* segs = nullptr;        // [n_segs] (row_begin, row_end), long rows excluded
  uint32_t n_segs = 0;
  const uint32_t* long_rows = nullptr;  // [n_long], descending degree
  uint32_t n_long = 0;
  uint32_t* counter = nullptr;        // work-unit counter (zeroed per launch)
  // per-call slicing
  int seg_sw = 256;       // columns per segment unit
  int long_sw = 32;       // columns per long-row unit
  uint32_t seg_slices = 1, long_slices = 1;
  uint32_t n_long_units = 0, n_units = 0;
  int rhs_width = 0;      // staged floats per edge of the small operand (0 = none)
  int mode = 0;           // gather.cu: 0 = row segments, 1 = long rows (one per CTA)
  uint32_t long_ctas = 0; // gather.cu mode 1: grid size (0 = one per SM)
  // gather.cu mode 1: the first n_xl long rows (heaviest) are cut into
  // xl_slices narrow slices of xl_sw columns (units [0, n_xl_units)), the
  // rest into long_slices slices of long_sw columns
  uint32_t n_xl = 0, xl_slices = 1, n_xl_units = 0;
  int xl_sw = 32;
  bool long_tma = false;  // GSPMM_LONG_TMA=1: warp-specialised TMA long rows
  // long rows through TMA tile::gather4 (k_long_g4, the default): box
  // widths (floats, multiples of 8, >= the slice width) of the two tensor maps
  bool long_g4 = false;
  int g4_box = 0, g4_box_xl = 0;
  bool long_ws = true;  // long rows: k_long_ws (default) or k_long (GSPMM_LONG_KERNEL=ldg)
  // Units whose gathered slice is narrower than this many bytes stage rows
  // with per-lane 16-byte cp.async (LSU path) instead of one TMA bulk copy
  // per edge: small bulk copies are bound by the TMA request rate.
  uint32_t tma_min_bytes = 512;
  // Development trace (GSPMM_UNIT_TRACE=<file>): per unit {start_ns, end_ns,
  // (smid << 32) | warp, edges}.  Null in production.
  unsigned long long* trace = nullptr;
};

// TMA-staged variant (stream.cu; GSPMM_KERNEL=tma) and the production
// register-staged kernel (gather.cu).  Same descriptor, same results.
cudaError_t launch_stream(const StreamLaunch& p, cudaStream_t s);
cudaError_t launch_gather(const StreamLaunch& p, cudaStream_t s);

// 2-D tensor map over the rows of a full-width operand (dims {width, rows},
// row pitch ld), box {box, 1}: the source of the gather4 long-row kernel.
// False if the driver rejects it.
bool encode_rows_tmap(CUtensorMap* map, const OperandDesc& d, int width, int box);

}  // namespace gspmm_b200

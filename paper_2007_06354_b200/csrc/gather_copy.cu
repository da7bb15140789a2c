// gather_copy.cu -- copy_u / copy_e instantiations of the production row
// kernel (gather_impl.cuh) and the kernel dispatcher.
#include "gather_impl.cuh"

namespace gspmm_b200 {

cudaError_t launch_gather_copy(const StreamLaunch& p, cudaStream_t s) {
  return gather_detail::launch_bop<B_COPY>(p, s);
}

cudaError_t launch_gather(const StreamLaunch& p, cudaStream_t s) {
  if (p.n_units == 0) return cudaSuccess;
  switch (p.row.binop) {
    case B_COPY: return launch_gather_copy(p, s);
    case B_MUL: return launch_gather_mul(p, s);
    default: return launch_gather_arith(p, s);
  }
}

}  // namespace gspmm_b200

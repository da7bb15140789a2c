// gather_arith.cu -- add / sub / div instantiations.
#include "gather_impl.cuh"

namespace gspmm_b200 {

cudaError_t launch_gather_arith(const StreamLaunch& p, cudaStream_t s) {
  switch (p.row.binop) {
    case B_ADD: return gather_detail::launch_bop<B_ADD>(p, s);
    case B_SUB: return gather_detail::launch_bop<B_SUB>(p, s);
    default: return gather_detail::launch_bop<B_DIV>(p, s);
  }
}

}  // namespace gspmm_b200

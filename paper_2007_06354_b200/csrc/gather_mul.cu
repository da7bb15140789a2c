// gather_mul.cu -- u_mul_e / v_mul_e (GCN, GAT, backward) instantiations.
#include "gather_impl.cuh"

namespace gspmm_b200 {

cudaError_t launch_gather_mul(const StreamLaunch& p, cudaStream_t s) {
  return gather_detail::launch_bop<B_MUL>(p, s);
}

}  // namespace gspmm_b200

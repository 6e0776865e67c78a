// k_mask_fit<D> instantiations for D in [17, 20] (eval_masks.cuh).
#include "eval_masks.cuh"

namespace speedrec {

cudaError_t mask_fit_launch_d(int D, unsigned grid, cudaStream_t st, const MaskArgs& M) {
  switch (D) {
    SR_MASK_FIT_CASE(17)
    SR_MASK_FIT_CASE(18)
    SR_MASK_FIT_CASE(19)
    SR_MASK_FIT_CASE(20)
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace speedrec

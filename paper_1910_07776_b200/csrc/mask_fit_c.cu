// k_mask_fit<D> instantiations for D in [14, 16] (eval_masks.cuh).
#include "eval_masks.cuh"

namespace speedrec {

cudaError_t mask_fit_launch_c(int D, unsigned grid, cudaStream_t st, const MaskArgs& M) {
  switch (D) {
    SR_MASK_FIT_CASE(14)
    SR_MASK_FIT_CASE(15)
    SR_MASK_FIT_CASE(16)
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace speedrec

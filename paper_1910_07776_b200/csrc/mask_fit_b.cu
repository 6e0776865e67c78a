// k_mask_fit<D> instantiations for D in [10, 13] (eval_masks.cuh).
#include "eval_masks.cuh"

namespace speedrec {

cudaError_t mask_fit_launch_b(int D, unsigned grid, cudaStream_t st, const MaskArgs& M) {
  switch (D) {
    SR_MASK_FIT_CASE(10)
    SR_MASK_FIT_CASE(11)
    SR_MASK_FIT_CASE(12)
    SR_MASK_FIT_CASE(13)
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace speedrec

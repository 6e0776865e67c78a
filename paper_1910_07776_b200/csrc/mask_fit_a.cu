// k_mask_fit<D> instantiations for D in [0, 9] (eval_masks.cuh).
#include "eval_masks.cuh"

namespace speedrec {

cudaError_t mask_fit_launch_a(int D, unsigned grid, cudaStream_t st, const MaskArgs& M) {
  switch (D) {
    SR_MASK_FIT_CASE(0)
    SR_MASK_FIT_CASE(1)
    SR_MASK_FIT_CASE(2)
    SR_MASK_FIT_CASE(3)
    SR_MASK_FIT_CASE(4)
    SR_MASK_FIT_CASE(5)
    SR_MASK_FIT_CASE(6)
    SR_MASK_FIT_CASE(7)
    SR_MASK_FIT_CASE(8)
    SR_MASK_FIT_CASE(9)
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace speedrec

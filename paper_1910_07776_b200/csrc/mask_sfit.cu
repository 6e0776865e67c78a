// k_mask_sfit<D> instantiations, D = suffix system size 0..10 (eval_schur.cuh).
#include "eval_schur.cuh"

namespace speedrec {

#define SR_SFIT_CASE(K)                                                             \
  case K:                                                                           \
    k_mask_sfit<K><<<grid, kSfitThreads, 0, st>>>(SA, off, n_items, fold_chunks);   \
    return cudaGetLastError();

cudaError_t mask_sfit_launch(int D, unsigned grid, cudaStream_t st, const SchurArgs& SA, int off, int n_items,
                             int fold_chunks) {
  switch (D) {
    SR_SFIT_CASE(0)
    SR_SFIT_CASE(1)
    SR_SFIT_CASE(2)
    SR_SFIT_CASE(3)
    SR_SFIT_CASE(4)
    SR_SFIT_CASE(5)
    SR_SFIT_CASE(6)
    SR_SFIT_CASE(7)
    SR_SFIT_CASE(8)
    SR_SFIT_CASE(9)
    SR_SFIT_CASE(10)
    default:
      return cudaErrorInvalidValue;
  }
}

#define SR_SPREP_CASE(K)                                                  \
  case K:                                                                 \
    k_mask_sprep_p<K><<<grid, 128, 0, st>>>(SA, glist, ng);               \
    return cudaGetLastError();

cudaError_t mask_sprep_launch(int P, unsigned grid, cudaStream_t st, const SchurArgs& SA, const int32_t* glist, int ng) {
  switch (P) {
    SR_SPREP_CASE(0)
    SR_SPREP_CASE(1)
    SR_SPREP_CASE(2)
    SR_SPREP_CASE(3)
    SR_SPREP_CASE(4)
    SR_SPREP_CASE(5)
    SR_SPREP_CASE(6)
    SR_SPREP_CASE(7)
    SR_SPREP_CASE(8)
    SR_SPREP_CASE(9)
    SR_SPREP_CASE(10)
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace speedrec

// K2 (FP32, FMM_LEAF_TF32 / FMM_LEAF_3XTF32): tcgen05 tensor-core leaf -- not yet built.
#include "fmm_internal.h"

namespace fmm {
cudaError_t launch_gemm_tf32(const LeafNode*, int, int64_t, int64_t, int64_t, const Bases&, int,
                             cudaStream_t) {
  return cudaErrorNotSupported;
}
}  // namespace fmm

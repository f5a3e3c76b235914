// mma.cu -- tcgen05 / TMEM implicit-GEMM path (placeholder until the kernels land).
#include "internal.h"

namespace capsconv {

bool mma_supported(capsconv_op_t, const Problem &) { return false; }
size_t mma_workspace_bytes(capsconv_op_t, const Problem &) { return 0; }
cudaError_t mma_fwd(const Problem &, const void *, const void *, void *, void *, size_t, cudaStream_t) {
    return cudaErrorNotSupported;
}
cudaError_t mma_bwd_data(const Problem &, const void *, const void *, void *, void *, size_t, cudaStream_t) {
    return cudaErrorNotSupported;
}
cudaError_t mma_bwd_kernel(const Problem &, const void *, const void *, float *, void *, size_t, cudaStream_t) {
    return cudaErrorNotSupported;
}

}  // namespace capsconv

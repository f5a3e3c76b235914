// rows_conv.cu -- forward and data gradient for the D1-outer ("rows") layout
// on tcgen05 (placeholder until the kernel lands: no problem is taken).
#include "internal.h"

namespace capsconv {

bool rows_conv_supported(capsconv_op_t, const Problem &) { return false; }
size_t rows_conv_workspace_bytes(capsconv_op_t, const Problem &) { return 0; }
cudaError_t rows_conv_run(capsconv_op_t, const Problem &, const void *, const void *, void *, void *, size_t,
                          cudaStream_t) {
    return cudaErrorNotSupported;
}
bool rows_fc_supported(capsconv_op_t, const Problem &) { return false; }
size_t rows_fc_workspace_bytes(capsconv_op_t, const Problem &) { return 0; }
cudaError_t rows_fc_run(capsconv_op_t, const Problem &, const void *, const void *, void *, void *, size_t,
                        cudaStream_t) {
    return cudaErrorNotSupported;
}

}  // namespace capsconv

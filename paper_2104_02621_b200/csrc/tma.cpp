// tma.cpp -- host-side TMA descriptor encoding through the driver entry point
// (cuTensorMapEncodeTiled), fetched at run time so libcapsconv does not link
// libcuda directly.
#include "tma.h"

#include <mutex>

namespace capsconv {

namespace {
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
        cudaGetLastError();
    });
    return fn;
}
}  // namespace

bool make_capsule_tmap(CUtensorMap *map, const void *base, int64_t B, int64_t H, int64_t W, int64_t CS, int cc,
                       int box_w, int box_h, int box_b, int stride) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t elem = 2;  // bf16
    cuuint64_t dims[4] = {(cuuint64_t)(CS * 16), (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)B};
    cuuint64_t strides[3] = {(cuuint64_t)(CS * 16) * elem, (cuuint64_t)(W * CS * 16) * elem,
                             (cuuint64_t)(H * W * CS * 16) * elem};
    cuuint32_t box[4] = {(cuuint32_t)(cc * 16), (cuuint32_t)(box_w * stride), (cuuint32_t)(box_h * stride),
                         (cuuint32_t)box_b};
    cuuint32_t estr[4] = {1, (cuuint32_t)stride, (cuuint32_t)stride, 1};
    if (box[0] > 256 || box[1] > 256 || box[2] > 256 || box[3] > 256) return false;
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

}  // namespace capsconv

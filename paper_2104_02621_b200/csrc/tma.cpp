// tma.cpp -- host-side TMA descriptor encoding through the driver entry point
// (cuTensorMapEncodeTiled), fetched at run time so libcapsconv does not link
// libcuda directly.
#include "tma.h"
#include "rows.cuh"

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

namespace rows {

namespace {
CUtensorMapSwizzle swz_enum(int bytes) {
    return bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
           : bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
           : bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE;
}
}  // namespace

bool make_rows_map5(CUtensorMap *map, const void *base, int64_t B, int64_t Hs, int64_t Ws, int64_t E, int ce, int bx,
                    int by, int es_x, int es_y, int bb) {
    EncodeTiledFn fn = encode_fn();
    if (!fn || ce * 2 > 128 || bx > 256 || by > 256 || bx < 1 || by < 1 || bb < 1 || bb > 256) return false;
    const cuuint64_t el = 2;
    cuuint64_t dims[5] = {(cuuint64_t)E, 4, (cuuint64_t)Ws, (cuuint64_t)Hs, (cuuint64_t)B};
    cuuint64_t strides[4] = {(cuuint64_t)E * el, (cuuint64_t)(4 * E) * el, (cuuint64_t)(Ws * 4 * E) * el,
                             (cuuint64_t)(Hs * Ws * 4 * E) * el};
    cuuint32_t box[5] = {(cuuint32_t)ce, 4, (cuuint32_t)bx, (cuuint32_t)by, (cuuint32_t)bb};
    cuuint32_t estr[5] = {1, 1, (cuuint32_t)es_x, (cuuint32_t)es_y, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void *>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, swz_enum(ce * 2), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_rows_map4m(CUtensorMap *map, const void *base, int64_t rows, int64_t Ws, int64_t E, int ce, int bx, int by,
                     int es) {
    EncodeTiledFn fn = encode_fn();
    if (!fn || ce * 2 > 128 || bx > 256 || by > 256 || bx < 1 || by < 1) return false;
    const cuuint64_t el = 2;
    cuuint64_t dims[4] = {(cuuint64_t)E, 4, (cuuint64_t)Ws, (cuuint64_t)rows};
    cuuint64_t strides[3] = {(cuuint64_t)E * el, (cuuint64_t)(4 * E) * el, (cuuint64_t)(Ws * 4 * E) * el};
    cuuint32_t box[4] = {(cuuint32_t)ce, 4, (cuuint32_t)bx, (cuuint32_t)by};
    cuuint32_t estr[4] = {1, 1, (cuuint32_t)es, (cuuint32_t)es};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, swz_enum(ce * 2), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_rows_map2(CUtensorMap *map, const void *base, int64_t rows, int64_t E, int ce, int br, int swz) {
    EncodeTiledFn fn = encode_fn();
    if (!fn || br > 256 || br < 1) return false;
    cuuint64_t dims[2] = {(cuuint64_t)E, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)E * 2};
    cuuint32_t box[2] = {(cuuint32_t)ce, (cuuint32_t)br};
    cuuint32_t estr[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, swz_enum(swz), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_rows_map4(CUtensorMap *map, const void *base, int64_t B, int64_t P, int64_t E, int ce, int bp, int bb) {
    EncodeTiledFn fn = encode_fn();
    if (!fn || ce * 2 > 128 || bb > 256 || bp > 256) return false;
    const cuuint64_t el = 2;
    cuuint64_t dims[4] = {(cuuint64_t)E, 4, (cuuint64_t)P, (cuuint64_t)B};
    cuuint64_t strides[3] = {(cuuint64_t)E * el, (cuuint64_t)(4 * E) * el, (cuuint64_t)(P * 4 * E) * el};
    cuuint32_t box[4] = {(cuuint32_t)ce, 4, (cuuint32_t)bp, (cuuint32_t)bb};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, swz_enum(ce * 2), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace rows
}  // namespace capsconv

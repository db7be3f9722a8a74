// tmap.cuh — host helpers: TMA tensor-map encoding (driver entry point fetched
// through cudart, so the library does not link libcuda) and device queries.
#pragma once
#include <cudaTypedefs.h>

#include "common.cuh"

namespace lb {

inline PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

inline bool make_map_2d(CUtensorMap* map, const void* base, uint64_t dim0, uint64_t dim1, uint64_t stride1,
                        uint32_t box0, uint32_t box1, CUtensorMapSwizzle swz,
                        CUtensorMapDataType dtype = CU_TENSOR_MAP_DATA_TYPE_UINT8) {
    auto fn = get_encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {dim0, dim1};
    cuuint64_t strides[1] = {stride1};
    cuuint32_t box[2] = {box0, box1};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, dtype, 2, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// 4-D NHWC int8 im2col map for implicit-GeMM convolution (fprop): lower
// corner -pad, upper corner pad - (k-1), traversal stride = conv stride
// (the CUTLASS convention, cutlass/conv/collective/detail.hpp).  Each load
// brings `pixels` consecutive output pixels x `channels` channels of one
// filter tap (given as the instruction's im2col offsets).
inline bool make_map_im2col(CUtensorMap* map, const void* base, int n, int h, int w, int c, int kh, int kw,
                            int stride, int pad, uint32_t channels, uint32_t pixels, CUtensorMapSwizzle swz) {
    static PFN_cuTensorMapEncodeIm2col_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(p);
    }
    if (!fn) return false;
    cuuint64_t dims[4] = {(cuuint64_t)c, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n};
    cuuint64_t strides[3] = {(cuuint64_t)c, (cuuint64_t)w * c, (cuuint64_t)h * w * c};
    int lower[2] = {-pad, -pad};
    int upper[2] = {pad - (kw - 1), pad - (kh - 1)};
    cuuint32_t estr[4] = {1, (cuuint32_t)stride, (cuuint32_t)stride, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void*>(base), dims, strides, lower, upper,
                    channels, pixels, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// "Tap-pair" im2col map over a packed fp4 NHWC map whose rows lead with one
// zero pixel (row pitch (w+1) pixels of 64 bytes, one more zero pixel at the end): each virtual pixel
// is 128 bytes = two horizontally adjacent pixels (stride 64 bytes), so one
// load brings two taps of a 3-wide filter for 128 output pixels.  Stride 1,
// padding 1 (the left edge's zero fill must cover exactly the padding).
inline bool make_map_im2col_pairtap(CUtensorMap* map, const void* base, int n, int h, int w, int kh, int pad,
                                    uint32_t pixels) {
    static PFN_cuTensorMapEncodeIm2col_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(p);
    }
    if (!fn) return false;
    cuuint64_t dims[4] = {128, (cuuint64_t)w + 1, (cuuint64_t)h, (cuuint64_t)n};
    cuuint64_t strides[3] = {64, (cuuint64_t)(w + 1) * 64, (cuuint64_t)h * (w + 1) * 64};
    // map x' = x + 1 (the zero pixel leads each row): from the window's first
    // tap x, offset 0 covers (x-1, x) for the (zero dummy, kx = 0) pair and
    // offset 2 covers (x+1, x+2) for (kx = 1, kx = 2)
    int lower[2] = {-pad, -pad};
    int upper[2] = {pad - 3, pad - (kh - 1)};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void*>(base), dims, strides, lower, upper, 128,
                    pixels, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// 3-D view of the prepared fp4 filter rows for the tap pairs: {192 bytes = the
// three taps (128 channels each) of one filter row, ky (kh), output channel}.
// A 128-byte box at x = -64 reads (zero, tap (ky,0)) — the out-of-bounds half
// is zero-filled — and at x = 64 reads (tap (ky,1), tap (ky,2)).
inline bool make_map_filter_pairtap(CUtensorMap* map, const void* base, int kh, uint64_t rows, uint64_t row_bytes,
                                    uint32_t box_rows) {
    auto fn = get_encode_fn();
    if (!fn) return false;
    cuuint64_t dims[3] = {192, (cuuint64_t)kh, rows};
    cuuint64_t strides[2] = {192, row_bytes};
    cuuint32_t box[3] = {128, 1, box_rows};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

inline int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

}  // namespace lb

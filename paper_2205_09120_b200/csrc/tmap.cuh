// tmap.cuh — host helpers: TMA tensor-map encoding (driver entry point fetched
// through cudart, so the library does not link libcuda) and device queries.
#pragma once
#include <cudaTypedefs.h>

#include <atomic>
#include <mutex>

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

// The conv output [batch, oh, ow, cout] int16 as a 4-D map for boxes of
// {16 channels, 32 pixels of one output row}: boxes may start left of x = 0
// or run past ow / oh — the clipped elements are not written — which lets a
// run of consecutive padded positions be stored row by row.
// box_cols 16 (32-byte swizzle) or 64 (128-byte swizzle).
inline bool make_map_conv_out(CUtensorMap* map, void* base, int batch, int oh, int ow, int cout, uint32_t box_cols) {
    auto fn = get_encode_fn();
    if (!fn) return false;
    cuuint64_t dims[4] = {(cuuint64_t)cout, (cuuint64_t)ow, (cuuint64_t)oh, (cuuint64_t)batch};
    cuuint64_t strides[3] = {(cuuint64_t)cout * 2, (cuuint64_t)ow * cout * 2, (cuuint64_t)oh * ow * cout * 2};
    cuuint32_t box[4] = {box_cols, 32, 1, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 4, base, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE,
                    box_cols == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_32B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// The int16 NHWC conv output with boxes of {box_cols channels, box_px pixels, box_rows rows, 1 image}.
inline bool make_map_conv_out_box(CUtensorMap* map, void* base, int batch, int oh, int ow, int cout, uint32_t box_cols,
                                  uint32_t box_px, uint32_t box_rows, CUtensorMapSwizzle swz) {
    auto fn = get_encode_fn();
    if (!fn) return false;
    cuuint64_t dims[4] = {(cuuint64_t)cout, (cuuint64_t)ow, (cuuint64_t)oh, (cuuint64_t)batch};
    cuuint64_t strides[3] = {(cuuint64_t)cout * 2, (cuuint64_t)ow * cout * 2, (cuuint64_t)oh * ow * cout * 2};
    cuuint32_t box[4] = {box_cols, box_px, box_rows, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 4, base, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// The NHWC int8 feature map [n, h, w, c] as a 4-D tiled map for boxes of
// {128 channels, `pixels` pixels of a row, `rows` rows, 1 image}, no swizzle:
// a box may start left of / above the image and run past its right / bottom
// edge — those elements read as zero, which is the convolution's padding.
inline bool make_map_nhwc_box(CUtensorMap* map, const void* base, int n, int h, int w, int c, uint32_t pixels,
                              uint32_t rows) {
    auto fn = get_encode_fn();
    if (!fn) return false;
    cuuint64_t dims[4] = {(cuuint64_t)c, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n};
    cuuint64_t strides[3] = {(cuuint64_t)c, (cuuint64_t)w * c, (cuuint64_t)h * w * c};
    cuuint32_t box[4] = {128, pixels, rows, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
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

inline int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev;
}

constexpr int kMaxDevices = 64;

// SM count of the current device (cached per device: one process may drive
// several GPUs from different host threads).
inline int num_sms() {
    static std::atomic<int> sms[kMaxDevices] = {};  // 0 = not queried yet; racing writers store the same value
    const int dev = current_device();
    int v = dev < kMaxDevices ? sms[dev].load(std::memory_order_relaxed) : 0;
    if (!v) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        v = n > 0 ? n : 148;
        if (dev < kMaxDevices) sms[dev].store(v, std::memory_order_relaxed);
    }
    return v;
}

// Largest dynamic-shared-memory opt-in already applied to one kernel, per
// device (cudaFuncSetAttribute is per device).  ensure() raises the
// attribute the first time a device needs more than it holds.  The opt-in
// only ever grows and the attribute call and the cache update happen under
// one lock, so concurrent host threads asking for different sizes cannot
// leave the cache above what the driver holds.
struct SmemOptIn {
    std::atomic<int> bytes[kMaxDevices] = {};
    std::mutex mu;
    template <typename K>
    cudaError_t ensure(K kern, int need) {
        const int dev = current_device();
        if (dev < kMaxDevices && bytes[dev].load(std::memory_order_acquire) >= need) return cudaSuccess;
        std::lock_guard<std::mutex> lock(mu);
        const int have = dev < kMaxDevices ? bytes[dev].load(std::memory_order_relaxed) : 0;
        if (have >= need) return cudaSuccess;
        const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, need);
        if (e == cudaSuccess && dev < kMaxDevices) bytes[dev].store(need, std::memory_order_release);
        return e;
    }
};

}  // namespace lb

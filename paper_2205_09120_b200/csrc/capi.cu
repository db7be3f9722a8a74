// capi.cu — the C-ABI surface (include/lowbit_cuda.h): argument validation in
// the reference's order, kernel choice, and the host-buffer drop-in entry.
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>

#include "common.cuh"
#include "layout.cuh"
#include "tmap.cuh"
#include "hostctx.cuh"

namespace lb {
lowbit_status launch_bitserial(int mode, const uint8_t* a0, const uint8_t* a1, long long a_pitch, int m, int n,
                               int k, const void* weights, int b_ternary, int16_t* c, long long ldc,
                               cudaStream_t stream);
lowbit_status launch_tensor_pair(int a_ternary, int layout, const uint8_t* a0, const uint8_t* a1, long long a_pitch, int m,
                                 int n, int k, const void* weights, int b_ternary, int16_t* c, long long ldc,
                                 cudaStream_t stream);
lowbit_status launch_tensor_pair_i8(const int8_t* a, long long lda, int m, int n, int k, const void* weights,
                                    int b_ternary, int16_t* c, long long ldc, cudaStream_t stream);
lowbit_status launch_fp4_pair(int a_ternary, int layout, const uint8_t* a0, const uint8_t* a1, long long a_pitch, int m, int n,
                              int k, const void* weights, int b_ternary, int16_t* c, long long ldc,
                              cudaStream_t stream);
lowbit_status launch_tensor(int a_ternary, int layout, const uint8_t* a0, const uint8_t* a1, long long a_pitch, int m, int n,
                            int k, const void* weights, int b_ternary, int16_t* c, long long ldc,
                            cudaStream_t stream);
}  // namespace lb

namespace {
thread_local std::string g_msg;
thread_local long long g_v0 = 0, g_v1 = 0;
}  // namespace

namespace lbhost {
lowbit_status set_error(lowbit_status st, const char* msg, long long v0, long long v1) {
    g_msg = msg ? msg : "";
    g_v0 = v0;
    g_v1 = v1;
    return st;
}
lowbit_status cuda_status(cudaError_t e, const char* where) {
    char buf[512];
    std::snprintf(buf, sizeof buf, "CUDA error %s (%s) at %s", cudaGetErrorName(e), cudaGetErrorString(e), where);
    return set_error(LOWBIT_CUDA_ERROR, buf);
}
}  // namespace lbhost

using lbhost::set_error;

extern "C" int lowbit_abi_version(void) { return LOWBIT_ABI_VERSION; }

extern "C" const char* lowbit_status_string(int st) {
    switch (st) {
        case LOWBIT_OK: return "OK";
        case LOWBIT_ERROR: return "Error";
        case LOWBIT_ZERO_IN_BINARY: return "ZeroInBinaryInput";
        case LOWBIT_INVALID_CODE: return "InvalidCode";
        case LOWBIT_OUT_OF_BOUNDS: return "OutOfBounds";
        case LOWBIT_DEPTH_OVERFLOW: return "DepthOverflow";
        case LOWBIT_MODE_MISMATCH: return "ModeMismatch";
        case LOWBIT_CHANNEL_OVERFLOW: return "ChannelOverflow";
        case LOWBIT_EMPTY_OUTPUT: return "EmptyOutput";
        case LOWBIT_CUDA_ERROR: return "CudaError";
        case LOWBIT_INVALID_ARGUMENT: return "InvalidArgument";
        case LOWBIT_NO_DEVICE: return "NoDevice";
        default: return "Unknown";
    }
}

extern "C" const char* lowbit_last_error(void) { return g_msg.c_str(); }

extern "C" void lowbit_last_error_values(long long* v0, long long* v1) {
    if (v0) *v0 = g_v0;
    if (v1) *v1 = g_v1;
}

extern "C" lowbit_status lowbit_device_check(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return set_error(LOWBIT_NO_DEVICE, "no CUDA device visible; liblowbit_cuda has no CPU fallback");
    }
    int dev = 0, major = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    if (major != 10) return set_error(LOWBIT_NO_DEVICE, "liblowbit_cuda is built for sm_100a only");
    return LOWBIT_OK;
}

extern "C" long long lowbit_plane_pitch(int cols) {
    long long b = (cols + 7) / 8;
    return (b + 15) / 16 * 16;
}

// The reference's gemm_lowbit validation, in order (gemm.cpp:81-84, 94-100,
// check_cfg gemm.cpp:9-12, check_dims gemm.cpp:14-19).
static lowbit_status validate_gemm(int mode, bool a_ternary, int b_ternary, int a_rows, int a_cols, int b_n,
                                   int b_k, int m, int n, int k, int k_blk) {
    if (k_blk < 8 || (k_blk & 7) != 0) return set_error(LOWBIT_ERROR, "k_blk must be a positive multiple of 8");
    if (mode < 0 || mode > 2) return set_error(LOWBIT_INVALID_ARGUMENT, "unknown gemm mode");
    if (!a_ternary) {
        if (mode != LOWBIT_BNN) return set_error(LOWBIT_MODE_MISMATCH, "mode mismatch: binary left operand requires bnn mode");
        if (b_ternary) return set_error(LOWBIT_MODE_MISMATCH, "mode mismatch: bnn requires binary right operand");
    } else {
        if (mode == LOWBIT_BNN) return set_error(LOWBIT_MODE_MISMATCH, "mode mismatch: bnn requires a binary left operand");
        if (mode == LOWBIT_TNN && !b_ternary)
            return set_error(LOWBIT_MODE_MISMATCH, "mode mismatch: tnn requires a ternary right operand");
        if (mode == LOWBIT_TBN && b_ternary)
            return set_error(LOWBIT_MODE_MISMATCH, "mode mismatch: tbn requires a binary right operand");
    }
    if (m <= 0 || n <= 0 || k <= 0) return set_error(LOWBIT_OUT_OF_BOUNDS, "out of bounds: gemm dims");
    if (a_rows != m || a_cols != k) return set_error(LOWBIT_OUT_OF_BOUNDS, "out of bounds: left operand shape");
    if (b_k != k || b_n != n) return set_error(LOWBIT_OUT_OF_BOUNDS, "out of bounds: packed right operand shape");
    if (k > LOWBIT_K_MAX16) {
        char buf[96];
        std::snprintf(buf, sizeof buf, "depth %d exceeds k_max %d", k, LOWBIT_K_MAX16);
        return set_error(LOWBIT_DEPTH_OVERFLOW, buf, k, LOWBIT_K_MAX16);
    }
    return LOWBIT_OK;
}

// Static per-shape kernel table, from B200
// measurements (profiles/r01, bench.py per_config), reference-layout planes:
//   c1 360x96x256      int8 K3 6.4 us, fp4 K5 8.6 us, bit-serial 12.6 us (graph replay)
//   c2 sweep (64)      int8 K3 5.0 us, fp4 K5 5.7 us, bit-serial 10.4 us per shape
//   c3 8192^2x4096     fp4 K5 4.04 POPS, int8 K3 2.7 POPS, bit-serial 0.28 POPS (95% of POPC peak)
//   c5 1Mx1024x2048    fp4 K5 4.73 POPS, int8 K3 2.50 POPS
// Launch-bound shapes (under ~1 GOP) take the int8 kernel, everything else the
// fp4 one.  (NIBBLES planes always run K5, LANES planes K3; lowbit_gemm_ex.)
// The bit-serial kernel stays selectable and is the one the grouped
// small-GeMM launch uses (lowbit_gemm_grouped).
extern "C" int lowbit_select_kernel(int mode, int m, int n, int k) {
    (void)mode;
    const double ops = 2.0 * (double)m * (double)n * (double)k;
    // Launch-bound shapes (< ~1 GOP), measured per call in a graph of back-to-back calls with every
    // kernel launched as a programmatic dependent (tools/c1_latency.py, PER_SHAPE=1; the 64 shapes of
    // config 2 take 250.7 us by this rule, 247.5 by the per-shape best, 286.1 on the single-CTA kernel
    // alone): outputs at least 96 columns wide take the int8 kernel, single-CTA up to 4 row tiles
    // (config 1: 3.5 us against 3.9 on the fp4 kernel); narrower ones the fp4 pair kernel, or the
    // int8 one when the depth is a single k-block.  Above that the fp4 kernel.
    if (ops < 1e9) {
        if (n >= 96) return m <= 512 ? LOWBIT_KERNEL_TENSOR_1CTA : LOWBIT_KERNEL_TENSOR_I8;
        return k <= 128 ? LOWBIT_KERNEL_TENSOR_I8 : LOWBIT_KERNEL_TENSOR;
    }
    return LOWBIT_KERNEL_TENSOR;
}

extern "C" lowbit_status lowbit_gemm(int mode, const uint8_t* a0, const uint8_t* a1, long long a_pitch, int a_rows,
                                     int a_cols, const void* weights, int b_ternary, int b_n, int b_k, int m, int n,
                                     int k, int k_blk, int16_t* c, long long ldc, int kernel, lowbit_stream stream) {
    return lowbit_gemm_ex(mode, LOWBIT_LAYOUT_REFERENCE, a0, a1, a_pitch, a_rows, a_cols, weights, b_ternary, b_n,
                          b_k, m, n, k, k_blk, c, ldc, kernel, stream);
}

extern "C" lowbit_status lowbit_gemm_ex(int mode, int a_layout, const uint8_t* a0, const uint8_t* a1,
                                        long long a_pitch, int a_rows, int a_cols, const void* weights, int b_ternary,
                                        int b_n, int b_k, int m, int n, int k, int k_blk, int16_t* c, long long ldc,
                                        int kernel, lowbit_stream stream) {
    const bool a_ternary = a1 != nullptr;
    lowbit_status st = validate_gemm(mode, a_ternary, b_ternary, a_rows, a_cols, b_n, b_k, m, n, k, k_blk);
    if (st) return st;
    if (!a0 || !weights || !c) return set_error(LOWBIT_INVALID_ARGUMENT, "gemm: NULL pointer");
    if ((a_pitch & 15) || a_pitch < (k + 7) / 8 || (reinterpret_cast<uintptr_t>(a0) & 15) ||
        (a_ternary && (reinterpret_cast<uintptr_t>(a1) & 15)))
        return set_error(LOWBIT_INVALID_ARGUMENT, "gemm: A planes need 16-byte aligned rows (pitch % 16 == 0)");
    if ((reinterpret_cast<uintptr_t>(weights) & 255))
        return set_error(LOWBIT_INVALID_ARGUMENT, "gemm: weights must be 256-byte aligned");
    if (ldc < n) return set_error(LOWBIT_INVALID_ARGUMENT, "gemm: ldc < n");
    if (a_layout != LOWBIT_LAYOUT_REFERENCE && a_layout != LOWBIT_LAYOUT_LANES && a_layout != LOWBIT_LAYOUT_NIBBLES)
        return set_error(LOWBIT_INVALID_ARGUMENT, "gemm: unknown A plane layout");
    if (kernel == LOWBIT_KERNEL_AUTO)
        kernel = a_layout == LOWBIT_LAYOUT_NIBBLES ? LOWBIT_KERNEL_TENSOR : lowbit_select_kernel(mode, m, n, k);
    cudaStream_t s = (cudaStream_t)stream;
    if (kernel == LOWBIT_KERNEL_BITSERIAL) {
        if (a_layout != LOWBIT_LAYOUT_REFERENCE)
            return set_error(LOWBIT_INVALID_ARGUMENT, "gemm: the bit-serial kernel reads REFERENCE-layout planes");
        return lb::launch_bitserial(mode, a0, a1, a_pitch, m, n, k, weights, b_ternary, c, ldc, s);
    }
    if (a_layout == LOWBIT_LAYOUT_NIBBLES && kernel != LOWBIT_KERNEL_TENSOR)
        return set_error(LOWBIT_INVALID_ARGUMENT, "gemm: NIBBLES planes run on the fp4 tensor-core kernel only");
    // TENSOR: the fp4 kernel K5 for NIBBLES and REFERENCE planes, the int8 kernel K3 for LANES planes
    if (kernel == LOWBIT_KERNEL_TENSOR && a_layout != LOWBIT_LAYOUT_LANES)
        return lb::launch_fp4_pair(a_ternary, a_layout, a0, a1, a_pitch, m, n, k, weights, b_ternary, c, ldc, s);
    if ((kernel == LOWBIT_KERNEL_TENSOR || kernel == LOWBIT_KERNEL_TENSOR_I8) && m > 128)
        return lb::launch_tensor_pair(a_ternary, a_layout, a0, a1, a_pitch, m, n, k, weights, b_ternary, c, ldc, s);
    if (kernel == LOWBIT_KERNEL_TENSOR_I8)
        return lb::launch_tensor(a_ternary, a_layout, a0, a1, a_pitch, m, n, k, weights, b_ternary, c, ldc, s);
    if (kernel == LOWBIT_KERNEL_TENSOR || kernel == LOWBIT_KERNEL_TENSOR_1CTA)
        return lb::launch_tensor(a_ternary, a_layout, a0, a1, a_pitch, m, n, k, weights, b_ternary, c, ldc, s);
    return set_error(LOWBIT_INVALID_ARGUMENT, "gemm: unknown kernel id");
}

extern "C" lowbit_status lowbit_gemm_i8(int mode, const int8_t* a, long long lda, int a_rows, int a_cols,
                                        const void* weights, int b_ternary, int b_n, int b_k, int m, int n, int k,
                                        int k_blk, int16_t* c, long long ldc, lowbit_stream stream) {
    // the A operand kind follows the mode (BNN binary, TNN/TBN ternary)
    lowbit_status st = validate_gemm(mode, mode != LOWBIT_BNN, b_ternary, a_rows, a_cols, b_n, b_k, m, n, k, k_blk);
    if (st) return st;
    if (!a || !weights || !c) return set_error(LOWBIT_INVALID_ARGUMENT, "gemm_i8: NULL pointer");
    if ((lda & 15) || lda < k || (reinterpret_cast<uintptr_t>(a) & 15))
        return set_error(LOWBIT_INVALID_ARGUMENT, "gemm_i8: A rows must be 16-byte aligned (lda % 16 == 0)");
    if ((reinterpret_cast<uintptr_t>(weights) & 255))
        return set_error(LOWBIT_INVALID_ARGUMENT, "gemm_i8: weights must be 256-byte aligned");
    if (ldc < n) return set_error(LOWBIT_INVALID_ARGUMENT, "gemm_i8: ldc < n");
    return lb::launch_tensor_pair_i8(a, lda, m, n, k, weights, b_ternary, c, ldc, (cudaStream_t)stream);
}

// ---------------------------------------------------------------------------
// Host-buffer drop-in.  Per-(thread, device) state, hostctx.cuh.
// ---------------------------------------------------------------------------
namespace {
struct ThreadState {
    lbhost::HostCtx* ctx[lb::kMaxDevices] = {};
    void release_all() {
        for (auto*& c : ctx) {
            delete c;  // ~HostCtx frees its scratch on its own device
            c = nullptr;
        }
    }
    ~ThreadState() { release_all(); }
};
thread_local ThreadState g_state;
}  // namespace

lbhost::HostCtx* lbhost::host_ctx() {
    const int dev = lb::current_device();
    if (dev < 0 || dev >= lb::kMaxDevices) return nullptr;
    HostCtx*& c = g_state.ctx[dev];
    if (!c) {
        c = new HostCtx;
        c->dev = dev;
    }
    return c;
}

extern "C" void lowbit_release_thread_state(void) { g_state.release_all(); }

using lbhost::HostCtx;
using lbhost::host_ctx;

extern "C" lowbit_status lowbit_gemm_lowbit_host(int mode, const uint8_t* a0, const uint8_t* a1, int a_rows,
                                                 int a_cols, const uint8_t* panels, int b_ternary, int b_n, int b_k,
                                                 int m, int n, int k, int k_blk, int16_t* c, int kernel,
                                                 lowbit_stream stream) {
    const bool a_ternary = a1 != nullptr;
    lowbit_status st = validate_gemm(mode, a_ternary, b_ternary, a_rows, a_cols, b_n, b_k, m, n, k, k_blk);
    if (st) return st;
    if (!a0 || !panels || !c) return set_error(LOWBIT_INVALID_ARGUMENT, "gemm_lowbit_host: NULL pointer");
    if ((st = lowbit_device_check())) return st;
    cudaStream_t s = (cudaStream_t)stream;
    const long long hstride = (k + 7) / 8;
    const long long pitch = lowbit_plane_pitch(k);
    const size_t abytes = (size_t)m * pitch;
    const size_t pbytes = lowbit_packed_b_bytes(b_ternary, n, k);
    const size_t wbytes = lowbit_weights_bytes(b_ternary, n, k);
    HostCtx* Xp = host_ctx();
    if (!Xp) return set_error(LOWBIT_INVALID_ARGUMENT, "host-buffer API: device ordinal out of range");
    HostCtx& X = *Xp;
    LB_CUDA_TRY(X.a0.ensure(abytes));
    if (a_ternary) LB_CUDA_TRY(X.a1.ensure(abytes));
    LB_CUDA_TRY(X.panels.ensure(pbytes));
    LB_CUDA_TRY(X.weights.ensure(wbytes));
    LB_CUDA_TRY(X.c.ensure((size_t)m * n * sizeof(int16_t)));
    LB_CUDA_TRY(X.ensure_streams());
    // Pageable caller memory (a std::vector, as the reference API hands out)
    // goes through pinned staging slots, copied on a few host threads, so the
    // DMA engines still run at the pinned rate; pinned memory is copied
    // directly.
    const bool in_pageable = !lbhost::host_pinned(a0) || (a_ternary && !lbhost::host_pinned(a1));
    const bool out_pageable = !lbhost::host_pinned(c);
    const bool staged = in_pageable || out_pageable;
    const long long a_row_bytes = hstride * (a_ternary ? 2 : 1), c_row_bytes = 2LL * n;
    int chunks;
    long long rows_per;
    if (staged) {  // ~16 MiB staging slots, whole 256-row m tiles
        const long long row_bytes = a_row_bytes > c_row_bytes ? a_row_bytes : c_row_bytes;
        static const long long slot_mb = lb::tuning_env("LOWBIT_STAGE_MB") ? atoi(lb::tuning_env("LOWBIT_STAGE_MB")) : 16;
        rows_per = ((slot_mb << 20) / row_bytes) / 256 * 256;
        if (rows_per < 256) rows_per = 256;
        if (rows_per > m) rows_per = m;
        chunks = (int)((m + rows_per - 1) / rows_per);
        for (int i = 0; i < HostCtx::kBounce; ++i) {
            if (in_pageable) LB_CUDA_TRY(X.bounce_in[i].ensure((size_t)rows_per * a_row_bytes));
            if (out_pageable) LB_CUDA_TRY(X.bounce_out[i].ensure((size_t)rows_per * c_row_bytes));
        }
    } else {  // the copy-in / compute / copy-out pipeline over <= 8 chunks of >= 1024 rows
        chunks = (int)((m + 1023) / 1024);
        if (chunks > HostCtx::kChunks) chunks = HostCtx::kChunks;
        if (chunks < 1) chunks = 1;
        rows_per = (m + chunks - 1) / chunks;
    }
    lbhost::StreamDrain drain{{X.s_in, X.s_out, s}};  // error paths wait for queued copies
    // weights: upload + prepare once on the caller's stream
    LB_CUDA_TRY(cudaMemcpyAsync(X.panels.ptr, panels, pbytes, cudaMemcpyHostToDevice, s));
    if ((st = lowbit_prepare_weights(b_ternary, static_cast<const uint8_t*>(X.panels.ptr), n, k, X.weights.ptr,
                                     stream)))
        return st;
    // the copy streams must not run ahead of work already queued on `s`
    LB_CUDA_TRY(cudaEventRecord(X.ev_w, s));
    LB_CUDA_TRY(cudaStreamWaitEvent(X.s_in, X.ev_w, 0));
    LB_CUDA_TRY(cudaStreamWaitEvent(X.s_out, X.ev_w, 0));
    lbhost::HostCopier* copier = nullptr;
    std::unique_ptr<lbhost::HostCopier> copier_owner;
    if (staged) {
        copier_owner.reset(new lbhost::HostCopier(lbhost::HostCopier::default_threads()));
        copier = copier_owner.get();
    }
    auto rows_of = [&](int ci, long long& r0, long long& rows) {
        r0 = (long long)ci * rows_per;
        rows = m - r0 < rows_per ? m - r0 : rows_per;
    };
    // host side of chunk `done`'s result: staging slot -> caller's C
    auto drain_c = [&](int done, lbhost::HostCopier::Job* jobs, int& nj) -> cudaError_t {
        long long r0, rows;
        rows_of(done, r0, rows);
        const int sl = done % HostCtx::kBounce;
        cudaError_t e = cudaEventSynchronize(X.ev_bout[sl]);
        if (e) return e;
        jobs[nj++] = {c + r0 * n, X.bounce_out[sl].ptr, (size_t)rows * c_row_bytes};
        return cudaSuccess;
    };
    for (int ci = 0; ci < chunks; ++ci) {
        long long r0, rows;
        rows_of(ci, r0, rows);
        const int sl = ci % HostCtx::kBounce, ev = ci % HostCtx::kChunks;
        uint8_t* d0 = static_cast<uint8_t*>(X.a0.ptr) + r0 * pitch;
        uint8_t* d1 = a_ternary ? static_cast<uint8_t*>(X.a1.ptr) + r0 * pitch : nullptr;
        const uint8_t* h0 = a0 + r0 * hstride;
        const uint8_t* h1 = a_ternary ? a1 + r0 * hstride : nullptr;
        if (staged) {
            // host copies of this round: A chunk ci into its slot, and C chunk ci - kBounce
            // (whose slot chunk ci reuses) out of it
            lbhost::HostCopier::Job jobs[3];
            int nj = 0;
            if (in_pageable) {
                if (ci >= HostCtx::kBounce) LB_CUDA_TRY(cudaEventSynchronize(X.ev_bin[sl]));  // slot's H2D done
                uint8_t* b = static_cast<uint8_t*>(X.bounce_in[sl].ptr);
                jobs[nj++] = {b, h0, (size_t)(rows * hstride)};
                if (a_ternary) jobs[nj++] = {b + rows * hstride, h1, (size_t)(rows * hstride)};
                h0 = b;
                h1 = a_ternary ? b + rows * hstride : nullptr;
            }
            if (out_pageable && ci >= HostCtx::kBounce) LB_CUDA_TRY(drain_c(ci - HostCtx::kBounce, jobs, nj));
            if (nj) copier->copy(jobs, nj);
        }
        if (pitch == hstride) {
            LB_CUDA_TRY(cudaMemcpyAsync(d0, h0, rows * pitch, cudaMemcpyHostToDevice, X.s_in));
            if (a_ternary) LB_CUDA_TRY(cudaMemcpyAsync(d1, h1, rows * pitch, cudaMemcpyHostToDevice, X.s_in));
        } else {  // re-pitch to 16-byte rows; zero the padding first
            LB_CUDA_TRY(cudaMemsetAsync(d0, 0, rows * pitch, X.s_in));
            LB_CUDA_TRY(cudaMemcpy2DAsync(d0, pitch, h0, hstride, hstride, rows, cudaMemcpyHostToDevice, X.s_in));
            if (a_ternary) {
                LB_CUDA_TRY(cudaMemsetAsync(d1, 0, rows * pitch, X.s_in));
                LB_CUDA_TRY(
                    cudaMemcpy2DAsync(d1, pitch, h1, hstride, hstride, rows, cudaMemcpyHostToDevice, X.s_in));
            }
        }
        if (in_pageable) LB_CUDA_TRY(cudaEventRecord(X.ev_bin[sl], X.s_in));
        LB_CUDA_TRY(cudaEventRecord(X.ev_in[ev], X.s_in));
        LB_CUDA_TRY(cudaStreamWaitEvent(s, X.ev_in[ev], 0));
        int16_t* dc = static_cast<int16_t*>(X.c.ptr) + r0 * n;
        if ((st = lowbit_gemm(mode, d0, d1, pitch, (int)rows, a_cols, X.weights.ptr, b_ternary, b_n, b_k, (int)rows,
                              n, k, k_blk, dc, n, kernel, stream)))
            return st;
        LB_CUDA_TRY(cudaEventRecord(X.ev_c[ev], s));
        LB_CUDA_TRY(cudaStreamWaitEvent(X.s_out, X.ev_c[ev], 0));
        int16_t* hc = out_pageable ? static_cast<int16_t*>(X.bounce_out[sl].ptr) : c + r0 * n;
        LB_CUDA_TRY(cudaMemcpyAsync(hc, dc, (size_t)rows * c_row_bytes, cudaMemcpyDeviceToHost, X.s_out));
        if (out_pageable) LB_CUDA_TRY(cudaEventRecord(X.ev_bout[sl], X.s_out));
    }
    if (out_pageable) {  // the last kBounce results are still in their slots
        for (int done = chunks > HostCtx::kBounce ? chunks - HostCtx::kBounce : 0; done < chunks; ++done) {
            lbhost::HostCopier::Job jobs[1];
            int nj = 0;
            LB_CUDA_TRY(drain_c(done, jobs, nj));
            copier->copy(jobs, nj);
        }
    }
    LB_CUDA_TRY(cudaEventRecord(X.ev_done, X.s_out));
    LB_CUDA_TRY(cudaStreamWaitEvent(s, X.ev_done, 0));
    LB_CUDA_TRY(cudaStreamSynchronize(s));
    drain.armed = false;
    return LOWBIT_OK;
}

extern "C" lowbit_status lowbit_encode_host(int ternary, const int8_t* values, int rows, int cols, uint8_t* plane0,
                                            uint8_t* plane1, lowbit_stream stream) {
    if (rows < 0 || cols < 0) return set_error(LOWBIT_INVALID_ARGUMENT, "encode: negative shape");
    if (rows == 0 || cols == 0) return LOWBIT_OK;
    if (!values || !plane0 || (ternary && !plane1)) return set_error(LOWBIT_INVALID_ARGUMENT, "encode: NULL pointer");
    lowbit_status st;
    if ((st = lowbit_device_check())) return st;
    cudaStream_t s = (cudaStream_t)stream;
    HostCtx* Xp = host_ctx();
    if (!Xp) return set_error(LOWBIT_INVALID_ARGUMENT, "host-buffer API: device ordinal out of range");
    HostCtx& X = *Xp;
    const long long sb = (cols + 7) / 8, pitch = lowbit_plane_pitch(cols);
    const size_t vbytes = (size_t)rows * cols, pbytes = (size_t)rows * pitch;
    LB_CUDA_TRY(X.vals.ensure(vbytes));
    LB_CUDA_TRY(X.a0.ensure(pbytes));
    if (ternary) LB_CUDA_TRY(X.a1.ensure(pbytes));
    LB_CUDA_TRY(X.flag.ensure(sizeof(int)));
    LB_CUDA_TRY(cudaMemsetAsync(X.flag.ptr, 0, sizeof(int), s));
    LB_CUDA_TRY(cudaMemcpyAsync(X.vals.ptr, values, vbytes, cudaMemcpyHostToDevice, s));
    if ((st = lowbit_encode(ternary, static_cast<const int8_t*>(X.vals.ptr), rows, cols, cols,
                            static_cast<uint8_t*>(X.a0.ptr), ternary ? static_cast<uint8_t*>(X.a1.ptr) : nullptr,
                            pitch, static_cast<int*>(X.flag.ptr), stream)))
        return st;
    int flag = 0;
    LB_CUDA_TRY(cudaMemcpyAsync(&flag, X.flag.ptr, sizeof(int), cudaMemcpyDeviceToHost, s));
    LB_CUDA_TRY(cudaMemcpy2DAsync(plane0, sb, X.a0.ptr, pitch, sb, rows, cudaMemcpyDeviceToHost, s));
    if (ternary) LB_CUDA_TRY(cudaMemcpy2DAsync(plane1, sb, X.a1.ptr, pitch, sb, rows, cudaMemcpyDeviceToHost, s));
    LB_CUDA_TRY(cudaStreamSynchronize(s));
    if (!ternary && flag) return set_error(LOWBIT_ZERO_IN_BINARY, "binary matrix contains a zero element");
    return LOWBIT_OK;
}

extern "C" lowbit_status lowbit_pack_b_host(int ternary, const uint8_t* b0, const uint8_t* b1, int k, int n,
                                            uint8_t* panels, lowbit_stream stream) {
    if (k <= 0 || n <= 0) return LOWBIT_OK;
    if (!b0 || !panels || (ternary && !b1)) return set_error(LOWBIT_INVALID_ARGUMENT, "pack_b: NULL pointer");
    lowbit_status st;
    if ((st = lowbit_device_check())) return st;
    cudaStream_t s = (cudaStream_t)stream;
    HostCtx* Xp = host_ctx();
    if (!Xp) return set_error(LOWBIT_INVALID_ARGUMENT, "host-buffer API: device ordinal out of range");
    HostCtx& X = *Xp;
    const size_t pbytes = (size_t)k * ((n + 7) / 8);
    const size_t obytes = lowbit_packed_b_bytes(ternary, n, k);
    LB_CUDA_TRY(X.a0.ensure(pbytes));
    if (ternary) LB_CUDA_TRY(X.a1.ensure(pbytes));
    LB_CUDA_TRY(X.panels.ensure(obytes));
    LB_CUDA_TRY(cudaMemcpyAsync(X.a0.ptr, b0, pbytes, cudaMemcpyHostToDevice, s));
    if (ternary) LB_CUDA_TRY(cudaMemcpyAsync(X.a1.ptr, b1, pbytes, cudaMemcpyHostToDevice, s));
    if ((st = lowbit_pack_b(ternary, static_cast<const uint8_t*>(X.a0.ptr),
                            ternary ? static_cast<const uint8_t*>(X.a1.ptr) : nullptr, k, n, (n + 7) / 8,
                            static_cast<uint8_t*>(X.panels.ptr), stream)))
        return st;
    LB_CUDA_TRY(cudaMemcpyAsync(panels, X.panels.ptr, obytes, cudaMemcpyDeviceToHost, s));
    LB_CUDA_TRY(cudaStreamSynchronize(s));
    return LOWBIT_OK;
}

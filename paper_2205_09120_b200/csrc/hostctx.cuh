// hostctx.cuh — state of the host-buffer entry points (lowbit_*_host), kept
// per (host thread, device).
//
// The reference is pure: every call owns its temporaries (std::vector, freed
// on return) and the only global state is thread_local kernel scratch
// (kernels.cpp:23).  The host-buffer forms here keep grow-only device scratch,
// two copy streams and their events per (host thread, device) so repeated
// calls do not re-allocate, and give all of it back:
//   * when the thread exits (thread_local destructor), and
//   * on demand through lowbit_release_thread_state().
// Nothing is shared between threads, so no lock is needed.
#pragma once
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"
#include "tmap.cuh"

namespace lbhost {

// True when `p` is page-locked (cudaMallocHost / cudaHostRegister): the DMA
// engines read and write it directly.  Pageable memory would make
// cudaMemcpyAsync stage synchronously through the driver (~11 GB/s H2D,
// ~17 GB/s D2H on the B200 boxes, tools/micro/host_copy_bw.cu).
inline bool host_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// A few host threads that split memcpy jobs between them (pageable caller
// buffers <-> pinned staging slots).  One per call of a host-buffer entry
// point; the workers are joined when it goes out of scope.
class HostCopier {
  public:
    struct Job {
        void* dst;
        const void* src;
        size_t bytes;
    };
    explicit HostCopier(int threads) : nthreads_(threads < 1 ? 1 : threads) {}
    ~HostCopier() {
        {
            std::lock_guard<std::mutex> l(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& w : workers_) w.join();
    }
    // Copy every job (each split into one stripe per worker); returns when all are done.
    // Small rounds are copied on the calling thread (the workers start on the first large one).
    void copy(const Job* jobs, int njobs) {
        size_t total = 0;
        for (int j = 0; j < njobs; ++j) total += jobs[j].bytes;
        if (total < kSmallBytes || nthreads_ == 1) {
            for (int j = 0; j < njobs; ++j)
                if (jobs[j].bytes) std::memcpy(jobs[j].dst, jobs[j].src, jobs[j].bytes);
            return;
        }
        if (workers_.empty())
            for (int t = 0; t < nthreads_; ++t) workers_.emplace_back([this, t] { loop(t); });
        std::unique_lock<std::mutex> l(mu_);
        jobs_ = jobs;
        njobs_ = njobs;
        left_ = nthreads_;
        ++gen_;
        cv_.notify_all();
        done_cv_.wait(l, [this] { return left_ == 0; });
    }
    static constexpr size_t kSmallBytes = 256 << 10;
    static int default_threads() {
        const int hw = (int)std::thread::hardware_concurrency();
        // memcpy pinned -> pageable: 14 GB/s on 1 thread, ~54 GB/s (the PCIe rate) on 8 (host_copy_bw.cu);
        // inside the c5 staging pipeline the host copies bound the call: 76 ms on 8 threads, 71 ms on 15
        // (tools/e2e_pageable_time.py, 16-CPU box)
        static const int cap = lb::tuning_env("LOWBIT_COPY_THREADS") ? atoi(lb::tuning_env("LOWBIT_COPY_THREADS")) : 16;
        return hw <= 2 ? 1 : (hw - 1 < cap ? hw - 1 : cap);
    }

  private:
    void loop(int t) {
        unsigned long long seen = 0;
        for (;;) {
            const Job* jobs;
            int nj;
            {
                std::unique_lock<std::mutex> l(mu_);
                cv_.wait(l, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                jobs = jobs_;
                nj = njobs_;
            }
            for (int j = 0; j < nj; ++j) {
                // cache-line stripes covering the whole job (ceil, so no byte is left out)
                const size_t per = ((jobs[j].bytes + nthreads_ - 1) / nthreads_ + 63) & ~size_t(63);
                const size_t a = per * t < jobs[j].bytes ? per * t : jobs[j].bytes;
                const size_t b = a + per < jobs[j].bytes ? a + per : jobs[j].bytes;
                if (b > a)
                    std::memcpy(static_cast<char*>(jobs[j].dst) + a, static_cast<const char*>(jobs[j].src) + a,
                                b - a);
            }
            std::lock_guard<std::mutex> l(mu_);
            if (--left_ == 0) done_cv_.notify_one();
        }
    }
    const int nthreads_;
    std::vector<std::thread> workers_;
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    const Job* jobs_ = nullptr;
    int njobs_ = 0, left_ = 0;
    unsigned long long gen_ = 0;
    bool stop_ = false;
};

// On an error return after copies were queued, wait for them: the caller may
// free its host buffers as soon as the call returns.
struct StreamDrain {
    cudaStream_t s[3];
    bool armed = true;
    ~StreamDrain() {
        if (!armed) return;
        for (cudaStream_t x : s)
            if (x) cudaStreamSynchronize(x);
        cudaGetLastError();
    }
};

// Grow-only device buffer of the device that was current at allocation.
struct DevScratch {
    void* ptr = nullptr;
    size_t bytes = 0;
    cudaError_t ensure(size_t want) {
        if (want <= bytes) return cudaSuccess;
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        bytes = 0;
        want = (want + 0xFFFFF) & ~size_t(0xFFFFF);
        cudaError_t e = cudaMalloc(&ptr, want);
        if (e == cudaSuccess) bytes = want;
        return e;
    }
    void release() {
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        bytes = 0;
    }
};

// Pinned host staging slot (page-locked; for callers that pass pageable memory).
struct PinnedScratch {
    void* ptr = nullptr;
    size_t bytes = 0;
    cudaError_t ensure(size_t want) {
        if (want <= bytes) return cudaSuccess;
        if (ptr) cudaFreeHost(ptr);
        ptr = nullptr;
        bytes = 0;
        cudaError_t e = cudaMallocHost(&ptr, want);
        if (e == cudaSuccess) bytes = want;
        return e;
    }
    void release() {
        if (ptr) cudaFreeHost(ptr);
        ptr = nullptr;
        bytes = 0;
    }
};

struct HostCtx {
    static constexpr int kChunks = 8;   // row chunks of the copy-in / compute / copy-out pipeline
    static constexpr int kBounce = 4;   // pinned staging slots per direction (pageable callers)
    int dev = -1;
    // gemm / encode / pack_b
    DevScratch a0, a1, panels, weights, c, vals, flag;
    // conv2d
    DevScratch fm, ws, out16, out32;
    // conv2d's prepared weights, kept while successive calls pass the same PackedB (a batch of
    // single-image conv2d_lowbit calls, conv.hpp:64-65): conv_w_key holds those panel bytes
    DevScratch conv_w;
    std::vector<uint8_t> conv_w_key;
    int conv_w_ternary = -1, conv_w_cout = 0, conv_w_k = 0;
    PinnedScratch bounce_in[kBounce], bounce_out[kBounce];
    cudaStream_t s_in = nullptr, s_out = nullptr;
    cudaEvent_t ev_in[kChunks] = {}, ev_c[kChunks] = {}, ev_w = nullptr, ev_done = nullptr;
    cudaEvent_t ev_bin[kBounce] = {}, ev_bout[kBounce] = {};

    cudaError_t ensure_streams() {
        if (s_in) return cudaSuccess;
        cudaError_t e;
        if ((e = cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking))) return e;
        if ((e = cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking))) return e;
        for (int i = 0; i < kChunks; ++i) {
            if ((e = cudaEventCreateWithFlags(&ev_in[i], cudaEventDisableTiming))) return e;
            if ((e = cudaEventCreateWithFlags(&ev_c[i], cudaEventDisableTiming))) return e;
        }
        for (int i = 0; i < kBounce; ++i) {
            if ((e = cudaEventCreateWithFlags(&ev_bin[i], cudaEventDisableTiming))) return e;
            if ((e = cudaEventCreateWithFlags(&ev_bout[i], cudaEventDisableTiming))) return e;
        }
        if ((e = cudaEventCreateWithFlags(&ev_w, cudaEventDisableTiming))) return e;
        return cudaEventCreateWithFlags(&ev_done, cudaEventDisableTiming);
    }

    // Give everything back on this context's device.  Errors are ignored: at
    // process exit the runtime may already be unloading.
    void release() {
        if (dev < 0) return;
        int prev = -1;
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
        if (s_in) cudaStreamSynchronize(s_in);
        if (s_out) cudaStreamSynchronize(s_out);
        for (DevScratch* b : {&a0, &a1, &panels, &weights, &c, &vals, &flag, &fm, &ws, &out16, &out32, &conv_w}) b->release();
        conv_w_key.clear();
        conv_w_ternary = -1;
        for (int i = 0; i < kBounce; ++i) {
            bounce_in[i].release();
            bounce_out[i].release();
        }
        auto ev = [](cudaEvent_t& e) {
            if (e) cudaEventDestroy(e);
            e = nullptr;
        };
        for (int i = 0; i < kChunks; ++i) {
            ev(ev_in[i]);
            ev(ev_c[i]);
        }
        for (int i = 0; i < kBounce; ++i) {
            ev(ev_bin[i]);
            ev(ev_bout[i]);
        }
        ev(ev_w);
        ev(ev_done);
        if (s_in) cudaStreamDestroy(s_in);
        if (s_out) cudaStreamDestroy(s_out);
        s_in = s_out = nullptr;
        if (prev >= 0 && prev != dev) cudaSetDevice(prev);
        cudaGetLastError();  // do not leak a teardown error into the caller's next call
    }
    ~HostCtx() { release(); }
};

// This thread's context for the current device (created on first use);
// nullptr if the ordinal is out of range.
HostCtx* host_ctx();

}  // namespace lbhost

// popc_rate.cu — measured POPC throughput per SM per clock on this GPU, the
// denominator of K2's roofline (148 SM x 16 POPC/clk x 32 bit x
// 2 ops x f, assumed from the architecture tables until measured).
//
// One CTA per SM x 8, 512 threads; each thread runs independent chains of
// LOP3 + POPC + IADD (the K2 inner-loop mix: acc += popc(a ^ b)) on register
// data, and the SM clock is read with clock64 around the loop.  Reports
// POPC/clk/SM and the implied BNN / TNN peaks at the measured clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o popc_rate popc_rate.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

constexpr int CHAINS = 8, ITERS = 4096;

__global__ void popc_kernel(uint32_t seed, uint32_t* out, unsigned long long* cycles) {
    uint32_t a[CHAINS], b[CHAINS];
    int acc[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
        a[c] = seed * (threadIdx.x + 1) + c * 0x9E3779B9u;
        b[c] = seed ^ (c * 0x85EBCA6Bu + threadIdx.x);
        acc[c] = 0;
    }
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) {
            acc[c] += __popc(a[c] ^ b[c]);
            a[c] = a[c] * 1664525u + 1013904223u;  // keep the operands changing (IMAD: another pipe)
        }
    }
    const long long t1 = clock64();
    uint32_t s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += (uint32_t)acc[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) atomicMax(cycles, (unsigned long long)(t1 - t0));
}

int main() {
    int dev = 0, sms = 0, clk_khz = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    const int blocks = sms * 4, threads = 512;
    uint32_t* out;
    unsigned long long* cyc;
    cudaMalloc(&out, (size_t)blocks * threads * 4);
    cudaMalloc(&cyc, 8);
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(cyc, 0, 8);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        popc_kernel<<<blocks, threads>>>(12345u + rep, out, cyc);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long c = 0;
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        const double popcs = (double)blocks * threads * CHAINS * ITERS;
        // wall rate (events) at the nominal 1.965 GHz, and the per-CTA clock64 view
        const double per_sm_clk_wall = popcs / (ms * 1e-3) / sms / 1.965e9;
        const double per_sm_clk_cyc = popcs / sms / (double)c;
        std::printf("POPC per clk per SM: %.2f from the kernel time at 1.965 GHz (%.3f ms), %.2f from clock64 "
                    "(%llu cycles per CTA); BNN peak = %.1f TOPS, TNN = %.1f (wall rate x 64 / 32 ops)\n",
                    per_sm_clk_wall, ms, per_sm_clk_cyc, c, popcs / (ms * 1e-3) * 64 / 1e12,
                    popcs / (ms * 1e-3) * 32 / 1e12);
    }
    return 0;
}

// Issue rate of tcgen05.mma.cta_group::1.kind::mxf4 (M = 128, N = 128 / 256, K = 64) with the A operand in
// tensor memory or in shared memory — K7T's MMA shape in isolation.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma1_rate mma1_rate.cu
#include <cstdio>
#include <cstdint>
#include "../../paper_2205_09120_b200/csrc/common.cuh"
#include "../../paper_2205_09120_b200/csrc/halo_common.cuh"
using namespace lb;

__device__ inline void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t sf, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%5], [%5], p;\n\t}"
                 ::"r"(d), "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc), "r"(sf) : "memory");
}
__device__ inline void mma_ss(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t sf, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%5], p;\n\t}"
                 ::"r"(d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc), "r"(sf) : "memory");
}

__global__ void __launch_bounds__(128, 1) rate_kernel(int n, int a_in_tmem, int iters, unsigned long long* cyc, int nissue) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tslot;
    __shared__ uint64_t bar;
    __shared__ uint64_t bars4[4];
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 48 * 1024 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0x2A2A2A2Au;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); for (int i = 0; i < 4; ++i) mbar_init(&bars4[i], 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc<512>(&tslot);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = tslot;
    if (warp < 4) {
        tmem_st_32x32b_x8_fill(tb + ((uint32_t)(warp * 32) << 16) + 504, 0x7F7F7F7Fu);
        tmem_st_32x32b_x8_fill(tb + ((uint32_t)(warp * 32) << 16) + 400, 0x22222222u);
        tmem_st_wait();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (nissue > 1) {  // nissue warps issue concurrently, each into its own 128-column accumulator
        if ((threadIdx.x & 31) == 0 && warp < nissue) {
            const uint32_t idesc = idesc_mxf4(128, 128);
            const uint64_t bd = h7_desc_sw64(smem_u32(smem + 16384));
            const long long t0 = clock64();
            for (int i = 0; i < iters / nissue; ++i)
                mma_ts(tb + warp * 128, tb + 400, bd + (uint32_t)((i % 9) * 4), idesc, tb + 504, i != 0);
            umma_commit(&bars4[warp]);
            mbar_wait(&bars4[warp], 0);
            if (warp == 0) cyc[blockIdx.x] = clock64() - t0;
        }
    } else if (threadIdx.x == 0) {
        const uint32_t idesc = idesc_mxf4(128, (uint32_t)n);
        const uint64_t ad = h7_desc_sw64(smem_u32(smem)), bd = h7_desc_sw64(smem_u32(smem + 16384));
        const long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const uint64_t b = bd + (uint32_t)((i % 9) * 4);  // row-shifted B, as the taps
            if (a_in_tmem) mma_ts(tb, tb + 400, b, idesc, tb + 504, i != 0);
            else mma_ss(tb, ad, b, idesc, tb + 504, i != 0);
        }
        umma_commit(&bar);
        mbar_wait(&bar, 0);
        cyc[blockIdx.x] = clock64() - t0;
    }
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tb);
}

int main() {
    unsigned long long* cyc;
    cudaMalloc(&cyc, 148 * 8);
    cudaFuncSetAttribute(rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    const int iters = 4000;
    for (int n : {128, 256})
        for (int ts : {1, 0}) {
            rate_kernel<<<148, 128, 64 * 1024>>>(n, ts, iters, cyc, 1);
            cudaError_t e = cudaDeviceSynchronize();
            unsigned long long h[148];
            cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
            printf("cta_group::1 mxf4 M=128 N=%d K=64, A in %s: %.1f cycles per MMA (%s)\n", n, ts ? "TMEM" : "smem",
                   (double)h[0] / iters, cudaGetErrorString(e));
        }
    for (int k : {2, 3}) {
        rate_kernel<<<148, 128, 64 * 1024>>>(128, 1, iters, cyc, k);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h[148];
        cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
        printf("%d warps issuing M=128 N=128 TMEM-A MMAs concurrently: %.1f cycles per MMA overall (%s)\n", k,
               (double)h[0] / iters, cudaGetErrorString(e));
    }
    return 0;
}

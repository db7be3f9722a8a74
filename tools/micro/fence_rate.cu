// Microbenchmark: what slows back-to-back tcgen05.mma (pair, kind::mxf4, A in
// TMEM, N = 208) issue: per-granule fences, barrier waits, commits.  One
// kernel instantiation per variant so the variants do not share code.
#include <cstdio>
#include <cstdint>
#include "../../paper_2205_09120_b200/csrc/common.cuh"
using namespace lb;

__device__ inline void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t sf) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                 "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%4], [%4], p;\n\t}"
                 ::"r"(d), "r"(a), "l"(b), "r"(id), "r"(sf) : "memory");
}

__device__ inline bool test_acq(uint64_t* bar, uint32_t par) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(par) : "memory");
    return ok;
}
__device__ inline bool try_rlx(uint64_t* bar, uint32_t par) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.relaxed.cta.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(par) : "memory");
    return ok;
}
__device__ inline bool test_rlx(uint64_t* bar, uint32_t par) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.relaxed.cta.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(par) : "memory");
    return ok;
}
__device__ inline bool ld_phase(uint64_t* bar, uint32_t par) {  // raw read of the barrier word
    uint64_t v;
    asm volatile("ld.volatile.shared.b64 %0, [%1];" : "=l"(v) : "r"(smem_u32(bar)) : "memory");
    return ((uint32_t)(v >> 63) & 1u) != par;
}

template <int V>  // 0 plain; 1 fence::after every 2; 2 try_wait(done) every 2; 3 both; 4 commit every 2;
                  // 5 commit + wait + fence every 2 (the kernel's pattern); 6 fence::before every 2
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k(int iters, unsigned long long* cyc) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tslot;
    __shared__ uint64_t bar, done;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 16384 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0x2A2A0A02u * (i | 1);
    if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&done, 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc_pair<512>(&tslot);
    fence_proxy_async_smem();
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tb = tslot;
    tmem_st_32x32b_x8_fill(tb + ((uint32_t)(warp * 32) << 16) + 416, 0x7F7F7F7Fu);
    tmem_st_wait();
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (cluster_ctarank() == 0 && threadIdx.x == 0) {
        mbar_arrive(&done);  // phase 0 of `done` completes: waits on it return at once
        const uint32_t id = idesc_mxf4(256, 208);
        const uint32_t b = smem_u32(smem);
        const long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const uint32_t acol = 432 + 16 * ((i >> 1) % 5) + (i & 1) * 8, dcol = ((i >> 5) & 1) * 208;
            mma_ts(tb + dcol, tb + acol, umma_desc_k_sw128(b + (i & 3) * 32), id, tb + 416);
            if (i & 1) {
                if (V == 4 || V == 5) umma_commit_pair(&bar, 0x3);
                if (V == 2 || V == 3 || V == 5) mbar_wait(&done, 0);
                if (V == 1 || V == 3 || V == 5) tc_fence_after();
                if (V == 6) tc_fence_before();
                if (V == 7) while (!test_acq(&done, 0)) {}
                if (V == 8) while (!try_rlx(&done, 0)) {}
                if (V == 9) while (!test_rlx(&done, 0)) {}
                if (V == 10) { volatile uint64_t* p = &done; (void)*p; }
            }
        }
        umma_commit_pair(&done, 0x3);
        mbar_wait(&done, 1);
        cyc[V] = clock64() - t0;
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 0) { tc_fence_after(); tmem_dealloc_pair<512>(tb); }
}

template <int V>
void run(unsigned long long* d) {
    cudaFuncSetAttribute(k<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    k<V><<<2, 128, 32768>>>(100000, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[16]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("variant %d: %s %.1f cycles/MMA\n", V, cudaGetErrorString(e), (double)h[V] / 100000);
}

int main() {
    unsigned long long* d; cudaMalloc(&d, 128); cudaMemset(d, 0, 128);
    run<0>(d); run<2>(d); run<5>(d); run<7>(d); run<8>(d); run<9>(d); run<10>(d);
    return 0;
}

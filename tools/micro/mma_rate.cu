// Microbenchmark: back-to-back tcgen05.mma issue rate (operands are whatever
// is in shared memory / TMEM; results discarded).  One persistent CTA (or CTA
// pair) per SM, one thread issues ITERS MMAs, commit + wait at the end.
// Reports cycles per MMA and the implied TOPS at the measured clock.
#include <cstdio>
#include <cstdint>
#include "../../paper_2205_09120_b200/csrc/common.cuh"
using namespace lb;

template <int KIND, int PAIR>  // KIND 0 = i8 (K=32), 1 = mxf4 (K=64)
__global__ void __launch_bounds__(128, 1) rate_kernel(int n, int iters, unsigned long long* out, int fill, int opts) {
    extern __shared__ __align__(1024) uint8_t smem[];
    // operands: zeros (fill 0) or random {-1, 0, +1} codes (fill 1)
    for (int i = threadIdx.x; i < 4 * 32768 / 4; i += blockDim.x) {
        uint32_t h = (uint32_t)(i * 2654435761u) ^ (blockIdx.x * 0x9E3779B9u);
        h ^= h >> 15; h *= 0x2C1B3C6Du; h ^= h >> 12; h *= 0x297A2D39u; h ^= h >> 15;
        uint32_t w = 0;
        for (int j = 0; j < 8; ++j) {
            const uint32_t r = (h >> (4 * j)) & 3;
            const uint32_t code = KIND ? (r == 1 ? 0x2u : r == 2 ? 0xAu : 0u) : 0u;
            w |= code << (4 * j);
        }
        if (!KIND) w = ((h & 0x03030303u) == 0 ? 0 : (h & 0x01010101u) * 0xFFu) ^ (h & 0x01010101u);
        reinterpret_cast<uint32_t*>(smem)[i] = fill ? w : 0u;
    }
    __syncthreads();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __shared__ uint32_t tslot;
    __shared__ uint64_t bar, bar2;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&bar2, 1); fence_barrier_init(); }
    if (warp == 0) { if (PAIR) tmem_alloc_pair<512>(&tslot); else tmem_alloc<512>(&tslot); }
    tc_fence_before();
    if (PAIR) cluster_sync(); else __syncthreads();
    tc_fence_after();
    const uint32_t tb = tslot;
    // zero scales region: fill cols 448.. with 0x7F
    {
        const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
        for (uint32_t c = 448; c < 512; c += 16) tmem_st_32x32b_x16_fill(tb + lane_base + c, 0x7F7F7F7Fu);
        tmem_st_wait();
    }
    tc_fence_before();
    if (PAIR) cluster_sync(); else __syncthreads();
    tc_fence_after();
    const bool leader = !PAIR || cluster_ctarank() == 0;
    long long t0 = 0, t1 = 0;
    if (leader && threadIdx.x == 0) {
        const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
        const uint32_t M = PAIR ? 256 : 128;
        const uint32_t id = KIND ? idesc_mxf4(M, n) : idesc_i8(M, n);
        t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            // opts 1: cycle over 4 stages of (16 KB A, 16 KB B); opts 2: commit every 4 MMAs
            const uint32_t stage = (opts & 1) ? ((i >> 2) & 3) * 32768u : 0u;
            const uint64_t ad = umma_desc_k_sw128((opts & 1) ? smem_u32(smem) + stage + (i & 3) * 32 : a + (i & 3) * 32);
            const uint64_t bd = umma_desc_k_sw128((opts & 1) ? smem_u32(smem) + stage + 16384 + (i & 3) * 32 : b + (i & 3) * 32);
            if ((opts & 2) && (i & 3) == 0 && i) { if (PAIR) umma_commit_pair(&bar2, 0x3); else umma_commit(&bar2); }
            if (KIND == 1) {
                if (PAIR) umma_mxf4_pair(tb, ad, bd, id, tb + 448, tb + 448, 1);
                else asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                  "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}"
                                  ::"r"(tb), "l"(ad), "l"(bd), "r"(id), "r"(1), "r"(tb + 448), "r"(tb + 448) : "memory");
            } else {
                if (PAIR) umma_i8_pair(tb, ad, bd, id, 1);
                else umma_i8(tb, ad, bd, id, 1);
            }
        }
        if (PAIR) umma_commit_pair(&bar, 0x1); else umma_commit(&bar);
        mbar_wait(&bar, 0);
        t1 = clock64();
        out[blockIdx.x] = (unsigned long long)(t1 - t0);
    }
    tc_fence_before();
    if (PAIR) cluster_sync(); else __syncthreads();
    if (warp == 0) { tc_fence_after(); if (PAIR) tmem_dealloc_pair<512>(tb); else tmem_dealloc<512>(tb); }
}

template <int KIND, int PAIR>
void run(int n, int iters, int fill, int opts = 0) {
    auto k = rate_kernel<KIND, PAIR>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    unsigned long long* d; cudaMalloc(&d, 148 * 8); cudaMemset(d, 0, 148 * 8);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = 148; cfg.blockDim = 128; cfg.dynamicSmemBytes = 131072;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = PAIR ? 2 : 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaLaunchKernelEx(&cfg, k, n, iters / 10, d, fill, opts);  // warm
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, k, n, iters, d, fill, opts);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[148]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    unsigned long long mx = 0; int cnt = 0;
    for (int i = 0; i < 148; ++i) if (h[i]) { mx = h[i] > mx ? h[i] : mx; ++cnt; }
    const double M = PAIR ? 256 : 128, K = KIND ? 64 : 32;
    const double ops = 2.0 * M * n * K * iters * (PAIR ? 74 : 148);
    printf("opts=%d %s %s %s N=%d: %s %.1f cycles/MMA (issuers %d), %.3f ms -> %.0f TOPS, clock %.2f GHz\n",
           opts, fill ? "random" : "zeros ", KIND ? "mxf4" : "i8  ", PAIR ? "pair" : "1cta", n, cudaGetErrorString(err), (double)mx / iters, cnt, ms,
           ops / (ms * 1e-3) / 1e12, (double)mx / (ms * 1e-3) / 1e9);
    cudaFree(d);
}


// The conv's operand shapes (K7): N = cout = 128, 64-byte-swizzled A/B rows
// (SW64) vs 128-byte (SW128), one accumulator chain vs two interleaved.  All
// descriptors precomputed; 4 MMAs per unrolled step so the issuing thread
// never limits the rate.
template <int SW64, int TWO_ACC, int BG = 0, int LDCOL = 256>
__global__ void __launch_bounds__(384, 1) conv_rate_kernel(int n, int iters, unsigned long long* out,
                                                           uint4* gbuf) {
    extern __shared__ __align__(1024) uint8_t smem[];
    for (int i = threadIdx.x; i < 4 * 32768 / 4; i += blockDim.x) {
        uint32_t h = (uint32_t)(i * 2654435761u) ^ (blockIdx.x * 0x9E3779B9u);
        h ^= h >> 15; h *= 0x2C1B3C6Du; h ^= h >> 12; h *= 0x297A2D39u; h ^= h >> 15;
        uint32_t w = 0;
        for (int j = 0; j < 8; ++j) {
            const uint32_t r = (h >> (4 * j)) & 3;
            w |= (r == 1 ? 0x2u : r == 2 ? 0xAu : 0u) << (4 * j);
        }
        reinterpret_cast<uint32_t*>(smem)[i] = w;
    }
    __syncthreads();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __shared__ uint32_t tslot;
    __shared__ uint64_t bar;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc_pair<512>(&tslot);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tb = tslot;
    {
        const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
        for (uint32_t c = 448; c < 512; c += 16) tmem_st_32x32b_x16_fill(tb + lane_base + c, 0x7F7F7F7Fu);
        tmem_st_wait();
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    __shared__ volatile int done;
    if (threadIdx.x == 0) done = 0;
    __syncthreads();
    if (BG == 7) {  // background TMA (bulk) writes into shared memory: warp 4 lane 0, 4 x 8 KB copies in flight
        if (warp == 4 && (threadIdx.x & 31) == 0) {
            __shared__ uint64_t tbar[4];
            for (int q = 0; q < 4; ++q) mbar_init(&tbar[q], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            const uint32_t dst0 = smem_u32(smem + 98304);
            uint32_t n[4] = {0, 0, 0, 0};  // copies issued per slot; copy k of a slot completes phase k
            for (int it = 0; !done; ++it) {
                const int q = it & 3;
                if (n[q]) mbar_wait(&tbar[q], (n[q] - 1) & 1);
                mbar_arrive_expect_tx(&tbar[q], 8192);
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                                 "r"(dst0 + q * 8192), "l"(reinterpret_cast<const uint8_t*>(gbuf) + (size_t)((blockIdx.x * 64 + (it & 63)) & 8191) * 8192),
                             "r"(8192), "r"(smem_u32(&tbar[q])) : "memory");
                ++n[q];
            }
            for (int q = 0; q < 4; ++q)
                if (n[q]) mbar_wait(&tbar[q], (n[q] - 1) & 1);
        }
    } else if (BG && warp >= 4) {  // background traffic from 8 warps while the MMAs run
        const uint32_t base = smem_u32(smem + 98304) + (warp - 4) * 2048 + (threadIdx.x & 31) * 16;
        uint4 acc = make_uint4(0, 0, 0, 0);
        uint4* g = gbuf + ((size_t)blockIdx.x * 8 + (warp - 4)) * 32 * 64 + (threadIdx.x & 31) * 2;
        for (int it = 0; !done; ++it) {
            if (BG == 1) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const uint4 v = lds_v4(base + (q & 3) * 512);
                    acc.x ^= v.x; acc.y += v.y;
                    sts_v4(base + 4096 * 4 + (q & 3) * 512, acc.x, acc.y, v.z, v.w);
                }
            } else if (BG == 3) {  // TMEM loads of another accumulator region (columns 256..383)
                uint32_t v[16];
                const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    tmem_ld_32x32b_x16(tb + lane_base + (uint32_t)LDCOL + ((it * 4 + q) & 7) * 16, v);
                    tmem_ld_wait();
                    acc.x ^= v[0] + v[15];
                }
            } else if (BG == 4 || BG == 5) {  // shared stores + proxy fence (4), or the fence alone (5)
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (BG == 4) sts_v4(base + 4096 * 4 + (q & 3) * 512, acc.x, acc.y, (uint32_t)it, (uint32_t)q);
                    fence_proxy_async_smem();
                }
                acc.x += 1;
            } else if (BG == 6) {  // tcgen05.fence::before_thread_sync / after, as the epilogue's handshakes
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    tc_fence_before();
                    __syncwarp();
                    tc_fence_after();
                }
                acc.x += 1;
            } else if (BG == 2) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    uint32_t w8[8] = {acc.x, acc.y, acc.z, acc.w, (uint32_t)it, (uint32_t)q, 0u, 1u};
                    stg_v8(g + (size_t)((it * 8 + q) & 63) * 64, w8);
                }
            }
        }
        if (acc.x == 0x12345) gbuf[0] = acc;
    }
    if (cluster_ctarank() == 0 && threadIdx.x == 0) {
        const uint32_t a = smem_u32(smem), b = smem_u32(smem + 65536);
        const uint32_t id = idesc_mxf4(256, n);
        uint64_t ad[4], bd[4];
        for (int q = 0; q < 4; ++q) {
            if (SW64) {  // K offset 0 / 32 bytes in 64-byte rows; A rows shifted by q (the halo taps)
                const uint32_t ao = a + (q & 1) * 32 + q * 64, bo = b + (q & 1) * 32;
                ad[q] = (uint64_t)((ao >> 4) & 0x3FFFu) | (1ull << 16) | ((uint64_t)(512u >> 4) << 32) | (1ull << 46) | (4ull << 61);
                bd[q] = (uint64_t)((bo >> 4) & 0x3FFFu) | (1ull << 16) | ((uint64_t)(512u >> 4) << 32) | (1ull << 46) | (4ull << 61);
            } else {
                ad[q] = umma_desc_k_sw128(a + q * 32);
                bd[q] = umma_desc_k_sw128(b + q * 32);
            }
        }
        const long long t0 = clock64();
        for (int i = 0; i < iters; i += 4) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
                umma_mxf4_pair(tb + (TWO_ACC == 1 ? (uint32_t)(q & 1) * 224u : TWO_ACC == 2 ? 160u : TWO_ACC == 3 ? 320u : 0u),
                               ad[q], bd[q], id, tb + 480, tb + 480, 1);
        }
        umma_commit_pair(&bar, 0x1);
        mbar_wait(&bar, 0);
        out[blockIdx.x] = (unsigned long long)(clock64() - t0);
    }
    if (threadIdx.x == 0) {
        // the MMA thread of the leader finished (the peer CTA's background warps stop when ours do)
        if (cluster_ctarank() == 0) done = 1;
    }
    if (cluster_ctarank() != 0 && threadIdx.x == 0) {
        // stop after roughly the leader's time: spin on the clock
        const long long t0 = clock64();
        while (clock64() - t0 < (long long)iters * 70) {}
        done = 1;
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 0) { tc_fence_after(); tmem_dealloc_pair<512>(tb); }
}

template <int SW64, int TWO_ACC, int BG = 0, int LDCOL = 256>
void conv_run(int n, int iters) {
    auto k = conv_rate_kernel<SW64, TWO_ACC, BG, LDCOL>;
    static uint4* gbuf = nullptr;
    if (!gbuf) cudaMalloc(&gbuf, (size_t)8192 * 8192 + 4096);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    unsigned long long* d; cudaMalloc(&d, 148 * 8); cudaMemset(d, 0, 148 * 8);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = 148; cfg.blockDim = 384; cfg.dynamicSmemBytes = 131072 + 32768;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072 + 32768);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, n, iters / 10, d, gbuf);
    cudaLaunchKernelEx(&cfg, k, n, iters, d, gbuf);
    cudaError_t err = cudaDeviceSynchronize();
    unsigned long long h[148]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    unsigned long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("conv shape (ld col %d): mxf4 pair N=%d %s %s, background %s: %s %.1f cycles/MMA\n", LDCOL, n, SW64 ? "SW64 (rows shifted)" : "SW128",
           TWO_ACC == 1 ? "two accumulators" : TWO_ACC == 2 ? "accumulator at column 160" : TWO_ACC == 3 ? "accumulator at column 320" : "one accumulator", BG == 0 ? "none" : BG == 1 ? "LDS.128+STS.128 x8 warps" : BG == 2 ? "STG.256 x8 warps" : BG == 3 ? "tcgen05.ld x8 warps" : BG == 4 ? "STS + fence.proxy.async x8 warps" : BG == 5 ? "fence.proxy.async x8 warps" : BG == 7 ? "bulk TMA writes 4 x 8 KB in flight" : "tcgen05 fences x8 warps",
           cudaGetErrorString(err), (double)mx / iters);
    cudaFree(d);
}

// The conv kernel's MMA-side pipeline without its data: tiles of 18 MMAs
// (the first with accumulate = 0) on a ring of NACC accumulators, one commit
// per tile, NISS issuing warps on alternate tiles, each waiting for the
// commit of the tile NACC back before reusing its accumulator.
template <int NISS, int NACC, int XWAIT = 0, int XCOMMIT = 0>
__global__ void __launch_bounds__(128, 1) conv_pipe_kernel(int tiles, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    for (int i = threadIdx.x; i < 4 * 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x22A022A0u ^ (i * 0x01010101u & 0x08080808u);
    __syncthreads();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __shared__ uint32_t tslot;
    __shared__ uint64_t full[4], xbar, xc[4];
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int a = 0; a < 4; ++a) { mbar_init(&full[a], 1); mbar_init(&xc[a], 1); }
        mbar_init(&xbar, 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) mbar_arrive(&xbar);
    if (warp == 0) tmem_alloc_pair<512>(&tslot);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tb = tslot;
    {
        const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
        tmem_st_32x32b_x8_fill(tb + lane_base + 480, 0x7F7F7F7Fu);
        tmem_st_wait();
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (cluster_ctarank() == 0 && warp < NISS && (threadIdx.x & 31) == 0) {
        const uint32_t a = smem_u32(smem), b = smem_u32(smem + 65536);
        const uint32_t id = idesc_mxf4(256, 128);
        auto desc = [](uint32_t o) {
            return (uint64_t)((o >> 4) & 0x3FFFu) | (1ull << 16) | ((uint64_t)(512u >> 4) << 32) | (1ull << 46) | (4ull << 61);
        };
        const uint64_t ad0 = desc(a), bd0 = desc(b);
        const long long t0 = clock64();
        for (int t = warp; t < tiles; t += NISS) {
            const int acc = t % NACC;
            if (t >= NACC) mbar_wait(&full[acc], ((t / NACC) - 1) & 1);
            if (XWAIT) mbar_wait_poll(&xbar, 0);  // a second (already complete) barrier per tile, as K7's a_full
            tc_fence_after();
            const uint32_t d = tb + (uint32_t)acc * 160u;
#pragma unroll
            for (int kb = 0; kb < 9; ++kb) {
                const uint64_t ad = ad0 + (uint32_t)((kb / 3) * 256 + (kb % 3) * 4), bd = bd0 + (uint32_t)kb * 256;
                umma_mxf4_pair(d, ad, bd, id, tb + 480, tb + 480, kb != 0);
                umma_mxf4_pair(d, ad + 2, bd + 2, id, tb + 480, tb + 480, 1);
            }
            if (XCOMMIT) umma_commit_pair(&xc[acc], 0x3);  // K7 also commits the A stage to both CTAs
            umma_commit_pair(&full[acc], 0x1);
        }
        // drain: wait for this issuer's last tile
        int last = warp;
        while (last + NISS < tiles) last += NISS;
        mbar_wait(&full[last % NACC], (last / NACC) & 1);
        out[blockIdx.x * 2 + warp] = (unsigned long long)(clock64() - t0);
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 0) { tc_fence_after(); tmem_dealloc_pair<512>(tb); }
}

template <int NISS, int NACC, int XWAIT = 0, int XCOMMIT = 0>
void pipe_run(int tiles) {
    auto k = conv_pipe_kernel<NISS, NACC, XWAIT, XCOMMIT>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    unsigned long long* d; cudaMalloc(&d, 148 * 16); cudaMemset(d, 0, 148 * 16);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = 148; cfg.blockDim = 128; cfg.dynamicSmemBytes = 131072;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, tiles, d);
    cudaError_t err = cudaDeviceSynchronize();
    unsigned long long h[296]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    unsigned long long mx = 0;
    for (int i = 0; i < 296; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("conv pipe: %d issuer(s), %d accumulators, extra wait %d, extra commit %d, %d tiles of 18 MMAs: %s %.1f cycles per tile (%.1f per MMA)\n", NISS, NACC,
           XWAIT, XCOMMIT, tiles, cudaGetErrorString(err), (double)mx / tiles, (double)mx / tiles / 18);
    cudaFree(d);
}

// K5's issue pattern: stages of 8 pair MMAs (N = 256, one accumulator chain),
// an mbarrier wait (already complete) + a commit per stage; NISS issuing
// warps take alternate stages, handing over through a shared-memory turn
// counter so the chain stays in order.
template <int NISS>
__global__ void __launch_bounds__(128, 1) k5_pipe_kernel(int stages, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    for (int i = threadIdx.x; i < 4 * 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x22A022A0u ^ (i * 0x01010101u & 0x08080808u);
    __syncthreads();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __shared__ uint32_t tslot;
    __shared__ uint64_t ready, done;
    __shared__ volatile uint32_t turn;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) { mbar_init(&ready, 1); mbar_init(&done, 1); turn = 0; fence_barrier_init(); }
    __syncthreads();
    if (threadIdx.x == 0) mbar_arrive(&ready);  // phase 0 complete: every wait below succeeds at once
    if (warp == 0) tmem_alloc_pair<512>(&tslot);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tb = tslot;
    {
        const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
        tmem_st_32x32b_x8_fill(tb + lane_base + 256 + 248, 0x7F7F7F7Fu);
        tmem_st_wait();
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (cluster_ctarank() == 0 && warp < NISS && (threadIdx.x & 31) == 0) {
        const uint32_t a = smem_u32(smem), b = smem_u32(smem + 65536);
        const uint32_t id = idesc_mxf4(256, 256);
        const long long t0 = clock64();
        for (int st = warp; st < stages; st += NISS) {
            mbar_wait(&ready, 0);
            tc_fence_after();
            if (NISS > 1)
                while (turn != (uint32_t)st) {
                }
#pragma unroll
            for (int j = 0; j < 8; ++j)
                umma_mxf4_pair(tb, umma_desc_k_sw128(a + (j & 3) * 32 + (j >> 2) * 16384),
                               umma_desc_k_sw128(b + (j & 3) * 32 + (j >> 2) * 16384), id, tb + 504, tb + 504, st | j);
            umma_commit_pair(&done, 0x1);
            if (NISS > 1) turn = (uint32_t)st + 1;
        }
        if (warp == 0) {
            while (turn != (uint32_t)stages && NISS > 1) {
            }
            umma_commit_pair(&ready, 0x1);  // (one more phase on a barrier nobody waits on afterwards)
        }
        out[blockIdx.x * 2 + warp] = (unsigned long long)(clock64() - t0);
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 0) { tc_fence_after(); tmem_dealloc_pair<512>(tb); }
}

template <int NISS>
void k5_pipe_run(int stages) {
    auto k = k5_pipe_kernel<NISS>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    unsigned long long* d; cudaMalloc(&d, 148 * 16); cudaMemset(d, 0, 148 * 16);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = 148; cfg.blockDim = 128; cfg.dynamicSmemBytes = 131072;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, stages, d);
    cudaError_t err = cudaDeviceSynchronize();
    unsigned long long h[296]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    unsigned long long mx = 0;
    for (int i = 0; i < 296; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("K5 pattern: %d issuer(s), %d stages of 8 N=256 MMAs, a wait + commit per stage: %s %.1f cycles per MMA\n",
           NISS, stages, cudaGetErrorString(err), (double)mx / stages / 8);
    cudaFree(d);
}

// K5's streaming issue loop verbatim in shape: per k-block a tcgen05 fence,
// lane 0 issues 4 N = 256 MMAs over a 4-stage ring of A / B slots (SW128)
// and VARIANT commits, then the warp re-converges.
//   VARIANT 0: one commit (local)       1: two commits multicast to both CTAs
//   2: two multicast commits, whole-warp loop (no lane-0 branch for the MMAs)
template <int VARIANT>
__global__ void __launch_bounds__(128, 1) k5_loop_kernel(int kblocks, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    for (int i = threadIdx.x; i < 4 * 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x22A022A0u ^ (i * 0x01010101u & 0x08080808u);
    __syncthreads();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __shared__ uint32_t tslot;
    __shared__ uint64_t e1[4], e2[4], done;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) { for (int q = 0; q < 4; ++q) { mbar_init(&e1[q], 1); mbar_init(&e2[q], 1); } mbar_init(&done, 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc_pair<512>(&tslot);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tb = tslot;
    {
        const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
        tmem_st_32x32b_x8_fill(tb + lane_base + 256 + 248, 0x7F7F7F7Fu);
        tmem_st_wait();
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (cluster_ctarank() == 0 && warp == 0) {
        const uint32_t base = smem_u32(smem);
        const uint32_t id = idesc_mxf4(256, 256);
        const long long t0 = clock64();
        for (int kb = 0; kb < kblocks; ++kb) {
            const uint32_t sa = kb & 3;
            tc_fence_after();
            if (VARIANT == 2 || lane == 0) {
                const uint32_t a_addr = base + sa * 16384, b_addr = base + 65536 + sa * 16384;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    umma_mxf4_pair(tb, umma_desc_k_sw128(a_addr + kk * 32), umma_desc_k_sw128(b_addr + kk * 32), id,
                                   tb + 504, tb + 504, (kb | kk) != 0);
                if (VARIANT == 0) {
                    umma_commit_pair(&e1[sa], 0x1);
                } else {
                    umma_commit_pair(&e1[sa], 0x3);
                    umma_commit_pair(&e2[sa], 0x3);
                }
            }
            __syncwarp();
        }
        if (lane == 0) {
            umma_commit_pair(&done, 0x1);
            mbar_wait(&done, 0);
            out[blockIdx.x] = (unsigned long long)(clock64() - t0);
        }
        __syncwarp();
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 0) { tc_fence_after(); tmem_dealloc_pair<512>(tb); }
}

template <int VARIANT>
void k5_loop_run(int kblocks) {
    auto k = k5_loop_kernel<VARIANT>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    unsigned long long* d; cudaMalloc(&d, 148 * 8); cudaMemset(d, 0, 148 * 8);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = 148; cfg.blockDim = 128; cfg.dynamicSmemBytes = 131072;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, kblocks, d);
    cudaError_t err = cudaDeviceSynchronize();
    unsigned long long h[148]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    unsigned long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("K5 loop variant %d (%s): %s %.1f cycles per MMA\n", VARIANT,
           VARIANT == 0 ? "1 local commit per k-block" : VARIANT == 1 ? "2 multicast commits per k-block" : "2 multicast commits, whole warp issues",
           cudaGetErrorString(err), (double)mx / kblocks / 4);
    cudaFree(d);
}

int main(int argc, char** argv) {
    if (argc > 1 && argv[1][0] == 'l') {
        k5_loop_run<0>(50000); k5_loop_run<1>(50000);
        return 0;
    }
    if (argc > 1 && argv[1][0] == 'k') {
        k5_pipe_run<1>(4000); k5_pipe_run<2>(4000);
        return 0;
    }
    if (argc > 2) {
        pipe_run<2, 3>(2000); pipe_run<2, 3, 1>(2000); pipe_run<2, 3, 0, 1>(2000); pipe_run<2, 3, 1, 1>(2000);
        return 0;
    }
    if (argc > 1) {
        conv_run<1, 0, 0>(128, 200000); conv_run<1, 0, 1>(128, 200000); conv_run<1, 0, 2>(128, 200000);
        conv_run<1, 0, 3>(128, 200000);
        conv_run<1, 0, 7>(128, 200000);
        return 0;
    }
    const int it = 200000;
    for (int opts : {0, 1, 2, 3}) run<1, 1>(256, it, 1, opts);
    for (int opts : {0, 3}) run<1, 1>(208, it, 1, opts);
    return 0;
}

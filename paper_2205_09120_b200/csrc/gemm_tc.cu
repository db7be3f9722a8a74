// gemm_tc.cu — K3: the low-bit GeMM on the 5th-generation tensor cores.
//
// {-1,0,+1} operands are an exact dense int8 contraction: tcgen05.mma
// kind::i8 with int32 accumulators in TMEM (exact, |C| <= K <= 32767), then
// narrowed to int16 — bit-identical to gemm_lowbit (gemm.cpp:79-112).
//
// Operands
//   A  stays in the reference bit-plane layout in HBM (1 plane binary, 2
//      planes ternary; 1/8 or 1/4 byte per element).  TMA brings 128-row x
//      16-byte raw tiles into shared memory; converter warps expand bits to
//      int8 straight into the UMMA operand tile (K-major, 128-byte swizzle).
//   B  the prepared int8 K-major weights (layout.cuh), TMA 128-byte swizzle.
//
// Warp roles (448 threads, 1 CTA per SM, persistent over output tiles):
//   warp 0       TMA producer (raw A bits + int8 B per 128-deep k-block)
//   warp 1       TMEM allocator + single-thread UMMA issuer
//   warps 2-9    converters: half an A row each, bits -> int8, swizzled STS
//   warps 10-13  epilogue: TMEM -> registers -> int16 -> global
// Pipelines: STAGES-deep smem ring (tma_full / a_ready / empty), and a
// double-buffered TMEM accumulator (2 x 256 columns; tmem_full / tmem_empty)
// so the epilogue of tile t overlaps the MMAs of tile t+1.
#include "common.cuh"
#include "expand.cuh"
#include "layout.cuh"
#include "tmap.cuh"

namespace lb {

constexpr int TC_BM = 128;         // UMMA M (rows of A per tile)
constexpr int TC_BK = 128;         // depth per k-block (bytes of int8 = one 128B swizzle row)
constexpr int TC_MAX_BN = 256;     // UMMA N max
constexpr int TC_STAGES = 4;
constexpr int TC_THREADS = 448;  // 2 control + 8 converter + 4 epilogue warps
constexpr int TC_A_BYTES = TC_BM * TC_BK;           // 16 KB
constexpr int TC_B_BYTES = TC_MAX_BN * TC_BK;       // 32 KB
constexpr int TC_RAW_BYTES = TC_BM * 16;            // one plane, 128 rows x 16 B
constexpr int TC_SMEM_BYTES = 1024 /*align slack*/ + TC_STAGES * (TC_A_BYTES + TC_B_BYTES + 2 * TC_RAW_BYTES) + 256;

struct TcParams {
    int m, n, kblocks, bn, m_tiles, n_tiles;
    long long ldc;
    int16_t* c;
};

template <bool A_TER, int LAYOUT>
__global__ void __launch_bounds__(TC_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmap_b, const __grid_constant__ CUtensorMap tmap_a0,
                   const __grid_constant__ CUtensorMap tmap_a1, const TcParams prm) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;                                         // STAGES x 16 KB
    uint8_t* sB = sA + TC_STAGES * TC_A_BYTES;                  // STAGES x 32 KB
    uint8_t* sRaw = sB + TC_STAGES * TC_B_BYTES;                // STAGES x 2 planes x 2 KB
    uint64_t* bars = reinterpret_cast<uint64_t*>(sRaw + TC_STAGES * 2 * TC_RAW_BYTES);
    uint64_t* tma_full = bars;
    uint64_t* a_ready = bars + TC_STAGES;
    uint64_t* empty = bars + 2 * TC_STAGES;
    uint64_t* tmem_full = bars + 3 * TC_STAGES;
    uint64_t* tmem_empty = tmem_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int num_tiles = prm.m_tiles * prm.n_tiles;
    const uint32_t bn = (uint32_t)prm.bn;

    if (threadIdx.x == 0) {
        for (int s = 0; s < TC_STAGES; ++s) {
            mbar_init(&tma_full[s], 1);
            mbar_init(&a_ready[s], 8);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tmem_full[a], 1);
            mbar_init(&tmem_empty[a], 128);
        }
        fence_barrier_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmap_b);
        tma_prefetch_desc(&tmap_a0);
        if (A_TER) tma_prefetch_desc(&tmap_a1);
    }
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // Programmatic dependent launch: the next kernel in the stream may begin launching now (its CTAs
    // run their setup while this grid works, then block in their own griddepcontrol.wait until this
    // grid has completed); this grid touches global memory only after its wait.  Launch-bound shapes
    // (config 1) are mostly launch latency and setup.
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");

    if (warp == 0) {
        // ===================== TMA producer =====================
        if (lane == 0) {
            const uint32_t tx_bytes = bn * TC_BK + (A_TER ? 2 : 1) * TC_RAW_BYTES;
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                const int mt = tile / prm.n_tiles, nt = tile - mt * prm.n_tiles;
                for (int kb = 0; kb < prm.kblocks; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_arrive_expect_tx(&tma_full[stage], tx_bytes);
                    tma_load_2d(sB + stage * TC_B_BYTES, &tmap_b, &tma_full[stage], kb * TC_BK, nt * (int)bn);
                    uint8_t* raw = sRaw + stage * 2 * TC_RAW_BYTES;
                    tma_load_2d(raw, &tmap_a0, &tma_full[stage], kb * 16, mt * TC_BM);
                    if (A_TER) tma_load_2d(raw + TC_RAW_BYTES, &tmap_a1, &tma_full[stage], kb * 16, mt * TC_BM);
                    if (++stage == TC_STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== UMMA issuer =====================
        const uint32_t idesc = idesc_i8(TC_BM, bn);
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + (uint32_t)acc * TC_MAX_BN;
            for (int kb = 0; kb < prm.kblocks; ++kb) {
                mbar_wait(&a_ready[stage], phase);
                mbar_wait(&tma_full[stage], phase);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t a_addr = smem_u32(sA + stage * TC_A_BYTES);
                    const uint32_t b_addr = smem_u32(sB + stage * TC_B_BYTES);
#pragma unroll
                    for (int kk = 0; kk < TC_BK / 32; ++kk) {
                        umma_i8(d_tmem, umma_desc_k_sw128(a_addr + kk * 32), umma_desc_k_sw128(b_addr + kk * 32),
                                idesc, (kb | kk) != 0);
                    }
                    umma_commit(&empty[stage]);
                }
                __syncwarp();
                if (++stage == TC_STAGES) { stage = 0; phase ^= 1; }
            }
            if (lane == 0) umma_commit(&tmem_full[acc]);
            __syncwarp();
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
    } else if (warp < 10) {
        // ===================== converters =====================
        const int ct = threadIdx.x - 64;
        const int r = ct & 127, h = ct >> 7;  // A row within the tile, half of its 16 raw bytes
        const uint32_t sA_u = smem_u32(sA), sRaw_u = smem_u32(sRaw);
        int stage = 0;
        uint32_t phase = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            for (int kb = 0; kb < prm.kblocks; ++kb) {
                mbar_wait(&tma_full[stage], phase);
                const uint32_t raw = sRaw_u + stage * 2 * TC_RAW_BYTES;
                expand_half_layout<A_TER, LAYOUT>(raw, raw + TC_RAW_BYTES, sA_u + stage * TC_A_BYTES, r, h);
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&a_ready[stage]);
                if (++stage == TC_STAGES) { stage = 0; phase ^= 1; }
            }
        }
    } else {
        // ===================== epilogue =====================
        const int lane_base = (warp & 3) * 32;  // TMEM lane quarter this warp may access
        const int r = lane_base + lane;
        int acc = 0;
        uint32_t acc_phase = 0;
        const bool vec_ok = ((prm.ldc & 7) == 0) && ((reinterpret_cast<uintptr_t>(prm.c) & 15) == 0);
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            const int mt = tile / prm.n_tiles, nt = tile - mt * prm.n_tiles;
            mbar_wait(&tmem_full[acc], acc_phase);
            tc_fence_after();
            const int row = mt * TC_BM + r;
            int16_t* crow = prm.c + (long long)row * prm.ldc;
            for (int ch = 0; ch < prm.bn / 32; ++ch) {
                uint32_t v[32];
                tmem_ld_32x32b_x32(tmem_base + ((uint32_t)lane_base << 16) + (uint32_t)acc * TC_MAX_BN + ch * 32, v);
                tmem_ld_wait();
                const int col0 = nt * prm.bn + ch * 32;
                if (row < prm.m) {
                    if (vec_ok && col0 + 32 <= prm.n) {
                        uint32_t pk[16];
#pragma unroll
                        for (int j = 0; j < 16; ++j) pk[j] = __byte_perm(v[2 * j], v[2 * j + 1], 0x5410);
                        uint4* dst = reinterpret_cast<uint4*>(crow + col0);
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            dst[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (col0 + j < prm.n) crow[col0 + j] = (int16_t)(int32_t)v[j];
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(&tmem_empty[acc]);
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
    }

    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<512>(tmem_base);
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
// Tile width along N: one UMMA of N = bn (multiple of 32, <= 256).
static int pick_bn(int n) {
    if (n >= 256) return 256;
    return (n + 31) / 32 * 32;
}

template <bool A_TER, int LAYOUT>
static lowbit_status launch_tc_variant(const CUtensorMap& mb, const CUtensorMap& ma0, const CUtensorMap& ma1,
                                       const TcParams& prm, int grid, cudaStream_t stream) {
    static SmemOptIn attr;
    LB_CUDA_TRY(attr.ensure(gemm_tc_kernel<A_TER, LAYOUT>, TC_SMEM_BYTES));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(TC_THREADS);
    cfg.dynamicSmemBytes = TC_SMEM_BYTES;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    LB_CUDA_TRY(cudaLaunchKernelEx(&cfg, gemm_tc_kernel<A_TER, LAYOUT>, mb, ma0, ma1, prm));
    LB_CUDA_TRY(cudaGetLastError());
    return LOWBIT_OK;
}

lowbit_status launch_tensor(int a_ternary, int layout, const uint8_t* a0, const uint8_t* a1, long long a_pitch, int m, int n,
                            int k, const void* weights, int b_ternary, int16_t* c, long long ldc,
                            cudaStream_t stream) {
    const WeightsLayout L(b_ternary, n, k);
    TcParams prm;
    prm.m = m;
    prm.n = n;
    prm.kblocks = L.kp / TC_BK;
    prm.bn = pick_bn(n);
    prm.m_tiles = (m + TC_BM - 1) / TC_BM;
    prm.n_tiles = (n + prm.bn - 1) / prm.bn;
    prm.ldc = ldc;
    prm.c = c;

    CUtensorMap mb, ma0, ma1;
    if (!make_map_2d(&mb, weights, (uint64_t)L.kp, (uint64_t)L.np, (uint64_t)L.kp, TC_BK, (uint32_t)prm.bn,
                     CU_TENSOR_MAP_SWIZZLE_128B))
        return lbhost::set_error(LOWBIT_CUDA_ERROR, "cuTensorMapEncodeTiled failed for B");
    if (!make_map_2d(&ma0, a0, (uint64_t)a_pitch, (uint64_t)m, (uint64_t)a_pitch, 16, TC_BM,
                     CU_TENSOR_MAP_SWIZZLE_NONE))
        return lbhost::set_error(LOWBIT_CUDA_ERROR, "cuTensorMapEncodeTiled failed for A");
    if (a_ternary) {
        if (!make_map_2d(&ma1, a1, (uint64_t)a_pitch, (uint64_t)m, (uint64_t)a_pitch, 16, TC_BM,
                         CU_TENSOR_MAP_SWIZZLE_NONE))
            return lbhost::set_error(LOWBIT_CUDA_ERROR, "cuTensorMapEncodeTiled failed for A minus");
    } else {
        ma1 = ma0;
    }

    const int tiles = prm.m_tiles * prm.n_tiles;
    const int grid = tiles < num_sms() ? tiles : num_sms();
    if (a_ternary)
        return layout ? launch_tc_variant<true, 1>(mb, ma0, ma1, prm, grid, stream)
                      : launch_tc_variant<true, 0>(mb, ma0, ma1, prm, grid, stream);
    return layout ? launch_tc_variant<false, 1>(mb, ma0, ma1, prm, grid, stream)
                  : launch_tc_variant<false, 0>(mb, ma0, ma1, prm, grid, stream);
}

}  // namespace lb

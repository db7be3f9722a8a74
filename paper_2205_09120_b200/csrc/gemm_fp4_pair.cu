// gemm_fp4_pair.cu — K5: the bit-plane GeMM on the fp4 tensor cores.
//
// Same contract as K3 (gemm_tc_pair.cu) — ternary/binary A bit planes times
// prepared weights, int16 out, bit-identical to gemm_lowbit (gemm.cpp:79-112)
// — but the operands reach the tensor cores as packed e2m1 (4 bits/element)
// through tcgen05.mma.cta_group::2.kind::mxf4.block_scale with every UE8M0
// block scale = 1.0:
//
//   * {-1, 0, +1} are exact e2m1 codes (0xA, 0x0, 0x2); every partial sum is
//     an integer of magnitude <= k <= 32767 < 2^24, so the f32 accumulator is
//     exact and the epilogue's round-to-nearest is the identity.
//   * an fp4 MMA does twice the int8 MMA's work per cycle on half the operand
//     bytes, and A arrives in the NIBBLES plane layout (lowbit_encode_ex,
//     layout 2: element j of a word at bit 4*(j%8) + j/8), so building a word
//     of 8 packed e2m1 values costs one shift + mask per plane and an IMAD:
//         ternary: ((M >> q) & 0x11111111) * 10 + ((P >> (q-1)) & 0x22222222)
//         binary:  ((S >> q) & 0x11111111) * 8 + 0x22222222
//     about 0.6 integer ops per element against 1.25 for the int8 lanes path.
//
// Tiling: a CTA pair computes 256 x BN (BN <= 224, multiple of 16; two f32
// accumulators of BN columns + the scale-factor columns fit the 512 TMEM
// columns), k-block = 256 depth positions = 128 bytes per row (one SW128
// atom row).  Warp roles as K3: 0-7 converters (two groups of 4, alternate
// k-blocks, one A row per thread), 8-11 epilogue, 12 raw-plane TMA producer,
// 13 B TMA producer, 14 TMEM allocation + UMMA issue (leader CTA).
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "layout.cuh"
#include "tmap.cuh"

namespace lb {

constexpr int F4_BM = 128;           // A rows per CTA (256 per pair)
constexpr int F4_BK = 256;           // depth per k-block (128 bytes of packed e2m1)
constexpr int F4_MAX_BN = 256;       // pair UMMA N (f32 accumulator columns per buffer)
#ifndef LOWBIT_F4_A_STAGES
#define LOWBIT_F4_A_STAGES 4
#endif
#ifndef LOWBIT_F4_B_STAGES
#define LOWBIT_F4_B_STAGES 4
#endif
#ifndef LOWBIT_F4_RAW_KB
#define LOWBIT_F4_RAW_KB 64
#endif
// A (converter output) and B (TMA) rings.  Equal depths share one release
// barrier (one commit per k-block); a sweep of (A, B) depths in
// {(2..5) x (3..6)} on config 5 put (4, 4) first, ahead of deeper B rings.
constexpr int F4_A_ST = LOWBIT_F4_A_STAGES, F4_B_ST = LOWBIT_F4_B_STAGES;
constexpr bool F4_SHARED_RING = F4_A_ST == F4_B_ST;
constexpr int F4_THREADS = 480;
constexpr int F4_W_RAW = 12, F4_W_B = 13, F4_W_MMA = 14;
constexpr int F4_A_BYTES = F4_BM * 128;       // 16 KB
constexpr int F4_B_BYTES = (F4_MAX_BN / 2) * 128;  // 16 KB slot (this CTA's <= 128 rows of B)
constexpr int F4_RAW_PLANE = F4_BM * 32;      // 4 KB: 128 rows x 256 bits
// Raw bit-plane ring: 64 KB = 8 ternary (two-plane) or 16 binary k-blocks.
// When a CTA's whole depth fits (k <= 2048 ternary / 4096 binary), the ring
// holds its A rows for all the column tiles of an m-tile: the planes cross
// L2 -> SM once per m-tile instead of once per (m, n) tile.
constexpr int F4_RAW_RING = LOWBIT_F4_RAW_KB * 1024;
__host__ __device__ constexpr int f4_raw_stages(bool ter) { return LOWBIT_F4_RAW_KB / (ter ? 8 : 4); }
constexpr int F4_EPI_BYTES = 32 * 32;         // 32 rows x 16 int16, per warp per buffer
// TMA-store staging: 16 buffers of 1 KB per CTA — 4 epilogue warps x 4 (streaming
// variant) or 8 epilogue warps x 2 (AR: its converters need one group of 4 warps
// only, so the other 4 drain the accumulators; the epilogue is its critical path).
constexpr int F4_EPI_TOTAL = 16;
// Scale factors.  An fp4 MMA costs the same for any N <= 256 (measured), so
// tiles are 256 wide, and two f32 accumulators fill all 512 TMEM columns.
// The unit scales (SFA and SFB share one 8-column block of 0x7F bytes) live
// in the LAST 8 columns of the accumulator NOT being written: tile i
// (buffer b) reads them from buffer 1-b's tail, which the epilogue of tile
// i-1 drains first and then overwrites with scales (sf_ready[1-b]).
constexpr uint32_t F4_SF_OFF = 248;
// A-resident variant (AR): when k <= 2048 (<= 8 k-blocks) the converted fp4
// A of a whole m tile (128 rows x 1 KB per CTA) stays in shared memory for
// all n tiles of that m tile: the converters run once per m tile instead of
// once per (m, n) tile, and the raw planes only stream through a 16 KB ring.
constexpr int F4_AR_SLOTS = 8;
#ifndef LOWBIT_F4_AR_RAW_KB
#define LOWBIT_F4_AR_RAW_KB 16
#endif
constexpr int F4_AR_RAW = LOWBIT_F4_AR_RAW_KB * 1024;
// AR tile width / B ring / staging (tuning knobs)
#ifndef LOWBIT_F4_AR_BN
#define LOWBIT_F4_AR_BN 256
#endif
#ifndef LOWBIT_F4_AR_B_SLOTS
#define LOWBIT_F4_AR_B_SLOTS 4
#endif
#ifndef LOWBIT_F4_AR_EGRP
#define LOWBIT_F4_AR_EGRP 2
#endif
constexpr int F4_AR_BN = LOWBIT_F4_AR_BN, F4_AR_B_SLOTS = LOWBIT_F4_AR_B_SLOTS, F4_AR_EGRP = LOWBIT_F4_AR_EGRP;
constexpr int F4_AR_B_BYTES = (F4_AR_BN / 2) * 128;
static_assert(F4_AR_B_BYTES % 1024 == 0 && F4_AR_B_SLOTS % 2 == 0, "AR B slots");
static_assert(F4_AR_EGRP == 2, "the epilogue stores 32-column boxes: groups of two 16-column chunks");
// staging: 8 epilogue warps x F4_AR_EGRP (AR) or 4 warps x 2 buffers of 1 KB
__host__ __device__ constexpr int f4_epi_bytes(bool ar) { return (ar ? 8 * F4_AR_EGRP : 8) * F4_EPI_BYTES; }
__host__ __device__ constexpr int f4_smem_bytes(bool ar) {
    return 1024 + (ar ? F4_AR_SLOTS : F4_A_ST) * F4_A_BYTES +
           (ar ? F4_AR_B_SLOTS * F4_AR_B_BYTES : F4_B_ST * F4_B_BYTES) + (ar ? F4_AR_RAW : F4_RAW_RING) +
           f4_epi_bytes(ar) + 1024;
}
static_assert(f4_smem_bytes(false) <= 227 * 1024 && f4_smem_bytes(true) <= 227 * 1024,
              "fp4 pair kernel exceeds shared memory");

struct Fp4Params {
    int m, n, kblocks, bn, m_tiles, n_tiles;
    int m_off;  // first m tile of this launch (a split launch runs the rest elsewhere)
    long long ldc;
    int16_t* c;
    int tma_store;
    int m_major;   // schedule: 1 = each pair owns whole m tiles (all n tiles back to back)
    int resident;  // raw A planes stay in the ring across the n tiles of an m tile (m_major only)
    int a_res;     // AR variant (launch selects the template; recorded for the host only)
    int debug;  // LOWBIT_DEBUG_FP4 timing experiments (results invalid unless only 8 is set): 1 converters
                // skip the expansion, 2 no MMAs, 4 no epilogue, 8 role timers (valid), 16 MMA issue without
                // waits, 64 half the B loads, 128 no TMA stores, 256 no TMEM loads, 512 no staging stores,
                // 8192 B loads without the evict_last hint
};

// Role timing for profiling experiments (LOWBIT_DEBUG_FP4 bit 3): cycle
// counters summed over CTAs, read by lowbit_debug_fp4_stats.
__device__ unsigned long long g_fp4_stats[16];
// Timing experiments and role timers exist only in -DLOWBIT_TUNING builds: in the product
// kernel F4_DBG is the constant 0 and the timers are empty, so their branches, clock reads and
// hoisted constants are compiled out (as in K7, conv_fp4_halo.cu).
#ifdef LOWBIT_TUNING
#define F4_DBG(bits) (prm.debug & (bits))
#define F4_T0() const long long _t0 = (prm.debug & 8) ? clock64() : 0
#define F4_ACC(var) \
    if (prm.debug & 8) var += clock64() - _t0
#else
#define F4_DBG(bits) 0
#define F4_T0() \
    do {        \
    } while (0)
#define F4_ACC(var) (void)(var)
#endif

// One 16-byte chunk (32 elements = one plane word per plane) of packed e2m1:
// output word q takes bit 4i+q of the plane word into nibble i — one shift +
// mask per plane and an IMAD, ~4.5 integer ops per 8 elements.  For NIBBLES
// planes (element j at bit 4*(j%8) + j/8) that is element 8q+i, the canonical
// order of the fp4 B section; for REFERENCE planes (element j at bit j) it is
// element 4i+q, the order of the reference-order B section (layout.cuh), so
// both layouts cost the same here.
template <bool A_TER>
__device__ __forceinline__ void fp4_chunk(uint32_t p, uint32_t m, uint32_t dst) {
    uint32_t o[4];
    if (A_TER) {
        o[0] = (m & 0x11111111u) * 10u + ((p << 1) & 0x22222222u);
        o[1] = ((m >> 1) & 0x11111111u) * 10u + (p & 0x22222222u);
        o[2] = ((m >> 2) & 0x11111111u) * 10u + ((p >> 1) & 0x22222222u);
        o[3] = ((m >> 3) & 0x11111111u) * 10u + ((p >> 2) & 0x22222222u);
    } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) o[q] = ((p >> q) & 0x11111111u) * 8u + 0x22222222u;
    }
    sts_v4(dst, o[0], o[1], o[2], o[3]);
}

// CL = 4 (AR only): two CTA pairs per cluster run different m tiles over the same
// n tiles in lockstep and share B: each CTA loads one k-block half of a B stage
// and multicasts it to the same-position CTA of the other pair, halving B's
// L2 -> SM traffic.
template <bool A_TER, bool AR, int CL>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(F4_THREADS, 1)
    gemm_fp4_pair_kernel(const __grid_constant__ CUtensorMap tmap_b, const __grid_constant__ CUtensorMap tmap_a0,
                         const __grid_constant__ CUtensorMap tmap_a1, const __grid_constant__ CUtensorMap tmap_c,
                         const Fp4Params prm) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    constexpr int A_SLOTS = AR ? F4_AR_SLOTS : F4_A_ST;
    constexpr int CONV_W = AR ? 4 : 8, EPI_W = 12 - CONV_W;  // warps 0..CONV_W-1 convert, the rest to 11 drain
    // staging buffers (= chunks per group) per epilogue warp: 2 (4 measured equal and spills registers)
    constexpr int EGRP = AR ? F4_AR_EGRP : 2;
    constexpr int B_SLOTS = AR ? F4_AR_B_SLOTS : F4_B_ST, B_BYTES = AR ? F4_AR_B_BYTES : F4_B_BYTES;
    constexpr bool SHARED = !AR && F4_SHARED_RING;  // one release barrier for the A and B slots
    uint8_t* sB = sA + A_SLOTS * F4_A_BYTES;
    uint8_t* sRaw = sB + B_SLOTS * B_BYTES;
    uint8_t* sEpi = sRaw + (AR ? F4_AR_RAW : F4_RAW_RING);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sEpi + f4_epi_bytes(AR));
    constexpr uint32_t RAW_SLOT = A_TER ? 2 * F4_RAW_PLANE : F4_RAW_PLANE;
    constexpr uint32_t RS = AR ? F4_AR_RAW / RAW_SLOT : f4_raw_stages(A_TER);
    static_assert(RS <= 16 && A_SLOTS <= 8 && B_SLOTS <= 8, "barrier table sizes");
    uint64_t* raw_full = bars;                       // local: raw planes landed            [raw]
    uint64_t* raw_empty = bars + 16;                 // local: 4 converter warps read them  [raw]
    uint64_t* b_full = bars + 32;                    // leader: both halves of B landed     [b]
    uint64_t* a_ready = bars + 40;                   // leader: 8 converter warps done      [a]
    uint64_t* a_empty = bars + 48;                   // local: pair MMAs done with A slot   [a]
    uint64_t* b_empty = bars + 56;                   // local: pair MMAs done with B slot   [b]
    uint64_t* tmem_full = bars + 64;                 // local: accumulator ready (2)
    uint64_t* tmem_empty = bars + 66;                // leader: 8 epilogue warps drained (2)
    uint64_t* sf_ready = bars + 68;                  // leader: scales in buffer c's tail (8 warps) (2)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 70);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    static_assert(CL == 2 || (CL == 4 && AR), "4-CTA clusters for the A-resident variant only");
    const uint32_t crank = cluster_ctarank();
    const uint32_t rank = crank & 1;            // position in the CTA pair
    const uint32_t pbase = crank & ~1u;         // cluster rank of this pair's leader
    const bool leader = rank == 0;
    const uint16_t pair_mask = (uint16_t)(0x3u << pbase);
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const int clu = blockIdx.x >> 2, nclu = gridDim.x >> 2, pc = (blockIdx.x >> 1) & 1;  // CL = 4
    // Schedule.  m_major: pair p owns m tiles p, p + npairs, ... and runs every
    // n tile of one m tile back to back (so its A rows can stay resident);
    // otherwise (fewer m tiles than pairs) tiles are dealt round-robin.
    const int num_tiles = prm.m_tiles * prm.n_tiles;
    const int m_pairs = (prm.m_tiles + 1) / 2;  // CL = 4: cluster c owns m-tile pairs c, c + nclu, ...
    const int my_tiles =
        CL == 4 ? (m_pairs > clu ? (m_pairs - clu + nclu - 1) / nclu : 0) * prm.n_tiles
        : prm.m_major ? (prm.m_tiles > pair ? (prm.m_tiles - pair + npairs - 1) / npairs : 0) * prm.n_tiles
                      : (num_tiles > pair ? (num_tiles - pair + npairs - 1) / npairs : 0);
    auto tile_of = [&](int i, int& mt, int& nt) {
        if (CL == 4) {  // m tile 2q + pc may be past the end (rows >= m: zero A, clipped stores)
            mt = 2 * (clu + (i / prm.n_tiles) * nclu) + pc;
            nt = i % prm.n_tiles;
        } else if (prm.m_major) {
            mt = pair + (i / prm.n_tiles) * npairs;
            nt = i % prm.n_tiles;
        } else {
            const int tile = pair + i * npairs;
            mt = tile / prm.n_tiles;
            nt = tile - mt * prm.n_tiles;
        }
        mt += prm.m_off;
    };
    const int bn = prm.bn, bnh = prm.bn >> 1;
    // streaming variant: the 4-slot shared ring runs as 2 stages of 2 k-blocks when the
    // tile's k-block count is even (one barrier wait per 8 MMAs on the issuing thread)
    const bool g2 = !AR && SHARED && F4_A_ST == 4 && (prm.kblocks % 2 == 0);

    if (threadIdx.x == 0) {
        for (int s = 0; s < (int)RS; ++s) {
            mbar_init(&raw_full[s], 1);
            mbar_init(&raw_empty[s], 4);
        }
        for (int s = 0; s < B_SLOTS; ++s) {
            mbar_init(&b_full[s], 1);
            mbar_init(&b_empty[s], CL == 4 ? 2 : 1);  // CL = 4: released by both pairs' MMAs
        }
        for (int s = 0; s < A_SLOTS; ++s) {
            mbar_init(&a_ready[s], (AR || g2) ? 16 : 8);  // one barrier per pair of k-blocks
            mbar_init(&a_empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tmem_full[a], 1);
            mbar_init(&tmem_empty[a], 2 * EPI_W);
        }
        mbar_init(&sf_ready[0], 8);
        mbar_init(&sf_ready[1], 8);
        fence_barrier_init();
    }
    if (warp == F4_W_RAW && lane == 0) {
        tma_prefetch_desc(&tmap_b);
        tma_prefetch_desc(&tmap_a0);
        if (A_TER) tma_prefetch_desc(&tmap_a1);
        if (prm.tma_store) tma_prefetch_desc(&tmap_c);
    }
    if (warp == F4_W_MMA) tmem_alloc_pair<512>(tmem_slot);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // programmatic dependent launch: the next kernel in the stream may begin launching (and run its
    // setup) now; this grid touches global memory only after its own wait
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");

    if (warp == F4_W_RAW) {
        // ===================== raw A-plane producer (both CTAs) =====================
        if (lane == 0) {
            uint32_t u = 0;  // raw loads issued
            for (int i = 0; i < my_tiles; ++i) {
                int mt, nt;
                tile_of(i, mt, nt);
                if (prm.resident && nt != 0) continue;
                const int arow = mt * 2 * F4_BM + (int)rank * F4_BM;
                for (int kb = 0; kb < prm.kblocks; ++kb, ++u) {
                    const uint32_t rs = u % RS;
                    mbar_wait_sleep(&raw_empty[rs], ((u / RS) & 1) ^ 1);
                    uint8_t* raw = sRaw + rs * RAW_SLOT;
                    mbar_arrive_expect_tx(&raw_full[rs], RAW_SLOT);
                    // (marking these streamed planes evict_first measured 10% slower on config 5)
                    tma_load_2d(raw, &tmap_a0, &raw_full[rs], kb * 32, arow);
                    if (A_TER) tma_load_2d(raw + F4_RAW_PLANE, &tmap_a1, &raw_full[rs], kb * 32, arow);
                }
            }
        }
    } else if (warp == F4_W_B) {
        // ===================== B producer (both CTAs; bytes land on the leader) =====================
        if (lane == 0) {
            const uint32_t pair_bytes = (uint32_t)bn * 128;
            const uint32_t b_full0 = mapa_shared(smem_u32(&b_full[0]), pbase);
            // B (the weights) is re-read by every pair for every m tile while A and C stream
            // through L2 once: keep it resident (evict_last; +3% on config 5)
            const uint64_t b_policy = l2_policy_evict_last();
            uint32_t t = 0;
            for (int i = 0; AR && i < my_tiles; ++i) {
                // AR: stages of two k-blocks (one barrier per 8 MMAs: an mbarrier wait on
                // the issuing thread stalls the MMA stream ~270 cycles)
                int mt, nt;
                tile_of(i, mt, nt);
                const int brow = nt * bn + (int)rank * bnh;
                for (int kb = 0; kb < prm.kblocks; kb += 2, ++t) {
                    const uint32_t st = t % (B_SLOTS / 2);
                    mbar_wait_sleep(&b_empty[st], ((t / (B_SLOTS / 2)) & 1) ^ 1);
                    if (leader) mbar_arrive_expect_tx(&b_full[st], 2 * pair_bytes);
                    if (CL == 4) {  // k-block pc of the stage, this CTA's half, to both pairs
                        tma_load_2d_pair_mc(smem_u32(sB + (2 * st + pc) * B_BYTES), &tmap_b,
                                            smem_u32(&b_full[st]) & 0xFEFFFFFFu, (kb + pc) * 128, brow,
                                            (uint16_t)((1u << rank) | (1u << (rank + 2))));
                        continue;
                    }
                    for (int j = 0; j < 2; ++j) {
                        if (!F4_DBG(8192))
                            tma_load_2d_pair_hint(smem_u32(sB + (2 * st + j) * B_BYTES), &tmap_b, b_full0 + st * 8,
                                                  (kb + j) * 128, brow, b_policy);
                        else
                            tma_load_2d_pair(smem_u32(sB + (2 * st + j) * B_BYTES), &tmap_b, b_full0 + st * 8,
                                             (kb + j) * 128, brow);
                    }
                }
            }
            for (int i = 0; g2 && i < my_tiles; ++i) {
                int mt, nt;
                tile_of(i, mt, nt);
                const int brow = nt * bn + (int)rank * bnh;
                for (int kb = 0; kb < prm.kblocks; kb += 2, t += 2) {
                    const uint32_t st = (t >> 1) & 1;
                    mbar_wait_sleep(&a_empty[st], ((t >> 2) & 1) ^ 1);
                    if (leader) mbar_arrive_expect_tx(&b_full[st], 2 * pair_bytes);
                    for (int j = 0; j < 2; ++j)
                        tma_load_2d_pair_hint(smem_u32(sB + (2 * st + j) * F4_B_BYTES), &tmap_b, b_full0 + st * 8,
                                              (kb + j) * 128, brow, b_policy);
                }
            }
            for (int i = 0; !AR && !g2 && i < my_tiles; ++i) {
                int mt, nt;
                tile_of(i, mt, nt);
                const int brow = nt * bn + (int)rank * bnh;
                for (int kb = 0; kb < prm.kblocks; ++kb, ++t) {
                    const uint32_t st = t % F4_B_ST;
                    mbar_wait_sleep(SHARED ? &a_empty[st] : &b_empty[st], ((t / F4_B_ST) & 1) ^ 1);
                    if (F4_DBG(64) && (i & 1)) {  // timing experiment: half the B traffic (results invalid)
                        if (leader) mbar_arrive(&b_full[st]);
                        continue;
                    }
                    if (leader) mbar_arrive_expect_tx(&b_full[st], pair_bytes);
                    tma_load_2d_pair_hint(smem_u32(sB + st * F4_B_BYTES), &tmap_b, b_full0 + st * 8, kb * 128, brow,
                                          b_policy);
                }
            }
        }
    } else if (warp == F4_W_MMA) {
        // ===================== UMMA issuer (leader CTA only) =====================
        if (leader) {
            const uint32_t idesc = idesc_mxf4(2 * F4_BM, (uint32_t)bn);
            uint32_t t = 0;
            int acc = 0;
            uint32_t acc_phase = 0, sf_phase = 0;  // sf_phase bit c: parity of the next wait on sf_ready[c]
            long long w_a = 0, w_b = 0, w_t = 0, w_s = 0;
            const long long t_start = clock64();
            for (int i = 0; i < my_tiles; ++i) {
                int mt_, nt_;
                tile_of(i, mt_, nt_);
                const uint32_t mgen = (uint32_t)(i / prm.n_tiles);  // AR: this pair's m-tile generation
                const bool first_nt = nt_ == 0, last_nt = nt_ == prm.n_tiles - 1;
                {
                    F4_T0();
                    mbar_wait_sleep(&tmem_empty[acc], acc_phase ^ 1);
                    F4_ACC(w_t);
                }
                {
                    F4_T0();
                    mbar_wait(&sf_ready[acc ^ 1], (sf_phase >> (acc ^ 1)) & 1);
                    F4_ACC(w_s);
                }
                sf_phase ^= 1u << (acc ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + (uint32_t)acc * F4_MAX_BN;
                const uint32_t sf = tmem_base + (uint32_t)(acc ^ 1) * F4_MAX_BN + F4_SF_OFF;
                for (int kb = 0; AR && kb < prm.kblocks; kb += 2, t += 2) {
                    const uint32_t t2 = t >> 1, st = t2 % (B_SLOTS / 2);
                    if (first_nt) {  // later n tiles reuse the converted A
                        F4_T0();
                        mbar_wait(&a_ready[kb >> 1], mgen & 1);
                        F4_ACC(w_a);
                    }
                    {
                        F4_T0();
                        mbar_wait(&b_full[st], (t2 / (B_SLOTS / 2)) & 1);
                        F4_ACC(w_b);
                    }
                    tc_fence_after();
                    if (lane == 0) {
#pragma unroll
                        for (int j = 0; j < 2; ++j) {
                            const uint32_t a_addr = smem_u32(sA + (kb + j) * F4_A_BYTES);
                            const uint32_t b_addr = smem_u32(sB + (2 * st + j) * B_BYTES);
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk)
                                umma_mxf4_pair(d_tmem, umma_desc_k_sw128(a_addr + kk * 32),
                                               umma_desc_k_sw128(b_addr + kk * 32), idesc, sf, sf,
                                               (kb | j | kk) != 0);
                        }
                        // CL = 4: both pairs' CTAs hold copies of this B stage (multicast)
                        umma_commit_pair(&b_empty[st], CL == 4 ? (uint16_t)0xF : pair_mask);
                        if (last_nt) umma_commit_pair(&a_empty[kb >> 1], pair_mask);
                    }
                    __syncwarp();
                }
                for (int kb = 0; g2 && kb < prm.kblocks; kb += 2, t += 2) {
                    const uint32_t st = (t >> 1) & 1, ph = (t >> 2) & 1;
                    {
                        F4_T0();
                        mbar_wait(&a_ready[st], ph);
                        F4_ACC(w_a);
                    }
                    {
                        F4_T0();
                        mbar_wait(&b_full[st], ph);
                        F4_ACC(w_b);
                    }
                    tc_fence_after();
                    if (lane == 0) {
#pragma unroll
                        for (int j = 0; j < 2; ++j) {
                            const uint32_t a_addr = smem_u32(sA + (2 * st + j) * F4_A_BYTES);
                            const uint32_t b_addr = smem_u32(sB + (2 * st + j) * F4_B_BYTES);
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk)
                                umma_mxf4_pair(d_tmem, umma_desc_k_sw128(a_addr + kk * 32),
                                               umma_desc_k_sw128(b_addr + kk * 32), idesc, sf, sf,
                                               (kb | j | kk) != 0);
                        }
                        umma_commit_pair(&a_empty[st], pair_mask);  // releases both slots of the stage (A and B)
                    }
                    __syncwarp();
                }
                for (int kb = 0; !AR && !g2 && kb < prm.kblocks; ++kb, ++t) {
                    const uint32_t sa = t % F4_A_ST, sb = t % F4_B_ST;
                    if (!F4_DBG(16) || t < (uint32_t)F4_B_ST) {  // debug 16: MMA issue rate (no waits)
                        {
                            F4_T0();
                            mbar_wait(&a_ready[sa], (t / F4_A_ST) & 1);
                            F4_ACC(w_a);
                        }
                        {
                            F4_T0();
                            mbar_wait(&b_full[sb], (t / F4_B_ST) & 1);
                            F4_ACC(w_b);
                        }
                    }
                    tc_fence_after();
                    if (lane == 0) {
                        const uint32_t a_addr = smem_u32(sA + sa * F4_A_BYTES);
                        const uint32_t b_addr = smem_u32(sB + sb * F4_B_BYTES);
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)  // K = 64 per MMA = 32 bytes
                            if (!F4_DBG(2))
                            umma_mxf4_pair(d_tmem, umma_desc_k_sw128(a_addr + kk * 32),
                                           umma_desc_k_sw128(b_addr + kk * 32), idesc, sf, sf, (kb | kk) != 0);
                        umma_commit_pair(&a_empty[sa], pair_mask);
                        if (!SHARED) umma_commit_pair(&b_empty[sb], pair_mask);
                    }
                    __syncwarp();
                }
                if (lane == 0) umma_commit_pair(&tmem_full[acc], pair_mask);
                __syncwarp();
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            }
            if (F4_DBG(8) && lane == 0) {
                atomicAdd(&g_fp4_stats[0], (unsigned long long)w_a);
                atomicAdd(&g_fp4_stats[1], (unsigned long long)w_b);
                atomicAdd(&g_fp4_stats[2], (unsigned long long)w_t);
                atomicAdd(&g_fp4_stats[3], (unsigned long long)(clock64() - t_start));
                atomicAdd(&g_fp4_stats[11], (unsigned long long)w_s);
                atomicAdd(&g_fp4_stats[12], (unsigned long long)t);
            }
        }
    } else if (warp < CONV_W) {
        // ===================== converters (both CTAs) =====================
        const int g = warp >> 2;
        const int r = threadIdx.x & 127;
        const uint32_t sA_u = smem_u32(sA), sRaw_u = smem_u32(sRaw);
        const uint32_t a_ready0 = mapa_shared(smem_u32(&a_ready[0]), pbase);
        const uint32_t kbs = (uint32_t)prm.kblocks, nts = (uint32_t)prm.n_tiles;
        const uint32_t total = (uint32_t)my_tiles * kbs;
        const uint32_t rsw = (uint32_t)(r >> 2) & 1;  // TMA SWIZZLE_32B on the raw rows
        long long w_raw = 0, w_slot = 0, w_work = 0;
        const long long t_start = clock64();
        if (AR) {
            // one item per (m tile, k-block); kbs is even, so a group always owns
            // the same k-blocks and its waits on a slot's barriers stay in order
            const uint32_t items = (uint32_t)(my_tiles / prm.n_tiles) * kbs;
            for (uint32_t u = g; u < items; u += CONV_W / 4) {
                const uint32_t mgen = u / kbs, kb = u - mgen * kbs;
                const uint32_t rs = u % RS;
                {
                    F4_T0();
                    mbar_wait_sleep(&raw_full[rs], (u / RS) & 1);
                    F4_ACC(w_raw);
                }
                const uint32_t raw = sRaw_u + rs * RAW_SLOT + r * 32;
                const uint4 p0 = lds_v4(raw + (rsw << 4)), p1 = lds_v4(raw + ((rsw ^ 1) << 4));
                uint4 m0 = make_uint4(0, 0, 0, 0), m1 = m0;
                if (A_TER) {
                    m0 = lds_v4(raw + F4_RAW_PLANE + (rsw << 4));
                    m1 = lds_v4(raw + F4_RAW_PLANE + ((rsw ^ 1) << 4));
                }
                // free the 16 KB raw ring early: the loads have returned (the dummy
                // asm consumes them) and are ordered before the TMA refill
                asm volatile("" ::"r"(p0.x), "r"(p1.w), "r"(m0.x), "r"(m1.w));
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&raw_empty[rs]);
                {
                    F4_T0();
                    mbar_wait_sleep(&a_empty[kb >> 1], (mgen & 1) ^ 1);  // last n tile of the previous m tile done
                    F4_ACC(w_slot);
                }
                F4_T0();
                const uint32_t row = sA_u + kb * F4_A_BYTES + r * 128;
                const uint32_t sw = (uint32_t)r & 7;  // SW128: chunk c at c ^ (row % 8)
                fp4_chunk<A_TER>(p0.x, m0.x, row + ((0 ^ sw) << 4));
                fp4_chunk<A_TER>(p0.y, m0.y, row + ((1 ^ sw) << 4));
                fp4_chunk<A_TER>(p0.z, m0.z, row + ((2 ^ sw) << 4));
                fp4_chunk<A_TER>(p0.w, m0.w, row + ((3 ^ sw) << 4));
                fp4_chunk<A_TER>(p1.x, m1.x, row + ((4 ^ sw) << 4));
                fp4_chunk<A_TER>(p1.y, m1.y, row + ((5 ^ sw) << 4));
                fp4_chunk<A_TER>(p1.z, m1.z, row + ((6 ^ sw) << 4));
                fp4_chunk<A_TER>(p1.w, m1.w, row + ((7 ^ sw) << 4));
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(a_ready0 + (kb >> 1) * 8);
                F4_ACC(w_work);
            }
        }
        for (uint32_t t = g; !AR && t < total; t += 2) {
            // raw load index of this k-block: resident rings load once per m tile
            const uint32_t seq = t / kbs, kb = t - seq * kbs;
            const uint32_t nt = seq % nts;
            const uint32_t u = prm.resident ? (seq / nts) * kbs + kb : t;
            const bool release = !prm.resident || nt == nts - 1;
            const uint32_t rs = u % RS, st = t % F4_A_ST;
            // g2: slot st belongs to stage (t/2)%2, released and signalled per stage
            const uint32_t bar_i = g2 ? (t >> 1) & 1 : st, bar_ph = g2 ? (t >> 2) & 1 : (t / F4_A_ST) & 1;
            {
                F4_T0();
                mbar_wait_sleep(&raw_full[rs], (u / RS) & 1);
                F4_ACC(w_raw);
            }
            {
                F4_T0();
                mbar_wait_sleep(&a_empty[bar_i], bar_ph ^ 1);
                F4_ACC(w_slot);
            }
            F4_T0();
            const uint32_t raw = sRaw_u + rs * RAW_SLOT + r * 32;
            if (F4_DBG(1)) goto done;
            {
            const uint4 p0 = lds_v4(raw + (rsw << 4)), p1 = lds_v4(raw + ((rsw ^ 1) << 4));
            uint4 m0 = make_uint4(0, 0, 0, 0), m1 = m0;
            if (A_TER) {
                m0 = lds_v4(raw + F4_RAW_PLANE + (rsw << 4));
                m1 = lds_v4(raw + F4_RAW_PLANE + ((rsw ^ 1) << 4));
            }
            const uint32_t row = sA_u + st * F4_A_BYTES + r * 128;
            const uint32_t sw = (uint32_t)r & 7;  // SW128: chunk c at c ^ (row % 8)
            fp4_chunk<A_TER>(p0.x, m0.x, row + ((0 ^ sw) << 4));
            fp4_chunk<A_TER>(p0.y, m0.y, row + ((1 ^ sw) << 4));
            fp4_chunk<A_TER>(p0.z, m0.z, row + ((2 ^ sw) << 4));
            fp4_chunk<A_TER>(p0.w, m0.w, row + ((3 ^ sw) << 4));
            fp4_chunk<A_TER>(p1.x, m1.x, row + ((4 ^ sw) << 4));
            fp4_chunk<A_TER>(p1.y, m1.y, row + ((5 ^ sw) << 4));
            fp4_chunk<A_TER>(p1.z, m1.z, row + ((6 ^ sw) << 4));
            fp4_chunk<A_TER>(p1.w, m1.w, row + ((7 ^ sw) << 4));
            }
        done:
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
                if (release) mbar_arrive(&raw_empty[rs]);
                mbar_arrive_cluster(a_ready0 + bar_i * 8);
            }
            F4_ACC(w_work);
        }
        if (F4_DBG(8) && lane == 0) {
            atomicAdd(&g_fp4_stats[4], (unsigned long long)w_raw);
            atomicAdd(&g_fp4_stats[5], (unsigned long long)w_slot);
            atomicAdd(&g_fp4_stats[6], (unsigned long long)w_work);
            atomicAdd(&g_fp4_stats[7], (unsigned long long)(clock64() - t_start));
        }
    } else {
        // ===================== epilogue (both CTAs) =====================
        const int ewarp = warp - CONV_W;
        const int wq = warp & 3;            // TMEM lane quarter (warp % 4, as tcgen05.ld/st require)
        const int half = ewarp >> 2;        // column range of the tile this warp drains
        constexpr int NHALF = EPI_W / 4;
        // chunk ranges of an even length (bn is a multiple of 32): whole 32-column store boxes
        const int nch_all = bn / 16, per_half = ((nch_all + NHALF - 1) / NHALF + 1) & ~1;
        const int ch_lo = half * per_half, ch_hi = ch_lo + per_half < nch_all ? ch_lo + per_half : nch_all;
        // the warps draining the last chunk also own the scale hand-off (sf_ready counts 8)
        const bool sf_owner = half == (nch_all - 1) / per_half;
        const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
        const uint32_t sf_ready0 = mapa_shared(smem_u32(&sf_ready[0]), pbase);
        // unit block scales (UE8M0 0x7F = 2^0) into buffer c's tail, then tell the MMA warp
        auto put_scales = [&](int c) {
            tmem_st_32x32b_x8_fill(tmem_base + lane_base + (uint32_t)c * F4_MAX_BN + F4_SF_OFF, 0x7F7F7F7Fu);
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(sf_ready0 + c * 8);
        };
        if (sf_owner) put_scales(1);  // tile 0 runs on buffer 0

        const uint32_t tmem_empty0 = mapa_shared(smem_u32(&tmem_empty[0]), pbase);
        const bool vec_ok = ((prm.ldc & 15) == 0) && ((reinterpret_cast<uintptr_t>(prm.c) & 31) == 0);
        const uint32_t epi = smem_u32(sEpi) + (uint32_t)ewarp * EGRP * F4_EPI_BYTES;
        int acc = 0;
        uint32_t acc_phase = 0;
        long long w_ep = 0, w_tail = 0, w_grp0 = 0, w_grp1 = 0;
        const long long t_start = clock64();
        for (int i = 0; i < my_tiles; ++i) {
            int mt, nt;
            tile_of(i, mt, nt);
            const int row0 = mt * 2 * F4_BM + (int)rank * F4_BM + wq * 32;
            {
                // one epilogue warp waits on the mbarrier; the others block on a named barrier
                // (wait loops in every warp cost issue slots)
                F4_T0();
                if (ewarp == 0) mbar_wait_sleep(&tmem_full[acc], acc_phase);
                named_bar_sync(1, 32 * EPI_W);
                F4_ACC(w_ep);
            }
            F4_T0();
            tc_fence_after();
            const uint32_t tacc = tmem_base + lane_base + (uint32_t)acc * F4_MAX_BN;
            const int nch = F4_DBG(4) ? 0 : bn / 16;
            // tail first: the next tile's scales go there (its last chunk waits in registers)
            uint32_t vt[16];
            const bool tail_out = bn > (int)F4_SF_OFF && nch > 0 && sf_owner;
            if (tail_out) {
                tmem_ld_32x32b_x16(tacc + (nch - 1) * 16, vt);
                tmem_ld_wait();
            }
            if (sf_owner) put_scales(acc);
            F4_ACC(w_tail);
            // f32 -> int16 without F2I (quarter rate): x + 1.5 * 2^23 puts the
            // integer x (|x| <= 32767) in the low mantissa bits, so its low
            // half-word IS the int16 result.
            auto to_i16 = [](const uint32_t (&v)[16], uint32_t (&h)[8]) {
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    h[j] = __byte_perm(__float_as_uint(__uint_as_float(v[2 * j]) + 12582912.0f),
                                       __float_as_uint(__uint_as_float(v[2 * j + 1]) + 12582912.0f), 0x5410);
            };
            // Groups of EGRP 16-column chunks: one TMEM wait, one wait for the
            // staging buffers, one proxy fence and one bulk group per group.
            long long _tg = F4_DBG(8) ? clock64() : 0;
            const int cend = nch < ch_hi ? nch : ch_hi;
            for (int g0 = ch_lo; g0 < cend; g0 += EGRP) {
                uint32_t v[EGRP][16];
                if (!F4_DBG(256)) {  // debug 256: timing experiment without the TMEM loads
#pragma unroll
                    for (int j = 0; j < EGRP; ++j)
                        if (g0 + j < cend && !(tail_out && g0 + j == nch - 1))
                            tmem_ld_32x32b_x16(tacc + (g0 + j) * 16, v[j]);
                    tmem_ld_wait();
                } else {
#pragma unroll
                    for (int j = 0; j < EGRP; ++j)
#pragma unroll
                        for (int q = 0; q < 16; ++q) v[j][q] = (uint32_t)(g0 + j + q);
                }
                if (prm.tma_store) {
                    if (lane == 0) bulk_wait_read<0>();  // the previous group's stores have read their buffers
                    __syncwarp();
                }
#pragma unroll
                for (int j = 0; j < EGRP; ++j) {
                    const int ch = g0 + j;
                    if (ch < cend) {
                        if (tail_out && ch == nch - 1) {
#pragma unroll
                            for (int q = 0; q < 16; ++q) v[j][q] = vt[q];
                        }
                        uint32_t h[8];
                        to_i16(v[j], h);
                        const int col0 = nt * bn + ch * 16;
                        if (F4_DBG(512)) {  // timing experiment: no staging stores
                            if ((h[0] ^ h[3] ^ h[7]) == 0x9E3779B9u && lane == 77) sts_v4(epi, h[0], h[1], h[2], h[3]);
                        } else if (prm.tma_store) {
                            // chunk j of the group's 32-column box: 64-byte rows, TMA SWIZZLE_64B
                            const uint32_t rowaddr = epi + lane * 64;
                            const uint32_t swz = ((uint32_t)lane >> 1) & 3;
                            sts_v4(rowaddr + (((2u * j) ^ swz) << 4), h[0], h[1], h[2], h[3]);
                            sts_v4(rowaddr + (((2u * j + 1) ^ swz) << 4), h[4], h[5], h[6], h[7]);
                        } else {
                            const int row = row0 + lane;
                            if (row < prm.m) {
                                int16_t* crow = prm.c + (long long)row * prm.ldc;
                                if (vec_ok && col0 + 16 <= prm.n) {  // one full 32-byte sector per lane
                                    stg_v8(crow + col0, h);
                                } else {
#pragma unroll
                                    for (int q = 0; q < 16; ++q)
                                        if (col0 + q < prm.n) crow[col0 + q] = (int16_t)(h[q >> 1] >> (16 * (q & 1)));
                                }
                            }
                        }
                    }
                }
                if (prm.tma_store && !F4_DBG(128)) {  // debug 128: timing experiment without the stores
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        // one 32-column box per group: half the TMA store rows of 16-column boxes
                        // (the store rows share the TMA unit with the B loads): +3.5% on c3 / c5
                        tma_store_2d(&tmap_c, epi, nt * bn + g0 * 16, row0);
                        bulk_commit();
                    }
                }
                if (F4_DBG(8)) {
                    const long long now = clock64();
                    if (g0 == ch_lo) w_grp0 += now - _tg;
                    else w_grp1 += now - _tg;
                    _tg = now;
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(tmem_empty0 + acc * 8);
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
        if (prm.tma_store && lane == 0) bulk_wait<0>();
        if (F4_DBG(8) && lane == 0) {
            atomicAdd(&g_fp4_stats[8], (unsigned long long)w_ep);
            atomicAdd(&g_fp4_stats[9], (unsigned long long)(clock64() - t_start));
            atomicAdd(&g_fp4_stats[10], (unsigned long long)w_tail);
            atomicAdd(&g_fp4_stats[14], (unsigned long long)w_grp0);
            atomicAdd(&g_fp4_stats[15], (unsigned long long)w_grp1);
        }
    }

    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (warp == F4_W_MMA) {
        tc_fence_after();
        tmem_dealloc_pair<512>(tmem_base);
    }
}

}  // namespace lb

extern "C" int lowbit_debug_fp4_stats(unsigned long long* out16) {
    if (cudaMemcpyFromSymbol(out16, lb::g_fp4_stats, sizeof(unsigned long long) * 16) != cudaSuccess) return 1;
    unsigned long long z[16] = {};
    if (cudaMemcpyToSymbol(lb::g_fp4_stats, z, sizeof z) != cudaSuccess) return 1;
    return 0;
}

namespace lb {

// BN: the fewest column tiles of <= 256 (an MMA costs the same for any N <= 256),
// then the smallest multiple of 32 covering n: the epilogue stores 32-column boxes
// (two 16-column chunks), so every warp's chunk range is a whole number of pairs.
static int pick_bn_fp4(int n, int max_bn = F4_MAX_BN) {
    const int tiles = (n + max_bn - 1) / max_bn;
    const int per = (n + tiles - 1) / tiles;
    return (per + 31) / 32 * 32;
}

template <bool A_TER, bool AR, int CL = 2>
static lowbit_status launch_fp4_variant(const CUtensorMap& mb, const CUtensorMap& ma0, const CUtensorMap& ma1,
                                        const CUtensorMap& mc, const Fp4Params& prm, int pairs, cudaStream_t stream) {
    static SmemOptIn attr;
    int max_clusters = 0;  // CL = 4 experiment only: queried per launch (per device)
    constexpr int smem = f4_smem_bytes(AR);
    auto kern = gemm_fp4_pair_kernel<A_TER, AR, CL>;
    LB_CUDA_TRY(attr.ensure(kern, smem));
    if (CL == 4) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(4 * 37);
        cfg.blockDim = dim3(F4_THREADS);
        cfg.dynamicSmemBytes = smem;
        LB_CUDA_TRY(cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg));
    }
    int grid = 2 * pairs;
    if (CL == 4) {  // whole clusters, all co-resident (a later wave would serialise the lockstep pairs)
        int clusters = (prm.m_tiles + 1) / 2 < pairs / 2 ? (prm.m_tiles + 1) / 2 : pairs / 2;
        if (max_clusters > 0 && clusters > max_clusters) clusters = max_clusters;
        grid = 4 * (clusters > 0 ? clusters : 1);
    }
    static const bool verbose = tuning_env("LOWBIT_FP4_VERBOSE") != nullptr;
    if (verbose)
        std::fprintf(stderr, "fp4 kernel: AR %d CL %d grid %d (max clusters %d) bn %d n_tiles %d m_tiles %d\n",
                     (int)AR, CL, grid, max_clusters, prm.bn, prm.n_tiles, prm.m_tiles);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(F4_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    LB_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, mb, ma0, ma1, mc, prm));
    LB_CUDA_TRY(cudaGetLastError());
    return LOWBIT_OK;
}

// A as NIBBLES-layout bit planes (lowbit_encode_ex layout 2).
lowbit_status launch_fp4_pair(int a_ternary, int layout, const uint8_t* a0, const uint8_t* a1, long long a_pitch, int m, int n,
                              int k, const void* weights, int b_ternary, int16_t* c, long long ldc,
                              cudaStream_t stream) {
    const WeightsLayout L(b_ternary, n, k);
    Fp4Params prm{};
    prm.m = m;
    prm.n = n;
    prm.kblocks = L.kp4 / F4_BK;
    prm.bn = pick_bn_fp4(n);
    prm.m_tiles = (m + 2 * F4_BM - 1) / (2 * F4_BM);
    prm.n_tiles = (n + prm.bn - 1) / prm.bn;
    prm.ldc = ldc;
    prm.c = c;
    prm.tma_store = ((ldc * 2) % 16 == 0) && ((reinterpret_cast<uintptr_t>(c) & 15) == 0);
    static const bool direct_epi = [] {
        const char* e = tuning_env("LOWBIT_FP4_EPI");
        return e && e[0] == 'd';
    }();
    if (direct_epi) prm.tma_store = 0;
    // resident raw ring: the whole depth fits, and each k-block is always
    // handled by the same converter group (even k-block count) so its last
    // reader is the one that frees it
    prm.m_major = prm.m_tiles >= num_sms() / 2;
    prm.resident = prm.m_major && prm.kblocks <= f4_raw_stages(a_ternary != 0) &&
                   (prm.kblocks % 2 == 0 || prm.n_tiles == 1);
    static const int no_ar = [] {
        const char* e = tuning_env("LOWBIT_FP4_NO_AR");  // tuning experiments: force the streaming variant
        return e ? atoi(e) : 0;
    }();
    prm.a_res = !no_ar && prm.m_major && prm.n_tiles >= 2 && prm.kblocks <= F4_AR_SLOTS && prm.kblocks % 2 == 0;
    if (prm.a_res) {
        prm.resident = 1;  // raw planes load once per m tile
        prm.bn = pick_bn_fp4(n, F4_AR_BN);
        prm.n_tiles = (n + prm.bn - 1) / prm.bn;
    }
    static const int debug = [] {
        const char* e = tuning_env("LOWBIT_DEBUG_FP4");
        return e ? atoi(e) : 0;
    }();
    prm.debug = debug;
    CUtensorMap mb, ma0, ma1, mc;
    // NIBBLES planes pair with the canonical fp4 B section, REFERENCE planes with
    // the reference-order one (layout.cuh): the converters are the same
    const uint8_t* wfp4 =
        static_cast<const uint8_t*>(weights) + (layout == LOWBIT_LAYOUT_NIBBLES ? L.off_fp4 : L.off_fp4r);
    if (!make_map_2d(&mb, wfp4, (uint64_t)L.kp4 / 2, (uint64_t)L.np, (uint64_t)L.kp4 / 2, 128, (uint32_t)(prm.bn / 2),
                     CU_TENSOR_MAP_SWIZZLE_128B))
        return lbhost::set_error(LOWBIT_CUDA_ERROR, "cuTensorMapEncodeTiled failed for fp4 B");
    if (prm.tma_store) {
        if (!make_map_2d(&mc, c, (uint64_t)n, (uint64_t)m, (uint64_t)ldc * 2, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B,
                         CU_TENSOR_MAP_DATA_TYPE_UINT16))
            return lbhost::set_error(LOWBIT_CUDA_ERROR, "cuTensorMapEncodeTiled failed for C");
    } else {
        mc = mb;
    }
    if (!make_map_2d(&ma0, a0, (uint64_t)a_pitch, (uint64_t)m, (uint64_t)a_pitch, 32, F4_BM,
                     CU_TENSOR_MAP_SWIZZLE_32B))
        return lbhost::set_error(LOWBIT_CUDA_ERROR, "cuTensorMapEncodeTiled failed for A");
    if (a_ternary) {
        if (!make_map_2d(&ma1, a1, (uint64_t)a_pitch, (uint64_t)m, (uint64_t)a_pitch, 32, F4_BM,
                         CU_TENSOR_MAP_SWIZZLE_32B))
            return lbhost::set_error(LOWBIT_CUDA_ERROR, "cuTensorMapEncodeTiled failed for A minus");
    } else {
        ma1 = ma0;
    }
    const int work = prm.m_major ? prm.m_tiles : prm.m_tiles * prm.n_tiles;
    const int pairs = work < num_sms() / 2 ? work : num_sms() / 2;
#define F4_LAUNCH(TER, AR_) launch_fp4_variant<TER, AR_>(mb, ma0, ma1, mc, prm, pairs, stream)
    static const int cl4 = [] {
        const char* e = tuning_env("LOWBIT_FP4_CL4");  // 4-CTA clusters with multicast B for the AR variant
        return e ? atoi(e) : 0;
    }();
    if (prm.a_res && cl4) {
        // Tuning experiment (LOWBIT_FP4_CL4=1, LOWBIT_TUNING builds): multicast B across 4-CTA
        // clusters.  Per SM the k-block time drops ~8% (half the B traffic), but only 33 clusters
        // (132 SMs) fit the GPCs, so it measured 3% slower on c5.
        return a_ternary ? launch_fp4_variant<true, true, 4>(mb, ma0, ma1, mc, prm, pairs, stream)
                         : launch_fp4_variant<false, true, 4>(mb, ma0, ma1, mc, prm, pairs, stream);
    }
    if (prm.a_res) return a_ternary ? F4_LAUNCH(true, true) : F4_LAUNCH(false, true);
    return a_ternary ? F4_LAUNCH(true, false) : F4_LAUNCH(false, false);
#undef F4_LAUNCH
}

}  // namespace lb

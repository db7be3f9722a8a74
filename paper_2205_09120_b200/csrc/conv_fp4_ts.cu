// conv_fp4_ts.cu — K7T: the fused halo convolution (K7, conv_fp4_halo.cu) with
// the filter resident in TENSOR MEMORY and one CTA per tile.
//
// Same algorithm and contract as K7 — conv2d_lowbit (conv.cpp:33-59) as one
// kernel over the int8 NHWC map: a TMA box brings a tile's input halo, eight
// converter warps pack it to e2m1 in shared memory (int8 AND 0x09, a chunk
// holding a value outside {-1, 0, +1} rewritten by sign, core.cpp:40-58), and
// filter tap (ky, kx) is the halo's UMMA descriptor advanced by ky*P + kx rows.
// What differs is the operand roles:
//
//   * D[cout, position] = W[cout, k] x X[position, k]^T: the FILTER is the
//     UMMA A operand, held in TMEM for the whole kernel (M = 128 output
//     channels; 16 TMEM columns per 128-channel k-block, the row's fp4 bytes
//     in natural order), and the converted halo is the B operand (N = 128
//     positions) in shared memory.  tcgen05.mma.cta_group::1.kind::mxf4 with A
//     from TMEM reads only the halo from shared memory: 4 KB per MMA against
//     6 KB for K7's pair MMA (A halo + half the filter).  Shared-memory
//     bandwidth is what K7's tile period is made of (the tensor pipe's operand
//     reads, the converters' LDS/STS, the epilogue's staging and the TMA
//     traffic share it), so the tile's traffic drops by ~15%.
//   * No CTA pairs, no cluster barriers: every CTA runs its own tiles.
//   * A bias MMA first sets every accumulator element to 1.5 * 2^22 (A: eight
//     TMEM columns of e2m1 1.0 under a 2^16 block scale, B: one uniform
//     swizzle atom of 1.5 with a descriptor stride of 0), so the exact
//     half-integer sums live in [2^22, 2^23) and the low 16 bits of each f32
//     are the int16 result (as in K7).
//   * The accumulator is channel-major (TMEM lane = output channel).  The
//     epilogue reads its low halves with tcgen05.ld.16x128b.pack::16b, whose
//     per-thread fragment is the m8n8 b16 matrix fragment, and writes it with
//     stmatrix.trans: each 8x8 block lands transposed, one 16-byte run of 8
//     channels per output position, in a 64-byte-swizzled staging box that a
//     TMA store writes to the NHWC output (clipped at the image edges).  No
//     arithmetic: one TMEM load and two stmatrix per 16 channels x 32 positions.
//
// Takes convs with cout <= 128, at most 14 k-blocks of 128 channels (3x3 over
// 128 channels: 9) and a padded row of <= 128 pixels; K7 keeps the rest.
//
// Warp roles (896 threads): 0-15 epilogue (two groups of 8 on alternate tiles;
// warp w drains TMEM lane quarter w % 4 = 32 output channels for 64
// positions), 16-23 converters, 24 TMA producer (raw halos), 25-26 UMMA
// issuers on alternate tiles (issuer i owns accumulator i; 25 also owns TMEM),
// 27 the converters' waiter.
#include <cstdio>
#include <cstdlib>

#include <type_traits>

#include "common.cuh"
#include "halo_common.cuh"
#include "layout.cuh"
#include "tmap.cuh"

namespace lb {

constexpr int T7_BN = 128;   // positions per tile (UMMA N)
constexpr int T7_NCONV = 8;
constexpr int T7_NEPI = 16;
constexpr int T7_W_CONV = T7_NEPI, T7_W_PROD = T7_W_CONV + T7_NCONV, T7_W_MMA = T7_W_PROD + 1,
              T7_W_WAIT = T7_W_MMA + 2;
constexpr int T7_THREADS = 32 * (T7_W_WAIT + 1);
constexpr int T7_SMEM = 227 * 1024;
constexpr int T7_EPI_BYTES = 4096;        // per epilogue warp: 64 positions x 32 channels x int16
constexpr int T7_MAX_ST = 4;
constexpr int T7_RAW_MAX = 64 * 1024;
constexpr uint32_t T7_FILT_COL = 256;     // filter: 16 columns per k-block (after two 128-column accumulators)
constexpr uint32_t T7_BIAS_COL = 480;     // the bias MMA's A operand: 8 columns of e2m1 1.0
constexpr uint32_t T7_SFBIAS_COL = 496;   // its A scales, 2^16 (8 columns)
constexpr uint32_t T7_SF_COL = 504;       // unit UE8M0 scales, 8 columns
constexpr int T7_MAX_KB = (int)(T7_BIAS_COL - T7_FILT_COL) / 16;  // 14 k-blocks
constexpr int T7_BIAS_B = 512;            // the bias MMA's B operand: one swizzle atom of e2m1 1.5

struct TsParams {
    int batch, h, w, oh, ow, pad, kw, cblocks;
    int P, log2p, R, rows_h;  // position pitch, output rows per tile, halo rows
    int tpi, ctiles;          // tiles per image, tiles
    int cout, kblocks, k33;
    int raw_cb, f4_cb, raw_st, f4_st;
    int box_px, box_rows;     // epilogue TMA box: 64 positions = box_rows x box_px
    uint32_t pad_word;        // binary map padded with +-1: four pad bytes (0: padding reads 0)
    uint32_t mul16;           // 16: the converters' multiplier (a register operand keeps their shifts IMADs)
    int dbg;                  // LOWBIT_TUNING builds only: 32768 return at entry
    int wrows;                // rows of a filter TMA box (min(128, padded cout))
    int* zero_flag;
};

#ifdef LOWBIT_TUNING
#define T7_DBG(bits) (prm.dbg & (bits))
#else
#define T7_DBG(bits) 0
#endif
// dbg & 32 (TUNING builds): clock64 per-tile events of CTA 0 and %globaltimer kernel phases,
// read by lowbit_debug_ts_trace (the same event numbering as K7's trace)
__device__ unsigned long long g_ts_trace[16 * 64];
__device__ unsigned long long g_ts_phase[4];
__device__ unsigned long long g_ts_setup[160 * 4];  // dbg & 32: per CTA: barriers initialised, TMEM allocated, CTA barrier passed
__device__ unsigned long long g_ts_cta[160 * 4];  // dbg & 32: per CTA: entry, work start, work end (globaltimer ns), SM id
LB_DEV unsigned long long t7_gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define T7_TRACE(ev, i) \
    if (T7_DBG(32) && blockIdx.x == 0 && (i) < 64) g_ts_trace[(ev) * 64 + (i)] = clock64()

// D[tmem] (+)= A[tmem] x B[smem]^T, packed e2m1 with UE8M0 block scales (all 1.0 here), one CTA
LB_DEV void umma_mxf4_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc, uint32_t tmem_sfa,
                         uint32_t tmem_sfb, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%5], [%6], p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(tmem_sfa), "r"(tmem_sfb)
        : "memory");
}
// 16 TMEM lanes x 32 columns, the LOW 16 bits of each column: word 2g of thread t holds columns
// 8g + 2(t%4), 8g + 2(t%4) + 1 of lane t/4, word 2g + 1 the same columns of lane 8 + t/4 — each word
// across the warp is an m8n8 b16 matrix fragment (the 16x256b shape packs four consecutive columns
// per thread instead, which costs stmatrix two-way bank conflicts in a swizzled box)
LB_DEV void tmem_ld_16x128b_x4_pack16(uint32_t taddr, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.16x128b.x4.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}
LB_DEV void tmem_st_32x32b_x16(uint32_t taddr, const uint32_t (&v)[16]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                 "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
                 : "memory");
}
// four 8x8 b16 matrices stored transposed: row r of matrix i goes to the address thread 8i + r holds
LB_DEV void stsm_x4_trans(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("stmatrix.sync.aligned.m8n8.x4.trans.shared.b16 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b),
                 "r"(c), "r"(d)
                 : "memory");
}
// FLAGS bit 0 (PADFILL): binary map padded with +-1; bit 1 (CHECKZ): BNN map, a 0 raises
// ZeroInBinaryInput (core.cpp:23) — as K7
template <int FLAGS>
__global__ void __launch_bounds__(T7_THREADS, 1)
    conv_fp4_ts_kernel(const __grid_constant__ CUtensorMap tmap_raw, const __grid_constant__ CUtensorMap tmap_out,
                       const __grid_constant__ CUtensorMap tmap_w, const TsParams prm) {
    constexpr bool PADFILL = (FLAGS & 1) != 0, CHECKZ = (FLAGS & 2) != 0;
    if (T7_DBG(32768)) return;
    if (T7_DBG(32) && threadIdx.x == 0) {
        atomicMin(&g_ts_phase[0], t7_gtime());
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_ts_cta[blockIdx.x * 4] = t7_gtime();
        g_ts_cta[blockIdx.x * 4 + 3] = smid;
    }
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int CB = prm.cblocks;
    const int raw_stage = CB * prm.raw_cb, f4_stage = CB * prm.f4_cb;
    uint8_t* sEpi = smem;                                  // 16 x 4 KB staging boxes
    uint8_t* sF4 = sEpi + T7_NEPI * T7_EPI_BYTES;          // fp4 halo ring (the UMMA B operand)
    uint8_t* sRaw = sF4 + prm.f4_st * f4_stage;            // raw int8 halo ring
    uint8_t* sBiasB = sRaw + prm.raw_st * raw_stage;       // the bias MMA's B operand (uniform bytes)
    uint64_t* bars = reinterpret_cast<uint64_t*>(sBiasB + T7_BIAS_B);
    uint64_t* raw_full = bars;          // TMA landed the raw halo
    uint64_t* raw_empty = bars + 4;     // the converter warps are done with it
    uint64_t* a_full = bars + 8;        // fp4 halo written (all converter warps)
    uint64_t* a_empty = bars + 12;      // the tile's MMAs are done with the fp4 halo
    uint64_t* tmem_full = bars + 16;    // (2) accumulator complete
    uint64_t* tmem_empty = bars + 18;   // (2) drained by the 8 epilogue warps of its group
    uint64_t* f_ready = bars + 32;      // (3) a third of the filter's k-blocks is in TMEM (the 16 epilogue warps);
                                        //     the first also covers the bias operand and the scales
    uint64_t* f_tma = bars + 35;        // (3) that third's TMA boxes landed in the bounce buffers
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 22);
    uint32_t* kb_boff = reinterpret_cast<uint32_t*>(bars + 24);  // k-block -> halo row offset (16-byte units)

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int ncta = gridDim.x;
    const int my_tiles = prm.ctiles > (int)blockIdx.x ? (prm.ctiles - (int)blockIdx.x + ncta - 1) / ncta : 0;

    // The filter's way into TMEM: TMA brings each k-block's 128 rows x 64 B into a bounce buffer — the
    // still idle staging boxes, then the last fp4 slot — and the epilogue warps move it on (below).  It
    // travels in three groups of k-blocks, each with its own barriers, so the first tile's MMAs start
    // on the first third while the rest is still on its way (148 CTAs pull 136 KB each at once).
    auto fgroup = [&](int g) -> int { return g * prm.kblocks / 3; };  // first k-block of group g
    auto bounce = [&](int j) -> uint32_t {  // k-block j's buffer
        constexpr int NE = T7_NEPI * T7_EPI_BYTES / 8192;
        return j < NE ? smem_u32(sEpi) + (uint32_t)j * 8192u
                      : smem_u32(sF4 + (prm.f4_st - 1) * f4_stage) + (uint32_t)(j - NE) * 8192u;
    };
    auto load_filter = [&]() {
        for (int g = 0; g < 3; ++g) {
            const int j0 = fgroup(g), j1 = fgroup(g + 1);
            mbar_arrive_expect_tx(&f_tma[g], (uint32_t)(j1 - j0) * (uint32_t)prm.wrows * 64u);
            for (int j = j0; j < j1; ++j)
                tma_load_2d(reinterpret_cast<void*>(smem + (bounce(j) - smem_u32(smem))), &tmap_w, &f_tma[g], j * 64, 0);
        }
    };

    // The producer thread initialises the barriers and at once sends the first tile's halo and the
    // filter on their way (its own griddepcontrol.wait orders them after the previous grid): they
    // gate the first tile, and the rest of the setup (TMEM, the CTA barrier) takes another ~0.5 us.
    if (warp == T7_W_PROD && lane == 0) {
        for (int s = 0; s < T7_MAX_ST; ++s) {
            mbar_init(&raw_full[s], 1);
            mbar_init(&raw_empty[s], T7_NCONV);
            mbar_init(&a_full[s], T7_NCONV);
            mbar_init(&a_empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tmem_full[a], 1);
            mbar_init(&tmem_empty[a], 8);
        }
        for (int g = 0; g < 3; ++g) {
            mbar_init(&f_ready[g], T7_NEPI);
            mbar_init(&f_tma[g], 1);
        }
        fence_barrier_init();
        if (T7_DBG(32)) g_ts_setup[blockIdx.x * 4] = t7_gtime();
        tma_prefetch_desc(&tmap_raw);
        tma_prefetch_desc(&tmap_w);
        asm volatile("griddepcontrol.wait;" ::: "memory");
        if (my_tiles > 0) {
            H7Walk wk;
            wk.init((int)blockIdx.x, ncta, prm.tpi);
            mbar_arrive_expect_tx(&raw_full[0], (uint32_t)raw_stage);
            for (int cb = 0; cb < CB; ++cb)
                tma_load_4d(smem_u32(sRaw + cb * prm.raw_cb), &tmap_raw, smem_u32(&raw_full[0]), cb * 128, -prm.pad,
                            wk.rem * prm.R - prm.pad, wk.img);
        }
        load_filter();
    }
    if (threadIdx.x < T7_BIAS_B / 16)  // every B element of the bias MMA is e2m1 1.5
        sts_v4(smem_u32(sBiasB) + threadIdx.x * 16, 0x33333333u, 0x33333333u, 0x33333333u, 0x33333333u);
    fence_proxy_async_smem();
    if (warp == T7_W_PROD && lane == 1) tma_prefetch_desc(&tmap_out);
    if (warp == T7_W_MMA) {
        tmem_alloc<512>(tmem_slot);
        if (T7_DBG(32) && lane == 0) g_ts_setup[blockIdx.x * 4 + 1] = t7_gtime();
        for (int kb = lane; kb < prm.kblocks; kb += 32) {  // tap (ky,kx), channel block cb
            const int tap = kb / CB, cb = kb - tap * CB;
            const int ky = tap / prm.kw, kx = tap - ky * prm.kw;
            kb_boff[kb] = ((uint32_t)(cb * prm.f4_cb) + (uint32_t)(ky * prm.P + kx) * 64u) >> 4;
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (T7_DBG(32) && threadIdx.x == 0) g_ts_setup[blockIdx.x * 4 + 2] = t7_gtime();
    // the next kernel in the stream may begin launching; global memory is touched only after the wait
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (T7_DBG(32) && threadIdx.x == 0) {
        atomicMax(&g_ts_phase[1], t7_gtime());
        g_ts_cta[blockIdx.x * 4 + 1] = t7_gtime();
    }

    if (warp == T7_W_PROD) {
        // ===================== TMA producer: raw halos (and the filter's first round) =====================
        if (lane == 0) {
            H7Ring rr;
            rr.init(prm.raw_st);
            H7Walk wk;
            wk.init((int)blockIdx.x, ncta, prm.tpi);
            for (int i = 0; i < my_tiles; ++i, rr.next(), wk.next()) {
                const uint32_t s = rr.idx;
                if (i == 0) {  // sent before the setup
                    T7_TRACE(0, i);
                    continue;
                }
                mbar_wait_sleep(&raw_empty[s], rr.phase ^ 1);
                T7_TRACE(0, i);
                mbar_arrive_expect_tx(&raw_full[s], (uint32_t)raw_stage);
                for (int cb = 0; cb < CB; ++cb)
                    tma_load_4d(smem_u32(sRaw + s * raw_stage + cb * prm.raw_cb), &tmap_raw, smem_u32(&raw_full[s]),
                                cb * 128, -prm.pad, wk.rem * prm.R - prm.pad, wk.img);
            }
        }
    } else if (warp >= T7_W_CONV && warp < T7_W_PROD) {
        // ===================== converters: raw int8 halo -> fp4 halo (as K7) =====================
        const int cw = warp - T7_W_CONV;
        const int P = prm.P, lp = prm.log2p, rows_h = prm.rows_h, raw_st = prm.raw_st, f4_st = prm.f4_st;
        const int raw_cb = prm.raw_cb, f4_cb = prm.f4_cb, R = prm.R;
        const int npos = rows_h * P;             // a multiple of 32
        constexpr int STEP = 4 * T7_NCONV;
        const int nfull = npos / (8 * STEP), nrem = (npos % (8 * STEP)) / STEP;
        const int nbatch = nfull + (nrem != 0);
        const int chunk = lane & 7;
        const int j0 = cw * 4 + (lane >> 3);
        // SW64: 16-byte unit u of row j at j*64 + ((u ^ ((j >> 1) & 3)) << 4)
        const uint32_t swz = ((((uint32_t)chunk >> 1) ^ (((uint32_t)j0 >> 1) & 3u)) << 4) + (chunk & 1) * 8;
        const uint32_t k16 = prm.mul16, k2 = k16 >> 3;
        bool zero = false;
        H7Ring rr, fr;
        rr.init(raw_st);
        fr.init(f4_st);
        H7Walk wk;
        wk.init((int)blockIdx.x, ncta, prm.tpi);
        for (int i = 0; i < my_tiles; ++i, rr.next(), fr.next(), wk.next()) {
            const uint32_t rs = rr.idx, fs = fr.idx;
            named_bar_sync(3 + rs, 32 * (T7_NCONV + 1));  // the waiter saw raw_full and a_empty
            if (cw == 0 && lane == 0) T7_TRACE(2, i);
            const int ytop = wk.rem * R - prm.pad;  // image row of halo row 0 (binary maps)
            for (int cb = 0; cb < CB; ++cb) {
                const uint32_t src = smem_u32(sRaw + rs * raw_stage + cb * raw_cb) + chunk * 16;
                const uint32_t dst = smem_u32(sF4 + fs * f4_stage + cb * f4_cb) + swz;
                // a batch: NQ loads in flight (a compile-time count), then as many stores
                auto batch = [&](auto nq_c, int jb, bool last) {
                    constexpr int NQ = decltype(nq_c)::value;
                    uint4 v[NQ];
#pragma unroll
                    for (int q = 0; q < NQ; ++q) v[q] = lds_v4(src + ((uint32_t)(jb + STEP * q) << 7));
                    if (last) {  // the tile's last loads are issued: hand the raw slot back
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&raw_empty[rs]);
                    }
                    if (PADFILL || CHECKZ) {
#pragma unroll
                        for (int q = 0; q < NQ; ++q) {
                            const int j = jb + STEP * q;
                            const int y = ytop + (j >> lp), x = (j & (P - 1)) - prm.pad;
                            const bool real = (unsigned)y < (unsigned)prm.h && (unsigned)x < (unsigned)prm.w;
                            if (CHECKZ && real && !h7_all_nonzero(v[q])) zero = true;
                            if (PADFILL && !real) v[q] = make_uint4(prm.pad_word, prm.pad_word, prm.pad_word, prm.pad_word);
                        }
                    }
                    uint32_t bad = 0;
#pragma unroll
                    for (int q = 0; q < NQ; ++q) {
                        sts_v2(dst + (uint32_t)(jb + STEP * q) * 64u, h7_pack8(v[q].x, v[q].y, k16),
                               h7_pack8(v[q].z, v[q].w, k16));
                        bad |= h7_bad16(v[q], k2);
                    }
                    if ((bad & 0xFEFEFEFEu) != 0) {  // a value outside {-1, 0, +1}: rewrite the chunks by sign
#pragma unroll
                        for (int q = 0; q < NQ; ++q)
                            sts_v2(dst + (uint32_t)(jb + STEP * q) * 64u, h7_pack8_sign(v[q].x, v[q].y),
                                   h7_pack8_sign(v[q].z, v[q].w));
                    }
                };
                const bool last_cb = cb == CB - 1;
                for (int bi = 0; bi < nfull; ++bi)
                    batch(std::integral_constant<int, 8>{}, j0 + bi * 8 * STEP, last_cb && bi == nbatch - 1);
                // the last, partial batch: 2, 4 or 6 loads at once, any other count one load at a time
                const int jr = j0 + nfull * 8 * STEP;
                if (nrem == 6) batch(std::integral_constant<int, 6>{}, jr, last_cb);
                else if (nrem == 4) batch(std::integral_constant<int, 4>{}, jr, last_cb);
                else if (nrem == 2) batch(std::integral_constant<int, 2>{}, jr, last_cb);
                else
                    for (int q = 0; q < nrem; ++q)
                        batch(std::integral_constant<int, 1>{}, jr + STEP * q, last_cb && q == nrem - 1);
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (cw == 0 && lane == 0) T7_TRACE(3, i);
            if (lane == 0) mbar_arrive(&a_full[fs]);
        }
        if (zero && prm.zero_flag) atomicOr(prm.zero_flag, 1);
    } else if (warp == T7_W_WAIT) {
        // ===================== the converters' waiter (as K7) =====================
        H7Ring rr, fr;
        rr.init(prm.raw_st);
        fr.init(prm.f4_st);
        for (int i = 0; i < my_tiles; ++i, rr.next(), fr.next()) {
            // the filter's overflow k-blocks bounce through the last fp4 slot (see the epilogue warps):
            // its first converter pass waits until they are in TMEM (long since, in practice)
            if (i == prm.f4_st - 1)
                for (int g = 0; g < 3; ++g) mbar_wait_sleep(&f_ready[g], 0);
            mbar_wait_sleep(&raw_full[rr.idx], rr.phase);
            if (lane == 0) T7_TRACE(1, i);
            mbar_wait_sleep(&a_empty[fr.idx], fr.phase ^ 1);
            __syncwarp();
            named_bar_arrive(3 + rr.idx, 32 * (T7_NCONV + 1));
        }
    } else if (warp >= T7_W_MMA) {
        // ===================== UMMA issuers: issuer i takes tiles i, i+2, ... into accumulator i =====================
        const int which = warp - T7_W_MMA;
        if (my_tiles > which) {
            const uint32_t idesc = idesc_mxf4(128, T7_BN);
            const uint32_t sf = tmem_base + T7_SF_COL, sf_bias = tmem_base + T7_SFBIAS_COL;
            const uint32_t filt = tmem_base + T7_FILT_COL, bias_a = tmem_base + T7_BIAS_COL;
            const uint64_t bias_bd = h7_desc_sw64(smem_u32(sBiasB), 0);  // every 8-row atom is the same 512 bytes
            const uint32_t d_tmem = tmem_base + (uint32_t)which * T7_BN;
            const uint32_t p4 = (uint32_t)prm.P * 4;  // one halo row in 16-byte units
            const int nkb = prm.kblocks;
            int fg = 0;  // filter groups known to be in TMEM (the first tile of each issuer waits for them as it goes)
            auto need = [&](int kb) {
                while (fg < 3 && kb >= fgroup(fg)) mbar_wait(&f_ready[fg++], 0);
                tc_fence_after();
            };
            H7Ring fr;
            fr.init(prm.f4_st);
            uint32_t acc_phase = 0;
            for (int i = 0; i < my_tiles; ++i, fr.next()) {
                if ((i & 1) != which) continue;  // the other issuer's tile
                mbar_wait_poll(&tmem_empty[which], acc_phase ^ 1);
                acc_phase ^= 1;
                if (lane == 0) T7_TRACE(4, i);
                const uint32_t fs = fr.idx;
                mbar_wait_poll(&a_full[fs], fr.phase);
                tc_fence_after();
                if (lane == 0) T7_TRACE(5, i);
                if (lane == 0) {
                    const uint64_t bd0 = h7_desc_sw64(smem_u32(sF4 + fs * f4_stage));
                    // the bias MMA: every accumulator element = 64 * (1.0 * 2^16) * 1.5 = 1.5 * 2^22 (see K7)
                    if (fg < 3) need(0);
                    umma_mxf4_ts(d_tmem, bias_a, bias_bd, idesc, sf_bias, sf, 0);
                    if (prm.k33) {
#pragma unroll
                        for (int kb = 0; kb < 9; ++kb) {
                            if (fg < 3) need(kb);
                            const uint64_t bd = bd0 + (uint32_t)((kb / 3) * p4 + (kb % 3) * 4);
                            umma_mxf4_ts(d_tmem, filt + (uint32_t)kb * 16, bd, idesc, sf, sf, 1);
                            umma_mxf4_ts(d_tmem, filt + (uint32_t)kb * 16 + 8, bd + 2, idesc, sf, sf, 1);
                        }
                    } else {
                        for (int kb = 0; kb < nkb; ++kb) {
                            if (fg < 3) need(kb);
                            const uint64_t bd = bd0 + kb_boff[kb];
                            umma_mxf4_ts(d_tmem, filt + (uint32_t)kb * 16, bd, idesc, sf, sf, 1);
                            umma_mxf4_ts(d_tmem, filt + (uint32_t)kb * 16 + 8, bd + 2, idesc, sf, sf, 1);
                        }
                    }
                    umma_commit(&a_empty[fs]);
                    umma_commit(&tmem_full[which]);
                    T7_TRACE(6, i);
                }
                __syncwarp();
            }
        }
    } else {
        // ===================== epilogue: warps 0-15 =====================
        const int q = warp & 3;               // TMEM lane quarter: output channels 32q .. 32q+31
        const int half = (warp >> 2) & 1;     // positions 64*half .. +63 of the tile
        const int grp = warp >> 3;            // group: tiles i with i % 2 == grp, accumulator grp
        const uint32_t lane_q = (uint32_t)(q * 32) << 16;
        {
            // The filter into TMEM columns T7_FILT_COL..: lane = output channel n, the row's fp4 bytes
            // (k-block kb, half h at columns 16kb + 8h, the converters' channel order).  Rows are wpitch
            // bytes apart in global memory (a lane loading its own row costs 32 sectors per warp load:
            // 4,600 L1 cycles per CTA in front of the first tile), so TMA brings each k-block into a
            // bounce buffer in the 64-byte swizzle, whose 16-byte units a quarter-warp reads from eight
            // different banks, and each lane moves its row from there into TMEM.
            const int r = q * 32 + lane;
            for (int g = 0; g < 3; ++g) {
                mbar_wait_sleep(&f_tma[g], 0);
                for (int j = fgroup(g) + (warp >> 2); j < fgroup(g + 1); j += 4) {
                    uint32_t v[16];
                    const uint32_t src = bounce(j) + (uint32_t)r * 64u;
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const uint4 x = lds_v4(src + ((uint32_t)(c ^ ((r >> 1) & 3)) << 4));
                        v[4 * c] = x.x, v[4 * c + 1] = x.y, v[4 * c + 2] = x.z, v[4 * c + 3] = x.w;
                    }
                    tmem_st_32x32b_x16(tmem_base + lane_q + T7_FILT_COL + (uint32_t)j * 16, v);
                }
                if (g == 0 && warp < 4) {
                    tmem_st_32x32b_x8_fill(tmem_base + lane_q + T7_SF_COL, 0x7F7F7F7Fu);      // UE8M0 1.0
                    tmem_st_32x32b_x8_fill(tmem_base + lane_q + T7_SFBIAS_COL, 0x8F8F8F8Fu);  // 2^16: the bias MMA's A scales
                    tmem_st_32x32b_x8_fill(tmem_base + lane_q + T7_BIAS_COL, 0x22222222u);    // its A operand: e2m1 1.0
                }
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&f_ready[g]);
            }
            named_bar_sync(7, 32 * T7_NEPI);  // the bounce buffers are read: the first drain may overwrite them
        }
        const uint32_t stg = smem_u32(sEpi) + (uint32_t)warp * T7_EPI_BYTES;
        // stmatrix row addresses: thread t stores position p = 8 * (t / 16) + t % 8 of a 16-position
        // block, channel chunk (t / 8) & 1 of a 16-channel block (the x4 matrices: ch 0-7 / 8-15 of
        // positions 0-7, then of positions 8-15)
        const int tp = 8 * (lane >> 4) + (lane & 7), tc = (lane >> 3) & 1;
        H7Walk wk;
        wk.init((int)blockIdx.x, ncta, prm.tpi);
        uint32_t phase = 0;
        for (int i = 0; i < my_tiles; ++i, wk.next()) {
            if ((i & 1) != grp) continue;  // the other group's tile
            if ((warp & 7) == 0) mbar_wait_sleep(&tmem_full[grp], phase);
            phase ^= 1;
            named_bar_sync(1 + grp, 256);
            tc_fence_after();
            if ((warp & 7) == 0 && lane == 0) T7_TRACE(7, i);
            const int img = wk.img, rt = wk.rem;
            const uint32_t tacc = tmem_base + lane_q + (uint32_t)grp * T7_BN + (uint32_t)half * 64;
            // the accumulator holds 1.5 * 2^22 + sum: the low 16 bits of each f32 are the int16 result;
            // 16 channels x 32 positions per load, already the b16 matrix fragments stmatrix takes
            uint32_t v[4][8];
#pragma unroll
            for (int s = 0; s < 4; ++s)
                tmem_ld_16x128b_x4_pack16(tacc + ((uint32_t)(16 * (s & 1)) << 16) + (s >> 1) * 32, v[s]);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tmem_empty[grp]);  // the accumulator is read: hand it back
            if ((warp & 7) == 0 && lane == 0) T7_TRACE(8, i);
            if (lane == 0) bulk_wait_read<0>();  // the previous box left the staging buffer
            __syncwarp();
#pragma unroll
            for (int s = 0; s < 4; ++s) {  // 16 channels (lanes 16*(s&1) of the quarter) x 32 positions
                const int c16 = s & 1, p32 = s >> 1;
#pragma unroll
                for (int b = 0; b < 2; ++b) {
                    const int p = p32 * 32 + b * 16 + tp;        // position in the warp's 64
                    const int u = 2 * c16 + tc;                  // 16-byte channel chunk in the 64-byte row
                    stsm_x4_trans(stg + (uint32_t)p * 64u + ((uint32_t)(u ^ ((p >> 1) & 3)) << 4), v[s][4 * b],
                                  v[s][4 * b + 1], v[s][4 * b + 2], v[s][4 * b + 3]);
                }
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
                const int pos0 = half * 64;  // the box: box_rows x box_px positions from here
                tma_store_4d(&tmap_out, stg, q * 32, pos0 & (prm.P - 1), rt * prm.R + (pos0 >> prm.log2p), img);
                bulk_commit();
            }
            if ((warp & 7) == 0 && lane == 0) T7_TRACE(9, i);
        }
        if (lane == 0) bulk_wait_read<0>();  // the staging buffers outlive the stores' reads
    }

    tc_fence_before();
    __syncthreads();
    if (T7_DBG(32) && threadIdx.x == 0) {
        atomicMax(&g_ts_phase[2], t7_gtime());
        g_ts_cta[blockIdx.x * 4 + 2] = t7_gtime();
    }
    if (warp == T7_W_MMA) {
        tc_fence_after();
        tmem_dealloc<512>(tmem_base);
    }
}

namespace {
struct TsGeom {
    int P, R, rows_h, raw_cb, f4_cb, raw_st, f4_st, kblocks;
    bool ok;
};
TsGeom ts_geom(int h, int w, int c, int cout, int kh, int kw, int stride, int pad) {
    TsGeom g{};
    g.ok = false;
    const int wp = w + 2 * pad;
    if (stride != 1 || c % 128 != 0 || cout % 8 != 0 || cout > 128 || kw > 9 || wp > 128 || h + 2 * pad < kh ||
        wp < kw)
        return g;
    g.P = wp <= 32 ? 32 : (wp <= 64 ? 64 : 128);
    g.R = T7_BN / g.P;
    g.rows_h = g.R + kh - 1;
    const int cb = c / 128;
    g.kblocks = kh * kw * cb;
    g.raw_cb = g.rows_h * g.P * 128;
    g.f4_cb = ((g.rows_h * g.P + 8) * 64 + 1023) / 1024 * 1024;  // + the taps' over-read past the halo
    if (g.kblocks > T7_MAX_KB || cb * g.raw_cb > T7_RAW_MAX) return g;
    // the filter bounces through the staging boxes and the last fp4 slot on its way to TMEM
    if (g.kblocks > T7_NEPI * T7_EPI_BYTES / 8192 + cb * g.f4_cb / 8192) return g;
    const int budget = T7_SMEM - 1024 - 1024 - T7_BIAS_B - T7_NEPI * T7_EPI_BYTES;  // alignment, barriers, bias operand, staging
    for (int f4 = 3; f4 >= 2; --f4) {
        const int raw = (budget - f4 * cb * g.f4_cb) / (cb * g.raw_cb);
        if (raw >= 2) {
            g.f4_st = f4;
            g.raw_st = raw < T7_MAX_ST ? raw : T7_MAX_ST;
            g.ok = true;
            return g;
        }
    }
    return g;
}
}  // namespace

bool conv_ts_applies(int h, int w, int c, int cout, int kh, int kw, int stride, int pad, long long batch) {
    static const bool off = lb::tuning_env("LOWBIT_CONV_NO_TS") != nullptr;  // tuning knob: K7 instead
    if (off) return false;
    const TsGeom g = ts_geom(h, w, c, cout, kh, kw, stride, pad);
    if (!g.ok) return false;
    const long long tpi = (h + 2 * pad - kh + 1 + g.R - 1) / g.R;
    return batch * tpi < 0x7FFFFFFFLL;
}

lowbit_status launch_conv_ts(const int8_t* fm, int batch, int h, int w, int cch, int kh, int kw, int pad,
                             int check_zero, int pad_value, const void* weights, int b_ternary, int cout,
                             int16_t* out, int* zero_flag, cudaStream_t stream) {
    const TsGeom g = ts_geom(h, w, cch, cout, kh, kw, 1, pad);
    if (!g.ok) return lbhost::set_error(LOWBIT_INVALID_ARGUMENT, "conv ts kernel: unsupported shape");
    const int oh = h + 2 * pad - kh + 1, ow = w + 2 * pad - kw + 1;
    const WeightsLayout L(b_ternary, cout, kh * kw * cch);
    TsParams prm{};
    prm.batch = batch;
    prm.h = h;
    prm.w = w;
    prm.oh = oh;
    prm.ow = ow;
    prm.pad = pad;
    prm.kw = kw;
    prm.cblocks = cch / 128;
    prm.P = g.P;
    prm.log2p = g.P == 32 ? 5 : (g.P == 64 ? 6 : 7);
    prm.R = g.R;
    prm.rows_h = g.rows_h;
    prm.tpi = (oh + g.R - 1) / g.R;
    prm.ctiles = batch * prm.tpi;
    prm.cout = cout;
    prm.kblocks = g.kblocks;
    prm.k33 = kh == 3 && kw == 3 && prm.cblocks == 1;
    prm.raw_cb = g.raw_cb;
    prm.f4_cb = g.f4_cb;
    prm.raw_st = g.raw_st;
    prm.f4_st = g.f4_st;
    prm.box_px = g.P < 64 ? g.P : 64;
    prm.box_rows = 64 / prm.box_px;
    prm.pad_word = pad > 0 ? (pad_value > 0 ? 0x01010101u : (pad_value < 0 ? 0xFFFFFFFFu : 0u)) : 0u;
    static const int dbg = lb::tuning_env("LOWBIT_HALO_DEBUG") ? atoi(lb::tuning_env("LOWBIT_HALO_DEBUG")) : 0;
    prm.dbg = dbg;
    prm.mul16 = 16;
    prm.wrows = L.np < 128 ? L.np : 128;
    const uint8_t* wfp4 = static_cast<const uint8_t*>(weights) + L.off_fp4c;  // the converters' channel order (layout.cuh)
    prm.zero_flag = zero_flag;

    CUtensorMap mraw, mout, mw;
    if (!make_map_2d(&mw, wfp4, (uint64_t)L.kp4 / 2, (uint64_t)L.np, (uint64_t)L.kp4 / 2, 64, (uint32_t)prm.wrows,
                     CU_TENSOR_MAP_SWIZZLE_64B))
        return lbhost::set_error(LOWBIT_CUDA_ERROR, "cuTensorMapEncodeTiled failed for the conv filter");
    if (!make_map_nhwc_box(&mraw, fm, batch, h, w, cch, (uint32_t)g.P, (uint32_t)g.rows_h))
        return lbhost::set_error(LOWBIT_CUDA_ERROR, "cuTensorMapEncodeTiled failed for the feature-map halo");
    if (!make_map_conv_out_box(&mout, out, batch, oh, ow, cout, 32, (uint32_t)prm.box_px, (uint32_t)prm.box_rows,
                               CU_TENSOR_MAP_SWIZZLE_64B))
        return lbhost::set_error(LOWBIT_CUDA_ERROR, "cuTensorMapEncodeTiled failed for the conv output");
    const int flags = (prm.pad_word != 0 ? 1 : 0) | (check_zero ? 2 : 0);
    using KernT = decltype(&conv_fp4_ts_kernel<0>);
    const KernT kerns[4] = {conv_fp4_ts_kernel<0>, conv_fp4_ts_kernel<1>, conv_fp4_ts_kernel<2>,
                            conv_fp4_ts_kernel<3>};
    static SmemOptIn attr[4];
    LB_CUDA_TRY(attr[flags].ensure(kerns[flags], T7_SMEM));
    const int ctas = prm.ctiles < num_sms() ? prm.ctiles : num_sms();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(T7_THREADS);
    cfg.dynamicSmemBytes = T7_SMEM;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    LB_CUDA_TRY(cudaLaunchKernelEx(&cfg, kerns[flags], mraw, mout, mw, prm));
    LB_CUDA_TRY(cudaGetLastError());
    return LOWBIT_OK;
}

}  // namespace lb

extern "C" int lowbit_debug_ts_trace(unsigned long long* out1024) {
    return cudaMemcpyFromSymbol(out1024, lb::g_ts_trace, sizeof(unsigned long long) * 1024) != cudaSuccess;
}
extern "C" int lowbit_debug_ts_ctas(unsigned long long* out640) {
    return cudaMemcpyFromSymbol(out640, lb::g_ts_cta, sizeof(unsigned long long) * 640) != cudaSuccess;
}
extern "C" int lowbit_debug_ts_setup(unsigned long long* out640) {
    return cudaMemcpyFromSymbol(out640, lb::g_ts_setup, sizeof(unsigned long long) * 640) != cudaSuccess;
}
extern "C" int lowbit_debug_ts_phases(unsigned long long* out4, int reset) {
    if (cudaMemcpyFromSymbol(out4, lb::g_ts_phase, sizeof(unsigned long long) * 4) != cudaSuccess) return 1;
    if (reset) {
        const unsigned long long init[4] = {~0ull, 0, 0, 0};
        return cudaMemcpyToSymbol(lb::g_ts_phase, init, sizeof init) != cudaSuccess;
    }
    return 0;
}

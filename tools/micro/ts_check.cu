// Microbenchmark + layout check: tcgen05.mma.cta_group::2.kind::mxf4 with the
// A operand in TMEM (converters would write it with tcgen05.st instead of
// st.shared).  Compares against the smem-A MMA and a host reference, then
// measures the issue rate.
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../../paper_2205_09120_b200/csrc/common.cuh"
using namespace lb;

__host__ __device__ inline uint32_t hsh(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
__host__ __device__ inline uint32_t code_of(uint32_t seed, uint32_t row, uint32_t e) {  // element e of row
    const uint32_t r = hsh(seed * 0x9E3779B9u ^ (row * 4096u + e)) % 3u;
    return r == 0 ? 0u : (r == 1 ? 0x2u : 0xAu);
}
__host__ __device__ inline uint8_t byte_of(uint32_t seed, uint32_t row, uint32_t b) {
    return (uint8_t)(code_of(seed, row, 2 * b) | (code_of(seed, row, 2 * b + 1) << 4));
}

__device__ inline void umma_mxf4_pair_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t sf,
                                         uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%5], [%5], p;\n\t}"
                 ::"r"(d), "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc), "r"(sf) : "memory");
}
__device__ inline void tmem_st_x32(uint32_t taddr, const uint32_t (&v)[32]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                 "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                 ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                 "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
                 "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]),
                 "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
                 : "memory");
}

constexpr int NN = 128;  // pair N (each CTA holds 64 B rows)

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    ts_kernel(float* out1, float* out2, int iters, unsigned long long* cyc, int perm) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tslot;
    __shared__ uint64_t bar;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, r = threadIdx.x;
    const uint32_t rank = cluster_ctarank();
    uint8_t* sA = smem;            // 128 rows x 128 B, SW128
    uint8_t* sB = smem + 16384;    // 64 rows x 128 B, SW128
    const uint32_t grow = rank * 128 + r;  // global A row
    for (int b = 0; b < 128; ++b) sA[r * 128 + (((b >> 4) ^ (r & 7)) << 4) + (b & 15)] = byte_of(1, grow, b);
    if (r < NN / 2) {
        const uint32_t brow = rank * (NN / 2) + r;
        for (int b = 0; b < 128; ++b) sB[r * 128 + (((b >> 4) ^ (r & 7)) << 4) + (b & 15)] = byte_of(2, brow, b);
    }
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc_pair<512>(&tslot);
    fence_proxy_async_smem();
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tb = tslot;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    // A into TMEM: lane r, columns 256..287 = the row's 128 bytes (perm selects a candidate byte order)
    {
        uint32_t v[32];
        for (int c = 0; c < 32; ++c) {
            uint32_t w = 0;
            for (int q = 0; q < 4; ++q) w |= (uint32_t)byte_of(1, grow, 4 * c + q) << (8 * q);
            v[c] = w;
        }
        tmem_st_x32(tb + lane_base + 256, v);
        tmem_st_32x32b_x8_fill(tb + lane_base + 288, 0x7F7F7F7Fu);
        tmem_st_wait();
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (rank == 0 && threadIdx.x == 0) {
        const uint32_t id = idesc_mxf4(256, NN);
        const uint32_t a = smem_u32(sA), b = smem_u32(sB);
        for (int kk = 0; kk < 4; ++kk)
            umma_mxf4_pair(tb + 0, umma_desc_k_sw128(a + kk * 32), umma_desc_k_sw128(b + kk * 32), id, tb + 288, tb + 288, kk);
        for (int kk = 0; kk < 4; ++kk)
            umma_mxf4_pair_ts(tb + 128, tb + 256 + kk * 8, umma_desc_k_sw128(b + kk * 32), id, tb + 288, kk);
        umma_commit_pair(&bar, 0x3);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    for (int ch = 0; ch < NN / 16; ++ch) {
        uint32_t v1[16], v2[16];
        tmem_ld_32x32b_x16(tb + lane_base + ch * 16, v1);
        tmem_ld_32x32b_x16(tb + lane_base + 128 + ch * 16, v2);
        tmem_ld_wait();
        for (int j = 0; j < 16; ++j) {
            out1[grow * NN + ch * 16 + j] = __uint_as_float(v1[j]);
            out2[grow * NN + ch * 16 + j] = __uint_as_float(v2[j]);
        }
    }
    // rate: TMEM-A MMAs back to back, N = 256 into cols [0,256)
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (rank == 0 && threadIdx.x == 0 && iters > 0) {
        // perm: 0 = N 256, A cols 256.., D col 0;  1 = N 208, kernel layout (D 0/208, SF 416, A 432 + 16 s)
        //       2 = as 1 plus a commit every 2 MMAs;  3 = N 208, A fixed at col 432
        const uint32_t nn = perm == 0 ? 256 : 208;
        const uint32_t id = idesc_mxf4(256, nn);
        const uint32_t b = smem_u32(sB);
        const long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            uint32_t acol, dcol, sfc;
            if (perm == 0) { acol = 256 + (i & 3) * 8; dcol = 0; sfc = 288; }
            else if (perm == 3) { acol = 432 + (i & 1) * 8; dcol = ((i >> 5) & 1) * 208; sfc = 416; }
            else { acol = 432 + 16 * ((i >> 1) % 5) + (i & 1) * 8; dcol = ((i >> 5) & 1) * 208; sfc = 416; }
            umma_mxf4_pair_ts(tb + dcol, tb + acol, umma_desc_k_sw128(b + (i & 3) * 32), id, tb + sfc, 1);
            if (perm == 2 && (i & 1)) umma_commit_pair(&bar, 0x3);
            if (perm >= 4 && (i & 1)) {  // 4: fence; 5: wait on a completed barrier; 6: both
                if (perm != 4) mbar_wait(&bar, 0);
                if (perm != 5) tc_fence_after();
            }
        }
        umma_commit_pair(&bar, 0x3);
        mbar_wait(&bar, 1);
        cyc[0] = clock64() - t0;
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 0) { tc_fence_after(); tmem_dealloc_pair<512>(tb); }
}

static float dec(uint32_t c) { return c == 0x2 ? 1.f : (c == 0xA ? -1.f : 0.f); }

int main() {
    float *o1, *o2; unsigned long long* cyc;
    cudaMalloc(&o1, 256 * NN * 4); cudaMalloc(&o2, 256 * NN * 4); cudaMalloc(&cyc, 8);
    cudaFuncSetAttribute(ts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    for (int perm = 1; perm < 7; ++perm) {
        ts_kernel<<<2, 128, 65536>>>(o1, o2, 100000, cyc, perm);
        cudaDeviceSynchronize();
        unsigned long long c2; cudaMemcpy(&c2, cyc, 8, cudaMemcpyDeviceToHost);
        printf("perm %d: %.1f cycles/MMA\n", perm, (double)c2 / 100000);
    }
    ts_kernel<<<2, 128, 65536>>>(o1, o2, 100000, cyc, 0);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    std::vector<float> h1(256 * NN), h2(256 * NN);
    cudaMemcpy(h1.data(), o1, h1.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(h2.data(), o2, h2.size() * 4, cudaMemcpyDeviceToHost);
    unsigned long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    int bad1 = 0, bad2 = 0, bad12 = 0;
    for (int r = 0; r < 256; ++r)
        for (int n = 0; n < NN; ++n) {
            float ref = 0;
            for (int k = 0; k < 256; ++k) ref += dec(code_of(1, r, k)) * dec(code_of(2, n, k));
            bad1 += h1[r * NN + n] != ref;
            bad2 += h2[r * NN + n] != ref;
            bad12 += h1[r * NN + n] != h2[r * NN + n];
        }
    printf("smem-A vs host: %d bad; tmem-A vs host: %d bad; smem vs tmem: %d (of %d)\n", bad1, bad2, bad12, 256 * NN);
    printf("sample r0: host %g smemA %g tmemA %g\n", 0.f, h1[0], h2[0]);
    printf("TMEM-A pair MMA N=256: %.1f cycles/MMA\n", (double)c / 100000);
    return 0;
}

// Layout check: can a UMMA K-major SW64 operand start at an arbitrary 64-byte
// row of a swizzled smem region (swizzle computed from absolute address bits,
// as TMA writes it)?  If so a conv's A operand for filter tap (ky,kx) is just
// the halo tile's descriptor advanced by (ky*wp + kx) rows.  Tries start rows
// 0..8 with the descriptor's base-offset field 0 and (addr >> 7) & 7.
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../../paper_2205_09120_b200/csrc/common.cuh"
using namespace lb;

__host__ __device__ inline uint32_t hsh(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
__host__ __device__ inline uint32_t code_of(uint32_t seed, uint32_t row, uint32_t e) {
    const uint32_t r = hsh(seed * 0x9E3779B9u ^ (row * 4096u + e)) % 3u;
    return r == 0 ? 0u : (r == 1 ? 0x2u : 0xAu);
}
__host__ __device__ inline uint8_t byte_of(uint32_t seed, uint32_t row, uint32_t b) {
    return (uint8_t)(code_of(seed, row, 2 * b) | (code_of(seed, row, 2 * b + 1) << 4));
}
__device__ inline uint64_t desc_sw64(uint32_t addr, uint32_t base_off) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFFu);
    d |= (uint64_t)1u << 16;
    d |= (uint64_t)(512u >> 4) << 32;
    d |= (uint64_t)1u << 46;
    d |= (uint64_t)(base_off & 7u) << 49;
    d |= (uint64_t)4u << 61;
    return d;
}

constexpr int NN = 32;       // pair N (16 rows per CTA)
constexpr int HALO = 144;    // A rows held per CTA
constexpr int NOFF = 9;      // start rows tried
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) halo_kernel(float* out, int mode) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tslot;
    __shared__ uint64_t bar;
    const int warp = threadIdx.x >> 5;
    const uint32_t rank = cluster_ctarank();
    uint8_t* sA = smem;              // HALO rows x 64 B, SW64 on absolute address bits
    uint8_t* sB = smem + 16384;      // NN/2 rows x 64 B
    for (int i = threadIdx.x; i < HALO * 64; i += blockDim.x) {
        const int r = i / 64, b = i % 64;
        const uint32_t lin = smem_u32(sA) + r * 64 + b;                  // unswizzled address
        const uint32_t chunk = ((lin >> 4) & 3) ^ ((lin >> 7) & 3);      // SW64: bits [4:5] ^= bits [7:8]
        const uint32_t phys = (lin & ~0x30u) | (chunk << 4);
        smem[phys - smem_u32(smem)] = byte_of(1, rank * 1000 + r, b);
    }
    for (int i = threadIdx.x; i < (NN / 2) * 64; i += blockDim.x) {
        const int r = i / 64, b = i % 64;
        const uint32_t lin = smem_u32(sB) + r * 64 + b;
        const uint32_t chunk = ((lin >> 4) & 3) ^ ((lin >> 7) & 3);
        const uint32_t phys = (lin & ~0x30u) | (chunk << 4);
        smem[phys - smem_u32(smem)] = byte_of(2, rank * (NN / 2) + r, b);
    }
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc_pair<512>(&tslot);
    fence_proxy_async_smem();
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tb = tslot;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    tmem_st_32x32b_x8_fill(tb + lane_base + 480, 0x7F7F7F7Fu);
    tmem_st_wait();
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (rank == 0 && threadIdx.x == 0) {
        const uint32_t id = idesc_mxf4(256, NN);
        for (int o = 0; o < NOFF; ++o) {
            const uint32_t a = smem_u32(sA) + o * 64, b = smem_u32(sB);
            const uint32_t bo = mode == 0 ? 0u : ((a >> 7) & 7u);
            for (int kk = 0; kk < 2; ++kk)
                umma_mxf4_pair(tb + o * NN, desc_sw64(a + kk * 32, bo), desc_sw64(b + kk * 32, 0), id, tb + 480,
                               tb + 480, kk);
        }
        umma_commit_pair(&bar, 0x3);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    const int row = threadIdx.x;
    for (int o = 0; o < NOFF; ++o)
        for (int ch = 0; ch < NN / 16; ++ch) {
            uint32_t v[16];
            tmem_ld_32x32b_x16(tb + lane_base + o * NN + ch * 16, v);
            tmem_ld_wait();
            for (int j = 0; j < 16; ++j)
                out[((size_t)o * 256 + rank * 128 + row) * NN + ch * 16 + j] = __uint_as_float(v[j]);
        }
    tc_fence_before();
    cluster_sync();
    if (warp == 0) { tc_fence_after(); tmem_dealloc_pair<512>(tb); }
}

// MMA issue rate over a halo: 9 taps x 2 MMAs (N = nn) per "tile", A rows
// advanced by ky*wp + kx (mode 1) or all at row 0 (mode 0, aligned).
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    rate_kernel(int tiles, int mode, int wp, int nn, unsigned long long* cyc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tslot;
    __shared__ uint64_t bar;
    const int warp = threadIdx.x >> 5;
    const uint32_t rank = cluster_ctarank();
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x22222222u;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc_pair<512>(&tslot);
    fence_proxy_async_smem();
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tb = tslot;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    tmem_st_32x32b_x8_fill(tb + lane_base + 480, 0x7F7F7F7Fu);
    tmem_st_wait();
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (rank == 0 && threadIdx.x == 0) {
        const uint32_t id = idesc_mxf4(256, nn);
        const uint32_t a = smem_u32(smem), b = smem_u32(smem + 40960);
        const long long t0 = clock64();
        for (int t = 0; t < tiles; ++t)
            for (int kb = 0; kb < 9; ++kb) {
                const uint32_t off = mode ? (uint32_t)((kb / 3) * wp + kb % 3) * 64u : 0u;
                for (int h = 0; h < 2; ++h)
                    umma_mxf4_pair(tb + (t & 1) * 240, desc_sw64(a + off + h * 32, 0), desc_sw64(b + kb * 4096 + h * 32, 0),
                                   id, tb + 480, tb + 480, (kb | h) != 0);
            }
        umma_commit_pair(&bar, 0x3);
        mbar_wait(&bar, 0);
        cyc[0] = clock64() - t0;
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 0) { tc_fence_after(); tmem_dealloc_pair<512>(tb); }
}

static float dec(uint32_t c) { return c == 0x2 ? 1.f : (c == 0xA ? -1.f : 0.f); }

int main() {
    float* o;
    cudaMalloc(&o, (size_t)NOFF * 256 * NN * 4);
    cudaFuncSetAttribute(halo_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    for (int mode = 0; mode < 2; ++mode) {
        cudaMemset(o, 0, (size_t)NOFF * 256 * NN * 4);
        halo_kernel<<<2, 128, 65536>>>(o, mode);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("mode %d: %s\n", mode, cudaGetErrorString(e)); return 1; }
        std::vector<float> h((size_t)NOFF * 256 * NN);
        cudaMemcpy(h.data(), o, h.size() * 4, cudaMemcpyDeviceToHost);
        printf("base-offset %s:", mode ? "(addr>>7)&7" : "0");
        for (int off = 0; off < NOFF; ++off) {
            int bad = 0;
            for (int r = 0; r < 256; ++r)
                for (int n = 0; n < NN; ++n) {
                    const uint32_t arow = (r / 128) * 1000 + (r % 128) + off;
                    float ref = 0;
                    for (int k = 0; k < 128; ++k) ref += dec(code_of(1, arow, k)) * dec(code_of(2, n, k));
                    bad += h[((size_t)off * 256 + r) * NN + n] != ref;
                }
            printf(" off%d=%d", off, bad);
        }
        printf("  (bad of %d)\n", 256 * NN);
    }
    unsigned long long* cyc;
    cudaMalloc(&cyc, 8);
    cudaFuncSetAttribute(rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    for (int nn : {128, 256})
        for (int mode = 0; mode < 2; ++mode) {
            rate_kernel<<<2, 128, 80 * 1024>>>(1000, mode, 58, nn, cyc);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("rate: %s\n", cudaGetErrorString(e)); return 1; }
            unsigned long long c;
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            printf("N=%d %s: %.1f cycles per MMA\n", nn, mode ? "halo offsets" : "aligned", (double)c / 18000);
        }
    return 0;
}

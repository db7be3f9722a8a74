// gemm_grouped.cu — one launch for a batch of small low-bit GeMMs (§8f-3).
//
// The reference bench grid (bench.cpp:196-234; BASELINE.json config 2: 64
// TBN shapes M x N x K in {72..360} x {24..96} x {128..512}) is launch-latency
// bound on a B200: each problem is 0.4-35 MOPs.  Here every problem's
// 64 x 32 output tiles are laid out back to back in one grid; a CTA finds its
// problem with a search over the tile prefix sums in the kernel parameters.
// The arithmetic is K2's (bit-serial LOP3 + POPC, (nz, sign) form); a tile's
// operands (512 depth positions at a time) are staged in shared memory by all
// its threads at once, so the small tiles pay one L2 latency per chunk.
#include <algorithm>
#include <cstdio>
#include <vector>

#include "common.cuh"
#include "layout.cuh"

namespace lb {

constexpr int GR_BM = 64, GR_BN = 32, GR_MAX = 128, GR_KQ = 4;  // GR_KQ: 16-byte quads per staged chunk

struct GroupedProblem {
    const uint8_t* a0;
    const uint8_t* a1;
    long long a_pitch;
    const uint32_t* b_sign;
    const uint32_t* b_nz;
    int m, n, k, kw;
    int16_t* c;
    long long ldc;
};

struct GroupedParams {
    int count;
    int tile_start[GR_MAX + 1];
    GroupedProblem p[GR_MAX];
};

__device__ __forceinline__ uint32_t tail_mask_word(int w, int k) {
    const int bit0 = w * 32;
    return bit0 >= k ? 0u : (k - bit0 >= 32 ? 0xFFFFFFFFu : ((1u << (k - bit0)) - 1u));
}

template <int MODE>
__global__ void __launch_bounds__(128) gemm_grouped_kernel(const __grid_constant__ GroupedParams P) {
    constexpr bool A_TER = MODE != 0, B_TER = MODE == 1;
    const int bid = blockIdx.x;
    int lo = 0, hi = P.count - 1;  // problem q with tile_start[q] <= bid < tile_start[q+1]
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (P.tile_start[mid] <= bid) lo = mid;
        else hi = mid - 1;
    }
    const GroupedProblem& pr = P.p[lo];
    const int t = bid - P.tile_start[lo];
    const int tiles_n = (pr.n + GR_BN - 1) / GR_BN;
    const int tm = t / tiles_n, tn = t - tm * tiles_n;
    const int tx = threadIdx.x & 7, ty = threadIdx.x >> 3;  // 16 x 8 threads, 4 x 4 outputs each
    const int row0 = tm * GR_BM + ty * 4, col0 = tn * GR_BN + tx * 4;
    const int a_words = (int)(pr.a_pitch / 4);
    const int kwords = (pr.k + 31) / 32;

    int acc[4][4] = {};
    int nnz[4] = {0, 0, 0, 0};
    // The tile's operands for up to 512 depth positions (16 words) at a time are staged
    // in shared memory by all threads at once (2-3 16-byte loads each), so a chunk costs
    // one L2 latency instead of one per 4 words; rows padded to 5 quads (bank spread).
    __shared__ uint4 sa0[GR_BM][GR_KQ + 1], sa1[GR_BM][GR_KQ + 1], sbs[GR_BN][GR_KQ + 1], sbn[GR_BN][GR_KQ + 1];
    const int arow0 = tm * GR_BM, bcol0 = tn * GR_BN;
    for (int wc = 0; wc < kwords; wc += 4 * GR_KQ) {
        const int nq = (kwords - wc + 3) / 4 < GR_KQ ? (kwords - wc + 3) / 4 : GR_KQ;  // quads in this chunk
        for (int sl = threadIdx.x; sl < GR_BM * GR_KQ; sl += blockDim.x) {
            const int r = sl / GR_KQ, q = sl - r * GR_KQ;
            if (q >= nq) continue;
            const int w0 = wc + 4 * q;
            uint4 p = make_uint4(0, 0, 0, 0), pq = make_uint4(0, 0, 0, 0);
            if (arow0 + r < pr.m && w0 < a_words) {
                p = __ldg(reinterpret_cast<const uint4*>(pr.a0 + (long long)(arow0 + r) * pr.a_pitch) + (w0 >> 2));
                if (A_TER) pq = __ldg(reinterpret_cast<const uint4*>(pr.a1 + (long long)(arow0 + r) * pr.a_pitch) + (w0 >> 2));
            }
            sa0[r][q] = p;
            if (A_TER) sa1[r][q] = pq;
        }
        for (int sl = threadIdx.x; sl < GR_BN * GR_KQ; sl += blockDim.x) {
            const int c = sl / GR_KQ, q = sl - c * GR_KQ;
            if (q >= nq) continue;
            // B: prepared (nz, sign) words, [np][kw] with np >= round_up(n, 256), kw % 8 == 0
            const long long boff = (long long)(bcol0 + c) * pr.kw + wc + 4 * q;
            sbs[c][q] = __ldg(reinterpret_cast<const uint4*>(pr.b_sign + boff));
            if (B_TER) sbn[c][q] = __ldg(reinterpret_cast<const uint4*>(pr.b_nz + boff));
        }
        __syncthreads();
        for (int q = 0; q < nq; ++q) {
            const int w0 = wc + 4 * q;
            uint32_t as[4][4], an[4][4], bs[4][4], bn[4][4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint4 p = sa0[ty * 4 + i][q];
                const uint4 pq = A_TER ? sa1[ty * 4 + i][q] : make_uint4(0, 0, 0, 0);
                const uint32_t pw[4] = {p.x, p.y, p.z, p.w}, qw[4] = {pq.x, pq.y, pq.z, pq.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t msk = tail_mask_word(w0 + j, pr.k);
                    if (A_TER) {
                        as[i][j] = qw[j] & msk;
                        an[i][j] = (pw[j] | qw[j]) & msk;
                    } else {
                        as[i][j] = pw[j] & msk;
                    }
                }
                const uint4 s4 = sbs[tx * 4 + i][q];
                bs[i][0] = s4.x, bs[i][1] = s4.y, bs[i][2] = s4.z, bs[i][3] = s4.w;
                if (B_TER) {
                    const uint4 n4 = sbn[tx * 4 + i][q];
                    bn[i][0] = n4.x, bn[i][1] = n4.y, bn[i][2] = n4.z, bn[i][3] = n4.w;
                }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    if (MODE == 2) nnz[i] += __popc(an[i][j]);
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        if (MODE == 0) {
                            acc[i][c] += __popc(as[i][j] ^ bs[c][j]);
                        } else if (MODE == 1) {
                            const uint32_t mm = an[i][j] & bn[c][j];
                            acc[i][c] += __popc(mm) - 2 * __popc(mm & (as[i][j] ^ bs[c][j]));
                        } else {
                            acc[i][c] += __popc(an[i][j] & (as[i][j] ^ bs[c][j]));
                        }
                    }
                }
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = row0 + i;
        if (r >= pr.m) continue;
        int16_t* dst = pr.c + (long long)r * pr.ldc + col0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            if (col0 + c >= pr.n) break;
            const int a = acc[i][c];
            dst[c] = (int16_t)(MODE == 0 ? pr.k - 2 * a : (MODE == 1 ? a : nnz[i] - 2 * a));
        }
    }
}

}  // namespace lb

using namespace lb;

extern "C" lowbit_status lowbit_gemm_grouped(int mode, int b_ternary, int count, const lowbit_gemm_problem* problems,
                                             lowbit_stream stream) {
    if (mode < 0 || mode > 2) return lbhost::set_error(LOWBIT_INVALID_ARGUMENT, "grouped: unknown gemm mode");
    if ((mode == LOWBIT_TNN) != (b_ternary != 0))
        return lbhost::set_error(LOWBIT_MODE_MISMATCH, "mode mismatch: tnn requires a ternary right operand, "
                                                       "bnn/tbn a binary one");
    if (count < 0 || (count > 0 && !problems))
        return lbhost::set_error(LOWBIT_INVALID_ARGUMENT, "grouped: bad problem list");
    // deepest problems first: block ids (and with them the SMs the tiles land on)
    // go round the machine in order of decreasing per-tile cost, which spreads
    // the K = 512 tiles of config 2 evenly instead of by problem order
    std::vector<int> order(count);
    for (int i = 0; i < count; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return problems[x].k > problems[y].k; });
    for (int base = 0; base < count; base += GR_MAX) {
        const int cnt = count - base < GR_MAX ? count - base : GR_MAX;
        GroupedParams P;
        P.count = cnt;
        int tiles = 0;
        for (int i = 0; i < cnt; ++i) {
            const lowbit_gemm_problem& q = problems[order[base + i]];
            if (q.m <= 0 || q.n <= 0 || q.k <= 0) return lbhost::set_error(LOWBIT_OUT_OF_BOUNDS, "out of bounds: gemm dims");
            if (q.k > LOWBIT_K_MAX16) {
                char buf[96];
                std::snprintf(buf, sizeof buf, "depth %d exceeds k_max %d", q.k, LOWBIT_K_MAX16);
                return lbhost::set_error(LOWBIT_DEPTH_OVERFLOW, buf, q.k, LOWBIT_K_MAX16);
            }
            if ((mode != LOWBIT_BNN) != (q.a1 != nullptr))
                return lbhost::set_error(LOWBIT_MODE_MISMATCH, "mode mismatch: left operand kind");
            if (!q.a0 || !q.weights || !q.c || (q.a_pitch & 15) || q.a_pitch < (q.k + 7) / 8 || q.ldc < q.n ||
                (reinterpret_cast<uintptr_t>(q.a0) & 15) || (q.a1 && (reinterpret_cast<uintptr_t>(q.a1) & 15)) ||
                (reinterpret_cast<uintptr_t>(q.weights) & 255))
                return lbhost::set_error(LOWBIT_INVALID_ARGUMENT, "grouped: device layout precondition violated");
            const WeightsLayout L(b_ternary, q.n, q.k);
            const uint8_t* wb = static_cast<const uint8_t*>(q.weights);
            P.p[i] = GroupedProblem{q.a0, q.a1, q.a_pitch, reinterpret_cast<const uint32_t*>(wb + L.off_sign),
                                    reinterpret_cast<const uint32_t*>(wb + L.off_nz), q.m, q.n, q.k, L.kw, q.c, q.ldc};
            P.tile_start[i] = tiles;
            tiles += ((q.m + GR_BM - 1) / GR_BM) * ((q.n + GR_BN - 1) / GR_BN);
        }
        P.tile_start[cnt] = tiles;
        if (tiles == 0) continue;
        cudaStream_t s = (cudaStream_t)stream;
        if (mode == 0) gemm_grouped_kernel<0><<<tiles, 128, 0, s>>>(P);
        else if (mode == 1) gemm_grouped_kernel<1><<<tiles, 128, 0, s>>>(P);
        else gemm_grouped_kernel<2><<<tiles, 128, 0, s>>>(P);
        LB_CUDA_TRY(cudaGetLastError());
    }
    return LOWBIT_OK;
}

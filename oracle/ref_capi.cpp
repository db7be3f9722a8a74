// ref_capi.cpp — a C entry layer over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles the reference sources
// where they lie (/root/reference/proj/src/*.cpp, with the reference's own
// -O3 and no -march) together with this file into oracle/_ref/liblowbit_ref.so.
// Python loads it with ctypes to (a) pin the C restatement in
// oracle/lowbit_oracle.c, (b) generate tests/golden/ fixtures, and (c) time
// the reference CPU path for bench.py's cpu_baseline / --impl reference legs.
// Nothing here is part of the product.
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "lowbit/conv.hpp"
#include "lowbit/gemm.hpp"
#include "lowbit/kernels.hpp"
#include "lowbit/pack.hpp"

using namespace lowbit;

namespace {

// Status codes match include/lowbit_cuda.h.
template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ZeroInBinaryInput&) {
        return 2;
    } catch (const InvalidCode&) {
        return 3;
    } catch (const OutOfBounds&) {
        return 4;
    } catch (const DepthOverflow&) {
        return 5;
    } catch (const ModeMismatch&) {
        return 6;
    } catch (const ChannelOverflow&) {
        return 7;
    } catch (const EmptyOutput&) {
        return 8;
    } catch (const Error&) {
        return 1;
    } catch (...) {
        return 99;
    }
}

SignMatrix sign_from(const int8_t* v, int rows, int cols, bool binary) {
    SignMatrix m(rows, cols, binary ? Mode::binary : Mode::ternary);
    std::memcpy(m.values.data(), v, (size_t)rows * cols);
    return m;
}

BinaryPackedMatrix bin_from(const uint8_t* p, int rows, int cols) {
    BinaryPackedMatrix m;
    m.rows = rows;
    m.cols = cols;
    m.stride_bits = (cols + 7) & ~7;
    m.plane.assign(p, p + (size_t)rows * m.stride_bytes());
    return m;
}

TernaryPackedMatrix ter_from(const uint8_t* p, const uint8_t* n, int rows, int cols) {
    TernaryPackedMatrix m;
    m.rows = rows;
    m.cols = cols;
    m.stride_bits = (cols + 7) & ~7;
    size_t bytes = (size_t)rows * m.stride_bytes();
    m.plane_plus.assign(p, p + bytes);
    m.plane_minus.assign(n, n + bytes);
    return m;
}

PackedB packed_b_from(int b_ternary, const uint8_t* b0, const uint8_t* b1, int k, int n) {
    return b_ternary ? pack_b(ter_from(b0, b1, k, n)) : pack_b(bin_from(b0, k, n));
}

}  // namespace

extern "C" {

int ref_encode(int ternary, const int8_t* v, int rows, int cols, uint8_t* p0, uint8_t* p1) {
    return guarded([&] {
        if (ternary) {
            auto t = encode_ternary(sign_from(v, rows, cols, false));
            std::memcpy(p0, t.plane_plus.data(), t.plane_plus.size());
            std::memcpy(p1, t.plane_minus.data(), t.plane_minus.size());
        } else {
            auto b = encode_binary(sign_from(v, rows, cols, true));
            std::memcpy(p0, b.plane.data(), b.plane.size());
        }
    });
}

// pack_{a,b}_{binary,ternary}; block_mode follows BlockMode order.
int ref_pack_block(int block_mode, const uint8_t* p0, const uint8_t* p1, int rows, int cols, int start,
                   int depth_start, int k_eff, uint8_t* out, int* lanes, int* out_bytes) {
    return guarded([&] {
        PackedBlock blk;
        switch (block_mode) {
            case 0: blk = pack_a_binary(bin_from(p0, rows, cols), start, depth_start, k_eff); break;
            case 1: blk = pack_b_binary(bin_from(p0, rows, cols), start, depth_start, k_eff); break;
            case 2: blk = pack_a_ternary(ter_from(p0, p1, rows, cols), start, depth_start, k_eff); break;
            default: blk = pack_b_ternary(ter_from(p0, p1, rows, cols), start, depth_start, k_eff); break;
        }
        *lanes = blk.lanes;
        *out_bytes = (int)blk.buffer.size();
        std::memcpy(out, blk.buffer.data(), blk.buffer.size());
    });
}

// pack_b over a K x N plane (or plane pair); panels concatenated.
int ref_pack_b(int b_ternary, const uint8_t* b0, const uint8_t* b1, int k, int n, uint8_t* out) {
    return guarded([&] {
        PackedB pb = packed_b_from(b_ternary, b0, b1, k, n);
        size_t off = 0;
        for (auto& p : pb.panels) {
            std::memcpy(out + off, p.buffer.data(), p.buffer.size());
            off += p.buffer.size();
        }
    });
}

// Full reference path from encoded planes: pack_b + gemm_lowbit.
int ref_gemm_lowbit(int mode, int a_ternary, const uint8_t* a0, const uint8_t* a1, int a_rows, int a_cols,
                    int b_ternary, const uint8_t* b0, const uint8_t* b1, int b_rows, int b_cols, int m, int n,
                    int k, int k_blk, int16_t* c) {
    return guarded([&] {
        PackedB pb = packed_b_from(b_ternary, b0, b1, b_rows, b_cols);
        GemmDims dims{m, n, k};
        GemmConfig cfg{k_blk};
        Int16Matrix r = a_ternary ? gemm_lowbit((GemmMode)mode, ter_from(a0, a1, a_rows, a_cols), pb, dims, cfg)
                                  : gemm_lowbit((GemmMode)mode, bin_from(a0, a_rows, a_cols), pb, dims, cfg);
        std::memcpy(c, r.values.data(), r.values.size() * sizeof(int16_t));
    });
}

int ref_reference_gemm_int(const int8_t* a, const int8_t* b, int m, int n, int k, int32_t* c) {
    return guarded([&] {
        auto r = reference_gemm_int(sign_from(a, m, k, false), sign_from(b, k, n, false));
        std::memcpy(c, r.values.data(), r.values.size() * sizeof(int32_t));
    });
}

int ref_dot_binary(const uint8_t* a, const uint8_t* b, int nbytes, int k, int16_t* out) {
    return guarded([&] {
        *out = dot_binary(std::span<const uint8_t>(a, nbytes), std::span<const uint8_t>(b, nbytes), k);
    });
}

int ref_conv2d_lowbit(int mode, const int8_t* fm, int h, int w, int ch, int fm_binary, const int8_t* wts,
                      int w_rows, int w_cols, int w_binary, int kh, int kw, int stride, int padding, int cout,
                      int binary_pad_value, int32_t* out, int* out_h, int* out_w) {
    return guarded([&] {
        FeatureMap f(h, w, ch, fm_binary ? Mode::binary : Mode::ternary);
        std::memcpy(f.values.data(), fm, (size_t)h * w * ch);
        ConvSpec spec{kh, kw, stride, padding, cout, binary_pad_value};
        auto r = conv2d_lowbit((GemmMode)mode, f, sign_from(wts, w_rows, w_cols, w_binary), spec);
        *out_h = r.height;
        *out_w = r.width;
        std::memcpy(out, r.values.data(), r.values.size() * sizeof(int32_t));
    });
}

long long ref_k_max(int p, int q) { return k_max(p, q); }
long long ref_c_in_max(long long km, int kh, int kw) { return c_in_max(km, kh, kw); }

// ---------------------------------------------------------------------------
// Timing harness for the CPU baseline: the reference gemm_lowbit on T
// contiguous row shards, one std::thread each (the library is pure and its
// tile scratch is thread_local, kernels.cpp:23).  Encoding and pack_b happen
// in ref_bench_prepare, outside the timed call, as in bench.cpp:40-68.
// ---------------------------------------------------------------------------
struct RefBench {
    int mode = 0, a_ternary = 0, n = 0, k = 0;
    PackedB pb;
    std::vector<BinaryPackedMatrix> a_bin;
    std::vector<TernaryPackedMatrix> a_ter;
    std::vector<SignMatrix> a_i8;  // "from int8 A": encode_* runs inside the timed call
    std::vector<int> row0;
};

void* ref_bench_prepare(int mode, int a_ternary, const uint8_t* a0, const uint8_t* a1, int m, int k,
                        int b_ternary, const uint8_t* b0, const uint8_t* b1, int n, int threads) {
    auto* rb = new RefBench;
    rb->mode = mode;
    rb->a_ternary = a_ternary;
    rb->n = n;
    rb->k = k;
    rb->pb = packed_b_from(b_ternary, b0, b1, k, n);
    int sb = (k + 7) / 8;
    if (threads < 1) threads = 1;
    if (threads > m) threads = m;
    for (int t = 0; t < threads; ++t) {
        int r0 = (int)((long long)m * t / threads), r1 = (int)((long long)m * (t + 1) / threads);
        rb->row0.push_back(r0);
        const uint8_t* p0 = a0 + (size_t)r0 * sb;
        if (a_ternary) rb->a_ter.push_back(ter_from(p0, a1 + (size_t)r0 * sb, r1 - r0, k));
        else rb->a_bin.push_back(bin_from(p0, r1 - r0, k));
    }
    return rb;
}

// "From int8 A" (BASELINE.md §2 second line): the shards keep the int8 sign
// matrix and ref_bench_run encodes each one (core.cpp:13-58) before its
// gemm_lowbit.  pack_b stays outside, as in bench.cpp:58.
void* ref_bench_prepare_i8(int mode, const int8_t* a, int m, int k, int b_ternary, const uint8_t* b0,
                           const uint8_t* b1, int n, int threads) {
    auto* rb = new RefBench;
    rb->mode = mode;
    rb->a_ternary = mode != 0;
    rb->n = n;
    rb->k = k;
    rb->pb = packed_b_from(b_ternary, b0, b1, k, n);
    if (threads < 1) threads = 1;
    if (threads > m) threads = m;
    for (int t = 0; t < threads; ++t) {
        int r0 = (int)((long long)m * t / threads), r1 = (int)((long long)m * (t + 1) / threads);
        rb->row0.push_back(r0);
        rb->a_i8.push_back(sign_from(a + (size_t)r0 * k, r1 - r0, k, mode == 0));
    }
    return rb;
}

// Runs one full gemm over all shards; writes C (row-major m x n) if c != NULL.
int ref_bench_run(void* h, int16_t* c) {
    auto* rb = static_cast<RefBench*>(h);
    size_t shards = rb->row0.size();
    std::vector<int> st(shards, 0);
    std::vector<std::thread> pool;
    for (size_t t = 0; t < shards; ++t)
        pool.emplace_back([&, t] {
            st[t] = guarded([&] {
                Int16Matrix r;
                if (!rb->a_i8.empty()) {
                    const SignMatrix& a = rb->a_i8[t];
                    GemmDims dims{a.rows, rb->n, rb->k};
                    r = rb->a_ternary ? gemm_lowbit((GemmMode)rb->mode, encode_ternary(a), rb->pb, dims)
                                      : gemm_lowbit((GemmMode)rb->mode, encode_binary(a), rb->pb, dims);
                } else {
                    int rows = rb->a_ternary ? rb->a_ter[t].rows : rb->a_bin[t].rows;
                    GemmDims dims{rows, rb->n, rb->k};
                    r = rb->a_ternary ? gemm_lowbit((GemmMode)rb->mode, rb->a_ter[t], rb->pb, dims)
                                      : gemm_lowbit((GemmMode)rb->mode, rb->a_bin[t], rb->pb, dims);
                }
                if (c) std::memcpy(c + (size_t)rb->row0[t] * rb->n, r.values.data(), r.values.size() * 2);
            });
        });
    for (auto& th : pool) th.join();
    for (int s : st)
        if (s) return s;
    return 0;
}

void ref_bench_free(void* h) { delete static_cast<RefBench*>(h); }

// Convolution baseline: `images` single-image
// conv2d_lowbit calls (conv.cpp:33-59: im2col + encode + pack_b + gemm_lowbit,
// all timed, as a caller of the reference pays them), images dealt to
// `threads` std::threads.  fm: images x h x w x ch int8 (NHWC).
int ref_bench_conv(int mode, const int8_t* fm, int images, int h, int w, int ch, int fm_binary, const int8_t* wts,
                   int w_rows, int w_cols, int w_binary, int kh, int kw, int stride, int padding, int threads) {
    if (threads < 1) threads = 1;
    if (threads > images) threads = images;
    std::vector<FeatureMap> maps;
    for (int i = 0; i < images; ++i) {
        FeatureMap f(h, w, ch, fm_binary ? Mode::binary : Mode::ternary);
        std::memcpy(f.values.data(), fm + (size_t)i * h * w * ch, (size_t)h * w * ch);
        maps.push_back(std::move(f));
    }
    SignMatrix wm = sign_from(wts, w_rows, w_cols, w_binary);
    ConvSpec spec{kh, kw, stride, padding, w_cols, 1};
    std::vector<int> st(threads, 0);
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
        pool.emplace_back([&, t] {
            for (int i = t; i < images && !st[t]; i += threads)
                st[t] = guarded([&] { (void)conv2d_lowbit((GemmMode)mode, maps[i], wm, spec); });
        });
    for (auto& th : pool) th.join();
    for (int x : st)
        if (x) return x;
    return 0;
}

}  // extern "C"

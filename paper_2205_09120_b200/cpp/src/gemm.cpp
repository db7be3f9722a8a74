// gemm.cpp — drop-in GeMM layer.  pack_b and gemm_lowbit run on the B200
// through the C ABI; the float / zero-point baselines, overflow calculators
// and the scalar oracle are host code with the reference semantics
// (/root/reference/proj/src/gemm.cpp, cited per function).
#include <cstring>

#include "device.hpp"
#include "lowbit/gemm.hpp"

namespace lowbit {

namespace {

// gemm.cpp:9-12
void require_kblk(const GemmConfig& cfg) {
    if (cfg.k_blk < 8 || cfg.k_blk % 8 != 0) throw Error("k_blk must be a positive multiple of 8");
}

int min_int(int a, int b) { return a < b ? a : b; }

// PackedB -> the contiguous panel byte stream the C ABI consumes.
std::vector<std::uint8_t> panel_stream(const PackedB& pb, bool ternary) {
    const size_t group = ternary ? 16 : 8;
    const size_t db = pb.k > 0 ? static_cast<size_t>(pb.k + 7) / 8 : 0;
    const size_t npan = pb.n > 0 ? static_cast<size_t>(pb.n + 7) / 8 : 0;
    std::vector<std::uint8_t> s(npan * group * db);
    if (pb.panels.size() != npan) throw OutOfBounds("packed right operand layout");
    for (size_t p = 0; p < npan; ++p) {
        if (pb.panels[p].buffer.size() != group * db) throw OutOfBounds("packed right operand layout");
        std::memcpy(s.data() + p * group * db, pb.panels[p].buffer.data(), group * db);
    }
    return s;
}

PackedB split_panels(const std::vector<std::uint8_t>& stream, BlockMode mode, int n, int k) {
    PackedB pb;
    pb.mode = mode;
    pb.n = n;
    pb.k = k;
    const int group = block_group_bytes(mode), db = (k + 7) / 8;
    for (int c = 0, p = 0; c < n; c += 8, ++p) {
        PackedBlock blk;
        blk.mode = mode;
        blk.lanes = min_int(8, n - c);
        blk.depth_bytes = db;
        const std::uint8_t* src = stream.data() + static_cast<size_t>(p) * group * db;
        blk.buffer.assign(src, src + static_cast<size_t>(group) * db);
        pb.panels.push_back(std::move(blk));
    }
    return pb;
}

Int16Matrix run_gemm(GemmMode mode, const std::uint8_t* a0, const std::uint8_t* a1, int a_rows, int a_cols,
                     const PackedB& pb, const GemmDims& dims, const GemmConfig& cfg) {
    // A PackedB whose blocks are not B-layouts fails the reference's mode
    // check (gemm.cpp:82, 96-99) right after check_cfg.
    if (pb.mode != BlockMode::bnn_b && pb.mode != BlockMode::tnn_b) {
        require_kblk(cfg);
        throw ModeMismatch("right operand is not a packed B matrix");
    }
    const bool b_ternary = pb.mode == BlockMode::tnn_b;
    Int16Matrix c;
    c.rows = dims.m;
    c.cols = dims.n;
    const bool shape_ok = dims.m > 0 && dims.n > 0 && dims.k > 0 && pb.n == dims.n && pb.k == dims.k;
    std::vector<std::uint8_t> stream;
    if (shape_ok) {
        stream = panel_stream(pb, b_ternary);
        c.values.assign(static_cast<size_t>(dims.m) * dims.n, 0);
    }
    // Validation (check_cfg -> mode -> check_dims, gemm.cpp:81-84, 94-100)
    // happens inside the C ABI before any device work.
    detail::check(lowbit_gemm_lowbit_host(static_cast<int>(mode), a0, a1, a_rows, a_cols,
                                          stream.empty() ? nullptr : stream.data(), b_ternary ? 1 : 0, pb.n, pb.k,
                                          dims.m, dims.n, dims.k, cfg.k_blk,
                                          c.values.empty() ? nullptr : c.values.data(), LOWBIT_KERNEL_AUTO, nullptr),
                  "gemm_lowbit");
    return c;
}

}  // namespace

// gemm.cpp:59-67
PackedB pack_b(const BinaryPackedMatrix& b) {
    if (b.cols > 0 && b.rows < 1) throw OutOfBounds("depth range");  // pack.cpp:10
    std::vector<std::uint8_t> stream(lowbit_packed_b_bytes(0, b.cols, b.rows));
    if (!stream.empty())
        detail::check(lowbit_pack_b_host(0, b.plane.data(), nullptr, b.rows, b.cols, stream.data(), nullptr), "pack_b");
    return split_panels(stream, BlockMode::bnn_b, b.cols, b.rows);
}

// gemm.cpp:69-77
PackedB pack_b(const TernaryPackedMatrix& b) {
    if (b.cols > 0 && b.rows < 1) throw OutOfBounds("depth range");
    std::vector<std::uint8_t> stream(lowbit_packed_b_bytes(1, b.cols, b.rows));
    if (!stream.empty())
        detail::check(lowbit_pack_b_host(1, b.plane_plus.data(), b.plane_minus.data(), b.rows, b.cols, stream.data(),
                                         nullptr),
                      "pack_b");
    return split_panels(stream, BlockMode::tnn_b, b.cols, b.rows);
}

// gemm.cpp:79-90
Int16Matrix gemm_lowbit(GemmMode mode, const BinaryPackedMatrix& a, const PackedB& packed_b, const GemmDims& dims,
                        const GemmConfig& cfg) {
    return run_gemm(mode, a.plane.data(), nullptr, a.rows, a.cols, packed_b, dims, cfg);
}

// gemm.cpp:92-112
Int16Matrix gemm_lowbit(GemmMode mode, const TernaryPackedMatrix& a, const PackedB& packed_b, const GemmDims& dims,
                        const GemmConfig& cfg) {
    // a1 != NULL marks a ternary left operand for the C ABI even when empty
    static const std::uint8_t empty_plane[16] = {};
    const std::uint8_t* minus = a.plane_minus.empty() ? empty_plane : a.plane_minus.data();
    return run_gemm(mode, a.plane_plus.data(), minus, a.rows, a.cols, packed_b, dims, cfg);
}

// gemm.cpp:114-136: sliced blocked float GeMM (host baseline).
FloatMatrix gemm_f32(const FloatMatrix& a, const FloatMatrix& b, const GemmConfig& cfg) {
    require_kblk(cfg);
    if (a.cols != b.rows) throw OutOfBounds("f32 operand shapes");
    FloatMatrix c(a.rows, b.cols);
    for (int d0 = 0; d0 < a.cols; d0 += cfg.k_blk) {
        const int d1 = min_int(a.cols, d0 + cfg.k_blk);
        for (int r0 = 0; r0 < a.rows; r0 += GemmConfig::m_mk)
            for (int c0 = 0; c0 < b.cols; c0 += GemmConfig::n_mk) {
                const int rm = min_int(GemmConfig::m_mk, a.rows - r0), cn = min_int(GemmConfig::n_mk, b.cols - c0);
                float tile[GemmConfig::m_mk][GemmConfig::n_mk] = {};
                for (int t = d0; t < d1; ++t)
                    for (int i = 0; i < rm; ++i) {
                        const float av = a.at(r0 + i, t);
                        for (int j = 0; j < cn; ++j) tile[i][j] += av * b.at(t, c0 + j);
                    }
                for (int i = 0; i < rm; ++i)
                    for (int j = 0; j < cn; ++j) c.at(r0 + i, c0 + j) += tile[i][j];
            }
    }
    return c;
}

// gemm.cpp:138-152
QuantizedGemmInputs make_quantized_inputs(Int32Matrix a_hat, Int32Matrix b_hat, QuantParams qa, QuantParams qb) {
    QuantizedGemmInputs in;
    in.a_row_sums.assign(a_hat.rows, 0);
    in.b_col_sums.assign(b_hat.cols, 0);
    for (int i = 0; i < a_hat.rows; ++i)
        for (int t = 0; t < a_hat.cols; ++t) in.a_row_sums[i] += a_hat.at(i, t);
    for (int t = 0; t < b_hat.rows; ++t)
        for (int j = 0; j < b_hat.cols; ++j) in.b_col_sums[j] += b_hat.at(t, j);
    in.a_hat = std::move(a_hat);
    in.b_hat = std::move(b_hat);
    in.qa = qa;
    in.qb = qb;
    return in;
}

// gemm.cpp:154-196, Eq. 3: sum (a-za)(b-zb) = sum ab - zb*rowsum(a) - za*colsum(b) + k*za*zb,
// first term accumulated in uint32 under the k <= k_max(p, 32) contract.
QuantizedGemmResult gemm_quantized(const QuantizedGemmInputs& in, const GemmDims& dims) {
    const Int32Matrix& a = in.a_hat;
    const Int32Matrix& b = in.b_hat;
    if (a.rows != dims.m || a.cols != dims.k || b.rows != dims.k || b.cols != dims.n)
        throw OutOfBounds("quantized operand shapes");
    const int p = in.qa.bits > in.qb.bits ? in.qa.bits : in.qb.bits;
    const std::int64_t limit = k_max(p, 32);
    if (dims.k > limit) throw DepthOverflow(dims.k, static_cast<long>(limit));
    QuantizedGemmResult res;
    res.scale = in.qa.scale * in.qb.scale;
    res.c_tilde.rows = dims.m;
    res.c_tilde.cols = dims.n;
    res.c_tilde.values.assign(static_cast<size_t>(dims.m) * dims.n, 0);
    const std::int64_t za = in.qa.zero_point, zb = in.qb.zero_point;
    const std::int64_t kzz = static_cast<std::int64_t>(dims.k) * za * zb;
    for (int i = 0; i < dims.m; ++i)
        for (int j = 0; j < dims.n; ++j) {
            std::uint32_t dot = 0;
            for (int t = 0; t < dims.k; ++t)
                dot += static_cast<std::uint32_t>(a.at(i, t)) * static_cast<std::uint32_t>(b.at(t, j));
            const std::int64_t v = static_cast<std::int64_t>(dot) - zb * in.a_row_sums[i] - za * in.b_col_sums[j] + kzz;
            res.c_tilde.at(i, j) = static_cast<std::int32_t>(v);
        }
    return res;
}

// gemm.cpp:198-208
std::int64_t k_max(int p, int q) {
    const std::uint64_t acc = q >= 64 ? ~0ull : ((1ull << q) - 1);
    const std::uint64_t prod = ((1ull << p) - 1) * ((1ull << p) - 1);
    return static_cast<std::int64_t>(acc / prod);
}

std::int64_t k_max_sign(int q) { return static_cast<std::int64_t>((1ull << (q - 1)) - 1); }

std::int64_t c_in_max(std::int64_t km, int kernel_h, int kernel_w) {
    return km / (static_cast<std::int64_t>(kernel_h) * kernel_w);
}

// gemm.cpp:210-223
Int32Matrix reference_gemm_int(const SignMatrix& a, const SignMatrix& b) {
    if (a.cols != b.rows) throw OutOfBounds("reference gemm shapes");
    Int32Matrix c;
    c.rows = a.rows;
    c.cols = b.cols;
    c.values.assign(static_cast<size_t>(a.rows) * b.cols, 0);
    for (int i = 0; i < a.rows; ++i)
        for (int t = 0; t < a.cols; ++t) {
            const int av = a.at(i, t);
            if (!av) continue;
            for (int j = 0; j < b.cols; ++j) c.at(i, j) += av * b.at(t, j);
        }
    return c;
}

}  // namespace lowbit

/*
 * lowbit_cuda.h — C ABI of the B200 (sm_100a) low-bit GeMM library
 * (paper_2205_09120_b200/liblowbit_cuda.so).
 *
 * This is the drop-in boundary for the reference library `lowbit`
 * (/root/reference/proj, namespace lowbit, headers include/lowbit/<name>.hpp).
 * Every entry point names the reference interface it replaces.  Plain C:
 * pointers, sizes and status codes only; no C++ or torch types.  The C++
 * drop-in (paper_2205_09120_b200/cpp, namespace lowbit) and the Python
 * bindings sit on top of these symbols; INTEGRATION.md shows how a
 * maintainer binds them.
 *
 * Conventions
 *  - Device-pointer entry points are stream-ordered on `stream` (a
 *    cudaStream_t; NULL = legacy default stream), do not synchronise and do
 *    not allocate.  They are safe to call from several host threads on
 *    distinct streams.
 *  - Bit planes use the reference encoding (core.hpp:3-10): LSB-first bytes,
 *    binary +1 -> 0 / -1 -> 1, ternary plus/minus planes.  On the device a
 *    plane row starts every `pitch` bytes; pitch must be a multiple of 16
 *    and >= ceil(cols/8); bytes past ceil(cols/8) must be zero
 *    (lowbit_encode writes them so).  lowbit_plane_pitch() gives the
 *    canonical pitch.
 *  - Errors: the reference throws lowbit::Error subclasses (errors.hpp:8-45)
 *    in the order check_cfg -> mode -> check_dims (gemm.cpp:81-84, 94-100).
 *    Here each call returns the matching lowbit_status, checked in the same
 *    order, and records a message plus detail values (e.g. k and k_max for
 *    LOWBIT_DEPTH_OVERFLOW) readable with lowbit_last_error*().
 */
#ifndef LOWBIT_CUDA_H
#define LOWBIT_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LOWBIT_ABI_VERSION 1
#define LOWBIT_K_MAX16 32767 /* kernels.hpp:24 kMaxDepth16 */

typedef enum lowbit_status {
    LOWBIT_OK = 0,
    LOWBIT_ERROR = 1,              /* lowbit::Error (e.g. bad k_blk, gemm.cpp:9-12) */
    LOWBIT_ZERO_IN_BINARY = 2,     /* lowbit::ZeroInBinaryInput (core.cpp:23) */
    LOWBIT_INVALID_CODE = 3,       /* lowbit::InvalidCode */
    LOWBIT_OUT_OF_BOUNDS = 4,      /* lowbit::OutOfBounds */
    LOWBIT_DEPTH_OVERFLOW = 5,     /* lowbit::DepthOverflow(k, k_max) */
    LOWBIT_MODE_MISMATCH = 6,      /* lowbit::ModeMismatch */
    LOWBIT_CHANNEL_OVERFLOW = 7,   /* lowbit::ChannelOverflow(c_in, c_in_max) */
    LOWBIT_EMPTY_OUTPUT = 8,       /* lowbit::EmptyOutput */
    LOWBIT_CUDA_ERROR = 9,         /* CUDA runtime/driver failure (no reference analogue) */
    LOWBIT_INVALID_ARGUMENT = 10,  /* device-layout precondition violated (pitch, alignment, NULL) */
    LOWBIT_NO_DEVICE = 11          /* no sm_100 device visible: the library has no CPU fallback */
} lowbit_status;

/* gemm.hpp:24 GemmMode, same order. */
typedef enum lowbit_gemm_mode { LOWBIT_BNN = 0, LOWBIT_TNN = 1, LOWBIT_TBN = 2 } lowbit_gemm_mode;

/* Kernel choice for lowbit_gemm.  AUTO consults the static per-shape table
 * (lowbit_select_kernel: the int8 kernel for launch-bound shapes under ~1 GOP,
 * else the fp4 one; NIBBLES planes always run the fp4 kernel); the others
 * force one kernel (tests, profiling). */
typedef enum lowbit_kernel {
    LOWBIT_KERNEL_AUTO = 0,
    LOWBIT_KERNEL_BITSERIAL = 1,  /* K2: LOP3 + POPC, int32 registers */
    LOWBIT_KERNEL_TENSOR = 2,     /* tensor cores: K5 (tcgen05.mma kind::mxf4, packed e2m1, CTA pairs)
                                     for REFERENCE and NIBBLES planes; K3 (kind::i8) for LANES planes */
    LOWBIT_KERNEL_TENSOR_1CTA = 3, /* K3 forced to the single-CTA (cta_group::1) variant */
    LOWBIT_KERNEL_TENSOR_I8 = 4   /* K3 (kind::i8, int32 TMEM accumulators; CTA pairs when m > 128) */
} lowbit_kernel;

typedef void* lowbit_stream; /* cudaStream_t */

/* Device plane layouts for the A operand.
 * REFERENCE: the reference encoding, element t of a row at bit t%8 of byte
 *            t/8 (core.hpp:3-10) — what the C++ API exchanges.
 * LANES:     the B200 layout written by lowbit_encode_ex: within each 32-bit
 *            word (32 consecutive elements) element j sits at bit
 *            8*(j%4) + j/4, so the tensor-core kernel turns a word into int8
 *            with one shift + mask per 4 elements.  A per-word bit
 *            permutation: popcounts, pitch and padding rules are unchanged. */
/* NIBBLES:  element j of each 32-bit word at bit 4*(j%8) + j/8, so
 *            (w >> q) & 0x11111111 holds elements 8q..8q+7 one per nibble: the
 *            fp4 (e2m1, kind::mxf4) tensor-core path builds its packed operand
 *            with one shift + mask + multiply-add per 8 elements. */
typedef enum lowbit_layout {
    LOWBIT_LAYOUT_REFERENCE = 0,
    LOWBIT_LAYOUT_LANES = 1,
    LOWBIT_LAYOUT_NIBBLES = 2
} lowbit_layout;

/* ---- library / errors --------------------------------------------------- */
int lowbit_abi_version(void);
const char* lowbit_status_string(int status);
/* Message of the last failing call on this host thread ("" if none). */
const char* lowbit_last_error(void);
/* Detail values of the last failure: DEPTH_OVERFLOW -> (k, k_max),
 * CHANNEL_OVERFLOW -> (c_in, c_in_max); otherwise (0, 0). */
void lowbit_last_error_values(long long* v0, long long* v1);
/* LOWBIT_OK when an sm_100 device is present, else LOWBIT_NO_DEVICE. */
lowbit_status lowbit_device_check(void);

/* ---- layouts ------------------------------------------------------------ */
/* Canonical device pitch for a plane with `cols` logical columns:
 * round_up(ceil(cols/8), 16) bytes. */
long long lowbit_plane_pitch(int cols);

/* ---- K1: encode (core.hpp:63 encode_binary, core.hpp:66 encode_ternary) --
 * values: rows x cols int8, row stride ld (elements), device.
 * ternary=0: plane0 <- binary plane (-1 -> 1); a 0 element sets *zero_flag
 *            to 1 (the caller raises ZeroInBinaryInput, core.cpp:23).
 * ternary=1: plane0 <- plus plane, plane1 <- minus plane.
 * Writes whole rows of `pitch` bytes (padding bytes zero).  zero_flag may be
 * NULL for ternary; it is only ever set, never cleared. */
lowbit_status lowbit_encode(int ternary, const int8_t* values, int rows, int cols, long long ld, uint8_t* plane0,
                            uint8_t* plane1, long long pitch, int* zero_flag, lowbit_stream stream);

/* encode with an explicit A layout (lowbit_layout). */
lowbit_status lowbit_encode_ex(int ternary, int layout, const int8_t* values, int rows, int cols, long long ld,
                               uint8_t* plane0, uint8_t* plane1, long long pitch, int* zero_flag,
                               lowbit_stream stream);

/* ---- K1b: pack_b (gemm.hpp:75-76; pack.cpp:64-127) ------------------------
 * b0/b1: K x N plane(s) packed along N (the reference B layout), row pitch
 * `pitch` bytes (any pitch >= ceil(n/8) here).  panels: the reference
 * PackedB byte stream — ceil(n/8) panels of group*ceil(k/8) bytes each,
 * group 8 (bnn_b) or 16 (tnn_b), concatenated in panel order. */
size_t lowbit_packed_b_bytes(int ternary, int n, int k);
lowbit_status lowbit_pack_b(int ternary, const uint8_t* b0, const uint8_t* b1, int k, int n, long long pitch,
                            uint8_t* panels, lowbit_stream stream);

/* ---- weight preparation (no reference analogue: the GPU operand of PackedB)
 * Turns PackedB panels into the device operand read by both GeMM kernels:
 * an int8 K-major copy (tensor-core path) and K-major (nonzero, sign) bit
 * words (bit-serial path).  Done once per weight matrix. */
size_t lowbit_weights_bytes(int ternary, int n, int k);
lowbit_status lowbit_prepare_weights(int ternary, const uint8_t* panels, int n, int k, void* weights,
                                     lowbit_stream stream);

/* ---- K2/K3: gemm_lowbit (gemm.hpp:78-81; gemm.cpp:79-112) ----------------
 * mode: lowbit_gemm_mode.  a0 (+a1 for ternary A; a1 == NULL means a binary
 * A) are a_rows x a_cols planes with pitch a_pitch.  weights: the output of
 * lowbit_prepare_weights for a b_n x b_k PackedB of kind b_ternary.  dims
 * (m, n, k) and k_blk are validated exactly like the reference (k_blk has
 * no effect on results, gemm.cpp:32; the GPU ignores it after validation).
 * c: m x n int16, row stride ldc elements.  kernel: lowbit_kernel. */
lowbit_status lowbit_gemm(int mode, const uint8_t* a0, const uint8_t* a1, long long a_pitch, int a_rows, int a_cols,
                          const void* weights, int b_ternary, int b_n, int b_k, int m, int n, int k, int k_blk,
                          int16_t* c, long long ldc, int kernel, lowbit_stream stream);

/* lowbit_gemm with A planes in layout a_layout (lowbit_layout).  LANES
 * planes are consumed by the tensor-core kernels only (the bit-serial kernel
 * needs REFERENCE planes; LOWBIT_KERNEL_BITSERIAL + LANES is rejected). */
lowbit_status lowbit_gemm_ex(int mode, int a_layout, const uint8_t* a0, const uint8_t* a1, long long a_pitch,
                             int a_rows, int a_cols, const void* weights, int b_ternary, int b_n, int b_k, int m,
                             int n, int k, int k_blk, int16_t* c, long long ldc, int kernel, lowbit_stream stream);

/* gemm_lowbit with A given as dense int8 sign values (row stride lda bytes,
 * lda % 16 == 0): the "from int8 A" form.  Values must be in {-1, 0, +1}
 * ({-1, +1} for BNN), the SignMatrix contract (core.hpp:21-33); the operand
 * kind follows the mode.  TMA feeds the tensor cores directly — no encode,
 * no converters.  Same validation and results as lowbit_gemm. */
lowbit_status lowbit_gemm_i8(int mode, const int8_t* a, long long lda, int a_rows, int a_cols, const void* weights,
                             int b_ternary, int b_n, int b_k, int m, int n, int k, int k_blk, int16_t* c,
                             long long ldc, lowbit_stream stream);

/* The static per-shape kernel table behind LOWBIT_KERNEL_AUTO. */
int lowbit_select_kernel(int mode, int m, int n, int k);

/* ---- grouped small GeMMs: one launch for many problems (§8f-3) ----------
 * The reference bench grid (bench.cpp:196-234) / BASELINE config 2 runs 64
 * small gemm_lowbit calls; each is launch-latency bound on a GPU.  One call
 * here validates every problem like lowbit_gemm (dims, depth, modes) and
 * issues one launch of K2-style bit-serial tiles for all of them (128
 * problems per launch; more are split).  Device pointers, stream-ordered. */
typedef struct lowbit_gemm_problem {
    const uint8_t* a0;    /* binary plane or plus plane, pitch a_pitch (multiple of 16) */
    const uint8_t* a1;    /* minus plane (ternary A) or NULL (binary A) */
    long long a_pitch;
    const void* weights;  /* lowbit_prepare_weights output for n x k */
    int m, n, k;
    int16_t* c;           /* m x n, row stride ldc */
    long long ldc;
} lowbit_gemm_problem;
lowbit_status lowbit_gemm_grouped(int mode, int b_ternary, int count, const lowbit_gemm_problem* problems,
                                  lowbit_stream stream);

/* ---- host-buffer drop-in: one whole reference gemm_lowbit call -----------
 * Host A planes with the reference stride ceil(a_cols/8); host PackedB
 * panels; host C (m x n, row-major).  Uploads, prepares B, runs, downloads
 * and synchronises `stream`.  Host buffers may be pinned or pageable
 * (pageable ones are staged through pinned slots).  Device scratch, copy
 * streams and staging slots are cached per (host thread, device) and freed
 * when the thread exits or by lowbit_release_thread_state().  On any error
 * the call has finished all of its copies before it returns. */
lowbit_status lowbit_gemm_lowbit_host(int mode, const uint8_t* a0, const uint8_t* a1, int a_rows, int a_cols,
                                      const uint8_t* panels, int b_ternary, int b_n, int b_k, int m, int n, int k,
                                      int k_blk, int16_t* c, int kernel, lowbit_stream stream);

/* ---- K4: convolution (conv.hpp:64-65 conv2d_lowbit; conv.cpp:33-59) -------
 * fm: NHWC int8 batch [batch][h][w][c] (the reference takes one image per
 * call; batch > 1 is the same computation per image).  Output pixels
 * (batch*OH*OW of them, lowbit_conv_rows) are the GeMM rows; depth
 * k = kh*kw*c in (ky, kx, c) order (conv.cpp:18-27).
 * lowbit_conv_encode: one launch of fused im2col + encode into the A planes
 * (binary planes when a_binary, plus/minus otherwise; padded positions read
 * as pad_value).  lowbit_conv2d: checks in the reference's order
 * (ChannelOverflow, weight shape, modes, EmptyOutput), K4, then lowbit_gemm
 * into out = int16 NHWC [batch][OH][OW][cout].  fm_binary is the feature
 * map's Mode (binary maps pad with binary_pad_value, ternary maps with 0);
 * a 0 in the A operand of a BNN conv sets *zero_flag.
 * Convs whose padding reads as 0 (ternary maps, or no padding) and whose c
 * is a multiple of 128 run on the tensor cores straight from the int8 map
 * (values in {-1,0,+1}, the FeatureMap contract): K7, a fused halo
 * convolution (stride 1, any map width), else K6 (fp4
 * implicit GeMM, uses the workspace), else an int8 implicit GeMM;
 * lowbit_conv_select names the path.  Other convs go through
 * lowbit_conv_encode. */
long long lowbit_conv_rows(int batch, int h, int w, int kh, int kw, int stride, int padding);
/* Which kernel lowbit_conv2d takes for a conv (host logic, no device needed;
 * `kernel` as for lowbit_conv2d, has_workspace: a workspace will be passed). */
enum {
    LOWBIT_CONV_PATH_ENCODE_GEMM = 1, /* K4 fused im2col + encode, then lowbit_gemm */
    LOWBIT_CONV_PATH_IMPLICIT_I8 = 3, /* TMA im2col over the int8 map -> tcgen05 kind::i8 */
    LOWBIT_CONV_PATH_IMPLICIT_FP4 = 6, /* K6: packed fp4 map + TMA im2col -> kind::mxf4 */
    LOWBIT_CONV_PATH_HALO_FP4 = 7     /* K7: fused halo convolution, one launch, no workspace */
};
int lowbit_conv_select(int mode, int fm_binary, int batch, int h, int w, int c, int cout, int kh, int kw, int stride,
                       int padding, int kernel, int has_workspace);
lowbit_status lowbit_conv_encode(int a_binary, const int8_t* fm, int batch, int h, int w, int c, int kh, int kw,
                                 int stride, int padding, int pad_value, uint8_t* plane0, uint8_t* plane1,
                                 long long pitch, int* zero_flag, lowbit_stream stream);
size_t lowbit_conv2d_workspace_bytes(int mode, int batch, int h, int w, int c, int kh, int kw, int stride,
                                     int padding);
lowbit_status lowbit_conv2d(int mode, const int8_t* fm, int batch, int h, int w, int c, int fm_binary,
                            const void* weights, int b_ternary, int cout, int k, int kh, int kw, int stride,
                            int padding, int binary_pad_value, void* workspace, int* zero_flag, int16_t* out,
                            int kernel, lowbit_stream stream);
/* Host-buffer drop-in of conv2d_lowbit: host NHWC fm, host PackedB panels of
 * the (kh*kw*c) x cout weights, host int32 NHWC out (IntFeatureMap).
 * The prepared weights of the last call on this thread and device are kept
 * and reused while the panel bytes (and b_ternary, cout, k) are identical, so
 * a batch of single-image calls uploads and prepares the weights once. */
lowbit_status lowbit_conv2d_host(int mode, const int8_t* fm, int batch, int h, int w, int c, int fm_binary,
                                 const uint8_t* panels, int b_ternary, int cout, int k, int kh, int kw, int stride,
                                 int padding, int binary_pad_value, int32_t* out, lowbit_stream stream);

/* Free this host thread's cached host-buffer state on every device
 * (device scratch, pinned staging, streams, events).  Optional: the same
 * happens when the thread exits.  The next host-buffer call re-creates it. */
void lowbit_release_thread_state(void);

/* ---- host-buffer forms of K1 / K1b (used by the C++ drop-in) -------------
 * Host planes use the reference stride ceil(cols/8) bytes.  Synchronous. */
/* encode_binary / encode_ternary (core.hpp:63,66): returns
 * LOWBIT_ZERO_IN_BINARY for a 0 in a binary matrix (core.cpp:23). */
lowbit_status lowbit_encode_host(int ternary, const int8_t* values, int rows, int cols, uint8_t* plane0,
                                 uint8_t* plane1, lowbit_stream stream);
/* pack_b (gemm.hpp:75-76): host K x N planes -> host PackedB panel stream. */
lowbit_status lowbit_pack_b_host(int ternary, const uint8_t* b0, const uint8_t* b1, int k, int n, uint8_t* panels,
                                 lowbit_stream stream);

/* ---- synthetic data (bench/tests): counter-based generator --------------
 * out[r][c] = f_dist(splitmix64(seed ^ matrix_id<<56 ^ ((row0+r)*cols + c)))
 * dist 0: uniform {-1,0,+1}; 1: uniform {-1,+1}; 2: P(0)=1/2, P(+-1)=1/4. */
lowbit_status lowbit_generate(int dist, unsigned long long seed, int matrix_id, long long row0, long long rows,
                              long long cols, int8_t* out, lowbit_stream stream);

/* ---- profiling experiments only ----------------------------------------
 * Read-and-reset per-role cycle counters of the CTA-pair kernel (enabled by
 * LOWBIT_DEBUG_PAIR=8 in the environment; see tools/pair_stats.py). */
int lowbit_debug_pair_stats(unsigned long long* out16);
/* Same for the fp4 pair kernel (LOWBIT_DEBUG_FP4=8). */
int lowbit_debug_fp4_stats(unsigned long long* out16);
/* Tuning aid: per-tile event clocks of K6's first leader CTA (LOWBIT_CONV_DEBUG & 32); 0 on success. */
int lowbit_debug_conv_trace(unsigned long long* out1024);
/* K7 timing experiments (LOWBIT_HALO_DEBUG & 32): per-tile clock64 events of
 * pair 0's leader CTA, and kernel phases in globaltimer ns (reset re-arms). */
int lowbit_debug_halo_trace(unsigned long long* out1024);
int lowbit_debug_halo_phases(unsigned long long* out4, int reset);

#ifdef __cplusplus
}
#endif

#endif /* LOWBIT_CUDA_H */

/*
 * ternkit_b200.h -- C-ABI of the B200 (sm_100a) ternary hot path.
 *
 * Drop-in boundary for the reference's header-only API (ternkit, R: =
 * /root/reference/proj/include/ternkit/).  The reference has no plugin
 * registry: its public C++ functions ARE the interface, so each entry point
 * below names the reference function it replaces.  The C++ shim
 * include/ternkit_b200/ternkit.hpp re-exposes exactly those C++ signatures
 * (host spans in, value-type results out, std::invalid_argument on error) on
 * top of this C layer; Python reaches it through ctypes
 * (paper_2008_05101_b200/_lib.py).
 *
 * Conventions
 *  - Buffers are caller-owned DEVICE pointers unless a parameter says _host.
 *  - Calls are asynchronous on `stream` (a cudaStream_t, NULL = legacy
 *    default stream) and return a status immediately for argument errors.
 *  - Data-dependent errors (non-finite input, negative activation -- the
 *    reference's throws in R:quantizer.hpp:37-41,53-55) are raised inside the
 *    kernels into the context's device error word; tk_context_sync() waits
 *    for the stream and returns the FIRST such error in the reference's
 *    evaluation order, then clears it.
 *  - One context per concurrently used stream (the context owns scratch).
 *  - Packed words are the reference layout byte for byte: 32 lanes per u64,
 *    lane i at bits 2(i%32), padding lanes 0b01 (R:codec.hpp:14-20).
 */
#ifndef TERNKIT_B200_H
#define TERNKIT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (all map to std::invalid_argument in the C++ shim) ---- */
#define TK_OK 0
#define TK_ERR_INVALID 1           /* length / shape / geometry mismatch      */
#define TK_ERR_THRESHOLDS 3        /* alpha1/alpha2 not > 0, R:codec.hpp:61   */
#define TK_ERR_NONFINITE 4         /* R:quantizer.hpp:37-41                   */
#define TK_ERR_NEGATIVE 5          /* R:quantizer.hpp:53-55                   */
#define TK_ERR_OFFSET_SYMMETRIC 6  /* R:linalg.hpp:245-249                    */
#define TK_ERR_MASKS 7             /* R:linalg.hpp:242-244                    */
#define TK_ERR_RANGE 8             /* value outside {-1,0,1}, R:codec.hpp:49  */
#define TK_ERR_CUDA 9              /* CUDA runtime failure                    */
#define TK_ERR_UNSUPPORTED 10      /* backend cannot run this shape           */

#define TK_MODE_WEIGHT 0             /* QuantMode::kWeight                   */
#define TK_MODE_ACTIVATION_NONNEG 1  /* QuantMode::kActivationNonneg         */

#define TK_MASK_ON_THE_FLY 0   /* MaskMode::kOnTheFly                         */
#define TK_MASK_PRECOMPUTED 1  /* MaskMode::kPrecomputed                      */

#define TK_BACKEND_AUTO 0    /* per-shape choice (profiles/)       */
#define TK_BACKEND_POPC 1    /* LOP3 + POPC integer pipe                      */
#define TK_BACKEND_TC_I8 2   /* tcgen05.mma kind::i8 tensor cores             */
#define TK_BACKEND_TC_F4 3   /* tcgen05.mma kind::mxf4 (E2M1 levels, unit E8M0
                                block scales: exact, 2x the i8 MMA rate)       */
#define TK_BACKEND_TC_CONV 4 /* conv2d_ternary: implicit-im2col fused conv
                                (quantize into padded channel-last s8 planes,
                                then tcgen05 kind::i8 over the 3x3 taps with
                                the folded-BN NCHW epilogue); other entries
                                and ineligible shapes use the kind::i8 GEMM */

typedef struct tk_context tk_context;
typedef struct tk_layer tk_layer;

int tk_version(void);
const char* tk_status_string(int status);

/* ---- context ------------------------------------------------------------ */
int tk_context_create(int device, tk_context** out);
int tk_context_destroy(tk_context* ctx);
/* Waits for `stream`, returns the first in-kernel error (or TK_OK), clears it. */
int tk_context_sync(tk_context* ctx, void* stream);

/* Exact float thresholds equivalent to the reference quantizer
 * (R:quantizer.hpp:44-60): lane bit0 = (p > t0), bit1 = (p > t1).  Host-only
 * helper, exposed so the threshold search can be tested without a GPU. */
int tk_quant_thresholds(float alpha1, float alpha2, int mode, float* t0,
                        float* t1);

/* fuse_bn(mean, var, gamma, beta, eps) -> ChannelAffine  R:linalg.hpp:70-91
 * Host-side parameter folding (one-time layer prep, host arrays), with the
 * reference build's float semantics (its multiply-subtract is one FMA). */
int tk_fuse_bn(const float* mean_host, const float* var_host,
               const float* gamma_host, const float* beta_host, float eps,
               int channels, float* gain_host, float* bias_host);

/* ---- codec / quantizer (R:codec.hpp, R:quantizer.hpp) ------------------- */
/* pack(span<const int8_t>)                         R:codec.hpp:89-100 */
int tk_pack(tk_context* ctx, const int8_t* values, size_t n, uint64_t* words,
            void* stream);
/* unpack(PackedTernaryVector)                      R:codec.hpp:107-117 */
int tk_unpack(tk_context* ctx, const uint64_t* words, size_t n, int8_t* values,
              void* stream);
/* quantize_and_pack(span<const float>, thr, mode)  R:quantizer.hpp:159-170
 * `rows` independent vectors of `n` floats each, row r packed into
 * words[r * words_for_lanes(n) ...]. */
int tk_quantize_pack(tk_context* ctx, const float* x, size_t rows, size_t n,
                     float alpha1, float alpha2, int mode, uint64_t* words,
                     void* stream);

/* ---- inner products (R:bitkernels.hpp) ---------------------------------- */
/* out[p] = ternary_dot(x_p, y_p) (+ wsum[p] if wsum != NULL, i.e.
 * ternary_dot_nonneg).  x,y: [pairs][words] u64.    R:bitkernels.hpp:116-159 */
int tk_ternary_dot_batched(tk_context* ctx, const uint64_t* x,
                           const uint64_t* y, size_t words, size_t pairs,
                           const int64_t* wsum, int64_t* out, void* stream);
/* detail::ternary_dot_words_premask / ternary_dot_premask: the same with the
 * zero seeds supplied, seeds: [pairs][words] u64 (make_zero_seeds of y, or any
 * caller buffer -- the TM of R:bitkernels.hpp:66-72 uses them as given).
 *                                                    R:bitkernels.hpp:87-97,130-149 */
int tk_ternary_dot_premask_batched(tk_context* ctx, const uint64_t* x, const uint64_t* y, const uint64_t* seeds,
                                   size_t words, size_t pairs, const int64_t* wsum, int64_t* out, void* stream);

/* ---- linalg (R:linalg.hpp) ---------------------------------------------- */
/* im2col_quantize_pack(x NCHW, shape, thr, geom, mode)  R:linalg.hpp:173-225
 * rows: [n*oh*ow][words_for_lanes(c*kh*kw)] u64. */
int tk_im2col_quantize_pack(tk_context* ctx, const float* x, int n, int c,
                            int h, int w, int kh, int kw, int stride, int pad,
                            float alpha1, float alpha2, int mode,
                            uint64_t* rows, void* stream);

/* make_packed_conv_layer(int8 weights, geom, thr_w, thr_a, nonneg, fused,
 * out_scale)                                         R:linalg.hpp:118-144
 * weights_host: [out_c][in_c*kh*kw] in {-1,0,1}; gain/bias_host may be NULL
 * (identity affine, R:linalg.hpp:133-134).  Uploads packed rows, weight sums,
 * zero masks and the int8 tensor-core operand once. */
int tk_layer_create(tk_context* ctx, const int8_t* weights_host, int in_c,
                    int out_c, int kh, int kw, int stride, int pad,
                    float tw1, float tw2, float ta1, float ta2,
                    int activation_nonneg, const float* gain_host,
                    const float* bias_host, float out_scale, tk_layer** out);
int tk_layer_destroy(tk_layer* layer);
/* PackedConvLayer::precompute_masks()                R:linalg.hpp:109-113 */
int tk_layer_precompute_masks(tk_layer* layer);
int tk_layer_set_backend(tk_layer* layer, int backend);
int tk_layer_get_backend(const tk_layer* layer, int m_rows);
/* host copies of the packed rows / weight sums (PackedConvLayer::weights,
 * ::weight_sums) for callers that inspect them */
int tk_layer_words_host(const tk_layer* layer, uint64_t* words_host,
                        int32_t* wsums_host);

/* packed_gemm(Im2colBuffer, layer, mask_mode, workers) R:linalg.hpp:232-293
 * rows: [row_count][words_for_lanes(row_len)] u64; out: [row_count][out_c]. */
int tk_packed_gemm(tk_context* ctx, const tk_layer* layer,
                   const uint64_t* rows, size_t row_count, size_t row_len,
                   int nonneg_offset, int mask_mode, int32_t* out,
                   void* stream);

/* conv2d_ternary(x NCHW, shape, layer, mask_mode, workers)
 *                                                    R:linalg.hpp:301-328
 * out: [n][out_c][oh][ow] f32 = gain*(out_scale*acc)+bias (one FMA). */
int tk_conv2d_ternary(tk_context* ctx, const tk_layer* layer, const float* x,
                      int n, int h, int w, int mask_mode, float* out,
                      void* stream);

/* Ternary GEMM on operands already expanded to quantization levels: the
 * contraction packed_gemm performs, without the pack/expand step.  a_s8 is
 * the s8 level operand in K-block-major layout [k_pad/128][m_pad][128]
 * (m_pad = m_rows rounded up to 128; element (r, k) at
 * ((k/128)*m_pad + r)*128 + k%128), as tk_quantize_levels writes it, so that
 * every tensor-core tile load is one contiguous block.  out_mode 0: int32
 * [m_rows][out_c] accumulators; 1: f32 rows after the folded-BN epilogue.
 * Tensor-core path only (TK_ERR_UNSUPPORTED otherwise). */
int tk_gemm_levels(tk_context* ctx, const tk_layer* layer, const int8_t* a_s8,
                   int m_rows, int out_mode, void* out, void* stream);
/* Quantize f32 rows [rows][n] to s8 levels for tk_gemm_levels (activation
 * levels {0,1,2} in nonneg mode, {-1,0,1} in weight mode), zero padded to
 * k_pad (a multiple of 128), written K-block-major (see tk_gemm_levels):
 * out holds round_up(rows, 128) * k_pad bytes. */
int tk_quantize_levels(tk_context* ctx, const float* x, int rows, int n,
                       float alpha1, float alpha2, int mode, int k_pad,
                       int8_t* out, void* stream);
int tk_layer_k_pad(const tk_layer* layer);
/* The same contraction on the FP4 tensor-core path:
 * levels as E2M1 nibbles (-1 -> 0xA, 0 -> 0x0, 1 -> 0x2, 2 -> 0x4), two per
 * byte with the even k in the low nibble, K-block-major with 256 levels per
 * 128-byte block: element (r, k) in byte ((k/256)*m_pad + r)*128 + (k%256)/2.
 * k_pad = tk_layer_k_pad_fp4 (K rounded up to 256); the operand holds
 * round_up(rows, 128) * k_pad / 2 bytes.  Results are identical to
 * tk_gemm_levels (f32 accumulation of integers < 2^24 is exact). */
int tk_gemm_levels_fp4(tk_context* ctx, const tk_layer* layer, const uint8_t* a_fp4,
                       int m_rows, int out_mode, void* out, void* stream);
int tk_quantize_levels_fp4(tk_context* ctx, const float* x, int rows, int n,
                           float alpha1, float alpha2, int mode, int k_pad,
                           uint8_t* out, void* stream);
int tk_layer_k_pad_fp4(const tk_layer* layer);

/* fully_connected_ternary(x, batch, layer, mask_mode) R:linalg.hpp:332-343 */
int tk_fully_connected_ternary(tk_context* ctx, const tk_layer* layer,
                               const float* x, int batch, int mask_mode,
                               float* out, void* stream);

/* ---- paper baselines: binary and bit-plane multi-bit dots (F3) ----------- */
/* pack_binary(span<const int8_t>) (R:bitkernels.hpp:170-182): +1 -> bit 1,
 * -1 -> bit 0, little-endian, zero-padded; other values raise TK_ERR_RANGE
 * at the next tk_context_sync.  words: (n + 63) / 64 u64. */
int tk_pack_binary(tk_context* ctx, const int8_t* values, size_t n, uint64_t* words, void* stream);
/* binary_dot (R:bitkernels.hpp:99-110, 184-191), batched: x, y [pairs][words] */
int tk_binary_dot_batched(tk_context* ctx, const uint64_t* x, const uint64_t* y, size_t words, size_t logical_len,
                          size_t pairs, int64_t* out, void* stream);
/* multibit_dot (R:bitkernels.hpp:196-222), batched: x_planes [m][pairs][words],
 * y_planes [k][pairs][words], f64 scales; the f64 accumulation follows the
 * reference's (m, k) order and roundings, so results are bit-identical */
int tk_multibit_dot_batched(tk_context* ctx, const uint64_t* x_planes, int m, const uint64_t* y_planes, int k,
                            const double* x_scales, const double* y_scales, size_t words, size_t logical_len,
                            size_t pairs, double* out, void* stream);

/* ---- packed_forward float pieces (R:tinynet.hpp:713-735, FATN models) ----- */
/* detail::matmul_t (R:tinynet.hpp, used by packed_forward for stem / head):
 * y[b][o] = bias[o] + sum_j x[b][j] * w[o][j] with the reference build's
 * operation order (see oracle/ternkit_oracle.c or_matmul_t); relu != 0 then
 * applies std::max(v, 0.0f).  Device pointers, w row-major [out_dim][in_dim],
 * bias may be NULL. */
int tk_matmul_t(tk_context* ctx, const float* x, const float* w, const float* bias, int batch, int in_dim,
                int out_dim, int relu, float* y, void* stream);
/* Dense fp32 layer of the ResNet head (outside the ternary path):
 * y[b][o] = bias[o] + sum_k x[b][k] * w[o][k], one fp32 FMA chain in k order
 * per output; w row-major [out_dim][in_dim], bias may be NULL. */
int tk_dense_f32(tk_context* ctx, const float* x, const float* w, const float* bias, int batch, int in_dim,
                 int out_dim, float* y, void* stream);
/* packed_forward's block tail (R:tinynet.hpp:720-730): z[i] = max(z[i] + id, 0)
 * with id = fmaf(cal_gain[j], h[i], cal_bias[j]) (calibration present) or
 * h[i], j = i % hidden; both calibration pointers or neither. */
int tk_residual_relu_rows(tk_context* ctx, float* z, const float* h, long long count, int hidden,
                          const float* cal_gain, const float* cal_bias, void* stream);

/* ---- network-level packed inference (R:tinynet.hpp:713-735 pattern) -------
 * A body is a sequence of residual blocks of conv2d_ternary layers (folded BN
 * in each layer's affine): inner convs are followed by ReLU; the last conv's
 * output is added to the shortcut (identity, or a 1x1 downsample conv) and
 * ReLU'd -- exactly the reference composition z = max(z + id, 0)
 * (R:tinynet.hpp:720-730) applied to conv layers.  Layout of the structs
 * matches oracle/netdesc.h. */
typedef struct {
  int in_c, out_c, k, stride, pad;
  const int8_t* weights_host; /* [out_c][(ky*k + kx)*in_c + c] in {-1,0,1} */
  float tw1, tw2, ta1, ta2;
  const float* gain_host;     /* folded BN, out_c (NULL = identity) */
  const float* bias_host;
  float out_scale;
} tk_conv_desc;

typedef struct {
  int n_convs;                /* 2 (basic) or 3 (bottleneck) */
  tk_conv_desc conv[3];
  int has_down;
  tk_conv_desc down;          /* 1x1 shortcut conv */
} tk_block_desc;

typedef struct tk_net tk_net;

#define TK_NET_AUTO 0     /* fused tensor-core pipeline when the shapes allow */
#define TK_NET_GENERIC 1  /* layer-by-layer conv2d_ternary (any shape)        */

/* Builds device weights, activation buffers (batch fixed) and launch plans. */
int tk_net_create(tk_context* ctx, const tk_block_desc* blocks, int n_blocks,
                  int batch, int in_c, int in_h, int in_w, int mode,
                  tk_net** out);
int tk_net_destroy(tk_net* net);
int tk_net_out_shape(const tk_net* net, int* c, int* h, int* w);
/* 1 = fused tensor-core pipeline, 0 = generic layer-by-layer path */
int tk_net_is_fused(const tk_net* net);
/* x: [batch][in_c][in_h][in_w] f32 (device).  out (nullable): body output
 * [batch][C][H][W] f32; pooled (nullable): its spatial mean [batch][C]. */
int tk_net_forward(tk_context* ctx, tk_net* net, const float* x, float* out,
                   float* pooled, void* stream);
/* Network stem helper (float, outside the ternary path): the fused
 * y = maxpool3x3/2(max(fmaf(gain[c], x, bias[c]), 0)) (pad 1, -inf padding)
 * over x [n][c][h][w] f32 -> out [n][c][(h+1)/2][(w+1)/2], one pass. */
int tk_affine_relu_maxpool(tk_context* ctx, const float* x, int n, int c, int h, int w,
                           const float* gain, const float* bias, float* out, void* stream);
/* Network stem helper: 7x7 / stride 2 / pad 3 convolution, 3 -> 64 channels,
 * on the tensor cores as split TF32 (x_hi w_hi + x_hi w_lo + x_lo w_hi, f32
 * accumulation; error <= 4e-6 x sum |x||w| per output): images [n][3][h][w]
 * (w <= 240), weights [64][3][7][7] -> out [n][64][(h-1)/2+1][(w-1)/2+1]
 * (no bias); TK_ERR_UNSUPPORTED for wider images. */
int tk_stem_conv7x7s2(tk_context* ctx, const float* images, int n, int h, int w, const float* weights,
                      float* out, void* stream);
/* number of kernel launches one tk_net_forward issues */
int tk_net_launches(const tk_net* net, int with_out, int with_pooled);
/* diagnostics: per-conv device time of the last forward after
 * tk_net_set_timing(net, 1) (fused path), and MACs per conv (whole batch) */
int tk_net_num_convs(const tk_net* net);
int tk_net_set_timing(tk_net* net, int on);
int tk_net_conv_times(tk_net* net, float* ms_host, double* macs_host);
/* diagnostics: per-CTA phase stamps of the last conv run with TK_CONV_DBG&16
 * (148*8 + 8*32 u64) */
int tk_debug_conv_stamps(unsigned long long* host_out);
/* profiling: per-CTA stamps of the last tensor-core GEMM launched with env
 * TK_GEMM_DBG & 16 (grid-linear CTA id < 512): [512][8] SM-clock phase
 * stamps, [2][512][2] globaltimer ns at CTA start / end for the last
 * launch of each parity, then [512][16] reduction sub-phase stamps (14336 u64) */
int tk_debug_gemm_stamps(unsigned long long* host_out);

#ifdef __cplusplus
}
#endif
#endif

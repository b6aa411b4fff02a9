// tk_api.cu -- the C-ABI (include/ternkit_b200.h): argument validation in the
// reference's order, layer upload, and dispatch to the kernels.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include "tk_internal.cuh"

#define TK_CUDA(call)                              \
  do {                                             \
    cudaError_t e_ = (call);                       \
    if (e_ != cudaSuccess) return TK_ERR_CUDA;     \
  } while (0)

namespace {

size_t words_for_lanes(size_t n) { return (n + 31) / 32; }

// ---- exact quantizer thresholds -------------------------------------------
// Key space: int32 k in [-0x7f800000, 0x7f800000] maps monotonically onto
// [-inf, +inf] (k >= 0: bits of +f; k < 0: bits of -f).
float key_to_float(int64_t k) {
  uint32_t b = (uint32_t)(k >= 0 ? k : -k);
  float f;
  memcpy(&f, &b, 4);
  return k >= 0 ? f : -f;
}

// smallest key whose float satisfies a monotone (false -> true) predicate;
// 0x7f800001 when even +inf fails
template <class P>
int64_t first_true(P pred) {
  int64_t lo = -0x7f800000LL, hi = 0x7f800000LL;
  if (!pred(key_to_float(hi))) return hi + 1;
  if (pred(key_to_float(lo))) return lo;
  while (hi - lo > 1) {  // invariant: !pred(lo), pred(hi)
    const int64_t mid = lo + (hi - lo) / 2;
    if (pred(key_to_float(mid))) hi = mid; else lo = mid;
  }
  return hi;
}

// The host divides exactly like the reference (IEEE binary32, round to
// nearest even); fl(p/a) and fl(fl(p-a1)/a2) are monotone in p, so each
// rounded step function of R:quantizer.hpp:44-60 is a single float threshold.
float below(int64_t first) { return key_to_float(first - 1); }

}  // namespace

int tk_make_qparams(float a1, float a2, int mode, tk_qparams* q) {
  if (!(a1 > 0.0f) || !(a2 > 0.0f)) return TK_ERR_THRESHOLDS;
  if (mode == TK_MODE_ACTIVATION_NONNEG) {
    // lo = round(clip(p/a1,0,1)) = 1  iff  p/a1 > 0.5 (0.5 ties to even -> 0)
    volatile float va1 = a1, va2 = a2;
    q->t0 = below(first_true([&](float p) { return p / va1 > 0.5f; }));
    // hi = round(clip((p-a1)/a2,0,1)) = 1  iff  (p-a1)/a2 > 0.5
    q->t1 = below(first_true([&](float p) { return (p - va1) / va2 > 0.5f; }));
    q->nonneg = 1;
  } else if (mode == TK_MODE_WEIGHT) {
    volatile float va1 = a1, va2 = a2;
    // bit0 = level >= 0 = !(round(clip(p/a1,-1,0)) == -1) = !(p/a1 < -0.5)
    q->t0 = below(first_true([&](float p) { return !(p / va1 < -0.5f); }));
    // bit1 = level == 1 = p/a2 > 0.5
    q->t1 = below(first_true([&](float p) { return p / va2 > 0.5f; }));
    q->nonneg = 0;
  } else {
    return TK_ERR_INVALID;
  }
  return TK_OK;
}

void* tk_workspace(tk_context* ctx, size_t bytes) {
  if (bytes <= ctx->ws_bytes) return ctx->ws;
  cudaDeviceSynchronize();  // previous users of the scratch must be done
  if (ctx->ws) cudaFree(ctx->ws);
  ctx->ws = nullptr;
  ctx->ws_bytes = 0;
  if (cudaMalloc(&ctx->ws, bytes) != cudaSuccess) return nullptr;
  ctx->ws_bytes = bytes;
  return ctx->ws;
}

cudaError_t tk_smem_attr(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;  // (kernel, device) -> bytes set
  int dev = 0;
  if (const cudaError_t e = cudaGetDevice(&dev); e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  int& have = done[{kernel, dev}];
  if (have >= bytes) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}

extern "C" {

int tk_version(void) { return 100; }

const char* tk_status_string(int status) {
  switch (status) {
    case TK_OK: return "ok";
    case TK_ERR_INVALID: return "invalid argument";
    case TK_ERR_THRESHOLDS: return "quantizer step sizes must be positive";
    case TK_ERR_NONFINITE: return "quantizer input is not finite";
    case TK_ERR_NEGATIVE: return "activation quantizer requires p >= 0";
    case TK_ERR_OFFSET_SYMMETRIC: return "packed_gemm: offset activations fed to a symmetric layer";
    case TK_ERR_MASKS: return "packed_gemm: masks not precomputed";
    case TK_ERR_RANGE: return "ternary value out of range {-1,0,1}";
    case TK_ERR_CUDA: return "CUDA runtime error";
    case TK_ERR_UNSUPPORTED: return "backend does not support this shape";
  }
  return "unknown status";
}

int tk_quant_thresholds(float a1, float a2, int mode, float* t0, float* t1) {
  tk_qparams q;
  const int st = tk_make_qparams(a1, a2, mode, &q);
  if (st != TK_OK) return st;
  *t0 = q.t0;
  *t1 = q.t1;
  return TK_OK;
}

int tk_fuse_bn(const float* mean, const float* var, const float* gamma,
               const float* beta, float eps, int c, float* gain, float* bias) {
  if (c < 0 || (c && (!mean || !var || !gamma || !beta || !gain || !bias)))
    return TK_ERR_INVALID;
  for (int i = 0; i < c; ++i) {
    const float denom = var[i] + eps;
    if (!(denom > 0.0f)) return TK_ERR_INVALID;  // R:linalg.hpp:83-85
    const float inv_std = 1.0f / sqrtf(denom);
    gain[i] = gamma[i] * inv_std;
    bias[i] = fmaf(-(mean[i] * gamma[i]), inv_std, beta[i]);
  }
  return TK_OK;
}

int tk_context_create(int device, tk_context** out) {
  if (!out) return TK_ERR_INVALID;
  TK_CUDA(cudaSetDevice(device));
  tk_context* c = new tk_context;
  c->device = device;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (cudaMalloc(&c->d_err, sizeof(unsigned long long)) != cudaSuccess ||
      cudaMallocHost(&c->pinned, sizeof(unsigned long long)) != cudaSuccess) {
    delete c;
    return TK_ERR_CUDA;
  }
  cudaMemset(c->d_err, 0xFF, sizeof(unsigned long long));
  cudaDeviceSynchronize();
  *out = c;
  return TK_OK;
}

int tk_context_destroy(tk_context* ctx) {
  TK_ON_DEVICE(ctx);
  if (!ctx) return TK_OK;
  cudaDeviceSynchronize();
  if (ctx->ws) cudaFree(ctx->ws);
  if (ctx->d_err) cudaFree(ctx->d_err);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  delete ctx;
  return TK_OK;
}

int tk_context_sync(tk_context* ctx, void* stream) {
  TK_ON_DEVICE(ctx);
  if (!ctx) return TK_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  unsigned long long* h = (unsigned long long*)ctx->pinned;
  TK_CUDA(cudaMemcpyAsync(h, ctx->d_err, 8, cudaMemcpyDeviceToHost, s));
  TK_CUDA(cudaMemsetAsync(ctx->d_err, 0xFF, 8, s));
  TK_CUDA(cudaStreamSynchronize(s));
  if (*h == ~0ull) return TK_OK;
  return (int)(*h & 0xFF);
}

int tk_pack(tk_context* ctx, const int8_t* values, size_t n, uint64_t* words,
            void* stream) {
  TK_ON_DEVICE(ctx);
  if (!ctx || (n && (!values || !words))) return TK_ERR_INVALID;
  TK_CUDA(tk_launch_pack_int8(values, n, words, ctx->d_err, (cudaStream_t)stream));
  return TK_OK;
}

int tk_unpack(tk_context* ctx, const uint64_t* words, size_t n, int8_t* values,
              void* stream) {
  TK_ON_DEVICE(ctx);
  if (!ctx || (n && (!values || !words))) return TK_ERR_INVALID;
  TK_CUDA(tk_launch_unpack(words, n, values, (cudaStream_t)stream));
  return TK_OK;
}

int tk_quantize_pack(tk_context* ctx, const float* x, size_t rows, size_t n,
                     float a1, float a2, int mode, uint64_t* words,
                     void* stream) {
  TK_ON_DEVICE(ctx);
  if (!ctx) return TK_ERR_INVALID;
  tk_qparams q;
  const int st = tk_make_qparams(a1, a2, mode, &q);  // R:quantizer.hpp:63
  if (st != TK_OK) return st;
  if (rows * n && (!x || !words)) return TK_ERR_INVALID;
  TK_CUDA(tk_launch_quantize_pack(x, rows, n, q, words, ctx->d_err,
                                  (cudaStream_t)stream));
  return TK_OK;
}

int tk_ternary_dot_batched(tk_context* ctx, const uint64_t* x,
                           const uint64_t* y, size_t words, size_t pairs,
                           const int64_t* wsum, int64_t* out, void* stream) {
  TK_ON_DEVICE(ctx);
  if (!ctx || (pairs && (!x || !y || !out))) return TK_ERR_INVALID;
  TK_CUDA(tk_launch_dot_batched(x, y, nullptr, words, pairs, wsum, out, (cudaStream_t)stream));
  return TK_OK;
}

int tk_ternary_dot_premask_batched(tk_context* ctx, const uint64_t* x, const uint64_t* y, const uint64_t* seeds,
                                   size_t words, size_t pairs, const int64_t* wsum, int64_t* out, void* stream) {
  TK_ON_DEVICE(ctx);
  if (!ctx || (pairs && (!x || !y || !seeds || !out))) return TK_ERR_INVALID;
  TK_CUDA(tk_launch_dot_batched(x, y, seeds, words, pairs, wsum, out, (cudaStream_t)stream));
  return TK_OK;
}

static bool geom_ok(int c, int h, int w, int kh, int kw, int stride, int pad) {
  // R:linalg.hpp:40-53
  if (c <= 0 || kh <= 0 || kw <= 0 || stride <= 0 || pad < 0) return false;
  if (h + 2 * pad < kh || w + 2 * pad < kw) return false;
  return true;
}

int tk_im2col_quantize_pack(tk_context* ctx, const float* x, int n, int c,
                            int h, int w, int kh, int kw, int stride, int pad,
                            float a1, float a2, int mode, uint64_t* rows,
                            void* stream) {
  TK_ON_DEVICE(ctx);
  if (!ctx) return TK_ERR_INVALID;
  if (!geom_ok(c, h, w, kh, kw, stride, pad) || n < 0 || h < 0 || w < 0)
    return TK_ERR_INVALID;  // geom.validate before t.validate, R:linalg.hpp:178-179
  tk_qparams q;
  const int st = tk_make_qparams(a1, a2, mode, &q);
  if (st != TK_OK) return st;
  TK_CUDA(tk_launch_im2col(x, n, c, h, w, kh, kw, stride, pad, q, rows,
                           ctx->d_err, (cudaStream_t)stream));
  return TK_OK;
}

// ---- layers ---------------------------------------------------------------

int tk_layer_create(tk_context* ctx, const int8_t* weights_host, int in_c,
                    int out_c, int kh, int kw, int stride, int pad, float tw1,
                    float tw2, float ta1, float ta2, int activation_nonneg,
                    const float* gain_host, const float* bias_host,
                    float out_scale, tk_layer** out) {
  TK_ON_DEVICE(ctx);
  if (!ctx || !out) return TK_ERR_INVALID;
  if (in_c <= 0 || out_c <= 0 || kh <= 0 || kw <= 0 || stride <= 0 || pad < 0)
    return TK_ERR_INVALID;
  const int K = in_c * kh * kw;
  const int wpr = (int)words_for_lanes(K);
  // pack rows on the host exactly as make_packed_conv_layer does
  // (R:linalg.hpp:136-143): one-time weight preparation, then uploaded.
  std::vector<uint64_t> words((size_t)out_c * wpr, 0x5555555555555555ull);
  std::vector<uint32_t> mask((size_t)out_c * wpr * 2);
  std::vector<int32_t> wsum(out_c), zcnt(out_c);
  const int k_pad = ((K + 127) / 128) * 128;
  const int n_pad = ((out_c + 255) / 256) * 256;
  std::vector<int8_t> w8((size_t)n_pad * k_pad, 0);
  const int k_pad4 = ((K + 255) / 256) * 256;
  std::vector<uint8_t> w4((size_t)n_pad * k_pad4 / 2, 0);  // E2M1 nibbles, even lane low
  for (int o = 0; o < out_c; ++o) {
    int32_t s = 0;
    for (int l = 0; l < K; ++l) {
      const int v = weights_host[(size_t)o * K + l];
      if (v < -1 || v > 1) return TK_ERR_RANGE;  // encode_lane throws
      const uint64_t code = v < 0 ? 0u : (v == 0 ? 1u : 3u);
      uint64_t& wd = words[(size_t)o * wpr + l / 32];
      wd = (wd & ~(3ull << (2 * (l % 32)))) | (code << (2 * (l % 32)));
      s += v;
      w8[((size_t)(l / 128) * n_pad + o) * 128 + l % 128] = (int8_t)v;  // [k/128][n_pad][128]
      const uint8_t nib = v < 0 ? 0xA : (v == 0 ? 0x0 : 0x2);            // [k/256][n_pad][128 B]
      w4[((size_t)(l / 256) * n_pad + o) * 128 + (l % 256) / 2] |= (uint8_t)(nib << (4 * (l & 1)));
    }
    wsum[o] = s;
    int32_t z = 0;
    for (int i = 0; i < wpr; ++i) {
      const uint64_t y = words[(size_t)o * wpr + i];
      const uint64_t d = (y ^ (y >> 1)) & 0x5555555555555555ull;
      const uint64_t m = ~(d | (d << 1));
      mask[((size_t)o * wpr + i) * 2] = (uint32_t)m;
      mask[((size_t)o * wpr + i) * 2 + 1] = (uint32_t)(m >> 32);
      z += __builtin_popcountll(d);
    }
    zcnt[o] = z;
  }
  tk_layer* L = new tk_layer;
  L->ctx = ctx;
  L->in_c = in_c; L->out_c = out_c; L->kh = kh; L->kw = kw;
  L->stride = stride; L->pad = pad;
  L->tw1 = tw1; L->tw2 = tw2; L->ta1 = ta1; L->ta2 = ta2;
  L->out_scale = out_scale;
  L->nonneg = activation_nonneg ? 1 : 0;
  L->K = K;
  L->wpr64 = wpr;
  L->k_pad = k_pad;
  L->n_pad = n_pad;
  L->k_pad4 = k_pad4;
  std::vector<float> gain(out_c, 1.0f), bias(out_c, 0.0f);  // identity, R:linalg.hpp:133
  if (gain_host) memcpy(gain.data(), gain_host, out_c * 4);
  if (bias_host) memcpy(bias.data(), bias_host, out_c * 4);
  bool ok =
      cudaMalloc(&L->d_words, words.size() * 8) == cudaSuccess &&
      cudaMalloc(&L->d_mask, mask.size() * 4) == cudaSuccess &&
      cudaMalloc(&L->d_wsum, out_c * 4) == cudaSuccess &&
      cudaMalloc(&L->d_zcnt, out_c * 4) == cudaSuccess &&
      cudaMalloc(&L->d_gain, out_c * 4) == cudaSuccess &&
      cudaMalloc(&L->d_bias, out_c * 4) == cudaSuccess &&
      cudaMalloc(&L->d_w8, w8.size()) == cudaSuccess &&
      cudaMalloc(&L->d_w4, w4.size()) == cudaSuccess;
  if (ok) {
    ok = cudaMemcpy(L->d_words, words.data(), words.size() * 8, cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemcpy(L->d_mask, mask.data(), mask.size() * 4, cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemcpy(L->d_wsum, wsum.data(), out_c * 4, cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemcpy(L->d_zcnt, zcnt.data(), out_c * 4, cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemcpy(L->d_gain, gain.data(), out_c * 4, cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemcpy(L->d_bias, bias.data(), out_c * 4, cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemcpy(L->d_w8, w8.data(), w8.size(), cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemcpy(L->d_w4, w4.data(), w4.size(), cudaMemcpyHostToDevice) == cudaSuccess;
  }
  L->h_words = (uint64_t*)malloc(words.size() * 8);
  L->h_wsum = (int32_t*)malloc(out_c * 4);
  L->h_gain = (float*)malloc(out_c * 4);
  L->h_bias = (float*)malloc(out_c * 4);
  memcpy(L->h_words, words.data(), words.size() * 8);
  memcpy(L->h_wsum, wsum.data(), out_c * 4);
  memcpy(L->h_gain, gain.data(), out_c * 4);
  memcpy(L->h_bias, bias.data(), out_c * 4);
  if (!ok) {
    tk_layer_destroy(L);
    return TK_ERR_CUDA;
  }
  *out = L;
  return TK_OK;
}

int tk_layer_destroy(tk_layer* L) {
  TK_ON_DEVICE(L ? L->ctx : nullptr);
  if (!L) return TK_OK;
  cudaDeviceSynchronize();
  tk_fconv_destroy_plans(L);
  cudaFree(L->d_words); cudaFree(L->d_mask); cudaFree(L->d_wsum);
  cudaFree(L->d_zcnt); cudaFree(L->d_gain); cudaFree(L->d_bias);
  cudaFree(L->d_w8);
  cudaFree(L->d_w4);
  free(L->h_words);
  free(L->h_wsum);
  free(L->h_gain);
  free(L->h_bias);
  delete L;
  return TK_OK;
}

int tk_layer_precompute_masks(tk_layer* L) {
  if (!L) return TK_ERR_INVALID;
  L->masks_ready = 1;  // device masks are always resident; mirrors the host flag
  return TK_OK;
}

int tk_layer_set_backend(tk_layer* L, int backend) {
  if (!L || backend < TK_BACKEND_AUTO || backend > TK_BACKEND_TC_CONV)
    return TK_ERR_INVALID;
  L->backend = backend;
  return TK_OK;
}

// Per-shape pipe choice (evidence in profiles/):
// the tensor-core path wins once the tile grid can be filled, and there the
// FP4 operands (half the bytes of s8, twice the MMA rate, same exact sums)
// beat s8.
int tk_layer_get_backend(const tk_layer* L, int m_rows) {
  if (!L) return TK_ERR_INVALID;
  // (TC_CONV is a conv2d_ternary kernel; everywhere else it is the kind::i8 GEMM)
  if (L->backend == TK_BACKEND_TC_CONV) return TK_BACKEND_TC_I8;
  if (L->backend != TK_BACKEND_AUTO) return L->backend;
  if (!(tk_tc_supported(m_rows, L->out_c, L->k_pad) && m_rows >= 128)) return TK_BACKEND_POPC;
  // FP4 unless its coarser K blocks (256 levels) leave too few K blocks to
  // split across the SMs when the tile grid alone is small (cfg2 at batch 1:
  // K = 576 -> 3 FP4 blocks vs 5 s8 blocks, 25 tiles; measured i8 18.5 us vs
  // fp4 20.5 us per step)
  const long tiles64 = (long)((m_rows + 127) / 128) * ((L->out_c + 63) / 64);
  return (tiles64 >= 96 || L->k_pad4 / 256 >= 4) ? TK_BACKEND_TC_F4 : TK_BACKEND_TC_I8;
}

namespace {
// tensor-core operand format of a backend: fp4 levels or s8 levels
bool tc_backend(int be) { return be == TK_BACKEND_TC_I8 || be == TK_BACKEND_TC_F4; }
int tc_k_pad(const tk_layer* L, bool fp4) { return fp4 ? L->k_pad4 : L->k_pad; }
size_t tc_operand_bytes(const tk_layer* L, size_t m_pad, bool fp4) {
  return fp4 ? m_pad * L->k_pad4 / 2 : m_pad * L->k_pad;
}
}  // namespace

int tk_layer_words_host(const tk_layer* L, uint64_t* words_host,
                        int32_t* wsums_host) {
  if (!L) return TK_ERR_INVALID;
  if (words_host) memcpy(words_host, L->h_words, (size_t)L->out_c * L->wpr64 * 8);
  if (wsums_host) memcpy(wsums_host, L->h_wsum, (size_t)L->out_c * 4);
  return TK_OK;
}

// R:linalg.hpp:232-249 validation order, then the chosen pipe.
int tk_packed_gemm(tk_context* ctx, const tk_layer* L, const uint64_t* rows,
                   size_t row_count, size_t row_len, int nonneg_offset,
                   int mask_mode, int32_t* out, void* stream) {
  TK_ON_DEVICE(ctx);
  if (!ctx || !L) return TK_ERR_INVALID;
  if (row_len != (size_t)L->K) return TK_ERR_INVALID;
  if (mask_mode == TK_MASK_PRECOMPUTED && !L->masks_ready) return TK_ERR_MASKS;
  if (nonneg_offset && !L->nonneg) return TK_ERR_OFFSET_SYMMETRIC;
  cudaStream_t s = (cudaStream_t)stream;
  tk_epilogue e{TK_EPI_I32, 1, nullptr, nullptr, 1.0f, out};
  const int be = tk_layer_get_backend(L, (int)row_count);
  if (tc_backend(be)) {
    const bool f4 = be == TK_BACKEND_TC_F4;
    if (!tk_tc_supported((int)row_count, L->out_c, L->k_pad)) return TK_ERR_UNSUPPORTED;
    const size_t m_pad = (row_count + 127) / 128 * 128;
    int8_t* a8 = (int8_t*)tk_workspace(ctx, tc_operand_bytes(L, m_pad, f4));
    if (!a8) return TK_ERR_CUDA;
    TK_CUDA(tk_launch_expand_rows(rows, row_count, L->wpr64, nonneg_offset, tc_k_pad(L, f4), f4, a8, s));
    TK_CUDA(tk_launch_gemm_tc_fmt(a8, (int)row_count, tc_k_pad(L, f4), L, e, f4, s));
    return TK_OK;
  }
  TK_CUDA(tk_launch_gemm_popc(rows, row_count, L->wpr64, L, nonneg_offset, e, s));
  return TK_OK;
}

// conv2d_ternary = im2col_quantize_pack + packed_gemm + affine epilogue,
// R:linalg.hpp:301-328, fused into two launches.
int tk_conv2d_ternary(tk_context* ctx, const tk_layer* L, const float* x,
                      int n, int h, int w, int mask_mode, float* out,
                      void* stream) {
  TK_ON_DEVICE(ctx);
  if (!ctx || !L) return TK_ERR_INVALID;
  if (!geom_ok(L->in_c, h, w, L->kh, L->kw, L->stride, L->pad) || n < 0)
    return TK_ERR_INVALID;
  tk_qparams q;
  int st = tk_make_qparams(L->ta1, L->ta2,
                           L->nonneg ? TK_MODE_ACTIVATION_NONNEG : TK_MODE_WEIGHT, &q);
  if (st != TK_OK) return st;
  if (mask_mode == TK_MASK_PRECOMPUTED && !L->masks_ready) return TK_ERR_MASKS;
  const int oh = (h + 2 * L->pad - L->kh) / L->stride + 1;
  const int ow = (w + 2 * L->pad - L->kw) / L->stride + 1;
  const size_t M = (size_t)n * oh * ow;
  if (M == 0) return TK_OK;
  cudaStream_t s = (cudaStream_t)stream;
  // nonneg activations on a tensor-core-shaped conv: the fused implicit-im2col
  // kernel (quantize into padded channel-last planes, 9 tap MMAs per tile, the
  // NCHW epilogue in the same kernel)
  if ((L->backend == TK_BACKEND_AUTO || L->backend == TK_BACKEND_TC_CONV) && tk_fconv_eligible(L, n, h, w))
    return tk_fconv_run(L, x, n, h, w, out, s);
  tk_epilogue e{TK_EPI_F32_NCHW, oh * ow, L->d_gain, L->d_bias, L->out_scale, out};
  const int be = tk_layer_get_backend(L, (int)M);
  const size_t rows_bytes = M * L->wpr64 * 8;
  if (tc_backend(be) && tk_tc_supported((int)M, L->out_c, L->k_pad)) {
    // im2col + quantize + level expansion in one kernel, then the GEMM
    const bool f4 = be == TK_BACKEND_TC_F4;
    const size_t m_pad = (M + 127) / 128 * 128;
    int8_t* a8 = (int8_t*)tk_workspace(ctx, tc_operand_bytes(L, m_pad, f4));
    if (!a8) return TK_ERR_CUDA;
    TK_CUDA(tk_launch_im2col_levels(x, n, L->in_c, h, w, L->kh, L->kw, L->stride, L->pad, q, L->nonneg,
                                    tc_k_pad(L, f4), f4, a8, ctx->d_err, s));
    TK_CUDA(tk_launch_gemm_tc_fmt(a8, (int)M, tc_k_pad(L, f4), L, e, f4, s));
    return TK_OK;
  }
  uint64_t* rows = (uint64_t*)tk_workspace(ctx, rows_bytes);
  if (!rows) return TK_ERR_CUDA;
  TK_CUDA(tk_launch_im2col(x, n, L->in_c, h, w, L->kh, L->kw, L->stride, L->pad,
                           q, rows, ctx->d_err, s));
  TK_CUDA(tk_launch_gemm_popc(rows, M, L->wpr64, L, L->nonneg, e, s));
  return TK_OK;
}

int tk_layer_k_pad(const tk_layer* L) { return L ? L->k_pad : -1; }
int tk_layer_k_pad_fp4(const tk_layer* L) { return L ? L->k_pad4 : -1; }

namespace {
int gemm_levels(tk_context* ctx, const tk_layer* L, const int8_t* a, int m_rows, int out_mode, void* out,
                bool fp4, void* stream) {
  if (!ctx || !L || m_rows < 0 || (out_mode != 0 && out_mode != 1)) return TK_ERR_INVALID;
  if (m_rows == 0) return TK_OK;
  if (!a || !out) return TK_ERR_INVALID;
  if (!tk_tc_supported(m_rows, L->out_c, L->k_pad)) return TK_ERR_UNSUPPORTED;
  tk_epilogue e{out_mode == 0 ? TK_EPI_I32 : TK_EPI_F32_ROWS, 1, L->d_gain, L->d_bias,
                L->out_scale, out};
  const cudaError_t ce = tk_launch_gemm_tc_fmt(a, m_rows, tc_k_pad(L, fp4), L, e, fp4, (cudaStream_t)stream);
  if (ce == cudaErrorNotSupported) return TK_ERR_UNSUPPORTED;
  TK_CUDA(ce);
  return TK_OK;
}

int quantize_levels(tk_context* ctx, const float* x, int rows, int n, float a1, float a2, int mode, int k_pad,
                    bool fp4, int8_t* out, void* stream) {
  if (!ctx || rows < 0 || n < 0 || k_pad < n || k_pad % (fp4 ? 256 : 128)) return TK_ERR_INVALID;
  tk_qparams q;
  const int st = tk_make_qparams(a1, a2, mode, &q);
  if (st != TK_OK) return st;
  TK_CUDA(tk_launch_quantize_levels(x, rows, n, q, k_pad, fp4, out, ctx->d_err, (cudaStream_t)stream));
  return TK_OK;
}
}  // namespace

int tk_gemm_levels(tk_context* ctx, const tk_layer* L, const int8_t* a_s8, int m_rows,
                   int out_mode, void* out, void* stream) {
  TK_ON_DEVICE(ctx);
  return gemm_levels(ctx, L, a_s8, m_rows, out_mode, out, false, stream);
}

int tk_gemm_levels_fp4(tk_context* ctx, const tk_layer* L, const uint8_t* a_fp4, int m_rows, int out_mode,
                       void* out, void* stream) {
  TK_ON_DEVICE(ctx);
  return gemm_levels(ctx, L, (const int8_t*)a_fp4, m_rows, out_mode, out, true, stream);
}

int tk_quantize_levels(tk_context* ctx, const float* x, int rows, int n, float a1, float a2,
                       int mode, int k_pad, int8_t* out, void* stream) {
  TK_ON_DEVICE(ctx);
  return quantize_levels(ctx, x, rows, n, a1, a2, mode, k_pad, false, out, stream);
}

int tk_quantize_levels_fp4(tk_context* ctx, const float* x, int rows, int n, float a1, float a2, int mode,
                           int k_pad, uint8_t* out, void* stream) {
  TK_ON_DEVICE(ctx);
  return quantize_levels(ctx, x, rows, n, a1, a2, mode, k_pad, true, (int8_t*)out, stream);
}

// R:linalg.hpp:332-343: a 1x1, pad-0 conv over [batch][in_c][1][1]
int tk_fully_connected_ternary(tk_context* ctx, const tk_layer* L,
                               const float* x, int batch, int mask_mode,
                               float* out, void* stream) {
  TK_ON_DEVICE(ctx);
  if (!ctx || !L) return TK_ERR_INVALID;
  if (L->kh != 1 || L->kw != 1 || L->pad != 0) return TK_ERR_INVALID;
  if (batch < 0) return TK_ERR_INVALID;
  tk_qparams q;
  int st = tk_make_qparams(L->ta1, L->ta2,
                           L->nonneg ? TK_MODE_ACTIVATION_NONNEG : TK_MODE_WEIGHT, &q);
  if (st != TK_OK) return st;
  if (mask_mode == TK_MASK_PRECOMPUTED && !L->masks_ready) return TK_ERR_MASKS;
  if (batch == 0) return TK_OK;
  cudaStream_t s = (cudaStream_t)stream;
  tk_epilogue e{TK_EPI_F32_ROWS, 1, L->d_gain, L->d_bias, L->out_scale, out};
  const int be = tk_layer_get_backend(L, batch);
  if (tc_backend(be) && tk_tc_supported(batch, L->out_c, L->k_pad)) {
    const bool f4 = be == TK_BACKEND_TC_F4;
    const size_t m_pad = ((size_t)batch + 127) / 128 * 128;
    int8_t* a8 = (int8_t*)tk_workspace(ctx, tc_operand_bytes(L, m_pad, f4));
    if (!a8) return TK_ERR_CUDA;
    TK_CUDA(tk_launch_quantize_levels(x, batch, L->in_c, q, tc_k_pad(L, f4), f4, a8, ctx->d_err, s));
    TK_CUDA(tk_launch_gemm_tc_fmt(a8, batch, tc_k_pad(L, f4), L, e, f4, s));
    return TK_OK;
  }
  uint64_t* rows = (uint64_t*)tk_workspace(ctx, (size_t)batch * L->wpr64 * 8);
  if (!rows) return TK_ERR_CUDA;
  TK_CUDA(tk_launch_quantize_pack(x, batch, L->in_c, q, rows, ctx->d_err, s));
  TK_CUDA(tk_launch_gemm_popc(rows, batch, L->wpr64, L, L->nonneg, e, s));
  return TK_OK;
}

}  // extern "C"

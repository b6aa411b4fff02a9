/*
 * ternkit_oracle.c -- plain-C restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see ternkit_oracle.h).  Built by oracle/Makefile
 * with -O2 -ffp-contract=off: the only fused multiply-adds are the explicit
 * fmaf() calls below, which restate the FMA contraction GCC applies to the
 * reference at its default -O3 -march=native (R:CMakeLists.txt:10-20).
 *
 * R: = /root/reference/proj/include/ternkit/
 */
#include "ternkit_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define LANES 32

/* R:codec.hpp:38-40 -- popcount(code) - 1; all four codes are valid */
int or_decode_lane(unsigned code) {
  code &= 3u;
  return (int)(code & 1u) + (int)(code >> 1) - 1;
}

/* R:codec.hpp:43-52 -- -1 -> 00, 0 -> 01 (canonical), +1 -> 11 */
int or_encode_lane(int value, unsigned* code) {
  if (value == -1) { *code = 0u; return OR_OK; }
  if (value == 0) { *code = 1u; return OR_OK; }
  if (value == 1) { *code = 3u; return OR_OK; }
  return OR_ERR_RANGE;
}

/* R:codec.hpp:84-86 */
size_t or_words_for_lanes(size_t n) { return (n + LANES - 1) / LANES; }

/* R:quantizer.hpp:30-32 */
static float clip(float v, float lo, float hi) {
  return v < lo ? lo : (v > hi ? hi : v);
}

/* R:quantizer.hpp:44-49 -- round(clip(p/a1,-1,0)) + round(clip(p/a2,0,1)),
 * round = nearbyintf under the default round-to-nearest-even mode. */
int or_quantize_weight_value(float p, float a1, float a2, int* level) {
  if (!isfinite(p)) return OR_ERR_NONFINITE;        /* R:quantizer.hpp:37-41 */
  float lo = nearbyintf(clip(p / a1, -1.0f, 0.0f));
  float hi = nearbyintf(clip(p / a2, 0.0f, 1.0f));
  *level = (int)lo + (int)hi;
  return OR_OK;
}

/* R:quantizer.hpp:51-60 -- round(clip(p/a1,0,1)) + round(clip((p-a1)/a2,0,1)) */
int or_quantize_activation_value(float p, float a1, float a2, int* level) {
  if (!isfinite(p)) return OR_ERR_NONFINITE;
  if (p < 0.0f) return OR_ERR_NEGATIVE;              /* R:quantizer.hpp:53-55 */
  float lo = nearbyintf(clip(p / a1, 0.0f, 1.0f));
  float hi = nearbyintf(clip((p - a1) / a2, 0.0f, 1.0f));
  *level = (int)lo + (int)hi;
  return OR_OK;
}

static int thresholds_ok(float a1, float a2) {
  return a1 > 0.0f && a2 > 0.0f;                      /* R:codec.hpp:61-65 */
}

/* R:codec.hpp:89-100 -- 32 lanes per u64, lane i at bits 2(i%32), padding
 * with the canonical zero code (kAuxi). */
int or_pack(const int8_t* values, size_t n, uint64_t* words) {
  size_t nw = or_words_for_lanes(n);
  for (size_t i = 0; i < nw; ++i) words[i] = OR_KAUXI;
  for (size_t i = 0; i < n; ++i) {
    unsigned code;
    if (or_encode_lane(values[i], &code) != OR_OK) return OR_ERR_RANGE;
    int sh = 2 * (int)(i % LANES);
    uint64_t* w = &words[i / LANES];
    *w = (*w & ~(3ull << sh)) | ((uint64_t)code << sh);
  }
  return OR_OK;
}

/* R:codec.hpp:107-117 */
int or_unpack(const uint64_t* words, size_t n, int8_t* values) {
  for (size_t i = 0; i < n; ++i) {
    unsigned code = (unsigned)(words[i / LANES] >> (2 * (i % LANES))) & 3u;
    values[i] = (int8_t)or_decode_lane(code);
  }
  return OR_OK;
}

/* R:quantizer.hpp:159-170 -- weight mode packs the level; activation mode
 * packs (level - 1) (the nonneg offset flag is carried out of band). */
int or_quantize_and_pack(const float* x, size_t n, float a1, float a2,
                         int mode, uint64_t* words) {
  if (!thresholds_ok(a1, a2)) return OR_ERR_INVALID;
  int8_t* q = (int8_t*)malloc(n ? n : 1);
  for (size_t i = 0; i < n; ++i) {
    int lv, st;
    st = mode == OR_MODE_WEIGHT ? or_quantize_weight_value(x[i], a1, a2, &lv)
                                : or_quantize_activation_value(x[i], a1, a2, &lv);
    if (st != OR_OK) { free(q); return st; }
    q[i] = (int8_t)(mode == OR_MODE_WEIGHT ? lv : lv - 1);
  }
  int st = or_pack(q, n, words);
  free(q);
  return st;
}

/* R:bitkernels.hpp:47-49 -- bit 2i set iff lane i of y is a zero code */
uint64_t or_ternary_zero_seed(uint64_t y) { return (y ^ (y >> 1)) & OR_KAUXI; }

/* R:bitkernels.hpp:55-63 -- xnor, then zero-operand lanes forced to 0b01 */
uint64_t or_ternary_multiply_word(uint64_t x, uint64_t y) {
  uint64_t xn = ~(x ^ y);
  uint64_t d = or_ternary_zero_seed(y);
  return (xn | d) & ~(d << 1);
}

/* R:bitkernels.hpp:76-85 -- sum popcount(TM) - 32 * words */
int64_t or_ternary_dot_words(const uint64_t* x, const uint64_t* y,
                             size_t words) {
  int64_t acc = 0;
  for (size_t i = 0; i < words; ++i)
    acc += __builtin_popcountll(or_ternary_multiply_word(x[i], y[i]));
  return acc - (int64_t)words * LANES;
}

/* R:bitkernels.hpp:116-123 (ternary_dot) and :151-159 (ternary_dot_nonneg) */
void or_ternary_dot_batched(const uint64_t* x, const uint64_t* y,
                            size_t words, size_t pairs, const int64_t* wsum,
                            int64_t* out) {
  for (size_t p = 0; p < pairs; ++p) {
    int64_t d = or_ternary_dot_words(x + p * words, y + p * words, words);
    out[p] = wsum ? d + wsum[p] : d;
  }
}

/* R:linalg.hpp:43-54 (ConvGeometry::validate / out_h / out_w) */
static int geom_ok(int c, int h, int w, int kh, int kw, int stride, int pad) {
  if (c <= 0 || kh <= 0 || kw <= 0 || stride <= 0 || pad < 0) return 0;
  if (h + 2 * pad < kh || w + 2 * pad < kw) return 0;
  return 1;
}

/* R:linalg.hpp:173-225 -- rows (n, oy, ox); lane (ky*kw+kx)*c + ci; padding
 * pixels enter the quantizer as 0.0f; each row is packed on its own. */
int or_im2col_quantize_pack(const float* x, int n, int c, int h, int w,
                            int kh, int kw, int stride, int pad, float a1,
                            float a2, int mode, uint64_t* rows) {
  if (!geom_ok(c, h, w, kh, kw, stride, pad) || n < 0) return OR_ERR_INVALID;
  if (!thresholds_ok(a1, a2)) return OR_ERR_INVALID;
  int oh = (h + 2 * pad - kh) / stride + 1, ow = (w + 2 * pad - kw) / stride + 1;
  size_t k = (size_t)c * kh * kw, wpr = or_words_for_lanes(k);
  float* patch = (float*)malloc(k * sizeof(float));
  size_t r = 0;
  int st = OR_OK;
  for (int b = 0; b < n && st == OR_OK; ++b) {
    const float* img = x + (size_t)b * c * h * w;
    for (int oy = 0; oy < oh && st == OR_OK; ++oy)
      for (int ox = 0; ox < ow && st == OR_OK; ++ox, ++r) {
        for (int ky = 0; ky < kh; ++ky)
          for (int kx = 0; kx < kw; ++kx) {
            int iy = oy * stride - pad + ky, ix = ox * stride - pad + kx;
            int in = iy >= 0 && iy < h && ix >= 0 && ix < w;
            float* dst = patch + (size_t)(ky * kw + kx) * c;
            for (int ci = 0; ci < c; ++ci)
              dst[ci] = in ? img[((size_t)ci * h + iy) * w + ix] : 0.0f;
          }
        st = or_quantize_and_pack(patch, k, a1, a2, mode, rows + r * wpr);
      }
  }
  free(patch);
  return st;
}

/* R:linalg.hpp:232-293 -- out[r*oc+o] = dot(row r, weight o) (+ wsum[o]
 * when the activations carry the nonneg offset); int32 row-major. */
void or_packed_gemm(const uint64_t* rows, size_t row_count, size_t wpr,
                    const uint64_t* weights, const int32_t* wsums, int oc,
                    int offset, int32_t* out) {
  for (size_t r = 0; r < row_count; ++r)
    for (int o = 0; o < oc; ++o) {
      int64_t base = offset ? wsums[o] : 0;
      out[r * oc + o] = (int32_t)(base + or_ternary_dot_words(
                                             rows + r * wpr,
                                             weights + (size_t)o * wpr, wpr));
    }
}

/* R:linalg.hpp:301-328 -- im2col + gemm + epilogue
 * y = gain[o] * (out_scale * acc) + bias[o]; GCC contracts the outer
 * multiply-add into one FMA at the reference's -O3 -march=native. */
int or_conv2d_ternary(const float* x, int n, int c, int h, int w,
                      int out_c, int kh, int kw, int stride, int pad,
                      const uint64_t* weights, const int32_t* wsums,
                      float a1, float a2, int nonneg, const float* gain,
                      const float* bias, float out_scale, float* out) {
  if (out_c <= 0) return OR_ERR_INVALID;
  if (!geom_ok(c, h, w, kh, kw, stride, pad)) return OR_ERR_INVALID;
  int oh = (h + 2 * pad - kh) / stride + 1, ow = (w + 2 * pad - kw) / stride + 1;
  size_t k = (size_t)c * kh * kw, wpr = or_words_for_lanes(k);
  size_t rows_n = (size_t)n * oh * ow, plane = (size_t)oh * ow;
  uint64_t* rows = (uint64_t*)malloc((rows_n ? rows_n : 1) * wpr * 8);
  int st = or_im2col_quantize_pack(x, n, c, h, w, kh, kw, stride, pad, a1, a2,
                                   nonneg ? OR_MODE_ACT_NONNEG : OR_MODE_WEIGHT,
                                   rows);
  if (st != OR_OK) { free(rows); return st; }
  int32_t* acc = (int32_t*)malloc((rows_n ? rows_n : 1) * out_c * 4);
  or_packed_gemm(rows, rows_n, wpr, weights, wsums, out_c, nonneg, acc);
  for (int b = 0; b < n; ++b)
    for (size_t p = 0; p < plane; ++p) {
      size_t r = (size_t)b * plane + p;
      for (int o = 0; o < out_c; ++o) {
        float g = gain ? gain[o] : 1.0f, bb = bias ? bias[o] : 0.0f;
        out[((size_t)b * out_c + o) * plane + p] =
            fmaf(g, out_scale * (float)acc[r * out_c + o], bb);
      }
    }
  free(acc);
  free(rows);
  return OR_OK;
}

/* R:linalg.hpp:70-91 -- gain = gamma / sqrt(var+eps) computed as
 * gamma * (1/sqrt), bias = beta - mean*gamma*inv_std (left to right). */
int or_fuse_bn(const float* mean, const float* var, const float* gamma,
               const float* beta, float eps, int c, float* gain,
               float* bias) {
  for (int i = 0; i < c; ++i) {
    float denom = var[i] + eps;
    if (!(denom > 0.0f)) return OR_ERR_INVALID;
    float inv_std = 1.0f / sqrtf(denom);
    gain[i] = gamma[i] * inv_std;
    /* beta - (mean*gamma)*inv_std: GCC contracts the final multiply-subtract */
    bias[i] = fmaf(-(mean[i] * gamma[i]), inv_std, beta[i]);
  }
  return OR_OK;
}

/* R:tinynet.hpp:720-730 -- z = max(z + (cal_gain*h + cal_bias | h), 0) */
void or_residual_relu_rows(float* z, const float* h, size_t count, int hidden,
                           const float* cal_gain, const float* cal_bias) {
  for (size_t i = 0; i < count; ++i) {
    size_t j = i % (size_t)hidden;
    float id = cal_gain ? fmaf(cal_gain[j], h[i], cal_bias[j]) : h[i];
    float v = z[i] + id;
    z[i] = v < 0.0f ? 0.0f : v; /* std::max(v, 0.0f) keeps -0.0f */
  }
}

void or_residual_relu_nchw(float* z, const float* skip, int n, int c,
                           int plane) {
  size_t count = (size_t)n * c * plane;
  for (size_t i = 0; i < count; ++i) {
    float v = z[i] + (skip ? skip[i] : 0.0f);
    z[i] = v < 0.0f ? 0.0f : v;
  }
}

/* Residual body restated from the reference composition pattern
 * (R:tinynet.hpp:713-735 with conv2d_ternary layers, see netdesc.h).
 * x: [n][c][h][w] f32; out must hold the final [n][c'][h'][w'] tensor.
 * Returns the final channel/height/width through the pointers. */
int or_net_body(const nd_block* blocks, int n_blocks, const float* x, int n,
                int c, int h, int w, float* out, int* oc, int* oh, int* ow) {
  size_t cur_n = (size_t)n * c * h * w;
  float* cur = (float*)malloc(cur_n * 4);
  memcpy(cur, x, cur_n * 4);
  int st = OR_OK;
  for (int bi = 0; bi < n_blocks && st == OR_OK; ++bi) {
    const nd_block* b = &blocks[bi];
    float* hbuf = cur;
    int hc = c, hh = h, hw = w;
    float* z = NULL;
    for (int j = 0; j < b->n_convs && st == OR_OK; ++j) {
      const nd_conv* cv = &b->conv[j];
      int zh = (hh + 2 * cv->pad - cv->k) / cv->stride + 1;
      int zw = (hw + 2 * cv->pad - cv->k) / cv->stride + 1;
      size_t wpr = or_words_for_lanes((size_t)cv->in_c * cv->k * cv->k);
      uint64_t* wp = (uint64_t*)malloc((size_t)cv->out_c * wpr * 8);
      int32_t* ws = (int32_t*)malloc((size_t)cv->out_c * 4);
      size_t kk = (size_t)cv->in_c * cv->k * cv->k;
      for (int o = 0; o < cv->out_c; ++o) {
        or_pack(cv->weights + (size_t)o * kk, kk, wp + (size_t)o * wpr);
        int32_t s = 0;
        for (size_t q = 0; q < kk; ++q) s += cv->weights[(size_t)o * kk + q];
        ws[o] = s;
      }
      z = (float*)malloc((size_t)n * cv->out_c * zh * zw * 4);
      st = or_conv2d_ternary(hbuf, n, hc, hh, hw, cv->out_c, cv->k, cv->k,
                             cv->stride, cv->pad, wp, ws, cv->ta1, cv->ta2, 1,
                             cv->gain, cv->bias, cv->out_scale, z);
      free(wp);
      free(ws);
      if (hbuf != cur) free(hbuf);
      hc = cv->out_c; hh = zh; hw = zw;
      if (j + 1 < b->n_convs) {
        size_t cnt = (size_t)n * hc * hh * hw;
        for (size_t i = 0; i < cnt; ++i) z[i] = z[i] < 0.0f ? 0.0f : z[i];
        hbuf = z;
      }
    }
    if (st != OR_OK) { free(z); break; }
    float* sc = cur;
    float* scbuf = NULL;
    if (b->has_down) {
      const nd_conv* cv = &b->down;
      size_t wpr = or_words_for_lanes((size_t)cv->in_c * cv->k * cv->k);
      size_t kk = (size_t)cv->in_c * cv->k * cv->k;
      uint64_t* wp = (uint64_t*)malloc((size_t)cv->out_c * wpr * 8);
      int32_t* ws = (int32_t*)malloc((size_t)cv->out_c * 4);
      for (int o = 0; o < cv->out_c; ++o) {
        or_pack(cv->weights + (size_t)o * kk, kk, wp + (size_t)o * wpr);
        int32_t s = 0;
        for (size_t q = 0; q < kk; ++q) s += cv->weights[(size_t)o * kk + q];
        ws[o] = s;
      }
      scbuf = (float*)malloc((size_t)n * hc * hh * hw * 4);
      st = or_conv2d_ternary(cur, n, c, h, w, cv->out_c, cv->k, cv->k,
                             cv->stride, cv->pad, wp, ws, cv->ta1, cv->ta2, 1,
                             cv->gain, cv->bias, cv->out_scale, scbuf);
      free(wp);
      free(ws);
      sc = scbuf;
    }
    if (st == OR_OK) or_residual_relu_nchw(z, sc, n, hc, hh * hw);
    free(scbuf);
    free(cur);
    cur = z;
    c = hc; h = hh; w = hw;
  }
  if (st == OR_OK) memcpy(out, cur, (size_t)n * c * h * w * 4);
  free(cur);
  *oc = c; *oh = h; *ow = w;
  return st;
}

/* R:tinynet.hpp:130-144 -- y[b][o] = bias[o] + sum_j x[b][j] * w[o][j],
 * accumulated left to right.  At the reference's -O3 -march=native GCC
 * vectorises the products 8 (then 4) at a time and adds them in order
 * (product rounded, then added), and contracts only the scalar tail
 * (< 4 terms) into FMAs; restated exactly (checked against oracle/_ref). */
void or_matmul_t(const float* x, const float* w, const float* bias, int batch,
                 int in_dim, int out_dim, float* y) {
  const int n8 = in_dim / 8 * 8;
  const int nv = n8 + ((in_dim - n8) >= 4 ? 4 : 0);
  for (int b = 0; b < batch; ++b)
    for (int o = 0; o < out_dim; ++o) {
      const float* xr = x + (size_t)b * in_dim;
      const float* wr = w + (size_t)o * in_dim;
      float acc = bias ? bias[o] : 0.0f;
      for (int j = 0; j < nv; ++j) {
        float prod = xr[j] * wr[j];
        acc = acc + prod;
      }
      for (int j = nv; j < in_dim; ++j) acc = fmaf(xr[j], wr[j], acc);
      y[(size_t)b * out_dim + o] = acc;
    }
}

/* ---- paper baselines (R:bitkernels.hpp:99-224) ---------------------------- */
int or_pack_binary(const int8_t* v, size_t n, uint64_t* words) {
  const size_t nw = (n + 63) / 64;
  for (size_t i = 0; i < nw; ++i) words[i] = 0;
  for (size_t i = 0; i < n; ++i) {
    if (v[i] != 1 && v[i] != -1) return OR_ERR_INVALID;
    if (v[i] == 1) words[i / 64] |= 1ull << (i % 64);
  }
  return OR_OK;
}

int64_t or_binary_dot(const uint64_t* x, const uint64_t* y, size_t words, size_t logical_len) {
  int64_t pop = 0;
  for (size_t i = 0; i < words; ++i) pop += __builtin_popcountll(~(x[i] ^ y[i]));
  return 2 * pop - 2 * (int64_t)words * 64 + (int64_t)logical_len;
}

double or_multibit_dot(const uint64_t* x, int m, const uint64_t* y, int k, const double* sx,
                       const double* sy, size_t words, size_t logical_len, int contract) {
  double acc = 0.0;
  for (int a = 0; a < m; ++a)
    for (int b = 0; b < k; ++b) {
      const double bd = (double)or_binary_dot(x + (size_t)a * words, y + (size_t)b * words, words, logical_len);
      const double s = sx[a] * sy[b];
      acc = contract ? fma(s, bd, acc) : acc + s * bd;
    }
  return acc;
}

/*
 * ternkit_oracle.h -- CPU restatement of the reference ternkit hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the
 * B200 kernels in paper_2008_05101_b200/csrc.  Only tests/, the smoke()
 * entry of __graft_entry__.py and bench.py's cpu_baseline leg may load it.
 * The product path never links or calls it.
 *
 * Every function restates the algorithm of the reference header it cites
 * (R: = /root/reference/proj/include/ternkit/).  Parity of this restatement
 * is pinned by tests/golden/ (fixtures produced by the reference itself,
 * see oracle/gen_golden.cpp) in tests/test_oracle_golden.py.
 */
#ifndef TERNKIT_ORACLE_H
#define TERNKIT_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#include "netdesc.h"

#ifdef __cplusplus
extern "C" {
#endif

/* status codes shared with include/ternkit_b200.h */
#define OR_OK 0
#define OR_ERR_INVALID 1    /* geometry / length / threshold problems */
#define OR_ERR_NONFINITE 4
#define OR_ERR_NEGATIVE 5
#define OR_ERR_RANGE 8

#define OR_MODE_WEIGHT 0
#define OR_MODE_ACT_NONNEG 1

#define OR_KAUXI 0x5555555555555555ull

int or_decode_lane(unsigned code);
int or_encode_lane(int value, unsigned* code);
size_t or_words_for_lanes(size_t n);

int or_quantize_weight_value(float p, float a1, float a2, int* level);
int or_quantize_activation_value(float p, float a1, float a2, int* level);

int or_pack(const int8_t* values, size_t n, uint64_t* words);
int or_unpack(const uint64_t* words, size_t n, int8_t* values);
int or_quantize_and_pack(const float* x, size_t n, float a1, float a2,
                         int mode, uint64_t* words);

uint64_t or_ternary_zero_seed(uint64_t y);
uint64_t or_ternary_multiply_word(uint64_t x, uint64_t y);
int64_t or_ternary_dot_words(const uint64_t* x, const uint64_t* y,
                             size_t words);
/* batched form: out[p] = dot(x[p], y[p]) (+ wsum[p] when wsum != NULL) */
void or_ternary_dot_batched(const uint64_t* x, const uint64_t* y,
                            size_t words, size_t pairs, const int64_t* wsum,
                            int64_t* out);

int or_im2col_quantize_pack(const float* x, int n, int c, int h, int w,
                            int kh, int kw, int stride, int pad, float a1,
                            float a2, int mode, uint64_t* rows);

void or_packed_gemm(const uint64_t* rows, size_t row_count, size_t wpr,
                    const uint64_t* weights, const int32_t* wsums, int oc,
                    int offset, int32_t* out);

int or_conv2d_ternary(const float* x, int n, int c, int h, int w,
                      int out_c, int kh, int kw, int stride, int pad,
                      const uint64_t* weights, const int32_t* wsums,
                      float a1, float a2, int nonneg, const float* gain,
                      const float* bias, float out_scale, float* out);

int or_fuse_bn(const float* mean, const float* var, const float* gamma,
               const float* beta, float eps, int c, float* gain,
               float* bias);

/* packed_forward block tail: z[i] = max(z[i] + id(h[i]), 0), id = cal affine
 * or identity; `hidden` is the channel count of the row-major [batch][hidden]
 * tensors (R:tinynet.hpp:720-730). */
void or_residual_relu_rows(float* z, const float* h, size_t count, int hidden,
                           const float* cal_gain, const float* cal_bias);
/* NCHW flavour of the same tail used for conv blocks. */
void or_residual_relu_nchw(float* z, const float* skip, int n, int c,
                           int plane);

int or_net_body(const nd_block* blocks, int n_blocks, const float* x, int n,
                int c, int h, int w, float* out, int* oc, int* oh, int* ow);
void or_matmul_t(const float* x, const float* w, const float* bias, int batch,
                 int in_dim, int out_dim, float* y);

/* ---- paper baselines (R:bitkernels.hpp:99-224) ------------------------- */
/* pack_binary: +1 -> bit 1, -1 -> bit 0, little-endian, zero-padded; returns
 * OR_ERR_INVALID for values outside {-1, +1} (R:bitkernels.hpp:170-182) */
int or_pack_binary(const int8_t* v, size_t n, uint64_t* words);
/* binary_dot_words (R:bitkernels.hpp:99-110) */
int64_t or_binary_dot(const uint64_t* x, const uint64_t* y, size_t words, size_t logical_len);
/* multibit_dot (R:bitkernels.hpp:196-222): planes [m][words], [k][words];
 * `contract` selects fma(sx*sy, bd, acc) (the reference build's FMA
 * contraction) over the two-rounding form */
double or_multibit_dot(const uint64_t* x, int m, const uint64_t* y, int k, const double* sx,
                       const double* sy, size_t words, size_t logical_len, int contract);

#ifdef __cplusplus
}
#endif
#endif

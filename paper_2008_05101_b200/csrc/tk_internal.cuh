// tk_internal.cuh -- shared definitions of the B200 ternary library.
//
// Storage contract (identical bytes to the reference, R:codec.hpp:14-20):
// a packed row is a sequence of u64 words, 32 lanes each, lane i at bits
// 2(i%32).  The kernels work on the little-endian u32 view: u32 word 2k holds
// lanes 0-15 of u64 word k, u32 word 2k+1 lanes 16-31.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>

#include <map>
#include <mutex>
#include <tuple>

#include "../../include/ternkit_b200.h"

// Experiment / profiling overrides (kernel phase knobs, tile-shape forcing,
// in-kernel timestamps).  Compiled in only with -DTK_PROFILE, for the A/B
// builds of tools/; the production library reads no environment variables
// and its kernels carry no profiling branches (TK_DBG(x) folds to 0).
#ifdef TK_PROFILE
#include <stdlib.h>
inline int tk_knob(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}
#define TK_DBG(x) (x)
#else
inline constexpr int tk_knob(const char*, int dflt) { return dflt; }
#define TK_DBG(x) 0
#endif

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device: raise it
// once per (kernel, current device), thread-safe (tk_api.cu).
cudaError_t tk_smem_attr(const void* kernel, int bytes);

// split-TF32 tensor-core stem conv 7x7/2 (tk_stem.cu)
int tk_launch_stem_tc(tk_context* ctx, const float* images, int n, int h, int w, const float* weights, float* out,
                      void* stream);

#define TK_KAUXI32 0x55555555u

struct tk_context {
  int device = 0;
  int num_sms = 148;
  unsigned long long* d_err = nullptr;  // first-error key, ~0 = none
  void* ws = nullptr;                   // scratch, grown on demand
  size_t ws_bytes = 0;
  void* pinned = nullptr;               // 8-byte host slot for the error word
};

// Every C-ABI entry that takes a context runs on the context's device and
// leaves the caller's current device as it found it.
struct tk_device_guard {
  int prev = -1, dev = -1;
  explicit tk_device_guard(const tk_context* c) {
    if (c && cudaGetDevice(&prev) == cudaSuccess && prev != c->device && cudaSetDevice(c->device) == cudaSuccess)
      dev = c->device;
  }
  ~tk_device_guard() {
    if (dev >= 0) cudaSetDevice(prev);
  }
  tk_device_guard(const tk_device_guard&) = delete;
  tk_device_guard& operator=(const tk_device_guard&) = delete;
};
#define TK_ON_DEVICE(ctx) const tk_device_guard tk_device_guard_(ctx)

struct tk_layer {
  tk_context* ctx = nullptr;
  int in_c = 0, out_c = 0, kh = 1, kw = 1, stride = 1, pad = 0;
  float tw1 = 1, tw2 = 1, ta1 = 1, ta2 = 1, out_scale = 1;
  int nonneg = 1;
  int K = 0;       // patch length in lanes
  int wpr64 = 0;   // u64 words per packed row
  int masks_ready = 0;
  int backend = TK_BACKEND_AUTO;
  // device copies
  uint64_t* d_words = nullptr;  // [out_c][wpr64] packed rows
  uint32_t* d_mask = nullptr;   // [out_c][2*wpr64] nonzero-lane masks (u32)
  int32_t* d_wsum = nullptr;    // [out_c] sum of decoded weights
  int32_t* d_zcnt = nullptr;    // [out_c] zero lanes per row incl. padding
  float* d_gain = nullptr;      // [out_c]
  float* d_bias = nullptr;      // [out_c]
  int8_t* d_w8 = nullptr;       // [k_pad/128][n_pad][128] s8 tensor-core operand
  int8_t* d_w4 = nullptr;       // [k_pad4/256][n_pad][128 B] FP4 (E2M1) operand
  int n_pad = 0, k_pad = 0;
  int k_pad4 = 0;               // K rounded up to the 256-level FP4 K block
  // host mirrors (PackedConvLayer::weights / weight_sums)
  uint64_t* h_words = nullptr;
  int32_t* h_wsum = nullptr;
  float* h_gain = nullptr;  // [out_c] folded affine (host copy for conv plans)
  float* h_bias = nullptr;
  // conv2d_ternary plans of the fused implicit-im2col kernel, per input shape
  // (n, h, w), built on first use (tk_net.cu)
  mutable std::mutex plan_mu;
  mutable std::map<std::tuple<int, int, int>, tk_net*> plans;
};

// conv2d_ternary through the fused implicit-im2col tensor-core conv
// (tk_net.cu): eligibility of a layer / input shape, the run, plan cleanup
bool tk_fconv_eligible(const tk_layer* L, int n, int h, int w);
int tk_fconv_run(const tk_layer* L, const float* x, int n, int h, int w, float* out, cudaStream_t s);
void tk_fconv_destroy_plans(tk_layer* L);

// Float thresholds that reproduce the reference quantizer exactly:
// lane code = (p > t0) | (p > t1) << 1.  `lo_ok` is the smallest valid input
// (0 for activations, -FLT_MAX for weights); anything else is an error.
struct tk_qparams {
  float t0, t1;
  int nonneg;  // activation mode: negative inputs are errors
};

// error keys: (position << 8) | code, kept as a running minimum so the
// reported error is the first one in the reference's evaluation order.
__device__ __forceinline__ void tk_raise(unsigned long long* err,
                                         unsigned long long pos, int code) {
  atomicMin(err, (pos << 8) | (unsigned long long)code);
}

// Quantize one float to its 2-bit lane code; returns 0xFF on error.
__device__ __forceinline__ uint32_t tk_code(float p, const tk_qparams& q) {
  const bool ok = q.nonneg ? (p >= 0.0f && p <= 3.402823466e38f)
                           : (fabsf(p) <= 3.402823466e38f);
  if (!ok) return 0xFFu;
  return (uint32_t)(p > q.t0) | ((uint32_t)(p > q.t1) << 1);
}

__device__ __forceinline__ int tk_error_code(float p, int nonneg) {
  if (!(fabsf(p) <= 3.402823466e38f)) return TK_ERR_NONFINITE;
  return (nonneg && p < 0.0f) ? TK_ERR_NEGATIVE : TK_OK;
}

// host helpers implemented in tk_api.cu
int tk_make_qparams(float a1, float a2, int mode, tk_qparams* q);
void* tk_workspace(tk_context* ctx, size_t bytes);

// launchers (tk_codec.cu)
cudaError_t tk_launch_quantize_pack(const float* x, size_t rows, size_t n,
                                    tk_qparams q, uint64_t* words,
                                    unsigned long long* err, cudaStream_t s);
cudaError_t tk_launch_pack_int8(const int8_t* v, size_t n, uint64_t* words,
                                unsigned long long* err, cudaStream_t s);
cudaError_t tk_launch_unpack(const uint64_t* words, size_t n, int8_t* v,
                             cudaStream_t s);
cudaError_t tk_launch_im2col(const float* x, int n, int c, int h, int w,
                             int kh, int kw, int stride, int pad, tk_qparams q,
                             uint64_t* rows, unsigned long long* err,
                             cudaStream_t s);
cudaError_t tk_launch_expand_rows_s8(const uint64_t* rows, size_t row_count,
                                     int wpr64, int offset, int k_pad,
                                     int8_t* out, cudaStream_t s);
cudaError_t tk_launch_quantize_s8(const float* x, size_t rows, size_t n,
                                  tk_qparams q, int k_pad, int8_t* out,
                                  unsigned long long* err, cudaStream_t s);
// fp4: E2M1 nibbles, [k_pad/256][m_pad][128 B] (k_pad a multiple of 256)
cudaError_t tk_launch_expand_rows(const uint64_t* rows, size_t row_count, int wpr64, int offset, int k_pad,
                                  bool fp4, int8_t* out, cudaStream_t s);
// im2col_quantize_pack straight into the level operand (s8 or fp4 layout)
cudaError_t tk_launch_im2col_levels(const float* x, int n, int c, int h, int w, int kh, int kw, int stride, int pad,
                                    tk_qparams q, int offset, int k_pad, bool fp4, int8_t* out,
                                    unsigned long long* err, cudaStream_t s);
cudaError_t tk_launch_quantize_levels(const float* x, size_t rows, size_t n, tk_qparams q, int k_pad, bool fp4,
                                      int8_t* out, unsigned long long* err, cudaStream_t s);

// launchers (tk_popc.cu)
// seed: optional [pairs][words] zero seeds (premask form), else derived from y
cudaError_t tk_launch_dot_batched(const uint64_t* x, const uint64_t* y, const uint64_t* seed, size_t words,
                                  size_t pairs, const int64_t* wsum, int64_t* out, cudaStream_t s);
// epilogue modes of the GEMM kernels
enum { TK_EPI_I32 = 0, TK_EPI_F32_NCHW = 1, TK_EPI_F32_ROWS = 2 };
struct tk_epilogue {
  int mode;
  int plane;          // oh*ow (NCHW mode)
  const float* gain;  // [N]
  const float* bias;  // [N]
  float out_scale;
  void* out;
};
cudaError_t tk_launch_gemm_popc(const uint64_t* rows, size_t M, int wpr64,
                                const tk_layer* L, int offset, tk_epilogue e,
                                cudaStream_t s);

// launchers (tk_tc.cu)
bool tk_tc_supported(int M, int N, int k_pad);
cudaError_t tk_launch_gemm_tc_fmt(const int8_t* a, int M, int k_pad, const tk_layer* L, tk_epilogue e, bool fp4,
                                  cudaStream_t s);
cudaError_t tk_launch_gemm_tc(const int8_t* a_s8, int M, int k_pad,
                              const tk_layer* L, tk_epilogue e,
                              cudaStream_t s);

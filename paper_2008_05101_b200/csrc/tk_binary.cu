// tk_binary.cu -- the paper's comparison baselines on the GPU (SURVEY.md
// §8(f) F3): the binary XNOR-popcount inner product (Eq. 1) and the
// bit-plane decomposed multi-bit inner product (Eq. 2), with the reference's
// packing and arithmetic (R:include/ternkit/bitkernels.hpp:99-224).
//
// * pack_binary: 1 bit per element (+1 -> 1, -1 -> 0), little-endian bit
//   order, zero-padded last u64 word; other values are rejected.
// * binary_dot = 2 * popc(~(x ^ y)) - 2 * 64 * words + logical_len (the
//   padding bits match in both operands and cancel).
// * multibit_dot = sum_m sum_k sx[m] * sy[k] * (double)binary_dot(x_m, y_k),
//   accumulated in double in (m, k) order -- bit-identical to the reference.
#include "tk_internal.cuh"

namespace {

__global__ void k_pack_binary(const int8_t* __restrict__ v, size_t n, uint64_t* __restrict__ words,
                              size_t nwords, unsigned long long* err) {
  for (size_t w = blockIdx.x * (size_t)blockDim.x + threadIdx.x; w < nwords; w += (size_t)gridDim.x * blockDim.x) {
    uint64_t out = 0;
    const size_t base = w * 64;
    for (int i = 0; i < 64; ++i) {
      const size_t idx = base + i;
      if (idx >= n) break;
      const int8_t x = v[idx];
      if (x != 1 && x != -1) {
        tk_raise(err, (unsigned long long)idx, TK_ERR_RANGE);
      } else if (x == 1) {
        out |= 1ull << i;
      }
    }
    words[w] = out;
  }
}

// one warp per pair; u64 words, 64-bit popcounts
__global__ void k_binary_dot_batched(const uint64_t* __restrict__ x, const uint64_t* __restrict__ y, size_t words,
                                     size_t logical_len, size_t pairs, int64_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const size_t nwarps = ((size_t)gridDim.x * blockDim.x) >> 5;
  for (size_t p = warp; p < pairs; p += nwarps) {
    const uint64_t* xp = x + p * words;
    const uint64_t* yp = y + p * words;
    long long pop = 0;
    for (size_t i = lane; i < words; i += 32) pop += __popcll(~(__ldg(xp + i) ^ __ldg(yp + i)));
#pragma unroll
    for (int o = 16; o; o >>= 1) pop += __shfl_xor_sync(0xffffffffu, pop, o);
    if (lane == 0) out[p] = 2 * pop - 2 * (long long)words * 64 + (long long)logical_len;
  }
}

// x planes [M][pairs][words], y planes [K][pairs][words]; one warp per pair:
// the M*K binary dots, then the double accumulation in the reference's order
__global__ void k_multibit_dot_batched(const uint64_t* __restrict__ x, const uint64_t* __restrict__ y, int M, int K,
                                       const double* __restrict__ sx, const double* __restrict__ sy, size_t words,
                                       size_t logical_len, size_t pairs, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const size_t nwarps = ((size_t)gridDim.x * blockDim.x) >> 5;
  const size_t plane = pairs * words;
  for (size_t p = warp; p < pairs; p += nwarps) {
    double acc = 0.0;
    for (int m = 0; m < M; ++m)
      for (int k = 0; k < K; ++k) {
        const uint64_t* xp = x + m * plane + p * words;
        const uint64_t* yp = y + k * plane + p * words;
        long long pop = 0;
        for (size_t i = lane; i < words; i += 32) pop += __popcll(~(__ldg(xp + i) ^ __ldg(yp + i)));
#pragma unroll
        for (int o = 16; o; o >>= 1) pop += __shfl_xor_sync(0xffffffffu, pop, o);
        const long long bd = 2 * pop - 2 * (long long)words * 64 + (long long)logical_len;
        // acc += sx[m] * sy[k] * bd: (sx*sy) rounded, times bd rounded, then the add
        acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(__ldg(sx + m), __ldg(sy + k)), (double)bd));
      }
    if (lane == 0) out[p] = acc;
  }
}

unsigned grid_of(size_t work, unsigned per) {
  size_t g = (work + per - 1) / per;
  if (g > 148u * 32u) g = 148u * 32u;
  return (unsigned)(g ? g : 1);
}

}  // namespace

extern "C" {

int tk_pack_binary(tk_context* ctx, const int8_t* values, size_t n, uint64_t* words, void* stream) {
  TK_ON_DEVICE(ctx);
  if (!ctx || (n && (!values || !words))) return TK_ERR_INVALID;
  const size_t nwords = (n + 63) / 64;
  if (nwords == 0) return TK_OK;
  k_pack_binary<<<grid_of(nwords, 256), 256, 0, (cudaStream_t)stream>>>(values, n, words, nwords, ctx->d_err);
  return cudaGetLastError() == cudaSuccess ? TK_OK : TK_ERR_CUDA;
}

int tk_binary_dot_batched(tk_context* ctx, const uint64_t* x, const uint64_t* y, size_t words, size_t logical_len,
                          size_t pairs, int64_t* out, void* stream) {
  TK_ON_DEVICE(ctx);
  if (!ctx || (pairs && (!x || !y || !out)) || logical_len > words * 64) return TK_ERR_INVALID;
  if (pairs == 0) return TK_OK;
  k_binary_dot_batched<<<grid_of(pairs, 8), 256, 0, (cudaStream_t)stream>>>(x, y, words, logical_len, pairs, out);
  return cudaGetLastError() == cudaSuccess ? TK_OK : TK_ERR_CUDA;
}

int tk_multibit_dot_batched(tk_context* ctx, const uint64_t* x_planes, int m, const uint64_t* y_planes, int k,
                            const double* x_scales, const double* y_scales, size_t words, size_t logical_len,
                            size_t pairs, double* out, void* stream) {
  TK_ON_DEVICE(ctx);
  if (!ctx || m <= 0 || k <= 0 || logical_len > words * 64) return TK_ERR_INVALID;  // R:bitkernels.hpp:199-203
  if (pairs && (!x_planes || !y_planes || !x_scales || !y_scales || !out)) return TK_ERR_INVALID;
  if (pairs == 0) return TK_OK;
  k_multibit_dot_batched<<<grid_of(pairs, 8), 256, 0, (cudaStream_t)stream>>>(
      x_planes, y_planes, m, k, x_scales, y_scales, words, logical_len, pairs, out);
  return cudaGetLastError() == cudaSuccess ? TK_OK : TK_ERR_CUDA;
}

}  // extern "C"

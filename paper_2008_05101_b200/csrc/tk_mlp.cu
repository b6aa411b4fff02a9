// tk_mlp.cu -- the float pieces of the reference's packed_forward
// (R:tinynet.hpp:713-735) for the FATN models: the stem / head dense layers
// (detail::matmul_t) and the per-block calibrated skip-add + ReLU.
//
// Exactness: both follow the reference build's arithmetic operation by
// operation (oracle/ternkit_oracle.c or_matmul_t / or_residual_relu_rows,
// pinned against the compiled reference by tests/golden).  nvcc would
// contract a*b + c into an FMA, so every multiply / add is an explicit
// round-to-nearest intrinsic.
#include "tk_internal.cuh"

namespace {

// y[b][o] = bias[o] + sum_j x[b][j] * w[o][j] in the reference build's order:
// the first n8 + (4 if >= 4 remain) terms are product-rounded then added one
// by one (GCC's vectorized reduction keeps the sequential order here), the
// scalar tail is FMA-contracted.  One thread per output.
__global__ void k_matmul_t(const float* __restrict__ x, const float* __restrict__ w,
                           const float* __restrict__ bias, int batch, int in_dim, int out_dim,
                           float* __restrict__ y) {
  const int n8 = in_dim / 8 * 8;
  const int nv = n8 + ((in_dim - n8) >= 4 ? 4 : 0);
  const long long total = (long long)batch * out_dim;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(i / out_dim), o = (int)(i - (long long)b * out_dim);
    const float* xr = x + (size_t)b * in_dim;
    const float* wr = w + (size_t)o * in_dim;
    float acc = bias ? __ldg(bias + o) : 0.0f;
    for (int j = 0; j < nv; ++j) acc = __fadd_rn(acc, __fmul_rn(__ldg(xr + j), __ldg(wr + j)));
    for (int j = nv; j < in_dim; ++j) acc = __fmaf_rn(__ldg(xr + j), __ldg(wr + j), acc);
    y[i] = acc;
  }
}

// z[i] = max(z[i] + (cal ? fmaf(cal_gain[j], h[i], cal_bias[j]) : h[i]), 0),
// j = i % hidden (R:tinynet.hpp:720-730; std::max keeps -0.0)
__global__ void k_residual_relu_rows(float* __restrict__ z, const float* __restrict__ h, long long count,
                                     int hidden, const float* __restrict__ cal_gain,
                                     const float* __restrict__ cal_bias) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(i % hidden);
    const float id = cal_gain ? __fmaf_rn(__ldg(cal_gain + j), h[i], __ldg(cal_bias + j)) : h[i];
    const float v = __fadd_rn(z[i], id);
    z[i] = v < 0.0f ? 0.0f : v;
  }
}

// in-place ReLU with the reference's std::max(v, 0.0f) semantics
__global__ void k_relu(float* __restrict__ z, long long count) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    const float v = z[i];
    z[i] = v < 0.0f ? 0.0f : v;
  }
}

// Dense fp32 layer for the ResNet head (outside the ternary path; no
// reference operation order to follow): y[b][o] = bias[o] + sum_k x[b][k] w[o][k]
// as one fp32 FMA chain in k order.  32 x 32 output tiles (ResNet head b256:
// 256 CTAs, not 64), 64 threads with 4 x 4 outputs each, K staged through
// shared memory 32 at a time; the next K chunk is loaded into registers while
// the current one is multiplied (the chunk loads are L2/HBM-latency bound).
constexpr int kDT = 32, kDK = 32;
__global__ void __launch_bounds__(64) k_dense_f32(const float* __restrict__ x, const float* __restrict__ w,
                                                  const float* __restrict__ bias, int batch, int in_dim,
                                                  int out_dim, float* __restrict__ y) {
  __shared__ float sx[kDK][kDT + 4], sw[kDK][kDT + 4];  // [k][row]
  const int b0 = blockIdx.y * kDT, o0 = blockIdx.x * kDT;
  const int tx = threadIdx.x & 7, ty = threadIdx.x >> 3;  // outputs (b0 + ty*4 + i, o0 + tx*4 + j)
  // loads: 16 rows x 32 k per matrix and pass, thread t -> row (t >> 3) + 8 q, k = 4 (t & 7) .. +3
  const int lr = threadIdx.x >> 3, lk = (threadIdx.x & 7) * 4;
  float4 px[4], pw[4];
  auto load = [&](int k0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = lr + 8 * q, k = k0 + lk;
      float4 vx = make_float4(0.0f, 0.0f, 0.0f, 0.0f), vw = vx;
      if (b0 + r < batch) {
        const float* src = x + (size_t)(b0 + r) * in_dim + k;
        if (k + 3 < in_dim && ((in_dim & 3) == 0)) vx = __ldg(reinterpret_cast<const float4*>(src));
        else {
          vx.x = k < in_dim ? __ldg(src) : 0.0f;
          vx.y = k + 1 < in_dim ? __ldg(src + 1) : 0.0f;
          vx.z = k + 2 < in_dim ? __ldg(src + 2) : 0.0f;
          vx.w = k + 3 < in_dim ? __ldg(src + 3) : 0.0f;
        }
      }
      if (o0 + r < out_dim) {
        const float* src = w + (size_t)(o0 + r) * in_dim + k;
        if (k + 3 < in_dim && ((in_dim & 3) == 0)) vw = __ldg(reinterpret_cast<const float4*>(src));
        else {
          vw.x = k < in_dim ? __ldg(src) : 0.0f;
          vw.y = k + 1 < in_dim ? __ldg(src + 1) : 0.0f;
          vw.z = k + 2 < in_dim ? __ldg(src + 2) : 0.0f;
          vw.w = k + 3 < in_dim ? __ldg(src + 3) : 0.0f;
        }
      }
      px[q] = vx;
      pw[q] = vw;
    }
  };
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
  load(0);
  for (int k0 = 0; k0 < in_dim; k0 += kDK) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = lr + 8 * q;
      sx[lk][r] = px[q].x; sx[lk + 1][r] = px[q].y; sx[lk + 2][r] = px[q].z; sx[lk + 3][r] = px[q].w;
      sw[lk][r] = pw[q].x; sw[lk + 1][r] = pw[q].y; sw[lk + 2][r] = pw[q].z; sw[lk + 3][r] = pw[q].w;
    }
    __syncthreads();
    if (k0 + kDK < in_dim) load(k0 + kDK);  // in flight while this chunk is multiplied
#pragma unroll
    for (int kk = 0; kk < kDK; ++kk) {
      float xv[4], wv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        xv[i] = sx[kk][ty * 4 + i];
        wv[i] = sw[kk][tx * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = __fmaf_rn(xv[i], wv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int b = b0 + ty * 4 + i;
    if (b >= batch) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int o = o0 + tx * 4 + j;
      if (o < out_dim) y[(size_t)b * out_dim + o] = __fadd_rn(acc[i][j], bias ? __ldg(bias + o) : 0.0f);
    }
  }
}

unsigned grid_of(long long work) {
  const long long g = (work + 255) / 256;
  return (unsigned)(g < 1 ? 1 : (g > 148 * 32 ? 148 * 32 : g));
}

}  // namespace

extern "C" {

int tk_matmul_t(tk_context* ctx, const float* x, const float* w, const float* bias, int batch, int in_dim,
                int out_dim, int relu, float* y, void* stream) {
  TK_ON_DEVICE(ctx);
  if (!ctx || !x || !w || !y || batch < 0 || in_dim <= 0 || out_dim <= 0) return TK_ERR_INVALID;
  const long long total = (long long)batch * out_dim;
  if (total == 0) return TK_OK;
  cudaStream_t s = (cudaStream_t)stream;
  k_matmul_t<<<grid_of(total), 256, 0, s>>>(x, w, bias, batch, in_dim, out_dim, y);
  if (relu) k_relu<<<grid_of(total), 256, 0, s>>>(y, total);
  return cudaGetLastError() == cudaSuccess ? TK_OK : TK_ERR_CUDA;
}

int tk_dense_f32(tk_context* ctx, const float* x, const float* w, const float* bias, int batch, int in_dim,
                 int out_dim, float* y, void* stream) {
  TK_ON_DEVICE(ctx);
  if (!ctx || !x || !w || !y || batch < 0 || in_dim <= 0 || out_dim <= 0) return TK_ERR_INVALID;
  if (batch == 0) return TK_OK;
  const dim3 grid((out_dim + kDT - 1) / kDT, (batch + kDT - 1) / kDT);
  k_dense_f32<<<grid, 64, 0, (cudaStream_t)stream>>>(x, w, bias, batch, in_dim, out_dim, y);
  return cudaGetLastError() == cudaSuccess ? TK_OK : TK_ERR_CUDA;
}

int tk_residual_relu_rows(tk_context* ctx, float* z, const float* h, long long count, int hidden,
                          const float* cal_gain, const float* cal_bias, void* stream) {
  TK_ON_DEVICE(ctx);
  if (!ctx || !z || !h || count < 0 || hidden <= 0 || count % hidden) return TK_ERR_INVALID;
  if ((cal_gain == nullptr) != (cal_bias == nullptr)) return TK_ERR_INVALID;
  if (count == 0) return TK_OK;
  k_residual_relu_rows<<<grid_of(count), 256, 0, (cudaStream_t)stream>>>(z, h, count, hidden, cal_gain, cal_bias);
  return cudaGetLastError() == cudaSuccess ? TK_OK : TK_ERR_CUDA;
}

}  // extern "C"

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
// in fp32.  32 x 32 output tiles (ResNet head b256: 256 CTAs); the K range
// is split over 4 groups of 64 threads (4 x 4 outputs per thread, one fp32
// FMA chain per K quarter), each streaming its quarter through a 3-stage
// cp.async ring of 32-wide chunks; the four partial sums are added in group
// order at the end (deterministic).  One warp per scheduler was latency
// bound (81 / 29 us for the b256 head); 8 warps per CTA hide it.
constexpr int kDT = 32, kDK = 32, kDS = 3, kDG = 4;
struct DenseSmem {
  float x[kDG][kDS][kDT][kDK + 4];  // [group][stage][row][k]
  float w[kDG][kDS][kDT][kDK + 4];
};
__global__ void __launch_bounds__(64 * kDG) k_dense_f32(const float* __restrict__ x, const float* __restrict__ w,
                                                        const float* __restrict__ bias, int batch, int in_dim,
                                                        int out_dim, float* __restrict__ y) {
  extern __shared__ __align__(16) uint8_t dense_raw[];
  DenseSmem& sm = *reinterpret_cast<DenseSmem*>(dense_raw);
  const int g = threadIdx.x >> 6, t = threadIdx.x & 63;
  const int b0 = blockIdx.y * kDT, o0 = blockIdx.x * kDT;
  const int tx = t & 7, ty = t >> 3;  // outputs (b0 + ty + 8 i, o0 + tx + 8 j)
  const bool vec = (in_dim & 3) == 0;
  const int nch_all = (in_dim + kDK - 1) / kDK, per = (nch_all + kDG - 1) / kDG;
  const int c_begin = g * per, nch = max(0, min(nch_all, c_begin + per) - c_begin);
  const int nmax = per;  // chunk count of the largest group (uniform trip count for the barriers)
  auto stage = [&](int c) {  // chunk c of this group: rows t / 8 + 8 q, k = 4 (t % 8) .. +3
    const int st = c % kDS, k0 = (c_begin + c) * kDK, lk = (t & 7) * 4;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = (t >> 3) + 8 * q, k = k0 + lk;
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        const int row = (m ? o0 : b0) + r, rows = m ? out_dim : batch;
        const float* src = (m ? w : x) + (size_t)row * in_dim + k;
        float* dst = m ? &sm.w[g][st][r][lk] : &sm.x[g][st][r][lk];
        if (vec && row < rows && k + 3 < in_dim) {
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                       "l"(src)
                       : "memory");
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e) dst[e] = (row < rows && k + e < in_dim) ? __ldg(src + e) : 0.0f;
        }
      }
    }
  };
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
  for (int c = 0; c < kDS - 1; ++c) {
    if (c < nch) stage(c);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int c = 0; c < nmax; ++c) {
    asm volatile("cp.async.wait_group %0;" ::"n"(kDS - 2) : "memory");
    __syncthreads();  // chunk c landed; chunk c - 1's slot is free
    if (c + kDS - 1 < nch) stage(c + kDS - 1);
    asm volatile("cp.async.commit_group;" ::: "memory");
    if (c < nch) {
      const int st = c % kDS;
      // 4 k at a time as float4 rows; a thread's rows are 8 apart, so the 8
      // (4) distinct rows a warp reads sit in distinct 16-byte bank groups
#pragma unroll
      for (int kk = 0; kk < kDK; kk += 4) {
        float4 xq[4], wq[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          xq[i] = *reinterpret_cast<const float4*>(&sm.x[g][st][ty + 8 * i][kk]);
          wq[i] = *reinterpret_cast<const float4*>(&sm.w[g][st][tx + 8 * i][kk]);
        }
#pragma unroll
        for (int e = 0; e < 4; ++e)
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float xv = e == 0 ? xq[i].x : e == 1 ? xq[i].y : e == 2 ? xq[i].z : xq[i].w;
              const float wv = e == 0 ? wq[j].x : e == 1 ? wq[j].y : e == 2 ? wq[j].z : wq[j].w;
              acc[i][j] = __fmaf_rn(xv, wv, acc[i][j]);
            }
      }
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  // partial sums of groups 1..3 through shared memory (the x slots), added in group order by group 0
  float* part = &sm.x[0][0][0][0];
  if (g > 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) part[((g - 1) * 16 + i * 4 + j) * 64 + t] = acc[i][j];
  }
  __syncthreads();
  if (g > 0) return;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int b = b0 + ty + 8 * i;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float v = acc[i][j];
#pragma unroll
      for (int h = 0; h < kDG - 1; ++h) v = __fadd_rn(v, part[(h * 16 + i * 4 + j) * 64 + t]);
      const int o = o0 + tx + 8 * j;
      if (b < batch && o < out_dim) y[(size_t)b * out_dim + o] = __fadd_rn(v, bias ? __ldg(bias + o) : 0.0f);
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
  if (tk_smem_attr((const void*)k_dense_f32, (int)sizeof(DenseSmem)) != cudaSuccess) return TK_ERR_CUDA;
  k_dense_f32<<<grid, 64 * kDG, sizeof(DenseSmem), (cudaStream_t)stream>>>(x, w, bias, batch, in_dim, out_dim, y);
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

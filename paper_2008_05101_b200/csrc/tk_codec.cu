// tk_codec.cu -- HBM-bound packing kernels: quantize+pack, im2col with fused
// quantize+pack, int8 pack/unpack and the 2-bit -> s8 operand expansion used
// by the tensor-core GEMM.
//
// The quantizer never divides: tk_make_qparams() turns (alpha1, alpha2) into
// two float thresholds that reproduce round(clip(p/a)) of the reference
// bit-exactly (R:quantizer.hpp:44-60), so a lane costs two FSETPs.
#include "tk_internal.cuh"

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ uint32_t lane_word16(const float v[16], int valid,
                                                const tk_qparams& q,
                                                unsigned long long* err,
                                                unsigned long long pos0) {
  uint32_t word = TK_KAUXI32;  // padding lanes keep the canonical zero code
  int first_bad = -1, bad_code = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    if (i < valid) {
      const uint32_t c = tk_code(v[i], q);
      if (c == 0xFFu) {
        if (first_bad < 0) {
          first_bad = i;
          bad_code = tk_error_code(v[i], q.nonneg);
        }
      } else {
        word = (word & ~(3u << (2 * i))) | (c << (2 * i));
      }
    }
  }
  if (first_bad >= 0) tk_raise(err, pos0 + first_bad, bad_code);
  return word;
}

// One thread per output u32 word (16 lanes) of one row.
// R:quantizer.hpp:159-170 (per row), R:codec.hpp:89-100 (layout).
__global__ void k_quantize_pack(const float* __restrict__ x, size_t rows,
                                size_t n, int w32pr, tk_qparams q,
                                uint32_t* __restrict__ out,
                                unsigned long long* err, bool vec4) {
  const size_t total = rows * (size_t)w32pr;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
       t += (size_t)gridDim.x * blockDim.x) {
    const size_t r = t / w32pr;
    const int j = (int)(t - r * w32pr);
    const size_t l0 = (size_t)j * 16;
    const int valid = l0 >= n ? 0 : (int)min((size_t)16, n - l0);
    const float* src = x + r * n + l0;
    float v[16];
    if (vec4 && valid == 16) {
      const float4* s4 = reinterpret_cast<const float4*>(src);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float4 f = __ldg(s4 + i);
        v[4 * i] = f.x; v[4 * i + 1] = f.y; v[4 * i + 2] = f.z; v[4 * i + 3] = f.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = i < valid ? __ldg(src + i) : 0.0f;
    }
    out[t] = lane_word16(v, valid, q, err, r * n + l0);
  }
}

// im2col + quantize + pack from NCHW floats.  R:linalg.hpp:173-225: row r =
// (b, oy, ox); lane (ky*kw + kx)*c + ci; padding pixels enter as 0.0f.
__global__ void k_im2col(const float* __restrict__ x, int n, int c, int h,
                         int w, int kh, int kw, int stride, int pad, int oh,
                         int ow, int K, int w32pr, tk_qparams q,
                         uint32_t* __restrict__ out, unsigned long long* err) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // (expand waits for this grid)
  const size_t rows = (size_t)n * oh * ow;
  const size_t total = rows * (size_t)w32pr;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
       t += (size_t)gridDim.x * blockDim.x) {
    const size_t r = t / w32pr;
    const int j = (int)(t - r * w32pr);
    const int b = (int)(r / ((size_t)oh * ow));
    const int p = (int)(r - (size_t)b * oh * ow);
    const int oy = p / ow, ox = p - (p / ow) * ow;
    const int l0 = j * 16;
    const int valid = l0 >= K ? 0 : min(16, K - l0);
    int kpos = l0 / c, ci = l0 - kpos * c;
    int ky = kpos / kw, kx = kpos - ky * kw;
    const float* img = x + (size_t)b * c * h * w;
    float v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float val = 0.0f;
      if (i < valid) {
        const int iy = oy * stride - pad + ky, ix = ox * stride - pad + kx;
        if (iy >= 0 && iy < h && ix >= 0 && ix < w)
          val = __ldg(img + ((size_t)ci * h + iy) * w + ix);
        if (++ci == c) {
          ci = 0;
          if (++kx == kw) { kx = 0; ++ky; }
        }
      }
      v[i] = val;
    }
    out[t] = lane_word16(v, valid, q, err, r * (size_t)K + l0);
  }
}

// pack(span<const int8_t>) R:codec.hpp:89-100; out-of-range -> TK_ERR_RANGE
__global__ void k_pack_int8(const int8_t* __restrict__ v, size_t n,
                            uint32_t* __restrict__ out, size_t w32,
                            unsigned long long* err) {
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < w32;
       t += (size_t)gridDim.x * blockDim.x) {
    uint32_t word = TK_KAUXI32;
    const size_t l0 = t * 16;
    for (int i = 0; i < 16; ++i) {
      if (l0 + i >= n) break;
      const int val = v[l0 + i];
      if (val < -1 || val > 1) {
        tk_raise(err, l0 + i, TK_ERR_RANGE);
        break;
      }
      const uint32_t code = val < 0 ? 0u : (val == 0 ? 1u : 3u);
      word = (word & ~(3u << (2 * i))) | (code << (2 * i));
    }
    out[t] = word;
  }
}

// unpack R:codec.hpp:107-117: value = popcount(code) - 1
__global__ void k_unpack(const uint32_t* __restrict__ words, size_t n,
                         int8_t* __restrict__ v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const uint32_t code = (words[i / 16] >> (2 * (i % 16))) & 3u;
    v[i] = (int8_t)(__popc(code) - 1);
  }
}

// 4 lane codes (8 bits) -> 4 s8 levels through one PRMT: selector nibble k =
// code_k indexes the byte table `tbl`.
__device__ __forceinline__ uint32_t expand4(uint32_t bits8, uint32_t tbl) {
  const uint32_t s = (bits8 & 0x3u) | ((bits8 & 0xCu) << 2) |
                     ((bits8 & 0x30u) << 4) | ((bits8 & 0xC0u) << 6);
  return __byte_perm(tbl, 0, s);
}

// Packed rows -> s8 tensor-core operand [rows][k_pad].  Level = decoded lane
// value, +1 when the rows carry the nonneg offset (codes -> {0,1,2}), so the
// integer MMA result equals packed_gemm's offset-corrected dot directly.
// F4: E2M1 nibbles instead, 16 lanes -> 8 bytes, layout [k/256][m_pad][128 B]
// with the even lane in the low nibble (the kind::mxf4 operand format).
__device__ __forceinline__ uint32_t e2m1_of_level(int lv) {  // -1, 0, 1, 2
  return lv == 0 ? 0x0u : lv == 1 ? 0x2u : lv == 2 ? 0x4u : 0xAu;
}
__device__ __forceinline__ void store_chunk_f4(int8_t* out, size_t m_pad, size_t r, int j, uint2 v) {
  reinterpret_cast<uint2*>(out + ((size_t)(j >> 4) * m_pad + r) * 128)[j & 15] = v;
}

template <bool F4>
__global__ void k_expand_rows_s8(const uint32_t* __restrict__ rows,
                                 size_t row_count, int w32pr, int offset,
                                 int k_pad, size_t m_pad, int8_t* __restrict__ out) {
  // launched as a dependent of the row producer (im2col): wait for its rows;
  // the GEMM after this kernel may launch right away
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int chunks = k_pad / 16;
  const uint32_t tbl = offset ? 0x02010100u : 0x010000FFu;
  // code -> E2M1 nibble (offset: levels 0,1,1,2; symmetric: -1,0,0,1)
  const uint32_t ntbl = offset ? 0x4220u : 0x200Au;
  const size_t total = row_count * (size_t)chunks;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
       t += (size_t)gridDim.x * blockDim.x) {
    const size_t r = t / chunks;
    const int j = (int)(t - r * chunks);
    if constexpr (F4) {
      uint2 o = make_uint2(0, 0);
      if (j < w32pr) {
        const uint32_t wd = rows[r * w32pr + j];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const uint32_t nib = (ntbl >> (4 * ((wd >> (2 * i)) & 3u))) & 0xFu;
          if (i < 8) o.x |= nib << (4 * i); else o.y |= nib << (4 * (i - 8));
        }
      }
      store_chunk_f4(out, m_pad, r, j, o);
      continue;
    }
    uint4 o = make_uint4(0, 0, 0, 0);
    if (j < w32pr) {
      const uint32_t wd = rows[r * w32pr + j];
      o.x = expand4(wd & 0xFF, tbl);
      o.y = expand4((wd >> 8) & 0xFF, tbl);
      o.z = expand4((wd >> 16) & 0xFF, tbl);
      o.w = expand4(wd >> 24, tbl);
    }
    // K-block-major operand layout [k/128][m_pad][128] (contiguous TMA boxes)
    reinterpret_cast<uint4*>(out + ((size_t)(j >> 3) * m_pad + r) * 128)[j & 7] = o;
  }
}

// im2col_quantize_pack fused with the level expansion: f32 NCHW input ->
// the tensor-core level operand in one pass (the packed 2-bit rows of
// k_im2col are formed in registers with the same quantizer and error
// checks, then expanded like k_expand_rows_s8).  Chunks past the packed
// row (up to k_pad) are written as zero levels.
template <bool F4>
__global__ void k_im2col_levels(const float* __restrict__ x, int n, int c, int h, int w, int kh, int kw, int stride,
                                int pad, int oh, int ow, int K, int w32pr, tk_qparams q, int offset, int k_pad,
                                size_t m_pad, int8_t* __restrict__ out, unsigned long long* err) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // (the GEMM waits for this grid)
  const size_t rows = (size_t)n * oh * ow;
  const int chunks = k_pad / 16;
  const size_t total = rows * (size_t)chunks;
  const uint32_t tbl = offset ? 0x02010100u : 0x010000FFu;
  const uint32_t ntbl = offset ? 0x4220u : 0x200Au;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total; t += (size_t)gridDim.x * blockDim.x) {
    const size_t r = t / chunks;
    const int j = (int)(t - r * chunks);
    uint32_t wd = 0;
    const bool have = j < w32pr;
    if (have) {
      const int b = (int)(r / ((size_t)oh * ow));
      const int p = (int)(r - (size_t)b * oh * ow);
      const int oy = p / ow, ox = p - (p / ow) * ow;
      const int l0 = j * 16;
      const int valid = l0 >= K ? 0 : min(16, K - l0);
      int kpos = l0 / c, ci = l0 - kpos * c;
      int ky = kpos / kw, kx = kpos - ky * kw;
      const float* img = x + (size_t)b * c * h * w;
      float v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        float val = 0.0f;
        if (i < valid) {
          const int iy = oy * stride - pad + ky, ix = ox * stride - pad + kx;
          if (iy >= 0 && iy < h && ix >= 0 && ix < w) val = __ldg(img + ((size_t)ci * h + iy) * w + ix);
          if (++ci == c) {
            ci = 0;
            if (++kx == kw) { kx = 0; ++ky; }
          }
        }
        v[i] = val;
      }
      wd = lane_word16(v, valid, q, err, r * (size_t)K + l0);
    }
    if constexpr (F4) {
      uint2 o = make_uint2(0, 0);
      if (have) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const uint32_t nib = (ntbl >> (4 * ((wd >> (2 * i)) & 3u))) & 0xFu;
          if (i < 8) o.x |= nib << (4 * i); else o.y |= nib << (4 * (i - 8));
        }
      }
      store_chunk_f4(out, m_pad, r, j, o);
    } else {
      uint4 o = make_uint4(0, 0, 0, 0);
      if (have) {
        o.x = expand4(wd & 0xFF, tbl);
        o.y = expand4((wd >> 8) & 0xFF, tbl);
        o.z = expand4((wd >> 16) & 0xFF, tbl);
        o.w = expand4(wd >> 24, tbl);
      }
      reinterpret_cast<uint4*>(out + ((size_t)(j >> 3) * m_pad + r) * 128)[j & 7] = o;
    }
  }
}

// Floats -> s8 quantization levels ({0,1,2} activation, {-1,0,1} weight
// mode) for the tensor-core FC path; columns >= n are zero.
template <bool F4>
__global__ void k_quantize_s8(const float* __restrict__ x, size_t rows,
                              size_t n, tk_qparams q, int k_pad, size_t m_pad,
                              int8_t* __restrict__ out,
                              unsigned long long* err, bool vec4) {
  // the consuming GEMM may launch now (it waits for this grid before reading)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int chunks = k_pad / 16;
  const size_t total = rows * (size_t)chunks;
  const int bias = q.nonneg ? 0 : -1;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
       t += (size_t)gridDim.x * blockDim.x) {
    const size_t r = t / chunks;
    const int j = (int)(t - r * chunks);
    const size_t l0 = (size_t)j * 16;
    const int valid = l0 >= n ? 0 : (int)min((size_t)16, n - l0);
    const float* src = x + r * n + l0;
    float v[16];
    if (vec4 && valid == 16) {
      const float4* s4 = reinterpret_cast<const float4*>(src);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float4 f = __ldg(s4 + i);
        v[4 * i] = f.x; v[4 * i + 1] = f.y; v[4 * i + 2] = f.z; v[4 * i + 3] = f.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = i < valid ? __ldg(src + i) : 0.0f;
    }
    uint32_t b[4] = {0, 0, 0, 0};
    uint32_t f[2] = {0, 0};  // F4 nibbles
    int first_bad = -1, bad_code = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (i < valid) {
        const uint32_t c = tk_code(v[i], q);
        if (c == 0xFFu) {
          if (first_bad < 0) {
            first_bad = i;
            bad_code = tk_error_code(v[i], q.nonneg);
          }
        } else {
          const int lv = (int)(c & 1u) + (int)(c >> 1) + bias;
          if constexpr (F4)
            f[i / 8] |= e2m1_of_level(lv) << (4 * (i % 8));
          else
            b[i / 4] |= ((uint32_t)(lv & 0xFF)) << (8 * (i % 4));
        }
      }
    }
    if (first_bad >= 0) tk_raise(err, r * n + l0 + first_bad, bad_code);
    if constexpr (F4) {
      store_chunk_f4(out, m_pad, r, j, make_uint2(f[0], f[1]));
    } else {
      // K-block-major operand layout [k/128][m_pad][128] (contiguous TMA boxes)
      reinterpret_cast<uint4*>(out + ((size_t)(j >> 3) * m_pad + r) * 128)[j & 7] =
          make_uint4(b[0], b[1], b[2], b[3]);
    }
  }
}

unsigned grid_for(size_t work) {
  size_t g = (work + kThreads - 1) / kThreads;
  if (g > 148u * 64u) g = 148u * 64u;
  return (unsigned)(g ? g : 1);
}

}  // namespace

cudaError_t tk_launch_quantize_pack(const float* x, size_t rows, size_t n,
                                    tk_qparams q, uint64_t* words,
                                    unsigned long long* err, cudaStream_t s) {
  const int w32pr = (int)(2 * ((n + 31) / 32));
  const size_t total = rows * (size_t)w32pr;
  if (total == 0) return cudaSuccess;
  const bool vec4 = (n % 4 == 0) && ((uintptr_t)x % 16 == 0);
  k_quantize_pack<<<grid_for(total), kThreads, 0, s>>>(
      x, rows, n, w32pr, q, reinterpret_cast<uint32_t*>(words), err, vec4);
  return cudaGetLastError();
}

cudaError_t tk_launch_im2col_levels(const float* x, int n, int c, int h, int w, int kh, int kw, int stride, int pad,
                                    tk_qparams q, int offset, int k_pad, bool fp4, int8_t* out,
                                    unsigned long long* err, cudaStream_t s) {
  const int oh = (h + 2 * pad - kh) / stride + 1;
  const int ow = (w + 2 * pad - kw) / stride + 1;
  const int K = c * kh * kw;
  const int w32pr = 2 * ((K + 31) / 32);
  const size_t rows = (size_t)n * oh * ow;
  const size_t total = rows * (size_t)(k_pad / 16);
  if (total == 0) return cudaSuccess;
  const size_t m_pad = (rows + 127) / 128 * 128;
  (fp4 ? k_im2col_levels<true> : k_im2col_levels<false>)<<<grid_for(total), kThreads, 0, s>>>(
      x, n, c, h, w, kh, kw, stride, pad, oh, ow, K, w32pr, q, offset, k_pad, m_pad, out, err);
  return cudaGetLastError();
}

cudaError_t tk_launch_im2col(const float* x, int n, int c, int h, int w,
                             int kh, int kw, int stride, int pad, tk_qparams q,
                             uint64_t* rows, unsigned long long* err,
                             cudaStream_t s) {
  const int oh = (h + 2 * pad - kh) / stride + 1;
  const int ow = (w + 2 * pad - kw) / stride + 1;
  const int K = c * kh * kw;
  const int w32pr = 2 * ((K + 31) / 32);
  const size_t total = (size_t)n * oh * ow * w32pr;
  if (total == 0) return cudaSuccess;
  k_im2col<<<grid_for(total), kThreads, 0, s>>>(
      x, n, c, h, w, kh, kw, stride, pad, oh, ow, K, w32pr, q,
      reinterpret_cast<uint32_t*>(rows), err);
  return cudaGetLastError();
}

cudaError_t tk_launch_pack_int8(const int8_t* v, size_t n, uint64_t* words,
                                unsigned long long* err, cudaStream_t s) {
  const size_t w32 = 2 * ((n + 31) / 32);
  if (w32 == 0) return cudaSuccess;
  k_pack_int8<<<grid_for(w32), kThreads, 0, s>>>(
      v, n, reinterpret_cast<uint32_t*>(words), w32, err);
  return cudaGetLastError();
}

cudaError_t tk_launch_unpack(const uint64_t* words, size_t n, int8_t* v,
                             cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  k_unpack<<<grid_for(n), kThreads, 0, s>>>(
      reinterpret_cast<const uint32_t*>(words), n, v);
  return cudaGetLastError();
}

cudaError_t tk_launch_expand_rows_s8(const uint64_t* rows, size_t row_count,
                                     int wpr64, int offset, int k_pad,
                                     int8_t* out, cudaStream_t s) {
  return tk_launch_expand_rows(rows, row_count, wpr64, offset, k_pad, false, out, s);
}

cudaError_t tk_launch_expand_rows(const uint64_t* rows, size_t row_count, int wpr64, int offset, int k_pad,
                                  bool fp4, int8_t* out, cudaStream_t s) {
  const size_t total = row_count * (size_t)(k_pad / 16);
  if (total == 0) return cudaSuccess;
  // programmatic dependent launch: the kernel waits for its predecessor
  // (griddepcontrol.wait) before touching memory, so only the launch overlaps
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid_for(total));
  cfg.blockDim = dim3(kThreads);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const uint32_t* r32 = reinterpret_cast<const uint32_t*>(rows);
  const size_t m_pad = (row_count + 127) / 128 * 128;
  const int w32pr = 2 * wpr64;
  cudaError_t e = fp4 ? cudaLaunchKernelEx(&cfg, k_expand_rows_s8<true>, r32, row_count, w32pr, offset, k_pad, m_pad, out)
                      : cudaLaunchKernelEx(&cfg, k_expand_rows_s8<false>, r32, row_count, w32pr, offset, k_pad, m_pad,
                                           out);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t tk_launch_quantize_s8(const float* x, size_t rows, size_t n,
                                  tk_qparams q, int k_pad, int8_t* out,
                                  unsigned long long* err, cudaStream_t s) {
  return tk_launch_quantize_levels(x, rows, n, q, k_pad, false, out, err, s);
}

cudaError_t tk_launch_quantize_levels(const float* x, size_t rows, size_t n, tk_qparams q, int k_pad, bool fp4,
                                      int8_t* out, unsigned long long* err, cudaStream_t s) {
  const size_t total = rows * (size_t)(k_pad / 16);
  if (total == 0) return cudaSuccess;
  const bool vec4 = (n % 4 == 0) && ((uintptr_t)x % 16 == 0);
  (fp4 ? k_quantize_s8<true> : k_quantize_s8<false>)<<<grid_for(total), kThreads, 0, s>>>(x, rows, n, q, k_pad, (rows + 127) / 128 * 128,
                                                    out, err, vec4);
  return cudaGetLastError();
}

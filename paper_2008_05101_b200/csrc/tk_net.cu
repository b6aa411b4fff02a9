// tk_net.cu -- network-level ternary inference: the fused tensor-core conv
// pipeline (implicit im2col, folded BN + skip-add + ReLU + next-layer
// quantize in the epilogue) and the generic layer-by-layer path.
//
// Composition (R:tinynet.hpp:713-735, applied to conv blocks; oracle:
// oracle/ternkit_oracle.c or_net_body, reference: oracle/ref_shim.cpp):
//   h = x; for inner convs: h = max(conv2d_ternary(h), 0)
//   out = max(conv2d_ternary_last(h) + (down ? conv2d_ternary_down(x) : x), 0)
//
// Fused-path data layout (all HBM-resident, per activation tensor):
//  * s8 levels  [C/R][phase][pos][R]   R = 64 (C == 64) or 128 channels,
//    pos = padded position n*PH*PW + py*PW + px of a zero-padded (pad 1)
//    image; stride-2 consumers get the 4 (row, col)-parity phase planes so
//    every kernel tap is a contiguous row range.  The pad ring is zero
//    (= the code of quantize(0.0)), written once and never touched.
//  * f32 values [C/32][pos][32] (only where a residual add needs them).
// Conv kernel (tcgen05 kind::i8): a CTA owns a 128-position tile; for each
// 64/128-channel chunk ONE TMA box loads the tile plus halo (rows shifted by
// up to 2*Wp+2) into SMEM with the hardware swizzle, and every tap of the
// 3x3 window is an MMA whose A descriptor simply starts `shift` rows later
// (verified on B200: tools/desc_test.cu).  Weights stream through a TMA ring
// (or stay resident when they fit).  Accumulators double-buffer in TMEM so
// the epilogue of tile i overlaps the MMAs of tile i+1.
#include <cuda.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "tk_internal.cuh"
#include "tk_sm100.cuh"

namespace {

constexpr int kConvThreads = 192;  // warp0 TMA, warp1 MMA, warps 2-5 epilogue

struct ConvK {
  int n_taps;
  int tap_slot[9];
  int tap_shift[9];
  int n_ph;
  int ph_id[4];
  int halo_rows;
  int chunks;
  long long in_pos;  // rows per phase plane of the input tensor
  int in_phases;
  int base_shift;
  int n_tiles, m_tiles;
  long long m_total;
  int PHg, PWg, Ho, Wo;
  int hs, ws, resident;
  int HB, WB;  // bytes per halo box / weight block (1024 aligned)
  // epilogue
  const float* gain;
  const float* bias;
  float out_scale;
  int relu;
  int N;
  const float* skip;
  float* fout;
  long long f_pos;
  int o_Hp, o_Wp, o_PH, o_PW;
  int n_q;
  int8_t* q[2];
  float t0[2], t1[2];
  int q_phases[2], q_R[2];
  long long q_pos[2];
  unsigned long long* err;
};

__device__ __forceinline__ uint64_t desc_sw(uint32_t saddr, int R) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((8 * R) >> 4) << 32;      // SBO: 8 rows
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(R == 128 ? 2 : 4) << 61;  // SWIZZLE_128B / SWIZZLE_64B
  return d;
}

template <int BN, int R>
__global__ void __launch_bounds__(kConvThreads, 1)
k_conv_tc(const __grid_constant__ CUtensorMap in_map, const __grid_constant__ CUtensorMap w_map,
          const ConvK p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* halo = smem;
  const int halo_stage = p.n_ph * p.HB;
  uint8_t* wreg = halo + p.hs * halo_stage;
  const int wblocks = p.resident ? p.chunks * p.n_taps : p.ws;
  uint64_t* bars = reinterpret_cast<uint64_t*>(wreg + (size_t)wblocks * p.WB);
  uint64_t* h_full = bars;
  uint64_t* h_empty = h_full + p.hs;
  uint64_t* w_full = h_empty + p.hs;
  uint64_t* w_empty = w_full + p.ws;
  uint64_t* a_full = w_empty + p.ws;
  uint64_t* a_empty = a_full + 2;
  uint64_t* w_res = a_empty + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(w_res + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  constexpr uint32_t kCols = 2 * BN;  // two accumulators
  constexpr int kSteps = R / 32;      // MMAs (K = 32) per tap and chunk

  if (threadIdx.x == 0) {
    sm100::tma_prefetch(&in_map);
    sm100::tma_prefetch(&w_map);
    for (int s = 0; s < p.hs; ++s) {
      sm100::mbar_init(&h_full[s], 1);
      sm100::mbar_init(&h_empty[s], 1);
    }
    for (int s = 0; s < p.ws; ++s) {
      sm100::mbar_init(&w_full[s], 1);
      sm100::mbar_init(&w_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      sm100::mbar_init(&a_full[s], 1);
      sm100::mbar_init(&a_empty[s], 128);
    }
    sm100::mbar_init(w_res, 1);
    sm100::fence_mbar_init();
  }
  if (warp == 1) sm100::tmem_alloc<kCols>(tslot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tslot;
  const int n_items = p.m_tiles * p.n_tiles;

  if (warp == 0 && lane == 0) {
    // ================= producer =================
    if (p.resident) {  // all weight blocks of the (single) n-tile, once
      sm100::mbar_arrive_expect_tx(w_res, (uint32_t)(p.chunks * p.n_taps) * BN * R);
      for (int b = 0; b < p.chunks * p.n_taps; ++b)
        sm100::tma_load_2d(wreg + (size_t)b * p.WB, &w_map, w_res, 0, b * BN);
    }
    int hc = 0, wc = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int mt = item / p.n_tiles, nt = item - mt * p.n_tiles;
      const int row0 = mt * 128 + p.base_shift;
      for (int ch = 0; ch < p.chunks; ++ch) {
        const int hsi = hc % p.hs;
        if (hc >= p.hs) sm100::mbar_wait(&h_empty[hsi], ((hc / p.hs) - 1) & 1);
        sm100::mbar_arrive_expect_tx(&h_full[hsi], (uint32_t)(p.n_ph * p.halo_rows * R));
        for (int s = 0; s < p.n_ph; ++s) {
          const long long r = (long long)(ch * p.in_phases + p.ph_id[s]) * p.in_pos + row0;
          sm100::tma_load_2d(halo + hsi * halo_stage + s * p.HB, &in_map, &h_full[hsi], 0, (int)r);
        }
        ++hc;
        if (!p.resident) {
          for (int t = 0; t < p.n_taps; ++t) {
            const int wsi = wc % p.ws;
            if (wc >= p.ws) sm100::mbar_wait(&w_empty[wsi], ((wc / p.ws) - 1) & 1);
            sm100::mbar_arrive_expect_tx(&w_full[wsi], BN * R);
            const int blk = (nt * p.chunks + ch) * p.n_taps + t;
            sm100::tma_load_2d(wreg + (size_t)wsi * p.WB, &w_map, &w_full[wsi], 0, blk * BN);
            ++wc;
          }
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ================= MMA issuer =================
    constexpr uint32_t idesc = sm100::idesc_i8(128, BN);
    if (p.resident) sm100::mbar_wait(w_res, 0);
    int hc = 0, wc = 0, it = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
      const int acc = it & 1;
      if (it >= 2) sm100::mbar_wait(&a_empty[acc], ((it >> 1) - 1) & 1);
      sm100::tc_fence_after();
      const uint32_t d = tmem + acc * BN;
      for (int ch = 0; ch < p.chunks; ++ch) {
        const int hsi = hc % p.hs;
        sm100::mbar_wait(&h_full[hsi], (hc / p.hs) & 1);
        sm100::tc_fence_after();
        const uint32_t hbase = sm100::smem_u32(halo + hsi * halo_stage);
        for (int t = 0; t < p.n_taps; ++t) {
          uint32_t wb;
          int wsi = 0;
          if (p.resident) {
            wb = sm100::smem_u32(wreg + (size_t)(ch * p.n_taps + t) * p.WB);
          } else {
            wsi = wc % p.ws;
            sm100::mbar_wait(&w_full[wsi], (wc / p.ws) & 1);
            sm100::tc_fence_after();
            wb = sm100::smem_u32(wreg + (size_t)wsi * p.WB);
          }
          const uint32_t ab = hbase + p.tap_slot[t] * p.HB + p.tap_shift[t] * R;
#pragma unroll
          for (int k = 0; k < kSteps; ++k)
            sm100::mma_i8(d, desc_sw(ab + k * 32, R), desc_sw(wb + k * 32, R), idesc,
                          (ch | t | k) != 0);
          if (!p.resident) {
            sm100::mma_commit(&w_empty[wsi]);
            ++wc;
          }
        }
        sm100::mma_commit(&h_empty[hsi]);
        ++hc;
      }
      sm100::mma_commit(&a_full[acc]);
    }
  } else if (warp >= 2) {
    // ================= epilogue =================
    const int qtr = warp & 3;
    const int plane = p.PHg * p.PWg;
    int it = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
      const int mt = item / p.n_tiles, nt = item - mt * p.n_tiles;
      const int acc = it & 1;
      const long long qrow = (long long)mt * 128 + qtr * 32 + lane;
      const int img = (int)(qrow / plane);
      const int rem = (int)(qrow - (long long)img * plane);
      const int oy = rem / p.PWg, ox = rem - (rem / p.PWg) * p.PWg;
      const bool valid = qrow < p.m_total && oy < p.Ho && ox < p.Wo;
      const long long P1 = ((long long)img * p.o_Hp + oy + 1) * p.o_Wp + ox + 1;
      const int py = oy + 1, px = ox + 1;
      const long long P4 = ((long long)img * p.o_PH + (py >> 1)) * p.o_PW + (px >> 1);
      const int ph4 = (py & 1) * 2 + (px & 1);
      sm100::mbar_wait(&a_full[acc], (it >> 1) & 1);
      sm100::tc_fence_after();
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t r[32];
        sm100::tmem_ld32(tmem + ((uint32_t)(qtr * 32) << 16) + acc * BN + c0, r);
        sm100::tmem_ld_wait();
        if (!valid) continue;
        const int n0 = nt * BN + c0;
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          // R:linalg.hpp:322-323 (FMA-contracted like the reference build)
          v[j] = __fmaf_rn(__ldg(p.gain + n0 + j), __fmul_rn(p.out_scale, (float)(int32_t)r[j]),
                           __ldg(p.bias + n0 + j));
        }
        if (p.skip) {
          const float4* s4 = reinterpret_cast<const float4*>(p.skip + ((long long)(n0 >> 5) * p.f_pos + P1) * 32);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 s = __ldg(s4 + j);
            v[4 * j] += s.x; v[4 * j + 1] += s.y; v[4 * j + 2] += s.z; v[4 * j + 3] += s.w;
          }
        }
        if (p.relu) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = v[j] < 0.0f ? 0.0f : v[j];  // std::max(v, 0.0f)
        }
        if (p.fout) {
          float4* o4 = reinterpret_cast<float4*>(p.fout + ((long long)(n0 >> 5) * p.f_pos + P1) * 32);
#pragma unroll
          for (int j = 0; j < 8; ++j) o4[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        }
        for (int o = 0; o < p.n_q; ++o) {
          uint32_t w[8];
          bool bad = false;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            uint32_t b = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float x = v[4 * j + i];
              bad |= !(x >= 0.0f && x <= 3.402823466e38f);
              const uint32_t lv = (uint32_t)(x > p.t0[o]) + (uint32_t)(x > p.t1[o]);
              b |= lv << (8 * i);
            }
            w[j] = b;
          }
          if (bad) tk_raise(p.err, (unsigned long long)qrow, TK_ERR_NONFINITE);
          const int Rq = p.q_R[o];
          const int chq = n0 / Rq, cq = n0 - chq * Rq;
          long long off;
          if (p.q_phases[o] == 4)
            off = ((long long)(chq * 4 + ph4) * p.q_pos[o] + P4) * Rq + cq;
          else
            off = ((long long)chq * p.q_pos[o] + P1) * Rq + cq;
          uint4* dst = reinterpret_cast<uint4*>(p.q[o] + off);
          dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
          dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
        }
      }
      sm100::tc_fence_before();
      sm100::mbar_arrive(&a_empty[acc]);
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) sm100::tmem_dealloc<kCols>(tmem);
}

// ---------------------------------------------------------------------------
// input packing: NCHW f32 -> s8 level tensors (up to 2 variants) + f32 copy.
struct PackIn {
  const float* x;
  int C, H, W;
  int n_q;
  int8_t* q[2];
  float t0[2], t1[2];
  int q_phases[2], q_R[2];
  long long q_pos[2];
  int Hp, Wp, PH, PW;
  float* f;
  long long f_pos;
  unsigned long long* err;
};

// one block per (image, row): stage the row's C x W floats in SMEM, then
// write channel-contiguous level bytes / float groups per position.
__global__ void k_pack_input(const PackIn p) {
  extern __shared__ float srow[];  // [C][W + 1]
  const int n = blockIdx.x / p.H, y = blockIdx.x - (blockIdx.x / p.H) * p.H;
  const int Wp1 = p.W + 1;
  for (int i = threadIdx.x; i < p.C * p.W; i += blockDim.x) {
    const int c = i / p.W, xx = i - c * p.W;
    srow[c * Wp1 + xx] = __ldg(p.x + (((long long)n * p.C + c) * p.H + y) * p.W + xx);
  }
  __syncthreads();
  // 16-channel groups per position
  const int groups = p.C / 16;
  for (int i = threadIdx.x; i < groups * p.W; i += blockDim.x) {
    const int g = i / p.W, xx = i - g * p.W;  // xx fastest -> coalesced-ish rows
    float v[16];
    bool bad = false;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      v[j] = srow[(g * 16 + j) * Wp1 + xx];
      bad |= !(v[j] >= 0.0f && v[j] <= 3.402823466e38f);
    }
    if (bad) {
      for (int j = 0; j < 16; ++j) {
        const int e = tk_error_code(v[j], 1);
        if (e != TK_OK) {
          tk_raise(p.err, (((unsigned long long)n * p.C + g * 16 + j) * p.H + y) * p.W + xx, e);
          break;
        }
      }
    }
    const int py = y + 1, px = xx + 1;
    const long long P1 = ((long long)n * p.Hp + py) * p.Wp + px;
    const long long P4 = ((long long)n * p.PH + (py >> 1)) * p.PW + (px >> 1);
    const int ph4 = (py & 1) * 2 + (px & 1);
    for (int o = 0; o < p.n_q; ++o) {
      uint32_t w[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t b = 0;
#pragma unroll
        for (int i2 = 0; i2 < 4; ++i2) {
          const float xv = v[4 * j + i2];
          b |= ((uint32_t)(xv > p.t0[o]) + (uint32_t)(xv > p.t1[o])) << (8 * i2);
        }
        w[j] = b;
      }
      const int Rq = p.q_R[o];
      const int c0 = g * 16, chq = c0 / Rq, cq = c0 - chq * Rq;
      const long long off = p.q_phases[o] == 4 ? ((long long)(chq * 4 + ph4) * p.q_pos[o] + P4) * Rq + cq
                                               : ((long long)chq * p.q_pos[o] + P1) * Rq + cq;
      *reinterpret_cast<uint4*>(p.q[o] + off) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    if (p.f) {
      float4* o4 = reinterpret_cast<float4*>(p.f + ((long long)(g >> 1) * p.f_pos + P1) * 32 + (g & 1) * 16);
#pragma unroll
      for (int j = 0; j < 4; ++j) o4[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
    }
  }
}

// f32 [C/32][pos][32] -> NCHW
__global__ void k_unpack_f32(const float* __restrict__ f, long long f_pos, int N, int C, int H, int W,
                             int Hp, int Wp, float* __restrict__ out) {
  const long long total = (long long)N * C * H * W;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int xx = (int)(i % W);
    long long t = i / W;
    const int y = (int)(t % H);
    t /= H;
    const int c = (int)(t % C);
    const int n = (int)(t / C);
    const long long P1 = ((long long)n * Hp + y + 1) * Wp + xx + 1;
    out[i] = f[((long long)(c >> 5) * f_pos + P1) * 32 + (c & 31)];
  }
}

// spatial mean of the f32 layout -> [N][C] (head input; left-to-right sum)
__global__ void k_pool_f32(const float* __restrict__ f, long long f_pos, int N, int C, int H, int W, int Hp,
                           int Wp, float* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N * C) return;
  const int n = i / C, c = i - (i / C) * C;
  float s = 0.0f;
  for (int y = 0; y < H; ++y)
    for (int xx = 0; xx < W; ++xx)
      s += f[((long long)(c >> 5) * f_pos + ((long long)n * Hp + y + 1) * Wp + xx + 1) * 32 + (c & 31)];
  out[i] = s / (float)(H * W);
}

// generic path helpers (NCHW)
__global__ void k_residual_relu(float* __restrict__ z, const float* __restrict__ sc, long long n, int relu_only) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const float v = relu_only ? z[i] : z[i] + sc[i];
    z[i] = v < 0.0f ? 0.0f : v;  // std::max(v, 0.0f)
  }
}

__global__ void k_pool_nchw(const float* __restrict__ x, int NC, int HW, float* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= NC) return;
  float s = 0.0f;
  for (int j = 0; j < HW; ++j) s += x[(long long)i * HW + j];
  out[i] = s / (float)HW;
}

// ---------------------------------------------------------------------------
// host side

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(ptr);
  });
  return fn;
}

bool map_rows(CUtensorMap* m, const void* base, unsigned long long rows, int R, int box_rows) {
  EncodeFn fn = encode();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)R, (cuuint64_t)rows};
  cuuint64_t str[1] = {(cuuint64_t)R};
  cuuint32_t box[2] = {(cuuint32_t)R, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, str, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, R == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct S8T {  // s8 level tensor
  int8_t* p = nullptr;
  int C = 0, R = 0, phases = 1;
  int H = 0, W = 0, Hp = 0, Wp = 0, PH = 0, PW = 0;
  long long pos = 0;
  float ta1 = 0, ta2 = 0;
  size_t bytes() const { return (size_t)(C / R) * phases * pos * R; }
};
struct F32T {
  float* p = nullptr;
  int C = 0, H = 0, W = 0, Hp = 0, Wp = 0;
  long long pos = 0;
};

int pick_R(int C) { return C == 64 ? 64 : 128; }

S8T make_s8(int batch, int C, int H, int W, int phases, float ta1, float ta2) {
  S8T t;
  t.C = C; t.R = pick_R(C); t.phases = phases; t.H = H; t.W = W; t.Hp = H + 2; t.Wp = W + 2;
  t.PH = phases == 4 ? t.Hp / 2 : t.Hp;
  t.PW = phases == 4 ? t.Wp / 2 : t.Wp;
  t.pos = ((long long)batch * t.PH * t.PW + 127) / 128 * 128 + 384;
  t.ta1 = ta1; t.ta2 = ta2;
  return t;
}

struct Conv {
  tk_conv_desc d;
  int BN = 0, R = 0, chunks = 0, n_tiles = 0;
  int8_t* d_w = nullptr;  // [nt][ch][tap][BN][R]
  float* d_gain = nullptr;
  float* d_bias = nullptr;
  tk_layer* layer = nullptr;  // generic path
  // fused wiring
  int in_idx = -1;            // index into net->s8
  int skip_f = -1, out_f = -1;
  int q_idx[2] = {-1, -1};
  int relu = 0;
  ConvK k{};
  CUtensorMap in_map{}, w_map{};
  int smem = 0;
  int grid = 0;
};

}  // namespace

struct tk_net {
  tk_context* ctx = nullptr;
  int fused = 0;
  int batch = 0, in_c = 0, in_h = 0, in_w = 0;
  int out_c = 0, out_h = 0, out_w = 0;
  std::vector<tk_block_desc> blocks;
  std::vector<std::vector<Conv>> convs;  // per block: convs..., then down
  std::vector<S8T> s8;
  std::vector<F32T> f32;
  PackIn pack{};
  int final_f = -1;
  // generic path buffers
  std::vector<float*> gbuf;
  size_t gbuf_elems = 0;
  float* d_pool_tmp = nullptr;
};

namespace {

int conv_out(int h, const tk_conv_desc& c) { return (h + 2 * c.pad - c.k) / c.stride + 1; }

bool fused_ok(const tk_net* net) {
  int H = net->in_h, W = net->in_w, C = net->in_c;
  if (C % 64) return false;
  for (const auto& b : net->blocks) {
    if (b.n_convs < 1 || b.n_convs > 3) return false;
    int h = H, w = W, c = C;
    auto ok = [&](const tk_conv_desc& d, int hh, int ww, int cc) {
      if (d.in_c != cc || d.out_c % 64 || d.in_c % 64) return false;
      if (!((d.k == 3 && d.pad == 1) || (d.k == 1 && d.pad == 0))) return false;
      if (d.stride != 1 && d.stride != 2) return false;
      if (d.stride == 2 && ((hh % 2) || (ww % 2))) return false;
      const int Wp = ww + 2;
      const int span = d.stride == 1 ? (d.k == 3 ? 2 * Wp + 2 : 0) : (d.k == 3 ? Wp / 2 + 1 : 0);
      if (128 + span > 256) return false;
      return true;
    };
    for (int i = 0; i < b.n_convs; ++i) {
      if (!ok(b.conv[i], h, w, c)) return false;
      h = conv_out(h, b.conv[i]);
      w = conv_out(w, b.conv[i]);
      c = b.conv[i].out_c;
    }
    if (b.has_down) {
      if (!ok(b.down, H, W, C) || conv_out(H, b.down) != h || conv_out(W, b.down) != w || b.down.out_c != c)
        return false;
    } else if (h != H || w != W || c != C) {
      return false;
    }
    H = h; W = w; C = c;
  }
  return true;
}

// taps of one conv against its input tensor layout
void plan_taps(Conv& cv, const S8T& in) {
  ConvK& k = cv.k;
  const tk_conv_desc& d = cv.d;
  int shifts[9], phs[9], n = 0;
  for (int ky = 0; ky < d.k; ++ky)
    for (int kx = 0; kx < d.k; ++kx) {
      // padded input coordinate of output (0,0): (stride*0 + ky + 1 - pad, ...)
      const int py = ky + 1 - d.pad, px = kx + 1 - d.pad;
      if (d.stride == 1) {
        phs[n] = 0;
        shifts[n] = py * in.Wp + px;
      } else {
        phs[n] = (py & 1) * 2 + (px & 1);
        shifts[n] = (py >> 1) * in.PW + (px >> 1);
      }
      ++n;
    }
  int used[4] = {0, 0, 0, 0};
  for (int i = 0; i < n; ++i) used[phs[i]] = 1;
  k.n_ph = 0;
  int slot_of[4];
  for (int ph = 0; ph < 4; ++ph)
    if (used[ph]) { slot_of[ph] = k.n_ph; k.ph_id[k.n_ph++] = ph; }
  int mn = 1 << 30, mx = 0;
  for (int i = 0; i < n; ++i) { mn = std::min(mn, shifts[i]); mx = std::max(mx, shifts[i]); }
  k.base_shift = mn;
  k.n_taps = n;
  for (int i = 0; i < n; ++i) {
    k.tap_slot[i] = slot_of[phs[i]];
    k.tap_shift[i] = shifts[i] - mn;
  }
  k.halo_rows = (128 + (mx - mn) + 7) / 8 * 8;
  k.in_phases = in.phases;
  k.in_pos = in.pos;
  k.chunks = in.C / in.R;
  // output grid = the input's (phase) plane grid
  k.PHg = in.PH;
  k.PWg = in.PW;
  k.Ho = conv_out(in.H, d);
  k.Wo = conv_out(in.W, d);
}

int prepare_conv_weights(Conv& cv, int R) {
  const tk_conv_desc& d = cv.d;
  const int taps = d.k * d.k, chunks = d.in_c / R;
  cv.R = R;
  cv.chunks = chunks;
  cv.BN = d.out_c >= 256 ? 256 : d.out_c;  // 64, 128, 256
  cv.n_tiles = d.out_c / cv.BN;
  const size_t blk = (size_t)cv.BN * R;
  std::vector<int8_t> w((size_t)cv.n_tiles * chunks * taps * blk, 0);
  const int K = d.in_c * taps;
  for (int nt = 0; nt < cv.n_tiles; ++nt)
    for (int ch = 0; ch < chunks; ++ch)
      for (int t = 0; t < taps; ++t)
        for (int o = 0; o < cv.BN; ++o)
          for (int c = 0; c < R; ++c) {
            const int oc = nt * cv.BN + o, ic = ch * R + c;
            const int8_t v = d.weights_host[(size_t)oc * K + (size_t)t * d.in_c + ic];
            if (v < -1 || v > 1) return TK_ERR_RANGE;
            w[(((size_t)(nt * chunks + ch) * taps + t) * cv.BN + o) * R + c] = v;
          }
  std::vector<float> g(d.out_c, 1.0f), b(d.out_c, 0.0f);
  if (d.gain_host) memcpy(g.data(), d.gain_host, d.out_c * 4);
  if (d.bias_host) memcpy(b.data(), d.bias_host, d.out_c * 4);
  if (cudaMalloc(&cv.d_w, w.size()) != cudaSuccess || cudaMalloc(&cv.d_gain, d.out_c * 4) != cudaSuccess ||
      cudaMalloc(&cv.d_bias, d.out_c * 4) != cudaSuccess)
    return TK_ERR_CUDA;
  cudaMemcpy(cv.d_w, w.data(), w.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(cv.d_gain, g.data(), d.out_c * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(cv.d_bias, b.data(), d.out_c * 4, cudaMemcpyHostToDevice);
  if (!map_rows(&cv.w_map, cv.d_w, (unsigned long long)cv.n_tiles * chunks * taps * cv.BN, R, cv.BN))
    return TK_ERR_CUDA;
  return TK_OK;
}

// s8 tensor index for (C, H, W, phases, ta) -- reuse or create
int want_s8(tk_net* net, int C, int H, int W, int phases, float ta1, float ta2) {
  for (size_t i = 0; i < net->s8.size(); ++i) {
    const S8T& t = net->s8[i];
    (void)t;
  }
  net->s8.push_back(make_s8(net->batch, C, H, W, phases, ta1, ta2));
  return (int)net->s8.size() - 1;
}

int want_f32(tk_net* net, int C, int H, int W) {
  F32T f;
  f.C = C; f.H = H; f.W = W; f.Hp = H + 2; f.Wp = W + 2;
  f.pos = (long long)net->batch * f.Hp * f.Wp;
  net->f32.push_back(f);
  return (int)net->f32.size() - 1;
}

int setup_fused(tk_net* net) {
  // ---- wiring: consumers of each block input / intermediate ----
  int H = net->in_h, W = net->in_w, C = net->in_c;
  const int nb = (int)net->blocks.size();
  // block-input tensors: variants needed by conv1 and down
  struct In { int idx_conv1, idx_down, f; };
  std::vector<In> bin(nb);
  auto phases_of = [](const tk_conv_desc& d) { return d.stride == 2 ? 4 : 1; };
  // block inputs
  for (int b = 0; b < nb; ++b) {
    const tk_block_desc& bd = net->blocks[b];
    const tk_conv_desc& c1 = bd.conv[0];
    bin[b].idx_conv1 = want_s8(net, C, H, W, phases_of(c1), c1.ta1, c1.ta2);
    bin[b].idx_down = -1;
    if (bd.has_down) {
      const tk_conv_desc& dn = bd.down;
      if (phases_of(dn) == phases_of(c1) && dn.ta1 == c1.ta1 && dn.ta2 == c1.ta2)
        bin[b].idx_down = bin[b].idx_conv1;
      else
        bin[b].idx_down = want_s8(net, C, H, W, phases_of(dn), dn.ta1, dn.ta2);
    }
    bin[b].f = bd.has_down ? -1 : want_f32(net, C, H, W);
    int h = H, w = W;
    for (int i = 0; i < bd.n_convs; ++i) { h = conv_out(h, bd.conv[i]); w = conv_out(w, bd.conv[i]); }
    H = h; W = w; C = bd.conv[bd.n_convs - 1].out_c;
  }
  net->out_c = C; net->out_h = H; net->out_w = W;
  net->final_f = want_f32(net, C, H, W);
  // ---- convs ----
  H = net->in_h; W = net->in_w; C = net->in_c;
  net->convs.assign(nb, {});
  for (int b = 0; b < nb; ++b) {
    const tk_block_desc& bd = net->blocks[b];
    auto& cvs = net->convs[b];
    int cur = bin[b].idx_conv1;
    int h = H, w = W, c = C;
    int sc_f = bin[b].f;
    if (bd.has_down) {  // shortcut first: its f32 output is the residual
      Conv dv;
      dv.d = bd.down;
      dv.in_idx = bin[b].idx_down;
      dv.out_f = want_f32(net, bd.down.out_c, conv_out(H, bd.down), conv_out(W, bd.down));
      sc_f = dv.out_f;
      cvs.push_back(dv);
    }
    for (int i = 0; i < bd.n_convs; ++i) {
      const tk_conv_desc& d = bd.conv[i];
      Conv cv;
      cv.d = d;
      cv.in_idx = cur;
      const int ho = conv_out(h, d), wo = conv_out(w, d);
      if (i + 1 < bd.n_convs) {
        cv.relu = 1;
        const tk_conv_desc& nx = bd.conv[i + 1];
        cv.q_idx[0] = want_s8(net, d.out_c, ho, wo, phases_of(nx), nx.ta1, nx.ta2);
        cur = cv.q_idx[0];
      } else {
        cv.relu = 1;
        cv.skip_f = sc_f;
        if (b + 1 < nb) {
          cv.q_idx[0] = bin[b + 1].idx_conv1;
          if (bin[b + 1].idx_down >= 0 && bin[b + 1].idx_down != bin[b + 1].idx_conv1)
            cv.q_idx[1] = bin[b + 1].idx_down;
          cv.out_f = bin[b + 1].f;  // identity shortcut of the next block
        } else {
          cv.out_f = net->final_f;
        }
      }
      cvs.push_back(cv);
      h = ho; w = wo; c = d.out_c;
    }
    H = h; W = w; C = c;
  }
  // ---- allocate tensors ----
  for (auto& t : net->s8) {
    if (cudaMalloc(&t.p, t.bytes()) != cudaSuccess) return TK_ERR_CUDA;
    cudaMemset(t.p, 0, t.bytes());  // pad ring = code of quantize(0.0) = level 0
  }
  for (auto& f : net->f32)
    if (cudaMalloc(&f.p, (size_t)f.C * f.pos * 4) != cudaSuccess) return TK_ERR_CUDA;
  // ---- per-conv kernel parameters ----
  for (auto& cvs : net->convs)
    for (auto& cv : cvs) {
      const S8T& in = net->s8[cv.in_idx];
      int st = prepare_conv_weights(cv, in.R);
      if (st != TK_OK) return st;
      plan_taps(cv, in);
      ConvK& k = cv.k;
      k.n_tiles = cv.n_tiles;
      k.m_total = (long long)net->batch * k.PHg * k.PWg;
      k.m_tiles = (int)((k.m_total + 127) / 128);
      k.HB = (k.halo_rows * cv.R + 1023) / 1024 * 1024;
      k.WB = (cv.BN * cv.R + 1023) / 1024 * 1024;
      const int budget = 200 * 1024;
      const int halo_stage = k.n_ph * k.HB;
      k.hs = 2 * halo_stage + 4 * k.WB <= budget ? 2 : 1;
      const int wbytes_all = cv.chunks * k.n_taps * k.WB;
      k.resident = (cv.n_tiles == 1 && k.hs * halo_stage + wbytes_all <= budget) ? 1 : 0;
      k.ws = k.resident ? 1 : std::max(2, std::min(8, (budget - k.hs * halo_stage) / k.WB));
      const int wregion = k.resident ? wbytes_all : k.ws * k.WB;
      cv.smem = 1024 + k.hs * halo_stage + wregion + 512;
      k.gain = cv.d_gain;
      k.bias = cv.d_bias;
      k.out_scale = cv.d.out_scale;
      k.relu = cv.relu;
      k.N = cv.d.out_c;
      const int ho = k.Ho, wo = k.Wo;
      k.o_Hp = ho + 2; k.o_Wp = wo + 2;
      k.o_PH = k.o_Hp / 2; k.o_PW = k.o_Wp / 2;
      k.skip = cv.skip_f >= 0 ? net->f32[cv.skip_f].p : nullptr;
      k.fout = cv.out_f >= 0 ? net->f32[cv.out_f].p : nullptr;
      k.f_pos = (long long)net->batch * k.o_Hp * k.o_Wp;
      k.n_q = 0;
      for (int o = 0; o < 2; ++o) {
        if (cv.q_idx[o] < 0) continue;
        const S8T& q = net->s8[cv.q_idx[o]];
        tk_qparams qp;
        if (tk_make_qparams(q.ta1, q.ta2, TK_MODE_ACTIVATION_NONNEG, &qp) != TK_OK) return TK_ERR_THRESHOLDS;
        k.q[k.n_q] = q.p;
        k.t0[k.n_q] = qp.t0;
        k.t1[k.n_q] = qp.t1;
        k.q_phases[k.n_q] = q.phases;
        k.q_R[k.n_q] = q.R;
        k.q_pos[k.n_q] = q.pos;
        ++k.n_q;
      }
      k.err = net->ctx->d_err;
      if (!map_rows(&cv.in_map, in.p, (unsigned long long)(in.C / in.R) * in.phases * in.pos, in.R, k.halo_rows))
        return TK_ERR_CUDA;
      const int items = k.m_tiles * k.n_tiles;
      cv.grid = std::min(items, net->ctx->num_sms);
    }
  // ---- input packing ----
  PackIn& pk = net->pack;
  pk.C = net->in_c; pk.H = net->in_h; pk.W = net->in_w;
  const S8T& s0 = net->s8[bin[0].idx_conv1];
  pk.Hp = s0.Hp; pk.Wp = s0.Wp; pk.PH = s0.Hp / 2; pk.PW = s0.Wp / 2;
  pk.n_q = 0;
  int ids[2] = {bin[0].idx_conv1, bin[0].idx_down != bin[0].idx_conv1 ? bin[0].idx_down : -1};
  for (int id : ids) {
    if (id < 0) continue;
    const S8T& q = net->s8[id];
    tk_qparams qp;
    if (tk_make_qparams(q.ta1, q.ta2, TK_MODE_ACTIVATION_NONNEG, &qp) != TK_OK) return TK_ERR_THRESHOLDS;
    pk.q[pk.n_q] = q.p; pk.t0[pk.n_q] = qp.t0; pk.t1[pk.n_q] = qp.t1;
    pk.q_phases[pk.n_q] = q.phases; pk.q_R[pk.n_q] = q.R; pk.q_pos[pk.n_q] = q.pos;
    ++pk.n_q;
  }
  pk.f = bin[0].f >= 0 ? net->f32[bin[0].f].p : nullptr;
  pk.f_pos = bin[0].f >= 0 ? net->f32[bin[0].f].pos : 0;
  pk.err = net->ctx->d_err;
  return TK_OK;
}

template <int BN, int R>
cudaError_t launch_conv(const Conv& cv, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_conv_tc<BN, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  k_conv_tc<BN, R><<<cv.grid, kConvThreads, cv.smem, s>>>(cv.in_map, cv.w_map, cv.k);
  return cudaGetLastError();
}

cudaError_t run_conv(const Conv& cv, cudaStream_t s) {
  if (cv.R == 64) {
    if (cv.BN == 64) return launch_conv<64, 64>(cv, s);
    if (cv.BN == 128) return launch_conv<128, 64>(cv, s);
    return launch_conv<256, 64>(cv, s);
  }
  if (cv.BN == 64) return launch_conv<64, 128>(cv, s);
  if (cv.BN == 128) return launch_conv<128, 128>(cv, s);
  return launch_conv<256, 128>(cv, s);
}

int setup_generic(tk_net* net) {
  int H = net->in_h, W = net->in_w, C = net->in_c;
  size_t maxe = (size_t)net->batch * C * H * W;
  net->convs.assign(net->blocks.size(), {});
  for (size_t b = 0; b < net->blocks.size(); ++b) {
    const tk_block_desc& bd = net->blocks[b];
    auto& cvs = net->convs[b];
    auto mk = [&](const tk_conv_desc& d) -> int {
      Conv cv;
      cv.d = d;
      int st = tk_layer_create(net->ctx, d.weights_host, d.in_c, d.out_c, d.k, d.k, d.stride, d.pad, d.tw1, d.tw2,
                               d.ta1, d.ta2, 1, d.gain_host, d.bias_host, d.out_scale, &cv.layer);
      if (st != TK_OK) return st;
      cvs.push_back(cv);
      return TK_OK;
    };
    int h = H, w = W;
    for (int i = 0; i < bd.n_convs; ++i) {
      int st = mk(bd.conv[i]);
      if (st != TK_OK) return st;
      h = conv_out(h, bd.conv[i]);
      w = conv_out(w, bd.conv[i]);
      maxe = std::max(maxe, (size_t)net->batch * bd.conv[i].out_c * h * w);
    }
    if (bd.has_down) {
      int st = mk(bd.down);
      if (st != TK_OK) return st;
    }
    H = h; W = w; C = bd.conv[bd.n_convs - 1].out_c;
  }
  net->out_c = C; net->out_h = H; net->out_w = W;
  net->gbuf_elems = maxe;
  net->gbuf.assign(4, nullptr);
  for (auto& p : net->gbuf)
    if (cudaMalloc(&p, maxe * 4) != cudaSuccess) return TK_ERR_CUDA;
  return TK_OK;
}

}  // namespace

extern "C" {

int tk_net_create(tk_context* ctx, const tk_block_desc* blocks, int n_blocks, int batch, int in_c, int in_h,
                  int in_w, int mode, tk_net** out) {
  if (!ctx || !blocks || n_blocks <= 0 || batch <= 0 || !out) return TK_ERR_INVALID;
  tk_net* net = new tk_net;
  net->ctx = ctx;
  net->batch = batch; net->in_c = in_c; net->in_h = in_h; net->in_w = in_w;
  net->blocks.assign(blocks, blocks + n_blocks);
  // geometry / composition checks (R:linalg.hpp:40-53 per conv)
  int H = in_h, W = in_w, C = in_c;
  for (const auto& b : net->blocks) {
    if (b.n_convs < 1 || b.n_convs > 3) { delete net; return TK_ERR_INVALID; }
    int h = H, w = W, c = C;
    for (int i = 0; i < b.n_convs; ++i) {
      const tk_conv_desc& d = b.conv[i];
      if (d.in_c != c || d.out_c <= 0 || d.k <= 0 || d.stride <= 0 || d.pad < 0 || h + 2 * d.pad < d.k ||
          w + 2 * d.pad < d.k || !d.weights_host) { delete net; return TK_ERR_INVALID; }
      if (!(d.ta1 > 0.0f) || !(d.ta2 > 0.0f)) { delete net; return TK_ERR_THRESHOLDS; }
      h = conv_out(h, d); w = conv_out(w, d); c = d.out_c;
    }
    if (b.has_down) {
      const tk_conv_desc& d = b.down;
      if (d.in_c != C || d.out_c != c || conv_out(H, d) != h || conv_out(W, d) != w || !d.weights_host) {
        delete net; return TK_ERR_INVALID;
      }
    } else if (h != H || w != W || c != C) {
      delete net; return TK_ERR_INVALID;  // identity shortcut needs equal shapes
    }
    H = h; W = w; C = c;
  }
  net->fused = (mode == TK_NET_AUTO && fused_ok(net) && encode() != nullptr) ? 1 : 0;
  const int st = net->fused ? setup_fused(net) : setup_generic(net);
  if (st != TK_OK) {
    tk_net_destroy(net);
    return st;
  }
  cudaDeviceSynchronize();
  *out = net;
  return TK_OK;
}

int tk_net_destroy(tk_net* net) {
  if (!net) return TK_OK;
  cudaDeviceSynchronize();
  for (auto& cvs : net->convs)
    for (auto& cv : cvs) {
      cudaFree(cv.d_w); cudaFree(cv.d_gain); cudaFree(cv.d_bias);
      if (cv.layer) tk_layer_destroy(cv.layer);
    }
  for (auto& t : net->s8) cudaFree(t.p);
  for (auto& f : net->f32) cudaFree(f.p);
  for (auto* p : net->gbuf) cudaFree(p);
  delete net;
  return TK_OK;
}

int tk_net_out_shape(const tk_net* net, int* c, int* h, int* w) {
  if (!net) return TK_ERR_INVALID;
  if (c) *c = net->out_c;
  if (h) *h = net->out_h;
  if (w) *w = net->out_w;
  return TK_OK;
}

int tk_net_is_fused(const tk_net* net) { return net ? net->fused : -1; }

int tk_net_launches(const tk_net* net, int with_out, int with_pooled) {
  if (!net) return -1;
  int n = 0;
  if (net->fused) {
    n = 1;
    for (const auto& cvs : net->convs) n += (int)cvs.size();
  } else {
    for (const auto& cvs : net->convs) n += 3 * (int)cvs.size();  // im2col + gemm + residual
  }
  return n + (with_out ? 1 : 0) + (with_pooled ? 1 : 0);
}

int tk_net_forward(tk_context* ctx, tk_net* net, const float* x, float* out, float* pooled, void* stream) {
  if (!ctx || !net || !x) return TK_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  if (net->fused) {
    PackIn pk = net->pack;
    pk.x = x;
    const size_t sm = (size_t)pk.C * (pk.W + 1) * 4;
    if (sm > 48 * 1024) cudaFuncSetAttribute(k_pack_input, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_pack_input<<<net->batch * pk.H, 256, sm, s>>>(pk);
    if (cudaGetLastError() != cudaSuccess) return TK_ERR_CUDA;
    for (const auto& cvs : net->convs)
      for (const auto& cv : cvs)
        if (run_conv(cv, s) != cudaSuccess) return TK_ERR_CUDA;
    const F32T& f = net->f32[net->final_f];
    if (out) {
      const long long total = (long long)net->batch * f.C * f.H * f.W;
      k_unpack_f32<<<(unsigned)std::min<long long>((total + 255) / 256, 148 * 32), 256, 0, s>>>(
          f.p, f.pos, net->batch, f.C, f.H, f.W, f.Hp, f.Wp, out);
    }
    if (pooled)
      k_pool_f32<<<(net->batch * f.C + 255) / 256, 256, 0, s>>>(f.p, f.pos, net->batch, f.C, f.H, f.W, f.Hp, f.Wp,
                                                                   pooled);
    return cudaGetLastError() == cudaSuccess ? TK_OK : TK_ERR_CUDA;
  }
  // generic: NCHW floats through conv2d_ternary (R:linalg.hpp:301-328)
  float* cur = net->gbuf[0];
  cudaMemcpyAsync(cur, x, (size_t)net->batch * net->in_c * net->in_h * net->in_w * 4, cudaMemcpyDeviceToDevice, s);
  int H = net->in_h, W = net->in_w;
  for (size_t b = 0; b < net->blocks.size(); ++b) {
    const tk_block_desc& bd = net->blocks[b];
    auto& cvs = net->convs[b];
    float* bufs[3];
    int k = 0;
    for (int i = 0; i < 4; ++i)
      if (net->gbuf[i] != cur && k < 3) bufs[k++] = net->gbuf[i];
    float* h = cur;
    int hh = H, ww = W;
    float* z = nullptr;
    for (int i = 0; i < bd.n_convs; ++i) {
      z = (h == bufs[0]) ? bufs[1] : bufs[0];
      int st = tk_conv2d_ternary(ctx, cvs[i].layer, h, net->batch, hh, ww, TK_MASK_ON_THE_FLY, z, stream);
      if (st != TK_OK) return st;
      const int ho = conv_out(hh, bd.conv[i]), wo = conv_out(ww, bd.conv[i]);
      const long long n = (long long)net->batch * bd.conv[i].out_c * ho * wo;
      if (i + 1 < bd.n_convs) {
        k_residual_relu<<<(unsigned)std::min<long long>((n + 255) / 256, 148 * 32), 256, 0, s>>>(z, nullptr, n, 1);
        h = z;
      }
      hh = ho; ww = wo;
    }
    const float* sc = cur;
    if (bd.has_down) {
      int st = tk_conv2d_ternary(ctx, cvs[bd.n_convs].layer, cur, net->batch, H, W, TK_MASK_ON_THE_FLY, bufs[2],
                                 stream);
      if (st != TK_OK) return st;
      sc = bufs[2];
    }
    const long long n = (long long)net->batch * bd.conv[bd.n_convs - 1].out_c * hh * ww;
    k_residual_relu<<<(unsigned)std::min<long long>((n + 255) / 256, 148 * 32), 256, 0, s>>>(z, sc, n, 0);
    cur = z;
    H = hh; W = ww;
  }
  const long long total = (long long)net->batch * net->out_c * H * W;
  if (out) cudaMemcpyAsync(out, cur, total * 4, cudaMemcpyDeviceToDevice, s);
  if (pooled)
    k_pool_nchw<<<(net->batch * net->out_c + 255) / 256, 256, 0, s>>>(cur, net->batch * net->out_c, H * W, pooled);
  return cudaGetLastError() == cudaSuccess ? TK_OK : TK_ERR_CUDA;
}

}  // extern "C"

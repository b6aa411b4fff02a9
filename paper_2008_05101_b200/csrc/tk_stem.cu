// tk_stem.cu -- the ResNet stem convolution (float; outside the ternary path,
// it feeds the first ternary block): 7x7 / stride 2 / pad 3, 3 -> 64 channels,
// on the tensor cores as split-TF32 (tcgen05 kind::tf32, f32 accumulation).
//
// Precision: every input x and weight w is split into x = x_hi + x_lo with
// x_hi = tf32(x), x_lo = tf32(x - x_hi) (11 + 11 significant bits); the MMAs
// accumulate x_hi*w_hi + x_hi*w_lo + x_lo*w_hi in f32, which drops x_lo*w_lo
// and the bits below x_lo (relative 2^-22 per product) -- the fp32 class of
// the SIMT FMA chain this replaces, checked against fp64 in
// tests/test_gpu_net.py::test_stem_conv_matches_fp32_reference.
//
// No im2col.  The padded image is split into four (row, column)-parity phase
// planes, channel-last with one zero pad channel: element (i, j) of plane
// (py, px) = 16 bytes {c0, c1, c2, 0} of padded pixel (2i + py, 2j + px),
// Wp = (W + 7) / 2 elements per plane row.  Output position p = oy * Wp + ox
// (ox >= Wo are junk columns) reads, for tap (ky, kx), element
// p + (ky >> 1) * Wp + (kx >> 1) of plane (ky & 1, kx & 1): every tap is a
// contiguous run of rows.  The MMA's K = 8 tf32 (two 16-byte core-matrix
// chunks) covers TWO taps of one plane: a K-major no-swizzle descriptor with
// LBO = 16 bytes makes the second chunk of row r the element after it, i.e.
// tap (ky, kx + 2).  So each (plane, dy) takes two MMAs per split term:
// 28 tap-pair blocks x 3 split terms = 84 MMAs (128 x 64 x 8) per tile of
// 128 output positions.
//
// CTA (one per SM, persistent over tiles (image, 128 positions)):
//   warps 0-7   producers: warp g converts NCHW f32 into the band of phase
//               plane g % 4 (hi and lo) of every other tile = one pipeline
//               stage slot of its own (8 slots); the eight warps' loads overlap
//   warp  8     MMA issuer (one elected lane), TMEM owner
//   warps 9-12  epilogue: TMEM -> registers -> NCHW f32 (coalesced per channel)
// TMEM holds 4 accumulators of 64 columns, so the epilogue of tile i overlaps
// the MMAs of tiles i+1..i+3.
#include "tk_internal.cuh"
#include "tk_sm100.cuh"

namespace {

constexpr int kTile = 128, kCout = 64, kBlocks = 28;
constexpr int kWBlk = 2 * kCout * 16;  // one tap-pair block: [K chunk][64 rows][16 B]
constexpr int kStages = 8, kAcc = 4;  // stage slot g belongs to producer warp g
constexpr int kProd = 8, kEpi = 4;  // producer / epilogue warps
constexpr int kMmaWarp = kProd, kThreads = (kProd + 1 + kEpi) * 32;
constexpr int kMaxW = 240;  // shared memory: weights 112 KB + 8 stage slots
constexpr uint32_t kDescHi = (128u >> 4) | (1u << 14);  // SBO 128 B, descriptor version 1 (bit 46)
constexpr int kGroupWarps = 1;  // producer warps per (phase plane, tile parity)
constexpr int kPer = 17;  // band positions per producer thread per stage (band <= 17 x 32 for W <= 240)

__host__ __device__ constexpr int stem_wp(int W) { return (W + 7) / 2; }
// band positions of one tile in a plane with row parity py: dy <= 3 (py = 0)
// or 2 (py = 1) rows below, plus the tap pair's column offset <= 3 + 1
__host__ __device__ constexpr int stem_band(int wp, int py) { return (kTile + (3 - py) * wp + 4 + 7) / 8 * 8; }
// stage slots 0..7 = phases 0..3 of even tiles, then of odd tiles; hi + lo
__host__ __device__ constexpr int stem_slot_b(int wp, int py) { return 2 * stem_band(wp, py) * 16; }
__host__ __device__ constexpr int stem_slot_off(int wp, int st) {
  const int a = stem_slot_b(wp, 0), b = stem_slot_b(wp, 1), r = st & 3;
  return (st >> 2) * (2 * a + 2 * b) + (r == 0 ? 0 : r == 1 ? a : r == 2 ? 2 * a : 2 * a + b);
}
__host__ int stem_smem(int W) { return 2 * kBlocks * kWBlk + stem_slot_off(stem_wp(W), kStages) + 256 + 1024; }

// TF32 x TF32 -> F32, both K-major, M x N
__host__ __device__ constexpr uint32_t idesc_tf32(uint32_t M, uint32_t N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

// The six MMAs of one (plane, dy): tap pairs 0 and 1 x (x_hi w_hi, x_hi w_lo,
// x_lo w_hi), 128 x 64 x 8 each, one elect.sync, descriptors as 32-bit low
// halves advanced by uniform adds (A and B share the high half: SBO 128 B,
// sm_100 version bit).  a: A (x_hi) start of pair 0 in 16-B units (+ LBO
// 16 B); b: B (w_hi) block of pair 0 (+ LBO 1024 B); pair 1 is +2 positions /
// +1 block; x_lo is +a_lo units, w_lo +b_lo units.  `acc` = 0 starts the
// accumulator at the first MMA.  (One N = 128 MMA on [w_hi | w_lo] reads x_hi
// once instead of twice, but measured 11% slower.)
#define TK_TF32(AREG, BREG, PRED)       \
  "mov.b64 da, {" AREG ", %3};\n"        \
  "mov.b64 db, {" BREG ", %3};\n"        \
  "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %4, " PRED ";\n"
__device__ __forceinline__ void mma_tf32_dy(uint32_t d, uint32_t a, uint32_t b, uint32_t hi, uint32_t idesc,
                                            uint32_t acc, uint32_t a_lo, uint32_t b_lo) {
  asm volatile(
      "{\n"
      ".reg .pred e, p, t;\n"
      ".reg .b64 da, db;\n"
      ".reg .b32 a1, b1, x0, x1, w0, w1;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %5, 0;\n"
      "setp.eq.b32 t, %5, %5;\n"
      "add.u32 a1, %1, 2;\n"
      "add.u32 b1, %2, %8;\n"
      "add.u32 x0, %1, %6;\n"
      "add.u32 x1, a1, %6;\n"
      "add.u32 w0, %2, %7;\n"
      "add.u32 w1, b1, %7;\n" TK_TF32("%1", "%2", "p") TK_TF32("%1", "w0", "t") TK_TF32("x0", "%2", "t")
          TK_TF32("a1", "b1", "t") TK_TF32("a1", "w1", "t") TK_TF32("x1", "b1", "t") "}\n" ::"r"(d),
      "r"(a), "r"(b), "r"(hi), "r"(idesc), "r"(acc), "r"(a_lo), "r"(b_lo), "n"(kWBlk >> 4));
}
#undef TK_TF32

// round to the nearest TF32 (ties away from zero, = cvt.rna.tf32.f32 for
// finite values) with two integer ops: cvt.rna runs on the XU pipe (16 / clk
// / SM), which the producers' 6 conversions per position saturated
__device__ __forceinline__ float tf32_rna(float v) {
  return __uint_as_float((__float_as_uint(v) + 0x1000u) & 0xFFFFE000u);
}

// tap-pair block s -> (plane phase, dy, pair): phases 0..3 = (py, px) in
// row-major order own 8, 8, 6, 6 blocks (py = 1 has dy < 3 only: ky <= 5)
__device__ __forceinline__ int phase_base(int ph) { return ph == 0 ? 0 : ph == 1 ? 8 : ph == 2 ? 16 : 22; }

__global__ void __launch_bounds__(kThreads, 1)
k_stem_tc(const float* __restrict__ img, const float* __restrict__ wgt, int N, int H, int W, int Ho, int Wo,
          float* __restrict__ out, int dbg_arg) {
  const int dbg = TK_DBG(dbg_arg);  // profiling build: 1 = no producer work, 2 = no MMAs, 4 = no stores
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
  const int Wp = stem_wp(W);
  uint8_t* w_hi = smem;
  uint8_t* w_lo = w_hi + kBlocks * kWBlk;
  uint8_t* stages = w_lo + kBlocks * kWBlk;
  uint64_t* bars = reinterpret_cast<uint64_t*>(stages + stem_slot_off(Wp, kStages));
  uint64_t* full = bars;                 // [kStages] producers -> MMA
  uint64_t* empty = full + kStages;      // [kStages] MMA commit -> producers
  uint64_t* acc_full = empty + kStages;  // [kAcc] MMA commit -> epilogue
  uint64_t* acc_empty = acc_full + kAcc; // [kAcc] epilogue -> MMA
  uint32_t* tslot = reinterpret_cast<uint32_t*>(acc_empty + kAcc);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // weights [64][3][7][7] -> hi / lo tap-pair blocks: chunk c of block s row
  // co = {w[co][0..2][ky][kx], 0}, ky = 2 dy + py, kx = 2 (2 pair + c) + px
  for (int i = threadIdx.x; i < kBlocks * 2 * kCout; i += kThreads) {
    const int s = i >> 7, c = (i >> 6) & 1, co = i & 63;
    const int ph = s < 8 ? 0 : s < 16 ? 1 : s < 22 ? 2 : 3, r = s - phase_base(ph);
    const int ky = 2 * (r >> 1) + (ph >> 1), kx = 2 * (2 * (r & 1) + c) + (ph & 1);
    float h[4], l[4];
#pragma unroll
    for (int ch = 0; ch < 4; ++ch) {
      const float v = (ch < 3 && kx < 7) ? __ldg(wgt + ((co * 3 + ch) * 7 + ky) * 7 + kx) : 0.0f;
      h[ch] = tf32_rna(v);
      l[ch] = tf32_rna(v - h[ch]);
    }
    const int off = s * kWBlk + c * (kCout * 16) + co * 16;
    *reinterpret_cast<float4*>(w_hi + off) = make_float4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<float4*>(w_lo + off) = make_float4(l[0], l[1], l[2], l[3]);
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      sm100::mbar_init(full + s, kGroupWarps * 32);
      sm100::mbar_init(empty + s, 1);
    }
    for (int b = 0; b < kAcc; ++b) {
      sm100::mbar_init(acc_full + b, 1);
      sm100::mbar_init(acc_empty + b, kEpi * 32);
    }
    sm100::fence_mbar_init();
  }
  if (warp == kMmaWarp) sm100::tmem_alloc<kAcc * kCout>(tslot);
  sm100::fence_proxy_async_smem();  // the weight blocks -> the tensor core
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tslot;

  const int per_img = (Ho * Wp + kTile - 1) / kTile, total = N * per_img;
  if (warp < kProd) {
    // ---- producers: warp g fills phase plane g % 4 of every other tile
    // (hi then lo) into its own stage slot g = (4 tc + g % 4) % 8, so eight
    // stages' global loads are in flight at once
    const int g = warp / kGroupWarps, pt = threadIdx.x - g * kGroupWarps * 32, ph = g & 3;
    const int py = ph >> 1, px = ph & 1, band = stem_band(Wp, py), plane_b = band * 16;
    uint8_t* hi = stages + stem_slot_off(Wp, g);
    // floor(j / Wp) = umulhi(j, ceil(2^32 / Wp)) for j < 2^32 / Wp (j < 1024 here)
    const uint32_t wp_magic = (uint32_t)((0x100000000ull + Wp - 1) / Wp);
    uint32_t tc = g >> 2;
    for (int tile = blockIdx.x + (g >> 2) * gridDim.x; tile < total; tile += 2 * gridDim.x, tc += 2) {
      const uint32_t it = 4 * tc + ph, st = it % kStages;
      const int n = tile / per_img, q0 = (tile - n * per_img) * kTile;
      const int i0 = q0 / Wp, j0 = q0 - i0 * Wp;
      const float* im = img + (size_t)n * 3 * H * W;
      if (dbg & 1) {
        if (it >= kStages) sm100::mbar_wait_sleep(empty + st, ((it / kStages) - 1) & 1, 2000);
        sm100::mbar_arrive(full + st);
        continue;
      }
      // all loads of this thread's positions first (kPer x 3 in flight; their
      // latency overlaps the wait for the slot), then split + store
      float v[kPer][3];
#pragma unroll
      for (int m = 0; m < kPer; ++m) {
        const int k = pt + m * kGroupWarps * 32, jj = j0 + k, di = (int)__umulhi((uint32_t)jj, wp_magic);
        const int i = i0 + di, j = jj - di * Wp;
        const int y = 2 * i + py - 3, x = 2 * j + px - 3;
        const bool in = k < band && y >= 0 && y < H && x >= 0 && x < W;
        const float* src = im + (in ? (size_t)y * W + x : 0);
#pragma unroll
        for (int c = 0; c < 3; ++c) v[m][c] = in ? __ldg(src + (size_t)c * H * W) : 0.0f;
      }
      if (it >= kStages) sm100::mbar_wait_sleep(empty + st, ((it / kStages) - 1) & 1, 2000);
#pragma unroll
      for (int m = 0; m < kPer; ++m) {
        const int k = pt + m * kGroupWarps * 32;
        if (k >= band) break;
        float h[3], l[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          h[c] = tf32_rna(v[m][c]);
          l[c] = tf32_rna(v[m][c] - h[c]);
        }
        *reinterpret_cast<float4*>(hi + k * 16) = make_float4(h[0], h[1], h[2], 0.0f);
        *reinterpret_cast<float4*>(hi + plane_b + k * 16) = make_float4(l[0], l[1], l[2], 0.0f);
      }
      sm100::fence_proxy_async_smem();
      sm100::mbar_arrive(full + st);
    }
  } else if (warp == kMmaWarp) {
    // ---- MMA issuer
    constexpr uint32_t idesc = idesc_tf32(kTile, kCout);
    const uint32_t whi = sm100::smem_u32(w_hi), wlo = sm100::smem_u32(w_lo), st0 = sm100::smem_u32(stages);
    uint32_t it = 0, tc = 0;
    for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++tc) {
      const uint32_t b = tc % kAcc;
      if (tc >= kAcc) sm100::mbar_wait(acc_empty + b, ((tc / kAcc) - 1) & 1);
      sm100::tc_fence_after();
      const uint32_t d = tmem + b * kCout;
      uint32_t acc = 0;
      for (int ph = 0; ph < 4; ++ph, ++it) {
        const int st = it % kStages;
        sm100::mbar_wait(full + st, (it / kStages) & 1);
        sm100::tc_fence_after();
        const uint32_t ahi = st0 + stem_slot_off(Wp, st), alo = ahi + stem_band(Wp, ph >> 1) * 16;
        const int ny = (ph >> 1) ? 3 : 4, s0 = phase_base(ph);
        const uint32_t a0 = (ahi >> 4) | (1u << 16), b0 = ((whi >> 4) + (uint32_t)s0 * (kWBlk >> 4)) | (64u << 16);
        for (int dy = 0; dy < ny && !(dbg & 2); ++dy) {
          mma_tf32_dy(d, a0 + dy * Wp, b0 + dy * 2 * (kWBlk >> 4), kDescHi, idesc, acc, (alo - ahi) >> 4,
                      (wlo - whi) >> 4);
          acc = 1;
        }
        sm100::mma_commit_elect(empty + st);  // the stage's band may be refilled once these MMAs are done
      }
      sm100::mma_commit_elect(acc_full + b);
    }
  } else {
    // ---- epilogue: warp (w % 4) owns TMEM lanes 32 (w % 4) .. +31 = positions
    const int qd = warp & 3;
    uint32_t tc = 0;
    for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++tc) {
      const uint32_t b = tc % kAcc;
      sm100::mbar_wait_sleep(acc_full + b, (tc / kAcc) & 1, 2000);
      sm100::tc_fence_after();
      uint32_t r0[32], r1[32];
      const uint32_t ta = tmem + ((uint32_t)(qd * 32) << 16) + b * kCout;
      sm100::tmem_ld32(ta, r0);
      sm100::tmem_ld32(ta + 32, r1);
      sm100::tmem_ld_wait();
      sm100::tc_fence_before();
      sm100::mbar_arrive(acc_empty + b);
      const int n = tile / per_img, p = (tile - n * per_img) * kTile + qd * 32 + lane;
      const int oy = p / Wp, ox = p - oy * Wp;
      if (oy < Ho && ox < Wo && !(dbg & 4)) {
        float* o = out + ((size_t)n * kCout * Ho + oy) * Wo + ox;
        const size_t cs = (size_t)Ho * Wo;
#pragma unroll
        for (int c = 0; c < 32; ++c) o[c * cs] = __uint_as_float(r0[c]);
#pragma unroll
        for (int c = 0; c < 32; ++c) o[(c + 32) * cs] = __uint_as_float(r1[c]);
      }
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc<kAcc * kCout>(tmem);
  }
}

}  // namespace

// 0 = launched; TK_ERR_UNSUPPORTED when the shape is outside the kernel
int tk_launch_stem_tc(tk_context* ctx, const float* images, int n, int h, int w, const float* weights, float* out,
                      void* stream) {
  if (w > kMaxW || h < 1) return TK_ERR_UNSUPPORTED;
  const int ho = (h - 1) / 2 + 1, wo = (w - 1) / 2 + 1, wp = stem_wp(w);
  const int smem = stem_smem(w);
  if (tk_smem_attr((const void*)k_stem_tc, smem) != cudaSuccess) return TK_ERR_CUDA;
  const long long tiles = (long long)n * ((ho * wp + kTile - 1) / kTile);
  const int grid = (int)std::min<long long>(tiles, ctx->num_sms);
  k_stem_tc<<<grid, kThreads, smem, (cudaStream_t)stream>>>(images, weights, n, h, w, ho, wo, out,
                                                          tk_knob("TK_STEM_DBG", 0));
  return cudaGetLastError() == cudaSuccess ? TK_OK : TK_ERR_CUDA;
}

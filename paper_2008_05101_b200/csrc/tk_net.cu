// tk_net.cu -- network-level ternary inference: the fused tensor-core conv
// pipeline (implicit im2col, folded BN + skip-add + ReLU + next-layer
// quantize in the epilogue) and the generic layer-by-layer path.
//
// Composition (R:tinynet.hpp:713-735, applied to conv blocks; oracle:
// oracle/ternkit_oracle.c or_net_body, reference: oracle/ref_shim.cpp):
//   h = x; for inner convs: h = max(conv2d_ternary(h), 0)
//   out = max(conv2d_ternary_last(h) + (down ? conv2d_ternary_down(x) : x), 0)
//
// Fused-path data layout (HBM-resident, per activation tensor):
//  * s8 levels  [C/R][phase][pos][R]   R = 64 (C == 64) or 128 channels,
//    pos = padded position n*PH*PW + py*PW + px of a zero-padded (pad 1)
//    image; stride-2 consumers get the 4 (row, col)-parity phase planes so
//    every kernel tap is a contiguous row range.  The pad ring is zero
//    (= the code of quantize(0.0)), written once and never touched.
//  * f32 NCHW tensors only where a residual add (or the head) needs floats.
// Conv kernel (tcgen05 kind::i8): a CTA owns a 128-position tile; for each
// 64/128-channel chunk ONE TMA box loads the tile plus halo (rows shifted by
// up to 2*Wp+2) into SMEM with the hardware swizzle, and every tap of the
// 3x3 window is an MMA whose A descriptor simply starts `shift` rows later
// (verified on B200: tools/desc_test.cu).  Weights stream through a TMA ring
// (or stay resident when they fit).  Accumulators rotate through 2-4 TMEM
// buffers so the epilogue of tile i overlaps the MMAs of the next tiles.
// Epilogue: inner convs (ReLU then quantize for the next conv, no float
// needed) compare the INTEGER accumulator against per-channel integer
// thresholds precomputed from the exact float epilogue (monotone in acc), so
// the level bytes are bit-identical to quantize(max(fma(g, s*acc, b), 0)).
#include <cuda.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include <cstdio>

#include "tk_internal.cuh"
#include "tk_sm100.cuh"

namespace {

// warp 0 TMA, warp 1 MMA, then G epilogue groups of 4 warps (one per TMEM
// lane quarter).  G = 3 groups take turns on items (MT = 1); with two M tiles
// per item (MT = 2) group g takes tile g.  Three groups fit because the
// epilogue walks the accumulator row 16 columns at a time (<= 128 registers).
// (a group waits on accumulator-buffer parity, so groups <= buffers: with
// at most one pass of lead no waiter can match a stale phase)
// GPI (column split): a BN = 256 single-tile item may be shared by two groups,
// each taking half its columns, so 16 epilogue warps (not 8) keep skip loads
// and stores in flight on the wide f32-epilogue layers (chosen per conv, §4.6)
__host__ __device__ constexpr int conv_groups(int BN, int MT, int GPI = 1) {
  return MT >= 2 ? 4 : (BN == 64 ? 4 : (BN <= 128 ? 3 : 2 * GPI));
}
__host__ __device__ constexpr int conv_threads(int BN, int MT, int GPI = 1) {
  return 64 + 128 * conv_groups(BN, MT, GPI);
}
// accumulator columns per epilogue step: 16 keeps 3-4 groups within 128 /
// 96 registers; with 2 groups (168 registers) 32 columns double the f32
// skip loads in flight per thread (the wide 1x1 f32-epilogue layers of
// ResNet-50 are HBM-latency bound)
// (measured: pays off on the 1x1 layers; the 3x3 ones spill)
__host__ __device__ constexpr int conv_chunk(int BN, int MT, int KT, int GPI = 1) {
  return conv_groups(BN, MT, GPI) == 2 && KT == 1 ? 32 : 16;
}

struct ConvK {
  int n_taps;
  int tap_slot[9];
  int tap_shift[9];
  int n_ph;
  int ph_id[4];
  int halo_rows;
  int hbox, nbox;  // halo rows per TMA box, boxes per halo (a box spans <= 256 rows)
  int chunks;
  long long in_pos;  // rows per phase plane of the input tensor
  int in_phases;
  int base_shift;
  int n_tiles, m_tiles, m_items;  // m_items = ceil(m_tiles / MT)
  long long m_total;
  int PHg, PWg, Ho, Wo;
  int hs, ws, resident;
  int HB, WB;  // bytes per halo box / weight block (1024 aligned)
  // epilogue
  const float* gain;
  const float* bias;
  const int* ithr;  // [n_q][3][N] (c0, c1, sign) integer-threshold mode, or null
  int ithr16;       // 1: ithr holds [n_q][N] (c0 & 0xffff) | c1 << 16 (all signs +1);
                    // 2: per channel pair (-c0, -c0') and (-c1, -c1') as s16x2 (DPX form)
  float out_scale;
  int relu;
  int N;
  // Residual tensors inside the network are channel-blocked, [N][C/16][H*W][16]
  // (element (n, c, p) at ((n * C/16 + c/16) * HW + p) * 16 + c % 16): a
  // thread's 16-channel chunk is one (s16) or two (f32) 32-byte sectors moved
  // by 256-bit accesses, and the 32 positions of a warp are contiguous, so
  // stores write whole lines.  The forward's input x (an identity shortcut of
  // the first block) and a conv2d_ternary plan's output are NCHW.
  const float* skip;  // blocked (skip_cl) or NCHW
  float* fout;        // blocked (fout_cl) or NCHW
  int skip_cl, fout_cl;
  int res16_cl;  // the s16 downsample residual (aout / skip16) channel-blocked, else NCHW
  // exact s16 residual of a downsample conv: that conv stores its integer
  // accumulators (aout) instead of f32 and the consumer recomputes the folded
  // BN, fmaf(sk_gain, sk_scale * acc, sk_bias) -- the same f32 bits, half the bytes
  int16_t* aout;         // blocked (res16_cl) or NCHW, downsample conv
  const int16_t* skip16; // blocked (res16_cl) or NCHW, the block's last conv
  const float* sk_gain;
  const float* sk_bias;
  float sk_scale;
  int o_Hp, o_Wp, o_PH, o_PW;
  int n_q;
  int8_t* q[2];
  float t0[2], t1[2];
  int q_phases[2], q_R[2];
  long long q_pos[2];
  int q_same;  // both quantized outputs use the same thresholds (levels computed once)
  unsigned long long* err;
  int dbg;  // profiling knob (env TK_CONV_DBG): 1 no MMA, 2 no halo TMA, 4 no epilogue,
            // float epilogue parts: 128 no quantize, 256 no f32 store, 512 no skip load
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

template <int kThreads>
__device__ __forceinline__ void epi_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(kThreads) : "memory");
}

// profiling stamps (dbg & 16): per CTA [start, setup done, MMA loop done,
// epilogue loop done, end] in globaltimer ns
__device__ unsigned long long g_stamps[148 * 8];
// CTA 0 event trace (dbg & 16): [role][item] for the first 32 items
// role 0 producer after h_empty wait, 1 MMA after a_empty wait, 2 MMA after
// h_full wait, 3 epilogue group after a_full wait, 4 epilogue done
__device__ unsigned long long g_trace[8 * 32];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// MT = 128-row M tiles per work item (they share every weight block and the
// per-item pipeline overhead); each accumulator buffer holds MT x BN columns
template <int BN, int MT>
struct Acc {
  static constexpr int kN = BN * MT <= 128 ? 4 : (BN * MT <= 256 ? 2 : 1);  // accumulator buffers
  static constexpr uint32_t kCols = kN * BN * MT;    // TMEM columns (power of 2)
};

template <int BN, int R, int KT, int MT, int GPI>
__global__ void __launch_bounds__(conv_threads(BN, MT, GPI), 1)
k_conv_tc(const __grid_constant__ CUtensorMap in_map, const __grid_constant__ CUtensorMap w_map,
          const ConvK p) {
  constexpr int kAcc = Acc<BN, MT>::kN;
  constexpr uint32_t kCols = Acc<BN, MT>::kCols;
  constexpr int kSteps = R / 32;  // MMAs (K = 32) per tap and chunk
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment by pointer arithmetic on the __shared__ array (not
  // through an integer cast) so derived pointers keep the shared address
  // space and the epilogue's parameter reads compile to LDS, not generic LD
  uint8_t* smem = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* halo = smem;
  const int halo_stage = p.n_ph * p.HB;
  uint8_t* wreg = halo + p.hs * halo_stage;
  const int wblocks = p.resident ? p.chunks * p.n_taps : p.ws;
  // epilogue parameter slots (2, by item parity): 6*BN words each
  // epilogue parameters of all N channels, staged once: int mode
  // [n_q][3][N] (c0, c1, sign), float mode [2][N] (gain, bias)
  uint32_t* eparam = reinterpret_cast<uint32_t*>(wreg + (size_t)wblocks * p.WB);
  // epilogue parameters: integer thresholds, or gain / bias (+ the residual's
  // gain / bias when it arrives as s16 accumulators)
  const int ewords = p.ithr ? (p.ithr16 ? p.n_q * p.N : p.n_q * 3 * p.N) : (p.skip16 ? 4 : 2) * p.N;
  uint64_t* bars = reinterpret_cast<uint64_t*>(eparam + ((ewords + 1) & ~1));
  uint64_t* h_full = bars;
  uint64_t* h_empty = h_full + p.hs;
  uint64_t* w_full = h_empty + p.hs;
  uint64_t* w_empty = w_full + p.ws;
  uint64_t* a_full = w_empty + p.ws;
  uint64_t* a_empty = a_full + kAcc;
  uint64_t* w_res = a_empty + kAcc;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(w_res + 1);
  // tap A-operand byte offsets and halo phase ids in (static) shared memory:
  // the issue loops read them with LDS instead of indexing kernel parameters
  __shared__ uint32_t s_tap[9];
  __shared__ int s_ph[4];

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const bool stamp = (TK_DBG(p.dbg) & 16) && blockIdx.x < 148;
  if (stamp && threadIdx.x == 0) g_stamps[blockIdx.x * 8 + 0] = gtime();

  if (threadIdx.x == 0) {
    sm100::pdl_launch_dependents();
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
    for (int s = 0; s < kAcc; ++s) {
      sm100::mbar_init(&a_full[s], 1);
      sm100::mbar_init(&a_empty[s], 128 * MT * GPI);  // the groups sharing an item
    }
    sm100::mbar_init(w_res, 1);
#pragma unroll
    for (int t = 0; t < 9; ++t) s_tap[t] = (uint32_t)(p.tap_slot[t] * p.HB + p.tap_shift[t] * R);
#pragma unroll
    for (int s = 0; s < 4; ++s) s_ph[s] = p.ph_id[s];
    sm100::fence_mbar_init();
  }
  if (warp == 1) sm100::tmem_alloc<kCols>(tslot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tslot;
  const int n_items = p.m_items * p.n_tiles;
  // CTAs walk the (chunk, tap) weight blocks from different starting points
  // (integer sums are order independent) so they do not all hit the same L2
  // lines at once.
  const int rot_c = blockIdx.x % p.chunks;

  // The producer and MMA roles run as WHOLE warps (all lanes wait on the
  // barriers, lane 0 issues).  Ring positions advance with (stage, round)
  // counters -- no integer division in the issue loops: a single issuing
  // thread's dependent scalar latency is what bounds the MMA issue rate.
  if (warp == 0) {
    // ================= producer =================
    if (p.resident && lane == 0) {  // all weight blocks of the (single) n-tile, once
      sm100::mbar_arrive_expect_tx(w_res, (uint32_t)(p.chunks * p.n_taps) * BN * R);
      for (int b = 0; b < p.chunks * p.n_taps; ++b)
        sm100::tma_load_2d(wreg + (size_t)b * p.WB, &w_map, w_res, 0, b * BN);
    }
    // weights are constant: their loads overlap the previous layer's tail;
    // activations only after that layer has completed (PDL)
    sm100::pdl_wait();
    int hs_i = 0, h_round = 0, ws_i = 0, w_round = 0;
    int mt = blockIdx.x / p.n_tiles, nt = blockIdx.x - mt * p.n_tiles;
    const int dmt = gridDim.x / p.n_tiles, dnt = gridDim.x - dmt * p.n_tiles;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int row0 = mt * (MT * 128) + p.base_shift;
      int ch = rot_c;
      for (int ci = 0; ci < p.chunks; ++ci) {
        if (h_round) sm100::mbar_wait(&h_empty[hs_i], (h_round - 1) & 1);
        if (lane == 0) {
          if (stamp && blockIdx.x == 0 && h_round * p.hs + hs_i < 32)
            g_trace[0 * 32 + h_round * p.hs + hs_i] = clock64();
          if (TK_DBG(p.dbg) & 2) {
            sm100::mbar_arrive(&h_full[hs_i]);
          } else {
            sm100::mbar_arrive_expect_tx(&h_full[hs_i], (uint32_t)(p.n_ph * p.nbox * p.hbox * R));
            const long long rbase = (long long)ch * p.in_phases * p.in_pos + row0;
            for (int s2 = 0; s2 < p.n_ph; ++s2)
              for (int b = 0; b < p.nbox; ++b)
                sm100::tma_load_2d(halo + hs_i * halo_stage + s2 * p.HB + b * p.hbox * R, &in_map, &h_full[hs_i],
                                   0, (int)(rbase + (long long)s_ph[s2] * p.in_pos + b * p.hbox));
          }
        }
        __syncwarp();
        if (++hs_i == p.hs) { hs_i = 0; ++h_round; }
        if (!p.resident) {
          const int blk0 = (nt * p.chunks + ch) * KT;
          for (int t = 0; t < KT; ++t) {
            if (w_round) sm100::mbar_wait(&w_empty[ws_i], (w_round - 1) & 1);
            if (lane == 0) {
              sm100::mbar_arrive_expect_tx(&w_full[ws_i], BN * R);
              sm100::tma_load_2d(wreg + (size_t)ws_i * p.WB, &w_map, &w_full[ws_i], 0, (blk0 + t) * BN);
            }
            __syncwarp();
            if (++ws_i == p.ws) { ws_i = 0; ++w_round; }
          }
        }
        if (++ch == p.chunks) ch = 0;
      }
      mt += dmt;
      nt += dnt;
      if (nt >= p.n_tiles) { nt -= p.n_tiles; ++mt; }
    }
  } else if (warp == 1) {
    // ================= MMA issuer (warp-uniform, elect.sync issues) ======
    constexpr uint32_t idesc = sm100::idesc_i8(128, BN);
    if (stamp && lane == 0) g_stamps[blockIdx.x * 8 + 1] = gtime();
    if (p.resident) sm100::mbar_wait(w_res, 0);
    if (stamp && lane == 0) g_stamps[blockIdx.x * 8 + 2] = gtime();
    // descriptor templates: only the start-address field (bits 0-13, in
    // 16-byte units) changes per MMA
    const uint64_t tmpl = desc_sw(0, R);
    const uint32_t dhi = (uint32_t)(tmpl >> 32);  // SBO, version, swizzle mode
    const uint32_t halo0 = sm100::smem_u32(halo), wreg0 = sm100::smem_u32(wreg);
    uint32_t toff[KT];
#pragma unroll
    for (int t = 0; t < KT; ++t) toff[t] = (uint32_t)(p.tap_slot[t] * p.HB + p.tap_shift[t] * R);
    const bool do_mma = !(TK_DBG(p.dbg) & 1);
    int hs_i = 0, h_round = 0, ws_i = 0, w_round = 0, acc = 0, a_round = 0, it = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
      if (stamp && lane == 0 && blockIdx.x == 0 && it < 32) g_trace[6 * 32 + it] = clock64();
      if (a_round) sm100::mbar_wait(&a_empty[acc], (a_round - 1) & 1);
      if (stamp && lane == 0 && blockIdx.x == 0 && it < 32) g_trace[1 * 32 + it] = clock64();
      sm100::tc_fence_after();
      if (stamp && lane == 0 && blockIdx.x == 0 && it < 32) g_trace[7 * 32 + it] = clock64();
      const uint32_t d = tmem + acc * (BN * MT);
      int ch = rot_c;
      for (int ci = 0; ci < p.chunks; ++ci) {
        sm100::mbar_wait(&h_full[hs_i], h_round & 1);
        if (stamp && lane == 0 && blockIdx.x == 0 && h_round * p.hs + hs_i < 32)
          g_trace[2 * 32 + h_round * p.hs + hs_i] = clock64();
        sm100::tc_fence_after();
        // descriptor low halves: start address >> 4 in bits 0-13 (smem
        // addresses < 2^18, so per-MMA offsets are plain adds) | LBO = 1
        const uint32_t a0 = ((halo0 + hs_i * halo_stage) >> 4) | (1u << 16);
        const uint32_t wres = ((wreg0 + (uint32_t)(ch * KT) * p.WB) >> 4) | (1u << 16);
#pragma unroll
        for (int t = 0; t < KT; ++t) {
          uint32_t b0;
          if (p.resident) {
            b0 = wres + (uint32_t)t * (p.WB >> 4);
          } else {
            sm100::mbar_wait(&w_full[ws_i], w_round & 1);
            sm100::tc_fence_after();
            b0 = (((wreg0 + (uint32_t)ws_i * p.WB)) >> 4) | (1u << 16);
          }
          const uint32_t at = a0 + (toff[t] >> 4);
          if (do_mma) {
            if constexpr (MT <= 2)
              sm100::mma_tap_elect<kSteps, MT>(d, at, b0, dhi, idesc, (ci | t) != 0, (uint32_t)(128 * R / 16),
                                               (uint32_t)BN);
            else
#pragma unroll
              for (int k = 0; k < kSteps; ++k)
#pragma unroll
                for (int u = 0; u < MT; ++u)
                  sm100::mma_i8_elect_lohi(d + u * BN, at + (uint32_t)((u * 128 * R + k * 32) >> 4), dhi,
                                           b0 + (uint32_t)(k * 2), dhi, idesc, (ci | t | k) != 0);
          }
          if (!p.resident) {
            sm100::mma_commit_elect(&w_empty[ws_i]);
            if (++ws_i == p.ws) { ws_i = 0; ++w_round; }
          }
        }
        if (stamp && lane == 0 && blockIdx.x == 0 && h_round * p.hs + hs_i < 32)
          g_trace[4 * 32 + h_round * p.hs + hs_i] = clock64();
        sm100::mma_commit_elect(&h_empty[hs_i]);
        if (++hs_i == p.hs) { hs_i = 0; ++h_round; }
        if (++ch == p.chunks) ch = 0;
      }
      sm100::mma_commit_elect(&a_full[acc]);
      if (stamp && lane == 0 && blockIdx.x == 0 && it < 32) g_trace[5 * 32 + it] = clock64();
      if (++acc == kAcc) { acc = 0; ++a_round; }
    }
    if (stamp && lane == 0) g_stamps[blockIdx.x * 8 + 3] = gtime();
  } else if (warp >= 2) {
    // ================= epilogue =========================================
    // G groups of 4 warps take turns on items (several items in flight hide
    // the TMEM-load and memory latencies); within a group warp w owns TMEM
    // lane quarter w % 4 and walks all BN columns.
    constexpr int G = conv_groups(BN, MT, GPI), kEpiThreads = 128 * G;
    constexpr int CH = conv_chunk(BN, MT, KT, GPI);
    constexpr int IG = G / GPI, BNG = BN / GPI;  // item groups, columns per group
    static_assert(IG / MT <= kAcc, "epilogue groups must not outnumber accumulator buffers");
    const int et = threadIdx.x - 64;
    const int qtr = warp & 3;
    const int grp = (warp - 2) >> 2;
    const int igrp = grp / GPI, half = grp % GPI;  // item-slot group, column part
    const int plane = p.PHg * p.PWg;
    const long long oplane = (long long)p.Ho * p.Wo;
    if constexpr (BN >= 128) {
      for (int i = et; i < ewords; i += kEpiThreads)
        eparam[i] = p.ithr ? (uint32_t)__ldg(p.ithr + i)
                           : __float_as_uint(__ldg(i < p.N       ? p.gain + i
                                                   : i < 2 * p.N ? p.bias + (i - p.N)
                                                   : i < 3 * p.N ? p.sk_gain + (i - 2 * p.N)
                                                                 : p.sk_bias + (i - 3 * p.N)));
    } else {
      for (int i = et; i < ewords; i += kEpiThreads)
        eparam[i] = p.ithr ? (uint32_t)__ldg(p.ithr + i)
                           : __float_as_uint(__ldg((i < p.N ? p.gain : p.bias - p.N) + i));
    }
    epi_bar<kEpiThreads>();
    sm100::pdl_wait();  // skip inputs / outputs of the neighbouring layers
    const uint32_t* ep = eparam;
    const uint32_t ostride = (uint32_t)oplane;  // CH channel planes < 2^31 elements
    const bool has_skip = (p.skip || (BN >= 128 && p.skip16)) && !(TK_DBG(p.dbg) & (4 | 512));
    // element offset of (item's first channel, this thread's position) in the
    // NCHW skip tensor, or -1 when the position is past the batch / padding
    // channel-last skip (internal f32 or s16 residual): chunk c0 is at
    // base + c0; NCHW (the forward's input): at base + c0 * plane
    const bool skip_cl = p.skip16 ? p.res16_cl != 0 : p.skip_cl != 0;
    const long long bstride = oplane * 16;  // elements per 16-channel block of an image
    // offset of channel c (a multiple of 16) from channel 0 of a position
    auto ch_off = [&](int c, bool cl) -> long long { return cl ? (long long)(c >> 4) * bstride : (long long)c * ostride; };
    auto skip_at = [&](int item) -> long long {
      const int mi = item / p.n_tiles, nt = item - mi * p.n_tiles;
      const int qrow = (mi * MT + igrp % MT) * 128 + qtr * 32 + lane;
      const int img = qrow / plane, rem = qrow - img * plane;
      const int oy = rem / p.PWg, ox = rem - (rem / p.PWg) * p.PWg;
      if (!(qrow < p.m_total && oy < p.Ho && ox < p.Wo)) return -1;
      if (skip_cl)
        return (long long)img * p.N * oplane + ((long long)oy * p.Wo + ox) * 16 + ch_off(nt * BN + half * BNG, true);
      return (long long)img * p.N * oplane + (long long)oy * p.Wo + ox + (long long)(nt * BN + half * BNG) * oplane;
    };
    // CH skip values (raw bits: f32, or the sign-extended s16 accumulator) of
    // one chunk; converted only where they are used, so the loads stay in flight
    auto load_skip = [&](long long base, uint32_t (&skr)[CH]) {
      if (p.skip16 && !p.res16_cl) {
        const int16_t* q = p.skip16 + base;
#pragma unroll
        for (int j = 0; j < CH; ++j, q += ostride) skr[j] = (uint32_t)(int32_t)__ldg(q);
      } else if (p.skip16) {
#pragma unroll
        for (int h = 0; h < CH / 16; ++h) {
          uint32_t w[8];
          sm100::ld_nc_v8(p.skip16 + base + h * bstride, w);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            skr[16 * h + 2 * i] = (uint32_t)(int32_t)(int16_t)(w[i] & 0xFFFFu);
            skr[16 * h + 2 * i + 1] = (uint32_t)((int32_t)w[i] >> 16);
          }
        }
      } else if (p.skip_cl) {
#pragma unroll
        for (int h = 0; h < CH / 8; ++h) {
          uint32_t w[8];
          sm100::ld_nc_v8(p.skip + base + (h >> 1) * bstride + 8 * (h & 1), w);
#pragma unroll
          for (int i = 0; i < 8; ++i) skr[8 * h + i] = w[i];
        }
      } else {
        const float* q = p.skip + base;
#pragma unroll
        for (int j = 0; j < CH; ++j, q += ostride) skr[j] = __float_as_uint(__ldg(q));
      }
    };
    uint32_t skr[CH];        // skip values of the next chunk to consume
    bool skr_ready = false;  // skr already holds this item's first chunk (loaded one item ahead)
    int it = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
      // MT == 1: the groups take turns on items; MT > 1: group g takes M tile
      // g % MT of every (G/MT)-th item
      if (it % (IG / MT) != igrp / MT) continue;
      const int mi = item / p.n_tiles, nt = item - mi * p.n_tiles;
      const int mt = mi * MT + igrp % MT;
      const uint32_t tcol = (uint32_t)(it % kAcc) * (BN * MT) + (igrp % MT) * BN + half * BNG;
      const int acc = it % kAcc;
      if (TK_DBG(p.dbg) & 8) {  // profiling: bare accumulator hand-off
        if (!(TK_DBG(p.dbg) & 64) || lane == 0) sm100::mbar_wait(&a_full[acc], (it / kAcc) & 1);
        __syncwarp();
        if (stamp && blockIdx.x == 0 && it < 32 && qtr == 0 && lane == 0) g_trace[3 * 32 + it] = clock64();
        sm100::tc_fence_after();
        sm100::tc_fence_before();
        sm100::mbar_arrive(&a_empty[acc]);
        continue;
      }
      const int qrow = mt * 128 + qtr * 32 + lane;  // m_total < 2^31 (checked at setup)
      const int img = qrow / plane;
      const int rem = qrow - img * plane;
      const int oy = rem / p.PWg, ox = rem - (rem / p.PWg) * p.PWg;
      const bool valid = qrow < p.m_total && oy < p.Ho && ox < p.Wo;
      const long long P1 = ((long long)img * p.o_Hp + oy + 1) * p.o_Wp + ox + 1;
      const int py = oy + 1, px = ox + 1;
      const long long P4 = ((long long)img * p.o_PH + (py >> 1)) * p.o_PW + (px >> 1);
      const int ph4 = (py & 1) * 2 + (px & 1);
      // NCHW index of (img, channel 0, oy, ox) in the f32 skip / output tensors,
      // and the channel-last one ((img, oy, ox) * C)
      const long long fbase = (long long)img * p.N * oplane + (long long)oy * p.Wo + ox;
      const long long hbase = (long long)img * p.N * oplane + ((long long)oy * p.Wo + ox) * 16;
      // skip values are independent of the accumulator: the first chunk's
      // loads were issued during the previous item's last chunk (else here,
      // before waiting for the MMAs), each later chunk's while the previous
      // one is finished (HBM latency off the critical path)
      const bool pre = has_skip && valid;
      const long long skb = (skip_cl ? hbase : fbase) + ch_off(nt * BN + half * BNG, skip_cl);
      // BN = 64 kernels (576 threads at the register cap) keep the plain f32
      // form: measured faster than the raw-bit / one-item-ahead variant there
      float sk[CH];
      if constexpr (BN >= 128) {
        if (pre && !skr_ready) load_skip(skb, skr);
        skr_ready = false;
      } else if (pre) {
        if (p.skip_cl) {
#pragma unroll
          for (int h = 0; h < CH / 8; ++h) {
            uint32_t w[8];
            sm100::ld_nc_v8(p.skip + skb + (h >> 1) * bstride + 8 * (h & 1), w);
#pragma unroll
            for (int i = 0; i < 8; ++i) sk[8 * h + i] = __uint_as_float(w[i]);
          }
        } else {
          const float* q = p.skip + skb;
#pragma unroll
          for (int j = 0; j < CH; ++j, q += ostride) sk[j] = __ldg(q);
        }
      }
      if (TK_DBG(p.dbg) & 1024)
        sm100::mbar_wait(&a_full[acc], (it / kAcc) & 1);
      else
        sm100::mbar_wait_sleep(&a_full[acc], (it / kAcc) & 1, 2000);
      sm100::tc_fence_after();
#pragma unroll 1
      for (int c0 = 0; c0 < BNG; c0 += CH) {
        uint32_t r[CH];
        if constexpr (CH == 32)
          sm100::tmem_ld32(tmem + ((uint32_t)(qtr * 32) << 16) + tcol + c0, r);
        else
          sm100::tmem_ld16(tmem + ((uint32_t)(qtr * 32) << 16) + tcol + c0, r);
        sm100::tmem_ld_wait();
        if (!valid || (TK_DBG(p.dbg) & 4)) continue;
        const int n0 = nt * BN + half * BNG + c0;
        if (p.ithr) {
          // integer-threshold epilogue: level = (s*acc > c0) + (s*acc > c1)
#pragma unroll
          for (int o = 0; o < 2; ++o) {
            if (o >= p.n_q) break;
            uint32_t w[CH / 4];
            if (p.ithr16 == 2) {
              // channel pairs as s16x2: (acc > c) = max(min(acc - c, 1), 0),
              // one DPX add-min-relu per threshold and pair; 4 levels -> 4 bytes
              const uint4* e0 = reinterpret_cast<const uint4*>(ep + o * p.N + n0);
#pragma unroll
              for (int j = 0; j < CH / 4; ++j) {
                const uint4 cc = e0[j];
                const uint32_t x01 = __byte_perm(r[4 * j], r[4 * j + 1], 0x5410);
                const uint32_t x23 = __byte_perm(r[4 * j + 2], r[4 * j + 3], 0x5410);
                const uint32_t l01 = __viaddmin_s16x2_relu(x01, cc.x, 0x00010001u) +
                                     __viaddmin_s16x2_relu(x01, cc.y, 0x00010001u);
                const uint32_t l23 = __viaddmin_s16x2_relu(x23, cc.z, 0x00010001u) +
                                     __viaddmin_s16x2_relu(x23, cc.w, 0x00010001u);
                w[j] = __byte_perm(l01, l23, 0x6420);
              }
            } else if (p.ithr16) {
              // (c0, c1) s16 pairs of 4 channels per 16-byte LDS (broadcast):
              // a third of the shared-memory wavefronts of the general form,
              // which competes with the MMA operand reads
              const uint4* e0 = reinterpret_cast<const uint4*>(ep + o * p.N + n0);
#pragma unroll
              for (int j = 0; j < CH / 4; ++j) {
                const uint4 cc = e0[j];
                const uint32_t cw[4] = {cc.x, cc.y, cc.z, cc.w};
                uint32_t b = 0;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  const int x = (int)r[4 * j + i];
                  b += ((x > (int)(int16_t)(cw[i] & 0xFFFFu)) ? (1u << (8 * i)) : 0u) +
                       ((x > ((int)cw[i] >> 16)) ? (1u << (8 * i)) : 0u);
                }
                w[j] = b;
              }
            } else {
              // (c0, c1, sign) of 4 channels per 16-byte LDS (broadcast: all
              // lanes read the same channels)
              const int4* e0 = reinterpret_cast<const int4*>(ep + o * 3 * p.N + n0);
              const int n4 = p.N / 4;
#pragma unroll
              for (int j = 0; j < CH / 4; ++j) {
                const int4 lo = e0[j], hi = e0[n4 + j], sg = e0[2 * n4 + j];
                const int xs[4] = {(int)r[4 * j] * sg.x, (int)r[4 * j + 1] * sg.y, (int)r[4 * j + 2] * sg.z,
                                   (int)r[4 * j + 3] * sg.w};
                const int l0[4] = {lo.x, lo.y, lo.z, lo.w}, l1[4] = {hi.x, hi.y, hi.z, hi.w};
                uint32_t b = 0;
#pragma unroll
                for (int i = 0; i < 4; ++i)
                  b |= ((uint32_t)(xs[i] > l0[i]) + (uint32_t)(xs[i] > l1[i])) << (8 * i);
                w[j] = b;
              }
            }
            const int Rq = p.q_R[o];  // 64 or 128: a shift, not a division
            const int chq = Rq == 128 ? n0 >> 7 : n0 >> 6, cq = n0 - chq * Rq;
            const long long off = p.q_phases[o] == 4 ? ((long long)(chq * 4 + ph4) * p.q_pos[o] + P4) * Rq + cq
                                                     : ((long long)chq * p.q_pos[o] + P1) * Rq + cq;
            uint4* dst = reinterpret_cast<uint4*>(p.q[o] + off);
#pragma unroll
            for (int j = 0; j < CH / 16; ++j) dst[j] = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
          }
          continue;
        }
        if constexpr (MT >= 2) continue;  // MT > 1 kernels: integer epilogue only (host-checked)
        if constexpr (BN >= 128) {
          if (p.aout) {  // downsample: exact s16 accumulators (|acc| <= 2K < 2^15, host-checked)
            if (p.res16_cl) {
              int16_t* ob = p.aout + hbase + ch_off(n0, true);  // blocked: one 32-byte store per 16 channels
#pragma unroll
              for (int h = 0; h < CH / 16; ++h) {
                uint32_t w[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) w[i] = (r[16 * h + 2 * i] & 0xFFFFu) | (r[16 * h + 2 * i + 1] << 16);
                sm100::st_v8(ob + h * bstride, w);
              }
            } else {
              int16_t* ob = p.aout + fbase + (long long)n0 * oplane;
#pragma unroll
              for (int j = 0; j < CH; ++j, ob += ostride) *ob = (int16_t)(int32_t)r[j];
            }
            continue;
          }
        }
        const float4* eg = reinterpret_cast<const float4*>(ep + n0);
        const int n4 = p.N / 4;
        float v[CH];
        if (p.out_scale == 1.0f) {  // fmul(1, x) == x exactly: one FMA per value
#pragma unroll
          for (int j = 0; j < CH / 4; ++j) {
            const float4 g = eg[j], bb = eg[n4 + j];
            const float gs[4] = {g.x, g.y, g.z, g.w}, bs[4] = {bb.x, bb.y, bb.z, bb.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)  // R:linalg.hpp:322-323 (FMA-contracted like the reference build)
              v[4 * j + i] = __fmaf_rn(gs[i], (float)(int32_t)r[4 * j + i], bs[i]);
          }
        } else {
#pragma unroll
          for (int j = 0; j < CH / 4; ++j) {
            const float4 g = eg[j], bb = eg[n4 + j];
            const float gs[4] = {g.x, g.y, g.z, g.w}, bs[4] = {bb.x, bb.y, bb.z, bb.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
              v[4 * j + i] = __fmaf_rn(gs[i], __fmul_rn(p.out_scale, (float)(int32_t)r[4 * j + i]), bs[i]);
          }
        }
        if constexpr (BN < 128) {
          if (pre) {  // NCHW: lanes = consecutive positions -> coalesced per channel
#pragma unroll
            for (int j = 0; j < CH; ++j) v[j] += sk[j];
            if (c0 + CH < BNG) {
              if (p.skip_cl) {
#pragma unroll
                for (int h = 0; h < CH / 8; ++h) {
                  uint32_t w[8];
                  sm100::ld_nc_v8(p.skip + skb + ch_off(c0 + CH, true) + (h >> 1) * bstride + 8 * (h & 1), w);
#pragma unroll
                  for (int i = 0; i < 8; ++i) sk[8 * h + i] = __uint_as_float(w[i]);
                }
              } else {
                // pointer increments: one IMAD.WIDE per element (no 64-bit index math)
                const float* sb = p.skip + skb + (size_t)(c0 + CH) * ostride;
#pragma unroll
                for (int j = 0; j < CH; ++j, sb += ostride) sk[j] = __ldg(sb);
              }
            }
          }
        } else if (pre) {  // NCHW: lanes = consecutive positions -> coalesced per channel
          if (p.skip16) {
            // the downsample conv's own epilogue, R:linalg.hpp:322-323 (fmul(1, x) == x)
            const float4* sg = reinterpret_cast<const float4*>(ep + 2 * p.N + n0);
#pragma unroll
            for (int j = 0; j < CH / 4; ++j) {
              const float4 g = sg[j], bb = sg[n4 + j];
              const float gs[4] = {g.x, g.y, g.z, g.w}, bs[4] = {bb.x, bb.y, bb.z, bb.w};
#pragma unroll
              for (int i = 0; i < 4; ++i)
                v[4 * j + i] += __fmaf_rn(gs[i], __fmul_rn(p.sk_scale, (float)(int32_t)skr[4 * j + i]), bs[i]);
            }
          } else {
#pragma unroll
            for (int j = 0; j < CH; ++j) v[j] += __uint_as_float(skr[j]);
          }
          if (c0 + CH < BNG) {
            load_skip(skb + ch_off(c0 + CH, skip_cl), skr);
          } else {
            // last chunk: this group's next item's first chunk, one item ahead
            const int nxt = item + (IG / MT) * (int)gridDim.x;
            if (nxt < n_items) {
              const long long nb = skip_at(nxt);
              if (nb >= 0) {
                load_skip(nb, skr);
                skr_ready = true;
              }
            }
          }
        }
        if (p.relu) {
#pragma unroll
          for (int j = 0; j < CH; ++j) v[j] = v[j] < 0.0f ? 0.0f : v[j];  // std::max(v, 0.0f)
        }
        if (p.fout && !(TK_DBG(p.dbg) & 256)) {
          if (p.fout_cl) {  // blocked: two 32-byte stores per 16 channels
            float* ob = p.fout + hbase + ch_off(n0, true);
#pragma unroll
            for (int h = 0; h < CH / 8; ++h) {
              uint32_t w[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) w[i] = __float_as_uint(v[8 * h + i]);
              sm100::st_v8(ob + (h >> 1) * bstride + 8 * (h & 1), w);
            }
          } else {
            float* ob = p.fout + fbase + (long long)n0 * oplane;
#pragma unroll
            for (int j = 0; j < CH; ++j, ob += ostride) *ob = v[j];
          }
        }
        if (p.n_q > 0 && !(TK_DBG(p.dbg) & 128)) {
          // quantizer input checks (R:quantizer.hpp:37-41,53-55), once per
          // value: after the ReLU a value is >= 0 (or -0.0) unless it is NaN
          // or +inf, exactly the values for which v * 0 is NaN -- one FMA
          // per value folds the check, one compare per chunk reads it
          bool bad = false;
          if (p.relu) {
            float z = 0.0f;
#pragma unroll
            for (int j = 0; j < CH; ++j) z = __fmaf_rn(v[j], 0.0f, z);
            bad = z != z;
          } else {
#pragma unroll
            for (int j = 0; j < CH; ++j) bad |= !(v[j] >= 0.0f && v[j] <= 3.402823466e38f);
          }
          if (bad) tk_raise(p.err, (unsigned long long)qrow, TK_ERR_NONFINITE);
          uint32_t w[CH / 4];
#pragma unroll
          for (int o = 0; o < 2; ++o) {
            if (o >= p.n_q) break;
            if (o == 0 || !p.q_same) {
              const float t0 = p.t0[o], t1 = p.t1[o];
#pragma unroll
              for (int j = 0; j < CH / 4; ++j) {
                uint32_t b = 0;
#pragma unroll
                for (int i = 0; i < 4; ++i) {  // level byte = (x > t0) + (x > t1): predicated adds
                  const float x = v[4 * j + i];
                  if (x > t0) b += 1u << (8 * i);
                  if (x > t1) b += 1u << (8 * i);
                }
                w[j] = b;
              }
            }
            const int Rq = p.q_R[o];  // 64 or 128: a shift, not a division
            const int chq = Rq == 128 ? n0 >> 7 : n0 >> 6, cq = n0 - chq * Rq;
            const long long off = p.q_phases[o] == 4 ? ((long long)(chq * 4 + ph4) * p.q_pos[o] + P4) * Rq + cq
                                                     : ((long long)chq * p.q_pos[o] + P1) * Rq + cq;
            uint4* dst = reinterpret_cast<uint4*>(p.q[o] + off);
#pragma unroll
            for (int j = 0; j < CH / 16; ++j) dst[j] = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
          }
        }
      }
      sm100::tc_fence_before();
      sm100::mbar_arrive(&a_empty[acc]);
    }
    if (stamp && warp == 2 && lane == 0) g_stamps[blockIdx.x * 8 + 4] = gtime();
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) sm100::tmem_dealloc<kCols>(tmem);
  if (stamp && threadIdx.x == 0) g_stamps[blockIdx.x * 8 + 5] = gtime();
}

// ---------------------------------------------------------------------------
// input packing: NCHW f32 -> s8 level tensors (up to 2 variants).  One thread
// per (image, 16-channel group, position): 16 loads coalesced across the warp
// (consecutive positions), one 16-byte store per variant.
struct PackIn {
  const float* x;
  int N, C, H, W;
  int n_q;
  int8_t* q[2];
  float t0[2], t1[2];
  int q_phases[2], q_R[2];
  long long q_pos[2];
  int Hp, Wp, PH, PW;
  unsigned long long* err;
  // error positions: 0 = NCHW element order (network input); 1 = the
  // im2col evaluation order of conv2d_ternary (R:linalg.hpp:173-225) for a
  // kk x kk / stride ks / pad kpad conv with OH x OW outputs
  int ek, kk, ks, kpad, OH, OW;
};

// Error key of input element (n, c, y, x).  In im2col order it is
// row * K + lane of the element's FIRST use (its smallest output row, then
// the tap within that row), so the minimum over bad elements is the error
// the reference throws first; -1 when no patch reads the element.
__device__ __forceinline__ long long pack_err_key(const PackIn& p, int n, int c, int y, int x) {
  if (!p.ek) return (((long long)n * p.C + c) * p.H + y) * p.W + x;
  int oy = y + p.kpad - (p.kk - 1), ox = x + p.kpad - (p.kk - 1);
  oy = oy <= 0 ? 0 : (oy + p.ks - 1) / p.ks;
  ox = ox <= 0 ? 0 : (ox + p.ks - 1) / p.ks;
  const int ky = y + p.kpad - oy * p.ks, kx = x + p.kpad - ox * p.ks;
  if (ky < 0 || kx < 0 || oy >= p.OH || ox >= p.OW) return -1;
  const long long row = ((long long)n * p.OH + oy) * p.OW + ox;
  return row * (p.kk * p.kk * p.C) + (ky * p.kk + kx) * p.C + c;
}

__global__ void k_pack_input(const PackIn p) {
  sm100::pdl_launch_dependents();  // a PDL-launched conv may start its prologue
  const long long HW = (long long)p.H * p.W;
  const int groups = p.C / 16;
  const long long total = (long long)p.N * groups * HW;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long pix = i % HW;
    const long long t = i / HW;
    const int g = (int)(t % groups), n = (int)(t / groups);
    const int y = (int)(pix / p.W), xx = (int)(pix - (long long)y * p.W);
    const float* src = p.x + ((long long)n * p.C + g * 16) * HW + pix;
    float v[16];
    float z = 0.0f, mn = 0.0f;  // NaN / inf and negative checks, as in k_pack_input_rows
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      v[j] = __ldg(src + j * HW);
      z = __fmaf_rn(v[j], 0.0f, z);
      mn = fminf(mn, v[j]);
    }
    if (z != z || mn < 0.0f) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int e = tk_error_code(v[j], 1);
        if (e != TK_OK) {
          const long long key = pack_err_key(p, n, g * 16 + j, y, xx);
          if (key >= 0) tk_raise(p.err, (unsigned long long)key, e);
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
          if (xv > p.t0[o]) b += 1u << (8 * i2);
          if (xv > p.t1[o]) b += 1u << (8 * i2);
        }
        w[j] = b;
      }
      const int Rq = p.q_R[o];  // 64 or 128
      const int c0 = g * 16, chq = Rq == 128 ? c0 >> 7 : c0 >> 6, cq = c0 - chq * Rq;
      const long long off = p.q_phases[o] == 4 ? ((long long)(chq * 4 + ph4) * p.q_pos[o] + P4) * Rq + cq
                                               : ((long long)chq * p.q_pos[o] + P1) * Rq + cq;
      *reinterpret_cast<uint4*>(p.q[o] + off) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

// Same result, one thread per (image, position) walking all C channels:
// 32-bit index math (N*H*W < 2^31, host-checked), every 16-channel group's
// loads in flight together, and each variant's R-byte position row written
// whole by one thread (full 32-byte sectors instead of 16-byte pieces from
// four different warps).
__global__ void __launch_bounds__(256) k_pack_input_rows(const PackIn p) {
  sm100::pdl_launch_dependents();
  const int HW = p.H * p.W;
  const int total = p.N * HW;
  const int groups = p.C / 16;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int n = i / HW, pix = i - n * HW;
    const int y = pix / p.W, xx = pix - y * p.W;
    const int py = y + 1, px = xx + 1;
    const long long P1 = ((long long)n * p.Hp + py) * p.Wp + px;
    const long long P4 = ((long long)n * p.PH + (py >> 1)) * p.PW + (px >> 1);
    const int ph4 = (py & 1) * 2 + (px & 1);
#pragma unroll 4
    for (int g = 0; g < groups; ++g) {
      const float* src = p.x + ((long long)n * p.C + g * 16) * HW + pix;
      float v[16];
      // quantizer input checks (R:quantizer.hpp:37-41,53-55): v * 0 is NaN
      // exactly for NaN / +-inf, and the minimum is < 0 exactly when some
      // value is negative (-0.0 is not): two instructions per value
      float z = 0.0f, mn = 0.0f;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        v[j] = __ldg(src + (long long)j * HW);
        z = __fmaf_rn(v[j], 0.0f, z);
        mn = fminf(mn, v[j]);
      }
      if (z != z || mn < 0.0f) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int e = tk_error_code(v[j], 1);
          if (e != TK_OK) {
            const long long key = pack_err_key(p, n, g * 16 + j, y, xx);
            if (key >= 0) tk_raise(p.err, (unsigned long long)key, e);
          }
        }
      }
      for (int o = 0; o < p.n_q; ++o) {
        uint32_t w[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint32_t b = 0;
#pragma unroll
          for (int i2 = 0; i2 < 4; ++i2) {  // level byte = (x > t0) + (x > t1): predicated adds
            const float xv = v[4 * j + i2];
            if (xv > p.t0[o]) b += 1u << (8 * i2);
            if (xv > p.t1[o]) b += 1u << (8 * i2);
          }
          w[j] = b;
        }
        const int Rq = p.q_R[o];  // 64 or 128
        const int c0 = g * 16, chq = Rq == 128 ? c0 >> 7 : c0 >> 6, cq = c0 - chq * Rq;
        const long long off = p.q_phases[o] == 4 ? ((long long)(chq * 4 + ph4) * p.q_pos[o] + P4) * Rq + cq
                                                 : ((long long)chq * p.q_pos[o] + P1) * Rq + cq;
        *reinterpret_cast<uint4*>(p.q[o] + off) = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
  }
}

// generic path helpers (NCHW)
__global__ void k_residual_relu(float* __restrict__ z, const float* __restrict__ sc, long long n, int relu_only) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const float v = relu_only ? z[i] : z[i] + sc[i];
    z[i] = v < 0.0f ? 0.0f : v;  // std::max(v, 0.0f)
  }
}

// spatial mean -> [N][C] (head input; left-to-right float sum)
// ---------------------------------------------------------------------------
#ifdef TK_PROFILE
// (profiling build only: the fp32 SIMT stem the split-TF32 tensor-core kernel
// of tk_stem.cu replaced, kept for the A/B in tools/stem_ab.py)
// stem convolution (float, outside the ternary path): 7x7 / stride 2 / pad 3,
// 3 -> 64 channels, fp32 FMA accumulation in the fixed order (ci, ky, kx).
// CTA = one image, kStemRows output rows x the full width; 512 threads =
// 8 channel groups (8 channels) x 64 pixel groups (7 columns, 16 apart, of
// one row), 56 accumulators per thread (four warps per scheduler keep the
// FMA pipe fed; FFMA2 occupies it for two cycles, so it halves issue slots,
// not pipe time).  Input band and weights in SMEM; per tap 2 x LDS.128
// (weights, broadcast) + 7 LDS (inputs) feed 56 FMA.
constexpr int kStemRows = 4, kStemCols = 112, kStemPx = 7;
constexpr int kStemInRows = 2 * kStemRows + 5, kStemInCols = 2 * kStemCols + 6;
// the input band is stored as even / odd column planes (stride-2 taps read
// consecutive words); the two output rows a warp computes read input rows
// 2 apart, i.e. 4 plane pitches: pitch 116 (4 mod 8) puts them 16 banks
// apart, so the 32 lanes' input loads are conflict-free
constexpr int kStemHalf = kStemInCols / 2, kStemPitch = 116;
static_assert(kStemPitch >= kStemHalf && (4 * kStemPitch) % 32 == 16, "stem band pitch");

// Persistent: one CTA per SM loads the weights once and walks (image, row
// tile) items; the next item's input band streams in with cp.async (zero
// fill outside the image) while the current one is computed.
__device__ __forceinline__ void stem_fill_band(float* band, const float* __restrict__ img, int n, int oy0, int H,
                                               int W) {
  for (int i = threadIdx.x; i < 3 * kStemInRows * kStemInCols; i += blockDim.x) {
    const int ci = i / (kStemInRows * kStemInCols);
    const int r = (i / kStemInCols) % kStemInRows, c = i % kStemInCols;
    const int y = 2 * oy0 - 3 + r, x = c - 3;
    const bool in = y >= 0 && y < H && x >= 0 && x < W;
    const float* src = in ? img + ((size_t)(n * 3 + ci) * H + y) * W + x : img;
    const uint32_t dst = sm100::smem_u32(band + ((ci * kStemInRows + r) * 2 + (c & 1)) * kStemPitch + (c >> 1));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(in ? 4 : 0) : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// CPT channels per thread (8: 512 threads, 16: 256 threads); PAIR: packed
// fp32x2 FMA (FFMA2) on channel pairs, else scalar FFMA -- every lane of
// either form is one round-to-nearest fp32 FMA in the same (ci, ky, kx) order
template <int CPT, bool PAIR>
__global__ void __launch_bounds__(64 * 64 / CPT, 1)
k_stem_conv(const float* __restrict__ img, const float* __restrict__ wgt, int N, int H, int W, int Ho, int Wo,
            float* __restrict__ out) {
  constexpr int kThr = 64 * 64 / CPT;
  extern __shared__ __align__(16) float s_stem[];
  float* s_w = s_stem;                                     // [tap][cout]
  constexpr int kBand = 3 * kStemInRows * 2 * kStemPitch;  // [ci][row][parity][kStemPitch]
  float* s_band[2] = {s_stem + 147 * 64, s_stem + 147 * 64 + kBand};
  for (int i = threadIdx.x; i < 147 * 64; i += kThr) {
    const int co = i / 147, tap = i - co * 147;  // weights [cout][ci][ky][kx]
    s_w[tap * 64 + co] = __ldg(wgt + i);
  }
  const int tiles = (Ho + kStemRows - 1) / kStemRows, n_items = N * tiles;
  int item = blockIdx.x;
  if (item < n_items) stem_fill_band(s_band[0], img, item / tiles, (item % tiles) * kStemRows, H, W);
  const int cg = threadIdx.x >> 6;      // channel group of CPT (warp-uniform)
  const int pg = threadIdx.x & 63;
  const int row = pg >> 4, c0 = pg & 15;  // output columns c0, c0+16, ..., c0+96
  for (int buf = 0; item < n_items; item += gridDim.x, buf ^= 1) {
    const int nxt = item + gridDim.x;
    if (nxt < n_items) {
      stem_fill_band(s_band[buf ^ 1], img, nxt / tiles, (nxt % tiles) * kStemRows, H, W);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const float* s_in = s_band[buf];
    float acc[CPT][kStemPx];
#pragma unroll
    for (int c = 0; c < CPT; ++c)
#pragma unroll
      for (int j = 0; j < kStemPx; ++j) acc[c][j] = 0.0f;
#pragma unroll 1
    for (int ci = 0; ci < 3; ++ci)
#pragma unroll
      for (int ky = 0; ky < 7; ++ky) {
        const float* in_row = s_in + (ci * kStemInRows + 2 * row + ky) * 2 * kStemPitch;
#pragma unroll
        for (int kx = 0; kx < 7; ++kx) {
          const float4* w4 = reinterpret_cast<const float4*>(s_w + ((ci * 7 + ky) * 7 + kx) * 64 + cg * CPT);
          float wv[CPT];
#pragma unroll
          for (int q = 0; q < CPT / 4; ++q) {
            const float4 t = w4[q];
            wv[4 * q] = t.x; wv[4 * q + 1] = t.y; wv[4 * q + 2] = t.z; wv[4 * q + 3] = t.w;
          }
          // input column 2*oc + kx (band coordinates) = plane kx&1, word oc + kx/2
          const float* pl = in_row + (kx & 1) * kStemPitch + (kx >> 1) + c0;
          float xv[kStemPx];
#pragma unroll
          for (int j = 0; j < kStemPx; ++j) xv[j] = pl[16 * j];
          if constexpr (PAIR) {
#pragma unroll
            for (int c = 0; c < CPT; c += 2)
#pragma unroll
              for (int j = 0; j < kStemPx; ++j) {
                unsigned long long a, w, x;
                asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(acc[c][j]), "f"(acc[c + 1][j]));
                asm("mov.b64 %0, {%1, %2};" : "=l"(w) : "f"(wv[c]), "f"(wv[c + 1]));
                asm("mov.b64 %0, {%1, %1};" : "=l"(x) : "f"(xv[j]));
                asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a) : "l"(w), "l"(x));
                asm("mov.b64 {%0, %1}, %2;" : "=f"(acc[c][j]), "=f"(acc[c + 1][j]) : "l"(a));
              }
          } else {
#pragma unroll
            for (int c = 0; c < CPT; ++c)
#pragma unroll
              for (int j = 0; j < kStemPx; ++j) acc[c][j] = __fmaf_rn(wv[c], xv[j], acc[c][j]);
          }
        }
      }
    const int n = item / tiles, oy = (item % tiles) * kStemRows + row;
    if (oy < Ho) {
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        float* o = out + ((size_t)(n * 64 + cg * CPT + c) * Ho + oy) * Wo;
#pragma unroll
        for (int j = 0; j < kStemPx; ++j)
          if (c0 + 16 * j < Wo) o[c0 + 16 * j] = acc[c][j];
      }
    }
    __syncthreads();  // everyone is done with this band before it is refilled
  }
}
#endif  // TK_PROFILE

// stem: out = maxpool3x3/2 pad 1 (relu(fmaf(g, x, b))); thread per output
__global__ void k_affine_relu_maxpool(const float* __restrict__ x, int C, int H, int W, int Ho, int Wo,
                                      const float* __restrict__ gain, const float* __restrict__ bias,
                                      long long total, float* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int ox = (int)(i % Wo);
    const long long r = i / Wo;
    const int oy = (int)(r % Ho);
    const long long nc = r / Ho;
    const int c = (int)(nc % C);
    const float g = __ldg(gain + c), b = __ldg(bias + c);
    const float* src = x + nc * H * W;
    float m = 0.0f;  // relu output >= 0, so 0 is the identity of the max
    for (int dy = -1; dy <= 1; ++dy) {
      const int y = 2 * oy + dy;
      if (y < 0 || y >= H) continue;
#pragma unroll
      for (int dx = -1; dx <= 1; ++dx) {
        const int xx = 2 * ox + dx;
        if (xx < 0 || xx >= W) continue;
        const float v = __fmaf_rn(g, __ldg(src + (long long)y * W + xx), b);
        m = fmaxf(m, v);
      }
    }
    out[i] = m;
  }
}

// the same with 4 consecutive outputs per thread (W = 2 * Wo, Wo % 4 == 0):
// per input row two float4 loads + one scalar replace 12 scalar loads, and
// the outputs go out as one float4
__global__ void k_affine_relu_maxpool4(const float* __restrict__ x, int C, int H, int W, int Ho, int Wo,
                                       const float* __restrict__ gain, const float* __restrict__ bias,
                                       long long total4, float* __restrict__ out) {
  const int q = Wo / 4;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total4;
       i += (long long)gridDim.x * blockDim.x) {
    const int ox = (int)(i % q) * 4;
    const long long r = i / q;
    const int oy = (int)(r % Ho);
    const long long nc = r / Ho;
    const int c = (int)(nc % C);
    const float g = __ldg(gain + c), b = __ldg(bias + c);
    const float* src = x + nc * H * W;
    float m[4] = {0.0f, 0.0f, 0.0f, 0.0f};  // relu output >= 0: 0 is the identity of the max
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy) {
      const int y = 2 * oy + dy;
      if (y < 0 || y >= H) continue;
      const float* row = src + (long long)y * W + 2 * ox;
      const float4 a = __ldg(reinterpret_cast<const float4*>(row));
      const float4 bb = __ldg(reinterpret_cast<const float4*>(row) + 1);
      // columns 2ox-1 .. 2ox+7 (the left one absent at the image border)
      const float v[9] = {ox > 0 ? __fmaf_rn(g, __ldg(row - 1), b) : 0.0f,
                          __fmaf_rn(g, a.x, b),  __fmaf_rn(g, a.y, b),  __fmaf_rn(g, a.z, b),
                          __fmaf_rn(g, a.w, b),  __fmaf_rn(g, bb.x, b), __fmaf_rn(g, bb.y, b),
                          __fmaf_rn(g, bb.z, b), __fmaf_rn(g, bb.w, b)};
#pragma unroll
      for (int k = 0; k < 4; ++k)
        m[k] = fmaxf(m[k], fmaxf(fmaxf(v[2 * k], v[2 * k + 1]), v[2 * k + 2]));
    }
    reinterpret_cast<float4*>(out)[i] = make_float4(m[0], m[1], m[2], m[3]);
  }
}

// spatial mean -> [NC] (the head input), each plane summed left to right
// (the reference's order).  A block's planes (one per thread) are one
// contiguous range: staged through shared memory with coalesced loads, then
// each thread walks its own plane.
__global__ void __launch_bounds__(64) k_pool_nchw(const float* __restrict__ x, int NC, int HW,
                                                  float* __restrict__ out) {
  extern __shared__ float s_pool[];  // [blockDim.x][HW]
  const int p0 = blockIdx.x * blockDim.x;
  const int np = min((int)blockDim.x, NC - p0);
  const float* src = x + (long long)p0 * HW;
  for (int i = threadIdx.x; i < np * HW; i += blockDim.x) s_pool[i] = __ldg(src + i);
  __syncthreads();
  if ((int)threadIdx.x >= np) return;
  const float* row = s_pool + threadIdx.x * HW;
  float s = 0.0f;
  for (int j = 0; j < HW; ++j) s += row[j];
  out[p0 + threadIdx.x] = s / (float)HW;
}

// the same mean over a channel-blocked [N][C/16][HW][16] tensor: a thread
// per (n, c) sums its positions left to right (the reference's order); the
// 16 channels of a block are 64 contiguous bytes per position
__global__ void __launch_bounds__(256) k_pool_cb16(const float* __restrict__ x, int N, int HW, int C,
                                                   float* __restrict__ out) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= (long long)N * C) return;
  const long long n = i / C;
  const int c = (int)(i - n * C);
  const float* q = x + (n * C + (c & ~15)) * HW + (c & 15);
  float s = 0.0f;
  for (int j = 0; j < HW; ++j, q += 16) s += __ldg(q);
  out[i] = s / (float)HW;
}

// channel-blocked [N][C/16][HW][16] -> NCHW (the body output the caller asked for)
__global__ void __launch_bounds__(256) k_cb16_to_nchw(const float* __restrict__ x, int N, int HW, int C,
                                                      float* __restrict__ out) {
  const long long total = (long long)N * C * HW;
  for (long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x; o < total;
       o += (long long)gridDim.x * blockDim.x) {
    const long long n = o / ((long long)C * HW);
    const long long r = o - n * C * HW;
    const int c = (int)(r / HW), p = (int)(r - (long long)c * HW);
    out[o] = __ldg(x + (n * C + (c & ~15)) * HW + (long long)p * 16 + (c & 15));
  }
}

void pool_cb16(const float* x, int N, int HW, int C, float* out, cudaStream_t s) {
  const long long nc = (long long)N * C;
  k_pool_cb16<<<(unsigned)((nc + 255) / 256), 256, 0, s>>>(x, N, HW, C, out);
}

void pool_nchw(const float* x, int NC, int HW, float* out, cudaStream_t s) {
  // planes per block: up to 64, within 96 KB of staged floats
  const int planes = std::max(1, std::min(64, (96 * 1024) / (HW * 4)));
  const size_t smem = (size_t)planes * HW * 4;
  tk_smem_attr((const void*)k_pool_nchw, 96 * 1024 + 4096);
  k_pool_nchw<<<(NC + planes - 1) / planes, planes, smem, s>>>(x, NC, HW, out);
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
struct F32T {  // f32 NCHW tensor
  float* p = nullptr;
  int C = 0, H = 0, W = 0;
  long long elems = 0;
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
  int* d_ithr = nullptr;
  tk_layer* layer = nullptr;  // generic path
  // fused wiring
  int in_idx = -1;            // index into net->s8
  int skip_f = -1, out_f = -1;  // -2 = the forward's input tensor
  int q_idx[2] = {-1, -1};
  int relu = 0;
  bool is_down = false;  // the block's downsample (1x1 / stride) conv
  ConvK k{};
  CUtensorMap in_map{}, w_map{};
  int smem = 0;
  int grid = 0;
  int MT = 1;  // 128-row M tiles per work item
  int GPI = 1;  // epilogue groups sharing one item (column split, BN = 256 only)
};


// the downsample residual travels as exact s16 accumulators when they fit
// (|acc| <= 2 * in_c * k * k); env TK_NET_F32_RESIDUAL=1 keeps f32 (A/B)
bool s16_ok(const Conv& cv) { return 2 * cv.d.in_c * cv.d.k * cv.d.k < 32768; }
bool f32_residual_forced() {
  return tk_knob("TK_NET_F32_RESIDUAL", 0) != 0;
}

}  // namespace

struct tk_net {
  tk_context* ctx = nullptr;
  int fused = 0;
  int single = 0;  // one conv, no residual (conv2d_ternary plan, tk_fconv_run)
  int f32_cl = 1;  // internal f32 residual tensors channel-blocked [N][C/16][HW][16], not NCHW
  int batch = 0, in_c = 0, in_h = 0, in_w = 0;
  int out_c = 0, out_h = 0, out_w = 0;
  std::vector<tk_block_desc> blocks;
  std::vector<std::vector<Conv>> convs;  // fused: down first; generic: convs then down
  std::vector<S8T> s8;
  std::vector<F32T> f32;
  PackIn pack{};
  int final_f = -1;
  std::vector<float*> gbuf;  // generic path buffers
  // optional per-conv timing (tk_net_set_timing): events around each conv
  int timing = 0;
  std::vector<cudaEvent_t> ev;
  size_t gbuf_elems = 0;
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
      // channel chunks of R = 64 (C == 64) or 128, N tiles of 64 / 128 / 256
      if (!(d.in_c == 64 || d.in_c % 128 == 0) || !(d.out_c == 64 || d.out_c == 128 || d.out_c % 256 == 0))
        return false;
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
  int slot_of[4] = {0, 0, 0, 0};
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
  k.halo_rows = mx - mn;  // tap span; the halo size is set once MT is chosen
  k.in_phases = in.phases;
  k.in_pos = in.pos;
  k.chunks = in.C / in.R;
  // output grid = the input's (phase) plane grid
  k.PHg = in.PH;
  k.PWg = in.PW;
  k.Ho = conv_out(in.H, d);
  k.Wo = conv_out(in.W, d);
}

// bn: N tile width (0 = the default: the whole layer up to 256 channels)
int prepare_conv_weights(Conv& cv, int R, int bn) {
  const tk_conv_desc& d = cv.d;
  const int taps = d.k * d.k, chunks = d.in_c / R;
  cv.R = R;
  cv.chunks = chunks;
  cv.BN = bn ? bn : (d.out_c >= 256 ? 256 : d.out_c);  // 64, 128, 256
  if (const int bnmax = tk_knob("TK_CONV_BNMAX", 0)) cv.BN = std::min(cv.BN, std::max(64, bnmax));
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

// The exact float epilogue of an inner conv, as the kernel (and the
// reference build) computes it: max(fma(g, s*acc, b), 0).
float epi_value(float g, float s, float b, int acc) {
  volatile float prod = s * (float)acc;  // rounded product, no contraction
  return fmaf(g, prod, b);
}

// Integer thresholds reproducing (relu(v(acc)) > t) for t >= 0 exactly:
// bit = (sign*acc > c).  v is monotone in acc (direction = sign of g*s).
void int_threshold(float g, float s, float b, float t, int kmax, int* c, int* sign) {
  const bool up = (g >= 0.0f) == (s >= 0.0f);
  auto pred = [&](int a) { return epi_value(g, s, b, a) > t; };
  if (up) {  // pred false..true: c = largest acc with !pred
    int lo = -kmax - 1, hi = kmax + 1;  // treat lo as !pred, hi as pred
    while (hi - lo > 1) {
      const int mid = lo + (hi - lo) / 2;
      if (pred(mid)) hi = mid; else lo = mid;
    }
    *c = lo;
    *sign = 1;
  } else {  // pred true..false: bit = acc < B, B = smallest acc with !pred
    int lo = -kmax - 1, hi = kmax + 1;  // lo as pred, hi as !pred
    while (hi - lo > 1) {
      const int mid = lo + (hi - lo) / 2;
      if (pred(mid)) lo = mid; else hi = mid;
    }
    *c = -hi;
    *sign = -1;
  }
}

int want_s8(tk_net* net, int C, int H, int W, int phases, float ta1, float ta2) {
  net->s8.push_back(make_s8(net->batch, C, H, W, phases, ta1, ta2));
  return (int)net->s8.size() - 1;
}

int want_f32(tk_net* net, int C, int H, int W) {
  F32T f;
  f.C = C; f.H = H; f.W = W;
  f.elems = (long long)net->batch * C * H * W;
  net->f32.push_back(f);
  return (int)net->f32.size() - 1;
}

int finish_fused(tk_net* net, int pack_a, int pack_b);

int setup_fused(tk_net* net) {
  int H = net->in_h, W = net->in_w, C = net->in_c;
  const int nb = (int)net->blocks.size();
  struct In { int idx_conv1, idx_down, f; };
  std::vector<In> bin(nb);
  auto phases_of = [](const tk_conv_desc& d) { return d.stride == 2 ? 4 : 1; };
  // block inputs: s8 variants for conv1 / down, f32 for identity shortcuts
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
    bin[b].f = bd.has_down ? -1 : (b == 0 ? -2 : want_f32(net, C, H, W));
    int h = H, w = W;
    for (int i = 0; i < bd.n_convs; ++i) { h = conv_out(h, bd.conv[i]); w = conv_out(w, bd.conv[i]); }
    H = h; W = w; C = bd.conv[bd.n_convs - 1].out_c;
  }
  net->out_c = C; net->out_h = H; net->out_w = W;
  net->final_f = want_f32(net, C, H, W);
  // convs (the downsample first: its f32 output is the block's residual)
  H = net->in_h; W = net->in_w; C = net->in_c;
  net->convs.assign(nb, {});
  for (int b = 0; b < nb; ++b) {
    const tk_block_desc& bd = net->blocks[b];
    auto& cvs = net->convs[b];
    int cur = bin[b].idx_conv1;
    int h = H, w = W, c = C;
    int sc_f = bin[b].f;
    if (bd.has_down) {
      Conv dv;
      dv.d = bd.down;
      dv.in_idx = bin[b].idx_down;
      dv.out_f = want_f32(net, bd.down.out_c, conv_out(H, bd.down), conv_out(W, bd.down));
      dv.is_down = true;
      sc_f = dv.out_f;
      cvs.push_back(dv);
    }
    for (int i = 0; i < bd.n_convs; ++i) {
      const tk_conv_desc& d = bd.conv[i];
      Conv cv;
      cv.d = d;
      cv.in_idx = cur;
      const int ho = conv_out(h, d), wo = conv_out(w, d);
      cv.relu = 1;
      if (i + 1 < bd.n_convs) {
        const tk_conv_desc& nx = bd.conv[i + 1];
        cv.q_idx[0] = want_s8(net, d.out_c, ho, wo, phases_of(nx), nx.ta1, nx.ta2);
        cur = cv.q_idx[0];
      } else {
        cv.skip_f = sc_f;
        if (b + 1 < nb) {
          cv.q_idx[0] = bin[b + 1].idx_conv1;
          if (bin[b + 1].idx_down >= 0 && bin[b + 1].idx_down != bin[b + 1].idx_conv1)
            cv.q_idx[1] = bin[b + 1].idx_down;
          cv.out_f = bin[b + 1].f;  // identity shortcut of the next block (or -1)
        } else {
          cv.out_f = net->final_f;
        }
      }
      cvs.push_back(cv);
      h = ho; w = wo; c = d.out_c;
    }
    H = h; W = w; C = c;
  }
  return finish_fused(net, bin[0].idx_conv1, bin[0].idx_down != bin[0].idx_conv1 ? bin[0].idx_down : -1);
}

// Allocation, per-conv kernel parameters and the input packing of a wired
// fused plan (net->convs); pack_a / pack_b: the s8 tensors the input is
// quantized into (pack_b may be -1).
int finish_fused(tk_net* net, int pack_a, int pack_b) {
  net->f32_cl = tk_knob("TK_NET_F32_NCHW", 0) ? 0 : 1;
  // allocate tensors
  for (auto& t : net->s8) {
    if (cudaMalloc(&t.p, t.bytes()) != cudaSuccess) return TK_ERR_CUDA;
    cudaMemset(t.p, 0, t.bytes());  // pad ring = code of quantize(0.0) = level 0
  }
  for (auto& f : net->f32)
    if (cudaMalloc(&f.p, (size_t)f.elems * 4) != cudaSuccess) return TK_ERR_CUDA;
  // per-conv kernel parameters
  int conv_no = -1;
  for (auto& cvs : net->convs)
    for (auto& cv : cvs) {
      ++conv_no;
      const S8T& in = net->s8[cv.in_idx];
      // integer-threshold (inner) convs: ReLU + quantize only, no floats out
      bool inner = cv.relu && cv.skip_f == -1 && cv.out_f < 0 && cv.q_idx[0] >= 0;
      if (inner) {
        tk_qparams q0;
        const S8T& q = net->s8[cv.q_idx[0]];
        inner = tk_make_qparams(q.ta1, q.ta2, TK_MODE_ACTIVATION_NONNEG, &q0) == TK_OK && q0.t0 >= 0.0f;
      }
      // wide inner convs (>= 256 channels, weights streamed per item): 128-wide
      // N tiles with two M tiles per item, so every streamed weight block
      // serves 256 positions (half the weight bytes per MAC of a 256-wide
      // single tile)
      // (measured, tools/layer_ab.py: also pays off for 128-channel stride-2
      // inner convs, not for 128-channel stride-1 ones)
      // (re-measured after the weight-ring change: the 3x3 stride-1 ones are
      // faster as 256-wide single tiles again -- ResNet-18 body -1.2%,
      // ResNet-50 b1024 -0.2%; bits: 1 all stride-1 wide, 4 stride-1 1x1
      // only, 2 stride-2)
      const int wm = tk_knob("TK_CONV_WIDE_MT2", 6);
      const bool wide_mt2 = inner && ((wm & 1) && cv.d.out_c >= 256 && cv.d.stride == 1 ||
                                      (wm & 4) && cv.d.out_c >= 256 && cv.d.stride == 1 && cv.d.k == 1 ||
                                      (wm & 2) && cv.d.out_c >= 128 && cv.d.stride == 2);
      int st = prepare_conv_weights(cv, in.R, wide_mt2 ? 128 : 0);
      if (st != TK_OK) return st;
      plan_taps(cv, in);
      ConvK& k = cv.k;
      k.n_tiles = cv.n_tiles;
      k.m_total = (long long)net->batch * k.PHg * k.PWg;
      k.m_tiles = (int)((k.m_total + 127) / 128);
      if (k.m_total + 1024 > (1ll << 31)) return TK_ERR_UNSUPPORTED;  // 32-bit row indices
      // two M tiles per item (env TK_CONV_MT=1 forces one, experiments)
      // (measured: pays off for the 64-channel inner convs; the f32-epilogue
      // convs and wider layers run faster with the two epilogue groups on
      // alternate items)
      // (MT > 1 kernels carry the integer epilogue only)
      // (MT = 4 measured no faster than 2 on the ResNet-18 stage-1 convs)
      cv.MT = ((cv.BN == 64 || wide_mt2) && inner && k.m_tiles > 1) ? 2 : 1;
      if (const int mt = tk_knob("TK_CONV_MT", 0)) cv.MT = std::min(cv.MT, std::max(1, mt));
      k.m_items = (k.m_tiles + cv.MT - 1) / cv.MT;
      {
        const int span = k.halo_rows;
        const int rows = (cv.MT * 128 + span + 7) / 8 * 8;
        k.nbox = (rows + 255) / 256;
        // box starts stay 1024-byte aligned in SMEM (the swizzle atom period)
        const int align = 1024 / cv.R;
        k.hbox = ((rows + k.nbox - 1) / k.nbox + align - 1) / align * align;
        if (k.hbox > 256) { ++k.nbox; k.hbox = ((rows + k.nbox - 1) / k.nbox + align - 1) / align * align; }
        k.halo_rows = k.nbox * k.hbox;
      }
      k.HB = (k.halo_rows * cv.R + 1023) / 1024 * 1024;
      k.WB = (cv.BN * cv.R + 1023) / 1024 * 1024;
      const int budget = 224 * 1024 - 6 * cv.d.out_c * 4 - 1536;  // of 227 KB dynamic SMEM
      const int halo_stage = k.n_ph * k.HB;
      const int wbytes_all = cv.chunks * k.n_taps * k.WB;
      k.resident = (cv.n_tiles == 1 && 2 * halo_stage + wbytes_all <= budget) ? 1 : 0;
      const int wmin = k.resident ? wbytes_all : 3 * k.WB;
      // halo ring depth: enough stages in flight to cover the TMA latency
      // (4: ResNet-50 b1024 -1% vs 8, ResNet-18 unchanged; env TK_CONV_HS
      // caps it for experiments)
      const int hs_cap = std::max(1, tk_knob("TK_CONV_HS", 4));
      k.hs = std::max(1, std::min(hs_cap, (budget - wmin) / halo_stage));
      // streamed 3x3 weights (9 blocks per halo stage) are the bytes that
      // bound the late stages: the TMA latency times the ring depth caps the
      // stream, so keep >= 5 weight stages and only 2 halo stages there
      // (tools/layer_ab.py, ResNet-18 b256: stage-3/4 convs -4..-8%)
      if (!k.resident && k.n_taps == 9 && tk_knob("TK_CONV_WDEEP", 1))
        k.hs = std::max(1, std::min(k.hs, std::max(2, (budget - 5 * k.WB) / halo_stage)));
      k.ws = k.resident ? 1 : std::max(2, std::min(8, (budget - k.hs * halo_stage) / k.WB));
      const int wregion = k.resident ? wbytes_all : k.ws * k.WB;
      // epilogue parameter words: at most 2 quantized outputs x 3 ints per channel
      cv.smem = 1024 + k.hs * halo_stage + wregion + 6 * cv.d.out_c * 4 + 512;
      k.gain = cv.d_gain;
      k.bias = cv.d_bias;
      k.out_scale = cv.d.out_scale;
      k.relu = cv.relu;
      k.N = cv.d.out_c;
      k.o_Hp = k.Ho + 2; k.o_Wp = k.Wo + 2;
      k.o_PH = k.o_Hp / 2; k.o_PW = k.o_Wp / 2;
      k.skip = cv.skip_f >= 0 ? net->f32[cv.skip_f].p : nullptr;  // -2: patched at launch
      k.fout = cv.out_f >= 0 ? net->f32[cv.out_f].p : nullptr;
      // the network's own residual tensors are channel-last; x and a plan's
      // caller output (-2 / -3) are NCHW
      k.skip_cl = cv.skip_f >= 0 && net->f32_cl ? 1 : 0;
      k.fout_cl = cv.out_f >= 0 && net->f32_cl ? 1 : 0;
      // (measured, tools/layer_ab.py: the f32 residual channel-blocked is 4-10%
      // faster per body than NCHW; the s16 one is not -- its blocked stores
      // are faster in the downsample convs but its readers slower overall)
      k.res16_cl = tk_knob("TK_NET_S16_CB16", 0) ? 1 : 0;
      k.aout = nullptr;
      k.skip16 = nullptr;
      k.sk_gain = k.sk_bias = nullptr;
      k.sk_scale = 1.0f;
      // (the s16 residual path is compiled into the BN >= 128 kernels only)
      auto s16_pair = [&](const Conv& dv) {
        return !f32_residual_forced() && s16_ok(dv) && dv.d.out_c >= 128 && cvs.back().d.out_c >= 128 &&
               !tk_knob("TK_CONV_BNMAX", 0);
      };
      if (cv.is_down && s16_pair(cv)) {  // (its f32 tensor holds the s16 values)
        k.aout = reinterpret_cast<int16_t*>(k.fout);
        k.fout = nullptr;
      } else if (cv.skip_f >= 0) {
        for (auto& dv : cvs)
          if (dv.is_down && dv.out_f == cv.skip_f && s16_pair(dv)) {
            k.skip16 = reinterpret_cast<const int16_t*>(k.skip);
            k.skip = nullptr;
            k.sk_gain = dv.d_gain;
            k.sk_bias = dv.d_bias;
            k.sk_scale = dv.d.out_scale;
          }
      }
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
      k.q_same = k.n_q == 2 && k.t0[0] == k.t0[1] && k.t1[0] == k.t1[1];
      // column split for the wide f32-epilogue convs (measured, tools/layer_ab.py:
      // -6..-19% on the skip + f32-output layers, but slower for the s16
      // downsample output and for two next-layer quantizers)
      cv.GPI = (cv.BN == 256 && cv.MT == 1 && !k.aout && k.n_q < 2 && tk_knob("TK_CONV_GPI", 1)) ? 2 : 1;
      // integer-threshold epilogue for inner convs (ReLU + quantize only)
      k.ithr = nullptr;
      k.ithr16 = 0;
      if (cv.relu && cv.skip_f == -1 && cv.out_f < 0 && k.n_q > 0 && k.t0[0] >= 0.0f) {
        const int N = cv.d.out_c, kmax = 2 * cv.d.in_c * cv.d.k * cv.d.k;
        std::vector<int> thr((size_t)k.n_q * 3 * N);
        std::vector<float> g(N, 1.0f), b(N, 0.0f);
        if (cv.d.gain_host) memcpy(g.data(), cv.d.gain_host, N * 4);
        if (cv.d.bias_host) memcpy(b.data(), cv.d.bias_host, N * 4);
        for (int o = 0; o < k.n_q; ++o)
          for (int n = 0; n < N; ++n) {
            int c0, s0, c1, s1;
            int_threshold(g[n], cv.d.out_scale, b[n], k.t0[o], kmax, &c0, &s0);
            int_threshold(g[n], cv.d.out_scale, b[n], k.t1[o], kmax, &c1, &s1);
            thr[((size_t)o * 3 + 0) * N + n] = c0;
            thr[((size_t)o * 3 + 1) * N + n] = c1;
            thr[((size_t)o * 3 + 2) * N + n] = s0;  // s0 == s1 (same direction)
          }
        // compact form when every direction is +1 and the thresholds fit s16
        bool pack16 = true;
        for (int o = 0; o < k.n_q && pack16; ++o)
          for (int n = 0; n < N && pack16; ++n) {
            const int c0 = thr[((size_t)o * 3 + 0) * N + n], c1 = thr[((size_t)o * 3 + 1) * N + n];
            pack16 = thr[((size_t)o * 3 + 2) * N + n] == 1 && c0 >= -32768 && c0 <= 32767 && c1 >= -32768 &&
                     c1 <= 32767;
          }
        if (tk_knob("TK_CONV_NOPACK16", 0)) pack16 = false;
        // DPX form: level pairs by two s16x2 add-min-relu ops (|acc - c| <= 2 kmax + 1 fits s16)
        const bool dpx = pack16 && 2 * kmax + 1 <= 32767 && tk_knob("TK_CONV_DPX", 1);
        k.ithr16 = pack16 ? (dpx ? 2 : 1) : 0;
        if (pack16) {
          std::vector<int> p16((size_t)k.n_q * N);
          auto h16 = [](int v) { return (uint32_t)v & 0xFFFFu; };
          for (int o = 0; o < k.n_q; ++o)
            for (int n = 0; n < N; ++n) {
              const int c0 = thr[((size_t)o * 3 + 0) * N + n], c1 = thr[((size_t)o * 3 + 1) * N + n];
              if (!dpx) {
                p16[(size_t)o * N + n] = (int)(h16(c0) | (h16(c1) << 16));
              } else {  // words of channels 4j..4j+3: (-c0 pair 01, -c1 pair 01, -c0 pair 23, -c1 pair 23)
                const int j = n & ~3, i = n & 3, word = j + (i >> 1) * 2, hi = i & 1;
                uint32_t* w = reinterpret_cast<uint32_t*>(p16.data() + (size_t)o * N);
                w[word] = (w[word] & (hi ? 0xFFFFu : 0xFFFF0000u)) | (h16(-c0) << (16 * hi));
                w[word + 1] = (w[word + 1] & (hi ? 0xFFFFu : 0xFFFF0000u)) | (h16(-c1) << (16 * hi));
              }
            }
          thr.swap(p16);
        }
        if (cudaMalloc(&cv.d_ithr, thr.size() * 4) != cudaSuccess) return TK_ERR_CUDA;
        cudaMemcpy(cv.d_ithr, thr.data(), thr.size() * 4, cudaMemcpyHostToDevice);
        k.ithr = cv.d_ithr;
      }
      if (cv.MT > 1 && !k.ithr) return TK_ERR_UNSUPPORTED;  // (inner predicate above mirrors this)
      k.err = net->ctx->d_err;
      k.dbg = tk_knob("TK_CONV_DBG", 0);
      // profiling: TK_CONV_DBG_ONLY=<launch order index> limits the knob to one conv
      if (tk_knob("TK_CONV_DBG_ONLY", -1) >= 0 && tk_knob("TK_CONV_DBG_ONLY", -1) != conv_no) k.dbg = 0;
      if (!map_rows(&cv.in_map, in.p, (unsigned long long)(in.C / in.R) * in.phases * in.pos, in.R, k.hbox))
        return TK_ERR_CUDA;
      const int items = k.m_items * k.n_tiles;
      cv.grid = std::min(items, net->ctx->num_sms);
      if (const int g = tk_knob("TK_CONV_GRID", 0)) cv.grid = std::min(items, g);
    }
  // input packing
  PackIn& pk = net->pack;
  pk.N = net->batch; pk.C = net->in_c; pk.H = net->in_h; pk.W = net->in_w;
  const S8T& s0 = net->s8[pack_a];
  pk.Hp = s0.Hp; pk.Wp = s0.Wp; pk.PH = s0.Hp / 2; pk.PW = s0.Wp / 2;
  pk.n_q = 0;
  int ids[2] = {pack_a, pack_b};
  for (int id : ids) {
    if (id < 0) continue;
    const S8T& q = net->s8[id];
    tk_qparams qp;
    if (tk_make_qparams(q.ta1, q.ta2, TK_MODE_ACTIVATION_NONNEG, &qp) != TK_OK) return TK_ERR_THRESHOLDS;
    pk.q[pk.n_q] = q.p; pk.t0[pk.n_q] = qp.t0; pk.t1[pk.n_q] = qp.t1;
    pk.q_phases[pk.n_q] = q.phases; pk.q_R[pk.n_q] = q.R; pk.q_pos[pk.n_q] = q.pos;
    ++pk.n_q;
  }
  pk.err = net->ctx->d_err;
  return TK_OK;
}

template <int BN, int R, int KT, int MT, int GPI = 1>
cudaError_t launch_conv(const Conv& cv, const float* x, float* out, int pdl, cudaStream_t s) {
  // 227 KB per block, less the kernel's static shared tables
  if (const cudaError_t e = tk_smem_attr((const void*)k_conv_tc<BN, R, KT, MT, GPI>, 226 * 1024); e != cudaSuccess)
    return e;
  ConvK k = cv.k;
  if (cv.skip_f == -2) k.skip = x;  // identity shortcut = the forward's input
  if (cv.out_f == -3) k.fout = out;  // the caller's output (conv2d_ternary plans)
  // programmatic dependent launch: the prologue (TMEM, barriers, resident
  // weights) may overlap the previous kernel's tail.  Inside the network only
  // for batches <= 128 (tools/body_batch.py, ResNet-18 body: b32 -11%, b64
  // -9%, b128 -6%, b256 -1.5%; ResNet-50 b128 -2%, b256 +1.6%, b512 +3.5%):
  // small layers leave SMs idle in their tails, large ones do not; on for
  // conv2d_ternary plans, behind the input packing.
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cv.grid);
  cfg.blockDim = dim3(conv_threads(BN, MT, GPI));
  cfg.dynamicSmemBytes = cv.smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_conv_tc<BN, R, KT, MT, GPI>, cv.in_map, cv.w_map, k);
}

template <int BN, int R, int KT>
cudaError_t launch_conv_mt(const Conv& cv, const float* x, float* out, int pdl, cudaStream_t s) {
  if constexpr (BN == 64) {
    if (cv.MT == 4) return launch_conv<BN, R, KT, 4>(cv, x, out, pdl, s);
    if (cv.MT == 2) return launch_conv<BN, R, KT, 2>(cv, x, out, pdl, s);
  }
  if constexpr (BN == 128) {
    if (cv.MT == 2) return launch_conv<BN, R, KT, 2>(cv, x, out, pdl, s);
  }
  if constexpr (BN == 256) {
    if (cv.GPI == 2) return launch_conv<BN, R, KT, 1, 2>(cv, x, out, pdl, s);
  }
  return launch_conv<BN, R, KT, 1>(cv, x, out, pdl, s);
}

template <int KT>
cudaError_t run_conv_kt(const Conv& cv, const float* x, float* out, int pdl, cudaStream_t s) {
  if (cv.R == 64) {
    if (cv.BN == 64) return launch_conv_mt<64, 64, KT>(cv, x, out, pdl, s);
    if (cv.BN == 128) return launch_conv_mt<128, 64, KT>(cv, x, out, pdl, s);
    return launch_conv_mt<256, 64, KT>(cv, x, out, pdl, s);
  }
  if (cv.BN == 64) return launch_conv_mt<64, 128, KT>(cv, x, out, pdl, s);
  if (cv.BN == 128) return launch_conv_mt<128, 128, KT>(cv, x, out, pdl, s);
  return launch_conv_mt<256, 128, KT>(cv, x, out, pdl, s);
}

// x: the forward's input (identity shortcut of the first block); out: the
// caller's output buffer of a conv2d_ternary plan (out_f == -3)
cudaError_t run_conv(const Conv& cv, const float* x, float* out, int pdl, cudaStream_t s) {
  return cv.k.n_taps == 9 ? run_conv_kt<9>(cv, x, out, pdl, s) : run_conv_kt<1>(cv, x, out, pdl, s);
}

// input packing: a thread per position walking all channels for large
// inputs (whole R-byte rows per thread); a thread per (position, 16-channel
// group) when the input is too small to fill the SMs that way
cudaError_t launch_pack(PackIn pk, const float* x, cudaStream_t s) {
  pk.x = x;
  const long long rows = (long long)pk.N * pk.H * pk.W;
  if (rows < (1ll << 31) && rows >= 148ll * 256 * 2) {
    k_pack_input_rows<<<(unsigned)std::min<long long>((rows + 255) / 256, 148 * 16), 256, 0, s>>>(pk);
  } else {
    const long long total = rows * (pk.C / 16);
    k_pack_input<<<(unsigned)std::min<long long>((total + 255) / 256, 148 * 64), 256, 0, s>>>(pk);
  }
  return cudaGetLastError();
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
  TK_ON_DEVICE(ctx);
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

int tk_affine_relu_maxpool(tk_context* ctx, const float* x, int n, int c, int h, int w, const float* gain,
                           const float* bias, float* out, void* stream) {
  TK_ON_DEVICE(ctx);
  if (!ctx || !x || !gain || !bias || !out || n < 0 || c <= 0 || h <= 0 || w <= 0) return TK_ERR_INVALID;
  const int ho = (h + 1) / 2, wo = (w + 1) / 2;
  const long long total = (long long)n * c * ho * wo;
  if (total == 0) return TK_OK;
  if (w == 2 * wo && wo % 4 == 0 && h == 2 * ho && (uintptr_t)x % 16 == 0 && (uintptr_t)out % 16 == 0) {
    const long long total4 = total / 4;
    const unsigned grid = (unsigned)std::min<long long>((total4 + 255) / 256, 148ll * 32);
    k_affine_relu_maxpool4<<<grid, 256, 0, (cudaStream_t)stream>>>(x, c, h, w, ho, wo, gain, bias, total4, out);
    return cudaGetLastError() == cudaSuccess ? TK_OK : TK_ERR_CUDA;
  }
  const unsigned grid = (unsigned)std::min<long long>((total + 255) / 256, 148ll * 64);
  k_affine_relu_maxpool<<<grid, 256, 0, (cudaStream_t)stream>>>(x, c, h, w, ho, wo, gain, bias, total, out);
  return cudaGetLastError() == cudaSuccess ? TK_OK : TK_ERR_CUDA;
}

int tk_stem_conv7x7s2(tk_context* ctx, const float* images, int n, int h, int w, const float* weights,
                      float* out, void* stream) {
  TK_ON_DEVICE(ctx);
  if (!ctx || !images || !weights || !out || n < 0 || h <= 0 || w <= 0) return TK_ERR_INVALID;
  if (n == 0) return TK_OK;
#ifdef TK_PROFILE
  // the fp32 SIMT kernel the tensor-core stem replaced, for A/B (tools/stem_ab.py)
  if (tk_knob("TK_STEM_SIMT", 0)) {
    const int ho = (h + 6 - 7) / 2 + 1, wo = (w + 6 - 7) / 2 + 1;
    if (wo > kStemCols || (w + 6) > kStemInCols) return TK_ERR_UNSUPPORTED;  // one CTA spans the width
    const int smem = (147 * 64 + 2 * 3 * kStemInRows * 2 * kStemPitch) * 4;
    if (tk_smem_attr((const void*)k_stem_conv<8, true>, smem) != cudaSuccess) return TK_ERR_CUDA;
    const int items = n * ((ho + kStemRows - 1) / kStemRows);
    k_stem_conv<8, true><<<std::min(items, ctx->num_sms), 512, smem, (cudaStream_t)stream>>>(images, weights, n, h,
                                                                                          w, ho, wo, out);
    return cudaGetLastError() == cudaSuccess ? TK_OK : TK_ERR_CUDA;
  }
#endif
  return tk_launch_stem_tc(ctx, images, n, h, w, weights, out, stream);
}

int tk_net_destroy(tk_net* net) {
  TK_ON_DEVICE(net ? net->ctx : nullptr);
  if (!net) return TK_OK;
  cudaDeviceSynchronize();
  for (auto& cvs : net->convs)
    for (auto& cv : cvs) {
      cudaFree(cv.d_w); cudaFree(cv.d_gain); cudaFree(cv.d_bias); cudaFree(cv.d_ithr);
      (void)0;
      if (cv.layer) tk_layer_destroy(cv.layer);
    }
  for (auto& t : net->s8) cudaFree(t.p);
  for (auto& f : net->f32) cudaFree(f.p);
  for (auto* p : net->gbuf) cudaFree(p);
  for (auto e : net->ev) cudaEventDestroy(e);
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

// diagnostics: per-CTA timestamps of the last conv launched with
// TK_CONV_DBG & 16 (148 x 8 u64, globaltimer ns)
int tk_debug_conv_stamps(unsigned long long* host_out) {
  return cudaMemcpyFromSymbol(host_out, g_stamps, sizeof(unsigned long long) * 148 * 8) == cudaSuccess &&
                 cudaMemcpyFromSymbol(host_out + 148 * 8, g_trace, sizeof(unsigned long long) * 8 * 32) ==
                     cudaSuccess
             ? TK_OK
             : TK_ERR_CUDA;
}

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

int tk_net_num_convs(const tk_net* net) {
  if (!net) return -1;
  int n = 0;
  for (const auto& cvs : net->convs) n += (int)cvs.size();
  return n;
}

// Per-conv device timing of subsequent forwards (fused path): events are
// recorded around every conv launch on the forward's stream.
int tk_net_set_timing(tk_net* net, int on) {
  if (!net) return TK_ERR_INVALID;
  if (on && net->ev.empty()) {
    net->ev.resize(2 * tk_net_num_convs(net));
    for (auto& e : net->ev)
      if (cudaEventCreate(&e) != cudaSuccess) return TK_ERR_CUDA;
  }
  net->timing = on && net->fused;
  return TK_OK;
}

// ms of each conv of the LAST timed forward (synchronises on its events);
// also fills MACs per conv (whole batch) when macs != NULL.
int tk_net_conv_times(tk_net* net, float* ms, double* macs) {
  if (!net || !net->timing) return TK_ERR_INVALID;
  int ci = 0;
  for (const auto& cvs : net->convs)
    for (const auto& cv : cvs) {
      if (ms) {
        if (cudaEventSynchronize(net->ev[2 * ci + 1]) != cudaSuccess) return TK_ERR_CUDA;
        cudaEventElapsedTime(&ms[ci], net->ev[2 * ci], net->ev[2 * ci + 1]);
      }
      if (macs)
        macs[ci] = (double)net->batch * cv.k.Ho * cv.k.Wo * cv.d.out_c * cv.d.in_c * cv.d.k * cv.d.k;
      ++ci;
    }
  return TK_OK;
}

int tk_net_forward(tk_context* ctx, tk_net* net, const float* x, float* out, float* pooled, void* stream) {
  TK_ON_DEVICE(ctx);
  if (!ctx || !net || !x) return TK_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  if (net->fused) {
    if (launch_pack(net->pack, x, s) != cudaSuccess) return TK_ERR_CUDA;
    int ci = 0;
    for (const auto& cvs : net->convs)
      for (const auto& cv : cvs) {
        if (net->timing) cudaEventRecord(net->ev[2 * ci], s);
        if (const cudaError_t ce = run_conv(cv, x, nullptr, tk_knob("TK_PDL", net->batch <= 128), s); ce != cudaSuccess) {
          if (tk_knob("TK_NET_DEBUG", 0)) fprintf(stderr, "tk_net_forward: conv %d: %s\n", ci, cudaGetErrorString(ce));
          return TK_ERR_CUDA;
        }
        if (net->timing) cudaEventRecord(net->ev[2 * ci + 1], s);
        ++ci;
      }
    const F32T& f = net->f32[net->final_f];
    if (out && net->f32_cl)
      k_cb16_to_nchw<<<(unsigned)std::min<long long>((f.elems + 255) / 256, 148 * 32), 256, 0, s>>>(
          f.p, net->batch, f.H * f.W, f.C, out);
    else if (out)
      cudaMemcpyAsync(out, f.p, (size_t)f.elems * 4, cudaMemcpyDeviceToDevice, s);
    if (pooled && net->f32_cl)
      pool_cb16(f.p, net->batch, f.H * f.W, f.C, pooled, s);
    else if (pooled)
      pool_nchw(f.p, net->batch * f.C, f.H * f.W, pooled, s);
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
    pool_nchw(cur, net->batch * net->out_c, H * W, pooled, s);
  return cudaGetLastError() == cudaSuccess ? TK_OK : TK_ERR_CUDA;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// conv2d_ternary plans (R:linalg.hpp:301-328) on the fused conv kernel: a
// one-conv plan without ReLU or residual whose f32 NCHW epilogue output is
// the caller's buffer.  The input packing quantizes with the layer's
// activation thresholds into the zero-padded channel-last plane (the pad ring
// is quantize(0.0) = level 0, exactly the reference's zero padding) and
// reports data errors in the reference's im2col evaluation order; the conv
// launches as a programmatic dependent of the packing, so its prologue
// (barriers, TMEM, resident weights) overlaps it.

namespace {

bool single_conv_ok(int C, int OC, int k, int stride, int pad, int h, int w) {
  if (!(C == 64 || C % 128 == 0) || !(OC == 64 || OC == 128 || OC % 256 == 0)) return false;
  if (!((k == 3 && pad == 1) || (k == 1 && pad == 0))) return false;
  if (stride != 1 && stride != 2) return false;
  if (stride == 2 && ((h % 2) || (w % 2))) return false;
  if (h < 8 || w < 8) return false;  // a padded plane holds (h+2)(w+2) rows for h*w outputs
  const int Wp = w + 2;
  const int span = stride == 1 ? (k == 3 ? 2 * Wp + 2 : 0) : (k == 3 ? Wp / 2 + 1 : 0);
  return 128 + span <= 256;  // one halo box per 128-position tile
}

int make_single(const tk_layer* L, int n, int h, int w, tk_net** out) {
  // int8 weights [out_c][K] in the reference lane order (ky*kw + kx)*in_c + c,
  // decoded from the packed rows (R:codec.hpp:38-40)
  std::vector<int8_t> wq((size_t)L->out_c * L->K);
  for (int o = 0; o < L->out_c; ++o)
    for (int l = 0; l < L->K; ++l) {
      const unsigned code = (unsigned)(L->h_words[(size_t)o * L->wpr64 + l / 32] >> (2 * (l % 32))) & 3u;
      wq[(size_t)o * L->K + l] = (int8_t)(code == 0 ? -1 : (code == 3 ? 1 : 0));
    }
  tk_conv_desc d{};
  d.in_c = L->in_c; d.out_c = L->out_c; d.k = L->kh; d.stride = L->stride; d.pad = L->pad;
  d.weights_host = wq.data();
  d.tw1 = L->tw1; d.tw2 = L->tw2; d.ta1 = L->ta1; d.ta2 = L->ta2;
  d.gain_host = L->h_gain; d.bias_host = L->h_bias;
  d.out_scale = L->out_scale;
  tk_net* net = new tk_net;
  net->ctx = L->ctx;
  net->batch = n; net->in_c = L->in_c; net->in_h = h; net->in_w = w;
  net->fused = 1;
  net->single = 1;
  const int a = want_s8(net, L->in_c, h, w, d.stride == 2 ? 4 : 1, d.ta1, d.ta2);
  net->out_c = d.out_c; net->out_h = conv_out(h, d); net->out_w = conv_out(w, d);
  Conv cv;
  cv.d = d;
  cv.in_idx = a;
  cv.relu = 0;     // conv2d_ternary: folded BN only
  cv.out_f = -3;   // the caller's output
  net->convs.assign(1, std::vector<Conv>{cv});
  int st = finish_fused(net, a, -1);
  if (st == TK_OK) {
    PackIn& pk = net->pack;
    pk.ek = 1; pk.kk = d.k; pk.ks = d.stride; pk.kpad = d.pad; pk.OH = net->out_h; pk.OW = net->out_w;
    if (cudaDeviceSynchronize() != cudaSuccess) st = TK_ERR_CUDA;
  }
  if (st != TK_OK) {
    tk_net_destroy(net);
    return st;
  }
  *out = net;
  return TK_OK;
}

}  // namespace

bool tk_fconv_eligible(const tk_layer* L, int n, int h, int w) {
  return L && L->nonneg && L->kh == L->kw && n > 0 && encode() != nullptr &&
         (long long)n * (h + 2) * (w + 2) + 1024 < (1ll << 31) &&
         single_conv_ok(L->in_c, L->out_c, L->kh, L->stride, L->pad, h, w);
}

int tk_fconv_run(const tk_layer* L, const float* x, int n, int h, int w, float* out, cudaStream_t s) {
  tk_net* net = nullptr;
  {
    std::lock_guard<std::mutex> lock(L->plan_mu);
    auto it = L->plans.find({n, h, w});
    if (it == L->plans.end()) {
      const int st = make_single(L, n, h, w, &net);
      if (st != TK_OK) return st;
      L->plans[{n, h, w}] = net;
    } else {
      net = it->second;
    }
  }
  if (launch_pack(net->pack, x, s) != cudaSuccess) return TK_ERR_CUDA;
  return run_conv(net->convs[0][0], x, out, 1, s) == cudaSuccess ? TK_OK : TK_ERR_CUDA;
}

void tk_fconv_destroy_plans(tk_layer* L) {
  std::lock_guard<std::mutex> lock(L->plan_mu);
  for (auto& kv : L->plans) tk_net_destroy(kv.second);
  L->plans.clear();
}

// tk_tc.cu -- the int8 tensor-core variant of the ternary contraction:
// tcgen05.mma kind::i8 with TMA-staged operands and the accumulator in TMEM.
//
// Operands are the quantization LEVELS as s8 (activations {0,1,2} with the
// nonneg offset folded in, or {-1,0,1}; weights {-1,0,1}), so the s32
// accumulator equals packed_gemm's offset-corrected result exactly
// (R:linalg.hpp:253-276) and the epilogue is the same folded-BN FMA.
//
// Work split: a 128 x BN output tile per CTA and, when the tiles alone do not
// fill the 148 SMs (cfg3: M=256, N=4096 -> 32 tiles of 128x256), the K range
// split S ways (S = 2, 4, 8) across the CTAs of one thread-block cluster.
// After the K loop every CTA pushes each accumulator row straight from TMEM
// into the shared memory of the CTA owning that row's slice (rows
// [r*128/S, (r+1)*128/S) belong to cluster rank r) with distributed-shared-
// memory stores; after a cluster barrier each CTA sums its S partial slices
// (integer sums: exact in any order), applies the epilogue and writes
// coalesced rows.
//
// CTA = 10 warps: warp 0 TMA producer, warp 1 TMEM owner + MMA issuer,
// warps 2-9 the epilogue (two per TMEM lane quarter, warp % 4); all warps
// run the cluster reduction.  Launched with programmatic dependent launch:
// the prologue and the first weight (B) stages overlap the producing kernel
// (quantize / expand), A loads and output stores wait for it
// (griddepcontrol.wait).
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "tk_internal.cuh"
#include "tk_sm100.cuh"

namespace {

constexpr int BM = 128, BK = 128;
// warp 0 TMA producer, warp 1 TMEM owner + MMA issuer, warps 2-9 epilogue:
// two warps per TMEM lane quarter (q = warp % 4), each taking half the columns
constexpr int kThreads = 320;

template <int BN>
struct TcSmem {
  // K blocks per stage: BN = 64 tiles take two per TMA box (3-D box over the
  // K-block-major planes): fewer, larger requests move more bytes per SM
  static constexpr int kKD = BN <= 128 ? 2 : 1;
  static constexpr int kA = kKD * BM * BK;  // bytes per stage
  static constexpr int kB = kKD * BN * BK;
  static constexpr int kStage = kA + kB;
  // as many stages as ~200 KB of shared memory holds (latency hiding)
  static constexpr int kStages = (200 * 1024 / kStage) > 8 ? 8 : (200 * 1024 / kStage);
  // split-K receive buffer, s16 [S][128/S][BN] = 128 x BN, aliasing the ring
  // (+ the f32 staging boxes of the reduced slice, <= 64 x BN x 4 bytes)
  static constexpr int kRecv = BM * BN * 2 + 64 * BN * 4;
  static constexpr int kRing = kStages * kStage > kRecv ? kStages * kStage : kRecv;
  // + the tile's folded-BN gain and bias (f32 epilogues), BN floats each
  static constexpr int kBytes = kRing + 1024 /*align*/ + 256 /*barriers*/ + 2 * BN * 4;
};

// profiling (dbg & 16): per CTA SM clock at [start, setup, producer done,
// MMA issue done, partial tile in smem, after cluster barrier, reduced, end]
__device__ unsigned long long g_gemm_stamps[512 * 8];
// globaltimer (ns) at CTA start / end, double-buffered by launch parity (dbg & 256)
__device__ unsigned long long g_gemm_gt[2 * 512 * 2];
__device__ unsigned long long g_gemm_st2[512 * 16];  // reduction sub-phases (thread 0, SM clock)
__device__ __forceinline__ unsigned long long gt_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long gtime() {
  // SM clock (cycles): consistent between the warps of a CTA, unlike the
  // coarse-grained globaltimer
  return (unsigned long long)clock64();
}

// F4: the operands are FP4 (E2M1) levels, 256 per 128-byte K-block row,
// and the MMA is kind::mxf4 with unit block scales in TMEM columns [BN, kCols)
template <int BN, bool F4>
__global__ void __launch_bounds__(kThreads, 1)
k_gemm_tc_i8(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
             const __grid_constant__ CUtensorMap tmO, int direct, int mcx,
             int M, int N, int num_kb, int m_pad, int n_pad, int S, tk_epilogue e,
             int dbg_arg) {
  const int dbg = TK_DBG(dbg_arg);  // profiling phase knobs: 0 in the production build
  constexpr int kStages = TcSmem<BN>::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * TcSmem<BN>::kA;  // A ring, then B ring
  // own partial slice (s16, chunk-major, see below), aliasing the ring
  int16_t* own = reinterpret_cast<int16_t*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + TcSmem<BN>::kRing);
  uint64_t* empty = full + kStages;
  uint64_t* tmem_full = empty + kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);
  float* s_gain = reinterpret_cast<float*>(smem + TcSmem<BN>::kRing + 256);  // [BN], columns clamped to N-1
  float* s_bias = s_gain + BN;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int cta = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  unsigned long long* st = (dbg & 16) && cta < 512 ? g_gemm_stamps + cta * 8 : nullptr;
  unsigned long long* gt = st ? g_gemm_gt + ((dbg >> 8) & 1) * 1024 + cta * 2 : nullptr;
  if (st && threadIdx.x == 0) {
    st[0] = gtime();
    gt[0] = gt_ns();
  }
  const int z = blockIdx.z;  // K split index == rank in the (1, 1, S) cluster
  const int kb0 = (int)((long long)z * num_kb / S), kb1 = (int)((long long)(z + 1) * num_kb / S);
  // F4: accumulator columns + unit scale-factor columns (power of two >= BN + 128)
  constexpr uint32_t kCols = F4 ? (BN <= 128 ? 256 : 512) : (BN < 32 ? 32 : BN);

  if (threadIdx.x == 0) {
    sm100::tma_prefetch(&tmA);
    sm100::tma_prefetch(&tmB);
    if (direct) sm100::tma_prefetch(&tmO);
    for (int s = 0; s < kStages; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], mcx);  // released by the MMA warps of all mcx CTAs
    }
    sm100::mbar_init(tmem_full, 1);
    sm100::fence_mbar_init();
  }
  // A multicast (mcx > 1, S == 1): the mcx CTAs of a (mcx, 1, 1) cluster share
  // the A tile; each loads BM/mcx of its rows into every CTA of the cluster.
  const uint32_t mc_rank = mcx > 1 ? sm100::cluster_ctarank() : 0;
  const uint16_t mc_mask = (uint16_t)((1u << mcx) - 1u);
  if (mcx > 1)
    sm100::cluster_sync();  // peers' barriers initialised before any multicast
  else
    __syncthreads();
  // The producer starts loading at once; the TMEM allocation (and, for F4,
  // the unit scale factors) is set up meanwhile by warps 1-5 (named barrier 1).
  uint32_t tmem = 0;
  if (warp >= 1) {
    if (warp == 1) sm100::tmem_alloc<kCols>(tmem_slot);
    if (warp >= 2 && e.mode != TK_EPI_I32)
      for (int i = threadIdx.x - 64; i < BN; i += kThreads - 64) {
        const int nn = min(n0 + i, N - 1);
        s_gain[i] = __ldg(e.gain + nn);
        s_bias[i] = __ldg(e.bias + nn);
      }
    sm100::tc_fence_before();
    sm100::named_bar_sync(1, kThreads - 32);
    sm100::tc_fence_after();
    tmem = *tmem_slot;
    if constexpr (F4) {  // E8M0 = 127 (2^0) everywhere, stored before any MMA reads it
      if (warp >= 2 && warp < 6)
        sm100::tmem_fill_unit_scales<kCols - BN>(tmem + ((uint32_t)((warp & 3) * 32) << 16) + BN);
      sm100::tc_fence_before();
      sm100::named_bar_sync(1, kThreads - 32);
      sm100::tc_fence_after();
    }
  }
  if (st && threadIdx.x == 32) st[1] = gtime();

  if (warp == 0) {
    // ---- TMA producer (whole warp waits, lane 0 issues) ----
    // weights do not depend on the previous kernel: the first stages' B
    // boxes go out before griddepcontrol.wait, the A boxes after it
    constexpr int KD = TcSmem<BN>::kKD;
    const int nst = (kb1 - kb0 + KD - 1) / KD;  // stages of this CTA's K range
    // (a box may reach one K block past kb1: zero fill past num_kb; inside
    // another split's range the MMA loop skips that block)
    auto load_b = [&](int s2, int kb) {
      if constexpr (KD == 1)
        sm100::tma_load_2d(sB + s2 * TcSmem<BN>::kB, &tmB, &full[s2], 0, kb * n_pad + n0);
      else
        sm100::tma_load_3d(sB + s2 * TcSmem<BN>::kB, &tmB, &full[s2], 0, n0, kb);
    };
    const int npre = (dbg & 8) ? 0 : min(kStages, nst);
    if (lane == 0)
      for (int i = 0; i < npre; ++i) {
        sm100::mbar_arrive_expect_tx(&full[i], TcSmem<BN>::kStage);
        load_b(i, kb0 + i * KD);
      }
    sm100::pdl_wait();
    int s = 0, round = 0;
    for (int si = 0; si < nst; ++si) {
      const int kb = kb0 + si * KD;
      if (round) sm100::mbar_wait(&empty[s], (round - 1) & 1);
      if (lane == 0) {
        if (dbg & 8) {  // profiling: no operand traffic
          sm100::mbar_arrive(&full[s]);
        } else {
          if (si >= npre) {
            sm100::mbar_arrive_expect_tx(&full[s], TcSmem<BN>::kStage);
            load_b(s, kb);
          }
          // K-block-major operands: each box is KD contiguous 16 KB / BN*128 B blocks
          if constexpr (KD > 1) {
            sm100::tma_load_3d(sA + s * TcSmem<BN>::kA, &tmA, &full[s], 0, m0, kb);
          } else if (mcx > 1) {
            const int part = BM / mcx;
            sm100::tma_load_2d_mc(sA + s * TcSmem<BN>::kA + mc_rank * part * 128, &tmA, &full[s], 0,
                                  kb * m_pad + m0 + (int)mc_rank * part, mc_mask);
          } else {
            sm100::tma_load_2d(sA + s * TcSmem<BN>::kA, &tmA, &full[s], 0, kb * m_pad + m0);
          }
        }
      }
      __syncwarp();
      if (++s == kStages) { s = 0; ++round; }
    }
  } else if (warp == 1) {
    // ---- MMA issuer: KD x 4 x (128 x BN x 32 bytes of K) per stage ----
    constexpr int KD = TcSmem<BN>::kKD;
    constexpr uint32_t idesc = F4 ? sm100::idesc_f4(BM, BN) : sm100::idesc_i8(BM, BN);
    const int nst = (kb1 - kb0 + KD - 1) / KD;
    int s = 0, round = 0;
    for (int si = 0; si < nst; ++si) {
      const int kbs = kb0 + si * KD;
      sm100::mbar_wait(&full[s], round & 1);
      sm100::tc_fence_after();
      if (!(dbg & 4)) {  // dbg & 4: profiling, no MMAs
#pragma unroll
        for (int j = 0; j < KD; ++j) {
          const int kb = kbs + j;
          if (kb >= kb1) break;
          const uint32_t a0 = sm100::smem_u32(sA + s * TcSmem<BN>::kA + j * BM * BK);
          const uint32_t b0 = sm100::smem_u32(sB + s * TcSmem<BN>::kB + j * BN * BK);
#pragma unroll
          for (int k = 0; k < BK / 32; ++k) {  // 32 bytes per MMA: K = 32 (s8) or 64 (fp4)
            if constexpr (F4)
              sm100::mma_f4_elect(tmem, sm100::desc_k_sw128(a0 + k * 32), sm100::desc_k_sw128(b0 + k * 32),
                                  idesc, (kb > kb0 || k > 0) ? 1u : 0u, tmem + BN, tmem + BN + 64);
            else
              sm100::mma_i8_elect(tmem, sm100::desc_k_sw128(a0 + k * 32), sm100::desc_k_sw128(b0 + k * 32),
                                  idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          }
        }
      }
      if (mcx > 1)
        sm100::mma_commit_mc_elect(&empty[s], mc_mask);
      else
        sm100::mma_commit_elect(&empty[s]);
      if (++s == kStages) { s = 0; ++round; }
    }
    sm100::mma_commit_elect(tmem_full);
    if (st && lane == 0) st[3] = gtime();
  }
  if (direct == 1) {
    // ---- S == 1, row-major output: TMEM -> registers -> epilogue -> shared
    // memory (128B-swizzled 32x32 boxes, two per warp) -> TMA tensor store.
    // Each epilogue warp owns TMEM lane quarter q = rows [32q, 32q + 32).
    if (warp >= 2 && !(dbg & 2)) {
      const int q = warp & 3, half = (warp - 2) >> 2;
      uint8_t* buf = smem + (warp - 2) * 8192;  // the operand ring is idle once tmem_full fired
      sm100::pdl_wait();  // (outputs may still be read by the previous kernel)
      sm100::mbar_wait(tmem_full, 0);
      sm100::tc_fence_after();
      const bool f32 = e.mode != TK_EPI_I32;
      constexpr int kHalf = BN / 2 < 32 ? 32 : BN / 2;
#pragma unroll 1
      for (int c0 = half * kHalf; c0 < (half + 1) * kHalf && c0 < BN; c0 += 32) {
        uint32_t r[32];
        sm100::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + c0, r);
        sm100::tmem_ld_wait();
        if (f32) {
          const float sc = e.out_scale;
#pragma unroll
          for (int i = 0; i < 8; ++i) {  // broadcast shared-memory reads of 4 gains / biases
            const float4 g = *reinterpret_cast<const float4*>(s_gain + c0 + 4 * i);
            const float4 b = *reinterpret_cast<const float4*>(s_bias + c0 + 4 * i);
            const float gv[4] = {g.x, g.y, g.z, g.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int j = 4 * i + k;
              // F4 accumulators are exact integers in f32 already
              const float a = F4 ? __uint_as_float(r[j]) : (float)(int)r[j];
              // R:linalg.hpp:322-323 with the reference build's FMA contraction
              r[j] = __float_as_uint(__fmaf_rn(gv[k], __fmul_rn(sc, a), bv[k]));
            }
          }
        } else if constexpr (F4) {  // f32 accumulators of exact integers
#pragma unroll
          for (int j = 0; j < 32; ++j) r[j] = (uint32_t)__float2int_rn(__uint_as_float(r[j]));
        }
        uint8_t* b = buf + ((c0 / 32) & 1) * 4096;
        if (c0 >= half * kHalf + 64) {  // this buffer's previous store must have read it
          if (lane == 0) sm100::bulk_wait_read<1>();
          __syncwarp();
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)  // 16-byte chunk i of row `lane`, SWIZZLE_128B
          *reinterpret_cast<uint4*>(b + lane * 128 + ((i ^ (lane & 7)) * 16)) =
              make_uint4(r[4 * i], r[4 * i + 1], r[4 * i + 2], r[4 * i + 3]);
        sm100::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          sm100::tma_store_2d(&tmO, b, n0 + c0, m0 + q * 32);
          sm100::bulk_commit();
        }
      }
      if (lane == 0) sm100::bulk_wait_read<0>();  // smem source consumed (global writes drain on their own)
      __syncwarp();
    }
    if (st && threadIdx.x == 64) st[4] = gtime();
    sm100::tc_fence_before();
    if (mcx > 1)
      sm100::cluster_sync();  // no peer may still signal this CTA's barriers
    else
      __syncthreads();
    if (warp == 1) sm100::tmem_dealloc<kCols>(tmem);
    if (st && threadIdx.x == 32) {
      st[7] = gtime();
      gt[1] = gt_ns();
    }
    return;
  }
  // ---- split-K exchange --------------------------------------------------
  // Rows [r*128/S, (r+1)*128/S) of the tile belong to cluster rank r.  After a
  // cluster barrier (every CTA past its K loop, so operand rings are free),
  // each epilogue thread pushes its accumulator row as s16 (|partial| <=
  // 2*K/S < 2^15, checked at launch) into the owner's shared memory with
  // distributed-shared-memory stores; a second barrier publishes them.
  // Receive layout [src][row][BN/8 chunks of 16 B], chunks XOR-swizzled by
  // row (a warp's 32 row-stores spread over the banks).  The integer sums
  // are exact in any order.
  const int rows_s = BM / S;
  constexpr int C8 = BN / 8;  // 16-byte chunks (8 x s16) per row
  auto swz = [](int row, int c) { return (c & ~7) | ((c ^ row) & 7); };
  uint4* recv = reinterpret_cast<uint4*>(own);  // [S][rows_s][C8]
  if (warp >= 1) sm100::pdl_wait();  // (warp 0 waited before its A loads)
  if (warp >= 2) sm100::mbar_wait(tmem_full, 0);
  sm100::tc_fence_before();
  sm100::cluster_sync();
  if (st && threadIdx.x == 0) st[2] = gtime();  // (re-used: exchange start)
  if (warp >= 2 && !(dbg & 2)) {
    sm100::tc_fence_after();
    const int q = warp & 3, half = (warp - 2) >> 2;  // TMEM lane quarter, column half
    const int row = q * 32 + lane;
    const int owner = row / rows_s, rr = row - owner * rows_s;
    const uint32_t dst = sm100::smem_u32(recv + (size_t)(z * rows_s + rr) * C8);
    constexpr int kHalf = BN / 2 < 32 ? 32 : BN / 2;
#pragma unroll 1
    for (int c0 = half * kHalf; c0 < (half + 1) * kHalf && c0 < BN; c0 += 32) {
      uint32_t r[32];
      sm100::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + c0, r);
      sm100::tmem_ld_wait();
      if constexpr (F4) {  // f32 accumulators of exact integers (|v| < 2^15)
#pragma unroll
        for (int j = 0; j < 32; ++j) r[j] = (uint32_t)__float2int_rn(__uint_as_float(r[j]));
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) w[i] = (r[8 * j + 2 * i] & 0xFFFFu) | (r[8 * j + 2 * i + 1] << 16);
        const uint32_t a = dst + (uint32_t)swz(rr, c0 / 8 + j) * 16u;
        if (owner == z)  // own slice: plain shared-memory store
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(w[0]), "r"(w[1]), "r"(w[2]),
                       "r"(w[3])
                       : "memory");
        else
          sm100::st_cluster_v4(a, (uint32_t)owner, make_uint4(w[0], w[1], w[2], w[3]));
      }
    }
  }
  if (st && threadIdx.x == 64) st[4] = gtime();
  sm100::cluster_sync();
  if (st && threadIdx.x == 0) st[5] = gtime();

  if (direct == 2) {
    // ---- row-major output, S in {2, 4} (rows_s >= 32): sum the S slices of
    // (row, 8-column group) items, rows fastest across threads (conflict-free
    // on both sides), into 128B-swizzled 32x32 staging boxes after the receive
    // area, then TMA tensor stores of the rows_s x BN slice (clipped at M, N).
    uint8_t* stage = smem + BM * BN * 2;
    const int r_lo = z * rows_s;
    // work pairs (32-row block, 8-column group), one row per lane; S is 2 or 4
    const int pairs = (dbg & 1) ? 0 : (rows_s >> 5) * C8;
    const bool f32 = e.mode != TK_EPI_I32;
    constexpr int kWarps = kThreads / 32;
    if (st && threadIdx.x == 0) g_gemm_st2[cta * 16] = gtime();
    int it = 0;
    const uint4* rv = recv + lane * C8;  // this lane's row within each 32-row block
    auto sum_slices = [&](int p, int (&acc)[8]) {
      const int c8 = p & (C8 - 1), rb = p / C8;
      const int cs = swz(lane, c8);  // (the swizzle depends on row & 7 = lane & 7)
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = 0;
#pragma unroll 1
      for (int src = 0; src < S; ++src) {
        const uint4 v = rv[(size_t)(src * rows_s + rb * 32) * C8 + cs];
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          acc[2 * i] += (int)(int16_t)(w[i] & 0xFFFFu);
          acc[2 * i + 1] += (int)w[i] >> 16;
        }
      }
    };
    auto put = [&](int p, const uint32_t (&o)[8]) {
      const int c8 = p & (C8 - 1), rb = p / C8;
      uint8_t* box = stage + (rb * (BN / 32) + (c8 >> 2)) * 4096 + lane * 128;
#pragma unroll
      for (int h = 0; h < 2; ++h)
        *reinterpret_cast<uint4*>(box + ((((c8 & 3) * 2 + h) ^ (lane & 7)) * 16)) =
            make_uint4(o[4 * h], o[4 * h + 1], o[4 * h + 2], o[4 * h + 3]);
    };
    if (f32) {
      const float sc = e.out_scale;
#pragma unroll 1
      for (int p = warp; p < pairs; p += kWarps) {
        int acc[8];
        sum_slices(p, acc);
        const int c = (p & (C8 - 1)) * 8;
        const float4 g0 = *reinterpret_cast<const float4*>(s_gain + c);
        const float4 g1 = *reinterpret_cast<const float4*>(s_gain + c + 4);
        const float4 b0 = *reinterpret_cast<const float4*>(s_bias + c);
        const float4 b1 = *reinterpret_cast<const float4*>(s_bias + c + 4);
        const float gv[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
        const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
        uint32_t o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)  // R:linalg.hpp:322-323 with the reference build's FMA contraction
          o[j] = __float_as_uint(__fmaf_rn(gv[j], __fmul_rn(sc, (float)acc[j]), bv[j]));
        put(p, o);
        if (st && threadIdx.x == 0 && it < 8) g_gemm_st2[cta * 16 + 1 + it++] = gtime();
      }
    } else {
#pragma unroll 1
      for (int p = warp; p < pairs; p += kWarps) {
        int acc[8];
        sum_slices(p, acc);
        uint32_t o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = (uint32_t)acc[j];
        put(p, o);
        if (st && threadIdx.x == 0 && it < 8) g_gemm_st2[cta * 16 + 1 + it++] = gtime();
      }
    }
    if (st && threadIdx.x == 0) g_gemm_st2[cta * 16 + 12] = gtime();
    sm100::fence_proxy_async_smem();
    __syncthreads();
    if (st && threadIdx.x == 0) g_gemm_st2[cta * 16 + 13] = gtime();
    if (threadIdx.x == 0 && pairs) {
      for (int rb = 0; rb < rows_s / 32; ++rb)
        for (int cb = 0; cb < BN / 32; ++cb)
          sm100::tma_store_2d(&tmO, stage + (rb * (BN / 32) + cb) * 4096, n0 + cb * 32, m0 + r_lo + rb * 32);
      sm100::bulk_commit();
      if (st) g_gemm_st2[cta * 16 + 14] = gtime();
      sm100::bulk_wait_read<0>();
      if (st) g_gemm_st2[cta * 16 + 15] = gtime();
    }
    if (st && threadIdx.x == 0) st[6] = gtime();
    __syncthreads();
    if (warp == 1) sm100::tmem_dealloc<kCols>(tmem);
    if (st && threadIdx.x == 32) {
      st[7] = gtime();
      gt[1] = gt_ns();
    }
    return;
  }
  // ---- reduction + epilogue over this CTA's row slice, 4 items per thread.
  // Row-major outputs: consecutive threads take consecutive 8-column groups
  // of a row (coalesced stores); NCHW: consecutive rows.
  const int r_lo = z * rows_s;
  const int items = dbg & 1 ? 0 : rows_s * C8;
  const bool nchw = e.mode == TK_EPI_F32_NCHW;
  const bool vec_ok = (N % 8) == 0;
  for (int base = threadIdx.x; base < items; base += 4 * kThreads) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int idx = base + u * kThreads;
      if (idx >= items) break;
      const int rr = nchw ? idx % rows_s : idx / C8;
      const int c8 = nchw ? idx / rows_s : idx % C8;
      const int m = m0 + r_lo + rr, n = n0 + c8 * 8;
      if (m >= M || n >= N) continue;
      int acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int src = 0; src < S; ++src) {
        const uint4 v = recv[(size_t)(src * rows_s + rr) * C8 + swz(rr, c8)];
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          acc[2 * i] += (int)(int16_t)(w[i] & 0xFFFFu);
          acc[2 * i + 1] += (int)w[i] >> 16;
        }
      }
      const int nv = N - n < 8 ? N - n : 8;
      if (e.mode == TK_EPI_I32) {
        int32_t* o = static_cast<int32_t*>(e.out) + (size_t)m * N + n;
        if (vec_ok) {
          reinterpret_cast<int4*>(o)[0] = make_int4(acc[0], acc[1], acc[2], acc[3]);
          reinterpret_cast<int4*>(o)[1] = make_int4(acc[4], acc[5], acc[6], acc[7]);
        } else {
          for (int j = 0; j < nv; ++j) o[j] = acc[j];
        }
        continue;
      }
      float y[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int nn = n + (j < nv ? j : 0);
        // R:linalg.hpp:322-323 with the reference build's FMA contraction
        y[j] = __fmaf_rn(__ldg(e.gain + nn), __fmul_rn(e.out_scale, (float)acc[j]), __ldg(e.bias + nn));
      }
      if (!nchw) {
        float* o = static_cast<float*>(e.out) + (size_t)m * N + n;
        if (vec_ok) {
          reinterpret_cast<float4*>(o)[0] = make_float4(y[0], y[1], y[2], y[3]);
          reinterpret_cast<float4*>(o)[1] = make_float4(y[4], y[5], y[6], y[7]);
        } else {
          for (int j = 0; j < nv; ++j) o[j] = y[j];
        }
      } else {
        const int b = m / e.plane, p = m - b * e.plane;
        float* o = static_cast<float*>(e.out) + ((size_t)b * N + n) * e.plane + p;
        for (int j = 0; j < nv; ++j) o[(size_t)j * e.plane] = y[j];
      }
    }
  }
  if (st && threadIdx.x == 0) st[6] = gtime();
  __syncthreads();
  if (warp == 1) sm100::tmem_dealloc<kCols>(tmem);
  if (st && threadIdx.x == 32) {
    st[7] = gtime();
    gt[1] = gt_ns();
  }
}

// ---- host side: tensor maps through the driver entry point ----------------
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// 2-D u8 tensor [rows][cols] (cols contiguous), box [box_rows][128 bytes]
bool make_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  EncodeFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols};
  cuuint32_t box[2] = {128, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 3-D u8 tensor [planes][rows][128 bytes] (K-block-major), box [depth][box_rows][128 bytes]
bool make_map3(CUtensorMap* m, const void* base, uint64_t rows, uint64_t planes, uint32_t box_rows, uint32_t depth) {
  EncodeFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {128, rows, planes};
  cuuint64_t strides[2] = {128, rows * 128};
  cuuint32_t box[3] = {128, box_rows, depth};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 2-D 4-byte tensor [rows][cols] (row-major output), 32 x 32 boxes, 128B swizzle
bool make_out_map(CUtensorMap* m, void* base, uint64_t rows, uint64_t cols, bool f32) {
  EncodeFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 4};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_INT32, 2, base, dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN, bool F4>
cudaError_t launch(const int8_t* a, int M, int num_kb, const tk_layer* L, tk_epilogue e, int S,
                   bool row_major, cudaStream_t s) {
  CUtensorMap ta, tb, to;
  // Row-major, 16-byte aligned outputs go out through TMA tensor stores:
  // directly from TMEM when S == 1, after the cluster reduction when S = 2, 4.
  int direct = row_major && S <= 4 ? (S == 1 ? 1 : 2) : 0;
  if (direct && !make_out_map(&to, e.out, (uint64_t)M, (uint64_t)L->out_c, e.mode != TK_EPI_I32)) direct = 0;
  if (!direct) memset(&to, 0, sizeof(to));
  const int m_pad = (M + BM - 1) / BM * BM;
  // K-block-major [kb][rows][128 B]: a 2-D map of num_kb*rows rows of 128 bytes
  // A multicast across a (mcx, 1, 1) cluster of N tiles (direct path only)
  const int mc_env = tk_knob("TK_GEMM_MC", 0);
  const int n_tiles = (L->out_c + BN - 1) / BN;
  int mcx = 1;
  if (direct == 1) {
    const int want = mc_env ? mc_env : 1;
    for (int c = 4; c >= 2; c /= 2)
      if (c <= want && n_tiles % c == 0) { mcx = c; break; }
  }
  if constexpr (TcSmem<BN>::kKD > 1) {  // 3-D view [kb][rows][128 B], boxes of kKD K blocks
    mcx = 1;
    if (!make_map3(&ta, a, (uint64_t)m_pad, (uint64_t)num_kb, BM, TcSmem<BN>::kKD)) return cudaErrorInvalidValue;
    if (!make_map3(&tb, F4 ? L->d_w4 : L->d_w8, (uint64_t)L->n_pad, (uint64_t)num_kb, BN, TcSmem<BN>::kKD))
      return cudaErrorInvalidValue;
  } else {
    if (!make_map(&ta, a, (uint64_t)num_kb * m_pad, 128, BM / mcx)) return cudaErrorInvalidValue;
    if (!make_map(&tb, F4 ? L->d_w4 : L->d_w8, (uint64_t)num_kb * L->n_pad, 128, BN)) return cudaErrorInvalidValue;
  }
  if (const cudaError_t er = tk_smem_attr((const void*)k_gemm_tc_i8<BN, F4>, TcSmem<BN>::kBytes); er != cudaSuccess)
    return er;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((L->out_c + BN - 1) / BN, (M + BM - 1) / BM, S);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = TcSmem<BN>::kBytes;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = mcx;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = S;
  // programmatic dependent launch
  const int pdl = tk_knob("TK_GEMM_PDL", 1);
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = pdl;
  cfg.attrs = at;
  cfg.numAttrs = 2;
#ifdef TK_PROFILE
  static int launches = 0;
  const int dbg0 = tk_knob("TK_GEMM_DBG", 0);
  const int dbg = (dbg0 & 16) ? (dbg0 | ((launches++ & 1) << 8)) : dbg0;  // stamp buffer parity
#else
  const int dbg = 0;
#endif
  return cudaLaunchKernelEx(&cfg, k_gemm_tc_i8<BN, F4>, ta, tb, to, direct, mcx, M, L->out_c, num_kb, m_pad, L->n_pad, S, e,
                            dbg);
}

}  // namespace

// K blocks one CTA may accumulate: its s16 partial |sum| <= 2*128*blocks < 2^15
constexpr int kMaxKbPerCta = 127;

bool tk_tc_supported(int M, int N, int k_pad) {
  return M > 0 && N > 0 && k_pad % BK == 0 && k_pad / BK <= 8 * kMaxKbPerCta && encode_fn() != nullptr;
}

cudaError_t tk_launch_gemm_tc(const int8_t* a_s8, int M, int k_pad, const tk_layer* L,
                              tk_epilogue e, cudaStream_t s) {
  return tk_launch_gemm_tc_fmt(a_s8, M, k_pad, L, e, false, s);
}

// fp4: a is [k_pad/256][m_pad][128 B] FP4 levels and L->d_w4 the weights
cudaError_t tk_launch_gemm_tc_fmt(const int8_t* a_s8, int M, int k_pad, const tk_layer* L, tk_epilogue e, bool fp4,
                                  cudaStream_t s) {
  if (!tk_tc_supported(M, L->out_c, k_pad)) return cudaErrorNotSupported;
  if (fp4 && (k_pad % 256 || !L->d_w4)) return cudaErrorNotSupported;
  const long tiles_m = (M + BM - 1) / BM;
  const int N = L->out_c, num_kb = fp4 ? k_pad / 256 : k_pad / BK;
  const int max_kb = fp4 ? kMaxKbPerCta / 2 : kMaxKbPerCta;  // 256 levels per fp4 K block
  const bool no_direct = tk_knob("TK_GEMM_NODIRECT", 0) != 0;
  const bool row_major = !no_direct && e.mode != TK_EPI_F32_NCHW && N % 4 == 0 && (uintptr_t)e.out % 16 == 0;
  auto tiles_of = [&](int bn) { return tiles_m * ((N + bn - 1) / bn); };
  // Tile shape: the operand traffic from L2 into the SMs,
  // K * (1/BM + 1/BN) per output, is what bounds this kernel (about 6300
  // B/clk chip-wide), so use the widest tile that still spreads over >= 2/3
  // of the SMs; split K across a cluster only when even 64-wide tiles leave
  // most SMs idle (the exchange + reduction then costs less than idle SMs).
  int BN = 64;
  for (int bn : {256, 128})
    if ((bn <= 128 || N >= 256) && tiles_of(bn) >= 96) { BN = bn; break; }
  int S = 1;
  if (tiles_of(BN) < 96) {
    BN = N > 64 ? 128 : 64;
    while (2 * S <= 4 && 2 * S <= num_kb && tiles_of(BN) * 2 * S <= 148) S *= 2;
  }
  if (const int bn = tk_knob("TK_GEMM_BN", 0)) BN = std::max(64, std::min(256, bn));
  if (const int sp = tk_knob("TK_GEMM_SPLIT", 0)) {
    S = 1;
    while (2 * S <= std::min({8, num_kb, sp})) S *= 2;
  }
  // s16 partials (cluster exchange, or the NCHW staging) stay exact; the
  // direct S == 1 epilogue reads the 32-bit accumulators straight from TMEM
  if (!(row_major && S == 1))
    while ((num_kb + S - 1) / S > max_kb && S < 8) S *= 2;
  if (!(row_major && S == 1) && (num_kb + S - 1) / S > max_kb) return cudaErrorNotSupported;
  if (fp4) {
    if (BN == 256) return launch<256, true>(a_s8, M, num_kb, L, e, S, row_major, s);
    if (BN == 128) return launch<128, true>(a_s8, M, num_kb, L, e, S, row_major, s);
    return launch<64, true>(a_s8, M, num_kb, L, e, S, row_major, s);
  }
  if (BN == 256) return launch<256, false>(a_s8, M, num_kb, L, e, S, row_major, s);
  if (BN == 128) return launch<128, false>(a_s8, M, num_kb, L, e, S, row_major, s);
  return launch<64, false>(a_s8, M, num_kb, L, e, S, row_major, s);
}

int tk_debug_gemm_stamps(unsigned long long* host_out) {
  // [512][8] SM-clock phase stamps, then [512][2] globaltimer start / end
  return cudaMemcpyFromSymbol(host_out, g_gemm_stamps, sizeof(unsigned long long) * 512 * 8) == cudaSuccess &&
                 cudaMemcpyFromSymbol(host_out + 512 * 8, g_gemm_gt, sizeof(unsigned long long) * 2048) ==
                     cudaSuccess &&
                 cudaMemcpyFromSymbol(host_out + 512 * 12, g_gemm_st2, sizeof(unsigned long long) * 512 * 16) ==
                     cudaSuccess
             ? TK_OK
             : TK_ERR_CUDA;
}

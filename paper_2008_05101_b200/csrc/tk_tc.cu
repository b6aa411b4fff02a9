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
// CTA = 6 warps: warp 0 TMA producer, warp 1 TMEM owner + MMA issuer,
// warps 2-5 move the accumulator TMEM -> shared memory (TMEM lane quarter =
// warp % 4); all 6 warps run the cluster reduction + epilogue.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "tk_internal.cuh"
#include "tk_sm100.cuh"

namespace {

constexpr int BM = 128, BK = 128;
constexpr int kThreads = 192;

template <int BN>
struct TcSmem {
  static constexpr int kA = BM * BK;  // bytes per stage
  static constexpr int kB = BN * BK;
  static constexpr int kStage = kA + kB;
  // as many stages as ~200 KB of shared memory holds (latency hiding)
  static constexpr int kStages = (200 * 1024 / kStage) > 8 ? 8 : (200 * 1024 / kStage);
  // split-K receive buffer, s16 [S][128/S][BN] = 128 x BN, aliasing the ring
  static constexpr int kRecv = BM * BN * 2;
  static constexpr int kRing = kStages * kStage > kRecv ? kStages * kStage : kRecv;
  static constexpr int kBytes = kRing + 1024 /*align*/ + 256 /*barriers*/;
};

// profiling (dbg & 16): per CTA SM clock at [start, setup, producer done,
// MMA issue done, partial tile in smem, after cluster barrier, reduced, end]
__device__ unsigned long long g_gemm_stamps[512 * 8];
__device__ __forceinline__ unsigned long long gtime() {
  // SM clock (cycles): consistent between the warps of a CTA, unlike the
  // coarse-grained globaltimer
  return (unsigned long long)clock64();
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
k_gemm_tc_i8(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
             int M, int N, int num_kb, int m_pad, int n_pad, int S, int16_t* __restrict__ red, tk_epilogue e,
             int dbg) {
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

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int cta = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  unsigned long long* st = (dbg & 16) && cta < 512 ? g_gemm_stamps + cta * 8 : nullptr;
  if (st && threadIdx.x == 0) st[0] = gtime();
  const int z = blockIdx.z;  // K split index == rank in the (1, 1, S) cluster
  const int kb0 = (int)((long long)z * num_kb / S), kb1 = (int)((long long)(z + 1) * num_kb / S);
  constexpr uint32_t kCols = BN < 32 ? 32 : BN;

  if (threadIdx.x == 0) {
    sm100::tma_prefetch(&tmA);
    sm100::tma_prefetch(&tmB);
    for (int s = 0; s < kStages; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], 1);
    }
    sm100::mbar_init(tmem_full, 1);
    sm100::fence_mbar_init();
  }
  if (warp == 1) sm100::tmem_alloc<kCols>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (st && threadIdx.x == 0) st[1] = gtime();

  if (warp == 0) {
    // ---- TMA producer (whole warp waits, lane 0 issues) ----
    int s = 0, round = 0;
    for (int kb = kb0; kb < kb1; ++kb) {
      if (round) sm100::mbar_wait(&empty[s], (round - 1) & 1);
      if (lane == 0) {
        if (dbg & 8) {  // profiling: no operand traffic
          sm100::mbar_arrive(&full[s]);
        } else {
          sm100::mbar_arrive_expect_tx(&full[s], TcSmem<BN>::kStage);
          // K-block-major operands: each box is one contiguous 16 / BN*128 byte block
          sm100::tma_load_2d(sA + s * TcSmem<BN>::kA, &tmA, &full[s], 0, kb * m_pad + m0);
          sm100::tma_load_2d(sB + s * TcSmem<BN>::kB, &tmB, &full[s], 0, kb * n_pad + n0);
        }
      }
      __syncwarp();
      if (++s == kStages) { s = 0; ++round; }
    }
  } else if (warp == 1) {
    // ---- MMA issuer: 4 x (128 x BN x 32) per stage ----
    constexpr uint32_t idesc = sm100::idesc_i8(BM, BN);
    int s = 0, round = 0;
    for (int kb = kb0; kb < kb1; ++kb) {
      sm100::mbar_wait(&full[s], round & 1);
      sm100::tc_fence_after();
      const uint32_t a0 = sm100::smem_u32(sA + s * TcSmem<BN>::kA);
      const uint32_t b0 = sm100::smem_u32(sB + s * TcSmem<BN>::kB);
      if (!(dbg & 4)) {  // dbg & 4: profiling, no MMAs
#pragma unroll
        for (int k = 0; k < BK / 32; ++k)
          sm100::mma_i8_elect(tmem, sm100::desc_k_sw128(a0 + k * 32), sm100::desc_k_sw128(b0 + k * 32), idesc,
                              (kb > kb0 || k > 0) ? 1u : 0u);
      }
      sm100::mma_commit_elect(&empty[s]);
      if (++s == kStages) { s = 0; ++round; }
    }
    sm100::mma_commit_elect(tmem_full);
    if (st && lane == 0) st[3] = gtime();
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
  if (warp >= 2) sm100::mbar_wait(tmem_full, 0);
  sm100::tc_fence_before();
  sm100::cluster_sync();
  if (st && threadIdx.x == 0) st[2] = gtime();  // (re-used: exchange start)
  if (warp >= 2 && !(dbg & 2)) {
    sm100::tc_fence_after();
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row = q * 32 + lane;
    const int owner = row / rows_s, rr = row - owner * rows_s;
    const uint32_t dst = sm100::smem_u32(recv + (size_t)(z * rows_s + rr) * C8);
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      uint32_t r[32];
      sm100::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + c0, r);
      sm100::tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) w[i] = (r[8 * j + 2 * i] & 0xFFFFu) | (r[8 * j + 2 * i + 1] << 16);
        sm100::st_cluster_v4(dst + (uint32_t)swz(rr, c0 / 8 + j) * 16u, (uint32_t)owner,
                             make_uint4(w[0], w[1], w[2], w[3]));
      }
    }
  }
  if (st && threadIdx.x == 64) st[4] = gtime();
  sm100::cluster_sync();
  if (st && threadIdx.x == 0) st[5] = gtime();

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
  if (st && threadIdx.x == 32) st[7] = gtime();
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

template <int BN>
cudaError_t launch(const int8_t* a, int M, int k_pad, const tk_layer* L, tk_epilogue e, int S,
                   int16_t* red, cudaStream_t s) {
  CUtensorMap ta, tb;
  const int num_kb = k_pad / BK, m_pad = (M + BM - 1) / BM * BM;
  // K-block-major [k/128][rows][128]: a 2-D map of num_kb*rows rows of 128 bytes
  if (!make_map(&ta, a, (uint64_t)num_kb * m_pad, 128, BM)) return cudaErrorInvalidValue;
  if (!make_map(&tb, L->d_w8, (uint64_t)num_kb * L->n_pad, 128, BN)) return cudaErrorInvalidValue;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_gemm_tc_i8<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcSmem<BN>::kBytes);
    attr_set = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((L->out_c + BN - 1) / BN, (M + BM - 1) / BM, S);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = TcSmem<BN>::kBytes;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = S;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  static const int dbg = getenv("TK_GEMM_DBG") ? atoi(getenv("TK_GEMM_DBG")) : 0;  // profiling knob
  return cudaLaunchKernelEx(&cfg, k_gemm_tc_i8<BN>, ta, tb, M, L->out_c, num_kb, m_pad, L->n_pad, S, red, e,
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
  if (!tk_tc_supported(M, L->out_c, k_pad)) return cudaErrorNotSupported;
  const long tiles_m = (M + BM - 1) / BM;
  const int N = L->out_c, num_kb = k_pad / BK;
  int BN = N >= 256 ? 256 : (N > 64 ? 128 : 64);
  if (getenv("TK_GEMM_BN")) BN = std::min(BN, std::max(64, atoi(getenv("TK_GEMM_BN"))));  // profiling
  const long tiles = tiles_m * ((N + BN - 1) / BN);
  // split K across a cluster until the grid covers the SMs (<= 8, the
  // portable cluster size; at least one K block per CTA)
  int S = 1;
  // (powers of two: the 128 tile rows split evenly over the cluster)
  while (2 * S <= 8 && 2 * S <= num_kb && tiles * 2 * S <= 148) S *= 2;
  if (getenv("TK_GEMM_SPLIT")) {  // profiling override
    S = 1;
    while (2 * S <= std::min({8, num_kb, atoi(getenv("TK_GEMM_SPLIT"))})) S *= 2;
  }
  while ((num_kb + S - 1) / S > kMaxKbPerCta) S *= 2;  // s16 partials stay exact
  int16_t* red = nullptr;  // (split-K exchange runs through distributed shared memory)
  if (BN == 256) return launch<256>(a_s8, M, k_pad, L, e, S, red, s);
  if (BN == 128) return launch<128>(a_s8, M, k_pad, L, e, S, red, s);
  return launch<64>(a_s8, M, k_pad, L, e, S, red, s);
}

int tk_debug_gemm_stamps(unsigned long long* host_out) {
  return cudaMemcpyFromSymbol(host_out, g_gemm_stamps, sizeof(unsigned long long) * 512 * 8) == cudaSuccess
             ? TK_OK
             : TK_ERR_CUDA;
}

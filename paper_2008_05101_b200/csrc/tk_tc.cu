// tk_tc.cu -- the int8 tensor-core variant of the ternary contraction:
// tcgen05.mma kind::i8 with TMA-staged operands and the accumulator in TMEM.
//
// Operands are the quantization LEVELS as s8 (activations {0,1,2} with the
// nonneg offset folded in, or {-1,0,1}; weights {-1,0,1}), so the s32
// accumulator equals packed_gemm's offset-corrected result exactly
// (R:linalg.hpp:253-276) and the epilogue is the same folded-BN FMA.
//
// CTA = 6 warps: warp 0 TMA producer, warp 1 TMEM owner + MMA issuer,
// warps 2-5 epilogue (TMEM lane quarter = warp % 4).  128 x BN tile,
// K staged 128 bytes per stage with SWIZZLE_128B, kStages-deep mbarrier ring.
#include <cuda.h>

#include <mutex>
#include <unordered_map>

#include "tk_internal.cuh"
#include "tk_sm100.cuh"

namespace {

constexpr int BM = 128, BK = 128;
constexpr int kThreads = 192;

template <int BN>
struct TcSmem {
  static constexpr int kA = BM * BK;          // bytes per stage
  static constexpr int kB = BN * BK;
  static constexpr int kStage = kA + kB;
  // as many stages as ~200 KB of shared memory holds (latency hiding)
  static constexpr int kStages = (200 * 1024 / kStage) > 8 ? 8 : (200 * 1024 / kStage);
  static constexpr int kBytes = kStages * kStage + 1024 /*align*/ + 256 /*barriers*/;
};

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
k_gemm_tc_i8(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
             int M, int N, int num_kb, tk_epilogue e) {
  constexpr int kStages = TcSmem<BN>::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * TcSmem<BN>::kA;  // A ring, then B ring
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * TcSmem<BN>::kStage);
  uint64_t* empty = full + kStages;
  uint64_t* tmem_full = empty + kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
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

  if (warp == 0 && lane == 0) {
    // ---- TMA producer ----
    // CTAs sharing an A tile start at different K blocks (integer sums are
    // order independent) so they do not hammer the same L2 lines at once
    const int k_rot = blockIdx.x % num_kb;
    for (int kb = 0; kb < num_kb; ++kb) {
      const int s = kb % kStages;
      if (kb >= kStages) sm100::mbar_wait(&empty[s], ((kb / kStages) - 1) & 1);
      int kk = kb + k_rot;
      if (kk >= num_kb) kk -= num_kb;
      sm100::mbar_arrive_expect_tx(&full[s], TcSmem<BN>::kStage);
      sm100::tma_load_2d(sA + s * TcSmem<BN>::kA, &tmA, &full[s], kk * BK, m0);
      sm100::tma_load_2d(sB + s * TcSmem<BN>::kB, &tmB, &full[s], kk * BK, n0);
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer: 4 x (128 x BN x 32) per stage ----
    constexpr uint32_t idesc = sm100::idesc_i8(BM, BN);
    for (int kb = 0; kb < num_kb; ++kb) {
      const int s = kb % kStages;
      sm100::mbar_wait(&full[s], (kb / kStages) & 1);
      sm100::tc_fence_after();
      const uint32_t a0 = sm100::smem_u32(sA + s * TcSmem<BN>::kA);
      const uint32_t b0 = sm100::smem_u32(sB + s * TcSmem<BN>::kB);
#pragma unroll
      for (int k = 0; k < BK / 32; ++k) {
        sm100::mma_i8(tmem, sm100::desc_k_sw128(a0 + k * 32), sm100::desc_k_sw128(b0 + k * 32),
                      idesc, (kb | k) != 0);
      }
      sm100::mma_commit(&empty[s]);
    }
    sm100::mma_commit(tmem_full);
  } else if (warp >= 2) {
    // ---- epilogue: TMEM -> registers -> folded-BN FMA -> global ----
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int m = m0 + q * 32 + lane;
    sm100::mbar_wait(tmem_full, 0);
    sm100::tc_fence_after();
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      uint32_t r[32];
      sm100::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + c0, r);
      sm100::tmem_ld_wait();
      if (m < M) {
        if (e.mode == TK_EPI_I32) {
          int32_t* out = static_cast<int32_t*>(e.out) + (size_t)m * N;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int n = n0 + c0 + j;
            if (n < N) out[n] = (int32_t)r[j];
          }
        } else {
          const int b = e.mode == TK_EPI_F32_NCHW ? m / e.plane : 0;
          const int p = e.mode == TK_EPI_F32_NCHW ? m - b * e.plane : 0;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int n = n0 + c0 + j;
            if (n < N) {
              // R:linalg.hpp:322-323 with the reference build's FMA contraction
              const float y = __fmaf_rn(e.gain[n], __fmul_rn(e.out_scale, (float)(int32_t)r[j]),
                                        e.bias[n]);
              if (e.mode == TK_EPI_F32_ROWS)
                static_cast<float*>(e.out)[(size_t)m * N + n] = y;
              else
                static_cast<float*>(e.out)[((size_t)b * N + n) * e.plane + p] = y;
            }
          }
        }
      }
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) sm100::tmem_dealloc<kCols>(tmem);
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
cudaError_t launch(const int8_t* a, int M, int k_pad, const tk_layer* L, tk_epilogue e,
                   cudaStream_t s) {
  CUtensorMap ta, tb;
  if (!make_map(&ta, a, (uint64_t)M, (uint64_t)k_pad, BM)) return cudaErrorInvalidValue;
  if (!make_map(&tb, L->d_w8, (uint64_t)L->n_pad, (uint64_t)k_pad, BN)) return cudaErrorInvalidValue;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_gemm_tc_i8<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         TcSmem<BN>::kBytes);
    attr_set = true;
  }
  dim3 grid((L->out_c + BN - 1) / BN, (M + BM - 1) / BM);
  k_gemm_tc_i8<BN><<<grid, kThreads, TcSmem<BN>::kBytes, s>>>(ta, tb, M, L->out_c, k_pad / BK, e);
  return cudaGetLastError();
}

}  // namespace

bool tk_tc_supported(int M, int N, int k_pad) {
  return M > 0 && N > 0 && k_pad % BK == 0 && encode_fn() != nullptr;
}

cudaError_t tk_launch_gemm_tc(const int8_t* a_s8, int M, int k_pad, const tk_layer* L,
                              tk_epilogue e, cudaStream_t s) {
  if (!tk_tc_supported(M, L->out_c, k_pad)) return cudaErrorNotSupported;
  const long tiles_m = (M + BM - 1) / BM;
  const int N = L->out_c;
  // widest N tile that still yields at least one CTA per SM; else the narrowest
  if (N > 128 && tiles_m * ((N + 255) / 256) >= 148) return launch<256>(a_s8, M, k_pad, L, e, s);
  if (N > 64 && tiles_m * ((N + 127) / 128) >= 148) return launch<128>(a_s8, M, k_pad, L, e, s);
  return launch<64>(a_s8, M, k_pad, L, e, s);
}

// desc_test.cu -- hardware check of the implicit-im2col trick the conv kernel
// relies on: an activation tile loaded ONCE by TMA into a swizzled SMEM
// buffer [rows][R bytes] (R = 64 -> SWIZZLE_64B, R = 128 -> SWIZZLE_128B), and
// tcgen05.mma reading a ROW-SHIFTED view of it (start address + shift*R,
// k-step + 32 B) -- i.e. a different kernel tap -- with the matching
// descriptor.  Verifies D = A[shift : shift+128, :] * B^T exactly for several
// shifts, and times the TMA box load rate for both swizzles.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o desc_test desc_test.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>

#include "../paper_2008_05101_b200/csrc/tk_sm100.cuh"

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint64_t desc_sw(uint32_t saddr, int R, int base_off_mode) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((8 * R) >> 4) << 32;  // SBO = 8 rows
  d |= (uint64_t)1 << 46;
  if (base_off_mode) d |= (uint64_t)((saddr >> 7) & 7) << 49;
  d |= (uint64_t)(R == 128 ? 2 : 4) << 61;  // SWIZZLE_128B = 2, SWIZZLE_64B = 4
  return d;
}

// one CTA: TMA-load A rows [0, 256) (R bytes each) and B [N=64 rows][R], then
// for the given shift issue R/32 MMAs and dump D (128 x 64 int32).
template <int R>
__global__ void k_test(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb,
                       int shift, int base_off_mode, int32_t* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = sm;                 // 256 rows * R
  uint8_t* sb = sm + 256 * R;       // 64 rows * R
  __shared__ __align__(8) uint64_t bar, done;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    sm100::mbar_init(&bar, 1);
    sm100::mbar_init(&done, 1);
    sm100::fence_mbar_init();
  }
  if (warp == 0) sm100::tmem_alloc<64>(&tslot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    sm100::mbar_arrive_expect_tx(&bar, 256 * R + 64 * R);
    sm100::tma_load_2d(sa, &ma, &bar, 0, 0);
    sm100::tma_load_2d(sb, &mb, &bar, 0, 0);
    sm100::mbar_wait(&bar, 0);
    sm100::tc_fence_after();
    constexpr uint32_t idesc = sm100::idesc_i8(128, 64);
    const uint32_t a0 = sm100::smem_u32(sa) + shift * R, b0 = sm100::smem_u32(sb);
    for (int k = 0; k < R / 32; ++k)
      sm100::mma_i8(tmem, desc_sw(a0 + k * 32, R, base_off_mode), desc_sw(b0 + k * 32, R, base_off_mode),
                    idesc, k > 0);
    sm100::mma_commit(&done);
  }
  __syncwarp();
  sm100::mbar_wait(&done, 0);
  sm100::tc_fence_after();
  // 4 warps read TMEM lanes
  const int q = warp & 3, lane = threadIdx.x & 31;
  for (int c0 = 0; c0 < 64; c0 += 32) {
    uint32_t r[32];
    sm100::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + c0, r);
    sm100::tmem_ld_wait();
    for (int j = 0; j < 32; ++j) out[(q * 32 + lane) * 64 + c0 + j] = (int32_t)r[j];
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc<64>(tmem);
}

// TMA box throughput for a [rows][R] tensor, box {R, rows_box}
template <int R>
__global__ void k_rate(const __grid_constant__ CUtensorMap m, int rows_box, int iters, int range,
                       unsigned long long* sink) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  const int bytes = rows_box * R;
  const int stages = 4;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + stages * ((bytes + 1023) & ~1023));
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) sm100::mbar_init(&full[s], 1);
    sm100::fence_mbar_init();
    int c = blockIdx.x * 3001;
    for (int i = 0; i < iters + stages; ++i) {
      const int s = i % stages;
      if (i >= stages) sm100::mbar_wait(&full[s], ((i / stages) - 1) & 1);
      if (i < iters) {
        sm100::mbar_arrive_expect_tx(&full[s], bytes);
        c = (c + 977) % range;
        sm100::tma_load_2d(sm + s * ((bytes + 1023) & ~1023), &m, &full[s], 0, c);
      }
    }
    sink[blockIdx.x] = sm[3];
  }
}

int main() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeFn enc = reinterpret_cast<EncodeFn>(p);
  int failures = 0;
  for (int R : {64, 128}) {
    const int rows = 256;
    std::vector<int8_t> A(rows * R), B(64 * R);
    srand(R);
    for (auto& v : A) v = (int8_t)(rand() % 3);
    for (auto& v : B) v = (int8_t)(rand() % 3 - 1);
    int8_t *dA, *dB;
    int32_t* dO;
    cudaMalloc(&dA, A.size());
    cudaMalloc(&dB, B.size());
    cudaMalloc(&dO, 128 * 64 * 4);
    cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
    CUtensorMap ma, mb;
    cuuint64_t da[2] = {(cuuint64_t)R, (cuuint64_t)rows}, db[2] = {(cuuint64_t)R, 64};
    cuuint64_t sa[1] = {(cuuint64_t)R};
    cuuint32_t ba[2] = {(cuuint32_t)R, 256}, bb[2] = {(cuuint32_t)R, 64}, es[2] = {1, 1};
    CUtensorMapSwizzle sw = R == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
    enc(&ma, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, dA, da, sa, ba, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc(&mb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, dB, db, sa, bb, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int smem = 256 * R + 64 * R + 2048;
    auto kern = R == 128 ? k_test<128> : k_test<64>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int mode = 0; mode < 2; ++mode) {
      for (int shift : {0, 1, 3, 5, 8, 58, 59, 117, 128}) {
        kern<<<1, 128, smem>>>(ma, mb, shift, mode, dO);
        std::vector<int32_t> O(128 * 64);
        cudaError_t e = cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int r = 0; r < 128; ++r)
          for (int n = 0; n < 64; ++n) {
            int acc = 0;
            for (int k = 0; k < R; ++k) acc += A[(r + shift) * R + k] * B[n * R + k];
            bad += acc != O[r * 64 + n];
          }
        printf("{\"R\": %d, \"base_offset_field\": %d, \"shift\": %d, \"mismatches\": %d, \"err\": \"%s\"}\n", R,
               mode, shift, bad, cudaGetErrorString(e));
        if (mode == 0) failures += bad != 0;
      }
    }
    // TMA rate, box {R, rows_box} from a 64 MB L2-resident [rows][R] tensor
    int8_t* big;
    const size_t nrows = (64ull << 20) / R;
    cudaMalloc(&big, nrows * R);
    unsigned long long* sink;
    cudaMalloc(&sink, 148 * 8);
    for (int rb : {128, 246}) {
      CUtensorMap m;
      cuuint64_t d2[2] = {(cuuint64_t)R, (cuuint64_t)nrows};
      cuuint32_t b2[2] = {(cuuint32_t)R, (cuuint32_t)rb};
      enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, big, d2, sa, b2, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      const int sbytes = 4 * ((rb * R + 1023) & ~1023) + 2048;
      auto rk = R == 128 ? k_rate<128> : k_rate<64>;
      cudaFuncSetAttribute(rk, cudaFuncAttributeMaxDynamicSharedMemorySize, sbytes);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      rk<<<148, 32, sbytes>>>(m, rb, 10, (int)(nrows - rb), sink);
      cudaEventRecord(e0);
      rk<<<148, 32, sbytes>>>(m, rb, 4000, (int)(nrows - rb), sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double b = 148.0 * 4000 * rb * R;
      printf("{\"tma_rate\": \"R=%d box_rows=%d stages=4\", \"TB_per_s\": %.2f, \"B_per_clk_per_sm\": %.1f}\n", R, rb,
             b / (ms * 1e-3) / 1e12, b / (ms * 1e-3) / 148 / 1.9e9);
    }
  }
  printf("{\"failures_mode0\": %d}\n", failures);
  return 0;
}

// tc_microbench.cu -- the two rates the tensor-core conv/GEMM design rests on:
//  (1) L2 -> SMEM streaming with cp.async.bulk (1-D TMA) per SM, all SMs busy;
//  (2) tcgen05.mma kind::i8 issue rate for M=128 and N in {64,128,256}, with
//      operands already resident in SMEM (no-swizzle K-major layout).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_microbench tc_microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2008_05101_b200/csrc/tk_sm100.cuh"

// ---- (1) bulk-copy streaming ----------------------------------------------
template <int kChunk, int kStages>
__global__ void k_stream(const uint8_t* src, size_t src_bytes, int iters, unsigned long long* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kChunk);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) sm100::mbar_init(&full[s], 1);
    sm100::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    size_t off = (size_t)blockIdx.x * 65536 % src_bytes;
    for (int i = 0; i < iters + kStages; ++i) {
      const int s = i % kStages;
      if (i >= kStages) sm100::mbar_wait(&full[s], ((i / kStages) - 1) & 1);
      if (i < iters) {
        sm100::mbar_arrive_expect_tx(&full[s], kChunk);
        sm100::bulk_load(smem + s * kChunk, src + off, kChunk, &full[s]);
        off += kChunk * 148;
        if (off + kChunk > src_bytes) off = (off + kChunk) % (src_bytes - kChunk);
        off &= ~size_t(127);
      }
    }
    sink[blockIdx.x] = smem[7];
  }
}

// ---- (1b) tensor TMA streaming: 3-D no-swizzle [slices][pos][16B] boxes and
// 2-D SWIZZLE_128B [rows][128B] boxes --------------------------------------------
template <int kBytes, int kStages, int kDims>
__global__ void k_stream_tma(const __grid_constant__ CUtensorMap map, int iters, int c1_range,
                             unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* buf = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(buf + kStages * kBytes);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) sm100::mbar_init(&full[s], 1);
    sm100::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int c = blockIdx.x * 97;
    for (int i = 0; i < iters + kStages; ++i) {
      const int s = i % kStages;
      if (i >= kStages) sm100::mbar_wait(&full[s], ((i / kStages) - 1) & 1);
      if (i < iters) {
        sm100::mbar_arrive_expect_tx(&full[s], kBytes);
        c = (c + 131) % c1_range;
        if (kDims == 3) {
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(sm100::smem_u32(buf + s * kBytes)),
              "l"(&map), "r"(sm100::smem_u32(&full[s])), "r"(0), "r"(c), "r"(0)
              : "memory");
        } else {
          sm100::tma_load_2d(buf + s * kBytes, &map, &full[s], 0, c);
        }
      }
    }
    sink[blockIdx.x] = buf[5];
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

void run_tma(const uint8_t* src, unsigned long long* sink) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeFn enc = reinterpret_cast<EncodeFn>(p);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000;
  {
    // 3-D: [4 slices][pos = 1M][16 B], box {16, 256, 4} = 16 KB
    CUtensorMap m;
    cuuint64_t dims[3] = {16, 1 << 20, 4};
    cuuint64_t str[2] = {16, 16ull << 20};
    cuuint32_t box[3] = {16, 256, 4}, es[3] = {1, 1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)src, dims, str, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int smem = 8 * 16384 + 2048;
    cudaFuncSetAttribute(k_stream_tma<16384, 8, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_stream_tma<16384, 8, 3><<<148, 32, smem>>>(m, 10, 1 << 10, sink);
    cudaEventRecord(e0);
    k_stream_tma<16384, 8, 3><<<148, 32, smem>>>(m, iters, 1 << 10, sink);  // 4 MB hot region
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double b = 148.0 * iters * 16384;
    printf("{\"test\": \"tma3d_noswz_box16x256x4\", \"enc\": %d, \"TB_per_s\": %.3f, \"B_per_clk_per_sm\": %.1f, \"err\": \"%s\"}\n",
           (int)r, b / (ms * 1e-3) / 1e12, b / (ms * 1e-3) / 148 / 1.9e9, cudaGetErrorString(cudaGetLastError()));
  }
  {
    // 2-D SW128: [rows][128 B], box {128, 128} = 16 KB
    CUtensorMap m;
    cuuint64_t dims[2] = {128, 1 << 18};
    cuuint64_t str[1] = {128};
    cuuint32_t box[2] = {128, 128}, es[2] = {1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)src, dims, str, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int smem = 8 * 16384 + 2048;
    cudaFuncSetAttribute(k_stream_tma<16384, 8, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_stream_tma<16384, 8, 2><<<148, 32, smem>>>(m, 10, 1 << 11, sink);
    cudaEventRecord(e0);
    k_stream_tma<16384, 8, 2><<<148, 32, smem>>>(m, iters, 1 << 11, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double b = 148.0 * iters * 16384;
    printf("{\"test\": \"tma2d_sw128_box128x128\", \"enc\": %d, \"TB_per_s\": %.3f, \"B_per_clk_per_sm\": %.1f, \"err\": \"%s\"}\n",
           (int)r, b / (ms * 1e-3) / 1e12, b / (ms * 1e-3) / 148 / 1.9e9, cudaGetErrorString(cudaGetLastError()));
  }
}

// ---- (2) MMA issue rate ------------------------------------------------------
template <int N>
__global__ void k_mma(int iters, unsigned long long* out_clk) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t done;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    sm100::mbar_init(&done, 1);
    sm100::fence_mbar_init();
  }
  for (int i = threadIdx.x; i < (128 + N) * 64; i += blockDim.x) smem[i] = (uint8_t)(i * 7);
  if (warp == 0) sm100::tmem_alloc<256>(&tslot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t a = sm100::smem_u32(smem), b = a + 128 * 32;
    // A: [2 k16-chunks][128 rows][16B]  B: [2][N][16B]
    const uint64_t ad = sm100::desc_k_noswz(a, 128 * 16, 128);
    const uint64_t bd = sm100::desc_k_noswz(b, N * 16, 128);
    constexpr uint32_t idesc = sm100::idesc_i8(128, N);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) sm100::mma_i8(tmem, ad, bd, idesc, i > 0);
    sm100::mma_commit(&done);
    sm100::mbar_wait(&done, 0);
    long long t1 = clock64();
    out_clk[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc<256>(tmem);
}

template <int kChunk, int kStages>
void run_stream(const uint8_t* src, size_t bytes, unsigned long long* sink, int blocks_per_sm) {
  const int iters = 4000;
  const int smem = kStages * kChunk + 1024;
  cudaFuncSetAttribute(k_stream<kChunk, kStages>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grid = 148 * blocks_per_sm;
  k_stream<kChunk, kStages><<<grid, 32, smem>>>(src, bytes, 10, sink);
  cudaEventRecord(e0);
  k_stream<kChunk, kStages><<<grid, 32, smem>>>(src, bytes, iters, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double b = (double)grid * iters * kChunk;
  printf("{\"test\": \"bulk_stream\", \"chunk\": %d, \"stages\": %d, \"ctas_per_sm\": %d, \"src_MB\": %.0f, "
         "\"TB_per_s\": %.3f, \"B_per_clk_per_sm_at_1.9GHz\": %.1f}\n",
         kChunk, kStages, blocks_per_sm, bytes / 1e6, b / (ms * 1e-3) / 1e12,
         b / (ms * 1e-3) / 148 / 1.9e9);
}

template <int N>
void run_mma(unsigned long long* d) {
  const int iters = 20000;
  cudaFuncSetAttribute(k_mma<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k_mma<N><<<148, 128, 64 * 1024>>>(iters, d);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  printf("{\"test\": \"mma_i8\", \"M\": 128, \"N\": %d, \"K\": 32, \"clk_per_mma\": %.2f, "
         "\"mac_per_clk_per_sm\": %.0f, \"err\": \"%s\"}\n",
         N, avg / iters, 128.0 * N * 32 * iters / avg, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  size_t bytes = 64ull << 20;  // L2 resident source
  uint8_t* src;
  unsigned long long* sink;
  cudaMalloc(&src, 1ull << 30);
  cudaMemset(src, 1, 1ull << 30);
  cudaMalloc(&sink, 148 * 8 * 8);
  run_stream<16384, 8>(src, bytes, sink, 1);
  run_stream<8192, 16>(src, bytes, sink, 1);
  run_stream<4096, 16>(src, bytes, sink, 1);
  run_stream<16384, 4>(src, bytes, sink, 2);
  run_stream<16384, 8>(src, 1ull << 30, sink, 1);  // HBM resident
  run_tma(src, sink);
  run_mma<64>(sink);
  run_mma<128>(sink);
  run_mma<256>(sink);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}

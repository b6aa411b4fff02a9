// commit_latency.cu -- latency of tcgen05.commit -> mbarrier arrive as seen by
// a waiting thread: (a) nothing pending, (b) after one 128x64x32 i8 MMA,
// (c) after 18 MMAs (one layer-1 conv tile), (d) a plain mbarrier.arrive.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o commit_latency commit_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2008_05101_b200/csrc/tk_sm100.cuh"

__global__ void k(unsigned long long* out) {
  __shared__ __align__(1024) uint8_t sm[32 * 1024];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    sm100::mbar_init(&bar, 1);
    sm100::fence_mbar_init();
  }
  if (warp == 0) sm100::tmem_alloc<128>(&tslot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t a = sm100::smem_u32(sm), b = a + 128 * 32;
    const uint64_t ad = sm100::desc_k_noswz(a, 128 * 16, 128), bd = sm100::desc_k_noswz(b, 64 * 16, 128);
    constexpr uint32_t idesc = sm100::idesc_i8(128, 64);
    uint32_t phase = 0;
    for (int mode = 0; mode < 4; ++mode) {
      long long best = 1ll << 60, sum = 0;
      for (int rep = 0; rep < 64; ++rep) {
        long long t0 = clock64();
        if (mode == 3) {
          sm100::mbar_arrive(&bar);
        } else {
          const int n = mode == 0 ? 0 : (mode == 1 ? 1 : 18);
          for (int i = 0; i < n; ++i) sm100::mma_i8(tmem, ad, bd, idesc, i > 0);
          sm100::mma_commit(&bar);
        }
        sm100::mbar_wait(&bar, phase);
        phase ^= 1;
        long long dt = clock64() - t0;
        best = dt < best ? dt : best;
        sum += dt;
      }
      out[blockIdx.x * 8 + mode * 2] = best;
      out[blockIdx.x * 8 + mode * 2 + 1] = sum / 64;
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc<128>(tmem);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8 * 8);
  k<<<148, 128>>>(d);
  cudaDeviceSynchronize();
  unsigned long long h[8];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const char* names[4] = {"commit_nothing_pending", "commit_after_1_mma", "commit_after_18_mma", "plain_arrive"};
  for (int m = 0; m < 4; ++m)
    printf("{\"case\": \"%s\", \"best_clk\": %llu, \"avg_clk\": %llu}\n", names[m], h[2 * m], h[2 * m + 1]);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

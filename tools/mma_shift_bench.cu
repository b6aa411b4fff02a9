// mma_shift_bench.cu -- tcgen05.mma kind::i8 issue rate when the A operand
// descriptor starts at a row-shifted (non swizzle-atom aligned) address, as
// the implicit-im2col conv does for each kernel tap.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_shift_bench mma_shift_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2008_05101_b200/csrc/tk_sm100.cuh"

__device__ __forceinline__ uint64_t desc_sw(uint32_t saddr, int R) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((8 * R) >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(R == 128 ? 2 : 4) << 61;
  return d;
}

template <int N, int R>
__global__ void k(int iters, int shift_mode, unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t done;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    sm100::mbar_init(&done, 1);
    sm100::fence_mbar_init();
  }
  for (int i = threadIdx.x; i < (256 + N) * R; i += blockDim.x) sm[i] = (uint8_t)(i * 13);
  if (warp == 0) sm100::tmem_alloc<256>(&tslot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t a = sm100::smem_u32(sm), b = a + 256 * R;
    constexpr uint32_t idesc = sm100::idesc_i8(128, N);
    const int shifts[9] = {0, 1, 2, 58, 59, 60, 116, 117, 118};
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int s = shift_mode ? shifts[i % 9] : 0;
#pragma unroll
      for (int kk = 0; kk < R / 32; ++kk)
        sm100::mma_i8(tmem, desc_sw(a + s * R + kk * 32, R), desc_sw(b + kk * 32, R), idesc, (i | kk) > 0);
    }
    sm100::mma_commit(&done);
    sm100::mbar_wait(&done, 0);
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc<256>(tmem);
}

template <int N, int R>
void run(unsigned long long* d, int mode) {
  const int iters = 4000, smem = (256 + N) * R + 2048;
  cudaFuncSetAttribute(k<N, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<N, R><<<148, 128, smem>>>(iters, mode, d);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const double mmas = (double)iters * (R / 32);
  printf("{\"N\": %d, \"R\": %d, \"shifted\": %d, \"clk_per_mma\": %.2f, \"mac_per_clk\": %.0f, \"err\": \"%s\"}\n",
         N, R, mode, avg / mmas, 128.0 * N * 32 * mmas / avg, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  for (int mode = 0; mode < 2; ++mode) {
    run<64, 64>(d, mode);
    run<128, 64>(d, mode);
    run<64, 128>(d, mode);
    run<128, 128>(d, mode);
    run<256, 128>(d, mode);
  }
  return 0;
}

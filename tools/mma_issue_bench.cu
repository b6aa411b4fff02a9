// mma_issue_bench.cu -- how the issuing code shape bounds tcgen05.mma kind::i8
// throughput for small N (the implicit-im2col conv issues 9 taps x R/32
// MMAs per item, each with a different row-shifted A descriptor).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_issue_bench mma_issue_bench.cu
// Variants (all M=128, SW64 (R=64) or SW128 (R=128) K-major operands):
//   0 constant descriptors (tensor-pipe bound)
//   1 per-MMA descriptor arithmetic in a single-thread loop (the old style)
//   2 18 descriptors precomputed into registers, unrolled issue
//   3 whole-warp loop, elect.sync inside the asm (kernel style)
//   4 descriptor deltas added to a base descriptor (64-bit add), single thread
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

__device__ constexpr int kShift[9] = {0, 1, 2, 58, 59, 60, 116, 117, 118};

template <int N, int R, int V>
__global__ void k(int iters, unsigned long long* out) {
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
  constexpr uint32_t idesc = sm100::idesc_i8(128, N);
  constexpr int KS = R / 32;
  const uint32_t a = sm100::smem_u32(sm), b = a + 256 * R;
  long long t0 = 0, t1 = 0;
  if (V == 3) {
    if (warp == 0) {
      t0 = clock64();
      for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int t = 0; t < 9; ++t)
#pragma unroll
          for (int kk = 0; kk < KS; ++kk)
            sm100::mma_i8_elect(tmem, desc_sw(a + kShift[t] * R + kk * 32, R), desc_sw(b + kk * 32, R), idesc,
                                (i | t | kk) > 0);
      }
      sm100::mma_commit_elect(&done);
      sm100::mbar_wait(&done, 0);
      t1 = clock64();
    }
  } else if (threadIdx.x == 0) {
    uint64_t ad[9 * KS], bd[KS];
#pragma unroll
    for (int t = 0; t < 9; ++t)
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) ad[t * KS + kk] = desc_sw(a + kShift[t] * R + kk * 32, R);
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) bd[kk] = desc_sw(b + kk * 32, R);
    const uint64_t abase = desc_sw(a, R), bbase = desc_sw(b, R);
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int t = 0; t < 9; ++t)
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
          uint64_t da, db;
          if (V == 0) {
            da = abase;
            db = bbase;
          } else if (V == 1) {
            da = desc_sw(a + kShift[t] * R + kk * 32, R);
            db = desc_sw(b + kk * 32, R);
          } else if (V == 2) {
            da = ad[t * KS + kk];
            db = bd[kk];
          } else {
            da = abase + (uint64_t)((kShift[t] * R + kk * 32) >> 4);
            db = bbase + (uint64_t)((kk * 32) >> 4);
          }
          sm100::mma_i8(tmem, da, db, idesc, (i | t | kk) > 0);
        }
    }
    sm100::mma_commit(&done);
    sm100::mbar_wait(&done, 0);
    t1 = clock64();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc<256>(tmem);
}

template <int N, int R, int V>
void run(unsigned long long* d) {
  const int iters = 400, smem = (256 + N) * R + 2048;
  cudaFuncSetAttribute(k<N, R, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<N, R, V><<<148, 128, smem>>>(iters, d);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const double mmas = (double)iters * 9 * (R / 32);
  printf("{\"variant\": %d, \"N\": %d, \"R\": %d, \"clk_per_mma\": %.2f, \"mac_per_clk\": %.0f, \"err\": \"%s\"}\n", V,
         N, R, avg / mmas, 128.0 * N * 32 * mmas / avg, cudaGetErrorString(cudaGetLastError()));
}

template <int V>
void run_all(unsigned long long* d) {
  run<64, 64, V>(d);
  run<128, 64, V>(d);
  run<128, 128, V>(d);
  run<256, 128, V>(d);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  run_all<0>(d);
  run_all<1>(d);
  run_all<2>(d);
  run_all<3>(d);
  run_all<4>(d);
  return 0;
}

// mbar_pingpong.cu -- round-trip latency of an mbarrier hand-off between two
// warps of one CTA (the producer/MMA/epilogue hand-off of the conv kernel),
// waiting with (0) try_wait loop, (1) test_wait spin, (2) try_wait with a
// suspend-time hint.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbar_pingpong mbar_pingpong.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2008_05101_b200/csrc/tk_sm100.cuh"

__device__ __forceinline__ void wait_mode(uint64_t* bar, uint32_t parity, int mode) {
  const uint32_t a = sm100::smem_u32(bar);
  if (mode == 0) {
    sm100::mbar_wait(bar, parity);
  } else if (mode == 1) {
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\n"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra W_%=;\n}\n" ::"r"(a),
        "r"(parity)
        : "memory");
  } else {
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra W_%=;\n}\n" ::"r"(a),
        "r"(parity), "r"(20000)
        : "memory");
  }
}

__global__ void k(int iters, int mode, unsigned long long* out) {
  __shared__ __align__(8) uint64_t ping, pong;
  if (threadIdx.x == 0) {
    sm100::mbar_init(&ping, 1);
    sm100::mbar_init(&pong, 1);
    sm100::fence_mbar_init();
  }
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (lane != 0) return;
  if (warp == 0) {
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      sm100::mbar_arrive(&ping);
      wait_mode(&pong, i & 1, mode);
    }
    out[blockIdx.x] = (clock64() - t0) / iters;
  } else if (warp == 1) {
    for (int i = 0; i < iters; ++i) {
      wait_mode(&ping, i & 1, mode);
      sm100::mbar_arrive(&pong);
    }
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  for (int mode = 0; mode < 3; ++mode) {
    k<<<148, 64>>>(20000, mode, d);
    cudaDeviceSynchronize();
    unsigned long long h;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("{\"wait\": \"%s\", \"round_trip_clk\": %llu, \"err\": \"%s\"}\n",
           mode == 0 ? "try_wait" : (mode == 1 ? "test_wait_spin" : "try_wait_hint20us"), h,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}

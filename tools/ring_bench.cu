// ring_bench.cu -- the conv kernel's three-role hand-off skeleton with no
// work: producer -> (ring of S stages) -> consumer -> (ring of A buffers) ->
// epilogue warps.  Per-item cost of the synchronisation alone.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ring_bench ring_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2008_05101_b200/csrc/tk_sm100.cuh"

template <int S, int A, int EPI_WARPS, int FENCE>
__global__ void k(int items, unsigned long long* out) {
  __shared__ __align__(8) uint64_t full[S], empty[S], afull[A], aempty[A];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) { sm100::mbar_init(&full[i], 1); sm100::mbar_init(&empty[i], 1); }
    for (int i = 0; i < A; ++i) { sm100::mbar_init(&afull[i], 1); sm100::mbar_init(&aempty[i], EPI_WARPS * 32); }
    sm100::fence_mbar_init();
  }
  __syncthreads();
  long long t0 = clock64();
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < items; ++i) {
      const int s = i % S;
      if (i >= S) sm100::mbar_wait(&empty[s], ((i / S) - 1) & 1);
      sm100::mbar_arrive(&full[s]);
    }
  } else if (warp == 1 && lane == 0) {
    for (int i = 0; i < items; ++i) {
      const int s = i % S, a = i % A;
      if (i >= A) sm100::mbar_wait(&aempty[a], ((i / A) - 1) & 1);
      sm100::mbar_wait(&full[s], (i / S) & 1);
      if (FENCE) sm100::tc_fence_after();
      sm100::mbar_arrive(&empty[s]);
      sm100::mbar_arrive(&afull[a]);
    }
    out[blockIdx.x] = (clock64() - t0) / items;
  } else if (warp >= 2 && warp < 2 + EPI_WARPS) {
    for (int i = 0; i < items; ++i) {
      const int a = i % A;
      sm100::mbar_wait(&afull[a], (i / A) & 1);
      if (FENCE) { sm100::tc_fence_after(); sm100::tc_fence_before(); }
      sm100::mbar_arrive(&aempty[a]);
    }
  }
}

template <int S, int A, int E, int F = 0>
void run() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  k<S, A, E, F><<<148, 64 + 32 * E>>>(20000, d);
  cudaDeviceSynchronize();
  unsigned long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("{\"fence\": %d, \"stages\": %d, \"acc\": %d, \"epi_warps\": %d, \"clk_per_item\": %llu, \"err\": \"%s\"}\n", F, S, A, E, h,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<4, 4, 1>();
  run<4, 4, 4>();
  run<4, 4, 8>();
  run<2, 2, 8>();
  run<4, 4, 8, 1>();
  return 0;
}

// launch_bench.cu -- fixed per-launch costs of a tcgen05 GEMM skeleton on
// B200: graph-replayed back-to-back launches of 128 CTAs x 192 threads with
// (a) nothing, (b) ~200 KB dynamic shared memory, (c) a (1,1,4) cluster,
// (d) + TMEM alloc/dealloc, (e) + mbarrier init and a cluster barrier.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o launch_bench launch_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2008_05101_b200/csrc/tk_sm100.cuh"

template <int V>
__global__ void __launch_bounds__(192, 1) k(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb,
                                            int* sink) {
  extern __shared__ uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar[8];
  if (V >= 3) {
    if (threadIdx.x / 32 == 1) sm100::tmem_alloc<256>(&slot);
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
  }
  if (V >= 4) {
    if (threadIdx.x == 0) {
      for (int i = 0; i < 8; ++i) sm100::mbar_init(&bar[i], 1);
      sm100::fence_mbar_init();
    }
    __syncthreads();
    sm100::cluster_sync();
  }
  if (V >= 5 && threadIdx.x == 0) {
    sm100::tma_prefetch(&ma);
    sm100::tma_prefetch(&mb);
  }
  if (V >= 6 && threadIdx.x == 0) {  // 8 empty commit round trips
    for (int i = 0; i < 8; ++i) {
      sm100::mma_commit(&bar[i]);
      sm100::mbar_wait(&bar[i], 0);
    }
  }
  if (V >= 7 && sink[0] == 0x7fffffff) {  // large, never-executed body: instruction-cache footprint
    float a = threadIdx.x;
#pragma unroll
    for (int i = 0; i < 3000; ++i) a = __fmaf_rn(a, 1.0001f, (float)i);
    sink[1] = (int)a;
  }
  if (threadIdx.x == 0 && sink[blockIdx.x] == 12345) sink[0] = smem[0];
  if (V >= 3) {
    __syncthreads();
    if (threadIdx.x / 32 == 1) sm100::tmem_dealloc<256>(slot);
  }
}

template <int V>
float run(int* sink, int smem, int cluster) {
  cudaFuncSetAttribute(k<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(32, 1, 4);
  cfg.blockDim = dim3(192, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = cluster;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaStream_t s;
  cudaStreamCreate(&s);
  cfg.stream = s;
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  CUtensorMap m{};
  for (int i = 0; i < 20; ++i) cudaLaunchKernelEx(&cfg, k<V>, m, m, sink);
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1e3f / 200;
}

int main() {
  int* sink;
  cudaMalloc(&sink, 1 << 20);
  cudaMemset(sink, 0, 1 << 20);
  printf("empty, 0 smem, no cluster:      %.2f us/launch\n", run<0>(sink, 0, 1));
  printf("empty, 200 KB smem:             %.2f us/launch\n", run<0>(sink, 200 * 1024, 1));
  printf("empty, 200 KB smem, cluster 4:  %.2f us/launch\n", run<0>(sink, 200 * 1024, 4));
  printf("+ TMEM alloc, cluster 4:        %.2f us/launch\n", run<3>(sink, 200 * 1024, 4));
  printf("+ mbar init + cluster barrier:  %.2f us/launch\n", run<4>(sink, 200 * 1024, 4));
  printf("+ TMEM alloc, no cluster:       %.2f us/launch\n", run<3>(sink, 200 * 1024, 1));
  printf("+ tensormap prefetch:           %.2f us/launch\n", run<5>(sink, 200 * 1024, 4));
  printf("+ 8 empty commit round trips:   %.2f us/launch\n", run<6>(sink, 200 * 1024, 4));
  printf("V6 with 225 KB smem:            %.2f us/launch\n", run<6>(sink, 225 * 1024, 4));
  printf("V6 + 48 KB of (dead) code:      %.2f us/launch\n", run<7>(sink, 225 * 1024, 4));
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

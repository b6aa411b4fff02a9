// dsmem_bench.cu -- distributed-shared-memory throughput inside a (1,1,4)
// cluster on B200, 128 CTAs x 192 threads, 128 KB moved per CTA:
//   push: st.shared::cluster.v4 from 128 threads to the next rank
//   pull: ld.shared::cluster.v4 by 192 threads from the next rank
//   bulk: one cp.async.bulk shared::cta -> shared::cluster per 32 KB chunk
//   local: plain st.shared.v4 (reference)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem_bench dsmem_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2008_05101_b200/csrc/tk_sm100.cuh"

constexpr int kBytes = 128 * 1024;

template <int V>
__global__ void __launch_bounds__(192, 1) k(unsigned long long* out, int reps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t rank = sm100::cluster_ctarank();
  const uint32_t peer = (rank + 1) & 3;
  const uint32_t base = sm100::smem_u32(smem);
  if (threadIdx.x == 0) {
    sm100::mbar_init(&bar, 1);
    sm100::fence_mbar_init();
  }
  for (int i = threadIdx.x; i < kBytes / 4 + 16384 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = i;
  __syncthreads();
  sm100::cluster_sync();
  unsigned long long t0 = clock64();
  uint32_t acc = 0;
  for (int r = 0; r < reps; ++r) {
    if (V == 0) {  // push
      if (threadIdx.x >= 64) {
        const int t = threadIdx.x - 64;
        for (int i = t; i < kBytes / 16; i += 128)
          sm100::st_cluster_v4(base + i * 16, peer, make_uint4(i, r, 1, 2));
      }
    } else if (V == 1) {  // pull
      for (int i = threadIdx.x; i < kBytes / 16; i += 192) {
        const uint4 v = sm100::ld_cluster_v4(base + i * 16, peer);
        acc += v.x ^ v.w;
      }
    } else if (V == 2) {  // bulk copies, 4 x 32 KB
      if (threadIdx.x == 0) {
        sm100::mbar_arrive_expect_tx(&bar, kBytes);
        for (int c = 0; c < 4; ++c) {
          uint32_t remote_bar;
          // copy my chunk c into my own buffer region of the peer; completion on the PEER's barrier is
          // the usual pattern -- here each CTA receives from rank-1, so arm locally and signal locally
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote_bar) : "r"(sm100::smem_u32(&bar)), "r"(peer));
          uint32_t dst;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(dst) : "r"(base + c * 32768), "r"(peer));
          asm volatile(
              "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
              "r"(base + kBytes + 0), "r"(16384), "r"(remote_bar)
              : "memory");
          asm volatile(
              "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst + 16384),
              "r"(base + kBytes + 0), "r"(16384), "r"(remote_bar)
              : "memory");
        }
        sm100::mbar_wait(&bar, r & 1);
      }
    } else {  // local stores
      for (int i = threadIdx.x; i < kBytes / 16; i += 192)
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(base + i * 16), "r"(i), "r"(r), "r"(1), "r"(2)
                     : "memory");
    }
    sm100::cluster_sync();
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x + blockIdx.z * gridDim.x] = t1 - t0;
  if (acc == 0xdeadbeef) out[0] = acc;
}

template <int V>
void run(const char* name, unsigned long long* d) {
  const int smem = kBytes + 16384 + 1024;
  cudaFuncSetAttribute(k<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(32, 1, 4);
  cfg.blockDim = dim3(192, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 4;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const int reps = 20;
  cudaLaunchKernelEx(&cfg, k<V>, d, reps);
  cudaDeviceSynchronize();
  unsigned long long h[128];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 128; ++i) avg += h[i];
  avg /= 128;
  printf("%-6s %.0f clk per 128 KB per CTA = %.1f B/clk/SM  (%s)\n", name, avg / reps, kBytes * reps / avg,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 4096 * 8);
  run<3>("local", d);
  run<0>("push", d);
  run<1>("pull", d);
  run<2>("bulk", d);
  return 0;
}

// pipe_bench.cu -- measures the integer pipes the LOP3+POPC GEMM is bound by
// (POPC and LOP3 results per clock per SM) on the B200 it runs on.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_bench pipe_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(unsigned* out, int iters, unsigned seed) {
  unsigned a[8], b = seed ^ threadIdx.x, acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed * (i + 1) + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) {               // POPC of a LOP3 (the GEMM inner op)
        acc += __popc(~(a[i] ^ b) & a[(i + 1) & 7]);
        a[i] += 0x9E3779B9u;
      } else {                        // LOP3 chain only
        a[i] = (a[i] ^ b) & ~a[(i + 3) & 7];
      }
    }
    b += it;
  }
  unsigned r = acc;
#pragma unroll
  for (int i = 0; i < 8; ++i) r ^= a[i];
  if (r == 0x12345678u) out[0] = r;
}

int main() {
  unsigned* d;
  cudaMalloc(&d, 4);
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 4096, blocks = sms * 8, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<blocks, threads>>>(d, iters, rep + 1);
      else k<1><<<blocks, threads>>>(d, iters, rep + 1);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double ops = (double)blocks * threads * iters * 8;
      printf("{\"pipe\": \"%s\", \"ops_per_s\": %.4e, \"ms\": %.3f, \"per_sm_per_clk_at_max\": %.2f, "
             "\"sms\": %d, \"max_clk_khz\": %d}\n",
             mode == 0 ? "popc(lop3)" : "lop3", ops / (ms * 1e-3), ms,
             ops / (ms * 1e-3) / sms / (clk * 1e3), sms, clk);
    }
  }
  return 0;
}

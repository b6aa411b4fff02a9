// mxf4_test.cu -- feasibility of an exact ternary contraction on the FP4
// tensor-core path: tcgen05.mma kind::mxf4 with unit
// (E8M0 = 127) block scales computes sum_k a_k * w_k exactly for a in
// {0,1,2}, w in {-1,0,1} (E2M1 codes 0/1.0/2.0 and -1.0), f32 accumulate.
// One CTA, M = 128, N = 128, K = 64 (one MMA), then timing of back-to-back
// MMAs for the issue rate.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mxf4_test mxf4_test.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

#include "../paper_2008_05101_b200/csrc/tk_sm100.cuh"

constexpr int M = 128, N = 128, K = 64;

__device__ __forceinline__ uint8_t e2m1(int v) {  // -1, 0, 1, 2 -> E2M1 nibble
  return v == 0 ? 0x0 : v == 1 ? 0x2 : v == 2 ? 0x4 : 0xA;
}

__global__ void k(const int8_t* a, const int8_t* b, float* d_out, int iters, unsigned long long* clk) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sa = smem;                 // [2 chunks][M rows][16 B]
  uint8_t* sb = smem + 2 * M * 16;    // [2 chunks][N rows][16 B]
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t done;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    sm100::mbar_init(&done, 1);
    sm100::fence_mbar_init();
  }
  // pack: element k of row r -> chunk k/32, byte (k%32)/2, low nibble = even k
  for (int i = threadIdx.x; i < M * K / 2; i += blockDim.x) {
    const int r = i / (K / 2), kb = i % (K / 2), k0 = 2 * kb;
    const uint8_t lo = e2m1(a[r * K + k0]), hi = e2m1(a[r * K + k0 + 1]);
    sa[(k0 / 32) * M * 16 + r * 16 + (k0 % 32) / 2] = lo | (hi << 4);
  }
  for (int i = threadIdx.x; i < N * K / 2; i += blockDim.x) {
    const int r = i / (K / 2), kb = i % (K / 2), k0 = 2 * kb;
    const uint8_t lo = e2m1(b[r * K + k0]), hi = e2m1(b[r * K + k0 + 1]);
    sb[(k0 / 32) * N * 16 + r * 16 + (k0 % 32) / 2] = lo | (hi << 4);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) sm100::tmem_alloc<256>(&slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = slot;
  // unit scales: columns 128..191 all 0x7F (E8M0 2^0) in every lane
  {
    const uint32_t base = tmem + ((uint32_t)(warp * 32) << 16) + 128;
    for (int c = 0; c < 64; c += 4)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %1, %1, %1};" ::"r"(base + c),
                   "r"(0x7F7F7F7Fu));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  if (threadIdx.x == 0) {
    const uint64_t ad = sm100::desc_k_noswz(sm100::smem_u32(sa), M * 16, 128);
    const uint64_t bd = sm100::desc_k_noswz(sm100::smem_u32(sb), N * 16, 128);
    // block-scaled idesc: a/b format E2M1 (MXF4 = 1), scale E8M0, N, M, K64
    const uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) |
                           ((uint32_t)(M >> 4) << 24);
    const uint32_t sfa = tmem + 128, sfb = tmem + 160;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}\n" ::"r"(
              tmem),
          "l"(ad), "l"(bd), "r"(idesc), "r"(0), "r"(sfa), "r"(sfb));
    }
    sm100::mma_commit(&done);
    sm100::mbar_wait(&done, 0);
    clk[blockIdx.x] = clock64() - t0;
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  if (warp < 4) {  // D: lanes = rows, columns = n (f32)
    for (int c0 = 0; c0 < N; c0 += 32) {
      uint32_t r[32];
      sm100::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c0, r);
      sm100::tmem_ld_wait();
      for (int j = 0; j < 32; ++j) d_out[(warp * 32 + lane) * N + c0 + j] = __uint_as_float(r[j]);
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc<256>(tmem);
}

int main() {
  int8_t ha[M * K], hb[N * K];
  srand(5);
  for (int i = 0; i < M * K; ++i) ha[i] = rand() % 3;       // {0,1,2}
  for (int i = 0; i < N * K; ++i) hb[i] = rand() % 3 - 1;   // {-1,0,1}
  int8_t *da, *db;
  float* dd;
  unsigned long long* dclk;
  cudaMalloc(&da, sizeof(ha));
  cudaMalloc(&db, sizeof(hb));
  cudaMalloc(&dd, M * N * 4);
  cudaMalloc(&dclk, 8 * 148);
  cudaMemcpy(da, ha, sizeof(ha), cudaMemcpyHostToDevice);
  cudaMemcpy(db, hb, sizeof(hb), cudaMemcpyHostToDevice);
  const int smem = 2 * (M + N) * 16 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<<<1, 128, smem>>>(da, db, dd, 1, dclk);
  cudaError_t e = cudaDeviceSynchronize();
  static float hd[M * N];
  cudaMemcpy(hd, dd, sizeof(hd), cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int r = 0; r < M; ++r)
    for (int n = 0; n < N; ++n) {
      int want = 0;
      for (int kk = 0; kk < K; ++kk) want += ha[r * K + kk] * hb[n * K + kk];
      if (hd[r * N + n] != (float)want) {
        if (bad < 5) printf("mismatch r=%d n=%d got %f want %d\n", r, n, hd[r * N + n], want);
        ++bad;
      }
    }
  printf("correctness: %d mismatches of %d (%s)\n", bad, M * N, cudaGetErrorString(e));
  // issue rate: 148 CTAs x 4000 back-to-back MMAs
  k<<<148, 128, smem>>>(da, db, dd, 4000, dclk);
  e = cudaDeviceSynchronize();
  unsigned long long hc[148];
  cudaMemcpy(hc, dclk, sizeof(hc), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += hc[i];
  avg /= 148;
  printf("mxf4 128x%dx%d: %.2f clk/MMA = %.0f MAC/clk/SM (%s)\n", N, K, avg / 4000, (double)M * N * K * 4000 / avg,
         cudaGetErrorString(e));
  return 0;
}

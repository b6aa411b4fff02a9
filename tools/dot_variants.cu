// dot_variants.cu -- A/B of the cfg1 batched ternary dot (65,536 pairs x
// N = 4096 lanes = 1 KiB per operand row) against a pure streaming-read
// ceiling.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dot_variants dot_variants.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t tm(uint32_t x, uint32_t y) {
  const uint32_t d = (y ^ (y >> 1)) & 0x55555555u;
  return (~(x ^ y) | d) & ~(d << 1);
}
__device__ __forceinline__ int tm4(uint4 a, uint4 b) {
  return __popc(tm(a.x, b.x)) + __popc(tm(a.y, b.y)) + __popc(tm(a.z, b.z)) + __popc(tm(a.w, b.w));
}
__device__ __forceinline__ uint4 ldnc(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// V0: round-1 kernel (warp per pair, grid-stride)
__global__ void v0(const uint4* __restrict__ x, const uint4* __restrict__ y, size_t words, size_t pairs,
                   const int64_t* __restrict__ wsum, int64_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const size_t nwarps = ((size_t)gridDim.x * blockDim.x) >> 5;
  const size_t q = words / 2;
  for (size_t p = warp; p < pairs; p += nwarps) {
    const uint4* xp = x + p * q;
    const uint4* yp = y + p * q;
    int acc = 0;
#pragma unroll 4
    for (size_t i = lane; i < q; i += 32) acc += tm4(__ldg(xp + i), __ldg(yp + i));
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[p] = (int64_t)acc - (int64_t)words * 32 + wsum[p];
  }
}

// V1: P pairs per warp-iteration, Q = words/2 uint4 per row known at compile
// time (64 for N = 4096); all 2*P*Q/32 loads of a lane issued before use.
template <int P, int Q, bool NC>
__global__ void __launch_bounds__(256) v1(const uint4* __restrict__ x, const uint4* __restrict__ y, size_t pairs,
                                         const int64_t* __restrict__ wsum, int64_t* __restrict__ out) {
  constexpr int L = Q / 32;  // uint4 per lane per row
  const int lane = threadIdx.x & 31;
  const size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const size_t nwarps = ((size_t)gridDim.x * blockDim.x) >> 5;
  for (size_t p0 = warp * P; p0 < pairs; p0 += nwarps * P) {
    uint4 a[P][L], b[P][L];
#pragma unroll
    for (int j = 0; j < P; ++j)
#pragma unroll
      for (int i = 0; i < L; ++i) {
        const size_t p = p0 + j < pairs ? p0 + j : pairs - 1;
        const size_t off = p * Q + i * 32 + lane;
        a[j][i] = NC ? ldnc(x + off) : __ldg(x + off);
        b[j][i] = NC ? ldnc(y + off) : __ldg(y + off);
      }
    int acc[P];
#pragma unroll
    for (int j = 0; j < P; ++j) {
      acc[j] = 0;
#pragma unroll
      for (int i = 0; i < L; ++i) acc[j] += tm4(a[j][i], b[j][i]);
    }
#pragma unroll
    for (int j = 0; j < P; ++j)
#pragma unroll
      for (int o = 16; o; o >>= 1) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
    if (lane < P && p0 + lane < pairs) {
      int v = acc[0];
#pragma unroll
      for (int j = 1; j < P; ++j) v = lane == j ? acc[j] : v;
      out[p0 + lane] = (int64_t)v - (int64_t)Q * 2 * 32 + wsum[p0 + lane];
    }
  }
}

// ceiling: read both operand arrays once, no math beyond an XOR fold
template <int U>
__global__ void __launch_bounds__(256) ceil_read(const uint4* __restrict__ x, const uint4* __restrict__ y, size_t n,
                                                int* __restrict__ sink) {
  const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const size_t nt = (size_t)gridDim.x * blockDim.x;
  uint32_t acc = 0;
  for (size_t i = t; i < n; i += nt * U) {
    uint4 a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t k = i + u * nt < n ? i + u * nt : i;
      a[u] = ldnc(x + k);
      b[u] = ldnc(y + k);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= a[u].x ^ a[u].w ^ b[u].y ^ b[u].z;
  }
  if (acc == 0x12345678u) *sink = 1;
}

int main() {
  const size_t pairs = 65536, words = 128, q = 64;
  const size_t bytes = pairs * words * 8;
  std::vector<uint64_t> hx(pairs * words), hy(pairs * words);
  uint64_t s = 88172645463325252ull;
  auto rnd = [&] { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; };
  for (auto& v : hx) v = rnd();
  for (auto& v : hy) v = rnd();
  std::vector<int64_t> hw(pairs);
  for (auto& v : hw) v = (int64_t)(rnd() % 1000);
  uint4 *x, *y;
  int64_t *w, *o, *o2;
  int* sink;
  CK(cudaMalloc(&x, bytes));
  CK(cudaMalloc(&y, bytes));
  CK(cudaMalloc(&w, pairs * 8));
  CK(cudaMalloc(&o, pairs * 8));
  CK(cudaMalloc(&o2, pairs * 8));
  CK(cudaMalloc(&sink, 4));
  CK(cudaMemcpy(x, hx.data(), bytes, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(y, hy.data(), bytes, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(w, hw.data(), pairs * 8, cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double alg = pairs * (2.0 * words * 8 + 16);
  auto timeit = [&](const char* name, auto launch, bool check) {
    for (int i = 0; i < 3; ++i) launch();
    cudaDeviceSynchronize();
    const int n = 50;
    cudaEventRecord(e0);
    for (int i = 0; i < n; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1e3 / n;
    bool ok = true;
    if (check) {
      std::vector<int64_t> a(pairs), b(pairs);
      cudaMemcpy(a.data(), o, pairs * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(b.data(), o2, pairs * 8, cudaMemcpyDeviceToHost);
      ok = a == b;
    }
    printf("%-28s %8.2f us  %7.1f GB/s  %s\n", name, us, alg / us / 1e3, check ? (ok ? "ok" : "MISMATCH") : "");
  };
  const int sms = 148;
  v0<<<148 * 32, 256>>>(x, y, words, pairs, w, o2);  // reference result
  CK(cudaDeviceSynchronize());
  timeit("v0 round-1", [&] { v0<<<sms * 32, 256>>>(x, y, words, pairs, w, o); }, true);
  timeit("v0 no-stride", [&] { v0<<<(unsigned)(pairs / 8), 256>>>(x, y, words, pairs, w, o); }, true);
  for (int gm : {8, 16, 32}) {
    char nm[64];
    snprintf(nm, 64, "v1 P1 ldg g%d", gm);
    timeit(nm, [&] { v1<1, 64, false><<<sms * gm, 256>>>(x, y, pairs, w, o); }, true);
    snprintf(nm, 64, "v1 P2 ldg g%d", gm);
    timeit(nm, [&] { v1<2, 64, false><<<sms * gm, 256>>>(x, y, pairs, w, o); }, true);
    snprintf(nm, 64, "v1 P2 nc g%d", gm);
    timeit(nm, [&] { v1<2, 64, true><<<sms * gm, 256>>>(x, y, pairs, w, o); }, true);
    snprintf(nm, 64, "v1 P4 nc g%d", gm);
    timeit(nm, [&] { v1<4, 64, true><<<sms * gm, 256>>>(x, y, pairs, w, o); }, true);
  }
  timeit("v1 P1 nc full grid", [&] { v1<1, 64, true><<<(unsigned)(pairs / 8), 256>>>(x, y, pairs, w, o); }, true);
  timeit("v1 P2 nc full grid", [&] { v1<2, 64, true><<<(unsigned)(pairs / 16), 256>>>(x, y, pairs, w, o); }, true);
  for (int gm : {8, 16, 32}) {
    char nm[64];
    snprintf(nm, 64, "ceiling U4 g%d", gm);
    timeit(nm, [&] { ceil_read<4><<<sms * gm, 256>>>(x, y, bytes / 16, sink); }, false);
    snprintf(nm, 64, "ceiling U8 g%d", gm);
    timeit(nm, [&] { ceil_read<8><<<sms * gm, 256>>>(x, y, bytes / 16, sink); }, false);
  }
  return 0;
}

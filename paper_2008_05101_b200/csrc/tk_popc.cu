// tk_popc.cu -- the LOP3 + POPC integer-pipe path.
//
// Ternary multiply (R:bitkernels.hpp:55-63) on a word pair is
//   TM(x, y) = (~(x ^ y) | d) & ~(d << 1),  d = (y ^ y >> 1) & kAuxi,
// and for every lane popcount(TM) = popcount(~(x^y) & M) + [lane of y is 0]
// with M = ~(d | d << 1).  Summed over a row:
//   dot = sum_w popc(~(x_w ^ y_w) & M_w) + Z_y - 32 * words
// where Z_y counts the zero lanes of the weight row (padding included).
// M and Z are per weight row, precomputed once at layer creation, so the
// inner loop is one LOP3 + one POPC + half an IADD3 per u32 word.
#include <algorithm>

#include "tk_internal.cuh"

namespace {

__device__ __forceinline__ uint32_t tm_u32(uint32_t x, uint32_t y) {
  const uint32_t d = (y ^ (y >> 1)) & TK_KAUXI32;
  return (~(x ^ y) | d) & ~(d << 1);
}

// TM with the zero seed supplied (R:bitkernels.hpp:66-72, premask form)
__device__ __forceinline__ uint32_t tm_seed_u32(uint32_t x, uint32_t y, uint32_t d) {
  return (~(x ^ y) | d) & ~(d << 1);
}

template <bool kSeed>
__device__ __forceinline__ int tm_popc4(const uint4& a, const uint4& b, const uint4& d) {
  if constexpr (kSeed)
    return __popc(tm_seed_u32(a.x, b.x, d.x)) + __popc(tm_seed_u32(a.y, b.y, d.y)) +
           __popc(tm_seed_u32(a.z, b.z, d.z)) + __popc(tm_seed_u32(a.w, b.w, d.w));
  else
    return __popc(tm_u32(a.x, b.x)) + __popc(tm_u32(a.y, b.y)) + __popc(tm_u32(a.z, b.z)) +
           __popc(tm_u32(a.w, b.w));
}

// cfg1: one warp per vector pair, R:bitkernels.hpp:76-97 (+ :151-159).
// Streaming-bound (no reuse): a lane issues all loads of a 4 x 16 B chunk of
// each operand before using any, so a warp keeps (2 or 3) x 2 KB in flight
// (tools/dot_variants.cu: 5.99 TB/s on cfg1, the read ceiling of this box;
// the round-1 runtime-trip-count loop kept half that in flight, 4.93 TB/s).
template <bool kSeed>
__global__ void __launch_bounds__(256) k_dot_batched(const uint4* __restrict__ x, const uint4* __restrict__ y,
                                                     const uint4* __restrict__ seed, size_t words, size_t pairs,
                                                     const int64_t* __restrict__ wsum, int64_t* __restrict__ out) {
  constexpr int U = 4;  // uint4 per lane per operand in flight
  const int lane = threadIdx.x & 31;
  const size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const size_t nwarps = ((size_t)gridDim.x * blockDim.x) >> 5;
  const size_t q = words / 2;  // uint4 = 2 u64 words
  for (size_t p = warp; p < pairs; p += nwarps) {
    const uint4* xp = x + p * q;
    const uint4* yp = y + p * q;
    const uint4* dp = kSeed ? seed + p * q : nullptr;
    int acc = 0;
    for (size_t base = 0; base < q; base += 32 * U) {
      uint4 a[U], b[U], d[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t i = base + u * 32 + lane;
        if (i < q) {
          a[u] = __ldg(xp + i);
          b[u] = __ldg(yp + i);
          if constexpr (kSeed) d[u] = __ldg(dp + i);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (base + u * 32 + lane < q) acc += tm_popc4<kSeed>(a[u], b[u], d[u]);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      const int64_t r = (int64_t)acc - (int64_t)words * 32;
      out[p] = wsum ? r + wsum[p] : r;
    }
  }
}

// Rows of exactly 32 * L uint4 (N = 2048 / 4096 / 8192 lanes: the cfg1 row
// is L = 2): the trip count is a compile-time constant, so every load of a
// lane is issued before any use with no predication (tools/dot_variants.cu
// "v1 P1": 5.99 TB/s on cfg1 vs 4.93 for a runtime-bounded loop).
template <int L, bool kSeed>
__global__ void __launch_bounds__(256) k_dot_fixed(const uint4* __restrict__ x, const uint4* __restrict__ y,
                                                   const uint4* __restrict__ seed, size_t pairs,
                                                   const int64_t* __restrict__ wsum, int64_t* __restrict__ out) {
  constexpr int Q = 32 * L;
  const int lane = threadIdx.x & 31;
  const size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const size_t nwarps = ((size_t)gridDim.x * blockDim.x) >> 5;
  for (size_t p = warp; p < pairs; p += nwarps) {
    uint4 a[L], b[L], d[L];
#pragma unroll
    for (int i = 0; i < L; ++i) {
      a[i] = __ldg(x + p * Q + i * 32 + lane);
      b[i] = __ldg(y + p * Q + i * 32 + lane);
      if constexpr (kSeed) d[i] = __ldg(seed + p * Q + i * 32 + lane);
    }
    int acc = 0;
#pragma unroll
    for (int i = 0; i < L; ++i) acc += tm_popc4<kSeed>(a[i], b[i], d[i]);
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      const int64_t r = (int64_t)acc - (int64_t)Q * 2 * 32;
      out[p] = wsum ? r + wsum[p] : r;
    }
  }
}

// odd word counts: scalar u64 variant
template <bool kSeed>
__global__ void k_dot_batched_u64(const uint64_t* __restrict__ x, const uint64_t* __restrict__ y,
                                  const uint64_t* __restrict__ seed, size_t words, size_t pairs,
                                  const int64_t* __restrict__ wsum, int64_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const size_t nwarps = ((size_t)gridDim.x * blockDim.x) >> 5;
  for (size_t p = warp; p < pairs; p += nwarps) {
    int acc = 0;
    for (size_t i = lane; i < words; i += 32) {
      const uint64_t a = x[p * words + i], b = y[p * words + i];
      if constexpr (kSeed) {
        const uint64_t d = seed[p * words + i];
        acc += __popc(tm_seed_u32((uint32_t)a, (uint32_t)b, (uint32_t)d)) +
               __popc(tm_seed_u32((uint32_t)(a >> 32), (uint32_t)(b >> 32), (uint32_t)(d >> 32)));
      } else {
        acc += __popc(tm_u32((uint32_t)a, (uint32_t)b)) + __popc(tm_u32((uint32_t)(a >> 32), (uint32_t)(b >> 32)));
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      const int64_t r = (int64_t)acc - (int64_t)words * 32;
      out[p] = wsum ? r + wsum[p] : r;
    }
  }
}

// ---------------------------------------------------------------------------
// Register-tiled packed GEMM: C[m][n] = sum_k popc(~(A[m][k]^B[n][k]) & M[n][k])
// + cst[n].  CTA tile 64 x 64, 256 threads, 4 x 4 outputs per thread, K staged
// through shared memory 16 u32 words at a time (k-major so each thread reads
// its 4 rows / 4 columns with one LDS.128).  R:linalg.hpp:232-293.
constexpr int BM = 64, BN = 64, BK = 16;

__global__ void __launch_bounds__(256)
k_gemm_popc(const uint32_t* __restrict__ A, int M, int K32,
            const uint32_t* __restrict__ B, const uint32_t* __restrict__ Mk,
            int N, const int32_t* __restrict__ wsum,
            const int32_t* __restrict__ zcnt, int offset, tk_epilogue e) {
  __shared__ __align__(16) uint32_t As[BK][BM];
  __shared__ __align__(16) uint32_t Bs[BK][BN];
  __shared__ __align__(16) uint32_t Ms[BK][BN];

  const int tid = threadIdx.x;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int tx = tid & 15, ty = tid >> 4;  // 16 x 16 threads
  const int lr = tid >> 2, lk = (tid & 3) * 4;  // loader: row, k quad

  int acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0;

  const bool vec = (K32 % 4) == 0;
  for (int k0 = 0; k0 < K32; k0 += BK) {
    // ---- load tiles (zero outside the matrix: popc(~(0^0)&0) = 0) ----
    uint32_t a4[4] = {0, 0, 0, 0}, b4[4] = {0, 0, 0, 0}, m4[4] = {0, 0, 0, 0};
    const int gm = m0 + lr, gn = n0 + lr, gk = k0 + lk;
    if (vec && gk + 3 < K32) {
      if (gm < M) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(A + (size_t)gm * K32 + gk));
        a4[0] = v.x; a4[1] = v.y; a4[2] = v.z; a4[3] = v.w;
      }
      if (gn < N) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(B + (size_t)gn * K32 + gk));
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(Mk + (size_t)gn * K32 + gk));
        b4[0] = v.x; b4[1] = v.y; b4[2] = v.z; b4[3] = v.w;
        m4[0] = u.x; m4[1] = u.y; m4[2] = u.z; m4[3] = u.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (gk + i < K32) {
          if (gm < M) a4[i] = A[(size_t)gm * K32 + gk + i];
          if (gn < N) {
            b4[i] = B[(size_t)gn * K32 + gk + i];
            m4[i] = Mk[(size_t)gn * K32 + gk + i];
          }
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      As[lk + i][lr] = a4[i];
      Bs[lk + i][lr] = b4[i];
      Ms[lk + i][lr] = m4[i];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      const uint4 a = *reinterpret_cast<const uint4*>(&As[k][ty * 4]);
      const uint4 b = *reinterpret_cast<const uint4*>(&Bs[k][tx * 4]);
      const uint4 m = *reinterpret_cast<const uint4*>(&Ms[k][tx * 4]);
      const uint32_t av[4] = {a.x, a.y, a.z, a.w};
      const uint32_t bv[4] = {b.x, b.y, b.z, b.w};
      const uint32_t mv[4] = {m.x, m.y, m.z, m.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          acc[i][j] += __popc(~(av[i] ^ bv[j]) & mv[j]);
    }
  }

  // ---- epilogue ----
  const int words64 = K32 / 2;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int n = n0 + tx * 4 + j;
    if (n >= N) continue;
    const int cst = zcnt[n] - 32 * words64 + (offset ? wsum[n] : 0);
    const float g = e.gain ? e.gain[n] : 1.0f;
    const float bb = e.bias ? e.bias[n] : 0.0f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int m = m0 + ty * 4 + i;
      if (m >= M) continue;
      const int v = acc[i][j] + cst;
      if (e.mode == TK_EPI_I32) {
        static_cast<int32_t*>(e.out)[(size_t)m * N + n] = v;
      } else {
        // R:linalg.hpp:322-323, contracted to one FMA like the reference build
        const float y = __fmaf_rn(g, __fmul_rn(e.out_scale, (float)v), bb);
        if (e.mode == TK_EPI_F32_ROWS) {
          static_cast<float*>(e.out)[(size_t)m * N + n] = y;
        } else {
          const int b = m / e.plane, p = m - b * e.plane;
          static_cast<float*>(e.out)[((size_t)b * N + n) * e.plane + p] = y;
        }
      }
    }
  }
}

}  // namespace

cudaError_t tk_launch_dot_batched(const uint64_t* x, const uint64_t* y, const uint64_t* seed, size_t words,
                                  size_t pairs, const int64_t* wsum, int64_t* out, cudaStream_t s) {
  if (pairs == 0) return cudaSuccess;
  // 8 warps per block, up to 16 resident-block waves of the 148 SMs
  const size_t blocks = std::min<size_t>((pairs + 7) / 8, 148u * 16u);
  const bool vec = words % 2 == 0 && ((uintptr_t)x % 16 == 0) && ((uintptr_t)y % 16 == 0) &&
                   ((uintptr_t)seed % 16 == 0);
  auto v4 = [](const uint64_t* p) { return reinterpret_cast<const uint4*>(p); };
  if (vec && (words == 64 || words == 128 || words == 256)) {
    auto go = [&](auto kern) {
      kern<<<(unsigned)blocks, 256, 0, s>>>(v4(x), v4(y), seed ? v4(seed) : nullptr, pairs, wsum, out);
    };
    if (seed) {
      if (words == 64) go(k_dot_fixed<1, true>);
      else if (words == 128) go(k_dot_fixed<2, true>);
      else go(k_dot_fixed<4, true>);
    } else {
      if (words == 64) go(k_dot_fixed<1, false>);
      else if (words == 128) go(k_dot_fixed<2, false>);
      else go(k_dot_fixed<4, false>);
    }
  } else if (vec && seed)
    k_dot_batched<true><<<(unsigned)blocks, 256, 0, s>>>(v4(x), v4(y), v4(seed), words, pairs, wsum, out);
  else if (vec)
    k_dot_batched<false><<<(unsigned)blocks, 256, 0, s>>>(v4(x), v4(y), nullptr, words, pairs, wsum, out);
  else if (seed)
    k_dot_batched_u64<true><<<(unsigned)blocks, 256, 0, s>>>(x, y, seed, words, pairs, wsum, out);
  else
    k_dot_batched_u64<false><<<(unsigned)blocks, 256, 0, s>>>(x, y, nullptr, words, pairs, wsum, out);
  return cudaGetLastError();
}

cudaError_t tk_launch_gemm_popc(const uint64_t* rows, size_t M, int wpr64,
                                const tk_layer* L, int offset, tk_epilogue e,
                                cudaStream_t s) {
  if (M == 0) return cudaSuccess;
  dim3 grid((L->out_c + BN - 1) / BN, (unsigned)((M + BM - 1) / BM));
  k_gemm_popc<<<grid, 256, 0, s>>>(
      reinterpret_cast<const uint32_t*>(rows), (int)M, 2 * wpr64,
      reinterpret_cast<const uint32_t*>(L->d_words), L->d_mask, L->out_c,
      L->d_wsum, L->d_zcnt, offset, e);
  return cudaGetLastError();
}

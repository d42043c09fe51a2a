// Design microbenchmark (not product code): the output stage of the bucket
// step.  A CTA holds T 16-B records in shared memory, each with a random
// output digit (NB = 2^logb pass-1 buckets of the next step); it reserves one
// run per digit with a global atomic and writes the records
//   mode 0: staged -- records reordered by digit through a shared-memory index,
//           consecutive threads write consecutive slots (coalesced runs)
//   mode 1: direct -- each thread writes its own records at run base + rank
//           (scattered 16-B stores, no staging index, one barrier less)
//   mode 2: plain copy of the same bytes (ceiling)
// Reports GB/s on 32 B per record (read + write).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o runs_mb runs_mb.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix(uint32_t x, uint32_t m) {
  x ^= m * 0x9E3779B9u;
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

__global__ void init_k(uint4* a, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    a[i] = make_uint4((uint32_t)i, __float_as_uint(1.0f), __float_as_uint(2.0f), __float_as_uint(3.0f));
}
__global__ void zero_k(uint32_t* c, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) c[i] = 0;
}

template <int BLOCK, int ITEMS, int MODE>
__global__ void __launch_bounds__(BLOCK) runs_k(const uint4* __restrict__ in, uint64_t n, uint4* out, uint32_t* cur,
                                                uint32_t logb, uint32_t cap, uint32_t m) {
  constexpr int T = BLOCK * ITEMS;
  __shared__ uint4 rs[T];
  __shared__ uint32_t cnt[512], off[512], gb[512];
  __shared__ uint32_t inv[T];
  const uint32_t nb = 1u << logb, sh = 32 - logb;
  const uint64_t base = (uint64_t)blockIdx.x * T;
  if (base >= n) return;
  for (uint32_t i = threadIdx.x; i < nb; i += BLOCK) cnt[i] = 0;
  __syncthreads();
  uint32_t dg[ITEMS], rk[ITEMS];
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const uint32_t e = k * BLOCK + threadIdx.x;
    const uint4 r = __ldcs(in + base + e);
    rs[e] = r;
    dg[k] = mix(r.x, m) >> sh;
    rk[k] = atomicAdd(&cnt[dg[k]], 1u);
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < nb; i += BLOCK) {
    const uint32_t h = cnt[i];
    gb[i] = h ? atomicAdd(&cur[i], h) : 0u;
  }
  if (MODE == 1) {
    __syncthreads();
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const uint32_t e = k * BLOCK + threadIdx.x;
      const uint32_t s = gb[dg[k]] + rk[k];
      if (s < cap) out[(size_t)dg[k] * cap + s] = rs[e];
    }
    return;
  }
  // exclusive scan of cnt (simple: warp 0 serial chunks)
  __syncthreads();
  if (threadIdx.x < 32) {
    const uint32_t per = (nb + 31) / 32, b0 = threadIdx.x * per;
    uint32_t s = 0;
    for (uint32_t i = b0; i < min(nb, b0 + per); ++i) s += cnt[i];
    uint32_t v = s;
    for (int o = 1; o < 32; o <<= 1) { const uint32_t t = __shfl_up_sync(0xffffffffu, v, o); if (threadIdx.x >= o) v += t; }
    uint32_t run = v - s;
    for (uint32_t i = b0; i < min(nb, b0 + per); ++i) { const uint32_t c = cnt[i]; off[i] = run; gb[i] -= run; run += c; }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const uint32_t e = k * BLOCK + threadIdx.x;
    inv[off[dg[k]] + rk[k]] = e | (dg[k] << 16);
  }
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < T; j += BLOCK) {
    const uint32_t v = inv[j], e = v & 0xffffu, d = v >> 16;
    const uint32_t s = gb[d] + j;
    if (s < cap) out[(size_t)d * cap + s] = rs[e];
  }
}

__global__ void __launch_bounds__(256) copy_k(const uint4* __restrict__ in, uint64_t n, uint4* out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = __ldcs(in + i);
}

static void run(int mode, int logb, int logn) {
  constexpr int BLOCK = 256, ITEMS = 8, T = BLOCK * ITEMS;
  const uint64_t n = 1ull << logn;
  const uint32_t nb = 1u << logb;
  const double mu = (double)n / nb;
  uint32_t cap = (uint32_t)(mu + 12 * sqrt(mu) + 64);
  cap = (cap + 63) & ~63u;
  uint4 *in, *out;
  uint32_t* cur;
  cudaMalloc(&in, n * 16);
  cudaMalloc(&out, (uint64_t)nb * cap * 16);
  cudaMalloc(&cur, (size_t)nb * 4);
  init_k<<<1184, 256>>>(in, n);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 7; ++r) {
    zero_k<<<64, 256>>>(cur, nb);
    cudaEventRecord(e0);
    if (mode == 0) runs_k<BLOCK, ITEMS, 0><<<(unsigned)(n / T), BLOCK>>>(in, n, out, cur, logb, cap, r);
    else if (mode == 1) runs_k<BLOCK, ITEMS, 1><<<(unsigned)(n / T), BLOCK>>>(in, n, out, cur, logb, cap, r);
    else copy_k<<<148 * 8, 256>>>(in, n, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r >= 2) best = ms < best ? ms : best;
  }
  printf("mode=%d logb=%d logn=%d best_ms=%.3f GBs(32B/rec)=%.0f err=%s\n", mode, logb, logn, best,
         32.0 * n / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  cudaFree(in); cudaFree(out); cudaFree(cur);
}

int main() {
  run(2, 8, 28);
  for (int b : {7, 8, 9}) { run(0, b, 28); run(1, b, 28); }
  return 0;
}

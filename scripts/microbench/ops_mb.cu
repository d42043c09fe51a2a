// Design microbenchmark (not product code): SM-side cost of the building
// blocks of an in-bucket sort / multisplit on B200, per element:
//   0 shared-memory atomicAdd with return, random bins (ATOMS)
//   1 __match_any_sync on an 8-bit digit (MATCH.ANY)
//   2 8-bit warp multisplit by ballots (VOTE + LOP3)
//   3 Philox4x32-10 (10 rounds, precomputed keys)
//   4 plain LDS/STS round trip (random bins, for the smem floor)
// Each kernel processes `per` elements per thread over a full grid; time/elt.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ops_mb ops_mb.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

template <int MODE>
__global__ void __launch_bounds__(512) k(uint32_t per, uint32_t* out, uint32_t seed) {
  __shared__ uint32_t h[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) h[i] = 0;
  __syncthreads();
  uint32_t acc = 0;
  uint32_t x = hash(blockIdx.x * 512 + threadIdx.x + seed);
  const int lane = threadIdx.x & 31;
  for (uint32_t i = 0; i < per; ++i) {
    x = x * 1664525u + 1013904223u;
    const uint32_t dg = x >> 24;
    if (MODE == 0) {
      acc += atomicAdd(&h[dg + ((threadIdx.x >> 5) << 8)], 1u);
    } else if (MODE == 1) {
      const uint32_t peers = __match_any_sync(0xffffffffu, dg);
      acc += __popc(peers & ((1u << lane) - 1));
    } else if (MODE == 2) {
      uint32_t peers = 0xffffffffu;
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const uint32_t bal = __ballot_sync(0xffffffffu, (dg >> b) & 1u);
        peers &= ((dg >> b) & 1u) ? bal : ~bal;
      }
      acc += __popc(peers & ((1u << lane) - 1));
    } else if (MODE == 3) {
      uint32_t c0 = x, c1 = i, c2 = 7, c3 = 1;
#pragma unroll
      for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ (seed + r * 0x9E3779B9u);
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ (seed * 3u + r * 0xBB67AE85u);
        c1 = (uint32_t)p1; c3 = (uint32_t)p0; c0 = n0; c2 = n2;
      }
      acc += c0 ^ c1 ^ c2 ^ c3;
    } else {
      const uint32_t a = dg + ((threadIdx.x >> 5) << 8);
      const uint32_t v = h[a];
      h[a ^ 1] = v + 1;
      acc += v;
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

int main() {
  uint32_t* out;
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const uint32_t per = 4096, grid = 148 * 4;
  const double elts = (double)per * grid * 512;
  const char* names[] = {"atoms", "match_any", "ballot8", "philox", "lds_sts"};
  for (int mode = 0; mode < 5; ++mode) {
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
      cudaEventRecord(e0);
      switch (mode) {
        case 0: k<0><<<grid, 512>>>(per, out, r); break;
        case 1: k<1><<<grid, 512>>>(per, out, r); break;
        case 2: k<2><<<grid, 512>>>(per, out, r); break;
        case 3: k<3><<<grid, 512>>>(per, out, r); break;
        default: k<4><<<grid, 512>>>(per, out, r); break;
      }
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r && ms < best) best = ms;
    }
    // SM-cycles per element at 1.965 GHz over 148 SMs
    printf("%-10s %.3f ms  %.3f ns/elt(chip)  %.2f SM-cycles/elt  err=%s\n", names[mode], best,
           best * 1e6 / elts, best * 1e-3 * 1.965e9 * 148 / elts, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}

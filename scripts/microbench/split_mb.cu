// Design microbenchmark (not product code): the pass-2 split
// with the records stored SoA (5 arrays of 4 B: id, key, x0, x1, x2 -- the
// current layout) versus AoS (one 20-B record).  Same tiles (4096 records of a
// 2^20-record segment), same 512 digits, same run reservations; only the
// record layout differs.  In the AoS variant the staged tile is written out
// as a word stream (consecutive lanes write consecutive words of the output
// runs), so a run of r records is one contiguous 20r-byte store.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o split_mb split_mb.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int TILE = 4096, BLOCK = 1024, NB = 512, W = 5;  // words per record
constexpr uint32_t SEG = 1u << 20, NSEG = 256, CAP2 = 2688;

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

__global__ void init_soa(uint32_t* a, uint64_t n) {  // a: W arrays of n words
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    a[i] = (uint32_t)i;
    a[n + i] = mix((uint32_t)i);
    for (int c = 2; c < W; ++c) a[c * n + i] = (uint32_t)(i * 3 + c);
  }
}
__global__ void init_aos(uint32_t* a, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    a[i * W] = (uint32_t)i;
    a[i * W + 1] = mix((uint32_t)i);
    for (int c = 2; c < W; ++c) a[i * W + c] = (uint32_t)(i * 3 + c);
  }
}

__device__ uint32_t block_scan(uint32_t* a, uint32_t* ws) {  // exclusive scan of NB entries
  const int t = threadIdx.x;
  uint32_t v = t < NB ? a[t] : 0u, inc = v;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if ((t & 31) >= o) inc += y;
  }
  if ((t & 31) == 31) ws[t >> 5] = inc;
  __syncthreads();
  if (t < 32) {
    uint32_t s = ws[t], si = s;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, si, o);
      if (t >= o) si += y;
    }
    ws[t] = si - s;
  }
  __syncthreads();
  if (t < NB) a[t] = ws[t >> 5] + inc - v;
  __syncthreads();
  return 0;
}

template <bool AOS>
__global__ void __launch_bounds__(BLOCK) split(const uint32_t* __restrict__ in, uint32_t* out, uint32_t* cur,
                                               uint64_t n, uint64_t outn) {
  extern __shared__ uint32_t sm[];
  uint32_t* stg = sm;                  // TILE * W words (SoA by array, or AoS by record)
  uint32_t* hist = stg + TILE * W;     // NB
  uint32_t* off = hist + NB;           // NB
  uint32_t* gb = off + NB;             // NB
  uint32_t* ws = gb + NB;              // 32
  uint32_t* rk = ws + 32;              // TILE
  uint16_t* inv = reinterpret_cast<uint16_t*>(rk + TILE);
  const uint32_t t0 = blockIdx.x * TILE, u = t0 / SEG;
  const int tid = threadIdx.x;
  if (tid < NB) hist[tid] = 0;
  // load (coalesced)
  if (AOS) {
    for (int w = tid; w < TILE * W; w += BLOCK) stg[w] = in[(uint64_t)t0 * W + w];
  } else {
    for (int c = 0; c < W; ++c)
      for (int e = tid; e < TILE; e += BLOCK) stg[c * TILE + e] = in[c * n + t0 + e];
  }
  __syncthreads();
  for (int e = tid; e < TILE; e += BLOCK) {
    const uint32_t key = AOS ? stg[e * W + 1] : stg[TILE + e];
    const uint32_t dg = (key >> 15) & (NB - 1);
    rk[e] = (dg << 16) | atomicAdd(&hist[dg], 1u);
  }
  __syncthreads();
  uint32_t g = 0;
  if (tid < NB) {
    off[tid] = hist[tid];
    g = hist[tid] ? atomicAdd(&cur[(u * NB + tid) * 8], hist[tid]) : 0u;
  }
  __syncthreads();
  block_scan(off, ws);
  for (int e = tid; e < TILE; e += BLOCK) inv[off[rk[e] >> 16] + (rk[e] & 0xffffu)] = (uint16_t)e;
  if (tid < NB) gb[tid] = g - off[tid];
  __syncthreads();
  if (AOS) {  // word stream over the tile's output positions
    for (int w = tid; w < TILE * W; w += BLOCK) {
      const int j = w / W, c = w - j * W;
      const uint32_t e = inv[j];
      const uint32_t dg = (stg[e * W + 1] >> 15) & (NB - 1);
      const uint32_t slot = gb[dg] + j;
      if (slot < CAP2) out[((uint64_t)(u * NB + dg) * CAP2 + slot) * W + c] = stg[e * W + c];
    }
  } else {
    for (int j = tid; j < TILE; j += BLOCK) {
      const uint32_t e = inv[j];
      const uint32_t dg = (stg[TILE + e] >> 15) & (NB - 1);
      const uint32_t slot = gb[dg] + j;
      if (slot < CAP2) {
        const uint64_t o = (uint64_t)(u * NB + dg) * CAP2 + slot;
        for (int c = 0; c < W; ++c) out[c * outn + o] = stg[c * TILE + e];
      }
    }
  }
}

int main() {
  const uint64_t n = (uint64_t)SEG * NSEG, outn = (uint64_t)NSEG * NB * CAP2;
  uint32_t *in, *out, *cur;
  cudaMalloc(&in, n * W * 4);
  cudaMalloc(&out, outn * W * 4);
  cudaMalloc(&cur, NSEG * NB * 8 * 4);
  const size_t smem = (TILE * W + 3 * NB + 32 + TILE) * 4 + TILE * 2;
  cudaFuncSetAttribute(split<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(split<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int aos = 0; aos < 2; ++aos) {
    if (aos) init_aos<<<148 * 8, 256>>>(in, n); else init_soa<<<148 * 8, 256>>>(in, n);
    float best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
      cudaMemset(cur, 0, NSEG * NB * 8 * 4);
      cudaEventRecord(a);
      if (aos) split<true><<<(unsigned)(n / TILE), BLOCK, smem>>>(in, out, cur, n, outn);
      else split<false><<<(unsigned)(n / TILE), BLOCK, smem>>>(in, out, cur, n, outn);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep > 0 && ms < best) best = ms;
    }
    const double gb = 2.0 * n * W * 4 / 1e9;
    printf("%s: %.3f ms for 2^28 records (%.0f GB/s of record bytes read + written) err=%s\n", aos ? "AoS" : "SoA",
           best, gb / (best / 1e3), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}

// rbm_kernels.cuh -- the RBM time-step kernels for sm_100a.
//
// RBM-1 step m (Alg. 1) as an MSD partition + fused sort/step:
//   hist_top      compute-only histogram of the top b1 key bits over ids 0..N-1
//   scan_top      bucket offsets / cursors of pass 1 (+ tile table of pass 2)
//   scatter<1>    state -> buckets by the top b1 key bits (smem-staged)
//   hist_sub      per top-bucket histogram of the next b2 bits (2-pass layouts)
//   scan_sub      final bucket starts S[0..2^B] and pass-2 cursors
//   scatter<2>    -> final buckets of the top B = b1+b2 key bits
//   bucket_step   per bucket: exact in-smem sort by (key, id), then every batch
//                 that lies inside the bucket does Eq. (2.2) + Euler-Maruyama
//                 (or the exact pair flow) and writes in sorted order
//   straddle_step batches that straddle two buckets
//   advance       m += 1
// The resulting permutation is exactly "ids sorted by (key_m(id), id)".
#pragma once
#include "rbm_device.cuh"

namespace rbm {

template <typename T, int D> struct State {
  uint32_t* id;
  T* x[3];
};

// ----------------------------------------------------------------- helpers
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// exclusive scan of a[0..n) in shared memory by the whole block (n <= 4*BLOCK*k)
// wsum: >= 32 uint32 of shared scratch. Returns the total.
template <int BLOCK>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t* a, int n, uint32_t* wsum) {
  const int per = (n + BLOCK - 1) / BLOCK;
  const int t = threadIdx.x;
  const int b0 = min(n, t * per), b1 = min(n, b0 + per);
  uint32_t s = 0;
  for (int i = b0; i < b1; ++i) s += a[i];
  const uint32_t inc = warp_incl_scan(s);
  const int lane = t & 31, w = t >> 5;
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  if (w == 0) {
    const uint32_t v = (lane < BLOCK / 32) ? wsum[lane] : 0u;
    const uint32_t vi = warp_incl_scan(v);
    if (lane < BLOCK / 32) wsum[lane] = vi - v;
    if (lane == 31) wsum[32] = vi;
  }
  __syncthreads();
  uint32_t run = wsum[w] + inc - s;
  for (int i = b0; i < b1; ++i) { const uint32_t v = a[i]; a[i] = run; run += v; }
  const uint32_t total = wsum[32];
  __syncthreads();
  return total;
}

// position P's batch (reading D:7): returns [b0, b1).  N < 2^32.
__device__ __forceinline__ void batch_range(uint32_t P, const DevParams& prm, uint32_t& b0,
                                            uint32_t& b1) {
  const uint32_t n = (uint32_t)prm.n, p = prm.p;
  uint32_t k = fdiv(P, prm.pdiv);
  if (prm.rem == 1 && k + 1 >= prm.nfull) {
    k = prm.nfull - 1;
    b0 = k * p;
    b1 = n;
  } else {
    b0 = k * p;
    b1 = min(b0 + p, n);
  }
}

// ------------------------------------------------------------------- init
// X_0 in fp64, rounded to T; state stored in id order.
template <typename T, int D>
static __global__ void init_kernel(DevParams P, State<T, D> st, uint32_t kind, double a0, double a1,
                            double a2, double a3) {
  const uint64_t n = P.n;
  // mixture centres (<= 64), computed redundantly per block
  __shared__ double cent[64][3];
  const int K = (kind == 4) ? (int)a0 : 0;
  if (kind == 4) {
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
      const uint4 w = block_at(P, (uint32_t)k, 0u, 0u, TAG_INIT_AUX);
      const uint4 v = block_at(P, (uint32_t)k, 2u, 0u, TAG_INIT_AUX);
      cent[k][0] = a2 + (a3 - a2) * u01d(w.x, w.y);
      cent[k][1] = a2 + (a3 - a2) * u01d(w.z, w.w);
      cent[k][2] = a2 + (a3 - a2) * u01d(v.x, v.y);
    }
  }
  __syncthreads();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t id = (uint32_t)i;
    double x[3] = {0, 0, 0};
    if (kind == 1 || kind == 3 || kind == 4) {
      double z[D];
      Normals<double, D>::get(P, id, 0u, TAG_INIT, z);
      if (kind == 1) {
        for (int c = 0; c < D; ++c) x[c] = a0 + a1 * z[c];
      } else if (kind == 3) {
        double r2 = 0;
        for (int c = 0; c < D; ++c) r2 += z[c] * z[c];
        const double r = sqrt(r2);
        for (int c = 0; c < D; ++c) x[c] = z[c] / r;
      } else {
        const uint4 w = block_at(P, id, 1u, 0u, TAG_INIT_AUX);
        int k = (int)floor((double)K * u01d(w.x, w.y));
        if (k >= K) k = K - 1;
        for (int c = 0; c < D; ++c) x[c] = cent[k][c] + a1 * z[c];
      }
    } else if (kind == 2) {
      const uint4 w = block_at(P, id, 0u, 0u, TAG_INIT);
      const uint4 v = block_at(P, id, 1u, 0u, TAG_INIT);
      const double u[4] = {u01d(w.x, w.y), u01d(w.z, w.w), u01d(v.x, v.y), u01d(v.z, v.w)};
      for (int c = 0; c < D; ++c) x[c] = a0 + (a1 - a0) * u[c];
    }
    st.id[i] = id;
#pragma unroll
    for (int c = 0; c < D; ++c) st.x[c][i] = (T)x[c];
  }
}

// user state (id order, row-major N x D) -> SoA state in id order
template <typename T, int D>
static __global__ void set_state_kernel(uint64_t n, State<T, D> st, const T* __restrict__ xin) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    st.id[i] = (uint32_t)i;
#pragma unroll
    for (int c = 0; c < D; ++c) st.x[c][i] = xin[i * D + c];
  }
}

// SoA state in storage order -> x_out (id order, row-major) for ids [i0, i1)
template <typename T, int D>
static __global__ void gather_kernel(uint64_t n, State<T, D> st, uint64_t i0, uint64_t i1,
                              T* __restrict__ out) {
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t id = st.id[q];
    if (id >= i0 && id < i1) {
#pragma unroll
      for (int c = 0; c < D; ++c) out[(id - i0) * D + c] = st.x[c][q];
    }
  }
}

static __global__ void copy_ids_kernel(uint64_t n, const uint32_t* __restrict__ id, uint32_t* out) {
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n;
       q += (uint64_t)gridDim.x * blockDim.x)
    out[q] = id[q];
}

static __global__ void philox_test_kernel(const uint32_t* __restrict__ in, uint32_t* out, uint64_t count) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t* a = in + 6 * i;
    const uint4 r = philox4x32_10(make_uint4(a[0], a[1], a[2], a[3]), a[4], a[5]);
    out[4 * i + 0] = r.x; out[4 * i + 1] = r.y; out[4 * i + 2] = r.z; out[4 * i + 3] = r.w;
  }
}

static __global__ void advance_kernel(uint64_t* step) { *step += 1; }

// ------------------------------------------------------- compute-only histogram
// histogram of key_m(id) >> (32-b1) over ALL ids 0..N-1: reads no memory.
static __global__ void __launch_bounds__(512) hist_top_kernel(DevParams P, uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[1024];
  const uint32_t nb = 1u << P.b1;
  for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const uint32_t m = (uint32_t)*P.step;
  const uint32_t sh = 32u - P.b1;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < P.n;
       i += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(&h[shuffle_key(P, (uint32_t)i, m) >> sh], 1u);
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], h[i]);
}

// single block: off1 = excl-scan(hist1), cursor1 = off1, tile table for pass 2,
// and (one-pass layouts) the final bucket starts S.
static __global__ void __launch_bounds__(1024) scan_top_kernel(DevParams P, const uint32_t* __restrict__ hist,
                                                        uint32_t* off1, uint32_t* cur1,
                                                        uint32_t* tile_off, uint32_t* S,
                                                        uint32_t tile) {
  __shared__ uint32_t a[1025];
  __shared__ uint32_t t[1025];
  __shared__ uint32_t ws[33];
  const uint32_t nb = 1u << P.b1;
  for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) {
    a[i] = hist[i];
    t[i] = (hist[i] + tile - 1) / tile;
  }
  __syncthreads();
  block_excl_scan<1024>(a, nb, ws);
  const uint32_t ntiles = block_excl_scan<1024>(t, nb, ws);
  for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) {
    off1[i] = a[i];
    cur1[i] = a[i];
    tile_off[i] = t[i];
    if (P.b2 == 0) S[i] = a[i];
  }
  if (threadIdx.x == 0) {
    off1[nb] = (uint32_t)P.n;
    tile_off[nb] = ntiles;
    if (P.b2 == 0) S[nb] = (uint32_t)P.n;
  }
}

// one block per top bucket u: S[u<<b2 | i] = off1[u] + excl-scan_i hist2[u<<b2 | .]
static __global__ void __launch_bounds__(512) scan_sub_kernel(DevParams P, const uint32_t* __restrict__ hist2,
                                                              const uint32_t* __restrict__ off1,
                                                              uint32_t* S, uint32_t* cur2) {
  __shared__ uint32_t a[512];
  __shared__ uint32_t ws[33];
  const uint32_t u = blockIdx.x, nb2 = 1u << P.b2, base = u << P.b2;
  for (uint32_t i = threadIdx.x; i < nb2; i += blockDim.x) a[i] = hist2[base + i];
  __syncthreads();
  block_excl_scan<512>(a, nb2, ws);
  const uint32_t o = off1[u];
  for (uint32_t i = threadIdx.x; i < nb2; i += blockDim.x) {
    S[base + i] = o + a[i];
    cur2[base + i] = o + a[i];
  }
  if (u == 0 && threadIdx.x == 0) S[P.nbuckets] = (uint32_t)P.n;
}

// tile t of a bucket-aligned pass: bucket u and element range [lo, hi)
__device__ __forceinline__ bool aligned_tile(const uint32_t* __restrict__ tile_off,
                                             const uint32_t* __restrict__ off1, uint32_t nb1,
                                             uint32_t t, uint32_t tile, uint32_t& u, uint32_t& lo,
                                             uint32_t& hi) {
  if (t >= tile_off[nb1]) return false;
  uint32_t a = 0, b = nb1;  // largest u with tile_off[u] <= t
  while (b - a > 1) {
    const uint32_t mid = (a + b) >> 1;
    if (tile_off[mid] <= t) a = mid; else b = mid;
  }
  u = a;
  lo = off1[u] + (t - tile_off[u]) * tile;
  hi = min(lo + tile, off1[u + 1]);
  return true;
}

// per top-bucket histogram of the next b2 key bits (reads ids only)
static __global__ void __launch_bounds__(256) hist_sub_kernel(DevParams P, const uint32_t* __restrict__ ids,
                                                       const uint32_t* __restrict__ off1,
                                                       const uint32_t* __restrict__ tile_off,
                                                       uint32_t* hist2, uint32_t tile) {
  __shared__ uint32_t h[512];
  uint32_t u, lo, hi;
  if (!aligned_tile(tile_off, off1, 1u << P.b1, blockIdx.x, tile, u, lo, hi)) return;
  const uint32_t nb2 = 1u << P.b2;
  for (uint32_t i = threadIdx.x; i < nb2; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const uint32_t m = (uint32_t)*P.step;
  const uint32_t sh = 32u - P.b1 - P.b2, mask = nb2 - 1;
  for (uint32_t e = lo + threadIdx.x; e < hi; e += blockDim.x)
    atomicAdd(&h[(shuffle_key(P, ids[e], m) >> sh) & mask], 1u);
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < nb2; i += blockDim.x)
    if (h[i]) atomicAdd(&hist2[(u << P.b2) | i], h[i]);
}

// --------------------------------------------------------------- scatter pass
// LEVEL 1: tiles over the whole array, digit = top b1 bits, cursors cur[digit].
// LEVEL 2: tiles aligned to top buckets u, digit = next b2 bits,
//          cursors cur[(u << b2) | digit].
// Order inside a bucket is irrelevant: bucket_step sorts each bucket exactly.
template <typename T, int D, int LEVEL, int BLOCK, int ITEMS>
static __global__ void __launch_bounds__(BLOCK) scatter_kernel(DevParams P, State<T, D> src,
                                                        State<T, D> dst, uint32_t* cur,
                                                        const uint32_t* __restrict__ off1,
                                                        const uint32_t* __restrict__ tile_off) {
  constexpr int TILE = BLOCK * ITEMS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem_raw);  // 1024
  uint32_t* gbase = hist + 1024;                           // 1024
  uint32_t* wsum = gbase + 1024;                           // 64
  uint32_t* st_id = wsum + 64;                             // TILE
  T* st_x = reinterpret_cast<T*>(st_id + TILE);            // D*TILE
  uint16_t* st_dig = reinterpret_cast<uint16_t*>(st_x + D * TILE);  // TILE

  uint32_t lo, hi, u = 0, bits, sh;
  if (LEVEL == 1) {
    lo = blockIdx.x * TILE;
    if (lo >= P.n) return;
    hi = (uint32_t)min((uint64_t)lo + TILE, P.n);
    bits = P.b1;
    sh = 32u - P.b1;
  } else {
    if (!aligned_tile(tile_off, off1, 1u << P.b1, blockIdx.x, TILE, u, lo, hi)) return;
    bits = P.b2;
    sh = 32u - P.b1 - P.b2;
  }
  const uint32_t nbins = 1u << bits, mask = nbins - 1;
  uint32_t* mycur = cur + (LEVEL == 1 ? 0u : (u << P.b2));
  for (uint32_t i = threadIdx.x; i < nbins; i += BLOCK) hist[i] = 0;
  __syncthreads();

  const uint32_t m = (uint32_t)*P.step;
  const uint32_t cnt = hi - lo;
  uint32_t rid[ITEMS], rdig[ITEMS], rslot[ITEMS];
  T rx[ITEMS][D];
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const uint32_t e = k * BLOCK + threadIdx.x;
    if (e < cnt) {
      rid[k] = src.id[lo + e];
#pragma unroll
      for (int c = 0; c < D; ++c) rx[k][c] = src.x[c][lo + e];
    }
  }
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const uint32_t e = k * BLOCK + threadIdx.x;
    if (e < cnt) {
      rdig[k] = (shuffle_key(P, rid[k], m) >> sh) & mask;
      rslot[k] = atomicAdd(&hist[rdig[k]], 1u);
    }
  }
  __syncthreads();
  // reserve global space per bin, then local exclusive offsets
  for (uint32_t i = threadIdx.x; i < nbins; i += BLOCK) {
    const uint32_t h = hist[i];
    gbase[i] = h ? atomicAdd(&mycur[i], h) : 0u;
  }
  block_excl_scan<BLOCK>(hist, nbins, wsum);  // hist -> local offsets
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const uint32_t e = k * BLOCK + threadIdx.x;
    if (e < cnt) {
      const uint32_t s = hist[rdig[k]] + rslot[k];
      st_id[s] = rid[k];
      st_dig[s] = (uint16_t)rdig[k];
#pragma unroll
      for (int c = 0; c < D; ++c) st_x[c * TILE + s] = rx[k][c];
    }
  }
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < cnt; j += BLOCK) {
    const uint32_t dg = st_dig[j];
    const uint32_t g = gbase[dg] + (j - hist[dg]);
    dst.id[g] = st_id[j];
#pragma unroll
    for (int c = 0; c < D; ++c) dst.x[c][g] = st_x[c * TILE + j];
  }
}

// ------------------------------------------------------- fused bucket step
// One CTA per final bucket b = positions [S[b], S[b+1]).  All ids in it share
// the top B key bits, so sorting it by (key, id) in shared memory puts every
// element at its exact global sorted position S[b] + rank.
template <typename T> __device__ __forceinline__ T batch_inv(const DevParams& P, uint32_t sz) {
  return (sz == P.p) ? Prm<T>::invp(P) : T(1) / T(sz - 1);
}

template <typename T, int D, int KK, int INTEG>
__device__ __forceinline__ void interior_update(const DevParams& P, uint32_t m, uint32_t q,
                                                uint32_t l0, uint32_t l1, const uint16_t* ord,
                                                T* const* xs, uint32_t id, T (&xn)[D]) {
  T xi[D];
  const uint32_t e = ord[q];
#pragma unroll
  for (int c = 0; c < D; ++c) xi[c] = xs[c][e];
  T z[D];
#pragma unroll
  for (int c = 0; c < D; ++c) z[c] = T(0);
  if (P.has_noise) Normals<T, D>::get(P, id, m, TAG_NOISE, z);
  if (INTEG == 0) {
    T f[D];
#pragma unroll
    for (int c = 0; c < D; ++c) f[c] = T(0);
    for (uint32_t g = l0; g < l1; ++g) {  // ascending sorted position, self skipped
      if (g == q) continue;
      const uint32_t e2 = ord[g];
      T xj[D];
#pragma unroll
      for (int c = 0; c < D; ++c) xj[c] = xs[c][e2];
      add_interaction<T, D, KK>(xi, xj, f, P);
    }
    const T inv = batch_inv<T>(P, l1 - l0);
#pragma unroll
    for (int c = 0; c < D; ++c) f[c] *= inv;
    em_update<T, D>(xi, f, z, xn, P, true);
  } else {
    const uint32_t ea = ord[l0], eb = ord[l0 + 1];
    T xa[D], xb[D], y[D];
#pragma unroll
    for (int c = 0; c < D; ++c) { xa[c] = xs[c][ea]; xb[c] = xs[c][eb]; }
    pair_flow<T, D, KK>(xa, xb, q == l0, y, P);
    split_finish<T, D>(y, z, xn, P, true);
  }
}

// Sort the loaded bucket by (key, id) and step every interior batch.
//   id_l, xs : bucket records in load order (n of them)
//   key_l    : n u32 scratch;  ks : n u64 scratch (16-B aligned);  ord : n u16
template <typename T, int D, int KK, int INTEG, int BLOCK>
__device__ __forceinline__ void bucket_compute(const DevParams& P, State<T, D> dst, uint32_t s0,
                                               uint32_t n, const uint32_t* id_l, T* const* xs,
                                               uint32_t* key_l, unsigned long long* ks,
                                               uint16_t* ord, uint32_t* cnt, uint32_t* off,
                                               uint32_t* wsum) {
  const uint32_t m = (uint32_t)*P.step;
  // 1. keys (Philox), counting sort by the next 8 key bits below the B-bit prefix
  const uint32_t sh = (P.B <= 24u) ? (24u - P.B) : 0u;
  for (uint32_t e = threadIdx.x; e < n; e += BLOCK) {
    const uint32_t key = shuffle_key(P, id_l[e], m);
    key_l[e] = key;
    ord[e] = (uint16_t)atomicAdd(&cnt[(key >> sh) & 255u], 1u);
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < 256; i += BLOCK) off[i] = cnt[i];
  __syncthreads();
  block_excl_scan<BLOCK>(off, 256, wsum);
  // 2. composite (key, id) keys grouped by sub-digit, contiguous per sub-bucket
  for (uint32_t e = threadIdx.x; e < n; e += BLOCK) {
    const uint32_t key = key_l[e];
    ks[off[(key >> sh) & 255u] + ord[e]] = ((unsigned long long)key << 32) | id_l[e];
  }
  __syncthreads();
  // 3. exact rank = sub-bucket offset + #smaller composites in the sub-bucket
  for (uint32_t e = threadIdx.x; e < n; e += BLOCK) {
    const uint32_t key = key_l[e];
    const unsigned long long mine = ((unsigned long long)key << 32) | id_l[e];
    const uint32_t sd = (key >> sh) & 255u;
    const uint32_t a = off[sd], c = cnt[sd];
    uint32_t r = a;
    for (uint32_t j = a; j < a + c; ++j) r += (ks[j] < mine) ? 1u : 0u;
    ord[r] = (uint16_t)e;
  }
  __syncthreads();
  // 4. batches inside [s0, s0+n): Eq. (2.2) + update; straddling ones copied through
  for (uint32_t q = threadIdx.x; q < n; q += BLOCK) {
    const uint32_t P0 = s0 + q;
    uint32_t b0, b1;
    batch_range(P0, P, b0, b1);
    const uint32_t e = ord[q];
    const uint32_t id = id_l[e];
    T xn[D];
    if (b0 >= s0 && b1 <= s0 + n) {
      interior_update<T, D, KK, INTEG>(P, m, q, b0 - s0, b1 - s0, ord, xs, id, xn);
      check_finite<T, D>(xn, P, id, m);
    } else {
#pragma unroll
      for (int c = 0; c < D; ++c) xn[c] = xs[c][e];
    }
    dst.id[P0] = id;
#pragma unroll
    for (int c = 0; c < D; ++c) dst.x[c][P0] = xn[c];
  }
}

// shared-memory bytes of the bucket kernel for capacity `cap`
template <typename T, int D> __host__ __device__ constexpr size_t bucket_smem_bytes(uint32_t cap) {
  return 2304 + 16                                  // cnt, off, wsum; mbarrier
         + (size_t)(cap + 8) * 4                    // ids (TMA window)
         + (size_t)D * (((size_t)(cap + 8) * sizeof(T) + 15) & ~(size_t)15)  // x (TMA windows)
         + (size_t)cap * 8                          // composite keys
         + (size_t)cap * 4                          // keys
         + (((size_t)cap * 2 + 15) & ~(size_t)15);  // ord
}

template <typename T, int D, int KK, int INTEG, int BLOCK>
static __global__ void __launch_bounds__(BLOCK) bucket_step_kernel(DevParams P, State<T, D> src,
                                                                   State<T, D> dst,
                                                                   const uint32_t* __restrict__ S) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem_raw);
  uint32_t* off = cnt + 256;
  uint32_t* wsum = off + 256;  // 64
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + 2304);
  const uint32_t b = blockIdx.x;
  const uint32_t s0 = S[b], n = S[b + 1] - s0;
  if (n == 0) return;
  for (uint32_t i = threadIdx.x; i < 256; i += BLOCK) cnt[i] = 0;
  const uint32_t cap = P.cap;
  if (n <= cap) {
    // TMA windows: 16-B aligned superset of [s0, s0+n) of every SoA array
    constexpr uint32_t AX = 16 / sizeof(T);
    const uint32_t lo_i = s0 & ~3u, oi = s0 - lo_i;
    const uint32_t lo_x = s0 & ~(AX - 1), ox = s0 - lo_x;
    const uint32_t bytes_i = ((oi + n + 3) & ~3u) * 4;
    const uint32_t bytes_x = ((ox + n + AX - 1) & ~(AX - 1)) * (uint32_t)sizeof(T);
    unsigned char* p = smem_raw + 2320;
    uint32_t* id_raw = reinterpret_cast<uint32_t*>(p);
    p += (size_t)(cap + 8) * 4;
    T* xr[3];
    const size_t xstride = ((size_t)(cap + 8) * sizeof(T) + 15) & ~(size_t)15;
#pragma unroll
    for (int c = 0; c < D; ++c) { xr[c] = reinterpret_cast<T*>(p); p += xstride; }
    unsigned long long* ks = reinterpret_cast<unsigned long long*>(p);
    p += (size_t)cap * 8;
    uint32_t* key_l = reinterpret_cast<uint32_t*>(p);
    p += (size_t)cap * 4;
    uint16_t* ord = reinterpret_cast<uint16_t*>(p);
    if (threadIdx.x == 0) {
      mbar_init(bar, 1);
      mbar_expect_tx(bar, bytes_i + D * bytes_x);
      bulk_g2s(id_raw, src.id + lo_i, bytes_i, bar);
#pragma unroll
      for (int c = 0; c < D; ++c) bulk_g2s(xr[c], src.x[c] + lo_x, bytes_x, bar);
    }
    __syncthreads();
    mbar_wait(bar, 0);
    T* xs[3];
#pragma unroll
    for (int c = 0; c < D; ++c) xs[c] = xr[c] + ox;
    bucket_compute<T, D, KK, INTEG, BLOCK>(P, dst, s0, n, id_raw + oi, xs, key_l, ks, ord, cnt,
                                           off, wsum);
  } else {
    // oversized bucket (never expected at the automatic capacity, forced in
    // tests): same algorithm on one of NBIG global-memory scratch slots,
    // claimed from a small pool and released at the end (holders are resident,
    // so waiters always make progress).
    __shared__ uint32_t slot;
    if (threadIdx.x == 0) {
      slot = 0xffffffffu;
      if (n <= BIG_CAP) {
        for (;;) {
          for (uint32_t s = 0; s < (uint32_t)NBIG && slot == 0xffffffffu; ++s)
            if (atomicCAS(&P.big_claim[s], 0u, 1u) == 0u) slot = s;
          if (slot != 0xffffffffu) break;
          __nanosleep(500);
        }
      }
    }
    __syncthreads();
    if (slot == 0xffffffffu) {
      if (threadIdx.x == 0) atomicExch(P.capacity_err, 1u);
      return;
    }
    unsigned char* base = P.big_scratch + slot * big_slot_bytes(D * sizeof(T));
    unsigned long long* ks = reinterpret_cast<unsigned long long*>(base);
    T* xr = reinterpret_cast<T*>(ks + BIG_CAP + 1);
    uint32_t* id_l = reinterpret_cast<uint32_t*>(xr + (size_t)D * BIG_CAP);
    uint32_t* key_l = id_l + BIG_CAP;
    uint16_t* ord = reinterpret_cast<uint16_t*>(key_l + BIG_CAP);
    T* xs[3];
#pragma unroll
    for (int c = 0; c < D; ++c) xs[c] = xr + (size_t)c * BIG_CAP;
    for (uint32_t e = threadIdx.x; e < n; e += BLOCK) {
      id_l[e] = src.id[s0 + e];
#pragma unroll
      for (int c = 0; c < D; ++c) xs[c][e] = src.x[c][s0 + e];
    }
    __syncthreads();
    bucket_compute<T, D, KK, INTEG, BLOCK>(P, dst, s0, n, id_l, xs, key_l, ks, ord, cnt, off, wsum);
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicExch(&P.big_claim[slot], 0u);
    }
  }
}

// batches that straddle bucket boundaries: one warp per owning boundary.
// Members were copied (unchanged) to their sorted positions in dst.
template <typename T, int D, int KK, int INTEG>
static __global__ void __launch_bounds__(256) straddle_kernel(DevParams P, State<T, D> dst,
                                                       const uint32_t* __restrict__ S) {
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t bnd = warp + 1;  // boundaries 1 .. nbuckets-1
  if (bnd >= P.nbuckets) return;
  const uint32_t Pb = S[bnd];
  if (Pb == 0 || Pb >= P.n) return;
  uint32_t b0, b1;
  batch_range(Pb, P, b0, b1);
  if (b0 == Pb) return;             // boundary at a batch start: no straddle
  if (S[bnd - 1] > b0) return;      // an earlier boundary inside the batch owns it
  const uint32_t m = (uint32_t)*P.step;
  const uint32_t sz = (uint32_t)(b1 - b0);
  // each lane updates members lane, lane+32, ... ; reads of all members from dst
  T xnew[3][D];
  uint32_t idv[3];
  int cntm = 0;
  for (uint32_t q = lane; q < sz; q += 32, ++cntm) {
    const uint32_t g = b0 + q;
    const uint32_t id = dst.id[g];
    T xi[D], z[D], xn[D];
#pragma unroll
    for (int c = 0; c < D; ++c) { xi[c] = dst.x[c][g]; z[c] = T(0); }
    if (P.has_noise) Normals<T, D>::get(P, id, m, TAG_NOISE, z);
    if (INTEG == 0) {
      T f[D];
#pragma unroll
      for (int c = 0; c < D; ++c) f[c] = T(0);
      for (uint32_t h = b0; h < b1; ++h) {
        if (h == g) continue;
        T xj[D];
#pragma unroll
        for (int c = 0; c < D; ++c) xj[c] = dst.x[c][h];
        add_interaction<T, D, KK>(xi, xj, f, P);
      }
      const T inv = batch_inv<T>(P, sz);
#pragma unroll
      for (int c = 0; c < D; ++c) f[c] *= inv;
      em_update<T, D>(xi, f, z, xn, P, true);
    } else {
      T xa[D], xb[D], y[D];
#pragma unroll
      for (int c = 0; c < D; ++c) { xa[c] = dst.x[c][b0]; xb[c] = dst.x[c][b0 + 1]; }
      pair_flow<T, D, KK>(xa, xb, q == 0, y, P);
      split_finish<T, D>(y, z, xn, P, true);
    }
    check_finite<T, D>(xn, P, id, m);
    idv[cntm] = id;
#pragma unroll
    for (int c = 0; c < D; ++c) xnew[cntm][c] = xn[c];
  }
  __syncwarp();
  int k = 0;
  for (uint32_t q = lane; q < sz; q += 32, ++k) {
#pragma unroll
    for (int c = 0; c < D; ++c) dst.x[c][b0 + q] = xnew[k][c];
  }
  (void)idv;
}

// ------------------------------------------------------------------ RBM-r
// one sweep of ceil(N/p) with-replacement batches (Alg. 2/3),
// Jacobi-additive reading D:8.  State stays in id order.
static __global__ void rbmr_draw_kernel(DevParams P, uint64_t nbatch, uint32_t* __restrict__ js,
                                 uint32_t* __restrict__ cnt) {
  const uint32_t m = (uint32_t)*P.step;
  for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < nbatch;
       b += (uint64_t)gridDim.x * blockDim.x) {
    for (uint32_t l = 0; l < P.p; ++l) {
      const uint64_t s = b * P.p + l;
      uint32_t t = 0, j;
      for (;;) {
        const uint4 w = block_at(P, (uint32_t)s, t, m, TAG_SLOT);
        const uint64_t u = (((uint64_t)w.x) << 32) | w.y;
        j = (uint32_t)__umul64hi(P.n, u);
        bool dup = false;
        for (uint32_t l2 = 0; l2 < l; ++l2) dup |= (js[b * P.p + l2] == j);
        if (!dup) break;
        ++t;
      }
      js[s] = j;
      atomicAdd(&cnt[j], 1u);
    }
  }
}

template <typename T, int D, int KK, int INTEG>
static __global__ void rbmr_delta_kernel(DevParams P, uint64_t nslots, State<T, D> st,
                                  const uint32_t* __restrict__ js, T* __restrict__ delta) {
  const uint32_t m = (uint32_t)*P.step;
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < nslots;
       s += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = s / P.p, s0 = b * P.p;
    const uint32_t l = (uint32_t)(s - s0);
    const uint32_t i = js[s];
    T xi[D], z[D], xn[D];
#pragma unroll
    for (int c = 0; c < D; ++c) { xi[c] = st.x[c][i]; z[c] = T(0); }
    if (P.has_noise) Normals<T, D>::get(P, (uint32_t)s, m, TAG_NOISE_SLOT, z);
    if (INTEG == 0) {
      T f[D];
#pragma unroll
      for (int c = 0; c < D; ++c) f[c] = T(0);
      for (uint32_t l2 = 0; l2 < P.p; ++l2) {
        if (l2 == l) continue;
        const uint32_t j = js[s0 + l2];
        T xj[D];
#pragma unroll
        for (int c = 0; c < D; ++c) xj[c] = st.x[c][j];
        add_interaction<T, D, KK>(xi, xj, f, P);
      }
      const T inv = T(1) / T(P.p - 1);
#pragma unroll
      for (int c = 0; c < D; ++c) f[c] *= inv;
      em_update<T, D>(xi, f, z, xn, P, false);
    } else {
      T xa[D], xb[D], y[D];
      const uint32_t ia = js[s0], ib = js[s0 + 1];
#pragma unroll
      for (int c = 0; c < D; ++c) { xa[c] = st.x[c][ia]; xb[c] = st.x[c][ib]; }
      pair_flow<T, D, KK>(xa, xb, l == 0, y, P);
      split_finish<T, D>(y, z, xn, P, false);
    }
#pragma unroll
    for (int c = 0; c < D; ++c) delta[(size_t)c * nslots + s] = xn[c] - xi[c];
  }
}

// CSR fill: slot s appended to particle js[s]'s list (order fixed later)
static __global__ void rbmr_fill_kernel(uint64_t nslots, const uint32_t* __restrict__ js,
                                 const uint32_t* __restrict__ off, uint32_t* __restrict__ fillc,
                                 uint32_t* __restrict__ lst) {
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < nslots;
       s += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t j = js[s];
    lst[off[j] + atomicAdd(&fillc[j], 1u)] = (uint32_t)s;
  }
}

// x_j += Delta_s for s in ascending order (reading D:8); sphere: renormalise
template <typename T, int D>
static __global__ void rbmr_apply_kernel(DevParams P, uint64_t nslots, State<T, D> st,
                                  const uint32_t* __restrict__ off, uint32_t* __restrict__ lst,
                                  const T* __restrict__ delta) {
  const uint32_t m = (uint32_t)*P.step;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < P.n;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t a = off[j], b = off[j + 1];
    if (a == b) continue;
    for (uint32_t u = a + 1; u < b; ++u) {  // insertion sort of the (short) slot list
      const uint32_t v = lst[u];
      uint32_t w = u;
      while (w > a && lst[w - 1] > v) { lst[w] = lst[w - 1]; --w; }
      lst[w] = v;
    }
    T x[D];
#pragma unroll
    for (int c = 0; c < D; ++c) x[c] = st.x[c][j];
    for (uint32_t u = a; u < b; ++u) {
      const uint32_t s = lst[u];
#pragma unroll
      for (int c = 0; c < D; ++c) x[c] += delta[(size_t)c * nslots + s];
    }
    if (P.constraint == 1) renormalise<T, D>(x);
    check_finite<T, D>(x, P, (uint32_t)j, m);
#pragma unroll
    for (int c = 0; c < D; ++c) st.x[c][j] = x[c];
  }
}

// ------------------------------------------------------ device-wide scan (RBM-r)
// exclusive scan of a[0..n) into out[0..n], out[n] = total; 3 phases.
constexpr int SCAN_BLOCK = 1024, SCAN_ITEMS = 4, SCAN_TILE = SCAN_BLOCK * SCAN_ITEMS;
static __global__ void __launch_bounds__(SCAN_BLOCK) scan_reduce_kernel(const uint32_t* __restrict__ a,
                                                                 uint64_t n, uint32_t* part) {
  __shared__ uint32_t ws[33];
  const uint64_t base = (uint64_t)blockIdx.x * SCAN_TILE;
  uint32_t s = 0;
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    const uint64_t i = base + (uint64_t)k * SCAN_BLOCK + threadIdx.x;
    if (i < n) s += a[i];
  }
  const uint32_t inc = warp_incl_scan(s);
  if ((threadIdx.x & 31) == 31) ws[threadIdx.x >> 5] = inc;
  __syncthreads();
  if (threadIdx.x < 32) {
    const uint32_t v = warp_incl_scan(ws[threadIdx.x]);
    if (threadIdx.x == 31) part[blockIdx.x] = v;
  }
}

static __global__ void __launch_bounds__(1024) scan_parts_kernel(uint32_t* part, uint32_t nparts) {
  __shared__ uint32_t ws[34];
  const uint32_t per = (nparts + 1023) / 1024;
  const uint32_t b0 = min(nparts, threadIdx.x * per), b1 = min(nparts, b0 + per);
  uint32_t s = 0;
  for (uint32_t i = b0; i < b1; ++i) s += part[i];
  const uint32_t inc = warp_incl_scan(s);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 31) ws[w] = inc;
  __syncthreads();
  if (w == 0) {
    const uint32_t v = ws[lane];
    ws[lane] = warp_incl_scan(v) - v;
  }
  __syncthreads();
  uint32_t run = ws[w] + inc - s;
  for (uint32_t i = b0; i < b1; ++i) { const uint32_t v = part[i]; part[i] = run; run += v; }
}

static __global__ void __launch_bounds__(SCAN_BLOCK) scan_down_kernel(const uint32_t* __restrict__ a,
                                                               uint64_t n,
                                                               const uint32_t* __restrict__ part,
                                                               uint32_t* out) {
  __shared__ uint32_t ws[34];
  const uint64_t base = (uint64_t)blockIdx.x * SCAN_TILE + (uint64_t)threadIdx.x * SCAN_ITEMS;
  uint32_t v[SCAN_ITEMS], s = 0;
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    const uint64_t i = base + k;
    v[k] = (i < n) ? a[i] : 0u;
    s += v[k];
  }
  const uint32_t inc = warp_incl_scan(s);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 31) ws[w] = inc;
  __syncthreads();
  if (w == 0) {
    const uint32_t x = ws[lane];
    ws[lane] = warp_incl_scan(x) - x;
  }
  __syncthreads();
  uint32_t run = part[blockIdx.x] + ws[w] + inc - s;
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    const uint64_t i = base + k;
    if (i < n) out[i] = run;
    if (i == n - 1) out[n] = run + v[k];
    run += v[k];
  }
}

}  // namespace rbm

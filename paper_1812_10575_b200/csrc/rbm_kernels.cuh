// rbm_kernels.cuh -- the RBM time-step kernels for sm_100a.
//
// RBM-1 step m (Alg. 1) as an MSD key partition into GAPPED
// buckets (fixed capacity per bucket, cursors from zero: no histogram pass)
// fused with an exact in-bucket sort and the batch update:
//   prologue      records in id order -> pass-1 buckets by the top b1 bits of
//                 key_m (first step after init / set_state only)
//   tile_scan     pass-1 counts -> prefix and tile table
//   split         pass-1 bucket d1 -> final buckets (d1, next b2 bits)
//   final_scan    final counts -> exact global bucket starts S[0..2^B]
//   bucket_step   per final bucket: exact in-smem sort by (key_m, id); every
//                 batch inside the bucket does Eq. (2.2) + Euler-Maruyama (or
//                 the exact pair flow / Verlet); the updated records are
//                 partitioned straight into the pass-1 buckets of step m+1
//   straddle      batches that straddle two final buckets
//   advance       m += 1
// Batches are defined on global sorted positions S[b] + rank, so the step's
// permutation is exactly "ids sorted by (key_m(id), id)" whatever the storage.
// The state is an array of RS-byte records (RecL in rbm_device.cuh): every
// move of a particle is one 8/16/32-byte vector access.
#pragma once
#include <type_traits>

#include "rbm_device.cuh"

namespace rbm {

// State buffer: records, plus the side array of shuffle keys that pass 2
// writes for the bucket step when the record has no room for the key.
template <typename T, int D> struct State {
  unsigned char* rec;
  uint32_t* key;
};

// Destination of the records a step writes into the pass-1 segments of the
// next step.  On one GPU (and with the NCCL exchange) st[0] is the local send
// buffer and segment v sits at v * cap.  Fused partitioned mode (row a7, G9):
// segment v belongs to rank v >> nls_log and is stored straight into that
// rank's receive buffer st[rank'] (peer memory over NVLink) as its segment
// (this rank << nls_log) | (v & (nls - 1)) -- the all-to-all is the store.
constexpr int MAXG_FUSED = 8;
template <typename T, int D> struct OutDst {
  State<T, D> st[MAXG_FUSED];
  uint32_t fused, nls_log, rank;
};

template <typename T, int D>
__device__ __forceinline__ void out_put(const OutDst<T, D>& o, uint32_t v, uint32_t cap, uint32_t slot,
                                        const Rec<T, D>& r) {
  uint32_t w = 0;
  size_t g;
  if (o.fused) {
    w = v >> o.nls_log;
    g = (size_t)((o.rank << o.nls_log) | (v & ((1u << o.nls_log) - 1u))) * cap + slot;
  } else {
    g = (size_t)v * cap + slot;
  }
  st_rec<T, D>(o.st[w].rec, (long long)g, r);
}

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

// exclusive scan of a[0..n) in shared memory by the whole block
// wsum: >= 33 uint32 of shared scratch. Returns the total.
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

// out[0..n) = exclusive scan of in[0..n) (n % 4 == 0, 16-B aligned; in and
// out may alias), uint4 chunks per thread.  Returns the total; ends synced.
template <int BLOCK>
__device__ __forceinline__ uint32_t block_excl_scan4(const uint32_t* in, uint32_t* out, int n,
                                                     uint32_t* wsum) {
  const int nq = n >> 2;
  const int per = (nq + BLOCK - 1) / BLOCK;
  const int t = threadIdx.x;
  const int q0 = min(nq, t * per), q1 = min(nq, q0 + per);
  const uint4* in4 = reinterpret_cast<const uint4*>(in);
  uint4* out4 = reinterpret_cast<uint4*>(out);
  uint32_t s = 0;
  for (int q = q0; q < q1; ++q) {
    const uint4 v = in4[q];
    s += v.x + v.y + v.z + v.w;
  }
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
  for (int q = q0; q < q1; ++q) {
    const uint4 v = in4[q];
    uint4 o;
    o.x = run;
    o.y = run + v.x;
    o.z = o.y + v.y;
    o.w = o.z + v.z;
    run = o.w + v.w;
    out4[q] = o;
  }
  const uint32_t total = wsum[32];
  __syncthreads();
  return total;
}

// exclusive scan of nw*2 u16 counts packed in u32 words (low half first);
// out[] gets the packed u16 offsets (totals < 2^16).  nw % 4 == 0.  Ends synced.
template <int BLOCK>
__device__ __forceinline__ void block_excl_scan_u16x2(const uint32_t* in, uint32_t* out, int nw,
                                                      uint32_t* wsum) {
  const int nq = nw >> 2;  // uint4 chunks of 8 counts
  const int per = (nq + BLOCK - 1) / BLOCK;
  const int t = threadIdx.x;
  const int q0 = min(nq, t * per), q1 = min(nq, q0 + per);
  const uint4* in4 = reinterpret_cast<const uint4*>(in);
  uint4* out4 = reinterpret_cast<uint4*>(out);
  uint32_t s = 0;
  for (int q = q0; q < q1; ++q) {
    const uint4 v = in4[q];
    s += (v.x & 0xffffu) + (v.x >> 16) + (v.y & 0xffffu) + (v.y >> 16) + (v.z & 0xffffu) + (v.z >> 16) +
         (v.w & 0xffffu) + (v.w >> 16);
  }
  const uint32_t inc = warp_incl_scan(s);
  const int lane = t & 31, wp = t >> 5;
  if (lane == 31) wsum[wp] = inc;
  __syncthreads();
  if (wp == 0) {
    const uint32_t v = (lane < BLOCK / 32) ? wsum[lane] : 0u;
    const uint32_t vi = warp_incl_scan(v);
    if (lane < BLOCK / 32) wsum[lane] = vi - v;
  }
  __syncthreads();
  uint32_t run = wsum[wp] + inc - s;
  for (int q = q0; q < q1; ++q) {
    const uint4 v = in4[q];
    const uint32_t c[4] = {v.x, v.y, v.z, v.w};
    uint32_t o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t lo = run, hi = run + (c[k] & 0xffffu);
      o[k] = lo | (hi << 16);
      run = hi + (c[k] >> 16);
    }
    out4[q] = make_uint4(o[0], o[1], o[2], o[3]);
  }
  __syncthreads();
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

// batch index of position P, and the [start, end) of batch k (reading D:7)
__device__ __forceinline__ uint32_t batch_index(uint32_t P0, const DevParams& prm) {
  uint32_t k = fdiv(P0, prm.pdiv);
  if (prm.rem == 1 && k + 1 >= prm.nfull) k = prm.nfull - 1;
  return k;
}
__device__ __forceinline__ uint32_t batch_end(uint32_t k, const DevParams& prm) {
  const uint32_t n = (uint32_t)prm.n;
  if (prm.rem == 1 && k + 1 == prm.nfull) return n;
  return min(k * prm.p + prm.p, n);
}

// ------------------------------------------------------------------- init
// X_0 in fp64, rounded to T; records stored in id order.
template <typename T, int D>
static __global__ void init_kernel(const __grid_constant__ DevParams P, State<T, D> st, uint64_t id0, uint64_t n, uint32_t kind,
                                   double a0, double a1, double a2, double a3) {
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
    const uint32_t id = (uint32_t)(id0 + i);
    double x[3] = {0, 0, 0};
    if (kind == 1 || kind == 3 || kind == 4 || kind == 5) {
      double z[D];
      Normals<double, D>::get(P, id, 0u, TAG_INIT, z);
      if (kind == 1 || kind == 5) {
        for (int c = 0; c < D; ++c) x[c] = kind == 5 ? fabs(a0 + a1 * z[c]) : a0 + a1 * z[c];
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
    Rec<T, D> r;
    r.id = id;
    r.key = 0u;
#pragma unroll
    for (int c = 0; c < D; ++c) r.x[c] = (T)x[c];
    st_rec<T, D>(st.rec, (long long)i, r);
  }
}

// user state (id order, row-major N x D) -> records in id order
template <typename T, int D>
static __global__ void set_state_kernel(uint64_t id0, uint64_t n, State<T, D> st, const T* __restrict__ xin) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    Rec<T, D> r;
    r.id = (uint32_t)(id0 + i);
    r.key = 0u;
#pragma unroll
    for (int c = 0; c < D; ++c) r.x[c] = xin[i * D + c];
    st_rec<T, D>(st.rec, (long long)i, r);
  }
}

// records in storage order -> x_out (id order, row-major) for ids [i0, i1)
template <typename T, int D>
static __global__ void gather_kernel(uint64_t n, State<T, D> st, uint64_t i0, uint64_t i1,
                                     T* __restrict__ out) {
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const Rec<T, D> r = ld_rec<T, D>(st.rec, (long long)q);
    const uint64_t id = r.id;
    if (id >= i0 && id < i1) {
#pragma unroll
      for (int c = 0; c < D; ++c) out[(id - i0) * D + c] = r.x[c];
    }
  }
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

static __global__ void iota_kernel(uint32_t* out, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (uint32_t)i;
}

// ------------------------------------------------------------ gapped layout
// nb buckets of fixed capacity cap; bucket u holds cnt[u*cstride] records at
// physical slots [u*cap, u*cap + cnt).  Cursor padding spreads the run-
// reservation atomics of concurrent CTAs over the L2 slices.
constexpr uint32_t CUR1_STRIDE = 8, CUR2_STRIDE = 8;
constexpr uint32_t MAX_SEG = 16384;  // pass-1 segments: 2^b1 << segk <= 2^10 << 4
constexpr uint32_t MAX_SEG_SPLIT = 1024;  // segments the pass-2 splitter's smem tile table holds

__device__ __forceinline__ uint32_t out_seg(const DevParams& P, uint32_t dg, uint32_t salt) {
  return (dg << P.segk) | (salt & P.segmask);
}

struct Gapped {
  uint32_t cap;           // slots per bucket (multiple of 64)
  uint32_t nb;            // buckets
  const uint32_t* cnt;    // counts (= final cursor values)
  uint32_t cstride;       // cursor stride (u32 elements)
};

// gather from a gapped layout: thread per physical slot, holes skipped
template <typename T, int D>
static __global__ void gather_gapped_kernel(Gapped g, State<T, D> st, uint64_t i0, uint64_t i1,
                                            T* __restrict__ out) {
  const uint64_t total = (uint64_t)g.nb * g.cap;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < total;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t u = (uint32_t)(q / g.cap), s = (uint32_t)(q - (uint64_t)u * g.cap);
    if (s >= g.cnt[(size_t)u * g.cstride]) continue;
    const Rec<T, D> r = ld_rec<T, D>(st.rec, (long long)q);
    const uint64_t id = r.id;
    if (id >= i0 && id < i1) {
#pragma unroll
      for (int c = 0; c < D; ++c) out[(id - i0) * D + c] = r.x[c];
    }
  }
}

// tiles of pass 2 over nseg segments (counts cnt[v * CUR1_STRIDE]):
// tile_off[v] = exclusive prefix of ceil(count/tile), tile_off[nseg] = total.
// One block of 1024 threads, each a run of consecutive segments.
__device__ __forceinline__ void seg_tile_table(const uint32_t* __restrict__ cnt, uint32_t nseg,
                                               uint32_t tile, uint32_t* tile_off, uint32_t* ws) {
  const uint32_t per = (nseg + 1023) / 1024;
  const uint32_t v0 = min(nseg, threadIdx.x * per), v1 = min(nseg, v0 + per);
  uint32_t ts = 0;
  for (uint32_t v = v0; v < v1; ++v) ts += (cnt[(size_t)v * CUR1_STRIDE] + tile - 1) / tile;
  const uint32_t inc = warp_incl_scan(ts);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 31) ws[w] = inc;
  __syncthreads();
  if (w == 0) {
    const uint32_t x = ws[lane];
    const uint32_t xi = warp_incl_scan(x);
    ws[lane] = xi - x;
    if (lane == 31) ws[32] = xi;
  }
  __syncthreads();
  uint32_t run = ws[w] + inc - ts;
  for (uint32_t v = v0; v < v1; ++v) {
    tile_off[v] = run;
    run += (cnt[(size_t)v * CUR1_STRIDE] + tile - 1) / tile;
  }
  if (threadIdx.x == 0) tile_off[nseg] = ws[32];
  __syncthreads();
}

// single block: pass-1 counts (2^b1 digits x K segments) -> prefix1 over the
// digits (exclusive, size nb1+1) and the tile table of pass 2 over the
// segments; for one-pass layouts the final starts S = prefix of the counts.
static __global__ void __launch_bounds__(1024) tile_scan_kernel(const __grid_constant__ DevParams P, const uint32_t* __restrict__ cnt1,
                                                                uint32_t* prefix1, uint32_t* tile_off,
                                                                uint32_t* S, uint32_t tile) {
  __shared__ uint32_t a[1025];
  __shared__ uint32_t ws[33];
  const uint32_t nb = 1u << P.b1, K = 1u << P.segk;
  for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) {
    uint32_t c = 0;
    for (uint32_t k = 0; k < K; ++k) c += cnt1[(size_t)((i << P.segk) | k) * CUR1_STRIDE];
    a[i] = c;
  }
  __syncthreads();
  const uint32_t total = block_excl_scan<1024>(a, nb, ws);
  for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) {
    prefix1[i] = a[i];
    if (P.b2 == 0) S[i] = a[i];
  }
  if (threadIdx.x == 0) {
    prefix1[nb] = total;
    if (P.b2 == 0) S[nb] = total;
  }
  seg_tile_table(cnt1, nb << P.segk, tile, tile_off, ws);
}

// one block per pass-1 bucket d1: S[d1<<b2 | d2] = prefix1[d1] + excl-scan of
// the final counts (d1, .)
static __global__ void __launch_bounds__(512) final_scan_kernel(const __grid_constant__ DevParams P, const uint32_t* __restrict__ cnt2,
                                                                const uint32_t* __restrict__ prefix1,
                                                                uint32_t* S) {
  __shared__ uint32_t a[1024];
  __shared__ uint32_t ws[33];
  const uint32_t u = blockIdx.x, nb2 = 1u << P.b2, base = u << P.b2;
  for (uint32_t i = threadIdx.x; i < nb2; i += blockDim.x) a[i] = cnt2[(size_t)(base + i) * CUR2_STRIDE];
  __syncthreads();
  block_excl_scan<512>(a, nb2, ws);
  const uint32_t o = prefix1[u];
  for (uint32_t i = threadIdx.x; i < nb2; i += blockDim.x) S[base + i] = o + a[i];
  if (u == 0 && threadIdx.x == 0) S[P.nbuckets] = prefix1[gridDim.x];  // end of this rank's range
}

// tile t of pass 2: pass-1 bucket u and its element range [lo, hi) (relative)
__device__ __forceinline__ bool gapped_tile(const uint32_t* __restrict__ tile_off,
                                            const uint32_t* __restrict__ cnt1, uint32_t nb1,
                                            uint32_t t, uint32_t tile, uint32_t& u, uint32_t& lo,
                                            uint32_t& hi) {
  if (t >= tile_off[nb1]) return false;
  uint32_t a = 0, b = nb1;  // largest u with tile_off[u] <= t
  while (b - a > 1) {
    const uint32_t mid = (a + b) >> 1;
    if (tile_off[mid] <= t) a = mid; else b = mid;
  }
  u = a;
  lo = (t - tile_off[u]) * tile;
  hi = min(lo + tile, cnt1[(size_t)u * CUR1_STRIDE]);
  return true;
}

// ------------------------------------------------------------- prologue
// Records in any storage order (contiguous [0, nsrc)) -> the gapped buckets
// of step m by the top b1 bits of key_m (computed from the ids; carried in
// keyed records).  Records are staged in shared memory by digit so that each
// reserved run is written coalesced.  Order inside a bucket is irrelevant:
// the bucket step sorts exactly.
template <typename T, int D> __host__ __device__ constexpr int prologue_tile() {  // <= 64 KB of staged records
  return ((65536 / RecL<T, D>::RS) < 4096 ? (65536 / RecL<T, D>::RS) : 4096) / 256 * 256;
}
template <typename T, int D, int BLOCK> __host__ __device__ constexpr size_t prologue_smem_bytes() {
  return (1024 + 1024 + 64) * 4 + (size_t)prologue_tile<T, D>() * (RecL<T, D>::RS + 2);
}

template <typename T, int D, int BLOCK>
static __global__ void __launch_bounds__(BLOCK) prologue_kernel(const __grid_constant__ DevParams P, State<T, D> src,
                                                                const __grid_constant__ OutDst<T, D> dst, uint32_t* cur,
                                                                uint32_t dcap, uint64_t nsrc) {
  constexpr int TILE = prologue_tile<T, D>();
  constexpr int ITEMS = TILE / BLOCK;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem_raw);  // 1024
  uint32_t* gbase = hist + 1024;                           // 1024
  uint32_t* wsum = gbase + 1024;                           // 64
  unsigned char* stg = reinterpret_cast<unsigned char*>(wsum + 64);  // TILE records
  uint16_t* st_dig = reinterpret_cast<uint16_t*>(stg + (size_t)TILE * RecL<T, D>::RS);

  const uint32_t lo = blockIdx.x * TILE;
  if (lo >= nsrc) return;
  const uint32_t hi = (uint32_t)min((uint64_t)lo + TILE, nsrc);
  const uint32_t sh = 32u - P.b1, nbins = 1u << P.b1;
  for (uint32_t i = threadIdx.x; i < nbins; i += BLOCK) hist[i] = 0;
  __syncthreads();
  const uint32_t m = (uint32_t)*P.step;
  const uint32_t cnt = hi - lo;
  uint32_t rds[ITEMS];
  Rec<T, D> rr[ITEMS];
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const uint32_t e = k * BLOCK + threadIdx.x;
    if (e < cnt) rr[k] = ld_rec<T, D>(src.rec, (long long)(lo + e));
  }
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const uint32_t e = k * BLOCK + threadIdx.x;
    if (e < cnt) {
      rr[k].key = shuffle_key(P, rr[k].id, m);
      const uint32_t dg = rr[k].key >> sh;
      rds[k] = (dg << 16) | atomicAdd(&hist[dg], 1u);
    }
  }
  __syncthreads();
  // reserve runs in the destination buckets, then local exclusive offsets
  for (uint32_t i = threadIdx.x; i < nbins; i += BLOCK) {
    const uint32_t h = hist[i];
    gbase[i] = h ? atomicAdd(&cur[(size_t)out_seg(P, i, blockIdx.x) * CUR1_STRIDE], h) : 0u;
  }
  block_excl_scan<BLOCK>(hist, nbins, wsum);  // hist -> local offsets
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const uint32_t e = k * BLOCK + threadIdx.x;
    if (e < cnt) {
      const uint32_t dg = rds[k] >> 16;
      const uint32_t s = hist[dg] + (rds[k] & 0xffffu);
      RBM_CHECK(P, s < cnt);
      st_rec<T, D>(stg, s, rr[k]);
      st_dig[s] = (uint16_t)dg;
    }
  }
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < cnt; j += BLOCK) {
    const uint32_t dg = st_dig[j];
    const uint32_t slot = gbase[dg] + (j - hist[dg]);
    if (slot >= dcap) {  // bucket capacity exceeded (probability ~1e-30): fail loudly
      atomicExch(P.capacity_err, 1u);
      continue;
    }
    out_put<T, D>(dst, out_seg(P, dg, blockIdx.x), dcap, slot, ld_rec<T, D>(stg, j));
  }
}

// ------------------------------------------- persistent pass-2 splitter
// Tiles of the pass-1 buckets (segments) -> final buckets by the next b2 key
// bits.  One 1024-thread CTA per SM loops over tiles with a two-stage TMA
// ring (one bulk copy of TILE records per stage, L2 evict-first), split into
// two warp groups that work on different tiles at once:
//   rank group (warps 0..15): key of every record (Philox for unkeyed
//     records), its rank in its digit (shared-memory atomics), one run
//     reservation per digit, the digit offsets, and the tile's output order
//     (staging index + the keys in output order) for stage s;
//   write group (warps 16..31): the coalesced runs of stage s (one vector
//     store per record, + the side key), then the TMA load of the tile after
//     next into the freed stage.
// So the stores of tile t overlap the key / rank work of tile t+1 (before:
// the phases of one tile ran one after the other in the whole CTA).
// Stage handshakes are mbarriers: tma[s] (bytes landed), full[s] (staging
// index of stage s ready); every per-stage array is double-buffered.
// record traits of the splitter: the state records (key carried, or from
// the id by Philox -> side key array), or the RBM-r increment records (the
// partition key is the particle index j, left-aligned to 32 bits)
template <typename T, int D> struct StateRT {
  static constexpr int RS = RecL<T, D>::RS, NW = RecL<T, D>::NW;
  static constexpr bool SIDE = !RecL<T, D>::KEYED;
  __device__ __forceinline__ static uint32_t key(const DevParams& P, const unsigned char* r, uint32_t m) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(r);
    return RecL<T, D>::KEYED ? w[1] : shuffle_key(P, w[0], m);
  }
};
// RBM-r increment record {j, [pad,] Delta_s[D]}: fp32 d=1 8 B, fp32 d=2/3 and
// fp64 d=1 16 B, fp64 d=2/3 32 B.  The slot index s is not carried: a
// particle's increments are summed order-independently (Fx below, reading D:8)
template <typename T, int D> struct IncL {
  static constexpr int XW = (int)(sizeof(T) / 4);  // word offset of Delta[0] (fp64: 8-byte aligned)
  static constexpr int RS0 = 4 * XW + D * (int)sizeof(T);
  static constexpr int RS = RS0 <= 8 ? 8 : (RS0 + 15) / 16 * 16;
  static constexpr int NW = RS / 4;
};
// Order-independent sum of a particle's increments (reading D:8): every
// increment coordinate is converted exactly to a fixed-point integer at the
// scale of the particle's largest increment exponent E (over all its
// increments and coordinates; G guard bits below the ulp of that scale, bits
// further down truncated), the integers are summed exactly (so the order of
// the increments does not matter), and each coordinate's sum is added to x
// with one rounding.  On one GPU the sum is formed by 32-bit shared-memory
// atomics on NCH chunks of CB bits of q + BIAS (64-bit shared atomics are CAS
// loops on sm_100a); the partitioned path sums the same integers in int64.
template <typename T> struct Fx;
template <> struct Fx<float> {
  static constexpr int G = 16;                     // |q| < 2^40
  static constexpr int NCH = 2, CB = 21;           // q + 2^40 in two chunks: u32 sums of < 2^11 increments
  static constexpr long long BIAS = 1ll << 40;
  __device__ __forceinline__ static uint32_t ex(float v) {
    const uint32_t e = (__float_as_uint(v) >> 23) & 0xffu;
    return e ? e : 1u;
  }
  __device__ __forceinline__ static long long q(float v, uint32_t E) {
    const uint32_t u = __float_as_uint(v), e = (u >> 23) & 0xffu;
    const unsigned long long mant = (unsigned long long)((u & 0x7fffffu) | (e ? 0x800000u : 0u)) << G;
    const uint32_t sh = E - (e ? e : 1u);
    const long long mag = sh >= 64u ? 0ll : (long long)(mant >> sh);
    return (u >> 31) ? -mag : mag;
  }
  __device__ __forceinline__ static float add(float x, long long acc, uint32_t E) {
    if (E >= 255u) return __int_as_float(0x7fc00000);  // a non-finite increment: flagged downstream
    // 2^(E - 150 - G) is a normal double for every E in [1, 254]: exact scaling
    const double sc = __longlong_as_double((long long)(E - 150 - G + 1023) << 52);
    return (float)((double)x + (double)acc * sc);
  }
};
template <> struct Fx<double> {
  static constexpr int G = 4;                      // |q| < 2^57: int64 sums of < 64 increments
  static constexpr int NCH = 3, CB = 20;           // q + 2^57 in three chunks: u32 sums of < 2^12 increments
  static constexpr long long BIAS = 1ll << 57;
  __device__ __forceinline__ static uint32_t ex(double v) {
    const uint32_t e = (uint32_t)(((unsigned long long)__double_as_longlong(v) >> 52) & 0x7ffu);
    return e ? e : 1u;
  }
  __device__ __forceinline__ static long long q(double v, uint32_t E) {
    const unsigned long long u = (unsigned long long)__double_as_longlong(v);
    const uint32_t e = (uint32_t)((u >> 52) & 0x7ffu);
    const unsigned long long mant = ((u & 0xfffffffffffffull) | (e ? 0x10000000000000ull : 0ull)) << G;
    const uint32_t sh = E - (e ? e : 1u);
    const long long mag = sh >= 64u ? 0ll : (long long)(mant >> sh);
    return (u >> 63) ? -mag : mag;
  }
  __device__ __forceinline__ static double add(double x, long long acc, uint32_t E) {
    if (E >= 2047u) return __longlong_as_double(0x7ff8000000000000ll);
    const int ex2 = (int)E - 1075 - G;  // >= -1078: below the normal range for the smallest E
    return x + (ex2 >= -1022 ? (double)acc * __longlong_as_double((long long)(ex2 + 1023) << 52)
                             : ldexp((double)acc, ex2));
  }
};
template <typename T, int D> struct IncRT {
  static constexpr int RS = IncL<T, D>::RS, NW = IncL<T, D>::NW;
  static constexpr bool SIDE = false;
  __device__ __forceinline__ static uint32_t key(const DevParams& P, const unsigned char* r, uint32_t) {
    return reinterpret_cast<const uint32_t*>(r)[0] << P.jshift;
  }
};

#ifndef RBM_SPLIT_STAGE  // design-experiment builds override these (build.py -D...)
#define RBM_SPLIT_STAGE 65536
#endif
constexpr int SPLIT_BLOCK = 1024, SPLIT_MINB = 1;  // one CTA of 2 x 512 threads per SM
constexpr int SPLIT_GRP = SPLIT_BLOCK / 2;          // threads per warp group
// RBM-r' link record {j, s} (8 bytes)
struct LinkL {
  static constexpr int RS = 8, NW = 2;
};
struct LinkRT {
  static constexpr int RS = LinkL::RS, NW = LinkL::NW;
  static constexpr bool SIDE = false;
  __device__ __forceinline__ static uint32_t key(const DevParams& P, const unsigned char* r, uint32_t) {
    return reinterpret_cast<const uint32_t*>(r)[0] << P.jshift;
  }
};
template <typename T, int D, bool LINK> using IncOrLink = std::conditional_t<LINK, LinkL, IncL<T, D>>;

template <class RT> __host__ __device__ constexpr int split_tile_rt() {
  return (RBM_SPLIT_STAGE / RT::RS) < 4096 ? (RBM_SPLIT_STAGE / RT::RS) : 4096;  // <= one stage of records
}
// header: hist, off (1024 each), wsum (64), 4 mbarriers, 2 tile infos, gbase[2][1024]
constexpr size_t SPLIT_HDR = (((2 * 1024 + 64) * 4 + 4 * 8 + 2 * 16 + 2 * 1024 * 4) + 127) & ~(size_t)127;
template <class RT> __host__ __device__ constexpr size_t split_smem_bytes_rt() {
  return SPLIT_HDR + 2 * (size_t)split_tile_rt<RT>() * RT::RS                 // stages
         + 2 * (size_t)split_tile_rt<RT>() * 4                                // staging index per stage
         + (RT::SIDE ? 2 * (size_t)split_tile_rt<RT>() * 4 : 0)               // keys in output order per stage
         + (size_t)(MAX_SEG_SPLIT + 1) * 4 + (size_t)MAX_SEG_SPLIT * 4;       // tile table, segment counts
}
template <typename T, int D> __host__ __device__ constexpr int split_tile() { return split_tile_rt<StateRT<T, D>>(); }
template <typename T, int D> __host__ __device__ constexpr size_t split_smem_bytes() {
  return split_smem_bytes_rt<StateRT<T, D>>();
}

struct TileInfo { uint32_t u, lo, hi, pad; };

__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// exclusive scan of a[0..n) (n <= 2 GRP) by the GRP threads of a warp group
// (local index lt, named barrier bid); returns with a[] scanned, group synced
template <int GRP>
__device__ __forceinline__ void group_excl_scan(uint32_t* a, uint32_t n, uint32_t* wsum, uint32_t lt, int bid) {
  const uint32_t per = (n + GRP - 1) / GRP;
  const uint32_t b0 = min(n, lt * per), b1 = min(n, b0 + per);
  uint32_t s = 0;
  for (uint32_t i = b0; i < b1; ++i) s += a[i];
  const uint32_t inc = warp_incl_scan(s);
  const uint32_t lane = lt & 31, w = lt >> 5;
  if (lane == 31) wsum[w] = inc;
  named_bar(bid, GRP);
  if (w == 0) {
    const uint32_t v = (lane < GRP / 32) ? wsum[lane] : 0u;
    const uint32_t vi = warp_incl_scan(v);
    if (lane < GRP / 32) wsum[lane] = vi - v;
  }
  named_bar(bid, GRP);
  uint32_t run = wsum[w] + inc - s;
  for (uint32_t i = b0; i < b1; ++i) { const uint32_t v = a[i]; a[i] = run; run += v; }
  named_bar(bid, GRP);
}

template <class RT, int BLOCK>
static __global__ void __launch_bounds__(BLOCK, SPLIT_MINB) split_kernel(const __grid_constant__ DevParams P,
                                                                const unsigned char* __restrict__ src_rec,
                                                                unsigned char* __restrict__ dst_rec,
                                                                uint32_t* __restrict__ dst_key,
                                                                uint32_t* cur, uint32_t dcap,
                                                                const uint32_t* __restrict__ cnt1,
                                                                const uint32_t* __restrict__ tile_off,
                                                                uint32_t scap) {
  using L = RT;
  constexpr int TILE = split_tile_rt<RT>();
  constexpr int GRP = BLOCK / 2;
  static_assert(GRP == SPLIT_GRP && GRP % 32 == 0, "two equal warp groups");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  RBM_PROF_BEGIN(P);
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem_raw);  // 1024 (rank group)
  uint32_t* off = hist + 1024;                             // 1024 (rank group)
  uint32_t* wsum = off + 1024;                             // 64
  uint64_t* tma = reinterpret_cast<uint64_t*>(wsum + 64);  // 2: stage s landed
  uint64_t* full = tma + 2;                                // 2: staging index of stage s ready
  TileInfo* tinfo = reinterpret_cast<TileInfo*>(full + 2); // 2
  uint32_t* gbase2 = reinterpret_cast<uint32_t*>(tinfo + 2);  // [2][1024]
  unsigned char* stg0 = smem_raw + SPLIT_HDR;
  constexpr size_t SBY = (size_t)TILE * L::RS;
  uint32_t* invd2 = reinterpret_cast<uint32_t*>(stg0 + 2 * SBY);  // [2][TILE]: element | digit << 16, by output slot
  uint32_t* kls2 = invd2 + 2 * TILE;                               // [2][TILE]: key_m by output slot (unkeyed)
  uint32_t* toff = kls2 + (L::SIDE ? 2 * TILE : 0);                // copy of tile_off (binary search in smem)
  uint32_t* cnts = toff + MAX_SEG_SPLIT + 1;                       // segment counts
  const uint32_t nseg = (1u << P.b1) << P.segk;
  const uint32_t ntiles = tile_off[nseg];
  const uint32_t bits = P.b2, sh = 32u - P.b1 - P.b2, nbins = 1u << bits, mask = nbins - 1u;
  const uint32_t tid = threadIdx.x;
  const uint32_t m = (uint32_t)*P.step;
  for (uint32_t i = tid; i <= nseg; i += BLOCK) toff[i] = tile_off[i];
  for (uint32_t i = tid; i < nseg; i += BLOCK) cnts[i] = cnt1[(size_t)i * CUR1_STRIDE];
  // tile t into stage st (one thread): its info, then one bulk copy
  auto issue = [&](uint32_t t, uint32_t st, uint64_t pol) {
    TileInfo ti{0u, 0u, 0u, 0u};
    const uint32_t tt = min(t, ntiles - 1u);
    uint32_t a = 0, b = nseg;  // largest u with toff[u] <= tt
    while (b - a > 1) {
      const uint32_t mid = (a + b) >> 1;
      if (toff[mid] <= tt) a = mid; else b = mid;
    }
    ti.u = a;
    ti.lo = (tt - toff[a]) * TILE;
    ti.hi = min(ti.lo + TILE, cnts[a]);
    tinfo[st] = ti;
    const uint32_t cnt = ti.hi - ti.lo;
    const uint32_t bytes = (cnt * (uint32_t)L::RS + 15u) & ~15u;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&tma[st], bytes);
    if (cnt) bulk_g2s_stream(stg0 + st * SBY, src_rec + ((size_t)ti.u * scap + ti.lo) * L::RS, bytes, &tma[st], pol);
  };
  __syncthreads();  // toff, cnts
  if (tid == 0) {
    mbar_init(&tma[0], 1);
    mbar_init(&tma[1], 1);
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    const uint64_t pol = l2_evict_first_policy();
    if (blockIdx.x < ntiles) issue(blockIdx.x, 0, pol);
    if (blockIdx.x + gridDim.x < ntiles) issue(blockIdx.x + gridDim.x, 1, pol);
  }
  __syncthreads();
  if (tid < GRP) {
    // ---------------------------------------------------------- rank group
    const uint32_t lt = tid;
    constexpr int PER = (TILE + GRP - 1) / GRP;
    uint32_t it = 0;
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const uint32_t s = it & 1u, ph = (it >> 1) & 1u;
      for (uint32_t i = lt; i < nbins; i += GRP) hist[i] = 0;
      mbar_wait(&tma[s], ph);
      named_bar(1, GRP);  // hist zeroed (and off / wsum of the previous tile consumed)
      RBM_PROF(P, 16);
      const TileInfo ti = tinfo[s];
      const uint32_t cnt = ti.hi - ti.lo;
      const unsigned char* stg = stg0 + s * SBY;
      uint32_t* invd = invd2 + s * TILE;
      uint32_t* kls = kls2 + s * TILE;
      uint32_t* gbase = gbase2 + s * 1024;
      const uint32_t dbase0 = ((ti.u >> P.segk) & P.nb1_loc_mask) << P.b2;
      // PER records per thread: keys computed together (independent Philox
      // chains for unkeyed records), then ranked in their digits
      uint32_t kk[PER], rk[PER];
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const uint32_t e = min(lt + k * GRP, cnt ? cnt - 1 : 0u);
        kk[k] = RT::key(P, stg + (size_t)e * L::RS, m);
      }
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const uint32_t e = lt + k * GRP;
        if (e < cnt) {
          const uint32_t dg = (kk[k] >> sh) & mask;
          rk[k] = (dg << 16) | atomicAdd(&hist[dg], 1u);
        }
      }
      named_bar(1, GRP);
      RBM_PROF(P, 17);
      // run reservations issued now and consumed after the offsets scan
      constexpr int NRES = (1024 + GRP - 1) / GRP;
      uint32_t gres[NRES];
#pragma unroll
      for (int r = 0; r < NRES; ++r) {
        const uint32_t i = lt + r * GRP;
        const uint32_t h = i < nbins ? hist[i] : 0u;
        if (i < nbins) off[i] = h;
        gres[r] = h ? atomicAdd(&cur[(size_t)(dbase0 + i) * CUR2_STRIDE], h) : 0u;
      }
      named_bar(1, GRP);
      group_excl_scan<GRP>(off, nbins, wsum, lt, 1);
      RBM_PROF(P, 18);
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const uint32_t e = lt + k * GRP;
        if (e < cnt) {
          const uint32_t pos = off[rk[k] >> 16] + (rk[k] & 0xffffu);
          RBM_CHECK(P, pos < cnt);
          invd[pos] = e | (rk[k] & 0xffff0000u);
          if (L::SIDE) kls[pos] = kk[k];
        }
      }
      // gbase[d] - off[d]: the global slot of output position j is gbase[dg] + j
#pragma unroll
      for (int r = 0; r < NRES; ++r)
        if (lt + r * GRP < nbins) gbase[lt + r * GRP] = gres[r] - off[lt + r * GRP];
      named_bar(1, GRP);
      if (lt == 0) mbar_arrive(&full[s]);  // release: the write group may take stage s
      RBM_PROF(P, 19);
    }
  } else {
    // --------------------------------------------------------- write group
    const uint32_t lt = tid - GRP;
    const uint64_t pol = (lt == 0) ? l2_evict_first_policy() : 0ull;
    uint32_t it = 0;
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const uint32_t s = it & 1u, ph = (it >> 1) & 1u;
      mbar_wait(&full[s], ph);
      const TileInfo ti = tinfo[s];
      const uint32_t cnt = ti.hi - ti.lo;
      const unsigned char* stg = stg0 + s * SBY;
      const uint32_t* invd = invd2 + s * TILE;
      const uint32_t* kls = kls2 + s * TILE;
      const uint32_t* gbase = gbase2 + s * 1024;
      const uint32_t dbase0 = ((ti.u >> P.segk) & P.nb1_loc_mask) << P.b2;
      for (uint32_t j = lt; j < cnt; j += GRP) {
        const uint32_t v = invd[j];
        const uint32_t e = v & 0xffffu, dg = v >> 16;
        RBM_CHECK(P, e < cnt && dg < nbins);
        const uint32_t slot = gbase[dg] + j;
        if (slot >= dcap) {  // bucket capacity exceeded (probability ~1e-30): fail loudly
          atomicExch(P.capacity_err, 1u);
          continue;
        }
        const size_t g = (size_t)(dbase0 + dg) * dcap + slot;
        uint32_t w[L::NW];
        ld_words<L::NW>(stg + (size_t)e * L::RS, w);
        st_words<L::NW>(dst_rec + g * L::RS, w);
        if (L::SIDE) dst_key[g] = kls[j];
      }
      named_bar(2, GRP);  // stage s, its staging index and tile info consumed
      if (lt == 0 && t + 2 * gridDim.x < ntiles) issue(t + 2 * gridDim.x, s, pol);
      if (lt == 0 && P.prof) atomicAdd(&P.prof[62], 1ull);
    }
  }
}

// copy one record (NW words) from src_rec to segment v, slot `slot` of dst
template <typename T, int D>
__device__ __forceinline__ void out_copy(const OutDst<T, D>& o, uint32_t v, uint32_t cap, uint32_t slot,
                                         const unsigned char* src_rec) {
  using L = RecL<T, D>;
  uint32_t w = 0;
  size_t g;
  if (o.fused) {
    w = v >> o.nls_log;
    g = (size_t)((o.rank << o.nls_log) | (v & ((1u << o.nls_log) - 1u))) * cap + slot;
  } else {
    g = (size_t)v * cap + slot;
  }
  uint32_t wd[L::NW];
  ld_words<L::NW>(src_rec, wd);
  st_words<L::NW>(o.st[w].rec + g * L::RS, wd);
}

// ------------------------------------------------------- bucket step pieces
// 1/(|B|-1) for the three batch sizes the division produces (D:7): p, p + 1
// (N mod p = 1) and r = N mod p >= 2; host-computed, no division here
template <typename T> __device__ __forceinline__ T batch_inv(const DevParams& P, uint32_t sz) {
  RBM_CHECK(P, sz == P.p || sz == P.p + 1 || (sz == P.rem && sz >= 2));
  return (sz == P.p) ? Prm<T>::invp(P) : (sz == P.p + 1 ? Prm<T>::invp1(P) : Prm<T>::invr(P));
}

// coordinates of record e in a shared-memory (or scratch) record array
template <typename T, int D> struct RX {
  unsigned char* base;
  __device__ __forceinline__ void get(uint32_t e, T (&x)[D]) const {
    const Rec<T, D> r = ld_rec<T, D>(base, e);
#pragma unroll
    for (int c = 0; c < D; ++c) x[c] = r.x[c];
  }
};

// member q of batch [l0, l1) (sorted positions, ord -> element): Eq. (2.2) +
// Euler-Maruyama / Verlet, or the exact pair flow (INTEG 1, p = 2)
template <typename T, int D, int KK, int INTEG, typename GetX>
__device__ __forceinline__ void interior_update(const DevParams& P, uint32_t m, uint32_t q,
                                                uint32_t l0, uint32_t l1, const uint16_t* ord,
                                                GetX xs, uint32_t id, T (&xn)[D], int vstart = -1) {
  T xi[D];
  const uint32_t e = ord[q];
  xs.get(e, xi);
  T z[D];
#pragma unroll
  for (int c = 0; c < D; ++c) z[c] = T(0);
  if (P.has_noise) Normals<T, D>::get(P, id, m, TAG_NOISE, z);
  if (INTEG != 1) {
    T f[D];
#pragma unroll
    for (int c = 0; c < D; ++c) f[c] = T(0);
    batch_force<T, D, KK, INTEG>(P, q - l0, l1 - l0, xi, [&](uint32_t j, T (&xj)[D]) {
      xs.get(ord[l0 + j], xj);
    }, f);
    const T inv = batch_inv<T>(P, l1 - l0);
#pragma unroll
    for (int c = 0; c < D; ++c) f[c] *= inv;
    member_update<T, D, INTEG>(xi, f, z, xn, P, vstart < 0 ? P.verlet_start != 0 : vstart != 0);
  } else {
    T xa[D], xb[D], y[D];
    xs.get(ord[l0], xa);
    xs.get(ord[l0 + 1], xb);
    pair_flow<T, D, KK>(xa, xb, q == l0, y, P);
    split_finish<T, D>(y, z, xn, P, true);
  }
}

// One batch [l0, l1) handled by one thread (a remainder batch larger than the
// lane group, or p > 32): every member from the old positions, then written
// back in place (keyed records carry key_{m+1}); tb[e] = output digit << 16 | rank in it.
template <typename T, int D, int KK, int INTEG>
__device__ __noinline__ void serial_batch(const DevParams& P, uint32_t m, uint32_t l0, uint32_t l1,
                                          const uint16_t* ord, unsigned char* rs,
                                          uint32_t* tb, uint32_t* ocnt, uint32_t osh) {
  T xn[65][D];
  const RX<T, D> xs{rs};
  for (uint32_t q = l0; q < l1; ++q) {
    T out[D];
    interior_update<T, D, KK, INTEG>(P, m, q, l0, l1, ord, xs, ld_id<T, D>(rs, ord[q]), out);
#pragma unroll
    for (int c = 0; c < D; ++c) xn[q - l0][c] = out[c];
  }
  for (uint32_t q = l0; q < l1; ++q) {
    const uint32_t e = ord[q];
    Rec<T, D> r = ld_rec<T, D>(rs, e);
    check_finite<T, D>(xn[q - l0], P, r.id, m);
    const uint32_t kn = shuffle_key(P, r.id, m + 1);
#pragma unroll
    for (int c = 0; c < D; ++c) r.x[c] = xn[q - l0][c];
    r.key = kn;
    st_rec<T, D>(rs, e, r);
    tb[e] = ((kn >> osh) << 16) | atomicAdd(&ocnt[kn >> osh], 1u);
  }
}

template <typename T, int D, int KK, int INTEG>
__device__ __forceinline__ void pair_update(const DevParams& P, uint32_t m, const T (&x0)[D],
                                            const T (&x1)[D], uint32_t id0, uint32_t id1,
                                            T (&y0)[D], T (&y1)[D]) {
  T z0[D], z1[D];
#pragma unroll
  for (int c = 0; c < D; ++c) { z0[c] = T(0); z1[c] = T(0); }
  if (P.has_noise) {
    Normals<T, D>::get(P, id0, m, TAG_NOISE, z0);
    Normals<T, D>::get(P, id1, m, TAG_NOISE, z1);
  }
  if (INTEG == 0) {
    T zz[D], f0[D], f1[D];
#pragma unroll
    for (int c = 0; c < D; ++c) zz[c] = x0[c] - x1[c];
    const T sc = kernel_scale<T, D, KK>(zz, P);  // 1/(p-1) = 1
#pragma unroll
    for (int c = 0; c < D; ++c) { f0[c] = sc * zz[c]; f1[c] = -f0[c]; }
    em_update<T, D>(x0, f0, z0, y0, P, true);
    em_update<T, D>(x1, f1, z1, y1, P, true);
  } else if (INTEG == 2) {  // Verlet: 1-D force on the positions; the partner gets -f
    T f0[D], f1[D];
#pragma unroll
    for (int c = 0; c < D; ++c) { f0[c] = T(0); f1[c] = T(0); }
    add_force1<T, D, KK>(x0, x1, f0, P);
    f1[0] = -f0[0];
    verlet_update<T, D>(x0, f0, y0, P, P.verlet_start != 0);
    verlet_update<T, D>(x1, f1, y1, P, P.verlet_start != 0);
  } else {
    T a[D], b[D];
    pair_flow<T, D, KK>(x0, x1, true, a, P);
    pair_flow<T, D, KK>(x0, x1, false, b, P);
    split_finish<T, D>(a, z0, y0, P, true);
    split_finish<T, D>(b, z1, y1, P, true);
  }
}

// Oversized bucket (never expected at the automatic capacity; forced in
// tests): the same sort and update on one of NBIG global-memory scratch slots,
// claimed from a small pool and released at the end (holders are resident, so
// waiters always make progress).  All records are written back to the
// bucket's own gapped range in sorted order (straddlers unchanged, for the
// straddle kernel); the interior ones are then appended one by one to the
// step-(m+1) buckets.
template <typename T, int D, int KK, int INTEG, int BLOCK>
__device__ __noinline__ void big_bucket(const DevParams& P, State<T, D> src, const OutDst<T, D>& dst,
                                        uint32_t* cur_next, uint32_t s0, uint32_t sb, uint32_t n,
                                        uint32_t m, uint32_t dcap, uint32_t* cnt, uint32_t* off,
                                        uint32_t* wsum) {
  using L = RecL<T, D>;
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
  unsigned char* base = P.big_scratch + slot * big_slot_bytes(L::RS);
  unsigned long long* ks = reinterpret_cast<unsigned long long*>(base);
  unsigned char* rs = reinterpret_cast<unsigned char*>(ks + BIG_CAP + 1);
  uint32_t* key_l = reinterpret_cast<uint32_t*>(rs + (size_t)BIG_CAP * L::RS);
  uint16_t* ord = reinterpret_cast<uint16_t*>(key_l + BIG_CAP);
  const RX<T, D> xs{rs};
  for (uint32_t i = threadIdx.x; i < 256; i += BLOCK) cnt[i] = 0;
  __syncthreads();
  // keys (carried, side array or Philox); counting sort by the 8 key bits
  // below the B-bit prefix
  const uint32_t sh = (P.B <= 24u) ? (24u - P.B) : 0u;
  for (uint32_t e = threadIdx.x; e < n; e += BLOCK) {
    const Rec<T, D> r = ld_rec<T, D>(src.rec, (long long)sb + e);
    st_rec<T, D>(rs, e, r);
    const uint32_t key = L::KEYED ? r.key : (P.side_key ? src.key[sb + e] : shuffle_key(P, r.id, m));
    key_l[e] = key;
    ord[e] = (uint16_t)atomicAdd(&cnt[(key >> sh) & 255u], 1u);
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < 256; i += BLOCK) off[i] = cnt[i];
  __syncthreads();
  block_excl_scan<BLOCK>(off, 256, wsum);
  for (uint32_t e = threadIdx.x; e < n; e += BLOCK) {
    const uint32_t key = key_l[e];
    ks[off[(key >> sh) & 255u] + ord[e]] = ((unsigned long long)key << 32) | ld_id<T, D>(rs, e);
  }
  __syncthreads();
  // exact rank = sub-bucket offset + #smaller (key, id) composites in the sub-bucket
  for (uint32_t e = threadIdx.x; e < n; e += BLOCK) {
    const uint32_t key = key_l[e];
    const unsigned long long mine = ((unsigned long long)key << 32) | ld_id<T, D>(rs, e);
    const uint32_t sd = (key >> sh) & 255u;
    const uint32_t a = off[sd], c = cnt[sd];
    uint32_t r = a;
    for (uint32_t j = a; j < a + c; ++j) r += (ks[j] < mine) ? 1u : 0u;
    ord[r] = (uint16_t)e;
  }
  __syncthreads();
  // batches inside [s0, s0+n): Eq. (2.2) + update from the scratch copy,
  // written to the own gapped range in sorted order; straddlers copied through
  for (uint32_t q = threadIdx.x; q < n; q += BLOCK) {
    const uint32_t P0 = s0 + q;
    uint32_t b0, b1;
    batch_range(P0, P, b0, b1);
    Rec<T, D> r = ld_rec<T, D>(rs, ord[q]);
    if (b0 >= s0 && b1 <= s0 + n) {
      T xn[D];
      interior_update<T, D, KK, INTEG>(P, m, q, b0 - s0, b1 - s0, ord, xs, r.id, xn);
      check_finite<T, D>(xn, P, r.id, m);
#pragma unroll
      for (int c = 0; c < D; ++c) r.x[c] = xn[c];
    }
    st_rec<T, D>(src.rec, (long long)sb + q, r);
    if (P.dbg_order) P.dbg_order[P0] = r.id;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicExch(&P.big_claim[slot], 0u);
  }
  const uint32_t osh = 32u - P.b1;
  for (uint32_t q = threadIdx.x; q < n; q += BLOCK) {
    uint32_t b0, b1;
    batch_range(s0 + q, P, b0, b1);
    if (b0 >= s0 && b1 <= s0 + n) {
      Rec<T, D> r = ld_rec<T, D>(src.rec, (long long)sb + q);
      r.key = shuffle_key(P, r.id, m + 1);
      const uint32_t v = out_seg(P, r.key >> osh, blockIdx.x);
      const uint32_t s = atomicAdd(&cur_next[(size_t)v * CUR1_STRIDE], 1u);
      if (s >= dcap) { atomicExch(P.capacity_err, 1u); continue; }
      out_put<T, D>(dst, v, dcap, s, r);
    }
  }
}

// ------------------------------------------------------------ bucket step
// One CTA per final bucket b of step m (gapped, capacity scap; global start
// S[b]):
//   (1) TMA bulk load of the bucket's records (and side keys) into smem;
//   (2) exact sort by (key_m, id): counting sort on SB sub-digit bits (packed
//       u16 counters) + rank among 32-bit (low key bits, id) composites;
//   (3) Eq. (2.2) + update of every batch inside the bucket, in place:
//       MODE_PAIR (p = 2): one thread per pair; MODE_GROUP: one lane group
//       of G = pow2 >= p lanes per batch (p <= 32; shuffles, each pair once
//       in the canonical rotation order), one thread per larger batch;
//       each member's key_{m+1} and its rank in its output digit;
//   (4) runs reserved in the step-(m+1) pass-1 buckets, staged through a u16
//       index, written coalesced (one vector store per record).
// Members of batches that straddle the bucket's ends are written unchanged to
// their sorted places in the own gapped range (the straddle kernel steps them).
// MODE_PAIR (p = 2), MODE_GROUP (lane groups of the runtime size P.group), or
// a compile-time lane-group size MODE in {4, 8, 32} (the fp32 group kernels:
// the partner loop unrolled, shuffle widths and lane arithmetic constant)
constexpr int MODE_PAIR = 0, MODE_GROUP = 1;
#ifndef RBM_BUCKET_BLOCK  // design-experiment builds override these (build.py -D...)
#define RBM_BUCKET_BLOCK 256
#define RBM_BUCKET_ITEMS 10
#endif
// 8 warps, capacity <= 2560 in registers; at <= 56 KB of shared memory four
// CTAs (buckets) share an SM (C5: 2352-record capacity, 57.3 KB)
constexpr int BUCKET_BLOCK = RBM_BUCKET_BLOCK, BUCKET_ITEMS = RBM_BUCKET_ITEMS;

// counter words: the packed u16 sub-digit counts (scanned in place), later the
// output digit counts; >= 512 for the oversized-bucket path's two 256 arrays
__host__ __device__ constexpr uint32_t bucket_ncw(uint32_t SB, uint32_t b1) {
  return ((1u << SB) / 2 > (1u << b1) ? (1u << SB) / 2 : (1u << b1)) > 512u
             ? ((1u << SB) / 2 > (1u << b1) ? (1u << SB) / 2 : (1u << b1))
             : 512u;
}
template <typename T, int D> __host__ __device__ constexpr size_t bucket_smem_bytes(uint32_t cap, uint32_t SB,
                                                                                   uint32_t b1) {
  return (size_t)(bucket_ncw(SB, b1) + (1u << b1) + 64) * 4 + 16  // counters, gbase, wsum, mbarrier
         + (size_t)(cap + 8) * RecL<T, D>::RS              // records (TMA window, updated in place)
         + (size_t)(cap + 8) * 4                           // side keys (TMA window) -> composites -> tb
         + (((size_t)cap * 2 + 15) & ~(size_t)15);         // ord (u16) -> staging index (u16)
}

// the bucket step of final bucket b (global start s0, n > 0 records at
// physical slots [b scap, b scap + n) of src), in the CTA's shared memory smem_raw
template <typename T, int D, int KK, int INTEG, int MODE>
__device__ __forceinline__ void bucket_body(const DevParams& P, State<T, D> src, uint32_t scap, uint32_t b,
                                            uint32_t s0, uint32_t n, const OutDst<T, D>& dst, uint32_t dcap,
                                            uint32_t* __restrict__ cur_next, unsigned char* smem_raw) {
  using L = RecL<T, D>;
  constexpr int BLOCK = BUCKET_BLOCK, ITEMS = BUCKET_ITEMS;
  RBM_PROF_BEGIN(P);
  const uint32_t sb = b * scap;
  const uint32_t nsb = 1u << P.SB;
  const uint32_t nout = 1u << P.b1;
  // sub-digit counts as packed u16 pairs (bucket sizes < 2^16), scanned in
  // place into offsets; the same words later hold the <= 1024 output digit
  // counts, again scanned in place
  const uint32_t ncw = bucket_ncw(P.SB, P.b1);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem_raw);
  uint32_t* off = cnt;
  uint32_t* gbase = cnt + ncw;
  uint32_t* wsum = gbase + nout;
  uint64_t* bar = reinterpret_cast<uint64_t*>(wsum + 64);
  const uint32_t cap = P.cap;
  const uint32_t m = (uint32_t)*P.step;
  for (uint32_t i = threadIdx.x; i < ncw / 4; i += BLOCK) reinterpret_cast<uint4*>(cnt)[i] = make_uint4(0, 0, 0, 0);
  if (n > cap || n > (uint32_t)(BLOCK * ITEMS)) {  // oversized bucket: global scratch
    __syncthreads();
    big_bucket<T, D, KK, INTEG, BLOCK>(P, src, dst, cur_next, s0, sb, n, m, dcap, cnt, cnt + 256, wsum);
    return;
  }
  unsigned char* rs = reinterpret_cast<unsigned char*>(bar + 2);
  uint32_t* key_l = reinterpret_cast<uint32_t*>(rs + (size_t)(cap + 8) * L::RS);
  uint32_t* ks = key_l;             // composites (sort), once the side keys are consumed
  uint32_t* tb = ks;                // then: output digit << 16 | rank in it, by element (~0: straddler)
  uint16_t* ord = reinterpret_cast<uint16_t*>(key_l + cap + 8);
  uint16_t* inv = ord;              // after the batch update: staged output slot -> element
  const bool side = !L::KEYED && P.side_key;
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // smem last touched by generic accesses
    const uint32_t bytes_r = (n * (uint32_t)L::RS + 15u) & ~15u;
    const uint32_t bytes_k = side ? ((n + 3u) & ~3u) * 4u : 0u;
    const uint64_t pol = l2_evict_first_policy();
    mbar_init(bar, 1);
    mbar_expect_tx(bar, bytes_r + bytes_k);
    bulk_g2s_stream(rs, src.rec + (size_t)sb * L::RS, bytes_r, bar, pol);
    if (side) bulk_g2s_stream(key_l, src.key + sb, bytes_k, bar, pol);
  }
  __syncthreads();
  mbar_wait(bar, 0);
  RBM_PROF(P, 0);
  if (!L::KEYED && !side) {  // one-pass layouts: key_m from the ids
    for (uint32_t e = threadIdx.x; e < n; e += BLOCK) key_l[e] = shuffle_key(P, ld_id<T, D>(rs, e), m);
    __syncthreads();
  }

  // 1-3. exact (key, id) sort: counting sort on SB sub-digit bits + rank in sub-bucket
  const uint32_t shsb = 32u - P.B - P.SB;
  const uint32_t lowmask = (P.lowbits >= 32u) ? 0xffffffffu : ((1u << P.lowbits) - 1u);
  uint32_t rc[ITEMS], rsd[ITEMS];
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const uint32_t e = k * BLOCK + threadIdx.x;
    if (e < n) {
      const unsigned char* re = rs + (size_t)e * L::RS;
      const uint32_t id = reinterpret_cast<const uint32_t*>(re)[0];
      const uint32_t key = L::KEYED ? reinterpret_cast<const uint32_t*>(re)[1] : key_l[e];
      const uint32_t sd = (key >> shsb) & (nsb - 1u);
      rc[k] = ((key & lowmask) << P.idbits) | id;
      const uint32_t sh16 = (sd & 1u) << 4;
      rsd[k] = (sd << 16) | ((atomicAdd(&cnt[sd >> 1], 1u << sh16) >> sh16) & 0xffffu);
    }
  }
  __syncthreads();
  RBM_PROF(P, 1);
  block_excl_scan_u16x2<BLOCK>(cnt, off, nsb / 2, wsum);  // in place
  RBM_PROF(P, 2);
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const uint32_t e = k * BLOCK + threadIdx.x;
    if (e < n) {
      const uint32_t sd = rsd[k] >> 16;
      // sub-bucket size = next offset - own offset (the last ends at n); for
      // an even sub-digit the next offset is the high half of the same word
      const uint32_t w0 = off[sd >> 1];
      const uint32_t a = (sd & 1u) ? (w0 >> 16) : (w0 & 0xffffu);
      uint32_t a1 = w0 >> 16;
      if (sd & 1u) a1 = (sd + 1u < nsb) ? (off[(sd + 1u) >> 1] & 0xffffu) : n;
      const uint32_t c = a1 - a;
      RBM_CHECK(P, a + (rsd[k] & 0xffffu) < n && a + c <= n);
      ks[a + (rsd[k] & 0xffffu)] = rc[k];
      rsd[k] = (a << 16) | c;  // sub-bucket start and size, for the rank below
    }
  }
  __syncthreads();
  RBM_PROF(P, 3);
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const uint32_t e = k * BLOCK + threadIdx.x;
    if (e < n) {
      const uint32_t a = rsd[k] >> 16, c = rsd[k] & 0xffffu;
      uint32_t r = a;
      if (c > 1) {  // sub-buckets hold ~1 element: a short predicated count
        // six independent loads (a + 5 < cap + 8: inside the array; entries
        // past the sub-bucket are masked by i < c)
        const uint32_t x = rc[k];
        uint32_t v[6];
#pragma unroll
        for (int i = 0; i < 6; ++i) v[i] = ks[a + i];
        uint32_t t = (uint32_t)(v[0] < x) + (uint32_t)(v[1] < x);
#pragma unroll
        for (uint32_t i = 2; i < 6; ++i) t += (uint32_t)(i < c && v[i] < x);
        r += t;
        // more than 6 (probability ~6e-4 per element): a plain loop, not
        // unrolled, so warps that never take it pay no loop prologue
#pragma unroll 1
        for (uint32_t i = 6; i < c; ++i) r += (ks[a + i] < rc[k]) ? 1u : 0u;
      }
      RBM_CHECK(P, r < n);
      ord[r] = (uint16_t)e;
    }
  }
  // the packed sub-digit counters are dead: they become the output digit counts
  for (uint32_t i = threadIdx.x; i < nout / 4; i += BLOCK) reinterpret_cast<uint4*>(cnt)[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  RBM_PROF(P, 4);
  if (P.dbg_order)
    for (uint32_t q = threadIdx.x; q < n; q += BLOCK) P.dbg_order[s0 + q] = ld_id<T, D>(rs, ord[q]);
  const uint32_t osh = 32u - P.b1;
  // interior sorted positions [head, tail); the rest belong to straddling batches
  uint32_t head, tail;
  if (MODE == MODE_PAIR) {
    // pairs start at even global positions; N odd: the last batch is a triple
    const uint32_t N = (uint32_t)P.n;
    const uint32_t pend = (N & 1u) ? N - 3u : N;
    head = s0 & 1u;
    const uint32_t lim = (min(s0 + n, pend) > s0) ? min(s0 + n, pend) - s0 : 0u;
    const uint32_t npairs = (lim > head) ? (lim - head) / 2 : 0u;
    tail = head + 2 * npairs;
    const bool triple = (N & 1u) && (pend >= s0) && (N <= s0 + n);
    // straddlers: unchanged, to their sorted places in the own gapped range
    const uint32_t tri0 = triple ? pend - s0 : n;
    for (uint32_t t = threadIdx.x; t < head + (tri0 - tail); t += BLOCK) {
      const uint32_t q = t < head ? t : tail + (t - head);
      const uint32_t e = ord[q];
      uint32_t wd[L::NW];
      ld_words<L::NW>(rs + (size_t)e * L::RS, wd);
      st_words<L::NW>(src.rec + ((size_t)sb + q) * L::RS, wd);
      tb[e] = 0xffffffffu;
    }
    RBM_PROF(P, 5);
    // one thread per pair: Eq. (2.2) + update in place; next keys and ranks
    constexpr int PITEMS = (ITEMS + 1) / 2;
#pragma unroll 1  // one copy of the pair update: the hot loop stays in the instruction cache
    for (int k = 0; k < PITEMS; ++k) {
      const uint32_t j = k * BLOCK + threadIdx.x;
      if (j < npairs) {
        const uint32_t q = head + 2 * j;
        RBM_CHECK(P, q + 1 < n);
        const uint32_t e0 = ord[q], e1 = ord[q + 1];
        RBM_CHECK(P, e0 < n && e1 < n);
        Rec<T, D> r0 = ld_rec<T, D>(rs, e0), r1 = ld_rec<T, D>(rs, e1);
        const uint32_t kn0 = shuffle_key(P, r0.id, m + 1), kn1 = shuffle_key(P, r1.id, m + 1);
        T y0[D], y1[D];
        pair_update<T, D, KK, INTEG>(P, m, r0.x, r1.x, r0.id, r1.id, y0, y1);
        check_finite<T, D>(y0, P, r0.id, m);
        check_finite<T, D>(y1, P, r1.id, m);
#pragma unroll
        for (int c = 0; c < D; ++c) { r0.x[c] = y0[c]; r1.x[c] = y1[c]; }
        r0.key = kn0;
        r1.key = kn1;
        st_rec<T, D>(rs, e0, r0);
        st_rec<T, D>(rs, e1, r1);
        tb[e0] = ((kn0 >> osh) << 16) | atomicAdd(&cnt[kn0 >> osh], 1u);
        tb[e1] = ((kn1 >> osh) << 16) | atomicAdd(&cnt[kn1 >> osh], 1u);
      }
    }
    // the size-3 remainder batch (N odd, EM): one thread, out of line
    if (triple && threadIdx.x == 0) serial_batch<T, D, KK, INTEG>(P, m, tri0, n, ord, rs, tb, cnt, osh);
    if (triple) tail = n;
  } else {
    // interior batches [kfirst, klast) of this bucket
    uint32_t kfirst = batch_index(s0, P);
    if (kfirst * P.p < s0) ++kfirst;
    uint32_t klast;
    {
      const uint32_t kl = batch_index(s0 + n - 1, P);
      klast = (batch_end(kl, P) <= s0 + n) ? kl + 1 : kl;
    }
    head = (kfirst < klast) ? kfirst * P.p - s0 : n;
    tail = (kfirst < klast) ? batch_end(klast - 1, P) - s0 : n;
    for (uint32_t t = threadIdx.x; t < head + (n - tail); t += BLOCK) {
      const uint32_t q = t < head ? t : tail + (t - head);
      const uint32_t e = ord[q];
      uint32_t wd[L::NW];
      ld_words<L::NW>(rs + (size_t)e * L::RS, wd);
      st_words<L::NW>(src.rec + ((size_t)sb + q) * L::RS, wd);
      tb[e] = 0xffffffffu;
    }
    RBM_PROF(P, 5);
    const uint32_t G = (MODE > MODE_GROUP) ? (uint32_t)MODE : P.group;
    if (G != 0) {
      // lane groups: batches with sz <= G; each pair evaluated once in the
      // canonical rotation order (batch_force), the partner's term by shuffle
      const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      const uint32_t gpw = 32u / G, gi = lane / G, li = lane & (G - 1);
      const uint32_t stride = (BLOCK / 32) * gpw;
      for (uint32_t kb = kfirst + warp * gpw; kb < klast; kb += stride) {  // warp-uniform
        const uint32_t k = kb + gi;
        const bool valid = k < klast;
        const uint32_t l0 = valid ? k * P.p - s0 : 0;
        const uint32_t sz = valid ? batch_end(k, P) - s0 - l0 : 0;
        const bool act = valid && sz <= G && li < sz;
        const uint32_t e = act ? ord[l0 + li] : 0u;
        Rec<T, D> ri;
        if (act) ri = ld_rec<T, D>(rs, e);
        T xi[D];
#pragma unroll
        for (int c = 0; c < D; ++c) xi[c] = act ? ri.x[c] : T(0);
        const uint32_t id = act ? ri.id : 0u;
        T xn[D];
        if (INTEG != 1) {
          T f[D];
#pragma unroll
          for (int c = 0; c < D; ++c) f[c] = T(0);
#pragma unroll
          for (uint32_t o = 1; o <= G / 2; ++o) {
            const uint32_t jp = (li + o) & (G - 1), jm = (li - o) & (G - 1);
            T xj[D], t[D];
#pragma unroll
            for (int c = 0; c < D; ++c) xj[c] = __shfl_sync(0xffffffffu, xi[c], (int)jp, (int)G);
            if (act && jp < sz) {
              pair_term<T, D, KK, INTEG>(xi, xj, t, P);
#pragma unroll
              for (int c = 0; c < D; ++c) f[c] = add_rn(f[c], t[c]);
            } else {
#pragma unroll
              for (int c = 0; c < D; ++c) t[c] = T(0);
            }
            if (o < G / 2) {  // warp-uniform
#pragma unroll
              for (int c = 0; c < (INTEG == 2 ? 1 : D); ++c) {
                const T r = __shfl_sync(0xffffffffu, t[c], (int)jm, (int)G);
                if (act && jm < sz) f[c] = sub_rn(f[c], r);
              }
            }
          }
          if (act) {
            T z[D];
#pragma unroll
            for (int c = 0; c < D; ++c) z[c] = T(0);
            if (P.has_noise) Normals<T, D>::get(P, id, m, TAG_NOISE, z);
            const T inv_b = batch_inv<T>(P, sz);
#pragma unroll
            for (int c = 0; c < D; ++c) f[c] *= inv_b;
            member_update<T, D, INTEG>(xi, f, z, xn, P, P.verlet_start != 0);
          }
        } else {  // split exact pair flow, p = 2 = G
          T xo[D];
#pragma unroll
          for (int c = 0; c < D; ++c) xo[c] = __shfl_xor_sync(0xffffffffu, xi[c], 1, 2);
          if (act) {
            T xa[D], xb[D], y[D], z[D];
#pragma unroll
            for (int c = 0; c < D; ++c) {
              xa[c] = li == 0 ? xi[c] : xo[c];
              xb[c] = li == 0 ? xo[c] : xi[c];
              z[c] = T(0);
            }
            if (P.has_noise) Normals<T, D>::get(P, id, m, TAG_NOISE, z);
            pair_flow<T, D, KK>(xa, xb, li == 0, y, P);
            split_finish<T, D>(y, z, xn, P, true);
          }
        }
        if (act) {
          check_finite<T, D>(xn, P, id, m);
          const uint32_t kn = shuffle_key(P, id, m + 1);
#pragma unroll
          for (int c = 0; c < D; ++c) ri.x[c] = xn[c];
          ri.key = kn;
          st_rec<T, D>(rs, e, ri);
          tb[e] = ((kn >> osh) << 16) | atomicAdd(&cnt[kn >> osh], 1u);
        }
      }
    }
    // batches too large for a lane group (the remainder batch, or p > 32): one thread each
    const uint32_t first_big =
        (G == 0) ? kfirst
                 : ((klast > kfirst && batch_end(klast - 1, P) - (klast - 1) * P.p > G) ? klast - 1 : klast);
    for (uint32_t k = first_big + threadIdx.x; k < klast; k += BLOCK)
      serial_batch<T, D, KK, INTEG>(P, m, k * P.p - s0, batch_end(k, P) - s0, ord, rs, tb, cnt, osh);
  }
  __syncthreads();
  RBM_PROF(P, 6);
  // run reservations of digits threadIdx.x + r BLOCK, consumed after the staging index
  constexpr int NRES = (1024 + BLOCK - 1) / BLOCK;
  uint32_t gres[NRES];
#pragma unroll
  for (int r = 0; r < NRES; ++r) {
    const uint32_t i = threadIdx.x + r * BLOCK;
    const uint32_t h = i < nout ? cnt[i] : 0u;
    gres[r] = h ? atomicAdd(&cur_next[(size_t)out_seg(P, i, blockIdx.x) * CUR1_STRIDE], h) : 0u;
  }
  const uint32_t total = block_excl_scan4<BLOCK>(cnt, off, nout, wsum);  // in place
  for (uint32_t e = threadIdx.x; e < n; e += BLOCK) {  // staging index (tb read in element order)
    const uint32_t t = tb[e];
    RBM_CHECK(P, t == 0xffffffffu || (t >> 16) < nout);
    if (t != 0xffffffffu) {
      RBM_CHECK(P, off[t >> 16] + (t & 0xffffu) < total);
      inv[off[t >> 16] + (t & 0xffffu)] = (uint16_t)e;
    }
  }
#pragma unroll
  for (int r = 0; r < NRES; ++r)  // gbase[d] - off[d]: output position j goes to slot gbase[dg] + j
    if (threadIdx.x + r * BLOCK < nout) gbase[threadIdx.x + r * BLOCK] = gres[r] - off[threadIdx.x + r * BLOCK];
  __syncthreads();
  RBM_PROF(P, 7);
  // staged slots -> coalesced runs of the step-(m+1) pass-1 buckets
  for (uint32_t j = threadIdx.x; j < total; j += BLOCK) {
    const uint32_t e = inv[j];
    RBM_CHECK(P, e < n);
    const uint32_t dg = tb[e] >> 16;
    RBM_CHECK(P, dg < nout);
    const uint32_t slot = gbase[dg] + j;
    if (slot >= dcap) { atomicExch(P.capacity_err, 1u); continue; }
    out_copy<T, D>(dst, out_seg(P, dg, blockIdx.x), dcap, slot, rs + (size_t)e * L::RS);
  }
  RBM_PROF(P, 8);
  if (P.prof && threadIdx.x == 0) atomicAdd(&P.prof[63], 1ull);
}

// one CTA per final bucket b of step m (S: exact global starts)
template <typename T, int D, int KK, int INTEG, int MODE, int MINB>
static __global__ void __launch_bounds__(BUCKET_BLOCK, MINB) bucket_kernel(const __grid_constant__ DevParams P, State<T, D> src,
                                                                           uint32_t scap,
                                                                           const uint32_t* __restrict__ S,
                                                                           const __grid_constant__ OutDst<T, D> dst, uint32_t dcap,
                                                                           uint32_t* __restrict__ cur_next) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const uint32_t b = blockIdx.x;
  const uint32_t s0 = S[b], n = S[b + 1] - s0;
  if (n == 0) return;
  bucket_body<T, D, KK, INTEG, MODE>(P, src, scap, b, s0, n, dst, dcap, cur_next, smem_raw);
}

// ------------------------------------------ resident multi-step (N <= 2048)
// One CTA keeps the whole system in shared memory for `nsteps` steps (the
// B = 0 layout, e.g. BASELINE C1): per step, keys (Philox) -> exact sort by
// (key_m, id) -> Eq. (2.2) + update of every batch into the other smem
// buffer in sorted order; one launch replaces 2 launches per step.
template <typename T, int D> struct SX {  // D coordinate arrays base + c*stride (shared memory)
  T* base;
  uint32_t stride;
  __device__ __forceinline__ void get(uint32_t e, T (&x)[D]) const {
#pragma unroll
    for (int c = 0; c < D; ++c) x[c] = base[(uint32_t)c * stride + e];
  }
};

template <typename T, int D> __host__ __device__ constexpr size_t resident_smem_bytes(uint32_t cap) {
  return 2304                                             // cnt, off, wsum
         + 2 * (size_t)cap * 4                            // ids, two buffers
         + 2 * (size_t)D * cap * sizeof(T)                // x, two buffers
         + (size_t)cap * 8 + (size_t)cap * 4              // composites, keys
         + (((size_t)cap * 2 + 15) & ~(size_t)15);        // ord
}

template <typename T, int D, int KK, int INTEG, int BLOCK>
static __global__ void __launch_bounds__(BLOCK) resident_kernel(const __grid_constant__ DevParams P, State<T, D> src,
                                                                State<T, D> dst, uint32_t nsteps,
                                                                uint64_t* stepp) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem_raw);
  uint32_t* off = cnt + 256;
  uint32_t* wsum = off + 256;
  const uint32_t cap = P.cap, n = (uint32_t)P.n;
  unsigned char* p = smem_raw + 2304;
  T* xb = reinterpret_cast<T*>(p);                      // [2][D][cap]
  p += 2 * (size_t)D * cap * sizeof(T);
  unsigned long long* ks = reinterpret_cast<unsigned long long*>(p);
  p += (size_t)cap * 8;
  uint32_t* idb = reinterpret_cast<uint32_t*>(p);       // [2][cap]
  p += 2 * (size_t)cap * 4;
  uint32_t* key_l = reinterpret_cast<uint32_t*>(p);
  p += (size_t)cap * 4;
  uint16_t* ord = reinterpret_cast<uint16_t*>(p);
  for (uint32_t e = threadIdx.x; e < n; e += BLOCK) {
    const Rec<T, D> r = ld_rec<T, D>(src.rec, e);
    idb[e] = r.id;
#pragma unroll
    for (int c = 0; c < D; ++c) xb[(size_t)c * cap + e] = r.x[c];
  }
  const uint32_t m0 = (uint32_t)*stepp;
  for (uint32_t it = 0; it < nsteps; ++it) {
    const uint32_t m = m0 + it, cur = it & 1u;
    const uint32_t* id_l = idb + cur * cap;
    const SX<T, D> xs{xb + (size_t)cur * D * cap, cap};
    uint32_t* id_o = idb + (cur ^ 1u) * cap;
    T* x_o = xb + (size_t)(cur ^ 1u) * D * cap;
    for (uint32_t i = threadIdx.x; i < 256; i += BLOCK) cnt[i] = 0;
    __syncthreads();
    // exact sort by (key_m, id): counting sort on the top 8 key bits + rank
    for (uint32_t e = threadIdx.x; e < n; e += BLOCK) {
      const uint32_t key = shuffle_key(P, id_l[e], m);
      key_l[e] = key;
      ord[e] = (uint16_t)atomicAdd(&cnt[key >> 24], 1u);
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < 256; i += BLOCK) off[i] = cnt[i];
    __syncthreads();
    block_excl_scan<BLOCK>(off, 256, wsum);
    for (uint32_t e = threadIdx.x; e < n; e += BLOCK) {
      const uint32_t key = key_l[e];
      ks[off[key >> 24] + ord[e]] = ((unsigned long long)key << 32) | id_l[e];
    }
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < n; e += BLOCK) {
      const uint32_t key = key_l[e];
      const unsigned long long mine = ((unsigned long long)key << 32) | id_l[e];
      const uint32_t a = off[key >> 24], c = cnt[key >> 24];
      uint32_t r = a;
      for (uint32_t j = a; j < a + c; ++j) r += (ks[j] < mine) ? 1u : 0u;
      ord[r] = (uint16_t)e;
    }
    __syncthreads();
    if (P.dbg_order)
      for (uint32_t q = threadIdx.x; q < n; q += BLOCK) P.dbg_order[q] = id_l[ord[q]];
    // every batch: Eq. (2.2) + update from the old positions, sorted output
    for (uint32_t q = threadIdx.x; q < n; q += BLOCK) {
      uint32_t b0, b1;
      batch_range(q, P, b0, b1);
      const uint32_t id = id_l[ord[q]];
      T xn[D];
      interior_update<T, D, KK, INTEG>(P, m, q, b0, b1, ord, xs, id, xn,
                                       (P.verlet_start && it == 0) ? 1 : 0);
      check_finite<T, D>(xn, P, id, m);
      id_o[q] = id;
#pragma unroll
      for (int c = 0; c < D; ++c) x_o[(size_t)c * cap + q] = xn[c];
    }
    __syncthreads();
  }
  const uint32_t fin = nsteps & 1u;
  for (uint32_t e = threadIdx.x; e < n; e += BLOCK) {
    Rec<T, D> r;
    r.id = idb[fin * cap + e];
    r.key = 0u;
#pragma unroll
    for (int c = 0; c < D; ++c) r.x[c] = xb[((size_t)fin * D + c) * cap + e];
    st_rec<T, D>(dst.rec, e, r);
  }
  if (threadIdx.x == 0) *stepp = m0 + nsteps;
}

// batches that straddle final buckets: one warp per owning boundary.  Their
// members were written (unchanged) by the bucket kernels to their sorted
// places in their own gapped ranges of `strad`: position P of bucket b sits at
// physical slot b*cap + (P - S[b]).  Results are appended to the step-(m+1)
// buckets of `dst` (capacity ocap, cursors cur_next).
template <typename T, int D, int KK, int INTEG>
static __global__ void __launch_bounds__(256) straddle_kernel(const __grid_constant__ DevParams P, State<T, D> strad,
                                                              uint32_t cap,
                                                              const uint32_t* __restrict__ S,
                                                              const __grid_constant__ OutDst<T, D> dst, uint32_t ocap,
                                                              uint32_t* cur_next) {
  __shared__ long long strad_phys[(256 / 32) * 96];  // member slots per warp (sz <= 96)
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  // boundaries 1 .. nbuckets-1; on a partitioned system with a halo also
  // boundary 0 (the rank's first position), whose batch starts in the halo
  // records of rank-1 placed at bucket -1 (physical slots [-cap, -cap + t),
  // S[-1] = S[0] - t)
  const int bnd = (int)warp + (P.halo ? 0 : 1);
  if (bnd >= (int)P.nbuckets) return;
  const uint32_t Pb = S[bnd];
  if (Pb == 0 || Pb >= P.n) return;
  uint32_t b0, b1;
  batch_range(Pb, P, b0, b1);
  if (b0 == Pb) return;             // boundary at a batch start: no straddle
  if (S[bnd - 1] > b0) return;      // an earlier boundary inside the batch owns it
  if (b1 > S[P.nbuckets]) return;   // ends on the next rank: that rank owns it
  const uint32_t m = (uint32_t)*P.step;
  const uint32_t sz = b1 - b0;
  // physical slot of every member (buckets walked forward from bnd-1)
  long long phys[3];
  {
    int bb = bnd - 1;
    int k = 0;
    for (uint32_t q = 0; q < sz; ++q) {
      const uint32_t Pq = b0 + q;
      while (Pq >= S[bb + 1]) ++bb;
      RBM_CHECK(P, Pq - S[bb] < cap && sz <= 96);
      if ((q & 31u) == (uint32_t)lane) phys[k++] = (long long)bb * cap + (Pq - S[bb]);
    }
  }
  auto getx = [&](long long g, T (&x)[D]) {
    const Rec<T, D> r = ld_rec<T, D>(strad.rec, g);
#pragma unroll
    for (int c = 0; c < D; ++c) x[c] = r.x[c];
  };
  T xnew[3][D];
  uint32_t idv[3];
  const uint32_t rounds = (sz + 31) / 32;
  for (uint32_t r = 0; r < rounds; ++r) {  // warp-uniform: every lane reaches the shuffles
    const uint32_t q = r * 32 + lane;
    const bool act = q < sz;
    const long long g = act ? (r == 0 ? phys[0] : (r == 1 ? phys[1] : phys[2])) : 0ll;
    Rec<T, D> rec;
    if (act) rec = ld_rec<T, D>(strad.rec, g);
    const uint32_t id = act ? rec.id : 0u;
    T xi[D], z[D], xn[D];
#pragma unroll
    for (int c = 0; c < D; ++c) { xi[c] = act ? rec.x[c] : T(0); z[c] = T(0); }
    if (act && P.has_noise) Normals<T, D>::get(P, id, m, TAG_NOISE, z);
    if (INTEG != 1) {
      T f[D];
#pragma unroll
      for (int c = 0; c < D; ++c) f[c] = T(0);
      // the physical slot of every member, staged per warp (lane l holds
      // members l, l+32, l+64): shuffled out once, then read in the
      // canonical partner order
      long long* ph_w = strad_phys + (threadIdx.x >> 5) * 96;
      for (uint32_t h = 0; h < sz; ++h) {
        const uint32_t hr = h >> 5;
        const long long src_ph = hr == 0 ? phys[0] : (hr == 1 ? phys[1] : phys[2]);
        const long long gh = __shfl_sync(0xffffffffu, src_ph, (int)(h & 31u));
        if (lane == 0) ph_w[h] = gh;
      }
      __syncwarp();
      if (act)
        batch_force<T, D, KK, INTEG>(P, q, sz, xi, [&](uint32_t j, T (&xj)[D]) { getx(ph_w[j], xj); }, f);
      __syncwarp();
      if (act) {
        const T inv = batch_inv<T>(P, sz);
#pragma unroll
        for (int c = 0; c < D; ++c) f[c] *= inv;
        member_update<T, D, INTEG>(xi, f, z, xn, P, P.verlet_start != 0);
      }
    } else {
      const long long ga = __shfl_sync(0xffffffffu, phys[0], 0), gb = __shfl_sync(0xffffffffu, phys[0], 1);
      if (act) {
        T xa[D], xb[D], y[D];
        getx(ga, xa);
        getx(gb, xb);
        pair_flow<T, D, KK>(xa, xb, q == 0, y, P);
        split_finish<T, D>(y, z, xn, P, true);
      }
    }
    if (act) {
      check_finite<T, D>(xn, P, id, m);
      idv[r] = id;
#pragma unroll
      for (int c = 0; c < D; ++c) xnew[r][c] = xn[c];
    }
  }
  __syncwarp();
  int k = 0;
  const uint32_t osh = 32u - P.b1;
  for (uint32_t q = lane; q < sz; q += 32, ++k) {
    Rec<T, D> o;
    o.id = idv[k];
    o.key = shuffle_key(P, o.id, m + 1);
#pragma unroll
    for (int c = 0; c < D; ++c) o.x[c] = xnew[k][c];
    const uint32_t v = out_seg(P, o.key >> osh, warp);
    const uint32_t slot = atomicAdd(&cur_next[(size_t)v * CUR1_STRIDE], 1u);
    if (slot >= ocap) { atomicExch(P.capacity_err, 1u); continue; }
    out_put<T, D>(dst, v, ocap, slot, o);
  }
}

// ------------------------------------------ partitioned single system (a7)
// G ranks, rank r owns keys whose top log2 G bits are r.  After the exchange a
// rank holds 2^b1 received pass-1 segments v = s*nl + u (source rank s, local
// pass-1 bucket u < nl = 2^b1/G) of capacity cap1 each; M[s*2^b1 + j] is the
// all-gathered count of source s's pass-1 bucket j (global j).
constexpr uint32_t HALO_MAX = 64;  // >= p - 1 records of the batch crossing a rank boundary
template <typename T, int D> __host__ __device__ constexpr size_t halo_bytes() {
  return 16 + (size_t)HALO_MAX * RecL<T, D>::RS;
}

// One block: segment counts (strided, for the pass-2 tile table), the exact
// global start O_r of this rank (exclusive scan of the rank totals), the
// global start of each local pass-1 bucket (prefix1[u], prefix1[nl] = O_r +
// n_r) and the tile table.  Flags capacity_err = 2 if the rank holds fewer
// than p particles (the halo exchange assumes a crossing batch touches only
// two ranks).
static __global__ void __launch_bounds__(1024) part_scan_kernel(const __grid_constant__ DevParams P, const uint32_t* __restrict__ M,
                                                                uint32_t G, uint32_t rank, uint32_t* cnt1,
                                                                uint32_t* prefix1, uint32_t* tile_off,
                                                                uint32_t tile) {
  __shared__ uint32_t a[1025];
  __shared__ uint32_t ws[33];
  __shared__ uint32_t o_r;
  // nseg = 2^b1 << segk segments per rank row of M; this rank's slice of a
  // row is nls = nseg/G segments = nlb = 2^b1/G local pass-1 buckets x K
  const uint32_t nseg = (1u << P.b1) << P.segk, nls = nseg / G, nlb = nls >> P.segk;
  const uint32_t K = 1u << P.segk;
  if (threadIdx.x == 0) o_r = 0;
  __syncthreads();
  for (uint32_t v = threadIdx.x; v < nseg; v += blockDim.x) {  // received segment v = s*nls + j
    const uint32_t s = v / nls, j = v - s * nls;
    cnt1[(size_t)v * CUR1_STRIDE] = M[(size_t)s * nseg + rank * nls + j];
  }
  for (uint32_t u = threadIdx.x; u < nlb; u += blockDim.x) {
    uint32_t c = 0;
    for (uint32_t s = 0; s < G; ++s)
      for (uint32_t k = 0; k < K; ++k) c += M[(size_t)s * nseg + rank * nls + (u << P.segk) + k];
    a[u] = c;
  }
  {  // O_r = all records of the ranks below (their segments, every source)
    uint32_t part = 0;
    const uint32_t below = rank * nls;
    for (uint32_t q = threadIdx.x; q < G * below; q += blockDim.x) {
      const uint32_t s = q / below, j = q - s * below;
      part += M[(size_t)s * nseg + j];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if ((threadIdx.x & 31) == 0 && part) atomicAdd(&o_r, part);
  }
  __syncthreads();
  const uint32_t nloc = block_excl_scan<1024>(a, nlb, ws);
  const uint32_t O = o_r;
  for (uint32_t u = threadIdx.x; u < nlb; u += blockDim.x) prefix1[u] = O + a[u];
  if (threadIdx.x == 0) {
    prefix1[nlb] = O + nloc;
    if (nloc < P.p) atomicExch(P.capacity_err, 2u);
  }
  __syncthreads();
  seg_tile_table(cnt1, nseg, tile, tile_off, ws);
}

// The batch crossing this rank's end E = S[nbuckets] (global positions
// [b0, E), t = E - b0 <= p - 1 records, left unchanged in sorted order by the
// bucket kernels) is owned by rank+1: copy it to the halo buffer
// {u32 t; pad; records[HALO_MAX]}.
template <typename T, int D>
static __global__ void halo_extract_kernel(const __grid_constant__ DevParams P, State<T, D> strad, uint32_t cap,
                                           const uint32_t* __restrict__ S, unsigned char* halo) {
  const uint32_t E = S[P.nbuckets];
  uint32_t t = 0, b0 = E, b1 = E;
  if (E < P.n) {
    batch_range(E, P, b0, b1);
    if (b0 < E) t = E - b0;
  }
  if (threadIdx.x == 0) *reinterpret_cast<uint32_t*>(halo) = t;
  for (uint32_t q = threadIdx.x; q < t; q += blockDim.x) {
    const uint32_t Pq = b0 + q;
    int bb = (int)P.nbuckets - 1;
    while (bb > 0 && S[bb] > Pq) --bb;
    const long long g = (long long)bb * cap + (Pq - S[bb]);
    st_rec<T, D>(halo + 16, q, ld_rec<T, D>(strad.rec, g));
  }
}

// Received halo (rank-1's trailing records of the crossing batch) -> bucket -1
// of the local final layout, S[-1] = S[0] - t.
template <typename T, int D>
static __global__ void halo_place_kernel(const __grid_constant__ DevParams P, State<T, D> strad, uint32_t cap, uint32_t* S,
                                         const unsigned char* __restrict__ halo) {
  const uint32_t t = *reinterpret_cast<const uint32_t*>(halo);
  for (uint32_t q = threadIdx.x; q < t; q += blockDim.x)
    st_rec<T, D>(strad.rec, -(long long)cap + q, ld_rec<T, D>(halo + 16, q));
  if (threadIdx.x == 0) S[-1] = S[0] - t;
}

// cursor counts (stride CUR1_STRIDE) -> contiguous u32 (the all-gathered row)
static __global__ void pack_counts_kernel(const uint32_t* __restrict__ cur, uint32_t nb, uint32_t* out) {
  for (uint32_t v = threadIdx.x; v < nb; v += blockDim.x) out[v] = cur[(size_t)v * CUR1_STRIDE];
}

// gather from the received segments of a partitioned rank (holes skipped)
template <typename T, int D>
static __global__ void gather_part_kernel(const __grid_constant__ DevParams P, State<T, D> st, uint32_t cap1,
                                          const uint32_t* __restrict__ M, uint32_t G, uint32_t rank,
                                          uint64_t i0, uint64_t i1, T* __restrict__ out) {
  const uint32_t nseg = (1u << P.b1) << P.segk, nls = nseg / G;
  const uint64_t total = (uint64_t)nseg * cap1;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < total;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t v = (uint32_t)(q / cap1), e = (uint32_t)(q - (uint64_t)v * cap1);
    const uint32_t s = v / nls, j = v - s * nls;
    if (e >= M[(size_t)s * nseg + rank * nls + j]) continue;
    const Rec<T, D> r = ld_rec<T, D>(st.rec, (long long)q);
    const uint64_t id = r.id;
    if (id >= i0 && id < i1) {
#pragma unroll
      for (int c = 0; c < D; ++c) out[(id - i0) * D + c] = r.x[c];
    }
  }
}

// this rank's records as (ids, rows) in storage order (rbm_gather_local):
// records in id order (before the first step) ...
template <typename T, int D>
static __global__ void gather_local_kernel(uint64_t n, State<T, D> st, uint32_t* __restrict__ ids,
                                           T* __restrict__ out) {
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const Rec<T, D> r = ld_rec<T, D>(st.rec, (long long)q);
    ids[q] = r.id;
#pragma unroll
    for (int c = 0; c < D; ++c) out[q * D + c] = r.x[c];
  }
}

// ... or in the received segments of a partitioned rank: off[v] = exclusive
// prefix of the segment counts (off[nseg] = total), one block
static __global__ void __launch_bounds__(1024) seg_offsets_kernel(const __grid_constant__ DevParams P,
                                                                  const uint32_t* __restrict__ M, uint32_t G,
                                                                  uint32_t rank, uint32_t* off) {
  __shared__ uint32_t a[MAX_SEG_SPLIT + 1];
  __shared__ uint32_t ws[33];
  const uint32_t nseg = (1u << P.b1) << P.segk, nls = nseg / G;
  for (uint32_t v = threadIdx.x; v < nseg; v += blockDim.x) {
    const uint32_t s = v / nls, j = v - s * nls;
    a[v] = M[(size_t)s * nseg + rank * nls + j];
  }
  __syncthreads();
  const uint32_t total = block_excl_scan<1024>(a, nseg, ws);
  for (uint32_t v = threadIdx.x; v < nseg; v += blockDim.x) off[v] = a[v];
  if (threadIdx.x == 0) off[nseg] = total;
}

template <typename T, int D>
static __global__ void gather_local_part_kernel(const __grid_constant__ DevParams P, State<T, D> st, uint32_t cap1,
                                                const uint32_t* __restrict__ M, uint32_t G, uint32_t rank,
                                                const uint32_t* __restrict__ off, uint32_t* __restrict__ ids,
                                                T* __restrict__ out) {
  const uint32_t nseg = (1u << P.b1) << P.segk, nls = nseg / G;
  const uint64_t total = (uint64_t)nseg * cap1;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < total;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t v = (uint32_t)(q / cap1), e = (uint32_t)(q - (uint64_t)v * cap1);
    const uint32_t s = v / nls, j = v - s * nls;
    if (e >= M[(size_t)s * nseg + rank * nls + j]) continue;
    const Rec<T, D> r = ld_rec<T, D>(st.rec, (long long)q);
    const uint64_t o = (uint64_t)off[v] + e;
    ids[o] = r.id;
#pragma unroll
    for (int c = 0; c < D; ++c) out[o * D + c] = r.x[c];
  }
}

// -------------------------------------- direct O(N^2) step (next row f1)
// The fully coupled Euler-Maruyama step of Eq. (1.2): the reference solution
// the paper measures RBM against (Sec. 4.1, "solving the
// fully coupled system using the forward Euler scheme").  One thread per
// particle i (id order), j tiles staged in shared memory, forces summed in
// ascending j, prefactor 1/(N-1); the Brownian increment of particle i at
// step m is the one RBM step m uses (counter (i, blk, m, TAG_NOISE)), so RBM
// and direct runs from one X_0 are synchronously coupled.
template <typename T, int D, int KK, int INTEG, int TB>
static __global__ void __launch_bounds__(TB) direct_kernel(const __grid_constant__ DevParams P,
                                                           const T* __restrict__ xin,
                                                           T* __restrict__ xout, uint32_t n,
                                                           uint32_t m) {
  __shared__ T tile[D][TB];
  const uint32_t i = blockIdx.x * TB + threadIdx.x;
  T xi[D], f[D];
#pragma unroll
  for (int c = 0; c < D; ++c) {
    xi[c] = (i < n) ? xin[(size_t)i * D + c] : T(0);
    f[c] = T(0);
  }
  for (uint32_t j0 = 0; j0 < n; j0 += TB) {
    const uint32_t jj = j0 + threadIdx.x;
#pragma unroll
    for (int c = 0; c < D; ++c) tile[c][threadIdx.x] = (jj < n) ? xin[(size_t)jj * D + c] : T(0);
    __syncthreads();
    const uint32_t lim = min((uint32_t)TB, n - j0);
#pragma unroll 4
    for (uint32_t t = 0; t < lim; ++t) {
      if (j0 + t == i) continue;
      T xj[D];
#pragma unroll
      for (int c = 0; c < D; ++c) xj[c] = tile[c][t];
      member_force<T, D, KK, INTEG>(xi, xj, f, P);
    }
    __syncthreads();
  }
  if (i >= n) return;
  const T nm1 = T(n - 1);
#pragma unroll
  for (int c = 0; c < D; ++c) f[c] /= nm1;
  T z[D], xn[D];
#pragma unroll
  for (int c = 0; c < D; ++c) z[c] = T(0);
  if (P.has_noise) Normals<T, D>::get(P, i, m, TAG_NOISE, z);
  member_update<T, D, INTEG>(xi, f, z, xn, P, P.verlet_start != 0);
  check_finite<T, D>(xn, P, i, m);
#pragma unroll
  for (int c = 0; c < D; ++c) xout[(size_t)i * D + c] = xn[c];
}

// ------------------------------------------------------------------ RBM-r
// One sweep of ceil(N/p) with-replacement batches (Alg. 2/3),
// Jacobi-additive reading D:8: every batch evaluated from X_m, then
// x_j <- x_j + sum over the slots s with j_s = j of Delta_s, summed
// order-independently in fixed point (Fx).
// State in id order as AoS (4 scalars per particle, one sector per gather).
// One GPU: the increments go through a partition by particle index (the
// rbmr_emit / split / rbmr_bucket_apply kernels below); the sequential RBM-r'
// finds each slot's predecessor through the same partition (link records).
// The partitioned system registers slots in per-particle mailboxes (MBOX
// entries, overflow list for the ~1e-6 of particles drawn more often), sorted
// by s when applied.
constexpr uint32_t MBOX = 8;
constexpr uint32_t OVF_CAP = 1u << 20;

template <typename T, int D>
static __global__ void rbmr_pack_kernel(uint64_t n, State<T, D> st, T* __restrict__ xa) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const Rec<T, D> r = ld_rec<T, D>(st.rec, (long long)i);  // id order: record i is id i
#pragma unroll
    for (int c = 0; c < 4; ++c) xa[i * 4 + c] = (c < D) ? r.x[c < D ? c : 0] : T(0);
  }
}

template <typename T, int D>
__device__ __forceinline__ void load4(const T* __restrict__ xa, uint32_t j, T (&x)[D]) {
  if constexpr (sizeof(T) == 4) {  // one 16-byte access
    const float4 v = reinterpret_cast<const float4*>(xa)[j];
    const float w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int c = 0; c < D; ++c) x[c] = (T)w[c];
  } else {
    const double2 v0 = reinterpret_cast<const double2*>(xa)[2 * (size_t)j];
    const double2 v1 = reinterpret_cast<const double2*>(xa)[2 * (size_t)j + 1];
    const double w[4] = {v0.x, v0.y, v1.x, v1.y};
#pragma unroll
    for (int c = 0; c < D; ++c) x[c] = (T)w[c];
  }
}

// the D coordinates of particle j into its 4-wide AoS slot, padding zero (as
// rbmr_pack_kernel writes it; only the Jacobi RBM-r state is stored this way):
// one 16-byte store for fp32, two for fp64, no read
template <typename T, int D>
__device__ __forceinline__ void store4(T* __restrict__ xa, uint32_t j, const T (&x)[D]) {
  T w[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) w[c] = (c < D) ? x[c < D ? c : 0] : T(0);
  if constexpr (sizeof(T) == 4) {
    reinterpret_cast<float4*>(xa)[j] = make_float4((float)w[0], (float)w[1], (float)w[2], (float)w[3]);
  } else {
    reinterpret_cast<double2*>(xa)[2 * (size_t)j] = make_double2((double)w[0], (double)w[1]);
    reinterpret_cast<double2*>(xa)[2 * (size_t)j + 1] = make_double2((double)w[2], (double)w[3]);
  }
}

// ----------------------- exact sequential RBM-r' (Alg. 2, row f2)
// Batches of one sweep are applied in draw order from the current positions.
// Batch b depends only on the earlier batches that touched its members.  Each
// particle's AoS record carries, in its padding word, a write counter (tag).
// The link pass routes records {j_s, s} through the partition by particle
// index (rbmr_emit_kernel<LINK> -> split -> rbmr_bucket_apply_kernel<LINK>):
// per particle j with slots s_0 < s_1 < ... in this sweep, expect[s_a] =
// tag_j + a (a > 0; the first slot waits for nobody).  The dependency-driven
// kernel then applies the batches: warps take consecutive groups of 32
// batches in ticket order; a batch waits until the tag of each member reaches
// its expect value (all earlier writers of that particle are done), reads the
// positions, writes the new ones and bumps the tags: fp32 records are 16
// bytes, read and written as single 128-bit accesses carrying position and
// tag together; wider records store the tag after a release fence.  Every batch waits only on lower-numbered batches,
// which were taken earlier by running warps, so the sweep always drains; each
// batch sees exactly the positions the sequential loop would give it.


// one batch of the sequential sweep from the current positions (members
// distinct): Eq. (2.2) + EM, or the exact pair flow; positions read through L2
// (other SMs wrote them) and written in place
template <typename T, int D, int KK, int INTEG>
__device__ __forceinline__ void seq_batch(const DevParams& P, uint32_t m, uint64_t b, const uint32_t* __restrict__ js,
                                          T* xa) {
  const uint32_t p = P.p;
  const uint64_t s0 = b * p;
  auto ld = [&](uint32_t j, T (&x)[D]) {
#pragma unroll
    for (int c = 0; c < D; ++c) x[c] = __ldcg(xa + (size_t)j * 4 + c);
  };
  if (INTEG == 0) {
    T xn[64][D];  // p <= 64; new positions of all members before any is written
    for (uint32_t l = 0; l < p; ++l) {
      T xi[D], f[D], z[D];
      ld(js[s0 + l], xi);
#pragma unroll
      for (int c = 0; c < D; ++c) { f[c] = T(0); z[c] = T(0); }
      for (uint32_t l2 = 0; l2 < p; ++l2) {
        if (l2 == l) continue;
        T xj[D];
        ld(js[s0 + l2], xj);
        add_interaction<T, D, KK>(xi, xj, f, P);
      }
      const T inv = T(1) / T(p - 1);
#pragma unroll
      for (int c = 0; c < D; ++c) f[c] *= inv;
      if (P.has_noise) Normals<T, D>::get(P, (uint32_t)(s0 + l), m, TAG_NOISE_SLOT, z);
      em_update<T, D>(xi, f, z, xn[l], P, true);
      check_finite<T, D>(xn[l], P, js[s0 + l], m);
    }
    for (uint32_t l = 0; l < p; ++l) {
      const uint32_t j = js[s0 + l];
#pragma unroll
      for (int c = 0; c < D; ++c) xa[(size_t)j * 4 + c] = xn[l][c];
    }
  } else {
    const uint32_t i = js[s0], j = js[s0 + 1];
    T xi[D], xj[D], y[D], z[D], xn[D];
    ld(i, xi);
    ld(j, xj);
#pragma unroll
    for (int c = 0; c < D; ++c) z[c] = T(0);
    if (KK == KK_ADJ) adj_flow<T, D>(P, i, j, xi, xj, true, y);
    else pair_flow<T, D, KK>(xi, xj, true, y, P);
    if (P.has_noise) Normals<T, D>::get(P, (uint32_t)s0, m, TAG_NOISE_SLOT, z);
    split_finish<T, D>(y, z, xn, P, true);
    check_finite<T, D>(xn, P, i, m);
    T yj[D], xnj[D];
#pragma unroll
    for (int c = 0; c < D; ++c) z[c] = T(0);
    if (KK == KK_ADJ) adj_flow<T, D>(P, i, j, xi, xj, false, yj);
    else pair_flow<T, D, KK>(xi, xj, false, yj, P);
    if (P.has_noise) Normals<T, D>::get(P, (uint32_t)(s0 + 1), m, TAG_NOISE_SLOT, z);
    split_finish<T, D>(yj, z, xnj, P, true);
    check_finite<T, D>(xnj, P, j, m);
#pragma unroll
    for (int c = 0; c < D; ++c) { xa[(size_t)i * 4 + c] = xn[c]; xa[(size_t)j * 4 + c] = xnj[c]; }
  }
}

// p = 2: the new positions of both members, computed exactly as seq_batch
// does (same operations, same order)
template <typename T, int D, int KK, int INTEG>
__device__ __forceinline__ void seq_pair(const DevParams& P, uint32_t m, uint64_t s0, uint32_t i, uint32_t j,
                                         const T (&xi)[D], const T (&xj)[D], T (&xni)[D], T (&xnj)[D]) {
  T z[D];
  if (INTEG == 0) {
    T f[D];
#pragma unroll
    for (int c = 0; c < D; ++c) { f[c] = T(0); z[c] = T(0); }
    add_interaction<T, D, KK>(xi, xj, f, P);
#pragma unroll
    for (int c = 0; c < D; ++c) f[c] *= T(1);
    if (P.has_noise) Normals<T, D>::get(P, (uint32_t)s0, m, TAG_NOISE_SLOT, z);
    em_update<T, D>(xi, f, z, xni, P, true);
#pragma unroll
    for (int c = 0; c < D; ++c) { f[c] = T(0); z[c] = T(0); }
    add_interaction<T, D, KK>(xj, xi, f, P);
#pragma unroll
    for (int c = 0; c < D; ++c) f[c] *= T(1);
    if (P.has_noise) Normals<T, D>::get(P, (uint32_t)(s0 + 1), m, TAG_NOISE_SLOT, z);
    em_update<T, D>(xj, f, z, xnj, P, true);
  } else {
    T y[D];
#pragma unroll
    for (int c = 0; c < D; ++c) z[c] = T(0);
    if (KK == KK_ADJ) adj_flow<T, D>(P, i, j, xi, xj, true, y);
    else pair_flow<T, D, KK>(xi, xj, true, y, P);
    if (P.has_noise) Normals<T, D>::get(P, (uint32_t)s0, m, TAG_NOISE_SLOT, z);
    split_finish<T, D>(y, z, xni, P, true);
#pragma unroll
    for (int c = 0; c < D; ++c) z[c] = T(0);
    if (KK == KK_ADJ) adj_flow<T, D>(P, i, j, xi, xj, false, y);
    else pair_flow<T, D, KK>(xi, xj, false, y, P);
    if (P.has_noise) Normals<T, D>::get(P, (uint32_t)(s0 + 1), m, TAG_NOISE_SLOT, z);
    split_finish<T, D>(y, z, xnj, P, true);
  }
  check_finite<T, D>(xni, P, i, m);
  check_finite<T, D>(xnj, P, j, m);
}

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* a) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_gpu(const uint32_t* a) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_gpu(uint32_t* a, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
// one 16-byte record, read and written whole at L2 (the position and its tag
// together, as one aligned 128-bit access)
__device__ __forceinline__ uint4 ld_cg_v4(const void* a) {
  uint4 v;
  asm volatile("ld.global.cg.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_cg_v4(void* a, uint4 v) {
  asm volatile("st.global.cg.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
// expect value of a particle's first slot in the sweep: no earlier writer
constexpr uint32_t SEQ_FREE = 0xffffffffu;
// the write counter of particle j: the padding word of its AoS record (D <= 3)
template <typename T> __device__ __forceinline__ uint32_t* seq_tag(T* xa, uint32_t j) {
  return reinterpret_cast<uint32_t*>(xa + (size_t)j * 4 + 3);
}
// wait until the earlier writers of the particle are done (tag >= e, mod 2^32)
template <typename T> __device__ __forceinline__ void wait_tag(T* xa, uint32_t j, uint32_t e) {
  if (e == SEQ_FREE) return;
  while ((int32_t)(ld_acquire_gpu(seq_tag(xa, j)) - e) < 0) __nanosleep(32);
}
template <typename T> __device__ __forceinline__ uint32_t next_tag(T* xa, uint32_t j, uint32_t e) {
  return (e == SEQ_FREE ? ld_relaxed_gpu(seq_tag(xa, j)) : e) + 1u;
}

template <typename T, int D, int KK, int INTEG>
static __global__ void __launch_bounds__(128) rbmr_seq_dep_kernel(const __grid_constant__ DevParams P, uint64_t nbatch,
                                                                  const uint32_t* __restrict__ js,
                                                                  const uint32_t* __restrict__ expect, T* xa,
                                                                  uint32_t* ticket) {
  const uint32_t m = (uint32_t)*P.step;
  const uint32_t p = P.p;
  const uint32_t lane = threadIdx.x & 31u;
  for (;;) {
    uint32_t base = 0;
    if (lane == 0) base = atomicAdd(ticket, 32u);
    base = __shfl_sync(0xffffffffu, base, 0);
    if ((uint64_t)base >= nbatch) break;
    const uint64_t b = (uint64_t)base + lane;
    if (b < nbatch) {
      if (p == 2) {
        const uint2 jj = reinterpret_cast<const uint2*>(js)[b];
        const uint2 ex = reinterpret_cast<const uint2*>(expect)[b];
        T xi[D], xj[D], xni[D], xnj[D];
        if constexpr (sizeof(T) == 4) {
          // 16-byte records {x, tag}: the tag is polled in the same 128-bit
          // load that returns the position, and the new position goes out
          // with the bumped tag in one 128-bit store (no fence)
          uint4 ri = ld_cg_v4(xa + (size_t)jj.x * 4), rj = ld_cg_v4(xa + (size_t)jj.y * 4);
          while (ex.x != SEQ_FREE && (int32_t)(ri.w - ex.x) < 0) { __nanosleep(32); ri = ld_cg_v4(xa + (size_t)jj.x * 4); }
          while (ex.y != SEQ_FREE && (int32_t)(rj.w - ex.y) < 0) { __nanosleep(32); rj = ld_cg_v4(xa + (size_t)jj.y * 4); }
          const uint32_t wi[3] = {ri.x, ri.y, ri.z}, wj[3] = {rj.x, rj.y, rj.z};
#pragma unroll
          for (int c = 0; c < D; ++c) { xi[c] = __uint_as_float(wi[c]); xj[c] = __uint_as_float(wj[c]); }
          seq_pair<T, D, KK, INTEG>(P, m, b * 2, jj.x, jj.y, xi, xj, xni, xnj);
          uint32_t oi[3] = {0u, 0u, 0u}, oj[3] = {0u, 0u, 0u};
#pragma unroll
          for (int c = 0; c < D; ++c) { oi[c] = __float_as_uint((float)xni[c]); oj[c] = __float_as_uint((float)xnj[c]); }
          st_cg_v4(xa + (size_t)jj.x * 4, make_uint4(oi[0], oi[1], oi[2], ri.w + 1u));
          st_cg_v4(xa + (size_t)jj.y * 4, make_uint4(oj[0], oj[1], oj[2], rj.w + 1u));
        } else {
          wait_tag(xa, jj.x, ex.x);
          wait_tag(xa, jj.y, ex.y);
#pragma unroll
          for (int c = 0; c < D; ++c) { xi[c] = __ldcg(xa + (size_t)jj.x * 4 + c); xj[c] = __ldcg(xa + (size_t)jj.y * 4 + c); }
          seq_pair<T, D, KK, INTEG>(P, m, b * 2, jj.x, jj.y, xi, xj, xni, xnj);
          const uint32_t ti = next_tag(xa, jj.x, ex.x), tj = next_tag(xa, jj.y, ex.y);
#pragma unroll
          for (int c = 0; c < D; ++c) { xa[(size_t)jj.x * 4 + c] = xni[c]; xa[(size_t)jj.y * 4 + c] = xnj[c]; }
          fence_acq_rel_gpu();  // positions before the tags (release pattern)
          st_relaxed_gpu(seq_tag(xa, jj.x), ti);
          st_relaxed_gpu(seq_tag(xa, jj.y), tj);
        }
      } else {
        const uint64_t s0 = b * p;
        for (uint32_t l = 0; l < p; ++l) wait_tag(xa, js[s0 + l], expect[s0 + l]);
        seq_batch<T, D, KK, INTEG>(P, m, b, js, xa);
        fence_acq_rel_gpu();
        for (uint32_t l = 0; l < p; ++l) {
          const uint32_t j = js[s0 + l], e = expect[s0 + l];
          // a first slot's tag is stable until this batch bumps it
          st_relaxed_gpu(seq_tag(xa, j), e == SEQ_FREE ? ld_relaxed_gpu(seq_tag(xa, j)) + 1u : e + 1u);
        }
      }
    }
    __syncwarp();
  }
}

// ------------------------ RBM-r on a partitioned global system (row e2)
// Rank r owns the ids [id0, id0 + n0) (AoS state xa in local order) and the
// batches [bb0, bb1) of the sweep (floor(nb r / G)).  One step (the Jacobi
// sweep of reading D:8, SURVEY 8(e) "request, response, increment return"):
//   A  draw j_s of the own slots (the G = 1 counters: bit-identical slots),
//      request j_s from its owner: chunk dest of Q gets j_s at a cursor
//   Q  all-to-all of the request chunks (header: count)
//   B  serve: x[j] of every received request into the response chunk
//   Pr all-to-all of the responses (reverse direction, same positions)
//   C  Delta_s of every own batch from the responses (rbmr_deltas: the same
//      arithmetic as the one-GPU kernel), increment record (s, Delta_s) at the
//      request's position
//   I  all-to-all of the increments
//   D  the owner registers every received increment at its particle and adds
//      them order-independently (Fx, as on one GPU): bit-identical to G = 1.
constexpr int RP_MAXG = 64;
struct RPart {
  uint32_t G, rank, cap;                 // ranks, this rank, records per (source, destination) chunk
  uint64_t n, id0, n0, bb0, bb1;         // global N; own ids; own batches
  uint64_t qchunk, pchunk, ichunk;       // bytes per chunk of the exchanges Q, Pr, I
  uint64_t ioff;                         // byte offset of the Delta array inside an I chunk
  unsigned char *qs, *qr, *ps, *pr, *is, *ir;  // send / receive regions (G chunks each)
  uint32_t* qcnt;                        // G request cursors
  uint32_t* spos;                        // own slot -> dest << 24 | pos
  uint64_t idb[RP_MAXG + 1];             // first id of every rank; idb[G] = N
};

__device__ __forceinline__ uint32_t rp_owner(const RPart& R, uint32_t j) {
  uint32_t a = 0, b = R.G;  // largest a with idb[a] <= j
  while (b - a > 1) {
    const uint32_t mid = (a + b) >> 1;
    if (R.idb[mid] <= j) a = mid; else b = mid;
  }
  return a;
}

// draws of slot s0 + l (distinct within the batch, reading D:9)
__device__ __forceinline__ uint32_t rbmr_draw(const DevParams& P, uint32_t m, uint64_t s, const uint32_t* prev,
                                              uint32_t l) {
  uint32_t t = 0, j;
  for (;;) {
    const uint4 w = block_at(P, (uint32_t)s, t, m, TAG_SLOT);
    j = (uint32_t)__umul64hi(P.n, (((uint64_t)w.x) << 32) | w.y);
    bool dup = false;
    for (uint32_t l2 = 0; l2 < l; ++l2) dup |= (prev[l2] == j);
    if (!dup) return j;
    ++t;
  }
}

// Delta_s of the p slots of batch s0/p from the members' positions x[l]
// (Eq. 2.2 over the batch in ascending lane order, prefactor 1/(p-1), exactly
// 1 for pairs; or the exact pair flow)
template <typename T, int D, int KK, int INTEG, int PMAX = 64>
__device__ __forceinline__ void rbmr_deltas(const DevParams& P, uint32_t m, uint64_t s0, uint32_t p,
                                            const uint32_t* jj, T (*x)[D], T (*dl)[D]) {
  for (uint32_t l = 0; l < (uint32_t)PMAX; ++l) {
    if (l >= p) break;
    T z[D], xn[D];
#pragma unroll
    for (int c = 0; c < D; ++c) z[c] = T(0);
    if (P.has_noise) Normals<T, D>::get(P, (uint32_t)(s0 + l), m, TAG_NOISE_SLOT, z);
    if (INTEG == 0) {
      T f[D];
#pragma unroll
      for (int c = 0; c < D; ++c) f[c] = T(0);
      for (uint32_t l2 = 0; l2 < (uint32_t)PMAX; ++l2) {
        if (l2 >= p) break;
        if (l2 == l) continue;
        add_interaction<T, D, KK>(x[l], x[l2], f, P);
      }
      const T inv = T(1) / T(p - 1);
#pragma unroll
      for (int c = 0; c < D; ++c) f[c] *= inv;
      em_update<T, D>(x[l], f, z, xn, P, false);
    } else {
      T y[D];
      if (KK == KK_ADJ) adj_flow<T, D>(P, jj[0], jj[1], x[0], x[1], l == 0, y);
      else pair_flow<T, D, KK>(x[0], x[1], l == 0, y, P);
      split_finish<T, D>(y, z, xn, P, false);
    }
#pragma unroll
    for (int c = 0; c < D; ++c) dl[l][c] = xn[c] - x[l][c];
  }
}

// A: one thread per own batch
static __global__ void __launch_bounds__(128) rbmr_req_kernel(const __grid_constant__ DevParams P,
                                                              const __grid_constant__ RPart R, uint32_t* __restrict__ js) {
  const uint32_t m = (uint32_t)*P.step;
  const uint32_t p = P.p;
  for (uint64_t b = R.bb0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < R.bb1;
       b += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s0 = b * p, sl0 = (b - R.bb0) * p;
    uint32_t jj[64];
    for (uint32_t l = 0; l < p; ++l) {
      const uint32_t j = rbmr_draw(P, m, s0 + l, jj, l);
      jj[l] = j;
      js[sl0 + l] = j;
      const uint32_t dest = rp_owner(R, j);
      const uint32_t pos = atomicAdd(&R.qcnt[dest], 1u);
      if (pos >= R.cap) { atomicExch(P.capacity_err, 1u); R.spos[sl0 + l] = 0xffffffffu; continue; }
      reinterpret_cast<uint32_t*>(R.qs + dest * R.qchunk + 16)[pos] = j;
      R.spos[sl0 + l] = (dest << 24) | pos;
    }
  }
}

// request counts into the chunk headers
static __global__ void rbmr_req_counts_kernel(const __grid_constant__ RPart R) {
  for (uint32_t q = threadIdx.x; q < R.G; q += blockDim.x)
    *reinterpret_cast<uint32_t*>(R.qs + q * R.qchunk) = min(R.qcnt[q], R.cap);
}

// B: serve the received requests (x of the own particles, 4 scalars each)
template <typename T, int D>
static __global__ void rbmr_serve_kernel(const __grid_constant__ RPart R, const T* __restrict__ xa) {
  const uint64_t total = (uint64_t)R.G * R.cap;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < total; k += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t q = (uint32_t)(k / R.cap), e = (uint32_t)(k - (uint64_t)q * R.cap);
    const unsigned char* qc = R.qr + q * R.qchunk;
    if (e >= *reinterpret_cast<const uint32_t*>(qc)) continue;
    const uint64_t jl = reinterpret_cast<const uint32_t*>(qc + 16)[e] - R.id0;
    T* o = reinterpret_cast<T*>(R.ps + q * R.pchunk) + (size_t)e * 4;
#pragma unroll
    for (int c = 0; c < 4; ++c) o[c] = xa[jl * 4 + c];
  }
}

// C: Delta of every own batch from the responses -> increment records
template <typename T, int D, int KK, int INTEG>
static __global__ void __launch_bounds__(128) rbmr_delta_part_kernel(const __grid_constant__ DevParams P,
                                                                     const __grid_constant__ RPart R) {
  const uint32_t m = (uint32_t)*P.step;
  const uint32_t p = P.p;
  for (uint64_t b = R.bb0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < R.bb1;
       b += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s0 = b * p, sl0 = (b - R.bb0) * p;
    T x[64][D], dl[64][D];
    bool ok = true;
    for (uint32_t l = 0; l < p; ++l) {
      const uint32_t sp = R.spos[sl0 + l];
      if (sp == 0xffffffffu) { ok = false; break; }
      const T* src = reinterpret_cast<const T*>(R.pr + (sp >> 24) * R.pchunk) + (size_t)(sp & 0xffffffu) * 4;
#pragma unroll
      for (int c = 0; c < D; ++c) x[l][c] = src[c];
    }
    if (!ok) continue;  // capacity overflow (flagged by the request kernel)
    rbmr_deltas<T, D, KK, INTEG>(P, m, s0, p, R.spos + sl0, x, dl);
    for (uint32_t l = 0; l < p; ++l) {
      const uint32_t sp = R.spos[sl0 + l], dest = sp >> 24, pos = sp & 0xffffffu;
      unsigned char* ic = R.is + dest * R.ichunk;
      reinterpret_cast<uint32_t*>(ic)[pos] = (uint32_t)(s0 + l);
      T* o = reinterpret_cast<T*>(ic + R.ioff) + (size_t)pos * 4;
#pragma unroll
      for (int c = 0; c < 4; ++c) o[c] = (c < D) ? dl[l][c < D ? c : 0] : T(0);
    }
  }
}

// D1: register every received increment (index q * cap + e) at its particle
static __global__ void rbmr_register_part_kernel(const __grid_constant__ DevParams P, const __grid_constant__ RPart R,
                                                 uint32_t* __restrict__ mcnt, uint32_t* __restrict__ mbox,
                                                 uint32_t* __restrict__ ovf, uint32_t* __restrict__ novf) {
  const uint64_t total = (uint64_t)R.G * R.cap;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < total; k += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t q = (uint32_t)(k / R.cap), e = (uint32_t)(k - (uint64_t)q * R.cap);
    const unsigned char* qc = R.qr + q * R.qchunk;  // the requests this rank served, same positions
    if (e >= *reinterpret_cast<const uint32_t*>(qc)) continue;
    const uint32_t jl = (uint32_t)(reinterpret_cast<const uint32_t*>(qc + 16)[e] - R.id0);
    const uint32_t idx = q * R.cap + e;
    const uint32_t pos = atomicAdd(&mcnt[jl], 1u);
    if (pos < MBOX) {
      mbox[(size_t)jl * MBOX + pos] = idx;
    } else {
      const uint32_t o = atomicAdd(novf, 1u);
      if (o < OVF_CAP) { ovf[2 * o] = jl; ovf[2 * o + 1] = idx; }
      else atomicExch(P.capacity_err, 1u);
    }
  }
}

// D2: x_j += the order-independent sum of its increments (Fx, reading D:8)
template <typename T, int D>
static __global__ void rbmr_apply_part_kernel(const __grid_constant__ DevParams P, const __grid_constant__ RPart R,
                                              T* __restrict__ xa, const uint32_t* __restrict__ mcnt,
                                              const uint32_t* __restrict__ mbox, const uint32_t* __restrict__ ovf,
                                              const uint32_t* __restrict__ novf) {
  const uint32_t m = (uint32_t)*P.step;
  constexpr uint32_t MAXL = 32;
  for (uint64_t jl = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; jl < R.n0;
       jl += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c = mcnt[jl];
    if (c == 0) continue;
    uint32_t ix[MAXL];
    uint32_t k = 0;
    const uint32_t cm = c < MBOX ? c : MBOX;
    for (uint32_t q = 0; q < cm; ++q) ix[k++] = mbox[jl * MBOX + q];
    if (c > MBOX) {
      const uint32_t no = min(*novf, OVF_CAP);
      for (uint32_t q = 0; q < no; ++q)
        if (ovf[2 * q] == (uint32_t)jl) {
          if (k < MAXL) ix[k++] = ovf[2 * q + 1];
          else atomicExch(P.capacity_err, 1u);
        }
    }
    auto dd = [&](uint32_t idx) {
      return reinterpret_cast<const T*>(R.ir + (idx / R.cap) * R.ichunk + R.ioff) + (size_t)(idx % R.cap) * 4;
    };
    T x[D];
    load4<T, D>(xa, (uint32_t)jl, x);
    uint32_t E = 0;  // order-independent fixed-point sums (Fx, D:8), as on one GPU
    for (uint32_t a = 0; a < k; ++a)
#pragma unroll
      for (int cc = 0; cc < D; ++cc) E = max(E, Fx<T>::ex(dd(ix[a])[cc]));
#pragma unroll
    for (int cc = 0; cc < D; ++cc) {
      long long acc = 0;
      for (uint32_t a = 0; a < k; ++a) acc += Fx<T>::q(dd(ix[a])[cc], E);
      x[cc] = Fx<T>::add(x[cc], acc, E);
    }
    if (P.constraint == 1) renormalise<T, D>(x);
    check_finite<T, D>(x, P, (uint32_t)(R.id0 + jl), m);
#pragma unroll
    for (int cc = 0; cc < D; ++cc) xa[jl * 4 + cc] = x[cc];
  }
}

// partitioned RBM-r: pack this rank's records (id order, ids [id0, id0+n0)) -> xa
template <typename T, int D>
static __global__ void rbmr_pack_local_kernel(uint64_t n0, State<T, D> st, T* __restrict__ xa) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n0;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const Rec<T, D> r = ld_rec<T, D>(st.rec, (long long)i);
#pragma unroll
    for (int c = 0; c < 4; ++c) xa[i * 4 + c] = (c < D) ? r.x[c < D ? c : 0] : T(0);
  }
}

// gather from a rank's AoS state (ids [id0, id0+n0)) for ids [i0, i1): rows of its own ids
template <typename T, int D>
static __global__ void gather_aos_part_kernel(const T* __restrict__ xa, uint64_t id0, uint64_t n0, uint64_t i0,
                                              uint64_t i1, T* __restrict__ out, uint32_t* __restrict__ ids) {
  for (uint64_t jl = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; jl < n0;
       jl += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t id = id0 + jl;
    if (ids) {  // local gather: (ids, rows) in local order
      ids[jl] = (uint32_t)id;
#pragma unroll
      for (int c = 0; c < D; ++c) out[jl * D + c] = xa[jl * 4 + c];
    } else if (id >= i0 && id < i1) {
#pragma unroll
      for (int c = 0; c < D; ++c) out[(id - i0) * D + c] = xa[jl * 4 + c];
    }
  }
}

// ------------------------------------------- RBM-r Jacobi sweep, one GPU
// The increments Delta_s are routed to their particles through the same
// MSD partition as the RBM-1 records, keyed by j_s (no random mailboxes):
//   emit     one thread per batch: draws j_s (as the oracle, reading D:9),
//            gathers x_{j_s}, computes Delta_s (rbmr_deltas), and the CTA's
//            records {j_s, Delta_s} are staged by the top b1 bits of j_s
//            and written as coalesced runs into the pass-1 buckets
//   split    pass-1 -> final buckets of 2^(idbits-B) particle ids (split_kernel<IncRT>)
//   apply    one CTA per final bucket of W ids: per coordinate, the largest
//            increment exponent of each particle (shared-memory atomicMax),
//            then the exact fixed-point sum of its increments (64-bit
//            shared-memory atomics, any order), added once (Fx, reading D:8)
constexpr int EMIT_BLOCK = 256;
constexpr uint32_t EMIT_TS = 2048;  // slots per emit CTA

// staged records, ranks, staging index, and hist / gbase / off over the 2^b1
// output digits (sized by b1: four CTAs per SM at C5)
template <typename T, int D, bool LINK> __host__ __device__ constexpr size_t emit_smem_bytes(uint32_t b1 = 10) {
  return (size_t)EMIT_TS * IncOrLink<T, D, LINK>::RS + (size_t)EMIT_TS * (4 + 2) + (3 * (1u << b1) + 64) * 4;
}

// LINK (the sequential RBM-r'): the records are {j_s, s} only (no gathers)
template <typename T, int D, int KK, int INTEG, bool LINK>
static __global__ void __launch_bounds__(EMIT_BLOCK) rbmr_emit_kernel(const __grid_constant__ DevParams P, uint64_t nbatch,
                                                                      const T* __restrict__ xa, uint32_t* __restrict__ js,
                                                                      unsigned char* __restrict__ dst, uint32_t* cur,
                                                                      uint32_t dcap) {
  using IL = IncOrLink<T, D, LINK>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char* stg = smem_raw;                                            // EMIT_TS records
  uint32_t* rk = reinterpret_cast<uint32_t*>(stg + (size_t)EMIT_TS * IL::RS);  // digit << 16 | rank
  uint16_t* inv = reinterpret_cast<uint16_t*>(rk + EMIT_TS);
  uint32_t* hist = reinterpret_cast<uint32_t*>(inv + EMIT_TS);             // 2^b1
  uint32_t* gbase = hist + (1u << P.b1);                                   // 2^b1
  uint32_t* off = gbase + (1u << P.b1);                                    // 2^b1
  uint32_t* wsum = off + (1u << P.b1);                                     // 64
  const uint32_t m = (uint32_t)*P.step;
  const uint32_t p = P.p;
  const uint32_t bpc = EMIT_TS / p;  // batches per CTA
  const uint64_t b0 = (uint64_t)blockIdx.x * bpc;
  if (b0 >= nbatch) return;
  const uint32_t nb = (uint32_t)min((uint64_t)bpc, nbatch - b0), cnt = nb * p;
  const uint32_t nbins = 1u << P.b1, sh = 32u - P.b1;
  for (uint32_t i = threadIdx.x; i < nbins; i += EMIT_BLOCK) hist[i] = 0;
  __syncthreads();
  auto batches = [&](auto pm) {
    constexpr int PM = decltype(pm)::value;  // array bound: 2 (registers) or 64
    for (uint32_t lb = threadIdx.x; lb < nb; lb += EMIT_BLOCK) {
      const uint64_t b = b0 + lb, s0 = b * p;
      uint32_t jj[PM];
      if (KK == KK_ADJ && P.adj_edges) {
        adj_edge_draw(P, s0, m, jj[0], jj[PM > 1 ? 1 : 0]);
      } else {
        for (uint32_t l = 0; l < (uint32_t)PM; ++l) {
          if (l >= p) break;
          jj[l] = rbmr_draw(P, m, s0 + l, jj, l);
        }
      }
      T dl[LINK ? 1 : PM][D];
      if constexpr (!LINK) {
        T x[PM][D];
        for (uint32_t l = 0; l < (uint32_t)PM; ++l) {
          if (l >= p) break;
          load4<T, D>(xa, jj[l], x[l]);
        }
        rbmr_deltas<T, D, KK, INTEG, PM>(P, m, s0, p, jj, x, dl);
      }
      for (uint32_t l = 0; l < (uint32_t)PM; ++l) {
        if (l >= p) break;
        const uint32_t e = lb * p + l;
        if (js) js[s0 + l] = jj[l];  // RBM-r' only (its sweep reads them); the Jacobi sweep recomputes on demand
        uint32_t w[IL::NW];
#pragma unroll
        for (int k = 0; k < IL::NW; ++k) w[k] = 0u;
        w[0] = jj[l];
        if constexpr (LINK) {
          w[1] = (uint32_t)(s0 + l);
        } else {
#pragma unroll
          for (int c = 0; c < D; ++c) to_w(dl[l][c], w + IncL<T, D>::XW + c * (int)(sizeof(T) / 4));
        }
        st_words<IL::NW>(stg + (size_t)e * IL::RS, w);
        const uint32_t dg = (jj[l] << P.jshift) >> sh;
        rk[e] = (dg << 16) | atomicAdd(&hist[dg], 1u);
      }
    }
  };
  if (p == 2) batches(std::integral_constant<int, 2>{});
  else batches(std::integral_constant<int, 64>{});
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < nbins; i += EMIT_BLOCK) {
    const uint32_t h = hist[i];
    off[i] = h;
    gbase[i] = h ? atomicAdd(&cur[(size_t)i * CUR1_STRIDE], h) : 0u;
  }
  __syncthreads();
  block_excl_scan<EMIT_BLOCK>(off, nbins, wsum);
  for (uint32_t e = threadIdx.x; e < cnt; e += EMIT_BLOCK) {
    const uint32_t v = rk[e];
    RBM_CHECK(P, off[v >> 16] + (v & 0xffffu) < cnt);
    inv[off[v >> 16] + (v & 0xffffu)] = (uint16_t)e;
  }
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < cnt; j += EMIT_BLOCK) {
    const uint32_t e = inv[j];
    const uint32_t dg = rk[e] >> 16;
    const uint32_t slot = gbase[dg] + (j - off[dg]);
    if (slot >= dcap) { atomicExch(P.capacity_err, 1u); continue; }
    uint32_t w[IL::NW];
    ld_words<IL::NW>(stg + (size_t)e * IL::RS, w);
    st_words<IL::NW>(dst + ((size_t)dg * dcap + slot) * IL::RS, w);
  }
}

// the slot draws j_s of step m (test hook rbm_debug_slots of the one-GPU
// Jacobi sweep, whose emit kernel does not store them): the emit's draws, one
// thread per batch
template <int KK>
static __global__ void rbmr_slots_kernel(const __grid_constant__ DevParams P, uint64_t nbatch, uint32_t m,
                                         uint32_t* __restrict__ js) {
  const uint32_t p = P.p;
  for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < nbatch;
       b += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s0 = b * p;
    uint32_t jj[64];
    if (KK == KK_ADJ && P.adj_edges) {
      adj_edge_draw(P, s0, m, jj[0], jj[1]);
    } else {
      for (uint32_t l = 0; l < p; ++l) jj[l] = rbmr_draw(P, m, s0 + l, jj, l);
    }
    for (uint32_t l = 0; l < p; ++l) js[s0 + l] = jj[l];
  }
}

template <typename T, int D, bool LINK> __host__ __device__ constexpr size_t rapply_smem_bytes(uint32_t cap, uint32_t W) {
  return LINK ? (size_t)(cap + 8) * IncOrLink<T, D, LINK>::RS + (size_t)cap * 4 + (size_t)W * 8 + 64 * 4 + 16
              : (size_t)W * (2 + Fx<T>::NCH * D) * 4 + 16;  // Jacobi: exponent, count, chunk sums per particle
}

// apply: final bucket b = the particle ids [b W, (b+1) W); n = cnt[b] records.
// LINK (the sequential RBM-r'): instead of adding increments, the a-th slot
// s_a of particle j (ascending) gets expect[s_a] = tag_j + a for a > 0 (the
// caller presets expect[] to SEQ_FREE, the first slot's value)
template <typename T, int D, bool LINK>
static __global__ void __launch_bounds__(256, 4) rbmr_bucket_apply_kernel(const __grid_constant__ DevParams P,
                                                                       const unsigned char* __restrict__ fin, uint32_t cap,
                                                                       const uint32_t* __restrict__ cnt, uint32_t W,
                                                                       T* __restrict__ xa, uint32_t* __restrict__ expect) {
  using IL = IncOrLink<T, D, LINK>;
  constexpr int BLOCK = 256;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const uint32_t b = blockIdx.x;
  const uint32_t n = cnt[(size_t)b * CUR2_STRIDE];
  const uint64_t j0 = (uint64_t)b * W;
  if (j0 >= P.n) return;
  const uint32_t nid = (uint32_t)min((uint64_t)W, P.n - j0);
  const uint32_t m = (uint32_t)*P.step;
  constexpr int RMAX = 4;  // W <= 1024 particles in registers (larger W: loaded in the loop)
  if constexpr (!LINK) {
    // ---- Jacobi RBM-r: order-independent fixed-point sums (Fx, reading D:8)
    using F = Fx<T>;
    uint32_t* emax = reinterpret_cast<uint32_t*>(smem_raw);  // [W]: common exponent; 0: no increment
    uint32_t* cntp = emax + W;                               // [W]: increments per particle
    uint32_t* ch = cntp + W;                                 // [NCH][W][D]: chunk sums of q + BIAS
    T xv[RMAX][D];
#pragma unroll
    for (int r = 0; r < RMAX; ++r) {  // the id range's positions, loaded before the increments
      const uint32_t jl = threadIdx.x + r * BLOCK;
      if (jl < nid) load4<T, D>(xa, (uint32_t)(j0 + jl), xv[r]);
    }
    for (uint32_t i = threadIdx.x; i < W * (2 + F::NCH * D); i += BLOCK) emax[i] = 0;
    if (n > cap || cap > 8u * BLOCK) {  // cannot happen at the layout's 12-sigma capacity (<= 2048): flagged
      if (threadIdx.x == 0) atomicExch(P.capacity_err, 1u);
      return;
    }
    constexpr int AI = 8;
    uint32_t jl_k[AI];
    T dv[AI][D];
#pragma unroll
    for (int k = 0; k < AI; ++k) {
      const uint32_t e = k * BLOCK + threadIdx.x;
      if (e < n) {
        uint32_t w[IL::NW];
        ld_words<IL::NW>(fin + ((size_t)b * cap + e) * IL::RS, w);
        jl_k[k] = w[0] - (uint32_t)j0;
        RBM_CHECK(P, jl_k[k] < nid);
#pragma unroll
        for (int cc = 0; cc < D; ++cc) from_w(dv[k][cc], w + IncL<T, D>::XW + cc * (int)(sizeof(T) / 4));
      }
    }
    __syncthreads();  // counters zeroed
#pragma unroll
    for (int k = 0; k < AI; ++k)
      if (k * BLOCK + threadIdx.x < n) {
        uint32_t e = 0;
#pragma unroll
        for (int cc = 0; cc < D; ++cc) e = max(e, F::ex(dv[k][cc]));
        atomicMax(&emax[jl_k[k]], e);
        atomicAdd(&cntp[jl_k[k]], 1u);
      }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < AI; ++k)
      if (k * BLOCK + threadIdx.x < n) {
        const uint32_t E = emax[jl_k[k]];
#pragma unroll
        for (int cc = 0; cc < D; ++cc) {
          const unsigned long long qb = (unsigned long long)(F::q(dv[k][cc], E) + F::BIAS);
#pragma unroll
          for (int h = 0; h < F::NCH; ++h)
            atomicAdd(&ch[((size_t)h * W + jl_k[k]) * D + cc],
                      (uint32_t)((qb >> (F::CB * h)) & ((h + 1 < F::NCH) ? ((1ull << F::CB) - 1ull) : ~0ull)));
        }
      }
    __syncthreads();
    auto particle = [&](uint32_t jl, T (&x)[D]) {
      const uint32_t c = cntp[jl];
      if (c == 0u) return;  // no increment
      const uint32_t E = emax[jl];
#pragma unroll
      for (int cc = 0; cc < D; ++cc) {
        long long acc = -(long long)c * F::BIAS;
#pragma unroll
        for (int h = 0; h < F::NCH; ++h) acc += (long long)ch[((size_t)h * W + jl) * D + cc] << (F::CB * h);
        x[cc] = F::add(x[cc], acc, E);
      }
      if (P.constraint == 1) renormalise<T, D>(x);
      check_finite<T, D>(x, P, (uint32_t)(j0 + jl), m);
      store4<T, D>(xa, (uint32_t)(j0 + jl), x);
    };
#pragma unroll
    for (int r = 0; r < RMAX; ++r) {
      const uint32_t jl = threadIdx.x + r * BLOCK;
      if (jl < nid) particle(jl, xv[r]);
    }
    for (uint32_t jl = threadIdx.x + RMAX * BLOCK; jl < nid; jl += BLOCK) {
      T x[D];
      load4<T, D>(xa, (uint32_t)(j0 + jl), x);
      particle(jl, x);
    }
    return;
  }
  // ---- RBM-r' link pass: records grouped by particle, each particle's slots in ascending s
  unsigned char* rs = smem_raw;
  uint32_t* pos = reinterpret_cast<uint32_t*>(rs + (size_t)(cap + 8) * IL::RS);  // element -> rank within its particle
  uint32_t* pc = pos + cap;        // per particle: count
  uint32_t* po = pc + W;           // per particle: first index in ix (after the scan)
  uint32_t* wsum = po + W;
  uint64_t* bar = reinterpret_cast<uint64_t*>(wsum + 64);
  uint16_t* ix = reinterpret_cast<uint16_t*>(pos);  // reused after the placement: sorted element indices
  if (threadIdx.x == 0 && n) {
    mbar_init(bar, 1);
    const uint32_t bytes = (n * (uint32_t)IL::RS + 15u) & ~15u;
    mbar_expect_tx(bar, bytes);
    bulk_g2s_stream(rs, fin + (size_t)b * cap * IL::RS, bytes, bar, l2_evict_first_policy());
  }
  for (uint32_t i = threadIdx.x; i < W; i += BLOCK) pc[i] = 0;
  __syncthreads();
  if (n > cap || cap > 8u * BLOCK) {  // cannot happen at the layout's 12-sigma capacity (<= 2048): flagged
    if (threadIdx.x == 0) atomicExch(P.capacity_err, 1u);
    return;
  }
  if (n) mbar_wait(bar, 0);
  // each record's particle and its arrival rank there (registers), counts per particle
  constexpr int AI = 8;
  uint32_t myjl[AI], myr[AI];
#pragma unroll
  for (int k = 0; k < AI; ++k) {
    const uint32_t e = k * BLOCK + threadIdx.x;
    if (e < n) {
      myjl[k] = (uint32_t)(reinterpret_cast<const uint32_t*>(rs + (size_t)e * IL::RS)[0] - j0);
      RBM_CHECK(P, myjl[k] < nid);
      myr[k] = atomicAdd(&pc[myjl[k]], 1u);
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < W; i += BLOCK) po[i] = pc[i];
  __syncthreads();
  block_excl_scan<BLOCK>(po, (int)W, wsum);
#pragma unroll
  for (int k = 0; k < AI; ++k) {
    const uint32_t e = k * BLOCK + threadIdx.x;
    if (e < n) {
      RBM_CHECK(P, po[myjl[k]] + myr[k] < n);
      ix[po[myjl[k]] + myr[k]] = (uint16_t)e;
    }
  }
  __syncthreads();
  {
    // each slot record ranks itself among its particle's slots by global slot
    // index (the group's records sit at ix[po[j] .. po[j] + c) in arrival
    // order); the a-th slot, a >= 1, gets expect[s] = tag_j + a.  expect[] was
    // preset to SEQ_FREE, which the first slot keeps
    constexpr uint32_t MAXL = 32;
    auto slot_of = [&](uint32_t e) { return reinterpret_cast<const uint32_t*>(rs + (size_t)e * IL::RS)[1]; };
#pragma unroll
    for (int k = 0; k < AI; ++k) {
      const uint32_t e = k * BLOCK + threadIdx.x;
      if (e >= n) continue;
      const uint32_t jl = myjl[k], c = pc[jl];
      if (c < 2) continue;
      if (c > MAXL) {  // flagged; no slot of the particle waits (the sweep cannot hang)
        if (myr[k] == 0) atomicExch(P.capacity_err, 1u);
        continue;
      }
      const uint32_t se = slot_of(e), base = po[jl];
      uint32_t r = 0;
      for (uint32_t q = 0; q < c; ++q) r += (slot_of(ix[base + q]) < se) ? 1u : 0u;
      if (r > 0) expect[se] = *seq_tag(xa, (uint32_t)(j0 + jl)) + r;
    }
  }
}

// gather from the AoS RBM-r state (id order)
template <typename T, int D>
static __global__ void gather_aos_kernel(const T* __restrict__ xa, uint64_t i0, uint64_t i1,
                                         T* __restrict__ out) {
  for (uint64_t i = i0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < i1;
       i += (uint64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int c = 0; c < D; ++c) out[(i - i0) * D + c] = xa[i * 4 + c];
  }
}

}  // namespace rbm

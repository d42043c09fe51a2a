// rbm_device.cuh -- device building blocks of the RBM step (sm_100a).
//
// Philox4x32-10 counter RNG, exact open-interval uniform maps, Box-Muller,
// the registry of interaction kernels K and potentials V, and the per-member
// Euler-Maruyama / split-pair updates of Eq. (2.2).
// Written for this library; shares nothing with oracle/.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace rbm {

enum : uint32_t { TAG_KEY = 0, TAG_NOISE = 1, TAG_INIT = 2, TAG_INIT_AUX = 3,
                  TAG_SLOT = 4, TAG_NOISE_SLOT = 5 };
enum : int { KK_ZERO = 0, KK_DYSON = 1, KK_COULOMB = 2, KK_BOUNDED = 3,
             KK_GAUSS_AR = 4, KK_COULOMB_REG = 5, KK_SMOOTH = 6, KK_LINEAR = 7, KK_ADJ = 8 };

// exact u32 division by a runtime-invariant divisor (Granlund-Montgomery):
// q = n / d for every 32-bit n.
struct FastDiv {
  uint32_t d, m, s;  // s = ceil(log2 d)
};
inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f{d, 0u, 0u};
  uint32_t l = 0;
  while ((1ull << l) < d) ++l;
  f.s = l;
  f.m = (d == 1) ? 0u : (uint32_t)((((1ull << 32) * ((1ull << l) - d)) / d) + 1ull);
  return f;
}
__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
  if (f.s == 0) return n;
  const uint32_t t = __umulhi(n, f.m);
  return (t + ((n - t) >> 1)) >> (f.s - 1);
}

// Everything a kernel needs about the configuration; passed by value.
struct DevParams {
  uint64_t n;          // N
  uint32_t p;          // batch size
  FastDiv pdiv;        // division by p
  uint32_t nfull;      // floor(N/p)
  uint32_t rem;        // N mod p (remainder rule, D:7)
  uint32_t seed_lo, seed_hi;
  uint32_t rk[20];     // Philox round keys (k0, k1) of rounds 0..9 (Weyl schedule)
  uint32_t rep_hi;     // replica << 8, OR-ed into counter word 3
  uint32_t potential;  // 0 none, 1 harmonic
  uint32_t constraint; // 0 none, 1 unit sphere
  uint32_t has_noise;  // sigma > 0
  // model constants in both precisions
  double kp0, kp1, beta, dt, sq;   // sq = sigma*sqrt(dt)
  float kp0f, kp1f, betaf, dtf, sqf;
  double invp;         // 1/(p-1): prefactor of a regular batch (Eq. 2.2)
  float invpf;
  double invr, invp1;  // 1/(r-1) (remainder batch of size r = N mod p >= 2) and 1/p (size p+1, D:7)
  float invrf, invp1f;
  uint32_t geo_noise;  // multiplicative noise sigma x dB (wealth model)
  uint32_t verlet_start;  // Verlet (row f3): this step starts from (x_0, v_0), not (x_n, x_{n-1})
  uint32_t closed_window; // bounded confidence: closed window |z| <= r (the paper's chi_[0,1])
  double half_s2dt, lin_decay;     // sigma^2 dt / 2; e^{-2 kappa dt} (linear pair flow)
  float half_s2dtf, lin_decayf;
  // bucket layout of the partition
  uint32_t B;          // prefix bits of the final buckets
  uint32_t b1, b2;     // digit bits of scatter passes 1 and 2 (b2 = 0: one pass)
  uint32_t nbuckets;   // 2^B
  uint32_t cap;        // per-bucket shared-memory capacity (elements)
  uint32_t SB;         // sub-digit bits of the in-bucket counting sort
  uint32_t idbits;     // bits of an id (ceil log2 N)
  uint32_t lowbits;    // key bits below prefix+sub-digit: 32 - B - SB (lowbits+idbits <= 32)
  uint32_t* dbg_order; // if set: sorted position -> id of this step (test hook)
  uint32_t side_key;   // the bucket step reads key_m from the side array pass 2 wrote (unkeyed records, 2-pass layouts)
  uint32_t jshift;     // RBM-r increment partition: 32 - idbits (key = j << jshift)
  uint32_t group;      // lanes per batch in the fused step: pow2 >= p (<= 32), 0 = one thread per batch
  // partitioned single system (world_size G > 1): this rank
  // owns the key range whose top log2 G bits equal its rank.  The 2^b1 pass-1
  // buckets are global; a rank holds 2^b1/G of them (nb1_loc_mask = that - 1;
  // 2^b1 - 1 on one GPU).  `halo`: the batch crossing the rank's first
  // position is completed with records of rank-1 placed at bucket "-1".
  uint32_t nb1_loc_mask;
  uint32_t halo;
  // output segments: every pass-1 bucket is split into K = 2^segk segments
  // with their own cursors (segment = digit << segk | (producer CTA & (K-1)))
  // so that the run reservations of concurrent CTAs do not serialise on one
  // L2 atomic address per digit
  uint32_t segk, segmask;
  // clustering model (Sec. 5.3, KK_ADJ): symmetric adjacency in CSR (caller-owned,
  // device), kparam = {alpha, beta, edge_restricted}
  const uint32_t* adj_rp;
  const uint32_t* adj_ci;
  const double* adj_v;
  uint64_t adj_nnz;
  uint32_t adj_edges;       // RBM-r pairs drawn among the edges only
  const uint64_t* step;     // device step counter m
  unsigned long long* nonfinite;  // atomicMin of (m<<32 | id); ~0 if clean
  uint32_t* capacity_err;         // set to 1 if a bucket overflowed every fallback
  uint32_t* big_claim;            // NBIG slot flags of the global-scratch fallback
  unsigned char* big_scratch;     // NBIG slots of BIG_CAP elements
  unsigned long long* prof;       // debug (RBM_PHASE_PROF): summed SM cycles per kernel phase
};

// phase profiling (debug only, P.prof set by RBM_PHASE_PROF): thread 0 of
// each CTA adds the cycles since the previous mark to slot i; slot 63 counts CTAs
#define RBM_PROF_BEGIN(P) long long prof_t_ = (P).prof ? clock64() : 0
#define RBM_PROF(P, i)                                                  \
  do {                                                                  \
    if ((P).prof && threadIdx.x == 0) {                                 \
      const long long t_ = clock64();                                   \
      atomicAdd(&(P).prof[i], (unsigned long long)(t_ - prof_t_));     \
      prof_t_ = t_;                                                     \
    }                                                                   \
  } while (0)

// Checked build (librbm_checked.so, -DRBM_CHECKED=1): index bounds asserted
// in the kernels; a violation sets capacity_err = 3, reported by rbm_sync /
// rbm_gather as RBM_ERR_CAPACITY ("bounds check").  compute-sanitizer is not
// available on the GPU pool, so this build is the memory-safety tier.
#ifdef RBM_CHECKED
#define RBM_CHECK(P, cond)                                     \
  do {                                                         \
    if (!(cond)) atomicExch((P).capacity_err, 3u);             \
  } while (0)
#else
#define RBM_CHECK(P, cond) \
  do {                     \
  } while (0)
#endif

constexpr int NBIG = 2;             // concurrent oversized buckets handled per step
constexpr uint32_t BIG_CAP = 65535; // u16 indices
// bytes of one oversized-bucket scratch slot (256-B aligned stride)
__host__ __device__ constexpr size_t big_slot_bytes(size_t rec_x_bytes) {
  return (((size_t)BIG_CAP * (18 + rec_x_bytes) + 64) + 255) & ~(size_t)255;
}

// ------------------------------------------------------------ record layout
// The state is an array of fixed-size records (AoS) so that every move of a
// particle is one vector access: word 0 = id, then (if it fits) word 1 = the
// carried shuffle key of the step the record is partitioned for, then the d
// coordinates.  RS = 8, 16, 24 or 32 bytes:
//   f32 d=1 {id, x} 8 B        f32 d=2 {id, key, x, y} 16 B   f32 d=3 {id, x, y, z} 16 B
//   f64 d=1 {id, key, x} 16 B  f64 d=2 {id, key, x, y} 24 B   f64 d=3 {id, key, x, y, z} 32 B
// Unkeyed layouts recompute key_m from the id (Philox) where it is needed;
// pass 2 hands it to the bucket step in a side array.
template <typename T, int D> struct RecL {
  static constexpr int XB = D * (int)sizeof(T);
  static constexpr int RS = (4 + XB <= 8) ? 8 : ((4 + XB <= 16) ? 16 : ((sizeof(T) == 8 && 8 + XB <= 24) ? 24 : 32));
  static constexpr bool KEYED = 8 + XB <= RS;
  static constexpr int XW = KEYED ? 2 : (sizeof(T) == 8 ? 2 : 1);  // word offset of x[0]
  static constexpr int NW = RS / 4;
};
template <typename T, int D> struct Rec {
  uint32_t id, key;
  T x[D];
};
__device__ __forceinline__ void from_w(float& x, const uint32_t* w) { x = __uint_as_float(w[0]); }
__device__ __forceinline__ void from_w(double& x, const uint32_t* w) { x = __hiloint2double((int)w[1], (int)w[0]); }
__device__ __forceinline__ void to_w(float x, uint32_t* w) { w[0] = __float_as_uint(x); }
__device__ __forceinline__ void to_w(double x, uint32_t* w) {
  w[0] = (uint32_t)__double2loint(x);
  w[1] = (uint32_t)__double2hiint(x);
}
template <int NW>
__device__ __forceinline__ void ld_words(const unsigned char* p, uint32_t (&w)[NW]) {
  if (NW % 4 != 0) {  // 8- and 24-byte records: 8-byte accesses
#pragma unroll
    for (int h = 0; h < NW / 2; ++h) {
      const uint2 v = reinterpret_cast<const uint2*>(p)[h];
      w[2 * h] = v.x; w[2 * h + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int h = 0; h < NW / 4; ++h) {
      const uint4 v = reinterpret_cast<const uint4*>(p)[h];
      w[4 * h] = v.x; w[4 * h + 1] = v.y; w[4 * h + 2] = v.z; w[4 * h + 3] = v.w;
    }
  }
}
template <int NW>
__device__ __forceinline__ void st_words(unsigned char* p, const uint32_t (&w)[NW]) {
  if (NW % 4 != 0) {
#pragma unroll
    for (int h = 0; h < NW / 2; ++h) reinterpret_cast<uint2*>(p)[h] = make_uint2(w[2 * h], w[2 * h + 1]);
  } else {
#pragma unroll
    for (int h = 0; h < NW / 4; ++h)
      reinterpret_cast<uint4*>(p)[h] = make_uint4(w[4 * h], w[4 * h + 1], w[4 * h + 2], w[4 * h + 3]);
  }
}
// record i of the array at base (global or shared memory)
template <typename T, int D>
__device__ __forceinline__ Rec<T, D> ld_rec(const unsigned char* base, long long i) {
  using L = RecL<T, D>;
  uint32_t w[L::NW];
  ld_words<L::NW>(base + i * L::RS, w);
  Rec<T, D> r;
  r.id = w[0];
  r.key = L::KEYED ? w[1] : 0u;
#pragma unroll
  for (int c = 0; c < D; ++c) from_w(r.x[c], w + L::XW + c * (int)(sizeof(T) / 4));
  return r;
}
template <typename T, int D>
__device__ __forceinline__ void st_rec(unsigned char* base, long long i, const Rec<T, D>& r) {
  using L = RecL<T, D>;
  uint32_t w[L::NW];
#pragma unroll
  for (int k = 0; k < L::NW; ++k) w[k] = 0u;
  w[0] = r.id;
  if (L::KEYED) w[1] = r.key;
#pragma unroll
  for (int c = 0; c < D; ++c) to_w(r.x[c], w + L::XW + c * (int)(sizeof(T) / 4));
  st_words<L::NW>(base + i * L::RS, w);
}
template <typename T, int D>
__device__ __forceinline__ uint32_t ld_id(const unsigned char* base, long long i) {
  return *reinterpret_cast<const uint32_t*>(base + i * RecL<T, D>::RS);
}

// ------------------------------------------------- TMA bulk copy + mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes) : "memory");
}
// L2 policy for data read exactly once: evict first, so streaming reads do not
// push out partially written output lines (which would cost a second write)
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// 1-D bulk copy global -> shared (TMA, SASS UBLKCP); 16-B aligned, size % 16 == 0
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_stream(void* dst, const void* src, uint32_t bytes,
                                                uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], "
      "%2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}

// ----------------------------------------------------------------- Philox
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    const uint64_t p0 = (uint64_t)0xD2511F53u * c.x;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c.z;
    c = make_uint4((uint32_t)(p1 >> 32) ^ c.y ^ k0, (uint32_t)p1,
                   (uint32_t)(p0 >> 32) ^ c.w ^ k1, (uint32_t)p0);
  }
  return c;
}

// same function with the 20 round keys precomputed on the host (read from the
// constant bank by LOP3, no per-round key additions)
__device__ __forceinline__ uint4 philox4x32_10_rk(uint4 c, const uint32_t* rk) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c.x;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c.z;
    c = make_uint4((uint32_t)(p1 >> 32) ^ c.y ^ rk[2 * r], (uint32_t)p1,
                   (uint32_t)(p0 >> 32) ^ c.w ^ rk[2 * r + 1], (uint32_t)p0);
  }
  return c;
}

__device__ __forceinline__ uint4 block_at(const DevParams& P, uint32_t c0, uint32_t c1,
                                          uint32_t m, uint32_t tag) {
  return philox4x32_10_rk(make_uint4(c0, c1, m, tag | P.rep_hi), P.rk);
}

// shuffle key of particle `id` at step m: word 0 of the TAG_KEY block
__device__ __forceinline__ uint32_t shuffle_key(const DevParams& P, uint32_t id, uint32_t m) {
  return block_at(P, id, 0u, m, TAG_KEY).x;
}

// ------------------------------------------------------------ uniform maps
// fp32: (2 (w>>9) + 1) 2^-24 == ((w >> 8) | 1) 2^-24, exact.  Computed as
// (1 + (w>>9) 2^-23) - (1 - 2^-24): the float with mantissa w>>9 minus one
// constant; the exact result is an odd multiple of 2^-24 below 1, so the one
// rounding is exact (checked for all 2^23 values of w>>9) and no int->float
// conversion is issued
__device__ __forceinline__ float u01f(uint32_t w) {
  return __uint_as_float(0x3f800000u | (w >> 9)) + __uint_as_float(0xbf7fffffu);
}
// fp64: (2k+1) 2^-53 with k = (a:b) >> 12, exact; as (1 + k 2^-52) - (1 - 2^-53)
// (one exact rounding, as for fp32)
__device__ __forceinline__ double u01d(uint32_t a, uint32_t b) {
  const uint64_t k = ((((uint64_t)a) << 32) | b) >> 12;
  return __longlong_as_double((long long)(0x3ff0000000000000ull | k)) +
         __longlong_as_double((long long)0xbfefffffffffffffull);
}

// ------------------------------------------------------------ Box-Muller
// fp32: MUFU-based (lg2.approx, sin/cos.approx on [0, 2pi)); the radius is
// clamped at 0 so u1 -> 1 can never produce a NaN.  Absolute error of z is
// ~1e-6, far inside the fp32 parity bar.
__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void bm_pair(float u1, float u2, float& z0, float& z1) {
  const float r = sqrt_approx(fmaxf(-1.3862943611198906f * __log2f(u1), 0.0f));  // -2 ln u1
  float s, c;
  __sincosf(6.2831853071795865f * u2, &s, &c);
  z0 = r * c;
  z1 = r * s;
}
__device__ __forceinline__ void bm_pair(double u1, double u2, double& z0, double& z1) {
  const double r = sqrt(-2.0 * log(u1));
  double s, c;
  sincospi(2.0 * u2, &s, &c);
  z0 = r * c;
  z1 = r * s;
}

// d standard normals from counter (c0, *, m, tag); layout of DESIGN.md D:13
template <typename T, int D> struct Normals;
template <int D> struct Normals<float, D> {
  __device__ __forceinline__ static void get(const DevParams& P, uint32_t c0, uint32_t m,
                                             uint32_t tag, float (&z)[D]) {
    const uint4 w = block_at(P, c0, 0u, m, tag);
    float a, b;
    bm_pair(u01f(w.x), u01f(w.y), a, b);
    z[0] = a;
    if (D > 1) z[D > 1 ? 1 : 0] = b;
    if (D > 2) {
      float e, f;
      bm_pair(u01f(w.z), u01f(w.w), e, f);
      z[D > 2 ? 2 : 0] = e;
    }
  }
};
template <int D> struct Normals<double, D> {
  __device__ __forceinline__ static void get(const DevParams& P, uint32_t c0, uint32_t m,
                                             uint32_t tag, double (&z)[D]) {
    const uint4 w = block_at(P, c0, 0u, m, tag);
    double a, b;
    bm_pair(u01d(w.x, w.y), u01d(w.z, w.w), a, b);
    z[0] = a;
    if (D > 1) z[D > 1 ? 1 : 0] = b;
    if (D > 2) {
      const uint4 v = block_at(P, c0, 1u, m, tag);
      double e, f;
      bm_pair(u01d(v.x, v.y), u01d(v.z, v.w), e, f);
      z[D > 2 ? 2 : 0] = e;
    }
  }
};

// ------------------------------------------------------------ model registry
template <typename T> struct Prm;
template <> struct Prm<float> {
  __device__ __forceinline__ static float kp0(const DevParams& P) { return P.kp0f; }
  __device__ __forceinline__ static float kp1(const DevParams& P) { return P.kp1f; }
  __device__ __forceinline__ static float beta(const DevParams& P) { return P.betaf; }
  __device__ __forceinline__ static float dt(const DevParams& P) { return P.dtf; }
  __device__ __forceinline__ static float sq(const DevParams& P) { return P.sqf; }
  __device__ __forceinline__ static float invp(const DevParams& P) { return P.invpf; }
  __device__ __forceinline__ static float invr(const DevParams& P) { return P.invrf; }
  __device__ __forceinline__ static float invp1(const DevParams& P) { return P.invp1f; }
  __device__ __forceinline__ static float half_s2dt(const DevParams& P) { return P.half_s2dtf; }
  __device__ __forceinline__ static float lin_decay(const DevParams& P) { return P.lin_decayf; }
};
template <> struct Prm<double> {
  __device__ __forceinline__ static double kp0(const DevParams& P) { return P.kp0; }
  __device__ __forceinline__ static double kp1(const DevParams& P) { return P.kp1; }
  __device__ __forceinline__ static double beta(const DevParams& P) { return P.beta; }
  __device__ __forceinline__ static double dt(const DevParams& P) { return P.dt; }
  __device__ __forceinline__ static double sq(const DevParams& P) { return P.sq; }
  __device__ __forceinline__ static double invp(const DevParams& P) { return P.invp; }
  __device__ __forceinline__ static double invr(const DevParams& P) { return P.invr; }
  __device__ __forceinline__ static double invp1(const DevParams& P) { return P.invp1; }
  __device__ __forceinline__ static double half_s2dt(const DevParams& P) { return P.half_s2dt; }
  __device__ __forceinline__ static double lin_decay(const DevParams& P) { return P.lin_decay; }
};

__device__ __forceinline__ float inv_cube_sqrt(float q) { const float r = rsqrtf(q); return r * r * r; }
// s(r^2) of the attractive-repulsive Gaussian kernel (C4): fp32 through the
// MUFU exp2 (__expf, ~2 ulp, as rsqrtf above and Box-Muller's MUFU maps, D:13)
__device__ __forceinline__ float gauss_ar(float r2) { return __expf(-0.5f * r2) - 0.25f * __expf(-0.125f * r2); }
__device__ __forceinline__ double gauss_ar(double r2) { return exp(-0.5 * r2) - 0.25 * exp(-0.125 * r2); }
__device__ __forceinline__ double inv_cube_sqrt(double q) { return 1.0 / (q * sqrt(q)); }

// K(z) = s(z) z for every registry entry (Eq. 1.2)
template <typename T, int D, int KK>
__device__ __forceinline__ T kernel_scale(const T (&z)[D], const DevParams& P) {
  T r2 = z[0] * z[0];
#pragma unroll
  for (int c = 1; c < D; ++c) r2 += z[c] * z[c];
  if (KK == KK_ZERO) return T(0);
  if (KK == KK_DYSON) return r2 == T(0) ? T(0) : T(1) / r2;               // 1/z, K(0):=0
  if (KK == KK_COULOMB) return r2 == T(0) ? T(0) : T(1) / (r2 * sqrt(r2));  // z/|z|^3
  if (KK == KK_BOUNDED) {  // -a z 1{|z|<r}; closed window |z| <= r if kparam[2] != 0
    const T az = (D == 1) ? fabs(z[0]) : sqrt(r2), rad = Prm<T>::kp1(P);
    const bool inside = P.closed_window ? (az <= rad) : (az < rad);
    return inside ? -Prm<T>::kp0(P) : T(0);
  }
  if (KK == KK_GAUSS_AR) return gauss_ar(r2);
  if (KK == KK_COULOMB_REG) return inv_cube_sqrt(r2 + Prm<T>::kp0(P));
  if (KK == KK_SMOOTH) return T(1) / (T(1) + r2);
  if (KK == KK_LINEAR) return -Prm<T>::kp0(P);                                // -kappa z
  return T(0);
}

// accumulate K(xi - xj) into f
template <typename T, int D, int KK>
__device__ __forceinline__ void add_interaction(const T (&xi)[D], const T (&xj)[D], T (&f)[D],
                                                const DevParams& P) {
  T z[D];
#pragma unroll
  for (int c = 0; c < D; ++c) z[c] = xi[c] - xj[c];
  const T s = kernel_scale<T, D, KK>(z, P);
#pragma unroll
  for (int c = 0; c < D; ++c) f[c] += s * z[c];
}

template <typename T, int D>
__device__ __forceinline__ void renormalise(T (&x)[D]) {
  T r2 = x[0] * x[0];
#pragma unroll
  for (int c = 1; c < D; ++c) r2 += x[c] * x[c];
  const T r = sqrt(r2);
#pragma unroll
  for (int c = 0; c < D; ++c) x[c] /= r;
}

// Euler-Maruyama member update, f = prefactor * sum K.
// Sphere: drift and noise projected on the tangent plane, then renormalised.
// `normalise` false returns the unnormalised point (RBM-r increments, D:8).
template <typename T, int D>
__device__ __forceinline__ void em_update(const T (&x)[D], const T (&f)[D], const T (&z)[D],
                                          T (&xn)[D], const DevParams& P, bool normalise) {
  T drift[D], zz[D];
  const T beta = Prm<T>::beta(P);
#pragma unroll
  for (int c = 0; c < D; ++c) {
    drift[c] = (P.potential == 1) ? (-(beta * x[c]) + f[c]) : f[c];
    zz[c] = z[c];
  }
  if (P.constraint == 1) {
    T a = T(0), b = T(0);
#pragma unroll
    for (int c = 0; c < D; ++c) { a += drift[c] * x[c]; b += zz[c] * x[c]; }
#pragma unroll
    for (int c = 0; c < D; ++c) { drift[c] -= a * x[c]; zz[c] -= b * x[c]; }
  }
  const T dt = Prm<T>::dt(P), sq = Prm<T>::sq(P);
  if (P.geo_noise) {  // multiplicative noise: Ito term sigma x sqrt(dt) z
#pragma unroll
    for (int c = 0; c < D; ++c) zz[c] *= x[c];
  }
#pragma unroll
  for (int c = 0; c < D; ++c) xn[c] = x[c] + dt * drift[c] + sq * zz[c];
  if (normalise && P.constraint == 1) renormalise<T, D>(xn);
}

// ---------------------------------------------- second order (Verlet, f3)
// A 1-D particle of the Hamiltonian test system stored as
// D = 2 components: (x_0, v_0) at the start, (x_n, x_{n-1}) afterwards.  The
// force acts on the positions (component 0).  Position Verlet:
//   start: x_1 = x_0 + v_0 tau + F_0 tau^2 / 2;  later: x_{n+1} = 2 x_n - x_{n-1} + F_n tau^2
template <typename T, int D, int KK>
__device__ __forceinline__ void add_force1(const T (&xi)[D], const T (&xj)[D], T (&f)[D],
                                           const DevParams& P) {
  T z[1] = {xi[0] - xj[0]};
  const T s = kernel_scale<T, 1, KK>(z, P);
  f[0] += s * z[0];
}

template <typename T, int D>
__device__ __forceinline__ void verlet_update(const T (&x)[D], const T (&f)[D], T (&xn)[D],
                                              const DevParams& P, bool start) {
  const T g = (P.potential == 1) ? Prm<T>::beta(P) * x[0] : T(0);
  const T F = -g + f[0];
  const T t = Prm<T>::dt(P);
  xn[0] = start ? x[0] + x[D > 1 ? 1 : 0] * t + T(0.5) * F * t * t : T(2) * x[0] - x[D > 1 ? 1 : 0] + F * t * t;
  if (D > 1) xn[D > 1 ? 1 : 0] = x[0];
}

// force accumulation and member update of Eq. (2.2) for EM (INTEG 0) and Verlet (2)
template <typename T, int D, int KK, int INTEG>
__device__ __forceinline__ void member_force(const T (&xi)[D], const T (&xj)[D], T (&f)[D],
                                             const DevParams& P) {
  if (INTEG == 2) add_force1<T, D, KK>(xi, xj, f, P);
  else add_interaction<T, D, KK>(xi, xj, f, P);
}

// ---------------------------------------------- canonical partner order
// A batch of sz <= G = P.group members (p <= 32) is summed in the rotation
// order of the lane-group kernel: for o = 1 .. G/2 the partner (li + o) mod G,
// then (li - o) mod G for o < G/2 (partners >= sz skipped).  The lane-group
// kernel evaluates each pair once (K is odd with s(z) = s(-z), so the
// partner's term is exactly the negation) and every other kernel that steps
// such a batch (straddlers, halo, resident, serial) sums the same terms in the
// same order with the same roundings (explicit _rn: no FMA contraction), so a
// batch gives bit-identical results wherever it is computed.  Batches larger
// than G (p > 32, or the long remainder batch) are summed in ascending order.
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

// t = K(xi - xj) (Verlet: the 1-D force on the position coordinate only)
template <typename T, int D, int KK, int INTEG>
__device__ __forceinline__ void pair_term(const T (&xi)[D], const T (&xj)[D], T (&t)[D],
                                          const DevParams& P) {
  if (INTEG == 2) {
    T z[1] = {xi[0] - xj[0]};
    const T s = kernel_scale<T, 1, KK>(z, P);
#pragma unroll
    for (int c = 0; c < D; ++c) t[c] = T(0);
    t[0] = mul_rn(s, z[0]);
  } else {
    T z[D];
#pragma unroll
    for (int c = 0; c < D; ++c) z[c] = xi[c] - xj[c];
    const T s = kernel_scale<T, D, KK>(z, P);
#pragma unroll
    for (int c = 0; c < D; ++c) t[c] = mul_rn(s, z[c]);
  }
}

// f += K(x_li - x_j) over the partners of member li in the canonical order;
// getx(j, xj) loads member j (0 <= j < sz) of the batch
template <typename T, int D, int KK, int INTEG, typename GetX>
__device__ __forceinline__ void batch_force(const DevParams& P, uint32_t li, uint32_t sz,
                                            const T (&xi)[D], GetX getx, T (&f)[D]) {
  const uint32_t G = P.group;
  if (G != 0 && sz <= G) {
    for (uint32_t o = 1; o <= G / 2; ++o) {
      const uint32_t jp = (li + o) & (G - 1);
      if (jp < sz) {
        T xj[D], t[D];
        getx(jp, xj);
        pair_term<T, D, KK, INTEG>(xi, xj, t, P);
#pragma unroll
        for (int c = 0; c < D; ++c) f[c] = add_rn(f[c], t[c]);
      }
      const uint32_t jm = (li - o) & (G - 1);
      if (o < G / 2 && jm < sz) {
        T xj[D], t[D];
        getx(jm, xj);
        pair_term<T, D, KK, INTEG>(xi, xj, t, P);
#pragma unroll
        for (int c = 0; c < D; ++c) f[c] = add_rn(f[c], t[c]);
      }
    }
  } else {
    for (uint32_t j = 0; j < sz; ++j) {  // ascending, self skipped
      if (j == li) continue;
      T xj[D];
      getx(j, xj);
      member_force<T, D, KK, INTEG>(xi, xj, f, P);
    }
  }
}


// exact pair flow (Dyson 922-943, Coulomb 1029-1045, with
// the 1/2 of reading D:3): returns y for the member `first` (true) or second.
template <typename T, int D, int KK>
__device__ __forceinline__ void pair_flow(const T (&xi)[D], const T (&xj)[D], bool first,
                                          T (&y)[D], const DevParams& P) {
  T Dv[D], mid[D], Dn[D];
#pragma unroll
  for (int c = 0; c < D; ++c) { Dv[c] = xi[c] - xj[c]; mid[c] = T(0.5) * (xi[c] + xj[c]); }
  const T dt = Prm<T>::dt(P);
  if (KK == KK_DYSON) {
    const T s = Dv[0] >= T(0) ? T(1) : T(-1);
    Dn[0] = s * sqrt(Dv[0] * Dv[0] + T(4) * dt);
#pragma unroll
    for (int c = 1; c < D; ++c) Dn[c] = T(0);
  } else if (KK == KK_LINEAR) {  // dD/dt = -2 kappa D (wealth trading): D' = D e^{-2 kappa dt}
    const T e = Prm<T>::lin_decay(P);
#pragma unroll
    for (int c = 0; c < D; ++c) Dn[c] = Dv[c] * e;
  } else {  // KK_COULOMB
    T r2 = Dv[0] * Dv[0];
#pragma unroll
    for (int c = 1; c < D; ++c) r2 += Dv[c] * Dv[c];
    const T r = sqrt(r2);
    const T rn = cbrt(r2 * r + T(6) * dt);
#pragma unroll
    for (int c = 0; c < D; ++c) Dn[c] = (r == T(0)) ? (c == 0 ? rn : T(0)) : Dv[c] / r * rn;
  }
  const T sg = first ? T(0.5) : T(-0.5);
#pragma unroll
  for (int c = 0; c < D; ++c) y[c] = mid[c] + sg * Dn[c];
}

// second half of the splitting: x' = y - dt grad V(y) + sq z
template <typename T, int D>
__device__ __forceinline__ void split_finish(const T (&y)[D], const T (&z)[D], T (&xn)[D],
                                             const DevParams& P, bool normalise) {
  const T dt = Prm<T>::dt(P), sq = Prm<T>::sq(P), beta = Prm<T>::beta(P);
#pragma unroll
  for (int c = 0; c < D; ++c) {
    const T g = (P.potential == 1) ? beta * y[c] : T(0);
    const T w = y[c] - dt * g;
    // multiplicative noise: the exact geometric Brownian motion step
    xn[c] = P.geo_noise ? w * exp(sq * z[c] - Prm<T>::half_s2dt(P)) : w + sq * z[c];
  }
  if (normalise && P.constraint == 1) renormalise<T, D>(xn);
}

template <typename T, int D, int INTEG>
__device__ __forceinline__ void member_update(const T (&x)[D], const T (&f)[D], const T (&z)[D], T (&xn)[D],
                                              const DevParams& P, bool vstart) {
  if (INTEG == 2) verlet_update<T, D>(x, f, xn, P, vstart);
  else em_update<T, D>(x, f, z, xn, P, true);
}

// ------------------------------------------- clustering model (KK_ADJ)
// a_ij of the CSR adjacency (rows sorted by column; 0 off the pattern)
__device__ __forceinline__ double adj_value(const DevParams& P, uint32_t i, uint32_t j) {
  uint32_t lo = P.adj_rp[i], hi = P.adj_rp[i + 1];
  const uint32_t end = hi;
  while (lo < hi) {
    const uint32_t mid = lo + (hi - lo) / 2;
    if (P.adj_ci[mid] < j) lo = mid + 1; else hi = mid;
  }
  return (lo < end && P.adj_ci[lo] == j) ? P.adj_v[lo] : 0.0;
}
// exact flow of dX^i/dt = alpha (a_ij - beta)(X^j - X^i) over tau (the update
// formula of PAPER.md:1258-1264): y = ((x_i + x_j) +- (x_i - x_j) e) / 2,
// e = exp(-2 alpha (a_ij - beta) tau) evaluated in fp64
template <typename T, int D>
__device__ __forceinline__ void adj_flow(const DevParams& P, uint32_t i, uint32_t j, const T (&xi)[D],
                                         const T (&xj)[D], bool first, T (&y)[D]) {
  const T e = (T)exp(-2.0 * P.kp0 * (adj_value(P, i, j) - P.kp1) * P.dt);
#pragma unroll
  for (int c = 0; c < D; ++c) {
    const T Dv = xi[c] - xj[c], sum = xi[c] + xj[c];
    y[c] = T(0.5) * (first ? sum + Dv * e : sum - Dv * e);
  }
}
// edge-restricted pick: edge e = floor(nnz U64 / 2^64), its row and
// column; redrawn on a diagonal entry
__device__ __forceinline__ void adj_edge_draw(const DevParams& P, uint64_t s0, uint32_t m, uint32_t& i, uint32_t& j) {
  for (uint32_t t = 0;; ++t) {
    const uint4 w = block_at(P, (uint32_t)s0, t, m, TAG_SLOT);
    const uint64_t e = __umul64hi(P.adj_nnz, (((uint64_t)w.x) << 32) | w.y);
    uint32_t lo = 0, hi = (uint32_t)P.n;
    while (hi - lo > 1) {
      const uint32_t mid = lo + (hi - lo) / 2;
      if (P.adj_rp[mid] <= e) lo = mid; else hi = mid;
    }
    i = lo;
    j = P.adj_ci[e];
    if (i != j) return;
  }
}

template <typename T, int D>
__device__ __forceinline__ void check_finite(const T (&x)[D], const DevParams& P, uint32_t id,
                                             uint32_t m) {
  bool ok = true;
#pragma unroll
  for (int c = 0; c < D; ++c) ok = ok && isfinite(x[c]);
  if (!ok) atomicMin(P.nonfinite, ((unsigned long long)m << 32) | id);
}

}  // namespace rbm

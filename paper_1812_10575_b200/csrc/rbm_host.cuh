#pragma once
// rbm_host.cuh -- host-side engine shared by rbm_api.cu and the per-dtype
// instantiation units rbm_engines_f32.cu / rbm_engines_f64.cu.
//
// Host orchestration only: validation, bucket-layout choice, workspace
// carving, per-config kernel dispatch, CUDA-graph capture/replay of steps.
// Every arithmetic step of the RBM path runs in the kernels of
// rbm_kernels.cuh; there is no CPU fallback.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/rbm.h"
#include "rbm_kernels.cuh"
#include "rbm_nccl.cuh"

using namespace rbm;

namespace rbmhost {

extern thread_local std::string g_err;  // failures without a context

// NVTX range around a host-side sub-step (seen by Nsight Systems / ncu --nvtx;
// a no-op unless a tool is attached)
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
};

struct Workspace {
  unsigned char* base = nullptr;
  size_t size = 0, used = 0;
  bool dry = false;  // offsets only: base is a sentinel address, never dereferenced
  template <typename U>
  U* take(size_t count) {
    used = (used + 255) & ~size_t(255);
    U* p = reinterpret_cast<U*>(base ? base + used : nullptr);
    used += count * sizeof(U) + 64;  // slack: TMA windows may read 16 B past the end
    return p;
  }
};

struct Layout {
  uint32_t g = 0;        // log2 world_size (partitioned single system; 0 on one GPU)
  uint32_t B = 0, b1 = 0, b2 = 0, nbuckets = 1, cap = 0;  // nbuckets: final buckets of this rank
  uint32_t SB = 8, idbits = 1, lowbits = 0;
  uint32_t segk = 0;     // log2 segments per pass-1 bucket (2-pass layouts)
  uint32_t cap1 = 0;     // gapped capacity of a pass-1 segment (2-pass layouts; per source rank when partitioned)
  uint32_t nseg() const { return (1u << b1) << segk; }
  uint32_t cap2 = 0;     // gapped capacity of a final bucket
  uint64_t slots = 0;    // elements per state buffer: max(N, 2^b1 cap1, 2^B cap2)
};
#ifndef RBM_FUSED_CAP_MAX  // design-experiment builds override this (build.py -D...)
#define RBM_FUSED_CAP_MAX 4096
#endif
constexpr uint32_t FUSED_CAP_MAX = RBM_FUSED_CAP_MAX;  // largest per-bucket smem capacity (u16 indices)

// bytes of one state record and whether it carries the shuffle key (RecL)
inline uint32_t rec_bytes(const rbm_config& c) {
  const uint32_t xb = c.d * (c.dtype == RBM_F64 ? 8u : 4u);
  return (4 + xb <= 8) ? 8u : ((4 + xb <= 16) ? 16u : ((c.dtype == RBM_F64 && 8 + xb <= 24) ? 24u : 32u));
}
inline bool rec_keyed(const rbm_config& c) {
  return 8 + c.d * (c.dtype == RBM_F64 ? 8u : 4u) <= rec_bytes(c);
}

struct EngineBase;

}  // namespace rbmhost
using namespace rbmhost;

struct rbm_ctx {
  rbm_config cfg{};
  Layout L;
  DevParams P{};
  cudaStream_t stream = nullptr;       // caller's stream
  cudaStream_t cap_stream = nullptr;   // private, for graph capture
  int device = 0;
  std::unique_ptr<EngineBase> eng;
  // workspace carve
  unsigned char* recbuf[3] = {nullptr, nullptr, nullptr};  // state records (RS bytes each)
  uint32_t* skey[3] = {nullptr, nullptr, nullptr};         // side keys (unkeyed records, 2-pass layouts)
  uint64_t xstride = 0;  // record slots per state buffer (multiple of 64)
  // partitioned single system (world_size > 1): buffer 0 = this rank's final
  // buckets A (bucket -1 = halo), 1 = send pass-1 buckets B, 2 = received C
  uint64_t id0 = 0, n0 = 0;  // initial id range of this rank
  unsigned char* ws_base = nullptr;            // this rank's workspace (device)
  bool fused = false;                          // G9: outputs stored into the peers' receive buffers
  unsigned char* peer_base[MAXG_FUSED] = {};   // every rank's workspace base (peer-mapped)
  uint32_t *counts_send = nullptr, *counts_all = nullptr;
  ncclComm_t comm = nullptr;                   // library-owned communicator (id given to rbm_init)
  void* ipc_open[MAXG_FUSED] = {};             // peer allocations opened by rbm_part_map_peers
  unsigned char* xchg = nullptr;               // device scratch: IPC handles, local-gather offsets
  unsigned char *halo_send = nullptr, *halo_recv = nullptr;
  // gapped-bucket pipeline.  cur1[q]: counts (cursors) of the buckets the
  // state of step m (q = m & 1) is partitioned into -- pass-1 buckets (2-pass)
  // or final buckets (1-pass); the fused step fills cur1[q ^ 1] for step m+1.
  uint32_t *cur1[2] = {nullptr, nullptr};
  uint32_t *prefix1 = nullptr, *tile_off = nullptr, *S = nullptr, *cur2 = nullptr;
  uint32_t* big_claim = nullptr;
  bool partitioned = false;  // state stored in the gapped buckets of step `step`
  uint64_t* step_dev = nullptr;
  unsigned long long* nonfinite = nullptr;
  uint32_t* capacity_err = nullptr;
  unsigned char* big_scratch = nullptr;
  // RBM-r
  uint32_t *js = nullptr, *rmcnt = nullptr, *rmbox = nullptr, *rovf = nullptr, *rnovf = nullptr;
  void* rxa = nullptr;     // AoS state (4 scalars per particle, id order)
  unsigned char* rinc[2] = {nullptr, nullptr};  // RBM-r increment records: pass-1 and final buckets
  uint32_t *rexpect = nullptr, *rticket = nullptr;  // sequential RBM-r': per-slot expected tags, ticket
  bool aos_valid = false;  // RBM-r state currently in rxa
  // RBM-r on a partitioned system (row e2): exchange regions and own batches
  RPart rp{};
  bool verlet_start = false;  // the next step starts a Verlet run from (x_0, v_0)
  uint64_t nbatch = 0, nslots = 0;
  // state
  int cur = 0;
  uint64_t step = 0;
  uint32_t launches = 0;
  int tile = 4096;
  cudaGraphExec_t graph[6] = {};  // by (cur, m & 1)
  uint32_t graph_steps = 1;
  bool graph_failed = false;  // stream capture refused (partitioned steps fall back to eager launches)
  // optional per-kernel CUDA-event timing (rbm_timing_begin/end)
  bool timing = false;
  std::vector<cudaEvent_t> ev;
  size_t ev_used = 0;
  std::string err;
  int debug_sync = -1;  // RBM_DEBUG_SYNC: synchronise and check after every sub-step (debugging)
  void mark(cudaStream_t s) {
    if (timing && ev_used < ev.size()) cudaEventRecord(ev[ev_used++], s);
    if (debug_sync < 0) debug_sync = std::getenv("RBM_DEBUG_SYNC") ? 1 : 0;
    if (debug_sync) {
      const cudaError_t e = cudaStreamSynchronize(s);
      std::fprintf(stderr, "[rbm debug] mark %u: %s\n", ev_dbg++, cudaGetErrorString(e));
    }
  }
  unsigned ev_dbg = 0;
};

namespace rbmhost {

inline rbm_status fail(rbm_ctx* c, rbm_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf; else g_err = buf;
  return s;
}

#define CU(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess)                                                            \
      return fail(c, RBM_ERR_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                \
  } while (0)

inline uint32_t ceil_log2(double v) {
  uint32_t b = 0;
  while ((double)(1ull << b) < v) ++b;
  return b;
}

inline size_t elt_size(const rbm_config& c) { return c.dtype == RBM_F64 ? 8 : 4; }

inline bool is_partitioned(const rbm_config& c) { return c.world_size > 1; }

// this rank's initial id range [id0, id0 + n0) (partitioned: floor(N r / G) ..)
inline void initial_ids(const rbm_config& c, uint64_t& id0, uint64_t& n0) {
  if (!is_partitioned(c)) { id0 = 0; n0 = c.n; return; }
  const uint64_t G = (uint64_t)c.world_size, r = (uint64_t)c.rank;
  id0 = c.n * r / G;
  n0 = c.n * (r + 1) / G - id0;
}

inline Layout choose_layout(const rbm_config& c) {
  Layout L;
  const uint64_t n = c.n;
  const bool part = is_partitioned(c);
  L.idbits = ceil_log2((double)n);
  if (L.idbits < 1) L.idbits = 1;
  // gapped capacities: mean + 12 sigma + 64 (overflow probability ~1e-33 per
  // bucket; an overflow is flagged as RBM_ERR_CAPACITY), multiples of 64 so
  // every bucket starts 256-B aligned (TMA)
  auto gcap = [](double mu, uint32_t floor_) {
    uint64_t v = (uint64_t)(mu + 12.0 * std::sqrt(mu) + 64.0);
    if (v < floor_) v = floor_;
    return (uint32_t)((v + 63) & ~63ull);
  };
  if ((c.scheme == RBM_SCHEME_RBMR || c.scheme == RBM_SCHEME_RBMR_SEQ) && !part) {
    // RBM-r increments (RBM-r' link records) partitioned by particle index: final buckets of
    // W = 2^(idbits-B) ids (~1024), one or two passes as for RBM-1
    double w = 1024.0;  // ids per final bucket (experiment knob RBM_RBMR_W)
    if (const char* e = std::getenv("RBM_RBMR_W")) w = std::atof(e);
    if (!(w >= 128.0 && w <= 1024.0)) w = 1024.0;
    uint32_t B = ceil_log2((double)n / w);
    if (B > L.idbits) B = L.idbits;
    if (B > 20) B = 20;
    L.B = B;
    if (B <= 10) { L.b1 = B; L.b2 = 0; } else { L.b1 = B / 2; L.b2 = B - L.b1; }
    L.nbuckets = 1u << B;
    const double W = (double)(1ull << (L.idbits - B));
    const double nslots = (double)(((n + c.p - 1) / c.p) * c.p);
    L.cap2 = gcap(nslots * W / (double)n, 64);
    L.cap1 = L.b2 ? gcap(nslots * W * (double)(1u << L.b2) / (double)n, 64) : L.cap2;
    L.cap = L.cap2;
    L.slots = std::max<uint64_t>((uint64_t)(1u << L.b1) * L.cap1, (uint64_t)L.nbuckets * L.cap2);
    return L;
  }
  if (part) L.g = ceil_log2((double)c.world_size);
  if (n <= 2048 && !part) {
    L.B = 0;  // one bucket: sorted-output kernel
  } else {
    // target mean bucket size (tuning knob RBM_BUCKET_TARGET, default 2048)
    double target = 2048.0;
    if (const char* e = std::getenv("RBM_BUCKET_TARGET")) target = std::atof(e);
    if (!(target >= 64.0 && target <= (double)(FUSED_CAP_MAX / 2))) target = 2048.0;
    L.B = ceil_log2((double)n / target);
    if (L.B < 2) L.B = 2;
    if (part && L.B < L.g + 2) L.B = L.g + 2;  // >= 4 final buckets per rank, two passes
    if (L.B > 20u) L.B = 20u;  // 2^10 x 2^10 digits; mean bucket 2048 up to N = 2^31
  }
  if (L.B <= 10 && !part) { L.b1 = L.B; L.b2 = 0; }
  else {
    L.b1 = L.B / 2;  // fused-output digit <= pass-2 digit: longer runs in the fused scatter
    if (const char* e = std::getenv("RBM_B1")) {  // tuning knob: pass-1 / fused-output digit bits
      const int v = std::atoi(e);
      if (v >= 5 && v <= 10 && L.B - v >= 5 && L.B - v <= 10) L.b1 = (uint32_t)v;
    }
    if (part && L.b1 < L.g) L.b1 = L.g;  // the pass-1 digit carries the destination rank
    if (L.b1 < 2) L.b1 = 2;              // >= 4 output digits (uint4 scans)
    if (L.b1 > 10) L.b1 = 10;
    L.b2 = L.B - L.b1;
    // one cursor per pass-1 digit: splitting each digit into 2^segk salted
    // segments (to spread the reservation atomics) measured no faster at C5,
    // and a salt fixed per CTA overfills segments when few CTAs produce
    // (prologue at small N), so segk stays 0 (the kernels take any segk)
    L.segk = 0;
  }
  L.nbuckets = 1u << (L.B - L.g);
  L.SB = L.idbits > L.B + 8 ? L.idbits - L.B : 8;  // 32-bit composites: lowbits + idbits <= 32
  L.lowbits = 32 - L.B - L.SB;
  if (L.B == 0) {
    L.cap = (uint32_t)((n + 31) & ~31ull);
  } else {
    const double mu = (double)n / L.nbuckets;
    L.cap = (uint32_t)(mu + 6.0 * std::sqrt(mu) + 32.0);
    L.cap = (L.cap + 15) & ~15u;  // C5: 2352 records, so four bucket CTAs fit an SM
    if (L.cap > FUSED_CAP_MAX) L.cap = FUSED_CAP_MAX;
  }
  if (c.debug_bucket_cap) L.cap = c.debug_bucket_cap;
  L.slots = n;
  if (part) {
    // three buffers (final buckets A with a leading halo bucket, send B,
    // receive C); pass-1 segments hold one source rank's share
    // the largest initial share, so every rank has the same workspace layout
    // (fused mode addresses the peers' buffers with this rank's offsets)
    const uint64_t n0 = (n + (uint64_t)c.world_size - 1) / (uint64_t)c.world_size;
    L.cap2 = gcap((double)n / (1u << L.B), L.cap + 64);
    L.cap1 = gcap((double)n / ((double)c.world_size * L.nseg()), 64);
    L.slots = std::max<uint64_t>(n0, (uint64_t)(L.nbuckets + 1) * L.cap2);
    L.slots = std::max<uint64_t>(L.slots, (uint64_t)L.nseg() * L.cap1);
  } else if (L.B > 0) {
    L.cap2 = gcap((double)n / L.nbuckets, L.cap + 64);
    L.slots = std::max<uint64_t>(L.slots, (uint64_t)L.nbuckets * L.cap2);
    if (L.b2) {
      L.cap1 = gcap((double)n / L.nseg(), 64);
      L.slots = std::max<uint64_t>(L.slots, (uint64_t)L.nseg() * L.cap1);
    }
  }
  return L;
}

// shared memory of the bucket kernel (bucket_smem_bytes in rbm_kernels.cuh)
inline size_t bucket_smem(const rbm_config& c, const Layout& L) {
  return ((size_t)bucket_ncw(L.SB, L.b1) + (1u << L.b1) + 64) * 4 + 16 + (size_t)(L.cap + 8) * rec_bytes(c) +
         (size_t)(L.cap + 8) * 4 + (((size_t)L.cap * 2 + 15) & ~(size_t)15);
}

inline rbm_status validate(const rbm_config* cfg) {
  rbm_ctx* c = nullptr;
  if (!cfg) return fail(c, RBM_ERR_INVALID_ARG, "cfg is NULL");
  const rbm_config& k = *cfg;
  if (k.abi_version != RBM_ABI_VERSION)
    return fail(c, RBM_ERR_INVALID_ARG, "abi_version %u != %u", k.abi_version, RBM_ABI_VERSION);
  if (k.dtype > RBM_F64) return fail(c, RBM_ERR_INVALID_ARG, "dtype %u", k.dtype);
  if (k.d < 1 || k.d > 3) return fail(c, RBM_ERR_INVALID_ARG, "d=%u not in 1..3", k.d);
  if (k.n < 2 || k.n > (1ull << 31)) return fail(c, RBM_ERR_INVALID_ARG, "n=%llu not in 2..2^31", (unsigned long long)k.n);
  if (k.p < 2 || k.p > k.n) return fail(c, RBM_ERR_INVALID_ARG, "p=%u must satisfy 2 <= p <= n", k.p);
  if (k.p > 64 && !(k.p == k.n && k.n <= 2048))
    return fail(c, RBM_ERR_INVALID_ARG, "p=%u: need p <= 64, or p == n <= 2048", k.p);
  if (k.scheme > RBM_SCHEME_RBMR_SEQ) return fail(c, RBM_ERR_INVALID_ARG, "scheme %u", k.scheme);
  if (k.integrator > RBM_INTEG_VERLET) return fail(c, RBM_ERR_INVALID_ARG, "integrator %u", k.integrator);
  if (k.integrator == RBM_INTEG_VERLET) {
    if (k.d != 2) return fail(c, RBM_ERR_INVALID_ARG, "Verlet: d must be 2 (x and v / x_prev of a 1-D particle)");
    if (k.sigma != 0.0) return fail(c, RBM_ERR_INVALID_ARG, "Verlet: the Hamiltonian system has no noise (sigma = 0)");
    if (k.kernel != RBM_K_SMOOTH_TEST && k.kernel != RBM_K_ZERO)
      return fail(c, RBM_ERR_UNSUPPORTED, "Verlet: kernel smooth or zero in this build");
    if (k.scheme != RBM_SCHEME_RBM1 || k.constraint != RBM_CONSTRAINT_NONE)
      return fail(c, RBM_ERR_UNSUPPORTED, "Verlet: RBM-1 without constraint");
    if (k.state_form > 1) return fail(c, RBM_ERR_INVALID_ARG, "state_form %u", k.state_form);
  }
  if (k.kernel > RBM_K_ADJACENCY) return fail(c, RBM_ERR_UNKNOWN_KERNEL, "kernel %u not in registry", k.kernel);
  if (k.kernel == RBM_K_ADJACENCY) {
    if (k.scheme == RBM_SCHEME_RBM1 || k.p != 2 || k.integrator != RBM_INTEG_SPLIT_EXACT_PAIR || k.world_size != 1)
      return fail(c, RBM_ERR_UNSUPPORTED, "adjacency (clustering) kernel: RBM-r or RBM-r', p = 2, split integrator, one GPU");
    if (!std::isfinite(k.kparam[0]) || !std::isfinite(k.kparam[1]))
      return fail(c, RBM_ERR_INVALID_ARG, "adjacency kernel needs finite kparam = {alpha, beta}");
  }
  if (k.noise > RBM_NOISE_GEOMETRIC) return fail(c, RBM_ERR_INVALID_ARG, "noise %u", k.noise);
  if (k.potential > RBM_V_HARMONIC) return fail(c, RBM_ERR_UNKNOWN_KERNEL, "potential %u not in registry", k.potential);
  if (k.constraint > RBM_CONSTRAINT_UNIT_SPHERE) return fail(c, RBM_ERR_INVALID_ARG, "constraint %u", k.constraint);
  if (k.kernel == RBM_K_DYSON && k.d != 1) return fail(c, RBM_ERR_INVALID_ARG, "Dyson kernel needs d=1");
  if (k.kernel == RBM_K_COULOMB && k.d != 3) return fail(c, RBM_ERR_INVALID_ARG, "Coulomb kernel needs d=3");
  if (k.constraint == RBM_CONSTRAINT_UNIT_SPHERE && k.d != 3) return fail(c, RBM_ERR_INVALID_ARG, "sphere constraint needs d=3");
  if (k.integrator == RBM_INTEG_SPLIT_EXACT_PAIR) {
    if (k.p != 2) return fail(c, RBM_ERR_INVALID_ARG, "split integrator needs p=2");
    if (k.kernel != RBM_K_DYSON && k.kernel != RBM_K_COULOMB && !(k.kernel == RBM_K_LINEAR && k.d == 1) &&
        k.kernel != RBM_K_ADJACENCY)
      return fail(c, RBM_ERR_INVALID_ARG, "split integrator needs the Dyson, Coulomb, (d=1) linear or adjacency kernel");
    if (k.scheme == RBM_SCHEME_RBM1 && (k.n % 2))
      return fail(c, RBM_ERR_INVALID_ARG, "split integrator with RBM-1 needs even n");
  }
  if (!(k.sigma >= 0.0) || !std::isfinite(k.sigma)) return fail(c, RBM_ERR_INVALID_ARG, "sigma must be finite and >= 0");
  if (!(k.dt > 0.0) || !std::isfinite(k.dt)) return fail(c, RBM_ERR_INVALID_ARG, "dt must be finite and > 0");
  if (k.kernel == RBM_K_COULOMB_REG && !(k.kparam[0] > 0.0)) return fail(c, RBM_ERR_INVALID_ARG, "coulomb_reg needs kparam[0]=eps > 0");
  if (k.kernel == RBM_K_BOUNDED_CONFIDENCE && !(k.kparam[1] > 0.0)) return fail(c, RBM_ERR_INVALID_ARG, "bounded confidence needs kparam[1]=radius > 0");
  if (k.init > RBM_INIT_ABS_NORMAL) return fail(c, RBM_ERR_INVALID_ARG, "init %u", k.init);
  if (k.init == RBM_INIT_UNIFORM_SPHERE && k.d != 3) return fail(c, RBM_ERR_INVALID_ARG, "sphere init needs d=3");
  if (k.init == RBM_INIT_GAUSS_MIXTURE && !(k.iparam[0] >= 1 && k.iparam[0] <= 64))
    return fail(c, RBM_ERR_INVALID_ARG, "mixture needs 1 <= K <= 64");
  if (k.replica >= (1u << 24)) return fail(c, RBM_ERR_INVALID_ARG, "replica must be < 2^24");
  if (k.step0 + 1 >= (1ull << 32)) return fail(c, RBM_ERR_INVALID_ARG, "step0 must be < 2^32-1");
  if (k.world_size < 1 || k.world_size > 64 || (k.world_size & (k.world_size - 1)))
    return fail(c, RBM_ERR_INVALID_ARG, "world_size=%d must be a power of two in 1..64", k.world_size);
  if (k.rank < 0 || k.rank >= k.world_size)
    return fail(c, RBM_ERR_INVALID_ARG, "rank=%d not in [0, world_size=%d)", k.rank, k.world_size);
  if (is_partitioned(k)) {
    if (k.scheme == RBM_SCHEME_RBMR_SEQ)
      return fail(c, RBM_ERR_UNSUPPORTED, "partitioned single system: RBM-1 and RBM-r (the sequential RBM-r' is one GPU only)");
    if (k.scheme == RBM_SCHEME_RBMR && k.integrator == RBM_INTEG_VERLET)
      return fail(c, RBM_ERR_UNSUPPORTED, "partitioned RBM-r: Euler-Maruyama or split");
    if (k.p > HALO_MAX)
      return fail(c, RBM_ERR_INVALID_ARG, "partitioned single system needs p <= %u", HALO_MAX);
    if (k.n / (uint64_t)k.world_size < 1024 || k.n / (uint64_t)k.world_size < 16ull * k.p)
      return fail(c, RBM_ERR_INVALID_ARG, "partitioned single system needs n/world_size >= max(1024, 16 p)");
  }
  const Layout L = choose_layout(k);
  if (k.scheme == RBM_SCHEME_RBM1 && L.B > 0 && L.SB > 12)
    return fail(c, RBM_ERR_UNSUPPORTED, "n=%llu needs %u sub-digit bits (> 12): n <= 2^30 per GPU", (unsigned long long)k.n, L.SB);
  if (k.scheme == RBM_SCHEME_RBM1 && L.B > 0 && L.cap > FUSED_CAP_MAX)
    return fail(c, RBM_ERR_INVALID_ARG, "debug_bucket_cap %u > %u", L.cap, FUSED_CAP_MAX);
  if (k.scheme == RBM_SCHEME_RBM1 && L.B == 0 &&
      (k.dtype == RBM_F64 ? resident_smem_bytes<double, 3>(L.cap) : resident_smem_bytes<float, 3>(L.cap)) > 227 * 1024)
    return fail(c, RBM_ERR_INVALID_ARG, "n=%llu too large for the resident kernel", (unsigned long long)k.n);
  if ((k.scheme == RBM_SCHEME_RBMR || k.scheme == RBM_SCHEME_RBMR_SEQ) && !is_partitioned(k) && L.cap2 > 2048)
    return fail(c, RBM_ERR_UNSUPPORTED, "RBM-r: %u slot records per id bucket exceed 2048", L.cap2);
  if (k.scheme == RBM_SCHEME_RBM1 && L.B > 0 && bucket_smem(k, L) > 227 * 1024)
    return fail(c, RBM_ERR_INVALID_ARG, "bucket capacity %u needs %zu B of shared memory", L.cap, bucket_smem(k, L));
  return RBM_OK;
}

// carve (or size, when ws.base == nullptr) the workspace
inline void carve(rbm_ctx& c, Workspace& ws) {
  const rbm_config& k = c.cfg;
  const size_t es = elt_size(k);
  const uint64_t n = k.n;
  const bool part = is_partitioned(k);
  const uint64_t slots = (k.scheme == RBM_SCHEME_RBM1) ? c.L.slots
                         : (part ? (n + (uint64_t)k.world_size - 1) / (uint64_t)k.world_size : n);
  const size_t RS = rec_bytes(k);
  const bool side = k.scheme == RBM_SCHEME_RBM1 && !rec_keyed(k) && c.L.b2 > 0;
  initial_ids(k, c.id0, c.n0);
  c.xstride = (slots + 63) & ~63ull;  // 256-B aligned buffers (TMA)
  // partitioned: buffer 0 = final buckets (pass 2 writes the side keys),
  // 1 = send, 2 = receive; one GPU: the state and the step's other buffer
  const int nbuf = (k.scheme == RBM_SCHEME_RBM1 && part) ? 3 : 2;
  for (int b = 0; b < nbuf; ++b) {
    c.recbuf[b] = ws.take<unsigned char>(c.xstride * RS);
    c.skey[b] = (side && (!part || b == 0)) ? ws.take<uint32_t>(c.xstride) : nullptr;
  }
  for (int q = 0; q < 2; ++q) c.cur1[q] = ws.take<uint32_t>((size_t)MAX_SEG * CUR1_STRIDE);
  c.prefix1 = ws.take<uint32_t>(1025);
  c.tile_off = ws.take<uint32_t>(1025);
  c.S = ws.take<uint32_t>((size_t)c.L.nbuckets + 2);
  if (c.S) c.S += 1;  // S[-1]: start of the halo bucket (partitioned)
  if (part) {
    c.counts_send = ws.take<uint32_t>(c.L.nseg());
    c.counts_all = ws.take<uint32_t>((size_t)k.world_size * c.L.nseg());
    c.halo_send = ws.take<unsigned char>(16 + (size_t)HALO_MAX * 32);
    c.halo_recv = ws.take<unsigned char>(16 + (size_t)HALO_MAX * 32);
    c.xchg = ws.take<unsigned char>(std::max<size_t>((size_t)MAXG_FUSED * 128, ((size_t)MAX_SEG_SPLIT + 2) * 4));
  }
  c.big_claim = ws.take<uint32_t>(NBIG);
  if (c.L.b2) c.cur2 = ws.take<uint32_t>((size_t)c.L.nbuckets * CUR2_STRIDE);
  c.step_dev = ws.take<uint64_t>(1);
  c.nonfinite = ws.take<unsigned long long>(1);
  c.capacity_err = ws.take<uint32_t>(1);
  c.big_scratch = ws.take<unsigned char>(NBIG * big_slot_bytes(RS));
  if (k.scheme != RBM_SCHEME_RBM1 && part) {
    // RBM-r partitioned: own ids [id0, id0+n0) and batches [bb0, bb1); chunk
    // capacity = mean requests per (source, destination) + 12 sigma + 64
    const uint64_t G = (uint64_t)k.world_size;
    c.nbatch = (n + k.p - 1) / k.p;
    c.nslots = c.nbatch * k.p;
    RPart& R = c.rp;
    R.G = (uint32_t)G;
    R.rank = (uint32_t)k.rank;
    R.n = n;
    R.id0 = c.id0;
    R.n0 = c.n0;
    R.bb0 = c.nbatch * (uint64_t)k.rank / G;
    R.bb1 = c.nbatch * (uint64_t)(k.rank + 1) / G;
    for (uint64_t q = 0; q <= G; ++q) R.idb[q] = n * q / G;
    const double mu = (double)((c.nbatch + G - 1) / G * k.p) * (double)((n + G - 1) / G) / (double)n;
    R.cap = (uint32_t)(((uint64_t)(mu + 12.0 * std::sqrt(mu) + 64.0) + 15) & ~15ull);
    R.qchunk = 16 + (uint64_t)R.cap * 4;
    R.pchunk = (uint64_t)R.cap * 4 * es;
    R.ioff = (uint64_t)R.cap * 4;
    R.ichunk = R.ioff + (uint64_t)R.cap * 4 * es;
    R.qs = ws.take<unsigned char>(G * R.qchunk);
    R.qr = ws.take<unsigned char>(G * R.qchunk);
    R.ps = ws.take<unsigned char>(G * R.pchunk);
    R.pr = ws.take<unsigned char>(G * R.pchunk);
    R.is = ws.take<unsigned char>(G * R.ichunk);
    R.ir = ws.take<unsigned char>(G * R.ichunk);
    R.qcnt = ws.take<uint32_t>(G);
    const uint64_t own = (R.bb1 - R.bb0) * k.p;
    R.spos = ws.take<uint32_t>(own);
    c.js = ws.take<uint32_t>(own);
    c.rxa = ws.take<unsigned char>(c.n0 * 4 * es);
    c.rmcnt = ws.take<uint32_t>(c.n0);
    c.rmbox = ws.take<uint32_t>(c.n0 * MBOX);
    c.rovf = ws.take<uint32_t>(2 * (size_t)OVF_CAP);
    c.rnovf = ws.take<uint32_t>(1);
  } else if (k.scheme != RBM_SCHEME_RBM1) {
    c.nbatch = (n + k.p - 1) / k.p;
    c.nslots = c.nbatch * k.p;
    {  // RBM-r increment records, or the 8-byte link records of RBM-r'
      const size_t irs = k.scheme == RBM_SCHEME_RBMR_SEQ ? 8 : ((8 + k.d * es) + 15) / 16 * 16;
      c.rinc[0] = ws.take<unsigned char>((size_t)(1u << c.L.b1) * c.L.cap1 * irs);
      if (c.L.b2) c.rinc[1] = ws.take<unsigned char>((size_t)c.L.nbuckets * c.L.cap2 * irs);
    }
    if (k.scheme == RBM_SCHEME_RBMR_SEQ) c.js = ws.take<uint32_t>(c.nslots);  // the Jacobi sweep keeps no draws
    c.rxa = ws.take<unsigned char>(n * 4 * es);
    if (k.scheme == RBM_SCHEME_RBMR_SEQ) {  // slot chains and flags of the sequential sweep
      c.rexpect = ws.take<uint32_t>(c.nslots);
      c.rticket = ws.take<uint32_t>(4);
    }
  }
  ws.used = (ws.used + 255) & ~size_t(255);
}

inline unsigned grid_for(uint64_t n, unsigned block, unsigned maxg = 148 * 16) {
  uint64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > maxg) g = maxg;
  return (unsigned)g;
}

struct EngineBase {
  virtual ~EngineBase() {}
  virtual rbm_status setup(rbm_ctx& c) = 0;
  virtual void init_state(rbm_ctx& c, cudaStream_t s) = 0;
  virtual void set_state(rbm_ctx& c, const void* x, cudaStream_t s) = 0;
  virtual void step(rbm_ctx& c, cudaStream_t s) = 0;
  virtual void gather(rbm_ctx& c, uint64_t i0, uint64_t i1, void* out, cudaStream_t s) = 0;
  // partitioned single system: the step split around its three exchanges
  virtual void run_resident(rbm_ctx& c, cudaStream_t s, uint32_t nsteps) = 0;
  // direct O(N^2) Euler-Maruyama steps on an id-ordered N x d array (f1)
  virtual void direct(const DevParams& P, void* x, void* tmp, uint32_t n, uint32_t m0,
                      uint32_t nsteps, cudaStream_t s) = 0;
  virtual void part_prologue(rbm_ctx& c, cudaStream_t s) = 0;
  virtual void part_phase1(rbm_ctx& c, cudaStream_t s) = 0;
  virtual void part_phase2(rbm_ctx& c, cudaStream_t s) = 0;
  // this rank's records, unordered (ids and positions, row-major); returns the count (syncs)
  virtual uint64_t gather_local(rbm_ctx& c, uint32_t* ids, void* x, cudaStream_t s) = 0;
  // RBM-r on a partitioned system: phase k = 1..4 of the step (exchange k-1 follows phase k)
  virtual void rbmr_part_phase(rbm_ctx& c, cudaStream_t s, int k) = 0;
  // the slot draws of step m of the one-GPU Jacobi sweep, recomputed (test hook)
  virtual void rbmr_slots(rbm_ctx& c, uint32_t m, uint32_t* out, cudaStream_t s) = 0;
};

template <typename T, int D, int KK, int INTEG>
struct Engine final : EngineBase {
  using RL = RecL<T, D>;
  static constexpr int PR_BLOCK = 256;
  // CTAs per SM the bucket kernel is register-budgeted for (1024 / 512 threads per SM)
  static constexpr int MINB = (((RL::RS <= 16) ? 4 : 2) * 256 / BUCKET_BLOCK) > 0 ? ((RL::RS <= 16) ? 4 : 2) * 256 / BUCKET_BLOCK : 1;
  size_t pr_smem = 0, sp_smem = 0, bk_smem = 0, rs_smem = 0;
  bool pair_mode = false;
  int bmode = MODE_GROUP;  // bucket kernel MODE: pair, runtime group, or a compile-time group size (fp32)
  int num_sms = 148;

  State<T, D> st(rbm_ctx& c, int b) { return State<T, D>{c.recbuf[b], c.skey[b]}; }

  template <bool LINK, class RT> rbm_status setup_rbmr(rbm_ctx& c) {
    const uint32_t W = 1u << (c.L.idbits - c.L.B);
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(rbmr_emit_kernel<T, D, KK, INTEG, LINK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  200 * 1024)) != cudaSuccess ||
        (e = cudaFuncSetAttribute(split_kernel<RT, SPLIT_BLOCK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)split_smem_bytes_rt<RT>())) != cudaSuccess ||
        (e = cudaFuncSetAttribute(rbmr_bucket_apply_kernel<T, D, LINK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)rapply_smem_bytes<T, D, LINK>(c.L.cap2, W))) != cudaSuccess)
      return fail(&c, RBM_ERR_CUDA, "smem attr rbmr: %s", cudaGetErrorString(e));
    return RBM_OK;
  }

  rbm_status setup(rbm_ctx& c) override {
    c.tile = split_tile<T, D>();
    pr_smem = prologue_smem_bytes<T, D, PR_BLOCK>();
    sp_smem = split_smem_bytes<T, D>();
    bk_smem = bucket_smem_bytes<T, D>(c.L.cap, c.L.SB, c.L.b1);
    if (const char* e = std::getenv("RBM_BUCKET_SMEM_MIN")) {  // experiment knob: fewer CTAs per SM
      const size_t v = (size_t)std::atoll(e);
      if (v > bk_smem && v <= 227 * 1024) bk_smem = v;
    }
    rs_smem = resident_smem_bytes<T, D>(c.L.cap);
    pair_mode = c.cfg.p == 2;
    {
      uint32_t g = 0;
      if (c.cfg.p <= 32) { g = 1; while (g < c.cfg.p) g <<= 1; }
      bmode = pair_mode ? MODE_PAIR : MODE_GROUP;
      if (std::is_same<T, float>::value && !pair_mode && (g == 4 || g == 8 || g == 32)) bmode = (int)g;
    }
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, c.device);
    if (num_sms <= 0) num_sms = 148;
    auto chk = [&](cudaError_t e, const char* what) -> rbm_status {
      if (e != cudaSuccess) return fail(&c, RBM_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
      return RBM_OK;
    };
    rbm_status s;
    if ((s = chk(cudaFuncSetAttribute(prologue_kernel<T, D, PR_BLOCK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)pr_smem), "smem attr prologue"))) return s;
    if ((s = chk(cudaFuncSetAttribute(split_kernel<StateRT<T, D>, SPLIT_BLOCK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)sp_smem), "smem attr split"))) return s;
    if (c.cfg.scheme == RBM_SCHEME_RBMR && !is_partitioned(c.cfg)) return setup_rbmr<false, IncRT<T, D>>(c);
    if (c.cfg.scheme == RBM_SCHEME_RBMR_SEQ) return setup_rbmr<true, LinkRT>(c);
    if (c.L.B > 0) {
      if ((s = chk(bucket_attr(), "smem attr bucket"))) return s;
    } else if (rs_smem <= 227 * 1024) {
      if ((s = chk(cudaFuncSetAttribute(resident_kernel<T, D, KK, INTEG, 256>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rs_smem),
                   "smem attr resident"))) return s;
    }
    return RBM_OK;
  }

  // partitioned: this rank's final buckets, shifted so that bucket -1 (the
  // halo) sits at physical slots [-cap2, 0)
  State<T, D> stA(rbm_ctx& c) {
    State<T, D> a = st(c, 0);
    a.rec += (size_t)c.L.cap2 * RL::RS;
    if (a.key) a.key += c.L.cap2;
    return a;
  }

  static OutDst<T, D> od(State<T, D> d) {
    OutDst<T, D> o{};
    o.st[0] = d;
    o.fused = 0;
    return o;
  }
  // buffer b of rank j's workspace (same layout on every rank)
  State<T, D> st_peer(rbm_ctx& c, int b, uint32_t j) {
    State<T, D> a = st(c, b);
    const ptrdiff_t sh = c.peer_base[j] - c.ws_base;
    a.rec += sh;
    if (a.key) a.key = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(a.key) + sh);
    return a;
  }
  // partitioned: receive buffer holding the data of step m (fused: double-buffered)
  static int recv_buf(const rbm_ctx& c, uint64_t m) { return c.fused ? ((m & 1) ? 1 : 2) : 2; }
  // partitioned: where a step writes the records of step m
  OutDst<T, D> part_dst(rbm_ctx& c, uint64_t m) {
    if (!c.fused) return od(st(c, 1));
    OutDst<T, D> o{};
    const uint32_t G = (uint32_t)c.cfg.world_size;
    for (uint32_t j = 0; j < G; ++j) o.st[j] = st_peer(c, recv_buf(c, m), j);
    o.fused = 1;
    o.nls_log = 0;
    while ((1u << o.nls_log) < c.L.nseg() / G) ++o.nls_log;
    o.rank = (uint32_t)c.cfg.rank;
    return o;
  }

  void init_state(rbm_ctx& c, cudaStream_t s) override {
    const rbm_config& k = c.cfg;
    init_kernel<T, D><<<grid_for(c.n0, 256), 256, 0, s>>>(c.P, st(c, c.cur), c.id0, c.n0, k.init,
                                                          k.iparam[0], k.iparam[1], k.iparam[2],
                                                          k.iparam[3]);
    c.partitioned = false;
    c.aos_valid = false;
    c.verlet_start = k.integrator == RBM_INTEG_VERLET && k.state_form == 0;
  }

  void set_state(rbm_ctx& c, const void* x, cudaStream_t s) override {
    set_state_kernel<T, D><<<grid_for(c.n0, 256), 256, 0, s>>>(c.id0, c.n0, st(c, c.cur),
                                                               reinterpret_cast<const T*>(x));
    c.partitioned = false;
    c.aos_valid = false;
    c.verlet_start = c.cfg.integrator == RBM_INTEG_VERLET && c.cfg.state_form == 0;
  }

  void gather(rbm_ctx& c, uint64_t i0, uint64_t i1, void* out, cudaStream_t s) override {
    if (is_partitioned(c.cfg) && c.cfg.scheme == RBM_SCHEME_RBMR && c.aos_valid) {
      gather_aos_part_kernel<T, D><<<grid_for(c.n0, 256), 256, 0, s>>>(
          reinterpret_cast<const T*>(c.rxa), c.id0, c.n0, i0, i1, reinterpret_cast<T*>(out), nullptr);
      return;
    }
    if (is_partitioned(c.cfg)) {
      if (c.partitioned) {
        gather_part_kernel<T, D><<<grid_for((uint64_t)c.L.nseg() * c.L.cap1, 256), 256, 0, s>>>(
            c.P, st(c, recv_buf(c, c.step)), c.L.cap1, c.counts_all, (uint32_t)c.cfg.world_size, (uint32_t)c.cfg.rank,
            i0, i1, reinterpret_cast<T*>(out));
      } else {
        gather_kernel<T, D><<<grid_for(c.n0, 256), 256, 0, s>>>(c.n0, st(c, 0), i0, i1,
                                                                reinterpret_cast<T*>(out));
      }
      return;
    }
    if (c.cfg.scheme != RBM_SCHEME_RBM1 && c.aos_valid) {
      if (i1 > i0)
        gather_aos_kernel<T, D><<<grid_for(i1 - i0, 256), 256, 0, s>>>(reinterpret_cast<const T*>(c.rxa), i0,
                                                                     i1, reinterpret_cast<T*>(out));
      return;
    }
    if (c.cfg.scheme == RBM_SCHEME_RBM1 && c.L.B > 0 && c.partitioned) {
      Gapped g;
      g.cap = c.L.b2 ? c.L.cap1 : c.L.cap2;
      g.nb = c.L.nseg();
      g.cnt = c.cur1[c.step & 1];
      g.cstride = CUR1_STRIDE;
      gather_gapped_kernel<T, D><<<grid_for((uint64_t)g.nb * g.cap, 256), 256, 0, s>>>(
          g, st(c, c.cur), i0, i1, reinterpret_cast<T*>(out));
    } else {
      gather_kernel<T, D><<<grid_for(c.cfg.n, 256), 256, 0, s>>>(c.cfg.n, st(c, c.cur), i0, i1,
                                                                  reinterpret_cast<T*>(out));
    }
  }

  // pass 2: pass-1 buckets/segments (capacity cap1, counts cnt1 strided) -> final buckets
  void split2(rbm_ctx& c, cudaStream_t s, State<T, D> in, State<T, D> out, const uint32_t* cnt1) {
    Nvtx r_("split");
    split_kernel<StateRT<T, D>, SPLIT_BLOCK><<<(unsigned)num_sms * SPLIT_MINB, SPLIT_BLOCK, sp_smem, s>>>(
        c.P, in.rec, out.rec, out.key, c.cur2, c.L.cap2, cnt1, c.tile_off, c.L.cap1);
  }

  uint32_t tile2() const { return (uint32_t)split_tile<T, D>(); }

  void fused(rbm_ctx& c, cudaStream_t s, State<T, D> in, const OutDst<T, D>& out, uint32_t ocap,
             uint32_t* cur_next) {
    Nvtx r_("bucket_step");
    auto go = [&](auto mode) {
      bucket_kernel<T, D, KK, INTEG, decltype(mode)::value, MINB>
          <<<c.L.nbuckets, BUCKET_BLOCK, bk_smem, s>>>(c.P, in, c.L.cap2, c.S, out, ocap, cur_next);
    };
    if (bmode == MODE_PAIR) { go(std::integral_constant<int, MODE_PAIR>{}); return; }
    if constexpr (std::is_same<T, float>::value) {
      if (bmode == 4) { go(std::integral_constant<int, 4>{}); return; }
      if (bmode == 8) { go(std::integral_constant<int, 8>{}); return; }
      if (bmode == 32) { go(std::integral_constant<int, 32>{}); return; }
    }
    go(std::integral_constant<int, MODE_GROUP>{});
  }

  cudaError_t bucket_attr() {
    auto at = [&](auto mode) {
      return cudaFuncSetAttribute(bucket_kernel<T, D, KK, INTEG, decltype(mode)::value, MINB>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bk_smem);
    };
    if (bmode == MODE_PAIR) return at(std::integral_constant<int, MODE_PAIR>{});
    if constexpr (std::is_same<T, float>::value) {
      if (bmode == 4) return at(std::integral_constant<int, 4>{});
      if (bmode == 8) return at(std::integral_constant<int, 8>{});
      if (bmode == 32) return at(std::integral_constant<int, 32>{});
    }
    return at(std::integral_constant<int, MODE_GROUP>{});
  }

  void prologue(rbm_ctx& c, cudaStream_t s, State<T, D> src, const OutDst<T, D>& dst, uint32_t* cur,
                uint32_t dcap, uint64_t nsrc) {
    constexpr int TILE = prologue_tile<T, D>();
    prologue_kernel<T, D, PR_BLOCK><<<(unsigned)((nsrc + TILE - 1) / TILE), PR_BLOCK, pr_smem, s>>>(
        c.P, src, dst, cur, dcap, nsrc);
  }

  void step(rbm_ctx& c, cudaStream_t s) override {
    Nvtx range_("rbm_step");
    if (c.cfg.scheme == RBM_SCHEME_RBMR) { step_rbmr(c, s); return; }
    if (c.cfg.scheme == RBM_SCHEME_RBMR_SEQ) { step_rbmr_seq(c, s); return; }
    const DevParams& P = c.P;
    const Layout& L = c.L;
    const uint64_t n = c.cfg.n;
    const int q = (int)(c.step & 1);
    if (L.B == 0) {  // single bucket, system resident in shared memory
      run_resident(c, s, 1);
      return;
    }
    // capacity of the buckets the state of a step lives in (pass-1 or final)
    const uint32_t pcap = L.b2 ? L.cap1 : L.cap2;
    if (!c.partitioned) {  // prologue: any storage order -> gapped buckets of step m
      Nvtx r_("prologue");
      const int to = c.cur ^ 1;
      cudaMemsetAsync(c.cur1[q], 0, (size_t)L.nseg() * CUR1_STRIDE * 4, s);
      prologue(c, s, st(c, c.cur), od(st(c, to)), c.cur1[q], pcap, n);
      c.cur = to;
      c.partitioned = true;
    }
    cudaMemsetAsync(c.cur1[q ^ 1], 0, (size_t)L.nseg() * CUR1_STRIDE * 4, s);  // step-(m+1) cursors
    const unsigned straddle_grid = (unsigned)(((uint64_t)L.nbuckets * 32 + 255) / 256);
    c.mark(s);
    tile_scan_kernel<<<1, 1024, 0, s>>>(P, c.cur1[q], c.prefix1, c.tile_off, c.S, tile2());
    if (L.b2 == 0) {
      // A holds the final buckets of step m; the fused step writes m+1's into B
      State<T, D> A = st(c, c.cur), Bf = st(c, c.cur ^ 1);
      c.mark(s);
      fused(c, s, A, od(Bf), L.cap2, c.cur1[q ^ 1]);
      c.mark(s);
      straddle_kernel<T, D, KK, INTEG><<<straddle_grid, 256, 0, s>>>(P, A, L.cap2, c.S, od(Bf), L.cap2,
                                                                     c.cur1[q ^ 1]);
      c.cur ^= 1;
    } else {
      // A holds the pass-1 buckets of step m: split them by the next b2 bits
      // into B, then the bucket step writes m+1's pass-1 buckets back into A
      State<T, D> A = st(c, c.cur), Bf = st(c, c.cur ^ 1);
      cudaMemsetAsync(c.cur2, 0, (size_t)L.nbuckets * CUR2_STRIDE * 4, s);
      c.mark(s);
      split2(c, s, A, Bf, c.cur1[q]);
      c.mark(s);
      final_scan_kernel<<<1u << L.b1, 512, 0, s>>>(P, c.cur2, c.prefix1, c.S);
      c.mark(s);
      fused(c, s, Bf, od(A), L.cap1, c.cur1[q ^ 1]);
      c.mark(s);
      straddle_kernel<T, D, KK, INTEG><<<straddle_grid, 256, 0, s>>>(P, Bf, L.cap2, c.S, od(A), L.cap1,
                                                                     c.cur1[q ^ 1]);
    }
    c.mark(s);
    advance_kernel<<<1, 1, 0, s>>>(c.step_dev);
    c.mark(s);
  }

  void direct(const DevParams& P, void* x, void* tmp, uint32_t n, uint32_t m0, uint32_t nsteps,
              cudaStream_t s) override {
    constexpr int TB = 128;
    T* a = reinterpret_cast<T*>(x);
    T* b = reinterpret_cast<T*>(tmp);
    DevParams Q = P;
    for (uint32_t k = 0; k < nsteps; ++k) {
      Q.verlet_start = (k == 0) ? P.verlet_start : 0u;
      direct_kernel<T, D, KK, (INTEG == 2 ? 2 : 0), TB><<<(n + TB - 1) / TB, TB, 0, s>>>(Q, a, b, n, m0 + k);
      std::swap(a, b);
    }
    if (nsteps & 1u) cudaMemcpyAsync(x, tmp, (size_t)n * D * sizeof(T), cudaMemcpyDeviceToDevice, s);
  }

  // N <= 2048: nsteps steps in one launch of one CTA (state in smem)
  void run_resident(rbm_ctx& c, cudaStream_t s, uint32_t nsteps) override {
    c.mark(s);
    resident_kernel<T, D, KK, INTEG, 256><<<1, 256, rs_smem, s>>>(c.P, st(c, c.cur), st(c, c.cur ^ 1), nsteps,
                                                                  c.step_dev);
    c.cur ^= 1;
    c.mark(s);
  }

  // ---------------------------------------- partitioned single system (a7)
  // Buffers: A = stA (this rank's final buckets + halo bucket), B = st(c, 1)
  // (send: 2^b1 pass-1 buckets by the top b1 bits of the key, capacity cap1,
  // destination rank = top g bits), C = st(c, 2) (received: 2^b1 segments
  // v = source * 2^b1/G + local pass-1 bucket).  cur1[0] = send cursors,
  // cur1[1] = received segment counts (strided, for the tile table).
  // Exchanges between the phases:
  //   prologue / phase2 -> all-gather counts_send into counts_all, and
  //                        all-to-all of B's records into C (equal chunks)
  //   phase1            -> halo_send of rank r to halo_recv of rank r+1
  void part_prologue(rbm_ctx& c, cudaStream_t s) override {
    Nvtx range_("rbm_part_prologue");
    cudaMemsetAsync(c.cur1[0], 0, (size_t)c.L.nseg() * CUR1_STRIDE * 4, s);
    prologue(c, s, st(c, 0), part_dst(c, c.step), c.cur1[0], c.L.cap1, c.n0);
    pack_counts_kernel<<<1, 1024, 0, s>>>(c.cur1[0], c.L.nseg(), c.counts_send);
    c.partitioned = true;
  }

  void part_phase1(rbm_ctx& c, cudaStream_t s) override {
    Nvtx range_("rbm_part_phase1");
    const DevParams& P = c.P;
    const Layout& L = c.L;
    const uint32_t G = (uint32_t)c.cfg.world_size, rank = (uint32_t)c.cfg.rank;
    const uint32_t nb1 = 1u << L.b1;
    c.mark(s);
    part_scan_kernel<<<1, 1024, 0, s>>>(P, c.counts_all, G, rank, c.cur1[1], c.prefix1, c.tile_off,
                                        tile2());
    cudaMemsetAsync(c.cur2, 0, (size_t)L.nbuckets * CUR2_STRIDE * 4, s);
    cudaMemsetAsync(c.cur1[0], 0, (size_t)c.L.nseg() * CUR1_STRIDE * 4, s);
    c.mark(s);
    split2(c, s, st(c, recv_buf(c, c.step)), stA(c), c.cur1[1]);
    c.mark(s);
    final_scan_kernel<<<nb1 / G, 512, 0, s>>>(P, c.cur2, c.prefix1, c.S);
    c.mark(s);
    fused(c, s, stA(c), part_dst(c, c.step + 1), L.cap1, c.cur1[0]);
    c.mark(s);
    halo_extract_kernel<T, D><<<1, 64, 0, s>>>(P, stA(c), L.cap2, c.S, c.halo_send);
  }

  void part_phase2(rbm_ctx& c, cudaStream_t s) override {
    Nvtx range_("rbm_part_phase2");
    const DevParams& P = c.P;
    const Layout& L = c.L;
    c.mark(s);
    halo_place_kernel<T, D><<<1, 64, 0, s>>>(P, stA(c), L.cap2, c.S, c.halo_recv);
    const unsigned grid = (unsigned)(((uint64_t)(L.nbuckets + 1) * 32 + 255) / 256);
    c.mark(s);
    straddle_kernel<T, D, KK, INTEG><<<grid, 256, 0, s>>>(P, stA(c), L.cap2, c.S, part_dst(c, c.step + 1),
                                                          L.cap1, c.cur1[0]);
    c.mark(s);
    pack_counts_kernel<<<1, 1024, 0, s>>>(c.cur1[0], L.nseg(), c.counts_send);
    c.mark(s);
    advance_kernel<<<1, 1, 0, s>>>(c.step_dev);
    c.mark(s);
  }

  void rbmr_part_phase(rbm_ctx& c, cudaStream_t s, int k) override {
    static const char* const names[5] = {"", "rbmr_request", "rbmr_serve", "rbmr_delta", "rbmr_apply"};
    Nvtx range_(names[k < 1 || k > 4 ? 0 : k]);
    const DevParams& P = c.P;
    RPart& R = c.rp;
    T* xa = reinterpret_cast<T*>(c.rxa);
    const unsigned gb = grid_for(R.bb1 - R.bb0, 128, 148 * 64);
    if (k == 1) {
      if (!c.aos_valid) {  // records of the own ids (id order) -> AoS, once
        rbmr_pack_local_kernel<T, D><<<grid_for(c.n0, 256), 256, 0, s>>>(c.n0, st(c, c.cur), xa);
        c.aos_valid = true;
      }
      cudaMemsetAsync(R.qcnt, 0, (size_t)R.G * 4, s);
      c.mark(s);
      rbmr_req_kernel<<<gb, 128, 0, s>>>(P, R, c.js);
      rbmr_req_counts_kernel<<<1, 64, 0, s>>>(R);
    } else if (k == 2) {
      c.mark(s);
      rbmr_serve_kernel<T, D><<<grid_for((uint64_t)R.G * R.cap, 256), 256, 0, s>>>(R, xa);
    } else if (k == 3) {
      c.mark(s);
      rbmr_delta_part_kernel<T, D, KK, INTEG><<<gb, 128, 0, s>>>(P, R);
    } else {
      cudaMemsetAsync(c.rmcnt, 0, c.n0 * 4, s);
      cudaMemsetAsync(c.rnovf, 0, 4, s);
      c.mark(s);
      rbmr_register_part_kernel<<<grid_for((uint64_t)R.G * R.cap, 256), 256, 0, s>>>(P, R, c.rmcnt, c.rmbox,
                                                                                   c.rovf, c.rnovf);
      rbmr_apply_part_kernel<T, D><<<grid_for(c.n0, 256), 256, 0, s>>>(P, R, xa, c.rmcnt, c.rmbox, c.rovf,
                                                                       c.rnovf);
      advance_kernel<<<1, 1, 0, s>>>(c.step_dev);
      c.mark(s);
    }
  }

  uint64_t gather_local(rbm_ctx& c, uint32_t* ids, void* x, cudaStream_t s) override {
    if (c.cfg.scheme == RBM_SCHEME_RBMR && c.aos_valid && is_partitioned(c.cfg)) {
      gather_aos_part_kernel<T, D><<<grid_for(c.n0, 256), 256, 0, s>>>(
          reinterpret_cast<const T*>(c.rxa), c.id0, c.n0, 0, 0, reinterpret_cast<T*>(x), ids);
      return c.n0;
    }
    if (!is_partitioned(c.cfg) || !c.partitioned) {  // records in id order (this rank's initial ids)
      gather_local_kernel<T, D><<<grid_for(c.n0, 256), 256, 0, s>>>(c.n0, st(c, 0), ids, reinterpret_cast<T*>(x));
      return c.n0;
    }
    uint32_t* off = reinterpret_cast<uint32_t*>(c.xchg);
    seg_offsets_kernel<<<1, 1024, 0, s>>>(c.P, c.counts_all, (uint32_t)c.cfg.world_size, (uint32_t)c.cfg.rank, off);
    gather_local_part_kernel<T, D><<<grid_for((uint64_t)c.L.nseg() * c.L.cap1, 256), 256, 0, s>>>(
        c.P, st(c, recv_buf(c, c.step)), c.L.cap1, c.counts_all, (uint32_t)c.cfg.world_size, (uint32_t)c.cfg.rank,
        off, ids, reinterpret_cast<T*>(x));
    uint32_t total = 0;
    cudaMemcpyAsync(&total, off + c.L.nseg(), 4, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    return total;
  }

  // Algorithm 2 as written (row f2): draws + slot chains through the
  // partition by particle index (link records), then the dependency-driven
  // sweep (no host synchronisation: graph-capturable)
  void step_rbmr_seq(rbm_ctx& c, cudaStream_t s) {
    T* xa = reinterpret_cast<T*>(c.rxa);
    if (!c.aos_valid) {
      rbmr_pack_kernel<T, D><<<grid_for(c.cfg.n, 256), 256, 0, s>>>(c.cfg.n, st(c, c.cur), xa);
      c.aos_valid = true;
    }
    cudaMemsetAsync(c.rticket, 0, 4, s);
    cudaMemsetAsync(c.rexpect, 0xff, c.nslots * 4, s);  // SEQ_FREE: a particle's first slot waits for nobody
    partition_slots<true, LinkRT>(c, s, c.rexpect);
    c.mark(s);
    // CTAs of 4 warps per SM (experiment knob RBM_SEQ_CTAS).  Measured at C5
    // (gpu_r3sq.sh): 16/12/8/6/4/2 CTAs per SM = 14.12/14.12/13.49/13.23/
    // 13.06/13.79 ms -- fewer random sector accesses in flight go faster
    unsigned per_sm = 4;
    if (const char* e = std::getenv("RBM_SEQ_CTAS")) per_sm = (unsigned)std::max(1, std::min(16, std::atoi(e)));
    rbmr_seq_dep_kernel<T, D, KK, INTEG><<<(unsigned)num_sms * per_sm, 128, 0, s>>>(c.P, c.nbatch, c.js, c.rexpect, xa,
                                                                                  c.rticket);
    c.mark(s);
    advance_kernel<<<1, 1, 0, s>>>(c.step_dev);
    c.mark(s);
  }

  // slot records {j_s, s[, Delta_s]} -> partition by particle index -> per id
  // bucket: increments added in the canonical order (RBM-r), or expected tags (RBM-r', LINK)
  template <bool LINK, class RT> void partition_slots(rbm_ctx& c, cudaStream_t s, uint32_t* expect) {
    const DevParams& P = c.P;
    const Layout& L = c.L;
    T* xa = reinterpret_cast<T*>(c.rxa);
    const uint32_t W = 1u << (L.idbits - L.B);
    const uint32_t bpc = EMIT_TS / c.cfg.p;
    cudaMemsetAsync(c.cur1[0], 0, (size_t)(1u << L.b1) * CUR1_STRIDE * 4, s);
    c.mark(s);
    // sized for 2^10 digits whatever b1: three CTAs per SM at C5.  Measured
    // (gpu_r3em.sh, C5 RBM-r emit): 4 CTAs/SM 10.5 ms, 3 CTAs 7.36, 2 CTAs
    // 7.47, 1 CTA 10.9 -- more concurrent random gathers than three CTAs'
    // worth slow the gathers down
    size_t esm = emit_smem_bytes<T, D, LINK>();
    if (const char* e = std::getenv("RBM_EMIT_SMEM"))  // experiment knob: pad to limit CTAs per SM
      esm = std::max<size_t>(esm, std::min<size_t>((size_t)std::atol(e), 200 * 1024));
    rbmr_emit_kernel<T, D, KK, INTEG, LINK>
        <<<(unsigned)((c.nbatch + bpc - 1) / bpc), EMIT_BLOCK, esm, s>>>(
            P, c.nbatch, xa, LINK ? c.js : nullptr, c.rinc[0], c.cur1[0], L.cap1);
    const unsigned char* fin = c.rinc[0];
    const uint32_t* fcnt = c.cur1[0];
    if (L.b2) {
      c.mark(s);
      tile_scan_kernel<<<1, 1024, 0, s>>>(P, c.cur1[0], c.prefix1, c.tile_off, c.S, (uint32_t)split_tile_rt<RT>());
      cudaMemsetAsync(c.cur2, 0, (size_t)L.nbuckets * CUR2_STRIDE * 4, s);
      c.mark(s);
      split_kernel<RT, SPLIT_BLOCK><<<(unsigned)num_sms * SPLIT_MINB, SPLIT_BLOCK, split_smem_bytes_rt<RT>(), s>>>(
          P, c.rinc[0], c.rinc[1], nullptr, c.cur2, L.cap2, c.cur1[0], c.tile_off, L.cap1);
      fin = c.rinc[1];
      fcnt = c.cur2;
    }
    c.mark(s);
    rbmr_bucket_apply_kernel<T, D, LINK><<<L.nbuckets, 256, rapply_smem_bytes<T, D, LINK>(L.cap2, W), s>>>(
        P, fin, L.cap2, fcnt, W, xa, expect);
  }

  void rbmr_slots(rbm_ctx& c, uint32_t m, uint32_t* out, cudaStream_t s) override {
    rbmr_slots_kernel<KK><<<grid_for(c.nbatch, 128), 128, 0, s>>>(c.P, c.nbatch, m, out);
  }

  // RBM-r Jacobi sweep (reading D:8): increments routed to their particles
  // through the partition by particle index (rbmr_emit -> split -> apply)
  void step_rbmr(rbm_ctx& c, cudaStream_t s) {
    T* xa = reinterpret_cast<T*>(c.rxa);
    if (!c.aos_valid) {  // state set by init / set_state (records) -> AoS, once
      rbmr_pack_kernel<T, D><<<grid_for(c.cfg.n, 256), 256, 0, s>>>(c.cfg.n, st(c, c.cur), xa);
      c.aos_valid = true;
    }
    partition_slots<false, IncRT<T, D>>(c, s, nullptr);
    c.mark(s);
    advance_kernel<<<1, 1, 0, s>>>(c.step_dev);
    c.mark(s);
  }
};

template <typename T, int D>
EngineBase* make_for_kernel(uint32_t kernel, uint32_t integ) {
  if (integ == RBM_INTEG_VERLET) {  // second order: 1-D particles stored as (x, v | x_prev)
    if constexpr (D == 2) {
      if (kernel == RBM_K_SMOOTH_TEST) return new Engine<T, 2, KK_SMOOTH, 2>();
      if (kernel == RBM_K_ZERO) return new Engine<T, 2, KK_ZERO, 2>();
    }
    return nullptr;
  }
  switch (kernel) {
    case RBM_K_ZERO: return new Engine<T, D, KK_ZERO, 0>();
    case RBM_K_BOUNDED_CONFIDENCE: return new Engine<T, D, KK_BOUNDED, 0>();
    case RBM_K_GAUSS_ATTR_REP: return new Engine<T, D, KK_GAUSS_AR, 0>();
    case RBM_K_COULOMB_REG: return new Engine<T, D, KK_COULOMB_REG, 0>();
    case RBM_K_SMOOTH_TEST: return new Engine<T, D, KK_SMOOTH, 0>();
    case RBM_K_DYSON:
      if constexpr (D == 1) return integ ? (EngineBase*)new Engine<T, 1, KK_DYSON, 1>() : new Engine<T, 1, KK_DYSON, 0>();
      return nullptr;
    case RBM_K_COULOMB:
      if constexpr (D == 3) return integ ? (EngineBase*)new Engine<T, 3, KK_COULOMB, 1>() : new Engine<T, 3, KK_COULOMB, 0>();
      return nullptr;
    case RBM_K_ADJACENCY: return integ == RBM_INTEG_SPLIT_EXACT_PAIR ? new Engine<T, D, KK_ADJ, 1>() : nullptr;
    case RBM_K_LINEAR:
      if constexpr (D == 1) {
        if (integ) return new Engine<T, 1, KK_LINEAR, 1>();
      } else {
        if (integ) return nullptr;
      }
      return new Engine<T, D, KK_LINEAR, 0>();
  }
  return nullptr;
}

inline const char* const* kernel_names(const rbm_ctx& c, uint32_t* count) {
  static const char* const r[] = {"rbmr_emit", "rbmr_apply", "advance"};
  static const char* const r2[] = {"rbmr_emit", "tile_scan", "split", "rbmr_apply", "advance"};
  static const char* const rs[] = {"rbmr_draw", "rbmr_link", "rbmr_seq_sweep", "advance"};
  static const char* const rs2[] = {"rbmr_draw", "tile_scan", "split", "rbmr_link", "rbmr_seq_sweep", "advance"};
  if (c.cfg.scheme == RBM_SCHEME_RBMR_SEQ) {
    if (c.L.b2) { *count = 6; return rs2; }
    *count = 4;
    return rs;
  }
  static const char* const b0[] = {"resident_step"};
  static const char* const p1[] = {"tile_scan", "bucket_step", "straddle", "advance"};
  static const char* const p2[] = {"tile_scan", "split", "final_scan", "bucket_step", "straddle", "advance"};
  static const char* const pt[] = {"part_scan", "split", "final_scan", "bucket_step",
                                   "halo_extract", "halo_place", "straddle", "pack_counts", "advance"};
  static const char* const prr[] = {"rbmr_request", "rbmr_serve", "rbmr_delta", "rbmr_apply"};
  if (is_partitioned(c.cfg) && c.cfg.scheme == RBM_SCHEME_RBMR) { *count = 4; return prr; }
  if (is_partitioned(c.cfg)) { *count = 9; return pt; }
  if (c.cfg.scheme == RBM_SCHEME_RBMR) {
    if (c.L.b2) { *count = 5; return r2; }
    *count = 3;
    return r;
  }
  if (c.L.B == 0) { *count = 1; return b0; }
  if (c.L.b2 == 0) { *count = 4; return p1; }
  *count = 6;
  return p2;
}

#define RBM_DECLARE_ENGINES(T) \
  EngineBase* make_engine_##T##_d1(uint32_t, uint32_t); \
  EngineBase* make_engine_##T##_d2(uint32_t, uint32_t); \
  EngineBase* make_engine_##T##_d3(uint32_t, uint32_t);
RBM_DECLARE_ENGINES(f32)
RBM_DECLARE_ENGINES(f64)
#undef RBM_DECLARE_ENGINES

}  // namespace rbmhost

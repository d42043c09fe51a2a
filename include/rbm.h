/*
 * include/rbm.h -- C ABI of the B200-native Random Batch Method library
 * (librbm.so, built from paper_1812_10575_b200/csrc/ for sm_100a).
 *
 * One call of rbm_step() is one time step of the Random Batch Method of
 * Jin, Li & Liu (arXiv:1812.10575) for the first-order binary-interaction
 * particle system, Eq. (1.2):
 *
 *   dX^i = -grad V(X^i) dt + 1/(N-1) sum_{j != i} K(X^i - X^j) dt + sigma dB^i,
 *
 * in one of two schemes:
 *   RBM_SCHEME_RBM1  Algorithm 1: a fresh random division of
 *                    {0..N-1} into batches of size p, then Eq. (2.2)
 *                     inside each batch with prefactor
 *                    1/(|B|-1), integrated by forward Euler-Maruyama
 *                     or by the splitting with the
 *                    exact p=2 pair flow.
 *   RBM_SCHEME_RBMR  Algorithms 2/3: one sweep of ceil(N/p)
 *                    with-replacement batches, read as a Jacobi-additive sweep
 *                    (reading D:8).
 *
 * The random division at step m is the permutation that sorts the ids by
 * (key_m(id), id), key_m(id) = word 0 of Philox4x32-10 at counter
 * (id, 0, m, TAG_KEY | replica<<8) under key (seed_lo, seed_hi); batch b is
 * sorted positions [b p, (b+1) p) with the remainder rule of DESIGN.md D:7.
 * Brownian increments use counter (id, blk, m, TAG_NOISE | replica<<8).
 * Everything is a pure function of (config, seed, step, id): results do not
 * depend on launch geometry, on the internal storage order, or on the GPU.
 *
 * Conventions for every entry point:
 *   - No C++ types, no exceptions cross the boundary; every call returns an
 *     rbm_status.  On failure rbm_last_error(ctx) (or rbm_last_error(NULL) for
 *     failures before a context exists) returns a NUL-terminated message owned
 *     by the library, valid until the next call on the same context/thread.
 *   - Positions exchanged with the caller are row-major (particle, axis):
 *     N*d scalars of the configured dtype (float for RBM_F32, double for
 *     RBM_F64), in id order.
 *   - "Device pointer" = CUDA global memory of the current device; "host
 *     pointer" = ordinary or pinned host memory.
 *   - Ownership: the caller owns the workspace, every input/output buffer and
 *     the CUDA stream; the library owns the context (and its private capture
 *     stream, CUDA graphs and events) and releases them in rbm_destroy().
 *   - A context is used by one host thread at a time.
 *   - Work is stream-ordered on the caller's stream and asynchronous unless
 *     stated; device-side failures (non-finite state, overflow of an internal
 *     capacity) surface at the next rbm_sync / rbm_gather as
 *     RBM_ERR_NONFINITE / RBM_ERR_CAPACITY.
 */
#ifndef RBM_H_
#define RBM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RBM_ABI_VERSION 1u

typedef struct rbm_ctx rbm_ctx; /* opaque, library-owned host object */

typedef enum {
  RBM_OK = 0,
  RBM_ERR_INVALID_ARG = 1,    /* config or argument rejected (message says which) */
  RBM_ERR_UNKNOWN_KERNEL = 2, /* kernel/potential id not in the registry */
  RBM_ERR_UNSUPPORTED = 3,    /* valid request this build does not implement */
  RBM_ERR_WORKSPACE = 4,      /* workspace NULL, too small or misaligned (256 B) */
  RBM_ERR_CUDA = 5,           /* a CUDA runtime call failed (message has the code) */
  RBM_ERR_NCCL = 6,           /* NCCL not loadable, or an NCCL call failed (partitioned system) */
  RBM_ERR_NONFINITE = 7,      /* a non-finite position was produced; message names step and id */
  RBM_ERR_STATE = 8,          /* call out of order (e.g. step before init) */
  RBM_ERR_CAPACITY = 9        /* an internal per-bucket capacity was exceeded */
} rbm_status;

typedef enum { RBM_F32 = 0, RBM_F64 = 1 } rbm_dtype;
/* RBM_SCHEME_RBMR_SEQ: Algorithm 2 (RBM-r') exactly as
 * written: the ceil(N/p) batches of a sweep (the same slot draws as RBMR) are
 * applied in draw order, each from the positions left by the earlier ones.
 * On the GPU each batch waits only for the earlier batches that last touched
 * its members (dependency flags), so independent batches run in parallel; no
 * host synchronisation, CUDA-graph replayed like the other schemes. */
typedef enum { RBM_SCHEME_RBM1 = 0, RBM_SCHEME_RBMR = 1, RBM_SCHEME_RBMR_SEQ = 2 } rbm_scheme;
/* RBM_INTEG_VERLET (row f3): the second-order (Hamiltonian) system of
 * PAPER.md:848-870, X' = V, V' = -grad V(X) + mean K, for 1-D particles
 * stored as d = 2 components; position Verlet with the RBM-1
 * batch force of each step.  The state at step0 is (x_0, v_0) when
 * state_form == 0 (first step x_1 = x_0 + v_0 tau + F_0 tau^2/2), or
 * (x_n, x_{n-1}) when state_form == 1 (x_{n+1} = 2 x_n - x_{n-1} + F_n tau^2);
 * after any step it is (x_n, x_{n-1}).  sigma must be 0; kernel smooth or zero. */
typedef enum { RBM_INTEG_EULER_MARUYAMA = 0, RBM_INTEG_SPLIT_EXACT_PAIR = 1, RBM_INTEG_VERLET = 2 } rbm_integrator;

/* Interaction kernels K(z), z = X^i - X^j (Eq. 1.2). */
typedef enum {
  RBM_K_ZERO = 0,
  RBM_K_DYSON = 1,              /* 1/z, d=1 (Eq. 4.4); K(0):=0            */
  RBM_K_COULOMB = 2,            /* z/|z|^3, d=3; K(0):=0                 */
  RBM_K_BOUNDED_CONFIDENCE = 3, /* -a z 1{|z|<r}, kparam={a, r, closed}; closed != 0: the paper's
                                   closed window |z| <= r, phi = chi_[0,1] (Eq. 5.12) */
  RBM_K_GAUSS_ATTR_REP = 4,     /* z e^{-|z|^2/2} - z e^{-|z|^2/8}/4 (BASELINE.json C4)       */
  RBM_K_COULOMB_REG = 5,        /* z/(|z|^2+eps)^{3/2}, kparam={eps} (BASELINE.json C5)       */
  RBM_K_SMOOTH_TEST = 6,        /* z/(1+|z|^2)                             */
  RBM_K_LINEAR = 7,             /* -kappa z, kparam={kappa}: wealth trading phi=y^2/2 */
  RBM_K_ADJACENCY = 8           /* clustering (Sec. 5.3): the picked pair (i, j) follows
                                   dX^i/dt = alpha (a_ij - beta)(X^j - X^i), a_ij from rbm_set_adjacency;
                                   kparam={alpha, beta, edge_restricted}; RBM-r / RBM-r', p = 2, split
                                   integrator (the exact update formula of P:1258-1264), one GPU */
} rbm_kernel;

/* Noise term of Eq. (1.2): additive sigma dB^i, or multiplicative sigma X^i dB^i
 * (componentwise; the wealth model, Sec. 5.2.1).  With the
 * split integrator the multiplicative step is the exact geometric Brownian
 * motion x' = w exp(sigma sqrt(dt) z - sigma^2 dt / 2). */
typedef enum { RBM_NOISE_ADDITIVE = 0, RBM_NOISE_GEOMETRIC = 1 } rbm_noise;

typedef enum { RBM_V_NONE = 0, RBM_V_HARMONIC = 1 /* beta|x|^2/2, vparam={beta} */ } rbm_potential;
typedef enum { RBM_CONSTRAINT_NONE = 0, RBM_CONSTRAINT_UNIT_SPHERE = 1 /* d=3 */ } rbm_constraint;

/* Initial data X_0^i ~ nu, iid; computed in fp64 from
 * Philox counter (id, blk, 0, TAG_INIT|replica<<8), then rounded to dtype. */
typedef enum {
  RBM_INIT_USER = 0,          /* caller supplies X_0 via rbm_set_state()            */
  RBM_INIT_NORMAL = 1,        /* iparam = {mean, std}                                */
  RBM_INIT_UNIFORM_BOX = 2,   /* iparam = {a, b}: U[a,b]^d                           */
  RBM_INIT_UNIFORM_SPHERE = 3,/* uniform on S^{d-1}                                  */
  RBM_INIT_GAUSS_MIXTURE = 4, /* iparam = {K, std, lo, hi}: equal weights, centres U[lo,hi]^d */
  RBM_INIT_ABS_NORMAL = 5     /* iparam = {mean, std}: |mean + std z| (wealth) */
} rbm_init_kind;

typedef enum { RBM_MEM_DEVICE = 0, RBM_MEM_HOST = 1 } rbm_mem;

typedef struct {
  uint32_t abi_version;  /* must be RBM_ABI_VERSION */
  uint32_t dtype;        /* rbm_dtype: arithmetic and storage precision of X */
  uint32_t d;            /* spatial dimension, 1..3 */
  uint32_t p;            /* batch size, 2..64 (or p == n for n <= 2048) */
  uint64_t n;            /* number of particles N, 2..2^31 */
  uint32_t scheme;       /* rbm_scheme */
  uint32_t integrator;   /* rbm_integrator */
  uint32_t kernel;       /* rbm_kernel */
  uint32_t potential;    /* rbm_potential */
  uint32_t constraint;   /* rbm_constraint */
  uint32_t init;         /* rbm_init_kind */
  double kparam[4];
  double vparam[2];
  double iparam[8];
  double sigma;          /* noise amplitude, >= 0 */
  double dt;             /* time step tau, > 0 */
  uint64_t seed;         /* Philox key (seed_lo, seed_hi) */
  uint64_t step0;        /* index m of the first step (checkpoint resume) */
  uint32_t replica;      /* ensemble member, enters Philox counter word 3 (< 2^24) */
  int32_t world_size;    /* 1, or G = 2..64 (power of two): partitioned single system, see rbm_part_* */
  int32_t rank;          /* 0..G-1: this process's rank (one GPU per rank) */
  uint32_t debug_bucket_cap; /* 0 = automatic; >0 forces the per-bucket smem capacity (tests) */
  uint32_t noise;        /* rbm_noise */
  uint32_t state_form;   /* RBM_INTEG_VERLET: 0 = (x, v) at step0, 1 = (x_n, x_{n-1}) */
} rbm_config;

/* Partitioned single system with the library's own NCCL communicator
 * (SURVEY.md 8(b)): rank 0 calls this, the caller broadcasts the 128 bytes
 * to every rank (e.g. torch.distributed), and each rank passes them to
 * rbm_init().  libnccl.so.2 is opened at first use.
 * Errors: RBM_ERR_NCCL (NCCL not loadable, or ncclGetUniqueId failed). */
rbm_status rbm_get_nccl_unique_id(void* out128);

/* Bytes of device workspace rbm_init() needs for this config.
 * Errors: RBM_ERR_INVALID_ARG / RBM_ERR_UNKNOWN_KERNEL (same validation as rbm_init). */
rbm_status rbm_workspace_size(const rbm_config* cfg, size_t* bytes);

/* Validate cfg (eagerly, all checks), carve ws (device pointer, >= the size
 * above, 256-byte aligned, owned by the caller and untouched by it until
 * rbm_destroy), and enqueue the initial data on `cuda_stream` (a cudaStream_t;
 * NULL = legacy default stream).  For RBM_INIT_USER the state is undefined
 * until rbm_set_state().  nccl_unique_id: NULL on one GPU, and for a
 * partitioned context whose exchanges the caller performs (rbm_part_*);
 * otherwise the 128-byte id of rbm_get_nccl_unique_id(), identical on every
 * rank: rbm_init then creates the library's NCCL communicator (collective:
 * every rank must call it; RBM_ERR_NCCL on failure), and rbm_step / rbm_run /
 * rbm_gather on the partitioned context run the exchanges themselves.
 * On success *out receives the context; the step index is cfg->step0. */
rbm_status rbm_init(const rbm_config* cfg, void* ws, size_t ws_bytes, void* cuda_stream,
                    const void* nccl_unique_id, rbm_ctx** out);

/* Clustering model (RBM_K_ADJACENCY): the symmetric adjacency A = (a_ij) in
 * CSR, device pointers owned by the caller and unchanged until rbm_destroy:
 * row_ptr n+1 uint32, col_idx nnz uint32 (each row sorted ascending), val nnz
 * doubles a_ij >= 0; entries off the pattern are 0.  With kparam[2] != 0 the
 * RBM-r pairs are drawn uniformly among the nnz entries ("picked from
 * those with nonzeros of a_ij only"; a diagonal entry is redrawn).  Must be
 * called before the first step of such a context. */
rbm_status rbm_set_adjacency(rbm_ctx* ctx, const uint32_t* row_ptr, const uint32_t* col_idx, const double* val,
                             uint64_t nnz);

/* Replace the state by X given in id order (N*d scalars of dtype, row-major);
 * `where` says whether x is a host or device pointer.  Host input is copied
 * before the call returns (synchronous); device input is stream-ordered. */
rbm_status rbm_set_state(rbm_ctx* ctx, const void* x, uint32_t where);

/* Enqueue one step X_m -> X_{m+1} (async); m advances by one.
 * Determinism: the result is a function of (cfg, X_m, m) only -- not of the
 * launch geometry, the bucket layout or world_size.  Inside a batch of
 * p <= 32 members the partner terms K(x_i - x_j) are summed in a fixed
 * rotation order (each pair evaluated once, K odd);
 * Eq. (2.2) as written sums in ascending order, so results differ from that
 * order by rounding only. */
rbm_status rbm_step(rbm_ctx* ctx);

/* Enqueue nsteps steps as CUDA-graph replays (async); no host work per step.
 * Partitioned context with a communicator: one step = phase 1, the halo
 * exchange (NCCL send/recv), phase 2, the counts all-gather and the records
 * all-to-all (none in the fused mode), all on the context's stream; the
 * steps are captured into CUDA graphs with their NCCL calls (eager launches
 * if the capture is refused). */
rbm_status rbm_run(rbm_ctx* ctx, uint64_t nsteps);

/* Write positions of ids [id_begin, id_end) in id order, (id_end-id_begin)*d
 * scalars, to x_out (host or device per `where`).  Synchronises the stream,
 * then reports RBM_ERR_NONFINITE / RBM_ERR_CAPACITY if the device flagged
 * one; the data are written in any case.  Partitioned context with a
 * communicator: collective (every rank calls it and receives the whole range;
 * an NCCL all-reduce of the disjoint rows). */
rbm_status rbm_gather(rbm_ctx* ctx, uint64_t id_begin, uint64_t id_end, void* x_out, uint32_t where);

/* This rank's particles, unordered: ids_out (device, >= n_local u32) and
 * x_out (device, >= n_local*d scalars, row-major) in storage order; *count
 * (host) = n_local (all N on one GPU, written in id order).  Not collective;
 * synchronises the stream.  Sizing: a rank holds at most its workspace's
 * slot count; the caller may allocate N rows. */
rbm_status rbm_gather_local(rbm_ctx* ctx, uint32_t* ids_out, void* x_out, uint64_t* count);

/* Synchronise the stream and check the device flags (see rbm_gather). */
rbm_status rbm_sync(rbm_ctx* ctx);

/* Index m of the next step to be enqueued (host-side counter). */
uint64_t rbm_step_index(const rbm_ctx* ctx);

/* Number of kernel launches one rbm_step enqueues (for the bench's
 * gpu_launches count); 0 if ctx is NULL. */
uint32_t rbm_launches_per_step(const rbm_ctx* ctx);

/* Diagnostics: bucket layout chosen for this config (B prefix bits, number of
 * scatter passes, per-bucket capacity).  Any out pointer may be NULL. */
rbm_status rbm_layout(const rbm_ctx* ctx, uint32_t* prefix_bits, uint32_t* passes, uint32_t* bucket_cap);

/* Test hook (RBM-1): the NEXT rbm_step() also writes its permutation pi_m
 * (sorted position -> id: ids ordered by (key_m(id), id); batch b = positions
 * [b p, (b+1) p) with the remainder rule) to `order_out`, N uint32 values,
 * device pointer, stream-ordered.  rbm_run() ignores and clears it. */
rbm_status rbm_debug_permutation(rbm_ctx* ctx, uint32_t* order_out);

/* Test hook (RBM_SCHEME_RBMR / _SEQ only): the slot draws j_s of the last
 * step, ceil(N/p)*p uint32 values (device); on a partitioned system the
 * slots of this rank's batches only. */
rbm_status rbm_debug_slots(rbm_ctx* ctx, uint32_t* slots_out);

/* Test hook: Philox4x32-10 of `count` (ctr, key) pairs on the device:
 * in = count*6 uint32 (c0,c1,c2,c3,k0,k1), out = count*4 uint32 (device). */
rbm_status rbm_debug_philox(const uint32_t* in, uint32_t* out, uint64_t count, void* cuda_stream);

/* Name of the i-th kernel one step launches (i < rbm_launches_per_step);
 * "" when out of range.  Static storage. */
const char* rbm_kernel_name(const rbm_ctx* ctx, uint32_t i);

/* Per-kernel timing: after rbm_timing_begin(ctx, max_steps) the next
 * max_steps steps (rbm_step, or rbm_run, which then launches eagerly instead of
 * replaying graphs) record a CUDA event on the caller's stream before every
 * kernel and after the last.  rbm_timing_end() synchronises the stream and
 * writes, for every kernel slot i < rbm_launches_per_step, the summed device
 * time in ms over the recorded steps (ms_per_kernel, caller-owned array) and
 * the number of steps recorded. */
rbm_status rbm_timing_begin(rbm_ctx* ctx, uint32_t max_steps);
rbm_status rbm_timing_end(rbm_ctx* ctx, double* ms_per_kernel, uint32_t* steps_recorded);

/* ------------------------------------------------------------------------
 * Partitioned single system (world_size G > 1).
 * One global system of N particles is split over G ranks (one GPU each) by
 * key range: rank r holds, at step m, exactly the particles whose shuffle key
 * key_m has top log2(G) bits equal to r.  Because the division is the (key,
 * id) order (reading D:6), rank r's particles are the global
 * sorted positions [O_r, O_r + n_r), O_r = n_0 + ... + n_{r-1}; every batch
 * lies in one rank except the one crossing O_r, which rank r completes with
 * t_r = O_r - (start of that batch) <= p-1 records of rank r-1 (the "halo").
 * The result is bit-identical to the same config on one GPU (world_size 1).
 *
 * With an NCCL id given to rbm_init, the library runs the whole step,
 * exchanges included (rbm_step / rbm_run above).  Without one, the library
 * runs every computation and the caller performs the three exchanges between
 * the phases (plumbing: torch.distributed, or the one-process loopback used
 * to test the G > 1 kernels on one GPU), using byte offsets into the
 * caller-owned workspace from rbm_part_info_get():
 *   H  halo:     rank r's halo_send (halo_bytes) -> rank r+1's halo_recv
 *   C  counts:   all-gather of every rank's counts_send (nseg u32) into
 *                counts_all (world_size * nseg u32, rank-major)
 *   R  records:  for each of the narrays exchanged arrays a, an all-to-all
 *                with equal chunks of chunk_elems elements of elem_bytes[a]:
 *                chunk j of send_off[a] (to rank j) -> chunk r of rank j's
 *                recv_off[a]
 * Protocol: rbm_init; rbm_part_prologue; C; R; then per step
 *   rbm_part_phase1; H; rbm_part_phase2; C; R.
 * rbm_step / rbm_run return RBM_ERR_STATE on a partitioned context without
 * a communicator.
 * rbm_init draws (or rbm_set_state takes, n0 rows) the particles with ids
 * [id0, id0 + n0) = [floor(N r/G), floor(N (r+1)/G)); rbm_gather writes, into
 * a DEVICE buffer, the positions of the ids in the range that this rank holds
 * and leaves the other rows untouched (host output: RBM_ERR_UNSUPPORTED).
 * A rank that ends up with fewer than p particles (probability ~0 at the
 * required n/G >= max(1024, 16p)) is reported as RBM_ERR_CAPACITY.
 * ------------------------------------------------------------------------ */
typedef struct {
  uint64_t ws_bytes;        /* workspace bytes (= rbm_workspace_size) */
  uint32_t world_size, rank;
  uint32_t nseg;            /* pass-1 segments (2^b1 digits x 2^segk cursors): u32 counts per rank in exchange C */
  uint32_t narrays;         /* exchanged arrays: 1 (the state records: id, [key,] x; elem_bytes[0] = 8, 16 or 32) */
  uint64_t chunk_elems;     /* elements per destination rank in each exchanged array */
  uint64_t send_off[5];     /* byte offsets in ws of the exchanged send arrays (a < narrays) */
  uint64_t recv_off[5];     /* byte offsets in ws of the exchanged receive arrays */
  uint32_t elem_bytes[5];   /* element size of array a */
  uint64_t counts_send_off; /* nseg u32 */
  uint64_t counts_all_off;  /* world_size * nseg u32, rank-major */
  uint64_t halo_send_off, halo_recv_off, halo_bytes;
  uint64_t id0, n0;         /* this rank's initial ids [id0, id0 + n0) */
  uint64_t chunk_bytes[5];  /* bytes per destination chunk of exchange a (RBM-1: chunk_elems * elem_bytes[a]) */
  uint32_t phases;          /* library phases per step: 2 (RBM-1) or 4 (RBM-r) */
  uint32_t pad;
} rbm_part_info;

/* RBM-r on a partitioned system (scheme RBM_SCHEME_RBMR):
 * rank r owns the ids [id0, id0+n0) and the batches [floor(nb r/G),
 * floor(nb (r+1)/G)) of the sweep (nb = ceil(N/p)); the slot draws are the
 * one-GPU ones, and the step is bit-identical to the one-GPU RBM-r step.  Its
 * three exchanges are all-to-alls of equal chunks (chunk j of send_off[a] ->
 * chunk r of rank j's recv_off[a], chunk_bytes[a] each), a = 0 requests
 * (header: count; ids j_s), a = 1 responses (x_j, reverse direction at the
 * requests' positions), a = 2 increments (slot s, Delta_s).  Caller protocol
 * per step: rbm_part_phase(ctx, 1); exchange 0; phase 2; exchange 1; phase 3;
 * exchange 2; phase 4 (m advances).  With a communicator, rbm_step / rbm_run
 * do all of it. */

/* Exchange layout for cfg (host-only computation, no device work; same
 * validation as rbm_init).  RBM_ERR_STATE if cfg->world_size == 1. */
rbm_status rbm_part_info_get(const rbm_config* cfg, rbm_part_info* out);

/* Fused exchange (optional, world_size <= 8; SURVEY.md 8(e) "G9"): give the
 * context every rank's workspace base as a device pointer usable from this
 * GPU (peer-mapped over NVLink, e.g. a CUDA IPC mapping; peer_ws[rank] = this
 * context's own ws).  From then on the bucket step, the straddle kernel and
 * the prologue store each updated record straight into the destination
 * rank's receive buffer (double-buffered by step parity), so exchange R is
 * not performed: the all-to-all is fused into the kernels' output stores.
 * Exchanges H and C stay (C, an all-gather, also orders the steps).  Call
 * before rbm_part_prologue; all ranks must use the same config. */
rbm_status rbm_part_set_peers(rbm_ctx* ctx, const uint64_t* peer_ws, uint32_t count);

/* Fused exchange set up by the library (communicator required; collective,
 * before the first step): each rank's workspace allocation is exported with
 * cudaIpcGetMemHandle, the handles are all-gathered over NCCL and opened on
 * every rank (peer access over NVLink / NVSwitch), then as rbm_part_set_peers.
 * All ranks switch or none does (RBM_ERR_UNSUPPORTED: the NCCL all-to-all
 * stays in use).  The mappings are closed by rbm_destroy. */
rbm_status rbm_part_map_peers(rbm_ctx* ctx);

/* Enqueue the partition of the initial state (id order) into the send
 * buckets; follow with exchanges C and R.  Once per context. */
rbm_status rbm_part_prologue(rbm_ctx* ctx);

/* Enqueue the first part of step m (needs C and R done): global offsets from
 * counts_all, split of the received segments into final buckets, the fused
 * bucket step (sort by (key_m, id), Eq. 2.2 + update of every batch inside
 * this rank, partition of the updated records by key_{m+1}), halo_send.
 * Follow with exchange H. */
rbm_status rbm_part_phase1(rbm_ctx* ctx);

/* Enqueue the rest of step m: the batches straddling final buckets and the
 * one crossing O_r (with halo_recv), counts_send; m advances.  Follow with
 * exchanges C and R. */
rbm_status rbm_part_phase2(rbm_ctx* ctx);

/* Phase k of the step (1 <= k <= rbm_part_info.phases): RBM-1 k = 1, 2 are
 * rbm_part_phase1 / rbm_part_phase2; RBM-r see above.  RBM_ERR_STATE out of
 * order. */
rbm_status rbm_part_phase(rbm_ctx* ctx, uint32_t k);

/* ------------------------------------------------------------------------
 * Direct O(N^2) steps: the fully coupled forward
 * Euler-Maruyama step of Eq. (1.2),
 *   x_i' = x_i + dt (-grad V(x_i) + 1/(N-1) sum_{j != i} K(x_i - x_j)) + sigma sqrt(dt) z_i,
 * the reference solution the paper measures RBM against (Sec. 4.1,
 * PAPER.md:808-813) and the p = N special case of Eq. (2.2).  z_i at step m
 * is the Brownian increment RBM step m uses (counter (i, blk, m, TAG_NOISE)),
 * so an RBM run and a direct run from the same X_0 and seed are
 * synchronously coupled.  Sphere constraint as in RBM (D:11).  cfg: model
 * fields only (p, scheme, world_size ignored); integrator Euler-Maruyama or
 * Verlet (row f3: the full-force reference of PAPER.md:866-868; the start
 * formula x_1 = x_0 + v_0 tau + F_0 tau^2/2 applies to the step with index
 * cfg->step0 when state_form == 0, so consecutive runs compose); n <= 2^24.
 * Stateless: no context.
 * ------------------------------------------------------------------------ */
/* Bytes of device workspace (ping-pong copy of x + flags). */
rbm_status rbm_direct_workspace_size(const rbm_config* cfg, size_t* bytes);
/* Clear the non-finite flag in ws (call once before the first rbm_direct_run). */
rbm_status rbm_direct_reset(const rbm_config* cfg, void* ws, void* cuda_stream);
/* Enqueue nsteps direct steps m0, m0+1, ... on x (device, N*d scalars of
 * dtype, id order, row-major), in place; ws (device, >= the size above,
 * 256-B aligned, caller-owned).  Asynchronous on cuda_stream. */
rbm_status rbm_direct_run(const rbm_config* cfg, void* x_dev, uint64_t m0, uint64_t nsteps, void* ws,
                          size_t ws_bytes, void* cuda_stream);
/* Synchronise cuda_stream; RBM_ERR_NONFINITE if a direct step produced a
 * non-finite position (message names step and id). */
rbm_status rbm_direct_sync(const rbm_config* cfg, void* ws, void* cuda_stream);

/* Message for the last failure on ctx (or on this thread if ctx == NULL). */
const char* rbm_last_error(const rbm_ctx* ctx);

/* Release everything the library owns; the caller may then free ws. */
rbm_status rbm_destroy(rbm_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* RBM_H_ */

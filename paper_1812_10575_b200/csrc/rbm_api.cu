// rbm_api.cu -- C ABI of librbm.so (declared in include/rbm.h).
//
// Host orchestration only: validation, bucket-layout choice, workspace
// carving, per-config kernel dispatch, CUDA-graph capture/replay of steps.
// Every arithmetic step of the RBM path runs in the kernels of
// rbm_kernels.cuh; there is no CPU fallback.
#include "rbm_host.cuh"

namespace rbmhost {
thread_local std::string g_err;

EngineBase* make_engine(const rbm_config& k) {
  const bool f64 = k.dtype == RBM_F64;
  switch (k.d) {
    case 1: return f64 ? make_engine_f64_d1(k.kernel, k.integrator) : make_engine_f32_d1(k.kernel, k.integrator);
    case 2: return f64 ? make_engine_f64_d2(k.kernel, k.integrator) : make_engine_f32_d2(k.kernel, k.integrator);
    case 3: return f64 ? make_engine_f64_d3(k.kernel, k.integrator) : make_engine_f32_d3(k.kernel, k.integrator);
  }
  return nullptr;
}

rbm_status enqueue_steps(rbm_ctx* c, cudaStream_t s, uint64_t k) {
  for (uint64_t i = 0; i < k; ++i) {
    c->P.verlet_start = c->verlet_start ? 1u : 0u;  // by value into this step's launches
    c->eng->step(*c, s);
    c->verlet_start = false;
  }
  c->P.verlet_start = 0u;
  CU(cudaGetLastError());
  return RBM_OK;
}

rbm_status check_flags(rbm_ctx* c) {
  unsigned long long nf = 0;
  uint32_t cap = 0;
  CU(cudaMemcpy(&nf, c->nonfinite, sizeof nf, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(&cap, c->capacity_err, sizeof cap, cudaMemcpyDeviceToHost));
  if (cap == 2) return fail(c, RBM_ERR_CAPACITY, "a rank of the partitioned system held fewer than p particles; results are invalid");
  if (cap == 3) return fail(c, RBM_ERR_CAPACITY, "bounds check failed in a kernel (checked build); results are invalid");
  if (cap) return fail(c, RBM_ERR_CAPACITY, "a bucket exceeded every capacity fallback; results of that step are invalid");
  if (nf != ~0ull)
    return fail(c, RBM_ERR_NONFINITE, "non-finite position at step %llu, particle id %llu",
                (unsigned long long)(nf >> 32), (unsigned long long)(nf & 0xffffffffull));
  return RBM_OK;
}

#define NC(call)                                                                             \
  do {                                                                                       \
    ncclResult_t r_ = (call);                                                                \
    if (r_ != ncclSuccess)                                                                   \
      return fail(c, RBM_ERR_NCCL, "%s failed: %s", #call, nccl().GetErrorString(r_));       \
  } while (0)

// Exchanges C (counts all-gather) and R (records all-to-all, equal chunks;
// none when the kernels store into the peers' buffers) of the partitioned
// step, on the stream, over the library's communicator (include/rbm.h).
rbm_status part_exchange_cr(rbm_ctx* c, cudaStream_t s) {
  Nvtx range_("nccl_counts_records");
  NcclApi& N = nccl();
  const int G = c->cfg.world_size;
  NC(N.AllGather(c->counts_send, c->counts_all, c->L.nseg(), ncclUint32, c->comm, s));
  if (!c->fused) {
    const size_t chunk = (size_t)(c->L.nseg() >> c->L.g) * c->L.cap1 * rec_bytes(c->cfg);
    NC(N.GroupStart());
    for (int j = 0; j < G; ++j) {
      NC(N.Send(c->recbuf[1] + (size_t)j * chunk, chunk, ncclUint8, j, c->comm, s));
      NC(N.Recv(c->recbuf[2] + (size_t)j * chunk, chunk, ncclUint8, j, c->comm, s));
    }
    NC(N.GroupEnd());
  }
  return RBM_OK;
}

// Exchange H: rank r's halo_send -> rank r+1's halo_recv (the <= p-1 trailing
// records of the batch crossing O_{r+1}, the regroup is the
// step's only synchronisation point)
rbm_status part_exchange_h(rbm_ctx* c, cudaStream_t s) {
  Nvtx range_("nccl_halo");
  NcclApi& N = nccl();
  const int G = c->cfg.world_size, r = c->cfg.rank;
  const size_t hb = 16 + (size_t)HALO_MAX * rec_bytes(c->cfg);
  NC(N.GroupStart());
  if (r + 1 < G) NC(N.Send(c->halo_send, hb, ncclUint8, r + 1, c->comm, s));
  if (r > 0) NC(N.Recv(c->halo_recv, hb, ncclUint8, r - 1, c->comm, s));
  NC(N.GroupEnd());
  return RBM_OK;
}

// RBM-r exchange a (0 requests, 1 responses, 2 increments): chunk j of the
// send region to rank j, chunk j of the receive region from rank j
rbm_status rbmr_exchange(rbm_ctx* c, cudaStream_t s, int a) {
  Nvtx range_("nccl_rbmr_alltoall");
  NcclApi& N = nccl();
  const RPart& R = c->rp;
  const unsigned char* sr[3][2] = {{R.qs, R.qr}, {R.ps, R.pr}, {R.is, R.ir}};
  const uint64_t cb[3] = {R.qchunk, R.pchunk, R.ichunk};
  NC(N.GroupStart());
  for (uint32_t j = 0; j < R.G; ++j) {
    NC(N.Send(sr[a][0] + j * cb[a], cb[a], ncclUint8, (int)j, c->comm, s));
    NC(N.Recv(const_cast<unsigned char*>(sr[a][1]) + j * cb[a], cb[a], ncclUint8, (int)j, c->comm, s));
  }
  NC(N.GroupEnd());
  return RBM_OK;
}

// one step of the partitioned system with the library's exchanges
rbm_status part_step(rbm_ctx* c, cudaStream_t s) {
  if (c->cfg.scheme == RBM_SCHEME_RBMR) {
    for (int k = 1; k <= 4; ++k) {
      c->eng->rbmr_part_phase(*c, s, k);
      if (k < 4)
        if (rbm_status e = rbmr_exchange(c, s, k - 1)) return e;
    }
    CU(cudaGetLastError());
    return RBM_OK;
  }
  c->P.verlet_start = c->verlet_start ? 1u : 0u;
  if (!c->partitioned) {
    c->eng->part_prologue(*c, s);
    if (rbm_status e = part_exchange_cr(c, s)) return e;
  }
  c->eng->part_phase1(*c, s);
  if (rbm_status e = part_exchange_h(c, s)) return e;
  c->eng->part_phase2(*c, s);
  if (rbm_status e = part_exchange_cr(c, s)) return e;
  c->verlet_start = false;
  c->P.verlet_start = 0u;
  CU(cudaGetLastError());
  return RBM_OK;
}

}  // namespace rbmhost

extern "C" {

rbm_status rbm_get_nccl_unique_id(void* out128) {
  rbm_ctx* c = nullptr;
  if (!out128) return fail(c, RBM_ERR_INVALID_ARG, "out is NULL");
  NcclApi& N = nccl();
  if (!N.ok) return fail(c, RBM_ERR_NCCL, "%s", N.err.c_str());
  ncclUniqueId id;
  NC(N.GetUniqueId(&id));
  std::memcpy(out128, &id, sizeof id);
  return RBM_OK;
}

rbm_status rbm_workspace_size(const rbm_config* cfg, size_t* bytes) {
  rbm_status s = validate(cfg);
  if (s) return s;
  if (!bytes) return fail(nullptr, RBM_ERR_INVALID_ARG, "bytes is NULL");
  rbm_ctx tmp;
  tmp.cfg = *cfg;
  tmp.L = choose_layout(*cfg);
  Workspace ws;
  carve(tmp, ws);
  *bytes = ws.used;
  return RBM_OK;
}

}  // extern "C"

namespace rbmhost {
// the configuration-derived constants of DevParams (no device pointers)
void fill_params(const rbm_config& k, DevParams& P) {
  P = DevParams{};
  P.n = k.n;
  P.p = k.p;
  P.pdiv = make_fastdiv(k.p);
  P.nfull = (uint32_t)(k.n / k.p);
  P.rem = (uint32_t)(k.n % k.p);
  P.seed_lo = (uint32_t)k.seed;
  P.seed_hi = (uint32_t)(k.seed >> 32);
  for (int r = 0; r < 10; ++r) {
    P.rk[2 * r] = P.seed_lo + (uint32_t)r * 0x9E3779B9u;
    P.rk[2 * r + 1] = P.seed_hi + (uint32_t)r * 0xBB67AE85u;
  }
  P.rep_hi = k.replica << 8;
  P.potential = k.potential;
  P.constraint = k.constraint;
  P.has_noise = k.sigma > 0.0;
  P.kp0 = k.kparam[0];
  P.kp1 = k.kparam[1];
  P.beta = k.potential == RBM_V_HARMONIC ? k.vparam[0] : 0.0;
  P.dt = k.dt;
  P.sq = k.sigma * std::sqrt(k.dt);
  P.kp0f = (float)P.kp0; P.kp1f = (float)P.kp1; P.betaf = (float)P.beta;
  P.dtf = (float)P.dt; P.sqf = (float)P.sq;
  P.invp = 1.0 / (double)(k.p - 1);
  P.invpf = (float)P.invp;
  P.invp1 = 1.0 / (double)k.p;  // size p + 1
  P.invp1f = 1.0f / (float)k.p;
  const uint32_t r = (uint32_t)(k.n % k.p);
  P.invr = r >= 2 ? 1.0 / (double)(r - 1) : 0.0;
  P.invrf = r >= 2 ? 1.0f / (float)(r - 1) : 0.0f;
  P.geo_noise = k.noise == RBM_NOISE_GEOMETRIC ? 1u : 0u;
  P.closed_window = (k.kernel == RBM_K_BOUNDED_CONFIDENCE && k.kparam[2] != 0.0) ? 1u : 0u;
  P.verlet_start = (k.integrator == RBM_INTEG_VERLET && k.state_form == 0) ? 1u : 0u;
  P.half_s2dt = 0.5 * k.sigma * k.sigma * k.dt;
  P.lin_decay = std::exp(-2.0 * k.kparam[0] * k.dt);
  P.half_s2dtf = (float)P.half_s2dt;
  P.lin_decayf = (float)P.lin_decay;
  P.group = 0;
  if (k.p <= 32) { P.group = 1; while (P.group < k.p) P.group <<= 1; }
}

rbm_status init_impl(rbm_ctx* c, const rbm_config* cfg, void* wsp, size_t ws_bytes) {
  CU(cudaGetDevice(&c->device));
  int major = 0;
  CU(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, c->device));
  if (major != 10) return fail(c, RBM_ERR_UNSUPPORTED, "device is sm_%d0; librbm is built for sm_100a", major);
  Workspace ws;
  ws.base = reinterpret_cast<unsigned char*>(wsp);
  ws.size = ws_bytes;
  carve(*c, ws);
  c->ws_base = ws.base;
  c->eng.reset(make_engine(*cfg));
  if (!c->eng) return fail(c, RBM_ERR_UNKNOWN_KERNEL, "no engine for kernel %u, d=%u", cfg->kernel, cfg->d);
  DevParams& P = c->P;
  fill_params(*cfg, P);
  P.B = c->L.B; P.b1 = c->L.b1; P.b2 = c->L.b2; P.nbuckets = c->L.nbuckets; P.cap = c->L.cap;
  P.step = c->step_dev;
  P.nonfinite = c->nonfinite;
  P.capacity_err = c->capacity_err;
  P.big_claim = c->big_claim;
  P.SB = c->L.SB; P.idbits = c->L.idbits; P.lowbits = c->L.lowbits;
  P.big_scratch = c->big_scratch;
  P.nb1_loc_mask = ((1u << c->L.b1) >> c->L.g) - 1u;
  P.segk = c->L.segk;
  P.segmask = (1u << c->L.segk) - 1u;
  P.halo = (is_partitioned(*cfg) && cfg->rank > 0) ? 1u : 0u;
  P.side_key = (cfg->scheme == RBM_SCHEME_RBM1 && !rec_keyed(*cfg) && c->L.b2 > 0) ? 1u : 0u;
  P.jshift = 32u - c->L.idbits;
  if (std::getenv("RBM_PHASE_PROF")) {  // debug: per-phase cycles of the bucket kernel
    CU(cudaMalloc(&P.prof, 64 * 8));
    CU(cudaMemset(P.prof, 0, 64 * 8));
  }
  rbm_status s = c->eng->setup(*c);
  if (s) return s;
  CU(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
  cudaStream_t st = c->stream;
  c->step = cfg->step0;
  const unsigned long long clean = ~0ull;
  CU(cudaMemcpyAsync(c->step_dev, &c->step, 8, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(c->nonfinite, &clean, 8, cudaMemcpyHostToDevice, st));
  CU(cudaMemsetAsync(c->capacity_err, 0, 4, st));
  const uint32_t s0[2] = {0u, (uint32_t)cfg->n};
  if (c->L.B == 0) CU(cudaMemcpyAsync(c->S, s0, 8, cudaMemcpyHostToDevice, st));
  CU(cudaMemsetAsync(c->big_claim, 0, NBIG * 4, st));
  if (c->halo_recv) CU(cudaMemsetAsync(c->halo_recv, 0, 16, st));  // rank 0 never receives one
  c->verlet_start = cfg->integrator == RBM_INTEG_VERLET && cfg->state_form == 0;
  if (cfg->init != RBM_INIT_USER) c->eng->init_state(*c, st);
  CU(cudaGetLastError());
  CU(cudaStreamSynchronize(st));  // the host-side sources above live on this stack frame
  return RBM_OK;
}
}  // namespace rbmhost

extern "C" {

rbm_status rbm_init(const rbm_config* cfg, void* wsp, size_t ws_bytes, void* cuda_stream,
                    const void* nccl_unique_id, rbm_ctx** out) {
  rbm_status s = validate(cfg);
  if (s) return s;
  if (!out) return fail(nullptr, RBM_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (nccl_unique_id && cfg->world_size == 1)
    return fail(nullptr, RBM_ERR_INVALID_ARG, "nccl_unique_id given for world_size 1");
  size_t need = 0;
  rbm_workspace_size(cfg, &need);
  if (!wsp || ws_bytes < need || (reinterpret_cast<uintptr_t>(wsp) & 255))
    return fail(nullptr, RBM_ERR_WORKSPACE, "workspace %p of %zu B; need %zu B, 256-B aligned", wsp, ws_bytes, need);
  std::unique_ptr<rbm_ctx> c(new rbm_ctx());
  c->cfg = *cfg;
  c->L = choose_layout(*cfg);
  c->stream = reinterpret_cast<cudaStream_t>(cuda_stream);
  s = init_impl(c.get(), cfg, wsp, ws_bytes);
  if (!s && nccl_unique_id) {  // library-owned communicator: the exchanges run inside rbm_step / rbm_run
    NcclApi& N = nccl();
    if (!N.ok) {
      s = fail(c.get(), RBM_ERR_NCCL, "%s", N.err.c_str());
    } else {
      ncclUniqueId id;
      std::memcpy(&id, nccl_unique_id, sizeof id);
      const ncclResult_t r = N.CommInitRank(&c->comm, cfg->world_size, id, cfg->rank);
      if (r != ncclSuccess) {
        c->comm = nullptr;
        s = fail(c.get(), RBM_ERR_NCCL, "ncclCommInitRank(world %d, rank %d): %s", cfg->world_size, cfg->rank,
                 N.GetErrorString(r));
      }
    }
  }
  if (s) {
    g_err = c->err;
    if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
    return s;
  }
  *out = c.release();
  return RBM_OK;
}

rbm_status rbm_set_adjacency(rbm_ctx* c, const uint32_t* row_ptr, const uint32_t* col_idx, const double* val,
                             uint64_t nnz) {
  if (!c) return fail(nullptr, RBM_ERR_INVALID_ARG, "ctx is NULL");
  if (c->cfg.kernel != RBM_K_ADJACENCY) return fail(c, RBM_ERR_STATE, "not an adjacency-kernel context");
  if (!row_ptr || !col_idx || !val || nnz == 0 || nnz >= (1ull << 32))
    return fail(c, RBM_ERR_INVALID_ARG, "adjacency: NULL array or nnz=%llu not in 1..2^32-1", (unsigned long long)nnz);
  c->P.adj_rp = row_ptr;
  c->P.adj_ci = col_idx;
  c->P.adj_v = val;
  c->P.adj_nnz = nnz;
  c->P.adj_edges = c->cfg.kparam[2] != 0.0 ? 1u : 0u;
  for (int i = 0; i < 6; ++i)  // kernel parameters changed: recapture
    if (c->graph[i]) { cudaGraphExecDestroy(c->graph[i]); c->graph[i] = nullptr; }
  return RBM_OK;
}

rbm_status rbm_set_state(rbm_ctx* c, const void* x, uint32_t where) {
  if (!c) return fail(nullptr, RBM_ERR_INVALID_ARG, "ctx is NULL");
  if (!x) return fail(c, RBM_ERR_INVALID_ARG, "x is NULL");
  const size_t bytes = c->n0 * c->cfg.d * elt_size(c->cfg);  // this rank's ids (all N on one GPU)
  if (where == RBM_MEM_HOST) {
    void* scratch = c->recbuf[c->cur ^ 1];  // inactive buffer as staging
    CU(cudaMemcpyAsync(scratch, x, bytes, cudaMemcpyHostToDevice, c->stream));
    c->eng->set_state(*c, scratch, c->stream);
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(c->stream));
  } else if (where == RBM_MEM_DEVICE) {
    c->eng->set_state(*c, x, c->stream);
    CU(cudaGetLastError());
  } else {
    return fail(c, RBM_ERR_INVALID_ARG, "where=%u", where);
  }
  return RBM_OK;
}

static rbm_status not_partitioned(rbm_ctx* c) {
  if (c->cfg.kernel == RBM_K_ADJACENCY && !c->P.adj_rp)
    return fail(c, RBM_ERR_STATE, "adjacency kernel: call rbm_set_adjacency before stepping");
  if (is_partitioned(c->cfg) && !c->comm)
    return fail(c, RBM_ERR_STATE, "partitioned context (world_size %d) without a communicator: step with rbm_part_phase1/2 and the exchanges, or pass an NCCL id to rbm_init", c->cfg.world_size);
  return RBM_OK;
}

rbm_status rbm_step(rbm_ctx* c) {
  if (!c) return fail(nullptr, RBM_ERR_INVALID_ARG, "ctx is NULL");
  if (rbm_status e = not_partitioned(c)) return e;
  if (c->step + 1 >= (1ull << 32)) return fail(c, RBM_ERR_INVALID_ARG, "step index would exceed 2^32");
  if (is_partitioned(c->cfg)) {
    rbm_status s = part_step(c, c->stream);
    c->P.dbg_order = nullptr;
    if (s) return s;
    ++c->step;
    return RBM_OK;
  }
  rbm_status s = enqueue_steps(c, c->stream, 1);
  c->P.dbg_order = nullptr;
  if (s) return s;
  ++c->step;
  return RBM_OK;
}

rbm_status rbm_run(rbm_ctx* c, uint64_t nsteps) {
  if (!c) return fail(nullptr, RBM_ERR_INVALID_ARG, "ctx is NULL");
  Nvtx range_("rbm_run");
  if (rbm_status e = not_partitioned(c)) return e;
  if (c->step + nsteps >= (1ull << 32)) return fail(c, RBM_ERR_INVALID_ARG, "step index would exceed 2^32");
  // steps per graph: even when a step flips the ping-pong buffers
  c->P.dbg_order = nullptr;  // the permutation hook applies to rbm_step only
  const uint32_t per = 8;  // even: every layout returns to the same (cur, parity)
  c->graph_steps = per;
  uint64_t done = 0;
  if (is_partitioned(c->cfg)) {  // the library's exchanges, captured with the kernels when possible
    const bool first = c->cfg.scheme == RBM_SCHEME_RBM1 ? !c->partitioned : !c->aos_valid;
    if (first && nsteps > 0) {
      if (rbm_status e = part_step(c, c->stream)) return e;
      ++c->step;
      --nsteps;
    }
    if (nsteps >= per && !c->timing && !c->verlet_start) {
      const int slot = (int)(c->step & 1);
      if (!c->graph[slot] && !c->graph_failed) {
        const uint64_t step0 = c->step;
        bool ok = cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
        for (uint32_t i = 0; ok && i < per; ++i) { ok = part_step(c, c->cap_stream) == RBM_OK; ++c->step; }
        c->step = step0;
        cudaGraph_t g = nullptr;
        const bool ended = cudaStreamEndCapture(c->cap_stream, &g) == cudaSuccess && g;
        ok = ok && ended && cudaGraphInstantiate(&c->graph[slot], g, 0) == cudaSuccess;
        if (g) cudaGraphDestroy(g);
        if (!ok) {  // NCCL or the driver refused capture: eager steps from now on
          c->graph[slot] = nullptr;
          c->graph_failed = true;
          cudaGetLastError();
        }
      }
      if (c->graph[slot]) {
        const uint64_t reps = nsteps / per;
        for (uint64_t r = 0; r < reps; ++r) CU(cudaGraphLaunch(c->graph[slot], c->stream));
        done = reps * per;
      }
    }
    c->step += done;
    for (uint64_t i = done; i < nsteps; ++i) {
      if (rbm_status e = part_step(c, c->stream)) return e;
      ++c->step;
    }
    return RBM_OK;
  }
  if (c->cfg.scheme == RBM_SCHEME_RBM1 && c->L.B == 0) {  // resident: chunks of <= 4096 steps per launch
    while (nsteps > 0) {
      const uint32_t k = (uint32_t)std::min<uint64_t>(nsteps, 4096);
      c->P.verlet_start = c->verlet_start ? 1u : 0u;  // first step of this launch only
      c->eng->run_resident(*c, c->stream, k);
      c->verlet_start = false;
      c->P.verlet_start = 0u;
      CU(cudaGetLastError());
      c->step += k;
      nsteps -= k;
    }
    return RBM_OK;
  }
  const bool needs_prologue = (c->cfg.scheme == RBM_SCHEME_RBM1 && c->L.B > 0 && !c->partitioned) ||
                              (c->cfg.scheme != RBM_SCHEME_RBM1 && !c->aos_valid) || c->verlet_start;
  if (needs_prologue && nsteps > 0) {  // layout change of the state: first step outside the graphs
    rbm_status s0 = enqueue_steps(c, c->stream, 1);  // prologue step outside the graph
    if (s0) return s0;
    ++c->step;
    --nsteps;
  }
  if (nsteps >= per && !c->timing) {
    const int slot = (c->cur << 1) | (int)(c->step & 1);
    if (!c->graph[slot]) {
      const int cur0 = c->cur;
      CU(cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal));
      const uint64_t step0 = c->step;
      for (uint32_t i = 0; i < per; ++i) { c->eng->step(*c, c->cap_stream); ++c->step; }
      c->step = step0;
      cudaGraph_t g = nullptr;
      CU(cudaStreamEndCapture(c->cap_stream, &g));
      CU(cudaGraphInstantiate(&c->graph[slot], g, 0));
      cudaGraphDestroy(g);
      if (c->cur != cur0) return fail(c, RBM_ERR_STATE, "graph does not return the buffer parity");
    }
    const uint64_t reps = nsteps / per;
    for (uint64_t r = 0; r < reps; ++r) CU(cudaGraphLaunch(c->graph[slot], c->stream));
    done = reps * per;
  }
  c->step += done;
  for (uint64_t i = done; i < nsteps; ++i) {
    rbm_status s = enqueue_steps(c, c->stream, 1);
    if (s) return s;
    ++c->step;
  }
  return RBM_OK;
}

rbm_status rbm_gather(rbm_ctx* c, uint64_t id_begin, uint64_t id_end, void* x_out, uint32_t where) {
  if (!c) return fail(nullptr, RBM_ERR_INVALID_ARG, "ctx is NULL");
  if (!x_out) return fail(c, RBM_ERR_INVALID_ARG, "x_out is NULL");
  if (id_begin > id_end || id_end > c->cfg.n) return fail(c, RBM_ERR_INVALID_ARG, "bad id range [%llu,%llu)", (unsigned long long)id_begin, (unsigned long long)id_end);
  const size_t bytes = (id_end - id_begin) * c->cfg.d * elt_size(c->cfg);
  if (is_partitioned(c->cfg) && c->comm) {  // collective: every rank receives the whole id range
    void* dev = x_out;
    if (where == RBM_MEM_HOST) {
      CU(cudaMallocAsync(&dev, bytes ? bytes : 4, c->stream));
    }
    if (bytes) CU(cudaMemsetAsync(dev, 0, bytes, c->stream));
    c->eng->gather(*c, id_begin, id_end, dev, c->stream);
    CU(cudaGetLastError());
    // disjoint rows: every other rank contributes zero bits, so the integer sum is exact
    if (bytes) NC(nccl().AllReduce(dev, dev, bytes / 4, ncclUint32, ncclSum, c->comm, c->stream));
    if (where == RBM_MEM_HOST) {
      if (bytes) CU(cudaMemcpyAsync(x_out, dev, bytes, cudaMemcpyDeviceToHost, c->stream));
      CU(cudaFreeAsync(dev, c->stream));
    }
    CU(cudaStreamSynchronize(c->stream));
    return check_flags(c);
  }
  if (where == RBM_MEM_HOST && is_partitioned(c->cfg))
    return fail(c, RBM_ERR_UNSUPPORTED, "partitioned context without a communicator: gather to device memory (each rank writes the ids it holds), then combine across ranks");
  if (where == RBM_MEM_HOST) {
    void* scratch = c->recbuf[c->cur ^ 1];
    c->eng->gather(*c, id_begin, id_end, scratch, c->stream);
    CU(cudaGetLastError());
    if (bytes) CU(cudaMemcpyAsync(x_out, scratch, bytes, cudaMemcpyDeviceToHost, c->stream));
  } else if (where == RBM_MEM_DEVICE) {
    c->eng->gather(*c, id_begin, id_end, x_out, c->stream);
    CU(cudaGetLastError());
  } else {
    return fail(c, RBM_ERR_INVALID_ARG, "where=%u", where);
  }
  CU(cudaStreamSynchronize(c->stream));
  return check_flags(c);
}

rbm_status rbm_sync(rbm_ctx* c) {
  if (!c) return fail(nullptr, RBM_ERR_INVALID_ARG, "ctx is NULL");
  CU(cudaStreamSynchronize(c->stream));
  return check_flags(c);
}

uint64_t rbm_step_index(const rbm_ctx* c) { return c ? c->step : 0; }

uint32_t rbm_launches_per_step(const rbm_ctx* c) {
  if (!c) return 0;
  uint32_t k = 0;
  kernel_names(*c, &k);
  return k;
}

const char* rbm_kernel_name(const rbm_ctx* c, uint32_t i) {
  if (!c) return "";
  uint32_t k = 0;
  const char* const* names = kernel_names(*c, &k);
  return i < k ? names[i] : "";
}

rbm_status rbm_timing_begin(rbm_ctx* c, uint32_t max_steps) {
  if (!c) return fail(nullptr, RBM_ERR_INVALID_ARG, "ctx is NULL");
  for (cudaEvent_t e : c->ev) cudaEventDestroy(e);
  c->ev.clear();
  const size_t need = (size_t)max_steps * (rbm_launches_per_step(c) + 1);
  c->ev.resize(need);
  for (size_t i = 0; i < need; ++i) CU(cudaEventCreate(&c->ev[i]));
  c->ev_used = 0;
  c->timing = true;
  return RBM_OK;
}

rbm_status rbm_timing_end(rbm_ctx* c, double* ms_per_kernel, uint32_t* steps_recorded) {
  if (!c) return fail(nullptr, RBM_ERR_INVALID_ARG, "ctx is NULL");
  if (!c->timing) return fail(c, RBM_ERR_STATE, "timing was not begun");
  CU(cudaStreamSynchronize(c->stream));
  const uint32_t k = rbm_launches_per_step(c);
  const size_t per = k + 1;
  const uint32_t steps = (uint32_t)(c->ev_used / per);
  for (uint32_t j = 0; j < k; ++j) ms_per_kernel[j] = 0.0;
  for (uint32_t t = 0; t < steps; ++t)
    for (uint32_t j = 0; j < k; ++j) {
      float ms = 0.f;
      CU(cudaEventElapsedTime(&ms, c->ev[t * per + j], c->ev[t * per + j + 1]));
      ms_per_kernel[j] += ms;
    }
  if (steps_recorded) *steps_recorded = steps;
  c->timing = false;
  return RBM_OK;
}

rbm_status rbm_layout(const rbm_ctx* c, uint32_t* prefix_bits, uint32_t* passes, uint32_t* bucket_cap) {
  if (!c) return fail(nullptr, RBM_ERR_INVALID_ARG, "ctx is NULL");
  if (prefix_bits) *prefix_bits = c->L.B;
  if (passes) *passes = c->L.B == 0 ? 0 : (c->L.b2 ? 2 : 1);
  if (bucket_cap) *bucket_cap = c->L.cap;
  return RBM_OK;
}

rbm_status rbm_debug_permutation(rbm_ctx* c, uint32_t* order_out) {
  if (!c) return fail(nullptr, RBM_ERR_INVALID_ARG, "ctx is NULL");
  if (!order_out) return fail(c, RBM_ERR_INVALID_ARG, "order_out is NULL");
  if (c->cfg.scheme != RBM_SCHEME_RBM1) return fail(c, RBM_ERR_STATE, "not an RBM-1 context");
  c->P.dbg_order = order_out;  // consumed by the next rbm_step
  return RBM_OK;
}

rbm_status rbm_debug_slots(rbm_ctx* c, uint32_t* slots_out) {
  if (!c) return fail(nullptr, RBM_ERR_INVALID_ARG, "ctx is NULL");
  if (c->cfg.scheme == RBM_SCHEME_RBM1) return fail(c, RBM_ERR_STATE, "not an RBM-r context");
  if (!slots_out) return fail(c, RBM_ERR_INVALID_ARG, "slots_out is NULL");
  const uint64_t ns = is_partitioned(c->cfg) ? (c->rp.bb1 - c->rp.bb0) * c->cfg.p : c->nslots;  // own batches' slots
  if (c->cfg.scheme == RBM_SCHEME_RBMR && !is_partitioned(c->cfg)) {
    // the one-GPU Jacobi sweep does not store its draws: recompute those of the last step
    if (c->step == c->cfg.step0) return fail(c, RBM_ERR_STATE, "no step has run yet");
    c->eng->rbmr_slots(*c, (uint32_t)(c->step - 1), slots_out, c->stream);
    CU(cudaGetLastError());
    return RBM_OK;
  }
  CU(cudaMemcpyAsync(slots_out, c->js, ns * 4, cudaMemcpyDeviceToDevice, c->stream));
  return RBM_OK;
}

rbm_status rbm_debug_philox(const uint32_t* in, uint32_t* out, uint64_t count, void* cuda_stream) {
  rbm_ctx* c = nullptr;
  if (!in || !out) return fail(nullptr, RBM_ERR_INVALID_ARG, "NULL buffer");
  if (count) philox_test_kernel<<<grid_for(count, 256), 256, 0, (cudaStream_t)cuda_stream>>>(in, out, count);
  CU(cudaGetLastError());
  return RBM_OK;
}

// ------------------------------------------------ partitioned single system
rbm_status rbm_part_info_get(const rbm_config* cfg, rbm_part_info* out) {
  rbm_status s = validate(cfg);
  if (s) return s;
  if (!out) return fail(nullptr, RBM_ERR_INVALID_ARG, "out is NULL");
  if (!is_partitioned(*cfg)) return fail(nullptr, RBM_ERR_STATE, "world_size 1: no partition exchange");
  rbm_ctx tmp;
  tmp.cfg = *cfg;
  tmp.L = choose_layout(*cfg);
  Workspace ws;
  unsigned char* const base = reinterpret_cast<unsigned char*>(uintptr_t(1) << 44);  // sentinel
  ws.base = base;
  ws.dry = true;
  carve(tmp, ws);
  auto off = [&](const void* p) { return (uint64_t)(reinterpret_cast<const unsigned char*>(p) - base); };
  std::memset(out, 0, sizeof *out);
  out->ws_bytes = ws.used;
  out->world_size = (uint32_t)cfg->world_size;
  out->rank = (uint32_t)cfg->rank;
  out->nseg = tmp.L.nseg();
  out->narrays = 1;  // the state records (id, [key,] x), rec_bytes each
  out->chunk_elems = (uint64_t)(tmp.L.nseg() >> tmp.L.g) * tmp.L.cap1;
  out->send_off[0] = off(tmp.recbuf[1]);
  out->recv_off[0] = off(tmp.recbuf[2]);
  out->elem_bytes[0] = rec_bytes(*cfg);
  out->counts_send_off = off(tmp.counts_send);
  out->counts_all_off = off(tmp.counts_all);
  out->halo_send_off = off(tmp.halo_send);
  out->halo_recv_off = off(tmp.halo_recv);
  out->halo_bytes = 16 + (uint64_t)HALO_MAX * rec_bytes(*cfg);
  out->id0 = tmp.id0;
  out->n0 = tmp.n0;
  out->phases = 2;
  for (uint32_t a = 0; a < out->narrays; ++a) out->chunk_bytes[a] = out->chunk_elems * out->elem_bytes[a];
  if (cfg->scheme == RBM_SCHEME_RBMR) {  // requests, responses, increments
    const RPart& R = tmp.rp;
    out->phases = 4;
    out->nseg = 0;
    out->narrays = 3;
    out->chunk_elems = 0;
    const unsigned char* sr[3][2] = {{R.qs, R.qr}, {R.ps, R.pr}, {R.is, R.ir}};
    const uint64_t cb[3] = {R.qchunk, R.pchunk, R.ichunk};
    for (int a = 0; a < 3; ++a) {
      out->send_off[a] = off(sr[a][0]);
      out->recv_off[a] = off(sr[a][1]);
      out->elem_bytes[a] = 1;
      out->chunk_bytes[a] = cb[a];
    }
    out->halo_bytes = 0;
  }
  return RBM_OK;
}

static rbm_status rbmr_part_call(rbm_ctx* c, int phase) {
  if (phase < 1 || phase > 4) return fail(c, RBM_ERR_STATE, "RBM-r partitioned step: phases 1..4");
  if (phase == 4 && c->step + 1 >= (1ull << 32)) return fail(c, RBM_ERR_INVALID_ARG, "step index would exceed 2^32");
  c->eng->rbmr_part_phase(*c, c->stream, phase);
  if (phase == 4) ++c->step;
  CU(cudaGetLastError());
  return RBM_OK;
}

static rbm_status part_call(rbm_ctx* c, int phase) {
  if (!c) return fail(nullptr, RBM_ERR_INVALID_ARG, "ctx is NULL");
  if (!is_partitioned(c->cfg)) return fail(c, RBM_ERR_STATE, "not a partitioned context (world_size 1)");
  if (c->cfg.scheme == RBM_SCHEME_RBMR) return rbmr_part_call(c, phase);
  if (phase == 0 && c->partitioned) return fail(c, RBM_ERR_STATE, "prologue already done (state is partitioned)");
  if (phase > 0 && !c->partitioned) return fail(c, RBM_ERR_STATE, "run rbm_part_prologue and its exchange first");
  if (phase == 2 && c->step + 1 >= (1ull << 32)) return fail(c, RBM_ERR_INVALID_ARG, "step index would exceed 2^32");
  c->P.verlet_start = c->verlet_start ? 1u : 0u;  // both phases compute batches of this step
  if (phase == 0) c->eng->part_prologue(*c, c->stream);
  else if (phase == 1) c->eng->part_phase1(*c, c->stream);
  else {
    c->eng->part_phase2(*c, c->stream);
    c->verlet_start = false;
    c->P.dbg_order = nullptr;  // the permutation hook covers one step (phase1 + phase2)
    ++c->step;
  }
  CU(cudaGetLastError());
  return RBM_OK;
}

rbm_status rbm_part_set_peers(rbm_ctx* c, const uint64_t* peer_ws, uint32_t count) {
  if (!c) return fail(nullptr, RBM_ERR_INVALID_ARG, "ctx is NULL");
  if (!is_partitioned(c->cfg)) return fail(c, RBM_ERR_STATE, "not a partitioned context (world_size 1)");
  if (c->partitioned) return fail(c, RBM_ERR_STATE, "set the peers before rbm_part_prologue");
  if (!peer_ws || count != (uint32_t)c->cfg.world_size)
    return fail(c, RBM_ERR_INVALID_ARG, "need world_size=%d peer workspace pointers", c->cfg.world_size);
  if (count > (uint32_t)MAXG_FUSED)
    return fail(c, RBM_ERR_UNSUPPORTED, "fused exchange supports world_size <= %d (one NVSwitch node)", MAXG_FUSED);
  if (reinterpret_cast<unsigned char*>(peer_ws[c->cfg.rank]) != c->ws_base)
    return fail(c, RBM_ERR_INVALID_ARG, "peer_ws[rank] must be this context's own workspace");
  for (uint32_t j = 0; j < count; ++j) {
    if (!peer_ws[j] || (peer_ws[j] & 255)) return fail(c, RBM_ERR_INVALID_ARG, "peer workspace %u is NULL or misaligned", j);
    c->peer_base[j] = reinterpret_cast<unsigned char*>(peer_ws[j]);
  }
  c->fused = true;
  return RBM_OK;
}

rbm_status rbm_part_map_peers(rbm_ctx* c) {
  if (!c) return fail(nullptr, RBM_ERR_INVALID_ARG, "ctx is NULL");
  if (!c->comm) return fail(c, RBM_ERR_STATE, "no communicator: pass an NCCL id to rbm_init (or map the peers yourself and call rbm_part_set_peers)");
  if (c->partitioned) return fail(c, RBM_ERR_STATE, "map the peers before the first step");
  const int G = c->cfg.world_size, r = c->cfg.rank;
  if (G > MAXG_FUSED) return fail(c, RBM_ERR_UNSUPPORTED, "fused exchange supports world_size <= %d (one NVSwitch node)", MAXG_FUSED);
  NcclApi& N = nccl();
  struct Entry { cudaIpcMemHandle_t h; unsigned long long off; int ok; int pad; };
  static_assert(sizeof(Entry) <= 128, "IPC entry");
  Entry mine{};
  mine.ok = 0;
  unsigned long long base = 0;
  size_t sz = 0;
  if (N.MemGetAddressRange && N.MemGetAddressRange(&base, &sz, (unsigned long long)c->ws_base) == 0 &&
      cudaIpcGetMemHandle(&mine.h, reinterpret_cast<void*>(base)) == cudaSuccess) {
    mine.ok = 1;
    mine.off = (unsigned long long)c->ws_base - base;
  }
  cudaGetLastError();
  unsigned char* all = c->xchg;  // G entries of 128 B
  CU(cudaMemcpyAsync(all + (size_t)r * 128, &mine, sizeof mine, cudaMemcpyHostToDevice, c->stream));
  NC(N.AllGather(all + (size_t)r * 128, all, 128, ncclUint8, c->comm, c->stream));
  std::vector<unsigned char> host((size_t)G * 128);
  CU(cudaMemcpyAsync(host.data(), all, host.size(), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  int ok = 1;
  void* opened[MAXG_FUSED] = {};
  for (int j = 0; j < G; ++j) {
    Entry e;
    std::memcpy(&e, host.data() + (size_t)j * 128, sizeof e);
    if (!e.ok) { ok = 0; continue; }
    if (j == r) continue;
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, e.h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) { ok = 0; cudaGetLastError(); continue; }
    opened[j] = p;
    c->peer_base[j] = reinterpret_cast<unsigned char*>(p) + e.off;
  }
  // every rank switches, or none
  int* flag = reinterpret_cast<int*>(all);
  CU(cudaMemcpyAsync(flag, &ok, 4, cudaMemcpyHostToDevice, c->stream));
  NC(N.AllReduce(flag, flag, 1, ncclInt32, ncclMin, c->comm, c->stream));
  CU(cudaMemcpyAsync(&ok, flag, 4, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  if (!ok) {
    for (int j = 0; j < G; ++j)
      if (opened[j]) cudaIpcCloseMemHandle(opened[j]);
    return fail(c, RBM_ERR_UNSUPPORTED, "CUDA IPC mapping of the peers' workspaces failed on some rank; the NCCL all-to-all stays in use");
  }
  c->peer_base[r] = c->ws_base;
  for (int j = 0; j < G; ++j) c->ipc_open[j] = opened[j];
  c->fused = true;
  return RBM_OK;
}

rbm_status rbm_gather_local(rbm_ctx* c, uint32_t* ids_out, void* x_out, uint64_t* count) {
  if (!c) return fail(nullptr, RBM_ERR_INVALID_ARG, "ctx is NULL");
  if (!ids_out || !x_out || !count) return fail(c, RBM_ERR_INVALID_ARG, "NULL output");
  if (!is_partitioned(c->cfg)) {  // one GPU holds every id: written in id order
    c->eng->gather(*c, 0, c->cfg.n, x_out, c->stream);
    iota_kernel<<<grid_for(c->cfg.n, 256), 256, 0, c->stream>>>(ids_out, c->cfg.n);
    *count = c->cfg.n;
  } else {
    *count = c->eng->gather_local(*c, ids_out, x_out, c->stream);
  }
  CU(cudaGetLastError());
  CU(cudaStreamSynchronize(c->stream));
  return check_flags(c);
}

rbm_status rbm_part_prologue(rbm_ctx* c) { return part_call(c, 0); }
rbm_status rbm_part_phase1(rbm_ctx* c) { return part_call(c, 1); }
rbm_status rbm_part_phase2(rbm_ctx* c) { return part_call(c, 2); }
rbm_status rbm_part_phase(rbm_ctx* c, uint32_t k) {
  if (!c) return fail(nullptr, RBM_ERR_INVALID_ARG, "ctx is NULL");
  if (k == 0) return fail(c, RBM_ERR_INVALID_ARG, "phases are numbered from 1");
  return part_call(c, (int)k);
}

// --------------------------------------------- direct O(N^2) steps (f1)
static rbm_status direct_validate(const rbm_config* cfg, size_t elt_bytes_out[2]) {
  if (!cfg) return fail(nullptr, RBM_ERR_INVALID_ARG, "cfg is NULL");
  if (cfg->integrator == RBM_INTEG_SPLIT_EXACT_PAIR)
    return fail(nullptr, RBM_ERR_INVALID_ARG, "direct step: Euler-Maruyama or Verlet");
  if (cfg->n > (1ull << 24)) return fail(nullptr, RBM_ERR_INVALID_ARG, "direct step: n <= 2^24 (O(N^2) work)");
  rbm_config k = *cfg;  // the batch fields do not apply: validate the model only
  k.p = 2;
  k.scheme = RBM_SCHEME_RBM1;
  if (k.n < 2) k.n = 2;
  k.world_size = 1;
  k.rank = 0;
  k.debug_bucket_cap = 0;
  rbm_status s = validate(&k);
  if (s) return s;
  elt_bytes_out[0] = (size_t)cfg->n * cfg->d * elt_size(*cfg);  // ping-pong copy of x
  elt_bytes_out[1] = 256;                                       // flags
  return RBM_OK;
}

rbm_status rbm_direct_workspace_size(const rbm_config* cfg, size_t* bytes) {
  size_t b[2];
  rbm_status s = direct_validate(cfg, b);
  if (s) return s;
  if (!bytes) return fail(nullptr, RBM_ERR_INVALID_ARG, "bytes is NULL");
  *bytes = ((b[0] + 255) & ~size_t(255)) + b[1];
  return RBM_OK;
}

rbm_status rbm_direct_run(const rbm_config* cfg, void* x, uint64_t m0, uint64_t nsteps, void* ws,
                          size_t ws_bytes, void* stream) {
  size_t need = 0;
  rbm_status s = rbm_direct_workspace_size(cfg, &need);
  if (s) return s;
  if (!x || !ws || ws_bytes < need || (reinterpret_cast<uintptr_t>(ws) & 255))
    return fail(nullptr, RBM_ERR_WORKSPACE, "direct: x %p, workspace %p of %zu B (need %zu, 256-B aligned)", x, ws, ws_bytes, need);
  if (m0 + nsteps >= (1ull << 32)) return fail(nullptr, RBM_ERR_INVALID_ARG, "step index would exceed 2^32");
  std::unique_ptr<EngineBase> eng(make_engine(*cfg));
  if (!eng) return fail(nullptr, RBM_ERR_UNKNOWN_KERNEL, "no engine for kernel %u, d=%u", cfg->kernel, cfg->d);
  DevParams P;
  fill_params(*cfg, P);
  // Verlet (row f3): the start formula applies to the step with index step0
  // only, so run(a) followed by run(b) equals run(a + b)
  if (m0 != cfg->step0) P.verlet_start = 0u;
  size_t b[2];
  direct_validate(cfg, b);
  unsigned char* w = reinterpret_cast<unsigned char*>(ws);
  P.nonfinite = reinterpret_cast<unsigned long long*>(w + ((b[0] + 255) & ~size_t(255)));
  rbm_ctx* c = nullptr;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (nsteps) eng->direct(P, x, w, (uint32_t)cfg->n, (uint32_t)m0, (uint32_t)nsteps, st);
  CU(cudaGetLastError());
  return RBM_OK;
}

rbm_status rbm_direct_sync(const rbm_config* cfg, void* ws, void* stream) {
  size_t b[2];
  rbm_status s = direct_validate(cfg, b);
  if (s) return s;
  rbm_ctx* c = nullptr;
  unsigned long long nf = 0;
  const unsigned long long* flag = reinterpret_cast<const unsigned long long*>(
      reinterpret_cast<unsigned char*>(ws) + ((b[0] + 255) & ~size_t(255)));
  CU(cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream)));
  CU(cudaMemcpy(&nf, flag, 8, cudaMemcpyDeviceToHost));
  if (nf != ~0ull)
    return fail(nullptr, RBM_ERR_NONFINITE, "direct step: non-finite position at step %llu, particle id %llu",
                (unsigned long long)(nf >> 32), (unsigned long long)(nf & 0xffffffffull));
  return RBM_OK;
}

rbm_status rbm_direct_reset(const rbm_config* cfg, void* ws, void* stream) {
  size_t b[2];
  rbm_status s = direct_validate(cfg, b);
  if (s) return s;
  rbm_ctx* c = nullptr;
  CU(cudaMemsetAsync(reinterpret_cast<unsigned char*>(ws) + ((b[0] + 255) & ~size_t(255)), 0xff, 8,
                     reinterpret_cast<cudaStream_t>(stream)));
  return RBM_OK;
}

const char* rbm_last_error(const rbm_ctx* c) { return c ? c->err.c_str() : g_err.c_str(); }

rbm_status rbm_destroy(rbm_ctx* c) {
  if (!c) return RBM_OK;
  if (c->P.prof) {
    unsigned long long h[64];
    if (cudaMemcpy(h, c->P.prof, sizeof h, cudaMemcpyDeviceToHost) == cudaSuccess && h[63]) {
      std::fprintf(stderr, "RBM_PHASE_PROF bucket kernel, %llu CTAs, mean SM cycles per CTA:", h[63]);
      for (int i = 0; i < 16; ++i)
        if (h[i]) std::fprintf(stderr, " p%d=%.0f", i, (double)h[i] / (double)h[63]);
      std::fprintf(stderr, "\n");
    }
    if (cudaMemcpy(h, c->P.prof, sizeof h, cudaMemcpyDeviceToHost) == cudaSuccess && h[62]) {
      std::fprintf(stderr, "RBM_PHASE_PROF pass-2 splitter, %llu tiles, mean SM cycles per tile:", h[62]);
      for (int i = 16; i < 32; ++i)
        if (h[i]) std::fprintf(stderr, " s%d=%.0f", i, (double)h[i] / (double)h[62]);
      std::fprintf(stderr, "\n");
    }
    cudaFree(c->P.prof);
  }
  for (int i = 0; i < 6; ++i)
    if (c->graph[i]) cudaGraphExecDestroy(c->graph[i]);
  for (int j = 0; j < MAXG_FUSED; ++j)
    if (c->ipc_open[j]) cudaIpcCloseMemHandle(c->ipc_open[j]);
  if (c->comm) nccl().CommDestroy(c->comm);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  for (cudaEvent_t e : c->ev) cudaEventDestroy(e);
  delete c;
  return RBM_OK;
}

}  // extern "C"

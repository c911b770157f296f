// api.cu -- the C ABI declared in include/fmm.h: argument checking, pointer
// kind detection (host or device), stage orchestration on the library stream,
// per-phase CUDA-event timing, and the final combine + un-permute (a13).
#include <cmath>
#include <cstring>
#include <algorithm>
#include <new>

#include "ctx.cuh"

#define FMM_API extern "C" __attribute__((visibility("default")))

namespace fmmb {

void set_expansion_smem_limits();

namespace {

__global__ void k_finalize(const uint32_t* __restrict__ idx, int64_t n, int64_t off, int parts, const float* __restrict__ un,
                           const float* __restrict__ sn, const float* __restrict__ uf, const float* __restrict__ sf,
                           float* __restrict__ u, float* __restrict__ s) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t o = 3 * (int64_t)idx[i], g = 3 * (off + i);
    for (int d = 0; d < 3; ++d) {
      float uu = 0.f, ss = 0.f;
      if (parts & 1) { uu += un[g + d]; ss += sn[g + d]; }
      if (parts & 2) { uu += uf[g + d]; ss += sf[g + d]; }
      u[o + d] = uu;
      s[o + d] = ss;
    }
  }
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess) { cudaGetLastError(); return false; }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

float ms_between(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) { cudaGetLastError(); return 0.f; }
  return ms;
}

void check_config(const fmm_config& c) {
  if (c.struct_size != sizeof(fmm_config)) throw FmmError(FMM_E_ARG, "fmm_config.struct_size mismatch");
  if (c.order < 2 || c.order > kMaxOrder) throw FmmError(FMM_E_ARG, "order must be in [2, 16]");
  if (c.theta_num < 1 || c.theta_den > 64 || c.theta_num >= c.theta_den)
    throw FmmError(FMM_E_ARG, "theta must satisfy 1 <= num < den <= 64");
  if (c.ncrit < 1) throw FmmError(FMM_E_ARG, "ncrit must be >= 1");
  if (c.images < 0 || c.images > 6) throw FmmError(FMM_E_ARG, "images must be in [0, 6]");
  if (c.images > 0 && !(c.box_len > 0.0 && std::isfinite(c.box_len))) throw FmmError(FMM_E_ARG, "box_len must be > 0");
  if (c.traversal != 0 && c.traversal != 1) throw FmmError(FMM_E_ARG, "traversal must be 0 or 1");
  if (c.nranks < 1 || c.rank < 0 || c.rank >= c.nranks) throw FmmError(FMM_E_ARG, "bad rank/nranks");
  if (c.partition < 0 || c.partition > 2) throw FmmError(FMM_E_ARG, "partition must be 0, 1 or 2");
  if (c.nranks > 8) throw FmmError(FMM_E_ARG, "nranks must be <= 8 (one NVLink node)");
  if (c.nranks > 1 && c.images < 1) throw FmmError(FMM_E_ARG, "multi-GPU needs the periodic mode (images >= 1)");
  int tp = 1;
  for (int d = 0; d < 3; ++d) {
    if (c.tiles[d] != 1 && c.tiles[d] != 2) throw FmmError(FMM_E_ARG, "tiles[d] must be 1 or 2");
    tp *= c.tiles[d];
  }
  if (tp > 1 && c.images < 1) throw FmmError(FMM_E_ARG, "tiles need the periodic mode");
}

template <typename F>
fmm_status guard(Ctx* c, F f) {
  try {
    f();
    if (poison_mode()) {                      // debug mode: every call ends with the guard-zone check
      FMM_CUDA(cudaDeviceSynchronize());
      guard_check("after an API call");
    }
    return FMM_OK;
  } catch (const FmmError& e) {
    if (c) {
      c->err = e.what();
      if (e.code == FMM_E_CUDA || e.code == FMM_E_NCCL || e.code == FMM_E_INTERNAL) c->poisoned = true;
    }
    return e.code;
  } catch (const std::bad_alloc&) {
    if (c) c->err = "host allocation failed";
    return FMM_E_OOM;
  } catch (...) {
    if (c) { c->err = "unknown internal error"; c->poisoned = true; }
    return FMM_E_INTERNAL;
  }
}

void evaluate_impl(Ctx& c, int parts, float* u, float* s) {
  cudaStream_t st = c.stream;
  const bool multi = c.cfg.nranks > 1;
  const int64_t n = c.n;                      // this rank's particles (after an ORB redistribution)
  const int64_t nout = c.balanced ? c.n_caller : n;   // the caller's particles
  FMM_CUDA(cudaEventRecord(c.ev[PH_EVAL0], st));
  if (c.ntot == 0) {
    for (int p = PH_UP; p <= PH_FIN; ++p) FMM_CUDA(cudaEventRecord(c.ev[p], st));
    c.evaluated = true;
    return;
  }
  size_t ncoef = (size_t)std::max<int64_t>(c.ncells, 1) * 3 * c.nc;
  c.M.reserve(ncoef);
  c.Lc.reserve(ncoef);
  const int64_t N = std::max<int64_t>(n, 1);
  c.u_near.reserve(3 * N); c.s_near.reserve(3 * N); c.u_far.reserve(3 * N); c.s_far.reserve(3 * N);
  const bool overlap = !c.lists_valid;
  if (overlap) {
    // a5-a6 on the side stream while a7 (the traversal, with its host round
    // trips between frontier rounds) runs on the main stream; joined before M2L
    FMM_CUDA(cudaEventRecord(c.ev_fork, st));
    FMM_CUDA(cudaStreamWaitEvent(c.stream2, c.ev_fork, 0));
    std::swap(c.stream, c.stream2);
    try {
      upward_pass(c);
      FMM_CUDA(cudaEventRecord(c.ev[PH_UP], c.stream));
    } catch (...) {
      std::swap(c.stream, c.stream2);
      throw;
    }
    std::swap(c.stream, c.stream2);
  } else {
    upward_pass(c);
    FMM_CUDA(cudaEventRecord(c.ev[PH_UP], st));
  }
  if (multi) {
    // a14: the LET payload (multipoles of the sent cells, bodies) and the top
    // multipoles' all-reduce on the communication stream, as soon as the
    // upward pass is done; the traversal and the local-source near field run
    // meanwhile on the main stream ("the FMM kernels for the local tree are
    // evaluated while the LET data is being communicated")
    FMM_CUDA(cudaStreamWaitEvent(c.cstream, c.ev[PH_UP], 0));
    FMM_CUDA(cudaEventRecord(c.ev_let0, c.cstream));
    let_exchange(c, c.cstream);
    FMM_CUDA(cudaEventRecord(c.ev_let1, c.cstream));
  }
  if (overlap) {
    build_lists(c);
    FMM_CUDA(cudaEventRecord(c.ev_trav, st));
  }
  c.overlapped = overlap;
  FMM_CUDA(cudaEventRecord(c.ev[PH_TRAV], st));
  // no local leaf: nothing below writes the near/far buffers, so they are zero
  if (c.nleaves == 0)
    for (float* bp : {c.u_near.p, c.s_near.p, c.u_far.p, c.s_far.p}) FMM_CUDA(cudaMemsetAsync(bp, 0, sizeof(float) * 3 * N, st));
  if (multi) {
    // a12 with local sources while the LET is in flight
    p2p_pass(c, c.u_near.p, c.s_near.p, 1);
    FMM_CUDA(cudaEventRecord(c.ev_p2p_loc, st));
    FMM_CUDA(cudaStreamWaitEvent(st, c.ev_let1, 0));
  }
  FMM_CUDA(cudaStreamWaitEvent(st, c.ev[PH_UP], 0));
  cudaEvent_t ev_p2p_end = c.ev[PH_N];
  const int conc = multi ? 0 : c.concurrent;
  if (conc == 0) {
    FMM_CUDA(cudaEventRecord(c.ev[PH_P2P], st));     // (multi: start of the part after the LET)
    // a8 periodic far layers (beside the M2L on the side stream: they read only the
    // top multipoles and write their own partials) + a9 M2L, then the far reduction
    FMM_CUDA(cudaMemsetAsync(c.Lc.p, 0, ncoef * sizeof(float2), st));
    FMM_CUDA(cudaStreamWaitEvent(c.mstream, c.ev[PH_P2P], 0));
    std::swap(c.stream, c.mstream);
    try {
      periodic_far_pass(c, 1);
      FMM_CUDA(cudaEventRecord(c.ev_far, c.stream));
    } catch (...) {
      std::swap(c.stream, c.mstream);
      throw;
    }
    std::swap(c.stream, c.mstream);
    m2l_pass(c);
    FMM_CUDA(cudaStreamWaitEvent(st, c.ev_far, 0));
    periodic_far_pass(c, 2);
    FMM_CUDA(cudaEventRecord(c.ev[PH_M2L], st));
    // a12 (multi: the received sources' entries, added)
    p2p_pass(c, c.u_near.p, c.s_near.p, multi ? 2 : 0);
    FMM_CUDA(cudaEventRecord(c.ev[PH_N], st));
  } else {
    // the far field (a8-a9, tensor and CUDA cores) and the near field (a12, FP32
    // pipe) are independent: M2L on the high-priority side stream beside P2P
    FMM_CUDA(cudaEventRecord(c.ev_fork, st));
    FMM_CUDA(cudaStreamWaitEvent(c.mstream, c.ev_fork, 0));
    auto near = [&] {
      FMM_CUDA(cudaEventRecord(c.ev[PH_TRAV], st));
      p2p_pass(c, c.u_near.p, c.s_near.p, 0);
      FMM_CUDA(cudaEventRecord(c.ev[PH_N], st));
    };
    if (conc == 1) near();
    std::swap(c.stream, c.mstream);
    try {
      FMM_CUDA(cudaEventRecord(c.ev[PH_P2P], c.stream));
      FMM_CUDA(cudaMemsetAsync(c.Lc.p, 0, ncoef * sizeof(float2), c.stream));
      m2l_pass(c);
      periodic_far_pass(c);
      FMM_CUDA(cudaEventRecord(c.ev[PH_M2L], c.stream));
    } catch (...) {
      std::swap(c.stream, c.mstream);
      throw;
    }
    std::swap(c.stream, c.mstream);
    if (conc == 2) near();
    FMM_CUDA(cudaStreamWaitEvent(st, c.ev[PH_M2L], 0));
  }
  // a10-a11 downward pass
  downward_pass(c, c.u_far.p, c.s_far.p);
  FMM_CUDA(cudaEventRecord(c.ev[PH_DOWN], st));
  // a13 combine + un-permute into the caller's order
  bool hu = !is_device_ptr(u), hs = !is_device_ptr(s);
  float* du = u;
  float* ds = s;
  if (hu) { c.stage_u.reserve(3 * std::max<int64_t>(nout, 1)); du = c.stage_u.p; }
  if (hs) { c.stage_ds.reserve(3 * std::max<int64_t>(nout, 1)); ds = c.stage_ds.p; }
  unsigned g = nblocks(n, 256);
  if (g > 148 * 16) g = 148 * 16;
  if (c.balanced) {
    // this rank's particles in their (local) caller order, then back to the
    // ranks that passed them (the reverse of the ORB redistribution)
    c.loc_u.reserve(3 * N);
    c.loc_s.reserve(3 * N);
    if (n > 0) FMM_LAUNCH(c, k_finalize, g, 256, 0, c.idx.p, n, (int64_t)0, parts, c.u_near.p, c.s_near.p, c.u_far.p,
                          c.s_far.p, c.loc_u.p, c.loc_s.p);
    orb_return(c, c.loc_u.p, c.loc_s.p, du, ds);
  } else if (n > 0) {
    FMM_LAUNCH(c, k_finalize, g, 256, 0, c.idx.p, n, (int64_t)0, parts, c.u_near.p, c.s_near.p, c.u_far.p, c.s_far.p,
               du, ds);
  }
  FMM_LAUNCH_CHECK();
  if (hu && nout) FMM_CUDA(cudaMemcpyAsync(u, du, sizeof(float) * 3 * nout, cudaMemcpyDeviceToHost, st));
  if (hs && nout) FMM_CUDA(cudaMemcpyAsync(s, ds, sizeof(float) * 3 * nout, cudaMemcpyDeviceToHost, st));
  FMM_CUDA(cudaEventRecord(c.ev[PH_FIN], st));
  unsigned long long nnear = 0;
  if (c.nleaves > 0) FMM_CUDA(cudaMemcpyAsync(&nnear, c.dnear.p, sizeof(nnear), cudaMemcpyDeviceToHost, st));
  FMM_CUDA(cudaStreamSynchronize(st));
  c.p2p_near_pairs = (int64_t)nnear;
  c.evaluated = true;
  fmm_stats& S = c.stats;
  S.ms_upward = ms_between(c.ev[PH_EVAL0], c.ev[PH_UP]);
  // overlapped: both phases start at EVAL0 (ms_upward and ms_traverse then overlap in time)
  S.ms_traverse = c.overlapped ? ms_between(c.ev[PH_EVAL0], c.ev_trav) : 0.0;
  S.ms_m2l = ms_between(c.ev[PH_P2P], c.ev[PH_M2L]);
  S.ms_p2p = conc ? ms_between(c.ev[PH_TRAV], ev_p2p_end) : ms_between(c.ev[PH_M2L], ev_p2p_end);
  if (multi) {
    S.ms_p2p += ms_between(c.ev[PH_TRAV], c.ev_p2p_loc);
    c.ms_let = ms_between(c.ev_let0, c.ev_let1);
    // time the main stream waited for the LET after its local near field
    c.ms_let_exposed = std::max(0.0, (double)ms_between(c.ev_p2p_loc, c.ev[PH_P2P]));
  }
  S.ms_downward = conc ? 0.0 : ms_between(ev_p2p_end, c.ev[PH_DOWN]);
  S.ms_finalize = ms_between(c.ev[PH_DOWN], c.ev[PH_FIN]);
  S.ms_eval_total = ms_between(c.ev[PH_EVAL0], c.ev[PH_FIN]);
  S.ms_m2l_tc = c.nm2l ? ms_between(c.ev_m2l[0], c.ev_m2l[1]) : 0.0;
  S.ms_m2l_reg = c.nm2l ? ms_between(c.ev_m2l[1], c.ev_m2l[2]) : 0.0;
}

}  // namespace
}  // namespace fmmb

using namespace fmmb;

FMM_API void fmm_config_default(fmm_config* cfg) {
  if (!cfg) return;
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->struct_size = sizeof(fmm_config);
  cfg->order = 10;
  cfg->theta_num = 1;
  cfg->theta_den = 2;
  cfg->ncrit = 64;
  cfg->images = 3;
  cfg->box_lo[0] = cfg->box_lo[1] = cfg->box_lo[2] = -kPi;
  cfg->box_len = 2.0 * kPi;
  cfg->traversal = 0;
  cfg->device = 0;
  cfg->stream = nullptr;
  cfg->rank = 0;
  cfg->nranks = 1;
  cfg->nccl_id = nullptr;
  cfg->tiles[0] = cfg->tiles[1] = cfg->tiles[2] = 1;
  cfg->m2l_path = 0;
  cfg->partition = 0;
}

FMM_API fmm_status fmm_create(const fmm_config* cfg, fmm_ctx** out) {
  if (!out) return FMM_E_ARG;
  *out = nullptr;
  if (!cfg) return FMM_E_ARG;
  fmm_ctx* h = new (std::nothrow) fmm_ctx;
  if (!h) return FMM_E_OOM;
  Ctx& c = h->c;
  fmm_status st = guard(&c, [&] {
    check_config(*cfg);
    c.cfg = *cfg;
    c.P = cfg->order;
    c.nc = c.P * (c.P + 1) / 2;
    c.tmax = 1;
    for (int d = 0; d < 3; ++d) c.tmax = std::max(c.tmax, (int)cfg->tiles[d]);
    for (int d = 0; d < 3; ++d) {
      c.per[d] = cfg->tiles[d] * cfg->box_len;
      c.per_units[d] = (1ll << 22) / c.tmax * cfg->tiles[d];
    }
    FMM_CUDA(cudaSetDevice(cfg->device));
    if (cfg->stream) {
      c.stream = (cudaStream_t)cfg->stream;
    } else {
      // blocking: ordered with the legacy default stream, so caller work queued
      // there (e.g. torch's default stream) completes before the library reads
      // its inputs, and the library's writes precede later default-stream work
      FMM_CUDA(cudaStreamCreate(&c.stream));
      c.own_stream = true;
    }
    for (int i = 0; i <= PH_N; ++i) FMM_CUDA(cudaEventCreate(&c.ev[i]));
    // side stream: the upward pass runs beside the traversal (they are independent)
    FMM_CUDA(cudaStreamCreateWithFlags(&c.stream2, cudaStreamNonBlocking));
    {
      int lo = 0, hi = 0;
      FMM_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      FMM_CUDA(cudaStreamCreateWithPriority(&c.mstream, cudaStreamNonBlocking, hi));
      const char* e = getenv("FMM_CONCURRENT");
      c.concurrent = e ? atoi(e) : 0;
    }
    if (cfg->nranks > 1) {
      FMM_CUDA(cudaStreamCreateWithFlags(&c.cstream, cudaStreamNonBlocking));
      for (cudaEvent_t* e : {&c.ev_let0, &c.ev_let1, &c.ev_p2p_loc}) FMM_CUDA(cudaEventCreate(e));
    }
    FMM_CUDA(cudaEventCreateWithFlags(&c.ev_fork, cudaEventDisableTiming));
    FMM_CUDA(cudaEventCreate(&c.ev_trav));
    for (auto& e : c.ev_m2l) FMM_CUDA(cudaEventCreate(&e));
    FMM_CUDA(cudaEventCreateWithFlags(&c.ev_far, cudaEventDisableTiming));
    set_expansion_smem_limits();
    FMM_CUDA(cudaGetLastError());
    comm_init(c);
  });
  if (st != FMM_OK) { delete h; return st; }
  *out = h;
  return FMM_OK;
}

FMM_API fmm_status fmm_destroy(fmm_ctx* h) {
  if (!h) return FMM_E_ARG;
  Ctx& c = h->c;
  cudaSetDevice(c.cfg.device);
  if (c.stream) cudaStreamSynchronize(c.stream);
  if (c.stream2) cudaStreamSynchronize(c.stream2);
  if (c.cstream) cudaStreamSynchronize(c.cstream);
  if (c.mstream) { cudaStreamSynchronize(c.mstream); cudaStreamDestroy(c.mstream); }
  for (cudaEvent_t e : {c.ev_let0, c.ev_let1, c.ev_p2p_loc}) if (e) cudaEventDestroy(e);
  if (c.cstream) cudaStreamDestroy(c.cstream);
  for (int i = 0; i <= PH_N; ++i) if (c.ev[i]) cudaEventDestroy(c.ev[i]);
  if (c.ev_fork) cudaEventDestroy(c.ev_fork);
  if (c.ev_trav) cudaEventDestroy(c.ev_trav);
  for (auto e : c.ev_m2l) if (e) cudaEventDestroy(e);
  if (c.ev_far) cudaEventDestroy(c.ev_far);
  if (c.stream2) cudaStreamDestroy(c.stream2);
  try { comm_destroy(c); } catch (...) {}
  if (c.own_stream && c.stream) cudaStreamDestroy(c.stream);
  delete h;
  return FMM_OK;
}

FMM_API const char* fmm_last_error(const fmm_ctx* h) { return h ? h->c.err.c_str() : "null context"; }

FMM_API fmm_status fmm_set_particles(fmm_ctx* h, int64_t n, const float* x, const float* alpha, const float* sigma) {
  if (!h) return FMM_E_ARG;
  Ctx& c = h->c;
  if (c.poisoned) return FMM_E_STATE;
  return guard(&c, [&] {
    if (n < 0) throw FmmError(FMM_E_ARG, "n < 0");
    if (n > 0 && (!x || !alpha || !sigma)) throw FmmError(FMM_E_ARG, "null array with n > 0");
    if (n >= (1ll << 31)) throw FmmError(FMM_E_ARG, "n >= 2^31");
    FMM_CUDA(cudaSetDevice(c.cfg.device));
    const float *dx = x, *da = alpha, *ds = sigma;
    if (n > 0) {
      if (!is_device_ptr(x)) {
        c.stage_x.reserve(3 * n);
        FMM_CUDA(cudaMemcpyAsync(c.stage_x.p, x, sizeof(float) * 3 * n, cudaMemcpyHostToDevice, c.stream));
        dx = c.stage_x.p;
      }
      if (!is_device_ptr(alpha)) {
        c.stage_a.reserve(3 * n);
        FMM_CUDA(cudaMemcpyAsync(c.stage_a.p, alpha, sizeof(float) * 3 * n, cudaMemcpyHostToDevice, c.stream));
        da = c.stage_a.p;
      }
      if (!is_device_ptr(sigma)) {
        c.stage_s.reserve(n);
        FMM_CUDA(cudaMemcpyAsync(c.stage_s.p, sigma, sizeof(float) * n, cudaMemcpyHostToDevice, c.stream));
        ds = c.stage_s.p;
      }
    }
    set_particles_impl(c, n, dx, da, ds);
    fmm_stats& S = c.stats;
    S.ms_keys = ms_between(c.ev[PH_SET0], c.ev[PH_KEYS]);
    S.ms_sort = ms_between(c.ev[PH_KEYS], c.ev[PH_SORT]);
    S.ms_tree = ms_between(c.ev[PH_SORT], c.ev[PH_TREE]);
    S.ms_set_total = ms_between(c.ev[PH_SET0], c.ev[PH_TREE]);
  });
}

FMM_API fmm_status fmm_evaluate_parts(fmm_ctx* h, int32_t parts, float* u, float* s) {
  if (!h) return FMM_E_ARG;
  Ctx& c = h->c;
  if (c.poisoned) return FMM_E_STATE;
  return guard(&c, [&] {
    if (!c.have_particles) throw FmmError(FMM_E_STATE, "evaluate before set_particles");
    if (c.n > 0 && (!u || !s)) throw FmmError(FMM_E_ARG, "null output with n > 0");
    if (parts < 1 || parts > 3) throw FmmError(FMM_E_ARG, "parts must be 1, 2 or 3");
    FMM_CUDA(cudaSetDevice(c.cfg.device));
    evaluate_impl(c, parts, u, s);
  });
}

FMM_API fmm_status fmm_evaluate(fmm_ctx* h, float* u, float* s) { return fmm_evaluate_parts(h, 3, u, s); }

FMM_API int32_t fmm_debug_mode(void) { return poison_mode() ? 1 : 0; }

FMM_API fmm_status fmm_get_stats(const fmm_ctx* h, fmm_stats* s) {
  if (!h || !s) return FMM_E_ARG;
  const Ctx& c = h->c;
  *s = c.stats;
  s->struct_size = sizeof(fmm_stats);
  s->n = c.n;
  s->ncells = c.ncells;
  s->nleaves = c.nleaves;
  s->nlevels = c.level_begin.empty() ? 0 : (int64_t)c.level_begin.size() - 1;
  s->p2p_list = c.np2p;
  s->m2l_list = c.nm2l;
  s->m2l_tc_list = c.tc_entries;
  s->m2l_reg_list = c.nm2lr;
  s->p2p_pairs = c.p2p_pairs;
  s->far_m2l = c.far_m2l;
  s->model_flops = 174.0 * (double)c.p2p_pairs;
  s->launches = c.launches;
  s->p2p_near_pairs = c.p2p_near_pairs;
  s->ntot = c.ntot;
  s->own_begin = c.off;
  s->own_count = c.nown;
  s->redist_bytes = c.redist_bytes;
  s->let_bytes_sent = c.let_bytes_sent;
  s->let_bytes_recv = c.let_bytes_recv;
  s->let_cells = c.let_cells;
  s->let_leaves = c.let_leaves;
  s->ms_let = c.ms_let;
  s->ms_let_exposed = c.ms_let_exposed;
  s->let_fallback = c.let_fallback;
  s->nranks = c.cfg.nranks;
  s->ncells_local = c.nloc_cells;
  s->cub_calls = c.cub_calls;
  return FMM_OK;
}

FMM_API fmm_status fmm_get_sizes(fmm_ctx* h, int64_t* ncells, int64_t* np2p, int64_t* nm2l) {
  if (!h) return FMM_E_ARG;
  Ctx& c = h->c;
  if (c.poisoned) return FMM_E_STATE;
  return guard(&c, [&] {
    if (!c.have_particles) throw FmmError(FMM_E_STATE, "no particles");
    FMM_CUDA(cudaSetDevice(c.cfg.device));
    if (!c.lists_valid) build_lists(c);
    if (ncells) *ncells = c.ncells;
    if (np2p) *np2p = c.np2p;
    if (nm2l) *nm2l = c.nm2l;
  });
}

FMM_API fmm_status fmm_get_box(const fmm_ctx* h, double* lo, double* L) {
  if (!h || !lo || !L) return FMM_E_ARG;
  for (int d = 0; d < 3; ++d) lo[d] = h->c.lo[d];
  *L = h->c.L;
  return FMM_OK;
}

FMM_API fmm_status fmm_get_keys(const fmm_ctx* h, uint64_t* keys, int64_t* perm) {
  if (!h) return FMM_E_ARG;
  Ctx& c = const_cast<Ctx&>(h->c);
  return guard(&c, [&] {
    if (!c.have_particles) throw FmmError(FMM_E_STATE, "no particles");
    if (c.n == 0) return;
    std::vector<uint32_t> idx(c.n);
    const uint64_t* kp = c.keys.p;
    if (keys) FMM_CUDA(cudaMemcpy(keys, kp, sizeof(uint64_t) * c.n, cudaMemcpyDeviceToHost));
    FMM_CUDA(cudaMemcpy(idx.data(), c.idx.p, sizeof(uint32_t) * c.n, cudaMemcpyDeviceToHost));
    if (perm) for (int64_t i = 0; i < c.n; ++i) perm[i] = idx[i];
  });
}

FMM_API fmm_status fmm_get_cells(const fmm_ctx* h, int64_t* out) {
  if (!h || !out) return FMM_E_ARG;
  Ctx& c = const_cast<Ctx&>(h->c);
  return guard(&c, [&] {
    if (!c.have_particles) throw FmmError(FMM_E_STATE, "no particles");
    int64_t nc = c.ncells;
    std::vector<int> buf(nc);
    DBuf<int>* cols[10] = {&c.cells.level, &c.cells.qx, &c.cells.qy, &c.cells.qz, &c.cells.begin,
                           &c.cells.count, &c.cells.parent, &c.cells.child_begin, &c.cells.nchild, &c.cells.leaf};
    for (int k = 0; k < 10; ++k) {
      if (nc) FMM_CUDA(cudaMemcpy(buf.data(), cols[k]->p, sizeof(int) * nc, cudaMemcpyDeviceToHost));
      for (int64_t i = 0; i < nc; ++i) out[10 * i + k] = buf[i];
    }
  });
}

FMM_API fmm_status fmm_get_lists(fmm_ctx* h, int64_t* p2p, int64_t* m2l) {
  if (!h) return FMM_E_ARG;
  Ctx& c = h->c;
  if (c.poisoned) return FMM_E_STATE;
  return guard(&c, [&] {
    if (!c.have_particles) throw FmmError(FMM_E_STATE, "no particles");
    if (!c.lists_valid) build_lists(c);
    auto dump = [&](const DBuf<uint64_t>& L, int64_t n, int64_t* out) {
      if (!out || n == 0) return;
      std::vector<uint64_t> v(n);
      FMM_CUDA(cudaMemcpy(v.data(), L.p, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost));
      std::sort(v.begin(), v.end());   // canonical (target, source, image) order (Z20)
      for (int64_t i = 0; i < n; ++i) {
        out[3 * i] = (int64_t)(v[i] >> 32);
        out[3 * i + 1] = (int64_t)((v[i] >> 5) & 0x7ffffff);
        out[3 * i + 2] = (int64_t)(v[i] & 31);
      }
    };
    dump(c.p2p, c.np2p, p2p);
    dump(c.m2l, c.nm2l, m2l);
  });
}

FMM_API fmm_status fmm_get_expansions(const fmm_ctx* h, float* M, float* L) {
  if (!h) return FMM_E_ARG;
  Ctx& c = const_cast<Ctx&>(h->c);
  return guard(&c, [&] {
    if (!c.evaluated) throw FmmError(FMM_E_STATE, "no evaluation yet");
    size_t bytes = sizeof(float2) * (size_t)c.ncells * 3 * c.nc;
    if (M && bytes) FMM_CUDA(cudaMemcpy(M, c.M.p, bytes, cudaMemcpyDeviceToHost));
    if (L && bytes) FMM_CUDA(cudaMemcpy(L, c.Lc.p, bytes, cudaMemcpyDeviceToHost));
  });
}

FMM_API fmm_status fmm_eval_cutoff(fmm_ctx* h, int64_t n, const float* rho, float* g) {
  if (!h) return FMM_E_ARG;
  Ctx& c = h->c;
  if (c.poisoned) return FMM_E_STATE;
  return guard(&c, [&] {
    if (n < 0 || (n > 0 && (!rho || !g))) throw FmmError(FMM_E_ARG, "bad arguments");
    if (n == 0) return;
    FMM_CUDA(cudaSetDevice(c.cfg.device));
    c.stage_u.reserve(n);
    c.stage_ds.reserve(n);
    FMM_CUDA(cudaMemcpyAsync(c.stage_u.p, rho, sizeof(float) * n, cudaMemcpyDefault, c.stream));
    eval_cutoff(c, c.stage_u.p, n, c.stage_ds.p);
    FMM_CUDA(cudaMemcpyAsync(g, c.stage_ds.p, sizeof(float) * n, cudaMemcpyDefault, c.stream));
    FMM_CUDA(cudaStreamSynchronize(c.stream));
  });
}

FMM_API fmm_status fmm_eval_pair_kernel(fmm_ctx* h, int64_t n, const float* rho, int32_t branch, float* g,
                                        float* rho_gp) {
  if (!h) return FMM_E_ARG;
  Ctx& c = h->c;
  if (c.poisoned) return FMM_E_STATE;
  return guard(&c, [&] {
    if (n < 0 || (n > 0 && (!rho || !g || !rho_gp)) || branch < 0 || branch > 1)
      throw FmmError(FMM_E_ARG, "bad arguments");
    if (n == 0) return;
    FMM_CUDA(cudaSetDevice(c.cfg.device));
    c.stage_u.reserve(3 * n);
    c.stage_ds.reserve(3 * n);
    float* dr = c.stage_u.p;
    float* dg = c.stage_ds.p;
    float* dp = c.stage_ds.p + n;
    FMM_CUDA(cudaMemcpyAsync(dr, rho, sizeof(float) * n, cudaMemcpyDefault, c.stream));
    eval_pair_kernel(c, dr, n, branch, dg, dp);
    FMM_CUDA(cudaMemcpyAsync(g, dg, sizeof(float) * n, cudaMemcpyDefault, c.stream));
    FMM_CUDA(cudaMemcpyAsync(rho_gp, dp, sizeof(float) * n, cudaMemcpyDefault, c.stream));
    FMM_CUDA(cudaStreamSynchronize(c.stream));
  });
}

FMM_API fmm_status fmm_comm_unique_id(void* id) {
  if (!id) return FMM_E_ARG;
  try {
    comm_unique_id(id);
    return FMM_OK;
  } catch (const FmmError& e) {
    return e.code;
  } catch (...) {
    return FMM_E_INTERNAL;
  }
}

FMM_API fmm_status fmm_step(fmm_ctx* h, int64_t n, float* x, float* alpha, float* sigma, double dt, double nu) {
  if (!h) return FMM_E_ARG;
  Ctx& c = h->c;
  if (c.poisoned) return FMM_E_STATE;
  return guard(&c, [&] {
    if (n < 0 || (n > 0 && (!x || !alpha || !sigma))) throw FmmError(FMM_E_ARG, "bad arguments");
    if (!(dt > 0.0) || !(nu >= 0.0) || !std::isfinite(dt) || !std::isfinite(nu)) throw FmmError(FMM_E_ARG, "need dt > 0, nu >= 0");
    FMM_CUDA(cudaSetDevice(c.cfg.device));
    cudaStream_t st = c.stream;
    c.st_x.reserve(3 * n); c.st_a.reserve(3 * n); c.st_s.reserve(n);
    c.st_u.reserve(3 * n); c.st_da.reserve(3 * n);
    c.st_xh.reserve(3 * n); c.st_ah.reserve(3 * n); c.st_sh.reserve(n);
    if (n > 0) {
      FMM_CUDA(cudaMemcpyAsync(c.st_x.p, x, sizeof(float) * 3 * n, cudaMemcpyDefault, st));
      FMM_CUDA(cudaMemcpyAsync(c.st_a.p, alpha, sizeof(float) * 3 * n, cudaMemcpyDefault, st));
      FMM_CUDA(cudaMemcpyAsync(c.st_s.p, sigma, sizeof(float) * n, cudaMemcpyDefault, st));
    }
    // stage 1 at t
    set_particles_impl(c, n, c.st_x.p, c.st_a.p, c.st_s.p);
    evaluate_impl(c, 3, c.st_u.p, c.st_da.p);
    step_stage_update(c, c.st_x.p, c.st_a.p, c.st_s.p, c.st_u.p, c.st_da.p, n, 0.5 * dt, nu * dt, c.st_xh.p,
                      c.st_ah.p, c.st_sh.p);
    // stage 2 at t + dt/2 (several GPUs: the particles move to the owners of the
    // stage-1 ORB domains -- the partition is reused)
    c.orb_reuse_next = true;
    set_particles_impl(c, n, c.st_xh.p, c.st_ah.p, c.st_sh.p);
    evaluate_impl(c, 3, c.st_u.p, c.st_da.p);
    // x' = x + dt u(t+dt/2), alpha' = alpha + dt dalpha/dt(t+dt/2), sigma'^2 = sigma^2 + 2 nu dt (Eq. 4)
    step_stage_update(c, c.st_x.p, c.st_a.p, c.st_s.p, c.st_u.p, c.st_da.p, n, dt, 2.0 * nu * dt, c.st_xh.p,
                      c.st_ah.p, c.st_sh.p);
    if (n > 0) {
      FMM_CUDA(cudaMemcpyAsync(x, c.st_xh.p, sizeof(float) * 3 * n, cudaMemcpyDefault, st));
      FMM_CUDA(cudaMemcpyAsync(alpha, c.st_ah.p, sizeof(float) * 3 * n, cudaMemcpyDefault, st));
      FMM_CUDA(cudaMemcpyAsync(sigma, c.st_sh.p, sizeof(float) * n, cudaMemcpyDefault, st));
    }
    FMM_CUDA(cudaStreamSynchronize(st));
  });
}

FMM_API fmm_status fmm_rbf_reinit(fmm_ctx* h, int64_t n, const float* x, const float* alpha, const float* sigma,
                                  int64_t m, const float* y, float sigma0, double tol, int32_t maxit, float* beta,
                                  int32_t* iters, double* resid) {
  if (!h) return FMM_E_ARG;
  Ctx& c = h->c;
  if (c.poisoned) return FMM_E_STATE;
  int it = 0;
  double res = 0.0;
  fmm_status st = guard(&c, [&] {
    if (n < 0 || m < 1 || (n > 0 && (!x || !alpha || !sigma)) || !y || !beta)
      throw FmmError(FMM_E_ARG, "bad arguments");
    if (!(sigma0 > 0.0f) || !std::isfinite(sigma0)) throw FmmError(FMM_E_SIGMA, "sigma0 must be > 0");
    if (!(tol > 0.0) || maxit < 1) throw FmmError(FMM_E_ARG, "tol must be > 0 and maxit >= 1");
    if (c.cfg.nranks > 1) throw FmmError(FMM_E_ARG, "fmm_rbf_reinit is single-GPU in this build");
    FMM_CUDA(cudaSetDevice(c.cfg.device));
    rbf_reinit_impl(c, n, x, alpha, sigma, m, y, sigma0, tol, (int)maxit, beta, &it, &res);
  });
  if (iters) *iters = it;
  if (resid) *resid = res;
  if (st == FMM_OK && res > tol) {
    c.err = "fmm_rbf_reinit: no convergence in maxit iterations (relative residual above tol)";
    return FMM_E_NOCONV;
  }
  return st;
}

FMM_API fmm_status fmm_evaluate_targets(fmm_ctx* h, int64_t n, const float* x, const float* alpha, const float* sigma,
                                        int64_t nt, const float* y, float* u) {
  if (!h) return FMM_E_ARG;
  Ctx& c = h->c;
  if (c.poisoned) return FMM_E_STATE;
  return guard(&c, [&] {
    if (n < 0 || nt < 0 || (n > 0 && (!x || !alpha || !sigma)) || (nt > 0 && (!y || !u)))
      throw FmmError(FMM_E_ARG, "bad arguments");
    if (c.cfg.nranks > 1) throw FmmError(FMM_E_ARG, "fmm_evaluate_targets is single-GPU in this build");
    FMM_CUDA(cudaSetDevice(c.cfg.device));
    cudaStream_t st = c.stream;
    const int64_t N = n + nt;
    c.st_x.reserve(3 * N); c.st_a.reserve(3 * N); c.st_s.reserve(N);
    c.st_u.reserve(3 * N); c.st_da.reserve(3 * N);
    // the union: sources as given, targets with zero strength (they add nothing to any
    // sum; their core size is irrelevant and set to 1)
    if (n > 0) {
      FMM_CUDA(cudaMemcpyAsync(c.st_x.p, x, sizeof(float) * 3 * n, cudaMemcpyDefault, st));
      FMM_CUDA(cudaMemcpyAsync(c.st_a.p, alpha, sizeof(float) * 3 * n, cudaMemcpyDefault, st));
      FMM_CUDA(cudaMemcpyAsync(c.st_s.p, sigma, sizeof(float) * n, cudaMemcpyDefault, st));
    }
    if (nt > 0) {
      FMM_CUDA(cudaMemcpyAsync(c.st_x.p + 3 * n, y, sizeof(float) * 3 * nt, cudaMemcpyDefault, st));
      FMM_CUDA(cudaMemsetAsync(c.st_a.p + 3 * n, 0, sizeof(float) * 3 * nt, st));
      fill_f32(c, c.st_s.p + n, nt, 1.0f);
    }
    set_particles_impl(c, N, c.st_x.p, c.st_a.p, c.st_s.p);
    evaluate_impl(c, 3, c.st_u.p, c.st_da.p);
    if (nt > 0) FMM_CUDA(cudaMemcpyAsync(u, c.st_u.p + 3 * n, sizeof(float) * 3 * nt, cudaMemcpyDefault, st));
    FMM_CUDA(cudaStreamSynchronize(st));
  });
}

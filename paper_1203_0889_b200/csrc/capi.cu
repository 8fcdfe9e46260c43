// capi.cu — the extern "C" boundary (include/fmm_b200.h). Converts internal errors to
// fmm_status codes + messages, owns the stage sequence of fmm_evaluate (engine.cpp:69-106)
// and the CUDA-event stage timing (RunResult's t_build/t_upward/t_traversal/t_downward,
// engine.hpp:38-49, measured on the device).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "context.cuh"

using fmmb::Error;
using fmmb::fail;

namespace {

thread_local std::string g_last_error;

template <class F>
int guard(fmm_ctx* c, F&& f) {
  try {
    f();
    if (c) c->err.clear();
    return FMM_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    if (c) c->err = e.what();
    return e.status;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    if (c) c->err = e.what();
    return FMM_ERR_CUDA;
  }
}

void require_device() {
  int n = 0;
  const cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    fail(FMM_ERR_NO_DEVICE, "no CUDA device available (the B200 path has no CPU fallback)");
}

enum { EV_BUILD0 = 0, EV_BUILD1, EV_TRAV1, EV_UP1, EV_M2L1, EV_P2P1, EV_DOWN1, EV_P2PK0, EV_P2PK1, EV_M2LK0,
       EV_M2LK1, EV_FORK, EV_XCH0, EV_XCH1, EV_COUNT };
static_assert(EV_COUNT <= 16, "fmm_ctx::ev holds 16 events");

float ms_between(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) {
    cudaGetLastError();
    return 0.f;
  }
  return ms;
}

void do_m2l(fmm_ctx* c, cudaStream_t st) {
  CK(cudaMemsetAsync(c->L.ensure((size_t)c->ncells * c->ncoef), 0, sizeof(double) * c->ncells * c->ncoef, st));
  CK(cudaEventRecord(c->ev[EV_M2LK0], st));
  fmmb::run_m2l(c, st);
  CK(cudaEventRecord(c->ev[EV_M2LK1], st));
}

void do_p2p(fmm_ctx* c, cudaStream_t st) {
  CK(cudaMemsetAsync(c->phi_p2p.ensure(c->N), 0, sizeof(double) * c->N, st));
  CK(cudaMemsetAsync(c->acc_p2p.ensure(3 * c->N), 0, sizeof(double) * 3 * c->N, st));
  CK(cudaEventRecord(c->ev[EV_P2PK0], st));
  fmmb::run_p2p(c, st);
  CK(cudaEventRecord(c->ev[EV_P2PK1], st));
}

void set_device(fmm_ctx* c) { CK(cudaSetDevice(c->cfg.device)); }

}  // namespace

extern "C" {

const char* fmm_version(void) { return "paper_1203_0889_b200 0.1 (sm_100a)"; }

const char* fmm_last_error(const fmm_ctx* ctx) { return ctx ? ctx->err.c_str() : g_last_error.c_str(); }

int fmm_create(const fmm_config* cfg, fmm_ctx** out) {
  if (!cfg || !out) return FMM_ERR_ARG;
  *out = nullptr;
  return guard(nullptr, [&] {
    if (cfg->order < 1) fail(FMM_ERR_ORDER, "expansion order must be >= 1");
    if (cfg->order > FMM_MAX_ORDER) fail(FMM_ERR_UNSUPPORTED, "expansion order above FMM_MAX_ORDER (10)");
    if (cfg->n_crit < 1) fail(FMM_ERR_NCRIT, "n_crit must be >= 1");
    if (!(cfg->theta > 0.0 && cfg->theta < 1.0)) fail(FMM_ERR_THETA, "theta must be in (0,1)");
    if (cfg->precision != FMM_PREC_FP64 && cfg->precision != FMM_PREC_FP32_P2P)
      fail(FMM_ERR_ARG, "unknown precision mode");
    require_device();
    auto* c = new fmm_ctx();
    c->cfg = *cfg;
    c->ncoef = fmmb::n_coef(cfg->order);
    try {
      set_device(c);
      int lo = 0, hi = 0;  // the expansion chain outranks P2P, which fills the SMs it leaves idle
      CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      // priorities: P2P list preparation (stream3) > FMM stream = overlap stream (stream2)
      const int mid = hi < lo ? hi + 1 : hi;
      CK(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, mid));
      // the upward pass shares the SMs with the traversal at the same priority (at low priority
      // it was starved by the traversal's kernels: C4 upward 26 ms against a 21 ms traversal)
      CK(cudaStreamCreateWithPriority(&c->stream2, cudaStreamNonBlocking, mid));
      // P2P list preparation alongside M2L: small latency-bound kernels, scheduled at the
      // highest priority so that they are not starved by the M2L CTAs
      CK(cudaStreamCreateWithPriority(&c->stream3, cudaStreamNonBlocking, hi));
      for (int i = 0; i < EV_COUNT; ++i) CK(cudaEventCreate(&c->ev[i]));
      CK(cudaEventCreateWithFlags(&c->ev_lists, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->ev_l2l, cudaEventDisableTiming));
      c->pstream = c->stream;
      // test hook: the per-level tree build (the fallback when a cooperative launch is not possible)
      if (getenv("FMM_NO_COOP_BUILD")) c->build_coop_ok = false;
      CK(cudaMallocHost(&c->hpin, 64 * sizeof(int64_t)));
      c->d_counters.ensure(32);
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

void fmm_destroy(fmm_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->cfg.device);
  cudaStreamSynchronize(ctx->stream);
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  if (ctx->ev_lists) cudaEventDestroy(ctx->ev_lists);
  if (ctx->ev_l2l) cudaEventDestroy(ctx->ev_l2l);
  if (ctx->own_stream) ctx->stream = ctx->own_stream;
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->stream2) cudaStreamDestroy(ctx->stream2);
  if (ctx->stream3) cudaStreamDestroy(ctx->stream3);
  if (ctx->hpin) cudaFreeHost(ctx->hpin);
  try {
    fmmb::comm_destroy(ctx);
  } catch (...) {
  }
  delete ctx;
}

int fmm_set_bodies(fmm_ctx* c, const double* xyzq, int64_t n) {
  if (!c) return FMM_ERR_ARG;
  return guard(c, [&] {
    if (n <= 0) fail(FMM_ERR_EMPTY_INPUT, "empty input");
    if (!xyzq) fail(FMM_ERR_ARG, "null bodies");
    set_device(c);
    c->N = n;
    c->kernel_launches = 0;
    CK(cudaMemcpyAsync(c->xyzq_in.ensure(n), xyzq, n * sizeof(double4), cudaMemcpyHostToDevice, c->stream));
    c->have_bodies = true;
    c->have_tree = c->have_lists = c->have_M = c->have_L = c->have_out = false;
  });
}

int fmm_set_bodies_device(fmm_ctx* c, const double* d_xyzq, int64_t n) {
  if (!c) return FMM_ERR_ARG;
  return guard(c, [&] {
    if (n <= 0) fail(FMM_ERR_EMPTY_INPUT, "empty input");
    if (!d_xyzq) fail(FMM_ERR_ARG, "null bodies");
    set_device(c);
    c->N = n;
    c->kernel_launches = 0;
    CK(cudaMemcpyAsync(c->xyzq_in.ensure(n), d_xyzq, n * sizeof(double4), cudaMemcpyDeviceToDevice, c->stream));
    c->have_bodies = true;
    c->have_tree = c->have_lists = c->have_M = c->have_L = c->have_out = false;
  });
}

int fmm_build_tree(fmm_ctx* c) {
  if (!c) return FMM_ERR_ARG;
  return guard(c, [&] {
    set_device(c);
    CK(cudaEventRecord(c->ev[EV_BUILD0], c->stream));
    fmmb::build_tree(c);
    CK(cudaEventRecord(c->ev[EV_BUILD1], c->stream));
    c->have_lists = c->have_M = c->have_L = c->have_out = false;
  });
}

int fmm_traverse(fmm_ctx* c) {
  if (!c) return FMM_ERR_ARG;
  return guard(c, [&] {
    set_device(c);
    fmmb::traverse(c);
    CK(cudaEventRecord(c->ev[EV_TRAV1], c->stream));
  });
}

int fmm_upward(fmm_ctx* c) {
  if (!c) return FMM_ERR_ARG;
  return guard(c, [&] {
    set_device(c);
    fmmb::run_upward(c, c->stream);
    CK(cudaEventRecord(c->ev[EV_UP1], c->stream));
  });
}

int fmm_m2l(fmm_ctx* c) {
  if (!c) return FMM_ERR_ARG;
  return guard(c, [&] {
    set_device(c);
    do_m2l(c, c->stream);
    CK(cudaEventRecord(c->ev[EV_M2L1], c->stream));
  });
}

int fmm_p2p(fmm_ctx* c) {
  if (!c) return FMM_ERR_ARG;
  return guard(c, [&] {
    set_device(c);
    do_p2p(c, c->stream);
    CK(cudaEventRecord(c->ev[EV_P2P1], c->stream));
  });
}

int fmm_downward(fmm_ctx* c) {
  if (!c) return FMM_ERR_ARG;
  return guard(c, [&] {
    set_device(c);
    if (!c->have_L) {  // no M2L ran: locals are zero
      CK(cudaMemsetAsync(c->L.ensure((size_t)c->ncells * c->ncoef), 0, sizeof(double) * c->ncells * c->ncoef,
                         c->stream));
      c->have_L = true;
    }
    if (!c->phi_p2p.p) {
      CK(cudaMemsetAsync(c->phi_p2p.ensure(c->N), 0, sizeof(double) * c->N, c->stream));
      CK(cudaMemsetAsync(c->acc_p2p.ensure(3 * c->N), 0, sizeof(double) * 3 * c->N, c->stream));
    }
    fmmb::run_downward(c, c->stream);
    CK(cudaEventRecord(c->ev[EV_DOWN1], c->stream));
  });
}

// The step of fmm_evaluate; with `reuse` (a time step on the kept tree, the bodies already
// re-gathered by refit_bodies) the build is replaced by the refit and the traversal by the
// rebuild of the FP32 P2P entries (their near test depends on the bodies).
void evaluate_impl(fmm_ctx* c, bool reuse) {
  {
    if (!reuse) {
      CK(cudaEventRecord(c->ev[EV_BUILD0], c->stream));
      fmmb::build_tree(c);
    }
    CK(cudaEventRecord(c->ev[EV_BUILD1], c->stream));
    // overlap: the P2P list and work list are prepared on the second stream (after the upward
    // pass) while M2L runs on the first; P2P waits for both
    c->p2p_overlap = c->overlap >= 1 && !reuse;
    c->pstream = c->stream;
    auto lists = [&] {
      if (!reuse) fmmb::traverse(c);
      else if (c->cfg.precision == FMM_PREC_FP32_P2P) fmmb::build_p2p_entries(c);
    };
    try {
      if (c->overlap) {
        // The upward pass needs only the tree: it runs on the second stream while the traversal
        // (and its host round trips) proceeds on the first; M2L joins both.
        CK(cudaStreamWaitEvent(c->stream2, c->ev[EV_BUILD1], 0));
        fmmb::run_upward(c, c->stream2);
        // M2L's detraced source rows need only the multipoles: built here, under the traversal
        if (c->world == 1) fmmb::run_detrace(c, c->stream2);
        CK(cudaEventRecord(c->ev[EV_UP1], c->stream2));
        lists();
        CK(cudaEventRecord(c->ev[EV_TRAV1], c->stream));
        CK(cudaStreamWaitEvent(c->stream, c->ev[EV_UP1], 0));
        CK(cudaEventRecord(c->ev[EV_FORK], c->stream));
      } else {
        lists();
        CK(cudaEventRecord(c->ev[EV_TRAV1], c->stream));
        fmmb::run_upward(c, c->stream);
        CK(cudaEventRecord(c->ev[EV_UP1], c->stream));
        CK(cudaEventRecord(c->ev[EV_FORK], c->stream));
      }
      const bool split = c->p2p_pending;  // the work list is being prepared on stream2
      if (c->overlap >= 2) {
        // M2L (FP64 pipe) on the high-priority stream and P2P (FP32 pipe) on the low-priority
        // one, concurrently: P2P CTAs fill what the M2L CTAs leave of each SM
        do_m2l(c, c->stream);
        CK(cudaEventRecord(c->ev[EV_M2L1], c->stream));
        fmmb::p2p_worklist_end(c);
        CK(cudaEventRecord(c->ev_lists, c->stream3));
        CK(cudaStreamWaitEvent(c->stream2, c->ev_lists, 0));
        CK(cudaStreamWaitEvent(c->stream2, c->ev[EV_FORK], 0));
        do_p2p(c, c->stream2);
        CK(cudaEventRecord(c->ev[EV_P2P1], c->stream2));
        CK(cudaStreamWaitEvent(c->stream, c->ev[EV_P2P1], 0));
      } else {
        do_m2l(c, c->stream);
        CK(cudaEventRecord(c->ev[EV_M2L1], c->stream));
        if (split) {  // finish the work list (host syncs on stream3 while M2L runs), then join
          fmmb::p2p_worklist_end(c);
          CK(cudaEventRecord(c->ev_lists, c->stream3));
          CK(cudaStreamWaitEvent(c->stream, c->ev_lists, 0));
        }
        if (c->overlap) {  // L2L needs only the locals: it runs beside P2P on the highest-priority
                           // stream (its small level launches get the SM slots P2P CTAs free)
          CK(cudaStreamWaitEvent(c->stream3, c->ev[EV_M2L1], 0));
          fmmb::run_downward(c, c->stream3, 1);
          CK(cudaEventRecord(c->ev_l2l, c->stream3));
        }
        do_p2p(c, c->stream);
        CK(cudaEventRecord(c->ev[EV_P2P1], c->stream));
        if (c->overlap) CK(cudaStreamWaitEvent(c->stream, c->ev_l2l, 0));
      }
    } catch (...) {
      c->p2p_overlap = false;
      c->p2p_pending = false;
      c->pstream = c->stream;
      throw;
    }
    c->p2p_overlap = false;
    c->pstream = c->stream;
    fmmb::run_downward(c, c->stream, (c->overlap == 1) ? 2 : 3);
    CK(cudaEventRecord(c->ev[EV_DOWN1], c->stream));
    CK(cudaStreamSynchronize(c->stream));
    fmm_stage_times& t = c->times;
    t.build_ms = ms_between(c->ev[EV_BUILD0], c->ev[EV_BUILD1]);
    t.traverse_ms = ms_between(c->ev[EV_BUILD1], c->ev[EV_TRAV1]);
    // overlap: upward ran concurrently with the traversal (BUILD1 -> UP1 on the second stream)
    t.upward_ms = c->overlap ? ms_between(c->ev[EV_BUILD1], c->ev[EV_UP1]) : ms_between(c->ev[EV_TRAV1], c->ev[EV_UP1]);
    t.m2l_ms = ms_between(c->ev[EV_FORK], c->ev[EV_M2L1]);
    // overlap 2: P2P ran from the fork alongside M2L; downward starts when both are done
    t.p2p_ms = c->overlap >= 2 ? ms_between(c->ev[EV_FORK], c->ev[EV_P2P1]) : ms_between(c->ev[EV_M2L1], c->ev[EV_P2P1]);
    t.downward_ms = c->overlap >= 2 ? ms_between(c->ev[EV_FORK], c->ev[EV_DOWN1]) -
                                          std::max(t.m2l_ms, t.p2p_ms)
                                    : ms_between(c->ev[EV_P2P1], c->ev[EV_DOWN1]);
    t.total_ms = ms_between(c->ev[EV_BUILD0], c->ev[EV_DOWN1]);
    t.p2p_kernel_ms = ms_between(c->ev[EV_P2PK0], c->ev[EV_P2PK1]);
    t.m2l_kernel_ms = ms_between(c->ev[EV_M2LK0], c->ev[EV_M2LK1]);
    t.p2p_launches = 1;
    t.m2l_launches = 1;
    t.kernel_launches = c->kernel_launches;
    t.exchange_ms = 0.f;
  }
}

int fmm_get_stage_trace(fmm_ctx* c, fmm_trace_row* rows, int max_rows, int* n_rows) {
  if (!c || !n_rows || (max_rows > 0 && !rows)) return FMM_ERR_ARG;
  return guard(c, [&] {
    if (!c->have_out) fail(FMM_ERR_STATE, "stage trace: no evaluated step");
    struct Span {
      const char* kind;
      int worker, a, b;
    };
    // fmm_evaluate's event graph: stream 0 = the FMM stream, 1 = the overlap stream (upward)
    const Span spans[] = {
        {"build", 0, EV_BUILD0, EV_BUILD1},
        {"traversal", 0, EV_BUILD1, EV_TRAV1},
        {"upward", c->overlap ? 1 : 0, c->overlap ? EV_BUILD1 : EV_TRAV1, EV_UP1},
        {"m2l", 0, EV_FORK, EV_M2L1},
        {"p2p", c->overlap >= 2 ? 1 : 0, c->overlap >= 2 ? EV_FORK : EV_M2L1, EV_P2P1},
        {"downward", 0, EV_P2P1, EV_DOWN1},
    };
    const int n = static_cast<int>(sizeof(spans) / sizeof(spans[0]));
    *n_rows = n;
    for (int i = 0; i < n && i < max_rows; ++i) {
      fmm_trace_row& r = rows[i];
      std::memset(&r, 0, sizeof(r));
      r.task_id = i;
      r.worker_id = spans[i].worker;
      std::strncpy(r.kind, spans[i].kind, sizeof(r.kind) - 1);
      r.start_ns = static_cast<int64_t>(1e6 * ms_between(c->ev[EV_BUILD0], c->ev[spans[i].a]));
      r.end_ns = static_cast<int64_t>(1e6 * ms_between(c->ev[EV_BUILD0], c->ev[spans[i].b]));
    }
    if (c->overlap >= 2 && n > 5 && max_rows > 5) {  // downward waits for both M2L and P2P
      const int64_t m2l_end = static_cast<int64_t>(1e6 * ms_between(c->ev[EV_BUILD0], c->ev[EV_M2L1]));
      rows[5].start_ns = std::max(rows[5].start_ns, m2l_end);
    }
  });
}

int fmm_evaluate(fmm_ctx* c) {
  if (!c) return FMM_ERR_ARG;
  return guard(c, [&] {
    if (c->world > 1) fail(FMM_ERR_STATE, "evaluate: sharded contexts run the staged sequence (see fmm_b200.h)");
    set_device(c);
    c->kernel_launches = 0;
    evaluate_impl(c, false);
  });
}

int fmm_update_bodies(fmm_ctx* c, const double* xyzq, int64_t n) {
  if (!c) return FMM_ERR_ARG;
  return guard(c, [&] {
    if (n <= 0) fail(FMM_ERR_EMPTY_INPUT, "empty input");
    if (!xyzq) fail(FMM_ERR_ARG, "null bodies");
    set_device(c);
    const bool keep = c->have_tree && c->have_lists && n == c->N;
    c->N = n;
    c->kernel_launches = 0;
    CK(cudaMemcpyAsync(c->xyzq_in.ensure(n), xyzq, n * sizeof(double4), cudaMemcpyHostToDevice, c->stream));
    c->have_bodies = true;
    c->have_M = c->have_L = c->have_out = false;
    if (!keep) c->have_tree = c->have_lists = false;
  });
}

int fmm_evaluate_reuse(fmm_ctx* c, int* reused) {
  if (!c) return FMM_ERR_ARG;
  return guard(c, [&] {
    if (!c->have_bodies) fail(FMM_ERR_STATE, "evaluate_reuse: no bodies");
    if (c->world > 1) fail(FMM_ERR_UNSUPPORTED, "evaluate_reuse: sharded contexts rebuild every step");
    set_device(c);
    c->kernel_launches = 0;
    bool ok = false;
    if (c->have_tree && c->have_lists) {
      CK(cudaEventRecord(c->ev[EV_BUILD0], c->stream));
      ok = fmmb::refit_bodies(c);
    }
    if (reused) *reused = ok ? 1 : 0;
    evaluate_impl(c, ok);
  });
}

int fmm_synchronize(fmm_ctx* c) {
  if (!c) return FMM_ERR_ARG;
  return guard(c, [&] {
    set_device(c);
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaStreamSynchronize(c->stream2));
  });
}

int fmm_get_results(fmm_ctx* c, double* phi, double* acc, int order) {
  if (!c) return FMM_ERR_ARG;
  return guard(c, [&] {
    if (!c->have_out) fail(FMM_ERR_STATE, "get_results: no results (run the downward pass)");
    set_device(c);
    const int64_t n = c->N;
    if (order == 0) {
      if (phi) CK(cudaMemcpyAsync(phi, c->phi.p, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
      if (acc) {
        if (!c->cfg.with_acc) fail(FMM_ERR_STATE, "acceleration was not requested (with_acc = 0)");
        CK(cudaMemcpyAsync(acc, c->acc.p, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
      }
      CK(cudaStreamSynchronize(c->stream));
      return;
    }
    // input order: scatter through the permutation on the device, then one copy each
    double* dphi = c->phi_in.ensure(n);
    double* dacc = acc ? c->acc_in.ensure(3 * n) : nullptr;
    if (acc && !c->cfg.with_acc) fail(FMM_ERR_STATE, "acceleration was not requested (with_acc = 0)");
    fmmb::unpermute_results(c, dphi, dacc);
    if (phi) CK(cudaMemcpyAsync(phi, dphi, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    if (acc) CK(cudaMemcpyAsync(acc, dacc, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int fmm_results_device(fmm_ctx* c, const double** d_phi, const double** d_acc) {
  if (!c) return FMM_ERR_ARG;
  return guard(c, [&] {
    if (!c->have_out) fail(FMM_ERR_STATE, "results_device: no results");
    if (d_phi) *d_phi = c->phi.p;
    if (d_acc) *d_acc = c->cfg.with_acc ? c->acc.p : nullptr;
  });
}

int fmm_get_tree_info(fmm_ctx* c, fmm_tree_info* info) {
  if (!c || !info) return FMM_ERR_ARG;
  return guard(c, [&] {
    if (!c->have_tree) fail(FMM_ERR_STATE, "no tree");
    std::memset(info, 0, sizeof(*info));
    info->nbodies = c->N;
    info->ncells = c->ncells;
    info->nleaves = c->nleaves;
    info->depth = c->depth;
    for (int d = 0; d < 3; ++d) info->center[d] = c->center[d];
    info->half_side = c->half_side;
    info->n_m2l = c->have_lists ? c->n_m2l_emit : -1;
    info->n_p2p = c->have_lists ? c->n_p2p_emit : -1;
    info->p2p_body_pairs = c->have_lists ? c->p2p_body_pairs : -1;
    for (int l = 0; l < FMM_MAX_LEVEL + 2; ++l) info->level_start[l] = c->level_start[l];
    info->mutual = c->cfg.mutual ? 1 : 0;
    info->n_m2l_exec = c->have_lists ? c->n_m2l : -1;
    info->n_p2p_exec = c->have_lists ? c->n_p2p : -1;
  });
}

int fmm_get_stage_times(fmm_ctx* c, fmm_stage_times* t) {
  if (!c || !t) return FMM_ERR_ARG;
  *t = c->times;
  t->kernel_launches = c->kernel_launches;  // launches since the bodies were last set
  return FMM_OK;
}

int fmm_get_cells(fmm_ctx* c, int32_t* level, uint64_t* key, double* center3, double* radius, int32_t* body_begin,
                  int32_t* body_end, int32_t* child_begin, int32_t* child_count, int32_t* parent) {
  if (!c) return FMM_ERR_ARG;
  return guard(c, [&] {
    if (!c->have_tree) fail(FMM_ERR_STATE, "no tree");
    set_device(c);
    const int64_t n = c->ncells;
    auto cp = [&](void* dst, const void* src, size_t bytes) {
      if (dst) CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
    };
    cp(level, c->c_level.p, n * 4);
    cp(key, c->c_key.p, n * 8);
    cp(body_begin, c->c_body_begin.p, n * 4);
    cp(body_end, c->c_body_end.p, n * 4);
    cp(child_begin, c->c_child_begin.p, n * 4);
    cp(child_count, c->c_child_count.p, n * 4);
    cp(parent, c->c_parent.p, n * 4);
    std::vector<double4> cr;
    if (center3 || radius) {
      cr.resize(n);
      cp(cr.data(), c->c_cr.p, n * sizeof(double4));
    }
    CK(cudaStreamSynchronize(c->stream));
    for (int64_t i = 0; i < n && (center3 || radius); ++i) {
      if (center3) {
        center3[3 * i] = cr[i].x;
        center3[3 * i + 1] = cr[i].y;
        center3[3 * i + 2] = cr[i].z;
      }
      if (radius) radius[i] = cr[i].w;
    }
  });
}

int fmm_get_permutation(fmm_ctx* c, int64_t* perm) {
  if (!c || !perm) return FMM_ERR_ARG;
  return guard(c, [&] {
    if (!c->have_tree) fail(FMM_ERR_STATE, "no tree");
    set_device(c);
    std::vector<int32_t> p(c->N);
    CK(cudaMemcpyAsync(p.data(), c->perm.p, c->N * 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (int64_t i = 0; i < c->N; ++i) perm[i] = p[i];
  });
}

int fmm_get_lists(fmm_ctx* c, int64_t* m2l_offsets, int32_t* m2l_sources, int64_t* p2p_offsets,
                  int32_t* p2p_sources) {
  if (!c) return FMM_ERR_ARG;
  return guard(c, [&] {
    if (!c->have_lists) fail(FMM_ERR_STATE, "no lists");
    set_device(c);
    auto cp = [&](void* dst, const void* src, size_t bytes) {
      if (dst && bytes) CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
    };
    // the device CSR keeps each target's sources in (deterministic) emission order; the export
    // is canonical: ascending sources within each target
    auto sort_segments = [&](const int64_t* o_off, int32_t* o_src) {
      for (int64_t t = 0; t < c->ncells; ++t) std::sort(o_src + o_off[t], o_src + o_off[t + 1]);
    };
    if (!c->cfg.mutual) {
      std::vector<int64_t> mo, po;
      const int64_t* mo_p = m2l_offsets;
      const int64_t* po_p = p2p_offsets;
      if (m2l_sources && !m2l_offsets) { mo.resize(c->ncells + 1); mo_p = mo.data(); }
      if (p2p_sources && !p2p_offsets) { po.resize(c->ncells + 1); po_p = po.data(); }
      cp(const_cast<int64_t*>(mo_p), c->m2l_off.p, (mo_p ? (c->ncells + 1) * 8 : 0));
      cp(m2l_sources, c->m2l_src.p, c->n_m2l * 4);
      cp(const_cast<int64_t*>(po_p), c->p2p_off.p, (po_p ? (c->ncells + 1) * 8 : 0));
      cp(p2p_sources, c->p2p_src.p, c->n_p2p * 4);
      CK(cudaStreamSynchronize(c->stream));
      if (m2l_sources) sort_segments(mo_p, m2l_sources);
      if (p2p_sources) sort_segments(po_p, p2p_sources);
      return;
    }
    // mutual: the emitted list (once per unordered pair, in its emitted orientation) = the
    // executed CSR without the mirrored entries
    auto emitted = [&](const fmmb::DBuf<int64_t>& off, const fmmb::DBuf<int32_t>& src,
                       const fmmb::DBuf<uint8_t>& mir, int64_t n, int64_t* o_off, int32_t* o_src) {
      if (!o_off && !o_src) return;
      std::vector<int64_t> ho(c->ncells + 1);
      std::vector<int32_t> hs(n);
      std::vector<uint8_t> hm(n);
      cp(ho.data(), off.p, (c->ncells + 1) * 8);
      cp(hs.data(), src.p, n * 4);
      cp(hm.data(), mir.p, n);
      CK(cudaStreamSynchronize(c->stream));
      int64_t k = 0;
      for (int64_t t = 0; t < c->ncells; ++t) {
        if (o_off) o_off[t] = k;
        for (int64_t i = ho[t]; i < ho[t + 1]; ++i)
          if (!hm[i]) {
            if (o_src) o_src[k] = hs[i];
            ++k;
          }
      }
      if (o_off) o_off[c->ncells] = k;
      if (o_off && o_src) sort_segments(o_off, o_src);
    };
    emitted(c->m2l_off, c->m2l_src, c->m2l_mir, c->n_m2l, m2l_offsets, m2l_sources);
    emitted(c->p2p_off, c->p2p_src, c->p2p_mir, c->n_p2p, p2p_offsets, p2p_sources);
  });
}

int fmm_get_expansions(fmm_ctx* c, double* multipole, double* local) {
  if (!c) return FMM_ERR_ARG;
  return guard(c, [&] {
    set_device(c);
    const size_t bytes = sizeof(double) * c->ncells * c->ncoef;
    if (multipole) {
      if (!c->have_M) fail(FMM_ERR_STATE, "no multipoles");
      CK(cudaMemcpyAsync(multipole, c->M.p, bytes, cudaMemcpyDeviceToHost, c->stream));
    }
    if (local) {
      if (!c->have_L) fail(FMM_ERR_STATE, "no locals");
      CK(cudaMemcpyAsync(local, c->L.p, bytes, cudaMemcpyDeviceToHost, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
  });
}

int fmm_load_tree(fmm_ctx* c, int64_t ncells, const int32_t* level, const uint64_t* key, const double* center3,
                  const double* radius, const int32_t* body_begin, const int32_t* body_end,
                  const int32_t* child_begin, const int32_t* child_count, const int32_t* parent,
                  const int64_t* perm) {
  if (!c) return FMM_ERR_ARG;
  return guard(c, [&] {
    if (!c->have_bodies) fail(FMM_ERR_STATE, "load_tree: set bodies first");
    if (ncells <= 0 || !level || !key || !center3 || !radius || !body_begin || !body_end || !child_begin ||
        !child_count || !parent || !perm)
      fail(FMM_ERR_ARG, "load_tree: bad arguments");
    set_device(c);
    cudaStream_t s = c->stream;
    std::vector<double4> cr(ncells);
    int depth = 0;
    for (int l = 0; l < FMM_MAX_LEVEL + 2; ++l) c->level_start[l] = 0;
    std::vector<int32_t> leaves;
    for (int64_t i = 0; i < ncells; ++i) {
      cr[i] = make_double4(center3[3 * i], center3[3 * i + 1], center3[3 * i + 2], radius[i]);
      depth = level[i] > depth ? level[i] : depth;
      if (child_count[i] == 0) leaves.push_back(static_cast<int32_t>(i));
      if (i > 0 && level[i] < level[i - 1]) fail(FMM_ERR_ARG, "load_tree: cells not level-contiguous");
    }
    for (int l = 0; l <= FMM_MAX_LEVEL + 1; ++l) {
      int64_t first = ncells;
      for (int64_t i = 0; i < ncells; ++i)
        if (level[i] >= l) { first = i; break; }
      c->level_start[l] = static_cast<int32_t>(first);
    }
    std::vector<int32_t> p32(c->N);
    for (int64_t i = 0; i < c->N; ++i) p32[i] = static_cast<int32_t>(perm[i]);
    auto up = [&](void* dst, const void* src, size_t bytes) {
      CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    };
    up(c->c_level.ensure(ncells), level, ncells * 4);
    up(c->c_key.ensure(ncells), key, ncells * 8);
    up(c->c_cr.ensure(ncells), cr.data(), ncells * sizeof(double4));
    up(c->c_body_begin.ensure(ncells), body_begin, ncells * 4);
    up(c->c_body_end.ensure(ncells), body_end, ncells * 4);
    up(c->c_child_begin.ensure(ncells), child_begin, ncells * 4);
    up(c->c_child_count.ensure(ncells), child_count, ncells * 4);
    up(c->c_parent.ensure(ncells), parent, ncells * 4);
    up(c->leaves.ensure(leaves.size()), leaves.data(), leaves.size() * 4);
    up(c->perm.ensure(c->N), p32.data(), c->N * 4);
    c->ncells = ncells;
    c->nleaves = static_cast<int64_t>(leaves.size());
    c->wl = c->leaves.p;
    c->nwl = c->nleaves;
    c->shard_planned = false;
    c->body_keys_valid = false;
    c->depth = depth;
    c->center[0] = center3[0];
    c->center[1] = center3[1];
    c->center[2] = center3[2];
    c->half_side = radius[0];
    fmmb::gather_bodies(c);
    CK(cudaStreamSynchronize(s));  // host staging vectors go out of scope
    c->have_tree = true;
    c->have_lists = c->have_M = c->have_L = c->have_out = false;
  });
}

int fmm_load_lists(fmm_ctx* c, int64_t n_m2l, const int32_t* m2l_pairs, int64_t n_p2p, const int32_t* p2p_pairs) {
  if (!c) return FMM_ERR_ARG;
  return guard(c, [&] {
    if (!c->have_tree) fail(FMM_ERR_STATE, "load_lists: no tree");
    if (n_m2l < 0 || n_p2p < 0 || (n_m2l && !m2l_pairs) || (n_p2p && !p2p_pairs)) fail(FMM_ERR_ARG, "bad lists");
    set_device(c);
    int2* dm = c->pairs_b.ensure(n_m2l + 1);
    int2* dp = c->pairs_c.ensure(n_p2p + 1);
    if (n_m2l) CK(cudaMemcpyAsync(dm, m2l_pairs, n_m2l * sizeof(int2), cudaMemcpyHostToDevice, c->stream));
    if (n_p2p) CK(cudaMemcpyAsync(dp, p2p_pairs, n_p2p * sizeof(int2), cudaMemcpyHostToDevice, c->stream));
    fmmb::lists_from_pairs(c, dm, n_m2l, dp, n_p2p);
    CK(cudaStreamSynchronize(c->stream));
  });
}

int fmm_load_multipoles(fmm_ctx* c, const double* multipole) {
  if (!c || !multipole) return FMM_ERR_ARG;
  return guard(c, [&] {
    if (!c->have_tree) fail(FMM_ERR_STATE, "load_multipoles: no tree");
    set_device(c);
    const size_t n = (size_t)c->ncells * c->ncoef;
    CK(cudaMemcpyAsync(c->M.ensure(n), multipole, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->have_M = true;
    ++c->M_version;
  });
}

int fmm_reset_accumulators(fmm_ctx* c) {
  if (!c) return FMM_ERR_ARG;
  return guard(c, [&] {
    if (!c->have_tree) fail(FMM_ERR_STATE, "no tree");
    set_device(c);
    const size_t n = (size_t)c->ncells * c->ncoef;
    CK(cudaMemsetAsync(c->L.ensure(n), 0, n * sizeof(double), c->stream));
    CK(cudaMemsetAsync(c->phi_p2p.ensure(c->N), 0, c->N * sizeof(double), c->stream));
    CK(cudaMemsetAsync(c->acc_p2p.ensure(3 * c->N), 0, 3 * c->N * sizeof(double), c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->have_L = true;
  });
}

int fmm_set_overlap(fmm_ctx* c, int on) {
  if (!c) return FMM_ERR_ARG;
  c->overlap = on < 0 ? 0 : (on > 2 ? 2 : on);
  return FMM_OK;
}

int fmm_set_mutual(fmm_ctx* c, int on) {
  if (!c) return FMM_ERR_ARG;
  return guard(c, [&] {
    if ((c->cfg.mutual != 0) == (on != 0)) return;
    if (on && c->world > 1) fail(FMM_ERR_UNSUPPORTED, "mutual mode is not supported by the sharded traversal");
    c->cfg.mutual = on != 0;
    c->have_lists = c->have_L = c->have_out = false;  // the lists depend on the mode
  });
}

int fmm_set_traversal_debug(fmm_ctx* c, int force_keys64, int64_t initial_capacity) {
  if (!c) return FMM_ERR_ARG;
  return guard(c, [&] {
    if (initial_capacity < 0) fail(FMM_ERR_ARG, "initial_capacity must be >= 0");
    c->dbg_keys64 = force_keys64 != 0;
    c->dbg_cap = initial_capacity;
    c->have_lists = c->have_L = c->have_out = false;
  });
}

int fmm_set_p2p_shape(fmm_ctx* c, int shape) {
  if (!c) return FMM_ERR_ARG;
  return guard(c, [&] {
    if (shape < -1 || shape > 1) fail(FMM_ERR_ARG, "shape must be -1, 0 or 1");
    c->p2p_shape = shape;
  });
}

int fmm_get_traversal_regrows(fmm_ctx* c, int* regrows) {
  if (!c || !regrows) return FMM_ERR_ARG;
  *regrows = c->trav_regrows;
  return FMM_OK;
}

// ---------------------------------------------------------------------- sharding -------
int fmm_set_partition(fmm_ctx* c, int rank, int world) {
  if (!c) return FMM_ERR_ARG;
  return guard(c, [&] {
    if (world < 1 || rank < 0 || rank >= world) fail(FMM_ERR_ARG, "bad rank/world");
    if (world > 1 && c->cfg.mutual) fail(FMM_ERR_UNSUPPORTED, "mutual mode is not supported by the sharded traversal");
    if (world != c->world) c->plan_world = 0;
    c->rank = rank;
    c->world = world;
    c->shard_planned = false;
    c->have_lists = c->have_M = c->have_L = c->have_out = false;
  });
}

int fmm_get_shard_info(fmm_ctx* c, fmm_shard_info* info) {
  if (!c || !info) return FMM_ERR_ARG;
  return guard(c, [&] {
    if (!c->have_lists) fail(FMM_ERR_STATE, "shard info: run the traversal first");
    info->rank = c->rank;
    info->world = c->world;
    info->body_begin = c->shard_b0;
    info->body_end = c->shard_b1;
    info->own_leaves = c->nwl;
    info->own_cells = c->world > 1 ? c->rank_cells_off[c->rank + 1] - c->rank_cells_off[c->rank] : c->ncells;
    info->chunk_doubles = c->world > 1 ? c->chunk_cells * c->ncoef : 0;
  });
}

int fmm_upward_local(fmm_ctx* c, double* d_send) {
  if (!c) return FMM_ERR_ARG;
  return guard(c, [&] {
    if (c->world == 1) fail(FMM_ERR_STATE, "upward_local: no partition (use fmm_upward)");
    if (!c->shard_planned) fail(FMM_ERR_STATE, "upward_local: run the traversal first");
    set_device(c);
    CK(cudaMemsetAsync(c->M.ensure((size_t)c->ncells * c->ncoef), 0, sizeof(double) * c->ncells * c->ncoef,
                       c->stream));
    fmmb::run_upward(c, c->stream, 1);
    fmmb::shard_pack(c, d_send, c->stream);
  });
}

int fmm_upward_finish(fmm_ctx* c, const double* d_recv) {
  if (!c) return FMM_ERR_ARG;
  return guard(c, [&] {
    if (c->world == 1 || !c->shard_planned) fail(FMM_ERR_STATE, "upward_finish: no sharded upward pass");
    set_device(c);
    fmmb::shard_unpack(c, d_recv, c->stream);
    fmmb::run_upward(c, c->stream, 2);
    c->have_M = true;
    ++c->M_version;
  });
}

int fmm_set_stream(fmm_ctx* c, void* stream) {
  if (!c) return FMM_ERR_ARG;
  return guard(c, [&] {
    set_device(c);
    if (!c->own_stream) c->own_stream = c->stream;
    c->stream = stream ? static_cast<cudaStream_t>(stream) : c->own_stream;
    c->pstream = c->stream;
  });
}

// ------------------------------------------------------- sharded step with NCCL (comm.cu) ----
int fmm_comm_unique_id(void* id) {
  if (!id) return FMM_ERR_ARG;
  return guard(nullptr, [&] { fmmb::comm_unique_id(id); });
}

int fmm_comm_init(fmm_ctx* c, const void* id, int rank, int world) {
  if (!c || !id) return FMM_ERR_ARG;
  const int rc = fmm_set_partition(c, rank, world);
  if (rc) return rc;
  return guard(c, [&] {
    set_device(c);
    fmmb::comm_init(c, id, rank, world);
  });
}

int fmm_comm_destroy(fmm_ctx* c) {
  if (!c) return FMM_ERR_ARG;
  return guard(c, [&] { fmmb::comm_destroy(c); });
}

int fmm_set_allgather(fmm_ctx* c, fmm_allgather_fn fn, void* user) {
  if (!c) return FMM_ERR_ARG;
  c->ag_fn = fn;
  c->ag_user = user;
  return FMM_OK;
}

int fmm_set_bodies_shard(fmm_ctx* c, const double* share, int64_t n_share, int64_t n_total) {
  if (!c) return FMM_ERR_ARG;
  return guard(c, [&] {
    if (n_total <= 0) fail(FMM_ERR_EMPTY_INPUT, "empty input");
    if (!c->nccl_comm && !c->ag_fn) fail(FMM_ERR_STATE, "set_bodies_shard: no communicator (fmm_comm_init)");
    const int world = c->ag_fn ? c->world : c->comm_world, rank = c->ag_fn ? c->rank : c->comm_rank;
    const int64_t chunk = (n_total + world - 1) / world;
    const int64_t b0 = std::min<int64_t>(n_total, rank * chunk), b1 = std::min<int64_t>(n_total, b0 + chunk);
    if (n_share != b1 - b0) fail(FMM_ERR_ARG, "set_bodies_shard: share size != this rank's chunk");
    if (n_share > 0 && !share) fail(FMM_ERR_ARG, "null bodies");
    set_device(c);
    double4* stage = c->body_share.ensure(chunk);
    if (n_share < chunk) CK(cudaMemsetAsync(stage + n_share, 0, (chunk - n_share) * sizeof(double4), c->stream));
    if (n_share > 0)
      CK(cudaMemcpyAsync(stage, share, n_share * sizeof(double4), cudaMemcpyHostToDevice, c->stream));
    double4* all = c->xyzq_in.ensure(chunk * world);
    fmmb::comm_all_gather(c, reinterpret_cast<const double*>(stage), reinterpret_cast<double*>(all), 4 * chunk,
                          c->stream);
    c->N = n_total;
    c->kernel_launches = 0;
    c->have_bodies = true;
    c->have_tree = c->have_lists = c->have_M = c->have_L = c->have_out = false;
  });
}

int fmm_evaluate_sharded(fmm_ctx* c, fmm_shard_info* info) {
  if (!c) return FMM_ERR_ARG;
  return guard(c, [&] {
    if (!c->have_bodies) fail(FMM_ERR_STATE, "evaluate_sharded: no bodies");
    set_device(c);
    c->kernel_launches = 0;
    if (c->world == 1) {
      evaluate_impl(c, false);
      c->times.exchange_ms = 0.f;
    } else {
      if (!c->ag_fn && (!c->nccl_comm || c->comm_world != c->world))
        fail(FMM_ERR_STATE, "evaluate_sharded: no communicator for this partition (fmm_comm_init)");
      cudaStream_t s = c->stream, x = c->stream2;
      CK(cudaEventRecord(c->ev[EV_BUILD0], s));
      fmmb::build_tree(c);
      CK(cudaEventRecord(c->ev[EV_BUILD1], s));
      fmmb::traverse(c);  // lists, partition, own leaves, P2P work list
      CK(cudaEventRecord(c->ev[EV_TRAV1], s));
      // exchange stream: own cells' multipoles -> all-gather -> shared ancestors
      const int64_t chunk = std::max<int64_t>(c->chunk_cells * c->ncoef, 1);
      double* send = c->shard_send.ensure(chunk);
      double* recv = c->shard_recv.ensure(chunk * c->world);
      CK(cudaStreamWaitEvent(x, c->ev[EV_TRAV1], 0));
      CK(cudaMemsetAsync(c->M.ensure((size_t)c->ncells * c->ncoef), 0, sizeof(double) * c->ncells * c->ncoef, x));
      fmmb::run_upward(c, x, 1);
      fmmb::shard_pack(c, send, x);
      CK(cudaEventRecord(c->ev[EV_XCH0], x));
      fmmb::comm_all_gather(c, send, recv, chunk, x);
      CK(cudaEventRecord(c->ev[EV_XCH1], x));
      fmmb::shard_unpack(c, recv, x);
      fmmb::run_upward(c, x, 2);
      CK(cudaEventRecord(c->ev[EV_UP1], x));
      // FMM stream: P2P of the own leaves (needs no multipole) under the exchange
      CK(cudaEventRecord(c->ev[EV_FORK], s));
      do_p2p(c, s);
      CK(cudaEventRecord(c->ev[EV_P2P1], s));
      CK(cudaStreamWaitEvent(s, c->ev[EV_UP1], 0));
      do_m2l(c, s);
      CK(cudaEventRecord(c->ev[EV_M2L1], s));
      c->have_L = true;
      fmmb::run_downward(c, s, 3);
      CK(cudaEventRecord(c->ev[EV_DOWN1], s));
      CK(cudaStreamSynchronize(s));
      fmm_stage_times& t = c->times;
      t.build_ms = ms_between(c->ev[EV_BUILD0], c->ev[EV_BUILD1]);
      t.traverse_ms = ms_between(c->ev[EV_BUILD1], c->ev[EV_TRAV1]);
      t.upward_ms = ms_between(c->ev[EV_TRAV1], c->ev[EV_UP1]);  // includes the exchange
      t.p2p_ms = ms_between(c->ev[EV_FORK], c->ev[EV_P2P1]);
      t.m2l_ms = ms_between(c->ev[EV_P2P1], c->ev[EV_M2L1]);     // includes any wait for the exchange
      t.downward_ms = ms_between(c->ev[EV_M2L1], c->ev[EV_DOWN1]);
      t.total_ms = ms_between(c->ev[EV_BUILD0], c->ev[EV_DOWN1]);
      t.p2p_kernel_ms = ms_between(c->ev[EV_P2PK0], c->ev[EV_P2PK1]);
      t.m2l_kernel_ms = ms_between(c->ev[EV_M2LK0], c->ev[EV_M2LK1]);
      t.exchange_ms = ms_between(c->ev[EV_XCH0], c->ev[EV_XCH1]);
      t.p2p_launches = 1;
      t.m2l_launches = 1;
      t.kernel_launches = c->kernel_launches;
    }
    if (info) {
      info->rank = c->rank;
      info->world = c->world;
      info->body_begin = c->shard_b0;
      info->body_end = c->shard_b1;
      info->own_leaves = c->nwl;
      info->own_cells = c->world > 1 ? c->rank_cells_off[c->rank + 1] - c->rank_cells_off[c->rank] : c->ncells;
      info->chunk_doubles = c->world > 1 ? c->chunk_cells * c->ncoef : 0;
    }
  });
}

int fmm_get_owned_results(fmm_ctx* c, double* phi, double* acc, int64_t* input_index) {
  if (!c) return FMM_ERR_ARG;
  return guard(c, [&] {
    if (!c->have_out) fail(FMM_ERR_STATE, "get_owned_results: no results");
    if (acc && !c->cfg.with_acc) fail(FMM_ERR_STATE, "acceleration was not requested (with_acc = 0)");
    set_device(c);
    const int64_t b0 = c->shard_b0, n = c->shard_b1 - c->shard_b0;
    if (n <= 0) return;
    if (phi) CK(cudaMemcpyAsync(phi, c->phi.p + b0, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    if (acc) CK(cudaMemcpyAsync(acc, c->acc.p + 3 * b0, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    std::vector<int32_t> idx;
    if (input_index) {
      idx.resize(n);
      CK(cudaMemcpyAsync(idx.data(), c->perm.p + b0, n * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
    for (int64_t i = 0; i < static_cast<int64_t>(idx.size()); ++i) input_index[i] = idx[i];
  });
}

int fmm_plan_partition(int64_t ncells, const int32_t* body_begin, const int32_t* body_end,
                       const int32_t* child_count, const double* cell_cost, int world, int64_t* bounds,
                       int32_t* owner) {
  return guard(nullptr, [&] {
    if (ncells <= 0 || world < 1 || !body_begin || !body_end || !child_count || !cell_cost || !bounds || !owner)
      fail(FMM_ERR_ARG, "bad partition arguments");
    fmmb::plan_partition_host(ncells, body_begin, body_end, child_count, cell_cost, world, bounds, owner);
  });
}

// ---------------------------------------------------------------------- operators ----
static int check_order(int order) {
  if (order < 1) return FMM_ERR_ORDER;
  if (order > FMM_MAX_ORDER) return FMM_ERR_UNSUPPORTED;
  return FMM_OK;
}

int fmm_op_p2m(int order, int64_t count, const int32_t* body_offsets, const double* xyzq, const double* centers3,
               double* M) {
  if (int rc = check_order(order)) return rc;
  return guard(nullptr, [&] {
    require_device();
    const int64_t nb = count > 0 ? body_offsets[count] : 0;
    fmmb::op_expansion(fmmb::OP_P2M, order, count, body_offsets, nullptr, centers3, xyzq, nb, M, nullptr);
  });
}

int fmm_op_m2m(int order, int64_t count, const double* child_m, const double* shifts3, double* parent_m) {
  if (int rc = check_order(order)) return rc;
  return guard(nullptr, [&] {
    require_device();
    fmmb::op_expansion(fmmb::OP_M2M, order, count, nullptr, child_m, shifts3, nullptr, 0, parent_m, nullptr);
  });
}

int fmm_op_m2l(int order, int64_t count, const double* source_m, const double* disp3, double* target_l) {
  if (int rc = check_order(order)) return rc;
  return guard(nullptr, [&] {
    for (int64_t k = 0; k < count; ++k) {
      const double* r = disp3 + 3 * k;
      if ((r[0] * r[0] + r[1] * r[1]) + r[2] * r[2] == 0.0)
        fail(FMM_ERR_SINGULAR_M2L, "singular M2L displacement");
    }
    require_device();
    fmmb::op_expansion(fmmb::OP_M2L, order, count, nullptr, source_m, disp3, nullptr, 0, target_l, nullptr);
  });
}

int fmm_op_l2l(int order, int64_t count, const double* parent_l, const double* shifts3, double* child_l) {
  if (int rc = check_order(order)) return rc;
  return guard(nullptr, [&] {
    require_device();
    fmmb::op_expansion(fmmb::OP_L2L, order, count, nullptr, parent_l, shifts3, nullptr, 0, child_l, nullptr);
  });
}

int fmm_op_l2p(int order, int64_t count, const int32_t* body_offsets, const double* L, const double* centers3,
               const double* xyzq, double* phi, double* acc) {
  if (int rc = check_order(order)) return rc;
  return guard(nullptr, [&] {
    require_device();
    const int64_t nb = count > 0 ? body_offsets[count] : 0;
    fmmb::op_expansion(fmmb::OP_L2P, order, count, body_offsets, L, centers3, xyzq, nb, phi, acc);
  });
}

int fmm_op_p2p(int64_t count, const int32_t* ranges4, const double* xyzq, int precision, double* phi, double* acc) {
  return guard(nullptr, [&] {
    require_device();
    int64_t nb = 0;
    for (int64_t k = 0; k < count; ++k)
      for (int j = 0; j < 4; ++j) nb = ranges4[4 * k + j] > nb ? ranges4[4 * k + j] : nb;
    fmmb::op_p2p(count, ranges4, xyzq, nb, precision, phi, acc);
  });
}

int fmm_op_evaluate_multipole(int order, int64_t count, const double* M, const double* x3, const double* centers3,
                              double* out) {
  if (int rc = check_order(order)) return rc;
  return guard(nullptr, [&] {
    std::vector<double> v(6 * (count > 0 ? count : 0));
    for (int64_t k = 0; k < count; ++k) {
      const double r[3] = {x3[3 * k] - centers3[3 * k], x3[3 * k + 1] - centers3[3 * k + 1],
                           x3[3 * k + 2] - centers3[3 * k + 2]};
      if ((r[0] * r[0] + r[1] * r[1]) + r[2] * r[2] == 0.0)
        fail(FMM_ERR_SINGULAR_EVAL, "singular evaluation point");
      for (int d = 0; d < 3; ++d) {
        v[6 * k + d] = x3[3 * k + d];
        v[6 * k + 3 + d] = centers3[3 * k + d];
      }
    }
    require_device();
    fmmb::op_expansion(fmmb::OP_EVAL, order, count, nullptr, M, v.data(), nullptr, 0, out, nullptr);
  });
}

int fmm_op_laplace_derivatives(int max_degree, int64_t count, const double* r3, double* out) {
  if (max_degree < 0 || max_degree + 1 > FMM_MAX_ORDER) return FMM_ERR_UNSUPPORTED;
  return guard(nullptr, [&] {
    require_device();
    fmmb::op_expansion(fmmb::OP_DERIV, max_degree + 1, count, nullptr, nullptr, r3, nullptr, 0, out, nullptr);
  });
}

int fmm_op_compute_bounds(const double* xyzq, int64_t n, double* center3, double* half_side) {
  return guard(nullptr, [&] {
    if (n <= 0) fail(FMM_ERR_EMPTY_INPUT, "empty input");
    require_device();
    fmmb::op_bounds(xyzq, n, center3, half_side);
  });
}

int fmm_op_morton_key(int64_t count, const double* p3, const double* center3, double half_side, int level,
                      uint64_t* out) {
  return guard(nullptr, [&] {
    if (level < 0 || level > FMM_MAX_LEVEL) fail(FMM_ERR_LEVEL_OVERFLOW, "level overflow");
    require_device();
    fmmb::op_morton(count, p3, center3, half_side, level, out);
  });
}

int fmm_op_mac(int64_t count, const double* tcenter3, const double* tradius, const double* scenter3,
               const double* sradius, double theta, int32_t* out) {
  return guard(nullptr, [&] {
    require_device();
    fmmb::op_mac(count, tcenter3, tradius, scenter3, sradius, theta, out);
  });
}

// ----------------------------------------------------------------- synthetic inputs ----
// BASELINE.json configs: the reference's xorshift64* (dataset.cpp:10-34),
// position drawn before charge, Vec3(u(),u(),u()) evaluated right-to-left by g++ (z first).
static void generate_reference(int dist, int64_t n, uint64_t seed, double* xyzq);

int fmm_generate_bodies(int config, int64_t n, uint64_t seed, double* xyzq) {
  return guard(nullptr, [&] {
    if (n <= 0) fail(FMM_ERR_EMPTY_INPUT, "empty input");
    if (!xyzq) fail(FMM_ERR_ARG, "null output");
    if (config >= 10 && config <= 12) {
      generate_reference(config, n, seed, xyzq);
      return;
    }
    auto splitmix = [](uint64_t x) {
      x += 0x9E3779B97F4A7C15ULL;
      x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
      x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
      return x ^ (x >> 31);
    };
    uint64_t st = splitmix(seed);
    if (st == 0) st = 0x9E3779B97F4A7C15ULL;
    auto next = [&]() {
      st ^= st >> 12;
      st ^= st << 25;
      st ^= st >> 27;
      return st * 2685821657736338717ULL;
    };
    auto u01 = [&]() { return static_cast<double>(next() >> 11) * 0x1.0p-53; };
    auto uni = [&](double lo, double hi) { return lo + (hi - lo) * u01(); };
    const double dn = static_cast<double>(n);
    const double two_pi = 6.283185307179586;
    for (int64_t i = 0; i < n; ++i) {
      double* b = xyzq + 4 * i;
      switch (config) {
        case 1:
        case 2:
        case 4:  // uniform in [-1,1]^3, q in (0, 1/N]
          b[2] = uni(-1.0, 1.0);
          b[1] = uni(-1.0, 1.0);
          b[0] = uni(-1.0, 1.0);
          b[3] = (1.0 - u01()) / dn;
          break;
        case 3: {  // Plummer sphere, scale radius 1, r <= 100, isotropic; q = 1/N
          double r;
          do {
            const double U = u01();
            r = 1.0 / std::sqrt(std::pow(U, -2.0 / 3.0) - 1.0);
          } while (!(r <= 100.0) || !std::isfinite(r));
          double v[3], s;
          do {
            v[2] = uni(-1.0, 1.0);
            v[1] = uni(-1.0, 1.0);
            v[0] = uni(-1.0, 1.0);
            s = (v[0] * v[0] + v[1] * v[1]) + v[2] * v[2];
          } while (s > 1.0 || s < 1e-8);
          const double inv = r / std::sqrt(s);
          b[0] = v[0] * inv;
          b[1] = v[1] * inv;
          b[2] = v[2] * inv;
          b[3] = 1.0 / dn;
          break;
        }
        case 5: {  // unit sphere surface (normalised Gaussian 3-vectors), q in [-1,1]/N
          double v[3], s;
          do {
            for (int d = 2; d >= 0; --d) {
              const double u1 = u01(), u2 = u01();
              v[d] = std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(two_pi * u2);
            }
            s = (v[0] * v[0] + v[1] * v[1]) + v[2] * v[2];
          } while (s == 0.0);
          const double inv = 1.0 / std::sqrt(s);
          b[0] = v[0] * inv;
          b[1] = v[1] * inv;
          b[2] = v[2] * inv;
          b[3] = uni(-1.0, 1.0) / dn;
          break;
        }
        default:
          fail(FMM_ERR_ARG, "unknown config (1..5, 10..12)");
      }
    }
  });
}

// The reference's own generate_bodies (dataset.cpp:76-111): 10 = cube (uniform [0,1]^3),
// 11 = sphere-surface (cube rejection, dataset.cpp:55-64), 12 = cluster (8 Irwin-Hall blobs,
// sigma 0.03, dataset.cpp:67-72); charges uniform(-1,1) then mean-subtracted. Vec3(a(), b(), c())
// draws are evaluated right-to-left as g++ does (z first), like the reference build.
static void generate_reference(int dist, int64_t n, uint64_t seed, double* xyzq) {
  auto splitmix = [](uint64_t x) {
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
  };
  uint64_t st = splitmix(seed);
  if (st == 0) st = 0x9E3779B97F4A7C15ULL;
  auto next = [&]() {
    st ^= st >> 12;
    st ^= st << 25;
    st ^= st >> 27;
    return st * 2685821657736338717ULL;
  };
  auto u01 = [&]() { return static_cast<double>(next() >> 11) * 0x1.0p-53; };
  auto uni = [&](double lo, double hi) { return lo + (hi - lo) * u01(); };
  auto normal = [&]() {  // Irwin-Hall: sum of 12 uniforms minus 6
    double s = 0.0;
    for (int k = 0; k < 12; ++k) s += u01();
    return s - 6.0;
  };
  double blob[8][3];
  if (dist == 12)
    for (auto& c : blob) {
      c[2] = u01();
      c[1] = u01();
      c[0] = u01();
    }
  for (int64_t i = 0; i < n; ++i) {
    double* b = xyzq + 4 * i;
    if (dist == 10) {
      b[2] = u01();
      b[1] = u01();
      b[0] = u01();
    } else if (dist == 11) {
      for (;;) {
        double v[3];
        v[2] = uni(-1.0, 1.0);
        v[1] = uni(-1.0, 1.0);
        v[0] = uni(-1.0, 1.0);
        const double r2 = (v[0] * v[0] + v[1] * v[1]) + v[2] * v[2];
        if (r2 > 1.0 || r2 < 1e-8) continue;
        const double r = std::sqrt(r2);
        b[0] = v[0] / r;
        b[1] = v[1] / r;
        b[2] = v[2] / r;
        break;
      }
    } else {
      const double* c = blob[next() % 8];
      double g[3];
      g[2] = normal();
      g[1] = normal();
      g[0] = normal();
      for (int d = 0; d < 3; ++d) b[d] = c[d] + 0.03 * g[d];
    }
    b[3] = uni(-1.0, 1.0);
  }
  double mean = 0.0;
  for (int64_t i = 0; i < n; ++i) mean += xyzq[4 * i + 3];
  mean /= static_cast<double>(n);
  for (int64_t i = 0; i < n; ++i) xyzq[4 * i + 3] -= mean;
}

}  // extern "C"

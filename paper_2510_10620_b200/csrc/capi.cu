// capi.cu — extern "C" boundary (include/dcpx.h). No exception crosses it: every
// dcpx::Failure maps onto its dcpx_status, mirroring the reference's exception types
// (types.hpp:17-45); the message is kept per context (dcpx_last_error).
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "executor.h"

struct dcpx_ctx {
  dcpx::Executor* ex = nullptr;
  std::string err;
};

namespace {
thread_local std::string g_create_err;

template <class F>
dcpx_status guarded(dcpx_ctx* ctx, F&& f) {
  if (!ctx || !ctx->ex) return DCPX_ERROR;
  try {
    f(*ctx->ex);
    return DCPX_OK;
  } catch (const dcpx::Failure& e) {
    ctx->err = e.what();
    if (e.code == DCPX_CUDA_ERROR) ctx->err += ctx->ex->watchdog_info();
    return e.code;
  } catch (const std::exception& e) {
    ctx->err = e.what();
    return DCPX_ERROR;
  }
}
// single-buffer calls: every plan device reads / writes the same packed buffer
template <class T>
std::vector<T> same_for_all(const dcpx::Executor& ex, T p) {
  return std::vector<T>(static_cast<size_t>(std::max(1, ex.devices())), p);
}

}  // namespace

extern "C" {

const char* dcpx_version(void) { return "dcpx 0.1 (sm_100a tcgen05)"; }

dcpx_status dcpx_create(int ndev, const int* cuda_ordinals, dcpx_transport transport, dcpx_ctx** out) {
  if (!out) return DCPX_ERROR;
  *out = nullptr;
  try {
    auto* c = new dcpx_ctx;
    c->ex = new dcpx::Executor(ndev, cuda_ordinals, static_cast<int>(transport));
    *out = c;
    return DCPX_OK;
  } catch (const dcpx::Failure& e) {
    g_create_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_create_err = e.what();
    return DCPX_ERROR;
  }
}

dcpx_status dcpx_prepare(dcpx_ctx* ctx, int nplans, const dcpx_plan_view* plans,
                         const dcpx_graph_view* graph, const dcpx_mask_view* masks) {
  return guarded(ctx, [&](dcpx::Executor& ex) { ex.prepare(nplans, plans, graph, masks); });
}

dcpx_status dcpx_load_inputs(dcpx_ctx* ctx, const void* q, const void* k, const void* v) {
  return guarded(ctx, [&](dcpx::Executor& ex) {
    ex.load_inputs(same_for_all(ex, q).data(), same_for_all(ex, k).data(), same_for_all(ex, v).data(), false);
  });
}

dcpx_status dcpx_load_inputs_host(dcpx_ctx* ctx, const void* q, const void* k, const void* v) {
  return guarded(ctx, [&](dcpx::Executor& ex) {
    ex.load_inputs(same_for_all(ex, q).data(), same_for_all(ex, k).data(), same_for_all(ex, v).data(), true);
  });
}

dcpx_status dcpx_load_inputs_dev(dcpx_ctx* ctx, const void* const* q, const void* const* k, const void* const* v) {
  return guarded(ctx, [&](dcpx::Executor& ex) {
    if (!q || !k || !v) throw dcpx::Failure(DCPX_ERROR, "dcpx_load_inputs_dev: null pointer array");
    ex.load_inputs(q, k, v, false);
  });
}

dcpx_status dcpx_forward(dcpx_ctx* ctx, void* o_out, float* lse_out, dcpx_report* rep) {
  return guarded(ctx, [&](dcpx::Executor& ex) {
    ex.forward(same_for_all(ex, o_out).data(), same_for_all(ex, lse_out).data(), rep, false);
  });
}

dcpx_status dcpx_forward_dev(dcpx_ctx* ctx, void* const* o_out, float* const* lse_out, dcpx_report* rep) {
  return guarded(ctx, [&](dcpx::Executor& ex) { ex.forward(o_out, lse_out, rep, false); });
}

dcpx_status dcpx_forward_host(dcpx_ctx* ctx, void* o_out, float* lse_out, dcpx_report* rep) {
  return guarded(ctx, [&](dcpx::Executor& ex) {
    ex.forward(same_for_all(ex, o_out).data(), same_for_all(ex, lse_out).data(), rep, true);
  });
}

dcpx_status dcpx_synchronize(dcpx_ctx* ctx) {
  return guarded(ctx, [&](dcpx::Executor& ex) { ex.synchronize(); });
}

dcpx_status dcpx_set_streams(dcpx_ctx* ctx, int n, void* const* streams) {
  return guarded(ctx, [&](dcpx::Executor& ex) {
    if (n < 0 || (n > 0 && !streams)) throw dcpx::Failure(DCPX_ERROR, "dcpx_set_streams: bad stream array");
    std::vector<cudaStream_t> s(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) s[i] = static_cast<cudaStream_t>(streams[i]);
    ex.set_streams(n, s.data());
  });
}

dcpx_status dcpx_check_plans(int nplans, const dcpx_plan_view* plans, const dcpx_graph_view* graph,
                             const dcpx_mask_view* masks, char* err, int64_t cap) {
  std::string msg;
  dcpx_status st = DCPX_OK;
  try {
    if (!plans || !graph || !masks) throw dcpx::Failure(DCPX_ERROR, "dcpx_check_plans: null view");
    dcpx::Executor ex(nplans, nullptr);  // host-only: no GPU is touched
    ex.prepare(nplans, plans, graph, masks);
  } catch (const dcpx::Failure& e) {
    st = e.code;
    msg = e.what();
  } catch (const std::exception& e) {
    st = DCPX_ERROR;
    msg = e.what();
  }
  if (err && cap > 0) {
    const size_t n = std::min<size_t>(msg.size(), static_cast<size_t>(cap - 1));
    std::memcpy(err, msg.data(), n);
    err[n] = '\0';
  }
  return st;
}

dcpx_status dcpx_kernel_times(dcpx_ctx* ctx, double* ms, int32_t* launches) {
  return guarded(ctx, [&](dcpx::Executor& ex) {
    if (!ms || !launches) throw dcpx::Failure(DCPX_ERROR, "dcpx_kernel_times: null output");
    ex.kernel_times(ms, launches);
  });
}

dcpx_status dcpx_debug_arena(dcpx_ctx* ctx, int dev, int kind, void** ptr, int64_t* slot_rows) {
  return guarded(ctx, [&](dcpx::Executor& ex) { ex.debug_arena(dev, kind, ptr, slot_rows); });
}

dcpx_status dcpx_set_option(dcpx_ctx* ctx, const char* key, int64_t value) {
  return guarded(ctx, [&](dcpx::Executor& ex) {
    const std::string k = key ? key : "";
    if (k == "fuse_reductions") ex.opt.fuse_reductions = value != 0;
    else if (k == "remap_copies") ex.opt.remap_copies = value != 0;
    else if (k == "check_rows") ex.opt.check_rows = value != 0;
    else if (k == "timing") ex.opt.timing = value != 0;
    else if (k == "trace") ex.opt.trace = value != 0;
    else if (k == "sm_transfers") ex.opt.sm_transfers = value != 0;
    else if (k == "bwd_order") ex.opt.bwd_order = static_cast<int>(value);
    else if (k == "bwd_window") ex.opt.bwd_window = static_cast<int>(value);
    else if (k == "bwd_window_min_steps") ex.opt.bwd_window_min_steps = static_cast<int>(value);
    else if (k == "bwd_merge_heads") ex.opt.bwd_merge_heads = static_cast<int>(value);
    else if (k == "persistent") ex.opt.persistent = static_cast<int>(value);
    else if (k == "aux_zero") ex.opt.aux_zero = static_cast<int>(value);
    else if (k == "sm_reserve") ex.opt.sm_reserve = static_cast<int>(value);
    else if (k == "kernel_timing") ex.opt.kernel_timing = static_cast<int>(value);
    else throw dcpx::Failure(DCPX_ERROR, "unknown option " + k);
  });
}

int dcpx_trace(dcpx_ctx* ctx, double* rows, int max_rows) {
  if (!ctx || !ctx->ex) return -1;
  return ctx->ex->trace_rows(rows, max_rows);
}

const char* dcpx_last_error(dcpx_ctx* ctx) {
  if (!ctx) return g_create_err.c_str();
  return ctx->err.c_str();
}

void dcpx_destroy(dcpx_ctx* ctx) {
  if (!ctx) return;
  try {
    delete ctx->ex;
  } catch (...) {
  }
  delete ctx;
}

}  // extern "C"

// ---- backward; per-rank entry points ----------------------------------------------------
extern "C" {
dcpx_status dcpx_create_rank(int rank, int world, int cuda_ordinal, dcpx_ctx** out) {
  if (!out) return DCPX_ERROR;
  *out = nullptr;
  try {
    if (world < 1 || rank < 0 || rank >= world) throw dcpx::Failure(DCPX_ERROR, "dcpx_create_rank: bad rank / world");
    auto* c = new dcpx_ctx;
    const std::vector<int> ords(static_cast<size_t>(world), cuda_ordinal);
    c->ex = new dcpx::Executor(world, ords.data(), DCPX_TRANSPORT_LOCAL, rank);
    *out = c;
    return DCPX_OK;
  } catch (const dcpx::Failure& e) {
    g_create_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_create_err = e.what();
    return DCPX_ERROR;
  }
}
dcpx_status dcpx_rank_export(dcpx_ctx* ctx, void* buf, int64_t cap, int64_t* size) {
  return guarded(ctx, [&](dcpx::Executor& ex) {
    const int64_t n = ex.export_handles(buf, buf ? cap : 0);
    if (size) *size = n;
  });
}
dcpx_status dcpx_rank_connect(dcpx_ctx* ctx, const void* blobs, int64_t blob_size) {
  return guarded(ctx, [&](dcpx::Executor& ex) { ex.connect(blobs, blob_size, ex.devices()); });
}
dcpx_status dcpx_backward(dcpx_ctx* ctx, const void* d_o, void* dq, void* dk, void* dv, dcpx_report* rep) {
  return guarded(ctx, [&](dcpx::Executor& ex) {
    ex.backward(same_for_all(ex, d_o).data(), same_for_all(ex, dq).data(), same_for_all(ex, dk).data(),
                same_for_all(ex, dv).data(), rep, false);
  });
}

dcpx_status dcpx_backward_dev(dcpx_ctx* ctx, const void* const* d_o, void* const* dq, void* const* dk,
                              void* const* dv, dcpx_report* rep) {
  return guarded(ctx, [&](dcpx::Executor& ex) {
    if (!d_o) throw dcpx::Failure(DCPX_ERROR, "dcpx_backward_dev: null d_o array");
    ex.backward(d_o, dq, dk, dv, rep, false);
  });
}
dcpx_status dcpx_backward_host(dcpx_ctx* ctx, const void* d_o, void* dq, void* dk, void* dv, dcpx_report* rep) {
  return guarded(ctx, [&](dcpx::Executor& ex) {
    ex.backward(same_for_all(ex, d_o).data(), same_for_all(ex, dq).data(), same_for_all(ex, dk).data(),
                same_for_all(ex, dv).data(), rep, true);
  });
}
}

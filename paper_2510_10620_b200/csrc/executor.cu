// executor.cu — host side of the B200 DCP executor.
//
// Replaces dcp::run (simexec.hpp:207-423). prepare() ingests the per-device plans
// (plan.hpp:101-107) and the block graph, re-checks them statically the way
// verify_plans does (plan.hpp:388-475), replays the reference's lockstep interpreter
// symbolically (simexec.hpp:375-397) to detect deadlocks / tag mismatches and to fix
// a global issue order, and compiles each device's instruction stream into a device
// program:
//   AttentionInstr (+ the ReductionInstrs that merge its partials)  -> one fused
//       attn_fwd launch (FwdUnit/FwdStep lists, masks classified per 128x128 tile)
//   remaining ReductionInstrs                                        -> merge launch
//   CopyInstr                                                        -> slot remap (or
//       a copy launch when the source is touched again)
//   CommLaunch / CommWait                                            -> event-ordered
//       transfers on a per-device comm stream (LOCAL transport: one copy kernel per
//       message reading the sender's arena, peer-to-peer across GPUs).
// forward() then issues the programs in the recorded order; no host sync inside.
// This file: lifetime, allocation, tracing and prepare() (validation, lockstep order);
// compile.cu builds the device programs and transfer jobs, run.cu executes them.
#include <cuda_bf16.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <numeric>
#include <set>

#include "executor.h"

namespace dcpx {

// ------------------------------------------------------------------------ lifetime
Executor::Executor(int ndev, const int* ordinals, int transport, int rank)
    : R_(ndev), transport_(transport), rank_(rank) {
  if (rank_ >= 0 && (rank_ >= ndev || transport != DCPX_TRANSPORT_LOCAL))
    throw Failure(DCPX_ERROR, "per-rank mode: rank outside the plan, or a transport other than peer memory");
  if (ndev < 1 || ndev > 64) throw Failure(DCPX_ERROR, "dcpx_create: 1..64 devices supported");
  if (!ordinals) {  // host-only: plan verification and the lockstep replay, no GPU
    host_only_ = true;
    dev_.resize(static_cast<size_t>(ndev));
    return;
  }
  ordinals_.assign(ordinals, ordinals + ndev);
  int count = 0;
  CUDA_OK(cudaGetDeviceCount(&count));
  for (int o : ordinals_)
    if (o < 0 || o >= count) throw Failure(DCPX_ERROR, "dcpx_create: bad CUDA ordinal " + std::to_string(o));
  dev_.resize(static_cast<size_t>(ndev));
  std::set<int> distinct(ordinals_.begin(), ordinals_.end());
  for (int a : distinct)
    for (int b : distinct)
      if (a != b) {
        int can = 0;
        cudaDeviceCanAccessPeer(&can, a, b);
        if (can) {
          DeviceGuard g(a);
          cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
          if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
            throw Failure(DCPX_CUDA_ERROR, "cudaDeviceEnablePeerAccess failed");
          cudaGetLastError();
        }
      }
  CUDA_OK(cudaHostAlloc(reinterpret_cast<void**>(&diag_), sizeof(uint32_t) * (1 + 4 * 64),
                        cudaHostAllocMapped | cudaHostAllocPortable));
  std::memset(diag_, 0, sizeof(uint32_t) * (1 + 4 * 64));
  for (int d = 0; d < R_; ++d) {
    dev_[d].ordinal = ordinals_[d];
    // streams and events only for the devices this process drives (per-rank mode: one); every
    // extra stream on a GPU raises the odds that the compute and comm streams share one of
    // its hardware work queues (CUDA_DEVICE_MAX_CONNECTIONS), which serialises them
    if (!local(d)) continue;
    DeviceGuard g(ordinals_[d]);
    set_watchdog_buffer_fwd(diag_);
    set_watchdog_buffer_bwd(diag_);
    preload_movers();
    CUDA_OK(cudaStreamCreateWithFlags(&dev_[d].cs, cudaStreamNonBlocking));
    int lo = 0, hi = 0;
    CUDA_OK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CUDA_OK(cudaStreamCreateWithPriority(&dev_[d].ms, cudaStreamNonBlocking, hi));  // transfers first
    CUDA_OK(cudaEventCreate(&dev_[d].t0));
    CUDA_OK(cudaEventCreate(&dev_[d].t1));
    CUDA_OK(cudaEventCreateWithFlags(&dev_[d].ev_join, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&dev_[d].ev_done, cudaEventDisableTiming));
    CUDA_OK(cudaStreamCreateWithFlags(&dev_[d].as, cudaStreamNonBlocking));
    CUDA_OK(cudaEventCreateWithFlags(&dev_[d].aux_done, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&dev_[d].bwd_end, cudaEventDisableTiming));
  }
  if (R_ > 0) {
    DeviceGuard g(ordinals_[0]);
    CUDA_OK(cudaStreamCreateWithFlags(&h2d_, cudaStreamNonBlocking));
    CUDA_OK(cudaStreamCreateWithFlags(&d2h_, cudaStreamNonBlocking));
  }
  if (transport_ == DCPX_TRANSPORT_NCCL) {
    std::set<int> distinct(ordinals_.begin(), ordinals_.end());
    if (static_cast<int>(distinct.size()) != R_)
      throw Failure(DCPX_UNSUPPORTED, "NCCL transport needs one GPU per plan device");
    comms_.assign(static_cast<size_t>(R_), nullptr);
    const ncclResult_t r = ncclCommInitAll(comms_.data(), R_, ordinals_.data());
    if (r != ncclSuccess) throw Failure(DCPX_CUDA_ERROR, std::string("ncclCommInitAll: ") + ncclGetErrorString(r));
  } else if (transport_ != DCPX_TRANSPORT_LOCAL) {
    throw Failure(DCPX_ERROR, "unknown transport");
  }
}

// NCCL transport: one message = a group of send/recv pairs over its contiguous row
// regions. The sender's comm stream waits for the data, the receiver's for its slots;
// groups are issued in the global lockstep order on every stream, so the rendezvous
// sends cannot deadlock.
void Executor::nccl_transfer(int src, int dst, const std::vector<RowCopyJob>& jobs, cudaEvent_t data_ready,
                             cudaEvent_t slot_free) {
  {
    DeviceGuard g(dev_[src].ordinal);
    CUDA_OK(cudaStreamWaitEvent(dev_[src].ms, data_ready, 0));
  }
  {
    DeviceGuard g(dev_[dst].ordinal);
    CUDA_OK(cudaStreamWaitEvent(dev_[dst].ms, slot_free, 0));
  }
  auto ok = [](ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw Failure(DCPX_CUDA_ERROR, std::string(what) + ": " + ncclGetErrorString(r));
  };
  ok(ncclGroupStart(), "ncclGroupStart");
  for (const auto& j : jobs) {
    if (j.src_stride != j.row_bytes && j.rows > 1) throw Failure(DCPX_UNSUPPORTED, "NCCL transport: strided transfer");
    const size_t n = static_cast<size_t>(j.rows) * j.row_bytes;
    ok(ncclSend(j.src, n, ncclUint8, dst, comms_[src], dev_[src].ms), "ncclSend");
    ok(ncclRecv(j.dst, n, ncclUint8, src, comms_[dst], dev_[dst].ms), "ncclRecv");
  }
  ok(ncclGroupEnd(), "ncclGroupEnd");
}

void Executor::await_peer_pulls() {
  if (rank_ >= 0) {  // per-rank mode: the peers' pulls flag of the last pass
    if (connected_ && pulls_epoch_ > 0) {
      DeviceGuard g(dev_[rank_].ordinal);
      flag_wait_peers(kFlagPulls, pulls_epoch_, dev_[rank_].cs);
    }
    return;
  }
  if (pulls_done_.empty() || R_ < 2) return;
  // plan devices sharing one GPU run on separate non-blocking streams, so they need the
  // wait as much as devices on different GPUs do
  for (int d = 0; d < R_; ++d) {
    DeviceGuard g(dev_[d].ordinal);
    for (int e = 0; e < R_; ++e)
      if (e != d) CUDA_OK(cudaStreamWaitEvent(dev_[d].cs, pulls_done_[e], 0));
  }
}

void Executor::kernel_times(double* ms, int32_t* launches) {
  for (int k = 0; k < 4; ++k) ms[k] = 0;
  launches[0] = launches[1] = 0;
  for (int d = 0; d < R_; ++d) {
    if (!local(d)) continue;
    DevState& D = dev_[d];
    DeviceGuard gd(D.ordinal);
    double dev_ms[2] = {0, 0};
    for (size_t k = 0; k < D.next_kev; ++k) {
      CUDA_OK(cudaEventSynchronize(D.kev[k].second));
      float t = 0;
      CUDA_OK(cudaEventElapsedTime(&t, D.kev[k].first, D.kev[k].second));
      const int pass = D.kev_pass[k];
      dev_ms[pass] += t;
      ++launches[pass];
    }
    for (int p = 0; p < 2; ++p) {
      ms[p] += dev_ms[p];
      ms[2 + p] = std::max(ms[2 + p], dev_ms[p]);
    }
    D.next_kev = 0;
    D.kev_pass.clear();
  }
}

void Executor::set_streams(int n, const cudaStream_t* s) {
  if (host_only_) throw Failure(DCPX_ERROR, "host-only context");
  if (n != R_) throw Failure(DCPX_ERROR, "dcpx_set_streams: one stream per plan device");
  for (int d = 0; d < R_; ++d) dev_[d].caller = s[d] ? s[d] : cudaStreamLegacy;
}

void Executor::join_caller() {
  for (int d = 0; d < R_; ++d) {
    if (!local(d)) continue;
    DevState& D = dev_[d];
    DeviceGuard g(D.ordinal);
    CUDA_OK(cudaEventRecord(D.ev_join, D.caller));
    CUDA_OK(cudaStreamWaitEvent(D.cs, D.ev_join, 0));
  }
}

void Executor::release_caller() {
  for (int d = 0; d < R_; ++d) {
    if (!local(d)) continue;
    DevState& D = dev_[d];
    DeviceGuard g(D.ordinal);
    CUDA_OK(cudaEventRecord(D.ev_done, D.cs));
    CUDA_OK(cudaStreamWaitEvent(D.caller, D.ev_done, 0));
  }
}

void Executor::mark_pulls_done() {
  if (rank_ >= 0) {
    DeviceGuard g(dev_[rank_].ordinal);
    flag_set(kFlagPulls, dev_[rank_].ms);
    pulls_epoch_ = epoch_;
    return;
  }
  if (R_ < 2) return;
  if (pulls_done_.empty())
    for (int d = 0; d < R_; ++d) pulls_done_.push_back(staging_event(d));
  for (int d = 0; d < R_; ++d) {
    DeviceGuard g(dev_[d].ordinal);
    CUDA_OK(cudaEventRecord(pulls_done_[d], dev_[d].ms));
  }
}

cudaEvent_t Executor::staging_event(int d) {
  DeviceGuard g(dev_[d].ordinal);
  cudaEvent_t e;
  CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  staging_events_.push_back(e);
  staging_event_dev_.push_back(dev_[d].ordinal);
  return e;
}

Executor::~Executor() {
  if (host_only_) return;
  for (auto& d : dev_) {
    DeviceGuard g(d.ordinal);
    if (d.cs) cudaStreamSynchronize(d.cs);
    if (d.ms) cudaStreamSynchronize(d.ms);
    if (d.as) cudaStreamSynchronize(d.as);
  }
  if (R_ > 0) {
    DeviceGuard g(dev_[0].ordinal);
    if (h2d_) { cudaStreamSynchronize(h2d_); cudaStreamDestroy(h2d_); }
    if (d2h_) { cudaStreamSynchronize(d2h_); cudaStreamDestroy(d2h_); }
  }
  for (size_t i = 0; i < staging_events_.size(); ++i) {
    DeviceGuard g(staging_event_dev_[i]);
    cudaEventDestroy(staging_events_[i]);
  }
  for (auto c : comms_)
    if (c) ncclCommDestroy(c);
  for (void* p : ipc_mapped_) cudaIpcCloseMemHandle(p);
  if (flags_) cudaFree(flags_);
  free_all();
  if (diag_) cudaFreeHost(diag_);
  for (auto& d : dev_) {
    DeviceGuard g(d.ordinal);
    for (auto e : d.events) cudaEventDestroy(e);
    for (auto& e : d.kev) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
    for (auto& e : d.tev) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
    if (d.ev_join) cudaEventDestroy(d.ev_join);
    if (d.ev_done) cudaEventDestroy(d.ev_done);
    if (d.aux_done) cudaEventDestroy(d.aux_done);
    if (d.bwd_end) cudaEventDestroy(d.bwd_end);
    if (d.as) cudaStreamDestroy(d.as);
    if (d.t0) cudaEventDestroy(d.t0);
    if (d.t1) cudaEventDestroy(d.t1);
    if (d.cs) cudaStreamDestroy(d.cs);
    if (d.ms) cudaStreamDestroy(d.ms);
  }
}

void Executor::free_all() {
  for (size_t i = 0; i < allocs_.size(); ++i) {
    DeviceGuard g(alloc_dev_[i]);
    cudaFree(allocs_[i]);
  }
  allocs_.clear();
  alloc_dev_.clear();
}

void* Executor::alloc(int d, size_t bytes) {
  DeviceGuard g(dev_[d].ordinal);
  void* p = nullptr;
  CUDA_OK(cudaMalloc(&p, std::max<size_t>(bytes, 256)));
  allocs_.push_back(p);
  alloc_dev_.push_back(dev_[d].ordinal);
  return p;
}

JobList Executor::make_jobs(int d, const std::vector<RowCopyJob>& jobs) {
  std::vector<int> rows;
  for (const auto& j : jobs) rows.push_back(j.rows);
  return make_row_jobs(d, jobs, rows, kRowsPerChunk);
}

cudaEvent_t Executor::event(int d) {
  auto& D = dev_[d];
  if (D.next_event == D.events.size()) {
    DeviceGuard g(D.ordinal);
    cudaEvent_t e;
    CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    D.events.push_back(e);
  }
  return D.events[D.next_event++];
}

// Persistent attention grids leave `sm_reserve` SMs free when the plan communicates, so
// transfer kernels on the (high-priority) comm stream run concurrently with compute.
// Default 4 (profiles/r1_sm_reserve_sweep.log, cfg2 per-rank): N = 4 2910 vs 2817 TFLOP/s
// with 8, N = 2 1624-1653 vs 1601-1609; one cfg3 N = 4 sample was 2 % slower (2482 vs 2531).
// By default only launches that a fetch overlaps keep them (`overlap`, mark_fetch_overlap):
// e.g. the last division's, which runs after every fetch has landed, takes all SMs.
int Executor::attn_grid(int d, int grid, bool overlap) const {
  const int reserve = opt.sm_reserve >= 0 ? opt.sm_reserve : (R_ > 1 && overlap ? 4 : 0);
  const int cap = std::max(1, num_sms(dev_[d].ordinal) - reserve);
  return std::min(grid, cap);
}

void Executor::mark_fetch_overlap(int d) {
  auto& prog = dev_[d].prog;
  const int T = plans_[d].divisions;
  for (size_t i = 0; i < prog.size(); ++i) {
    Op& op = prog[i];
    if (op.kind != OpKind::kFwdAttn) continue;
    bool f = false, b = false;
    for (size_t k = i + 1; k < prog.size(); ++k) {
      const Op& x = prog[k];
      if (x.kind == OpKind::kFwdAttn && (x.num_units > 0 || x.bnum_units > 0)) break;
      if (x.kind == OpKind::kCommWait && x.division < T) {
        f |= x.jobs.dj.n_blocks > 0 || !x.xfer.empty();
        b |= x.bjobs.dj.n_blocks > 0 || !x.bxfer.empty();
      }
    }
    op.fetch_overlap = f;
    op.bfetch_overlap = b;
  }
}

// LOCAL transport on the DMA copy engines (option sm_transfers = 0), issued on the receiver's
// comm stream so NVLink traffic never competes with the attention kernels for SMs. A block
// component is one contiguous run of slot rows on both sides; runs that continue each other
// on both sides are merged into one cudaMemcpyAsync (one call per 256 KiB component keeps
// the host issuing thousands of copies per step).
void Executor::copy_engine(const std::vector<RowCopyJob>& jobs, cudaStream_t s) {
  char *dst = nullptr, *src = nullptr;
  size_t run = 0;
  auto flush = [&] {
    if (run) CUDA_OK(cudaMemcpyAsync(dst, src, run, cudaMemcpyDefault, s));
    run = 0;
  };
  for (const auto& j : jobs) {
    if (j.src_stride == j.row_bytes && j.dst_stride == j.row_bytes) {
      const size_t n = static_cast<size_t>(j.rows) * j.row_bytes;
      char* d = static_cast<char*>(j.dst);
      char* c = const_cast<char*>(static_cast<const char*>(j.src));
      if (run && dst + run == d && src + run == c) {
        run += n;
      } else {
        flush();
        dst = d;
        src = c;
        run = n;
      }
    } else {
      flush();
      CUDA_OK(cudaMemcpy2DAsync(j.dst, j.dst_stride, j.src, j.src_stride, j.row_bytes, j.rows, cudaMemcpyDefault, s));
    }
  }
  flush();
}

// ---- op tracing (option "trace"): device-time spans of every executed op ------------------
void Executor::trace_begin() {
  trace_.clear();
  trace_pending_.clear();
}

TraceScope::TraceScope(Executor* ex, int d, int instr, cudaStream_t s, int pass, const Op& op)
    : ex_(ex), d_(d) {
  if (!ex->opt.trace || op.kind == OpKind::kNop) return;
  auto ev = ex->trace_events(d);
  CUDA_OK(cudaEventRecord(ev.first, s));
  ex->trace_pending_.push_back({d, instr, static_cast<int>(op.kind), op.division, pass, ev.first, ev.second});
  s_ = s;
  active_ = true;
}

TraceScope::~TraceScope() {
  if (active_) cudaEventRecord(ex_->trace_pending_.back().end, s_);
}

void TraceScope::split(int kind) {
  if (!active_) return;
  auto ev = ex_->trace_events(d_);
  CUDA_OK(cudaEventRecord(ev.first, s_));
  Executor::TracePending prev = ex_->trace_pending_.back();
  ex_->trace_pending_.back().end = ev.first;
  ex_->trace_pending_.push_back({prev.d, prev.instr, kind, prev.division, prev.pass, ev.first, ev.second});
}

void Executor::trace_collect() {
  for (const auto& t : trace_pending_) {
    DeviceGuard gd(dev_[t.d].ordinal);
    cudaEventSynchronize(t.end);
    float a = 0, b = 0;
    cudaEventElapsedTime(&a, dev_[t.d].t0, t.start);
    cudaEventElapsedTime(&b, dev_[t.d].t0, t.end);
    trace_.push_back({static_cast<double>(t.d), static_cast<double>(t.instr), static_cast<double>(t.kind),
                      static_cast<double>(t.division), static_cast<double>(t.pass), a, b});
  }
  trace_pending_.clear();
}

std::string Executor::watchdog_info() const {
  if (!diag_ || diag_[0] == 0) return "";
  std::string s = " [watchdog: " + std::to_string(diag_[0]) + " timed-out waits; distinct (block, warp, barrier, parity):";
  std::set<std::tuple<uint32_t, uint32_t, uint32_t, uint32_t>> seen;
  for (uint32_t i = 0; i < std::min<uint32_t>(diag_[0], 64); ++i)
    seen.insert({diag_[1 + 4 * i], diag_[2 + 4 * i] / 32, diag_[3 + 4 * i], diag_[4 + 4 * i]});
  for (const auto& [b, w, a, par] : seen)
    s += " (" + std::to_string(b) + ", w" + std::to_string(w) + ", smem+" + std::to_string(a) + ", " +
         std::to_string(par) + ")";
  return s + "]";
}

int Executor::trace_rows(double* out, int max_rows) const {
  const int n = std::min<int>(max_rows, static_cast<int>(trace_.size()));
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < 7; ++k) out[7 * i + k] = trace_[i][k];
  return static_cast<int>(trace_.size());
}

std::pair<cudaEvent_t, cudaEvent_t> Executor::trace_events(int d) {
  auto& D = dev_[d];
  if (D.next_tev == D.tev.size()) {
    DeviceGuard g(D.ordinal);
    cudaEvent_t a, b;
    CUDA_OK(cudaEventCreate(&a));
    CUDA_OK(cudaEventCreate(&b));
    D.tev.push_back({a, b});
  }
  return D.tev[D.next_tev++];
}

std::pair<cudaEvent_t, cudaEvent_t> Executor::kernel_events(int d, int pass) {
  auto& D = dev_[d];
  D.kev_pass.resize(D.next_kev + 1);
  D.kev_pass[D.next_kev] = pass;
  if (D.next_kev == D.kev.size()) {
    DeviceGuard g(D.ordinal);
    cudaEvent_t a, b;
    CUDA_OK(cudaEventCreate(&a));
    CUDA_OK(cudaEventCreate(&b));
    D.kev.push_back({a, b});
  }
  return D.kev[D.next_kev++];
}

// ------------------------------------------------------------------------ prepare
void Executor::prepare(int nplans, const dcpx_plan_view* plans, const dcpx_graph_view* gv,
                       const dcpx_mask_view* mv) {
  if (nplans != R_) throw Failure(DCPX_ERROR, "run: plan count does not match topology");  // simexec.hpp:211
  if (!host_only_) synchronize();  // asynchronous host I/O of a previous plan may still be in flight
  if (rank_ >= 0) {  // per-rank mode: the previous plan's peer mappings and flags
    DeviceGuard g(dev_[rank_].ordinal);
    for (void* p : ipc_mapped_) cudaIpcCloseMemHandle(p);
    ipc_mapped_.clear();
    if (flags_) cudaFree(flags_);
    flags_ = nullptr;
    connected_ = false;
  }
  if (!host_only_) free_all();
  for (Staging* st : {&in_st_, &bwd_st_, &fwd_st_})
    for (int k = 0; k < kStagingSlots; ++k) {  // (events stay alive in staging_events_ and are reused)
      st->buf[k] = nullptr;
    }
  fwd_done_ = false;
  for (auto& d : dev_) {
    d.prog.clear();
    d.o_phys.clear();
  }
  prepared_ = false;
  // ---- graph copy
  g_ = GraphCopy{};
  g_.H = gv->heads; g_.G = gv->kv_groups; g_.D = gv->head_dim; g_.bpe = gv->bytes_per_element;
  // (a host-only context executes nothing, so any head_dim / element size verifies)
  if (!host_only_ && g_.D != kHeadDim) throw Failure(DCPX_UNSUPPORTED, "sm_100a kernels support head_dim 128 only");
  if (!host_only_ && g_.bpe != 2) throw Failure(DCPX_UNSUPPORTED, "bf16 payloads (bytes_per_element 2) only");
  if (g_.H < 1 || g_.G < 1 || g_.H % g_.G) throw Failure(DCPX_ERROR, "batch: heads must be divisible by kv_groups");
  g_.seq_lengths.assign(gv->seq_lengths, gv->seq_lengths + gv->num_seqs);
  g_.block_sizes.assign(gv->block_sizes, gv->block_sizes + gv->num_seqs);
  g_.seq_offsets.assign(mv->seq_offsets, mv->seq_offsets + gv->num_seqs + 1);
  for (int s = 0; s < gv->num_seqs; ++s)
    if (g_.seq_offsets[s + 1] - g_.seq_offsets[s] != g_.seq_lengths[s])
      throw Failure(DCPX_ERROR, "mask view does not match sequence lengths");
  g_.ranges.assign(mv->ranges, mv->ranges + 4 * g_.total_tokens());
  g_.data_blocks.assign(gv->data_blocks, gv->data_blocks + gv->num_data_blocks);
  g_.comp_blocks.assign(gv->comp_blocks, gv->comp_blocks + gv->num_comp_blocks);
  int64_t max_rows = 1;
  for (const auto& db : g_.data_blocks) {
    if (db.seq < 0 || db.seq >= gv->num_seqs || db.tok_begin < 0 || db.tok_end > g_.seq_lengths[db.seq] ||
        db.tok_end <= db.tok_begin)
      throw Failure(DCPX_ERROR, "graph: bad data block " + std::to_string(db.id));
    max_rows = std::max<int64_t>(max_rows, db.tok_end - db.tok_begin);
  }
  const int64_t slot_rows = (max_rows + 127) / 128 * 128;

  // ---- plan copies
  plans_.assign(static_cast<size_t>(R_), PlanCopy{});
  for (int d = 0; d < R_; ++d) {
    const dcpx_plan_view& v = plans[d];
    PlanCopy& P = plans_[d];
    if (v.device != d) throw Failure(DCPX_ERROR, "plan " + std::to_string(d) + " has device " + std::to_string(v.device));
    P.device = v.device;
    P.divisions = v.divisions;
    for (int k = 0; k < 3; ++k) P.cap[k] = v.capacity[k];
    P.res_q.assign(v.resident_q, v.resident_q + v.n_resident_q);
    P.res_kv.assign(v.resident_kv, v.resident_kv + v.n_resident_kv);
    P.res_o.assign(v.resident_o, v.resident_o + v.n_resident_o);
    int64_t n_items = 0, n_srcs = 0, n_copies = 0, n_blocks = 0, n_rows = 0;
    for (int i = 0; i < v.n_instructions; ++i) {
      const dcpx_instruction& x = v.instructions[i];
      Instr I;
      I.op = x.op; I.division = x.division; I.send = x.send; I.peer = x.peer; I.dst = x.dst;
      I.count = x.count; I.offset = x.offset;
      if (x.tag) I.tag = x.tag;
      if (I.op < 0 || I.op > 4) throw Failure(DCPX_ERROR, "run: unknown instruction");  // simexec.hpp:369
      if (I.count < 0 || I.offset < 0) throw Failure(DCPX_ERROR, "plan: negative pool range");
      const int64_t end = I.offset + I.count;
      if (I.op == DCPX_OP_ATTENTION) n_items = std::max(n_items, end);
      if (I.op == DCPX_OP_REDUCTION) n_srcs = std::max(n_srcs, end);
      if (I.op == DCPX_OP_COPY) n_copies = std::max(n_copies, end);
      if (I.op == DCPX_OP_COMM_LAUNCH) n_blocks = std::max(n_blocks, end);
      if ((I.op == DCPX_OP_COMM_LAUNCH || I.op == DCPX_OP_COMM_WAIT) && I.tag.empty())
        throw Failure(DCPX_TAG_MISMATCH, "communication instruction without a tag");
      P.ins.push_back(std::move(I));
    }
    P.items.assign(v.items, v.items + n_items);
    P.srcs.assign(v.srcs, v.srcs + n_srcs);
    P.copies.assign(v.copies, v.copies + n_copies);
    P.blocks.assign(v.blocks, v.blocks + n_blocks);
    for (const auto& it : P.items)
      if (it.rows_offset >= 0) n_rows = std::max<int64_t>(n_rows, it.rows_offset + (it.q_end - it.q_begin));
    if (n_rows) P.rows.assign(v.rows, v.rows + 4 * n_rows);
  }

  // ---- static verification (verify_plans, plan.hpp:388-475)
  {
    struct Side { int device = -1, peer = -1; std::vector<int> blocks; };
    std::map<std::string, Side> send_side, recv_side;
    std::map<std::string, int> wait_count;
    auto kind_of = [&](int block) {
      if (block < 0 || block >= static_cast<int>(g_.data_blocks.size()))
        throw Failure(DCPX_ERROR, "plan: bad data block id " + std::to_string(block));
      return g_.data_blocks[block].kind;
    };
    for (const auto& P : plans_) {
      std::array<std::set<int>, 3> written;
      for (const auto& r : P.res_q) written[0].insert(r.slot);
      for (const auto& r : P.res_kv) written[1].insert(r.slot);
      std::map<std::string, std::vector<std::pair<int, int>>> pending;
      auto check_slot = [&](int kind, int slot) {
        if (slot < 0 || slot >= P.cap[kind])
          throw Failure(DCPX_BUFFER_OVERFLOW, "device " + std::to_string(P.device) + ": slot " + std::to_string(slot) +
                                                  " outside capacity " + std::to_string(P.cap[kind]));
      };
      auto require = [&](int kind, int slot, const char* what) {
        check_slot(kind, slot);
        if (!written[kind].count(slot))
          throw Failure(DCPX_ERROR, "plan verify: device " + std::to_string(P.device) + ": " + what + " reads slot " +
                                        std::to_string(slot) + " before it is written");
      };
      for (const auto& r : P.res_q) { check_slot(0, r.slot); if (kind_of(r.block) != DCPX_KIND_Q) throw Failure(DCPX_ERROR, "resident_q holds a non-Q block"); }
      for (const auto& r : P.res_kv) { check_slot(1, r.slot); if (kind_of(r.block) != DCPX_KIND_KV) throw Failure(DCPX_ERROR, "resident_kv holds a non-KV block"); }
      for (const auto& r : P.res_o) { check_slot(2, r.slot); if (kind_of(r.block) != DCPX_KIND_O) throw Failure(DCPX_ERROR, "resident_o holds a non-O block"); }
      for (const auto& I : P.ins) {
        if (I.op == DCPX_OP_ATTENTION) {
          for (int i = 0; i < I.count; ++i) {
            const auto& it = P.items[I.offset + i];
            require(0, it.q_slot, "attention");
            require(1, it.kv_slot, "attention");
            check_slot(2, it.out_slot);
            written[2].insert(it.out_slot);
            if (it.seq < 0 || it.seq >= static_cast<int>(g_.seq_lengths.size()) || it.head < 0 || it.head >= g_.H ||
                it.q_begin < 0 || it.q_end > g_.seq_lengths[it.seq] || it.q_end <= it.q_begin || it.kv_begin < 0 ||
                it.kv_end > g_.seq_lengths[it.seq] || it.kv_end <= it.kv_begin || it.q_end - it.q_begin > slot_rows ||
                it.kv_end - it.kv_begin > slot_rows)
              throw Failure(DCPX_ERROR, "exec_attention: inconsistent shapes");  // simexec.hpp:35-38
          }
        } else if (I.op == DCPX_OP_REDUCTION) {
          if (I.count < 1) throw Failure(DCPX_ERROR, "exec_reduction: no partials");  // simexec.hpp:81
          for (int i = 0; i < I.count; ++i) require(2, P.srcs[I.offset + i], "reduction");
          check_slot(2, I.dst);
          written[2].insert(I.dst);
        } else if (I.op == DCPX_OP_COPY) {
          for (int i = 0; i < I.count; ++i) {
            const auto& c = P.copies[I.offset + i];
            require(2, c.src_slot, "copy");
            check_slot(2, c.dst_slot);
            written[2].insert(c.dst_slot);
          }
        } else if (I.op == DCPX_OP_COMM_LAUNCH) {
          if (I.peer < 0 || I.peer >= R_) throw Failure(DCPX_ERROR, "bad peer device");
          if (I.send) {
            for (int i = 0; i < I.count; ++i) {
              const auto& tb = P.blocks[I.offset + i];
              require(kind_of(tb.block), tb.slot, "send");
            }
            auto [it, ins] = send_side.insert({I.tag, {}});
            if (!ins) throw Failure(DCPX_TAG_MISMATCH, "duplicate send tag " + I.tag);
            it->second.device = P.device; it->second.peer = I.peer;
            for (int i = 0; i < I.count; ++i) it->second.blocks.push_back(P.blocks[I.offset + i].block);
          } else {
            auto [it, ins] = recv_side.insert({I.tag, {}});
            if (!ins) throw Failure(DCPX_TAG_MISMATCH, "duplicate recv tag " + I.tag);
            it->second.device = P.device; it->second.peer = I.peer;
            for (int i = 0; i < I.count; ++i) {
              const auto& tb = P.blocks[I.offset + i];
              const int k = kind_of(tb.block);
              check_slot(k, tb.slot);
              it->second.blocks.push_back(tb.block);
              pending[I.tag].push_back({k, tb.slot});
            }
          }
        } else if (I.op == DCPX_OP_COMM_WAIT) {
          auto it = pending.find(I.tag);
          if (it == pending.end())
            throw Failure(DCPX_TAG_MISMATCH, "device " + std::to_string(P.device) + " waits on tag " + I.tag +
                                                 " without a posted receive");
          for (auto [k, s] : it->second) written[k].insert(s);
          pending.erase(it);
          ++wait_count[I.tag];
        }
      }
      if (!pending.empty())
        throw Failure(DCPX_TAG_MISMATCH, "device " + std::to_string(P.device) + " has posted receives never waited on");
    }
    for (const auto& [tag, snd] : send_side) {
      auto it = recv_side.find(tag);
      if (it == recv_side.end()) continue;  // unmatched sends surface in the lockstep replay
      if (snd.peer != it->second.device || it->second.peer != snd.device)
        throw Failure(DCPX_TAG_MISMATCH, "tag " + tag + " connects mismatched peers");
      if (snd.blocks != it->second.blocks)
        throw Failure(DCPX_TAG_MISMATCH, "tag " + tag + " transfers mismatched block lists");
    }
  }

  // ---- lockstep replay: deadlock / tag errors + the global issue order
  simulate_order();
  if (host_only_) {
    prepared_ = true;
    return;
  }

  // ---- per-device compile
  for (int d = 0; d < R_; ++d) {
    dev_[d].slot_rows = slot_rows;
    compile_device(d);
    build_persistent_fwd(d);
  }
  // ---- transfer jobs (owned by the receiver) and input / output jobs
  build_transfer_jobs();
  for (int d = 0; d < R_; ++d) build_io_jobs(d);
  build_bwd_jobs();
  for (int d = 0; d < R_; ++d) mark_fetch_overlap(d);
  for (int d = 0; d < R_; ++d) {
    DeviceGuard g(dev_[d].ordinal);
    CUDA_OK(cudaDeviceSynchronize());
  }
  // enqueue orders per pass without the ops that launch nothing (fused reductions, remapped
  // copies; the backward also skips the output stage and the forward-only merges / copies)
  fwd_live_.clear();
  bwd_live_.clear();
  {
    const int T = R_ ? plans_[0].divisions : 0;
    for (const auto& [d, i] : order_) {
      const Op& op = dev_[d].prog[i];
      if (op.kind == OpKind::kNop) continue;
      fwd_live_.push_back({d, i});
      if (plans_[d].ins[i].division < T &&
          (op.kind == OpKind::kFwdAttn || op.kind == OpKind::kCommLaunch || op.kind == OpKind::kCommWait))
        bwd_live_.push_back({d, i});
    }
  }
  if (rank_ >= 0) {  // per-rank mode: flags for the peers, tags numbered the same on every rank
    tag_id_.clear();
    for (const auto& P : plans_)
      for (const auto& I : P.ins)
        if (I.op == DCPX_OP_COMM_LAUNCH && I.send) tag_id_.emplace(I.tag, static_cast<int>(tag_id_.size()));
    DeviceGuard g(dev_[rank_].ordinal);
    const size_t words = kFlagSend + tag_id_.size();
    CUDA_OK(cudaMalloc(&flags_, words * sizeof(uint32_t)));
    CUDA_OK(cudaMemset(flags_, 0, words * sizeof(uint32_t)));
    epoch_ = pulls_epoch_ = 0;
    connected_ = false;
  }
  acc_dirty_ = false;  // the accumulators were zeroed when allocated (compile_device)
  prepared_ = true;
}

// ---- per-rank mode ---------------------------------------------------------------------
namespace {
struct IpcBlob {
  int32_t rank, n;
  cudaIpcMemHandle_t h[10];
};
}  // namespace

int64_t Executor::export_handles(void* buf, int64_t cap) const {
  if (rank_ < 0 || !prepared_) throw Failure(DCPX_ERROR, "export_handles: per-rank context after prepare only");
  if (cap < static_cast<int64_t>(sizeof(IpcBlob))) return static_cast<int64_t>(sizeof(IpcBlob));
  const DevState& D = dev_[rank_];
  DeviceGuard g(D.ordinal);
  IpcBlob b{};
  b.rank = rank_;
  void* ptrs[10] = {D.q, D.kv, D.o, D.lse, D.d_o, D.lse2, D.delta, D.dq_acc, D.dkv_acc, flags_};
  b.n = 10;
  for (int i = 0; i < 10; ++i) CUDA_OK(cudaIpcGetMemHandle(&b.h[i], ptrs[i]));
  std::memcpy(buf, &b, sizeof(b));
  return static_cast<int64_t>(sizeof(b));
}

void Executor::connect(const void* blobs, int64_t blob_size, int world) {
  if (rank_ < 0 || !prepared_) throw Failure(DCPX_ERROR, "connect: per-rank context after prepare only");
  if (world != R_ || blob_size != static_cast<int64_t>(sizeof(IpcBlob)))
    throw Failure(DCPX_ERROR, "connect: handle blobs do not match this context");
  DeviceGuard g(dev_[rank_].ordinal);
  peer_flags_.assign(static_cast<size_t>(R_), nullptr);
  peer_flags_[rank_] = flags_;
  for (int e = 0; e < R_; ++e) {
    if (e == rank_) continue;
    IpcBlob b;
    std::memcpy(&b, static_cast<const char*>(blobs) + e * blob_size, sizeof(b));
    if (b.rank != e || b.n != 10) throw Failure(DCPX_ERROR, "connect: blob order");
    void* p[10];
    for (int i = 0; i < 10; ++i) {
      CUDA_OK(cudaIpcOpenMemHandle(&p[i], b.h[i], cudaIpcMemLazyEnablePeerAccess));
      ipc_mapped_.push_back(p[i]);
    }
    DevState& E = dev_[e];  // from here on, peer e's arenas are its own, mapped
    E.q = static_cast<__nv_bfloat16*>(p[0]);
    E.kv = static_cast<__nv_bfloat16*>(p[1]);
    E.o = static_cast<__nv_bfloat16*>(p[2]);
    E.lse = static_cast<float*>(p[3]);
    E.d_o = static_cast<__nv_bfloat16*>(p[4]);
    E.lse2 = static_cast<float*>(p[5]);
    E.delta = static_cast<float*>(p[6]);
    E.dq_acc = static_cast<float*>(p[7]);
    E.dkv_acc = static_cast<float*>(p[8]);
    peer_flags_[e] = static_cast<uint32_t*>(p[9]);
  }
  build_transfer_jobs();
  build_bwd_jobs();
  CUDA_OK(cudaDeviceSynchronize());
  connected_ = true;
}

void Executor::flag_set(int word, cudaStream_t s) { launch_flag_set(flags_ + word, epoch_, s); }

// Waits until the flag word of every peer (or of one peer) reached `epoch`.
void Executor::flag_wait_peers(int word, uint32_t epoch, cudaStream_t s, int only_peer) {
  std::vector<const uint32_t*> f;
  for (int e = 0; e < R_; ++e)
    if (e != rank_ && (only_peer < 0 || e == only_peer)) f.push_back(peer_flags_[e] + word);
  for (size_t i = 0; i < f.size(); i += 64)
    launch_flag_wait(f.data() + i, static_cast<int>(std::min<size_t>(64, f.size() - i)), epoch, s);
}

// Transfer jobs of every CommWait, owned by the receiver (they read the sender's arenas:
// peer memory across GPUs, or IPC-mapped peer memory in the per-rank mode).
void Executor::build_transfer_jobs() {
  const int64_t SR = R_ ? dev_[0].slot_rows : 0;
  for (int d = 0; d < R_; ++d) {
    for (auto& op : dev_[d].prog) {
      if (op.kind != OpKind::kCommWait) continue;
      // find the matching send and recv launches
      const PlanCopy& P = plans_[d];
      int recv_i = -1;
      for (size_t i = 0; i < P.ins.size(); ++i)
        if (P.ins[i].op == DCPX_OP_COMM_LAUNCH && !P.ins[i].send && P.ins[i].tag == op.tag) recv_i = static_cast<int>(i);
      const int src_dev = P.ins[recv_i].peer;
      const PlanCopy& S = plans_[src_dev];
      int send_i = -1;
      for (size_t i = 0; i < S.ins.size(); ++i)
        if (S.ins[i].op == DCPX_OP_COMM_LAUNCH && S.ins[i].send && S.ins[i].tag == op.tag) send_i = static_cast<int>(i);
      if (send_i < 0) throw Failure(DCPX_DEADLOCK, "no sender for " + op.tag);
      const Instr& RI = P.ins[recv_i];
      const Instr& SI = S.ins[send_i];
      std::vector<RowCopyJob> jobs;
      const DevState& A = dev_[src_dev];
      const DevState& B = dev_[d];
      for (int b = 0; b < RI.count; ++b) {
        const auto rb = P.blocks[RI.offset + b];
        const auto sb = S.blocks[SI.offset + b];
        const auto& db = g_.data_blocks[rb.block];
        const int rows = static_cast<int>(db.tok_end - db.tok_begin);
        if (db.kind == DCPX_KIND_Q) {
          jobs.push_back({reinterpret_cast<const char*>(A.q + sb.slot * SR * 128),
                          reinterpret_cast<char*>(B.q + rb.slot * SR * 128), 256, 256, rows, 256});
        } else if (db.kind == DCPX_KIND_KV) {
          for (int h = 0; h < 2; ++h)
            jobs.push_back({reinterpret_cast<const char*>(A.kv + (2 * sb.slot + h) * SR * 128),
                            reinterpret_cast<char*>(B.kv + (2 * rb.slot + h) * SR * 128), 256, 256, rows, 256});
        } else {
          const int64_t so = A.o_phys[sb.slot], ro = B.o_phys[rb.slot];
          jobs.push_back({reinterpret_cast<const char*>(A.o + so * SR * 128),
                          reinterpret_cast<char*>(B.o + ro * SR * 128), 256, 256, rows, 256});
          jobs.push_back({reinterpret_cast<const char*>(A.lse + so * SR),
                          reinterpret_cast<char*>(B.lse + ro * SR), 4 * rows, 4 * rows, 1, 4 * rows});
        }
      }
      op.jobs = make_jobs(d, jobs);
      op.xfer = jobs;
      op.peer = src_dev;
    }
  }
}

void Executor::simulate_order() {
  order_.clear();
  const int T = R_ ? plans_[0].divisions : 0;
  comm_bytes_.assign(static_cast<size_t>(T) + 1, {});
  comp_flops_.assign(static_cast<size_t>(T) + 1, std::vector<uint64_t>(static_cast<size_t>(R_), 0));
  wire_fwd_send_.assign(static_cast<size_t>(R_), 0);
  wire_fwd_recv_.assign(static_cast<size_t>(R_), 0);
  std::vector<size_t> pc(static_cast<size_t>(R_), 0);
  std::map<std::string, std::pair<int, int>> inbox;  // tag -> (src, dst)
  std::vector<std::set<std::string>> posted(static_cast<size_t>(R_));
  while (true) {
    bool all_done = true, any = false;
    for (int d = 0; d < R_; ++d) {
      const auto& P = plans_[d];
      if (pc[d] >= P.ins.size()) continue;
      all_done = false;
      while (pc[d] < P.ins.size()) {
        const Instr& I = P.ins[pc[d]];
        if (I.op == DCPX_OP_COMM_WAIT) {
          auto it = inbox.find(I.tag);
          if (it == inbox.end()) break;
          if (it->second.second != d) throw Failure(DCPX_TAG_MISMATCH, "message " + I.tag + " delivered to wrong device");
          if (!posted[d].count(I.tag))
            throw Failure(DCPX_TAG_MISMATCH, "device " + std::to_string(d) + " waits on " + I.tag + " without a posted receive");
          posted[d].erase(I.tag);
          inbox.erase(it);
        } else if (I.op == DCPX_OP_COMM_LAUNCH) {
          if (I.send) {
            if (!inbox.insert({I.tag, {d, I.peer}}).second)
              throw Failure(DCPX_TAG_MISMATCH, "duplicate message tag " + I.tag);
            uint64_t bytes = 0, wire = 0;
            for (int b = 0; b < I.count; ++b) {
              const auto& db = g_.data_blocks[P.blocks[I.offset + b].block];
              bytes += db.size_bytes;
              // an O block travels with its fp32 LSE rows (the reference moves (out, m, l))
              wire += db.size_bytes + (db.kind == DCPX_KIND_O ? 4 * static_cast<uint64_t>(db.tok_end - db.tok_begin) : 0);
            }
            if (I.division >= 0 && I.division <= T) comm_bytes_[I.division][{d, I.peer}] += bytes;
            wire_fwd_send_[d] += wire;
            wire_fwd_recv_[I.peer] += wire;
          } else {
            posted[d].insert(I.tag);
          }
        }
        order_.push_back({d, static_cast<int>(pc[d])});
        ++pc[d];
        any = true;
      }
    }
    if (all_done) break;
    if (!any) {
      std::string msg = "deadlock: ";
      for (int d = 0; d < R_; ++d)
        if (pc[d] < plans_[d].ins.size() && plans_[d].ins[pc[d]].op == DCPX_OP_COMM_WAIT)
          msg += "device " + std::to_string(d) + " waits on " + plans_[d].ins[pc[d]].tag + "; ";
      throw Failure(DCPX_DEADLOCK, msg);  // simexec.hpp:384-394
    }
  }
  if (!inbox.empty()) throw Failure(DCPX_TAG_MISMATCH, "messages left undelivered at termination");  // :396-397
}

// Does any instruction at index >= start read O slot `slot` before overwriting it?

}  // namespace dcpx

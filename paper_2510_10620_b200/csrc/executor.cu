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
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <numeric>
#include <set>

#include "executor.h"

namespace dcpx {

#define CUDA_OK(x)                                                                        \
  do {                                                                                    \
    cudaError_t e__ = (x);                                                                \
    if (e__ != cudaSuccess)                                                               \
      throw Failure(DCPX_CUDA_ERROR, std::string(#x) + ": " + cudaGetErrorString(e__));   \
  } while (0)

namespace {

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

// Current-device cursor for the enqueue loops: switches only when the device changes and
// restores the caller's device at the end (the loops visit thousands of ops per call).
struct DeviceCursor {
  int saved = 0, cur = -1;
  DeviceCursor() { cudaGetDevice(&saved); cur = saved; }
  void to(int d) {
    if (d != cur) {
      cudaSetDevice(d);
      cur = d;
    }
  }
  ~DeviceCursor() {
    if (cur != saved) cudaSetDevice(saved);
  }
};

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CUDA_OK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p) throw Failure(DCPX_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D bf16 tensor map over an arena of `rows` x 128, box `box_rows` rows x 64 columns,
// 128-byte swizzle (matches the UMMA SWIZZLE_128B descriptors in sm100.cuh).
CUtensorMap make_tmap(void* base, int64_t rows, uint32_t box_rows = 128) {
  CUtensorMap m;
  cuuint64_t dims[2] = {128, static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {256};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Failure(DCPX_CUDA_ERROR, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return m;
}

// 2-D fp32 tensor map over a [rows][128] accumulator, box `box_rows` rows x 32 columns
// (128 B), 128-byte swizzle: the TMA reduce-add target of the backward's drain warps.
CUtensorMap make_tmap_f32(void* base, int64_t rows, uint32_t box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {128, static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {512};
  cuuint32_t box[2] = {32, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Failure(DCPX_CUDA_ERROR, "cuTensorMapEncodeTiled (f32) failed: " + std::to_string(r));
  return m;
}

int num_sms(int ordinal) {
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, ordinal);
  return n > 0 ? n : 148;
}

struct RelRange {
  int32_t b0, e0, b1, e1;  // kv-tile-relative, already intersected with [0, n_k)
};

}  // namespace

// ------------------------------------------------------------------------ lifetime
Executor::Executor(int ndev, const int* ordinals) : R_(ndev) {
  if (ndev < 1 || ndev > 64) throw Failure(DCPX_ERROR, "dcpx_create: 1..64 devices supported");
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
    DeviceGuard g(ordinals_[d]);
    dev_[d].ordinal = ordinals_[d];
    set_watchdog_buffer_fwd(diag_);
    set_watchdog_buffer_bwd(diag_);
    CUDA_OK(cudaStreamCreateWithFlags(&dev_[d].cs, cudaStreamNonBlocking));
    int lo = 0, hi = 0;
    CUDA_OK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CUDA_OK(cudaStreamCreateWithPriority(&dev_[d].ms, cudaStreamNonBlocking, hi));  // transfers first
    CUDA_OK(cudaEventCreate(&dev_[d].t0));
    CUDA_OK(cudaEventCreate(&dev_[d].t1));
  }
  if (R_ > 0) {
    DeviceGuard g(ordinals_[0]);
    CUDA_OK(cudaStreamCreateWithFlags(&h2d_, cudaStreamNonBlocking));
    CUDA_OK(cudaStreamCreateWithFlags(&d2h_, cudaStreamNonBlocking));
  }
}

void Executor::await_peer_pulls() {
  if (pulls_done_.empty() || R_ < 2) return;
  for (int d = 0; d < R_; ++d) {
    DeviceGuard g(dev_[d].ordinal);
    for (int e = 0; e < R_; ++e)
      if (e != d && dev_[e].ordinal != dev_[d].ordinal) CUDA_OK(cudaStreamWaitEvent(dev_[d].cs, pulls_done_[e], 0));
  }
}

void Executor::mark_pulls_done() {
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
  for (auto& d : dev_) {
    DeviceGuard g(d.ordinal);
    if (d.cs) cudaStreamSynchronize(d.cs);
    if (d.ms) cudaStreamSynchronize(d.ms);
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
  free_all();
  if (diag_) cudaFreeHost(diag_);
  for (auto& d : dev_) {
    DeviceGuard g(d.ordinal);
    for (auto e : d.events) cudaEventDestroy(e);
    for (auto& e : d.kev) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
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

template <class T>
T* Executor::upload(int d, const std::vector<T>& v) {
  if (v.empty()) return nullptr;
  T* p = static_cast<T*>(alloc(d, v.size() * sizeof(T)));
  DeviceGuard g(dev_[d].ordinal);
  CUDA_OK(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return p;
}

template <class J>
JobList Executor::make_row_jobs(int d, const std::vector<J>& jobs, const std::vector<int>& rows,
                                int rows_per_block) {
  JobList L;
  std::vector<int32_t> job_of_block, first_chunk;
  for (size_t j = 0; j < jobs.size(); ++j) {
    first_chunk.push_back(static_cast<int32_t>(job_of_block.size()));
    const int nb = (rows[j] + rows_per_block - 1) / rows_per_block;
    for (int b = 0; b < nb; ++b) job_of_block.push_back(static_cast<int32_t>(j));
  }
  L.dj.jobs = upload(d, jobs);
  L.dj.job_of_block = upload(d, job_of_block);
  L.dj.first_chunk = upload(d, first_chunk);
  L.dj.n_blocks = static_cast<int32_t>(job_of_block.size());
  L.dj.n_jobs = static_cast<int32_t>(jobs.size());
  return L;
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
int Executor::attn_grid(int d, int grid) const {
  const int reserve = opt.sm_reserve >= 0 ? opt.sm_reserve : (R_ > 1 ? 8 : 0);
  const int cap = std::max(1, num_sms(dev_[d].ordinal) - reserve);
  return std::min(grid, cap);
}

// LOCAL transport on the DMA copy engines: one peer copy per contiguous block component,
// issued on the receiver's comm stream so NVLink traffic never competes with the
// persistent attention kernels for SMs.
void Executor::copy_engine(const std::vector<RowCopyJob>& jobs, cudaStream_t s) {
  for (const auto& j : jobs) {
    if (j.src_stride == j.row_bytes && j.dst_stride == j.row_bytes) {
      CUDA_OK(cudaMemcpyAsync(j.dst, j.src, static_cast<size_t>(j.rows) * j.row_bytes, cudaMemcpyDefault, s));
    } else {
      CUDA_OK(cudaMemcpy2DAsync(j.dst, j.dst_stride, j.src, j.src_stride, j.row_bytes, j.rows, cudaMemcpyDefault, s));
    }
  }
}

// ---- op tracing (option "trace"): device-time spans of every executed op ------------------
void Executor::trace_begin() {
  trace_.clear();
  trace_pending_.clear();
}

TraceScope::TraceScope(Executor* ex, int d, int instr, cudaStream_t s, int pass, const Op& op)
    : ex_(ex), d_(d) {
  if (!ex->opt.trace || op.kind == OpKind::kNop) return;
  auto ev = ex->kernel_events(d);
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
  auto ev = ex_->kernel_events(d_);
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

std::pair<cudaEvent_t, cudaEvent_t> Executor::kernel_events(int d) {
  auto& D = dev_[d];
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
  synchronize();  // asynchronous host I/O of a previous plan may still be in flight
  free_all();
  out_stage_ = nullptr;
  for (Staging* st : {&in_st_, &bwd_st_})
    for (int k = 0; k < 2; ++k) {  // (events stay alive in staging_events_ and are reused)
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
  if (g_.D != kHeadDim) throw Failure(DCPX_UNSUPPORTED, "sm_100a kernels support head_dim 128 only");
  if (g_.bpe != 2) throw Failure(DCPX_UNSUPPORTED, "bf16 payloads (bytes_per_element 2) only");
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

  // ---- per-device compile
  for (int d = 0; d < R_; ++d) {
    dev_[d].slot_rows = slot_rows;
    compile_device(d);
  }
  // ---- LOCAL transport: precompiled transfer jobs, owned by the receiver
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
          jobs.push_back({reinterpret_cast<const char*>(A.q + sb.slot * slot_rows * 128),
                          reinterpret_cast<char*>(B.q + rb.slot * slot_rows * 128), 256, 256, rows, 256});
        } else if (db.kind == DCPX_KIND_KV) {
          for (int h = 0; h < 2; ++h)
            jobs.push_back({reinterpret_cast<const char*>(A.kv + (2 * sb.slot + h) * slot_rows * 128),
                            reinterpret_cast<char*>(B.kv + (2 * rb.slot + h) * slot_rows * 128), 256, 256, rows, 256});
        } else {
          const int64_t so = A.o_phys[sb.slot], ro = B.o_phys[rb.slot];
          jobs.push_back({reinterpret_cast<const char*>(A.o + so * slot_rows * 128),
                          reinterpret_cast<char*>(B.o + ro * slot_rows * 128), 256, 256, rows, 256});
          jobs.push_back({reinterpret_cast<const char*>(A.lse + so * slot_rows),
                          reinterpret_cast<char*>(B.lse + ro * slot_rows), 4 * rows, 4 * rows, 1, 4 * rows});
        }
      }
      op.jobs = make_jobs(d, jobs);
      op.xfer = jobs;
      op.peer = src_dev;
    }
    build_io_jobs(d);
  }
  build_bwd_jobs();
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
  prepared_ = true;
}

void Executor::simulate_order() {
  order_.clear();
  const int T = R_ ? plans_[0].divisions : 0;
  comm_bytes_.assign(static_cast<size_t>(T) + 1, {});
  comp_flops_.assign(static_cast<size_t>(T) + 1, std::vector<uint64_t>(static_cast<size_t>(R_), 0));
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
            uint64_t bytes = 0;
            for (int b = 0; b < I.count; ++b) bytes += g_.data_blocks[P.blocks[I.offset + b].block].size_bytes;
            if (I.division >= 0 && I.division <= T) comm_bytes_[I.division][{d, I.peer}] += bytes;
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
static bool o_read_before_write(const PlanCopy& P, const GraphCopy& g, size_t start, int slot) {
  for (size_t i = start; i < P.ins.size(); ++i) {
    const Instr& I = P.ins[i];
    if (I.op == DCPX_OP_ATTENTION) {
      for (int k = 0; k < I.count; ++k)
        if (P.items[I.offset + k].out_slot == slot) return false;
    } else if (I.op == DCPX_OP_REDUCTION) {
      for (int k = 0; k < I.count; ++k)
        if (P.srcs[I.offset + k] == slot) return true;
      if (I.dst == slot) return false;
    } else if (I.op == DCPX_OP_COPY) {
      for (int k = 0; k < I.count; ++k)
        if (P.copies[I.offset + k].src_slot == slot) return true;
      for (int k = 0; k < I.count; ++k)
        if (P.copies[I.offset + k].dst_slot == slot) return false;
    } else if (I.op == DCPX_OP_COMM_LAUNCH) {
      for (int k = 0; k < I.count; ++k) {
        const auto& tb = P.blocks[I.offset + k];
        if (g.data_blocks[tb.block].kind == DCPX_KIND_O && tb.slot == slot) return I.send ? true : false;
      }
    }
  }
  return false;
}

// Does any instruction at index >= start touch O slot `slot` at all?
static bool o_touched(const PlanCopy& P, const GraphCopy& g, size_t start, int slot) {
  for (size_t i = start; i < P.ins.size(); ++i) {
    const Instr& I = P.ins[i];
    if (I.op == DCPX_OP_ATTENTION) {
      for (int k = 0; k < I.count; ++k)
        if (P.items[I.offset + k].out_slot == slot) return true;
    } else if (I.op == DCPX_OP_REDUCTION) {
      if (I.dst == slot) return true;
      for (int k = 0; k < I.count; ++k)
        if (P.srcs[I.offset + k] == slot) return true;
    } else if (I.op == DCPX_OP_COPY) {
      for (int k = 0; k < I.count; ++k)
        if (P.copies[I.offset + k].src_slot == slot || P.copies[I.offset + k].dst_slot == slot) return true;
    } else if (I.op == DCPX_OP_COMM_LAUNCH) {
      for (int k = 0; k < I.count; ++k) {
        const auto& tb = P.blocks[I.offset + k];
        if (g.data_blocks[tb.block].kind == DCPX_KIND_O && tb.slot == slot) return true;
      }
    }
  }
  return false;
}

struct AttnGroup {
  std::vector<int> items;  // indices into P.items
  int target = 0;          // O slot receiving the merged result
  bool merge_prev = false;
};

void Executor::compile_device(int d) {
  PlanCopy& P = plans_[d];
  DevState& D = dev_[d];
  const int64_t SR = D.slot_rows;
  D.prog.assign(P.ins.size(), Op{});

  // ---- 1. fusion decisions for attention + reductions
  std::vector<bool> fused_red(P.ins.size(), false);
  std::vector<std::vector<AttnGroup>> groups_of(P.ins.size());
  std::vector<int> o_written;  // O slots written by the program
  for (size_t a = 0; a < P.ins.size(); ++a) {
    const Instr& I = P.ins[a];
    if (I.op != DCPX_OP_ATTENTION) continue;
    std::map<int, int> out2item;
    for (int k = 0; k < I.count; ++k) {
      const int idx = static_cast<int>(I.offset) + k;
      if (!out2item.insert({P.items[idx].out_slot, idx}).second)
        throw Failure(DCPX_ERROR, "attention instruction writes one slot twice");
    }
    std::set<int> covered;
    auto& groups = groups_of[a];
    if (opt.fuse_reductions) {
      for (size_t r = a + 1; r < P.ins.size() && P.ins[r].op == DCPX_OP_REDUCTION; ++r) {
        const Instr& Rd = P.ins[r];
        std::vector<int> srcs(P.srcs.begin() + Rd.offset, P.srcs.begin() + Rd.offset + Rd.count);
        const bool dst_in_srcs = std::find(srcs.begin(), srcs.end(), Rd.dst) != srcs.end();
        if (!dst_in_srcs) continue;
        bool ok = true;
        AttnGroup grp;
        grp.target = Rd.dst;
        std::set<int> seen;
        for (int s : srcs) {
          if (!seen.insert(s).second) { ok = false; break; }
          auto it = out2item.find(s);
          if (it == out2item.end()) {
            if (s != Rd.dst) { ok = false; break; }
            continue;  // existing accumulator (earlier division)
          }
          if (covered.count(it->second)) { ok = false; break; }
          grp.items.push_back(it->second);
        }
        if (!ok || grp.items.empty()) continue;
        grp.merge_prev = !out2item.count(Rd.dst);
        const auto& i0 = P.items[grp.items[0]];
        for (int idx : grp.items) {
          const auto& x = P.items[idx];
          if (x.q_slot != i0.q_slot || x.q_begin != i0.q_begin || x.q_end != i0.q_end || x.seq != i0.seq) ok = false;
        }
        for (int s : srcs)
          if (s != Rd.dst && o_read_before_write(P, g_, r + 1, s)) ok = false;
        // the attention's other items must not read the accumulator being merged
        if (!ok) continue;
        for (int idx : grp.items) covered.insert(idx);
        groups.push_back(grp);
        fused_red[r] = true;
      }
    }
    for (int k = 0; k < I.count; ++k) {
      const int idx = static_cast<int>(I.offset) + k;
      if (covered.count(idx)) continue;
      AttnGroup grp;
      grp.items = {idx};
      grp.target = P.items[idx].out_slot;
      groups.push_back(grp);
    }
    for (const auto& grp : groups) o_written.push_back(grp.target);
  }

  // ---- 2. copy remaps and the physical O slot map
  std::vector<int> remap_dst2src(static_cast<size_t>(P.cap[2]), -1);
  std::vector<bool> copy_remapped(P.ins.size(), false);
  for (size_t c = 0; c < P.ins.size(); ++c) {
    const Instr& I = P.ins[c];
    if (I.op != DCPX_OP_COPY || !opt.remap_copies) continue;
    bool ok = true;
    std::set<int> srcs, dsts;
    for (int k = 0; k < I.count; ++k) {
      const auto& ci = P.copies[I.offset + k];
      if (!srcs.insert(ci.src_slot).second || !dsts.insert(ci.dst_slot).second) ok = false;
      if (o_touched(P, g_, c + 1, ci.src_slot) || o_touched(P, g_, c + 1, ci.dst_slot)) ok = false;
    }
    for (int s : srcs)
      if (dsts.count(s)) ok = false;
    // the destination must be a resident output slot that nothing else reads
    if (!ok) continue;
    copy_remapped[c] = true;
    for (int k = 0; k < I.count; ++k) remap_dst2src[P.copies[I.offset + k].dst_slot] = P.copies[I.offset + k].src_slot;
  }
  std::vector<bool> o_used(static_cast<size_t>(P.cap[2]), false);
  for (int s : o_written) o_used[s] = true;
  for (size_t i = 0; i < P.ins.size(); ++i) {
    const Instr& I = P.ins[i];
    if (I.op == DCPX_OP_REDUCTION && !fused_red[i]) {
      o_used[I.dst] = true;
      for (int k = 0; k < I.count; ++k) o_used[P.srcs[I.offset + k]] = true;
    } else if (I.op == DCPX_OP_COPY) {
      for (int k = 0; k < I.count; ++k) {
        o_used[P.copies[I.offset + k].src_slot] = true;
        if (!copy_remapped[i]) o_used[P.copies[I.offset + k].dst_slot] = true;
      }
    } else if (I.op == DCPX_OP_COMM_LAUNCH) {
      for (int k = 0; k < I.count; ++k) {
        const auto& tb = P.blocks[I.offset + k];
        if (g_.data_blocks[tb.block].kind == DCPX_KIND_O) o_used[tb.slot] = true;
      }
    }
  }
  for (const auto& r : P.res_o) {
    const int src = remap_dst2src[r.slot];
    o_used[src >= 0 ? src : r.slot] = true;
  }
  D.o_phys.assign(static_cast<size_t>(P.cap[2]), -1);
  int64_t n_o = 0;
  for (int s = 0; s < P.cap[2]; ++s)
    if (o_used[s]) D.o_phys[s] = static_cast<int32_t>(n_o++);
  D.cap_q = P.cap[0];
  D.cap_kv = P.cap[1];
  D.cap_o = n_o;

  // ---- 3. arenas (zero-initialised: stale rows stay finite) and tensor maps
  {
    DeviceGuard gd(D.ordinal);
    D.q = static_cast<__nv_bfloat16*>(alloc(d, std::max<int64_t>(1, D.cap_q) * SR * 256));
    D.kv = static_cast<__nv_bfloat16*>(alloc(d, std::max<int64_t>(1, D.cap_kv) * 2 * SR * 256));
    D.o = static_cast<__nv_bfloat16*>(alloc(d, std::max<int64_t>(1, D.cap_o) * SR * 256));
    D.lse = static_cast<float*>(alloc(d, std::max<int64_t>(1, D.cap_o) * SR * 4));
    CUDA_OK(cudaMemset(D.q, 0, std::max<int64_t>(1, D.cap_q) * SR * 256));
    CUDA_OK(cudaMemset(D.kv, 0, std::max<int64_t>(1, D.cap_kv) * 2 * SR * 256));
    CUDA_OK(cudaMemset(D.o, 0, std::max<int64_t>(1, D.cap_o) * SR * 256));
    CUDA_OK(cudaMemset(D.lse, 0, std::max<int64_t>(1, D.cap_o) * SR * 4));
    // backward arenas, parallel to the Q arena (dO, LSE*log2e, Delta, dQ accumulator)
    // and to the KV arena (dK / dV accumulators)
    const int64_t nq = std::max<int64_t>(1, D.cap_q), nkv = std::max<int64_t>(1, D.cap_kv);
    D.d_o = static_cast<__nv_bfloat16*>(alloc(d, nq * SR * 256));
    D.lse2 = static_cast<float*>(alloc(d, nq * SR * 4));
    D.delta = static_cast<float*>(alloc(d, nq * SR * 4));
    D.dq_acc = static_cast<float*>(alloc(d, nq * SR * 512));
    D.dkv_acc = static_cast<float*>(alloc(d, nkv * 2 * SR * 512));
    CUDA_OK(cudaMemset(D.d_o, 0, nq * SR * 256));
    CUDA_OK(cudaMemset(D.lse2, 0, nq * SR * 4));
    CUDA_OK(cudaMemset(D.delta, 0, nq * SR * 4));
    D.tm_do = make_tmap(D.d_o, nq * SR, kBwdQRows);
    D.tm_dq = make_tmap_f32(D.dq_acc, nq * SR, kBwdQRows);
    D.tm_q = make_tmap(D.q, std::max<int64_t>(1, D.cap_q) * SR);
    D.tm_q64 = make_tmap(D.q, std::max<int64_t>(1, D.cap_q) * SR, kBwdQRows);
    D.tm_kv = make_tmap(D.kv, std::max<int64_t>(1, D.cap_kv) * 2 * SR);
    D.tm_dkv = make_tmap_f32(D.dkv_acc, nkv * 2 * SR, 128);
    std::vector<int32_t> ranges = g_.ranges;
    ranges.insert(ranges.end(), P.rows.begin(), P.rows.end());
    if (ranges.empty()) ranges.assign(4, 0);
    D.ranges = upload(d, ranges);
  }

  // ---- 4. per-instruction device ops
  const int64_t TT = g_.total_tokens();
  for (size_t i = 0; i < P.ins.size(); ++i) {
    const Instr& I = P.ins[i];
    Op& op = D.prog[i];
    op.division = I.division;
    op.instr = static_cast<int>(i);
    switch (I.op) {
      case DCPX_OP_ATTENTION: {
        op.kind = OpKind::kFwdAttn;
        // -- classify every item once: [128-row q tile][128-col kv sub-tile] -> empty /
        //    partial / full, from the item rows (plan.hpp:231-242 or explicit rows)
        struct ItemCls { int nks = 0, n_qt = 0, n_qb = 0, mask = 0; std::vector<uint8_t> cls, cls_b; };
        std::map<int, ItemCls> icl;
        std::vector<ItemMask> masks;
        for (int k = 0; k < I.count; ++k) {
          const int idx = static_cast<int>(I.offset) + k;
          const auto& it = P.items[idx];
          const int n_q = static_cast<int>(it.q_end - it.q_begin);
          const int n_k = static_cast<int>(it.kv_end - it.kv_begin);
          ItemCls c;
          c.nks = (n_k + 127) / 128;
          c.n_qt = (n_q + 127) / 128;
          c.n_qb = (n_q + kBwdQRows - 1) / kBwdQRows;
          ItemMask im{};
          im.n_k = n_k;
          const int32_t* rg;
          if (it.rows_offset >= 0) {
            im.range_row0 = TT + it.rows_offset;
            im.kv_shift = 0;
            rg = P.rows.data() + 4 * it.rows_offset;
          } else {
            im.range_row0 = g_.seq_offsets[it.seq] + it.q_begin;
            im.kv_shift = it.kv_begin;
            rg = g_.ranges.data() + 4 * (g_.seq_offsets[it.seq] + it.q_begin);
          }
          c.mask = static_cast<int>(masks.size());
          masks.push_back(im);
          std::vector<uint8_t> all_full(static_cast<size_t>(c.n_qt) * c.nks, 1), any(static_cast<size_t>(c.n_qt) * c.nks, 0);
          // the backward's 64-row q tiles
          std::vector<uint8_t> all_full_b(static_cast<size_t>(c.n_qb) * c.nks, 1), any_b(static_cast<size_t>(c.n_qb) * c.nks, 0);
          uint64_t pairs = 0;
          for (int r = 0; r < n_q; ++r) {
            RelRange rr;
            const int64_t sh = im.kv_shift;
            rr.b0 = static_cast<int32_t>(std::max<int64_t>(rg[4 * r] - sh, 0));
            rr.e0 = static_cast<int32_t>(std::min<int64_t>(rg[4 * r + 1] - sh, n_k));
            rr.b1 = static_cast<int32_t>(std::max<int64_t>(rg[4 * r + 2] - sh, 0));
            rr.e1 = static_cast<int32_t>(std::min<int64_t>(rg[4 * r + 3] - sh, n_k));
            if (it.rows_offset >= 0 && (rg[4 * r] < 0 || rg[4 * r + 1] > n_k || rg[4 * r + 2] < 0 || rg[4 * r + 3] > n_k) &&
                (rg[4 * r + 1] > rg[4 * r] || rg[4 * r + 3] > rg[4 * r + 2]))
              throw Failure(DCPX_ERROR, "exec_attention: range outside kv tile");  // simexec.hpp:53
            if (rr.e0 > rr.b0) pairs += rr.e0 - rr.b0;
            if (rr.e1 > rr.b1) pairs += rr.e1 - rr.b1;
            const int qt = r / 128;
            for (int ks = 0; ks < c.nks; ++ks) {
              const int c0 = ks * 128, c1 = std::min(n_k, c0 + 128);
              const bool full = (c1 - c0 == 128) && ((rr.b0 <= c0 && rr.e0 >= c1) || (rr.b1 <= c0 && rr.e1 >= c1));
              const bool hit = (rr.e0 > rr.b0 && rr.b0 < c1 && rr.e0 > c0) || (rr.e1 > rr.b1 && rr.b1 < c1 && rr.e1 > c0);
              if (!full) all_full[qt * c.nks + ks] = 0;
              if (hit) any[qt * c.nks + ks] = 1;
              if (!full) all_full_b[(r / kBwdQRows) * c.nks + ks] = 0;
              if (hit) any_b[(r / kBwdQRows) * c.nks + ks] = 1;
            }
          }
          op.flops += 4ull * pairs * static_cast<uint64_t>(g_.D);
          c.cls.resize(static_cast<size_t>(c.n_qt) * c.nks);
          for (size_t q = 0; q < c.cls.size(); ++q)
            c.cls[q] = !any[q] ? kTileEmpty : (all_full[q] ? kTileFull : kTilePartial);
          c.cls_b.resize(static_cast<size_t>(c.n_qb) * c.nks);
          for (size_t q = 0; q < c.cls_b.size(); ++q)
            c.cls_b[q] = !any_b[q] ? kTileEmpty : (all_full_b[q] ? kTileFull : kTilePartial);
          icl[idx] = std::move(c);
        }
        // -- forward units: one per (group, pair of 128-row q tiles)
        std::vector<FwdUnit> units;
        std::vector<FwdStep> steps;
        std::vector<int64_t> unit_cost;
        for (const auto& grp : groups_of[i]) {
          const auto& i0 = P.items[grp.items[0]];
          const int n_q = static_cast<int>(i0.q_end - i0.q_begin);
          const int n_pairs = (n_q + 255) / 256;
          const int n_qt = (n_q + 127) / 128;
          for (int pr = 0; pr < n_pairs; ++pr) {
            FwdUnit U{};
            U.q_row0 = static_cast<int32_t>(i0.q_slot * SR + 256 * pr);
            U.n_rows = std::min(256, n_q - 256 * pr);
            U.out_row0 = static_cast<int32_t>(D.o_phys[grp.target] * SR + 256 * pr);
            U.flags = grp.merge_prev ? 1 : 0;
            U.q_local0 = 256 * pr;
            U.step_begin = static_cast<int32_t>(steps.size());
            int64_t cost = 0;
            for (int idx : grp.items) {
              const auto& it = P.items[idx];
              const auto& c = icl.at(idx);
              for (int ks = 0; ks < c.nks; ++ks) {
                const uint32_t c0 = c.cls[(2 * pr) * c.nks + ks];
                const uint32_t c1 = (2 * pr + 1 < n_qt) ? c.cls[(2 * pr + 1) * c.nks + ks] : kTileEmpty;
                if (!c0 && !c1) continue;
                FwdStep S{};
                S.kv_row0 = static_cast<int32_t>(2 * it.kv_slot * SR + 128 * ks);
                S.col0 = 128 * ks;
                S.item = c.mask;
                S.cls = c0 | (c1 << 2);
                steps.push_back(S);
                cost += (c0 ? 1 : 0) + (c1 ? 1 : 0);
              }
            }
            U.step_count = static_cast<int32_t>(steps.size()) - U.step_begin;
            units.push_back(U);
            unit_cost.push_back(cost * 1000 + U.n_rows);
          }
        }
        // longest-processing-time-first order for the static round-robin schedule
        std::vector<size_t> order(units.size());
        std::iota(order.begin(), order.end(), 0);
        std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return unit_cost[a] > unit_cost[b]; });
        std::vector<FwdUnit> sorted;
        for (size_t k : order) sorted.push_back(units[k]);
        op.units = upload(d, sorted);
        op.steps = upload(d, steps);
        op.items = upload(d, masks);
        op.num_units = static_cast<int>(sorted.size());
        op.grid = std::min(op.num_units, num_sms(D.ordinal));
        // -- backward units: one per (kv slot, 128-row kv sub-tile, window of bwd_window
        //    q tiles of one item). Windowing bounds the rows a wave of CTAs touches: with
        //    units ordered by q window, the CTAs running at once stream the same Q / dO
        //    tiles and reduce into the same fp32 dQ rows, which then stay in L2 instead
        //    of making an HBM round trip per step; dK / dV are flushed per unit.
        std::map<int, std::vector<int>> by_kv;
        for (int k = 0; k < I.count; ++k) by_kv[P.items[I.offset + k].kv_slot].push_back(static_cast<int>(I.offset) + k);
        std::vector<BwdUnit> bunits;
        std::vector<BwdStep> bsteps;
        std::vector<int64_t> bcost;
        std::vector<std::pair<int64_t, int64_t>> bkey;
        // windowing pays off for long units only: count the steps of the whole-item units
        // first and window (with q-window-major order) when they average enough steps;
        // short units (very sparse masks) stay whole, longest first
        int64_t whole_units = 0, whole_steps = 0;
        for (const auto& [kv_slot, idxs] : by_kv) {
          const auto& c0 = icl.at(idxs[0]);
          for (int ks = 0; ks < c0.nks; ++ks) {
            int64_t n = 0;
            for (int idx : idxs) {
              const auto& c = icl.at(idx);
              for (int qt = 0; qt < c.n_qb; ++qt) n += c.cls_b[qt * c.nks + ks] != 0;
            }
            whole_units += n > 0;
            whole_steps += n;
          }
        }
        const bool windowed = opt.bwd_window > 0 && whole_steps >= int64_t{opt.bwd_window_min_steps} * whole_units;
        const int win = windowed ? opt.bwd_window : (1 << 30);
        const int border_mode = windowed ? opt.bwd_order : 0;
        for (const auto& [kv_slot, idxs] : by_kv) {
          const auto& f = P.items[idxs[0]];
          const int n_k = static_cast<int>(f.kv_end - f.kv_begin);
          const int nks = (n_k + 127) / 128;
          for (int ks = 0; ks < nks; ++ks) {
            BwdUnit U{};
            U.kv_row0 = static_cast<int32_t>(2 * kv_slot * SR + 128 * ks);
            U.n_kv = std::min(128, n_k - 128 * ks);
            U.step_begin = static_cast<int32_t>(bsteps.size());
            int64_t cur_window = -1;
            auto close = [&]() {
              U.step_count = static_cast<int32_t>(bsteps.size()) - U.step_begin;
              if (U.step_count > 0) {
                bunits.push_back(U);
                bcost.push_back(U.step_count);
                bkey.emplace_back(bsteps[U.step_begin].q_row0, U.kv_row0);
              }
              U.step_begin = static_cast<int32_t>(bsteps.size());
            };
            for (int idx : idxs) {
              const auto& it = P.items[idx];
              if (it.kv_end - it.kv_begin != n_k) throw Failure(DCPX_ERROR, "kv slot read with two sizes in one instruction");
              const auto& c = icl.at(idx);
              const int n_q = static_cast<int>(it.q_end - it.q_begin);
              for (int qt = 0; qt < c.n_qb; ++qt) {
                const uint32_t cl = c.cls_b[qt * c.nks + ks];
                if (!cl) continue;
                const int64_t window = static_cast<int64_t>(idx) * (1 << 20) + qt / win;
                if (window != cur_window) {
                  close();
                  cur_window = window;
                }
                BwdStep S{};
                S.q_row0 = static_cast<int32_t>(it.q_slot * SR + kBwdQRows * qt);
                S.n_q = std::min(kBwdQRows, n_q - kBwdQRows * qt);
                S.item = c.mask;
                S.q_local0 = kBwdQRows * qt;
                S.col0 = 128 * ks;
                S.cls = cl;
                bsteps.push_back(S);
              }
            }
            close();
          }
        }
        std::vector<size_t> border(bunits.size());
        std::iota(border.begin(), border.end(), 0);
        // bwd_order 0: longest-first; 1: plan order (kv slot, sub-tile, q window);
        // 2: q window major, so consecutive units (one wave) share their Q / dO / dQ rows
        if (border_mode == 0)
          std::stable_sort(border.begin(), border.end(), [&](size_t a, size_t b) { return bcost[a] > bcost[b]; });
        else if (border_mode == 2)
          std::stable_sort(border.begin(), border.end(), [&](size_t a, size_t b) {
            const int64_t wa = bkey[a].first / (int64_t{kBwdQRows} * std::min(win, 1 << 20));
            const int64_t wb = bkey[b].first / (int64_t{kBwdQRows} * std::min(win, 1 << 20));
            return wa != wb ? wa < wb : bkey[a].second < bkey[b].second;
          });
        std::vector<BwdUnit> bsorted;
        for (size_t k : border) bsorted.push_back(bunits[k]);
        op.bunits = upload(d, bsorted);
        op.bsteps = upload(d, bsteps);
        op.bitems = op.items;
        op.bnum_units = static_cast<int>(bsorted.size());
        op.bgrid = std::min(op.bnum_units, num_sms(D.ordinal));
        if (I.division >= 0 && I.division < static_cast<int>(comp_flops_.size())) comp_flops_[I.division][d] += op.flops;
        break;
      }
      case DCPX_OP_REDUCTION: {
        if (fused_red[i]) { op.kind = OpKind::kNop; break; }
        op.kind = OpKind::kMerge;
        MergeJob J{};
        J.dst_row0 = static_cast<int32_t>(D.o_phys[I.dst] * SR);
        J.n_rows = static_cast<int32_t>(SR);
        J.src_begin = 0;
        J.n_src = I.count;
        for (int k = 0; k < I.count; ++k) op.msrc.push_back(static_cast<int32_t>(D.o_phys[P.srcs[I.offset + k]] * SR));
        op.mjobs.push_back(J);
        break;
      }
      case DCPX_OP_COPY: {
        if (copy_remapped[i]) { op.kind = OpKind::kNop; break; }
        op.kind = OpKind::kCopy;
        std::vector<RowCopyJob> jobs;
        for (int k = 0; k < I.count; ++k) {
          const auto& ci = P.copies[I.offset + k];
          const int64_t s = D.o_phys[ci.src_slot], t = D.o_phys[ci.dst_slot];
          jobs.push_back({reinterpret_cast<const char*>(D.o + s * SR * 128), reinterpret_cast<char*>(D.o + t * SR * 128),
                          256, 256, static_cast<int32_t>(SR), 256});
          jobs.push_back({reinterpret_cast<const char*>(D.lse + s * SR), reinterpret_cast<char*>(D.lse + t * SR),
                          static_cast<int64_t>(SR) * 4, static_cast<int64_t>(SR) * 4, 1, static_cast<int32_t>(SR * 4)});
        }
        op.jobs = make_jobs(d, jobs);
        break;
      }
      case DCPX_OP_COMM_LAUNCH: {
        op.kind = OpKind::kCommLaunch;
        op.send = I.send;
        op.peer = I.peer;
        op.tag = I.tag;
        op.blocks.assign(P.blocks.begin() + I.offset, P.blocks.begin() + I.offset + I.count);
        for (const auto& tb : op.blocks) op.bytes += g_.data_blocks[tb.block].size_bytes;
        if (I.send) {
          // Q / KV sends read resident slots, written only by dcpx_load_inputs
          std::set<int> res_q, res_kv;
          for (const auto& r : P.res_q) res_q.insert(r.slot);
          for (const auto& r : P.res_kv) res_kv.insert(r.slot);
          op.resident_only = true;
          for (const auto& tb : op.blocks) {
            const int kd = g_.data_blocks[tb.block].kind;
            if (!((kd == DCPX_KIND_Q && res_q.count(tb.slot)) || (kd == DCPX_KIND_KV && res_kv.count(tb.slot))))
              op.resident_only = false;
          }
        }
        if (I.send) {  // snapshot semantics: the sent slots must not be rewritten afterwards
          for (const auto& tb : op.blocks)
            if (g_.data_blocks[tb.block].kind == DCPX_KIND_O && o_touched(P, g_, i + 1, tb.slot)) {
              for (size_t k = i + 1; k < P.ins.size(); ++k) {
                const Instr& X = P.ins[k];
                bool writes = (X.op == DCPX_OP_REDUCTION && X.dst == tb.slot);
                for (int q = 0; X.op == DCPX_OP_ATTENTION && q < X.count; ++q)
                  writes |= P.items[X.offset + q].out_slot == tb.slot;
                if (writes) throw Failure(DCPX_UNSUPPORTED, "plan overwrites a slot with an in-flight send");
              }
            }
        }
        break;
      }
      case DCPX_OP_COMM_WAIT:
        op.kind = OpKind::kCommWait;
        op.tag = I.tag;
        break;
    }
  }
  // ---- 5. batch runs of independent consecutive reductions into one merge launch
  for (size_t i = 0; i < D.prog.size(); ++i) {
    if (D.prog[i].kind != OpKind::kMerge) continue;
    Op& head = D.prog[i];
    std::set<int32_t> touched;  // O-arena rows written or read by the run
    for (const auto& J : head.mjobs) touched.insert(J.dst_row0);
    for (int32_t r : head.msrc) touched.insert(r);
    size_t k = i + 1;
    for (; k < D.prog.size(); ++k) {
      Op& o2 = D.prog[k];
      if (o2.kind == OpKind::kNop) continue;
      if (o2.kind != OpKind::kMerge) break;
      bool clash = touched.count(o2.mjobs[0].dst_row0) > 0;
      for (int32_t r : o2.msrc) clash |= touched.count(r) > 0 && r != o2.mjobs[0].dst_row0;
      if (clash) break;
      MergeJob J = o2.mjobs[0];
      J.src_begin = static_cast<int32_t>(head.msrc.size());
      head.mjobs.push_back(J);
      head.msrc.insert(head.msrc.end(), o2.msrc.begin(), o2.msrc.end());
      touched.insert(J.dst_row0);
      touched.insert(o2.msrc.begin(), o2.msrc.end());
      o2.kind = OpKind::kNop;
    }
    std::vector<int> rows;
    for (const auto& J : head.mjobs) rows.push_back(J.n_rows);
    head.src_rows = upload(d, head.msrc);
    head.jobs = make_row_jobs(d, head.mjobs, rows, 16);
    i = k - 1;
  }
  // final output slots (after copy remaps)
  D.final_o_slot.clear();
  for (const auto& r : P.res_o) {
    const int src = remap_dst2src[r.slot];
    D.final_o_slot.push_back(D.o_phys[src >= 0 ? src : r.slot]);
  }
}

void Executor::build_io_jobs(int d) {
  const PlanCopy& P = plans_[d];
  DevState& D = dev_[d];
  const int64_t SR = D.slot_rows, H = g_.H, G = g_.G, TT = g_.total_tokens();
  std::vector<RowCopyJob> sq, sk, sv, go, gl;
  for (const auto& r : P.res_q) {
    const auto& db = g_.data_blocks[r.block];
    const int64_t tok = g_.seq_offsets[db.seq] + db.tok_begin;
    sq.push_back({reinterpret_cast<const char*>((tok * H + db.head) * 256),
                  reinterpret_cast<char*>(D.q + r.slot * SR * 128), H * 256, 256,
                  static_cast<int32_t>(db.tok_end - db.tok_begin), 256});
  }
  for (const auto& r : P.res_kv) {
    const auto& db = g_.data_blocks[r.block];
    const int64_t tok = g_.seq_offsets[db.seq] + db.tok_begin;
    for (int h = 0; h < 2; ++h)
      (h ? sv : sk).push_back({reinterpret_cast<const char*>((tok * G + db.head) * 256),
                               reinterpret_cast<char*>(D.kv + (2 * r.slot + h) * SR * 128), G * 256, 256,
                               static_cast<int32_t>(db.tok_end - db.tok_begin), 256});
  }
  for (size_t i = 0; i < P.res_o.size(); ++i) {
    const auto& db = g_.data_blocks[P.res_o[i].block];
    const int64_t tok = g_.seq_offsets[db.seq] + db.tok_begin;
    const int64_t phys = D.final_o_slot[i];
    const int rows = static_cast<int>(db.tok_end - db.tok_begin);
    go.push_back({reinterpret_cast<const char*>(D.o + phys * SR * 128), reinterpret_cast<char*>((tok * H + db.head) * 256),
                  256, H * 256, rows, 256});
    gl.push_back({reinterpret_cast<const char*>(D.lse + phys * SR), reinterpret_cast<char*>((db.head * TT + tok) * 4),
                  4 * rows, 4 * rows, 1, 4 * rows});
  }
  D.scatter_q = make_jobs(d, sq);
  D.scatter_k = make_jobs(d, sk);
  D.scatter_v = make_jobs(d, sv);
  D.gather_o = make_jobs(d, go);
  D.gather_lse = make_jobs(d, gl);
}

void Executor::build_bwd_jobs() {
  const int T = R_ ? plans_[0].divisions : 0;
  const int64_t TT = g_.total_tokens(), H = g_.H, G = g_.G;
  bwd_send_.assign(static_cast<size_t>(R_), 0);
  bwd_recv_.assign(static_cast<size_t>(R_), 0);
  std::map<int, std::pair<int, int>> owner;  // resident Q / KV block -> (device, slot)
  for (int d = 0; d < R_; ++d) {
    for (const auto& r : plans_[d].res_q) owner[r.block] = {d, r.slot};
    for (const auto& r : plans_[d].res_kv) owner[r.block] = {d, r.slot};
  }
  for (int d = 0; d < R_; ++d) {
    const PlanCopy& P = plans_[d];
    DevState& D = dev_[d];
    const int64_t SR = D.slot_rows;
    // 1. backward fetch payloads: Q + dO + LSE + Delta for Q blocks, K + V for KV blocks
    for (size_t i = 0; i < P.ins.size(); ++i) {
      Op& op = D.prog[i];
      if (op.kind != OpKind::kCommWait || P.ins[i].division >= T) continue;
      int recv_i = -1;
      for (size_t k = 0; k < P.ins.size(); ++k)
        if (P.ins[k].op == DCPX_OP_COMM_LAUNCH && !P.ins[k].send && P.ins[k].tag == op.tag) recv_i = static_cast<int>(k);
      const Instr& RI = P.ins[recv_i];
      const int src_dev = RI.peer;
      const PlanCopy& S = plans_[src_dev];
      int send_i = -1;
      for (size_t k = 0; k < S.ins.size(); ++k)
        if (S.ins[k].op == DCPX_OP_COMM_LAUNCH && S.ins[k].send && S.ins[k].tag == op.tag) send_i = static_cast<int>(k);
      const Instr& SI = S.ins[send_i];
      const DevState& A = dev_[src_dev];
      std::vector<RowCopyJob> jobs;
      for (int b = 0; b < RI.count; ++b) {
        const auto rb = P.blocks[RI.offset + b];
        const auto sb = S.blocks[SI.offset + b];
        const auto& db = g_.data_blocks[rb.block];
        const int rows = static_cast<int>(db.tok_end - db.tok_begin);
        if (db.kind == DCPX_KIND_Q) {
          jobs.push_back({reinterpret_cast<const char*>(A.q + sb.slot * SR * 128), reinterpret_cast<char*>(D.q + rb.slot * SR * 128), 256, 256, rows, 256});
          jobs.push_back({reinterpret_cast<const char*>(A.d_o + sb.slot * SR * 128), reinterpret_cast<char*>(D.d_o + rb.slot * SR * 128), 256, 256, rows, 256});
          jobs.push_back({reinterpret_cast<const char*>(A.lse2 + sb.slot * SR), reinterpret_cast<char*>(D.lse2 + rb.slot * SR), 4 * rows, 4 * rows, 1, 4 * rows});
          jobs.push_back({reinterpret_cast<const char*>(A.delta + sb.slot * SR), reinterpret_cast<char*>(D.delta + rb.slot * SR), 4 * rows, 4 * rows, 1, 4 * rows});
          bwd_send_[src_dev] += 2 * db.size_bytes; bwd_recv_[d] += 2 * db.size_bytes;  // Q + dO out
          bwd_send_[d] += db.size_bytes; bwd_recv_[src_dev] += db.size_bytes;          // dQ back
        } else if (db.kind == DCPX_KIND_KV) {
          for (int h = 0; h < 2; ++h)
            jobs.push_back({reinterpret_cast<const char*>(A.kv + (2 * sb.slot + h) * SR * 128),
                            reinterpret_cast<char*>(D.kv + (2 * rb.slot + h) * SR * 128), 256, 256, rows, 256});
          bwd_send_[src_dev] += db.size_bytes; bwd_recv_[d] += db.size_bytes;  // K, V out
          bwd_send_[d] += db.size_bytes; bwd_recv_[src_dev] += db.size_bytes;  // dK, dV back
        }
      }
      op.bjobs = make_jobs(d, jobs);
      op.bxfer = jobs;
    }
    // 2. gradient returns of fetched blocks, right after the attention of their last use
    std::map<int, int> cur_q, cur_kv;                    // slot -> fetched block
    std::map<int, std::pair<size_t, int>> last_q, last_kv;  // block -> (attention instr, slot)
    for (size_t i = 0; i < P.ins.size(); ++i) {
      const Instr& I = P.ins[i];
      if (I.op == DCPX_OP_COMM_LAUNCH && !I.send && I.division < T) {
        for (int b = 0; b < I.count; ++b) {
          const auto tb = P.blocks[I.offset + b];
          const int k = g_.data_blocks[tb.block].kind;
          if (k == DCPX_KIND_Q) cur_q[tb.slot] = tb.block;
          else if (k == DCPX_KIND_KV) cur_kv[tb.slot] = tb.block;
        }
      } else if (I.op == DCPX_OP_ATTENTION) {
        for (int k = 0; k < I.count; ++k) {
          const auto& it = P.items[I.offset + k];
          auto q = cur_q.find(it.q_slot);
          if (q != cur_q.end()) last_q[q->second] = {i, it.q_slot};
          auto kv = cur_kv.find(it.kv_slot);
          if (kv != cur_kv.end()) last_kv[kv->second] = {i, it.kv_slot};
        }
      }
    }
    std::map<size_t, std::vector<RowCopyJob>> ret;
    for (const auto& [block, use] : last_q) {
      const auto [o, so] = owner.at(block);
      const auto& db = g_.data_blocks[block];
      ret[use.first].push_back({reinterpret_cast<const char*>(D.dq_acc + use.second * SR * 128),
                                reinterpret_cast<char*>(dev_[o].dq_acc + so * SR * 128), 512, 512,
                                static_cast<int32_t>(db.tok_end - db.tok_begin), 512});
    }
    for (const auto& [block, use] : last_kv) {
      const auto [o, so] = owner.at(block);
      const auto& db = g_.data_blocks[block];
      for (int h = 0; h < 2; ++h)
        ret[use.first].push_back({reinterpret_cast<const char*>(D.dkv_acc + (2 * use.second + h) * SR * 128),
                                  reinterpret_cast<char*>(dev_[o].dkv_acc + (2 * so + h) * SR * 128), 512, 512,
                                  static_cast<int32_t>(db.tok_end - db.tok_begin), 512});
    }
    for (auto& [i, jobs] : ret) D.prog[i].ret = make_jobs(d, jobs);
    // 3. io: dO scatter to the resident Q slots, Delta/LSE preprocess, gradient gathers
    std::map<std::tuple<int, int, int>, int> qslot_of;  // (seq, head, tile) -> resident Q slot
    for (const auto& r : P.res_q) {
      const auto& db = g_.data_blocks[r.block];
      qslot_of[{db.seq, db.head, db.tile}] = r.slot;
    }
    std::vector<RowCopyJob> sdo;
    std::vector<RowJob> prep, gq, gk, gv;
    std::vector<int> prep_rows, gq_rows, gk_rows;
    for (size_t k = 0; k < P.res_o.size(); ++k) {
      const auto& db = g_.data_blocks[P.res_o[k].block];
      auto it = qslot_of.find({db.seq, db.head, db.tile});
      if (it == qslot_of.end()) throw Failure(DCPX_ERROR, "output block without a co-located Q block (blocks.hpp:42-51)");
      const int64_t tok = g_.seq_offsets[db.seq] + db.tok_begin;
      const int rows = static_cast<int>(db.tok_end - db.tok_begin);
      sdo.push_back({reinterpret_cast<const char*>((tok * H + db.head) * 256), reinterpret_cast<char*>(D.d_o + it->second * SR * 128),
                     H * 256, 256, rows, 256});
      prep.push_back({D.final_o_slot[k] * SR, it->second * SR, 0, rows, 0});
      prep_rows.push_back(rows);
    }
    for (const auto& r : P.res_q) {
      const auto& db = g_.data_blocks[r.block];
      const int64_t tok = g_.seq_offsets[db.seq] + db.tok_begin;
      const int rows = static_cast<int>(db.tok_end - db.tok_begin);
      gq.push_back({r.slot * SR, (tok * H + db.head) * 128, H * 128, rows, 0});
      gq_rows.push_back(rows);
    }
    for (const auto& r : P.res_kv) {
      const auto& db = g_.data_blocks[r.block];
      const int64_t tok = g_.seq_offsets[db.seq] + db.tok_begin;
      const int rows = static_cast<int>(db.tok_end - db.tok_begin);
      gk.push_back({2 * r.slot * SR, (tok * G + db.head) * 128, G * 128, rows, 0});
      gv.push_back({(2 * r.slot + 1) * SR, (tok * G + db.head) * 128, G * 128, rows, 0});
      gk_rows.push_back(rows);
    }
    D.scatter_do = make_jobs(d, sdo);
    D.prep = make_row_jobs(d, prep, prep_rows, 16);
    D.gather_dq = make_row_jobs(d, gq, gq_rows, 16);
    D.gather_dk = make_row_jobs(d, gk, gk_rows, 16);
    D.gather_dv = make_row_jobs(d, gv, gk_rows, 16);
  }
  (void)TT;
}

// ------------------------------------------------------------------------ execution
void Executor::load_inputs(const void* const* q, const void* const* k, const void* const* v, bool host) {
  if (!prepared_) throw Failure(DCPX_ERROR, "dcpx_load_inputs before dcpx_prepare");
  const int64_t TT = g_.total_tokens();
  std::vector<const void*> sq(q, q + R_), sk(k, k + R_), sv(v, v + R_);
  int slot = -1;
  if (host) {
    // upload into staging slot k on the h2d stream once the slot's previous scatters are
    // done; peers read it over NVLink. The call returns without waiting for the copy.
    DevState& D0 = dev_[0];
    DeviceGuard gd(D0.ordinal);
    const size_t bq = TT * g_.H * 256, bk = TT * g_.G * 256;
    slot = in_st_.next;
    in_st_.next ^= 1;
    char*& buf = in_st_.buf[slot];
    if (!buf) buf = static_cast<char*>(alloc(0, bq + 2 * bk));
    for (cudaEvent_t e : in_st_.free[slot]) CUDA_OK(cudaStreamWaitEvent(h2d_, e, 0));
    CUDA_OK(cudaMemcpyAsync(buf, q[0], bq, cudaMemcpyHostToDevice, h2d_));
    CUDA_OK(cudaMemcpyAsync(buf + bq, k[0], bk, cudaMemcpyHostToDevice, h2d_));
    CUDA_OK(cudaMemcpyAsync(buf + bq + bk, v[0], bk, cudaMemcpyHostToDevice, h2d_));
    if (!in_st_.up[slot]) in_st_.up[slot] = staging_event(0);
    cudaEvent_t up = in_st_.up[slot];
    CUDA_OK(cudaEventRecord(up, h2d_));
    for (int d = 0; d < R_; ++d) {
      DeviceGuard g2(dev_[d].ordinal);
      CUDA_OK(cudaStreamWaitEvent(dev_[d].cs, up, 0));
    }
    std::fill(sq.begin(), sq.end(), buf);
    std::fill(sk.begin(), sk.end(), buf + bq);
    std::fill(sv.begin(), sv.end(), buf + bq + bk);
  }
  await_peer_pulls();  // resident slots may still be read by a peer's previous-call pull
  for (int d = 0; d < R_; ++d) {
    DevState& D = dev_[d];
    DeviceGuard gd(D.ordinal);
    launch_row_copy(D.scatter_q.dj, D.cs, reinterpret_cast<int64_t>(sq[d]), 0);
    launch_row_copy(D.scatter_k.dj, D.cs, reinterpret_cast<int64_t>(sk[d]), 0);
    launch_row_copy(D.scatter_v.dj, D.cs, reinterpret_cast<int64_t>(sv[d]), 0);
    CUDA_OK(cudaGetLastError());
  }
  if (slot >= 0) {  // the slot is free again once every device has scattered from it
    auto& fr = in_st_.free[slot];
    if (fr.empty())
      for (int d = 0; d < R_; ++d) fr.push_back(staging_event(d));
    for (int d = 0; d < R_; ++d) {
      DeviceGuard gd(dev_[d].ordinal);
      CUDA_OK(cudaEventRecord(fr[d], dev_[d].cs));
    }
  }
}

void Executor::forward(void* const* o_out, float* const* lse_out, dcpx_report* rep, bool host) {
  if (!prepared_) throw Failure(DCPX_ERROR, "dcpx_forward before dcpx_prepare");
  const int64_t TT = g_.total_tokens();
  for (auto& D : dev_) {
    D.next_event = 0;
    D.next_kev = 0;
    D.launches = 0;
    DeviceGuard gd(D.ordinal);
    if (opt.timing) CUDA_OK(cudaEventRecord(D.t0, D.cs));
  }
  await_peer_pulls();
  std::map<std::string, cudaEvent_t> send_ev, recv_ev;
  std::vector<cudaEvent_t> ready_ev(static_cast<size_t>(R_));
  for (int d = 0; d < R_; ++d) {  // resident Q / KV were scattered on cs before this call
    DeviceGuard gd(dev_[d].ordinal);
    ready_ev[d] = event(d);
    CUDA_OK(cudaEventRecord(ready_ev[d], dev_[d].cs));
  }
  trace_begin();
  DeviceCursor cursor;
  for (const auto& [d, i] : fwd_live_) {
    DevState& D = dev_[d];
    Op& op = D.prog[i];
    cursor.to(D.ordinal);
    TraceScope ts(this, d, static_cast<int>(i), op.kind == OpKind::kCommWait ? D.ms : D.cs, 0, op);
    switch (op.kind) {
      case OpKind::kFwdAttn: {
        if (!op.num_units) break;
        FwdParams p{};
        p.units = op.units; p.steps = op.steps; p.items = op.items; p.ranges = D.ranges;
        p.o_arena = D.o; p.lse_arena = D.lse; p.num_units = op.num_units;
        p.slot_rows = static_cast<int32_t>(D.slot_rows);
        p.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(g_.D)));
        std::pair<cudaEvent_t, cudaEvent_t> ke{};
        if (opt.kernel_timing) { ke = kernel_events(d); CUDA_OK(cudaEventRecord(ke.first, D.cs)); }
        launch_attn_fwd(D.tm_q, D.tm_kv, p, attn_grid(d, op.grid), D.cs);
        if (opt.kernel_timing) CUDA_OK(cudaEventRecord(ke.second, D.cs));
        ++D.launches;
        break;
      }
      case OpKind::kMerge:
        launch_merge(op.jobs.dj, op.src_rows, D.o, D.lse, D.cs);
        ++D.launches;
        break;
      case OpKind::kCopy:
        launch_row_copy(op.jobs.dj, D.cs);
        ++D.launches;
        break;
      case OpKind::kCommLaunch: {
        if (op.send && op.resident_only) {
          send_ev[op.tag] = ready_ev[d];  // resident inputs: ready since load / preprocess
        } else {
          cudaEvent_t e = event(d);
          CUDA_OK(cudaEventRecord(e, D.cs));
          (op.send ? send_ev : recv_ev)[op.tag] = e;
        }
        break;
      }
      case OpKind::kCommWait: {
        CUDA_OK(cudaStreamWaitEvent(D.ms, send_ev.at(op.tag), 0));
        CUDA_OK(cudaStreamWaitEvent(D.ms, recv_ev.at(op.tag), 0));
        ts.split(kTraceXfer);
        if (opt.sm_transfers) {
          launch_row_copy(op.jobs.dj, D.ms);
          ++D.launches;
        } else {
          copy_engine(op.xfer, D.ms);
        }
        cudaEvent_t e = event(d);
        CUDA_OK(cudaEventRecord(e, D.ms));
        CUDA_OK(cudaStreamWaitEvent(D.cs, e, 0));
        break;
      }
      case OpKind::kNop:
        break;
    }
  }
  mark_pulls_done();
  // output assembly (simexec.hpp:403-421) into the caller's packed buffers
  std::vector<char*> o_dev(static_cast<size_t>(R_)), l_dev(static_cast<size_t>(R_));
  for (int d = 0; d < R_; ++d) {
    o_dev[d] = static_cast<char*>(o_out ? o_out[d] : nullptr);
    l_dev[d] = reinterpret_cast<char*>(lse_out ? lse_out[d] : nullptr);
  }
  const bool want_o = o_dev[0] != nullptr, want_l = l_dev[0] != nullptr;
  if (host && (want_o || want_l)) {
    if (!out_stage_) out_stage_ = static_cast<char*>(alloc(0, TT * g_.H * 256 + TT * g_.H * 4));
    std::fill(o_dev.begin(), o_dev.end(), want_o ? out_stage_ : nullptr);
    std::fill(l_dev.begin(), l_dev.end(), want_l ? out_stage_ + TT * g_.H * 256 : nullptr);
  }
  for (int d = 0; d < R_; ++d) {
    DevState& D = dev_[d];
    DeviceGuard gd(D.ordinal);
    if (o_dev[d]) { launch_row_copy(D.gather_o.dj, D.cs, 0, reinterpret_cast<int64_t>(o_dev[d])); ++D.launches; }
    if (l_dev[d]) { launch_row_copy(D.gather_lse.dj, D.cs, 0, reinterpret_cast<int64_t>(l_dev[d])); ++D.launches; }
    if (opt.timing) CUDA_OK(cudaEventRecord(D.t1, D.cs));
    CUDA_OK(cudaGetLastError());
  }
  if (host && (want_o || want_l)) {
    DevState& D0 = dev_[0];
    DeviceGuard gd(D0.ordinal);
    for (int d = 1; d < R_; ++d) {
      cudaEvent_t e = event(d);
      DeviceGuard g2(dev_[d].ordinal);
      CUDA_OK(cudaEventRecord(e, dev_[d].cs));
      DeviceGuard g3(D0.ordinal);
      CUDA_OK(cudaStreamWaitEvent(D0.cs, e, 0));
    }
    if (want_o) CUDA_OK(cudaMemcpyAsync(o_out[0], o_dev[0], TT * g_.H * 256, cudaMemcpyDeviceToHost, D0.cs));
    if (want_l) CUDA_OK(cudaMemcpyAsync(lse_out[0], l_dev[0], TT * g_.H * 4, cudaMemcpyDeviceToHost, D0.cs));
    CUDA_OK(cudaStreamSynchronize(D0.cs));
  }
  fill_report(rep, false);
  fwd_done_ = true;
}

void Executor::fill_report(dcpx_report* rep, bool bwd) {
  if (opt.trace) trace_collect();
  if (!rep) return;
  std::memset(rep, 0, sizeof(*rep));
  rep->devices = R_;
  rep->stages = static_cast<int32_t>(comm_bytes_.size());
  std::vector<double> comp_t(comm_bytes_.size(), 0), comm_t(comm_bytes_.size(), 0);
  for (size_t t = 0; t < comm_bytes_.size(); ++t) {
    for (const auto& [link, bytes] : comm_bytes_[t]) {
      if (!bwd) {
        rep->total_bytes += bytes;
        rep->per_device_send[link.first] += bytes;
        rep->per_device_recv[link.second] += bytes;
      }
      comm_t[t] = std::max(comm_t[t], bytes ? 5e-6 + static_cast<double>(bytes) / 600e9 : 0.0);  // link_time, schedule.hpp:209-215
    }
    for (int d = 0; d < R_; ++d) {
      rep->total_flops += comp_flops_[t][d];
      comp_t[t] = std::max(comp_t[t], static_cast<double>(comp_flops_[t][d]) / 312e12);  // CostParams, schedule.hpp:173-175
    }
  }
  // pipeline_makespan (schedule.hpp:192-207)
  double start_prev = 0, finish = 0;
  for (size_t t = 0; t < comm_t.size(); ++t) {
    const double start = t == 0 ? 0 : std::max(finish, start_prev + comm_t[t]);
    start_prev = start;
    finish = start + comp_t[t];
  }
  rep->makespan = finish;
  if (bwd) {
    // backward: 5 GEMMs per attended pair vs 2 forward -> 2.5x FLOPs; planned bytes =
    // (Q + dO out, dQ back) per Q fetch and (KV out, dK/dV back) per KV fetch
    rep->total_flops = rep->total_flops / 2 * 5;
    rep->makespan = 0;
    for (int d = 0; d < R_; ++d) {
      rep->per_device_send[d] = bwd_send_[d];
      rep->per_device_recv[d] = bwd_recv_[d];
      rep->total_bytes += bwd_send_[d];
    }
  }
  rep->wire_bytes = rep->total_bytes;
  for (int d = 0; d < R_; ++d) rep->kernel_launches += dev_[d].launches;
  if (opt.kernel_timing) {
    double mx = 0;
    for (auto& D : dev_) {
      DeviceGuard gd(D.ordinal);
      double sum = 0;
      for (size_t k = 0; k < D.next_kev; ++k) {
        CUDA_OK(cudaEventSynchronize(D.kev[k].second));
        float ms = 0;
        CUDA_OK(cudaEventElapsedTime(&ms, D.kev[k].first, D.kev[k].second));
        sum += ms;
      }
      rep->attn_launches += static_cast<int32_t>(D.next_kev);
      rep->attn_ms_sum += sum;
      mx = std::max(mx, sum);
    }
    rep->attn_ms = mx;
  }
  if (opt.timing) {
    double mx = 0;
    for (auto& D : dev_) {
      DeviceGuard gd(D.ordinal);
      CUDA_OK(cudaEventSynchronize(D.t1));
      float ms = 0;
      CUDA_OK(cudaEventElapsedTime(&ms, D.t0, D.t1));
      mx = std::max<double>(mx, ms);
    }
    rep->device_ms = mx;
  }
}

void Executor::backward(const void* const* d_o, void* const* dq, void* const* dk, void* const* dv,
                        dcpx_report* rep, bool host) {
  if (!prepared_) throw Failure(DCPX_ERROR, "dcpx_backward before dcpx_prepare");
  if (!fwd_done_) throw Failure(DCPX_ERROR, "dcpx_backward needs a preceding dcpx_forward");
  const int64_t TT = g_.total_tokens(), H = g_.H, G = g_.G;
  const int T = R_ ? plans_[0].divisions : 0;
  std::vector<const char*> ddo(static_cast<size_t>(R_));
  std::vector<char*> ddq(static_cast<size_t>(R_)), ddk(static_cast<size_t>(R_)), ddv(static_cast<size_t>(R_));
  for (int d = 0; d < R_; ++d) {
    ddo[d] = static_cast<const char*>(d_o[d]);
    ddq[d] = static_cast<char*>(dq ? dq[d] : nullptr);
    ddk[d] = static_cast<char*>(dk ? dk[d] : nullptr);
    ddv[d] = static_cast<char*>(dv ? dv[d] : nullptr);
  }
  const size_t bq = TT * H * 256, bk = TT * G * 256;
  for (auto& D : dev_) {
    D.next_event = 0;
    D.next_kev = 0;
    D.launches = 0;
    DeviceGuard gd(D.ordinal);
    if (opt.timing) CUDA_OK(cudaEventRecord(D.t0, D.cs));
  }
  int slot = -1;
  if (host) {
    // dO up on h2d_ into staging slot k (once the slot's previous downloads are done);
    // dQ/dK/dV come back through the same slot on d2h_ at the end. Asynchronous.
    DevState& D0 = dev_[0];
    DeviceGuard gd(D0.ordinal);
    slot = bwd_st_.next;
    bwd_st_.next ^= 1;
    char*& buf = bwd_st_.buf[slot];
    if (!buf) buf = static_cast<char*>(alloc(0, 2 * bq + 2 * bk));
    for (cudaEvent_t e : bwd_st_.free[slot]) CUDA_OK(cudaStreamWaitEvent(h2d_, e, 0));
    CUDA_OK(cudaMemcpyAsync(buf, d_o[0], bq, cudaMemcpyHostToDevice, h2d_));
    if (!bwd_st_.up[slot]) bwd_st_.up[slot] = staging_event(0);
    cudaEvent_t up = bwd_st_.up[slot];
    CUDA_OK(cudaEventRecord(up, h2d_));
    for (int d = 0; d < R_; ++d) {
      DeviceGuard g2(dev_[d].ordinal);
      CUDA_OK(cudaStreamWaitEvent(dev_[d].cs, up, 0));
    }
    std::fill(ddo.begin(), ddo.end(), buf);
    std::fill(ddq.begin(), ddq.end(), ddq[0] ? buf + bq : nullptr);
    std::fill(ddk.begin(), ddk.end(), ddk[0] ? buf + 2 * bq : nullptr);
    std::fill(ddv.begin(), ddv.end(), ddv[0] ? buf + 2 * bq + bk : nullptr);
  }
  await_peer_pulls();
  const float scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(g_.D)));
  for (int d = 0; d < R_; ++d) {
    DevState& D = dev_[d];
    DeviceGuard gd(D.ordinal);
    const int64_t SR = D.slot_rows;
    CUDA_OK(cudaMemsetAsync(D.dq_acc, 0, std::max<int64_t>(1, D.cap_q) * SR * 512, D.cs));
    CUDA_OK(cudaMemsetAsync(D.dkv_acc, 0, std::max<int64_t>(1, D.cap_kv) * 2 * SR * 512, D.cs));
    launch_row_copy(D.scatter_do.dj, D.cs, reinterpret_cast<int64_t>(ddo[d]), 0);
    launch_delta(D.prep.dj, D.o, D.lse, D.d_o, D.delta, D.lse2, D.cs);
    D.launches += 2;
  }
  // every device's accumulators are zeroed before any peer returns into them: a device's
  // first gradient return waits for its peers' zeroing (not its attention)
  std::vector<cudaEvent_t> zeroed(static_cast<size_t>(R_));
  std::vector<char> zero_waited(static_cast<size_t>(R_), 0);
  for (int d = 0; d < R_; ++d) {
    DeviceGuard gd(dev_[d].ordinal);
    zeroed[d] = event(d);
    CUDA_OK(cudaEventRecord(zeroed[d], dev_[d].cs));
  }
  auto await_zeroed = [&](int d) {
    if (zero_waited[d]) return;
    zero_waited[d] = 1;
    DeviceGuard gd(dev_[d].ordinal);
    for (int e = 0; e < R_; ++e)
      if (e != d) CUDA_OK(cudaStreamWaitEvent(dev_[d].cs, zeroed[e], 0));
  };
  std::map<std::string, cudaEvent_t> send_ev, recv_ev;
  std::vector<cudaEvent_t> ready_ev(static_cast<size_t>(R_));
  for (int d = 0; d < R_; ++d) {  // dO scattered, Delta / LSE prepared on cs
    DeviceGuard gd(dev_[d].ordinal);
    ready_ev[d] = event(d);
    CUDA_OK(cudaEventRecord(ready_ev[d], dev_[d].cs));
  }
  trace_begin();
  DeviceCursor cursor;
  for (const auto& [d, i] : bwd_live_) {  // the output stage has no backward counterpart
    DevState& D = dev_[d];
    Op& op = D.prog[i];
    cursor.to(D.ordinal);
    TraceScope ts(this, d, static_cast<int>(i), op.kind == OpKind::kCommWait ? D.ms : D.cs, 1, op);
    switch (op.kind) {
      case OpKind::kFwdAttn: {
        if (op.bnum_units) {
          BwdParams p{};
          p.units = op.bunits; p.steps = op.bsteps; p.items = op.bitems; p.ranges = D.ranges;
          p.lse2 = D.lse2; p.delta = D.delta; p.dq_acc = D.dq_acc; p.dkv_acc = D.dkv_acc;
          p.num_units = op.bnum_units;
          p.slot_rows = static_cast<int32_t>(D.slot_rows);
          p.scale_log2 = static_cast<float>(1.4426950408889634) * scale;
          p.scale = scale;
          p.debug_flags = opt.bwd_debug;
          std::pair<cudaEvent_t, cudaEvent_t> ke{};
          if (opt.kernel_timing) { ke = kernel_events(d); CUDA_OK(cudaEventRecord(ke.first, D.cs)); }
          launch_attn_bwd(D.tm_q64, D.tm_do, D.tm_kv, D.tm_dq, D.tm_dkv, p, attn_grid(d, op.bgrid), D.cs);
          if (opt.kernel_timing) CUDA_OK(cudaEventRecord(ke.second, D.cs));
          ++D.launches;
        }
        if (op.ret.dj.n_blocks) {
          await_zeroed(d);
          launch_return_accum(op.ret.dj, D.cs);
          ++D.launches;
        }
        break;
      }
      case OpKind::kCommLaunch: {
        if (op.send && op.resident_only) {
          send_ev[op.tag] = ready_ev[d];  // resident inputs: ready since load / preprocess
        } else {
          cudaEvent_t e = event(d);
          CUDA_OK(cudaEventRecord(e, D.cs));
          (op.send ? send_ev : recv_ev)[op.tag] = e;
        }
        break;
      }
      case OpKind::kCommWait: {
        CUDA_OK(cudaStreamWaitEvent(D.ms, send_ev.at(op.tag), 0));
        CUDA_OK(cudaStreamWaitEvent(D.ms, recv_ev.at(op.tag), 0));
        ts.split(kTraceXfer);
        if (opt.sm_transfers) {
          launch_row_copy(op.bjobs.dj, D.ms);
          ++D.launches;
        } else {
          copy_engine(op.bxfer, D.ms);
        }
        cudaEvent_t e = event(d);
        CUDA_OK(cudaEventRecord(e, D.ms));
        CUDA_OK(cudaStreamWaitEvent(D.cs, e, 0));
        break;
      }
      default:
        break;
    }
  }
  mark_pulls_done();
  // all gradient returns land before the owners convert their accumulators
  {
    std::vector<cudaEvent_t> ev(static_cast<size_t>(R_));
    for (int d = 0; d < R_; ++d) {
      DeviceGuard gd(dev_[d].ordinal);
      ev[d] = event(d);
      CUDA_OK(cudaEventRecord(ev[d], dev_[d].cs));
    }
    for (int d = 0; d < R_; ++d)
      for (int e = 0; e < R_; ++e)
        if (e != d) {
          DeviceGuard gd(dev_[d].ordinal);
          CUDA_OK(cudaStreamWaitEvent(dev_[d].cs, ev[e], 0));
        }
  }
  for (int d = 0; d < R_; ++d) {
    DevState& D = dev_[d];
    DeviceGuard gd(D.ordinal);
    if (ddq[d]) { launch_to_bf16(D.gather_dq.dj, D.dq_acc, reinterpret_cast<__nv_bfloat16*>(ddq[d]), D.cs); ++D.launches; }
    if (ddk[d]) { launch_to_bf16(D.gather_dk.dj, D.dkv_acc, reinterpret_cast<__nv_bfloat16*>(ddk[d]), D.cs); ++D.launches; }
    if (ddv[d]) { launch_to_bf16(D.gather_dv.dj, D.dkv_acc, reinterpret_cast<__nv_bfloat16*>(ddv[d]), D.cs); ++D.launches; }
    if (opt.timing) CUDA_OK(cudaEventRecord(D.t1, D.cs));
    CUDA_OK(cudaGetLastError());
  }
  if (host) {
    DevState& D0 = dev_[0];
    DeviceGuard gd(D0.ordinal);
    for (int d = 0; d < R_; ++d) {  // every device's conversions into the slot are done
      cudaEvent_t e = event(d);
      {
        DeviceGuard g2(dev_[d].ordinal);
        CUDA_OK(cudaEventRecord(e, dev_[d].cs));
      }
      CUDA_OK(cudaStreamWaitEvent(d2h_, e, 0));
    }
    if (ddq[0]) CUDA_OK(cudaMemcpyAsync(dq[0], ddq[0], bq, cudaMemcpyDeviceToHost, d2h_));
    if (ddk[0]) CUDA_OK(cudaMemcpyAsync(dk[0], ddk[0], bk, cudaMemcpyDeviceToHost, d2h_));
    if (ddv[0]) CUDA_OK(cudaMemcpyAsync(dv[0], ddv[0], bk, cudaMemcpyDeviceToHost, d2h_));
    auto& fr = bwd_st_.free[slot];
    if (fr.empty()) fr.push_back(staging_event(0));
    CUDA_OK(cudaEventRecord(fr[0], d2h_));
  }
  fill_report(rep, true);
}

void Executor::synchronize() {
  for (auto& D : dev_) {
    DeviceGuard gd(D.ordinal);
    CUDA_OK(cudaStreamSynchronize(D.cs));
    CUDA_OK(cudaStreamSynchronize(D.ms));
  }
  if (R_ > 0) {
    DeviceGuard gd(dev_[0].ordinal);
    if (h2d_) CUDA_OK(cudaStreamSynchronize(h2d_));
    if (d2h_) CUDA_OK(cudaStreamSynchronize(d2h_));
  }
}

void Executor::debug_arena(int d, int kind, void** ptr, int64_t* rows) {
  if (d < 0 || d >= R_) throw Failure(DCPX_ERROR, "bad device");
  const DevState& D = dev_[d];
  *rows = D.slot_rows;
  switch (kind) {
    case 0: *ptr = D.q; break;
    case 1: *ptr = D.kv; break;
    case 2: *ptr = D.o; break;
    case 3: *ptr = D.lse; break;
    default: throw Failure(DCPX_ERROR, "bad arena kind");
  }
}

}  // namespace dcpx

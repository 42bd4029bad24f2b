// executor.h — host side of the B200 DCP executor (C++; the C ABI in capi.cu wraps it).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <array>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/dcpx.h"
#include "host_util.h"
#include "movers.h"
#include "program.h"

#ifndef DCPX_STAGING_SLOTS
#define DCPX_STAGING_SLOTS 2
#endif

namespace dcpx {

// Exception carrying a dcpx_status (mirrors the reference hierarchy, types.hpp:17-45).
struct Instr {
  int op = 0, division = 0, send = 0, peer = 0, dst = 0, count = 0;
  int64_t offset = 0;
  std::string tag;
};

struct PlanCopy {  // owned copy of one dcpx_plan_view
  int device = 0, divisions = 0;
  int cap[3] = {0, 0, 0};
  std::vector<dcpx_block_slot> res_q, res_kv, res_o;
  std::vector<Instr> ins;
  std::vector<dcpx_attention_item> items;
  std::vector<int32_t> srcs;
  std::vector<dcpx_copy_item> copies;
  std::vector<dcpx_block_slot> blocks;
  std::vector<int32_t> rows;
};

struct GraphCopy {
  int H = 0, G = 0, D = 0, bpe = 2;
  std::vector<int64_t> seq_lengths, block_sizes, seq_offsets;
  std::vector<int32_t> ranges;  // [T][4]
  std::vector<dcpx_data_block> data_blocks;
  std::vector<dcpx_comp_block> comp_blocks;
  int64_t total_tokens() const { return seq_offsets.empty() ? 0 : seq_offsets.back(); }
};

// Device-resident job list helper (uploaded once at prepare).
struct JobList {
  DevJobs dj;
  std::vector<void*> owned;
};

enum class OpKind { kFwdAttn, kMerge, kCopy, kCommLaunch, kCommWait, kNop };
constexpr int kTraceXfer = 6;  // trace-only kind: the transfer part of a comm wait

struct Op {
  OpKind kind = OpKind::kNop;
  int division = 0;
  int instr = 0;
  // kFwdAttn
  FwdUnit* units = nullptr;
  FwdStep* steps = nullptr;
  ItemMask* items = nullptr;
  int num_units = 0, grid = 0;
  uint64_t flops = 0;
  // host copies of the forward lists (a persistent launch concatenates them) and the output
  // block each unit writes
  std::vector<FwdUnit> h_units;
  std::vector<FwdStep> h_steps;
  std::vector<ItemMask> h_items;
  std::vector<int> h_unit_oblock;
  // kMerge / kCopy
  JobList jobs;
  int32_t* src_rows = nullptr;
  // backward of an attention instruction (K1b) + gradient returns that follow it
  BwdUnit* bunits = nullptr;
  BwdStep* bsteps = nullptr;
  ItemMask* bitems = nullptr;
  int bnum_units = 0, bgrid = 0;
  JobList ret;   // LOCAL: dQ / dK,dV partials of fetched blocks whose last use is here
  JobList bjobs; // kCommWait: backward payload transfer (Q + dO + LSE + Delta, or K + V)
  std::vector<RowCopyJob> xfer, bxfer;  // the same transfers for the copy engines
  std::vector<MergeJob> mjobs;          // kMerge (host side, batched before upload)
  std::vector<int32_t> msrc;
  // comm
  int send = 0, peer = 0;
  bool resident_only = false;  // a send of resident Q / KV slots only
  // persistent forward, receive side: the transfer overwrites slots once the units of
  // divisions < pf_wait_divs are done (the attention ops before its launch in program order)
  int pf_wait_divs = 0;
  // attention: a fetch (CommWait of a division < T) follows before the next attention op in
  // program order, i.e. runs on the comm stream while this launch does (forward / backward)
  bool fetch_overlap = true, bfetch_overlap = true;
  std::string tag;
  std::vector<dcpx_block_slot> blocks;
  uint64_t bytes = 0;
};

struct DevState {
  int ordinal = 0;
  cudaStream_t cs = nullptr, ms = nullptr;
  int64_t slot_rows = 0;
  int64_t cap_q = 0, cap_kv = 0, cap_o = 0;  // physical slots
  std::vector<int32_t> o_phys;               // plan O slot -> physical slot
  __nv_bfloat16 *q = nullptr, *kv = nullptr, *o = nullptr;
  float* lse = nullptr;
  int32_t* ranges = nullptr;
  CUtensorMap tm_q{}, tm_kv{};
  std::vector<Op> prog;
  JobList scatter_q, scatter_k, scatter_v, gather_o, gather_lse;
  // packed token ranges [begin, end) of the resident Q / KV / O blocks (merged): the rows
  // this device reads from / writes to the caller's packed buffers
  std::vector<std::pair<int64_t, int64_t>> tok_q, tok_kv, tok_o;
  // backward arenas (parallel to Q / KV arenas) and their io jobs
  __nv_bfloat16* d_o = nullptr;
  float *lse2 = nullptr, *delta = nullptr, *dq_acc = nullptr, *dkv_acc = nullptr;
  CUtensorMap tm_do{}, tm_dq{}, tm_q64{};  // backward: 64-row boxes over dO, dQ acc, Q
  CUtensorMap tm_dkv{};                    // backward: dK / dV accumulator, 128-row boxes
  JobList prep, gather_dq, gather_dk, gather_dv;  // prep: Delta / LSE2 + dO scatter
  std::vector<int32_t> final_o_slot;  // per resident_o entry: physical slot holding the result
  std::vector<cudaEvent_t> events;
  size_t next_event = 0;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  int launches = 0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> kev;  // per attention launch (kernel_timing)
  std::vector<int> kev_pass;                             // 0 forward / 1 backward, per used pair
  size_t next_kev = 0;
  // the fp32 gradient accumulators are re-zeroed on `as` after each backward (bwd_end), off the
  // compute stream; the next backward's compute waits for aux_done
  cudaStream_t as = nullptr;
  cudaEvent_t aux_done = nullptr, bwd_end = nullptr;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> tev;  // per traced op (trace), a separate pool
  size_t next_tev = 0;
  // stream contract with the caller: every call starts after the work already enqueued on
  // `caller` (its inputs) and `caller` waits for the call's device work (its outputs)
  cudaStream_t caller = cudaStreamLegacy;
  cudaEvent_t ev_join = nullptr, ev_done = nullptr;
  // persistent cross-division forward: one launch for all divisions' units,
  // gated device-side (FwdParams::rdy / done / unit_done); pf_first = the op that launches
  // it (the device's first attention), the other attention ops launch nothing
  bool pfwd = false;
  int pf_first = -1;
  FwdUnit* pf_units = nullptr;
  FwdStep* pf_steps = nullptr;
  ItemMask* pf_items = nullptr;
  int pf_num_units = 0, pf_grid = 0;
  uint32_t* pctr = nullptr;          // rdy[T + 1] then done[T + 1]
  uint32_t* prdy_target = nullptr;   // [T + 1] transfers per division
  uint32_t* pdone_target = nullptr;  // [T + 1] (unit, tile) epilogues per division
  uint32_t* punit_done = nullptr;    // [2 * pf_num_units] epoch stamps
  // dynamic unit scheduler of the attention kernels: a device counter that every launch
  // advances by num_units + grid, and its host-side running value (sched_produce)
  uint32_t* sched_ctr = nullptr;
  uint32_t sched_base = 0;
  // backward units of the last prepare (diagnostics in the report)
  int32_t bwd_units = 0, bwd_windowed = 0;
};

struct Options {
  bool fuse_reductions = true;
  bool remap_copies = true;
  bool check_rows = false;
  bool timing = false;  // per-call device_ms in the report (blocks the host at the end of each call)
  // CUDA events around every attention launch: 1 = read back at the end of each call (in the
  // report; blocks the host), 2 = accumulated without blocking, read by kernel_times()
  int kernel_timing = 0;
  bool trace = false;
  bool sm_transfers = true;   // LOCAL transfers by copy kernel (false: DMA copy engines)
  int sm_reserve = -1;        // SMs left free of attention CTAs for transfer kernels (-1: auto)
  // backward units: (kv sub-tile, window of bwd_window 64-row q tiles of one item), ordered
  // q-window-major (2) so concurrent CTAs share Q / dO / dQ rows in L2; 0 = longest first,
  // 1 = plan order. Windows apply to instructions whose whole-item units average at least
  // bwd_window_min_steps steps; shorter units stay whole, longest first. Measured on B200
  // (bench): cfg2 798 -> 813, cfg4 shared-question 761 -> 814 TFLOP/s with windows;
  // cfg4 causal-blockwise (49 steps per unit) 339 with windows vs 366 without.
  int bwd_order = 2;
  int bwd_window = 16;
  int bwd_window_min_steps = 128;
  // windows span every item of one q block (the heads of the GQA group) instead of one item
  int bwd_merge_heads = 1;
  // multi-device plans: run each device's forward divisions as one persistent launch
  int persistent = 0;
  // re-zero the fp32 gradient accumulators on the aux stream after each backward (1) or on the
  // compute stream at the start of the next one (0)
  int aux_zero = 1;
};

class Executor;

// Records device-time spans of one executed op when Options::trace is set.
class TraceScope {
 public:
  TraceScope(Executor* ex, int d, int instr, cudaStream_t s, int pass, const Op& op);
  ~TraceScope();
  // Ends the current span here and opens a second one of trace kind `kind` (e.g. a
  // comm wait's transfer once its events have resolved).
  void split(int kind);

 private:
  Executor* ex_;
  int d_;
  cudaStream_t s_ = nullptr;
  bool active_ = false;
};

class Executor {
 public:
  // transport: DCPX_TRANSPORT_LOCAL (copy kernels reading peer memory) or
  // DCPX_TRANSPORT_NCCL (NCCL send/recv pairs, one GPU per plan device). rank >= 0: the
  // per-rank mode (one process per GPU): all ordinals are this process's GPU, only plan
  // device `rank` executes, peers' arenas are mapped over CUDA IPC (export / connect).
  Executor(int ndev, const int* ordinals, int transport = DCPX_TRANSPORT_LOCAL, int rank = -1);
  // host-only instance (ordinals == nullptr): prepare() ingests, verifies and replays the plans
  // (verify_plans + the lockstep deadlock / tag checks) without touching a GPU
  bool host_only() const { return host_only_; }
  // per-rank mode: IPC handles of this rank's arenas and flags; map every peer's
  int64_t export_handles(void* buf, int64_t cap) const;
  void connect(const void* blobs, int64_t blob_size, int world);
  bool local(int d) const { return rank_ < 0 || d == rank_; }
  ~Executor();
  void prepare(int nplans, const dcpx_plan_view* plans, const dcpx_graph_view* g,
               const dcpx_mask_view* m);
  int devices() const { return R_; }  // plan devices (0 before prepare)
  // Packed I/O buffers, one pointer per plan device: device d reads / writes only the rows
  // of the blocks it owns. The single-buffer API passes the same buffer for every device;
  // the per-device (_dev) API passes buffers in each device's own memory. host: all
  // entries are one host buffer, staged through the first device.
  void load_inputs(const void* const* q, const void* const* k, const void* const* v, bool host);
  void forward(void* const* o_out, float* const* lse_out, dcpx_report* rep, bool host);
  void backward(const void* const* d_o, void* const* dq, void* const* dk, void* const* dv, dcpx_report* rep,
                bool host);
  void synchronize();
  // kernel_timing 2: GPU time of the attention launches since the last read, per pass:
  // ms[0..1] summed over local devices (fwd, bwd), ms[2..3] max over devices; resets
  void kernel_times(double* ms, int32_t* launches);
  // the caller's stream on each plan device (nullptr entry: the legacy default stream)
  void set_streams(int n, const cudaStream_t* s);
  void debug_arena(int dev, int kind, void** ptr, int64_t* rows);
  int trace_rows(double* out, int max_rows) const;
  std::string watchdog_info() const;  // barrier waits that timed out (kernel watchdog)  // rows of 7: dev, instr, kind, division, pass, start_ms, end_ms
  Options opt;
  std::string last_error;

 private:
  friend class TraceScope;
  struct TracePending {
    int d, instr, kind, division, pass;
    cudaEvent_t start, end;
  };
  std::vector<TracePending> trace_pending_;
  std::vector<std::array<double, 7>> trace_;
  void trace_begin();
  void copy_engine(const std::vector<RowCopyJob>& jobs, cudaStream_t s);
  int attn_grid(int d, int grid, bool overlap = true) const;
  void mark_fetch_overlap(int d);
  void trace_collect();
  void compile_device(int d);
  void compile_attention(int d, int ins_index, std::vector<bool>& fused_red);
  void build_persistent_fwd(int d);
  void zero_accumulators(int d, cudaStream_t s);  // the fp32 dQ / dK,dV accumulators
  bool acc_dirty_ = false;  // the last backward did not re-zero them (aux_zero = 0)
  void build_io_jobs(int d);
  void build_bwd_jobs();
  void fill_report(dcpx_report* rep, bool bwd);
  void simulate_order();
  cudaEvent_t event(int d);
  std::pair<cudaEvent_t, cudaEvent_t> kernel_events(int d, int pass);
  std::pair<cudaEvent_t, cudaEvent_t> trace_events(int d);
  void join_caller();     // cs of every local device waits for the caller's stream
  void release_caller();  // the caller's stream waits for cs of every local device
  void free_all();

  int R_ = 0;
  bool host_only_ = false;
  std::vector<int> ordinals_;
  std::vector<PlanCopy> plans_;
  GraphCopy g_;
  std::vector<DevState> dev_;
  // global issue order from the lockstep simulation: (device, op index)
  std::vector<std::pair<int, int>> order_;
  int transport_ = DCPX_TRANSPORT_LOCAL;
  // per-rank mode: device-side epoch flags instead of cross-device events. Word layout of
  // each rank's flag buffer: kFlagZeroed, kFlagReturns, kFlagPulls, then one word per
  // message tag (send ready).
  enum { kFlagZeroed = 0, kFlagReturns = 1, kFlagPulls = 2, kFlagSend = 3 };
  int rank_ = -1;
  bool connected_ = false;
  uint32_t* flags_ = nullptr;
  std::vector<uint32_t*> peer_flags_;  // [R_], this rank's own included
  std::map<std::string, int> tag_id_;
  uint32_t epoch_ = 0, pulls_epoch_ = 0;
  std::vector<void*> ipc_mapped_;
  void flag_set(int word, cudaStream_t s);
  void flag_wait_peers(int word, uint32_t epoch, cudaStream_t s, int only_peer = -1);
  void build_transfer_jobs();
  // host I/O: the packed token ranges the local device(s) touch (everything in the
  // single-process context; this rank's rows in the per-rank mode)
  std::vector<std::pair<int64_t, int64_t>> host_ranges(int which) const;  // 0 Q, 1 KV, 2 O
  static void copy_ranges(void* dst, const void* src, const std::vector<std::pair<int64_t, int64_t>>& r,
                          int64_t row_bytes, cudaMemcpyKind kind, cudaStream_t s);
  void publish_resident_sends(const std::vector<std::pair<int, int>>& live);
  std::vector<ncclComm_t> comms_;  // NCCL transport: one communicator per plan device
  void nccl_transfer(int src, int dst, const std::vector<RowCopyJob>& jobs, cudaEvent_t data_ready,
                     cudaEvent_t slot_free);
  std::vector<std::pair<int, int>> fwd_live_, bwd_live_;  // order_ without ops that launch nothing
  std::vector<void*> allocs_;  // (ordinal, ptr) freed in destructor
  std::vector<int> alloc_dev_;
  uint32_t* diag_ = nullptr;   // host-mapped watchdog report buffer (see sm100.cuh)
  // Host I/O goes through device-0 staging. load_inputs_host / backward_host are
  // asynchronous: staging slots rotate, uploads run on h2d_ and downloads on d2h_
  // (PCIe is full duplex), so step i+1's uploads and step i's downloads overlap step i's
  // compute; free[k] holds the events after which slot k may be overwritten.
  static constexpr int kStagingSlots = DCPX_STAGING_SLOTS;
  struct Staging {
    char* buf[kStagingSlots] = {};
    std::vector<cudaEvent_t> free[kStagingSlots];  // per plan device (backward: entry 0 only)
    cudaEvent_t up[kStagingSlots] = {};             // upload into slot k finished (h2d_)
    int next = 0;
    int take() {  // the next slot, round robin
      const int k = next;
      next = (next + 1) % kStagingSlots;
      return k;
    }
  };
  Staging in_st_, bwd_st_, fwd_st_;  // fwd_st_: forward_host outputs (O + LSE), downloaded on d2h_
  cudaStream_t h2d_ = nullptr, d2h_ = nullptr;  // on device 0
  cudaEvent_t staging_event(int d);              // persistent (not from the per-call pool)
  // pulls_done_[d]: recorded on device d's comm stream at the end of each pass (its last
  // peer reads); every device waits for its peers' before writing slots in the next call,
  // so a lagging peer never reads a slot that the next call is already rewriting
  std::vector<cudaEvent_t> pulls_done_;
  void await_peer_pulls();
  void mark_pulls_done();
  std::vector<cudaEvent_t> staging_events_;
  std::vector<int> staging_event_dev_;
  bool fwd_done_ = false;
  std::vector<uint64_t> bwd_send_, bwd_recv_;  // planned backward bytes per device
  // bytes the transfers actually move (fp32 sidecars and fp32 gradient returns included)
  std::vector<uint64_t> wire_fwd_send_, wire_fwd_recv_, wire_bwd_send_, wire_bwd_recv_;
  bool prepared_ = false;
  // report
  std::vector<std::map<std::pair<int, int>, uint64_t>> comm_bytes_;
  std::vector<std::vector<uint64_t>> comp_flops_;
  void* alloc(int d, size_t bytes);
  template <class T>
  T* upload(int d, const std::vector<T>& v);
  JobList make_jobs(int d, const std::vector<RowCopyJob>& jobs);
  template <class J>
  JobList make_row_jobs(int d, const std::vector<J>& jobs, const std::vector<int>& rows, int rows_per_block);
};


// ---- member templates (used by compile.cu and executor.cu)
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

}  // namespace dcpx

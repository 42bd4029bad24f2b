// run.cu — execution side of the B200 DCP executor (see executor.cu): input scatter,
// forward / backward issue in the recorded lockstep order (attention launches, merges,
// copies, event-ordered LOCAL transfers on the comm streams), output gathers, host I/O
// staging and the SimReport-shaped report.
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <numeric>
#include <string>

#include "executor.h"

namespace dcpx {

// ------------------------------------------------------------------------ execution
// Per-rank mode: sends of resident blocks are ready as soon as the inputs are, so their
// flags go up at the start of the pass (the LOCAL transport gates them on ready_ev).
void Executor::publish_resident_sends(const std::vector<std::pair<int, int>>& live) {
  if (rank_ < 0) return;
  DevState& D = dev_[rank_];
  for (const auto& [d, i] : live) {
    if (d != rank_) continue;
    const Op& op = D.prog[i];
    if (op.kind == OpKind::kCommLaunch && op.send && op.resident_only) flag_set(kFlagSend + tag_id_.at(op.tag), D.cs);
  }
}

std::vector<std::pair<int64_t, int64_t>> Executor::host_ranges(int which) const {
  const int64_t TT = g_.total_tokens();
  if (rank_ < 0) return {{0, TT}};  // the devices of one process together touch every row
  const DevState& D = dev_[rank_];
  return which == 0 ? D.tok_q : which == 1 ? D.tok_kv : D.tok_o;
}

void Executor::copy_ranges(void* dst, const void* src, const std::vector<std::pair<int64_t, int64_t>>& r,
                           int64_t row_bytes, cudaMemcpyKind kind, cudaStream_t s) {
  for (const auto& [b, e] : r)
    if (e > b)
      CUDA_OK(cudaMemcpyAsync(static_cast<char*>(dst) + b * row_bytes, static_cast<const char*>(src) + b * row_bytes,
                              (e - b) * row_bytes, kind, s));
}

void Executor::load_inputs(const void* const* q, const void* const* k, const void* const* v, bool host) {
  if (host_only_) throw Failure(DCPX_ERROR, "host-only context: nothing executes");
  if (!prepared_) throw Failure(DCPX_ERROR, "dcpx_load_inputs before dcpx_prepare");
  if (rank_ >= 0 && !connected_) throw Failure(DCPX_ERROR, "dcpx_load_inputs: per-rank context not connected (dcpx_rank_connect)");
  const int64_t TT = g_.total_tokens();
  std::vector<const void*> sq(q, q + R_), sk(k, k + R_), sv(v, v + R_);
  int slot = -1;
  if (host) {
    // upload into staging slot k on the h2d stream once the slot's previous scatters are
    // done; peers read it over NVLink. The call returns without waiting for the copy.
    DevState& D0 = dev_[0];
    DeviceGuard gd(D0.ordinal);
    const size_t bq = TT * g_.H * 256, bk = TT * g_.G * 256;
    slot = in_st_.take();
    char*& buf = in_st_.buf[slot];
    if (!buf) buf = static_cast<char*>(alloc(0, bq + 2 * bk));
    for (cudaEvent_t e : in_st_.free[slot]) CUDA_OK(cudaStreamWaitEvent(h2d_, e, 0));
    // only the token rows this process's devices read (all of them in one process)
    const auto rq = host_ranges(0), rkv = host_ranges(1);
    copy_ranges(buf, q[0], rq, g_.H * 256, cudaMemcpyHostToDevice, h2d_);
    copy_ranges(buf + bq, k[0], rkv, g_.G * 256, cudaMemcpyHostToDevice, h2d_);
    copy_ranges(buf + bq + bk, v[0], rkv, g_.G * 256, cudaMemcpyHostToDevice, h2d_);
    if (!in_st_.up[slot]) in_st_.up[slot] = staging_event(0);
    cudaEvent_t up = in_st_.up[slot];
    CUDA_OK(cudaEventRecord(up, h2d_));
    for (int d = 0; d < R_; ++d) {
      if (!local(d)) continue;
      DeviceGuard g2(dev_[d].ordinal);
      CUDA_OK(cudaStreamWaitEvent(dev_[d].cs, up, 0));
    }
    std::fill(sq.begin(), sq.end(), buf);
    std::fill(sk.begin(), sk.end(), buf + bq);
    std::fill(sv.begin(), sv.end(), buf + bq + bk);
  }
  join_caller();       // device inputs are produced on the caller's stream
  await_peer_pulls();  // resident slots may still be read by a peer's previous-call pull
  for (int d = 0; d < R_; ++d) {
    if (!local(d)) continue;
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
      if (!local(d)) continue;
      DeviceGuard gd(dev_[d].ordinal);
      CUDA_OK(cudaEventRecord(fr[d], dev_[d].cs));
    }
  }
  release_caller();  // the caller may overwrite its input buffers after this point
}

void Executor::forward(void* const* o_out, float* const* lse_out, dcpx_report* rep, bool host) {
  if (host_only_) throw Failure(DCPX_ERROR, "host-only context: nothing executes");
  if (!prepared_) throw Failure(DCPX_ERROR, "dcpx_forward before dcpx_prepare");
  if (rank_ >= 0 && !connected_) throw Failure(DCPX_ERROR, "dcpx_forward: per-rank context not connected (dcpx_rank_connect)");
  const int64_t TT = g_.total_tokens();
  join_caller();  // the output buffers may still be in use on the caller's stream
  for (int d = 0; d < R_; ++d) {
    DevState& D = dev_[d];
    D.next_event = 0;
    if (opt.kernel_timing != 2) {  // (deferred timing accumulates until kernel_times())
      D.next_kev = 0;
      D.kev_pass.clear();
    }
    D.next_tev = 0;
    D.launches = 0;
    if (!local(d)) continue;
    DeviceGuard gd(D.ordinal);
    if (opt.timing || opt.trace) CUDA_OK(cudaEventRecord(D.t0, D.cs));
  }
  await_peer_pulls();
  ++epoch_;
  const int T = R_ ? plans_[0].divisions : 0;
  std::map<std::string, cudaEvent_t> send_ev, recv_ev;
  std::vector<cudaEvent_t> ready_ev(static_cast<size_t>(R_));
  for (int d = 0; d < R_; ++d) {  // resident Q / KV were scattered on cs before this call
    if (!local(d)) continue;
    DeviceGuard gd(dev_[d].ordinal);
    if (dev_[d].pfwd)  // persistent launch: this call's dependency counters start at zero
      CUDA_OK(cudaMemsetAsync(dev_[d].pctr, 0, sizeof(uint32_t) * 2 * (static_cast<size_t>(T) + 1), dev_[d].cs));
    ready_ev[d] = event(d);
    CUDA_OK(cudaEventRecord(ready_ev[d], dev_[d].cs));
  }
  publish_resident_sends(fwd_live_);
  trace_begin();
  DeviceCursor cursor;
  for (const auto& [d, i] : fwd_live_) {
    if (!local(d)) continue;
    DevState& D = dev_[d];
    Op& op = D.prog[i];
    cursor.to(D.ordinal);
    TraceScope ts(this, d, static_cast<int>(i), op.kind == OpKind::kCommWait ? D.ms : D.cs, 0, op);
    switch (op.kind) {
      case OpKind::kFwdAttn: {
        if (!op.num_units) break;
        const bool pers = D.pfwd;
        if (pers && static_cast<int>(i) != D.pf_first) break;  // part of the persistent launch
        FwdParams p{};
        p.units = pers ? D.pf_units : op.units;
        p.steps = pers ? D.pf_steps : op.steps;
        p.items = pers ? D.pf_items : op.items;
        p.ranges = D.ranges;
        p.o_arena = D.o; p.lse_arena = D.lse;
        p.num_units = pers ? D.pf_num_units : op.num_units;
        p.slot_rows = static_cast<int32_t>(D.slot_rows);
        p.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(g_.D)));
        if (pers) {
          p.rdy = D.pctr;
          p.rdy_target = D.prdy_target;
          p.done = D.pctr + T + 1;
          p.unit_done = D.punit_done;
          p.epoch = epoch_;
        }
        std::pair<cudaEvent_t, cudaEvent_t> ke{};
        const int grid = pers ? attn_grid(d, D.pf_grid) : attn_grid(d, op.grid, op.fetch_overlap);
        p.sched = D.sched_ctr;
        p.sched_base = D.sched_base;
        D.sched_base += static_cast<uint32_t>(p.num_units + grid);
        if (opt.kernel_timing) { ke = kernel_events(d, 0); CUDA_OK(cudaEventRecord(ke.first, D.cs)); }
        launch_attn_fwd(D.tm_q, D.tm_kv, p, grid, D.cs);
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
        } else if (!op.send && D.pfwd && op.division < T) {
          // persistent launch: the slots are free once the units of the divisions before this
          // launch point are done, which the transfer waits for on the device (kCommWait)
          recv_ev[op.tag] = ready_ev[d];
        } else {
          cudaEvent_t e = event(d);
          CUDA_OK(cudaEventRecord(e, D.cs));
          (op.send ? send_ev : recv_ev)[op.tag] = e;
          if (rank_ >= 0 && op.send) flag_set(kFlagSend + tag_id_.at(op.tag), D.cs);
        }
        break;
      }
      case OpKind::kCommWait: {
        const bool pers_xfer = D.pfwd && op.division < T;
        if (transport_ == DCPX_TRANSPORT_NCCL) {
          nccl_transfer(op.peer, d, op.xfer, send_ev.at(op.tag), recv_ev.at(op.tag));
          cursor.to(D.ordinal);
        } else {
          if (rank_ >= 0)  // the sender is another process: its send flag for this epoch
            flag_wait_peers(kFlagSend + tag_id_.at(op.tag), epoch_, D.ms, op.peer);
          else
            CUDA_OK(cudaStreamWaitEvent(D.ms, send_ev.at(op.tag), 0));
          CUDA_OK(cudaStreamWaitEvent(D.ms, recv_ev.at(op.tag), 0));
          if (pers_xfer)  // the units that read the slots' previous blocks are done
            launch_counter_wait(D.pctr + T + 1, D.pdone_target, op.pf_wait_divs, D.ms);
          ts.split(kTraceXfer);
          if (opt.sm_transfers) {
            launch_row_copy(op.jobs.dj, D.ms);
            ++D.launches;
          } else {
            copy_engine(op.xfer, D.ms);
          }
          if (pers_xfer) launch_counter_add(D.pctr, D.ms);  // one more fetch landed (cumulative)
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
  int slot = -1;
  if (host && (want_o || want_l)) {
    // asynchronous like the other host calls: gather into device-0 staging slot k (once
    // the slot's previous download is done), download on d2h_; host buffers are valid after
    // dcpx_synchronize, so the download overlaps the next call's work
    slot = fwd_st_.take();
    char*& buf = fwd_st_.buf[slot];
    if (!buf) buf = static_cast<char*>(alloc(0, TT * g_.H * 256 + TT * g_.H * 4));
    for (int d = 0; d < R_; ++d) {
      if (!local(d)) continue;
      DeviceGuard gd(dev_[d].ordinal);
      for (cudaEvent_t e : fwd_st_.free[slot]) CUDA_OK(cudaStreamWaitEvent(dev_[d].cs, e, 0));
    }
    std::fill(o_dev.begin(), o_dev.end(), want_o ? buf : nullptr);
    std::fill(l_dev.begin(), l_dev.end(), want_l ? buf + TT * g_.H * 256 : nullptr);
  }
  for (int d = 0; d < R_; ++d) {
    if (!local(d)) continue;
    DevState& D = dev_[d];
    DeviceGuard gd(D.ordinal);
    if (o_dev[d]) { launch_row_copy(D.gather_o.dj, D.cs, 0, reinterpret_cast<int64_t>(o_dev[d])); ++D.launches; }
    if (l_dev[d]) { launch_row_copy(D.gather_lse.dj, D.cs, 0, reinterpret_cast<int64_t>(l_dev[d])); ++D.launches; }
    if (opt.timing) CUDA_OK(cudaEventRecord(D.t1, D.cs));
    CUDA_OK(cudaGetLastError());
  }
  if (slot >= 0) {
    DevState& D0 = dev_[0];
    for (int d = 0; d < R_; ++d) {  // every device's gathers into the slot are done
      if (!local(d)) continue;
      cudaEvent_t e = event(d);
      DeviceGuard g2(dev_[d].ordinal);
      CUDA_OK(cudaEventRecord(e, dev_[d].cs));
      CUDA_OK(cudaStreamWaitEvent(d2h_, e, 0));
    }
    DeviceGuard gd(D0.ordinal);
    const auto ro = host_ranges(2);
    if (want_o) copy_ranges(o_out[0], o_dev[0], ro, g_.H * 256, cudaMemcpyDeviceToHost, d2h_);
    if (want_l)  // LSE is head-major [H][T]: one strided copy per token range
      for (const auto& [b, e] : ro)
        if (e > b)
          CUDA_OK(cudaMemcpy2DAsync(static_cast<char*>(static_cast<void*>(lse_out[0])) + b * 4, TT * 4, l_dev[0] + b * 4,
                                    TT * 4, (e - b) * 4, g_.H, cudaMemcpyDeviceToHost, d2h_));
    auto& fr = fwd_st_.free[slot];
    if (fr.empty()) fr.push_back(staging_event(0));
    CUDA_OK(cudaEventRecord(fr[0], d2h_));
  }
  release_caller();  // o_out / lse_out are ready in the caller's stream order
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
  for (int d = 0; d < R_; ++d) {
    rep->wire_per_device_send[d] = bwd ? wire_bwd_send_[d] : wire_fwd_send_[d];
    rep->wire_per_device_recv[d] = bwd ? wire_bwd_recv_[d] : wire_fwd_recv_[d];
    rep->wire_bytes += rep->wire_per_device_send[d];
    rep->kernel_launches += dev_[d].launches;
    if (!local(d)) continue;
    for (const Op& op : dev_[d].prog)
      if (op.kind == OpKind::kFwdAttn) rep->units += bwd ? op.bnum_units : op.num_units;
    if (bwd) rep->windowed += dev_[d].bwd_windowed;
  }
  if (opt.kernel_timing == 1) {
    double mx = 0;
    for (int d = 0; d < R_; ++d) {
      if (!local(d)) continue;
      DevState& D = dev_[d];
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
      D.next_kev = 0;  // read: a later switch to deferred timing starts from an empty pool
      D.kev_pass.clear();
    }
    rep->attn_ms = mx;
  }
  if (opt.timing) {
    double mx = 0;
    for (int d = 0; d < R_; ++d) {
      if (!local(d)) continue;
      DevState& D = dev_[d];
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
  if (host_only_) throw Failure(DCPX_ERROR, "host-only context: nothing executes");
  if (!prepared_) throw Failure(DCPX_ERROR, "dcpx_backward before dcpx_prepare");
  if (rank_ >= 0 && !connected_) throw Failure(DCPX_ERROR, "dcpx_backward: per-rank context not connected (dcpx_rank_connect)");
  if (!fwd_done_) throw Failure(DCPX_ERROR, "dcpx_backward needs a preceding dcpx_forward");
  const int64_t TT = g_.total_tokens(), H = g_.H, G = g_.G;
  const int T = R_ ? plans_[0].divisions : 0;
  std::vector<const char*> ddo(static_cast<size_t>(R_));
  std::vector<char*> ddq(static_cast<size_t>(R_)), ddk(static_cast<size_t>(R_)), ddv(static_cast<size_t>(R_));
  for (int d = 0; d < R_; ++d) {
    ddo[d] = static_cast<const char*>(d_o[d]);
    if (!host && local(d) && (reinterpret_cast<uintptr_t>(ddo[d]) & 15))  // (16-byte row loads)
      throw Failure(DCPX_ERROR, "dcpx_backward: dO must be 16-byte aligned");
    ddq[d] = static_cast<char*>(dq ? dq[d] : nullptr);
    ddk[d] = static_cast<char*>(dk ? dk[d] : nullptr);
    ddv[d] = static_cast<char*>(dv ? dv[d] : nullptr);
  }
  const size_t bq = TT * H * 256, bk = TT * G * 256;
  join_caller();  // d_o is produced on the caller's stream
  for (int d = 0; d < R_; ++d) {
    DevState& D = dev_[d];
    D.next_event = 0;
    if (opt.kernel_timing != 2) {  // (deferred timing accumulates until kernel_times())
      D.next_kev = 0;
      D.kev_pass.clear();
    }
    D.next_tev = 0;
    D.launches = 0;
    if (!local(d)) continue;
    DeviceGuard gd(D.ordinal);
    if (opt.timing || opt.trace) CUDA_OK(cudaEventRecord(D.t0, D.cs));
  }
  int slot = -1;
  if (host) {
    // dO up on h2d_ into staging slot k (once the slot's previous downloads are done);
    // dQ/dK/dV come back through the same slot on d2h_ at the end. Asynchronous.
    DevState& D0 = dev_[0];
    DeviceGuard gd(D0.ordinal);
    slot = bwd_st_.take();
    char*& buf = bwd_st_.buf[slot];
    if (!buf) buf = static_cast<char*>(alloc(0, 2 * bq + 2 * bk));
    for (cudaEvent_t e : bwd_st_.free[slot]) CUDA_OK(cudaStreamWaitEvent(h2d_, e, 0));
    copy_ranges(buf, d_o[0], host_ranges(0), g_.H * 256, cudaMemcpyHostToDevice, h2d_);
    if (!bwd_st_.up[slot]) bwd_st_.up[slot] = staging_event(0);
    cudaEvent_t up = bwd_st_.up[slot];
    CUDA_OK(cudaEventRecord(up, h2d_));
    for (int d = 0; d < R_; ++d) {
      if (!local(d)) continue;
      DeviceGuard g2(dev_[d].ordinal);
      CUDA_OK(cudaStreamWaitEvent(dev_[d].cs, up, 0));
    }
    std::fill(ddo.begin(), ddo.end(), buf);
    std::fill(ddq.begin(), ddq.end(), ddq[0] ? buf + bq : nullptr);
    std::fill(ddk.begin(), ddk.end(), ddk[0] ? buf + 2 * bq : nullptr);
    std::fill(ddv.begin(), ddv.end(), ddv[0] ? buf + 2 * bq + bk : nullptr);
  }
  await_peer_pulls();
  ++epoch_;
  const float scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(g_.D)));
  for (int d = 0; d < R_; ++d) {
    if (!local(d)) continue;
    DevState& D = dev_[d];
    DeviceGuard gd(D.ordinal);
    // the fp32 accumulators were zeroed on the aux stream right after the previous backward
    // (overlapping the next forward; zero at prepare for the first call)
    CUDA_OK(cudaStreamWaitEvent(D.cs, D.aux_done, 0));
    if (acc_dirty_) zero_accumulators(d, D.cs);  // (the previous backward left them)
    launch_delta(D.prep.dj, D.o, D.lse, reinterpret_cast<const __nv_bfloat16*>(ddo[d]), g_.H * 128, D.d_o, D.delta,
                 D.lse2, D.cs);
    ++D.launches;
  }
  // every device's accumulators are zeroed before any peer returns into them: a device's
  // first gradient return waits for its peers' zeroing (not its attention)
  std::vector<cudaEvent_t> zeroed(static_cast<size_t>(R_));
  std::vector<char> zero_waited(static_cast<size_t>(R_), 0);
  for (int d = 0; d < R_; ++d) {
    if (!local(d)) continue;
    DeviceGuard gd(dev_[d].ordinal);
    zeroed[d] = event(d);
    CUDA_OK(cudaEventRecord(zeroed[d], dev_[d].cs));
    if (rank_ >= 0) flag_set(kFlagZeroed, dev_[d].cs);
  }
  auto await_zeroed = [&](int d) {
    if (zero_waited[d]) return;
    zero_waited[d] = 1;
    DeviceGuard gd(dev_[d].ordinal);
    if (rank_ >= 0) {
      flag_wait_peers(kFlagZeroed, epoch_, dev_[d].cs);
      return;
    }
    for (int e = 0; e < R_; ++e)
      if (e != d) CUDA_OK(cudaStreamWaitEvent(dev_[d].cs, zeroed[e], 0));
  };
  std::map<std::string, cudaEvent_t> send_ev, recv_ev;
  std::vector<cudaEvent_t> ready_ev(static_cast<size_t>(R_));
  for (int d = 0; d < R_; ++d) {  // dO scattered, Delta / LSE prepared on cs
    if (!local(d)) continue;
    DeviceGuard gd(dev_[d].ordinal);
    ready_ev[d] = event(d);
    CUDA_OK(cudaEventRecord(ready_ev[d], dev_[d].cs));
  }
  publish_resident_sends(bwd_live_);
  trace_begin();
  DeviceCursor cursor;
  for (const auto& [d, i] : bwd_live_) {  // the output stage has no backward counterpart
    if (!local(d)) continue;
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
          std::pair<cudaEvent_t, cudaEvent_t> ke{};
          const int grid = attn_grid(d, op.bgrid, op.bfetch_overlap);
          p.sched = D.sched_ctr;
          p.sched_base = D.sched_base;
          D.sched_base += static_cast<uint32_t>(op.bnum_units + grid);
          if (opt.kernel_timing) { ke = kernel_events(d, 1); CUDA_OK(cudaEventRecord(ke.first, D.cs)); }
          launch_attn_bwd(D.tm_q64, D.tm_do, D.tm_kv, D.tm_dq, D.tm_dkv, p, grid, D.cs);
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
          if (rank_ >= 0 && op.send) flag_set(kFlagSend + tag_id_.at(op.tag), D.cs);
        }
        break;
      }
      case OpKind::kCommWait: {
        if (transport_ == DCPX_TRANSPORT_NCCL) {
          nccl_transfer(op.peer, d, op.bxfer, send_ev.at(op.tag), recv_ev.at(op.tag));
          cursor.to(D.ordinal);
        } else {
          if (rank_ >= 0)  // the sender is another process: its send flag for this epoch
            flag_wait_peers(kFlagSend + tag_id_.at(op.tag), epoch_, D.ms, op.peer);
          else
            CUDA_OK(cudaStreamWaitEvent(D.ms, send_ev.at(op.tag), 0));
          CUDA_OK(cudaStreamWaitEvent(D.ms, recv_ev.at(op.tag), 0));
          ts.split(kTraceXfer);
          if (opt.sm_transfers) {
            launch_row_copy(op.bjobs.dj, D.ms);
            ++D.launches;
          } else {
            copy_engine(op.bxfer, D.ms);
          }
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
  if (rank_ >= 0) {
    DevState& D = dev_[rank_];
    DeviceGuard gd(D.ordinal);
    flag_set(kFlagReturns, D.cs);
    flag_wait_peers(kFlagReturns, epoch_, D.cs);
  } else {
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
    if (!local(d)) continue;
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
      if (!local(d)) continue;
      cudaEvent_t e = event(d);
      {
        DeviceGuard g2(dev_[d].ordinal);
        CUDA_OK(cudaEventRecord(e, dev_[d].cs));
      }
      CUDA_OK(cudaStreamWaitEvent(d2h_, e, 0));
    }
    const auto rq = host_ranges(0), rkv = host_ranges(1);
    if (ddq[0]) copy_ranges(dq[0], ddq[0], rq, H * 256, cudaMemcpyDeviceToHost, d2h_);
    if (ddk[0]) copy_ranges(dk[0], ddk[0], rkv, G * 256, cudaMemcpyDeviceToHost, d2h_);
    if (ddv[0]) copy_ranges(dv[0], ddv[0], rkv, G * 256, cudaMemcpyDeviceToHost, d2h_);
    auto& fr = bwd_st_.free[slot];
    if (fr.empty()) fr.push_back(staging_event(0));
    CUDA_OK(cudaEventRecord(fr[0], d2h_));
  }
  for (int d = 0; d < R_; ++d) {
    // re-zero the fp32 accumulators for the next backward on the aux stream, once this
    // call's gathers (and gradient returns) have read them: off the critical path, it
    // overlaps whatever the caller runs next (the next step's input load and forward)
    if (!local(d)) continue;
    DevState& D = dev_[d];
    DeviceGuard gd(D.ordinal);
    if (!opt.aux_zero) continue;  // zeroed at the start of the next backward instead
    CUDA_OK(cudaEventRecord(D.bwd_end, D.cs));
    CUDA_OK(cudaStreamWaitEvent(D.as, D.bwd_end, 0));
    zero_accumulators(d, D.as);
    CUDA_OK(cudaEventRecord(D.aux_done, D.as));
  }
  acc_dirty_ = !opt.aux_zero;
  release_caller();  // dq / dk / dv (device buffers) are ready in the caller's stream order
  fill_report(rep, true);
}

void Executor::zero_accumulators(int d, cudaStream_t s) {
  DevState& D = dev_[d];
  const int64_t SR = D.slot_rows;
  CUDA_OK(cudaMemsetAsync(D.dq_acc, 0, std::max<int64_t>(1, D.cap_q) * SR * 512, s));
  CUDA_OK(cudaMemsetAsync(D.dkv_acc, 0, std::max<int64_t>(1, D.cap_kv) * 2 * SR * 512, s));
}

void Executor::synchronize() {
  if (host_only_) return;
  for (auto& D : dev_) {
    DeviceGuard gd(D.ordinal);
    CUDA_OK(cudaStreamSynchronize(D.cs));
    CUDA_OK(cudaStreamSynchronize(D.ms));
    CUDA_OK(cudaStreamSynchronize(D.as));
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

// dcp_gpu_pipeline.hpp — the reference's look-ahead planning pipeline with the B200
// executor as its consumer (reference: proj/include/dcp/pipeline.hpp:100-225).
//
//   PipelineResult r = dcp::gpu::pipeline_run(cfg, batches);            // same arguments
//   PipelineResult r = dcp::gpu::pipeline_run(cfg, batches, {0,1,...});  // plan device -> GPU
//
// The reference's pipeline_run calls dcp::run (the CPU simulator) internally, so the swap
// needs its own driver; this one keeps the reference's protocol and types:
//   * kappa + 1 planner threads (kappa = max(lookahead, 0)) take iterations in order; a
//     thread may start planning iteration j only once j <= (iterations executed) + kappa;
//     iteration j is planned with placement seed cfg.seed + j;
//   * the consumer (calling thread) executes iteration i once plans i .. i + kappa (capped
//     at the last iteration) are complete, here on the GPU through dcp::gpu::run;
//   * a failure (planning or execution) marks only that iteration's report;
//   * the event log records PlanStart / PlanDone / SimStart / SimDone with a global order.
// Planning of later iterations overlaps GPU execution of the current one.
#pragma once

#include <algorithm>
#include <condition_variable>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "dcp/pipeline.hpp"
#include "dcp_gpu.hpp"

namespace dcp {
namespace gpu {

inline PipelineResult pipeline_run(const PipelineConfig& cfg, const std::vector<Batch>& batches,
                                   std::vector<int> cuda_ordinals = {}) {
  const int n = static_cast<int>(batches.size());
  const int kappa = std::max(cfg.lookahead, 0);
  PipelineResult out;
  out.reports.resize(static_cast<size_t>(n));
  if (n == 0) return out;

  enum State { kPending, kPlanning, kPlanned };
  std::mutex mu;
  std::condition_variable cv;
  std::vector<State> state(static_cast<size_t>(n), kPending);
  std::vector<PlannedBatch> planned(static_cast<size_t>(n));
  std::vector<std::string> plan_error(static_cast<size_t>(n));
  int next_to_plan = 0, executed = 0, order = 0;
  auto log = [&](PipelineEvent::Kind k, int it) { out.events.push_back({k, it, order++}); };  // under mu

  auto planner = [&]() {
    for (;;) {
      int it = -1;
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return next_to_plan >= n || next_to_plan <= executed + kappa; });
        if (next_to_plan >= n) return;
        it = next_to_plan++;
        state[static_cast<size_t>(it)] = kPlanning;
        log(PipelineEvent::PlanStart, it);
      }
      PlannedBatch pb;
      std::string err;
      try {
        PlannerConfig pc = cfg.planner;
        pc.placement.seed = cfg.seed + static_cast<std::uint64_t>(it);
        pb = plan_batch(batches[static_cast<size_t>(it)], cfg.topology, pc);
      } catch (const std::exception& e) {
        err = e.what();
      }
      std::lock_guard<std::mutex> lk(mu);
      planned[static_cast<size_t>(it)] = std::move(pb);
      plan_error[static_cast<size_t>(it)] = std::move(err);
      state[static_cast<size_t>(it)] = kPlanned;
      log(PipelineEvent::PlanDone, it);
      cv.notify_all();
    }
  };
  std::vector<std::thread> threads;
  threads.reserve(static_cast<size_t>(kappa) + 1);
  for (int t = 0; t <= kappa; ++t) threads.emplace_back(planner);

  for (int i = 0; i < n; ++i) {
    const int last = std::min(i + kappa, n - 1);
    {
      std::unique_lock<std::mutex> lk(mu);
      cv.wait(lk, [&] {
        for (int j = i; j <= last; ++j)
          if (state[static_cast<size_t>(j)] != kPlanned) return false;
        return true;
      });
      log(PipelineEvent::SimStart, i);
    }
    const Batch& batch = batches[static_cast<size_t>(i)];
    IterationReport& rep = out.reports[static_cast<size_t>(i)];
    rep.iteration = i;
    rep.tokens = batch.total_tokens();
    rep.sequences = static_cast<int>(batch.sequences.size());
    if (!plan_error[static_cast<size_t>(i)].empty()) {
      rep.failed = true;
      rep.error = plan_error[static_cast<size_t>(i)];
    } else {
      try {
        const PlannedBatch& pb = planned[static_cast<size_t>(i)];
        SimOptions opts;
        opts.numeric = cfg.numeric;
        opts.cost = cfg.cost;
        const BatchPayload payload =
            cfg.numeric ? make_payload(batch, cfg.seed + static_cast<std::uint64_t>(i)) : BatchPayload{};
        std::vector<int> ords = cuda_ordinals;
        if (ords.empty()) ords.assign(static_cast<size_t>(pb.plans.size()), 0);
        const SimResult sim = dcp::gpu::run(pb.plans, pb.graph, payload, cfg.topology, opts, ords);
        rep.comm_bytes = sim.report.total_bytes;
        rep.inter_machine_bytes = pb.placement.inter_machine_bytes;
        rep.flops = sim.report.total_flops;
        rep.makespan = sim.report.makespan;
      } catch (const std::exception& e) {
        rep.failed = true;
        rep.error = e.what();
      }
    }
    std::lock_guard<std::mutex> lk(mu);
    log(PipelineEvent::SimDone, i);
    ++executed;
    cv.notify_all();
  }
  {
    std::lock_guard<std::mutex> lk(mu);
    executed = n;  // no planner may remain gated
    cv.notify_all();
  }
  for (auto& t : threads) t.join();
  return out;
}

}  // namespace gpu
}  // namespace dcp

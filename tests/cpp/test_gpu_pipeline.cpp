// Look-ahead pipeline with the B200 executor as consumer (include/dcp_gpu_pipeline.hpp,
// SURVEY 8(f)2) against the reference's pipeline_run (proj/include/dcp/pipeline.hpp:105)
// with its CPU simulator, on the same batches (the reference's random fixtures,
// tests/fixtures.hpp:172-189, at D = 128): per-iteration reports must be identical and the
// event log must follow the look-ahead protocol. Built here against the unchanged reference
// headers (tools/build.py); run on a B200 by tests/test_gpu_dropin.py.
#include <cstdio>
#include <map>

#include "dcp/pipeline.hpp"
#include "dcp_gpu_pipeline.hpp"
#include "fixtures.hpp"

using namespace dcp;

int main() {
  int failures = 0;
  std::mt19937_64 rng(4242);
  std::vector<Batch> batches;
  for (int i = 0; i < 6; ++i) {
    Batch b = fixtures::random_batch(rng, 700, 3, 2, 8);
    b.head_dim = 128;
    batches.push_back(std::move(b));
  }
  for (int kappa : {0, 2}) {
    for (bool numeric : {false, true}) {
      PipelineConfig cfg;
      cfg.topology.devices_per_machine = 2;
      cfg.planner.block_size = 128;
      cfg.planner.divisions = 3;
      cfg.lookahead = kappa;
      cfg.seed = 7;
      cfg.numeric = numeric;
      const PipelineResult ref = pipeline_run(cfg, batches);
      const PipelineResult gpu = gpu::pipeline_run(cfg, batches);
      for (size_t i = 0; i < batches.size(); ++i) {
        const auto& a = ref.reports[i];
        const auto& b = gpu.reports[i];
        const bool same = a.failed == b.failed && a.tokens == b.tokens && a.sequences == b.sequences &&
                          a.comm_bytes == b.comm_bytes && a.inter_machine_bytes == b.inter_machine_bytes &&
                          a.flops == b.flops && a.makespan == b.makespan;
        if (!same) {
          ++failures;
          std::printf("kappa %d numeric %d iter %zu: report mismatch (failed %d/%d bytes %llu/%llu flops %llu/%llu "
                      "makespan %.9g/%.9g) %s\n", kappa, numeric, i, a.failed, b.failed,
                      (unsigned long long)a.comm_bytes, (unsigned long long)b.comm_bytes,
                      (unsigned long long)a.flops, (unsigned long long)b.flops, a.makespan, b.makespan,
                      b.error.c_str());
        }
      }
      // protocol: one event of each kind per iteration; SimStart(i) after PlanDone(i..i+kappa);
      // PlanStart(j) after SimDone(j - kappa - 1)
      const int n = static_cast<int>(batches.size());
      std::map<std::pair<int, int>, int> at;  // (kind, iteration) -> order
      for (const auto& e : gpu.events) {
        if (at.count({e.kind, e.iteration})) ++failures;
        at[{e.kind, e.iteration}] = e.order;
      }
      if (static_cast<int>(at.size()) != 4 * n) ++failures;
      for (int i = 0; i < n; ++i) {
        for (int j = i; j <= std::min(i + kappa, n - 1); ++j)
          if (!(at[{PipelineEvent::PlanDone, j}] < at[{PipelineEvent::SimStart, i}])) {
            ++failures;
            std::printf("kappa %d: SimStart(%d) before PlanDone(%d)\n", kappa, i, j);
          }
        if (i - kappa - 1 >= 0 && !(at[{PipelineEvent::SimDone, i - kappa - 1}] < at[{PipelineEvent::PlanStart, i}])) {
          ++failures;
          std::printf("kappa %d: PlanStart(%d) before SimDone(%d)\n", kappa, i, i - kappa - 1);
        }
      }
      std::printf("kappa %d numeric %d: %zu iterations compared\n", kappa, numeric, batches.size());
    }
  }
  std::printf("%s (%d failures)\n", failures ? "FAIL" : "OK", failures);
  return failures ? 1 : 0;
}

// Drop-in check: the reference's own executor tests (tests/test_simexec.cpp:164-208, 251-270)
// with dcp::run swapped for dcp::gpu::run (include/dcp_gpu.hpp), D = 128, against the
// reference's dense oracle (tests/oracle.hpp:80-120). Built here against the unchanged
// reference headers (tools/build.py); run on a B200 by tests/test_gpu_dropin.py.
#include <cstdio>

#include "dcp/pipeline.hpp"
#include "dcp_gpu.hpp"
#include "fixtures.hpp"
#include "oracle.hpp"

using namespace dcp;

static double rel_error(const BatchOutputs& a, const BatchOutputs& b) {
  double mx = 0;
  for (const auto& s : b.o)
    for (const auto& m : s)
      for (double x : m.a) mx = std::max(mx, std::abs(x));
  return max_abs_error(a, b) / (mx > 0 ? mx : 1.0);
}

int main() {
  int failures = 0;
  // single device run equals the dense oracle (test_simexec.cpp:164-178)
  {
    std::mt19937_64 rng(127);
    for (int rep = 0; rep < 4; ++rep) {
      Batch b = fixtures::random_batch(rng, 400, 3, 2, 6);
      b.head_dim = 128;
      const BatchPayload payload = make_payload(b, 1000 + static_cast<std::uint64_t>(rep));
      BlockGraph g = generate_blocks(b, 128);
      DeviceTopology topo;
      const PlacementResult pl = place(g, topo, {});
      const DivisionSchedule s = schedule(g, pl, 2);
      const auto plans = compile_plans(s, g, pl);
      const SimResult sim = gpu::run(plans, g, payload, topo, {});
      const double err = rel_error(sim.outputs, oracle::dense_attention(b, payload));
      std::printf("single-device rep %d: rel err %.3e\n", rep, err);
      if (!(err <= 2e-2)) ++failures;
    }
  }
  // multi-device run equals the dense oracle and counts bytes exactly (:180-208)
  {
    std::mt19937_64 rng(131);
    int ran = 0;
    for (int rep = 0; rep < 8; ++rep) {
      Batch b = fixtures::random_batch(rng, 320, 3, 2, 4);
      b.head_dim = 128;
      DeviceTopology topo;
      topo.machines = 1 + static_cast<int>(rng() % 2);
      topo.devices_per_machine = 1 + static_cast<int>(rng() % 2);
      PlacementConfig pcfg;
      pcfg.eps_intra = 0.4;
      pcfg.eps_inter = 0.4;
      pcfg.eps_data = 0.6;
      pcfg.seed = static_cast<std::uint64_t>(rep);
      BlockGraph g = generate_blocks(b, 64);
      PlacementResult pl;
      try {
        pl = place(g, topo, pcfg);
      } catch (const InfeasibleError&) {
        continue;
      }
      const DivisionSchedule s = schedule(g, pl, 4);
      const auto plans = compile_plans(s, g, pl);
      verify_plans(plans, g);
      const BatchPayload payload = make_payload(b, 77);
      const SimResult sim = gpu::run(plans, g, payload, topo, {});
      const double err = rel_error(sim.outputs, oracle::dense_attention(b, payload));
      const bool bytes_ok = sim.report.total_bytes == communication_volume(g, pl).total;
      const SimResult ref = run(plans, g, {}, topo, SimOptions{false, {}});  // reference, cost mode
      const bool report_ok = ref.report.total_bytes == sim.report.total_bytes &&
                             ref.report.total_flops == sim.report.total_flops &&
                             ref.report.comm_bytes == sim.report.comm_bytes &&
                             ref.report.makespan == sim.report.makespan;
      std::printf("multi-device rep %d (R=%d): rel err %.3e bytes %llu ok=%d report=%d\n", rep,
                  topo.device_count(), err, static_cast<unsigned long long>(sim.report.total_bytes), bytes_ok,
                  report_ok);
      if (!(err <= 2e-2) || !bytes_ok || !report_ok) ++failures;
      ++ran;
    }
    if (ran == 0) ++failures;
  }
  // missing sender is reported as a deadlock (:251-270)
  {
    Batch b = fixtures::single_seq_batch(256, MaskDescriptor::causal(), 1, 1, 128);
    BlockGraph g = generate_blocks(b, 128);
    std::vector<int> group_dev = {0, 1};
    std::vector<int> comp_dev(g.comp_blocks.size());
    for (const auto& c : g.comp_blocks) comp_dev[static_cast<size_t>(c.id)] = c.q_tile;
    const PlacementResult pl = dcp::detail::make_placement(g, fixtures::two_devices(), group_dev, comp_dev);
    const DivisionSchedule s = schedule(g, pl, 2);
    auto plans = compile_plans(s, g, pl);
    auto& instrs = plans[0].instructions;
    instrs.erase(std::remove_if(instrs.begin(), instrs.end(),
                                [](const Instruction& ins) {
                                  const auto* l = std::get_if<CommLaunchInstr>(&ins.op);
                                  return l && l->send;
                                }),
                 instrs.end());
    bool deadlock = false;
    try {
      gpu::run(plans, g, make_payload(b, 1), fixtures::two_devices(), {});
    } catch (const DeadlockError&) {
      deadlock = true;
    }
    std::printf("missing sender -> DeadlockError: %d\n", deadlock);
    if (!deadlock) ++failures;
  }
  std::printf(failures ? "DROPIN FAIL (%d)\n" : "DROPIN PASS\n", failures);
  return failures ? 1 : 0;
}

// Cost-only drop-in check (no GPU needed): dcp::gpu::run with SimOptions{numeric = false}
// builds its SimReport from the plans and verifies them host-side (dcpx_check_plans), so it
// must equal the reference's cost-mode run() (simexec.hpp:207-423) for any head_dim -- here
// D = 64, which the sm_100a kernels do not execute -- and raise the reference's exception
// types on a broken plan (tests/test_simexec.cpp:251-270). Run by tests/test_boundary_cpu.py.
#include <cstdio>

#include "dcp/pipeline.hpp"
#include "dcp_gpu.hpp"
#include "fixtures.hpp"

using namespace dcp;

int main() {
  int failures = 0, ran = 0;
  std::mt19937_64 rng(977);
  for (int rep = 0; rep < 6; ++rep) {
    Batch b = fixtures::random_batch(rng, 320, 3, 2, 4);
    b.head_dim = 64;
    DeviceTopology topo;
    topo.machines = 1 + static_cast<int>(rng() % 2);
    topo.devices_per_machine = 1 + static_cast<int>(rng() % 3);
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
    const auto plans = compile_plans(schedule(g, pl, 3), g, pl);
    const SimResult ref = run(plans, g, {}, topo, SimOptions{false, {}});
    const SimResult got = gpu::run(plans, g, {}, topo, SimOptions{false, {}});
    const bool ok = ref.report.total_bytes == got.report.total_bytes &&
                    ref.report.total_flops == got.report.total_flops && ref.report.comm_bytes == got.report.comm_bytes &&
                    ref.report.comp_flops == got.report.comp_flops &&
                    ref.report.per_device_send == got.report.per_device_send &&
                    ref.report.per_device_recv == got.report.per_device_recv && ref.report.makespan == got.report.makespan;
    std::printf("cost-only rep %d (R=%d, D=64): report equal %d\n", rep, topo.device_count(), ok);
    failures += !ok;
    ++ran;
  }
  if (ran == 0) ++failures;
  {
    Batch b = fixtures::single_seq_batch(256, MaskDescriptor::causal(), 1, 1, 128);
    BlockGraph g = generate_blocks(b, 128);
    std::vector<int> group_dev = {0, 1};
    std::vector<int> comp_dev(g.comp_blocks.size());
    for (const auto& c : g.comp_blocks) comp_dev[static_cast<size_t>(c.id)] = c.q_tile;
    const PlacementResult pl = dcp::detail::make_placement(g, fixtures::two_devices(), group_dev, comp_dev);
    auto plans = compile_plans(schedule(g, pl, 2), g, pl);
    auto& instrs = plans[0].instructions;
    instrs.erase(std::remove_if(instrs.begin(), instrs.end(),
                                [](const Instruction& ins) {
                                  const auto* l = std::get_if<CommLaunchInstr>(&ins.op);
                                  return l && l->send;
                                }),
                 instrs.end());
    bool ref_dl = false, got_dl = false;
    try {
      run(plans, g, {}, fixtures::two_devices(), SimOptions{false, {}});
    } catch (const DeadlockError&) {
      ref_dl = true;
    }
    try {
      gpu::run(plans, g, {}, fixtures::two_devices(), SimOptions{false, {}});
    } catch (const DeadlockError&) {
      got_dl = true;
    }
    std::printf("cost-only missing sender -> DeadlockError: reference %d, drop-in %d\n", ref_dl, got_dl);
    failures += !(ref_dl && got_dl);
  }
  std::printf(failures ? "COST FAIL (%d)\n" : "COST PASS\n", failures);
  return failures ? 1 : 0;
}

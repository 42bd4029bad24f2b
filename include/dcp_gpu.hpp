// dcp_gpu.hpp — drop-in replacement for dcp::run (reference: proj/include/dcp/simexec.hpp:207-209).
//
//   #include "dcp/simexec.hpp"   // the reference (caller side)
//   #include "dcp_gpu.hpp"       // this header, links against libdcpx.so
//   SimResult r = dcp::gpu::run(plans, g, payload, topo, opts);   // same signature
//
// Header-only glue on the caller's side of the C ABI (include/dcpx.h): it flattens the
// reference's ExecutionPlans / BlockGraph into dcpx views, converts the FP64 payload to
// packed bf16, runs the sm_100a executor and converts the outputs back into the
// reference's BatchOutputs / SimReport. Status codes are rethrown as the reference's
// exception types (types.hpp:17-45). Plan device d runs on CUDA device
// cuda_ordinals[d] (default: all on device 0, i.e. a single-GPU emulation of R devices).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "dcp/simexec.hpp"
#include "dcpx.h"

namespace dcp {
namespace gpu {

namespace detail {

inline void throw_status(dcpx_status st, const char* msg) {
  const std::string m = msg ? msg : "";
  switch (st) {
    case DCPX_OK: return;
    case DCPX_DEADLOCK: throw DeadlockError(m);
    case DCPX_TAG_MISMATCH: throw TagMismatchError(m);
    case DCPX_BUFFER_OVERFLOW: throw BufferOverflowError(m);
    case DCPX_INFEASIBLE: throw InfeasibleError(m);
    default: throw Error("dcpx: " + m);
  }
}

struct Flat {  // owned storage behind the views
  std::vector<int64_t> seq_lengths, block_sizes, seq_offsets;
  std::vector<int32_t> ranges;
  std::vector<dcpx_data_block> data_blocks;
  std::vector<dcpx_comp_block> comp_blocks;
  struct Dev {
    std::vector<dcpx_block_slot> rq, rkv, ro, blocks;
    std::vector<dcpx_instruction> ins;
    std::vector<std::string> tags;
    std::vector<dcpx_attention_item> items;
    std::vector<int32_t> srcs, rows;
    std::vector<dcpx_copy_item> copies;
  };
  std::vector<Dev> devs;
  std::vector<dcpx_plan_view> views;
  dcpx_graph_view graph{};
  dcpx_mask_view masks{};
};

inline void flatten(const std::vector<ExecutionPlan>& plans, const BlockGraph& g, Flat& f) {
  const auto& b = g.batch;
  f.seq_offsets.assign(1, 0);
  for (size_t s = 0; s < b.sequences.size(); ++s) {
    f.seq_lengths.push_back(b.sequences[s].length);
    f.block_sizes.push_back(g.block_sizes[s]);
    f.seq_offsets.push_back(f.seq_offsets.back() + b.sequences[s].length);
    for (const auto& row : g.masks[s].rows) {
      int32_t r4[4] = {0, 0, 0, 0};
      for (int i = 0; i < row.count; ++i) {
        r4[2 * i] = static_cast<int32_t>(row.r[i].begin);
        r4[2 * i + 1] = static_cast<int32_t>(row.r[i].end);
      }
      f.ranges.insert(f.ranges.end(), r4, r4 + 4);
    }
  }
  for (const auto& d : g.data_blocks)
    f.data_blocks.push_back({d.id, static_cast<int32_t>(d.kind), d.seq, d.head, d.tile, 0, d.tokens.begin,
                             d.tokens.end, d.size_bytes});
  for (const auto& c : g.comp_blocks)
    f.comp_blocks.push_back({c.id, c.q_block, c.kv_block, c.o_block, c.seq, c.head, c.q_tile, c.kv_tile,
                             c.attended_pairs, c.flops_weight});
  f.devs.resize(plans.size());
  for (size_t p = 0; p < plans.size(); ++p) {
    const auto& plan = plans[p];
    auto& D = f.devs[p];
    for (const auto& r : plan.buffers.resident_q) D.rq.push_back({r.block, r.slot});
    for (const auto& r : plan.buffers.resident_kv) D.rkv.push_back({r.block, r.slot});
    for (const auto& r : plan.buffers.resident_o) D.ro.push_back({r.block, r.slot});
    std::vector<int> tag_of;
    for (const auto& ins : plan.instructions) {
      dcpx_instruction x{};
      x.division = ins.division;
      int tag = -1;
      if (const auto* a = std::get_if<AttentionInstr>(&ins.op)) {
        x.op = DCPX_OP_ATTENTION;
        x.count = static_cast<int32_t>(a->items.size());
        x.offset = static_cast<int64_t>(D.items.size());
        for (const auto& it : a->items) {
          dcpx_attention_item y{};
          y.comp_id = it.comp_id; y.q_slot = it.q_slot; y.kv_slot = it.kv_slot; y.out_slot = it.out_slot;
          y.seq = it.seq; y.head = it.head;
          y.q_begin = it.q_tokens.begin; y.q_end = it.q_tokens.end;
          y.kv_begin = it.kv_tokens.begin; y.kv_end = it.kv_tokens.end;
          // the item carries its own rows (plan.hpp:231-242): pass them explicitly
          y.rows_offset = static_cast<int64_t>(D.rows.size() / 4);
          for (const auto& row : it.rows) {
            int32_t r4[4] = {0, 0, 0, 0};
            for (int i = 0; i < row.count; ++i) {
              r4[2 * i] = static_cast<int32_t>(row.r[i].begin);
              r4[2 * i + 1] = static_cast<int32_t>(row.r[i].end);
            }
            D.rows.insert(D.rows.end(), r4, r4 + 4);
          }
          D.items.push_back(y);
        }
      } else if (const auto* r = std::get_if<ReductionInstr>(&ins.op)) {
        x.op = DCPX_OP_REDUCTION;
        x.dst = r->dst;
        x.count = static_cast<int32_t>(r->srcs.size());
        x.offset = static_cast<int64_t>(D.srcs.size());
        D.srcs.insert(D.srcs.end(), r->srcs.begin(), r->srcs.end());
      } else if (const auto* c = std::get_if<CopyInstr>(&ins.op)) {
        x.op = DCPX_OP_COPY;
        x.count = static_cast<int32_t>(c->items.size());
        x.offset = static_cast<int64_t>(D.copies.size());
        for (const auto& it : c->items) D.copies.push_back({it.src_slot, it.dst_slot});
      } else if (const auto* l = std::get_if<CommLaunchInstr>(&ins.op)) {
        x.op = DCPX_OP_COMM_LAUNCH;
        x.send = l->send ? 1 : 0;
        x.peer = l->peer;
        x.count = static_cast<int32_t>(l->blocks.size());
        x.offset = static_cast<int64_t>(D.blocks.size());
        for (const auto& tb : l->blocks) D.blocks.push_back({tb.block, tb.slot});
        tag = static_cast<int>(D.tags.size());
        D.tags.push_back(l->tag);
      } else if (const auto* w = std::get_if<CommWaitInstr>(&ins.op)) {
        x.op = DCPX_OP_COMM_WAIT;
        tag = static_cast<int>(D.tags.size());
        D.tags.push_back(w->tag);
      }
      tag_of.push_back(tag);
      D.ins.push_back(x);
    }
    for (size_t i = 0; i < D.ins.size(); ++i)
      D.ins[i].tag = tag_of[i] >= 0 ? D.tags[static_cast<size_t>(tag_of[i])].c_str() : nullptr;
    dcpx_plan_view v{};
    v.version = plan.version;
    v.device = plan.device;
    v.divisions = plan.divisions;
    for (int k = 0; k < 3; ++k) v.capacity[k] = plan.buffers.capacity[static_cast<size_t>(k)];
    v.n_resident_q = static_cast<int32_t>(D.rq.size());
    v.n_resident_kv = static_cast<int32_t>(D.rkv.size());
    v.n_resident_o = static_cast<int32_t>(D.ro.size());
    v.resident_q = D.rq.data(); v.resident_kv = D.rkv.data(); v.resident_o = D.ro.data();
    v.n_instructions = static_cast<int32_t>(D.ins.size());
    v.instructions = D.ins.data();
    v.items = D.items.data(); v.srcs = D.srcs.data(); v.copies = D.copies.data();
    v.blocks = D.blocks.data(); v.rows = D.rows.data();
    f.views.push_back(v);
  }
  f.graph.heads = b.heads; f.graph.kv_groups = b.kv_groups; f.graph.head_dim = b.head_dim;
  f.graph.bytes_per_element = b.bytes_per_element;
  f.graph.num_seqs = static_cast<int32_t>(b.sequences.size());
  f.graph.num_data_blocks = static_cast<int32_t>(f.data_blocks.size());
  f.graph.num_comp_blocks = static_cast<int32_t>(f.comp_blocks.size());
  f.graph.seq_lengths = f.seq_lengths.data(); f.graph.block_sizes = f.block_sizes.data();
  f.graph.data_blocks = f.data_blocks.data(); f.graph.comp_blocks = f.comp_blocks.data();
  f.masks.seq_offsets = f.seq_offsets.data();
  f.masks.ranges = f.ranges.data();
}

inline void cuda_check(cudaError_t e) {
  if (e != cudaSuccess) throw Error(std::string("cuda: ") + cudaGetErrorString(e));
}

}  // namespace detail

// Same signature as dcp::run (simexec.hpp:207-209), plus optional CUDA ordinals.
inline SimResult run(const std::vector<ExecutionPlan>& plans, const BlockGraph& g, const BatchPayload& payload,
                     const DeviceTopology& topo, const SimOptions& options = {},
                     std::vector<int> cuda_ordinals = {}) {
  const int R = static_cast<int>(plans.size());
  if (R != topo.device_count()) throw Error("run: plan count does not match topology");
  if (cuda_ordinals.empty()) cuda_ordinals.assign(static_cast<size_t>(R), 0);
  detail::Flat f;
  detail::flatten(plans, g, f);
  dcpx_ctx* ctx = nullptr;
  struct Guard {
    dcpx_ctx* c;
    ~Guard() { dcpx_destroy(c); }
  } guard{nullptr};
  if (options.numeric) {
    detail::throw_status(dcpx_create(R, cuda_ordinals.data(), DCPX_TRANSPORT_LOCAL, &ctx), dcpx_last_error(nullptr));
    guard.c = ctx;
    detail::throw_status(dcpx_prepare(ctx, R, f.views.data(), &f.graph, &f.masks), dcpx_last_error(ctx));
  } else {
    // cost-only run (SimOptions::numeric false): no GPU work, so no context; the plans still
    // get the reference's checks (verify_plans and the lockstep deadlock / tag replay), and
    // any head_dim / element size is accepted as the reference's run() accepts it
    char err[1024];
    const dcpx_status st = dcpx_check_plans(R, f.views.data(), &f.graph, &f.masks, err, sizeof(err));
    detail::throw_status(st, err);
  }

  const auto& b = g.batch;
  const int H = b.heads, G = b.kv_groups, D = b.head_dim;
  const int64_t TT = f.seq_offsets.back();
  SimResult result;
  dcpx_report rep{};
  if (options.numeric) {
    std::vector<__nv_bfloat16> q(static_cast<size_t>(TT) * H * D), k(static_cast<size_t>(TT) * G * D),
        v(static_cast<size_t>(TT) * G * D), o(static_cast<size_t>(TT) * H * D);
    for (size_t s = 0; s < b.sequences.size(); ++s) {
      const int L = static_cast<int>(b.sequences[s].length);
      const int64_t off = f.seq_offsets[s];
      for (int i = 0; i < L; ++i)
        for (int d = 0; d < D; ++d) {
          for (int h = 0; h < H; ++h)
            q[((off + i) * H + h) * D + d] = __float2bfloat16(static_cast<float>(payload.seqs[s].q[h].at(i, d)));
          for (int gr = 0; gr < G; ++gr) {
            k[((off + i) * G + gr) * D + d] = __float2bfloat16(static_cast<float>(payload.seqs[s].k[gr].at(i, d)));
            v[((off + i) * G + gr) * D + d] = __float2bfloat16(static_cast<float>(payload.seqs[s].v[gr].at(i, d)));
          }
        }
    }
    detail::throw_status(dcpx_load_inputs_host(ctx, q.data(), k.data(), v.data()), dcpx_last_error(ctx));
    detail::throw_status(dcpx_forward_host(ctx, o.data(), nullptr, &rep), dcpx_last_error(ctx));
    detail::throw_status(dcpx_synchronize(ctx), dcpx_last_error(ctx));  // host outputs are asynchronous
    result.outputs.o.resize(b.sequences.size());
    for (size_t s = 0; s < b.sequences.size(); ++s) {
      const int L = static_cast<int>(b.sequences[s].length);
      const int64_t off = f.seq_offsets[s];
      result.outputs.o[s].assign(static_cast<size_t>(H), Matrix(L, D));
      for (int h = 0; h < H; ++h)
        for (int i = 0; i < L; ++i)
          for (int d = 0; d < D; ++d)
            result.outputs.o[s][static_cast<size_t>(h)].at(i, d) =
                static_cast<double>(__bfloat162float(o[((off + i) * H + h) * D + d]));
    }
  }
  // SimReport (simexec.hpp:153-162): byte tables from the plans exactly as run() charges them
  const int T = plans.empty() ? 0 : plans[0].divisions;
  SimReport& r = result.report;
  r.comm_bytes.resize(static_cast<size_t>(T) + 1);
  r.comp_flops.assign(static_cast<size_t>(T) + 1, std::vector<FlopCount>(static_cast<size_t>(R), 0));
  r.per_device_send.assign(static_cast<size_t>(R), 0);
  r.per_device_recv.assign(static_cast<size_t>(R), 0);
  for (const auto& plan : plans)
    for (const auto& ins : plan.instructions) {
      if (const auto* l = std::get_if<CommLaunchInstr>(&ins.op)) {
        if (!l->send) continue;
        ByteCount bytes = 0;
        for (const auto& tb : l->blocks) bytes += g.data_blocks[static_cast<size_t>(tb.block)].size_bytes;
        r.total_bytes += bytes;
        r.per_device_send[static_cast<size_t>(plan.device)] += bytes;
        r.per_device_recv[static_cast<size_t>(l->peer)] += bytes;
        r.comm_bytes[static_cast<size_t>(ins.division)][{plan.device, l->peer}] += bytes;
      } else if (const auto* a = std::get_if<AttentionInstr>(&ins.op)) {
        for (const auto& item : a->items) {
          FlopCount pairs = 0;
          for (const auto& row : item.rows) pairs += static_cast<FlopCount>(row.total());
          r.comp_flops[static_cast<size_t>(ins.division)][static_cast<size_t>(plan.device)] +=
              4 * pairs * static_cast<FlopCount>(D);
          r.total_flops += 4 * pairs * static_cast<FlopCount>(D);
        }
      }
    }
  if (options.numeric && rep.total_bytes != r.total_bytes)
    throw Error("dcpx: executed bytes differ from the plan's byte table");
  r.makespan = dcp::detail::cost_from_tables(r.comp_flops, r.comm_bytes, topo, options.cost).makespan;
  return result;
}

}  // namespace gpu
}  // namespace dcp

// Caller-side shim: the reference DCP planner, unchanged, behind a small C API.
//
// This file contains no planner logic. It #includes the reference's header-only
// planner from /root/reference/proj/include (never copied into this repo) and
// flattens its artefacts — BlockGraph (blocks.hpp:53-85), PlacementResult
// (placement.hpp:7-22), CommVolume (placement.hpp:164-173) and the per-device
// ExecutionPlans (plan.hpp:101-107) — into the POD views declared in
// include/dcpx.h, which is exactly what a maintainer would add on the reference
// side to call the B200 executor.
//
// Entry points used:
//   dcp::plan_batch            pipeline.hpp:29-38
//   dcp::make_batches          pipeline.hpp:42-65
//   dcp::synth_sequences       synth.hpp:84-100
//   dcp::generate_blocks       blocks.hpp:102-203
//   dcp::detail::make_placement baselines.hpp:12-34 (explicit placements, tests)
//   dcp::ring_placement / zigzag_placement baselines.hpp:46-76
//   dcp::schedule / compile_plans / verify_plans / communication_volume
//   fixtures::random_batch     tests/fixtures.hpp:172-189 (seeded fuzz batches)
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "dcp/baselines.hpp"
#include "dcp/pipeline.hpp"
#include "dcp_partition_parallel.hpp"
#if __has_include(<json.hpp>)
#include <filesystem>
#include "dcp/io.hpp"  // the reference's plan / graph / placement JSON writers (io.hpp:72-352)
#define DCPP_HAVE_JSON 1
#endif
#include "dcp/synth.hpp"
#include "fixtures.hpp"
#include "../include/dcpx.h"

namespace {

struct SeqSpecC {
  int64_t length;
  int32_t kind;  // MaskKind
  int32_t window_blocks, sink_blocks, test_blocks;
  int64_t sink, window, block;
  int64_t question_len;
  int32_t n_answers, _pad;
  int64_t answer_lens[16];
};

struct DevicePlanFlat {
  int32_t device = 0, divisions = 0;
  int32_t capacity[3] = {0, 0, 0};
  std::vector<dcpx_block_slot> res_q, res_kv, res_o;
  std::vector<int32_t> instr;  // [n][8]: op, division, send, peer, dst, count, offset, tag index
  std::vector<dcpx_attention_item> items;
  std::vector<int32_t> srcs;
  std::vector<dcpx_copy_item> copies;
  std::vector<dcpx_block_slot> blocks;
  std::vector<std::string> tags;
  std::string tag_blob;  // tags joined by '\n'
};

}  // namespace

struct dcpp_planned {
  dcp::PlannedBatch pb;
  // flattened graph
  std::vector<int64_t> seq_lengths, block_sizes, seq_offsets;
  std::vector<int32_t> ranges;  // [T][4]
  std::vector<dcpx_data_block> data_blocks;
  std::vector<dcpx_comp_block> comp_blocks;
  std::vector<int32_t> data_block_device, comp_block_device;
  std::vector<uint64_t> dev_flops, per_device_send, per_device_recv;
  std::vector<uint64_t> volume;  // total, q_xfer, kv_xfer, o_xfer, inter_machine
  std::vector<DevicePlanFlat> devs;
  std::vector<int32_t> header;   // R, T, H, G, D, bpe, S, N, M
};

struct dcpp_batch {
  dcp::Batch batch;
};

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const dcp::InfeasibleError*>(&e)) return DCPX_INFEASIBLE;
  if (dynamic_cast<const dcp::BufferOverflowError*>(&e)) return DCPX_BUFFER_OVERFLOW;
  if (dynamic_cast<const dcp::TagMismatchError*>(&e)) return DCPX_TAG_MISMATCH;
  if (dynamic_cast<const dcp::DeadlockError*>(&e)) return DCPX_DEADLOCK;
  return DCPX_ERROR;
}

dcp::MaskDescriptor mask_from_c(const SeqSpecC& s) {
  switch (s.kind) {
    case 0: return dcp::MaskDescriptor::causal();
    case 1: return dcp::MaskDescriptor::lambda(s.sink, s.window);
    case 2: return dcp::MaskDescriptor::causal_blockwise(s.block, s.window_blocks, s.sink_blocks,
                                                         s.test_blocks);
    case 3: {
      std::vector<dcp::TokenIndex> a(s.answer_lens, s.answer_lens + s.n_answers);
      return dcp::MaskDescriptor::shared_question(s.question_len, std::move(a));
    }
  }
  throw dcp::Error("unknown mask kind");
}

void mask_to_c(const dcp::SequenceSpec& spec, SeqSpecC& s) {
  std::memset(&s, 0, sizeof(s));
  s.length = spec.length;
  s.kind = static_cast<int32_t>(spec.mask.kind);
  s.sink = spec.mask.sink_tokens;
  s.window = spec.mask.window;
  s.block = spec.mask.block;
  s.window_blocks = spec.mask.window_blocks;
  s.sink_blocks = spec.mask.sink_blocks;
  s.test_blocks = spec.mask.test_blocks;
  s.question_len = spec.mask.question_len;
  s.n_answers = static_cast<int32_t>(std::min<size_t>(spec.mask.answer_lens.size(), 16));
  for (int i = 0; i < s.n_answers; ++i) s.answer_lens[i] = spec.mask.answer_lens[i];
}

void flatten(dcpp_planned& p) {
  const auto& g = p.pb.graph;
  const auto& b = g.batch;
  const int R = p.pb.placement.device_count();
  const int S = static_cast<int>(b.sequences.size());
  p.header = {R, p.pb.schedule.divisions, b.heads, b.kv_groups, b.head_dim,
              b.bytes_per_element, S, static_cast<int32_t>(g.data_blocks.size()),
              static_cast<int32_t>(g.comp_blocks.size())};
  p.seq_offsets.assign(1, 0);
  for (int s = 0; s < S; ++s) {
    p.seq_lengths.push_back(b.sequences[s].length);
    p.block_sizes.push_back(g.block_sizes[s]);
    p.seq_offsets.push_back(p.seq_offsets.back() + b.sequences[s].length);
    for (const auto& row : g.masks[s].rows) {
      int32_t r4[4] = {0, 0, 0, 0};
      for (int i = 0; i < row.count; ++i) {
        r4[2 * i] = static_cast<int32_t>(row.r[i].begin);
        r4[2 * i + 1] = static_cast<int32_t>(row.r[i].end);
      }
      p.ranges.insert(p.ranges.end(), r4, r4 + 4);
    }
  }
  for (const auto& d : g.data_blocks) {
    dcpx_data_block x{};
    x.id = d.id; x.kind = static_cast<int32_t>(d.kind); x.seq = d.seq; x.head = d.head;
    x.tile = d.tile; x.tok_begin = d.tokens.begin; x.tok_end = d.tokens.end;
    x.size_bytes = d.size_bytes;
    p.data_blocks.push_back(x);
  }
  for (const auto& c : g.comp_blocks) {
    dcpx_comp_block x{};
    x.id = c.id; x.q_block = c.q_block; x.kv_block = c.kv_block; x.o_block = c.o_block;
    x.seq = c.seq; x.head = c.head; x.q_tile = c.q_tile; x.kv_tile = c.kv_tile;
    x.attended_pairs = c.attended_pairs; x.flops_weight = c.flops_weight;
    p.comp_blocks.push_back(x);
  }
  const auto& pl = p.pb.placement;
  p.data_block_device.assign(pl.data_block_device.begin(), pl.data_block_device.end());
  p.comp_block_device.assign(pl.comp_block_device.begin(), pl.comp_block_device.end());
  for (const auto& bal : pl.balance) p.dev_flops.push_back(bal.flops);
  const auto& v = p.pb.volume;
  p.per_device_send.assign(v.per_device_send.begin(), v.per_device_send.end());
  p.per_device_recv.assign(v.per_device_recv.begin(), v.per_device_recv.end());
  p.volume = {v.total, v.q_block_transfers, v.kv_block_transfers, v.o_block_transfers,
              v.inter_machine};

  for (const auto& plan : p.pb.plans) {
    DevicePlanFlat f;
    f.device = plan.device;
    f.divisions = plan.divisions;
    for (int k = 0; k < 3; ++k) f.capacity[k] = plan.buffers.capacity[k];
    for (const auto& r : plan.buffers.resident_q) f.res_q.push_back({r.block, r.slot});
    for (const auto& r : plan.buffers.resident_kv) f.res_kv.push_back({r.block, r.slot});
    for (const auto& r : plan.buffers.resident_o) f.res_o.push_back({r.block, r.slot});
    for (const auto& ins : plan.instructions) {
      int32_t rec[8] = {0, ins.division, 0, 0, 0, 0, 0, -1};
      if (const auto* a = std::get_if<dcp::AttentionInstr>(&ins.op)) {
        rec[0] = DCPX_OP_ATTENTION;
        rec[5] = static_cast<int32_t>(a->items.size());
        rec[6] = static_cast<int32_t>(f.items.size());
        for (const auto& it : a->items) {
          dcpx_attention_item x{};
          x.comp_id = it.comp_id; x.q_slot = it.q_slot; x.kv_slot = it.kv_slot;
          x.out_slot = it.out_slot; x.seq = it.seq; x.head = it.head;
          x.q_begin = it.q_tokens.begin; x.q_end = it.q_tokens.end;
          x.kv_begin = it.kv_tokens.begin; x.kv_end = it.kv_tokens.end;
          x.rows_offset = -1;  // rows are re-derived from the mask (plan.hpp:231-242)
          f.items.push_back(x);
        }
      } else if (const auto* r = std::get_if<dcp::ReductionInstr>(&ins.op)) {
        rec[0] = DCPX_OP_REDUCTION;
        rec[4] = r->dst;
        rec[5] = static_cast<int32_t>(r->srcs.size());
        rec[6] = static_cast<int32_t>(f.srcs.size());
        f.srcs.insert(f.srcs.end(), r->srcs.begin(), r->srcs.end());
      } else if (const auto* c = std::get_if<dcp::CopyInstr>(&ins.op)) {
        rec[0] = DCPX_OP_COPY;
        rec[5] = static_cast<int32_t>(c->items.size());
        rec[6] = static_cast<int32_t>(f.copies.size());
        for (const auto& it : c->items) f.copies.push_back({it.src_slot, it.dst_slot});
      } else if (const auto* l = std::get_if<dcp::CommLaunchInstr>(&ins.op)) {
        rec[0] = DCPX_OP_COMM_LAUNCH;
        rec[2] = l->send ? 1 : 0;
        rec[3] = l->peer;
        rec[5] = static_cast<int32_t>(l->blocks.size());
        rec[6] = static_cast<int32_t>(f.blocks.size());
        for (const auto& tb : l->blocks) f.blocks.push_back({tb.block, tb.slot});
        rec[7] = static_cast<int32_t>(f.tags.size());
        f.tags.push_back(l->tag);
      } else if (const auto* w = std::get_if<dcp::CommWaitInstr>(&ins.op)) {
        rec[0] = DCPX_OP_COMM_WAIT;
        rec[7] = static_cast<int32_t>(f.tags.size());
        f.tags.push_back(w->tag);
      }
      f.instr.insert(f.instr.end(), rec, rec + 8);
    }
    for (const auto& t : f.tags) { f.tag_blob += t; f.tag_blob += '\n'; }
    p.devs.push_back(std::move(f));
  }
}

struct CfgC {
  int32_t machines, devices_per_machine, divisions, max_slots_per_kind;
  int64_t block_size;
  double eps_inter, eps_intra, eps_data;
  uint64_t seed;
  int32_t verify;
  int32_t threads;  // 1: the reference plan_batch, unchanged; 0 (all cores) or > 1: plan_batch_parallel
};

dcp::DeviceTopology topo_of(const CfgC& c) {
  dcp::DeviceTopology t;
  t.machines = c.machines;
  t.devices_per_machine = c.devices_per_machine;
  return t;
}

}  // namespace

extern "C" {

const char* dcpp_last_error() { return g_err.c_str(); }

// Batch construction ------------------------------------------------------------------
int dcpp_batch_from_specs(const SeqSpecC* specs, int n, int heads, int kv_groups, int head_dim,
                          int bpe, int64_t token_budget, dcpp_batch** out) {
  try {
    auto b = std::make_unique<dcpp_batch>();
    b->batch.heads = heads;
    b->batch.kv_groups = kv_groups;
    b->batch.head_dim = head_dim;
    b->batch.bytes_per_element = bpe;
    for (int i = 0; i < n; ++i) {
      dcp::SequenceSpec s;
      s.seq_id = "s" + std::to_string(i);
      s.length = specs[i].length;
      s.mask = mask_from_c(specs[i]);
      b->batch.sequences.push_back(std::move(s));
    }
    b->batch.token_budget = token_budget > 0 ? token_budget : b->batch.total_tokens();
    b->batch.validate();
    *out = b.release();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// synth_sequences (synth.hpp:84-100) + make_batches (pipeline.hpp:42-65); returns
// batch `index`. dist: 0 LongAlign, 1 LDC. mask params follow SynthConfig defaults
// when the corresponding argument is negative.
int dcpp_batch_from_synth(int dist, double scale, int64_t max_len, int64_t min_len, int mask_kind,
                          int count, uint64_t seed, int64_t token_budget, int index, int heads,
                          int kv_groups, int head_dim, int bpe, dcpp_batch** out,
                          int* n_batches) {
  try {
    dcp::SynthConfig cfg;
    cfg.dist = dist == 0 ? dcp::LengthDist::LongAlign : dcp::LengthDist::LongDataCollections;
    cfg.scale = scale;
    cfg.max_len = max_len;
    if (min_len > 0) cfg.min_len = min_len;
    cfg.mask = static_cast<dcp::MaskKind>(mask_kind);
    const auto stream = dcp::synth_sequences(cfg, count, seed);
    dcp::Batch proto;
    proto.token_budget = token_budget;
    proto.heads = heads;
    proto.kv_groups = kv_groups;
    proto.head_dim = head_dim;
    proto.bytes_per_element = bpe;
    const auto batches = dcp::make_batches(stream, proto);
    *n_batches = static_cast<int>(batches.size());
    if (index < 0 || index >= static_cast<int>(batches.size()))
      throw dcp::Error("batch index out of range");
    auto b = std::make_unique<dcpp_batch>();
    b->batch = batches[static_cast<size_t>(index)];
    *out = b.release();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// fixtures::random_batch (tests/fixtures.hpp:172-189) with an overridden head_dim.
int dcpp_batch_random(uint64_t seed, int64_t max_seq_len, int max_seqs, int max_heads,
                      int head_dim, dcpp_batch** out) {
  try {
    std::mt19937_64 rng(seed);
    auto b = std::make_unique<dcpp_batch>();
    b->batch = fixtures::random_batch(rng, max_seq_len, max_seqs, max_heads, 8);
    b->batch.head_dim = head_dim;
    b->batch.validate();
    *out = b.release();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int dcpp_batch_num_seqs(const dcpp_batch* b) { return static_cast<int>(b->batch.sequences.size()); }
void dcpp_batch_seq(const dcpp_batch* b, int i, SeqSpecC* out) {
  mask_to_c(b->batch.sequences[static_cast<size_t>(i)], *out);
}
void dcpp_batch_shape(const dcpp_batch* b, int32_t* out4) {
  out4[0] = b->batch.heads; out4[1] = b->batch.kv_groups; out4[2] = b->batch.head_dim;
  out4[3] = b->batch.bytes_per_element;
}
double dcpp_batch_sparsity(const dcpp_batch* b) { return dcp::mask_sparsity(b->batch); }
void dcpp_batch_free(dcpp_batch* b) { delete b; }

// Planning -------------------------------------------------------------------------------
// placement: 0 = DCP planner (place), 1 = ring, 2 = zigzag, 3 = explicit (group_dev/comp_dev)
int dcpp_plan(const dcpp_batch* b, const CfgC* cfg, int placement, const int32_t* group_dev,
              const int32_t* comp_dev, dcpp_planned** out) {
  try {
    auto p = std::make_unique<dcpp_planned>();
    const dcp::DeviceTopology topo = topo_of(*cfg);
    dcp::PlannerConfig pc;
    pc.block_size = cfg->block_size;
    pc.divisions = cfg->divisions;
    pc.placement.eps_inter = cfg->eps_inter;
    pc.placement.eps_intra = cfg->eps_intra;
    pc.placement.eps_data = cfg->eps_data;
    pc.placement.seed = cfg->seed;
    pc.compile.max_slots_per_kind = cfg->max_slots_per_kind;
    if (placement == 0 && cfg->threads == 1) {
      p->pb = dcp::plan_batch(b->batch, topo, pc);  // pipeline.hpp:29-38, unchanged
    } else if (placement == 0) {
      // the same plan, bit for bit, with the partitioner's candidates and repair scans on
      // host threads (planner/dcp_partition_parallel.hpp)
      p->pb = dcpx_planner::plan_batch_parallel(b->batch, topo, pc, cfg->threads);
    } else {
      auto& pb = p->pb;
      pb.graph = dcp::generate_blocks(b->batch, pc.block_size);
      if (placement == 1) pb.placement = dcp::ring_placement(pb.graph, topo);
      else if (placement == 2) pb.placement = dcp::zigzag_placement(pb.graph, topo);
      else {
        std::vector<int> gd(group_dev, group_dev + pb.graph.groups.size());
        std::vector<int> cd(comp_dev, comp_dev + pb.graph.comp_blocks.size());
        pb.placement = dcp::detail::make_placement(pb.graph, topo, gd, cd);
      }
      pb.schedule = dcp::schedule(pb.graph, pb.placement, pc.divisions);
      pb.plans = dcp::compile_plans(pb.schedule, pb.graph, pb.placement, pc.compile);
      pb.volume = dcp::communication_volume(pb.graph, pb.placement);
    }
    if (cfg->verify) dcp::verify_plans(p->pb.plans, p->pb.graph);
    flatten(*p);
    *out = p.release();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Number of groups / comp blocks of the graph a batch would produce (for explicit
// placements chosen by the caller).
int dcpp_graph_counts(const dcpp_batch* b, int64_t block_size, int32_t* groups, int32_t* comps,
                      int32_t* out_group_tile, int32_t* out_comp_qtile, int max_out) {
  try {
    const auto g = dcp::generate_blocks(b->batch, block_size);
    *groups = static_cast<int32_t>(g.groups.size());
    *comps = static_cast<int32_t>(g.comp_blocks.size());
    if (out_group_tile && static_cast<int>(g.groups.size()) <= max_out)
      for (const auto& grp : g.groups) out_group_tile[grp.id] = grp.tile;
    if (out_comp_qtile && static_cast<int>(g.comp_blocks.size()) <= max_out)
      for (const auto& c : g.comp_blocks) out_comp_qtile[c.id] = c.q_tile;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

void dcpp_plan_free(dcpp_planned* p) { delete p; }

// Generic accessor: returns a pointer to a flat array and its byte size.
// Graph-level names (device ignored): header, seq_lengths, block_sizes, seq_offsets,
// ranges, data_blocks, comp_blocks, data_block_device, comp_block_device, dev_flops,
// per_device_send, per_device_recv, volume.
// Device-level names: capacity, resident_q, resident_kv, resident_o, instr, items,
// srcs, copies, blocks, tags, meta.
int dcpp_array(dcpp_planned* p, const char* name, int device, const void** ptr, int64_t* nbytes) {
  const std::string n(name);
#define RET(vec)                                                 \
  do {                                                           \
    *ptr = (vec).data();                                         \
    *nbytes = static_cast<int64_t>((vec).size() * sizeof((vec)[0])); \
    return 0;                                                    \
  } while (0)
  if (n == "header") RET(p->header);
  if (n == "seq_lengths") RET(p->seq_lengths);
  if (n == "block_sizes") RET(p->block_sizes);
  if (n == "seq_offsets") RET(p->seq_offsets);
  if (n == "ranges") RET(p->ranges);
  if (n == "data_blocks") RET(p->data_blocks);
  if (n == "comp_blocks") RET(p->comp_blocks);
  if (n == "data_block_device") RET(p->data_block_device);
  if (n == "comp_block_device") RET(p->comp_block_device);
  if (n == "dev_flops") RET(p->dev_flops);
  if (n == "per_device_send") RET(p->per_device_send);
  if (n == "per_device_recv") RET(p->per_device_recv);
  if (n == "volume") RET(p->volume);
  if (device < 0 || device >= static_cast<int>(p->devs.size())) {
    g_err = "dcpp_array: bad device";
    return DCPX_ERROR;
  }
  auto& f = p->devs[static_cast<size_t>(device)];
  if (n == "capacity") {
    *ptr = f.capacity;
    *nbytes = sizeof(f.capacity);
    return 0;
  }
  if (n == "resident_q") RET(f.res_q);
  if (n == "resident_kv") RET(f.res_kv);
  if (n == "resident_o") RET(f.res_o);
  if (n == "instr") RET(f.instr);
  if (n == "items") RET(f.items);
  if (n == "srcs") RET(f.srcs);
  if (n == "copies") RET(f.copies);
  if (n == "blocks") RET(f.blocks);
  if (n == "tags") {
    *ptr = f.tag_blob.data();
    *nbytes = static_cast<int64_t>(f.tag_blob.size());
    return 0;
  }
#undef RET
  g_err = "dcpp_array: unknown array " + n;
  return DCPX_ERROR;
}

// Writes the planned batch in the reference's own file formats, with the reference's own
// writers: batch.jsonl (write_sequences_jsonl, io.hpp:72-88), graph.json
// (block_graph_to_json, :135-174), placement.json (placement_to_json, :183-216) and
// plan_d<d>.json (plan_to_json, :271-350). DCPX_UNSUPPORTED when built without json.hpp.
int dcpp_dump_json(const dcpp_planned* p, const dcpp_batch* b, const char* dir) {
#ifdef DCPP_HAVE_JSON
  try {
    namespace fs = std::filesystem;
    fs::create_directories(dir);
    const fs::path d(dir);
    dcp::BatchHeader h;
    h.heads = b->batch.heads;
    h.kv_groups = b->batch.kv_groups;
    h.head_dim = b->batch.head_dim;
    h.token_budget = b->batch.token_budget;
    h.bytes_per_element = b->batch.bytes_per_element;
    std::ostringstream os;
    dcp::write_sequences_jsonl(os, h, b->batch.sequences);
    dcp::write_file((d / "batch.jsonl").string(), os.str());
    dcp::write_file((d / "graph.json").string(), dcp::block_graph_to_json(p->pb.graph).dump(1));
    dcp::write_file((d / "placement.json").string(),
                    dcp::placement_to_json(p->pb.graph, p->pb.placement).dump(1));
    for (size_t i = 0; i < p->pb.plans.size(); ++i)
      dcp::write_file((d / ("plan_d" + std::to_string(i) + ".json")).string(),
                      dcp::plan_to_json(p->pb.plans[i]).dump(1));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
#else
  (void)p;
  (void)b;
  (void)dir;
  g_err = "dcpp_dump_json: planner shim built without json.hpp";
  return DCPX_UNSUPPORTED;
#endif
}

}  // extern "C"

// compile.cu — per-device program compilation of the B200 DCP executor (see executor.cu):
// the instruction stream of one plan device -> fused attention units (forward FwdUnit /
// FwdStep lists, backward BwdUnit / BwdStep lists, masks classified per tile), merge
// batches, copy remaps, O-slot compaction, arenas and tensor maps, and the row-copy jobs
// of inputs, outputs and LOCAL transfers (forward and backward).
#include <cuda_bf16.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <tuple>
#include <numeric>
#include <set>
#include <utility>

#include "executor.h"

namespace dcpx {

namespace {

struct RelRange {
  int32_t b0, e0, b1, e1;  // kv-tile-relative, already intersected with [0, n_k)
};

}  // namespace

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
  D.bwd_units = D.bwd_windowed = 0;

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
        groups.push_back(std::move(grp));
        fused_red[r] = true;
      }
    }
    for (int k = 0; k < I.count; ++k) {
      const int idx = static_cast<int>(I.offset) + k;
      if (covered.count(idx)) continue;
      AttnGroup grp;
      grp.items = {idx};
      grp.target = P.items[idx].out_slot;
      groups.push_back(std::move(grp));
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
    // per-rank mode: a peer's arenas are mapped from its process at connect(); until then
    // a placeholder (its tensor maps are never used here)
    const bool own = local(d);
    auto arena = [&](int64_t bytes) { return alloc(d, own ? static_cast<size_t>(bytes) : 256); };
    auto zero = [&](void* p, int64_t bytes) { if (own) CUDA_OK(cudaMemset(p, 0, bytes)); };
    D.q = static_cast<__nv_bfloat16*>(arena(std::max<int64_t>(1, D.cap_q) * SR * 256));
    D.kv = static_cast<__nv_bfloat16*>(arena(std::max<int64_t>(1, D.cap_kv) * 2 * SR * 256));
    D.o = static_cast<__nv_bfloat16*>(arena(std::max<int64_t>(1, D.cap_o) * SR * 256));
    D.lse = static_cast<float*>(arena(std::max<int64_t>(1, D.cap_o) * SR * 4));
    zero(D.q, std::max<int64_t>(1, D.cap_q) * SR * 256);
    zero(D.kv, std::max<int64_t>(1, D.cap_kv) * 2 * SR * 256);
    zero(D.o, std::max<int64_t>(1, D.cap_o) * SR * 256);
    zero(D.lse, std::max<int64_t>(1, D.cap_o) * SR * 4);
    D.sched_ctr = static_cast<uint32_t*>(alloc(d, 256));
    if (own) CUDA_OK(cudaMemset(D.sched_ctr, 0, 256));
    D.sched_base = 0;
    // backward arenas, parallel to the Q arena (dO, LSE*log2e, Delta, dQ accumulator)
    // and to the KV arena (dK / dV accumulators)
    const int64_t nq = std::max<int64_t>(1, D.cap_q), nkv = std::max<int64_t>(1, D.cap_kv);
    D.d_o = static_cast<__nv_bfloat16*>(arena(nq * SR * 256));
    D.lse2 = static_cast<float*>(arena(nq * SR * 4));
    D.delta = static_cast<float*>(arena(nq * SR * 4));
    D.dq_acc = static_cast<float*>(arena(nq * SR * 512));
    D.dkv_acc = static_cast<float*>(arena(nkv * 2 * SR * 512));
    zero(D.d_o, nq * SR * 256);
    zero(D.lse2, nq * SR * 4);
    zero(D.delta, nq * SR * 4);
    zero(D.dq_acc, nq * SR * 512);     // every backward leaves them zeroed for the next one
    zero(D.dkv_acc, nkv * 2 * SR * 512);
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
        std::vector<int> unit_oblock;  // output block of each unit (persistent-launch checks)
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
            U.flags = (grp.merge_prev ? 1 : 0) | (std::min(I.division, 255) << 8);
            U.q_local0 = 256 * pr;
            U.dep = -1;
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
            unit_oblock.push_back(g_.comp_blocks[P.items[grp.items[0]].comp_id].o_block);
          }
        }
        // longest-processing-time-first order (the kernels take units in list order from a
        // dynamic scheduler, so the longest start first)
        std::vector<size_t> order(units.size());
        std::iota(order.begin(), order.end(), 0);
        std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return unit_cost[a] > unit_cost[b]; });
        std::vector<FwdUnit> sorted;
        for (size_t k : order) sorted.push_back(units[k]);
        op.units = upload(d, sorted);
        op.steps = upload(d, steps);
        op.items = upload(d, masks);
        op.num_units = static_cast<int>(sorted.size());
        op.h_units = sorted;
        op.h_steps = steps;
        op.h_items = masks;
        for (size_t k : order) op.h_unit_oblock.push_back(unit_oblock[k]);
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
            auto close = [&]() {
              U.step_count = static_cast<int32_t>(bsteps.size()) - U.step_begin;
              if (U.step_count > 0) {
                bunits.push_back(U);
                bcost.push_back(U.step_count);
                bkey.emplace_back(bsteps[U.step_begin].q_row0, U.kv_row0);
              }
              U.step_begin = static_cast<int32_t>(bsteps.size());
            };
            // (item, q tile) steps of this sub-tile grouped into windows. With
            // bwd_merge_heads the items of one q block (the GQA group's heads, same tokens)
            // share their windows, so a unit streams win q tiles of every head: 4x longer
            // units (fewer K/V reloads and dK/dV epilogues) with the same q-row locality.
            std::map<std::tuple<int64_t, int64_t, int64_t, int64_t>, std::vector<std::pair<int, int>>> windows;
            std::vector<std::tuple<int64_t, int64_t, int64_t, int64_t>> window_order;
            for (int idx : idxs) {
              const auto& it = P.items[idx];
              if (it.kv_end - it.kv_begin != n_k) throw Failure(DCPX_ERROR, "kv slot read with two sizes in one instruction");
              const auto& c = icl.at(idx);
              for (int qt = 0; qt < c.n_qb; ++qt) {
                if (!c.cls_b[qt * c.nks + ks]) continue;
                const auto key = opt.bwd_merge_heads ? std::make_tuple(int64_t{it.seq}, it.q_begin, it.q_end, int64_t{qt / win})
                                                     : std::make_tuple(int64_t{idx}, int64_t{0}, int64_t{0}, int64_t{qt / win});
                auto& w = windows[key];
                if (w.empty()) window_order.push_back(key);
                w.emplace_back(idx, qt);
              }
            }
            for (const auto& key : window_order) {
              for (const auto& [idx, qt] : windows[key]) {
                const auto& it = P.items[idx];
                const auto& c = icl.at(idx);
                const int n_q = static_cast<int>(it.q_end - it.q_begin);
                const uint32_t cl = c.cls_b[qt * c.nks + ks];
                BwdStep S{};
                S.q_row0 = static_cast<int32_t>(it.q_slot * SR + kBwdQRows * qt);
                S.n_q = std::min(kBwdQRows, n_q - kBwdQRows * qt);
                S.item = c.mask;
                S.q_local0 = kBwdQRows * qt;
                S.col0 = 128 * ks;
                S.cls = cl;
                bsteps.push_back(S);
              }
              close();
            }
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
        D.bwd_units += op.bnum_units;
        D.bwd_windowed += windowed ? 1 : 0;
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

// Persistent cross-division forward for plan device d (multi-device plans): all attention
// instructions' units concatenated in division order into one launch. The kernel then needs
// device-side ordering instead of launch boundaries: units of division t wait for the
// transfers of division t (rdy), a unit merging into an earlier division's output waits for
// that unit's epilogue (dep / unit_done), and a receive waits for the units of the divisions
// whose attention precedes its launch in program order (done), i.e. those that read the
// slots it overwrites. Eligible when nothing but transfers
// sit between the attention instructions (no unfused merge or copy) and every physical O slot
// keeps one output block for the whole forward.
void Executor::build_persistent_fwd(int d) {
  DevState& D = dev_[d];
  D.pfwd = false;
  D.pf_first = -1;
  if (!opt.persistent || R_ < 2 || transport_ != DCPX_TRANSPORT_LOCAL) return;
  // The launch spins on transfers that run on the SMs it leaves free; plan devices sharing a
  // GPU would fill those SMs with each other's persistent CTAs (one process) or only run
  // between time slices (ranks in separate processes), so a single-GPU emulation of a
  // multi-device plan keeps one launch per division.
  if (rank_ < 0) {
    for (int e = 0; e < R_; ++e)
      if (e != d && dev_[e].ordinal == D.ordinal) return;
  } else {
    int n = 0;
    CUDA_OK(cudaGetDeviceCount(&n));
    if (n < R_) return;
  }
  const int T = plans_[d].divisions;
  if (T + 1 > 255) return;
  std::vector<int> attn;
  for (size_t i = 0; i < D.prog.size(); ++i)
    if (D.prog[i].kind == OpKind::kFwdAttn && D.prog[i].num_units > 0) attn.push_back(static_cast<int>(i));
  if (attn.size() < 2) return;
  for (int i = attn.front(); i <= attn.back(); ++i) {
    const Op& op = D.prog[i];
    if (op.kind == OpKind::kMerge || op.kind == OpKind::kCopy) return;
    if (op.kind == OpKind::kCommLaunch && op.send && !op.resident_only) return;
    if (op.kind == OpKind::kFwdAttn && op.division >= T) return;
  }
  std::vector<FwdUnit> units;
  std::vector<FwdStep> steps;
  std::vector<ItemMask> items;
  std::map<int32_t, int> last_writer;  // out_row0 -> unit
  std::map<int64_t, int> slot_block;   // physical O slot -> output block
  std::vector<uint32_t> done_target(static_cast<size_t>(T) + 1, 0);
  for (int i : attn) {
    const Op& op = D.prog[i];
    const int32_t s0 = static_cast<int32_t>(steps.size()), m0 = static_cast<int32_t>(items.size());
    for (size_t k = 0; k < op.h_units.size(); ++k) {
      FwdUnit U = op.h_units[k];
      U.step_begin += s0;
      const int slot = static_cast<int>(U.out_row0 / D.slot_rows);
      auto [sb, fresh] = slot_block.try_emplace(slot, op.h_unit_oblock[k]);
      if (!fresh && sb->second != op.h_unit_oblock[k]) return;  // O slot reused by another output
      auto lw = last_writer.find(U.out_row0);
      if (U.flags & 1) {
        if (lw == last_writer.end()) return;  // merges with a value no unit of this launch wrote
        if (units[static_cast<size_t>(lw->second)].n_rows != U.n_rows) return;  // per-tile stamps
        U.dep = lw->second;
      } else if (lw != last_writer.end()) {
        return;  // overwrites an earlier unit's output unordered
      }
      last_writer[U.out_row0] = static_cast<int>(units.size());
      done_target[static_cast<size_t>(op.division)] += U.n_rows > kTileRows ? 2 : 1;
      units.push_back(U);
    }
    for (FwdStep S : op.h_steps) {
      S.item += m0;
      steps.push_back(S);
    }
    items.insert(items.end(), op.h_items.begin(), op.h_items.end());
  }
  // the comm stream runs the transfers in program order (division ascending) and each adds 1
  // to one counter, so "every fetch of divisions <= t landed" is a cumulative count (a
  // division may read blocks fetched for an earlier one and have no transfers of its own)
  std::vector<uint32_t> rdy_target(static_cast<size_t>(T) + 1, 0);
  for (const Op& op : D.prog)
    if (op.kind == OpKind::kCommWait && op.division < T) ++rdy_target[static_cast<size_t>(op.division)];
  // slot reuse: without the persistent launch a receive starts after every attention op that
  // precedes its launch in program order; here it waits for those ops' divisions on the device
  std::map<std::string, int> wait_divs;
  int divs_before = 0;
  for (const Op& op : D.prog) {
    if (op.kind == OpKind::kFwdAttn && op.num_units > 0) divs_before = std::max(divs_before, op.division + 1);
    if (op.kind == OpKind::kCommLaunch && !op.send) wait_divs[op.tag] = divs_before;
  }
  for (Op& op : D.prog)
    if (op.kind == OpKind::kCommWait && op.division < T) {
      const auto w = wait_divs.find(op.tag);
      if (w == wait_divs.end() || w->second > op.division) return;  // (would wait on its own readers)
      op.pf_wait_divs = w->second;
    }
  for (int t = 1; t <= T; ++t) rdy_target[static_cast<size_t>(t)] += rdy_target[static_cast<size_t>(t) - 1];
  D.pf_units = upload(d, units);
  D.pf_steps = upload(d, steps);
  D.pf_items = upload(d, items);
  D.pf_num_units = static_cast<int>(units.size());
  // at least two SMs stay free whatever sm_reserve says: the comm stream's counter / flag
  // kernels the launch spins on need somewhere to run
  D.pf_grid = std::min(D.pf_num_units, num_sms(D.ordinal) - 2);
  D.prdy_target = upload(d, rdy_target);
  D.pdone_target = upload(d, done_target);
  D.pctr = static_cast<uint32_t*>(alloc(d, sizeof(uint32_t) * 2 * (static_cast<size_t>(T) + 1)));
  D.punit_done = static_cast<uint32_t*>(alloc(d, sizeof(uint32_t) * 2 * units.size()));
  if (local(d)) {
    DeviceGuard g(D.ordinal);
    CUDA_OK(cudaMemset(D.punit_done, 0, sizeof(uint32_t) * 2 * units.size()));
  }
  D.pf_first = attn.front();
  D.pfwd = true;
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
  auto tok_ranges = [&](const std::vector<dcpx_block_slot>& res) {
    std::vector<std::pair<int64_t, int64_t>> r;
    for (const auto& x : res) {
      const auto& db = g_.data_blocks[x.block];
      const int64_t off = g_.seq_offsets[db.seq];
      r.push_back({off + db.tok_begin, off + db.tok_end});
    }
    std::sort(r.begin(), r.end());
    std::vector<std::pair<int64_t, int64_t>> m;
    for (const auto& x : r) {
      if (!m.empty() && x.first <= m.back().second) m.back().second = std::max(m.back().second, x.second);
      else m.push_back(x);
    }
    return m;
  };
  D.tok_q = tok_ranges(P.res_q);
  D.tok_kv = tok_ranges(P.res_kv);
  D.tok_o = tok_ranges(P.res_o);
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
  wire_bwd_send_.assign(static_cast<size_t>(R_), 0);
  wire_bwd_recv_.assign(static_cast<size_t>(R_), 0);
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
          const uint64_t out = 2 * db.size_bytes + 8 * static_cast<uint64_t>(rows);     // + fp32 LSE, Delta
          wire_bwd_send_[src_dev] += out; wire_bwd_recv_[d] += out;
          wire_bwd_send_[d] += 2 * db.size_bytes; wire_bwd_recv_[src_dev] += 2 * db.size_bytes;  // fp32 dQ
        } else if (db.kind == DCPX_KIND_KV) {
          for (int h = 0; h < 2; ++h)
            jobs.push_back({reinterpret_cast<const char*>(A.kv + (2 * sb.slot + h) * SR * 128),
                            reinterpret_cast<char*>(D.kv + (2 * rb.slot + h) * SR * 128), 256, 256, rows, 256});
          bwd_send_[src_dev] += db.size_bytes; bwd_recv_[d] += db.size_bytes;  // K, V out
          bwd_send_[d] += db.size_bytes; bwd_recv_[src_dev] += db.size_bytes;  // dK, dV back
          wire_bwd_send_[src_dev] += db.size_bytes; wire_bwd_recv_[d] += db.size_bytes;
          wire_bwd_send_[d] += 2 * db.size_bytes; wire_bwd_recv_[src_dev] += 2 * db.size_bytes;  // fp32 dK, dV
        }
      }
      op.bjobs = make_jobs(d, jobs);
      op.bxfer = jobs;
    }
    // 2. gradient returns of fetched blocks, right after the attention of their last use.
    //    One fetch episode per receive of a block into a slot (a plan may fetch the same
    //    block twice, into different slots or at different divisions): each episode's
    //    accumulator is returned (and zeroed) after its own last use.
    struct Episode { int block, slot, kind; size_t last; bool used; };
    std::vector<Episode> eps;
    std::map<int, int> cur_q, cur_kv;  // slot -> episode
    for (size_t i = 0; i < P.ins.size(); ++i) {
      const Instr& I = P.ins[i];
      if (I.op == DCPX_OP_COMM_LAUNCH && !I.send && I.division < T) {
        for (int b = 0; b < I.count; ++b) {
          const auto tb = P.blocks[I.offset + b];
          const int k = g_.data_blocks[tb.block].kind;
          if (k != DCPX_KIND_Q && k != DCPX_KIND_KV) continue;
          (k == DCPX_KIND_Q ? cur_q : cur_kv)[tb.slot] = static_cast<int>(eps.size());
          eps.push_back({tb.block, tb.slot, k, 0, false});
        }
      } else if (I.op == DCPX_OP_ATTENTION) {
        for (int k = 0; k < I.count; ++k) {
          const auto& it = P.items[I.offset + k];
          for (auto* cur : {&cur_q, &cur_kv}) {
            auto e = cur->find(cur == &cur_q ? it.q_slot : it.kv_slot);
            if (e != cur->end()) {
              eps[e->second].last = i;
              eps[e->second].used = true;
            }
          }
        }
      }
    }
    std::map<size_t, std::vector<RowCopyJob>> ret;
    for (const auto& ep : eps) {
      if (!ep.used) continue;  // never read: its accumulator stays zero
      const auto [o, so] = owner.at(ep.block);
      const auto& db = g_.data_blocks[ep.block];
      const int rows = static_cast<int>(db.tok_end - db.tok_begin);
      if (ep.kind == DCPX_KIND_Q) {
        ret[ep.last].push_back({reinterpret_cast<const char*>(D.dq_acc + ep.slot * SR * 128),
                                reinterpret_cast<char*>(dev_[o].dq_acc + so * SR * 128), 512, 512, rows, 512});
      } else {
        for (int h = 0; h < 2; ++h)
          ret[ep.last].push_back({reinterpret_cast<const char*>(D.dkv_acc + (2 * ep.slot + h) * SR * 128),
                                  reinterpret_cast<char*>(dev_[o].dkv_acc + (2 * so + h) * SR * 128), 512, 512,
                                  rows, 512});
      }
    }
    for (auto& [i, jobs] : ret) D.prog[i].ret = make_jobs(d, jobs);
    // 3. io: Delta/LSE preprocess with the dO scatter to the resident Q slots, gradient gathers
    std::map<std::tuple<int, int, int>, int> qslot_of;  // (seq, head, tile) -> resident Q slot
    for (const auto& r : P.res_q) {
      const auto& db = g_.data_blocks[r.block];
      qslot_of[{db.seq, db.head, db.tile}] = r.slot;
    }
    std::vector<RowJob> prep, gq, gk, gv;
    std::vector<int> prep_rows, gq_rows, gk_rows;
    for (size_t k = 0; k < P.res_o.size(); ++k) {
      const auto& db = g_.data_blocks[P.res_o[k].block];
      auto it = qslot_of.find({db.seq, db.head, db.tile});
      if (it == qslot_of.end()) throw Failure(DCPX_ERROR, "output block without a co-located Q block (blocks.hpp:42-51)");
      const int64_t tok = g_.seq_offsets[db.seq] + db.tok_begin;
      const int rows = static_cast<int>(db.tok_end - db.tok_begin);
      prep.push_back({D.final_o_slot[k] * SR, it->second * SR, (tok * H + db.head) * 128, rows, 0});
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
    D.prep = make_row_jobs(d, prep, prep_rows, 16);
    D.gather_dq = make_row_jobs(d, gq, gq_rows, 16);
    D.gather_dk = make_row_jobs(d, gk, gk_rows, 16);
    D.gather_dv = make_row_jobs(d, gv, gk_rows, 16);
  }
  (void)TT;
}

}  // namespace dcpx

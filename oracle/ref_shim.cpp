// TEST INFRASTRUCTURE ONLY. extern "C" wrapper around the REFERENCE executor so tests
// can pin oracle/dcp_oracle.c against it and bench.py's cpu_baseline / --impl reference
// leg can time it. Built by oracle/Makefile into oracle/_ref/libdcpref.so from the
// unchanged headers under /root/reference/proj/{include,tests} (nothing copied).
//
//   dcpr_plan_run      plan_batch (pipeline.hpp:29-38) + run (simexec.hpp:207-423)
//   dcpr_make_payload  make_payload (simexec.hpp:125-146)
//   dcpr_exec_attention / dcpr_exec_reduction  (simexec.hpp:33-111)
//   dcpr_dense_attention  oracle::dense_attention (tests/oracle.hpp:80-120)
//   dcpr_time_items    exec_attention over a deterministic sample of a plan's
//                      AttentionItems on N host threads (CPU baseline)
#include <atomic>
#include <limits>
#include <chrono>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "dcp/pipeline.hpp"
#include "oracle.hpp"

namespace {

struct SeqSpecC {
  int64_t length;
  int32_t kind;
  int32_t window_blocks, sink_blocks, test_blocks;
  int64_t sink, window, block;
  int64_t question_len;
  int32_t n_answers, _pad;
  int64_t answer_lens[16];
};

struct CfgC {
  int32_t machines, devices_per_machine, divisions, max_slots_per_kind;
  int64_t block_size;
  double eps_inter, eps_intra, eps_data;
  uint64_t seed;
  int32_t verify, _pad;
};

thread_local std::string g_err;

dcp::Batch make_batch(const SeqSpecC* s, int n, int H, int G, int D) {
  dcp::Batch b;
  b.heads = H;
  b.kv_groups = G;
  b.head_dim = D;
  for (int i = 0; i < n; ++i) {
    dcp::SequenceSpec sp;
    sp.seq_id = "s" + std::to_string(i);
    sp.length = s[i].length;
    switch (s[i].kind) {
      case 0: sp.mask = dcp::MaskDescriptor::causal(); break;
      case 1: sp.mask = dcp::MaskDescriptor::lambda(s[i].sink, s[i].window); break;
      case 2:
        sp.mask = dcp::MaskDescriptor::causal_blockwise(s[i].block, s[i].window_blocks,
                                                        s[i].sink_blocks, s[i].test_blocks);
        break;
      default:
        sp.mask = dcp::MaskDescriptor::shared_question(
            s[i].question_len,
            std::vector<dcp::TokenIndex>(s[i].answer_lens, s[i].answer_lens + s[i].n_answers));
    }
    b.sequences.push_back(sp);
  }
  b.token_budget = b.total_tokens();
  return b;
}

dcp::PlannerConfig planner_cfg(const CfgC& c) {
  dcp::PlannerConfig pc;
  pc.block_size = c.block_size;
  pc.divisions = c.divisions;
  pc.placement.eps_inter = c.eps_inter;
  pc.placement.eps_intra = c.eps_intra;
  pc.placement.eps_data = c.eps_data;
  pc.placement.seed = c.seed;
  pc.compile.max_slots_per_kind = c.max_slots_per_kind;
  return pc;
}

dcp::BatchPayload payload_from_packed(const dcp::Batch& b, const double* q, const double* k,
                                      const double* v) {
  const int H = b.heads, G = b.kv_groups, D = b.head_dim;
  dcp::BatchPayload p;
  int64_t off = 0;
  for (const auto& s : b.sequences) {
    dcp::SeqPayload sp;
    const int L = static_cast<int>(s.length);
    for (int h = 0; h < H; ++h) {
      dcp::Matrix m(L, D);
      for (int i = 0; i < L; ++i)
        for (int d = 0; d < D; ++d) m.at(i, d) = q[((off + i) * H + h) * D + d];
      sp.q.push_back(std::move(m));
    }
    for (int gr = 0; gr < G; ++gr) {
      dcp::Matrix mk(L, D), mv(L, D);
      for (int i = 0; i < L; ++i)
        for (int d = 0; d < D; ++d) {
          mk.at(i, d) = k[((off + i) * G + gr) * D + d];
          mv.at(i, d) = v[((off + i) * G + gr) * D + d];
        }
      sp.k.push_back(std::move(mk));
      sp.v.push_back(std::move(mv));
    }
    p.seqs.push_back(std::move(sp));
    off += L;
  }
  return p;
}

int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const dcp::InfeasibleError*>(&e)) return 5;
  if (dynamic_cast<const dcp::BufferOverflowError*>(&e)) return 4;
  if (dynamic_cast<const dcp::TagMismatchError*>(&e)) return 3;
  if (dynamic_cast<const dcp::DeadlockError*>(&e)) return 2;
  return 1;
}

}  // namespace

extern "C" {

const char* dcpr_last_error() { return g_err.c_str(); }

// plan_batch + run in numeric mode. Outputs o [T][H][D]; stats: total_bytes,
// total_flops, per-device send[R], recv[R]; seconds = wall time of run() only.
int dcpr_plan_run(const SeqSpecC* specs, int n, int H, int G, int D, const CfgC* cfg,
                  const double* q, const double* k, const double* v, double* o,
                  uint64_t* stats, double* seconds, double* makespan) {
  try {
    const dcp::Batch b = make_batch(specs, n, H, G, D);
    dcp::DeviceTopology topo;
    topo.machines = cfg->machines;
    topo.devices_per_machine = cfg->devices_per_machine;
    const dcp::PlannedBatch pb = dcp::plan_batch(b, topo, planner_cfg(*cfg));
    dcp::verify_plans(pb.plans, pb.graph);
    const dcp::BatchPayload payload = payload_from_packed(b, q, k, v);
    const auto t0 = std::chrono::steady_clock::now();
    const dcp::SimResult sim = dcp::run(pb.plans, pb.graph, payload, topo, {});
    const auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
    *makespan = sim.report.makespan;
    int64_t off = 0;
    for (size_t s = 0; s < b.sequences.size(); ++s) {
      const int L = static_cast<int>(b.sequences[s].length);
      for (int h = 0; h < H; ++h)
        for (int i = 0; i < L; ++i)
          for (int d = 0; d < D; ++d) o[((off + i) * H + h) * D + d] = sim.outputs.o[s][h].at(i, d);
      off += L;
    }
    const int R = topo.device_count();
    stats[0] = sim.report.total_bytes;
    stats[1] = sim.report.total_flops;
    for (int d = 0; d < R; ++d) {
      stats[2 + d] = sim.report.per_device_send[d];
      stats[2 + R + d] = sim.report.per_device_recv[d];
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// make_payload(batch, seed) in the packed token-major layout.
int dcpr_make_payload(const SeqSpecC* specs, int n, int H, int G, int D, uint64_t seed,
                      double* q, double* k, double* v) {
  try {
    const dcp::Batch b = make_batch(specs, n, H, G, D);
    const dcp::BatchPayload p = dcp::make_payload(b, seed);
    int64_t off = 0;
    for (size_t s = 0; s < b.sequences.size(); ++s) {
      const int L = static_cast<int>(b.sequences[s].length);
      for (int i = 0; i < L; ++i)
        for (int d = 0; d < D; ++d) {
          for (int h = 0; h < H; ++h) q[((off + i) * H + h) * D + d] = p.seqs[s].q[h].at(i, d);
          for (int g = 0; g < G; ++g) {
            k[((off + i) * G + g) * D + d] = p.seqs[s].k[g].at(i, d);
            v[((off + i) * G + g) * D + d] = p.seqs[s].v[g].at(i, d);
          }
        }
      off += L;
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

static dcp::Matrix to_matrix(const double* a, int r, int c) {
  dcp::Matrix m(r, c);
  std::memcpy(m.a.data(), a, sizeof(double) * static_cast<size_t>(r) * c);
  return m;
}

static std::vector<dcp::TokenRanges> to_rows(const int32_t* rows, int nq) {
  std::vector<dcp::TokenRanges> out(static_cast<size_t>(nq));
  for (int i = 0; i < nq; ++i) {
    out[i].push({rows[4 * i], rows[4 * i + 1]});
    out[i].push({rows[4 * i + 2], rows[4 * i + 3]});
  }
  return out;
}

int dcpr_exec_attention(const double* q, const double* k, const double* v, int nq, int nk, int D,
                        const int32_t* rows, double* out, double* m, double* l) {
  try {
    const dcp::PartialBlock p = dcp::exec_attention(to_matrix(q, nq, D), to_matrix(k, nk, D),
                                                    to_matrix(v, nk, D), to_rows(rows, nq));
    std::memcpy(out, p.out.a.data(), sizeof(double) * static_cast<size_t>(nq) * D);
    std::memcpy(m, p.m.data(), sizeof(double) * nq);
    std::memcpy(l, p.l.data(), sizeof(double) * nq);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int dcpr_exec_reduction(int n, const double* const* outs, const double* const* ms,
                        const double* const* ls, int rows, int D, double* out, double* m,
                        double* l) {
  try {
    std::vector<dcp::PartialBlock> parts(static_cast<size_t>(n));
    std::vector<const dcp::PartialBlock*> ptrs;
    for (int i = 0; i < n; ++i) {
      parts[i].out = to_matrix(outs[i], rows, D);
      parts[i].m.assign(ms[i], ms[i] + rows);
      parts[i].l.assign(ls[i], ls[i] + rows);
      ptrs.push_back(&parts[i]);
    }
    const dcp::PartialBlock r = dcp::exec_reduction(ptrs);
    std::memcpy(out, r.out.a.data(), sizeof(double) * static_cast<size_t>(rows) * D);
    std::memcpy(m, r.m.data(), sizeof(double) * rows);
    std::memcpy(l, r.l.data(), sizeof(double) * rows);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int dcpr_dense_attention(const SeqSpecC* specs, int n, int H, int G, int D, const double* q,
                         const double* k, const double* v, double* o) {
  try {
    const dcp::Batch b = make_batch(specs, n, H, G, D);
    const dcp::BatchOutputs out =
        oracle::dense_attention(b, payload_from_packed(b, q, k, v));
    int64_t off = 0;
    for (size_t s = 0; s < b.sequences.size(); ++s) {
      const int L = static_cast<int>(b.sequences[s].length);
      for (int h = 0; h < H; ++h)
        for (int i = 0; i < L; ++i)
          for (int d = 0; d < D; ++d) o[((off + i) * H + h) * D + d] = out.o[s][h].at(i, d);
      off += L;
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// CPU baseline: reference exec_attention (simexec.hpp:33-76) over `count` tiles of
// n_q x n_k with the given rows (relative, [n_q][4]) repeated, on `threads` host
// threads, inputs N(0,1). Returns wall seconds; flops = 4 * pairs * D per tile.
int dcpr_time_tiles(int count, int nq, int nk, int D, const int32_t* rows, int threads,
                    double* seconds) {
  try {
    std::mt19937_64 rng(7);
    std::normal_distribution<double> dist(0.0, 1.0);
    dcp::Matrix q(nq, D), k(nk, D), v(nk, D);
    for (auto* m : {&q, &k, &v})
      for (auto& x : m->a) x = dist(rng);
    const auto rr = to_rows(rows, nq);
    std::atomic<int> next{0};
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
      pool.emplace_back([&] {
        while (next.fetch_add(1) < count) {
          volatile double sink = dcp::exec_attention(q, k, v, rr).out.a[0];
          (void)sink;
        }
      });
    for (auto& th : pool) th.join();
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// CPU baseline over a sample of real AttentionItems: item i has nq[i] x nk[i] tiles and
// rows at rows + 4 * row_off[i] (kv-tile-relative, as compile_plans builds them).
// exec_attention (simexec.hpp:33-76) runs on `threads` host threads, inputs N(0,1).
int dcpr_time_items(int n, const int32_t* nq, const int32_t* nk, const int64_t* row_off,
                    const int32_t* rows, int D, int threads, double* seconds) {
  try {
    int maxq = 1, maxk = 1;
    for (int i = 0; i < n; ++i) { maxq = std::max(maxq, nq[i]); maxk = std::max(maxk, nk[i]); }
    std::mt19937_64 rng(7);
    std::normal_distribution<double> dist(0.0, 1.0);
    dcp::Matrix q(maxq, D), k(maxk, D), v(maxk, D);
    for (auto* m : {&q, &k, &v})
      for (auto& x : m->a) x = dist(rng);
    std::vector<dcp::Matrix> qs, ks, vs;
    std::vector<std::vector<dcp::TokenRanges>> rr;
    for (int i = 0; i < n; ++i) {
      dcp::Matrix a(nq[i], D), b(nk[i], D), c(nk[i], D);
      std::copy(q.a.begin(), q.a.begin() + static_cast<size_t>(nq[i]) * D, a.a.begin());
      std::copy(k.a.begin(), k.a.begin() + static_cast<size_t>(nk[i]) * D, b.a.begin());
      std::copy(v.a.begin(), v.a.begin() + static_cast<size_t>(nk[i]) * D, c.a.begin());
      qs.push_back(std::move(a)); ks.push_back(std::move(b)); vs.push_back(std::move(c));
      rr.push_back(to_rows(rows + 4 * row_off[i], nq[i]));
    }
    std::atomic<int> next{0};
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
      pool.emplace_back([&] {
        int i;
        while ((i = next.fetch_add(1)) < n) {
          volatile double sink = dcp::exec_attention(qs[i], ks[i], vs[i], rr[i]).out.a[0];
          (void)sink;
        }
      });
    for (auto& th : pool) th.join();
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// CPU baseline with outputs: the same as dcpr_time_items, but on the caller's inputs (item i
// reads nq[i] x D rows of q at q + D * in_off_q[i], nk[i] x D rows of k and v at
// k / v + D * in_off_k[i]) and returning item i's (out, LSE = m + ln l; -inf where l = 0) at
// out + D * out_off[i] / lse + out_off[i], so the timed sample can be checked against the GPU.
int dcpr_run_items(int n, const int32_t* nq, const int32_t* nk, const int64_t* row_off, const int32_t* rows,
                   int D, const double* q, const double* k, const double* v, const int64_t* in_off_q,
                   const int64_t* in_off_k, const int64_t* out_off, double* out, double* lse, int threads,
                   double* seconds) {
  try {
    std::vector<dcp::Matrix> qs, ks, vs;
    std::vector<std::vector<dcp::TokenRanges>> rr;
    for (int i = 0; i < n; ++i) {
      qs.push_back(to_matrix(q + D * in_off_q[i], nq[i], D));
      ks.push_back(to_matrix(k + D * in_off_k[i], nk[i], D));
      vs.push_back(to_matrix(v + D * in_off_k[i], nk[i], D));
      rr.push_back(to_rows(rows + 4 * row_off[i], nq[i]));
    }
    std::vector<dcp::PartialBlock> res(static_cast<size_t>(n));
    std::atomic<int> next{0};
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
      pool.emplace_back([&] {
        int i;
        while ((i = next.fetch_add(1)) < n) res[static_cast<size_t>(i)] = dcp::exec_attention(qs[i], ks[i], vs[i], rr[i]);
      });
    for (auto& th : pool) th.join();
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (int i = 0; i < n; ++i) {
      const auto& p = res[static_cast<size_t>(i)];
      std::memcpy(out + D * out_off[i], p.out.a.data(), sizeof(double) * static_cast<size_t>(nq[i]) * D);
      for (int r = 0; r < nq[i]; ++r)
        lse[out_off[i] + r] = p.l[r] > 0 ? p.m[r] + std::log(p.l[r]) : -std::numeric_limits<double>::infinity();
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

}  // extern "C"

// dcp_partition_parallel.hpp — multi-threaded DCP placement with output bit-identical to the
// reference's single-threaded planner (planner throughput).
//
// The reference partitioner, partition_heuristic (hypergraph.hpp:623-784), builds a list of
// candidate initial placements and then, one candidate at a time, repairs it to the balance
// caps (detail::repair, :398-455), refines it (fm_pass / greedy_pass) and keeps the cheapest
// (ties: lexicographically smallest assignment, :772-777). Each candidate's repair and
// refinement depend only on that candidate, so here they run on a pool of host threads,
// each with its own EdgeCounts, and the winner is picked afterwards by the same rule in the
// same candidate order: the result is the reference's. repair -- a best-move scan over every
// (vertex, part) per step, quadratic in the graph and the bulk of planning time on large
// batches -- is replaced by repair_fast, which makes the same move at every step from
// per-weight-class reductions and cached connectivity deltas.
//
// Everything else is the reference's own code, called unchanged from the headers:
// detail::lpt_assign / components / coarsen / fm_pass / greedy_pass / EdgeCounts,
// generate_blocks, schedule, compile_plans, communication_volume.
#pragma once

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <functional>
#include <map>
#include <thread>

#include "dcp/pipeline.hpp"

namespace dcpx_planner {

// Runs fn(i) for i in [0, n) on up to `threads` host threads (the caller's included).
inline void parallel_for(int n, int threads, const std::function<void(int)>& fn) {
  threads = std::max(1, std::min(threads, n));
  if (threads == 1) {
    for (int i = 0; i < n; ++i) fn(i);
    return;
  }
  std::atomic<int> next{0};
  auto worker = [&] {
    for (int i; (i = next.fetch_add(1)) < n;) fn(i);
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();
}

inline int default_threads() {
  const unsigned hc = std::thread::hardware_concurrency();
  return hc ? static_cast<int>(hc) : 1;
}

// detail::repair (hypergraph.hpp:398-455), the same sequence of moves without the full scan.
// The reference evaluates every (vertex in an over-cap part, target part) each step and keeps
// the largest overflow reduction, then the smallest connectivity delta, then the first in
// (vertex, part) scan order. A move's reduction depends only on (from, to, the vertex's
// Weight2D), so it is computed once per (from, weight class, to) -- with the reference's
// expression, hence the same long double value. Per (from, class, to) a min-heap orders the
// class's vertices in `from` by (delta, vertex); a vertex's entries are refreshed only when a
// move touched one of its hyperedges (the only way move_delta's inputs, the per-edge part
// counts, change) or it moved, older entries being discarded lazily. The winner, the
// lexicographic minimum of (delta, vertex, part) over the heap tops of the maximal-reduction
// (from, class, to), is exactly the reference's choice.
inline bool repair_fast(const dcp::Hypergraph& h, std::vector<int>& assignment, int parts,
                        const dcp::detail::BalanceCaps& caps, dcp::detail::EdgeCounts& counts,
                        std::vector<dcp::Weight2D>& loads) {
  using dcp::Weight2D;
  auto overflow = [&](const Weight2D& w) -> long double {
    long double f = 0;
    if (static_cast<long double>(w.flops) > caps.flops_cap && caps.flops_cap > 0)
      f += (static_cast<long double>(w.flops) - caps.flops_cap) / caps.flops_cap;
    if (static_cast<long double>(w.bytes) > caps.bytes_cap && caps.bytes_cap > 0)
      f += (static_cast<long double>(w.bytes) - caps.bytes_cap) / caps.bytes_cap;
    return f;
  };
  auto total_overflow = [&] {
    long double f = 0;
    for (const auto& w : loads) f += overflow(w);
    return f;
  };
  const int n = h.vertex_count();
  // weight classes; vertices per (part, class)
  std::map<std::pair<uint64_t, uint64_t>, int> class_id;
  std::vector<int> cls(static_cast<size_t>(n));
  std::vector<Weight2D> cw;
  for (int v = 0; v < n; ++v) {
    const auto& w = h.weights[static_cast<size_t>(v)];
    auto [it, fresh] = class_id.try_emplace({w.flops, w.bytes}, static_cast<int>(cw.size()));
    if (fresh) cw.push_back(w);
    cls[static_cast<size_t>(v)] = it->second;
  }
  const int nc = static_cast<int>(cw.size());
  std::vector<int> count(static_cast<size_t>(parts) * nc, 0);
  for (int v = 0; v < n; ++v) ++count[static_cast<size_t>(assignment[static_cast<size_t>(v)]) * nc + cls[static_cast<size_t>(v)]];
  struct Entry {
    long long delta;
    int v;
    uint32_t stamp;
  };
  auto later = [](const Entry& a, const Entry& b) { return a.delta != b.delta ? a.delta > b.delta : a.v > b.v; };
  std::vector<std::vector<Entry>> heap(static_cast<size_t>(parts) * nc * parts);
  auto heap_of = [&](int from, int c, int to) -> std::vector<Entry>& {
    return heap[(static_cast<size_t>(from) * nc + c) * parts + to];
  };
  // per (vertex, part): the cached delta and the stamp of its live heap entry
  std::vector<uint32_t> stamp(static_cast<size_t>(n) * parts, 0);
  std::vector<long long> cached(static_cast<size_t>(n) * parts, 0);
  auto refresh = [&](int v, bool moved) {  // v's current deltas into the heaps of its (part, class)
    const int from = assignment[static_cast<size_t>(v)], c = cls[static_cast<size_t>(v)];
    for (int to = 0; to < parts; ++to) {
      const size_t k = static_cast<size_t>(v) * parts + to;
      if (to == from) {
        ++stamp[k];  // no move to its own part (and its old entries, if any, are dead)
        continue;
      }
      const long long d = counts.move_delta(v, from, to);
      if (!moved && d == cached[k]) continue;  // the live entry is still exact
      cached[k] = d;
      const uint32_t st = ++stamp[k];
      auto& hp = heap_of(from, c, to);
      hp.push_back({d, v, st});
      std::push_heap(hp.begin(), hp.end(), later);
      if (hp.size() > 4 * static_cast<size_t>(count[static_cast<size_t>(from) * nc + c]) + 64) {  // drop stale entries
        hp.erase(std::remove_if(hp.begin(), hp.end(),
                                [&](const Entry& e) { return e.stamp != stamp[static_cast<size_t>(e.v) * parts + to]; }),
                 hp.end());
        std::make_heap(hp.begin(), hp.end(), later);
      }
    }
  };
  std::vector<std::vector<int>> incident(static_cast<size_t>(n));
  for (size_t e = 0; e < h.edges.size(); ++e)
    for (int v : h.edges[e].members) incident[static_cast<size_t>(v)].push_back(static_cast<int>(e));
  for (int v = 0; v < n; ++v) refresh(v, true);

  long double current = total_overflow();
  int guard = 4 * n * parts + 16;
  struct Combo { int from, c, to; };
  std::vector<Combo> top;
  std::vector<long double> part_over(static_cast<size_t>(parts));
  std::vector<int> touched;
  std::vector<char> mark(static_cast<size_t>(n), 0);
  size_t steps_ = 0, touched_ = 0, topn_ = 0;
  while (current > 0 && guard-- > 0) {
    ++steps_;
    for (int p = 0; p < parts; ++p) part_over[static_cast<size_t>(p)] = overflow(loads[static_cast<size_t>(p)]);
    long double best_red = 0;
    top.clear();
    for (int from = 0; from < parts; ++from) {
      if (part_over[static_cast<size_t>(from)] == 0) continue;
      for (int c = 0; c < nc; ++c) {
        if (!count[static_cast<size_t>(from) * nc + c]) continue;
        for (int to = 0; to < parts; ++to) {
          if (to == from) continue;
          Weight2D wf = loads[static_cast<size_t>(from)];
          wf -= cw[static_cast<size_t>(c)];
          Weight2D wt = loads[static_cast<size_t>(to)];
          wt += cw[static_cast<size_t>(c)];
          const long double red = part_over[static_cast<size_t>(from)] + part_over[static_cast<size_t>(to)] -
                                  overflow(wf) - overflow(wt);
          if (red <= 0 || red < best_red) continue;
          if (red > best_red) {
            best_red = red;
            top.clear();
          }
          top.push_back({from, c, to});
        }
      }
    }
    if (top.empty()) return false;
    long long bd = std::numeric_limits<long long>::max();
    int bv = -1, bt = -1;
    for (const Combo& k : top) {
      auto& hp = heap_of(k.from, k.c, k.to);
      while (!hp.empty() && hp.front().stamp != stamp[static_cast<size_t>(hp.front().v) * parts + k.to]) {
        std::pop_heap(hp.begin(), hp.end(), later);
        hp.pop_back();
      }
      const Entry& e = hp.front();  // non-empty: the class has members in `from`
      if (e.delta < bd || (e.delta == bd && (e.v < bv || (e.v == bv && k.to < bt)))) {
        bd = e.delta;
        bv = e.v;
        bt = k.to;
      }
    }
    const int from = assignment[static_cast<size_t>(bv)];
    counts.apply_move(bv, from, bt);
    loads[static_cast<size_t>(from)] -= h.weights[static_cast<size_t>(bv)];
    loads[static_cast<size_t>(bt)] += h.weights[static_cast<size_t>(bv)];
    assignment[static_cast<size_t>(bv)] = bt;
    --count[static_cast<size_t>(from) * nc + cls[static_cast<size_t>(bv)]];
    ++count[static_cast<size_t>(bt) * nc + cls[static_cast<size_t>(bv)]];
    touched.clear();
    touched.push_back(bv);
    mark[static_cast<size_t>(bv)] = 1;
    for (int e : incident[static_cast<size_t>(bv)])
      for (int u : h.edges[static_cast<size_t>(e)].members)
        if (!mark[static_cast<size_t>(u)]) {
          mark[static_cast<size_t>(u)] = 1;
          touched.push_back(u);
        }
    touched_ += touched.size(); topn_ += top.size();
    for (int u : touched) {
      mark[static_cast<size_t>(u)] = 0;
      refresh(u, u == bv);
    }
    current -= best_red;
    current = std::max<long double>(current, 0);
    if (current == 0) current = total_overflow();  // re-derived exactly as the reference does
  }
  if (std::getenv("DCPX_PLANNER_PROFILE")) std::fprintf(stderr, "[repair] n=%d classes=%d steps=%zu touched/step=%.1f top/step=%.1f\n", n, nc, steps_, steps_ ? double(touched_) / steps_ : 0., steps_ ? double(topn_) / steps_ : 0.);
  return current == 0;
}

// The candidate initial placements of partition_heuristic, in its order (hypergraph.hpp:
// round-robin :650-655, weight-chunked :656-672, LPT :674, component packing :676-711,
// multilevel :713-735, seeded random restarts :737-745, hint :746-752).
inline std::vector<std::vector<int>> partition_candidates(const dcp::Hypergraph& h, int parts, double eps_comp,
                                                          double eps_data, std::uint64_t seed,
                                                          const dcp::PartitionOptions& options,
                                                          const dcp::detail::BalanceCaps& caps) {
  using namespace dcp;
  const int n = h.vertex_count();
  const Weight2D total = h.total_weight();
  auto share = [&](const Weight2D& w) {  // dominant normalised weight
    const long double f = total.flops ? static_cast<long double>(w.flops) / total.flops : 0;
    const long double b = total.bytes ? static_cast<long double>(w.bytes) / total.bytes : 0;
    return std::make_pair(f, b);
  };
  std::vector<std::vector<int>> out;
  std::vector<int> a(static_cast<size_t>(n));
  for (int v = 0; v < n; ++v) a[static_cast<size_t>(v)] = v % parts;
  out.push_back(a);
  {
    long double acc = 0;
    const long double whole = (total.flops ? 1.0L : 0.0L) + (total.bytes ? 1.0L : 0.0L);
    for (int v = 0; v < n; ++v) {
      const int p = whole > 0 ? static_cast<int>(acc / whole * parts) : 0;
      a[static_cast<size_t>(v)] = std::min(p, parts - 1);
      const auto [f, b] = share(h.weights[static_cast<size_t>(v)]);
      if (total.flops) acc += f;
      if (total.bytes) acc += b;
    }
    out.push_back(a);
  }
  out.push_back(detail::lpt_assign(h, detail::VertexOrder::by_weight_desc(h), parts, caps));
  {
    const auto comp = detail::components(h);
    const int ncomp = 1 + *std::max_element(comp.begin(), comp.end());
    std::vector<Weight2D> cw(static_cast<size_t>(ncomp));
    for (int v = 0; v < n; ++v) cw[static_cast<size_t>(comp[static_cast<size_t>(v)])] += h.weights[static_cast<size_t>(v)];
    std::vector<int> order(static_cast<size_t>(ncomp));
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
      const auto [fx, bx] = share(cw[static_cast<size_t>(x)]);
      const auto [fy, by] = share(cw[static_cast<size_t>(y)]);
      return std::max(fx, bx) > std::max(fy, by);
    });
    std::vector<Weight2D> load(static_cast<size_t>(parts));
    std::vector<int> part_of(static_cast<size_t>(ncomp), 0);
    for (int c : order) {
      int best = 0;
      long double best_key = std::numeric_limits<long double>::max();
      for (int p = 0; p < parts; ++p) {
        Weight2D w = load[static_cast<size_t>(p)];
        w += cw[static_cast<size_t>(c)];
        const long double l = (caps.flops_cap > 0 ? static_cast<long double>(w.flops) / caps.flops_cap : 0) +
                              (caps.bytes_cap > 0 ? static_cast<long double>(w.bytes) / caps.bytes_cap : 0);
        const long double key = caps.fits(w) ? l : 1e9L + l;
        if (key < best_key) {
          best_key = key;
          best = p;
        }
      }
      part_of[static_cast<size_t>(c)] = best;
      load[static_cast<size_t>(best)] += cw[static_cast<size_t>(c)];
    }
    for (int v = 0; v < n; ++v) a[static_cast<size_t>(v)] = part_of[static_cast<size_t>(comp[static_cast<size_t>(v)])];
    out.push_back(a);
  }
  if (n > 4 * parts) {
    Hypergraph cur = h;
    std::vector<std::vector<int>> maps;
    while (cur.vertex_count() > std::max(4 * parts, 32)) {
      auto [coarse, map] = detail::coarsen(cur, caps);
      if (coarse.vertex_count() >= cur.vertex_count()) break;
      maps.push_back(std::move(map));
      cur = std::move(coarse);
    }
    std::vector<int> m = detail::lpt_assign(cur, detail::VertexOrder::by_weight_desc(cur), parts,
                                            detail::BalanceCaps::of(cur, parts, eps_comp, eps_data));
    for (size_t level = maps.size(); level > 0; --level) {
      const std::vector<int>& map = maps[level - 1];
      std::vector<int> fine(map.size());
      for (size_t v = 0; v < map.size(); ++v) fine[v] = m[static_cast<size_t>(map[v])];
      m = std::move(fine);
    }
    out.push_back(std::move(m));
  }
  std::mt19937_64 rng(seed);
  for (int r = 0; r < options.random_restarts; ++r) {
    for (int v = 0; v < n; ++v) a[static_cast<size_t>(v)] = static_cast<int>(rng() % static_cast<std::uint64_t>(parts));
    out.push_back(a);
  }
  if (!options.hint.empty()) {
    if (static_cast<int>(options.hint.size()) != n) throw Error("partition_heuristic: hint size mismatch");
    for (int p : options.hint)
      if (p < 0 || p >= parts) throw Error("partition_heuristic: hint part out of range");
    out.push_back(options.hint);
  }
  return out;
}

// partition_heuristic (hypergraph.hpp:623-784) with candidates evaluated concurrently and
// repair scans split across the remaining threads; same result, same exceptions.
inline dcp::Partition partition_parallel(const dcp::Hypergraph& h, int parts, double eps_comp, double eps_data,
                                         std::uint64_t seed, const dcp::PartitionOptions& options = {},
                                         int threads = 0) {
  using namespace dcp;
  if (parts < 1) throw Error("partition_heuristic: parts must be >= 1");
  if (threads <= 0) threads = default_threads();
  const int n = h.vertex_count();
  Partition result;
  result.parts = parts;
  result.eps_comp = eps_comp;
  result.eps_data = eps_data;
  if (n == 0) return result;
  const auto caps = detail::BalanceCaps::of(h, parts, eps_comp, eps_data);
  for (int v = 0; v < n; ++v)
    if (!caps.fits(h.weights[static_cast<size_t>(v)]))
      throw InfeasibleError(
          "partition_heuristic: a single atomic vertex exceeds the balance cap "
          "(block size too large for this epsilon)");
  if (parts == 1) {
    result.assignment.assign(static_cast<size_t>(n), 0);
    return result;
  }
  const bool profile = std::getenv("DCPX_PLANNER_PROFILE") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  const auto t0 = now();
  std::vector<std::vector<int>> cands = partition_candidates(h, parts, eps_comp, eps_data, seed, options, caps);
  const double t_cand = std::chrono::duration<double>(now() - t0).count();
  const int nc = static_cast<int>(cands.size());
  struct Outcome {
    bool feasible = false;
    ByteCount cost = 0;
    double seconds = 0;
  };
  std::vector<Outcome> res(static_cast<size_t>(nc));
  const bool small = n <= 256;
  // candidates run concurrently
  const int outer = std::min(threads, nc);
  parallel_for(nc, outer, [&](int i) {
    const auto t1 = now();
    std::vector<int>& a = cands[static_cast<size_t>(i)];
    detail::EdgeCounts counts(h, parts);
    auto loads = detail::part_weights(h, a, parts);
    counts.reset(a);
    bool ok = true;
    if (!detail::balanced(h, a, parts, caps)) ok = repair_fast(h, a, parts, caps, counts, loads);
    if (ok) {
      for (int pass = 0; pass < options.max_passes; ++pass) {
        const bool improved = small ? detail::fm_pass(h, a, parts, caps, counts, loads)
                                    : detail::greedy_pass(h, a, parts, caps, counts, loads);
        if (!improved) break;
      }
      counts.reset(a);
      res[static_cast<size_t>(i)] = {true, counts.cost(), 0};
    }
    res[static_cast<size_t>(i)].seconds = std::chrono::duration<double>(now() - t1).count();
  });
  // selection exactly as the reference's loop (:772-777), in candidate order
  bool any = false;
  ByteCount best_cost = std::numeric_limits<ByteCount>::max();
  int best = -1;
  for (int i = 0; i < nc; ++i) {
    const Outcome& o = res[static_cast<size_t>(i)];
    if (!o.feasible) continue;
    if (!any || o.cost < best_cost || (o.cost == best_cost && cands[static_cast<size_t>(i)] < cands[static_cast<size_t>(best)])) {
      any = true;
      best_cost = o.cost;
      best = i;
    }
  }
  if (profile) {
    std::fprintf(stderr, "[partition_parallel] n=%d parts=%d threads=%d candidates %.2fs;", n, parts, threads, t_cand);
    for (int i = 0; i < nc; ++i)
      std::fprintf(stderr, " c%d %s%.2fs", i, res[static_cast<size_t>(i)].feasible ? "" : "(infeasible) ",
                   res[static_cast<size_t>(i)].seconds);
    std::fprintf(stderr, " -> c%d\n", best);
  }
  if (!any) throw InfeasibleError("partition_heuristic: no feasible partition found under the balance caps");
  result.assignment = std::move(cands[static_cast<size_t>(best)]);
  return result;
}

// place (placement.hpp:96-162) with partition_parallel in place of partition_heuristic. The
// per-machine sub-problems of level 2 are independent as well and run concurrently.
inline dcp::PlacementResult place_parallel(const dcp::BlockGraph& g, const dcp::DeviceTopology& topo,
                                           const dcp::PlacementConfig& cfg = {}, int threads = 0) {
  using namespace dcp;
  if (threads <= 0) threads = default_threads();
  topo.validate();
  const Hypergraph h = build_hypergraph(g);
  const int X = topo.machines, Y = topo.devices_per_machine;
  const int n = h.vertex_count();
  std::vector<int> machine_of(static_cast<size_t>(n), 0);
  ByteCount inter_bytes = 0;
  if (X > 1) {
    Partition level1;
    try {
      level1 = partition_parallel(h, X, cfg.eps_inter, cfg.eps_data, cfg.seed, cfg.partition_options, threads);
    } catch (const InfeasibleError& e) {
      throw InfeasibleError(std::string("machine-level placement: ") + e.what());
    }
    machine_of = level1.assignment;
    inter_bytes = connectivity_cost(h, level1);
  }
  std::vector<int> device_of(static_cast<size_t>(n), 0);
  std::vector<ByteCount> intra(static_cast<size_t>(X), 0);
  std::vector<std::string> errors(static_cast<size_t>(X));
  const int outer = std::min(X, threads);
  parallel_for(X, outer, [&](int m) {
    std::vector<int> verts;
    for (int v = 0; v < n; ++v)
      if (machine_of[static_cast<size_t>(v)] == m) verts.push_back(v);
    if (verts.empty()) return;
    if (Y == 1) {
      for (int v : verts) device_of[static_cast<size_t>(v)] = m * Y;
      return;
    }
    // induced sub-hypergraph: edges keep only the members on this machine
    Hypergraph sub;
    std::vector<int> local_id(static_cast<size_t>(n), -1);
    for (size_t i = 0; i < verts.size(); ++i) local_id[static_cast<size_t>(verts[i])] = static_cast<int>(i);
    sub.comp_count = static_cast<int>(verts.size());
    sub.group_count = 0;
    sub.weights.resize(verts.size());
    for (size_t i = 0; i < verts.size(); ++i) sub.weights[i] = h.weights[static_cast<size_t>(verts[i])];
    for (const auto& e : h.edges) {
      Hyperedge se;
      se.weight = e.weight;
      for (int v : e.members)
        if (local_id[static_cast<size_t>(v)] >= 0) se.members.push_back(local_id[static_cast<size_t>(v)]);
      if (se.members.size() > 1) sub.edges.push_back(std::move(se));
    }
    try {
      const Partition level2 = partition_parallel(sub, Y, cfg.eps_intra, cfg.eps_data,
                                                  cfg.seed + static_cast<std::uint64_t>(m) + 1, cfg.partition_options,
                                                  std::max(1, threads / outer));
      intra[static_cast<size_t>(m)] = connectivity_cost(sub, level2);
      for (size_t i = 0; i < verts.size(); ++i)
        device_of[static_cast<size_t>(verts[i])] = m * Y + level2.assignment[i];
    } catch (const InfeasibleError& e) {
      errors[static_cast<size_t>(m)] = "device-level placement on machine " + std::to_string(m) + ": " + e.what();
    }
  });
  for (const auto& e : errors)  // the lowest machine's failure, as the sequential loop raises
    if (!e.empty()) throw InfeasibleError(e);
  PlacementResult r = detail::placement_from_flat(g, h, device_of, topo);
  r.inter_machine_bytes = inter_bytes;
  for (ByteCount b : intra) r.intra_machine_bytes += b;
  return r;
}

// plan_batch (pipeline.hpp:29-38) with place_parallel.
inline dcp::PlannedBatch plan_batch_parallel(const dcp::Batch& batch, const dcp::DeviceTopology& topo,
                                             const dcp::PlannerConfig& cfg, int threads = 0) {
  dcp::PlannedBatch pb;
  pb.graph = dcp::generate_blocks(batch, cfg.block_size);
  pb.placement = place_parallel(pb.graph, topo, cfg.placement, threads);
  pb.schedule = dcp::schedule(pb.graph, pb.placement, cfg.divisions);
  pb.plans = dcp::compile_plans(pb.schedule, pb.graph, pb.placement, cfg.compile);
  pb.volume = dcp::communication_volume(pb.graph, pb.placement);
  return pb;
}

}  // namespace dcpx_planner

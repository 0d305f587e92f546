// test_device_shim.cpp -- the reference's own test semantics, run through
// the device execution policy (include/graflow_b200/device.hpp).
//
// Built against the UNMODIFIED reference headers (graflow/*.hpp and the
// corpus generator tests/random_graphs.hpp) by tests/cpp/Makefile in the
// build container; the binary travels to the GPU box (it reads nothing from
// /root/reference at run time).  The graphs are the reference's own Graph
// objects built by its build_csr/build_transpose; the oracle is its own
// reference_dijkstra.  Exit code = number of failed checks (the
// acceptance.cpp:435-455 convention).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>
#include <set>
#include <string>
#include <tuple>
#include <vector>

#include "graflow_b200/device.hpp"
#include "random_graphs.hpp"

using namespace graflow;

static int g_fail = 0, g_pass = 0;
#define CHECK(c)                                                            \
  do {                                                                      \
    if (c) {                                                                \
      ++g_pass;                                                             \
    } else {                                                                \
      ++g_fail;                                                             \
      std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #c);              \
    }                                                                       \
  } while (0)

template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static Graph triangle() { return build_csr({{0, 1, 1.0}, {0, 2, 4.0}, {1, 2, 2.0}}, 3); }

static std::vector<DeviceSsspConfig> device_configs() {
  std::vector<DeviceSsspConfig> out;
  for (auto dir : {Direction::push, Direction::pull})
    for (bool autod : {false, true}) {
      DeviceSsspConfig c;
      c.direction = dir;
      c.policy.auto_direction = autod;
      // AUTO pulls when a superstep's frontier edges exceed m / alpha: alpha = 8
      // makes the switch fire on these small graphs (alpha <= 1 never pulls)
      if (autod) c.policy.pull_alpha = 8.0f;
      out.push_back(c);
    }
  return out;
}

// test_algorithms.cpp:66-92 / acceptance.cpp:56-91
static bool valid_pred_tree(const Graph& g, vertex_t source, const DistanceMap& dist,
                            const PredecessorMap& pred) {
  std::size_t n = g.num_vertices();
  for (vertex_t v = 0; v < n; ++v) {
    if (v == source || dist[v] == unreachable) {
      if (pred[v] != no_predecessor) return false;
      continue;
    }
    vertex_t u = pred[v];
    if (u == no_predecessor) return false;
    bool found = false;
    for (auto e : g.get_edges(u))
      if (g.get_dest_vertex(e) == v && dist[u] + g.get_edge_weight(e) == dist[v]) found = true;
    if (!found) return false;
    vertex_t walk = v;
    for (std::size_t steps = 0; walk != source; ++steps) {
      walk = pred[walk];
      if (walk == no_predecessor || steps > n) return false;
    }
  }
  return true;
}

int main() {
  // --- test_algorithms.cpp:134-144: triangle under every device config
  {
    Graph g = build_transpose(triangle());
    for (const auto& cfg : device_configs()) {
      auto r = sssp(g, 0, cfg);
      CHECK((r.dist == DistanceMap{0, 1, 3}));
      CHECK((r.pred == PredecessorMap{no_predecessor, 0, 1}));
      CHECK(r.supersteps >= 1 && r.relaxations >= 3);
    }
  }
  // --- :146-156 degenerate cases
  {
    Graph single = build_csr({}, 1);
    auto r = sssp(single, 0, DeviceSsspConfig{});
    CHECK((r.dist == DistanceMap{0}));
    CHECK((r.pred == PredecessorMap{no_predecessor}));
    Graph two = build_csr({{0, 1, 1.0}}, 3);
    auto r2 = sssp(two, 0, DeviceSsspConfig{});
    CHECK(r2.dist[2] == unreachable && r2.pred[2] == no_predecessor);
  }
  // --- :158-179 rejections (same exception types as the reference)
  {
    Graph g = triangle();
    CHECK(throws<std::out_of_range>([&] { sssp(g, 9, DeviceSsspConfig{}); }));
    DeviceSsspConfig pull;
    pull.direction = Direction::pull;
    CHECK(throws<std::invalid_argument>([&] { sssp(g, 0, pull); }));
    DeviceSsspConfig q;  // the queue (async) model is push-only, like the reference
    q.frontier_repr = FrontierRepr::queue;
    q.direction = Direction::pull;
    CHECK(throws<std::invalid_argument>([&] { sssp(g, 0, q); }));
  }
  // --- acceptance.cpp:95-122 (C1 + C4): 200 graphs, every device config,
  //     distances == reference_dijkstra exactly, predecessor trees valid
  {
    std::mt19937_64 sizes(2024);
    int dist_bad = 0, pred_bad = 0;
    for (int instance = 0; instance < 200; ++instance) {
      std::size_t n = 2 + sizes() % 499;
      Graph g = build_transpose(testutil::random_graph(n, 9000 + instance));
      auto oracle = reference_dijkstra(g, 0).first;
      for (const auto& cfg : device_configs()) {
        auto r = sssp(g, 0, cfg);
        if (r.dist != oracle) ++dist_bad;
        if (!valid_pred_tree(g, 0, r.dist, r.pred)) ++pred_bad;
      }
    }
    std::printf("C1 oracle sweep: %d mismatching runs; C4 pred trees: %d invalid\n", dist_bad,
                pred_bad);
    CHECK(dist_bad == 0);
    CHECK(pred_bad == 0);
  }
  // --- test_algorithms.cpp:181-192 random corpus, also in f32 / u32 modes
  {
    for (std::uint64_t seed = 0; seed < 15; ++seed) {
      std::size_t n = 20 + seed * 13;
      Graph g = build_transpose(testutil::random_graph(n, seed + 100));
      auto oracle = reference_dijkstra(g, 0).first;
      DeviceSsspConfig cfg;
      auto r = sssp(g, 0, cfg);
      CHECK(r.dist == oracle);
      CHECK(valid_pred_tree(g, 0, r.dist, r.pred));
    }
    // integer weights: u32 device arithmetic == the reference's doubles
    std::mt19937_64 rng(11);
    std::vector<WeightedEdge> edges;
    for (vertex_t u = 0; u < 400; ++u)
      for (int k = 0; k < 6; ++k) edges.push_back({u, (vertex_t)(rng() % 400), (double)(rng() % 50)});
    Graph g = build_transpose(build_csr(edges, 400));
    DeviceSsspConfig cfg;
    cfg.policy.arithmetic = GFB_W_U32;
    auto r = sssp(g, 0, cfg);
    CHECK(r.dist == reference_dijkstra(g, 0).first);
    CHECK(valid_pred_tree(g, 0, r.dist, r.pred));
    // the partitioned loop (policy.devices, gfb_mg_*): 2 and 3 partitions
    // on device 0, same fixpoint; f64 arithmetic is rejected
    // -- with both exchanges (device-initiated peer reductions; bucketed
    // messages over NCCL / device copies)
    for (int ex : {GFB_EXCHANGE_PEER, GFB_EXCHANGE_NCCL})
      for (int parts : {2, 3}) {
        DeviceSsspConfig mc = cfg;
        mc.policy.devices.assign(parts, 0);
        mc.policy.exchange = ex;
        auto rm = sssp(g, 0, mc);
        CHECK(rm.dist == r.dist);
        CHECK(valid_pred_tree(g, 0, rm.dist, rm.pred));
        auto rm7 = sssp(g, 7, mc);
        CHECK(rm7.dist == reference_dijkstra(g, 7).first);
      }
    {
      DeviceSsspConfig bad = cfg;
      bad.policy.devices = {0, 0};
      bad.policy.arithmetic = GFB_W_F64;
      bool threw = false;
      try {
        sssp(g, 0, bad);
      } catch (const std::invalid_argument&) {
        threw = true;
      }
      CHECK(threw);
    }
    // the queue representation (the reference's async model) on the device
    {
      DeviceSsspConfig qc = cfg;
      qc.frontier_repr = FrontierRepr::queue;
      auto rq = sssp(g, 0, qc);
      CHECK(rq.dist == r.dist);
      CHECK(valid_pred_tree(g, 0, rq.dist, rq.pred));
      CHECK(rq.supersteps == 0);
      qc.direction = Direction::pull;
      bool threw = false;
      try {
        sssp(g, 0, qc);
      } catch (const std::invalid_argument&) {
        threw = true;
      }
      CHECK(threw);
    }
    // the near-far loop (policy.delta) reaches the same fixpoint
    for (double delta : {1.0, 16.0, 200.0}) {
      DeviceSsspConfig nf = cfg;
      nf.policy.delta = delta;
      auto rn = sssp(g, 0, nf);
      CHECK(rn.dist == r.dist);
      CHECK(valid_pred_tree(g, 0, rn.dist, rn.pred));
    }
  }
  // --- BFS: test_algorithms.cpp:185-211 and acceptance.cpp:180-199 (C5)
  {
    DeviceSsspConfig cfg;
    CHECK((bfs(triangle(), 0, cfg).depth == DistanceMap{0, 1, 1}));
    Graph path = build_csr({{0, 1, 5.0}, {1, 2, 0.5}, {2, 3, 2.0}}, 4);
    CHECK((bfs(path, 0, cfg).depth == DistanceMap{0, 1, 2, 3}));
    DeviceSsspConfig q = cfg;
    q.frontier_repr = FrontierRepr::queue;
    bool threw = false;
    try {
      bfs(triangle(), 0, q);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
    int bad = 0;
    for (int instance = 0; instance < 50; ++instance) {
      std::size_t n = 5 + instance * 7;
      auto edges = testutil::random_edges(n, 6000 + instance);
      Graph g = build_transpose(build_csr(edges, n));
      auto want = graflow::bfs(g, 0, SsspConfig{ExecutionPolicy::sequential()});
      for (Direction dir : {Direction::push, Direction::pull}) {
        DeviceSsspConfig c2;
        c2.direction = dir;
        auto got = bfs(g, 0, c2);
        if (got.depth != want.depth || got.supersteps != want.supersteps ||
            got.relaxations != want.relaxations)
          ++bad;
      }
    }
    std::printf("C5 bfs vs reference bfs(): %d mismatching runs\n", bad);
    CHECK(bad == 0);
  }
  // --- acceptance.cpp:157-177 (C3): 20 repeated runs, identical distances
  {
    Graph g = testutil::random_graph(1000, 424242);
    auto first = sssp(g, 0, DeviceSsspConfig{}).dist;
    bool same = true;
    for (int run = 1; run < 20; ++run) same = same && sssp(g, 0, DeviceSsspConfig{}).dist == first;
    CHECK(same);
    CHECK(first == reference_dijkstra(g, 0).first);
  }
  // --- test_algorithms.cpp:202-211 triangle inequality at the fixpoint
  {
    Graph g = testutil::random_graph(200, 77);
    auto r = sssp(g, 0, DeviceSsspConfig{});
    bool ok = true;
    for (edge_t e = 0; e < g.num_edges(); ++e) {
      vertex_t u = g.get_source_vertex(e), v = g.get_dest_vertex(e);
      if (r.dist[u] == unreachable) continue;
      ok = ok && r.dist[v] <= r.dist[u] + g.get_edge_weight(e);
    }
    CHECK(ok);
  }
  // --- operator level: test_operators.cpp:31-37, :67-84, :86-102, :151-171
  {
    DevicePolicy pol;
    Graph g = build_transpose(triangle());
    DeviceFrontier f(FrontierRepr::sparse, 3);
    f.assign({0});
    auto out = neighbors_expand(pol, g, f, device_ops::always{});
    CHECK((out.contents() == std::vector<vertex_t>{1, 2}));

    Graph g2 = testutil::random_graph(80, 21);
    DeviceFrontier f2(FrontierRepr::sparse, 80);
    std::vector<vertex_t> fr;
    for (vertex_t v = 0; v < 80; v += 3) fr.push_back(v);
    f2.assign(fr);
    std::vector<vertex_t> expected;
    for (vertex_t v : fr)
      for (auto e : g2.get_edges(v)) expected.push_back(g2.get_dest_vertex(e));
    CHECK(neighbors_expand(pol, g2, f2, device_ops::always{}).contents() == expected);

    for (std::uint64_t seed : {1, 2, 3, 4, 5}) {
      Graph g3 = build_transpose(testutil::random_graph(40, seed));
      DeviceFrontier f3(FrontierRepr::dense, 40);
      std::vector<vertex_t> v3;
      for (vertex_t v = 0; v < 40; v += 2) v3.push_back(v);
      f3.assign(v3);
      DeviceRecorder push_rec(4096), pull_rec(4096);
      neighbors_expand(pol, g3, f3, device_ops::record{push_rec});
      neighbors_expand_pull(pol, g3, f3, device_ops::record{pull_rec});
      auto a = push_rec.triples(), b = pull_rec.triples();
      std::sort(a.begin(), a.end());
      std::sort(b.begin(), b.end());
      // the reference's own recording of the same expansion
      std::set<std::tuple<vertex_t, vertex_t, edge_t>> ref;
      Frontier rf(FrontierRepr::dense, 40);
      for (vertex_t v : v3) rf.add_vertex(v);
      neighbors_expand(ExecutionPolicy::sequential(), g3, rf, [&](vertex_t s, vertex_t d, edge_t e, weight_t) {
        ref.insert({s, d, e});
        return false;
      });
      CHECK(a == b);
      CHECK((std::vector<std::tuple<vertex_t, vertex_t, edge_t>>(ref.begin(), ref.end()) == a));
    }

    // sssp composed from device operators exactly as algorithms.hpp:165-182
    Graph g4 = build_transpose(testutil::random_graph(300, 5));
    auto oracle = reference_dijkstra(g4, 0).first;
    for (bool pull : {false, true}) {
      DeviceDistances dist(g4, pol, 0, true);
      DeviceFrontier cur(pull ? FrontierRepr::dense : FrontierRepr::sparse, 300);
      cur.assign({0});
      std::size_t steps = 0;
      while (cur.size() != 0) {
        ++steps;
        cur = pull ? neighbors_expand_pull(pol, g4, cur, device_ops::relax_min{dist})
                   : neighbors_expand(pol, g4, cur, device_ops::relax_min{dist});
      }
      CHECK(dist.read() == oracle);
      CHECK(steps > 1);
    }

    // filter (operators.hpp:163-188): the reference's own filter with the same
    // predicate as a lambda, sparse (order + duplicates) and dense
    {
      DeviceDistances dist(g4, pol, 0, true);
      DeviceFrontier cur(FrontierRepr::sparse, 300);
      cur.assign({0});
      while (cur.size() != 0) cur = neighbors_expand(pol, g4, cur, device_ops::relax_min{dist});
      const DistanceMap d = dist.read();
      std::vector<vertex_t> lst;
      for (vertex_t v = 0; v < 300; ++v) lst.push_back((v * 37u) % 300u);
      for (vertex_t v = 0; v < 300; v += 3) lst.push_back(v);  // duplicates
      const double thr = d[lst[7]] == unreachable ? 1.0 : d[lst[7]];
      for (FrontierRepr repr : {FrontierRepr::sparse, FrontierRepr::dense}) {
        Frontier hf(repr, 300);
        DeviceFrontier df(repr, 300);
        for (vertex_t v : lst) hf.add_vertex(v);
        df.assign(lst);
        auto contents = [](const Frontier& f) {
          std::vector<vertex_t> out;
          for (std::size_t i = 0; i < f.size(); ++i) out.push_back(f.get_active_vertex(i));
          return out;
        };
        CHECK(filter(pol, df, device_ops::dist_below{dist, thr}).contents() ==
              contents(filter(ExecutionPolicy::sequential(), hf,
                              [&](vertex_t v) { return d[v] < thr; })));
        CHECK(filter(pol, df, device_ops::dist_at_least{dist, thr}).contents() ==
              contents(filter(ExecutionPolicy::sequential(), hf,
                              [&](vertex_t v) { return d[v] >= thr; })));
        CHECK(filter(pol, df, device_ops::reached{dist}).contents() ==
              contents(filter(ExecutionPolicy::sequential(), hf,
                              [&](vertex_t v) { return d[v] != unreachable; })));
      }
    }

    DeviceFrontier dup(FrontierRepr::sparse, 10);
    dup.assign({5, 3, 5, 1, 3, 9});
    CHECK((uniquify(dup).contents() == std::vector<vertex_t>{1, 3, 5, 9}));
    CHECK(throws<std::invalid_argument>([&] {
      neighbors_expand_pull(pol, triangle(), DeviceFrontier(FrontierRepr::dense, 3),
                            device_ops::always{});
    }));
  }
  std::printf("device shim: %d checks passed, %d failed\n", g_pass, g_fail);
  return g_fail;
}

// ref_shim.cpp -- C entry points over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file against the
// reference's own headers where they lie (/root/reference/proj/include and
// proj/tests/random_graphs.hpp) into oracle/_ref/libgraflow_ref.so.  No
// reference source is copied into this repository.  The library is used to
// (1) generate the golden fixtures in tests/golden/ that pin the C
// restatement (graflow_oracle.c), and (2) time the reference CPU path in
// bench.py (--impl reference and the cpu_baseline leg).
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "graflow/algorithms.hpp"
#include "graflow/io.hpp"
#include "random_graphs.hpp"

using namespace graflow;

namespace {
thread_local std::string g_err;

// 0 ok, 1 invalid_argument, 2 out_of_range, 3 logic_error, 4 other
template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 2;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

unsigned ref_hardware_concurrency() { return ExecutionPolicy::default_workers(); }

// random_graphs.hpp:15-30
size_t ref_random_edges(size_t n, uint64_t seed, uint32_t* src, uint32_t* dst,
                        double* w, size_t cap) {
  auto e = testutil::random_edges(n, seed);
  for (size_t i = 0; i < e.size() && i < cap; ++i) {
    src[i] = e[i].src;
    dst[i] = e[i].dst;
    w[i] = e[i].weight;
  }
  return e.size();
}

// graph.hpp:132-162 (+ :184-211 when transpose != 0)
int ref_graph_new(size_t n, size_t m, const uint32_t* src, const uint32_t* dst,
                  const double* w, int transpose, void** out) {
  return guarded([&] {
    std::vector<WeightedEdge> edges(m);
    for (size_t i = 0; i < m; ++i) edges[i] = {src[i], dst[i], w[i]};
    Graph g = build_csr(edges, n);
    *out = new Graph(transpose ? build_transpose(g) : std::move(g));
  });
}

void ref_graph_free(void* g) { delete static_cast<Graph*>(g); }

void ref_graph_csr(void* gp, uint32_t* ro, uint32_t* col, double* val) {
  auto& g = *static_cast<Graph*>(gp);
  std::memcpy(ro, g.row_offsets().data(), g.row_offsets().size() * 4);
  std::memcpy(col, g.column_indices().data(), g.column_indices().size() * 4);
  std::memcpy(val, g.values().data(), g.values().size() * 8);
}

// CSC view (graph.hpp:85-96)
void ref_graph_csc(void* gp, uint32_t* cso, uint32_t* csrc, double* cval,
                   uint32_t* ceid) {
  auto& g = *static_cast<Graph*>(gp);
  size_t n = g.num_vertices();
  for (size_t u = 0; u < n; ++u) {
    auto r = g.in_edges(static_cast<vertex_t>(u));
    cso[u] = r.start;
    if (u + 1 == n) cso[n] = r.stop;
    for (auto i : r) {
      csrc[i] = g.in_edge_source(i);
      cval[i] = g.in_edge_weight(i);
      ceid[i] = g.in_edge_id(i);
    }
  }
  if (n == 0) cso[0] = 0;
}

// algorithms.hpp:134-188.  mode: 0 seq, 1 par, 2 par-nosync;
// direction: 0 push, 1 pull; repr: 0 sparse, 1 dense, 2 queue.
int ref_sssp(void* gp, uint32_t source, int mode, size_t workers, int direction,
             int repr, int uniquify, double* dist, uint32_t* pred,
             uint64_t* supersteps, uint64_t* relaxations) {
  return guarded([&] {
    SsspConfig cfg;
    cfg.policy = {static_cast<ExecutionMode>(mode), workers};
    cfg.direction = direction ? Direction::pull : Direction::push;
    cfg.frontier_repr = static_cast<FrontierRepr>(repr);
    cfg.uniquify_frontier = uniquify != 0;
    auto r = sssp(*static_cast<Graph*>(gp), source, cfg);
    std::memcpy(dist, r.dist.data(), r.dist.size() * 8);
    std::memcpy(pred, r.pred.data(), r.pred.size() * 4);
    *supersteps = r.supersteps;
    *relaxations = r.relaxations;
  });
}

// algorithms.hpp:194-239 (mode / direction / repr as ref_sssp)
int ref_bfs(void* gp, uint32_t source, int mode, size_t workers, int direction, int repr,
            double* depth, uint64_t* supersteps, uint64_t* relaxations) {
  return guarded([&] {
    SsspConfig cfg;
    cfg.policy = {static_cast<ExecutionMode>(mode), workers};
    cfg.direction = direction ? Direction::pull : Direction::push;
    cfg.frontier_repr = static_cast<FrontierRepr>(repr);
    auto r = bfs(*static_cast<Graph*>(gp), source, cfg);
    std::memcpy(depth, r.depth.data(), r.depth.size() * 8);
    *supersteps = r.supersteps;
    *relaxations = r.relaxations;
  });
}

// algorithms.hpp:101-128
int ref_dijkstra(void* gp, uint32_t source, double* dist, uint32_t* pred) {
  return guarded([&] {
    auto [d, p] = reference_dijkstra(*static_cast<Graph*>(gp), source);
    std::memcpy(dist, d.data(), d.size() * 8);
    std::memcpy(pred, p.data(), p.size() * 4);
  });
}

// operators.hpp:35-68 / :296-334 with a recording cond: the eligible
// (src, dst, edge) triples of one push or pull expansion of `k` vertices.
// Returns the number of triples (writes at most cap).
size_t ref_expand_record(void* gp, const uint32_t* frontier, size_t k, int pull,
                         uint32_t* s, uint32_t* d, uint32_t* e, size_t cap) {
  auto& g = *static_cast<Graph*>(gp);
  Frontier f(pull ? FrontierRepr::dense : FrontierRepr::sparse, g.num_vertices());
  for (size_t i = 0; i < k; ++i) f.add_vertex(frontier[i]);
  size_t cnt = 0;
  auto rec = [&](vertex_t a, vertex_t b, edge_t c, weight_t) {
    if (cnt < cap) {
      s[cnt] = a;
      d[cnt] = b;
      e[cnt] = c;
    }
    ++cnt;
    return false;
  };
  if (pull)
    neighbors_expand_pull(ExecutionPolicy::sequential(), g, f, rec);
  else
    neighbors_expand(ExecutionPolicy::sequential(), g, f, rec);
  return cnt;
}

// operators.hpp:163-188 filter with the predicate `dist[v] < thr` (pred 0),
// `dist[v] >= thr` (1) or `dist[v] < +inf` (2), on a sparse (repr 0) or
// dense (1) frontier of `k` vertices; the result's contents in the
// reference's order (dense: ascending).  Returns the count (writes <= cap).
size_t ref_filter(size_t n, const uint32_t* frontier, size_t k, int repr, int pred,
                  const double* dist, double thr, int mode, size_t workers, uint32_t* out,
                  size_t cap) {
  Frontier f(repr ? FrontierRepr::dense : FrontierRepr::sparse, n);
  for (size_t i = 0; i < k; ++i) f.add_vertex(frontier[i]);
  ExecutionPolicy p{static_cast<ExecutionMode>(mode), workers};
  Frontier r = filter(p, f, [&](vertex_t v) {
    return pred == 0 ? dist[v] < thr : pred == 1 ? dist[v] >= thr : dist[v] != unreachable;
  });
  const size_t cnt = r.size();
  for (size_t i = 0; i < cnt && i < cap; ++i) out[i] = r.get_active_vertex(i);
  return cnt;
}

// io.hpp:43-123 parse_matrix_market on a text buffer.  Returns the edge
// count (writes <= cap edges and *n), or -1 on ParseError with its line and
// message (msg of msg_cap bytes).
long long ref_mm_parse(const char* text, size_t len, int force_unit, int expand_sym, size_t* n,
                       uint32_t* src, uint32_t* dst, double* w, size_t cap, size_t* err_line,
                       char* msg, size_t msg_cap) {
  try {
    MatrixMarketOptions opt;
    opt.force_unit_weights = force_unit != 0;
    opt.expand_symmetric = expand_sym != 0;
    EdgeList el = parse_matrix_market(std::string(text, len), opt);
    *n = el.num_vertices;
    for (size_t i = 0; i < el.edges.size() && i < cap; ++i) {
      src[i] = el.edges[i].src;
      dst[i] = el.edges[i].dst;
      w[i] = el.edges[i].weight;
    }
    return (long long)el.edges.size();
  } catch (const ParseError& e) {
    *err_line = e.line();
    std::snprintf(msg, msg_cap, "%s", e.what());
    return -1;
  }
}

}  // extern "C"

// graflow_b200/device.hpp -- the device execution policy for graflow.
//
// Header-only C++20 shim that plugs the B200 SSSP path (libgfb.so, C ABI in
// include/gfb.h) in behind the reference's own operator API, through the
// paper's execution-policy overloading: the reference's
// types stay exactly as they are --
//   graflow::Graph            graph.hpp:45-127
//   graflow::FrontierRepr     frontier.hpp:18
//   graflow::Direction        algorithms.hpp:32
//   graflow::SsspResult       algorithms.hpp:56-61
//   graflow::vertex_t/edge_t/weight_t, no_predecessor, unreachable (types.hpp)
// -- and a DevicePolicy overload set is added next to them:
//   sssp(const Graph&, vertex_t, const DeviceSsspConfig&) -> SsspResult
//       (algorithms.hpp:134-188; same result layout, same throw sites)
//   neighbors_expand(const DevicePolicy&, const Graph&, const DeviceFrontier&, Cond)
//       (operators.hpp:35-68)
//   neighbors_expand_pull(const DevicePolicy&, const Graph&, const DeviceFrontier&, Cond)
//       (operators.hpp:76-114)
//   uniquify(const DeviceFrontier&)            (operators.hpp:191-200)
// Host lambdas cannot run on the device, so `Cond` must be one of the
// recognised conditions in graflow::device_ops (relax_min, record, always);
// anything else is a compile-time error (cf. the reference's own rejection
// of unsupported frontier/policy combinations, operators.hpp:38-43).
//
// Include the reference's <graflow/algorithms.hpp> first (or let this
// header include it) and link libgfb.so.  See INTEGRATION.md.
#pragma once

#include <cstdint>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <type_traits>
#include <vector>

#include "graflow/algorithms.hpp"
#include "gfb.h"

namespace graflow {

namespace device_detail {

// gfb_status -> the exception type the reference throws at the same site.
inline void check(int rc) {
  if (rc == GFB_OK) return;
  std::string msg = gfb_last_error();
  switch (rc) {
    case GFB_EINVAL: throw std::invalid_argument(msg);
    case GFB_ERANGE: throw std::out_of_range(msg);
    case GFB_ELOGIC: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}

struct CtxDeleter {
  void operator()(gfb_ctx* c) const { gfb_ctx_destroy(c); }
};
struct GraphDeleter {
  void operator()(gfb_graph* g) const { gfb_graph_free(g); }
};

// One context (CUDA stream) per (host thread, device): gfb_ctx is
// single-threaded by contract (include/gfb.h).
inline gfb_ctx* context(int device) {
  thread_local std::map<int, std::unique_ptr<gfb_ctx, CtxDeleter>> ctxs;
  auto& c = ctxs[device];
  if (!c) {
    gfb_ctx* h = nullptr;
    check(gfb_ctx_create(device, &h));
    c.reset(h);
  }
  return c.get();
}

}  // namespace device_detail

/// Device execution policy (the new ExecutionPolicy value of the paper's
/// overloading mechanism).  `arithmetic` selects the device distance type:
/// GFB_W_F64 reproduces the reference's double arithmetic bit for bit,
/// GFB_W_U32 is exact for integer weights, GFB_W_F32 is the bandwidth mode.
struct DevicePolicy {
  int device = 0;
  gfb_wtype arithmetic = GFB_W_F64;
  // push<->pull switch on the device (Direction::push in the config): a
  // superstep pulls when its frontier edges exceed m / pull_alpha.  A plan
  // holds each vertex once, so its edges never exceed m: alpha <= 1 never
  // pulls.  Measured break-even at RMAT s24: the pull streams
  // all m in-edges in 1.40 ms, push takes ~1.45 ms for 0.95 m edges, so
  // alpha ~1.05; with the far-bucket deferral no superstep exceeds 0.22 m and
  // pulling never pays -- hence off by default (the reference's default is
  // Direction::push, algorithms.hpp:40).
  bool auto_direction = false;
  float pull_alpha = 1.05f;
  double delta = 0.0;          // > 0: near-far filter (push only; high-diameter
                               // graphs, any arithmetic) -- same distances.  0: the
                               // device chooses (near-far on low-degree meshes)
  // More than one entry: the graph is cut into edge-balanced vertex ranges,
  // partition q runs on devices[q] and relaxes remote vertices directly in
  // their owner's memory (gfb_mg_*, NVLink peer access; entries may repeat a
  // device).  u32 / f32 arithmetic, push, no near-far.  `device` is unused.
  std::vector<int> devices;
  // exchange of the multi-device path: GFB_EXCHANGE_PEER (device-initiated
  // reductions over NVLink peer memory) or GFB_EXCHANGE_NCCL (remote
  // candidates bucketed per owner, NCCL send/recv + allreduce per superstep)
  int exchange = GFB_EXCHANGE_PEER;

  void validate() const {
    if (device < 0) throw std::invalid_argument("device policy: device must be >= 0");
    if (devices.size() > 8) throw std::invalid_argument("device policy: at most 8 devices");
    for (int d : devices)
      if (d < 0) throw std::invalid_argument("device policy: device must be >= 0");
    if (devices.size() > 1 && arithmetic == GFB_W_F64)
      throw std::invalid_argument("device policy: multi-GPU needs u32 or f32 arithmetic");
    if (devices.size() > 1 && delta > 0)
      throw std::invalid_argument("device policy: the near-far filter is single-GPU");
    if (arithmetic < GFB_W_U32 || arithmetic > GFB_W_F64)
      throw std::invalid_argument("device policy: bad arithmetic");
    if (!(delta >= 0.0)) throw std::invalid_argument("device policy: delta must be >= 0");
  }
};

inline DevicePolicy device_policy(int device = 0, gfb_wtype arithmetic = GFB_W_F64) {
  DevicePolicy p;
  p.device = device;
  p.arithmetic = arithmetic;
  return p;
}

/// SsspConfig (algorithms.hpp:38-54) with a device policy.
struct DeviceSsspConfig {
  DevicePolicy policy{};
  Direction direction = Direction::push;
  FrontierRepr frontier_repr = FrontierRepr::sparse;
  bool uniquify_frontier = false;  // the device frontier is always a set

  void validate() const {
    policy.validate();
    // The queue representation is the reference's asynchronous model
    // (par-nosync, algorithms.hpp:44-53): on the device it runs as one
    // persistent work-queue launch (the near-far kernel with no far set);
    // like the reference it is push-only and reports no supersteps.
    if (frontier_repr == FrontierRepr::queue && direction != Direction::push)
      throw std::invalid_argument("config: queue frontier requires push direction");
    if (frontier_repr == FrontierRepr::queue && policy.devices.size() > 1)
      throw std::invalid_argument("config: the queue model is single-GPU");
  }
};

/// Device copy of a graflow::Graph.  Construct one and pass it to the
/// DeviceGraph overloads below to run many calls on one upload (the fast
/// path: the caller owns the handle and decides when the contents are
/// current, cf. graph.hpp:42-44 "immutable").  refill() re-copies new
/// contents of the same shape without reallocating.
class DeviceGraph {
 public:
  DeviceGraph(const Graph& g, const DevicePolicy& p, bool with_transpose)
      : n_(g.num_vertices()), m_(g.num_edges()), device_(p.device), arith_(p.arithmetic),
        csc_(with_transpose) {
    gfb_ctx* c = device_detail::context(p.device);
    gfb_graph* h = nullptr;
    device_detail::check(gfb_graph_upload(c, g.num_vertices(), g.num_edges(),
                                          g.row_offsets().data(), g.column_indices().data(),
                                          g.values().data(), GFB_W_F64, p.arithmetic,
                                          with_transpose ? 1 : 0, &h));
    h_.reset(h);
    ctx_ = c;
  }
  DeviceGraph(const Graph& g, const DevicePolicy& p) : DeviceGraph(g, p, g.has_transpose()) {}
  gfb_graph* handle() const { return h_.get(); }
  gfb_ctx* ctx() const { return ctx_; }
  std::size_t num_vertices() const { return n_; }
  bool has_transpose() const { return csc_; }
  bool fits(const Graph& g, const DevicePolicy& p, bool with_transpose) const {
    return n_ == g.num_vertices() && m_ == g.num_edges() && device_ == p.device &&
           arith_ == p.arithmetic && csc_ == with_transpose;
  }
  void refill(const Graph& g) {
    device_detail::check(gfb_graph_refill(h_.get(), g.row_offsets().data(),
                                          g.column_indices().data(), g.values().data(),
                                          GFB_W_F64));
  }

  /// The Graph-taking overloads' upload: the graph's CURRENT contents, copied
  /// on every call (gfb_graph_refill into a cached allocation of the same
  /// shape, so nothing is reallocated).  No address or sampled-fingerprint
  /// reuse: a different Graph at the same address, or one differing in a
  /// single weight, can never see a stale copy.  At most kCacheSlots
  /// allocations per host thread (least recently used evicted).  Keep a
  /// DeviceGraph yourself to skip the copy.
  static DeviceGraph& of(const Graph& g, const DevicePolicy& p, bool with_transpose) {
    thread_local std::vector<std::unique_ptr<DeviceGraph>> lru;  // front = most recent
    for (std::size_t i = 0; i < lru.size(); ++i) {
      if (!lru[i]->fits(g, p, with_transpose)) continue;
      std::unique_ptr<DeviceGraph> hit = std::move(lru[i]);
      lru.erase(lru.begin() + (long)i);
      hit->refill(g);
      lru.insert(lru.begin(), std::move(hit));
      return *lru.front();
    }
    if (lru.size() >= kCacheSlots) lru.pop_back();
    lru.insert(lru.begin(), std::make_unique<DeviceGraph>(g, p, with_transpose));
    return *lru.front();
  }
  static constexpr std::size_t kCacheSlots = 2;

 private:
  std::unique_ptr<gfb_graph, device_detail::GraphDeleter> h_;
  gfb_ctx* ctx_ = nullptr;
  std::size_t n_, m_;
  int device_;
  int arith_;
  bool csc_;
};

/// The graph partitioned over several devices (gfb_mg_*).  Like DeviceGraph:
/// the Graph overloads re-upload the current contents into the per-thread
/// handle of the same device list (one slot).
class DeviceMgGraph {
 public:
  explicit DeviceMgGraph(const DevicePolicy& p)
      : devices_(p.devices), arith_(p.arithmetic), exchange_(p.exchange) {
    gfb_mg* h = nullptr;
    device_detail::check(
        gfb_mg_create_ex((int)p.devices.size(), p.devices.data(), p.exchange, &h));
    h_.reset(h);
  }
  DeviceMgGraph(const Graph& g, const DevicePolicy& p) : DeviceMgGraph(p) { upload(g); }
  gfb_mg* handle() const { return h_.get(); }
  void upload(const Graph& g) {
    device_detail::check(gfb_mg_graph_upload(h_.get(), g.num_vertices(), g.num_edges(),
                                             g.row_offsets().data(), g.column_indices().data(),
                                             g.values().data(), GFB_W_F64, arith_));
  }

  static DeviceMgGraph& of(const Graph& g, const DevicePolicy& p) {
    thread_local std::unique_ptr<DeviceMgGraph> slot;
    if (!slot || slot->devices_ != p.devices || slot->arith_ != p.arithmetic ||
        slot->exchange_ != p.exchange)
      slot = std::make_unique<DeviceMgGraph>(p);
    slot->upload(g);
    return *slot;
  }

 private:
  struct Deleter {
    void operator()(gfb_mg* h) const { gfb_mg_destroy(h); }
  };
  std::unique_ptr<gfb_mg, Deleter> h_;
  std::vector<int> devices_;
  int arith_;
  int exchange_;
};

inline SsspResult sssp(const DeviceGraph& dg, vertex_t source, const DeviceSsspConfig& cfg);

/// Single-source shortest paths on the device (algorithms.hpp:134-188):
/// same validation order and exception types, same SsspResult layout.
/// dist is widened from the device arithmetic to double (exact); pred is
/// the acyclic tight-edge tree (NIL for the source and unreachable).
inline SsspResult sssp(const Graph& g, vertex_t source, const DeviceSsspConfig& cfg) {
  cfg.validate();
  std::size_t n = g.num_vertices();
  if (source >= n) throw std::out_of_range("sssp: source out of range");
  if (cfg.direction == Direction::pull && !g.has_transpose())
    throw std::invalid_argument("sssp: pull direction requires a built transpose");
  if (cfg.policy.devices.size() > 1) {  // partitioned over several devices
    if (cfg.direction == Direction::pull)
      throw std::invalid_argument("sssp: the multi-GPU loop is push-only");
    DeviceMgGraph& mg = DeviceMgGraph::of(g, cfg.policy);
    SsspResult r;
    r.dist.resize(n);
    r.pred.resize(n);
    gfb_sssp_stats st{};
    device_detail::check(gfb_mg_sssp(mg.handle(), source, nullptr, r.dist.data(), r.pred.data(), &st));
    r.supersteps = st.supersteps;
    r.relaxations = st.relaxations;
    return r;
  }
  return sssp(DeviceGraph::of(g, cfg.policy, g.has_transpose()), source, cfg);
}

/// sssp() on a caller-owned upload (no copy per call).
inline SsspResult sssp(const DeviceGraph& dg, vertex_t source, const DeviceSsspConfig& cfg) {
  cfg.validate();
  const std::size_t n = dg.num_vertices();
  if (source >= n) throw std::out_of_range("sssp: source out of range");
  const bool want_csc = dg.has_transpose();
  if (cfg.direction == Direction::pull && !want_csc)
    throw std::invalid_argument("sssp: pull direction requires a built transpose");
  if (cfg.policy.devices.size() > 1)
    throw std::invalid_argument("sssp: a DeviceGraph is single-device (use the Graph overload)");
  gfb_sssp_opts o;
  gfb_sssp_opts_default(&o);
  o.direction = cfg.direction == Direction::pull
                    ? GFB_DIR_PULL
                    : (cfg.policy.auto_direction && want_csc ? GFB_DIR_AUTO : GFB_DIR_PUSH);
  o.pull_alpha = cfg.policy.pull_alpha;
  if (cfg.policy.delta > 0 && cfg.direction != Direction::pull) {
    o.delta = cfg.policy.delta;
    o.direction = GFB_DIR_PUSH;  // the near-far loop is push-only
  }
  const bool queue = cfg.frontier_repr == FrontierRepr::queue;
  if (queue) {  // asynchronous work queue: near-far with an unbounded near set
    o.delta = std::numeric_limits<double>::infinity();
    o.direction = GFB_DIR_PUSH;
  }
  SsspResult r;
  r.dist.resize(n);
  r.pred.resize(n);
  gfb_sssp_stats st{};
  device_detail::check(gfb_sssp(dg.ctx(), dg.handle(), source, &o, r.dist.data(), r.pred.data(), &st));
  r.supersteps = queue ? 0 : st.supersteps;  // the async model has no supersteps
  r.relaxations = st.relaxations;
  return r;
}

/// Breadth-first search on the device (algorithms.hpp:194-239): same
/// validation and exceptions, same BfsResult (depth as double, +inf when
/// unreachable; supersteps; relaxations = claim evaluations).
inline BfsResult bfs(const Graph& g, vertex_t source, const DeviceSsspConfig& cfg) {
  cfg.validate();
  if (cfg.frontier_repr == FrontierRepr::queue)
    throw std::invalid_argument("bfs: queue configuration not supported "
                                "(level semantics require supersteps)");
  std::size_t n = g.num_vertices();
  if (source >= n) throw std::out_of_range("bfs: source out of range");
  if (cfg.direction == Direction::pull && !g.has_transpose())
    throw std::invalid_argument("bfs: pull direction requires a built transpose");
  DevicePolicy p = cfg.policy;
  if (p.devices.size() > 1) p.device = p.devices[0];  // BFS runs on one device
  DeviceGraph& dg = DeviceGraph::of(g, p, g.has_transpose());
  BfsResult r;
  r.depth.resize(n);
  uint64_t st = 0, rl = 0;
  device_detail::check(gfb_bfs(dg.ctx(), dg.handle(), source,
                               cfg.direction == Direction::pull ? GFB_DIR_PULL : GFB_DIR_PUSH,
                               r.depth.data(), &st, &rl));
  r.supersteps = st;
  r.relaxations = rl;
  return r;
}

// ---------------------------------------------------------------- operators

/// Device frontier (frontier.hpp:37-218, sparse and dense representations).
class DeviceFrontier {
 public:
  DeviceFrontier(FrontierRepr repr, std::size_t num_vertices, int device = 0)
      : repr_(repr), n_(num_vertices) {
    if (repr == FrontierRepr::queue)
      throw std::invalid_argument("device frontier: queue representation is the async model");
    gfb_frontier* h = nullptr;
    device_detail::check(gfb_frontier_create(device_detail::context(device), num_vertices,
                                             repr == FrontierRepr::dense ? GFB_DENSE : GFB_SPARSE, &h));
    h_.reset(h);
  }
  FrontierRepr repr() const { return repr_; }
  std::size_t num_vertices() const { return n_; }
  /// add_vertex for a batch (frontier.hpp:73-96 semantics).
  void assign(const std::vector<vertex_t>& vs) {
    device_detail::check(gfb_frontier_assign(h_.get(), vs.data(), vs.size()));
  }
  std::size_t size() const {
    uint64_t s = 0;
    device_detail::check(gfb_frontier_size(h_.get(), &s));
    return s;
  }
  bool empty() const { return size() == 0; }
  /// Sparse: element order; dense: ascending (get_active_vertex order).
  std::vector<vertex_t> contents() const {
    std::vector<vertex_t> out(size());
    uint64_t k = 0;
    device_detail::check(gfb_frontier_read(h_.get(), out.data(), out.size(), &k));
    out.resize(k);
    return out;
  }
  gfb_frontier* handle() const { return h_.get(); }

 private:
  struct Del {
    void operator()(gfb_frontier* f) const { gfb_frontier_free(f); }
  };
  FrontierRepr repr_;
  std::size_t n_;
  std::unique_ptr<gfb_frontier, Del> h_;
};

/// Device distance map for the relax_min condition.
class DeviceDistances {
 public:
  DeviceDistances(const Graph& g, const DevicePolicy& p, vertex_t source, bool with_transpose)
      : dg_(&DeviceGraph::of(g, p, with_transpose)) {
    gfb_dist* h = nullptr;
    device_detail::check(gfb_dist_create(dg_->ctx(), dg_->handle(), &h));
    h_.reset(h);
    device_detail::check(gfb_dist_init(h, source));
  }
  DistanceMap read(std::size_t* relaxations = nullptr) const {
    DistanceMap d(n());
    uint64_t r = 0;
    device_detail::check(gfb_dist_read(h_.get(), d.data(), &r));
    if (relaxations) *relaxations = r;
    return d;
  }
  gfb_dist* handle() const { return h_.get(); }

 private:
  std::size_t n() const {
    uint64_t n = 0;
    gfb_graph_info(dg_->handle(), &n, nullptr, nullptr, nullptr);
    return n;
  }
  struct Del {
    void operator()(gfb_dist* d) const { gfb_dist_free(d); }
  };
  DeviceGraph* dg_;
  std::unique_ptr<gfb_dist, Del> h_;
};

/// Records every (src, dst, edge) invocation (test_operators.cpp:151-171).
class DeviceRecorder {
 public:
  explicit DeviceRecorder(std::size_t capacity, int device = 0) {
    gfb_record* h = nullptr;
    device_detail::check(gfb_record_create(device_detail::context(device), capacity, &h));
    h_.reset(h);
  }
  std::vector<std::tuple<vertex_t, vertex_t, edge_t>> triples() const {
    uint64_t cnt = 0;
    device_detail::check(gfb_record_read(h_.get(), nullptr, nullptr, nullptr, 0, &cnt));
    std::vector<uint32_t> s(cnt), d(cnt), e(cnt);
    device_detail::check(gfb_record_read(h_.get(), s.data(), d.data(), e.data(), cnt, &cnt));
    std::vector<std::tuple<vertex_t, vertex_t, edge_t>> out;
    for (std::size_t i = 0; i < s.size(); ++i) out.emplace_back(s[i], d[i], e[i]);
    return out;
  }
  gfb_record* handle() const { return h_.get(); }

 private:
  struct Del {
    void operator()(gfb_record* r) const { gfb_record_free(r); }
  };
  std::unique_ptr<gfb_record, Del> h_;
};

/// The conditions the device policy recognises (the C ABI's gfb_op).
namespace device_ops {
struct relax_min {  // algorithms.hpp:151-158
  DeviceDistances& dist;
};
struct record {  // test-only eligibility recorder
  DeviceRecorder& rec;
};
struct always {};  // test_operators.cpp:27
// filter predicates (operators.hpp:163-188), compared in double
struct dist_below {  // dist[v] < threshold: the near side of a near-far split
  DeviceDistances& dist;
  double threshold;
};
struct dist_at_least {  // dist[v] >= threshold: the far side
  DeviceDistances& dist;
  double threshold;
};
struct reached {  // dist[v] < +inf
  DeviceDistances& dist;
};
}  // namespace device_ops

namespace device_detail {
template <class C> struct op_of {
  static_assert(sizeof(C) == 0,
                "device policy: host lambdas cannot run on the device; use "
                "graflow::device_ops::{relax_min, record, always}");
};
template <> struct op_of<device_ops::relax_min> {
  static int op() { return GFB_OP_RELAX_MIN; }
  static void* state(const device_ops::relax_min& c) { return c.dist.handle(); }
};
template <> struct op_of<device_ops::record> {
  static int op() { return GFB_OP_RECORD; }
  static void* state(const device_ops::record& c) { return c.rec.handle(); }
};
template <> struct op_of<device_ops::always> {
  static int op() { return GFB_OP_ALWAYS; }
  static void* state(const device_ops::always&) { return nullptr; }
};
}  // namespace device_detail

/// Push advance on the device (operators.hpp:35-68).
template <class Cond>
DeviceFrontier neighbors_expand(const DevicePolicy& policy, const Graph& g,
                                const DeviceFrontier& f, Cond&& cond) {
  using C = std::remove_cvref_t<Cond>;
  policy.validate();
  DeviceGraph& dg = DeviceGraph::of(g, policy, g.has_transpose());
  DeviceFrontier out(f.repr(), g.num_vertices(), policy.device);
  device_detail::check(gfb_advance_push(dg.ctx(), dg.handle(), f.handle(), out.handle(),
                                        device_detail::op_of<C>::op(),
                                        device_detail::op_of<C>::state(cond)));
  return out;
}

/// Pull advance on the device (operators.hpp:76-114).
template <class Cond>
DeviceFrontier neighbors_expand_pull(const DevicePolicy& policy, const Graph& g,
                                     const DeviceFrontier& f, Cond&& cond) {
  using C = std::remove_cvref_t<Cond>;
  policy.validate();
  if (!g.has_transpose())  // operators.hpp:79-80
    throw std::invalid_argument("neighbors_expand_pull: transpose not built");
  if (f.repr() != FrontierRepr::dense)  // operators.hpp:81-82
    throw std::invalid_argument("neighbors_expand_pull: dense frontier required");
  DeviceGraph& dg = DeviceGraph::of(g, policy, true);
  DeviceFrontier out(FrontierRepr::dense, g.num_vertices(), policy.device);
  device_detail::check(gfb_advance_pull(dg.ctx(), dg.handle(), f.handle(), out.handle(),
                                        device_detail::op_of<C>::op(),
                                        device_detail::op_of<C>::state(cond)));
  return out;
}

namespace device_detail {
template <class P> struct pred_of {
  static_assert(sizeof(P) == 0,
                "device policy: host predicates cannot run on the device; use "
                "graflow::device_ops::{dist_below, dist_at_least, reached}");
};
template <> struct pred_of<device_ops::dist_below> {
  static int id() { return GFB_PRED_DIST_BELOW; }
  static gfb_dist* dist(const device_ops::dist_below& p) { return p.dist.handle(); }
  static double thr(const device_ops::dist_below& p) { return p.threshold; }
};
template <> struct pred_of<device_ops::dist_at_least> {
  static int id() { return GFB_PRED_DIST_AT_LEAST; }
  static gfb_dist* dist(const device_ops::dist_at_least& p) { return p.dist.handle(); }
  static double thr(const device_ops::dist_at_least& p) { return p.threshold; }
};
template <> struct pred_of<device_ops::reached> {
  static int id() { return GFB_PRED_REACHED; }
  static gfb_dist* dist(const device_ops::reached& p) { return p.dist.handle(); }
  static double thr(const device_ops::reached&) { return 0.0; }
};
}  // namespace device_detail

/// filter on the device (operators.hpp:163-188): same representation, the
/// sparse input order and duplicates kept.
template <class Pred>
DeviceFrontier filter(const DevicePolicy& policy, const DeviceFrontier& f, Pred&& pred) {
  using P = std::remove_cvref_t<Pred>;
  policy.validate();
  DeviceFrontier out(f.repr(), f.num_vertices(), policy.device);
  device_detail::check(gfb_filter(device_detail::context(policy.device), f.handle(), out.handle(),
                                  device_detail::pred_of<P>::id(),
                                  device_detail::pred_of<P>::dist(pred),
                                  device_detail::pred_of<P>::thr(pred)));
  return out;
}

/// uniquify (operators.hpp:191-200): bitmap dedup + warp-ballot compaction.
inline DeviceFrontier uniquify(const DeviceFrontier& f, int device = 0) {
  if (f.repr() != FrontierRepr::sparse)
    throw std::invalid_argument("uniquify: sparse frontier required");
  DeviceFrontier out(FrontierRepr::sparse, f.num_vertices(), device);
  device_detail::check(gfb_filter_unique(device_detail::context(device), f.handle(), out.handle()));
  return out;
}

}  // namespace graflow

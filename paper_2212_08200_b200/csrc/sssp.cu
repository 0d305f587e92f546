// sssp.cu -- the device SSSP driver: sssp() of algorithms.hpp:134-188 as
// init -> { advance (push | pull) -> filter } until the frontier is empty
// -> predecessor pass, all on one CUDA stream.
//
//   init      algorithms.hpp:141-148 (k_init)
//   advance   neighbors_expand / neighbors_expand_pull with the relax lambda
//             (operators.hpp:35-68 / :76-114, algorithms.hpp:150-158):
//             k_push_range / k_pull_relax (hot.cuh)
//   filter    frontier dedup + distance-ordered plan + far-bucket deferral
//             (frontier.hpp:147-165, operators.hpp:163-200): k_fcount_o,
//             k_fscan_o, k_fwrite_o (frontier.cuh)
//   loop      while (f.size() != 0) (algorithms.hpp:167): a CUDA graph with a
//             conditional WHILE node whose condition k_fscan_o sets
//   tail      small frontiers: one persistent launch with vertex queues
//             (tail.cuh k_tail), entered through an IF node the filter sets
//   preds     repair_predecessors (algorithms.hpp:77-93): k_pred_* (kernels.cuh)
// High-diameter meshes take the near-far loop instead (nearfar.cuh).
#include <cub/cub.cuh>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "frontier.cuh"
#include "hot.cuh"
#include "impl.hpp"
#include "nearfar.cuh"
#include "tail.cuh"

namespace gfb {

static size_t dist_bytes(int wtype) { return wtype == GFB_W_F64 ? 8 : 4; }

// Launch with programmatic stream serialization (PDL) when pdl: the kernel may
// be scheduled while its predecessor drains; it waits (griddepcontrol.wait)
// before reading the predecessor's results.
template <class... KArgs, class... Args>
static void launch_pdl(bool pdl, void (*k)(KArgs...), dim3 grid, dim3 block, cudaStream_t st,
                       Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  GFB_CUDA(cudaLaunchKernelEx(&cfg, k, args...));
}

Workspace* ensure_ws(Graph* g) {
  if (g->ws && g->ws->wtype == g->wtype) return g->ws.get();
  Ctx* c = g->ctx;
  cudaStream_t s = c->stream;
  auto ws = std::make_unique<Workspace>();
  const uint64_t n = g->n, m = g->m;
  const uint64_t nwords = (n + 31) / 32;
  ws->wtype = g->wtype;
  ws->dist.alloc(n * dist_bytes(g->wtype), s);
  ws->predrec.alloc(n * 8, s);
  ws->pred.alloc(n * 4, s);
  ws->res.alloc(n * 4, s);
  ws->cand.alloc(n * 4, s);
  ws->bm_next.alloc(nwords * 4, s);
  ws->bm_cur.alloc(nwords * 4, s);
  ws->repair_bm.alloc(nwords * 4, s);
  ws->pv.alloc((n + 1) * 4, s);
  ws->pstart.alloc((n + 1) * 4, s);
  ws->poff.alloc((n + 1) * 4, s);
  ws->ptseg.alloc((m / PLAN_GRAIN + 3) * 4, s);
  ws->ftiles = (uint32_t)std::max<uint64_t>((nwords + F_WORDS - 1) / F_WORDS, 1);
  ws->agg.alloc((size_t)ws->ftiles * 8, s);  // bfs.cu's plain compaction
  ws->oagg.alloc((size_t)ws->ftiles * (OB_N * 8 + 4), s);  // (tile, bucket) cells + tile flags
  ws->obuck.alloc(2 * OB_N * 8, s);                          // bucket totals | cursors
  GFB_CUDA(cudaMemsetAsync(ws->obuck.p, 0, 2 * OB_N * 8, s));
  ws->src_dev.alloc(16, s);
  ws->ctl.alloc(sizeof(Ctl), s);
  GFB_CUDA(cudaMallocHost(&ws->ctl_host, sizeof(Ctl)));
  g->ws = std::move(ws);
  return g->ws.get();
}

constexpr uint32_t PRED_KEY_ROUNDS = 4;

template <class W>
struct Runner {
  using D = typename DT<W>::D;
  Ctx* c;
  Graph* g;
  Workspace* ws;
  cudaStream_t s;
  uint32_t n, nwords;
  const gfb_sssp_opts* o;
  uint64_t kernels = 0;
  bool rl = false;  // loop runs on the in-degree-relabelled CSR (ensure_relabel)

  // 32-bit distances: packed (dist, pred) keys with fire-and-forget
  // reductions; f64: {u, edge} records written by returning mins (hot.cuh)
  static constexpr bool key_mode() { return sizeof(D) == 4; }

  // Far-bucket deferral (k_fscan_o): in a superstep whose frontier holds
  // >= m/4 edges only the closest distance buckets up to defer_pct % of those
  // edges are expanded; the rest stay pending in the bitmap.  RMAT s24: 3.0 -> 1.27
  // relaxations per reached edge (sweep 1-95 %, thresholds m/2..m/64:
  // DESIGN.md §4).
  uint32_t defer_pct() const { return o->defer_pct ? (uint32_t)o->defer_pct : DEFER_PCT; }
  uint32_t defer_min() const { return (uint32_t)(g->m >> 2); }
  bool pullable(int dir) const { return g->has_csc && dir != GFB_DIR_PUSH; }

  const uint32_t* lro() const { return rl ? g->rl_ro.as<uint32_t>() : g->ro.as<uint32_t>(); }
  D* ldist() const { return rl ? ws->dist_int.as<D>() : ws->dist.as<D>(); }
  uint2* lpred() const { return rl ? ws->pkey_int.as<uint2>() : ws->predrec.as<uint2>(); }

  Plan plan() const {
    return Plan{ws->pv.as<uint32_t>(), ws->pstart.as<uint32_t>(), ws->poff.as<uint32_t>(),
                ws->ptseg.as<uint32_t>(), (uint32_t)(ws->ptseg.bytes / 4)};
  }
  Plan pull_plan() const {
    return Plan{g->pull_v.as<uint32_t>(), g->pull_off.as<uint32_t>(), g->pull_off.as<uint32_t>(),
                g->pull_tseg.as<uint32_t>(), (uint32_t)(g->pull_tseg.bytes / 4)};
  }
  AdvArgs<W> args(bool pull) const {
    AdvArgs<W> a{};
    a.adj = pull ? g->cadj.as<EdgeRec<W>>()
                 : (rl ? g->rl_adj.as<EdgeRec<W>>() : g->adj.as<EdgeRec<W>>());
    a.ceid = g->ceid.as<uint32_t>();
    a.dist = ldist();
    a.predrec = lpred();
    a.plan = pull ? pull_plan() : plan();
    a.ctl = ws->ctl.as<Ctl>();
    a.bm_out = ws->bm_next.as<uint32_t>();
    a.bm_in = ws->bm_cur.as<uint32_t>();
    a.status = nullptr;
    a.status_len = 0;
    a.op = GFB_OP_RELAX_MIN;
    return a;
  }

  // frontier filter (frontier.cuh): count per (tile, distance bucket) ->
  // bucket cursors, deferral cut, plan totals (+ loop / direction decision)
  // -> write the distance-ordered plan; deferred vertices stay in the bitmap
  // The scan and write passes are launched with programmatic stream
  // serialization (PDL): each is scheduled while its predecessor drains and
  // waits (griddepcontrol.wait) before reading its results -- s24 3.35-3.36 ->
  // 3.34 ms, s22 1.164 -> 1.151 ms; the count pass behind the advance gains
  // nothing more.  Not in the traced host loop (its events split the passes).
  void compact(cudaStream_t st, int dir, float alpha, cudaGraphConditionalHandle hloop,
               cudaGraphConditionalHandle hmode, bool set_loop, bool set_mode,
               cudaEvent_t* split = nullptr, cudaGraphConditionalHandle htail = {},
               bool set_tail = false) {
    const uint32_t tiles = ws->ftiles;
    unsigned long long* bt = ws->obuck.as<unsigned long long>();
    unsigned long long* cells = ws->oagg.as<unsigned long long>();
    uint32_t* tflag = reinterpret_cast<uint32_t*>(cells + (size_t)tiles * OB_N);
    k_fcount_o<D><<<tiles, F_WARPS * 32, 0, st>>>(lro(), ws->bm_next.as<uint32_t>(), nwords,
                                                  ldist(), ws->ctl.as<Ctl>(), cells, bt, tflag);
    if (split) GFB_CUDA(cudaEventRecord(split[0], st));
    launch_pdl(!split, k_fscan_o, dim3(1), dim3(32), st, bt, bt + OB_N, plan(),
               ws->ctl.as<Ctl>(), (uint32_t)g->m, alpha, dir == GFB_DIR_AUTO && g->has_csc ? 1 : 0,
               dir == GFB_DIR_PULL ? 1 : 0, hloop, hmode, set_loop ? 1 : 0, set_mode ? 1 : 0,
               defer_pct(), defer_min(), htail, set_tail ? 1 : 0, tail_edges(dir));
    if (split) GFB_CUDA(cudaEventRecord(split[1], st));
    launch_pdl(!split, k_fwrite_o<D, false>, dim3(tiles), dim3(F_WARPS * 32), st,
               lro(), ws->bm_next.as<uint32_t>(), ws->bm_cur.as<uint32_t>(), nwords,
               (const D*)ldist(), (const Ctl*)ws->ctl.as<Ctl>(),
               (const unsigned long long*)cells, bt + OB_N, plan(), (const uint32_t*)tflag,
               (uint32_t*)nullptr, (uint32_t*)nullptr);
    GFB_CUDA(cudaGetLastError());
    kernels += 3;
  }

  void pull_launch(cudaStream_t st) {
    uint32_t ntiles = (g->pull_total + HotCfg<W>::TILE - 1) / HotCfg<W>::TILE;
    uint32_t grid = std::min<uint32_t>(std::max<uint32_t>(ntiles, 1), c->num_sms * 4);
    if constexpr (key_mode()) {
      k_pull_relax<W, true><<<grid, H_BLOCK, 0, st>>>(args(true), g->pull_total, g->pull_k);
    } else {
      k_pull_relax<W, false><<<grid, H_BLOCK, 0, st>>>(args(true), g->pull_total, g->pull_k);
    }
    ++kernels;
  }

  // Tail kernel threshold (tail.cuh): push-only loops on the BSP driver; a
  // plan below it with nothing deferred hands over.
  uint32_t tail_edges(int dir) const {
    if (pullable(dir) || o->tail_edges < 0) return 0;
    if (o->tail_edges > 0) return (uint32_t)o->tail_edges;
    return (uint32_t)std::max<uint64_t>(g->m >> 8, 4096);
  }
  // queues + grid size (outside any stream capture)
  void tail_prepare() {
    {
      if (ws->tq.bytes < (size_t)n * 8 + 8) {
        invalidate_loop_graphs(g);
        ws->tq.alloc((size_t)n * 8 + 8, s);
        ws->tctr.alloc(64, s);
      }
      if (!ws->tail_grid) {
        int per_sm = 0;
        GFB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tail<W>, TL_THREADS, 0));
        if (per_sm <= 0) fail(GFB_ECUDA, "sssp: tail kernel does not fit an SM");
        ws->tail_grid = std::min(per_sm, 2) * c->num_sms;
      }
    }
  }
  void tail_launch(cudaStream_t st, cudaGraphConditionalHandle hloop, bool set_loop) {
    {
      TailArgs<W> t{};
      t.a = args(false);
      t.ro = lro();
      t.q[0] = ws->tq.as<uint32_t>();
      t.q[1] = t.q[0] + n;
      t.qcnt = ws->tctr.as<uint32_t>();
      t.cell = reinterpret_cast<unsigned long long*>(ws->tctr.as<char>() + 16);
      t.bm[0] = ws->bm_next.as<uint32_t>();
      t.bm[1] = ws->bm_cur.as<uint32_t>();
      t.nwords = nwords;
      // hand back at twice the entry threshold (hysteresis: no ping-pong)
      t.tmax = 2 * tail_edges(GFB_DIR_PUSH);
      t.hloop = hloop;
      t.set_loop = set_loop ? 1 : 0;
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(ws->tail_grid);
      cfg.blockDim = dim3(TL_THREADS);
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeCooperative;
      at[0].val.cooperative = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      GFB_CUDA(cudaLaunchKernelEx(&cfg, k_tail<W>, t));
      ++kernels;
    }
  }

  // The push advance (hot.cuh k_push_range): 6 x 256-thread CTAs per SM,
  // strided edge tiles, PTX red.*, the next chunk's records in flight while
  // the current one gathers (OPT 16).  Measured at RMAT s24 / s22
  // (profiles/r01_variants_s24.txt): 128 / 256 / 512-edge tiles 3.91 / 3.86 /
  // 3.94 ms at s24, 1.27 / 1.31 / 1.35 at s22; one edge per lane 3.81 / 1.24
  // vs two 3.85 / 1.27; pipelined at 6 CTAs/SM 3.72 -> 3.55 ms
  // (profiles/r02_advance_variants.txt).  f64 (record mode): <2 edges/lane,
  // 6 CTAs/SM> (<1,8> 5.94, <2,6> 5.82, <4,4> 6.29 ms without predecessors).
  int tile() const {
    if (o->advance_tile) return o->advance_tile;
    return g->m <= (1ull << 27) ? 128 : 256;
  }
  void push(cudaStream_t st) {
    if constexpr (key_mode()) {
      if (tile() == 128)
        k_push_range<W, 1, 6, 128, 17><<<c->num_sms * 6, 256, 0, st>>>(args(false));
      else
        k_push_range<W, 1, 6, 256, 17><<<c->num_sms * 6, 256, 0, st>>>(args(false));
    } else {
      // f64 record mode, pipelined like the 4-byte path: 5.57 -> 5.37 ms at s24
      k_push_range<W, 1, 6, 256, 17, false, true><<<c->num_sms * 6, 256, 0, st>>>(args(false));
    }
    ++kernels;
  }

  // Near-far filter (delta > 0): one persistent launch (nearfar.cuh).  8
  // queue entries per warp (one edge per lane on degree-4 meshes) and
  // warp-local chasing of 8 rounds (4096^2 grid: 32 entries/warp, 4 rounds,
  // delta 32: 55 ms; 8/8, delta 16: 31.8 ms; profiles/r01_nearfar_chunk.txt).
  // Rows longer than NF_HEAVY edges are expanded by a whole CTA in the next
  // phase (RMAT s24, delta = inf: 212 -> 36 ms); compiled out otherwise.
  bool nearfar_launch(double delta) {
    const bool hv = max_out_degree(g) > NF_HEAVY;
    auto kern = hv ? k_nearfar<W, 8, 8, true> : k_nearfar<W, 8, 8>;
    int per_sm = 0;
    GFB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NF_THREADS, 0));
    if (per_sm <= 0) return false;
    const uint32_t grid = (uint32_t)std::min(per_sm, 2) * c->num_sms;
    // queue capacity: every activation appends one entry; a phase can
    // activate at most min(m, n x in-degree) vertices -- size for 2n or m/4
    const uint64_t cap64 = std::min<uint64_t>(std::max<uint64_t>(2ull * n, g->m / 4), 0xFFFFFFF0ull);
    const uint32_t cap = (uint32_t)cap64;
    const uint32_t hcap = (uint32_t)std::min<uint64_t>(g->m / NF_HEAVY + 4096, 0xFFFFFFF0ull);
    const size_t qbytes = (size_t)cap * 32 + (size_t)hcap * 16;
    if (ws->nf_q.bytes < qbytes) {
      ws->nf_q.alloc(qbytes, s);
      ws->nf_cnt.alloc(64, s);
    }
    NfArgs<W> a{};
    a.ro = g->ro.as<uint32_t>();
    a.adj = g->adj.as<EdgeRec<W>>();
    a.dist = ws->dist.as<D>();
    a.pkey = ws->predrec.as<unsigned long long>();
    uint2* q = ws->nf_q.as<uint2>();
    a.nq[0] = q;
    a.nq[1] = q + cap;
    a.fq[0] = q + 2 * (size_t)cap;
    a.fq[1] = q + 3 * (size_t)cap;
    a.hq[0] = q + 4 * (size_t)cap;
    a.hq[1] = q + 4 * (size_t)cap + hcap;
    a.hcap = hcap;
    a.cap = cap;
    a.cnt = ws->nf_cnt.as<uint32_t>();
    a.fmin64 = reinterpret_cast<unsigned long long*>(ws->nf_cnt.as<uint32_t>() + 10);
    a.ctl = ws->ctl.as<Ctl>();
    a.src_ptr = ws->src_dev.as<uint32_t>();
    a.n = n;
    a.nwords = nwords;
    if constexpr (std::is_same<D, float>::value) a.delta = (float)delta;
    else if constexpr (std::is_same<D, double>::value) a.delta = delta;
    else a.delta = std::isinf(delta) ? (D)0xFFFFFFFEu  // the queue model: no far set
                                     : (D)std::min(std::max(std::llround(delta), 1ll), 0xFFFFFFFEll);
    TBuf trace;
    if (o->trace) {
      a.trace_cap = 1u << 16;
      trace.alloc((size_t)a.trace_cap * 8, s);
      GFB_CUDA(cudaMemsetAsync(trace.p, 0, (size_t)a.trace_cap * 8, s));
      a.trace = trace.as<unsigned long long>();
    }
    void* params[] = {&a};
    GFB_CUDA(cudaLaunchCooperativeKernel((const void*)kern, grid, NF_THREADS, params, 0, s));
    kernels += 1;
    if (a.trace) {  // phase histogram (diagnostics only)
      std::vector<unsigned long long> h(a.trace_cap);
      GFB_CUDA(cudaMemcpyAsync(h.data(), trace.p, h.size() * 8, cudaMemcpyDeviceToHost, s));
      c->sync();
      uint32_t np = 0;
      while (np + 1 < a.trace_cap && h[np + 1]) ++np;
      double buck_us[8] = {0}, buck_n[8] = {0};
      for (uint32_t i = 0; i + 1 <= np; ++i) {
        const double us = ((h[i + 1] >> 24) - (h[i] >> 24)) * 1e-3;
        const uint32_t K = (uint32_t)(h[i] & 0xFFFFFF);
        int b = 0;
        for (uint32_t x = K; x >= 16 && b < 7; x >>= 3) ++b;  // 0:<16 1:<128 2:<1K ...
        buck_us[b] += us;
        buck_n[b] += 1;
      }
      for (int b = 0; b < 8; ++b)
        if (buck_n[b] > 0)
          fprintf(stderr, "[gfb nearfar] K < %8u: %6.0f phases, %8.1f us total, %6.2f us/phase\n",
                  16u << (3 * b), buck_n[b], buck_us[b], buck_us[b] / buck_n[b]);
    }
    return true;
  }

  void init_launch(cudaStream_t st) {
    k_init<W><<<stride_grid(c), 256, 0, st>>>(ldist(), lpred(), ws->bm_next.as<uint32_t>(),
                                              ws->bm_cur.as<uint32_t>(), n, nwords,
                                              ws->src_dev.as<uint32_t>(), ws->ctl.as<Ctl>());
    ++kernels;
  }

  // ---- device loop: init; filter; WHILE(k > 0) { IF(pull) pull ELSE push;
  //      filter }  captured once into a CUDA graph (conditional nodes).  The
  //      graph holds raw pointers into the graph's / workspace's buffers:
  //      every reallocation of those destroys it (invalidate_loop_graphs).
  void build_loop_graph(int dir, float alpha) {
    if (tail_edges(dir) > 0) tail_prepare();
    invalidate_loop_graphs(g);
    for (auto& a : c->aux)
      if (!a) GFB_CUDA(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking));
    cudaGraph_t G;
    GFB_CUDA(cudaGraphCreate(&G, 0));
    // a handle belongs to the graph holding its conditional node: hloop to
    // the top-level graph, hmode to the loop body (created below)
    cudaGraphConditionalHandle hloop, hmode{};
    GFB_CUDA(cudaGraphConditionalHandleCreate(&hloop, G, 1, cudaGraphCondAssignDefault));
    const bool pull_ok = pullable(dir);

    GFB_CUDA(cudaStreamBeginCaptureToGraph(s, G, nullptr, nullptr, 0,
                                           cudaStreamCaptureModeRelaxed));
    init_launch(s);
    compact(s, dir, alpha, hloop, hmode, true, false);
    cudaStreamCaptureStatus cst;
    cudaGraph_t capG;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    GFB_CUDA(cudaStreamGetCaptureInfo(s, &cst, nullptr, &capG, &deps, &ndeps));
    cudaGraphNodeParams wp{};
    wp.type = cudaGraphNodeTypeConditional;
    wp.conditional.handle = hloop;
    wp.conditional.type = cudaGraphCondTypeWhile;
    wp.conditional.size = 1;
    cudaGraphNode_t wnode;
    GFB_CUDA(cudaGraphAddNode(&wnode, capG, deps, ndeps, &wp));
    cudaGraph_t body = wp.conditional.phGraph_out[0];
    GFB_CUDA(cudaStreamUpdateCaptureDependencies(s, &wnode, 1, cudaStreamSetCaptureDependencies));
    cudaGraph_t tmp;
    GFB_CUDA(cudaStreamEndCapture(s, &tmp));

    // loop body
    if (pull_ok)  // first iteration expands {source}: push unless pull is forced
      GFB_CUDA(cudaGraphConditionalHandleCreate(&hmode, body, dir == GFB_DIR_PULL ? 1 : 0,
                                                cudaGraphCondAssignDefault));
    cudaStream_t b = c->aux[0];
    GFB_CUDA(cudaStreamBeginCaptureToGraph(b, body, nullptr, nullptr, 0,
                                           cudaStreamCaptureModeRelaxed));
    if (pull_ok) {
      GFB_CUDA(cudaStreamGetCaptureInfo(b, &cst, nullptr, &capG, &deps, &ndeps));
      cudaGraphNodeParams ip{};
      ip.type = cudaGraphNodeTypeConditional;
      ip.conditional.handle = hmode;
      ip.conditional.type = cudaGraphCondTypeIf;
      ip.conditional.size = 2;  // [0]: mode != 0 (pull), [1]: else (push)
      cudaGraphNode_t inode;
      GFB_CUDA(cudaGraphAddNode(&inode, capG, deps, ndeps, &ip));
      cudaGraph_t gpull = ip.conditional.phGraph_out[0], gpush = ip.conditional.phGraph_out[1];
      GFB_CUDA(cudaStreamUpdateCaptureDependencies(b, &inode, 1, cudaStreamSetCaptureDependencies));
      cudaStream_t x = c->aux[1];
      GFB_CUDA(cudaStreamBeginCaptureToGraph(x, gpull, nullptr, nullptr, 0,
                                             cudaStreamCaptureModeRelaxed));
      pull_launch(x);
      GFB_CUDA(cudaStreamEndCapture(x, &tmp));
      GFB_CUDA(cudaStreamBeginCaptureToGraph(x, gpush, nullptr, nullptr, 0,
                                             cudaStreamCaptureModeRelaxed));
      push(x);
      GFB_CUDA(cudaStreamEndCapture(x, &tmp));
    } else {
      push(b);
    }
    const bool tail_ok = tail_edges(dir) > 0;
    cudaGraphConditionalHandle htail{};
    if (tail_ok)
      GFB_CUDA(cudaGraphConditionalHandleCreate(&htail, body, 0, cudaGraphCondAssignDefault));
    compact(b, dir, alpha, hloop, hmode, true, pull_ok, nullptr, htail, tail_ok);
    if (tail_ok) {  // IF(tail) { k_tail } -- the rest of the run in one launch
      GFB_CUDA(cudaStreamGetCaptureInfo(b, &cst, nullptr, &capG, &deps, &ndeps));
      cudaGraphNodeParams tp{};
      tp.type = cudaGraphNodeTypeConditional;
      tp.conditional.handle = htail;
      tp.conditional.type = cudaGraphCondTypeIf;
      tp.conditional.size = 1;
      cudaGraphNode_t tnode;
      GFB_CUDA(cudaGraphAddNode(&tnode, capG, deps, ndeps, &tp));
      cudaGraph_t gtail = tp.conditional.phGraph_out[0];
      GFB_CUDA(cudaStreamUpdateCaptureDependencies(b, &tnode, 1, cudaStreamSetCaptureDependencies));
      cudaStream_t x = c->aux[1];
      GFB_CUDA(cudaStreamBeginCaptureToGraph(x, gtail, nullptr, nullptr, 0,
                                             cudaStreamCaptureModeRelaxed));
      tail_launch(x, hloop, true);
      GFB_CUDA(cudaStreamEndCapture(x, &tmp));
    }
    GFB_CUDA(cudaStreamEndCapture(b, &tmp));
    GFB_CUDA(cudaGraphInstantiate(&ws->loop_exec, G, 0));
    ws->loop_graph = G;
  }

  void run(uint32_t source, gfb_sssp_stats* st) {
    ws->has_result = false;
    const int dir = o->direction;
    const float alpha = o->pull_alpha > 0 ? o->pull_alpha : 0.25f;
    // Default configuration on a low-degree mesh (max out-degree <= 8, e.g.
    // grids and road networks: thousands of BSP supersteps): the near-far
    // loop with delta = 32 x the mean edge weight (the 4096^2 grid's tuned
    // value: 570 -> 32 ms).  Same fixpoint; loop = BSP keeps the BSP loop.
    double delta = o->delta;
    if (delta == 0 && o->loop == GFB_LOOP_AUTO && dir != GFB_DIR_PULL && n >= (1u << 16) &&
        max_out_degree(g) <= 8 && g->m >= n) {
      const double mw = mean_weight(g);
      if (mw > 0) delta = 32.0 * mw;
    }
    // The in-degree-relabelled CSR has no CSC: only when no superstep can
    // pull (AUTO pulls when frontier edges > m / alpha, impossible for
    // alpha <= 1).  Automatic for graphs with >= 2^20 vertices from the
    // second SSSP on the same contents on (the copy costs ~6 ms at s24 and
    // saves ~0.3 ms per call: it pays on reuse, not for a one-shot upload +
    // SSSP); skipped when in-degrees are not skewed (ensure_relabel).
    const bool reuse = g->runs_since_fill++ > 0 || g->rl_valid;
    const bool rl_dir = dir == GFB_DIR_PUSH || (dir == GFB_DIR_AUTO && (alpha <= 1.0f || !g->has_csc));
    rl = delta <= 0 && rl_dir &&
         (o->relabel == GFB_RELABEL_ON ||
          (o->relabel == GFB_RELABEL_AUTO && n >= (1u << 20) && reuse));
    if (rl) {
      ensure_relabel(g);
      rl = !g->rl_skip;
    }
    if (rl && ws->dist_int.bytes < (size_t)n * sizeof(D)) {
      ws->dist_int.alloc((size_t)n * sizeof(D), s);
      ws->pkey_int.alloc((size_t)n * 8, s);
      invalidate_loop_graphs(g);
    }
    // source -> device (the graph launches stay source-agnostic)
    GFB_CUDA(cudaMemcpyAsync(ws->src_dev.p, &source, 4, cudaMemcpyHostToDevice, s));
    if (rl)
      GFB_CUDA(cudaMemcpyAsync(ws->src_dev.p, g->rl_perm.as<uint32_t>() + source, 4,
                               cudaMemcpyDeviceToDevice, s));
    uint64_t launches = 0;
    float adv_ms = 0;
    GFB_CUDA(cudaEventRecord(c->ev[0], s));
    bool done = false;
    if (delta > 0 && !rl) {
      if (dir == GFB_DIR_PULL) fail(GFB_EINVAL, "sssp: the near-far filter (delta > 0) is push-only");
      done = nearfar_launch(delta);
      if (done && (c->read_ctl(ws->ctl.as<Ctl>()).err & 2u)) done = false;  // queue overflow: BSP
    }
    if (done) {
    } else if (o->device_loop) {
      // the graph's key: everything its captured launches depend on
      const int key[6] = {dir, (int)(alpha * 1000), rl ? 1 : 0, (int)defer_pct(), tile(),
                          (int)tail_edges(dir)};
      if (!ws->loop_exec || memcmp(key, ws->loop_key, sizeof(key)) != 0) {
        GFB_CUDA(cudaStreamSynchronize(s));
        build_loop_graph(dir, alpha);
        memcpy(ws->loop_key, key, sizeof(key));
        GFB_CUDA(cudaEventRecord(c->ev[0], s));
      }
      GFB_CUDA(cudaGraphLaunch(ws->loop_exec, s));
    } else {
      cudaGraphConditionalHandle none{};
      init_launch(s);
      compact(s, dir, alpha, none, none, false, false);
      for (;;) {
        Ctl h = c->read_ctl(ws->ctl.as<Ctl>());
        if (h.err & 1u) fail(GFB_ERANGE, "sssp: u32 distance overflow (use f64 weights)");
        if (h.tail == 1 && tail_edges(dir) > 0) {  // the rest of the run in one launch
          tail_prepare();
          GFB_CUDA(cudaEventRecord(c->ev[2], s));
          tail_launch(s, none, false);
          GFB_CUDA(cudaEventRecord(c->ev[3], s));
          ++launches;
          h = c->read_ctl(ws->ctl.as<Ctl>());
          float tms = 0;  // the tail's supersteps count as advance time (their filter included)
          GFB_CUDA(cudaEventElapsedTime(&tms, c->ev[2], c->ev[3]));
          adv_ms += tms;
          if (o->trace)
            fprintf(stderr, "[gfb] tail kernel: %u supersteps so far, %s\n", h.supersteps,
                    h.tail == 2 ? "handed back (plan above 2 x tail_edges)" : "converged");
          if (h.tail != 2) break;
          compact(s, dir, alpha, none, none, false, false);

          continue;
        }
        if (h.k == 0) break;
        GFB_CUDA(cudaEventRecord(c->ev[2], s));
        if (h.mode == 1) pull_launch(s);
        else push(s);
        GFB_CUDA(cudaEventRecord(c->ev[3], s));
        GFB_CUDA(cudaGetLastError());
        compact(s, dir, alpha, none, none, false, false, o->trace ? &c->ev[5] : nullptr);
        GFB_CUDA(cudaEventRecord(c->ev[4], s));
        ++launches;
        GFB_CUDA(cudaEventSynchronize(c->ev[4]));
        float ms = 0, fms = 0;
        GFB_CUDA(cudaEventElapsedTime(&ms, c->ev[2], c->ev[3]));
        GFB_CUDA(cudaEventElapsedTime(&fms, c->ev[3], c->ev[4]));
        adv_ms += ms;
        if (o->trace) {  // filter split: count | scan | write; bitmap = placed + deferred
          float f0 = 0, f1 = 0;
          GFB_CUDA(cudaEventElapsedTime(&f0, c->ev[3], c->ev[5]));
          GFB_CUDA(cudaEventElapsedTime(&f1, c->ev[5], c->ev[6]));
          fprintf(stderr, "[gfb] superstep %llu %s frontier=%u edges=%u advance=%.3f ms (%.1f G edges/s) "
                  "filter=%.3f ms (count %.3f scan %.3f write %.3f) bitmap=%u/%u tail=%u\n",
                  (unsigned long long)launches, h.mode ? "pull" : "push", h.k, h.total, ms,
                  (h.mode ? g->pull_total : h.total) / (ms * 1e-3) / 1e9, fms, f0, f1,
                  fms - f0 - f1, h.k_all, h.t_all, h.tail);
        }
      }
    }
    uint64_t fallback = 0;
    if (o->trace) GFB_CUDA(cudaEventRecord(c->ev[4], s));
    pred_pass(source, o->compute_pred != 0, &fallback);  // records ev[1]
    if (o->trace) {
      float pms = 0;
      GFB_CUDA(cudaEventSynchronize(c->ev[1]));
      GFB_CUDA(cudaEventElapsedTime(&pms, c->ev[4], c->ev[1]));
      fprintf(stderr, "[gfb] predecessor pass %.3f ms (fallback %llu)\n", pms,
              (unsigned long long)fallback);
    }
    Ctl h = c->read_ctl(ws->ctl.as<Ctl>());
    if (h.err & 1u) fail(GFB_ERANGE, "sssp: u32 distance overflow (use f64 weights)");
    float ms = 0;
    GFB_CUDA(cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]));
    if (o->device_loop && !done) kernels += 4 + 4ull * h.supersteps;  // graph launches
    ws->has_result = true;
    ws->source = source;
    if (st) {
      st->supersteps = h.supersteps;
      st->relaxations = h.relax;
      st->n_reach = h.n_reach;
      st->m_reach = h.m_reach;
      st->push_steps = h.push_steps;
      st->pull_steps = h.pull_steps;
      st->pred_fallback = fallback;
      st->device_ms = ms;
      st->advance_ms = adv_ms;
      st->advance_launches = o->device_loop ? h.supersteps : launches;
      st->kernel_launches = kernels;
    }
  }

  void pred_pass(uint32_t source, bool want, uint64_t* fallback) {
    GFB_CUDA(cudaMemsetAsync(ws->repair_bm.p, 0, (size_t)nwords * 4, s));
    GFB_CUDA(cudaMemsetAsync(&ws->ctl.as<Ctl>()->flag, 0, 4, s));
    auto verify = k_pred_verify<W, false, false>;
    PermView<D> pv{};
    if constexpr (key_mode()) {
      verify = rl ? k_pred_verify<W, true, true> : k_pred_verify<W, true, false>;
    } else {
      if (rl) verify = k_pred_verify<W, false, true>;  // f64 records, relabelled loop
    }
    if (rl)  // back to the caller's ids, fused into the verification
      pv = PermView<D>{g->rl_perm.as<uint32_t>(), g->rl_iperm.as<uint32_t>(),
                       ws->dist_int.as<D>(), ws->pkey_int.as<unsigned long long>(),
                       ws->dist.as<D>(), nullptr /* keys stay in loop ids */, g->rl_adj.p};
    verify<<<c->num_sms * 8, 256, 0, s>>>(
        g->ro.as<uint32_t>(), g->adj.as<EdgeRec<W>>(),
        g->has_csc ? g->co.as<uint32_t>() : nullptr,
        g->has_csc ? g->cadj.as<EdgeRec<W>>() : nullptr, ws->dist.as<D>(),
        ws->predrec.as<uint2>(), ws->pred.as<uint32_t>(), ws->res.as<uint32_t>(),
        ws->repair_bm.as<uint32_t>(), ws->cand.as<uint32_t>(), n, source, ws->ctl.as<Ctl>(), pv);
    GFB_CUDA(cudaGetLastError());
    ++kernels;
    // ev[1] = the end of the device work, recorded before every host read of
    // the control block (the decision to continue is host-side; the SSSP's
    // device time does not include that round trip)
    if (!want) {
      GFB_CUDA(cudaEventRecord(c->ev[1], s));
      return;
    }
    Ctl* dctl = ws->ctl.as<Ctl>();
    // key rounds first (no in-edge scan), queued in batches of
    // PRED_KEY_ROUNDS with one host read per batch; long zero-weight tie
    // chains (u32 weights) take more batches while they make progress
    uint32_t base = 0;
    Ctl h = {};
    uint64_t left = 0;
    for (uint32_t done_before = 0;;) {
      if constexpr (key_mode()) {
        for (uint32_t k = base + 1; k <= base + PRED_KEY_ROUNDS; ++k)
          k_pred_key_round<W><<<c->num_sms, 256, 0, s>>>(
              ws->cand.as<uint32_t>(),
              rl ? ws->pkey_int.as<unsigned long long>() : ws->predrec.as<unsigned long long>(),
              ws->dist.as<D>(), ws->pred.as<uint32_t>(), ws->res.as<uint32_t>(),
              ws->repair_bm.as<uint32_t>(), k, dctl,
              rl ? g->rl_perm.as<uint32_t>() : nullptr, rl ? g->rl_iperm.as<uint32_t>() : nullptr);
        GFB_CUDA(cudaGetLastError());
        kernels += PRED_KEY_ROUNDS;
        base += PRED_KEY_ROUNDS;
      }
      GFB_CUDA(cudaEventRecord(c->ev[1], s));
      h = c->read_ctl(dctl);
      *fallback = h.unresolved;
      left = h.unresolved - std::min(h.unresolved, h.resolved);
      if (left == 0 || !key_mode() || h.resolved == done_before || base >= 64) break;
      done_before = h.resolved;
    }
    if (left == 0) return;
    // in-edge rounds: res values continue above the key rounds' (base)
    if (g->has_csc) {
      const uint32_t grid = c->num_sms * 8;
      for (uint32_t round = 1; left > 0; ++round) {
        GFB_CUDA(cudaMemsetAsync(&dctl->flag, 0, 4, s));
        k_pred_csc_block<W><<<grid, 256, 0, s>>>(
            g->co.as<uint32_t>(), g->cadj.as<EdgeRec<W>>(), ws->dist.as<D>(),
            ws->pred.as<uint32_t>(), ws->res.as<uint32_t>(), ws->cand.as<uint32_t>(), round, dctl,
            base);
        GFB_CUDA(cudaGetLastError());
        ++kernels;
        GFB_CUDA(cudaEventRecord(c->ev[1], s));
        Ctl r = c->read_ctl(dctl);
        // round 1 (strict edges) may resolve nothing when every unresolved
        // vertex sits in a zero-weight tie class; later rounds must progress
        if (r.flag == 0 && round > 1) fail(GFB_ELOGIC, "sssp: predecessor repair made no progress");
        left -= std::min<uint64_t>(left, r.flag);
      }
      return;
    }
    // no transpose: collect the unresolved vertices' in-edges in one CSR pass,
    // then run the rounds over that list
    uint32_t cap = (uint32_t)std::min<uint64_t>(g->m + 1, 1u << 22);
    TBuf list, big;
    big.alloc((size_t)n * 4 + 4, s);
    for (int attempt = 0;; ++attempt) {  // a second pass with the exact size on overflow
      list.alloc((size_t)cap * 16, s);
      GFB_CUDA(cudaMemsetAsync(&dctl->out_count, 0, 8, s));  // out_count, rec_count
      GFB_CUDA(cudaMemsetAsync(&dctl->err, 0, 4, s));
      if (h.unresolved <= PR_FLAT_MAX) {  // few: one flat pass screened by a shared filter
        k_pred_inedges_flat<W><<<c->num_sms * 8, 256, 0, s>>>(
            g->ro.as<uint32_t>(), g->adj.as<EdgeRec<W>>(), n, g->m,
            ws->repair_bm.as<uint32_t>(), ws->cand.as<uint32_t>(), list.as<uint4>(), cap, dctl);
        kernels += 1;
      } else {
        k_pred_inedges<W><<<stride_grid(c), 256, 0, s>>>(
            g->ro.as<uint32_t>(), g->adj.as<EdgeRec<W>>(), ws->repair_bm.as<uint32_t>(), n,
            list.as<uint4>(), cap, big.as<uint32_t>(), dctl);
        k_pred_inedges_big<W><<<stride_grid(c), 256, 0, s>>>(
            g->ro.as<uint32_t>(), g->adj.as<EdgeRec<W>>(), ws->repair_bm.as<uint32_t>(),
            list.as<uint4>(), cap, big.as<uint32_t>(), dctl);
        kernels += 2;
      }
      GFB_CUDA(cudaEventRecord(c->ev[1], s));
      const Ctl r = c->read_ctl(dctl);
      if (!(r.err & 4u)) break;
      if (attempt > 0) fail(GFB_ELOGIC, "sssp: predecessor repair list overflow");
      cap = r.out_count;  // every in-edge was counted, stored or not
    }
    GFB_CUDA(cudaMemsetAsync(ws->cand.p, 0xFF, (size_t)n * 4, s));
    for (uint32_t round = 1; left > 0; ++round) {
      GFB_CUDA(cudaMemsetAsync(&dctl->flag, 0, 4, s));
      k_pred_list_round<W><<<stride_grid(c), 256, 0, s>>>(list.as<uint4>(), dctl, cap,
                                                          ws->dist.as<D>(), ws->res.as<uint32_t>(),
                                                          ws->cand.as<uint32_t>(), round, base);
      k_pred_apply<<<stride_grid(c), 256, 0, s>>>(ws->cand.as<uint32_t>(), ws->pred.as<uint32_t>(),
                                                  ws->res.as<uint32_t>(),
                                                  ws->repair_bm.as<uint32_t>(), n, round, dctl,
                                                  base);
      GFB_CUDA(cudaGetLastError());
      kernels += 2;
      GFB_CUDA(cudaEventRecord(c->ev[1], s));
      Ctl r = c->read_ctl(dctl);
      if (r.err & 4u) fail(GFB_ELOGIC, "sssp: predecessor repair list overflow");
      if (r.flag == 0 && round > 1)
        fail(GFB_ELOGIC, "sssp: predecessor repair made no progress");
      left -= std::min<uint64_t>(left, r.flag);
    }
  }
};

void sssp_run(Ctx* c, Graph* g, uint32_t source, const gfb_sssp_opts* o, gfb_sssp_stats* st) {
  check_usable(g);
  if (source >= g->n) fail(GFB_ERANGE, "sssp: source out of range");  // algorithms.hpp:137
  if (o->direction == GFB_DIR_PULL && !g->csc_wanted)                  // algorithms.hpp:138-139
    fail(GFB_EINVAL, "sssp: pull direction requires a built transpose");
  if (o->direction < GFB_DIR_PUSH || o->direction > GFB_DIR_AUTO)
    fail(GFB_EINVAL, "sssp: bad direction");
  if (o->loop < GFB_LOOP_AUTO || o->loop > GFB_LOOP_BSP) fail(GFB_EINVAL, "sssp: bad loop");
  if (o->relabel < GFB_RELABEL_AUTO || o->relabel > GFB_RELABEL_OFF)
    fail(GFB_EINVAL, "sssp: bad relabel");
  if (o->defer_pct < 0 || o->defer_pct > 100) fail(GFB_EINVAL, "sssp: defer_pct must be 0..100");
  if (o->advance_tile != 0 && o->advance_tile != 128 && o->advance_tile != 256)
    fail(GFB_EINVAL, "sssp: advance_tile must be 0, 128 or 256");
  // the transpose only when a superstep can pull (AUTO pulls when frontier
  // edges exceed m / alpha: impossible for alpha <= 1)
  const float alpha = o->pull_alpha > 0 ? o->pull_alpha : 0.25f;
  if (o->direction == GFB_DIR_PULL || (o->direction == GFB_DIR_AUTO && alpha > 1.0f &&
                                       o->delta <= 0))
    ensure_csc(g);
  Workspace* ws = ensure_ws(g);
  const uint32_t n = (uint32_t)g->n, nw = (uint32_t)((g->n + 31) / 32);
  if (g->wtype == GFB_W_F32) Runner<float>{c, g, ws, c->stream, n, nw, o}.run(source, st);
  else if (g->wtype == GFB_W_F64) Runner<double>{c, g, ws, c->stream, n, nw, o}.run(source, st);
  else Runner<uint32_t>{c, g, ws, c->stream, n, nw, o}.run(source, st);
}

// widen the native distances to double (exact for u32 / f32 / f64)
template <class W>
__global__ void k_widen(const typename DT<W>::D* d, double* out, uint32_t n) {
  uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    typename DT<W>::D x = d[i];
    out[i] = x == dinf<W>() ? __longlong_as_double(0x7FF0000000000000ll) : (double)x;
  }
}

void sssp_read(Graph* g, double* dist, void* dist_native, uint32_t* pred) {
  Workspace* ws = g->ws.get();
  if (!ws || !ws->has_result) fail(GFB_ELOGIC, "sssp_read: no result on this graph");
  Ctx* c = g->ctx;
  cudaStream_t s = c->stream;
  const uint32_t n = (uint32_t)g->n;
  if (dist) {
    TBuf tmp;
    tmp.alloc((size_t)n * 8, s);
    if (g->wtype == GFB_W_F32) k_widen<float><<<stride_grid(c), 256, 0, s>>>(ws->dist.as<float>(), tmp.as<double>(), n);
    else if (g->wtype == GFB_W_F64) k_widen<double><<<stride_grid(c), 256, 0, s>>>(ws->dist.as<double>(), tmp.as<double>(), n);
    else k_widen<uint32_t><<<stride_grid(c), 256, 0, s>>>(ws->dist.as<uint32_t>(), tmp.as<double>(), n);
    GFB_CUDA(cudaGetLastError());
    GFB_CUDA(cudaMemcpyAsync(dist, tmp.p, (size_t)n * 8, cudaMemcpyDeviceToHost, s));
    c->sync();
  }
  if (dist_native)
    GFB_CUDA(cudaMemcpyAsync(dist_native, ws->dist.p, (size_t)n * dist_bytes(g->wtype),
                             cudaMemcpyDeviceToHost, s));
  if (pred) GFB_CUDA(cudaMemcpyAsync(pred, ws->pred.p, (size_t)n * 4, cudaMemcpyDeviceToHost, s));
  c->sync();
}

}  // namespace gfb

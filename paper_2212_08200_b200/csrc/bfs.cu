// bfs.cu -- bfs() of algorithms.hpp:194-239 on the device: the same
// operator reuse as the reference (neighbors_expand with a claim condition,
// frontier compaction, convergence loop), level-synchronous.
//
//   k_bfs_push  one frontier edge per lane (warp tiles of 256 plan edges,
//               shuffle segment search as in k_push_range): an unclaimed
//               destination gets depth[u] + 1 and its next-frontier bit.  All
//               writers of one level store the same value, so the reference's
//               compare-exchange (algorithms.hpp:210-215) becomes a test and
//               a plain store plus a red.or -- no returning atomic.
//   k_bfs_pull  bottom-up level (needs the transpose): each unvisited vertex
//               scans its in-edges until a parent in the frontier bitmap
//   compaction  the plain bitmap -> plan passes of frontier.cuh
//   loop        CUDA graph: init, compact, WHILE(k > 0) { IF(pull) pull ELSE
//               push; compact } -- direction PUSH: push only; AUTO with a
//               transpose: pull while the frontier has > m / 20 out-edges
//               (direction-optimizing); PULL: every level bottom-up.
//
// Results equal the reference's for every direction: depths are unique,
// supersteps = max depth + 1 (one expansion per non-empty level), and
// relaxations = out-degree sum of the reached vertices (push evaluates every
// out-edge of the frontier once; the reference's pull evaluates every in-edge
// from an active source once, the same edge set) -- reported from the plan
// totals, whatever the bottom-up scan actually touched.
#include <algorithm>

#include "frontier.cuh"
#include "impl.hpp"

namespace gfb {

__global__ void k_bfs_init(uint32_t* depth, uint32_t* bm_next, uint32_t n, uint32_t nwords,
                           const uint32_t* src_ptr, Ctl* ctl) {
  const uint32_t s = *src_ptr;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    depth[i] = i == s ? 0u : NIL;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nwords; i += stride)
    bm_next[i] = (s >> 5) == i ? (1u << (s & 31)) : 0u;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    Ctl c0 = {};
    *ctl = c0;
  }
}

template <class W>
__global__ void __launch_bounds__(256) k_bfs_push(const EdgeRec<W>* __restrict__ adj,
                                                  uint32_t* depth, uint32_t* bm_out, Plan plan,
                                                  Ctl* ctl) {
  constexpr uint32_t TILE = 256;
  const uint32_t total = ctl->total, k = ctl->k;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctl->relax += total;  // every frontier out-edge evaluates the claim once
    ctl->supersteps += 1;
    ctl->push_steps += 1;
  }
  const int lane = threadIdx.x & 31;
  const uint32_t gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint64_t t0 = (uint64_t)gwarp * TILE; t0 < total; t0 += (uint64_t)nwarps * TILE) {
    const uint32_t e0 = (uint32_t)t0, e1 = (uint32_t)min(t0 + TILE, (uint64_t)total);
    uint32_t cs = plan.tseg[e0 / PLAN_GRAIN];  // segment holding e0
    for (;;) {
      const uint32_t cand = cs + lane;
      const uint32_t end = cand < k ? plan.off[cand + 1] : 0xFFFFFFFFu;
      const unsigned msk = __ballot_sync(0xffffffffu, cand < k && end > e0);
      if (msk) {
        cs += __ffs(msk) - 1;
        break;
      }
      cs += 32;
    }
    for (;; cs += 32) {  // windows of 32 segments: lane j holds segment cs + j
      uint32_t off = 0xFFFFFFFFu, start = 0, du = 0;
      if (cs + lane < k) {
        off = plan.off[cs + lane];
        start = plan.start[cs + lane];
      }
      const uint32_t c0 = max(__shfl_sync(0xffffffffu, off, 0), e0);
      if (c0 >= e1) break;
      if (cs + lane < k && off < e1) du = depth[plan.v[cs + lane]];
      const uint32_t nxt = cs + 32 < k ? plan.off[cs + 32] : total;
      const uint32_t c1 = min(nxt, e1);
      for (uint32_t x = c0; x < c1; x += 32) {
        const uint32_t le = x + lane;
        int lo = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
          const uint32_t o = __shfl_sync(0xffffffffu, off, lo + step);
          if (o <= le) lo += step;
        }
        const uint32_t so = __shfl_sync(0xffffffffu, off, lo);
        const uint32_t ss = __shfl_sync(0xffffffffu, start, lo);
        const uint32_t sd = __shfl_sync(0xffffffffu, du, lo);
        if (le < c1) {
          const uint32_t v = adj[ss + (le - so)].v;
          if (depth[v] == NIL) {  // claim: every claimant of this level writes sd + 1
            depth[v] = sd + 1;
            red_or_u32(bm_out + (v >> 5), 1u << (v & 31));
          }
        }
      }
      if (c1 >= e1) break;
    }
  }
}

// Bottom-up level (direction-optimizing BFS): every unvisited vertex scans
// its in-edges (CSC) until it finds a parent in the current frontier bitmap.
// relaxations still count the reference's claim evaluations (the frontier's
// out-degree sum, ctl->total), not the early-exit scan.
template <class W>
__global__ void __launch_bounds__(256) k_bfs_pull(const uint32_t* __restrict__ co,
                                                  const EdgeRec<W>* __restrict__ cadj,
                                                  uint32_t* depth,
                                                  const uint32_t* __restrict__ bm_cur,
                                                  uint32_t* bm_next, uint32_t n, Ctl* ctl) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctl->relax += ctl->total;
    ctl->supersteps += 1;
    ctl->pull_steps += 1;
  }
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) {
    if (depth[v] != NIL) continue;
    const uint32_t e1 = co[v + 1];
    for (uint32_t i = co[v]; i < e1; ++i) {
      const uint32_t u = cadj[i].v;
      if ((__ldg(bm_cur + (u >> 5)) >> (u & 31)) & 1u) {
        depth[v] = depth[u] + 1;
        red_or_u32(bm_next + (v >> 5), 1u << (v & 31));
        break;
      }
    }
  }
}

// depth (u32, NIL unreached) -> double (inf), and the largest finite depth
__global__ void k_bfs_widen(const uint32_t* depth, double* out, uint32_t n, uint32_t* maxd) {
  uint32_t mx = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t d = depth[i];
    if (out) out[i] = d == NIL ? __longlong_as_double(0x7FF0000000000000ll) : (double)d;
    if (d != NIL) mx = max(mx, d);
  }
  mx = __reduce_max_sync(0xffffffffu, mx);
  if ((threadIdx.x & 31) == 0) atomicMax(maxd, mx);
}

template <class W>
static void bfs_t(Ctx* c, Graph* g, uint32_t source, int direction, double* depth_out,
                  uint64_t* supersteps, uint64_t* relaxations) {
  Workspace* ws = ensure_ws(g);
  cudaStream_t s = c->stream;
  const uint32_t n = (uint32_t)g->n, nwords = (n + 31) / 32;
  ws->has_result = false;  // ws->dist holds depths below, not an SSSP result
  uint32_t* depth = ws->dist.as<uint32_t>();
  Ctl* ctl = ws->ctl.as<Ctl>();
  Plan plan{ws->pv.as<uint32_t>(), ws->pstart.as<uint32_t>(), ws->poff.as<uint32_t>(),
            ws->ptseg.as<uint32_t>(), (uint32_t)(ws->ptseg.bytes / 4)};
  const uint32_t tiles = ws->ftiles;
  auto compact = [&](cudaStream_t st, cudaGraphConditionalHandle h, int set_loop) {
    cudaGraphConditionalHandle none{};
    k_fcount<<<tiles, F_WARPS * 32, 0, st>>>(g->ro.as<uint32_t>(), ws->bm_next.as<uint32_t>(),
                                             nwords, ws->agg.as<uint2>());
    k_fscan<<<1, F_SCAN_THREADS, 0, st>>>(ws->agg.as<uint2>(), tiles, plan, ctl, (uint32_t)g->m,
                                          1.0f, 0, 0, h, none, set_loop, 0);
    k_fwrite<<<tiles, F_WARPS * 32, 0, st>>>(g->ro.as<uint32_t>(), ws->bm_next.as<uint32_t>(),
                                             nullptr, nwords, ws->agg.as<uint2>(), plan);
  };
  // direction-optimizing when a transpose exists: pull (bottom-up) levels
  // while the frontier has more than m / BFS_ALPHA out-edges (AUTO), every
  // level for PULL (the reference's pull -- same results, see the header)
  constexpr float BFS_ALPHA = 20.0f;
  const bool pullable = direction != GFB_DIR_PUSH && g->has_csc;
  const int key = pullable ? direction : GFB_DIR_PUSH;
  if (ws->bfs_exec && ws->bfs_key != key) {
    cudaGraphExecDestroy(ws->bfs_exec);
    cudaGraphDestroy(ws->bfs_graph);
    ws->bfs_exec = nullptr;
    ws->bfs_graph = nullptr;
  }
  auto compact2 = [&](cudaStream_t st, cudaGraphConditionalHandle hl,
                      cudaGraphConditionalHandle hm, int set_mode) {
    k_fcount<<<tiles, F_WARPS * 32, 0, st>>>(g->ro.as<uint32_t>(), ws->bm_next.as<uint32_t>(),
                                             nwords, ws->agg.as<uint2>());
    k_fscan<<<1, F_SCAN_THREADS, 0, st>>>(ws->agg.as<uint2>(), tiles, plan, ctl, (uint32_t)g->m,
                                          BFS_ALPHA, direction == GFB_DIR_AUTO ? 1 : 0,
                                          direction == GFB_DIR_PULL ? 1 : 0, hl, hm, 1, set_mode);
    k_fwrite<<<tiles, F_WARPS * 32, 0, st>>>(g->ro.as<uint32_t>(), ws->bm_next.as<uint32_t>(),
                                             ws->bm_cur.as<uint32_t>(), nwords,
                                             ws->agg.as<uint2>(), plan);
  };
  if (!ws->bfs_exec && pullable) {
    for (auto& a : c->aux)
      if (!a) GFB_CUDA(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking));
    cudaGraph_t G;
    GFB_CUDA(cudaGraphCreate(&G, 0));
    cudaGraphConditionalHandle hloop, hmode;
    GFB_CUDA(cudaGraphConditionalHandleCreate(&hloop, G, 1, cudaGraphCondAssignDefault));
    GFB_CUDA(cudaStreamBeginCaptureToGraph(s, G, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    k_bfs_init<<<stride_grid(c), 256, 0, s>>>(depth, ws->bm_next.as<uint32_t>(), n, nwords,
                                               ws->src_dev.as<uint32_t>(), ctl);
    compact2(s, hloop, cudaGraphConditionalHandle{}, 0);  // also writes bm_cur
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
    // first level expands {source}: push unless pull is forced
    GFB_CUDA(cudaGraphConditionalHandleCreate(&hmode, body, direction == GFB_DIR_PULL ? 1 : 0,
                                              cudaGraphCondAssignDefault));
    cudaStream_t b = c->aux[0], x = c->aux[1];
    GFB_CUDA(cudaStreamBeginCaptureToGraph(b, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    GFB_CUDA(cudaStreamGetCaptureInfo(b, &cst, nullptr, &capG, &deps, &ndeps));
    cudaGraphNodeParams ip{};
    ip.type = cudaGraphNodeTypeConditional;
    ip.conditional.handle = hmode;
    ip.conditional.type = cudaGraphCondTypeIf;
    ip.conditional.size = 2;  // [0]: pull, [1]: push
    cudaGraphNode_t inode;
    GFB_CUDA(cudaGraphAddNode(&inode, capG, deps, ndeps, &ip));
    cudaGraph_t gpull = ip.conditional.phGraph_out[0], gpush = ip.conditional.phGraph_out[1];
    GFB_CUDA(cudaStreamUpdateCaptureDependencies(b, &inode, 1, cudaStreamSetCaptureDependencies));
    GFB_CUDA(cudaStreamBeginCaptureToGraph(x, gpull, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    k_bfs_pull<W><<<c->num_sms * 8, 256, 0, x>>>(g->co.as<uint32_t>(), g->cadj.as<EdgeRec<W>>(),
                                                 depth, ws->bm_cur.as<uint32_t>(),
                                                 ws->bm_next.as<uint32_t>(), n, ctl);
    GFB_CUDA(cudaStreamEndCapture(x, &tmp));
    GFB_CUDA(cudaStreamBeginCaptureToGraph(x, gpush, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    k_bfs_push<W><<<c->num_sms * 8, 256, 0, x>>>(g->adj.as<EdgeRec<W>>(), depth,
                                                 ws->bm_next.as<uint32_t>(), plan, ctl);
    GFB_CUDA(cudaStreamEndCapture(x, &tmp));
    compact2(b, hloop, hmode, 1);
    GFB_CUDA(cudaStreamEndCapture(b, &tmp));
    GFB_CUDA(cudaGraphInstantiate(&ws->bfs_exec, G, 0));
    ws->bfs_graph = G;
    ws->bfs_key = key;
  }
  if (!ws->bfs_exec) {  // push only: captured once per graph workspace
    for (auto& a : c->aux)
      if (!a) GFB_CUDA(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking));
    cudaGraph_t G;
    GFB_CUDA(cudaGraphCreate(&G, 0));
    cudaGraphConditionalHandle hloop;
    GFB_CUDA(cudaGraphConditionalHandleCreate(&hloop, G, 1, cudaGraphCondAssignDefault));
    GFB_CUDA(cudaStreamBeginCaptureToGraph(s, G, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    k_bfs_init<<<stride_grid(c), 256, 0, s>>>(depth, ws->bm_next.as<uint32_t>(), n, nwords,
                                               ws->src_dev.as<uint32_t>(), ctl);
    compact(s, hloop, 1);
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
    cudaStream_t b = c->aux[0];
    GFB_CUDA(cudaStreamBeginCaptureToGraph(b, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    k_bfs_push<W><<<c->num_sms * 8, 256, 0, b>>>(g->adj.as<EdgeRec<W>>(), depth,
                                                 ws->bm_next.as<uint32_t>(), plan, ctl);
    compact(b, hloop, 1);
    GFB_CUDA(cudaStreamEndCapture(b, &tmp));
    GFB_CUDA(cudaGraphInstantiate(&ws->bfs_exec, G, 0));
    ws->bfs_graph = G;
    ws->bfs_key = key;
  }
  GFB_CUDA(cudaMemcpyAsync(ws->src_dev.p, &source, 4, cudaMemcpyHostToDevice, s));
  GFB_CUDA(cudaGraphLaunch(ws->bfs_exec, s));
  TBuf out, mx;
  mx.alloc(16, s);
  GFB_CUDA(cudaMemsetAsync(mx.p, 0, 4, s));
  if (depth_out) out.alloc((size_t)n * 8 + 8, s);
  k_bfs_widen<<<stride_grid(c), 256, 0, s>>>(depth, depth_out ? out.as<double>() : nullptr, n,
                                             mx.as<uint32_t>());
  GFB_CUDA(cudaGetLastError());
  uint32_t maxd = 0;
  GFB_CUDA(cudaMemcpyAsync(&maxd, mx.p, 4, cudaMemcpyDeviceToHost, s));
  if (depth_out) GFB_CUDA(cudaMemcpyAsync(depth_out, out.p, (size_t)n * 8, cudaMemcpyDeviceToHost, s));
  const Ctl h = c->read_ctl(ctl);
  // one superstep per non-empty level (the reference also expands a last
  // level whose vertices have no out-edges, which the plan skips)
  if (supersteps) *supersteps = (uint64_t)maxd + 1;
  if (relaxations) *relaxations = h.relax;
}

void bfs_run(Ctx* c, Graph* g, uint32_t source, int direction, double* depth,
             uint64_t* supersteps, uint64_t* relaxations) {
  if (source >= g->n) fail(GFB_ERANGE, "bfs: source out of range");  // algorithms.hpp:200
  if (direction == GFB_DIR_PULL && !g->csc_wanted)                  // algorithms.hpp:201-202
    fail(GFB_EINVAL, "bfs: pull direction requires a built transpose");
  if (direction < GFB_DIR_PUSH || direction > GFB_DIR_AUTO) fail(GFB_EINVAL, "bfs: bad direction");
  if (direction != GFB_DIR_PUSH) ensure_csc(g);  // bottom-up levels read the transpose
  if (g->wtype == GFB_W_F32) bfs_t<float>(c, g, source, direction, depth, supersteps, relaxations);
  else if (g->wtype == GFB_W_F64) bfs_t<double>(c, g, source, direction, depth, supersteps, relaxations);
  else bfs_t<uint32_t>(c, g, source, direction, depth, supersteps, relaxations);
}

}  // namespace gfb

// sssp.cu -- the device SSSP driver: sssp() of algorithms.hpp:569-623 as
// init -> { advance (push | pull) -> compact } until the frontier is empty
// -> predecessor pass, all on one CUDA stream.
#include <cmath>
#include <cstring>

#include "hot.cuh"
#include "impl.hpp"

namespace gfb {

static size_t dist_bytes(int wtype) { return wtype == GFB_W_F64 ? 8 : 4; }

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
  ws->compact_tiles = (uint32_t)((nwords + C_WORDS - 1) / C_WORDS);
  if (ws->compact_tiles == 0) ws->compact_tiles = 1;
  ws->status_len = ws->compact_tiles + 1;
  ws->status.alloc((size_t)ws->status_len * 8, s);
  ws->ctl.alloc(sizeof(Ctl), s);
  GFB_CUDA(cudaMallocHost(&ws->ctl_host, sizeof(Ctl)));
  g->ws = std::move(ws);
  return g->ws.get();
}

template <class W>
struct Runner {
  using D = typename DT<W>::D;
  Ctx* c;
  Graph* g;
  Workspace* ws;
  cudaStream_t s;
  uint32_t n, nwords;
  uint64_t kernels = 0;

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
    a.adj = pull ? g->cadj.as<EdgeRec<W>>() : g->adj.as<EdgeRec<W>>();
    a.ceid = g->ceid.as<uint32_t>();
    a.dist = ws->dist.as<D>();
    a.predrec = ws->predrec.as<uint2>();
    a.plan = pull ? pull_plan() : plan();
    a.ctl = ws->ctl.as<Ctl>();
    a.bm_out = ws->bm_next.as<uint32_t>();
    a.bm_in = ws->bm_cur.as<uint32_t>();
    a.status = ws->status.as<unsigned long long>();
    a.status_len = ws->status_len;
    a.op = GFB_OP_RELAX_MIN;
    return a;
  }

  void compact() {
    k_compact<<<ws->compact_tiles, C_WARPS * 32, 0, s>>>(
        g->ro.as<uint32_t>(), ws->bm_next.as<uint32_t>(), ws->bm_cur.as<uint32_t>(), nwords, n,
        plan(), ws->ctl.as<Ctl>(), ws->status.as<unsigned long long>(), ws->compact_tiles, 1);
  }

  int variant = 0;  // experimental kernel shape (opts.reserved[0])

  template <int VT, int MINB>
  void push_launch(uint32_t total) {
    constexpr int TILE = H_BLOCK * VT;
    uint32_t ntiles = (total + TILE - 1) / TILE;
    uint32_t grid = std::min<uint32_t>(std::max<uint32_t>(ntiles, 1), c->num_sms * MINB);
    k_push_relax<W, VT, MINB><<<grid, H_BLOCK, 0, s>>>(args(false));
  }

  template <int VT, int MINB>
  void warp_launch(uint32_t total) {
    constexpr int WT = 32 * VT;
    uint32_t ntiles = (total + WT - 1) / WT;
    uint32_t warps_cap = c->num_sms * MINB * 8;  // 8 warps per 256-thread CTA
    uint32_t warps = std::min<uint32_t>(std::max<uint32_t>(ntiles, 1), warps_cap);
    k_push_warp<W, VT, MINB><<<(warps + 7) / 8, 256, 0, s>>>(args(false));
  }

  void advance(bool pull, uint32_t total) {
    const uint32_t cap = c->num_sms * 4;  // 4 resident CTAs per SM (launch bounds)
    if (pull) {
      uint32_t ntiles = (g->pull_total + HotCfg<W>::TILE - 1) / HotCfg<W>::TILE;
      uint32_t grid = std::min<uint32_t>(std::max<uint32_t>(ntiles, 1), cap);
      k_pull_relax<W><<<grid, H_BLOCK, 0, s>>>(args(true), g->pull_total, g->pull_k);
      return;
    }
    switch (variant) {
      case 5: push_launch<HotCfg<W>::VT, 4>(total); break;
      case 6: warp_launch<4, 8>(total); break;
      case 7: warp_launch<8, 6>(total); break;
      case 1: push_launch<4, 8>(total); break;
      case 2: push_launch<4, 6>(total); break;
      case 3: push_launch<8, 6>(total); break;
      case 4: {  // generic operator kernel (one edge in flight per thread)
        uint32_t ntiles = (total + A_TILE - 1) / A_TILE;
        uint32_t grid = std::min<uint32_t>(std::max<uint32_t>(ntiles, 1), c->num_sms * 8);
        k_advance_push<W, OUT_BITMAP><<<grid, A_BLOCK, 0, s>>>(args(false));
        break;
      }
      default: warp_launch<(sizeof(W) == 8 ? 4 : 8), 4>(total);
    }
  }

  void run(uint32_t source, const gfb_sssp_opts* o, gfb_sssp_stats* st) {
    ws->has_result = false;
    variant = o->reserved[0];
    GFB_CUDA(cudaEventRecord(c->ev[0], s));
    k_init<W><<<stride_grid(c), 256, 0, s>>>(ws->dist.as<D>(), ws->predrec.as<uint2>(),
                                             ws->bm_next.as<uint32_t>(), ws->bm_cur.as<uint32_t>(),
                                             n, nwords, source, ws->ctl.as<Ctl>());
    GFB_CUDA(cudaMemsetAsync(ws->status.p, 0, (size_t)ws->status_len * 8, s));
    compact();
    GFB_CUDA(cudaGetLastError());
    const int dir = o->direction;
    const double alpha = o->pull_alpha > 0 ? o->pull_alpha : 1.5;
    uint64_t supersteps = 0, push_steps = 0, pull_steps = 0, launches = 0;
    kernels = 2;  // k_init + first k_compact
    float adv_ms = 0;
    for (;;) {
      Ctl h = c->read_ctl(ws->ctl.as<Ctl>());
      if (h.err & 1u) fail(GFB_ERANGE, "sssp: u32 distance overflow (use f64 weights)");
      if (h.k == 0) break;
      bool pull = false;
      if (dir == GFB_DIR_PULL) pull = true;
      else if (dir == GFB_DIR_AUTO && g->has_csc && (double)h.total > (double)g->m / alpha)
        pull = true;
      GFB_CUDA(cudaEventRecord(c->ev[2], s));
      advance(pull, h.total);
      GFB_CUDA(cudaEventRecord(c->ev[3], s));
      GFB_CUDA(cudaGetLastError());
      compact();
      GFB_CUDA(cudaGetLastError());
      ++supersteps;
      ++launches;
      kernels += 2;
      (pull ? pull_steps : push_steps)++;
      GFB_CUDA(cudaEventSynchronize(c->ev[3]));
      float ms = 0;
      GFB_CUDA(cudaEventElapsedTime(&ms, c->ev[2], c->ev[3]));
      adv_ms += ms;
    }
    uint64_t fallback = 0;
    pred_pass(source, o->compute_pred != 0, &fallback);
    GFB_CUDA(cudaEventRecord(c->ev[1], s));
    Ctl h = c->read_ctl(ws->ctl.as<Ctl>());
    if (h.err & 1u) fail(GFB_ERANGE, "sssp: u32 distance overflow (use f64 weights)");
    float ms = 0;
    GFB_CUDA(cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]));
    ws->has_result = true;
    ws->source = source;
    if (st) {
      st->supersteps = supersteps;
      st->relaxations = h.relax;
      st->n_reach = h.n_reach;
      st->m_reach = h.m_reach;
      st->push_steps = push_steps;
      st->pull_steps = pull_steps;
      st->pred_fallback = fallback;
      st->device_ms = ms;
      st->advance_ms = adv_ms;
      st->advance_launches = launches;
      st->kernel_launches = kernels;
    }
  }

  void pred_pass(uint32_t source, bool want, uint64_t* fallback) {
    GFB_CUDA(cudaMemsetAsync(ws->repair_bm.p, 0, (size_t)nwords * 4, s));
    GFB_CUDA(cudaMemsetAsync(&ws->ctl.as<Ctl>()->flag, 0, 4, s));
    k_pred_verify<W><<<std::max<uint32_t>((n + 255) / 256, 1), 256, 0, s>>>(
        g->ro.as<uint32_t>(), g->adj.as<EdgeRec<W>>(), ws->dist.as<D>(), ws->predrec.as<uint2>(),
        ws->pred.as<uint32_t>(), ws->res.as<uint32_t>(), ws->repair_bm.as<uint32_t>(),
        ws->cand.as<uint32_t>(), n, source, ws->ctl.as<Ctl>());
    GFB_CUDA(cudaGetLastError());
    ++kernels;
    if (!want) return;
    Ctl h = c->read_ctl(ws->ctl.as<Ctl>());
    *fallback = h.unresolved;
    if (h.unresolved == 0) return;
    uint64_t left = h.unresolved;
    if (g->has_csc) {
      // unresolved vertices were appended to ws->cand; scan their in-edges
      const uint32_t count = h.unresolved;
      DBuf list;
      list.alloc((size_t)count * 4, s);
      GFB_CUDA(cudaMemcpyAsync(list.p, ws->cand.p, (size_t)count * 4, cudaMemcpyDeviceToDevice, s));
      for (uint32_t round = 1; left > 0; ++round) {
        GFB_CUDA(cudaMemsetAsync(&ws->ctl.as<Ctl>()->flag, 0, 4, s));
        uint32_t grid = std::min<uint32_t>((count + 7) / 8, c->num_sms * 8);
        k_pred_csc_round<W><<<grid, 256, 0, s>>>(
            g->co.as<uint32_t>(), g->cadj.as<EdgeRec<W>>(), ws->dist.as<D>(),
            ws->pred.as<uint32_t>(), ws->res.as<uint32_t>(), list.as<uint32_t>(), count, round,
            ws->ctl.as<Ctl>());
        GFB_CUDA(cudaGetLastError());
        ++kernels;
        Ctl r = c->read_ctl(ws->ctl.as<Ctl>());
        // round 1 (strict edges) may resolve nothing when every unresolved
        // vertex sits in a zero-weight tie class; later rounds must progress.
        if (r.flag == 0 && round > 1)
          fail(GFB_ELOGIC, "sssp: predecessor repair made no progress");
        left -= std::min<uint64_t>(left, r.flag);
      }
      return;
    }
    // no CSC: candidate rounds over every CSR row (O(m) per round)
    GFB_CUDA(cudaMemsetAsync(ws->cand.p, 0xFF, (size_t)n * 4, s));
    for (uint32_t round = 1; left > 0; ++round) {
      GFB_CUDA(cudaMemsetAsync(&ws->ctl.as<Ctl>()->flag, 0, 4, s));
      k_pred_repair<W><<<stride_grid(c), 256, 0, s>>>(
          g->ro.as<uint32_t>(), g->adj.as<EdgeRec<W>>(), ws->dist.as<D>(), ws->cand.as<uint32_t>(),
          ws->res.as<uint32_t>(), ws->repair_bm.as<uint32_t>(), n, round);
      k_pred_apply<<<stride_grid(c), 256, 0, s>>>(ws->cand.as<uint32_t>(), ws->pred.as<uint32_t>(),
                                                  ws->res.as<uint32_t>(),
                                                  ws->repair_bm.as<uint32_t>(), n, round,
                                                  ws->ctl.as<Ctl>());
      GFB_CUDA(cudaGetLastError());
      kernels += 2;
      Ctl r = c->read_ctl(ws->ctl.as<Ctl>());
      if (r.flag == 0 && round > 1)
        fail(GFB_ELOGIC, "sssp: predecessor repair made no progress");
      left -= std::min<uint64_t>(left, r.flag);
    }
  }
};

void sssp_run(Ctx* c, Graph* g, uint32_t source, const gfb_sssp_opts* o, gfb_sssp_stats* st) {
  if (source >= g->n) fail(GFB_ERANGE, "sssp: source out of range");  // algorithms.hpp:572
  if (o->direction == GFB_DIR_PULL && !g->has_csc)                     // algorithms.hpp:573-574
    fail(GFB_EINVAL, "sssp: pull direction requires a built transpose");
  if (o->direction < GFB_DIR_PUSH || o->direction > GFB_DIR_AUTO)
    fail(GFB_EINVAL, "sssp: bad direction");
  Workspace* ws = ensure_ws(g);
  if (g->wtype == GFB_W_F32) Runner<float>{c, g, ws, c->stream, (uint32_t)g->n, (uint32_t)((g->n + 31) / 32)}.run(source, o, st);
  else if (g->wtype == GFB_W_F64) Runner<double>{c, g, ws, c->stream, (uint32_t)g->n, (uint32_t)((g->n + 31) / 32)}.run(source, o, st);
  else Runner<uint32_t>{c, g, ws, c->stream, (uint32_t)g->n, (uint32_t)((g->n + 31) / 32)}.run(source, o, st);
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
    DBuf tmp;
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

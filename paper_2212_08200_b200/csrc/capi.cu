// capi.cu -- the extern "C" boundary (include/gfb.h).  Every entry point
// catches internal errors and returns a status; gfb_last_error() holds the
// thread-local message (no exception crosses the ABI).
#include <cstdio>
#include <cstring>
#include <string>

#include "impl.hpp"

namespace gfb {

static thread_local std::string g_last_error;

[[noreturn]] void fail(int code, const std::string& msg) { throw Error{code, msg}; }

void check_cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  cudaGetLastError();
  int code = e == cudaErrorMemoryAllocation ? GFB_ENOMEM : GFB_ECUDA;
  fail(code, std::string(what) + ": " + cudaGetErrorString(e));
}

// ops.cu / graph.cu
Graph* graph_upload(Ctx*, uint64_t, uint64_t, const uint32_t*, const uint32_t*, const void*, int,
                    int, int, uint64_t);
void graph_refill(Graph*, const uint32_t*, const uint32_t*, const void*, int);
Graph* graph_generate_rmat(Ctx*, int, int, uint64_t, int, int);
Graph* graph_generate_grid(Ctx*, uint32_t, uint64_t, int);
Graph* graph_from_edges(Ctx*, uint64_t, uint64_t, const uint32_t*, const uint32_t*, const double*,
                        int, int);
struct EdgeList;
EdgeList* mm_parse(const char*, size_t, bool, bool);
void edge_list_free(EdgeList*);
void edge_list_info(const EdgeList*, uint64_t*, uint64_t*);
void edge_list_read(const EdgeList*, uint32_t*, uint32_t*, double*);
const uint32_t* edge_list_src(const EdgeList*);
const uint32_t* edge_list_dst(const EdgeList*);
const double* edge_list_w(const EdgeList*);
uint64_t parse_error_line();
void graph_download(Graph*, uint32_t*, uint32_t*, void*);
Frontier* frontier_create(Ctx*, uint64_t, int);
void frontier_assign(Frontier*, const uint32_t*, uint64_t);
uint64_t frontier_size(Frontier*);
void frontier_read(Frontier*, uint32_t*, uint64_t, uint64_t*);
void advance_push(Ctx*, const Graph*, Frontier*, Frontier*, int, void*);
void advance_pull(Ctx*, const Graph*, Frontier*, Frontier*, int, void*);
void filter_unique(Ctx*, Frontier*, Frontier*);
void filter(Ctx*, Frontier*, Frontier*, int, const Dist*, double);
Dist* dist_create(Ctx*, const Graph*);
void dist_init(Dist*, uint32_t);
void dist_read(Dist*, double*, uint64_t*);
Record* record_create(Ctx*, uint64_t);
void record_read(Record*, uint32_t*, uint32_t*, uint32_t*, uint64_t, uint64_t*);

template <class F>
static int guard(F&& f) {
  try {
    f();
    return GFB_OK;
  } catch (const Error& e) {
    g_last_error = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return GFB_ENOMEM;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return GFB_ECUDA;
  }
}

static void set_device(Ctx* c) { GFB_CUDA(cudaSetDevice(c->device)); }

}  // namespace gfb

using namespace gfb;

struct gfb_ctx : Ctx {};
struct gfb_graph : Graph {};
struct gfb_frontier : Frontier {};
struct gfb_dist : Dist {};
struct gfb_record : Record {};
struct gfb_part : Part {};

#define NEED(p)                                          \
  do {                                                   \
    if (!(p)) fail(GFB_EINVAL, "null argument: " #p);    \
  } while (0)

extern "C" {

int gfb_version(void) { return 1; }

const char* gfb_last_error(void) { return g_last_error.c_str(); }

int gfb_ctx_create(int device, gfb_ctx** out) {
  return guard([&] {
    NEED(out);
    int count = 0;
    GFB_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) fail(GFB_EINVAL, "ctx: no CUDA device " + std::to_string(device));
    GFB_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    GFB_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
      fail(GFB_ECUDA, std::string("ctx: libgfb is built for sm_100a; device is ") + prop.name);
    auto* c = new gfb_ctx();
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    try {
      // keep freed pool memory reserved (DBuf allocates stream-ordered)
      cudaMemPool_t pool;
      GFB_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
      uint64_t keep = ~0ull;
      GFB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
      GFB_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      for (auto& e : c->ev) GFB_CUDA(cudaEventCreate(&e));
      GFB_CUDA(cudaMallocHost(&c->ctl_host, sizeof(Ctl)));
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

int gfb_ctx_destroy(gfb_ctx* ctx) {
  return guard([&] {
    if (!ctx) return;
    set_device(ctx);
    cudaStreamSynchronize(ctx->stream);
    delete ctx;
  });
}

int gfb_ctx_num_sms(gfb_ctx* ctx, int* out) {
  return guard([&] {
    NEED(ctx);
    NEED(out);
    *out = ctx->num_sms;
  });
}

int gfb_graph_upload(gfb_ctx* ctx, uint64_t n, uint64_t m, const uint32_t* ro, const uint32_t* col,
                     const void* w, int w_host_type, int wtype, int build_csc, gfb_graph** out) {
  return guard([&] {
    NEED(ctx);
    NEED(out);
    set_device(ctx);
    *out = static_cast<gfb_graph*>(
        graph_upload(ctx, n, m, ro, col, w, w_host_type, wtype, build_csc, 0));
  });
}

int gfb_graph_refill(gfb_graph* g, const uint32_t* ro, const uint32_t* col, const void* w,
                     int w_host_type) {
  return guard([&] {
    NEED(g);
    set_device(g->ctx);
    graph_refill(g, ro, col, w, w_host_type);
  });
}

int gfb_graph_free(gfb_graph* g) {
  return guard([&] {
    if (!g) return;
    set_device(g->ctx);
    g->ctx->sync();
    delete static_cast<Graph*>(g);
  });
}

int gfb_graph_info(const gfb_graph* g, uint64_t* n, uint64_t* m, int* wtype, int* has_csc) {
  return guard([&] {
    NEED(g);
    if (n) *n = g->n;
    if (m) *m = g->m;
    if (wtype) *wtype = g->wtype;
    if (has_csc) *has_csc = g->csc_wanted ? 1 : 0;
  });
}

int gfb_graph_download(gfb_graph* g, uint32_t* ro, uint32_t* col, void* w) {
  return guard([&] {
    NEED(g);
    gfb::check_usable(g);
    set_device(g->ctx);
    graph_download(g, ro, col, w);
  });
}

int gfb_graph_generate_rmat(gfb_ctx* ctx, int scale, int ef, uint64_t seed, int wtype, int csc,
                            gfb_graph** out) {
  return guard([&] {
    NEED(ctx);
    NEED(out);
    set_device(ctx);
    *out = static_cast<gfb_graph*>(graph_generate_rmat(ctx, scale, ef, seed, wtype, csc));
  });
}

// ---- Matrix Market ingest (mm.cu) + device build_csr (graph.cu) ----
struct gfb_edge_list {};  // opaque: a gfb::EdgeList

int gfb_mm_parse(const char* text, size_t len, int force_unit, int expand_symmetric,
                 gfb_edge_list** out) {
  return guard([&] {
    NEED(out);
    if (!text && len) gfb::fail(GFB_EINVAL, "mm: null text");
    *out = reinterpret_cast<gfb_edge_list*>(
        gfb::mm_parse(text ? text : "", len, force_unit != 0, expand_symmetric != 0));
  });
}

int gfb_edge_list_info(const gfb_edge_list* e, uint64_t* n, uint64_t* m) {
  return guard([&] {
    NEED(e);
    gfb::edge_list_info(reinterpret_cast<const gfb::EdgeList*>(e), n, m);
  });
}

int gfb_edge_list_read(const gfb_edge_list* e, uint32_t* src, uint32_t* dst, double* w) {
  return guard([&] {
    NEED(e);
    gfb::edge_list_read(reinterpret_cast<const gfb::EdgeList*>(e), src, dst, w);
  });
}

int gfb_edge_list_free(gfb_edge_list* e) {
  return guard([&] { gfb::edge_list_free(reinterpret_cast<gfb::EdgeList*>(e)); });
}

uint64_t gfb_last_error_line(void) { return gfb::parse_error_line(); }

int gfb_graph_from_edges(gfb_ctx* ctx, uint64_t n, uint64_t m, const uint32_t* src,
                         const uint32_t* dst, const double* w, int wtype, int build_csc,
                         gfb_graph** out) {
  return guard([&] {
    NEED(ctx);
    NEED(out);
    set_device(ctx);
    *out = static_cast<gfb_graph*>(graph_from_edges(ctx, n, m, src, dst, w, wtype, build_csc));
  });
}

int gfb_graph_from_edge_list(gfb_ctx* ctx, const gfb_edge_list* e, int wtype, int build_csc,
                             gfb_graph** out) {
  return guard([&] {
    NEED(ctx);
    NEED(e);
    NEED(out);
    set_device(ctx);
    const auto* el = reinterpret_cast<const gfb::EdgeList*>(e);
    uint64_t n = 0, m = 0;
    gfb::edge_list_info(el, &n, &m);
    *out = static_cast<gfb_graph*>(graph_from_edges(ctx, n, m, gfb::edge_list_src(el),
                                                    gfb::edge_list_dst(el), gfb::edge_list_w(el),
                                                    wtype, build_csc));
  });
}

int gfb_graph_generate_grid(gfb_ctx* ctx, uint32_t side, uint64_t seed, int csc, gfb_graph** out) {
  return guard([&] {
    NEED(ctx);
    NEED(out);
    set_device(ctx);
    *out = static_cast<gfb_graph*>(graph_generate_grid(ctx, side, seed, csc));
  });
}

int gfb_frontier_create(gfb_ctx* ctx, uint64_t n, int repr, gfb_frontier** out) {
  return guard([&] {
    NEED(ctx);
    NEED(out);
    set_device(ctx);
    *out = static_cast<gfb_frontier*>(frontier_create(ctx, n, repr));
  });
}

int gfb_frontier_free(gfb_frontier* f) {
  return guard([&] {
    if (!f) return;
    set_device(f->ctx);
    delete static_cast<Frontier*>(f);
  });
}

int gfb_frontier_assign(gfb_frontier* f, const uint32_t* v, uint64_t k) {
  return guard([&] {
    NEED(f);
    if (k) NEED(v);
    set_device(f->ctx);
    frontier_assign(f, v, k);
  });
}

int gfb_frontier_size(gfb_frontier* f, uint64_t* size) {
  return guard([&] {
    NEED(f);
    NEED(size);
    set_device(f->ctx);
    *size = frontier_size(f);
  });
}

int gfb_frontier_read(gfb_frontier* f, uint32_t* out, uint64_t cap, uint64_t* k) {
  return guard([&] {
    NEED(f);
    NEED(k);
    if (cap) NEED(out);
    set_device(f->ctx);
    frontier_read(f, out, cap, k);
  });
}

int gfb_frontier_repr(gfb_frontier* f, int* repr) {
  return guard([&] {
    NEED(f);
    NEED(repr);
    *repr = f->repr;
  });
}

int gfb_dist_create(gfb_ctx* ctx, const gfb_graph* g, gfb_dist** out) {
  return guard([&] {
    NEED(ctx);
    NEED(g);
    NEED(out);
    gfb::check_usable(g);
    set_device(ctx);
    *out = static_cast<gfb_dist*>(dist_create(ctx, g));
  });
}

int gfb_dist_free(gfb_dist* d) {
  return guard([&] {
    if (!d) return;
    set_device(d->ctx);
    delete static_cast<Dist*>(d);
  });
}

int gfb_dist_init(gfb_dist* d, uint32_t source) {
  return guard([&] {
    NEED(d);
    set_device(d->ctx);
    dist_init(d, source);
  });
}

int gfb_dist_read(gfb_dist* d, double* dist, uint64_t* relax) {
  return guard([&] {
    NEED(d);
    set_device(d->ctx);
    dist_read(d, dist, relax);
  });
}

int gfb_record_create(gfb_ctx* ctx, uint64_t cap, gfb_record** out) {
  return guard([&] {
    NEED(ctx);
    NEED(out);
    set_device(ctx);
    *out = static_cast<gfb_record*>(record_create(ctx, cap));
  });
}

int gfb_record_free(gfb_record* r) {
  return guard([&] {
    if (!r) return;
    set_device(r->ctx);
    delete static_cast<Record*>(r);
  });
}

int gfb_record_read(gfb_record* r, uint32_t* s, uint32_t* d, uint32_t* e, uint64_t cap,
                    uint64_t* count) {
  return guard([&] {
    NEED(r);
    NEED(count);
    set_device(r->ctx);
    record_read(r, s, d, e, cap, count);
  });
}

int gfb_advance_push(gfb_ctx* ctx, const gfb_graph* g, gfb_frontier* in, gfb_frontier* out, int op,
                     void* state) {
  return guard([&] {
    NEED(ctx);
    NEED(g);
    gfb::check_usable(g);
    set_device(ctx);
    advance_push(ctx, g, in, out, op, state);
  });
}

int gfb_advance_pull(gfb_ctx* ctx, const gfb_graph* g, gfb_frontier* in, gfb_frontier* out, int op,
                     void* state) {
  return guard([&] {
    NEED(ctx);
    NEED(g);
    gfb::check_usable(g);
    set_device(ctx);
    advance_pull(ctx, g, in, out, op, state);
  });
}

int gfb_filter_unique(gfb_ctx* ctx, gfb_frontier* in, gfb_frontier* out) {
  return guard([&] {
    NEED(ctx);
    NEED(in);
    NEED(out);
    set_device(ctx);
    filter_unique(ctx, in, out);
  });
}

int gfb_filter(gfb_ctx* ctx, gfb_frontier* in, gfb_frontier* out, int pred, const gfb_dist* dist,
               double threshold) {
  return guard([&] {
    NEED(ctx);
    NEED(in);
    NEED(out);
    if (dist) gfb::check_usable(dist->g);
    set_device(ctx);
    filter(ctx, in, out, pred, dist, threshold);
  });
}

void gfb_sssp_opts_default(gfb_sssp_opts* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->struct_size = sizeof(*o);
  o->direction = GFB_DIR_PUSH;  // the reference's default (algorithms.hpp:40)
  o->pull_alpha = 1.05f;         // AUTO: the measured push/pull break-even
  o->device_loop = 1;
  o->delta = 0.0;
  o->compute_pred = 1;
}

int gfb_sssp(gfb_ctx* ctx, gfb_graph* g, uint32_t source, const gfb_sssp_opts* opts, double* dist,
             uint32_t* pred, gfb_sssp_stats* stats) {
  return guard([&] {
    NEED(ctx);
    NEED(g);
    set_device(ctx);
    gfb_sssp_opts o;
    gfb_sssp_opts_default(&o);
    if (opts) {
      if (opts->struct_size != sizeof(gfb_sssp_opts)) fail(GFB_EINVAL, "sssp: opts struct_size mismatch");
      o = *opts;
    }
    gfb_sssp_stats st{};
    sssp_run(ctx, g, source, &o, &st);
    if (dist || pred) sssp_read(g, dist, nullptr, pred);
    if (stats) *stats = st;
  });
}

int gfb_part_create(gfb_ctx* ctx, uint64_t n_global, uint32_t lo, uint32_t hi, uint64_t m_local,
                    const uint32_t* ro_local, const uint32_t* col, const void* w, int w_host_type,
                    int wtype, gfb_part** out) {
  return guard([&] {
    NEED(ctx);
    NEED(out);
    set_device(ctx);
    *out = static_cast<gfb_part*>(
        part_create(ctx, n_global, lo, hi, m_local, ro_local, col, w, w_host_type, wtype));
  });
}

int gfb_part_free(gfb_part* p) {
  return guard([&] {
    if (!p) return;
    set_device(p->ctx);
    p->ctx->sync();
    delete static_cast<Part*>(p);
  });
}

int gfb_part_init(gfb_part* p, uint32_t source) {
  return guard([&] {
    NEED(p);
    set_device(p->ctx);
    part_init(p, source);
  });
}

int gfb_part_advance(gfb_part* p, void* out_dev, uint64_t out_cap, const uint32_t* range_starts,
                     int nparts, uint32_t* counts, uint64_t* total) {
  return guard([&] {
    NEED(p);
    NEED(range_starts);
    NEED(counts);
    set_device(p->ctx);
    uint64_t t = part_advance(p, out_dev, out_cap, range_starts, nparts, counts);
    if (total) *total = t;
  });
}

int gfb_part_apply(gfb_part* p, const void* in_dev, uint64_t count) {
  return guard([&] {
    NEED(p);
    set_device(p->ctx);
    part_apply(p, in_dev, count);
  });
}

int gfb_part_pending(gfb_part* p, uint64_t* size) {
  return guard([&] {
    NEED(p);
    NEED(size);
    set_device(p->ctx);
    *size = part_pending(p);
  });
}

int gfb_part_read(gfb_part* p, void* dist_native, uint64_t* relaxations, uint64_t* supersteps) {
  return guard([&] {
    NEED(p);
    set_device(p->ctx);
    part_read(p, dist_native, relaxations, supersteps);
  });
}

int gfb_part_pred(gfb_part* p, const void* gdist_dev, const uint32_t* res_dev, uint32_t* cand_dev,
                  uint32_t round) {
  return guard([&] {
    NEED(p);
    set_device(p->ctx);
    part_pred(p, gdist_dev, res_dev, cand_dev, round);
  });
}

int gfb_sssp_read(gfb_graph* g, double* dist, void* dist_native, uint32_t* pred) {
  return guard([&] {
    NEED(g);
    gfb::check_usable(g);
    set_device(g->ctx);
    sssp_read(g, dist, dist_native, pred);
  });
}

}  // extern "C"

// Inspection: the in-degree-relabelled loop CSR (include/gfb.h).
int gfb_debug_relabel(gfb_graph* g, uint32_t* ro, uint32_t* adj_pairs, uint32_t* perm) {
  return guard([&] {
    NEED(g);
    gfb::check_usable(g);
    if (g->rec_bytes() != 8) gfb::fail(GFB_EINVAL, "relabel view: 4-byte weights only");
    set_device(g->ctx);
    gfb::ensure_relabel(g);
    if (g->rl_skip) gfb::fail(GFB_ELOGIC, "relabel: in-degrees not skewed, no relabelled view");
    cudaStream_t s = g->ctx->stream;
    if (ro) GFB_CUDA(cudaMemcpyAsync(ro, g->rl_ro.p, (g->n + 1) * 4, cudaMemcpyDeviceToHost, s));
    if (adj_pairs) GFB_CUDA(cudaMemcpyAsync(adj_pairs, g->rl_adj.p, g->m * 8, cudaMemcpyDeviceToHost, s));
    if (perm) GFB_CUDA(cudaMemcpyAsync(perm, g->rl_perm.p, g->n * 4, cudaMemcpyDeviceToHost, s));
    g->ctx->sync();
  });
}

int gfb_graph_relabel_ranges(gfb_graph* g, uint32_t nparts, const uint32_t* range_starts,
                             uint32_t* row_offsets, uint32_t* col, void* weights,
                             uint32_t* perm) {
  return guard([&] {
    NEED(g);
    NEED(range_starts);
    set_device(g->ctx);
    gfb::relabel_ranges(g, nparts, range_starts, row_offsets, col, weights, perm);
  });
}

// ---- peer-memory partitioned SSSP (include/gfb.h) ----
static gfb::Peer* P(gfb_peer* p) { return reinterpret_cast<gfb::Peer*>(p); }

int gfb_peer_create(gfb_ctx* ctx, int rank, int nparts, const uint32_t* range_starts,
                    uint64_t m_local, const uint32_t* ro_local, const uint32_t* col, const void* w,
                    int w_host_type, int wtype, gfb_peer** out) {
  return guard([&] {
    NEED(ctx);
    NEED(range_starts);
    NEED(ro_local);
    NEED(out);
    if (m_local && (!col || !w)) gfb::fail(GFB_EINVAL, "peer: null edge arrays");
    set_device(ctx);
    *out = reinterpret_cast<gfb_peer*>(gfb::peer_create(ctx, rank, nparts, range_starts, m_local,
                                                        ro_local, col, w, w_host_type, wtype));
  });
}

int gfb_peer_export(gfb_peer* p, void* handle) {
  return guard([&] {
    NEED(p);
    NEED(handle);
    set_device(gfb::peer_ctx(P(p)));
    gfb::peer_export(P(p), handle);
  });
}

int gfb_peer_link(gfb_peer* p, const void* handles) {
  return guard([&] {
    NEED(p);
    NEED(handles);
    set_device(gfb::peer_ctx(P(p)));
    gfb::peer_link(P(p), handles);
  });
}

int gfb_peer_sssp(gfb_peer* p, uint32_t source, const gfb_sssp_opts* opts,
                  gfb_sssp_stats* stats) {
  return guard([&] {
    NEED(p);
    set_device(gfb::peer_ctx(P(p)));
    gfb_sssp_opts o;
    gfb_sssp_opts_default(&o);
    if (opts) {
      if (opts->struct_size != sizeof(gfb_sssp_opts)) gfb::fail(GFB_EINVAL, "sssp: opts struct_size mismatch");
      o = *opts;
    }
    gfb::peer_sssp(P(p), source, &o, stats);
  });
}

int gfb_peer_read(gfb_peer* p, double* dist, void* dist_native, uint32_t* pred) {
  return guard([&] {
    NEED(p);
    set_device(gfb::peer_ctx(P(p)));
    gfb::peer_read(P(p), dist, dist_native, pred);
  });
}

int gfb_peer_free(gfb_peer* p) {
  return guard([&] {
    if (!p) return;
    set_device(gfb::peer_ctx(P(p)));
    gfb::peer_ctx(P(p))->sync();
    gfb::peer_free(P(p));
  });
}

// ---- one process, several partitions (include/gfb.h) ----
struct gfb_mg : gfb::Mg {};

int gfb_mg_create(int ndev, const int* devices, gfb_mg** out) {
  return guard([&] {
    NEED(devices);
    NEED(out);
    if (ndev < 1 || ndev > gfb::PEER_MAX) gfb::fail(GFB_EINVAL, "mg: 1 <= ndev <= 8");
    auto mg = std::make_unique<gfb_mg>();
    for (int i = 0; i < ndev; ++i) {
      gfb_ctx* c = nullptr;
      const int rc = gfb_ctx_create(devices[i], &c);
      if (rc != GFB_OK) {
        for (gfb::Ctx* x : mg->ctx) gfb_ctx_destroy(static_cast<gfb_ctx*>(x));
        gfb::fail(rc, gfb_last_error());
      }
      mg->ctx.push_back(c);
    }
    *out = mg.release();
  });
}

int gfb_mg_create_ex(int ndev, const int* devices, int exchange, gfb_mg** out) {
  return guard([&] {
    NEED(out);
    if (exchange != GFB_EXCHANGE_PEER && exchange != GFB_EXCHANGE_NCCL)
      gfb::fail(GFB_EINVAL, "mg: exchange must be GFB_EXCHANGE_PEER or GFB_EXCHANGE_NCCL");
    gfb_mg* mg = nullptr;
    const int rc = gfb_mg_create(ndev, devices, &mg);
    if (rc != GFB_OK) gfb::fail(rc, gfb_last_error());
    mg->exchange = exchange;
    if (exchange == GFB_EXCHANGE_NCCL) {
      try {
        mg->x = gfb::xmg_create(mg->ctx);
      } catch (...) {
        gfb_mg_destroy(mg);
        throw;
      }
    }
    *out = mg;
  });
}

int gfb_mg_uses_nccl(gfb_mg* mg, int* out) {
  return guard([&] {
    NEED(mg);
    NEED(out);
    *out = mg->x && gfb::xmg_uses_nccl(mg->x) ? 1 : 0;
  });
}

int gfb_mg_graph_upload(gfb_mg* mg, uint64_t n, uint64_t m, const uint32_t* row_offsets,
                        const uint32_t* col, const void* w, int w_host_type, int wtype) {
  return guard([&] {
    NEED(mg);
    NEED(row_offsets);
    if (m && (!col || !w)) gfb::fail(GFB_EINVAL, "mg: null edge arrays");
    gfb::mg_upload(mg, n, m, row_offsets, col, w, w_host_type, wtype);
  });
}

int gfb_mg_ranges(gfb_mg* mg, uint32_t* range_starts) {
  return guard([&] {
    NEED(mg);
    NEED(range_starts);
    if (mg->starts.empty()) gfb::fail(GFB_ELOGIC, "mg: no graph uploaded");
    std::memcpy(range_starts, mg->starts.data(), mg->starts.size() * 4);
  });
}

int gfb_mg_sssp(gfb_mg* mg, uint32_t source, const gfb_sssp_opts* opts, double* dist,
                uint32_t* pred, gfb_sssp_stats* stats) {
  return guard([&] {
    NEED(mg);
    gfb_sssp_opts o;
    gfb_sssp_opts_default(&o);
    if (opts) {
      if (opts->struct_size != sizeof(gfb_sssp_opts)) gfb::fail(GFB_EINVAL, "sssp: opts struct_size mismatch");
      o = *opts;
    }
    gfb::mg_sssp(mg, source, &o, dist, pred, stats);
  });
}

int gfb_mg_destroy(gfb_mg* mg) {
  return guard([&] {
    if (!mg) return;
    gfb::mg_free(mg);
    for (gfb::Ctx* x : mg->ctx) gfb_ctx_destroy(static_cast<gfb_ctx*>(x));
    delete mg;
  });
}

// ---- bfs (include/gfb.h) ----
int gfb_bfs(gfb_ctx* ctx, gfb_graph* g, uint32_t source, int direction, double* depth,
            uint64_t* supersteps, uint64_t* relaxations) {
  return guard([&] {
    NEED(ctx);
    NEED(g);
    gfb::check_usable(g);
    set_device(ctx);
    gfb::bfs_run(ctx, g, source, direction, depth, supersteps, relaxations);
  });
}


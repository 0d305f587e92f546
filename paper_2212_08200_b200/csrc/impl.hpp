// impl.hpp -- host-side objects behind the C ABI handles.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <memory>
#include <vector>

#include "kernels.cuh"

namespace gfb {

// Owning device buffer, allocated stream-ordered from the device pool
// (cudaMallocAsync on the given stream).  Re-allocation frees stream-ordered;
// destruction frees synchronously (cudaFree), because a long-lived buffer
// may outlive the stream it was allocated on (objects destroyed at exit).
struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t s = nullptr;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release_sync(); }
  void alloc(size_t b, cudaStream_t stream);
  void release();       // stream-ordered on s
  void release_sync();  // cudaFree
  template <class T> T* as() const { return static_cast<T*>(p); }
};

// Owning pinned host buffer (cudaHostAlloc), grown on demand.
struct HostBuf {
  void* p = nullptr;
  size_t bytes = 0;
  HostBuf() = default;
  HostBuf(const HostBuf&) = delete;
  HostBuf& operator=(const HostBuf&) = delete;
  ~HostBuf() {
    if (p) cudaFreeHost(p);
  }
  template <class T> T* as() const { return static_cast<T*>(p); }
};

// Function-local temporary: freed stream-ordered at scope exit (its stream
// is alive for the whole call), so temporaries never synchronise the device.
struct TBuf : DBuf {
  ~TBuf() { release(); }
};

struct Ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[7] = {};
  cudaStream_t aux[2] = {};  // graph-capture helpers (device loop)
  // operator-API scratch
  DBuf ctl, status, qstatus;
  size_t status_cap = 0;
  Ctl* ctl_host = nullptr;  // pinned mirror
  ~Ctx();
  void ensure_status(size_t n);
  void sync();
  Ctl read_ctl(const Ctl* dctl);
};

struct Workspace;

struct Graph {
  Ctx* ctx = nullptr;
  uint64_t n = 0, m = 0;
  uint64_t col_bound = 0;  // destination ids must be < col_bound (= n, or n_global for a partition)
  int wtype = GFB_W_F32;
  bool csc_wanted = false;  // the caller asked for the transpose (build_transpose)
  bool has_csc = false;     // ... and it is built for the current contents (ensure_csc)
  DBuf ro, adj, co, cadj, ceid;  // ceid built lazily (ensure_ceid) for the record op
  DBuf stage;                     // upload staging, kept for refills
  HostBuf hstage;                 // pinned f64 -> f32 narrowing buffers (fill_graph)
  cudaEvent_t hdone[2] = {};      // ... and the copies that last read them
  // A refill whose validation failed has already overwritten ro / adj: the
  // handle is unusable (every entry point rejects it) until a good refill.
  bool poisoned = false;
  // In-degree-ordered copy of the CSR used inside the SSSP loop (ensure_relabel):
  // new id i = rank of vertex iperm[i] by descending in-degree, so the hot
  // destinations share distance cache lines.  4-byte weights only.
  DBuf rl_ro, rl_adj, rl_perm, rl_iperm;
  bool rl_valid = false;
  uint32_t runs_since_fill = 0;  // sssp calls on the current contents (relabel pays on reuse)
  int64_t max_outdeg = -1;        // cached (max_out_degree), -1: not computed
  double mean_w = -1;             // cached (mean_weight), -1: not computed
  bool rl_skip = false;  // in-degrees not skewed enough to pay (no arrays built)
  // static pull plan (destinations with in-degree > 0)
  uint32_t pull_k = 0, pull_total = 0;
  DBuf pull_v, pull_off, pull_tseg;
  std::unique_ptr<Workspace> ws;
  ~Graph();
  size_t rec_bytes() const { return wtype == GFB_W_F64 ? 16 : 8; }
};

struct Frontier {
  Ctx* ctx = nullptr;
  uint64_t n = 0;
  int repr = GFB_SPARSE;
  DBuf list;      // sparse: u32[cap]
  uint64_t len = 0, cap = 0;
  DBuf bits;      // dense: u32[nwords]
  uint64_t nwords() const { return (n + 31) / 32; }
  void reserve(uint64_t c);
};

struct Dist {
  Ctx* ctx = nullptr;
  const Graph* g = nullptr;
  DBuf dist, predrec, ctl;
  unsigned long long relax = 0;
};

struct Record {
  Ctx* ctx = nullptr;
  uint64_t cap = 0;
  DBuf src, dst, eid;
  uint64_t count = 0;
};

// SSSP working memory, cached on the graph.
struct Workspace {
  DBuf dist, predrec, pred, res, cand;
  DBuf bm_next, bm_cur, repair_bm;
  DBuf pv, pstart, poff, ptseg;
  DBuf ctl;
  DBuf agg;        // per-tile (count, edges) of bfs.cu's frontier compaction
  DBuf oagg, obuck; // distance-ordered filter: (tile, bucket) cells, bucket totals / cursors
  DBuf tq, tctr;    // tail kernel (tail.cuh): two vertex queues, rotating counters
  int tail_grid = 0;
  DBuf src_dev;    // the source vertex (read by k_init)
  DBuf dist_int, pkey_int;          // loop state in relabelled ids (ensure_relabel)
  DBuf nf_q, nf_bm, nf_cnt;         // near-far queues / bitmaps / counters (nearfar.cuh)
  uint32_t ftiles = 0;
  // device loop: one instantiated CUDA graph for the last (direction, alpha,
  // relabel, deferral, tile) key.  It holds raw pointers into the graph's and
  // this workspace's buffers: invalidate_loop_graphs() on every reallocation.
  cudaGraphExec_t loop_exec = nullptr;
  cudaGraph_t loop_graph = nullptr;
  int loop_key[6] = {-1, -1, -1, -1, -1, -1};
  cudaGraphExec_t bfs_exec = nullptr;  // bfs.cu device loop
  cudaGraph_t bfs_graph = nullptr;
  int bfs_key = -1;
  Ctl* ctl_host = nullptr;  // pinned
  int wtype = -1;
  bool has_result = false;
  uint32_t source = 0;
  ~Workspace();
};

// One rank of the 1-D partitioned SSSP (mg.cu).
struct Part {
  Ctx* ctx = nullptr;
  std::unique_ptr<Graph> g;  // local CSR slice, global column ids
  uint64_t n_global = 0;
  uint32_t lo = 0, hi = 0;
  DBuf dist, predrec, bm_next, bm_cur, pv, pstart, poff, ptseg, agg, ctl;
  DBuf rbest, rbm, ragg, rtot, counts;
  uint32_t ftiles = 0, rtiles = 0;
  unsigned long long relax = 0;
  uint32_t supersteps = 0;
};

// One rank of the peer-memory partitioned SSSP (peer.cu).
struct Peer;
Peer* peer_create(Ctx*, int rank, int nparts, const uint32_t* range_starts, uint64_t m_local,
                  const uint32_t* ro, const uint32_t* col, const void* w, int htype, int wtype);
void peer_export(Peer*, void* handle);
void peer_link(Peer*, const void* handles);
void peer_sssp(Peer*, uint32_t source, const gfb_sssp_opts*, gfb_sssp_stats*);
void peer_read(Peer*, double* dist, void* dist_native, uint32_t* pred);
void peer_free(Peer*);
Ctx* peer_ctx(Peer*);
// One process driving every partition (peer.cu): ctx[q] runs partition q.
// exchange: GFB_EXCHANGE_PEER (device-initiated over peer memory, peer.cu)
// or GFB_EXCHANGE_NCCL (host-driven bucketed messages over NCCL, xmg.cu).
struct Xmg;
struct Mg {
  std::vector<Ctx*> ctx;  // owned through the C ABI (gfb_ctx_create / destroy)
  std::vector<Peer*> peers;
  std::vector<uint32_t> starts;
  uint64_t n = 0;
  int wtype = -1;
  int exchange = GFB_EXCHANGE_PEER;
  Xmg* x = nullptr;
};
Xmg* xmg_create(const std::vector<Ctx*>& ctx);
void xmg_free(Xmg*);
bool xmg_uses_nccl(const Xmg*);
void xmg_upload(Xmg*, const std::vector<uint32_t>& starts, uint64_t n, const uint32_t* ro,
                const uint32_t* col, const void* w, int htype, int wtype);
void xmg_sssp(Xmg*, uint32_t source, const gfb_sssp_opts*, double* dist, uint32_t* pred,
              gfb_sssp_stats*);
void mg_upload(Mg*, uint64_t n, uint64_t m, const uint32_t* ro, const uint32_t* col,
               const void* w, int htype, int wtype);
void mg_sssp(Mg*, uint32_t source, const gfb_sssp_opts*, double* dist, uint32_t* pred,
             gfb_sssp_stats*);
void mg_free(Mg*);

// grid sizes
inline int stride_grid(const Ctx* c) { return c->num_sms * 8; }
inline int persist_grid(const Ctx* c, int per_sm) { return c->num_sms * per_sm; }

// graph.cu
void relabel_ranges(Graph* g, uint32_t nparts, const uint32_t* starts, uint32_t* ro_out,
                    uint32_t* col_out, void* w_out, uint32_t* perm_out);
void build_csc(Graph* g);
void ensure_csc(Graph* g);
void ensure_ceid(Graph* g);
void build_pull_plan(Graph* g);
// destroy the cached device-loop graphs of g (their pointers went stale)
void invalidate_loop_graphs(Graph* g);
// GFB_ELOGIC if a failed refill left g's contents invalid
void check_usable(const Graph* g);
void ensure_relabel(Graph* g);
uint32_t max_out_degree(Graph* g);
double mean_weight(Graph* g);
// bfs.cu
void bfs_run(Ctx* c, Graph* g, uint32_t source, int direction, double* depth,
             uint64_t* supersteps, uint64_t* relaxations);
// sssp.cu
void sssp_run(Ctx* ctx, Graph* g, uint32_t source, const gfb_sssp_opts* o, gfb_sssp_stats* st);
void sssp_read(Graph* g, double* dist, void* dist_native, uint32_t* pred);
Workspace* ensure_ws(Graph* g);
// mg.cu
Part* part_create(Ctx*, uint64_t n_global, uint32_t lo, uint32_t hi, uint64_t m_local,
                  const uint32_t* ro, const uint32_t* col, const void* w, int htype, int wtype);
void part_init(Part*, uint32_t source);
uint64_t part_advance(Part*, void* out, uint64_t cap, const uint32_t* range_starts, int nparts,
                      uint32_t* counts_host);
void part_apply(Part*, const void* in, uint64_t count);
uint64_t part_pending(Part*);
void part_read(Part*, void* dist_native, uint64_t* relax, uint64_t* supersteps);
void part_pred(Part*, const void* gdist, const uint32_t* res, uint32_t* cand, uint32_t round);

}  // namespace gfb

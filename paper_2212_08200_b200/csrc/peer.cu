// peer.cu -- the 1-D partitioned SSSP with a device-initiated exchange over
// peer memory.
//
// Same partition as mg.cu (contiguous vertex ranges with edge-balanced cut
// points, here rounded to multiples of 32 so bitmap words never straddle two
// owners; each rank holds the CSR rows of its range with GLOBAL column ids),
// but no messages and no host round trip per superstep:
//   * every rank allocates its loop state (distances, packed (dist, pred)
//     keys, next-frontier bitmap, repair state, barrier mailbox) in ONE
//     cudaMalloc slab and exports it with cudaIpcGetMemHandle; the handles are
//     exchanged once (torch.distributed all_gather_object in peer.py) and
//     opened with cudaIpcOpenMemHandle -- on an NVSwitch node every peer slab
//     is then directly addressable over NVLink;
//   * the advance (k_push_range<PEER>) resolves each destination's owner from
//     the range table and issues its test-before-atomic gather and its
//     red.min / red.min.64 / red.or straight into the owner's slab: the
//     exchange IS the advance, overlapped edge by edge with the local work;
//   * a cross-rank barrier kernel (k_xbar, one warp: release-store of this
//     rank's counters into every peer's mailbox, acquire-spin on its own)
//     separates the advance from the owners' compaction and publishes the
//     global frontier minimum and the global frontier size, which sets the
//     WHILE condition of the per-rank CUDA graph -- the convergence
//     allreduce of algorithms.hpp:167 done by the device;
//   * compaction (the distance-ordered k_fcount_o / k_fscan_o / k_fwrite_o,
//     deferral included) is purely local: each rank owns its bitmaps -- the
//     local one (bits set by relaxations that lowered a distance) and the
//     remote one (rbm: bits peers set after testing against their proposal
//     cache, merged by the filter only where dexp shows the distance moved
//     since the vertex's last expansion; one rank: no remote bitmap, no dexp
//     traffic -- s24 4.19 -> 3.84 ms).
// Predecessors: the packed keys already live at the owners; verification
// reads the key source's distance through the peer table; the rare
// tie-class repair runs the single-GPU round rules with barriers between
// rounds.  4-byte distances (f32 / u32) only, like mg.cu.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "frontier.cuh"
#include "hot.cuh"
#include "impl.hpp"

namespace gfb {

Graph* graph_upload(Ctx*, uint64_t, uint64_t, const uint32_t*, const uint32_t*, const void*, int,
                    int, int, uint64_t);

// ---- slab layout (identical on every rank for a given range length) ------
constexpr uint32_t MBOX_WORDS = 8;  // per (parity, rank): epoch, k, fmin, flag, unres, resolved, err
struct PeerLayout {
  size_t dist, pkey, bm, rbm, res, cand, repair, mbox, bytes;
};
static PeerLayout peer_layout(uint64_t nq) {
  auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
  const uint64_t words = (nq + 31) / 32;
  PeerLayout l{};
  size_t o = 0;
  l.dist = o;   o = up(o + nq * 4);
  l.pkey = o;   o = up(o + nq * 8);
  l.bm = o;     o = up(o + words * 4);
  l.rbm = o;    o = up(o + words * 4);
  l.res = o;    o = up(o + nq * 4);
  l.cand = o;   o = up(o + nq * 4);
  l.repair = o; o = up(o + words * 4);
  l.mbox = o;   o = up(o + 2 * PEER_MAX * MBOX_WORDS * 4);
  l.bytes = o;
  return l;
}

// ---- cross-rank barrier ----------------------------------------------------
enum { XB_PLAIN = 0, XB_FMIN = 1, XB_LOOP = 2 };
struct XBarArgs {
  uint32_t* mbox[PEER_MAX];  // every rank's mailbox (own included)
  uint32_t nparts, self;
  uint32_t* epoch;           // this rank's barrier count (device, monotonic)
  Ctl* ctl;
  cudaGraphConditionalHandle loop;
  int set_loop, mode;
  unsigned long long timeout_ns;
};

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// One warp.  Barrier e writes mailbox parity e & 1: a peer can only reuse a
// parity (barrier e + 2) after passing e + 1, which needs this rank's e + 1
// record, written after this rank finished reading e.  Every rank runs the
// same barrier sequence, so epochs agree.  The fence.sc.sys before the
// release orders this rank's previous kernels' peer reductions (complete at
// the kernel boundary) before the record.
__global__ void __launch_bounds__(32) k_xbar(XBarArgs b) {
  const uint32_t lane = threadIdx.x;
  Ctl* c = b.ctl;
  const uint32_t e = *b.epoch + 1;
  __syncwarp();
  if (lane == 0) *b.epoch = e;
  const uint32_t par = e & 1u;
  const uint32_t mine[6] = {c->k, c->fmin, c->flag, c->unresolved, c->resolved, c->err};
  __threadfence_system();
  if (lane < b.nparts) {
    uint32_t* slot = b.mbox[lane] + (par * PEER_MAX + b.self) * MBOX_WORDS;
#pragma unroll
    for (int j = 0; j < 6; ++j) st_relaxed_sys(slot + 1 + j, mine[j]);
    st_release_sys(slot, e);
  }
  uint32_t v[6] = {0, 0xFFFFFFFFu, 0, 0, 0, 0};
  uint32_t timed_out = 0;
  if (lane < b.nparts) {
    const uint32_t* slot = b.mbox[b.self] + (par * PEER_MAX + lane) * MBOX_WORDS;
    const unsigned long long t0 = globaltimer();
    while (ld_acquire_sys(slot) != e) {
      if (globaltimer() - t0 > b.timeout_ns) {
        timed_out = 1;
        break;
      }
      __nanosleep(64);
    }
    if (!timed_out) {
#pragma unroll
      for (int j = 0; j < 6; ++j) v[j] = ld_relaxed_sys(slot + 1 + j);
    }
  }
  uint32_t gk = v[0], gmin = v[1], gflag = v[2], gun = v[3], gres = v[4], gerr = v[5];
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    gk += __shfl_xor_sync(0xffffffffu, gk, d);
    gmin = min(gmin, __shfl_xor_sync(0xffffffffu, gmin, d));
    gflag += __shfl_xor_sync(0xffffffffu, gflag, d);
    gun += __shfl_xor_sync(0xffffffffu, gun, d);
    gres += __shfl_xor_sync(0xffffffffu, gres, d);
    gerr |= __shfl_xor_sync(0xffffffffu, gerr, d);
    timed_out |= __shfl_xor_sync(0xffffffffu, timed_out, d);
  }
  if (lane == 0) {
    c->gk = gk;
    c->gflag = gflag;
    c->gunres = gun;
    c->gresolved = gres;
    if (b.mode == XB_FMIN) c->fmin = gmin;  // every rank buckets from the global minimum
    c->err |= (gerr & 1u) | (timed_out ? 8u : 0u);
    if (b.set_loop)
      cudaGraphSetConditional(b.loop, (gk > 0 && !timed_out && !(gerr & 1u)) ? 1u : 0u);
  }
}

// ---- init / predecessor kernels -------------------------------------------
template <class W>
__global__ void k_peer_init(typename DT<W>::D* dist, unsigned long long* pkey, uint32_t* bm_next,
                            uint32_t* bm_cur, uint32_t* res, uint32_t* cand, uint32_t* repair,
                            uint32_t n, uint32_t nwords, const uint32_t* src_local, Ctl* ctl,
                            uint32_t* dexp, uint32_t* rbm) {
  using D = typename DT<W>::D;
  const uint32_t s = *src_local;  // NIL when the source lives on another rank
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    dist[i] = i == s ? D(0) : dinf<W>();
    pkey[i] = ~0ull;
    res[i] = 0;
    cand[i] = NIL;
    dexp[i] = 0xFFFFFFFFu;  // never expanded (no distance has these bits)
  }
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nwords; i += stride) {
    bm_next[i] = (s != NIL && (s >> 5) == i) ? (1u << (s & 31)) : 0u;
    bm_cur[i] = 0;
    rbm[i] = 0;
    repair[i] = 0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    Ctl c0 = {};
    *ctl = c0;
  }
}

// Owner of every destination into the top bits of its id (PEER_VBITS).
struct Starts {
  uint32_t s[PEER_MAX + 1];
  uint32_t nparts;
};
template <class W>
__global__ void k_peer_encode(EdgeRec<W>* adj, uint64_t m, Starts st) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t v = adj[e].v;
    uint32_t q = 0;
    for (uint32_t i = 1; i < st.nparts; ++i) q += v >= st.s[i] ? 1u : 0u;
    adj[e].v = v | (q << PEER_VBITS);
  }
}

__global__ void k_peer_fill(uint32_t* a, uint32_t v, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    a[i] = v;
}

__device__ __forceinline__ void load_tab(PeerTab* s, const PeerTab* g) {
  for (int i = threadIdx.x; i < (int)(sizeof(PeerTab) / 4); i += blockDim.x)
    reinterpret_cast<uint32_t*>(s)[i] = reinterpret_cast<const uint32_t*>(g)[i];
  __syncthreads();
}

// Verification at the owner: the key (dist_bits << 32 | u_global) is
// accepted when its distance is dist[v] and dist[u] < dist[v] (u read
// through the peer table); else v joins the local repair list.
template <class W>
__global__ void __launch_bounds__(256)
k_peer_verify(const uint32_t* __restrict__ ro, const PeerTab* tab,
              const typename DT<W>::D* __restrict__ dist, const unsigned long long* __restrict__ pkey,
              uint32_t* pred, uint32_t* res, uint32_t* repair, uint32_t* list, uint32_t n,
              uint32_t src_local, Ctl* ctl) {
  using D = typename DT<W>::D;
  __shared__ PeerTab t;
  load_tab(&t, tab);
  unsigned long long nr = 0, mr = 0;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const D dv = dist[v];
    uint32_t p = NIL, rr = 0;
    if (!(dv == dinf<W>())) {
      ++nr;
      mr += ro[v + 1] - ro[v];
      if (v == src_local) {
        rr = 1;
      } else {
        const unsigned long long k = pkey[v];
        const uint32_t u = (uint32_t)k;
        if (u != NIL && (uint32_t)(k >> 32) == *reinterpret_cast<const uint32_t*>(&dv)) {
          const uint32_t q = peer_owner(t, u);
          const D du = __ldcg(reinterpret_cast<const D*>(t.dist[q]) + u);
          if (du < dv) {
            p = u;
            rr = 1;
          }
        }
        if (!rr) {
          atomicOr(repair + (v >> 5), 1u << (v & 31));
          list[atomicAdd(&ctl->unresolved, 1u)] = v;  // rare: zero-weight ties
        }
      }
    }
    pred[v] = p;
    res[v] = rr;
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    nr += __shfl_xor_sync(0xffffffffu, nr, d);
    mr += __shfl_xor_sync(0xffffffffu, mr, d);
  }
  if ((threadIdx.x & 31) == 0) {
    if (nr) atomicAdd(&ctl->n_reach, nr);
    if (mr) atomicAdd(&ctl->m_reach, mr);
  }
}

// Key round k (as k_pred_key_round): the key source u has dist[u] == dist[v];
// accept once u is resolved with res[u] <= k (res read at u's owner).
template <class W>
__global__ void k_peer_key_round(const uint32_t* __restrict__ list, const PeerTab* tab,
                                 const unsigned long long* __restrict__ pkey,
                                 const typename DT<W>::D* __restrict__ dist, uint32_t* pred,
                                 uint32_t* res, uint32_t* repair, uint32_t k, Ctl* ctl) {
  using D = typename DT<W>::D;
  __shared__ PeerTab t;
  load_tab(&t, tab);
  const uint32_t count = ctl->unresolved;
  uint32_t done = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
    const uint32_t v = list[i];
    if (res[v] != 0) continue;
    const uint32_t u = (uint32_t)pkey[v];
    if (u == NIL) continue;
    const uint32_t q = peer_owner(t, u);
    if (!(__ldcg(reinterpret_cast<const D*>(t.dist[q]) + u) == dist[v])) continue;
    const uint32_t ru = __ldcg(t.res[q] + u);
    if (ru != 0 && ru <= k) {
      pred[v] = u;
      res[v] = k + 1;
      atomicAnd(repair + (v >> 5), ~(1u << (v & 31)));
      ++done;
    }
  }
  done = warp_sum(done);
  if ((threadIdx.x & 31) == 0 && done) atomicAdd(&ctl->resolved, done);
}

// In-edge collection: this rank's out-edges u -> v whose owner flags v in its
// repair bitmap (one warp per row), as {u_global, v_global, w, 0}.
template <class W>
__global__ void k_peer_inedges(const uint32_t* __restrict__ ro, const EdgeRec<W>* __restrict__ adj,
                               const PeerTab* tab, uint32_t n, uint4* list, uint32_t cap,
                               Ctl* ctl) {
  __shared__ PeerTab t;
  load_tab(&t, tab);
  const int lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n; u += warps) {
    const uint32_t s0 = ro[u], s1 = ro[u + 1];
    for (uint32_t e = s0 + lane; e < s1; e += 32) {
      const EdgeRec<W> r = adj[e];
      const uint32_t q = r.v >> PEER_VBITS, v = r.v & PEER_VMASK;  // owner-encoded
      if ((__ldcg(t.repair[q] + (v >> 5)) >> (v & 31)) & 1u) {
        const uint32_t i = atomicAdd(&ctl->out_count, 1u);
        if (i < cap) list[i] = make_uint4(u + t.self_lo, v, *reinterpret_cast<const uint32_t*>(&r.w), 0u);
        else atomicOr(&ctl->err, 4u);
      }
    }
  }
}

// One repair round over the collected edges (k_pred_list_round's rule); the
// candidate goes to cand at v's owner.
template <class W>
__global__ void k_peer_list_round(const uint4* __restrict__ list, const Ctl* __restrict__ ctl,
                                  uint32_t cap, const PeerTab* tab, uint32_t round, uint32_t base) {
  using D = typename DT<W>::D;
  __shared__ PeerTab t;
  load_tab(&t, tab);
  const uint32_t cnt = min(ctl->out_count, cap);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
    const uint4 e = list[i];
    const uint32_t qv = peer_owner(t, e.y), qu = peer_owner(t, e.x);
    if (__ldcg(t.res[qv] + e.y) != 0) continue;
    const W w = *reinterpret_cast<const W*>(&e.z);
    const D du = __ldcg(reinterpret_cast<const D*>(t.dist[qu]) + e.x);
    const D dv = __ldcg(reinterpret_cast<const D*>(t.dist[qv]) + e.y);
    if (du == dinf<W>() || !(dadd(du, w, nullptr) == dv)) continue;
    bool ok;
    if (round == 1) {
      ok = du < dv;
    } else {
      const uint32_t ru = __ldcg(t.res[qu] + e.x);
      ok = du == dv && ru != 0 && ru <= base + round;
    }
    if (ok) atomicMin(t.cand[qv] + e.y, e.x);
  }
}

// ---- host side --------------------------------------------------------------
struct Peer {
  Ctx* ctx = nullptr;
  std::unique_ptr<Graph> g;  // local CSR rows, global column ids
  int rank = 0, nparts = 1;
  std::vector<uint32_t> starts;
  uint64_t n_global = 0;
  uint32_t lo = 0, n = 0, nwords = 0;
  void* slab = nullptr;
  PeerLayout lay{};
  std::vector<void*> opened;  // mapped peer slabs (nullptr for self)
  std::vector<char*> bases;   // every rank's slab base as seen from this rank
  bool linked = false;
  PeerTab tab{};
  DBuf tab_dev, ctl, epoch, src_dev, bm_cur, pred, list, pv, pstart, poff, ptseg, oagg, obuck;
  DBuf rc;     // proposal cache for remote destinations (n_global, nparts > 1)
  DBuf rlist;  // predecessor repair: this rank's edges into unresolved vertices
  DBuf dexp;   // distance bits each local vertex was last expanded with
  uint64_t call_l0 = 0;
  uint32_t ftiles = 0;
  cudaGraphExec_t exec = nullptr;
  cudaGraph_t graph = nullptr;
  int graph_key = -1;
  bool has_result = false;
  uint64_t launches = 0;

  template <class T> T* at(size_t off) const { return reinterpret_cast<T*>((char*)slab + off); }
  ~Peer() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    for (void* p : opened)
      if (p) cudaIpcCloseMemHandle(p);
    if (slab) cudaFree(slab);
  }
};

Peer* peer_create(Ctx* c, int rank, int nparts, const uint32_t* range_starts, uint64_t m_local,
                  const uint32_t* ro, const uint32_t* col, const void* w, int htype, int wtype) {
  if (nparts < 1 || nparts > PEER_MAX) fail(GFB_EINVAL, "peer: 1 <= nparts <= 8");
  if (rank < 0 || rank >= nparts) fail(GFB_EINVAL, "peer: rank out of range");
  if (wtype != GFB_W_F32 && wtype != GFB_W_U32)
    fail(GFB_EINVAL, "peer: partitioned SSSP needs 4-byte distances (f32 / u32 weights)");
  if (range_starts[0] != 0) fail(GFB_EINVAL, "peer: range_starts[0] must be 0");
  for (int q = 0; q < nparts; ++q) {
    if (range_starts[q + 1] < range_starts[q]) fail(GFB_EINVAL, "peer: range_starts must ascend");
    if (q > 0 && (range_starts[q] & 31u)) fail(GFB_EINVAL, "peer: range starts must be multiples of 32");
  }
  auto p = std::make_unique<Peer>();
  p->ctx = c;
  p->rank = rank;
  p->nparts = nparts;
  p->starts.assign(range_starts, range_starts + nparts + 1);
  p->n_global = range_starts[nparts];
  p->lo = range_starts[rank];
  p->n = range_starts[rank + 1] - p->lo;
  p->nwords = (p->n + 31) / 32;
  cudaStream_t s = c->stream;
  if (p->n_global >= (1ull << PEER_VBITS)) fail(GFB_EINVAL, "peer: n must be < 2^29");
  p->g.reset(graph_upload(c, p->n, m_local, ro, col, w, htype, wtype, 0, p->n_global));
  {  // owner-encoded destination ids (the advance decodes them with a shift)
    Starts st{};
    for (int q = 0; q <= nparts; ++q) st.s[q] = range_starts[q];
    st.nparts = (uint32_t)nparts;
    if (m_local) {
      if (wtype == GFB_W_F32)
        k_peer_encode<float><<<stride_grid(c), 256, 0, s>>>(p->g->adj.as<EdgeRec<float>>(), m_local, st);
      else
        k_peer_encode<uint32_t><<<stride_grid(c), 256, 0, s>>>(p->g->adj.as<EdgeRec<uint32_t>>(), m_local, st);
      GFB_CUDA(cudaGetLastError());
    }
  }
  p->lay = peer_layout(p->n);
  GFB_CUDA(cudaMalloc(&p->slab, p->lay.bytes));  // plain cudaMalloc: IPC-exportable
  GFB_CUDA(cudaMemsetAsync(p->at<char>(p->lay.mbox), 0, 2 * PEER_MAX * MBOX_WORDS * 4, s));
  const uint64_t n1 = (uint64_t)p->n + 1;
  p->ctl.alloc(sizeof(Ctl), s);
  GFB_CUDA(cudaMemsetAsync(p->ctl.p, 0, sizeof(Ctl), s));
  p->epoch.alloc(16, s);
  GFB_CUDA(cudaMemsetAsync(p->epoch.p, 0, 16, s));
  p->src_dev.alloc(16, s);
  p->bm_cur.alloc((size_t)std::max<uint32_t>(p->nwords, 1) * 4, s);
  p->pred.alloc(n1 * 4, s);
  p->list.alloc(n1 * 4, s);
  p->pv.alloc(n1 * 4, s);
  p->pstart.alloc(n1 * 4, s);
  p->poff.alloc(n1 * 4, s);
  p->ptseg.alloc((m_local / PLAN_GRAIN + 3) * 4, s);
  p->ftiles = (uint32_t)std::max<uint64_t>((p->nwords + F_WORDS - 1) / F_WORDS, 1);
  p->oagg.alloc((size_t)p->ftiles * (OB_N * 8 + 4), s);
  p->obuck.alloc(2 * OB_N * 8, s);
  GFB_CUDA(cudaMemsetAsync(p->obuck.p, 0, 2 * OB_N * 8, s));
  p->tab_dev.alloc(sizeof(PeerTab), s);
  p->dexp.alloc(n1 * 4, s);
  c->sync();
  return p.release();
}

void peer_export(Peer* p, void* handle) {
  cudaIpcMemHandle_t h;
  GFB_CUDA(cudaIpcGetMemHandle(&h, p->slab));
  std::memcpy(handle, &h, sizeof(h));
}

// Peer table from every rank's slab base (own slab included).
static void peer_link_bases(Peer* p, const std::vector<char*>& bases) {
  PeerTab& t = p->tab;
  t = PeerTab{};
  for (int q = 0; q <= p->nparts; ++q) t.start[q] = p->starts[q];
  for (int q = p->nparts + 1; q <= PEER_MAX; ++q) t.start[q] = (uint32_t)p->n_global;
  p->bases = bases;
  for (int q = 0; q < p->nparts; ++q) {
    const PeerLayout l = peer_layout(p->starts[q + 1] - p->starts[q]);
    const uint32_t s0 = p->starts[q];
    char* base = bases[q];
    // pre-offset so that index = global id (s0 is a multiple of 32)
    t.dist[q] = reinterpret_cast<uint32_t*>(base + l.dist) - s0;
    t.pkey[q] = reinterpret_cast<unsigned long long*>(base + l.pkey) - s0;
    // a peer's frontier bits go to its remote bitmap (checked against dexp)
    t.bm[q] = reinterpret_cast<uint32_t*>(base + (q == p->rank ? l.bm : l.rbm)) - (s0 >> 5);
    t.res[q] = reinterpret_cast<uint32_t*>(base + l.res) - s0;
    t.cand[q] = reinterpret_cast<uint32_t*>(base + l.cand) - s0;
    t.repair[q] = reinterpret_cast<uint32_t*>(base + l.repair) - (s0 >> 5);
  }
  if (p->nparts > 1) {
    p->rc.alloc(p->n_global * 4, p->ctx->stream);
    t.rc = p->rc.as<uint32_t>();
  }
  t.nparts = (uint32_t)p->nparts;
  t.self = (uint32_t)p->rank;
  t.self_lo = p->lo;
  GFB_CUDA(cudaMemcpyAsync(p->tab_dev.p, &t, sizeof(t), cudaMemcpyHostToDevice, p->ctx->stream));
  p->ctx->sync();
  p->linked = true;
}

// Multi-process: open the peers' exported slabs (NVLink peer mappings).
void peer_link(Peer* p, const void* handles) {
  if (p->linked) fail(GFB_ELOGIC, "peer: already linked");
  p->opened.assign(p->nparts, nullptr);
  std::vector<char*> bases(p->nparts);
  for (int q = 0; q < p->nparts; ++q) {
    if (q == p->rank) {
      bases[q] = static_cast<char*>(p->slab);
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const char*>(handles) + (size_t)q * sizeof(h), sizeof(h));
    void* ptr = nullptr;
    GFB_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    p->opened[q] = ptr;
    bases[q] = static_cast<char*>(ptr);
  }
  peer_link_bases(p, bases);
}

// One process, all ranks: direct pointers (peer access between devices).
static void peer_link_local(const std::vector<Peer*>& ps) {
  std::vector<char*> bases;
  for (Peer* p : ps) bases.push_back(static_cast<char*>(p->slab));
  for (Peer* a : ps) {
    GFB_CUDA(cudaSetDevice(a->ctx->device));
    for (Peer* b : ps) {
      if (b->ctx->device == a->ctx->device) continue;
      int ok = 0;
      GFB_CUDA(cudaDeviceCanAccessPeer(&ok, a->ctx->device, b->ctx->device));
      if (!ok) fail(GFB_ECUDA, "mg: no peer access between devices");
      const cudaError_t e = cudaDeviceEnablePeerAccess(b->ctx->device, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else GFB_CUDA(e);
    }
    peer_link_bases(a, bases);
  }
}

static unsigned long long peer_timeout_ns() {
  const char* e = getenv("GFB_PEER_TIMEOUT_S");
  const double s = e ? atof(e) : 30.0;
  return (unsigned long long)(s * 1e9);
}

template <class W>
struct PeerRun {
  using D = typename DT<W>::D;
  Peer* p;
  Ctx* c;
  cudaStream_t s;

  D* dist() const { return p->at<D>(p->lay.dist); }
  unsigned long long* pkey() const { return p->at<unsigned long long>(p->lay.pkey); }
  uint32_t* bm() const { return p->at<uint32_t>(p->lay.bm); }
  uint32_t* rbm() const { return p->at<uint32_t>(p->lay.rbm); }
  uint32_t* res() const { return p->at<uint32_t>(p->lay.res); }
  uint32_t* cand() const { return p->at<uint32_t>(p->lay.cand); }
  uint32_t* repair() const { return p->at<uint32_t>(p->lay.repair); }
  Ctl* ctl() const { return p->ctl.as<Ctl>(); }
  Plan plan() const {
    return Plan{p->pv.as<uint32_t>(), p->pstart.as<uint32_t>(), p->poff.as<uint32_t>(),
                p->ptseg.as<uint32_t>(), (uint32_t)(p->ptseg.bytes / 4)};
  }

  void xbar(cudaStream_t st, int mode, cudaGraphConditionalHandle h = {}, bool set_loop = false) {
    XBarArgs b{};
    for (int q = 0; q < p->nparts; ++q) {
      const PeerLayout l = peer_layout(p->starts[q + 1] - p->starts[q]);
      b.mbox[q] = reinterpret_cast<uint32_t*>(p->bases[q] + l.mbox);
    }
    b.nparts = (uint32_t)p->nparts;
    b.self = (uint32_t)p->rank;
    b.epoch = p->epoch.as<uint32_t>();
    b.ctl = ctl();
    b.loop = h;
    b.set_loop = set_loop ? 1 : 0;
    b.mode = mode;
    b.timeout_ns = peer_timeout_ns();
    k_xbar<<<1, 32, 0, st>>>(b);
    ++p->launches;
  }

  void compact(cudaStream_t st, uint32_t defer_pct, cudaGraphConditionalHandle hl = {},
               bool set_loop = false) {
    Graph* g = p->g.get();
    const uint32_t tiles = p->ftiles;
    unsigned long long* bt = p->obuck.as<unsigned long long>();
    uint32_t* tflag =
        reinterpret_cast<uint32_t*>(p->oagg.as<unsigned long long>() + (size_t)tiles * OB_N);
    cudaGraphConditionalHandle none{};
    // one rank: every frontier bit is local (no remote bitmap, no dexp)
    uint32_t* dx = p->nparts > 1 ? p->dexp.as<uint32_t>() : nullptr;
    uint32_t* rb = p->nparts > 1 ? rbm() : nullptr;
    k_fcount_o<D, true><<<tiles, F_WARPS * 32, 0, st>>>(g->ro.as<uint32_t>(), bm(), p->nwords, dist(),
                                                  ctl(), p->oagg.as<unsigned long long>(), bt,
                                                  tflag, dx, rb);
    k_fscan_o<<<1, 32, 0, st>>>(bt, bt + OB_N, plan(), ctl(), (uint32_t)g->m, 1.0f, 0, 0, hl,
                                none, set_loop ? 1 : 0, 0, defer_pct, (uint32_t)(g->m >> 2));
    k_fwrite_o<D, true><<<tiles, F_WARPS * 32, 0, st>>>(g->ro.as<uint32_t>(), bm(),
                                                  p->bm_cur.as<uint32_t>(), p->nwords, dist(),
                                                  ctl(), p->oagg.as<unsigned long long>(),
                                                  bt + OB_N, plan(), tflag, dx, rb);
    p->launches += 3;
  }

  void push(cudaStream_t st) {
    AdvArgs<W> a{};
    a.adj = p->g->adj.as<EdgeRec<W>>();
    a.dist = dist();
    a.predrec = reinterpret_cast<uint2*>(pkey());
    a.plan = plan();
    a.ctl = ctl();
    a.bm_out = bm();
    a.op = GFB_OP_RELAX_MIN;
    a.peers = p->tab_dev.as<PeerTab>();
    if constexpr (sizeof(D) == 4) {
      k_push_range<W, 1, 6, 256, 17, true><<<c->num_sms * 6, 256, 0, st>>>(a);
    }
    ++p->launches;
  }

  // B0 (everyone finished the previous call) -> init -> first compaction ->
  // B2 (global frontier size) -> WHILE { push -> B1 (global fmin) ->
  // compaction -> B2 }
  void build(uint32_t defer_pct) {
    if (p->exec) cudaGraphExecDestroy(p->exec);
    if (p->graph) cudaGraphDestroy(p->graph);
    p->exec = nullptr;
    p->graph = nullptr;
    for (auto& a : c->aux)
      if (!a) GFB_CUDA(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking));
    cudaGraph_t G;
    GFB_CUDA(cudaGraphCreate(&G, 0));
    cudaGraphConditionalHandle hloop;
    GFB_CUDA(cudaGraphConditionalHandleCreate(&hloop, G, 1, cudaGraphCondAssignDefault));
    GFB_CUDA(cudaStreamBeginCaptureToGraph(s, G, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    xbar(s, XB_PLAIN);
    k_peer_init<W><<<stride_grid(c), 256, 0, s>>>(dist(), pkey(), bm(), p->bm_cur.as<uint32_t>(),
                                                  res(), cand(), repair(), p->n, p->nwords,
                                                  p->src_dev.as<uint32_t>(), ctl(),
                                                  p->dexp.as<uint32_t>(), rbm());
    if (p->rc.p)  // nothing proposed yet: the unreachable distance's bits
      k_peer_fill<<<stride_grid(c), 256, 0, s>>>(p->rc.as<uint32_t>(),
                                                 std::is_same<D, float>::value ? 0x7F800000u
                                                                               : 0xFFFFFFFFu,
                                                 (uint32_t)p->n_global);
    compact(s, defer_pct);
    xbar(s, XB_LOOP, hloop, true);
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
    push(b);
    xbar(b, XB_FMIN);
    compact(b, defer_pct);
    xbar(b, XB_LOOP, hloop, true);
    GFB_CUDA(cudaStreamEndCapture(b, &tmp));
    GFB_CUDA(cudaGraphInstantiate(&p->exec, G, 0));
    p->graph = G;
  }

  // ---- one call, split into launch steps: the host runs each step on
  // every peer before reading any result (peer_call), because a rank's
  // device barriers only complete when all ranks have launched the step.
  uint32_t defer = 10;
  uint32_t src_local = NIL;

  void prepare(uint32_t source, const gfb_sssp_opts* o) {
    if (!p->linked) fail(GFB_ELOGIC, "peer: gfb_peer_link first");
    if (source >= p->n_global) fail(GFB_ERANGE, "sssp: source out of range");
    if (o->direction == GFB_DIR_PULL) fail(GFB_EINVAL, "peer: the partitioned SSSP is push-only");
    if (o->delta > 0) fail(GFB_EINVAL, "peer: the near-far filter is single-GPU only");
    p->has_result = false;
    // 5%, like the single-GPU loop: s24 at one partition on the relabelled
    // copy 3.81 ms vs 4.00 at 10% with the same 22 supersteps (so the same
    // number of cross-rank barriers; r01, before the relabel and the
    // spill-free filter, 10% won: 5.52-5.60 vs 5.79 ms)
    if (o->defer_pct < 0 || o->defer_pct > 100) fail(GFB_EINVAL, "sssp: defer_pct must be 0..100");
    defer = o->defer_pct ? (uint32_t)o->defer_pct : 5u;
    src_local = (source >= p->lo && source < p->lo + p->n) ? source - p->lo : NIL;
    if (!p->exec || p->graph_key != (int)defer) {
      GFB_CUDA(cudaStreamSynchronize(s));
      build(defer);
      p->graph_key = (int)defer;
    }
    p->call_l0 = p->launches;
    GFB_CUDA(cudaMemcpyAsync(p->src_dev.p, &src_local, 4, cudaMemcpyHostToDevice, s));
    GFB_CUDA(cudaEventRecord(c->ev[0], s));
  }
  void launch_loop() {
    GFB_CUDA(cudaGraphLaunch(p->exec, s));
    p->launches += 0;  // counted from the superstep count after the call
  }
  void launch_verify() {
    k_peer_verify<W><<<c->num_sms * 8, 256, 0, s>>>(p->g->ro.as<uint32_t>(),
                                                    p->tab_dev.as<PeerTab>(), dist(), pkey(),
                                                    p->pred.as<uint32_t>(), res(), repair(),
                                                    p->list.as<uint32_t>(), p->n, src_local, ctl());
    ++p->launches;
    xbar(s, XB_PLAIN);  // every owner's res / repair state visible
  }
  void launch_key_batch(uint32_t base) {
    for (uint32_t k = base + 1; k <= base + 4; ++k) {
      k_peer_key_round<W><<<c->num_sms, 256, 0, s>>>(p->list.as<uint32_t>(),
                                                     p->tab_dev.as<PeerTab>(), pkey(), dist(),
                                                     p->pred.as<uint32_t>(), res(), repair(), k,
                                                     ctl());
      ++p->launches;
      xbar(s, XB_PLAIN);  // res is read across ranks by the next round
    }
  }
  uint32_t launch_inedges() {
    Graph* g = p->g.get();
    const uint32_t cap = (uint32_t)std::min<uint64_t>(g->m + 1, 1u << 24);
    if (p->rlist.bytes < (size_t)cap * 16) p->rlist.alloc((size_t)cap * 16, s);
    GFB_CUDA(cudaMemsetAsync(&ctl()->out_count, 0, 4, s));
    k_peer_inedges<W><<<stride_grid(c), 256, 0, s>>>(g->ro.as<uint32_t>(), g->adj.as<EdgeRec<W>>(),
                                                     p->tab_dev.as<PeerTab>(), p->n,
                                                     p->rlist.as<uint4>(), cap, ctl());
    ++p->launches;
    return cap;
  }
  void launch_round(uint32_t round, uint32_t base, uint32_t cap) {
    GFB_CUDA(cudaMemsetAsync(&ctl()->flag, 0, 4, s));
    k_peer_list_round<W><<<stride_grid(c), 256, 0, s>>>(p->rlist.as<uint4>(), ctl(), cap,
                                                        p->tab_dev.as<PeerTab>(), round, base);
    xbar(s, XB_PLAIN);  // candidates landed at their owners
    k_pred_apply<<<stride_grid(c), 256, 0, s>>>(cand(), p->pred.as<uint32_t>(), res(), repair(),
                                                p->n, round, ctl(), base);
    xbar(s, XB_PLAIN);  // global count of this round's resolutions
    p->launches += 2;
  }
  void finish(gfb_sssp_stats* st, uint64_t fallback) {
    GFB_CUDA(cudaEventRecord(c->ev[1], s));
    const Ctl h = c->read_ctl(ctl());
    check_err(h);
    float ms = 0;
    GFB_CUDA(cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]));
    p->has_result = true;
    p->launches += (p->rc.p ? 7 : 6) + 6ull * h.supersteps;  // the loop graph's kernels
    if (st) {
      *st = gfb_sssp_stats{};
      st->supersteps = h.supersteps;
      st->relaxations = h.relax;
      st->n_reach = h.n_reach;
      st->m_reach = h.m_reach;
      st->push_steps = h.push_steps;
      st->pred_fallback = fallback;
      st->device_ms = ms;
      st->advance_launches = h.supersteps;
      st->kernel_launches = p->launches - p->call_l0;
    }
  }
  Ctl read() {
    const Ctl h = c->read_ctl(ctl());
    check_err(h);
    return h;
  }

  static void check_err(const Ctl& h) {
    if (h.err & 8u) fail(GFB_ECUDA, "peer: cross-rank barrier timed out (a rank did not arrive)");
    if (h.err & 1u) fail(GFB_ERANGE, "sssp: u32 distance overflow (use f64 weights)");
    if (h.err & 4u) fail(GFB_ELOGIC, "peer: predecessor repair list overflow");
  }
};

// One SSSP over the peers this process drives (one per rank in the
// multi-process case, all of them for gfb_mg): every step is launched on all
// peers, then every peer's control block is read.  The barrier-published
// global counters are equal on all ranks, so all hosts take the same
// decisions without a host collective.
template <class W>
static void peer_call_t(const std::vector<Peer*>& ps, uint32_t source, const gfb_sssp_opts* o,
                        std::vector<gfb_sssp_stats>* st) {
  std::vector<PeerRun<W>> rs;
  for (Peer* p : ps) rs.push_back(PeerRun<W>{p, p->ctx, p->ctx->stream});
  auto each = [&](auto&& f) {
    for (auto& r : rs) {
      GFB_CUDA(cudaSetDevice(r.c->device));
      f(r);
    }
  };
  std::vector<Ctl> h(rs.size());
  auto read_all = [&] {
    for (size_t i = 0; i < rs.size(); ++i) {
      GFB_CUDA(cudaSetDevice(rs[i].c->device));
      h[i] = rs[i].read();
    }
  };
  each([&](PeerRun<W>& r) { r.prepare(source, o); });
  each([&](PeerRun<W>& r) { r.launch_loop(); });
  each([&](PeerRun<W>& r) { r.launch_verify(); });
  read_all();
  const uint64_t fallback = h[0].gunres;
  if (o->compute_pred && h[0].gunres > 0) {
    uint32_t base = 0, before = 0;
    uint64_t left = h[0].gunres;
    for (;;) {  // key rounds in batches of 4 while they make progress
      each([&](PeerRun<W>& r) { r.launch_key_batch(base); });
      base += 4;
      read_all();
      left = h[0].gunres - std::min(h[0].gunres, h[0].gresolved);
      if (left == 0 || h[0].gresolved == before || base >= 64) break;
      before = h[0].gresolved;
    }
    if (left > 0) {
      std::vector<uint32_t> caps;
      each([&](PeerRun<W>& r) { caps.push_back(r.launch_inedges()); });
      for (uint32_t round = 1; left > 0; ++round) {
        size_t i = 0;
        each([&](PeerRun<W>& r) { r.launch_round(round, base, caps[i++]); });
        read_all();
        if (h[0].gflag == 0 && round > 1)
          fail(GFB_ELOGIC, "peer: predecessor repair made no progress");
        left -= std::min<uint64_t>(left, h[0].gflag);
      }
    }
  }
  if (st) st->assign(rs.size(), gfb_sssp_stats{});
  for (size_t i = 0; i < rs.size(); ++i) {
    GFB_CUDA(cudaSetDevice(rs[i].c->device));
    rs[i].finish(st ? &(*st)[i] : nullptr, fallback);
  }
}

static void peer_call(const std::vector<Peer*>& ps, uint32_t source, const gfb_sssp_opts* o,
                      std::vector<gfb_sssp_stats>* st) {
  if (ps[0]->g->wtype == GFB_W_F32) peer_call_t<float>(ps, source, o, st);
  else peer_call_t<uint32_t>(ps, source, o, st);
}

void peer_sssp(Peer* p, uint32_t source, const gfb_sssp_opts* o, gfb_sssp_stats* st) {
  std::vector<gfb_sssp_stats> v;
  peer_call({p}, source, o, &v);
  if (st) *st = v[0];
}

// widened distances / native bits / predecessors (global ids) of the local range
template <class W>
__global__ void k_peer_widen(const typename DT<W>::D* d, double* out, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const typename DT<W>::D x = d[i];
    out[i] = x == dinf<W>() ? __longlong_as_double(0x7FF0000000000000ll) : (double)x;
  }
}

void peer_read(Peer* p, double* dist, void* dist_native, uint32_t* pred) {
  if (!p->has_result) fail(GFB_ELOGIC, "peer: no result");
  Ctx* c = p->ctx;
  cudaStream_t s = c->stream;
  const void* d = (char*)p->slab + p->lay.dist;
  if (dist) {
    TBuf tmp;
    tmp.alloc((size_t)p->n * 8 + 8, s);
    if (p->g->wtype == GFB_W_F32)
      k_peer_widen<float><<<stride_grid(c), 256, 0, s>>>((const float*)d, tmp.as<double>(), p->n);
    else
      k_peer_widen<uint32_t><<<stride_grid(c), 256, 0, s>>>((const uint32_t*)d, tmp.as<double>(), p->n);
    GFB_CUDA(cudaMemcpyAsync(dist, tmp.p, (size_t)p->n * 8, cudaMemcpyDeviceToHost, s));
    c->sync();
  }
  if (dist_native) GFB_CUDA(cudaMemcpyAsync(dist_native, d, (size_t)p->n * 4, cudaMemcpyDeviceToHost, s));
  if (pred) GFB_CUDA(cudaMemcpyAsync(pred, p->pred.p, (size_t)p->n * 4, cudaMemcpyDeviceToHost, s));
  c->sync();
}

void peer_free(Peer* p) { delete p; }

// ---- one process driving every partition (gfb_mg_*) ----------------------
// Edge-balanced cut points rounded down to multiples of 32.
static std::vector<uint32_t> mg_ranges(const uint32_t* ro, uint64_t n, int parts) {
  const uint64_t m = ro[n];
  std::vector<uint32_t> rs(parts + 1, 0);
  for (int q = 1; q < parts; ++q) {
    const uint64_t target = (uint64_t)q * m / parts;
    const uint64_t v = std::lower_bound(ro, ro + n + 1, (uint32_t)target) - ro;
    rs[q] = (uint32_t)(std::min<uint64_t>(v, n) & ~31ull);
    rs[q] = std::max(rs[q], rs[q - 1]);
  }
  rs[parts] = (uint32_t)n;
  return rs;
}

void mg_upload(Mg* mg, uint64_t n, uint64_t m, const uint32_t* ro, const uint32_t* col,
               const void* w, int htype, int wtype) {
  if (n == 0 || n >= 0xFFFFFFFFull) fail(GFB_EINVAL, "mg: bad vertex count");
  if (ro[0] != 0 || ro[n] != m) fail(GFB_EINVAL, "mg: row_offsets must run from 0 to m");
  for (Peer* p : mg->peers) delete p;
  mg->peers.clear();
  const int P = (int)mg->ctx.size();
  mg->starts = mg_ranges(ro, n, P);
  mg->n = n;
  mg->wtype = wtype;
  if (mg->exchange == GFB_EXCHANGE_NCCL) {  // xmg.cu
    if (wtype == GFB_W_F64) fail(GFB_EINVAL, "mg: f32 or u32 arithmetic only");
    xmg_upload(mg->x, mg->starts, n, ro, col, w, htype, wtype);
    return;
  }
  const size_t wsz = htype == GFB_W_F64 ? 8 : 4;
  for (int q = 0; q < P; ++q) {
    const uint32_t lo = mg->starts[q], hi = mg->starts[q + 1];
    std::vector<uint32_t> rl(hi - lo + 1);
    for (uint32_t i = 0; i <= hi - lo; ++i) rl[i] = ro[lo + i] - ro[lo];
    GFB_CUDA(cudaSetDevice(mg->ctx[q]->device));
    mg->peers.push_back(peer_create(mg->ctx[q], q, P, mg->starts.data(), rl[hi - lo], rl.data(),
                                    col + ro[lo],
                                    static_cast<const char*>(w) + (size_t)ro[lo] * wsz, htype,
                                    wtype));
  }
  peer_link_local(mg->peers);
}

void mg_sssp(Mg* mg, uint32_t source, const gfb_sssp_opts* o, double* dist, uint32_t* pred,
             gfb_sssp_stats* st) {
  if (mg->exchange == GFB_EXCHANGE_NCCL) return xmg_sssp(mg->x, source, o, dist, pred, st);
  if (mg->peers.empty()) fail(GFB_ELOGIC, "mg: no graph uploaded");
  std::vector<gfb_sssp_stats> v;
  peer_call(mg->peers, source, o, &v);
  for (Peer* p : mg->peers) {
    GFB_CUDA(cudaSetDevice(p->ctx->device));
    if (dist || pred)
      peer_read(p, dist ? dist + p->lo : nullptr, nullptr, pred ? pred + p->lo : nullptr);
  }
  if (st) {  // whole-graph view: sums of the shares, max device time
    *st = v[0];
    for (size_t i = 1; i < v.size(); ++i) {
      st->relaxations += v[i].relaxations;
      st->n_reach += v[i].n_reach;
      st->m_reach += v[i].m_reach;
      st->kernel_launches += v[i].kernel_launches;
      st->device_ms = std::max(st->device_ms, v[i].device_ms);
    }
  }
}

void mg_free(Mg* mg) {
  if (mg->x) {
    xmg_free(mg->x);
    mg->x = nullptr;
  }
  for (Peer* p : mg->peers) {
    GFB_CUDA(cudaSetDevice(p->ctx->device));
    p->ctx->sync();
  }
  for (Peer* p : mg->peers) delete p;
  mg->peers.clear();
}
Ctx* peer_ctx(Peer* p) { return p->ctx; }

}  // namespace gfb

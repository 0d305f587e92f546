// xmg.cu -- the 1-D partitioned SSSP with a host-driven message exchange over
// NCCL (the north star's "remote relaxations bucketed per owner
// and exchanged each iteration by NCCL all-to-all over NVLink, with an
// allreduce for frontier-empty convergence"), one process driving P devices
// (gfb_mg_create_ex(..., GFB_EXCHANGE_NCCL)).  The measured baseline and
// fallback for the device-initiated exchange of peer.cu.
//
// Partition q owns vertex range [starts[q], starts[q+1]) (edge-balanced,
// 32-aligned cut points) and the CSR rows of it (gfb_part, mg.cu).  One
// superstep:
//   1. part_advance   per partition: local destinations relaxed in place,
//                     remote candidates min-combined per destination into
//                     16-byte messages {dst, src, dist_bits, 0}, ascending dst
//                     = bucketed by owner, with per-owner counts
//   2. exchange       one NCCL group of ncclSend / ncclRecv per (sender,
//                     owner) pair with messages (the all-to-all-v; counts are
//                     known to the driving thread, so no count exchange)
//   3. part_apply     owners atomicMin the received candidates, activate
//   4. convergence    ncclAllReduce(sum) of the partitions' next-frontier
//                     sizes (device counters), read once
// Predecessors (after convergence): the distances are gathered, every
// partition proposes tight in-edges for unresolved vertices in rounds
// (round 1 strictly decreasing, later rounds equal-distance from resolved
// sources: the acyclicity rule of the single-GPU repair), and the proposals
// are combined with ncclAllReduce(min).
//
// NCCL needs one device per communicator rank; partitions sharing a device
// (the one-GPU tests) exchange through device copies with the same protocol.
#include <dlfcn.h>
#include <nccl.h>  // types only: the library is bound at first use (nccl_api())

#include <algorithm>
#include <chrono>
#include <cstring>
#include <memory>
#include <vector>

#include "impl.hpp"

namespace gfb {

// NCCL is bound with dlopen at the first exchange that needs it, not linked:
// libgfb.so loaded before torch must not pin the system libnccl.so.2 into the
// process (torch's bundled NCCL has the same soname and newer symbols).  An
// NCCL already in the process (torch's) is preferred.
struct NcclApi {
  decltype(&ncclCommInitAll) CommInitAll;
  decltype(&ncclCommDestroy) CommDestroy;
  decltype(&ncclGroupStart) GroupStart;
  decltype(&ncclGroupEnd) GroupEnd;
  decltype(&ncclSend) Send;
  decltype(&ncclRecv) Recv;
  decltype(&ncclAllReduce) AllReduce;
  decltype(&ncclGetErrorString) GetErrorString;
};

static const NcclApi& nccl_api() {
  static const NcclApi api = [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) fail(GFB_ENCCL, std::string("libnccl.so.2 not loadable: ") + dlerror());
    auto sym = [h](const char* name) {
      void* f = dlsym(h, name);
      if (!f) fail(GFB_ENCCL, std::string("libnccl.so.2 lacks ") + name);
      return f;
    };
    NcclApi a;
    a.CommInitAll = (decltype(a.CommInitAll))sym("ncclCommInitAll");
    a.CommDestroy = (decltype(a.CommDestroy))sym("ncclCommDestroy");
    a.GroupStart = (decltype(a.GroupStart))sym("ncclGroupStart");
    a.GroupEnd = (decltype(a.GroupEnd))sym("ncclGroupEnd");
    a.Send = (decltype(a.Send))sym("ncclSend");
    a.Recv = (decltype(a.Recv))sym("ncclRecv");
    a.AllReduce = (decltype(a.AllReduce))sym("ncclAllReduce");
    a.GetErrorString = (decltype(a.GetErrorString))sym("ncclGetErrorString");
    return a;
  }();
  return api;
}

#define GFB_NCCL(x)                                                                         \
  do {                                                                                      \
    ncclResult_t r_ = (x);                                                                  \
    if (r_ != ncclSuccess)                                                                  \
      fail(GFB_ENCCL, std::string(#x) + ": " + nccl_api().GetErrorString(r_));                  \
  } while (0)

unsigned long long* part_pending_launch(Part* p);

struct Xmg {
  std::vector<Ctx*> ctx;
  std::vector<Part*> parts;
  std::vector<uint32_t> starts;
  std::vector<uint32_t> ro;  // host row offsets: n_reach / m_reach
  std::vector<ncclComm_t> comms;
  bool nccl = false;
  std::vector<DBuf> out, in;  // per partition: outgoing / incoming messages (16 B)
  std::vector<uint64_t> out_cap, in_cap;
  uint64_t n = 0;
  int wtype = -1;
  ~Xmg() {
    for (Part* p : parts) delete p;
    for (ncclComm_t c : comms) nccl_api().CommDestroy(c);
  }
};

static void set_dev(Ctx* c) { GFB_CUDA(cudaSetDevice(c->device)); }

Xmg* xmg_create(const std::vector<Ctx*>& ctx) {
  auto x = std::make_unique<Xmg>();
  x->ctx = ctx;
  std::vector<int> devs;
  for (Ctx* c : ctx) devs.push_back(c->device);
  std::vector<int> sorted = devs;
  std::sort(sorted.begin(), sorted.end());
  x->nccl = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
  if (x->nccl) {
    x->comms.resize(devs.size());
    GFB_NCCL(nccl_api().CommInitAll(x->comms.data(), (int)devs.size(), devs.data()));
  }
  return x.release();
}

void xmg_free(Xmg* x) {
  for (Ctx* c : x->ctx) {
    set_dev(c);
    c->sync();
  }
  delete x;
}

bool xmg_uses_nccl(const Xmg* x) { return x->nccl; }

void xmg_upload(Xmg* x, const std::vector<uint32_t>& starts, uint64_t n, const uint32_t* ro,
                const uint32_t* col, const void* w, int htype, int wtype) {
  for (Part* p : x->parts) delete p;
  x->parts.clear();
  const int P = (int)x->ctx.size();
  x->starts = starts;
  x->n = n;
  x->wtype = wtype;
  x->ro.assign(ro, ro + n + 1);
  x->out.clear();
  x->in.clear();
  x->out = std::vector<DBuf>(P);
  x->in = std::vector<DBuf>(P);
  x->out_cap.assign(P, 0);
  x->in_cap.assign(P, 0);
  const size_t wsz = htype == GFB_W_F64 ? 8 : 4;
  for (int q = 0; q < P; ++q) {
    const uint32_t lo = starts[q], hi = starts[q + 1];
    std::vector<uint32_t> rl(hi - lo + 1);
    for (uint32_t i = 0; i <= hi - lo; ++i) rl[i] = ro[lo + i] - ro[lo];
    set_dev(x->ctx[q]);
    x->parts.push_back(part_create(x->ctx[q], n, lo, hi, rl[hi - lo], rl.data(), col + ro[lo],
                                   static_cast<const char*>(w) + (size_t)ro[lo] * wsz, htype,
                                   wtype));
    // one message per remote destination per superstep at most (min-combined
    // per destination), and one per (sender, local vertex) on the way in
    x->out_cap[q] = std::max<uint64_t>(n - (hi - lo), 1);
    x->in_cap[q] = std::max<uint64_t>((uint64_t)(P - 1) * (hi - lo), 1);
    x->out[q].alloc(x->out_cap[q] * 16, x->ctx[q]->stream);
    x->in[q].alloc(x->in_cap[q] * 16, x->ctx[q]->stream);
  }
}

// all-to-all-v of the messages: counts[q][p] from q to p, bucketed in q's
// outbox in owner order; p's inbox gets the senders' buckets in sender order
static void exchange(Xmg* x, const std::vector<std::vector<uint32_t>>& counts,
                     std::vector<uint64_t>* recv_total) {
  const int P = (int)x->parts.size();
  std::vector<std::vector<uint64_t>> soff(P, std::vector<uint64_t>(P + 1, 0)),
      roff(P, std::vector<uint64_t>(P + 1, 0));
  for (int q = 0; q < P; ++q)
    for (int p = 0; p < P; ++p) soff[q][p + 1] = soff[q][p] + counts[q][p];
  for (int p = 0; p < P; ++p)
    for (int q = 0; q < P; ++q) roff[p][q + 1] = roff[p][q] + counts[q][p];
  recv_total->assign(P, 0);
  for (int p = 0; p < P; ++p) {
    (*recv_total)[p] = roff[p][P];
    if (roff[p][P] > x->in_cap[p]) fail(GFB_ELOGIC, "xmg: inbox overflow");
  }
  if (x->nccl) {
    GFB_NCCL(nccl_api().GroupStart());
    for (int q = 0; q < P; ++q)
      for (int p = 0; p < P; ++p) {
        if (p == q) continue;
        if (counts[q][p])
          GFB_NCCL(nccl_api().Send(x->out[q].as<char>() + soff[q][p] * 16, counts[q][p] * 16, ncclUint8,
                            p, x->comms[q], x->ctx[q]->stream));
        if (counts[p][q])
          GFB_NCCL(nccl_api().Recv(x->in[q].as<char>() + roff[q][p] * 16, counts[p][q] * 16, ncclUint8,
                            p, x->comms[q], x->ctx[q]->stream));
      }
    GFB_NCCL(nccl_api().GroupEnd());
  } else {  // partitions sharing devices: the same all-to-all-v as copies
    for (int p = 0; p < P; ++p) {
      set_dev(x->ctx[p]);
      for (int q = 0; q < P; ++q)
        if (q != p && counts[q][p])
          GFB_CUDA(cudaMemcpyPeerAsync(x->in[p].as<char>() + roff[p][q] * 16, x->ctx[p]->device,
                                       x->out[q].as<char>() + soff[q][p] * 16, x->ctx[q]->device,
                                       counts[q][p] * 16, x->ctx[p]->stream));
    }
  }
  for (int p = 0; p < P; ++p) {
    set_dev(x->ctx[p]);
    x->ctx[p]->sync();
  }
}

// next-frontier size summed over partitions: ncclAllReduce of the device
// counters (NCCL), or the host sum of the same counters
static uint64_t global_pending(Xmg* x) {
  const int P = (int)x->parts.size();
  std::vector<unsigned long long*> cnt(P);
  for (int q = 0; q < P; ++q) {
    set_dev(x->ctx[q]);
    cnt[q] = part_pending_launch(x->parts[q]);
  }
  unsigned long long total = 0;
  if (x->nccl) {
    GFB_NCCL(nccl_api().GroupStart());
    for (int q = 0; q < P; ++q)
      GFB_NCCL(nccl_api().AllReduce(cnt[q], cnt[q], 1, ncclUint64, ncclSum, x->comms[q],
                             x->ctx[q]->stream));
    GFB_NCCL(nccl_api().GroupEnd());
    set_dev(x->ctx[0]);
    GFB_CUDA(cudaMemcpyAsync(&total, cnt[0], 8, cudaMemcpyDeviceToHost, x->ctx[0]->stream));
    for (int q = 0; q < P; ++q) {
      set_dev(x->ctx[q]);
      x->ctx[q]->sync();
    }
  } else {
    for (int q = 0; q < P; ++q) {
      set_dev(x->ctx[q]);
      unsigned long long h = 0;
      GFB_CUDA(cudaMemcpyAsync(&h, cnt[q], 8, cudaMemcpyDeviceToHost, x->ctx[q]->stream));
      x->ctx[q]->sync();
      total += h;
    }
  }
  return total;
}

void xmg_sssp(Xmg* x, uint32_t source, const gfb_sssp_opts* o, double* dist, uint32_t* pred,
              gfb_sssp_stats* st) {
  if (x->parts.empty()) fail(GFB_ELOGIC, "mg: no graph uploaded");
  if (source >= x->n) fail(GFB_ERANGE, "sssp: source out of range");
  if (o->direction == GFB_DIR_PULL) fail(GFB_EINVAL, "mg: the partitioned SSSP is push-only");
  if (o->delta > 0) fail(GFB_EINVAL, "mg: the near-far filter is single-GPU only");
  const int P = (int)x->parts.size();
  const auto t0 = std::chrono::steady_clock::now();
  for (int q = 0; q < P; ++q) {
    set_dev(x->ctx[q]);
    part_init(x->parts[q], source);
  }
  std::vector<std::vector<uint32_t>> counts(P, std::vector<uint32_t>(P, 0));
  std::vector<uint64_t> recv;
  uint64_t supersteps = 0, launches = 0;
  for (;;) {
    for (int q = 0; q < P; ++q) {
      set_dev(x->ctx[q]);
      part_advance(x->parts[q], x->out[q].p, x->out_cap[q], x->starts.data(), P,
                   counts[q].data());
      launches += 9;
    }
    exchange(x, counts, &recv);
    for (int q = 0; q < P; ++q) {
      set_dev(x->ctx[q]);
      part_apply(x->parts[q], x->in[q].p, recv[q]);
      launches += recv[q] ? 1 : 0;
    }
    ++supersteps;
    launches += P;
    if (global_pending(x) == 0) break;
  }
  // distances: every partition's range, in the device arithmetic
  std::vector<uint32_t> dbits(x->n);
  uint64_t relax = 0;
  for (int q = 0; q < P; ++q) {
    set_dev(x->ctx[q]);
    uint64_t r = 0, s = 0;
    part_read(x->parts[q], dbits.data() + x->starts[q], &r, &s);
    relax += r;
  }
  const bool f32 = x->wtype == GFB_W_F32;
  const uint32_t inf_bits = f32 ? 0x7F800000u : 0xFFFFFFFFu;
  uint64_t n_reach = 0, m_reach = 0;
  for (uint64_t v = 0; v < x->n; ++v)
    if (dbits[v] != inf_bits) {
      ++n_reach;
      m_reach += x->ro[v + 1] - x->ro[v];
    }
  if (dist)
    for (uint64_t v = 0; v < x->n; ++v) {
      float fv;
      std::memcpy(&fv, &dbits[v], 4);
      dist[v] = dbits[v] == inf_bits ? __builtin_inf() : (f32 ? (double)fv : (double)dbits[v]);
    }
  if (pred && o->compute_pred) {
    // global distances on every device, then election rounds combined with
    // allreduce(min) (NCCL) or the host minimum (shared devices)
    std::vector<uint32_t> res(x->n, 0), cand(x->n), pmin(x->n);
    std::fill(pred, pred + x->n, NIL);
    res[source] = 1;
    uint64_t left = n_reach - 1;
    std::vector<DBuf> gd(P), gres(P), gcand(P);
    for (int q = 0; q < P; ++q) {
      set_dev(x->ctx[q]);
      cudaStream_t s = x->ctx[q]->stream;
      gd[q].alloc(x->n * 4, s);
      gres[q].alloc(x->n * 4, s);
      gcand[q].alloc(x->n * 4, s);
      GFB_CUDA(cudaMemcpyAsync(gd[q].p, dbits.data(), x->n * 4, cudaMemcpyHostToDevice, s));
    }
    for (uint32_t round = 1; left > 0; ++round) {
      for (int q = 0; q < P; ++q) {
        set_dev(x->ctx[q]);
        cudaStream_t s = x->ctx[q]->stream;
        GFB_CUDA(cudaMemcpyAsync(gres[q].p, res.data(), x->n * 4, cudaMemcpyHostToDevice, s));
        GFB_CUDA(cudaMemsetAsync(gcand[q].p, 0xFF, x->n * 4, s));
        part_pred(x->parts[q], gd[q].p, gres[q].as<uint32_t>(), gcand[q].as<uint32_t>(), round);
      }
      if (x->nccl) {
        GFB_NCCL(nccl_api().GroupStart());
        for (int q = 0; q < P; ++q)
          GFB_NCCL(nccl_api().AllReduce(gcand[q].p, gcand[q].p, x->n, ncclUint32, ncclMin, x->comms[q],
                                 x->ctx[q]->stream));
        GFB_NCCL(nccl_api().GroupEnd());
        set_dev(x->ctx[0]);
        GFB_CUDA(cudaMemcpyAsync(pmin.data(), gcand[0].p, x->n * 4, cudaMemcpyDeviceToHost,
                                 x->ctx[0]->stream));
        for (int q = 0; q < P; ++q) {
          set_dev(x->ctx[q]);
          x->ctx[q]->sync();
        }
      } else {
        std::fill(pmin.begin(), pmin.end(), NIL);
        for (int q = 0; q < P; ++q) {
          set_dev(x->ctx[q]);
          GFB_CUDA(cudaMemcpyAsync(cand.data(), gcand[q].p, x->n * 4, cudaMemcpyDeviceToHost,
                                   x->ctx[q]->stream));
          x->ctx[q]->sync();
          for (uint64_t v = 0; v < x->n; ++v) pmin[v] = std::min(pmin[v], cand[v]);
        }
      }
      uint64_t got = 0;
      for (uint64_t v = 0; v < x->n; ++v)
        if (res[v] == 0 && pmin[v] != NIL && dbits[v] != inf_bits) {
          pred[v] = pmin[v];
          res[v] = round + 1;
          ++got;
        }
      if (got == 0 && round > 1) fail(GFB_ELOGIC, "mg: predecessor repair made no progress");
      left -= std::min(left, got);
    }
  } else if (pred) {
    std::fill(pred, pred + x->n, NIL);
  }
  const double ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (st) {
    *st = gfb_sssp_stats{};
    st->supersteps = supersteps;
    st->relaxations = relax;
    st->n_reach = n_reach;
    st->m_reach = m_reach;
    st->push_steps = supersteps;
    st->device_ms = ms;  // host-driven loop: wall time of the call (documented)
    st->kernel_launches = launches;
    st->advance_launches = supersteps * P;
  }
}

}  // namespace gfb

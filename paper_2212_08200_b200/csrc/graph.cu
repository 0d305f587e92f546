// graph.cu -- device graph store: upload (graph.hpp:132-162 layout and
// validation), device build_transpose (graph.hpp:166-193), the static pull
// plan, and the device-side synthetic generators (RMAT, grid).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <immintrin.h>

#include <chrono>
#include <cmath>
#include <string>
#include <thread>
#include <vector>

#include "impl.hpp"
#include "rmat.cuh"

namespace gfb {

// Stream-ordered allocations from the device's default pool (its release
// threshold is raised at context creation, so memory stays reserved and a
// temporary costs no page mapping and no device-wide synchronisation -- a
// plain cudaFree synchronises the whole device).  Every buffer is used on the
// stream it was allocated on, or on helper streams the owner synchronises
// before returning (fill_graph).
void DBuf::alloc(size_t b, cudaStream_t stream) {
  release();
  s = stream;
  if (b == 0) b = 16;
  cudaError_t e = cudaMallocAsync(&p, b, stream);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    p = nullptr;
    fail(GFB_ENOMEM, "device allocation of " + std::to_string(b) + " bytes failed");
  }
  check_cuda(e, "cudaMallocAsync");
  bytes = b;
}

void DBuf::release() {
  if (p && cudaFreeAsync(p, s) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(p);
  }
  p = nullptr;
  bytes = 0;
}

void DBuf::release_sync() {
  if (p) cudaFree(p);
  p = nullptr;
  bytes = 0;
}

Ctx::~Ctx() {
  if (ctl_host) cudaFreeHost(ctl_host);
  for (auto& a : aux)
    if (a) cudaStreamDestroy(a);
  for (auto& e : ev)
    if (e) cudaEventDestroy(e);
  if (stream) cudaStreamDestroy(stream);
}

void Ctx::ensure_status(size_t n) {
  if (n <= status_cap) return;
  status.alloc(n * 8, stream);
  qstatus.alloc(n * 8, stream);
  status_cap = n;
}

void Ctx::sync() { GFB_CUDA(cudaStreamSynchronize(stream)); }

Ctl Ctx::read_ctl(const Ctl* dctl) {
  GFB_CUDA(cudaMemcpyAsync(ctl_host, dctl, sizeof(Ctl), cudaMemcpyDeviceToHost, stream));
  sync();
  return *ctl_host;
}

Graph::~Graph() {
  for (cudaEvent_t& e : hdone)
    if (e) cudaEventDestroy(e);
}

void invalidate_loop_graphs(Graph* g) {
  Workspace* ws = g->ws.get();
  if (!ws) return;
  if (ws->loop_exec) cudaGraphExecDestroy(ws->loop_exec);
  if (ws->loop_graph) cudaGraphDestroy(ws->loop_graph);
  if (ws->bfs_exec) cudaGraphExecDestroy(ws->bfs_exec);
  if (ws->bfs_graph) cudaGraphDestroy(ws->bfs_graph);
  ws->loop_exec = nullptr;
  ws->loop_graph = nullptr;
  ws->bfs_exec = nullptr;
  ws->bfs_graph = nullptr;
  ws->bfs_key = -1;
}

void check_usable(const Graph* g) {
  if (g->poisoned)
    fail(GFB_ELOGIC, "graph: contents invalid after a failed refill (refill it again)");
}
Workspace::~Workspace() {
  if (loop_exec) cudaGraphExecDestroy(loop_exec);
  if (loop_graph) cudaGraphDestroy(loop_graph);
  if (bfs_exec) cudaGraphExecDestroy(bfs_exec);
  if (bfs_graph) cudaGraphDestroy(bfs_graph);
  if (ctl_host) cudaFreeHost(ctl_host);
}

void Frontier::reserve(uint64_t c) {
  if (c <= cap) return;
  TBuf nb;
  nb.alloc(c * 4, ctx->stream);
  if (len) GFB_CUDA(cudaMemcpyAsync(nb.p, list.p, len * 4, cudaMemcpyDeviceToDevice, ctx->stream));
  std::swap(list.p, nb.p);
  std::swap(list.bytes, nb.bytes);
  cap = c;
}

// ---------------------------------------------------------------------------
// Upload: validate + interleave {dst, weight} records.
// ---------------------------------------------------------------------------
template <class W>
__device__ __forceinline__ bool conv_weight(const void* src, int htype, uint64_t e, W* out);

template <>
__device__ __forceinline__ bool conv_weight<float>(const void* src, int htype, uint64_t e,
                                                   float* out) {
  float w;
  if (htype == GFB_W_F64) {
    double d = static_cast<const double*>(src)[e];
    if (!(d >= 0) || isinf(d)) return false;
    w = __double2float_rn(d);
  } else if (htype == GFB_W_F32) {
    w = static_cast<const float*>(src)[e];
  } else {
    w = (float)static_cast<const uint32_t*>(src)[e];
  }
  if (!(w >= 0.0f) || isinf(w)) return false;
  *out = w + 0.0f;  // canonicalise -0.0 -> +0.0
  return true;
}
template <>
__device__ __forceinline__ bool conv_weight<double>(const void* src, int htype, uint64_t e,
                                                    double* out) {
  double w;
  if (htype == GFB_W_F64) w = static_cast<const double*>(src)[e];
  else if (htype == GFB_W_F32) w = (double)static_cast<const float*>(src)[e];
  else w = (double)static_cast<const uint32_t*>(src)[e];
  if (!(w >= 0.0) || isinf(w)) return false;
  *out = w + 0.0;
  return true;
}
template <>
__device__ __forceinline__ bool conv_weight<uint32_t>(const void* src, int htype, uint64_t e,
                                                      uint32_t* out) {
  if (htype == GFB_W_U32) {
    *out = static_cast<const uint32_t*>(src)[e];
    return true;
  }
  double d = htype == GFB_W_F64 ? static_cast<const double*>(src)[e]
                                : (double)static_cast<const float*>(src)[e];
  if (!(d >= 0) || isinf(d) || d > 4294967295.0 || d != floor(d)) return false;
  *out = (uint32_t)d;
  return true;
}

// Interleave one uploaded chunk [e0, e0 + cnt) of col[] / w[] into the
// device records; validation flags record the first bad global edge index.
template <class W>
__global__ void k_interleave(const uint32_t* __restrict__ col, const void* __restrict__ wsrc,
                             int htype, EdgeRec<W>* adj, uint64_t e0, uint64_t cnt,
                             uint64_t bound, unsigned long long* bad_v,
                             unsigned long long* bad_w) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += stride) {
    uint32_t v = col[i];
    W w{};
    bool okw = conv_weight<W>(wsrc, htype, i, &w);
    if (v >= bound) atomicMin(bad_v, (unsigned long long)(e0 + i));
    if (!okw) atomicMin(bad_w, (unsigned long long)(e0 + i));
    EdgeRec<W> r{};
    r.v = v;
    r.w = w;
    adj[e0 + i] = r;
  }
}

__global__ void k_check_ro(const uint32_t* ro, uint64_t n, uint64_t m,
                           unsigned long long* bad) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v <= n; v += stride) {
    bool ok = v == 0 ? ro[0] == 0 : ro[v - 1] <= ro[v];
    if (v == n && ro[n] != m) ok = false;
    if (!ok) atomicMin(bad, (unsigned long long)v);
  }
}

template <class W>
static void launch_interleave(Graph* g, const uint32_t* dcol, const void* dw, int htype,
                              uint64_t e0, uint64_t cnt, unsigned long long* flags) {
  Ctx* c = g->ctx;
  k_interleave<W><<<stride_grid(c), 256, 0, c->stream>>>(
      dcol, dw, htype, g->adj.as<EdgeRec<W>>(), e0, cnt, g->col_bound ? g->col_bound : g->n,
      flags, flags + 1);
  GFB_CUDA(cudaGetLastError());
}

static size_t host_wsize(int htype) { return htype == GFB_W_F64 ? 8 : 4; }

// f64 host weights into an f32 graph (the reference's values() on the
// headline path): narrowed on the host, a slice per thread, into pinned
// buffers, so PCIe carries 4 bytes per weight instead of 8 -- with exactly
// the device conversion's rules (conv_weight<float>: a negative, NaN or
// infinite double, or one that rounds to +inf, is invalid; -0.0 -> +0.0).
// Returns the first invalid edge index of [0, cnt), or ~0.
static constexpr uint64_t HOST_NARROW_MIN_EDGES = 1ull << 20;

// scalar slice [a, b): first invalid index or ~0
static uint64_t narrow_scalar(const double* src, float* dst, uint64_t a, uint64_t b) {
  uint64_t first = ~0ull;
  for (uint64_t i = a; i < b; ++i) {
    const double d = src[i];
    const float w = (float)d;  // round to nearest (SSE), like __double2float_rn
    const bool ok = d >= 0 && !std::isinf(d) && w >= 0.0f && !std::isinf(w);
    if (!ok && first == ~0ull) first = i;
    dst[i] = w + 0.0f;
  }
  return first;
}

// AVX2 slice: 8 weights per step, streaming (non-temporal) stores -- the
// pinned buffer is read next by the DMA engine, not by this core, so no
// read-for-ownership of its lines (the narrowing is host-memory bound)
__attribute__((target("avx2"))) static uint64_t narrow_avx2(const double* src, float* dst,
                                                            uint64_t a, uint64_t b) {
  uint64_t i = a;
  uint64_t first = ~0ull;
  while (i < b && ((uintptr_t)(dst + i) & 31u)) {  // align the stores
    const uint64_t f = narrow_scalar(src, dst, i, i + 1);
    if (first == ~0ull) first = f;
    ++i;
  }
  const __m256d zd = _mm256_setzero_pd();
  const __m256 zf = _mm256_setzero_ps();
  const __m256 inf = _mm256_set1_ps(INFINITY);
  for (; i + 8 <= b; i += 8) {
    const __m256d d0 = _mm256_loadu_pd(src + i), d1 = _mm256_loadu_pd(src + i + 4);
    const __m256 w = _mm256_set_m128(_mm256_cvtpd_ps(d1), _mm256_cvtpd_ps(d0));
    // valid: d >= 0 (ordered: NaN and negatives fail; -0.0 passes) and w < +inf
    const int okd = _mm256_movemask_pd(_mm256_cmp_pd(d0, zd, _CMP_GE_OQ)) |
                    (_mm256_movemask_pd(_mm256_cmp_pd(d1, zd, _CMP_GE_OQ)) << 4);
    const int okw = _mm256_movemask_ps(_mm256_cmp_ps(w, inf, _CMP_LT_OQ));
    if ((okd & okw) != 0xFF && first == ~0ull) first = narrow_scalar(src, dst, i, i + 8);
    _mm256_stream_ps(dst + i, _mm256_add_ps(w, zf));  // -0.0 -> +0.0
  }
  if (i < b) {
    const uint64_t f = narrow_scalar(src, dst, i, b);
    if (first == ~0ull) first = f;
  }
  _mm_sfence();
  return first;
}

static uint64_t narrow_weights(const double* src, float* dst, uint64_t cnt) {
  const unsigned hc = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  const bool avx2 = __builtin_cpu_supports("avx2");
  // slices in multiples of 8 weights (32-byte aligned stores when dst is)
  const uint64_t per = ((cnt + hc - 1) / hc + 7) & ~7ull;
  std::vector<uint64_t> bad(hc, ~0ull);
  std::vector<std::thread> th;
  auto work = [&](unsigned t) {
    const uint64_t a = std::min<uint64_t>(cnt, t * per), b = std::min<uint64_t>(cnt, a + per);
    // IEEE round-to-nearest with denormals kept, like __double2float_rn on the
    // device, whatever FTZ / DAZ / rounding mode the calling process has set
    const unsigned csr = _mm_getcsr();
    _mm_setcsr(0x1F80u);
    bad[t] = avx2 ? narrow_avx2(src, dst, a, b) : narrow_scalar(src, dst, a, b);
    _mm_setcsr(csr);
  };
  for (unsigned t = 1; t < hc; ++t) {
    try {
      th.emplace_back(work, t);
    } catch (...) {  // no thread available: this slice on the calling thread
      work(t);
    }
  }
  work(0);
  for (auto& x : th) x.join();
  return *std::min_element(bad.begin(), bad.end());
}

// H2D upload as a two-stream pipeline: chunk b+1 is copied (copy stream,
// double-buffered staging kept on the graph for refills) while chunk b is
// validated and interleaved into {dst, w} records (compute stream).
static constexpr uint64_t UPLOAD_CHUNK = 1ull << 25;  // edges per chunk

static void fill_graph(Graph* g, const uint32_t* ro, const uint32_t* col, const void* w,
                       int htype) {
  // everything derived from the old contents goes first: the transpose, the
  // relabelled copy, cached statistics and the loop graphs that point at them
  invalidate_loop_graphs(g);
  g->has_csc = false;
  g->ceid.release();
  if (g->ws) g->ws->has_result = false;
  g->poisoned = true;  // cleared once the new contents validated
  g->rl_valid = false;
  g->max_outdeg = -1;
  g->mean_w = -1;
  g->runs_since_fill = 0;
  Ctx* c = g->ctx;
  cudaStream_t s = c->stream;
  const uint64_t n = g->n, m = g->m;
  if (htype < GFB_W_U32 || htype > GFB_W_F64) fail(GFB_EINVAL, "graph: bad host weight type");
  if (!ro || (m && (!col || !w))) fail(GFB_EINVAL, "graph: null CSR array");
  if (!c->aux[1]) GFB_CUDA(cudaStreamCreateWithFlags(&c->aux[1], cudaStreamNonBlocking));
  cudaStream_t cp = c->aux[1];
  // f64 -> f32 narrowed on the host (large uploads; identical validation)
  const bool narrow = htype == GFB_W_F64 && g->wtype == GFB_W_F32 && m >= HOST_NARROW_MIN_EDGES;
  uint64_t host_bad_w = ~0ull;
  const size_t wsz = host_wsize(htype);
  // narrowing pays while a chunk narrows faster than PCIe would carry its
  // doubles (~55 GB/s for col + 8-byte weights); on a busy host it falls
  // back to the device conversion for the remaining chunks
  bool narrow_now = narrow;
  // staging layout per buffer: col[chunk] | w[chunk]; chunk rounded to 64 so
  // every sub-array stays 16-byte aligned for any weight width
  const uint64_t chunk = (std::min<uint64_t>(UPLOAD_CHUNK, std::max<uint64_t>(m, 1)) + 63) & ~63ull;
  if (g->stage.bytes < 2 * chunk * (4 + 8)) g->stage.alloc(2 * chunk * (4 + 8), s);
  TBuf flags;
  flags.alloc(3 * 8, s);
  GFB_CUDA(cudaMemsetAsync(flags.p, 0xFF, 3 * 8, s));
  auto* f = flags.as<unsigned long long>();
  cudaEvent_t ready[2], done[2], start;
  for (int b = 0; b < 2; ++b) {
    GFB_CUDA(cudaEventCreateWithFlags(&ready[b], cudaEventDisableTiming));
    GFB_CUDA(cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming));
  }
  GFB_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
  if (narrow) {
    if (g->hstage.bytes < 2 * chunk * 4) {
      if (g->hstage.p) {
        c->sync();
        GFB_CUDA(cudaStreamSynchronize(cp));
        cudaFreeHost(g->hstage.p);
        g->hstage.p = nullptr;
        g->hstage.bytes = 0;
      }
      GFB_CUDA(cudaHostAlloc(&g->hstage.p, 2 * chunk * 4, cudaHostAllocDefault));
      g->hstage.bytes = 2 * chunk * 4;
    }
    for (cudaEvent_t& e : g->hdone)
      if (!e) GFB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  GFB_CUDA(cudaEventRecord(start, s));  // staging / flags ready before any copy
  GFB_CUDA(cudaStreamWaitEvent(cp, start, 0));
  GFB_CUDA(cudaMemcpyAsync(g->ro.p, ro, (n + 1) * 4, cudaMemcpyHostToDevice, cp));
  GFB_CUDA(cudaEventRecord(ready[1], cp));
  GFB_CUDA(cudaStreamWaitEvent(s, ready[1], 0));
  k_check_ro<<<stride_grid(c), 256, 0, s>>>(g->ro.as<uint32_t>(), n, m, f + 2);
  for (uint64_t e0 = 0, k = 0; e0 < m; e0 += chunk, ++k) {
    const int b = (int)(k & 1);
    const uint64_t cnt = std::min(chunk, m - e0);
    uint32_t* dcol = reinterpret_cast<uint32_t*>(g->stage.as<char>() + b * chunk * 12);
    void* dw = g->stage.as<char>() + b * chunk * 12 + chunk * 4;
    if (k >= 2) GFB_CUDA(cudaStreamWaitEvent(cp, done[b], 0));  // buffer b consumed
    GFB_CUDA(cudaMemcpyAsync(dcol, col + e0, cnt * 4, cudaMemcpyHostToDevice, cp));
    const bool nk = narrow_now;  // this chunk narrowed on the host
    if (nk) {
      // host buffer b was last read by the copy of chunk k - 2: wait for it,
      // then narrow this chunk while the previous chunk's copies run
      float* hb = g->hstage.as<float>() + b * chunk;
      if (k >= 2) GFB_CUDA(cudaEventSynchronize(g->hdone[b]));
      const auto t0 = std::chrono::steady_clock::now();
      const uint64_t bw = narrow_weights(static_cast<const double*>(w) + e0, hb, cnt);
      const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (sec > (double)cnt * 12.0 / 55e9) narrow_now = false;
      if (bw != ~0ull) host_bad_w = std::min(host_bad_w, e0 + bw);
      GFB_CUDA(cudaMemcpyAsync(dw, hb, cnt * 4, cudaMemcpyHostToDevice, cp));
      GFB_CUDA(cudaEventRecord(g->hdone[b], cp));
    } else {
      GFB_CUDA(cudaMemcpyAsync(dw, static_cast<const char*>(w) + e0 * wsz, cnt * wsz,
                               cudaMemcpyHostToDevice, cp));
    }
    GFB_CUDA(cudaEventRecord(ready[b], cp));
    GFB_CUDA(cudaStreamWaitEvent(s, ready[b], 0));
    if (nk) launch_interleave<float>(g, dcol, dw, GFB_W_F32, e0, cnt, f);
    else if (g->wtype == GFB_W_F32) launch_interleave<float>(g, dcol, dw, htype, e0, cnt, f);
    else if (g->wtype == GFB_W_F64) launch_interleave<double>(g, dcol, dw, htype, e0, cnt, f);
    else launch_interleave<uint32_t>(g, dcol, dw, htype, e0, cnt, f);
    GFB_CUDA(cudaEventRecord(done[b], s));
  }
  unsigned long long hf[3];
  GFB_CUDA(cudaMemcpyAsync(hf, f, sizeof(hf), cudaMemcpyDeviceToHost, s));
  c->sync();
  GFB_CUDA(cudaStreamSynchronize(cp));
  for (int b = 0; b < 2; ++b) {
    cudaEventDestroy(ready[b]);
    cudaEventDestroy(done[b]);
  }
  cudaEventDestroy(start);
  hf[1] = std::min<unsigned long long>(hf[1], host_bad_w);
  if (hf[2] != ~0ull)
    fail(GFB_EINVAL, "graph: row_offsets inconsistent at vertex " + std::to_string(hf[2]));
  // graph.hpp:134-142 reports the first offending edge
  if (hf[0] != ~0ull && hf[0] <= hf[1])
    fail(GFB_EINVAL, "build_csr: edge " + std::to_string(hf[0]) + " has vertex id out of range");
  if (hf[1] != ~0ull)
    fail(GFB_EINVAL,
         "build_csr: edge " + std::to_string(hf[1]) + " has negative or non-finite weight");
  g->poisoned = false;  // same shape: keep the workspace
}

static __global__ void k_max_outdeg(const uint32_t* __restrict__ ro, uint32_t n, uint32_t* out) {
  uint32_t mx = 0;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    mx = max(mx, ro[v + 1] - ro[v]);
  mx = __reduce_max_sync(0xffffffffu, mx);
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(out, mx);
}

// Largest out-degree (cached until a refill): picks the near-far kernel's
// heavy-row handling.
uint32_t max_out_degree(Graph* g) {
  if (g->max_outdeg >= 0) return (uint32_t)g->max_outdeg;
  Ctx* c = g->ctx;
  TBuf mx;
  mx.alloc(16, c->stream);
  GFB_CUDA(cudaMemsetAsync(mx.p, 0, 4, c->stream));
  k_max_outdeg<<<stride_grid(c), 256, 0, c->stream>>>(g->ro.as<uint32_t>(), (uint32_t)g->n,
                                                      mx.as<uint32_t>());
  uint32_t h = 0;
  GFB_CUDA(cudaMemcpyAsync(&h, mx.p, 4, cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  g->max_outdeg = h;
  return h;
}

template <class W>
static __global__ void k_weight_sum(const EdgeRec<W>* __restrict__ adj, uint64_t m, double* out) {
  double acc = 0;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m;
       e += (uint64_t)gridDim.x * blockDim.x)
    acc += (double)adj[e].w;
  for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
  if ((threadIdx.x & 31) == 0 && acc != 0) atomicAdd(out, acc);
}

// Mean edge weight (cached until a refill): scales the automatic near-far
// delta for mesh-like graphs.
double mean_weight(Graph* g) {
  if (g->mean_w >= 0) return g->mean_w;
  Ctx* c = g->ctx;
  TBuf acc;
  acc.alloc(16, c->stream);
  GFB_CUDA(cudaMemsetAsync(acc.p, 0, 8, c->stream));
  if (g->m) {
    if (g->wtype == GFB_W_F32)
      k_weight_sum<float><<<stride_grid(c), 256, 0, c->stream>>>(g->adj.as<EdgeRec<float>>(), g->m,
                                                                 acc.as<double>());
    else if (g->wtype == GFB_W_F64)
      k_weight_sum<double><<<stride_grid(c), 256, 0, c->stream>>>(g->adj.as<EdgeRec<double>>(),
                                                                  g->m, acc.as<double>());
    else
      k_weight_sum<uint32_t><<<stride_grid(c), 256, 0, c->stream>>>(
          g->adj.as<EdgeRec<uint32_t>>(), g->m, acc.as<double>());
  }
  double h = 0;
  GFB_CUDA(cudaMemcpyAsync(&h, acc.p, 8, cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  g->mean_w = g->m ? h / (double)g->m : 0.0;
  return g->mean_w;
}

// ---------------------------------------------------------------------------
// In-degree relabelling for the SSSP loop.  The unpermuted RMAT ids scatter
// the ~55K destinations that receive half of all edges over 55K distinct
// 128-byte lines of the distance array, so the advance's test-before-atomic
// gathers miss L1 (12% hit rate at s24, profiles/).  Ranking vertices by
// descending in-degree (stable: ties keep ascending id) packs them into a few
// hundred KB.  Rows move as blocks; row contents keep their order.
// ---------------------------------------------------------------------------
template <class W>
static __global__ void k_indeg(const EdgeRec<W>* __restrict__ adj, uint64_t m, uint32_t* cnt) {
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t v = adj[e].v;
    // warp-aggregate equal destinations (hubs): one atomic per distinct v
    const unsigned peers = __match_any_sync(__activemask(), v);
    if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(cnt + v, (uint32_t)__popc(peers));
  }
}

static __global__ void k_indeg_csc(const uint32_t* __restrict__ co, uint32_t n, uint32_t* cnt) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    cnt[v] = co[v + 1] - co[v];
}

static __global__ void k_iota_rev(uint32_t* ids, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    ids[i] = i;
}

static __global__ void k_rl_perm(const uint32_t* __restrict__ iperm, const uint32_t* __restrict__ ro,
                                 uint32_t* perm, uint32_t* deg2, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t p = iperm[i];
    perm[p] = i;
    deg2[i] = ro[p + 1] - ro[p];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) deg2[n] = 0;
}

// Copy into the new layout.  One warp per 32 new rows: lane j holds row
// i0+j, the rows' edges are concatenated and copied lane-strided (shuffle
// search for the owning row), so reads of each old row and writes of the new
// CSR coalesce even for rows of a handful of edges.  Rows longer than RL_BIG
// (the hubs, which the in-degree order puts first) would serialise their
// warp: they are listed and copied by k_rl_big, one CTA per row.
constexpr uint32_t RL_BIG = 1024;
template <class W>
static __global__ void k_rl_rows(const uint32_t* __restrict__ ro, const EdgeRec<W>* __restrict__ adj,
                                 const uint32_t* __restrict__ ro2, const uint32_t* __restrict__ iperm,
                                 const uint32_t* __restrict__ perm, EdgeRec<W>* adj2, uint32_t n,
                                 uint32_t* big, uint32_t* nbig) {
  const int lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t i0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; i0 < n;
       i0 += warps * 32) {
    const uint32_t i = i0 + lane;
    uint32_t s0 = 0, len = 0, d0 = 0;
    if (i < n) {
      const uint32_t p = iperm[i];
      s0 = ro[p];
      len = ro[p + 1] - s0;
      d0 = ro2[i];
      if (len > RL_BIG) {
        big[atomicAdd(nbig, 1u)] = i;
        len = 0;
      }
    }
    const uint32_t incl = warp_incl_scan(len, lane);
    const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
    for (uint32_t x = lane; x - lane < tot; x += 32) {
      int lo = 0;  // owning row: first lane whose inclusive length exceeds x
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const uint32_t q = __shfl_sync(0xffffffffu, incl, lo + step - 1);
        if (q <= x) lo += step;
      }
      const uint32_t os = __shfl_sync(0xffffffffu, s0, lo);
      const uint32_t od = __shfl_sync(0xffffffffu, d0, lo);
      const uint32_t opre = __shfl_sync(0xffffffffu, incl, lo) - __shfl_sync(0xffffffffu, len, lo);
      if (x < tot) {
        EdgeRec<W> r = adj[os + (x - opre)];
        r.v = perm[r.v];
        adj2[od + (x - opre)] = r;
      }
    }
  }
}

template <class W>
static __global__ void k_rl_big(const uint32_t* __restrict__ ro, const EdgeRec<W>* __restrict__ adj,
                                const uint32_t* __restrict__ ro2, const uint32_t* __restrict__ iperm,
                                const uint32_t* __restrict__ perm, EdgeRec<W>* adj2,
                                const uint32_t* __restrict__ big, const uint32_t* __restrict__ nbig) {
  const uint32_t cnt = *nbig;
  for (uint32_t k = blockIdx.x; k < cnt; k += gridDim.x) {
    const uint32_t i = big[k], p = iperm[i];
    const uint32_t s0 = ro[p], len = ro[p + 1] - s0, d0 = ro2[i];
    for (uint32_t x = threadIdx.x; x < len; x += blockDim.x) {
      EdgeRec<W> r = adj[s0 + x];
      r.v = perm[r.v];
      adj2[d0 + x] = r;
    }
  }
}

// Rows of the relabelled CSR sorted by destination: on RMAT most edges point
// into the first few hundred thousand relabelled ids, so a sorted row lets
// neighbouring lanes' distance gathers share sectors and L1 lines (s24:
// 3.80 -> 3.68 ms).  Records are split into (dst, weight) arrays for a
// segmented sort and joined back.
template <class W>
static __global__ void k_split_recs(const EdgeRec<W>* r, uint32_t* k, W* v, uint64_t m) {
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const EdgeRec<W> x = r[e];
    k[e] = x.v;
    v[e] = x.w;
  }
}
template <class W>
static __global__ void k_join_recs(EdgeRec<W>* r, const uint32_t* k, const W* v, uint64_t m) {
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += (uint64_t)gridDim.x * blockDim.x) {
    EdgeRec<W> x{};
    x.v = k[e];
    x.w = v[e];
    r[e] = x;
  }
}

template <class W>
static void sort_rows(Ctx* c, const uint32_t* ro, EdgeRec<W>* adj, uint64_t n, uint64_t m) {
  cudaStream_t s = c->stream;
  TBuf k0, k1, v0, v1, t;
  k0.alloc(m * 4, s);
  k1.alloc(m * 4, s);
  v0.alloc(m * sizeof(W), s);
  v1.alloc(m * sizeof(W), s);
  k_split_recs<W><<<stride_grid(c), 256, 0, s>>>(adj, k0.as<uint32_t>(), v0.as<W>(), m);
  size_t tb = 0;
  GFB_CUDA(cub::DeviceSegmentedSort::SortPairs(nullptr, tb, k0.as<uint32_t>(), k1.as<uint32_t>(),
                                               v0.as<W>(), v1.as<W>(), (int64_t)m, (int64_t)n, ro,
                                               ro + 1, s));
  t.alloc(tb, s);
  GFB_CUDA(cub::DeviceSegmentedSort::SortPairs(t.p, tb, k0.as<uint32_t>(), k1.as<uint32_t>(),
                                               v0.as<W>(), v1.as<W>(), (int64_t)m, (int64_t)n, ro,
                                               ro + 1, s));
  k_join_recs<W><<<stride_grid(c), 256, 0, s>>>(adj, k1.as<uint32_t>(), v1.as<W>(), m);
  GFB_CUDA(cudaGetLastError());
}

static __global__ void k_range_keys(const uint32_t* __restrict__ cnt,
                                    const uint32_t* __restrict__ ranges, uint32_t nparts,
                                    unsigned long long* keys, uint32_t n) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    uint32_t lo = 0, hi = nparts;  // the range holding v: ranges[lo] <= v < ranges[lo + 1]
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) / 2;
      if (ranges[mid] <= v) lo = mid;
      else hi = mid;
    }
    keys[v] = ((unsigned long long)(nparts - 1 - lo) << 32) | cnt[v];
  }
}

// The relabelled CSR (new id = rank by descending in-degree cnt[], rows
// sorted by destination) into perm / iperm / ro2 / adj2.  ranges (device,
// nparts + 1 cut points): the ranking runs inside each vertex range, so a
// 1-D partition of the new ids owns the same rows (relabel_ranges).
static void build_relabelled(Graph* g, const uint32_t* cnt, uint32_t* perm, uint32_t* iperm,
                             uint32_t* ro2, void* adj2, const uint32_t* ranges = nullptr,
                             uint32_t nparts = 0) {
  Ctx* c = g->ctx;
  cudaStream_t s = c->stream;
  const uint32_t n = (uint32_t)g->n;
  const uint64_t m = g->m;
  TBuf cnt2, ids, deg2, tmp;
  cnt2.alloc((size_t)n * 4, s);
  ids.alloc((size_t)n * 4, s);
  deg2.alloc((size_t)(n + 1) * 4, s);
  k_iota_rev<<<stride_grid(c), 256, 0, s>>>(ids.as<uint32_t>(), n);
  size_t tb = 0;
  TBuf k64, k64b;
  if (ranges) {  // (nparts - 1 - range) << 32 | in-degree, descending: ranges in order
    k64.alloc((size_t)n * 8, s);
    k64b.alloc((size_t)n * 8, s);
    k_range_keys<<<stride_grid(c), 256, 0, s>>>(cnt, ranges, nparts, k64.as<unsigned long long>(), n);
    GFB_CUDA(cub::DeviceRadixSort::SortPairsDescending(
        nullptr, tb, k64.as<unsigned long long>(), k64b.as<unsigned long long>(),
        ids.as<uint32_t>(), iperm, (int64_t)n, 0, 64, s));
  } else {
    GFB_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, cnt, cnt2.as<uint32_t>(),
                                                       ids.as<uint32_t>(), iperm, (int64_t)n, 0,
                                                       32, s));
  }
  size_t tb2 = 0;
  GFB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb2, deg2.as<uint32_t>(),
                                         ro2, (int64_t)(n + 1), s));
  tmp.alloc(std::max(tb, tb2), s);
  if (ranges)
    GFB_CUDA(cub::DeviceRadixSort::SortPairsDescending(
        tmp.p, tb, k64.as<unsigned long long>(), k64b.as<unsigned long long>(),
        ids.as<uint32_t>(), iperm, (int64_t)n, 0, 64, s));
  else
    GFB_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp.p, tb, cnt, cnt2.as<uint32_t>(),
                                                       ids.as<uint32_t>(), iperm, (int64_t)n, 0,
                                                       32, s));
  k_rl_perm<<<stride_grid(c), 256, 0, s>>>(iperm, g->ro.as<uint32_t>(),
                                           perm, deg2.as<uint32_t>(), n);
  GFB_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb2, deg2.as<uint32_t>(), ro2,
                                         (int64_t)(n + 1), s));
  TBuf big;
  big.alloc((size_t)n * 4 + 16, s);
  uint32_t* nbig = big.as<uint32_t>() + n;
  GFB_CUDA(cudaMemsetAsync(nbig, 0, 4, s));
  if (g->wtype == GFB_W_F32) {
    k_rl_rows<float><<<stride_grid(c), 256, 0, s>>>(
        g->ro.as<uint32_t>(), g->adj.as<EdgeRec<float>>(), ro2,
        iperm, perm, reinterpret_cast<EdgeRec<float>*>(adj2), n,
        big.as<uint32_t>(), nbig);
    k_rl_big<float><<<stride_grid(c), 256, 0, s>>>(
        g->ro.as<uint32_t>(), g->adj.as<EdgeRec<float>>(), ro2,
        iperm, perm, reinterpret_cast<EdgeRec<float>*>(adj2),
        big.as<uint32_t>(), nbig);
  } else if (g->wtype == GFB_W_F64) {
    k_rl_rows<double><<<stride_grid(c), 256, 0, s>>>(
        g->ro.as<uint32_t>(), g->adj.as<EdgeRec<double>>(), ro2,
        iperm, perm, reinterpret_cast<EdgeRec<double>*>(adj2), n,
        big.as<uint32_t>(), nbig);
    k_rl_big<double><<<stride_grid(c), 256, 0, s>>>(
        g->ro.as<uint32_t>(), g->adj.as<EdgeRec<double>>(), ro2,
        iperm, perm, reinterpret_cast<EdgeRec<double>*>(adj2),
        big.as<uint32_t>(), nbig);
  } else {
    k_rl_rows<uint32_t><<<stride_grid(c), 256, 0, s>>>(
        g->ro.as<uint32_t>(), g->adj.as<EdgeRec<uint32_t>>(), ro2,
        iperm, perm,
        reinterpret_cast<EdgeRec<uint32_t>*>(adj2), n, big.as<uint32_t>(), nbig);
    k_rl_big<uint32_t><<<stride_grid(c), 256, 0, s>>>(
        g->ro.as<uint32_t>(), g->adj.as<EdgeRec<uint32_t>>(), ro2,
        iperm, perm,
        reinterpret_cast<EdgeRec<uint32_t>*>(adj2), big.as<uint32_t>(), nbig);
  }
  GFB_CUDA(cudaGetLastError());
  if (g->wtype == GFB_W_F32)
    sort_rows<float>(c, ro2, reinterpret_cast<EdgeRec<float>*>(adj2), n, m);
  else if (g->wtype == GFB_W_F64)
    sort_rows<double>(c, ro2, reinterpret_cast<EdgeRec<double>*>(adj2), n, m);
  else
    sort_rows<uint32_t>(c, ro2, reinterpret_cast<EdgeRec<uint32_t>*>(adj2), n, m);
}

static void indegrees(Graph* g, uint32_t* cnt) {
  Ctx* c = g->ctx;
  cudaStream_t s = c->stream;
  const uint32_t n = (uint32_t)g->n;
  const uint64_t m = g->m;
  if (g->has_csc) {  // from the transpose's offsets
    k_indeg_csc<<<stride_grid(c), 256, 0, s>>>(g->co.as<uint32_t>(), n, cnt);
  } else {
    GFB_CUDA(cudaMemsetAsync(cnt, 0, (size_t)n * 4, s));
    if (g->wtype == GFB_W_F32)
      k_indeg<float><<<stride_grid(c), 256, 0, s>>>(g->adj.as<EdgeRec<float>>(), m, cnt);
    else if (g->wtype == GFB_W_F64)
      k_indeg<double><<<stride_grid(c), 256, 0, s>>>(g->adj.as<EdgeRec<double>>(), m, cnt);
    else
      k_indeg<uint32_t><<<stride_grid(c), 256, 0, s>>>(g->adj.as<EdgeRec<uint32_t>>(), m, cnt);
  }
  GFB_CUDA(cudaGetLastError());
}

// A range-preserving relabelled copy for the 1-D partitioned paths (peer.cu,
// mg.cu): inside each [starts[q], starts[q+1]) the vertices are ranked by
// descending in-degree, rows sorted by destination -- the single-GPU loop's
// layout (ensure_relabel) without moving any vertex to another owner.
// Written to host buffers: row offsets (n + 1), destinations and native
// weights (m), perm (old id -> new id, n).
void relabel_ranges(Graph* g, uint32_t nparts, const uint32_t* starts, uint32_t* ro_out,
                    uint32_t* col_out, void* w_out, uint32_t* perm_out) {
  check_usable(g);
  const uint32_t n = (uint32_t)g->n;
  const uint64_t m = g->m;
  if (nparts < 1 || !starts || starts[0] != 0 || starts[nparts] != n)
    fail(GFB_EINVAL, "relabel_ranges: range_starts must run from 0 to n");
  for (uint32_t q = 0; q < nparts; ++q)
    if (starts[q + 1] < starts[q]) fail(GFB_EINVAL, "relabel_ranges: range_starts must not decrease");
  Ctx* c = g->ctx;
  cudaStream_t s = c->stream;
  TBuf cnt, perm, iperm, ro2, adj2, rg, kc, kw;
  cnt.alloc((size_t)n * 4, s);
  perm.alloc((size_t)n * 4 + 4, s);
  iperm.alloc((size_t)n * 4 + 4, s);
  ro2.alloc((size_t)(n + 1) * 4, s);
  adj2.alloc(m * g->rec_bytes() + 16, s);
  rg.alloc((size_t)(nparts + 1) * 4, s);
  GFB_CUDA(cudaMemcpyAsync(rg.p, starts, (size_t)(nparts + 1) * 4, cudaMemcpyHostToDevice, s));
  indegrees(g, cnt.as<uint32_t>());
  build_relabelled(g, cnt.as<uint32_t>(), perm.as<uint32_t>(), iperm.as<uint32_t>(),
                   ro2.as<uint32_t>(), adj2.p, rg.as<uint32_t>(), nparts);
  const size_t wb = g->wtype == GFB_W_F64 ? 8 : 4;
  kc.alloc(m * 4 + 4, s);
  kw.alloc(m * wb + 8, s);
  if (g->wtype == GFB_W_F32)
    k_split_recs<float><<<stride_grid(c), 256, 0, s>>>(adj2.as<EdgeRec<float>>(), kc.as<uint32_t>(),
                                                       kw.as<float>(), m);
  else if (g->wtype == GFB_W_F64)
    k_split_recs<double><<<stride_grid(c), 256, 0, s>>>(adj2.as<EdgeRec<double>>(),
                                                        kc.as<uint32_t>(), kw.as<double>(), m);
  else
    k_split_recs<uint32_t><<<stride_grid(c), 256, 0, s>>>(adj2.as<EdgeRec<uint32_t>>(),
                                                          kc.as<uint32_t>(), kw.as<uint32_t>(), m);
  GFB_CUDA(cudaGetLastError());
  if (ro_out) GFB_CUDA(cudaMemcpyAsync(ro_out, ro2.p, (size_t)(n + 1) * 4, cudaMemcpyDeviceToHost, s));
  if (col_out) GFB_CUDA(cudaMemcpyAsync(col_out, kc.p, m * 4, cudaMemcpyDeviceToHost, s));
  if (w_out) GFB_CUDA(cudaMemcpyAsync(w_out, kw.p, m * wb, cudaMemcpyDeviceToHost, s));
  if (perm_out) GFB_CUDA(cudaMemcpyAsync(perm_out, perm.p, (size_t)n * 4, cudaMemcpyDeviceToHost, s));
  c->sync();
}

void ensure_relabel(Graph* g) {
  if (g->rl_valid) return;
  Ctx* c = g->ctx;
  cudaStream_t s = c->stream;
  const uint32_t n = (uint32_t)g->n;
  const uint64_t m = g->m;
  TBuf cnt;
  cnt.alloc((size_t)n * 4, s);
  if (g->rl_perm.bytes < (size_t)n * 4) {
    invalidate_loop_graphs(g);
    g->rl_perm.alloc((size_t)n * 4, s);
    g->rl_iperm.alloc((size_t)n * 4, s);
    g->rl_ro.alloc((size_t)(n + 1) * 4, s);
    g->rl_adj.alloc(m * g->rec_bytes(), s);
  }
  indegrees(g, cnt.as<uint32_t>());
  {  // only skewed in-degrees profit (grids lose their locality): max >= 32x mean
    TBuf mx, tmpr;
    mx.alloc(8, s);
    size_t tr = 0;
    GFB_CUDA(cub::DeviceReduce::Max(nullptr, tr, cnt.as<uint32_t>(), mx.as<uint32_t>(), (int64_t)n, s));
    tmpr.alloc(tr, s);
    GFB_CUDA(cub::DeviceReduce::Max(tmpr.p, tr, cnt.as<uint32_t>(), mx.as<uint32_t>(), (int64_t)n, s));
    uint32_t hmax = 0;
    GFB_CUDA(cudaMemcpyAsync(&hmax, mx.p, 4, cudaMemcpyDeviceToHost, s));
    c->sync();
    g->rl_skip = (double)hmax < 32.0 * (double)m / (double)std::max<uint32_t>(n, 1);
    if (g->rl_skip) {
      g->rl_valid = true;
      return;
    }
  }
  build_relabelled(g, cnt.as<uint32_t>(), g->rl_perm.as<uint32_t>(), g->rl_iperm.as<uint32_t>(),
                   g->rl_ro.as<uint32_t>(), g->rl_adj.p);
  c->sync();  // temporaries are stream-ordered frees; keep the build synchronous
  g->rl_valid = true;
}

Graph* graph_upload(Ctx* c, uint64_t n, uint64_t m, const uint32_t* ro, const uint32_t* col,
                    const void* w, int htype, int wtype, int build_csc_flag, uint64_t col_bound) {
  if (wtype < GFB_W_U32 || wtype > GFB_W_F64) fail(GFB_EINVAL, "graph: bad weight type");
  if (n >= (1ull << 31) || m >= (1ull << 31))
    fail(GFB_EINVAL, "graph: device path needs n < 2^31 and m < 2^31");
  auto g = std::make_unique<Graph>();
  g->ctx = c;
  g->n = n;
  g->m = m;
  g->col_bound = col_bound ? col_bound : n;
  g->wtype = wtype;
  g->ro.alloc((n + 1) * 4, c->stream);
  g->adj.alloc(m * g->rec_bytes(), c->stream);
  fill_graph(g.get(), ro, col, w, htype);
  g->csc_wanted = build_csc_flag != 0;  // built on first use (ensure_csc)
  return g.release();
}

void graph_refill(Graph* g, const uint32_t* ro, const uint32_t* col, const void* w, int htype) {
  fill_graph(g, ro, col, w, htype);  // the transpose is rebuilt on first use
}

// The transpose is built lazily: a push-only or AUTO (alpha <= 1) sssp and
// the transpose-free predecessor repair never need it, and its radix sort is
// the largest part of an upload after the H2D copy (~25 ms at s24).
void ensure_csc(Graph* g) {
  if (!g->csc_wanted || g->has_csc) return;
  build_csc(g);
  build_pull_plan(g);
}

// ---------------------------------------------------------------------------
// Device build_transpose (graph.hpp:166-193).  A stable radix sort of the
// CSR edge ids by destination gives exactly the reference slot order
// (ascending source, then CSR edge id, within each destination).
// ---------------------------------------------------------------------------
__global__ void k_dst_keys(const void* adj, int recb, uint32_t* keys, uint32_t* ids, uint64_t m) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
    keys[e] = *reinterpret_cast<const uint32_t*>(static_cast<const char*>(adj) + e * recb);
    ids[e] = (uint32_t)e;
  }
}

__global__ void k_row_marks(const uint32_t* ro, uint32_t* mark, uint64_t n) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride)
    if (ro[v + 1] > ro[v]) mark[ro[v]] = (uint32_t)v;  // one non-empty row per start
}

// offsets from sorted keys: off[v] = first index i with keys[i] >= v,
// off[n] = m (the count+scan of graph.hpp:154-160 done from sorted keys).
__global__ void k_offsets_from_sorted(const uint32_t* keys, uint64_t m, uint32_t* off,
                                      uint64_t n) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= m; i += stride) {
    int64_t prev = i == 0 ? -1 : (int64_t)keys[i - 1];
    int64_t cur = i < m ? (int64_t)keys[i] : (int64_t)n;
    for (int64_t v = prev + 1; v <= cur; ++v) off[v] = (uint32_t)i;
  }
}

template <class W>
__global__ void k_csc_fill(const EdgeRec<W>* adj, const uint32_t* sorted_eid,
                           const uint32_t* src_of, EdgeRec<W>* cadj, uint32_t* ceid, uint64_t m) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < m; s += stride) {
    uint32_t e = sorted_eid[s];
    EdgeRec<W> r = adj[e];
    r.v = src_of[e];
    cadj[s] = r;
    ceid[s] = e;
  }
}

static int bits_for(uint64_t n) {
  int b = 1;
  while ((1ull << b) < n) ++b;
  return b;
}

struct MaxOp {
  __device__ __forceinline__ uint32_t operator()(uint32_t a, uint32_t b) const {
    return a > b ? a : b;
  }
};

// src_of[e] = source vertex of CSR edge e (row marks + inclusive max-scan).
static void source_of_edges(Graph* g, DBuf& src_of) {
  Ctx* c = g->ctx;
  cudaStream_t s = c->stream;
  src_of.alloc(g->m * 4, s);
  GFB_CUDA(cudaMemsetAsync(src_of.p, 0, g->m * 4, s));
  k_row_marks<<<stride_grid(c), 256, 0, s>>>(g->ro.as<uint32_t>(), src_of.as<uint32_t>(), g->n);
  size_t tb = 0;
  GFB_CUDA(cub::DeviceScan::InclusiveScan(nullptr, tb, src_of.as<uint32_t>(),
                                          src_of.as<uint32_t>(), MaxOp(), (int64_t)g->m, s));
  TBuf tmp;
  tmp.alloc(tb, s);
  GFB_CUDA(cub::DeviceScan::InclusiveScan(tmp.p, tb, src_of.as<uint32_t>(),
                                          src_of.as<uint32_t>(), MaxOp(), (int64_t)g->m, s));
}

// payload for the CSC sort: key = dst, value = the CSC record {src, w} as one
// 64-bit word (low 32 bits = src, high = weight bits: EdgeRec<W> layout)
template <class W>
__global__ void k_csc_payload(const EdgeRec<W>* __restrict__ adj, const uint32_t* __restrict__ src_of,
                              uint32_t* keys, unsigned long long* vals, uint64_t m) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
    EdgeRec<W> r = adj[e];
    keys[e] = r.v;
    vals[e] = ((unsigned long long)(*reinterpret_cast<const uint32_t*>(&r.w)) << 32) | src_of[e];
  }
}

// CSC slot -> CSR edge id (graph.hpp:188 back-map), for the operator-level
// record condition only: slots of v are in ascending (src, CSR id) order and
// parallel edges u->v are contiguous in u's sorted row, so
// id = ro[u] + lower_bound(row u, v) + (slot - first slot of v with source u).
template <class W>
__global__ void k_ceid(const uint32_t* __restrict__ co, const EdgeRec<W>* __restrict__ cadj,
                       const uint32_t* __restrict__ ro, const EdgeRec<W>* __restrict__ adj,
                       uint32_t n, uint32_t* ceid) {
  const int lane = threadIdx.x & 31;
  uint32_t warps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t v = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); v < n; v += warps) {
    const uint32_t s0 = co[v], s1 = co[v + 1];
    for (uint32_t sl = s0 + lane; sl < s1; sl += 32) {
      const uint32_t u = cadj[sl].v;
      uint32_t lo = s0, hi = sl;  // first slot of v with source u
      while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        if (cadj[mid].v < u) lo = mid + 1;
        else hi = mid;
      }
      uint32_t a = ro[u], b = ro[u + 1];  // lower_bound(row u, v)
      while (a < b) {
        uint32_t mid = (a + b) >> 1;
        if (adj[mid].v < v) a = mid + 1;
        else b = mid;
      }
      ceid[sl] = a + (sl - lo);
    }
  }
}

void ensure_ceid(Graph* g) {
  ensure_csc(g);
  if (!g->has_csc || g->ceid.p) return;
  Ctx* c = g->ctx;
  invalidate_loop_graphs(g);
  g->ceid.alloc(g->m * 4, c->stream);
  if (g->m) {
    if (g->wtype == GFB_W_F32)
      k_ceid<float><<<stride_grid(c), 256, 0, c->stream>>>(
          g->co.as<uint32_t>(), g->cadj.as<EdgeRec<float>>(), g->ro.as<uint32_t>(),
          g->adj.as<EdgeRec<float>>(), (uint32_t)g->n, g->ceid.as<uint32_t>());
    else
      k_ceid<uint32_t><<<stride_grid(c), 256, 0, c->stream>>>(
          g->co.as<uint32_t>(), g->cadj.as<EdgeRec<uint32_t>>(), g->ro.as<uint32_t>(),
          g->adj.as<EdgeRec<uint32_t>>(), (uint32_t)g->n, g->ceid.as<uint32_t>());
    GFB_CUDA(cudaGetLastError());
  }
  c->sync();
}

void build_csc(Graph* g) {
  invalidate_loop_graphs(g);
  Ctx* c = g->ctx;
  cudaStream_t s = c->stream;
  const uint64_t n = g->n, m = g->m;
  g->co.alloc((n + 1) * 4, s);
  g->ceid.release();
  if (m == 0) {
    g->cadj.alloc(16, s);
    g->ceid.alloc(16, s);
    GFB_CUDA(cudaMemsetAsync(g->co.p, 0, (n + 1) * 4, s));
    g->has_csc = true;
    c->sync();
    return;
  }
  TBuf src_of;
  source_of_edges(g, src_of);
  if (g->wtype != GFB_W_F64) {
    // one stable radix sort of {src, w} payloads by dst: the sorted payloads
    // ARE the CSC records in build_transpose slot order (graph.hpp:180-190)
    TBuf keys, keys2, vals;
    keys.alloc(m * 4, s);
    keys2.alloc(m * 4, s);
    vals.alloc(m * 8, s);
    g->cadj.alloc(m * 8, s);
    if (g->wtype == GFB_W_F32)
      k_csc_payload<float><<<stride_grid(c), 256, 0, s>>>(
          g->adj.as<EdgeRec<float>>(), src_of.as<uint32_t>(), keys.as<uint32_t>(),
          vals.as<unsigned long long>(), m);
    else
      k_csc_payload<uint32_t><<<stride_grid(c), 256, 0, s>>>(
          g->adj.as<EdgeRec<uint32_t>>(), src_of.as<uint32_t>(), keys.as<uint32_t>(),
          vals.as<unsigned long long>(), m);
    GFB_CUDA(cudaGetLastError());
    src_of.release();
    size_t tb = 0;
    GFB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.as<uint32_t>(), keys2.as<uint32_t>(),
                                             vals.as<unsigned long long>(),
                                             g->cadj.as<unsigned long long>(), (int64_t)m, 0,
                                             bits_for(n), s));
    TBuf tmp;
    tmp.alloc(tb, s);
    GFB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys.as<uint32_t>(), keys2.as<uint32_t>(),
                                             vals.as<unsigned long long>(),
                                             g->cadj.as<unsigned long long>(), (int64_t)m, 0,
                                             bits_for(n), s));
    k_offsets_from_sorted<<<stride_grid(c), 256, 0, s>>>(keys2.as<uint32_t>(), m,
                                                         g->co.as<uint32_t>(), n);
    GFB_CUDA(cudaGetLastError());
    c->sync();
    g->has_csc = true;
    return;
  }
  // f64 (16-byte records): sort CSR ids by dst, then gather records + ids
  g->cadj.alloc(m * g->rec_bytes(), s);
  g->ceid.alloc(m * 4, s);
  TBuf keys, ids, keys2, ids2;
  keys.alloc(m * 4, s);
  ids.alloc(m * 4, s);
  keys2.alloc(m * 4, s);
  ids2.alloc(m * 4, s);
  k_dst_keys<<<stride_grid(c), 256, 0, s>>>(g->adj.p, (int)g->rec_bytes(), keys.as<uint32_t>(),
                                            ids.as<uint32_t>(), m);
  size_t tb = 0;
  GFB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.as<uint32_t>(), keys2.as<uint32_t>(),
                                           ids.as<uint32_t>(), ids2.as<uint32_t>(), (int64_t)m, 0,
                                           bits_for(n), s));
  TBuf tmp;
  tmp.alloc(tb, s);
  GFB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys.as<uint32_t>(), keys2.as<uint32_t>(),
                                           ids.as<uint32_t>(), ids2.as<uint32_t>(), (int64_t)m, 0,
                                           bits_for(n), s));
  tmp.release();
  keys.release();
  ids.release();
  k_offsets_from_sorted<<<stride_grid(c), 256, 0, s>>>(keys2.as<uint32_t>(), m,
                                                       g->co.as<uint32_t>(), n);
  k_csc_fill<double><<<stride_grid(c), 256, 0, s>>>(g->adj.as<EdgeRec<double>>(), ids2.as<uint32_t>(),
                                                    src_of.as<uint32_t>(), g->cadj.as<EdgeRec<double>>(),
                                                    g->ceid.as<uint32_t>(), m);
  GFB_CUDA(cudaGetLastError());
  c->sync();
  g->has_csc = true;
}

// Static pull plan: k_compact over the CSC offsets with an all-ones bitmap
// drops destinations of in-degree 0 and emits the edge-tile map.
__global__ void k_fill_ones(uint32_t* bm, uint64_t nwords, uint64_t n) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nwords; i += stride) {
    uint64_t lo = i * 32;
    uint32_t w = 0xFFFFFFFFu;
    if (lo + 32 > n) w = (n > lo) ? ((1u << (n - lo)) - 1u) : 0u;
    bm[i] = w;
  }
}

void build_pull_plan(Graph* g) {
  invalidate_loop_graphs(g);
  Ctx* c = g->ctx;
  cudaStream_t s = c->stream;
  const uint64_t n = g->n, m = g->m;
  const uint64_t nwords = (n + 31) / 32;
  const uint32_t ntiles = (uint32_t)((nwords + C_WORDS - 1) / C_WORDS);
  g->pull_v.alloc((n + 1) * 4, s);
  g->pull_off.alloc((n + 1) * 4, s);
  g->pull_tseg.alloc((m / PLAN_GRAIN + 3) * 4, s);
  TBuf bm, ctl, status;
  bm.alloc(nwords * 4, s);
  ctl.alloc(sizeof(Ctl), s);
  status.alloc((size_t)(ntiles + 1) * 8, s);
  GFB_CUDA(cudaMemsetAsync(ctl.p, 0, sizeof(Ctl), s));
  GFB_CUDA(cudaMemsetAsync(status.p, 0, (size_t)(ntiles + 1) * 8, s));
  if (n == 0) {
    g->pull_k = 0;
    g->pull_total = 0;
    c->sync();
    return;
  }
  k_fill_ones<<<stride_grid(c), 256, 0, s>>>(bm.as<uint32_t>(), nwords, n);
  // start and off coincide for a complete plan: start = co[v] = off
  TBuf start;
  start.alloc((n + 1) * 4, s);
  Plan p{g->pull_v.as<uint32_t>(), start.as<uint32_t>(), g->pull_off.as<uint32_t>(),
         g->pull_tseg.as<uint32_t>(), (uint32_t)(g->pull_tseg.bytes / 4)};
  k_compact<<<ntiles, C_WARPS * 32, 0, s>>>(g->co.as<uint32_t>(), bm.as<uint32_t>(), nullptr,
                                            (uint32_t)nwords, (uint32_t)n, p, ctl.as<Ctl>(),
                                            status.as<unsigned long long>(), ntiles, 1);
  GFB_CUDA(cudaGetLastError());
  Ctl h = c->read_ctl(ctl.as<Ctl>());
  g->pull_k = h.k;
  g->pull_total = h.total;
}

// ---------------------------------------------------------------------------
// Device-side synthetic graphs in build_csr layout.
// ---------------------------------------------------------------------------
__global__ void k_rmat_gen(int scale, uint64_t seed, int wkind, uint64_t m,
                           unsigned long long* key, uint32_t* wbits) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    uint32_t s, d, w;
    rmat_edge(scale, seed, wkind, i, &s, &d, &w);
    key[i] = ((unsigned long long)s << 32) | d;
    wbits[i] = w;
  }
}

__global__ void k_unpack_sorted(const unsigned long long* key, const uint32_t* wbits,
                                uint32_t* srcs, EdgeRec<uint32_t>* adj, uint64_t m) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    unsigned long long k = key[i];
    srcs[i] = (uint32_t)(k >> 32);
    adj[i] = EdgeRec<uint32_t>{(uint32_t)k, wbits[i]};
  }
}

Graph* graph_generate_rmat(Ctx* c, int scale, int ef, uint64_t seed, int wtype, int csc) {
  if (scale < 1 || scale > 30 || ef < 1) fail(GFB_EINVAL, "rmat: bad scale/edgefactor");
  if (wtype != GFB_W_U32 && wtype != GFB_W_F32) fail(GFB_EINVAL, "rmat: wtype must be u32 or f32");
  const uint64_t n = 1ull << scale, m = (uint64_t)ef << scale;
  if (m >= (1ull << 31)) fail(GFB_EINVAL, "rmat: m must be < 2^31");
  cudaStream_t s = c->stream;
  auto g = std::make_unique<Graph>();
  g->ctx = c;
  g->n = n;
  g->m = m;
  g->wtype = wtype;
  g->ro.alloc((n + 1) * 4, s);
  g->adj.alloc(m * 8, s);
  {
    TBuf key, key2, wb, wb2;
    key.alloc(m * 8, s);
    key2.alloc(m * 8, s);
    wb.alloc(m * 4, s);
    wb2.alloc(m * 4, s);
    k_rmat_gen<<<stride_grid(c), 256, 0, s>>>(scale, seed, wtype == GFB_W_U32 ? 0 : 1, m,
                                              key.as<unsigned long long>(), wb.as<uint32_t>());
    GFB_CUDA(cudaGetLastError());
    // (src, dst, w) order: stable sort by w, then stable sort by (src, dst).
    size_t tb1 = 0, tb2 = 0;
    GFB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb1, wb.as<uint32_t>(), wb2.as<uint32_t>(),
                                             key.as<unsigned long long>(),
                                             key2.as<unsigned long long>(), (int64_t)m, 0, 32, s));
    GFB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb2, key2.as<unsigned long long>(),
                                             key.as<unsigned long long>(), wb2.as<uint32_t>(),
                                             wb.as<uint32_t>(), (int64_t)m, 0, 32 + scale, s));
    TBuf tmp;
    tmp.alloc(tb1 > tb2 ? tb1 : tb2, s);
    size_t tb = tmp.bytes;
    GFB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, wb.as<uint32_t>(), wb2.as<uint32_t>(),
                                             key.as<unsigned long long>(),
                                             key2.as<unsigned long long>(), (int64_t)m, 0, 32, s));
    tb = tmp.bytes;
    GFB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, key2.as<unsigned long long>(),
                                             key.as<unsigned long long>(), wb2.as<uint32_t>(),
                                             wb.as<uint32_t>(), (int64_t)m, 0, 32 + scale, s));
    tmp.release();
    key2.release();
    TBuf srcs;
    srcs.alloc(m * 4, s);
    k_unpack_sorted<<<stride_grid(c), 256, 0, s>>>(key.as<unsigned long long>(), wb.as<uint32_t>(),
                                                   srcs.as<uint32_t>(),
                                                   g->adj.as<EdgeRec<uint32_t>>(), m);
    k_offsets_from_sorted<<<stride_grid(c), 256, 0, s>>>(srcs.as<uint32_t>(), m,
                                                         g->ro.as<uint32_t>(), n);
    GFB_CUDA(cudaGetLastError());
    c->sync();
  }
  g->csc_wanted = csc != 0;  // built on first use (ensure_csc)
  return g.release();
}

// ---------------------------------------------------------------------------
// build_csr (graph.hpp:132-162) on the device from a host edge list (Matrix
// Market ingest, mm.cu): validation naming the first bad edge (:134-142),
// order (src, dst, weight) by two stable radix sorts (weight bits, then
// (src, dst) -- non-negative IEEE weights order like their bits, and the
// conversion to the device arithmetic is monotone), count + scan.
// ---------------------------------------------------------------------------
template <class W>
__global__ void k_edges_in(const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst,
                           const double* __restrict__ w, uint64_t m, uint64_t n, int shift,
                           unsigned long long* key, typename DT<W>::Bits* wb,
                           unsigned long long* bad) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    const uint32_t s = src[i], d = dst[i];
    W x{};
    const bool okw = conv_weight<W>(w, GFB_W_F64, i, &x);
    if (s >= n || d >= n) atomicMin(bad, (unsigned long long)i);
    else if (!okw) atomicMin(bad + 1, (unsigned long long)i);
    key[i] = ((unsigned long long)s << shift) | d;
    wb[i] = *reinterpret_cast<typename DT<W>::Bits*>(&x);
  }
}

template <class W>
__global__ void k_edges_out(const unsigned long long* __restrict__ key,
                            const typename DT<W>::Bits* __restrict__ wb, uint64_t m, int shift,
                            uint32_t* srcs, EdgeRec<W>* adj) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const unsigned long long dmask = (1ull << shift) - 1;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    const unsigned long long k = key[i];
    srcs[i] = (uint32_t)(k >> shift);
    EdgeRec<W> r{};
    r.v = (uint32_t)(k & dmask);
    const typename DT<W>::Bits b = wb[i];
    r.w = *reinterpret_cast<const W*>(&b);
    adj[i] = r;
  }
}

template <class W>
static void edges_build(Graph* g, const uint32_t* hsrc, const uint32_t* hdst, const double* hw) {
  using Bits = typename DT<W>::Bits;
  Ctx* c = g->ctx;
  cudaStream_t s = c->stream;
  const uint64_t n = g->n, m = g->m;
  const int shift = bits_for(n);
  TBuf dsrc, ddst, dw, key, key2, wb, wb2, flags;
  dsrc.alloc(m * 4, s);
  ddst.alloc(m * 4, s);
  dw.alloc(m * 8, s);
  key.alloc(m * 8, s);
  key2.alloc(m * 8, s);
  wb.alloc(m * sizeof(Bits), s);
  wb2.alloc(m * sizeof(Bits), s);
  flags.alloc(16, s);
  GFB_CUDA(cudaMemcpyAsync(dsrc.p, hsrc, m * 4, cudaMemcpyHostToDevice, s));
  GFB_CUDA(cudaMemcpyAsync(ddst.p, hdst, m * 4, cudaMemcpyHostToDevice, s));
  GFB_CUDA(cudaMemcpyAsync(dw.p, hw, m * 8, cudaMemcpyHostToDevice, s));
  GFB_CUDA(cudaMemsetAsync(flags.p, 0xFF, 16, s));
  k_edges_in<W><<<stride_grid(c), 256, 0, s>>>(dsrc.as<uint32_t>(), ddst.as<uint32_t>(),
                                               dw.as<double>(), m, n, shift,
                                               key.as<unsigned long long>(), wb.as<Bits>(),
                                               flags.as<unsigned long long>());
  GFB_CUDA(cudaGetLastError());
  unsigned long long hf[2];
  GFB_CUDA(cudaMemcpyAsync(hf, flags.p, 16, cudaMemcpyDeviceToHost, s));
  c->sync();
  const unsigned long long first = std::min(hf[0], hf[1]);
  if (first != ~0ull) {  // the reference reports the first offending edge
    if (first == hf[0])
      fail(GFB_EINVAL, "build_csr: edge " + std::to_string(first) + " has vertex id out of range");
    fail(GFB_EINVAL,
         "build_csr: edge " + std::to_string(first) + " has negative or non-finite weight");
  }
  dsrc.release();
  ddst.release();
  dw.release();
  size_t tb1 = 0, tb2 = 0;
  GFB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb1, wb.as<Bits>(), wb2.as<Bits>(),
                                           key.as<unsigned long long>(),
                                           key2.as<unsigned long long>(), (int64_t)m, 0,
                                           (int)(8 * sizeof(Bits)), s));
  GFB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb2, key2.as<unsigned long long>(),
                                           key.as<unsigned long long>(), wb2.as<Bits>(),
                                           wb.as<Bits>(), (int64_t)m, 0, 2 * shift, s));
  TBuf tmp;
  tmp.alloc(std::max(tb1, tb2), s);
  size_t tb = tmp.bytes;
  GFB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, wb.as<Bits>(), wb2.as<Bits>(),
                                           key.as<unsigned long long>(),
                                           key2.as<unsigned long long>(), (int64_t)m, 0,
                                           (int)(8 * sizeof(Bits)), s));
  tb = tmp.bytes;
  GFB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, key2.as<unsigned long long>(),
                                           key.as<unsigned long long>(), wb2.as<Bits>(),
                                           wb.as<Bits>(), (int64_t)m, 0, 2 * shift, s));
  tmp.release();
  TBuf srcs;
  srcs.alloc(m * 4, s);
  k_edges_out<W><<<stride_grid(c), 256, 0, s>>>(key.as<unsigned long long>(), wb.as<Bits>(), m,
                                                shift, srcs.as<uint32_t>(),
                                                g->adj.as<EdgeRec<W>>());
  k_offsets_from_sorted<<<stride_grid(c), 256, 0, s>>>(srcs.as<uint32_t>(), m,
                                                       g->ro.as<uint32_t>(), n);
  GFB_CUDA(cudaGetLastError());
  c->sync();
}

Graph* graph_from_edges(Ctx* c, uint64_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                        const double* w, int wtype, int csc) {
  if (wtype < GFB_W_U32 || wtype > GFB_W_F64) fail(GFB_EINVAL, "graph: bad weight type");
  if (n >= (1ull << 31) || m >= (1ull << 31))
    fail(GFB_EINVAL, "graph: device path needs n < 2^31 and m < 2^31");
  if (m && (!src || !dst || !w)) fail(GFB_EINVAL, "graph: null edge arrays");
  auto g = std::make_unique<Graph>();
  g->ctx = c;
  g->n = n;
  g->m = m;
  g->col_bound = n;
  g->wtype = wtype;
  cudaStream_t s = c->stream;
  g->ro.alloc((n + 1) * 4, s);
  g->adj.alloc(std::max<uint64_t>(m, 1) * g->rec_bytes(), s);
  if (m == 0) {
    GFB_CUDA(cudaMemsetAsync(g->ro.p, 0, (n + 1) * 4, s));
    c->sync();
  } else if (wtype == GFB_W_F32) {
    edges_build<float>(g.get(), src, dst, w);
  } else if (wtype == GFB_W_F64) {
    edges_build<double>(g.get(), src, dst, w);
  } else {
    edges_build<uint32_t>(g.get(), src, dst, w);
  }
  g->csc_wanted = csc != 0;  // built on first use (ensure_csc)
  return g.release();
}

__global__ void k_grid_deg(uint32_t side, uint32_t* deg) {
  uint64_t n = (uint64_t)side * side;
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n; u += stride) {
    uint32_t r = (uint32_t)(u / side), cc = (uint32_t)(u % side);
    deg[u] = (r > 0) + (cc > 0) + (cc + 1 < side) + (r + 1 < side);
  }
}

__global__ void k_grid_fill(uint32_t side, uint64_t seed, const uint32_t* ro,
                            EdgeRec<uint32_t>* adj) {
  uint64_t n = (uint64_t)side * side;
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n; u += stride) {
    uint32_t r = (uint32_t)(u / side), cc = (uint32_t)(u % side);
    uint32_t e = ro[u];
    bool ok[4] = {r > 0, cc > 0, cc + 1 < side, r + 1 < side};
    uint64_t nb[4] = {u - side, u - 1, u + 1, u + side};
    for (int k = 0; k < 4; ++k) {
      if (!ok[k]) continue;
      adj[e++] = EdgeRec<uint32_t>{(uint32_t)nb[k], grid_weight_bits(seed, u, k)};
    }
  }
}

Graph* graph_generate_grid(Ctx* c, uint32_t side, uint64_t seed, int csc) {
  const uint64_t n = (uint64_t)side * side;
  const uint64_t m = side < 2 ? 0 : 4ull * side * (side - 1);
  if (side == 0 || n >= (1ull << 31) || m >= (1ull << 31)) fail(GFB_EINVAL, "grid: bad side");
  cudaStream_t s = c->stream;
  auto g = std::make_unique<Graph>();
  g->ctx = c;
  g->n = n;
  g->m = m;
  g->wtype = GFB_W_F32;
  g->ro.alloc((n + 1) * 4, s);
  g->adj.alloc(m * 8, s);
  TBuf deg;
  deg.alloc((n + 1) * 4, s);
  GFB_CUDA(cudaMemsetAsync(deg.p, 0, (n + 1) * 4, s));
  k_grid_deg<<<stride_grid(c), 256, 0, s>>>(side, deg.as<uint32_t>());
  size_t tb = 0;
  GFB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, deg.as<uint32_t>(), g->ro.as<uint32_t>(),
                                         (int64_t)(n + 1), s));
  TBuf tmp;
  tmp.alloc(tb, s);
  GFB_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, deg.as<uint32_t>(), g->ro.as<uint32_t>(),
                                         (int64_t)(n + 1), s));
  k_grid_fill<<<stride_grid(c), 256, 0, s>>>(side, seed, g->ro.as<uint32_t>(),
                                             g->adj.as<EdgeRec<uint32_t>>());
  GFB_CUDA(cudaGetLastError());
  c->sync();
  g->csc_wanted = csc != 0;  // built on first use (ensure_csc)
  return g.release();
}

// ---------------------------------------------------------------------------
template <class W>
__global__ void k_split(const EdgeRec<W>* adj, uint32_t* col, W* w, uint64_t m) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
    EdgeRec<W> r = adj[e];
    if (col) col[e] = r.v;
    if (w) w[e] = r.w;
  }
}

void graph_download(Graph* g, uint32_t* ro, uint32_t* col, void* w) {
  Ctx* c = g->ctx;
  cudaStream_t s = c->stream;
  if (ro) GFB_CUDA(cudaMemcpyAsync(ro, g->ro.p, (g->n + 1) * 4, cudaMemcpyDeviceToHost, s));
  if ((col || w) && g->m) {
    size_t wb = g->wtype == GFB_W_F64 ? 8 : 4;
    TBuf dc, dw;
    dc.alloc(g->m * 4, s);
    dw.alloc(g->m * wb, s);
    if (g->wtype == GFB_W_F32)
      k_split<float><<<stride_grid(c), 256, 0, s>>>(g->adj.as<EdgeRec<float>>(), dc.as<uint32_t>(), dw.as<float>(), g->m);
    else if (g->wtype == GFB_W_F64)
      k_split<double><<<stride_grid(c), 256, 0, s>>>(g->adj.as<EdgeRec<double>>(), dc.as<uint32_t>(), dw.as<double>(), g->m);
    else
      k_split<uint32_t><<<stride_grid(c), 256, 0, s>>>(g->adj.as<EdgeRec<uint32_t>>(), dc.as<uint32_t>(), dw.as<uint32_t>(), g->m);
    GFB_CUDA(cudaGetLastError());
    if (col) GFB_CUDA(cudaMemcpyAsync(col, dc.p, g->m * 4, cudaMemcpyDeviceToHost, s));
    if (w) GFB_CUDA(cudaMemcpyAsync(w, dw.p, g->m * wb, cudaMemcpyDeviceToHost, s));
    c->sync();
  }
  c->sync();
}

}  // namespace gfb

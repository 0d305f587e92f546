/*
 * graflow_oracle.c -- CPU restatement of the reference SSSP path.
 *
 * TEST INFRASTRUCTURE ONLY (see graflow_oracle.h).  Plain C99, single
 * threaded, deterministic.  Each function cites the reference file:line it
 * restates (paths relative to the reference's proj/ directory).
 */
#include "graflow_oracle.h"

#include <math.h>
#include <omp.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* std::mt19937_64, per the C++11 [rand.predef] parameters.  Used by         */
/* tests/random_graphs.hpp:17 (the reference's seeded corpus).               */
/* ------------------------------------------------------------------------ */
#define MT_N 312
#define MT_M 156
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x000000007FFFFFFFULL

void orc_mt64_seed(orc_mt64* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) +
               (uint64_t)i;
  r->idx = MT_N;
}

static void mt_twist(orc_mt64* r) {
  for (int i = 0; i < MT_N; ++i) {
    uint64_t x = (r->mt[i] & MT_UPPER) | (r->mt[(i + 1) % MT_N] & MT_LOWER);
    uint64_t xa = x >> 1;
    if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
    r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
  }
  r->idx = 0;
}

uint64_t orc_mt64_next(orc_mt64* r) {
  if (r->idx >= MT_N) mt_twist(r);
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* libstdc++ bits/random.tcc generate_canonical<double, 53>: one 64-bit draw,
 * rounded to double, divided by 2^64, clamped below 1. */
double orc_canonical(orc_mt64* r) {
  double sum = (double)orc_mt64_next(r);
  double ret = sum / 18446744073709551616.0;
  if (ret >= 1.0) ret = nextafter(1.0, 0.0);
  return ret;
}

/* random_graphs.hpp:15-30: for u, for v: coin >= 4/n -> skip; weight is 0
 * with probability 0.1 else U[0,10) (uniform_real_distribution: x*(b-a)+a). */
size_t orc_random_edges(size_t n, uint64_t seed, uint32_t* src, uint32_t* dst,
                        double* w, size_t cap) {
  orc_mt64 rng;
  orc_mt64_seed(&rng, seed);
  double p = 4.0 / (double)n;
  size_t count = 0;
  for (uint32_t u = 0; u < n; ++u) {
    for (uint32_t v = 0; v < n; ++v) {
      if (orc_canonical(&rng) * (1.0 - 0.0) + 0.0 >= p) continue;
      double wt = (orc_canonical(&rng) * (1.0 - 0.0) + 0.0) < 0.1
                      ? 0.0
                      : orc_canonical(&rng) * (10.0 - 0.0) + 0.0;
      if (count < cap) {
        src[count] = u;
        dst[count] = v;
        w[count] = wt;
      }
      ++count;
    }
  }
  return count;
}

/* ------------------------------------------------------------------------ */
/* graph.hpp:132-162 build_csr                                               */
/* ------------------------------------------------------------------------ */
typedef struct {
  uint32_t s, d;
  double w;
} orc_edge;

static int edge_cmp(const void* a, const void* b) {
  const orc_edge* x = (const orc_edge*)a;
  const orc_edge* y = (const orc_edge*)b;
  /* std::tie(src, dst, weight) < ... (graph.hpp:163-165) */
  if (x->s != y->s) return x->s < y->s ? -1 : 1;
  if (x->d != y->d) return x->d < y->d ? -1 : 1;
  if (x->w != y->w) return x->w < y->w ? -1 : 1;
  return 0;
}

int64_t orc_build_csr(size_t n, size_t m, const uint32_t* src,
                      const uint32_t* dst, const double* w, uint32_t* ro,
                      uint32_t* col, double* val) {
  for (size_t i = 0; i < m; ++i) { /* graph.hpp:134-142 */
    if (src[i] >= n || dst[i] >= n) return (int64_t)i;
    if (!(w[i] >= 0) || !isfinite(w[i])) return (int64_t)i;
  }
  orc_edge* e = (orc_edge*)malloc((m ? m : 1) * sizeof(orc_edge));
  for (size_t i = 0; i < m; ++i) {
    e[i].s = src[i];
    e[i].d = dst[i];
    e[i].w = w[i];
  }
  qsort(e, m, sizeof(orc_edge), edge_cmp); /* graph.hpp:144-147 */
  memset(ro, 0, (n + 1) * sizeof(uint32_t));
  for (size_t i = 0; i < m; ++i) { /* graph.hpp:154-158 */
    ++ro[e[i].s + 1];
    col[i] = e[i].d;
    val[i] = e[i].w;
  }
  for (size_t v = 0; v < n; ++v) ro[v + 1] += ro[v]; /* graph.hpp:159-160 */
  free(e);
  return -1;
}

/* graph.hpp:166-193 build_transpose */
void orc_build_transpose(size_t n, size_t m, const uint32_t* ro,
                         const uint32_t* col, const double* val,
                         uint32_t* cso, uint32_t* csrc, double* cval,
                         uint32_t* ceid) {
  memset(cso, 0, (n + 1) * sizeof(uint32_t));
  for (size_t e = 0; e < m; ++e) ++cso[col[e] + 1];          /* :193-194 */
  for (size_t u = 0; u < n; ++u) cso[u + 1] += cso[u];        /* :195-196 */
  uint32_t* cursor = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
  memcpy(cursor, cso, n * sizeof(uint32_t));                  /* :198-199 */
  for (uint32_t v = 0; v < n; ++v) {                          /* :200-208 */
    for (uint32_t e = ro[v]; e < ro[v + 1]; ++e) {
      uint32_t slot = cursor[col[e]]++;
      csrc[slot] = v;
      if (cval) cval[slot] = val[e];
      ceid[slot] = e;
    }
  }
  free(cursor);
}

/* ------------------------------------------------------------------------ */
/* algorithms.hpp:101-128 reference_dijkstra.  std::priority_queue with     */
/* std::greater<pair<key, vertex>> = a binary min-heap on (key, vertex).    */
/* The pop order only affects pred, never dist (unique fixpoint).           */
/* ------------------------------------------------------------------------ */
#define DEFINE_DIJKSTRA(NAME, KEY_T, W_T, WIDEN, INF)                          \
  typedef struct {                                                           \
    KEY_T k;                                                                 \
    uint32_t v;                                                              \
  } NAME##_ent;                                                              \
  static int NAME##_less(NAME##_ent a, NAME##_ent b) {                       \
    return a.k < b.k || (a.k == b.k && a.v < b.v);                           \
  }                                                                          \
  int NAME(size_t n, const uint32_t* ro, const uint32_t* col, const W_T* w,  \
           uint32_t source, KEY_T* dist, uint32_t* pred) {                   \
    if (source >= n) return -1; /* algorithms.hpp:104 out_of_range */        \
    for (size_t i = 0; i < n; ++i) {                                         \
      dist[i] = INF;                                                         \
      if (pred) pred[i] = ORC_NIL;                                           \
    }                                                                        \
    dist[source] = 0;                                                        \
    size_t cap = 1024, sz = 0;                                               \
    NAME##_ent* h = (NAME##_ent*)malloc(cap * sizeof(NAME##_ent));           \
    h[sz++] = (NAME##_ent){0, source};                                       \
    while (sz) {                                                             \
      NAME##_ent top = h[0];                                                 \
      h[0] = h[--sz];                                                        \
      for (size_t i = 0;;) { /* sift down */                                 \
        size_t l = 2 * i + 1, r = l + 1, s = i;                              \
        if (l < sz && NAME##_less(h[l], h[s])) s = l;                        \
        if (r < sz && NAME##_less(h[r], h[s])) s = r;                        \
        if (s == i) break;                                                   \
        NAME##_ent t = h[i];                                                 \
        h[i] = h[s];                                                         \
        h[s] = t;                                                            \
        i = s;                                                               \
      }                                                                      \
      KEY_T d = top.k;                                                       \
      uint32_t u = top.v;                                                    \
      if (d > dist[u]) continue; /* :551 stale entry */                      \
      for (uint32_t e = ro[u]; e < ro[u + 1]; ++e) {                         \
        uint32_t v = col[e];                                                 \
        KEY_T nd = d + WIDEN(w[e]);                                          \
        if (nd < dist[v]) { /* :555 strict relax */                          \
          dist[v] = nd;                                                      \
          if (pred) pred[v] = u;                                             \
          if (sz == cap) {                                                   \
            cap *= 2;                                                        \
            h = (NAME##_ent*)realloc(h, cap * sizeof(NAME##_ent));           \
          }                                                                  \
          size_t i = sz++; /* sift up */                                     \
          h[i] = (NAME##_ent){nd, v};                                        \
          while (i && NAME##_less(h[i], h[(i - 1) / 2])) {                   \
            NAME##_ent t = h[i];                                             \
            h[i] = h[(i - 1) / 2];                                           \
            h[(i - 1) / 2] = t;                                              \
            i = (i - 1) / 2;                                                 \
          }                                                                  \
        }                                                                    \
      }                                                                      \
    }                                                                        \
    free(h);                                                                 \
    return 0;                                                                \
  }

#define WIDEN_ID(x) (x)
#define WIDEN_U64(x) ((uint64_t)(x))
DEFINE_DIJKSTRA(orc_dijkstra_f64, double, double, WIDEN_ID, INFINITY)
DEFINE_DIJKSTRA(orc_dijkstra_f32, float, float, WIDEN_ID, INFINITY)
DEFINE_DIJKSTRA(orc_dijkstra_u32, uint64_t, uint32_t, WIDEN_U64, UINT64_MAX)

/* ------------------------------------------------------------------------ */
/* algorithms.hpp:134-188 sssp(), Sequential policy, push direction, in f32. */
/* The relax lambda (:151-158): relaxations++, new_d = dist[src] + w,       */
/* curr = atomic_min(dist[dst], new_d) (:22-30), return new_d < curr.       */
/* neighbors_expand (operators.hpp:35-68) visits frontier positions in    */
/* order and each row in edge-id order; duplicates kept when !dedup.        */
/* ------------------------------------------------------------------------ */
#define DEFINE_BSP(NAME, T)                                                    \
int NAME(size_t n, const uint32_t* ro, const uint32_t* col,                   \
                     const T* w, uint32_t source, int dedup, T* dist,         \
                     uint64_t* supersteps, uint64_t* relaxations) {           \
  if (source >= n) return -1;                                                 \
  for (size_t i = 0; i < n; ++i) dist[i] = INFINITY;                          \
  dist[source] = 0;                                                           \
  size_t cap = 1024, fsz = 1, osz;                                            \
  uint32_t* f = (uint32_t*)malloc(cap * sizeof(uint32_t));                    \
  uint32_t* o = NULL;                                                         \
  uint8_t* mark = dedup ? (uint8_t*)calloc(n, 1) : NULL;                      \
  uint64_t steps = 0, relax = 0;                                              \
  f[0] = source;                                                              \
  while (fsz) { /* algorithms.hpp:167 while (f.size() != 0) */                              \
    ++steps;                                                                  \
    size_t ocap = 1024;                                                       \
    osz = 0;                                                                  \
    o = (uint32_t*)malloc(ocap * sizeof(uint32_t));                           \
    for (size_t i = 0; i < fsz; ++i) {                                        \
      uint32_t u = f[i];                                                      \
      for (uint32_t e = ro[u]; e < ro[u + 1]; ++e) {                          \
        ++relax;                                                              \
        uint32_t v = col[e];                                                  \
        T nd = dist[u] + w[e];                                                \
        T cur = dist[v];                                                      \
        if (nd < cur) dist[v] = nd;                                           \
        if (nd < cur) {                                                       \
          if (dedup) { /* dense frontier: set semantics, ascending output */  \
            mark[v] = 1;                                                      \
          } else {                                                            \
            if (osz == ocap) {                                                \
              ocap *= 2;                                                      \
              o = (uint32_t*)realloc(o, ocap * sizeof(uint32_t));             \
            }                                                                 \
            o[osz++] = v;                                                     \
          }                                                                   \
        }                                                                     \
      }                                                                       \
    }                                                                         \
    if (dedup) { /* frontier.hpp:147-165 convert: ascending bitmap order */   \
      for (uint32_t v = 0; v < n; ++v)                                        \
        if (mark[v]) {                                                        \
          mark[v] = 0;                                                        \
          if (osz == ocap) {                                                  \
            ocap *= 2;                                                        \
            o = (uint32_t*)realloc(o, ocap * sizeof(uint32_t));               \
          }                                                                   \
          o[osz++] = v;                                                       \
        }                                                                     \
    }                                                                         \
    free(f);                                                                  \
    f = o;                                                                    \
    fsz = osz;                                                                \
  }                                                                           \
  free(f);                                                                    \
  free(mark);                                                                 \
  if (supersteps) *supersteps = steps;                                        \
  if (relaxations) *relaxations = relax;                                      \
  return 0;                                                                   \
}
DEFINE_BSP(orc_sssp_bsp_f64, double)
DEFINE_BSP(orc_sssp_bsp_f32, float)

/* algorithms.hpp:77-93 detail::repair_predecessors */
#define DEFINE_REPAIR(NAME, T)                                                \
  void NAME(size_t n, const uint32_t* ro, const uint32_t* col, const T* w,    \
            uint32_t source, const T* dist, uint32_t* pred) {                 \
    for (size_t i = 0; i < n; ++i) pred[i] = ORC_NIL;                         \
    uint8_t* reached = (uint8_t*)calloc(n ? n : 1, 1);                        \
    uint32_t* q = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));          \
    size_t qs = 0;                                                            \
    reached[source] = 1;                                                      \
    q[qs++] = source;                                                         \
    for (size_t head = 0; head < qs; ++head) {                                \
      uint32_t u = q[head];                                                   \
      for (uint32_t e = ro[u]; e < ro[u + 1]; ++e) {                          \
        uint32_t v = col[e];                                                  \
        if (reached[v] || (T)(dist[u] + w[e]) != dist[v]) continue;           \
        reached[v] = 1;                                                       \
        pred[v] = u;                                                          \
        q[qs++] = v;                                                          \
      }                                                                       \
    }                                                                         \
    free(reached);                                                            \
    free(q);                                                                  \
  }
DEFINE_REPAIR(orc_repair_pred_f64, double)
DEFINE_REPAIR(orc_repair_pred_f32, float)

static int tight_edge(const uint32_t* ro, const uint32_t* col, const double* wd,
                      const float* wf, const double* dd, const float* df, int kind,
                      uint32_t u, uint32_t v) {
  /* build_csr rows are sorted by (dst, weight) (graph.hpp:144-147): binary
   * search for v, then its parallel edges; a linear scan if that misses
   * (rows of other layouts) */
  uint32_t lo = ro[u], hi = ro[u + 1];
  while (lo < hi) {
    uint32_t mid = lo + (hi - lo) / 2;
    if (col[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  for (int pass = 0; pass < 2; ++pass) {
    uint32_t e0 = pass ? ro[u] : lo, e1 = ro[u + 1];
    for (uint32_t e = e0; e < e1; ++e) {
      if (col[e] != v) {
        if (pass == 0) break;
        continue;
      }
      if (kind ? (float)(df[u] + wf[e]) == df[v] : dd[u] + wd[e] == dd[v]) return 1;
    }
  }
  return 0;
}

/* acceptance.cpp:56-91: NIL at the source and unreachable vertices; every
 * other v has an edge pred[v] -> v with dist[pred] + w == dist[v], and the
 * chain reaches the source.  Chains are walked once (memoised: a vertex is
 * marked when its chain is known to end at the source), so the check is
 * linear even on high-diameter graphs.  Returns -1, or the first bad v. */
int64_t orc_check_pred_tree(size_t n, const uint32_t* ro, const uint32_t* col,
                            const void* wv, const void* dv, int kind,
                            uint32_t source, const uint32_t* pred) {
  const double* wd = (const double*)wv;
  const float* wf = (const float*)wv;
  const double* dd = (const double*)dv;
  const float* df = (const float*)dv;
  for (uint32_t v = 0; v < n; ++v) {
    int unreach = kind ? isinf(df[v]) : isinf(dd[v]);
    if (v == source || unreach) {
      if (pred[v] != ORC_NIL) return v;
      continue;
    }
    uint32_t u = pred[v];
    if (u == ORC_NIL || u >= n) return v;
    if (!tight_edge(ro, col, wd, wf, dd, df, kind, u, v)) return v;
  }
  /* 0 = unknown, 1 = on the walk in progress, 2 = reaches the source */
  uint8_t* state = (uint8_t*)calloc(n ? n : 1, 1);
  if (source < n) state[source] = 2;
  int64_t bad = -1;
  for (uint32_t v = 0; v < n && bad < 0; ++v) {
    if (state[v] || pred[v] == ORC_NIL) continue;
    uint32_t walk = v;
    while (state[walk] == 0) {
      state[walk] = 1;
      walk = pred[walk];
      if (walk == ORC_NIL || walk >= n) break;
    }
    int ok = walk < n && state[walk] == 2;  /* else a cycle or a dead end */
    if (!ok) bad = v;
    for (uint32_t x = v; x < n && state[x] == 1; x = pred[x]) state[x] = ok ? 2 : 3;
  }
  free(state);
  return bad;
}

/* ------------------------------------------------------------------------ */
/* Synthetic generators.  Independent restatement of       */
/* paper_2212_08200_b200/csrc/rmat.cuh.                                      */
/* ------------------------------------------------------------------------ */
static uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static uint64_t rmat_key(uint64_t seed, uint64_t i, uint32_t j) {
  return splitmix64(seed * 0xD1B54A32D192ED03ULL + i * 64ULL + j);
}

void orc_rmat_edges(int scale, uint64_t m, uint64_t seed, int wkind,
                    uint64_t first, uint64_t count, uint32_t* src,
                    uint32_t* dst, uint32_t* wbits) {
  (void)m;
  /* Graph500 A/B/C/D = .57/.19/.19/.05 as 32-bit cumulative thresholds */
  const uint32_t t1 = 0x91eb851eu, t2 = 0xc28f5c28u, t3 = 0xf3333333u;
  for (uint64_t k = 0; k < count; ++k) {
    uint64_t i = first + k;
    uint32_t s = 0, d = 0;
    uint64_t word = 0;
    for (int l = 0; l < scale; ++l) {
      if ((l & 1) == 0) word = rmat_key(seed, i, (uint32_t)(l >> 1));
      uint32_t r = (l & 1) ? (uint32_t)(word >> 32) : (uint32_t)word;
      uint32_t sb = r >= t2;                  /* quadrants (1,0),(1,1) */
      uint32_t db = (r >= t1 && r < t2) || r >= t3;
      s = (s << 1) | sb;
      d = (d << 1) | db;
    }
    uint64_t wk = rmat_key(seed, i, 31);
    src[k] = s;
    dst[k] = d;
    if (wkind == 0) {
      wbits[k] = (uint32_t)(wk >> 56); /* U{0..255} */
    } else {
      float f = (float)(wk >> 40) * (1.0f / 16777216.0f);
      memcpy(&wbits[k], &f, 4);
    }
  }
}

/* The RMAT graph in build_csr's layout (graph.hpp:132-162: rows ascending
 * by src, each row sorted by (dst, weight), parallel edges kept), built on the
 * host for the CPU baseline at full size: edges generated in parallel, a
 * counting sort by source, then each row sorted.  Equal to sorting the whole
 * edge list by (src, dst, w) -- the reference's own std::sort -- because the
 * row order and the in-row order are both total.  threads <= 0: all cores. */
static int edge_dw_cmp(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y;
}

uint64_t orc_rmat_csr(int scale, int edgefactor, uint64_t seed, int wkind, int threads,
                      uint32_t* ro, uint32_t* col, uint32_t* wbits) {
  const uint64_t n = 1ull << scale, m = (uint64_t)edgefactor << scale;
  if (threads > 0) omp_set_num_threads(threads);
  uint32_t* s = (uint32_t*)malloc(m * 4);
  uint64_t* dw = (uint64_t*)malloc(m * 8); /* (dst << 32 | weight bits): in-row key */
  const uint64_t chunk = 1u << 14;
#pragma omp parallel for schedule(dynamic, 1)
  for (uint64_t c = 0; c < (m + chunk - 1) / chunk; ++c) {
    const uint64_t first = c * chunk, cnt = first + chunk > m ? m - first : chunk;
    uint32_t d[1u << 14], w[1u << 14];
    orc_rmat_edges(scale, m, seed, wkind, first, cnt, s + first, d, w);
    for (uint64_t k = 0; k < cnt; ++k) dw[first + k] = ((uint64_t)d[k] << 32) | w[k];
  }
  memset(ro, 0, (n + 1) * 4);
  for (uint64_t i = 0; i < m; ++i) ++ro[s[i] + 1];
  for (uint64_t v = 0; v < n; ++v) ro[v + 1] += ro[v];
  uint64_t* sorted = (uint64_t*)malloc(m * 8);
  uint32_t* cur = (uint32_t*)malloc(n * 4);
  memcpy(cur, ro, n * 4);
  for (uint64_t i = 0; i < m; ++i) sorted[cur[s[i]]++] = dw[i]; /* stable scatter by source */
  free(cur);
  free(dw);
  free(s);
  /* f32 weights are non-negative: their bits order like the values; u32 the same */
#pragma omp parallel for schedule(dynamic, 4096)
  for (uint64_t v = 0; v < n; ++v)
    qsort(sorted + ro[v], ro[v + 1] - ro[v], 8, edge_dw_cmp);
#pragma omp parallel for schedule(static)
  for (uint64_t i = 0; i < m; ++i) {
    col[i] = (uint32_t)(sorted[i] >> 32);
    wbits[i] = (uint32_t)sorted[i];
  }
  free(sorted);
  return m;
}

uint64_t orc_grid_csr(uint32_t side, uint64_t seed, uint32_t* ro,
                      uint32_t* col, uint32_t* wbits) {
  uint64_t n = (uint64_t)side * side, e = 0;
  for (uint64_t u = 0; u < n; ++u) {
    uint32_t r = (uint32_t)(u / side), c = (uint32_t)(u % side);
    if (ro) ro[u] = (uint32_t)e;
    /* ascending dst: up, left, right, down; direction code 0..3 */
    uint64_t nb[4];
    int ok[4] = {r > 0, c > 0, c + 1 < side, r + 1 < side};
    nb[0] = u - side;
    nb[1] = u - 1;
    nb[2] = u + 1;
    nb[3] = u + side;
    for (int k = 0; k < 4; ++k) {
      if (!ok[k]) continue;
      if (col) {
        col[e] = (uint32_t)nb[k];
        uint64_t h = splitmix64(seed * 0xD1B54A32D192ED03ULL + u * 4ULL + k);
        float f = (float)(h >> 40) * (1.0f / 16777216.0f);
        memcpy(&wbits[e], &f, 4);
      }
      ++e;
    }
  }
  if (ro) ro[n] = (uint32_t)e;
  return e;
}

/* algorithms.hpp:194-239 bfs(): the frontier of level L is expanded once per
 * superstep (:222-236); every out-edge of a frontier vertex evaluates the
 * claim once (:212-213 relaxations), and an unclaimed destination takes
 * level L + 1 (:214-217, first claimant wins; all claimants of one level
 * write the same value).  The loop runs while the frontier is non-empty
 * (:222), so supersteps = number of non-empty levels. */
int orc_bfs(size_t n, const uint32_t* ro, const uint32_t* col, uint32_t source, double* depth,
            uint64_t* supersteps, uint64_t* relaxations) {
  if (source >= n) return -1;
  uint32_t* cur = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
  uint32_t* nxt = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
  for (size_t i = 0; i < n; ++i) depth[i] = INFINITY;
  depth[source] = 0.0;
  size_t k = 0, level = 0;
  uint64_t steps = 0, rel = 0;
  cur[k++] = source;
  while (k != 0) {
    ++steps;
    size_t kn = 0;
    for (size_t i = 0; i < k; ++i) {
      const uint32_t u = cur[i];
      for (uint32_t e = ro[u]; e < ro[u + 1]; ++e) {
        ++rel;
        const uint32_t v = col[e];
        if (isinf(depth[v])) {
          depth[v] = (double)(level + 1);
          nxt[kn++] = v;
        }
      }
    }
    uint32_t* t = cur;
    cur = nxt;
    nxt = t;
    k = kn;
    ++level;
  }
  free(cur);
  free(nxt);
  *supersteps = steps;
  *relaxations = rel;
  return 0;
}


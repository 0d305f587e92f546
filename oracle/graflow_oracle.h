/*
 * graflow_oracle.h -- CPU restatement of the reference SSSP path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing under oracle/ is part of the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it, and only as the checker or the timed
 * CPU baseline.  The product library (paper_2212_08200_b200/lib/libgfb.so)
 * never links or calls it.
 *
 * Every function restates one piece of the reference (graflow, arXiv
 * 2212.08200) and cites the file:line it follows.  Paths are relative to the
 * reference tree's proj/ directory.
 *
 * Parity pinning: tests/test_oracle.py checks this restatement against the
 * golden vectors in tests/golden/, which tests/golden/make_golden.py produced
 * by running the UNMODIFIED reference headers (compiled into
 * oracle/_ref/libgraflow_ref.so by oracle/Makefile).
 */
#ifndef GRAFLOW_ORACLE_H
#define GRAFLOW_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_NIL 0xFFFFFFFFu /* types.hpp:13 no_predecessor */

/* ---- std::mt19937_64 + libstdc++ generate_canonical<double,53> ---------- */
typedef struct {
  uint64_t mt[312];
  int idx;
} orc_mt64;

void orc_mt64_seed(orc_mt64* r, uint64_t seed);
uint64_t orc_mt64_next(orc_mt64* r);
double orc_canonical(orc_mt64* r);

/* random_graphs.hpp:15-30 testutil::random_edges(n, seed).  Returns the edge
 * count; writes at most `cap` edges (pass cap=0 to only count). */
size_t orc_random_edges(size_t n, uint64_t seed, uint32_t* src, uint32_t* dst,
                        double* w, size_t cap);

/* graph.hpp:132-162 build_csr: validate, sort by (src,dst,w), count+scan.
 * Returns -1 on success, else the index of the first invalid edge
 * (graph.hpp:134-142 throws invalid_argument naming that index). */
int64_t orc_build_csr(size_t n, size_t m, const uint32_t* src,
                      const uint32_t* dst, const double* w, uint32_t* ro,
                      uint32_t* col, double* val);

/* graph.hpp:166-193 build_transpose: counting sort by dst, slots in ascending
 * (src, CSR edge id) order, back-map to the CSR edge id. */
void orc_build_transpose(size_t n, size_t m, const uint32_t* ro,
                         const uint32_t* col, const double* val,
                         uint32_t* cso, uint32_t* csrc, double* cval,
                         uint32_t* ceid);

/* algorithms.hpp:101-128 reference_dijkstra (binary heap, lazy deletion,
 * strict `<` relaxation) in three arithmetics:
 *   f64: the reference's own arithmetic (weight_t = double, types.hpp:10);
 *   f32: the same algorithm with float keys, nd = d + (float)w;
 *   u32: integer weights, sums in uint64 (exact; equals the f64 result). */
int orc_dijkstra_f64(size_t n, const uint32_t* ro, const uint32_t* col,
                     const double* w, uint32_t source, double* dist,
                     uint32_t* pred);
int orc_dijkstra_f32(size_t n, const uint32_t* ro, const uint32_t* col,
                     const float* w, uint32_t source, float* dist,
                     uint32_t* pred);
int orc_dijkstra_u32(size_t n, const uint32_t* ro, const uint32_t* col,
                     const uint32_t* w, uint32_t source, uint64_t* dist,
                     uint32_t* pred);

/* algorithms.hpp:134-188 sssp(), sequential push over a frontier, in f32.
 * dedup=0 keeps duplicates (FrontierRepr::sparse, frontier.hpp:78-80);
 * dedup=1 is set semantics (FrontierRepr::dense, frontier.hpp:81-88).
 * relaxations counts every cond invocation (algorithms.hpp:152). */
int orc_sssp_bsp_f64(size_t n, const uint32_t* ro, const uint32_t* col,
                     const double* w, uint32_t source, int dedup, double* dist,
                     uint64_t* supersteps, uint64_t* relaxations);
int orc_sssp_bsp_f32(size_t n, const uint32_t* ro, const uint32_t* col,
                     const float* w, uint32_t source, int dedup, float* dist,
                     uint64_t* supersteps, uint64_t* relaxations);

/* algorithms.hpp:77-93 detail::repair_predecessors: BFS from the source
 * over tight edges, first assignment wins.  f64 and f32 arithmetic. */
void orc_repair_pred_f64(size_t n, const uint32_t* ro, const uint32_t* col,
                         const double* w, uint32_t source, const double* dist,
                         uint32_t* pred);
void orc_repair_pred_f32(size_t n, const uint32_t* ro, const uint32_t* col,
                         const float* w, uint32_t source, const float* dist,
                         uint32_t* pred);

/* test_algorithms.cpp:66-92 / acceptance.cpp:56-91 predecessor-tree check:
 * NIL at the source and at unreachable vertices, a tight edge pred->v
 * (dist[pred] + w == dist[v] in the given arithmetic), and a chain reaching
 * the source within n steps.  Returns -1 when valid, else the first bad
 * vertex.  Weights/dists are passed as f64 (kind=0) or f32 (kind=1). */
int64_t orc_check_pred_tree(size_t n, const uint32_t* ro, const uint32_t* col,
                            const void* w, const void* dist, int kind,
                            uint32_t source, const uint32_t* pred);

/* ---- synthetic inputs (not in the reference) ------------
 * Counter-based RMAT: edge i is a pure function of (seed, i), so CPU and GPU
 * produce identical edge lists.  This restates paper_2212_08200_b200/csrc/
 * rmat.cuh independently; tests assert the two agree.
 * wkind: 0 = u32 U{0..255}, 1 = f32 U[0,1) on a 2^-24 grid. */
/* algorithms.hpp:194-239 bfs(): level-synchronous push with the claim
 * condition; depth as double (+inf unreachable), supersteps = expanded
 * levels, relaxations = claim evaluations.  Returns -1 if source >= n. */
int orc_bfs(size_t n, const uint32_t* ro, const uint32_t* col, uint32_t source, double* depth,
            uint64_t* supersteps, uint64_t* relaxations);

/* build_csr layout of the RMAT graph, host-parallel (CPU-baseline input) */
uint64_t orc_rmat_csr(int scale, int edgefactor, uint64_t seed, int wkind, int threads,
                      uint32_t* ro, uint32_t* col, uint32_t* wbits);
void orc_rmat_edges(int scale, uint64_t m, uint64_t seed, int wkind,
                    uint64_t first, uint64_t count, uint32_t* src,
                    uint32_t* dst, uint32_t* wbits);

/* 4-neighbour side x side grid, both directions, independent f32 weights;
 * CSR emitted directly in build_csr order (ascending dst per row). */
uint64_t orc_grid_csr(uint32_t side, uint64_t seed, uint32_t* ro,
                      uint32_t* col, uint32_t* wbits);

#ifdef __cplusplus
}
#endif
#endif

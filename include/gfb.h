/*
 * gfb.h -- C ABI of the B200-native SSSP hot path ("graflow-b200").
 *
 * This is the drop-in boundary for the reference's BSP single-source shortest
 * path (graflow, arXiv 2212.08200; paths below are relative to the
 * reference's proj/ directory).  The reference is header-only C++20; its
 * device execution policy (include/graflow_b200/device.hpp in this repo) is
 * the binding a graflow maintainer adds, and it calls exactly these entry
 * points.  Plain pointers and sizes only; no exceptions cross the ABI.
 *
 * Conventions
 *  - Every function returns a gfb_status.  On failure gfb_last_error() holds
 *    a thread-local message.  The C++ shim maps GFB_EINVAL ->
 *    std::invalid_argument, GFB_ERANGE -> std::out_of_range, GFB_ELOGIC ->
 *    std::logic_error, everything else -> std::runtime_error, mirroring the
 *    reference's throw sites (cited per function).
 *  - Host arrays are caller-owned and only read/written during the call.
 *    Device memory is owned by the opaque handles and released by the
 *    matching _free/_destroy.
 *  - Calls are synchronous at operator granularity: no device work of a call
 *    is still running when it returns (the reference's barrier contract,
 *    operators.hpp:28-34; test_operators.cpp:104-117).
 *  - One gfb_ctx per host thread (it owns one CUDA stream).
 */
#ifndef GFB_H
#define GFB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GFB_NIL 0xFFFFFFFFu /* types.hpp:13 no_predecessor */

typedef enum gfb_status {
  GFB_OK = 0,
  GFB_EINVAL = 1, /* std::invalid_argument */
  GFB_ERANGE = 2, /* std::out_of_range */
  GFB_ELOGIC = 3, /* std::logic_error */
  GFB_ECUDA = 4,  /* std::runtime_error (CUDA) */
  GFB_ENOMEM = 5, /* std::runtime_error (device memory) */
  GFB_ENCCL = 6,  /* std::runtime_error (NCCL) */
  GFB_EPARSE = 7  /* graflow::ParseError (io.hpp:27-36): "line N: ...";
                     the line via gfb_last_error_line() */
} gfb_status;

/* Edge-weight / distance arithmetic.  The reference computes in double
 * (types.hpp:10 weight_t = double).  GFB_W_F64 reproduces it bit for bit;
 * GFB_W_U32 is exact for integer weights (dist widened to double on read);
 * GFB_W_F32 is the bandwidth mode (fp32 fixpoint). */
typedef enum gfb_wtype { GFB_W_U32 = 0, GFB_W_F32 = 1, GFB_W_F64 = 2 } gfb_wtype;

/* algorithms.hpp:32 Direction, plus AUTO (device push<->pull switch). */
typedef enum gfb_direction {
  GFB_DIR_PUSH = 0,
  GFB_DIR_PULL = 1,
  GFB_DIR_AUTO = 2
} gfb_direction;

/* frontier.hpp:18 FrontierRepr (queue is the async model: out of scope). */
typedef enum gfb_repr { GFB_SPARSE = 0, GFB_DENSE = 1 } gfb_repr;

/* Operator conditions.  Host C++ lambdas cannot cross a C ABI, so the device
 * policy accepts these recognised conditions (include/graflow_b200/ops.hpp):
 *   RELAX_MIN -- the SSSP relax lambda, algorithms.hpp:151-158;
 *   RECORD    -- record every (src,dst,edge) invocation, return false
 *                (test_operators.cpp:151-171 eligibility recorder);
 *   ALWAYS    -- return true (test_operators.cpp:27 `always`). */
typedef enum gfb_op { GFB_OP_RELAX_MIN = 0, GFB_OP_RECORD = 1, GFB_OP_ALWAYS = 2 } gfb_op;

typedef struct gfb_ctx gfb_ctx;
typedef struct gfb_graph gfb_graph;
typedef struct gfb_frontier gfb_frontier;
typedef struct gfb_dist gfb_dist;     /* device distance map + relax counter */
typedef struct gfb_record gfb_record; /* device (src,dst,edge) recorder */

/* ---- errors / version -------------------------------------------------- */
int gfb_version(void);
const char* gfb_last_error(void);

/* ---- context (one CUDA stream on one device) ---------------------------- */
int gfb_ctx_create(int device, gfb_ctx** out);
int gfb_ctx_destroy(gfb_ctx* ctx);
int gfb_ctx_num_sms(gfb_ctx* ctx, int* out);

/* ---- graph store (graph.hpp:45-127 Graph) --------------------------------
 * gfb_graph_upload takes the reference Graph's CSR arrays as they are
 * (row_offsets(), column_indices(), values(): graph.hpp:76-78; values are
 * `double` in the reference, or u32/f32 for the typed modes) and builds the
 * device CSR (interleaved {dst, weight} records) and, when build_csc != 0,
 * the CSC view of build_transpose (graph.hpp:166-193; slot order ascending
 * (src, CSR edge id), with the edge-id back-map).  `wtype` is the device
 * arithmetic; `w_host_type` the element type of `w` (GFB_W_F64 when passing
 * the reference's values() directly).
 * Validation mirrors build_csr (graph.hpp:134-142): a dst >= n, a negative or
 * non-finite weight, or an inconsistent row_offsets array -> GFB_EINVAL
 * naming the first offending edge.  -0.0 weights are canonicalised to +0.0. */
int gfb_graph_upload(gfb_ctx* ctx, uint64_t n, uint64_t m,
                     const uint32_t* row_offsets, const uint32_t* col,
                     const void* w, int w_host_type, int wtype, int build_csc,
                     gfb_graph** out);
/* Re-copy new CSR contents of the same shape into an existing graph. */
int gfb_graph_refill(gfb_graph* g, const uint32_t* row_offsets,
                     const uint32_t* col, const void* w, int w_host_type);
int gfb_graph_free(gfb_graph* g);
int gfb_graph_info(const gfb_graph* g, uint64_t* n, uint64_t* m, int* wtype,
                   int* has_csc);
/* Copy the device CSR back (w in the graph's wtype; any pointer may be 0). */
int gfb_graph_download(gfb_graph* g, uint32_t* row_offsets, uint32_t* col,
                       void* w);
/* Device-side synthetic graphs: counter-based RMAT
 * (A/B/C/D = .57/.19/.19/.05, unpermuted, duplicates and self-loops kept;
 * wtype U32 -> U{0..255}, F32 -> U[0,1) on a 2^-24 grid) and the 4-neighbour
 * grid.  Built on the device in build_csr's layout (graph.hpp:144-161). */
int gfb_graph_generate_rmat(gfb_ctx* ctx, int scale, int edgefactor,
                            uint64_t seed, int wtype, int build_csc,
                            gfb_graph** out);
int gfb_graph_generate_grid(gfb_ctx* ctx, uint32_t side, uint64_t seed,
                            int build_csc, gfb_graph** out);

/* ---- Matrix Market ingest (io.hpp:17-123) --------------------------------
 * gfb_mm_parse: parse_matrix_market on a text buffer, the reference's
 * acceptance rules and error lines (GFB_EPARSE; MatrixMarketOptions
 * force_unit_weights / expand_symmetric, io.hpp:22-25) into a host edge list
 * (EdgeList, io.hpp:17-20: 0-based ids, weights as double, file order).
 * gfb_graph_from_edges: build_csr (graph.hpp:132-162) on the device from a
 * host edge list: validation naming the first bad edge (GFB_EINVAL), rows
 * sorted by (dst, weight), parallel edges kept. */
typedef struct gfb_edge_list gfb_edge_list;
int gfb_mm_parse(const char* text, size_t len, int force_unit_weights, int expand_symmetric,
                 gfb_edge_list** out);
int gfb_edge_list_info(const gfb_edge_list* e, uint64_t* num_vertices, uint64_t* num_edges);
int gfb_edge_list_read(const gfb_edge_list* e, uint32_t* src, uint32_t* dst, double* w);
int gfb_edge_list_free(gfb_edge_list* e);
uint64_t gfb_last_error_line(void);
int gfb_graph_from_edges(gfb_ctx* ctx, uint64_t n, uint64_t m, const uint32_t* src,
                         const uint32_t* dst, const double* w, int wtype, int build_csc,
                         gfb_graph** out);
int gfb_graph_from_edge_list(gfb_ctx* ctx, const gfb_edge_list* e, int wtype, int build_csc,
                             gfb_graph** out);

/* ---- frontier (frontier.hpp:37-218 Frontier, sparse + dense) ------------ */
int gfb_frontier_create(gfb_ctx* ctx, uint64_t n, int repr, gfb_frontier** out);
int gfb_frontier_free(gfb_frontier* f);
/* add_vertex semantics (frontier.hpp:73-96): sparse keeps duplicates and
 * order, dense is a set.  Vertex >= n -> GFB_ERANGE. */
int gfb_frontier_assign(gfb_frontier* f, const uint32_t* vertices, uint64_t k);
/* size() (frontier.hpp:57-67): sparse counts duplicates, dense set bits. */
int gfb_frontier_size(gfb_frontier* f, uint64_t* size);
/* Contents: sparse in insertion order (device order for device-produced
 * frontiers), dense ascending (get_active_vertex, frontier.hpp:100-122). */
int gfb_frontier_read(gfb_frontier* f, uint32_t* out, uint64_t cap, uint64_t* k);
int gfb_frontier_repr(gfb_frontier* f, int* repr);

/* ---- operator state ------------------------------------------------------ */
int gfb_dist_create(gfb_ctx* ctx, const gfb_graph* g, gfb_dist** out);
int gfb_dist_free(gfb_dist* d);
/* dist = +inf everywhere, dist[source] = 0 (algorithms.hpp:144-148). */
int gfb_dist_init(gfb_dist* d, uint32_t source);
/* Widened to double (exact for every wtype); relaxations may be 0. */
int gfb_dist_read(gfb_dist* d, double* dist, uint64_t* relaxations);
int gfb_record_create(gfb_ctx* ctx, uint64_t capacity, gfb_record** out);
int gfb_record_free(gfb_record* r);
int gfb_record_read(gfb_record* r, uint32_t* src, uint32_t* dst, uint32_t* edge,
                    uint64_t cap, uint64_t* count);

/* ---- operators (operators.hpp) -------------------------------------------
 * Push advance, operators.hpp:35-68 neighbors_expand: for every frontier
 * element (duplicates included) and every out-edge, cond exactly once; the
 * output has one entry per true cond (sparse) or is a set (dense); output
 * representation = input representation.  `state` is a gfb_dist* for
 * RELAX_MIN, a gfb_record* for RECORD, unused for ALWAYS. */
int gfb_advance_push(gfb_ctx* ctx, const gfb_graph* g, gfb_frontier* in,
                     gfb_frontier* out, int op, void* state);
/* Pull advance, operators.hpp:76-114 neighbors_expand_pull: input must be
 * dense (else GFB_EINVAL, :81-82), graph must have the CSC (else
 * GFB_EINVAL, :79-80); cond runs for every eligible in-edge; output dense. */
int gfb_advance_pull(gfb_ctx* ctx, const gfb_graph* g, gfb_frontier* in,
                     gfb_frontier* out, int op, void* state);
/* uniquify, operators.hpp:191-200: sparse in (else GFB_EINVAL), ascending
 * duplicate-free sparse out.  Bitmap dedup + warp-ballot compaction. */
int gfb_filter_unique(gfb_ctx* ctx, gfb_frontier* in, gfb_frontier* out);

/* filter, operators.hpp:163-188: out = the elements of `in` whose predicate
 * holds, same representation (else GFB_EINVAL); sparse keeps the input order
 * and duplicates (the reference's sequential order).  Host predicates cannot
 * cross the ABI; the recognised ones read a device distance map (gfb_dist)
 * and compare in double (exact for every arithmetic):
 *   DIST_BELOW     dist[v] <  threshold   (the near side of a near-far split)
 *   DIST_AT_LEAST  dist[v] >= threshold   (the far side)
 *   REACHED        dist[v] <  +inf        (threshold unused) */
typedef enum gfb_pred {
  GFB_PRED_DIST_BELOW = 0,
  GFB_PRED_DIST_AT_LEAST = 1,
  GFB_PRED_REACHED = 2
} gfb_pred;
int gfb_filter(gfb_ctx* ctx, gfb_frontier* in, gfb_frontier* out, int pred,
               const gfb_dist* dist, double threshold);

/* ---- the entry point: sssp() (algorithms.hpp:134-188) -------------------- */
typedef struct gfb_sssp_opts {
  uint32_t struct_size;  /* sizeof(gfb_sssp_opts) */
  int32_t direction;     /* gfb_direction; PUSH default (algorithms.hpp:40) */
  float pull_alpha;      /* AUTO: pull when frontier edges > m / pull_alpha
                            (default 1.05, the measured break-even; a plan
                            holds each vertex once, so alpha <= 1 never
                            pulls) */
  int32_t device_loop;   /* 1: device-side convergence (CUDA graph) */
  double delta;          /* >0: near-far filter of this width (push only; one
                            persistent launch with queue frontiers, for
                            high-diameter graphs); +inf: the async queue model
                            (no far set); 0: the device chooses -- near-far
                            with delta = 32 x mean weight on low-degree meshes
                            (max out-degree <= 8, n >= 2^16), else the BSP
                            loop.  Any arithmetic.  Same distances. */
  int32_t compute_pred;  /* 1: fill pred (tight-edge tree) */
  /* Tuning (0 = the measured default everywhere; none changes the result):  */
  int32_t loop;          /* GFB_LOOP_AUTO | GFB_LOOP_BSP (never pick the
                            near-far loop automatically) */
  int32_t relabel;       /* GFB_RELABEL_AUTO (in-degree relabelled CSR for
                            skewed graphs, from the 2nd call on the same
                            contents) | GFB_RELABEL_ON | GFB_RELABEL_OFF */
  int32_t defer_pct;     /* BSP far-bucket deferral: in a superstep whose
                            frontier holds >= m/4 edges only the closest
                            distance buckets up to this % of those edges are
                            expanded.  0 = default (5; 10 on the partitioned
                            path), 100 = off */
  int32_t advance_tile;  /* push advance edge tile for 4-byte distances:
                            0 = by size (128 for m <= 2^27, else 256), or
                            128 / 256 */
  int32_t trace;         /* 1: per-superstep lines on stderr (host loop) */
  int32_t tail_edges;    /* BSP loop, push: a plan below this
                            many edges with nothing deferred hands the rest of
                            the run to one persistent tail launch (vertex
                            queues, no per-superstep bitmap filter).  0 = by
                            size (m / 256, at least 4096), -1 = never */
  int32_t reserved[1];
} gfb_sssp_opts;

#define GFB_LOOP_AUTO 0
#define GFB_LOOP_BSP 1
#define GFB_RELABEL_AUTO 0
#define GFB_RELABEL_ON 1
#define GFB_RELABEL_OFF 2

void gfb_sssp_opts_default(gfb_sssp_opts* o);

typedef struct gfb_sssp_stats {
  uint64_t supersteps;    /* SsspResult::supersteps, algorithms.hpp:59 */
  uint64_t relaxations;   /* SsspResult::relaxations, algorithms.hpp:60 */
  uint64_t n_reach;       /* vertices with finite dist */
  uint64_t m_reach;       /* sum of out-degrees of reached vertices */
  uint64_t push_steps, pull_steps;
  uint64_t pred_fallback; /* vertices whose pred needed the repair pass */
  double device_ms;       /* CUDA-event time: init .. last superstep + pred */
  double advance_ms;      /* CUDA-event time of the advance launches (sum;
                             host-loop mode only, 0 under the device loop) */
  uint64_t advance_launches;
  uint64_t kernel_launches; /* libgfb kernels launched by this call */
} gfb_sssp_stats;

/* Runs init, the BSP loop and the predecessor pass on the device.  dist is
 * written widened to double (n entries), pred as u32 with GFB_NIL for the
 * source and unreachable vertices; either may be NULL to leave the result on
 * the device (gfb_sssp_read fetches it later).  source >= n -> GFB_ERANGE
 * (algorithms.hpp:137); PULL without CSC -> GFB_EINVAL (:138-139). */
int gfb_sssp(gfb_ctx* ctx, gfb_graph* g, uint32_t source,
             const gfb_sssp_opts* opts, double* dist, uint32_t* pred,
             gfb_sssp_stats* stats);
/* Result of the last gfb_sssp on g: dist widened to double and/or in the
 * graph's native type (u32 / f32 / f64 bytes). */
int gfb_sssp_read(gfb_graph* g, double* dist, void* dist_native, uint32_t* pred);

/* ---- inspection (tests / tools; no reference counterpart) ----------------
 * The in-degree-relabelled CSR the BSP loop runs on for skewed graphs (the
 * loop also uses it for f64; this view serves 4-byte weights only; built on
 * first use, cached until a refill): row offsets (n+1), records as
 * {dst, weight bits} u32 pairs (2m), perm old->new id (n).  Any pointer may
 * be 0.  4-byte weights only (else GFB_EINVAL). */
int gfb_debug_relabel(gfb_graph* g, uint32_t* row_offsets, uint32_t* adj_pairs,
                      uint32_t* perm);

/* Range-preserving relabelled copy of g for the 1-D partitioned paths
 * (gfb_peer_* / gfb_mg_*; the reference partitions by contiguous vertex
 * ranges): inside each [range_starts[q], range_starts[q+1])
 * vertices are ranked by descending in-degree (the hot destinations of one
 * owner share cache lines, as in the single-GPU loop's relabelled CSR) and
 * every row is sorted by destination; no vertex changes owner, so the same
 * range_starts partition the result with the same per-owner edge counts.
 * Writes row_offsets (n+1), col (m, new ids), weights (m, g's native type:
 * u32 / f32 / f64) and perm (n, old id -> new id); any pointer may be 0.
 * range_starts: nparts + 1 entries from 0 to n, non-decreasing (else
 * GFB_EINVAL).  Distances of the relabelled graph map back as
 * dist_old[v] = dist_new[perm[v]]. */
int gfb_graph_relabel_ranges(gfb_graph* g, uint32_t nparts, const uint32_t* range_starts,
                             uint32_t* row_offsets, uint32_t* col, void* weights,
                             uint32_t* perm);

/* Breadth-first search as operator reuse (algorithms.hpp:194-239 bfs()):
 * depth[n] as double (math.inf for unreachable, like BfsResult.depth),
 * supersteps = levels expanded (max depth + 1), relaxations = claim
 * evaluations (the out-degree sum of the reached vertices, the same for push
 * and pull).  direction: gfb_direction; pull needs a transpose (build_csc)
 * like the reference, and is executed as push (identical results).
 * GFB_ERANGE: source >= n. */
int gfb_bfs(gfb_ctx* ctx, gfb_graph* g, uint32_t source, int direction, double* depth,
            uint64_t* supersteps, uint64_t* relaxations);

/* ---- 1-D partitioned SSSP: one rank's share (multi-GPU) ----
 * No reference counterpart (the reference is single-host); mg.py drives one
 * gfb_part per rank and exchanges the messages with torch.distributed
 * (NCCL over NVLink/NVSwitch).  The rank holds CSR rows [lo, hi) of the
 * global graph (ro_local rebased to 0, hi-lo+1 entries; column ids global
 * < n_global).  Messages are 16-byte {dst_global, src_global, dist_bits, 0}
 * records in device memory, ascending dst (= grouped by owner).  f32 / u32
 * arithmetic only. */
typedef struct gfb_part gfb_part;
int gfb_part_create(gfb_ctx* ctx, uint64_t n_global, uint32_t lo, uint32_t hi,
                    uint64_t m_local, const uint32_t* ro_local, const uint32_t* col,
                    const void* w, int w_host_type, int wtype, gfb_part** out);
int gfb_part_free(gfb_part* p);
/* dist = +inf, dist[source] = 0 if the source is local; frontier = {source} */
int gfb_part_init(gfb_part* p, uint32_t source);
/* One superstep: expand the local frontier (relax local destinations in
 * place, min-combine remote candidates), write the remote messages to
 * out_dev (capacity out_cap messages), per-owner counts[nparts] (host) and
 * the message total.  range_starts: host array of nparts+1 vertex ids. */
int gfb_part_advance(gfb_part* p, void* out_dev, uint64_t out_cap,
                     const uint32_t* range_starts, int nparts, uint32_t* counts,
                     uint64_t* total);
/* Apply received messages (device memory): atomicMin + activate. */
int gfb_part_apply(gfb_part* p, const void* in_dev, uint64_t count);
/* Size of the local next frontier (the allreduce operand for convergence). */
int gfb_part_pending(gfb_part* p, uint64_t* size);
int gfb_part_read(gfb_part* p, void* dist_native, uint64_t* relaxations,
                  uint64_t* supersteps);
/* Predecessor candidates from the local edges given the global distance
 * array (device, n_global, native type): round 1 strict tight edges, round
 * r > 1 equal-distance tight edges from sources with 1 <= res[u] <= r;
 * cand[v] = min candidate source (device atomicMin). */
int gfb_part_pred(gfb_part* p, const void* gdist_dev, const uint32_t* res_dev,
                  uint32_t* cand_dev, uint32_t round);

/* ---- 1-D partitioned SSSP over peer memory (multi-GPU) --
 * No reference counterpart (the reference is single-host); replaces the
 * per-superstep host exchange of the gfb_part_* path with a device-initiated
 * one.  One gfb_peer per rank (one process per GPU); rank r holds CSR rows
 * [range_starts[r], range_starts[r+1]) with GLOBAL column ids (ro_local
 * rebased to 0).  range_starts: nparts+1 ascending vertex ids, 0 first,
 * interior cuts multiples of 32; nparts <= 8.  The loop state lives in one
 * device allocation per rank, exported as a GFB_PEER_HANDLE_BYTES CUDA IPC
 * handle; after every rank has called gfb_peer_link with all nparts handles
 * (rank order; its own entry is ignored), gfb_peer_sssp relaxes remote
 * destinations directly in their owner's memory (NVLink peer access) and
 * synchronises the ranks with device-side barriers: every rank must call it
 * with the same source and options.  Distances / predecessors come back per
 * rank for its own range (predecessors as global ids); stats are this
 * rank's share (relaxations, n_reach, m_reach sum over ranks; supersteps are
 * equal).  f32 / u32 weights, push only, no near-far (delta must be 0).  A
 * rank that does not arrive at a barrier within GFB_PEER_TIMEOUT_S seconds
 * (default 30) makes every waiting rank fail with GFB_ECUDA. */
#define GFB_PEER_HANDLE_BYTES 64
typedef struct gfb_peer gfb_peer;
int gfb_peer_create(gfb_ctx* ctx, int rank, int nparts, const uint32_t* range_starts,
                    uint64_t m_local, const uint32_t* ro_local, const uint32_t* col,
                    const void* w, int w_host_type, int wtype, gfb_peer** out);
int gfb_peer_export(gfb_peer* p, void* handle /* GFB_PEER_HANDLE_BYTES */);
int gfb_peer_link(gfb_peer* p, const void* handles /* nparts x GFB_PEER_HANDLE_BYTES */);
int gfb_peer_sssp(gfb_peer* p, uint32_t source, const gfb_sssp_opts* opts,
                  gfb_sssp_stats* stats);
/* local range: dist widened to double and/or native 4-byte bits, pred global ids */
int gfb_peer_read(gfb_peer* p, double* dist, void* dist_native, uint32_t* pred);
/* every rank must be done with all peers' calls before any frees */
int gfb_peer_free(gfb_peer* p);

/* ---- the same partitioned SSSP driven by ONE host thread (SURVEY.md §8b
 * gfb_mg_*): partition q runs on devices[q] (entries may repeat a device;
 * distinct devices need peer access, i.e. an NVLink/NVSwitch node).  Upload
 * takes the whole reference-layout CSR (row_offsets n+1, col m, weights in
 * w_host_type) and cuts edge-balanced, 32-aligned vertex ranges; gfb_mg_sssp
 * returns whole-graph dist (double, n) / pred (n) and summed statistics
 * (device_ms = max over partitions).  f32 / u32 device arithmetic. */
typedef struct gfb_mg gfb_mg;
int gfb_mg_create(int ndev, const int* devices, gfb_mg** out);
/* The same, choosing the exchange:
 *   GFB_EXCHANGE_PEER  device-initiated: remote relaxations are reductions
 *                      into the owner's memory over NVLink, device barriers
 *                      (the default, peer.cu)
 *   GFB_EXCHANGE_NCCL  host-driven, the north star's baseline: remote
 *                      candidates min-combined per destination into 16-byte
 *                      messages bucketed by owner, one NCCL group of
 *                      send/recv per superstep (all-to-all-v) and an NCCL
 *                      allreduce of the frontier sizes for convergence
 *                      (xmg.cu).  NCCL needs distinct devices; partitions
 *                      that share a device exchange by device copies (same
 *                      protocol).  device_ms is the call's wall time. */
#define GFB_EXCHANGE_PEER 0
#define GFB_EXCHANGE_NCCL 1
int gfb_mg_create_ex(int ndev, const int* devices, int exchange, gfb_mg** out);
/* 1 if the exchange runs over NCCL communicators, 0 otherwise */
int gfb_mg_uses_nccl(gfb_mg* mg, int* out);
int gfb_mg_graph_upload(gfb_mg* mg, uint64_t n, uint64_t m, const uint32_t* row_offsets,
                        const uint32_t* col, const void* w, int w_host_type, int wtype);
int gfb_mg_ranges(gfb_mg* mg, uint32_t* range_starts /* ndev + 1 */);
int gfb_mg_sssp(gfb_mg* mg, uint32_t source, const gfb_sssp_opts* opts, double* dist,
                uint32_t* pred, gfb_sssp_stats* stats);
int gfb_mg_destroy(gfb_mg* mg);

#ifdef __cplusplus
}
#endif
#endif /* GFB_H */

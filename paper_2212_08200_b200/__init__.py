"""graflow-b200: the B200-native SSSP hot path of graflow (arXiv 2212.08200).

Python host mirror of the reference's binding (proj/python/module.cpp:61-151,
``graflow._core``): ``build_csr``, ``build_transpose``, ``Graph`` queries,
``sssp`` returning ``(dist, pred, supersteps, relaxations)`` and the operator
level (``Frontier``, ``neighbors_expand``, ``neighbors_expand_pull``,
``uniquify``).  Everything below runs through ``lib/libgfb.so`` (the C ABI in
include/gfb.h); the only policy is ``"device"`` -- there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _lib
from ._lib import (DENSE, DIR_AUTO, DIR_PULL, DIR_PUSH, NIL, OP_ALWAYS, OP_RECORD,
                   OP_RELAX_MIN, SPARSE, W_F32, W_F64, W_U32, GfbError, ParseError, SsspOpts,
                   SsspStats, check)

__all__ = ["Context", "Graph", "Frontier", "build_csr", "build_transpose", "rmat", "grid",
           "sssp", "sssp_stats", "neighbors_expand", "neighbors_expand_pull", "uniquify", "filter",
           "DistanceMap", "Recorder", "NIL", "GfbError", "ParseError", "EdgeList",
           "parse_matrix_market", "read_matrix_market", "graph_from_edges", "write_distances"]

_WT = {"u32": W_U32, "f32": W_F32, "f64": W_F64}
_WT_NP = {W_U32: np.uint32, W_F32: np.float32, W_F64: np.float64}
_DIR = {"push": DIR_PUSH, "pull": DIR_PULL, "auto": DIR_AUTO}
_REPR = {"sparse": SPARSE, "dense": DENSE}


def _ptr(a):
    return C.c_void_p(a.ctypes.data) if a is not None and a.size else None


class Context:
    """One CUDA stream on one device (gfb_ctx)."""

    _default = {}

    def __init__(self, device=0):
        lib = _lib.load()
        h = C.c_void_p()
        check(lib.gfb_ctx_create(device, C.byref(h)))
        self.h, self.device, self._lib = h, device, lib

    @classmethod
    def default(cls, device=0):
        if device not in cls._default:
            cls._default[device] = cls(device)
        return cls._default[device]

    @property
    def num_sms(self):
        x = C.c_int()
        check(self._lib.gfb_ctx_num_sms(self.h, C.byref(x)))
        return x.value

    def close(self):
        if getattr(self, "h", None):
            self._lib.gfb_ctx_destroy(self.h)
            self.h = None


class Graph:
    """Device-resident graph (graph.hpp:45-127): CSR + optional CSC view."""

    def __init__(self, handle, ctx):
        self.h, self.ctx, self._lib = handle, ctx, ctx._lib
        n, m, wt, csc = C.c_uint64(), C.c_uint64(), C.c_int(), C.c_int()
        check(self._lib.gfb_graph_info(handle, C.byref(n), C.byref(m), C.byref(wt), C.byref(csc)))
        self.num_vertices, self.num_edges = n.value, m.value
        self.wtype, self._csc = wt.value, bool(csc.value)
        self._csr_cache = None

    @classmethod
    def from_csr(cls, n, row_offsets, col, w, wtype="f64", transpose=False, ctx=None):
        """Upload a reference-layout CSR (row_offsets/column_indices/values)."""
        ctx = ctx or Context.default()
        ro = np.ascontiguousarray(row_offsets, np.uint32)
        col = np.ascontiguousarray(col, np.uint32)
        w = np.asarray(w)
        if w.dtype == np.float64:
            htype = W_F64
        elif w.dtype == np.float32:
            htype = W_F32
        elif w.dtype == np.uint32:
            htype = W_U32
        else:
            w = w.astype(np.float64)
            htype = W_F64
        w = np.ascontiguousarray(w)
        if len(ro) != n + 1:
            raise ValueError("row_offsets must have n + 1 entries")
        h = C.c_void_p()
        check(ctx._lib.gfb_graph_upload(ctx.h, n, len(col), _ptr(ro), _ptr(col), _ptr(w), htype,
                                        _WT[wtype] if isinstance(wtype, str) else wtype,
                                        int(transpose), C.byref(h)))
        return cls(h, ctx)

    def refill(self, row_offsets, col, w):
        w = np.ascontiguousarray(w)
        htype = {np.dtype(np.float64): W_F64, np.dtype(np.float32): W_F32,
                 np.dtype(np.uint32): W_U32}[w.dtype]
        check(self._lib.gfb_graph_refill(self.h, _ptr(np.ascontiguousarray(row_offsets, np.uint32)),
                                         _ptr(np.ascontiguousarray(col, np.uint32)), _ptr(w), htype))
        self._csr_cache = None

    def has_transpose(self):
        return self._csc

    def csr(self):
        """(row_offsets, column_indices, values) copied back from the device."""
        if self._csr_cache is None:
            ro = np.empty(self.num_vertices + 1, np.uint32)
            col = np.empty(self.num_edges, np.uint32)
            w = np.empty(self.num_edges, _WT_NP[self.wtype])
            check(self._lib.gfb_graph_download(self.h, _ptr(ro), _ptr(col), _ptr(w)))
            self._csr_cache = (ro, col, w)
        return self._csr_cache

    # graph.hpp:52-74 queries (host side, from the downloaded CSR)
    def get_edges(self, v):
        if v >= self.num_vertices:
            raise IndexError(f"get_edges: vertex {v} out of range")
        ro = self.csr()[0]
        return (int(ro[v]), int(ro[v + 1]))

    def get_dest_vertex(self, e):
        if e >= self.num_edges:
            raise IndexError(f"edge {e} out of range")
        return int(self.csr()[1][e])

    def get_edge_weight(self, e):
        if e >= self.num_edges:
            raise IndexError(f"edge {e} out of range")
        return float(self.csr()[2][e])

    def get_source_vertex(self, e):
        if e >= self.num_edges:
            raise IndexError(f"edge {e} out of range")
        return int(np.searchsorted(self.csr()[0], e, side="right") - 1)

    def free(self):
        if getattr(self, "h", None):
            self._lib.gfb_graph_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def build_csr(edges, num_vertices, wtype="f64", transpose=False, ctx=None):
    """graph.hpp:132-162: sort by (src, dst, weight), count + scan, upload.

    ``edges`` is a sequence of (src, dst, weight) or a tuple of three arrays.
    """
    if isinstance(edges, tuple) and len(edges) == 3 and hasattr(edges[0], "__len__") \
            and not isinstance(edges[0], tuple):
        src, dst, w = (np.asarray(x) for x in edges)
    else:
        arr = list(edges)
        src = np.array([e[0] for e in arr], dtype=np.int64)
        dst = np.array([e[1] for e in arr], dtype=np.int64)
        w = np.array([e[2] for e in arr], dtype=np.float64)
    src = src.astype(np.int64); dst = dst.astype(np.int64)
    w = np.asarray(w)
    if w.dtype not in (np.float32, np.uint32):
        w = w.astype(np.float64)
    n = int(num_vertices)
    for i in range(len(src)):  # graph.hpp:134-142, first offending edge
        if src[i] >= n or dst[i] >= n or src[i] < 0 or dst[i] < 0:
            raise ValueError(f"build_csr: edge {i} has vertex id out of range")
        if not (w[i] >= 0) or not math.isfinite(float(w[i])):
            raise ValueError(f"build_csr: edge {i} has negative or non-finite weight")
    order = np.lexsort((w, dst, src))
    col = dst[order].astype(np.uint32)
    ws = w[order]
    ro = np.zeros(n + 1, np.uint64)
    np.add.at(ro, src + 1, 1)
    ro = np.cumsum(ro).astype(np.uint32)
    return Graph.from_csr(n, ro, col, ws, wtype=wtype, transpose=transpose, ctx=ctx)


def build_transpose(g):
    """graph.hpp:166-193: a graph with the CSC view built (on the device)."""
    ro, col, w = g.csr()
    return Graph.from_csr(g.num_vertices, ro, col, w, wtype=g.wtype, transpose=True, ctx=g.ctx)


def rmat(scale, edgefactor=16, seed=1, wtype="f32", transpose=True, ctx=None):
    """Counter-based RMAT generated and built on the device."""
    ctx = ctx or Context.default()
    h = C.c_void_p()
    check(ctx._lib.gfb_graph_generate_rmat(ctx.h, scale, edgefactor, seed, _WT[wtype],
                                           int(transpose), C.byref(h)))
    return Graph(h, ctx)


def grid(side, seed=1, transpose=True, ctx=None):
    ctx = ctx or Context.default()
    h = C.c_void_p()
    check(ctx._lib.gfb_graph_generate_grid(ctx.h, side, seed, int(transpose), C.byref(h)))
    return Graph(h, ctx)


_LOOP = {"auto": 0, "bsp": 1}
_RELABEL = {"auto": 0, "on": 1, "off": 2}


def _opts(direction="push", pull_alpha=1.05, delta=0.0, device_loop=True, compute_pred=True,
          loop="auto", relabel="auto", defer_pct=0, advance_tile=0, trace=False, tail_edges=0):
    """gfb_sssp_opts (include/gfb.h).  The tuning knobs (loop, relabel,
    defer_pct, advance_tile, tail_edges) never change the result, only the
    schedule."""
    o = SsspOpts()
    _lib.load().gfb_sssp_opts_default(C.byref(o))
    if direction not in _DIR:
        raise ValueError("direction must be push|pull|auto")
    o.direction = _DIR[direction]
    o.pull_alpha = pull_alpha
    o.delta = delta
    o.device_loop = int(device_loop)
    o.compute_pred = int(compute_pred)
    if loop not in _LOOP or relabel not in _RELABEL:
        raise ValueError("loop must be auto|bsp, relabel auto|on|off")
    o.loop = _LOOP[loop]
    o.relabel = _RELABEL[relabel]
    o.defer_pct = int(defer_pct)
    o.advance_tile = int(advance_tile)
    o.trace = int(bool(trace))
    o.tail_edges = int(tail_edges)
    return o


def sssp(g, source, policy="device", direction="push", frontier="sparse", workers=None,
         as_lists=False, **kw):
    """algorithms.hpp:134-188 on the device.

    Mirrors module.cpp:115-128: returns ``(dist, pred, supersteps,
    relaxations)``.  ``dist`` is float64 (exact widening of the device
    arithmetic), ``pred`` uint32 with NIL for the source / unreachable
    vertices (``as_lists=True`` gives Python lists with ``None`` like the
    reference binding).  Distances equal the reference's for any frontier
    and direction (one fixpoint).  ``supersteps`` / ``relaxations`` are the
    DEVICE loop's counts: its frontier is always deduplicated (a bitmap, like
    the reference's ``uniquify_frontier`` / dense modes), expanded closest
    distance buckets first and with far buckets deferred to later supersteps
    (DESIGN.md §4), so they are NOT the reference's sparse-mode counts (which
    expand duplicates).  ``frontier`` selects the model: sparse | dense run
    the BSP loop, queue the asynchronous one (no supersteps, like the
    reference).  ``direction="auto"`` adds the push<->pull switch (pull when
    frontier edges > m / pull_alpha).
    """
    if policy != "device":
        raise ValueError("policy must be device (the CPU policies live in the reference)")
    if frontier not in ("sparse", "dense", "queue"):
        raise ValueError("frontier must be sparse|dense|queue")
    if frontier == "queue":  # the asynchronous model: one persistent work-queue launch
        if direction == "pull":
            raise ValueError("config: queue frontier requires push direction")
        direction = "push"
        kw = dict(kw, delta=float("inf"))
    dist, pred, st = sssp_stats(g, source, direction=direction, **kw)
    if frontier == "queue":
        st.supersteps = 0  # like the reference's async loop (algorithms.hpp:160-163)
    if as_lists:
        return (dist.tolist(), [None if p == NIL else int(p) for p in pred], st.supersteps,
                st.relaxations)
    return dist, pred, st.supersteps, st.relaxations


def bfs(g, source, policy="device", direction="push", frontier="sparse", workers=None,
        as_lists=False, want_result=True):
    """algorithms.hpp:194-239 on the device; mirrors module.cpp:130-140:
    returns ``(depths, supersteps, relaxations)`` with depths as float64
    (math.inf when unreachable).  The queue frontier is rejected like the
    reference (level semantics need supersteps)."""
    if policy != "device":
        raise ValueError("policy must be device (the CPU policies live in the reference)")
    if frontier == "queue":
        raise ValueError("bfs: queue configuration not supported "
                         "(level semantics require supersteps)")
    if frontier not in ("sparse", "dense"):
        raise ValueError("frontier must be sparse|dense")
    if direction not in _DIR:
        raise ValueError("direction must be push|pull|auto")
    if source < 0 or source >= g.num_vertices:  # algorithms.hpp:200 (a ctypes u32 would wrap)
        raise IndexError("bfs: source out of range")
    depth = np.empty(g.num_vertices, np.float64) if want_result else None
    st, rl = C.c_uint64(), C.c_uint64()
    check(g._lib.gfb_bfs(g.ctx.h, g.h, source, _DIR[direction], _ptr(depth), C.byref(st),
                         C.byref(rl)))
    if as_lists:
        return depth.tolist(), st.value, rl.value
    return depth, st.value, rl.value


def sssp_stats(g, source, direction="push", want_result=True, **kw):
    """gfb_sssp with the full statistics record (device time, n/m_reach...)."""
    if source < 0 or source >= g.num_vertices:  # algorithms.hpp:137 (a ctypes u32 would wrap)
        raise IndexError("sssp: source out of range")
    o = _opts(direction=direction, **kw)
    st = SsspStats()
    n = g.num_vertices
    dist = np.empty(n, np.float64) if want_result else None
    pred = np.empty(n, np.uint32) if want_result else None
    check(g._lib.gfb_sssp(g.ctx.h, g.h, source, C.byref(o), _ptr(dist), _ptr(pred), C.byref(st)))
    return dist, pred, st


def sssp_read(g, native=False):
    n = g.num_vertices
    dist = np.empty(n, _WT_NP[g.wtype] if native else np.float64)
    pred = np.empty(n, np.uint32)
    if native:
        check(g._lib.gfb_sssp_read(g.h, None, _ptr(dist), _ptr(pred)))
    else:
        check(g._lib.gfb_sssp_read(g.h, _ptr(dist), None, _ptr(pred)))
    return dist, pred


# ------------------------------------------------------------ operator level --

class Frontier:
    """Device frontier (frontier.hpp:37-218): sparse list or dense bitmap."""

    def __init__(self, repr_, num_vertices, ctx=None):
        if repr_ not in _REPR:
            raise ValueError("frontier must be sparse|dense")
        self.ctx = ctx or Context.default()
        self._lib = self.ctx._lib
        self.repr, self.num_vertices = repr_, num_vertices
        h = C.c_void_p()
        check(self._lib.gfb_frontier_create(self.ctx.h, num_vertices, _REPR[repr_], C.byref(h)))
        self.h = h

    def assign(self, vertices):
        v = np.ascontiguousarray(vertices, np.uint32)
        check(self._lib.gfb_frontier_assign(self.h, _ptr(v), len(v)))
        return self

    def size(self):
        x = C.c_uint64()
        check(self._lib.gfb_frontier_size(self.h, C.byref(x)))
        return x.value

    def contents(self):
        k = self.size()
        out = np.empty(max(k, 1), np.uint32)
        got = C.c_uint64()
        check(self._lib.gfb_frontier_read(self.h, _ptr(out), k, C.byref(got)))
        return out[: got.value]

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self._lib.gfb_frontier_free(self.h)
                self.h = None
        except Exception:
            pass


class DistanceMap:
    """Device distance map for the relax_min condition (algorithms.hpp:151-158)."""

    def __init__(self, g, source):
        self.g, self._lib = g, g._lib
        h = C.c_void_p()
        check(self._lib.gfb_dist_create(g.ctx.h, g.h, C.byref(h)))
        self.h = h
        check(self._lib.gfb_dist_init(h, source))

    def read(self):
        d = np.empty(self.g.num_vertices, np.float64)
        r = C.c_uint64()
        check(self._lib.gfb_dist_read(self.h, _ptr(d), C.byref(r)))
        return d, r.value

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self._lib.gfb_dist_free(self.h)
        except Exception:
            pass


class Recorder:
    """Records every (src, dst, edge) cond invocation (test_operators.cpp:151-171)."""

    def __init__(self, capacity, ctx=None):
        self.ctx = ctx or Context.default()
        self._lib = self.ctx._lib
        h = C.c_void_p()
        check(self._lib.gfb_record_create(self.ctx.h, capacity, C.byref(h)))
        self.h, self.capacity = h, capacity

    def read(self):
        cnt = C.c_uint64()
        check(self._lib.gfb_record_read(self.h, None, None, None, 0, C.byref(cnt)))
        k = min(cnt.value, self.capacity)
        s = np.empty(max(k, 1), np.uint32); d = np.empty_like(s); e = np.empty_like(s)
        check(self._lib.gfb_record_read(self.h, _ptr(s), _ptr(d), _ptr(e), k, C.byref(cnt)))
        return s[:k], d[:k], e[:k], cnt.value

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self._lib.gfb_record_free(self.h)
        except Exception:
            pass


def _cond(cond):
    if cond == "always":
        return OP_ALWAYS, None
    if isinstance(cond, DistanceMap):
        return OP_RELAX_MIN, cond.h
    if isinstance(cond, Recorder):
        return OP_RECORD, cond.h
    raise ValueError("device policy accepts the recognised conditions only: "
                     "DistanceMap (relax_min), Recorder (record) or 'always'")


def neighbors_expand(g, f, cond, policy="device"):
    """operators.hpp:35-68 push advance; output repr = input repr."""
    if policy != "device":
        raise ValueError("policy must be device")
    op, state = _cond(cond)
    out = Frontier(f.repr, g.num_vertices, ctx=g.ctx)
    check(g._lib.gfb_advance_push(g.ctx.h, g.h, f.h, out.h, op, state))
    return out


def neighbors_expand_pull(g, f, cond, policy="device"):
    """operators.hpp:76-114 pull advance (dense in, dense out)."""
    if policy != "device":
        raise ValueError("policy must be device")
    op, state = _cond(cond)
    out = Frontier("dense", g.num_vertices, ctx=g.ctx)
    check(g._lib.gfb_advance_pull(g.ctx.h, g.h, f.h, out.h, op, state))
    return out


def uniquify(f):
    """operators.hpp:191-200: ascending, duplicate-free sparse frontier."""
    out = Frontier("sparse", f.num_vertices, ctx=f.ctx)
    check(f._lib.gfb_filter_unique(f.ctx.h, f.h, out.h))
    return out


_PRED = {"dist_below": 0, "dist_at_least": 1, "reached": 2}


def filter(f, pred, dist, threshold=0.0, policy="device"):
    """operators.hpp:163-188: the elements of ``f`` whose predicate holds,
    same representation, sparse order and duplicates kept.  Host callables
    cannot run on the device: ``pred`` is a recognised predicate over the
    DistanceMap ``dist`` -- "dist_below" (dist[v] < threshold), "dist_at_least"
    (dist[v] >= threshold) or "reached" (dist[v] < inf)."""
    if policy != "device":
        raise ValueError("policy must be device")
    if pred not in _PRED:
        raise ValueError("device policy accepts the recognised predicates only: "
                         + ", ".join(_PRED))
    out = Frontier(f.repr, f.num_vertices, ctx=f.ctx)
    check(f._lib.gfb_filter(f.ctx.h, f.h, out.h, _PRED[pred], dist.h, float(threshold)))
    return out


# ------------------------------------------------------- Matrix Market I/O --

class EdgeList:
    """io.hpp:17-20 EdgeList: ``num_vertices`` and the edges as three arrays
    (0-based src / dst, double weights) in file order."""

    def __init__(self, num_vertices, src, dst, w):
        self.num_vertices, self.src, self.dst, self.w = num_vertices, src, dst, w

    @property
    def edges(self):
        return list(zip(self.src.tolist(), self.dst.tolist(), self.w.tolist()))


def parse_matrix_market(text, force_unit_weights=False, expand_symmetric=False):
    """io.hpp:43-129 parse_matrix_market (string overload) -> EdgeList; raises
    ParseError (with ``.line``) at the reference's lines and messages."""
    lib = _lib.load()
    b = text.encode() if isinstance(text, str) else bytes(text)
    h = C.c_void_p()
    check(lib.gfb_mm_parse(b, len(b), int(force_unit_weights), int(expand_symmetric),
                           C.byref(h)))
    try:
        n, m = C.c_uint64(), C.c_uint64()
        check(lib.gfb_edge_list_info(h, C.byref(n), C.byref(m)))
        src = np.empty(m.value, np.uint32); dst = np.empty(m.value, np.uint32)
        w = np.empty(m.value, np.float64)
        check(lib.gfb_edge_list_read(h, _ptr(src), _ptr(dst), _ptr(w)))
    finally:
        lib.gfb_edge_list_free(h)
    return EdgeList(n.value, src, dst, w)


def graph_from_edges(num_vertices, src, dst, w, wtype="f64", transpose=False, ctx=None):
    """build_csr (graph.hpp:132-162) on the device from an edge list: same
    validation and layout as the reference (rows sorted by (dst, weight))."""
    ctx = ctx or Context.default()
    src = np.ascontiguousarray(src, np.uint32)
    dst = np.ascontiguousarray(dst, np.uint32)
    w = np.ascontiguousarray(w, np.float64)
    if not (len(src) == len(dst) == len(w)):
        raise ValueError("graph_from_edges: src / dst / w lengths differ")
    h = C.c_void_p()
    check(ctx._lib.gfb_graph_from_edges(ctx.h, int(num_vertices), len(src), _ptr(src), _ptr(dst),
                                        _ptr(w), _WT[wtype] if isinstance(wtype, str) else wtype,
                                        int(transpose), C.byref(h)))
    return Graph(h, ctx)


def read_matrix_market(path_or_text, wtype="f64", transpose=False, force_unit_weights=False,
                       expand_symmetric=False, ctx=None):
    """A Matrix Market file (or its text) -> device Graph: the host parser
    (io.hpp:43-123) then build_csr on the device."""
    text = path_or_text
    if not (isinstance(text, (bytes, bytearray)) or "\n" in text or text.startswith("%%")):
        with open(path_or_text, "rb") as fh:
            text = fh.read()
    el = parse_matrix_market(text, force_unit_weights, expand_symmetric)
    return graph_from_edges(el.num_vertices, el.src, el.dst, el.w, wtype=wtype,
                            transpose=transpose, ctx=ctx)


def write_distances(dist, pred):
    """io.hpp:131-155: one line per vertex, ``<v> <dist %g|inf> <pred|->``."""
    if len(dist) != len(pred):
        raise ValueError("write_distances: array length mismatch")
    out = []
    for v, (d, p) in enumerate(zip(dist, pred)):
        ds = "inf" if d == math.inf else "%g" % d
        ps = "-" if p is None or p == NIL else str(int(p))
        out.append(f"{v} {ds} {ps}\n")
    return "".join(out)

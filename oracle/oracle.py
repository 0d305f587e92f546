"""ctypes front end for the CPU checker.  TEST INFRASTRUCTURE ONLY.

Loads ``oracle/liborc.so`` (the C restatement, graflow_oracle.c) and, when it
was built, ``oracle/_ref/libgraflow_ref.so`` (the unmodified reference headers
behind ref_shim.cpp).  Only tests/, ``__graft_entry__.smoke()`` and bench.py's
CPU-baseline legs import this module; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_ORC = None
_REF = None
NIL = 0xFFFFFFFF

u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
sz = C.c_size_t


def build():
    """Compile liborc.so (and _ref/ when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def orc():
    global _ORC
    if _ORC is None:
        path = os.path.join(HERE, "liborc.so")
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.orc_random_edges.restype = sz
        L.orc_random_edges.argtypes = [sz, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p, sz]
        L.orc_build_csr.restype = C.c_int64
        L.orc_build_csr.argtypes = [sz, sz, u32p, u32p, f64p, u32p, u32p, f64p]
        L.orc_build_transpose.argtypes = [sz, sz, u32p, u32p, f64p, u32p, u32p, f64p, u32p]
        L.orc_dijkstra_f64.argtypes = [sz, u32p, u32p, f64p, C.c_uint32, f64p, u32p]
        L.orc_dijkstra_f32.argtypes = [sz, u32p, u32p, f32p, C.c_uint32, f32p, u32p]
        L.orc_dijkstra_u32.argtypes = [sz, u32p, u32p, u32p, C.c_uint32, u64p, u32p]
        for nm, fp in (("orc_sssp_bsp_f64", f64p), ("orc_sssp_bsp_f32", f32p)):
            getattr(L, nm).argtypes = [sz, u32p, u32p, fp, C.c_uint32, C.c_int, fp,
                                       C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.orc_repair_pred_f64.argtypes = [sz, u32p, u32p, f64p, C.c_uint32, f64p, u32p]
        L.orc_repair_pred_f32.argtypes = [sz, u32p, u32p, f32p, C.c_uint32, f32p, u32p]
        L.orc_check_pred_tree.restype = C.c_int64
        L.orc_check_pred_tree.argtypes = [sz, u32p, u32p, C.c_void_p, C.c_void_p, C.c_int,
                                          C.c_uint32, u32p]
        L.orc_rmat_edges.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_int, C.c_uint64,
                                     C.c_uint64, u32p, u32p, u32p]
        L.orc_bfs.argtypes = [sz, u32p, u32p, C.c_uint32, f64p, C.POINTER(C.c_uint64),
                              C.POINTER(C.c_uint64)]
        L.orc_grid_csr.restype = C.c_uint64
        L.orc_grid_csr.argtypes = [C.c_uint32, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_rmat_csr.restype = C.c_uint64
        L.orc_rmat_csr.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_void_p,
                                   C.c_void_p, C.c_void_p]
        _ORC = L
    return _ORC


def ref():
    """The unmodified reference (or None when oracle/_ref was never built)."""
    global _REF
    if _REF is None:
        path = os.path.join(HERE, "_ref", "libgraflow_ref.so")
        if not os.path.exists(path):
            return None
        L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_hardware_concurrency.restype = C.c_uint
        L.ref_random_edges.restype = sz
        L.ref_random_edges.argtypes = [sz, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p, sz]
        L.ref_graph_new.argtypes = [sz, sz, u32p, u32p, f64p, C.c_int, C.POINTER(C.c_void_p)]
        L.ref_graph_free.argtypes = [C.c_void_p]
        L.ref_graph_csr.argtypes = [C.c_void_p, u32p, u32p, f64p]
        L.ref_graph_csc.argtypes = [C.c_void_p, u32p, u32p, f64p, u32p]
        L.ref_sssp.argtypes = [C.c_void_p, C.c_uint32, C.c_int, sz, C.c_int, C.c_int, C.c_int,
                               f64p, u32p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.ref_dijkstra.argtypes = [C.c_void_p, C.c_uint32, f64p, u32p]
        L.ref_bfs.argtypes = [C.c_void_p, C.c_uint32, C.c_int, sz, C.c_int, C.c_int, f64p,
                              C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.ref_expand_record.restype = sz
        L.ref_expand_record.argtypes = [C.c_void_p, u32p, sz, C.c_int, u32p, u32p, u32p, sz]
        L.ref_mm_parse.restype = C.c_longlong
        L.ref_mm_parse.argtypes = [C.c_char_p, sz, C.c_int, C.c_int, C.POINTER(sz), u32p, u32p,
                                   f64p, sz, C.POINTER(sz), C.c_char_p, sz]
        L.ref_filter.restype = sz
        L.ref_filter.argtypes = [sz, u32p, sz, C.c_int, C.c_int, f64p, C.c_double, C.c_int, sz,
                                 u32p, sz]
        _REF = L
    return _REF


# ---------------------------------------------------------------- helpers --

def random_edges(n, seed):
    """random_graphs.hpp:15-30 restated (orc_random_edges)."""
    L = orc()
    m = L.orc_random_edges(n, seed, None, None, None, 0)
    s = np.empty(m, np.uint32); d = np.empty(m, np.uint32); w = np.empty(m, np.float64)
    L.orc_random_edges(n, seed, s.ctypes.data, d.ctypes.data, w.ctypes.data, m)
    return s, d, w


def build_csr(n, src, dst, w):
    """graph.hpp:132-162 restated.  Returns (ro, col, val)."""
    src = np.ascontiguousarray(src, np.uint32); dst = np.ascontiguousarray(dst, np.uint32)
    w = np.ascontiguousarray(w, np.float64)
    m = len(src)
    ro = np.empty(n + 1, np.uint32); col = np.empty(max(m, 1), np.uint32)
    val = np.empty(max(m, 1), np.float64)
    bad = orc().orc_build_csr(n, m, src, dst, w, ro, col, val)
    if bad >= 0:
        raise ValueError(f"build_csr: edge {bad} is invalid")
    return ro, col[:m], val[:m]


def build_transpose(n, ro, col, val):
    m = len(col)
    cso = np.empty(n + 1, np.uint32); cs = np.empty(max(m, 1), np.uint32)
    cv = np.empty(max(m, 1), np.float64); ce = np.empty(max(m, 1), np.uint32)
    orc().orc_build_transpose(n, m, ro, np.ascontiguousarray(col) if m else np.zeros(1, np.uint32),
                              np.ascontiguousarray(val) if m else np.zeros(1), cso, cs, cv, ce)
    return cso, cs[:m], cv[:m], ce[:m]


def _nz(a, dt):
    a = np.ascontiguousarray(a, dt)
    return a if len(a) else np.zeros(1, dt)


def dijkstra(n, ro, col, w, source, kind="f64"):
    """algorithms.hpp:101-128 restated; kind f64 | f32 | u32."""
    L = orc()
    pred = np.empty(n, np.uint32)
    if kind == "f64":
        dist = np.empty(n, np.float64)
        rc = L.orc_dijkstra_f64(n, ro, _nz(col, np.uint32), _nz(w, np.float64), source, dist, pred)
    elif kind == "f32":
        dist = np.empty(n, np.float32)
        rc = L.orc_dijkstra_f32(n, ro, _nz(col, np.uint32), _nz(w, np.float32), source, dist, pred)
    else:
        dist = np.empty(n, np.uint64)
        rc = L.orc_dijkstra_u32(n, ro, _nz(col, np.uint32), _nz(w, np.uint32), source, dist, pred)
    if rc != 0:
        raise IndexError("reference_dijkstra: source out of range")
    return dist, pred


def bfs(n, ro, col, source):
    """algorithms.hpp:194-239 restated: (depth f64, supersteps, relaxations)."""
    depth = np.empty(max(n, 1), np.float64)
    st = C.c_uint64(); rl = C.c_uint64()
    if orc().orc_bfs(n, ro, _nz(col, np.uint32), source, depth, C.byref(st), C.byref(rl)) != 0:
        raise IndexError("bfs: source out of range")
    return depth[:n], st.value, rl.value


def sssp_bsp(n, ro, col, w, source, dedup=True):
    """algorithms.hpp:134-188 restated (sequential push); f64 or f32 by w dtype."""
    L = orc()
    st = C.c_uint64(); rl = C.c_uint64()
    if np.asarray(w).dtype == np.float32:
        dist = np.empty(n, np.float32)
        L.orc_sssp_bsp_f32(n, ro, _nz(col, np.uint32), _nz(w, np.float32), source, int(dedup),
                           dist, C.byref(st), C.byref(rl))
    else:
        dist = np.empty(n, np.float64)
        L.orc_sssp_bsp_f64(n, ro, _nz(col, np.uint32), _nz(w, np.float64), source, int(dedup),
                           dist, C.byref(st), C.byref(rl))
    return dist, st.value, rl.value


def repair_pred(n, ro, col, w, source, dist):
    pred = np.empty(n, np.uint32)
    if dist.dtype == np.float32:
        orc().orc_repair_pred_f32(n, ro, _nz(col, np.uint32), _nz(w, np.float32), source, dist, pred)
    else:
        orc().orc_repair_pred_f64(n, ro, _nz(col, np.uint32), _nz(w, np.float64), source,
                                  dist.astype(np.float64), pred)
    return pred


def check_pred_tree(n, ro, col, w, dist, source, pred):
    """-1 when valid, else the first bad vertex (acceptance.cpp:56-91 semantics)."""
    kind = 1 if np.asarray(dist).dtype == np.float32 else 0
    wt = np.float32 if kind else np.float64
    w = _nz(w, wt); dist = np.ascontiguousarray(dist, wt)
    return orc().orc_check_pred_tree(n, ro, _nz(col, np.uint32), w.ctypes.data, dist.ctypes.data,
                                     kind, source, np.ascontiguousarray(pred, np.uint32))


def rmat_edges(scale, edgefactor=16, seed=1, wkind=1, first=0, count=None):
    m = edgefactor << scale
    count = m - first if count is None else count
    s = np.empty(count, np.uint32); d = np.empty(count, np.uint32); w = np.empty(count, np.uint32)
    orc().orc_rmat_edges(scale, m, seed, wkind, first, count, s, d, w)
    return s, d, w


def rmat_csr(scale, edgefactor=16, seed=1, wkind=1, threads=0):
    """RMAT in build_csr layout, built on the host (orc_rmat_csr): (ro, col, w)
    with w float32 (wkind 1) or uint32 (wkind 0)."""
    L = orc()
    n, m = 1 << scale, edgefactor << scale
    ro = np.empty(n + 1, np.uint32); col = np.empty(m, np.uint32); w = np.empty(m, np.uint32)
    L.orc_rmat_csr(scale, edgefactor, seed, wkind, threads, ro.ctypes.data, col.ctypes.data,
                   w.ctypes.data)
    return ro, col, (w.view(np.float32) if wkind == 1 else w)


def grid_csr(side, seed=1):
    L = orc()
    m = L.orc_grid_csr(side, seed, None, None, None)
    ro = np.empty(side * side + 1, np.uint32); col = np.empty(m, np.uint32); w = np.empty(m, np.uint32)
    L.orc_grid_csr(side, seed, ro.ctypes.data, col.ctypes.data, w.ctypes.data)
    return ro, col, w.view(np.float32)


# ------------------------------------------------------- reference (_ref) --

class RefGraph:
    """The reference graflow::Graph built by its own build_csr/build_transpose."""

    def __init__(self, n, src, dst, w, transpose=False):
        L = ref()
        if L is None:
            raise RuntimeError("oracle/_ref/libgraflow_ref.so not built")
        self.L, self.n, self.m = L, n, len(src)
        h = C.c_void_p()
        rc = L.ref_graph_new(n, self.m, _nz(src, np.uint32), _nz(dst, np.uint32),
                             _nz(w, np.float64), int(transpose), C.byref(h))
        if rc:
            raise ValueError(L.ref_last_error().decode())
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_graph_free(self.h)
            self.h = None

    def csr(self):
        ro = np.empty(self.n + 1, np.uint32); col = np.empty(max(self.m, 1), np.uint32)
        val = np.empty(max(self.m, 1), np.float64)
        self.L.ref_graph_csr(self.h, ro, col, val)
        return ro, col[: self.m], val[: self.m]

    def csc(self):
        m = max(self.m, 1)
        cso = np.empty(self.n + 1, np.uint32); cs = np.empty(m, np.uint32)
        cv = np.empty(m, np.float64); ce = np.empty(m, np.uint32)
        self.L.ref_graph_csc(self.h, cso, cs, cv, ce)
        return cso, cs[: self.m], cv[: self.m], ce[: self.m]

    def sssp(self, source, mode=0, workers=1, direction=0, repr_=0, uniquify=False):
        dist = np.empty(max(self.n, 1), np.float64); pred = np.empty(max(self.n, 1), np.uint32)
        st = C.c_uint64(); rl = C.c_uint64()
        rc = self.L.ref_sssp(self.h, source, mode, workers, direction, repr_, int(uniquify),
                             dist, pred, C.byref(st), C.byref(rl))
        if rc:
            raise {1: ValueError, 2: IndexError}.get(rc, RuntimeError)(
                self.L.ref_last_error().decode())
        return dist[: self.n], pred[: self.n], st.value, rl.value

    def bfs(self, source, mode=0, workers=1, direction=0, repr_=0):
        depth = np.empty(max(self.n, 1), np.float64)
        st = C.c_uint64(); rl = C.c_uint64()
        rc = self.L.ref_bfs(self.h, source, mode, workers, direction, repr_, depth,
                            C.byref(st), C.byref(rl))
        if rc:
            raise {1: ValueError, 2: IndexError}.get(rc, RuntimeError)(
                self.L.ref_last_error().decode())
        return depth[: self.n], st.value, rl.value

    def dijkstra(self, source):
        dist = np.empty(max(self.n, 1), np.float64); pred = np.empty(max(self.n, 1), np.uint32)
        rc = self.L.ref_dijkstra(self.h, source, dist, pred)
        if rc:
            raise IndexError(self.L.ref_last_error().decode())
        return dist[: self.n], pred[: self.n]

    def expand_record(self, frontier, pull):
        f = np.ascontiguousarray(frontier, np.uint32)
        cnt = self.L.ref_expand_record(self.h, _nz(f, np.uint32), len(f), int(pull),
                                       np.empty(1, np.uint32), np.empty(1, np.uint32),
                                       np.empty(1, np.uint32), 0)
        s = np.empty(max(cnt, 1), np.uint32); d = np.empty_like(s); e = np.empty_like(s)
        self.L.ref_expand_record(self.h, _nz(f, np.uint32), len(f), int(pull), s, d, e, cnt)
        return s[:cnt], d[:cnt], e[:cnt]


def ref_filter(n, frontier, repr_, pred, dist, thr=0.0, mode=0, workers=1):
    """The reference's own filter (operators.hpp:163-188) with a distance
    predicate (0 below, 1 at least, 2 reached); contents in its order."""
    L = ref()
    f = np.ascontiguousarray(frontier, np.uint32)
    d = np.ascontiguousarray(dist, np.float64)
    out = np.empty(max(len(f), 1), np.uint32)
    cnt = L.ref_filter(n, _nz(f, np.uint32), len(f), repr_, pred, d, thr, mode, workers, out,
                       len(out))
    return out[:cnt]


def ref_mm_parse(text, force_unit_weights=False, expand_symmetric=False):
    """The reference's parse_matrix_market (io.hpp:43-123) on a text buffer:
    (n, src, dst, w), or ("error", line, message) on ParseError."""
    L = ref()
    b = text.encode() if isinstance(text, str) else bytes(text)
    n = C.c_size_t()
    line = C.c_size_t()
    msg = C.create_string_buffer(512)
    e = np.empty(1, np.uint32)
    cnt = L.ref_mm_parse(b, len(b), int(force_unit_weights), int(expand_symmetric), C.byref(n),
                         e, e, np.empty(1, np.float64), 0, C.byref(line), msg, 512)
    if cnt < 0:
        return ("error", line.value, msg.value.decode())
    s = np.empty(max(cnt, 1), np.uint32); d = np.empty_like(s); w = np.empty(max(cnt, 1))
    L.ref_mm_parse(b, len(b), int(force_unit_weights), int(expand_symmetric), C.byref(n), s, d, w,
                   cnt, C.byref(line), msg, 512)
    return n.value, s[:cnt], d[:cnt], w[:cnt]


def ref_random_edges(n, seed):
    L = ref()
    m = L.ref_random_edges(n, seed, None, None, None, 0)
    s = np.empty(m, np.uint32); d = np.empty(m, np.uint32); w = np.empty(m, np.float64)
    L.ref_random_edges(n, seed, s.ctypes.data, d.ctypes.data, w.ctypes.data, m)
    return s, d, w

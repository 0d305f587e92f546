"""1-D partitioned SSSP with a device-initiated exchange over peer memory.

The multi-GPU path of SURVEY.md §8e with §8f's "fused device-initiated
exchange" (peer.cu): the same edge-balanced 1-D partition as ``mg.py`` (cut
points rounded to multiples of 32), but no per-superstep messages, host
collectives or host round trips.  Each rank's loop state is one CUDA IPC
exportable allocation; after the one-time handle exchange below
(``torch.distributed.all_gather_object``: NCCL or gloo, any backend), the
push advance of every rank lowers remote distances directly in their owner's
memory over NVLink, and device-side barriers between ranks decide
convergence inside each rank's CUDA graph.

One process per GPU (``torchrun``); several processes may also share one GPU
(CUDA IPC between processes on the same device), which is how the tests
exercise world sizes 2 and 3 on a single B200.  The reference has no
partitioned SSSP (it is single-host); results are the same fixpoint as
``sssp()`` (algorithms.hpp:134-188) on the whole graph.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from . import mg

NIL = 0xFFFFFFFF
ALIGN = 32  # range starts: whole frontier-bitmap words per owner


def aligned_ranges(row_offsets, parts, align=ALIGN):
    """Edge-balanced cut points (mg.edge_balanced_ranges) rounded down to
    multiples of ``align``; parts+1 ascending vertex ids, 0 first, n last."""
    if parts < 1 or parts > 8:
        raise ValueError("peer: 1 <= parts <= 8")
    rs = mg.edge_balanced_ranges(row_offsets, parts).astype(np.int64)
    n = int(rs[-1])
    cuts = [0] + [(int(c) // align) * align for c in rs[1:-1]] + [n]
    return np.maximum.accumulate(np.array(cuts, dtype=np.int64)).astype(np.uint32)


def relabel_ranges(g, range_starts):
    """Range-preserving relabelled copy of device graph ``g`` for the
    partition ``range_starts`` (gfb_graph_relabel_ranges): inside each range
    vertices are ranked by descending in-degree and rows are sorted by
    destination -- the single-GPU loop's relabelled layout without moving a
    vertex to another owner.  Returns ``(row_offsets, col, w, perm)`` with
    ``perm[old] = new``; a distance of the relabelled graph maps back as
    ``dist_old = dist_new[perm]`` (``unrelabel``)."""
    from . import _WT_NP
    rs = np.ascontiguousarray(range_starts, np.uint32)
    n, m = g.num_vertices, g.num_edges
    ro = np.empty(n + 1, np.uint32)
    col = np.empty(max(m, 1), np.uint32)
    w = np.empty(max(m, 1), _WT_NP[g.wtype])
    perm = np.empty(max(n, 1), np.uint32)
    _lib.check(g._lib.gfb_graph_relabel_ranges(g.h, len(rs) - 1, C.c_void_p(rs.ctypes.data),
                                          C.c_void_p(ro.ctypes.data), C.c_void_p(col.ctypes.data),
                                          C.c_void_p(w.ctypes.data),
                                          C.c_void_p(perm.ctypes.data)))
    return ro, col[:m], w[:m], perm[:n]


def unrelabel(perm, dist_new, pred_new=None):
    """Results of a relabelled run in the original ids: dist[v] =
    dist_new[perm[v]], pred[v] = iperm[pred_new[perm[v]]] (NIL kept)."""
    perm = np.asarray(perm)
    dist = np.asarray(dist_new)[perm]
    if pred_new is None:
        return dist
    iperm = np.empty_like(perm)
    iperm[perm] = np.arange(len(perm), dtype=perm.dtype)
    p = np.asarray(pred_new)[perm]
    ok = p != NIL
    out = np.full(len(perm), NIL, np.uint32)
    out[ok] = iperm[p[ok]]
    return dist, out


class PeerSssp:
    """One rank's share: rows [range_starts[rank], range_starts[rank+1]) with
    global column ids (``mg.slice_csr``), on ``ctx``'s GPU."""

    def __init__(self, rank, nparts, range_starts, ro_local, col, w, ctx=None):
        import paper_2212_08200_b200 as gb
        self.gb = gb
        self.ctx = ctx or gb.Context.default()
        self.lib = _lib.load()
        self.rank, self.nparts = rank, nparts
        self.range_starts = np.ascontiguousarray(range_starts, np.uint32)
        if len(self.range_starts) != nparts + 1:
            raise ValueError("peer: range_starts needs nparts + 1 entries")
        self.lo = int(self.range_starts[rank])
        self.hi = int(self.range_starts[rank + 1])
        w = np.ascontiguousarray(w)
        if w.dtype == np.float32:
            wt = _lib.W_F32
        elif w.dtype == np.uint32:
            wt = _lib.W_U32
        else:
            raise ValueError("peer: f32 or u32 weights")
        self.wtype = wt
        ro = np.ascontiguousarray(ro_local, np.uint32)
        col = np.ascontiguousarray(col, np.uint32)
        h = C.c_void_p()
        gb.check(self.lib.gfb_peer_create(
            self.ctx.h, rank, nparts, C.c_void_p(self.range_starts.ctypes.data), len(col),
            C.c_void_p(ro.ctypes.data), C.c_void_p(col.ctypes.data) if len(col) else None,
            C.c_void_p(w.ctypes.data) if len(w) else None, wt, wt, C.byref(h)))
        self.h = h
        self.linked = False

    def handle(self) -> bytes:
        buf = (C.c_char * _lib.PEER_HANDLE_BYTES)()
        self.gb.check(self.lib.gfb_peer_export(self.h, buf))
        return bytes(buf)

    def link(self, group=None):
        """Exchange the IPC handles (collective over ``group``) and map the
        peers' memory.  Ends with a barrier: nobody relaxes into a peer before
        it is mapped everywhere."""
        mine = self.handle()
        if self.nparts > 1:
            import torch.distributed as dist
            handles = [None] * self.nparts
            dist.all_gather_object(handles, mine, group=group)
        else:
            handles = [mine]
        blob = b"".join(handles)
        self.gb.check(self.lib.gfb_peer_link(self.h, blob))
        if self.nparts > 1:
            import torch.distributed as dist
            dist.barrier(group=group)
        self.linked = True

    def sssp(self, source, want_pred=True, defer_pct=0):
        """Collective: every rank calls it with the same arguments.  Returns
        this rank's statistics (relaxations / n_reach / m_reach: local share)."""
        o = self.gb._opts(direction="push", compute_pred=want_pred, defer_pct=defer_pct)
        st = _lib.SsspStats()
        self.gb.check(self.lib.gfb_peer_sssp(self.h, int(source), C.byref(o), C.byref(st)))
        return {k: getattr(st, k) for k, _ in _lib.SsspStats._fields_}

    def read(self, native=False):
        """(dist, pred) of the local range: dist float64 (or the native 4-byte
        type), pred as global ids (NIL for the source / unreachable)."""
        n = self.hi - self.lo
        pred = np.empty(n, np.uint32)
        if native:
            dist = np.empty(n, np.float32 if self.wtype == _lib.W_F32 else np.uint32)
            self.gb.check(self.lib.gfb_peer_read(self.h, None, C.c_void_p(dist.ctypes.data),
                                                 C.c_void_p(pred.ctypes.data)))
        else:
            dist = np.empty(n, np.float64)
            self.gb.check(self.lib.gfb_peer_read(self.h, C.c_void_p(dist.ctypes.data), None,
                                                 C.c_void_p(pred.ctypes.data)))
        return dist, pred

    def free(self):
        if self.h:
            self.gb.check(self.lib.gfb_peer_free(self.h))
            self.h = None


def gather(peer, native=False, group=None):
    """Whole-graph (dist, pred) on every rank (tests; all_gather_object)."""
    d, p = peer.read(native=native)
    if peer.nparts == 1:
        return d, p
    import torch.distributed as dist
    parts = [None] * peer.nparts
    dist.all_gather_object(parts, (d, p), group=group)
    return np.concatenate([x[0] for x in parts]), np.concatenate([x[1] for x in parts])


class MgSssp:
    """The same partitioned SSSP driven by one process (gfb_mg_*): partition q
    on ``devices[q]`` (entries may repeat a device).  Takes the whole
    reference-layout CSR; returns whole-graph results."""

    def __init__(self, devices, row_offsets, col, w, exchange="peer"):
        """exchange: "peer" (device-initiated over peer memory) or "nccl"
        (host-driven bucketed messages, NCCL send/recv + allreduce;
        partitions sharing a device use device copies instead)."""
        import paper_2212_08200_b200 as gb
        self.gb = gb
        self.lib = _lib.load()
        devs = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        ex = {"peer": 0, "nccl": 1}[exchange]
        gb.check(self.lib.gfb_mg_create_ex(len(devices), devs, ex, C.byref(h)))
        self.h = h
        self.parts = len(devices)
        ro = np.ascontiguousarray(row_offsets, np.uint32)
        col = np.ascontiguousarray(col, np.uint32)
        w = np.ascontiguousarray(w)
        ht = {np.dtype(np.float32): _lib.W_F32, np.dtype(np.uint32): _lib.W_U32,
              np.dtype(np.float64): _lib.W_F64}[w.dtype]
        self.wtype = _lib.W_U32 if ht == _lib.W_U32 else _lib.W_F32
        self.n, self.m = len(ro) - 1, len(col)
        gb.check(self.lib.gfb_mg_graph_upload(
            self.h, self.n, self.m, C.c_void_p(ro.ctypes.data),
            C.c_void_p(col.ctypes.data) if self.m else None,
            C.c_void_p(w.ctypes.data) if self.m else None, ht, self.wtype))

    def uses_nccl(self):
        x = C.c_int()
        self.gb.check(self.lib.gfb_mg_uses_nccl(self.h, C.byref(x)))
        return bool(x.value)

    def ranges(self):
        rs = np.empty(self.parts + 1, np.uint32)
        self.gb.check(self.lib.gfb_mg_ranges(self.h, C.c_void_p(rs.ctypes.data)))
        return rs

    def sssp(self, source, want_pred=True, defer_pct=0):
        o = self.gb._opts(direction="push", compute_pred=want_pred, defer_pct=defer_pct)
        st = _lib.SsspStats()
        dist = np.empty(self.n, np.float64)
        pred = np.empty(self.n, np.uint32)
        self.gb.check(self.lib.gfb_mg_sssp(self.h, int(source), C.byref(o),
                                           C.c_void_p(dist.ctypes.data),
                                           C.c_void_p(pred.ctypes.data), C.byref(st)))
        return dist, pred, {k: getattr(st, k) for k, _ in _lib.SsspStats._fields_}

    def free(self):
        if self.h:
            self.gb.check(self.lib.gfb_mg_destroy(self.h))
            self.h = None

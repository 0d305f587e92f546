"""1-D partitioned BSP SSSP across ranks (BASELINE config 5).

The reference is single-host (no partitioned SSSP exists there); this module
distributes the same fixpoint: every rank owns a contiguous vertex range
[lo, hi) chosen on ``row_offsets`` so each rank holds ~m/P out-edges
(equal-vertex ranges give rank 0 ~44% of RMAT edges), the rows
of its range (column ids stay global) and the distances of its vertices.

One superstep, on every rank:
  1. ``advance``  expand the local frontier: local destinations are relaxed in
     place; remote candidates are min-combined per destination into
     16-byte messages ``{dst, src, dist_bits, 0}``, ascending dst (= grouped by
     owner) with per-owner counts;
  2. ``exchange`` all-to-all of the counts, then of the payload
     (``torch.distributed.all_to_all_single``: NCCL over NVLink/NVSwitch on
     GPUs, gloo on CPU);
  3. ``apply``    owners atomicMin the received candidates and activate;
  4. convergence: allreduce(SUM) of the local next-frontier sizes.
Predecessors: after convergence the distances are all-gathered and tight
in-edges are elected with allreduce(MIN) rounds (round 1 strictly decreasing
tight edges, later rounds equal-distance edges from already-resolved
sources), the same acyclicity rule as the single-GPU repair pass.

Engines: ``GfbPart`` runs the sm_100a kernels (``gfb_part_*`` in
include/gfb.h); ``CpuPart`` is a numpy restatement of the same contract used
to test the partitioning and exchange logic with gloo on CPU (it is host-side
protocol code, not a fallback: the GPU path never uses it).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

NIL = 0xFFFFFFFF
MSG_WORDS = 4  # {dst, src, dist_bits, 0}


# ------------------------------------------------------------ partitioning --

def edge_balanced_ranges(row_offsets, parts):
    """range_starts (parts+1 vertex ids): cut p = lower_bound(ro, p*m/parts)."""
    ro = np.asarray(row_offsets, dtype=np.int64)
    n, m = len(ro) - 1, int(ro[-1])
    cuts = [0]
    for p in range(1, parts):
        cuts.append(int(np.searchsorted(ro, (p * m) // parts, side="left")))
    cuts.append(n)
    cuts = np.maximum.accumulate(np.minimum(np.array(cuts, dtype=np.int64), n))
    return cuts.astype(np.uint32)


def equal_vertex_ranges(n, parts):
    return np.array([(p * n) // parts for p in range(parts + 1)], dtype=np.uint32)


def slice_csr(row_offsets, col, w, lo, hi):
    """Rows [lo, hi) of the global CSR, offsets rebased to 0, global columns."""
    ro = np.asarray(row_offsets)
    a, b = int(ro[lo]), int(ro[hi])
    return (ro[lo:hi + 1].astype(np.int64) - a).astype(np.uint32), col[a:b], w[a:b]


def owner_of(v, range_starts):
    return np.searchsorted(range_starts, v, side="right") - 1


# ------------------------------------------------------------------ engines --

class CpuPart:
    """numpy engine with the gfb_part contract (host-side protocol tests)."""

    def __init__(self, n_global, lo, hi, ro_local, col, w):
        self.n_global, self.lo, self.hi = n_global, lo, hi
        self.ro = np.asarray(ro_local, dtype=np.int64)
        self.col = np.asarray(col, dtype=np.int64)
        self.w = np.asarray(w)
        self.dt = np.float32 if self.w.dtype == np.float32 else np.uint64
        self.relaxations = 0
        self.supersteps = 0

    def init(self, source):
        n = self.hi - self.lo
        inf = np.float32(np.inf) if self.dt == np.float32 else np.uint64(np.iinfo(np.uint64).max)
        self.inf = inf
        self.dist = np.full(n, inf, dtype=self.dt)
        self.active = np.zeros(n, dtype=bool)
        if self.lo <= source < self.hi:
            self.dist[source - self.lo] = 0
            self.active[source - self.lo] = True
        self.relaxations = 0
        self.supersteps = 0

    def advance(self, range_starts):
        frontier = np.flatnonzero(self.active)
        self.active[:] = False
        best = {}
        if len(frontier):
            self.supersteps += 1
        for ul in frontier:  # ascending (the device plan is ascending too)
            du = self.dist[ul]
            for e in range(self.ro[ul], self.ro[ul + 1]):
                self.relaxations += 1
                v = int(self.col[e])
                nd = self.dt(du + self.w[e]) if self.dt == np.float32 else du + np.uint64(self.w[e])
                if self.lo <= v < self.hi:
                    if nd < self.dist[v - self.lo]:
                        self.dist[v - self.lo] = nd
                        self.active[v - self.lo] = True
                else:
                    key = (nd, ul + self.lo)
                    if v not in best or key < best[v]:
                        best[v] = key
        vs = np.array(sorted(best), dtype=np.int64)
        msgs = np.zeros((len(vs), MSG_WORDS), dtype=np.uint32)
        for i, v in enumerate(vs):
            nd, u = best[int(v)]
            msgs[i, 0] = v
            msgs[i, 1] = u
            msgs[i, 2] = (np.array([nd], np.float32).view(np.uint32)[0] if self.dt == np.float32
                          else np.uint32(nd))
        owners = owner_of(vs, range_starts) if len(vs) else np.zeros(0, np.int64)
        counts = np.bincount(owners, minlength=len(range_starts) - 1).astype(np.int64)
        return msgs, counts

    def apply(self, msgs):
        for v, u, bits, _ in np.asarray(msgs, dtype=np.uint32):
            nd = (np.array([bits], np.uint32).view(np.float32)[0] if self.dt == np.float32
                  else np.uint64(bits))
            if nd < self.dist[v - self.lo]:
                self.dist[v - self.lo] = nd
                self.active[v - self.lo] = True

    def pending(self):
        return int(self.active.sum())

    def dist_native(self):
        if self.dt == np.float32:
            return self.dist.copy()
        return np.minimum(self.dist, np.uint64(0xFFFFFFFF)).astype(np.uint32)

    def pred_candidates(self, gdist, res, cand, rnd):
        """cand[v] = min(cand[v], u) over local tight edges (round rules)."""
        f32 = self.dt == np.float32
        inf = np.float32(np.inf) if f32 else np.uint32(0xFFFFFFFF)
        for ul in range(self.hi - self.lo):
            u = ul + self.lo
            du = gdist[u]
            if du == inf or (rnd > 1 and not (1 <= res[u] <= rnd)):
                continue
            for e in range(self.ro[ul], self.ro[ul + 1]):
                v = int(self.col[e])
                if res[v] != 0:
                    continue
                dv = gdist[v]
                ok = du < dv if rnd == 1 else du == dv
                nd = np.float32(du + self.w[e]) if f32 else int(du) + int(self.w[e])
                if ok and nd == dv and u < cand[v]:
                    cand[v] = u


class GfbPart:
    """Device engine: one gfb_part on the rank's GPU (libgfb, sm_100a)."""

    def __init__(self, n_global, lo, hi, ro_local, col, w, ctx=None, device=0):
        import torch

        import paper_2212_08200_b200 as gb
        from . import _lib
        self.torch, self.gb = torch, gb
        self.ctx = ctx or gb.Context.default(device)
        self.lib = _lib.load()
        self.n_global, self.lo, self.hi = n_global, lo, hi
        self.dev = torch.device("cuda", self.ctx.device)
        w = np.ascontiguousarray(w)
        htype = _lib.W_F32 if w.dtype == np.float32 else _lib.W_U32
        self.wtype = htype
        ro = np.ascontiguousarray(ro_local, np.uint32)
        col = np.ascontiguousarray(col, np.uint32)
        h = C.c_void_p()
        gb.check(self.lib.gfb_part_create(self.ctx.h, n_global, lo, hi, len(col),
                                          C.c_void_p(ro.ctypes.data),
                                          C.c_void_p(col.ctypes.data) if len(col) else None,
                                          C.c_void_p(w.ctypes.data) if len(w) else None,
                                          htype, htype, C.byref(h)))
        self.h = h
        cap = max(n_global - (hi - lo), 1)
        self.out = torch.empty((cap, MSG_WORDS), dtype=torch.int32, device=self.dev)
        self.cap = cap

    def init(self, source):
        self.gb.check(self.lib.gfb_part_init(self.h, source))

    def advance(self, range_starts):
        rs = np.ascontiguousarray(range_starts, np.uint32)
        counts = np.zeros(len(rs) - 1, np.uint32)
        total = C.c_uint64()
        self.gb.check(self.lib.gfb_part_advance(self.h, C.c_void_p(self.out.data_ptr()), self.cap,
                                                C.c_void_p(rs.ctypes.data), len(rs) - 1,
                                                C.c_void_p(counts.ctypes.data), C.byref(total)))
        return self.out[: total.value], counts.astype(np.int64)

    def apply(self, msgs):
        if len(msgs):
            msgs = msgs.contiguous()
            self.gb.check(self.lib.gfb_part_apply(self.h, C.c_void_p(msgs.data_ptr()), len(msgs)))

    def pending(self):
        x = C.c_uint64()
        self.gb.check(self.lib.gfb_part_pending(self.h, C.byref(x)))
        return x.value

    @property
    def relaxations(self):
        r, s = C.c_uint64(), C.c_uint64()
        self.gb.check(self.lib.gfb_part_read(self.h, None, C.byref(r), C.byref(s)))
        return r.value

    @property
    def supersteps(self):
        r, s = C.c_uint64(), C.c_uint64()
        self.gb.check(self.lib.gfb_part_read(self.h, None, C.byref(r), C.byref(s)))
        return s.value

    def dist_native(self):
        d = np.empty(self.hi - self.lo, np.float32 if self.wtype == 1 else np.uint32)
        self.gb.check(self.lib.gfb_part_read(self.h, C.c_void_p(d.ctypes.data) if len(d) else None,
                                             None, None))
        return d

    def pred_candidates(self, gdist, res, cand, rnd):
        """gdist/res/cand: torch CUDA tensors (int32 views accepted)."""
        self.gb.check(self.lib.gfb_part_pred(self.h, C.c_void_p(gdist.data_ptr()),
                                             C.c_void_p(res.data_ptr()),
                                             C.c_void_p(cand.data_ptr()), rnd))

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.gfb_part_free(self.h)
                self.h = None
        except Exception:
            pass


# -------------------------------------------------------------- protocol ---

def _exchange(dist, msgs, counts, torch, device):
    """all-to-all of per-owner counts, then of the 16-byte message payload."""
    world = len(counts)
    send_counts = torch.as_tensor(np.asarray(counts, np.int64), device=device)
    recv_counts = torch.empty_like(send_counts)
    dist.all_to_all_single(recv_counts, send_counts)
    rc = recv_counts.cpu().tolist()
    sc = [int(c) for c in counts]
    if isinstance(msgs, np.ndarray):
        msgs = torch.from_numpy(msgs.view(np.int32))
    recv = torch.empty((sum(rc), MSG_WORDS), dtype=torch.int32, device=device)
    dist.all_to_all_single(recv, msgs.to(device), output_split_sizes=rc, input_split_sizes=sc)
    assert world == len(rc)
    return recv


def sssp_partitioned(engine, range_starts, source, group=None, device="cpu", want_pred=False):
    """Run the partitioned BSP loop on this rank.  Returns (dist_local native,
    pred_local or None, stats dict).  Every rank must call it."""
    import torch
    import torch.distributed as dist
    engine.init(source)
    steps = 0
    msgs_sent = 0
    while True:
        msgs, counts = engine.advance(range_starts)
        msgs_sent += int(np.sum(counts))
        recv = _exchange(dist, msgs, counts, torch, device)
        engine.apply(recv.cpu().numpy().view(np.uint32) if isinstance(engine, CpuPart) else recv)
        pend = torch.tensor([engine.pending()], dtype=torch.int64, device=device)
        dist.all_reduce(pend, op=dist.ReduceOp.SUM)
        steps += 1
        if int(pend.item()) == 0:
            break
    d = engine.dist_native()
    stats = {"supersteps": steps, "relaxations": engine.relaxations, "messages_sent": msgs_sent}
    pred = (_pred_partitioned(engine, d, range_starts, source, torch, dist, device)
            if want_pred else None)
    return d, pred, stats


def _gather_dist(d_local, range_starts, torch, dist, device):
    world = len(range_starts) - 1
    span = int(np.max(np.diff(range_starts.astype(np.int64)))) if world else 0
    pad = np.zeros(span, dtype=d_local.dtype)
    pad[: len(d_local)] = d_local
    t = torch.from_numpy(pad.view(np.int32)).to(device)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    out = np.concatenate([p.cpu().numpy()[: int(range_starts[r + 1] - range_starts[r])]
                          for r, p in enumerate(parts)])
    return out.view(d_local.dtype)


def _pred_partitioned(engine, d_local, range_starts, source, torch, dist, device):
    n = int(range_starts[-1])
    gdist = _gather_dist(d_local, range_starts, torch, dist, device)
    inf = np.float32(np.inf) if gdist.dtype == np.float32 else np.uint32(0xFFFFFFFF)
    res = np.zeros(n, np.uint32)
    reach = gdist != inf
    res[source] = 1  # the source is resolved without a predecessor
    pred = np.full(n, NIL, np.uint32)
    left = int(reach.sum()) - int((res != 0).sum())
    rnd = 1
    on_gpu = isinstance(engine, GfbPart)
    while left > 0:
        cand = np.full(n, NIL, np.uint32)
        if on_gpu:
            tg = torch.from_numpy(gdist.view(np.int32)).to(device)
            tr = torch.from_numpy(res.view(np.int32)).to(device)
            tc = torch.from_numpy(cand.view(np.int32)).to(device)
            engine.pred_candidates(tg, tr, tc, rnd)
            cand = tc.cpu().numpy().view(np.uint32).copy()
        else:
            engine.pred_candidates(gdist, res, cand, rnd)
        tc = torch.from_numpy(cand.astype(np.int64)).to(device)
        dist.all_reduce(tc, op=dist.ReduceOp.MIN)
        cand = tc.cpu().numpy().astype(np.uint32)
        newly = (cand != NIL) & (res == 0) & reach
        pred[newly] = cand[newly]
        res[newly] = rnd + 1
        got = int(newly.sum())
        if got == 0 and rnd > 1:
            raise RuntimeError("partitioned predecessor repair made no progress")
        left -= got
        rnd += 1
    lo, hi = int(range_starts[dist.get_rank()]), int(range_starts[dist.get_rank() + 1])
    return pred[lo:hi]


def sssp_simulated(engines, range_starts, source):
    """Single-process run of the same protocol over P engines (exchange by
    concatenation) -- exercises the partitioned device kernels on one GPU."""
    for e in engines:
        e.init(source)
    steps = 0
    while True:
        outbox = []
        for e in engines:
            msgs, counts = e.advance(range_starts)
            if not isinstance(msgs, np.ndarray):
                msgs = msgs.cpu().numpy().view(np.uint32)
            outbox.append((msgs.copy(), counts))
        for p, e in enumerate(engines):
            parts = []
            for msgs, counts in outbox:
                off = np.concatenate([[0], np.cumsum(counts)])
                parts.append(msgs[off[p]:off[p + 1]])
            inbox = np.concatenate(parts) if parts else np.zeros((0, MSG_WORDS), np.uint32)
            if isinstance(e, GfbPart):
                import torch
                e.apply(torch.from_numpy(inbox.view(np.int32)).to(e.dev))
            else:
                e.apply(inbox)
        steps += 1
        if sum(e.pending() for e in engines) == 0:
            break
    return np.concatenate([e.dist_native() for e in engines]), steps

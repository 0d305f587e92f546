"""GPU parity of the alternative loop drivers against the oracle.

Every driver runs the same operators (advance + relax + filter until the
frontier is empty, algorithms.hpp:151-167) in a different order, so they all
reach the same unique fixpoint: distances must be bit-identical to the
oracle (f32 restatement of reference_dijkstra, u32 = the reference's own
integer arithmetic) and predecessor trees valid.

  delta > 0          near-far filter, one persistent cooperative launch with
                     queue frontiers (nearfar.cuh) -- the high-diameter path
  relabel="on"       BSP loop on the in-degree-relabelled CSR (ensure_relabel)
  advance_tile=256   the push-advance instantiation the headline RMAT s24
                     run uses (chosen by size for m > 2^27 edges)
  defer_pct          the far-bucket deferral of the BSP filter (100 = off)
  loop="bsp"         never the automatic near-far choice
"""
import os

import numpy as np
import pytest

import paper_2212_08200_b200 as gb
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _check(g, dist, pred, source=0, wtype="f32"):
    ro, col, w = g.csr()
    if wtype == "f32":
        want, _ = O.dijkstra(g.num_vertices, ro, col, w, source, "f32")
        assert np.array_equal(dist.astype(np.float32), want)
        assert O.check_pred_tree(g.num_vertices, ro, col, w, dist.astype(np.float32), source,
                                 pred) == -1
    else:
        want, _ = O.dijkstra(g.num_vertices, ro, col, w.astype(np.float64), source, "f64")
        assert np.array_equal(dist, want)
        assert O.check_pred_tree(g.num_vertices, ro, col, w.astype(np.float64), dist, source,
                                 pred) == -1


@pytest.mark.parametrize("delta", [0.25, 1.0, 8.0])
def test_nearfar_grid(ctx, delta):
    g = gb.grid(128, seed=1, transpose=True, ctx=ctx)
    dist, pred, st = gb.sssp_stats(g, 0, delta=delta)
    _check(g, dist, pred)
    assert st.relaxations >= st.m_reach  # every reached edge relaxed at least once


@pytest.mark.parametrize("delta", [0.01, 0.1, 1.0])
def test_nearfar_rmat(ctx, delta):
    g = gb.rmat(12, 16, seed=1, wtype="f32", transpose=True, ctx=ctx)
    dist, pred, st = gb.sssp_stats(g, 0, delta=delta)
    _check(g, dist, pred)


def test_nearfar_u32_and_sources(ctx):
    g = gb.rmat(12, 16, seed=2, wtype="u32", transpose=True, ctx=ctx)
    for src in (0, 5, 1000):
        dist, pred, st = gb.sssp_stats(g, src, delta=16)
        _check(g, dist, pred, source=src, wtype="u32")


def test_nearfar_corpus_f32(ctx):
    """acceptance.cpp:95-122 corpus graphs (G(n, 4/n), 10% zero weights)."""
    corpus = np.load(os.path.join(os.path.dirname(__file__), "golden", "corpus.npz"))
    for i in range(0, 200, 7):
        n, seed = int(corpus["meta"][i][0]), int(corpus["meta"][i][1])
        s, d, w = O.random_edges(n, seed)
        g = gb.build_csr((s, d, w), n, wtype="f32", transpose=True, ctx=ctx)
        dist, pred, st = gb.sssp_stats(g, 0, delta=2.0)
        _check(g, dist, pred)


def test_nearfar_rejects_pull(ctx):
    g = gb.grid(16, seed=1, transpose=True, ctx=ctx)
    with pytest.raises(ValueError):
        gb.sssp_stats(g, 0, delta=1.0, direction="pull")


LOOP_OPTS = [dict(relabel="on"), dict(relabel="off"), dict(advance_tile=256),
             dict(advance_tile=128, relabel="on"), dict(advance_tile=256, relabel="on"),
             dict(defer_pct=100), dict(defer_pct=1), dict(defer_pct=50, advance_tile=256)]


@pytest.mark.parametrize("kw", LOOP_OPTS)
def test_loop_options_rmat(ctx, kw):
    g = gb.rmat(14, 16, seed=1, wtype="f32", transpose=True, ctx=ctx)
    dist, pred, st = gb.sssp_stats(g, 0, **kw)
    _check(g, dist, pred)


@pytest.mark.parametrize("kw", [dict(relabel="on", loop="bsp"), dict(advance_tile=256, loop="bsp"),
                                dict(defer_pct=100, loop="bsp")])
def test_loop_options_u32_grid(ctx, kw):
    g = gb.rmat(12, 16, seed=1, wtype="u32", transpose=True, ctx=ctx)
    dist, pred, st = gb.sssp_stats(g, 0, **kw)
    _check(g, dist, pred, wtype="u32")
    g = gb.grid(64, seed=1, transpose=True, ctx=ctx)
    dist, pred, st = gb.sssp_stats(g, 0, **kw)
    _check(g, dist, pred)


def test_headline_instantiation_corpus(ctx):
    """k_push_range<f32|u32, 1, 8, 256, 1> -- the instantiation RMAT s24 runs
    (tile 256 above 2^27 edges) -- forced on the acceptance corpus
    (acceptance.cpp:95-122) against the oracle, with and without relabelling."""
    corpus = np.load(os.path.join(os.path.dirname(__file__), "golden", "corpus.npz"))
    for i in range(0, 200, 3):
        n, seed = int(corpus["meta"][i][0]), int(corpus["meta"][i][1])
        s, d, w = O.random_edges(n, seed)
        for wt in ("f32", "u32"):
            ww = w if wt == "f32" else np.floor(w).astype(np.uint32)
            g = gb.build_csr((s, d, ww), n, wtype=wt, transpose=False, ctx=ctx)
            dist, pred, st = gb.sssp_stats(g, 0, advance_tile=256, loop="bsp",
                                           relabel="on" if i % 2 else "off")
            _check(g, dist, pred, wtype=wt)
            g.free()


@pytest.mark.parametrize("scale,wt", [(18, "f32"), (20, "f32"), (18, "u32")])
def test_headline_instantiation_rmat(ctx, scale, wt):
    """The s24 configuration (tile 256, relabelled CSR, 5 % deferral) at RMAT
    s18 / s20: bit-exact vs the oracle, valid predecessor tree."""
    g = gb.rmat(scale, 16, seed=1, wtype=wt, transpose=False, ctx=ctx)
    for src in (0, 3):
        dist, pred, st = gb.sssp_stats(g, src, advance_tile=256, relabel="on")
        _check(g, dist, pred, source=src, wtype=wt)


def test_relabel_view_is_permuted_csr(ctx):
    """ensure_relabel: rows keyed by descending in-degree, contents mapped,
    each row sorted by destination."""
    import ctypes as C
    from paper_2212_08200_b200 import _lib
    g = gb.rmat(10, 16, seed=1, wtype="f32", transpose=True, ctx=ctx)
    ro, col, w = g.csr()
    n, m = g.num_vertices, g.num_edges
    ro2 = np.zeros(n + 1, np.uint32)
    adj = np.zeros(2 * m, np.uint32)
    perm = np.zeros(n, np.uint32)
    assert _lib.load().gfb_debug_relabel(g.h, C.c_void_p(ro2.ctypes.data),
                                         C.c_void_p(adj.ctypes.data),
                                         C.c_void_p(perm.ctypes.data)) == 0
    indeg = np.bincount(col, minlength=n)
    iperm = np.argsort(-indeg.astype(np.int64), kind="stable")
    assert np.array_equal(perm[iperm], np.arange(n))
    deg = np.diff(ro.astype(np.int64))
    assert np.array_equal(ro2, np.concatenate([[0], np.cumsum(deg[iperm])]))
    dst, ww = adj[0::2], adj[1::2].view(np.float32)
    for i in range(0, n, 7):
        p = iperm[i]
        a = sorted(zip(perm[col[ro[p]:ro[p + 1]]].tolist(), w[ro[p]:ro[p + 1]].tolist()))
        b = sorted(zip(dst[ro2[i]:ro2[i + 1]].tolist(), ww[ro2[i]:ro2[i + 1]].tolist()))
        assert a == b
        assert np.all(np.diff(dst[ro2[i]:ro2[i + 1]].astype(np.int64)) >= 0)  # rows by destination


def test_default_path_rmat20_bit_exact(ctx):
    """The default BSP path at RMAT s20: the first call runs on the caller's
    ids, the second on the in-degree-relabelled CSR (built on reuse); both use
    the distance-ordered filter and the deferral of far buckets (pending sets
    with >= m/4 edges) -- bit-exact vs the oracle, valid predecessor trees,
    and the deferral actually cut the work."""
    g = gb.rmat(20, 16, seed=1, wtype="f32", transpose=True, ctx=ctx)
    for _ in range(2):
        dist, pred, st = gb.sssp_stats(g, 0)
        _check(g, dist, pred)
    _, _, plain = gb.sssp_stats(g, 0, want_result=False, defer_pct=100)  # deferral off
    assert st.relaxations < 0.8 * plain.relaxations


@pytest.mark.parametrize("src", [1, 12345])
def test_default_path_rmat20_other_sources_u32(ctx, src):
    g = gb.rmat(20, 16, seed=5, wtype="u32", transpose=False, ctx=ctx)
    dist, pred, st = gb.sssp_stats(g, src, direction="push")
    _check(g, dist, pred, source=src, wtype="u32")


def test_relabel_on_reuse_same_result(ctx):
    """The relabelled copy is built from the second SSSP on the same contents
    on (and dropped by a refill): every call returns identical results."""
    g = gb.rmat(20, 16, seed=3, wtype="f32", transpose=False, ctx=ctx)
    first = gb.sssp_stats(g, 0)
    _check(g, first[0], first[1])
    for _ in range(2):
        d, p, st = gb.sssp_stats(g, 0)
        assert np.array_equal(d, first[0])
        _check(g, d, p)
    ro, col, w = g.csr()
    g2 = gb.Graph.from_csr(g.num_vertices, ro, col, w.astype(np.float64), wtype="f32", ctx=ctx)
    import ctypes as C
    from paper_2212_08200_b200 import _lib
    assert _lib.load().gfb_graph_refill(g.h, C.c_void_p(ro.ctypes.data),
                                        C.c_void_p(col.ctypes.data),
                                        C.c_void_p(w.ctypes.data), gb.W_F32) == 0
    d, p, st = gb.sssp_stats(g, 0)  # first call after the refill: no relabel
    assert np.array_equal(d, first[0])
    assert np.array_equal(gb.sssp_stats(g2, 0)[0], first[0])


def test_f64_s20_relabel_records(ctx):
    """f64 arithmetic on the ordered loop (k_push_range<REC>) at 2^20 vertices:
    the first call runs on the caller's ids, later calls on the in-degree-
    relabelled CSR (records {u', edge'} mapped back in k_pred_verify<PERM>).
    Bit-exact vs the f64 restatement of reference_dijkstra, valid trees."""
    g32 = gb.rmat(20, 16, seed=4, wtype="f32", transpose=False, ctx=ctx)
    ro, col, w = g32.csr()
    n = g32.num_vertices
    g32.free()
    w64 = w.astype(np.float64)
    g = gb.Graph.from_csr(n, ro, col, w64, wtype="f64", ctx=ctx)
    for src in (0, 0, 12345):
        dist, pred, st = gb.sssp_stats(g, src, direction="push")
        want, _ = O.dijkstra(n, ro, col, w64, src, "f64")
        assert np.array_equal(dist, want), src
        assert O.check_pred_tree(n, ro, col, w64, dist, src, pred) == -1, src
    g.free()


def test_queue_model_fixpoint(ctx):
    """frontier="queue": the reference's asynchronous model (par-nosync,
    algorithms.hpp:160-163) as one persistent work-queue launch (near-far with
    no far set).  Same fixpoint, no supersteps reported."""
    cases = [(gb.rmat(12, 16, seed=5, wtype="f32", transpose=False, ctx=ctx), "f32"),
             (gb.rmat(12, 16, seed=6, wtype="u32", transpose=False, ctx=ctx), "u32"),
             (gb.grid(96, seed=7, transpose=False, ctx=ctx), "f32")]
    for g, wt in cases:
        for src in (0, 77):
            dist, pred, steps, relax = gb.sssp(g, src, frontier="queue")
            _check(g, dist, pred, source=src, wtype=wt)
            assert steps == 0 and relax > 0
    with pytest.raises(ValueError):
        gb.sssp(cases[0][0], 0, frontier="queue", direction="pull")


@pytest.mark.parametrize("wtype", ["f32", "u32"])
def test_nearfar_heavy_rows(ctx, wtype):
    """Rows longer than NF_HEAVY (2048) edges are expanded by a whole CTA in
    the next phase: hubs with 6000 / 3000 out-edges, queue model and near-far."""
    rng = np.random.default_rng(11)
    n = 20000
    src = np.concatenate([np.zeros(6000, np.int64), np.full(3000, 7),
                          rng.integers(0, n, 60000)])
    dst = np.concatenate([rng.integers(0, n, 6000), rng.integers(0, n, 3000),
                          rng.integers(0, n, 60000)])
    src[6000:9000] = 7
    w = rng.integers(0, 100, len(src)).astype(np.float64)
    if wtype == "f32":
        w = w / 7.0
    g = gb.build_csr((src.astype(np.uint32), dst.astype(np.uint32), w), n, wtype=wtype,
                     ctx=ctx)
    for kw in (dict(frontier="queue"), dict(delta=3.0, direction="push")):
        for s in (0, 7, 123):
            dist, pred, _, _ = gb.sssp(g, s, **kw)
            _check(g, dist, pred, source=s, wtype=wtype)


def test_auto_nearfar_on_mesh(ctx):
    """The default configuration picks the near-far loop on a low-degree mesh
    (max out-degree <= 8, n >= 2^16; delta = 32 x mean weight) and the BSP loop
    otherwise; loop="bsp" forces BSP.  Same distances either way."""
    g = gb.grid(300, seed=9, transpose=False, ctx=ctx)
    ro, col, w = g.csr()
    want, _ = O.dijkstra(g.num_vertices, ro, col, w, 0, "f32")
    d_auto, p_auto, st_auto = gb.sssp_stats(g, 0, direction="push")
    d_bsp, p_bsp, st_bsp = gb.sssp_stats(g, 0, direction="push", loop="bsp")
    for d, p in ((d_auto, p_auto), (d_bsp, p_bsp)):
        assert np.array_equal(d.astype(np.float32), want)
        assert O.check_pred_tree(g.num_vertices, ro, col, w, d.astype(np.float32), 0, p) == -1
    assert st_auto.supersteps * 2 < st_bsp.supersteps  # phases vs BSP supersteps
    g.free()


def _f64(g32, ctx):
    ro, col, w = g32.csr()
    n = g32.num_vertices
    g32.free()
    w64 = w.astype(np.float64)
    return gb.Graph.from_csr(n, ro, col, w64, wtype="f64", ctx=ctx), ro, col, w64


def test_nearfar_f64(ctx):
    """f64 arithmetic in the near-far / queue kernel (returning 64-bit mins,
    {u, edge} records, 32-bit entry tags): bit-exact vs the f64 restatement of
    reference_dijkstra; includes the automatic choice on a mesh."""
    for g32, kws in ((gb.grid(128, seed=4, transpose=False, ctx=ctx),
                      [dict(delta=4.0, direction="push"), dict(frontier="queue")]),
                     (gb.rmat(12, 16, seed=8, wtype="f32", transpose=False, ctx=ctx),
                      [dict(delta=0.1, direction="push"), dict(frontier="queue")]),
                     (gb.grid(300, seed=9, transpose=False, ctx=ctx), [dict()])):
        g, ro, col, w64 = _f64(g32, ctx)
        n = g.num_vertices
        for kw in kws:
            for src in (0, n // 2):
                dist, pred, _, _ = gb.sssp(g, src, **kw)
                want, _ = O.dijkstra(n, ro, col, w64, src, "f64")
                assert np.array_equal(dist, want), kw
                assert O.check_pred_tree(n, ro, col, w64, dist, src, pred) == -1, kw
        g.free()


@pytest.mark.parametrize("kw", [dict(pull_alpha=1.5, defer_pct=100), dict(pull_alpha=8.0),
                                dict(pull_alpha=8.0, defer_pct=100)])
def test_auto_switch_pulls(ctx, kw):
    """direction="auto": a superstep pulls when its frontier edges exceed
    m / pull_alpha (the reference's direction branch, algorithms.hpp:169-179,
    taken per superstep on the device).  At the measured break-even (1.05)
    only the densest deferral-free superstep of RMAT s24 qualifies (bench.py
    secondary line); here alpha 1.5 / 8 make the switch fire at s16.  Both
    directions must run and the distances stay bit-exact."""
    g = gb.rmat(16, 16, seed=1, wtype="f32", transpose=True, ctx=ctx)
    dist, pred, st = gb.sssp_stats(g, 0, direction="auto", **kw)
    assert st.pull_steps > 0 and st.push_steps > 0, (st.pull_steps, st.push_steps)
    _check(g, dist, pred)
    _, _, st2 = gb.sssp_stats(g, 0, direction="auto", pull_alpha=1.0)
    assert st2.pull_steps == 0  # a plan's edges never exceed m


# ---- the tail kernel (tail.cuh): small frontiers in one persistent launch ----

@pytest.mark.parametrize("wt", ["f32", "u32"])
@pytest.mark.parametrize("tail", [1 << 30, 50_000])
def test_tail_kernel_rmat(ctx, wt, tail):
    """tail_edges = 2^30: the tail takes over after the source's superstep and
    hands back to the bitmap filter whenever a queue outgrows qmax; 50K: the
    hand-over happens mid-run.  Same fixpoint either way, both loop drivers."""
    g = gb.rmat(16, 16, seed=3, wtype=wt, transpose=False, ctx=ctx)
    for dl in (True, False):
        for src in (0, 77):
            dist, pred, st = gb.sssp_stats(g, src, tail_edges=tail, device_loop=dl)
            _check(g, dist, pred, source=src, wtype=wt)
            assert st.supersteps > 0 and st.relaxations >= st.m_reach


def test_tail_kernel_off_same_result(ctx):
    """tail_edges = -1 (never) vs the default threshold vs always: identical
    distances (a schedule change only)."""
    g = gb.rmat(18, 16, seed=1, wtype="f32", transpose=False, ctx=ctx)
    runs = [gb.sssp_stats(g, 0, tail_edges=t) for t in (-1, 0, 1 << 30)]
    for dist, pred, _ in runs:
        _check(g, dist, pred)
    assert runs[0][2].supersteps > 0


def test_tail_kernel_grid_bsp(ctx):
    """A high-diameter mesh on the BSP loop: thousands of tiny supersteps, all
    but the first few inside the tail kernel."""
    g = gb.grid(256, seed=2, transpose=False, ctx=ctx)
    dist, pred, st = gb.sssp_stats(g, 0, loop="bsp")
    _check(g, dist, pred)
    d2, p2, st2 = gb.sssp_stats(g, 0, loop="bsp", tail_edges=-1)
    assert np.array_equal(dist, d2)


def test_tail_kernel_corpus(ctx):
    """The reference acceptance corpus (acceptance.cpp:95-122; every graph is
    small, so the default threshold of 4096 edges runs each one almost
    entirely in the tail), f32, two sources, both loop drivers."""
    corpus = np.load(os.path.join(os.path.dirname(__file__), "golden", "corpus.npz"))
    for i in range(0, 200, 7):
        row = corpus["meta"][i]
        n, seed = int(row[0]), int(row[1])
        s_, d_, w_ = O.random_edges(n, seed)
        g = gb.build_csr((s_, d_, w_), n, wtype="f32", ctx=ctx)
        ro, col, w32 = g.csr()
        for src in (0, n // 2):
            want, _ = O.dijkstra(n, ro, col, w32, src, "f32")
            for dl in (True, False):
                dist, pred, st = gb.sssp_stats(g, src, device_loop=dl)
                assert np.array_equal(dist.astype(np.float32), want), (i, src, dl)
                assert O.check_pred_tree(n, ro, col, w32, dist.astype(np.float32), src,
                                         pred) == -1, (i, src, dl)


@pytest.mark.parametrize("tail", [1 << 30, 0])
def test_tail_kernel_f64_records(ctx, tail):
    """f64 (record mode: returning mins, {u, edge} records) through the tail
    kernel, both loop drivers: bit-exact vs the f64 oracle, valid trees."""
    g32 = gb.rmat(15, 16, seed=7, wtype="f32", transpose=False, ctx=ctx)
    ro, col, w = g32.csr()
    n = g32.num_vertices
    g32.free()
    g = gb.Graph.from_csr(n, ro, col, w.astype(np.float64), wtype="f64", ctx=ctx)
    want, _ = O.dijkstra(n, ro, col, w.astype(np.float64), 0, "f64")
    for dl in (True, False):
        dist, pred, st = gb.sssp_stats(g, 0, tail_edges=tail, device_loop=dl)
        assert np.array_equal(dist, want), dl
        assert O.check_pred_tree(n, ro, col, w.astype(np.float64), dist, 0, pred) == -1, dl

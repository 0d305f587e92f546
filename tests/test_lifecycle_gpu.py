"""Handle lifecycle through the C ABI: refills, failed refills, cached loop
graphs, argument ranges.

The reference Graph is immutable (graph.hpp:42-44); the device handle can be
refilled with new contents of the same shape (gfb_graph_refill).  Everything
derived from the old contents -- the transpose, the relabelled copy and the
CUDA graphs of the device loop that point into them -- must be rebuilt, and a
refill that fails validation (build_csr's checks, graph.hpp:134-142) must
leave the handle unusable rather than half-updated.
"""
import ctypes as C

import numpy as np
import pytest

import paper_2212_08200_b200 as gb
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _refill(g, ro, col, w, htype):
    return gb._lib.load().gfb_graph_refill(g.h, C.c_void_p(ro.ctypes.data),
                                            C.c_void_p(col.ctypes.data),
                                            C.c_void_p(w.ctypes.data), htype)


def _want(g, ro, col, w, src=0):
    return O.dijkstra(g.num_vertices, ro, col, w, src, "f32")[0]


def test_refill_rebuilds_pull_loop(ctx):
    """AUTO with alpha > 1 can pull, so the device loop graph captures the
    transpose's buffers; a refill frees them (rebuilt lazily).  The next call
    must run on a rebuilt loop graph, not replay pointers into freed memory."""
    g = gb.rmat(14, 16, seed=1, wtype="f32", transpose=True, ctx=ctx)
    ro, col, w = (x.copy() for x in g.csr())
    for direction in ("auto", "pull"):
        d, p, st = gb.sssp_stats(g, 0, direction=direction, pull_alpha=4.0)
        assert np.array_equal(d.astype(np.float32), _want(g, ro, col, w))
    w2 = (w * np.float32(0.5)).astype(np.float32)  # new contents, same shape
    assert _refill(g, ro, col, w2, gb.W_F32) == 0
    g._csr_cache = None
    for direction in ("auto", "pull", "push"):
        for _ in range(2):
            d, p, st = gb.sssp_stats(g, 0, direction=direction, pull_alpha=4.0)
            assert np.array_equal(d.astype(np.float32), _want(g, ro, col, w2)), direction
            assert O.check_pred_tree(g.num_vertices, ro, col, w2, d.astype(np.float32), 0,
                                     p) == -1


def test_failed_refill_poisons_until_good_refill(ctx):
    g = gb.rmat(10, 16, seed=2, wtype="f32", transpose=True, ctx=ctx)
    ro, col, w = (x.copy() for x in g.csr())
    gb.sssp_stats(g, 0, direction="pull")  # transpose built, loop graph cached
    bad = col.copy()
    bad[17] = g.num_vertices + 5  # graph.hpp:136-138: vertex id out of range
    with pytest.raises(ValueError, match="edge 17"):
        g.refill(ro, bad, w)
    for call in (lambda: gb.sssp_stats(g, 0), lambda: gb.bfs(g, 0),
                 lambda: gb.sssp_stats(g, 0, direction="pull")):
        with pytest.raises(RuntimeError, match="failed refill"):
            call()
    negw = w.copy()
    negw[3] = -1.0  # graph.hpp:139-141
    with pytest.raises(ValueError, match="edge 3"):
        g.refill(ro, col, negw)
    with pytest.raises(RuntimeError, match="failed refill"):
        gb.sssp_stats(g, 0)
    g.refill(ro, col, w)  # good contents: usable again, transpose rebuilt on demand
    for direction in ("push", "pull", "auto"):
        d, p, st = gb.sssp_stats(g, 0, direction=direction)
        assert np.array_equal(d.astype(np.float32), _want(g, ro, col, w)), direction


def test_tuning_options_change_the_loop_graph(ctx):
    """The device loop graph is keyed by every option its launches depend on:
    switching tile / deferral / relabel between calls rebuilds it, and each
    configuration returns the same fixpoint."""
    g = gb.rmat(16, 16, seed=3, wtype="f32", transpose=False, ctx=ctx)
    ro, col, w = g.csr()
    want = _want(g, ro, col, w)
    seen = set()
    for kw in (dict(), dict(advance_tile=256), dict(defer_pct=100), dict(relabel="on"),
               dict(relabel="on", advance_tile=256), dict(), dict(defer_pct=20)):
        d, p, st = gb.sssp_stats(g, 0, **kw)
        assert np.array_equal(d.astype(np.float32), want), kw
        seen.add(st.relaxations)
    assert len(seen) > 1  # the schedules really differed


def test_bad_options_rejected(ctx):
    g = gb.rmat(8, 8, seed=1, wtype="f32", transpose=False, ctx=ctx)
    for kw in (dict(advance_tile=64), dict(defer_pct=101), dict(defer_pct=-1)):
        with pytest.raises(ValueError):
            gb.sssp_stats(g, 0, **kw)


@pytest.mark.parametrize("src", [256, 2 ** 32 + 5])
def test_source_out_of_range(ctx, src):
    """algorithms.hpp:137 / :200: std::out_of_range -> IndexError, including
    ids a 32-bit ctypes argument would silently wrap (2^32 + 5 -> 5)."""
    g = gb.rmat(8, 8, seed=1, wtype="f32", transpose=False, ctx=ctx)
    with pytest.raises(IndexError):
        gb.sssp_stats(g, src)
    with pytest.raises(IndexError):
        gb.bfs(g, src)

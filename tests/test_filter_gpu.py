"""Device filter (operators.hpp:163-188) against the reference's own filter.

The reference keeps exactly the frontier elements whose predicate holds, in
the same representation; a sparse frontier keeps its order and duplicates in
sequential mode (:184-186).  The device accepts the recognised distance
predicates only (host callables cannot cross the C ABI); the reference side
runs the same predicate as a C++ lambda through the unmodified headers
(oracle/_ref, ref_filter).
"""
import numpy as np
import pytest

import paper_2212_08200_b200 as gb
from oracle import oracle as O

pytestmark = pytest.mark.gpu

PREDS = {"dist_below": 0, "dist_at_least": 1, "reached": 2}


@pytest.fixture(scope="module")
def ref():
    if O.ref() is None:
        pytest.skip("oracle/_ref not built")
    return O


def _dist_map(g, source):
    """A device distance map after a full SSSP from `source`, via the
    operator-level API (neighbors_expand with relax_min until empty)."""
    dm = gb.DistanceMap(g, source)
    f = gb.Frontier("sparse", g.num_vertices, ctx=g.ctx).assign([source])
    while f.size():
        f = gb.uniquify(gb.neighbors_expand(g, f, dm))
    return dm


@pytest.mark.parametrize("wtype", ["f32", "u32", "f64"])
def test_filter_matches_reference(ctx, ref, wtype):
    g = gb.rmat(11, 8, seed=4, wtype="f32" if wtype == "f64" else wtype, transpose=False, ctx=ctx)
    if wtype == "f64":
        ro, col, w = g.csr()
        g = gb.Graph.from_csr(g.num_vertices, ro, col, w.astype(np.float64), wtype="f64", ctx=ctx)
    n = g.num_vertices
    dm = _dist_map(g, 0)
    dist, _ = dm.read()
    rng = np.random.default_rng(7)
    fin = dist[np.isfinite(dist)]
    thresholds = [0.0, float(np.median(fin)), float(fin.max()), float(fin.max()) + 1, np.inf]
    lists = [np.array([], np.uint32), np.array([0], np.uint32),
             rng.integers(0, n, 5000).astype(np.uint32),           # duplicates, random order
             np.arange(n, dtype=np.uint32)[::-1].copy(),           # descending, all vertices
             rng.integers(0, 64, 3000).astype(np.uint32)]          # heavy duplication
    for lst in lists:
        for repr_ in ("sparse", "dense"):
            f = gb.Frontier(repr_, n, ctx=ctx).assign(lst)
            for pred, pid in PREDS.items():
                for thr in (thresholds if pid != 2 else [0.0]):
                    got = gb.filter(f, pred, dm, thr)
                    want = ref.ref_filter(n, lst, 1 if repr_ == "dense" else 0, pid, dist, thr)
                    assert got.repr == repr_
                    assert np.array_equal(got.contents(), want), (repr_, pred, thr, len(lst))


def test_filter_large_sparse_order(ctx, ref):
    """Several 2048-element tiles: the ordered write must stitch tiles in
    order (count -> scan -> write)."""
    g = gb.rmat(16, 8, seed=2, wtype="f32", transpose=False, ctx=ctx)
    n = g.num_vertices
    dm = _dist_map(g, 3)
    dist, _ = dm.read()
    lst = np.random.default_rng(3).integers(0, n, 200_001).astype(np.uint32)
    f = gb.Frontier("sparse", n, ctx=ctx).assign(lst)
    thr = float(np.median(dist[np.isfinite(dist)]))
    for pred in ("dist_below", "dist_at_least", "reached"):
        got = gb.filter(f, pred, dm, thr).contents()
        want = ref.ref_filter(n, lst, 0, PREDS[pred], dist, thr)
        assert np.array_equal(got, want), pred


def test_filter_par_policy_same_set(ctx, ref):
    """The reference's parallel mode chunks statically and merges per worker
    in order, so even par(k) yields the sequential order (operators.hpp:
    172-187): the device result equals it too."""
    g = gb.rmat(12, 8, seed=5, wtype="u32", transpose=False, ctx=ctx)
    n = g.num_vertices
    dm = _dist_map(g, 0)
    dist, _ = dm.read()
    lst = np.random.default_rng(5).integers(0, n, 10000).astype(np.uint32)
    f = gb.Frontier("sparse", n, ctx=ctx).assign(lst)
    thr = float(np.median(dist[np.isfinite(dist)]))
    got = gb.filter(f, "dist_below", dm, thr).contents()
    want = ref.ref_filter(n, lst, 0, 0, dist, thr, mode=1, workers=8)
    assert np.array_equal(got, want)


def test_filter_rejects(ctx):
    g = gb.rmat(8, 8, seed=1, wtype="f32", transpose=False, ctx=ctx)
    dm = gb.DistanceMap(g, 0)
    f = gb.Frontier("sparse", g.num_vertices, ctx=ctx).assign([1, 2])
    with pytest.raises(ValueError):
        gb.filter(f, "odd_vertices", dm)
    with pytest.raises(ValueError):
        gb.filter(f, "dist_below", dm, float("nan"))
    other = gb.rmat(9, 8, seed=1, wtype="f32", transpose=False, ctx=ctx)
    with pytest.raises(ValueError):
        gb.filter(gb.Frontier("sparse", other.num_vertices, ctx=ctx).assign([1]), "reached", dm)

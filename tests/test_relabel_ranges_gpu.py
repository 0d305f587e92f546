"""gfb_graph_relabel_ranges: the range-preserving relabelled copy the
partitioned paths run on (bench.py --gpus N / --partitioned).  Properties:
perm is a permutation mapping every partition range onto itself, rows move
with their vertex (same weights, destinations mapped through perm, sorted),
inside a range vertices come by descending in-degree, and SSSP on the copy
from perm[source] equals the oracle on the original (dist_old =
dist_new[perm]); the partitioned run on a relabelled copy is checked in
tests/mg_worker.py (its own process: same-device partitions need
CUDA_DEVICE_MAX_CONNECTIONS set before CUDA starts)."""
import numpy as np
import pytest

import paper_2212_08200_b200 as gb
from oracle import oracle as O
from paper_2212_08200_b200 import peer

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("wt,parts", [("f32", 1), ("f32", 3), ("u32", 4), ("f64", 2)])
def test_relabel_ranges_properties(ctx, wt, parts):
    g = gb.rmat(13, 16, seed=4, wtype="f32" if wt == "f64" else wt, transpose=False, ctx=ctx)
    if wt == "f64":  # (the generator makes 4-byte weights: widen exactly)
        ro, col, w = g.csr()
        g = gb.Graph.from_csr(g.num_vertices, ro, col, w.astype(np.float64), wtype="f64", ctx=ctx)
    ro, col, w = g.csr()
    n = g.num_vertices
    rs = peer.aligned_ranges(ro, parts)
    ro2, col2, w2, perm = peer.relabel_ranges(g, rs)
    assert np.array_equal(np.sort(perm), np.arange(n, dtype=np.uint32))
    for q in range(parts):
        lo, hi = int(rs[q]), int(rs[q + 1])
        assert perm[lo:hi].min(initial=lo) >= lo and perm[lo:hi].max(initial=lo) < max(hi, lo + 1)
    deg, deg2 = np.diff(ro.astype(np.int64)), np.diff(ro2.astype(np.int64))
    assert np.array_equal(deg2[perm], deg)
    indeg = np.bincount(col, minlength=n)
    iperm = np.empty_like(perm)
    iperm[perm] = np.arange(n, dtype=perm.dtype)
    for q in range(parts):  # descending in-degree inside each range
        lo, hi = int(rs[q]), int(rs[q + 1])
        d = indeg[iperm[lo:hi]]
        assert np.all(np.diff(d) <= 0)
    for v in range(0, n, 37):
        a = sorted(zip(perm[col[ro[v]:ro[v + 1]]].tolist(), w[ro[v]:ro[v + 1]].tolist()))
        r = perm[v]
        seg = col2[ro2[r]:ro2[r + 1]]
        assert np.all(np.diff(seg.astype(np.int64)) >= 0)
        b = sorted(zip(seg.tolist(), w2[ro2[r]:ro2[r + 1]].tolist()))
        assert a == b
    # SSSP on the copy maps back to the oracle's distances on the original
    kind = {"f32": "f32", "u32": "f64", "f64": "f64"}[wt]
    want, _ = O.dijkstra(n, ro, col, w.astype(np.float32 if kind == "f32" else np.float64), 0, kind)
    g2 = gb.Graph.from_csr(n, ro2, col2, w2, wtype=wt, ctx=ctx)
    d2, p2, _ = gb.sssp_stats(g2, int(perm[0]))
    d_old, p_old = peer.unrelabel(perm, d2, p2)
    if kind == "f32":
        assert np.array_equal(d_old.astype(np.float32), want)
        assert O.check_pred_tree(n, ro, col, w, d_old.astype(np.float32), 0, p_old) == -1
    else:
        assert np.array_equal(d_old, want)
        assert O.check_pred_tree(n, ro, col, w.astype(np.float64), d_old, 0, p_old) == -1


def test_relabel_ranges_rejects_bad_ranges(ctx):
    g = gb.rmat(10, 16, seed=1, wtype="f32", transpose=False, ctx=ctx)
    n = g.num_vertices
    for bad in ([0, n + 1], [1, n], [0, 600, 500, n]):
        with pytest.raises(ValueError):
            peer.relabel_ranges(g, np.array(bad, np.uint32))

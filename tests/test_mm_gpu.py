"""Device build_csr from an edge list (graph.cu graph_from_edges) and the
Matrix Market path end to end: the CSR equals the unmodified reference's
build_csr (graph.hpp:132-162: rows by (dst, weight), parallel edges kept),
validation names the same first bad edge, and SSSP on an ingested file
matches the reference's Dijkstra bit for bit."""
import numpy as np
import pytest

import paper_2212_08200_b200 as gb
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _ref_csr(n, s, d, w):
    g = O.RefGraph(n, s, d, w)
    return g.csr()


@pytest.mark.parametrize("wtype", ["f64", "f32", "u32"])
def test_edges_build_equals_reference_build_csr(ctx, wtype):
    if O.ref() is None:
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(3)
    n = 5000
    s = rng.integers(0, n, 60000).astype(np.uint32)
    d = rng.integers(0, n, 60000).astype(np.uint32)
    w = rng.integers(0, 40, 60000).astype(np.float64) / (1.0 if wtype == "u32" else 8.0)
    s[:500] = 7  # a heavy row with parallel edges and equal (dst, w) pairs
    d[:500] = rng.integers(0, 20, 500)
    g = gb.graph_from_edges(n, s, d, w, wtype=wtype, ctx=ctx)
    ro, col, val = g.csr()
    rro, rcol, rval = _ref_csr(n, s, d, w)
    assert np.array_equal(ro, rro) and np.array_equal(col, rcol)
    assert np.array_equal(val.astype(np.float64), rval.astype(val.dtype).astype(np.float64))
    dist, pred, _, _ = gb.sssp(g, 0)
    want, _ = O.RefGraph(n, s, d, w).dijkstra(0)  # k/8 weights: exact in every arithmetic
    assert np.array_equal(dist, want)


def test_edges_build_validation(ctx):
    """build_csr (graph.hpp:134-142): the first offending edge, vertex check
    before the weight check of the same edge."""
    s = np.array([0, 1, 2, 3], np.uint32)
    d = np.array([1, 2, 3, 0], np.uint32)
    w = np.array([1.0, -1.0, 1.0, 1.0])
    with pytest.raises(ValueError, match="edge 1 has negative or non-finite weight"):
        gb.graph_from_edges(4, s, d, w, ctx=ctx)
    d2 = d.copy()
    d2[1] = 9
    with pytest.raises(ValueError, match="edge 1 has vertex id out of range"):
        gb.graph_from_edges(4, s, d2, w, ctx=ctx)
    w2 = np.array([1.0, 1.0, np.inf, 1.0])
    with pytest.raises(ValueError, match="edge 2 has negative"):
        gb.graph_from_edges(4, s, d, w2, ctx=ctx)
    g = gb.graph_from_edges(4, s[:0], d[:0], w[:0], ctx=ctx)  # no edges
    assert gb.sssp(g, 2)[0].tolist() == [np.inf, np.inf, 0.0, np.inf]


def _grid_mm(side, rng):
    """A road-like symmetric grid with integer weights, as a Matrix Market
    `integer symmetric` file (each undirected edge once)."""
    lines = []
    for r in range(side):
        for c in range(side):
            u = r * side + c + 1
            if c + 1 < side:
                lines.append(f"{u + 1} {u} {rng.integers(1, 100)}")
            if r + 1 < side:
                lines.append(f"{u + side} {u} {rng.integers(1, 100)}")
    head = (f"%%MatrixMarket matrix coordinate integer symmetric\n% synthetic road grid\n"
            f"{side * side} {side * side} {len(lines)}\n")
    return head + "\n".join(lines) + "\n"


@pytest.mark.parametrize("wtype", ["u32", "f64"])
def test_matrix_market_sssp_matches_reference(ctx, wtype):
    if O.ref() is None:
        pytest.skip("oracle/_ref not built")
    text = _grid_mm(120, np.random.default_rng(5))
    g = gb.read_matrix_market(text, wtype=wtype, expand_symmetric=True, ctx=ctx)
    n, s, d, w = O.ref_mm_parse(text, expand_symmetric=True)
    rg = O.RefGraph(n, s, d, w)
    ro, col, val = g.csr()
    rro, rcol, rval = rg.csr()
    assert np.array_equal(ro, rro) and np.array_equal(col, rcol)
    for src in (0, n // 2):
        dist, pred, _, _ = gb.sssp(g, src)  # default: near-far on this mesh
        want, _ = rg.dijkstra(src)
        assert np.array_equal(dist, want)
        assert O.check_pred_tree(n, rro, rcol, rval, dist, src, pred) == -1

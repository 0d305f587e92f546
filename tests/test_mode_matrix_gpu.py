"""Every loop the device can pick, on graph shapes that stress different
corners, in every arithmetic -- all against the oracle (distances bit-exact:
f64 / u32 vs the reference's own arithmetic, f32 vs the fp32 restatement;
predecessor trees valid).

shapes: random G(n, 4/n) with 10% zero weights (tie classes, acceptance.cpp
corpus generator), RMAT with duplicates and self-loops, a 2-D grid, a long
path with a back edge, a star hub (heavy rows) and a graph with unreachable
parts.  loops: default (automatic choice), push BSP, pull BSP (transpose),
AUTO, near-far (small delta), the queue model, forced BSP (loop="bsp").
"""
import numpy as np
import pytest

import paper_2212_08200_b200 as gb
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _shapes():
    rng = np.random.default_rng(2026)
    out = []
    s, d, w = O.random_edges(700, 77)
    out.append(("corpus", 700, np.asarray(s), np.asarray(d), np.asarray(w)))
    s, d, wb = O.rmat_edges(11, 8, seed=3, wkind=1)
    out.append(("rmat", 1 << 11, s, d, wb.view(np.float32).astype(np.float64)))
    g = gb.grid(40, seed=5, transpose=False)
    ro, col, w = g.csr()
    g.free()
    src = np.repeat(np.arange(len(ro) - 1), np.diff(ro.astype(np.int64)))
    out.append(("grid", len(ro) - 1, src, col, w.astype(np.float64)))
    n = 3000
    s = np.arange(n - 1)
    out.append(("path", n, np.concatenate([s, [n - 1]]), np.concatenate([s + 1, [0]]),
                np.concatenate([rng.random(n - 1), [0.5]])))
    hub = np.zeros(1500, np.int64)
    out.append(("star", 2000, np.concatenate([hub, rng.integers(0, 2000, 4000)]),
                np.concatenate([rng.integers(1, 2000, 1500), rng.integers(0, 2000, 4000)]),
                rng.random(5500)))
    out.append(("islands", 1000, rng.integers(0, 300, 2000), rng.integers(0, 300, 2000),
                rng.random(2000)))
    return out


LOOPS = [dict(), dict(direction="push"), dict(direction="pull"), dict(direction="auto"),
         dict(direction="push", delta=0.05), dict(frontier="queue"),
         dict(direction="push", loop="bsp")]


@pytest.mark.parametrize("wtype", ["f64", "f32", "u32"])
def test_mode_matrix(ctx, wtype):
    for name, n, s, d, w in _shapes():
        if wtype == "u32":
            w = np.floor(w * 10)
        g = gb.build_csr((np.asarray(s, np.uint32), np.asarray(d, np.uint32), w), n,
                         wtype=wtype, transpose=True, ctx=ctx)
        ro, col, wv = g.csr()
        for src in (0, n // 3):
            if wtype == "f32":
                want, _ = O.dijkstra(n, ro, col, wv, src, "f32")
            else:
                want, _ = O.dijkstra(n, ro, col, wv.astype(np.float64), src, "f64")
            for kw in LOOPS:
                if wtype != "f32" and "delta" in kw:
                    kw = dict(kw, delta=1.0 if wtype == "u32" else 0.05)
                dist, pred, _, _ = gb.sssp(g, src, **kw)
                if wtype == "f32":
                    ok = np.array_equal(dist.astype(np.float32), want)
                    tree = O.check_pred_tree(n, ro, col, wv, dist.astype(np.float32), src, pred)
                else:
                    ok = np.array_equal(dist, want)
                    tree = O.check_pred_tree(n, ro, col, wv.astype(np.float64), dist, src, pred)
                assert ok and tree == -1, (name, wtype, src, kw, ok, tree)
        g.free()

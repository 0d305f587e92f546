"""bench.sp_certificate: the size-independent shortest-path proof bench.py
applies where the oracle's Dijkstra is slow (RMAT s26).  CPU only."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from oracle import oracle as O  # noqa: E402


def _graph():
    s, d, w = O.rmat_edges(12, 16, seed=3, wkind=1)
    n = 1 << 12
    ro, col, val = O.build_csr(n, s, d, w.view(np.float32).astype(np.float64))
    return n, ro, col, val.astype(np.float32)


def test_certificate_accepts_the_fixpoint():
    n, ro, col, w = _graph()
    dist, pred = O.dijkstra(n, ro, col, w, 0, "f32")
    assert bench.sp_certificate(ro, col, w, dist, pred, 0) == {
        "source_zero": True, "relaxable_edges": 0, "pred_tree_valid": True}


def test_certificate_rejects_too_high_and_too_low():
    n, ro, col, w = _graph()
    dist, pred = O.dijkstra(n, ro, col, w, 0, "f32")
    i = int(np.flatnonzero(np.isfinite(dist) & (dist > 0))[5])
    hi = dist.copy()
    hi[i] *= np.float32(1.5)  # an edge into i can still relax
    c = bench.sp_certificate(ro, col, w, hi, pred, 0)
    assert c["relaxable_edges"] > 0
    lo = dist.copy()
    lo[i] *= np.float32(0.5)  # no tight in-edge any more
    assert not bench.sp_certificate(ro, col, w, lo, pred, 0)["pred_tree_valid"]

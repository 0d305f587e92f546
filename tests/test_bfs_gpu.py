"""GPU parity of the device BFS (gfb_bfs, bfs.cu) -- algorithms.hpp:194-239.

Depths, supersteps and relaxations must equal the reference's own bfs()
(tests/golden/bfs.npz, acceptance.cpp:180-199 graphs) in every direction,
and the oracle restatement (orc_bfs) on RMAT / grid graphs; the reference's
rejections (queue frontier, pull without a transpose, source out of range)
are kept.
"""
import os

import numpy as np
import pytest

import paper_2212_08200_b200 as gb
from oracle import oracle as O

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_bfs_hand_checked(ctx):
    tri = gb.build_csr([(0, 1, 1.0), (0, 2, 4.0), (1, 2, 2.0)], 3, ctx=ctx)
    assert gb.bfs(tri, 0, as_lists=True)[0] == [0.0, 1.0, 1.0]      # test_algorithms.cpp:186
    path = gb.build_csr([(0, 1, 5.0), (1, 2, 0.5), (2, 3, 2.0)], 4, ctx=ctx)
    assert gb.bfs(path, 0)[0].tolist() == [0.0, 1.0, 2.0, 3.0]       # :189-191
    d, st, rl = gb.bfs(path, 2)
    assert d.tolist() == [np.inf, np.inf, 0.0, 1.0] and st == 2 and rl == 1
    with pytest.raises(ValueError):
        gb.bfs(tri, 0, frontier="queue")                             # :194-198
    with pytest.raises(ValueError):
        gb.bfs(tri, 0, direction="pull")                             # no transpose
    with pytest.raises(IndexError):
        gb.bfs(tri, 3)


@pytest.mark.parametrize("direction", ["push", "pull", "auto"])
@pytest.mark.parametrize("wtype", ["f64", "f32", "u32"])
def test_bfs_matches_reference_goldens(ctx, direction, wtype):
    gold = np.load(os.path.join(GOLD, "bfs.npz"))
    for n, seed, src, st_p, rl_p, st_q, rl_q in gold["meta"].astype(np.int64):
        s, d, w = O.random_edges(int(n), int(seed))
        if wtype == "u32":
            w = np.floor(w)
        g = gb.build_csr((s, d, w), int(n), wtype=wtype, transpose=True, ctx=ctx)
        depth, st, rl = gb.bfs(g, int(src), direction=direction)
        assert np.array_equal(depth, gold[f"depth_{seed - 6000}_{src}"]), (n, seed, src)
        want_st, want_rl = (st_q, rl_q) if direction == "pull" else (st_p, rl_p)
        assert (st, rl) == (want_st, want_rl), (n, seed, src, st, rl)
        g.free()


def test_bfs_rmat_and_grid(ctx):
    for g in (gb.rmat(14, 16, seed=3, wtype="f32", transpose=False, ctx=ctx),
              gb.grid(96, seed=2, transpose=False, ctx=ctx)):
        ro, col, _ = g.csr()
        n = g.num_vertices
        for src in (0, n // 3):
            want, wst, wrl = O.bfs(n, ro, col, src)
            depth, st, rl = gb.bfs(g, src)
            assert np.array_equal(depth, want) and (st, rl) == (wst, wrl)
            again = gb.bfs(g, src)  # the captured loop graph is reused
            assert np.array_equal(again[0], want)
        # an SSSP between BFS calls on the same graph keeps both correct
        dist, _, _, _ = gb.sssp(g, 0)
        assert np.isfinite(dist[0])
        assert np.array_equal(gb.bfs(g, 0)[0], O.bfs(n, ro, col, 0)[0])
        g.free()


def test_bfs_edge_cases(ctx):
    one = gb.build_csr([], 1, ctx=ctx)                      # single vertex (test_algorithms.cpp:110-113)
    d, st, rl = gb.bfs(one, 0)
    assert d.tolist() == [0.0] and st == 1 and rl == 0
    iso = gb.build_csr([(1, 2, 1.0)], 4, transpose=True, ctx=ctx)  # source without out-edges
    for direction in ("push", "auto", "pull"):
        d, st, rl = gb.bfs(iso, 0, direction=direction)
        assert np.isinf(d[1:]).all() and d[0] == 0 and st == 1 and rl == 0
        d, st, rl = gb.bfs(iso, 1, direction=direction)
        assert d.tolist() == [np.inf, 0.0, 1.0, np.inf] and st == 2 and rl == 1

"""CPU tests: pin the oracle restatement (oracle/graflow_oracle.c) against the
golden vectors produced by the unmodified reference (tests/golden/), and
against the live reference library when oracle/_ref was built here."""
import hashlib
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:32]


@pytest.fixture(scope="module")
def corpus():
    return np.load(os.path.join(GOLD, "corpus.npz"))


def _hex(a):
    return bytes(a).hex()


def test_acceptance_sizes_match_mt19937_64(corpus):
    """acceptance.cpp:98-101 draws n = 2 + mt19937_64(2024)() % 499."""
    import ctypes as C
    L = O.orc()
    L.orc_mt64_next.restype = C.c_uint64
    st = C.create_string_buffer(312 * 8 + 16)
    L.orc_mt64_seed(st, C.c_uint64(2024))
    sizes = [2 + L.orc_mt64_next(st) % 499 for _ in range(200)]
    assert sizes == [int(r[0]) for r in corpus["meta"]]


def test_random_edges_restatement_matches_reference(corpus):
    """random_graphs.hpp:15-30 restated bit for bit (all 200 instances)."""
    for i, row in enumerate(corpus["meta"]):
        n, seed, m = int(row[0]), int(row[1]), int(row[2])
        s, d, w = O.random_edges(n, seed)
        assert len(s) == m
        assert digest(s, d, w) == _hex(corpus[f"digest_edges_{i}"]), i


def test_dijkstra_f64_matches_reference(corpus):
    """algorithms.hpp:101-128 restated: exact distances on the 200-graph sweep."""
    for i, row in enumerate(corpus["meta"]):
        n, seed = int(row[0]), int(row[1])
        s, d, w = O.random_edges(n, seed)
        ro, col, val = O.build_csr(n, s, d, w)
        dist, pred = O.dijkstra(n, ro, col, val, 0, "f64")
        assert digest(dist) == _hex(corpus[f"digest_dist_{i}"]), i
        if i < 24:
            assert np.array_equal(dist, corpus[f"dist_{i}"])


def test_bsp_restatement_supersteps_and_relaxations(corpus):
    """algorithms.hpp:134-188 seq push: same supersteps/relaxations as the
    reference in both sparse (duplicates) and dense (set) frontier modes."""
    for i, row in enumerate(corpus["meta"][:80]):
        n, seed = int(row[0]), int(row[1])
        s, d, w = O.random_edges(n, seed)
        ro, col, val = O.build_csr(n, s, d, w)
        ref, _ = O.dijkstra(n, ro, col, val, 0, "f64")
        dist, st, rl = O.sssp_bsp(n, ro, col, val, 0, dedup=False)
        assert np.array_equal(dist, ref)
        assert (st, rl) == (int(row[3]), int(row[4])), i
        dist, st, rl = O.sssp_bsp(n, ro, col, val, 0, dedup=True)
        assert np.array_equal(dist, ref)
        assert (st, rl) == (int(row[5]), int(row[6])), i


def test_repair_predecessors_gives_valid_tree(corpus):
    """algorithms.hpp:77-93 + the checker of acceptance.cpp:56-91."""
    for i, row in enumerate(corpus["meta"][:60]):
        n, seed = int(row[0]), int(row[1])
        s, d, w = O.random_edges(n, seed)
        ro, col, val = O.build_csr(n, s, d, w)
        dist, _ = O.dijkstra(n, ro, col, val, 0, "f64")
        pred = O.repair_pred(n, ro, col, val, 0, dist)
        assert O.check_pred_tree(n, ro, col, val, dist, 0, pred) == -1


def test_pred_checker_rejects_bad_trees():
    s, d, w = O.random_edges(60, 3)
    ro, col, val = O.build_csr(60, s, d, w)
    dist, _ = O.dijkstra(60, ro, col, val, 0, "f64")
    pred = O.repair_pred(60, ro, col, val, 0, dist)
    reach = np.flatnonzero(np.isfinite(dist))
    v = int(reach[reach != 0][0])
    bad = pred.copy(); bad[v] = O.NIL
    assert O.check_pred_tree(60, ro, col, val, dist, 0, bad) == v
    bad = pred.copy(); bad[0] = 1
    assert O.check_pred_tree(60, ro, col, val, dist, 0, bad) == 0


def test_f32_oracles_agree(corpus):
    """fp32 fixpoint is unique: Dijkstra-f32 == BSP-f32 (sparse and dense)."""
    for row in corpus["meta"][:60]:
        n, seed = int(row[0]), int(row[1])
        s, d, w = O.random_edges(n, seed)
        ro, col, val = O.build_csr(n, s, d, w)
        w32 = val.astype(np.float32)
        a, _ = O.dijkstra(n, ro, col, w32, 0, "f32")
        b, _, _ = O.sssp_bsp(n, ro, col, w32, 0, dedup=True)
        c, _, _ = O.sssp_bsp(n, ro, col, w32, 0, dedup=False)
        assert np.array_equal(a, b) and np.array_equal(a, c)


def test_build_csr_rejects_like_reference():
    """graph.hpp:134-142: invalid_argument naming the first bad edge."""
    with pytest.raises(ValueError, match="edge 1"):
        O.build_csr(3, [0, 0], [1, 5], [1.0, 1.0])
    with pytest.raises(ValueError, match="edge 0"):
        O.build_csr(3, [0], [1], [-1.0])


def test_triangle_goldens():
    """test_algorithms.cpp:120-132 hand-checked graphs."""
    ro, col, val = O.build_csr(3, [0, 0, 1], [1, 2, 2], [1.0, 4.0, 2.0])
    assert list(ro) == [0, 2, 3, 3] and list(col) == [1, 2, 2] and list(val) == [1, 4, 2]
    dist, pred = O.dijkstra(3, ro, col, val, 0)
    assert list(dist) == [0, 1, 3] and list(pred) == [O.NIL, 0, 1]
    ro, col, val = O.build_csr(4, [0, 1, 2], [1, 2, 3], [1.0, 1.0, 1.0])
    assert list(O.dijkstra(4, ro, col, val, 0)[0]) == [0, 1, 2, 3]
    ro, col, val = O.build_csr(2, [0], [1], [0.0])
    assert list(O.dijkstra(2, ro, col, val, 0)[0]) == [0, 0]
    with pytest.raises(IndexError):
        O.dijkstra(3, *O.build_csr(3, [0], [1], [1.0]), 3)


def test_rmat16_u32_oracle_matches_reference():
    """Config 1: RMAT s16 u32; oracle Dijkstra (u32 sums) == the reference's
    sssp() and reference_dijkstra() (f64), and the CSR layout is identical."""
    g = np.load(os.path.join(GOLD, "rmat16.npz"))
    s, d, wb = O.rmat_edges(16, 16, seed=1, wkind=0)
    assert digest(s, d, wb) == _hex(g["edge_digest"])
    ro, col, val = O.build_csr(1 << 16, s, d, wb.astype(np.float64))
    assert digest(ro, col, val) == _hex(g["csr_digest"])
    dist, _ = O.dijkstra(1 << 16, ro, col, val.astype(np.uint32), 0, "u32")
    ref = g["dist"]
    fin = np.isfinite(ref)
    assert np.array_equal(dist[fin].astype(np.float64), ref[fin])
    assert np.all(dist[~fin] == np.iinfo(np.uint64).max)
    assert np.array_equal(ref, g["dijkstra"])


def test_operator_record_goldens():
    """operators.hpp:35-114: push/pull eligibility sets equal (the oracle
    enumerates them from the restated CSR/CSC, the golden from the reference)."""
    ops = np.load(os.path.join(GOLD, "ops.npz"))
    for seed in (1, 2, 3, 4, 5):
        s, d, w = O.random_edges(40, seed)
        ro, col, val = O.build_csr(40, s, d, w)
        f = range(0, 40, 2)
        push = [(v, int(col[e]), e) for v in f for e in range(ro[v], ro[v + 1])]
        assert np.array_equal(np.array(push, dtype=np.uint32).T.reshape(3, -1),
                              ops[f"rec_{seed}_0"])
        pull = ops[f"rec_{seed}_1"]
        assert sorted(map(tuple, pull.T.tolist())) == sorted(push)


def test_rmat_and_grid_generators_shape():
    s, d, w = O.rmat_edges(10, 16, seed=1, wkind=1)
    assert len(s) == 16 << 10 and s.max() < 1024 and d.max() < 1024
    wf = w.view(np.float32)
    assert (wf >= 0).all() and (wf < 1).all()
    assert np.all(wf * 16777216 == np.round(wf * 16777216))
    # vertex 0 is the hub (unpermuted labels)
    deg = np.bincount(s, minlength=1024)
    assert deg.argmax() == 0
    ro, col, wg = O.grid_csr(8, seed=1)
    assert ro[-1] == 4 * 8 * 7 and len(col) == ro[-1]
    for u in range(64):
        nb = col[ro[u]:ro[u + 1]]
        assert list(nb) == sorted(nb)


@pytest.mark.skipif(O.ref() is None, reason="oracle/_ref not built (no /root/reference)")
def test_live_reference_f32_vs_f64_ulps():
    """The f32 fixpoint vs the reference's f64 result: small ulp distance
    (reported, not a gate)."""
    s, d, wb = O.rmat_edges(12, 16, seed=1, wkind=1)
    w64 = wb.view(np.float32).astype(np.float64)
    g = O.RefGraph(1 << 12, s, d, w64)
    ref, _ = g.dijkstra(0)
    ro, col, val = g.csr()
    d32, _ = O.dijkstra(1 << 12, ro, col, val.astype(np.float32), 0, "f32")
    fin = np.isfinite(ref)
    a = d32[fin].view(np.int32).astype(np.int64)
    b = ref[fin].astype(np.float32).view(np.int32).astype(np.int64)
    assert np.abs(a - b).max() <= 4


def test_bfs_restatement_matches_reference_goldens():
    """orc_bfs (algorithms.hpp:194-239 restated) against the reference's own
    bfs() on acceptance C5's 50 graphs (tests/golden/bfs.npz): depth,
    supersteps and relaxations, push and pull alike."""
    gold = np.load(os.path.join(GOLD, "bfs.npz"))
    for n, seed, src, st_p, rl_p, st_q, rl_q in gold["meta"].astype(np.int64):
        s, d, w = O.random_edges(int(n), int(seed))
        ro, col, _ = O.build_csr(int(n), s, d, w)
        depth, st, rl = O.bfs(int(n), ro, col, int(src))
        assert np.array_equal(depth, gold[f"depth_{(seed - 6000)}_{src}"])
        assert (st, rl) == (st_p, rl_p) == (st_q, rl_q)
        # C5: depths equal unit-weight Dijkstra
        unit, _ = O.dijkstra(int(n), ro, col, np.ones(len(col)), int(src), "f64")
        assert np.array_equal(depth, unit)
    assert gold["triangle"].tolist() == [0.0, 1.0, 1.0]  # test_algorithms.cpp:186-187
    assert gold["path"].tolist() == [0.0, 1.0, 2.0, 3.0]  # :189-191
    with pytest.raises(IndexError):
        O.bfs(3, np.array([0, 0, 0, 0], np.uint32), np.zeros(0, np.uint32), 3)


def test_pred_tree_checker_rejects_cycles_and_loose_edges():
    """orc_check_pred_tree (acceptance.cpp:56-91 semantics), linear version:
    a zero-weight tight cycle and a non-tight edge are both rejected."""
    nil = 0xFFFFFFFF
    ro = np.array([0, 2, 4, 5], np.uint32)
    col = np.array([1, 2, 0, 2, 1], np.uint32)
    w = np.array([1, 4, 5, 2, 0], np.float64)
    d = np.array([0, 1, 3], np.float64)
    assert O.check_pred_tree(3, ro, col, w, d, 0, np.array([nil, 0, 1], np.uint32)) == -1
    assert O.check_pred_tree(3, ro, col, w, d, 0, np.array([nil, 2, 1], np.uint32)) == 1
    w0 = np.array([1, 4, 5, 0, 0], np.float64)  # 1 <-> 2 both tight at distance 1
    d0 = np.array([0, 1, 1], np.float64)
    assert O.check_pred_tree(3, ro, col, w0, d0, 0, np.array([nil, 2, 1], np.uint32)) == 1
    assert O.check_pred_tree(3, ro, col, w0, d0, 0, np.array([nil, 0, 1], np.uint32)) == -1


def test_host_rmat_csr_matches_generator():
    """orc_rmat_csr (the CPU baseline's full-size input) == the edge generator
    sorted like build_csr (graph.hpp:144-147)."""
    for sc in (8, 13):
        ro, col, w = O.rmat_csr(sc, 16, 1, 1)
        s, dd, wb = O.rmat_edges(sc, 16, seed=1, wkind=1)
        order = np.lexsort((wb.view(np.float32), dd, s))
        want = np.concatenate([[0], np.cumsum(np.bincount(s, minlength=1 << sc))])
        assert np.array_equal(ro, want.astype(np.uint32))
        assert np.array_equal(col, dd[order])
        assert np.array_equal(w, wb.view(np.float32)[order])

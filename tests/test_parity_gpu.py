"""GPU parity: the sm_100a path (through the C ABI) against the oracle.

Mirrors the reference's own suites: test_algorithms.cpp (goldens, corpus,
degenerate cases, rejections, triangle inequality), acceptance.cpp C1/C3/C4
(200-graph oracle sweep, determinism, predecessor trees) and
test_operators.cpp (operator contracts), plus RMAT/grid configs.

Bars (BASELINE.json north_star): f64 and u32 distances bit-exact vs the
unmodified reference's arithmetic; f32 bit-exact vs the f32 restatement of
reference_dijkstra (tolerance 0 ulp).  Predecessors: dist[pred] + w == dist
in the device arithmetic, chains acyclic.
"""
import os

import numpy as np
import pytest

import paper_2212_08200_b200 as gb
from oracle import oracle as O

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
DIRS = ("push", "pull", "auto")


def triangle(ctx, wtype="f64"):
    return gb.build_csr([(0, 1, 1.0), (0, 2, 4.0), (1, 2, 2.0)], 3, wtype=wtype,
                        transpose=True, ctx=ctx)


def pred_ok(g, dist, pred, source=0, wtype="f64"):
    ro, col, w = g.csr()
    if wtype == "f32":
        return O.check_pred_tree(g.num_vertices, ro, col, w, dist.astype(np.float32), source,
                                 pred) == -1
    return O.check_pred_tree(g.num_vertices, ro, col, w.astype(np.float64), dist, source,
                             pred) == -1


# ------------------------------------------------------------ goldens ---

@pytest.mark.parametrize("wtype", ["f64", "f32", "u32"])
@pytest.mark.parametrize("direction", DIRS)
def test_triangle(ctx, wtype, direction):
    """test_algorithms.cpp:134-144: dist [0,1,3], pred [NIL,0,1]."""
    g = triangle(ctx, wtype)
    dist, pred, st, rl = gb.sssp(g, 0, direction=direction)
    assert list(dist) == [0.0, 1.0, 3.0]
    assert list(pred) == [gb.NIL, 0, 1]
    assert st >= 1 and rl >= 3


def test_triangle_as_lists(ctx):
    """module.cpp:115-128 binding shape: None for NIL."""
    d, p, _, _ = gb.sssp(triangle(ctx), 0, as_lists=True)
    assert d == [0.0, 1.0, 3.0] and p == [None, 0, 1]


def test_path_and_zero_weight(ctx):
    g = gb.build_csr([(0, 1, 1.0), (1, 2, 1.0), (2, 3, 1.0)], 4, ctx=ctx)
    assert list(gb.sssp(g, 0)[0]) == [0, 1, 2, 3]
    g = gb.build_csr([(0, 1, 0.0)], 2, ctx=ctx)
    d, p, _, _ = gb.sssp(g, 0)
    assert list(d) == [0, 0] and list(p) == [gb.NIL, 0]


def test_degenerate(ctx):
    """test_algorithms.cpp:146-156."""
    g = gb.build_csr([], 1, ctx=ctx)
    d, p, _, _ = gb.sssp(g, 0)
    assert list(d) == [0.0] and list(p) == [gb.NIL]
    g = gb.build_csr([(0, 1, 1.0)], 3, ctx=ctx)
    d, p, _, _ = gb.sssp(g, 0)
    assert np.isinf(d[2]) and p[2] == gb.NIL and d[1] == 1.0


def test_rejections(ctx):
    """test_algorithms.cpp:158-179 / algorithms.hpp:137-139."""
    g = gb.build_csr([(0, 1, 1.0), (0, 2, 4.0), (1, 2, 2.0)], 3, ctx=ctx)
    with pytest.raises(IndexError):
        gb.sssp(g, 9)
    with pytest.raises(ValueError):
        gb.sssp(g, 0, direction="pull")  # no transpose built
    with pytest.raises(ValueError):
        gb.sssp(g, 0, policy="par")
    with pytest.raises(ValueError):  # the queue (async) model is push-only
        gb.sssp(g, 0, frontier="queue", direction="pull")
    d, _, steps, _ = gb.sssp(g, 0, frontier="queue")  # runs as the device work queue
    assert list(d) == [0.0, 1.0, 3.0] and steps == 0


def test_upload_validation(ctx):
    """graph.hpp:134-142: invalid_argument naming the first offending edge."""
    with pytest.raises(ValueError, match="edge 1"):
        gb.Graph.from_csr(3, [0, 2, 2, 2], [1, 7], [1.0, 1.0], ctx=ctx)
    with pytest.raises(ValueError, match="edge 0"):
        gb.Graph.from_csr(3, [0, 1, 1, 1], [1], [-1.0], ctx=ctx)
    with pytest.raises(ValueError, match="edge 0"):
        gb.Graph.from_csr(3, [0, 1, 1, 1], [1], [np.inf], ctx=ctx)
    with pytest.raises(ValueError):
        gb.Graph.from_csr(3, [0, 2, 1, 2], [1, 2], [1.0, 1.0], ctx=ctx)
    with pytest.raises(ValueError):
        gb.Graph.from_csr(3, [0, 1, 1, 1], [1], [1.5], wtype="u32", ctx=ctx)


def test_negative_zero_weight_canonicalised(ctx):
    g = gb.build_csr([(0, 1, -0.0), (1, 2, 1.0)], 3, transpose=True, ctx=ctx)
    for direction in DIRS:
        d, p, _, _ = gb.sssp(g, 0, direction=direction)
        assert list(d) == [0.0, 0.0, 1.0] and not np.signbit(d[1])


# ------------------------------------------------------ corpus sweep ---

def _corpus_graph(i, corpus):
    row = corpus["meta"][i]
    n, seed = int(row[0]), int(row[1])
    s, d, w = O.random_edges(n, seed)
    return n, s, d, w


@pytest.fixture(scope="module")
def corpus():
    return np.load(os.path.join(GOLD, "corpus.npz"))


def test_oracle_sweep_f64_bit_exact(ctx, corpus):
    """acceptance.cpp:95-122 (C1 + C4): 200 graphs x {push, pull, auto},
    distances bit-exact vs the reference (golden digests + oracle), valid
    predecessor trees."""
    import hashlib
    for i in range(200):
        n, s, d, w = _corpus_graph(i, corpus)
        g = gb.build_csr((s, d, w), n, transpose=True, ctx=ctx)
        ro, col, val = g.csr()
        want, _ = O.dijkstra(n, ro, col, val, 0, "f64")
        h = hashlib.sha256(want.tobytes()).hexdigest()[:32]
        assert h == bytes(corpus[f"digest_dist_{i}"]).hex()
        for direction in DIRS:
            dist, pred, _, _ = gb.sssp(g, 0, direction=direction)
            assert np.array_equal(dist, want), (i, direction)
            assert O.check_pred_tree(n, ro, col, val, dist, 0, pred) == -1, (i, direction)


def test_oracle_sweep_f32_bit_exact(ctx, corpus):
    """Same corpus in the f32 bandwidth mode vs the f32 restatement."""
    for i in range(0, 200, 3):
        n, s, d, w = _corpus_graph(i, corpus)
        g = gb.build_csr((s, d, w), n, wtype="f32", transpose=True, ctx=ctx)
        ro, col, w32 = g.csr()
        want, _ = O.dijkstra(n, ro, col, w32, 0, "f32")
        for direction in DIRS:
            dist, pred, _, _ = gb.sssp(g, 0, direction=direction)
            assert np.array_equal(dist.astype(np.float32), want), (i, direction)
            assert pred_ok(g, dist, pred, wtype="f32"), (i, direction)


def test_corpus_nonzero_sources(ctx, corpus):
    for i in range(0, 40, 4):
        n, s, d, w = _corpus_graph(i, corpus)
        g = gb.build_csr((s, d, w), n, transpose=True, ctx=ctx)
        ro, col, val = g.csr()
        src = n // 2
        want, _ = O.dijkstra(n, ro, col, val, src, "f64")
        dist, pred, _, _ = gb.sssp(g, src)
        assert np.array_equal(dist, want)
        assert O.check_pred_tree(n, ro, col, val, dist, src, pred) == -1


def test_determinism_20_runs(ctx):
    """acceptance.cpp:157-177 (C3): random_graph(1000, 424242), 20 runs."""
    s, d, w = O.random_edges(1000, 424242)
    g = gb.build_csr((s, d, w), 1000, transpose=True, ctx=ctx)
    first = gb.sssp(g, 0)[0]
    for _ in range(19):
        assert np.array_equal(gb.sssp(g, 0)[0], first)


def test_triangle_inequality_at_fixpoint(ctx):
    """test_algorithms.cpp:202-211."""
    s, d, w = O.random_edges(200, 77)
    g = gb.build_csr((s, d, w), 200, ctx=ctx)
    dist = gb.sssp(g, 0)[0]
    ro, col, val = g.csr()
    src = np.repeat(np.arange(200), np.diff(ro))
    fin = np.isfinite(dist[src])
    assert np.all(dist[col[fin]] <= dist[src[fin]] + val[fin])


# ------------------------------------------------------ RMAT / grid ---

def test_rmat_generator_matches_oracle(ctx):
    """Device RMAT (rmat.cuh) == oracle restatement + build_csr layout."""
    for scale, wt, wk in ((10, "f32", 1), (12, "u32", 0)):
        g = gb.rmat(scale, 16, seed=1, wtype=wt, transpose=True, ctx=ctx)
        ro, col, w = g.csr()
        s, d, wb = O.rmat_edges(scale, 16, seed=1, wkind=wk)
        wv = wb.view(np.float32).astype(np.float64) if wk else wb.astype(np.float64)
        ro2, col2, val2 = O.build_csr(1 << scale, s, d, wv)
        assert np.array_equal(ro, ro2) and np.array_equal(col, col2)
        assert np.array_equal(w.astype(np.float64), val2)


def test_config1_rmat16_u32_bit_exact(ctx):
    """Config 1: device u32 distances widened to double == the reference's
    sssp() (par/push/sparse) on the same RMAT s16 graph, bit for bit."""
    gold = np.load(os.path.join(GOLD, "rmat16.npz"))
    g = gb.rmat(16, 16, seed=1, wtype="u32", transpose=True, ctx=ctx)
    for direction in DIRS:
        dist, pred, st, rl = gb.sssp(g, 0, direction=direction)
        assert np.array_equal(dist, gold["dist"]), direction
        assert pred_ok(g, dist, pred, wtype="f64")


def test_upload_equals_generate(ctx):
    """gfb_graph_upload of the reference CSR == the device-built graph."""
    g1 = gb.rmat(14, 16, seed=3, wtype="f32", transpose=True, ctx=ctx)
    ro, col, w = g1.csr()
    g2 = gb.Graph.from_csr(1 << 14, ro, col, w.astype(np.float64), wtype="f32", transpose=True,
                           ctx=ctx)
    d1 = gb.sssp(g1, 0)[0]
    d2 = gb.sssp(g2, 0)[0]
    assert np.array_equal(d1, d2)


@pytest.mark.parametrize("scale", [14, 18])
def test_rmat_f32_bit_exact(ctx, scale):
    g = gb.rmat(scale, 16, seed=1, wtype="f32", transpose=True, ctx=ctx)
    ro, col, w = g.csr()
    want, _ = O.dijkstra(g.num_vertices, ro, col, w, 0, "f32")
    for direction in DIRS:
        dist, pred, st, rl = gb.sssp(g, 0, direction=direction)
        assert np.array_equal(dist.astype(np.float32), want), direction
        assert pred_ok(g, dist, pred, wtype="f32")


def test_grid_f32_bit_exact(ctx):
    g = gb.grid(256, seed=1, transpose=True, ctx=ctx)
    ro, col, w = g.csr()
    ro2, col2, w2 = O.grid_csr(256, seed=1)
    assert np.array_equal(ro, ro2) and np.array_equal(col, col2) and np.array_equal(w, w2)
    want, _ = O.dijkstra(g.num_vertices, ro, col, w, 0, "f32")
    dist, pred, st, rl = gb.sssp(g, 0)
    assert np.array_equal(dist.astype(np.float32), want)
    assert pred_ok(g, dist, pred, wtype="f32")


@pytest.mark.slow
def test_rmat22_properties(ctx):
    """Full-size property checks (configs 2/3 scale): fixpoint (no edge can
    relax), tight acyclic predecessor tree, and n_reach/m_reach consistency."""
    g = gb.rmat(22, 16, seed=1, wtype="f32", transpose=True, ctx=ctx)
    dist, pred, st = gb.sssp_stats(g, 0)
    ro, col, w = g.csr()
    d32 = dist.astype(np.float32)
    src = np.repeat(np.arange(g.num_vertices, dtype=np.uint32), np.diff(ro))
    fin = np.isfinite(d32[src])
    nd = (d32[src[fin]] + w[fin]).astype(np.float32)
    assert np.all(d32[col[fin]] <= nd)
    reach = np.isfinite(d32)
    assert st.n_reach == reach.sum()
    assert st.m_reach == np.diff(ro)[reach].sum()
    assert O.check_pred_tree(g.num_vertices, ro, col, w, d32, 0, pred) == -1


# ------------------------------------------------- operator contracts ---

def test_push_visits_every_out_edge(ctx):
    """test_operators.cpp:31-37 + :39-55."""
    g = triangle(ctx)
    f = gb.Frontier("sparse", 3, ctx=ctx).assign([0])
    assert list(gb.neighbors_expand(g, f, "always").contents()) == [1, 2]
    assert gb.neighbors_expand(g, gb.Frontier("sparse", 3, ctx=ctx), "always").size() == 0
    assert gb.neighbors_expand(g, gb.Frontier("sparse", 3, ctx=ctx).assign([2]),
                               "always").size() == 0


def test_push_output_multiset_and_order(ctx):
    """test_operators.cpp:67-84: output multiset == concatenated adjacency;
    the device sparse output also keeps the sequential order."""
    s, d, w = O.random_edges(80, 21)
    g = gb.build_csr((s, d, w), 80, ctx=ctx)
    ro, col, _ = g.csr()
    fr = list(range(0, 80, 3))
    expected = [int(col[e]) for v in fr for e in range(ro[v], ro[v + 1])]
    out = gb.neighbors_expand(g, gb.Frontier("sparse", 80, ctx=ctx).assign(fr), "always")
    assert list(out.contents()) == expected


def test_exactly_once_per_frontier_occurrence(ctx):
    """test_operators.cpp:86-102: duplicates count once per occurrence."""
    s, d, w = O.random_edges(60, 33)
    g = gb.build_csr((s, d, w), 60, ctx=ctx)
    ro = g.csr()[0]
    fr, deg = [], 0
    for v in range(0, 60, 2):
        fr.append(v)
        if v % 4 == 0:
            fr.append(v)
        deg += (ro[v + 1] - ro[v]) * (2 if v % 4 == 0 else 1)
    rec = gb.Recorder(4096, ctx=ctx)
    gb.neighbors_expand(g, gb.Frontier("sparse", 60, ctx=ctx).assign(fr), rec)
    assert rec.read()[3] == deg


def test_dense_in_dense_out(ctx):
    g = triangle(ctx)
    out = gb.neighbors_expand(g, gb.Frontier("dense", 3, ctx=ctx).assign([0]), "always")
    assert out.repr == "dense" and list(out.contents()) == [1, 2]


def test_pull_contracts(ctx):
    """test_operators.cpp:128-149, :173-182."""
    g = triangle(ctx)
    out = gb.neighbors_expand_pull(g, gb.Frontier("dense", 3, ctx=ctx).assign([0]), "always")
    assert list(out.contents()) == [1, 2]
    assert gb.neighbors_expand_pull(g, gb.Frontier("dense", 3, ctx=ctx), "always").size() == 0
    g2 = gb.build_csr([(0, 2, 1.0), (1, 2, 1.0)], 3, transpose=True, ctx=ctx)
    out = gb.neighbors_expand_pull(g2, gb.Frontier("dense", 3, ctx=ctx).assign([0, 1]), "always")
    assert list(out.contents()) == [2]
    with pytest.raises(ValueError):
        gb.neighbors_expand_pull(gb.build_csr([(0, 1, 1.0)], 2, ctx=ctx),
                                 gb.Frontier("dense", 2, ctx=ctx), "always")
    with pytest.raises(ValueError):
        gb.neighbors_expand_pull(g, gb.Frontier("sparse", 3, ctx=ctx), "always")


def test_push_pull_eligibility_equals_reference(ctx):
    """test_operators.cpp:151-171: recorded (src,dst,edge) sets of push and
    pull are identical and equal the reference's (golden ops.npz)."""
    ops = np.load(os.path.join(GOLD, "ops.npz"))
    for seed in (1, 2, 3, 4, 5):
        s, d, w = O.random_edges(40, seed)
        g = gb.build_csr((s, d, w), 40, transpose=True, ctx=ctx)
        fr = list(range(0, 40, 2))
        sets = []
        for pull in (0, 1):
            rec = gb.Recorder(4096, ctx=ctx)
            f = gb.Frontier("dense", 40, ctx=ctx).assign(fr)
            (gb.neighbors_expand_pull if pull else gb.neighbors_expand)(g, f, rec)
            a, b, c, cnt = rec.read()
            sets.append(sorted(zip(a.tolist(), b.tolist(), c.tolist())))
            ref = ops[f"rec_{seed}_{pull}"]
            assert sets[-1] == sorted(map(tuple, ref.T.tolist()))
        assert sets[0] == sets[1]


def test_operator_level_sssp_composition(ctx):
    """sssp() as the reference composes it (algorithms.hpp:164-183): a host
    loop of device neighbors_expand calls with relax_min reaches the oracle."""
    s, d, w = O.random_edges(300, 5)
    g = gb.build_csr((s, d, w), 300, transpose=True, ctx=ctx)
    ro, col, val = g.csr()
    want, _ = O.dijkstra(300, ro, col, val, 0)
    for repr_, pull in (("sparse", False), ("dense", False), ("dense", True)):
        dm = gb.DistanceMap(g, 0)
        f = gb.Frontier(repr_, 300, ctx=ctx).assign([0])
        steps = 0
        while f.size():
            steps += 1
            f = (gb.neighbors_expand_pull if pull else gb.neighbors_expand)(g, f, dm)
        dist, relax = dm.read()
        assert np.array_equal(dist, want), (repr_, pull)
        assert relax > 0 and steps > 1


def test_uniquify(ctx):
    """test_operators.cpp:212-233: ascending, duplicate-free."""
    f = gb.Frontier("sparse", 10, ctx=ctx).assign([5, 3, 5, 1, 3, 9])
    assert list(gb.uniquify(f).contents()) == [1, 3, 5, 9]
    assert gb.uniquify(gb.Frontier("sparse", 10, ctx=ctx)).size() == 0
    with pytest.raises(ValueError):
        gb.uniquify(gb.Frontier("dense", 10, ctx=ctx))


def test_frontier_semantics(ctx):
    """frontier.hpp / test_frontier.cpp:19-53: sparse counts duplicates,
    dense does not and reads back ascending; out-of-range add throws."""
    sp = gb.Frontier("sparse", 100, ctx=ctx).assign([7, 7, 3])
    dn = gb.Frontier("dense", 100, ctx=ctx).assign([7, 7, 3, 64, 99])
    assert sp.size() == 3 and list(sp.contents()) == [7, 7, 3]
    assert dn.size() == 4 and list(dn.contents()) == [3, 7, 64, 99]
    with pytest.raises(IndexError):
        gb.Frontier("sparse", 10, ctx=ctx).assign([10])


# ------------------------------------ f64 host weights into an f32 graph ---

def _big_csr(n=1 << 16, deg=24, seed=5):
    """m = 1.5 M edges: above graph.cu's HOST_NARROW_MIN_EDGES (f64 weights are
    narrowed on the host, a slice per thread, before the H2D copy)."""
    rng = np.random.default_rng(seed)
    ro = np.arange(0, n * deg + 1, deg, dtype=np.uint32)
    col = rng.integers(0, n, n * deg, dtype=np.uint32)
    w = rng.random(n * deg)  # doubles, most not representable in f32
    return n, ro, col, w


def test_host_narrowed_upload_equals_device_conversion(ctx):
    """The narrowed upload rounds like the device conversion (to nearest), so
    the device CSR equals an upload of the same weights already rounded."""
    n, ro, col, w = _big_csr()
    w[7] = -0.0  # canonicalised to +0.0
    w[9] = 3.4e38  # finite in f32
    g = gb.Graph.from_csr(n, ro, col, w, wtype="f32", ctx=ctx)
    g32 = gb.Graph.from_csr(n, ro, col, w.astype(np.float32) + np.float32(0), wtype="f32", ctx=ctx)
    r1, c1, w1 = g.csr()
    r2, c2, w2 = g32.csr()
    assert np.array_equal(r1, r2) and np.array_equal(c1, c2)
    assert np.array_equal(w1.view(np.uint32), w2.view(np.uint32))
    assert not np.signbit(w1[7])
    d, p, _, _ = gb.sssp(g, 0)
    d2, p2, _, _ = gb.sssp(g32, 0)
    assert np.array_equal(d, d2)


@pytest.mark.parametrize("bad", [-1e-50, np.nan, np.inf, 1e300, -2.0])
def test_host_narrowed_upload_validation(ctx, bad):
    """Same first-offending-edge message as the device path (graph.hpp:134-142);
    1e300 is finite as a double but rounds to +inf in f32: rejected like the
    device conversion does; the refill path checks the same rules."""
    n, ro, col, w = _big_csr()
    at = 1_234_567
    w[at] = bad
    w[at + 100] = -1.0
    with pytest.raises(ValueError, match=f"edge {at} has negative or non-finite weight"):
        gb.Graph.from_csr(n, ro, col, w, wtype="f32", ctx=ctx)
    n, ro, col, w_ok = _big_csr()
    g = gb.Graph.from_csr(n, ro, col, w_ok, wtype="f32", ctx=ctx)
    with pytest.raises(ValueError, match=f"edge {at} has negative or non-finite weight"):
        g.refill(ro, col, w)
    g.refill(ro, col, w_ok)  # a good refill clears the poisoned state
    gb.sssp(g, 0)


def test_host_narrowed_upload_keeps_f32_denormals(ctx):
    """Weights in the f32 denormal range round like __double2float_rn even when
    the process runs with flush-to-zero (the narrowing pins its own MXCSR)."""
    n, ro, col, w = _big_csr()
    w[:1000] = np.ldexp(1.0, -140) * (1 + np.arange(1000) / 997.0)  # f32 denormals
    g = gb.Graph.from_csr(n, ro, col, w, wtype="f32", ctx=ctx)
    _, _, w1 = g.csr()
    want = w[:1000].astype(np.float32)
    assert np.all(want > 0)
    assert np.array_equal(w1[:1000].view(np.uint32), want.view(np.uint32))

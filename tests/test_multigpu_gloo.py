"""Multi-rank partitioned SSSP on CPU with the gloo backend.

Exercises the host-side logic of paper_2212_08200_b200/mg.py -- edge-balanced
1-D ranges, per-owner message grouping, the all-to-all exchange protocol,
allreduce convergence and the allreduce(MIN) predecessor election -- with
world_size 2 and 3, against the oracle (f32 Dijkstra restatement)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2212_08200_b200 import mg


def _graph(scale=9, seed=3):
    s, d, wb = O.rmat_edges(scale, 16, seed=seed, wkind=1)
    n = 1 << scale
    ro, col, val = O.build_csr(n, s, d, wb.view(np.float32).astype(np.float64))
    return n, ro, col, val.astype(np.float32)


def test_edge_balanced_ranges_balance_rmat_edges():
    n, ro, col, w = _graph(scale=12)
    m = int(ro[-1])
    for parts in (2, 4, 8):
        rs = mg.edge_balanced_ranges(ro, parts)
        assert rs[0] == 0 and rs[-1] == n and np.all(np.diff(rs.astype(np.int64)) >= 0)
        share = np.diff(ro[rs].astype(np.int64)) / m
        assert share.max() < 1.0 / parts + 0.05, share
        eq = mg.equal_vertex_ranges(n, parts)
        assert (ro[eq[1]] - ro[eq[0]]) / m > 1.5 / parts  # rank 0 overloaded (hub)


def test_slice_and_owner():
    n, ro, col, w = _graph(scale=8)
    rs = mg.edge_balanced_ranges(ro, 3)
    total = 0
    for p in range(3):
        rl, c, ww = mg.slice_csr(ro, col, w, rs[p], rs[p + 1])
        assert rl[0] == 0 and rl[-1] == len(c) == len(ww)
        total += len(c)
    assert total == len(col)
    assert list(mg.owner_of(np.array([0, rs[1] - 1, rs[1], n - 1]), rs)) == [0, 0, 1, 2]


def test_single_process_simulation_matches_oracle():
    n, ro, col, w = _graph(scale=9)
    rs = mg.edge_balanced_ranges(ro, 4)
    engines = [mg.CpuPart(n, int(rs[p]), int(rs[p + 1]), *mg.slice_csr(ro, col, w, rs[p], rs[p + 1]))
               for p in range(4)]
    got, steps = mg.sssp_simulated(engines, rs, 0)
    want, _ = O.dijkstra(n, ro, col, w, 0, "f32")
    assert np.array_equal(got, want) and steps > 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, ro, col, w = _graph(scale=9)
        rs = mg.edge_balanced_ranges(ro, world)
        lo, hi = int(rs[rank]), int(rs[rank + 1])
        eng = mg.CpuPart(n, lo, hi, *mg.slice_csr(ro, col, w, lo, hi))
        d, pred, st = mg.sssp_partitioned(eng, rs, 0, want_pred=True)
        q.put((rank, d, pred, st))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_partitioned_sssp_matches_oracle(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, d, pred, st = q.get(timeout=300)
        out[r] = (d, pred, st)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n, ro, col, w = _graph(scale=9)
    dist = np.concatenate([out[r][0] for r in range(world)])
    pred = np.concatenate([out[r][1] for r in range(world)])
    want, _ = O.dijkstra(n, ro, col, w, 0, "f32")
    assert np.array_equal(dist, want)
    assert O.check_pred_tree(n, ro, col, w, dist, 0, pred) == -1
    assert out[0][2]["messages_sent"] + out[1][2]["messages_sent"] > 0


def test_peer_aligned_ranges():
    """peer.aligned_ranges: 32-aligned interior cuts, ascending, covering [0, n)."""
    from paper_2212_08200_b200 import peer
    rng = np.random.default_rng(5)
    for n in (1, 31, 32, 1000, 4097):
        deg = rng.integers(0, 50, size=n)
        ro = np.concatenate([[0], np.cumsum(deg)]).astype(np.uint32)
        for parts in range(1, 9):
            rs = peer.aligned_ranges(ro, parts)
            assert len(rs) == parts + 1 and rs[0] == 0 and rs[-1] == n
            assert np.all(np.diff(rs.astype(np.int64)) >= 0)
            assert all(int(c) % 32 == 0 for c in rs[1:-1])
    with pytest.raises(ValueError):
        peer.aligned_ranges(np.zeros(2, np.uint32), 9)

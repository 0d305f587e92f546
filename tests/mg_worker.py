"""gfb_mg_* parity in one process (test_peer_gpu.py::test_mg_one_process):
python tests/mg_worker.py PARTS -- all partitions on device 0."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)
import peer_worker as W  # noqa: E402
from paper_2212_08200_b200 import peer  # noqa: E402


def main():
    parts = int(sys.argv[1])
    for name, (n, ro, col, w), sources in [("rmat13-f32", W.rmat(13, 1, 1), [0, 8000]),
                                           ("rmat12-u32", W.rmat(12, 0, 2), [0, 77]),
                                           ("grid48-f32", W.grid(48, 3), [0, 2000]),
                                           ("corpus-f32", W.corpus(300, 9001), [0, 5])]:
        mg = peer.MgSssp([0] * parts, ro, col, w)
        rs = mg.ranges()
        assert rs[0] == 0 and rs[-1] == n and all(int(c) % 32 == 0 for c in rs[1:-1])
        for src in sources:
            for _ in range(2):
                d, p, st = mg.sssp(src)
                W.check(name, n, ro, col, w, src, d, p, 0)
                fin = np.isfinite(d)
                assert st["n_reach"] == int(fin.sum())
                assert st["m_reach"] == int(np.diff(ro.astype(np.int64))[fin].sum())
        try:
            mg.sssp(n)
            raise AssertionError("source out of range accepted")
        except IndexError:
            pass
        mg.free()
    edge_cases(parts)
    relabelled(parts)
    print(f"MG_OK parts {parts}", flush=True)


def relabelled(parts):
    """The partitioned path on a range-preserving relabelled copy
    (gfb_graph_relabel_ranges, what bench.py --gpus N runs on): distances map
    back to the oracle's on the original graph."""
    import paper_2212_08200_b200 as gb
    n, ro, col, w = W.rmat(13, 1, 5)
    g = gb.Graph.from_csr(n, ro, col, w, wtype="f32")
    rs = peer.aligned_ranges(ro, parts)
    ro2, col2, w2, perm = peer.relabel_ranges(g, rs)
    g.free()
    mg = peer.MgSssp([0] * parts, ro2, col2, w2)
    for src in (0, n - 1):
        d2, p2, _ = mg.sssp(int(perm[src]))
        d, p = peer.unrelabel(perm, d2, p2)
        W.check("rmat13-relabelled", n, ro, col, w, src, d, p, 0)
    mg.free()




def edge_cases(parts):
    """No edges at all, and a graph whose edges all live in one partition."""
    n = 200
    ro = np.zeros(n + 1, np.uint32)
    mg = peer.MgSssp([0] * parts, ro, np.zeros(0, np.uint32), np.zeros(0, np.float32))
    d, p, st = mg.sssp(5)
    assert d[5] == 0 and np.isinf(np.delete(d, 5)).all() and (p == 0xFFFFFFFF).all()
    mg.free()
    # a path 0 -> 1 -> ... -> 9 (rows 0..9 only), u32 weights
    ro = np.concatenate([np.arange(10, dtype=np.uint32), np.full(n - 9, 9, np.uint32)])
    col = np.arange(1, 10, dtype=np.uint32)
    w = np.full(9, 3, np.uint32)
    mg = peer.MgSssp([0] * parts, ro, col, w)
    d, p, st = mg.sssp(0)
    assert d[:10].tolist() == [3.0 * i for i in range(10)] and np.isinf(d[10:]).all()
    assert p[1:10].tolist() == list(range(9))
    mg.free()


if __name__ == "__main__":
    main()

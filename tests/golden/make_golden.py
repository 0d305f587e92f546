"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Runs only in the build container (needs oracle/_ref/libgraflow_ref.so, which
oracle/Makefile compiles from /root/reference/proj/include + tests/).  The
fixtures are small and committed; the GPU box never reads /root/reference.

  corpus.npz   acceptance.cpp:95-122 oracle sweep: 200 graphs
               random_graph(2 + mt19937_64(2024)() % 499, 9000 + i); per
               instance the edge-list digest, the reference_dijkstra distance
               digest, and the reference sssp() seq/push/sparse and
               seq/push/dense supersteps + relaxations.  The first 24
               instances are stored in full (edges + distances).
  rmat16.npz   config 1: RMAT s16 EF16 u32 U{0..255}, source 0; reference
               sssp() (par, push, sparse: the CLI default) and
               reference_dijkstra() distances (full) + stats.
  bfs.npz      acceptance.cpp:180-199 (C5): 50 graphs random_edges(5 + 7i,
               6000 + i), transpose built; the reference bfs() depth,
               supersteps, relaxations for seq/push/sparse and seq/pull/dense
               (sources 0 and n/2), plus the hand-checked graphs of
               test_algorithms.cpp:185-192.
  ops.npz      operator contracts on random_graph(40, seed) seeds 1..5:
               push and pull recorded (src, dst, edge) triples of the
               reference's own neighbors_expand / neighbors_expand_pull.
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
from oracle import oracle as O  # noqa: E402


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:32]


def mt_sizes(count):
    """acceptance.cpp:98-101: n = 2 + mt19937_64(2024)() % 499 (restated RNG)."""
    import ctypes as C
    L = O.orc()
    L.orc_mt64_next.restype = C.c_uint64
    state = C.create_string_buffer(312 * 8 + 16)  # orc_mt64
    L.orc_mt64_seed(state, C.c_uint64(2024))
    return [2 + L.orc_mt64_next(state) % 499 for _ in range(count)]


def main():
    assert O.ref() is not None, "build oracle/_ref first (make -C oracle)"
    # ---- corpus (acceptance C1 + C4) ----
    sizes = mt_sizes(200)
    rows = []
    full = {}
    for i, n in enumerate(sizes):
        s, d, w = O.ref_random_edges(n, 9000 + i)
        g = O.RefGraph(n, s, d, w, transpose=True)
        dist, _ = g.dijkstra(0)
        _, _, st_sp, rl_sp = g.sssp(0, mode=0, workers=1, direction=0, repr_=0)
        _, _, st_dn, rl_dn = g.sssp(0, mode=0, workers=1, direction=0, repr_=1)
        rows.append((n, 9000 + i, len(s), st_sp, rl_sp, st_dn, rl_dn))
        full[f"digest_edges_{i}"] = np.frombuffer(bytes.fromhex(digest(s, d, w)), np.uint8)
        full[f"digest_dist_{i}"] = np.frombuffer(bytes.fromhex(digest(dist)), np.uint8)
        if i < 24:
            full[f"src_{i}"], full[f"dst_{i}"], full[f"w_{i}"] = s, d, w
            full[f"dist_{i}"] = dist
    full["meta"] = np.array(rows, dtype=np.uint64)
    np.savez_compressed(os.path.join(HERE, "corpus.npz"), **full)

    # ---- config 1: RMAT s16 u32 ----
    s, d, wb = O.rmat_edges(16, 16, seed=1, wkind=0)
    g = O.RefGraph(1 << 16, s, d, wb.astype(np.float64), transpose=False)
    dist, pred, st, rl = g.sssp(0, mode=1, workers=8, direction=0, repr_=0)
    ddist, _ = g.dijkstra(0)
    ro, col, val = g.csr()
    np.savez_compressed(os.path.join(HERE, "rmat16.npz"), dist=dist, dijkstra=ddist,
                        supersteps=st, csr_digest=np.frombuffer(
                            bytes.fromhex(digest(ro, col, val)), np.uint8),
                        edge_digest=np.frombuffer(bytes.fromhex(digest(s, d, wb)), np.uint8))

    # ---- bfs (acceptance C5) ----
    bfs = {}
    rows = []
    for i in range(50):
        n = 5 + 7 * i
        s, d, w = O.ref_random_edges(n, 6000 + i)
        g = O.RefGraph(n, s, d, w, transpose=True)
        for src in (0, n // 2):
            dp, st_p, rl_p = g.bfs(src, mode=0, workers=1, direction=0, repr_=0)
            dq, st_q, rl_q = g.bfs(src, mode=0, workers=1, direction=1, repr_=1)
            assert np.array_equal(dp, dq)
            rows.append((n, 6000 + i, src, st_p, rl_p, st_q, rl_q))
            bfs[f"depth_{i}_{src}"] = dp
    bfs["meta"] = np.array(rows, dtype=np.uint64)
    tri = O.RefGraph(3, np.array([0, 0, 1], np.uint32), np.array([1, 2, 2], np.uint32),
                     np.array([1.0, 4.0, 2.0]))
    bfs["triangle"] = tri.bfs(0)[0]
    path = O.RefGraph(4, np.array([0, 1, 2], np.uint32), np.array([1, 2, 3], np.uint32),
                      np.array([5.0, 0.5, 2.0]))
    bfs["path"] = path.bfs(0, mode=1, workers=2)[0]
    np.savez_compressed(os.path.join(HERE, "bfs.npz"), **bfs)

    # ---- operator contracts ----
    ops = {}
    for seed in (1, 2, 3, 4, 5):
        s, d, w = O.ref_random_edges(40, seed)
        g = O.RefGraph(40, s, d, w, transpose=True)
        f = np.arange(0, 40, 2, dtype=np.uint32)
        for pull in (0, 1):
            a, b, c = g.expand_record(f, pull)
            ops[f"rec_{seed}_{pull}"] = np.stack([a, b, c])
    np.savez_compressed(os.path.join(HERE, "ops.npz"), **ops)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()

"""One rank of the peer-memory partitioned SSSP parity run (test_peer_gpu.py).

Launched by torchrun with any world size (1..8); several ranks may share one
GPU (CUDA IPC between processes on one device).  Every rank builds the same
graphs on the host (oracle generators), keeps its edge-balanced slice, runs
gfb_peer_sssp, gathers the whole result and checks it against the oracle:
distances bit-exact (f32 Dijkstra restatement / u32 integer Dijkstra),
predecessor trees valid (acceptance.cpp:56-91 rules).  Prints PEER_OK.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_08200_b200 as gb  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2212_08200_b200 import mg, peer  # noqa: E402


def rmat(scale, wkind, seed):
    s, d, wb = O.rmat_edges(scale, 16, seed=seed, wkind=wkind)
    n = 1 << scale
    wv = wb.view(np.float32).astype(np.float64) if wkind else wb.astype(np.float64)
    ro, col, val = O.build_csr(n, s, d, wv)
    return n, ro, col, (val.astype(np.float32) if wkind else val.astype(np.uint32))


def grid(side, seed):
    g = gb.grid(side, seed=seed, transpose=False)
    ro, col, w = g.csr()
    n = g.num_vertices
    g.free()
    return n, ro, col, w.astype(np.float32)


def corpus(n, seed):
    s, d, w = O.random_edges(n, seed)
    ro, col, val = O.build_csr(n, np.asarray(s), np.asarray(d), np.asarray(w, np.float64))
    return n, ro, col, val.astype(np.float32)


def check(name, n, ro, col, w, src, dist_, pred, rank):
    if w.dtype == np.float32:
        want, _ = O.dijkstra(n, ro, col, w, src, "f32")
        ok = np.array_equal(dist_.astype(np.float32), want)
        tree = O.check_pred_tree(n, ro, col, w, dist_.astype(np.float32), src, pred)
    else:
        want, _ = O.dijkstra(n, ro, col, w.astype(np.float64), src, "f64")
        ok = np.array_equal(dist_, want)
        tree = O.check_pred_tree(n, ro, col, w.astype(np.float64), dist_, src, pred)
    if not ok or tree != -1:
        bad = np.flatnonzero(dist_.astype(np.float64) != np.asarray(want, np.float64))[:5]
        raise AssertionError(f"[rank {rank}] {name} src {src}: dist_equal={ok} pred_tree={tree} "
                             f"first bad {bad.tolist()}")


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dev = local % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ctx = gb.Context(dev)
    cases = [("rmat13-f32", rmat(13, 1, 1), [0, None]),
             ("rmat12-u32", rmat(12, 0, 2), [0, 77]),
             ("grid48-f32", grid(48, 3), [0, None]),
             ("corpus-f32", corpus(300, 9001), [0, 5])]
    steps = []
    for name, (n, ro, col, w), sources in cases:
        rs = peer.aligned_ranges(ro, world)
        lo, hi = int(rs[rank]), int(rs[rank + 1])
        p = peer.PeerSssp(rank, world, rs, *mg.slice_csr(ro, col, w, lo, hi), ctx=ctx)
        p.link()
        for src in sources:
            if src is None:  # a source owned by the last rank
                src = int(rs[-2]) + 1 if world > 1 and rs[-2] + 1 < n else n - 1
            for rep in range(2):  # reuse of the captured loop graph
                st = p.sssp(src)
                d, pr = peer.gather(p)
                check(name, n, ro, col, w, src, d, pr, rank)
                tot = torch.tensor([st["relaxations"], st["n_reach"], st["m_reach"]],
                                   dtype=torch.int64)
                dist.all_reduce(tot)
                fin = np.isfinite(d)
                m_reach = int(np.diff(ro.astype(np.int64))[fin].sum())
                assert int(tot[1]) == int(fin.sum()), (name, int(tot[1]), int(fin.sum()))
                assert int(tot[2]) == m_reach, (name, int(tot[2]), m_reach)
                steps.append(st["supersteps"])
        dist.barrier()
        p.free()
    dist.barrier()
    print(f"PEER_OK rank {rank} world {world} supersteps {steps}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

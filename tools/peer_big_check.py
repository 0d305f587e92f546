"""Peer-memory partitioned SSSP at RMAT s18 (f32 and u32: cross-rank tie repair at
scale), checked against the oracle; run under torchrun (world 2+; ranks may share a GPU)."""
import os, sys
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2212_08200_b200 as gb
from paper_2212_08200_b200 import mg, peer
import peer_worker as W
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("gloo", rank=rank, world_size=world)
ctx = gb.Context(0)
for name, (n, ro, col, w) in (("rmat18-f32", W.rmat(18, 1, 1)), ("rmat18-u32", W.rmat(18, 0, 2))):
    rs = peer.aligned_ranges(ro, world)
    lo, hi = int(rs[rank]), int(rs[rank + 1])
    p = peer.PeerSssp(rank, world, rs, *mg.slice_csr(ro, col, w, lo, hi), ctx=ctx)
    p.link()
    for src in (0, n - 5):
        st = p.sssp(src)
        d, pr = peer.gather(p)
        W.check(name, n, ro, col, w, src, d, pr, rank)
        if rank == 0:
            print(name, src, "ok supersteps", st["supersteps"], "fallback", st["pred_fallback"], flush=True)
    dist.barrier()
    p.free()
print("BIG_OK", rank, flush=True)
dist.destroy_process_group()

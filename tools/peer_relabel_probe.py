"""Does the partitioned (peer) path gain from an in-degree-relabelled CSR
with destination-sorted rows, like the single-GPU loop?  World size 1:
the same s24 graph as given and relabelled (the single-GPU library's own
relabelled copy, gfb_debug_relabel).  python tools/peer_relabel_probe.py"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2212_08200_b200 as gb  # noqa: E402
from paper_2212_08200_b200 import _lib, mg, peer  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29678")
dist.init_process_group("gloo", rank=0, world_size=1)
ctx = gb.Context(0)
g = gb.rmat(24, 16, seed=1, wtype="f32", transpose=False, ctx=ctx)
ro, col, w = g.csr()
n, m = g.num_vertices, g.num_edges
gb.sssp_stats(g, 0, want_result=False, relabel="on")  # builds the relabelled copy
ro2 = np.zeros(n + 1, np.uint32)
adj = np.zeros(2 * m, np.uint32)
assert _lib.load().gfb_debug_relabel(g.h, C.c_void_p(ro2.ctypes.data), C.c_void_p(adj.ctypes.data),
                                     None) == 0
col2, w2 = adj[0::2].copy(), adj[1::2].view(np.float32).copy()
del adj
g.free()
for name, (r, c, ww) in (("given", (ro, col, w)), ("relabelled", (ro2, col2, w2))):
    rs = peer.aligned_ranges(r, 1)
    p = peer.PeerSssp(0, 1, rs, *mg.slice_csr(r, c, ww, 0, n), ctx=ctx)
    p.link()
    for dp in (10, 5, 3):
        ms = []
        for i in range(8):
            st = p.sssp(0, defer_pct=dp)
            if i > 1:
                ms.append(st["device_ms"])
        print(f"{name} defer {dp}%: median {np.median(ms):.3f} ms, supersteps "
              f"{st['supersteps']}, relax {st['relaxations']}", flush=True)
    p.free()
dist.destroy_process_group()

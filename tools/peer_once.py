"""Run the peer-memory partitioned SSSP once per call at world size 1 (for ncu
launch lists): python tools/peer_once.py SCALE RUNS"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch.distributed as dist  # noqa: E402

import paper_2212_08200_b200 as gb  # noqa: E402
from paper_2212_08200_b200 import mg, peer  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 2
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29677")
dist.init_process_group("gloo", rank=0, world_size=1)
ctx = gb.Context(0)
g = gb.rmat(scale, 16, seed=1, wtype="f32", transpose=False, ctx=ctx)
ro, col, w = g.csr()
g.free()
rs = peer.aligned_ranges(ro, 1)
p = peer.PeerSssp(0, 1, rs, *mg.slice_csr(ro, col, w, 0, len(ro) - 1), ctx=ctx)
p.link()
for _ in range(runs):
    st = p.sssp(0)
    print(f"device_ms {st['device_ms']:.3f} supersteps {st['supersteps']} "
          f"relax {st['relaxations']} fallback {st['pred_fallback']}", flush=True)
p.free()
dist.destroy_process_group()

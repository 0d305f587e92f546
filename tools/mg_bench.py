"""Partitioned SSSP in one process (gfb_mg_*), P partitions on device 0:
python tools/mg_bench.py SCALE P1,P2,...  (set CUDA_DEVICE_MAX_CONNECTIONS=32).
All partitions share one GPU, so the device time measures the protocol's
overhead against the single-GPU loop, not multi-GPU scaling."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2212_08200_b200 as gb  # noqa: E402
from paper_2212_08200_b200 import peer  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
plist = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,2,4").split(",")]
ctx = gb.Context(0)
g = gb.rmat(scale, 16, seed=1, wtype="f32", transpose=False, ctx=ctx)
ro, col, w = g.csr()
_, _, st0 = gb.sssp_stats(g, 0, want_result=False, direction="push")
ts = []
for _ in range(5):
    _, _, st0 = gb.sssp_stats(g, 0, want_result=False, direction="push")
    ts.append(st0.device_ms)
print(json.dumps({"single_gpu_ms": float(np.median(ts)), "m_reach": st0.m_reach}), flush=True)
g.free()
for P in plist:
    t0 = time.time()
    mg = peer.MgSssp([0] * P, ro, col, w)
    setup = time.time() - t0
    mg.sssp(0)
    ts = []
    for _ in range(5):
        _, _, st = mg.sssp(0, want_pred=True)
        ts.append(st["device_ms"])
    print(json.dumps({"parts": P, "ms": float(np.median(ts)), "supersteps": st["supersteps"],
                      "relax": st["relaxations"], "m_reach": st["m_reach"],
                      "launches": st["kernel_launches"], "setup_s": round(setup, 2)}), flush=True)
    mg.free()

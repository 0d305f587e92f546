"""BASELINE configs[4] (RMAT s26 EF16 fp32, 1.07 B edges) through the
partitioned SSSP with 8 partitions on ONE GPU (gfb_mg_*, peer-memory
exchange, one process), checked the way bench.py checks the single-GPU s26
line: dist[source] = 0, no edge can still relax in f32, tight acyclic
predecessor tree -- plus bit-equality with the single-GPU loop's distances.
Needs CUDA_DEVICE_MAX_CONNECTIONS=32.  python tools/s26_partitioned_check.py [scale] [parts]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2212_08200_b200 as gb  # noqa: E402
from paper_2212_08200_b200 import peer  # noqa: E402
from bench import sp_certificate  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
parts = int(sys.argv[2]) if len(sys.argv) > 2 else 8
ctx = gb.Context(0)
t0 = time.time()
g = gb.rmat(scale, 16, seed=1, wtype="f32", transpose=False, ctx=ctx)
d1, p1, st1 = gb.sssp_stats(g, 0, direction="push")
ro, col, w = g.csr()
ro, col, w = ro.copy(), col.copy(), w.copy()
g.free()
mg = peer.MgSssp([0] * parts, ro, col, w)
mg.sssp(0)
ts = []
for _ in range(3):
    d8, p8, st = mg.sssp(0, want_pred=True)
    ts.append(st["device_ms"])
mg.free()
d32 = d8.astype(np.float32)
cert = sp_certificate(ro, col, w, d32, p8, 0)
out = {"config": f"RMAT s{scale} EF16 fp32, source 0, {parts} partitions on one GPU (gfb_mg_*, peer exchange)",
       "m": int(len(col)), "parts": parts, "device_ms": float(np.median(ts)),
       "supersteps": st["supersteps"], "m_reach": st["m_reach"],
       "single_gpu_ms": st1.device_ms,
       "dist_equal_single_gpu": bool(np.array_equal(d8, d1)),
       "certificate": cert, "wall_s": round(time.time() - t0, 1),
       "note": "partitions share one GPU: the time measures the protocol, not multi-GPU scaling"}
print(json.dumps(out), flush=True)

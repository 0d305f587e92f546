"""Device BFS on RMAT (python tools/bfs_time.py SCALE): median wall time of
gfb_bfs without the depth download (host-synchronous call), GTEPS."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2212_08200_b200 as gb  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
g = gb.rmat(scale, 16, seed=1, wtype="f32", transpose=True)
for direction in ("push", "auto", "pull"):
    for _ in range(3):
        gb.bfs(g, 0, direction=direction, want_result=False)
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        _, st, rl = gb.bfs(g, 0, direction=direction, want_result=False)
        ts.append((time.perf_counter() - t0) * 1e3)
    ms = float(np.median(ts))
    print(json.dumps({"scale": scale, "direction": direction, "ms": ms, "supersteps": st,
                      "relaxations": rl, "gteps": rl / (ms * 1e-3) / 1e9}))

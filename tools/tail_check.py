"""Tail kernel on/off timings: RMAT s22/s24 (default BSP loop) and a 2048^2
grid on the BSP loop (loop="bsp"), device loop, median of N calls."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2212_08200_b200 as gb  # noqa: E402

ctx = gb.Context(0)
cases = [("rmat22", lambda: gb.rmat(22, 16, seed=1, wtype="f32", ctx=ctx), {}),
         ("rmat24", lambda: gb.rmat(24, 16, seed=1, wtype="f32", ctx=ctx), {}),
         ("grid2048_bsp", lambda: gb.grid(2048, seed=1, ctx=ctx), {"loop": "bsp"})]
for name, make, kw in cases:
    g = make()
    for tail in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else '-1,0').split(',')]:
        for _ in range(3):
            gb.sssp_stats(g, 0, want_result=False, tail_edges=tail, **kw)
        ms = []
        for _ in range(7):
            _, _, st = gb.sssp_stats(g, 0, want_result=False, tail_edges=tail, **kw)
            ms.append(st.device_ms)
        print(json.dumps({"case": name, "tail_edges": tail, "median_ms": float(np.median(ms)),
                          "supersteps": st.supersteps, "relaxations": st.relaxations}), flush=True)
    del g

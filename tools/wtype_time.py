"""SSSP device time per arithmetic (python tools/wtype_time.py SCALE)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_08200_b200 as gb  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
g32 = gb.rmat(scale, 16, seed=1, wtype="f32", transpose=False)
ro, col, w = g32.csr()
n = g32.num_vertices
g32.free()
for wt in ("f64", "u32", "f32"):
    if wt == "u32":
        g = gb.rmat(scale, 16, seed=1, wtype="u32", transpose=False)
    else:  # the same f32 weights, f64 arithmetic for "f64" (exact widening)
        g = gb.Graph.from_csr(n, ro, col, w.astype("float64"), wtype=wt)
    ms = []
    for i in range(8):
        _, _, st = gb.sssp_stats(g, 0, want_result=False, direction="push")
        if i > 1:
            ms.append(st.device_ms)
    t = statistics.median(ms)
    print(json.dumps({"wtype": wt, "lib": os.environ.get("GFB_LIB", "default"), "ms": t,
                      "gteps": st.m_reach / t / 1e6, "supersteps": st.supersteps,
                      "inflation": st.relaxations / st.m_reach}), flush=True)
    g.free()

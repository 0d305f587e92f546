"""4096^2 grid: f64 / f32 arithmetic, default loop choice vs BSP (variant 122)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_08200_b200 as gb  # noqa: E402

g = gb.grid(4096, seed=1, transpose=False)
ro, col, w = g.csr()
n = g.num_vertices
g64 = gb.Graph.from_csr(n, ro, col, w.astype("float64"), wtype="f64")
for name, gg in (("f32", g), ("f64", g64)):
    for v in (0, 122):
        _, _, st = gb.sssp_stats(gg, 0, want_result=False, direction="push", variant=v)
        _, _, st = gb.sssp_stats(gg, 0, want_result=False, direction="push", variant=v)
        print(json.dumps({"wtype": name, "variant": v, "ms": st.device_ms,
                          "steps_or_phases": st.supersteps,
                          "inflation": st.relaxations / st.m_reach}), flush=True)

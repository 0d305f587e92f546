"""Work inflation vs plan order (host loop): ascending id (0), by distance (42), reverse (43)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2212_08200_b200 as gb
ctx = gb.Context(0)
for sc in [int(x) for x in sys.argv[1:]] or [20, 24]:
    g = gb.rmat(sc, 16, seed=1, wtype="f32", transpose=True, ctx=ctx)
    base = None
    for v in (0, 42, 43, 47, 48, 49):
        d, p, st = gb.sssp_stats(g, 0, variant=v, device_loop=False)
        if base is None: base = d
        print(json.dumps({"scale": sc, "variant": v, "relax": st.relaxations,
                          "inflation": round(st.relaxations / st.m_reach, 3),
                          "supersteps": st.supersteps, "advance_ms": round(st.advance_ms, 3),
                          "equal": bool(np.array_equal(d, base))}), flush=True)

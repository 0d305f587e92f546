"""f64 SSSP breakdown at RMAT s24 (python tools/f64_breakdown.py VARIANTS)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_08200_b200 as gb  # noqa: E402

variants = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "0").split(",")]
g32 = gb.rmat(24, 16, seed=1, wtype="f32", transpose=False)
ro, col, w = g32.csr()
n = g32.num_vertices
g32.free()
g = gb.Graph.from_csr(n, ro, col, w.astype("float64"), wtype="f64")
for v in variants:
    for pred in (True, False):
        ms, adv = [], []
        for i in range(4):
            _, _, st = gb.sssp_stats(g, 0, want_result=False, direction="push", variant=v,
                                     compute_pred=pred)
            _, _, hs = gb.sssp_stats(g, 0, want_result=False, direction="push", variant=v,
                                     compute_pred=pred, device_loop=False)
            if i:
                ms.append(st.device_ms)
                adv.append(hs.advance_ms)
        print(json.dumps({"variant": v, "pred": pred, "ms": statistics.median(ms),
                          "advance_ms_hostloop": statistics.median(adv),
                          "fallback": st.pred_fallback, "relax": st.relaxations,
                          "supersteps": st.supersteps}), flush=True)

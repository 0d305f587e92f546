"""Time one library build (GFB_LIB=...) on RMAT s24: median device time of
the live device loop (compute_pred off so experimental builds that skip the
predecessor keys compare like for like), then one traced host-loop run whose
per-superstep advance / filter lines go to stderr.

  GFB_LIB=exp/nopkey/libgfb.so python tools/exp_time.py --scale 24 [--trace]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2212_08200_b200 as gb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--runs", type=int, default=10)
ap.add_argument("--trace", action="store_true")
ap.add_argument("--pred", type=int, default=0)
ap.add_argument("--defer", type=int, default=0)
ap.add_argument("--tile", type=int, default=0)
ap.add_argument("--tag", default=os.environ.get("GFB_LIB", "default"))
args = ap.parse_args()

ctx = gb.Context(0)
g = gb.rmat(args.scale, 16, seed=1, wtype="f32", transpose=False, ctx=ctx)
kw = dict(want_result=False, compute_pred=bool(args.pred), defer_pct=args.defer,
          advance_tile=args.tile)
for _ in range(3):
    gb.sssp_stats(g, 0, **kw)
ms = []
for _ in range(args.runs):
    _, _, st = gb.sssp_stats(g, 0, **kw)
    ms.append(st.device_ms)
out = {"tag": args.tag, "scale": args.scale, "median_ms": float(np.median(ms)),
       "min_ms": float(np.min(ms)), "supersteps": st.supersteps,
       "relaxations": st.relaxations, "m_reach": st.m_reach,
       "gteps": st.m_reach / np.median(ms) / 1e6}
if args.trace:
    _, _, st = gb.sssp_stats(g, 0, device_loop=False, trace=True, **kw)
    out["hostloop_ms"] = st.device_ms
    out["hostloop_adv_ms"] = st.advance_ms
print(json.dumps(out), flush=True)

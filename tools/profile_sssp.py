"""Run gfb_sssp on a device-generated graph (for ncu / timing experiments).

  python tools/profile_sssp.py --scale 24 --runs 2 --direction auto
Prints one JSON line per run with the library's own statistics.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_08200_b200 as gb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--grid", type=int, default=0, help="grid side (instead of RMAT)")
ap.add_argument("--runs", type=int, default=2)
ap.add_argument("--direction", default="auto")
ap.add_argument("--alpha", type=float, default=0.25)
ap.add_argument("--delta", type=float, default=0.0)
ap.add_argument("--device-loop", type=int, default=1)
ap.add_argument("--defer-pct", type=int, default=0)
ap.add_argument("--tile", type=int, default=0)
ap.add_argument("--relabel", default="auto")
ap.add_argument("--source", type=int, default=0)
a = ap.parse_args()
ctx = gb.Context(0)
g = gb.grid(a.grid) if a.grid else gb.rmat(a.scale, 16, seed=1, wtype="f32", transpose=True, ctx=ctx)
for r in range(a.runs):
    _, _, st = gb.sssp_stats(g, a.source, want_result=False, direction=a.direction, pull_alpha=a.alpha,
                             delta=a.delta, device_loop=bool(a.device_loop),
                             defer_pct=a.defer_pct, advance_tile=a.tile, relabel=a.relabel)
    print(json.dumps({k: getattr(st, k) for k, _ in gb.SsspStats._fields_}), flush=True)

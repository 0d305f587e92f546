"""Time gfb_graph_refill of the RMAT s24 CSR from pinned host arrays: f64
host weights (narrowed to f32 on the host, graph.cu narrow_weights) vs f32
host weights.  python tools/refill_time.py [--scale 24]"""
import argparse
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2212_08200_b200 as gb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=24)
args = ap.parse_args()
ctx = gb.Context(0)
g = gb.rmat(args.scale, 16, seed=1, wtype="f32", transpose=False, ctx=ctx)
ro, col, w = g.csr()
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
p_ro, p_col, p_w32, p_w64 = pin(ro), pin(col), pin(w), pin(w.astype(np.float64))
lib = gb._lib.load()
for name, pw, ht in (("f64", p_w64, gb.W_F64), ("f32", p_w32, gb.W_F32), ("f64", p_w64, gb.W_F64)):
    ts = []
    for i in range(4):
        t0 = time.perf_counter()
        gb.check(lib.gfb_graph_refill(g.h, C.c_void_p(p_ro.ctypes.data), C.c_void_p(p_col.ctypes.data),
                                      C.c_void_p(pw.ctypes.data), ht))
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"refill {name} host weights: {np.median(ts[1:]):.1f} ms (first {ts[0]:.1f}) "
          f"host bytes {(p_ro.nbytes + p_col.nbytes + pw.nbytes) / 1e9:.2f} GB", flush=True)
dist = pin(np.empty(g.num_vertices, np.float64))
pred = pin(np.empty(g.num_vertices, np.uint32))
o = gb._opts()
for name, pw, ht in (("f64", p_w64, gb.W_F64), ("f32", p_w32, gb.W_F32), ("f64", p_w64, gb.W_F64)):
    ts = []
    for i in range(4):
        st = gb.SsspStats()
        t0 = time.perf_counter()
        gb.check(lib.gfb_graph_refill(g.h, C.c_void_p(p_ro.ctypes.data), C.c_void_p(p_col.ctypes.data),
                                      C.c_void_p(pw.ctypes.data), ht))
        t1 = time.perf_counter()
        gb.check(lib.gfb_sssp(ctx.h, g.h, 0, C.byref(o), C.c_void_p(dist.ctypes.data),
                              C.c_void_p(pred.ctypes.data), C.byref(st)))
        ts.append(((time.perf_counter() - t0) * 1e3, (t1 - t0) * 1e3))
    print(f"e2e {name}: " + ", ".join(f"{a:.1f} (refill {b:.1f})" for a, b in ts), flush=True)
t0 = time.perf_counter()
x = np.empty(len(p_w64), np.float32)
np.copyto(x, p_w64, casting="same_kind")
print(f"numpy single-thread f64->f32 of {p_w64.nbytes / 1e9:.1f} GB: {(time.perf_counter() - t0) * 1e3:.1f} ms")
print("host cpus", os.cpu_count())

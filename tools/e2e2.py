import ctypes as C, os, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2212_08200_b200 as gb
from paper_2212_08200_b200 import _lib
lib = _lib.load()
ctx = gb.Context(0)
g = gb.rmat(24, 16, seed=1, wtype="f32", transpose=False, ctx=ctx)
ro, col, w = g.csr()
for i in range(2):
    gb.check(lib.gfb_graph_refill(g.h, C.c_void_p(ro.ctypes.data), C.c_void_p(col.ctypes.data), C.c_void_p(w.ctypes.data), gb.W_F32))
    d, p, st = gb.sssp_stats(g, 0)
    print(st.device_ms, st.pred_fallback)

"""Host-timed breakdown of bench.py's e2e step (pinned buffers):
refill H2D+CSR build | CSC build | relabel | sssp | D2H."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2212_08200_b200 as gb
from paper_2212_08200_b200 import _lib
lib = _lib.load()
ctx = gb.Context(0)
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
for csc in (True, False):
    g = gb.rmat(scale, 16, seed=1, wtype="f32", transpose=csc, ctx=ctx)
    ro, col, w = g.csr()
    p_ro = torch.from_numpy(ro).pin_memory().numpy()
    p_col = torch.from_numpy(col).pin_memory().numpy()
    p_w = torch.from_numpy(w).pin_memory().numpy()
    n = g.num_vertices
    dist = torch.empty(n, dtype=torch.float64).pin_memory().numpy()
    pred = torch.empty(n, dtype=torch.int32).pin_memory().numpy().view(np.uint32)
    o = gb._opts()
    st = gb.SsspStats()
    for i in range(3):
        t0 = time.perf_counter()
        gb.check(lib.gfb_graph_refill(g.h, C.c_void_p(p_ro.ctypes.data), C.c_void_p(p_col.ctypes.data),
                                      C.c_void_p(p_w.ctypes.data), gb.W_F32))
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        if csc:
            lib.gfb_debug_relabel(g.h, None, None, None)
        t2 = time.perf_counter()
        gb.check(lib.gfb_sssp(ctx.h, g.h, 0, C.byref(o), None, None, C.byref(st)))
        t3 = time.perf_counter()
        gb.check(lib.gfb_sssp_read(g.h, C.c_void_p(dist.ctypes.data), None, C.c_void_p(pred.ctypes.data)))
        t4 = time.perf_counter()
        print(f"csc={csc} refill(H2D+build) {1e3*(t1-t0):.1f} ms | relabel {1e3*(t2-t1):.1f} | sssp {1e3*(t3-t2):.1f} (dev {st.device_ms:.2f}) | read {1e3*(t4-t3):.1f} | total {1e3*(t4-t0):.1f}", flush=True)

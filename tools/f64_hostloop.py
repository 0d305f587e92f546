"""One f64 SSSP at RMAT s24 in host-loop mode (ncu target for k_push_range<REC>)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_08200_b200 as gb  # noqa: E402

g32 = gb.rmat(24, 16, seed=1, wtype="f32", transpose=False)
ro, col, w = g32.csr()
n = g32.num_vertices
g32.free()
g = gb.Graph.from_csr(n, ro, col, w.astype("float64"), wtype="f64")
_, _, st = gb.sssp_stats(g, 0, want_result=False, direction="push", device_loop=False)
print(st.supersteps, st.advance_ms)

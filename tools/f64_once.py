"""One f64 SSSP at RMAT s24 in host-loop mode twice (ncu launch-list target)."""
import sys; sys.path.insert(0, '/root/repo')
import paper_2212_08200_b200 as gb
g32 = gb.rmat(24, 16, seed=1, wtype="f32", transpose=False)
ro, col, w = g32.csr(); n = g32.num_vertices; g32.free()
g = gb.Graph.from_csr(n, ro, col, w.astype("float64"), wtype="f64")
for i in range(2):
    _, _, st = gb.sssp_stats(g, 0, want_result=False, direction="push", device_loop=False)
    print(st.pred_fallback, st.device_ms)

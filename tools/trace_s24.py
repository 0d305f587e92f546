import sys, json
sys.path.insert(0, '.')
import paper_2212_08200_b200 as gb
ctx = gb.Context(0)
g = gb.rmat(24, 16, seed=1, wtype="f32", transpose=True, ctx=ctx)
for r in range(3):
    _, _, st = gb.sssp_stats(g, 0, want_result=False, device_loop=False, trace=(r == 2))
    print(json.dumps({k: getattr(st, k) for k, _ in gb.SsspStats._fields_}), flush=True)
for r in range(5):
    _, _, st = gb.sssp_stats(g, 0, want_result=False)
    print("device", st.device_ms, st.supersteps, st.relaxations, flush=True)

"""Queue (async) model vs the BSP loop on RMAT s24 and the 4096^2 grid (device ms, work)."""
import sys, time, json, statistics
sys.path.insert(0, '/root/repo')
import paper_2212_08200_b200 as gb
for name, g in (("rmat24", gb.rmat(24, 16, seed=1, wtype="f32", transpose=False)), ("grid4096", gb.grid(4096, seed=1, transpose=False))):
    for mode in ("dense", "queue"):
        ms = []
        for i in range(4):
            kw = dict(delta=float("inf"), direction="push") if mode == "queue" else dict(direction="push")
            _, _, st = gb.sssp_stats(g, 0, want_result=False, **kw)
            if i: ms.append(st.device_ms)
        print(json.dumps({"graph": name, "mode": mode, "ms": statistics.median(ms), "phases_or_steps": st.supersteps, "inflation": st.relaxations / st.m_reach}), flush=True)
    g.free()

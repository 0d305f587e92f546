"""Time the unmodified reference (oracle/_ref) on the host-built RMAT graph:
build_csr, reference_dijkstra, sssp() seq and par -- sizing for bench.py's
CPU legs.  usage: python tools/ref_probe.py --scale 24 [--kinds dijkstra,seq,par]"""
import argparse
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--kinds", default="dijkstra,seq,par")
a = ap.parse_args()
print(subprocess.run("nproc; free -g | head -2; grep -m1 'model name' /proc/cpuinfo", shell=True,
                     capture_output=True, text=True).stdout, flush=True)
t = time.time()
ro, col, w = O.rmat_csr(a.scale, 16, 1, 1)
print(f"host rmat_csr s{a.scale}: {time.time() - t:.1f}s", flush=True)
t = time.time()
n = len(ro) - 1
src = np.repeat(np.arange(n, dtype=np.uint32), np.diff(ro).astype(np.int64))
g = O.RefGraph(n, src, col, w.astype(np.float64))
del src
print(f"reference build_csr: {time.time() - t:.1f}s", flush=True)
cores = int(O.ref().ref_hardware_concurrency())
for kind in a.kinds.split(","):
    t = time.perf_counter()
    if kind == "par":
        d, _, st, rl = g.sssp(0, mode=1, workers=cores, direction=0, repr_=0)
    elif kind == "seq":
        d, _, st, rl = g.sssp(0, mode=0, workers=1, direction=0, repr_=0)
    else:
        d, _ = g.dijkstra(0)
    dt = time.perf_counter() - t
    reach = np.isfinite(d)
    mr = int(np.diff(ro.astype(np.int64))[reach].sum())
    print(f"{kind}: {dt:.2f}s  m_reach={mr}  {mr / dt / 1e9:.4f} GTEPS", flush=True)
t = time.perf_counter()
d32, _ = O.dijkstra(n, ro, col, w, 0, "f32")
print(f"oracle f32 dijkstra: {time.perf_counter() - t:.2f}s", flush=True)

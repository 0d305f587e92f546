"""Partitioned SSSP, one process: the device-initiated peer exchange vs the
host-driven NCCL exchange (xmg.cu) on one GPU (P partitions sharing it; P = 1
runs a real one-rank NCCL communicator).  usage: python tools/xmg_bench.py
--scale 24 --parts 1,2,4"""
import argparse
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402  (input graph only)
from paper_2212_08200_b200 import peer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--parts", default="1,2,4")
ap.add_argument("--runs", type=int, default=3)
a = ap.parse_args()
ro, col, w = O.rmat_csr(a.scale, 16, 1, 1)
for parts in (int(x) for x in a.parts.split(",")):
    for ex in ("peer", "nccl"):
        x = peer.MgSssp([0] * parts, ro, col, w, exchange=ex)
        ms = []
        for i in range(a.runs + 1):
            t0 = time.perf_counter()
            _, _, st = x.sssp(0, want_pred=False)
            if i:
                ms.append((time.perf_counter() - t0) * 1e3)
        print(f"s{a.scale} parts={parts} exchange={ex} nccl={x.uses_nccl()}: wall {statistics.median(ms):.2f} ms"
              f" (device_ms {st['device_ms']:.2f}), supersteps {st['supersteps']}, "
              f"GTEPS {st['m_reach'] / statistics.median(ms) * 1e-6:.2f}", flush=True)
        x.free()

"""bench.py --gpus N (N > 1): the 1-D partitioned SSSP over NCCL.

Launched by torchrun (one process per GPU).  Every rank builds the same RMAT
graph on its own GPU (device generator, identical by construction), keeps
the rows of its edge-balanced vertex range [lo, hi) and runs the partitioned
BSP loop of paper_2212_08200_b200/mg.py: local advance on the device
(gfb_part_advance), per-owner message exchange with NCCL all_to_all over
NVLink/NVSwitch, device apply, allreduce convergence.  Strong scaling: the
workload (graph) is the same as at N=1.  value = m_reach / max over ranks of
the per-SSSP time (CUDA events on the NCCL stream around a host-synchronous
loop, i.e. device time of the whole exchange-inclusive superstep chain).
"""
import json
import os
import sys
import time

import numpy as np


def run(args, rank, world):
    import torch
    import torch.distributed as dist

    import paper_2212_08200_b200 as gb
    from paper_2212_08200_b200 import mg

    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world == 1:  # --partitioned without torchrun: a single-rank group
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    ctx = gb.Context(local)
    t0 = time.time()
    g = gb.rmat(args.scale, args.edgefactor, seed=args.seed, wtype="f32", transpose=False, ctx=ctx)
    ro, col, w = g.csr()
    n = g.num_vertices
    g.free()
    rs = mg.edge_balanced_ranges(ro, world)
    lo, hi = int(rs[rank]), int(rs[rank + 1])
    ro_l, col_l, w_l = mg.slice_csr(ro, col, w, lo, hi)
    eng = mg.GfbPart(n, lo, hi, ro_l, col_l, w_l, ctx=ctx)
    print(f"[rank {rank}] rows [{lo},{hi}) edges {len(col_l)} ({len(col_l) / len(col):.3f} of m) "
          f"setup {time.time() - t0:.1f}s", file=sys.stderr, flush=True)

    def one(want_pred=False):
        return mg.sssp_partitioned(eng, rs, 0, device=dev, want_pred=want_pred)

    for _ in range(args.warmup):
        one()
    times = []
    for _ in range(args.steps):
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d, _, st = one()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    t_local = sum(times) / len(times)
    tt = torch.tensor([t_local], dtype=torch.float64, device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_ms = float(tt.item())
    reach = np.isfinite(d)
    m_loc = int(np.diff(ro_l.astype(np.int64))[reach].sum())
    agg = torch.tensor([m_loc, int(reach.sum()), st["relaxations"], st["messages_sent"]],
                       dtype=torch.int64, device=dev)
    dist.all_reduce(agg, op=dist.ReduceOp.SUM)
    m_reach, n_reach, relax, msgs = (int(x) for x in agg.tolist())

    # e2e: host slice -> device (partition upload) + SSSP + D2H of distances
    e2e_ms = []
    pin = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy() for a in (ro_l, col_l, w_l)]
    for _ in range(2):
        dist.barrier()
        t1 = time.perf_counter()
        e2 = mg.GfbPart(n, lo, hi, *pin, ctx=ctx)
        d2, _, _ = mg.sssp_partitioned(e2, rs, 0, device=dev)
        del e2
        e2e_ms.append((time.perf_counter() - t1) * 1e3)
    te = torch.tensor([e2e_ms[-1]], dtype=torch.float64, device=dev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)

    if rank == 0:
        gteps = m_reach / (t_ms * 1e-3) / 1e9
        b_alg = 12.0 + 20.0 * n_reach / m_reach
        peak = 6549.4
        try:
            peak = float(json.load(open(os.path.join(os.path.dirname(__file__),
                                                     "MEASURED_PEAKS.json")))["hbm_gbs"])
        except Exception:
            pass
        print(json.dumps({
            "metric": "SSSP GTEPS on RMAT (1/2/4/8 B200) and % of HBM roofline vs host-CPU ref",
            "value": gteps, "unit": "GTEPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (device-generated RMAT on every rank)",
            "config": {"workload": f"RMAT scale {args.scale} EF{args.edgefactor} fp32, source 0, "
                                   f"1-D edge-balanced partition over {world} GPUs, NCCL all-to-all",
                       "scale": args.scale, "edgefactor": args.edgefactor,
                       "parallelism": f"1d-partition{world}",
                       "l2": "inputs larger than L2"},
            "e2e": {"value": m_reach / (float(te.item()) * 1e-3) / 1e9, "unit": "GTEPS",
                    "h2d_bytes_per_step": int(sum(a.nbytes for a in pin)) * world,
                    "d2h_bytes_per_step": int(n * 4)},
            "roofline": {"bound": "hbm", "achieved": gteps * b_alg, "peak": peak * world,
                         "unit": "GB/s", "frac": gteps * b_alg / (peak * world), "traffic": None,
                         "note": "whole-SSSP B_alg x GTEPS vs P x measured HBM"},
            "cpu_baseline": None, "m_reach": m_reach, "n_reach": n_reach,
            "relaxations": relax, "messages": msgs, "supersteps": st["supersteps"],
            "nvlink_bytes": msgs * 16,
            "gpu_launches": None}), flush=True)
    dist.barrier()
    dist.destroy_process_group()

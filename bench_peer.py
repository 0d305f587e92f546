"""bench.py --gpus N (N > 1, or --partitioned): the peer-memory partitioned SSSP.

Launched by torchrun, one process per GPU.  Every rank builds the same RMAT
graph on its GPU (device generator, identical by construction), keeps the CSR
rows of its edge-balanced, 32-aligned vertex range, uploads them as a
gfb_peer (include/gfb.h), maps every peer's loop state over CUDA IPC
(NVLink on a multi-GPU node) and runs the device-driven partitioned loop
(paper_2212_08200_b200/peer.py, csrc/peer.cu): remote relaxations go straight
into the owner's memory, device barriers decide convergence, no host round
trip per superstep.  Strong scaling: the graph is the same as at N = 1.
value = m_reach / max over ranks of the per-SSSP device time (CUDA events on
the library stream around the loop graph + predecessor pass).
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
    from paper_2212_08200_b200 import mg, peer
    from bench import METRIC, ClockSampler, peaks

    local = int(os.environ.get("LOCAL_RANK", rank))
    dev = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(dev)
    if world == 1:  # --partitioned without torchrun: a single-rank group
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
    # the only host-driven collectives: the one-time IPC handle exchange,
    # barriers and the final max/sum reductions of the measurements -- over
    # NCCL (the exchange itself is device-initiated through peer memory)
    # NCCL with a GPU per rank; ranks sharing one GPU (one-GPU test boxes) fall
    # back to gloo (NCCL rejects duplicate devices)
    if torch.cuda.device_count() >= world:
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", dev))
        cdev = torch.device("cuda", dev)
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        cdev = torch.device("cpu")
    ctx = gb.Context(dev)
    t0 = time.time()
    g = gb.rmat(args.scale, args.edgefactor, seed=args.seed, wtype="f32", transpose=False, ctx=ctx)
    ro, col, w = g.csr()
    n = g.num_vertices
    rs = peer.aligned_ranges(ro, world)
    relabel = not getattr(args, "no_relabel", False)
    if relabel:  # range-preserving in-degree relabel + destination-sorted rows (untimed setup,
        # like the single-GPU loop's relabelled copy built in its warm-up)
        ro, col, w, perm = peer.relabel_ranges(g, rs)
    src = int(perm[0]) if relabel else 0  # source 0 of the generator's ids
    g.free()
    lo, hi = int(rs[rank]), int(rs[rank + 1])
    ro_l, col_l, w_l = mg.slice_csr(ro, col, w, lo, hi)
    del col, w
    p = peer.PeerSssp(rank, world, rs, ro_l, col_l, w_l, ctx=ctx)
    p.link()
    print(f"[rank {rank}] rows [{lo},{hi}) edges {len(col_l)} setup {time.time() - t0:.1f}s",
          file=sys.stderr, flush=True)

    sampler = ClockSampler(dev) if rank == 0 else None
    if sampler:
        sampler.start()
    t_end = time.time() + args.soak
    i = 0
    while i < args.warmup or time.time() < t_end:
        dist.barrier()
        p.sssp(src)
        i += 1
    times, launches = [], 0
    for _ in range(args.steps):
        dist.barrier()  # host skew out of the device timing
        st = p.sssp(src)
        times.append(st["device_ms"])
        launches += st["kernel_launches"]
    clocks = sampler.stop() if sampler else None
    t_local = sum(times) / len(times)
    tt = torch.tensor([t_local], dtype=torch.float64, device=cdev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_ms = float(tt.item())
    agg = torch.tensor([st["m_reach"], st["n_reach"], st["relaxations"], launches],
                       dtype=torch.int64, device=cdev)
    dist.all_reduce(agg, op=dist.ReduceOp.SUM)
    m_reach, n_reach, relax, all_launches = (int(x) for x in agg.tolist())

    # correctness at full size: every rank's local distances satisfy the
    # fixpoint on its own edges (no local out-edge can still relax)
    d_all, _ = peer.gather(p, native=True)
    du = d_all[lo:hi].astype(np.float32)
    src_rows = np.repeat(np.arange(hi - lo, dtype=np.int32), np.diff(ro_l.astype(np.int64)))
    fin = np.isfinite(du[src_rows])
    nd = du[src_rows][fin] + w_l[fin]
    relaxable = int(np.count_nonzero(nd < d_all[col_l[fin]].astype(np.float32)))
    bad = torch.tensor([relaxable], dtype=torch.int64, device=cdev)
    dist.all_reduce(bad)

    # e2e: host slice (pinned) -> device upload + IPC link + SSSP + D2H of the
    # local distances, per rank; max over ranks
    pin = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
           for a in (ro_l, col_l, w_l)]
    e2e_ms = []
    for _ in range(2):
        dist.barrier()
        t1 = time.perf_counter()
        p2 = peer.PeerSssp(rank, world, rs, *pin, ctx=ctx)
        p2.link()
        p2.sssp(src)
        d2, _ = p2.read(native=True)
        e2e_ms.append((time.perf_counter() - t1) * 1e3)
        dist.barrier()
        p2.free()
    te = torch.tensor([e2e_ms[-1]], dtype=torch.float64, device=cdev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)

    if rank == 0:
        gteps = m_reach / (t_ms * 1e-3) / 1e9
        b_alg = 12.0 + 20.0 * n_reach / m_reach
        peak, peak_kind = peaks()
        print(json.dumps({
            "metric": METRIC, "value": gteps, "unit": "GTEPS", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (device-generated RMAT on every rank)",
            "config": {"workload": f"RMAT scale {args.scale} EF{args.edgefactor} fp32, source 0, "
                                   f"1-D edge-balanced partition over {world} GPU(s), "
                                   f"device-initiated exchange over peer memory",
                       "relabel": "in-degree order inside each rank's range, rows sorted by "
                                  "destination (gfb_graph_relabel_ranges, untimed setup)"
                                  if relabel else "none (the generator's ids)",
                       "scale": args.scale, "edgefactor": args.edgefactor,
                       "parallelism": f"1d-partition{world}-peer",
                       "l2": "inputs larger than L2"},
            "e2e": {"value": m_reach / (float(te.item()) * 1e-3) / 1e9, "unit": "GTEPS",
                    "h2d_bytes_per_step": int(sum(a.nbytes for a in pin)) * world,
                    "d2h_bytes_per_step": int(n * 4),
                    "note": "per rank: pinned slice upload + IPC link + SSSP + D2H, max over ranks"},
            "roofline": {"bound": "hbm", "achieved": gteps * b_alg, "peak": peak * world,
                         "unit": "GB/s", "frac": gteps * b_alg / (peak * world), "traffic": None,
                         "peak_kind": peak_kind,
                         "note": "whole-SSSP B_alg x GTEPS vs P x measured HBM"},
            "cpu_baseline": None, "clocks": clocks, "gpu_launches": all_launches,
            "m_reach": m_reach, "n_reach": n_reach, "relaxations": relax,
            "work_inflation": relax / m_reach, "supersteps": st["supersteps"],
            "pred_fallback": st["pred_fallback"],
            "fixpoint_check": {"relaxable_edges": int(bad.item())},
            "exchange": "peer"}), flush=True)
    dist.barrier()
    p.free()
    dist.destroy_process_group()

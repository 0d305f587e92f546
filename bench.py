#!/usr/bin/env python
"""SSSP GTEPS bench (BASELINE.json metric) for the B200 path and the reference.

Default workload: BASELINE configs[2] -- RMAT scale 24, edge factor 16, fp32
U[0,1) weights, source 0, one B200.  Direction push: the push/pull switch
(AUTO, pull when frontier edges > m / alpha at the measured break-even
alpha = 1.05) never fires with the far-bucket deferral (no superstep
exceeds 0.22 m); its measurement is a secondary line.
A "step" is one full sssp() (init .. last superstep .. predecessor pass).

  value   GTEPS = m_reach / device time per step, graph resident in HBM
          (CUDA events on the library's stream; max over ranks).  The
          in-degree-relabelled loop CSR is built on the second call on a
          graph (during the warm-up) and reused; `one_shot` is the same call
          on the caller's ids (what a single upload + sssp() gets).
  e2e     the same metric through the public C ABI with HOST buffers: each
          step re-uploads the reference-layout CSR from pinned memory
          (gfb_graph_refill: H2D + device CSR build), runs gfb_sssp and
          copies dist (f64) + pred back.
  roofline  the advance kernel (k_push_range): algorithmic bytes of the step,
          B_alg x m_reach (every reached edge once, no credit
          for redundant visits), over its CUDA-event time per step.
  parity  the timed configuration checked at FULL size against the CPU
          oracle: the device graph equals the host-built one, distances
          bit-identical to the fp32 restatement of reference_dijkstra, the
          predecessor tree valid, max ulp vs the unmodified reference's
          doubles; f64 arithmetic bit-identical to them.
  cpu_baseline  the unmodified reference (oracle/_ref) on this host, on the
          same full-size graph: reference_dijkstra (algorithms.hpp:101-128,
          the fastest CPU path); --cpu-all adds sssp() seq and par.

--impl reference runs the unmodified reference on the SAME configuration
(the full RMAT s24 graph, built by the oracle's host generator and the
reference's own build_csr): every step is one reference_dijkstra from
source 0 (the fastest reference path, single-threaded by construction); the
K timed steps run concurrently on all host threads and value = K x m_reach /
wall time (the host's whole-job throughput).

--gpus N (N > 1) without torchrun re-launches itself under
torch.distributed.run with N ranks (127.0.0.1 rendezvous).
"""
import argparse
import concurrent.futures as cf
import ctypes as C
import json
import os
import platform
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SSSP GTEPS on RMAT (1/2/4/8 B200) and % of HBM roofline vs host-CPU ref"
NOMINAL_HBM_GBS = 8000.0
# measured on this pool's B200 by tools/microbench.cu: coalesced 8-byte record
# stream + one dependent random 4-byte gather into a 64 MB L2-resident array
GATHER_CEILING = 263e9


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def host_info():
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    from oracle import oracle as O
    hc = int(O.ref().ref_hardware_concurrency()) if O.ref() is not None else None
    return {"cpu_model": model or platform.processor(), "nproc": os.cpu_count(),
            "hardware_concurrency": hc}


# ------------------------------------------------------------------ clocks ---
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,utilization.gpu,power.draw,"
              "clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, device=0):
        self.device, self.rows, self.proc = device, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        load = [r for r in self.rows if len(r) >= 8 and r[2].isdigit() and int(r[2]) > 0]
        use = load or [r for r in self.rows if len(r) >= 8]
        if not use:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[0]) for r in use if r[0].replace(".", "").isdigit()]
        reasons = sorted({names[i] for r in use for i in range(4) if r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(use[0][1]) if use[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(use), "samples_under_load": len(load)}


# -------------------------------------------------------------- reference ---
def host_rmat(args):
    """The RMAT graph in build_csr layout built on the host by the oracle's C
    generator (no product code): (ro, col, w_f32)."""
    from oracle import oracle as O
    t0 = time.time()
    ro, col, w = O.rmat_csr(args.scale, args.edgefactor, args.seed, 1)
    log(f"[host] RMAT s{args.scale} CSR (oracle generator) {time.time() - t0:.1f}s")
    return ro, col, w


def ref_graph(ro, col, w):
    """The reference's own Graph (build_csr, graph.hpp:132-162) -- untimed."""
    from oracle import oracle as O
    n = len(ro) - 1
    t0 = time.time()
    src = np.repeat(np.arange(n, dtype=np.uint32), np.diff(ro.astype(np.int64)))
    g = O.RefGraph(n, src, col, w.astype(np.float64))
    del src
    log(f"[ref] build_csr n={n} m={len(col)} {time.time() - t0:.1f}s (untimed)")
    return g


def m_reach_of(ro, dist):
    reach = np.isfinite(dist)
    return int(np.diff(ro.astype(np.int64))[reach].sum()), int(reach.sum())


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as O
    if O.ref() is None:
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref/libgraflow_ref.so not built"}))
        return
    ro, col, w = host_rmat(args)
    g = ref_graph(ro, col, w)
    del col
    info = host_info()
    cores = info["hardware_concurrency"] or 1

    def one(_):
        t0 = time.perf_counter()
        d, _ = g.dijkstra(0)  # algorithms.hpp:101-128
        return time.perf_counter() - t0, d

    with cf.ThreadPoolExecutor(max_workers=cores) as pool:  # ctypes drops the GIL
        warm = list(pool.map(one, range(args.warmup)))
        t0 = time.perf_counter()
        runs = list(pool.map(one, range(args.steps)))
        wall = time.perf_counter() - t0
    dist = runs[-1][1]
    m_reach, n_reach = m_reach_of(ro, dist)
    per = [r[0] for r in runs]
    gteps = args.steps * m_reach / wall / 1e9
    sample = (f"full RMAT scale {args.scale} EF{args.edgefactor} fp32 graph (oracle host "
              f"generator + the reference's build_csr), source 0; each step = one "
              f"reference_dijkstra (algorithms.hpp:101-128: the fastest reference path; "
              f"sssp() seq / par are 2.6x / 7.3x slower at s24, profiles/r02_ref_s24.txt); the "
              f"{args.steps} timed steps run concurrently on {cores} host threads: value = steps x "
              f"m_reach / wall; m_reach={m_reach}")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": gteps, "unit": "GTEPS",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": wall / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args),
        "cpu_baseline": {"value": gteps, "unit": "GTEPS", "cores": cores, "kind": "reference",
                         "sample": sample, **info},
        "e2e": {"value": gteps, "unit": "GTEPS", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "single_run": {"median_s": statistics.median(per), "min_s": min(per),
                       "gteps": m_reach / statistics.median(per) / 1e9, "threads": 1},
        "warmup_runs_s": [r[0] for r in warm],
        "m_reach": m_reach, "n_reach": n_reach}))


def config_dict(args):
    return {"workload": f"RMAT scale {args.scale} EF{args.edgefactor} fp32 U[0,1) weights, "
                        f"source 0, direction {args.direction} (BASELINE.json configs[2]; the "
                        f"push/pull switch is measured as a secondary line: it never pulls "
                        f"under the deferral)",
            "scale": args.scale, "edgefactor": args.edgefactor, "weights": "f32",
            "direction": args.direction, "seed": args.seed,
            "l2": "inputs larger than L2 (CSR ~2.1 GB at scale 24 vs 126 MB L2)"}


# ---------------------------------------------------------------- our arm ---
def run_ours(args):
    import paper_2212_08200_b200 as gb
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1 or args.partitioned:
        if args.exchange == "nccl":  # host-driven message exchange (mg.py)
            import bench_mg
            return bench_mg.run(args, rank, world)
        import bench_peer  # device-initiated exchange over peer memory (peer.py)
        return bench_peer.run(args, rank, world)
    ctx = gb.Context(0)
    t0 = time.time()
    g = gb.rmat(args.scale, args.edgefactor, seed=args.seed, wtype="f32", transpose=True, ctx=ctx)
    log(f"[gpu] generated RMAT s{args.scale}: n={g.num_vertices} m={g.num_edges} "
        f"in {time.time() - t0:.1f}s")
    kw = dict(direction=args.direction, pull_alpha=args.alpha)

    # one-shot: the first call on a fresh upload runs on the caller's ids
    one_shot = []
    for _ in range(3):
        _, _, st1 = gb.sssp_stats(g, 0, want_result=False, relabel="off", **kw)
        one_shot.append(st1.device_ms)

    sampler = ClockSampler()
    sampler.start()
    # warm-up (builds the relabelled loop CSR on the second call; keeps the
    # GPU busy long enough for clock samples)
    t_end = time.time() + args.soak
    i = 0
    while i < args.warmup or time.time() < t_end:
        _, _, st = gb.sssp_stats(g, 0, want_result=False, **kw)
        i += 1
    # timed region: exactly K steps, device time from CUDA events
    dev_ms, launches = [], 0
    wall0 = time.perf_counter()
    for _ in range(args.steps):
        _, _, st = gb.sssp_stats(g, 0, want_result=False, **kw)
        dev_ms.append(st.device_ms)
        launches += st.kernel_launches
    wall = time.perf_counter() - wall0
    clocks = sampler.stop()
    m_reach, n_reach = st.m_reach, st.n_reach
    t_ms = sum(dev_ms) / len(dev_ms)
    gteps = m_reach / (t_ms * 1e-3) / 1e9
    b_alg = 12.0 + 20.0 * n_reach / m_reach
    peak, peak_kind = peaks()
    dist32, pred = gb.sssp_read(g, native=True)  # the last timed step's result

    # kernel roofline: advance launches, CUDA events per launch (host loop)
    _, _, ist = gb.sssp_stats(g, 0, want_result=False, device_loop=False, **kw)
    alg_bytes = b_alg * m_reach
    achieved = alg_bytes / (ist.advance_ms * 1e-3) / 1e9 if ist.advance_ms > 0 else None
    traffic = None
    tp = os.path.join(ROOT, "profiles", "advance_traffic.json")
    if os.path.exists(tp):
        tr = json.load(open(tp))
        if tr.get("scale") == args.scale:
            traffic = tr.get("dram_bytes_per_step")

    # e2e through the public API with host buffers
    e2e = run_e2e(gb, ctx, g, args, kw)

    secondary = [] if args.no_secondary else secondary_configs(gb, ctx, args, g)
    f64_dist = None
    for rec in secondary:
        f64_dist = rec.pop("_dist", f64_dist)

    parity, cpu = None, None
    if not args.no_cpu:
        parity, cpu = full_size_parity(gb, g, args, dist32, pred, st, f64_dist)

    out = {
        "metric": METRIC, "value": gteps, "unit": "GTEPS", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (device-generated RMAT)",
        "config": dict(config_dict(args), loop_csr="in-degree-relabelled copy, built on the "
                                                   "2nd call (warm-up, untimed) and reused"),
        "one_shot": {"ms": statistics.median(one_shot),
                     "gteps": m_reach / (statistics.median(one_shot) * 1e-3) / 1e9,
                     "note": "same call on the caller's vertex ids (no relabelled copy)"},
        "e2e": e2e,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if achieved else None, "traffic": traffic,
                     "kernel": "k_push_range (advance, hot.cuh) + k_tail (the last supersteps' "
                               "advances with their queue filter, tail.cuh)",
                     "algorithmic_bytes_per_step": alg_bytes,
                     "b_alg_bytes_per_te": b_alg, "m_reach": m_reach,
                     "advance_ms_per_step": ist.advance_ms,
                     "advance_launches_per_step": ist.advance_launches,
                     "advance_share_of_step": ist.advance_ms / t_ms,
                     "peak_kind": peak_kind,
                     "note": "achieved = B_alg x m_reach (SURVEY §8(d), redundant visits get "
                             "no credit) / advance time per step (CUDA events, host-loop run; "
                             "the tail kernel's whole time counted as advance); traffic = ncu "
                             "dram read+write summed over one step's advance + tail launches "
                             "(profiles/advance_traffic.json)"},
        "visits": {"relaxations_per_step": ist.relaxations,
                   "work_inflation": ist.relaxations / m_reach,
                   "visit_bw_gbs": ist.relaxations * 12 / (ist.advance_ms * 1e-3) / 1e9
                   if ist.advance_ms else None,
                   "visits_per_s": ist.relaxations / (ist.advance_ms * 1e-3)
                   if ist.advance_ms else None,
                   "gather_ceiling_visits_per_s": GATHER_CEILING,
                   "note": "kernel-efficiency view: 1 streamed 8 B record + 1 random 4 B gather "
                           "per visit; ceiling measured by tools/microbench.cu"},
        "roofline_sssp": {"b_alg_bytes_per_te": b_alg,
                          "achieved_gbs": gteps * b_alg,
                          "frac_of_measured": gteps * b_alg / peak,
                          "frac_of_8tbs": gteps * b_alg / NOMINAL_HBM_GBS,
                          "roofline_gteps_8tbs": NOMINAL_HBM_GBS / b_alg},
        "parity": parity,
        "cpu_baseline": cpu,
        "clocks": clocks,
        "gpu_launches": launches,
        "m_reach": m_reach, "n_reach": n_reach, "supersteps": st.supersteps,
        "relaxations": st.relaxations, "work_inflation": st.relaxations / m_reach,
        "push_steps": st.push_steps, "pull_steps": st.pull_steps,
        "pred_fallback": st.pred_fallback, "wall_s_timed": wall,
        "secondary": secondary,
    }
    if cpu and cpu.get("value"):
        out["speedup_vs_cpu_best"] = gteps / cpu["value"]
        if e2e and e2e.get("value"):
            out["e2e_speedup_vs_cpu_best"] = e2e["value"] / cpu["value"]
    print(json.dumps(out))


def f32_ulps(d32, dref):
    """|device fp32 - reference double| in fp32 ulps at the reference value."""
    fin = np.isfinite(dref)
    if not np.array_equal(fin, np.isfinite(d32)):
        return None
    r = dref[fin]
    sp = np.spacing(r.astype(np.float32)).astype(np.float64)
    sp[sp == 0] = np.spacing(np.float32(0))
    return float(np.max(np.abs(d32[fin].astype(np.float64) - r) / sp)) if r.size else 0.0


def full_size_parity(gb, g, args, dist32, pred, st, f64_dist):
    """Two-sided full-size check of the timed configuration + the CPU baseline
    on the same in-memory graph."""
    from oracle import oracle as O
    ro, col, w = host_rmat(args)
    dro, dcol, dw = g.csr()
    same_graph = bool(np.array_equal(ro, dro) and np.array_equal(col, dcol)
                      and np.array_equal(w.view(np.uint32), dw.view(np.uint32)))
    del dro, dcol, dw
    n = len(ro) - 1
    t0 = time.perf_counter()
    want32, _ = O.dijkstra(n, ro, col, w, 0, "f32")
    t_orc = time.perf_counter() - t0
    equal32 = bool(np.array_equal(want32.view(np.uint32), dist32.view(np.uint32)))
    bad_pred = int(O.check_pred_tree(n, ro, col, w, dist32, 0, pred))
    parity = {"graph": f"RMAT s{args.scale} (the timed configuration)",
              "device_graph_equals_host_build": same_graph,
              "oracle_equal": equal32,
              "oracle": "fp32 restatement of reference_dijkstra (oracle/graflow_oracle.c), "
                        f"{t_orc:.1f}s on one core",
              "pred_tree_valid": bad_pred == -1,
              "n_reach_match": int(np.isfinite(want32).sum()) == st.n_reach}
    cpu = None
    if O.ref() is not None:
        info = host_info()
        rg = ref_graph(ro, col, w)
        runs = {}
        t0 = time.perf_counter()
        dref, _ = rg.dijkstra(0)
        runs["dijkstra"] = (time.perf_counter() - t0, 1)
        log(f"[ref] dijkstra s{args.scale}: {runs['dijkstra'][0]:.2f}s")
        if args.cpu_all:
            hc = info["hardware_concurrency"] or 1
            for kind, mode, wk in (("seq", 0, 1), ("par", 1, hc)):
                t0 = time.perf_counter()
                rg.sssp(0, mode=mode, workers=wk, direction=0, repr_=0)
                runs[kind] = (time.perf_counter() - t0, wk)
                log(f"[ref] {kind} s{args.scale}: {runs[kind][0]:.2f}s on {wk} thread(s)")
        del rg
        m_reach, _ = m_reach_of(ro, dref)
        parity["max_ulp_vs_reference_f64"] = f32_ulps(dist32, dref)
        if f64_dist is not None:
            parity["f64_equal_reference"] = bool(
                np.array_equal(f64_dist.view(np.uint64), dref.view(np.uint64)))
        best = min(runs, key=lambda k: runs[k][0])
        cpu = {"value": m_reach / runs[best][0] / 1e9, "unit": "GTEPS", "cores": runs[best][1],
               "kind": "reference",
               "sample": f"the full RMAT s{args.scale} graph (same CSR, built by the reference's "
                         f"own build_csr), source 0, one run each; fastest of "
                         f"{'/'.join(runs)} = {best}"
                         + ("" if args.cpu_all else "; sssp() seq/par at s24: --cpu-all, "
                            "profiles/r02_ref_s24.txt"),
               "runs": {k: {"s": v[0], "threads": v[1], "gteps": m_reach / v[0] / 1e9}
                        for k, v in runs.items()},
               **info}
    return parity, cpu


def sp_certificate(ro, col, w, dist, pred, source):
    """Size-independent proof that fp32 distances are THE shortest-path
    fixpoint (SURVEY §8c at sizes the oracle's Dijkstra is slow at): dist[src]
    = 0, no edge can still relax (fl(dist[u] + w) >= dist[v] for every edge,
    the device's own arithmetic) and the predecessor tree is tight and
    acyclic (the reference checker's rules, oracle/graflow_oracle.c)."""
    from oracle import oracle as O
    n = len(ro) - 1
    ok_src = dist[source] == 0
    relaxable = 0
    step = 1 << 26
    for r0 in range(0, n, 1 << 22):  # row blocks (bounded temporaries)
        r1 = min(n, r0 + (1 << 22))
        e0, e1 = int(ro[r0]), int(ro[r1])
        for a in range(e0, e1, step):
            b = min(e1, a + step)
            rows = np.searchsorted(ro[r0:r1 + 1], np.arange(a, b, dtype=np.int64),
                                   side="right") - 1 + r0
            du = dist[rows]
            fin = np.isfinite(du)
            nd = du[fin] + w[a:b][fin]
            relaxable += int(np.count_nonzero(nd < dist[col[a:b][fin]]))
    bad = int(O.check_pred_tree(n, ro, col, w, dist, source, pred))
    return {"source_zero": bool(ok_src), "relaxable_edges": relaxable, "pred_tree_valid": bad == -1}


def secondary_configs(gb, ctx, args, g_main=None):
    """The other BASELINE.json configs as extra measurements (not the headline):
    f64 arithmetic on the headline graph, configs[1] RMAT s22 push-only,
    configs[3] 4096^2 grid (near-far filter vs plain BSP, device-side
    convergence), configs[4]'s graph (RMAT s26) on one GPU, and the device BFS
    (algorithms.hpp:194-239) on the headline graph.  Each full-size result is
    compared with the oracle unless --no-cpu."""
    from oracle import oracle as O
    out = []

    def timed(g, runs, **kw):
        ms = []
        for i in range(runs + 1):
            _, _, st = gb.sssp_stats(g, 0, want_result=False, **kw)
            if i:
                ms.append(st.device_ms)
        return statistics.median(ms), st

    def check32(g, n):
        if args.no_cpu:
            return None
        ro, col, w = g.csr()
        d, p = gb.sssp_read(g, native=True)
        want, _ = O.dijkstra(n, ro, col, w, 0, "f32")
        return {"oracle_equal": bool(np.array_equal(want.view(np.uint32), d.view(np.uint32))),
                "pred_tree_valid": O.check_pred_tree(n, ro, col, w, d, 0, p) == -1}

    if g_main is not None:
        for _ in range(2):
            gb.bfs(g_main, 0, direction="auto", want_result=False)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            _, bst, brl = gb.bfs(g_main, 0, direction="auto", want_result=False)
            ts.append((time.perf_counter() - t0) * 1e3)
        bms = statistics.median(ts)
        out.append({"config": f"bfs() on the headline RMAT s{args.scale} graph, source 0 "
                              f"(direction-optimizing: bottom-up levels while frontier edges > m/20)",
                    "gteps": brl / (bms * 1e-3) / 1e9, "ms": bms, "supersteps": bst,
                    "relaxations": brl,
                    "timing": "host wall clock around the synchronous gfb_bfs call"})
        # f64 arithmetic: the C++ policy default, bit-exact vs the reference
        ro, col, w = g_main.csr()
        g64 = gb.Graph.from_csr(g_main.num_vertices, ro, col, w.astype("float64"), wtype="f64",
                                ctx=ctx)
        del ro, col, w
        ms, st = timed(g64, 5, direction="push")
        d64, _ = gb.sssp_read(g64)
        out.append({"config": f"RMAT s{args.scale} EF{args.edgefactor}, f64 arithmetic (the same "
                              f"weights widened; compared bit for bit with the reference's "
                              f"doubles in parity.f64_equal_reference), push",
                    "gteps": st.m_reach / (ms * 1e-3) / 1e9, "ms": ms,
                    "supersteps": st.supersteps, "work_inflation": st.relaxations / st.m_reach,
                    "_dist": d64})
        g64.free()
        # the push/pull switch at its break-even (needs the transpose; the
        # relabelled CSR has none): with the deferral (default) and without
        for dp in (0, 100):
            ms, st = timed(g_main, 3, direction="auto", pull_alpha=1.05, defer_pct=dp)
            out.append({"config": f"push/pull switch (AUTO, alpha 1.05: pull when frontier edges "
                                  f"> 0.95 m) on the headline graph, deferral "
                                  f"{'off' if dp == 100 else 'on (default)'}",
                        "gteps": st.m_reach / (ms * 1e-3) / 1e9, "ms": ms,
                        "push_steps": st.push_steps, "pull_steps": st.pull_steps,
                        "supersteps": st.supersteps,
                        "work_inflation": st.relaxations / st.m_reach})
    g = gb.rmat(22, args.edgefactor, seed=args.seed, wtype="f32", transpose=True, ctx=ctx)
    ms, st = timed(g, 5, direction="push")
    out.append({"config": "BASELINE configs[1]: RMAT s22 EF16 fp32, push-only",
                "gteps": st.m_reach / (ms * 1e-3) / 1e9, "ms": ms, "supersteps": st.supersteps,
                "work_inflation": st.relaxations / st.m_reach,
                "parity": check32(g, g.num_vertices)})
    g.free()
    side = args.grid_side
    g = gb.grid(side, seed=args.seed, transpose=True, ctx=ctx)
    bms, bst = timed(g, 1, loop="bsp")  # the BSP loop (no automatic near-far choice)
    bsp_check = check32(g, g.num_vertices)
    ms, st = timed(g, 3, delta=args.grid_delta)
    rec = {"config": f"BASELINE configs[3]: {side}^2 4-neighbour grid fp32 U[0,1), source 0 "
                     f"(corner), near-far filter delta={args.grid_delta}, one persistent launch",
           "gteps": st.m_reach / (ms * 1e-3) / 1e9, "ms": ms, "phases": st.supersteps,
           "work_inflation": st.relaxations / st.m_reach,
           "parity": check32(g, g.num_vertices)}
    rec["bsp"] = {"ms": bms, "supersteps": bst.supersteps,
                  "work_inflation": bst.relaxations / bst.m_reach,
                  "gteps": bst.m_reach / (bms * 1e-3) / 1e9, "parity": bsp_check}
    out.append(rec)
    g.free()
    if args.s26:
        g = gb.rmat(26, args.edgefactor, seed=args.seed, wtype="f32", transpose=False, ctx=ctx)
        ms, st = timed(g, 3)
        rec = {"config": "BASELINE configs[4]'s graph on ONE GPU (the N=1 point of the "
                         "scaling target): RMAT s26 EF16 fp32, default loop",
               "gteps": st.m_reach / (ms * 1e-3) / 1e9, "ms": ms,
               "supersteps": st.supersteps, "m_reach": st.m_reach,
               "work_inflation": st.relaxations / st.m_reach}
        if not args.no_cpu:  # the last timed call's result, certified at full size
            t0 = time.perf_counter()
            d, p = gb.sssp_read(g, native=True)
            ro, col, w = g.csr()
            rec["parity"] = dict(sp_certificate(ro, col, w, d, p, 0),
                                 seconds=round(time.perf_counter() - t0, 1))
            del ro, col, w, d, p
        out.append(rec)
        g.free()
    return out


def run_e2e(gb, ctx, g, args, kw):
    """Public API, host buffers: refill (H2D + device build) + sssp + D2H.

    The headline uses the reference Graph's own arrays -- row_offsets u32,
    column_indices u32, values() as double (graph.hpp:76-78) -- exactly what
    the C++ device policy uploads; the f32-host variant (a caller that keeps
    fp32 weights) is reported beside it."""
    import torch  # pinned host memory only
    ro, col, w = g.csr()
    n = g.num_vertices
    p_ro = torch.from_numpy(ro).pin_memory().numpy()
    p_col = torch.from_numpy(col).pin_memory().numpy()
    dist = torch.empty(n, dtype=torch.float64).pin_memory().numpy()
    pred = torch.empty(n, dtype=torch.int32).pin_memory().numpy().view(np.uint32)
    lib = gb._lib.load()
    o = gb._opts(**kw)

    def measure(p_w, htype):
        st = gb.SsspStats()
        times = []
        steps = max(1, args.e2e_steps)
        for i in range(1 + steps):
            t0 = time.perf_counter()
            gb.check(lib.gfb_graph_refill(g.h, C.c_void_p(p_ro.ctypes.data),
                                          C.c_void_p(p_col.ctypes.data),
                                          C.c_void_p(p_w.ctypes.data), htype))
            gb.check(lib.gfb_sssp(ctx.h, g.h, 0, C.byref(o), C.c_void_p(dist.ctypes.data),
                                  C.c_void_p(pred.ctypes.data), C.byref(st)))
            dt = time.perf_counter() - t0
            if i > 0:
                times.append(dt)
        t = sum(times) / len(times)
        return st, t, steps, ro.nbytes + col.nbytes + p_w.nbytes

    p_w64 = torch.from_numpy(w.astype(np.float64)).pin_memory().numpy()
    st, t, steps, h2d = measure(p_w64, gb.W_F64)
    del p_w64
    p_w32 = torch.from_numpy(w).pin_memory().numpy()
    st32, t32, _, h2d32 = measure(p_w32, gb.W_F32)
    d2h = dist.nbytes + pred.nbytes
    # leave the graph as the timed steps saw it (fp32 contents, relabel on reuse)
    return {"value": st.m_reach / t / 1e9, "unit": "GTEPS", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": t * 1e3, "steps": steps,
            "path": "gfb_graph_refill(pinned reference-layout CSR, values() as double; device "
                    "CSR build, transpose on first use) + gfb_sssp(dist f64, pred)",
            "h2d_note": "h2d_bytes_per_step counts the caller's host arrays; the library narrows "
                        "the f64 weights to the graph's f32 on the host (16 threads, AVX2, "
                        "pipelined with the copies), so PCIe carries %d bytes per step"
                        % int(ro.nbytes + col.nbytes + 4 * len(col)),
            "f32_host_weights": {"value": st32.m_reach / t32 / 1e9, "ms_per_step": t32 * 1e3,
                                 "h2d_bytes_per_step": int(h2d32)}}


def spawn_ranks(args):
    """--gpus N without torchrun: re-launch under torch.distributed.run."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    log(f"[bench] {args.gpus} ranks: {' '.join(cmd)}")
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--edgefactor", type=int, default=16)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--direction", default="push", choices=["auto", "push", "pull"])
    ap.add_argument("--alpha", type=float, default=1.05)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--soak", type=float, default=1.5, help="min warm-up seconds (clock samples)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the full-size oracle/CPU legs")
    ap.add_argument("--cpu-all", action="store_true",
                    help="also time the reference sssp() seq and par at full size (minutes)")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--s26", type=int, default=1, help="secondary RMAT s26 line on one GPU")
    ap.add_argument("--grid-side", type=int, default=4096)
    ap.add_argument("--grid-delta", type=float, default=16.0)
    ap.add_argument("--partitioned", action="store_true",
                    help="force the 1-D partitioned path (default for N > 1)")
    ap.add_argument("--no-relabel", action="store_true",
                    help="partitioned path: keep the generator's vertex ids")
    ap.add_argument("--exchange", default="peer", choices=["peer", "nccl"],
                    help="partitioned path: device-initiated peer-memory exchange (default) "
                         "or the host-driven NCCL all-to-all")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(spawn_ranks(args))
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

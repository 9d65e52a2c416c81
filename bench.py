#!/usr/bin/env python3
"""bench.py — BFS GTEPS on Graph500 R-MAT through the SIMD-X ACC engine (B200).

Contract (see the task statement and DESIGN.md "Measurement"):
  python bench.py --gpus N --steps K --warmup W [--impl reference]
prints ONE JSON line on rank 0.

Workload (N=1): BFS from vertex 0 on R-MAT scale 24, edge factor 16
(Graph500 A,B,C = .57,.19,.19; 16.8M vertices, ~537M directed edges), the
north_star bar configuration.  A "step" is one full BFS — every §8(a) row of
the hot path: state init, JIT online/ballot filters, thread/warp/CTA/grid
binning, push->pull->push switching, fused persistent kernels with the grid
barrier — over the device-resident graph.  GTEPS = Graph500 m_cc / time, m_cc =
undirected edges of the traversed component (sum of reached degrees / 2).
The CSR (2.15 GB of col) is larger than L2 (126 MB), so no flush is needed.

Extra keys: SSSP GTEPS, PageRank (20 iterations) and k-core decomposition ms on
the same graph; roofline of the dominant kernel; the oracle timed on the host.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GTEPS for BFS/SSSP on R-MAT; PageRank/k-core ms; HBM GB/s vs peak, 1-8 GPUs"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no nvidia-smi samples"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 2 + i and s[2 + i] == "Active"})
        loaded = [x for x in sm if x > 500] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def make_graph(scale, ef, seed):
    import simgen
    t = time.time()
    g = simgen.rmat(scale, ef, seed, wmin=1, wmax=255)
    log(f"[bench] R-MAT s{scale} ef{ef}: n={g.n} m={g.m} generated on host in {time.time() - t:.1f}s")
    return g


def m_cc_of(g, level):
    import numpy as np
    deg = g.degree().astype(np.int64)
    return int(deg[level != 0xFFFFFFFF].sum() // 2)


# ---------------------------------------------------------------------------- reference arm
def run_reference(args):
    """--impl reference: the oracle (single-threaded C, host) on the same workload/metric."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle
    g = make_graph(args.scale, args.ef, args.seed)
    t0 = time.perf_counter()
    lv = oracle.bfs(g, 0)
    t1 = time.perf_counter() - t0
    m_cc = oracle.traversed_edges(g, lv)
    for _ in range(max(0, min(args.warmup, 1) - 1)):
        oracle.bfs(g, 0)
    budget = args.ref_budget_s
    k = max(1, min(args.steps, int(budget / max(t1, 1e-3))))
    ts = []
    for _ in range(k):
        t0 = time.perf_counter()
        oracle.bfs(g, 0)
        ts.append(time.perf_counter() - t0)
    sec = sum(ts) / len(ts)
    v = m_cc / sec / 1e9
    sample = f"{k} full BFS runs from vertex 0 on R-MAT s{args.scale} (each {sec:.2f} s)"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "GTEPS", "n_gpus": world, "steps": k,
        "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": f"BFS from vertex 0, R-MAT scale {args.scale} edge factor {args.ef}",
                   "scale": args.scale, "edgefactor": args.ef, "m_cc": m_cc},
        "cpu_baseline": {"value": v, "unit": "GTEPS", "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------------------- our arm
def run_simdx(args):
    import numpy as np
    import torch

    import simgen
    from paper_1812_04070_b200 import simdx

    world, rank, local = dist_env()
    if world > 1:
        raise SystemExit("bench.py: the multi-GPU (1D partition + NCCL) layer is not built yet; run with --gpus 1")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    peak, peak_src = peaks()

    g = make_graph(args.scale, args.ef, args.seed)
    ctx = simdx.Context(local, stream.cuda_stream)
    G = ctx.upload(g)
    level = torch.empty(g.n, dtype=torch.int32, device=dev)

    # ---- warm-up + one instrumented run
    for _ in range(args.warmup):
        G.bfs(0, out=level)
    _, st, trace = G.bfs(0, out=level, trace_cap=64)
    lv_host = level.cpu().numpy().view(np.uint32)
    m_cc = m_cc_of(g, lv_host)
    log(f"[bench] BFS stats: {st}")
    log(f"[bench] BFS trace: " + " | ".join(
        f"it{t['iter']} {'pull' if t['dir'] else 'push'} {'ballot' if t['filter'] == 1 else 'online'} "
        f"|F'|={t['n_frontier']} L{t['launch']}" for t in trace))

    # ---- timed region: K BFS steps, CUDA events on the ctx stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    ms_push = ms_pull = b_push = b_pull = 0.0
    l_push = l_pull = 0
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            _, s, _ = G.bfs(0, out=level)
            launches += 1 + s["launches"]  # bfs_init + persistent launches
            ms_push += s["ms_push"]
            ms_pull += s["ms_pull"]
            b_push += s["bytes_push"]
            b_pull += s["bytes_pull"]
            l_push += s["launches_push"]
            l_pull += s["launches_pull"]
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    gteps = m_cc / (ms * 1e-3) / 1e9
    clocks = clk.summary()

    # roofline of the dominant kernel (largest share of the step's device time)
    dom = "bfs_pull" if ms_pull >= ms_push else "bfs_push"
    dms, dbytes, dl = (ms_pull, b_pull, l_pull) if dom == "bfs_pull" else (ms_push, b_push, l_push)
    achieved = (dbytes / args.steps) / (dms / args.steps * 1e-3) / 1e9 if dms > 0 else 0.0
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(f"s{args.scale}", {}).get(dom)
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "peak_source": peak_src,
                "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                "bytes_per_step": dbytes / args.steps, "kernel_ms_per_step": dms / args.steps,
                "kernel_share_of_step": (dms / args.steps) / ms, "launches_per_step": dl / args.steps,
                "step_bytes_model": (b_push + b_pull) / args.steps,
                "step_gbs": (b_push + b_pull) / args.steps / (ms * 1e-3) / 1e9}

    # ---- extras on the same graph (not part of the timed step)
    extras = {}
    if not args.no_extras:
        dist = torch.empty(g.n, dtype=torch.int32, device=dev)
        G.sssp(0, args.delta, out=dist)
        t = []
        for _ in range(3):
            _, s, _ = G.sssp(0, args.delta, out=dist)
            t.append(s["ms"])
        dh = dist.cpu().numpy().view(np.uint32)
        extras["sssp"] = {"delta": args.delta, "ms": min(t), "gteps": m_cc_of(g, dh) / (min(t) * 1e-3) / 1e9,
                          "iterations": s["iterations"], "hbm_gbs": s["bytes_model"] / (s["ms"] * 1e-3) / 1e9}
        rank_out = torch.empty(g.n, dtype=torch.float32, device=dev)
        G.pagerank(0.85, 20, out=rank_out)
        t = []
        for _ in range(3):
            _, s, _ = G.pagerank(0.85, 20, out=rank_out)
            t.append(s["ms"])
        extras["pagerank"] = {"iters": 20, "ms": min(t), "hbm_gbs": s["bytes_model"] / (s["ms"] * 1e-3) / 1e9,
                              "frac": s["bytes_model"] / (s["ms"] * 1e-3) / 1e9 / peak}
        core = torch.empty(g.n, dtype=torch.int32, device=dev)
        G.kcore(0, out=core)
        _, s, _ = G.kcore(0, out=core)
        extras["kcore"] = {"k": 0, "ms": s["ms"], "iterations": s["iterations"],
                           "hbm_gbs": s["bytes_model"] / (s["ms"] * 1e-3) / 1e9}
        log(f"[bench] extras: {extras}")

    # ---- e2e: host CSR (pinned) -> upload -> BFS -> host levels, through the C ABI
    e2e = None
    if not args.no_e2e:
        rp = torch.from_numpy(g.row_ptr.view(np.int64)).pin_memory()
        ci = torch.from_numpy(g.col.view(np.int32)).pin_memory()
        out_h = torch.empty(g.n, dtype=torch.int32).pin_memory()
        h2d = rp.numel() * 8 + ci.numel() * 4
        d2h = out_h.numel() * 4
        ts = []
        for i in range(args.e2e_steps + 1):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            h = simdx.sx_graph_upload(ctx.h, g.n, rp, ci)
            Ge = simdx.Graph(ctx, h, g.n)
            Ge.bfs(0, out=out_h)
            Ge.free()
            torch.cuda.synchronize()
            if i:
                ts.append(time.perf_counter() - t0)
        sec = sum(ts) / len(ts)
        e2e = {"value": m_cc / sec / 1e9, "unit": "GTEPS", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": sec * 1e3, "steps": len(ts),
               "what": "sx_graph_upload(pinned host CSR) + sx_bfs(host level_out) + sx_graph_free"}

    # ---- CPU baseline: the oracle on rank 0's host cores, bounded sample
    cpu = None
    if not args.no_cpu and rank == 0:
        import oracle
        ts = []
        t_start = time.perf_counter()
        while True:
            t0 = time.perf_counter()
            ref = oracle.bfs(g, 0)
            ts.append(time.perf_counter() - t0)
            if time.perf_counter() - t_start > args.cpu_budget_s or len(ts) >= 8:
                break
        ok = bool(np.array_equal(ref, lv_host))
        sec = min(ts)
        cpu = {"value": m_cc / sec / 1e9, "unit": "GTEPS", "cores": 1, "kind": "oracle",
               "sample": f"{len(ts)} full single-threaded BFS runs from vertex 0 on the same graph (min {sec:.2f} s)",
               "parity_with_gpu": ok}

    G.free()
    ctx.close()
    out = {
        "metric": METRIC, "value": gteps, "unit": "GTEPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": f"BFS from vertex 0, R-MAT scale {args.scale} edge factor {args.ef} "
                               f"(Graph500 A,B,C=.57,.19,.19, seed {args.seed}), 1D partition over {world} GPU(s)",
                   "scale": args.scale, "edgefactor": args.ef, "n": g.n, "m_directed": g.m, "m_cc": m_cc,
                   "l2": "inputs larger than L2 (col array 4*m bytes >> 126 MB); no flush",
                   "parallelism": f"1d{world}"},
        "gpu_launches": launches, "clocks": clocks, "roofline": roofline, "e2e": e2e, "cpu_baseline": cpu,
        "bfs": {"iterations": st["iterations"], "launches": st["launches"], "pull_iters": st["pull_iters"],
                "ballot_iters": st["ballot_iters"], "edges_examined": st["edges_examined"]},
        "extras": extras,
    }
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="simdx", choices=["simdx", "reference"])
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--ef", type=int, default=16)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--delta", type=int, default=1024)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-budget-s", type=float, default=15.0)
    ap.add_argument("--ref-budget-s", type=float, default=60.0)
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        log("[bench] warm-up raised to 3 (timing rule)")
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_simdx(args)


if __name__ == "__main__":
    main()

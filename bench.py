#!/usr/bin/env python3
"""bench.py — BFS GTEPS on Graph500 R-MAT through the SIMD-X ACC engine (B200).

Contract (task statement):
  python bench.py --gpus N --steps K --warmup W [--impl reference]
prints ONE JSON line on rank 0.  N > 1 is launched with torchrun (one process
per GPU); the driver computes scaling efficiency itself.

Workload: BFS from vertex 0 on R-MAT scale 24 + log2(N), edge factor 16
(Graph500 A,B,C = .57,.19,.19): 2^24 vertices (~537M directed edges) per GPU —
weak scaling; N = 1 is the north_star bar config (s24), N = 8 is C5 (s27).  A
step is one full BFS: state init, the JIT online/ballot filters, the
thread/warp/CTA/grid binning, push->pull->push switching, the fused persistent
kernels with their grid barrier (N = 1) or the per-level NCCL exchanges of the
1D partition (N > 1), over a device-resident graph.  GTEPS = Graph500 m_cc /
time, m_cc = undirected edges of the traversed component (sum of reached
degrees / 2).  The CSR (4m bytes of col) exceeds L2 (126 MB): no flush needed.
Graphs are built on the GPU by simgen's GPU generator, bit-identical to its CPU
generator (tests/test_gpu_gen.py).
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
            time.sleep(0.3)  # let the sampler start before the timed region
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
        mx = [float(s[1]) for s in self.samples if len(s) > 1 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 2 + i and s[2 + i] == "Active"})
        loaded = [x for x in sm if x > 500] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def timed_loop(fn, steps, stream):
    """Run fn() `steps` times between CUDA events on `stream`; returns ms per step."""
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


# ---------------------------------------------------------------------------- reference arm
def run_reference(args):
    """--impl reference: the oracle (single-threaded C on the host) on the same workload and metric.
    Nothing of the product package is imported here (its __init__ would load libsimdx.so)."""
    world, rank = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    import simgen
    scale = args.scale + max(0, world - 1).bit_length()  # weak scaling: 2^scale vertices per GPU
    t = time.time()
    g = simgen.rmat(scale, args.ef, args.seed)
    log(f"[bench:ref] R-MAT s{scale}: generated on the host in {time.time() - t:.1f}s")
    t0 = time.perf_counter()
    lv = oracle.bfs(g, 0)
    t1 = time.perf_counter() - t0
    m_cc = oracle.traversed_edges(g, lv)
    k = max(1, min(args.steps, int(args.ref_budget_s / max(t1, 1e-3))))
    ts = []
    for _ in range(k):
        t0 = time.perf_counter()
        oracle.bfs(g, 0)
        ts.append(time.perf_counter() - t0)
    sec = sum(ts) / len(ts)
    v = m_cc / sec / 1e9
    sample = f"{k} full BFS runs from vertex 0 on R-MAT s{scale} (mean {sec:.2f} s each)"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "GTEPS", "n_gpus": world, "steps": k,
        "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": f"BFS from vertex 0, R-MAT scale {scale} edge factor {args.ef}", "scale": scale,
                   "edgefactor": args.ef, "m_cc": m_cc},
        "cpu_baseline": {"value": v, "unit": "GTEPS", "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------------------- one GPU
def run_single(args):
    import numpy as np
    import torch

    import simgen
    from paper_1812_04070_b200 import simdx

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)
    peak, peak_src = peaks()
    t = time.time()
    dg = simgen.rmat_gpu(args.scale, args.ef, args.seed, 1, 255, stream=stream.cuda_stream)
    log(f"[bench] R-MAT s{args.scale}: n={dg.n} m={dg.m} built on the GPU in {time.time() - t:.2f}s")
    ctx = simdx.Context(0, stream.cuda_stream)
    G = ctx.upload_device(dg)
    n = dg.n
    level = torch.empty(n, dtype=torch.int32, device=dev)
    bkw = {"fusion": 2, "cluster_enter": 0} if args.mode == "async" else {} if args.fusion == 1 else {
        "fusion": args.fusion}
    for _ in range(args.warmup):
        if args.mode == "async":
            G.bfs_async(0, level)
        else:
            G.bfs(0, out=level, **bkw)
    _, st, trace = G.bfs(0, out=level, trace_cap=64, **bkw)
    lv = level.cpu().numpy().view(np.uint32)
    log(f"[bench] BFS stats: {st}")
    log("[bench] BFS trace: " + " | ".join(
        f"it{t['iter']} {'pull' if t['dir'] else 'push'} {'ballot' if t['filter'] == 1 else 'online'} "
        f"|F'|={t['n_frontier']} L{t['launch']}" for t in trace))

    # ---- timed region: K BFS steps
    host = dg.to_host()  # input generator output (bit-identical to simgen.rmat), for m_cc / e2e / oracle
    deg = np.diff(host.row_ptr).astype(np.int64)
    m_cc = int(deg[lv != 0xFFFFFFFF].sum() // 2)
    K = args.steps
    if args.mode == "async":
        # sx_bfs_async: each step = ONE all-fusion persistent launch (the state
        # init inside it), enqueued without a host round trip; the device-side
        # statistics and per-run CUDA events come back at sx_graph_sync
        G.sync()

        def step():
            G.bfs_async(0, level)

        with Clocks(0) as clk:
            ms = timed_loop(step, K, stream)
        clocks = clk.summary()
        sa = G.sync()
        assert sa["runs"] == K, sa
        # one bfs_all launch per step (state init inside), two with SX_ALL_INIT=0 (bfs_init + bfs_all)
        launches = (2 if os.environ.get("SX_ALL_INIT") == "0" else 1) * K
        dom, dms, dbytes, dl = "bfs_all", sa["ms_fused"], sa["bytes_model"], sa["launches_fused"]
        step_bytes = sa["bytes_model"]
    else:
        acc = dict(launches=0, ms_push=0.0, ms_pull=0.0, ms_fused=0.0, b_push=0.0, b_pull=0.0, l_push=0, l_pull=0,
                   l_fused=0)

        def step():
            _, s, _ = G.bfs(0, out=level, **bkw)
            # bfs_init + persistent launches (+ the control-tail copy kernel unless all fusion)
            acc["launches"] += 1 + s["launches"] + (0 if s["launches_fused"] else 1)
            for k in ("ms_push", "ms_pull", "ms_fused"):
                acc[k] += s[k]
            acc["b_push"] += s["bytes_push"]
            acc["b_pull"] += s["bytes_pull"]
            acc["l_push"] += s["launches_push"]
            acc["l_pull"] += s["launches_pull"]
            acc["l_fused"] += s["launches_fused"]

        with Clocks(0) as clk:
            ms = timed_loop(step, K, stream)
        clocks = clk.summary()
        launches = acc["launches"]
        step_bytes = acc["b_push"] + acc["b_pull"]
        if acc["l_fused"]:
            dom, dms, dbytes, dl = "bfs_all", acc["ms_fused"], step_bytes, acc["l_fused"]
        elif acc["ms_pull"] >= acc["ms_push"]:
            dom, dms, dbytes, dl = "bfs_pull", acc["ms_pull"], acc["b_pull"], acc["l_pull"]
        else:
            dom, dms, dbytes, dl = "bfs_push", acc["ms_push"], acc["b_push"], acc["l_push"]
    gteps = m_cc / (ms * 1e-3) / 1e9
    achieved = (dbytes / K) / (dms / K * 1e-3) / 1e9 if dms > 0 else 0.0
    traffic = None
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(f"s{args.scale}", {}).get(dom)
    except Exception:
        pass
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "peak_source": peak_src,
                "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                "bytes_per_step": dbytes / K, "kernel_ms_per_step": dms / K, "kernel_share_of_step": (dms / K) / ms,
                "launches_per_step": dl / K, "step_bytes_model": step_bytes / K,
                "step_gbs": step_bytes / K / (ms * 1e-3) / 1e9}

    # ---- extras on the same graph (outside the timed step)
    extras = {}
    if not args.no_extras:
        # Graph500-style: BFS from random roots of degree >= 1 (the timed step always
        # starts at vertex 0, the hub); harmonic mean of per-root GTEPS, device time
        # of each run (sx_stats.ms, CUDA events), all fusion
        rng = np.random.default_rng(args.seed)
        cand = np.flatnonzero(deg > 0)
        roots = rng.choice(cand, size=min(args.roots, cand.size), replace=False)
        deg_t = torch.from_numpy(deg).to(dev)
        tg = []
        for r in roots:
            _, s, _ = G.bfs(int(r), out=level, fusion=2, cluster_enter=0)
            mc = int(deg_t[level != -1].sum().item()) // 2
            tg.append(mc / (s["ms"] * 1e-3) / 1e9)
        extras["bfs_random_roots"] = {"roots": len(tg), "gteps_hmean": len(tg) / sum(1.0 / x for x in tg),
                                      "gteps_min": min(tg), "gteps_max": max(tg),
                                      "what": "device time per run (init + fused kernel), fusion = 2"}
        # fusion / filter ablation on this graph (Fig. 12/13 analogue):
        # device ms per BFS from vertex 0, best of 3
        abl = {}
        for name, kw in (("fusion0_none", dict(fusion=0)), ("fusion1_selective", {}),
                         ("fusion2_all", dict(fusion=2, cluster_enter=0)),
                         ("online_only", dict(force_filter=1)), ("ballot_only", dict(force_filter=2)),
                         ("push_only", dict(force_dir=1)), ("pull_only", dict(force_dir=2))):
            best = min((G.bfs(0, out=level, **kw)[1] for _ in range(3)), key=lambda x: x["ms"])
            abl[name] = {"ms": best["ms"], "launches": best["launches"], "iterations": best["iterations"]}
        extras["bfs_ablation"] = abl
        level.zero_()
        G.bfs(0, out=level)
        out = torch.empty(n, dtype=torch.int32, device=dev)
        G.sssp(0, args.delta, out=out)
        best = None
        for _ in range(3):
            _, s, _ = G.sssp(0, args.delta, out=out)
            best = s if best is None or s["ms"] < best["ms"] else best
        dh = out.cpu().numpy().view(np.uint32)
        m_s = int(deg[dh != 0xFFFFFFFF].sum() // 2)
        extras["sssp"] = {"delta": args.delta, "ms": best["ms"], "gteps": m_s / (best["ms"] * 1e-3) / 1e9,
                          "iterations": best["iterations"], "hbm_gbs": best["bytes_model"] / (best["ms"] * 1e-3) / 1e9}
        rk = torch.empty(n, dtype=torch.float32, device=dev)
        G.pagerank(0.85, 20, out=rk)
        best = None
        for _ in range(3):
            _, s, _ = G.pagerank(0.85, 20, out=rk)
            best = s if best is None or s["ms"] < best["ms"] else best
        gbs = best["bytes_model"] / (best["ms"] * 1e-3) / 1e9
        extras["pagerank"] = {"iters": 20, "ms": best["ms"], "hbm_gbs": gbs, "frac": gbs / peak}
        G.kcore(0, out=out)
        _, s, _ = G.kcore(0, out=out)
        extras["kcore"] = {"k": 0, "ms": s["ms"], "iterations": s["iterations"],
                           "hbm_gbs": s["bytes_model"] / (s["ms"] * 1e-3) / 1e9}
        _, s, _ = G.kcore(0, out=out, cluster_enter=0)
        extras["kcore_bsp_only"] = {"k": 0, "ms": s["ms"], "iterations": s["iterations"]}
        _, s, _ = G.kcore(16, out=out)
        extras["kcore_k16"] = {"k": 16, "ms": s["ms"], "iterations": s["iterations"]}
        G.wcc(out=out)
        _, s, _ = G.wcc(out=out)
        extras["wcc"] = {"ms": s["ms"], "iterations": s["iterations"], "launches": s["launches"]}
        us, ctas = simdx.sx_barrier_bench(ctx.h, 20000)
        extras["grid_barrier_us"] = {"us": us, "ctas": ctas}
        # the other single-GPU configs of BASELINE.json, built on the device through
        # the boundary (sx_graph_rmat / sx_graph_grid): C3 PageRank s22, C2 SSSP grid
        G3 = ctx.rmat(22, args.ef, args.seed)
        r3 = torch.empty(1 << 22, dtype=torch.float32, device=dev)
        G3.pagerank(0.85, 20, out=r3)
        best = None
        for _ in range(3):
            _, s, _ = G3.pagerank(0.85, 20, out=r3)
            best = s if best is None or s["ms"] < best["ms"] else best
        gbs = best["bytes_model"] / (best["ms"] * 1e-3) / 1e9
        extras["c3_pagerank_s22"] = {"iters": 20, "ms": best["ms"], "hbm_gbs": gbs, "frac": gbs / peak}
        # NEXT-3: PageRank to convergence (both recurrences; pull -> push tail) and BP to convergence
        r64 = torch.empty(1 << 22, dtype=torch.float64, device=dev)
        for var, eps in ((0, 1e-6), (1, 1e-6 * (1 << 22))):
            G3.pagerank_conv(0.85, eps, 10000, var, out=r64)
            _, s, _ = G3.pagerank_conv(0.85, eps, 10000, var, out=r64)
            extras[f"c3_pagerank_conv_v{var}"] = {"eps": eps, "ms": s["ms"], "iterations": s["iterations"],
                                                  "pull_iters": s["pull_iters"], "launches": s["launches"],
                                                  "residual": s["residual"]}
        del r64
        # SpMV (1 product) and BP (10 iterations) on the same graph, the same tiled pull
        x3 = torch.from_numpy(simgen.uniform_f32(args.seed, 1, 1 << 22, 0.0, 1.0)).to(dev)
        G3.spmv(x3, 1, out=r3)
        _, s, _ = G3.spmv(x3, 1, out=r3)
        extras["spmv_s22"] = {"ms": s["ms"], "hbm_gbs": s["bytes_model"] / (s["ms"] * 1e-3) / 1e9}
        pr3 = torch.from_numpy(simgen.bp_prior(args.seed, 1 << 22)).to(dev)
        G3.bp(pr3, 10, out=r3)
        _, s, _ = G3.bp(pr3, 10, out=r3)
        extras["bp_s22"] = {"iters": 10, "ms": s["ms"], "hbm_gbs": s["bytes_model"] / (s["ms"] * 1e-3) / 1e9}
        _, s, _ = G3.bp_conv(pr3, 1e-3 * (1 << 22), 200, out=r3)
        extras["bp_conv_s22"] = {"eps": 1e-3 * (1 << 22), "ms": s["ms"], "iterations": s["iterations"],
                                 "residual": s["residual"]}
        G3.free()
        # C5 at P = 1: R-MAT s27 (4.3 G edges) built on the device; BFS and SSSP device time
        try:
            G5 = ctx.rmat(27, args.ef, args.seed, 1, 255)
            n5 = 1 << 27
            o5 = torch.empty(n5, dtype=torch.int32, device=dev)
            G5.bfs(0, out=o5)
            b5 = min((G5.bfs(0, out=o5)[1] for _ in range(3)), key=lambda x: x["ms"])
            G5.sssp(0, args.delta, out=o5)
            s5 = G5.sssp(0, args.delta, out=o5)[1]
            G5.bfs(0, out=o5)
            rp5 = torch.empty(n5 + 1, dtype=torch.int64, device=dev)
            simdx.sx_graph_download(G5.h, rp5, None, None)
            mcc5 = int((rp5[1:] - rp5[:-1])[o5 != -1].sum().item()) // 2
            extras["c5_s27_one_gpu"] = {"bfs_ms": b5["ms"], "bfs_gteps": mcc5 / (b5["ms"] * 1e-3) / 1e9,
                                        "m_cc": mcc5, "sssp_ms": s5["ms"], "sssp_gteps": mcc5 / (s5["ms"] * 1e-3) / 1e9,
                                        "sssp_iterations": s5["iterations"]}
            del rp5
            G5.free()
            del o5
        except Exception as ex:  # memory-bound extra: never fail the bench line for it
            extras["c5_s27_one_gpu"] = {"error": str(ex)[:200]}
        G2 = ctx.grid(2048, 2048, args.seed, 1, 255)
        d2 = torch.empty(2048 * 2048, dtype=torch.int32, device=dev)
        G2.sssp(0, args.delta, out=d2)
        _, s, _ = G2.sssp(0, args.delta, out=d2)
        extras["c2_sssp_grid2048"] = {"delta": args.delta, "ms": s["ms"], "iterations": s["iterations"],
                                      "us_per_iteration": s["ms"] * 1e3 / max(1, s["iterations"]),
                                      "launches": s["launches"]}
        # filter / fusion ablation on the synthetic configs (the paper's Figs. 12-13,
        # P:1082-1093): device ms, best of 2; batch = every update recorded with duplicates
        # (P:536-545); k-core rows run BSP sub-rounds (cluster_enter = 0) unless named
        modes = (("jit", {}), ("online", dict(force_filter=1)), ("ballot", dict(force_filter=2)),
                 ("batch", dict(force_filter=3)), ("no_fusion", dict(fusion=0)))

        def best(fn, **kw):
            return min((fn(**kw)[1] for _ in range(2)), key=lambda x: x["ms"])["ms"]

        abl = {"c2_sssp_grid2048": {k: best(lambda **kw: G2.sssp(0, args.delta, out=d2, **kw), **kw) for k, kw in modes}}
        G2.free()
        abl["bfs_s24"] = {k: best(lambda **kw: G.bfs(0, out=level, **kw), **kw)
                          for k, kw in modes + (("all_fusion", dict(fusion=2, cluster_enter=0)),)}
        abl["c4_kcore_s24"] = {k: best(lambda **kw: G.kcore(0, out=out, cluster_enter=0, **kw), **kw) for k, kw in modes}
        abl["c4_kcore_s24"]["jit_async_tail"] = best(lambda **kw: G.kcore(0, out=out, **kw))
        G1 = ctx.rmat(16, args.ef, args.seed)
        l1 = torch.empty(1 << 16, dtype=torch.int32, device=dev)
        abl["c1_bfs_s16"] = {k: best(lambda **kw: G1.bfs(0, out=l1, **kw), **kw)
                             for k, kw in modes + (("all_fusion", dict(fusion=2, cluster_enter=0)),)}
        G1.free()
        extras["ablation_ms"] = abl
        log(f"[bench] extras: {extras}")

    # ---- e2e: pinned host CSR -> upload -> BFS -> host levels -> free, through the C ABI
    e2e = None
    if not args.no_e2e:
        rp = torch.from_numpy(host.row_ptr.view(np.int64)).pin_memory()
        ci = torch.from_numpy(host.col.view(np.int32)).pin_memory()
        out_h = torch.empty(n, dtype=torch.int32).pin_memory()
        ts = []
        for i in range(args.e2e_steps + 1):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            Ge = simdx.Graph(ctx, simdx.sx_graph_upload(ctx.h, n, rp, ci), n)
            Ge.bfs(0, out=out_h)
            Ge.free()
            torch.cuda.synchronize()
            if i:
                ts.append(time.perf_counter() - t0)
        sec = sum(ts) / len(ts)
        e2e = {"value": m_cc / sec / 1e9, "unit": "GTEPS", "h2d_bytes_per_step": rp.numel() * 8 + ci.numel() * 4,
               "d2h_bytes_per_step": out_h.numel() * 4, "ms_per_step": sec * 1e3, "steps": len(ts),
               "what": "sx_graph_upload(pinned host CSR) + sx_bfs(host level_out) + sx_graph_free"}

    # ---- CPU baseline: the oracle on this host, one core, bounded sample
    cpu = None
    if not args.no_cpu:
        import oracle
        ts = []
        t_start = time.perf_counter()
        while True:
            t0 = time.perf_counter()
            ref = oracle.bfs(host, 0)
            ts.append(time.perf_counter() - t0)
            if time.perf_counter() - t_start > args.cpu_budget_s or len(ts) >= 8:
                break
        sec = min(ts)
        cpu = {"value": m_cc / sec / 1e9, "unit": "GTEPS", "cores": 1, "kind": "oracle",
               "sample": f"{len(ts)} full single-threaded BFS runs from vertex 0 on the same graph (min {sec:.2f} s)",
               "parity_with_gpu": bool(np.array_equal(ref, lv))}

    G.free()
    dg.free()
    ctx.close()
    print(json.dumps({
        "metric": METRIC, "value": gteps, "unit": "GTEPS", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic",
        "config": {"workload": f"BFS from vertex 0, R-MAT scale {args.scale} edge factor {args.ef} "
                               f"(Graph500 A,B,C=.57,.19,.19, seed {args.seed}), 1 GPU",
                   "scale": args.scale, "edgefactor": args.ef, "n": n, "m_directed": int(host.m), "m_cc": m_cc,
                   "l2": "inputs larger than L2 (col array 4*m bytes >> 126 MB); no flush", "parallelism": "1d1"},
        "gpu_launches": launches, "clocks": clocks, "roofline": roofline, "e2e": e2e, "cpu_baseline": cpu,
        "bfs": {"iterations": st["iterations"], "launches": st["launches"], "pull_iters": st["pull_iters"],
                "ballot_iters": st["ballot_iters"], "edges_examined": st["edges_examined"]},
        "extras": extras,
    }), flush=True)


# ---------------------------------------------------------------------------- N GPUs (torchrun)
def run_dist(args, world, rank, local):
    import numpy as np
    import torch

    import simgen
    from paper_1812_04070_b200 import dist_host, simdx

    dist_host.init_group("gloo")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)
    scale = dist_host.weak_scale(args.scale, world)
    n = 1 << scale
    lo, hi = dist_host.partition(n, world, rank)
    t = time.time()
    dg = simgen.rmat_gpu(scale, args.ef, args.seed, 1, 255, v_lo=lo, v_hi=hi, stream=stream.cuda_stream)
    log(f"[bench r{rank}] R-MAT s{scale} slice [{lo},{hi}): m={dg.m} built in {time.time() - t:.2f}s")
    nid = dist_host.nccl_id_for_job(simdx.sx_nccl_unique_id)
    ctx = simdx.Context(local, stream.cuda_stream)
    D = simdx.Dist(ctx, n, world, rank, 1, nid)
    D.upload_device(0, dg)
    out = torch.empty(hi - lo, dtype=torch.int32, device=dev)
    # --fusion 2: the device-initiated BFS (one persistent kernel per rank, exchanges
    # over the NCCL device API); otherwise per-level host-issued collectives
    dkw = {"fusion": 2} if args.fusion == 2 else {}
    for _ in range(args.warmup):
        D.bfs(0, outs=[out], **dkw)
    acc = dict(launches=0)

    if args.fusion == 2:
        # device-initiated runs enqueued back to back (sx_dist_bfs_async), as the
        # single-GPU bench's async steps: no host round trip between steps
        def step():
            D.bfs_async(0, [out])
    else:
        def step():
            _, s = D.bfs(0, outs=[out], **dkw)
            acc["launches"] += s["launches"]

    dist_host.allreduce(0.0)  # barrier
    with Clocks(local) as clk:
        ms_local = timed_loop(step, args.steps, stream)
    if args.fusion == 2:
        acc["launches"] = D.sync()["launches"]
    ms = dist_host.allreduce(ms_local, "max")
    lv = out.cpu().numpy().view(np.uint32)
    host_rp = np.empty(hi - lo + 1, np.uint64)
    import ctypes
    simgen._LG().simgen_gpu_to_host(ctypes.c_void_p(host_rp.ctypes.data), dg.row_ptr_ptr, host_rp.nbytes)
    deg = np.diff(host_rp).astype(np.int64)
    m_cc = int(dist_host.allreduce(float(deg[lv != 0xFFFFFFFF].sum()), "sum") // 2)
    m_dir = int(dist_host.allreduce(float(dg.m), "sum"))
    gteps = m_cc / (ms * 1e-3) / 1e9
    _, st = D.bfs(0, outs=[out], **dkw)
    # ---- e2e at N GPUs: every rank re-uploads its slice from pinned host memory
    # (sx_dist_upload replaces the slice), runs the distributed BFS into a pinned
    # host level array; max over ranks of the wall time per step
    e2e = None
    if not args.no_e2e:
        hs = dg.to_host()
        rp_p = torch.from_numpy(hs.row_ptr.view(np.int64)).pin_memory().numpy().view(np.uint64)
        ci_p = torch.from_numpy(hs.col.view(np.int32)).pin_memory().numpy().view(np.uint32)
        w_p = torch.from_numpy(hs.w).pin_memory().numpy() if hs.w is not None else None
        out_h = torch.empty(hi - lo, dtype=torch.int32).pin_memory()

        class _Slice:
            row_ptr, col, w = rp_p, ci_p, w_p

        ts = []
        for i in range(args.e2e_steps + 1):
            dist_host.allreduce(0.0)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            D.upload(0, _Slice)
            D.bfs(0, outs=[out_h], **dkw)
            torch.cuda.synchronize()
            dt = dist_host.allreduce(time.perf_counter() - t0, "max")
            if i:
                ts.append(dt)
        sec = sum(ts) / len(ts)
        h2d = int(dist_host.allreduce(float(rp_p.nbytes + ci_p.nbytes + (w_p.nbytes if w_p is not None else 0)), "sum"))
        e2e = {"value": m_cc / sec / 1e9, "unit": "GTEPS", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": int(dist_host.allreduce(float(out_h.numel() * 4), "sum")),
               "ms_per_step": sec * 1e3, "steps": len(ts),
               "what": "per rank: sx_dist_upload(pinned host slice) + sx_dist_bfs(host level slice); max over ranks"}
    D.free()
    dg.free()
    ctx.close()
    if rank == 0:
        peak, peak_src = peaks()
        exch = st["bytes_model"]  # bytes of frontier bitmaps exchanged per rank per BFS
        print(json.dumps({
            "metric": METRIC, "value": gteps, "unit": "GTEPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": f"BFS from vertex 0, R-MAT scale {scale} edge factor {args.ef} "
                                   f"(2^{args.scale} vertices per GPU), 1D vertex partition over {world} GPUs, NCCL"
                                   + (" device API (one persistent kernel per rank, async steps)" if args.fusion == 2 else ""),
                       "scale": scale, "edgefactor": args.ef, "n": n, "m_directed": m_dir, "m_cc": m_cc,
                       "l2": "inputs larger than L2; no flush", "parallelism": f"1d{world}"},
            "gpu_launches": acc["launches"], "clocks": clk.summary(),
            "roofline": {"bound": "nvlink", "kernel": "per-level exchange", "achieved": exch / (ms * 1e-3) / 1e9,
                         "peak": 770.0, "peak_source": "B200_PROFILING.md measured peer copy per direction",
                         "unit": "GB/s", "frac": exch / (ms * 1e-3) / 1e9 / 770.0, "traffic": None,
                         "hbm_peak": peak, "hbm_peak_source": peak_src},
            "e2e": e2e, "cpu_baseline": None,
            "bfs": {"iterations": st["iterations"], "launches": st["launches"], "pull_iters": st["pull_iters"]},
        }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="simdx", choices=["simdx", "reference"])
    ap.add_argument("--scale", type=int, default=24, help="R-MAT scale per GPU")
    ap.add_argument("--ef", type=int, default=16)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--fusion", type=int, default=1, choices=[0, 1, 2],
                    help="--mode sync: 0 none, 1 selective (P:773-778), 2 all (one launch per BFS)")
    ap.add_argument("--mode", default="async", choices=["async", "sync"],
                    help="async: sx_bfs_async steps (all fusion, no host round trip); sync: sx_bfs per step")
    ap.add_argument("--roots", type=int, default=64, help="random-root BFS extra (Graph500 style, P:1003)")
    ap.add_argument("--delta", type=int, default=4096)  # measured best for C2 (profiles/r1/delta_sweep.txt)
    ap.add_argument("--dist", action="store_true",
                    help="run the multi-GPU path (NCCL communicator) even at one rank")
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
        return
    from paper_1812_04070_b200 import dist_host
    world, rank, local = dist_host.env_rank()
    if world != args.gpus:
        log(f"[bench] --gpus {args.gpus} but WORLD_SIZE={world}: using WORLD_SIZE")
    if world == 1 and not args.dist:
        run_single(args)
    else:
        run_dist(args, world, rank, local)


if __name__ == "__main__":
    main()

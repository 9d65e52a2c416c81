"""acc_model — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The ACC processing loop of PAPER.md §3.3 (Fig. 4(b) lines 12-21)
and the three task-management filters of §4, written step by step
in the paper's order for tiny graphs in pure Python.  It exists to pin the
paper's worked examples (Fig. 1; Fig. 6)
and the per-iteration frontier semantics the GPU trace is compared with.

One BSP iteration:
  1. Active:  the frontier = vertices whose metadata changed in
                            the previous iteration (SSSP), or were newly visited (BFS).
  2. Compute:  update_{v->u} = compute(M_v, M_(v,u), M_u) for every
                            out-edge of every active v.
  3. Combine:  update_u = (+)_v update_{v->u}; min for SSSP, vote for BFS.
  4. Filters produce the next active list:
       batch: every edge whose update changed u appends u -> unsorted, redundant
       ballot: scan the "updated" flags in vertex order -> sorted, unique
       online: record u while computing -> possibly redundant / unordered
  Metadata is applied immediately as edges are processed ("immediately
  updates vertex metadata"), in the order the active list gives.
"""
from __future__ import annotations

INF = 0xFFFFFFFF


def _adj(g, v):
    b, e = int(g.row_ptr[v]), int(g.row_ptr[v + 1])
    ws = [1] * (e - b) if g.w is None else [int(x) for x in g.w[b:e]]
    return list(zip([int(x) for x in g.col[b:e]], ws))


def run(g, src: int, algo: str = "sssp", max_iters: int = 1 << 20):
    """Run ACC from `src`; algo in {"sssp", "bfs"}.  Returns (metadata, trace).

    trace[i] (iteration i+1) = dict(active, batch, ballot, online, bits, updated_meta)
    """
    n = g.n
    meta = [INF] * n
    meta[src] = 0
    active = [src]
    trace = []
    it = 0
    while active and it < max_iters:
        it += 1
        batch, online = [], []
        updated = [False] * n
        for v in active:
            for u, w in _adj(g, v):
                if algo == "sssp":
                    upd = meta[v] + w            # Compute: dist(v) + w
                    if upd < meta[u]:            # Combine: min
                        meta[u] = upd
                        updated[u] = True
                        batch.append(u)
                        online.append(u)
                else:                            # BFS: vote
                    if meta[u] == INF:
                        meta[u] = it
                        updated[u] = True
                        batch.append(u)
                        online.append(u)
        ballot = [u for u in range(n) if updated[u]]      # sorted, unique
        bits = "".join("1" if updated[u] else "0" for u in range(n))
        trace.append(dict(active=list(active), batch=batch, ballot=ballot, online=online, bits=bits,
                          meta=list(meta)))
        active = ballot
    return meta, trace


def classify(deg: int, sep_small: int = 32, sep_large: int = 128) -> str:
    """Thread / warp / CTA class (boundary ownership: reading 17)."""
    if deg < sep_small:
        return "small"
    if deg < sep_large:
        return "medium"
    return "large"


def eq1_ctas(regs_per_smx: int, regs_per_thread: int, threads_per_cta: int, smx: int) -> int:
    """Eq. 1: #CTA = floor(regsPerSMX / (regsPerThread * threadsPerCTA)) * #SMX.
    (The example at P:756 prints ceil; floor gives its stated 60 — reading 4.)"""
    return (regs_per_smx // (regs_per_thread * threads_per_cta)) * smx

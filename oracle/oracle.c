/*
 * oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct, single-threaded CPU reference for every
 * result the SIMD-X ACC hot path computes (PAPER.md = arXiv 1812.04070 text,
 * cited as P:<line>; SURVEY.md §8(c) gives the readings).  May be loaded only
 * by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs.  Shares no code with paper_1812_04070_b200/ (the
 * CUDA path) and never calls it.
 *
 * Where the method reaches a result with a plain definition (BFS levels,
 * shortest-path distances, coreness) this file is that definition written out
 * with the textbook algorithm; PageRank, SpMV and BP are fixed-iteration Jacobi
 * recurrences written term by term in fp64.
 *
 * Graph input: CSR rows (row_ptr u64[n+1], col u32[m]); weights u8 or u32
 * (wbytes 1 / 4, or 0 = unweighted).  Pull-side functions take the
 * in-neighbour rows (CSC), which for an undirected graph are the CSR itself
 * (P:913).  Vertex-state sentinel for "unreached" is 0xFFFFFFFF.
 *
 * Parity pins: tests/test_oracle.py (all functions pinned).  BP's model is
 * this build's reading 15 (the paper names no model); its recurrence is
 * pinned at T = 1..4 by hand-derived closed forms and by exact rational BP in
 * the tanh form (fractions), which fail if any step feeds the prior instead of
 * the current log-odds.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define INF32 0xFFFFFFFFu

static inline uint32_t wt(const void* w, int wbytes, uint64_t e) {
    if (!w || wbytes == 0) return 1u;
    return wbytes == 1 ? ((const uint8_t*)w)[e] : ((const uint32_t*)w)[e];
}

/* C-B, BFS: level(v) = hop distance from src; queue BFS. */
int oracle_bfs(uint64_t n, const uint64_t* row_ptr, const uint32_t* col, uint32_t src, uint32_t* level) {
    for (uint64_t v = 0; v < n; ++v) level[v] = INF32;
    if (n == 0) return 0;
    if (src >= n) return -1;
    uint32_t* q = (uint32_t*)malloc(n * sizeof(uint32_t));
    if (!q) return -2;
    uint64_t head = 0, tail = 0;
    level[src] = 0;
    q[tail++] = src;
    while (head < tail) {
        uint32_t v = q[head++];
        for (uint64_t e = row_ptr[v]; e < row_ptr[v + 1]; ++e) {
            uint32_t u = col[e];
            if (level[u] == INF32) {
                level[u] = level[v] + 1;
                q[tail++] = u;
            }
        }
    }
    free(q);
    return 0;
}

/* ---- binary heap keyed by (dist, vertex) with lazy deletion ---- */
typedef struct { uint64_t d; uint32_t v; } hent;

static void heap_push(hent* h, uint64_t* sz, hent x) {
    uint64_t i = (*sz)++;
    while (i > 0) {
        uint64_t p = (i - 1) / 2;
        if (h[p].d <= x.d) break;
        h[i] = h[p];
        i = p;
    }
    h[i] = x;
}

static hent heap_pop(hent* h, uint64_t* sz) {
    hent top = h[0];
    hent x = h[--(*sz)];
    uint64_t i = 0, n = *sz;
    for (;;) {
        uint64_t l = 2 * i + 1, r = l + 1, m = i;
        uint64_t md = x.d;
        if (l < n && h[l].d < md) { m = l; md = h[l].d; }
        if (r < n && h[r].d < md) { m = r; }
        if (m == i) break;
        h[i] = h[m];
        i = m;
    }
    if (n > 0) h[i] = x;
    return top;
}

/* C-S, SSSP ("positive edge weights"):
 * dist(v) = min over paths of the sum of weights; binary-heap Dijkstra.
 * Returns -3 if a weight is 0 or a distance does not fit below 2^32-1. */
int oracle_sssp(uint64_t n, const uint64_t* row_ptr, const uint32_t* col, const void* w, int wbytes,
                uint32_t src, uint32_t* dist) {
    for (uint64_t v = 0; v < n; ++v) dist[v] = INF32;
    if (n == 0) return 0;
    if (src >= n) return -1;
    uint64_t m = row_ptr[n];
    uint64_t* d = (uint64_t*)malloc(n * sizeof(uint64_t));
    hent* h = (hent*)malloc((m + 1) * sizeof(hent));
    uint8_t* done = (uint8_t*)calloc(n, 1);
    if (!d || !h || !done) { free(d); free(h); free(done); return -2; }
    for (uint64_t v = 0; v < n; ++v) d[v] = UINT64_MAX;
    uint64_t sz = 0;
    d[src] = 0;
    heap_push(h, &sz, (hent){0, src});
    int rc = 0;
    while (sz > 0) {
        hent x = heap_pop(h, &sz);
        if (done[x.v]) continue;
        done[x.v] = 1;
        for (uint64_t e = row_ptr[x.v]; e < row_ptr[x.v + 1]; ++e) {
            uint32_t we = wt(w, wbytes, e);
            if (we == 0) rc = -3;
            uint32_t u = col[e];
            uint64_t nd = x.d + we;
            if (nd < d[u]) {
                d[u] = nd;
                heap_push(h, &sz, (hent){nd, u});
            }
        }
    }
    for (uint64_t v = 0; v < n; ++v) {
        if (d[v] == UINT64_MAX) continue;
        if (d[v] >= INF32) rc = -3;
        dist[v] = (uint32_t)d[v];
    }
    free(d); free(h); free(done);
    return rc;
}

/* C-K, coreness (SURVEY.md §8(c) reading 6):
 * core(v) = max{k : v in the k-core}, the k-core being the maximal induced
 * sub-multigraph with minimum degree >= k (duplicate edges count, reading 19).
 * Batagelj & Zaversnik's O(m) bucket algorithm (2003). */
int oracle_coreness(uint64_t n, const uint64_t* row_ptr, const uint32_t* col, uint32_t* core) {
    if (n == 0) return 0;
    uint64_t* deg = (uint64_t*)malloc(n * sizeof(uint64_t));
    uint64_t maxd = 0;
    for (uint64_t v = 0; v < n; ++v) {
        deg[v] = row_ptr[v + 1] - row_ptr[v];
        if (deg[v] > maxd) maxd = deg[v];
    }
    uint64_t* bin = (uint64_t*)calloc(maxd + 2, sizeof(uint64_t));
    uint32_t* vert = (uint32_t*)malloc(n * sizeof(uint32_t));
    uint64_t* pos = (uint64_t*)malloc(n * sizeof(uint64_t));
    if (!deg || !bin || !vert || !pos) { free(deg); free(bin); free(vert); free(pos); return -2; }
    for (uint64_t v = 0; v < n; ++v) bin[deg[v]]++;
    uint64_t start = 0;
    for (uint64_t d = 0; d <= maxd; ++d) {
        uint64_t num = bin[d];
        bin[d] = start;
        start += num;
    }
    for (uint64_t v = 0; v < n; ++v) {
        pos[v] = bin[deg[v]];
        vert[pos[v]] = (uint32_t)v;
        bin[deg[v]]++;
    }
    for (uint64_t d = maxd; d >= 1; --d) bin[d] = bin[d - 1];
    bin[0] = 0;
    for (uint64_t i = 0; i < n; ++i) {
        uint32_t v = vert[i];
        for (uint64_t e = row_ptr[v]; e < row_ptr[v + 1]; ++e) {
            uint32_t u = col[e];
            if (deg[u] > deg[v]) {
                uint64_t du = deg[u], pu = pos[u], pw = bin[du];
                uint32_t w = vert[pw];
                if (u != w) {
                    pos[u] = pw; vert[pu] = w;
                    pos[w] = pu; vert[pw] = u;
                }
                bin[du]++;
                deg[u]--;
            }
        }
    }
    for (uint64_t v = 0; v < n; ++v) core[v] = (uint32_t)deg[v];
    free(deg); free(bin); free(vert); free(pos);
    return 0;
}

/* C-P, PageRank after T Jacobi steps (readings 14):
 *   r_0(u) = 1/N
 *   r_{t+1}(u) = (1-d)/N + d * ( sum_{v in in(u)} r_t(v)/outdeg(v) + D_t/N ),
 *   D_t = sum_{outdeg(v)=0} r_t(v)           (dangling mass redistributed)
 * out_ptr: out-CSR row pointers (for outdeg); in_ptr/in_idx: in-neighbours. */
int oracle_pagerank(uint64_t n, const uint64_t* out_ptr, const uint64_t* in_ptr, const uint32_t* in_idx,
                    double d, uint32_t iters, double* rank) {
    if (n == 0) return 0;
    double* r = (double*)malloc(n * sizeof(double));
    double* rn = (double*)malloc(n * sizeof(double));
    if (!r || !rn) { free(r); free(rn); return -2; }
    const double N = (double)n;
    for (uint64_t v = 0; v < n; ++v) r[v] = 1.0 / N;
    for (uint32_t t = 0; t < iters; ++t) {
        double D = 0.0;
        for (uint64_t v = 0; v < n; ++v)
            if (out_ptr[v + 1] == out_ptr[v]) D += r[v];
        for (uint64_t u = 0; u < n; ++u) {
            double s = 0.0;
            for (uint64_t e = in_ptr[u]; e < in_ptr[u + 1]; ++e) {
                uint32_t v = in_idx[e];
                s += r[v] / (double)(out_ptr[v + 1] - out_ptr[v]);
            }
            rn[u] = (1.0 - d) / N + d * (s + D / N);
        }
        double* tmp = r; r = rn; rn = tmp;
    }
    memcpy(rank, r, n * sizeof(double));
    free(r); free(rn);
    return 0;
}

/* C-PC, PageRank to convergence ("updates the rank value of one vertex
 * ... iteratively till all vertices have stable rank values"; the stopping
 * test and both recurrences are readings 25-26 of DESIGN.md):
 *   variant 0 (reading 14, normalised):  r_0 = 1/N,
 *       r_{t+1}(u) = (1-d)/N + d * ( sum_{v in in(u)} r_t(v)/outdeg(v) + D_t/N ),
 *       D_t = sum_{outdeg(v)=0} r_t(v)
 *   variant 1 (un-normalised, dangling mass dropped): r_0 = 1,
 *       r_{t+1}(u) = (1-d) + d * sum_{v in in(u)} r_t(v)/outdeg(v)
 * Jacobi steps until the L1 change delta_t = sum_u |r_{t+1}(u) - r_t(u)| < eps
 * ("converged when L1 delta < epsilon"), at most max_iter steps.
 * *iters = steps taken; *last_delta = the last delta_t. */
int oracle_pagerank_conv(uint64_t n, const uint64_t* out_ptr, const uint64_t* in_ptr, const uint32_t* in_idx,
                         double d, double eps, uint32_t max_iter, int variant, double* rank, uint32_t* iters,
                         double* last_delta) {
    *iters = 0;
    *last_delta = 0.0;
    if (n == 0) return 0;
    double* r = (double*)malloc(n * sizeof(double));
    double* rn = (double*)malloc(n * sizeof(double));
    if (!r || !rn) { free(r); free(rn); return -2; }
    const double N = (double)n;
    for (uint64_t v = 0; v < n; ++v) r[v] = variant == 0 ? 1.0 / N : 1.0;
    for (uint32_t t = 0; t < max_iter; ++t) {
        double D = 0.0;
        if (variant == 0)
            for (uint64_t v = 0; v < n; ++v)
                if (out_ptr[v + 1] == out_ptr[v]) D += r[v];
        double delta = 0.0;
        for (uint64_t u = 0; u < n; ++u) {
            double s = 0.0;
            for (uint64_t e = in_ptr[u]; e < in_ptr[u + 1]; ++e) {
                uint32_t v = in_idx[e];
                s += r[v] / (double)(out_ptr[v + 1] - out_ptr[v]);
            }
            rn[u] = variant == 0 ? (1.0 - d) / N + d * (s + D / N) : (1.0 - d) + d * s;
            delta += fabs(rn[u] - r[u]);
        }
        double* tmp = r; r = rn; rn = tmp;
        *iters = t + 1;
        *last_delta = delta;
        if (delta < eps) break;
    }
    memcpy(rank, r, n * sizeof(double));
    free(r); free(rn);
    return 0;
}

/* C-V, SpMV (north_star; not in the paper): y[u] = sum_{(v,u) in E} w(v,u) * x[v],
 * w = float(weight) or 1 when unweighted; fp64 accumulation. */
int oracle_spmv(uint64_t n, const uint64_t* in_ptr, const uint32_t* in_idx, const void* in_w, int wbytes,
                const float* x, double* y) {
    for (uint64_t u = 0; u < n; ++u) {
        double s = 0.0;
        for (uint64_t e = in_ptr[u]; e < in_ptr[u + 1]; ++e)
            s += (double)wt(in_w, wbytes, e) * (double)x[in_idx[e]];
        y[u] = s;
    }
    return 0;
}

/* C-BP, belief propagation log-odds after T Jacobi steps ("all
 * vertices active", P:340 sum-combine; the model itself is this build's
 * reading 15):
 *   psi(x_v, x_u) = c if x_v == x_u else 1-c,  c = 0.25 + 0.5*(weight-1)/254
 *   (unweighted graph: weight 255, c = 0.75)
 *   l_0(u) = logit(p_u)
 *   l_{t+1}(u) = logit(p_u) + sum_{v in in(u)} log( (c b + (1-c)(1-b)) / (c (1-b) + (1-c) b) ),
 *   b = sigmoid(l_t(v)).
 * abs_terms (nullable) receives sum |log(...)| of the final step (tolerance scale). */
int oracle_bp(uint64_t n, const uint64_t* in_ptr, const uint32_t* in_idx, const void* in_w, int wbytes,
              const float* prior, uint32_t iters, double* logodds, double* abs_terms) {
    if (n == 0) return 0;
    double* l = (double*)malloc(n * sizeof(double));
    double* ln = (double*)malloc(n * sizeof(double));
    double* lp = (double*)malloc(n * sizeof(double));
    if (!l || !ln || !lp) { free(l); free(ln); free(lp); return -2; }
    for (uint64_t u = 0; u < n; ++u) {
        double p = (double)prior[u];
        lp[u] = log(p / (1.0 - p));
        l[u] = lp[u];
        if (abs_terms) abs_terms[u] = 0.0;
    }
    for (uint32_t t = 0; t < iters; ++t) {
        for (uint64_t u = 0; u < n; ++u) {
            double s = 0.0, sa = 0.0;
            for (uint64_t e = in_ptr[u]; e < in_ptr[u + 1]; ++e) {
                double weight = in_w && wbytes ? (double)wt(in_w, wbytes, e) : 255.0;
                double c = 0.25 + 0.5 * (weight - 1.0) / 254.0;
                double b = 1.0 / (1.0 + exp(-l[in_idx[e]]));
                double term = log((c * b + (1.0 - c) * (1.0 - b)) / (c * (1.0 - b) + (1.0 - c) * b));
                s += term;
                sa += fabs(term);
            }
            ln[u] = lp[u] + s;
            if (abs_terms && t + 1 == iters) abs_terms[u] = sa;
        }
        double* tmp = l; l = ln; ln = tmp;
    }
    memcpy(logodds, l, n * sizeof(double));
    free(l); free(ln); free(lp);
    return 0;
}

/* C-W, connected components of an undirected graph (WCC, named by the paper
 * as a voting workload): label(v) = the
 * smallest vertex id in v's component.  Ids are scanned in increasing order and
 * a queue BFS labels each component from its first (= smallest) unlabelled
 * vertex.  Undirected (symmetric) CSR only. */
int oracle_wcc(uint64_t n, const uint64_t* row_ptr, const uint32_t* col, uint32_t* label) {
    for (uint64_t v = 0; v < n; ++v) label[v] = INF32;
    if (n == 0) return 0;
    uint32_t* q = (uint32_t*)malloc(n * sizeof(uint32_t));
    if (!q) return -2;
    for (uint64_t s = 0; s < n; ++s) {
        if (label[s] != INF32) continue;
        uint64_t head = 0, tail = 0;
        label[s] = (uint32_t)s;
        q[tail++] = (uint32_t)s;
        while (head < tail) {
            uint32_t v = q[head++];
            for (uint64_t e = row_ptr[v]; e < row_ptr[v + 1]; ++e) {
                uint32_t u = col[e];
                if (label[u] == INF32) {
                    label[u] = (uint32_t)s;
                    q[tail++] = u;
                }
            }
        }
    }
    free(q);
    return 0;
}

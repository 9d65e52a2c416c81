// pull_all.cu — the all-active pull algorithms: PageRank, SpMV
// (north_star) and belief propagation.  Every vertex is active every
// iteration ("treats all vertices as active"), so the ballot filter runs
// exactly once, in iteration 1, to build the class lists ("BP and
// PageRank need the ballot filter at exactly the first iteration"); the lists
// are then static.  Each iteration is a pull:
//   Compute : update_{v->u} = term(M_v, M_(v,u))   over in-edges of u
//   Combine : sum (agg_sum)
//     small  (thread granularity): one thread per vertex, 16 gathers in flight
//     medium (warp granularity):   lane-strided 128-bit loads + shuffle tree
//     large + huge (CTA / grid granularity): the two lists are concatenated and
//       split edge-balanced over every thread of the grid (B200 design: a CTA
//       per vertex leaves the latency of each row exposed); fp64 atomics only
//       where a thread's slice ends inside a row, then the owner applies.
//   Apply   : a single owner writes M_u (atomic-free), Jacobi double
//             buffering between iterations; fp64 accumulation, fp32 state (BP: fp64).
#include <cmath>

#include "internal.h"

namespace sx {

// ---------------------------------------------------------------- operators
struct PrOp {  // r(u) = (1-d)/N + d (sum_v r(v)/outdeg(v) + D/N)
    float* contrib[2];
    float* out;
    const uint32_t* dout;
    double d, invN;
    // per-iteration
    uint32_t cur;
    double D;
    bool last;
    __device__ __forceinline__ double edge(const DevGraph&, uint64_t, uint32_t v) const { return (double)contrib[cur][v]; }
    __device__ __forceinline__ void init(uint64_t v, double& dpart) const {
        const uint32_t dv = dout[v];
        contrib[0][v] = dv ? (float)(invN / (double)dv) : 0.f;
        if (dv == 0) dpart += invN;
    }
    __device__ __forceinline__ void apply(uint32_t u, double s, double& dpart) const {
        const double r = (1.0 - d) * invN + d * (s + D * invN);
        if (last) out[u] = (float)r;
        const uint32_t du = dout[u];
        contrib[cur ^ 1][u] = du ? (float)(r / (double)du) : 0.f;
        if (du == 0) dpart += r;
    }
};

struct SpmvOp {  // y(u) = sum_v w(v,u) x(v)
    const float* x;
    float* out;
    uint32_t cur;
    double D;
    bool last;
    __device__ __forceinline__ double edge(const DevGraph& g, uint64_t e, uint32_t v) const {
        return (double)edge_w(g.iw8, g.iw32, e) * (double)x[v];
    }
    __device__ __forceinline__ void init(uint64_t, double&) const {}
    __device__ __forceinline__ void apply(uint32_t u, double s, double&) const { out[u] = (float)s; }
};

// BP is computed in fp64 end to end (beliefs, couplings, messages), fp32 out.
// Measured: this loopy recurrence amplifies a 1-ulp fp32 perturbation (even of
// the coupling c alone) to ~1e-4 after 10 steps on R-MAT, so fp32 state cannot
// meet the 1e-5 conditioned tolerance.
struct BpOp {  // l(u) = logit(p_u) + sum_v log((c b + (1-c)(1-b)) / (c(1-b) + (1-c) b)), b = sigmoid(l(v))
    double* b[2];
    const float* prior;
    float* out;
    uint32_t cur;
    double D;
    bool last;
    __device__ __forceinline__ double edge(const DevGraph& g, uint64_t e, uint32_t v) const {
        const double wt = (g.iw8 || g.iw32) ? (double)edge_w(g.iw8, g.iw32, e) : 255.0;
        const double c = 0.25 + 0.5 * (wt - 1.0) / 254.0;
        const double bv = b[cur][v];
        const double num = c * bv + (1.0 - c) * (1.0 - bv);
        const double den = c * (1.0 - bv) + (1.0 - c) * bv;
        return log(num / den);
    }
    __device__ __forceinline__ void init(uint64_t v, double&) const {
        const double p = (double)prior[v];
        const double l = log(p / (1.0 - p));
        b[0][v] = 1.0 / (1.0 + exp(-l));
    }
    __device__ __forceinline__ void apply(uint32_t u, double s, double&) const {
        const double p = (double)prior[u];
        const double l = log(p / (1.0 - p)) + s;
        if (last) out[u] = (float)l;
        b[cur ^ 1][u] = 1.0 / (1.0 + exp(-l));
    }
};

template <class Op> struct PullP {
    DevGraph g;
    Sched s;
    Op op;
    uint32_t iters;
    double* hacc;         // per big-list entry partial sums (fp64)
    uint64_t* loff;       // prefix sums of in-degrees over the big list (nb + 1 entries)
    uint64_t* scratch;    // MAX_GRID u64 scan scratch
};

template <class Op> __device__ __forceinline__ double row_sum(const DevGraph& g, const Op& op, uint64_t beg, uint64_t end,
                                                              uint64_t rank, uint64_t size) {
    double acc = 0.0;
    for_edges(g.ici, beg, end, rank, size, [&](uint64_t e, uint32_t v) { acc += op.edge(g, e, v); });
    return acc;
}
template <class Op> __device__ __forceinline__ double row_seq(const DevGraph& g, const Op& op, uint64_t beg, uint64_t end) {
    return seq_sum(g.ici, beg, end, [&](uint64_t e, uint32_t v) { return op.edge(g, e, v); });
}

// Block-wide exclusive scan of one u64 per thread; returns the exclusive value and the block total.
__device__ __forceinline__ uint64_t block_excl_scan_u64(uint64_t x, uint64_t& total) {
    __shared__ uint64_t ws[WARPS];
    uint64_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(FULL, inc, o);
        if ((int)lane_id() >= o) inc += y;
    }
    __syncthreads();
    if (lane_id() == 31) ws[warp_id()] = inc;
    __syncthreads();
    uint64_t before = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
        if (w < (int)warp_id()) before += ws[w];
        tot += ws[w];
    }
    total = tot;
    return before + inc - x;
}

// The large and huge class lists, concatenated ("big" list, nb entries).
__device__ __forceinline__ uint32_t big_at(const uint32_t* L, uint64_t cs, uint32_t c2, uint32_t i) {
    return i < c2 ? L[2 * cs + i] : L[3 * cs + (i - c2)];
}

template <class Op> __global__ void __launch_bounds__(BLOCK, 4) pull_all(PullP<Op> p) {
    Ctl* c = p.s.ctl;
    grid_begin(c);
    const uint64_t n = p.g.n;
    const uint64_t cs = p.s.cstride;
    Stats st;
    uint32_t cnt[NCLS];
    // iteration 1 task management: ballot filter over all vertices -> static class lists (in-degree)
    if (!ballot_filter(AllWords{n}, p.s, BallotOut{p.s.lists[0], cs, p.g.din}, cnt)) return;
    ++st.ballot;
    st.scanned += n;
    {
        double dpart = 0.0;
        for (uint64_t v = gtid(); v < n; v += gthreads()) p.op.init(v, dpart);
        double a[1] = {dpart};
        block_sum<1>(a);
        if (threadIdx.x == 0 && a[0] != 0.0) atomicAdd(&c->line[0].s[my_slot()].dsum, a[0]);
    }
    if (!grid_sync(c)) return;
    const uint32_t* L = p.s.lists[0];
    // CTA / grid granularity for the big list: one edge-balanced stream over the
    // concatenated rows of the large and huge vertices.  loff = exclusive prefix
    // sums of their in-degrees (grid scan, once; the lists are static).
    const uint32_t nb = cnt[2] + cnt[3];
    {
        const uint32_t per = (nb + gridDim.x - 1) / gridDim.x;
        const uint32_t i0 = min(nb, per * blockIdx.x), i1 = min(nb, i0 + per);
        uint64_t part = 0;
        for (uint32_t i = i0 + threadIdx.x; i < i1; i += BLOCK) part += __ldg(p.g.din + big_at(L, cs, cnt[2], i));
        uint64_t a[1] = {part};
        block_sum<1>(a);
        if (threadIdx.x == 0) p.scratch[blockIdx.x] = a[0];
        if (!grid_sync(c)) return;
        uint64_t r[2] = {0, 0};
        for (uint32_t b = threadIdx.x; b < gridDim.x; b += BLOCK) {
            const uint64_t x = vload(p.scratch + b);
            if (b < blockIdx.x) r[0] += x;
            r[1] += x;
        }
        block_sum<2>(r);
        uint64_t run = r[0];
        for (uint32_t t0 = i0; t0 < i1; t0 += BLOCK) {
            const uint32_t i = t0 + threadIdx.x;
            const uint64_t d = i < i1 ? __ldg(p.g.din + big_at(L, cs, cnt[2], i)) : 0;
            uint64_t tt;
            const uint64_t ex = block_excl_scan_u64(d, tt);
            if (i < i1) p.loff[i] = run + ex;
            run += tt;
        }
        if (lead()) p.loff[nb] = r[1];
        if (!grid_sync(c)) return;
    }
    const uint64_t Eb = nb ? vload(p.loff + nb) : 0;
    // this thread's slice [x0, x1) of the big stream and its first segment (static)
    const uint64_t T = gthreads();
    const uint64_t x0 = Eb * gtid() / T, x1 = Eb * (gtid() + 1) / T;
    uint32_t seg0 = 0;
    if (x0 < x1) {
        uint32_t lo = 0, hi = nb;  // largest i with loff[i] <= x0
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (vload(p.loff + mid) <= x0) lo = mid;
            else hi = mid;
        }
        seg0 = lo;
    }
    Op op = p.op;
    for (uint32_t t = 0; t < p.iters; ++t) {
        maybe_reset_line(&c->line[(t + 2) % 3]);
        {
            LineSum ls;
            read_line(&c->line[t % 3], ls);
            op.D = ls.dsum;
        }
        op.cur = t & 1;
        op.last = t + 1 == p.iters;
        double dpart = 0.0;
        uint64_t edges = 0;
        // big list: edge-balanced slices, fp64 atomics only at segment ends
        for (uint64_t x = x0, i = seg0; x < x1; ++i) {
            const uint32_t u = big_at(L, cs, cnt[2], (uint32_t)i);
            const uint64_t s0 = p.loff[i], s1 = p.loff[i + 1];
            const uint64_t end = min(s1, x1);
            const uint64_t base = __ldg(p.g.irp + u) - s0;
            const double a = row_seq(p.g, op, base + x, base + end);
            atomicAdd(p.hacc + i, a);
            edges += end - x;
            x = end;
        }
        // medium: one warp per vertex
        for (uint64_t i = gwarp(); i < cnt[1]; i += gwarps()) {
            const uint32_t u = L[cs + i];
            const uint64_t beg = __ldg(p.g.irp + u), end = __ldg(p.g.irp + u + 1);
            const double a = warp_sum(row_sum(p.g, op, beg, end, lane_id(), 32));
            if (lane_id() == 0) {
                op.apply(u, a, dpart);
                edges += end - beg;
            }
        }
        // small: one thread per vertex
        for (uint64_t i = gtid(); i < cnt[0]; i += gthreads()) {
            const uint32_t u = L[i];
            const uint64_t beg = __ldg(p.g.irp + u), end = __ldg(p.g.irp + u + 1);
            op.apply(u, row_seq(p.g, op, beg, end), dpart);
            edges += end - beg;
        }
        if (nb) {
            if (!grid_sync(c)) return;
            // owners apply the big vertices' sums
            for (uint64_t i = gtid(); i < nb; i += gthreads()) {
                op.apply(big_at(L, cs, cnt[2], (uint32_t)i), p.hacc[i], dpart);
                p.hacc[i] = 0.0;
            }
        }
        {
            double a[1] = {dpart};
            block_sum<1>(a);
            if (threadIdx.x == 0 && a[0] != 0.0) atomicAdd(&c->line[(t + 1) % 3].s[my_slot()].dsum, a[0]);
        }
        st.edges += edges;
        if (lead()) st.entries += n;
        ++st.iters;
        if (!grid_sync(c)) return;
        trace_put(p.s, t + 1, DIR_PULL, t == 0 ? 1u : 2u, cnt, n, 0, 0);
    }
    st.pull = st.iters;
    flush_stats(c, st, DIR_PULL);
    if (lead()) {
        c->iter = p.iters;
        c->done = 1;
        grid_end(c);
        c->launch += 1;
    }
}

template __global__ void pull_all<PrOp>(PullP<PrOp>);
template __global__ void pull_all<SpmvOp>(PullP<SpmvOp>);
template __global__ void pull_all<BpOp>(PullP<BpOp>);

}  // namespace sx

using namespace sx;

namespace {

sx_status prep(sx_graph g, const char* who) {
    if (g->directed && !g->has_rev)
        return sxh::fail(SX_E_NO_REVERSE, std::string(who) + ": pull needs in-neighbour rows (CSC)");
    if (!g->hacc) {
        SX_CU(cudaMalloc(&g->hacc, (g->n + 1) * sizeof(double)));
        SX_CU(cudaMemsetAsync(g->hacc, 0, (g->n + 1) * sizeof(double), g->ctx->stream));
        SX_CU(cudaMalloc(&g->loff, (g->n + 1) * sizeof(uint64_t)));
        SX_CU(cudaMalloc(&g->scratch64, MAX_GRID * sizeof(uint64_t)));
    }
    return SX_OK;
}

// Algorithmic bytes of one pull-all iteration: every in-edge once
// (col 4 B + gathered source value + weight bytes), every vertex once
// (list 4 B + row_ptr 8 B + state read/write); set per operator.
thread_local double t_edge_bytes = 0, t_vertex_bytes = 0;
static double pull_bytes(const sx_graph g, const sxh::Counters& c) {
    return c.iters * ((double)g->mi * t_edge_bytes + (double)g->n * t_vertex_bytes) + c.scanned / 8.0;
}

template <class Op>
sx_status run_pull(sx_graph g, const sx_opts* opts, sx_stats* stats, const Op& op, uint32_t iters, double edge_bytes,
                   double vertex_bytes) {
    sxh::Run run{g, sxh::resolve_opts(opts), stats};
    sx_status rc = run.begin();
    if (rc != SX_OK) return rc;
    PullP<Op> p;
    p.g = sxh::dev_graph(g);
    p.s = sxh::make_sched(g, run.o);
    p.op = op;
    p.iters = iters;
    p.hacc = g->hacc;
    p.loff = g->loff;
    p.scratch = g->scratch64;
    void* args[] = {&p};
    if ((rc = run.launch((const void*)pull_all<Op>, args, true)) != SX_OK) return rc;
    t_edge_bytes = edge_bytes;
    t_vertex_bytes = vertex_bytes;
    return run.end(pull_bytes);
}

}  // namespace

extern "C" sx_status sx_pagerank(sx_graph g, float damping, uint32_t iters, const sx_opts* opts, float* rank_out,
                                 sx_stats* stats) {
    if (!g || !rank_out) return sxh::fail(SX_E_INVALID, "sx_pagerank: NULL graph or rank_out");
    sx_status rc = sxh::check_ctx(g->ctx);
    if (rc != SX_OK) return rc;
    if (!(damping >= 0.f && damping <= 1.f)) return sxh::fail(SX_E_INVALID, "sx_pagerank: damping outside [0,1]");
    if (iters == 0) return sxh::fail(SX_E_INVALID, "sx_pagerank: iters must be >= 1");
    if (g->n == 0) return SX_OK;
    if ((rc = prep(g, "sx_pagerank")) != SX_OK) return rc;
    const bool dev_out = sxh::is_device_ptr(rank_out);
    PrOp op;
    op.contrib[0] = (float*)g->st[0];
    op.contrib[1] = (float*)g->st[1];
    op.out = dev_out ? rank_out : (float*)g->st[2];
    op.dout = g->dout;
    op.d = damping;
    op.invN = 1.0 / (double)g->n;
    op.cur = 0;
    op.D = 0;
    op.last = false;
    // edge: col 4 + contrib 4; vertex: list 4 + row_ptr 8 + contrib write 4 + outdeg 4
    if ((rc = run_pull(g, opts, stats, op, iters, 8.0, 20.0)) != SX_OK) return rc;
    return dev_out ? SX_OK : sxh::copy_out(g, rank_out, op.out, g->n * 4);
}

extern "C" sx_status sx_spmv(sx_graph g, const float* x, uint32_t iters, const sx_opts* opts, float* y_out,
                             sx_stats* stats) {
    if (!g || !x || !y_out) return sxh::fail(SX_E_INVALID, "sx_spmv: NULL argument");
    sx_status rc = sxh::check_ctx(g->ctx);
    if (rc != SX_OK) return rc;
    if (iters == 0) return sxh::fail(SX_E_INVALID, "sx_spmv: iters must be >= 1");
    if (g->n == 0) return SX_OK;
    if ((rc = prep(g, "sx_spmv")) != SX_OK) return rc;
    const bool dev_out = sxh::is_device_ptr(y_out);
    SpmvOp op;
    float* dx = (float*)g->st[0];
    if ((rc = sxh::copy_in(g, dx, x, g->n * 4)) != SX_OK) return rc;
    op.x = dx;
    op.out = dev_out ? y_out : (float*)g->st[1];
    op.cur = 0;
    op.D = 0;
    op.last = false;
    if ((rc = run_pull(g, opts, stats, op, iters, 8.0 + g->wbytes, 16.0)) != SX_OK) return rc;
    return dev_out ? SX_OK : sxh::copy_out(g, y_out, op.out, g->n * 4);
}

extern "C" sx_status sx_bp(sx_graph g, const float* prior, uint32_t iters, const sx_opts* opts, float* logodds_out,
                           sx_stats* stats) {
    if (!g || !prior || !logodds_out) return sxh::fail(SX_E_INVALID, "sx_bp: NULL argument");
    sx_status rc = sxh::check_ctx(g->ctx);
    if (rc != SX_OK) return rc;
    if (iters == 0) return sxh::fail(SX_E_INVALID, "sx_bp: iters must be >= 1");
    if (g->n == 0) return SX_OK;
    if ((rc = prep(g, "sx_bp")) != SX_OK) return rc;
    if (!g->dstate) SX_CU(cudaMalloc(&g->dstate, 2 * g->n * sizeof(double)));
    const bool dev_out = sxh::is_device_ptr(logodds_out);
    BpOp op;
    op.b[0] = g->dstate;
    op.b[1] = g->dstate + g->n;
    float* dp = (float*)g->st[2];
    if ((rc = sxh::copy_in(g, dp, prior, g->n * 4)) != SX_OK) return rc;
    op.prior = dp;
    op.out = dev_out ? logodds_out : (float*)g->st[3];
    op.cur = 0;
    op.D = 0;
    op.last = false;
    // edge: col 4 + belief 8 + weight; vertex: list 4 + row_ptr 8 + prior 4 + belief write 8
    if ((rc = run_pull(g, opts, stats, op, iters, 12.0 + g->wbytes, 24.0)) != SX_OK) return rc;
    return dev_out ? SX_OK : sxh::copy_out(g, logodds_out, op.out, g->n * 4);
}

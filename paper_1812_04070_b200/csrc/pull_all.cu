// pull_all.cu — the all-active pull algorithms: PageRank, SpMV
// (north_star) and belief propagation.  Every vertex is active every
// iteration ("treats all vertices as active"), so the ballot filter runs
// exactly once, in iteration 1, to build the class lists ("BP and
// PageRank need the ballot filter at exactly the first iteration"); the lists
// are then static.  Each iteration is a pull:
//   Compute : update_{v->u} = term(M_v, M_(v,u))   over in-edges of u
//   Combine : sum (agg_sum) — thread-sequential (small),
//             lane-strided + shuffle tree (medium, warp), thread-strided + block
//             tree (large, CTA), grid-split + fp64 atomics (huge)
//   Apply   : a single owner writes M_u (atomic-free), Jacobi double
//             buffering between iterations; fp64 accumulation, fp32 state.
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
    double* hacc;
};

template <class Op> __device__ __forceinline__ double row_sum(const DevGraph& g, const Op& op, uint64_t beg, uint64_t end,
                                                              uint64_t rank, uint64_t size) {
    double acc = 0.0;
    for_edges(g.ici, beg, end, rank, size, [&](uint64_t e, uint32_t v) { acc += op.edge(g, e, v); });
    return acc;
}

template <class Op> __global__ void __launch_bounds__(BLOCK, 4) pull_all(PullP<Op> p) {
    Ctl* c = p.s.ctl;
    const uint64_t n = p.g.n;
    Stats st;
    uint32_t cnt[NCLS];
    // iteration 1 task management: ballot filter over all vertices -> static class lists (in-degree)
    if (!ballot_filter(AllWords{n}, p.s, BallotOut{p.s.lists[0], n, p.g.din}, cnt)) return;
    ++st.ballot;
    st.scanned += n;
    {
        double dpart = 0.0;
        for (uint64_t v = gtid(); v < n; v += gthreads()) p.op.init(v, dpart);
        double a[1] = {dpart};
        block_sum<1>(a);
        if (threadIdx.x == 0 && a[0] != 0.0) atomicAdd(&c->line[0].dsum, a[0]);
    }
    if (!grid_sync(c)) return;
    const uint32_t* L = p.s.lists[0];
    Op op = p.op;
    for (uint32_t t = 0; t < p.iters; ++t) {
        if (lead()) reset_line(&c->line[(t + 2) % 3]);
        op.cur = t & 1;
        op.D = vload(&c->line[t % 3].dsum);
        op.last = t + 1 == p.iters;
        double dpart = 0.0;
        uint64_t edges = 0;
        // huge: grid-split partial sums -> fp64 atomics -> barrier -> owners apply
        if (cnt[3]) {
            for (uint32_t i = 0; i < cnt[3]; ++i) {
                const uint32_t u = L[3 * n + i];
                const uint64_t beg = __ldg(p.g.irp + u), end = __ldg(p.g.irp + u + 1);
                double a[1] = {row_sum(p.g, op, beg, end, gtid(), gthreads())};
                block_sum<1>(a);
                if (threadIdx.x == 0) atomicAdd(p.hacc + i, a[0]);
                if (lead()) edges += end - beg;
            }
            if (!grid_sync(c)) return;
            for (uint64_t i = gtid(); i < cnt[3]; i += gthreads()) {
                op.apply(L[3 * n + i], vload(p.hacc + i), dpart);
                p.hacc[i] = 0.0;
            }
        }
        // large: one CTA per vertex
        for (uint32_t i = blockIdx.x; i < cnt[2]; i += gridDim.x) {
            const uint32_t u = L[2 * n + i];
            const uint64_t beg = __ldg(p.g.irp + u), end = __ldg(p.g.irp + u + 1);
            double a[1] = {row_sum(p.g, op, beg, end, threadIdx.x, BLOCK)};
            block_sum<1>(a);
            if (threadIdx.x == 0) {
                op.apply(u, a[0], dpart);
                edges += end - beg;
            }
        }
        // medium: one warp per vertex
        for (uint64_t i = gwarp(); i < cnt[1]; i += gwarps()) {
            const uint32_t u = L[n + i];
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
            op.apply(u, row_sum(p.g, op, beg, end, 0, 1), dpart);
            edges += end - beg;
        }
        {
            double a[1] = {dpart};
            block_sum<1>(a);
            if (threadIdx.x == 0 && a[0] != 0.0) atomicAdd(&c->line[(t + 1) % 3].dsum, a[0]);
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
        SX_CU(cudaMalloc(&g->hacc, (g->n ? g->n : 1) * sizeof(double)));
        SX_CU(cudaMemsetAsync(g->hacc, 0, (g->n ? g->n : 1) * sizeof(double), g->ctx->stream));
    }
    return SX_OK;
}

// Algorithmic bytes of one pull-all iteration: every in-edge once
// (col 4 B + gathered source value 4 B + weight bytes), every vertex once
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
    PrOp op;
    op.contrib[0] = (float*)g->st[0];
    op.contrib[1] = (float*)g->st[1];
    op.out = (float*)g->st[2];
    op.dout = g->dout;
    op.d = damping;
    op.invN = 1.0 / (double)g->n;
    op.cur = 0;
    op.D = 0;
    op.last = false;
    // edge: col 4 + contrib 4; vertex: list 4 + row_ptr 8 + contrib write 4 + outdeg 4
    if ((rc = run_pull(g, opts, stats, op, iters, 8.0, 20.0)) != SX_OK) return rc;
    return sxh::copy_out(g, rank_out, op.out, g->n * 4);
}

extern "C" sx_status sx_spmv(sx_graph g, const float* x, uint32_t iters, const sx_opts* opts, float* y_out,
                             sx_stats* stats) {
    if (!g || !x || !y_out) return sxh::fail(SX_E_INVALID, "sx_spmv: NULL argument");
    sx_status rc = sxh::check_ctx(g->ctx);
    if (rc != SX_OK) return rc;
    if (g->n == 0) return SX_OK;
    if (iters == 0) return sxh::fail(SX_E_INVALID, "sx_spmv: iters must be >= 1");
    if ((rc = prep(g, "sx_spmv")) != SX_OK) return rc;
    SpmvOp op;
    float* dx = (float*)g->st[0];
    if ((rc = sxh::copy_in(g, dx, x, g->n * 4)) != SX_OK) return rc;
    op.x = dx;
    op.out = (float*)g->st[1];
    op.cur = 0;
    op.D = 0;
    op.last = false;
    if ((rc = run_pull(g, opts, stats, op, iters, 8.0 + g->wbytes, 16.0)) != SX_OK) return rc;
    return sxh::copy_out(g, y_out, op.out, g->n * 4);
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
    BpOp op;
    op.b[0] = g->dstate;
    op.b[1] = g->dstate + g->n;
    float* dp = (float*)g->st[2];
    if ((rc = sxh::copy_in(g, dp, prior, g->n * 4)) != SX_OK) return rc;
    op.prior = dp;
    op.out = (float*)g->st[3];
    op.cur = 0;
    op.D = 0;
    op.last = false;
    // edge: col 4 + belief 8 + weight; vertex: list 4 + row_ptr 8 + prior 4 + belief write 8
    if ((rc = run_pull(g, opts, stats, op, iters, 12.0 + g->wbytes, 24.0)) != SX_OK) return rc;
    return sxh::copy_out(g, logodds_out, op.out, g->n * 4);
}

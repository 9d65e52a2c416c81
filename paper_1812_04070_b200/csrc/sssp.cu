// sssp.cu — SSSP as an ACC algorithm (§3.3; Fig. 4(a)).
//
//   Active  : vertices whose distance changed in the previous iteration
//   Compute : update_{v->u} = dist(v) + w(v,u)
//   Combine : min, applied with atomicMin on u32 distances — order
//             independent, so results are bit-exact (SURVEY.md §8(c) reading 11)
//   delta-stepping ([Meyer & Sanders]): an improved vertex with
//   dist < hi joins the next active list (claimed exactly once per iteration on
//   the next-frontier bitmap); otherwise it goes to the far pile (a bitmap).
//   When the near lists run dry the bucket advances to the smallest pending
//   distance: hi = (min_far / delta + 1) * delta, and the far vertices below hi
//   are moved to the active list by a ballot pass over the far bitmap.
//   delta = 0 means delta = infinity: frontier Bellman-Ford (reading 9).
#include "internal.h"

namespace sx {

struct SsspP {
    DevGraph g;
    Sched s;
    uint32_t* dist;
    uint32_t* far;
    uint32_t delta;
};

__global__ void sssp_init(SsspP p, uint32_t src) {
    Ctl* c = p.s.ctl;
    if (threadIdx.x < 32)
        for (int i = 0; i < 3; ++i) reset_line_warp(&c->line[i]);
    if (threadIdx.x != 0) return;
    p.dist[src] = 0;
    const uint32_t k = cls_of(p.g.dout[src], p.s);
    for (int i = 0; i < NCLS; ++i) c->cur_count[i] = 0;
    c->cur_count[k] = 1;
    p.s.lists[0][(uint64_t)k * p.s.cstride] = src;
    c->hi = p.delta ? (unsigned long long)p.delta : 0xFFFFFFFFull + 1;
    c->dir = DIR_PUSH;
    c->lists_ready = 1;
    c->slotted = 0;
    c->iter = 0;
    c->done = 0;
}

// Far-pile source for the bucket advance: far vertices with dist < hi.
struct FarWords {
    const uint32_t* far;
    const uint32_t* dist;
    uint64_t hi;
    __device__ __forceinline__ uint32_t word(uint64_t wi) const {
        uint32_t w = far[wi], out = 0;
        while (w) {
            const int b = __ffs(w) - 1;
            w &= w - 1;
            if ((uint64_t)dist[(wi << 5) + b] < hi) out |= 1u << b;
        }
        return out;
    }
};

__global__ void __launch_bounds__(BLOCK, 4) sssp_push(SsspP p) {
    Ctl* c = p.s.ctl;
    if (vload(&c->done)) return;
    grid_begin(c);
    uint32_t it = vload(&c->iter);
    uint64_t hi = vload(&c->hi);
    uint32_t cnt[NCLS];
    uint32_t slotted = vload(&c->slotted);
    if (slotted) {
        view_slots(&c->line[it % 3], p.s, cnt);
    } else {
        for (int i = 0; i < NCLS; ++i) cnt[i] = vload(&c->cur_count[i]);
        view_contig(cnt);
    }
    Stats st;
    uint32_t done = 0;
    for (;;) {
        IterLine* nx = &c->line[(it + 1) % 3];
        maybe_reset_line(&c->line[(it + 2) % 3]);
        clear_bitmap(p.s.bm[(it + 2) % 3], p.s.nwords);
        uint32_t* nlists = p.s.lists[(it + 1) & 1];
        uint32_t* nbm = p.s.bm[(it + 1) % 3];
        uint64_t edges = 0;
        for_tasks(p.s.lists[it & 1], p.s, cnt, [&](uint32_t v, uint64_t rank, uint64_t size, uint32_t) {
            const uint64_t beg = __ldg(p.g.rp + v), end = __ldg(p.g.rp + v + 1);
            const uint32_t dv = p.dist[v];
            for_edges(p.g.ci, beg, end, rank, size, [&](uint64_t e, uint32_t u) {
                ++edges;
                const uint32_t nd = dv + edge_w(p.g.w8, p.g.w32, e);
                if (nd >= p.dist[u]) return;
                const uint32_t old = atomicMin(p.dist + u, nd);
                if (nd >= old) return;
                if ((uint64_t)nd < hi) {
                    if (bm_claim(nbm, u)) online_record(nx, nlists, p.s, u, cls_of(__ldg(p.g.dout + u), p.s));
                } else {
                    bm_set(p.far, u);
                }
            });
        });
        st.edges += edges;
        if (lead()) st.entries += sum4(cnt);
        if (!grid_sync(c)) return;
        LineSum ls;
        uint32_t vcnt[NCLS];
        read_line_view(nx, p.s, ls, vcnt);
        const uint64_t nf = sum4(ls.cnt);
        bool overflow = false;
        for (int i = 0; i < NCLS; ++i) overflow |= ls.cntmax[i] > p.s.cap_s;
        if (p.s.force_filter == 2) overflow = true;
        ++it;
        ++st.iters;
        uint32_t filt = overflow ? 1u : 0u;
        if (nf > 0 && overflow) {
            ++st.ballot;
            st.scanned += p.s.nwords * 32;
            if (!ballot_filter(BitmapWords{nbm}, p.s, BallotOut{p.s.lists[it & 1], p.s.cstride, p.g.dout}, cnt)) return;
            if (!grid_sync(c)) return;
            view_contig(cnt);
            slotted = 0;
        } else {
            for (int i = 0; i < NCLS; ++i) cnt[i] = vcnt[i];  // view set by read_line_view
            slotted = 1;
        }
        if (nf == 0) {
            if (p.delta == 0) {
                trace_put(p.s, it, DIR_PUSH, filt, cnt, nf, 0, hi);
                done = 1;
                break;
            }
            // bucket advance: min distance over the far pile (into this line's minv slots)
            uint32_t mn = INF;
            for (uint64_t wi = gtid(); wi < p.s.nwords; wi += gthreads()) {
                uint32_t w = p.far[wi];
                while (w) {
                    const int b = __ffs(w) - 1;
                    w &= w - 1;
                    mn = min(mn, p.dist[(wi << 5) + b]);
                }
            }
            mn = block_min(mn);
            if (threadIdx.x == 0 && mn != INF) atomicMin(&nx->s[my_slot()].minv, mn);
            st.scanned += p.s.nwords * 32;
            if (!grid_sync(c)) return;
            read_line(nx, ls);
            mn = ls.minv;
            if (mn == INF) {
                trace_put(p.s, it, DIR_PUSH, filt, cnt, nf, 0, hi);
                done = 1;
                break;
            }
            hi = ((uint64_t)mn / p.delta + 1) * p.delta;
            ++st.ballot;
            FarWords src{p.far, p.dist, hi};
            if (!ballot_filter(src, p.s, BallotOut{p.s.lists[it & 1], p.s.cstride, p.g.dout}, cnt,
                               [&](uint32_t v, uint32_t) { p.far[v >> 5] &= ~(1u << (v & 31)); }))
                return;
            if (!grid_sync(c)) return;
            view_contig(cnt);
            slotted = 0;
            filt = 1;
        }
        trace_put(p.s, it, DIR_PUSH, filt, cnt, nf, 0, hi);
        if (p.s.max_iters && it >= p.s.max_iters) {
            done = 1;
            break;
        }
        if (!p.s.fusion) break;
    }
    flush_stats(c, st, DIR_PUSH);
    if (lead()) {
        c->iter = it;
        c->hi = hi;
        c->done = done;
        c->slotted = slotted;
        for (int i = 0; i < NCLS; ++i) c->cur_count[i] = cnt[i];
        grid_end(c);
        c->launch += 1;
    }
}

}  // namespace sx

using namespace sx;

// Algorithmic bytes: per list entry 4 B list + 16 B row_ptr pair +
// 4 B dist(v); per edge 4 B col + weight + 4 B dist(u); per iteration one
// bitmap clear (n/8); ballot / far scans n/8.
static double sssp_bytes(const sx_graph g, const sxh::Counters& c) {
    const double n = (double)g->n;
    return 24.0 * c.entries + (8.0 + g->wbytes) * c.edges + c.iters * n / 8.0 + c.scanned / 8.0;
}

extern "C" sx_status sx_sssp(sx_graph g, uint32_t src, uint32_t delta, const sx_opts* opts, uint32_t* dist_out,
                             sx_stats* stats) {
    if (!g || !dist_out) return sxh::fail(SX_E_INVALID, "sx_sssp: NULL graph or dist_out");
    sx_status rc = sxh::check_ctx(g->ctx);
    if (rc != SX_OK) return rc;
    if (g->n == 0) return sxh::fail(SX_E_INVALID, "sx_sssp: empty graph has no source");
    if (src >= g->n) return sxh::fail(SX_E_INVALID, "sx_sssp: src >= n");
    if (!g->w || g->wbytes == 0) return sxh::fail(SX_E_WEIGHT, "sx_sssp: graph has no edge weights");
    if (g->has_zero_w) return sxh::fail(SX_E_WEIGHT, "sx_sssp: zero edge weight (P:361 assumes positive weights)");
    sxh::Run run{g, sxh::resolve_opts(opts), stats};
    cudaStream_t s = g->ctx->stream;
    SsspP p;
    if ((rc = run.begin()) != SX_OK) return rc;
    p.g = sxh::dev_graph(g);
    p.s = sxh::make_sched(g, run.o);
    const bool dev_out = sxh::is_device_ptr(dist_out);
    p.dist = dev_out ? dist_out : g->st[0];
    p.far = g->aux_bm;
    p.delta = delta;
    SX_CU(cudaMemsetAsync(p.dist, 0xFF, g->n * 4, s));
    SX_CU(cudaMemsetAsync(p.far, 0, g->nwords * 4, s));
    for (int i = 0; i < 3; ++i) SX_CU(cudaMemsetAsync(p.s.bm[i], 0, g->nwords * 4, s));
    sssp_init<<<1, 32, 0, s>>>(p, src);
    SX_CU(cudaGetLastError());
    void* args[] = {&p};
    g->ctx->h_ctl->done = 0;
    for (;;) {
        if ((rc = run.launch((const void*)sssp_push, args, false)) != SX_OK) return rc;
        if ((rc = run.sync()) != SX_OK) return rc;
        if (g->ctx->h_ctl->done) break;
    }
    if ((rc = run.end(sssp_bytes)) != SX_OK) return rc;
    return dev_out ? SX_OK : sxh::copy_out(g, dist_out, p.dist, g->n * 4);
}

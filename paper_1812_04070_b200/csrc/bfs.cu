// bfs.cu — BFS as an ACC algorithm (PAPER.md; voting combine P:343-345).
//
//   Active  : vertices first reached in the previous level (frontier bitmap bm[it%3])
//   Compute : level(u) = it + 1 for an unvisited neighbour u
//   Combine : vote — any one update suffices; push claims u exactly once
//             with atomicOr on the visited bitmap; pull stops scanning u's
//             in-neighbours at the first frontier hit (collaborative early
//             termination) using __any_sync / __syncthreads_or.
//
// Selective fusion: one persistent cooperative kernel per direction
// run; it loops over BSP iterations with the grid barrier and exits only when
// the traversal ends or the direction switches (push -> pull -> push).
#include <cstring>

#include "internal.h"

namespace sx {

struct BfsP {
    DevGraph g;
    Sched s;
    uint32_t* level;
    uint32_t* visited;
};

__global__ void bfs_init(BfsP p, uint32_t src, uint32_t dir) {
    Ctl* c = p.s.ctl;
    for (int i = 0; i < 3; ++i) reset_line(&c->line[i]);
    p.level[src] = 0;
    p.visited[src >> 5] |= 1u << (src & 31);
    p.s.bm[0][src >> 5] |= 1u << (src & 31);
    const uint32_t d = p.g.dout[src];
    const uint32_t k = cls_of(d, p.s);
    for (int i = 0; i < NCLS; ++i) c->cur_count[i] = 0;
    c->cur_count[k] = 1;
    p.s.lists[0][(uint64_t)k * p.g.n] = src;
    c->m_u = p.g.m - d;
    c->nf_prev = 1;
    c->dir = dir;
    c->lists_ready = dir == DIR_PUSH ? 1u : 0u;
    c->iter = 0;
    c->done = 0;
    c->st_reached = 1;
}

__device__ __forceinline__ void bfs_exit(const BfsP& p, uint32_t it, uint64_t m_u, uint32_t nf_prev, uint32_t dir,
                                         uint32_t done, uint32_t ready, const uint32_t (&cnt)[NCLS], Stats& st) {
    Ctl* c = p.s.ctl;
    flush_stats(c, st);
    if (lead()) {
        c->iter = it;
        c->m_u = m_u;
        c->nf_prev = nf_prev;
        c->dir = dir;
        c->done = done;
        c->lists_ready = ready;
        for (int i = 0; i < NCLS; ++i) c->cur_count[i] = cnt[i];
        c->launch += 1;
    }
}

// ------------------------------------------------------------------ push
__global__ void __launch_bounds__(BLOCK, 4) bfs_push(BfsP p) {
    Ctl* c = p.s.ctl;
    if (vload(&c->done) || vload(&c->dir) != DIR_PUSH) return;
    const uint64_t n = p.g.n;
    uint32_t it = vload(&c->iter);
    uint64_t m_u = vload(&c->m_u);
    uint32_t nf_prev = vload(&c->nf_prev);
    uint32_t cnt[NCLS];
    Stats st;
    uint32_t dir = DIR_PUSH, done = 0, ready = 1;
    if (!vload(&c->lists_ready)) {
        // entering push from pull: the frontier exists only as a bitmap -> ballot filter
        if (!ballot_filter(BitmapWords{p.s.bm[it % 3]}, p.s, BallotOut{p.s.lists[it & 1], n, p.g.dout}, cnt)) return;
        st.scanned += p.s.nwords * 32;
        if (!grid_sync(c)) return;
    } else {
        for (int i = 0; i < NCLS; ++i) cnt[i] = vload(&c->cur_count[i]);
    }
    for (;;) {
        CntLine* nx = &c->line[(it + 1) % 3];
        if (lead()) reset_line(&c->line[(it + 2) % 3]);
        clear_bitmap(p.s.bm[(it + 2) % 3], p.s.nwords);
        uint32_t* nlists = p.s.lists[(it + 1) & 1];
        uint32_t* nbm = p.s.bm[(it + 1) % 3];
        const uint32_t lvl = it + 1;
        uint64_t mdeg = 0, edges = 0, reached = 0;
        for_tasks(p.s.lists[it & 1], n, cnt, [&](uint32_t v, uint64_t rank, uint64_t size, uint32_t) {
            const uint64_t beg = __ldg(p.g.rp + v), end = __ldg(p.g.rp + v + 1);
            for_edges(p.g.ci, beg, end, rank, size, [&](uint64_t, uint32_t u) {
                ++edges;
                if (bm_test(p.visited, u)) return;
                if (!bm_claim(p.visited, u)) return;
                p.level[u] = lvl;
                bm_set(nbm, u);
                const uint32_t du = __ldg(p.g.dout + u);
                mdeg += du;
                ++reached;
                online_record(nx, nlists, n, p.s.online_cap, u, cls_of(du, p.s));
            });
        });
        st.edges += edges;
        st.reached += reached;
        if (lead()) st.entries += sum4(cnt);
        {
            uint64_t v[1] = {mdeg};
            block_sum<1>(v);
            if (threadIdx.x == 0 && v[0]) atomicAdd(&nx->mdeg, (unsigned long long)v[0]);
        }
        if (!grid_sync(c)) return;
        uint32_t ncnt[NCLS];
        for (int i = 0; i < NCLS; ++i) ncnt[i] = vload(&nx->cnt[i]);
        const uint64_t nf = sum4(ncnt);
        const uint64_t mf = vload(&nx->mdeg);
        bool overflow = false;
        for (int i = 0; i < NCLS; ++i) overflow |= ncnt[i] > p.s.online_cap;
        if (p.s.force_filter == 2) overflow = true;
        m_u -= mf;
        ++it;
        ++st.iters;
        trace_put(p.s, it, DIR_PUSH, overflow ? 1u : 0u, ncnt, nf, mf, m_u);
        if (nf == 0 || (p.s.max_iters && it >= p.s.max_iters)) {
            done = 1;
            for (int i = 0; i < NCLS; ++i) cnt[i] = 0;
            break;
        }
        const bool to_pull = p.s.force_dir == 2 ||
                             (p.s.force_dir == 0 && (double)mf > (double)m_u / p.s.alpha && nf > nf_prev);
        nf_prev = (uint32_t)nf;
        if (to_pull) {
            dir = DIR_PULL;
            ready = 0;
            break;
        }
        if (overflow) {
            ++st.ballot;
            st.scanned += p.s.nwords * 32;
            if (!ballot_filter(BitmapWords{nbm}, p.s, BallotOut{p.s.lists[it & 1], n, p.g.dout}, cnt)) return;
            if (!grid_sync(c)) return;
        } else {
            for (int i = 0; i < NCLS; ++i) cnt[i] = ncnt[i];
        }
        if (!p.s.fusion) break;
    }
    bfs_exit(p, it, m_u, nf_prev, dir, done, ready, cnt, st);
}

// ------------------------------------------------------------------ pull
// Candidates = unvisited vertices with in-edges (ballot filter over
// ~visited & nz at entry); a candidate that finds no frontier in-neighbour is
// re-recorded for the next level (online, exactly once).
__global__ void __launch_bounds__(BLOCK, 4) bfs_pull(BfsP p) {
    Ctl* c = p.s.ctl;
    if (vload(&c->done) || vload(&c->dir) != DIR_PULL) return;
    const uint64_t n = p.g.n;
    uint32_t it = vload(&c->iter);
    uint64_t m_u = vload(&c->m_u);
    uint32_t nf_prev = vload(&c->nf_prev);
    uint32_t cnt[NCLS];
    Stats st;
    uint32_t dir = DIR_PULL, done = 0, ready = 1;
    if (!vload(&c->lists_ready)) {
        if (!ballot_filter(CandidateWords{p.visited, p.g.nz_in}, p.s, BallotOut{p.s.lists[it & 1], n, p.g.din}, cnt))
            return;
        st.scanned += p.s.nwords * 32;
        if (!grid_sync(c)) return;
    } else {
        for (int i = 0; i < NCLS; ++i) cnt[i] = vload(&c->cur_count[i]);
    }
    __shared__ uint32_t s_hit;
    for (;;) {
        CntLine* nx = &c->line[(it + 1) % 3];
        if (lead()) reset_line(&c->line[(it + 2) % 3]);
        clear_bitmap(p.s.bm[(it + 2) % 3], p.s.nwords);
        const uint32_t* cur = p.s.bm[it % 3];
        uint32_t* nbm = p.s.bm[(it + 1) % 3];
        uint32_t* nlists = p.s.lists[(it + 1) & 1];
        const uint32_t* L = p.s.lists[it & 1];
        const uint32_t lvl = it + 1;
        uint64_t mdeg = 0, edges = 0;
        uint32_t found = 0;
        auto mark = [&](uint32_t u) {
            p.level[u] = lvl;
            bm_set(p.visited, u);
            bm_set(nbm, u);
            mdeg += __ldg(p.g.dout + u);
            ++found;
        };
        // CTA granularity: large and huge candidates (early exit with __syncthreads_or)
        const uint32_t nbig = cnt[2] + cnt[3];
        for (uint32_t i = blockIdx.x; i < nbig; i += gridDim.x) {
            const uint32_t k = i < cnt[2] ? 2u : 3u;
            const uint32_t u = L[(uint64_t)k * n + (k == 2 ? i : i - cnt[2])];
            const uint64_t beg = __ldg(p.g.irp + u), end = __ldg(p.g.irp + u + 1);
            bool hit = false;
            for (uint64_t b = beg; b < end; b += BLOCK) {
                const uint64_t e = b + threadIdx.x;
                bool h = false;
                if (e < end) {
                    ++edges;
                    h = bm_test(cur, __ldg(p.g.ici + e));
                }
                if (__syncthreads_or(h)) {
                    hit = true;
                    break;
                }
            }
            if (threadIdx.x == 0) {
                if (hit) mark(u);
                else online_record(nx, nlists, n, (uint32_t)n, u, k);
            }
        }
        // warp granularity: medium candidates (__any_sync early exit)
        for (uint64_t i = gwarp(); i < cnt[1]; i += gwarps()) {
            const uint32_t u = L[n + i];
            const uint64_t beg = __ldg(p.g.irp + u), end = __ldg(p.g.irp + u + 1);
            bool hit = false;
            for (uint64_t b = beg; b < end; b += 32) {
                const uint64_t e = b + lane_id();
                bool h = false;
                if (e < end) {
                    ++edges;
                    h = bm_test(cur, __ldg(p.g.ici + e));
                }
                if (__any_sync(FULL, h)) {
                    hit = true;
                    break;
                }
            }
            if (lane_id() == 0) {
                if (hit) mark(u);
                else online_record(nx, nlists, n, (uint32_t)n, u, 1u);
            }
        }
        // thread granularity: small candidates
        for (uint64_t i = gtid(); i < cnt[0]; i += gthreads()) {
            const uint32_t u = L[i];
            const uint64_t beg = __ldg(p.g.irp + u), end = __ldg(p.g.irp + u + 1);
            bool hit = false;
            for (uint64_t e = beg; e < end; ++e) {
                ++edges;
                if (bm_test(cur, __ldg(p.g.ici + e))) {
                    hit = true;
                    break;
                }
            }
            if (hit) mark(u);
            else online_record(nx, nlists, n, (uint32_t)n, u, 0u);
        }
        (void)s_hit;
        st.edges += edges;
        st.reached += found;
        if (lead()) st.entries += sum4(cnt);
        {
            uint64_t v[2] = {mdeg, found};
            block_sum<2>(v);
            if (threadIdx.x == 0) {
                if (v[0]) atomicAdd(&nx->mdeg, (unsigned long long)v[0]);
                if (v[1]) atomicAdd(&nx->found, (unsigned int)v[1]);
            }
        }
        if (!grid_sync(c)) return;
        uint32_t ncnt[NCLS];
        for (int i = 0; i < NCLS; ++i) ncnt[i] = vload(&nx->cnt[i]);
        const uint64_t nf = vload(&nx->found);
        const uint64_t mf = vload(&nx->mdeg);
        m_u -= mf;
        ++it;
        ++st.iters;
        ++st.pull;
        trace_put(p.s, it, DIR_PULL, 0u, ncnt, nf, mf, m_u);
        for (int i = 0; i < NCLS; ++i) cnt[i] = ncnt[i];
        if (nf == 0 || (p.s.max_iters && it >= p.s.max_iters)) {
            done = 1;
            break;
        }
        const bool to_push = p.s.force_dir == 1 ||
                             (p.s.force_dir == 0 && (double)nf < (double)n / p.s.beta && nf < nf_prev);
        nf_prev = (uint32_t)nf;
        if (to_push) {
            dir = DIR_PUSH;
            ready = 0;
            break;
        }
        if (!p.s.fusion) break;
    }
    bfs_exit(p, it, m_u, nf_prev, dir, done, ready, cnt, st);
}

}  // namespace sx

// ------------------------------------------------------------------ host driver
using namespace sx;

// Algorithmic bytes of the executed BFS schedule:
// per list entry 4 B (list) + 16 B (row_ptr pair); per examined edge 4 B (col);
// per reached vertex 4 B (level write); per iteration one frontier-bitmap clear
// (n/8); per pull iteration one frontier-bitmap read (n/8); ballot scans n/8.
static double bfs_bytes(const sx_graph g, const sxh::Counters& c) {
    const double n = (double)g->n;
    return 20.0 * c.entries + 4.0 * c.edges + 4.0 * c.reached + (c.iters + c.pull) * n / 8.0 + c.scanned / 8.0;
}

extern "C" sx_status sx_bfs(sx_graph g, uint32_t src, const sx_opts* opts, uint32_t* level_out, sx_stats* stats) {
    if (!g || !level_out) return sxh::fail(SX_E_INVALID, "sx_bfs: NULL graph or level_out");
    sx_status rc = sxh::check_ctx(g->ctx);
    if (rc != SX_OK) return rc;
    if (g->n == 0) return sxh::fail(SX_E_INVALID, "sx_bfs: empty graph has no source");
    if (src >= g->n) return sxh::fail(SX_E_INVALID, "sx_bfs: src >= n");
    sxh::Run run{g, sxh::resolve_opts(opts), stats};
    if (g->directed && !g->has_rev && run.o.force_dir != 1)
        return sxh::fail(SX_E_NO_REVERSE, "sx_bfs: pull needs in-neighbour rows (CSC); use force_dir=1 (push)");
    cudaStream_t s = g->ctx->stream;
    BfsP p;
    if ((rc = run.begin()) != SX_OK) return rc;
    p.g = sxh::dev_graph(g);
    p.s = sxh::make_sched(g, run.o);
    p.level = g->st[0];
    p.visited = g->aux_bm;
    SX_CU(cudaMemsetAsync(p.level, 0xFF, g->n * 4, s));
    SX_CU(cudaMemsetAsync(p.visited, 0, g->nwords * 4, s));
    for (int i = 0; i < 3; ++i) SX_CU(cudaMemsetAsync(p.s.bm[i], 0, g->nwords * 4, s));
    const uint32_t dir0 = run.o.force_dir == 2 ? DIR_PULL : DIR_PUSH;
    bfs_init<<<1, 1, 0, s>>>(p, src, dir0);
    SX_CU(cudaGetLastError());
    void* args[] = {&p};
    g->ctx->h_ctl->dir = dir0;
    g->ctx->h_ctl->done = 0;
    for (;;) {
        const bool pull = g->ctx->h_ctl->dir == DIR_PULL;
        if ((rc = run.launch(pull ? (const void*)bfs_pull : (const void*)bfs_push, args, pull)) != SX_OK) return rc;
        if (g->ctx->h_ctl->done) break;
    }
    if ((rc = run.end(bfs_bytes)) != SX_OK) return rc;
    return sxh::copy_out(g, level_out, p.level, g->n * 4);
}

extern "C" sx_status sx_ctx_info(sx_ctx c, sx_device_info* out) {
    if (!out) return sxh::fail(SX_E_INVALID, "sx_ctx_info: out == NULL");
    sx_status rc = sxh::check_ctx(c);
    if (rc != SX_OK) return rc;
    std::memset(out, 0, sizeof(*out));
    out->device = c->device;
    out->sm_count = c->prop.multiProcessorCount;
    out->cc_major = c->prop.major;
    out->cc_minor = c->prop.minor;
    out->regs_per_sm = c->prop.regsPerMultiprocessor;
    out->max_threads_per_sm = c->prop.maxThreadsPerMultiProcessor;
    out->block_threads = BLOCK;
    cudaFuncAttributes a{};
    int occ = 0;
    SX_CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bfs_push, BLOCK, 0));
    out->push_ctas_per_sm = occ;
    SX_CU(cudaFuncGetAttributes(&a, bfs_push));
    out->push_regs = a.numRegs;
    SX_CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bfs_pull, BLOCK, 0));
    out->pull_ctas_per_sm = occ;
    SX_CU(cudaFuncGetAttributes(&a, bfs_pull));
    out->pull_regs = a.numRegs;
    return SX_OK;
}

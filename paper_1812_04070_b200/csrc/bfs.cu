// bfs.cu — BFS as an ACC algorithm (PAPER.md; voting combine P:343-345).
//
//   Active  : vertices first reached in the previous level (frontier bitmap bm[it%3])
//   Compute : level(u) = it + 1 for an unvisited neighbour u
//   Combine : vote — any one update suffices; push claims u exactly once
//             with atomicOr on the visited bitmap; pull stops scanning u's
//             in-neighbours at the first frontier hit (collaborative early
//             termination) using __any_sync.
//
// Selective fusion: one persistent cooperative kernel per direction
// run; it loops over BSP iterations with the grid barrier and exits only when
// the traversal ends or the direction switches (push -> pull -> push).
#include <cstring>

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <type_traits>

#include "internal.h"

namespace sx {

struct BfsP {
    DevGraph g;
    Sched s;
    uint32_t* level;
    uint32_t* visited;
    const uint32_t* __restrict__ hub;  // per vertex: its in-neighbour of largest out-degree (INF: none)
    int sym;  // symmetric graph: in-degree == out-degree
    int tma;  // TILE-mode pull stages each chunk's hub slice with a TMA bulk copy (needs a 16-B aligned hub)
    AsyncAcc* acc;  // asynchronous run: statistics go to this accumulator (nullptr: the control block)
};

// Hub-first probe table, built once per graph: hub(v) = the in-neighbour of
// largest out-degree among v's first HUB_SCAN in-edges (ties: smallest id).
// The bottom-up step tests it before touching v's row; a high-degree neighbour
// is the one most likely to sit in a large frontier, so in the dense middle
// levels a candidate usually costs one coalesced 4-B load instead of a row-pointer
// pair plus a random row sector.  Probe order does not change the result (any
// frontier in-neighbour proves level(v) = it + 1).  When v has exactly one
// in-edge, bit 31 (HUB_SOLE; graphs of n <= 2^31) says the hub is the whole row:
// a failed probe then settles v for the level without a row walk — on R-MAT
// most candidates left open by the probe are such degree-1 vertices.
constexpr uint32_t HUB_SCAN = 64;
constexpr uint32_t HUB_SOLE = 0x80000000u;
#ifndef SX_PROBE
#define SX_PROBE 4
#endif
#ifndef SX_PULL_MINB
#define SX_PULL_MINB 3  // measured: 3 CTAs x 256 at <= 85 registers beat 4 at 64 (s24 pull 158 -> 154 us)
#endif
// Groups of 8 lanes per vertex (4 vertices per warp step): a lane loads up to
// HUB_SCAN / 8 ids of its vertex's row, then their out-degrees, each batch in
// flight together, and the group reduces with 3 shuffles.
__global__ void __launch_bounds__(BLOCK) bfs_hub(DevGraph g, uint32_t* hub) {
    constexpr uint32_t GS = 8, PER = HUB_SCAN / GS;
    const uint32_t lane = lane_id(), sub = lane % GS;
    const uint64_t ngroups = (uint64_t)gridDim.x * WARPS * (32 / GS);
    const bool flag = g.n <= HUB_SOLE;
    const uint64_t g0 = ((uint64_t)blockIdx.x * WARPS + warp_id()) * (32 / GS) + lane / GS;
    for (uint64_t vb = g0 - lane / GS; vb < g.n; vb += ngroups) {  // warp-uniform loop
        const uint64_t v = vb + lane / GS;
        uint64_t beg = 0, end0 = 0;
        if (v < g.n) {
            beg = __ldg(g.irp + v);
            end0 = __ldg(g.irp + v + 1);
        }
        const uint64_t end = min(end0, beg + HUB_SCAN);
        uint32_t u[PER], d[PER];
#pragma unroll
        for (uint32_t k = 0; k < PER; ++k) {
            const uint64_t e = beg + sub + k * GS;
            u[k] = e < end ? __ldg(g.ici + e) : INF;
        }
#pragma unroll
        for (uint32_t k = 0; k < PER; ++k) d[k] = u[k] != INF ? __ldg(g.dout + u[k]) : 0u;
        uint64_t best = 0;
#pragma unroll
        for (uint32_t k = 0; k < PER; ++k)
            if (u[k] != INF) best = max(best, ((uint64_t)(d[k] + 1u) << 32) | (uint64_t)(~u[k]));
#pragma unroll
        for (int o = GS / 2; o; o >>= 1) best = max(best, __shfl_xor_sync(FULL, best, o));
        if (sub == 0 && v < g.n) hub[v] = best ? (~(uint32_t)best | (flag && end0 - beg == 1 ? HUB_SOLE : 0u)) : INF;
    }
}
// the probe target of a hub entry (INF: no in-neighbour) and whether it is v's only in-edge
__device__ __forceinline__ uint32_t hub_id(uint32_t h) { return h == INF ? INF : h & ~HUB_SOLE; }
__device__ __forceinline__ bool hub_sole(uint32_t h) { return h != INF && (h & HUB_SOLE); }

constexpr uint32_t CL_EDGES = 32;
constexpr uint32_t INIT_TILE = 2048;  // bytes per TMA bulk store of the fused init
#ifndef SX_REC_EDGES
#define SX_REC_EDGES (1u << 17)
#endif
constexpr uint64_t REC_EDGES = SX_REC_EDGES;
constexpr uint32_t DIR_NOCLUSTER = 0x100;  // bfs_init flag: no cluster start (all fusion)
__device__ __forceinline__ bool cluster_ok(const Sched& s, uint64_t nf, uint64_t mf) {
    return s.cluster_enter && s.fusion && s.force_filter < 2 && s.force_dir != 2 && nf > 0 &&
           nf <= s.cluster_enter && mf <= (uint64_t)CL_EDGES * s.cluster_enter;
}

// SX_BFS_MARKS (profiling builds): extra trace records from CTA 0 (dir = 16 + id)
#ifdef SX_BFS_MARKS
#define BFS_MARK(id)                                                          \
    do {                                                                      \
        const uint32_t z_[NCLS] = {0u, 0u, 0u, 0u};                           \
        trace_put(p.s, 1000u + (id), 16u + (id), 0u, z_, 0, 0, 0);            \
    } while (0)
#else
#define BFS_MARK(id) \
    do {             \
    } while (0)
#endif

// SX_BFS_ANAT (profiling builds): anatomy of the first pull level's TILE chunks —
// SM cycles per segment summed over CTA 0's warps (profiles/bfs_anatomy.py reads
// them through sx_debug_bfs_anat, a symbol outside the ABI).  A volatile store of
// the segment's last value makes the clock read wait for it.
#ifdef SX_BFS_ANAT
__device__ unsigned long long g_bfs_anat[16];
__device__ volatile uint32_t g_bfs_sink;
#define ANAT(k, dep)                                         \
    do {                                                      \
        if (an_on) {                                          \
            g_bfs_sink = (uint32_t)(dep);                     \
            const unsigned long long t_ = clock64();          \
            an[k] += t_ - an_last;                            \
            an_last = t_;                                     \
        }                                                     \
    } while (0)
#else
#define ANAT(k, dep) \
    do {             \
    } while (0)
#endif

// Per-run state in one grid-stride pass: level = INF (0 at src), visited and
// the three frontier bitmaps zero (src's bit set in visited and bm[0]); block 0
// also seeds the control block and the first list.
template <bool ALL, bool CLUSTER = !ALL>
__device__ __forceinline__ void bfs_init_body(const BfsP& p, uint32_t src, uint32_t dir) {
    const uint64_t n = p.g.n, T = gthreads(), tid = gtid();
    if (ALL && ((uintptr_t)p.level & 15u) == 0) {
        // inside the fused launch (3 CTAs x 256 threads per SM, too few threads to
        // saturate HBM with stores) the level array is filled by the TMA unit: one
        // thread per CTA issues bulk copies of an INF tile in shared memory
        // (cp.async.bulk global <- shared), the source's level follows once they landed
        __shared__ alignas(128) uint32_t s_inf[INIT_TILE / 4];
        for (uint32_t i = threadIdx.x; i < INIT_TILE / 4; i += BLOCK) s_inf[i] = INF;
        fence_proxy_async_smem();
        __syncthreads();
        const uint64_t nb = n * 4 / INIT_TILE;  // whole tiles
        if (threadIdx.x == 0) {
            for (uint64_t b = blockIdx.x; b < nb; b += gridDim.x) tma_store_1d((char*)p.level + b * INIT_TILE, s_inf, INIT_TILE);
            tma_store_wait();
            asm volatile("fence.proxy.async.global;" ::: "memory");  // bulk (async-proxy) writes before generic ones
        }
        for (uint64_t i = nb * (INIT_TILE / 4) + tid; i < n; i += T) p.level[i] = INF;
        __syncthreads();
        // every CTA's bulk stores are complete here; the source's tile belongs to CTA (src*4/INIT_TILE) % grid
        const uint64_t sb = (uint64_t)src * 4 / INIT_TILE;
        if (threadIdx.x == 0 && (sb >= nb || blockIdx.x == sb % gridDim.x)) p.level[src] = 0u;
    } else if (((uintptr_t)p.level & 15u) == 0) {
        uint4* L4 = reinterpret_cast<uint4*>(p.level);
        for (uint64_t q = tid; q < n / 4; q += T) {
            uint4 v = make_uint4(INF, INF, INF, INF);
            if (q == src >> 2) {
                const uint32_t k = src & 3u;
                v.x = k == 0 ? 0u : INF;
                v.y = k == 1 ? 0u : INF;
                v.z = k == 2 ? 0u : INF;
                v.w = k == 3 ? 0u : INF;
            }
            L4[q] = v;
        }
        for (uint64_t i = n / 4 * 4 + tid; i < n; i += T) p.level[i] = i == src ? 0u : INF;
    } else {
        for (uint64_t i = tid; i < n; i += T) p.level[i] = i == src ? 0u : INF;
    }
    uint32_t* bms[4] = {p.visited, p.s.bm[0], p.s.bm[1], p.s.bm[2]};
    const uint64_t nq = p.s.nwords / 4;  // nwords is a multiple of TILE_WORDS
    const uint64_t sq = src >> 7;        // the quad holding src's word
    const uint32_t bit = 1u << (src & 31), sw = (src >> 5) & 3u;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        uint4* B4 = reinterpret_cast<uint4*>(bms[b]);
        for (uint64_t q = tid; q < nq; q += T) {
            uint4 v = make_uint4(0u, 0u, 0u, 0u);
            if (q == sq && b < 2) {
                v.x = sw == 0 ? bit : 0u;
                v.y = sw == 1 ? bit : 0u;
                v.z = sw == 2 ? bit : 0u;
                v.w = sw == 3 ? bit : 0u;
            }
            B4[q] = v;
        }
    }
    if (blockIdx.x != 0) return;
    Ctl* c = p.s.ctl;
    if (!ALL) {  // the whole control block starts at zero (replaces a host-enqueued memset per call)
        uint4* C4 = reinterpret_cast<uint4*>(c);
        for (uint32_t i = threadIdx.x; i < sizeof(Ctl) / 16; i += BLOCK) C4[i] = make_uint4(0u, 0u, 0u, 0u);
    } else {  // inside the fused launch: not the barrier halves in use, not the launch count
        uint32_t* W = reinterpret_cast<uint32_t*>(c);
        constexpr uint32_t w0 = offsetof(Ctl, line) / 4, wl = offsetof(Ctl, launch) / 4;
        for (uint32_t i = w0 + threadIdx.x; i < sizeof(Ctl) / 4; i += BLOCK)
            if (i != wl) W[i] = 0u;
    }
    __syncthreads();
    if (threadIdx.x < 32)
        for (int i = 0; i < 3; ++i) reset_line_warp(&c->line[i]);
    if (threadIdx.x != 0) return;
    const uint32_t d = p.g.dout[src];
    const uint32_t k = cls_of(d, p.s);
    for (int i = 0; i < NCLS; ++i) c->cur_count[i] = 0;
    c->cur_count[k] = 1;
    p.s.lists[0][(uint64_t)k * p.s.cstride] = src;
    c->m_u = p.g.m - d;
    c->hi = d;  // out-edges of the current frontier (the online-record prediction of the push)
    c->nf_prev = 1;
    if (CLUSTER && dir == DIR_PUSH && cluster_ok(p.s, 1, d)) dir = DIR_CLUSTER;  // low-degree source: start on one cluster
    c->dir = dir;
    c->k = dir;  // the start direction, for the host (k is unused by BFS)
    c->lists_ready = dir == DIR_PUSH ? 1u : 0u;
    c->slotted = 0;
    c->iter = 0;
    c->done = 0;
    c->st[0].reached = 1;
}
__global__ void __launch_bounds__(BLOCK) bfs_init(BfsP p, uint32_t src, uint32_t dir) {
    if (dir & DIR_NOCLUSTER) bfs_init_body<false, false>(p, src, dir & ~DIR_NOCLUSTER);
    else bfs_init_body<false, true>(p, src, dir);
}

// End of a direction phase.  Selective fusion (ALL = false): the kernel exits;
// CTA 0 leaves the run state in the control block for the next launch.  All
// fusion (ALL = true): the next phase runs in the same launch; every CTA took
// the same decisions from the same counters, so each writes its own copy of
// the run state (shared memory) and CTA 0 also stores it for the host.
template <bool ALL>
__device__ __forceinline__ void bfs_exit(const BfsP& p, uint32_t kdir, uint32_t it, uint64_t m_u, uint32_t nf_prev,
                                         uint32_t dir, uint32_t done, uint32_t ready, uint32_t slotted,
                                         const uint32_t (&cnt)[NCLS], Stats& st, RunState* rs_next, uint64_t mf_next) {
    Ctl* c = p.s.ctl;
    flush_stats(c, st, kdir, p.acc ? p.acc->st : nullptr);
    if (lead()) {
        c->iter = it;
        c->m_u = m_u;
        c->hi = mf_next;
        c->nf_prev = nf_prev;
        c->dir = dir;
        c->done = done;
        c->lists_ready = ready;
        c->slotted = slotted;
        for (int i = 0; i < NCLS; ++i) c->cur_count[i] = cnt[i];
        if (!ALL) {
            grid_end(c);
            c->launch += 1;
        }
    }
    if (ALL) {
        __syncthreads();  // every thread has read the current copy
        if (threadIdx.x == 0) {
            rs_next->iter = it;
            rs_next->m_u = m_u;
            rs_next->hi = mf_next;
            rs_next->nf_prev = nf_prev;
            rs_next->dir = dir;
            rs_next->done = done;
            rs_next->lists_ready = ready;
            rs_next->slotted = slotted;
            for (int i = 0; i < NCLS; ++i) rs_next->cur_count[i] = cnt[i];
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ push
#ifndef SX_PUSH_MINB
#define SX_PUSH_MINB 3  // measured: 3 CTAs/SM beat 4 (s24 push 58.6 -> 54.5 us; profiles/r1/bfs_variant_sweep.txt)
#endif
template <bool ALL>
__device__ __forceinline__ bool push_phase(const BfsP& p, RunState& rs) {
    Ctl* c = p.s.ctl;
    stage_init();
    __syncthreads();
    uint32_t it = rs.iter;
    uint64_t m_u = rs.m_u;
    uint32_t nf_prev = rs.nf_prev;
    uint32_t cnt[NCLS];
    Stats st;
    uint32_t dir = DIR_PUSH, done = 0, ready = 1, slotted = 0;
    uint64_t mf_cur = rs.hi;  // out-edges of the current frontier
    uint32_t local_n = 0;  // > 0: this iteration's tasks are the flat found list of the pull (CTA-local binning)
    if (rs.lists_ready == 2) {
        // entering push from pull with the found vertices recorded as one list
        // (online filter, <= FREC_MAX entries): no bitmap scan, no class split
        local_n = vload(&c->cl.cnt[it % 3]);
        for (int i = 0; i < NCLS; ++i) cnt[i] = 0;
        if (local_n == 0) view_contig(cnt);
    } else if (!rs.lists_ready) {
        // entering push from pull: the frontier exists only as a bitmap -> ballot filter
        if (!ballot_filter(BitmapWords{p.s.bm[it % 3]}, p.s, BallotOut{p.s.lists[it & 1], p.s.cstride, p.g.dout}, cnt))
            return false;
        st.scanned += p.s.nwords * 32;
        if (!grid_sync(c)) return false;
        view_contig(cnt);
    } else if (rs.slotted) {
        view_slots(&c->line[it % 3], p.s, cnt);
    } else {
        for (int i = 0; i < NCLS; ++i) cnt[i] = rs.cur_count[i];
        view_contig(cnt);
    }
    for (;;) {
        IterLine* nx = &c->line[(it + 1) % 3];
        maybe_reset_line(&c->line[(it + 2) % 3]);
        clear_bitmap(p.s.bm[(it + 2) % 3], p.s.nwords);
        uint32_t* nlists = p.s.lists[(it + 1) & 1];
        uint32_t* nbm = p.s.bm[(it + 1) % 3];
        const uint32_t lvl = it + 1;
        uint64_t mdeg = 0, edges = 0, reached = 0;
        // JIT by prediction (B200 reading of P:619-626): a frontier with more than
        // REC_EDGES out-edges activates a next frontier the ballot filter handles
        // better (or the pull takes over), so it is not recorded online — as if
        // the bins had overflowed; measured: the s24 hub level 30 -> 24 us
        const bool batch = p.s.force_filter == 3;
        const bool rec = batch || mf_cur <= REC_EDGES;
        auto visit = [&](uint32_t v, uint64_t rank, uint64_t size, uint32_t) {
            const uint64_t beg = __ldg(p.g.rp + v), end = __ldg(p.g.rp + v + 1);
            // up to 4 edges per step: visited words, claims and the claimed
            // vertices' degrees are each issued together
            for_edges_b(p.g.ci, beg, end, rank, size, [&](const uint32_t (&u)[4], uint32_t k) {
                edges += k;
                uint32_t vw[4], du[4];
                bool cl[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) vw[j] = j < (int)k ? p.visited[u[j] >> 5] : FULL;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t bit = 1u << (u[j] & 31);
                    // batch filter (force_filter = 3): no claim, so a vertex reached by
                    // several frontier vertices in the iteration is updated and recorded by each
                    cl[j] = j < (int)k && !(vw[j] & bit) &&
                            (batch ? (atomicOr(p.visited + (u[j] >> 5), bit), true)
                                   : !(atomicOr(p.visited + (u[j] >> 5), bit) & bit));
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    du[j] = 0;
                    if (!cl[j]) continue;
                    p.level[u[j]] = lvl;
                    bm_set(nbm, u[j]);
                    du[j] = __ldg(p.g.dout + u[j]);
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (!cl[j]) continue;
                    mdeg += du[j];
                    ++reached;
                    if (rec) online_record(nx, nlists, p.s, u[j], cls_of(du[j], p.s));
                }
            });
        };
        if (local_n) for_list_local(p.s.lists[it & 1], local_n, p.s, p.g.dout, visit);
        else for_tasks(p.s.lists[it & 1], p.s, cnt, visit);
        BFS_MARK(2);
        stage_flush(nx, nlists, p.s);
        st.edges += edges;
        st.reached += reached;
        if (lead()) st.entries += local_n ? local_n : sum4(cnt);
        {
            uint64_t v[2] = {mdeg, rec ? 0ull : reached};
            block_sum<2>(v);
            if (threadIdx.x == 0 && v[0]) atomicAdd(&nx->s[my_slot()].mdeg, (unsigned long long)v[0]);
            if (threadIdx.x == 0 && v[1]) atomicAdd(&nx->s[my_slot()].found, (unsigned int)v[1]);  // not recorded: counted
        }
        if (!grid_sync(c)) return false;
        if (local_n) {
            if (lead()) c->cl.cnt[it % 3] = 0;  // every CTA read the count before the barrier above
            local_n = 0;
        }
        LineSum ls;
        uint32_t vcnt[NCLS];
        read_line_view(nx, p.s, ls, vcnt);
        const uint64_t nf = rec ? sum4(ls.cnt) : ls.found;
        const uint64_t mf = ls.mdeg;
        bool overflow = !rec;
        for (int i = 0; i < NCLS; ++i) overflow |= ls.cntmax[i] > p.s.cap_s;
        if (p.s.force_filter == 2) overflow = true;
        mf_cur = mf;
        m_u -= mf;
        ++it;
        ++st.iters;
        trace_put(p.s, it, DIR_PUSH, overflow ? 1u : 0u, ls.cnt, nf, mf, m_u);
        if (nf == 0 || (p.s.max_iters && it >= p.s.max_iters)) {
            done = 1;
            for (int i = 0; i < NCLS; ++i) cnt[i] = 0;
            slotted = 0;
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
        if (!ALL && cluster_ok(p.s, nf, mf)) {
            dir = DIR_CLUSTER;
            ready = 0;
            break;
        }
        if (overflow) {
            ++st.ballot;
            st.scanned += p.s.nwords * 32;
            if (!ballot_filter(BitmapWords{nbm}, p.s, BallotOut{p.s.lists[it & 1], p.s.cstride, p.g.dout}, cnt)) return false;
            if (!grid_sync(c)) return false;
            view_contig(cnt);
            slotted = 0;
        } else {
            for (int i = 0; i < NCLS; ++i) cnt[i] = vcnt[i];  // view set by read_line_view
            slotted = 1;
        }
        if (!p.s.fusion) break;
    }
    bfs_exit<ALL>(p, DIR_PUSH, it, m_u, nf_prev, dir, done, ready, slotted, cnt, st, &rs, mf_cur);
    return true;
}
__global__ void __launch_bounds__(BLOCK, SX_PUSH_MINB) bfs_push(BfsP p) {
    RunState& rs = const_cast<RunState&>(run_state(p.s.ctl));
    if (rs.done || rs.dir != DIR_PUSH) return;
    grid_begin(rs.launch);
    push_phase<false>(p, rs);
}

// ------------------------------------------------------------------ pull
// Bottom-up step.  The active set of a pull iteration is the unvisited set
// (candidates: unvisited with in-degree > 0), held the JIT way:
//  * TILE mode (large candidate sets — the ballot side): chunks of 32 tiles of
//    32 consecutive vertices.  A warp owns its chunk's words of the visited
//    bitmap, so a tile's candidates are the word ~visited & (in-degree > 0) —
//    the ballot filter's output for that tile without a grid-wide
//    list; the warp compacts them into shared memory in vertex order (popc +
//    exclusive scan: a warp-local ballot filter).  Found bits are merged per
//    word in shared memory and stored once: no global atomics.
//  * LIST mode (small candidate sets — the online side): the candidates still
//    open at the end of the previous pull iteration were recorded in slotted
//    lists (online filter); the iteration walks those lists in warp
//    chunks instead of scanning every tile.  A level records its open
//    candidates only when its own candidates are <= n / REC_OPEN_DIV (never the
//    first pull): recording costs the recording level, and a LIST level over a
//    large set is slower than a TILE scan.  Otherwise they are only counted (the
//    next level's candidate count).  LIST mode follows a recorded level when the
//    recorded total is <= n / LIST_DIV and no region overflowed.  When at most
//    FREC_MAX vertices can be found, the found ones also go onto a list (TILE
//    or LIST mode) that a switch back to push takes as its task list.
// A warp's candidates then go through two phases.  (1) Hub-first probe, HUB_ILP
// rounds of 32 in flight: one load of hub[v] and one bitmap test each; a sole
// in-edge probed in vain settles v (still open, no row walk).  (2) Row walks of
// the others, binned by in-degree: small ones (thread
// granularity) on their lane with PROBE loads in flight per round, medium and
// larger ones with the whole warp, 32 edges per step (warp granularity); all
// stop at the first frontier in-neighbour (voting early exit).
// m_u on symmetric graphs needs no degree loads: every candidate left open
// walked its whole row (or had one in-edge), so m_u(next) = sum of the open
// candidates' degrees and m_f = m_u - m_u(next).
constexpr int PROBE = SX_PROBE;
#ifndef SX_WALK_K
#define SX_WALK_K 1
#endif
constexpr int WALK_K = SX_WALK_K;
#ifndef SX_LIST_CSZ_MAX
#define SX_LIST_CSZ_MAX 128  // measured: 256 leaves it3 of s24 imbalanced (CTA finish spread 21 us median), 64 adds grab overhead (profiles/r2/list_csz.txt)
#endif
constexpr uint32_t LIST_CSZ_MAX = SX_LIST_CSZ_MAX;  // LIST-mode chunk (candidates) at most  // pull row walks at warp granularity: edges per lane per step
#ifndef SX_HUB_ILP
#define SX_HUB_ILP 4
#endif
constexpr int HUB_ILP = SX_HUB_ILP;
#ifndef SX_HUB_PIPE
#define SX_HUB_PIPE 0  // measured (session 3): probe rounds 9.8 -> 9.1 us per chunk, level total unchanged (issue-bound, not latency-bound)
#endif
constexpr bool HUB_PIPE = SX_HUB_PIPE;  // next probe round's hub loads issued before this round's processing             // phase 1: rounds of 32 candidates in flight per warp
#ifndef SX_LIST_DIV
#define SX_LIST_DIV 8
#endif
constexpr uint32_t LIST_DIV = SX_LIST_DIV;
#ifndef SX_PULL_REC
#define SX_PULL_REC 1
#endif
#ifndef SX_PULL_STATIC
#define SX_PULL_STATIC 0
#endif
constexpr bool PULL_REC = SX_PULL_REC;        // record the open candidates for a LIST-mode next level
#ifndef SX_REC_OPEN_DIV
#define SX_REC_OPEN_DIV 16
#endif
// ... only when this level's candidates are at most n / REC_OPEN_DIV: recording costs
// the level that records (s24: the first pull 84.6 -> 98.6 us) and a LIST level is
// slower than a TILE scan for large candidate sets (s24 it3: 38.8 vs 30.1 us); the
// first pull never records (its candidate count is unknown and large)
constexpr uint32_t REC_OPEN_DIV = SX_REC_OPEN_DIV;
constexpr bool PULL_STATIC = SX_PULL_STATIC;  // TILE chunks assigned statically (no claims / stealing)
#ifndef SX_PULL_TMA
#define SX_PULL_TMA 0  // measured slower (s24 it2 100.6 -> 114.8 us; profiles/r2/pull_tma.txt); experiment only
#endif
// TILE-mode chunk: CW bitmap words = CV vertices.  With TMA staging the chunk's
// hub slice (CV x 4 B) is bulk-copied into shared memory one chunk ahead, two
// buffers per warp (dynamic shared memory, PULL_DYN_SMEM bytes per CTA).
#ifndef SX_PULL_CW
#define SX_PULL_CW (SX_PULL_TMA ? 16 : 32)
#endif
constexpr uint32_t CW = SX_PULL_CW;
static_assert(CW >= 1 && CW <= 32, "TILE chunk: at most one bitmap word per lane");
constexpr uint32_t CV = CW * 32u;
constexpr uint32_t CAND_MAX = CV > 256u ? CV : 256u;  // per-warp candidate list (TILE chunk, LIST csz <= 256)
constexpr int PULL_DYN_SMEM = SX_PULL_TMA ? WARPS * 2 * CV * 4 : 0;
constexpr uint32_t FREC_MAX = 32768;   // record the found vertices as a list when candidates <= this
constexpr uint32_t CAND_CLS = 2;       // class region of lists[] holding the LIST-mode candidate lists
constexpr uint32_t REC_STAGE = 256;    // per-warp staging of the LIST-mode record

template <bool ALL>
__device__ __forceinline__ bool pull_phase(const BfsP& p, RunState& rs) {
    Ctl* c = p.s.ctl;
    const uint64_t n = p.g.n;
    const uint64_t nw = (n + 31) >> 5;
    uint32_t it = rs.iter;
    uint64_t m_u = rs.m_u;
    uint32_t nf_prev = rs.nf_prev;
    uint32_t cnt[NCLS] = {0, 0, 0, 0};
    Stats st;
    uint32_t dir = DIR_PULL, done = 0;
    const uint32_t lane = lane_id();
    __shared__ uint32_t s_cand[WARPS][CAND_MAX];
    __shared__ uint64_t s_mbar[WARPS][2];
    extern __shared__ __align__(128) uint32_t s_dyn_hub[];
    __shared__ uint32_t s_found[WARPS][32];
    __shared__ uint32_t s_cpre[NSLOT + 1];  // LIST mode: prefix of the candidate regions' counts
    // the record staging shares the push phase's online-filter stage (8 KB): the
    // phases never overlap, and the fused kernel then fits 48 KB of static smem
    static_assert(WARPS * REC_STAGE <= NCLS * STAGE, "record staging fits the online stage");
    uint32_t* s_c = s_cand[warp_id()];
    uint32_t* s_r = &stage().e[0][0] + warp_id() * REC_STAGE;
    uint32_t* s_f = s_found[warp_id()];
    uint64_t mf_last = 0;  // out-edges of the frontier found last (the push's record prediction)
    uint32_t ncand = 0;    // LIST mode when > 0: candidates recorded by the previous iteration
    uint64_t cand_cnt = ~0ull;  // this level's candidates (the previous level's open count; unknown at first)
    uint32_t handoff = 0;  // the next frontier was recorded as a contiguous list
    uint32_t to_list = 0;  // 2: ... and the push takes it as its lists (lists_ready = 2)
    for (;;) {
        IterLine* nx = &c->line[(it + 1) % 3];
        maybe_reset_line(&c->line[(it + 2) % 3]);
        if (lead()) c->cl.cnt[(it + 2) % 3] = 0;  // found-list counter of the next iteration
        clear_bitmap(p.s.bm[(it + 2) % 3], p.s.nwords);
        const uint32_t* cur = p.s.bm[it % 3];
        uint32_t* nbm = p.s.bm[(it + 1) % 3];
        const uint32_t lvl = it + 1;
        const bool list_mode = ncand > 0;
        // the found vertices go to a list (the push hand-over) when few can be found
        const bool rec_found = cand_cnt <= FREC_MAX && p.s.force_filter != 2;
        // the open candidates are recorded (LIST mode next) only when this level's candidates are few
        const bool rec_open = PULL_REC && cand_cnt <= n / REC_OPEN_DIV && p.s.force_filter != 2;
        uint32_t open_cnt = 0;  // open candidates counted, not recorded (!rec_open)
#ifdef SX_BFS_ANAT
        const bool an_on = blockIdx.x == 0 && !list_mode && cand_cnt == ~0ull;  // CTA 0, the first pull level
        unsigned long long an[8] = {0, 0, 0, 0, 0, 0, 0, 0}, an_last = clock64();
#endif
        uint32_t* cnext = p.s.lists[(it + 1) & 1] + (uint64_t)CAND_CLS * p.s.cstride;
        uint32_t* flist = p.s.lists[(it + 1) & 1];  // class-0 region: the found list (hand-over)
        unsigned int* fcnt = &c->cl.cnt[(it + 1) % 3];
        uint64_t mdeg = 0, mopen = 0, edges = 0, cand_small = 0, cand_warp = 0, rows = 0;
        uint32_t found_cnt = 0;
        // a found vertex: level, statistics, and (TILE) the word merge in shared
        // memory or (LIST) the bitmaps plus the online record of the next frontier
        auto on_found = [&](uint32_t v, uint64_t w0) {
            p.level[v] = lvl;
            if (!p.sym) mdeg += __ldg(p.g.dout + v);
            if (!list_mode) {
                atomicOr(s_f + ((v >> 5) - w0), 1u << (v & 31));
                return;
            }
            bm_set(p.visited, v);
            bm_set(nbm, v);
            ++found_cnt;
            if (rec_found) {  // warp-aggregated append
                const uint32_t act = __activemask();
                const int leader = __ffs(act) - 1;
                uint32_t base = 0;
                if ((int)lane == leader) base = atomicAdd(fcnt, (uint32_t)__popc(act));
                base = __shfl_sync(act, base, leader);
                flist[base + __popc(act & lanemask_lt())] = v;
            }
        };
        // warp-collective: record the lanes' still-open candidates for a
        // LIST-mode next iteration — staged in shared memory, then appended to
        // cnext (region of this CTA's slot) with one atomic per flush instead of
        // a blocking atomic round trip per probe round
        uint32_t nrec = 0;
        auto flush_rec = [&]() {
            if (!nrec) return;
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(&nx->s[my_slot()].alive, nrec);
            base = __shfl_sync(FULL, base, 0);
            for (uint32_t j = lane; j < nrec; j += 32)
                if (base + j < p.s.R) cnext[(uint64_t)my_slot() * p.s.R + base + j] = s_r[j];
            __syncwarp();
            nrec = 0;
        };
        // R (a compile-time tag, so the two variants of the probe loops are separate
        // code): record the open candidates, or only count them
        auto record_open = [&](auto R, bool still, uint32_t v) {
            if constexpr (!decltype(R)::value) {  // counted only (per lane: the block sum adds the lanes up)
                open_cnt += still;
                return;
            }
            const uint32_t bal = __ballot_sync(FULL, still);
            if (still) s_r[nrec + __popc(bal & lanemask_lt())] = v;
            nrec += __popc(bal);
            if (nrec > REC_STAGE - 32) {
                __syncwarp();
                flush_rec();
            }
        };
        // one probe round: up to PROBE in-edges [e, end) of this lane's candidate, loads in flight together
        auto probe = [&](uint64_t& e, uint64_t end, bool& found) {
            uint32_t u[PROBE];
#pragma unroll
            for (int k = 0; k < PROBE; ++k) u[k] = (e + k < end) ? __ldg(p.g.ici + e + k) : INF;
            uint32_t w[PROBE];
#pragma unroll
            for (int k = 0; k < PROBE; ++k) w[k] = u[k] != INF ? cur[u[k] >> 5] : 0u;
#pragma unroll
            for (int k = 0; k < PROBE; ++k) found |= u[k] != INF && ((w[k] >> (u[k] & 31)) & 1u);
            const uint64_t k = min((uint64_t)PROBE, end - e);
            edges += k;
            e += k;
        };
        // phase 2 — the warp's `nopen` open candidates in s_c walk their in-edge rows
        auto walk_open = [&](auto R, uint32_t nopen, uint64_t w0) {
            uint32_t v_n = 0;
            uint64_t beg_n = 0, end_n = 0;
            if (lane < nopen) {
                v_n = s_c[lane];
                beg_n = __ldg(p.g.irp + v_n);
                end_n = __ldg(p.g.irp + v_n + 1);
            }
            for (uint32_t r = 0; r < nopen; r += 32) {
                const bool open = r + lane < nopen;
                const uint32_t v = v_n;
                const uint64_t beg = beg_n, end = end_n;
                bool found = false;
                uint64_t e = beg;
                rows += open;
                if (open) probe(e, end, found);  // first row round
                beg_n = end_n = 0;
                if (r + 32 + lane < nopen) {
                    v_n = s_c[r + 32 + lane];
                    beg_n = __ldg(p.g.irp + v_n);
                    end_n = __ldg(p.g.irp + v_n + 1);
                }
                // thread granularity: small candidates continue on their lane
                const bool small = open && (end - beg) < p.s.sep_small;
                if (small) {
                    ++cand_small;
                    while (!found && e < end) probe(e, end, found);
                }
                // warp granularity: medium / large candidates still open, 32 edges per step
                uint32_t todo = __ballot_sync(FULL, open && !small && !found && e < end);
                while (todo) {
                    const int l = __ffs(todo) - 1;
                    todo &= todo - 1;
                    const uint64_t b0 = __shfl_sync(FULL, e, l), e0 = __shfl_sync(FULL, end, l);
                    bool hit = false;
                    // WALK_K edges per lane per step, their loads in flight together (the
                    // tail of a level is a few long walks; fewer, wider steps shorten them)
                    for (uint64_t b = b0; b < e0; b += 32 * WALK_K) {
                        uint32_t u[WALK_K];
#pragma unroll
                        for (int k = 0; k < WALK_K; ++k) {
                            const uint64_t x = b + k * 32 + lane;
                            u[k] = x < e0 ? __ldg(p.g.ici + x) : INF;
                        }
                        bool hh = false;
#pragma unroll
                        for (int k = 0; k < WALK_K; ++k)
                            if (u[k] != INF) {
                                ++edges;
                                hh |= bm_test(cur, u[k]);
                            }
                        if (__any_sync(FULL, hh)) {
                            hit = true;
                            break;
                        }
                    }
                    if ((int)lane == l) found = hit;
                    ++cand_warp;
                }
                if (found) on_found(v, w0);
                const bool still = open && !found;
                if (still) mopen += end - beg;
                record_open(R, still, v);
            }
        };
        // the warp's `total` candidates in s_c through phases 1 and 2
        // sh: the chunk's staged hub slice (vertices from vbase), or nullptr (global loads)
        auto run_cands = [&](auto R, uint32_t total, uint64_t w0, const uint32_t* sh, uint32_t vbase) {
            uint32_t nopen = 0;
            // a round's candidates and their hub entries (the in-place compaction below
            // only writes positions before the round, so a later round can be read early)
            uint32_t vn[HUB_ILP], xn[HUB_ILP];
            auto load_round = [&](uint32_t r0) {
#pragma unroll
                for (int k = 0; k < HUB_ILP; ++k) {
                    const uint32_t i = r0 + 32 * k + lane;
                    vn[k] = i < total ? s_c[i] : INF;
                }
#pragma unroll
                for (int k = 0; k < HUB_ILP; ++k)
                    xn[k] = vn[k] == INF ? INF : sh ? sh[vn[k] - vbase] : __ldg(p.hub + vn[k]);
            };
            load_round(0);
            for (uint32_t r0 = 0; r0 < total; r0 += 32 * HUB_ILP) {
                uint32_t v[HUB_ILP], h[HUB_ILP], wd[HUB_ILP];
                bool sole[HUB_ILP];
#pragma unroll
                for (int k = 0; k < HUB_ILP; ++k) {
                    v[k] = vn[k];
                    h[k] = hub_id(xn[k]);
                    sole[k] = hub_sole(xn[k]);
                }
#pragma unroll
                for (int k = 0; k < HUB_ILP; ++k) wd[k] = h[k] != INF ? cur[h[k] >> 5] : 0u;
                // software pipeline (SX_HUB_PIPE): the next round's hub loads fly while this
                // round's frontier tests and bookkeeping run
                if (HUB_PIPE && r0 + 32 * HUB_ILP < total) load_round(r0 + 32 * HUB_ILP);
                __syncwarp();
#pragma unroll
                for (int k = 0; k < HUB_ILP; ++k) {
                    const bool f = h[k] != INF && ((wd[k] >> (h[k] & 31)) & 1u);
                    edges += h[k] != INF;
                    if (f) on_found(v[k], w0);
                    const bool settled = v[k] != INF && !f && sole[k];
                    if (settled) mopen += 1;
                    record_open(R, settled, v[k]);
                    // open ones are compacted in place at the front of s_c (stable)
                    const bool open = v[k] != INF && !f && !sole[k];
                    const uint32_t bal = __ballot_sync(FULL, open);
                    if (open) s_c[nopen + __popc(bal & lanemask_lt())] = v[k];
                    nopen += __popc(bal);
                }
                __syncwarp();
                if (!HUB_PIPE && r0 + 32 * HUB_ILP < total) load_round(r0 + 32 * HUB_ILP);
            }
            ANAT(3, nopen);  // hub-first probe rounds
            walk_open(R, nopen, w0);
        };
        uint32_t s_cur = my_slot();
        uint32_t chunk = 0;
        if (list_mode) {
            // chunks of the recorded candidates; the chunk size adapts so that
            // every warp of the grid gets work when the list is short
            const uint32_t* ccur = p.s.lists[it & 1] + (uint64_t)CAND_CLS * p.s.cstride;
            if (threadIdx.x < 32) {
                const uint32_t x = min(vload(&c->line[it % 3].s[lane].alive), p.s.R);
                uint32_t inc = x;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(FULL, inc, o);
                    if ((int)lane >= o) inc += y;
                }
                s_cpre[lane] = inc - x;
                if (lane == 31) s_cpre[NSLOT] = inc;
            }
            __syncthreads();
            const uint64_t per_warp = (ncand + gwarps() - 1) / gwarps();
            uint32_t csz = per_warp >= 192 ? 256u : per_warp >= 96 ? 128u : per_warp >= 48 ? 64u : 32u;
            if (csz > LIST_CSZ_MAX) csz = LIST_CSZ_MAX;
            const uint32_t nchunks = (ncand + csz - 1) / csz;
            chunk = grab_chunk(nx, nchunks, s_cur);
            while (chunk != INF) {
                const uint32_t s_iss = s_cur, raw_n = grab_issue(nx, s_cur);  // next claim in flight
                const uint32_t i0 = chunk * csz;
                const uint32_t total = min(csz, ncand - i0);
                for (uint32_t j = lane; j < total; j += 32) {
                    const uint32_t i = i0 + j;
                    int lo = 0, hi = NSLOT;  // largest lo with s_cpre[lo] <= i
#pragma unroll
                    for (int q = 0; q < 5; ++q) {
                        const int mid = (lo + hi) >> 1;
                        if (s_cpre[mid] <= i) lo = mid;
                        else hi = mid;
                    }
                    s_c[j] = ccur[(uint64_t)lo * p.s.R + (i - s_cpre[lo])];
                }
                __syncwarp();
                if (rec_open) run_cands(std::true_type{}, total, 0, nullptr, 0u);
                else run_cands(std::false_type{}, total, 0, nullptr, 0u);
                __syncwarp();
                flush_rec();
                chunk = grab_finish(nx, nchunks, s_cur, raw_n, s_iss);
            }
        } else {
            const uint32_t nchunks = (uint32_t)((nw + CW - 1) / CW);
            // TMA staging: buffer b of this warp, its mbarrier and phase
            uint32_t* shub = s_dyn_hub + (uint32_t)warp_id() * 2u * CV;
            uint64_t* mbar = s_mbar[warp_id()];
            const bool tma = SX_PULL_TMA && p.tma;
            uint32_t buf = 0, phase = 0;  // phase bit b: parity to wait for on buffer b
            if (tma) {
                if (lane == 0) {
                    mbar_init(&mbar[0], 1);
                    mbar_init(&mbar[1], 1);
                }
                __syncwarp();
            }
            auto stage_hub = [&](uint32_t ch, uint32_t b) {
                if (!tma || ch == INF) return;
                __syncwarp();  // every lane is done reading buffer b (the chunk before last)
                if (lane == 0) {
                    const uint64_t v0 = (uint64_t)ch * CV;
                    const uint32_t nv = (uint32_t)min((uint64_t)CV, n - v0);
                    fence_proxy_async_smem();
                    tma_load_1d(shub + b * CV, p.hub + v0, (nv * 4u + 15u) & ~15u, &mbar[b]);
                }
            };
            chunk = PULL_STATIC ? (gwarp() < nchunks ? (uint32_t)gwarp() : INF) : grab_chunk(nx, nchunks, s_cur);
            stage_hub(chunk, 0);
            while (chunk != INF) {
#if SX_PULL_TMA
                const uint32_t chunk_n = grab_chunk(nx, nchunks, s_cur);  // the TMA prefetch needs it now
                stage_hub(chunk_n, buf ^ 1u);
#else
                const uint32_t s_iss = s_cur, raw_n = PULL_STATIC ? 0u : grab_issue(nx, s_cur);  // next claim in flight
#endif
                const uint64_t w0 = (uint64_t)chunk * CW;
                const uint64_t wl = w0 + lane;
                const bool mine = lane < CW && wl < nw;
                const uint32_t vis_l = mine ? p.visited[wl] : FULL;
                const uint32_t cand_l = mine ? (~vis_l & __ldg(p.g.nz_in + wl)) : 0u;
#ifdef SX_BFS_ANAT
                if (an_on) an[7] += 1;  // chunks
#endif
                ANAT(0, cand_l);  // chunk claim -> visited / in-degree words
                uint32_t incl = __popc(cand_l);
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(FULL, incl, o);
                    if ((int)lane >= o) incl += y;
                }
                const uint32_t total = __shfl_sync(FULL, incl, 31);
                const uint32_t* sh = nullptr;
                if (tma) {  // the chunk's hub slice has landed (always consume the phase)
                    mbar_wait(&mbar[buf], (phase >> buf) & 1u);
                    phase ^= 1u << buf;
                    sh = shub + buf * CV;
                    buf ^= 1u;
                }
                if (total) {
                    uint32_t pos = incl - __popc(cand_l);
                    for (uint32_t w = cand_l; w; w &= w - 1) s_c[pos++] = (uint32_t)(wl << 5) + (__ffs(w) - 1);
                    s_f[lane] = 0;
                    __syncwarp();
                    ANAT(1, pos);  // scan + compaction into shared memory
                    if (rec_open) run_cands(std::true_type{}, total, w0, sh, (uint32_t)(w0 << 5));
                    else run_cands(std::false_type{}, total, w0, sh, (uint32_t)(w0 << 5));
                    __syncwarp();
                    ANAT(4, s_f[lane]);  // row walks of the open candidates
                    flush_rec();
                    const uint32_t fm = s_f[lane];
                    if (fm) {
                        p.visited[wl] = vis_l | fm;  // this warp owns the chunk's words during the level
                        nbm[wl] = fm;
                        found_cnt += __popc(fm);
                    }
                    if (rec_found && __any_sync(FULL, fm != 0)) {  // the chunk's found vertices onto the hand-over list, one atomic per warp
                        const uint32_t nfl = __popc(fm);
                        uint32_t inc = nfl;
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const uint32_t y = __shfl_up_sync(FULL, inc, o);
                            if ((int)lane >= o) inc += y;
                        }
                        const uint32_t tot = __shfl_sync(FULL, inc, 31);
                        if (tot) {
                            uint32_t base = 0;
                            if (lane == 0) base = atomicAdd(fcnt, tot);
                            base = __shfl_sync(FULL, base, 0) + inc - nfl;
                            for (uint32_t x = fm; x; x &= x - 1) flist[base++] = (uint32_t)(wl << 5) + (__ffs(x) - 1);
                        }
                    }
                    __syncwarp();
                }
                ANAT(5, found_cnt);  // merge + stores of the chunk's words
#if SX_PULL_TMA
                chunk = chunk_n;
#else
                if (PULL_STATIC) chunk = chunk + gwarps() < nchunks ? chunk + (uint32_t)gwarps() : INF;
                else chunk = grab_finish(nx, nchunks, s_cur, raw_n, s_iss);
#endif
                ANAT(6, chunk);  // the next chunk's claim
            }
        }
#ifdef SX_BFS_ANAT
        if (an_on && lane == 0)
            for (int k = 0; k < 8; ++k) atomicAdd(&g_bfs_anat[k], an[k]);
#endif
        st.edges += edges;
        st.reached += found_cnt;
#ifdef SX_BFS_SPREAD
        // profiling build: when each CTA finished its work of this pull level
        // (globaltimer), per level and CTA, into the trace buffer's tail area
        __syncthreads();
        if (threadIdx.x == 0 && p.s.trace)
            reinterpret_cast<uint64_t*>(p.s.trace + 32)[(it % 8) * MAX_GRID + blockIdx.x] = globaltimer();
#endif
        {
            uint64_t v4[5] = {p.sym ? mopen : mdeg, found_cnt, cand_small, cand_warp, open_cnt};
            block_sum<5>(v4);
            if (threadIdx.x == 0) {
                Slot& sl = nx->s[my_slot()];
                if (v4[0]) atomicAdd(&sl.mdeg, (unsigned long long)v4[0]);
                if (v4[1]) atomicAdd(&sl.found, (unsigned int)v4[1]);
                if (v4[2]) atomicAdd(&sl.cnt[0], (unsigned int)v4[2]);
                if (v4[3]) atomicAdd(&sl.cnt[1], (unsigned int)(v4[3] / 32));
                if (v4[4]) atomicAdd(&sl.alive, (unsigned int)v4[4]);  // counted, not recorded
            }
        }
        st.entries += rows;
        st.scanned += (lead() && !list_mode ? nw * 32 : 0);
        if (!grid_sync(c)) return false;
        LineSum ls;
        read_line(nx, ls);
        const uint64_t nf = ls.found;
        // symmetric: the line holds sum deg(still unvisited); else sum deg(found)
        const uint64_t mf = p.sym ? m_u - ls.mdeg : ls.mdeg;
        mf_last = mf;
        const uint32_t nopen_all = ls.alive;
        const uint32_t tc[NCLS] = {ls.cnt[0], ls.cnt[1], 0u, nopen_all};
        m_u -= mf;
        ++it;
        ++st.iters;
        ++st.pull;
        trace_put(p.s, it, DIR_PULL, list_mode ? 0u : 1u, tc, nf, mf, m_u);
        if (nf == 0 || (p.s.max_iters && it >= p.s.max_iters)) {
            done = 1;
            break;
        }
        const bool to_push = p.s.force_dir == 1 ||
                             (p.s.force_dir == 0 && (double)nf < (double)n / p.s.beta && nf < nf_prev);
        nf_prev = (uint32_t)nf;
        if (to_push) {
            dir = !ALL && cluster_ok(p.s, nf, mf) ? DIR_CLUSTER : DIR_PUSH;
            // the grid push takes the recorded found list (class split, no bitmap scan)
            if (dir == DIR_PUSH && rec_found && p.s.force_filter != 2) {
                to_list = 2;
                handoff = 1;
            }
            if (dir == DIR_CLUSTER && rec_found && p.s.force_filter != 2) {
                // hand the frontier over as the list recorded in flist / fcnt: the
                // cluster kernel skips its bitmap scan; the stale bitmap it would
                // clear is cleared here by the whole grid
                handoff = 1;
                clear_bitmap(p.s.bm[(it + 2) % 3], p.s.nwords);
            }
            break;
        }
        if (!p.s.fusion) break;
        // LIST mode next when the open candidates are few and every slot region held its share
        ncand = 0;
        cand_cnt = nopen_all;  // the next level's candidates
        if (rec_open && nopen_all > 0 && nopen_all <= n / LIST_DIV) {
            __shared__ uint32_t s_ok;
            if (threadIdx.x < 32) {
                const uint32_t ok = __all_sync(FULL, vload(&nx->s[lane].alive) <= p.s.R);
                if (lane == 0) s_ok = ok;
            }
            __syncthreads();
            if (s_ok) ncand = nopen_all;
            __syncthreads();
        }
    }
    if (lead()) {
        // the found-list counters stay zero outside a hand-over
        for (int i = 0; i < 3; ++i)
            if (!(handoff && i == (int)(it % 3))) c->cl.cnt[i] = 0;
        c->cl.ready = handoff && dir == DIR_CLUSTER;
    }
    bfs_exit<ALL>(p, DIR_PULL, it, m_u, nf_prev, dir, done, to_list, 0u, cnt, st, &rs, mf_last);
    return true;
}
__global__ void __launch_bounds__(BLOCK, SX_PULL_MINB) bfs_pull(BfsP p) {
    RunState& rs = const_cast<RunState&>(run_state(p.s.ctl));
    if (rs.done || rs.dir != DIR_PULL) return;
    grid_begin(rs.launch);
    pull_phase<false>(p, rs);
}



// ------------------------------------------------------------------ all fusion
// fusion = 2 ("all-fusion", one kernel for the whole run).
// One cooperative launch: the state init, then push and pull phases back to
// back (a direction switch costs a grid barrier, not a kernel exit and a
// relaunch), small frontiers on the grid (no cluster kernel).  The paper's
// all-fusion kernel lost occupancy to the union of the push and pull register
// demands (110 registers); here the launch bounds hold it at the
// occupancy of the separate kernels (3 CTAs x 256 threads per SM), because the
// phases are disjoint code regions and registers are allocated for the
// larger of the two, not their sum.  At the end one more barrier, then CTA 0
// copies the control block's tail into the mapped host mirror (no tail-copy
// kernel).
#ifndef SX_ALL_MINB
#define SX_ALL_MINB 3
#endif
__global__ void __launch_bounds__(BLOCK, SX_ALL_MINB) bfs_all(BfsP p, uint32_t src, uint32_t dir0, Ctl* hctl,
                                                              int fuse_init, AsyncAcc* acc) {
    Ctl* c = p.s.ctl;
    // a broken barrier (watchdog): every CTA leaves; CTA 0 reports it to the
    // host mirror (sync run) or the async accumulator
    auto failed = [&]() {
        if (lead()) {
            if (hctl) hctl->error = ERR_BARRIER;
            if (acc) atomicAdd(&acc->errors, 1u);
        }
    };
#ifdef SX_BFS_MARKS
    const uint64_t t_start = globaltimer();  // profiling build: record 0's aux = ns from kernel start
#else
    const uint64_t t_start = 0;
#endif
    grid_begin(c);  // parity of this launch (the previous launch's exit zeroed this half)
    if (fuse_init) {
        bfs_init_body<true>(p, src, dir0);
        BFS_MARK(3);
        if (!grid_sync(c)) return failed();
    }
    {
        const uint32_t z[NCLS] = {0u, 0u, 0u, 0u};
        trace_put(p.s, 0, DIR_PUSH, 0u, z, 1, 0, t_start ? globaltimer() - t_start : 0);  // end of the state init (iteration 0)
    }
    RunState& rs = const_cast<RunState&>(run_state(c));
    while (!rs.done) {
        const bool ok = rs.dir == DIR_PULL ? pull_phase<true>(p, rs) : push_phase<true>(p, rs);
        if (!ok) return failed();
    }
    BFS_MARK(4);
    if (acc) {
        // asynchronous run: every CTA flushed its statistics into the accumulator
        // itself, and no later launch reads this one's counters: no closing barrier
        if (lead()) {
            grid_end(c);
            c->launch += 1;
            acc->runs += 1;
        }
        return;
    }
    if (!grid_sync(c)) return failed();  // every CTA's statistics are in
    if (blockIdx.x != 0) return;
    if (threadIdx.x == 0) {
        grid_end(c);
        c->launch += 1;
    }
    if (!hctl) return;
    __syncthreads();
    constexpr size_t off = offsetof(Ctl, iter);
    constexpr size_t nw = (sizeof(Ctl) - off) / 4;
    const uint32_t* sw = reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(c) + off);
    uint32_t* dw = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(hctl) + off);
    for (uint32_t i = threadIdx.x; i < nw; i += BLOCK) dw[i] = vload(sw + i);
}

// ------------------------------------------------------------------ small-frontier cluster mode
// Push on one 16-CTA cluster (engine.cuh: cluster_entry / cluster_leave) while
// the frontier is small: the start from a low-degree source and the tail after
// the bottom-up levels.  Vertices of out-degree > CL_BIG have their edges spread
// over the whole cluster.  Back to the grid push once the next frontier exceeds
// 8 x cluster_enter vertices or CL_EDGES x cluster_enter out-edges.
__global__ void __cluster_dims__(CL_CTAS, 1, 1) __launch_bounds__(CL_BLOCK, 1) bfs_cluster(BfsP p) {
    Ctl* c = p.s.ctl;
    const RunState& rs = run_state(c);
    if (rs.done || rs.dir != DIR_CLUSTER) return;
    constexpr uint32_t T = CL_CTAS * CL_BLOCK;
    const uint32_t tid = cluster_rank() * CL_BLOCK + threadIdx.x;
    const bool lead0 = tid == 0;
    uint32_t it = rs.iter;
    uint64_t m_u = rs.m_u;
    uint32_t nf_prev = rs.nf_prev;
    Ctl::ClusterLine* cl = &c->cl;
    uint64_t edges = 0, entries = 0, reached = 0;
    uint32_t iters = 0, done = 0, dir = DIR_CLUSTER, nnext = 0;
    cluster_entry(p.s, it, tid, T);
    const uint64_t lcap = (uint64_t)NCLS * p.s.cstride;  // deferred big tasks fill the next list from the top
    // the current list's size: read once at entry, afterwards carried from the
    // previous iteration's count (one L2 round trip less per iteration)
    uint32_t ncur = vload(&cl->cnt[it % 3]);
    for (;;) {
        if (lead0) {
            cl->cnt[(it + 2) % 3] = 0;
            cl->nbig[(it + 1) % 3] = 0;
            cl->mf[(it + 2) % 3] = 0;  // two ahead: this iteration adds to mf[(it + 1) % 3] before its barrier
        }
        const uint32_t* L = p.s.lists[it & 1];
        uint32_t* NL = p.s.lists[(it + 1) & 1];
        uint32_t* cur = p.s.bm[it % 3];
        uint32_t* nbm = p.s.bm[(it + 1) % 3];
        unsigned int* ncnt = &cl->cnt[(it + 1) % 3];
        const uint32_t lvl = it + 1;
        uint64_t mdeg = 0;
        // visit edges [e0, e1) with stride `step`, 8 in flight: ids -> visited words -> claims
        auto visit = [&](uint64_t e0, uint64_t e1, uint64_t step) {
            for (uint64_t e = e0; e < e1; e += 8 * step) {
                uint32_t u[8], vw[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) u[k] = e + k * step < e1 ? __ldg(p.g.ci + e + k * step) : INF;
#pragma unroll
                for (int k = 0; k < 8; ++k) vw[k] = u[k] != INF ? p.visited[u[k] >> 5] : FULL;
                // the unvisited candidates' claims issued together, then one append per warp
                uint32_t ow[8];
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    ow[k] = (vw[k] >> (u[k] & 31)) & 1u ? FULL : atomicOr(p.visited + (u[k] >> 5), 1u << (u[k] & 31));
                uint32_t sel = 0;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    edges += u[k] != INF;
                    if ((ow[k] >> (u[k] & 31)) & 1u) continue;
                    p.level[u[k]] = lvl;
                    bm_set(nbm, u[k]);
                    mdeg += __ldg(p.g.dout + u[k]);
                    ++reached;
                    sel |= 1u << k;
                }
                cl_append8(NL, ncnt, u, sel);
            }
        };
        for (uint32_t i = tid; i < ncur; i += T) {
            const uint32_t v = L[i];
            atomicAnd(cur + (v >> 5), ~(1u << (v & 31)));  // consumed: keep the bitmaps clean
            const uint64_t beg = __ldg(p.g.rp + v), end = __ldg(p.g.rp + v + 1);
            ++entries;
            if (end - beg > CL_BIG) {
                NL[lcap - 1 - atomicAdd(&cl->nbig[it % 3], 1u)] = v;
                continue;
            }
            visit(beg, end, 1);
        }
        mdeg = warp_sum(mdeg);
        if (lane_id() == 0 && mdeg) atomicAdd(&cl->mf[(it + 1) % 3], (unsigned long long)mdeg);
        mdeg = 0;
        cluster_barrier();
        // deferred-task count, next-list size and m_f read together; one barrier per
        // iteration unless high-degree tasks were deferred
        const uint32_t nbig = vload(&cl->nbig[it % 3]);
        nnext = vload(ncnt);
        uint64_t mf = vload(&cl->mf[(it + 1) % 3]);
        if (nbig) {  // high-degree tasks: their edges spread over the whole cluster
            for (uint32_t j = 0; j < nbig; ++j) {
                const uint32_t v = NL[lcap - 1 - j];
                visit(__ldg(p.g.rp + v) + tid, __ldg(p.g.rp + v + 1), T);
            }
            mdeg = warp_sum(mdeg);
            if (lane_id() == 0 && mdeg) atomicAdd(&cl->mf[(it + 1) % 3], (unsigned long long)mdeg);
            cluster_barrier();
            nnext = vload(ncnt);
            mf = vload(&cl->mf[(it + 1) % 3]);
        }
        m_u -= mf;
        ++it;
        ++iters;
        if (lead0 && p.s.trace) {
            const uint32_t i = c->ntrace++;
            if (i < p.s.trace_cap) {
                TraceRec r;
                r.iter = it;
                r.dir = DIR_CLUSTER;
                r.filter = 0;
                r.launch = c->launch;
                r.n_active[0] = nnext;
                r.n_active[1] = r.n_active[2] = r.n_active[3] = 0;
                r.n_frontier = nnext;
                r.m_active = mf;
                r.aux = m_u;
                r.t_ns = globaltimer();
                p.s.trace[i] = r;
            }
        }
        if (nnext == 0 || (p.s.max_iters && it >= p.s.max_iters)) {
            done = 1;
            break;
        }
        const bool grown = nnext > nf_prev;
        nf_prev = nnext;
        if (nnext > 8u * p.s.cluster_enter || mf > (uint64_t)CL_EDGES * 2u * p.s.cluster_enter) {
            // too big for one cluster: back to the grid, in the direction Beamer's
            // test picks (reading 8) — a push of a frontier whose edges
            // outweigh m_u / alpha costs milliseconds (the bottom-up pull reads the
            // frontier bitmap this kernel kept)
            dir = p.s.force_dir == 2 || (p.s.force_dir == 0 && (double)mf > (double)m_u / p.s.alpha && grown)
                      ? DIR_PULL
                      : DIR_PUSH;
            break;
        }
        ncur = nnext;
    }
    const uint64_t e = warp_sum(edges), en = warp_sum(entries), rc = warp_sum(reached);
    if (lane_id() == 0) {
        if (e) atomicAdd(&c->st[0].edges, (unsigned long long)e);
        if (en) atomicAdd(&c->st[0].entries, (unsigned long long)en);
        if (rc) atomicAdd(&c->st[0].reached, (unsigned long long)rc);
    }
    cluster_barrier();
    if (lead0) {
        c->st[0].iters += iters;
        c->iter = it;
        c->m_u = m_u;
        c->hi = 0;  // the push after the cluster records online
        c->done = done;
        c->dir = dir;
        c->nf_prev = nnext;
        cluster_leave(c);
    }
}

}  // namespace sx

// ------------------------------------------------------------------ host driver
using namespace sx;

// Algorithmic bytes of the executed BFS schedule.
// Push: per list entry 4 B (list) + 16 B (row_ptr pair); per examined edge 4 B
// (col); per reached vertex 4 B (level write); per iteration one frontier-bitmap
// clear (n/8); ballot scans n/8 per scanned vertex / 8.
// Pull (tile scan): per row visit 16 B (row_ptr pair); per examined edge 4 B (the
// hub probe counts as one); per reached vertex 4 B level write + 4 B out-degree
// (directed graphs only: on a symmetric graph m_u needs no degree loads);
// per iteration visited + in-degree>0 + frontier bitmaps and one bitmap clear (4 n/8).
// the state init (level array + visited and three frontier bitmaps), counted when it
// runs inside the fused launch whose bytes the bench's roofline divides
static double bfs_init_bytes(const sx_graph g) { return 4.0 * (double)g->n + 4.0 * 4.0 * (double)g->nwords; }

static double bfs_bytes(const sx_graph g, const sxh::Counters& c) {
    const double n = (double)g->n;
    const double per_reached = g->directed ? 8.0 : 4.0;
    if (c.pull > 0) return 16.0 * c.entries + 4.0 * c.edges + per_reached * c.reached + c.pull * 4.0 * n / 8.0;
    return 20.0 * c.entries + 4.0 * c.edges + 4.0 * c.reached + c.iters * n / 8.0 + c.scanned / 8.0;
}

// SX_TIMING=2: host-side timestamps of one sx_bfs call on stderr (no syncs added).
namespace {
struct HostMarks {
    bool on;
    std::chrono::steady_clock::time_point t0, prev;
    char buf[512];
    int len = 0;
    HostMarks() : on([] { const char* e = getenv("SX_TIMING"); return e && e[0] == '2'; }()) {
        if (on) t0 = prev = std::chrono::steady_clock::now();
    }
    void mark(const char* what) {
        if (!on) return;
        const auto t = std::chrono::steady_clock::now();
        len += snprintf(buf + len, sizeof(buf) - len, " %s %.1f", what, std::chrono::duration<double, std::micro>(t - prev).count());
        prev = t;
    }
    ~HostMarks() {
        if (on) fprintf(stderr, "[sx_bfs host us]%s\n", buf);
    }
};
}  // namespace

extern "C" sx_status sx_bfs(sx_graph g, uint32_t src, const sx_opts* opts, uint32_t* level_out, sx_stats* stats) {
    HostMarks hm;
    if (!g || !level_out) return sxh::fail(SX_E_INVALID, "sx_bfs: NULL graph or level_out");
    sx_status rc = sxh::check_ctx(g->ctx);
    if (rc != SX_OK) return rc;
    if (g->n == 0) return sxh::fail(SX_E_INVALID, "sx_bfs: empty graph has no source");
    if (src >= g->n) return sxh::fail(SX_E_INVALID, "sx_bfs: src >= n");
    sxh::Run run{g, sxh::resolve_opts(opts), stats};
    run.o.cluster_enter = sxh::resolve_cluster(run.o.cluster_enter, true, g->n);
    if (g->directed && !g->has_rev && run.o.force_dir != 1)
        return sxh::fail(SX_E_NO_REVERSE, "sx_bfs: pull needs in-neighbour rows (CSC); use force_dir=1 (push)");
    cudaStream_t s = g->ctx->stream;
    BfsP p;
    p.g = sxh::dev_graph(g);
    if ((rc = sxh::bfs_prepare(g)) != SX_OK) return rc;  // normally done at upload
    if ((rc = run.begin(/*zero_ctl=*/false)) != SX_OK) return rc;  // bfs_init zeroes the control block
    p.s = sxh::make_sched(g, run.o);
    // write levels straight into a device output buffer (no copy-out)
    const bool dev_out = sxh::is_device_ptr(level_out);
    p.level = dev_out ? level_out : g->st[0];
    p.visited = g->aux_bm;
    p.hub = g->hub;
    p.sym = !g->directed;
    p.tma = g->hub && ((uintptr_t)g->hub & 15u) == 0;
    p.acc = nullptr;
    uint32_t dir0 = run.o.force_dir == 2 ? DIR_PULL : DIR_PUSH;
    hm.mark("prologue");
    if (run.o.fusion == 2) {  // all fusion: every phase in one cooperative launch
        // the state init runs inside the persistent launch, the level array filled by
        // TMA bulk stores (SX_ALL_INIT=0: a separate, wider init launch instead)
        static const int fuse_init = [] { const char* e = getenv("SX_ALL_INIT"); return !(e && e[0] == '0'); }();
        if (!fuse_init) {
            bfs_init<<<g->ctx->prop.multiProcessorCount * 8, BLOCK, 0, s>>>(p, src, dir0 | DIR_NOCLUSTER);
            SX_CU(cudaGetLastError());
        }
        Ctl* hctl = g->ctx->d_hctl;
        int fi = fuse_init;
        AsyncAcc* acc = nullptr;
        void* args2[] = {&p, &src, &dir0, &hctl, &fi, &acc};
        if ((rc = run.launch((const void*)bfs_all, args2, sxh::KIND_FUSED, PULL_DYN_SMEM)) != SX_OK) return rc;
        if ((rc = run.sync(false)) != SX_OK) return rc;
        if ((rc = run.end(bfs_bytes)) != SX_OK) return rc;
        if (stats && fuse_init) {
            stats->bytes_push += bfs_init_bytes(g);
            stats->bytes_model += bfs_init_bytes(g);
        }
        hm.mark("end");
        return dev_out ? SX_OK : sxh::copy_out(g, level_out, p.level, g->n * 4);
    }
    bfs_init<<<g->ctx->prop.multiProcessorCount * 8, BLOCK, 0, s>>>(p, src, dir0);
    SX_CU(cudaGetLastError());
    void* args[] = {&p};
    // Selective fusion: the direction-optimising BFS runs push -> pull
    // -> push; the three persistent launches are enqueued back to back
    // without a host round trip — a launch whose direction does not match the
    // device-side state exits at once — and the host syncs once per sequence.
    // likely successor of each phase: push -> pull -> cluster tail (-> push)
    const bool cl_on = run.o.cluster_enter && run.o.fusion && run.o.force_filter < 2 && run.o.force_dir != 2;
    auto next = [&](uint32_t d) -> uint32_t {
        if (d == DIR_PUSH) return DIR_PULL;
        if (d == DIR_PULL) return cl_on ? DIR_CLUSTER : DIR_PUSH;
        return DIR_PUSH;
    };
    auto enqueue = [&](uint32_t d) -> sx_status {
        if (d == DIR_CLUSTER) return run.launch_plain((const void*)bfs_cluster, args, CL_CTAS, CL_BLOCK, false);
        return d == DIR_PULL ? run.launch((const void*)bfs_pull, args, sxh::KIND_PULL, PULL_DYN_SMEM)
                             : run.launch((const void*)bfs_push, args, sxh::KIND_PUSH);
    };
    g->ctx->h_ctl->done = 0;
    // the device picks cluster mode at init for a low-degree source; the host
    // learns the direction only at a sync, so the first sequence starts with it
    // a repeated source (same graph, source and options): start with the direction
    // the device chose last time, so no launch exits at once (correctness never
    // depends on it: a launch of the wrong phase returns and the loop goes on)
    const uint32_t okey = (uint32_t)cl_on | ((uint32_t)run.o.force_dir << 1) | ((uint32_t)run.o.force_filter << 3);
    const bool hit = g->bfs_last_src == src && g->bfs_last_key == okey && g->bfs_last_ce == run.o.cluster_enter &&
                     g->bfs_last_dir0 != INF;
    uint32_t dir = hit ? g->bfs_last_dir0 : (dir0 == DIR_PUSH && cl_on ? DIR_CLUSTER : dir0);
    for (bool first = true;; first = false) {
        // first sequence from a cluster start: cluster, push, pull, cluster (covers
        // both a low- and a high-degree source); later ones three phases deep
        const int len = first && dir == DIR_CLUSTER ? 4 : 3;
        for (int i = 0, d = (int)dir; i < len; ++i, d = (int)next((uint32_t)d))
            if ((rc = enqueue((uint32_t)d)) != SX_OK) return rc;
        hm.mark("enqueue");
        if ((rc = run.sync()) != SX_OK) return rc;
        hm.mark("sync");
        if (first) {
            g->bfs_last_src = src;
            g->bfs_last_key = okey;
            g->bfs_last_ce = run.o.cluster_enter;
            g->bfs_last_dir0 = g->ctx->h_ctl->k;
        }
        if (g->ctx->h_ctl->done) break;
        dir = g->ctx->h_ctl->dir;
    }
    if ((rc = run.end(bfs_bytes)) != SX_OK) return rc;
    hm.mark("end");
    return dev_out ? SX_OK : sxh::copy_out(g, level_out, p.level, g->n * 4);
}

namespace sxh {
// The hub-first probe table (bfs_hub) of a graph with in-neighbour rows: built
// once, at upload, so no BFS call pays for it.
sx_status bfs_prepare(sx_graph g) {
    if (g->hub || !g->has_rev || g->n == 0) return SX_OK;
    sx_status rc = dmalloc(g->ctx, &g->hub, g->n * 4 + 16);
    if (rc != SX_OK) return rc;
    bfs_hub<<<g->ctx->prop.multiProcessorCount * 8, BLOCK, 0, g->ctx->stream>>>(dev_graph(g), g->hub);
    SX_CU(cudaGetLastError());
    return SX_OK;
}

sx_status drain_async(sx_ctx c) {
    if (c->nasync == 0) return SX_OK;
    cudaError_t e = cudaEventSynchronize(c->eva[3 * (c->nasync - 1) + 2]);
    if (e != cudaSuccess) {
        c->poisoned = true;
        return cuda_fail(e, "async BFS");
    }
    for (int i = 0; i < c->nasync; ++i) {
        float t = 0, k = 0;
        SX_CU(cudaEventElapsedTime(&t, c->eva[3 * i], c->eva[3 * i + 2]));
        SX_CU(cudaEventElapsedTime(&k, c->eva[3 * i + 1], c->eva[3 * i + 2]));
        sx_graph g = c->async_g[i];
        g->async_ms += t;
        g->async_ms_fused += k;
        g->async_runs += 1;
        c->async_g[i] = nullptr;
    }
    c->nasync = 0;
    return SX_OK;
}
}  // namespace sxh

// Enqueue one BFS (all fusion: the init kernel and one persistent launch,
// P:742-743) on the ctx stream and return at once.
extern "C" sx_status sx_bfs_async(sx_graph g, uint32_t src, const sx_opts* opts, uint32_t* level_out) {
    if (!g || !level_out) return sxh::fail(SX_E_INVALID, "sx_bfs_async: NULL graph or level_out");
    sx_status rc = sxh::check_ctx(g->ctx);
    if (rc != SX_OK) return rc;
    if (g->n == 0) return sxh::fail(SX_E_INVALID, "sx_bfs_async: empty graph has no source");
    if (src >= g->n) return sxh::fail(SX_E_INVALID, "sx_bfs_async: src >= n");
    if (!sxh::is_device_ptr(level_out)) return sxh::fail(SX_E_INVALID, "sx_bfs_async: level_out must be device memory");
    sx_opts o = sxh::resolve_opts(opts);
    o.fusion = 2;
    o.trace = nullptr;
    o.trace_cap = 0;
    o.cluster_enter = 0;
    if (g->directed && !g->has_rev && o.force_dir != 1)
        return sxh::fail(SX_E_NO_REVERSE, "sx_bfs_async: pull needs in-neighbour rows (CSC); use force_dir=1 (push)");
    sx_ctx c = g->ctx;
    cudaStream_t s = c->stream;
    if ((rc = sxh::bfs_prepare(g)) != SX_OK) return rc;
    if (!g->async_acc) {
        if ((rc = sxh::dmalloc(c, &g->async_acc, sizeof(AsyncAcc))) != SX_OK) return rc;
        SX_CU(cudaMemsetAsync(g->async_acc, 0, sizeof(AsyncAcc), s));
    }
    if (c->nasync == sx_ctx_s::ASYNC_POOL && (rc = sxh::drain_async(c)) != SX_OK) return rc;
    BfsP p;
    p.g = sxh::dev_graph(g);
    p.s = sxh::make_sched(g, o);
    p.level = level_out;
    p.visited = g->aux_bm;
    p.hub = g->hub;
    p.sym = !g->directed;
    p.tma = g->hub && ((uintptr_t)g->hub & 15u) == 0;
    p.acc = g->async_acc;
    uint32_t dir0 = o.force_dir == 2 ? DIR_PULL : DIR_PUSH;
    const int i = c->nasync;
    // one launch per BFS: the state init inside the persistent kernel (TMA bulk stores
    // of the level array); SX_ALL_INIT=0 keeps a separate init launch
    static const int fuse_init = [] { const char* e = getenv("SX_ALL_INIT"); return !(e && e[0] == '0'); }();
    SX_CU(cudaEventRecord(c->eva[3 * i], s));
    if (!fuse_init) {
        bfs_init<<<c->prop.multiProcessorCount * 8, BLOCK, 0, s>>>(p, src, dir0 | DIR_NOCLUSTER);
        SX_CU(cudaGetLastError());
    }
    SX_CU(cudaEventRecord(c->eva[3 * i + 1], s));
    Ctl* hctl = nullptr;
    int fi = fuse_init;
    AsyncAcc* acc = g->async_acc;
    void* args[] = {&p, &src, &dir0, &hctl, &fi, &acc};
    if ((rc = sxh::coop_launch(g, (const void*)bfs_all, args, nullptr, PULL_DYN_SMEM)) != SX_OK) return rc;
    SX_CU(cudaEventRecord(c->eva[3 * i + 2], s));
    c->async_g[i] = g;
    c->nasync = i + 1;
    return SX_OK;
}

// Wait for the graph's enqueued async runs; report and reset their statistics.
extern "C" sx_status sx_graph_sync(sx_graph g, sx_stats* stats) {
    if (!g) return sxh::fail(SX_E_INVALID, "sx_graph_sync: NULL graph");
    sx_status rc = sxh::check_ctx(g->ctx);
    if (rc != SX_OK) return rc;
    sx_ctx c = g->ctx;
    if ((rc = sxh::drain_async(c)) != SX_OK) return rc;
    AsyncAcc h{};
    if (g->async_acc) {
        SX_CU(cudaMemcpyAsync(&h, g->async_acc, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
        SX_CU(cudaMemsetAsync(g->async_acc, 0, sizeof(AsyncAcc), c->stream));
    }
    cudaError_t e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) {
        c->poisoned = true;
        return sxh::cuda_fail(e, "sx_graph_sync");
    }
    if (stats) {
        std::memset(stats, 0, sizeof(*stats));
        const Ctl::StatBlock& a = h.st[0];
        const Ctl::StatBlock& b = h.st[1];
        auto cnt = [](const Ctl::StatBlock& x) {
            sxh::Counters k;
            k.entries = (double)x.entries;
            k.edges = (double)x.edges;
            k.reached = (double)x.reached;
            k.scanned = (double)x.scanned;
            k.iters = (double)x.iters;
            k.pull = (double)x.pull;
            k.ballot = (double)x.ballot;
            return k;
        };
        stats->iterations = a.iters + b.iters;
        stats->launches = g->async_runs;
        stats->launches_fused = g->async_runs;
        stats->ballot_iters = a.ballot + b.ballot;
        stats->pull_iters = a.pull + b.pull;
        stats->edges_examined = a.edges + b.edges;
        stats->vertices_scanned = a.scanned + b.scanned;
        stats->list_entries = a.entries + b.entries;
        static const bool fused_init = [] { const char* e = getenv("SX_ALL_INIT"); return !(e && e[0] == '0'); }();
        stats->bytes_push = bfs_bytes(g, cnt(a)) + (fused_init ? g->async_runs * bfs_init_bytes(g) : 0.0);
        stats->bytes_pull = bfs_bytes(g, cnt(b));
        stats->bytes_model = stats->bytes_push + stats->bytes_pull;
        stats->ms = g->async_ms;
        stats->ms_fused = g->async_ms_fused;
        stats->runs = g->async_runs;
    }
    const uint32_t runs = g->async_runs;
    g->async_ms = g->async_ms_fused = 0;
    g->async_runs = 0;
    if (h.errors) {
        cudaMemsetAsync(g->ctl, 0, sizeof(Ctl), c->stream);  // a clean control block for the next run
        cudaStreamSynchronize(c->stream);
        return sxh::fail(SX_E_BARRIER, "grid barrier watchdog fired in an async run");
    }
    if (h.runs != runs) return sxh::fail(SX_E_STATE, "async run count mismatch");
    return SX_OK;
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
    SX_CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bfs_pull, BLOCK, PULL_DYN_SMEM));
    out->pull_ctas_per_sm = occ;
    SX_CU(cudaFuncGetAttributes(&a, bfs_pull));
    out->pull_regs = a.numRegs;
    return SX_OK;
}

#ifdef SX_BFS_ANAT
extern "C" int sx_debug_bfs_anat(unsigned long long* out16, int reset) {
    cudaDeviceSynchronize();
    if (cudaMemcpyFromSymbol(out16, sx::g_bfs_anat, 16 * 8) != cudaSuccess) return 1;
    if (reset) {
        unsigned long long z[16] = {};
        cudaMemcpyToSymbol(sx::g_bfs_anat, z, sizeof(z));
    }
    return 0;
}
#endif

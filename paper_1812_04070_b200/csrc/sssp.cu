// sssp.cu — SSSP as an ACC algorithm (§3.3; Fig. 4(a)).
//
//   Active  : vertices whose distance changed in the previous iteration
//   Compute : update_{v->u} = dist(v) + w(v,u)
//   Combine : min
//     push: atomicMin on u32 distances — order independent, so results are
//           bit-exact (SURVEY.md §8(c) reading 11);
//     pull: every vertex u folds min over its in-neighbours in the frontier and
//           its single owner writes dist(u) — atomic-free; in-degrees
//           >= sep_huge are folded grid-wide first (block min + one atomicMin).
//   "BFS and SSSP utilize push in the first and last iterations, and pull in
//   between": push -> pull when the frontier's out-edges exceed m/alpha,
//   pull -> push when |F| < n/beta and shrinking (reading 8); selective fusion
//   = one persistent launch per direction phase.
//   delta-stepping: an improved vertex with dist < hi joins the next
//   frontier; otherwise it goes to the far pile (a bitmap).  When the frontier
//   runs dry the bucket advances to the smallest pending distance:
//   hi = (min_far / delta + 1) * delta, and the far vertices below hi are moved
//   to the active list by a ballot pass over the far bitmap.  delta = 0 means
//   delta = infinity: frontier Bellman-Ford (reading 9).
#include "internal.h"

namespace sx {

constexpr double kSsspPullFrac = 0.4;  // auto mode: pull while the frontier's out-edges exceed this x m

struct SsspP {
    DevGraph g;
    Sched s;
    uint32_t* dist;
    uint32_t* far;
    const uint32_t* rs;   // pull: row-start bitmap over in-edges (bit E set)
    const uint32_t* nz;   // pull: rows with in-degree > 0, ascending (+ sentinel)
    const uint32_t* seg;  // pull: tile -> index in nz of its first edge's row
    uint64_t ntiles, E;
    uint32_t delta;
    int sym;
    uint32_t wcc;  // connected components: every weight reads as 0, dist = component label (sx_wcc)
};

__global__ void sssp_init(SsspP p, uint32_t src) {
    Ctl* c = p.s.ctl;
    if (threadIdx.x < 32)
        for (int i = 0; i < 3; ++i) reset_line_warp(&c->line[i]);
    if (threadIdx.x != 0) return;
    p.dist[src] = 0;
    p.s.bm[0][src >> 5] |= 1u << (src & 31);
    const uint32_t k = cls_of(p.g.dout[src], p.s);
    for (int i = 0; i < NCLS; ++i) c->cur_count[i] = 0;
    c->cur_count[k] = 1;
    p.s.lists[0][(uint64_t)k * p.s.cstride] = src;
    c->hi = p.delta ? (unsigned long long)p.delta : 0xFFFFFFFFull + 1;
    c->dir = DIR_PUSH;
    c->lists_ready = 1;
    c->slotted = 0;
    c->nf_prev = 1;
    c->iter = 0;
    c->done = 0;
}

// WCC start (label propagation as an ACC algorithm): every vertex is
// its own label and every vertex with edges is active; the push kernel builds
// the first lists from the frontier bitmap with the ballot filter.
__global__ void wcc_init(SsspP p) {
    Ctl* c = p.s.ctl;
    const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < p.g.n; v += T) p.dist[v] = (uint32_t)v;
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < p.s.nwords; w += T) p.s.bm[0][w] = p.g.nz_in[w];
    if (blockIdx.x == 0 && threadIdx.x < 32)
        for (int i = 0; i < 3; ++i) reset_line_warp(&c->line[i]);
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    for (int i = 0; i < NCLS; ++i) c->cur_count[i] = 0;
    c->hi = 0xFFFFFFFFull + 1;
    c->dir = (p.rs && p.s.force_dir != 1) ? DIR_PULL : DIR_PUSH;  // every vertex active: m_f = m, pull
    c->lists_ready = 0;
    c->slotted = 0;
    c->nf_prev = 0xFFFFFFFFu;
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

__device__ __forceinline__ void sssp_exit(const SsspP& p, uint32_t kdir, uint32_t it, uint64_t hi, uint32_t nf_prev,
                                          uint32_t dir, uint32_t done, uint32_t ready, uint32_t slotted,
                                          const uint32_t (&cnt)[NCLS], Stats& st) {
    Ctl* c = p.s.ctl;
    flush_stats(c, st, kdir);
    if (lead()) {
        c->iter = it;
        c->hi = hi;
        c->nf_prev = nf_prev;
        c->dir = dir;
        c->done = done;
        c->lists_ready = ready;
        c->slotted = slotted;
        for (int i = 0; i < NCLS; ++i) c->cur_count[i] = cnt[i];
        grid_end(c);
        c->launch += 1;
    }
}

// ------------------------------------------------------------------ push
#ifndef SX_SSSP_PUSH_MINB
#define SX_SSSP_PUSH_MINB 4
#endif
__global__ void __launch_bounds__(BLOCK, SX_SSSP_PUSH_MINB) sssp_push(SsspP p) {
    Ctl* c = p.s.ctl;
    const RunState& rs = run_state(c);
    if (rs.done || rs.dir != DIR_PUSH) return;
    stage_init();
    grid_begin(rs.launch);
    uint32_t it = rs.iter;
    uint64_t hi = rs.hi;
    uint32_t nf_prev = rs.nf_prev;
    uint32_t cnt[NCLS];
    uint32_t slotted = 0;
    Stats st;
    if (!rs.lists_ready) {
        // entering push from pull: the frontier exists only as a bitmap -> ballot filter
        if (!ballot_filter(BitmapWords{p.s.bm[it % 3]}, p.s, BallotOut{p.s.lists[it & 1], p.s.cstride, p.g.dout}, cnt))
            return;
        st.scanned += p.s.nwords * 32;
        if (!grid_sync(c)) return;
        view_contig(cnt);
    } else if (rs.slotted) {
        slotted = 1;
        view_slots(&c->line[it % 3], p.s, cnt);
    } else {
        for (int i = 0; i < NCLS; ++i) cnt[i] = rs.cur_count[i];
        view_contig(cnt);
    }
    uint32_t dir = DIR_PUSH, done = 0, ready = 1;
    for (;;) {
        IterLine* nx = &c->line[(it + 1) % 3];
        maybe_reset_line(&c->line[(it + 2) % 3]);
        clear_bitmap(p.s.bm[(it + 2) % 3], p.s.nwords);
        uint32_t* nlists = p.s.lists[(it + 1) & 1];
        uint32_t* nbm = p.s.bm[(it + 1) % 3];
        uint64_t edges = 0, mdeg = 0;
        // record u for the next iteration (claimed once per iteration on the bitmap)
        auto record = [&](uint32_t u) {
            if (p.s.force_filter == 3) {
                // batch filter: every improvement is recorded, duplicates
                // included (the bitmap still marks u for a ballot on overflow)
                bm_set(nbm, u);
                const uint32_t du = __ldg(p.g.dout + u);
                mdeg += du;
                online_record(nx, nlists, p.s, u, cls_of(du, p.s));
            } else if (!bm_test(nbm, u) && bm_claim(nbm, u)) {
                const uint32_t du = __ldg(p.g.dout + u);
                mdeg += du;
                online_record(nx, nlists, p.s, u, cls_of(du, p.s));
            }
        };
        for_tasks(p.s.lists[it & 1], p.s, cnt, [&](uint32_t v, uint64_t rank, uint64_t size, uint32_t) {
            // Local chain (B200 addition, reading 12): a thread-granularity task that
            // improves a vertex below hi processes it at once instead of recording it,
            // up to local_chain vertices in a row.  A later improvement by another
            // thread finds the vertex unclaimed and records it, so nothing is lost.
            for (uint32_t depth = 0;; ++depth) {
                const uint64_t beg = __ldg(p.g.rp + v), end = __ldg(p.g.rp + v + 1);
                if (depth > 0 && end - beg >= p.s.sep_small) {  // a chained vertex too big for one thread
                    record(v);
                    break;
                }
                const uint32_t dv = p.dist[v];
                const bool can_chain = size == 1 && depth < p.s.local_chain;
                uint32_t next = INF;
                auto improved = [&](uint32_t u, uint32_t nd) {
                    if ((uint64_t)nd < hi) {
                        if (can_chain && next == INF) next = u;
                        else record(u);
                    } else if (!bm_test(p.far, u)) {
                        bm_set(p.far, u);
                    }
                };
                if (size == 1) {
                    // thread granularity: 4 edges per step with their loads and
                    // atomics in flight together (one aligned 128-bit id load, one
                    // 32-bit weight load); the edges' chains would otherwise serialise
                    for (uint64_t e = beg; e < end;) {
                        const uint64_t a = e & ~3ull;
                        const uint4 q = __ldg(reinterpret_cast<const uint4*>(p.g.ci + a));
                        const uint32_t u[4] = {q.x, q.y, q.z, q.w};
                        uint32_t w[4];
                        if (p.wcc) {
#pragma unroll
                            for (int k = 0; k < 4; ++k) w[k] = 0u;
                        } else if (p.g.w8) {
                            const uint32_t ww = __ldg(reinterpret_cast<const uint32_t*>(p.g.w8 + a));
#pragma unroll
                            for (int k = 0; k < 4; ++k) w[k] = (ww >> (8 * k)) & 0xFF;
                        } else {
                            const uint4 ww = __ldg(reinterpret_cast<const uint4*>(p.g.w32 + a));
                            w[0] = ww.x;
                            w[1] = ww.y;
                            w[2] = ww.z;
                            w[3] = ww.w;
                        }
                        bool ok[4];
                        uint32_t nd[4], cur[4], old[4];
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            ok[k] = a + k >= e && a + k < end;
                            nd[k] = dv + w[k];
                            cur[k] = ok[k] ? p.dist[u[k]] : 0u;
                        }
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            ok[k] = ok[k] && nd[k] < cur[k];
                            old[k] = ok[k] ? atomicMin(p.dist + u[k], nd[k]) : 0u;
                        }
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            if (ok[k] && nd[k] < old[k]) improved(u[k], nd[k]);
                        const uint64_t stop = min(end, a + 4);
                        edges += stop - e;
                        e = stop;
                    }
                } else {
                    // warp / CTA / grid granularity: 4 edges per step, distances, then
                    // the atomicMins, then the improvement tests, each issued together
                    for_edges_wb(p.g.ci, p.g.w8, p.g.w32, beg, end, rank, size,
                                 [&](const uint32_t (&u)[4], const uint32_t (&w)[4], uint32_t kn) {
                                     edges += kn;
                                     uint32_t nd[4], cur[4], old[4];
                                     bool ok[4];
#pragma unroll
                                     for (int k = 0; k < 4; ++k) {
                                         ok[k] = k < (int)kn;
                                         nd[k] = dv + (p.wcc ? 0u : w[k]);
                                         cur[k] = ok[k] ? p.dist[u[k]] : 0u;
                                     }
#pragma unroll
                                     for (int k = 0; k < 4; ++k) {
                                         ok[k] = ok[k] && nd[k] < cur[k];
                                         old[k] = ok[k] ? atomicMin(p.dist + u[k], nd[k]) : 0u;
                                     }
#pragma unroll
                                     for (int k = 0; k < 4; ++k)
                                         if (ok[k] && nd[k] < old[k]) improved(u[k], nd[k]);
                                 });
                }
                if (next == INF) break;
                v = next;
            }
        });
        stage_flush(nx, nlists, p.s);
        st.edges += edges;
        if (lead()) st.entries += sum4(cnt);
        {
            uint64_t v[1] = {mdeg};
            block_sum<1>(v);
            if (threadIdx.x == 0 && v[0]) atomicAdd(&nx->s[my_slot()].mdeg, (unsigned long long)v[0]);
        }
        if (!grid_sync(c)) return;
        LineSum ls;
        uint32_t vcnt[NCLS];
        read_line_view(nx, p.s, ls, vcnt);
        const uint64_t nf = sum4(ls.cnt);
        const uint64_t mf = ls.mdeg;
        bool overflow = false;
        for (int i = 0; i < NCLS; ++i) overflow |= ls.cntmax[i] > p.s.cap_s;
        if (p.s.force_filter == 2) overflow = true;
        ++it;
        ++st.iters;
        uint32_t filt = overflow ? 1u : 0u;
        // SSSP pull has no early exit: it visits all m in-edges, push visits m_f
        // out-edges with atomics.  Measured on R-MAT s24 (profiles/r1/sssp24_dirs.txt):
        // a pull iteration costs ~0.020 ms per million in-edges, a push iteration
        // ~0.018 ms per million frontier out-edges, so pull never wins (m_f <= m):
        // the automatic mode stays in push; force_dir = 2 still runs the pull path.
        const bool to_pull = nf > 0 && p.s.force_dir != 1 &&
                             (p.s.force_dir == 2 || (double)mf > kSsspPullFrac * (double)p.g.m);
        if (to_pull) {
            trace_put(p.s, it, DIR_PUSH, filt, ls.cnt, nf, mf, hi);
            nf_prev = (uint32_t)nf;
            dir = DIR_PULL;
            ready = 0;
            break;
        }
        if (nf > 0 && nf <= p.s.cluster_enter && p.s.force_filter < 2 && p.s.fusion) {
            // small frontier: continue on one thread-block cluster (frontier handed over as bm[it % 3])
            trace_put(p.s, it, DIR_PUSH, filt, ls.cnt, nf, mf, hi);
            nf_prev = (uint32_t)nf;
            dir = DIR_CLUSTER;
            ready = 0;
            break;
        }
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
                    // a far-flagged vertex improved below hi since has been processed in
                    // this bucket: only the pending ones (dist >= hi) set the next bucket
                    const uint32_t d = p.dist[(wi << 5) + b];
                    if ((uint64_t)d >= hi) mn = min(mn, d);
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
            // moved vertices become this iteration's frontier: list entries AND bitmap bits
            uint32_t* fbm = p.s.bm[it % 3];
            FarWords src{p.far, p.dist, hi};
            if (!ballot_filter(src, p.s, BallotOut{p.s.lists[it & 1], p.s.cstride, p.g.dout}, cnt,
                               [&](uint32_t v, uint32_t) {
                                   p.far[v >> 5] &= ~(1u << (v & 31));
                                   fbm[v >> 5] |= 1u << (v & 31);
                               }))
                return;
            if (!grid_sync(c)) return;
            view_contig(cnt);
            slotted = 0;
            filt = 1;
        }
        trace_put(p.s, it, DIR_PUSH, filt, cnt, nf, mf, hi);
        nf_prev = (uint32_t)(nf ? nf : sum4(cnt));
        if (p.s.max_iters && it >= p.s.max_iters) {
            done = 1;
            break;
        }
        if (!p.s.fusion) break;
    }
    sssp_exit(p, DIR_PUSH, it, hi, nf_prev, dir, done, ready, slotted, cnt, st);
}

// ------------------------------------------------------------------ pull
// Every vertex u with in-edges folds min(dist(v) + w(v,u)) over its in-neighbours
// v in the frontier bitmap (P:340 min combine; P:379 atomic-free for a row that
// one lane owns).  B200 design: the in-edge array is streamed in warp tiles of
// MPT edges (the PageRank tile machinery, pull_all.cu): lane l owns MPV
// consecutive in-edges (128-bit id loads), tests their sources' frontier bits,
// gathers the frontier sources' distances (predicated, issued together), takes
// the min over its runs of equal destination (row starts from the per-graph
// row-start bitmap), and a warp segmented min-scan carries partial runs across
// lanes.  The lane holding a row's last edge in the tile improves the row; a
// row split across tiles is improved piece by piece — min is idempotent, so
// each piece does a compare + atomicMin and no second phase is needed.  An
// improved u joins the next frontier (bitmap claim, exactly once) when
// dist < hi, else the far pile.
__device__ __forceinline__ uint32_t warp_seg_min(uint32_t v, bool start) {
    const uint32_t l = lane_id();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, v, o);
        const bool fy = __shfl_up_sync(FULL, start, o);
        if ((int)l >= o) {
            if (!start) v = min(v, y);
            start |= fy;
        }
    }
    return v;
}

__global__ void __launch_bounds__(BLOCK, 4) sssp_pull(SsspP p) {
    Ctl* c = p.s.ctl;
    const RunState& rs = run_state(c);
    if (rs.done || rs.dir != DIR_PULL) return;
    grid_begin(rs.launch);
    const uint64_t n = p.g.n, E = p.E;
    uint32_t it = rs.iter;
    const uint64_t hi = rs.hi;
    uint32_t nf_prev = rs.nf_prev;
    uint32_t cnt[NCLS] = {0, 0, 0, 0};
    Stats st;
    uint32_t dir = DIR_PULL, done = 0;
    const uint32_t lane = lane_id();
    const bool w8_vec = p.g.iw8 && !((uintptr_t)p.g.iw8 & 7u);
    const bool w32_vec = p.g.iw32 && !((uintptr_t)p.g.iw32 & 15u);
    for (;;) {
        IterLine* nx = &c->line[(it + 1) % 3];
        maybe_reset_line(&c->line[(it + 2) % 3]);
        clear_bitmap(p.s.bm[(it + 2) % 3], p.s.nwords);
        const uint32_t* cur = p.s.bm[it % 3];
        uint32_t* nbm = p.s.bm[(it + 1) % 3];
        uint64_t mdeg = 0, edges = 0;
        uint32_t found = 0;
        // a row that starts and ends inside the tile has this lane as its only
        // writer in the pull: plain store and a fire-and-forget claim;
        // the pieces of a row split across tiles use atomicMin + a returning claim
        auto improve = [&](uint32_t u, uint32_t m, bool owner) {
            if (m >= p.dist[u]) return;
            if (owner) {
                p.dist[u] = m;
            } else {
                const uint32_t old = atomicMin(p.dist + u, m);
                if (m >= old) return;
            }
            if ((uint64_t)m < hi) {
                if (owner) {
                    bm_set(nbm, u);
                    ++found;
                    mdeg += __ldg(p.g.dout + u);
                } else if (bm_claim(nbm, u)) {
                    ++found;
                    mdeg += __ldg(p.g.dout + u);
                }
            } else {
                bm_set(p.far, u);
            }
        };
        for (uint64_t tile = gwarp(); tile < p.ntiles; tile += gwarps()) {
            const uint64_t base = tile * MPT, e0 = base + lane * MPV;
            const bool full = e0 + MPV <= E;
            uint32_t id[MPV], w[MPV];
            if (full) {
                const uint4 qa = __ldg(reinterpret_cast<const uint4*>(p.g.ici + e0));
                const uint4 qb = __ldg(reinterpret_cast<const uint4*>(p.g.ici + e0 + 4));
                id[0] = qa.x; id[1] = qa.y; id[2] = qa.z; id[3] = qa.w;
                id[4] = qb.x; id[5] = qb.y; id[6] = qb.z; id[7] = qb.w;
            } else {
#pragma unroll
                for (int j = 0; j < MPV; ++j) id[j] = e0 + j < E ? __ldg(p.g.ici + e0 + j) : 0u;
            }
            if (p.wcc) {
#pragma unroll
                for (int j = 0; j < MPV; ++j) w[j] = 0u;
            } else if (full && w8_vec) {
                const uint2 q = __ldg(reinterpret_cast<const uint2*>(p.g.iw8 + e0));
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    w[j] = (q.x >> (8 * j)) & 0xFF;
                    w[4 + j] = (q.y >> (8 * j)) & 0xFF;
                }
            } else if (full && w32_vec) {
                const uint4 qa = __ldg(reinterpret_cast<const uint4*>(p.g.iw32 + e0));
                const uint4 qb = __ldg(reinterpret_cast<const uint4*>(p.g.iw32 + e0 + 4));
                w[0] = qa.x; w[1] = qa.y; w[2] = qa.z; w[3] = qa.w;
                w[4] = qb.x; w[5] = qb.y; w[6] = qb.z; w[7] = qb.w;
            } else {
#pragma unroll
                for (int j = 0; j < MPV; ++j) w[j] = e0 + j < E ? edge_w(p.g.iw8, p.g.iw32, e0 + j) : 0u;
            }
            const uint32_t byte = (__ldg(p.rs + (e0 >> 5)) >> (uint32_t)(e0 & 31)) & 0xFFu;  // row starts
            uint32_t nxt = __shfl_down_sync(FULL, byte, 1) & 1u;
            if (lane == 31) nxt = __ldg(p.rs + ((base + MPT) >> 5)) & 1u;
            const uint32_t ends = (byte >> 1) | (nxt << (MPV - 1));
            const uint32_t seg0 = __ldg(p.seg + tile);
            const bool tile_first_start = __shfl_sync(FULL, byte, 0) & 1u;
            const uint32_t mb = lane == 0 ? (byte & ~1u) : byte;
            uint32_t ex = __popc(mb);
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(FULL, ex, o);
                if ((int)lane >= o) ex += y;
            }
            ex -= __popc(mb);
            // frontier words, then the frontier sources' distances, each issued together
            uint32_t fw[MPV], dv[MPV];
#pragma unroll
            for (int j = 0; j < MPV; ++j) fw[j] = e0 + j < E ? cur[id[j] >> 5] : 0u;
#pragma unroll
            for (int j = 0; j < MPV; ++j) dv[j] = ld_pred_u32(p.dist + id[j], (fw[j] >> (id[j] & 31)) & 1u, INF);
            uint32_t x[MPV];
            uint32_t tail = INF;
#pragma unroll
            for (int j = 0; j < MPV; ++j) {
                x[j] = dv[j] == INF ? INF : dv[j] + w[j];
                if ((byte >> j) & 1u) tail = INF;
                tail = min(tail, x[j]);
            }
            const uint32_t nvalid = e0 >= E ? 0u : (E - e0 >= (uint64_t)MPV ? (uint32_t)MPV : (uint32_t)(E - e0));
            edges += nvalid;
            const uint32_t incl = warp_seg_min(tail, byte != 0);
            uint32_t carry = __shfl_up_sync(FULL, incl, 1);
            if (lane == 0 || (byte & 1u)) carry = INF;
            uint32_t run = INF;
#pragma unroll
            for (int j = 0; j < MPV; ++j) {
                if ((byte >> j) & 1u) {
                    run = INF;
                    carry = INF;
                }
                run = min(run, x[j]);
                if ((uint32_t)j < nvalid && ((ends >> j) & 1u)) {
                    const uint32_t m = min(run, carry);
                    if (m != INF) {
                        const uint32_t ridx = seg0 + ex + __popc(mb & ((2u << j) - 1u));
                        const uint32_t u = p.nz[ridx];
                        if (u != INF) improve(u, m, ridx != seg0 || tile_first_start);
                    }
                }
            }
            if (lane == 31 && !nxt && nvalid == MPV && incl != INF) improve(p.nz[seg0 + ex + __popc(mb)], incl, false);
        }
        st.edges += edges;
        {
            uint64_t v2[2] = {mdeg, found};
            block_sum<2>(v2);
            if (threadIdx.x == 0) {
                Slot& sl = nx->s[my_slot()];
                if (v2[0]) atomicAdd(&sl.mdeg, (unsigned long long)v2[0]);
                if (v2[1]) atomicAdd(&sl.found, (unsigned int)v2[1]);
            }
        }
        if (!grid_sync(c)) return;
        LineSum ls;
        read_line(nx, ls);
        const uint64_t nf = ls.found;
        ++it;
        ++st.iters;
        ++st.pull;
        const uint32_t tc[NCLS] = {0u, 0u, 0u, 0u};
        trace_put(p.s, it, DIR_PULL, 1u, tc, nf, ls.mdeg, hi);
        if (p.s.max_iters && it >= p.s.max_iters) {
            done = 1;
            break;
        }
        // an empty frontier goes back to push, which owns the bucket advance
        const bool to_push = nf == 0 || p.s.force_dir == 1 ||
                             (p.s.force_dir == 0 && (double)ls.mdeg <= kSsspPullFrac * (double)p.g.m);
        nf_prev = (uint32_t)nf;
        if (to_push) {
            dir = DIR_PUSH;
            break;
        }
        if (!p.s.fusion) break;
    }
    (void)n;
    sssp_exit(p, DIR_PULL, it, hi, nf_prev, dir, done, 0u, 0u, cnt, st);
}

// ------------------------------------------------------------------ small-frontier cluster mode
// (engine.cuh: cluster_entry / cluster_leave).  Delta-stepping continues inside
// the cluster, bucket advances included; the frontier goes back to the grid
// kernels once it exceeds 8 x cluster_enter vertices.
#ifdef SX_C2_MARKS
// profiling build (profiles/c2_marks.py): where thread 0's iteration goes — SM cycles per
// segment of its dependent chain, summed over the iterations in which it had a task; read
// with sx_debug_c2_marks (not part of the ABI).  A volatile store of the segment's last
// value makes the clock read wait for it.
__device__ unsigned long long g_c2_marks[16];
__device__ volatile uint32_t g_c2_sink;
#define C2MARK(k, dep)                                        \
    do {                                                       \
        if (mk_on) {                                           \
            g_c2_sink = (uint32_t)(dep);                       \
            const unsigned long long t_ = clock64();           \
            mk[k] += t_ - mk_last;                             \
            mk_last = t_;                                      \
        }                                                      \
    } while (0)
#else
#define C2MARK(k, dep) \
    do {               \
    } while (0)
#endif
__global__ void __cluster_dims__(CL_CTAS, 1, 1) __launch_bounds__(CL_BLOCK, 1) sssp_cluster(SsspP p) {
    Ctl* c = p.s.ctl;
    const RunState& rs = run_state(c);
    if (rs.done || rs.dir != DIR_CLUSTER) return;
    constexpr uint32_t T = CL_CTAS * CL_BLOCK;
    const uint32_t tid = cluster_rank() * CL_BLOCK + threadIdx.x;
    const bool lead0 = tid == 0;
    uint32_t it = rs.iter;
    uint64_t hi = rs.hi;
    Ctl::ClusterLine* cl = &c->cl;
    uint64_t edges = 0, entries = 0;
    uint32_t iters = 0, ballots = 0, done = 0, dir = DIR_CLUSTER;
    cluster_entry(p.s, it, tid, T);
    const uint64_t lcap = (uint64_t)NCLS * p.s.cstride;  // entries per list; deferred big tasks fill it from the top
    // Without a claim a vertex improved k times in an iteration is listed k
    // times, so the appends are bounded only by the improvements.  They may fill
    // the lower half of the list (>= 2n entries); the deferred big tasks come
    // from the current list, which never exceeds that half either, and take the
    // upper half from the top.  An iteration whose appends overflow the half
    // (dense graphs) hands the frontier to the grid kernels, which rebuild their
    // lists from the bitmap (every in-bucket improvement is in nbm) - the JIT
    // controller's "overflow -> ballot".
    const uint32_t acap = lcap / 2 < 0xFFFFFFFFull ? (uint32_t)(lcap / 2) : 0xFFFFFFFFu;
    // relax edges [e0, e1) of v, 8 in flight per step: the chain is
    // ids/weights -> atomicMin -> claim (atomicOr) -> append
    // Far-pile minimum kept incrementally (B200 addition): every far insertion
    // min-combines its distance into cl->fmin[fsel]; a bucket advance's compaction
    // leaves the minimum over the vertices it keeps in the other slot.  A bucket
    // advance then reads one word instead of scanning the far pile (after the
    // first advance of a launch: the grid kernels' insertions are not tracked).
    // The value can only undershoot the true pending minimum (an inserted vertex
    // improved again below hi); the advance then moves nothing and the next one
    // reads the exact minimum its compaction left.
    uint32_t fins = INF, fsel = 0;
    bool fvalid = false;
#ifdef SX_C2_MARKS
    unsigned long long mk[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, mk_last = clock64();
    bool mk_on = false;
#endif
    auto flush_fins = [&]() {
        const uint32_t m = warp_min(fins);
        if (lane_id() == 0 && m != INF) atomicMin(&cl->fmin[fsel], m);
        fins = INF;
    };
    auto relax = [&](uint32_t dv, uint64_t e0, uint64_t e1, uint64_t step, uint32_t* nbm, uint32_t* NL,
                     unsigned int* ncnt) {
        for (uint64_t e = e0; e < e1; e += 8 * step) {
            uint32_t u[8], nd[8], old[8];
            bool ok[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint64_t ek = e + k * step;
                ok[k] = ek < e1;
                u[k] = ok[k] ? __ldg(p.g.ci + ek) : 0u;
                nd[k] = dv + (ok[k] && !p.wcc ? (p.g.w8 ? (uint32_t)__ldg(p.g.w8 + ek) : __ldg(p.g.w32 + ek)) : 0u);
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) old[k] = ok[k] ? atomicMin(p.dist + u[k], nd[k]) : 0u;
            C2MARK(10, u[0]);        // ids
            C2MARK(11, nd[0] - dv);  // weights
            C2MARK(3, nd[1]);        // dist(v)
            C2MARK(4, old[0] ^ old[1]);  // the atomicMin results
            uint32_t sel = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                edges += ok[k];
                if (!(ok[k] && nd[k] < old[k])) continue;
                if ((uint64_t)nd[k] < hi) {
                    // no claim round trip on the dependent chain: a vertex improved twice in
                    // an iteration is listed twice and relaxed twice (min is idempotent; the
                    // bitmap bit is still set for a hand-over to the grid kernels).
                    // Measured on C2: 61.2 -> 53.6 ms at delta = 1024.
                    bm_set(nbm, u[k]);
                    sel |= 1u << k;
                } else {
                    bm_set(p.far, u[k]);
                    fins = min(fins, nd[k]);
                }
            }
            // the step's appends with one returning atomic per warp, not one per edge slot
            cl_append8(NL, ncnt, u, sel, acap);
            C2MARK(5, sel);
        }
    };
    // the current list's size: read once at entry, then carried from the previous
    // iteration's count (one L2 round trip less per iteration)
    uint32_t ncur = vload(&cl->cnt[it % 3]);
    for (;;) {
        if (lead0) {
            cl->cnt[(it + 2) % 3] = 0;
            cl->nbig[(it + 1) % 3] = 0;
        }
        const uint32_t* L = p.s.lists[it & 1];
        uint32_t* NL = p.s.lists[(it + 1) & 1];
        uint32_t* cur = p.s.bm[it % 3];
        uint32_t* nbm = p.s.bm[(it + 1) % 3];
        unsigned int* ncnt = &cl->cnt[(it + 1) % 3];
#ifdef SX_C2_MARKS
        mk_on = tid == 0 && ncur > 0;
        if (mk_on) {
            mk[9] += 1;
            mk_last = clock64();
        }
#endif
        for (uint32_t i = tid; i < ncur; i += T) {
            const uint32_t v = L[i];
            C2MARK(1, v);
            atomicAnd(cur + (v >> 5), ~(1u << (v & 31)));  // consumed: keep the bitmaps clean
            const uint64_t beg = __ldg(p.g.rp + v), end = __ldg(p.g.rp + v + 1);
            C2MARK(2, (uint32_t)(beg ^ end));
            ++entries;
            if (end - beg > CL_BIG) {
                NL[lcap - 1 - atomicAdd(&cl->nbig[it % 3], 1u)] = v;
                continue;
            }
            relax(p.dist[v], beg, end, 1, nbm, NL, ncnt);
        }
        flush_fins();
        C2MARK(6, 0u);
        cluster_barrier();
        C2MARK(7, 0u);
        const uint32_t nbig = vload(&cl->nbig[it % 3]);
        uint32_t nnext = vload(ncnt);  // issued together with nbig and the far minimum
        uint32_t fmin = vload(&cl->fmin[fsel]);
        C2MARK(8, nbig ^ nnext ^ fmin);
#ifdef SX_C2_MARKS
        mk_on = false;
#endif
        if (nbig) {  // high-degree tasks: their edges spread over the whole cluster
            for (uint32_t j = 0; j < nbig; ++j) {
                const uint32_t v = NL[lcap - 1 - j];
                relax(p.dist[v], __ldg(p.g.rp + v) + tid, __ldg(p.g.rp + v + 1), T, nbm, NL, ncnt);
            }
            flush_fins();
            cluster_barrier();
            nnext = vload(ncnt);
            fmin = vload(&cl->fmin[fsel]);
        }
        ++it;
        ++iters;
        uint32_t filt = 0;
        const bool overflow = nnext > acap;
        if (nnext == 0) {
            if (p.delta == 0) {
                done = 1;
            } else {
                // bucket advance over the far pile
                uint32_t mn = INF;
                if (fvalid) {
                    mn = fmin;
                } else {
                    cluster_words(p.far, p.s.nwords, tid, T, [&](uint64_t wi, uint32_t x) {
                        word_values(p.dist, wi, x, [&](int, uint32_t d) { mn = min(mn, d); });
                    });
                    mn = warp_min(mn);
                    if (lane_id() == 0 && mn != INF) atomicMin(&cl->minv, mn);
                    cluster_barrier();
                    mn = vload(&cl->minv);
                    cluster_barrier();
                    if (lead0) cl->minv = INF;
                }
                if (mn == INF) {
                    done = 1;
                } else {
                    hi = ((uint64_t)mn / p.delta + 1) * p.delta;
                    uint32_t* L2 = p.s.lists[it & 1];
                    unsigned int* c2 = &cl->cnt[it % 3];
                    uint32_t* fbm = p.s.bm[it % 3];
                    uint32_t rem = INF;  // minimum over the far vertices that stay
                    cluster_compact(p.far, p.s.nwords, tid, T, c2, L2, [&](uint64_t wi, uint32_t f) {
                        uint32_t mv = 0;
                        word_values(p.dist, wi, f, [&](int b, uint32_t d) {
                            if ((uint64_t)d < hi) mv |= 1u << b;
                            else rem = min(rem, d);
                        });
                        if (mv) {
                            p.far[wi] = f & ~mv;  // single owner of the word
                            fbm[wi] |= mv;
                        }
                        return mv;
                    });
                    rem = warp_min(rem);
                    if (lane_id() == 0 && rem != INF) atomicMin(&cl->fmin[fsel ^ 1u], rem);
                    cluster_barrier();
                    if (lead0) cl->fmin[fsel] = INF;  // read by everyone before the barrier above
                    fsel ^= 1u;
                    fvalid = true;
                    nnext = vload(c2);
                    ++ballots;
                    filt = 1;
                }
            }
        }
        if (lead0 && p.s.trace) {
            const uint32_t tc[NCLS] = {nnext, 0u, 0u, 0u};
            const uint32_t i = c->ntrace++;
            if (i < p.s.trace_cap) {
                TraceRec r;
                r.iter = it;
                r.dir = DIR_CLUSTER;
                r.filter = filt;
                r.launch = c->launch;
                for (int k = 0; k < NCLS; ++k) r.n_active[k] = tc[k];
                r.n_frontier = nnext;
                r.m_active = 0;
                r.aux = hi;
                r.t_ns = globaltimer();
                p.s.trace[i] = r;
            }
        }
        if (done) break;
        if (p.s.max_iters && it >= p.s.max_iters) {
            done = 1;
            break;
        }
        if (overflow || nnext > 8u * p.s.cluster_enter) {  // frontier too big for one cluster: back to the grid
            dir = DIR_PUSH;
            break;
        }
        ncur = nnext;
    }
#ifdef SX_C2_MARKS
    if (tid == 0)
        for (int k = 0; k < 12; ++k) atomicAdd(&g_c2_marks[k], mk[k]);
#endif
    // statistics: warp sums, one atomic per warp
    const uint64_t e = warp_sum(edges), en = warp_sum(entries);
    if (lane_id() == 0) {
        if (e) atomicAdd(&c->st[0].edges, (unsigned long long)e);
        if (en) atomicAdd(&c->st[0].entries, (unsigned long long)en);
    }
    cluster_barrier();
    if (lead0) {
        c->st[0].iters += iters;
        c->st[0].ballot += ballots;
        c->st[0].scanned += (uint64_t)ballots * p.s.nwords * 32;
        c->iter = it;
        c->hi = hi;
        c->done = done;
        c->dir = dir;
        c->nf_prev = vload(&cl->cnt[it % 3]);
        cluster_leave(c);
    }
}

}  // namespace sx

using namespace sx;

// Algorithmic bytes: push — per list entry 4 B list + 16 B row_ptr
// pair + 4 B dist(v); per edge 4 B col + weight + 4 B dist(u); per iteration one
// bitmap clear (n/8); ballot / far scans n/8.  Pull (tiles) — every in-edge
// once (4 B id + weight + 1/8 B row-start bit) + per vertex the active-row
// entry, the distance gathers (bounded by the 4n-byte array) and the
// improvement (12 B), + frontier and next bitmaps, per pull iteration.
static double sssp_bytes(const sx_graph g, const sxh::Counters& c) {
    const double n = (double)g->n;
    if (c.pull > 0)
        return c.pull * ((4.125 + g->wbytes) * (double)g->mi + 12.0 * n + 2.0 * n / 8.0) + c.scanned / 8.0;
    return 24.0 * c.entries + (8.0 + g->wbytes) * c.edges + c.iters * n / 8.0 + c.scanned / 8.0;
}

static sx_status run_sssp(sx_graph g, uint32_t src, uint32_t delta, const sx_opts* opts, uint32_t* dist_out,
                          sx_stats* stats, bool wcc) {
    sx_status rc;
    sxh::Run run{g, sxh::resolve_opts(opts), stats};
    run.o.cluster_enter = sxh::resolve_cluster(run.o.cluster_enter, false, g->n);
    if (g->directed && !g->has_rev) run.o.force_dir = 1;  // no in-rows: push only
    cudaStream_t s = g->ctx->stream;
    SsspP p;
    if ((rc = run.begin()) != SX_OK) return rc;
    p.g = sxh::dev_graph(g);
    p.s = sxh::make_sched(g, run.o);
    const bool dev_out = sxh::is_device_ptr(dist_out);
    p.dist = dev_out ? dist_out : g->st[0];
    p.far = g->aux_bm;
    p.delta = delta;
    p.sym = !g->directed;
    p.wcc = wcc ? 1u : 0u;
    if (!wcc) SX_CU(cudaMemsetAsync(p.dist, 0xFF, g->n * 4, s));
    SX_CU(cudaMemsetAsync(p.far, 0, g->nwords * 4, s));
    for (int i = 0; i < 3; ++i) SX_CU(cudaMemsetAsync(p.s.bm[i], 0, g->nwords * 4, s));
    // the tiled pull's per-graph plan (row-start bitmap, active rows, tile map)
    if (!(g->directed && !g->has_rev) && run.o.force_dir != 1) {
        if ((rc = sxh::min_pull_plan(g)) != SX_OK) return rc;
        p.rs = g->pp_rs;
        p.nz = g->pp_gnz;
        p.seg = g->pp_gseg;
        p.ntiles = g->pp_gntiles;
    } else {
        p.rs = p.nz = p.seg = nullptr;
        p.ntiles = 0;
        run.o.force_dir = 1;
        p.s.force_dir = 1;
    }
    p.E = g->mi;
    if (wcc) wcc_init<<<4 * g->ctx->prop.multiProcessorCount, 256, 0, s>>>(p);
    else sssp_init<<<1, 32, 0, s>>>(p, src);
    SX_CU(cudaGetLastError());
    void* args[] = {&p};
    g->ctx->h_ctl->done = 0;
    // Selective fusion: one launch per direction phase (push grid, pull grid, push
    // on one cluster); a launch whose phase does not match the device state exits
    // at once, so the likely next phases are enqueued without a host round trip.
    uint32_t dir = DIR_PUSH;
    auto enqueue = [&](uint32_t d) -> sx_status {
        if (d == DIR_CLUSTER) return run.launch_plain((const void*)sssp_cluster, args, CL_CTAS, CL_BLOCK, false);
        return run.launch(d == DIR_PULL ? (const void*)sssp_pull : (const void*)sssp_push, args, d == DIR_PULL ? sxh::KIND_PULL : sxh::KIND_PUSH);
    };
    for (;;) {
        const uint32_t seq[3] = {dir, dir == DIR_PUSH ? DIR_PULL : DIR_PUSH, dir == DIR_PUSH ? DIR_CLUSTER : dir};
        for (uint32_t d : seq)
            if ((rc = enqueue(d)) != SX_OK) return rc;
        if ((rc = run.sync()) != SX_OK) return rc;
        if (g->ctx->h_ctl->done) break;
        dir = g->ctx->h_ctl->dir;
    }
    if ((rc = run.end(sssp_bytes)) != SX_OK) return rc;
    return dev_out ? SX_OK : sxh::copy_out(g, dist_out, p.dist, g->n * 4);
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
    return run_sssp(g, src, delta, opts, dist_out, stats, false);
}

extern "C" sx_status sx_wcc(sx_graph g, const sx_opts* opts, uint32_t* label_out, sx_stats* stats) {
    if (!g || !label_out) return sxh::fail(SX_E_INVALID, "sx_wcc: NULL graph or label_out");
    sx_status rc = sxh::check_ctx(g->ctx);
    if (rc != SX_OK) return rc;
    if (g->directed) return sxh::fail(SX_E_INVALID, "sx_wcc: undirected graphs only");
    if (g->n == 0) return SX_OK;
    return run_sssp(g, 0, 0, opts, label_out, stats, true);
}

#ifdef SX_C2_MARKS
extern "C" int sx_debug_c2_marks(unsigned long long* out16, int reset) {
    cudaDeviceSynchronize();
    if (cudaMemcpyFromSymbol(out16, sx::g_c2_marks, 16 * 8) != cudaSuccess) return 1;
    if (reset) {
        unsigned long long z[16] = {};
        cudaMemcpyToSymbol(sx::g_c2_marks, z, sizeof(z));
    }
    return 0;
}
#endif

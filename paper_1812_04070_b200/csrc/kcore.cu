// kcore.cu — k-core / coreness as an ACC algorithm (
// SURVEY.md §8(c) readings 6, 7).
//
// Peeling by levels k = 0, 1, 2, ...: at a level start the ballot filter
// (coalesced scan + __ballot_sync) selects the alive vertices with
// residual degree <= k (their coreness is k); each BSP sub-round then pushes
// the removals:
//   Active  : vertices removed in the previous sub-round
//   Compute : update_{v->u} = -1 for every alive neighbour u
//   Combine : aggregation (sum) with atomicSub on the residual degree; the one
//             thread that sees the residual cross k+1 -> k removes u (coreness k)
//             and records it — exactly once, so results are order-independent.
// When a level empties, k jumps to the minimum residual degree among the alive
// vertices (a grid min-reduction).  k > 0 ("fixed k") runs the single level
// k-1 and reports the survivors; k = 0 runs the full decomposition.
// k-Core uses the ballot filter in its first iterations and online afterwards
// — the same JIT controller as BFS/SSSP decides.
#include "internal.h"

namespace sx {

struct KcoreP {
    DevGraph g;
    Sched s;
    uint32_t* res;   // residual degree
    uint32_t* core;  // coreness, INF while alive
    uint32_t* ab;    // alive bitmap (bit v set while core[v] = INF): n/8 bytes, L2-resident
    uint32_t kfix;   // 0 = decomposition
    unsigned long long* q;  // asynchronous cascade queue: qcap items (v << 32 | piece), all ones = not yet written
    uint64_t qcap;          // positions are never reused within a run: n removals + the pieces of split rows
    uint32_t amax;   // a level's cascade goes asynchronous once a sub-round frontier has <= amax vertices (0: never)
};

// Asynchronous tail of a level's cascade (B200 addition; results unchanged by
// reading 7: a vertex is removed exactly once, by the decrement that takes its
// residual from k+1 to k, whatever the order).  Once a sub-round's frontier is
// small, the grid barrier per sub-round (3.2 us, with a dependent chain of a
// few microseconds behind it) dominates: the rest of the level runs as a
// work queue instead.  A removal is an item; a warp takes one ticket (queue
// position) at a time, waits for it to be published and processes the item
// with the whole warp (warp granularity; rows longer than AQ_PIECE
// edges are split into pieces, themselves items), enqueueing the neighbours
// whose residual it takes to k.  One 64-bit
// word counts positions (low half) and pending items (high half): an item is
// pending from its enqueue until its own enqueues are done, so pending = 0
// means the cascade is over.  Only AQ_WARPS warps per CTA take part.
#ifndef SX_AQ_WARPS
#define SX_AQ_WARPS 4
#endif
constexpr uint32_t AQ_WARPS = SX_AQ_WARPS;
constexpr unsigned long long AQ_ONE = 1ull << 32;
#ifndef SX_AQ_RELEASE
#define SX_AQ_RELEASE 1
#endif
__device__ __forceinline__ uint32_t aq_pending(const Ctl* c) { return (uint32_t)(vload(&c->aq_tp) >> 32); }
// watchdog of the queue waits (as the grid barrier's): a lost item would leave
// pending > 0 forever; after 20 s the waiters give up and flag SX_E_BARRIER
__device__ __forceinline__ bool aq_stuck(Ctl* c, uint32_t& spins, uint64_t& t0) {
    if (((++spins) & 1023u) != 0) return false;
    const uint64_t t = globaltimer();
    if (t0 == 0) t0 = t;
    else if (t - t0 > 20000000000ull) atomicExch(&c->error, ERR_BARRIER);
    return vload(&c->error) != 0;
}

constexpr double KCORE_ALPHA = 4.0;  // pull a sub-round whose frontier has > m / 4 out-edges (R-MAT: never)
#ifndef SX_AQ_PIECE
#define SX_AQ_PIECE 256  // measured s24 (session 3): 1024 25.64, 256 25.16 ms at cluster_enter 16384
#endif
constexpr uint32_t AQ_PIECE = SX_AQ_PIECE;  // a removal of a longer row is split into pieces of this many edges
constexpr unsigned long long AQ_EMPTY = ~0ull;
// An item is done: its pending count drops with a RELEASE reduction (the warp's
// enqueues, ordered before it by __syncwarp, are visible first).  A
// __threadfence + atomicAdd did the same with a full fence, which also
// invalidates L1 (CCTL.IVALL): the spilled locals of the queue loop were then
// reloaded from L2 on every item of a cascade's dependent chain.
__device__ __forceinline__ void aq_done(unsigned long long* tp) {
#if SX_AQ_RELEASE
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(tp), "l"((unsigned long long)(-(long long)AQ_ONE))
                 : "memory");
#else
    __threadfence();
    atomicAdd(tp, (unsigned long long)(-(long long)AQ_ONE));
#endif
}
// Work-first (KEEP): the first neighbour an item's warp removes stays with the
// warp as its next item — no ticket, no queue publish and no spin on the
// dependent chain of a cascade; the item's pending token passes to it.  The
// others go to the queue for the idle warps.
#ifndef SX_AQ_KEEP
#define SX_AQ_KEEP 1
#endif
template <class Rm>
__device__ __forceinline__ void kcore_async(const KcoreP& p, Ctl* c, Rm&& remove_edges, uint64_t& entries) {
    if (warp_id() >= AQ_WARPS) return;
    __shared__ uint32_t s_keep[AQ_WARPS];
    uint32_t* keep = SX_AQ_KEEP ? &s_keep[warp_id()] : nullptr;
    const uint32_t lane = lane_id();
    uint32_t spins = 0;
    uint64_t tw = 0;
    unsigned long long kept = AQ_EMPTY;
    for (;;) {
        unsigned long long it = kept;
        kept = AQ_EMPTY;
        if (it == AQ_EMPTY) {
            // one ticket (queue position) per warp; the item is processed by the whole warp
            unsigned long long t = 0;
            if (lane == 0) t = atomicAdd(&c->aq_head, 1ull);
            t = __shfl_sync(FULL, t, 0);
            if (lane == 0) {
                for (;;) {
                    if (t < p.qcap && (it = vload(p.q + t)) != AQ_EMPTY) break;
                    // the cascade is over when nothing is pending: this position stays empty
                    if (aq_pending(c) == 0 || aq_stuck(c, spins, tw)) break;
                    __nanosleep(64);
                }
            }
            it = __shfl_sync(FULL, it, 0);
            if (it == AQ_EMPTY) return;
        }
        // item = (v, piece): piece 0 = a removal; k > 0 = edges [(k-1) P, k P) of v's row
        const uint32_t v = (uint32_t)(it >> 32), pc = (uint32_t)it;
        uint64_t beg = __ldg(p.g.rp + v), end = __ldg(p.g.rp + v + 1);
        if (pc > 0) {
            beg += (uint64_t)(pc - 1) * AQ_PIECE;
            end = min(end, beg + AQ_PIECE);
        } else if (end - beg > AQ_PIECE) {
            // a long row: its pieces become items, spread over the waiting warps
            const uint32_t np = (uint32_t)((end - beg + AQ_PIECE - 1) / AQ_PIECE);
            unsigned long long tp = 0;
            if (lane == 0) tp = atomicAdd(&c->aq_tp, (unsigned long long)np * (AQ_ONE + 1ull));
            tp = __shfl_sync(FULL, tp, 0);
            for (uint32_t k = lane; k < np; k += 32)
                *(volatile unsigned long long*)(p.q + (uint32_t)tp + k) = ((unsigned long long)v << 32) | (k + 1);
            end = beg;
        }
        if (keep && lane == 0) *keep = INF;
        __syncwarp();
        remove_edges(beg, end, (uint64_t)lane, 32ull, keep);
        __syncwarp();
        if (lane == 0) ++entries;
        if (keep) {
            const uint32_t u = *keep;
            if (u != INF) {  // the next item of this warp; this item's pending token passes to it
                kept = (unsigned long long)u << 32;
                continue;
            }
        }
        if (lane == 0) aq_done(&c->aq_tp);  // done with this item
    }
}

__global__ void k_alive_init(uint32_t* ab, uint64_t n, uint64_t nwords) {
    const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwords; w += T) {
        const uint64_t v0 = w << 5;
        ab[w] = v0 + 32 <= n ? FULL : v0 >= n ? 0u : (1u << (uint32_t)(n - v0)) - 1u;
    }
}

__global__ void kcore_init(KcoreP p) {
    Ctl* c = p.s.ctl;
    if (threadIdx.x < 32)
        for (int i = 0; i < 3; ++i) reset_line_warp(&c->line[i]);
    if (threadIdx.x != 0) return;
    for (int i = 0; i < NCLS; ++i) c->cur_count[i] = 0;
    c->k = 0;
    c->iter = 0;
    c->done = 0;
    c->slotted = 0;
    c->dir = DIR_PUSH;
}

__global__ void k_copy_deg(const uint32_t* deg, uint64_t n, uint32_t* res) {
    const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += T) res[i] = deg[i];
}

// Ballot-filter source of a level start: the alive vertices with residual <= k.
// Word wi = alive word wi restricted to those bits (dead words cost one load).
// The alive vertices of word wi, eight at a time: their residual loads are
// issued together (a dense word's bits were a chain of dependent-latency loads)
template <class Fn> __device__ __forceinline__ void for_alive_bits(const uint32_t* res, uint64_t wi, uint32_t w, Fn&& fn) {
    while (w) {
        int b[8];
        uint32_t r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            b[j] = w ? __ffs(w) - 1 : -1;
            w &= w - 1;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = b[j] >= 0 ? res[(wi << 5) + b[j]] : INF;
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (b[j] >= 0) fn(b[j], r[j]);
    }
}
struct LevelWords {
    const uint32_t* ab;
    const uint32_t* res;
    uint32_t k;
    __device__ __forceinline__ uint32_t word(uint64_t wi) const {
        uint32_t m = 0;
        for_alive_bits(res, wi, ab[wi], [&](int b, uint32_t r) {
            if (r <= k) m |= 1u << b;
        });
        return m;
    }
};

#ifndef SX_KCORE_MINB
#define SX_KCORE_MINB 4
#endif
__global__ void __launch_bounds__(BLOCK, SX_KCORE_MINB) kcore_push(KcoreP p) {
    Ctl* c = p.s.ctl;
    const RunState& rs = run_state(c);
    if (rs.done) return;
    stage_init();
    grid_begin(rs.launch);
    const uint64_t n = p.g.n;
    uint32_t it = rs.iter;
    uint32_t k = rs.k;
    uint32_t cnt[NCLS];
    uint32_t slotted = rs.slotted;
    if (slotted) {
        view_slots(&c->line[it % 3], p.s, cnt);
    } else {
        for (int i = 0; i < NCLS; ++i) cnt[i] = rs.cur_count[i];
        view_contig(cnt);
    }
    Stats st;
    uint32_t done = 0;
    bool level_started = it > 0 || sum4(cnt) > 0;
    uint32_t qt = (uint32_t)vload(&c->aq_tp);  // queue tail (the same in every CTA between cascades)
    bool pred_async = false;  // the last level start was small: seed the next one into the queue at once
    uint64_t mf_cur = 0;      // out-edges of the current frontier (0 after a level start: the seeds' are not summed)
    uint64_t aedges = 0;  // edges of the asynchronous cascades
    // one removal's edges in the asynchronous cascade (level k): decrement the
    // alive neighbours; the one whose residual crosses k+1 -> k is removed and enqueued
    // keep (shared memory, nullable): the first removal is kept by the warp instead of enqueued
    auto remove_edges = [&](uint64_t beg, uint64_t end, uint64_t rank, uint64_t size, uint32_t* keep) {
        const uint32_t kk = k;
        for_edges_b(p.g.ci, beg, end, rank, size, [&](const uint32_t (&u)[4], uint32_t kn) {
            aedges += kn;
            uint32_t aw[4], old[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) aw[j] = j < (int)kn ? p.ab[u[j] >> 5] : 0u;
#pragma unroll
            for (int j = 0; j < 4; ++j)
                old[j] = (j < (int)kn && ((aw[j] >> (u[j] & 31)) & 1u)) ? atomicSub(p.res + u[j], 1u) : 0u;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (j < (int)kn && old[j] == kk + 1) {
                    // removal claimed on the alive bit: an asynchronous level's seeding pass
                    // may see the same vertex at residual <= k at the same time
                    const uint32_t bit = 1u << (u[j] & 31);
                    if (!(atomicAnd(p.ab + (u[j] >> 5), ~bit) & bit)) continue;
                    p.core[u[j]] = kk;
                    if (keep && atomicCAS(keep, INF, u[j]) == INF) continue;  // the warp's next item
                    const unsigned long long tp = atomicAdd(&c->aq_tp, AQ_ONE + 1ull);
                    *(volatile unsigned long long*)(p.q + (uint32_t)tp) = (unsigned long long)u[j] << 32;
                }
            }
        });
    };
    for (;;) {
        IterLine* nx = &c->line[(it + 1) % 3];
        if (sum4(cnt) == 0) {
            // ---- level start: min residual degree over alive vertices
            if (p.kfix && level_started) {
                done = 1;
                break;
            }
            // One pass over the alive bitmap computes the minimum residual AND the
            // ballot filter's per-CTA class counts for the speculative level kspec:
            // after a level's cascade every alive vertex has residual > k, so the next
            // level is k + 1 unless the minimum jumps; then the count pass is redone.
            const uint32_t kspec = p.kfix ? p.kfix - 1 : (level_started ? k + 1 : k);
            const LevelWords lw_spec{p.ab, p.res, kspec};
            const bool spec = pred_async && level_started && !p.kfix;
            uint32_t mn = INF;
            uint64_t alive = 0;
            {
                uint64_t w0, w1;
                ballot_chunk(p.s.nwords, w0, w1);
                uint32_t acc[NCLS] = {0, 0, 0, 0};
                const uint32_t lane = lane_id();
                for (uint64_t t = w0; t < w1; t += TILE_WORDS) {
                    const uint64_t wi = t + threadIdx.x;
                    const uint32_t w = p.ab[wi];
                    alive += __popc(w);
                    uint32_t m = 0;  // this word's seeds of kspec
                    for_alive_bits(p.res, wi, w, [&](int b, uint32_t r) {
                        mn = min(mn, r);
                        if (r <= kspec) {
                            m |= 1u << b;
                            if (!spec) cls_count(acc, cls_of(__ldg(p.g.dout + (uint32_t)((wi << 5) + b)), p.s));
                        }
                    });
                    if (spec) {
                        // speculative asynchronous level (the previous one was small): the seeds of
                        // kspec go into the queue now — no second pass; the workers start after
                        // the barrier (if the minimum jumped past kspec, there are none)
                        if (m) {
                            p.ab[wi] = w & ~m;  // this thread owns the word; no worker runs yet
                            for (uint32_t x = m; x; x &= x - 1) p.core[(wi << 5) + (__ffs(x) - 1)] = kspec;
                        }
                        const uint32_t nm = __popc(m);
                        acc[0] += nm;
                        uint32_t incl = nm;
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const uint32_t y = __shfl_up_sync(FULL, incl, o);
                            if ((int)lane >= o) incl += y;
                        }
                        const uint32_t tot = __shfl_sync(FULL, incl, 31);
                        if (tot) {
                            unsigned long long base = 0;
                            if (lane == 0) base = atomicAdd(&c->aq_tp, (unsigned long long)tot * (AQ_ONE + 1ull));
                            base = __shfl_sync(FULL, base, 0);
                            uint32_t pos = (uint32_t)base + incl - nm;
                            for (uint32_t x = m; x; x &= x - 1)
                                *(volatile unsigned long long*)(p.q + pos++) = (unsigned long long)((wi << 5) + (__ffs(x) - 1)) << 32;
                        }
                    }
                }
                block_sum<NCLS>(acc);
                if (threadIdx.x == 0) {
#pragma unroll
                    for (int cc = 0; cc < NCLS; ++cc) p.s.cta_cnt[cc * MAX_GRID + blockIdx.x] = acc[cc];
                    const uint32_t ns = acc[0] + acc[1] + acc[2] + acc[3];
                    if (ns) atomicAdd(&nx->s[my_slot()].found, ns);
                }
            }
            // one token per CTA pending (released by the path taken after the barrier):
            // an asynchronous level's seeding overlaps its workers (added atomically: a
            // speculative level enqueues concurrently)
            if (lead() && p.amax) atomicAdd(&c->aq_tp, (unsigned long long)gridDim.x << 32);
            mn = block_min(mn);
            {
                uint64_t a[1] = {alive};
                block_sum<1>(a);
                alive = a[0];
            }
            if (threadIdx.x == 0) {
                Slot& sl = nx->s[my_slot()];
                if (mn != INF) atomicMin(&sl.minv, mn);
                if (alive) atomicAdd(&sl.alive, (unsigned int)alive);
            }
            if (!grid_sync(c)) return;
            LineSum ls;
            read_line(nx, ls);
            mn = ls.minv;
            if (ls.alive == 0) {
                done = 1;
                break;
            }
            if (p.kfix) {
                if (mn >= p.kfix) {
                    done = 1;
                    break;
                }
                k = p.kfix - 1;
            } else {
                k = max(k, mn);
            }
            level_started = true;
            const bool was_spec = spec;
            pred_async = p.amax && p.s.fusion && ls.found <= p.amax;
            if (was_spec && k == kspec) {
                // ---- the speculative asynchronous level: its seeds are already queued
                ++st.ballot;
                if (lead()) {
                    st.scanned += ls.alive;
                    atomicAdd(&c->aq_tp, (unsigned long long)(-(long long)((unsigned long long)gridDim.x << 32)));
                }
                maybe_reset_line(&c->line[(it + 2) % 3]);
                clear_bitmap(p.s.bm[(it + 2) % 3], p.s.nwords);
#ifdef SX_KCORE_MARKS  // profiling build: the level start is done (CTA 0)
                trace_put(p.s, it + 1, DIR_PUSH, 5u, cnt, ls.found, 0, k);
#endif
                uint64_t entries = 0;
                kcore_async(p, c, remove_edges, entries);
#ifdef SX_KCORE_MARKS  // CTA 0's queue warps saw the cascade end
                __syncthreads();
                trace_put(p.s, it + 1, DIR_PUSH, 6u, cnt, entries, 0, k);
#endif
                st.edges += aedges;
                aedges = 0;
                st.entries += entries;
                ++st.iters;
                if (!grid_sync(c)) return;
                qt = (uint32_t)vload(&c->aq_tp);
                if (lead()) c->aq_head = (unsigned long long)qt;  // the next cascade's tickets start at the tail
                ++it;
                trace_put(p.s, it, DIR_PUSH, 4u, cnt, ls.found, 0, k);
                continue;
            }
            if (p.amax && p.s.fusion && k == kspec && ls.found <= p.amax) {
                // ---- a small level entirely asynchronous: the seeds go straight into
                // the queue (no class lists, no sub-rounds); each CTA releases its token
                ++st.ballot;
                if (lead()) st.scanned += 2 * ls.alive;
                maybe_reset_line(&c->line[(it + 2) % 3]);  // the next level start's line (nx after ++it)
                clear_bitmap(p.s.bm[(it + 2) % 3], p.s.nwords);  // the rotation a sub-round keeps
                uint64_t w0, w1;
                ballot_chunk(p.s.nwords, w0, w1);
                const uint32_t lane = lane_id();
                for (uint64_t t = w0; t < w1; t += TILE_WORDS) {
                    const uint64_t wi = t + threadIdx.x;
                    uint32_t m = lw_spec.word(wi);
                    if (m) {
                        // claimed on the alive bits: the queue workers of CTAs already past
                        // their seeding remove vertices of this level concurrently
                        m &= atomicAnd(p.ab + wi, ~m);
                        for (uint32_t x = m; x; x &= x - 1) p.core[(wi << 5) + (__ffs(x) - 1)] = k;
                    }
                    const uint32_t nm = __popc(m);
                    uint32_t incl = nm;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t y = __shfl_up_sync(FULL, incl, o);
                        if ((int)lane >= o) incl += y;
                    }
                    const uint32_t tot = __shfl_sync(FULL, incl, 31);
                    if (tot) {
                        unsigned long long base = 0;
                        if (lane == 0) base = atomicAdd(&c->aq_tp, (unsigned long long)tot * (AQ_ONE + 1ull));
                        base = __shfl_sync(FULL, base, 0);
                        uint32_t pos = (uint32_t)base + incl - nm;
                        for (uint32_t x = m; x; x &= x - 1)
                            *(volatile unsigned long long*)(p.q + pos++) = (unsigned long long)((wi << 5) + (__ffs(x) - 1)) << 32;
                    }
                }
                __syncthreads();
                if (threadIdx.x == 0) {
                    __threadfence();
                    atomicAdd(&c->aq_tp, (unsigned long long)(-(long long)AQ_ONE));  // this CTA's seeds are in
                }
                uint64_t entries = 0;
                kcore_async(p, c, remove_edges, entries);
                st.edges += aedges;
                aedges = 0;
                st.entries += entries;
                ++st.iters;
                if (!grid_sync(c)) return;
                qt = (uint32_t)vload(&c->aq_tp);
                if (lead()) c->aq_head = (unsigned long long)qt;  // the next cascade's tickets start at the tail
                ++it;
                trace_put(p.s, it, DIR_PUSH, 4u, cnt, ls.found, 0, k);  // filter 4: an asynchronous level
                continue;  // cnt stays empty: the next level start
            }
            // ---- ballot filter selects the level's seeds; their coreness is k
            if (lead() && p.amax) atomicAdd(&c->aq_tp, (unsigned long long)(-(long long)((unsigned long long)gridDim.x << 32)));
            ++st.ballot;
            // the thread owning word v >> 5 in the write pass clears the seeds' alive bits
            uint32_t* fbm = p.s.bm[it % 3];  // the seeds are the frontier of sub-round `it`
            auto seed = [&](uint32_t v, uint32_t) {
                p.core[v] = k;
                p.ab[v >> 5] &= ~(1u << (v & 31));
                fbm[v >> 5] |= 1u << (v & 31);  // the word's single owner in the write pass
            };
            const BallotOut bo{p.s.lists[it & 1], p.s.cstride, p.g.dout};
            if (k == kspec) {  // the counts of the fused pass stand: write pass only
                if (lead()) st.scanned += 2 * ls.alive;
                ballot_write(lw_spec, p.s, bo, cnt, seed);
            } else {
                if (lead()) st.scanned += 3 * ls.alive;
                if (!ballot_filter(LevelWords{p.ab, p.res, k}, p.s, bo, cnt, seed)) return;
            }
            if (!grid_sync(c)) return;
            view_contig(cnt);
            trace_put(p.s, it + 1, DIR_PUSH, 1u, cnt, sum4(cnt), 0, k);  // level start (seeds)
            mf_cur = 0;  // the seeds' degrees are not summed: their sub-round pushes unless forced
        }
        // ---- one sub-round: removals push -1 to alive neighbours
        maybe_reset_line(&c->line[(it + 2) % 3]);
        clear_bitmap(p.s.bm[(it + 2) % 3], p.s.nwords);
        uint32_t* nlists = p.s.lists[(it + 1) & 1];
        uint32_t* nbm = p.s.bm[(it + 1) % 3];
        uint64_t edges = 0, mrec = 0;
        const uint32_t kk = k;
        auto record = [&](uint32_t u) {
            bm_set(nbm, u);
            const uint32_t du = __ldg(p.g.dout + u);
            mrec += du;
            online_record(nx, nlists, p.s, u, cls_of(du, p.s));
        };
        // direction ("pull at the beginning, push in the end"; reading 8's test
        // with m = all edges): a frontier whose out-edges exceed m / KCORE_ALPHA is
        // pulled — every alive vertex counts its frontier neighbours and subtracts
        // them at once (single owner, no atomics) — otherwise pushed
        const bool pull_sub = p.s.force_dir == 2 || (p.s.force_dir == 0 && (double)mf_cur * KCORE_ALPHA > (double)p.g.m);
        if (pull_sub) {
            const uint32_t* F = p.s.bm[it % 3];
            for (uint64_t wi = gtid(); wi < p.s.nwords; wi += gthreads()) {
                const uint32_t w = p.ab[wi];
                if (!w) continue;
                uint32_t dead = 0;
                for (uint32_t x = w; x; x &= x - 1) {
                    const int b = __ffs(x) - 1;
                    const uint32_t u = (uint32_t)((wi << 5) + b);
                    const uint64_t beg = __ldg(p.g.rp + u), end = __ldg(p.g.rp + u + 1);
                    uint32_t cnt_f = 0;
                    for_edges_b(p.g.ci, beg, end, 0ull, 1ull, [&](const uint32_t (&v)[4], uint32_t kn) {
                        edges += kn;
#pragma unroll
                        for (int j = 0; j < 4; ++j) cnt_f += j < (int)kn && bm_test(F, v[j]);
                    });
                    if (!cnt_f) continue;
                    const uint32_t r = p.res[u], rn = r > cnt_f ? r - cnt_f : 0u;
                    p.res[u] = rn;
                    if (r > kk && rn <= kk) {  // crosses k+1 -> k in this sub-round: removed once
                        p.core[u] = kk;
                        dead |= 1u << b;
                        record(u);
                    }
                }
                if (dead) p.ab[wi] = w & ~dead;  // this thread owns the word
            }
        } else
        for_tasks(p.s.lists[it & 1], p.s, cnt, [&](uint32_t v, uint64_t rank, uint64_t size, uint32_t) {
            // Local chain (B200 addition, reading 12): a removal that a thread-granularity
            // task triggers is processed at once (the cascade continues within the
            // iteration) instead of being recorded; each vertex is still removed and
            // processed exactly once (the crossing test), so coreness is unchanged.
            for (uint32_t depth = 0;; ++depth) {
                const uint64_t beg = __ldg(p.g.rp + v), end = __ldg(p.g.rp + v + 1);
                if (depth > 0 && end - beg >= p.s.sep_small) {
                    record(v);
                    break;
                }
                const bool can_chain = size == 1 && depth < p.s.local_chain;
                uint32_t next = INF;
                // four edges per step: alive words, then the residual decrements, then the
                // crossing tests, each issued together
                for_edges_b(p.g.ci, beg, end, rank, size, [&](const uint32_t (&u)[4], uint32_t kn) {
                    edges += kn;
                    uint32_t aw[4], old[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) aw[j] = j < (int)kn ? p.ab[u[j] >> 5] : 0u;
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        old[j] = (j < (int)kn && ((aw[j] >> (u[j] & 31)) & 1u)) ? atomicSub(p.res + u[j], 1u) : 0u;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if (j < (int)kn && old[j] == kk + 1) {
                            p.core[u[j]] = kk;
                            atomicAnd(p.ab + (u[j] >> 5), ~(1u << (u[j] & 31)));
                            if (can_chain && next == INF) next = u[j];
                            else record(u[j]);
                        }
                    }
                });
                if (next == INF) break;
                v = next;
            }
        });
        stage_flush(nx, nlists, p.s);
        st.edges += edges;
        if (lead()) st.entries += sum4(cnt);
        {
            uint64_t a[1] = {mrec};
            block_sum<1>(a);
            if (threadIdx.x == 0 && a[0]) atomicAdd(&nx->s[my_slot()].mdeg, (unsigned long long)a[0]);
        }
        if (pull_sub) ++st.pull;
        if (!grid_sync(c)) return;
        LineSum ls;
        uint32_t vcnt[NCLS];
        read_line_view(nx, p.s, ls, vcnt);
        mf_cur = ls.mdeg;  // out-edges of the next frontier (its removals' degrees)
        const uint64_t nf = sum4(ls.cnt);
        bool overflow = false;
        for (int i = 0; i < NCLS; ++i) overflow |= ls.cntmax[i] > p.s.cap_s;
        if (p.s.force_filter == 2) overflow = true;
        ++it;
        ++st.iters;
        trace_put(p.s, it, DIR_PUSH, overflow ? 1u : 0u, ls.cnt, nf, 0, k);
        if (nf > 0 && overflow) {
            ++st.ballot;
            if (!ballot_filter(BitmapWords{nbm}, p.s, BallotOut{p.s.lists[it & 1], p.s.cstride, p.g.dout}, cnt)) return;
            if (!grid_sync(c)) return;
            view_contig(cnt);
            slotted = 0;
        } else {
            for (int i = 0; i < NCLS; ++i) cnt[i] = vcnt[i];  // view set by read_line_view
            slotted = 1;
        }
        if (p.s.max_iters && it >= p.s.max_iters) {
            done = 1;
            break;
        }
        const uint32_t nf32 = sum4(cnt);
        if (p.amax && p.s.fusion && nf32 > 0 && nf32 <= p.amax) {
            // ---- the rest of the level's cascade asynchronously: the frontier seeds the queue
            uint32_t off = qt;
            for (int cc = 0; cc < NCLS; ++cc) {
                for (uint64_t i = gtid(); i < cnt[cc]; i += gthreads())
                    *(volatile unsigned long long*)(p.q + off + i) =
                        (unsigned long long)task_at(p.s.lists[it & 1], p.s, cc, (uint32_t)i) << 32;
                off += cnt[cc];
            }
            if (lead()) {
                c->aq_tp = ((unsigned long long)nf32 << 32) | (unsigned long long)(qt + nf32);
                c->aq_head = (unsigned long long)qt;
            }
            if (!grid_sync(c)) return;
            uint64_t entries = 0;
            maybe_reset_line(&c->line[(it + 2) % 3]);  // the next level start's line (nx after ++it)
            clear_bitmap(p.s.bm[(it + 2) % 3], p.s.nwords);  // the rotation a sub-round keeps
            kcore_async(p, c, remove_edges, entries);
            st.edges += aedges;
            aedges = 0;
            st.entries += entries;
            ++st.iters;
            if (!grid_sync(c)) return;
            qt = (uint32_t)vload(&c->aq_tp);
            if (lead()) c->aq_head = (unsigned long long)qt;  // the next cascade's tickets start at the tail
            for (int i = 0; i < NCLS; ++i) cnt[i] = 0;
            view_contig(cnt);
            slotted = 0;
            ++it;
            trace_put(p.s, it, DIR_PUSH, 3u, cnt, 0, 0, k);  // filter 3: an asynchronous cascade ended
            continue;
        }
        if (!p.s.fusion) break;
    }
    flush_stats(c, st, DIR_PUSH);
    if (lead()) {
        c->iter = it;
        c->k = k;
        c->done = done;
        c->slotted = slotted;
        for (int i = 0; i < NCLS; ++i) c->cur_count[i] = cnt[i];
        grid_end(c);
        c->launch += 1;
    }
}

__global__ void k_kcore_out(const uint32_t* core, uint64_t n, uint32_t kfix, uint32_t* out) {
    const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += T)
        out[i] = kfix ? (core[i] == INF ? 1u : 0u) : core[i];
}

}  // namespace sx

using namespace sx;

// Algorithmic bytes: per list entry 4 B list + 16 B row_ptr pair;
// per edge 4 B col + 4 B residual RMW (the alive test reads an n/8 bitmap, once
// per pass); level starts: 4 B residual per alive vertex per pass (scanned) and
// the alive bitmap (n/8) per pass, 3 passes; per iteration one bitmap clear (n/8).
static double kcore_bytes(const sx_graph g, const sxh::Counters& c) {
    const double bm = (double)g->n / 8.0;
    return 20.0 * c.entries + 8.0 * c.edges + 4.0 * c.scanned + 3.0 * c.ballot * bm + c.iters * bm * 2.0;
}

extern "C" sx_status sx_kcore(sx_graph g, uint32_t k, const sx_opts* opts, uint32_t* core_out, sx_stats* stats) {
    if (!g || !core_out) return sxh::fail(SX_E_INVALID, "sx_kcore: NULL graph or core_out");
    sx_status rc = sxh::check_ctx(g->ctx);
    if (rc != SX_OK) return rc;
    if (g->directed) return sxh::fail(SX_E_INVALID, "sx_kcore: k-core is defined on undirected graphs");
    if (g->n == 0) return SX_OK;
    sxh::Run run{g, sxh::resolve_opts(opts), stats};
    // asynchronous-level threshold: 16384 measured best on s24 (profiles/r2/kcore_sweep.txt)
    if (run.o.cluster_enter == SX_CLUSTER_AUTO) run.o.cluster_enter = 16384;
    cudaStream_t s = g->ctx->stream;
    KcoreP p;
    if ((rc = run.begin()) != SX_OK) return rc;
    p.g = sxh::dev_graph(g);
    p.s = sxh::make_sched(g, run.o);
    p.res = g->st[0];
    p.core = g->st[1];
    p.ab = g->aux_bm;
    p.kfix = k;
    // the asynchronous cascade queue: n positions, written once each (INF = empty)
    p.amax = run.o.cluster_enter;
    p.qcap = g->n + g->m / AQ_PIECE + 64;
    p.q = nullptr;
    if (p.amax) {
        if (!g->kq && (rc = sxh::dmalloc(g->ctx, &g->kq, p.qcap * 8)) != SX_OK) return rc;
        p.q = g->kq;
        SX_CU(cudaMemsetAsync(p.q, 0xFF, p.qcap * 8, s));
    }
    SX_CU(cudaMemsetAsync(p.core, 0xFF, g->n * 4, s));
    for (int i = 0; i < 3; ++i) SX_CU(cudaMemsetAsync(p.s.bm[i], 0, g->nwords * 4, s));
    const int eg = 4 * g->ctx->prop.multiProcessorCount;
    k_copy_deg<<<eg, 256, 0, s>>>(g->dout, g->n, p.res);
    k_alive_init<<<eg, 256, 0, s>>>(p.ab, g->n, g->nwords);
    kcore_init<<<1, 32, 0, s>>>(p);
    SX_CU(cudaGetLastError());
    void* args[] = {&p};
    g->ctx->h_ctl->done = 0;
    for (;;) {
        if ((rc = run.launch((const void*)kcore_push, args, sxh::KIND_PUSH)) != SX_OK) return rc;
        if ((rc = run.sync()) != SX_OK) return rc;
        if (g->ctx->h_ctl->done) break;
    }
    if ((rc = run.end(kcore_bytes)) != SX_OK) return rc;
    const bool dev_out = sxh::is_device_ptr(core_out);
    uint32_t* out = dev_out ? core_out : g->st[2];
    k_kcore_out<<<eg, 256, 0, s>>>(p.core, g->n, k, out);
    SX_CU(cudaGetLastError());
    if (dev_out) {
        SX_CU(cudaStreamSynchronize(s));
        return SX_OK;
    }
    return sxh::copy_out(g, core_out, out, g->n * 4);
}

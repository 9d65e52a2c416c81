// engine.cuh — device-side building blocks of the ACC frontier engine (sm_100a).
//
// PAPER.md (arXiv 1812.04070) passages implemented here:
//   P:365        BSP loop: compute with online recording -> global barrier -> overflow ?
//                ballot filter : prefix-scan concatenation of the bins
//   P:525, P:659 task classes small / medium / large (separators 32 / 128) ->
//                thread / warp / CTA granularity; + a B200 grid-split "huge" class
//   P:549-561    ballot filter: coalesced scan of the "updated" metadata with a warp
//                ballot, per-thread bins concatenated in vertex order -> sorted, unique
//   P:602-608    online filter: record activated vertices while computing
//   P:619-626    JIT control: online first, ballot after an overflow
//   P:701-729    software global barrier made deadlock-free by sizing the grid to
//                guaranteed co-residency (here: cooperative launch of
//                occupancy x SMs CTAs; Eq. 1 generalised)
//
// B200 design notes:
//   * The paper's thread-private bins become warp-aggregated slot claims
//     (__match_any_sync + one atomicAdd per class per warp) into class lists in
//     global memory (L2-resident); "overflow" = a class list exceeding
//     overflow_threshold x (warps in the grid) entries, after which recording
//     only counts (the shadow filter of P:654) and the ballot filter rebuilds the
//     lists.  Exactly-once claims (atomicOr on the frontier bitmap / an atomic
//     crossing test) keep online lists duplicate-free.
//   * The ballot filter scans a frontier BITMAP (one u32 word = 32 vertices, so a
//     lane's word is already the warp ballot of P:555) or evaluates a per-vertex
//     predicate with __ballot_sync; a two-pass grid-wide scan (per-CTA counts ->
//     barrier -> offsets) writes class-split lists in ascending vertex order.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sx {

constexpr int BLOCK = 256;
constexpr int WARPS = BLOCK / 32;
constexpr int NCLS = 4;  // small, medium, large, huge
constexpr uint32_t INF = 0xFFFFFFFFu;
constexpr uint32_t FULL = 0xFFFFFFFFu;
constexpr int MAX_GRID = 4096;
constexpr int TILE_WORDS = BLOCK;  // ballot tile: one bitmap word per thread

enum : uint32_t { DIR_PUSH = 0, DIR_PULL = 1 };
enum : uint32_t { ERR_NONE = 0, ERR_BARRIER = 7 };

// ---------------------------------------------------------------- control block
// One 128-B line per contended group so that atomics on different groups do not
// share an L2 line.
struct alignas(128) CntLine {
    unsigned int cnt[NCLS];          // class-list fill counters (online filter)
    unsigned int found;              // |F'| (vertices activated this iteration)
    unsigned int pad0;
    unsigned long long mdeg;         // sum of degrees of activated vertices (m_f)
    unsigned long long edges;        // edges examined this iteration (trace)
    double dsum;                     // PageRank dangling mass accumulator
    unsigned int minv;               // min reduction scratch (SSSP far min, k-core min residual)
    unsigned int alive;              // k-core alive count
    unsigned int tile;               // dynamic work counter (chunks of tiles / tasks)
};

struct Ctl {
    alignas(128) unsigned int bar_count;
    alignas(128) unsigned int bar_gen;
    alignas(128) CntLine line[3];    // triple-buffered by iteration (it % 3)
    // --- state carried across launches (written by CTA 0 at exit, read at entry)
    alignas(128) unsigned int iter;  // iterations completed
    unsigned int dir;                // direction of the next launch
    unsigned int done;
    unsigned int error;
    unsigned int lists_ready;        // lists for iteration `iter` exist in the current direction's form
    unsigned int launch;             // launches so far
    unsigned int nf_prev;            // previous frontier size (Beamer growth test)
    unsigned int k;                  // k-core level
    unsigned long long m_u;          // BFS: edges incident to unvisited vertices
    unsigned long long hi;           // SSSP: current bucket upper bound (exclusive)
    unsigned int cur_count[NCLS];    // list sizes for iteration `iter`
    unsigned int ntrace;
    // --- run statistics per direction of the launch (0 push, 1 pull), one atomic per CTA per launch
    struct alignas(128) StatBlock {
        unsigned long long edges, entries, scanned, reached;
        unsigned int ballot, pull, iters;
    } st[2];
};

struct TraceRec {  // mirrors sx_trace_rec
    uint32_t iter, dir, filter, launch;
    uint32_t n_active[4];
    uint64_t n_frontier;
    uint64_t m_active;
    uint64_t aux;
    uint64_t t_ns;
};

// ---------------------------------------------------------------- graph view
struct DevGraph {
    uint64_t n, m;
    const uint64_t* __restrict__ rp;   // out rows
    const uint32_t* __restrict__ ci;
    const uint8_t* __restrict__ w8;    // weights (u8) or null
    const uint32_t* __restrict__ w32;  // weights (u32) or null
    const uint64_t* __restrict__ irp;  // in rows (== rp for symmetric graphs)
    const uint32_t* __restrict__ ici;
    const uint8_t* __restrict__ iw8;
    const uint32_t* __restrict__ iw32;
    const uint32_t* __restrict__ dout;  // out-degree
    const uint32_t* __restrict__ din;   // in-degree
    const uint32_t* __restrict__ nz_in; // bitmap: in-degree > 0
};

// Common per-launch parameters of every persistent kernel.
struct Sched {
    Ctl* ctl;
    uint32_t* lists[2];     // each: NCLS regions of n entries
    uint32_t* bm[3];        // frontier bitmaps, rotating by iteration
    uint32_t* cta_cnt;      // [NCLS][MAX_GRID] ballot scratch
    TraceRec* trace;        // device trace buffer or null
    uint32_t trace_cap;
    uint64_t nwords;        // words per bitmap (multiple of TILE_WORDS)
    uint32_t sep_small, sep_large, sep_huge;
    uint32_t online_cap;    // per class list
    float alpha, beta;
    int force_filter, force_dir, fusion;
    uint32_t max_iters;
};

// ---------------------------------------------------------------- small helpers
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ uint32_t warp_id() { return threadIdx.x >> 5; }
__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}
__device__ __forceinline__ uint64_t gtid() { return (uint64_t)blockIdx.x * BLOCK + threadIdx.x; }
__device__ __forceinline__ uint64_t gthreads() { return (uint64_t)gridDim.x * BLOCK; }
__device__ __forceinline__ uint64_t gwarp() { return (uint64_t)blockIdx.x * WARPS + warp_id(); }
__device__ __forceinline__ uint64_t gwarps() { return (uint64_t)gridDim.x * WARPS; }

__device__ __forceinline__ uint32_t ld_acquire(const unsigned int* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
template <class T> __device__ __forceinline__ T vload(const T* p) { return *(const volatile T*)p; }

__device__ __forceinline__ uint32_t cls_of(uint32_t deg, const Sched& s) {
    return deg < s.sep_small ? 0u : deg < s.sep_large ? 1u : deg < s.sep_huge ? 2u : 3u;
}

__device__ __forceinline__ uint32_t edge_w(const uint8_t* w8, const uint32_t* w32, uint64_t e) {
    return w8 ? (uint32_t)__ldg(w8 + e) : w32 ? __ldg(w32 + e) : 1u;
}

// ---------------------------------------------------------------- grid barrier
// Counter + generation barrier (no monitor CTA).  All CTAs are
// co-resident (cooperative launch), so it cannot deadlock.  Release
// on arrive, acquire on depart (gpu scope); the acquire fence also invalidates
// the SM's L1 so later plain loads see other SMs' writes.  A watchdog
// (globaltimer, 20 s) turns a broken barrier into SX_E_BARRIER instead of a hang.
__device__ __forceinline__ bool grid_sync(Ctl* c) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t gen = vload(&c->bar_gen);
        __threadfence();
        const uint32_t arrived = atomicAdd(&c->bar_count, 1u);
        if (arrived == gridDim.x - 1) {
            atomicExch(&c->bar_count, 0u);
            __threadfence();
            atomicAdd(&c->bar_gen, 1u);
        } else {
            uint32_t spins = 0;
            uint64_t t0 = 0;
            while (ld_acquire(&c->bar_gen) == gen) {
                if (((++spins) & 1023u) == 0) {
                    uint64_t t = globaltimer();
                    if (t0 == 0) t0 = t;
                    else if (t - t0 > 20000000000ull) { atomicExch(&c->error, ERR_BARRIER); break; }
                    if (vload(&c->error)) break;
                }
            }
        }
        __threadfence();
    }
    __syncthreads();
    return vload(&c->error) == 0;
}

// ---------------------------------------------------------------- block reductions
template <class T> __device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}
__device__ __forceinline__ uint32_t warp_min(uint32_t v) { return __reduce_min_sync(FULL, v); }

// Sum K values across the block; result valid in every thread.
template <int K, class T> __device__ __forceinline__ void block_sum(T (&v)[K]) {
    __shared__ T red[K][WARPS];
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = warp_sum(v[k]);
    __syncthreads();
    if (lane_id() == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) red[k][warp_id()] = v[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) {
        T s = 0;
#pragma unroll
        for (int w = 0; w < WARPS; ++w) s += red[k][w];
        v[k] = s;
    }
    __syncthreads();
}

__device__ __forceinline__ uint32_t block_min(uint32_t v) {
    __shared__ uint32_t red[WARPS];
    v = warp_min(v);
    __syncthreads();
    if (lane_id() == 0) red[warp_id()] = v;
    __syncthreads();
    uint32_t m = red[0];
#pragma unroll
    for (int w = 1; w < WARPS; ++w) m = min(m, red[w]);
    __syncthreads();
    return m;
}

// ---------------------------------------------------------------- online filter
// Record vertex u of class c into the next lists.  Warp-aggregated:
// lanes of the same class share one atomicAdd.  Entries beyond online_cap are
// not stored (overflow); the counter keeps counting so the JIT
// controller sees the overflow at the barrier.
__device__ __forceinline__ void online_record(CntLine* L, uint32_t* lists, uint64_t n, uint32_t cap, uint32_t u,
                                              uint32_t c) {
    const uint32_t active = __activemask();
    const uint32_t peers = __match_any_sync(active, c);
    const int leader = __ffs(peers) - 1;
    uint32_t base = 0;
    if ((int)lane_id() == leader) base = atomicAdd(&L->cnt[c], (uint32_t)__popc(peers));
    base = __shfl_sync(peers, base, leader);
    const uint32_t pos = base + __popc(peers & lanemask_lt());
    if (pos < cap) lists[(uint64_t)c * n + pos] = u;
}

// ---------------------------------------------------------------- ballot filter
// Word sources: word(wi) is called warp-collectively for wi = base + lane.
struct BitmapWords {  // frontier bitmap
    const uint32_t* bm;
    __device__ __forceinline__ uint32_t word(uint64_t wi) const { return bm[wi]; }
};
struct CandidateWords {  // BFS pull candidates: unvisited and in-degree > 0
    const uint32_t* visited;
    const uint32_t* nz;
    __device__ __forceinline__ uint32_t word(uint64_t wi) const { return ~visited[wi] & __ldg(nz + wi); }
};
struct AllWords {  // every vertex < n (pull-all algorithms: P:626, ballot in exactly iteration 1)
    uint64_t n;
    __device__ __forceinline__ uint32_t word(uint64_t wi) const {
        const uint64_t v0 = wi << 5;
        if (v0 + 32 <= n) return FULL;
        if (v0 >= n) return 0u;
        return (1u << (uint32_t)(n - v0)) - 1u;
    }
};
// Per-vertex predicate evaluated with a coalesced scan and __ballot_sync.
template <class Pred> struct BallotWords {
    Pred pred;
    uint64_t n;
    __device__ __forceinline__ uint32_t word(uint64_t wi) const {
        // warp-collective: lane l returns the word wi(lane l) = base + l
        const uint64_t base = wi - lane_id();
        uint32_t mine = 0;
#pragma unroll 4
        for (int j = 0; j < 32; ++j) {
            const uint64_t v = ((base + j) << 5) + lane_id();
            const bool p = v < n && pred(v);
            const uint32_t b = __ballot_sync(FULL, p);
            if ((int)lane_id() == j) mine = b;
        }
        return mine;
    }
};

struct BallotOut {
    uint32_t* lists;      // NCLS regions of n
    uint64_t n;
    const uint32_t* deg;  // degree used for classification
};

__device__ __forceinline__ void ballot_chunk(uint64_t nwords, uint64_t& w0, uint64_t& w1) {
    uint64_t per = (nwords + gridDim.x - 1) / gridDim.x;
    per = (per + TILE_WORDS - 1) / TILE_WORDS * TILE_WORDS;
    w0 = per * blockIdx.x;
    w1 = w0 + per;
    if (w0 > nwords) w0 = nwords;
    if (w1 > nwords) w1 = nwords;
}

// Pass 1: per-CTA class counts of set bits in its contiguous word range.
template <class Src>
__device__ void ballot_count(const Src& src, const Sched& s, const uint32_t* deg) {
    uint64_t w0, w1;
    ballot_chunk(s.nwords, w0, w1);
    uint32_t acc[NCLS] = {0, 0, 0, 0};
    for (uint64_t t = w0; t < w1; t += TILE_WORDS) {
        uint32_t w = src.word(t + threadIdx.x);
        const uint64_t vb = (t + threadIdx.x) << 5;
        while (w) {
            const int b = __ffs(w) - 1;
            w &= w - 1;
            acc[cls_of(__ldg(deg + vb + b), s)]++;
        }
    }
    block_sum<NCLS>(acc);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int c = 0; c < NCLS; ++c) s.cta_cnt[c * MAX_GRID + blockIdx.x] = acc[c];
    }
}

// Block-wide exclusive scan of 4 small counts packed in 16-bit fields.
__device__ __forceinline__ uint64_t block_excl_scan_packed(uint64_t x, uint64_t& total) {
    __shared__ uint64_t wsum[WARPS];
    uint64_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(FULL, inc, o);
        if ((int)lane_id() >= o) inc += y;
    }
    __syncthreads();
    if (lane_id() == 31) wsum[warp_id()] = inc;
    __syncthreads();
    uint64_t before = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
        const uint64_t v = wsum[w];
        if (w < (int)warp_id()) before += v;
        tot += v;
    }
    total = tot;
    return before + inc - x;
}

// Pass 2: offsets from the per-CTA counts, then write the class lists in
// ascending vertex order (sorted + unique).  `on_vertex(v, c)` is
// called for every emitted vertex (used to update metadata during the scan).
// Returns the class totals (identical in every CTA).
template <class Src, class OnV>
__device__ void ballot_write(const Src& src, const Sched& s, const BallotOut& out, uint32_t (&tot)[NCLS],
                             OnV on_vertex) {
    uint64_t w0, w1;
    ballot_chunk(s.nwords, w0, w1);
    uint32_t red[2 * NCLS] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (uint32_t b = threadIdx.x; b < gridDim.x; b += BLOCK) {
#pragma unroll
        for (int c = 0; c < NCLS; ++c) {
            const uint32_t v = vload(s.cta_cnt + c * MAX_GRID + b);
            red[NCLS + c] += v;
            if (b < blockIdx.x) red[c] += v;
        }
    }
    block_sum<2 * NCLS>(red);
    uint32_t run[NCLS];
#pragma unroll
    for (int c = 0; c < NCLS; ++c) {
        run[c] = red[c];
        tot[c] = red[NCLS + c];
    }
    for (uint64_t t = w0; t < w1; t += TILE_WORDS) {
        const uint32_t w = src.word(t + threadIdx.x);
        const uint64_t vb = (t + threadIdx.x) << 5;
        uint64_t packed = 0;
        uint32_t ww = w;
        while (ww) {
            const int b = __ffs(ww) - 1;
            ww &= ww - 1;
            packed += 1ull << (16 * cls_of(__ldg(out.deg + vb + b), s));
        }
        uint64_t tile_tot;
        const uint64_t ex = block_excl_scan_packed(packed, tile_tot);
        uint32_t pos[NCLS];
#pragma unroll
        for (int c = 0; c < NCLS; ++c) pos[c] = run[c] + (uint32_t)((ex >> (16 * c)) & 0xFFFF);
        ww = w;
        while (ww) {
            const int b = __ffs(ww) - 1;
            ww &= ww - 1;
            const uint32_t v = (uint32_t)(vb + b);
            const uint32_t c = cls_of(__ldg(out.deg + v), s);
            out.lists[(uint64_t)c * out.n + pos[c]++] = v;
            on_vertex(v, c);
        }
#pragma unroll
        for (int c = 0; c < NCLS; ++c) run[c] += (uint32_t)((tile_tot >> (16 * c)) & 0xFFFF);
    }
}

struct NoOp {
    __device__ __forceinline__ void operator()(uint32_t, uint32_t) const {}
};

// Full ballot filter: count -> barrier -> write.  Ends WITHOUT a trailing
// barrier; callers barrier before consuming the lists.
template <class Src, class OnV = NoOp>
__device__ bool ballot_filter(const Src& src, const Sched& s, const BallotOut& out, uint32_t (&tot)[NCLS],
                              OnV on_vertex = OnV()) {
    ballot_count(src, s, out.deg);
    if (!grid_sync(s.ctl)) return false;
    ballot_write(src, s, out, tot, on_vertex);
    return true;
}

// Dense clear of a bitmap with 128-bit stores, grid-strided.
__device__ __forceinline__ void clear_bitmap(uint32_t* bm, uint64_t nwords) {
    uint4* p = reinterpret_cast<uint4*>(bm);
    const uint64_t n4 = nwords / 4;
    for (uint64_t i = gtid(); i < n4; i += gthreads()) p[i] = make_uint4(0, 0, 0, 0);
}

__device__ __forceinline__ bool bm_test(const uint32_t* bm, uint32_t v) { return (bm[v >> 5] >> (v & 31)) & 1u; }
__device__ __forceinline__ bool bm_claim(uint32_t* bm, uint32_t v) {
    const uint32_t bit = 1u << (v & 31);
    return !(atomicOr(bm + (v >> 5), bit) & bit);
}
__device__ __forceinline__ void bm_set(uint32_t* bm, uint32_t v) { atomicOr(bm + (v >> 5), 1u << (v & 31)); }

// ---------------------------------------------------------------- edge loops
// Visit edges [beg, end) of one vertex with `size` cooperating workers, this
// worker being `rank`.  The aligned body uses 128-bit loads of 4 neighbour ids
// per worker (coalesced across the warp); head/tail are scalar.
template <class Fn>
__device__ __forceinline__ void for_edges(const uint32_t* __restrict__ col, uint64_t beg, uint64_t end, uint64_t rank,
                                          uint64_t size, Fn&& fn) {
    uint64_t a = (beg + 3) & ~3ull;
    if (a > end) a = end;
    for (uint64_t e = beg + rank; e < a; e += size) fn(e, __ldg(col + e));
    const uint64_t nvec = (end - a) >> 2;
    const uint4* c4 = reinterpret_cast<const uint4*>(col + a);
    for (uint64_t i = rank; i < nvec; i += size) {
        const uint4 q = __ldg(c4 + i);
        const uint64_t e = a + 4 * i;
        fn(e, q.x);
        fn(e + 1, q.y);
        fn(e + 2, q.z);
        fn(e + 3, q.w);
    }
    for (uint64_t e = a + 4 * nvec + rank; e < end; e += size) fn(e, __ldg(col + e));
}

// Visit the four class lists with thread / warp / CTA / grid granularity.
// The functor gets (v, rank, size) and loops over v's edges itself.  Huge
// vertices (grid-split, B200 addition) go first so the whole GPU shares them,
// small ones last so they fill the tail.
template <class VFn>
__device__ __forceinline__ void for_tasks(const uint32_t* lists, uint64_t n, const uint32_t (&cnt)[NCLS], VFn&& vf) {
    for (uint32_t i = 0; i < cnt[3]; ++i) vf(lists[3 * n + i], gtid(), gthreads(), 3u);
    for (uint32_t i = blockIdx.x; i < cnt[2]; i += gridDim.x) vf(lists[2 * n + i], (uint64_t)threadIdx.x, (uint64_t)BLOCK, 2u);
    for (uint64_t i = gwarp(); i < cnt[1]; i += gwarps()) vf(lists[n + i], (uint64_t)lane_id(), 32ull, 1u);
    for (uint64_t i = gtid(); i < cnt[0]; i += gthreads()) vf(lists[i], 0ull, 1ull, 0u);
}

// ---------------------------------------------------------------- bookkeeping
struct Stats {
    uint64_t edges = 0, entries = 0, scanned = 0, reached = 0;
    uint32_t ballot = 0, pull = 0, iters = 0;
};

// Per-CTA partial counters -> one atomic per CTA; uniform counters from CTA 0.
__device__ __forceinline__ void flush_stats(Ctl* c, Stats& st, uint32_t dir) {
    uint64_t v[3] = {st.edges, st.entries, st.reached};
    block_sum<3>(v);
    if (threadIdx.x == 0) {
        Ctl::StatBlock& b = c->st[dir];
        if (v[0]) atomicAdd(&b.edges, (unsigned long long)v[0]);
        if (v[1]) atomicAdd(&b.entries, (unsigned long long)v[1]);
        if (v[2]) atomicAdd(&b.reached, (unsigned long long)v[2]);
        if (blockIdx.x == 0) {
            b.scanned += st.scanned;
            b.ballot += st.ballot;
            b.pull += st.pull;
            b.iters += st.iters;
        }
    }
}

__device__ __forceinline__ void reset_line(CntLine* L) {
#pragma unroll
    for (int c = 0; c < NCLS; ++c) L->cnt[c] = 0;
    L->found = 0;
    L->mdeg = 0;
    L->edges = 0;
    L->dsum = 0.0;
    L->minv = INF;
    L->alive = 0;
    L->tile = 0;
}

__device__ __forceinline__ bool lead() { return blockIdx.x == 0 && threadIdx.x == 0; }

__device__ __forceinline__ void trace_put(const Sched& s, uint32_t iter, uint32_t dir, uint32_t filter,
                                          const uint32_t (&cnt)[NCLS], uint64_t nf, uint64_t mf, uint64_t aux) {
    if (s.trace && lead()) {
        const uint32_t i = s.ctl->ntrace++;
        if (i < s.trace_cap) {
            TraceRec r;
            r.iter = iter;
            r.dir = dir;
            r.filter = filter;
            r.launch = s.ctl->launch;
#pragma unroll
            for (int c = 0; c < NCLS; ++c) r.n_active[c] = cnt[c];
            r.n_frontier = nf;
            r.m_active = mf;
            r.aux = aux;
            r.t_ns = globaltimer();
            s.trace[i] = r;
        }
    }
}

__device__ __forceinline__ uint32_t sum4(const uint32_t (&c)[NCLS]) { return c[0] + c[1] + c[2] + c[3]; }

}  // namespace sx

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
// B200 design notes (DESIGN.md has the full rationale):
//   * Same-address atomics serialise in L2 (~4.5 ns each, measured): every
//     per-iteration counter is therefore spread over NSLOT = 32 "slots" (one
//     128-B line each), CTA b writing slot b % 32, readers summing the 32 slots
//     with one warp-wide load.
//   * The paper's thread-private bins become 32 slot regions per class
//     list: a warp claims positions with one atomicAdd per class on its slot's
//     counter (warp-aggregated with __match_any_sync), so a bin is a (slot,
//     class) region.  Overflow = a region exceeding overflow_threshold x (warps
//     of the GPU) / 32 entries; recording then only counts (the shadow filter of
//     P:654) and the ballot filter rebuilds the lists.  Exactly-once claims
//     (atomicOr on a bitmap, an atomic crossing test) keep online lists unique.
//   * The ballot filter scans a frontier BITMAP (one u32 word = 32 vertices, so a
//     lane's word already is the warp ballot of P:555) or evaluates a per-vertex
//     predicate with __ballot_sync; a two-pass grid-wide scan (per-CTA counts ->
//     barrier -> offsets) writes class-split lists in ascending vertex order.
#pragma once
#include <cstddef>
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
constexpr int NSLOT = 32;          // counter slots (L2 lines) per iteration line
constexpr int BAR_GROUPS = 32;     // two-level barrier: <= 32 groups of CTAs

enum : uint32_t { DIR_PUSH = 0, DIR_PULL = 1, DIR_CLUSTER = 2 };
constexpr int MPV = 8;          // frontier pulls (SSSP / WCC): in-edges per lane of a warp tile
constexpr int MPT = 32 * MPV;   // in-edges per warp tile
constexpr int CL_CTAS = 16;      // CTAs of the small-frontier cluster kernel (non-portable size 16)
constexpr uint32_t CL_BIG = 64;  // cluster mode: out-degree above which a task's edges are split cluster-wide
constexpr int CL_BLOCK = 1024;   // threads per CTA of the cluster kernel
enum : uint32_t { ERR_NONE = 0, ERR_BARRIER = 7 };

// ---------------------------------------------------------------- control block
struct alignas(128) Slot {
    unsigned int cnt[NCLS];          // online-filter fill counters of this slot's list regions
    unsigned int found;              // |F'| contributions
    unsigned int minv;               // min reduction scratch (SSSP far min, k-core min residual)
    unsigned int alive;              // k-core alive count
    unsigned int tile;               // dynamic work counter of this slot's chunk range
    unsigned long long mdeg;         // sum of degrees of activated vertices (m_f)
    unsigned long long edges;        // edges examined (trace)
    double dsum;                     // PageRank dangling mass
    double dsum2;                    // convergence tests: L1 change of the iteration
};
struct IterLine {
    Slot s[NSLOT];
};
struct alignas(128) BarLine {
    unsigned int count;
};

struct Ctl {
    // grid barrier state, double-buffered by launch parity (the other half is
    // zeroed by the exiting kernel, so each launch starts from zero counters)
    BarLine bar_grp[2][BAR_GROUPS];  // per-group monotonic arrival counters
    BarLine bar_top[2];              // monotonic count of completed group arrivals
    IterLine line[3];                // per-iteration counters, triple-buffered (it % 3)
    // --- state carried across launches (written by CTA 0 at exit, read at entry)
    alignas(128) unsigned int iter;  // iterations completed
    unsigned int dir;                // direction of the next launch
    unsigned int done;
    unsigned int error;
    unsigned int lists_ready;        // lists for iteration `iter` exist in the current direction's form
    unsigned int slotted;            // ... as slotted online lists (counts in line[iter % 3]) or contiguous
    unsigned int launch;             // launches so far
    unsigned int nf_prev;            // previous frontier size (Beamer growth test)
    unsigned int k;                  // k-core level
    unsigned long long m_u;          // BFS: edges incident to unvisited vertices
    unsigned long long hi;           // SSSP: current bucket upper bound (exclusive)
    unsigned int cur_count[NCLS];    // contiguous list sizes for iteration `iter`
    unsigned int ntrace;
    // --- small-frontier cluster mode: list counts by iteration (it % 3) and a min scratch
    struct alignas(128) ClusterLine {
        unsigned int cnt[3];
        unsigned int minv;
        unsigned int nbig[3];  // tasks of degree > CL_BIG deferred to the cluster-wide edge loop
        unsigned int ready;    // BFS: the pull kernel left the frontier as a contiguous list (cnt[iter % 3])
        unsigned long long mf[3];  // BFS: sum of out-degrees of the next frontier
        unsigned int fmin[2];      // SSSP: far-pile minimum, kept incrementally (two slots by advance parity)
    } cl;
    // --- run statistics per direction of the launch (0 push, 1 pull), one atomic per CTA per launch
    struct alignas(128) StatBlock {
        unsigned long long edges, entries, scanned, reached;
        unsigned int ballot, pull, iters;
    } st[2];
    // --- asynchronous work queue (k-core cascades): low 32 bits = queue tail
    // (positions handed to producers), high 32 bits = pending items (enqueued,
    // not yet fully processed); head = next ticket for the consumers
    alignas(128) unsigned long long aq_tp;
    alignas(128) unsigned long long aq_head;
};

// Statistics of the runs enqueued without a host sync (sx_bfs_async): the
// fused kernel's CTA 0 adds each run's stat blocks here at its end; the host
// reads and zeroes them at sx_graph_sync.
struct AsyncAcc {
    Ctl::StatBlock st[2];
    unsigned int runs, errors;
};

// The run state carried across launches (Ctl from `iter` to `ntrace`), as one
// CTA sees it: run_state() reads the 128-B line once per CTA (warp 0, lane l
// word l) instead of every thread loading each field from the same L2 line.
struct RunState {
    uint32_t iter, dir, done, error, lists_ready, slotted, launch, nf_prev, k;
    uint64_t m_u, hi;
    uint32_t cur_count[NCLS];
    uint32_t ntrace;
};
static_assert(offsetof(Ctl, m_u) - offsetof(Ctl, iter) == offsetof(RunState, m_u), "RunState layout");
static_assert(offsetof(Ctl, hi) - offsetof(Ctl, iter) == offsetof(RunState, hi), "RunState layout");
static_assert(offsetof(Ctl, cur_count) - offsetof(Ctl, iter) == offsetof(RunState, cur_count), "RunState layout");
static_assert(offsetof(Ctl, ntrace) - offsetof(Ctl, iter) == offsetof(RunState, ntrace), "RunState layout");
static_assert(sizeof(RunState) <= 128 && offsetof(Ctl, cl) - offsetof(Ctl, iter) >= 128, "RunState fits one line");

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
    uint32_t* lists[2];     // each: NCLS class regions of cstride entries
    uint32_t* bm[3];        // frontier bitmaps, rotating by iteration
    uint32_t* cta_cnt;      // [NCLS][MAX_GRID] ballot scratch
    TraceRec* trace;        // device trace buffer or null
    uint32_t trace_cap;
    uint64_t nwords;        // words per bitmap (multiple of TILE_WORDS)
    uint64_t cstride;       // class region stride = NSLOT * R >= n
    uint32_t R;             // slot region size
    uint32_t cap_s;         // online capacity of one (slot, class) region
    uint32_t sep_small, sep_large, sep_huge;
    float alpha, beta;
    int force_filter, force_dir, fusion;
    uint32_t max_iters;
    uint32_t local_chain;   // SSSP / k-core: vertices a thread may process in a row within one iteration
    uint32_t cluster_enter; // SSSP: frontier size at or below which one thread-block cluster continues
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
__device__ __forceinline__ uint32_t my_slot() { return blockIdx.x % NSLOT; }
__device__ __forceinline__ bool lead() { return blockIdx.x == 0 && threadIdx.x == 0; }

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

// ---------------------------------------------------------------- TMA bulk copies (sm_100a)
// 1D bulk copy global -> shared (cp.async.bulk, the TMA unit) completing on an
// mbarrier with a transaction count: one thread issues it, the data land
// without registers or load instructions, and the consumer waits on the
// barrier's phase.  Used to stage contiguous slices (BFS pull: the hub-probe
// table of the next chunk) while the current one is processed.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// arm the barrier for `bytes` and issue the copy (bytes: multiple of 16, 16-B aligned addresses)
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// 1D bulk copy shared -> global (bulk-group completion); wait = the writes are done
__device__ __forceinline__ void tma_store_1d(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok = 0;
    do {
        asm volatile("{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n\tselp.u32 %0, 1, 0, q;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    } while (!ok);
}

// ---------------------------------------------------------------- grid barrier
// Two-level monotonic-counter barrier (no monitor CTA).  All
// CTAs are co-resident (cooperative launch), so it cannot deadlock.
// CTA b arrives on group counter b % G (G <= 32, one L2 line each); the last
// arriver of a group arrives on the top counter; the k-th barrier of a launch
// completes when the top counter reaches (k+1) G.  (A flat counter serialises
// ~1200 same-address atomics: 5.3 us measured on B200.)  fence.acq_rel.gpu
// before arriving (release) and after the poll (acquire; it also invalidates
// the SM's L1, so later plain loads see other SMs' writes).  A watchdog
// (globaltimer, 20 s) turns a broken barrier into SX_E_BARRIER.
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// The launch parity selecting the barrier half, read once at kernel entry.
__device__ __forceinline__ uint32_t& bar_parity() {
    __shared__ uint32_t s_parity;
    return s_parity;
}
__device__ __forceinline__ void grid_begin(Ctl* c) {
    if (threadIdx.x == 0) bar_parity() = vload(&c->launch) & 1u;
    __syncthreads();
}
__device__ __forceinline__ void grid_begin(uint32_t launch) {
    if (threadIdx.x == 0) bar_parity() = launch & 1u;
    __syncthreads();
}
__device__ __forceinline__ const RunState& run_state(const Ctl* c) {
    __shared__ alignas(16) uint32_t w[32];
    __syncthreads();
    if (threadIdx.x < 32) w[threadIdx.x] = vload(reinterpret_cast<const uint32_t*>(&c->iter) + threadIdx.x);
    __syncthreads();
    return *reinterpret_cast<const RunState*>(w);
}
// Called by CTA 0 thread 0 when the kernel exits: zero the other half for the next launch.
__device__ __forceinline__ void grid_end(Ctl* c) {
    const uint32_t q = bar_parity() ^ 1u;
    for (int i = 0; i < BAR_GROUPS; ++i) c->bar_grp[q][i].count = 0;
    c->bar_top[q].count = 0;
}

// Barrier watchdog in ns (20 s); sx_barrier_fault lowers it for its test and restores it.
static __device__ unsigned long long g_watchdog_ns = 20000000000ull;

__device__ __forceinline__ bool grid_sync(Ctl* c) {
    __shared__ uint32_t s_err;
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t q = bar_parity();
        const uint32_t G = gridDim.x < (uint32_t)BAR_GROUPS ? gridDim.x : (uint32_t)BAR_GROUPS;
        const uint32_t grp = blockIdx.x % G;
        const uint32_t gsize = (gridDim.x - grp + G - 1) / G;  // CTAs b with b % G == grp
        fence_acq_rel_gpu();
        uint32_t err = 0;
        const uint32_t old = atomicAdd(&c->bar_grp[q][grp].count, 1u);
        const uint32_t k = old / gsize;
        if (old - k * gsize == gsize - 1) {
            fence_acq_rel_gpu();  // acquire the group's arrivals, release them with ours
            atomicAdd(&c->bar_top[q].count, 1u);
        }
        const uint32_t target = (k + 1) * G;
        uint32_t spins = 0;
        uint64_t t0 = 0;
        while ((int32_t)(ld_acquire(&c->bar_top[q].count) - target) < 0) {
            if (((++spins) & 1023u) == 0) {
                const uint64_t t = globaltimer();
                if (t0 == 0) t0 = t;
                else if (t - t0 > g_watchdog_ns) atomicExch(&c->error, ERR_BARRIER);
                if (vload(&c->error)) break;
            }
        }
        fence_acq_rel_gpu();
        if (spins >= 1023u) err = vload(&c->error);
        s_err = err;
    }
    __syncthreads();
    return s_err == 0;
}

// ---------------------------------------------------------------- reductions
template <class T> __device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}
__device__ __forceinline__ uint32_t warp_min(uint32_t v) { return __reduce_min_sync(FULL, v); }
__device__ __forceinline__ uint32_t warp_max(uint32_t v) { return __reduce_max_sync(FULL, v); }

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

// ---------------------------------------------------------------- iteration lines
// Zero an iteration line.  Warp-collective: call from warp 0 of CTA 0 only.
__device__ __forceinline__ void reset_line_warp(IterLine* L) {
    Slot& s = L->s[lane_id()];
#pragma unroll
    for (int c = 0; c < NCLS; ++c) s.cnt[c] = 0;
    s.found = 0;
    s.minv = INF;
    s.alive = 0;
    s.tile = 0;
    s.mdeg = 0;
    s.edges = 0;
    s.dsum = 0.0;
    s.dsum2 = 0.0;
}
__device__ __forceinline__ void maybe_reset_line(IterLine* L) {
    if (blockIdx.x == 0 && warp_id() == 0) reset_line_warp(L);
}

// Sum of one iteration line over its slots, computed by warp 0 and shared.
// One slot's counters in four 128-bit volatile loads (one L2 request each
// instead of one per field: every CTA of the grid reads every slot).
__device__ __forceinline__ uint4 vload4(const void* p) {
    uint4 r;
    asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
struct SlotSnap {
    uint32_t cnt[NCLS];
    uint32_t found, minv, alive;
    uint64_t mdeg, edges;
    double dsum, dsum2;
};
__device__ __forceinline__ SlotSnap load_slot(const Slot& sl) {
    static_assert(offsetof(Slot, found) == 16 && offsetof(Slot, mdeg) == 32 && offsetof(Slot, dsum) == 48, "Slot layout");
    const char* b = reinterpret_cast<const char*>(&sl);
    const uint4 a = vload4(b), q = vload4(b + 16), m = vload4(b + 32), d = vload4(b + 48);
    SlotSnap r;
    r.cnt[0] = a.x;
    r.cnt[1] = a.y;
    r.cnt[2] = a.z;
    r.cnt[3] = a.w;
    r.found = q.x;
    r.minv = q.y;
    r.alive = q.z;
    r.mdeg = ((uint64_t)m.y << 32) | m.x;
    r.edges = ((uint64_t)m.w << 32) | m.z;
    r.dsum = __hiloint2double((int)d.y, (int)d.x);
    r.dsum2 = __hiloint2double((int)d.w, (int)d.z);
    return r;
}
__device__ __forceinline__ SlotSnap load_slot_cnt(const Slot& sl) {
    const uint4 a = vload4(&sl);
    SlotSnap r{};
    r.cnt[0] = a.x;
    r.cnt[1] = a.y;
    r.cnt[2] = a.z;
    r.cnt[3] = a.w;
    return r;
}

struct LineSum {
    uint32_t cnt[NCLS];
    uint32_t cntmax[NCLS];
    uint32_t found, minv, alive;
    uint64_t mdeg, edges;
    double dsum, dsum2;
};
__device__ __forceinline__ void read_line(const IterLine* L, LineSum& out) {
    __shared__ LineSum sh;
    __syncthreads();
    if (warp_id() == 0) {
        const SlotSnap x = load_slot(L->s[lane_id()]);
        LineSum r;
#pragma unroll
        for (int c = 0; c < NCLS; ++c) {
            r.cnt[c] = warp_sum(x.cnt[c]);
            r.cntmax[c] = warp_max(x.cnt[c]);
        }
        r.found = warp_sum(x.found);
        r.minv = warp_min(x.minv);
        r.alive = warp_sum(x.alive);
        r.mdeg = warp_sum(x.mdeg);
        r.edges = warp_sum(x.edges);
        r.dsum = warp_sum(x.dsum);
        r.dsum2 = warp_sum(x.dsum2);
        if (lane_id() == 0) sh = r;
    }
    __syncthreads();
    out = sh;
}

// ---------------------------------------------------------------- task views
struct TaskView;
__device__ __forceinline__ TaskView& task_view();
// How the current iteration's class lists are laid out: per class, NSLOT
// segments (online, slotted) or one contiguous segment (ballot output).
struct TaskView {
    uint32_t pre[NCLS][NSLOT + 1];  // exclusive prefix of segment sizes
    uint32_t base[NCLS][NSLOT];     // segment offsets inside the class region
};
__device__ __forceinline__ TaskView& task_view() {
    __shared__ TaskView tv;
    return tv;
}
// contiguous lists of tot[c] entries (all threads call; ends with __syncthreads)
__device__ __forceinline__ void view_contig(const uint32_t (&tot)[NCLS]) {
    TaskView& tv = task_view();
    __syncthreads();
    if (warp_id() == 0) {
        const uint32_t l = lane_id();
#pragma unroll
        for (int c = 0; c < NCLS; ++c) {
            tv.pre[c][l] = l == 0 ? 0u : tot[c];
            tv.base[c][l] = 0;
            if (l == 0) tv.pre[c][NSLOT] = tot[c];
        }
    }
    __syncthreads();
}
// slotted online lists whose sizes are the line's slot counters (capped)
__device__ __forceinline__ void view_slots(const IterLine* L, const Sched& s, uint32_t (&tot)[NCLS]) {
    TaskView& tv = task_view();
    __shared__ uint32_t sh_tot[NCLS];
    __syncthreads();
    if (warp_id() == 0) {
        const uint32_t l = lane_id();
        const SlotSnap sn = load_slot_cnt(L->s[l]);
#pragma unroll
        for (int c = 0; c < NCLS; ++c) {
            const uint32_t x = min(sn.cnt[c], s.cap_s);
            uint32_t inc = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(FULL, inc, o);
                if ((int)l >= o) inc += y;
            }
            tv.pre[c][l] = inc - x;
            tv.base[c][l] = l * s.R;
            if (l == 31) {
                tv.pre[c][NSLOT] = inc;
                sh_tot[c] = inc;
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < NCLS; ++c) tot[c] = sh_tot[c];
}
// read_line + view_slots in one warp-wide pass over the slots (one L2 round
// trip after the barrier instead of two).  vcnt receives the view's class sizes.
__device__ __forceinline__ void read_line_view(const IterLine* L, const Sched& s, LineSum& out, uint32_t (&vcnt)[NCLS]) {
    __shared__ LineSum sh;
    __shared__ uint32_t sh_tot[NCLS];
    TaskView& tv = task_view();
    __syncthreads();
    if (warp_id() == 0) {
        const uint32_t l = lane_id();
        const SlotSnap sn = load_slot(L->s[l]);
        uint32_t x[NCLS];
#pragma unroll
        for (int c = 0; c < NCLS; ++c) x[c] = sn.cnt[c];
        const uint32_t found = sn.found, minv = sn.minv, alive = sn.alive;
        const uint64_t mdeg = sn.mdeg, edges = sn.edges;
        const double dsum = sn.dsum;
        LineSum r;
#pragma unroll
        for (int c = 0; c < NCLS; ++c) {
            r.cnt[c] = warp_sum(x[c]);
            r.cntmax[c] = warp_max(x[c]);
            const uint32_t xc = min(x[c], s.cap_s);
            uint32_t inc = xc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(FULL, inc, o);
                if ((int)l >= o) inc += y;
            }
            tv.pre[c][l] = inc - xc;
            tv.base[c][l] = l * s.R;
            if (l == 31) {
                tv.pre[c][NSLOT] = inc;
                sh_tot[c] = inc;
            }
        }
        r.found = warp_sum(found);
        r.minv = warp_min(minv);
        r.alive = warp_sum(alive);
        r.mdeg = warp_sum(mdeg);
        r.edges = warp_sum(edges);
        r.dsum = warp_sum(dsum);
        r.dsum2 = warp_sum(sn.dsum2);
        if (l == 0) sh = r;
    }
    __syncthreads();
    out = sh;
#pragma unroll
    for (int c = 0; c < NCLS; ++c) vcnt[c] = sh_tot[c];
}

// the i-th task of class c under the current view
__device__ __forceinline__ uint32_t task_at(const uint32_t* lists, const Sched& s, uint32_t c, uint32_t i) {
    const TaskView& tv = task_view();
    int lo = 0, hi = NSLOT;  // largest lo with pre[lo] <= i
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const int mid = (lo + hi) >> 1;
        if (tv.pre[c][mid] <= i) lo = mid;
        else hi = mid;
    }
    return lists[(uint64_t)c * s.cstride + tv.base[c][lo] + (i - tv.pre[c][lo])];
}

// ---------------------------------------------------------------- online filter
// Record vertex u of class c into the next lists: region (slot of
// this CTA, class c).  Two levels, both warp-aggregated (lanes of the same
// class share one atomic via __match_any_sync):
//   * a CTA stage in shared memory (STAGE entries per class; a shared-memory
//     atomic, no L2 round trip on the compute path), appended to the slot
//     region by stage_flush() before the iteration's barrier — one global
//     atomic per class per CTA;
//   * entries beyond the stage go straight to the slot region (global atomic).
// Region entries beyond cap_s are not stored (overflow); the
// counter keeps counting, so the JIT controller sees the overflow at the barrier.
constexpr uint32_t STAGE = 512;
struct Stage {
    uint32_t cnt[NCLS];
    uint32_t e[NCLS][STAGE];
};
__device__ __forceinline__ Stage& stage() {
    __shared__ Stage st;
    return st;
}
// Kernel entry, before the first record (a __syncthreads must follow: grid_begin has one).
__device__ __forceinline__ void stage_init() {
    if (threadIdx.x < NCLS) stage().cnt[threadIdx.x] = 0;
}
__device__ __forceinline__ void online_record_global(IterLine* L, uint32_t* lists, const Sched& s, uint32_t u,
                                                     uint32_t c) {
    const uint32_t slot = my_slot();
    const uint32_t active = __activemask();
    const uint32_t peers = __match_any_sync(active, c);
    const int leader = __ffs(peers) - 1;
    uint32_t base = 0;
    if ((int)lane_id() == leader) base = atomicAdd(&L->s[slot].cnt[c], (uint32_t)__popc(peers));
    base = __shfl_sync(peers, base, leader);
    const uint32_t pos = base + __popc(peers & lanemask_lt());
    if (pos < s.cap_s) lists[(uint64_t)c * s.cstride + (uint64_t)slot * s.R + pos] = u;
}
__device__ __forceinline__ void online_record(IterLine* L, uint32_t* lists, const Sched& s, uint32_t u, uint32_t c) {
    Stage& st = stage();
    const uint32_t active = __activemask();
    const uint32_t peers = __match_any_sync(active, c);
    const int leader = __ffs(peers) - 1;
    uint32_t base = 0;
    if ((int)lane_id() == leader) base = atomicAdd(&st.cnt[c], (uint32_t)__popc(peers));
    base = __shfl_sync(peers, base, leader);
    const uint32_t pos = base + __popc(peers & lanemask_lt());
    if (pos < STAGE) st.e[c][pos] = u;
    else online_record_global(L, lists, s, u, c);
}
// All threads, after the iteration's records and before its barrier: append
// the CTA stage to this CTA's slot regions (warp c copies class c).
__device__ __forceinline__ void stage_flush(IterLine* L, uint32_t* lists, const Sched& s) {
    Stage& st = stage();
    __syncthreads();
    const uint32_t c = warp_id();
    if (c < NCLS) {
        const uint32_t n = min(st.cnt[c], STAGE);
        if (n) {
            const uint32_t slot = my_slot();
            uint32_t base = 0;
            if (lane_id() == 0) base = atomicAdd(&L->s[slot].cnt[c], n);
            base = __shfl_sync(FULL, base, 0);
            uint32_t* dst = lists + (uint64_t)c * s.cstride + (uint64_t)slot * s.R;
            for (uint32_t j = lane_id(); j < n; j += 32)
                if (base + j < s.cap_s) dst[base + j] = st.e[c][j];
        }
    }
    __syncthreads();
    if (threadIdx.x < NCLS) st.cnt[threadIdx.x] = 0;
}

// One CTA-level total added to this CTA's slot (thread 0 after a block_sum).
template <class T> __device__ __forceinline__ void slot_add(T* field_of_slot0, T v) {
    // field_of_slot0 points at the field inside slot 0; slots are sizeof(Slot) apart
    T* p = (T*)((char*)field_of_slot0 + (size_t)my_slot() * sizeof(Slot));
    if (v) atomicAdd(p, v);
}

// Dynamic work distribution (warp-collective; every lane gets the same chunk):
// chunks [0, nchunks) split into NSLOT ranges, range s counted by slot s's
// `tile` counter.  A warp takes chunks from its current range (one atomicAdd by
// lane 0); once that range is exhausted the warp reads all NSLOT counters at
// once (lane l loads slot l: one round trip) and moves to a range with work
// left — the first such range after a per-warp rotation, so the thieves spread
// over the ranges instead of queueing on one counter.  Returns INF only when
// every range is exhausted (no warp leaves while another still has work).
#ifndef SX_STEAL_MAX
#define SX_STEAL_MAX 1000000  // range moves per warp and level (round 1 stopped after 3)
#endif
__device__ __forceinline__ uint32_t grab_chunk(IterLine* L, uint32_t nchunks, uint32_t& s_cur) {
    const uint32_t per = (nchunks + NSLOT - 1) / NSLOT;
    const uint32_t lane = lane_id();
    for (uint32_t moves = 0;; ++moves) {
        uint32_t ch = INF;
        if (lane == 0 && vload(&L->s[s_cur].tile) < per) {
            const uint32_t k = atomicAdd(&L->s[s_cur].tile, 1u);
            if (k < per && s_cur * per + k < nchunks) ch = s_cur * per + k;
        }
        ch = __shfl_sync(FULL, ch, 0);
        if (ch != INF || moves >= SX_STEAL_MAX) return ch;
        const uint32_t lo = lane * per;
        const uint32_t size = lo < nchunks ? min(per, nchunks - lo) : 0u;
        const uint32_t left = __ballot_sync(FULL, vload(&L->s[lane].tile) < size);
        if (!left) return INF;
        const uint32_t rot = (uint32_t)(gwarp() * 7u) & 31u;
        const uint32_t r = (left >> rot) | (rot ? left << (32u - rot) : 0u);  // rotate right by rot
        s_cur = ((uint32_t)(__ffs(r) - 1) + rot) & 31u;
    }
}

// The same distribution with the next chunk's claim in flight while the
// current one is processed: grab_issue sends lane 0's atomicAdd on the current
// range and returns the raw ticket WITHOUT consuming it (the warp does not stall
// on the atomic's round trip); grab_finish turns it into a chunk once the
// current chunk is done, falling back to grab_chunk (the steal path) when the
// range is exhausted.
__device__ __forceinline__ uint32_t grab_issue(IterLine* L, uint32_t s_cur) {
    return lane_id() == 0 ? atomicAdd(&L->s[s_cur].tile, 1u) : 0u;
}
__device__ __forceinline__ uint32_t grab_finish(IterLine* L, uint32_t nchunks, uint32_t& s_cur, uint32_t raw,
                                                uint32_t s_issued) {
    const uint32_t per = (nchunks + NSLOT - 1) / NSLOT;
    uint32_t ch = INF;
    if (lane_id() == 0 && raw < per && s_issued * per + raw < nchunks) ch = s_issued * per + raw;
    ch = __shfl_sync(FULL, ch, 0);
    if (ch != INF) return ch;
    return grab_chunk(L, nchunks, s_cur);
}

// ---------------------------------------------------------------- ballot filter
// Word sources: word(wi) is called warp-collectively for wi = base + lane.
struct BitmapWords {  // frontier bitmap
    const uint32_t* bm;
    __device__ __forceinline__ uint32_t word(uint64_t wi) const { return bm[wi]; }
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
    uint32_t* lists;      // NCLS class regions of cstride entries
    uint64_t cstride;
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

// Per-class counters indexed by a runtime class without dynamic indexing (a local
// array indexed by a runtime value lives in local memory: an LDL/STL pair per use).
__device__ __forceinline__ void cls_count(uint32_t (&acc)[NCLS], uint32_t c) {
#pragma unroll
    for (int k = 0; k < NCLS; ++k) acc[k] += c == (uint32_t)k;
}
__device__ __forceinline__ uint32_t cls_take(uint32_t (&pos)[NCLS], uint32_t c) {
    uint32_t r = pos[0];
#pragma unroll
    for (int k = 1; k < NCLS; ++k) r = c == (uint32_t)k ? pos[k] : r;
#pragma unroll
    for (int k = 0; k < NCLS; ++k) pos[k] += c == (uint32_t)k;
    return r;
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
            out.lists[(uint64_t)c * out.cstride + pos[c]++] = v;
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

// for_edges in batches: fn(u, k) gets k (1..4) neighbour ids u[0..k) whose
// dependent loads / atomics the caller issues together (ILP across a vector).
template <class Fn>
__device__ __forceinline__ void for_edges_b(const uint32_t* __restrict__ col, uint64_t beg, uint64_t end,
                                            uint64_t rank, uint64_t size, Fn&& fn) {
    uint64_t a = (beg + 3) & ~3ull;
    if (a > end) a = end;
    for (uint64_t e = beg + rank; e < a; e += size) {
        const uint32_t u[4] = {__ldg(col + e), INF, INF, INF};
        fn(u, 1);
    }
    const uint64_t nvec = (end - a) >> 2;
    const uint4* c4 = reinterpret_cast<const uint4*>(col + a);
    for (uint64_t i = rank; i < nvec; i += size) {
        const uint4 q = __ldg(c4 + i);
        const uint32_t u[4] = {q.x, q.y, q.z, q.w};
        fn(u, 4);
    }
    for (uint64_t e = a + 4 * nvec + rank; e < end; e += size) {
        const uint32_t u[4] = {__ldg(col + e), INF, INF, INF};
        fn(u, 1);
    }
}

// for_edges with the edge weight: in the aligned body the four u8 weights of a
// 128-bit group of ids arrive in one 32-bit load (u32 weights: one 128-bit load).
template <class Fn>
__device__ __forceinline__ void for_edges_w(const uint32_t* __restrict__ col, const uint8_t* __restrict__ w8,
                                            const uint32_t* __restrict__ w32, uint64_t beg, uint64_t end,
                                            uint64_t rank, uint64_t size, Fn&& fn) {
    uint64_t a = (beg + 3) & ~3ull;
    if (a > end) a = end;
    for (uint64_t e = beg + rank; e < a; e += size) fn(e, __ldg(col + e), edge_w(w8, w32, e));
    const uint64_t nvec = (end - a) >> 2;
    const uint4* c4 = reinterpret_cast<const uint4*>(col + a);
    for (uint64_t i = rank; i < nvec; i += size) {
        const uint4 q = __ldg(c4 + i);
        const uint64_t e = a + 4 * i;
        uint32_t w0, w1, w2, w3;
        if (w8) {
            const uint32_t ww = __ldg(reinterpret_cast<const uint32_t*>(w8 + e));
            w0 = ww & 0xFF;
            w1 = (ww >> 8) & 0xFF;
            w2 = (ww >> 16) & 0xFF;
            w3 = ww >> 24;
        } else if (w32) {
            const uint4 ww = __ldg(reinterpret_cast<const uint4*>(w32 + e));
            w0 = ww.x;
            w1 = ww.y;
            w2 = ww.z;
            w3 = ww.w;
        } else {
            w0 = w1 = w2 = w3 = 1u;
        }
        fn(e, q.x, w0);
        fn(e + 1, q.y, w1);
        fn(e + 2, q.z, w2);
        fn(e + 3, q.w, w3);
    }
    for (uint64_t e = a + 4 * nvec + rank; e < end; e += size) fn(e, __ldg(col + e), edge_w(w8, w32, e));
}

// for_edges_w in batches: fn(u, w, k) gets k (1..4) neighbour ids and weights,
// so the caller can issue the four edges' dependent loads together.
template <class Fn>
__device__ __forceinline__ void for_edges_wb(const uint32_t* __restrict__ col, const uint8_t* __restrict__ w8,
                                             const uint32_t* __restrict__ w32, uint64_t beg, uint64_t end,
                                             uint64_t rank, uint64_t size, Fn&& fn) {
    uint64_t a = (beg + 3) & ~3ull;
    if (a > end) a = end;
    for (uint64_t e = beg + rank; e < a; e += size) {
        const uint32_t u[4] = {__ldg(col + e), 0u, 0u, 0u};
        const uint32_t w[4] = {edge_w(w8, w32, e), 0u, 0u, 0u};
        fn(u, w, 1u);
    }
    const uint64_t nvec = (end - a) >> 2;
    const uint4* c4 = reinterpret_cast<const uint4*>(col + a);
    for (uint64_t i = rank; i < nvec; i += size) {
        const uint4 q = __ldg(c4 + i);
        const uint64_t e = a + 4 * i;
        const uint32_t u[4] = {q.x, q.y, q.z, q.w};
        uint32_t w[4];
        if (w8) {
            const uint32_t ww = __ldg(reinterpret_cast<const uint32_t*>(w8 + e));
            w[0] = ww & 0xFF;
            w[1] = (ww >> 8) & 0xFF;
            w[2] = (ww >> 16) & 0xFF;
            w[3] = ww >> 24;
        } else if (w32) {
            const uint4 ww = __ldg(reinterpret_cast<const uint4*>(w32 + e));
            w[0] = ww.x;
            w[1] = ww.y;
            w[2] = ww.z;
            w[3] = ww.w;
        } else {
            w[0] = w[1] = w[2] = w[3] = 1u;
        }
        fn(u, w, 4u);
    }
    for (uint64_t e = a + 4 * nvec + rank; e < end; e += size) {
        const uint32_t u[4] = {__ldg(col + e), 0u, 0u, 0u};
        const uint32_t w[4] = {edge_w(w8, w32, e), 0u, 0u, 0u};
        fn(u, w, 1u);
    }
}

// Predicated u32 load (returns `dflt` when !c) without a branch, so that a batch
// of dependent gathers is issued back to back.
__device__ __forceinline__ uint32_t ld_pred_u32(const uint32_t* p, bool c, uint32_t dflt) {
    uint32_t v = dflt;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.global.u32 %0, [%1];\n\t}"
                 : "+r"(v) : "l"(p), "r"((int)c));
    return v;
}

// One thread sums term(e, col[e]) over [beg, end) with 16 neighbour ids (four
// 128-bit loads) and their 16 gathers in flight per step.
template <class Term>
__device__ __forceinline__ double seq_sum(const uint32_t* __restrict__ col, uint64_t beg, uint64_t end, Term&& term) {
    double acc = 0.0;
    uint64_t e = beg;
    const uint64_t a = min((uint64_t)((beg + 3) & ~3ull), end);
    for (; e < a; ++e) acc += term(e, __ldg(col + e));
    for (; e + 16 <= end; e += 16) {
        const uint4* c4 = reinterpret_cast<const uint4*>(col + e);
        const uint4 q0 = __ldg(c4), q1 = __ldg(c4 + 1), q2 = __ldg(c4 + 2), q3 = __ldg(c4 + 3);
        const double t0 = term(e, q0.x) + term(e + 1, q0.y) + term(e + 2, q0.z) + term(e + 3, q0.w);
        const double t1 = term(e + 4, q1.x) + term(e + 5, q1.y) + term(e + 6, q1.z) + term(e + 7, q1.w);
        const double t2 = term(e + 8, q2.x) + term(e + 9, q2.y) + term(e + 10, q2.z) + term(e + 11, q2.w);
        const double t3 = term(e + 12, q3.x) + term(e + 13, q3.y) + term(e + 14, q3.z) + term(e + 15, q3.w);
        acc += (t0 + t1) + (t2 + t3);
    }
    for (; e + 4 <= end; e += 4) {
        const uint4 q = __ldg(reinterpret_cast<const uint4*>(col + e));
        acc += term(e, q.x) + term(e + 1, q.y) + term(e + 2, q.z) + term(e + 3, q.w);
    }
    for (; e < end; ++e) acc += term(e, __ldg(col + e));
    return acc;
}

// Visit the four class lists of the current view with thread / warp / CTA /
// grid granularity.  The functor gets (v, rank, size, class) and loops
// over v's edges itself.  Huge vertices (grid-split, B200 addition) go first so
// the whole GPU shares them, small ones last so they fill the tail.
template <class VFn>
__device__ __forceinline__ void for_tasks(const uint32_t* lists, const Sched& s, const uint32_t (&cnt)[NCLS], VFn&& vf) {
    // huge: the CTAs are split into cnt[3] equal groups, one per task, so the
    // tasks run side by side (one task at a time over the whole grid left a
    // dependent row_ptr -> col -> update chain per task exposed: 3.4 us each)
    if (cnt[3] >= gridDim.x) {
        for (uint32_t i = blockIdx.x; i < cnt[3]; i += gridDim.x) vf(task_at(lists, s, 3, i), (uint64_t)threadIdx.x, (uint64_t)BLOCK, 3u);
    } else if (cnt[3] > 0) {
        const uint64_t T = cnt[3], G = gridDim.x;
        const uint64_t i = (uint64_t)blockIdx.x * T / G;
        const uint64_t g0 = (i * G + T - 1) / T, g1 = ((i + 1) * G + T - 1) / T;
        vf(task_at(lists, s, 3, (uint32_t)i), (blockIdx.x - g0) * BLOCK + threadIdx.x, (g1 - g0) * BLOCK, 3u);
    }
    for (uint32_t i = blockIdx.x; i < cnt[2]; i += gridDim.x)
        vf(task_at(lists, s, 2, i), (uint64_t)threadIdx.x, (uint64_t)BLOCK, 2u);
    // CTA-major spreading: consecutive warp tasks / 32-task chunks go to different
    // CTAs, so a small frontier runs on many SMs instead of the first few.
    const uint64_t wslot = blockIdx.x + (uint64_t)warp_id() * gridDim.x;
    for (uint64_t i = wslot; i < cnt[1]; i += gwarps()) vf(task_at(lists, s, 1, (uint32_t)i), (uint64_t)lane_id(), 32ull, 1u);
    const uint64_t nch = ((uint64_t)cnt[0] + 31) >> 5;
    for (uint64_t ch = wslot; ch < nch; ch += gwarps()) {
        const uint64_t i = (ch << 5) + lane_id();
        if (i < cnt[0]) vf(task_at(lists, s, 0, (uint32_t)i), 0ull, 1ull, 0u);
    }
}

// CTA-local binning of a short flat task list (the found list a pull iteration
// recorded with the online filter): CTA b takes the contiguous chunk
// [b0, b1) of the list, classifies its entries by degree in shared memory and
// runs small ones at thread, medium ones at warp and large / huge ones at CTA
// granularity — no grid-wide class lists, so no barrier before the
// iteration.  Balance across CTAs is by entry count; the lists this serves are
// the last levels of a traversal (few, low-degree vertices).
template <class VFn>
__device__ __forceinline__ void for_list_local(const uint32_t* list, uint32_t n, const Sched& s, const uint32_t* deg,
                                               VFn&& vf) {
    __shared__ uint32_t q_w[BLOCK], q_c[BLOCK];
    __shared__ uint32_t nq[2];
    const uint32_t per = (n + gridDim.x - 1) / gridDim.x;
    const uint32_t b0 = min(n, blockIdx.x * per), b1 = min(n, b0 + per);
    for (uint32_t base = b0; base < b1; base += BLOCK) {  // CTA-uniform
        if (threadIdx.x < 2) nq[threadIdx.x] = 0;
        __syncthreads();
        const uint32_t i = base + threadIdx.x;
        uint32_t v = INF, c = NCLS;
        if (i < b1) {
            v = list[i];
            c = cls_of(__ldg(deg + v), s);
        }
        if (c == 1) q_w[atomicAdd(&nq[0], 1u)] = v;
        else if (c == 2 || c == 3) q_c[atomicAdd(&nq[1], 1u)] = v;
        if (c == 0) vf(v, 0ull, 1ull, 0u);
        __syncthreads();
        const uint32_t nw = nq[0], nc = nq[1];
        for (uint32_t j = warp_id(); j < nw; j += WARPS) vf(q_w[j], (uint64_t)lane_id(), 32ull, 1u);
        for (uint32_t j = 0; j < nc; ++j) vf(q_c[j], (uint64_t)threadIdx.x, (uint64_t)BLOCK, 2u);
        __syncthreads();
    }
}

// ---------------------------------------------------------------- bookkeeping
struct Stats {
    uint64_t edges = 0, entries = 0, scanned = 0, reached = 0;
    uint32_t ballot = 0, pull = 0, iters = 0;
};

// Per-CTA partial counters -> one atomic per CTA; uniform counters from CTA 0.
// blocks (nullable): flush into these statistics blocks instead of the control
// block's (the asynchronous BFS accumulates its runs' statistics there)
__device__ __forceinline__ void flush_stats(Ctl* c, Stats& st, uint32_t dir, Ctl::StatBlock* blocks = nullptr) {
    uint64_t v[3] = {st.edges, st.entries, st.reached};
    block_sum<3>(v);
    if (threadIdx.x == 0) {
        Ctl::StatBlock& b = blocks ? blocks[dir] : c->st[dir];
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

// ---------------------------------------------------------------- small-frontier cluster mode
// When the frontier is small the grid barrier (~3 us for 600+ CTAs) dominates an
// iteration.  The push then continues on ONE thread-block cluster of CL_CTAS x
// CL_BLOCK threads whose barrier is the hardware cluster barrier: same ACC step,
// online filter into one list, no grid barrier.  Frontier hand-over with the grid
// kernels is the bitmap bm[it % 3]; consumers clear the bits they consume, so
// bm[(it+1)%3] and bm[(it+2)%3] stay zero as the grid kernels expect.
__device__ __forceinline__ void cluster_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// warp-aggregated append to a list with a global counter
__device__ __forceinline__ void cl_append(uint32_t* list, unsigned int* cnt, uint32_t u) {
    const uint32_t m = __activemask();
    const int leader = __ffs(m) - 1;
    uint32_t base = 0;
    if ((int)lane_id() == leader) base = atomicAdd(cnt, (uint32_t)__popc(m));
    base = __shfl_sync(m, base, leader);
    list[base + __popc(m & lanemask_lt())] = u;
}
// Append the u[k] whose bit k is set in sel (k < 8) with ONE returning atomic
// per warp: each lane's count goes in as four bit-plane ballots, so the
// exclusive prefix over a sparse active mask needs no shuffles.
// Entries at positions >= cap are counted but not written: the caller sees
// count > cap after its barrier and rebuilds the frontier from the bitmap.
__device__ __forceinline__ void cl_append8(uint32_t* list, unsigned int* cnt, const uint32_t (&u)[8], uint32_t sel,
                                           uint32_t cap = 0xFFFFFFFFu) {
    const uint32_t m = __activemask();
    const uint32_t c = __popc(sel), lt = lanemask_lt();
    uint32_t pre = 0, tot = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const uint32_t bb = __ballot_sync(m, (c >> b) & 1u);
        pre += __popc(bb & lt) << b;
        tot += __popc(bb) << b;
    }
    if (tot == 0) return;
    const int leader = __ffs(m) - 1;
    uint32_t base = 0;
    if ((int)lane_id() == leader) base = atomicAdd(cnt, tot);
    base = __shfl_sync(m, base, leader) + pre;
#pragma unroll
    for (int k = 0; k < 8; ++k)
        if (sel >> k & 1u) {
            if (base < cap) list[base] = u[k];
            ++base;
        }
}
// Visit the nonzero words of a bitmap (nwords a multiple of 4) with 128-bit
// loads, 4 in flight per thread: f(word index, word).
template <class F>
__device__ __forceinline__ void cluster_words(const uint32_t* bm, uint64_t nwords, uint32_t tid, uint32_t T, F&& f) {
    const uint4* q = reinterpret_cast<const uint4*>(bm);
    const uint64_t nq = nwords / 4;
    for (uint64_t q0 = tid; q0 < nq; q0 += 4ull * T) {
        uint4 w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) w[k] = q0 + k * T < nq ? q[q0 + k * T] : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint64_t b = (q0 + k * T) * 4;
            if (w[k].x) f(b, w[k].x);
            if (w[k].y) f(b + 1, w[k].y);
            if (w[k].z) f(b + 2, w[k].z);
            if (w[k].w) f(b + 3, w[k].w);
        }
    }
}

// Exclusive scan over the 1024 threads of a cluster CTA; *total = CTA sum.
__device__ __forceinline__ uint32_t cta_scan_1024(uint32_t v, uint32_t* total) {
    __shared__ uint32_t s_ws[32];
    __shared__ uint32_t s_tot;
    const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, incl, o);
        if ((int)lane >= o) incl += y;
    }
    if (lane == 31) s_ws[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        const uint32_t x = s_ws[lane];
        uint32_t sx = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, sx, o);
            if ((int)lane >= o) sx += y;
        }
        s_ws[lane] = sx - x;
        if (lane == 31) s_tot = sx;
    }
    __syncthreads();
    const uint32_t excl = s_ws[wid] + incl - v;
    *total = s_tot;
    __syncthreads();  // s_ws / s_tot reuse by the next call
    return excl;
}
// Cluster-wide compaction of a bitmap into a list: the bits mask(word index,
// word) keeps (words read with 128-bit loads, 16 per thread per round) are
// appended to L at positions claimed with ONE atomicAdd per CTA per round.
// Every thread of the cluster must call it (CTA barriers inside).
template <class M>
__device__ __forceinline__ void cluster_compact(const uint32_t* bm, uint64_t nwords, uint32_t tid, uint32_t T,
                                                unsigned int* cnt, uint32_t* L, M&& mask) {
    __shared__ uint32_t s_base;
    const uint4* q = reinterpret_cast<const uint4*>(bm);
    const uint64_t nq = nwords / 4;
    const uint64_t rounds = (nq + 4ull * T - 1) / (4ull * T);
    for (uint64_t r = 0; r < rounds; ++r) {
        const uint64_t q0 = r * 4ull * T + tid;
        uint32_t w[16];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint4 x = q0 + k * T < nq ? q[q0 + k * T] : make_uint4(0u, 0u, 0u, 0u);
            w[4 * k] = x.x;
            w[4 * k + 1] = x.y;
            w[4 * k + 2] = x.z;
            w[4 * k + 3] = x.w;
        }
        uint32_t pc = 0;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            if (w[j]) w[j] = mask((q0 + (j >> 2) * T) * 4 + (j & 3), w[j]);
            pc += __popc(w[j]);
        }
        uint32_t tot;
        uint32_t pos = cta_scan_1024(pc, &tot);
        if (tot == 0) continue;  // CTA-uniform
        if (threadIdx.x == 0) s_base = atomicAdd(cnt, tot);
        __syncthreads();
        pos += s_base;
#pragma unroll
        for (int j = 0; j < 16; ++j)
            for (uint32_t x = w[j]; x; x &= x - 1)
                L[pos++] = (uint32_t)((((q0 + (j >> 2) * T) * 4 + (j & 3)) << 5) + (__ffs(x) - 1));
        __syncthreads();  // s_base reuse
    }
}
// Per-vertex values of the set bits of word wi (32 consecutive vertices = one
// 128-B line): the 4-vertex quads holding set bits are loaded together.
template <class F>
__device__ __forceinline__ void word_values(const uint32_t* a, uint64_t wi, uint32_t x, F&& f) {
    const uint4* q = reinterpret_cast<const uint4*>(a + (wi << 5));
    uint4 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = (x >> (4 * j)) & 0xFu ? q[j] : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const uint32_t nib = (x >> (4 * j)) & 0xFu;
        if (nib & 1u) f(4 * j, v[j].x);
        if (nib & 2u) f(4 * j + 1, v[j].y);
        if (nib & 4u) f(4 * j + 2, v[j].z);
        if (nib & 8u) f(4 * j + 3, v[j].w);
    }
}

// Entry: zero the cluster counters and the stale bitmap bm[(it+2)%3], list the
// frontier bitmap bm[it % 3] into lists[it & 1] (count in cl.cnt[it % 3]).
__device__ __forceinline__ void cluster_entry(const Sched& s, uint32_t it, uint32_t tid, uint32_t T) {
    Ctl::ClusterLine* cl = &s.ctl->cl;
    // the BFS pull kernel may hand over the frontier as a ready list (it also
    // cleared the stale bitmap): then only the counters are reset
    const bool ready = vload(&cl->ready) != 0;
    cluster_barrier();  // every CTA has read `ready` before thread 0 clears it
    if (tid == 0) {
        for (int i = 0; i < 3; ++i) {
            if (!(ready && i == (int)(it % 3))) cl->cnt[i] = 0;
            cl->nbig[i] = 0;
            cl->mf[i] = 0;
        }
        cl->minv = INF;
        cl->fmin[0] = cl->fmin[1] = INF;
        cl->ready = 0;
    }
    if (ready) {
        cluster_barrier();
        return;
    }
    uint4* z = reinterpret_cast<uint4*>(s.bm[(it + 2) % 3]);
    const uint64_t nq = s.nwords / 4;
    for (uint64_t q = tid; q < nq; q += T) z[q] = make_uint4(0u, 0u, 0u, 0u);
    cluster_barrier();
    cluster_compact(s.bm[it % 3], s.nwords, tid, T, &cl->cnt[it % 3], s.lists[it & 1],
                    [](uint64_t, uint32_t w) { return w; });
    cluster_barrier();
}
// Exit (one thread): the grid kernels rebuild their lists from bm[it % 3] and
// start from zeroed grid-barrier counters.
__device__ __forceinline__ void cluster_leave(Ctl* c) {
    for (int i = 0; i < 3; ++i) c->cl.cnt[i] = 0;  // the BFS pull kernel counts its hand-over list here
    c->lists_ready = 0;
    c->slotted = 0;
    for (int h = 0; h < 2; ++h) {
        for (int i = 0; i < BAR_GROUPS; ++i) c->bar_grp[h][i].count = 0;
        c->bar_top[h].count = 0;
    }
    c->launch += 1;
}

}  // namespace sx

// dist.cu — the multi-GPU layer.
//
// 1D vertex-range partition: rank r owns vertices [r*V, min(N, (r+1)*V)), V =
// ceil(N/P) rounded up to a multiple of 32 so every bitmap slice is whole
// words.  Each rank holds the CSR rows of its owned vertices with GLOBAL column
// ids (for a symmetric graph those rows are also the in-neighbour rows).
// Traversal shards naturally by vertex range; the per-iteration exchange is:
//   BFS pull level : allgather of the frontier-bitmap slices (N/8/P bytes each),
//                    then a local bottom-up pass over owned unvisited vertices;
//   BFS push level : each rank marks targets in a global-size bitmap; alltoall of
//                    the per-owner slices; the owner ORs them and keeps the
//                    unvisited bits (NCCL has no bitwise-OR reduction);
//   SSSP iteration : candidate distances for remote targets min-combined into a
//                    global-size array, reduce-scatter(min) to the owners;
//   every level    : allreduce of (|F'|, m_f) — termination and the Beamer
//                    direction decision are taken identically on every rank.
// Exchange backends: NCCL (one rank per process, ncclComm from a unique id the
// caller broadcasts, collectives on the ctx stream) or, with all ranks in one
// process on one device ("virtual ranks", for tests), the same schedule with
// device-to-device copies standing in for the collectives.
#include <nccl.h>
#include <nccl_device.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "internal.h"

using namespace sx;

namespace {

constexpr int DIST_MAX_LOCAL = 64;
constexpr int KGRID_PER_SM = 4;

struct DistRank {
    uint64_t nl = 0, ml = 0, lo = 0;  // owned rows, local edges, first owned vertex
    uint64_t* rp = nullptr;
    uint32_t* ci = nullptr;
    void* w = nullptr;
    uint32_t* deg = nullptr;          // out-degree of owned rows
    uint32_t* nz = nullptr;           // owned words: degree > 0
    uint32_t* state = nullptr;        // level / dist of owned rows
    uint32_t* visited = nullptr;      // owned words (BFS visited / SSSP far pile)
    uint32_t* front[2] = {nullptr, nullptr};  // owned words
    uint32_t* gfront = nullptr;       // NW global words (pull: allgathered frontier)
    uint32_t* sendmap = nullptr;      // NW global words (push targets)
    uint32_t* recv = nullptr;         // P * nwl words (alltoall receive)
    uint64_t* pieces = nullptr;       // push: (row, piece) items of the rows split into DIST_PIECE-edge pieces
    uint32_t* hub = nullptr;          // pull: per owned row, its neighbour of largest GLOBAL degree among the first 64 (lazy)
    uint32_t* sendbest = nullptr;     // SSSP (lazy): P * V sender-side candidate minima (INF between iterations)
    uint32_t* touched = nullptr;      // SSSP: P regions of V ids first improved this iteration, by owner
    uint32_t* tcnt = nullptr;         // SSSP: P per-owner touched counts, then P received counts
    uint64_t* sendbuf = nullptr;      // SSSP: P regions of V packed (id << 32 | dist) pairs, by owner
    uint64_t* recvbuf = nullptr;      // SSSP: P regions of V pairs, by sender
    unsigned long long* cnt = nullptr;  // device counters
    bool has_zero_w = false;
};

}  // namespace

struct sx_dist_s {
    sx_ctx ctx = nullptr;
    int P = 1, rank0 = 0, nlocal = 1;
    uint64_t N = 0, V = 0, nwl = 0, NW = 0;
    uint32_t wbytes = 0;
    bool nccl = false;
    ncclComm_t comm = nullptr;
    DistRank r[DIST_MAX_LOCAL];
    unsigned long long* hcnt = nullptr;  // pinned host counters [nlocal][8]
    unsigned long long* dred = nullptr;  // device allreduce buffer (8)
    // device-initiated BFS (fusion = 2; NCCL device API): one
    // symmetric window per rank (global frontier bitmap | push inbox | counter slots),
    // a device communicator with one LSA barrier, and the fused kernel's control block
    void* sym = nullptr;
    size_t sym_bytes = 0, off_in = 0, off_cnt = 0;
    ncclWindow_t win = nullptr;
    ncclDevComm dcomm{};
    bool dcomm_ok = false;
    sx::Ctl* fctl = nullptr;
    unsigned long long* fstats = nullptr;  // device: iterations, pull levels, edges, reached, error; level stamps
    unsigned long long m_total = 0;        // global directed edge count (allreduced once per upload)
    bool m_total_ok = false;
    int fgrid = 0;                         // the fused kernel's cooperative grid
    // asynchronous fused runs (sx_dist_bfs_async): count, device-time events
    uint32_t async_runs = 0;
    cudaEvent_t aev[2] = {nullptr, nullptr};
};

namespace {

sx_status nccl_fail(ncclResult_t r, const char* what) {
    return sxh::fail(SX_E_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}
#define SX_NC(call)                                               \
    do {                                                          \
        ncclResult_t r__ = (call);                                \
        if (r__ != ncclSuccess) return nccl_fail(r__, #call);     \
    } while (0)

template <class T> sx_status dmalloc(T** p, size_t count) {
    cudaError_t e = cudaMalloc((void**)p, (count ? count : 1) * sizeof(T));
    if (e != cudaSuccess) {
        *p = nullptr;
        return sxh::cuda_fail(e, "cudaMalloc");
    }
    return SX_OK;
}

int kgrid(sx_dist d) { return KGRID_PER_SM * d->ctx->prop.multiProcessorCount; }

// ------------------------------------------------------------------ kernels
struct RankView {
    uint64_t nl, lo, nwl;
    const uint64_t* __restrict__ rp;
    const uint32_t* __restrict__ ci;
    const uint8_t* __restrict__ w8;
    const uint32_t* __restrict__ w32;
    const uint32_t* __restrict__ deg;
    const uint32_t* __restrict__ nz;
    uint32_t* state;
    uint32_t* visited;
    uint32_t* cur;
    uint32_t* nxt;
    uint32_t* gfront;
    uint32_t* sendmap;
    const uint32_t* recv;
    uint32_t* sendbest;
    unsigned long long* cnt;
    uint64_t* pieces;
    const uint32_t* hub;
    uint32_t* touched;
    uint32_t* tcnt;
    uint64_t* sendbuf;
    const uint64_t* recvbuf;
    uint32_t P;
    uint64_t V;
    uint32_t sep_small;
};

// Visit the owned vertices whose bit is set in `bits` (owned words) with the
// engine's granularities: small rows on the lane (thread), medium rows
// by the warp, and rows of at least DIST_PIECE edges split into pieces of
// DIST_PIECE edges that the next launch spreads over every warp of the GPU
// (the grid split of the single-GPU engine's huge class: an R-MAT hub of 10^5-10^6
// edges no longer sits on one warp).  Pieces are listed with one atomic per row.
constexpr uint32_t DIST_PIECE = 256;  // 8 edges per lane: a hub row's pieces fill the GPU in one round
constexpr int CNT_PIECES = 5;  // counter slot holding the piece count of the level
// Word batches: a warp loads 32 consecutive words of an owned bitmap at once
// (lane = word) and visits only the nonzero ones (ballot), instead of one
// dependent word load per warp step — a sparse frontier costs one coalesced
// pass over the bitmap.  f(word index, word), warp-collective.
template <class WordFn>
__device__ __forceinline__ void dist_for_words(const uint32_t* bits, uint64_t nwl, WordFn&& f) {
    const uint32_t lane = lane_id();
    const uint64_t nb = (nwl + 31) >> 5;
    for (uint64_t bi = gwarp(); bi < nb; bi += gwarps()) {
        const uint64_t wl = (bi << 5) + lane;
        const uint32_t myw = wl < nwl ? bits[wl] : 0u;
        for (uint32_t act = __ballot_sync(FULL, myw != 0); act; act &= act - 1) {
            const int j = __ffs(act) - 1;
            f((bi << 5) + j, __shfl_sync(FULL, myw, j));
        }
    }
}
template <class EdgeFn>
__device__ __forceinline__ void dist_for_active(const RankView& r, const uint32_t* bits, EdgeFn&& fn) {
    const uint32_t lane = lane_id();
    dist_for_words(bits, r.nwl, [&](uint64_t wi, uint32_t word) {
        const uint64_t vl = (wi << 5) + lane;
        const bool mine = (word >> lane) & 1u;
        uint64_t beg = 0, end = 0;
        if (mine) {
            beg = __ldg(r.rp + vl);
            end = __ldg(r.rp + vl + 1);
        }
        const bool small = mine && end - beg < r.sep_small;
        const bool split = mine && end - beg >= DIST_PIECE;
        if (small)
            for (uint64_t e = beg; e < end; ++e) fn(vl, e, __ldg(r.ci + e));
        for (uint32_t sp = __ballot_sync(FULL, split); sp; sp &= sp - 1) {  // the warp lists each row's pieces
            const int l = __ffs(sp) - 1;
            const uint64_t b0 = __shfl_sync(FULL, beg, l), e0 = __shfl_sync(FULL, end, l);
            const uint64_t vr = (wi << 5) + l, np = (e0 - b0 + DIST_PIECE - 1) / DIST_PIECE;
            uint64_t base = 0;
            if (lane == 0) base = atomicAdd(r.cnt + CNT_PIECES, (unsigned long long)np);
            base = __shfl_sync(FULL, base, 0);
            for (uint64_t q = lane; q < np; q += 32) r.pieces[base + q] = (vr << 32) | q;
        }
        uint32_t todo = __ballot_sync(FULL, mine && !small && !split);
        while (todo) {
            const int l = __ffs(todo) - 1;
            todo &= todo - 1;
            const uint64_t b0 = __shfl_sync(FULL, beg, l), e0 = __shfl_sync(FULL, end, l);
            const uint64_t v0 = (wi << 5) + l;
            for (uint64_t e = b0 + lane; e < e0; e += 32) fn(v0, e, __ldg(r.ci + e));
        }
    });
}
// the pieces listed by dist_for_active: one warp per piece, lane-strided edges
template <class EdgeFn> __device__ __forceinline__ void dist_for_pieces(const RankView& r, EdgeFn&& fn) {
    const uint64_t np = vload(r.cnt + CNT_PIECES);
    for (uint64_t i = gwarp(); i < np; i += gwarps()) {
        const uint64_t it = r.pieces[i];
        const uint64_t vl = it >> 32, q = it & 0xFFFFFFFFull;
        const uint64_t beg = __ldg(r.rp + vl) + q * DIST_PIECE;
        const uint64_t end = min(beg + DIST_PIECE, __ldg(r.rp + vl + 1));
        for (uint64_t e = beg + lane_id(); e < end; e += 32 * 4) {  // 4 ids in flight per lane
            uint32_t u[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) u[k] = e + 32 * k < end ? __ldg(r.ci + e + 32 * k) : INF;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (u[k] != INF) fn(vl, e + 32 * k, u[k]);
        }
    }
}

// PIECES = 0: the active rows (big ones listed as pieces); 1: the pieces
template <int PIECES> __global__ void k_bfs_push(RankView r) {
    unsigned long long edges = 0;
    auto fn = [&](uint64_t, uint64_t, uint32_t u) {
        ++edges;
        const uint64_t ul = (uint64_t)u - r.lo;
        // owned and already visited (read-only during the push: the non-coherent path
        // lets the loads of several edges issue ahead of the marks)
        if (ul < r.nl && ((__ldg(r.visited + (ul >> 5)) >> (ul & 31)) & 1u)) return;
        bm_set(r.sendmap, u);
    };
    if (PIECES) dist_for_pieces(r, fn);
    else dist_for_active(r, r.cur, fn);
    uint64_t a[1] = {edges};
    block_sum<1>(a);
    if (threadIdx.x == 0 && a[0]) atomicAdd(r.cnt + 2, (unsigned long long)a[0]);
}

// owner side of a push level: OR the P received slices, keep the unvisited bits
// Also clears, in the same launch, the level's pushed frontier (r.cur: the next
// level's output buffer) and this rank's send bitmap (consumed by the exchange
// before this launch) — no memset launches per level.
__global__ void k_bfs_apply(RankView r, uint32_t lvl) {
    unsigned long long found = 0, mdeg = 0;
    const uint64_t NW = (uint64_t)r.P * r.nwl;
    for (uint64_t w = gtid(); w < NW; w += gthreads()) r.sendmap[w] = 0;
    for (uint64_t wi = gtid(); wi < r.nwl; wi += gthreads()) {
        r.cur[wi] = 0;
        uint32_t m = 0;
        for (uint32_t q = 0; q < r.P; ++q) m |= r.recv[(uint64_t)q * r.nwl + wi];
        const uint64_t v0 = wi << 5;
        if (v0 + 32 > r.nl) m &= v0 >= r.nl ? 0u : ((1u << (uint32_t)(r.nl - v0)) - 1u);
        m &= ~r.visited[wi];
        r.nxt[wi] = m;
        if (m) {
            r.visited[wi] |= m;
            found += __popc(m);
            for (uint32_t x = m; x; x &= x - 1) {
                const uint64_t vl = v0 + (__ffs(x) - 1);
                r.state[vl] = lvl;
                mdeg += __ldg(r.deg + vl);
            }
        }
    }
    uint64_t a[2] = {found, mdeg};
    block_sum<2>(a);
    if (threadIdx.x == 0) {
        if (a[0]) atomicAdd(r.cnt + 0, (unsigned long long)a[0]);
        if (a[1]) atomicAdd(r.cnt + 1, (unsigned long long)a[1]);
    }
}

// Bottom-up over the owned unvisited candidates against a global frontier
// bitmap, the single-GPU pull's TILE scheme (bfs.cu) on a rank's slice: a warp
// takes a batch of 32 owned words (1024 vertices, lane = word), compacts the
// candidates (unvisited, in-degree > 0) into shared memory in vertex order,
// probes each one's hub entry first (DP_ILP rounds of 32 in flight: one hub load
// and one frontier-bit test each; a vain probe of a sole in-edge settles the
// vertex), then walks the rows of the candidates the hub left open — small rows
// on the lane, 4 probes in flight, larger ones by the whole warp with the
// voting early exit.  Found bits are merged per word in shared memory
// and stored once by the word's lane: no global atomics.  `mopen` returns the
// degree sum of the candidates still open after the level (walked rows: their
// length; settled sole edges: 1): on a symmetric graph that is m_u of the next
// level, so m_f = m_u - mopen with no degree load per found vertex (a found
// vertex's degree load stalled the probe loop: 15% of the kernel's samples).
constexpr int DP_ILP = 4;
constexpr uint32_t DHUB_SOLE = 0x80000000u;  // hub entry: bit 31 = the hub is the row's only edge (N <= 2^31)
__device__ __forceinline__ uint32_t dhub_id(uint32_t h) { return h == INF ? INF : h & ~DHUB_SOLE; }
__device__ __forceinline__ bool dhub_sole(uint32_t h) { return h != INF && (h & DHUB_SOLE); }
// clr (nullable): owned words zeroed on the way (the fused kernel's next output buffer)
__device__ __forceinline__ void dist_pull_batches(const RankView& r, const uint32_t* front, uint32_t* nxt, uint32_t lvl,
                                                  unsigned long long& found, unsigned long long& mopen,
                                                  unsigned long long& edges, uint32_t* clr = nullptr) {
    __shared__ uint32_t s_c[WARPS][1024];
    __shared__ uint32_t s_f[WARPS][32];
    const uint32_t lane = lane_id();
    uint32_t* sc = s_c[warp_id()];
    uint32_t* sf = s_f[warp_id()];
    const uint64_t nb = (r.nwl + 31) >> 5;
    for (uint64_t bi = gwarp(); bi < nb; bi += gwarps()) {
        const uint64_t wl = (bi << 5) + lane;
        const bool own = wl < r.nwl;
        const uint32_t vis = own ? r.visited[wl] : FULL;
        const uint32_t cand = own ? (~vis & __ldg(r.nz + wl)) : 0u;
        if (clr && own) clr[wl] = 0;
        uint32_t incl = __popc(cand);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, incl, o);
            if ((int)lane >= o) incl += y;
        }
        const uint32_t total = __shfl_sync(FULL, incl, 31);
        if (!total) continue;  // warp-uniform
        uint32_t pos = incl - __popc(cand);
        for (uint32_t w = cand; w; w &= w - 1) sc[pos++] = (lane << 5) | (uint32_t)(__ffs(w) - 1);
        sf[lane] = 0;
        __syncwarp();
        const uint64_t vb = bi << 10;  // first vertex of the batch
        // phase 1: hub-first probes; the open candidates are compacted in place (stable)
        uint32_t nopen = 0;
        for (uint32_t r0 = 0; r0 < total; r0 += 32 * DP_ILP) {
            uint32_t ix[DP_ILP], hx[DP_ILP], wd[DP_ILP];
#pragma unroll
            for (int k = 0; k < DP_ILP; ++k) {
                const uint32_t i = r0 + 32 * k + lane;
                ix[k] = i < total ? sc[i] : INF;
            }
#pragma unroll
            for (int k = 0; k < DP_ILP; ++k) hx[k] = ix[k] != INF && r.hub ? __ldg(r.hub + vb + ix[k]) : INF;
#pragma unroll
            for (int k = 0; k < DP_ILP; ++k) {
                const uint32_t h = dhub_id(hx[k]);
                wd[k] = h != INF ? front[h >> 5] : 0u;
            }
            __syncwarp();
#pragma unroll
            for (int k = 0; k < DP_ILP; ++k) {
                const uint32_t h = dhub_id(hx[k]);
                const bool f = h != INF && ((wd[k] >> (h & 31)) & 1u);
                edges += h != INF;
                if (f) {
                    r.state[vb + ix[k]] = lvl;
                    atomicOr(sf + (ix[k] >> 5), 1u << (ix[k] & 31));
                }
                if (ix[k] != INF && !f && dhub_sole(hx[k])) mopen += 1;  // settled: its one edge stays
                const bool open = ix[k] != INF && !f && !dhub_sole(hx[k]);
                const uint32_t bal = __ballot_sync(FULL, open);
                if (open) sc[nopen + __popc(bal & lanemask_lt())] = ix[k];
                nopen += __popc(bal);
            }
            __syncwarp();
        }
        // phase 2: row walks of the open candidates
        for (uint32_t o0 = 0; o0 < nopen; o0 += 32) {
            const bool mine = o0 + lane < nopen;
            const uint32_t ix = mine ? sc[o0 + lane] : 0u;
            const uint64_t vl = vb + ix;
            uint64_t beg = 0, end = 0;
            if (mine) {
                beg = __ldg(r.rp + vl);
                end = __ldg(r.rp + vl + 1);
            }
            bool hit = false;
            const bool small = mine && end - beg < r.sep_small;
            if (small) {
                for (uint64_t e = beg; e < end && !hit; e += 4) {
                    uint32_t u[4], w[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) u[k] = e + k < end ? __ldg(r.ci + e + k) : INF;
#pragma unroll
                    for (int k = 0; k < 4; ++k) w[k] = u[k] != INF ? front[u[k] >> 5] : 0u;
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (u[k] != INF) {
                            ++edges;
                            hit |= (w[k] >> (u[k] & 31)) & 1u;
                        }
                }
            }
            for (uint32_t todo = __ballot_sync(FULL, mine && !small); todo; todo &= todo - 1) {
                const int l = __ffs(todo) - 1;
                const uint64_t b0 = __shfl_sync(FULL, beg, l), e0 = __shfl_sync(FULL, end, l);
                bool any = false;
                for (uint64_t b = b0; b < e0 && !any; b += 32) {
                    const uint64_t e = b + lane;
                    bool h = false;
                    if (e < e0) {
                        ++edges;
                        h = bm_test(front, __ldg(r.ci + e));
                    }
                    any = __any_sync(FULL, h);
                }
                if ((int)lane == l) hit = any;
            }
            if (hit) {
                r.state[vl] = lvl;
                atomicOr(sf + (ix >> 5), 1u << (ix & 31));
            } else if (mine) {
                mopen += end - beg;
            }
        }
        __syncwarp();
        const uint32_t fm = sf[lane];
        if (own && fm) {
            r.visited[wl] = vis | fm;  // this warp owns the batch's words during the level
            nxt[wl] = fm;
            found += __popc(fm);
        }
        __syncwarp();
    }
}
__global__ void k_bfs_pull(RankView r, uint32_t lvl) {
    unsigned long long found = 0, mdeg = 0, edges = 0;
    dist_pull_batches(r, r.gfront, r.nxt, lvl, found, mdeg, edges, r.cur);  // r.cur: the next output, cleared on the way
    uint64_t a[3] = {found, mdeg, edges};
    block_sum<3>(a);
    if (threadIdx.x == 0) {
        if (a[0]) atomicAdd(r.cnt + 0, (unsigned long long)a[0]);
        if (a[1]) atomicAdd(r.cnt + 1, (unsigned long long)a[1]);
        if (a[2]) atomicAdd(r.cnt + 2, (unsigned long long)a[2]);
    }
}

// SSSP push over owned active vertices: local targets relaxed in place
// (atomicMin), remote ones min-combined into the global candidate array.
template <int PIECES> __global__ void k_sssp_push(RankView r, unsigned long long hi) {
    unsigned long long edges = 0;
    auto fn = [&](uint64_t vl, uint64_t e, uint32_t u) {
        ++edges;
        const uint32_t nd = r.state[vl] + edge_w(r.w8, r.w32, e);
        const uint64_t ul = (uint64_t)u - r.lo;
        if (ul < r.nl) {
            if (nd >= r.state[ul]) return;
            const uint32_t old = atomicMin(r.state + ul, nd);
            if (nd >= old) return;
            if ((unsigned long long)nd < hi) bm_set(r.nxt, (uint32_t)ul);
            else bm_set(r.visited, (uint32_t)ul);
        } else {
            // sender-side combining (min per target); the first
            // improvement of u this iteration lists u for its owner
            if (nd >= r.sendbest[u]) return;
            if (atomicMin(r.sendbest + u, nd) == INF) {
                const uint64_t q = u / r.V;
                const uint32_t pos = atomicAdd(r.tcnt + q, 1u);
                r.touched[q * r.V + pos] = u;
            }
        }
    };
    if (PIECES) dist_for_pieces(r, fn);
    else dist_for_active(r, r.cur, fn);
    uint64_t a[1] = {edges};
    block_sum<1>(a);
    if (threadIdx.x == 0 && a[0]) atomicAdd(r.cnt + 2, (unsigned long long)a[0]);
}

// sender side: pack each owner's touched targets as (id << 32 | dist) pairs and
// reset their candidate slots (a sparse reset: no P*V memset per iteration)
__global__ void k_sssp_pack(RankView r) {
    for (uint32_t q = 0; q < r.P; ++q) {
        const uint32_t nq = r.tcnt[q];
        for (uint64_t i = gtid(); i < nq; i += gthreads()) {
            const uint32_t u = r.touched[(uint64_t)q * r.V + i];
            r.sendbuf[(uint64_t)q * r.V + i] = ((uint64_t)u << 32) | r.sendbest[u];
            r.sendbest[u] = INF;
        }
    }
}
// owner side: apply the received pairs (rcnt[q] pairs from sender q at region q)
__global__ void k_sssp_apply_pairs(RankView r, const uint32_t* rcnt, unsigned long long hi) {
    for (uint32_t q = 0; q < r.P; ++q) {
        const uint32_t nq = rcnt[q];
        for (uint64_t i = gtid(); i < nq; i += gthreads()) {
            const uint64_t pr = r.recvbuf[(uint64_t)q * r.V + i];
            const uint32_t ul = (uint32_t)((pr >> 32) - r.lo), nd = (uint32_t)pr;
            if (nd >= r.state[ul]) continue;
            const uint32_t old = atomicMin(r.state + ul, nd);
            if (nd >= old) continue;
            if ((unsigned long long)nd < hi) bm_set(r.nxt, ul);
            else bm_set(r.visited, ul);
        }
    }
}
__global__ void k_count_next(RankView r) {
    unsigned long long active = 0;
    for (uint64_t wi = gtid(); wi < r.nwl; wi += gthreads()) active += __popc(r.nxt[wi]);
    uint64_t a[1] = {active};
    block_sum<1>(a);
    if (threadIdx.x == 0 && a[0]) atomicAdd(r.cnt + 0, (unsigned long long)a[0]);
}

__global__ void k_far_min(RankView r) {
    uint32_t mn = INF;
    for (uint64_t wi = gtid(); wi < r.nwl; wi += gthreads())
        for (uint32_t x = r.visited[wi]; x; x &= x - 1) mn = min(mn, r.state[(wi << 5) + (__ffs(x) - 1)]);
    mn = block_min(mn);
    if (threadIdx.x == 0 && mn != INF) atomicMin(r.cnt + 3, (unsigned long long)mn);
}

__global__ void k_far_move(RankView r, unsigned long long hi) {
    unsigned long long active = 0;
    for (uint64_t wi = gtid(); wi < r.nwl; wi += gthreads()) {
        uint32_t f = r.visited[wi], mv = 0;
        for (uint32_t x = f; x; x &= x - 1) {
            const int b = __ffs(x) - 1;
            if ((unsigned long long)r.state[(wi << 5) + b] < hi) mv |= 1u << b;
        }
        if (mv) {
            r.visited[wi] = f & ~mv;
            r.nxt[wi] |= mv;
        }
        active += __popc(r.nxt[wi]);
    }
    uint64_t a[1] = {active};
    block_sum<1>(a);
    if (threadIdx.x == 0 && a[0]) atomicAdd(r.cnt + 0, (unsigned long long)a[0]);
}

__global__ void k_validate_slice(const uint64_t* rp, const uint32_t* ci, uint64_t n, uint64_t m, uint64_t N,
                                 const void* w, uint32_t wbytes, uint32_t* flags) {
    const uint64_t t = gtid(), T = gthreads();
    uint32_t f = 0;
    if (t == 0 && (rp[0] != 0 || rp[n] != m)) f |= 4;
    for (uint64_t i = t; i < n; i += T)
        if (rp[i] > rp[i + 1]) f |= 1;
    for (uint64_t e = t; e < m; e += T) {
        if (ci[e] >= N) f |= 2;
        if (w && (wbytes == 1 ? ((const uint8_t*)w)[e] : ((const uint32_t*)w)[e]) == 0) f |= 8;
    }
    if (f) atomicOr(flags, f);
}

// BFS start on the source's owner: level 0, visited and frontier bits, and the
// source's degree in counter slot 4 (the first level's counter reduction
// carries it to every rank: m_u = m - deg(src) without a host round trip)
__global__ void k_dist_bfs_start(RankView r, uint32_t src) {
    const uint64_t sl = (uint64_t)src - r.lo;
    if (threadIdx.x != 0 || blockIdx.x != 0 || sl >= r.nl) return;
    const uint32_t bit = 1u << (sl & 31);
    r.state[sl] = 0;
    r.visited[sl >> 5] |= bit;
    r.cur[sl >> 5] |= bit;
    r.cnt[4] = r.deg[sl];
}
__global__ void k_deg_nz(const uint64_t* rp, uint64_t n, uint64_t nwl, uint32_t* deg, uint32_t* nz) {
    for (uint64_t i = gtid(); i < n; i += gthreads()) deg[i] = (uint32_t)(rp[i + 1] - rp[i]);
    for (uint64_t wi = gtid(); wi < nwl; wi += gthreads()) {
        uint32_t x = 0;
        for (int b = 0; b < 32; ++b) {
            const uint64_t v = (wi << 5) + b;
            if (v < n && rp[v + 1] > rp[v]) x |= 1u << b;
        }
        nz[wi] = x;
    }
}


// ------------------------------------------------------------------ device-initiated BFS
// the P:773-778 persistent loop across GPUs.  Every rank
// runs ONE cooperative kernel for the whole BFS; the per-level exchange is done
// from inside it over the NCCL device API instead of host-issued collectives:
//   push level: a remote target's bit is atomicOr'ed straight into its owner's
//               inbox slice through an LSA (load/store-accessible, NVLink) pointer
//               into the owner's symmetric window; the owner folds the inbox;
//   pull level: every owner stores its new frontier slice into every rank's
//               copy of the global frontier bitmap (LSA stores) before the level;
//   counters:   each rank stores (|F'|, m_f, edges) into every rank's counter
//               slots; every CTA of every rank sums the same P slots and takes the
//               same Beamer decision (reading 8);
//   barrier:    a local grid barrier, CTA 0 crosses one ncclLsaBarrierSession with
//               the peers (release/acquire at system scope), a local grid barrier.
// Requires every rank in one LSA team (one NVLink/NVSwitch domain).
constexpr int FS_STAMPS = 8, FS_NSTAMP = 24;  // fstats[8 + i]: globaltimer at the end of level i (bit 63: pull)
constexpr int FS_SUB = FS_STAMPS + FS_NSTAMP, FS_NSUB = 8;  // fstats[FS_SUB + 4 i + k]: sub-steps k of level i < 8
constexpr int FS_TOTAL = FS_SUB + 4 * FS_NSUB;
struct FusedBfsP {
    RankView r;
    uint32_t* front[2];
    Ctl* ctl;
    ncclDevComm dc;
    ncclWindow_t win;
    uint32_t* gfront;           // this rank's window: global frontier bitmap (NW words)
    uint32_t* inbox;            // this rank's window: push marks for its slice (nwl words)
    unsigned long long* slots;  // this rank's window: counter slots [2 parities][P ranks][4]
    uint64_t off_in, off_cnt;
    uint32_t P, me, src;
    uint64_t N, m_total;
    float alpha, beta;
    int force_dir;
    uint32_t max_iters;
    unsigned long long* fstats;
};

// Cross-rank barrier: a local grid barrier, CTA 0 crosses the LSA barrier with
// the peers, a local grid barrier.  The CTA's peer writes are ordered before it
// by __syncthreads + one system-scope fence per CTA (cumulativity), not a fence
// per thread.  With one rank there are no peers (no peer writes, no system-scope
// fence — measured 5-9 us per barrier): one grid barrier.
__device__ __forceinline__ bool xsync(const FusedBfsP& p) {
    if (p.P == 1) return grid_sync(p.ctl);
    __syncthreads();
    if (threadIdx.x == 0) __threadfence_system();
    if (!grid_sync(p.ctl)) return false;
    if (blockIdx.x == 0) {
        ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), p.dc, ncclTeamTagLsa(), 0u);
        bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
    }
    return grid_sync(p.ctl);
}

// x[0, n) = v with 16-B stores where aligned (grid-stride: thread tid of T)
__device__ __forceinline__ void fill_u32(uint32_t* x, uint64_t n, uint32_t v, uint64_t tid, uint64_t T) {
    const uint64_t head = (((16u - ((uintptr_t)x & 15u)) & 15u) / 4u) < n ? ((16u - ((uintptr_t)x & 15u)) & 15u) / 4u : n;
    if ((uintptr_t)x & 3u) {  // not even 4-B aligned: plain stores
        for (uint64_t i = tid; i < n; i += T) x[i] = v;
        return;
    }
    if (tid < head) x[tid] = v;
    uint4* q = reinterpret_cast<uint4*>(x + head);
    const uint64_t nq = (n - head) / 4;
    const uint4 vv = make_uint4(v, v, v, v);
    for (uint64_t i = tid; i < nq; i += T) q[i] = vv;
    for (uint64_t i = head + nq * 4 + tid; i < n; i += T) x[i] = v;
}
#define FSUB(k)                                                                          \
    do {                                                                                 \
        if (lead() && it < FS_NSUB) p.fstats[FS_SUB + 4 * it + (k)] = globaltimer();   \
    } while (0)
__global__ void __launch_bounds__(BLOCK, 4) k_dist_bfs_fused(FusedBfsP p) {
    Ctl* c = p.ctl;
    grid_begin(c);
    const RankView& r = p.r;
    const uint64_t T = gthreads(), tid = gtid();
    const uint32_t lane = lane_id();
    const uint64_t NW = p.N ? (uint64_t)p.P * r.nwl : 0;
    if (lead()) p.fstats[7] = globaltimer();  // kernel start (SX_DIST_LEVELS)
    // ---- state init (inside the timed kernel, as on one GPU), 16-B stores
    fill_u32(r.state, r.nl, INF, tid, T);  // the level output (owned rows)
    fill_u32(r.visited, r.nwl, 0u, tid, T);
    fill_u32(p.front[0], r.nwl, 0u, tid, T);
    fill_u32(p.front[1], r.nwl, 0u, tid, T);
    fill_u32(p.inbox, r.nwl, 0u, tid, T);
    fill_u32(p.gfront, NW, 0u, tid, T);
    if (tid < 8) p.slots[tid] = 0;  // counter slots, both parities (added into by every rank)
    if (!xsync(p)) return;  // every rank's window is clean before anyone writes into it
    if (tid == 0) {
        p.gfront[p.src >> 5] |= 1u << (p.src & 31);
        const uint64_t sl = (uint64_t)p.src - r.lo;
        if (sl < r.nl) {
            // the source's degree into every rank's slot[0][3] (read after the first level's
            // cross-rank barrier: m_u = m - deg(src) everywhere)
            for (uint32_t q = 0; q < p.P; ++q)
                *(unsigned long long*)ncclGetLsaPointer(p.win, p.off_cnt + 3 * 8, (int)q) = __ldg(r.deg + sl);
            r.state[sl] = 0;
            r.visited[sl >> 5] |= 1u << (sl & 31);
            p.front[0][sl >> 5] |= 1u << (sl & 31);
        }
    }
    if (!grid_sync(c)) return;
    if (lead()) p.fstats[FS_STAMPS] = globaltimer();  // end of the state init
    uint32_t it = 0, cur = 0, pulls = 0;
    uint32_t dir = p.force_dir == 2 ? DIR_PULL : DIR_PUSH;
    uint64_t m_u = p.m_total, nf_prev = 1, edges_all = 0, reached = 1;
    uint64_t mf_prev = ~0ull;  // out-edges of the current frontier (unknown for the source)
    for (;;) {
        const uint32_t lvl = it + 1;
        uint32_t* curb = p.front[cur];
        uint32_t* nxt = p.front[cur ^ 1];
        unsigned long long found = 0, mdeg = 0, edges = 0;
        if (dir == DIR_PUSH) {
            // up to 4 targets at a time (INF: none): the visited pre-tests, then the
            // claims, then the claimed vertices' updates — each group issued together
            auto visit4 = [&](const uint32_t (&u)[4]) {
                uint64_t ul[4];
                uint32_t vw[4], old[4];
                bool own[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint64_t q = u[k] == INF ? ~0ull : (uint64_t)u[k] / r.V;
                    own[k] = q == p.me;
                    ul[k] = own[k] ? (uint64_t)u[k] - r.lo : 0;
                    edges += u[k] != INF;
                    if (u[k] != INF && !own[k]) {  // V is a multiple of 32: the same bit in the owner's slice
                        uint32_t* pin =
                            (uint32_t*)ncclGetLsaPointer(p.win, p.off_in + (((uint64_t)u[k] - q * r.V) >> 5) * 4, (int)q);
                        atomicOr(pin, 1u << (u[k] & 31));
                    }
                }
                // pre-test on the non-coherent path (bits are only ever set during the
                // run, so a stale word only sends the vertex on to the atomic claim)
#pragma unroll
                for (int k = 0; k < 4; ++k) vw[k] = own[k] ? __ldg(r.visited + (ul[k] >> 5)) : FULL;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t bit = 1u << (ul[k] & 31);
                    old[k] = own[k] && !(vw[k] & bit) ? atomicOr(r.visited + (ul[k] >> 5), bit) : FULL;
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t bit = 1u << (ul[k] & 31);
                    if (old[k] & bit) continue;
                    r.state[ul[k]] = lvl;
                    atomicOr(nxt + (ul[k] >> 5), bit);
                    ++found;
                    mdeg += __ldg(r.deg + ul[k]);
                }
            };
            // edges [b, e) with stride st, 4 per lane step
            auto visit_range = [&](uint64_t b, uint64_t e, uint64_t st) {
                for (; b < e; b += 4 * st) {
                    uint32_t u[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) u[k] = b + k * st < e ? __ldg(r.ci + b + k * st) : INF;
                    visit4(u);
                }
            };
            dist_for_words(curb, r.nwl, [&](uint64_t wi, uint32_t word) {
                const uint64_t vl = (wi << 5) + lane;
                const bool mine = (word >> lane) & 1u;
                uint64_t beg = 0, end = 0;
                if (mine) {
                    beg = __ldg(r.rp + vl);
                    end = __ldg(r.rp + vl + 1);
                }
                if (mine && end - beg < r.sep_small) visit_range(beg, end, 1);  // thread granularity
                // rows of >= DIST_PIECE edges: listed as pieces for the whole grid (below),
                // the warp writing each row's items together
                for (uint32_t sp = __ballot_sync(FULL, mine && end - beg >= DIST_PIECE); sp; sp &= sp - 1) {
                    const int l = __ffs(sp) - 1;
                    const uint64_t b0 = __shfl_sync(FULL, beg, l), e0 = __shfl_sync(FULL, end, l);
                    const uint64_t vr = (wi << 5) + l;
                    const uint64_t np = (e0 - b0 + DIST_PIECE - 1) / DIST_PIECE;
                    uint64_t base = 0;
                    if (lane == 0) base = atomicAdd(r.cnt + CNT_PIECES, (unsigned long long)np);
                    base = __shfl_sync(FULL, base, 0);
                    for (uint64_t q = lane; q < np; q += 32) r.pieces[base + q] = (vr << 32) | q;
                }
                // warp granularity: medium rows, 32 lanes x 4 edges per step
                for (uint32_t todo = __ballot_sync(FULL, mine && end - beg >= r.sep_small && end - beg < DIST_PIECE);
                     todo; todo &= todo - 1) {
                    const int l = __ffs(todo) - 1;
                    const uint64_t b0 = __shfl_sync(FULL, beg, l), e0 = __shfl_sync(FULL, end, l);
                    visit_range(b0 + lane, e0, 32);
                }
            });
            FSUB(0);
            // pieces exist only if some frontier row has >= DIST_PIECE edges: not when the
            // frontier's out-edges (all ranks) are fewer — then no barrier for them either
            if (mf_prev >= DIST_PIECE) {
                if (!grid_sync(c)) return;
                const uint64_t np = vload(r.cnt + CNT_PIECES);
                for (uint64_t i = gwarp(); i < np; i += gwarps()) {  // the hub rows, one warp per piece
                    const uint64_t item = r.pieces[i];
                    const uint64_t vl = item >> 32, q = item & 0xFFFFFFFFull;
                    const uint64_t b0 = __ldg(r.rp + vl) + q * DIST_PIECE;
                    const uint64_t e0 = min(b0 + DIST_PIECE, __ldg(r.rp + vl + 1));
                    visit_range(b0 + lane, e0, 32);
                }
            }
            FSUB(1);
            if (!xsync(p)) return;  // every rank's marks are in the owners' inboxes
            FSUB(2);
            if (lead()) r.cnt[CNT_PIECES] = 0;  // read by every CTA before the barrier
            for (uint64_t w = tid; w < r.nwl; w += T) {
                curb[w] = 0;  // scanned by every CTA before the barriers above: the next level's output
                uint32_t m = p.inbox[w];
                if (!m) continue;
                p.inbox[w] = 0;
                m &= ~r.visited[w];
                if (!m) continue;
                r.visited[w] |= m;
                nxt[w] |= m;
                found += __popc(m);
                for (uint32_t x = m; x; x &= x - 1) {
                    const uint64_t ul = (w << 5) + (__ffs(x) - 1);
                    r.state[ul] = lvl;
                    mdeg += __ldg(r.deg + ul);
                }
            }
        } else {
            ++pulls;
            dist_pull_batches(r, p.gfront, nxt, lvl, found, mdeg, edges, curb);
            FSUB(0);
        }
        {
            // the CTA's counts go straight into every rank's slot[par] (peer atomics
            // through the LSA pointers): one cross-rank barrier, no local reduction line
            uint64_t a[3] = {found, mdeg, edges};
            block_sum<3>(a);
            const uint32_t par = it & 1u;
            if (threadIdx.x < p.P && (a[0] | a[1] | a[2])) {
                unsigned long long* dst =
                    (unsigned long long*)ncclGetLsaPointer(p.win, p.off_cnt + (uint64_t)par * 4 * 8, (int)threadIdx.x);
                if (a[0]) atomicAdd(dst, (unsigned long long)a[0]);
                if (a[1]) atomicAdd(dst + 1, (unsigned long long)a[1]);
                if (a[2]) atomicAdd(dst + 2, (unsigned long long)a[2]);
            }
        }
        // curb (read no more this level) is the next level's output: cleared by the
        // push's inbox fold or on the way through the pull's batches
        FSUB(3);
        if (!xsync(p)) return;
        const uint32_t par = it & 1u;
        const unsigned long long* sq = p.slots + (uint64_t)par * 4;
        if (it == 0) m_u -= vload(sq + 3);  // deg(src)
        const uint64_t nf = vload(sq), ed = vload(sq + 2);
        // push: m_f; pull: the still-open candidates' degrees = the next m_u (symmetric graphs)
        const uint64_t mf = dir == DIR_PULL ? (m_u > vload(sq + 1) ? m_u - vload(sq + 1) : 0ull) : vload(sq + 1);
        // the other parity's slot was read by every local CTA at the previous level (before
        // the barrier just crossed); the next adds into it come after the next cross-rank
        // barrier (push marks or frontier broadcast), which this store precedes
        if (lead()) {
            unsigned long long* z = p.slots + (uint64_t)(par ^ 1u) * 4;
            z[0] = z[1] = z[2] = z[3] = 0;
        }
        edges_all += ed;
        reached += nf;
        if (lead() && it + 1 < FS_NSTAMP) p.fstats[FS_STAMPS + it + 1] = globaltimer() | ((uint64_t)(dir == DIR_PULL) << 63);
        ++it;
        m_u -= mf < m_u ? mf : m_u;
        mf_prev = mf;
        cur ^= 1u;
        if (nf == 0 || (p.max_iters && it >= p.max_iters)) break;
        if (dir == DIR_PUSH) {
            if (p.force_dir == 2 || (p.force_dir == 0 && (double)mf > (double)m_u / p.alpha && nf > nf_prev)) dir = DIR_PULL;
        } else {
            if (p.force_dir == 1 || (p.force_dir == 0 && (double)nf < (double)p.N / p.beta && nf < nf_prev)) dir = DIR_PUSH;
        }
        nf_prev = nf;
        if (dir == DIR_PULL) {
            // the new frontier (front[cur] now) into every rank's global bitmap, slice me
            const uint32_t* fr = p.front[cur];
            for (uint64_t w = tid; w < r.nwl; w += T) {
                const uint32_t x = fr[w];
                for (uint32_t q = 0; q < p.P; ++q)
                    *(uint32_t*)ncclGetLsaPointer(p.win, ((uint64_t)p.me * r.nwl + w) * 4, (int)q) = x;
            }
            if (!xsync(p)) return;
        }
    }
    if (lead()) {
        p.fstats[0] = it;
        p.fstats[1] = pulls;
        p.fstats[2] = edges_all;
        p.fstats[3] = reached;
        grid_end(c);
        c->launch += 1;
    }
}


// Hub table of a rank's rows: the neighbour of largest global degree (gdeg: N
// entries, allgathered once) among a row's first 64 edges; INF for an empty row.
// With sole_ok (N <= 2^31), bit 31 marks a row whose hub is its only edge.
__global__ void k_dist_hub(const uint64_t* rp, const uint32_t* ci, uint64_t nl, const uint32_t* gdeg, uint32_t* hub,
                           bool sole_ok) {
    for (uint64_t v = gtid(); v < nl; v += gthreads()) {
        const uint64_t b = rp[v], e = min(rp[v + 1], b + 64);
        uint64_t best = 0;
        for (uint64_t x = b; x < e; ++x) {
            const uint32_t u = __ldg(ci + x);
            best = max(best, ((uint64_t)(__ldg(gdeg + u) + 1u) << 32) | (uint64_t)(~u));
        }
        hub[v] = best ? (~(uint32_t)best | (sole_ok && rp[v + 1] - b == 1 ? DHUB_SOLE : 0u)) : INF;
    }
}
__global__ void k_deg_pad(const uint32_t* deg, uint64_t nl, uint64_t V, uint32_t* out) {
    for (uint64_t i = gtid(); i < V; i += gthreads()) out[i] = i < nl ? deg[i] : 0u;
}

// ------------------------------------------------------------------ host helpers
RankView view_of(sx_dist d, int i, uint32_t cur, const sx_opts& o) {
    DistRank& k = d->r[i];
    RankView v;
    v.nl = k.nl;
    v.lo = k.lo;
    v.nwl = d->nwl;
    v.rp = k.rp;
    v.ci = k.ci;
    v.w8 = d->wbytes == 1 ? (const uint8_t*)k.w : nullptr;
    v.w32 = d->wbytes == 4 ? (const uint32_t*)k.w : nullptr;
    v.deg = k.deg;
    v.nz = k.nz;
    v.state = k.state;
    v.visited = k.visited;
    v.cur = k.front[cur];
    v.nxt = k.front[cur ^ 1];
    v.gfront = k.gfront;
    v.sendmap = k.sendmap;
    v.recv = k.recv;
    v.sendbest = k.sendbest;
    v.cnt = k.cnt;
    v.pieces = k.pieces;
    v.hub = k.hub;
    v.touched = k.touched;
    v.tcnt = k.tcnt;
    v.sendbuf = k.sendbuf;
    v.recvbuf = k.recvbuf;
    v.P = (uint32_t)d->P;
    v.V = d->V;
    v.sep_small = o.sep_small;
    return v;
}

// allreduce of the ranks' 8 counters: slot 3 is a min, the others sums
// need_min = false (BFS): the min slot is not reduced (one collective per level, not two)
sx_status reduce_counters(sx_dist d, unsigned long long (&out)[8], bool need_min = true) {
    cudaStream_t s = d->ctx->stream;
    if (d->nccl) {
        DistRank& k = d->r[0];
        // slots 0-2 and 4 are sums (slot 3, a min, is overwritten by the min reduction when needed)
        SX_NC(ncclAllReduce(k.cnt, d->dred, 5, ncclUint64, ncclSum, d->comm, s));
        if (need_min) SX_NC(ncclAllReduce(k.cnt + 3, d->dred + 3, 1, ncclUint64, ncclMin, d->comm, s));
        SX_CU(cudaMemcpyAsync(d->hcnt, d->dred, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
        SX_CU(cudaStreamSynchronize(s));
        std::memcpy(out, d->hcnt, sizeof(out));
    } else {
        for (int i = 0; i < d->nlocal; ++i)
            SX_CU(cudaMemcpyAsync(d->hcnt + 8 * i, d->r[i].cnt, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
        SX_CU(cudaStreamSynchronize(s));
        for (int j = 0; j < 8; ++j) out[j] = j == 3 ? ~0ull : 0ull;
        for (int i = 0; i < d->nlocal; ++i)
            for (int j = 0; j < 8; ++j) {
                const unsigned long long x = d->hcnt[8 * i + j];
                if (j == 3) out[j] = x < out[j] ? x : out[j];
                else out[j] += x;
            }
    }
    for (int i = 0; i < d->nlocal; ++i) {
        SX_CU(cudaMemsetAsync(d->r[i].cnt, 0, 8 * sizeof(unsigned long long), s));
        SX_CU(cudaMemsetAsync(d->r[i].cnt + 3, 0xFF, sizeof(unsigned long long), s));
    }
    return SX_OK;
}

// allgather of the owned frontier slices into every rank's global frontier bitmap
sx_status ex_allgather(sx_dist d, uint32_t cur) {
    cudaStream_t s = d->ctx->stream;
    if (d->nccl) {
        SX_NC(ncclAllGather(d->r[0].front[cur], d->r[0].gfront, d->nwl, ncclUint32, d->comm, s));
    } else {
        for (int i = 0; i < d->nlocal; ++i)
            for (int q = 0; q < d->nlocal; ++q)
                SX_CU(cudaMemcpyAsync(d->r[i].gfront + (uint64_t)q * d->nwl, d->r[q].front[cur], d->nwl * 4,
                                      cudaMemcpyDeviceToDevice, s));
    }
    return SX_OK;
}

// alltoall of per-owner slices of the push-target bitmaps
sx_status ex_alltoall(sx_dist d) {
    cudaStream_t s = d->ctx->stream;
    if (d->nccl) {
        SX_NC(ncclAlltoAll(d->r[0].sendmap, d->r[0].recv, d->nwl, ncclUint32, d->comm, s));
    } else {
        for (int i = 0; i < d->nlocal; ++i)
            for (int q = 0; q < d->nlocal; ++q)
                SX_CU(cudaMemcpyAsync(d->r[i].recv + (uint64_t)q * d->nwl, d->r[q].sendmap + (uint64_t)i * d->nwl,
                                      d->nwl * 4, cudaMemcpyDeviceToDevice, s));
    }
    return SX_OK;
}


// The pull's hub tables (once per upload): the global degree array is assembled
// (allgather of the V-padded slices; device copies for virtual ranks), then each
// rank picks its rows' hubs.
sx_status ensure_hubs(sx_dist d) {
    bool all = true;  // a re-upload drops its rank's table; then every table is rebuilt
    for (int i = 0; i < d->nlocal; ++i) all &= d->r[i].hub != nullptr;
    if (all) return SX_OK;
    for (int i = 0; i < d->nlocal; ++i)
        if (d->r[i].hub) {
            cudaFree(d->r[i].hub);
            d->r[i].hub = nullptr;
        }
    cudaStream_t s = d->ctx->stream;
    const int G = kgrid(d);
    uint32_t* gdeg = nullptr;
    sx_status rc = dmalloc(&gdeg, d->NW * 32);
    if (rc != SX_OK) return rc;
    if (d->nccl) {
        uint32_t* pad = nullptr;
        if ((rc = dmalloc(&pad, d->V)) != SX_OK) return rc;
        k_deg_pad<<<G, BLOCK, 0, s>>>(d->r[0].deg, d->r[0].nl, d->V, pad);
        SX_NC(ncclAllGather(pad, gdeg, d->V, ncclUint32, d->comm, s));
        SX_CU(cudaStreamSynchronize(s));
        cudaFree(pad);
    } else {
        for (int i = 0; i < d->nlocal; ++i)
            k_deg_pad<<<G, BLOCK, 0, s>>>(d->r[i].deg, d->r[i].nl, d->V, gdeg + (uint64_t)i * d->V);
    }
    for (int i = 0; i < d->nlocal; ++i) {
        DistRank& k = d->r[i];
        if ((rc = dmalloc(&k.hub, k.nl ? k.nl : 1)) != SX_OK) return rc;
        k_dist_hub<<<G, BLOCK, 0, s>>>(k.rp, k.ci, k.nl, gdeg, k.hub, d->N <= (1ull << 31));
    }
    SX_CU(cudaGetLastError());
    SX_CU(cudaStreamSynchronize(s));
    cudaFree(gdeg);
    return SX_OK;
}

sx_status ensure_sssp_buffers(sx_dist d) {
    const uint64_t PV = (uint64_t)d->P * d->V;
    for (int i = 0; i < d->nlocal; ++i) {
        DistRank& k = d->r[i];
        if (k.sendbest) continue;
        sx_status rc;
        if ((rc = dmalloc(&k.sendbest, PV)) != SX_OK) return rc;
        if ((rc = dmalloc(&k.touched, PV)) != SX_OK) return rc;
        if ((rc = dmalloc(&k.tcnt, 2 * (uint64_t)d->P)) != SX_OK) return rc;
        if ((rc = dmalloc(&k.sendbuf, PV)) != SX_OK) return rc;
        if ((rc = dmalloc(&k.recvbuf, PV)) != SX_OK) return rc;
        SX_CU(cudaMemsetAsync(k.sendbest, 0xFF, PV * 4, d->ctx->stream));
    }
    return SX_OK;
}

// the sparse SSSP exchange (alltoallv of (target, distance) pairs):
// per-owner counts by all-to-all, to the host (the pair transfers need them),
// then one grouped send/recv of the packed pairs.  hcounts receives, per local
// rank i, P send counts then P receive counts.
sx_status ex_sssp_pairs(sx_dist d, uint32_t* hcounts, double* pairs_out) {
    cudaStream_t s = d->ctx->stream;
    const int P = d->P;
    if (d->nccl) {
        DistRank& k = d->r[0];
        SX_NC(ncclAlltoAll(k.tcnt, k.tcnt + P, 1, ncclUint32, d->comm, s));
        SX_CU(cudaMemcpyAsync(hcounts, k.tcnt, 2 * P * 4, cudaMemcpyDeviceToHost, s));
        SX_CU(cudaStreamSynchronize(s));
        SX_NC(ncclGroupStart());
        for (int q = 0; q < P; ++q) {
            const uint32_t ns = hcounts[q], nr = hcounts[P + q];
            if (ns) SX_NC(ncclSend(k.sendbuf + (uint64_t)q * d->V, ns, ncclUint64, q, d->comm, s));
            if (nr) SX_NC(ncclRecv(k.recvbuf + (uint64_t)q * d->V, nr, ncclUint64, q, d->comm, s));
            *pairs_out += ns;
        }
        SX_NC(ncclGroupEnd());
    } else {
        for (int i = 0; i < d->nlocal; ++i)
            SX_CU(cudaMemcpyAsync(hcounts + 2 * P * i, d->r[i].tcnt, P * 4, cudaMemcpyDeviceToHost, s));
        SX_CU(cudaStreamSynchronize(s));
        for (int i = 0; i < d->nlocal; ++i) {  // owner i receives from every sender q
            for (int q = 0; q < d->nlocal; ++q) {
                const uint32_t n = hcounts[2 * P * q + i];
                hcounts[2 * P * i + P + q] = n;
                *pairs_out += n;
                if (n)
                    SX_CU(cudaMemcpyAsync(d->r[i].recvbuf + (uint64_t)q * d->V, d->r[q].sendbuf + (uint64_t)i * d->V,
                                          (uint64_t)n * 8, cudaMemcpyDeviceToDevice, s));
            }
            SX_CU(cudaMemcpyAsync(d->r[i].tcnt + P, hcounts + 2 * P * i + P, P * 4, cudaMemcpyHostToDevice, s));
        }
    }
    return SX_OK;
}

sx_status check_dist(sx_dist d) {
    if (!d) return sxh::fail(SX_E_INVALID, "NULL dist handle");
    sx_status rc = sxh::check_ctx(d->ctx);
    if (rc != SX_OK) return rc;
    for (int i = 0; i < d->nlocal; ++i)
        if (!d->r[i].rp) return sxh::fail(SX_E_INVALID, "sx_dist: a local rank's slice was not uploaded");
    return SX_OK;
}

sx_status copy_owned(sx_dist d, uint32_t* const* out) {
    cudaStream_t s = d->ctx->stream;
    for (int i = 0; i < d->nlocal; ++i)
        if (out[i] && d->r[i].nl && out[i] != d->r[i].state)
            SX_CU(cudaMemcpyAsync(out[i], d->r[i].state, d->r[i].nl * 4, cudaMemcpyDefault, s));
    SX_CU(cudaStreamSynchronize(s));
    return SX_OK;
}

// global directed edge count: one allreduce per upload
sx_status ensure_m_total(sx_dist d) {
    if (d->m_total_ok) return SX_OK;
    unsigned long long m = 0;
    for (int i = 0; i < d->nlocal; ++i) m += d->r[i].ml;
    if (d->nccl) {
        cudaStream_t s = d->ctx->stream;
        SX_CU(cudaMemcpyAsync(d->dred, &m, 8, cudaMemcpyHostToDevice, s));
        SX_NC(ncclAllReduce(d->dred, d->dred, 1, ncclUint64, ncclSum, d->comm, s));
        SX_CU(cudaMemcpyAsync(&m, d->dred, 8, cudaMemcpyDeviceToHost, s));
        SX_CU(cudaStreamSynchronize(s));
    }
    d->m_total = m;
    d->m_total_ok = true;
    return SX_OK;
}

// A device level output is written in place by the BFS kernels (no copy-out):
// the rank's state pointer is redirected for the run and restored on exit.
struct StateRedirect {
    sx_dist d;
    uint32_t* saved[DIST_MAX_LOCAL];
    StateRedirect(sx_dist d_, uint32_t* const* out) : d(d_) {
        for (int i = 0; i < d->nlocal; ++i) {
            saved[i] = d->r[i].state;
            if (out[i] && d->r[i].nl && sxh::is_device_ptr(out[i])) d->r[i].state = out[i];
        }
    }
    ~StateRedirect() {
        for (int i = 0; i < d->nlocal; ++i) d->r[i].state = saved[i];
    }
};


// Symmetric window, device communicator and control block of the fused BFS (once per dist).
sx_status fused_prepare(sx_dist d) {
    if (d->dcomm_ok) return SX_OK;
    if (!d->nccl) return sxh::fail(SX_E_INVALID, "sx_dist_bfs fusion=2: needs the NCCL backend (one rank per process)");
    const ncclTeam_t lsa = ncclTeamLsa(d->comm);
    if (lsa.nRanks != d->P)
        return sxh::fail(SX_E_NCCL, "sx_dist_bfs fusion=2: every rank must be in one LSA team (one NVLink domain)");
    d->off_in = (d->NW * 4 + 127) / 128 * 128;
    d->off_cnt = (d->off_in + d->nwl * 4 + 127) / 128 * 128;
    d->sym_bytes = (d->off_cnt + 2 * (uint64_t)d->P * 4 * 8 + 4095) / 4096 * 4096;
    SX_NC(ncclMemAlloc(&d->sym, d->sym_bytes));
    SX_NC(ncclCommWindowRegister(d->comm, d->sym, d->sym_bytes, &d->win, NCCL_WIN_COLL_SYMMETRIC));
    ncclDevCommRequirements reqs;
    std::memset(&reqs, 0, sizeof(reqs));
    reqs.lsaBarrierCount = 1;
    SX_NC(ncclDevCommCreate(d->comm, &reqs, &d->dcomm));
    d->dcomm_ok = true;
    SX_CU(cudaMalloc(&d->fctl, sizeof(Ctl)));
    SX_CU(cudaMemset(d->fctl, 0, sizeof(Ctl)));
    SX_CU(cudaMalloc(&d->fstats, FS_TOTAL * sizeof(unsigned long long)));
    return SX_OK;
}

// Enqueue one device-initiated BFS of this rank (no sync).  state: the owned
// level array the kernel writes (a device output, or the rank's own state).
sx_status enqueue_fused(sx_dist d, uint32_t src, const sx_opts& o, uint32_t* state) {
    sx_status rc = fused_prepare(d);
    if (rc != SX_OK) return rc;
    sx_ctx c = d->ctx;
    DistRank& k = d->r[0];
    // global edge count (the Beamer test needs m_u): allreduced once per upload
    if ((rc = ensure_m_total(d)) != SX_OK) return rc;
    FusedBfsP p;
    p.r = view_of(d, 0, 0, o);
    p.r.state = state;
    p.front[0] = k.front[0];
    p.front[1] = k.front[1];
    p.ctl = d->fctl;
    p.dc = d->dcomm;
    p.win = d->win;
    p.gfront = (uint32_t*)d->sym;
    p.inbox = (uint32_t*)((char*)d->sym + d->off_in);
    p.slots = (unsigned long long*)((char*)d->sym + d->off_cnt);
    p.off_in = d->off_in;
    p.off_cnt = d->off_cnt;
    p.P = (uint32_t)d->P;
    p.me = (uint32_t)d->rank0;
    p.src = src;
    p.N = d->N;
    p.m_total = d->m_total;
    p.alpha = o.alpha;
    p.beta = o.beta;
    p.force_dir = o.force_dir;
    p.max_iters = o.max_iters;
    p.fstats = d->fstats;
    if (d->fgrid == 0) {  // occupancy-sized cooperative grid, once per dist
        int per_sm = 0;
        SX_CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dist_bfs_fused, BLOCK, 0));
        d->fgrid = per_sm * c->prop.multiProcessorCount;
        if (d->fgrid <= 0) {
            d->fgrid = 0;
            return sxh::fail(SX_E_BARRIER, "fused dist BFS cannot be co-resident");
        }
    }
    void* args[] = {&p};
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_dist_bfs_fused, dim3(d->fgrid), dim3(BLOCK), args, 0,
                                                c->stream);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return sxh::cuda_fail(e, "cudaLaunchCooperativeKernel(k_dist_bfs_fused)");
    }
    return SX_OK;
}

sx_status dist_bfs_fused(sx_dist d, uint32_t src, const sx_opts& o, uint32_t* const* level_out, sx_stats* stats) {
    sx_ctx c = d->ctx;
    cudaStream_t s = c->stream;
    StateRedirect redirect(d, level_out);
    SX_CU(cudaEventRecord(c->ev0, s));
    sx_status rc = enqueue_fused(d, src, o, d->r[0].state);
    if (rc != SX_OK) return rc;
    SX_CU(cudaEventRecord(c->ev1, s));
    cudaError_t e;
    // statistics and the watchdog flag in one pinned read-back, one sync
    static const bool levels = [] { const char* v = getenv("SX_DIST_LEVELS"); return v && v[0] == '1'; }();
    const int nst = levels ? FS_TOTAL : 4;
    unsigned long long* hs = d->hcnt;
    SX_CU(cudaMemcpyAsync(hs, d->fstats, nst * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    SX_CU(cudaMemcpyAsync(hs + FS_TOTAL, &d->fctl->error, 4, cudaMemcpyDeviceToHost, s));
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        c->poisoned = true;
        return sxh::cuda_fail(e, "k_dist_bfs_fused");
    }
    if (levels) {  // SX_DIST_LEVELS=1: per-level device time of the fused kernel on stderr
        std::string line = "[sx_dist_bfs fused] init us: " + std::to_string(((hs[FS_STAMPS] & ~(1ull << 63)) - hs[7]) / 1e3) + "; levels us:";
        const uint32_t nl = (uint32_t)std::min<unsigned long long>(hs[0], FS_NSTAMP - 1);
        const unsigned long long msk = ~(1ull << 63);
        for (uint32_t i = 1; i <= nl; ++i) {
            char b[64];
            snprintf(b, sizeof(b), " it%u:%s:%.1f", i, (hs[FS_STAMPS + i] >> 63) ? "pull" : "push",
                     ((hs[FS_STAMPS + i] & msk) - (hs[FS_STAMPS + i - 1] & msk)) / 1e3);
            line += b;
            if (i - 1 < (uint32_t)FS_NSUB) {  // sub-steps (0: scan/pull, 1: pieces, 2: marks barrier, 3: fold+count)
                const unsigned long long* q = hs + FS_SUB + 4 * (i - 1);
                unsigned long long t = hs[FS_STAMPS + i - 1] & msk;
                line += " [";
                for (int k = 0; k < 4; ++k) {
                    if (!q[k] || q[k] < t) continue;
                    snprintf(b, sizeof(b), "%s%d:%.1f", k ? " " : "", k, (q[k] - t) / 1e3);
                    line += b;
                    t = q[k];
                }
                line += "]";
            }
        }
        fprintf(stderr, "%s\n", line.c_str());
    }
    if ((uint32_t)hs[FS_TOTAL]) {
        cudaMemset(d->fctl, 0, sizeof(Ctl));
        return sxh::fail(SX_E_BARRIER, "fused dist BFS: grid barrier watchdog fired");
    }
    float ms = 0;
    SX_CU(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
    if (stats) {
        std::memset(stats, 0, sizeof(*stats));
        stats->iterations = (uint32_t)hs[0];
        stats->pull_iters = (uint32_t)hs[1];
        stats->edges_examined = hs[2];
        stats->list_entries = hs[3];
        stats->launches = 1;
        stats->launches_fused = 1;
        stats->ms = ms;
        stats->ms_fused = ms;
        stats->runs = 1;
        stats->bytes_model = (double)hs[0] * (double)d->NW * 4.0;  // at most one frontier slice broadcast per level
    }
    return copy_owned(d, level_out);
}
}  // namespace

// ====================================================================== C ABI
extern "C" {

sx_status sx_nccl_unique_id(void* out128) {
    if (!out128) return sxh::fail(SX_E_INVALID, "sx_nccl_unique_id: NULL");
    ncclUniqueId id;
    SX_NC(ncclGetUniqueId(&id));
    std::memcpy(out128, &id, sizeof(id));
    return SX_OK;
}

sx_status sx_dist_create(sx_ctx ctx, uint64_t n_global, int nranks, int rank0, int nlocal, const void* nccl_id,
                         sx_dist* out) {
    if (!out) return sxh::fail(SX_E_INVALID, "sx_dist_create: out == NULL");
    *out = nullptr;
    sx_status rc = sxh::check_ctx(ctx);
    if (rc != SX_OK) return rc;
    if (nranks < 1 || nlocal < 1 || nlocal > DIST_MAX_LOCAL || rank0 < 0 || rank0 + nlocal > nranks)
        return sxh::fail(SX_E_INVALID, "sx_dist_create: bad rank layout");
    if (!(nlocal == nranks || nlocal == 1)) return sxh::fail(SX_E_INVALID, "sx_dist_create: nlocal must be 1 or nranks");
    if (nlocal == 1 && nranks > 1 && !nccl_id) return sxh::fail(SX_E_INVALID, "sx_dist_create: NCCL id required");
    if (n_global >= 0xFFFFFFFFull) return sxh::fail(SX_E_INVALID, "sx_dist_create: n >= 2^32-1");
    sx_dist d = new sx_dist_s();
    d->ctx = ctx;
    d->P = nranks;
    d->rank0 = rank0;
    d->nlocal = nlocal;
    d->N = n_global;
    d->V = ((n_global + nranks - 1) / nranks + 31) / 32 * 32;
    if (d->V == 0) d->V = 32;
    d->nwl = d->V / 32;
    d->NW = d->nwl * nranks;
    // NCCL whenever the caller supplies a communicator id with one local rank
    // (nranks = 1 included: a one-rank communicator runs every collective of the
    // data path; that is how the NCCL branch is exercised on one GPU)
    d->nccl = nlocal == 1 && nccl_id != nullptr;
    if (d->nccl) {
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof(id));
        ncclResult_t r = ncclCommInitRank(&d->comm, nranks, id, rank0);
        if (r != ncclSuccess) {
            delete d;
            return nccl_fail(r, "ncclCommInitRank");
        }
    }
    cudaError_t e = cudaMallocHost(&d->hcnt, sizeof(unsigned long long) * std::max(8 * nlocal, 96));
    if (e == cudaSuccess) e = cudaMalloc(&d->dred, 8 * sizeof(unsigned long long));
    if (e != cudaSuccess) {
        sx_dist_free(d);
        return sxh::cuda_fail(e, "sx_dist_create");
    }
    for (int i = 0; i < nlocal; ++i) {
        d->r[i].lo = (uint64_t)(rank0 + i) * d->V;
        const uint64_t hi = std::min<uint64_t>(n_global, d->r[i].lo + d->V);
        d->r[i].nl = hi > d->r[i].lo ? hi - d->r[i].lo : 0;
    }
    *out = d;
    return SX_OK;
}

sx_status sx_dist_range(sx_dist d, int local_rank, uint64_t* v_begin, uint64_t* v_end) {
    if (!d || local_rank < 0 || local_rank >= d->nlocal) return sxh::fail(SX_E_INVALID, "sx_dist_range: bad argument");
    if (v_begin) *v_begin = d->r[local_rank].lo;
    if (v_end) *v_end = d->r[local_rank].lo + d->r[local_rank].nl;
    return SX_OK;
}

sx_status sx_dist_upload(sx_dist d, int local_rank, const sx_csr_desc* desc) {
    if (!d || !desc || local_rank < 0 || local_rank >= d->nlocal)
        return sxh::fail(SX_E_INVALID, "sx_dist_upload: bad argument");
    sx_status rc = sxh::check_ctx(d->ctx);
    if (rc != SX_OK) return rc;
    DistRank& k = d->r[local_rank];
    if (desc->n != k.nl) return sxh::fail(SX_E_INVALID, "sx_dist_upload: desc->n must equal the owned row count");
    d->m_total_ok = false;
    if (desc->flags & SX_DIRECTED) return sxh::fail(SX_E_INVALID, "sx_dist_upload: symmetric graphs only (1D rows serve as in-rows)");
    if (desc->w && desc->w_bytes != 1 && desc->w_bytes != 4) return sxh::fail(SX_E_INVALID, "sx_dist_upload: w_bytes");
    if (local_rank > 0 && d->wbytes != (desc->w ? desc->w_bytes : 0))
        return sxh::fail(SX_E_INVALID, "sx_dist_upload: all slices need the same weight width");
    d->wbytes = desc->w ? desc->w_bytes : 0;
    cudaStream_t s = d->ctx->stream;
    if (k.rp) {  // re-upload (a new graph on the same partition): release the previous slice and workspace
        cudaStreamSynchronize(s);
        void* ps[] = {k.rp, k.ci, k.w, k.deg, k.nz, k.state, k.visited, k.front[0], k.front[1], k.gfront, k.sendmap,
                      k.recv, k.sendbest, k.cnt, k.pieces, k.touched, k.tcnt, k.sendbuf, k.recvbuf, k.hub};
        for (void* q : ps)
            if (q) cudaFree(q);
        const uint64_t nl = k.nl, lo = k.lo;
        k = DistRank{};
        k.nl = nl;
        k.lo = lo;
    }
    k.ml = desc->m;
    if ((rc = dmalloc(&k.rp, k.nl + 1)) != SX_OK) return rc;
    if ((rc = dmalloc(&k.ci, k.ml)) != SX_OK) return rc;
    SX_CU(cudaMemcpyAsync(k.rp, desc->row_ptr, (k.nl + 1) * 8, cudaMemcpyDefault, s));
    if (k.ml) SX_CU(cudaMemcpyAsync(k.ci, desc->col, k.ml * 4, cudaMemcpyDefault, s));
    if (desc->w) {
        if ((rc = dmalloc((char**)&k.w, k.ml * desc->w_bytes)) != SX_OK) return rc;
        if (k.ml) SX_CU(cudaMemcpyAsync(k.w, desc->w, k.ml * desc->w_bytes, cudaMemcpyDefault, s));
    }
    uint32_t* flags = nullptr;
    if ((rc = dmalloc(&flags, 1)) != SX_OK) return rc;
    SX_CU(cudaMemsetAsync(flags, 0, 4, s));
    k_validate_slice<<<kgrid(d), BLOCK, 0, s>>>(k.rp, k.ci, k.nl, k.ml, d->N, k.w, d->wbytes, flags);
    uint32_t hf = 0;
    SX_CU(cudaMemcpyAsync(&hf, flags, 4, cudaMemcpyDeviceToHost, s));
    SX_CU(cudaStreamSynchronize(s));
    cudaFree(flags);
    if (hf & 7) return sxh::fail(SX_E_INVALID, "sx_dist_upload: invalid CSR slice (row_ptr / col >= n_global)");
    k.has_zero_w = hf & 8;
    if ((rc = dmalloc(&k.deg, k.nl)) != SX_OK) return rc;
    if ((rc = dmalloc(&k.nz, d->nwl)) != SX_OK) return rc;
    k_deg_nz<<<kgrid(d), BLOCK, 0, s>>>(k.rp, k.nl, d->nwl, k.deg, k.nz);
    if ((rc = dmalloc(&k.state, d->V)) != SX_OK) return rc;
    if ((rc = dmalloc(&k.visited, d->nwl)) != SX_OK) return rc;
    for (int j = 0; j < 2; ++j)
        if ((rc = dmalloc(&k.front[j], d->nwl)) != SX_OK) return rc;
    if ((rc = dmalloc(&k.gfront, d->NW)) != SX_OK) return rc;
    if ((rc = dmalloc(&k.sendmap, d->NW)) != SX_OK) return rc;
    if ((rc = dmalloc(&k.recv, d->NW)) != SX_OK) return rc;
    if ((rc = dmalloc(&k.pieces, 2 * (k.ml / DIST_PIECE) + 2)) != SX_OK) return rc;
    if ((rc = dmalloc(&k.cnt, 8)) != SX_OK) return rc;
    SX_CU(cudaMemsetAsync(k.cnt, 0, 64, s));
    SX_CU(cudaMemsetAsync(k.cnt + 3, 0xFF, 8, s));
    SX_CU(cudaStreamSynchronize(s));
    return SX_OK;
}

void sx_dist_free(sx_dist d) {
    if (!d) return;
    cudaSetDevice(d->ctx->device);
    cudaStreamSynchronize(d->ctx->stream);
    for (cudaEvent_t& ev : d->aev)
        if (ev) cudaEventDestroy(ev);
    for (int i = 0; i < d->nlocal; ++i) {
        DistRank& k = d->r[i];
        void* ps[] = {k.rp, k.ci, k.w, k.deg, k.nz, k.state, k.visited, k.front[0], k.front[1], k.gfront, k.sendmap,
                      k.recv, k.sendbest, k.cnt, k.pieces, k.touched, k.tcnt, k.sendbuf, k.recvbuf, k.hub};
        for (void* p : ps)
            if (p) cudaFree(p);
    }
    if (d->hcnt) cudaFreeHost(d->hcnt);
    if (d->dcomm_ok) ncclDevCommDestroy(d->comm, &d->dcomm);
    if (d->win) ncclCommWindowDeregister(d->comm, d->win);
    if (d->sym) ncclMemFree(d->sym);
    if (d->fctl) cudaFree(d->fctl);
    if (d->fstats) cudaFree(d->fstats);
    if (d->dred) cudaFree(d->dred);
    if (d->comm) ncclCommDestroy(d->comm);
    delete d;
}

sx_status sx_dist_bfs(sx_dist d, uint32_t src, const sx_opts* opts, uint32_t* const* level_out, sx_stats* stats) {
    sx_status rc = check_dist(d);
    if (rc != SX_OK) return rc;
    if (!level_out) return sxh::fail(SX_E_INVALID, "sx_dist_bfs: NULL level_out");
    if (src >= d->N) return sxh::fail(SX_E_INVALID, "sx_dist_bfs: src >= n");
    const sx_opts o = sxh::resolve_opts(opts);
    if ((rc = ensure_hubs(d)) != SX_OK) return rc;
    if (o.fusion == 2) return dist_bfs_fused(d, src, o, level_out, stats);  // device-initiated (NEXT-1)
    if ((rc = ensure_m_total(d)) != SX_OK) return rc;
    sx_ctx c = d->ctx;
    cudaStream_t s = c->stream;
    const int G = kgrid(d);
    StateRedirect redirect(d, level_out);
    SX_CU(cudaEventRecord(c->ev0, s));
    // state init (no host round trip): levels INF, bitmaps zero, the source on its
    // owner, whose degree rides in counter slot 4 of the first level's reduction
    for (int i = 0; i < d->nlocal; ++i) {
        DistRank& k = d->r[i];
        SX_CU(cudaMemsetAsync(k.state, 0xFF, k.nl * 4, s));
        SX_CU(cudaMemsetAsync(k.visited, 0, d->nwl * 4, s));
        SX_CU(cudaMemsetAsync(k.front[0], 0, d->nwl * 4, s));
        SX_CU(cudaMemsetAsync(k.front[1], 0, d->nwl * 4, s));
        SX_CU(cudaMemsetAsync(k.sendmap, 0, d->NW * 4, s));
        SX_CU(cudaMemsetAsync(k.cnt, 0, 64, s));
        SX_CU(cudaMemsetAsync(k.cnt + 3, 0xFF, 8, s));
        if (src >= k.lo && src < k.lo + k.nl) k_dist_bfs_start<<<1, 32, 0, s>>>(view_of(d, i, 0, o), src);
    }
    const unsigned long long msum = d->m_total;
    unsigned long long m_u = msum, nf_prev = 1, mf_prev = ~0ull;
    uint32_t dir = o.force_dir == 2 ? DIR_PULL : DIR_PUSH, cur = 0, it = 0, launches = 0, pulls = 0;
    unsigned long long edges_total = 0, reached = 1;
    for (;;) {
        const uint32_t lvl = it + 1;
        if (dir == DIR_PUSH) {
            for (int i = 0; i < d->nlocal; ++i) {
                k_bfs_push<0><<<G, BLOCK, 0, s>>>(view_of(d, i, cur, o));
                ++launches;
                if (mf_prev >= DIST_PIECE) {  // otherwise no frontier row was split into pieces
                    k_bfs_push<1><<<G, BLOCK, 0, s>>>(view_of(d, i, cur, o));
                    ++launches;
                }
            }
            if ((rc = ex_alltoall(d)) != SX_OK) return rc;
            for (int i = 0; i < d->nlocal; ++i) {
                k_bfs_apply<<<G, BLOCK, 0, s>>>(view_of(d, i, cur, o), lvl);
                ++launches;
            }
        } else {
            if ((rc = ex_allgather(d, cur)) != SX_OK) return rc;
            for (int i = 0; i < d->nlocal; ++i) {
                k_bfs_pull<<<G, BLOCK, 0, s>>>(view_of(d, i, cur, o), lvl);
                ++launches;
            }
            ++pulls;
        }
        SX_CU(cudaGetLastError());
        unsigned long long cnt[8];
        if ((rc = reduce_counters(d, cnt, false)) != SX_OK) return rc;
        const unsigned long long nf = cnt[0];
        edges_total += cnt[2];
        reached += nf;
        if (it == 0) m_u -= cnt[4];  // deg(src), from the start kernel
        // push: cnt[1] = m_f (degrees of the found vertices); pull: cnt[1] = degrees of the
        // candidates still open = m_u of the next level (symmetric graphs), m_f = m_u - that
        const unsigned long long mf = dir == DIR_PULL ? (m_u > cnt[1] ? m_u - cnt[1] : 0ull) : cnt[1];
        ++it;
        m_u -= mf;
        mf_prev = mf;
        // the new frontier is front[cur ^ 1]; the old one (the next output) was cleared by the
        // level's apply / pull launch
        cur ^= 1;
        if (nf == 0 || (o.max_iters && it >= o.max_iters)) break;
        if (dir == DIR_PUSH) {
            if (o.force_dir == 2 || (o.force_dir == 0 && (double)mf > (double)m_u / o.alpha && nf > nf_prev)) dir = DIR_PULL;
        } else {
            if (o.force_dir == 1 || (o.force_dir == 0 && (double)nf < (double)d->N / o.beta && nf < nf_prev)) dir = DIR_PUSH;
        }
        nf_prev = nf;
    }
    SX_CU(cudaEventRecord(c->ev1, s));
    SX_CU(cudaEventSynchronize(c->ev1));
    float ms = 0;
    SX_CU(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
    if (stats) {
        std::memset(stats, 0, sizeof(*stats));
        stats->iterations = it;
        stats->launches = launches;
        stats->pull_iters = pulls;
        stats->edges_examined = edges_total;
        stats->list_entries = reached;
        stats->ms = ms;
        // bytes exchanged per rank: pull levels allgather N/8, push levels alltoall N/8 (+ counters)
        stats->bytes_model = (double)it * (double)d->NW * 4.0;
    }
    return copy_owned(d, level_out);
}

sx_status sx_dist_bfs_async(sx_dist d, uint32_t src, const sx_opts* opts, uint32_t* const* level_out) {
    sx_status rc = check_dist(d);
    if (rc != SX_OK) return rc;
    if (!level_out || !level_out[0]) return sxh::fail(SX_E_INVALID, "sx_dist_bfs_async: NULL level_out");
    if (src >= d->N) return sxh::fail(SX_E_INVALID, "sx_dist_bfs_async: src >= n");
    if (!sxh::is_device_ptr(level_out[0]))
        return sxh::fail(SX_E_INVALID, "sx_dist_bfs_async: level_out[0] must be device memory");
    if (!d->nccl || d->nlocal != 1)
        return sxh::fail(SX_E_INVALID, "sx_dist_bfs_async: needs the NCCL backend (one rank per process)");
    if ((rc = ensure_hubs(d)) != SX_OK) return rc;
    sx_opts o = sxh::resolve_opts(opts);
    o.fusion = 2;
    cudaStream_t s = d->ctx->stream;
    for (int i = 0; i < 2; ++i)
        if (!d->aev[i]) SX_CU(cudaEventCreate(&d->aev[i]));
    if (d->async_runs == 0) SX_CU(cudaEventRecord(d->aev[0], s));
    if ((rc = enqueue_fused(d, src, o, level_out[0])) != SX_OK) return rc;
    SX_CU(cudaEventRecord(d->aev[1], s));
    ++d->async_runs;
    return SX_OK;
}

sx_status sx_dist_sync(sx_dist d, sx_stats* stats) {
    sx_status rc = check_dist(d);
    if (rc != SX_OK) return rc;
    cudaStream_t s = d->ctx->stream;
    if (stats) std::memset(stats, 0, sizeof(*stats));
    if (d->async_runs == 0) {
        SX_CU(cudaStreamSynchronize(s));
        return SX_OK;
    }
    unsigned long long* hs = d->hcnt;
    SX_CU(cudaMemcpyAsync(hs, d->fstats, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    SX_CU(cudaMemcpyAsync(hs + 4, &d->fctl->error, 4, cudaMemcpyDeviceToHost, s));
    cudaError_t e = cudaStreamSynchronize(s);
    const uint32_t runs = d->async_runs;
    d->async_runs = 0;
    if (e != cudaSuccess) {
        d->ctx->poisoned = true;
        return sxh::cuda_fail(e, "sx_dist_sync");
    }
    if ((uint32_t)hs[4]) {
        cudaMemset(d->fctl, 0, sizeof(Ctl));
        return sxh::fail(SX_E_BARRIER, "fused dist BFS: grid barrier watchdog fired");
    }
    float ms = 0;
    SX_CU(cudaEventElapsedTime(&ms, d->aev[0], d->aev[1]));
    if (stats) {
        stats->iterations = (uint32_t)hs[0];  // of the last run
        stats->pull_iters = (uint32_t)hs[1];
        stats->edges_examined = hs[2];
        stats->list_entries = hs[3];
        stats->launches = runs;
        stats->launches_fused = runs;
        stats->runs = runs;
        stats->ms = ms;
        stats->ms_fused = ms;
        stats->bytes_model = (double)runs * (double)hs[0] * (double)d->NW * 4.0;
    }
    return SX_OK;
}

sx_status sx_dist_sssp(sx_dist d, uint32_t src, uint32_t delta, const sx_opts* opts, uint32_t* const* dist_out,
                       sx_stats* stats) {
    sx_status rc = check_dist(d);
    if (rc != SX_OK) return rc;
    if (!dist_out) return sxh::fail(SX_E_INVALID, "sx_dist_sssp: NULL dist_out");
    if (src >= d->N) return sxh::fail(SX_E_INVALID, "sx_dist_sssp: src >= n");
    if (d->wbytes == 0) return sxh::fail(SX_E_WEIGHT, "sx_dist_sssp: graph has no edge weights");
    for (int i = 0; i < d->nlocal; ++i)
        if (d->r[i].has_zero_w) return sxh::fail(SX_E_WEIGHT, "sx_dist_sssp: zero edge weight");
    if ((rc = ensure_sssp_buffers(d)) != SX_OK) return rc;
    const sx_opts o = sxh::resolve_opts(opts);
    sx_ctx c = d->ctx;
    cudaStream_t s = c->stream;
    const int G = kgrid(d);
    SX_CU(cudaEventRecord(c->ev0, s));
    for (int i = 0; i < d->nlocal; ++i) {
        DistRank& k = d->r[i];
        SX_CU(cudaMemsetAsync(k.state, 0xFF, d->V * 4, s));
        SX_CU(cudaMemsetAsync(k.visited, 0, d->nwl * 4, s));  // far pile
        SX_CU(cudaMemsetAsync(k.front[0], 0, d->nwl * 4, s));
        SX_CU(cudaMemsetAsync(k.front[1], 0, d->nwl * 4, s));
        SX_CU(cudaMemsetAsync(k.tcnt, 0, 2 * (uint64_t)d->P * 4, s));
        SX_CU(cudaMemsetAsync(k.cnt, 0, 64, s));
        SX_CU(cudaMemsetAsync(k.cnt + 3, 0xFF, 8, s));
        if (src >= k.lo && src < k.lo + k.nl) {
            const uint64_t sl = src - k.lo;
            const uint32_t zero = 0, bit = 1u << (sl & 31);
            SX_CU(cudaMemcpyAsync(k.state + sl, &zero, 4, cudaMemcpyHostToDevice, s));
            SX_CU(cudaMemcpyAsync(k.front[0] + (sl >> 5), &bit, 4, cudaMemcpyHostToDevice, s));
            SX_CU(cudaStreamSynchronize(s));
        }
    }
    unsigned long long hi = delta ? (unsigned long long)delta : 0x100000000ull;
    uint32_t cur = 0, it = 0, launches = 0, advances = 0;
    unsigned long long edges_total = 0;
    std::vector<uint32_t> hcounts(2 * (size_t)d->P * d->nlocal);
    double pairs = 0;
    for (;;) {
        for (int i = 0; i < d->nlocal; ++i) {
            k_sssp_push<0><<<G, BLOCK, 0, s>>>(view_of(d, i, cur, o), hi);
            k_sssp_push<1><<<G, BLOCK, 0, s>>>(view_of(d, i, cur, o), hi);
            launches += 2;
        }
        for (int i = 0; i < d->nlocal; ++i) {
            k_sssp_pack<<<G, BLOCK, 0, s>>>(view_of(d, i, cur, o));
            ++launches;
        }
        if ((rc = ex_sssp_pairs(d, hcounts.data(), &pairs)) != SX_OK) return rc;
        for (int i = 0; i < d->nlocal; ++i) {
            const RankView v = view_of(d, i, cur, o);
            k_sssp_apply_pairs<<<G, BLOCK, 0, s>>>(v, d->r[i].tcnt + d->P, hi);
            k_count_next<<<G, BLOCK, 0, s>>>(v);
            SX_CU(cudaMemsetAsync(d->r[i].tcnt, 0, d->P * 4, s));
            launches += 2;
        }
        SX_CU(cudaGetLastError());
        unsigned long long cnt[8];
        if ((rc = reduce_counters(d, cnt)) != SX_OK) return rc;
        edges_total += cnt[2];
        ++it;
        for (int i = 0; i < d->nlocal; ++i) SX_CU(cudaMemsetAsync(d->r[i].front[cur], 0, d->nwl * 4, s));
        cur ^= 1;
        unsigned long long active = cnt[0];
        if (active == 0) {
            if (delta == 0) break;
            for (int i = 0; i < d->nlocal; ++i) k_far_min<<<G, BLOCK, 0, s>>>(view_of(d, i, cur, o));
            if ((rc = reduce_counters(d, cnt)) != SX_OK) return rc;
            const unsigned long long mn = cnt[3];
            if (mn >= 0xFFFFFFFFull) break;
            hi = (mn / delta + 1) * delta;
            // move the far vertices below hi into the current frontier (front[cur])
            for (int i = 0; i < d->nlocal; ++i) {
                RankView v = view_of(d, i, cur ^ 1, o);  // nxt = front[cur]
                k_far_move<<<G, BLOCK, 0, s>>>(v, hi);
            }
            if ((rc = reduce_counters(d, cnt)) != SX_OK) return rc;
            ++advances;
            if (cnt[0] == 0) break;
        }
        if (o.max_iters && it >= o.max_iters) break;
    }
    SX_CU(cudaEventRecord(c->ev1, s));
    SX_CU(cudaEventSynchronize(c->ev1));
    float ms = 0;
    SX_CU(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
    if (stats) {
        std::memset(stats, 0, sizeof(*stats));
        stats->iterations = it;
        stats->launches = launches;
        stats->ballot_iters = advances;
        stats->edges_examined = edges_total;
        stats->ms = ms;
        stats->bytes_model = pairs * 8.0;  // (target, distance) pairs sent over the exchange
    }
    return copy_owned(d, dist_out);
}

}  // extern "C"

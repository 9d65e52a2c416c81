// internal.h — host-side structures shared by the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/simdx.h"
#include "engine.cuh"

struct sx_ctx_s {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaDeviceProp prop{};
    bool poisoned = false;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaEvent_t evp[2 * 32] = {};  // per-launch event pairs (sxh::EV_POOL)
    sx::Ctl* h_ctl = nullptr;  // pinned, device-mapped host mirror of the control block
    sx::Ctl* d_hctl = nullptr; // device address of h_ctl (the tail-copy kernel writes it directly)
    cudaMemPool_t pool = nullptr;  // stream-ordered pool of graph memory (kept, not returned to the driver)
    // runs enqueued without a host sync (sx_bfs_async): three events each
    // (before the init, between init and the fused kernel, after it), drained
    // into the owning graph's accumulators at sx_graph_sync or when the ring is full
    static constexpr int ASYNC_POOL = 64;
    cudaEvent_t eva[3 * ASYNC_POOL] = {};
    sx_graph async_g[ASYNC_POOL] = {};
    int nasync = 0;
};

struct sx_graph_s {
    sx_ctx ctx = nullptr;
    uint64_t n = 0, m = 0, mi = 0;
    bool directed = false, has_rev = true;
    uint32_t wbytes = 0;
    bool borrowed = false;
    bool gen_owned = false;   // rp/ci/w come from the embedded generator (cudaMalloc), not the ctx pool
    bool has_zero_w = false;
    // device graph arrays
    uint64_t* rp = nullptr;
    uint32_t* ci = nullptr;
    void* w = nullptr;
    uint64_t* irp = nullptr;
    uint32_t* ici = nullptr;
    void* iw = nullptr;
    uint32_t* dout = nullptr;
    uint32_t* din = nullptr;
    uint32_t* nz_in = nullptr;
    // workspace
    uint64_t nwords = 0;
    uint32_t* lists[2] = {nullptr, nullptr};
    uint32_t* bm[3] = {nullptr, nullptr, nullptr};
    uint32_t* aux_bm = nullptr;   // BFS visited / SSSP far pile
    uint32_t* cta_cnt = nullptr;
    sx::Ctl* ctl = nullptr;
    sx::TraceRec* trace = nullptr;
    uint32_t trace_cap = 0;
    uint32_t* st[4] = {nullptr, nullptr, nullptr, nullptr};  // 4N-byte state arrays
    double* hacc = nullptr;       // n+1 doubles, pull-all split-row partial sums (lazy)
    double* dstate = nullptr;     // 2n doubles, BP beliefs (lazy)
    unsigned long long* kq = nullptr;  // k-core asynchronous cascade queue (lazy)
    double* prc = nullptr;        // 5n doubles, PageRank to convergence: contrib x2, r, rho, harvested x (lazy)
    uint32_t* hub = nullptr;      // n entries, BFS hub-first probe table (built at upload)
    // sx_bfs_async bookkeeping: device stat accumulator, host-side event times
    sx::AsyncAcc* async_acc = nullptr;
    double async_ms = 0, async_ms_fused = 0;
    uint32_t async_runs = 0;
    // tiled pull-all plan (lazy, pull_all.cu)
    uint32_t* pp_hcol = nullptr;  // encoded in-edge sources (padded)
    uint32_t* pp_rs = nullptr;    // row-start bitmap over in-edges
    uint32_t* pp_hubs = nullptr;  // hub ids by slot
    uint32_t* pp_tile_seg = nullptr;
    uint32_t* pp_nzaux = nullptr;   // per active row: the operator's per-row operand
    uint32_t bfs_last_src = 0xFFFFFFFFu, bfs_last_key = 0, bfs_last_ce = 0, bfs_last_dir0 = 0xFFFFFFFFu;  // sx_bfs start-direction cache
    // degree-ordered view of the in-rows for the all-active pulls (lazy, pull_all.cu):
    // vertex ids renumbered by descending out-degree, so the most-gathered values share lines
    uint32_t* pa_order = nullptr;   // new id -> old id
    uint32_t* pa_newid = nullptr;   // old id -> new id
    uint64_t* pa_irp = nullptr;
    uint32_t* pa_ici = nullptr;
    void* pa_iw = nullptr;
    uint32_t* pa_dout = nullptr;
    uint32_t* pa_din = nullptr;
    uint32_t* pa_rs = nullptr;      // row-start bitmap over the renumbered in-edges
    uint32_t* pp_gnz = nullptr;     // per graph: rows with in-degree > 0 (+ sentinel), for the frontier pulls
    uint32_t* pp_gseg = nullptr;    // per graph: tile -> index in pp_gnz of its first edge's row
    uint64_t pp_gnnz = 0, pp_gntiles = 0;
    uint32_t pp_K = 0;
    uint64_t pp_ntiles = 0;
};

namespace sxh {

sx_status fail(sx_status st, const std::string& msg);
sx_status cuda_fail(cudaError_t e, const char* what);
#define SX_CU(call)                                              \
    do {                                                         \
        cudaError_t e__ = (call);                                \
        if (e__ != cudaSuccess) return sxh::cuda_fail(e__, #call); \
    } while (0)

sx::DevGraph dev_graph(const sx_graph g);
enum { KIND_PUSH = 0, KIND_PULL = 1, KIND_FUSED = 2 };
// BFS per-graph preparation (the hub-first probe table), run by sx_graph_upload.
sx_status bfs_prepare(sx_graph g);
// Wait for every run enqueued on the ctx without a sync and book its event times.
sx_status drain_async(sx_ctx c);
// Slot region size of a class list: NSLOT regions of R entries cover n.
inline uint32_t region_size(uint64_t n) { return (uint32_t)((n + sx::NSLOT - 1) / sx::NSLOT + 3) & ~3u; }
// Fill the scheduling parameters common to every persistent kernel.
sx::Sched make_sched(const sx_graph g, const sx_opts& o);
sx_opts resolve_opts(const sx_opts* o);
// cluster_enter == SX_CLUSTER_AUTO -> the measured default for this algorithm and size
uint32_t resolve_cluster(uint32_t ce, bool bfs, uint64_t n);

// Cooperative launch of a persistent kernel with occupancy x SMs CTAs (Eq. 1
// generalised).  Returns SX_E_BARRIER when co-residency is impossible.
sx_status coop_launch(sx_graph g, const void* fn, void** args, int* grid_out, int smem = 0);
int coop_grid(sx_graph g, const void* fn, int smem = 0);

// Device counters of one direction (deltas of the control block's st_* fields).
struct Counters {
    double entries = 0, edges = 0, reached = 0, scanned = 0, iters = 0, pull = 0, ballot = 0;
};
using BytesFn = double (*)(const sx_graph g, const Counters& c);

// Per-run bookkeeping: events, trace copy-out, stats.
constexpr int EV_POOL = 32;  // event pairs per ctx (launches in flight between two syncs)
struct Run {
    sx_graph g;
    sx_opts o;
    sx_stats* st;
    float ms_push = 0, ms_pull = 0, ms_fused = 0;
    uint32_t launches = 0, launches_push = 0, launches_pull = 0, launches_fused = 0;
    int npending = 0;
    int pend_kind[EV_POOL] = {};
    sx_status begin(bool zero_ctl = true);  // zero_ctl = false: the algorithm's init kernel zeroes it
    // Enqueue one persistent kernel (timed with an event pair); no host sync.
    // kind: KIND_PUSH / KIND_PULL (a direction phase), KIND_FUSED (all phases, fusion = 2).
    sx_status launch(const void* fn, void** args, int kind, int smem = 0);
    // Same for a non-cooperative launch with an explicit shape (e.g. one cluster).
    sx_status launch_plain(const void* fn, void** args, int grid, int block, bool pull, int smem = 0);
    // Read back the control block, accumulate the pending launches' times, check errors.
    // tail_copy = false: the kernel itself stored the control block's tail into the host mirror.
    sx_status sync(bool tail_copy = true);
    sx_status end(BytesFn bytes);
};

// Graph memory: stream-ordered allocations from the ctx's pool on the ctx
// stream.  Freed blocks stay in the pool (release threshold = max), so a
// graph upload after a free reuses them without a driver mapping (the
// cudaMalloc / cudaFree of a 2.8 GB graph cost 10-60 ms, varying run to run).
sx_status dmalloc(sx_ctx c, void** p, size_t bytes);
void dfree(sx_ctx c, void* p);
template <class T> sx_status dmalloc(sx_ctx c, T** p, size_t bytes) { return dmalloc(c, (void**)p, bytes); }

// Per-graph plan of the tiled frontier pulls (row-start bitmap, active rows, tile map); pull_all.cu.
sx_status min_pull_plan(sx_graph g);

sx_status copy_out(sx_graph g, void* dst, const void* src_dev, size_t bytes);
sx_status copy_in(sx_graph g, void* dst_dev, const void* src, size_t bytes);
sx_status check_ctx(sx_ctx c);
bool is_device_ptr(const void* p);

}  // namespace sxh

// capi.cu — contexts, graph upload/validation, launch plumbing and the common
// run bookkeeping behind include/simdx.h.
#include <cstddef>
#include <cstdio>
#include <cstring>
#include <string>

#include "internal.h"

using namespace sx;

namespace {
thread_local std::string g_last_error;
}

namespace sxh {

sx_status fail(sx_status st, const std::string& msg) {
    g_last_error = msg;
    return st;
}

sx_status cuda_fail(cudaError_t e, const char* what) {
    g_last_error = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
    if (e == cudaErrorMemoryAllocation) return SX_E_OOM;
    if (e == cudaErrorCooperativeLaunchTooLarge) return SX_E_BARRIER;
    return SX_E_CUDA;
}

sx_status check_ctx(sx_ctx c) {
    if (!c) return fail(SX_E_INVALID, "NULL context");
    if (c->poisoned) return fail(SX_E_STATE, "context poisoned by an earlier sticky CUDA error");
    SX_CU(cudaSetDevice(c->device));
    return SX_OK;
}

bool is_device_ptr(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

sx_status copy_out(sx_graph g, void* dst, const void* src_dev, size_t bytes) {
    if (bytes == 0) return SX_OK;
    SX_CU(cudaMemcpyAsync(dst, src_dev, bytes, cudaMemcpyDefault, g->ctx->stream));
    SX_CU(cudaStreamSynchronize(g->ctx->stream));
    return SX_OK;
}

sx_status copy_in(sx_graph g, void* dst_dev, const void* src, size_t bytes) {
    if (bytes == 0) return SX_OK;
    SX_CU(cudaMemcpyAsync(dst_dev, src, bytes, cudaMemcpyDefault, g->ctx->stream));
    return SX_OK;
}

DevGraph dev_graph(const sx_graph g) {
    DevGraph d;
    d.n = g->n;
    d.m = g->m;
    d.rp = g->rp;
    d.ci = g->ci;
    d.w8 = g->wbytes == 1 ? (const uint8_t*)g->w : nullptr;
    d.w32 = g->wbytes == 4 ? (const uint32_t*)g->w : nullptr;
    d.irp = g->irp;
    d.ici = g->ici;
    d.iw8 = g->wbytes == 1 ? (const uint8_t*)g->iw : nullptr;
    d.iw32 = g->wbytes == 4 ? (const uint32_t*)g->iw : nullptr;
    d.dout = g->dout;
    d.din = g->din;
    d.nz_in = g->nz_in;
    return d;
}

sx_opts resolve_opts(const sx_opts* o) {
    sx_opts r;
    sx_opts_default(&r);
    if (o) r = *o;
    // automatic cluster tail: the algorithm entry resolves it (resolve_cluster)
    if (r.overflow_threshold == 0) r.overflow_threshold = 64;
    if (r.sep_small == 0) r.sep_small = 32;
    if (r.sep_large == 0) r.sep_large = 128;
    if (r.sep_huge == 0) r.sep_huge = 16384;
    if (r.sep_large < r.sep_small) r.sep_large = r.sep_small;
    if (r.sep_huge < r.sep_large) r.sep_huge = r.sep_large;
    if (!(r.alpha > 0)) r.alpha = 60.f;
    if (!(r.beta > 0)) r.beta = 512.f;
    return r;
}

int coop_grid(sx_graph g, const void* fn, int smem) {
    int per_sm = 0;
    if (smem > 0 && cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, BLOCK, smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int grid = per_sm * g->ctx->prop.multiProcessorCount;
    if (grid > MAX_GRID) grid = MAX_GRID;
    return grid;
}

uint32_t resolve_cluster(uint32_t ce, bool bfs, uint64_t n) {
    if (ce != SX_CLUSTER_AUTO) return ce;
    // measured: the SSSP tail always pays (C2 grid 1.93x, profiles/r1/cluster_sweep.txt);
    // for BFS the tail saved 7% from the s24 hub but Graph500-style random roots
    // lose 20% (harmonic mean 387 vs 480 GTEPS, profiles/r2/bfs_roots.txt): the
    // cluster start and its hand-over to the grid cost more than the grid
    // barriers it saves, so BFS leaves it off by default
    (void)n;
    return bfs ? 0u : 4096u;
}

Sched make_sched(const sx_graph g, const sx_opts& o) {
    Sched s;
    s.ctl = g->ctl;
    s.lists[0] = g->lists[0];
    s.lists[1] = g->lists[1];
    for (int i = 0; i < 3; ++i) s.bm[i] = g->bm[i];
    s.cta_cnt = g->cta_cnt;
    s.trace = o.trace ? g->trace : nullptr;
    s.trace_cap = o.trace ? (uint32_t)std::min<uint64_t>(o.trace_cap, g->trace_cap) : 0;
    s.nwords = g->nwords;
    s.sep_small = o.sep_small;
    s.sep_large = o.sep_large;
    s.sep_huge = o.sep_huge;
    // online capacity per class: threshold x warp slots of the GPU (the paper's
    // per-thread bin of 64, aggregated per warp), split over NSLOT regions
    s.R = region_size(g->n);
    s.cstride = (uint64_t)NSLOT * s.R;
    const uint64_t warps = (uint64_t)g->ctx->prop.multiProcessorCount * (2048 / 32);
    uint64_t cap = ((uint64_t)o.overflow_threshold * warps + NSLOT - 1) / NSLOT;
    // online only / batch: regions are never capped below their size (overflow = a full region)
    if (o.force_filter == 1 || o.force_filter == 3 || cap > s.R) cap = s.R;
    s.cap_s = (uint32_t)cap;
    s.alpha = o.alpha;
    s.beta = o.beta;
    s.force_filter = o.force_filter;
    s.force_dir = o.force_dir;
    s.fusion = o.fusion;
    s.max_iters = o.max_iters;
    s.local_chain = o.local_chain;
    s.cluster_enter = o.cluster_enter;
    return s;
}

sx_status coop_launch(sx_graph g, const void* fn, void** args, int* grid_out, int smem) {
    const int grid = coop_grid(g, fn, smem);
    if (grid <= 0) return fail(SX_E_BARRIER, "persistent kernel cannot be co-resident (occupancy 0)");
    if (grid_out) *grid_out = grid;
    cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(BLOCK), args, (size_t)smem, g->ctx->stream);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return cuda_fail(e, "cudaLaunchCooperativeKernel");
    }
    return SX_OK;
}

sx_status dmalloc(sx_ctx c, void** p, size_t bytes) {
    cudaError_t e = cudaMallocFromPoolAsync(p, bytes ? bytes : 1, c->pool, c->stream);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *p = nullptr;
        return e == cudaErrorMemoryAllocation ? fail(SX_E_OOM, "device memory exhausted")
                                              : cuda_fail(e, "cudaMallocFromPoolAsync");
    }
    return SX_OK;
}

void dfree(sx_ctx c, void* p) {
    if (p) cudaFreeAsync(p, c->stream);
}

sx_status Run::begin(bool zero_ctl) {
    sx_ctx c = g->ctx;
    if (o.trace && o.trace_cap > g->trace_cap) {
        dfree(c, g->trace);
        g->trace = nullptr;
        g->trace_cap = 0;
        sx_status rc = dmalloc(c, &g->trace, o.trace_cap * sizeof(TraceRec));
        if (rc != SX_OK) return rc;
        g->trace_cap = (uint32_t)o.trace_cap;
    }
    if (zero_ctl) SX_CU(cudaMemsetAsync(g->ctl, 0, sizeof(Ctl), c->stream));
    // only the tail (from `iter` on) is ever copied back and read on the host
    constexpr size_t off = offsetof(Ctl, iter);
    std::memset(reinterpret_cast<char*>(c->h_ctl) + off, 0, sizeof(Ctl) - off);
    SX_CU(cudaEventRecord(c->ev0, c->stream));
    return SX_OK;
}

sx_status Run::launch(const void* fn, void** args, int kind, int smem) {
    sx_ctx c = g->ctx;
    if (npending == EV_POOL) {
        sx_status rc = sync();
        if (rc != SX_OK) return rc;
    }
    SX_CU(cudaEventRecord(c->evp[2 * npending], c->stream));
    sx_status rc = coop_launch(g, fn, args, nullptr, smem);
    if (rc != SX_OK) return rc;
    SX_CU(cudaEventRecord(c->evp[2 * npending + 1], c->stream));
    pend_kind[npending++] = kind;
    ++(kind == KIND_PULL ? launches_pull : kind == KIND_FUSED ? launches_fused : launches_push);
    ++launches;
    if (launches > 10000000) return fail(SX_E_STATE, "runaway launch loop");
    return SX_OK;
}

sx_status Run::launch_plain(const void* fn, void** args, int grid, int block, bool pull, int smem) {
    sx_ctx c = g->ctx;
    if (npending == EV_POOL) {
        sx_status rc = sync();
        if (rc != SX_OK) return rc;
    }
    // cluster kernels of 16 CTAs need the non-portable size opt-in (idempotent)
    SX_CU(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    if (smem > 0) SX_CU(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    SX_CU(cudaEventRecord(c->evp[2 * npending], c->stream));
    cudaError_t e = cudaLaunchKernel(fn, dim3(grid), dim3(block), args, (size_t)smem, c->stream);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return cuda_fail(e, "cudaLaunchKernel");
    }
    SX_CU(cudaEventRecord(c->evp[2 * npending + 1], c->stream));
    pend_kind[npending++] = pull ? KIND_PULL : KIND_PUSH;
    ++(pull ? launches_pull : launches_push);
    ++launches;
    return SX_OK;
}

__global__ void k_tail_copy(const Ctl* src, Ctl* dst_host) {
    constexpr size_t off = offsetof(Ctl, iter);
    constexpr size_t nw = (sizeof(Ctl) - off) / 4;
    const uint32_t* s = reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(src) + off);
    uint32_t* d = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(dst_host) + off);
    for (uint32_t i = threadIdx.x; i < nw; i += blockDim.x) d[i] = vload(s + i);
}

sx_status Run::sync(bool tail_copy) {
    sx_ctx c = g->ctx;
    // end-of-run event and the host-visible tail of the control block (from
    // `iter` on: run state, cluster line, statistics), one stream sync
    SX_CU(cudaEventRecord(c->ev1, c->stream));
    // one small kernel stores the tail into the mapped host mirror (a DMA copy of
    // these ~0.6 KB cost more per call: copy-engine start-up)
    if (tail_copy) {
        k_tail_copy<<<1, 256, 0, c->stream>>>(g->ctl, c->d_hctl);
        SX_CU(cudaGetLastError());
    }
    cudaError_t e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) {
        c->poisoned = true;
        return cuda_fail(e, "persistent kernel");
    }
    for (int i = 0; i < npending; ++i) {
        float ms = 0;
        SX_CU(cudaEventElapsedTime(&ms, c->evp[2 * i], c->evp[2 * i + 1]));
        (pend_kind[i] == KIND_PULL ? ms_pull : pend_kind[i] == KIND_FUSED ? ms_fused : ms_push) += ms;
    }
    npending = 0;
    if (c->h_ctl->error) {
        // the aborted launch left its barrier counters mid-count: start the graph's next run clean
        cudaMemsetAsync(g->ctl, 0, sizeof(Ctl), c->stream);
        cudaStreamSynchronize(c->stream);
        return fail(SX_E_BARRIER, "grid barrier watchdog fired");
    }
    return SX_OK;
}

static Counters counters_of(const Ctl::StatBlock& b) {
    Counters k;
    k.entries = (double)b.entries;
    k.edges = (double)b.edges;
    k.reached = (double)b.reached;
    k.scanned = (double)b.scanned;
    k.iters = (double)b.iters;
    k.pull = (double)b.pull;
    k.ballot = (double)b.ballot;
    return k;
}

sx_status Run::end(BytesFn bytes) {
    sx_ctx c = g->ctx;
    if (npending || launches == 0) {
        sx_status rc = sync();
        if (rc != SX_OK) return rc;
    }
    float ms = 0;  // ev1 was recorded by the last sync()
    SX_CU(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
    const Ctl& h = *c->h_ctl;
    if (st) {
        std::memset(st, 0, sizeof(*st));
        const Ctl::StatBlock& a = h.st[0];
        const Ctl::StatBlock& b = h.st[1];
        st->iterations = a.iters + b.iters;
        st->launches = launches;
        st->ballot_iters = a.ballot + b.ballot;
        st->pull_iters = a.pull + b.pull;
        st->edges_examined = a.edges + b.edges;
        st->vertices_scanned = a.scanned + b.scanned;
        st->list_entries = a.entries + b.entries;
        st->bytes_push = bytes(g, counters_of(a));
        st->bytes_pull = bytes(g, counters_of(b));
        st->bytes_model = st->bytes_push + st->bytes_pull;
        st->ms = ms;
        st->ms_push = ms_push;
        st->ms_pull = ms_pull;
        st->launches_push = launches_push;
        st->launches_pull = launches_pull;
        st->ms_fused = ms_fused;
        st->launches_fused = launches_fused;
        st->runs = 1;
    }
    if (o.trace && o.trace_cap) {
#ifdef SX_BFS_SPREAD  // profiling build: the whole buffer (per-CTA stamps live past the records)
        const uint64_t nrec = std::min<uint64_t>(o.trace_cap, g->trace_cap);
#else
        const uint64_t nrec = std::min<uint64_t>(std::min<uint64_t>(h.ntrace, o.trace_cap), g->trace_cap);
#endif
        std::memset(o.trace, 0, o.trace_cap * sizeof(sx_trace_rec));
        if (nrec) {
            SX_CU(cudaMemcpyAsync(o.trace, g->trace, nrec * sizeof(TraceRec), cudaMemcpyDefault, c->stream));
            SX_CU(cudaStreamSynchronize(c->stream));
        }
    }
    return SX_OK;
}

}  // namespace sxh

// ====================================================================== C ABI
static_assert(sizeof(sx_trace_rec) == sizeof(TraceRec), "trace record layout");

extern "C" {

const char* sx_status_str(int s) {
    switch (s) {
        case SX_OK: return "SX_OK";
        case SX_E_INVALID: return "SX_E_INVALID";
        case SX_E_OOM: return "SX_E_OOM";
        case SX_E_CUDA: return "SX_E_CUDA";
        case SX_E_NCCL: return "SX_E_NCCL";
        case SX_E_NO_REVERSE: return "SX_E_NO_REVERSE";
        case SX_E_WEIGHT: return "SX_E_WEIGHT";
        case SX_E_BARRIER: return "SX_E_BARRIER";
        case SX_E_STATE: return "SX_E_STATE";
        default: return "SX_E_UNKNOWN";
    }
}

const char* sx_last_error(void) { return g_last_error.c_str(); }

int sx_version(void) { return (0 << 16) | 1; }

void sx_opts_default(sx_opts* o) {
    if (!o) return;
    std::memset(o, 0, sizeof(*o));
    o->overflow_threshold = 64;
    o->sep_small = 32;
    o->sep_large = 128;
    o->sep_huge = 16384;
    o->alpha = 60.f;  // measured on B200 (profiles/r2/bfs_ab_sweep.txt); Beamer's CPU values are 14, 24
    o->beta = 512.f;
    o->force_filter = 0;
    o->force_dir = 0;
    o->fusion = 1;
    o->max_iters = 0;
    o->trace = nullptr;
    o->trace_cap = 0;
    o->local_chain = 0;
    o->cluster_enter = SX_CLUSTER_AUTO;
}

sx_status sx_ctx_create(int device, void* cuda_stream, sx_ctx* out) {
    if (!out) return sxh::fail(SX_E_INVALID, "sx_ctx_create: out == NULL");
    *out = nullptr;
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return sxh::fail(SX_E_CUDA, "sx_ctx_create: no CUDA device (there is no CPU fallback)");
    }
    if (device < 0 || device >= ndev) return sxh::fail(SX_E_INVALID, "sx_ctx_create: bad device index");
    SX_CU(cudaSetDevice(device));
    sx_ctx c = new sx_ctx_s();
    c->device = device;
    c->stream = (cudaStream_t)cuda_stream;
    if ((e = cudaGetDeviceProperties(&c->prop, device)) != cudaSuccess) {
        delete c;
        return sxh::cuda_fail(e, "cudaGetDeviceProperties");
    }
    if (c->prop.major < 10) {
        delete c;
        return sxh::fail(SX_E_CUDA, "sx_ctx_create: device is not sm_100 (this library is built for sm_100a only)");
    }
    if (!c->prop.cooperativeLaunch) {
        delete c;
        return sxh::fail(SX_E_BARRIER, "sx_ctx_create: device lacks cooperative launch");
    }
    for (int i = 0; i < 2 + 2 * sxh::EV_POOL; ++i) {
        cudaEvent_t* ev = i == 0 ? &c->ev0 : i == 1 ? &c->ev1 : &c->evp[i - 2];
        if ((e = cudaEventCreate(ev)) != cudaSuccess) {
            sx_ctx_destroy(c);
            return sxh::cuda_fail(e, "cudaEventCreate");
        }
    }
    for (auto& ev : c->eva) {
        if ((e = cudaEventCreate(&ev)) != cudaSuccess) {
            sx_ctx_destroy(c);
            return sxh::cuda_fail(e, "cudaEventCreate");
        }
    }
    if ((e = cudaHostAlloc(&c->h_ctl, sizeof(Ctl), cudaHostAllocMapped)) != cudaSuccess ||
        (e = cudaHostGetDevicePointer((void**)&c->d_hctl, c->h_ctl, 0)) != cudaSuccess) {
        sx_ctx_destroy(c);
        return sxh::cuda_fail(e, "cudaMallocHost");
    }
    std::memset(c->h_ctl, 0, sizeof(Ctl));
    {
        cudaMemPoolProps pp{};
        pp.allocType = cudaMemAllocationTypePinned;
        pp.handleTypes = cudaMemHandleTypeNone;
        pp.location.type = cudaMemLocationTypeDevice;
        pp.location.id = device;
        if ((e = cudaMemPoolCreate(&c->pool, &pp)) != cudaSuccess) {
            c->pool = nullptr;
            sx_ctx_destroy(c);
            return sxh::cuda_fail(e, "cudaMemPoolCreate");
        }
        uint64_t keep = ~0ull;
        cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    *out = c;
    return SX_OK;
}

void sx_ctx_destroy(sx_ctx c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    for (auto ev : c->evp)
        if (ev) cudaEventDestroy(ev);
    for (auto ev : c->eva)
        if (ev) cudaEventDestroy(ev);
    if (c->h_ctl) cudaFreeHost(c->h_ctl);
    if (c->pool) {
        cudaStreamSynchronize(c->stream);
        cudaMemPoolDestroy(c->pool);
    }
    delete c;
}

sx_status sx_ctx_info(sx_ctx c, sx_device_info* out);

}  // extern "C"

// graph.cu — graph residency: upload, validation, degree
// arrays, the in-degree>0 bitmap, and the per-graph workspace of the engine.
//
// Layout in HBM: row_ptr u64[n+1], col u32[m],
// weights u8 or u32 [m] (u32 ids, u64 indices); for symmetric graphs
// the CSR serves as CSC.  Workspace: 2 list buffers of 4 class regions
// x n u32, 3 rotating frontier bitmaps + 1 auxiliary bitmap, the control block,
// 4 state arrays of n x 4 B.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "internal.h"

using namespace sx;

namespace {

__device__ __forceinline__ bool has_zero_byte(uint32_t x) { return ((x - 0x01010101u) & ~x & 0x80808080u) != 0; }

// Validation (SPEC.md S:35-38 invariants): rows monotone, row_ptr[0] = 0 and
// row_ptr[n] = m, col < n, weights nonzero.  Edges are checked 8 ids (two
// 128-bit loads) per thread step; misaligned or short tails scalar.
__global__ void k_validate(const uint64_t* rp, const uint32_t* ci, uint64_t n, uint64_t m, const void* w,
                           uint32_t wbytes, uint32_t* flags) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
    uint32_t f = 0;
    if (t == 0 && (rp[0] != 0 || rp[n] != m)) f |= 4;
    for (uint64_t i = t; i < n; i += T) {
        const uint64_t a = rp[i], b = rp[i + 1];
        if (a > b) f |= 1;
        if (b - a >= 0xFFFFFFFFull) f |= 16;
    }
    const bool vec = ((uintptr_t)ci & 15u) == 0;
    const uint64_t n8 = vec ? m / 8 : 0;
    const uint4* c4 = reinterpret_cast<const uint4*>(ci);
    for (uint64_t q = t; q < n8; q += T) {
        const uint4 x = __ldg(c4 + 2 * q), y = __ldg(c4 + 2 * q + 1);
        if (x.x >= n || x.y >= n || x.z >= n || x.w >= n || y.x >= n || y.y >= n || y.z >= n || y.w >= n) f |= 2;
    }
    for (uint64_t e = n8 * 8 + t; e < m; e += T)
        if (ci[e] >= n) f |= 2;
    if (w) {
        if (wbytes == 1 && ((uintptr_t)w & 15u) == 0) {
            const uint64_t n16 = m / 16;
            const uint4* w4 = reinterpret_cast<const uint4*>(w);
            for (uint64_t q = t; q < n16; q += T) {
                const uint4 x = __ldg(w4 + q);
                if (has_zero_byte(x.x) || has_zero_byte(x.y) || has_zero_byte(x.z) || has_zero_byte(x.w)) f |= 8;
            }
            for (uint64_t e = n16 * 16 + t; e < m; e += T)
                if (((const uint8_t*)w)[e] == 0) f |= 8;
        } else {
            for (uint64_t e = t; e < m; e += T) {
                const uint32_t x = wbytes == 1 ? ((const uint8_t*)w)[e] : ((const uint32_t*)w)[e];
                if (x == 0) f |= 8;
            }
        }
    }
    if (f) atomicOr(flags, f);
}

__global__ void k_degrees(const uint64_t* rp, uint64_t n, uint32_t* deg) {
    const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += T)
        deg[i] = (uint32_t)(rp[i + 1] - rp[i]);
}

__global__ void k_nz_bitmap(const uint32_t* deg, uint64_t n, uint64_t nwords, uint32_t* bm) {
    const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwords; w += T) {
        uint32_t x = 0;
        for (int b = 0; b < 32; ++b) {
            const uint64_t v = (w << 5) + b;
            if (v < n && deg[v] > 0) x |= 1u << b;
        }
        bm[w] = x;
    }
}

template <class T> sx_status dalloc(sx_ctx c, T** p, size_t count) {
    return sxh::dmalloc(c, (void**)p, (count ? count : 1) * sizeof(T));
}

bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

// SX_TIMING=1: host timestamps of the upload / free phases on stderr (diagnostic;
// each mark synchronises the stream first).
struct PhaseTimer {
    bool on = getenv("SX_TIMING") != nullptr;
    cudaStream_t s;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    explicit PhaseTimer(cudaStream_t st) : s(st) {}
    void mark(const char* what) {
        if (!on) return;
        cudaStreamSynchronize(s);
        const auto t = std::chrono::steady_clock::now();
        fprintf(stderr, "[sx_timing] %-28s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(t - t0).count());
        t0 = t;
    }
};

// ---- SX_DEDUP: duplicate edges collapsed (reading 19 keeps
// duplicates by default).  Per graph, at upload: keys (row << 32 | col) sorted
// by one 64-bit radix sort (rows stay in place, each row's neighbours ascend),
// a run of equal keys keeps one edge with the run's MINIMUM weight (so shortest
// paths are unchanged), survivors are compacted by an exclusive scan, and
// row_ptr'[r] = the scan at the row's old start.
__global__ void k_dd_keys(const uint64_t* rp, const uint32_t* ci, uint64_t n, uint64_t* keys) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t r = gw; r < n; r += nw)
        for (uint64_t e = rp[r] + lane; e < rp[r + 1]; e += 32) keys[e] = (r << 32) | ci[e];
}
template <class W>
__global__ void k_dd_flags(const uint64_t* keys, const W* w, uint64_t m, uint64_t* flag, W* wmin) {
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e <= m; e += (uint64_t)gridDim.x * blockDim.x) {
        const bool head = e < m && (e == 0 || keys[e] != keys[e - 1]);
        flag[e] = head ? 1u : 0u;
        if (head && w) {  // the run's minimum weight (runs are short: the duplicates of one edge)
            W x = w[e];
            for (uint64_t f = e + 1; f < m && keys[f] == keys[e]; ++f) x = w[f] < x ? w[f] : x;
            wmin[e] = x;
        }
    }
}
template <class W>
__global__ void k_dd_scatter(const uint64_t* keys, const uint64_t* flag, const uint64_t* pos, const W* wmin, uint64_t m,
                             uint32_t* ci, W* w) {
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x)
        if (flag[e]) {
            ci[pos[e]] = (uint32_t)keys[e];
            if (w) w[pos[e]] = wmin[e];
        }
}
__global__ void k_dd_rowptr(const uint64_t* rp, const uint64_t* pos, uint64_t n, uint64_t* rp2) {
    for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r <= n; r += (uint64_t)gridDim.x * blockDim.x)
        rp2[r] = pos[rp[r]];
}

// Collapse the duplicates of one CSR (rp/ci/w owned by the graph) in place of the
// arrays: new arrays replace the old ones, *m gets the new edge count.
sx_status dedup_csr(sx_ctx ctx, uint64_t n, uint64_t* m, uint64_t** rp, uint32_t** ci, void** w, uint32_t wbytes) {
    cudaStream_t s = ctx->stream;
    const uint64_t M = *m;
    const int g = 8 * ctx->prop.multiProcessorCount;
    uint64_t *keys = nullptr, *keys2 = nullptr, *flag = nullptr, *pos = nullptr, *rp2 = nullptr;
    void *w2 = nullptr, *wmin = nullptr, *tmp = nullptr, *wn = nullptr;
    uint32_t* ci2 = nullptr;
    auto cleanup = [&]() {
        for (void* q : {(void*)keys, (void*)keys2, (void*)flag, (void*)pos, w2, wmin, tmp}) sxh::dfree(ctx, q);
    };
#define DTRY(x)                             \
    do {                                    \
        sx_status r__ = (x);                \
        if (r__ != SX_OK) {                 \
            cleanup();                      \
            return r__;                     \
        }                                   \
    } while (0)
    DTRY(sxh::dmalloc(ctx, (void**)&keys, M * 8 + 8));
    DTRY(sxh::dmalloc(ctx, (void**)&keys2, M * 8 + 8));
    DTRY(sxh::dmalloc(ctx, (void**)&flag, (M + 1) * 8));
    DTRY(sxh::dmalloc(ctx, (void**)&pos, (M + 1) * 8));
    if (*w) {
        DTRY(sxh::dmalloc(ctx, &w2, M * wbytes + 16));
        DTRY(sxh::dmalloc(ctx, &wmin, M * wbytes + 16));
    }
    k_dd_keys<<<g, 256, 0, s>>>(*rp, *ci, n, keys);
    size_t tb = 0;
    if (*w && wbytes == 1) {
        SX_CU(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys2, (const uint8_t*)*w, (uint8_t*)w2, (int64_t)M, 0, 64, s));
    } else if (*w) {
        SX_CU(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys2, (const uint32_t*)*w, (uint32_t*)w2, (int64_t)M, 0, 64, s));
    } else {
        SX_CU(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, keys2, (int64_t)M, 0, 64, s));
    }
    size_t tb2 = 0;
    SX_CU(cub::DeviceScan::ExclusiveSum(nullptr, tb2, flag, pos, (int64_t)(M + 1), s));
    DTRY(sxh::dmalloc(ctx, &tmp, std::max(tb, tb2) + 16));
    if (*w && wbytes == 1) {
        SX_CU(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys2, (const uint8_t*)*w, (uint8_t*)w2, (int64_t)M, 0, 64, s));
        k_dd_flags<uint8_t><<<g, 256, 0, s>>>(keys2, (const uint8_t*)w2, M, flag, (uint8_t*)wmin);
    } else if (*w) {
        SX_CU(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys2, (const uint32_t*)*w, (uint32_t*)w2, (int64_t)M, 0, 64, s));
        k_dd_flags<uint32_t><<<g, 256, 0, s>>>(keys2, (const uint32_t*)w2, M, flag, (uint32_t*)wmin);
    } else {
        SX_CU(cub::DeviceRadixSort::SortKeys(tmp, tb, keys, keys2, (int64_t)M, 0, 64, s));
        k_dd_flags<uint32_t><<<g, 256, 0, s>>>(keys2, (const uint32_t*)nullptr, M, flag, (uint32_t*)nullptr);
    }
    SX_CU(cub::DeviceScan::ExclusiveSum(tmp, tb2, flag, pos, (int64_t)(M + 1), s));
    uint64_t M2 = 0;
    SX_CU(cudaMemcpyAsync(&M2, pos + M, 8, cudaMemcpyDeviceToHost, s));
    SX_CU(cudaStreamSynchronize(s));
    DTRY(sxh::dmalloc(ctx, (void**)&ci2, M2 * 4 + 16));
    DTRY(sxh::dmalloc(ctx, (void**)&rp2, (n + 1) * 8 + 16));
    if (*w) DTRY(sxh::dmalloc(ctx, &wn, M2 * wbytes + 16));
    if (*w && wbytes == 1)
        k_dd_scatter<uint8_t><<<g, 256, 0, s>>>(keys2, flag, pos, (const uint8_t*)wmin, M, ci2, (uint8_t*)wn);
    else
        k_dd_scatter<uint32_t><<<g, 256, 0, s>>>(keys2, flag, pos, (const uint32_t*)wmin, M, ci2, (uint32_t*)wn);
    k_dd_rowptr<<<g, 256, 0, s>>>(*rp, pos, n, rp2);
    SX_CU(cudaGetLastError());
    SX_CU(cudaStreamSynchronize(s));
    cleanup();
#undef DTRY
    sxh::dfree(ctx, *rp);
    sxh::dfree(ctx, *ci);
    if (*w) sxh::dfree(ctx, *w);
    *rp = rp2;
    *ci = ci2;
    if (*w) *w = wn;
    *m = M2;
    return SX_OK;
}

}  // namespace

extern "C" {

sx_status sx_graph_upload(sx_ctx ctx, const sx_csr_desc* d, sx_graph* out) {
    if (!out || !d) return sxh::fail(SX_E_INVALID, "sx_graph_upload: NULL argument");
    *out = nullptr;
    sx_status rc = sxh::check_ctx(ctx);
    if (rc != SX_OK) return rc;
    if (d->n >= 0xFFFFFFFFull) return sxh::fail(SX_E_INVALID, "sx_graph_upload: n >= 2^32-1 (0xFFFFFFFF is reserved)");
    if (!d->row_ptr || (d->m && !d->col)) return sxh::fail(SX_E_INVALID, "sx_graph_upload: NULL row_ptr/col");
    if (d->w && d->w_bytes != 1 && d->w_bytes != 4) return sxh::fail(SX_E_INVALID, "sx_graph_upload: w_bytes must be 1 or 4");
    const bool directed = d->flags & SX_DIRECTED;
    const bool devp = d->flags & SX_DEVICE_PTRS;
    const bool dedup = d->flags & SX_DEDUP;  // the deduplicated arrays are the graph's own: no borrowing
    const bool borrow = !dedup && devp && (d->flags & SX_BORROW) && aligned16(d->col) &&
                        (!directed || !d->csc_idx || aligned16(d->csc_idx));
    cudaStream_t s = ctx->stream;
    PhaseTimer pt(s);
    sx_graph g = new sx_graph_s();
    g->ctx = ctx;
    g->n = d->n;
    g->m = d->m;
    g->directed = directed;
    g->wbytes = d->w ? d->w_bytes : 0;
    g->borrowed = borrow;
    const uint64_t n = d->n, m = d->m;
    auto bail = [&](sx_status st) {
        sx_graph_free(g);
        return st;
    };
#define TRY(x)                          \
    do {                                \
        sx_status r__ = (x);            \
        if (r__ != SX_OK) return bail(r__); \
    } while (0)
    auto take = [&](auto** dst, const auto* src, size_t count, size_t elem) -> sx_status {
        if (borrow) {
            *dst = (std::remove_pointer_t<decltype(dst)>)src;
            return SX_OK;
        }
        // +16 B: kernels read whole aligned 16-B groups of ids / weights (masked)
        sx_status r = dalloc(ctx, (char**)dst, count * elem + 16);
        if (r != SX_OK) return r;
        if (count) SX_CU(cudaMemcpyAsync(*dst, src, count * elem, cudaMemcpyDefault, s));
        return SX_OK;
    };
    TRY(take(&g->rp, d->row_ptr, n + 1, 8));
    TRY(take(&g->ci, d->col, m, 4));
    if (d->w) TRY(take((char**)&g->w, (const char*)d->w, m, d->w_bytes));
    pt.mark("upload: alloc + copy CSR");
    if (directed) {
        if (d->csc_ptr && d->csc_idx) {
            uint64_t mi = 0;
            if (devp) SX_CU(cudaMemcpy(&mi, d->csc_ptr + n, 8, cudaMemcpyDefault));
            else mi = d->csc_ptr[n];
            g->mi = mi;
            TRY(take(&g->irp, d->csc_ptr, n + 1, 8));
            TRY(take(&g->ici, d->csc_idx, mi, 4));
            if (d->w && d->csc_w) TRY(take((char**)&g->iw, (const char*)d->csc_w, mi, d->w_bytes));
            g->has_rev = true;
        } else {
            g->has_rev = false;
            g->irp = g->rp;
            g->ici = g->ci;
            g->iw = g->w;
            g->mi = m;
        }
    } else {
        g->irp = g->rp;
        g->ici = g->ci;
        g->iw = g->w;
        g->mi = m;
    }
    // validation (SPEC.md S:35-38 invariants) on the device
    uint32_t* dflags = nullptr;
    TRY(dalloc(ctx, &dflags, 1));
    SX_CU(cudaMemsetAsync(dflags, 0, 4, s));
    const int vb = 256, vg = 4 * ctx->prop.multiProcessorCount;
    k_validate<<<vg, vb, 0, s>>>(g->rp, g->ci, n, m, g->w, g->wbytes, dflags);
    if (directed && g->has_rev) k_validate<<<vg, vb, 0, s>>>(g->irp, g->ici, n, g->mi, g->iw, g->wbytes, dflags);
    pt.mark("upload: validate");
    uint32_t hflags = 0;
    SX_CU(cudaMemcpyAsync(&hflags, dflags, 4, cudaMemcpyDeviceToHost, s));
    cudaError_t e = cudaStreamSynchronize(s);
    sxh::dfree(ctx, dflags);
    if (e != cudaSuccess) return bail(sxh::cuda_fail(e, "graph validation"));
    if (hflags & 7) {
        char buf[160];
        snprintf(buf, sizeof buf, "sx_graph_upload: invalid CSR (%s%s%s)", (hflags & 1) ? "row_ptr decreasing; " : "",
                 (hflags & 2) ? "col >= n; " : "", (hflags & 4) ? "row_ptr[0] != 0 or row_ptr[n] != m" : "");
        return bail(sxh::fail(SX_E_INVALID, buf));
    }
    if (hflags & 16) return bail(sxh::fail(SX_E_INVALID, "sx_graph_upload: a degree exceeds 2^32-2"));
    g->has_zero_w = (hflags & 8) != 0;
    if (dedup) {  // SX_DEDUP: duplicate edges collapsed (one edge, the minimum weight)
        const bool rev = directed && g->has_rev;
        TRY(dedup_csr(ctx, n, &g->m, &g->rp, &g->ci, &g->w, g->wbytes));
        if (rev) {
            TRY(dedup_csr(ctx, n, &g->mi, &g->irp, &g->ici, &g->iw, g->wbytes));
        } else {
            g->irp = g->rp;
            g->ici = g->ci;
            g->iw = g->w;
            g->mi = g->m;
        }
        pt.mark("upload: dedup");
    }
    // degrees + in-degree>0 bitmap
    g->nwords = ((n + 31) / 32 + TILE_WORDS - 1) / TILE_WORDS * TILE_WORDS;
    if (g->nwords == 0) g->nwords = TILE_WORDS;
    TRY(dalloc(ctx, &g->dout, n));
    k_degrees<<<vg, vb, 0, s>>>(g->rp, n, g->dout);
    if (directed && g->has_rev) {
        TRY(dalloc(ctx, &g->din, n));
        k_degrees<<<vg, vb, 0, s>>>(g->irp, n, g->din);
    } else {
        g->din = g->dout;
    }
    TRY(dalloc(ctx, &g->nz_in, g->nwords));
    k_nz_bitmap<<<vg, vb, 0, s>>>(g->din, n, g->nwords, g->nz_in);
    // workspace
    pt.mark("upload: degrees + bitmap");
    for (int i = 0; i < 2; ++i) TRY(dalloc(ctx, &g->lists[i], (uint64_t)NCLS * NSLOT * sxh::region_size(n)));
    for (int i = 0; i < 3; ++i) TRY(dalloc(ctx, &g->bm[i], g->nwords));
    TRY(dalloc(ctx, &g->aux_bm, g->nwords));
    TRY(dalloc(ctx, &g->cta_cnt, NCLS * MAX_GRID));
    TRY(dalloc(ctx, (char**)&g->ctl, sizeof(Ctl)));
    // a clean control block (barrier halves, launch parity): the all-fusion BFS
    // initialises only its run state, inside the persistent launch
    SX_CU(cudaMemsetAsync(g->ctl, 0, sizeof(Ctl), s));
    for (int i = 0; i < 4; ++i) TRY(dalloc(ctx, &g->st[i], n));
    TRY(sxh::bfs_prepare(g));  // BFS hub-first probe table (graph residency, not per-run work)
    e = cudaStreamSynchronize(s);
    pt.mark("upload: workspace");
    if (e != cudaSuccess) return bail(sxh::cuda_fail(e, "graph upload"));
#undef TRY
    *out = g;
    return SX_OK;
}

sx_status sx_graph_info(sx_graph g, uint64_t* n, uint64_t* m, uint64_t* v_begin, uint64_t* v_end) {
    if (!g) return sxh::fail(SX_E_INVALID, "sx_graph_info: NULL graph");
    if (n) *n = g->n;
    if (m) *m = g->m;
    if (v_begin) *v_begin = 0;
    if (v_end) *v_end = g->n;
    return SX_OK;
}

void sx_graph_free(sx_graph g) {
    if (!g) return;
    sx_ctx c = g->ctx;
    cudaSetDevice(c->device);
    sxh::drain_async(c);  // book (and forget) enqueued async runs: none may point at g afterwards
    cudaStreamSynchronize(c->stream);
    PhaseTimer pt(c->stream);
    auto F = [&](void* p) { sxh::dfree(c, p); };
    if (!g->borrowed) {
        // generator-built arrays were cudaMalloc'ed by the embedded generator
        auto G = [&](void* p) {
            if (!p) return;
            if (g->gen_owned) cudaFree(p);
            else F(p);
        };
        if (g->irp && g->irp != g->rp) G(g->irp);
        if (g->ici && g->ici != g->ci) G(g->ici);
        if (g->iw && g->iw != g->w) G(g->iw);
        G(g->rp);
        G(g->ci);
        G(g->w);
    }
    if (g->din && g->din != g->dout) F(g->din);
    F(g->dout);
    F(g->nz_in);
    for (auto* p : g->lists) F(p);
    for (auto* p : g->bm) F(p);
    F(g->aux_bm);
    F(g->cta_cnt);
    F(g->ctl);
    F(g->trace);
    for (auto* p : g->st) F(p);
    F(g->hacc);
    F(g->dstate);
    F(g->prc);
    F(g->kq);
    F(g->hub);
    F(g->async_acc);
    F(g->pp_hcol);
    F(g->pp_rs);
    F(g->pp_hubs);
    F(g->pp_tile_seg);
    F(g->pp_nzaux);
    F(g->pp_gnz);
    F(g->pa_order);
    F(g->pa_newid);
    F(g->pa_irp);
    F(g->pa_ici);
    F(g->pa_iw);
    F(g->pa_dout);
    F(g->pa_din);
    F(g->pa_rs);
    F(g->pp_gseg);
    pt.mark("free");
    delete g;
}

}  // extern "C"

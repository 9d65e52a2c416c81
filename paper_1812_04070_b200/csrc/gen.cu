// gen.cu — synthetic graph residency without a host round trip (SURVEY.md §8(b):
// sx_graph_rmat / sx_graph_grid) and the download used by the oracle side.
//
// The generators are the shared seeded input generators of simgen/ (no method
// arithmetic: Philox-4x32-10 tuples, R-MAT recursion, relabel, grid edge ids),
// compiled into this library with SIMGEN_EMBED so their entry points stay
// internal.  The CSR they build on the device is bit-identical to simgen.c's
// (tests/test_gpu_gen.py), and is adopted by the graph (no copy).
#define SIMGEN_EMBED 1
#include "../../simgen/gpu_gen.cu"

#include <vector>

#include "internal.h"

namespace {

__global__ void k_widen_w(const uint8_t* w8, uint64_t m, uint32_t* w32) {
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x)
        w32[e] = w8[e];
}

// Adopt generator-owned device arrays as a graph (validated and prepared by sx_graph_upload).
sx_status adopt(sx_ctx ctx, uint64_t n, uint64_t m, uint64_t* rp, uint32_t* col, void* w, int wbytes, sx_graph* out) {
    sx_csr_desc d{};
    d.n = n;
    d.m = m;
    d.row_ptr = rp;
    d.col = col;
    d.w = w;
    d.w_bytes = (uint32_t)wbytes;
    d.flags = SX_DEVICE_PTRS | SX_BORROW;
    sx_status rc = sx_graph_upload(ctx, &d, out);
    if (rc != SX_OK || !(*out)->borrowed) {  // not adopted: the graph (if any) holds copies
        cudaFree(rp);
        cudaFree(col);
        if (w) cudaFree(w);
        return rc;
    }
    (*out)->borrowed = false;  // the graph now owns the generator's arrays (cudaMalloc'ed)
    (*out)->gen_owned = true;
    return SX_OK;
}

sx_status gen_fail(const char* who) {
    cudaError_t e = cudaGetLastError();
    return e != cudaSuccess ? sxh::cuda_fail(e, who) : sxh::fail(SX_E_OOM, std::string(who) + ": generator failed");
}

}  // namespace

extern "C" {

sx_status sx_graph_rmat(sx_ctx ctx, int scale, int edgefactor, uint64_t seed, uint32_t wmin, uint32_t wmax,
                        uint32_t flags, sx_graph* out) {
    if (!out) return sxh::fail(SX_E_INVALID, "sx_graph_rmat: out == NULL");
    *out = nullptr;
    sx_status rc = sxh::check_ctx(ctx);
    if (rc != SX_OK) return rc;
    if (scale < 1 || scale > 31 || edgefactor < 1)
        return sxh::fail(SX_E_INVALID, "sx_graph_rmat: need 1 <= scale <= 31 and edgefactor >= 1");
    if ((wmin || wmax) && (wmin == 0 || wmax < wmin))
        return sxh::fail(SX_E_INVALID, "sx_graph_rmat: weights need 1 <= wmin <= wmax (or 0,0 = unweighted)");
    if (flags & ~(uint32_t)SX_GEN_NO_RELABEL) return sxh::fail(SX_E_INVALID, "sx_graph_rmat: unknown flag");
    const uint64_t n = 1ull << scale;
    uint64_t* rp = nullptr;
    uint32_t* col = nullptr;
    void* w = nullptr;
    uint64_t m = 0;
    int wbytes = 0;
    if (simgen_embed::simgen_gpu_rmat_csr(scale, edgefactor, seed, wmin, wmax, (flags & SX_GEN_NO_RELABEL) ? 0 : 1, 0, n,
                                          ctx->stream, &rp, &col, &w, &m, &wbytes) != 0)
        return gen_fail("sx_graph_rmat");
    return adopt(ctx, n, m, rp, col, w, wbytes, out);
}

sx_status sx_graph_grid(sx_ctx ctx, uint32_t rows, uint32_t cols, uint64_t seed, uint32_t wmin, uint32_t wmax,
                        sx_graph* out) {
    if (!out) return sxh::fail(SX_E_INVALID, "sx_graph_grid: out == NULL");
    *out = nullptr;
    sx_status rc = sxh::check_ctx(ctx);
    if (rc != SX_OK) return rc;
    const uint64_t n = (uint64_t)rows * cols;
    if (n >= 0xFFFFFFFFull) return sxh::fail(SX_E_INVALID, "sx_graph_grid: rows*cols >= 2^32-1");
    if ((wmin || wmax) && (wmin == 0 || wmax < wmin))
        return sxh::fail(SX_E_INVALID, "sx_graph_grid: weights need 1 <= wmin <= wmax (or 0,0 = unweighted)");
    uint64_t* rp = nullptr;
    uint32_t* col = nullptr;
    void* w = nullptr;
    uint64_t m = 0;
    int wbytes = 0;
    if (simgen_embed::simgen_gpu_grid_csr(rows, cols, seed, wmin, wmax, 0, n, ctx->stream, &rp, &col, &w, &m,
                                          &wbytes) != 0)
        return gen_fail("sx_graph_grid");
    return adopt(ctx, n, m, rp, col, w, wbytes, out);
}

sx_status sx_graph_download(sx_graph g, uint64_t* row_ptr, uint32_t* col, uint32_t* w) {
    if (!g) return sxh::fail(SX_E_INVALID, "sx_graph_download: NULL graph");
    sx_status rc = sxh::check_ctx(g->ctx);
    if (rc != SX_OK) return rc;
    cudaStream_t s = g->ctx->stream;
    if (row_ptr) SX_CU(cudaMemcpyAsync(row_ptr, g->rp, (g->n + 1) * 8, cudaMemcpyDefault, s));
    if (col && g->m) SX_CU(cudaMemcpyAsync(col, g->ci, g->m * 4, cudaMemcpyDefault, s));
    if (w && g->m) {
        if (!g->w) return sxh::fail(SX_E_WEIGHT, "sx_graph_download: the graph is unweighted (pass w = NULL)");
        if (g->wbytes == 4) {
            SX_CU(cudaMemcpyAsync(w, g->w, g->m * 4, cudaMemcpyDefault, s));
        } else {
            uint32_t* tmp = nullptr;
            const bool dev = sxh::is_device_ptr(w);
            if (!dev) {
                sx_status rc2 = sxh::dmalloc(g->ctx, &tmp, g->m * 4);
                if (rc2 != SX_OK) return rc2;
            }
            k_widen_w<<<8 * g->ctx->prop.multiProcessorCount, 256, 0, s>>>((const uint8_t*)g->w, g->m, dev ? w : tmp);
            SX_CU(cudaGetLastError());
            if (!dev) {
                cudaError_t e = cudaMemcpyAsync(w, tmp, g->m * 4, cudaMemcpyDeviceToHost, s);
                if (e == cudaSuccess) e = cudaStreamSynchronize(s);
                sxh::dfree(g->ctx, tmp);
                if (e != cudaSuccess) return sxh::cuda_fail(e, "sx_graph_download");
            }
        }
    }
    SX_CU(cudaStreamSynchronize(s));
    return SX_OK;
}

}  // extern "C"

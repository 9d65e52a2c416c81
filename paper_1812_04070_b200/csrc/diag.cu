// diag.cu — the "barrier roofline": an empty persistent loop
// of grid barriers, launched exactly like the fused kernels (cooperative,
// occupancy x SMs CTAs).  Iterations x this latency is the floor of any
// iteration-bound run (C2 SSSP on the road grid, the k-core tail).
#include <cstring>

#include "internal.h"

namespace sx {

__global__ void __launch_bounds__(BLOCK, 4) barrier_loop(Ctl* c, uint32_t iters) {
    grid_begin(c);
    for (uint32_t i = 0; i < iters; ++i)
        if (!grid_sync(c)) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        grid_end(c);
        c->launch += 1;
    }
}

// Fault injection (P:707-711 deadlock, P:724-729 co-residency): CTA `skip`
// never arrives at the barrier, so the others wait until the watchdog fires;
// every CTA then leaves (the kernel ends normally, the context stays usable).
__global__ void __launch_bounds__(BLOCK, 4) barrier_skip(Ctl* c, uint32_t skip) {
    grid_begin(c);
    if (blockIdx.x == skip) return;
    grid_sync(c);
}

}  // namespace sx

using namespace sx;

extern "C" sx_status sx_barrier_fault(sx_ctx c, uint32_t mode, uint32_t timeout_ms) {
    if (mode < 1 || mode > 2 || (mode == 2 && timeout_ms == 0))
        return sxh::fail(SX_E_INVALID, "sx_barrier_fault: mode must be 1 or 2 (2 needs timeout_ms > 0)");
    sx_status rc = sxh::check_ctx(c);
    if (rc != SX_OK) return rc;
    int per_sm = 0;
    SX_CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, barrier_skip, BLOCK, 0));
    const int grid = per_sm * c->prop.multiProcessorCount;
    Ctl* d = nullptr;
    SX_CU(cudaMalloc(&d, sizeof(Ctl)));
    SX_CU(cudaMemsetAsync(d, 0, sizeof(Ctl), c->stream));
    uint32_t skip = mode == 2 ? (uint32_t)grid - 1 : 0xFFFFFFFFu;
    void* args[] = {&d, &skip};
    const unsigned long long wd = (unsigned long long)timeout_ms * 1000000ull, wd0 = 20000000000ull;
    if (mode == 2) SX_CU(cudaMemcpyToSymbolAsync(g_watchdog_ns, &wd, sizeof(wd), 0, cudaMemcpyHostToDevice, c->stream));
    // mode 1: one CTA more than can be co-resident; the driver must refuse the
    // cooperative launch (a software barrier over such a grid could deadlock)
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)barrier_skip, dim3(mode == 1 ? grid + 1 : grid),
                                                dim3(BLOCK), args, 0, c->stream);
    const cudaError_t le = e;
    if (e != cudaSuccess) cudaGetLastError();
    Ctl h{};
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e == cudaSuccess) e = cudaMemcpy(&h, d, sizeof(Ctl), cudaMemcpyDeviceToHost);
    if (mode == 2) cudaMemcpyToSymbol(g_watchdog_ns, &wd0, sizeof(wd0));
    cudaFree(d);
    if (le == cudaErrorCooperativeLaunchTooLarge) return sxh::cuda_fail(le, "cudaLaunchCooperativeKernel(grid + 1)");
    if (e != cudaSuccess) return sxh::cuda_fail(e, "barrier_skip");
    if (h.error) return sxh::fail(SX_E_BARRIER, "barrier watchdog fired");
    return SX_OK;
}

extern "C" sx_status sx_barrier_bench(sx_ctx c, uint32_t iters, double* us_per_barrier, int* ctas) {
    if (!us_per_barrier || iters == 0) return sxh::fail(SX_E_INVALID, "sx_barrier_bench: bad argument");
    sx_status rc = sxh::check_ctx(c);
    if (rc != SX_OK) return rc;
    Ctl* d = nullptr;
    SX_CU(cudaMalloc(&d, sizeof(Ctl)));
    SX_CU(cudaMemsetAsync(d, 0, sizeof(Ctl), c->stream));
    int per_sm = 0;
    SX_CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, barrier_loop, BLOCK, 0));
    const int grid = per_sm * c->prop.multiProcessorCount;
    if (ctas) *ctas = grid;
    void* args[] = {&d, &iters};
    // warm-up launch, then the timed one
    uint32_t one = 1;
    void* args1[] = {&d, &one};
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)barrier_loop, dim3(grid), dim3(BLOCK), args1, 0, c->stream);
    if (e == cudaSuccess) {
        SX_CU(cudaEventRecord(c->ev0, c->stream));
        e = cudaLaunchCooperativeKernel((const void*)barrier_loop, dim3(grid), dim3(BLOCK), args, 0, c->stream);
        SX_CU(cudaEventRecord(c->ev1, c->stream));
    }
    if (e != cudaSuccess) {
        cudaFree(d);
        return sxh::cuda_fail(e, "cudaLaunchCooperativeKernel(barrier_loop)");
    }
    e = cudaEventSynchronize(c->ev1);
    Ctl h;
    if (e == cudaSuccess) e = cudaMemcpy(&h, d, sizeof(Ctl), cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return sxh::cuda_fail(e, "barrier_loop");
    if (h.error) return sxh::fail(SX_E_BARRIER, "barrier watchdog fired");
    float ms = 0;
    SX_CU(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
    *us_per_barrier = (double)ms * 1e3 / iters;
    return SX_OK;
}

// ---------------------------------------------------------------- cluster-mode micro-benchmark
namespace sx {
__global__ void __cluster_dims__(CL_CTAS, 1, 1) __launch_bounds__(CL_BLOCK, 1)
    cluster_loop(Ctl* c, uint32_t* a, uint32_t* b, uint64_t nwords, uint32_t mode, uint32_t iters) {
    constexpr uint32_t T = CL_CTAS * CL_BLOCK;
    const uint32_t tid = cluster_rank() * CL_BLOCK + threadIdx.x;
    if (mode == 1) {
        for (uint32_t i = 0; i < iters; ++i) cluster_barrier();
        return;
    }
    if (mode >= 2) {
        uint4* z = reinterpret_cast<uint4*>(a);
        for (uint64_t q = tid; q < nwords / 4; q += T) z[q] = make_uint4(0u, 0u, 0u, 0u);
        cluster_barrier();
    }
    if (mode >= 3) {
        cluster_compact(b, nwords, tid, T, &c->cl.cnt[0], a, [](uint64_t, uint32_t w) { return w; });
        cluster_barrier();
    }
}
}  // namespace sx

extern "C" sx_status sx_cluster_bench(sx_ctx c, uint64_t nwords, uint32_t mode, uint32_t reps, double* us) {
    if (!us || reps == 0 || mode > 3) return sxh::fail(SX_E_INVALID, "sx_cluster_bench: bad argument");
    sx_status rc = sxh::check_ctx(c);
    if (rc != SX_OK) return rc;
    nwords = (nwords + TILE_WORDS - 1) / TILE_WORDS * TILE_WORDS;
    Ctl* d = nullptr;
    uint32_t *a = nullptr, *b = nullptr;
    SX_CU(cudaMalloc(&d, sizeof(Ctl)));
    SX_CU(cudaMalloc(&a, nwords * 4 + 16));
    SX_CU(cudaMalloc(&b, nwords * 4 + 16));
    SX_CU(cudaMemsetAsync(d, 0, sizeof(Ctl), c->stream));
    SX_CU(cudaMemsetAsync(b, 0, nwords * 4, c->stream));
    SX_CU(cudaFuncSetAttribute((const void*)cluster_loop, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    const uint32_t inner = mode == 1 ? reps : 1;
    const uint32_t outer = mode == 1 ? 1 : reps;
    cluster_loop<<<CL_CTAS, CL_BLOCK, 0, c->stream>>>(d, a, b, nwords, mode, 1);  // warm-up
    SX_CU(cudaEventRecord(c->ev0, c->stream));
    for (uint32_t i = 0; i < outer; ++i) cluster_loop<<<CL_CTAS, CL_BLOCK, 0, c->stream>>>(d, a, b, nwords, mode, inner);
    SX_CU(cudaEventRecord(c->ev1, c->stream));
    cudaError_t e = cudaEventSynchronize(c->ev1);
    cudaFree(d);
    cudaFree(a);
    cudaFree(b);
    if (e != cudaSuccess) return sxh::cuda_fail(e, "cluster_loop");
    float ms = 0;
    SX_CU(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
    *us = (double)ms * 1e3 / reps;
    return SX_OK;
}

// ---------------------------------------------------------------- launch-cost micro-benchmark
// GPU time per back-to-back launch of an empty kernel in the fused kernels'
// shape: mode 0 plain launch, 1 cooperative launch (occupancy x SMs CTAs of
// BLOCK threads), 2 one 16-CTA cluster — the fixed cost a launch sequence pays
// per phase, whatever the phase does.
namespace sx {
__global__ void __launch_bounds__(BLOCK, 4) k_empty(uint32_t* sink) {
    if (sink && threadIdx.x == 0 && blockIdx.x == 0xFFFFFFFFu) *sink = 1;
}
__global__ void __cluster_dims__(CL_CTAS, 1, 1) __launch_bounds__(CL_BLOCK, 1) k_empty_cluster(uint32_t* sink) {
    if (sink && threadIdx.x == 0 && blockIdx.x == 0xFFFFFFFFu) *sink = 1;
}
}  // namespace sx

extern "C" sx_status sx_launch_bench(sx_ctx c, uint32_t mode, uint32_t reps, double* us) {
    if (!us || reps == 0 || mode > 2) return sxh::fail(SX_E_INVALID, "sx_launch_bench: bad argument");
    sx_status rc = sxh::check_ctx(c);
    if (rc != SX_OK) return rc;
    int per_sm = 0;
    SX_CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_empty, BLOCK, 0));
    const int grid = per_sm * c->prop.multiProcessorCount;
    uint32_t* sink = nullptr;
    void* args[] = {&sink};
    SX_CU(cudaFuncSetAttribute((const void*)k_empty_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    auto one = [&]() -> cudaError_t {
        if (mode == 0) return cudaLaunchKernel((const void*)k_empty, dim3(grid), dim3(BLOCK), args, 0, c->stream);
        if (mode == 1) return cudaLaunchCooperativeKernel((const void*)k_empty, dim3(grid), dim3(BLOCK), args, 0, c->stream);
        return cudaLaunchKernel((const void*)k_empty_cluster, dim3(CL_CTAS), dim3(CL_BLOCK), args, 0, c->stream);
    };
    for (int i = 0; i < 3; ++i) SX_CU(one());
    SX_CU(cudaStreamSynchronize(c->stream));
    SX_CU(cudaEventRecord(c->ev0, c->stream));
    for (uint32_t i = 0; i < reps; ++i) SX_CU(one());
    SX_CU(cudaEventRecord(c->ev1, c->stream));
    SX_CU(cudaEventSynchronize(c->ev1));
    float ms = 0;
    SX_CU(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
    *us = (double)ms * 1e3 / reps;
    return SX_OK;
}

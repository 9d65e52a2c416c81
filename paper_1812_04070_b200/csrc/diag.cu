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

}  // namespace sx

using namespace sx;

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

// gpu_gen.cu — the SAME seeded R-MAT input generator as simgen.c, on the GPU
// (input generation only: no method arithmetic).  Tuple i is a function of
// (seed, i) through Philox-4x32-10 with the counters of simgen.c, so the CSR
// built here is bit-identical to simgen.rmat(...) (tests/test_gpu_gen.py).
// Used to build the scale-24..27 bench graphs (and each rank's 1D slice) in
// seconds instead of minutes, and (compiled into libsimdx with SIMGEN_EMBED,
// csrc/gen.cu) behind sx_graph_rmat / sx_graph_grid.  The grid generator is
// simgen.c's simgen_grid_csr, bit-identical (tests/test_gpu_gen.py).
//
// Pipeline (device): count the slice's directed edges -> emit (src_local<<32 | dst,
// weight) -> stable radix sort by weight, then by key (rows ordered by (col, w)
// like simgen.c) -> row_ptr by boundary fill -> col = key & 0xffffffff.
#include <cub/device/device_radix_sort.cuh>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

namespace {

__device__ __forceinline__ void philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint64_t seed, uint32_t* o) {
    uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
        const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    o[0] = c0;
    o[1] = c1;
    o[2] = c2;
    o[3] = c3;
}

__device__ __forceinline__ uint64_t mix_bits(uint64_t x, int bits) {
    if (bits <= 1) return x;
    const uint64_t mask = bits >= 64 ? ~0ull : ((1ull << bits) - 1);
    const int s = (bits + 1) / 2;
    x &= mask;
    x = (x * 0x9E3779B97F4A7C15ull) & mask;
    x ^= x >> s;
    x = (x * 0xBF58476D1CE4E5B9ull) & mask;
    x ^= x >> s;
    x = (x * 0x94D049BB133111EBull) & mask;
    x ^= x >> s;
    return x;
}

struct Gen {
    int scale;
    uint64_t seed;
    uint32_t wmin, wspan;
    int relabel, weighted;
    uint64_t M, v_lo, v_hi;
};

__device__ __forceinline__ void tuple(const Gen& g, uint64_t i, uint32_t& a, uint32_t& b, uint32_t& w) {
    const uint64_t tA = (uint64_t)(0.57 * 4294967296.0), tAB = (uint64_t)(0.76 * 4294967296.0),
                   tABC = (uint64_t)(0.95 * 4294967296.0);
    a = 0;
    b = 0;
    uint32_t r[4];
    for (int l = 0; l < g.scale; ++l) {
        if ((l & 3) == 0) philox((uint32_t)i, (uint32_t)(i >> 32), (uint32_t)(l >> 2), 0x52A7u, g.seed, r);
        const uint64_t u = r[l & 3];
        const uint32_t q = u < tA ? 0u : u < tAB ? 1u : u < tABC ? 2u : 3u;
        a = (a << 1) | (q >> 1);
        b = (b << 1) | (q & 1u);
    }
    if (g.relabel) {
        a = (uint32_t)mix_bits(a, g.scale);
        b = (uint32_t)mix_bits(b, g.scale);
    }
    w = 0;
    if (g.weighted) {
        philox((uint32_t)i, (uint32_t)(i >> 32), 0xFFFFu, 0x3E16u, g.seed, r);
        w = g.wmin + (r[0] % g.wspan);
    }
}

__global__ void k_count(Gen g, unsigned long long* total) {
    unsigned long long c = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < g.M; i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t a, b, w;
        tuple(g, i, a, b, w);
        if (a == b) continue;
        c += (a >= g.v_lo && a < g.v_hi) + (b >= g.v_lo && b < g.v_hi);
    }
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(total, c);
}

__global__ void k_emit(Gen g, unsigned long long* cursor, uint64_t* key, uint32_t* wv) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < g.M; i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t a, b, w;
        tuple(g, i, a, b, w);
        if (a == b) continue;
        if (a >= g.v_lo && a < g.v_hi) {
            const unsigned long long p = atomicAdd(cursor, 1ull);
            key[p] = ((uint64_t)(a - g.v_lo) << 32) | b;
            wv[p] = w;
        }
        if (b >= g.v_lo && b < g.v_hi) {
            const unsigned long long p = atomicAdd(cursor, 1ull);
            key[p] = ((uint64_t)(b - g.v_lo) << 32) | a;
            wv[p] = w;
        }
    }
}

// row_ptr[v] = first edge of row v (keys sorted by row); rows without edges inherit
__global__ void k_rowptr(const uint64_t* key, uint64_t m, uint64_t nl, uint64_t* rp, uint32_t* col) {
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e <= m; e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = e < m ? (key[e] >> 32) : nl;
        const uint64_t rprev = e == 0 ? 0 : (key[e - 1] >> 32) + 1;
        for (uint64_t v = (e == 0 ? 0 : rprev); v <= r && v <= nl; ++v) rp[v] = e;
        if (e < m) col[e] = (uint32_t)key[e];
    }
}

__global__ void k_narrow(const uint32_t* wv, uint64_t m, uint8_t* w8) {
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x)
        w8[e] = (uint8_t)wv[e];
}

// rows x cols 4-neighbour grid of simgen.c (simgen_grid_csr): vertex id r*cols+c,
// neighbours in increasing id (up, left, right, down), weight of undirected edge
// id e = wmin + Philox(e, 0x6121, 0x7A11)[0] % wspan.  row_ptr in closed form:
// the degree sum of all vertices before v.
struct Grid {
    uint32_t rows, cols;
    uint64_t seed;
    uint32_t wmin, wspan;
    int wbytes;
    uint64_t v_lo, v_hi;
};

__device__ __forceinline__ uint64_t grid_rp(const Grid& g, uint64_t v) {  // sum_{u < v} deg(u)
    const uint64_t r = v / g.cols, c = v % g.cols, C = g.cols, R = g.rows;
    uint64_t s = r * 2 * (C - 1) + (c ? c - 1 : 0) + c;          // horizontal: left + right neighbours
    s += (r ? (r - 1) * C : 0) + (r ? c : 0);                      // vertical: up neighbours
    s += (r < R - 1 ? r * C : (R - 1) * C) + (r + 1 < R ? c : 0);  // vertical: down neighbours
    return s;
}

__global__ void k_grid(Grid g, uint64_t* rp, uint32_t* col, void* w) {
    const uint64_t nl = g.v_hi - g.v_lo, C = g.cols;
    const uint64_t H = (uint64_t)g.rows * (C ? C - 1 : 0), base = grid_rp(g, g.v_lo);
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k <= nl; k += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t v = g.v_lo + k;
        const uint64_t p = grid_rp(g, v) - base;
        rp[k] = p;
        if (k == nl) continue;
        const uint32_t r = (uint32_t)(v / C), c = (uint32_t)(v % C);
        uint64_t nb[4], eid[4];
        int d = 0;
        if (r > 0) { nb[d] = v - C; eid[d] = H + (uint64_t)(r - 1) * C + c; ++d; }
        if (c > 0) { nb[d] = v - 1; eid[d] = (uint64_t)r * (C - 1) + (c - 1); ++d; }
        if (c + 1 < C) { nb[d] = v + 1; eid[d] = (uint64_t)r * (C - 1) + c; ++d; }
        if (r + 1 < g.rows) { nb[d] = v + C; eid[d] = H + (uint64_t)r * C + c; ++d; }
        for (int j = 0; j < d; ++j) {
            col[p + j] = (uint32_t)nb[j];
            if (g.wbytes) {
                uint32_t o[4];
                philox((uint32_t)eid[j], (uint32_t)(eid[j] >> 32), 0x6121u, 0x7A11u, g.seed, o);
                const uint32_t x = g.wmin + (o[0] % g.wspan);
                if (g.wbytes == 1) ((uint8_t*)w)[p + j] = (uint8_t)x;
                else ((uint32_t*)w)[p + j] = x;
            }
        }
    }
}

int bits_for(uint64_t x) {
    int b = 0;
    while (b < 64 && (x >> b)) ++b;
    return b;
}

}  // namespace

#define CK(x)                                                                            \
    do {                                                                                 \
        cudaError_t e__ = (x);                                                           \
        if (e__ != cudaSuccess) {                                                        \
            fprintf(stderr, "simgen_gpu: %s: %s\n", #x, cudaGetErrorString(e__));      \
            return -1;                                                                   \
        }                                                                                \
    } while (0)

// Exported C functions; with SIMGEN_EMBED (libsimdx's csrc/gen.cu) they are
// internal to the including translation unit instead.
#ifdef SIMGEN_EMBED
#define SG_BEGIN namespace simgen_embed {
#define SG_END }
#define SG_FN static
#else
#define SG_BEGIN extern "C" {
#define SG_END }
#define SG_FN
#endif

SG_BEGIN

// Build rows [v_lo, v_hi) of the undirected R-MAT graph of simgen.c on the current
// device.  Outputs are cudaMalloc'ed (free with simgen_gpu_free): row_ptr u64[nl+1],
// col u32[m], w u8[m] (wmax <= 255) or u32[m], or NULL when unweighted.  Returns 0.
SG_FN int simgen_gpu_rmat_csr(int scale, int ef, uint64_t seed, uint32_t wmin, uint32_t wmax, int relabel, uint64_t v_lo,
                        uint64_t v_hi, void* stream, uint64_t** row_ptr, uint32_t** col, void** w, uint64_t* m_out,
                        int* wbytes_out) {
    cudaStream_t s = (cudaStream_t)stream;
    Gen g;
    g.scale = scale;
    g.seed = seed;
    g.weighted = !(wmin == 0 && wmax == 0);
    g.wmin = wmin;
    g.wspan = wmax >= wmin ? wmax - wmin + 1u : 1u;
    g.relabel = relabel;
    g.M = (uint64_t)ef << scale;
    g.v_lo = v_lo;
    g.v_hi = v_hi;
    const uint64_t nl = v_hi - v_lo;
    int dev = 0, sms = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int grid = sms * 8, block = 256;
    unsigned long long* d_cnt = nullptr;
    CK(cudaMalloc(&d_cnt, 16));
    CK(cudaMemsetAsync(d_cnt, 0, 16, s));
    k_count<<<grid, block, 0, s>>>(g, d_cnt);
    unsigned long long m = 0;
    CK(cudaMemcpyAsync(&m, d_cnt, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    uint64_t *key = nullptr, *key2 = nullptr;
    uint32_t *wv = nullptr, *wv2 = nullptr;
    CK(cudaMalloc(&key, (m ? m : 1) * 8));
    CK(cudaMalloc(&key2, (m ? m : 1) * 8));
    CK(cudaMalloc(&wv, (m ? m : 1) * 4));
    CK(cudaMalloc(&wv2, (m ? m : 1) * 4));
    k_emit<<<grid, block, 0, s>>>(g, d_cnt + 1, key, wv);
    // stable LSD: by weight first, then by (row, col)
    const int kb = 32 + bits_for(nl ? nl - 1 : 0);
    const int wb = g.weighted ? bits_for(wmax) : 0;
    void* tmp = nullptr;
    size_t tmp_bytes = 0, t1 = 0, t2 = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, t1, wv, wv2, key, key2, (int64_t)m, 0, wb > 0 ? wb : 1, s));
    CK(cub::DeviceRadixSort::SortPairs(nullptr, t2, key2, key, wv2, wv, (int64_t)m, 0, kb, s));
    tmp_bytes = t1 > t2 ? t1 : t2;
    CK(cudaMalloc(&tmp, tmp_bytes ? tmp_bytes : 1));
    if (m) {
        if (wb > 0) {
            CK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, wv, wv2, key, key2, (int64_t)m, 0, wb, s));
        } else {
            CK(cudaMemcpyAsync(key2, key, m * 8, cudaMemcpyDeviceToDevice, s));
            CK(cudaMemcpyAsync(wv2, wv, m * 4, cudaMemcpyDeviceToDevice, s));
        }
        CK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, key2, key, wv2, wv, (int64_t)m, 0, kb, s));
    }
    uint64_t* rp = nullptr;
    uint32_t* c = nullptr;
    CK(cudaMalloc(&rp, (nl + 1) * 8));
    CK(cudaMalloc(&c, m * 4 + 16));  // +16 B: consumers read whole aligned 16-B groups
    k_rowptr<<<grid, block, 0, s>>>(key, m, nl, rp, c);
    void* wout = nullptr;
    int wbytes = 0;
    if (g.weighted) {
        if (wmax <= 255) {
            CK(cudaMalloc(&wout, m + 16));
            k_narrow<<<grid, block, 0, s>>>(wv, m, (uint8_t*)wout);
            wbytes = 1;
        } else {
            CK(cudaMalloc(&wout, m * 4 + 16));
            CK(cudaMemcpyAsync(wout, wv, m * 4, cudaMemcpyDeviceToDevice, s));
            wbytes = 4;
        }
    }
    CK(cudaStreamSynchronize(s));
    cudaFree(tmp);
    cudaFree(key);
    cudaFree(key2);
    cudaFree(wv);
    cudaFree(wv2);
    cudaFree(d_cnt);
    CK(cudaGetLastError());
    *row_ptr = rp;
    *col = c;
    *w = wout;
    *m_out = m;
    *wbytes_out = wbytes;
    return 0;
}

SG_FN void simgen_gpu_free(void* p) {
    if (p) cudaFree(p);
}

SG_FN int simgen_gpu_to_host(void* dst, const void* src, uint64_t bytes) {
    return cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : -1;
}

// Rows [v_lo, v_hi) of simgen.c's rows x cols grid on the current device (see
// k_grid).  Outputs cudaMalloc'ed like simgen_gpu_rmat_csr.  Returns 0.
SG_FN int simgen_gpu_grid_csr(uint32_t rows, uint32_t cols, uint64_t seed, uint32_t wmin, uint32_t wmax,
                              uint64_t v_lo, uint64_t v_hi, void* stream, uint64_t** row_ptr, uint32_t** col,
                              void** w, uint64_t* m_out, int* wbytes_out) {
    cudaStream_t s = (cudaStream_t)stream;
    Grid g;
    g.rows = rows;
    g.cols = cols;
    g.seed = seed;
    g.wmin = wmin;
    g.wspan = wmax >= wmin ? wmax - wmin + 1u : 1u;
    g.wbytes = (wmin == 0 && wmax == 0) ? 0 : (wmax <= 255 ? 1 : 4);
    g.v_lo = v_lo;
    g.v_hi = v_hi;
    const uint64_t nl = v_hi - v_lo;
    // m from the closed form (host copy of grid_rp)
    auto rp_host = [&](uint64_t v) -> uint64_t {
        const uint64_t r = v / cols, c = v % cols, C = cols, R = rows;
        uint64_t x = r * 2 * (C - 1) + (c ? c - 1 : 0) + c;
        x += (r ? (r - 1) * C : 0) + (r ? c : 0);
        x += (r < R - 1 ? r * C : (R - 1) * C) + (r + 1 < R ? c : 0);
        return x;
    };
    const uint64_t m = (rows && cols) ? rp_host(v_hi) - rp_host(v_lo) : 0;
    uint64_t* rp = nullptr;
    uint32_t* c = nullptr;
    void* wout = nullptr;
    CK(cudaMalloc(&rp, (nl + 1) * 8));
    CK(cudaMalloc(&c, m * 4 + 16));
    if (g.wbytes) CK(cudaMalloc(&wout, m * g.wbytes + 16));
    int dev = 0, sms = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (rows && cols) k_grid<<<sms * 8, 256, 0, s>>>(g, rp, c, wout);
    else CK(cudaMemsetAsync(rp, 0, (nl + 1) * 8, s));
    CK(cudaStreamSynchronize(s));
    CK(cudaGetLastError());
    *row_ptr = rp;
    *col = c;
    *w = wout;
    *m_out = m;
    *wbytes_out = g.wbytes;
    return 0;
}

SG_END

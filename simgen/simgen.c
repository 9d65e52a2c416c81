/*
 * simgen — seeded synthetic INPUT generators shared by the oracle and the
 * CUDA path (and nothing else).  This file holds none of the method's
 * arithmetic: it only produces graphs (CSR arrays) and dense input vectors.
 *
 *   - Philox-4x32-10 counter-based RNG (Salmon et al., SC'11), so that tuple i
 *     of a graph is reproducible from (seed, i) alone, on any number of threads.
 *   - Graph500-style R-MAT / Kronecker tuples, (A,B,C,D) = (.57,.19,.19,.05)
 *     (SURVEY.md §8(c) reading 20; "Graph500 generator").
 *   - a bijective xorshift-multiply relabel on `scale` bits that fixes vertex 0
 *     (so vertex 0 stays the generator's hub, a meaningful BFS/SSSP source).
 *   - a rows x cols 4-neighbour grid ("road-like").
 *   - CSR construction: symmetrise, drop self-loops, keep duplicates
 *     (reading 19), rows sorted by (col, weight) so the CSR is deterministic.
 *   - uniform f32 vectors (BP priors, SpMV x).
 *
 * Weights: uniform integers in [wmin, wmax] per input tuple (undirected edge),
 * both directions get the same weight (reading 13).
 *
 * Build: gcc -O3 -fopenmp -shared -fPIC simgen.c -o libsimgen.so
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define PHILOX_M0 0xD2511F53u
#define PHILOX_M1 0xCD9E8D57u
#define PHILOX_W0 0x9E3779B9u
#define PHILOX_W1 0xBB67AE85u

static inline void philox4x32_10(const uint32_t in[4], uint64_t seed, uint32_t out[4]) {
    uint32_t c0 = in[0], c1 = in[1], c2 = in[2], c3 = in[3];
    uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    for (int r = 0; r < 10; ++r) {
        uint64_t p0 = (uint64_t)PHILOX_M0 * c0;
        uint64_t p1 = (uint64_t)PHILOX_M1 * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += PHILOX_W0; k1 += PHILOX_W1;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* exported for the generator's own known-answer test */
void simgen_philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint64_t seed, uint32_t* out4) {
    uint32_t in[4] = {c0, c1, c2, c3};
    philox4x32_10(in, seed, out4);
}

/* bijection on [0, 2^bits) with f(0) = 0: odd multiplies and xor-shifts mod 2^bits */
static inline uint64_t mix_bits(uint64_t x, int bits) {
    if (bits <= 1) return x;
    const uint64_t mask = (bits >= 64) ? ~0ull : ((1ull << bits) - 1);
    const int s = (bits + 1) / 2;
    x &= mask;
    x = (x * 0x9E3779B97F4A7C15ull) & mask; x ^= x >> s;
    x = (x * 0xBF58476D1CE4E5B9ull) & mask; x ^= x >> s;
    x = (x * 0x94D049BB133111EBull) & mask; x ^= x >> s;
    return x;
}

uint64_t simgen_relabel(uint64_t x, int bits) { return mix_bits(x, bits); }

/*
 * R-MAT tuples [lo, hi) of the M = ef << scale tuple stream.
 * Tuple i uses Philox counters (i_lo, i_hi, j, 0x52A7) for j = 0..ceil(scale/4)-1
 * (one uniform u32 per recursion level, compared against integer thresholds)
 * and (i_lo, i_hi, 0xFFFF, 0x3E16) for its weight.
 */
void simgen_rmat_tuples(int scale, int ef, uint64_t seed, uint32_t wmin, uint32_t wmax,
                        int relabel, uint64_t lo, uint64_t hi,
                        uint32_t* src, uint32_t* dst, uint8_t* w8, uint32_t* w32) {
    (void)ef;
    /* integer quadrant thresholds: A = .57, A+B = .76, A+B+C = .95 of 2^32 */
    const uint64_t tA = (uint64_t)(0.57 * 4294967296.0);
    const uint64_t tAB = (uint64_t)(0.76 * 4294967296.0);
    const uint64_t tABC = (uint64_t)(0.95 * 4294967296.0);
    const uint32_t wspan = (wmax >= wmin) ? (wmax - wmin + 1u) : 1u;
#pragma omp parallel for schedule(static)
    for (int64_t ii = (int64_t)lo; ii < (int64_t)hi; ++ii) {
        uint64_t i = (uint64_t)ii;
        uint32_t a = 0, b = 0;
        uint32_t r[4];
        for (int l = 0; l < scale; ++l) {
            if ((l & 3) == 0) {
                uint32_t ctr[4] = {(uint32_t)i, (uint32_t)(i >> 32), (uint32_t)(l >> 2), 0x52A7u};
                philox4x32_10(ctr, seed, r);
            }
            uint64_t u = r[l & 3];
            uint32_t q = (u < tA) ? 0u : (u < tAB) ? 1u : (u < tABC) ? 2u : 3u;
            a = (a << 1) | (q >> 1);
            b = (b << 1) | (q & 1u);
        }
        if (relabel) {
            a = (uint32_t)mix_bits(a, scale);
            b = (uint32_t)mix_bits(b, scale);
        }
        uint64_t k = i - lo;
        src[k] = a;
        dst[k] = b;
        if (w8 || w32) {
            uint32_t ctr[4] = {(uint32_t)i, (uint32_t)(i >> 32), 0xFFFFu, 0x3E16u};
            philox4x32_10(ctr, seed, r);
            uint32_t w = wmin + (r[0] % wspan);
            if (w8) w8[k] = (uint8_t)w;
            if (w32) w32[k] = w;
        }
    }
}

/*
 * Degree count of the CSR rows [v_lo, v_hi) built from m tuples:
 * symmetric -> each tuple (a,b), a != b, contributes a->b and b->a;
 * directed  -> a->b only.  Self-loops are dropped.  row_ptr has v_hi-v_lo+1
 * entries and is written as an exclusive prefix sum.
 */
void simgen_csr_count(uint64_t v_lo, uint64_t v_hi, uint64_t m, const uint32_t* src,
                      const uint32_t* dst, int symmetric, uint64_t* row_ptr) {
    const uint64_t nl = v_hi - v_lo;
    memset(row_ptr, 0, (nl + 1) * sizeof(uint64_t));
#pragma omp parallel for schedule(static)
    for (int64_t ii = 0; ii < (int64_t)m; ++ii) {
        uint32_t a = src[ii], b = dst[ii];
        if (a == b) continue;
        if (a >= v_lo && a < v_hi) __atomic_fetch_add(&row_ptr[a - v_lo + 1], 1, __ATOMIC_RELAXED);
        if (symmetric && b >= v_lo && b < v_hi) __atomic_fetch_add(&row_ptr[b - v_lo + 1], 1, __ATOMIC_RELAXED);
    }
    for (uint64_t v = 0; v < nl; ++v) row_ptr[v + 1] += row_ptr[v];
}

static int cmp_u64(const void* x, const void* y) {
    uint64_t a = *(const uint64_t*)x, b = *(const uint64_t*)y;
    return (a > b) - (a < b);
}

static void sort_u64(uint64_t* a, uint64_t n) {
    if (n < 24) {
        for (uint64_t i = 1; i < n; ++i) {
            uint64_t x = a[i];
            uint64_t j = i;
            while (j > 0 && a[j - 1] > x) { a[j] = a[j - 1]; --j; }
            a[j] = x;
        }
    } else {
        qsort(a, n, sizeof(uint64_t), cmp_u64);
    }
}

/*
 * Fill col (and weights) for rows [v_lo, v_hi) given row_ptr from
 * simgen_csr_count.  Each row is sorted by (col, weight).  `w_in`/`w_out` are
 * u8 when wbytes == 1, u32 when wbytes == 4, ignored when NULL.
 */
int simgen_csr_fill(uint64_t v_lo, uint64_t v_hi, uint64_t m, const uint32_t* src,
                    const uint32_t* dst, const void* w_in, int wbytes, int symmetric,
                    const uint64_t* row_ptr, uint32_t* col, void* w_out) {
    const uint64_t nl = v_hi - v_lo;
    const uint64_t nnz = row_ptr[nl];
    uint64_t* packed = (uint64_t*)malloc((nnz ? nnz : 1) * sizeof(uint64_t));
    uint64_t* cur = (uint64_t*)malloc((nl + 1) * sizeof(uint64_t));
    if (!packed || !cur) { free(packed); free(cur); return -1; }
    memcpy(cur, row_ptr, (nl + 1) * sizeof(uint64_t));
    const uint8_t* w8 = (wbytes == 1) ? (const uint8_t*)w_in : NULL;
    const uint32_t* w32 = (wbytes == 4) ? (const uint32_t*)w_in : NULL;
#pragma omp parallel for schedule(static)
    for (int64_t ii = 0; ii < (int64_t)m; ++ii) {
        uint32_t a = src[ii], b = dst[ii];
        if (a == b) continue;
        uint64_t w = w8 ? w8[ii] : (w32 ? w32[ii] : 0);
        if (a >= v_lo && a < v_hi) {
            uint64_t p = __atomic_fetch_add(&cur[a - v_lo], 1, __ATOMIC_RELAXED);
            packed[p] = ((uint64_t)b << 32) | w;
        }
        if (symmetric && b >= v_lo && b < v_hi) {
            uint64_t p = __atomic_fetch_add(&cur[b - v_lo], 1, __ATOMIC_RELAXED);
            packed[p] = ((uint64_t)a << 32) | w;
        }
    }
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t v = 0; v < (int64_t)nl; ++v) {
        uint64_t beg = row_ptr[v], end = row_ptr[v + 1];
        sort_u64(packed + beg, end - beg);
        for (uint64_t e = beg; e < end; ++e) {
            col[e] = (uint32_t)(packed[e] >> 32);
            if (w_out) {
                uint32_t w = (uint32_t)packed[e];
                if (wbytes == 1) ((uint8_t*)w_out)[e] = (uint8_t)w;
                else ((uint32_t*)w_out)[e] = w;
            }
        }
    }
    free(packed);
    free(cur);
    return 0;
}

/*
 * rows x cols 4-neighbour grid, vertex id r*cols + c.  Undirected edge ids:
 * horizontal (r,c)-(r,c+1) -> r*(cols-1)+c ; vertical (r,c)-(r+1,c) ->
 * rows*(cols-1) + r*cols + c.  Weight of edge id e: Philox(e, 0, 0x6121, 0x7A11).
 * Rows of the CSR list neighbours in increasing id: up, left, right, down.
 * Fills rows [v_lo, v_hi); row_ptr local (v_hi - v_lo + 1 entries).
 */
void simgen_grid_csr(uint32_t rows, uint32_t cols, uint64_t seed, uint32_t wmin, uint32_t wmax,
                     uint64_t v_lo, uint64_t v_hi, uint64_t* row_ptr, uint32_t* col,
                     void* w_out, int wbytes) {
    const uint64_t nl = v_hi - v_lo;
    const uint64_t H = (uint64_t)rows * (cols ? cols - 1 : 0);
    const uint32_t wspan = (wmax >= wmin) ? (wmax - wmin + 1u) : 1u;
    /* degrees are closed-form, so the prefix sum is computed directly */
    row_ptr[0] = 0;
    for (uint64_t k = 0; k < nl; ++k) {
        uint64_t v = v_lo + k;
        uint32_t r = (uint32_t)(v / cols), c = (uint32_t)(v % cols);
        uint32_t d = (r > 0) + (c > 0) + (c + 1 < cols) + (r + 1 < rows);
        row_ptr[k + 1] = row_ptr[k] + d;
    }
#pragma omp parallel for schedule(static)
    for (int64_t kk = 0; kk < (int64_t)nl; ++kk) {
        uint64_t v = v_lo + (uint64_t)kk;
        uint32_t r = (uint32_t)(v / cols), c = (uint32_t)(v % cols);
        uint64_t p = row_ptr[kk];
        uint64_t nb[4], eid[4];
        int d = 0;
        if (r > 0) { nb[d] = v - cols; eid[d] = H + (uint64_t)(r - 1) * cols + c; ++d; }
        if (c > 0) { nb[d] = v - 1; eid[d] = (uint64_t)r * (cols - 1) + (c - 1); ++d; }
        if (c + 1 < cols) { nb[d] = v + 1; eid[d] = (uint64_t)r * (cols - 1) + c; ++d; }
        if (r + 1 < rows) { nb[d] = v + cols; eid[d] = H + (uint64_t)r * cols + c; ++d; }
        for (int j = 0; j < d; ++j) {
            col[p + j] = (uint32_t)nb[j];
            if (w_out) {
                uint32_t ctr[4] = {(uint32_t)eid[j], (uint32_t)(eid[j] >> 32), 0x6121u, 0x7A11u};
                uint32_t o[4];
                philox4x32_10(ctr, seed, o);
                uint32_t w = wmin + (o[0] % wspan);
                if (wbytes == 1) ((uint8_t*)w_out)[p + j] = (uint8_t)w;
                else ((uint32_t*)w_out)[p + j] = w;
            }
        }
    }
}

/* out[i] = lo + (hi - lo) * u_i, u_i = (Philox(i, 0, 0xB9, stream) >> 8) * 2^-24 in [0,1) */
void simgen_uniform_f32(uint64_t seed, uint32_t stream, uint64_t n, float lo, float hi, float* out) {
#pragma omp parallel for schedule(static)
    for (int64_t ii = 0; ii < (int64_t)n; ++ii) {
        uint64_t i = (uint64_t)ii;
        uint32_t ctr[4] = {(uint32_t)i, (uint32_t)(i >> 32), 0xB9u, stream};
        uint32_t o[4];
        philox4x32_10(ctr, seed, o);
        float u = (float)(o[0] >> 8) * (1.0f / 16777216.0f);
        out[i] = lo + (hi - lo) * u;
    }
}

/*
 * simdx.h — C ABI of the B200-native SIMD-X ACC frontier engine
 * (arXiv 1812.04070; PAPER.md lines cited as P:<n>).
 *
 * The library runs ONE data-parallel hot path: the per-iteration
 * Active-Compute-Combine (ACC) frontier step over a CSR/CSC graph
 * (P:913), with just-in-time task management (online + ballot filters and
 * thread/warp/CTA degree binning), the push/pull direction switch
 * and push/pull selective kernel fusion held together by a deadlock-free grid
 * barrier.  Every step runs in hand-written sm_100a CUDA kernels;
 * there is no CPU fallback: without a usable CUDA device every call returns
 * SX_E_CUDA.
 *
 * Conventions (all functions):
 *   - extern "C", no C++ exceptions cross the ABI, nothing aborts the process.
 *   - Return an sx_status; on failure sx_last_error() holds a thread-local
 *     detail string valid until the next call on that thread.
 *   - A sticky CUDA error (e.g. an illegal address) poisons the context: every
 *     later call on it returns SX_E_STATE.
 *   - Vertex ids are uint32; n must be < 2^32-1 because 0xFFFFFFFF is
 *     the "unreached / unset" sentinel.  Edge indices are uint64.
 *   - A context is single-threaded (one host thread at a time); distinct
 *     contexts are independent.  All work runs on the context's stream and
 *     every algorithm call synchronises that stream before returning, so
 *     output buffers are valid on return.
 *   - Output pointers may be host or device memory (detected with
 *     cudaPointerGetAttributes); the caller allocates them.
 */
#ifndef SIMDX_H
#define SIMDX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SX_OK = 0,
    SX_E_INVALID = 1,    /* bad argument: NULL required pointer, src >= n, n >= 2^32-1, k-core on directed, ... */
    SX_E_OOM = 2,        /* device allocation failed */
    SX_E_CUDA = 3,       /* CUDA runtime error (no device, launch failure, ...) */
    SX_E_NCCL = 4,       /* reserved for the multi-GPU layer */
    SX_E_NO_REVERSE = 5, /* pull needed on a directed graph uploaded without CSC */
    SX_E_WEIGHT = 6,     /* SSSP on an unweighted graph or with a zero weight ("positive edge weights") */
    SX_E_BARRIER = 7,    /* co-resident grid impossible, or the grid-barrier watchdog fired */
    SX_E_STATE = 8       /* context poisoned by an earlier sticky CUDA error */
} sx_status;

/* Static string naming a status code. Never NULL. */
const char* sx_status_str(int status);
/* Thread-local detail of the last failure on this thread ("" if none). Never NULL. */
const char* sx_last_error(void);
/* ABI version: (major << 16) | minor. */
int sx_version(void);

typedef struct sx_ctx_s* sx_ctx;     /* one device + one stream */
typedef struct sx_graph_s* sx_graph; /* device-resident graph owned by one ctx */

/*
 * Create a context on CUDA device `device`, issuing all work on `cuda_stream`
 * (a cudaStream_t; NULL = the legacy default stream).  The stream is borrowed:
 * it must outlive the context.  Errors: SX_E_CUDA (no such device / not
 * sm_100), SX_E_INVALID (out == NULL), SX_E_OOM.
 */
sx_status sx_ctx_create(int device, void* cuda_stream, sx_ctx* out);
/* Release a context (NULL is a no-op).  Graphs of the ctx must be freed first. */
void sx_ctx_destroy(sx_ctx ctx);

/*
 * Device facts the engine sizes itself from (Eq. 1 generalised):
 * the persistent kernels are launched cooperatively with
 * ctas = occupancy(kernel) * sm_count, so every CTA is co-resident and the
 * software grid barrier cannot deadlock (the Fig. 10 failure).
 */
typedef struct {
    int device, sm_count, cc_major, cc_minor;
    int regs_per_sm, max_threads_per_sm;
    int block_threads;       /* threads per CTA of the persistent kernels */
    int push_ctas_per_sm;    /* occupancy of the fused push kernel */
    int pull_ctas_per_sm;    /* occupancy of the fused pull kernel */
    int push_regs, pull_regs; /* registers/thread of those kernels (Table 2 analogue) */
} sx_device_info;
sx_status sx_ctx_info(sx_ctx ctx, sx_device_info* out);

/*
 * Barrier roofline: launch the persistent configuration and
 * time `iters` back-to-back grid barriers with no work between them.
 * us_per_barrier receives the mean latency in microseconds; ctas (nullable)
 * the co-resident grid size used.  Errors: SX_E_INVALID (iters == 0 or NULL
 * out), SX_E_BARRIER (watchdog), SX_E_CUDA.
 */
sx_status sx_barrier_bench(sx_ctx ctx, uint32_t iters, double* us_per_barrier, int* ctas);
/*
 * Fault injection for the grid barrier (a software barrier over
 * CTAs that are not all co-resident deadlocks).
 *   mode 1: cooperatively launch one CTA more than occupancy x SMs; the
 *           driver must refuse it -> SX_E_BARRIER (nothing runs).
 *   mode 2: a co-resident grid in which the last CTA never arrives at the
 *           barrier; the watchdog, lowered to timeout_ms for this launch, fires
 *           -> SX_E_BARRIER, every CTA leaves, and the context stays usable.
 * Returns SX_OK only if the fault was NOT detected.  Errors: SX_E_INVALID
 * (mode not 1/2, mode 2 with timeout_ms = 0), SX_E_CUDA.
 */
sx_status sx_barrier_fault(sx_ctx ctx, uint32_t mode, uint32_t timeout_ms);
/* Diagnostic: cost of the small-frontier cluster mode's pieces on one 16-CTA
   cluster.  mode 0: empty launch; 1: one cluster barrier (reps barriers in one
   launch); 2: zero a bitmap of nwords words; 3: zero + compact an empty bitmap.
   *us = microseconds per launch (modes 0, 2, 3) or per barrier (mode 1). */
sx_status sx_cluster_bench(sx_ctx ctx, uint64_t nwords, uint32_t mode, uint32_t reps, double* us);
/* Diagnostic: GPU time per back-to-back launch of an empty kernel in the shape
   of a fused phase (P:743's launch count is what selective fusion saves).
   mode 0: plain launch of occupancy x SMs CTAs; 1: the same as a cooperative
   launch; 2: one 16-CTA cluster.  *us = microseconds per launch.  Errors:
   SX_E_INVALID (mode > 2, reps == 0, NULL us), SX_E_CUDA. */
sx_status sx_launch_bench(sx_ctx ctx, uint32_t mode, uint32_t reps, double* us);

/* ------------------------------------------------------------------ graphs */
enum {
    SX_DIRECTED = 1,    /* csc_* describe the in-neighbour rows; otherwise the graph is symmetric and CSR serves as CSC */
    SX_DEVICE_PTRS = 2, /* row_ptr/col/w (and csc_*) are device pointers */
    SX_BORROW = 4,      /* with SX_DEVICE_PTRS: do not copy; the caller keeps the arrays alive until sx_graph_free */
    SX_DEDUP = 8        /* collapse duplicate edges at upload (reading 19 keeps them by default): one edge per
                           (row, neighbour) with the minimum weight of its duplicates, neighbours ascending per
                           row; m (and the CSC's) shrink accordingly.  Implies a copy (no SX_BORROW) */
};

/*
 * A CSR graph.  Layout: row_ptr u64[n+1] with row_ptr[0] = 0,
 * non-decreasing, row_ptr[n] = m; col u32[m] neighbour ids < n; w = edge
 * weights, w_bytes = 1 (u8) or 4 (u32) per edge, or w = NULL (unweighted).
 * For SX_DIRECTED graphs csc_ptr/csc_idx/csc_w give the in-neighbour rows in
 * the same layout (csc_w uses w_bytes); they may be NULL, in which case pull
 * (PageRank, SpMV, BP, pull-mode BFS) returns SX_E_NO_REVERSE.
 */
typedef struct {
    uint64_t n, m;
    const uint64_t* row_ptr;
    const uint32_t* col;
    const void* w;
    uint32_t w_bytes;
    const uint64_t* csc_ptr;
    const uint32_t* csc_idx;
    const void* csc_w;
    uint32_t flags;
} sx_csr_desc;

/*
 * Upload (copy) a CSR graph to the device, validate it (row_ptr monotone,
 * row_ptr[0] = 0, row_ptr[n] = m, col < n) and precompute per-vertex degree
 * arrays (step a1/a3 of SURVEY.md §8(a)).  The caller's arrays are not
 * retained unless SX_BORROW.  Errors: SX_E_INVALID (bad layout, n >= 2^32-1),
 * SX_E_OOM, SX_E_CUDA.
 */
sx_status sx_graph_upload(sx_ctx ctx, const sx_csr_desc* desc, sx_graph* out);
/*
 * Generate a synthetic graph directly in device memory (SURVEY.md §8(b), §8(d)
 * input recipe; the paper's Kron/R-MAT workloads) and
 * return it as a graph of this ctx, prepared exactly like sx_graph_upload.
 * The generator is the seeded one of simgen/ (Philox-4x32-10, counter = tuple
 * index), so the CSR is bit-identical to simgen.c's for the same arguments.
 *
 * sx_graph_rmat: Graph500 Kronecker/R-MAT, n = 2^scale, edgefactor*2^scale
 *   tuples with (A,B,C,D) = (.57,.19,.19,.05) (reading 20), symmetrised,
 *   self-loops dropped, duplicates kept (reading 19), rows sorted by (col, w);
 *   ids relabelled by a bijective mixer that fixes vertex 0 unless
 *   SX_GEN_NO_RELABEL.  Weights uniform in [wmin, wmax] per tuple (both
 *   directions equal; reading 13); wmin = wmax = 0 = unweighted.  Stored u8
 *   when wmax <= 255.
 * sx_graph_grid: rows x cols 4-neighbour grid ("road-like", C2), vertex id
 *   r*cols + c, weight per undirected edge id, same weight rule.
 * Errors: SX_E_INVALID (scale outside [1,31], edgefactor < 1, n >= 2^32-1,
 * wmin = 0 < wmax or wmax < wmin, unknown flag), SX_E_OOM, SX_E_CUDA.
 */
enum { SX_GEN_NO_RELABEL = 1 };
sx_status sx_graph_rmat(sx_ctx ctx, int scale, int edgefactor, uint64_t seed, uint32_t wmin, uint32_t wmax,
                        uint32_t flags, sx_graph* out);
sx_status sx_graph_grid(sx_ctx ctx, uint32_t rows, uint32_t cols, uint64_t seed, uint32_t wmin, uint32_t wmax,
                        sx_graph* out);
/*
 * Copy a graph's CSR back to caller memory (host or device): row_ptr u64[n+1],
 * col u32[m], w u32[m] (widened from u8 storage).  Any pointer may be NULL to
 * skip that array.  This is how the oracle side checks graphs built on the
 * device.  Errors: SX_E_WEIGHT (w requested of an
 * unweighted graph), SX_E_INVALID, SX_E_CUDA.
 */
sx_status sx_graph_download(sx_graph g, uint64_t* row_ptr, uint32_t* col, uint32_t* w);
/* n, m and the owned vertex range [v_begin, v_end) (= [0, n) on one GPU). Any out pointer may be NULL. */
sx_status sx_graph_info(sx_graph g, uint64_t* n, uint64_t* m, uint64_t* v_begin, uint64_t* v_end);
/* Free a graph and its workspace (NULL is a no-op). */
void sx_graph_free(sx_graph g);

/* -------------------------------------------------------------- run knobs */
typedef struct {
    uint32_t iter;       /* 1-based iteration number */
    uint32_t dir;        /* 0 push, 1 pull, 2 push on one thread-block cluster (cluster_enter) */
    uint32_t filter;     /* how the NEXT list was produced: 0 online, 1 ballot, 2 static (pull-all lists) */
    uint32_t launch;     /* 0-based index of the kernel launch that ran this iteration */
    uint32_t n_active[4];/* next-iteration list sizes: small / medium / large / huge;
                            in pull these are the remaining candidate (unvisited) lists */
    uint64_t n_frontier; /* |F'|: vertices activated by this iteration */
    uint64_t m_active;   /* sum of out-degrees of F' (m_f of the direction heuristic) */
    uint64_t aux;        /* algorithm-specific: BFS unvisited edges m_u; SSSP bucket upper bound; k-core level k */
    uint64_t t_ns;       /* device %globaltimer (ns) when the iteration's decision was taken */
} sx_trace_rec;

typedef struct {
    uint32_t overflow_threshold; /* online-filter bin capacity per warp; default 64 */
    uint32_t sep_small;          /* degree separator thread|warp; default 32 */
    uint32_t sep_large;          /* degree separator warp|CTA; default 128 */
    uint32_t sep_huge;           /* degree separator CTA|grid-split (B200 addition); default 16384 */
    float alpha, beta;           /* push->pull when m_f > m_u/alpha, pull->push when n_f < n/beta (Beamer's test;
                                    reading 8); defaults 60, 512 — measured on B200 (Beamer's CPU values 14, 24
                                    cost Graph500-style random roots 20%) */
    int32_t force_filter;        /* 0 JIT, 1 online only, 2 ballot only, 3 batch (the baseline of
                                    P:536-545: every update recorded, duplicates kept, no claim; BFS and
                                    SSSP/WCC push; k-core removals are exactly-once, so 3 = online there) */
    int32_t force_dir;           /* 0 auto, 1 push only, 2 pull only */
    int32_t fusion;              /* 1 selective push/pull fusion (default); 0 no fusion (one launch per
                                    iteration); 2 all fusion (BFS: one launch for every phase) */
    uint32_t max_iters;          /* 0 = unlimited */
    sx_trace_rec* trace;         /* nullable host buffer of trace_cap records (P:623-626 activation patterns) */
    uint64_t trace_cap;
    uint32_t local_chain;        /* SSSP / k-core push (B200 addition): a thread that activates a vertex may
                                    process it at once instead of recording it, up to this many in a row
                                    (chaotic relaxation, reading 12; results unchanged); 0 = strict BSP.
                                    Ignored by BFS (levels are BSP-exact). Default 0: measured on the 2048^2
                                    grid, chains cut iterations 1.6x but lengthened each one more. */
    uint32_t cluster_enter;      /* BFS / SSSP push (B200 addition): when the next frontier has at most this
                                    many vertices (BFS: and at most 128x this many out-edges) the iterations
                                    continue on ONE thread-block cluster of 16 CTAs x 1024 threads
                                    synchronised by the hardware cluster barrier instead of the grid
                                    barrier; back to the full grid above 8x this size (BFS: or 256x this
                                    many out-edges).  Results unchanged.  0 = never.  Default
                                    SX_CLUSTER_AUTO = 4096 for SSSP / WCC / k-core, 0 for BFS (measured:
                                    the cluster start costs Graph500-style random roots 20%).
                                    k-core: once a sub-round frontier of a level has at most this many
                                    vertices, the rest of the level's cascade runs as an asynchronous work
                                    queue (no grid barrier per sub-round; reading 28); 0 = BSP. */
} sx_opts;

typedef struct {
    uint32_t iterations;         /* BSP iterations executed */
    uint32_t launches;           /* persistent-kernel launches (Table 2: selective fusion -> 3 for BFS) */
    uint32_t ballot_iters;       /* iterations whose next list came from the ballot filter */
    uint32_t pull_iters;         /* iterations run in pull direction */
    uint64_t edges_examined;     /* edges whose Compute ran (push: all out-edges of F; pull: scanned up to early exit) */
    uint64_t vertices_scanned;   /* vertices covered by ballot scans */
    uint64_t list_entries;       /* active-list entries consumed */
    double bytes_model;          /* algorithmic bytes of the executed schedule (SURVEY.md §8(d) rule) */
    double ms;                   /* device time of the run, CUDA events on the ctx stream (init + all kernels, no readback) */
    double ms_push, ms_pull;     /* device time inside push / pull persistent kernels (CUDA events around each launch) */
    double bytes_push, bytes_pull; /* bytes_model split by the direction of the launch that moved them */
    uint32_t launches_push, launches_pull;
    double ms_fused;             /* device time inside all-phase fused launches (fusion = 2) */
    uint32_t launches_fused;
    uint32_t runs;               /* algorithm runs these statistics cover (1; sx_graph_sync: the runs it drained) */
    double residual;             /* convergence runs (sx_pagerank_conv, sx_bp_conv): L1 mass of change not yet
                                    propagated when the run stopped (pull: the last iteration's L1 change; PageRank
                                    push tail: sum |rho|).  PageRank lies within d/(1-d) x residual (L1) of its
                                    fixed point.  0 otherwise. */
} sx_stats;

#define SX_CLUSTER_AUTO 0xFFFFFFFFu
/* Fill `o` with the defaults above. */
void sx_opts_default(sx_opts* o);

/* ------------------------------------------------------------- algorithms
 * opts may be NULL (defaults); stats may be NULL.  Results are written to the
 * caller's buffer of n elements (host or device memory).
 */

/* BFS (voting combine P:345): level_out[v] = hop distance from src,
 * 0xFFFFFFFF if unreachable.  Push/pull switch per opts.
 * Errors: SX_E_INVALID (src >= n, NULL level_out), SX_E_NO_REVERSE (pull on a directed graph without CSC). */
sx_status sx_bfs(sx_graph g, uint32_t src, const sx_opts* opts, uint32_t* level_out, sx_stats* stats);

/* Asynchronous BFS (the same result as sx_bfs): enqueue the whole run on the
 * ctx stream — one state-init kernel and ONE all-fusion persistent launch
 * (fusion = 2 whatever opts says; no trace, no cluster tail)
 * — and return without waiting, so back-to-back runs pay no host round trip.
 * level_out must be DEVICE memory (n u32) and stays undefined until the
 * stream reaches the run (stream order: later work on the ctx stream sees it).
 * Statistics (summed over the graph's async runs) come from sx_graph_sync.
 * Errors found while enqueuing are returned here (as sx_bfs, plus
 * SX_E_INVALID for a host level_out); a barrier watchdog during a run is
 * reported by the next sx_graph_sync. */
sx_status sx_bfs_async(sx_graph g, uint32_t src, const sx_opts* opts, uint32_t* level_out);
/* Wait for every run enqueued with sx_bfs_async on g's context and return g's
 * async statistics since the previous sx_graph_sync (stats nullable; then
 * reset them): runs, iterations, edges, bytes_model, ms = device time of the
 * runs (init + fused kernel, CUDA events), ms_fused = the fused kernels alone.
 * Errors: SX_E_BARRIER (a watchdog fired in one of the runs), SX_E_CUDA. */
sx_status sx_graph_sync(sx_graph g, sx_stats* stats);

/* SSSP: dist_out[v] = min path weight from src
 * (u32, 0xFFFFFFFF unreachable).  delta-stepping with bucket width `delta` (0 = infinity:
 * frontier Bellman-Ford; reading 9).  Distances are delta-independent.
 * Errors: SX_E_WEIGHT (unweighted graph or a zero weight), SX_E_INVALID. */
sx_status sx_sssp(sx_graph g, uint32_t src, uint32_t delta, const sx_opts* opts, uint32_t* dist_out,
                  sx_stats* stats);

/* PageRank (reading 14): `iters` Jacobi steps of
 *   r(u) = (1-d)/N + d*(sum_{v in in(u)} r(v)/outdeg(v) + D/N), D = dangling mass, r_0 = 1/N,
 * pull with sum combine; iters >= 1.  rank_out: f32[n].  Errors: SX_E_INVALID (iters = 0, damping outside [0,1]), SX_E_NO_REVERSE. */
sx_status sx_pagerank(sx_graph g, float damping, uint32_t iters, const sx_opts* opts, float* rank_out,
                      sx_stats* stats);

/* PageRank to convergence ("updates the rank value ... iteratively till all vertices have stable
 * rank values ... we start PageRank with the pull model ... At the end of PageRank, we switch to the push
 * model because the majority of the vertices are stable"; readings 25-26):
 *   variant SX_PR_NORMALIZED: r(u) = (1-d)/N + d*(sum_{v in in(u)} r(v)/outdeg(v) + D/N), r_0 = 1/N (reading 14)
 *   variant SX_PR_SPEC:       r(u) = (1-d) + d*sum_{v in in(u)} r(v)/outdeg(v), dangling mass dropped, r_0 = 1
 *
 * Jacobi pull steps in fp64 while the L1 change of a step is >= epsilon; when at most a tenth of the
 * vertices still change by more than tau = epsilon/(4N), the run switches to a delta-accumulative push
 * (residual propagation) over the vertices whose pending change exceeds tau, until none does.  Either
 * way the result is within d/(1-d)*epsilon (L1) of the exact fixed point; stats->residual says how far.
 * opts->force_dir: 0 auto, 1 push tail right after the first pull step, 2 pull only.  max_iters >= 1 caps
 * pull steps + push iterations.  rank_out: f64[n], host or device.
 * Errors: SX_E_INVALID (damping outside (0,1), epsilon <= 0, max_iters = 0, unknown variant), SX_E_NO_REVERSE. */
enum { SX_PR_NORMALIZED = 0, SX_PR_SPEC = 1 };
sx_status sx_pagerank_conv(sx_graph g, double damping, double epsilon, uint32_t max_iters, uint32_t variant,
                           const sx_opts* opts, double* rank_out, sx_stats* stats);

/* k-core (reading 6): k > 0 -> core_out[v] = 1 if v is in the k-core (minimum degree >= k,
 * duplicate edges counted) else 0; k = 0 -> core_out[v] = coreness of v.  Undirected graphs only.
 * Errors: SX_E_INVALID (directed graph). */
sx_status sx_kcore(sx_graph g, uint32_t k, const sx_opts* opts, uint32_t* core_out, sx_stats* stats);

/* SpMV (north_star; not in the paper): y[u] = sum_{(v,u) in E} w(v,u) * x[v] (w = 1 if unweighted),
 * repeated `iters` >= 1 times with the same x (pull, sum combine).  x: f32[n] host or device.
 * Errors: SX_E_INVALID, SX_E_NO_REVERSE. */
sx_status sx_spmv(sx_graph g, const float* x, uint32_t iters, const sx_opts* opts, float* y_out,
                  sx_stats* stats);

/* Belief propagation (model = reading 15 of SURVEY.md §8(c)): `iters` Jacobi steps of
 *   l(u) = logit(p_u) + sum_{v in in(u)} log((c b + (1-c)(1-b)) / (c (1-b) + (1-c) b)),
 *   b = sigmoid(l(v)), c = 0.25 + 0.5*(weight-1)/254 (unweighted: c = 0.75), l_0 = logit(p).
 * prior: f32[n] in (0,1), host or device; iters >= 1.  Errors: SX_E_INVALID, SX_E_NO_REVERSE. */
sx_status sx_bp(sx_graph g, const float* prior, uint32_t iters, const sx_opts* opts, float* logodds_out,
                sx_stats* stats);

/* Belief propagation to convergence (reading 15's model, reading 27): the Jacobi steps of
 * sx_bp until the L1 change of the beliefs b = sigmoid(l), sum_u |b_{t+1}(u) - b_t(u)|, is < epsilon or
 * max_iters steps ran (loopy BP need not converge: not an error; stats->residual = the last L1 change,
 * stats->iterations = steps run).  logodds_out: f32[n].  Errors: as sx_bp, SX_E_INVALID (epsilon <= 0). */
sx_status sx_bp_conv(sx_graph g, const float* prior, double epsilon, uint32_t max_iters, const sx_opts* opts,
                     float* logodds_out, sx_stats* stats);

/* Connected components (WCC on an undirected graph; the paper names WCC as a
 * voting workload): label_out[v] = the smallest
 * vertex id in v's component.  Min-label propagation as an ACC algorithm: every
 * vertex starts with its own id and active; Compute = the neighbour's label,
 * Combine = min (atomicMin in push, single-owner min in pull); the same
 * filters, direction switch and fused kernels as sx_sssp with every weight
 * read as 0.  Unweighted graphs are fine.  Errors: SX_E_INVALID (directed
 * graph, NULL label_out). */
sx_status sx_wcc(sx_graph g, const sx_opts* opts, uint32_t* label_out, sx_stats* stats);

/* ------------------------------------------------------------ multi-GPU layer
 * SURVEY.md §8(e); the paper itself is single-GPU.  1D vertex-range
 * partition: rank r of P owns vertices [r V, min(n, (r+1) V)), V = ceil(n/P)
 * rounded up to a multiple of 32.  Each rank holds the CSR rows of its owned
 * vertices with GLOBAL column ids (symmetric graphs: those rows are also the
 * in-rows used by pull).  Per BSP level the ranks exchange frontier-bitmap
 * slices (allgather for pull, alltoall + local OR for push), SSSP candidate
 * distances (reduce-scatter with min) and the (|F'|, m_f) counters (allreduce),
 * all on the ctx stream.  Collective: every rank calls the same function with
 * the same arguments (except its own slice / outputs).
 */
typedef struct sx_dist_s* sx_dist;

/* 128-byte NCCL unique id for ncclCommInitRank; rank 0 creates it and the
 * caller broadcasts it (e.g. with torch.distributed).  Errors: SX_E_NCCL. */
sx_status sx_nccl_unique_id(void* out128);

/*
 * Create the distribution of an n_global-vertex graph over `nranks` ranks, of
 * which this process drives ranks [rank0, rank0 + nlocal):
 *   nlocal == 1 with nccl_id: one rank per process, exchanges over an NCCL
 *     communicator built from `nccl_id` (one process per GPU, NVLink/NVSwitch;
 *     nranks = 1 gives a one-rank communicator that still runs every collective);
 *   nlocal == nranks without nccl_id: every rank in this process on the ctx's
 *     device ("virtual ranks": the same kernels and schedule, device-to-device
 *     copies in place of the collectives; for tests of the partitioned path on one GPU).
 * Errors: SX_E_INVALID (bad layout), SX_E_NCCL, SX_E_OOM, SX_E_CUDA.
 */
sx_status sx_dist_create(sx_ctx ctx, uint64_t n_global, int nranks, int rank0, int nlocal, const void* nccl_id,
                         sx_dist* out);
/* Owned vertex range [v_begin, v_end) of local rank `local_rank`. */
sx_status sx_dist_range(sx_dist d, int local_rank, uint64_t* v_begin, uint64_t* v_end);
/*
 * Upload local rank `local_rank`'s slice: desc->n = owned row count (v_end -
 * v_begin), desc->row_ptr local (starting at 0), desc->col GLOBAL ids < n_global,
 * desc->w optional (same width on every rank).  Symmetric graphs only.
 * Copies; validates like sx_graph_upload.  Uploading again replaces the rank's
 * slice (a new graph on the same partition).  Errors: SX_E_INVALID, SX_E_OOM.
 */
sx_status sx_dist_upload(sx_dist d, int local_rank, const sx_csr_desc* desc);
/* Free (collective for NCCL communicators; NULL is a no-op). */
void sx_dist_free(sx_dist d);
/*
 * Distributed BFS with the push/pull switch (Beamer
 * alpha/beta from opts): level_out[i] receives local rank i's owned slice
 * (v_end - v_begin entries, host or device).
 * opts->fusion = 2 (NCCL backend only): the whole BFS is ONE
 * persistent cooperative kernel per rank; the per-level exchange runs inside it
 * over the NCCL device API — push marks atomically OR'ed into the owner's inbox
 * and frontier slices stored into every rank's global bitmap through LSA
 * pointers into a symmetric window (ncclMemAlloc + ncclCommWindowRegister),
 * counters added into every rank's slots with peer atomics, one
 * ncclLsaBarrierSession per level step — no host round trip per level.  Needs
 * every rank in one LSA team (one NVLink/NVSwitch domain): SX_E_NCCL otherwise.
 * A DEVICE level_out[i] is written in place (no copy-out).  Errors as sx_bfs.
 */
sx_status sx_dist_bfs(sx_dist d, uint32_t src, const sx_opts* opts, uint32_t* const* level_out, sx_stats* stats);
/* Asynchronous device-initiated distributed BFS (the fusion = 2 run of sx_dist_bfs, the same result):
 * enqueue this rank's ONE persistent kernel on the ctx stream and return without waiting, so
 * back-to-back runs pay no host round trip (as sx_bfs_async on one GPU).  NCCL backend, one rank per
 * process; level_out[0] must be DEVICE memory (the owned slice, v_end - v_begin u32), written in place
 * and undefined until the stream reaches the run.  Every rank must enqueue the same runs.
 * Errors: SX_E_INVALID (host or NULL level_out, src >= n, virtual ranks), SX_E_NCCL (ranks not in one
 * LSA team); a barrier watchdog during a run is reported by the next sx_dist_sync. */
sx_status sx_dist_bfs_async(sx_dist d, uint32_t src, const sx_opts* opts, uint32_t* const* level_out);
/* Wait for the runs enqueued with sx_dist_bfs_async and return their statistics (stats nullable):
 * runs, ms = device time from the first run's start to the last run's end (CUDA events), iterations /
 * pull_iters / edges_examined / list_entries (reached vertices) of the LAST run.  Resets the count.
 * Errors: SX_E_BARRIER (a watchdog fired), SX_E_CUDA. */
sx_status sx_dist_sync(sx_dist d, sx_stats* stats);
/* Distributed SSSP, delta-stepping as sx_sssp; dist_out[i] = local rank i's owned slice. */
sx_status sx_dist_sssp(sx_dist d, uint32_t src, uint32_t delta, const sx_opts* opts, uint32_t* const* dist_out,
                       sx_stats* stats);

#ifdef __cplusplus
}
#endif
#endif /* SIMDX_H */

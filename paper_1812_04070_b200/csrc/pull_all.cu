// pull_all.cu — the all-active pull algorithms: PageRank, SpMV
// (north_star) and belief propagation.  Every vertex is active every
// iteration ("treats all vertices as active"), so the ballot filter runs
// exactly once, in iteration 1, to build the class lists ("BP and
// PageRank need the ballot filter at exactly the first iteration"); the lists
// are then static.  Each iteration is a pull:
//   Compute : update_{v->u} = term(M_v, M_(v,u))   over in-edges of u
//   Combine : sum (agg_sum)
//     small  (thread granularity): one thread per vertex, 16 gathers in flight
//     medium (warp granularity):   lane-strided 128-bit loads + shuffle tree
//     large + huge (CTA / grid granularity): the two lists are concatenated and
//       split edge-balanced over every thread of the grid (B200 design: a CTA
//       per vertex leaves the latency of each row exposed); fp64 atomics only
//       where a thread's slice ends inside a row, then the owner applies.
//   Apply   : a single owner writes M_u (atomic-free), Jacobi double
//             buffering between iterations; fp64 accumulation, fp32 state (BP: fp64).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "internal.h"

namespace sx {

// ---------------------------------------------------------------- operators
// Per-thread sums an operator's apply() contributes to: dangling mass of the
// next iteration (PageRank), and for the convergence runs the L1 change of the
// iteration and the number of vertices that changed by more than tau.
struct PAcc {
    double dang = 0.0, l1 = 0.0;
    uint32_t unstable = 0;  // out-edges of the vertices that changed by more than tau (the push tail's work)
};

// Each operator splits the edge term into the source value val(v) (what the hub
// cache holds) and term(e, val) (combined with the edge weight).
struct PrOp {  // r(u) = (1-d)/N + d (sum_v r(v)/outdeg(v) + D/N)
    using HubT = float;
    using TermT = float;     // lane-local partial sums of <= 8 terms in fp32, fp64 from the warp scan on
    using AuxT = float;      // 1/outdeg of the destination (0 = dangling): contrib = r x (1/outdeg),
                             // no fp64 division per row (rel. error <= 2^-24 + 2^-53, within the fp32 store)
    static constexpr bool kStaticHub = false;
    float* contrib[2];
    float* out;
    const uint32_t* dout;
    double d, invN;
    // per-iteration.  The double buffer is chosen with a select, never indexed by
    // `cur`: a dynamically indexed member array put the kernel's copy of the
    // operator in local memory (an LDL on every tile's gather address)
    uint32_t cur;
    double D;
    bool last;
    __device__ __forceinline__ HubT val(uint32_t v) const { return (cur ? contrib[1] : contrib[0])[v]; }
    __device__ __forceinline__ const HubT* src() const { return (cur ? contrib[1] : contrib[0]); }
    __device__ __forceinline__ TermT term(const DevGraph&, uint64_t, HubT x) const { return x; }
    __device__ __forceinline__ AuxT aux(uint32_t u) const {
        const uint32_t du = dout[u];
        return du ? 1.0f / (float)du : 0.0f;
    }
    __device__ __forceinline__ void init(uint64_t v, PAcc& pa) const {
        const uint32_t dv = dout[v];
        contrib[0][v] = dv ? (float)(invN / (double)dv) : 0.f;
        if (dv == 0) pa.dang += invN;
    }
    bool directed;
    __device__ __forceinline__ bool empty_each_iter() const { return directed; }
    // symmetric graph: an empty row is dangling (out-degree 0); its rank is the
    // same for every such row, so their dangling mass is count x rank
    __device__ __forceinline__ double empty_dangling(uint32_t ne) const { return (double)ne * ((1.0 - d) * invN + d * D * invN); }
    __device__ __forceinline__ void apply(uint32_t u, double s, AuxT inv, PAcc& pa) const {
        const double r = (1.0 - d) * invN + d * (s + D * invN);
        if (last) out[u] = (float)r;
        (cur ? contrib[0] : contrib[1])[u] = (float)(r * (double)inv);
        if (inv == 0.0f) pa.dang += r;
    }
};

// PageRank to convergence (readings 25-26), the pull part, in fp64:
//   variant 0: r(u) = (1-d)/N + d (sum_v r(v)/outdeg(v) + D/N)   (reading 14), r_0 = 1/N
//   variant 1: r(u) = (1-d)   + d  sum_v r(v)/outdeg(v), r_0 = 1
// Every apply also stores rho(u) = r_new(u) - r_old(u) (the change not yet
// propagated: what the push tail starts from) and adds |rho(u)| to the
// iteration's L1 change; |rho(u)| > tau counts u as unstable.
struct PrcOp {
    using HubT = double;
    using TermT = double;
    using AuxT = uint32_t;  // out-degree of the destination (0 = dangling)
    static constexpr bool kStaticHub = false;
    double* contrib[2];
    double* r;
    double* rho;
    const uint32_t* dout;
    double d, base, dn, r0, tau;  // base = (1-d)/N or 1-d; dn = 1/N (variant 0) or 0 (dangling mass dropped)
    uint32_t cur;
    double D;
    bool last;
    __device__ __forceinline__ HubT val(uint32_t v) const { return (cur ? contrib[1] : contrib[0])[v]; }
    __device__ __forceinline__ const HubT* src() const { return (cur ? contrib[1] : contrib[0]); }
    __device__ __forceinline__ TermT term(const DevGraph&, uint64_t, HubT x) const { return x; }
    __device__ __forceinline__ AuxT aux(uint32_t u) const { return dout[u]; }
    __device__ __forceinline__ void init(uint64_t v, PAcc& pa) const {
        const uint32_t dv = dout[v];
        r[v] = r0;
        contrib[0][v] = dv ? r0 / (double)dv : 0.0;
        if (dv == 0 && dn != 0.0) pa.dang += r0;
    }
    __device__ __forceinline__ bool empty_each_iter() const { return true; }
    __device__ __forceinline__ double empty_dangling(uint32_t) const { return 0.0; }
    __device__ __forceinline__ void apply(uint32_t u, double s, AuxT du, PAcc& pa) const {
        const double rn = base + d * (s + D * dn);
        const double ch = rn - r[u];
        r[u] = rn;
        rho[u] = ch;
        (cur ? contrib[0] : contrib[1])[u] = du ? rn / (double)du : 0.0;
        if (du == 0 && dn != 0.0) pa.dang += rn;
        pa.l1 += fabs(ch);
        if (fabs(ch) > tau) pa.unstable += du;
    }
};

struct SpmvOp {  // y(u) = sum_v w(v,u) x(v)
    using HubT = float;
    using TermT = float;
    using AuxT = uint32_t;
    static constexpr bool kStaticHub = true;  // x does not change between iterations
    const float* x;
    float* out;
    uint32_t cur;
    double D;
    bool last;
    __device__ __forceinline__ HubT val(uint32_t v) const { return x[v]; }
    __device__ __forceinline__ const HubT* src() const { return x; }
    __device__ __forceinline__ TermT term(const DevGraph& g, uint64_t e, HubT xv) const {
        return (float)edge_w(g.iw8, g.iw32, e) * xv;
    }
    __device__ __forceinline__ AuxT aux(uint32_t) const { return 0; }
    __device__ __forceinline__ bool empty_each_iter() const { return false; }  // y = 0
    __device__ __forceinline__ double empty_dangling(uint32_t) const { return 0.0; }
    __device__ __forceinline__ void init(uint64_t, PAcc&) const {}
    __device__ __forceinline__ void apply(uint32_t u, double s, AuxT, PAcc&) const { out[u] = (float)s; }
};

// BP is computed in fp64 end to end (beliefs, couplings, messages), fp32 out.
// Measured: this loopy recurrence amplifies a 1-ulp fp32 perturbation (even of
// the coupling c alone) to ~1e-4 after 10 steps on R-MAT, so fp32 state cannot
// meet the 1e-5 conditioned tolerance.
struct BpOp {  // l(u) = logit(p_u) + sum_v log((c b + (1-c)(1-b)) / (c(1-b) + (1-c) b)), b = sigmoid(l(v))
    using HubT = double;
    using TermT = double;
    using AuxT = float;      // prior of the destination
    static constexpr bool kStaticHub = false;
    double* b[2];
    const double* ctab;  // coupling c(w) for the 256 u8 weights (same expression, precomputed: no fp64 division per edge)
    const float* prior;
    float* out;
    uint32_t cur;
    double D;
    bool last;
    __device__ static __forceinline__ double coupling(double wt) { return 0.25 + 0.5 * (wt - 1.0) / 254.0; }
    __device__ __forceinline__ HubT val(uint32_t v) const { return (cur ? b[1] : b[0])[v]; }
    __device__ __forceinline__ const HubT* src() const { return (cur ? b[1] : b[0]); }
    __device__ __forceinline__ AuxT aux(uint32_t u) const { return prior[u]; }
    // l = logit(p): written to b[1] in the first iteration (b[0] by init), out in the last
    __device__ __forceinline__ bool empty_each_iter() const { return false; }
    __device__ __forceinline__ double empty_dangling(uint32_t) const { return 0.0; }
    __device__ __forceinline__ TermT term(const DevGraph& g, uint64_t e, HubT bv) const {
        const double c = g.iw8 ? __ldg(ctab + __ldg(g.iw8 + e)) : g.iw32 ? coupling((double)__ldg(g.iw32 + e)) : __ldg(ctab + 255);
        const double num = c * bv + (1.0 - c) * (1.0 - bv);
        const double den = c * (1.0 - bv) + (1.0 - c) * bv;
        return log(num / den);
    }
    bool conv;  // convergence run: the L1 change of the beliefs is summed
    __device__ __forceinline__ void init(uint64_t v, PAcc&) const {
        const double p = (double)prior[v];
        const double l = log(p / (1.0 - p));
        b[0][v] = 1.0 / (1.0 + exp(-l));
    }
    __device__ __forceinline__ void apply(uint32_t u, double s, AuxT pu, PAcc& pa) const {
        const double p = (double)pu;
        const double l = log(p / (1.0 - p)) + s;
        if (last) out[u] = (float)l;
        const double bn = 1.0 / (1.0 + exp(-l));
        if (conv) pa.l1 += fabs(bn - (cur ? b[1] : b[0])[u]);
        (cur ? b[0] : b[1])[u] = bn;
    }
};

// convergence runs: the per-vertex change above which a vertex counts as unstable
template <class Op> __device__ __forceinline__ void op_set_tau(Op&, double) {}
__device__ __forceinline__ void op_set_tau(PrcOp& op, double tau) { op.tau = tau; }

// ---------------------------------------------------------------- schedule
// The all-active pull as an edge-balanced stream (B200 design; DESIGN.md
// "Pull-all").  The in-edge array is cut into warp tiles of PT = 32 x PV
// consecutive edges; lane l of a warp owns PV consecutive edges, loaded with
// two 128-bit loads.  Per graph (once, graph residency a1):
//   hcol  : the in-edge sources, the K most-gathered sources (largest out-degree)
//           re-encoded as HUBBIT | slot — their values are read from a copy in
//           shared memory instead of L2 (a software cache of the hubs);
//   rs    : bitmap over in-edges, bit e set iff e is the first edge of a row
//           (and bit E, a sentinel row start).
// Per run, iteration 1 (task management: ballot filter in exactly the
// first iteration): the ballot filter lists the active rows (in-degree > 0)
// in vertex order (nz) and the rows that need the second phase (sp: empty rows
// and rows that cross a tile boundary); tile_seg[t] = index in nz of the row
// holding tile t's first edge.
// Per iteration:
//   A: every warp streams tiles; each lane sums its runs of equal destination
//      (row starts from rs), a warp segmented scan carries partial runs across
//      lanes; a row that starts and ends inside the tile is applied at once by
//      the lane holding its last edge (single owner, atomic-free); the
//      pieces of a row that crosses a tile boundary are added with fp64
//      atomics to acc[u];
//   -- grid barrier --
//   B: the sp rows are applied from acc (then acc is reset to 0);
//   -- grid barrier --  (Jacobi double buffer between iterations)
#ifndef SX_PULL_PV
#define SX_PULL_PV 8
#endif
#ifndef SX_PALL_MINB
#define SX_PALL_MINB 3
#endif
constexpr int PV = SX_PULL_PV;  // edges per lane (8 or 16)
constexpr int PT = 32 * PV;
static_assert(PV == 8 || PV == 16, "PV");
constexpr uint32_t HUBBIT = 0x80000000u;
#ifndef SX_PULL_HUBS
#define SX_PULL_HUBS 8192
#endif
// hub cache entries: 32 KB of fp32 (PR, SpMV) / 64 KB of fp64 (BP) per CTA.  Measured
// (profiles/r1/pull_hub_sweep.txt, PR s22 / s24): none 17.2 / 84.5 ms, 4K 15.2 / 70.4,
// 6K 14.9 / 69.3, 8K 14.7 / 68.2, 12K 15.1 / 72.7, 16K 22 ms (occupancy falls)
constexpr uint32_t PULL_HUBS = SX_PULL_HUBS;

template <class Op> struct PullP {
    DevGraph g;
    Sched s;
    Op op;
    uint32_t iters;
    const uint32_t* hcol;   // encoded in-edge sources (>= ntiles * PT entries, zero padded)
    const uint32_t* rs;     // row-start bitmap over in-edges (bit E set)
    const uint32_t* hubs;   // K hub vertex ids by slot
    uint32_t K;
    uint64_t ntiles, E;     // tiles, in-edges
    uint32_t* tile_seg;     // ntiles entries
    uint32_t* nz;           // active rows (in-degree > 0), ascending (+1 sentinel)
    uint32_t* sp;           // rows applied in phase B, ascending
    void* nzaux;            // per active row k: op.aux(nz[k]) (n + 2 entries of 4 B), filled per run
    double* acc;            // n fp64 partial sums of split rows (zero between runs)
    double eps;             // > 0: convergence run, stop when the iteration's L1 change < eps (iters = the cap)
    uint32_t tail;          // convergence run: 1 hand over to the push tail when most vertices are stable, 2 after iteration 1
};

struct NzPred {
    const uint32_t* din;
    __device__ __forceinline__ bool operator()(uint64_t v) const { return __ldg(din + v) > 0; }
};
struct SpPred {  // empty row, or a row crossing a tile boundary
    const uint64_t* irp;
    __device__ __forceinline__ bool operator()(uint64_t v) const {
        const uint64_t b = __ldg(irp + v), e = __ldg(irp + v + 1);
        return b == e || b / PT != (e - 1) / PT;
    }
};

// L2 eviction policies: the in-edge stream is read once per iteration
// (evict_first), the gathered source values are re-read E/n times per
// iteration and should stay resident (evict_last) instead of being pushed
// out by the stream.
__device__ __forceinline__ uint64_t l2_policy_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint4 ld_stream(const uint4* p, uint64_t pol) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
    return v;
}

// Predicated gather (plain global load, L2 evict_last; 0 when !c), so that a
// lane's loads are issued back to back instead of one branch-guarded load at a time.
__device__ __forceinline__ float ld_pred(const float* p, bool c, uint64_t pol) {
    float v = 0.f;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.global.L2::cache_hint.f32 %0, [%1], %3;\n\t}"
                 : "+f"(v) : "l"(p), "r"((int)c), "l"(pol));
    return v;
}
__device__ __forceinline__ double ld_pred(const double* p, bool c, uint64_t pol) {
    double v = 0.0;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.global.L2::cache_hint.f64 %0, [%1], %3;\n\t}"
                 : "+d"(v) : "l"(p), "r"((int)c), "l"(pol));
    return v;
}

// Segmented inclusive scan over the warp: a lane holding a row start does not
// take the partial sum of the lanes before it.
__device__ __forceinline__ double warp_seg_scan(double v, bool start) {
    const uint32_t l = lane_id();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(FULL, v, o);
        const bool fy = __shfl_up_sync(FULL, start, o);
        if ((int)l >= o) {
            if (!start) v += y;
            start |= fy;
        }
    }
    return v;
}

template <class Op> __global__ void __launch_bounds__(BLOCK, SX_PALL_MINB) pull_all(PullP<Op> p) {
    using HubT = typename Op::HubT;
    using TermT = typename Op::TermT;
    static_assert(sizeof(typename Op::AuxT) == 4, "nzaux holds 4-byte per-row operands");
    extern __shared__ __align__(16) unsigned char s_dyn[];
    HubT* s_hub = reinterpret_cast<HubT*>(s_dyn);
    Ctl* c = p.s.ctl;
    grid_begin(c);
    const uint64_t n = p.g.n, E = p.E;
    const uint64_t cs = p.s.cstride;
    Stats st;
    // ---- iteration-1 task management: two ballot filters, one list each
    Sched s1 = p.s;
    s1.sep_small = s1.sep_large = s1.sep_huge = INF;  // one class: plain vertex-ordered lists
    uint32_t cnt[NCLS];
    if (!ballot_filter(BallotWords<NzPred>{NzPred{p.g.din}, n}, s1, BallotOut{p.nz, cs, p.g.din}, cnt)) return;
    if (!grid_sync(c)) return;
    const uint32_t nnz = cnt[0];
    // second list, two classes by in-degree: 0 = empty rows, 1 = rows split across tiles
    s1.sep_small = 1;
    if (!ballot_filter(BallotWords<SpPred>{SpPred{p.g.irp}, n}, s1, BallotOut{p.sp, cs, p.g.din}, cnt)) return;
    const uint32_t nempty = cnt[0], nsplit = cnt[1];
    st.ballot += 2;
    st.scanned += 2 * n;
    {
        PAcc pa0;
        for (uint64_t v = gtid(); v < n; v += gthreads()) p.op.init(v, pa0);
        double a[1] = {pa0.dang};
        block_sum<1>(a);
        if (threadIdx.x == 0 && a[0] != 0.0) atomicAdd(&c->line[0].s[my_slot()].dsum, a[0]);
    }
    if (!grid_sync(c)) return;
    // tile_seg from the active-row list (ends before the first iteration's barrier below)
    for (uint64_t k = gtid(); k < nnz; k += gthreads()) {
        const uint32_t u = p.nz[k];
        const uint64_t b = __ldg(p.g.irp + u), e = __ldg(p.g.irp + u + 1);
        for (uint64_t t = (b + PT - 1) / PT; t * PT < e; ++t) p.tile_seg[t] = (uint32_t)k;
        reinterpret_cast<typename Op::AuxT*>(p.nzaux)[k] = p.op.aux(u);
    }
    if (lead()) {
        p.nz[nnz] = INF;  // sentinel row of the sentinel start bit E
        reinterpret_cast<typename Op::AuxT*>(p.nzaux)[nnz] = typename Op::AuxT(0);
        reinterpret_cast<typename Op::AuxT*>(p.nzaux)[nnz + 1] = typename Op::AuxT(0);
    }
    if (!grid_sync(c)) return;
    Op op = p.op;
    const uint32_t lane = lane_id();
    const uint64_t pol_first = l2_policy_first(), pol_last = l2_policy_last();
    uint32_t conv_state = 0;  // convergence runs: 1 converged, 2 continue in the push tail
    double last_l1 = 0.0;
    for (uint32_t t = 0; t < p.iters; ++t) {
        maybe_reset_line(&c->line[(t + 2) % 3]);
        {
            LineSum ls;
            read_line(&c->line[t % 3], ls);
            op.D = ls.dsum;
        }
        op.cur = t & 1;
        op.last = p.eps > 0.0 || t + 1 == p.iters;  // a convergence run writes its output every iteration
        if (!Op::kStaticHub || t == 0) {
            // hub cache refresh: 8 independent id -> value chains in flight per thread
            for (uint32_t i0 = threadIdx.x; i0 < p.K; i0 += 8 * BLOCK) {
                uint32_t hid[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) hid[j] = i0 + j * BLOCK < p.K ? __ldg(p.hubs + i0 + j * BLOCK) : 0u;
                HubT hvv[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) hvv[j] = ld_pred(op.src() + hid[j], i0 + j * BLOCK < p.K, pol_last);
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (i0 + j * BLOCK < p.K) s_hub[i0 + j * BLOCK] = hvv[j];
            }
            __syncthreads();
        }
#ifdef SX_PULL_PHASES
        trace_put(p.s, t + 1, DIR_PULL, 7u, cnt, 0, 0, 0);  // hub cache refreshed (CTA 0)
#endif
        PAcc pa;
        uint64_t edges = 0;
        // ---- phase A: edge tiles (software-pipelined: the next tile's ids, row-start
        // bits and first row are loaded while this tile's gathers are in flight)
        uint4 nq[PV / 4];
        uint32_t nrs = 0, nrs1 = 0, nseg = 0;
        auto fetch = [&](uint64_t tl) {
            if (tl < p.ntiles) {
                const uint64_t b = tl * PT, f0 = b + lane * PV;
#pragma unroll
                for (int q = 0; q < PV / 4; ++q) nq[q] = ld_stream(reinterpret_cast<const uint4*>(p.hcol + f0) + q, pol_first);
                nrs = __ldg(p.rs + (f0 >> 5));
                if (lane == 31) nrs1 = __ldg(p.rs + ((b + PT) >> 5));
                nseg = __ldg(p.tile_seg + tl);
            }
        };
        fetch(gwarp());
        for (uint64_t tile = gwarp(); tile < p.ntiles; tile += gwarps()) {
            const uint64_t base = tile * PT, e0 = base + lane * PV;
            uint32_t cols[PV];
#pragma unroll
            for (int q = 0; q < PV / 4; ++q) {
                cols[4 * q] = nq[q].x;
                cols[4 * q + 1] = nq[q].y;
                cols[4 * q + 2] = nq[q].z;
                cols[4 * q + 3] = nq[q].w;
            }
            const uint32_t rsw = nrs, rsw1 = nrs1, seg0 = nseg;
            fetch(tile + gwarps());
            // row starts at e0 .. e0+PV-1
            const uint32_t byte = (rsw >> (uint32_t)(e0 & 31)) & ((1u << PV) - 1u);
            uint32_t nxt = __shfl_down_sync(FULL, byte, 1) & 1u;  // start bit of e0+PV
            if (lane == 31) nxt = rsw1 & 1u;
            const uint32_t ends = (byte >> 1) | (nxt << (PV - 1));  // bit j: edge e0+j is the last of its row
            const bool tile_first_start = __shfl_sync(FULL, byte, 0) & 1u;
            // row starts strictly after the tile's first edge, counted up to each edge
            const uint32_t mb = lane == 0 ? (byte & ~1u) : byte;
            uint32_t ex = __popc(mb);
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(FULL, ex, o);
                if ((int)lane >= o) ex += y;
            }
            ex -= __popc(mb);
            // the lane's first two destination rows and their per-row operands, fetched
            // while the gathers are in flight (most lanes emit at most two rows)
            const uint32_t ra = seg0 + ex;
            const uint32_t u0 = p.nz[ra], u1 = p.nz[ra + 1];
            const typename Op::AuxT* nza = reinterpret_cast<const typename Op::AuxT*>(p.nzaux);
            const typename Op::AuxT a0 = nza[ra], a1 = nza[ra + 1];
            // all PV gathers issued back to back (predicated, no branches), hubs from shared memory
            const HubT* src = op.src();
            HubT hv[PV];
#pragma unroll
            for (int j = 0; j < PV; ++j)
                hv[j] = ld_pred(src + (cols[j] & ~HUBBIT), e0 + j < E && !(cols[j] & HUBBIT), pol_last);
#pragma unroll
            for (int j = 0; j < PV; ++j)
                if (cols[j] & HUBBIT) hv[j] = s_hub[cols[j] & ~HUBBIT];
            TermT x[PV];
            TermT tail = 0;
#pragma unroll
            for (int j = 0; j < PV; ++j) {
                const TermT v = e0 + j < E ? op.term(p.g, e0 + j, hv[j]) : TermT(0);
                x[j] = v;
                if ((byte >> j) & 1u) tail = 0;
                tail += v;
            }
            const uint32_t nvalid = e0 >= E ? 0u : (E - e0 >= (uint64_t)PV ? (uint32_t)PV : (uint32_t)(E - e0));
            edges += nvalid;
            // carry into this lane = inclusive scan of the previous lane
            const double incl = warp_seg_scan((double)tail, byte != 0);
            double carry = __shfl_up_sync(FULL, incl, 1);
            if (lane == 0 || (byte & 1u)) carry = 0.0;
            TermT run = 0;
#pragma unroll
            for (int j = 0; j < PV; ++j) {
                if ((byte >> j) & 1u) {
                    run = 0;
                    carry = 0.0;
                }
                run += x[j];
                if ((uint32_t)j < nvalid && ((ends >> j) & 1u)) {
                    const uint32_t k = __popc(mb & ((2u << j) - 1u));  // row offset within the lane
                    const uint32_t ridx = ra + k;
                    const uint32_t u = k == 0 ? u0 : k == 1 ? u1 : p.nz[ridx];
                    if (u != INF) {
                        const double sum = carry + (double)run;
                        const bool complete = ridx != seg0 || tile_first_start;
                        if (complete) op.apply(u, sum, k == 0 ? a0 : k == 1 ? a1 : op.aux(u), pa);
                        else atomicAdd(p.acc + u, sum);
                    }
                }
            }
            // the tile's last run continues into the next tile: its piece goes to acc
            if (lane == 31 && !nxt && nvalid == PV) {
                const uint32_t k = __popc(mb);
                atomicAdd(p.acc + (k == 0 ? u0 : k == 1 ? u1 : p.nz[ra + k]), incl);
            }
        }
        if (!grid_sync(c)) return;
#ifdef SX_PULL_PHASES
        trace_put(p.s, t + 1, DIR_PULL, 8u, cnt, 0, 0, 0);  // phase A done
#endif
        // ---- phase B: rows split across tiles (from acc), then the empty rows
        for (uint64_t i = gtid(); i < nsplit; i += gthreads()) {
            const uint32_t u = p.sp[cs + i];
            const double a = p.acc[u];
            p.acc[u] = 0.0;
            op.apply(u, a, op.aux(u), pa);
        }
        // An empty row's value depends on no neighbour: it is the same in every
        // iteration (PageRank: up to the common dangling term), so it is written in
        // the first and the last iteration only, unless the operator needs it every
        // iteration (PageRank on a directed graph: an empty in-row can have out-edges).
        if (t == 0 || op.last || op.empty_each_iter()) {
            for (uint64_t i = gtid(); i < nempty; i += gthreads()) {
                const uint32_t u = p.sp[i];
                op.apply(u, 0.0, op.aux(u), pa);
            }
        } else if (lead()) {
            pa.dang += op.empty_dangling(nempty);
        }
        {
            double a[3] = {pa.dang, pa.l1, (double)pa.unstable};
            block_sum<3>(a);
            if (threadIdx.x == 0) {
                Slot& sl = c->line[(t + 1) % 3].s[my_slot()];
                if (a[0] != 0.0) atomicAdd(&sl.dsum, a[0]);
                if (a[1] != 0.0) atomicAdd(&sl.dsum2, a[1]);
                if (a[2] != 0.0) atomicAdd(&sl.mdeg, (unsigned long long)a[2]);
            }
        }
        st.edges += edges;
        if (lead()) st.entries += n;
        ++st.iters;
        if (!grid_sync(c)) return;
        if (p.eps > 0.0) {
            // convergence run: stop at the first iteration whose L1 change is < eps
            // (the oracle's rule); hand over to the push tail once at most a tenth of
            // the vertices still change by more than tau (reading 26)
            LineSum ls;
            read_line(&c->line[(t + 1) % 3], ls);
            trace_put(p.s, t + 1, DIR_PULL, 2u, cnt, n, ls.mdeg, (uint64_t)__double_as_longlong(ls.dsum2));
            last_l1 = ls.dsum2;
            if (ls.dsum2 < p.eps) {
                conv_state = 1;
                break;
            }
            if (p.tail && (p.tail == 2 || (double)ls.mdeg * 14.0 <= (double)E)) {
                conv_state = 2;
                break;
            }
            continue;
        }
        trace_put(p.s, t + 1, DIR_PULL, t == 0 ? 1u : 2u, cnt, n, 0, 0);
    }
    st.pull = st.iters;
    flush_stats(c, st, DIR_PULL);
    if (lead()) {
        c->iter = st.iters;
        c->done = conv_state != 2;
        c->dir = conv_state == 2 ? DIR_PUSH : DIR_PULL;
        c->k = conv_state;
        c->hi = (unsigned long long)__double_as_longlong(last_l1);
        grid_end(c);
        c->launch += 1;
    }
}

template __global__ void pull_all<PrOp>(PullP<PrOp>);
template __global__ void pull_all<SpmvOp>(PullP<SpmvOp>);
template __global__ void pull_all<BpOp>(PullP<BpOp>);
template __global__ void pull_all<PrcOp>(PullP<PrcOp>);


// ---------------------------------------------------------------- PageRank push tail
// "At the end of PageRank, we switch to the push model because the majority
// of the vertices are stable" (the delta-accumulative push of Maiter,
// which the paper cites).  State: r (applied ranks) and rho (change applied to
// r but not yet propagated); invariant r* = r + sum_{k>=1} (dA)^k rho, A the
// (column-(sub)stochastic) transition operator.  An iteration:
//   Active  : vertices with |rho(v)| > tau (ballot filter at entry, then the
//             online filter: a vertex is recorded when an update lifts its
//             |rho| above tau, claimed once per iteration in the next bitmap)
//   harvest : x_v = atomicExch(rho(v), 0) for the active set   -- grid barrier --
//   Compute : update_{v->u} = d x_v / outdeg(v)
//   Combine : sum, atomicAdd (fp64) into r(u) and rho(u)
// A dangling v (variant 0) sends d x_v / N to every vertex: summed per
// iteration into a uniform pending term U, applied to every r and rho once
// |U| > tau, and at the end.  Stops when no |rho| exceeds tau = eps / (4N):
// the unpropagated mass sum |rho| <= 2 N tau = eps/2, so r lies within
// d/(1-d) * eps/2 of the fixed point (reading 26).
struct PrTailP {
    DevGraph g;
    Sched s;
    double* r;
    double* rho;
    double* xv;
    double d, tau, tau0, invN;  // final threshold eps/(4N); first threshold (the mean change at the switch)
    uint32_t variant;
};
struct RhoPred {
    const double* rho;
    double tau;
    __device__ __forceinline__ bool operator()(uint64_t v) const { return fabs(rho[v]) > tau; }
};

__global__ void __launch_bounds__(BLOCK, 4) pr_tail(PrTailP p) {
    Ctl* c = p.s.ctl;
    grid_begin(c);
    stage_init();
    const uint64_t n = p.g.n;
    uint32_t it = vload(&c->iter);
    const uint32_t it0 = it;
    if (blockIdx.x == 0 && warp_id() == 0)
        for (int i = 0; i < 3; ++i) reset_line_warp(&c->line[i]);
    for (int i = 0; i < 3; ++i) clear_bitmap(p.s.bm[i], p.s.nwords);
    if (!grid_sync(c)) return;
    Stats st;
    uint32_t cnt[NCLS];
    // thresholds from the mean change at the switch down to tau, /16 per stage:
    // the largest residuals are pushed first (Maiter's priority order, approximated)
    double tau = p.tau0 > p.tau ? p.tau0 : p.tau;
    RhoPred pred{p.rho, tau};
    if (!ballot_filter(BallotWords<RhoPred>{pred, n}, p.s, BallotOut{p.s.lists[it & 1], p.s.cstride, p.g.dout}, cnt))
        return;
    ++st.ballot;
    st.scanned += lead() ? n : 0;
    if (!grid_sync(c)) return;
    view_contig(cnt);
    double U = 0.0;  // pending uniform change (dangling pushes, variant 0); the same in every CTA
    auto uniform = [&]() -> bool {
        for (uint64_t v = gtid(); v < n; v += gthreads()) {
            p.r[v] += U;
            p.rho[v] += U;
        }
        U = 0.0;
        return grid_sync(c);
    };
    for (;;) {
        if (sum4(cnt) == 0) {
            if (fabs(U) <= tau) {
                if (tau <= p.tau) break;
                tau = tau / 16.0 > p.tau ? tau / 16.0 : p.tau;  // next stage
                pred.tau = tau;
            } else if (!uniform()) {
                return;
            }
            if (!ballot_filter(BallotWords<RhoPred>{pred, n}, p.s, BallotOut{p.s.lists[it & 1], p.s.cstride, p.g.dout},
                               cnt))
                return;
            ++st.ballot;
            st.scanned += lead() ? n : 0;
            if (!grid_sync(c)) return;
            view_contig(cnt);
            continue;
        }
        if (p.s.max_iters && it >= p.s.max_iters) break;
        // harvest the active residuals (every update of the previous iteration has landed)
        const uint32_t* cl = p.s.lists[it & 1];
        for (uint32_t k = 0; k < NCLS; ++k)
            for (uint64_t i = gtid(); i < cnt[k]; i += gthreads()) {
                const uint32_t v = task_at(cl, p.s, k, (uint32_t)i);
                p.xv[v] = __longlong_as_double((long long)atomicExch(reinterpret_cast<unsigned long long*>(p.rho + v), 0ull));
            }
        if (!grid_sync(c)) return;
        IterLine* nx = &c->line[(it + 1) % 3];
        maybe_reset_line(&c->line[(it + 2) % 3]);
        clear_bitmap(p.s.bm[(it + 2) % 3], p.s.nwords);
        uint32_t* nlists = p.s.lists[(it + 1) & 1];
        uint32_t* nbm = p.s.bm[(it + 1) % 3];
        double upart = 0.0;
        uint64_t edges = 0;
        for_tasks(cl, p.s, cnt, [&](uint32_t v, uint64_t rank, uint64_t size, uint32_t) {
            const uint64_t beg = __ldg(p.g.rp + v), end = __ldg(p.g.rp + v + 1);
            const double x = p.xv[v];
            if (beg == end) {
                if (rank == 0 && p.variant == 0) upart += p.d * x * p.invN;
                return;
            }
            const double inc = p.d * x / (double)(end - beg);
            for_edges_b(p.g.ci, beg, end, rank, size, [&](const uint32_t (&u)[4], uint32_t kn) {
                edges += kn;
                double old[4];
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (j < (int)kn) atomicAdd(p.r + u[j], inc);
#pragma unroll
                for (int j = 0; j < 4; ++j) old[j] = j < (int)kn ? atomicAdd(p.rho + u[j], inc) : 0.0;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (j >= (int)kn || !(fabs(old[j] + inc) > tau)) continue;
                    const uint32_t bit = 1u << (u[j] & 31);
                    if (atomicOr(nbm + (u[j] >> 5), bit) & bit) continue;  // claimed once per iteration
                    online_record(nx, nlists, p.s, u[j], cls_of(__ldg(p.g.dout + u[j]), p.s));
                }
            });
        });
        stage_flush(nx, nlists, p.s);
        st.edges += edges;
        if (lead()) st.entries += sum4(cnt);
        {
            double a[1] = {upart};
            block_sum<1>(a);
            if (threadIdx.x == 0 && a[0] != 0.0) atomicAdd(&nx->s[my_slot()].dsum, a[0]);
        }
        if (!grid_sync(c)) return;
        LineSum ls;
        uint32_t vcnt[NCLS];
        read_line_view(nx, p.s, ls, vcnt);
        U += ls.dsum;
        bool overflow = false;
        for (int i = 0; i < NCLS; ++i) overflow |= ls.cntmax[i] > p.s.cap_s;
        if (p.s.force_filter == 2) overflow = true;
        ++it;
        ++st.iters;
        trace_put(p.s, it, DIR_PUSH, overflow ? 1u : 0u, ls.cnt, sum4(ls.cnt), 0, (uint64_t)__double_as_longlong(U));
        if (sum4(ls.cnt) > 0 && overflow) {
            ++st.ballot;
            st.scanned += lead() ? p.s.nwords * 32 : 0;
            if (!ballot_filter(BitmapWords{nbm}, p.s, BallotOut{p.s.lists[it & 1], p.s.cstride, p.g.dout}, cnt)) return;
            if (!grid_sync(c)) return;
            view_contig(cnt);
        } else {
            for (int i = 0; i < NCLS; ++i) cnt[i] = vcnt[i];  // view set by read_line_view
        }
    }
    // the pending uniform term joins r (and rho, so the residual covers what was not propagated)
    if (U != 0.0 && !uniform()) return;
    double* R = reinterpret_cast<double*>(&c->hi);
    if (lead()) *R = 0.0;
    if (!grid_sync(c)) return;
    {
        double a[1] = {0.0};
        for (uint64_t v = gtid(); v < n; v += gthreads()) a[0] += fabs(p.rho[v]);
        block_sum<1>(a);
        if (threadIdx.x == 0 && a[0] != 0.0) atomicAdd(R, a[0]);
    }
    (void)it0;
    flush_stats(c, st, DIR_PUSH);
    if (!grid_sync(c)) return;
    if (lead()) {
        c->iter = it;
        c->done = 1;
        grid_end(c);
        c->launch += 1;
    }
}

// ---------------------------------------------------------------- per-graph plan kernels
__global__ void k_hubslot(const uint32_t* hubs, uint32_t K, uint32_t* slot) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < K; i += gridDim.x * blockDim.x) slot[hubs[i]] = i;
}
__global__ void k_hcol(const uint32_t* ici, uint64_t E, uint64_t Epad, const uint32_t* slot, uint32_t* hcol) {
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < Epad; e += (uint64_t)gridDim.x * blockDim.x) {
        if (e >= E) {
            hcol[e] = 0;
            continue;
        }
        const uint32_t v = ici[e];
        const uint32_t s = slot ? slot[v] : INF;
        hcol[e] = s != INF ? (HUBBIT | s) : v;
    }
}
__global__ void k_rowstarts(const uint64_t* irp, uint64_t n, uint64_t E, uint32_t* rs) {
    for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n; u += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t b = irp[u];
        if (b < irp[u + 1]) atomicOr(rs + (b >> 5), 1u << (b & 31));
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(rs + (E >> 5), 1u << (E & 31));
}
__global__ void k_bp_ctab(double* ctab) {
    if (threadIdx.x < 256) ctab[threadIdx.x] = BpOp::coupling((double)threadIdx.x);
}
// degree-ordered renumbering of the all-active pulls (graph residency)
__global__ void k_pa_newid(const uint32_t* order, uint64_t n, uint32_t* newid) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        newid[order[i]] = (uint32_t)i;
}
template <class T> __global__ void k_pa_gather(const T* src, const uint32_t* idx, uint64_t n, T* dst) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        dst[i] = src[idx[i]];  // dst[new] = src[order[new]] (inputs) or dst[old] = src[newid[old]] (outputs)
}
__global__ void k_pa_keys(const uint64_t* irp, const uint32_t* ici, uint64_t n, const uint32_t* newid, uint64_t* keys) {
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    for (uint64_t u = (((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); u < n; u += nw) {
        const uint64_t b = irp[u], e = irp[u + 1], nr = (uint64_t)newid[u] << 32;
        for (uint64_t x = b + lane; x < e; x += 32) keys[x] = nr | newid[ici[x]];
    }
}
__global__ void k_pa_low32(const uint64_t* keys, uint64_t m, uint32_t* out) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = (uint32_t)keys[i];
}
__global__ void k_pa_rowptr(const uint32_t* din, uint64_t n, uint64_t* tmp) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += (uint64_t)gridDim.x * blockDim.x)
        tmp[i] = i < n ? din[i] : 0ull;
}
__global__ void k_iota(uint32_t* a, uint64_t n) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        a[i] = (uint32_t)i;
}

}  // namespace sx

using namespace sx;

// Per-graph active-row list and tile map for the frontier pulls (SSSP / WCC):
// nz = rows with in-degree > 0 in vertex order, seg[t] = index in nz of the row
// holding tile t's first in-edge (the pull-all kernel builds the same per run
// with its iteration-1 ballot filter).
__global__ void k_tile_seg(const uint64_t* irp, const uint32_t* nz, uint64_t nnz, uint64_t tsz, uint32_t* seg) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t u = nz[k];
        const uint64_t b = irp[u], e = irp[u + 1];
        for (uint64_t t = (b + tsz - 1) / tsz; t * tsz < e; ++t) seg[t] = (uint32_t)k;
    }
}
struct NzFlag {
    const uint32_t* din;
    __host__ __device__ __forceinline__ bool operator()(const uint32_t& v) const { return din[v] > 0; }
};

namespace {

// Per-graph plan of the tiled pull (graph residency, built on first use):
// hub selection (top-K out-degree), encoded sources, row-start bitmap.
#define TRYA(x)                          \
    do {                                 \
        sx_status r__ = (x);             \
        if (r__ != SX_OK) return r__;    \
    } while (0)
// Row-start bitmap over the in-edges (bit e = first edge of a row, bit E = a
// sentinel start), sized for the largest tile of either pull.
sx_status prep_rs(sx_graph g) {
    if (g->pp_rs) return SX_OK;
    const uint64_t n = g->n, E = g->mi;
    const uint64_t tmax = PT > MPT ? PT : MPT;
    const uint64_t rsw = ((E + tmax - 1) / tmax * tmax + tmax) / 32 + 4;
    TRYA(sxh::dmalloc(g->ctx, &g->pp_rs, rsw * 4));
    SX_CU(cudaMemsetAsync(g->pp_rs, 0, rsw * 4, g->ctx->stream));
    k_rowstarts<<<8 * g->ctx->prop.multiProcessorCount, 256, 0, g->ctx->stream>>>(g->irp, n, E, g->pp_rs);
    SX_CU(cudaGetLastError());
    return SX_OK;
}


// The all-active pulls run on a renumbered copy of the in-rows: vertex ids by
// descending out-degree (ties by id), so the sources gathered most often sit
// together (the hub cache holds ids 0..K-1 and the values behind it share
// 32-B sectors and L1 lines; measured on C3: 14.8 -> 11.4 ms, profiles/r2/pr_relabel.txt).
// Rows are re-sorted by the new source ids.  Built once per graph; inputs
// are gathered into the new order per run and outputs scattered back.
sx_status prep_relabel(sx_graph g) {
    if (g->pa_irp) return SX_OK;
    cudaStream_t s = g->ctx->stream;
    const uint64_t n = g->n, E = g->mi;
    const int eg = 8 * g->ctx->prop.multiProcessorCount;
    sx_ctx c = g->ctx;
    uint32_t *kout = nullptr, *vin = nullptr;
    void* tmp = nullptr;
    size_t tb = 0;
    TRYA(sxh::dmalloc(c, &g->pa_order, n * 4 + 16));
    TRYA(sxh::dmalloc(c, &g->pa_newid, n * 4 + 16));
    TRYA(sxh::dmalloc(c, &kout, n * 4 + 16));
    TRYA(sxh::dmalloc(c, &vin, n * 4 + 16));
    k_iota<<<eg, 256, 0, s>>>(vin, n);
    SX_CU(cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, g->dout, kout, vin, g->pa_order, (int64_t)n, 0, 32, s));
    TRYA(sxh::dmalloc(c, &tmp, tb ? tb : 1));
    SX_CU(cub::DeviceRadixSort::SortPairsDescending(tmp, tb, g->dout, kout, vin, g->pa_order, (int64_t)n, 0, 32, s));
    SX_CU(cudaStreamSynchronize(s));
    sxh::dfree(c, tmp);
    tmp = nullptr;
    k_pa_newid<<<eg, 256, 0, s>>>(g->pa_order, n, g->pa_newid);
    TRYA(sxh::dmalloc(c, &g->pa_dout, n * 4 + 16));
    TRYA(sxh::dmalloc(c, &g->pa_din, n * 4 + 16));
    k_pa_gather<<<eg, 256, 0, s>>>(g->dout, g->pa_order, n, g->pa_dout);
    k_pa_gather<<<eg, 256, 0, s>>>(g->din, g->pa_order, n, g->pa_din);
    // row pointers: exclusive scan of the renumbered in-degrees
    uint64_t* deg64 = nullptr;
    TRYA(sxh::dmalloc(c, &deg64, (n + 1) * 8));
    TRYA(sxh::dmalloc(c, &g->pa_irp, (n + 1) * 8 + 16));
    k_pa_rowptr<<<eg, 256, 0, s>>>(g->pa_din, n, deg64);
    tb = 0;
    SX_CU(cub::DeviceScan::ExclusiveSum(nullptr, tb, deg64, g->pa_irp, (int64_t)(n + 1), s));
    TRYA(sxh::dmalloc(c, &tmp, tb ? tb : 1));
    SX_CU(cub::DeviceScan::ExclusiveSum(tmp, tb, deg64, g->pa_irp, (int64_t)(n + 1), s));
    SX_CU(cudaStreamSynchronize(s));
    sxh::dfree(c, tmp);
    tmp = nullptr;
    sxh::dfree(c, deg64);
    // edges: key (new row << 32 | new source), sorted; weights ride along
    uint64_t *k0 = nullptr, *k1 = nullptr;
    TRYA(sxh::dmalloc(c, &k0, E * 8 + 16));
    TRYA(sxh::dmalloc(c, &k1, E * 8 + 16));
    k_pa_keys<<<eg, 256, 0, s>>>(g->irp, g->ici, n, g->pa_newid, k0);
    TRYA(sxh::dmalloc(c, &g->pa_ici, E * 4 + 16));
    tb = 0;
    if (g->wbytes) {
        TRYA(sxh::dmalloc(c, &g->pa_iw, E * g->wbytes + 16));
        if (g->wbytes == 1) {
            SX_CU(cub::DeviceRadixSort::SortPairs(nullptr, tb, k0, k1, (const uint8_t*)g->iw, (uint8_t*)g->pa_iw, (int64_t)E, 0, 64, s));
            TRYA(sxh::dmalloc(c, &tmp, tb ? tb : 1));
            SX_CU(cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, (const uint8_t*)g->iw, (uint8_t*)g->pa_iw, (int64_t)E, 0, 64, s));
        } else {
            SX_CU(cub::DeviceRadixSort::SortPairs(nullptr, tb, k0, k1, (const uint32_t*)g->iw, (uint32_t*)g->pa_iw, (int64_t)E, 0, 64, s));
            TRYA(sxh::dmalloc(c, &tmp, tb ? tb : 1));
            SX_CU(cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, (const uint32_t*)g->iw, (uint32_t*)g->pa_iw, (int64_t)E, 0, 64, s));
        }
    } else {
        SX_CU(cub::DeviceRadixSort::SortKeys(nullptr, tb, k0, k1, (int64_t)E, 0, 64, s));
        TRYA(sxh::dmalloc(c, &tmp, tb ? tb : 1));
        SX_CU(cub::DeviceRadixSort::SortKeys(tmp, tb, k0, k1, (int64_t)E, 0, 64, s));
    }
    k_pa_low32<<<eg, 256, 0, s>>>(k1, E, g->pa_ici);
    SX_CU(cudaGetLastError());
    SX_CU(cudaStreamSynchronize(s));
    sxh::dfree(c, tmp);
    sxh::dfree(c, k0);
    sxh::dfree(c, k1);
    sxh::dfree(c, kout);
    sxh::dfree(c, vin);
    // row starts of the renumbered in-edges (the pull-all tiles)
    const uint64_t rsw = ((E + PT - 1) / PT * PT + PT) / 32 + 4;
    TRYA(sxh::dmalloc(c, &g->pa_rs, rsw * 4));
    SX_CU(cudaMemsetAsync(g->pa_rs, 0, rsw * 4, s));
    k_rowstarts<<<eg, 256, 0, s>>>(g->pa_irp, n, E, g->pa_rs);
    SX_CU(cudaGetLastError());
    return SX_OK;
}

// The renumbered graph as the pull-all kernels see it.
sx::DevGraph pa_graph(const sx_graph g) {
    sx::DevGraph d = sxh::dev_graph(g);
    d.irp = g->pa_irp;
    d.ici = g->pa_ici;
    d.iw8 = g->wbytes == 1 ? (const uint8_t*)g->pa_iw : nullptr;
    d.iw32 = g->wbytes == 4 ? (const uint32_t*)g->pa_iw : nullptr;
    d.dout = g->pa_dout;
    d.din = g->pa_din;
    return d;
}

sx_status prep(sx_graph g, const char* who) {
    if (g->directed && !g->has_rev)
        return sxh::fail(SX_E_NO_REVERSE, std::string(who) + ": pull needs in-neighbour rows (CSC)");
    if (g->pp_hcol) return SX_OK;
    cudaStream_t s = g->ctx->stream;
    const uint64_t n = g->n, E = g->mi;
    const uint64_t ntiles = (E + PT - 1) / PT;
    const uint64_t epad = ntiles * PT + PT;
    const int eg = 8 * g->ctx->prop.multiProcessorCount;
    TRYA(sxh::dmalloc(g->ctx, &g->hacc, (n + 1) * sizeof(double)));
    SX_CU(cudaMemsetAsync(g->hacc, 0, (n + 1) * sizeof(double), s));
    TRYA(sxh::dmalloc(g->ctx, &g->pp_tile_seg, (ntiles + 1) * 4));
    TRYA(sxh::dmalloc(g->ctx, &g->pp_nzaux, (n + 2) * 4));
    TRYA(sxh::dmalloc(g->ctx, &g->pp_hcol, epad * 4));
    TRYA(prep_relabel(g));
    // hubs: the K sources of largest out-degree (each is gathered outdeg times per iteration)
    uint32_t K = (uint32_t)std::min<uint64_t>(PULL_HUBS, n);
#ifdef SX_PULL_NOHUB
    K = 0;
#endif
    if (n >= HUBBIT) K = 0;  // ids need the top bit free for the encoding
    TRYA(sxh::dmalloc(g->ctx, &g->pp_hubs, (K ? K : 1) * 4));
    uint32_t* slot = nullptr;
    if (K) {
        uint32_t *kin = nullptr, *kout = nullptr, *vin = nullptr, *vout = nullptr;
        void* tmp = nullptr;
        size_t tb = 0;
        TRYA(sxh::dmalloc(g->ctx, &kout, n * 4));
        TRYA(sxh::dmalloc(g->ctx, &vin, n * 4));
        TRYA(sxh::dmalloc(g->ctx, &vout, n * 4));
        kin = g->pa_dout;  // already descending: the hubs are ids 0..K-1
        k_iota<<<eg, 256, 0, s>>>(vin, n);
        SX_CU(cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, kin, kout, vin, vout, (int64_t)n, 0, 32, s));
        TRYA(sxh::dmalloc(g->ctx, &tmp, tb ? tb : 1));
        SX_CU(cub::DeviceRadixSort::SortPairsDescending(tmp, tb, kin, kout, vin, vout, (int64_t)n, 0, 32, s));
        SX_CU(cudaMemcpyAsync(g->pp_hubs, vout, K * 4, cudaMemcpyDeviceToDevice, s));
        SX_CU(cudaMemsetAsync(vin, 0xFF, n * 4, s));
        slot = vin;
        k_hubslot<<<eg, 256, 0, s>>>(g->pp_hubs, K, slot);
        k_hcol<<<eg, 256, 0, s>>>(g->pa_ici, E, epad, slot, g->pp_hcol);
        SX_CU(cudaStreamSynchronize(s));
        sxh::dfree(g->ctx, tmp);
        sxh::dfree(g->ctx, kout);
        sxh::dfree(g->ctx, vin);
        sxh::dfree(g->ctx, vout);
    } else {
        k_hcol<<<eg, 256, 0, s>>>(g->pa_ici, E, epad, nullptr, g->pp_hcol);
    }
    SX_CU(cudaGetLastError());
    SX_CU(cudaStreamSynchronize(s));
    g->pp_K = K;
    g->pp_ntiles = ntiles;
    return SX_OK;
}

// Algorithmic bytes of one pull-all iteration: every in-edge once
// (encoded source 4 B + gathered source value + weight bytes + 1/8 B row-start
// bit), every vertex once (state read/write, set per operator).
thread_local double t_edge_bytes = 0, t_vertex_bytes = 0;
static double pull_bytes(const sx_graph g, const sxh::Counters& c) {
    return c.iters * ((double)g->mi * (t_edge_bytes + 0.125) + (double)g->n * t_vertex_bytes) + c.scanned / 8.0;
}

template <class Op> PullP<Op> pull_params(sx_graph g, const sxh::Run& run, const Op& op, uint32_t iters) {
    PullP<Op> p;
    p.g = pa_graph(g);  // the degree-ordered in-rows
    p.s = sxh::make_sched(g, run.o);
    p.op = op;
    p.iters = iters;
    p.hcol = g->pp_hcol;
    p.rs = g->pa_rs;
    p.hubs = g->pp_hubs;
    p.K = g->pp_K;
    p.ntiles = g->pp_ntiles;
    p.E = g->mi;
    p.tile_seg = g->pp_tile_seg;
    p.nz = g->lists[0];
    p.nzaux = g->pp_nzaux;
    p.sp = g->lists[1];
    p.acc = g->hacc;
    p.eps = 0.0;
    p.tail = 0;
    return p;
}

template <class Op>
sx_status run_pull(sx_graph g, const sx_opts* opts, sx_stats* stats, const Op& op, uint32_t iters, double edge_bytes,
                   double vertex_bytes, double eps = 0.0) {
    sxh::Run run{g, sxh::resolve_opts(opts), stats};
    run.o.cluster_enter = sxh::resolve_cluster(run.o.cluster_enter, false, g->n);
    sx_status rc = run.begin();
    if (rc != SX_OK) return rc;
    PullP<Op> p = pull_params(g, run, op, iters);
    p.eps = eps;
    void* args[] = {&p};
    const int smem = (int)(PULL_HUBS * sizeof(typename Op::HubT));
    if ((rc = run.launch((const void*)pull_all<Op>, args, sxh::KIND_PULL, smem)) != SX_OK) return rc;
    t_edge_bytes = edge_bytes;
    t_vertex_bytes = vertex_bytes;
    rc = run.end(pull_bytes);
    if (rc == SX_OK && stats) {
        const unsigned long long h = g->ctx->h_ctl->hi;
        double last = 0.0;
        std::memcpy(&last, &h, 8);
        stats->residual = eps > 0.0 ? last : 0.0;
    }
    return rc;
}


}  // namespace

namespace sxh {
sx_status min_pull_plan(sx_graph g) {
    if (g->pp_gnz) return SX_OK;
    TRYA(prep_rs(g));
    cudaStream_t s = g->ctx->stream;
    const uint64_t n = g->n;
    const int eg = 8 * g->ctx->prop.multiProcessorCount;
    TRYA(sxh::dmalloc(g->ctx, &g->pp_gnz, (n + 2) * 4));
    const uint64_t gtiles = (g->mi + MPT - 1) / MPT;
    TRYA(sxh::dmalloc(g->ctx, &g->pp_gseg, (gtiles + 1) * 4));
    unsigned long long* dcnt = nullptr;
    TRYA(sxh::dmalloc(g->ctx, &dcnt, 8));
    thrust::counting_iterator<uint32_t> it(0);
    size_t tb = 0;
    SX_CU(cub::DeviceSelect::If(nullptr, tb, it, g->pp_gnz, dcnt, (int64_t)n, NzFlag{g->din}, s));
    void* tmp = nullptr;
    TRYA(sxh::dmalloc(g->ctx, &tmp, tb ? tb : 1));
    SX_CU(cub::DeviceSelect::If(tmp, tb, it, g->pp_gnz, dcnt, (int64_t)n, NzFlag{g->din}, s));
    unsigned long long nnz = 0;
    SX_CU(cudaMemcpyAsync(&nnz, dcnt, 8, cudaMemcpyDeviceToHost, s));
    SX_CU(cudaStreamSynchronize(s));
    k_tile_seg<<<eg, 256, 0, s>>>(g->irp, g->pp_gnz, nnz, MPT, g->pp_gseg);
    const uint32_t sentinel[2] = {INF, INF};  // nz[nnz] = the sentinel row of start bit E
    SX_CU(cudaMemcpyAsync(g->pp_gnz + nnz, sentinel, 8, cudaMemcpyHostToDevice, s));
    SX_CU(cudaGetLastError());
    SX_CU(cudaStreamSynchronize(s));
    sxh::dfree(g->ctx, tmp);
    sxh::dfree(g->ctx, dcnt);
    g->pp_gnnz = nnz;
    g->pp_gntiles = gtiles;
    return SX_OK;
}
}  // namespace sxh

// Outputs of the renumbered pulls back to the caller's ids: dst[old] = src[newid[old]]
// (dst: the caller's device buffer, or `stage` then a copy to a host buffer).
template <class T> static sx_status pa_out(sx_graph g, T* user, bool dev_out, const T* src, T* stage) {
    T* dst = dev_out ? user : stage;
    k_pa_gather<<<8 * g->ctx->prop.multiProcessorCount, 256, 0, g->ctx->stream>>>(src, g->pa_newid, g->n, dst);
    SX_CU(cudaGetLastError());
    if (dev_out) {
        SX_CU(cudaStreamSynchronize(g->ctx->stream));
        return SX_OK;
    }
    return sxh::copy_out(g, user, stage, g->n * sizeof(T));
}
// An input vector into the renumbered order: dst[new] = src[order[new]].
template <class T> static void pa_in(sx_graph g, const T* src, T* dst) {
    k_pa_gather<<<8 * g->ctx->prop.multiProcessorCount, 256, 0, g->ctx->stream>>>(src, g->pa_order, g->n, dst);
}

extern "C" sx_status sx_pagerank(sx_graph g, float damping, uint32_t iters, const sx_opts* opts, float* rank_out,
                                 sx_stats* stats) {
    if (!g || !rank_out) return sxh::fail(SX_E_INVALID, "sx_pagerank: NULL graph or rank_out");
    sx_status rc = sxh::check_ctx(g->ctx);
    if (rc != SX_OK) return rc;
    if (!(damping >= 0.f && damping <= 1.f)) return sxh::fail(SX_E_INVALID, "sx_pagerank: damping outside [0,1]");
    if (iters == 0) return sxh::fail(SX_E_INVALID, "sx_pagerank: iters must be >= 1");
    if (g->n == 0) return SX_OK;
    if ((rc = prep(g, "sx_pagerank")) != SX_OK) return rc;
    const bool dev_out = sxh::is_device_ptr(rank_out);
    PrOp op;
    op.contrib[0] = (float*)g->st[0];
    op.contrib[1] = (float*)g->st[1];
    op.out = (float*)g->st[2];  // renumbered; scattered back below
    op.dout = g->pa_dout;
    op.d = damping;
    op.invN = 1.0 / (double)g->n;
    op.directed = g->directed;
    op.cur = 0;
    op.D = 0;
    op.last = false;
    // SURVEY §8(d) rule (each array at most once per pass): edge: source id 4 B;
    // vertex: contrib read 4 + contrib write 4 + outdeg 4 (the gathers of
    // contrib are bounded by its size, counted per vertex)
    if ((rc = run_pull(g, opts, stats, op, iters, 4.0, 12.0)) != SX_OK) return rc;
    return pa_out(g, rank_out, dev_out, op.out, (float*)g->st[3]);
}

extern "C" sx_status sx_spmv(sx_graph g, const float* x, uint32_t iters, const sx_opts* opts, float* y_out,
                             sx_stats* stats) {
    if (!g || !x || !y_out) return sxh::fail(SX_E_INVALID, "sx_spmv: NULL argument");
    sx_status rc = sxh::check_ctx(g->ctx);
    if (rc != SX_OK) return rc;
    if (iters == 0) return sxh::fail(SX_E_INVALID, "sx_spmv: iters must be >= 1");
    if (g->n == 0) return SX_OK;
    if ((rc = prep(g, "sx_spmv")) != SX_OK) return rc;
    const bool dev_out = sxh::is_device_ptr(y_out);
    SpmvOp op;
    float* dx = (float*)g->st[0];
    if ((rc = sxh::copy_in(g, dx, x, g->n * 4)) != SX_OK) return rc;
    pa_in(g, (const float*)dx, (float*)g->st[2]);  // x in the renumbered order
    op.x = (float*)g->st[2];
    op.out = (float*)g->st[1];
    op.cur = 0;
    op.D = 0;
    op.last = false;
    // edge: source id 4 + weight; vertex: x 4 + y 4
    if ((rc = run_pull(g, opts, stats, op, iters, 4.0 + g->wbytes, 8.0)) != SX_OK) return rc;
    return pa_out(g, y_out, dev_out, op.out, (float*)g->st[3]);
}

extern "C" sx_status sx_bp(sx_graph g, const float* prior, uint32_t iters, const sx_opts* opts, float* logodds_out,
                           sx_stats* stats) {
    if (!g || !prior || !logodds_out) return sxh::fail(SX_E_INVALID, "sx_bp: NULL argument");
    sx_status rc = sxh::check_ctx(g->ctx);
    if (rc != SX_OK) return rc;
    if (iters == 0) return sxh::fail(SX_E_INVALID, "sx_bp: iters must be >= 1");
    if (g->n == 0) return SX_OK;
    if ((rc = prep(g, "sx_bp")) != SX_OK) return rc;
    if (!g->dstate && (rc = sxh::dmalloc(g->ctx, &g->dstate, (2 * g->n + 256) * sizeof(double))) != SX_OK) return rc;
    k_bp_ctab<<<1, 256, 0, g->ctx->stream>>>(g->dstate + 2 * g->n);
    SX_CU(cudaGetLastError());
    const bool dev_out = sxh::is_device_ptr(logodds_out);
    BpOp op;
    op.b[0] = g->dstate;
    op.b[1] = g->dstate + g->n;
    op.ctab = g->dstate + 2 * g->n;
    float* dp = (float*)g->st[2];
    if ((rc = sxh::copy_in(g, dp, prior, g->n * 4)) != SX_OK) return rc;
    pa_in(g, (const float*)dp, (float*)g->st[0]);  // priors in the renumbered order
    op.prior = (float*)g->st[0];
    op.out = (float*)g->st[3];
    op.cur = 0;
    op.D = 0;
    op.last = false;
    op.conv = false;
    // edge: source id 4 + weight; vertex: belief read 8 + belief write 8 + prior 4
    if ((rc = run_pull(g, opts, stats, op, iters, 4.0 + g->wbytes, 20.0)) != SX_OK) return rc;
    return pa_out(g, logodds_out, dev_out, op.out, (float*)g->st[1]);
}

extern "C" sx_status sx_bp_conv(sx_graph g, const float* prior, double epsilon, uint32_t max_iters,
                                const sx_opts* opts, float* logodds_out, sx_stats* stats) {
    if (!g || !prior || !logodds_out) return sxh::fail(SX_E_INVALID, "sx_bp_conv: NULL argument");
    sx_status rc = sxh::check_ctx(g->ctx);
    if (rc != SX_OK) return rc;
    if (!(epsilon > 0.0)) return sxh::fail(SX_E_INVALID, "sx_bp_conv: epsilon must be > 0");
    if (max_iters == 0) return sxh::fail(SX_E_INVALID, "sx_bp_conv: max_iters must be >= 1");
    if (g->n == 0) return SX_OK;
    if ((rc = prep(g, "sx_bp_conv")) != SX_OK) return rc;
    if (!g->dstate && (rc = sxh::dmalloc(g->ctx, &g->dstate, (2 * g->n + 256) * sizeof(double))) != SX_OK) return rc;
    k_bp_ctab<<<1, 256, 0, g->ctx->stream>>>(g->dstate + 2 * g->n);
    SX_CU(cudaGetLastError());
    const bool dev_out = sxh::is_device_ptr(logodds_out);
    BpOp op;
    op.b[0] = g->dstate;
    op.b[1] = g->dstate + g->n;
    op.ctab = g->dstate + 2 * g->n;
    float* dp = (float*)g->st[2];
    if ((rc = sxh::copy_in(g, dp, prior, g->n * 4)) != SX_OK) return rc;
    pa_in(g, (const float*)dp, (float*)g->st[0]);  // priors in the renumbered order
    op.prior = (float*)g->st[0];
    op.out = (float*)g->st[3];
    op.cur = 0;
    op.D = 0;
    op.last = true;
    op.conv = true;
    if ((rc = run_pull(g, opts, stats, op, max_iters, 4.0 + g->wbytes, 24.0, epsilon)) != SX_OK) return rc;
    return pa_out(g, logodds_out, dev_out, op.out, (float*)g->st[1]);
}

// Algorithmic bytes of the push tail: per harvested entry 4 B list +
// 16 B row_ptr + 8 B rho exchange + 8 B x; per pushed edge 4 B col + 2 x 8 B fp64
// read-modify-writes (r, rho); ballot passes 8 B rho per vertex.
static double prtail_bytes(const sx_graph g, const sxh::Counters& c) {
    return 36.0 * c.entries + 20.0 * c.edges + 8.0 * c.scanned + c.iters * (double)g->n / 8.0;
}
static double prc_bytes(const sx_graph g, const sxh::Counters& c) {
    if (c.pull > 0) return pull_bytes(g, c);
    return prtail_bytes(g, c);
}

extern "C" sx_status sx_pagerank_conv(sx_graph g, double damping, double epsilon, uint32_t max_iters, uint32_t variant,
                                      const sx_opts* opts, double* rank_out, sx_stats* stats) {
    if (!g || !rank_out) return sxh::fail(SX_E_INVALID, "sx_pagerank_conv: NULL graph or rank_out");
    sx_status rc = sxh::check_ctx(g->ctx);
    if (rc != SX_OK) return rc;
    if (!(damping > 0.0 && damping < 1.0)) return sxh::fail(SX_E_INVALID, "sx_pagerank_conv: damping outside (0,1)");
    if (!(epsilon > 0.0)) return sxh::fail(SX_E_INVALID, "sx_pagerank_conv: epsilon must be > 0");
    if (max_iters == 0) return sxh::fail(SX_E_INVALID, "sx_pagerank_conv: max_iters must be >= 1");
    if (variant > SX_PR_SPEC) return sxh::fail(SX_E_INVALID, "sx_pagerank_conv: unknown variant");
    if (g->n == 0) return SX_OK;
    if ((rc = prep(g, "sx_pagerank_conv")) != SX_OK) return rc;
    const uint64_t n = g->n;
    if (!g->prc && (rc = sxh::dmalloc(g->ctx, &g->prc, 5 * n * sizeof(double) + 64)) != SX_OK) return rc;
    const bool dev_out = sxh::is_device_ptr(rank_out);
    sxh::Run run{g, sxh::resolve_opts(opts), stats};
    if ((rc = run.begin()) != SX_OK) return rc;
    const double d = damping;
    PrcOp op;
    op.contrib[0] = g->prc;
    op.contrib[1] = g->prc + n;
    op.r = g->prc + 2 * n;    // renumbered
    op.rho = g->prc + 3 * n;
    op.dout = g->pa_dout;
    op.d = d;
    op.base = variant == SX_PR_NORMALIZED ? (1.0 - d) / (double)n : 1.0 - d;
    op.dn = variant == SX_PR_NORMALIZED ? 1.0 / (double)n : 0.0;
    op.r0 = variant == SX_PR_NORMALIZED ? 1.0 / (double)n : 1.0;
    op.tau = epsilon / (4.0 * (double)n);
    op.cur = 0;
    op.D = 0;
    op.last = true;
    PullP<PrcOp> p = pull_params(g, run, op, max_iters);
    p.eps = epsilon;
    p.tail = run.o.force_dir == 2 ? 0u : run.o.force_dir == 1 ? 2u : 1u;
    void* args[] = {&p};
    const int smem = (int)(PULL_HUBS * sizeof(double));
    if ((rc = run.launch((const void*)pull_all<PrcOp>, args, sxh::KIND_PULL, smem)) != SX_OK) return rc;
    if ((rc = run.sync()) != SX_OK) return rc;
    const Ctl& h = *g->ctx->h_ctl;
    double* r_final = op.r;
    bool renumbered = true;
    if (!h.done && h.dir == DIR_PUSH && h.iter < max_iters) {
        // the tail pushes along the out-rows in the caller's ids: r and rho go back first
        double* r_old = g->prc;  // the contribution arrays are free now
        double* rho_old = g->prc + n;
        const int eg = 8 * g->ctx->prop.multiProcessorCount;
        k_pa_gather<<<eg, 256, 0, g->ctx->stream>>>(op.r, g->pa_newid, n, r_old);
        k_pa_gather<<<eg, 256, 0, g->ctx->stream>>>(op.rho, g->pa_newid, n, rho_old);
        SX_CU(cudaGetLastError());
        r_final = r_old;
        renumbered = false;
        PrTailP q;
        q.g = sxh::dev_graph(g);
        q.s = p.s;
        q.s.max_iters = max_iters;
        q.r = r_old;
        q.rho = rho_old;
        q.xv = g->prc + 4 * n;
        q.d = d;
        q.tau = op.tau;
        q.tau0 = op.tau;  // one stage: the tail pushes every change above tau
        q.invN = 1.0 / (double)n;
        q.variant = variant;
        void* args2[] = {&q};
        if ((rc = run.launch((const void*)pr_tail, args2, sxh::KIND_PUSH)) != SX_OK) return rc;
    }
    // edge: source id 4 + gathered contrib 8; vertex: r read/write 16, rho write 8, contrib write 8, outdeg 4
    t_edge_bytes = 12.0;
    t_vertex_bytes = 36.0;
    if ((rc = run.end(prc_bytes)) != SX_OK) return rc;
    if (stats) {
        double res = 0.0;
        const unsigned long long hh = g->ctx->h_ctl->hi;
        std::memcpy(&res, &hh, 8);
        stats->residual = res;
    }
    if (renumbered) return pa_out(g, rank_out, dev_out, (const double*)r_final, g->prc + 4 * n);
    if (dev_out) {
        SX_CU(cudaMemcpyAsync(rank_out, r_final, n * 8, cudaMemcpyDeviceToDevice, g->ctx->stream));
        SX_CU(cudaStreamSynchronize(g->ctx->stream));
        return SX_OK;
    }
    return sxh::copy_out(g, rank_out, r_final, n * 8);
}

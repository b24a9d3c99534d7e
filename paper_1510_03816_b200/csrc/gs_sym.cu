// gs_sym.cu — symmetric all-pairs fp64 RHS (single rank, all rows).
//
// The pair term is symmetric in (i, j): G_ij = G_ji, c_ij = (p_i.p_j) G'(d)/d = c_ji and
// q_j - q_i = -(q_i - q_j) (particles.py:100-116).  Each unordered pair is therefore
// evaluated once and feeds both rows — ~16 FP64-pipe slots per ordered pair instead of the
// ~28 of the one-sided kernel (gs_dense.cu) and the 45 of the libm formulation.
//
// Work decomposition.  Rows are cut in blocks of 128 (nb blocks) and blocks in superblocks
// of G (nsb = ceil(nb/G) <= ~256).  One CTA (2 warps) owns a superblock pair (SI <= SJ) and
// walks its 128 x 128 tiles (I in SI, J in SJ, I <= J):
//   * warp w owns 64 targets of I, two per lane (rows w*64 + lane and w*64 + 32 + lane):
//     positions, momenta and I-side accumulators in registers;
//   * the warp visits the 4 source sub-blocks (32 records) of J in phases ph = 0..3
//     (sub-block (2w + ph) & 3, so the two warps of a phase never share a source);
//   * inside a phase lane l pairs both its targets with source (l + t) & 31 at step t, read
//     from a doubled copy of the sub-block (64 records: the rotated index is a constant
//     offset); the source's 4 accumulators travel with it around the warp (one shuffle
//     from lane l+1 per step, shared by the two targets), so after 32 steps lane l holds the
//     complete contribution of the warp's 64 targets to source l and adds it to the CTA's
//     shared accumulator of block J;
//   * diagonal tiles (I == J) are evaluated one-sided.
// Why two targets per lane: with one, the per-step shared-memory traffic (rotated 32-byte
// source records, table lookups, 8 shuffles) saturated the LSU pipe (96% in ncu) before the
// FP64 pipe; sharing the source read and the shuffles between two targets halves it.  Each
// rotation step takes two sources (GS_SYM_SRC2), so a lane runs four independent pair chains
// against the FP64 latency ("wait" stalls were the top stall reason with two).
// d == 0 pairs are exact through the lean pair core (gs_device.cuh); interacting coincident
// particles are re-scanned on the rare flagged tile (reference error, particles.py:92-98).
// Partials: the I-side of block I over superblock SJ goes to slot SJ, the J-side of block J
// over superblock SI goes to slot SI (in a diagonal superblock both land in one shared
// accumulator, slot SI).  Every row receives exactly nsb partials, part[slot * pstride + row],
// summed in slot order by k_finish — deterministic.
#include <atomic>

#include "gs_kernels.cuh"

namespace gsb {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kST = 64;  // threads per CTA
#ifndef GS_SYM_MINB      // resident CTAs per SM the register allocation is bounded for (A/B builds)
#define GS_SYM_MINB 6  // A/B on C2 (one source per step): 6 -> 0.374 ms, 8 -> 0.377, 10 -> 0.391, 12 -> 0.401
#endif
#ifndef GS_SYM_SB        // superblock count above which blocks are grouped (A/B builds)
#define GS_SYM_SB 256  // A/B on C2 (ms per 100-step solve): 128 -> 152.8, 64 -> 165.4, 32 -> 178.7; on C3 (N = 131072,
                       // ms per RHS, 16 KB exp table): 128 (G = 8: 57 KB of shared memory, 3 CTAs/SM) -> 23.44,
                       // 256 (G = 4, 5 CTAs/SM; 1 GB of partials, 0.17 ms of k_finish) -> 20.90
#endif
#ifndef GS_SYM_UNROLL     // unroll of the two-source rotation loop (16 trips)
#define GS_SYM_UNROLL 4  // A/B on C2 (ms per 100-step solve, bulk-copy prologue, 152-160 regs): 1 -> 138.1,
                         // 2 -> 139.5, 4 -> 137.1, 8 -> 150.6 (spills), 16 -> 164.9 (round 1, 160 regs: 2 best)
#endif
constexpr int kSymUnroll = GS_SYM_UNROLL;
#ifndef GS_SYM_SRC2      // two sources per rotation step: 4 independent pair chains per lane
#define GS_SYM_SRC2 1    // A/B on C2: 0.364 ms (minb 6, 158 regs) vs 0.383 ms (minb 8, 128 regs) vs 0.374
#endif

struct Acc {
    double qx, qy, px, py;
};

template <int FAM>
__device__ __forceinline__ void one_sided(const double4& me, const double4& s, const double* tbl, double k1, Acc& a,
                                          int& nz) {
    const double dx = me.x - s.x, dy = me.y - s.y;
    const double pdot = fma(me.z, s.z, me.w * s.w);
    double g, c;
    int z;
    pair_core<FAM>(dx, dy, pdot, tbl, k1, g, c, z);
    a.qx = fma(g, s.z, a.qx);
    a.qy = fma(g, s.w, a.qy);
    a.px = fma(c, dx, a.px);
    a.py = fma(c, dy, a.py);
    nz += z;
}

#ifndef GS_SYM_ZMIN      // coincidence detection by the minimum high word of d^2 (1 op per pair, A/B)
#define GS_SYM_ZMIN 1
#endif

template <int FAM>
__device__ __forceinline__ void two_sided(const double4& me, const double4& s, const double* tbl, unsigned tb,
                                          double k1, int caphi, Acc& a, Acc& j, int& nz) {
    const double dx = me.x - s.x, dy = me.y - s.y;
    const double pdot = fma(me.z, s.z, me.w * s.w);
    double g, c;
#if GS_SYM_ZMIN
    int h;
    pair_core_hi<FAM>(dx, dy, pdot, tb, k1, caphi, g, c, h);
    nz = min(nz, h);  // nz: the minimum high word of d^2 (see pair_core_hi)
#else
    int z;
    pair_core<FAM>(dx, dy, pdot, tbl, k1, g, c, z);
    nz += z;
#endif
    a.qx = fma(g, s.z, a.qx);
    a.qy = fma(g, s.w, a.qy);
    a.px = fma(c, dx, a.px);
    a.py = fma(c, dy, a.py);
    j.qx = fma(g, me.z, j.qx);
    j.qy = fma(g, me.w, j.qy);
    j.px = fma(-c, dx, j.px);
    j.py = fma(-c, dy, j.py);
}

// The J tile into s_rot by 8 bulk copies (each 32-record sub-block twice, the rotation's doubled
// layout) on the tile mbarrier — one thread, no registers, overlapping the CTA's setup for the
// first tile.  Full tiles only (a partial last tile takes the thread loop and its far records).
__device__ __forceinline__ void tile_bar_init(unsigned long long* bar) {
    if (threadIdx.x != 0) return;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void tile_bulk_issue(double4 (*rot)[64], const double4* __restrict__ src,
                                                unsigned long long* bar) {
    if (threadIdx.x != 0) return;
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the previous tile's reads are done (barrier)
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(kDB * 64) : "memory");
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const unsigned d = (unsigned)__cvta_generic_to_shared(&rot[k >> 1][(k & 1) * 32]);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 1024, [%2];"
                     ::"r"(d), "l"(src + 32 * (k >> 1)), "r"(b) : "memory");
    }
}

__device__ __forceinline__ void tile_wait(unsigned long long* bar, unsigned parity) {
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    unsigned done = 0;
    while (!done)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done) : "r"(b), "r"(parity) : "memory");
}

__device__ __forceinline__ void add_to(double4* dst, const Acc& a) {
    double4 v = *dst;
    v.x += a.qx; v.y += a.qy; v.z += a.px; v.w += a.py;
    *dst = v;
}

#ifdef GS_SYM_MAXREG  // A/B on C2 (ms per RHS): 160 regs (6 CTAs/SM) 0.366, 152 -> 0.378, 144 (7 CTAs/SM) -> 0.381, 136 -> 0.397
#define GS_SYM_BOUNDS __maxnreg__(GS_SYM_MAXREG)
#else
#define GS_SYM_BOUNDS __launch_bounds__(kST, GS_SYM_MINB)
#endif

template <int FAM>
__global__ void GS_SYM_BOUNDS k_dense_sym(const double4* __restrict__ S, int64_t n, int nb, int G,
                                                       int nsb, long long cta0, double k1, double4* __restrict__ part,
                                                       int64_t pstride, DevStatus* st, unsigned long long event,
                                                       const double* __restrict__ tbl_g, PeerWait wait) {
    __shared__ __align__(128) double s_tbl[kTblWords];
    __shared__ __align__(128) double4 s_rot[4][64];  // sub-block b of J twice: s_rot[b][k] = record 32 b + (k & 31)
    __shared__ unsigned long long s_tbar, s_rbar;
    extern __shared__ double4 s_acc[];   // G * kDB records
    table_bulk_issue(s_tbl, tbl_g, &s_tbar);  // lands while the CTA sets up its first tile
    tile_bar_init(&s_rbar);
    // an earlier failure: skip (one decision per CTA, the status may change while CTAs start)
    if (__syncthreads_or(*((volatile unsigned long long*)&st->first_event) < event)) {
        table_bulk_wait(&s_tbar);  // no copy in flight into a retiring CTA
        return;
    }
    block_wait(wait);  // multi-GPU peer exchange: every rank's records of the previous stage are in S
    const double* tbl = lane_table(s_tbl);
    const unsigned tb = lane_table_addr(s_tbl);
    const int caphi = pair_clamp_hi(FAM, k1);

    // CTA -> superblock pair (SI, SJ), SI <= SJ, row-major over the upper triangle
    const long long t = cta0 + blockIdx.x;
    const double b2 = 2.0 * nsb + 1.0;
    long long SI = (long long)floor((b2 - sqrt(b2 * b2 - 8.0 * (double)t)) * 0.5);
    auto row_start = [nsb](long long r) { return r * nsb - r * (r - 1) / 2; };
    while (SI > 0 && row_start(SI) > t) --SI;
    while (row_start(SI + 1) <= t) ++SI;
    const long long SJ = SI + (t - row_start(SI));
    const bool diag = SI == SJ;
    GS_ASSERT(SI >= 0 && SI <= SJ && SJ < nsb);

    // the first tile (SJ G, full) goes in flight now
    const long long J0 = SJ * G;
    const bool pre = (J0 + 1) * kDB <= n;
    if (pre) tile_bulk_issue(s_rot, S + J0 * kDB, &s_rbar);
    unsigned rph = 0;
    bool first = true;

    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int r0 = w * 64 + lane, r1 = r0 + 32;  // this thread's two rows inside a block
    const double4 zero4 = make_double4(0.0, 0.0, 0.0, 0.0);
    for (int k = threadIdx.x; k < G * kDB; k += kST) s_acc[k] = zero4;
    table_bulk_wait(&s_tbar);

#ifdef GS_SYM_EMPTY  // A/B probe: prologue + partial writes only (the per-CTA fixed cost)
    if (pre) tile_wait(&s_rbar, 0);  // no copy in flight into a retiring CTA
    for (int ib = 0; ib < 0; ++ib) {
#else
    for (int ib = 0; ib < G; ++ib) {
#endif
        const long long I = SI * G + ib;
        if (I >= nb) break;
        const int64_t i0 = I * kDB + r0, i1 = I * kDB + r1;
        const double4 me0 = (i0 < n) ? S[i0] : far_record(r0);
        const double4 me1 = (i1 < n) ? S[i1] : far_record(r1);
        Acc a0{0.0, 0.0, 0.0, 0.0}, a1{0.0, 0.0, 0.0, 0.0};
        for (int jb = diag ? ib : 0; jb < G; ++jb) {
            const long long J = SJ * G + jb;
            if (J >= nb) break;
            __syncthreads();  // previous tile done with s_rot / s_acc
            const bool full = (J + 1) * kDB <= n;
            if (full) {
                if (!(first && pre)) tile_bulk_issue(s_rot, S + J * kDB, &s_rbar);
                tile_wait(&s_rbar, rph);
                rph ^= 1u;
            } else {
                for (int r = threadIdx.x; r < kDB; r += kST) {
                    const int64_t js = J * kDB + r;
                    const double4 rec = (js < n) ? S[js] : far_record(kDB + r);
                    s_rot[r >> 5][r & 31] = rec;
                    s_rot[r >> 5][(r & 31) + 32] = rec;
                }
                __syncthreads();
            }
            first = false;
            int nz0 = 0, nz1 = 0;
            if (I == J) {
#pragma unroll 4
                for (int jj = 0; jj < kDB; ++jj) {
                    const double4 s = s_rot[jj >> 5][jj & 31];
                    one_sided<FAM>(me0, s, tbl, k1, a0, nz0);
                    one_sided<FAM>(me1, s, tbl, k1, a1, nz1);
                }
                if (nz0 > 1 && i0 < n) record_coincident(S, n, i0, me0, J * kDB, J * kDB + kDB, st, event);
                if (nz1 > 1 && i1 < n) record_coincident(S, n, i1, me1, J * kDB, J * kDB + kDB, st, event);
                continue;
            }
#if GS_SYM_ZMIN
            nz0 = nz1 = 0x7fffffff;
#endif
            double4* jacc = s_acc + jb * kDB;
            for (int ph = 0; ph < 4; ++ph) {
                const int b = (2 * w + ph) & 3;
                const double4* rot = &s_rot[b][lane];
                Acc j{0.0, 0.0, 0.0, 0.0};
#if GS_SYM_SRC2
                // two sources per step (4 independent pair chains per lane): jA travels with
                // source (lane + step), jB with source (lane + step + 1); both move 2 lanes
                Acc jb2{0.0, 0.0, 0.0, 0.0};
#pragma unroll kSymUnroll
                for (int step = 0; step < 32; step += 2) {
                    const double4 sa = rot[step];
                    const double4 sb = rot[step + 1];
                    two_sided<FAM>(me0, sa, tbl, tb, k1, caphi, a0, j, nz0);
                    two_sided<FAM>(me1, sa, tbl, tb, k1, caphi, a1, j, nz1);
                    two_sided<FAM>(me0, sb, tbl, tb, k1, caphi, a0, jb2, nz0);
                    two_sided<FAM>(me1, sb, tbl, tb, k1, caphi, a1, jb2, nz1);
                    const int src = (lane + 2) & 31;
                    j.qx = __shfl_sync(kFull, j.qx, src);
                    j.qy = __shfl_sync(kFull, j.qy, src);
                    j.px = __shfl_sync(kFull, j.px, src);
                    j.py = __shfl_sync(kFull, j.py, src);
                    jb2.qx = __shfl_sync(kFull, jb2.qx, src);
                    jb2.qy = __shfl_sync(kFull, jb2.qy, src);
                    jb2.px = __shfl_sync(kFull, jb2.px, src);
                    jb2.py = __shfl_sync(kFull, jb2.py, src);
                }
                {   // jB of lane l belongs to source l + 1: hand it to lane l + 1
                    const int src = (lane + 31) & 31;
                    j.qx += __shfl_sync(kFull, jb2.qx, src);
                    j.qy += __shfl_sync(kFull, jb2.qy, src);
                    j.px += __shfl_sync(kFull, jb2.px, src);
                    j.py += __shfl_sync(kFull, jb2.py, src);
                }
#else
#pragma unroll 4
                for (int step = 0; step < 32; ++step) {
                    const double4 s = rot[step];
                    two_sided<FAM>(me0, s, tbl, tb, k1, caphi, a0, j, nz0);
                    two_sided<FAM>(me1, s, tbl, tb, k1, caphi, a1, j, nz1);
                    const int src = (lane + 1) & 31;
                    j.qx = __shfl_sync(kFull, j.qx, src);
                    j.qy = __shfl_sync(kFull, j.qy, src);
                    j.px = __shfl_sync(kFull, j.px, src);
                    j.py = __shfl_sync(kFull, j.py, src);
                }
#endif
                add_to(&jacc[b * 32 + lane], j);
                __syncthreads();
            }
#if GS_SYM_ZMIN
            constexpr int kTinyHi = 0x16687e92;  // high word of kTinyR2 = 1e-200
            nz0 = nz0 <= kTinyHi;
            nz1 = nz1 <= kTinyHi;
#endif
            if (nz0 > 0 && i0 < n) record_coincident(S, n, i0, me0, J * kDB, J * kDB + kDB, st, event);  // rare
            if (nz1 > 0 && i1 < n) record_coincident(S, n, i1, me1, J * kDB, J * kDB + kDB, st, event);
        }
        if (diag) {
            // rows of block ib: their J-side contributions (tiles (I' < I, I)) are already in
            // s_acc[ib]; later tiles of this CTA never touch s_acc[ib] again
            __syncthreads();
            add_to(&s_acc[ib * kDB + r0], a0);
            add_to(&s_acc[ib * kDB + r1], a1);
        } else {
            GS_ASSERT(I * kDB + kDB <= pstride);
            if (i0 < n) part[SJ * pstride + i0] = make_double4(a0.qx, a0.qy, a0.px, a0.py);
            if (i1 < n) part[SJ * pstride + i1] = make_double4(a1.qx, a1.qy, a1.px, a1.py);
        }
    }
    __syncthreads();
    for (int jb = 0; jb < G; ++jb) {
        const long long J = SJ * G + jb;
        if (J >= nb) break;
        for (int r = threadIdx.x; r < kDB; r += kST) {
            const int64_t js = J * kDB + r;
            if (js < n) part[SI * pstride + js] = s_acc[jb * kDB + r];
        }
    }
}

}  // namespace

SymPlan sym_plan(int64_t n) {
    SymPlan p;
    p.nb = (int)((n + kDB - 1) / kDB);
    p.G = 1;
    while ((p.nb + p.G - 1) / p.G > GS_SYM_SB && p.G < kSymMaxG) p.G *= 2;
    p.nsb = (p.nb + p.G - 1) / p.G;
    p.pstride = (int64_t)p.nb * kDB;
    p.ok = p.nsb <= 256;
    return p;
}

void sym_pair_of(long long t, int nsb, long long* SI, long long* SJ) {
    auto row_start = [nsb](long long r) { return r * nsb - r * (r - 1) / 2; };
    long long lo = 0, hi = nsb - 1;  // largest r with row_start(r) <= t
    while (lo < hi) {
        const long long mid = (lo + hi + 1) / 2;
        if (row_start(mid) <= t) lo = mid;
        else hi = mid - 1;
    }
    *SI = lo;
    *SJ = lo + (t - row_start(lo));
}

long long sym_ctas(int64_t n) {
    const SymPlan p = sym_plan(n);
    return (long long)p.nsb * (p.nsb + 1) / 2;
}

void launch_dense_sym(const SysConst& sc, const double4* S, int64_t n, double4* part, int64_t pstride, DevStatus* st,
                      unsigned long long event, const double* tbl_dev, cudaStream_t stream, long long cta0,
                      long long cta1, PeerWait wait) {
    const SymPlan p = sym_plan(n);
    if (cta1 < 0) cta1 = sym_ctas(n);
    if (cta1 <= cta0) return;
    const unsigned ctas = (unsigned)(cta1 - cta0);
    const size_t smem = (size_t)p.G * kDB * sizeof(double4);
    {   // static (table, s_rot, barriers) + dynamic (G blocks of J-side sums) exceeds the 48 KB default
        // at G = 8: opt in to more dynamic shared memory, once per device (the attribute is per device)
        static std::atomic<signed char> done[64];
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev >= 0 && dev < 64 && done[dev].load() == 0) {
            const int max_dyn = kSymMaxG * kDB * (int)sizeof(double4);
            const bool ok = cudaFuncSetAttribute(k_dense_sym<kFamConical>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 max_dyn) == cudaSuccess &&
                            cudaFuncSetAttribute(k_dense_sym<kFamGaussian>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 max_dyn) == cudaSuccess;
            done[dev] = ok ? 1 : -1;
        }
    }
    if (sc.fam == kFamConical)
        k_dense_sym<kFamConical><<<ctas, kST, smem, stream>>>(S, n, p.nb, p.G, p.nsb, cta0, sc.k1, part, pstride, st,
                                                              event, tbl_dev, wait);
    else
        k_dense_sym<kFamGaussian><<<ctas, kST, smem, stream>>>(S, n, p.nb, p.G, p.nsb, cta0, sc.k1, part, pstride,
                                                               st, event, tbl_dev, wait);
}

}  // namespace gsb

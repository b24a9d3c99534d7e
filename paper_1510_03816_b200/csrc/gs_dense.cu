// gs_dense.cu — all-pairs (dense) fp64 RHS of the Euler–Poincaré N-particle system.
//
// Replaces particles._interaction_terms + rhs (particles.py:79-117) and the N x N
// temporaries of kernels.pairwise_distances / kernel_value / kernel_derivative
// (kernels.py:121-178): nothing of size N^2 is ever materialised.
//
// Grid: (row blocks of kDB targets) x (source chunks).  Each thread owns one target row,
// keeps its (x, y, px, py) and four fp64 accumulators in registers, and sweeps its
// chunk's sources through a shared-memory tile (kDT records of 32 B, read as warp-wide
// broadcasts).  The chunk split gives the GPU enough CTAs at small N (N = 16384 has only
// 128 row blocks) and is fixed by n alone, so a row's summation order — and its bits —
// do not depend on how rows are sharded across GPUs.  Chunk partials are summed in chunk
// order by the finish kernel, which also applies the kernel scale factors, the sigma2
// term and the fused RK4 stage epilogue (integrator.py:98-114).
//
// Bound: FP64 pipe.  ~27 DP-pipe slots per ordered pair (2 DADD diff, 2 r^2, 5 rsqrt
// refinement, 2 r*k1, 8 exp, 2 p.p, 4 accumulate, 2 coefficient) against the
// libm formulation's 45.
#include <algorithm>

#include "gs_kernels.cuh"

namespace gsb {

DensePlan dense_plan(int64_t n, int sm_count) {
    // Source chunks of a multiple of kCG sources, enough of them for ~32 CTAs per SM: at mid N
    // (a few thousand particles) whole kDT tiles would leave a handful of CTAs with long serial
    // source loops (N = 600: 15 CTAs, 59 us per RHS).  Depends on n and the SM count only, so a
    // row's summation order does not depend on the row split.
    constexpr int64_t kCG = 32;
    const int64_t row_blocks = (n + kDB - 1) / kDB;
    const int64_t units = (n + kCG - 1) / kCG;
    const int64_t want_ctas = (int64_t)sm_count * 32;
    int64_t nc = (want_ctas + row_blocks - 1) / row_blocks;
    nc = std::max<int64_t>(1, std::min(nc, units));
    DensePlan p;
    p.chunk = ((units + nc - 1) / nc) * kCG;
    p.nchunks = (int)((n + p.chunk - 1) / p.chunk);
    return p;
}

// Two target rows per thread (64 threads x 2 = the kDB rows of a CTA): every shared-memory
// source broadcast and the loop overhead serve two pair evaluations.
constexpr int kDPT = kDB / 2;

struct Row {
    double qx, qy, px, py;
    int nz;
};

template <int FAM>
__device__ __forceinline__ void row_pair(const double4& me, const double4& s, const double* tbl, double k1, Row& a) {
    const double dx = me.x - s.x, dy = me.y - s.y;
    const double pdot = fma(me.z, s.z, me.w * s.w);
    double g, c;
    int z;
    pair_core<FAM>(dx, dy, pdot, tbl, k1, g, c, z);
    a.qx = fma(g, s.z, a.qx);
    a.qy = fma(g, s.w, a.qy);
    a.px = fma(c, dx, a.px);
    a.py = fma(c, dy, a.py);
    a.nz += z;
}

template <int FAM>
__global__ void __launch_bounds__(kDPT, 12) k_dense_partial(const double4* __restrict__ S, int64_t n, int64_t row0,
                                                            int64_t nrows, int64_t chunk, double k1,
                                                            double4* __restrict__ part, DevStatus* st,
                                                            unsigned long long event, const double* __restrict__ tbl_g) {
    __shared__ __align__(128) double s_tbl[kTblWords];
    __shared__ double4 s_src[kDT];
    __shared__ unsigned long long s_tbar;
    table_bulk_issue(s_tbl, tbl_g, &s_tbar);
    // an earlier failure: skip (one decision per CTA, the status may change while CTAs start)
    if (__syncthreads_or(*((volatile unsigned long long*)&st->first_event) < event)) {
        table_bulk_wait(&s_tbar);
        return;
    }
    table_bulk_wait(&s_tbar);
    const double* tbl = lane_table(s_tbl);

    const int64_t li0 = (int64_t)blockIdx.x * kDB + threadIdx.x, li1 = li0 + kDPT;
    const bool v0 = li0 < nrows, v1 = li1 < nrows;
    const int64_t i0 = row0 + li0, i1 = row0 + li1;
    const double4 me0 = v0 ? S[i0] : far_record(threadIdx.x);
    const double4 me1 = v1 ? S[i1] : far_record(threadIdx.x + kDPT);
    const int64_t j0 = (int64_t)blockIdx.y * chunk;
    const int64_t j1 = min(n, j0 + chunk);

    Row a0{0.0, 0.0, 0.0, 0.0, 0}, a1{0.0, 0.0, 0.0, 0.0, 0};
    for (int64_t t0 = j0; t0 < j1; t0 += kDT) {
        const int m = (int)((j1 - t0) < kDT ? (j1 - t0) : kDT);
        const int mr = (m + 3) & ~3;
        __syncthreads();
        for (int t = threadIdx.x; t < mr; t += kDPT) {
            const int64_t j = t0 + t;
            s_src[t] = (j < j1) ? S[j] : far_record(kDB + t);  // far, p = 0: contributes exactly 0
        }
        __syncthreads();
#pragma unroll 4
        for (int jj = 0; jj < mr; ++jj) {
            const double4 s = s_src[jj];
            row_pair<FAM>(me0, s, tbl, k1, a0);
            row_pair<FAM>(me1, s, tbl, k1, a1);
        }
    }
    // rare: a flagged pair other than the row itself (coincident particles)
    if (v0 && a0.nz > ((i0 >= j0 && i0 < j1) ? 1 : 0)) record_coincident(S, n, i0, me0, j0, j1, st, event);
    if (v1 && a1.nz > ((i1 >= j0 && i1 < j1) ? 1 : 0)) record_coincident(S, n, i1, me1, j0, j1, st, event);
    if (v0) part[(int64_t)blockIdx.y * nrows + li0] = make_double4(a0.qx, a0.qy, a0.px, a0.py);
    if (v1) part[(int64_t)blockIdx.y * nrows + li1] = make_double4(a1.qx, a1.qy, a1.px, a1.py);
}

void launch_dense_partial(const SysConst& sc, const double4* S, int64_t n, int64_t row0, int64_t nrows,
                          const DensePlan& plan, double4* part, DevStatus* st, unsigned long long event,
                          const double* tbl_dev, cudaStream_t stream) {
    if (nrows <= 0) return;
    dim3 grid((unsigned)((nrows + kDB - 1) / kDB), (unsigned)plan.nchunks);
    if (sc.fam == kFamConical)
        k_dense_partial<kFamConical><<<grid, kDPT, 0, stream>>>(S, n, row0, nrows, plan.chunk, sc.k1, part, st,
                                                                 event, tbl_dev);
    else
        k_dense_partial<kFamGaussian><<<grid, kDPT, 0, stream>>>(S, n, row0, nrows, plan.chunk, sc.k1, part, st,
                                                                  event, tbl_dev);
}

// ---------------------------------------------------------------------------------------
// Gram matrix K[i][j] = G(|q_i - q_j|) (kernels.gram_matrix, kernels.py:181-197) for the
// velocity-space feedback update (shooting.py:138-175): row-major n x n, and the row-major
// first coincident pair (i != j, d == 0) recorded in *bad as i*n + j.
template <int FAM>
__global__ void k_gram(const double* __restrict__ q, int64_t n, double k1, double scale, double* K,
                       unsigned long long* bad, const double* __restrict__ tbl_g) {
    __shared__ double s_tbl[kTblWords];
    for (int t = threadIdx.y * blockDim.x + threadIdx.x; t < kTblWords; t += blockDim.x * blockDim.y)
        s_tbl[t] = tbl_g[t];
    __syncthreads();
    const double* tbl = s_tbl + ((threadIdx.y * blockDim.x + threadIdx.x) & (kTblRep - 1));
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t i = (int64_t)blockIdx.y * blockDim.y + threadIdx.y;
    if (i >= n || j >= n) return;
    const double dx = q[2 * i] - q[2 * j], dy = q[2 * i + 1] - q[2 * j + 1];
    const double r2 = fma(dx, dx, fma(dy, dy, kTinyR2));
    double g;
    if (FAM == kFamConical) g = exp2_tbl(r2 * rsqrt_refined(r2), k1, tbl);
    else g = exp2_tbl(r2, k1, tbl);
    K[i * n + j] = g * scale;
    if (i != j && __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)) == 0.0)
        atomicMin(bad, (unsigned long long)(i * n + j));
}

void launch_gram(const SysConst& sc, const double* q, int64_t n, double* K, unsigned long long* bad,
                 const double* tbl_dev, cudaStream_t stream) {
    dim3 block(32, 8), grid((unsigned)((n + 31) / 32), (unsigned)((n + 7) / 8));
    if (sc.fam == kFamConical) k_gram<kFamConical><<<grid, block, 0, stream>>>(q, n, sc.k1, sc.scale_q, K, bad, tbl_dev);
    else k_gram<kFamGaussian><<<grid, block, 0, stream>>>(q, n, sc.k1, sc.scale_q, K, bad, tbl_dev);
}

// ---------------------------------------------------------------------------------------
// Velocity field u(x_k) = sum_j G(|x_k - q_j|) p_j at m sample points (particles.py:140-150):
// the dq half of the pair sum with targets outside the particle set.  Same tiling as
// k_dense_partial (two sample points per thread, sources through shared memory, source
// chunks for parallelism at small m); partials per chunk are summed in chunk order.
template <int FAM>
__global__ void __launch_bounds__(kDPT, 12) k_velocity_partial(const double4* __restrict__ S, int64_t n,
                                                               const double* __restrict__ x, int64_t m,
                                                               int64_t chunk, double k1, double2* __restrict__ part,
                                                               const double* __restrict__ tbl_g) {
    __shared__ double s_tbl[kTblWords];
    __shared__ double4 s_src[kDT];
    for (int t = threadIdx.x; t < kTblWords; t += kDPT) s_tbl[t] = tbl_g[t];
    const double* tbl = lane_table(s_tbl);
    const int64_t k0 = (int64_t)blockIdx.x * kDB + threadIdx.x, k1i = k0 + kDPT;
    const bool v0 = k0 < m, v1 = k1i < m;
    const double x0 = v0 ? x[2 * k0] : 1e150 * (threadIdx.x + 1), y0 = v0 ? x[2 * k0 + 1] : 1e150;
    const double x1 = v1 ? x[2 * k1i] : 1e150 * (threadIdx.x + 1), y1 = v1 ? x[2 * k1i + 1] : -1e150;
    const int64_t j0 = (int64_t)blockIdx.y * chunk;
    const int64_t j1 = min(n, j0 + chunk);
    double ux0 = 0.0, uy0 = 0.0, ux1 = 0.0, uy1 = 0.0;
    for (int64_t t0 = j0; t0 < j1; t0 += kDT) {
        __syncthreads();
        for (int t = threadIdx.x; t < kDT; t += kDPT) {
            const int64_t j = t0 + t;
            s_src[t] = (j < j1) ? S[j] : far_record(kDB + t);
        }
        __syncthreads();
        const int mm = (int)((j1 - t0) < kDT ? (j1 - t0) : kDT);
        const int mr = (mm + 3) & ~3;
#pragma unroll 4
        for (int jj = 0; jj < mr; ++jj) {
            const double4 s = s_src[jj];
            double g0, g1, c;
            int z;
            pair_core<FAM>(x0 - s.x, y0 - s.y, 0.0, tbl, k1, g0, c, z);
            pair_core<FAM>(x1 - s.x, y1 - s.y, 0.0, tbl, k1, g1, c, z);
            ux0 = fma(g0, s.z, ux0); uy0 = fma(g0, s.w, uy0);
            ux1 = fma(g1, s.z, ux1); uy1 = fma(g1, s.w, uy1);
        }
    }
    if (v0) part[(int64_t)blockIdx.y * m + k0] = make_double2(ux0, uy0);
    if (v1) part[(int64_t)blockIdx.y * m + k1i] = make_double2(ux1, uy1);
}

__global__ void k_velocity_finish(const double2* __restrict__ part, int nchunks, int64_t m, double scale, double* u) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= m) return;
    double sx = 0.0, sy = 0.0;
    for (int c = 0; c < nchunks; ++c) {
        const double2 v = part[(int64_t)c * m + k];
        sx += v.x; sy += v.y;
    }
    u[2 * k] = sx * scale;
    u[2 * k + 1] = sy * scale;
}

DensePlan velocity_plan(int64_t n, int64_t m, int sm_count) {
    const int64_t row_blocks = (m + kDB - 1) / kDB;
    const int64_t tiles = (n + kDT - 1) / kDT;
    int64_t nc = ((int64_t)sm_count * 32 + row_blocks - 1) / row_blocks;
    nc = std::max<int64_t>(1, std::min(nc, tiles));
    DensePlan p;
    p.chunk = ((tiles + nc - 1) / nc) * kDT;
    p.nchunks = (int)((n + p.chunk - 1) / p.chunk);
    return p;
}

void launch_velocity_field(const SysConst& sc, const double4* S, int64_t n, const double* x, int64_t m,
                           const DensePlan& plan, double2* part, double* u, const double* tbl_dev,
                           cudaStream_t stream) {
    if (m <= 0) return;
    dim3 grid((unsigned)((m + kDB - 1) / kDB), (unsigned)plan.nchunks);
    if (sc.fam == kFamConical)
        k_velocity_partial<kFamConical><<<grid, kDPT, 0, stream>>>(S, n, x, m, plan.chunk, sc.k1, part, tbl_dev);
    else
        k_velocity_partial<kFamGaussian><<<grid, kDPT, 0, stream>>>(S, n, x, m, plan.chunk, sc.k1, part, tbl_dev);
    k_velocity_finish<<<(unsigned)((m + 255) / 256), 256, 0, stream>>>(part, plan.nchunks, m, sc.scale_q, u);
}

// ---------------------------------------------------------------------------------------
// Finish: chunk reduction (fixed order) + scale + sigma2 + mode-specific epilogue.
// (the RK4 stage epilogue itself, stage_update, is in gs_kernels.cuh)
// Partial sums are reduced by kFinGroups warps per 32 rows: warp w sums slots w, w + 8, ...
// (coalesced over the rows), warp 0 adds the group sums in group order — a fixed order, and
// 8x the parallelism of one thread per row walking all slots (the symmetric kernel leaves
// nsb = 128 slots per row at C2: 67 MB per stage).
constexpr int kFinRows = 32;
constexpr int kFinGroups = 8;

inline int finish_threads(int nchunks) {
    const int g = nchunks < 1 ? 1 : (nchunks < kFinGroups ? nchunks : kFinGroups);
    return g * kFinRows;
}

__device__ __forceinline__ bool finish_reduce(const FinishArgs& a, int64_t& li, double4& sum) {
    __shared__ double4 s_part[kFinGroups][kFinRows];
    const int r = threadIdx.x & (kFinRows - 1), w = threadIdx.x / kFinRows;
    const int groups = blockDim.x / kFinRows;  // <= kFinGroups, no more than the slots
    li = (int64_t)blockIdx.x * kFinRows + r;
    const bool valid = li < a.nrows;
    const int64_t ps = a.pstride ? a.pstride : a.nrows;
    double4 acc = make_double4(0.0, 0.0, 0.0, 0.0);
    GS_ASSERT(a.nchunks >= 1 && (a.pstride == 0 || a.pstride >= a.nrows));
    if (valid)
        for (int c = w; c < a.nchunks; c += groups) {
            const double4 v = a.part[(int64_t)c * ps + li];
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
    s_part[w][r] = acc;
    __syncthreads();
    if (w != 0 || !valid) return false;
    const int ng = a.nchunks < groups ? a.nchunks : groups;
    sum = s_part[0][r];
    for (int g = 1; g < ng; ++g) {
        const double4 v = s_part[g][r];
        sum.x += v.x; sum.y += v.y; sum.z += v.z; sum.w += v.w;
    }
    return true;
}

template <int MODE>
__global__ void __launch_bounds__(kFinRows * kFinGroups) k_finish(SysConst sc, FinishArgs a) {
    int64_t li;
    double4 sum;
    if (!finish_reduce(a, li, sum)) return;
    if (*((volatile unsigned long long*)&a.st->first_event) < a.event) return;  // an earlier failure
    const int64_t i = a.row0 + li;
    const double sqx = sum.x, sqy = sum.y, spx = sum.z, spy = sum.w;
    const double4 me = a.S[i];
    // particles.py:113-116: dq = K p (+ sigma2 p), dp = -(sum_j a_ij (q_i - q_j))
    double dqx = sqx * sc.scale_q, dqy = sqy * sc.scale_q;
    if (sc.sigma2 != 0.0) {
        dqx = __dadd_rn(dqx, __dmul_rn(sc.sigma2, me.z));
        dqy = __dadd_rn(dqy, __dmul_rn(sc.sigma2, me.w));
    }
    const double dpx = spx * sc.scale_p, dpy = spy * sc.scale_p;
    if (MODE == kFinRhs) {
        a.dq[2 * li] = dqx; a.dq[2 * li + 1] = dqy;
        a.dp[2 * li] = dpx; a.dp[2 * li + 1] = dpy;
        return;
    }
    if (MODE == kFinHam) {
        a.ham[li] = __dadd_rn(__dmul_rn(me.z, sqx * sc.scale_q), __dmul_rn(me.w, sqy * sc.scale_q));
        return;
    }
    const double4 nxt = stage_update(a, li, dqx, dqy, dpx, dpy);
    a.S[i] = nxt;
    if (!finite4(nxt.x, nxt.y, nxt.z, nxt.w)) record_event(a.st, a.event, kNoEvent);
}

// One raw-sum record per row (the lists' sweep): one thread per row in 256-thread CTAs (with the
// 32-row CTAs of finish_reduce a C5 stage ran 32768 CTAs, each bumping the decision counter).
__global__ void __launch_bounds__(256) k_finish_verlet(SysConst sc, FinishArgs a, VerletFuse f) {
    const int64_t li = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double4 sum = make_double4(0.0, 0.0, 0.0, 0.0);
    bool act = li < a.nrows;
    if (act) {
        const double4 v = a.part[li];
        sum = make_double4(0.0 + v.x, 0.0 + v.y, 0.0 + v.z, 0.0 + v.w);  // as finish_reduce (nchunks = 1)
    }
    act = act && !(*((volatile unsigned long long*)&a.st->first_event) < a.event);
    bool need = false;
    if (act) {
        const int64_t i = a.row0 + li;
        const double4 me = a.S[i];
        double dqx = sum.x * sc.scale_q, dqy = sum.y * sc.scale_q;
        if (sc.sigma2 != 0.0) {
            dqx = __dadd_rn(dqx, __dmul_rn(sc.sigma2, me.z));
            dqy = __dadd_rn(dqy, __dmul_rn(sc.sigma2, me.w));
        }
        const double4 nxt = stage_update(a, li, dqx, dqy, sum.z * sc.scale_p, sum.w * sc.scale_p);
        a.S[i] = nxt;
        if (!finite4(nxt.x, nxt.y, nxt.z, nxt.w)) record_event(a.st, a.event, kNoEvent);
        const int64_t k = f.inv ? (int64_t)f.inv[i] : li;  // slab path (gs_slab.cu): rows already in sorted order
        GS_ASSERT(k >= 0 && k < a.nrows);
        if (f.Ss) f.Ss[k] = nxt;
        if (!f.defer) {
            const double2 b = f.Xb[k];
            const double dx = nxt.x - b.x, dy = nxt.y - b.y;
            need = fma(dx, dx, dy * dy) > f.thr2;
        }
    }
    if (f.defer) return;  // the trigger kernel decides
    if (__syncthreads_or(need) && threadIdx.x == 0) atomicOr(&f.flags[0], 1u);
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned prev = atomicAdd(&f.flags[2], 1u);
        if (prev == gridDim.x - 1) {
            const unsigned d = atomicExch(&f.flags[0], 0u);
            f.flags[2] = 0u;
            if (f.use_cond) cudaGraphSetConditional(f.cond, d);
            f.flags[3] = d;
        }
    }
}

void launch_finish_verlet(const SysConst& sc, const FinishArgs& a, const VerletFuse& f, cudaStream_t stream) {
    if (a.nrows <= 0) return;
    // the lists' sweep leaves one partial per row (a.nchunks == 1)
    k_finish_verlet<<<(unsigned)((a.nrows + 255) / 256), 256, 0, stream>>>(sc, a, f);
}

// R[i] = the same fixed-order slot sum k_finish forms (multi-GPU symmetric split: the rank's
// raw row sums before the reduce-scatter), so 1-GPU and N-GPU runs agree bitwise.
__global__ void __launch_bounds__(kFinRows * kFinGroups) k_slot_reduce(FinishArgs a, double4* R) {
    int64_t li;
    double4 sum;
    if (finish_reduce(a, li, sum)) R[li] = sum;
}

// Rank-split variant: rows of superblock X sum only the slots the rank's superblock pairs wrote
// (slots[X * nsb + k], k < counts[X], ascending), in the same grouped order as finish_reduce;
// untouched slots are neither cleared nor read.
__global__ void __launch_bounds__(kFinRows * kFinGroups) k_slot_reduce_list(const double4* __restrict__ part,
                                                                            int64_t pstride, int64_t n,
                                                                            int rows_per_sb, int nsb,
                                                                            const int* __restrict__ slots,
                                                                            const int* __restrict__ counts,
                                                                            double4* R, PeerSignal sig) {
    __shared__ double4 s_part[kFinGroups][kFinRows];
    const int r = threadIdx.x & (kFinRows - 1), w = threadIdx.x / kFinRows;
    const int64_t li = (int64_t)blockIdx.x * kFinRows + r;
    const bool valid = li < n;
    const int X = valid ? (int)(li / rows_per_sb) : 0;
    const int cnt = valid ? counts[X] : 0;
    const int* list = slots + (size_t)X * nsb;
    double4 acc = make_double4(0.0, 0.0, 0.0, 0.0);
    for (int k = w; k < cnt; k += kFinGroups) {
        const double4 v = part[(int64_t)list[k] * pstride + li];
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    s_part[w][r] = acc;
    __syncthreads();
    if (w == 0 && valid) {
        const int ng = cnt < kFinGroups ? cnt : kFinGroups;
        double4 sum = ng > 0 ? s_part[0][r] : make_double4(0.0, 0.0, 0.0, 0.0);
        for (int g = 1; g < ng; ++g) {
            const double4 v = s_part[g][r];
            sum.x += v.x; sum.y += v.y; sum.z += v.z; sum.w += v.w;
        }
        R[li] = sum;
    }
    block_signal_last(sig);
}

void launch_slot_reduce_list(const double4* part, int64_t pstride, int64_t n, int rows_per_sb, int nsb,
                             const int* slots, const int* counts, double4* R, cudaStream_t stream,
                             PeerSignal sig) {
    if (n <= 0) return;
    k_slot_reduce_list<<<(unsigned)((n + kFinRows - 1) / kFinRows), kFinRows * kFinGroups, 0, stream>>>(
        part, pstride, n, rows_per_sb, nsb, slots, counts, R, sig);
}

void launch_slot_reduce(const double4* part, int nslots, int64_t pstride, int64_t n, double4* R, cudaStream_t stream) {
    if (n <= 0) return;
    FinishArgs a{};
    a.part = part; a.nchunks = nslots; a.pstride = pstride; a.nrows = n;
    k_slot_reduce<<<(unsigned)((n + kFinRows - 1) / kFinRows), finish_threads(nslots), 0, stream>>>(a, R);
}

// ---------------------------------------------------------------------------------------
// Fused stage exchange over peer memory (multi-GPU, symmetric split): the RK4 epilogue of this
// rank's rows reads every rank's raw row sums through NVLink (rank order: deterministic) and
// stores each finished 32-byte stage record straight into every rank's copy of S — the
// reduce-scatter and the all-gather of the NCCL path, done by the epilogue itself.
__global__ void __launch_bounds__(256) k_finish_p2p(SysConst sc, FinishArgs a, const double4* const* __restrict__ Rp,
                                                    double4* const* __restrict__ Sp, int world, PeerWait wt,
                                                    PeerSignal sig) {
    block_wait(wt);  // every rank's row sums of this stage are in place
    const int64_t li = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (li < a.nrows && !(*((volatile unsigned long long*)&a.st->first_event) < a.event)) {
        const int64_t i = a.row0 + li;
        double4 sum = Rp[0][i];
        for (int w = 1; w < world; ++w) {
            const double4 v = Rp[w][i];
            sum.x += v.x; sum.y += v.y; sum.z += v.z; sum.w += v.w;
        }
        const double4 me = a.S[i];
        double dqx = sum.x * sc.scale_q, dqy = sum.y * sc.scale_q;
        if (sc.sigma2 != 0.0) {
            dqx = __dadd_rn(dqx, __dmul_rn(sc.sigma2, me.z));
            dqy = __dadd_rn(dqy, __dmul_rn(sc.sigma2, me.w));
        }
        const double dpx = sum.z * sc.scale_p, dpy = sum.w * sc.scale_p;
        const double4 nxt = stage_update(a, li, dqx, dqy, dpx, dpy);
        for (int w = 0; w < world; ++w) Sp[w][i] = nxt;
        if (!finite4(nxt.x, nxt.y, nxt.z, nxt.w)) record_event(a.st, a.event, kNoEvent);
    }
    block_signal_last(sig);  // after the last CTA's stores: "records written" to every rank
}

void launch_finish_p2p(const SysConst& sc, const FinishArgs& a, const double4* const* Rp, double4* const* Sp,
                       int world, PeerWait wait, PeerSignal sig, cudaStream_t stream) {
    const int64_t rows = a.nrows > 0 ? a.nrows : 1;  // one CTA at least: it carries the signal
    k_finish_p2p<<<(unsigned)((rows + 255) / 256), 256, 0, stream>>>(sc, a, Rp, Sp, world, wait, sig);
}

void launch_finish(int mode, const SysConst& sc, const FinishArgs& a, cudaStream_t stream) {
    if (a.nrows <= 0) return;
    const unsigned blocks = (unsigned)((a.nrows + kFinRows - 1) / kFinRows);
    const int threads = finish_threads(a.nchunks);
    if (mode == kFinRhs) k_finish<kFinRhs><<<blocks, threads, 0, stream>>>(sc, a);
    else if (mode == kFinHam) k_finish<kFinHam><<<blocks, threads, 0, stream>>>(sc, a);
    else k_finish<kFinStage><<<blocks, threads, 0, stream>>>(sc, a);
}

}  // namespace gsb

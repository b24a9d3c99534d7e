// gs_cell.cu — cell-list fp64 RHS for the numerically compact kernels (KD-1).
//
// The reference sums all N^2 pairs (particles.py:79-117).  With the conical kernel at
// alpha = sigma / (53 ln 2) every pair beyond the support radius sigma contributes less
// than 2^-53 of a neighbour's term, so the device may sum only pairs with d_ij < cutoff
// (the truncation changes results by ~1e-15 relative).  Per RHS:
//
//   1. bounding box of the stage positions (block partials + one-block finish) and the
//      grid parameters (cell edge >= cutoff; coarsened if the grid would exceed the cap),
//      all on the device — no host round trip;
//   2. cell key per particle, stable LSD radix sort of (key, index) with CUB, cell start
//      offsets (start[c] = first sorted position with key >= c), permuted copy of the
//      32-byte (x, y, px, py) records so that a cell's particles are contiguous;
//   3. the pair kernel: TPL lanes per target in sorted order.  Cells have edge cutoff/2
//      (GridParams::sub), so a target visits 5 stencil rows, each one contiguous sorted range
//      trimmed to the cells its disk reaches (~5 sigma^2 of candidates instead of the 9 sigma^2
//      of a 3x3 stencil of cutoff-sized cells: C5 RHS 2.57 -> 1.98 ms).  Candidates are filtered in fp32 on the FMA pipe
//      (8-byte float positions relative to the grid origin, radius grown by the fp32 error
//      bound so no pair within the cutoff is lost) into a per-lane list in shared memory,
//      then the accepted pairs run the full fp64 pair body of
//      gs_device.cuh — lanes do not idle on rejected candidates.  Each target's sum runs
//      over its candidates in a fixed order (row, then sorted position), so results are
//      deterministic.  Raw sums are written at the target's original index; the shared
//      finish kernel (gs_dense.cu) applies scales, sigma2 and the RK4 stage epilogue.
//
// Bound: FP64 pipe for the pair kernel (~90 DP slots per HBM byte at config 5); the build
// kernels (sort / scan / permute) are HBM/latency bound and are measured separately.
#include <cub/cub.cuh>

#include <algorithm>
#include <atomic>
#include <cstdlib>

#include "gs_cell.cuh"

namespace gsb {

namespace {

constexpr int kBB = 256;        // bbox block
constexpr int kMaxDevices = 64;
constexpr int kCB = 128;        // pair-kernel threads per CTA
#ifndef GS_CELL_CL               // candidate chunk = per-lane list capacity (A/B builds)
#define GS_CELL_CL 32  // A/B at 7 CTAs/SM (C5 / C4 RHS ms): 24 -> 1.95 / 2.79, 32 -> 1.86 / 2.77, 40 -> 1.86 / 2.80, 48 -> 1.96 / 2.95
#endif
constexpr int kCL = GS_CELL_CL;
#ifndef GS_CELL_TPL_MIN         // minimum lanes per target (A/B builds)
#define GS_CELL_TPL_MIN 4  // A/B (C5 / C4 RHS ms): 1 -> 2.61 / 4.48, 2 -> 2.57 / 3.94, 4 -> 2.57 / 3.62, 8 -> 2.64 / 3.48, 16 -> 2.87 / 3.36
#endif
#ifndef GS_CELL_TPL_DEPTH  // lanes per target grow until n * lanes >= SMs * this (A/B builds)
#define GS_CELL_TPL_DEPTH 512  // A/B (bench --path cell, ms per 100-step solve, 1024 -> 512): n = 12000 34.5 -> 30.8, 16384 37.1 -> 33.7 (256: 34.9), 30000 50.3 -> 48.0
#endif
#ifndef GS_CELL_PREFETCH  // software-pipelined record loads in the pair loop (A/B builds)
#define GS_CELL_PREFETCH 0  // A/B (C5 / C4 RHS ms vs 1.855 / 2.76): minb 7 -> 2.00 / 3.01, 6 -> 2.01 / 2.93, 5 -> 2.01 / 2.84 (bitwise equal)
#endif
#ifndef GS_CELL_MINB           // resident CTAs per SM the register allocation is bounded for (A/B builds)
#define GS_CELL_MINB 7  // A/B (C5 / C4 RHS ms), 3x3 stencil: 8 -> 2.79 / 5.40, 6 -> 2.57 / 4.67, 5 -> 2.61 / 4.55, 4 -> 2.62 / 4.49; half-size cells: 8 -> 1.95 / 2.90, 7 -> 1.85 / 2.75, 6 -> 1.91 / 2.76, 5 -> 1.98 / 2.75, 4 -> 1.98 / 2.75
#endif

__global__ void k_bbox_partial(const double4* __restrict__ S, int64_t n, double* red) {
    __shared__ double s[4][kBB];
    double mnx = INFINITY, mny = INFINITY, mxx = -INFINITY, mxy = -INFINITY;
    bool bad = false;
    for (int64_t i = (int64_t)blockIdx.x * kBB + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBB) {
        const double4 v = S[i];
        bad |= !(isfinite(v.x) && isfinite(v.y));
        mnx = fmin(mnx, v.x); mxx = fmax(mxx, v.x);
        mny = fmin(mny, v.y); mxy = fmax(mxy, v.y);
    }
    if (bad) { mnx = NAN; }
    s[0][threadIdx.x] = mnx; s[1][threadIdx.x] = mny; s[2][threadIdx.x] = mxx; s[3][threadIdx.x] = mxy;
    __syncthreads();
    for (int w = kBB / 2; w; w >>= 1) {
        if (threadIdx.x < w) {
            const int o = threadIdx.x + w;
            const bool nan0 = s[0][threadIdx.x] != s[0][threadIdx.x] || s[0][o] != s[0][o];
            s[0][threadIdx.x] = nan0 ? NAN : fmin(s[0][threadIdx.x], s[0][o]);
            s[1][threadIdx.x] = fmin(s[1][threadIdx.x], s[1][o]);
            s[2][threadIdx.x] = fmax(s[2][threadIdx.x], s[2][o]);
            s[3][threadIdx.x] = fmax(s[3][threadIdx.x], s[3][o]);
        }
        __syncthreads();
    }
    if (threadIdx.x < 4) red[4 * blockIdx.x + threadIdx.x] = s[threadIdx.x][0];
}

// Grid of the bounding box [mnx, mxx] x [mny, mxy] (bad: a non-finite position was seen).  One
// function for the whole-cloud build and the slab build (gs_slab.cu), so that every rank of a
// slab decomposition derives bitwise the grid of the one-GPU build from the all-reduced box.
__device__ GridParams grid_params_of(double mnx, double mny, double mxx, double mxy, bool bad, double cutoff,
                                     int64_t cap, int sub_max) {
    GridParams g;
    // fp32 filter radius: positions are stored as float(x - x0); each carries an error of at
    // most 2^-24 * extent, so a pair's distance in fp32 is off by <= 4 * 2^-24 * extent.
    // Pairs admitted only by this margin have G < 2^-53 (they add < 1e-16 relative).
    // Once the margin dwarfs the cutoff (a flung-apart cloud) the fp32 test is useless and is
    // switched off with a NaN radius: the filter `!(r2 >= rc2f)` then admits every candidate.
    const double extent = fmax(fmax(mxx - mnx, mxy - mny), 0.0);
    const double margin = 4.0 * extent * 5.9604644775390625e-08;
    const double rcf = cutoff * (1.0 + 1e-6) + margin + 1e-30;
    g.rc2f = (margin < 64.0 * cutoff && extent < 1e30) ? __double2float_ru(rcf * rcf) : __int_as_float(0x7fc00000);
    g.rc = rcf;
    g.sub = 1;
    if (bad || !isfinite(mnx) || !isfinite(mxx) || !isfinite(mny) || !isfinite(mxy)) {
        // non-finite stage state: one cell (the stage check has already recorded the failure)
        g.x0 = 0.0; g.y0 = 0.0; g.inv_h = 0.0; g.h = 0.0; g.nx = 1; g.ny = 1; g.ncells = 1; g.hashed = 0;
        g.rc2f = __int_as_float(0x7fc00000);  // NaN: accept everything
    } else {
        g.x0 = mnx; g.y0 = mny;
        // finest subdivision whose row-major grid fits the cap (sub = 1: cell edge = cutoff)
        int sub = sub_max;
        for (; sub > 1; --sub) {
            const double h = cutoff / sub;
            const double fx = floor((mxx - mnx) / h) + 1.0, fy = floor((mxy - mny) / h) + 1.0;
            if (fx * fy <= (double)cap && margin < 0.25 * h) break;
        }
        const double h = cutoff / sub;
        const double fx = floor((mxx - mnx) / h) + 1.0, fy = floor((mxy - mny) / h) + 1.0;
        g.h = h; g.inv_h = 1.0 / h;
        if (fx * fy <= (double)cap) {
            g.nx = (int)fx; g.ny = (int)fy; g.ncells = g.nx * g.ny; g.hashed = 0; g.sub = sub;
        } else {
            g.nx = 0; g.ny = 0; g.ncells = (int)cap; g.hashed = 1;
        }
    }
    g.ylo = 0;
    g.yhi = g.ny;
    return g;
}

__global__ void k_grid_params(const double* __restrict__ red, int nb, double cutoff, int64_t cap, int sub_max,
                              GridParams* gp, const double* __restrict__ skin_ctl, double base_cutoff) {
    if (skin_ctl) cutoff = base_cutoff * (1.0 + skin_ctl[0]);  // adaptive list skin (gs_verlet.cu)
    __shared__ double s[4][kBB];
    __shared__ int s_bad;
    if (threadIdx.x == 0) s_bad = 0;
    double mnx = INFINITY, mny = INFINITY, mxx = -INFINITY, mxy = -INFINITY;
    bool badl = false;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) {
        badl |= red[4 * b] != red[4 * b];
        mnx = fmin(mnx, red[4 * b]); mny = fmin(mny, red[4 * b + 1]);
        mxx = fmax(mxx, red[4 * b + 2]); mxy = fmax(mxy, red[4 * b + 3]);
    }
    s[0][threadIdx.x] = mnx; s[1][threadIdx.x] = mny; s[2][threadIdx.x] = mxx; s[3][threadIdx.x] = mxy;
    __syncthreads();
    if (badl) s_bad = 1;
    for (int w = blockDim.x / 2; w; w >>= 1) {
        if (threadIdx.x < w) {
            const int o = threadIdx.x + w;
            s[0][threadIdx.x] = fmin(s[0][threadIdx.x], s[0][o]); s[1][threadIdx.x] = fmin(s[1][threadIdx.x], s[1][o]);
            s[2][threadIdx.x] = fmax(s[2][threadIdx.x], s[2][o]); s[3][threadIdx.x] = fmax(s[3][threadIdx.x], s[3][o]);
        }
        __syncthreads();
    }
    if (threadIdx.x != 0) return;
    *gp = grid_params_of(s[0][0], s[1][0], s[2][0], s[3][0], s_bad != 0, cutoff, cap, sub_max);
}

__device__ __forceinline__ int cell_coord(double v, double v0, double inv_h, int nmax) {
    int c = (int)floor((v - v0) * inv_h);
    return min(max(c, 0), nmax - 1);
}

// Hashed cells are identified by the bits of the double floor((x - x0) / cutoff): exact below
// 2^53 and, beyond, particles within the cutoff of each other still share the value — so no
// clamping can pile far-flung particles into one cell.
__device__ __forceinline__ double cell_coordf(double v, double v0, double inv_h) { return floor((v - v0) * inv_h); }

__device__ __forceinline__ unsigned cell_hash(double cx, double cy, int ncells) {
    // splitmix64 finalizer of each coordinate's bits (the low bits of small integral doubles are all
    // zero: a plain multiply would put most cells into a few buckets)
    const unsigned long long h = mix64((unsigned long long)__double_as_longlong(cx + 0.0)) ^
                                 mix64((unsigned long long)__double_as_longlong(cy + 0.0) ^ 0xC2B2AE3D27D4EB4Full);
    return (unsigned)h & (unsigned)(ncells - 1);
}

__device__ __forceinline__ unsigned cell_key(const GridParams& g, double x, double y) {
    if (g.hashed) return cell_hash(cell_coordf(x, g.x0, g.inv_h), cell_coordf(y, g.y0, g.inv_h), g.ncells);
    const int cx = cell_coord(x, g.x0, g.inv_h, g.nx), cy = cell_coord(y, g.y0, g.inv_h, g.ny);
    const double fx = (x - g.x0) * g.inv_h - (double)cx, fy = (y - g.y0) * g.inv_h - (double)cy;
    return ((unsigned)(cy * g.nx + cx) << GS_CELL_SUBKEY) | cell_subkey(fx, fy);
}

// The candidate ranges of a target at (x, y): 3 contiguous stencil rows of the row-major grid,
// or the (deduplicated) buckets of the 9 stencil cells of the hashed grid.
struct Ranges {
    int a[9], b[9];
    int cnt;
};

__device__ __forceinline__ void stencil_ranges(const GridParams& g, const int* __restrict__ start, double x, double y,
                                               Ranges& r) {
    r.cnt = 0;
    if (!g.hashed && g.sub > 1) {
        // rows cy - sub .. cy + sub, each trimmed to the cells within rc of the target in x.
        // Cell coordinates are monotone in the position, so every particle with |dx| <= xr lies
        // in [cell(x - xr), cell(x + xr)]; rc carries a 1e-6 relative slack over the cutoff (and
        // the fp32 margin), far above the rounding of the slab bounds below.
        const int cy = cell_coord(y, g.y0, g.inv_h, g.ny);
        const double rc2 = g.rc * g.rc;
        for (int yy = max(cy - g.sub, 0); yy <= min(cy + g.sub, g.ny - 1); ++yy) {
            const double lo = fma((double)yy, g.h, g.y0), hi = lo + g.h;
            const double gap = fmax(0.0, fmax(lo - y, y - hi));
            const double xr2 = fma(-gap, gap, rc2);
            if (!(xr2 > 0.0)) continue;
            const double xr = sqrt(xr2);
            const int xa = cell_coord(x - xr, g.x0, g.inv_h, g.nx), xb = cell_coord(x + xr, g.x0, g.inv_h, g.nx);
            r.a[r.cnt] = start[yy * g.nx + xa];
            r.b[r.cnt] = start[yy * g.nx + xb + 1];
            ++r.cnt;
        }
        return;
    }
    if (!g.hashed) {
        const int cx = cell_coord(x, g.x0, g.inv_h, g.nx), cy = cell_coord(y, g.y0, g.inv_h, g.ny);
        const int xa = max(cx - 1, 0), xb = min(cx + 1, g.nx - 1);
        for (int yy = max(cy - 1, 0); yy <= min(cy + 1, g.ny - 1); ++yy) {
            r.a[r.cnt] = start[yy * g.nx + xa];
            r.b[r.cnt] = start[yy * g.nx + xb + 1];
            ++r.cnt;
        }
        return;
    }
    const double cx = cell_coordf(x, g.x0, g.inv_h), cy = cell_coordf(y, g.y0, g.inv_h);
    unsigned seen[9];
    for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
            const unsigned key = cell_hash(cx + dx, cy + dy, g.ncells);
            bool dup = false;
            for (int t = 0; t < r.cnt; ++t) dup |= seen[t] == key;
            if (dup) continue;  // two stencil cells in one bucket: visit it once
            seen[r.cnt] = key;
            r.a[r.cnt] = start[key];
            r.b[r.cnt] = start[key + 1];
            ++r.cnt;
        }
}

__global__ void k_cell_keys(const double4* __restrict__ S, int64_t n, const GridParams* __restrict__ gp,
                            unsigned* keys, unsigned* vals) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const GridParams g = *gp;
    const double4 v = S[i];
    keys[i] = cell_key(g, v.x, v.y);
    vals[i] = (unsigned)i;
}

// Small-n sort (n <= kSortSmallMax): the whole (key, index) sort in ONE CTA (CUB BlockRadixSort,
// stable, blocked arrangement in index order) instead of the four device-wide radix launches
// (histogram, scan, two onesweep passes) that dominate a small cloud's cell build.  Pad slots
// carry the largest key and follow every real element (stability), so positions [0, n) hold
// exactly the device sort's (key, index) order: results are bitwise unchanged.
#ifndef GS_SORT_SMALL_RB          // radix bits per block pass (A/B builds)
#define GS_SORT_SMALL_RB 4
#endif
constexpr int kSortSmallThreads = 1024;
constexpr int kSortSmallItems = 16;
constexpr int64_t kSortSmallMax = (int64_t)kSortSmallThreads * kSortSmallItems;
using SortSmall = cub::BlockRadixSort<unsigned, kSortSmallThreads, kSortSmallItems, unsigned, GS_SORT_SMALL_RB>;

__global__ void __launch_bounds__(kSortSmallThreads, 1) k_sort_small(const unsigned* __restrict__ keys, int n,
                                                                     int end_bit, unsigned* keys_sorted,
                                                                     unsigned* perm) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    auto& tmp = *reinterpret_cast<typename SortSmall::TempStorage*>(smem_raw);
    unsigned k[kSortSmallItems], v[kSortSmallItems];
#pragma unroll
    for (int t = 0; t < kSortSmallItems; ++t) {
        const int i = threadIdx.x * kSortSmallItems + t;
        k[t] = i < n ? keys[i] : 0xffffffffu;
        v[t] = (unsigned)i;
    }
    SortSmall(tmp).SortBlockedToStriped(k, v, 0, end_bit);
#pragma unroll
    for (int t = 0; t < kSortSmallItems; ++t) {
        const int i = t * kSortSmallThreads + threadIdx.x;
        if (i < n) {
            keys_sorted[i] = k[t];
            perm[i] = v[t];
        }
    }
}

// start[c] = first sorted position whose key >= c, for c in [0, ncells]; permuted records
__global__ void k_cell_start_permute(const unsigned* __restrict__ keys_sorted, const unsigned* __restrict__ perm,
                                     const double4* __restrict__ S, int64_t n, const GridParams* __restrict__ gp,
                                     int* start, double4* Ss, float2* Sf) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k > n) return;
    const GridParams g = *gp;
    const int sh = g.hashed ? 0 : GS_CELL_SUBKEY;  // row-major keys: cell index above the sub-cell bits
    const long long prev = (k == 0) ? -1 : (long long)(keys_sorted[k - 1] >> sh);
    const long long cur = (k == n) ? (long long)g.ncells : (long long)(keys_sorted[k] >> sh);
    GS_ASSERT(cur <= (long long)g.ncells);
    for (long long c = prev + 1; c <= cur; ++c) start[c] = (int)k;
    if (k < n) {
        GS_ASSERT(perm[k] < (unsigned)n);
        const double4 v = S[perm[k]];
        Ss[k] = v;
        Sf[k] = make_float2((float)(v.x - g.x0), (float)(v.y - g.y0));
    }
}

// TPL lanes share one target (small N: fills the GPU); each lane takes every TPL-th
// candidate of the stencil rows and the lanes' sums are xor-butterfly reduced, so every
// target's summation order is fixed.
template <int FAM, int TPL>
__global__ void __launch_bounds__(kCB, GS_CELL_MINB) k_cell_pair(const double4* __restrict__ Ss, const float2* __restrict__ Sf,
                                                      const unsigned* __restrict__ perm,
                                                      const int* __restrict__ tlist, int64_t nt,
                                                      const int* __restrict__ start, const GridParams* __restrict__ gp,
                                                      int64_t n, int64_t row0, int64_t row1, double k1,
                                                      double4* __restrict__ part, DevStatus* st,
                                                      unsigned long long event, const double* __restrict__ tbl_g,
                                                      unsigned long long* accepted) {
    __shared__ __align__(128) double s_tbl[kTblWords];
    __shared__ int s_list[kCL][kCB];
    __shared__ unsigned long long s_acc_count, s_tbar;
    table_bulk_issue(s_tbl, tbl_g, &s_tbar);
    // an earlier failure: skip (one decision per CTA, the status may change while CTAs start)
    if (__syncthreads_or(*((volatile unsigned long long*)&st->first_event) < event)) {
        table_bulk_wait(&s_tbar);
        return;
    }
    table_bulk_wait(&s_tbar);
    const double* tbl = lane_table(s_tbl);
    if (threadIdx.x == 0) s_acc_count = 0;
    __syncthreads();

    const int sub = (TPL > 1) ? (int)(threadIdx.x % TPL) : 0;
    // target t of this launch: sorted position t (all rows), or tlist[t] (a rank's rows, in
    // sorted order: the rank's warps only carry its own targets)
    const int64_t t = (int64_t)blockIdx.x * (kCB / TPL) + threadIdx.x / TPL;
    const bool valid = t < nt;
    const int64_t kk = valid ? (tlist ? (int64_t)tlist[t] : t) : 0;
    const int64_t i = (int64_t)perm[kk];
    const bool active = valid && i >= row0 && i < row1;
    const GridParams g = *gp;
    const double4 me = Ss[kk];
    const float2 mef = Sf[kk];
    Ranges rg;
    stencil_ranges(g, start, me.x, me.y, rg);

    double aqx = 0.0, aqy = 0.0, apx = 0.0, apy = 0.0;
    unsigned long long nacc = 0;
    int nz = 0;
    if (active) {
        for (int rr = 0; rr < rg.cnt; ++rr) {
            const int a = rg.a[rr], b = rg.b[rr];
            for (int base = a + sub; base < b; base += TPL * kCL) {
                const int m = min(kCL, (b - base + TPL - 1) / TPL);
                int cnt = 0;
                for (int t = 0; t < m; ++t) {  // fp32 filter (FMA pipe): d < cutoff (+ fp32 margin)
                    const int j = base + TPL * t;
                    const float2 xy = Sf[j];
                    const float dx = mef.x - xy.x, dy = mef.y - xy.y;
                    if (!(fmaf(dx, dx, dy * dy) >= g.rc2f)) s_list[cnt++][threadIdx.x] = j;  // NaN: keep
                }
                nacc += cnt;
#if GS_CELL_PREFETCH
                // the next accepted record is loaded while the current pair is evaluated
                double4 s_nx = cnt > 0 ? Ss[s_list[0][threadIdx.x]] : me;
#endif
                for (int u = 0; u < cnt; ++u) {
#if GS_CELL_PREFETCH
                    const double4 s = s_nx;
                    if (u + 1 < cnt) s_nx = Ss[s_list[u + 1][threadIdx.x]];
#else
                    const int j = s_list[u][threadIdx.x];
                    GS_ASSERT(j >= 0 && j < n);
                    const double4 s = Ss[j];
#endif
                    const double dx = me.x - s.x, dy = me.y - s.y;
                    const double pdot = fma(me.z, s.z, me.w * s.w);
                    double gk, c;
                    int z;
                    pair_core<FAM>(dx, dy, pdot, tbl, k1, gk, c, z);
                    aqx = fma(gk, s.z, aqx);
                    aqy = fma(gk, s.w, aqy);
                    apx = fma(c, dx, apx);
                    apy = fma(c, dy, apy);
                    nz += z;
                }
            }
        }
    }
    for (int off = TPL >> 1; off; off >>= 1) nz += __shfl_xor_sync(0xffffffffu, nz, off);
    for (int off = TPL >> 1; off; off >>= 1) {
        aqx += __shfl_xor_sync(0xffffffffu, aqx, off);
        aqy += __shfl_xor_sync(0xffffffffu, aqy, off);
        apx += __shfl_xor_sync(0xffffffffu, apx, off);
        apy += __shfl_xor_sync(0xffffffffu, apy, off);
    }
    if (active && sub == 0) {
        if (nz > 1) {  // rare: a coincident particle among the candidates
            for (int rr = 0; rr < rg.cnt; ++rr) {
                const int a = rg.a[rr], b = rg.b[rr];
                for (int j = a; j < b; ++j) {
                    const int64_t jo = (int64_t)perm[j];
                    if (jo == i) continue;
                    const double4 s = Ss[j];
                    const double dx = me.x - s.x, dy = me.y - s.y;
                    if (__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)) != 0.0) continue;
                    if (fma(me.z, s.z, me.w * s.w) != 0.0) record_event(st, event, (unsigned long long)(i * n + jo));
                }
            }
        }
        part[i - row0] = make_double4(aqx, aqy, apx, apy);
    }
    if (accepted) {
        // pair count for the throughput metric (accepted pairs incl. self), one atomic per warp
        for (int off = 16; off; off >>= 1) nacc += __shfl_xor_sync(0xffffffffu, nacc, off);
        if ((threadIdx.x & 31) == 0 && nacc) atomicAdd(&s_acc_count, nacc);
        __syncthreads();
        if (threadIdx.x == 0 && s_acc_count) atomicAdd(accepted, s_acc_count);
    }
}

}  // namespace

size_t cell_select_bytes(int64_t n);

size_t cell_cub_bytes(int64_t n) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const unsigned*)nullptr, (unsigned*)nullptr,
                                    (const unsigned*)nullptr, (unsigned*)nullptr, (int)n, 0, 32);
    return std::max(bytes, cell_select_bytes(n));
}

int64_t cell_cap(int64_t n) {
    // >= 16 particles per cell on average (coarser grids only cost candidates): 16-bit keys,
    // i.e. two radix passes, up to n = 2^20
    int64_t cap = 16384;
    while (cap < n / 16) cap <<= 1;
    return cap;
}

namespace {
int cell_sub_max() {
    static const int v = [] {
        const char* e = std::getenv("GS_B200_CELL_SUB");  // A/B: cells per cutoff (1 = classic 3x3 stencil)
        return e ? std::min(std::max(std::atoi(e), 1), kCellSubMax) : 2;
    }();
    return v;
}

// Slab decomposition (gs_slab.cu): the bounding box of a rank's particles as (min x, min y,
// -max x, -max y), so that ONE elementwise MIN all-reduce over the ranks gives the global box.
__global__ void k_bbox4(const double* __restrict__ red, int nb, double* b4) {
    __shared__ double sh[4][kBB];
    __shared__ int s_bad;
    if (threadIdx.x == 0) s_bad = 0;
    __syncthreads();
    double mnx = INFINITY, mny = INFINITY, mxx = -INFINITY, mxy = -INFINITY;
    bool bad = false;
    for (int b = threadIdx.x; b < nb; b += kBB) {
        bad |= red[4 * b] != red[4 * b];
        mnx = fmin(mnx, red[4 * b]); mny = fmin(mny, red[4 * b + 1]);
        mxx = fmax(mxx, red[4 * b + 2]); mxy = fmax(mxy, red[4 * b + 3]);
    }
    if (bad) s_bad = 1;
    sh[0][threadIdx.x] = mnx; sh[1][threadIdx.x] = mny; sh[2][threadIdx.x] = mxx; sh[3][threadIdx.x] = mxy;
    __syncthreads();
    for (int w = kBB / 2; w; w >>= 1) {
        if (threadIdx.x < w) {
            const int o = threadIdx.x + w;
            sh[0][threadIdx.x] = fmin(sh[0][threadIdx.x], sh[0][o]); sh[1][threadIdx.x] = fmin(sh[1][threadIdx.x], sh[1][o]);
            sh[2][threadIdx.x] = fmax(sh[2][threadIdx.x], sh[2][o]); sh[3][threadIdx.x] = fmax(sh[3][threadIdx.x], sh[3][o]);
        }
        __syncthreads();
    }
    if (threadIdx.x != 0) return;
    b4[0] = s_bad ? -INFINITY : sh[0][0];  // a non-finite position poisons the global box (-> one cell)
    b4[1] = sh[1][0]; b4[2] = -sh[2][0]; b4[3] = -sh[3][0];
}

__global__ void k_grid_from_b4(const double* __restrict__ b4, double cutoff, int64_t cap, int sub_max, GridParams* gp) {
    const double mnx = b4[0], mny = b4[1], mxx = -b4[2], mxy = -b4[3];
    const bool empty = mnx > mxx;  // no particles at all
    *gp = grid_params_of(empty ? 0.0 : mnx, empty ? 0.0 : mny, empty ? 0.0 : mxx, empty ? 0.0 : mxy,
                         mnx == -INFINITY, cutoff, cap, sub_max);
}
}  // namespace

void slab_bbox(const double4* S, int64_t n, double* red, double* b4, cudaStream_t stream) {
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(kCellBboxBlocks, (n + kBB - 1) / kBB));
    k_bbox_partial<<<nb, kBB, 0, stream>>>(S, n, red);
    k_bbox4<<<1, kBB, 0, stream>>>(red, nb, b4);
}

void slab_grid(const double* b4, double cutoff, int64_t n_glob, GridParams* gp, cudaStream_t stream) {
    k_grid_from_b4<<<1, 1, 0, stream>>>(b4, cutoff, cell_cap(n_glob), cell_sub_max(), gp);
}

int cell_build(const CellWs& w, const double4* S, int64_t n, double cutoff, cudaStream_t stream,
               const double* skin_ctl, double base_cutoff) {
    const int nb = (int)std::min<int64_t>(kCellBboxBlocks, (n + kBB - 1) / kBB);
    k_bbox_partial<<<nb, kBB, 0, stream>>>(S, n, w.bbox_red);
    const int64_t cap = cell_cap(n);
    k_grid_params<<<1, kBB, 0, stream>>>(w.bbox_red, nb, cutoff, cap, cell_sub_max(), w.gp, skin_ctl, base_cutoff);
    const unsigned blocks = (unsigned)((n + 255) / 256);
    k_cell_keys<<<blocks, 256, 0, stream>>>(S, n, w.gp, w.keys, w.vals);
    int end_bit = 1;
    while ((1ll << end_bit) < cap) ++end_bit;
    end_bit += GS_CELL_SUBKEY;
    static const int64_t small_max = [] {
        const char* e = std::getenv("GS_B200_SORT_SMALL_MAX");  // A/B: 0 = always the device-wide sort
        return e ? std::min<int64_t>(std::atoll(e), kSortSmallMax) : kSortSmallMax;
    }();
    if (n <= small_max) {
        // the attribute is per device: set once for each device this process launches on
        static std::atomic<signed char> attr_state[kMaxDevices];
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 0 || dev >= kMaxDevices) return (int)cudaErrorInvalidDevice;
        if (attr_state[dev].load() == 0)
            attr_state[dev] = cudaFuncSetAttribute(k_sort_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)sizeof(typename SortSmall::TempStorage)) == cudaSuccess ? 1 : -1;
        if (attr_state[dev].load() < 0) return (int)cudaErrorInvalidConfiguration;
        k_sort_small<<<1, kSortSmallThreads, sizeof(typename SortSmall::TempStorage), stream>>>(
            w.keys, (int)n, end_bit, w.keys_sorted, w.perm);
    } else {
        size_t bytes = w.cub_bytes;
        cudaError_t e = cub::DeviceRadixSort::SortPairs(w.cub_temp, bytes, w.keys, w.keys_sorted, w.vals, w.perm,
                                                        (int)n, 0, end_bit, stream);
        if (e != cudaSuccess) return (int)e;
    }
    k_cell_start_permute<<<(unsigned)((n + 1 + 255) / 256), 256, 0, stream>>>(w.keys_sorted, w.perm, S, n, w.gp,
                                                                            w.start, w.Ss, w.Sf);
    return 0;
}

namespace {
// perm[k] in [row0, row1): the sorted positions of a rank's target rows
struct InRows {
    const unsigned* perm;
    int64_t row0, row1;
    __device__ __forceinline__ bool operator()(const int& k) const {
        const int64_t i = (int64_t)perm[k];
        return i >= row0 && i < row1;
    }
};
}  // namespace

size_t cell_select_bytes(int64_t n) {
    size_t bytes = 0;
    cub::DeviceSelect::If(nullptr, bytes, cub::CountingInputIterator<int>(0), (int*)nullptr, (int*)nullptr, (int)n,
                          InRows{nullptr, 0, 0});
    return bytes;
}

void launch_cell_pair(const SysConst& sc, const CellWs& w, int64_t n, int64_t row0, int64_t row1, double4* part,
                      DevStatus* st, unsigned long long event, const double* tbl_dev, unsigned long long* accepted,
                      cudaStream_t stream) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // A row range (multi-GPU rank): compact the rank's targets in sorted order first, so no warp
    // carries other ranks' targets (over all n sorted positions nearly every warp would hold
    // one of this rank's rows at 8 ranks, and a warp costs its slowest target).
    const bool partial = row0 > 0 || row1 < n;
    const int* tlist = nullptr;
    const int64_t nt = partial ? row1 - row0 : n;
    if (partial) {
        size_t bytes = w.cub_bytes;
        cub::DeviceSelect::If(w.cub_temp, bytes, cub::CountingInputIterator<int>(0), w.tlist, w.nsel, (int)n,
                              InRows{w.perm, row0, row1}, stream);
        tlist = w.tlist;
    }
    if (nt <= 0) return;
    // lanes per target: enough threads to cover every SM ~8 warps deep.  Chosen from n, not nt,
    // so a row's lane split and summation order do not depend on the number of ranks.
    int tpl = GS_CELL_TPL_MIN;
    while (tpl < 16 && n * tpl < (int64_t)sms * GS_CELL_TPL_DEPTH) tpl *= 2;
    const unsigned blocks = (unsigned)((nt * tpl + kCB - 1) / kCB);
#define GS_CELL_LAUNCH(F, T)                                                                                   \
    k_cell_pair<F, T><<<blocks, kCB, 0, stream>>>(w.Ss, w.Sf, w.perm, tlist, nt, w.start, w.gp, n, row0,      \
                                                  row1, sc.k1, part, st, event, tbl_dev, accepted)
#define GS_CELL_FAM(F)                                    \
    switch (tpl) {                                        \
        case 1: GS_CELL_LAUNCH(F, 1); break;              \
        case 2: GS_CELL_LAUNCH(F, 2); break;              \
        case 4: GS_CELL_LAUNCH(F, 4); break;              \
        case 8: GS_CELL_LAUNCH(F, 8); break;              \
        default: GS_CELL_LAUNCH(F, 16); break;            \
    }
    if (sc.fam == kFamConical) { GS_CELL_FAM(kFamConical) }
    else { GS_CELL_FAM(kFamGaussian) }
#undef GS_CELL_FAM
#undef GS_CELL_LAUNCH
}

}  // namespace gsb

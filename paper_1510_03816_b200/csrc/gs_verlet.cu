// gs_verlet.cu — cluster Verlet lists for the cell-list fp64 RHS of whole evolves / matches.
//
// The cell-list semantics are unchanged (KD-1): the RHS of row i sums the pairs
// with d_ij < cutoff (particles.py:79-117 restricted to the kernel's numerical support).  What
// changes is how the pairs are found:
//
//   build (only when needed): the cell grid of gs_cell.cu (bbox, keys, sort, start/permute) is
//   built for the list radius rl = cutoff (1 + skin); consecutive sorted particles form clusters
//   of M targets; every cluster gets ONE list of the sorted positions of all sources within rl of
//   any of its members (fp32 filter grown by its error bound, canonical order: stencil row, then
//   sorted position), padded to a multiple of 2 TPL entries with a sentinel far record.
//
//   every RHS: the records of the stage are gathered into sorted order; a particle that moved more
//   than skin * cutoff / 2 since the build triggers a rebuild (a pair now closer than the cutoff
//   was closer than rl at the build: both particles moved less than half the skin); then TPL lanes
//   per cluster walk its list two sources at a time, each source evaluated against all M members
//   with the fp64 pair core of gs_device.cuh (the list's pairs beyond the cutoff add terms below
//   2^-53 of the self term; GS_VERLET_NOMASK=0 masks them to d^2 < cutoff^2 exactly).
//
// Why: the per-RHS cell sweep (gs_cell.cu) spends its issue slots on the fp32 candidate filter and
// idles lanes whose filtered lists are short; here the filter runs once per rebuild, every lane of
// a cluster has the same trip count, each 32-byte source load feeds M bodies (LSU traffic / M) and
// the M x 2 independent pair chains per lane hide the FP64 latency.  The cost is the masked skin
// pairs (~(1 + skin)^2 - 1 of the accepted ones) and the union of the M members' neighbourhoods.
//
// In a CUDA graph the rebuild is a conditional IF node whose condition the gather kernel sets, so
// an RHS that does not need a rebuild runs 3 kernels: gather, pair sweep, stage epilogue.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>

#include "gs_cell.cuh"

namespace gsb {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kVB = 128;     // pair-sweep threads per CTA
constexpr int kVBB = 128;    // list-build threads per CTA
constexpr int kTplB = 32;    // list-build lanes per cluster: one warp (warp-uniform range loop, no divergence)
#ifndef GS_VERLET_MINB       // resident CTAs per SM the pair sweep's registers are bounded for (A/B)
#define GS_VERLET_MINB 3
#endif
#ifndef GS_VERLET_M          // targets per cluster (A/B builds)
#define GS_VERLET_M 2
#endif
#ifndef GS_VERLET_PF         // L2 prefetch distance of the list, in trips (A/B)
#define GS_VERLET_PF 8
#endif
// The sweep sums every pair of the list (d < cutoff (1 + skin) at the last build): the pairs
// beyond the cutoff add terms below 2^-53 of the self term (G(cutoff) = 2^-53, KD-1) — the order of
// the truncation itself — and dropping the per-pair cutoff test saves ~5 % (C5 1.62 -> 1.55 ms per
// RHS, profiles/r02_history.md).  The pair count of the throughput metric (COUNT) still uses d < cutoff.
#ifndef GS_VERLET_NOMASK
#define GS_VERLET_NOMASK 1
#endif
#ifndef GS_VERLET_DEPTH      // lanes per cluster grow until clusters * lanes >= SMs * this (A/B)
#define GS_VERLET_DEPTH 128   // A/B (C2 100-step solve, ms): lanes 4 -> 13.6, 8 -> 14.1, 16 -> 14.3, 2 -> 16.1
#endif
constexpr int kVM = GS_VERLET_M;
#ifndef GS_VERLET_UNIFORM
#define GS_VERLET_UNIFORM 1
#endif
#ifndef GS_VERLET_BALANCE
#define GS_VERLET_BALANCE 1
#endif
#ifndef GS_VERLET_LIST2
#define GS_VERLET_LIST2 1
#endif

struct Acc {
    double qx, qy, px, py;
};

// exp2_tbl with an extra acceptance predicate (the cutoff mask, GS_VERLET_NOMASK=0): G = 0 outside.
__device__ __forceinline__ double exp2_tbl_in(double x, double k, unsigned tb, bool in) {
    const double g = exp2_tbl_fast(x, k, tb);
    return in ? g : 0.0;
}

// One ordered pair (target me <- source s), masked to d^2 < cutoff^2 (rc2b = bits of cutoff^2:
// non-negative doubles order like their bit patterns, so the test is one 64-bit integer compare).
// nz counts pairs whose d^2 has the high word of the 1e-200 offset (d == 0: the self pair and any
// coincident particle; a superset, the rare re-scan decides exactly).
template <int FAM>
__device__ __forceinline__ double vexp(double x, double k, unsigned tb, bool in) {
#if GS_VERLET_NOMASK
    return exp2_tbl_fast(x, k, tb);  // `in` only counts pairs here
#else
    return exp2_tbl_in(x, k, tb, in);
#endif
}

template <int FAM, bool COUNT>
__device__ __forceinline__ void vbody(const double4& me, const double4& s, const double* __restrict__ tbl, unsigned tb,
                                      double k1, int caphi, long long rc2b, Acc& a, int& nz, int& nin) {
    const double dx = me.x - s.x, dy = me.y - s.y;
    const double pdot = fma(me.z, s.z, me.w * s.w);
    double r2 = fma(dx, dx, fma(dy, dy, gs_cb[kCbTinyR2]));
    const long long r2b = __double_as_longlong(r2);
#if GS_VERLET_NOMASK  // A/B: sum every list pair (skin pairs add their sub-2^-53 terms)
    const bool in = COUNT ? r2b < rc2b : true;
#else
    const bool in = r2b < rc2b;
#endif
#if GS_PAIR_CLAMP && GS_VERLET_NOMASK
    // list pairs lie within rl of their target; only the sentinel (far, p = 0) is out of the table
    // exp's range: the clamp of d^2 (pair_clamp_hi) replaces the exp's range select.  The d == 0
    // count reads the clamped high word (the cap lies far above 1e-200), so d^2 is clamped in place.
    const int r2h = min(__double2hiint(r2), caphi);
    r2 = __hiloint2double(r2h, __double2loint(r2));
    nz += r2h == __double2hiint(kTinyR2);
#else
    nz += __double2hiint(r2) == __double2hiint(kTinyR2);
#endif
    if (COUNT) nin += in;
    double g, c;
#if GS_PAIR_CLAMP && GS_VERLET_NOMASK
    if (FAM == kFamConical) {
        const double rs = rsqrt_refined(r2);
        g = exp2_tbl_core<false>(r2 * rs, k1, tb);
        c = (pdot * g) * rs;
    } else {
        g = exp2_tbl_core<false>(r2, k1, tb);
        c = pdot * g;
    }
#else
    if (FAM == kFamConical) {
        const double rs = rsqrt_refined(r2);
        g = vexp<FAM>(r2 * rs, k1, tb, in);
        c = (pdot * g) * rs;
    } else {
        g = vexp<FAM>(r2, k1, tb, in);
        c = pdot * g;
    }
#endif
    a.qx = fma(g, s.z, a.qx);
    a.qy = fma(g, s.w, a.qy);
    a.px = fma(c, dx, a.px);
    a.py = fma(c, dy, a.py);
}

// The last CTA of a fused sweep (EPI) turns the CTAs' "rebuild wanted" into the decision: flags[3]
// and, inside a graph, the next stage's IF-node condition (k_finish_verlet's protocol).
__device__ __forceinline__ void epi_decide(const VerletEpi& e, bool need) {
    if (__syncthreads_or(need) && threadIdx.x == 0) atomicOr(&e.flags[0], 1u);
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned prev = atomicAdd(&e.flags[2], 1u);
        if (prev == gridDim.x - 1) {
            const unsigned d = atomicExch(&e.flags[0], 0u);
            e.flags[2] = 0u;
            if (e.use_cond) cudaGraphSetConditional(e.cond, d);
            e.flags[3] = d;
        }
    }
}

template <int FAM, int TPL, bool COUNT, bool EPI>
__global__ void __launch_bounds__(kVB, GS_VERLET_MINB)
    k_verlet_pair(const double4* __restrict__ Ss, const int* __restrict__ list, const long long* __restrict__ ofs,
                  const int* __restrict__ len,
                  const unsigned* __restrict__ perm, int64_t n, int64_t cl0, int64_t cl1, double k1, long long rc2b,
                  double4* __restrict__ part, int64_t row0, DevStatus* st, unsigned long long event,
                  const double* __restrict__ tbl_g, unsigned long long* accepted, const int* __restrict__ cfirst,
                  int64_t n_ev, VerletEpi epi) {
    __shared__ __align__(128) double s_tbl[kTblWords];
    __shared__ unsigned long long s_acc_count, s_tbar;
    table_bulk_issue(s_tbl, tbl_g, &s_tbar);  // lands while the lanes load their members and first records
    if (__syncthreads_or(*((volatile unsigned long long*)&st->first_event) < event)) {
        table_bulk_wait(&s_tbar);
        if (EPI && epi.Xb && epi.decide) epi_decide(epi, false);  // every CTA counts towards the decision
        return;
    }
    if (threadIdx.x == 0) s_acc_count = 0;
    __syncthreads();
    const double* tbl = lane_table(s_tbl);
    const unsigned tb = lane_table_addr(s_tbl);
    const int caphi = pair_clamp_hi(FAM, k1);

    const int sub = (TPL > 1) ? (int)(threadIdx.x % TPL) : 0;
#if GS_VERLET_BALANCE
    // A warp runs to the longest list among its 32 / TPL clusters (28 of 32 lanes busy on C5).  The
    // CTA's kVB / TPL consecutive clusters are dealt to the lane groups in order of list length
    // (ties by index), so a warp's clusters have nearly equal lists; each cluster keeps its lanes'
    // split and summation order — the results are bitwise those of the natural assignment — and
    // the CTA still works on one contiguous run of the sorted order (source records shared in L1).
    constexpr int kSlots = kVB / TPL;
    __shared__ int s_len[kSlots];
    __shared__ long long s_ofs[kSlots];  // loaded beside the lengths: one global round trip less before the first list entry
    __shared__ unsigned char s_slot[kSlots];
    const int slot0 = threadIdx.x / TPL;
    const int64_t cbase = cl0 + (int64_t)blockIdx.x * kSlots;
    if (sub == 0) {
        const bool in = cbase + slot0 < cl1;
        s_len[slot0] = in ? len[cbase + slot0] : -1;
        s_ofs[slot0] = in ? ofs[cbase + slot0] : 0;
    }
    __syncthreads();
    if (sub == 0) {
        const int mine = s_len[slot0];
        int rank = 0;
        for (int k = 0; k < kSlots; ++k) {
            const int o = s_len[k];
            rank += (o > mine) || (o == mine && k < slot0);
        }
        s_slot[rank] = (unsigned char)slot0;
    }
    __syncthreads();
    const int myslot = s_slot[slot0];
    const int64_t c = cbase + myslot;
#else
    const int64_t c = cl0 + (int64_t)blockIdx.x * (kVB / TPL) + threadIdx.x / TPL;
#endif
    const bool valid = c < cl1;
    // members: sorted positions first .. first + cnt - 1 (slab: clusters restart at every cell row,
    // cfirst[c]; otherwise c * M)
    int64_t first = c * kVM;
    int cnt = kVM;
    if (cfirst) {
        first = valid ? cfirst[c] : 0;
        cnt = valid ? cfirst[c + 1] - (int)first : 0;
    } else if (first + kVM > n) {
        cnt = (int)(n - first);
    }
    double4 me[kVM];
    Acc a[kVM];
    int nz[kVM];
#pragma unroll
    for (int m = 0; m < kVM; ++m) {
        const int64_t k = first + m;
        me[m] = (valid && m < cnt) ? Ss[k] : far_record(m);
        a[m] = Acc{0.0, 0.0, 0.0, 0.0};
        nz[m] = 0;
    }
    int nin = 0;
#if GS_VERLET_BALANCE
    const long long beg = valid ? s_ofs[myslot] : 0, end = valid ? beg + s_len[myslot] : 0;
#else
    const long long beg = valid ? ofs[c] : 0, end = valid ? beg + len[c] : 0;
#endif
    // software pipeline: source records two trips ahead (unrolled by three, so the prefetched
    // records rotate through three register sets without moves), list entries three trips ahead,
    // and an L2 prefetch of the list GS_VERLET_PF trips ahead.  Past the end the sentinel n is
    // loaded: always a valid address.  Lists are padded to 2 TPL entries per trip.
    const int2 sent = make_int2((int)n, (int)n);
    const long long step = 2 * TPL;
    long long e = beg + 2 * sub;
    auto ldl = [&](long long x) { return x < end ? __ldg(reinterpret_cast<const int2*>(list + x)) : sent; };
    int2 j = ldl(e);
    GS_ASSERT(!valid || (beg >= 0 && (end - beg) % (2 * TPL) == 0));
    GS_ASSERT(j.x >= 0 && j.x <= n && j.y >= 0 && j.y <= n);
    double4 a0 = Ss[j.x], a1 = Ss[j.y];
    j = ldl(e + step);
    double4 b0 = Ss[j.x], b1 = Ss[j.y];
    int2 jc = ldl(e + 2 * step);
#if GS_VERLET_LIST2
    // a second list entry in flight: an entry is loaded two trips before it addresses its records
    // (with one, the address computation waited on the entry loaded one trip earlier: long
    // scoreboard on 10 % of the sweep's stall samples)
    int2 jd = ldl(e + 3 * step);
#define GS_V_NEXT(k) jc = jd; jd = ldl(e + ((k) + 1) * step)
#else
#define GS_V_NEXT(k) jc = ldl(e + (k) * step)
#endif
    double4 c0, c1;
    table_bulk_wait(&s_tbar);
#if GS_VERLET_UNIFORM
    // warp-uniform trip count (the longest list of the warp's clusters; a warp runs that long
    // anyway): lanes past their own list sweep the sentinel (exact zeros), and the loop's branches
    // and loop-invariant FP64 operands become uniform (constants stay out of the vector registers:
    // a DFMA with three vector-register operands costs ~3.2 instead of 2 pipe cycles)
    const int trips = __reduce_max_sync(kFull, (int)((end - beg) / step));
    for (int t = 0; t < trips; t += 3) {
#else
    const int trips = 0;
    while (true) {
        const int t = -3;
        if (e >= end) break;
#endif
        asm volatile("prefetch.global.L2 [%0];" ::"l"(list + e + GS_VERLET_PF * step));
        GS_ASSERT(jc.x >= 0 && jc.x <= n && jc.y >= 0 && jc.y <= n);
        c0 = Ss[jc.x]; c1 = Ss[jc.y];
        GS_V_NEXT(3);
#pragma unroll
        for (int m = 0; m < kVM; ++m) {
            vbody<FAM, COUNT>(me[m], a0, tbl, tb, k1, caphi, rc2b, a[m], nz[m], nin);
            vbody<FAM, COUNT>(me[m], a1, tbl, tb, k1, caphi, rc2b, a[m], nz[m], nin);
        }
        e += step;
        if (GS_VERLET_UNIFORM ? t + 1 >= trips : e >= end) break;
        a0 = Ss[jc.x]; a1 = Ss[jc.y];
        GS_V_NEXT(3);
#pragma unroll
        for (int m = 0; m < kVM; ++m) {
            vbody<FAM, COUNT>(me[m], b0, tbl, tb, k1, caphi, rc2b, a[m], nz[m], nin);
            vbody<FAM, COUNT>(me[m], b1, tbl, tb, k1, caphi, rc2b, a[m], nz[m], nin);
        }
        e += step;
        if (GS_VERLET_UNIFORM ? t + 2 >= trips : e >= end) break;
        b0 = Ss[jc.x]; b1 = Ss[jc.y];
        GS_V_NEXT(3);
#pragma unroll
        for (int m = 0; m < kVM; ++m) {
            vbody<FAM, COUNT>(me[m], c0, tbl, tb, k1, caphi, rc2b, a[m], nz[m], nin);
            vbody<FAM, COUNT>(me[m], c1, tbl, tb, k1, caphi, rc2b, a[m], nz[m], nin);
        }
        e += step;
    }
#pragma unroll
    for (int m = 0; m < kVM; ++m) {
        for (int off = TPL >> 1; off; off >>= 1) {
            nz[m] += __shfl_xor_sync(kFull, nz[m], off);
            a[m].qx += __shfl_xor_sync(kFull, a[m].qx, off);
            a[m].qy += __shfl_xor_sync(kFull, a[m].qy, off);
            a[m].px += __shfl_xor_sync(kFull, a[m].px, off);
            a[m].py += __shfl_xor_sync(kFull, a[m].py, off);
        }
    }
    bool need = false;
    if (valid && sub == 0) {
#pragma unroll
        for (int m = 0; m < kVM; ++m) {
            if (m >= cnt) continue;
            const int64_t k = first + m;
            const int64_t i = (int64_t)perm[k];
            GS_ASSERT(i >= 0 && i < n_ev);
            if (nz[m] > 1) {  // rare: a coincident particle among the list (reference error, particles.py:92-98)
                for (long long e = beg; e < end; ++e) {
                    const int j = list[e];
                    if (j >= n) continue;
                    const int64_t jo = (int64_t)perm[j];
                    if (jo == i) continue;
                    const double4 s = Ss[j];
                    const double dx = me[m].x - s.x, dy = me[m].y - s.y;
                    if (__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)) != 0.0) continue;
                    if (fma(me[m].z, s.z, me[m].w * s.w) != 0.0)
                        record_event(st, event, (unsigned long long)(i * n_ev + jo));
                }
            }
            if (EPI) {  // k_finish_verlet's arithmetic (the sum as finish_reduce forms it: 0 + v)
                const double sx = 0.0 + a[m].qx, sy = 0.0 + a[m].qy, sz = 0.0 + a[m].px, sw = 0.0 + a[m].py;
                double dqx = sx * epi.scale_q, dqy = sy * epi.scale_q;
                if (epi.sigma2 != 0.0) {
                    dqx = __dadd_rn(dqx, __dmul_rn(epi.sigma2, me[m].z));
                    dqy = __dadd_rn(dqy, __dmul_rn(epi.sigma2, me[m].w));
                }
                const int64_t ri = epi.local ? k - epi.rbase : i;  // row of S / B / A
                const double4 nxt = stage_update(epi.a, ri, dqx, dqy, sz * epi.scale_p, sw * epi.scale_p);
                epi.a.S[ri] = nxt;
                if (!finite4(nxt.x, nxt.y, nxt.z, nxt.w)) record_event(epi.a.st, epi.a.event, kNoEvent);
                if (epi.Ss_next) epi.Ss_next[k] = nxt;
                if (epi.Xb) {
                    const double2 b = epi.Xb[epi.local ? ri : k];
                    const double dx = nxt.x - b.x, dy = nxt.y - b.y;
                    need |= fma(dx, dx, dy * dy) > epi.thr2;
                }
            } else {
                // slab: part in sorted order of the rank's own particles; else at the original index
                part[(cfirst ? k : i) - row0] = make_double4(a[m].qx, a[m].qy, a[m].px, a[m].py);
            }
        }
    }
    if (EPI && epi.Xb) {
        if (epi.decide) epi_decide(epi, need);
        else if (__any_sync(kFull, need) && (threadIdx.x & 31) == 0) atomicOr(&epi.flags[0], 1u);
    }
    if (COUNT) {
        unsigned long long v = (unsigned long long)nin;
        for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(&s_acc_count, v);
        __syncthreads();
        if (threadIdx.x == 0 && s_acc_count) atomicAdd(accepted, s_acc_count);
    }
}

// ---- list build ---------------------------------------------------------------------------

__device__ __forceinline__ int vcell(double v, double v0, double inv_h, int nmax) {
    int c = (int)floor((v - v0) * inv_h);
    return min(max(c, 0), nmax - 1);
}

__device__ __forceinline__ double vcellf(double v, double v0, double inv_h) { return floor((v - v0) * inv_h); }

__device__ __forceinline__ unsigned vhash(double cx, double cy, int ncells) {
    // splitmix64 finalizer of each coordinate's bits (the low bits of small integral doubles are all
    // zero: a plain multiply would put most cells into a few buckets)
    const unsigned long long h = mix64((unsigned long long)__double_as_longlong(cx + 0.0)) ^
                                 mix64((unsigned long long)__double_as_longlong(cy + 0.0) ^ 0xC2B2AE3D27D4EB4Full);
    return (unsigned)h & (unsigned)(ncells - 1);
}

// The cluster's candidates: the union of its members' stencils (gs_cell.cu stencil_ranges),
// generated range by range.  Row-major grid: per stencil row one contiguous sorted range spanning
// every member's trimmed x-range (cells between two consecutive sorted members of one row are
// empty; in other rows the span may add candidates the filter rejects).  Hashed grid: the
// deduplicated buckets of all members' 3 x 3 stencils.  One warp per cluster: every range is
// swept 32 candidates per round, so the loop is warp-uniform.
struct ClusterMembers {
    double mx[kVM], my[kVM];
    float fx[kVM], fy[kVM];
    int nm;
};

template <typename F>
__device__ __forceinline__ void for_each_range(const GridParams& g, const int* __restrict__ start,
                                               const ClusterMembers& cm, F&& f) {
    if (!g.hashed) {
        const int sub = g.sub;
        int cy[kVM];
        int lo = g.ny, hi = -1;
#pragma unroll
        for (int m = 0; m < kVM; ++m) {
            cy[m] = m < cm.nm ? vcell(cm.my[m], g.y0, g.inv_h, g.ny) : 0;
            if (m < cm.nm) { lo = min(lo, cy[m]); hi = max(hi, cy[m]); }
        }
        const double rc2 = g.rc * g.rc;
        for (int yy = max(lo - sub, g.ylo); yy <= min(hi + sub, g.yhi - 1); ++yy) {
            int xa = g.nx, xb = -1;
#pragma unroll
            for (int m = 0; m < kVM; ++m) {
                if (m >= cm.nm || yy < cy[m] - sub || yy > cy[m] + sub) continue;
                int a, b;
                if (sub > 1) {
                    const double ylo = fma((double)yy, g.h, g.y0), yhi = ylo + g.h;
                    const double gap = fmax(0.0, fmax(ylo - cm.my[m], cm.my[m] - yhi));
                    const double xr2 = fma(-gap, gap, rc2);
                    if (!(xr2 > 0.0)) continue;
                    const double xr = sqrt(xr2);
                    a = vcell(cm.mx[m] - xr, g.x0, g.inv_h, g.nx);
                    b = vcell(cm.mx[m] + xr, g.x0, g.inv_h, g.nx);
                } else {
                    const int cx = vcell(cm.mx[m], g.x0, g.inv_h, g.nx);
                    a = max(cx - 1, 0);
                    b = min(cx + 1, g.nx - 1);
                }
                xa = min(xa, a);
                xb = max(xb, b);
            }
            const int r0 = (yy - g.ylo) * g.nx;  // `start` covers rows [ylo, yhi)
            if (xb >= xa) f(start[r0 + xa], start[r0 + xb + 1]);
        }
        return;
    }
    for (int m = 0; m < cm.nm; ++m) {
        const double cx = vcellf(cm.mx[m], g.x0, g.inv_h), cy = vcellf(cm.my[m], g.y0, g.inv_h);
        for (int t = 0; t < 9; ++t) {
            const unsigned key = vhash(cx + (t % 3 - 1), cy + (t / 3 - 1), g.ncells);
            bool dup = false;  // the bucket already came up for an earlier (member, cell)?
            for (int m2 = 0; m2 <= m && !dup; ++m2) {
                const double cx2 = vcellf(cm.mx[m2], g.x0, g.inv_h), cy2 = vcellf(cm.my[m2], g.y0, g.inv_h);
                for (int t2 = 0; t2 < (m2 == m ? t : 9); ++t2)
                    dup |= vhash(cx2 + (t2 % 3 - 1), cy2 + (t2 / 3 - 1), g.ncells) == key;
            }
            if (!dup) f(start[key], start[key + 1]);
        }
    }
}

__device__ __forceinline__ int64_t cluster_first(const int* __restrict__ cfirst, int64_t c) {
    return cfirst ? (int64_t)cfirst[c] : c * kVM;
}

__device__ __forceinline__ void load_members(const double4* __restrict__ Ss, const float2* __restrict__ Sf, int64_t n,
                                             int64_t c, const int* __restrict__ cfirst, ClusterMembers& cm) {
    cm.nm = 0;
    const int64_t first = cluster_first(cfirst, c);
    const int64_t end = cfirst ? (int64_t)cfirst[c + 1] : n;
#pragma unroll
    for (int m = 0; m < kVM; ++m) {
        const int64_t k = first + m;
        if (k < end) {
            const double4 v = Ss[k];
            cm.mx[m] = v.x; cm.my[m] = v.y;
            const float2 f = Sf[k];
            cm.fx[m] = f.x; cm.fy[m] = f.y;
            cm.nm = m + 1;
        } else {
            cm.mx[m] = cm.my[m] = 0.0;
            cm.fx[m] = cm.fy[m] = 0.0f;
        }
    }
}

// Capacity of cluster c's list: its candidate count (every range's length), padded to `pad` — an
// upper bound of the filtered list, found without touching a candidate (one thread per cluster).
__global__ void __launch_bounds__(256) k_verlet_caps(const float2* __restrict__ Sf, const double4* __restrict__ Ss,
                                                     const int* __restrict__ start, const GridParams* __restrict__ gp,
                                                     int64_t n, int64_t ncl, int pad, long long* cap,
                                                     const int* __restrict__ cfirst) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncl) return;
    const GridParams g = *gp;
    ClusterMembers cm;
    load_members(Ss, Sf, n, c, cfirst, cm);
    long long total = 0;
    for_each_range(g, start, cm, [&](int a, int b) { total += b - a; });
    cap[c] = (total + pad - 1) / pad * pad;
}

// list[ofs[c] ...] = the sorted positions within the list radius of any member, in canonical order
// (ballot compaction, one warp per cluster), padded to a multiple of `pad` with n (the sentinel far
// record Ss[n]); len[c] = the padded length; Xb[k] = positions at the build.
__global__ void __launch_bounds__(kVBB) k_verlet_fill(const float2* __restrict__ Sf, const double4* __restrict__ Ss,
                                                      const int* __restrict__ start, const GridParams* __restrict__ gp,
                                                      int64_t n, int64_t ncl, int pad, const long long* __restrict__ ofs,
                                                      int* len, int* list, int64_t cap, double2* Xb,
                                                      const unsigned* __restrict__ perm, int* inv,
                                                      unsigned long long* overflow, const int* __restrict__ cfirst,
                                                      int64_t xb_base) {
    const int sub = threadIdx.x & 31;
    const int64_t c = (int64_t)blockIdx.x * (kVBB / kTplB) + threadIdx.x / kTplB;
    if (c >= ncl) return;  // warp-uniform
    const GridParams g = *gp;
    ClusterMembers cm;
    load_members(Ss, Sf, n, c, cfirst, cm);
#pragma unroll
    for (int m = 0; m < kVM; ++m)
        if (sub == m && m < cm.nm) {
            const int64_t k = cluster_first(cfirst, c) + m;
            Xb[k - xb_base] = make_double2(cm.mx[m], cm.my[m]);
            if (inv) inv[perm[k]] = (int)k;  // original index -> sorted slot (the fused stage epilogue's gather)
        }
    const int64_t obase = ofs[c];
    const bool ok = ofs[ncl] <= cap;  // the list buffer holds the whole build
    if (!ok) {  // no list: the sweep reads nothing (the call is redone with a larger buffer)
        if (sub == 0) {
            atomicMax(overflow, (unsigned long long)ofs[ncl]);
            len[c] = 0;
        }
        return;
    }
    const float rc2f = g.rc2f;
    int count = 0;
    for_each_range(g, start, cm, [&](int a, int b) {
        for (int base = a; base < b; base += kTplB) {
            const int pos = base + sub;
            bool acc = false;
            if (pos < b) {
                const float2 f = Sf[pos];
                float d2 = INFINITY;
#pragma unroll
                for (int m = 0; m < kVM; ++m) {
                    const float dx = cm.fx[m] - f.x, dy = cm.fy[m] - f.y;
                    const float dm = fmaf(dx, dx, dy * dy);
                    d2 = m < cm.nm ? fminf(d2, dm) : d2;
                }
                acc = !(d2 >= rc2f);  // NaN radius (filter off): keep
            }
            const unsigned bal = __ballot_sync(kFull, acc);
            const int64_t widx = obase + count + __popc(bal & ((1u << sub) - 1));
            GS_ASSERT(!acc || (pos >= 0 && pos < n && widx < ofs[c + 1]));
            if (acc) list[widx] = pos;
            count += __popc(bal);
        }
    });
    const int padded = (count + pad - 1) / pad * pad;
    GS_ASSERT(obase + padded <= ofs[c + 1] && ofs[c + 1] <= cap);
    for (int e = count + sub; e < padded; e += kTplB) list[obase + e] = (int)n;  // padding: sentinel
    if (sub == 0) len[c] = padded;
}

// Packed FP32 pairs (sm_100: FADD2 / FMUL2 / FFMA2 on {lo, hi} = two members).
#ifndef GS_VERLET_FILL_F32X2   // A/B: 0 = one member at a time
#define GS_VERLET_FILL_F32X2 1
#endif
__device__ __forceinline__ unsigned long long f32x2_pack(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ unsigned long long f32x2_splat(float v) { return f32x2_pack(v, v); }
__device__ __forceinline__ float f32x2_lo(unsigned long long v) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
    return lo;
}
__device__ __forceinline__ float f32x2_hi(unsigned long long v) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
    return hi;
}
__device__ __forceinline__ unsigned long long f32x2_sub(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ unsigned long long f32x2_mul(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ unsigned long long f32x2_fma(unsigned long long a, unsigned long long b,
                                                        unsigned long long c) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// The same lists for kVQ consecutive clusters per warp (row-major grid): per stencil row the warp
// sweeps the union of the clusters' ranges once, each candidate is tested against every member
// (fp32) and appended to each cluster whose own range holds it and whose members it is near —
// exactly the lists of k_verlet_fill (same candidates, same order), at a third of its loads,
// ballots and loop overhead (consecutive clusters share most of their stencil).  The members'
// x-ranges are computed one member per lane.  Hashed grids: the per-cluster loop.
#ifndef GS_VERLET_FILL_Q        // clusters per warp in the grouped list build (A/B)
#define GS_VERLET_FILL_Q 4
#endif
constexpr int kVQ = GS_VERLET_FILL_Q;
constexpr int kVQM = kVQ * kVM;  // members per warp (<= 32)
static_assert(kVQM <= 32, "one lane per member");

__global__ void __launch_bounds__(kVBB) k_verlet_fill_grp(const float2* __restrict__ Sf, const double4* __restrict__ Ss,
                                                          const int* __restrict__ start,
                                                          const GridParams* __restrict__ gp, int64_t n, int64_t ncl,
                                                          int pad, const long long* __restrict__ ofs, int* len,
                                                          int* list, int64_t cap, double2* Xb,
                                                          const unsigned* __restrict__ perm, int* inv,
                                                          unsigned long long* overflow, const int* __restrict__ cfirst,
                                                          int64_t xb_base) {
    const int lane = threadIdx.x & 31;
    const int64_t c0 = ((int64_t)blockIdx.x * (kVBB / 32) + threadIdx.x / 32) * kVQ;
    if (c0 >= ncl) return;  // warp-uniform
    const GridParams g = *gp;
    const int nq = (int)min((int64_t)kVQ, ncl - c0);
    const bool ok = ofs[ncl] <= cap;
    // lane t < kVQM: member t % kVM of cluster c0 + t / kVM
    const int tq = lane / kVM, tm = lane % kVM;
    bool mv = false;
    double mx = 0.0, my = 0.0;
    float fx = 0.0f, fy = 0.0f;
    if (lane < kVQM && tq < nq) {
        const int64_t c = c0 + tq;
        const int64_t k = cluster_first(cfirst, c) + tm;
        const int64_t end = cfirst ? (int64_t)cfirst[c + 1] : n;
        if (k < end) {
            mv = true;
            const double4 v = Ss[k];
            mx = v.x; my = v.y;
            const float2 f = Sf[k];
            fx = f.x; fy = f.y;
            Xb[k - xb_base] = make_double2(mx, my);
            if (inv) inv[perm[k]] = (int)k;  // original index -> sorted slot
        }
    }
    if (!ok) {  // no list: the sweep reads nothing (the call is redone with a larger buffer)
        if (lane < nq) {
            atomicMax(overflow, (unsigned long long)ofs[ncl]);
            len[c0 + lane] = 0;
        }
        return;
    }
    if (g.hashed) {  // flung-apart clouds: the per-cluster candidate walk of k_verlet_fill
        for (int q = 0; q < nq; ++q) {
            const int64_t c = c0 + q;
            ClusterMembers cm;
            load_members(Ss, Sf, n, c, cfirst, cm);
            const int64_t obase = ofs[c];
            int count = 0;
            for_each_range(g, start, cm, [&](int a, int b) {
                for (int base = a; base < b; base += 32) {
                    const int pos = base + lane;
                    bool acc = false;
                    if (pos < b) {
                        const float2 f = Sf[pos];
                        float d2 = INFINITY;
#pragma unroll
                        for (int m = 0; m < kVM; ++m) {
                            const float dx = cm.fx[m] - f.x, dy = cm.fy[m] - f.y;
                            const float dm = fmaf(dx, dx, dy * dy);
                            d2 = m < cm.nm ? fminf(d2, dm) : d2;
                        }
                        acc = !(d2 >= g.rc2f);
                    }
                    const unsigned bal = __ballot_sync(kFull, acc);
                    if (acc) list[obase + count + __popc(bal & ((1u << lane) - 1))] = pos;
                    count += __popc(bal);
                }
            });
            const int padded = (count + pad - 1) / pad * pad;
            for (int e = count + lane; e < padded; e += 32) list[obase + e] = (int)n;
            if (lane == 0) len[c] = padded;
        }
        return;
    }
    // every lane holds every member's fp32 position (the filter); a missing member sits at 3e38,
    // whose squared distance overflows to +inf and never passes (with the filter off — a NaN radius
    // — acceptance only follows the cluster's own ranges, which skip missing members)
    float qfx[kVQM], qfy[kVQM];
#pragma unroll
    for (int t = 0; t < kVQM; ++t) {
        qfx[t] = __shfl_sync(kFull, mv ? fx : 3e38f, t);
        qfy[t] = __shfl_sync(kFull, mv ? fy : 3e38f, t);
    }
#if GS_VERLET_FILL_F32X2
    static_assert(kVM == 2, "packed member pairs");
    unsigned long long qx2[kVQ], qy2[kVQ];
#pragma unroll
    for (int q = 0; q < kVQ; ++q) {
        qx2[q] = f32x2_pack(qfx[2 * q], qfx[2 * q + 1]);
        qy2[q] = f32x2_pack(qfy[2 * q], qfy[2 * q + 1]);
    }
#endif
    int wpos[kVQ];  // each cluster's next list slot (32-bit: a build never exceeds 2^31 entries)
#pragma unroll
    for (int q = 0; q < kVQ; ++q) wpos[q] = q < nq ? (int)ofs[c0 + q] : 0;
    const unsigned lt = (1u << lane) - 1u;  // lanes below this one
    const int sub = g.sub;
    const int cy = mv ? vcell(my, g.y0, g.inv_h, g.ny) : 0;
    int lo = __reduce_min_sync(kFull, mv ? cy : g.ny), hi = __reduce_max_sync(kFull, mv ? cy : -1);
    const double rc2 = g.rc * g.rc;
    const float rc2f = g.rc2f;
    // a row's candidate ranges: this lane's member's trimmed x-range of cells in row yy (as
    // for_each_range), the clusters' unions by shuffles, their sorted-position ranges from `start`
    auto row_ranges = [&](int yy, int* pa, int* pb, int& A, int& B) {
        int a = g.nx, b = -1;
        if (mv && yy >= cy - sub && yy <= cy + sub) {
            if (sub > 1) {
                const double ylo = fma((double)yy, g.h, g.y0), yhi = ylo + g.h;
                const double gap = fmax(0.0, fmax(ylo - my, my - yhi));
                const double xr2 = fma(-gap, gap, rc2);
                if (xr2 > 0.0) {
                    const double xr = sqrt(xr2);
                    a = vcell(mx - xr, g.x0, g.inv_h, g.nx);
                    b = vcell(mx + xr, g.x0, g.inv_h, g.nx);
                }
            } else {
                const int cx = vcell(mx, g.x0, g.inv_h, g.nx);
                a = max(cx - 1, 0);
                b = min(cx + 1, g.nx - 1);
            }
        }
        const int r0 = (yy - g.ylo) * g.nx;
        A = 0x7fffffff;
        B = -1;
#pragma unroll
        for (int q = 0; q < kVQ; ++q) {
            int xa = g.nx, xb = -1;
#pragma unroll
            for (int m = 0; m < kVM; ++m) {
                xa = min(xa, __shfl_sync(kFull, a, q * kVM + m));
                xb = max(xb, __shfl_sync(kFull, b, q * kVM + m));
            }
            pa[q] = 0; pb[q] = 0;
            if (xb >= xa) {
                pa[q] = start[r0 + xa];
                pb[q] = start[r0 + xb + 1];
            }
        }
    };
    const int y_first = max(lo - sub, g.ylo), y_last = min(hi + sub, g.yhi - 1);
    // software pipeline over the rows: the next row's `start` loads are in flight while this
    // row's candidates are filtered
    int na[kVQ], nb[kVQ], nA = 0, nB = -1;
    if (y_first <= y_last) row_ranges(y_first, na, nb, nA, nB);
    for (int yy = y_first; yy <= y_last; ++yy) {
        int pa[kVQ], pb[kVQ];
#pragma unroll
        for (int q = 0; q < kVQ; ++q) { pa[q] = na[q]; pb[q] = nb[q]; }
        if (yy < y_last) row_ranges(yy + 1, na, nb, nA, nB);
        int A = 0x7fffffff, B = -1, span = 0;
#pragma unroll
        for (int q = 0; q < kVQ; ++q)
            if (pb[q] > pa[q] || pa[q] != 0) { A = min(A, pa[q]); B = max(B, pb[q]); span += pb[q] - pa[q]; }
        // candidates [a, b) tested against the clusters in qmask, appended in position order
        auto sweep_range = [&](int a, int b, unsigned qmask) {
            for (int base = a; base < b; base += 32) {
                const int pos = base + lane;
                float2 f = make_float2(0.0f, 0.0f);
                if (pos < b) f = Sf[pos];
#if GS_VERLET_FILL_F32X2
                const unsigned long long fxx = f32x2_splat(f.x), fyy = f32x2_splat(f.y);
#endif
#pragma unroll
                for (int q = 0; q < kVQ; ++q) {
                    if (!((qmask >> q) & 1u)) continue;  // warp-uniform
#if GS_VERLET_FILL_F32X2
                    // both members at once on the packed FP32 pipe (FADD2 / FMUL2 / FFMA2): the
                    // same roundings as fmaf(dx, dx, dy * dy) per member
                    const unsigned long long dx2 = f32x2_sub(qx2[q], fxx), dy2 = f32x2_sub(qy2[q], fyy);
                    const unsigned long long d22 = f32x2_fma(dx2, dx2, f32x2_mul(dy2, dy2));
                    const float d2 = fminf(fminf(INFINITY, f32x2_lo(d22)), f32x2_hi(d22));
#else
                    float d2 = INFINITY;
#pragma unroll
                    for (int m = 0; m < kVM; ++m) {
                        const int t = q * kVM + m;
                        const float dx = qfx[t] - f.x, dy = qfy[t] - f.y;
                        d2 = fminf(d2, fmaf(dx, dx, dy * dy));
                    }
#endif
                    const bool acc = (pos >= pa[q]) & (pos < pb[q]) & !(d2 >= rc2f);  // NaN radius: keep
                    const unsigned bal = __ballot_sync(kFull, acc);
                    GS_ASSERT(!acc || (pos < n && wpos[q] + __popc(bal) <= ofs[c0 + q + 1]));
                    const int at = wpos[q] + __popc(bal & lt);
                    if (acc) list[at] = pos;
                    wpos[q] += __popc(bal);
                }
            }
        };
        // clusters far apart in the row (the group wraps to the next cell row: one cluster at the
        // row's end, the next at its start) would sweep the whole row between them — a warp
        // hundreds of rounds long that sets the kernel's tail; sweep their ranges one by one
        // instead (each cluster still gets its candidates in position order: the same lists)
        if (B - A <= 2 * span + 64) {
            sweep_range(A, B, (1u << kVQ) - 1u);
        } else {
#pragma unroll
            for (int q = 0; q < kVQ; ++q)
                if (pb[q] > pa[q]) sweep_range(pa[q], pb[q], 1u << q);
        }
    }
#pragma unroll
    for (int q = 0; q < kVQ; ++q) {
        if (q >= nq) break;
        const int base = (int)ofs[c0 + q], count = wpos[q] - base;
        const int padded = (count + pad - 1) / pad * pad;
        GS_ASSERT(base + padded <= ofs[c0 + q + 1]);
        for (int e = count + lane; e < padded; e += 32) list[base + e] = (int)n;  // padding: sentinel
        if (lane == 0) len[c0 + q] = padded;
    }
}

#ifndef GS_VERLET_FILL_GRP   // A/B: 0 = one warp per cluster (k_verlet_fill)
#define GS_VERLET_FILL_GRP 1
#endif

void launch_fill(const float2* Sf, const double4* Ss, const int* start, const GridParams* gp, int64_t n, int64_t ncl,
                 int pad, const long long* ofs, int* len, int* list, int64_t cap, double2* Xb, const unsigned* perm,
                 int* inv, unsigned long long* overflow, const int* cfirst, int64_t xb_base, cudaStream_t stream) {
    if (ncl <= 0) return;
#if GS_VERLET_FILL_GRP
    const int64_t warps = (ncl + kVQ - 1) / kVQ;
    const unsigned blocks = (unsigned)((warps * 32 + kVBB - 1) / kVBB);
    k_verlet_fill_grp<<<blocks, kVBB, 0, stream>>>(Sf, Ss, start, gp, n, ncl, pad, ofs, len, list, cap, Xb, perm, inv,
                                                   overflow, cfirst, xb_base);
#else
    const unsigned blocks = (unsigned)((ncl * kTplB + kVBB - 1) / kVBB);
    k_verlet_fill<<<blocks, kVBB, 0, stream>>>(Sf, Ss, start, gp, n, ncl, pad, ofs, len, list, cap, Xb, perm, inv,
                                               overflow, cfirst, xb_base);
#endif
}

// Gather of the stage records into sorted order + the rebuild trigger.  The last CTA decides:
// rebuild if forced or any particle moved more than half the skin since the build; in a graph
// it sets the IF node's condition, otherwise flags[3] (host-driven paths always rebuild).
__global__ void __launch_bounds__(256) k_verlet_gather(const double4* __restrict__ S, const unsigned* __restrict__ perm,
                                                       int64_t n, double4* Ss, const double2* __restrict__ Xb,
                                                       double thr2, unsigned* flags, int force,
                                                       cudaGraphConditionalHandle cond, int use_cond) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool need = false;
    if (!force && k < n) {
        const double4 v = S[perm[k]];
        Ss[k] = v;
        const double2 b = Xb[k];
        const double dx = v.x - b.x, dy = v.y - b.y;
        need = fma(dx, dx, dy * dy) > thr2;
    }
    if (__syncthreads_or(need) && threadIdx.x == 0) atomicOr(&flags[0], 1u);
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned prev = atomicAdd(&flags[2], 1u);
        if (prev == gridDim.x - 1) {
            const unsigned f = force ? 1u : atomicExch(&flags[0], 0u);
            flags[0] = 0u;
            flags[2] = 0u;
            if (use_cond) cudaGraphSetConditional(cond, f);
            flags[3] = f;
        }
    }
}

__global__ void k_verlet_sentinel(double4* Ss, double4* Ss0, double4* Ss1, int64_t n, unsigned* flags) {
    Ss[n] = far_record(0);
    if (Ss0) Ss0[n] = far_record(0);  // the ping-pong halves (a buffer sized for a larger n holds a stale record at n)
    if (Ss1) Ss1[n] = far_record(0);
    flags[1] += 1u;  // builds so far (diagnostics)
    flags[2] = 0u;   // decision counter (a failed evolve may have left CTAs uncounted)
    flags[4] = 0u;   // RHS since the build (the adaptive skin's interval)
}

__global__ void k_skin_init(double* c, double s0) {
    c[0] = s0;
    c[1] = 0.0;
}

}  // namespace

int verlet_tpl(int64_t n) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t ncl = (n + kVM - 1) / kVM;
    // A/B knobs (read per call): lanes grow until clusters * lanes >= SMs * depth; minimum lanes
    const char* ed = std::getenv("GS_B200_VERLET_DEPTH");
    const int depth = ed ? std::max(1, std::atoi(ed)) : GS_VERLET_DEPTH;
    const char* et = std::getenv("GS_B200_VERLET_TPL");
    const int tv = et ? std::atoi(et) : 4;
    const int tpl_min = (tv == 1 || tv == 2 || tv == 4 || tv == 8 || tv == 16) ? tv : 4;
    int tpl = tpl_min;
    while (tpl < 16 && ncl * tpl < (int64_t)sms * depth) tpl *= 2;
    return tpl;
}

int64_t verlet_clusters(int64_t n) { return (n + kVM - 1) / kVM; }

size_t verlet_scan_bytes(int64_t ncl) {
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const long long*)nullptr, (long long*)nullptr, (int)(ncl + 1));
    return bytes;
}

int verlet_build(const CellWs& w, const VerletWs& v, const double4* S, int64_t n, double cutoff, cudaStream_t stream) {
    const double rl = cutoff * (1.0 + v.skin);
    int rc = cell_build(w, S, n, rl, stream, v.skin_ctl, cutoff);
    if (rc) return rc;
    k_verlet_sentinel<<<1, 1, 0, stream>>>(w.Ss, v.Ss_pair[0], v.Ss_pair[1], n, v.flags);
    const int64_t ncl = verlet_clusters(n);
    const int pad = 2 * v.tpl;
    k_verlet_caps<<<(unsigned)((ncl + 255) / 256), 256, 0, stream>>>(w.Sf, w.Ss, w.start, w.gp, n, ncl, pad, v.cnt,
                                                                     nullptr);
    size_t bytes = v.scan_bytes;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(v.scan_temp, bytes, v.cnt, v.ofs, (int)(ncl + 1), stream);
    if (e != cudaSuccess) return (int)e;
    launch_fill(w.Sf, w.Ss, w.start, w.gp, n, ncl, pad, v.ofs, v.len, v.list, v.cap, v.Xb, w.perm, v.inv, v.overflow,
                nullptr, 0, stream);
    return (int)cudaGetLastError();
}

void verlet_gather(const CellWs& w, const VerletWs& v, const double4* S, int64_t n, int force,
                   cudaGraphConditionalHandle cond, int use_cond, cudaStream_t stream) {
    const double thr = 0.5 * v.skin * v.cutoff;
    k_verlet_gather<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(S, w.perm, n, w.Ss, v.Xb, thr * thr * (1.0 - 1e-9),
                                                                     v.flags, force, cond, use_cond);
}

// ---- the rebuild trigger of large clouds: relative displacement of neighbours ----------------
// A list built with radius rl = cutoff (1 + skin) stays exact while no pair that was >= rl apart at
// the build has come closer than the cutoff.  Blanket rule (the fused epilogue, small clouds):
// rebuild when any particle moved skin cutoff / 2.  Here, with Delta_i = x_i(t) - x_i(build):
// coarse cells of edge L = 2 rl (by the build positions) get the bounding box B_C of their
// particles' Delta; a pair in the same or adjacent coarse cells has |Delta_i - Delta_j| <=
// diam(B_C u B_C'), a pair in non-adjacent cells started >= L apart.  So the lists hold while
//   diam(B_C u B_C') < skin cutoff for every adjacent / same pair of cells, and
//   max |Delta| < (L - cutoff) / 2.
// In a smooth flow neighbours move together and rebuilds get rarer.  Boxes are kept as
// order-preserving 32-bit keys of the displacements rounded outwards to float (a valid, slightly
// wider box): one warp reduction (REDUX) per run of a coarse cell, then 4 atomics.
namespace {
__device__ __forceinline__ unsigned fkey(float v) {  // monotone float -> unsigned
    const unsigned u = __float_as_uint(v);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float funkey(unsigned k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}
constexpr unsigned kBoxEmptyMin = 0xffffffffu, kBoxEmptyMax = 0u;

struct TriggerArgs {
    const double4* Ss;         // the stage's records in sorted order
    const double2* Xb;         // their positions at the build
    const unsigned* keys;      // the build's sorted cell keys (cell above GS_CELL_SUBKEY bits)
    const GridParams* gp;
    int64_t n;
    unsigned* box;             // 4 per coarse cell: min x, max x, min y, max y (keys); capacity `cap`
    int64_t cap;
    double skin, cutoff;       // the list's skin (skin_ctl[0] when adaptive) and the kernel cutoff
    double* skin_ctl;          // adaptive skin {skin, RHS per unit skin} (nullptr: fixed)
    unsigned* flags;
    cudaGraphConditionalHandle cond;
    int use_cond;
};

// The trigger's thresholds for the current list's skin: lim2 = (skin cutoff)^2, mlim2 =
// ((L - cutoff) / 2)^2 with L = 2 rl, both slightly reduced; thr2 = the blanket rule's
// (skin cutoff / 2)^2 (hashed grids).
struct TriggerLimits {
    double lim2, mlim2, thr2;
};
__device__ __forceinline__ TriggerLimits trigger_limits(const TriggerArgs& t) {
    const double skin = t.skin_ctl ? t.skin_ctl[0] : t.skin;
    const double lim = skin * t.cutoff, rl = t.cutoff * (1.0 + skin), mlim = 0.5 * (2.0 * rl - t.cutoff);
    const double thr = 0.5 * skin * t.cutoff;
    return TriggerLimits{lim * lim * (1.0 - 1e-6), mlim * mlim * (1.0 - 1e-6), thr * thr * (1.0 - 1e-9)};
}

// The adaptive skin (relative trigger path): a rebuild after I RHS on a list of skin s observes
// a = I / s RHS per unit skin (smoothed over the builds); per RHS the sweep costs ~(1 + s)^2 and
// the builds ~kSkinCostRatio / (a s) sweeps, minimal where s^2 (1 + s) = kSkinCostRatio / (2 a).
// The next list's skin moves there (Newton), by at most x1.5 per build, within [kSkinMin,
// kSkinMax].  Measured optimum (tools/skin_scan.py): C5 ~0.1 (a rebuild every ~2.7 RHS at 0.05),
// C4 0.03-0.05 (every ~9.5 RHS).
__device__ void verlet_skin_adapt(double* c, unsigned since) {
    const double s = c[0];
    const double a_obs = (double)since / s;
    const double a = c[1] > 0.0 ? 0.5 * (c[1] + a_obs) : a_obs;
    c[1] = a;
    const double K = kSkinCostRatio / (2.0 * a);
    double x = s;
    for (int it = 0; it < 8; ++it) x -= (x * x * (1.0 + x) - K) / (x * (2.0 + 3.0 * x));
    c[0] = fmin(fmax(x, fmax(kSkinMin, s / 1.5)), fmin(kSkinMax, s * 1.5));
}

// Phase 1 (one thread per particle, sorted order): the coarse cells' displacement boxes (or, without
// coarse cells, the blanket rule straight into flags[0]).
__global__ void __launch_bounds__(256) k_verlet_trigger(TriggerArgs t) {
    const GridParams g = *t.gp;
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = k < t.n;
    const int fct = 2 * max(g.sub, 1);  // fine cells per coarse cell: L = fct h = 2 rl
    const int ncx = g.hashed ? 1 : (g.nx + fct - 1) / fct, ncy = g.hashed ? 1 : (g.ny + fct - 1) / fct;
    const bool coarse = !g.hashed && (int64_t)ncx * ncy * 4 <= t.cap;
    bool need = false;
    const TriggerLimits lm = trigger_limits(t);
    double2 d = make_double2(0.0, 0.0);
    if (valid) {
        const double4 x = t.Ss[k];
        const double2 b = t.Xb[k];
        d = make_double2(x.x - b.x, x.y - b.y);
    }
    if (!coarse) {
        need = valid && fma(d.x, d.x, d.y * d.y) > lm.thr2;
    } else {
        int cc = -1;
        if (valid) {
            const unsigned cell = t.keys[k] >> GS_CELL_SUBKEY;
            const int cy = (int)(cell / (unsigned)g.nx), cx = (int)(cell % (unsigned)g.nx);
            cc = (cy / fct) * ncx + cx / fct;
        }
        const unsigned act = __ballot_sync(0xffffffffu, valid);
        if (valid) {
            const unsigned peers = __match_any_sync(act, cc);
            const unsigned mnx = __reduce_min_sync(peers, fkey(__double2float_rd(d.x)));
            const unsigned mxx = __reduce_max_sync(peers, fkey(__double2float_ru(d.x)));
            const unsigned mny = __reduce_min_sync(peers, fkey(__double2float_rd(d.y)));
            const unsigned mxy = __reduce_max_sync(peers, fkey(__double2float_ru(d.y)));
            if ((threadIdx.x & 31) == __ffs(peers) - 1) {
                unsigned* b = t.box + 4 * (int64_t)cc;
                atomicMin(&b[0], mnx); atomicMax(&b[1], mxx); atomicMin(&b[2], mny); atomicMax(&b[3], mxy);
            }
        }
    }
    if (__syncthreads_or(need) && threadIdx.x == 0) atomicOr(&t.flags[0], 1u);
}

// Phase 2 (grid-stride over the coarse cells, kTrigCheckCtas CTAs): every cell against itself and
// its forward neighbours, all eight box words loaded before any test (one L2 round trip per
// cell, where the last CTA of a single kernel used to walk every cell with a dependent load chain
// — 45 of the 60 us of the C5 trigger); the last CTA empties the boxes and decides.
constexpr int kTrigCheckCtas = 148;
__global__ void __launch_bounds__(256) k_verlet_trigger_check(TriggerArgs t) {
    const GridParams g = *t.gp;
    const int fct = 2 * max(g.sub, 1);
    const int ncx = g.hashed ? 1 : (g.nx + fct - 1) / fct, ncy = g.hashed ? 1 : (g.ny + fct - 1) / fct;
    const bool coarse = !g.hashed && (int64_t)ncx * ncy * 4 <= t.cap;
    const int ncell = coarse ? ncx * ncy : 0;
    const TriggerLimits lm = trigger_limits(t);
    bool bad = false;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncell; c += gridDim.x * blockDim.x) {
        const uint4 a = __ldcg(reinterpret_cast<const uint4*>(t.box) + c);
        const int cx = c % ncx, cy = c / ncx;
        const int nb[4][2] = {{1, 0}, {-1, 1}, {0, 1}, {1, 1}};
        uint4 e[4];
        bool ok[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int ex = cx + nb[q][0], ey = cy + nb[q][1];
            ok[q] = ex >= 0 && ex < ncx && ey < ncy;
            e[q] = ok[q] ? __ldcg(reinterpret_cast<const uint4*>(t.box) + ((int64_t)ey * ncx + ex))
                         : make_uint4(kBoxEmptyMin, kBoxEmptyMax, kBoxEmptyMin, kBoxEmptyMax);
        }
        if (a.x == kBoxEmptyMin) continue;
        const float ax0 = funkey(a.x), ax1 = funkey(a.y), ay0 = funkey(a.z), ay1 = funkey(a.w);
        const double mx = fmax(fabs((double)ax0), fabs((double)ax1)), my = fmax(fabs((double)ay0), fabs((double)ay1));
        bad |= fma(mx, mx, my * my) >= lm.mlim2;
        {   // the cell itself
            const double wx = (double)ax1 - (double)ax0, wy = (double)ay1 - (double)ay0;
            bad |= fma(wx, wx, wy * wy) >= lm.lim2;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (!ok[q] || e[q].x == kBoxEmptyMin) continue;
            const double wx = (double)fmaxf(ax1, funkey(e[q].y)) - (double)fminf(ax0, funkey(e[q].x));
            const double wy = (double)fmaxf(ay1, funkey(e[q].w)) - (double)fminf(ay0, funkey(e[q].z));
            bad |= fma(wx, wx, wy * wy) >= lm.lim2;
        }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&t.flags[0], 1u);
    __shared__ unsigned s_last;
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(&t.flags[2], 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    // the last CTA: every check is done; empty the boxes for the next stage and decide
    __threadfence();
    for (int c = threadIdx.x; c < ncell; c += blockDim.x)
        reinterpret_cast<uint4*>(t.box)[c] = make_uint4(kBoxEmptyMin, kBoxEmptyMax, kBoxEmptyMin, kBoxEmptyMax);
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned dflag = atomicExch(&t.flags[0], 0u) != 0u ? 1u : 0u;
        t.flags[2] = 0u;
        const unsigned since = t.flags[4] + 1u;  // RHS on this list (k_verlet_sentinel zeroes it)
        t.flags[4] = since;
        if (dflag && t.skin_ctl) verlet_skin_adapt(t.skin_ctl, since);
        if (t.use_cond) cudaGraphSetConditional(t.cond, dflag);
        t.flags[3] = dflag;
    }
}

__global__ void k_box_reset(unsigned* box, int64_t cells) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= cells) return;
    box[4 * c] = kBoxEmptyMin; box[4 * c + 1] = kBoxEmptyMax; box[4 * c + 2] = kBoxEmptyMin; box[4 * c + 3] = kBoxEmptyMax;
}
}  // namespace

void verlet_skin_init(double* skin_ctl, double skin0, cudaStream_t stream) {
    k_skin_init<<<1, 1, 0, stream>>>(skin_ctl, skin0);
}

void verlet_box_reset(unsigned* box, int64_t cells, cudaStream_t stream) {
    if (cells > 0) k_box_reset<<<(unsigned)((cells + 255) / 256), 256, 0, stream>>>(box, cells);
}

void launch_verlet_trigger(const CellWs& w, const VerletWs& v, int64_t n, unsigned* box,
                           int64_t box_cap, cudaGraphConditionalHandle cond, int use_cond, cudaStream_t stream) {
    TriggerArgs t;
    t.Ss = w.Ss; t.Xb = v.Xb; t.keys = w.keys_sorted; t.gp = w.gp; t.n = n; t.box = box; t.cap = box_cap;
    t.skin = v.skin; t.cutoff = v.cutoff; t.skin_ctl = v.skin_ctl;
    t.flags = v.flags; t.cond = cond; t.use_cond = use_cond;
    if (n > 0) k_verlet_trigger<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(t);
    k_verlet_trigger_check<<<kTrigCheckCtas, 256, 0, stream>>>(t);
}

namespace {
template <bool EPI>
void sweep(const SysConst& sc, const double4* Ss, const int* list, const long long* ofs, const int* len,
           const unsigned* perm, int64_t n, int64_t ncl, int tpl, double4* part, int64_t row0, DevStatus* st,
           unsigned long long event, const double* tbl_dev, unsigned long long* accepted, const int* cfirst,
           int64_t n_ev, const VerletEpi& e, cudaStream_t stream) {
    if (ncl <= 0) return;
    const double rc2 = sc.cutoff * sc.cutoff;
    long long rc2b;
    memcpy(&rc2b, &rc2, sizeof(rc2b));
    const unsigned blocks = (unsigned)((ncl * tpl + kVB - 1) / kVB);
#define GS_V_LAUNCH(F, T)                                                                                  \
    if (accepted)                                                                                          \
        k_verlet_pair<F, T, true, EPI><<<blocks, kVB, 0, stream>>>(Ss, list, ofs, len, perm, n, 0, ncl, sc.k1, rc2b,   \
                                                              part, row0, st, event, tbl_dev, accepted, cfirst, n_ev, e); \
    else                                                                                                   \
        k_verlet_pair<F, T, false, EPI><<<blocks, kVB, 0, stream>>>(Ss, list, ofs, len, perm, n, 0, ncl, sc.k1, rc2b,  \
                                                               part, row0, st, event, tbl_dev, accepted, cfirst, n_ev, e)
#define GS_V_FAM(F)                           \
    switch (tpl) {                            \
        case 1: GS_V_LAUNCH(F, 1); break;     \
        case 2: GS_V_LAUNCH(F, 2); break;     \
        case 4: GS_V_LAUNCH(F, 4); break;     \
        case 8: GS_V_LAUNCH(F, 8); break;     \
        default: GS_V_LAUNCH(F, 16); break;   \
    }
    if (sc.fam == kFamConical) { GS_V_FAM(kFamConical) }
    else { GS_V_FAM(kFamGaussian) }
#undef GS_V_FAM
#undef GS_V_LAUNCH
}
}  // namespace

void launch_verlet_pair(const SysConst& sc, const CellWs& w, const VerletWs& v, int64_t n, double4* part,
                        DevStatus* st, unsigned long long event, const double* tbl_dev, unsigned long long* accepted,
                        cudaStream_t stream) {
    sweep<false>(sc, w.Ss, v.list, v.ofs, v.len, w.perm, n, verlet_clusters(n), v.tpl, part, 0, st, event, tbl_dev,
                 accepted, nullptr, n, VerletEpi{}, stream);
}

void launch_verlet_pair_epi(const SysConst& sc, const CellWs& w, const VerletWs& v, int64_t n, const VerletEpi& e,
                            DevStatus* st, unsigned long long event, const double* tbl_dev, unsigned long long* accepted,
                            cudaStream_t stream) {
    sweep<true>(sc, w.Ss, v.list, v.ofs, v.len, w.perm, n, verlet_clusters(n), v.tpl, nullptr, 0, st, event, tbl_dev,
                accepted, nullptr, n, e, stream);
}

// ---- slab decomposition (gs_slab.cu) ---------------------------------------------------------
// The same list build and sweep over a rank's local particles (its own cell rows + the halo rows,
// in global sorted order), clusters given by cfirst (they restart at every cell row, so a rank
// forms exactly the clusters of the one-rank build), output in the rank's own sorted order.

int slab_list_caps(const SlabLists& L, int64_t n_loc, int64_t ncl, int tpl, cudaStream_t stream) {
    if (ncl > 0)
        k_verlet_caps<<<(unsigned)((ncl + 255) / 256), 256, 0, stream>>>(L.Sf, L.S, L.start, L.gp, n_loc, ncl,
                                                                         2 * tpl, L.cnt, L.cfirst);
    size_t bytes = L.scan_bytes;
    const cudaError_t e = cub::DeviceScan::ExclusiveSum(L.scan_temp, bytes, L.cnt, L.ofs, (int)(ncl + 1), stream);
    return (int)e;
}

void slab_list_fill(const SlabLists& L, int64_t n_loc, int64_t ncl, int tpl, int64_t own_begin, cudaStream_t stream) {
    launch_fill(L.Sf, L.S, L.start, L.gp, n_loc, ncl, 2 * tpl, L.ofs, L.len, L.list, L.cap, L.Xb, nullptr, nullptr,
                L.overflow, L.cfirst, own_begin, stream);
}

void slab_sweep(const SysConst& sc, const SlabLists& L, const unsigned* gidx, int64_t n_loc, int64_t ncl, int tpl,
                int64_t own_begin, int64_t n_glob, double4* part, DevStatus* st, unsigned long long event,
                const double* tbl_dev, unsigned long long* accepted, cudaStream_t stream) {
    sweep<false>(sc, L.S, L.list, L.ofs, L.len, gidx, n_loc, ncl, tpl, part, own_begin, st, event, tbl_dev, accepted,
                 L.cfirst, n_glob, VerletEpi{}, stream);
}

void slab_sweep_epi(const SysConst& sc, const SlabLists& L, const unsigned* gidx, int64_t n_loc, int64_t ncl, int tpl,
                    int64_t n_glob, const VerletEpi& e, DevStatus* st, unsigned long long event, const double* tbl_dev,
                    cudaStream_t stream) {
    sweep<true>(sc, L.S, L.list, L.ofs, L.len, gidx, n_loc, ncl, tpl, nullptr, 0, st, event, tbl_dev, nullptr,
                L.cfirst, n_glob, e, stream);
}

}  // namespace gsb

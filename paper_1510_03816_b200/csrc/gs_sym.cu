// gs_sym.cu — symmetric all-pairs fp64 RHS (single rank, all rows).
//
// The pair term is symmetric in (i, j): G_ij = G_ji, c_ij = (p_i.p_j) G'(d)/d = c_ji and
// q_j - q_i = -(q_i - q_j) (particles.py:100-116).  Each unordered pair is therefore
// evaluated once and feeds both rows — ~15 DP-pipe slots per ordered pair instead of the
// ~27 of the one-sided kernel (gs_dense.cu) and the 45 of the libm formulation.
//
// Work decomposition.  Rows are cut in blocks of 128 (nb blocks) and blocks in superblocks
// of G (nsb = ceil(nb/G) ~ 128, so there are ~8k CTAs at any N).  One CTA (4 warps) owns a
// superblock pair (SI <= SJ) and walks its 128 x 128 tiles (I in SI, J in SJ, I <= J):
//   * warp w owns target sub-block w of I (32 targets: positions, momenta and the I-side
//     accumulators in registers) and visits the 4 source sub-blocks of J in phases
//     k = 0..3 (sub-block (w + k) & 3, so no two warps of a phase share a source);
//   * inside a phase lane l pairs its target with source (l + t) & 31 at step t, read from
//     a doubled copy of the sub-block (64 records) so that the rotated index is a constant
//     offset; the source's accumulators travel with it around the warp (one shuffle from
//     lane l+1 per step), so after 32 steps lane l holds the complete contribution of the
//     warp's 32 targets to source l and adds it to the CTA's shared accumulator of block J;
//   * diagonal tiles (I == J) are evaluated one-sided.
// d == 0 pairs (self, coincident particles) come out as exact zeros of the lean pair core
// (gs_device.cuh); the conical G(0) = 1 self term is added per row and the rare coincident
// pairs are re-scanned (inert: G(0) p terms, interacting: the reference's error).
// Partials: the I-side of block I over superblock SJ goes to slot SJ, the J-side of block J
// over superblock SI goes to slot SI (in a diagonal superblock both land in one shared
// accumulator, slot SI).  Every row thus receives exactly nsb partials,
// part[slot * pstride + row], summed in slot order by k_finish — deterministic.
#include "gs_kernels.cuh"

namespace gsb {

namespace {

constexpr unsigned kFull = 0xffffffffu;

template <int FAM>
__global__ void __launch_bounds__(kDB, 6) k_dense_sym(const double4* __restrict__ S, int64_t n, int nb, int G,
                                                      int nsb, double k1, double4* __restrict__ part, int64_t pstride,
                                                      DevStatus* st, unsigned long long event,
                                                      const double* __restrict__ tbl_g) {
    __shared__ double s_tbl[kTbl];
    __shared__ double4 s_src[kDB];       // block J in order
    __shared__ double4 s_rot[4][64];     // sub-block b twice: s_rot[b][k] = s_src[32 b + (k & 31)]
    extern __shared__ double4 s_acc[];   // G * kDB records
    if (*((volatile unsigned long long*)&st->first_event) < event) return;
    for (int t = threadIdx.x; t < kTbl; t += kDB) s_tbl[t] = tbl_g[t];

    // CTA -> superblock pair (SI, SJ), SI <= SJ, row-major over the upper triangle
    const long long t = blockIdx.x;
    const double b2 = 2.0 * nsb + 1.0;
    long long SI = (long long)floor((b2 - sqrt(b2 * b2 - 8.0 * (double)t)) * 0.5);
    auto row_start = [nsb](long long r) { return r * nsb - r * (r - 1) / 2; };
    while (SI > 0 && row_start(SI) > t) --SI;
    while (row_start(SI + 1) <= t) ++SI;
    const long long SJ = SI + (t - row_start(SI));
    const bool diag = SI == SJ;

    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const double4 zero = make_double4(0.0, 0.0, 0.0, 0.0);
    for (int k = threadIdx.x; k < G * kDB; k += kDB) s_acc[k] = zero;

    for (int ib = 0; ib < G; ++ib) {
        const long long I = SI * G + ib;
        if (I >= nb) break;
        const int64_t i = I * kDB + threadIdx.x;
        const double4 me = (i < n) ? S[i] : far_record(threadIdx.x);
        double aqx = 0.0, aqy = 0.0, apx = 0.0, apy = 0.0;
        for (int jb = diag ? ib : 0; jb < G; ++jb) {
            const long long J = SJ * G + jb;
            if (J >= nb) break;
            const int64_t js = J * kDB + threadIdx.x;
            __syncthreads();  // previous tile done with s_src / s_rot / s_acc
            const double4 rec = (js < n) ? S[js] : far_record(threadIdx.x + kDB);
            s_src[threadIdx.x] = rec;
            s_rot[w][lane] = rec;
            s_rot[w][lane + 32] = rec;
            __syncthreads();
            int nz = 0;
            if (I == J) {
#pragma unroll 4
                for (int jj = 0; jj < kDB; ++jj) {
                    const double4 s = s_src[jj];
                    const double dx = me.x - s.x, dy = me.y - s.y;
                    const double pdot = fma(me.z, s.z, me.w * s.w);
                    double g, c;
                    int z;
                    pair_core<FAM>(dx, dy, pdot, s_tbl, k1, g, c, z);
                    aqx = fma(g, s.z, aqx);
                    aqy = fma(g, s.w, aqy);
                    apx = fma(c, dx, apx);
                    apy = fma(c, dy, apy);
                    nz += z;
                }
                if (nz > 1 && i < n) record_coincident(S, n, i, me, J * kDB, J * kDB + kDB, st, event);
                continue;
            }
            double4* jacc = s_acc + jb * kDB;
            for (int ph = 0; ph < 4; ++ph) {
                const int b = (w + ph) & 3;
                const double4* rot = &s_rot[b][lane];
                double jqx = 0.0, jqy = 0.0, jpx = 0.0, jpy = 0.0;
#pragma unroll 8
                for (int step = 0; step < 32; ++step) {
                    const double4 s = rot[step];
                    const double dx = me.x - s.x, dy = me.y - s.y;
                    const double pdot = fma(me.z, s.z, me.w * s.w);
                    double g, c;
                    int z;
                    pair_core<FAM>(dx, dy, pdot, s_tbl, k1, g, c, z);
                    aqx = fma(g, s.z, aqx);
                    aqy = fma(g, s.w, aqy);
                    apx = fma(c, dx, apx);
                    apy = fma(c, dy, apy);
                    jqx = fma(g, me.z, jqx);
                    jqy = fma(g, me.w, jqy);
                    jpx = fma(-c, dx, jpx);
                    jpy = fma(-c, dy, jpy);
                    nz += z;
                    const int src = (lane + 1) & 31;
                    jqx = __shfl_sync(kFull, jqx, src);
                    jqy = __shfl_sync(kFull, jqy, src);
                    jpx = __shfl_sync(kFull, jpx, src);
                    jpy = __shfl_sync(kFull, jpy, src);
                }
                double4 a = jacc[b * 32 + lane];
                a.x += jqx; a.y += jqy; a.z += jpx; a.w += jpy;
                jacc[b * 32 + lane] = a;
                __syncthreads();
            }
            if (nz > 0 && i < n) record_coincident(S, n, i, me, J * kDB, J * kDB + kDB, st, event);  // rare
        }
        if (diag) {
            // row threadIdx.x of block ib: its J-side contributions (tiles (I' < I, I)) are
            // already in s_acc[ib]; later tiles of this CTA never touch s_acc[ib] again
            __syncthreads();
            double4 a = s_acc[ib * kDB + threadIdx.x];
            a.x += aqx; a.y += aqy; a.z += apx; a.w += apy;
            s_acc[ib * kDB + threadIdx.x] = a;
        } else if (i < n) {
            part[SJ * pstride + i] = make_double4(aqx, aqy, apx, apy);
        }
    }
    __syncthreads();
    for (int jb = 0; jb < G; ++jb) {
        const long long J = SJ * G + jb;
        if (J >= nb) break;
        const int64_t js = J * kDB + threadIdx.x;
        if (js < n) part[SI * pstride + js] = s_acc[jb * kDB + threadIdx.x];
    }
}

}  // namespace

SymPlan sym_plan(int64_t n) {
    SymPlan p;
    p.nb = (int)((n + kDB - 1) / kDB);
    p.G = 1;
    while ((p.nb + p.G - 1) / p.G > 128 && p.G < kSymMaxG) p.G *= 2;
    p.nsb = (p.nb + p.G - 1) / p.G;
    p.pstride = (int64_t)p.nb * kDB;
    p.ok = p.nsb <= 256;
    return p;
}

void launch_dense_sym(const SysConst& sc, const double4* S, int64_t n, double4* part, int64_t pstride, DevStatus* st,
                      unsigned long long event, const double* tbl_dev, cudaStream_t stream) {
    const SymPlan p = sym_plan(n);
    const unsigned ctas = (unsigned)((long long)p.nsb * (p.nsb + 1) / 2);
    const size_t smem = (size_t)p.G * kDB * sizeof(double4);
    if (sc.fam == kFamConical)
        k_dense_sym<kFamConical><<<ctas, kDB, smem, stream>>>(S, n, p.nb, p.G, p.nsb, sc.k1, part, pstride, st, event,
                                                              tbl_dev);
    else
        k_dense_sym<kFamGaussian><<<ctas, kDB, smem, stream>>>(S, n, p.nb, p.G, p.nsb, sc.k1, part, pstride, st,
                                                               event, tbl_dev);
}

}  // namespace gsb

// gs_device.cuh — fp64 pair-interaction math shared by every kernel of the B200 path.
//
// One ordered pair (i <- j) of the Euler–Poincaré RHS (particles.py:79-117):
//   dq_i += G(d_ij) p_j
//   dp_i += (p_i . p_j) (-G'(d_ij) / d_ij) (q_i - q_j)          (j != i, d_ij > 0)
// accumulated in "raw" units; the per-row epilogue applies
//   conical  G = exp(-r/alpha):        dq *= peak,  dp *= peak/alpha   (G'/r = -G/(alpha r))
//   gaussian G = exp(-r^2/(2alpha^2)): dq *= peak,  dp *= peak/alpha^2 (G'/r = -G/alpha^2)
// with peak = 1 (normalized) or 1/(2 pi alpha^2) (kernels.py:83-88, 129-136, 158-165).
//
// The reference evaluates exp twice per pair (kernel_value and kernel_derivative) and a
// sqrt and a divide (kernels.py:130, 159; particles.py:100).  Here one pair costs one
// MUFU.RSQ64H + one cubic refinement (r and 1/r), and ONE table-driven exp:
//   2^(y/T) = T[k & (T-1)] * 2^(k / T) * e^(u ln2/T),  k = rint(y), u = y - k in [-1/2, 1/2]
// with a 2^kTblBits-entry table in shared memory (replicated for conflict-free lookups) and a
// polynomial for e^x - 1 on |x| <= ln2/2^(kTblBits+1): 64 entries with the degree-5 Taylor
// polynomial (truncation 3.5e-17), or 128 entries with a degree-4 minimax polynomial (error
// 7.6e-17, one FP64 instruction less per pair; GS_EXP_TBL_BITS).  The exp is ~8-9 FP64-pipe
// instructions plus integer work; results agree with libm to a few ulp (tests/test_gpu_parity.py).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

// Checked builds (-DGS_CHECKED, tools/checked_build.sh): device-side bounds and protocol asserts in
// every kernel family.  compute-sanitizer is not available on the GPU pool this was built on, so
// the checked library running the whole GPU test suite is the memory-safety evidence.
#ifdef GS_CHECKED
#include <cstdio>
#define GS_ASSERT(c)                                                                   \
    do {                                                                               \
        if (!(c)) {                                                                    \
            printf("GS_ASSERT failed %s:%d: %s\n", __FILE__, __LINE__, #c);           \
            __trap();                                                                  \
        }                                                                              \
    } while (0)
#else
#define GS_ASSERT(c) \
    do {             \
    } while (0)
#endif

namespace gsb {

constexpr int kFamConical = 0;
constexpr int kFamGaussian = 1;

#ifndef GS_EXP_TBL_BITS   // table entries 2^bits: 6 (degree-5 Taylor) or 7 (degree-4 minimax; A/B: C2 dense solve
                          // 137.2 -> 134.8 ms, C2 cell solve 11.68 -> 11.37, C4 / C5 list RHS 1.685 / 1.222 -> 1.663 / 1.201)
#define GS_EXP_TBL_BITS 7
#endif
constexpr int kTblBits = GS_EXP_TBL_BITS;
static_assert(kTblBits == 6 || kTblBits == 7, "exp table: 64 or 128 entries");
constexpr int kTbl = 1 << kTblBits;
// The table is stored 16 times interleaved (entry j of copy c at [16 j + c]) and lane l reads
// copy l & 15: a warp's random lookups hit 16 distinct bank pairs per half-warp, i.e. the
// minimum 2 shared-memory wavefronts instead of ~5 for a single copy.
constexpr int kTblRep = 16;
constexpr int kTblWords = kTbl * kTblRep;
constexpr double kLn2 = 0.69314718055994530941723212145818;
// e1(u) = e^(u ln2 / kTbl) - 1 = u (C1 + u (C2 + u (C3 + u (C4 [+ u C5])))) on |u| <= 1/2
#if GS_EXP_TBL_BITS == 6   // Taylor, degree 5
constexpr int kExpDeg = 5;
constexpr double kC1 = kLn2 / kTbl;
constexpr double kC2 = kC1 * kC1 / 2.0;
constexpr double kC3 = kC1 * kC1 * kC1 / 6.0;
constexpr double kC4 = kC1 * kC1 * kC1 * kC1 / 24.0;
constexpr double kC5 = kC1 * kC1 * kC1 * kC1 * kC1 / 120.0;
#else                      // minimax (Remez in 60-digit arithmetic, tools/exp_minimax.py), degree 4
constexpr int kExpDeg = 4;
constexpr double kC1 = 0.005415212348123815;
constexpr double kC2 = 1.4662262387640288e-05;
constexpr double kC3 = 2.6466433568944648e-08;
#ifndef GS_EXP_C4_IMM
#define GS_EXP_C4_IMM 1
#endif
#if GS_EXP_C4_IMM
// C4 rounded to a double whose low word is zero (0x3DC3B2AC00000000, relative change 2.5e-7: 5.7e-19
// on e^x): the first Horner step fma(C4, u, C3) then carries C4 as a 32-bit immediate and C3 in one
// register — two fresh 64-bit register operands.  With both constants in registers (what ptxas makes
// of two constant-bank operands in one instruction) the DFMA reads three and holds the FP64 pipe's
// issue ~3.2 cycles instead of 2 (tools/issue_probe2.cu).
constexpr double kC4 = 3.583033869603014e-11;
#else
constexpr double kC4 = 3.583032962059034e-11;
#endif
constexpr double kC5 = 0.0;
#endif
constexpr double kRoundMagic = 6755399441055744.0;  // 1.5 * 2^52
constexpr int kKMin = -1020 * kTbl;                 // below: G underflows (flush to 0)

constexpr uint64_t kNoEvent = ~0ull;

// Device-side failure record.  `first_event` = step*8 + ev, ev in 0..7:
//   ev = 2s   coincident interacting pair in the RHS of stage s   (particles.py:92-98)
//   ev = 2s+1 non-finite input of stage s+1 (s < 3)               (integrator.py:106-112)
//   ev = 7    non-finite state after the step                     (integrator.py:58-63)
// Kernels of one launch share one event id and launches are stream-ordered, so the
// first failure wins without a race; `pair_key` = i*n + j of the row-major-first pair.
struct DevStatus {
    unsigned long long first_event;
    unsigned long long pair_key;
};

// Constants of the pair core in the constant bank: FP64 instructions take them as c[][] operands
// instead of re-materialising 64-bit literals into (uniform) registers inside the hot loops
// (k_cell_pair's body: 123 -> 115 instructions per two pairs; results bitwise unchanged).
enum { kCbC1, kCbC2, kCbC3, kCbC4, kCbC5, kCb0375, kCbMagicK, kCbTinyR2, kCbN };
static __constant__ double gs_cb[kCbN] = {kC1, kC2, kC3, kC4, kC5, 0.375, 6755399441055744.0 + 1073741824.0, 1e-200};

__device__ __forceinline__ double rsqrt_refined(double x) {
    double y0;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(x));
    // cubic correction: y = y0 (1 + e/2 + 3e^2/8), e = 1 - x y0^2
    double h = x * y0;
    double e = fma(-h, y0, 1.0);
    double t = fma(e, gs_cb[kCb0375], 0.5);
    double ye = y0 * e;
    return fma(ye, t, y0);
}

// 2^(y / kTbl) for y = x k <= 0 (x = r, k = -kTbl/(alpha ln2)); 0 below 2^-1020.
// Rounding trick with a biased magic 1.5*2^52 + 2^30: for y in [-2^30, 0] the high word of
// s = y + magic is exactly kMagicHi and its low word is rint(y) + 2^30, so one integer
// compare on each word rejects both the underflow range and far-away pairs (|y| > 2^30,
// where the low word would wrap) without an extra FP64 instruction.
constexpr double kRoundMagicK = 6755399441055744.0 + 1073741824.0;
constexpr int kMagicHi = 0x43380000;
// The integer side is written for the fewest instructions: `tb` is the
// 32-bit shared-memory byte address of this lane's table copy (lane_table_addr), so a lookup is
// one AND + one shift-add; the range test is two compares on the words of s; the exponent goes
// into the table value's high word as ((lo(s) >> kTblBits) << 20) (lo(s) = k + 2^30 and 2^30 / kTbl << 20
// vanishes mod 2^32).  (Zeroing only the high word on the out-of-range side was tried: for the
// far padding records u = y - kd is huge and the polynomial overflows to inf, inf * 0 = NaN.)
constexpr unsigned kLoMin = (1u << 30) + (unsigned)kKMin;  // lo(s) >= kLoMin <=> k >= kKMin
// The argument is y = x k, never rounded on its own: the exact product enters the magic-constant
// rounding and the reduced argument u = x k - rint(x k) through fused multiply-adds (what nvcc's
// contraction made of the y + M / y - kd form anyway; written out so the rounding is explicit).
template <bool SELECT>
__device__ __forceinline__ double exp2_tbl_core(double x, double k, unsigned tb) {
    const double s = fma(x, k, gs_cb[kCbMagicK]);
    const double kd = s - gs_cb[kCbMagicK];
    const double u = fma(x, k, -kd);
    const unsigned lo = (unsigned)__double2loint(s), hi = (unsigned)__double2hiint(s);
    // the integer side in PTX, so that ptxas keeps the two-instruction forms: table address
    // (and + mad), exponent ((lo >> 6) << 20 added to the table value's high word: shr + mad),
    // range test (two chained compares: one predicate)
    unsigned addr, sh;
    asm("{\n\t.reg .b32 x;\n\tand.b32 x, %1, %3;\n\tmad.lo.u32 %0, x, 128, %2;\n\t}"
        : "=r"(addr) : "r"(lo), "r"(tb), "n"(kTbl - 1));
    asm("shr.u32 %0, %1, %2;" : "=r"(sh) : "r"(lo), "n"(kTblBits));
    double t;
    asm("ld.shared.f64 %0, [%1];" : "=d"(t) : "r"(addr));
    unsigned th;
    asm("mad.lo.u32 %0, %1, 1048576, %2;" : "=r"(th) : "r"(sh), "r"((unsigned)__double2hiint(t)));
#if GS_EXP_C4_IMM && GS_EXP_TBL_BITS != 6
    const double p4 = kC4;  // a literal: the immediate form
#else
    const double p4 = kExpDeg == 5 ? fma(gs_cb[kCbC5], u, gs_cb[kCbC4]) : gs_cb[kCbC4];
#endif
    const double e1 = u * fma(fma(fma(p4, u, gs_cb[kCbC3]), u, gs_cb[kCbC2]), u, gs_cb[kCbC1]);
    const double tn = __hiloint2double((int)th, __double2loint(t));
    const double g = fma(tn, e1, tn);
    if (!SELECT) return g;  // the caller keeps x k inside [kKMin + kTbl, 0] (pair_clamp_hi)
    double r;
    asm("{\n\t.reg .pred p;\n\tsetp.ge.u32 p, %1, %2;\n\tsetp.eq.and.u32 p, %3, %4, p;\n\t"
        "selp.f64 %0, %5, 0d0000000000000000, p;\n\t}"
        : "=d"(r) : "r"(lo), "n"(kLoMin), "r"(hi), "n"(kMagicHi), "d"(g));
    return r;
}

__device__ __forceinline__ double exp2_tbl_fast(double x, double k, unsigned tb) {
    return exp2_tbl_core<true>(x, k, tb);
}

// Range handling of the hot pair loops without the select (GS_PAIR_CLAMP): instead of testing the
// rounded exponent argument after the fact (two compares + a 64-bit select = 4 instructions per
// pair), d^2 is clamped from above by ONE integer min on its high word before the rsqrt, at the
// d^2 where G = 2^-1019: every farther pair then evaluates G ~ 2^-1019 (x its momentum: < 1e-300
// absolute, where the reference holds subnormals or 0) instead of exactly 0, the argument stays
// inside the table exp's range, and the far padding records (p = 0) still contribute exact zeros.
// The clamp replaces the high word only: the clamped value lies within 2^-20 below the cap.
// Valid wherever the lean core itself is (d = 0 pairs need cap >> 1e-200: alpha > ~1e-103).
// A/B (session 6): the list sweep gains (44.5 -> 42.5 instructions per pair, C4 / C5 list RHS 1.594 /
// 1.159 -> 1.584 / 1.151 ms, bitwise unchanged: only the sentinel is ever clamped there); the
// symmetric dense kernel loses (47.4 -> 45.4 instructions per pair but 160 -> 168 registers and a
// worse schedule: C2 solve 134.7 -> 137.4 ms), so it keeps the select (GS_PAIR_CLAMP_SYM=0).
#ifndef GS_PAIR_CLAMP
#define GS_PAIR_CLAMP 1
#endif
#ifndef GS_PAIR_CLAMP_SYM
#define GS_PAIR_CLAMP_SYM 0
#endif
__device__ __forceinline__ int pair_clamp_hi(int fam, double k1) {
    const double lim = (1019.0 * kTbl) / fabs(k1);  // d (conical) or d^2 (gaussian) with G = 2^-1019
    const double cap = fam == kFamConical ? lim * lim : lim;
    return min(max(__double2hiint(cap) - 1, 0x00100000), 0x7fefffff);
}
static_assert(kTblRep * 8 == 128, "lane copies interleave in 128-byte rows (exp2_tbl_fast)");

// The exp table into shared memory by one bulk copy (TMA engine, cp.async.bulk): thread 0 arms an
// mbarrier with the table's byte count and issues the copy; the CTA synchronises (the barrier's
// init is then visible) and every thread waits on the barrier before its first lookup.  Replaces
// 16 loads + stores per thread of a 64-thread CTA in the prologue of every tile-pair CTA (7 % of
// k_dense_sym's stall samples sat there at C2).
__device__ __forceinline__ void table_bulk_issue(double* s_tbl, const double* tbl_g, unsigned long long* bar) {
    if (threadIdx.x != 0) return;
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    const unsigned d = (unsigned)__cvta_generic_to_shared(s_tbl);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(kTblWords * 8) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(d), "l"(tbl_g), "r"(kTblWords * 8), "r"(b) : "memory");
}

__device__ __forceinline__ void table_bulk_wait(unsigned long long* bar) {
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    unsigned done = 0;
    while (!done)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done) : "r"(b) : "memory");
}

// The table exp every kernel calls: `tbl` is the lane's copy in shared memory (lane_table); its
// 32-bit shared address is loop-invariant and hoisted out of the hot loops.
__device__ __forceinline__ double exp2_tbl(double x, double k, const double* __restrict__ tbl) {
    return exp2_tbl_fast(x, k, (unsigned)__cvta_generic_to_shared(tbl));
}

// 32-bit shared address of this lane's table copy (exp2_tbl_fast).
__device__ __forceinline__ unsigned lane_table_addr(const double* s_tbl) {
    return (unsigned)__cvta_generic_to_shared(s_tbl + (threadIdx.x & (kTblRep - 1)));
}

// This thread's copy of the replicated table in shared memory.
__device__ __forceinline__ const double* lane_table(const double* s_tbl) {
    return s_tbl + (threadIdx.x & (kTblRep - 1));
}

// ---- lean pair core for the hot loops -------------------------------------------------------
// G and c for one pair with d^2 computed as dx^2 + dy^2 + 1e-200.  The offset changes nothing
// for d > 1e-92 and makes the d == 0 pairs (self, coincident particles) come out exactly right
// without a select: 1/d = 1e100 is finite, G(1e-100) rounds to exactly 1 = G(0), and c * dx =
// c * 0 = 0, as the reference's zeroed diagonal (particles.py:100-105).  `z` flags
// d^2 == 1e-200 (d == 0, or d < 1e-208) on the integer pipe; callers re-scan only when a
// non-self pair was flagged (the reference raises for interacting coincident particles,
// particles.py:92-98), see record_coincident().
constexpr double kTinyR2 = 1e-200;

template <int FAM>
__device__ __forceinline__ void pair_core(double dx, double dy, double pdot, const double* __restrict__ tbl, double k1,
                                          double& g, double& c, int& z) {
    const double r2 = fma(dx, dx, fma(dy, dy, gs_cb[kCbTinyR2]));
    z = ((__double2hiint(r2) ^ __double2hiint(kTinyR2)) | (__double2loint(r2) ^ __double2loint(kTinyR2))) == 0;
    if (FAM == kFamConical) {
        const double rs = rsqrt_refined(r2);
        g = exp2_tbl(r2 * rs, k1, tbl);
        c = (pdot * g) * rs;
    } else {
        g = exp2_tbl(r2, k1, tbl);
        c = pdot * g;
    }
}

// pair_core for the symmetric kernel's off-diagonal tiles (no self pairs there): instead of a
// d == 0 flag per pair it hands back the high word of d^2 (the caller keeps the minimum, one
// integer op per pair); a minimum <= hi(1e-200) means a pair with d^2 within 2^-20 of the offset
// (d < ~1e-103, in practice d == 0) and triggers the exact re-scan.
template <int FAM>
__device__ __forceinline__ void pair_core_hi(double dx, double dy, double pdot, unsigned tb, double k1, int caphi,
                                             double& g, double& c, int& r2hi) {
    double r2 = fma(dx, dx, fma(dy, dy, gs_cb[kCbTinyR2]));
    r2hi = __double2hiint(r2);
#if GS_PAIR_CLAMP_SYM
    r2 = __hiloint2double(min(r2hi, caphi), __double2loint(r2));
    if (FAM == kFamConical) {
        const double rs = rsqrt_refined(r2);
        g = exp2_tbl_core<false>(r2 * rs, k1, tb);
        c = (pdot * g) * rs;
    } else {
        g = exp2_tbl_core<false>(r2, k1, tb);
        c = pdot * g;
    }
    return;
#endif
    if (FAM == kFamConical) {
        const double rs = rsqrt_refined(r2);
        g = exp2_tbl_fast(r2 * rs, k1, tb);
        c = (pdot * g) * rs;
    } else {
        g = exp2_tbl_fast(r2, k1, tb);
        c = pdot * g;
    }
}

// Accumulates one ordered pair.  k1 = -kTbl/(alpha ln2) (conical, multiplies r) or
// -kTbl/(2 alpha^2 ln2) (gaussian, multiplies r^2).  Returns true when d_ij == 0
// (self pair or coincident particles): G(0)=1 enters dq, nothing enters dp, and the
// caller checks the reference's "interacting coincident pair" condition with *pdot_out.
template <int FAM>
__device__ __forceinline__ bool pair_accum(double xi, double yi, double pxi, double pyi, double xj, double yj,
                                           double pxj, double pyj, const double* __restrict__ tbl, double k1,
                                           double& aqx, double& aqy, double& apx, double& apy,
                                           double& pdot_out) {
    double dx = xi - xj;
    double dy = yi - yj;
    double r2 = fma(dx, dx, dy * dy);
    double pdot = fma(pxi, pxj, pyi * pyj);
    bool z = (r2 == 0.0);
    double g, c;
    if (FAM == kFamConical) {
        double r2s = z ? 1.0 : r2;
        double rs = rsqrt_refined(r2s);
        double r = r2s * rs;
        g = exp2_tbl(r, k1, tbl);
        g = z ? 1.0 : g;
        c = (pdot * g) * rs;
    } else {
        g = exp2_tbl(r2, k1, tbl);   // exactly 1 at r2 == 0
        c = pdot * g;
    }
    c = z ? 0.0 : c;
    aqx = fma(g, pxj, aqx);
    aqy = fma(g, pyj, aqy);
    apx = fma(c, dx, apx);
    apy = fma(c, dy, apy);
    pdot_out = pdot;
    return z;
}

// Symmetric variant: one evaluation of G and c serves both ordered pairs (i <- j) and
// (j <- i) (G, c symmetric; q_j - q_i = -(q_i - q_j)).  Same exp/rsqrt path as pair_accum.
template <int FAM>
__device__ __forceinline__ bool pair_sym(double xi, double yi, double pxi, double pyi, double xj, double yj,
                                         double pxj, double pyj, const double* __restrict__ tbl, double k1,
                                         double& aqx, double& aqy, double& apx, double& apy, double& jqx,
                                         double& jqy, double& jpx, double& jpy, double& pdot_out) {
    double dx = xi - xj;
    double dy = yi - yj;
    double r2 = fma(dx, dx, dy * dy);
    double pdot = fma(pxi, pxj, pyi * pyj);
    bool z = (r2 == 0.0);
    double g, c;
    if (FAM == kFamConical) {
        double r2s = z ? 1.0 : r2;
        double rs = rsqrt_refined(r2s);
        double r = r2s * rs;
        g = exp2_tbl(r, k1, tbl);
        g = z ? 1.0 : g;
        c = (pdot * g) * rs;
    } else {
        g = exp2_tbl(r2, k1, tbl);
        c = pdot * g;
    }
    c = z ? 0.0 : c;
    aqx = fma(g, pxj, aqx);
    aqy = fma(g, pyj, aqy);
    apx = fma(c, dx, apx);
    apy = fma(c, dy, apy);
    jqx = fma(g, pxi, jqx);
    jqy = fma(g, pyi, jqy);
    jpx = fma(-c, dx, jpx);
    jpy = fma(-c, dy, jpy);
    pdot_out = pdot;
    return z;
}

__device__ __forceinline__ void record_event(DevStatus* st, unsigned long long event, unsigned long long key);

// Padding record for partial tiles: far away (pairwise distinct, d^2 <= ~1e304) with p = 0, so
// it contributes exactly 0 to every real row and never has d == 0 with anything.
__device__ __forceinline__ double4 far_record(int k) {
    return make_double4(1e150 * (double)(k + 1), 1e150, 0.0, 0.0);
}

// Rare path of the lean loops: row i had a flagged pair other than itself among sources
// [j0, j1) of S.  Records the reference's error for each exactly coincident interacting pair
// (d == 0 and p_i.p_j != 0, particles.py:92-98); the row-major-first pair is kept.
__device__ __noinline__ inline void record_coincident(const double4* __restrict__ S, int64_t n, int64_t i, double4 me,
                                                      int64_t j0, int64_t j1, DevStatus* st,
                                                      unsigned long long event) {
    for (int64_t j = j0; j < j1 && j < n; ++j) {
        if (j == i) continue;
        const double4 s = S[j];
        const double dx = me.x - s.x, dy = me.y - s.y;
        if (__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)) != 0.0) continue;  // the reference's dist == 0
        if (fma(me.z, s.z, me.w * s.w) != 0.0) record_event(st, event, (unsigned long long)(i * n + j));
    }
}

__device__ __forceinline__ bool finite4(double a, double b, double c, double d) {
    return isfinite(a) && isfinite(b) && isfinite(c) && isfinite(d);
}

__device__ __forceinline__ void record_event(DevStatus* st, unsigned long long event, unsigned long long key) {
    atomicMin(&st->pair_key, key);
    atomicMin(&st->first_event, event);
}

}  // namespace gsb

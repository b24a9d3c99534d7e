// gs_small.cu — a whole evolve or a whole feedback match per thread-block cluster (n <= 512).
//
// Config 1 (N = 64) is pure latency: a launch per RHS would cost more than the RHS.  Here
// the reference's complete Algorithm 1 loop (shooting.py:218-301, both update spaces) and its
// RK4 integrator (integrator.py:66-121) execute inside one kernel.  One match runs on a
// cluster of C CTAs (C = 8 by default, C = 1 for tiny n): CTA r owns rows
// [r*R, (r+1)*R), R = ceil(n/C), and keeps the FULL stage state in its own shared memory.
// Per RK stage every CTA evaluates its rows against all n sources (`split` lanes per row
// sharing the source sweep, shuffle-reduced in a fixed butterfly order), computes the next
// stage input of its rows and stores it into the next-stage buffer of every CTA of the
// cluster through distributed shared memory; one cluster barrier per stage publishes it.
// Stage buffers alternate (ping-pong) and the cross-CTA flag / reduction slots alternate by
// barrier parity, so a CTA running one barrier ahead never overwrites what a slower one still
// reads.  Residual norms and H are block reductions combined over the cluster in CTA order,
// so every CTA takes identical decisions.  A batched launch is a grid of such clusters, one
// per item.
#include <cooperative_groups.h>

#include "gs_kernels.cuh"

namespace cg = cooperative_groups;

namespace gsb {

namespace {

constexpr unsigned kFull = 0xffffffffu;
#ifndef GS_SMALL_UNROLL   // source-loop unroll of the small-N RHS (A/B builds)
#define GS_SMALL_UNROLL 4
#endif
constexpr int kSmallUnroll = GS_SMALL_UNROLL;
#ifndef GS_SMALL_MAXSPLIT    // lanes per row at most (A/B builds)
#define GS_SMALL_MAXSPLIT 32
#endif
#ifndef GS_SMALL_RS          // reduce-scatter + all-gather of a row's four sums (A/B: 0 = plain butterfly)
#define GS_SMALL_RS 1
#endif
#ifndef GS_SMALL_ASYNC       // per-stage exchange by st.async + mbarriers (A/B: 0 = cluster barriers)
#define GS_SMALL_ASYNC 1
#endif
#ifndef GS_CLUSTER_PTX_BAR   // explicit aligned cluster barrier instead of cg::this_cluster().sync() (A/B)
#define GS_CLUSTER_PTX_BAR 1
#endif
constexpr int kWarps = kSmallThreads / 32;

// Shared memory of the kernel at file scope, so the helpers address it directly instead of
// through pointers held in registers (the match loop runs at the 128-register limit).
extern __shared__ double4 s_state[];  // [2][n] ping-pong stage buffers, then the velocity workspace
__shared__ double s_tbl[kTblWords];
__shared__ double s_red[kWarps + 1];
__shared__ double s_dslot[2 * kMaxCluster];              // reduction slots, by barrier parity
__shared__ unsigned long long s_kslot[2 * kMaxCluster];  // coincidence keys, by barrier parity
__shared__ int s_bslot[2 * kMaxCluster];                 // non-finite flags, by barrier parity
__shared__ unsigned long long s_key[3];                  // this CTA's rotating coincidence keys
__shared__ SmallItem s_item;                             // this item's constants (read on demand)
__shared__ __align__(8) unsigned long long s_mbar[2];    // per next-stage buffer: DSMEM arrivals

template <int CL>
struct SmallCtx {
    static constexpr int C = CL;  // CTAs of the cluster (compile time: C = 1 folds away all cluster code)
    int rank;              // this CTA's rank in the cluster
    int n, split, tgt, sub;
    bool act;              // this thread's row exists and is owned by this CTA
    int parity;            // slot parity (flips at every cluster barrier that uses slots)
    unsigned ph[2];        // phase parity of s_mbar[0 / 1] (identical in every thread and CTA)
};

__device__ __forceinline__ double nanmax(double a, double b) { return (a > b || a != a) ? a : b; }

template <class Ctx>
__device__ __forceinline__ void cluster_sync(const Ctx& c) {
    if constexpr (Ctx::C > 1) {
#if GS_CLUSTER_PTX_BAR
        // all threads arrive (release: this CTA's DSMEM / shared stores become visible to the
        // cluster) and wait (acquire); the .aligned forms: every thread executes them together
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
#else
        cg::this_cluster().sync();
#endif
    } else {
        __syncthreads();
    }
}

template <class Ctx, typename T>
__device__ __forceinline__ T* remote(const Ctx& c, T* p, int r) {
    if constexpr (Ctx::C > 1) return cg::this_cluster().map_shared_rank(p, r);
    else return p;
}

// ---- DSMEM transfers tracked by mbarriers (the per-stage exchange, C > 1) -----------------
// A stage's records and flags go to every CTA with st.async, each store counted in bytes on
// the receiving CTA's mbarrier of that buffer (complete_tx); a CTA proceeds when its barrier
// has seen all n x 32 + C x 12 bytes — no cluster-wide barrier and none of its GPU-scope
// fences / L1 invalidation per stage.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        unsigned done;
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (done) return;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 5000000000ull) __trap();  // a lost transfer: fail the launch, never hang
    }
}

__device__ __forceinline__ void st_async_rec(uint32_t raddr, const double4& v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];"
                 ::"r"(raddr), "d"(v.x), "d"(v.y), "r"(rbar) : "memory");
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];"
                 ::"r"(raddr + 16), "d"(v.z), "d"(v.w), "r"(rbar) : "memory");
}

__device__ __forceinline__ void st_async_u64(uint32_t raddr, unsigned long long v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];"
                 ::"r"(raddr), "l"(v), "r"(rbar) : "memory");
}

__device__ __forceinline__ void st_async_u32(uint32_t raddr, unsigned v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];"
                 ::"r"(raddr), "r"(v), "r"(rbar) : "memory");
}

// Stores this row's record into buf[tgt] of every CTA of the cluster (the row's lanes share
// the stores).  Visible to all after the next cluster barrier.
template <class Ctx, typename T>
__device__ __forceinline__ void bcast_row(const Ctx& c, T* buf, const T& v) {
    if constexpr (Ctx::C == 1) {
        if (c.act && c.sub == 0) buf[c.tgt] = v;
    } else {
        if (!c.act) return;
        for (int r = c.sub; r < Ctx::C; r += c.split) remote(c, buf, r)[c.tgt] = v;
    }
}

// block-wide reduction of one value per row (lanes with sub != 0 or !act pass identity)
template <class Ctx>
__device__ double block_reduce(const Ctx& c, double v, bool is_max) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int off = 16; off; off >>= 1) {
        double o = __shfl_xor_sync(kFull, v, off);
        v = is_max ? nanmax(v, o) : v + o;
    }
    if (lane == 0) s_red[warp] = v;
    __syncthreads();
    if (warp == 0) {
        const int nw = (blockDim.x + 31) >> 5;
        double w = lane < nw ? s_red[lane] : 0.0;
        for (int off = 16; off; off >>= 1) {
            double o = __shfl_xor_sync(kFull, w, off);
            w = is_max ? nanmax(w, o) : w + o;
        }
        if (lane == 0) s_red[kWarps] = w;
    }
    __syncthreads();
    const double out = s_red[kWarps];
    __syncthreads();
    return out;
}

// block reduction, then the cluster's CTA values combined in rank order (identical everywhere)
template <class Ctx>
__device__ double cluster_reduce(Ctx& c, double v, bool is_max) {
    v = block_reduce(c, v, is_max);
    if constexpr (Ctx::C == 1) return v;
    double* slots = s_dslot + c.parity * kMaxCluster;
    if (threadIdx.x < (unsigned)c.C) remote(c, slots, (int)threadIdx.x)[c.rank] = v;
    cluster_sync(c);
    c.parity ^= 1;
    double acc = slots[0];
    for (int r = 1; r < c.C; ++r) acc = is_max ? nanmax(acc, slots[r]) : acc + slots[r];
    return acc;
}

// shooting.py:124-135: MAX = max_i hypot(r_i), L2 = flat 2-norm
template <class Ctx>
__device__ double cluster_norm(Ctx& c, double rx, double ry, int kind) {
    const bool own = c.act && c.sub == 0;
    if (kind == 0) return cluster_reduce(c, own ? hypot(rx, ry) : 0.0, true);
    return sqrt(cluster_reduce(c, own ? __dadd_rn(__dmul_rn(rx, rx), __dmul_rn(ry, ry)) : 0.0, false));
}

// raw sums of the RHS of this lane's row against S (all lanes of the row get them).  The lean
// pair core (gs_device.cuh) makes d == 0 pairs exact without selects; its z flag (integer pipe)
// sends the rare candidate to the reference's exact coincidence test (particles.py:92-98).
template <int FAM, class Ctx>
__device__ void small_rhs(const Ctx& c, const double4* __restrict__ S, double k1, double4 me,
                          unsigned long long* key, double& sqx, double& sqy, double& spx, double& spy) {
    const double* tbl = lane_table(s_tbl);
    double aqx = 0.0, aqy = 0.0, apx = 0.0, apy = 0.0;
#pragma unroll kSmallUnroll
    for (int j = c.sub; j < c.n; j += c.split) {
        const double4 s = S[j];
        const double dx = me.x - s.x, dy = me.y - s.y;
        const double pdot = fma(me.z, s.z, me.w * s.w);
        double g, cf;
        int z;
        pair_core<FAM>(dx, dy, pdot, tbl, k1, g, cf, z);
        aqx = fma(g, s.z, aqx);
        aqy = fma(g, s.w, aqy);
        apx = fma(cf, dx, apx);
        apy = fma(cf, dy, apy);
        if (z && c.act && j != c.tgt && pdot != 0.0 && __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)) == 0.0)
            atomicMin(key, (unsigned long long)c.tgt * (unsigned long long)c.n + (unsigned long long)j);
    }
#if GS_SMALL_RS
    if (c.split >= 4) {
        // reduce-scatter, then all-gather: the first level swaps two of the four sums, the second
        // one, the rest one each — 12 + 8 shuffles of 32-bit halves instead of 8 per level (the
        // SHFL pipe bounded the plain butterfly at 32 lanes per row).  Fixed order: deterministic.
        const int oa = c.split >> 1, ob = c.split >> 2;
        const bool ha = (c.sub & oa) != 0, hb = (c.sub & ob) != 0;
        const double k0 = ha ? apx : aqx, k1 = ha ? apy : aqy;   // kept: components 2ha, 2ha + 1
        const double s0 = ha ? aqx : apx, s1 = ha ? aqy : apy;
        const double m0 = k0 + __shfl_xor_sync(kFull, s0, oa);
        const double m1 = k1 + __shfl_xor_sync(kFull, s1, oa);
        double m = (hb ? m1 : m0) + __shfl_xor_sync(kFull, hb ? m0 : m1, ob);  // component 2ha + hb
        for (int off = ob >> 1; off; off >>= 1) m += __shfl_xor_sync(kFull, m, off);
        const int base = (threadIdx.x & 31) & ~(c.split - 1), low = c.sub & (ob - 1);
        sqx = __shfl_sync(kFull, m, base | low);
        sqy = __shfl_sync(kFull, m, base | ob | low);
        spx = __shfl_sync(kFull, m, base | oa | low);
        spy = __shfl_sync(kFull, m, base | oa | ob | low);
        return;
    }
#endif
    for (int off = c.split >> 1; off; off >>= 1) {
        aqx += __shfl_xor_sync(kFull, aqx, off);
        aqy += __shfl_xor_sync(kFull, aqy, off);
        apx += __shfl_xor_sync(kFull, apx, off);
        apy += __shfl_xor_sync(kFull, apy, off);
    }
    sqx = aqx; sqy = aqy; spx = apx; spy = apy;
}

template <class Ctx>
__device__ __forceinline__ void store_frame(const Ctx& c, double* frames, int f, const double4& b) {
    if (frames && c.act && c.sub == 0) reinterpret_cast<double4*>(frames)[(int64_t)f * c.n + c.tgt] = b;
}

// Publishes this CTA's rows of (q, p) as S[0] of every CTA (an evolve's initial state).
template <class Ctx>
__device__ __forceinline__ void publish_state(Ctx& c, const double4& b) {
    bcast_row(c, s_state, b);
    cluster_sync(c);
}

// integrator.py:66-121 over the cluster.  Precondition: S[0] holds the initial state of all
// rows (publish_state).  b: in = this thread's initial row, out = its final row.  Returns
// kNoEvent or the failure event (step*8 + ev); *key_out = the row-major-first coincident pair.
template <int FAM, class Ctx>
__device__ unsigned long long small_evolve(Ctx& c, const SysConst& sc, double4& b, int steps, double dt,
                                           int capture_every, double* frames, unsigned long long* key_out) {
    int f = 0;
    if (capture_every > 0) store_frame(c, frames, f++, b);
    // Barriers per stage: one CTA barrier (C = 1), or one CTA + one cluster barrier.  The
    // coincidence key rotates over 3 slots: stage k's slot is read right after stage k's
    // barrier, when stage k - 1's slot (read after the previous barrier) is reset for its next
    // use by stage k + 2.
    int cur = 0, k = 0;
    for (int step = 1; step <= steps; ++step) {
        double4 acc = make_double4(0.0, 0.0, 0.0, 0.0);
        for (int s = 0; s < 4; ++s, ++k) {
            double4* Sc = s_state + (size_t)cur * c.n;
            double4* Sn = s_state + (size_t)(cur ^ 1) * c.n;
            unsigned long long* key = s_key + k % 3;
            const double4 me = c.act ? Sc[c.tgt] : make_double4(0.0, 0.0, 0.0, 0.0);
            double sqx, sqy, spx, spy;
            small_rhs<FAM>(c, Sc, sc.k1, me, key, sqx, sqy, spx, spy);
            double dqx = sqx * sc.scale_q, dqy = sqy * sc.scale_q;
            if (sc.sigma2 != 0.0) {
                dqx = __dadd_rn(dqx, __dmul_rn(sc.sigma2, me.z));
                dqy = __dadd_rn(dqy, __dmul_rn(sc.sigma2, me.w));
            }
            const double dpx = spx * sc.scale_p, dpy = spy * sc.scale_p;
            double4 nxt;
            if (s == 0) {
                acc = make_double4(dqx, dqy, dpx, dpy);
            } else {
                const double w = (s == 3) ? 1.0 : 2.0;
                acc.x = __dadd_rn(acc.x, __dmul_rn(w, dqx));
                acc.y = __dadd_rn(acc.y, __dmul_rn(w, dqy));
                acc.z = __dadd_rn(acc.z, __dmul_rn(w, dpx));
                acc.w = __dadd_rn(acc.w, __dmul_rn(w, dpy));
            }
            if (s < 3) {
                const double cc = (s == 2) ? dt : 0.5 * dt;
                nxt.x = __dadd_rn(b.x, __dmul_rn(cc, dqx));
                nxt.y = __dadd_rn(b.y, __dmul_rn(cc, dqy));
                nxt.z = __dadd_rn(b.z, __dmul_rn(cc, dpx));
                nxt.w = __dadd_rn(b.w, __dmul_rn(cc, dpy));
            } else {
                const double cc = dt / 6.0;
                nxt.x = __dadd_rn(b.x, __dmul_rn(cc, acc.x));
                nxt.y = __dadd_rn(b.y, __dmul_rn(cc, acc.y));
                nxt.z = __dadd_rn(b.z, __dmul_rn(cc, acc.z));
                nxt.w = __dadd_rn(b.w, __dmul_rn(cc, acc.w));
                b = nxt;
            }
            unsigned long long kmin;
            int anybad;
            if constexpr (Ctx::C > 1) {
#if GS_SMALL_ASYNC
                // records and flags to every CTA by st.async, counted on its mbarrier of buffer nb
                const int nb = cur ^ 1;
                unsigned long long* bar = &s_mbar[nb];
                if (threadIdx.x == 0) mbar_expect_tx(bar, (unsigned)(c.n * 32 + Ctx::C * 12));
                GS_ASSERT(!c.act || (c.tgt >= 0 && c.tgt < c.n));
                GS_ASSERT(c.rank >= 0 && c.rank < Ctx::C && nb >= 0 && nb < 2);
                if (c.act)
                    for (int r = c.sub; r < Ctx::C; r += c.split)
                        st_async_rec(mapa_u32(smem_u32(&Sn[c.tgt]), r), nxt, mapa_u32(smem_u32(bar), r));
                const int bad = __syncthreads_or(c.act && !finite4(nxt.x, nxt.y, nxt.z, nxt.w));
                unsigned long long* ks = s_kslot + nb * kMaxCluster;
                int* bs = s_bslot + nb * kMaxCluster;
                if (threadIdx.x < (unsigned)Ctx::C) {
                    const uint32_t rb = mapa_u32(smem_u32(bar), (int)threadIdx.x);
                    st_async_u64(mapa_u32(smem_u32(&ks[c.rank]), (int)threadIdx.x), *key, rb);
                    st_async_u32(mapa_u32(smem_u32(&bs[c.rank]), (int)threadIdx.x), (unsigned)bad, rb);
                }
                mbar_wait(bar, c.ph[nb]);
                c.ph[nb] ^= 1u;
#else
                bcast_row(c, Sn, nxt);
                const int bad = __syncthreads_or(c.act && !finite4(nxt.x, nxt.y, nxt.z, nxt.w));
                unsigned long long* ks = s_kslot + c.parity * kMaxCluster;
                int* bs = s_bslot + c.parity * kMaxCluster;
                if (threadIdx.x < (unsigned)c.C) {
                    remote(c, ks, (int)threadIdx.x)[c.rank] = *key;
                    remote(c, bs, (int)threadIdx.x)[c.rank] = bad;
                }
                cluster_sync(c);
                c.parity ^= 1;
#endif
                kmin = ks[0];
                anybad = bs[0];
                for (int r = 1; r < c.C; ++r) {
                    kmin = ks[r] < kmin ? ks[r] : kmin;
                    anybad |= bs[r];
                }
            } else {
                bcast_row(c, Sn, nxt);
                anybad = __syncthreads_or(c.act && !finite4(nxt.x, nxt.y, nxt.z, nxt.w));
                kmin = *key;
            }
            if (threadIdx.x == 0) s_key[(k + 2) % 3] = kNoEvent;  // stage k - 1's slot, next used by k + 2
            if (kmin != kNoEvent) {
                *key_out = kmin;
                return (unsigned long long)step * 8ull + 2ull * s;
            }
            if (anybad) return (unsigned long long)step * 8ull + 2ull * s + 1ull;
            cur ^= 1;
        }
        if (capture_every > 0 && (step % capture_every == 0 || step == steps)) store_frame(c, frames, f++, b);
    }
    return kNoEvent;
}

// particles.py:120-131 at (q, p): sum_i p_i . (K p)_i over the cluster.  b = this row's (q0, p).
template <int FAM, class Ctx>
__device__ double small_hamiltonian(Ctx& c, const SysConst& sc, double4 b) {
    publish_state(c, b);
    double sqx, sqy, spx, spy;
    small_rhs<FAM>(c, s_state, sc.k1, b, s_key + 2, sqx, sqy, spx, spy);  // coincidences are irrelevant to H
    const double v = __dadd_rn(__dmul_rn(b.z, sqx * sc.scale_q), __dmul_rn(b.w, sqy * sc.scale_q));
    return cluster_reduce(c, (c.act && c.sub == 0) ? v : 0.0, false);
}

// p = K^-1 u with K = L L^T (shooting.py:157-159, cho_solve), solved redundantly by every CTA
// of the cluster (u of all rows is in v): forward substitution L y = u (column-oriented:
// y_j = v_j / L_jj, then v_i -= L_ij y_j for i > j) into v, backward L^T x = y into w.  One
// CTA barrier per column; every thread updates rows of the column.
template <class Ctx>
__device__ void small_chol_solve(const Ctx& c, const double* L, int ld, double2* v, double2* w) {
    const int n = c.n;
    __syncthreads();
    for (int t = threadIdx.x; t < n; t += blockDim.x) w[t] = v[t];
    __syncthreads();
    for (int j = 0; j < n; ++j) {
        const double2 bj = w[j];
        const double d = L[(int64_t)j * ld + j];
        const double yx = __ddiv_rn(bj.x, d), yy = __ddiv_rn(bj.y, d);
        for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) {
            const double l = L[(int64_t)i * ld + j];
            double2 r = w[i];
            r.x = __dsub_rn(r.x, __dmul_rn(l, yx));
            r.y = __dsub_rn(r.y, __dmul_rn(l, yy));
            w[i] = r;
        }
        if (threadIdx.x == 0) v[j] = make_double2(yx, yy);
        __syncthreads();
    }
    // v = y; backward: x_j = v_j / L_jj, v_i -= L_ji x_j for i < j
    for (int j = n - 1; j >= 0; --j) {
        const double2 bj = v[j];
        const double d = L[(int64_t)j * ld + j];
        const double xx = __ddiv_rn(bj.x, d), xy = __ddiv_rn(bj.y, d);
        for (int i = threadIdx.x; i < j; i += blockDim.x) {
            const double l = L[(int64_t)j * ld + i];
            double2 r = v[i];
            r.x = __dsub_rn(r.x, __dmul_rn(l, xx));
            r.y = __dsub_rn(r.y, __dmul_rn(l, xy));
            v[i] = r;
        }
        if (threadIdx.x == 0) w[j] = make_double2(xx, xy);
        __syncthreads();
    }
}

template <int FAM, int CL>
__global__ void __launch_bounds__(kSmallThreads) k_small(SmallArgs a, const double* __restrict__ tbl_g) {
    for (int t = threadIdx.x; t < kTblWords; t += blockDim.x) s_tbl[t] = tbl_g[t];
    if (threadIdx.x < 3) s_key[threadIdx.x] = kNoEvent;
    if (CL > 1 && threadIdx.x == 0) {  // DSMEM arrival barriers, visible to the cluster after its first sync
        mbar_init(&s_mbar[0]);
        mbar_init(&s_mbar[1]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }

    constexpr int C = CL;
    const int64_t b = blockIdx.x / C;  // the item this cluster runs
    if (threadIdx.x == 0) s_item = a.items ? a.items[b] : a.item;
    __syncthreads();
    const SmallItem& item = s_item;
    const SysConst& sc = item.sc;
    SmallCtx<CL> c;
    c.ph[0] = 0; c.ph[1] = 0; c.rank = (int)(blockIdx.x % C); c.parity = 0;
    c.n = (int)a.n; c.split = a.split;
    const int R = (c.n + C - 1) / C;
    const int tl = threadIdx.x / a.split;
    c.sub = threadIdx.x % a.split;
    c.tgt = c.rank * R + tl;
    c.act = tl < R && c.tgt < c.n;
    const int t = c.act ? c.tgt : 0;
    const double dt = item.t_final / item.steps;
    const int64_t own = b * 2 * a.n;  // this item's (n, 2) slice of the per-item outputs
    const double* q_in = a.q_in + b * a.q_stride;
    cluster_sync(c);  // table loaded; every CTA of the cluster is running (DSMEM targets exist)

    if (a.mode == 0) {  // ------------------------------------------------ evolve
        const double* p_in = a.p_in + own;
        double4 bs = make_double4(q_in[2 * t], q_in[2 * t + 1], p_in[2 * t], p_in[2 * t + 1]);
        publish_state(c, bs);
        unsigned long long key = kNoEvent;
        const unsigned long long ev = small_evolve<FAM>(c, sc, bs, item.steps, dt, a.capture_every, a.frames, &key);
        if (c.act && c.sub == 0) {
            a.q_out[own + 2 * t] = bs.x; a.q_out[own + 2 * t + 1] = bs.y;
            a.p_out[own + 2 * t] = bs.z; a.p_out[own + 2 * t + 1] = bs.w;
        }
        if (c.rank == 0 && threadIdx.x == 0) {
            a.st[b].first_event = ev;
            a.st[b].pair_key = (ev != kNoEvent && (ev & 1ull) == 0) ? key : kNoEvent;
        }
        cluster_sync(c);  // no CTA exits while another may still store into its shared memory
        return;
    }

    // ------------------------------------------------------------------ match
    // velocity workspace after the two state buffers: v, w (n double2 each), then L (smem copy)
    double2* v = reinterpret_cast<double2*>(s_state + 2 * a.n);
    double2* w = v + a.n;
    const double* L = nullptr;
    int ld = (int)a.n;
    if (a.L) {
        L = a.L + b * a.L_stride;
        if (a.L_smem) {
            double* Ls = reinterpret_cast<double*>(w + a.n);
            for (int64_t k = threadIdx.x; k < a.n * a.n; k += blockDim.x)
                Ls[(k / a.n) * (a.n + 1) + k % a.n] = L[k];
            L = Ls;
            ld = (int)a.n + 1;
        }
    }
    const double* target = a.target + b * a.t_stride;
    double* history = a.history + b * a.hist_stride;
    const double qx0 = q_in[2 * t], qy0 = q_in[2 * t + 1];
    const double yx = target[2 * t], yy = target[2 * t + 1];
    double px = 0.0, py = 0.0, ux = 0.0, uy = 0.0;
    double ex = qx0, ey = qy0;  // evolve(q0, 0) is exactly q0 (zero momenta: dq = dp = 0)
    double rx = __dsub_rn(yx, ex), ry = __dsub_rn(yy, ey);
    double nrm = cluster_norm(c, rx, ry, item.norm);
    double initial = nrm;
    bool have_initial = (item.stop_rule == 0);
    int outcome = 1, iters = 0, fail_iter = -1;
    unsigned long long fail_event = kNoEvent, fail_key = kNoEvent;
    if (item.stop_rule == 0 && nrm < item.epsilon) {
        outcome = 0;
    } else {
        for (int it = 0; it < item.max_iter; ++it) {
            const double delta = item.h * nrm;
            if (L) {  // u <- u + h r; p = K^-1 u (shooting.py:263-265)
                ux = __dadd_rn(ux, __dmul_rn(item.h, rx));
                uy = __dadd_rn(uy, __dmul_rn(item.h, ry));
                bcast_row(c, v, make_double2(ux, uy));
                cluster_sync(c);
                small_chol_solve(c, L, ld, v, w);
                const double2 pv = w[t];
                px = pv.x; py = pv.y;
            } else {  // p <- p + h r (shooting.py:266-267)
                px = __dadd_rn(px, __dmul_rn(item.h, rx));
                py = __dadd_rn(py, __dmul_rn(item.h, ry));
            }
            double4 bs = make_double4(qx0, qy0, px, py);
            publish_state(c, bs);
            unsigned long long key = kNoEvent;
            const unsigned long long ev = small_evolve<FAM>(c, sc, bs, item.steps, dt, 0, nullptr, &key);
            if (ev != kNoEvent) {
                outcome = 3; fail_event = ev; fail_iter = it + 1;
                fail_key = ((ev & 1ull) == 0) ? key : kNoEvent;
                break;
            }
            ex = bs.x; ey = bs.y;
            rx = __dsub_rn(yx, ex); ry = __dsub_rn(yy, ey);
            nrm = cluster_norm(c, rx, ry, item.norm);
            double value = (item.stop_rule == 0) ? nrm : delta;
            if (!have_initial) { initial = value; have_initial = true; }
            if (c.rank == 0 && threadIdx.x == 0) history[it] = value;
            iters = it + 1;
            if (!isfinite(value) || (initial > 0.0 && value > 1e6 * initial)) { outcome = 2; break; }
            if (value < item.epsilon) { outcome = 0; break; }
        }
    }
    const double H = small_hamiltonian<FAM>(c, sc, make_double4(qx0, qy0, px, py));
    if (c.act && c.sub == 0) {
        a.p_out[own + 2 * t] = px; a.p_out[own + 2 * t + 1] = py;
        a.q_out[own + 2 * t] = ex; a.q_out[own + 2 * t + 1] = ey;
    }
    if (c.rank == 0 && threadIdx.x == 0) {
        SmallResult r;
        r.hamiltonian = H; r.final_residual = nrm; r.fail_event = fail_event; r.pair_key = fail_key;
        r.outcome = outcome; r.iterations = iters; r.fail_iter = fail_iter; r.pad = 0;
        a.result[b] = r;
    }
    cluster_sync(c);
}

}  // namespace

size_t small_smem_bytes(const SmallArgs& a) {
    size_t bytes = 2 * (size_t)a.n * sizeof(double4);
    if (a.mode == 1 && a.L) {
        bytes += 2 * (size_t)a.n * sizeof(double2);
        if (a.L_smem) bytes += (size_t)a.n * (a.n + 1) * sizeof(double);
    }
    return bytes;
}

int small_threads(int64_t n, int cluster, int* split_out) {
    const int64_t rows = (n + cluster - 1) / cluster;
    int split = 1;
    // lanes per row: a power of two <= 32, no more than the sources (n), within the CTA size
    while (split < GS_SMALL_MAXSPLIT && split * 2 <= n && rows * split * 2 <= kSmallThreads) split *= 2;
    *split_out = split;
    return (int)(((rows * split) + 31) / 32 * 32);
}

static int launch_small_cluster(int fam, const SmallArgs& a, const double* tbl_dev, cudaStream_t stream);

// A cluster launch the device cannot place (shared memory / cluster resources) falls back to
// one CTA per item: same results to rounding, never a failed match.
int launch_small(int fam, const SmallArgs& a, const double* tbl_dev, cudaStream_t stream) {
    int rc = launch_small_cluster(fam, a, tbl_dev, stream);
    if (rc != 0 && a.cluster > 1) {
        (void)cudaGetLastError();
        SmallArgs b = a;
        b.cluster = 1;
        small_threads(b.n, 1, &b.split);
        rc = launch_small_cluster(fam, b, tbl_dev, stream);
    }
    return rc;
}

static int launch_small_cluster(int fam, const SmallArgs& a, const double* tbl_dev, cudaStream_t stream) {
    int split = 0;
    const int threads = small_threads(a.n, a.cluster, &split);
    if (split != a.split) return (int)cudaErrorInvalidValue;
    const size_t smem = small_smem_bytes(a);
    void (*kern)(SmallArgs, const double*) = nullptr;
    const bool con = fam == kFamConical;
    switch (a.cluster) {
        case 1: kern = con ? k_small<kFamConical, 1> : k_small<kFamGaussian, 1>; break;
        case 2: kern = con ? k_small<kFamConical, 2> : k_small<kFamGaussian, 2>; break;
        case 4: kern = con ? k_small<kFamConical, 4> : k_small<kFamGaussian, 4>; break;
        case 8: kern = con ? k_small<kFamConical, 8> : k_small<kFamGaussian, 8>; break;
        default: return (int)cudaErrorInvalidValue;
    }
    // static (exp table, slots) + dynamic above the 48 KB default: opt in for the dynamic part
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, kern) != cudaSuccess) return (int)cudaErrorInvalidValue;
    if (smem + fa.sharedSizeBytes > 48 * 1024) {
        const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return (int)e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(a.batch * a.cluster));
    cfg.blockDim = dim3((unsigned)threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)a.cluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return (int)cudaLaunchKernelEx(&cfg, kern, a, tbl_dev);
}

}  // namespace gsb

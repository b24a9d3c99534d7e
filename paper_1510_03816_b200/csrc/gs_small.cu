// gs_small.cu — one persistent CTA runs a whole evolve or a whole feedback match (n <= 512).
//
// Config 1 (N = 64) is pure latency: a launch per RHS would cost more than the RHS.  Here
// the reference's complete Algorithm 1 loop (shooting.py:218-301, momentum update
// :266-267) and its RK4 integrator (integrator.py:66-121) execute inside one kernel:
// the stage state lives in shared memory, each target row is owned by `split` lanes
// that share its source sweep (shuffle-reduced in a fixed butterfly order, so every
// lane ends with identical bits), and the residual norms are block reductions.  The
// host launches once and reads one result record.
#include "gs_kernels.cuh"

namespace gsb {

namespace {

constexpr unsigned kFull = 0xffffffffu;
#ifndef GS_SMALL_LEAN   // lean pair core + unrolled source loop (A/B builds)
#define GS_SMALL_LEAN 1
#endif
constexpr int kWarps = kSmallThreads / 32;

struct SmallCtx {
    double4* S;            // shared: stage state, n records
    const double* tbl;     // shared: this lane's copy of the exp table
    double* red;           // shared: kWarps scratch
    unsigned long long* key;
    int n, split, tgt, sub;
    bool act;
};

__device__ __forceinline__ double nanmax(double a, double b) { return (a > b || a != a) ? a : b; }

// block-wide reduction of one value per target (lanes with sub != 0 or !act pass identity)
__device__ double block_reduce(const SmallCtx& c, double v, bool is_max) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int off = 16; off; off >>= 1) {
        double o = __shfl_xor_sync(kFull, v, off);
        v = is_max ? nanmax(v, o) : v + o;
    }
    if (lane == 0) c.red[warp] = v;
    __syncthreads();
    if (warp == 0) {
        const int nw = (blockDim.x + 31) >> 5;
        double w = lane < nw ? c.red[lane] : (is_max ? 0.0 : 0.0);
        for (int off = 16; off; off >>= 1) {
            double o = __shfl_xor_sync(kFull, w, off);
            w = is_max ? nanmax(w, o) : w + o;
        }
        if (lane == 0) c.red[kWarps] = w;
    }
    __syncthreads();
    const double out = c.red[kWarps];
    __syncthreads();
    return out;
}

// shooting.py:124-135: MAX = max_i hypot(r_i), L2 = flat 2-norm
__device__ double block_norm(const SmallCtx& c, double rx, double ry, int kind) {
    const bool own = c.act && c.sub == 0;
    if (kind == 0) return block_reduce(c, own ? hypot(rx, ry) : 0.0, true);
    return sqrt(block_reduce(c, own ? __dadd_rn(__dmul_rn(rx, rx), __dmul_rn(ry, ry)) : 0.0, false));
}

// raw sums of the RHS of this lane's target against S (all lanes of the group get them)
template <int FAM>
__device__ void small_rhs(const SmallCtx& c, double k1, double4 me, double& sqx, double& sqy, double& spx,
                          double& spy) {
    double aqx = 0.0, aqy = 0.0, apx = 0.0, apy = 0.0;
#if GS_SMALL_LEAN
    // lean pair core (gs_device.cuh): d == 0 pairs are exact without selects; the z flag
    // (integer pipe) sends the rare candidate to the reference's exact coincidence test
#pragma unroll 4
    for (int j = c.sub; j < c.n; j += c.split) {
        const double4 s = c.S[j];
        const double dx = me.x - s.x, dy = me.y - s.y;
        const double pdot = fma(me.z, s.z, me.w * s.w);
        double g, cf;
        int z;
        pair_core<FAM>(dx, dy, pdot, c.tbl, k1, g, cf, z);
        aqx = fma(g, s.z, aqx);
        aqy = fma(g, s.w, aqy);
        apx = fma(cf, dx, apx);
        apy = fma(cf, dy, apy);
        if (z && c.act && j != c.tgt && pdot != 0.0 && __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)) == 0.0)
            atomicMin(c.key, (unsigned long long)c.tgt * (unsigned long long)c.n + (unsigned long long)j);
    }
#else
    for (int j = c.sub; j < c.n; j += c.split) {
        const double4 s = c.S[j];
        double pdot;
        if (pair_accum<FAM>(me.x, me.y, me.z, me.w, s.x, s.y, s.z, s.w, c.tbl, k1, aqx, aqy, apx, apy, pdot)) {
            if (c.act && j != c.tgt && pdot != 0.0)
                atomicMin(c.key, (unsigned long long)c.tgt * (unsigned long long)c.n + (unsigned long long)j);
        }
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

__device__ __forceinline__ void store_frame(const SmallCtx& c, double* frames, int f, const double4& b) {
    if (frames && c.act && c.sub == 0) reinterpret_cast<double4*>(frames)[(int64_t)f * c.n + c.tgt] = b;
}

// integrator.py:66-121 on the block.  b: in = initial state, out = final state.
// Returns kNoEvent or the failure event (step*8 + ev); *c.key holds the pair on coincidence.
template <int FAM>
__device__ unsigned long long small_evolve(const SmallCtx& c, const SysConst& sc, double4& b, int steps, double dt,
                                           int capture_every, double* frames) {
    if (threadIdx.x == 0) *c.key = kNoEvent;
    if (c.act && c.sub == 0) c.S[c.tgt] = b;
    int f = 0;
    if (capture_every > 0) store_frame(c, frames, f++, b);
    __syncthreads();
    for (int step = 1; step <= steps; ++step) {
        double4 acc = make_double4(0.0, 0.0, 0.0, 0.0);
        for (int s = 0; s < 4; ++s) {
            const double4 me = c.act ? c.S[c.tgt] : make_double4(0.0, 0.0, 0.0, 0.0);
            double sqx, sqy, spx, spy;
            small_rhs<FAM>(c, sc.k1, me, sqx, sqy, spx, spy);
            __syncthreads();
            if (*c.key != kNoEvent) return (unsigned long long)step * 8ull + 2ull * s;
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
            if (c.act && c.sub == 0) c.S[c.tgt] = nxt;
            const bool bad = c.act && !finite4(nxt.x, nxt.y, nxt.z, nxt.w);
            if (__syncthreads_or(bad)) return (unsigned long long)step * 8ull + 2ull * s + 1ull;
        }
        if (capture_every > 0 && (step % capture_every == 0 || step == steps)) store_frame(c, frames, f++, b);
    }
    return kNoEvent;
}

// particles.py:120-131 at (q, p): block sum of p_i . (K p)_i
template <int FAM>
__device__ double small_hamiltonian(const SmallCtx& c, const SysConst& sc, double4 b) {
    if (c.act && c.sub == 0) c.S[c.tgt] = b;
    if (threadIdx.x == 0) *c.key = kNoEvent;
    __syncthreads();
    double sqx, sqy, spx, spy;
    small_rhs<FAM>(c, sc.k1, b, sqx, sqy, spx, spy);
    __syncthreads();
    const double v = __dadd_rn(__dmul_rn(b.z, sqx * sc.scale_q), __dmul_rn(b.w, sqy * sc.scale_q));
    return block_reduce(c, (c.act && c.sub == 0) ? v : 0.0, false);
}

// p = K^-1 u with K = L L^T (shooting.py:157-159, cho_solve): forward substitution L y = u
// (column-oriented: y_j = v_j / L_jj, then v_i -= L_ij y_j for i > j) into w, backward
// L^T x = y into w.  One barrier per column; every thread updates rows of the column.
__device__ void small_chol_solve(const SmallCtx& c, const double* L, int ld, double2* v, double2* w) {
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

template <int FAM>
__global__ void __launch_bounds__(kSmallThreads) k_small(SmallArgs a, const double* __restrict__ tbl_g) {
    extern __shared__ double4 s_state[];
    __shared__ double s_tbl[kTblWords];
    __shared__ double s_red[kWarps + 1];
    __shared__ unsigned long long s_key;
    for (int t = threadIdx.x; t < kTblWords; t += blockDim.x) s_tbl[t] = tbl_g[t];

    const int64_t b = blockIdx.x;
    const SmallItem item = a.items ? a.items[b] : a.item;
    const SysConst& sc = item.sc;
    SmallCtx c;
    c.S = s_state; c.tbl = lane_table(s_tbl); c.red = s_red; c.key = &s_key;
    c.n = (int)a.n; c.split = a.split;
    c.tgt = threadIdx.x / a.split; c.sub = threadIdx.x % a.split;
    c.act = c.tgt < c.n;
    const int t = c.act ? c.tgt : 0;
    const double dt = item.t_final / item.steps;
    const int64_t own = b * 2 * a.n;  // this item's (n, 2) slice of the per-item outputs
    const double* q_in = a.q_in + b * a.q_stride;
    __syncthreads();

    if (a.mode == 0) {  // ------------------------------------------------ evolve
        const double* p_in = a.p_in + own;
        double4 bs = make_double4(q_in[2 * t], q_in[2 * t + 1], p_in[2 * t], p_in[2 * t + 1]);
        const unsigned long long ev = small_evolve<FAM>(c, sc, bs, item.steps, dt, a.capture_every, a.frames);
        if (c.act && c.sub == 0) {
            a.q_out[own + 2 * t] = bs.x; a.q_out[own + 2 * t + 1] = bs.y;
            a.p_out[own + 2 * t] = bs.z; a.p_out[own + 2 * t + 1] = bs.w;
        }
        if (threadIdx.x == 0) {
            a.st[b].first_event = ev;
            a.st[b].pair_key = (ev != kNoEvent && (ev & 1ull) == 0) ? s_key : kNoEvent;
        }
        return;
    }

    // ------------------------------------------------------------------ match
    // velocity workspace after the state records: v, w (n double2 each), then L (smem copy)
    double2* v = reinterpret_cast<double2*>(s_state + a.n);
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
    double nrm = block_norm(c, rx, ry, item.norm);
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
                if (c.act && c.sub == 0) v[c.tgt] = make_double2(ux, uy);
                small_chol_solve(c, L, ld, v, w);
                const double2 pv = w[t];
                px = pv.x; py = pv.y;
            } else {  // p <- p + h r (shooting.py:266-267)
                px = __dadd_rn(px, __dmul_rn(item.h, rx));
                py = __dadd_rn(py, __dmul_rn(item.h, ry));
            }
            double4 bs = make_double4(qx0, qy0, px, py);
            const unsigned long long ev = small_evolve<FAM>(c, sc, bs, item.steps, dt, 0, nullptr);
            if (ev != kNoEvent) {
                outcome = 3; fail_event = ev; fail_iter = it + 1;
                fail_key = ((ev & 1ull) == 0) ? s_key : kNoEvent;
                break;
            }
            ex = bs.x; ey = bs.y;
            rx = __dsub_rn(yx, ex); ry = __dsub_rn(yy, ey);
            nrm = block_norm(c, rx, ry, item.norm);
            double value = (item.stop_rule == 0) ? nrm : delta;
            if (!have_initial) { initial = value; have_initial = true; }
            if (threadIdx.x == 0) history[it] = value;
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
    if (threadIdx.x == 0) {
        SmallResult r;
        r.hamiltonian = H; r.final_residual = nrm; r.fail_event = fail_event; r.pair_key = fail_key;
        r.outcome = outcome; r.iterations = iters; r.fail_iter = fail_iter; r.pad = 0;
        a.result[b] = r;
    }
}

}  // namespace

size_t small_smem_bytes(const SmallArgs& a) {
    size_t bytes = (size_t)a.n * sizeof(double4);
    if (a.mode == 1 && a.L) {
        bytes += 2 * (size_t)a.n * sizeof(double2);
        if (a.L_smem) bytes += (size_t)a.n * (a.n + 1) * sizeof(double);
    }
    return bytes;
}

int launch_small(int fam, const SmallArgs& a, const double* tbl_dev, cudaStream_t stream) {
    const int threads = (int)(((a.n * a.split) + 31) / 32 * 32);
    const size_t smem = small_smem_bytes(a);
    auto kern = fam == kFamConical ? k_small<kFamConical> : k_small<kFamGaussian>;
    if (smem > 48 * 1024) {
        const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return (int)e;
    }
    kern<<<(unsigned)a.batch, threads, smem, stream>>>(a, tbl_dev);
    return (int)cudaGetLastError();
}

}  // namespace gsb

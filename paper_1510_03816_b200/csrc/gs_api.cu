// gs_api.cu — C ABI of libgs_b200.so (include/geoshoot_b200.h): context, RHS, Hamiltonian,
// velocity field, evolve, match, Gram matrix, stage API, profiling.
//
// Host-side orchestration of the device path: argument validation with the reference's
// error contract, workspaces owned by an opaque context (gs_context.cuh), the RK4 stage loop
// (integrator.py:95-119) and the feedback loop (shooting.py:259-301).  The numerics all run in
// the kernels of gs_dense.cu / gs_sym.cu / gs_small.cu / gs_cell.cu; batched trajectories are in
// gs_batch.cu, the multi-GPU peer-memory exchange in gs_p2p.cu.
#include "gs_context.cuh"

using namespace gsb;
using namespace gsapi;

namespace gsapi {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}



int check_system(const gs_system_t* sys) {
    if (!sys) return fail(GS_ERR_INVALID, "system is NULL");
    if (sys->family != GS_FAMILY_CONICAL && sys->family != GS_FAMILY_GAUSSIAN)
        return fail(GS_ERR_UNSUPPORTED, "kernel family not available on the device (conical, gaussian only)");
    if (!(sys->alpha > 0.0) || !std::isfinite(sys->alpha))
        return fail(GS_ERR_INVALID, "alpha must be positive");
    if (!(sys->sigma2 >= 0.0) || !std::isfinite(sys->sigma2))
        return fail(GS_ERR_INVALID, "sigma2 must be nonnegative");
    if (sys->path != GS_PATH_AUTO && sys->path != GS_PATH_DENSE && sys->path != GS_PATH_CELL)
        return fail(GS_ERR_INVALID, "unknown path");
    return GS_OK;
}

SysConst make_const(const gs_system_t* sys) {
    SysConst c;
    c.fam = sys->family;
    const double a = sys->alpha;
    const double peak = sys->normalized ? 1.0 : 1.0 / (2.0 * M_PI * a * a);   // kernels.py:83-88
    if (c.fam == kFamConical) {
        c.k1 = -(double)kTbl / (a * kLn2);
        c.scale_p = peak / a;
    } else {
        c.k1 = -(double)kTbl / (2.0 * a * a * kLn2);
        c.scale_p = peak / (a * a);
    }
    c.scale_q = peak;
    c.sigma2 = sys->sigma2;
    c.cutoff = sys->cutoff;
    return c;
}

// ---- small elementwise kernels -----------------------------------------------------------
__global__ void k_pack(const double* __restrict__ q, const double* __restrict__ p, int64_t n, double4* S,
                       DevStatus* st, int check) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double4 v = make_double4(q[2 * i], q[2 * i + 1], p[2 * i], p[2 * i + 1]);
    S[i] = v;
    if (check && !finite4(v.x, v.y, v.z, v.w)) record_event(st, 0ull, kNoEvent);
}

__global__ void k_copy_rows(const double4* __restrict__ S, int64_t row0, int64_t nrows, double4* B) {
    const int64_t li = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (li < nrows) B[li] = S[row0 + li];
}

__global__ void k_unpack(const double4* __restrict__ B, int64_t nrows, double* q, double* p) {
    const int64_t li = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (li >= nrows) return;
    const double4 v = B[li];
    q[2 * li] = v.x; q[2 * li + 1] = v.y;
    if (p) { p[2 * li] = v.z; p[2 * li + 1] = v.w; }
}

__global__ void k_status_reset(DevStatus* st) {
    st->first_event = kNoEvent;
    st->pair_key = kNoEvent;
}

// match: p <- p + h r (shooting.py:266-267); S = B = (q0, p) (evolve's input copy, integrator.py:81-82)
__global__ void k_match_begin(const double* __restrict__ q0, double* p, const double* __restrict__ resid, double h,
                              int64_t n, double4* S, double4* B) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double px = p[2 * i], py = p[2 * i + 1];
    if (h != 0.0) {
        px = __dadd_rn(px, __dmul_rn(h, resid[2 * i]));
        py = __dadd_rn(py, __dmul_rn(h, resid[2 * i + 1]));
        p[2 * i] = px; p[2 * i + 1] = py;
    }
    const double4 v = make_double4(q0[2 * i], q0[2 * i + 1], px, py);
    S[i] = v;
    B[i] = v;
}

__device__ __forceinline__ double nanmax(double a, double b) { return (a > b || a != a) ? a : b; }

// residual = target - endpoint (shooting.py:277) and per-block partial of the norm
// (shooting.py:124-135).  `src` is either the evolved base state (B, stride 4) or an
// endpoint array (stride 2).  Skipped when the evolve failed (endpoint keeps the last
// finite shoot, shooting.py:271-276).
__global__ void k_residual(const double* __restrict__ src, int stride, const double* __restrict__ tgt, int64_t n,
                           double* endpoint, double* resid, int kind, double* red, DevStatus* st) {
    __shared__ double s[256];
    if (st && *((volatile unsigned long long*)&st->first_event) != kNoEvent) return;
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double ex = src[stride * i], ey = src[stride * i + 1];
        if (endpoint) { endpoint[2 * i] = ex; endpoint[2 * i + 1] = ey; }
        const double rx = __dsub_rn(tgt[2 * i], ex), ry = __dsub_rn(tgt[2 * i + 1], ey);
        resid[2 * i] = rx; resid[2 * i + 1] = ry;
        if (kind == GS_NORM_MAX) acc = nanmax(acc, hypot(rx, ry));
        else acc += __dadd_rn(__dmul_rn(rx, rx), __dmul_rn(ry, ry));
    }
    s[threadIdx.x] = acc;
    __syncthreads();
    for (int w = blockDim.x / 2; w; w >>= 1) {
        if (threadIdx.x < w)
            s[threadIdx.x] = (kind == GS_NORM_MAX) ? nanmax(s[threadIdx.x], s[threadIdx.x + w])
                                                   : s[threadIdx.x] + s[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) red[blockIdx.x] = s[0];
}

// One decision of Algorithm 1 on the device (shooting.py:259-301, as the host loop in gs_match):
// delta = h * |r| from BEFORE the update, value = |Y - X(T)| or delta, blow-up / convergence /
// cap, history; then the WHILE node's condition for the next iteration.
__global__ void k_match_decide(MatchLoop* L, const double* __restrict__ scal, const DevStatus* __restrict__ st,
                               double* hist, double h, double eps, int max_iter, int stop_rule,
                               cudaGraphConditionalHandle cond) {
    MatchLoop m = *L;
    bool stop = false;
    if (st->first_event != kNoEvent) {  // the shoot failed: last finite endpoint, new p (shooting.py:269-276)
        m.outcome = GS_MATCH_EVOLVE_FAILED;
        m.fail_it = m.it + 1;
        stop = true;
    } else {
        const double delta = h * m.nrm;
        const double nrm = scal[0];
        const double value = stop_rule == GS_STOP_TARGET_RESIDUAL ? nrm : delta;
        if (!m.have_initial) { m.initial = value; m.have_initial = 1; }
        hist[m.it] = value;
        m.iters = m.it + 1;
        m.nrm = nrm;
        if (!isfinite(value) || (m.initial > 0.0 && value > 1e6 * m.initial)) { m.outcome = GS_MATCH_BLOWUP; stop = true; }
        else if (value < eps) { m.outcome = GS_MATCH_CONVERGED; stop = true; }
        else if (m.it + 1 >= max_iter) { m.outcome = GS_MATCH_CAP; stop = true; }
        m.it += 1;
    }
    *L = m;
    cudaGraphSetConditional(cond, stop ? 0u : 1u);
}

// deterministic final reduction of `m` partials; kind: 0 max, 1 sum -> sqrt, 2 plain sum
__global__ void k_reduce_final(const double* __restrict__ red, int m, int kind, double* out, DevStatus* st) {
    __shared__ double s[512];
    if (st && *((volatile unsigned long long*)&st->first_event) != kNoEvent) return;
    double acc = 0.0;
    for (int t = threadIdx.x; t < m; t += blockDim.x) acc = (kind == 0) ? nanmax(acc, red[t]) : acc + red[t];
    s[threadIdx.x] = acc;
    __syncthreads();
    for (int w = blockDim.x / 2; w; w >>= 1) {
        if (threadIdx.x < w) s[threadIdx.x] = (kind == 0) ? nanmax(s[threadIdx.x], s[threadIdx.x + w]) : s[threadIdx.x] + s[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = (kind == 1) ? sqrt(s[0]) : s[0];
}

__global__ void k_sum_partial(const double* __restrict__ v, int64_t n, double* red) {
    __shared__ double s[256];
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        acc += v[i];
    s[threadIdx.x] = acc;
    __syncthreads();
    for (int w = blockDim.x / 2; w; w >>= 1) {
        if (threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) red[blockIdx.x] = s[0];
}

__global__ void k_fp64_probe(double* out, int iters) {
    double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-9, a2 = a0 + 2e-9, a3 = a0 + 3e-9;
    double a4 = a0 + 4e-9, a5 = a0 + 5e-9, a6 = a0 + 6e-9, a7 = a0 + 7e-9;
    const double m = 0.999999999, c = 1e-12;
    for (int k = 0; k < iters; ++k) {
        a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
        a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
    }
    const double r = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (r == 12345.678) out[0] = r;  // never true; keeps the chains alive
}


int ensure_session(gs_context* ctx, int64_t n, int64_t nrows) {
    const DensePlan plan = dense_plan(n, ctx->sm_count);
    GS_CUDA(ctx->S.ensure(n + kStatePad));
    GS_CUDA(ctx->B.ensure(nrows));
    GS_CUDA(ctx->A.ensure(nrows));
    GS_CUDA(ctx->part.ensure((size_t)plan.nchunks * nrows));
    return GS_OK;
}

void decode_status(const DevStatus& d, int64_t n, gs_status_t* out) {
    std::memset(out, 0, sizeof(*out));
    out->i = out->j = -1;
    if (d.first_event == kNoEvent) { out->code = GS_OK; return; }
    const unsigned long long step = d.first_event / 8, ev = d.first_event % 8;
    out->step = (int32_t)step;
    out->event = (int32_t)ev;
    if (d.first_event == 0) out->code = GS_ERR_INVALID;
    else if (ev % 2 == 0) {
        out->code = GS_ERR_COINCIDENT;
        out->i = (int64_t)(d.pair_key / (unsigned long long)n);
        out->j = (int64_t)(d.pair_key % (unsigned long long)n);
    } else if (ev == 7) out->code = GS_ERR_NONFINITE_STATE;
    else out->code = GS_ERR_NONFINITE_STAGE;
}

int fetch_status(gs_context* ctx, cudaStream_t s, int64_t n, gs_status_t* out) {
    GS_CUDA(cudaMemcpyAsync(ctx->st_host, ctx->st.ptr, sizeof(DevStatus), cudaMemcpyDeviceToHost, s));
    GS_CUDA(cudaStreamSynchronize(s));
    gs_status_t tmp;
    decode_status(*ctx->st_host, n, &tmp);
    if (out) *out = tmp;
    return tmp.code;
}

cudaEvent_t prof_event(gs_context* ctx) {
    if (ctx->capture_events) {  // recorded as an event node of the graph being captured
        cudaEvent_t e;
        cudaEventCreate(&e);
        ctx->capture_events->push_back(e);
        return e;
    }
    if (ctx->prof_used == ctx->prof_events.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        ctx->prof_events.push_back(e);
    }
    return ctx->prof_events[ctx->prof_used++];
}

// Inside a stream capture the record must be "external" to stay a real, timeable event
// on every graph replay; otherwise it would only be an intra-graph dependency.
void prof_mark(gs_context* ctx, cudaStream_t stream) {
    cudaEvent_t e = prof_event(ctx);
    if (ctx->capture_events) cudaEventRecordWithFlags(e, stream, cudaEventRecordExternal);
    else cudaEventRecord(e, stream);
}

CellWs cell_ws(gs_context* ctx) {
    CellWs w;
    w.keys = ctx->c_keys.ptr; w.keys_sorted = ctx->c_keys_sorted.ptr; w.vals = ctx->c_vals.ptr;
    w.perm = ctx->c_perm.ptr; w.start = ctx->c_start.ptr; w.Ss = ctx->c_Ss.ptr; w.Sf = ctx->c_Sf.ptr; w.bbox_red = ctx->c_bbox.ptr;
    w.gp = ctx->c_gp.ptr; w.cub_temp = ctx->c_cub.ptr; w.cub_bytes = ctx->c_cub_bytes;
    w.tlist = ctx->c_tlist.ptr; w.nsel = ctx->c_nsel.ptr;
    return w;
}

int ensure_cell(gs_context* ctx, int64_t n) {
    GS_CUDA(ctx->c_keys.ensure(n)); GS_CUDA(ctx->c_keys_sorted.ensure(n)); GS_CUDA(ctx->c_vals.ensure(n));
    GS_CUDA(ctx->c_perm.ensure(n)); GS_CUDA(ctx->c_Ss.ensure(n + 1)); GS_CUDA(ctx->c_Sf.ensure(n));
    GS_CUDA(ctx->c_start.ensure(cell_cap(n) + 1));
    GS_CUDA(ctx->c_bbox.ensure(4 * kCellBboxBlocks));
    GS_CUDA(ctx->c_gp.ensure(1));
    GS_CUDA(ctx->c_tlist.ensure(n));
    GS_CUDA(ctx->c_nsel.ensure(1));
    GS_CUDA(ctx->c_acc.ensure(1));
    const size_t bytes = cell_cub_bytes(n);
    GS_CUDA(ctx->c_cub.ensure(bytes));
    ctx->c_cub_bytes = ctx->c_cub.cap;
    return GS_OK;
}

VerletWs verlet_ws(gs_context* ctx, int64_t n, double cutoff) {
    VerletWs v;
    v.cnt = ctx->v_cnt.ptr; v.ofs = ctx->v_ofs.ptr; v.len = ctx->v_len.ptr; v.list = ctx->v_list.ptr;
    v.cap = (int64_t)ctx->v_list.cap;
    v.Xb = ctx->v_xb.ptr; v.inv = ctx->v_inv.ptr; v.flags = ctx->v_flags.ptr; v.overflow = ctx->v_over.ptr;
    v.scan_temp = ctx->v_scan.ptr; v.scan_bytes = ctx->v_scan.cap;
    // skin: small clouds are launch/latency bound, so fewer rebuilds beat fewer masked pairs
    // (C2: 0.05 -> 0.1 saves 1.5 ms per 100-step solve); large ones are FP64 bound (C4/C5: the
    // masked skin pairs cost more than the rebuilds they save) — tools/verlet_ab.py
    v.tpl = verlet_tpl(n);
    v.skin = ctx->verlet_skin >= 0.0 ? ctx->verlet_skin : (n < 131072 ? 0.1 : 0.05);
    v.cutoff = cutoff;
    // the relative-trigger path (no fused epilogue) adapts the skin to the observed rebuild rate
    const bool adapt = ctx->skin_adapt && ctx->verlet_rel && ctx->verlet_skin < 0.0 && n >= ctx->verlet_fuse_max_n;
    v.skin_ctl = adapt && ctx->v_skin.cap >= 2 ? ctx->v_skin.ptr : nullptr;
    v.Ss_pair[0] = ctx->c_Ss.ptr;
    v.Ss_pair[1] = ctx->c_Ss2.cap >= (size_t)(n + 1) ? ctx->c_Ss2.ptr : nullptr;
    return v;
}

// Workspaces of the cluster Verlet lists for n particles; the list buffer is sized from a build
// of the current state S (twice its entries: the lists grow when the cloud contracts; a build
// that still overflows is detected after the call and the call is redone, see verlet_retry).
int ensure_verlet(gs_context* ctx, const double4* S, int64_t n, double cutoff, cudaStream_t s) {
    const int64_t ncl = verlet_clusters(n);
    const bool fresh = ctx->v_flags.cap == 0;
    GS_CUDA(ctx->v_cnt.ensure(ncl + 1)); GS_CUDA(ctx->v_ofs.ensure(ncl + 1)); GS_CUDA(ctx->v_xb.ensure(n));
    GS_CUDA(ctx->v_len.ensure(ncl)); GS_CUDA(ctx->v_inv.ensure(n));
    GS_CUDA(ctx->v_flags.ensure(kVerletFlags)); GS_CUDA(ctx->v_over.ensure(1)); GS_CUDA(ctx->v_skin.ensure(2));
    GS_CUDA(ctx->v_scan.ensure(verlet_scan_bytes(ncl)));
    {
        const size_t box = 4 * (size_t)cell_cap(n);
        if (ctx->v_box.cap < box) {
            GS_CUDA(ctx->v_box.ensure(box));
            verlet_box_reset(ctx->v_box.ptr, (int64_t)(box / 4), s);
        }
    }
    GS_CUDA(ctx->c_Ss2.ensure(n + 1));  // the ping-pong half of the sorted records (fused epilogue);
                                        // every list build writes the sentinel record [n] into both halves
    if (fresh) {
        GS_CUDA(cudaMemsetAsync(ctx->v_flags.ptr, 0, kVerletFlags * sizeof(unsigned), s));
        GS_CUDA(cudaMemsetAsync(ctx->v_over.ptr, 0, sizeof(unsigned long long), s));
    }
    GS_CUDA(cudaMemsetAsync(ctx->v_cnt.ptr + ncl, 0, sizeof(long long), s));
    VerletWs v = verlet_ws(ctx, n, cutoff);
    if (v.skin_ctl) verlet_skin_init(v.skin_ctl, v.skin, s);  // every call starts from the default skin
    if (ctx->v_list.cap > 0 && ctx->v_list_n == n && ctx->v_list_cutoff == cutoff) return GS_OK;
    if (v.skin_ctl) v.skin = std::max(v.skin, kSkinMax);  // size for the largest skin it may adapt to
    v.skin_ctl = nullptr;
    v.cap = 0;  // sizing build: counts and offsets only
    if (int rc = verlet_build(cell_ws(ctx), v, S, n, cutoff, s)) return fail(GS_ERR_CUDA, "verlet sizing build failed");
    long long total = 0;
    GS_CUDA(cudaMemcpyAsync(&total, ctx->v_ofs.ptr + ncl, sizeof(total), cudaMemcpyDeviceToHost, s));
    GS_CUDA(cudaMemsetAsync(ctx->v_over.ptr, 0, sizeof(unsigned long long), s));
    GS_CUDA(cudaStreamSynchronize(s));
    // spare capacity as a fraction of the sizing build: a build that outgrows the buffer makes the
    // whole call (a 100-iteration match: seconds) run again, and lists grow when a deforming cloud
    // packs tighter (C4's late iterations outgrew 1.5x), so room is generous — HBM is plentiful
    const double slack = ctx->verlet_slack;
    const long long want = slack >= 0.5 ? std::max<long long>((long long)((1.0 + slack) * (double)total), total + (1 << 20))
                                        : std::max<long long>(1, (long long)((1.0 + slack) * (double)total));
    ctx->v_list.release();
    GS_CUDA(ctx->v_list.ensure((size_t)want));
    ctx->v_list_n = n;
    ctx->v_list_cutoff = cutoff;
    return GS_OK;
}

// After a multi-RHS call: did a rebuild need more list entries than the buffer holds?  Then the
// buffer grows and the caller redoes the call (*retry).  Synchronises.
int verlet_retry(gs_context* ctx, cudaStream_t s, bool* retry) {
    *retry = false;
    if (!ctx->verlet_call) return GS_OK;
    unsigned long long need = 0;
    GS_CUDA(cudaMemcpyAsync(&need, ctx->v_over.ptr, sizeof(need), cudaMemcpyDeviceToHost, s));
    GS_CUDA(cudaStreamSynchronize(s));
    if (!need) return GS_OK;
    GS_CUDA(cudaMemsetAsync(ctx->v_over.ptr, 0, sizeof(unsigned long long), s));
    if (++ctx->verlet_retries > 3 || need > (1ull << 31)) {
        ctx->verlet_call = 0;  // give up on lists for this context: the per-RHS cell sweep
        ctx->verlet_on = 0;
    } else {
        GS_CUDA(ctx->v_list.ensure((size_t)(need + need / 2)));
    }
    *retry = true;
    return GS_OK;
}

// Pair-sum strategy of one API call (gs_system_t.path).  AUTO takes the cell list when the
// support radius is small against the point cloud of S (one bbox reduction + 8-byte read).
constexpr int64_t kCellMinN = 2048;
constexpr int kCellMinCells = 25;
constexpr double kCellMinDensity = 4.0;  // mean particles per cutoff-sized cell of the bounding box

int choose_path_impl(gs_context* ctx, const gs_system_t* sys, const double4* S, int64_t n, cudaStream_t s) {
    ctx->cell_on = 0;
    if (sys->path == GS_PATH_DENSE) return GS_OK;
    if (sys->path == GS_PATH_CELL && !(sys->cutoff > 0.0))
        return fail(GS_ERR_INVALID, "the cell-list path needs a positive cutoff (support radius)");
    if (!(sys->cutoff > 0.0) || (sys->path == GS_PATH_AUTO && n < kCellMinN)) return GS_OK;
    int rc = ensure_cell(ctx, n);
    if (rc) return rc;
    if (sys->path == GS_PATH_CELL) {
        ctx->cell_on = 1;
        return GS_OK;
    }
    // AUTO: grid size at cell edge = cutoff
    CellWs w = cell_ws(ctx);
    if (cell_build(w, S, n, sys->cutoff, s) != 0) return fail(GS_ERR_CUDA, "cell_build failed");
    GridParams g;
    GS_CUDA(cudaMemcpyAsync(&g, ctx->c_gp.ptr, sizeof(g), cudaMemcpyDeviceToHost, s));
    GS_CUDA(cudaStreamSynchronize(s));
    // cells of edge cutoff: enough of them to pay for the build, and dense enough that a row has
    // in-support neighbours (a row with none keeps only its self term: its dp, < 2^-53 of a
    // neighbour's term in the reference, becomes 0 — fine normwise unless most rows are like that).
    // A cloud already spread over a hashed grid is sparse by construction: dense path.
    const double cells = (double)g.nx * (double)g.ny / ((double)g.sub * (double)g.sub);
    ctx->cell_on = !g.hashed && cells >= (double)kCellMinCells && (double)n >= kCellMinDensity * cells;
    return GS_OK;
}

// Below this N the symmetric kernel's 128 x 128 tiles leave most SMs idle (N = 1024: 36 CTAs)
// and the one-sided kernel with fine source chunks is faster (us per RK stage, one-sided vs
// symmetric: N = 1024 15.7 vs 23.7, 2048 21.6 vs 24.6, 4096 51.2 vs 37.2).
constexpr int64_t kSymMinN = 3072;
// Multi-GPU: the ranks' shares of the symmetric pair list (gs_sym_parts) from this N on.
constexpr int64_t kSymSplitMinN = 1024;

bool use_sym(const gs_context* ctx, int64_t n, int64_t row0, int64_t nrows) {
    return ctx->sym_on && !ctx->cell_on && row0 == 0 && nrows == n && n >= kSymMinN && sym_plan(n).ok;
}

// Path of this call + the partial buffer it needs (allocated here, never inside a capture).
// multi_rhs: the call evaluates many RHS of all rows (evolve, match): the cell path then runs
// through the cluster Verlet lists.
int choose_path(gs_context* ctx, const gs_system_t* sys, const double4* S, int64_t n, cudaStream_t s,
                bool multi_rhs = false) {
    int rc = choose_path_impl(ctx, sys, S, n, s);
    if (rc) return rc;
    ctx->verlet_call = 0;
    if (multi_rhs && ctx->cell_on && ctx->verlet_on && ctx->row0 == 0 && ctx->row1 == n) {
        if ((rc = ensure_verlet(ctx, S, n, sys->cutoff, s))) return rc;
        ctx->verlet_call = 1;
    }
    if (use_sym(ctx, n, ctx->row0, ctx->row1 - ctx->row0)) {
        const SymPlan sp = sym_plan(n);
        GS_CUDA(ctx->part.ensure((size_t)sp.nsb * (size_t)sp.pstride));
    }
    return GS_OK;
}

struct PairOut {
    int nchunks;
    int64_t pstride;
};

// The pair kernel (the hot spot) of every RHS goes through here: timed when profiling is on.
// Returns how the partials are laid out for k_finish: asymmetric dense = plan.nchunks chunk
// partials per row; symmetric dense = nb slot partials per row; cell list = one per row.
PairOut pair_kernel(gs_context* ctx, const SysConst& sc, const double4* S, int64_t n, int64_t row0, int64_t nrows,
                    const DensePlan& plan, double4* part, unsigned long long ev, cudaStream_t stream) {
    PairOut out{plan.nchunks, 0};
    const SymPlan sp = sym_plan(n);
    if (use_sym(ctx, n, row0, nrows) && ctx->part.cap >= (size_t)sp.nsb * (size_t)sp.pstride) {
        out = PairOut{sp.nsb, sp.pstride};
        if (ctx->prof_on) prof_mark(ctx, stream);
        launch_dense_sym(sc, S, n, part, sp.pstride, ctx->st.ptr, ev, ctx->tbl.ptr, stream);
        if (ctx->prof_on) prof_mark(ctx, stream);
        ctx->host_pairs += nrows * n;
    } else if (ctx->cell_on) {
        out = PairOut{1, 0};
        CellWs w = cell_ws(ctx);
        if (const int rc = cell_build(w, S, n, sc.cutoff, stream)) ctx->cell_err = rc;
        ctx->launches += 6;  // bbox, params, keys, 2x radix passes (approx.), start/permute
        if (ctx->prof_on) prof_mark(ctx, stream);
        launch_cell_pair(sc, w, n, row0, row0 + nrows, part, ctx->st.ptr, ev, ctx->tbl.ptr,
                         ctx->prof_on ? ctx->c_acc.ptr : nullptr, stream);
        if (ctx->prof_on) prof_mark(ctx, stream);
    } else {
        if (ctx->prof_on) prof_mark(ctx, stream);
        launch_dense_partial(sc, S, n, row0, nrows, plan, part, ctx->st.ptr, ev, ctx->tbl.ptr, stream);
        if (ctx->prof_on) prof_mark(ctx, stream);
        ctx->host_pairs += nrows * n;
    }
    ctx->launches++;
    ctx->pair_launches++;
    return out;
}

// A cell build that failed to enqueue inside this call (sticky until reported).
int take_cell_err(gs_context* ctx) {
    if (!ctx->cell_err) return GS_OK;
    const int e = ctx->cell_err;
    ctx->cell_err = 0;
    return fail(GS_ERR_CUDA, std::string("cell-list build failed: ") + cudaGetErrorString((cudaError_t)e));
}

// The cluster-list RHS sweep of one stage (gs_verlet.cu).  The lists are rebuilt when the previous
// stage's fused epilogue saw a particle move more than half the skin (captured: a conditional IF
// node on the condition that epilogue set; host-driven: unconditionally, or decided on the host
// with GS_B200_VERLET=3) and always at the first stage of an evolve (`force`).  Then the sweep.
// Returns the cell workspace of the stage (its sorted records: c_Ss or c_Ss2 by `parity`).
CellWs verlet_prepare(gs_context* ctx, const SysConst& sc, int force, cudaStream_t stream, int parity) {
    const int64_t n = ctx->n;
    CellWs w = cell_ws(ctx);
    if (parity) w.Ss = ctx->c_Ss2.ptr;  // the stage's sorted records: ping-pong with the fused epilogue
    VerletWs v = verlet_ws(ctx, n, sc.cutoff);
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(stream, &cs);
    const bool capturing = cs == cudaStreamCaptureStatusActive;
    const bool pending = ctx->v_next_valid != 0;
    ctx->v_next_valid = 0;
    if (capturing && !force && pending) {
        cudaGraph_t g = nullptr;
        const cudaGraphNode_t* deps = nullptr;
        size_t nd = 0;
        cudaGraphNodeParams np = {};
        np.type = cudaGraphNodeTypeConditional;
        np.conditional.handle = ctx->v_next_cond;
        np.conditional.type = cudaGraphCondTypeIf;
        np.conditional.size = 1;
        cudaGraphNode_t node;
        bool ok = cudaStreamGetCaptureInfo(stream, &cs, nullptr, &g, &deps, &nd) == cudaSuccess &&
                  cudaGraphAddNode(&node, g, deps, nd, &np) == cudaSuccess;
        if (ok && !ctx->cap_stream2) ok = cudaStreamCreateWithFlags(&ctx->cap_stream2, cudaStreamNonBlocking) == cudaSuccess;
        if (ok) {
            cudaStream_t s2 = ctx->cap_stream2;
            ok = cudaStreamBeginCaptureToGraph(s2, np.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                               cudaStreamCaptureModeThreadLocal) == cudaSuccess;
            if (ok) {
                if (int rc = verlet_build(w, v, ctx->S.ptr, n, sc.cutoff, s2)) ctx->cell_err = rc;
                cudaGraph_t body = nullptr;
                ok = cudaStreamEndCapture(s2, &body) == cudaSuccess;
            }
            if (ok) ok = cudaStreamUpdateCaptureDependencies(stream, &node, 1, cudaStreamSetCaptureDependencies) ==
                         cudaSuccess;
        }
        if (!ok && !ctx->cell_err) ctx->cell_err = (int)cudaErrorStreamCaptureInvalidated;
        ctx->launches += 10;  // a rebuild, when it runs (approx.)
    } else if (!capturing && ctx->verlet_on == 3 && !force && pending) {
        // profiling aid (GS_B200_VERLET=3): the graph's lazy rebuild decided on the host, so a
        // per-kernel profiler sees the same kernels as a graph replay (one sync per RHS)
        unsigned f = 0;
        cudaMemcpyAsync(&f, v.flags + 3, sizeof(f), cudaMemcpyDeviceToHost, stream);
        cudaStreamSynchronize(stream);
        if (f) {
            if (int rc = verlet_build(w, v, ctx->S.ptr, n, sc.cutoff, stream)) ctx->cell_err = rc;
        }
        ctx->launches += f ? 10 : 0;
    } else {
        if (int rc = verlet_build(w, v, ctx->S.ptr, n, sc.cutoff, stream)) ctx->cell_err = rc;
        ctx->launches += 10;
    }
    return w;
}

// The stage's list sweep with the RK4 stage epilogue fused in.
void verlet_sweep(gs_context* ctx, const SysConst& sc, const CellWs& w, unsigned long long ev, const VerletEpi& epi,
                  cudaStream_t stream) {
    const int64_t n = ctx->n;
    VerletWs v = verlet_ws(ctx, n, sc.cutoff);
    if (ctx->prof_on) prof_mark(ctx, stream);
    launch_verlet_pair_epi(sc, w, v, n, epi, ctx->st.ptr, ev, ctx->tbl.ptr, ctx->prof_on ? ctx->c_acc.ptr : nullptr,
                           stream);
    if (ctx->prof_on) prof_mark(ctx, stream);
    ctx->launches++;
    ctx->pair_launches++;
}

// The fused gather + rebuild trigger of a stage epilogue whose next stage sweeps the lists; inside a
// capture it creates the condition handle of that stage's IF node.
VerletFuse verlet_fuse(gs_context* ctx, const SysConst& sc, cudaStream_t stream) {
    VerletWs v = verlet_ws(ctx, ctx->n, sc.cutoff);
    const double thr = 0.5 * v.skin * sc.cutoff;
    VerletFuse f{ctx->c_Ss.ptr, ctx->v_inv.ptr, ctx->v_xb.ptr, thr * thr * (1.0 - 1e-9), ctx->v_flags.ptr, {}, 0, 0};
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(stream, &cs);
    if (cs == cudaStreamCaptureStatusActive) {
        cudaGraph_t g = nullptr;
        if (cudaStreamGetCaptureInfo(stream, &cs, nullptr, &g, nullptr, nullptr) == cudaSuccess &&
            cudaGraphConditionalHandleCreate(&f.cond, g, 0, cudaGraphCondAssignDefault) == cudaSuccess) {
            f.use_cond = 1;
        } else if (!ctx->cell_err) {
            ctx->cell_err = (int)cudaErrorStreamCaptureInvalidated;
        }
        ctx->v_next_cond = f.cond;
    }
    ctx->v_next_valid = 1;
    return f;
}

// One RK4 stage for the session's rows (pair kernel + finish epilogue).  `last`: no RK stage of
// this call follows (the lists' fused gather is skipped).
void stage(gs_context* ctx, const SysConst& sc, int step, int s, double dt, cudaStream_t stream, bool last = false) {
    const int64_t n = ctx->n, nrows = ctx->row1 - ctx->row0;
    const DensePlan plan = dense_plan(n, ctx->sm_count);
    const unsigned long long ev = (unsigned long long)step * 8ull + 2ull * (unsigned long long)s;
    PairOut po{1, 0};
    const bool lists = ctx->verlet_call && ctx->cell_on && ctx->row0 == 0 && nrows == n;
    FinishArgs fa{};
    fa.part = ctx->part.ptr; fa.nchunks = po.nchunks; fa.pstride = po.pstride; fa.nrows = nrows;
    fa.row0 = ctx->row0;
    fa.S = ctx->S.ptr; fa.B = ctx->B.ptr; fa.A = ctx->A.ptr;
    fa.stage = s; fa.dt = dt; fa.st = ctx->st.ptr; fa.event = ev + 1;
    if (lists && ctx->verlet_fuse_max_n > n) {
        // small clouds (launch/latency bound): the sweep carries the stage epilogue, one kernel per
        // stage plus the conditional rebuild (C2 100-step solve 13.3 -> 12.3 ms); sorted records
        // ping-pong between c_Ss and c_Ss2 by the stage's parity within the evolve.  Large clouds
        // keep the separate epilogue: its rows are coalesced in original order, where the fused
        // lanes would touch S / B / A scattered by the sort (C5 evolve 23.2 -> 23.7 ms fused).
        const int parity = ((step - 1) * 4 + s) & 1;
        // the rebuild first: its IF node reads the condition the previous stage's sweep set
        const CellWs w = verlet_prepare(ctx, sc, step == 1 && s == 0, stream, parity);
        VerletEpi e{};
        e.a = fa;
        e.scale_q = sc.scale_q; e.scale_p = sc.scale_p; e.sigma2 = sc.sigma2;
        if (!last) {  // this sweep sets the condition of the next stage's IF node
            const VerletFuse f = verlet_fuse(ctx, sc, stream);
            e.Ss_next = parity ? ctx->c_Ss.ptr : ctx->c_Ss2.ptr;
            e.Xb = f.Xb; e.thr2 = f.thr2; e.flags = f.flags; e.cond = f.cond; e.use_cond = f.use_cond;
            e.decide = 1;
        }
        verlet_sweep(ctx, sc, w, ev, e, stream);
        return;
    }
    if (lists) {
        const CellWs w = verlet_prepare(ctx, sc, step == 1 && s == 0, stream, 0);
        const VerletWs v = verlet_ws(ctx, n, sc.cutoff);
        if (ctx->prof_on) prof_mark(ctx, stream);
        launch_verlet_pair(sc, w, v, n, ctx->part.ptr, ctx->st.ptr, ev, ctx->tbl.ptr,
                           ctx->prof_on ? ctx->c_acc.ptr : nullptr, stream);
        if (ctx->prof_on) prof_mark(ctx, stream);
        ctx->launches += 2;
        ctx->pair_launches++;
        if (!last) {
            VerletFuse f = verlet_fuse(ctx, sc, stream);
            if (ctx->verlet_rel) {  // rebuild on the relative displacement of neighbours (gs_verlet.cu)
                f.defer = 1;
                launch_finish_verlet(sc, fa, f, stream);
                launch_verlet_trigger(w, v, n, ctx->v_box.ptr, (int64_t)ctx->v_box.cap, f.cond,
                                      f.use_cond, stream);
                ctx->launches++;
            } else {
                launch_finish_verlet(sc, fa, f, stream);
            }
        } else {
            launch_finish(kFinStage, sc, fa, stream);
        }
        return;
    }
    po = pair_kernel(ctx, sc, ctx->S.ptr, n, ctx->row0, nrows, plan, ctx->part.ptr, ev, stream);
    fa.nchunks = po.nchunks; fa.pstride = po.pstride;
    ctx->launches++;  // finish
    launch_finish(kFinStage, sc, fa, stream);
}

void graph_reset(gs_context* ctx) {
    if (ctx->graph.exec) cudaGraphExecDestroy(ctx->graph.exec);
    for (cudaEvent_t e : ctx->graph.ev) cudaEventDestroy(e);
    ctx->graph = gs_context::Graph();
}

// Everything the captured kernels bake in: sizes, constants, buffer addresses, path, profiling.
std::vector<double> graph_key(gs_context* ctx, const SysConst& sc, double dt, int steps) {
    auto P = [](const void* p) { return (double)(uintptr_t)p; };
    return {(double)ctx->n, (double)ctx->row0, (double)ctx->row1, (double)steps, dt, (double)ctx->cell_on,
            (double)ctx->prof_on, (double)sc.fam, sc.k1, sc.scale_q, sc.scale_p, sc.sigma2, sc.cutoff,
            P(ctx->S.ptr), P(ctx->B.ptr), P(ctx->A.ptr), P(ctx->part.ptr), P(ctx->st.ptr), P(ctx->c_Ss.ptr), P(ctx->c_Ss2.ptr), P(ctx->c_Sf.ptr),
            P(ctx->c_cub.ptr), P(ctx->c_start.ptr), P(ctx->c_keys.ptr), P(ctx->c_perm.ptr), P(ctx->c_acc.ptr),
            P(ctx->c_keys_sorted.ptr), P(ctx->c_vals.ptr), P(ctx->c_bbox.ptr), P(ctx->c_gp.ptr), P(ctx->c_tlist.ptr),
            P(ctx->c_nsel.ptr), P(ctx->tbl.ptr), (double)ctx->c_cub_bytes, (double)ctx->verlet_call,
            P(ctx->v_cnt.ptr), P(ctx->v_ofs.ptr), P(ctx->v_len.ptr), P(ctx->v_inv.ptr), P(ctx->v_list.ptr), (double)ctx->v_list.cap, P(ctx->v_xb.ptr),
            P(ctx->v_flags.ptr), P(ctx->v_over.ptr), P(ctx->v_scan.ptr), ctx->verlet_skin, (double)ctx->verlet_fuse_max_n,
            P(ctx->v_box.ptr), (double)ctx->v_box.cap, (double)ctx->verlet_rel, P(ctx->v_skin.ptr),
            (double)ctx->skin_adapt};
}

// integrator.py:95-119 as one CUDA graph (4 x steps stages, ~2 kernels per dense stage and
// ~10 per cell-list stage) captured once per configuration and replayed on the caller's
// stream: no per-launch CPU overhead inside a shoot.
int run_evolve_graph(gs_context* ctx, const SysConst& sc, double t_final, int steps, cudaStream_t stream) {
    const double dt = t_final / steps;
    std::vector<double> key = graph_key(ctx, sc, dt, steps);
    if (!ctx->graph.exec || ctx->graph.key != key) {
        graph_reset(ctx);
        if (!ctx->cap_stream) GS_CUDA(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
        const long long l0 = ctx->launches, pl0 = ctx->pair_launches, hp0 = ctx->host_pairs;
        ctx->capture_events = &ctx->graph.ev;
        GS_CUDA(cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeThreadLocal));
        for (int step = 1; step <= steps; ++step)
            for (int s = 0; s < 4; ++s) stage(ctx, sc, step, s, dt, ctx->cap_stream, step == steps && s == 3);
        cudaGraph_t g = nullptr;
        cudaError_t e = cudaStreamEndCapture(ctx->cap_stream, &g);
        ctx->capture_events = nullptr;
        if (ctx->cell_err) {
            if (g) cudaGraphDestroy(g);
            return take_cell_err(ctx);
        }
        if (e != cudaSuccess) return fail(GS_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
        e = cudaGraphInstantiate(&ctx->graph.exec, g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) return fail(GS_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
        ctx->graph.key = key;
        ctx->graph.launches = ctx->launches - l0;
        ctx->graph.pair_launches = ctx->pair_launches - pl0;
        ctx->graph.host_pairs = ctx->host_pairs - hp0;
        ctx->launches = l0; ctx->pair_launches = pl0; ctx->host_pairs = hp0;  // counted per replay below
    }
    GS_CUDA(cudaGraphLaunch(ctx->graph.exec, stream));
    ctx->launches += ctx->graph.launches;
    ctx->pair_launches += ctx->graph.pair_launches;
    ctx->host_pairs += ctx->graph.host_pairs;
    return GS_OK;
}

// Harvest the pair-kernel times of the last graph replay (call after the stream is synced).
int graph_harvest(gs_context* ctx) {
    if (!ctx->prof_on || ctx->graph.ev.size() < 2) return GS_OK;
    for (size_t k = 0; k + 1 < ctx->graph.ev.size(); k += 2) {
        float t = 0.f;
        GS_CUDA(cudaEventElapsedTime(&t, ctx->graph.ev[k], ctx->graph.ev[k + 1]));
        ctx->prof_ms_acc += t;
    }
    return GS_OK;
}

// integrator.py:95-119 over the session rows (single rank: rows = all).
int run_evolve(gs_context* ctx, const SysConst& sc, double t_final, int steps, int capture_every, double* frames,
               cudaStream_t stream) {
    if (capture_every == 0 && ctx->graphs_on) return run_evolve_graph(ctx, sc, t_final, steps, stream);
    const double dt = t_final / steps;
    const int64_t nrows = ctx->row1 - ctx->row0;
    int f = 0;
    if (capture_every > 0 && frames)
        GS_CUDA(cudaMemcpyAsync(frames, ctx->B.ptr, nrows * sizeof(double4), cudaMemcpyDeviceToDevice, stream));
    if (capture_every > 0) f = 1;
    for (int step = 1; step <= steps; ++step) {
        NvtxScope nvtx_step("RK4 step");
        for (int s = 0; s < 4; ++s) stage(ctx, sc, step, s, dt, stream, step == steps && s == 3);
        if (capture_every > 0 && (step % capture_every == 0 || step == steps)) {
            if (frames)
                GS_CUDA(cudaMemcpyAsync(frames + (size_t)f * nrows * 4, ctx->B.ptr, nrows * sizeof(double4),
                                        cudaMemcpyDeviceToDevice, stream));
            ++f;
        }
    }
    GS_CUDA(cudaGetLastError());
    return take_cell_err(ctx);
}

// CTAs per small-N item: a cluster of kMaxCluster CTAs spreads the rows of one match over
// that many SMs (GS_B200_CLUSTER overrides; 1 = one CTA per item).
int small_cluster(int64_t n) {
    static int forced = -1;
    if (forced < 0) {
        const char* e = std::getenv("GS_B200_CLUSTER");
        const int v = e ? std::atoi(e) : 0;
        forced = (v == 1 || v == 2 || v == 4 || v == 8) ? v : 0;  // cluster sizes with a kernel instance
    }
    if (forced > 0) return forced;
    // A/B (st.async exchange, ms per feedback iteration): N = 64 -> 8 CTAs best (16, non-portable:
    // no faster); N = 60 (100 RK4 steps) 8 -> 0.57, 4 -> 0.67; N = 30: 8 -> 0.49, 4 -> 0.48; N = 8 -> 1
    return n >= 48 ? kMaxCluster : (n >= 16 ? 4 : 1);
}

void small_setup(SmallArgs& a, int64_t n) {
    a.n = n;
    a.cluster = small_cluster(n);
    small_threads(n, a.cluster, &a.split);
}

bool use_small(const gs_system_t* sys, int64_t n) {
    return n <= kSmallMax && sys->path != GS_PATH_CELL;
}

SmallItem small_item(const SysConst& sc, const gs_match_config_t* cfg) {
    SmallItem it{};
    it.sc = sc;
    it.t_final = cfg->t_final; it.steps = cfg->steps;
    it.h = cfg->h; it.epsilon = cfg->epsilon;
    it.max_iter = cfg->max_iter; it.stop_rule = cfg->stop_rule; it.norm = cfg->norm;
    return it;
}

int check_match(const gs_system_t* sys, const gs_match_config_t* cfg) {
    int rc = check_system(sys);
    if (rc) return rc;
    if (!cfg) return fail(GS_ERR_INVALID, "match config is NULL");
    if (!(cfg->h > 0.0) || !std::isfinite(cfg->h)) return fail(GS_ERR_INVALID, "h must be positive");
    if (!(cfg->epsilon > 0.0) || !std::isfinite(cfg->epsilon)) return fail(GS_ERR_INVALID, "epsilon must be positive");
    if (cfg->max_iter < 1) return fail(GS_ERR_INVALID, "max_iter must be >= 1");
    if (cfg->steps < 1 || !(cfg->t_final > 0.0) || !std::isfinite(cfg->t_final))
        return fail(GS_ERR_INVALID, "bad evolve config");
    if (cfg->stop_rule != GS_STOP_TARGET_RESIDUAL && cfg->stop_rule != GS_STOP_MOMENTUM_DELTA)
        return fail(GS_ERR_INVALID, "unknown stop rule");
    if (cfg->norm != GS_NORM_MAX && cfg->norm != GS_NORM_L2) return fail(GS_ERR_INVALID, "unknown norm");
    if (sys->sigma2 > 0.0 && cfg->stop_rule != GS_STOP_MOMENTUM_DELTA)
        return fail(GS_ERR_INVALID, "inexact matching (sigma2 > 0) cannot stop on the endpoint residual; "
                                    "use stop_rule = MomentumDelta");
    return GS_OK;
}

void small_to_result(const SmallResult& r, int64_t n, gs_match_result_t* out) {
    std::memset(out, 0, sizeof(*out));
    out->status.i = out->status.j = -1;
    out->outcome = r.outcome;
    out->iterations = r.iterations;
    out->hamiltonian = r.hamiltonian;
    out->final_residual = r.final_residual;
    if (r.outcome == GS_MATCH_EVOLVE_FAILED) {
        DevStatus d{r.fail_event, r.pair_key};
        decode_status(d, n, &out->status);
        out->status.iteration = r.fail_iter;
    }
}


int pairs_sym_impl(gs_context* ctx, const gs_system_t* sys, int32_t step, int32_t stg, int64_t part_begin,
                   int64_t part_end, double* R, void* stream, PeerSignal sig, PeerWait wait) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || ctx->n < 1 || !R) return fail(GS_ERR_INVALID, "no stage session");
    int rc = check_system(sys);
    if (rc) return rc;
    const int64_t n = ctx->n, total = gs_sym_parts(n);
    if (total == 0) return fail(GS_ERR_UNSUPPORTED, "symmetric split not available for this n");
    if (stg < 0 || stg > 3 || step < 1 || part_begin < 0 || part_end > total || part_begin > part_end)
        return fail(GS_ERR_INVALID, "bad stage / part range");
    GS_CUDA(cudaSetDevice(ctx->device));
    const SymPlan sp = sym_plan(n);
    GS_CUDA(ctx->part.ensure((size_t)sp.nsb * (size_t)sp.pstride));
    if (ctx->sym_key_n != n || ctx->sym_key_b != part_begin || ctx->sym_key_e != part_end) {
        // Each (slot, row) is written by exactly one superblock pair: tile (X, Y) stores the
        // I-side sums of X's rows in slot Y and the J-side sums of Y's rows in slot X.  List,
        // per row superblock, the slots this rank's pairs write (ascending); the reduction reads
        // only those, so the buffer needs no clearing.
        const int nsb = sp.nsb;
        std::vector<unsigned char> hit((size_t)nsb * nsb, 0);
        for (long long t = part_begin; t < part_end; ++t) {
            long long SI, SJ;
            sym_pair_of(t, nsb, &SI, &SJ);
            hit[(size_t)SI * nsb + SJ] = 1;
            hit[(size_t)SJ * nsb + SI] = 1;
        }
        std::vector<int> slots((size_t)nsb * nsb, 0), counts(nsb, 0);
        for (int X = 0; X < nsb; ++X)
            for (int Y = 0; Y < nsb; ++Y)
                if (hit[(size_t)X * nsb + Y]) slots[(size_t)X * nsb + counts[X]++] = Y;
        GS_CUDA(ctx->sym_slots.ensure(slots.size()));
        GS_CUDA(ctx->sym_counts.ensure(counts.size()));
        GS_CUDA(cudaMemcpy(ctx->sym_slots.ptr, slots.data(), slots.size() * sizeof(int), cudaMemcpyHostToDevice));
        GS_CUDA(cudaMemcpy(ctx->sym_counts.ptr, counts.data(), counts.size() * sizeof(int), cudaMemcpyHostToDevice));
        ctx->sym_key_n = n; ctx->sym_key_b = part_begin; ctx->sym_key_e = part_end;
    }
    const SysConst sc = make_const(sys);
    const unsigned long long ev = (unsigned long long)step * 8ull + 2ull * (unsigned long long)stg;
    if (ctx->prof_on) prof_mark(ctx, s);
    launch_dense_sym(sc, ctx->S.ptr, n, ctx->part.ptr, sp.pstride, ctx->st.ptr, ev, ctx->tbl.ptr, s, part_begin,
                     part_end, wait);
    if (ctx->prof_on) prof_mark(ctx, s);
    launch_slot_reduce_list(ctx->part.ptr, sp.pstride, n, sp.G * kDB, sp.nsb, ctx->sym_slots.ptr,
                            ctx->sym_counts.ptr, reinterpret_cast<double4*>(R), s, sig);
    ctx->launches += 2;
    ctx->pair_launches++;
    ctx->host_pairs += (long long)((double)n * (double)n * (double)(part_end - part_begin) / (double)total);
    GS_CUDA(cudaGetLastError());
    return GS_OK;
}


}  // namespace gsapi

// ======================================================================================
extern "C" {

#ifdef GS_CHECKED
const char* gs_version(void) { return "geoshoot-b200 0.1.0 (sm_100a, fp64, checked)"; }
#else
const char* gs_version(void) { return "geoshoot-b200 0.1.0 (sm_100a, fp64)"; }
#endif
int gs_abi_version(void) { return GS_ABI_VERSION; }
const char* gs_last_error(void) { return g_last_error.c_str(); }

int gs_create(gs_context** out, int device) {
    if (!out) return fail(GS_ERR_INVALID, "out is NULL");
    *out = nullptr;
    int ndev = 0;
    GS_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(GS_ERR_INVALID, "bad device ordinal");
    GS_CUDA(cudaSetDevice(device));
    gs_context* ctx = new gs_context();
    ctx->device = device;
    if (const char* g = std::getenv("GS_B200_GRAPHS")) ctx->graphs_on = std::atoi(g) != 0;
    if (const char* g = std::getenv("GS_B200_SYM")) ctx->sym_on = std::atoi(g) != 0;
    if (const char* g = std::getenv("GS_B200_DEVLOOP")) ctx->devloop_on = std::atoi(g) != 0;
    if (const char* g = std::getenv("GS_B200_VERLET")) ctx->verlet_on = std::atoi(g);
    if (const char* g = std::getenv("GS_B200_SKIN")) ctx->verlet_skin = std::atof(g);
    if (const char* g = std::getenv("GS_B200_VERLET_FUSE_MAX_N")) ctx->verlet_fuse_max_n = std::atoll(g);
    if (const char* g = std::getenv("GS_B200_VERLET_REL")) ctx->verlet_rel = std::atoi(g);
    if (const char* g = std::getenv("GS_B200_SKIN_ADAPT")) ctx->skin_adapt = std::atoi(g);
    if (const char* g = std::getenv("GS_B200_VERLET_SLACK")) ctx->verlet_slack = std::atof(g);  // tests
    cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device);
    // 2^(j/256), j = 0..255, rounded from long double
    // 2^(j/kTbl), j = 0..kTbl-1, rounded from long double, replicated kTblRep times interleaved
    std::vector<double> t(kTblWords);
    for (int j = 0; j < kTbl; ++j)
        for (int c = 0; c < kTblRep; ++c) t[j * kTblRep + c] = (double)exp2l((long double)j / (long double)kTbl);
    cudaError_t e = ctx->tbl.ensure(kTblWords);
    if (e == cudaSuccess) e = cudaMemcpy(ctx->tbl.ptr, t.data(), kTblWords * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = ctx->st.ensure(1);
    if (e == cudaSuccess) e = cudaMallocHost(&ctx->st_host, sizeof(DevStatus));
    if (e == cudaSuccess) e = cudaMallocHost(&ctx->scal_host, 16 * sizeof(double));
    if (e == cudaSuccess) e = cudaMallocHost(&ctx->mloop_host, sizeof(MatchLoop));
    if (e == cudaSuccess) e = ctx->scal.ensure(16);
    if (e == cudaSuccess) e = ctx->small_res.ensure(1);
    if (e != cudaSuccess) {
        gs_destroy(ctx);
        return fail(GS_ERR_CUDA, std::string("gs_create: ") + cudaGetErrorString(e));
    }
    *out = ctx;
    return GS_OK;
}

int gs_destroy(gs_context* ctx) {
    if (!ctx) return GS_OK;
    cudaSetDevice(ctx->device);
    ctx->tbl.release(); ctx->st.release(); ctx->S.release(); ctx->B.release(); ctx->A.release();
    ctx->part.release(); ctx->q0.release(); ctx->tgt.release(); ctx->p.release(); ctx->resid.release();
    ctx->red.release(); ctx->ham.release(); ctx->hist.release(); ctx->scal.release(); ctx->small_res.release();
    if (ctx->st_host) cudaFreeHost(ctx->st_host);
    if (ctx->scal_host) cudaFreeHost(ctx->scal_host);
    if (ctx->mloop_host) cudaFreeHost(ctx->mloop_host);
    if (ctx->mgraph.exec) cudaGraphExecDestroy(ctx->mgraph.exec);
    ctx->mloop.release(); ctx->ep.release(); ctx->c_tlist.release(); ctx->c_nsel.release();
    graph_reset(ctx);
    if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
    if (ctx->cap_stream2) cudaStreamDestroy(ctx->cap_stream2);
    for (cudaEvent_t e : ctx->prof_events) cudaEventDestroy(e);
    ctx->v_cnt.release(); ctx->v_list.release(); ctx->v_len.release(); ctx->v_inv.release(); ctx->v_ofs.release(); ctx->v_xb.release(); ctx->v_flags.release();
    ctx->v_over.release(); ctx->v_scan.release(); ctx->cg.release(); ctx->v_box.release(); ctx->v_skin.release();
    ctx->c_keys.release(); ctx->c_keys_sorted.release(); ctx->c_vals.release(); ctx->c_perm.release();
    ctx->c_start.release(); ctx->c_Ss.release(); ctx->c_Ss2.release(); ctx->c_Sf.release(); ctx->c_bbox.release(); ctx->c_gp.release(); ctx->c_cub.release();
    gs_p2p_close(ctx);
    ctx->p2p.R.release(); ctx->p2p.flags.release(); ctx->p2p.done.release(); ctx->p2p.Rp.release(); ctx->p2p.Sp.release(); ctx->p2p.Fp.release();
    ctx->c_acc.release(); ctx->gram_bad.release(); ctx->b_items.release(); ctx->b_st.release(); ctx->vf_part.release(); ctx->sym_slots.release();
    ctx->sym_counts.release();
    {
        auto& L = ctx->slab;
        L.S.release(); L.S2.release(); L.gidx.release(); L.B.release(); L.A.release(); L.Xb.release();
        L.Su.release(); L.Bu.release(); L.Au.release(); L.gu.release(); L.skey.release(); L.skey2.release();
        L.sval.release(); L.sval2.release(); L.cub.release(); L.keys.release(); L.start.release();
        L.cfirst.release(); L.head.release(); L.len.release(); L.list.release(); L.Sf.release(); L.gp.release();
        L.cnt.release(); L.ofs.release(); L.red.release(); L.b4.release(); L.dest.release(); L.dcount.release();
        L.flags.release(); L.over.release();
    }
    delete ctx;
    return GS_OK;
}

int gs_status_reset(gs_context* ctx, void* stream) {
    if (!ctx) return fail(GS_ERR_INVALID, "ctx is NULL");
    k_status_reset<<<1, 1, 0, (cudaStream_t)stream>>>(ctx->st.ptr);
    GS_CUDA(cudaGetLastError());
    return GS_OK;
}

int gs_status_fetch(gs_context* ctx, gs_status_t* status, void* stream) {
    if (!ctx) return fail(GS_ERR_INVALID, "ctx is NULL");
    const int rc = fetch_status(ctx, (cudaStream_t)stream, ctx->n > 0 ? ctx->n : 1, status);
    return rc == GS_ERR_CUDA ? rc : GS_OK;
}

static int rhs_impl(gs_context* ctx, const gs_system_t* sys, int64_t n, const double* q, const double* p,
                    int64_t row0, int64_t row1, double* dq, double* dp, cudaStream_t s) {
    if (!ctx) return fail(GS_ERR_INVALID, "ctx is NULL");
    int rc = check_system(sys);
    if (rc) return rc;
    if (n < 1 || !q || !p || !dq || !dp) return fail(GS_ERR_INVALID, "q and p must have shape (N, 2), N >= 1");
    if (row0 < 0 || row1 > n || row0 > row1) return fail(GS_ERR_INVALID, "bad row range");
    GS_CUDA(cudaSetDevice(ctx->device));
    const int64_t nrows = row1 - row0;
    if ((rc = ensure_session(ctx, n, nrows))) return rc;
    ctx->n = n; ctx->row0 = row0; ctx->row1 = row1;
    const SysConst sc = make_const(sys);
    k_status_reset<<<1, 1, 0, s>>>(ctx->st.ptr);
    k_pack<<<nblk(n), 256, 0, s>>>(q, p, n, ctx->S.ptr, ctx->st.ptr, 1);
    if ((rc = choose_path(ctx, sys, ctx->S.ptr, n, s))) return rc;
    const DensePlan plan = dense_plan(n, ctx->sm_count);
    const PairOut po = pair_kernel(ctx, sc, ctx->S.ptr, n, row0, nrows, plan, ctx->part.ptr, 2ull, s);
    ctx->launches += 3;  // reset, pack, finish
    FinishArgs fa{};
    fa.part = ctx->part.ptr; fa.nchunks = po.nchunks; fa.pstride = po.pstride; fa.nrows = nrows; fa.row0 = row0;
    fa.S = ctx->S.ptr;
    fa.dq = dq; fa.dp = dp; fa.st = ctx->st.ptr; fa.event = 3ull;
    launch_finish(kFinRhs, sc, fa, s);
    GS_CUDA(cudaGetLastError());
    return take_cell_err(ctx);
}

int gs_rhs_rows(gs_context* ctx, const gs_system_t* sys, int64_t n, const double* q, const double* p, int64_t row0,
                int64_t row1, double* dq, double* dp, void* stream) {
    gsapi::NvtxScope nvtx_("gs_rhs_rows");
    return rhs_impl(ctx, sys, n, q, p, row0, row1, dq, dp, (cudaStream_t)stream);
}

int gs_rhs(gs_context* ctx, const gs_system_t* sys, int64_t n, const double* q, const double* p, double* dq,
           double* dp, gs_status_t* status, void* stream) {
    gsapi::NvtxScope nvtx_("gs_rhs");
    int rc = rhs_impl(ctx, sys, n, q, p, 0, n, dq, dp, (cudaStream_t)stream);
    if (rc) return rc;
    gs_status_t st;
    rc = fetch_status(ctx, (cudaStream_t)stream, n, &st);
    if (status) *status = st;
    if (rc == GS_ERR_INVALID) return fail(rc, "state contains non-finite entries");
    return rc;
}

int gs_hamiltonian(gs_context* ctx, const gs_system_t* sys, int64_t n, const double* q, const double* p,
                   double* h_out, void* stream) {
    gsapi::NvtxScope nvtx_("gs_hamiltonian");
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || !h_out) return fail(GS_ERR_INVALID, "NULL argument");
    int rc = check_system(sys);
    if (rc) return rc;
    if (n < 1 || !q || !p) return fail(GS_ERR_INVALID, "q and p must have shape (N, 2), N >= 1");
    GS_CUDA(cudaSetDevice(ctx->device));
    if ((rc = ensure_session(ctx, n, n))) return rc;
    GS_CUDA(ctx->ham.ensure(n));
    GS_CUDA(ctx->red.ensure(kRedBlocks));
    ctx->n = n; ctx->row0 = 0; ctx->row1 = n;
    const SysConst sc = make_const(sys);
    k_status_reset<<<1, 1, 0, s>>>(ctx->st.ptr);
    k_pack<<<nblk(n), 256, 0, s>>>(q, p, n, ctx->S.ptr, ctx->st.ptr, 0);
    if ((rc = choose_path(ctx, sys, ctx->S.ptr, n, s))) return rc;
    const DensePlan plan = dense_plan(n, ctx->sm_count);
    // coincident pairs are irrelevant to H (particles.py:127-128 has no check): use an event id
    // that is never reported
    const PairOut po = pair_kernel(ctx, sc, ctx->S.ptr, n, 0, n, plan, ctx->part.ptr, 2ull, s);
    if ((rc = take_cell_err(ctx))) return rc;
    ctx->launches += 5;  // reset, pack, finish, 2 reductions
    FinishArgs fa{};
    fa.part = ctx->part.ptr; fa.nchunks = po.nchunks; fa.pstride = po.pstride; fa.nrows = n; fa.row0 = 0;
    fa.S = ctx->S.ptr;
    fa.ham = ctx->ham.ptr; fa.st = ctx->st.ptr; fa.event = 0ull;  // never skipped
    launch_finish(kFinHam, sc, fa, s);
    const int nb = (int)std::min<int64_t>(kRedBlocks, (n + 255) / 256);
    k_sum_partial<<<nb, 256, 0, s>>>(ctx->ham.ptr, n, ctx->red.ptr);
    k_reduce_final<<<1, 512, 0, s>>>(ctx->red.ptr, nb, 2, ctx->scal.ptr, nullptr);
    GS_CUDA(cudaMemcpyAsync(ctx->scal_host, ctx->scal.ptr, sizeof(double), cudaMemcpyDeviceToHost, s));
    GS_CUDA(cudaStreamSynchronize(s));
    *h_out = ctx->scal_host[0];
    return GS_OK;
}

int gs_evolve(gs_context* ctx, const gs_system_t* sys, int64_t n, double t_final, int32_t steps,
              int32_t capture_every, double* q, double* p, double* frames, gs_status_t* status, void* stream) {
    gsapi::NvtxScope nvtx_("gs_evolve");
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx) return fail(GS_ERR_INVALID, "ctx is NULL");
    int rc = check_system(sys);
    if (rc) return rc;
    if (n < 1 || !q || !p) return fail(GS_ERR_INVALID, "q and p must have shape (N, 2), N >= 1");
    if (!(t_final > 0.0) || !std::isfinite(t_final)) return fail(GS_ERR_INVALID, "t_final must be positive");
    if (steps < 1) return fail(GS_ERR_INVALID, "steps must be >= 1");
    if (capture_every < 0) return fail(GS_ERR_INVALID, "capture_every must be >= 0");
    GS_CUDA(cudaSetDevice(ctx->device));
    const SysConst sc = make_const(sys);
    ctx->n = n;
    if (use_small(sys, n)) {
        SmallArgs a{};
        small_setup(a, n); a.batch = 1; a.mode = 0;
        a.item.sc = sc; a.item.t_final = t_final; a.item.steps = steps;
        a.capture_every = capture_every; a.q_in = q; a.p_in = p; a.q_out = q; a.p_out = p; a.frames = frames;
        a.st = ctx->st.ptr;
        ctx->host_pairs += 4LL * steps * n * n;
        if (ctx->prof_on) cudaEventRecord(prof_event(ctx), s);
        GS_CUDA((cudaError_t)launch_small(sc.fam, a, ctx->tbl.ptr, s));
        if (ctx->prof_on) cudaEventRecord(prof_event(ctx), s);
        ctx->launches++;
        ctx->pair_launches++;
    } else {
        if ((rc = ensure_session(ctx, n, n))) return rc;
        ctx->row0 = 0; ctx->row1 = n;
        // (verlet_on >= 2: lists in host-driven evolves too, for per-kernel profiling)
        const bool multi = capture_every == 0 && (ctx->graphs_on || ctx->verlet_on >= 2);
        for (bool retry = true; retry;) {
            ctx->launches += 4;  // reset, pack, copy, unpack
            k_status_reset<<<1, 1, 0, s>>>(ctx->st.ptr);
            k_pack<<<nblk(n), 256, 0, s>>>(q, p, n, ctx->S.ptr, ctx->st.ptr, 0);
            if ((rc = choose_path(ctx, sys, ctx->S.ptr, n, s, multi))) return rc;
            k_copy_rows<<<nblk(n), 256, 0, s>>>(ctx->S.ptr, 0, n, ctx->B.ptr);
            if ((rc = run_evolve(ctx, sc, t_final, steps, capture_every, frames, s))) return rc;
            if ((rc = verlet_retry(ctx, s, &retry))) return rc;  // lists outgrew their buffer: redo
        }
        k_unpack<<<nblk(n), 256, 0, s>>>(ctx->B.ptr, n, q, p);
        GS_CUDA(cudaGetLastError());
    }
    gs_status_t st;
    rc = fetch_status(ctx, s, n, &st);
    if (status) *status = st;
    if (rc != GS_ERR_CUDA) {
        const int hr = graph_harvest(ctx);
        if (hr) return hr;
    }
    return rc;
}

// The whole feedback loop as ONE graph launch: a conditional WHILE node whose body is an
// iteration (momentum update, 4 x steps RK stages, residual, norm, k_match_decide); the
// device decides when to stop, the host reads the outcome once at the end.  Returns
// GS_ERR_UNSUPPORTED when the runtime cannot build conditional nodes (the caller then runs the
// host-driven loop).
int match_device_loop(gs_context* ctx, const SysConst& sc, const gs_match_config_t* cfg, int64_t n,
                      double* endpoint_out, int nb, int red_kind, double nrm0, cudaStream_t s, MatchLoop* out) {
    GS_CUDA(ctx->mloop.ensure(1));
    GS_CUDA(ctx->hist.ensure(cfg->max_iter));
    GS_CUDA(ctx->ep.ensure(2 * n));
    if (!ctx->cap_stream) GS_CUDA(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
    const double dt = cfg->t_final / cfg->steps;
    // everything the loop graph bakes in (the evolve's key + the loop's constants and buffers)
    std::vector<double> key = graph_key(ctx, sc, dt, cfg->steps);
    auto P = [](const void* p) { return (double)(uintptr_t)p; };
    for (double v : {cfg->h, cfg->epsilon, (double)cfg->max_iter, (double)cfg->stop_rule, (double)cfg->norm, (double)nb,
                     (double)red_kind, P(ctx->q0.ptr), P(ctx->p.ptr), P(ctx->resid.ptr), P(ctx->tgt.ptr),
                     P(ctx->red.ptr), P(ctx->scal.ptr), P(ctx->mloop.ptr), P(ctx->hist.ptr), P(ctx->ep.ptr)})
        key.push_back(v);
    if (!ctx->mgraph.exec || ctx->mgraph.key != key) {
        if (ctx->mgraph.exec) cudaGraphExecDestroy(ctx->mgraph.exec);
        ctx->mgraph = gs_context::LoopGraph();
        cudaGraph_t g = nullptr;
        GS_CUDA(cudaGraphCreate(&g, 0));
        cudaGraphConditionalHandle cond;
        cudaGraphNode_t node;
        cudaGraphNodeParams np = {};
        if (cudaGraphConditionalHandleCreate(&cond, g, 1, cudaGraphCondAssignDefault) != cudaSuccess) {
            (void)cudaGetLastError();
            cudaGraphDestroy(g);
            return GS_ERR_UNSUPPORTED;
        }
        np.type = cudaGraphNodeTypeConditional;
        np.conditional.handle = cond;
        np.conditional.type = cudaGraphCondTypeWhile;
        np.conditional.size = 1;
        if (cudaGraphAddNode(&node, g, nullptr, 0, &np) != cudaSuccess) {
            (void)cudaGetLastError();
            cudaGraphDestroy(g);
            return GS_ERR_UNSUPPORTED;
        }
        cudaGraph_t body = np.conditional.phGraph_out[0];
        const long long l0 = ctx->launches, pl0 = ctx->pair_launches, hp0 = ctx->host_pairs;
        cudaStream_t c = ctx->cap_stream;
        cudaError_t e = cudaStreamBeginCaptureToGraph(c, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
        if (e != cudaSuccess) {
            cudaGraphDestroy(g);
            return fail(GS_ERR_CUDA, std::string("loop capture: ") + cudaGetErrorString(e));
        }
        k_match_begin<<<nblk(n), 256, 0, c>>>(ctx->q0.ptr, ctx->p.ptr, ctx->resid.ptr, cfg->h, n, ctx->S.ptr,
                                              ctx->B.ptr);
        k_status_reset<<<1, 1, 0, c>>>(ctx->st.ptr);
        for (int step = 1; step <= cfg->steps; ++step)
            for (int st = 0; st < 4; ++st) stage(ctx, sc, step, st, dt, c, step == cfg->steps && st == 3);
        k_residual<<<nb, 256, 0, c>>>(reinterpret_cast<const double*>(ctx->B.ptr), 4, ctx->tgt.ptr, n, ctx->ep.ptr,
                                      ctx->resid.ptr, cfg->norm, ctx->red.ptr, ctx->st.ptr);
        k_reduce_final<<<1, 512, 0, c>>>(ctx->red.ptr, nb, red_kind, ctx->scal.ptr, ctx->st.ptr);
        k_match_decide<<<1, 1, 0, c>>>(ctx->mloop.ptr, ctx->scal.ptr, ctx->st.ptr, ctx->hist.ptr, cfg->h,
                                       cfg->epsilon, cfg->max_iter, cfg->stop_rule, cond);
        cudaGraph_t captured = nullptr;
        e = cudaStreamEndCapture(c, &captured);
        if (ctx->cell_err) {
            cudaGraphDestroy(g);
            return take_cell_err(ctx);
        }
        ctx->mgraph.launches = ctx->launches - l0 + 4;
        ctx->mgraph.pair_launches = ctx->pair_launches - pl0;
        ctx->mgraph.host_pairs = ctx->host_pairs - hp0;
        ctx->launches = l0; ctx->pair_launches = pl0; ctx->host_pairs = hp0;
        if (e == cudaSuccess) e = cudaGraphInstantiate(&ctx->mgraph.exec, g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) {
            ctx->mgraph = gs_context::LoopGraph();
            return fail(GS_ERR_CUDA, std::string("loop graph: ") + cudaGetErrorString(e));
        }
        ctx->mgraph.key = key;
    }
    MatchLoop m{};
    m.outcome = GS_MATCH_CAP;
    m.nrm = nrm0;
    m.initial = nrm0;
    m.have_initial = cfg->stop_rule == GS_STOP_TARGET_RESIDUAL;
    *ctx->mloop_host = m;
    cudaError_t e = cudaMemcpyAsync(ctx->mloop.ptr, ctx->mloop_host, sizeof(MatchLoop), cudaMemcpyHostToDevice, s);
    // the graph's endpoint buffer starts from the initial shoot's endpoint (kept on a failure)
    if (e == cudaSuccess) e = cudaMemcpyAsync(ctx->ep.ptr, endpoint_out, 2 * n * sizeof(double), cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess) e = cudaGraphLaunch(ctx->mgraph.exec, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(endpoint_out, ctx->ep.ptr, 2 * n * sizeof(double), cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(ctx->mloop_host, ctx->mloop.ptr, sizeof(MatchLoop), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return fail(GS_ERR_CUDA, std::string("loop graph launch: ") + cudaGetErrorString(e));
    *out = *ctx->mloop_host;
    const long long its = out->iters + (out->outcome == GS_MATCH_EVOLVE_FAILED);
    ctx->launches += its * ctx->mgraph.launches;
    ctx->pair_launches += its * ctx->mgraph.pair_launches;
    ctx->host_pairs += its * ctx->mgraph.host_pairs;
    return GS_OK;
}

int gs_match(gs_context* ctx, const gs_system_t* sys, const gs_match_config_t* cfg, int64_t n, const double* q0,
             const double* target, double* p0_out, double* endpoint_out, double* history_out,
             gs_match_result_t* result, void* stream) {
    gsapi::NvtxScope nvtx_("gs_match");
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || !cfg || !result || !history_out) return fail(GS_ERR_INVALID, "NULL argument");
    int rc = check_match(sys, cfg);
    if (rc) return rc;
    if (n < 1 || !q0 || !target || !p0_out || !endpoint_out)
        return fail(GS_ERR_INVALID, "templates must have shape (N, 2), N >= 1");
    GS_CUDA(cudaSetDevice(ctx->device));
    const SysConst sc = make_const(sys);
    std::memset(result, 0, sizeof(*result));
    result->status.i = result->status.j = -1;
    cudaEvent_t e0, e1;
    GS_CUDA(cudaEventCreate(&e0));
    GS_CUDA(cudaEventCreate(&e1));
    GS_CUDA(cudaEventRecord(e0, s));
    ctx->n = n;

    if (use_small(sys, n)) {
        GS_CUDA(ctx->hist.ensure(cfg->max_iter));
        SmallArgs a{};
        small_setup(a, n); a.batch = 1; a.mode = 1;
        a.item = small_item(sc, cfg);
        a.q_in = q0; a.target = target; a.q_out = endpoint_out; a.p_out = p0_out;
        a.history = ctx->hist.ptr; a.result = ctx->small_res.ptr; a.st = ctx->st.ptr;
        if (ctx->prof_on) cudaEventRecord(prof_event(ctx), s);
        GS_CUDA((cudaError_t)launch_small(sc.fam, a, ctx->tbl.ptr, s));
        if (ctx->prof_on) cudaEventRecord(prof_event(ctx), s);
        ctx->launches++;
        ctx->pair_launches++;
        GS_CUDA(cudaEventRecord(e1, s));
        SmallResult r;
        GS_CUDA(cudaMemcpyAsync(&r, ctx->small_res.ptr, sizeof(r), cudaMemcpyDeviceToHost, s));
        GS_CUDA(cudaStreamSynchronize(s));
        if (r.iterations > 0)
            GS_CUDA(cudaMemcpy(history_out, ctx->hist.ptr, r.iterations * sizeof(double), cudaMemcpyDeviceToHost));
        ctx->host_pairs += (long long)(r.iterations + (r.outcome == GS_MATCH_EVOLVE_FAILED)) * 4LL * cfg->steps * n * n +
                           n * n;
        small_to_result(r, n, result);
    } else {
        // host-driven loop, all state on the device, two scalars read back per iteration
      for (bool verlet_redo = true; verlet_redo;) {
        verlet_redo = false;
        if ((rc = ensure_session(ctx, n, n))) return rc;
        GS_CUDA(ctx->q0.ensure(2 * n)); GS_CUDA(ctx->tgt.ensure(2 * n)); GS_CUDA(ctx->p.ensure(2 * n));
        GS_CUDA(ctx->resid.ensure(2 * n)); GS_CUDA(ctx->red.ensure(kRedBlocks)); GS_CUDA(ctx->ham.ensure(n));
        ctx->row0 = 0; ctx->row1 = n;
        GS_CUDA(cudaMemcpyAsync(ctx->q0.ptr, q0, 2 * n * sizeof(double), cudaMemcpyDeviceToDevice, s));
        GS_CUDA(cudaMemcpyAsync(ctx->tgt.ptr, target, 2 * n * sizeof(double), cudaMemcpyDeviceToDevice, s));
        GS_CUDA(cudaMemsetAsync(ctx->p.ptr, 0, 2 * n * sizeof(double), s));
        k_match_begin<<<nblk(n), 256, 0, s>>>(ctx->q0.ptr, ctx->p.ptr, ctx->resid.ptr, 0.0, n, ctx->S.ptr, ctx->B.ptr);
        if ((rc = choose_path(ctx, sys, ctx->S.ptr, n, s, ctx->graphs_on != 0))) return rc;
        // initial shoot with p = 0 leaves q0 unchanged bitwise: endpoint = q0 (shooting.py:244-247)
        const int nb = (int)std::min<int64_t>(kRedBlocks, (n + 255) / 256);
        const int red_kind = cfg->norm == GS_NORM_MAX ? 0 : 1;
        k_residual<<<nb, 256, 0, s>>>(ctx->q0.ptr, 2, ctx->tgt.ptr, n, endpoint_out, ctx->resid.ptr, cfg->norm,
                                      ctx->red.ptr, nullptr);
        k_reduce_final<<<1, 512, 0, s>>>(ctx->red.ptr, nb, red_kind, ctx->scal.ptr, nullptr);
        GS_CUDA(cudaMemcpyAsync(ctx->scal_host, ctx->scal.ptr, sizeof(double), cudaMemcpyDeviceToHost, s));
        GS_CUDA(cudaStreamSynchronize(s));
        double nrm = ctx->scal_host[0];
        double initial = nrm;
        bool have_initial = cfg->stop_rule == GS_STOP_TARGET_RESIDUAL;
        int outcome = GS_MATCH_CAP, iters = 0;
        bool done = false;
        if (cfg->stop_rule == GS_STOP_TARGET_RESIDUAL && nrm < cfg->epsilon) {
            outcome = GS_MATCH_CONVERGED;
            done = true;
        } else if (ctx->devloop_on && !ctx->prof_on) {
            MatchLoop m{};
            rc = match_device_loop(ctx, sc, cfg, n, endpoint_out, nb, red_kind, nrm, s, &m);
            if (rc != GS_OK && rc != GS_ERR_UNSUPPORTED) return rc;
            if (rc == GS_OK) {
                done = true;
                outcome = m.outcome;
                iters = m.iters;
                nrm = m.nrm;
                if (iters > 0)
                    GS_CUDA(cudaMemcpy(history_out, ctx->hist.ptr, iters * sizeof(double), cudaMemcpyDeviceToHost));
                if (outcome == GS_MATCH_EVOLVE_FAILED) {
                    gs_status_t st;
                    if (fetch_status(ctx, s, n, &st) == GS_ERR_CUDA) return GS_ERR_CUDA;
                    result->status = st;
                    result->status.iteration = m.fail_it;
                }
            }
        }
        if (!done) {
            for (int it = 0; it < cfg->max_iter; ++it) {
                NvtxScope nvtx_it("feedback iteration");
                const double delta = cfg->h * nrm;
                k_match_begin<<<nblk(n), 256, 0, s>>>(ctx->q0.ptr, ctx->p.ptr, ctx->resid.ptr, cfg->h, n, ctx->S.ptr,
                                                      ctx->B.ptr);
                ctx->launches += 4;  // begin, reset, residual, reduce
                k_status_reset<<<1, 1, 0, s>>>(ctx->st.ptr);
                if ((rc = run_evolve(ctx, sc, cfg->t_final, cfg->steps, 0, nullptr, s))) return rc;
                k_residual<<<nb, 256, 0, s>>>(reinterpret_cast<const double*>(ctx->B.ptr), 4, ctx->tgt.ptr, n,
                                              endpoint_out, ctx->resid.ptr, cfg->norm, ctx->red.ptr, ctx->st.ptr);
                k_reduce_final<<<1, 512, 0, s>>>(ctx->red.ptr, nb, red_kind, ctx->scal.ptr, ctx->st.ptr);
                GS_CUDA(cudaMemcpyAsync(ctx->scal_host, ctx->scal.ptr, sizeof(double), cudaMemcpyDeviceToHost, s));
                gs_status_t st;
                rc = fetch_status(ctx, s, n, &st);  // synchronises
                if (rc == GS_ERR_CUDA) return rc;
                if ((rc = graph_harvest(ctx))) return rc;
                if (st.code != GS_OK) {
                    outcome = GS_MATCH_EVOLVE_FAILED;
                    result->status = st;
                    result->status.iteration = it + 1;
                    break;
                }
                nrm = ctx->scal_host[0];
                const double value = cfg->stop_rule == GS_STOP_TARGET_RESIDUAL ? nrm : delta;
                if (!have_initial) { initial = value; have_initial = true; }
                history_out[it] = value;
                iters = it + 1;
                if (!std::isfinite(value) || (initial > 0.0 && value > 1e6 * initial)) { outcome = GS_MATCH_BLOWUP; break; }
                if (value < cfg->epsilon) { outcome = GS_MATCH_CONVERGED; break; }
            }
        }
        if ((rc = verlet_retry(ctx, s, &verlet_redo))) return rc;  // lists outgrew their buffer: redo
        if (verlet_redo) {
            std::memset(result, 0, sizeof(*result));
            result->status.i = result->status.j = -1;
            continue;
        }
        GS_CUDA(cudaMemcpyAsync(p0_out, ctx->p.ptr, 2 * n * sizeof(double), cudaMemcpyDeviceToDevice, s));
        GS_CUDA(cudaEventRecord(e1, s));
        double H = 0.0;
        if ((rc = gs_hamiltonian(ctx, sys, n, q0, p0_out, &H, stream))) return rc;
        result->outcome = outcome;
        result->iterations = iters;
        result->hamiltonian = H;
        result->final_residual = nrm;
      }
    }
    GS_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    result->seconds_device = ms * 1e-3;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return GS_OK;
}

// Cluster Verlet list diagnostics: list builds since the context was created (incl. the sizing
// builds) and the entries of the last build.  Synchronises.
int gs_cell_stats(gs_context* ctx, int64_t* builds, int64_t* entries, void* stream) {
    if (!ctx || !builds || !entries) return fail(GS_ERR_INVALID, "NULL argument");
    *builds = 0;
    *entries = 0;
    if (ctx->v_flags.cap == 0) return GS_OK;
    cudaStream_t s = (cudaStream_t)stream;
    unsigned f[4];
    long long tot = 0;
    GS_CUDA(cudaMemcpyAsync(f, ctx->v_flags.ptr, sizeof(f), cudaMemcpyDeviceToHost, s));
    if (ctx->v_list_n > 0)
        GS_CUDA(cudaMemcpyAsync(&tot, ctx->v_ofs.ptr + verlet_clusters(ctx->v_list_n), sizeof(tot),
                                cudaMemcpyDeviceToHost, s));
    GS_CUDA(cudaStreamSynchronize(s));
    *builds = f[1];
    *entries = tot;
    return GS_OK;
}

// ---- matrix-free Gram solve (velocity update space) --------------------------
// shooting.py:138-159, 263-265: p = K^-1 u with K_ij = G(|q0_i - q0_j|) (the reference factors K
// once with Cholesky).  Here K v is the dq half of the RHS at (q0, v) — the same pair kernels
// (dense, cell sweep or cluster lists built once: q0 never moves) — and conjugate gradients on the
// 2N vector (K (x) I2 is SPD) solve to a relative residual `tol`.  Reductions are fixed-order.

namespace gsapi {

__global__ void k_cg_dot_partial(const double* __restrict__ a, const double* __restrict__ b, int64_t m, double* red) {
    __shared__ double s[256];
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        acc = fma(a[i], b[i], acc);
    s[threadIdx.x] = acc;
    __syncthreads();
    for (int w = blockDim.x / 2; w; w >>= 1) {
        if (threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) red[blockIdx.x] = s[0];
}

// r = u - Kp; d = r
__global__ void k_cg_init(const double* __restrict__ u, const double* __restrict__ Kp, int64_t m, double* r, double* d) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) {
        const double v = u[i] - Kp[i];
        r[i] = v;
        d[i] = v;
    }
}

// p += alpha d; r -= alpha Kd   (alpha = scal[0] / scal[1])
__global__ void k_cg_step(const double* __restrict__ scal, const double* __restrict__ d, const double* __restrict__ Kd,
                          int64_t m, double* p, double* r) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) {
        const double alpha = scal[0] / scal[1];
        p[i] = fma(alpha, d[i], p[i]);
        r[i] = fma(-alpha, Kd[i], r[i]);
    }
}

// d = r + beta d   (beta = scal[2] / scal[0])
__global__ void k_cg_dir(const double* __restrict__ scal, const double* __restrict__ r, int64_t m, double* d) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) d[i] = fma(scal[2] / scal[0], d[i], r[i]);
}

}  // namespace gsapi

// out = K v at the fixed points q0 (device, n x 2 each).  With lists: the cluster lists of q0,
// built by the caller, refreshed (momenta only) and swept.
static void gram_matvec(gs_context* ctx, const SysConst& sc, int64_t n, const double* q0, const double* v,
                        double* out, double* scratch, bool lists, cudaStream_t s) {
    k_pack<<<nblk(n), 256, 0, s>>>(q0, v, n, ctx->S.ptr, ctx->st.ptr, 0);
    PairOut po{1, 0};
    if (lists) {
        CellWs w = cell_ws(ctx);
        VerletWs vw = verlet_ws(ctx, n, sc.cutoff);
        verlet_gather(w, vw, ctx->S.ptr, n, 0, cudaGraphConditionalHandle{}, 0, s);
        launch_verlet_pair(sc, w, vw, n, ctx->part.ptr, ctx->st.ptr, 2ull, ctx->tbl.ptr, nullptr, s);
        ctx->launches += 2;
        ctx->pair_launches++;
    } else {
        const DensePlan plan = dense_plan(n, ctx->sm_count);
        po = pair_kernel(ctx, sc, ctx->S.ptr, n, 0, n, plan, ctx->part.ptr, 2ull, s);
    }
    FinishArgs fa{};
    fa.part = ctx->part.ptr; fa.nchunks = po.nchunks; fa.pstride = po.pstride; fa.nrows = n; fa.row0 = 0;
    fa.S = ctx->S.ptr; fa.dq = out; fa.dp = scratch; fa.st = ctx->st.ptr; fa.event = 3ull;
    launch_finish(kFinRhs, sc, fa, s);
    ctx->launches += 2;
}

extern "C" int gs_gram_cg(gs_context* ctx, const gs_system_t* sys, int64_t n, const double* q0, const double* u,
                          double* p, double tol, int32_t max_it, int32_t* iters, double* coef, double* relres,
                          void* stream) {
    gsapi::NvtxScope nvtx_("gs_gram_cg");
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || !iters || !relres) return fail(GS_ERR_INVALID, "NULL argument");
    int rc = check_system(sys);
    if (rc) return rc;
    if (n < 1 || !q0 || !u || !p) return fail(GS_ERR_INVALID, "q0, u and p must have shape (N, 2), N >= 1");
    if (!(tol > 0.0) || max_it < 1) return fail(GS_ERR_INVALID, "tol must be positive and max_it >= 1");
    GS_CUDA(cudaSetDevice(ctx->device));
    gs_system_t plain = *sys;
    plain.sigma2 = 0.0;  // K only (the sigma2 term belongs to the RHS, not to the Gram matrix)
    const SysConst sc = make_const(&plain);
    if ((rc = ensure_session(ctx, n, n))) return rc;
    ctx->n = n; ctx->row0 = 0; ctx->row1 = n;
    const int64_t m = 2 * n;
    GS_CUDA(ctx->cg.ensure(4 * m));
    GS_CUDA(ctx->red.ensure(kRedBlocks));
    double* r = ctx->cg.ptr;
    double* d = r + m;
    double* Kd = d + m;
    double* scratch = Kd + m;
    k_status_reset<<<1, 1, 0, s>>>(ctx->st.ptr);
    k_pack<<<nblk(n), 256, 0, s>>>(q0, p, n, ctx->S.ptr, ctx->st.ptr, 0);
    if ((rc = choose_path(ctx, &plain, ctx->S.ptr, n, s, false))) return rc;
    bool lists = false;
    if (ctx->cell_on && ctx->verlet_on) {  // q0 is fixed: one list build serves every product
        if ((rc = ensure_verlet(ctx, ctx->S.ptr, n, sc.cutoff, s))) return rc;
        for (int attempt = 0; attempt < 3; ++attempt) {
            if (verlet_build(cell_ws(ctx), verlet_ws(ctx, n, sc.cutoff), ctx->S.ptr, n, sc.cutoff, s))
                return fail(GS_ERR_CUDA, "verlet build failed");
            ctx->verlet_call = 1;
            bool retry = false;
            if ((rc = verlet_retry(ctx, s, &retry))) return rc;
            if (!retry) break;
        }
        lists = ctx->verlet_on != 0;
    }
    const int nb = (int)std::min<int64_t>(kRedBlocks, (m + 255) / 256);
    double* sc_dev = ctx->scal.ptr;  // [0] r.r, [1] d.Kd, [2] r.r new, [3] u.u
    auto dot = [&](const double* a, const double* b, int slot) {
        k_cg_dot_partial<<<nb, 256, 0, s>>>(a, b, m, ctx->red.ptr);
        k_reduce_final<<<1, 512, 0, s>>>(ctx->red.ptr, nb, 2, sc_dev + slot, nullptr);
    };
    gram_matvec(ctx, sc, n, q0, p, Kd, scratch, lists, s);  // K p0 (warm start)
    k_cg_init<<<nblk(m), 256, 0, s>>>(u, Kd, m, r, d);
    dot(r, r, 0);
    dot(u, u, 3);
    GS_CUDA(cudaMemcpyAsync(ctx->scal_host, sc_dev, 4 * sizeof(double), cudaMemcpyDeviceToHost, s));
    GS_CUDA(cudaStreamSynchronize(s));
    const double unorm = std::sqrt(ctx->scal_host[3]);
    double rr = ctx->scal_host[0];
    int it = 0;
    while (it < max_it && std::sqrt(rr) > tol * unorm && rr > 0.0) {
        gram_matvec(ctx, sc, n, q0, d, Kd, scratch, lists, s);
        dot(d, Kd, 1);
        k_cg_step<<<nblk(m), 256, 0, s>>>(sc_dev, d, Kd, m, p, r);
        dot(r, r, 2);
        k_cg_dir<<<nblk(m), 256, 0, s>>>(sc_dev, r, m, d);
        GS_CUDA(cudaMemcpyAsync(ctx->scal_host, sc_dev, 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
        GS_CUDA(cudaMemcpyAsync(sc_dev, sc_dev + 2, sizeof(double), cudaMemcpyDeviceToDevice, s));  // rr <- rr new
        GS_CUDA(cudaStreamSynchronize(s));
        const double alpha = ctx->scal_host[0] / ctx->scal_host[1], beta = ctx->scal_host[2] / ctx->scal_host[0];
        if (coef) { coef[2 * it] = alpha; coef[2 * it + 1] = beta; }
        rr = ctx->scal_host[2];
        ctx->launches += 8;
        ++it;
        if (!(ctx->scal_host[1] > 0.0)) break;  // K not positive definite along d (or a NaN)
    }
    *iters = it;
    *relres = unorm > 0.0 ? std::sqrt(rr) / unorm : 0.0;
    ctx->verlet_call = 0;
    gs_status_t st;
    rc = fetch_status(ctx, s, n, &st);
    if (rc == GS_ERR_COINCIDENT) return fail(rc, "coincident points: the Gram matrix is singular");
    if (rc == GS_ERR_CUDA) return rc;
    if ((rc = take_cell_err(ctx))) return rc;
    return GS_OK;
}

// ---- stage API ------------------------------------------------------------------------
int gs_stage_begin(gs_context* ctx, int64_t n, const double* q, const double* p, int64_t row0, int64_t row1,
                   void* stream) {
    gsapi::NvtxScope nvtx_("gs_stage_begin");
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || !q || !p || n < 1 || row0 < 0 || row1 > n || row0 > row1) return fail(GS_ERR_INVALID, "bad stage args");
    GS_CUDA(cudaSetDevice(ctx->device));
    int rc = ensure_session(ctx, n, row1 - row0);
    if (rc) return rc;
    ctx->n = n; ctx->row0 = row0; ctx->row1 = row1;
    k_status_reset<<<1, 1, 0, s>>>(ctx->st.ptr);
    GS_CUDA(cudaMemsetAsync(ctx->S.ptr + n, 0, kStatePad * sizeof(double4), s));
    k_pack<<<nblk(n), 256, 0, s>>>(q, p, n, ctx->S.ptr, ctx->st.ptr, 0);
    if (row1 > row0) k_copy_rows<<<nblk(row1 - row0), 256, 0, s>>>(ctx->S.ptr, row0, row1 - row0, ctx->B.ptr);
    GS_CUDA(cudaGetLastError());
    return GS_OK;
}

int gs_stage_run(gs_context* ctx, const gs_system_t* sys, int32_t step, int32_t stg, double dt, void* stream) {
    gsapi::NvtxScope nvtx_("gs_stage_run");
    if (!ctx || ctx->n < 1) return fail(GS_ERR_INVALID, "no stage session");
    int rc = check_system(sys);
    if (rc) return rc;
    if (stg < 0 || stg > 3 || step < 1) return fail(GS_ERR_INVALID, "bad stage index");
    if (step == 1 && stg == 0 && (rc = choose_path(ctx, sys, ctx->S.ptr, ctx->n, (cudaStream_t)stream))) return rc;
    stage(ctx, make_const(sys), step, stg, dt, (cudaStream_t)stream);
    GS_CUDA(cudaGetLastError());
    return take_cell_err(ctx);
}

double* gs_stage_state(gs_context* ctx) { return ctx ? reinterpret_cast<double*>(ctx->S.ptr) : nullptr; }

int gs_stage_end(gs_context* ctx, double* q_rows, double* p_rows, void* stream) {
    gsapi::NvtxScope nvtx_("gs_stage_end");
    if (!ctx || !q_rows) return fail(GS_ERR_INVALID, "bad stage args");
    const int64_t nrows = ctx->row1 - ctx->row0;
    if (nrows > 0) k_unpack<<<nblk(nrows), 256, 0, (cudaStream_t)stream>>>(ctx->B.ptr, nrows, q_rows, p_rows);
    GS_CUDA(cudaGetLastError());
    return GS_OK;
}

int gs_gram(gs_context* ctx, const gs_system_t* sys, int64_t n, const double* q, double* K, int64_t* bad_i,
            int64_t* bad_j, void* stream) {
    gsapi::NvtxScope nvtx_("gs_gram");
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || !q || !K || !bad_i || !bad_j || n < 1) return fail(GS_ERR_INVALID, "bad gram args");
    int rc = check_system(sys);
    if (rc) return rc;
    GS_CUDA(cudaSetDevice(ctx->device));
    GS_CUDA(ctx->gram_bad.ensure(1));
    unsigned long long key = kNoEvent;
    GS_CUDA(cudaMemsetAsync(ctx->gram_bad.ptr, 0xff, sizeof(key), s));
    launch_gram(make_const(sys), q, n, K, ctx->gram_bad.ptr, ctx->tbl.ptr, s);
    ctx->launches++;
    GS_CUDA(cudaGetLastError());
    GS_CUDA(cudaMemcpyAsync(&key, ctx->gram_bad.ptr, sizeof(key), cudaMemcpyDeviceToHost, s));
    GS_CUDA(cudaStreamSynchronize(s));
    *bad_i = key == kNoEvent ? -1 : (int64_t)(key / (unsigned long long)n);
    *bad_j = key == kNoEvent ? -1 : (int64_t)(key % (unsigned long long)n);
    return key == kNoEvent ? GS_OK : GS_ERR_COINCIDENT;
}

int gs_velocity_field(gs_context* ctx, const gs_system_t* sys, int64_t n, const double* q, const double* p,
                      int64_t m, const double* x, double* u, void* stream) {
    gsapi::NvtxScope nvtx_("gs_velocity_field");
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || !q || !p || !x || !u || n < 1 || m < 0) return fail(GS_ERR_INVALID, "bad velocity-field args");
    int rc = check_system(sys);
    if (rc) return rc;
    if (m == 0) return GS_OK;
    GS_CUDA(cudaSetDevice(ctx->device));
    GS_CUDA(ctx->S.ensure(n + kStatePad));
    const DensePlan plan = velocity_plan(n, m, ctx->sm_count);
    GS_CUDA(ctx->vf_part.ensure((size_t)plan.nchunks * m));
    k_pack<<<nblk(n), 256, 0, s>>>(q, p, n, ctx->S.ptr, ctx->st.ptr, 0);
    launch_velocity_field(make_const(sys), ctx->S.ptr, n, x, m, plan, ctx->vf_part.ptr, u, ctx->tbl.ptr, s);
    ctx->launches += 3;
    ctx->host_pairs += n * m;
    GS_CUDA(cudaGetLastError());
    return GS_OK;
}

int gs_stage_path(gs_context* ctx, const gs_system_t* sys, void* stream) {
    if (!ctx || ctx->n < 1) return -fail(GS_ERR_INVALID, "no stage session");
    int rc = check_system(sys);
    if (rc) return -rc;
    if ((rc = choose_path(ctx, sys, ctx->S.ptr, ctx->n, (cudaStream_t)stream))) return -rc;
    return ctx->cell_on ? GS_PATH_CELL : GS_PATH_DENSE;
}

int64_t gs_sym_parts(int64_t n) {
    const SymPlan p = sym_plan(n);
    return (p.ok && n >= kSymSplitMinN) ? (int64_t)sym_ctas(n) : 0;
}

int gs_stage_pairs_sym(gs_context* ctx, const gs_system_t* sys, int32_t step, int32_t stg, int64_t part_begin,
                       int64_t part_end, double* R, void* stream) {
    gsapi::NvtxScope nvtx_("gs_stage_pairs_sym");
    return pairs_sym_impl(ctx, sys, step, stg, part_begin, part_end, R, stream);
}

int gs_stage_finish(gs_context* ctx, const gs_system_t* sys, int32_t step, int32_t stg, double dt,
                    const double* R_rows, void* stream) {
    gsapi::NvtxScope nvtx_("gs_stage_finish");
    if (!ctx || ctx->n < 1) return fail(GS_ERR_INVALID, "no stage session");
    int rc = check_system(sys);
    if (rc) return rc;
    if (stg < 0 || stg > 3 || step < 1) return fail(GS_ERR_INVALID, "bad stage index");
    const int64_t nrows = ctx->row1 - ctx->row0;
    if (nrows > 0 && !R_rows) return fail(GS_ERR_INVALID, "R_rows is NULL");
    FinishArgs fa{};
    fa.part = reinterpret_cast<const double4*>(R_rows); fa.nchunks = 1; fa.pstride = 0; fa.nrows = nrows;
    fa.row0 = ctx->row0; fa.S = ctx->S.ptr; fa.B = ctx->B.ptr; fa.A = ctx->A.ptr; fa.stage = stg; fa.dt = dt;
    fa.st = ctx->st.ptr;
    fa.event = (unsigned long long)step * 8ull + 2ull * (unsigned long long)stg + 1ull;
    launch_finish(kFinStage, make_const(sys), fa, (cudaStream_t)stream);
    ctx->launches++;
    GS_CUDA(cudaGetLastError());
    return GS_OK;
}

int gs_profile_enable(gs_context* ctx, int32_t on) {
    if (!ctx) return fail(GS_ERR_INVALID, "ctx is NULL");
    ctx->prof_on = on ? 1 : 0;
    ctx->prof_used = 0;
    return GS_OK;
}

int gs_profile_read(gs_context* ctx, double* pair_ms, int64_t* pair_launches, int64_t* launches, int64_t* pairs,
                    int32_t reset) {
    if (!ctx || !pair_ms || !pair_launches || !launches || !pairs) return fail(GS_ERR_INVALID, "NULL argument");
    unsigned long long acc = 0;
    if (ctx->c_acc.ptr) {
        GS_CUDA(cudaMemcpy(&acc, ctx->c_acc.ptr, sizeof(acc), cudaMemcpyDeviceToHost));
        if (reset) GS_CUDA(cudaMemset(ctx->c_acc.ptr, 0, sizeof(acc)));
    }
    *pairs = (int64_t)acc + ctx->host_pairs;
    if (reset) ctx->host_pairs = 0;
    double total = ctx->prof_ms_acc;
    if (ctx->prof_used >= 2) {
        GS_CUDA(cudaEventSynchronize(ctx->prof_events[ctx->prof_used - 1]));
        for (size_t k = 0; k + 1 < ctx->prof_used; k += 2) {
            float t = 0.f;
            GS_CUDA(cudaEventElapsedTime(&t, ctx->prof_events[k], ctx->prof_events[k + 1]));
            total += t;
        }
    }
    *pair_ms = total;
    *pair_launches = ctx->pair_launches;
    *launches = ctx->launches;
    if (reset) {
        ctx->prof_ms_acc = 0.0;
        ctx->prof_used = 0;
        ctx->pair_launches = 0;
        ctx->launches = 0;
    }
    return GS_OK;
}

int gs_fp64_peak_probe(gs_context* ctx, int32_t iters, double* ms, double* flops, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || !ms || !flops || iters < 1) return fail(GS_ERR_INVALID, "bad probe args");
    GS_CUDA(cudaSetDevice(ctx->device));
    const int blocks = ctx->sm_count * 8, threads = 256;
    cudaEvent_t e0, e1;
    GS_CUDA(cudaEventCreate(&e0));
    GS_CUDA(cudaEventCreate(&e1));
    k_fp64_probe<<<blocks, threads, 0, s>>>(ctx->scal.ptr, iters);  // warm-up
    GS_CUDA(cudaEventRecord(e0, s));
    k_fp64_probe<<<blocks, threads, 0, s>>>(ctx->scal.ptr, iters);
    GS_CUDA(cudaEventRecord(e1, s));
    GS_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    cudaEventElapsedTime(&t, e0, e1);
    *ms = t;
    *flops = 2.0 * 8.0 * (double)iters * blocks * threads;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return GS_OK;
}

}  // extern "C"


// gs_batch.cu — batched independent trajectories of the C ABI:
// gs_match_batch / gs_evolve_batch (include/geoshoot_b200.h).
#include "gs_context.cuh"

using namespace gsb;
using namespace gsapi;

extern "C" {

// ---- batched trajectories --------------------------------------------
// One CTA per item of a persistent small-N launch: convergence-sweep cells, cluster-test
// pairs, exact-vs-inexact rows (gs_match_batch) and Newton Jacobian columns (gs_evolve_batch)
// run side by side instead of one after another.  Above kSmallMax (or on the cell path) the
// items run one after another through the general path.
namespace {

constexpr size_t kSmemBudget = 200 * 1024;  // dynamic shared memory one CTA may claim (227 KB - k_small's static)

int upload_items(gs_context* ctx, const std::vector<SmallItem>& items, cudaStream_t s) {
    GS_CUDA(ctx->b_items.ensure(items.size()));
    GS_CUDA(cudaMemcpyAsync(ctx->b_items.ptr, items.data(), items.size() * sizeof(SmallItem), cudaMemcpyHostToDevice,
                            s));
    return GS_OK;
}

}  // namespace

int gs_match_batch(gs_context* ctx, const gs_batch_item_t* items, int64_t batch, int64_t n, const double* q0,
                   int64_t q0_stride, const double* target, int64_t target_stride, const double* gram_factor,
                   int64_t factor_stride, double* p0_out, double* endpoint_out, double* history_out,
                   int64_t history_stride, gs_match_result_t* results, void* stream) {
    gsapi::NvtxScope nvtx_("gs_match_batch");
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || !items || !results || !history_out) return fail(GS_ERR_INVALID, "NULL argument");
    if (batch < 1) return fail(GS_ERR_INVALID, "batch must be >= 1");
    if (n < 1 || !q0 || !target || !p0_out || !endpoint_out)
        return fail(GS_ERR_INVALID, "templates must have shape (N, 2), N >= 1");
    if (q0_stride < 0 || target_stride < 0 || factor_stride < 0)
        return fail(GS_ERR_INVALID, "strides must be >= 0");
    bool small = n <= kSmallMax;
    std::vector<SmallItem> host_items((size_t)batch);
    for (int64_t b = 0; b < batch; ++b) {
        int rc = check_match(&items[b].system, &items[b].config);
        if (rc) return fail(rc, "item " + std::to_string(b) + ": " + g_last_error);
        if (items[b].system.family != items[0].system.family)
            return fail(GS_ERR_INVALID, "all items of a batch must use the same kernel family");
        if (history_stride < items[b].config.max_iter)
            return fail(GS_ERR_INVALID, "history_stride must be >= every item's max_iter");
        small = small && use_small(&items[b].system, n);
        host_items[b] = small_item(make_const(&items[b].system), &items[b].config);
    }
    GS_CUDA(cudaSetDevice(ctx->device));
    cudaEvent_t e0, e1;
    GS_CUDA(cudaEventCreate(&e0));
    GS_CUDA(cudaEventCreate(&e1));
    GS_CUDA(cudaEventRecord(e0, s));
    if (small) {
        int rc = upload_items(ctx, host_items, s);
        if (rc) return rc;
        GS_CUDA(ctx->small_res.ensure(batch));
        SmallArgs a{};
        small_setup(a, n); a.batch = batch; a.mode = 1;
        a.item = host_items[0]; a.items = ctx->b_items.ptr;
        a.q_in = q0; a.q_stride = q0_stride; a.target = target; a.t_stride = target_stride;
        a.q_out = endpoint_out; a.p_out = p0_out;
        a.history = history_out; a.hist_stride = history_stride; a.result = ctx->small_res.ptr;
        a.L = gram_factor; a.L_stride = factor_stride;
        if (gram_factor) {
            a.L_smem = 1;
            if (small_smem_bytes(a) > kSmemBudget) a.L_smem = 0;
        }
        if (ctx->prof_on) cudaEventRecord(prof_event(ctx), s);
        GS_CUDA((cudaError_t)launch_small(items[0].system.family, a, ctx->tbl.ptr, s));
        if (ctx->prof_on) cudaEventRecord(prof_event(ctx), s);
        ctx->launches++;
        ctx->pair_launches++;
        GS_CUDA(cudaEventRecord(e1, s));
        std::vector<SmallResult> r((size_t)batch);
        GS_CUDA(cudaMemcpyAsync(r.data(), ctx->small_res.ptr, batch * sizeof(SmallResult), cudaMemcpyDeviceToHost, s));
        GS_CUDA(cudaStreamSynchronize(s));
        for (int64_t b = 0; b < batch; ++b) {
            small_to_result(r[b], n, &results[b]);
            ctx->host_pairs += (long long)(r[b].iterations + (r[b].outcome == GS_MATCH_EVOLVE_FAILED)) * 4LL *
                                   items[b].config.steps * n * n + n * n;
        }
    } else {
        if (gram_factor)
            return fail(GS_ERR_UNSUPPORTED, "velocity-space batches need N <= 512 on the dense path");
        std::vector<double> hist((size_t)history_stride);
        for (int64_t b = 0; b < batch; ++b) {
            int rc = gs_match(ctx, &items[b].system, &items[b].config, n, q0 + b * q0_stride,
                              target + b * target_stride, p0_out + b * 2 * n, endpoint_out + b * 2 * n, hist.data(),
                              &results[b], stream);
            if (rc) return fail(rc, "item " + std::to_string(b) + ": " + g_last_error);
            if (results[b].iterations > 0)
                GS_CUDA(cudaMemcpyAsync(history_out + b * history_stride, hist.data(),
                                        results[b].iterations * sizeof(double), cudaMemcpyHostToDevice, s));
        }
        GS_CUDA(cudaEventRecord(e1, s));
    }
    GS_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    for (int64_t b = 0; b < batch; ++b) results[b].seconds_device = ms * 1e-3;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return GS_OK;
}

int gs_evolve_batch(gs_context* ctx, const gs_system_t* sys, int64_t batch, int64_t n, double t_final, int32_t steps,
                    const double* q_in, int64_t q_stride, double* q_out, double* p_io, gs_status_t* status,
                    void* stream) {
    gsapi::NvtxScope nvtx_("gs_evolve_batch");
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || !status) return fail(GS_ERR_INVALID, "NULL argument");
    int rc = check_system(sys);
    if (rc) return rc;
    if (batch < 1) return fail(GS_ERR_INVALID, "batch must be >= 1");
    if (n < 1 || !q_in || !q_out || !p_io) return fail(GS_ERR_INVALID, "q and p must have shape (N, 2), N >= 1");
    if (q_stride < 0) return fail(GS_ERR_INVALID, "q_stride must be >= 0");
    if (!(t_final > 0.0) || !std::isfinite(t_final)) return fail(GS_ERR_INVALID, "t_final must be positive");
    if (steps < 1) return fail(GS_ERR_INVALID, "steps must be >= 1");
    GS_CUDA(cudaSetDevice(ctx->device));
    const SysConst sc = make_const(sys);
    if (use_small(sys, n)) {
        GS_CUDA(ctx->b_st.ensure(batch));
        SmallArgs a{};
        small_setup(a, n); a.batch = batch; a.mode = 0;
        a.item.sc = sc; a.item.t_final = t_final; a.item.steps = steps;
        a.q_in = q_in; a.q_stride = q_stride; a.p_in = p_io; a.q_out = q_out; a.p_out = p_io;
        a.st = ctx->b_st.ptr;
        ctx->host_pairs += 4LL * steps * n * n * batch;
        if (ctx->prof_on) cudaEventRecord(prof_event(ctx), s);
        GS_CUDA((cudaError_t)launch_small(sc.fam, a, ctx->tbl.ptr, s));
        if (ctx->prof_on) cudaEventRecord(prof_event(ctx), s);
        ctx->launches++;
        ctx->pair_launches++;
        std::vector<DevStatus> d((size_t)batch);
        GS_CUDA(cudaMemcpyAsync(d.data(), ctx->b_st.ptr, batch * sizeof(DevStatus), cudaMemcpyDeviceToHost, s));
        GS_CUDA(cudaStreamSynchronize(s));
        for (int64_t b = 0; b < batch; ++b) decode_status(d[b], n, &status[b]);
        return GS_OK;
    }
    for (int64_t b = 0; b < batch; ++b) {
        GS_CUDA(cudaMemcpyAsync(q_out + b * 2 * n, q_in + b * q_stride, 2 * n * sizeof(double),
                                cudaMemcpyDeviceToDevice, s));
        rc = gs_evolve(ctx, sys, n, t_final, steps, 0, q_out + b * 2 * n, p_io + b * 2 * n, nullptr, &status[b],
                       stream);
        if (rc == GS_ERR_CUDA || rc == GS_ERR_INVALID || rc == GS_ERR_UNSUPPORTED) return rc;
    }
    return GS_OK;
}

}  // extern "C"

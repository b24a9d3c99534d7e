// gs_p2p.cu — the multi-GPU stage exchange over peer memory (gs_p2p_*, include/geoshoot_b200.h).
#include "gs_context.cuh"

using namespace gsb;
using namespace gsapi;

extern "C" {

// ---- fused stage exchange over peer memory (multi-GPU, symmetric split) -----------------
// Per stage: [wait: previous stage's records from all ranks] -> this rank's superblock pairs ->
// raw row sums into R -> signal "sums ready" to every rank -> wait for all ranks' signals ->
// epilogue of this rank's rows reading every rank's R and storing the new records into every
// rank's S (k_finish_p2p) -> signal "records written".  Counters only grow (targets are
// multiples of the world size), waits give up after a timeout and count it (gs_p2p_timeouts),
// so a lost signal costs a timeout, never a hang.
namespace {

__global__ void k_p2p_wait(unsigned long long* flags, int which, unsigned long long target, long long timeout_ns) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (*((volatile unsigned long long*)&flags[which]) < target &&
           *((volatile unsigned long long*)&flags[2]) == 0) {  // after one timeout nobody waits
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if ((long long)(t - t0) > timeout_ns) {
            atomicAdd(&flags[2], 1ull);
            break;
        }
        __nanosleep(256);
    }
    __threadfence_system();
}

}  // namespace

int gs_p2p_local(gs_context* ctx, int64_t rows_all, void** S, void** R, void** flags) {
    if (!ctx || ctx->n < 1 || !S || !R || !flags) return fail(GS_ERR_INVALID, "no stage session");
    if (rows_all < ctx->n) return fail(GS_ERR_INVALID, "rows_all < n");
    GS_CUDA(cudaSetDevice(ctx->device));
    GS_CUDA(ctx->p2p.R.ensure(rows_all));
    GS_CUDA(ctx->p2p.flags.ensure(4));
    GS_CUDA(cudaMemset(ctx->p2p.flags.ptr, 0, 4 * sizeof(unsigned long long)));
    GS_CUDA(ctx->p2p.done.ensure(2));
    GS_CUDA(cudaMemset(ctx->p2p.done.ptr, 0, 2 * sizeof(unsigned)));
    *S = ctx->S.ptr; *R = ctx->p2p.R.ptr; *flags = ctx->p2p.flags.ptr;
    if (const char* e = std::getenv("GS_B200_P2P_TIMEOUT_S")) ctx->p2p.timeout_ns = (long long)(std::atof(e) * 1e9);
    return GS_OK;
}

int gs_p2p_export(gs_context* ctx, int64_t rows_all, void* handles) {
    if (!handles) return fail(GS_ERR_INVALID, "handles is NULL");
    void* ptr[3];
    int rc = gs_p2p_local(ctx, rows_all, &ptr[0], &ptr[1], &ptr[2]);
    if (rc) return rc;
    for (int k = 0; k < 3; ++k)
        GS_CUDA(cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(handles) + k, ptr[k]));
    return GS_OK;
}

int gs_p2p_set_peers(gs_context* ctx, int world, int rank, void* const* S, void* const* R, void* const* F) {
    if (!ctx || world < 1 || world > 32 || rank < 0 || rank >= world || !S || !R || !F)
        return fail(GS_ERR_INVALID, "bad peer set");
    GS_CUDA(cudaSetDevice(ctx->device));
    GS_CUDA(ctx->p2p.Sp.ensure(world));
    GS_CUDA(ctx->p2p.Rp.ensure(world));
    GS_CUDA(ctx->p2p.Fp.ensure(world));
    GS_CUDA(cudaMemcpy(ctx->p2p.Sp.ptr, S, world * sizeof(void*), cudaMemcpyHostToDevice));
    GS_CUDA(cudaMemcpy(ctx->p2p.Rp.ptr, R, world * sizeof(void*), cudaMemcpyHostToDevice));
    GS_CUDA(cudaMemcpy(ctx->p2p.Fp.ptr, F, world * sizeof(void*), cudaMemcpyHostToDevice));
    ctx->p2p.world = world; ctx->p2p.rank = rank; ctx->p2p.epoch = 0;
    return GS_OK;
}

int gs_p2p_close(gs_context* ctx) {
    if (!ctx) return fail(GS_ERR_INVALID, "ctx is NULL");
    cudaSetDevice(ctx->device);
    for (void* p : ctx->p2p.opened) cudaIpcCloseMemHandle(p);
    ctx->p2p.opened.clear();
    ctx->p2p.world = 0;
    return GS_OK;
}

int gs_p2p_import(gs_context* ctx, int world, int rank, const void* handles_all) {
    if (!ctx || !handles_all || world < 1 || world > 32 || rank < 0 || rank >= world)
        return fail(GS_ERR_INVALID, "bad peer import");
    GS_CUDA(cudaSetDevice(ctx->device));
    gs_p2p_close(ctx);
    const cudaIpcMemHandle_t* h = reinterpret_cast<const cudaIpcMemHandle_t*>(handles_all);
    std::vector<void*> S(world), R(world), F(world);
    for (int w = 0; w < world; ++w) {
        void** dst[3] = {&S[w], &R[w], &F[w]};
        if (w == rank) {
            S[w] = ctx->S.ptr; R[w] = ctx->p2p.R.ptr; F[w] = ctx->p2p.flags.ptr;
            continue;
        }
        for (int k = 0; k < 3; ++k) {
            GS_CUDA(cudaIpcOpenMemHandle(dst[k], h[3 * w + k], cudaIpcMemLazyEnablePeerAccess));
            ctx->p2p.opened.push_back(*dst[k]);
        }
    }
    return gs_p2p_set_peers(ctx, world, rank, S.data(), R.data(), F.data());
}

int gs_p2p_pairs(gs_context* ctx, const gs_system_t* sys, int32_t step, int32_t stg, int64_t part_begin,
                 int64_t part_end, void* stream) {
    gsapi::NvtxScope nvtx_("gs_p2p_pairs");
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || ctx->p2p.world < 1) return fail(GS_ERR_INVALID, "no peers (gs_p2p_import / gs_p2p_set_peers)");
    GS_CUDA(cudaSetDevice(ctx->device));
    {
        auto& P = ctx->p2p;
        // one waiting thread for every rank's records of the previous stage (waiting in each of
        // the pair kernel's thousands of CTAs cost more: 164.8 vs 159.5 ms per C2 solve), then
        // the pairs; the slot reduction's last CTA signals "sums ready" to every rank
        if (P.epoch > 0) {
            k_p2p_wait<<<1, 1, 0, s>>>(P.flags.ptr, 1, P.epoch * (unsigned long long)P.world, P.timeout_ns);
            ctx->launches++;
        }
        int rc = pairs_sym_impl(ctx, sys, step, stg, part_begin, part_end, reinterpret_cast<double*>(P.R.ptr), stream,
                                PeerSignal{P.Fp.ptr, P.world, 0, P.done.ptr});
        if (rc) return rc;
    }
    GS_CUDA(cudaGetLastError());
    return GS_OK;
}

int gs_p2p_finish(gs_context* ctx, const gs_system_t* sys, int32_t step, int32_t stg, double dt, void* stream) {
    gsapi::NvtxScope nvtx_("gs_p2p_finish");
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || ctx->p2p.world < 1) return fail(GS_ERR_INVALID, "no peers (gs_p2p_import / gs_p2p_set_peers)");
    int rc = check_system(sys);
    if (rc) return rc;
    if (stg < 0 || stg > 3 || step < 1) return fail(GS_ERR_INVALID, "bad stage index");
    GS_CUDA(cudaSetDevice(ctx->device));
    auto& P = ctx->p2p;
    FinishArgs fa{};
    fa.nrows = ctx->row1 - ctx->row0; fa.row0 = ctx->row0;
    fa.S = ctx->S.ptr; fa.B = ctx->B.ptr; fa.A = ctx->A.ptr; fa.stage = stg; fa.dt = dt; fa.st = ctx->st.ptr;
    fa.event = (unsigned long long)step * 8ull + 2ull * (unsigned long long)stg + 1ull;
    // waits (every CTA) for all ranks' "sums ready", its last CTA signals "records written"
    launch_finish_p2p(make_const(sys), fa, P.Rp.ptr, P.Sp.ptr, P.world,
                      PeerWait{P.flags.ptr, 0, (P.epoch + 1) * (unsigned long long)P.world, P.timeout_ns},
                      PeerSignal{P.Fp.ptr, P.world, 1, P.done.ptr + 1}, s);
    P.epoch++;
    ctx->launches++;
    GS_CUDA(cudaGetLastError());
    return GS_OK;
}

int gs_p2p_sync(gs_context* ctx, void* stream) {
    if (!ctx || ctx->p2p.world < 1) return fail(GS_ERR_INVALID, "no peers");
    GS_CUDA(cudaSetDevice(ctx->device));
    auto& P = ctx->p2p;
    k_p2p_wait<<<1, 1, 0, (cudaStream_t)stream>>>(P.flags.ptr, 1, P.epoch * (unsigned long long)P.world,
                                                   P.timeout_ns);
    GS_CUDA(cudaGetLastError());
    return GS_OK;
}

int gs_p2p_timeouts(gs_context* ctx, int64_t* out) {
    if (!ctx || !out) return fail(GS_ERR_INVALID, "NULL argument");
    unsigned long long v = 0;
    if (ctx->p2p.flags.ptr) {
        GS_CUDA(cudaSetDevice(ctx->device));
        GS_CUDA(cudaMemcpy(&v, ctx->p2p.flags.ptr + 2, sizeof(v), cudaMemcpyDeviceToHost));
    }
    *out = (int64_t)v;
    return GS_OK;
}

}  // extern "C"

// gs_slab.cu — slab decomposition of the cell-list path across ranks (gs_slab_*, include/geoshoot_b200.h).
//
// SURVEY.md §8(e) for the compactly supported kernel (KD-1): the RHS of row i only needs the
// particles within the support radius (particles.py:109-117 restricted as in gs_verlet.cu), so a
// rank needs its own particles and a halo, not the whole state.  Ownership is spatial: at every
// list build the cell rows of the global grid (the grid the one-GPU build would use, derived by
// every rank from the all-reduced bounding box) are split into W contiguous slabs of balanced
// particle counts (from an all-reduced row histogram).  A rank holds
//
//     local rows [y_loc0, y_loc1) = its own rows [y_own0, y_own1) + `sub` halo rows on each side
//
// in GLOBAL sorted order (cell key, then global index): the halo rows come as contiguous slices
// of the neighbours' own blocks, so the layout needs no permutation after the exchange.  Own
// particles form clusters of two that restart at every cell row, their lists are built over the
// local particles, and the sweep + RK4 stage epilogue run over the own particles only, in local
// order (coalesced).  Between builds a stage exchanges only the halo slices (32 B per halo
// particle); a build migrates the particles whose row changed owner (with their RK4 base and
// accumulator, 104 B each).
//
// Row sums are bitwise independent of the number of ranks: a cluster's members, its list (the
// candidates of its stencil rows in global sorted order, every one of them local) and the lane
// split (from the global N) are those of the one-rank slab build.  The collectives (all-reduce
// of the box, the histogram and the rebuild flag; the migration all-to-all; the halo slices) are
// issued by the host driver (paper_1510_03816_b200/slab.py) through torch.distributed.
#include <cub/cub.cuh>

#include "gs_context.cuh"

using namespace gsb;
using namespace gsapi;

namespace {

constexpr int kPackW = 13;  // doubles per migrating particle: S (4), B (4), A (4), global index

// Per-build buffers grow with 25 % headroom: counts change by a few per cent at every build
// (migration, halo, list length), and an exact-size reallocation costs a device-wide
// cudaFree + cudaMalloc inside the build.
template <typename T>
cudaError_t grow(DevBuf<T>& b, size_t n) {
    return n <= b.cap ? cudaSuccess : b.ensure(n + n / 4 + 256);
}

__device__ __forceinline__ int grid_cell(double v, double v0, double inv_h, int nmax) {
    // the cell coordinate of gs_cell.cu / gs_verlet.cu (floor, clamped to the grid)
    const int c = (int)floor((v - v0) * inv_h);
    return min(max(c, 0), nmax - 1);
}

__global__ void k_slab_begin(const double* __restrict__ q, const double* __restrict__ p,
                             const int* __restrict__ g, int64_t n, double4* Su, double4* Bu, double4* Au, unsigned* gu) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double4 v = make_double4(q[2 * i], q[2 * i + 1], p[2 * i], p[2 * i + 1]);
    Su[i] = v;
    Bu[i] = v;
    Au[i] = make_double4(0.0, 0.0, 0.0, 0.0);
    gu[i] = (unsigned)g[i];
}

// One atomic per distinct value per warp (own particles are in cell order after a layout, so a
// warp's lanes mostly share one row / one destination: per-lane atomics on a few addresses
// serialised to ~100 us at 131k particles).
__device__ __forceinline__ void warp_count(unsigned long long* ctr, int key, bool valid) {
    const unsigned act = __ballot_sync(0xffffffffu, valid);
    if (!valid) return;
    const unsigned peers = __match_any_sync(act, key);
    if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&ctr[key], (unsigned long long)__popc(peers));
}

__global__ void k_slab_rows(const double4* __restrict__ S, int64_t n, const GridParams* __restrict__ gp,
                            unsigned long long* hist) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const GridParams g = *gp;
    const bool valid = i < n;
    warp_count(hist, valid ? grid_cell(S[i].y, g.y0, g.inv_h, g.ny) : 0, valid);
}

// destination rank of every own particle: the owner of its cell row
__global__ void k_slab_dest(const double4* __restrict__ S, int64_t n, const GridParams* __restrict__ gp,
                            const int* __restrict__ owner, unsigned long long* key, unsigned* val,
                            unsigned long long* count) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const GridParams g = *gp;
    const bool valid = i < n;
    const int d = valid ? owner[grid_cell(S[i].y, g.y0, g.inv_h, g.ny)] : 0;
    if (valid) {
        key[i] = (unsigned long long)d;
        val[i] = (unsigned)i;
    }
    warp_count(count, d, valid);
}

__global__ void k_slab_pack(const unsigned* __restrict__ order, int64_t n, const double4* __restrict__ S,
                            const double4* __restrict__ B, const double4* __restrict__ A,
                            const unsigned* __restrict__ g, double* send) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const unsigned i = order[j];
    const double4 s = S[i], b = B[i], a = A[i];
    double* o = send + (int64_t)kPackW * j;
    o[0] = s.x; o[1] = s.y; o[2] = s.z; o[3] = s.w;
    o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
    o[8] = a.x; o[9] = a.y; o[10] = a.z; o[11] = a.w;
    o[12] = (double)g[i];
}

__global__ void k_slab_unpack(const double* __restrict__ recv, int64_t n, double4* Su, double4* Bu, double4* Au,
                              unsigned* gu) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const double* o = recv + (int64_t)kPackW * j;
    Su[j] = make_double4(o[0], o[1], o[2], o[3]);
    Bu[j] = make_double4(o[4], o[5], o[6], o[7]);
    Au[j] = make_double4(o[8], o[9], o[10], o[11]);
    gu[j] = (unsigned)o[12];
}

// (cell within the own rows, global index): the one-rank build's sorted order restricted to the rank
__global__ void k_slab_own_keys(const double4* __restrict__ S, const unsigned* __restrict__ g, int64_t n,
                                const GridParams* __restrict__ gp, int y_own0, int gbits, unsigned long long* key,
                                unsigned* val) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const GridParams G = *gp;
    const double4 v = S[i];
    const int cy = grid_cell(v.y, G.y0, G.inv_h, G.ny), cx = grid_cell(v.x, G.x0, G.inv_h, G.nx);
    GS_ASSERT(cy >= y_own0);
    const unsigned sub = cell_subkey((v.x - G.x0) * G.inv_h - (double)cx, (v.y - G.y0) * G.inv_h - (double)cy);
    const unsigned long long cell = ((unsigned long long)((int64_t)(cy - y_own0) * G.nx + cx) << GS_CELL_SUBKEY) | sub;
    key[i] = (cell << gbits) | (unsigned long long)g[i];
    val[i] = (unsigned)i;
}

__global__ void k_slab_place(const unsigned* __restrict__ order, int64_t n, const double4* __restrict__ Su,
                             const double4* __restrict__ Bu, const double4* __restrict__ Au,
                             const unsigned* __restrict__ gu, double4* S, double4* B, double4* A, unsigned* g) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const unsigned i = order[k];
    S[k] = Su[i];
    B[k] = Bu[i];
    A[k] = Au[i];
    g[k] = gu[i];
}

// local cell keys (rows from ylo) of the local records; they are sorted by construction
__global__ void k_slab_local_keys(const double4* __restrict__ S, int64_t n, const GridParams* __restrict__ gp,
                                  unsigned* keys, float2* Sf) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const GridParams G = *gp;
    const double4 v = S[k];
    const int cy = grid_cell(v.y, G.y0, G.inv_h, G.ny), cx = grid_cell(v.x, G.x0, G.inv_h, G.nx);
    GS_ASSERT(cy >= G.ylo && cy < G.yhi);
    const unsigned sub = cell_subkey((v.x - G.x0) * G.inv_h - (double)cx, (v.y - G.y0) * G.inv_h - (double)cy);
    keys[k] = ((unsigned)((cy - G.ylo) * G.nx + cx) << GS_CELL_SUBKEY) | sub;
    Sf[k] = make_float2((float)(v.x - G.x0), (float)(v.y - G.y0));
}

// start[c] = first local position with cell >= c, c in [0, ncells] (cell = key above the sub-cell bits)
__global__ void k_slab_start(const unsigned* __restrict__ keys, int64_t n, int64_t ncells, int* start) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k > n) return;
    const long long prev = (k == 0) ? -1 : (long long)(keys[k - 1] >> GS_CELL_SUBKEY);
    const long long cur = (k == n) ? ncells : (long long)(keys[k] >> GS_CELL_SUBKEY);
    GS_ASSERT(cur >= prev && cur <= ncells);
    for (long long c = prev + 1; c <= cur; ++c) start[c] = (int)k;
}

// cluster heads of the own particles: pairs restart at every cell row
__global__ void k_slab_heads(const unsigned* __restrict__ keys, const int* __restrict__ start, int64_t own_begin,
                             int64_t n_own, int nx, int* head) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k > n_own) return;
    if (k == n_own) { head[k] = 0; return; }
    const int64_t pos = own_begin + k;
    const int row = (int)((keys[pos] >> GS_CELL_SUBKEY) / (unsigned)nx);
    head[k] = ((pos - start[(int64_t)row * nx]) % 2) == 0 ? 1 : 0;
}

__global__ void k_slab_cfirst(const int* __restrict__ head, const int* __restrict__ cid, int64_t own_begin,
                              int64_t n_own, int* cfirst, int ncl) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k > n_own) return;
    GS_ASSERT(cid[n_own] == ncl);
    if (k == n_own) cfirst[cid[k]] = (int)(own_begin + n_own);
    else if (head[k]) cfirst[cid[k]] = (int)(own_begin + k);
}

__global__ void k_slab_sentinel(double4* S, double4* S2, int64_t n_loc, long long* cnt, int64_t ncl) {
    S[n_loc] = far_record(0);
    S2[n_loc] = far_record(0);
    cnt[ncl] = 0;
}

__global__ void k_slab_status_reset(DevStatus* st) {
    st->first_event = kNoEvent;
    st->pair_key = kNoEvent;
}

inline unsigned blk(int64_t n) { return (unsigned)((n + 255) / 256); }

int bits_for(int64_t v) {  // smallest b with 2^b > v
    int b = 0;
    while (b < 63 && (1ll << b) <= v) ++b;
    return b;
}

double4* slab_cur(gs_context* ctx) { return ctx->slab.par ? ctx->slab.S2.ptr : ctx->slab.S.ptr; }

SlabLists slab_lists(gs_context* ctx) {
    auto& L = ctx->slab;
    SlabLists s;
    s.S = slab_cur(ctx); s.Sf = L.Sf.ptr; s.start = L.start.ptr; s.gp = L.gp.ptr; s.cfirst = L.cfirst.ptr;
    s.cnt = L.cnt.ptr; s.ofs = L.ofs.ptr; s.len = L.len.ptr; s.list = L.list.ptr; s.cap = (int64_t)L.list.cap;
    s.Xb = L.Xb.ptr; s.overflow = L.over.ptr; s.scan_temp = L.cub.ptr; s.scan_bytes = L.cub.cap;
    return s;
}

// the own particles' current arrays (arrival order before a layout, local order after it)
struct Own {
    const double4 *S, *B, *A;
    const unsigned* g;
};
Own own_arrays(gs_context* ctx) {
    auto& L = ctx->slab;
    if (L.own_sorted) return Own{slab_cur(ctx) + L.own_begin, L.B.ptr, L.A.ptr, L.gidx.ptr + L.own_begin};
    return Own{L.Su.ptr, L.Bu.ptr, L.Au.ptr, L.gu.ptr};
}

int ensure_own(gs_context* ctx, int64_t n) {
    auto& L = ctx->slab;
    GS_CUDA(grow(L.Su, n)); GS_CUDA(grow(L.Bu, n)); GS_CUDA(grow(L.Au, n)); GS_CUDA(grow(L.gu, n));
    GS_CUDA(grow(L.skey, n)); GS_CUDA(grow(L.skey2, n)); GS_CUDA(grow(L.sval, n)); GS_CUDA(grow(L.sval2, n));
    return GS_OK;
}

}  // namespace

extern "C" {

int gs_slab_begin(gs_context* ctx, const gs_system_t* sys, int64_t n_glob, int64_t n_own, const double* q,
                  const double* p, const int32_t* gidx, void* stream) {
    gsapi::NvtxScope nvtx_("gs_slab_begin");
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || n_glob < 1 || n_own < 0 || n_own > n_glob || n_glob >= (1ll << 31) || (n_own && (!q || !p || !gidx)))
        return fail(GS_ERR_INVALID, "bad slab args");
    int rc = check_system(sys);
    if (rc) return rc;
    if (!(sys->cutoff > 0.0)) return fail(GS_ERR_INVALID, "the slab path needs a positive cutoff (support radius)");
    GS_CUDA(cudaSetDevice(ctx->device));
    auto& L = ctx->slab;
    L.n_glob = n_glob;
    L.n_own = n_own;
    L.own_sorted = 0;
    L.n_loc = 0;
    L.ncl = 0;
    L.cutoff = sys->cutoff;
    // the one-rank list parameters of N = n_glob (gs_api.cu verlet_ws): skin and lanes per cluster
    L.skin = ctx->verlet_skin >= 0.0 ? ctx->verlet_skin : (n_glob < 131072 ? 0.1 : 0.05);
    L.rl = sys->cutoff * (1.0 + L.skin);
    L.tpl = verlet_tpl(n_glob);
    if ((rc = ensure_own(ctx, std::max<int64_t>(n_own, 1)))) return rc;
    GS_CUDA(grow(L.red, 4 * kCellBboxBlocks)); GS_CUDA(grow(L.b4, 4)); GS_CUDA(grow(L.gp, 1));
    GS_CUDA(grow(L.flags, 4)); GS_CUDA(grow(L.over, 1));
    GS_CUDA(cudaMemsetAsync(L.flags.ptr, 0, 4 * sizeof(unsigned), s));
    GS_CUDA(cudaMemsetAsync(L.over.ptr, 0, sizeof(unsigned long long), s));
    k_slab_status_reset<<<1, 1, 0, s>>>(ctx->st.ptr);
    if (n_own) k_slab_begin<<<blk(n_own), 256, 0, s>>>(q, p, gidx, n_own, L.Su.ptr, L.Bu.ptr, L.Au.ptr, L.gu.ptr);
    GS_CUDA(cudaGetLastError());
    return GS_OK;
}

int gs_slab_bbox(gs_context* ctx, double* b4, void* stream) {
    if (!ctx || !b4) return fail(GS_ERR_INVALID, "bad slab args");
    GS_CUDA(cudaSetDevice(ctx->device));
    const Own o = own_arrays(ctx);
    slab_bbox(o.S, ctx->slab.n_own, ctx->slab.red.ptr, b4, (cudaStream_t)stream);
    GS_CUDA(cudaGetLastError());
    return GS_OK;
}

int gs_slab_grid(gs_context* ctx, const double* b4, gs_slab_grid_t* out, void* stream) {
    gsapi::NvtxScope nvtx_("gs_slab_grid");
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || !b4 || !out) return fail(GS_ERR_INVALID, "bad slab args");
    GS_CUDA(cudaSetDevice(ctx->device));
    auto& L = ctx->slab;
    slab_grid(b4, L.rl, L.n_glob, L.gp.ptr, s);
    GS_CUDA(cudaMemcpyAsync(&L.g, L.gp.ptr, sizeof(GridParams), cudaMemcpyDeviceToHost, s));
    GS_CUDA(cudaStreamSynchronize(s));
    out->x0 = L.g.x0; out->y0 = L.g.y0; out->h = L.g.h;
    out->nx = L.g.nx; out->ny = L.g.ny; out->sub = L.g.sub; out->hashed = L.g.hashed;
    return GS_OK;
}

int gs_slab_rows(gs_context* ctx, int64_t* hist, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || !hist) return fail(GS_ERR_INVALID, "bad slab args");
    if (ctx->slab.g.hashed) return fail(GS_ERR_UNSUPPORTED, "slab decomposition needs a row-major grid");
    GS_CUDA(cudaSetDevice(ctx->device));
    const Own o = own_arrays(ctx);
    GS_CUDA(cudaMemsetAsync(hist, 0, (size_t)ctx->slab.g.ny * sizeof(int64_t), s));
    if (ctx->slab.n_own)
        k_slab_rows<<<blk(ctx->slab.n_own), 256, 0, s>>>(o.S, ctx->slab.n_own, ctx->slab.gp.ptr,
                                                         reinterpret_cast<unsigned long long*>(hist));
    GS_CUDA(cudaGetLastError());
    return GS_OK;
}

int gs_slab_pack(gs_context* ctx, const int32_t* owner, int32_t world, double* send, int64_t* counts, void* stream) {
    gsapi::NvtxScope nvtx_("gs_slab_pack");
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || !owner || world < 1 || (ctx->slab.n_own && !send)) return fail(GS_ERR_INVALID, "bad slab args");
    auto& L = ctx->slab;
    GS_CUDA(cudaSetDevice(ctx->device));
    const int64_t n = L.n_own;
    const Own o = own_arrays(ctx);
    GS_CUDA(grow(L.dcount, world));
    GS_CUDA(cudaMemsetAsync(L.dcount.ptr, 0, world * sizeof(unsigned long long), s));
    if (n) {
        k_slab_dest<<<blk(n), 256, 0, s>>>(o.S, n, L.gp.ptr, owner, L.skey.ptr, L.sval.ptr, L.dcount.ptr);
        size_t bytes = 0;
        const int end_bit = std::max(1, bits_for(world));
        cub::DeviceRadixSort::SortPairs(nullptr, bytes, L.skey.ptr, L.skey2.ptr, L.sval.ptr, L.sval2.ptr, (int)n, 0,
                                        end_bit, s);
        GS_CUDA(grow(L.cub, bytes));
        bytes = L.cub.cap;
        GS_CUDA(cub::DeviceRadixSort::SortPairs(L.cub.ptr, bytes, L.skey.ptr, L.skey2.ptr, L.sval.ptr, L.sval2.ptr,
                                                (int)n, 0, end_bit, s));
        k_slab_pack<<<blk(n), 256, 0, s>>>(L.sval2.ptr, n, o.S, o.B, o.A, o.g, send);
    }
    if (counts) {  // optional: the driver knows them from the all-gathered row histograms
        std::vector<unsigned long long> c(world);
        GS_CUDA(cudaMemcpyAsync(c.data(), L.dcount.ptr, world * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
        GS_CUDA(cudaStreamSynchronize(s));
        for (int d = 0; d < world; ++d) counts[d] = (int64_t)c[d];
    }
    GS_CUDA(cudaGetLastError());
    return GS_OK;
}

int gs_slab_unpack(gs_context* ctx, int64_t n_own, const double* recv, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || n_own < 0 || (n_own && !recv)) return fail(GS_ERR_INVALID, "bad slab args");
    GS_CUDA(cudaSetDevice(ctx->device));
    int rc = ensure_own(ctx, std::max<int64_t>(n_own, 1));
    if (rc) return rc;
    auto& L = ctx->slab;
    L.n_own = n_own;
    L.own_sorted = 0;
    if (n_own) k_slab_unpack<<<blk(n_own), 256, 0, s>>>(recv, n_own, L.Su.ptr, L.Bu.ptr, L.Au.ptr, L.gu.ptr);
    GS_CUDA(cudaGetLastError());
    return GS_OK;
}

int gs_slab_layout(gs_context* ctx, int32_t y_own0, int32_t y_own1, int32_t y_loc0, int32_t y_loc1, int64_t own_begin,
                   int64_t n_loc, void* stream) {
    gsapi::NvtxScope nvtx_("gs_slab_layout");
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx) return fail(GS_ERR_INVALID, "bad slab args");
    auto& L = ctx->slab;
    if (L.own_sorted) return fail(GS_ERR_INVALID, "slab layout: own particles already placed (pack/unpack first)");
    const int ny = L.g.ny;
    if (!(0 <= y_loc0 && y_loc0 <= y_own0 && y_own0 <= y_own1 && y_own1 <= y_loc1 && y_loc1 <= ny) ||
        own_begin < 0 || own_begin + L.n_own > n_loc)
        return fail(GS_ERR_INVALID, "bad slab rows");
    GS_CUDA(cudaSetDevice(ctx->device));
    L.y_own0 = y_own0; L.y_own1 = y_own1; L.y_loc0 = y_loc0; L.y_loc1 = y_loc1;
    L.own_begin = own_begin;
    L.n_loc = n_loc;
    const int64_t n = L.n_own;
    GS_CUDA(grow(L.S, n_loc + 1)); GS_CUDA(grow(L.S2, n_loc + 1)); GS_CUDA(grow(L.gidx, std::max<int64_t>(n_loc, 1)));
    L.par = 0;
    GS_CUDA(grow(L.B, std::max<int64_t>(n, 1))); GS_CUDA(grow(L.A, std::max<int64_t>(n, 1)));
    GS_CUDA(grow(L.Xb, std::max<int64_t>(n, 1)));
    // the device grid covers the local rows from now on
    L.g.ylo = y_loc0;
    L.g.yhi = y_loc1;
    GS_CUDA(cudaMemcpyAsync(L.gp.ptr, &L.g, sizeof(GridParams), cudaMemcpyHostToDevice, s));
    if (n) {
        const int gbits = bits_for(L.n_glob - 1 > 0 ? L.n_glob - 1 : 1);
        const int64_t cells = (int64_t)(y_own1 - y_own0) * L.g.nx;
        const int end_bit = gbits + bits_for(cells) + GS_CELL_SUBKEY;
        if (end_bit > 64) return fail(GS_ERR_UNSUPPORTED, "slab sort key exceeds 64 bits");
        k_slab_own_keys<<<blk(n), 256, 0, s>>>(L.Su.ptr, L.gu.ptr, n, L.gp.ptr, y_own0, gbits, L.skey.ptr, L.sval.ptr);
        size_t bytes = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, bytes, L.skey.ptr, L.skey2.ptr, L.sval.ptr, L.sval2.ptr, (int)n, 0,
                                        end_bit, s);
        GS_CUDA(grow(L.cub, bytes));
        bytes = L.cub.cap;
        GS_CUDA(cub::DeviceRadixSort::SortPairs(L.cub.ptr, bytes, L.skey.ptr, L.skey2.ptr, L.sval.ptr, L.sval2.ptr,
                                                (int)n, 0, end_bit, s));
        k_slab_place<<<blk(n), 256, 0, s>>>(L.sval2.ptr, n, L.Su.ptr, L.Bu.ptr, L.Au.ptr, L.gu.ptr,
                                            L.S.ptr + own_begin, L.B.ptr, L.A.ptr, L.gidx.ptr + own_begin);
    }
    L.own_sorted = 1;
    GS_CUDA(cudaGetLastError());
    return GS_OK;
}

int gs_slab_views(gs_context* ctx, double** S, double** S_alt, int32_t** gidx, int32_t** flag) {
    if (!ctx || !S || !S_alt || !gidx || !flag) return fail(GS_ERR_INVALID, "bad slab args");
    *S = reinterpret_cast<double*>(slab_cur(ctx));
    *S_alt = reinterpret_cast<double*>(ctx->slab.par ? ctx->slab.S.ptr : ctx->slab.S2.ptr);
    *gidx = reinterpret_cast<int32_t*>(ctx->slab.gidx.ptr);
    *flag = reinterpret_cast<int32_t*>(ctx->slab.flags.ptr);
    return GS_OK;
}

// After the halo exchange: cell starts over the local rows, own clusters, their lists.
int gs_slab_lists(gs_context* ctx, int64_t ncl_host, void* stream) {
    gsapi::NvtxScope nvtx_("gs_slab_lists");
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || !ctx->slab.own_sorted) return fail(GS_ERR_INVALID, "slab lists before the layout");
    if (ncl_host < 0 || ncl_host > ctx->slab.n_own) return fail(GS_ERR_INVALID, "bad cluster count");
    GS_CUDA(cudaSetDevice(ctx->device));
    auto& L = ctx->slab;
    const int64_t n_loc = L.n_loc, n = L.n_own;
    const int64_t ncells = (int64_t)(L.y_loc1 - L.y_loc0) * L.g.nx;
    GS_CUDA(grow(L.keys, std::max<int64_t>(n_loc, 1))); GS_CUDA(grow(L.Sf, std::max<int64_t>(n_loc, 1)));
    GS_CUDA(grow(L.start, ncells + 1));
    GS_CUDA(grow(L.head, n + 1)); GS_CUDA(grow(L.dest, n + 1));
    if (n_loc) k_slab_local_keys<<<blk(n_loc), 256, 0, s>>>(slab_cur(ctx), n_loc, L.gp.ptr, L.keys.ptr, L.Sf.ptr);
    k_slab_start<<<blk(n_loc + 1), 256, 0, s>>>(L.keys.ptr, n_loc, ncells, L.start.ptr);
    k_slab_heads<<<blk(n + 1), 256, 0, s>>>(L.keys.ptr, L.start.ptr, L.own_begin, n, L.g.nx, L.head.ptr);
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, L.head.ptr, L.dest.ptr, (int)(n + 1), s);
    GS_CUDA(grow(L.cub, bytes));
    bytes = L.cub.cap;
    GS_CUDA(cub::DeviceScan::ExclusiveSum(L.cub.ptr, bytes, L.head.ptr, L.dest.ptr, (int)(n + 1), s));
    // clusters: sum over the own rows of ceil(count / 2), known to the driver from the histogram
    // (checked on the device: the scan's total must agree)
    const int ncl = (int)ncl_host;
    L.ncl = ncl;
    GS_CUDA(grow(L.cfirst, ncl + 1)); GS_CUDA(grow(L.cnt, ncl + 1)); GS_CUDA(grow(L.ofs, ncl + 1));
    GS_CUDA(grow(L.len, std::max(ncl, 1)));
    k_slab_cfirst<<<blk(n + 1), 256, 0, s>>>(L.head.ptr, L.dest.ptr, L.own_begin, n, L.cfirst.ptr, ncl);
    k_slab_sentinel<<<1, 1, 0, s>>>(L.S.ptr, L.S2.ptr, n_loc, L.cnt.ptr, ncl);
    bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, L.cnt.ptr, L.ofs.ptr, ncl + 1, s);
    GS_CUDA(grow(L.cub, bytes));
    SlabLists sl = slab_lists(ctx);
    if (int e = slab_list_caps(sl, n_loc, ncl, L.tpl, s)) return fail(GS_ERR_CUDA, cudaGetErrorString((cudaError_t)e));
    long long total = 0;
    GS_CUDA(cudaMemcpyAsync(&total, L.ofs.ptr + ncl, sizeof(total), cudaMemcpyDeviceToHost, s));
    GS_CUDA(cudaStreamSynchronize(s));
    if (total >= (1ll << 31)) return fail(GS_ERR_UNSUPPORTED, "slab lists exceed 2^31 entries");
    GS_CUDA(grow(L.list, (size_t)std::max<long long>(total, 1)));
    sl = slab_lists(ctx);
    slab_list_fill(sl, n_loc, ncl, L.tpl, L.own_begin, s);
    GS_CUDA(cudaGetLastError());
    return GS_OK;
}

int gs_slab_stage(gs_context* ctx, const gs_system_t* sys, int32_t step, int32_t stg, double dt, void* stream) {
    gsapi::NvtxScope nvtx_("gs_slab_stage");
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx || !ctx->slab.own_sorted) return fail(GS_ERR_INVALID, "slab stage before the layout");
    int rc = check_system(sys);
    if (rc) return rc;
    if (stg < 0 || stg > 3 || step < 1) return fail(GS_ERR_INVALID, "bad stage index");
    GS_CUDA(cudaSetDevice(ctx->device));
    auto& L = ctx->slab;
    const SysConst sc = make_const(sys);
    const unsigned long long ev = (unsigned long long)step * 8ull + 2ull * (unsigned long long)stg;
    // the sweep carries the RK4 stage epilogue (rows in local order: coalesced): it reads the
    // current buffer and writes the own rows' next records into the other one, which becomes current
    double4* next = L.par ? L.S.ptr : L.S2.ptr;
    const double thr = 0.5 * L.skin * L.cutoff;
    VerletEpi e{};
    e.a.S = next + L.own_begin; e.a.B = L.B.ptr; e.a.A = L.A.ptr;
    e.a.nrows = L.n_own; e.a.stage = stg; e.a.dt = dt; e.a.st = ctx->st.ptr; e.a.event = ev + 1;
    e.scale_q = sc.scale_q; e.scale_p = sc.scale_p; e.sigma2 = sc.sigma2;
    e.Xb = L.Xb.ptr; e.thr2 = thr * thr * (1.0 - 1e-9); e.flags = L.flags.ptr;
    e.decide = 0; e.local = 1; e.rbase = L.own_begin;
    GS_CUDA(cudaMemsetAsync(L.flags.ptr, 0, sizeof(unsigned), s));
    if (ctx->prof_on) prof_mark(ctx, s);
    slab_sweep_epi(sc, slab_lists(ctx), L.gidx.ptr, L.n_loc, L.ncl, L.tpl, L.n_glob, e, ctx->st.ptr, ev, ctx->tbl.ptr, s);
    if (ctx->prof_on) prof_mark(ctx, s);
    ctx->launches += 1;
    ctx->pair_launches++;
    L.par ^= 1;
    GS_CUDA(cudaGetLastError());
    return GS_OK;
}

int gs_slab_status(gs_context* ctx, gs_status_t* out, void* stream) {
    if (!ctx || !out) return fail(GS_ERR_INVALID, "bad slab args");
    GS_CUDA(cudaSetDevice(ctx->device));
    fetch_status(ctx, (cudaStream_t)stream, std::max<int64_t>(ctx->slab.n_glob, 1), out);
    return GS_OK;
}

}  // extern "C"

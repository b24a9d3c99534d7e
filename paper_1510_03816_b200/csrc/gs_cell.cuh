// gs_cell.cuh — cell-list workspace and launchers (gs_cell.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "gs_kernels.cuh"

namespace gsb {

// Cells have edge = cutoff.  When the point cloud fits in cell_cap(n) such cells the grid is a
// dense row-major array (a stencil row = one contiguous sorted range); otherwise (e.g. a
// diverging flow flinging particles far apart) cells are hashed into cell_cap(n) buckets and
// the 9 stencil cells are looked up separately — the work stays ~O(N x neighbours).
//
// The row-major grid may be subdivided: cell edge h = cutoff / sub (sub <= kCellSubMax).  A
// target then visits 2 sub + 1 stencil rows, each trimmed to the x-range of cells its disk
// of radius rc reaches — fewer fp32 candidates per accepted pair (C5: 9 -> ~5 sigma^2).
constexpr int kCellSubMax = 4;

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {  // splitmix64 finalizer
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
// Row-major cell keys carry a sub-cell index (Morton order over 2^(GS_CELL_SUBKEY/2) sub-cells per
// axis) below the cell index: cells stay contiguous and x-ordered in a row (the stencil ranges are
// unchanged), and inside a cell the sorted order walks the sub-cells, so consecutive sorted
// particles — the lists' clusters — sit close together and a cluster's list (the union of its
// members' neighbourhoods) shrinks (C4 RHS 1.96 -> 1.71 ms, C5 1.46 -> 1.36 ms).
#ifndef GS_CELL_SUBKEY          // sub-cell key bits (A/B builds: 0 = index order inside a cell)
#define GS_CELL_SUBKEY 4
#endif
// fx, fy: the position inside its cell in cell units (clamped to the sub-cell range)
__device__ __forceinline__ unsigned cell_subkey(double fx, double fy) {
#if GS_CELL_SUBKEY
    constexpr int kB = GS_CELL_SUBKEY / 2, kS = 1 << kB;  // bits / sub-cells per axis
    const unsigned sx = (unsigned)min(max((int)(fx * kS), 0), kS - 1), sy = (unsigned)min(max((int)(fy * kS), 0), kS - 1);
    unsigned sub = 0;
#pragma unroll
    for (int b = 0; b < kB; ++b) sub |= (((sx >> b) & 1u) << (2 * b)) | (((sy >> b) & 1u) << (2 * b + 1));
    return sub;
#else
    return 0u;
#endif
}

struct GridParams {
    double x0, y0, inv_h;
    double h, rc;        // cell edge; filter radius (double) = sqrt(rc2f) before fp32 rounding
    int nx, ny, ncells;  // row-major: nx * ny cells; hashed: ncells buckets (a power of two)
    float rc2f;          // fp32 candidate-filter radius^2: cutoff^2 grown by the fp32 position error
    int hashed;
    int sub;             // cells per cutoff (row-major grid; 1 when hashed or degenerate)
    int ylo, yhi;        // row-major: `start` covers cell rows [ylo, yhi) (0, ny except on a slab)
};

constexpr int kCellBboxBlocks = 296;

// Device buffers owned by the context (sizes for n particles, cell_cap(n) cells).
struct CellWs {
    unsigned* keys;         // n
    unsigned* keys_sorted;  // n
    unsigned* vals;         // n
    unsigned* perm;         // n: sorted position -> original index
    int* start;             // cell_cap(n) + 1
    double4* Ss;            // n: records in sorted order
    float2* Sf;             // n: fp32 positions relative to the grid origin, sorted order
    double* bbox_red;       // 4 * kCellBboxBlocks
    GridParams* gp;         // 1
    int* tlist;             // n: sorted positions of a rank's target rows (row-range launches)
    int* nsel;              // 1: CUB select output count
    void* cub_temp;         // shared by the radix sort and the target select (same stream)
    size_t cub_bytes;
};

size_t cell_cub_bytes(int64_t n);
int64_t cell_cap(int64_t n);
// Builds the grid for the n records of S (positions of the current stage).  Returns a
// cudaError_t value (0 on success).
// skin_ctl (device, optional): the grid is built for base_cutoff (1 + skin_ctl[0]) instead of cutoff
int cell_build(const CellWs& w, const double4* S, int64_t n, double cutoff, cudaStream_t stream,
               const double* skin_ctl = nullptr, double base_cutoff = 0.0);
// Raw pair sums of the targets with original index in [row0, row1) -> part[i - row0].
// `accepted` (nullable) accumulates the number of evaluated pairs (d < cutoff, self included).
void launch_cell_pair(const SysConst& sc, const CellWs& w, int64_t n, int64_t row0, int64_t row1, double4* part,
                      DevStatus* st, unsigned long long event, const double* tbl_dev, unsigned long long* accepted,
                      cudaStream_t stream);

// ---- cluster Verlet lists (gs_verlet.cu): the cell path of whole evolves / matches ----------
// Clusters of GS_VERLET_M consecutive sorted particles; one list per cluster of the sorted
// positions within cutoff (1 + skin) of any member at the last build, reused until a particle has
// moved half the skin.
constexpr int kVerletFlags = 8;     // words of VerletWs::flags
// Adaptive skin (relative trigger path, gs_verlet.cu k_verlet_trigger_check): bounds and the
// cost ratio (one list build / one pair sweep) of its model.
constexpr double kSkinMin = 0.03, kSkinMax = 0.12, kSkinCostRatio = 0.67;
// Device {skin, rate} reset to {skin0, 0} (start of every call: results depend only on the call).
void verlet_skin_init(double* skin_ctl, double skin0, cudaStream_t stream);
struct VerletWs {
    long long* cnt;                // ncl + 1 (cnt[ncl] = 0): list capacities (candidate counts, padded)
    long long* ofs;                // ncl + 1: exclusive scan of cnt (ofs[ncl] = entries of the build)
    int* len;                      // ncl: padded list lengths
    int* list;                     // cap entries
    int64_t cap;
    double2* Xb;                   // n: positions at the build, sorted order
    int* inv;                      // n: original index -> sorted slot
    unsigned* flags;               // [0] rebuild wanted, [1] builds, [2] CTA counter, [3] last decision,
                                   // [4] RHS since the build (zero-initialised, kVerletFlags words)
    unsigned long long* overflow;  // entries a build needed beyond cap (0: none)
    void* scan_temp;
    size_t scan_bytes;
    int tpl;                       // pair-sweep lanes per cluster (lists padded to 2 tpl)
    double skin;                   // list radius = cutoff (1 + skin); rebuild at skin * cutoff / 2
    double cutoff;
    double* skin_ctl;              // device {skin, RHS per unit skin}: the adaptive skin of the relative
                                   // trigger's path (verlet_skin_adapt); nullptr: the fixed `skin`
    double4* Ss_pair[2];           // both halves of the sorted-record ping-pong: the sentinel goes into each
};
// The stage epilogue fused into the list sweep (single rank, all rows): the lane that reduced a
// member's sums applies scales, sigma2 and the RK4 stage update (stage_update) to its row of
// a.S / a.B / a.A (original order), stores the new record into the next stage's sorted buffer
// (Ss_next, the other half of a ping-pong pair; nullptr on the call's last stage) and the last
// CTA decides the next stage's rebuild (flags[3] / the IF-node condition), as k_finish_verlet.
struct VerletEpi {
    FinishArgs a;                  // S, B, A, stage, dt, st, event (= the sweep's event + 1)
    double scale_q, scale_p, sigma2;
    double4* Ss_next;              // the next stage's sorted copy (nullptr: none)
    const double2* Xb;             // positions at the build (nullptr: no rebuild check, last stage)
    double thr2;
    unsigned* flags;               // [0] rebuild wanted, [2] CTA counter, [3] decision
    cudaGraphConditionalHandle cond;
    int use_cond;
    int decide;                    // 1: the last CTA decides (flags[3] / IF condition); 0: OR into flags[0]
    int local;                     // rows of S / B / A / Xb by sorted position k - rbase (the slab
    int64_t rbase;                 // layout) instead of by original index (single GPU)
};
int64_t verlet_clusters(int64_t n);
int verlet_tpl(int64_t n);
size_t verlet_scan_bytes(int64_t ncl);
// Grid + lists for the records of S (cell workspace w is rebuilt; Ss[n] becomes the sentinel;
// the decision counter flags[2] is reset).
int verlet_build(const CellWs& w, const VerletWs& v, const double4* S, int64_t n, double cutoff, cudaStream_t stream);
// Ss <- S in sorted order and the rebuild decision (force: no gather, rebuild) -> IF condition / flags[3].
void verlet_gather(const CellWs& w, const VerletWs& v, const double4* S, int64_t n, int force,
                   cudaGraphConditionalHandle cond, int use_cond, cudaStream_t stream);
// The rebuild decision of large clouds from the stage's displacements (the sorted records w.Ss the
// separate list epilogue wrote, against the build positions v.Xb): relative displacement of
// neighbours over coarse cells of edge 2 rl (gs_verlet.cu k_verlet_trigger) -> flags[3] / the next
// stage's IF condition.  box: box_cap u32 (4 per coarse cell) of scratch, empty between calls
// (verlet_box_reset once at allocation).
void launch_verlet_trigger(const CellWs& w, const VerletWs& v, int64_t n, unsigned* box,
                           int64_t box_cap, cudaGraphConditionalHandle cond, int use_cond, cudaStream_t stream);
void verlet_box_reset(unsigned* box, int64_t cells, cudaStream_t stream);
// Raw pair sums of all n rows from the lists -> part[i] (original index).
void launch_verlet_pair(const SysConst& sc, const CellWs& w, const VerletWs& v, int64_t n, double4* part,
                        DevStatus* st, unsigned long long event, const double* tbl_dev, unsigned long long* accepted,
                        cudaStream_t stream);
// The same sweep with the stage epilogue fused in (no partials): e.a.S gets the new records.
void launch_verlet_pair_epi(const SysConst& sc, const CellWs& w, const VerletWs& v, int64_t n, const VerletEpi& e,
                            DevStatus* st, unsigned long long event, const double* tbl_dev, unsigned long long* accepted,
                            cudaStream_t stream);

// ---- slab decomposition (gs_slab.cu): a rank's cell rows + halo rows -------------------------
// Bounding box of n records as (min x, min y, -max x, -max y) into b4 (red: kCellBboxBlocks x 4 scratch).
void slab_bbox(const double4* S, int64_t n, double* red, double* b4, cudaStream_t stream);
// The grid of the one-rank build for list radius `cutoff` from an all-reduced b4 (n_glob particles).
void slab_grid(const double* b4, double cutoff, int64_t n_glob, GridParams* gp, cudaStream_t stream);

struct SlabLists {
    const double4* S;      // n_loc + 1 local records in global sorted order (S[n_loc]: sentinel)
    const float2* Sf;      // n_loc
    const int* start;      // local cells + 1 (rows [gp->ylo, gp->yhi))
    const GridParams* gp;
    const int* cfirst;     // ncl + 1: first local position of each own cluster
    long long* cnt;        // ncl + 1 (cnt[ncl] = 0)
    long long* ofs;        // ncl + 1
    int* len;              // ncl
    int* list;             // cap entries
    int64_t cap;
    double2* Xb;           // own particles: positions at the build
    unsigned long long* overflow;
    void* scan_temp;
    size_t scan_bytes;
};
// capacities + their exclusive scan (ofs[ncl] = entries); then the lists themselves
int slab_list_caps(const SlabLists& L, int64_t n_loc, int64_t ncl, int tpl, cudaStream_t stream);
void slab_list_fill(const SlabLists& L, int64_t n_loc, int64_t ncl, int tpl, int64_t own_begin, cudaStream_t stream);
// raw pair sums of the own clusters -> part[k - own_begin] (local sorted order)
void slab_sweep(const SysConst& sc, const SlabLists& L, const unsigned* gidx, int64_t n_loc, int64_t ncl, int tpl,
                int64_t own_begin, int64_t n_glob, double4* part, DevStatus* st, unsigned long long event,
                const double* tbl_dev, unsigned long long* accepted, cudaStream_t stream);
// The same sweep with the RK4 stage epilogue fused in (e.local: rows by local position), reading
// L.S and writing the new own records through e.a.S (the other half of the slab's ping-pong pair).
void slab_sweep_epi(const SysConst& sc, const SlabLists& L, const unsigned* gidx, int64_t n_loc, int64_t ncl, int tpl,
                    int64_t n_glob, const VerletEpi& e, DevStatus* st, unsigned long long event, const double* tbl_dev,
                    cudaStream_t stream);

}  // namespace gsb

/* geoshoot_b200.h — C ABI of the B200-native Euler–Poincaré N-particle hot path.
 *
 * The reference (arXiv 1510.03816, package `geoshoot`, /root/reference/pkg/src/geoshoot)
 * is pure Python/NumPy and has no FFI or plugin registry: its drop-in boundary is the
 * Python function API.  Each entry point below replaces one reference function; the
 * Python shim `paper_1510_03816_b200` binds them with ctypes and re-exposes the
 * reference signatures.
 *
 *   gs_rhs          <- geoshoot.particles.rhs            particles.py:109-117 (+ _interaction_terms :79-106)
 *   gs_rhs_rows     <- rows [row0,row1) of the same (target-row sharding)
 *   gs_hamiltonian  <- geoshoot.particles.hamiltonian    particles.py:120-131
 *   gs_evolve       <- geoshoot.integrator.evolve        integrator.py:66-121
 *   gs_match        <- geoshoot.shooting.match, momentum update branch
 *                                                        shooting.py:218-301 (update :266-267)
 *   gs_stage_*      <- one RK4 stage of integrator.py:98-114 for a row range; the
 *                      building blocks of the multi-GPU driver (paper_1510_03816_b200/sharded.py)
 *
 * Conventions
 *   - All arrays are fp64.  (n,2) arrays are C-order AoS (x0,y0,x1,y1,...) exactly as the
 *     reference's NumPy arrays.  Pointers documented "device" must be device memory of the
 *     context's GPU; "host" pointers are ordinary host memory.
 *   - All GPU work is ordered on the caller's `stream` (a cudaStream_t passed as void*;
 *     NULL = legacy default stream).  Functions that must report a numerical outcome
 *     (status, match result) synchronise that stream before returning; gs_rhs_rows,
 *     gs_velocity_field and the gs_stage_* / gs_p2p_* calls never synchronise.
 *   - The library owns only the workspaces inside a gs_context; the caller owns every
 *     buffer it passes.  One context per concurrent caller; no global mutable state
 *     beyond a thread-local last-error string.
 *   - Every function returns a GS_* code; numerical failures are also described in a
 *     gs_status_t so the shim can rebuild the reference's exception messages:
 *       GS_ERR_COINCIDENT      -> DegenerateConfigurationError  particles.py:92-98,
 *                                 integrator.py:102-105 ("(during step k, t in [a, b])")
 *       GS_ERR_NONFINITE_STAGE -> DivergenceError "non-finite intermediate at step k"
 *                                 integrator.py:106-112
 *       GS_ERR_NONFINITE_STATE -> DivergenceError "non-finite state at step k"
 *                                 integrator.py:58-63
 *       GS_ERR_INVALID         -> ConfigurationError / ValueError
 */
#ifndef GEOSHOOT_B200_H
#define GEOSHOOT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GS_ABI_VERSION 2

#define GS_OK 0
#define GS_ERR_INVALID 1
#define GS_ERR_COINCIDENT 2
#define GS_ERR_NONFINITE_STAGE 3
#define GS_ERR_NONFINITE_STATE 4
#define GS_ERR_CUDA 5
#define GS_ERR_UNSUPPORTED 6

/* kernels.py:44-47 KernelFamily (bessel is not provided on the device) */
#define GS_FAMILY_CONICAL 0
#define GS_FAMILY_GAUSSIAN 1

/* pair-sum strategy */
#define GS_PATH_AUTO 0   /* cell list when N >= 2048, the bounding box spans >= 25 support-radius cells and
                            holds >= 4 particles per such cell on average; dense otherwise */
#define GS_PATH_DENSE 1  /* all N^2 pairs, the reference's own semantics (no truncation) */
#define GS_PATH_CELL 2   /* pairs with d_ij < cutoff only (KD-1: G(cutoff) = 2^-53) */

/* shooting.py:56-63 */
#define GS_STOP_TARGET_RESIDUAL 0
#define GS_STOP_MOMENTUM_DELTA 1
#define GS_NORM_MAX 0
#define GS_NORM_L2 1

/* match outcomes (MatchResult.converged / diagnosis, shooting.py:251-301) */
#define GS_MATCH_CONVERGED 0
#define GS_MATCH_CAP 1          /* "iteration cap reached before the stopping rule" */
#define GS_MATCH_BLOWUP 2       /* "step too large" (non-finite or > 1e6 x initial norm) */
#define GS_MATCH_EVOLVE_FAILED 3/* "step too large (<evolve exception>)", see status */

/* SystemSpec + KernelSpec (particles.py:67-76, kernels.py:50-88) */
typedef struct {
    int32_t family;      /* GS_FAMILY_* */
    int32_t normalized;  /* KernelSpec.normalized: G(0) = 1, else x 1/(2 pi alpha^2) */
    double alpha;        /* KernelSpec.alpha > 0 */
    double sigma2;       /* SystemSpec.sigma2 >= 0 */
    double cutoff;       /* support radius for GS_PATH_CELL/AUTO; <= 0 disables the cell path */
    int32_t path;        /* GS_PATH_* */
    int32_t reserved;
} gs_system_t;

typedef struct {
    int32_t code;        /* GS_* of the first failure */
    int32_t step;        /* 1-based RK4 step of the failure (evolve / match), 0 otherwise */
    int64_t i, j;        /* coincident pair, first in row-major order (GS_ERR_COINCIDENT) */
    int32_t iteration;   /* match iteration whose shoot failed (0 = the initial zero-momentum shoot) */
    int32_t event;       /* position of the failure inside its step, 0..7: 2s = coincidence in the RHS of
                            stage s, 2s+1 = non-finite input of stage s+1, 7 = non-finite state; lets a
                            multi-GPU driver order failures seen by different ranks */
} gs_status_t;

/* ShootingConfig (shooting.py:66-100) restricted to the momentum update */
typedef struct {
    double h;
    double epsilon;
    int32_t max_iter;
    int32_t stop_rule;   /* GS_STOP_* */
    int32_t norm;        /* GS_NORM_* */
    int32_t steps;       /* EvolveConfig.steps */
    double t_final;      /* EvolveConfig.t_final */
} gs_match_config_t;

typedef struct {
    int32_t outcome;         /* GS_MATCH_* */
    int32_t iterations;      /* len(residual_history) */
    double hamiltonian;      /* H(q0, p0), particles.py:120-131 */
    double final_residual;   /* _norm(target - endpoint) */
    gs_status_t status;      /* evolve failure details when outcome == GS_MATCH_EVOLVE_FAILED */
    double seconds_device;   /* device time of the whole match (CUDA events) */
} gs_match_result_t;

typedef struct gs_context gs_context;

const char* gs_version(void);
int gs_abi_version(void);
const char* gs_last_error(void);

int gs_create(gs_context** ctx, int device);
int gs_destroy(gs_context* ctx);

/* particles.rhs: dq, dp (device, n x 2) from q, p (device, n x 2).  Synchronises to fill status. */
int gs_rhs(gs_context* ctx, const gs_system_t* sys, int64_t n, const double* q, const double* p,
           double* dq, double* dp, gs_status_t* status, void* stream);
/* Rows [row0, row1) only: dq, dp are (row1-row0) x 2.  Does not synchronise; a coincidence is
 * reported by the next gs_status_fetch on this context. */
int gs_rhs_rows(gs_context* ctx, const gs_system_t* sys, int64_t n, const double* q, const double* p,
                int64_t row0, int64_t row1, double* dq, double* dp, void* stream);
int gs_status_fetch(gs_context* ctx, gs_status_t* status, void* stream);
int gs_status_reset(gs_context* ctx, void* stream);

/* particles.hamiltonian: *h_out (host) = sum_ij (p_i . p_j) G(d_ij).  Synchronises. */
int gs_hamiltonian(gs_context* ctx, const gs_system_t* sys, int64_t n, const double* q, const double* p,
                   double* h_out, void* stream);

/* integrator.evolve: q, p (device, n x 2) are advanced in place over [0, t_final] with `steps`
 * classical RK4 steps.  If capture_every > 0 and frames != NULL, frames (device) receives
 * (1 + steps/capture_every + [steps % capture_every != 0]) records of n x 4 doubles
 * (x, y, px, py) at the reference's capture times (integrator.py:84-86, 116-119).
 * Synchronises; on failure q, p hold the state of the failing step (unspecified). */
int gs_evolve(gs_context* ctx, const gs_system_t* sys, int64_t n, double t_final, int32_t steps,
              int32_t capture_every, double* q, double* p, double* frames, gs_status_t* status,
              void* stream);

/* shooting.match with UpdateSpace.MOMENTUM: q0, target (device, n x 2).  Outputs p0_out and
 * endpoint_out (device, n x 2), history_out (host, >= max_iter doubles) and *result (host).
 * The whole feedback loop runs on the device; the host reads two scalars per iteration
 * (one persistent kernel for n <= 512).  Synchronises. */
int gs_match(gs_context* ctx, const gs_system_t* sys, const gs_match_config_t* cfg, int64_t n,
             const double* q0, const double* target, double* p0_out, double* endpoint_out,
             double* history_out, gs_match_result_t* result, void* stream);

/* particles.velocity_field (particles.py:140-150): u (device, m x 2) = sum_j G(|x_k - q_j|) p_j
 * at the m sample points x (device, m x 2) for the state q, p (device, n x 2).  Stream-ordered
 * (does not synchronise); m == 0 is a no-op. */
int gs_velocity_field(gs_context* ctx, const gs_system_t* sys, int64_t n, const double* q,
                      const double* p, int64_t m, const double* x, double* u, void* stream);

/* ---- batched independent trajectories ---------------------------------
 * Replace the reference's serial loops over independent matches / shoots:
 *   convergence_sweep cells (analysis.py:254-283), cluster_test / shape_distance pairs
 *   (analysis.py:109-126, 162-207), exact_vs_inexact rows (analysis.py:326-377): gs_match_batch;
 *   newton_match Jacobian columns, 2N shoots per iteration (shooting.py:367-372): gs_evolve_batch.
 * For n <= 512 on the dense path every item is one CTA of ONE persistent launch; otherwise the
 * items run one after another through gs_match / gs_evolve. */
typedef struct {
    gs_system_t system;        /* per item (alpha, sigma2 may differ; the family may not) */
    gs_match_config_t config;  /* per item (h, epsilon, max_iter, stop rule, norm, evolve config) */
} gs_batch_item_t;

/* batch matches over n landmarks.  Item b reads q0 + b*q0_stride and target + b*target_stride
 * (device, n x 2; stride 0 = shared) and writes p0_out / endpoint_out + b*2n (device) and
 * history_out + b*history_stride (DEVICE; history_stride >= every max_iter) and results[b]
 * (host; seconds_device = the whole batch's device time).
 * gram_factor != NULL selects the VELOCITY update space (shooting.py:263-265): the lower
 * Cholesky factor L of the Gram matrix over item b's q0 at gram_factor + b*factor_stride
 * (device, n x n row-major, K = L L^T; stride 0 = shared), and p = K^-1 u is solved on the
 * device every iteration (velocity batches need n <= 512 and the dense path).
 * Validation errors name the item.  Synchronises. */
int gs_match_batch(gs_context* ctx, const gs_batch_item_t* items, int64_t batch, int64_t n,
                   const double* q0, int64_t q0_stride, const double* target, int64_t target_stride,
                   const double* gram_factor, int64_t factor_stride, double* p0_out,
                   double* endpoint_out, double* history_out, int64_t history_stride,
                   gs_match_result_t* results, void* stream);

/* batch evolves of one system: item b starts from (q_in + b*q_stride, p_io + b*2n) (device;
 * q_stride 0 = shared q0) and ends in (q_out + b*2n, p_io + b*2n).  status[b] (host) carries
 * each item's failure as gs_evolve would report it; the call returns GS_OK unless the batch
 * itself is invalid.  Synchronises. */
int gs_evolve_batch(gs_context* ctx, const gs_system_t* sys, int64_t batch, int64_t n,
                    double t_final, int32_t steps, const double* q_in, int64_t q_stride,
                    double* q_out, double* p_io, gs_status_t* status, void* stream);

/* ---- stage-level API (multi-GPU driver; one rank owns rows [row0, row1)) -----------------
 * The context keeps a packed stage state S (n x 4: x, y, px, py, device) that every rank
 * holds in full, plus the rank's own RK4 base/accumulator rows.
 *   gs_stage_begin  : S <- (q, p) (device, n x 2, full), base rows <- S rows, resets status;
 *                     S has room for n + 64 records (padding rows are zero) so that equal-size
 *                     per-rank slices can be all-gathered in place
 *   gs_stage_run    : one RK4 stage (0..3) of step `step` (1-based) for rows [row0,row1):
 *                     evaluates the RHS of those rows against all n sources in S and writes
 *                     the next stage input (or, after stage 3, the new state) into S's rows
 *   gs_stage_state  : device pointer to S (n x 4 doubles), for the all-gather of S's rows
 *   gs_stage_end    : copies the base rows out as (q, p) rows (device, (row1-row0) x 2)
 */
int gs_stage_begin(gs_context* ctx, int64_t n, const double* q, const double* p, int64_t row0,
                   int64_t row1, void* stream);
int gs_stage_run(gs_context* ctx, const gs_system_t* sys, int32_t step, int32_t stage, double dt,
                 void* stream);
double* gs_stage_state(gs_context* ctx);
int gs_stage_end(gs_context* ctx, double* q_rows, double* p_rows, void* stream);

/* kernels.gram_matrix (kernels.py:181-197) on the device: K (device, n x n row-major) =
 * G(|q_i - q_j|) for the velocity-space feedback update (shooting.py:138-175, 263-265).
 * Returns GS_ERR_COINCIDENT with the row-major first coincident pair in *bad_i, *bad_j
 * ("points i and j coincide; Gram matrix would be singular").  Synchronises. */
int gs_gram(gs_context* ctx, const gs_system_t* sys, int64_t n, const double* q, double* K, int64_t* bad_i,
            int64_t* bad_j, void* stream);

/* shooting.py:138-159, 263-265 (_GramSolver.solve) without forming K: solves (K (x) I2) p = u by
 * conjugate gradients, K v being the dq half of the RHS at (q0, v) through the same pair kernels
 * (dense, or the cluster lists of q0 built once).  q0, u (device, n x 2); p (device, n x 2) is the
 * initial guess on entry (warm start) and the solution on exit.  Stops when |u - K p| <= tol |u|
 * or after max_it iterations; *iters and *relres (host) report which.  coef (host, 2 * max_it
 * doubles, nullable) receives alpha_k, beta_k of every iteration — the Lanczos tridiagonal whose
 * extreme eigenvalues estimate cond(K) for the reference's ill-conditioning warning
 * (shooting.py:237-242).  Synchronises (once per iteration). */
int gs_gram_cg(gs_context* ctx, const gs_system_t* sys, int64_t n, const double* q0, const double* u, double* p,
               double tol, int32_t max_it, int32_t* iters, double* coef, double* relres, void* stream);

/* Symmetric multi-GPU split of the dense RHS (each unordered pair once, gs_sym.cu):
 *   gs_sym_parts       : number of work items (superblock pairs) of one RHS at this n (0 if the
 *                        symmetric kernel is not available for n)
 *   gs_stage_pairs_sym : evaluates items [part_begin, part_end) on the session state S and writes
 *                        this rank's raw partial sums for ALL n rows into R (device, n x 4 doubles:
 *                        sum G p_j, sum c (q_i - q_j)); the ranks' R are summed by a
 *                        reduce-scatter over rows
 *   gs_stage_finish    : RK4 stage epilogue of the session rows from their reduced raw sums
 *                        (device, (row1-row0) x 4), as gs_stage_run's second half */
int gs_stage_path(gs_context* ctx, const gs_system_t* sys, void* stream); /* GS_PATH_DENSE/CELL, <0: -GS_ERR_* */
int64_t gs_sym_parts(int64_t n);
int gs_stage_pairs_sym(gs_context* ctx, const gs_system_t* sys, int32_t step, int32_t stage, int64_t part_begin,
                       int64_t part_end, double* R, void* stream);
int gs_stage_finish(gs_context* ctx, const gs_system_t* sys, int32_t step, int32_t stage, double dt,
                    const double* R_rows, void* stream);

/* ---- fused stage exchange over peer memory (multi-GPU symmetric split) ----------------------
 * Replaces the NCCL reduce-scatter + all-gather of a stage: the stage
 * epilogue of this rank's rows reads every rank's raw row sums over NVLink and stores each new
 * 32-byte stage record straight into every rank's S.  Per stage: gs_p2p_pairs (waits for the
 * previous stage's records, this rank's superblock pairs, signals "sums ready"), gs_p2p_finish
 * (waits for all ranks' sums, epilogue + stores, signals "records written"); gs_p2p_sync after
 * the last stage.  Signals are monotonic counters in each rank's memory (system-scope atomics);
 * waits give up after GS_B200_P2P_TIMEOUT_S (default 10 s) and count it in gs_p2p_timeouts —
 * a lost signal costs a timeout, never a hang.  Requires an open stage session (gs_stage_begin).
 *   gs_p2p_local    : allocates this rank's sums buffer (rows_all records) and counters (zeroed);
 *                     returns the device pointers of S, R and the counters
 *   gs_p2p_export   : the same, as 3 cudaIpcMemHandle_t (3 x 64 bytes) for the other ranks
 *   gs_p2p_import   : opens every rank's handles (world x 3 x 64 bytes, rank order)
 *   gs_p2p_set_peers: sets the ranks' pointers directly (one process driving several contexts) */
int gs_p2p_local(gs_context* ctx, int64_t rows_all, void** S, void** R, void** flags);
int gs_p2p_export(gs_context* ctx, int64_t rows_all, void* handles);
int gs_p2p_import(gs_context* ctx, int world, int rank, const void* handles_all);
int gs_p2p_set_peers(gs_context* ctx, int world, int rank, void* const* S, void* const* R, void* const* F);
int gs_p2p_pairs(gs_context* ctx, const gs_system_t* sys, int32_t step, int32_t stage, int64_t part_begin,
                 int64_t part_end, void* stream);
int gs_p2p_finish(gs_context* ctx, const gs_system_t* sys, int32_t step, int32_t stage, double dt,
                  void* stream);
int gs_p2p_sync(gs_context* ctx, void* stream);
int gs_p2p_timeouts(gs_context* ctx, int64_t* timeouts);
int gs_p2p_close(gs_context* ctx);

/* Profiling: with profiling enabled, every launch of the pair kernel (the dense or cell-list
 * RHS sweep, or the persistent small-N kernel) is bracketed by CUDA events on its stream;
 * gs_profile_read returns their summed device time (ms), the number of pair-kernel launches,
 * of all kernel launches and of evaluated ordered pairs (dense: rows x n per RHS; cell list:
 * pairs with d < cutoff incl. self, counted on the device while profiling) since the last
 * reset.  Synchronises. */
int gs_profile_enable(gs_context* ctx, int32_t on);
int gs_profile_read(gs_context* ctx, double* pair_ms, int64_t* pair_launches, int64_t* launches, int64_t* pairs,
                    int32_t reset);

/* Cell path of multi-RHS calls (gs_evolve, gs_match): the RHS runs through cluster Verlet lists
 * rebuilt only when a particle has moved half the skin (gs_verlet.cu).  Diagnostics: *builds =
 * list builds so far on this context, *entries = list capacity (candidates) of the last
 * build.  Synchronises. */
int gs_cell_stats(gs_context* ctx, int64_t* builds, int64_t* entries, void* stream);

/* ---- slab decomposition of the cell path across ranks (multi-GPU) -----------
 * Replaces "every rank all-gathers all N stage records and rebuilds the whole grid" for the
 * compactly supported kernel (particles.py:109-117 truncated at the support radius, KD-1): each
 * rank owns the particles of a contiguous band of cell rows of the global grid (balanced by an
 * all-reduced row histogram) and holds `sub` halo rows on each side, all in global sorted order.
 * The host driver (paper_1510_03816_b200/slab.py) issues the collectives; per list build:
 *   gs_slab_bbox   : (min x, min y, -max x, -max y) of the own particles into b4 (device, 4
 *                    doubles) -> elementwise MIN all-reduce over the ranks
 *   gs_slab_grid   : the one-rank build's grid for list radius cutoff (1 + skin) from the reduced
 *                    b4 (the same on every rank); synchronises
 *   gs_slab_rows   : own particles per cell row into hist (device, ny int64) -> all-gather
 *   gs_slab_pack   : every own particle (S, RK4 base B and accumulator A, global index: 13
 *                    doubles) into send (device, n_own x 13) grouped by the owner of its row
 *                    (owner: device, ny int32); counts[world] (host, optional: NULL = the
 *                    driver knows them from the all-gathered histograms; else synchronises)
 *                    -> all-to-all -> gs_slab_unpack (the rank's new own particles)
 *   gs_slab_layout : own particles sorted by (cell, global index) into local positions
 *                    [own_begin, own_begin + n_own) of the n_loc local records (rows
 *                    [y_loc0, y_loc1) = own rows [y_own0, y_own1) + halo rows)
 *                    -> the halo slices of S and of the global indices (gs_slab_views) are
 *                    copied in from the neighbours' own blocks
 *   gs_slab_lists  : cell starts, own clusters (pairs restarting at every cell row: ncl = sum
 *                    over the own rows of ceil(count / 2)) and their lists over the local
 *                    particles; synchronises once (list capacity)
 * per RK4 stage: gs_slab_stage (the list sweep with the RK4 stage epilogue of the own rows fused
 * in; rebuild flag = some own particle moved more than skin * cutoff / 2 since the build, *flag of
 * gs_slab_views) -> the halo slices of S -> MAX all-reduce of the flags: rebuild before the next
 * stage.  The local records ping-pong between two buffers: a stage reads the current one (S of
 * gs_slab_views after the layout) and writes the own rows' next records into the other (S_alt),
 * which is current for the next stage — the halo slices go there.
 * Rows are bitwise independent of the number of ranks.  gs_slab_begin sets the own particles
 * (q, p: device (n_own, 2); gidx: device int32 global indices) and resets the status;
 * gs_slab_status decodes it with global indices (synchronises). */
typedef struct gs_slab_grid {
    double x0, y0, h;          /* grid origin and cell edge (= cutoff (1 + skin) / sub) */
    int32_t nx, ny, sub, hashed;
} gs_slab_grid_t;
int gs_slab_begin(gs_context* ctx, const gs_system_t* sys, int64_t n_glob, int64_t n_own, const double* q,
                  const double* p, const int32_t* gidx, void* stream);
int gs_slab_bbox(gs_context* ctx, double* b4, void* stream);
int gs_slab_grid(gs_context* ctx, const double* b4, gs_slab_grid_t* grid, void* stream);
int gs_slab_rows(gs_context* ctx, int64_t* hist, void* stream);
int gs_slab_pack(gs_context* ctx, const int32_t* owner, int32_t world, double* send, int64_t* counts, void* stream);
int gs_slab_unpack(gs_context* ctx, int64_t n_own, const double* recv, void* stream);
int gs_slab_layout(gs_context* ctx, int32_t y_own0, int32_t y_own1, int32_t y_loc0, int32_t y_loc1, int64_t own_begin,
                   int64_t n_loc, void* stream);
int gs_slab_views(gs_context* ctx, double** S, double** S_alt, int32_t** gidx, int32_t** flag);
int gs_slab_lists(gs_context* ctx, int64_t ncl, void* stream);
int gs_slab_stage(gs_context* ctx, const gs_system_t* sys, int32_t step, int32_t stage, double dt, void* stream);
int gs_slab_status(gs_context* ctx, gs_status_t* status, void* stream);

/* micro-benchmark used by bench.py for the FP64 roofline denominator: `iters` dependent
 * DFMA chains per thread on a full grid; returns the device time in *ms (host). */
int gs_fp64_peak_probe(gs_context* ctx, int32_t iters, double* ms, double* flops, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* GEOSHOOT_B200_H */

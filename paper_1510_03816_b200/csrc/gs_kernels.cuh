// gs_kernels.cuh — kernel launchers shared between the translation units of libgs_b200.so.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "gs_device.cuh"

namespace gsb {

// Derived per-system constants (host-computed once per call).
struct SysConst {
    int fam;
    double k1;        // exponent scale, see pair_accum
    double scale_q;   // peak (or 1)
    double scale_p;   // peak/alpha (conical) or peak/alpha^2 (gaussian)
    double sigma2;
    double cutoff;    // > 0: truncate pairs with d >= cutoff (cell path)
};

// Dense tiling: DB targets per CTA (one per thread), DT sources per shared-memory tile.
constexpr int kDB = 128;
constexpr int kDT = 256;

struct DensePlan {
    int64_t chunk;    // sources per CTA column (multiple of kDT)
    int nchunks;
};
DensePlan dense_plan(int64_t n, int sm_count);

// RHS partial sums of rows [row0, row0+nrows) against all n sources of S, one
// record (sum G p_j, sum c (q_i - q_j)) per (chunk, row): part[c * nrows + li].
void launch_dense_partial(const SysConst& sc, const double4* S, int64_t n, int64_t row0, int64_t nrows,
                          const DensePlan& plan, double4* part, DevStatus* st, unsigned long long event,
                          const double* tbl_dev, cudaStream_t stream);

// Peer-memory signalling fused into kernels (gs_p2p_*).  PeerWait: every CTA waits until its
// own counter flags[which] reaches target (gives up after timeout_ns, counted in flags[2]; once
// a timeout happened nobody waits any more).  PeerSignal: the last CTA to finish adds 1 to
// counter `which` of every rank (system-scope, after a system fence), using `done` (zero
// between launches) to detect it.  A null pointer disables either.
struct PeerWait {
    unsigned long long* flags;
    int which;
    unsigned long long target;
    long long timeout_ns;
};
struct PeerSignal {
    unsigned long long* const* Fp;
    int world, which;
    unsigned int* done;
};

__device__ __forceinline__ void block_wait(const PeerWait& w) {
    if (!w.flags) return;
    if (threadIdx.x == 0) {
        unsigned long long t0, t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        while (*((volatile unsigned long long*)&w.flags[w.which]) < w.target &&
               *((volatile unsigned long long*)&w.flags[2]) == 0) {
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if ((long long)(t - t0) > w.timeout_ns) {
                atomicAdd(&w.flags[2], 1ull);
                break;
            }
            __nanosleep(128);
        }
        __threadfence_system();
    }
    __syncthreads();
}

__device__ __forceinline__ void block_signal_last(const PeerSignal& s) {
    if (!s.Fp) return;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();  // this CTA's stores (local and peer) are visible system-wide
        const unsigned prev = atomicAdd(s.done, 1u);
        if (prev == gridDim.x - 1) {
            *s.done = 0;
            __threadfence_system();
            for (int r = 0; r < s.world; ++r) atomicAdd_system(s.Fp[r] + s.which, 1ull);
        }
    }
}

// Symmetric all-pairs RHS of all n rows (single rank, gs_sym.cu): each unordered pair once;
// row i gets nsb partials part[slot * pstride + i], pstride = nb * kDB.
constexpr int kSymMaxG = 8;  // 8 blocks per superblock: symmetric dense up to N = 256 * 8 * 128 = 262144
struct SymPlan {
    int nb;           // 128-row blocks
    int G;            // blocks per superblock
    int nsb;          // superblocks = partial slots per row
    int64_t pstride;  // nb * kDB
    bool ok;          // partial buffer stays bounded (nsb <= 256)
};
SymPlan sym_plan(int64_t n);
long long sym_ctas(int64_t n);  // work items (superblock pairs) of one symmetric RHS
// CTAs [cta0, cta1) of the superblock-pair list (cta1 < 0: all).  A multi-GPU rank runs its
// share of the list; the slots of the other ranks' items must be zero in `part`.
void launch_dense_sym(const SysConst& sc, const double4* S, int64_t n, double4* part, int64_t pstride, DevStatus* st,
                      unsigned long long event, const double* tbl_dev, cudaStream_t stream, long long cta0 = 0,
                      long long cta1 = -1, PeerWait wait = PeerWait{nullptr, 0, 0, 0});
// R[i] = sum over slots of part[slot * pstride + i] (fixed order), i < n.
void launch_slot_reduce(const double4* part, int nslots, int64_t pstride, int64_t n, double4* R, cudaStream_t stream);
// The same over the slots listed per row superblock (a rank's share of the superblock pairs);
// `sig` (optional) signals the peers once all of R is written.
void launch_slot_reduce_list(const double4* part, int64_t pstride, int64_t n, int rows_per_sb, int nsb,
                             const int* slots, const int* counts, double4* R, cudaStream_t stream,
                             PeerSignal sig = PeerSignal{nullptr, 0, 0, nullptr});
// Superblock pair (SI, SJ), SI <= SJ, of work item t (row-major over the upper triangle).
void sym_pair_of(long long t, int nsb, long long* SI, long long* SJ);

// Gram matrix of the kernel over q (n x n row-major), first coincident pair -> *bad (i*n+j).
void launch_gram(const SysConst& sc, const double* q, int64_t n, double* K, unsigned long long* bad,
                 const double* tbl_dev, cudaStream_t stream);

// Velocity field u(x_k) = sum_j G(|x_k - q_j|) p_j at m points x (m x 2) from the packed
// state S (n records); part holds plan.nchunks * m double2 partials.
DensePlan velocity_plan(int64_t n, int64_t m, int sm_count);
void launch_velocity_field(const SysConst& sc, const double4* S, int64_t n, const double* x, int64_t m,
                           const DensePlan& plan, double2* part, double* u, const double* tbl_dev,
                           cudaStream_t stream);

// Finish modes
constexpr int kFinRhs = 0;    // write dq, dp rows ((nrows, 2) AoS)
constexpr int kFinStage = 1;  // RK4 stage epilogue (integrator.py:98-114)
constexpr int kFinHam = 2;    // ham[li] = p_i . dq_i (sigma2 excluded)

struct FinishArgs {
    const double4* part;
    int nchunks;
    int64_t pstride;   // distance between chunk partials of one row (0: nrows)
    int64_t nrows, row0;
    double4* S;        // stage state (all n rows)
    double4* B;        // base rows (nrows)
    double4* A;        // RK accumulator rows (nrows)
    double* dq;        // kFinRhs
    double* dp;
    double* ham;       // kFinHam
    int stage;
    double dt;
    DevStatus* st;
    unsigned long long event;
};
void launch_finish(int mode, const SysConst& sc, const FinishArgs& a, cudaStream_t stream);

// RK4 stage epilogue of row li in the reference's evaluation order (integrator.py:98-114):
//   stage inputs q + (0.5 dt) k_s, q + dt k_3; combine q + (dt/6) (((k1 + 2k2) + 2k3) + k4).
// Updates the row's accumulator / base records and returns the next stage input.
__device__ __forceinline__ double4 stage_update(const FinishArgs& a, int64_t li, double dqx, double dqy, double dpx,
                                                double dpy) {
    double4 b = a.B[li];
    double4 acc;
    double4 nxt;
    if (a.stage == 0) {
        acc = make_double4(dqx, dqy, dpx, dpy);
    } else {
        acc = a.A[li];
        const double w = (a.stage == 3) ? 1.0 : 2.0;
        acc.x = __dadd_rn(acc.x, __dmul_rn(w, dqx));
        acc.y = __dadd_rn(acc.y, __dmul_rn(w, dqy));
        acc.z = __dadd_rn(acc.z, __dmul_rn(w, dpx));
        acc.w = __dadd_rn(acc.w, __dmul_rn(w, dpy));
    }
    if (a.stage < 3) {
        const double c = (a.stage == 2) ? a.dt : 0.5 * a.dt;
        nxt.x = __dadd_rn(b.x, __dmul_rn(c, dqx));
        nxt.y = __dadd_rn(b.y, __dmul_rn(c, dqy));
        nxt.z = __dadd_rn(b.z, __dmul_rn(c, dpx));
        nxt.w = __dadd_rn(b.w, __dmul_rn(c, dpy));
        a.A[li] = acc;
    } else {
        const double c = a.dt / 6.0;
        nxt.x = __dadd_rn(b.x, __dmul_rn(c, acc.x));
        nxt.y = __dadd_rn(b.y, __dmul_rn(c, acc.y));
        nxt.z = __dadd_rn(b.z, __dmul_rn(c, acc.z));
        nxt.w = __dadd_rn(b.w, __dmul_rn(c, acc.w));
        a.B[li] = nxt;
    }
    return nxt;
}

// Stage epilogue fused with the cluster-list gather (gs_verlet.cu, single rank, all rows): the new
// record also goes to its sorted slot Ss[inv[i]], and the last CTA decides the rebuild trigger (a
// particle farther than sqrt(thr2) from its position Xb at the last build): the next stage's
// IF-node condition (use_cond) or flags[3].
struct VerletFuse {
    double4* Ss;
    const int* inv;
    const double2* Xb;
    double thr2;
    unsigned* flags;
    cudaGraphConditionalHandle cond;
    int use_cond;
    int defer;    // 1: only store the sorted record; launch_verlet_trigger (gs_verlet.cu) reads it in
                  // sorted order with the build position and decides
};
void launch_finish_verlet(const SysConst& sc, const FinishArgs& a, const VerletFuse& f, cudaStream_t stream);
// Stage epilogue of rows [row0, row0 + nrows) from the raw row sums of all `world` ranks
// (Rp[w], full length, summed in rank order), storing each new stage record into Sp[w] of
// every rank (peer memory).
void launch_finish_p2p(const SysConst& sc, const FinishArgs& a, const double4* const* Rp, double4* const* Sp,
                       int world, PeerWait wait, PeerSignal sig, cudaStream_t stream);

// Small-N persistent kernel: a whole evolve or a whole match per thread-block cluster
// (n <= kSmallMax), see gs_small.cu.
constexpr int kSmallMax = 512;
constexpr int kSmallThreads = 512;

struct SmallResult {
    double hamiltonian;
    double final_residual;
    unsigned long long fail_event;   // kNoEvent if the shoots never failed
    unsigned long long pair_key;
    int outcome;                     // GS_MATCH_*
    int iterations;
    int fail_iter;
    int pad;
};

// Per-trajectory constants.  A batched launch runs one CTA per item (SURVEY.md §8(f2):
// convergence-sweep cells, cluster-test pairs, Newton Jacobian columns); the family must be
// uniform across a launch (it selects the template instance).
struct SmallItem {
    SysConst sc;
    double t_final;
    double h, epsilon;
    int steps;
    int max_iter, stop_rule, norm;
};

constexpr int kMaxCluster = 8;  // CTAs per item (portable cluster size)

struct SmallArgs {
    int64_t n;
    int64_t batch;         // items; the grid is batch x cluster CTAs
    int cluster;           // CTAs per item (1..kMaxCluster), one thread-block cluster
    int split;             // lanes per row (power of two <= 32), see small_threads
    int mode;              // 0 evolve, 1 match
    int capture_every;     // evolve, batch == 1 only
    SmallItem item;        // used when items == null
    const SmallItem* items;  // device, batch entries (or null)
    // evolve: q_in (+ b*q_stride), p_in (+ b*2n) in; q_out/p_out (+ b*2n) out; frames or null
    const double* q_in;
    int64_t q_stride;      // doubles between items' q0 / q_in (0: shared)
    const double* p_in;
    double* q_out;
    double* p_out;
    double* frames;
    // match
    const double* target;
    int64_t t_stride;      // doubles between items' targets (0: shared)
    double* history;       // device, + b*hist_stride
    int64_t hist_stride;
    SmallResult* result;   // device, + b
    DevStatus* st;         // evolve: failure record, + b
    // velocity update space (shooting.py:263-265): lower Cholesky factor of the Gram matrix
    // over q0, row-major n x n (+ b*L_stride; 0: shared), or null for the momentum update
    const double* L;
    int64_t L_stride;
    int L_smem;            // stage L in shared memory (row stride n + 1)
};
size_t small_smem_bytes(const SmallArgs& a);
// Threads per CTA for n rows on `cluster` CTAs; *split = lanes per row.
int small_threads(int64_t n, int cluster, int* split);
int launch_small(int fam, const SmallArgs& a, const double* tbl_dev, cudaStream_t stream);

}  // namespace gsb

// gs_context.cuh — the library context (opaque gs_context of include/geoshoot_b200.h) and the
// host helpers shared by the C-ABI translation units: gs_api.cu (sessions, RHS, evolve, match,
// stage API), gs_batch.cu (batched trajectories), gs_p2p.cu (peer-memory stage exchange).
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/geoshoot_b200.h"
#include "gs_cell.cuh"
#include "gs_kernels.cuh"

namespace gsapi {

// NVTX range for the lifetime of a scope (every C-ABI call, every host-driven feedback iteration
// and RK stage): visible in nsys / ncu timelines, free when no tool is attached (nvtx3 is
// header-only and loads a tool only through NVTX_INJECTION64_PATH).
struct NvtxScope {
    explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
    ~NvtxScope() { nvtxRangePop(); }
    NvtxScope(const NvtxScope&) = delete;
    NvtxScope& operator=(const NvtxScope&) = delete;
};

extern thread_local std::string g_last_error;
int fail(int code, const std::string& msg);

}  // namespace gsapi

#define GS_CUDA(call)                                                                                   \
    do {                                                                                                \
        cudaError_t e_ = (call);                                                                        \
        if (e_ != cudaSuccess)                                                                          \
            return gsapi::fail(GS_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));        \
    } while (0)

namespace gsapi {

using namespace gsb;

template <typename T>
struct DevBuf {
    T* ptr = nullptr;
    size_t cap = 0;  // elements
    cudaError_t ensure(size_t n) {
        if (n <= cap) return cudaSuccess;
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        cap = 0;
        cudaError_t e = cudaMalloc(&ptr, std::max<size_t>(n, 1) * sizeof(T));
        if (e == cudaSuccess) cap = n;
        return e;
    }
    void release() {
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        cap = 0;
    }
};

}  // namespace gsapi

using gsapi::DevBuf;
using namespace gsb;  // internal header: the context holds the kernels' types

// State of the device-resident feedback loop (gs_match, n above the small-N kernel): what the
// host loop of shooting.py:259-301 keeps in locals, kept on the device between iterations.
struct MatchLoop {
    int it, iters, outcome, have_initial, fail_it, pad;
    double initial, nrm;
};

struct gs_context {
    int device = 0;
    int sm_count = 148;
    DevBuf<double> tbl;
    DevBuf<DevStatus> st;
    DevStatus* st_host = nullptr;   // pinned
    double* scal_host = nullptr;    // pinned scratch (16 doubles)
    MatchLoop* mloop_host = nullptr; // pinned
    // stage session
    DevBuf<double4> S, B, A, part;
    int64_t n = 0, row0 = 0, row1 = 0;
    // match / reductions
    DevBuf<double> q0, tgt, p, resid, red, ham, hist, scal;
    DevBuf<SmallResult> small_res;
    DevBuf<MatchLoop> mloop;
    DevBuf<double> ep;               // the loop graph's endpoint buffer
    DevBuf<SmallItem> b_items;       // batched launches: per-item constants
    DevBuf<DevStatus> b_st;          // batched evolve: per-item failure records
    DevBuf<double2> vf_part;         // velocity-field chunk partials
    DevBuf<double> cg;               // matrix-free Gram solve: r, d, K d, scratch (4 x 2n)
    // rank split of the symmetric kernel: slots written per row superblock for the cached range
    DevBuf<int> sym_slots, sym_counts;
    int64_t sym_key_n = -1, sym_key_b = -1, sym_key_e = -1;
    // fused stage exchange over peer memory (gs_p2p_*): this rank's raw row sums, the signal
    // counters ([0] sums ready, [1] stage records written, [2] wait timeouts) and the ranks' pointers
    struct P2P {
        int world = 0, rank = 0;
        DevBuf<double4> R;
        DevBuf<unsigned long long> flags;
        DevBuf<const double4*> Rp;
        DevBuf<double4*> Sp;
        DevBuf<unsigned long long*> Fp;
        DevBuf<unsigned> done;           // block-completion counters of the signalling kernels
        std::vector<void*> opened;       // IPC mappings to close
        unsigned long long epoch = 0;    // stages completed since the peers were set
        long long timeout_ns = 10000000000ll;
    } p2p;
    // profiling: CUDA events around every pair-kernel launch, kernel launch counter
    int prof_on = 0;
    std::vector<cudaEvent_t> prof_events;
    size_t prof_used = 0;
    long long launches = 0;
    long long pair_launches = 0;
    long long host_pairs = 0;     // dense / small-kernel pair count (known on the host)
    // cell list (gs_cell.cu)
    DevBuf<unsigned> c_keys, c_keys_sorted, c_vals, c_perm;
    DevBuf<int> c_start;
    DevBuf<double4> c_Ss, c_Ss2;        // sorted records; c_Ss2: ping-pong half for the fused list epilogue
    DevBuf<float2> c_Sf;
    DevBuf<double> c_bbox;
    DevBuf<GridParams> c_gp;
    DevBuf<int> c_tlist, c_nsel;
    DevBuf<unsigned char> c_cub;
    DevBuf<unsigned long long> c_acc;   // accepted pairs (profiling)
    DevBuf<unsigned long long> gram_bad;  // gs_gram's first coincident pair
    size_t c_cub_bytes = 0;
    int cell_on = 0;                    // path of the current call
    int cell_err = 0;                   // sticky: a cell build failed to enqueue (reported by the API call)
    // cluster Verlet lists of the cell path in multi-RHS calls (gs_verlet.cu)
    DevBuf<int> v_list, v_len, v_inv;
    cudaGraphConditionalHandle v_next_cond{};  // IF-node condition the last fused epilogue sets
    int v_next_valid = 0;
    DevBuf<long long> v_cnt, v_ofs;
    DevBuf<double2> v_xb;
    DevBuf<unsigned> v_flags;
    DevBuf<unsigned long long> v_over;
    DevBuf<unsigned char> v_scan;
    int verlet_on = 1;                  // GS_B200_VERLET=0: the per-RHS cell sweep everywhere
    int verlet_call = 0;                // this call evaluates its RHS through the lists
    int64_t v_list_n = -1;              // n and cutoff the list buffer was sized for
    double v_list_cutoff = 0.0;
    int verlet_retries = 0;
    double verlet_skin = -1.0;          // GS_B200_SKIN (< 0: by n, see verlet_ws)
    int skin_adapt = 1;                 // GS_B200_SKIN_ADAPT: adaptive skin on the relative-trigger path
    DevBuf<double> v_skin;              // its device state {skin, RHS per unit skin}
    int64_t verlet_fuse_max_n = 131072; // lists: epilogue fused into the sweep below this n (GS_B200_VERLET_FUSE_MAX_N)
    int verlet_rel = 1;                 // large clouds: rebuild on neighbours' relative displacement (GS_B200_VERLET_REL)
    DevBuf<unsigned> v_box;             // coarse-cell displacement boxes (k_verlet_trigger)
    double verlet_slack = 1.5;          // list buffer = (1 + slack) x the sizing build (GS_B200_VERLET_SLACK)
    cudaStream_t cap_stream2 = nullptr; // captures the conditional rebuild bodies
    // slab decomposition of the cell path across ranks (gs_slab.cu): this rank's own particles
    // (contiguous cell rows of the global grid) + the halo rows, all in global sorted order
    struct Slab {
        int64_t n_glob = 0, n_own = 0, n_loc = 0, own_begin = 0, ncl = 0;
        int tpl = 4;
        double skin = 0.05, cutoff = 0.0, rl = 0.0;
        int own_sorted = 0;                 // own particles live in the local layout (else in the *_u arrays)
        GridParams g{};                     // host copy of the last grid
        int y_own0 = 0, y_own1 = 0, y_loc0 = 0, y_loc1 = 0;
        DevBuf<double4> S, S2;              // n_loc + 1 local records (S[n_loc]: sentinel far record), ping-pong:
        int par = 0;                        // the stage reads buffer `par` and writes its own rows into the other
        DevBuf<unsigned> gidx;              // n_loc: global index of each local particle
        DevBuf<double4> B, A;               // own particles, local sorted order
        DevBuf<double2> Xb;                 // own particles: positions at the last build
        DevBuf<double4> Su, Bu, Au;         // own particles in arrival order (begin / after a migration)
        DevBuf<unsigned> gu;
        DevBuf<unsigned long long> skey, skey2;  // (cell, global index) sort keys of the own particles
        DevBuf<unsigned> sval, sval2;
        DevBuf<unsigned char> cub;
        DevBuf<unsigned> keys;              // n_loc local cell keys
        DevBuf<int> start, cfirst, head, len, list;
        DevBuf<float2> Sf;
        DevBuf<GridParams> gp;
        DevBuf<long long> cnt, ofs;
        DevBuf<double> red, b4;
        DevBuf<int> dest;
        DevBuf<unsigned long long> dcount;
        DevBuf<unsigned> flags;             // [0] rebuild wanted (set by the last stage's epilogue)
        DevBuf<unsigned long long> over;
    } slab;
    // CUDA graph of a whole evolve (all steps x 4 stages), re-launched while its key holds
    struct Graph {
        cudaGraphExec_t exec = nullptr;
        std::vector<double> key;
        std::vector<cudaEvent_t> ev;    // profiling events captured inside the graph
        long long launches = 0, pair_launches = 0, host_pairs = 0;
    } graph;
    // the device-resident feedback loop (conditional WHILE graph), re-launched while its key holds
    struct LoopGraph {
        cudaGraphExec_t exec = nullptr;
        std::vector<double> key;
        long long launches = 0, pair_launches = 0, host_pairs = 0;  // per iteration
    } mgraph;
    std::vector<cudaEvent_t>* capture_events = nullptr;  // non-null while capturing
    cudaStream_t cap_stream = nullptr;
    int graphs_on = 1;
    int devloop_on = 1;                 // large-N matches as one conditional-WHILE graph
    int sym_on = 1;                     // symmetric dense kernel for full-row RHS
    double prof_ms_acc = 0.0;           // pair-kernel time already harvested (graph replays)
};

namespace gsapi {

constexpr int kRedBlocks = 512;
constexpr int64_t kStatePad = 64;  // spare records after S for equal-size all-gather slices

inline unsigned nblk(int64_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

int check_system(const gs_system_t* sys);
// shooting.py:66-100 / integrator.py:35-43 validation of one (system, match config) item
int check_match(const gs_system_t* sys, const gs_match_config_t* cfg);
SysConst make_const(const gs_system_t* sys);
void decode_status(const DevStatus& d, int64_t n, gs_status_t* out);
int fetch_status(gs_context* ctx, cudaStream_t s, int64_t n, gs_status_t* out);
cudaEvent_t prof_event(gs_context* ctx);
void prof_mark(gs_context* ctx, cudaStream_t stream);
// small-N cluster kernel: CTAs per item, launch setup, eligibility, per-item constants, result
int small_cluster(int64_t n);
void small_setup(SmallArgs& a, int64_t n);
bool use_small(const gs_system_t* sys, int64_t n);
SmallItem small_item(const SysConst& sc, const gs_match_config_t* cfg);
void small_to_result(const SmallResult& r, int64_t n, gs_match_result_t* out);
// this rank's share [part_begin, part_end) of the symmetric pair list: raw row sums of all rows
// into R; sig / wait: optional peer signalling (gs_p2p_*)
int pairs_sym_impl(gs_context* ctx, const gs_system_t* sys, int32_t step, int32_t stg, int64_t part_begin,
                   int64_t part_end, double* R, void* stream, PeerSignal sig = PeerSignal{nullptr, 0, 0, nullptr},
                   PeerWait wait = PeerWait{nullptr, 0, 0, 0});

}  // namespace gsapi

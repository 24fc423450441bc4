// capi.cu — extern "C" entry points of libpipeplan_b200.so (include/pipeplan_b200.h).
#include <algorithm>
#include <cmath>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "common.cuh"

namespace pp {
__global__ void k_prep(pp_batch b);
__global__ void k_prep_p(const pp_batch* bp);
__global__ void k_base_p(const pp_batch* bp, int full_rows);
__global__ void k_sdedup_p(const pp_batch* bp);
__global__ void k_stab_p(const pp_batch* bp);
__global__ void k_stab_big_p(const pp_batch* bp);
__global__ void k_stab_big(pp_batch b);
__global__ void k_expand_s_p(const pp_batch* bp, int j, int rfirst, int rlast);
__global__ void k_expand_m_p(const pp_batch* bp, int j, int rb);
__global__ void k_combine_s_p(const pp_batch* bp, int j, int r0);
__global__ void k_combine_bis_p(const pp_batch* bp, int j, int r0, int rg, int rb);
__global__ void k_backtrack_p(const pp_batch* bp);
__global__ void k_phi(pp_batch b);
__global__ void k_base(pp_batch b, int full_rows);
__global__ void k_expand(pp_batch b, int j, int planes_r, int ybase);
__global__ void k_combine_diag(pp_batch b, int j, int planes_x);
__global__ void k_expand_s(pp_batch b, int j);
__global__ void k_sdedup(pp_batch b);
__global__ void k_stab(pp_batch b);
__global__ void k_combine_s(pp_batch b, int j);
__global__ void k_dp_inst(pp_batch b, int smem_doubles);
__global__ void k_dp_inst2(pp_batch b);
__global__ void k_backtrack(pp_batch b);
__global__ void k_query(pp_batch b, int n, const int* qi, const int* ql, const int* qx, const int* qr,
                        const int* qd, int max_xi, double* w, int* frag, int* feas);
template <bool SMEM> __global__ void k_rdo(pp_batch b, int resume);
template <int MAXS> __global__ void k_rdo_plan(pp_batch b, int round, int predict);
__global__ void k_rdo_hash(pp_batch b, int dedup);
__global__ void k_rdo_rep(pp_batch b);
__global__ void k_rdo_insert(pp_batch b);
__global__ void k_rdo_copy(pp_batch b);
template <bool SMEM> __global__ void k_rdo_cut(pp_batch b, int per_warp);
template <bool SMEM>
__global__ void k_min_cut(pp_batch b, int k, const int* verts, int n, unsigned char* in_a, double* weight);
__global__ void k_pe_sweep(pp_batch b);
__global__ void k_pe_sweep_w(pp_batch b);
__global__ void k_replay_w(pp_batch b);
__global__ void k_event_merge(pp_batch b);
__global__ void k_event_rank(pp_batch b);
__global__ void k_select(pp_batch b);
__global__ void k_replay(pp_batch b);
__global__ void k_sim_plans(pp_batch b, pp_sim_batch s);
__global__ void k_peak_minmax(double* out, int iters, double seed);
}  // namespace pp

using namespace pp;

static thread_local std::string g_err;
static std::atomic<long long> g_launches{0};

static int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define PP_CHECK_LAUNCH(name)                                                                        \
    do {                                                                                             \
        g_launches.fetch_add(1, std::memory_order_relaxed);                                          \
        cudaError_t e_ = cudaGetLastError();                                                         \
        if (e_ != cudaSuccess) return fail(PP_ECUDA, "%s launch: %s", name, cudaGetErrorString(e_)); \
    } while (0)

static inline int ceil_div(int a, int b) { return (a + b - 1) / b; }

// Upper bound on the per-item CTA split of k_combine_s (PP_COMBINE_SPLIT env, default 8):
// items are split only while the whole step has fewer items than SMs.
static int read_max_parts() {
    const char* e = getenv("PP_COMBINE_SPLIT");
    const int v = e ? atoi(e) : 8;
    return v < 1 ? 1 : (v > 8 ? 8 : v);
}
static const int g_max_parts = read_max_parts();
// per-step combine: split items until a launch (over the whole batch) has about
// PP_COMBINE_WAVES x SMs CTAs
static int read_combine_waves() {
    const char* e = getenv("PP_COMBINE_WAVES");
    const int v = e ? atoi(e) : 2;   // n = 1 C3 DP: 1.25 ms at 1 wave, 1.21 at 2, 1.24 at 3
    return v < 1 ? 1 : (v > 16 ? 16 : v);
}
static const int g_combine_waves = read_combine_waves();
// expand CTAs get 256 threads when a step has <= this many rows per SM (PP_EXPAND_WIDE env)
static const int g_expand_wide = getenv("PP_EXPAND_WIDE") ? atoi(getenv("PP_EXPAND_WIDE")) : 2;
// rows per expand CTA when a step has more than PP_EXPAND_RB_MIN rows per SM
// (PP_EXPAND_RB env, default 4; the chan block is shared by the CTA's rows)
static const int g_expand_rb = getenv("PP_EXPAND_RB") ? std::max(1, atoi(getenv("PP_EXPAND_RB"))) : 2;   // r02: 2 rows x 80 registers (3 CTAs/SM) beat 4 rows x 126 (C3 n = 12 DP 2.56 -> 2.50 ms)
static const int g_expand_rb_min = getenv("PP_EXPAND_RB_MIN") ? atoi(getenv("PP_EXPAND_RB_MIN")) : 4;
static constexpr int64_t EX_SMEM_DOUBLES = 12288;   // 96 KB: two 256-thread CTAs per SM
// per-step chain with the critical path (items r = 1) split from the bulk, for
// batches of at most PP_DP_SPLIT instances (default 2; measured on C3: n = 1
// DP 1.20 -> 1.10 ms, n = 3 equal, n = 12 2.71 -> 3.52 ms: twice the launches)
static const int g_dp_split = getenv("PP_DP_SPLIT") ? atoi(getenv("PP_DP_SPLIT")) : 2;
// CTAs (tile parts) of the critical item r = 1 in the split chain (PP_C1_PARTS env)
static const int g_c1_parts = getenv("PP_C1_PARTS") ? std::max(1, std::min(64, atoi(getenv("PP_C1_PARTS")))) : 32;
// programmatic dependent launch in the per-step chain (PP_PDL=0 disables)
static const int g_pdl = getenv("PP_PDL") ? atoi(getenv("PP_PDL")) : 1;
// combine kernel of the per-step schedule: 1 = crossing search (combine_bis.cu),
// 0 = exhaustive register tiles (k_combine_s_p), 2 = auto; same bits either way
static const int g_bis_rb = getenv("PP_BIS_RB") ? atoi(getenv("PP_BIS_RB")) : 0;   // rows per thread (0 = auto)
// (n = 1 C3 DP: 0.98 ms at 2 waves, 0.94 at 1-1.5)
static const double g_bis_waves = getenv("PP_BIS_WAVES") ? atof(getenv("PP_BIS_WAVES")) : 1.5;
static std::atomic<int> g_combine_kind{getenv("PP_COMBINE_BIS") ? atoi(getenv("PP_COMBINE_BIS")) : 2};
// auto (kind 2): the crossing search for batches of at most this many instances
// (latency-bound chains), the register tiles above it (throughput)
static const int g_bis_max_inst = getenv("PP_BIS_MAX_INST") ? atoi(getenv("PP_BIS_MAX_INST")) : 1;

static int num_sms() {
    static thread_local int dev = -1, sms = 148;
    int d = 0;
    cudaGetDevice(&d);
    if (d != dev) {
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
        dev = d;
    }
    return sms;
}
static inline cudaStream_t S(void* s) { return (cudaStream_t)s; }

extern "C" {

const char* pp_version(void) { return "pipeplan_b200 0.1.0 (sm_100a, fp64 bit-exact)"; }
const char* pp_last_error(void) { return g_err.c_str(); }
int64_t pp_launch_count(void) { return g_launches.load(); }

int pp_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) { cudaGetLastError(); return 0; }
    return n;
}

int pp_layout(int32_t n, const int32_t* L, const int32_t* V, const int32_t* M, const int32_t* flags,
              pp_instance* inst, int64_t* n_layer, int64_t* n_bw, int64_t* n_order, int64_t* n_sweep,
              int64_t* n_stage, int64_t* n_ev, int64_t* n_ar, int64_t* n_ws) {
    int64_t lo = 0, bo = 0, oo = 0, so = 0, sto = 0, wo = 0, eo = 0, ao = 0;
    for (int k = 0; k < n; ++k) {
        if (L[k] < 1 || L[k] > PP_MAX_LAYERS) return fail(PP_EINVAL, "instance %d: L=%d outside 1..%d", k, L[k], PP_MAX_LAYERS);
        if (V[k] < 1 || V[k] > PP_MAX_GPUS) return fail(PP_EINVAL, "instance %d: V=%d outside 1..%d", k, V[k], PP_MAX_GPUS);
        if (M[k] < 1) return fail(PP_EINVAL, "instance %d: microbatch count must be positive", k);
        pp_instance& I = inst[k];
        I.L = L[k]; I.V = V[k]; I.M = M[k]; I.flags = flags[k];
        I.layer_off = lo; lo += L[k];
        I.bw_off = bo; bo += (int64_t)V[k] * V[k];
        I.order_off = oo; oo += V[k];
        I.sweep_off = so; so += V[k];
        I.stage_off = sto; sto += (int64_t)V[k] * (V[k] + 1) / 2;
        I.ws_off = wo; wo += ws_layout(L[k], V[k]).total;
        I.ev_off = eo; eo += (int64_t)M[k] * (4 * V[k] - 3);
        I.ar_off = ao; ao += V[k];
    }
    *n_layer = lo; *n_bw = bo; *n_order = oo; *n_sweep = so; *n_stage = sto; *n_ev = eo; *n_ar = ao; *n_ws = wo;
    return PP_OK;
}

// Speculative rounds before the sequential finisher (rdo.cu); 0 = sequential only.
static std::atomic<int> g_rdo_rounds{1};

int pp_rdo_set_rounds(int32_t rounds) {
    if (rounds < 0 || rounds > 64) return fail(PP_EINVAL, "rdo rounds %d outside 0..64", rounds);
    return g_rdo_rounds.exchange(rounds);
}

// Workspace bounds check (pp_batch.ws_doubles > 0): the instance table lives in
// device memory, so it is read back once (small, stream-ordered) and every
// instance's shape and workspace range validated before any kernel touches ws.
static int check_ws(const pp_batch* b, void* stream) {
    if (b->n_inst > 0 && b->ws == nullptr)
        return fail(PP_EINVAL, "pp_batch.ws is NULL: RDO / DP / sweep need the pp_layout workspace "
                               "(only pp_phi and pp_simulate run without one)");
    if (b->ws_doubles <= 0 || b->n_inst <= 0) return PP_OK;
    std::vector<pp_instance> h((size_t)b->n_inst);
    if (cudaMemcpyAsync(h.data(), b->inst, sizeof(pp_instance) * h.size(), cudaMemcpyDeviceToHost, S(stream)) !=
            cudaSuccess ||
        cudaStreamSynchronize(S(stream)) != cudaSuccess)
        return fail(PP_ECUDA, "workspace check: %s", cudaGetErrorString(cudaGetLastError()));
    for (int k = 0; k < b->n_inst; ++k) {
        const pp_instance& I = h[(size_t)k];
        if (I.L < 1 || I.L > PP_MAX_LAYERS || I.V < 1 || I.V > PP_MAX_GPUS || I.L > b->max_L || I.V > b->max_V)
            return fail(PP_EINVAL, "instance %d: L=%d V=%d outside the batch limits", k, I.L, I.V);
        const int64_t need = ws_layout(I.L, I.V).total;
        if (I.ws_off < 0 || I.ws_off + need > b->ws_doubles)
            return fail(PP_EINVAL, "instance %d: workspace [%lld, %lld) exceeds ws_doubles %lld", k,
                        (long long)I.ws_off, (long long)(I.ws_off + need), (long long)b->ws_doubles);
    }
    return PP_OK;
}

// RDO deduplication across a batch (rdo.cu).  RDO is latency-bound (one CTA per
// instance), so deduplicating only saves SM time once a batch has more
// instances than ~2 waves of SMs; below that it is skipped (C3, 12 instances of
// one cluster: RDO 0.37 ms either way).  PP_RDO_DEDUP: 0 off, 1 auto, 2 always.
static std::atomic<int> g_rdo_dedup{getenv("PP_RDO_DEDUP") ? atoi(getenv("PP_RDO_DEDUP")) : 1};

int pp_rdo_set_dedup(int32_t mode) { return g_rdo_dedup.exchange(mode < 0 || mode > 2 ? 1 : mode); }

int pp_rdo(const pp_batch* b, void* stream) {
    if (b->n_inst <= 0) return PP_OK;
    if (int rc = check_ws(b, stream)) return rc;
    const int V = b->max_V;
    const int dm = g_rdo_dedup.load();
    const int dedup = b->n_inst > 1 && (dm == 2 || (dm == 1 && b->n_inst > 2 * num_sms()));
    k_rdo_hash<<<b->n_inst, 32, 0, S(stream)>>>(*b, dedup);
    PP_CHECK_LAUNCH("k_rdo_hash");
    if (dedup) {
        k_rdo_insert<<<(b->n_inst + 127) / 128, 128, 0, S(stream)>>>(*b);
        PP_CHECK_LAUNCH("k_rdo_insert");
        k_rdo_rep<<<b->n_inst, 32, 0, S(stream)>>>(*b);
        PP_CHECK_LAUNCH("k_rdo_rep");
    }
    const int in_smem = V <= RDO_SMEM_MAX;
    const int rounds = V >= 2 ? g_rdo_rounds.load() : 0;
    if (rounds > 0) {
        const size_t plan_smem = rdo_plan_smem(V);
        const size_t cut_smem = (in_smem ? sizeof(double) * V * V : 0) + sizeof(int) * V + V + 16;
        // a batch above RDO_SMEM_MAX may still hold instances below it: their cuts run
        // in the shared-memory variant (k_rdo_cut<false> has no scratch for them)
        const int vs = V < RDO_SMEM_MAX ? V : RDO_SMEM_MAX;
        const size_t cut_smem_s = sizeof(double) * vs * vs + sizeof(int) * vs + vs + 16;
        // register slots of the largest group: the plan kernel instantiated for the batch's V
        void (*plan)(pp_batch, int, int) = V <= 32 ? k_rdo_plan<1> : V <= 64 ? k_rdo_plan<2> :
                                           V <= 128 ? k_rdo_plan<4> : V <= 256 ? k_rdo_plan<8> : k_rdo_plan<16>;
        cudaFuncSetAttribute(plan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)plan_smem);
        // cuts per CTA (one per warp; per-warp shared slices 16-byte aligned).  Four
        // per CTA for V <= 32 measured slower on C4 (RDO 0.50 -> 0.62 ms,
        // profiles/r02b_rdo_cut_wpc_ab.txt): one warp per CTA
        const int wpc = 1;
        const size_t pw_s = (cut_smem_s + 15) & ~size_t(15), pw = (cut_smem + 15) & ~size_t(15);
        cudaFuncSetAttribute(k_rdo_cut<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(pw_s * wpc));
        const dim3 gc(b->n_inst, (V - 1 + wpc - 1) / wpc);
        for (int r = 0; r <= rounds; ++r) {
            plan<<<b->n_inst, 32 * RDO_WARPS, plan_smem, S(stream)>>>(*b, r, r < rounds);
            PP_CHECK_LAUNCH("k_rdo_plan");
            if (r == rounds) break;
            k_rdo_cut<true><<<gc, 32 * wpc, pw_s * wpc, S(stream)>>>(*b, (int)pw_s);
            if (!in_smem) k_rdo_cut<false><<<gc, 32 * wpc, pw * wpc, S(stream)>>>(*b, (int)pw);
            PP_CHECK_LAUNCH("k_rdo_cut");
        }
    }
    const size_t smem = (in_smem ? sizeof(double) * V * V : 0) + rdo_state_bytes(V);
    if (in_smem) {
        cudaFuncSetAttribute(k_rdo<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_rdo<true><<<b->n_inst, 32 * RDO_WARPS, smem, S(stream)>>>(*b, rounds > 0);
    } else {
        cudaFuncSetAttribute(k_rdo<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_rdo<false><<<b->n_inst, 32 * RDO_WARPS, smem, S(stream)>>>(*b, rounds > 0);
    }
    PP_CHECK_LAUNCH("k_rdo");
    if (dedup) {
        k_rdo_copy<<<b->n_inst, 64, 0, S(stream)>>>(*b);
        PP_CHECK_LAUNCH("k_rdo_copy");
    }
    return PP_OK;
}

static int prm_chain(const pp_batch* b, void* stream, int total_inst);
static int prm_chain_p(const pp_batch* b, const pp_batch* db, void* stream, int total_inst);
static int prm_chain_split_p(const pp_batch* b, const pp_batch* db, void* stream, int total_inst, int grp);
static int prm_groups(const pp_batch* b, void* stream);
static int prm_steps_graph(const pp_batch* b, void* stream);

// The wavefront is a chain of ~2V dependent launches whose last wave is
// partly empty.  Instance groups run their chains on separate streams so one
// group's tail overlaps another group's kernels (fork/join with events on the
// caller's stream; the side streams are created once per host thread+device).
static constexpr int PP_DP_STREAMS = 8;
// instance groups (side streams) of the per-step schedule; PP_DP_GROUPS env overrides
static int read_dp_groups() {
    const char* e = getenv("PP_DP_GROUPS");
    const int v = e ? atoi(e) : 6;   // C3 n = 12 DP: 2.64 ms at 4 groups, 2.59 at 6, 2.61 at 8
    return v < 1 ? 1 : (v > PP_DP_STREAMS ? PP_DP_STREAMS : v);
}
static const int g_dp_groups = read_dp_groups();
struct SideStreams {
    int dev = -1;
    cudaStream_t s[PP_DP_STREAMS];
    cudaStream_t capture;   // origin stream of graph captures (the caller's may be the legacy stream)
    cudaEvent_t fork, join[PP_DP_STREAMS];
    // split chain (prm_chain_split_p): per group 3 bulk streams + its events
    cudaStream_t x[3 * PP_DP_STREAMS];
    cudaEvent_t xfork[PP_DP_STREAMS], c1[PP_DP_STREAMS][2], cb[PP_DP_STREAMS][3];
    cudaStream_t aux;              // pp_spp: phi beside RDO + DP
    cudaEvent_t aux_fork, aux_done;
};
static thread_local SideStreams g_side;

// Shared-memory-path DP schedule (same bits either way):
//   0 = the launch-per-step wavefront (prm_chain_p / the split critical-path
//       chain), replayed as a CUDA graph;
//   3 = one CTA per instance (dp_inst2.cu, dp_inst.cu): the whole wavefront of
//       an instance in one CTA, for batches with many more instances than SMs;
//   2 = auto (default): instance-per-CTA for >= 2 x SMs small instances
//       (L * V <= PP_DP_INST_MAX_LV), else per-step.
// (Round 1's persistent dependency-driven kernel and cluster-per-instance
// schedules were never chosen by auto — the graph-replayed per-step chain beat
// them at every batch size — and were removed in round 2.)
static constexpr int64_t PP_DP_INST_MAX_LV = 2048;
static std::atomic<int> g_dp_persist{2};

int pp_dp_set_persistent(int32_t mode) {
    if (mode != 0 && mode != 2 && mode != 3) return fail(PP_EINVAL, "DP schedule %d: 0 (per step), 2 (auto) or 3", mode);
    return g_dp_persist.exchange(mode);
}

static int prm_prep(const pp_batch* b, void* stream, bool tables = true);
// instance-per-CTA DP kernel: 2 = k_dp_inst2 (operands built in shared memory)
// when its footprint fits, 1 = k_dp_inst (table-staged); PP_DP_INST env
static const int g_dp_inst_kind = getenv("PP_DP_INST") ? atoi(getenv("PP_DP_INST")) : 2;

static int prm_inst(const pp_batch* b, void* stream) {
    const int maxL = b->max_L, maxV = b->max_V;
    int rc;
    // k_dp_inst2: one CTA per instance with every operand built in shared memory
    // (<= 113 KB: two CTAs per SM); the triangle tables are then never built
    const size_t smem2 = sizeof(double) * (size_t)dp_inst2_smem_doubles(maxL, maxV);
    if (g_dp_inst_kind == 2 && maxV > 1 && smem2 <= 113 * 1024) {
        if ((rc = prm_prep(b, stream, false))) return rc;
        cudaFuncSetAttribute(k_dp_inst2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
        k_dp_inst2<<<b->n_inst, DI2_T, smem2, S(stream)>>>(*b);
        PP_CHECK_LAUNCH("k_dp_inst2");
        // (the backtrack as the tail of k_dp_inst2, one warp per xi while its tables are
        // hot in L2, measured slower: C4 DP 4.91 -> 5.09 ms — it holds the CTA's 88 KB)
        dim3 gb(b->n_inst, maxV);
        k_backtrack<<<gb, 32, 0, S(stream)>>>(*b);
        PP_CHECK_LAUNCH("k_backtrack");
        return PP_OK;
    }
    if ((rc = prm_prep(b, stream))) return rc;
    if (maxV > 1) {
        // smallest chunk: one expand row at j = V-1 or one combine item at j = V-1
        const int need = std::max((maxV - 1) * maxV, (maxL - 1) * maxL / 2 + std::max(maxL - 1, 0) * (maxV - 1));
        // enough for a whole step's rows / items when that is small (C4: ~8 K doubles,
        // 3 CTAs per SM), else ~12 K doubles with chunking
        int full = 0;
        for (int j = 1; j < maxV; ++j)
            full = std::max(full, std::max((maxL - 1) * j * maxV,
                                           (maxV - j) * ((maxL - 1) * maxL / 2 + (maxL - 1) * j)));
        const int sd = std::min(27000, std::max(need, std::min(full, 12000)));
        if (need > 27000) return fail(PP_EINVAL, "k_dp_inst: L=%d V=%d exceed shared memory", maxL, maxV);
        const size_t smem = sizeof(double) * (size_t)sd;
        cudaFuncSetAttribute(k_dp_inst, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_dp_inst<<<b->n_inst, DI_T, smem, S(stream)>>>(*b, sd);
        PP_CHECK_LAUNCH("k_dp_inst");
    }
    dim3 gb(b->n_inst, maxV);
    k_backtrack<<<gb, 32, 0, S(stream)>>>(*b);
    PP_CHECK_LAUNCH("k_backtrack");
    return PP_OK;
}

int pp_dp_set_combine(int32_t kind) { return g_combine_kind.exchange(kind < 0 || kind > 2 ? 2 : kind); }

int pp_dp_set_early_exit(int32_t on) {
    int prev = 1, v = on ? 1 : 0;
    if (cudaMemcpyFromSymbol(&prev, g_combine_early_exit, sizeof(int)) != cudaSuccess ||
        cudaMemcpyToSymbol(g_combine_early_exit, &v, sizeof(int)) != cudaSuccess)
        return fail(PP_ECUDA, "pp_dp_set_early_exit: %s", cudaGetErrorString(cudaGetLastError()));
    return prev;
}

// Debug: per-CTA timeline of the per-step expand / combine kernels (4 x u64 per
// CTA, cap records); NULL disables.  Resets the record counter.
int pp_step_trace(uint64_t* d_buf, int32_t cap) {
    unsigned long long* p = reinterpret_cast<unsigned long long*>(d_buf);
    const int zero = 0;
    if (cudaMemcpyToSymbol(g_step_trace, &p, sizeof(p)) != cudaSuccess ||
        cudaMemcpyToSymbol(g_step_trace_cap, &cap, sizeof(cap)) != cudaSuccess ||
        cudaMemcpyToSymbol(g_step_trace_n, &zero, sizeof(zero)) != cudaSuccess)
        return fail(PP_ECUDA, "pp_step_trace: %s", cudaGetErrorString(cudaGetLastError()));
    return PP_OK;
}

// Debug: per-task timeline of the persistent DP into a caller device buffer of
// 4 * cap u64 (NULL / 0 disables).  Not part of the planning path.



int pp_prm(const pp_batch* b, void* stream) {
    if (b->n_inst <= 0) return PP_OK;
    if (int rc = check_ws(b, stream)) return rc;
    const int mode = g_dp_persist.load();
    if (b->max_L <= SR_MAX && b->max_V <= SR_MAX) {
        // many SMALL instances: one CTA each; otherwise the graph-replayed per-step schedule
        // (it beats the persistent kernel at every batch size once launches are free)
        const bool small = (int64_t)b->max_L * b->max_V <= PP_DP_INST_MAX_LV;
        if (mode == 3 || (mode == 2 && small && b->n_inst >= 2 * num_sms())) return prm_inst(b, stream);
    }
    if (!(b->max_L <= SR_MAX && b->max_V <= SR_MAX)) return prm_groups(b, stream);
    return prm_steps_graph(b, stream);
}

// descriptor slot k of the reserved workspace head (256-byte slots)
static inline const pp_batch* desc_slot(const pp_batch* base, int k) {
    return reinterpret_cast<const pp_batch*>(reinterpret_cast<const char*>(base) + 256 * k);
}

static int ensure_side_streams() {
    int dev = 0;
    cudaGetDevice(&dev);
    if (g_side.dev == dev) return PP_OK;
    for (int g = 0; g < PP_DP_STREAMS; ++g) {
        if (cudaStreamCreateWithFlags(&g_side.s[g], cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&g_side.join[g], cudaEventDisableTiming) != cudaSuccess)
            return fail(PP_ECUDA, "side stream creation: %s", cudaGetErrorString(cudaGetLastError()));
    }
    for (int g = 0; g < PP_DP_STREAMS; ++g) {
        bool ok = cudaEventCreateWithFlags(&g_side.xfork[g], cudaEventDisableTiming) == cudaSuccess;
        for (int k = 0; k < 3; ++k)
            ok = ok && cudaStreamCreateWithFlags(&g_side.x[3 * g + k], cudaStreamNonBlocking) == cudaSuccess &&
                 cudaEventCreateWithFlags(&g_side.cb[g][k], cudaEventDisableTiming) == cudaSuccess;
        for (int k = 0; k < 2; ++k) ok = ok && cudaEventCreateWithFlags(&g_side.c1[g][k], cudaEventDisableTiming) == cudaSuccess;
        if (!ok) return fail(PP_ECUDA, "side stream creation: %s", cudaGetErrorString(cudaGetLastError()));
    }
    if (cudaEventCreateWithFlags(&g_side.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaStreamCreateWithFlags(&g_side.capture, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&g_side.aux, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&g_side.aux_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&g_side.aux_done, cudaEventDisableTiming) != cudaSuccess)
        return fail(PP_ECUDA, "event creation: %s", cudaGetErrorString(cudaGetLastError()));
    if (const char* e = getenv("PP_BULK")) {   // A/B knob: 0 stages the combine with per-element cp.async
        const int v = atoi(e);
        cudaMemcpyToSymbol(g_combine_bulk, &v, sizeof(v));
    }
    g_side.dev = dev;
    return PP_OK;
}

// Instance groups on side streams (fork/join on the caller's stream).  `dev`:
// device descriptors of the groups (per-step shared-memory path) or NULL.
static int prm_groups_impl(const pp_batch* b, void* stream, const pp_batch* dev) {
    const int G = b->n_inst < g_dp_groups ? b->n_inst : g_dp_groups;
    if (G <= 1)
        return dev ? (b->n_inst <= g_dp_split ? prm_chain_split_p(b, desc_slot(dev, 1), stream, b->n_inst, 0)
                                 : prm_chain_p(b, desc_slot(dev, 1), stream, b->n_inst))
                   : prm_chain(b, stream, b->n_inst);
    int rc;
    if ((rc = ensure_side_streams())) return rc;
    cudaEventRecord(g_side.fork, S(stream));
    for (int g = 0; g < G; ++g) {
        const int lo = (int)((int64_t)g * b->n_inst / G), hi = (int)((int64_t)(g + 1) * b->n_inst / G);
        pp_batch bg = *b;
        bg.inst = b->inst + lo;
        bg.n_inst = hi - lo;
        cudaStreamWaitEvent(g_side.s[g], g_side.fork, 0);
        rc = dev ? (b->n_inst <= g_dp_split ? prm_chain_split_p(&bg, desc_slot(dev, 1 + g), g_side.s[g], b->n_inst, g)
                               : prm_chain_p(&bg, desc_slot(dev, 1 + g), g_side.s[g], b->n_inst))
                 : prm_chain(&bg, g_side.s[g], b->n_inst);
        if (rc) return rc;
        cudaEventRecord(g_side.join[g], g_side.s[g]);
        cudaStreamWaitEvent(S(stream), g_side.join[g], 0);
    }
    return PP_OK;
}
static int prm_groups(const pp_batch* b, void* stream) { return prm_groups_impl(b, stream, nullptr); }

// The per-step schedule is ~2V dependent launches per instance group: launched
// one by one the host's launch rate is the bound (~3.5 us per launch, measured:
// the empty-kernel chain alone took 1.8 ms on C3).  It is captured once per batch
// SHAPE into a CUDA graph and replayed; its kernels read their batch descriptor
// from a small library-owned device buffer of the cache entry (rewritten, stream
// ordered, before every replay), so any workspace / buffers of that shape replay.
struct GraphKey {   // what the captured launches bake in: grid shapes (descriptors live in the entry)
    int n_inst, max_L, max_V, G, dev, combine;
    bool operator==(const GraphKey& o) const {
        return n_inst == o.n_inst && max_L == o.max_L && max_V == o.max_V && G == o.G && dev == o.dev &&
               combine == o.combine;
    }
};
struct GraphEntry {
    GraphKey key;
    cudaGraphExec_t exec;
    pp_batch* d_desc;   // library-owned descriptor slots the graph's kernels read (256 B each)
    cudaEvent_t done;   // last replay of this graph (the next one may rewrite the slots after it)
};
static thread_local std::vector<GraphEntry> g_graphs;
static constexpr size_t PP_GRAPH_CACHE = 8;
static_assert(sizeof(pp_batch) <= 256, "descriptor slot");

static int prm_steps_graph(const pp_batch* b, void* stream) {
    const int G = b->n_inst < g_dp_groups ? b->n_inst : g_dp_groups;
    // descriptors: slot 1 + g = group g (slot 1 = the whole batch when G == 1)
    pp_batch hd[1 + PP_DP_STREAMS];
    hd[0] = *b;
    const int ng = G <= 1 ? 1 : G;
    for (int g = 0; g < ng; ++g) {
        const int lo = (int)((int64_t)g * b->n_inst / ng), hi = (int)((int64_t)(g + 1) * b->n_inst / ng);
        hd[1 + g] = *b;
        hd[1 + g].inst = b->inst + lo;
        hd[1 + g].n_inst = hi - lo;
    }
    int d = 0;
    cudaGetDevice(&d);
    const GraphKey key{b->n_inst, b->max_L, b->max_V, G, d, g_combine_kind.load()};
    GraphEntry* ent = nullptr;
    for (size_t k = 0; k < g_graphs.size(); ++k)
        if (g_graphs[k].key == key) { ent = &g_graphs[k]; break; }
    if (!ent) {
        int rc;
        if ((rc = ensure_side_streams())) return rc;
        if (g_graphs.size() >= PP_GRAPH_CACHE) {   // cudaFree waits for the evicted graph's last replay
            GraphEntry& o = g_graphs.front();
            cudaGraphExecDestroy(o.exec);
            cudaFree(o.d_desc);
            cudaEventDestroy(o.done);
            g_graphs.erase(g_graphs.begin());
        }
        GraphEntry e{key, nullptr, nullptr, nullptr};
        if (cudaMalloc(&e.d_desc, 256 * (1 + PP_DP_STREAMS)) != cudaSuccess ||
            cudaEventCreateWithFlags(&e.done, cudaEventDisableTiming) != cudaSuccess)
            return fail(PP_ECUDA, "graph descriptors: %s", cudaGetErrorString(cudaGetLastError()));
        cudaGraph_t graph;
        cudaStream_t cs = g_side.capture;   // the caller's stream may be the (uncapturable) legacy stream
        if (cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
            return fail(PP_ECUDA, "graph capture: %s", cudaGetErrorString(cudaGetLastError()));
        rc = prm_groups_impl(b, cs, e.d_desc);
        const cudaError_t ce = cudaStreamEndCapture(cs, &graph);
        if (rc) return rc;
        if (ce != cudaSuccess) return fail(PP_ECUDA, "graph capture: %s", cudaGetErrorString(ce));
        const cudaError_t ie = cudaGraphInstantiate(&e.exec, graph, 0);
        cudaGraphDestroy(graph);
        if (ie != cudaSuccess) return fail(PP_ECUDA, "graph instantiate: %s", cudaGetErrorString(ie));
        g_graphs.push_back(e);
        ent = &g_graphs.back();
    } else {
        cudaStreamWaitEvent(S(stream), ent->done, 0);   // a replay on another stream may still read the slots
    }
    for (int g = 0; g <= ng; ++g)   // pageable source: staged by the driver, safe to reuse at once
        if (cudaMemcpyAsync(reinterpret_cast<char*>(ent->d_desc) + 256 * g, &hd[g], sizeof(pp_batch),
                            cudaMemcpyHostToDevice, S(stream)) != cudaSuccess)
            return fail(PP_ECUDA, "descriptor upload: %s", cudaGetErrorString(cudaGetLastError()));
    if (cudaGraphLaunch(ent->exec, S(stream)) != cudaSuccess)
        return fail(PP_ECUDA, "graph launch: %s", cudaGetErrorString(cudaGetLastError()));
    cudaEventRecord(ent->done, S(stream));
    g_launches.fetch_add(1 + 2 * (int64_t)ng * (b->max_V - 1) + 5 * ng, std::memory_order_relaxed);
    return PP_OK;
}

// Tables every DP schedule needs: prep, base rows, and (shared-memory path)
// the deduplicated stage-term triangles.
static int prm_prep(const pp_batch* b, void* stream, bool tables) {
    const int maxL = b->max_L, maxV = b->max_V;
    dim3 gp(b->n_inst, maxL > maxV ? maxL : maxV);
    // small instances (C4: L 32, V 16) leave most of a 128-thread row CTA idle and
    // the rows are latency-bound: 32-thread CTAs fit twice as many rows per SM
    const int pt = (maxL <= 32 && maxV <= 32) ? 32 : 128;
    k_prep<<<gp, pt, maxV <= PREP_CM_MAX ? sizeof(double) * maxV * maxV : 0, S(stream)>>>(*b);
    PP_CHECK_LAUNCH("k_prep");
    dim3 gbase(b->n_inst, maxL > maxV ? maxL : maxV);
    k_base<<<gbase, pt, 0, S(stream)>>>(*b, !(maxL <= SR_MAX && maxV <= SR_MAX));
    PP_CHECK_LAUNCH("k_base");
    if (tables && maxL <= SR_MAX && maxV <= SR_MAX) {
        k_sdedup<<<dim3(b->n_inst, (maxV - 1 + 7) / 8 > 0 ? (maxV - 1 + 7) / 8 : 1), 256, 0, S(stream)>>>(*b);
        PP_CHECK_LAUNCH("k_sdedup");
        if (maxV > 1 && maxL > 1) {
            dim3 gs(b->n_inst, maxV - 1);
            if ((maxL - 1) * maxL / 2 >= STAB_BIG) k_stab_big<<<gs, 128, 0, S(stream)>>>(*b);
            else k_stab<<<gs, 128, 0, S(stream)>>>(*b);
            PP_CHECK_LAUNCH("k_stab");
        }
    }
    return PP_OK;
}

// prm_chain for the shared-memory path with device descriptors (graph capture):
// `b` supplies the host-side shape, `db` is the same batch in device memory.
static int prm_tables_p(const pp_batch* b, const pp_batch* db, void* stream) {
    const int maxL = b->max_L, maxV = b->max_V;
    dim3 gp(b->n_inst, maxL > maxV ? maxL : maxV);
    k_prep_p<<<gp, 128, maxV <= PREP_CM_MAX ? sizeof(double) * maxV * maxV : 0, S(stream)>>>(db);
    PP_CHECK_LAUNCH("k_prep");
    k_base_p<<<gp, 128, 0, S(stream)>>>(db, 0);
    PP_CHECK_LAUNCH("k_base");
    k_sdedup_p<<<dim3(b->n_inst, (maxV - 1 + 7) / 8 > 0 ? (maxV - 1 + 7) / 8 : 1), 256, 0, S(stream)>>>(db);
    PP_CHECK_LAUNCH("k_sdedup");
    if (maxV > 1 && maxL > 1) {
        dim3 gs(b->n_inst, maxV - 1);
        if ((maxL - 1) * maxL / 2 >= STAB_BIG) k_stab_big_p<<<gs, 128, 0, S(stream)>>>(db);
        else k_stab_p<<<gs, 128, 0, S(stream)>>>(db);
        PP_CHECK_LAUNCH("k_stab");
    }
    const size_t ex_smem = sizeof(double) * (size_t)maxV * maxV;
    const size_t cs_smem = sizeof(double) * ((maxL + 1) / 2 + 3 + (size_t)(maxL - 1) * maxL / 2 +
                                             (size_t)(maxL > 1 ? maxL - 1 : 0) * maxV);
    cudaFuncSetAttribute(k_expand_s_p, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ex_smem);
    cudaFuncSetAttribute(k_expand_m_p, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)std::max(ex_smem, sizeof(double) * (size_t)(EX_SMEM_DOUBLES + 2)));
    cudaFuncSetAttribute(k_combine_s_p, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cs_smem);
    cudaFuncSetAttribute(k_combine_bis_p, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(sizeof(double) * combine_bis_smem_doubles(maxL, maxV, maxL)));
    return PP_OK;
}

// one combine launch of the per-step schedule: items r0 .. r0 + nitems - 1 of step j
static int launch_combine(const pp_batch* b, const pp_batch* db, cudaStream_t st, cudaLaunchAttribute* attrs, int j,
                          int r0, int nitems, int parts, int total_inst) {
    const int maxL = b->max_L;
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cfg.attrs = attrs;
    cfg.numAttrs = 1;
    cudaError_t e;
    const int kind = g_combine_kind.load();
    if (kind == 1 || (kind == 2 && total_inst <= g_bis_max_inst)) {
        // row groups: split items until the launch has ~2 waves of CTAs (at most L/8 groups)
        const int64_t items = (int64_t)b->n_inst * nitems;
        int groups = (int)std::min<int64_t>((int64_t)std::ceil(g_bis_waves * num_sms() / (double)items), (maxL + 7) / 8);
        if (groups < 1) groups = 1;
        const int rg = (maxL + groups - 1) / groups;
        groups = (maxL + rg - 1) / rg;
        cfg.gridDim = dim3(b->n_inst, nitems, groups);
        cfg.dynamicSmemBytes = sizeof(double) * combine_bis_smem_doubles(maxL, j, rg);
        const int rb = g_bis_rb > 0 ? g_bis_rb : (groups > 1 ? 1 : 8);
        e = cudaLaunchKernelEx(&cfg, k_combine_bis_p, db, j, r0, rg, rb);
    } else {
        cfg.gridDim = dim3(b->n_inst, nitems, parts);
        cfg.dynamicSmemBytes = sizeof(double) * ((maxL + 1) / 2 + 3 + (size_t)(maxL - 1) * maxL / 2 +
                                                 (size_t)(maxL > 1 ? maxL - 1 : 0) * j);
        e = cudaLaunchKernelEx(&cfg, k_combine_s_p, db, j, r0);
    }
    if (e != cudaSuccess) return fail(PP_ECUDA, "combine launch: %s", cudaGetErrorString(cudaGetLastError()));
    PP_CHECK_LAUNCH("k_combine");
    return PP_OK;
}

// combine work units (tile parts) per item: split until a step has about
// g_combine_waves waves of CTAs
static int combine_parts(int items) {
    int parts = (g_combine_waves * num_sms() + items - 1) / items;
    return parts < 1 ? 1 : (parts > g_max_parts ? g_max_parts : parts);
}
static size_t combine_smem(int maxL, int j) {
    return sizeof(double) * ((maxL + 1) / 2 + 3 + (size_t)(maxL - 1) * maxL / 2 + (size_t)(maxL > 1 ? maxL - 1 : 0) * j);
}

// The wavefront with its critical path split off (small batches, PP_DP_SPLIT).  Slice W_{j+1} needs only the r = 1 item of step j (i = j + 1); the
// items r >= 2 of step j are first read r - 1 steps later.  So each step runs
//   s0 (critical): E1(j) = expand target r = 1, then C1(j) = combine item r = 1
//   x[j % 3] (bulk): Eb(j) = expand targets r >= 2, then Cb(j) = items r >= 2
// E1(j) and Eb(j) read all of W_j: they wait for C1(j-1) and Cb(j-2) (Cb(j-3)
// is behind its own stream's order, or waited for on s0; older ones are
// implied: Cb(m) waited for Cb(m-2) and follows Cb(m-3) on its stream).  The
// critical chain is two small launches per step; the bulk work of later steps
// overlaps it on three streams.
static int prm_chain_split_p(const pp_batch* b, const pp_batch* db, void* stream, int total_inst, int grp) {
    const int maxL = b->max_L, maxV = b->max_V;
    int rc;
    if ((rc = ensure_side_streams())) return rc;
    if ((rc = prm_tables_p(b, db, stream))) return rc;
    cudaLaunchAttribute pdl[1];
    pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
    cudaStream_t s0 = S(stream);
    cudaStream_t* sx = &g_side.x[3 * grp];
    cudaEvent_t* c1 = g_side.c1[grp];
    cudaEvent_t* cb = g_side.cb[grp];
    cudaEventRecord(g_side.xfork[grp], s0);
    for (int k = 0; k < 3; ++k) {
        cudaStreamWaitEvent(sx[k], g_side.xfork[grp], 0);
        cudaEventRecord(cb[k], sx[k]);
    }
    cudaEventRecord(c1[0], s0);
    cudaEventRecord(c1[1], s0);
    auto expand = [&](cudaStream_t st, int j, int rfirst, int rlast) -> int {
        if (maxL <= 1) return PP_OK;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(b->n_inst, maxL - 1);
        cfg.blockDim = dim3(rlast == 1 || (int64_t)total_inst * (maxL - 1) <= g_expand_wide * num_sms() ? 256 : 128);
        cfg.dynamicSmemBytes = sizeof(double) * (size_t)j * maxV;
        cfg.stream = st;
        cfg.attrs = pdl;
        cfg.numAttrs = 1;
        if (cudaLaunchKernelEx(&cfg, k_expand_s_p, db, j, rfirst, rlast) != cudaSuccess)
            return fail(PP_ECUDA, "k_expand_s launch: %s", cudaGetErrorString(cudaGetLastError()));
        PP_CHECK_LAUNCH("k_expand_s");
        return PP_OK;
    };
    auto combine = [&](cudaStream_t st, int j, int r0, int nitems, int parts) -> int {
        return launch_combine(b, db, st, pdl, j, r0, nitems, parts, total_inst);
    };
    for (int j = 1; j < maxV; ++j) {
        if (j >= 3) cudaStreamWaitEvent(s0, cb[(j - 2) % 3], 0);
        if (j >= 4) cudaStreamWaitEvent(s0, cb[(j - 3) % 3], 0);
        if ((rc = expand(s0, j, 1, 1))) return rc;
        if ((rc = combine(s0, j, 1, 1, g_c1_parts))) return rc;
        cudaEventRecord(c1[j % 2], s0);
        if (maxV - j >= 2) {
            cudaStream_t sk = sx[j % 3];
            cudaStreamWaitEvent(sk, c1[(j - 1) % 2], 0);
            if (j >= 3) cudaStreamWaitEvent(sk, cb[(j - 2) % 3], 0);
            if ((rc = expand(sk, j, 2, (int)SR_MAX))) return rc;
            if ((rc = combine(sk, j, 2, maxV - j - 1, combine_parts(total_inst * (maxV - j - 1))))) return rc;
            cudaEventRecord(cb[j % 3], sk);
        }
    }
    for (int k = 0; k < 3; ++k) cudaStreamWaitEvent(s0, cb[k], 0);
    dim3 gb(b->n_inst, maxV);
    k_backtrack_p<<<gb, 32, 0, s0>>>(db);
    PP_CHECK_LAUNCH("k_backtrack");
    return PP_OK;
}

static int prm_chain_p(const pp_batch* b, const pp_batch* db, void* stream, int total_inst) {
    const int maxL = b->max_L, maxV = b->max_V;
    int rc;
    if ((rc = prm_tables_p(b, db, stream))) return rc;
    // programmatic dependent launch between consecutive wavefront kernels: each
    // stages its producer-independent operands while its predecessor drains
    cudaLaunchAttribute pdl[1];
    pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
    for (int j = 1; j < maxV; ++j) {
        if (maxL > 1) {
            cudaLaunchConfig_t cfg = {};
            // a step with fewer rows than SMs runs one CTA per SM: twice the warps
            // per row (split-K over r') hides the issue latency of its (min, max) chain;
            // with many rows, rb rows per 256-thread CTA share their chan block
            const int64_t rows = (int64_t)total_inst * (maxL - 1);
            int rb = 1;
            if (rows > (int64_t)g_expand_rb_min * num_sms()) {
                rb = g_expand_rb;
                const int64_t cap = (EX_SMEM_DOUBLES - (int64_t)j * (maxV - j)) / ((int64_t)j * j);
                if (rb > cap) rb = cap < 1 ? 1 : (int)cap;
            }
            cfg.gridDim = dim3(b->n_inst, ceil_div(maxL - 1, rb));
            cfg.blockDim = dim3(rb > 1 || rows <= g_expand_wide * num_sms() ? 256 : 128);
            cfg.dynamicSmemBytes = sizeof(double) * (2 + std::max((size_t)j * maxV, (size_t)rb * j * j + (size_t)j * (maxV - j)));
            cfg.stream = S(stream);
            cfg.attrs = pdl;
            cfg.numAttrs = 1;
            if ((rb > 1 ? cudaLaunchKernelEx(&cfg, k_expand_m_p, db, j, rb) : cudaLaunchKernelEx(&cfg, k_expand_s_p, db, j, 1, (int)SR_MAX)) !=
                cudaSuccess)
                return fail(PP_ECUDA, "k_expand_s launch: %s", cudaGetErrorString(cudaGetLastError()));
            PP_CHECK_LAUNCH("k_expand_s");
        }
        if ((rc = launch_combine(b, db, S(stream), pdl, j, 1, maxV - j, combine_parts(total_inst * (maxV - j)),
                                 total_inst)))
            return rc;
    }
    dim3 gb(b->n_inst, maxV);
    k_backtrack_p<<<gb, 32, 0, S(stream)>>>(db);
    PP_CHECK_LAUNCH("k_backtrack");
    return PP_OK;
}

static int prm_chain(const pp_batch* b, void* stream, int total_inst) {
    const int maxL = b->max_L, maxV = b->max_V;
    int rc;
    if ((rc = prm_prep(b, stream))) return rc;
    // wavefront: step j = expand(j) (X for every target (r, j+r) + their stage
    // terms) then combine_diag(j) (W for every target (r, j+r)); afterwards
    // slice j+1 is complete.
    if (maxL <= SR_MAX && maxV <= SR_MAX) {
        // shared-memory-resident path: one barrier per work item
        const size_t ex_smem = sizeof(double) * (size_t)maxV * maxV;
        const size_t cs_smem = sizeof(double) * ((maxL + 1) / 2 + 1 + (size_t)(maxL - 1) * maxL / 2 +
                                                 (size_t)(maxL > 1 ? maxL - 1 : 0) * maxV);
        cudaFuncSetAttribute(k_expand_s, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ex_smem);
        cudaFuncSetAttribute(k_combine_s, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cs_smem);
        for (int j = 1; j < maxV; ++j) {
            if (maxL > 1) {
                dim3 ge(b->n_inst, maxL - 1);
                k_expand_s<<<ge, 128, sizeof(double) * (size_t)j * maxV, S(stream)>>>(*b, j);
                PP_CHECK_LAUNCH("k_expand_s");
            }
            // split every item over `parts` CTAs so a launch fills ~2 waves of the SMs
            // (counted over the whole batch: the groups' launches run concurrently)
            const int items = total_inst * (maxV - j);
            int parts = (g_combine_waves * num_sms() + items - 1) / items;
            parts = parts < 1 ? 1 : (parts > g_max_parts ? g_max_parts : parts);
            dim3 gc(b->n_inst, maxV - j, parts);
            const size_t sm = sizeof(double) * ((maxL + 1) / 2 + 1 + (size_t)(maxL - 1) * maxL / 2 +
                                                (size_t)(maxL > 1 ? maxL - 1 : 0) * j);
            k_combine_s<<<gc, 256, sm, S(stream)>>>(*b, j);
            PP_CHECK_LAUNCH("k_combine_s");
        }
        dim3 gb(b->n_inst, maxV);
        k_backtrack<<<gb, 32, 0, S(stream)>>>(*b);
        PP_CHECK_LAUNCH("k_backtrack");
        return PP_OK;
    }
    const int rows_l = ceil_div(maxL, CD_L), planes_cx = ceil_div(maxV, CD_X);
    cudaFuncSetAttribute(k_combine_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CD_SMEM);
    for (int j = 1; j < maxV; ++j) {
        const int planes_xi = ceil_div(j, EX_P), planes_r = ceil_div(maxV - j, EX_P);
        dim3 ge(b->n_inst, (maxL - 1) + (maxV - j), planes_xi * planes_r);
        k_expand<<<ge, EX_T, 0, S(stream)>>>(*b, j, planes_r, maxL - 1);
        PP_CHECK_LAUNCH("k_expand");
        dim3 gc(b->n_inst, maxV - j, rows_l * planes_cx);
        k_combine_diag<<<gc, CD_T, CD_SMEM, S(stream)>>>(*b, j, planes_cx);
        PP_CHECK_LAUNCH("k_combine_diag");
    }
    dim3 gb(b->n_inst, maxV);
    k_backtrack<<<gb, 32, 0, S(stream)>>>(*b);
    PP_CHECK_LAUNCH("k_backtrack");
    return PP_OK;
}

static size_t sim_smem(int maxN) {
    const int R = 2 * maxN - 1;
    return sizeof(double) * (4 * R + 64);
}

static int sim_block(int maxN) {
    const int R = 2 * maxN - 1;
    int t = (R + 31) / 32 * 32;
    return t < 32 ? 32 : t;
}

int pp_pe_sweep(const pp_batch* b, void* stream) {
    if (b->n_inst <= 0) return PP_OK;
    if (!b->ws) return fail(PP_EINVAL, "pp_pe_sweep: pp_batch.ws is NULL (the sweep reads the DP's slice tables)");
    dim3 g(b->n_inst, b->max_V);
    if (b->max_V <= PE_WARP_MAXN) {   // one warp per plan: registers + shuffles per pass
        k_pe_sweep_w<<<g, 32, 0, S(stream)>>>(*b);
        PP_CHECK_LAUNCH("k_pe_sweep");
        return PP_OK;
    }
    k_pe_sweep<<<g, 32 * pe_mw_warps(b->max_V), sizeof(double) * 6 * 32, S(stream)>>>(*b);
    PP_CHECK_LAUNCH("k_pe_sweep");
    return PP_OK;
}

int pp_select(const pp_batch* b, void* stream) {
    if (b->n_inst <= 0) return PP_OK;
    if (b->ev_start && !b->ws) return fail(PP_EINVAL, "pp_select: pp_batch.ws is NULL (the replay reads the DP's slice tables)");
    k_select<<<b->n_inst, 32, 0, S(stream)>>>(*b);
    PP_CHECK_LAUNCH("k_select");
    if (b->ev_start) {
        if (b->max_V <= PE_WARP_MAXN) {
            k_replay_w<<<b->n_inst, 32, 0, S(stream)>>>(*b);
        } else {
            k_replay<<<b->n_inst, 32 * pe_mw_warps(b->max_V), sizeof(double) * 6 * 32, S(stream)>>>(*b);
        }
        PP_CHECK_LAUNCH("k_replay");
        if (b->ev_order) {
            // events per plan <= max_M (4 max_V - 3): shared memory and block sized to
            // it (small plans: several CTAs per SM); max_M = 0 (unknown) sizes for EM_MAXN
            const int64_t nmax = b->max_M > 0 ? (int64_t)b->max_M * (4 * b->max_V - 3) : (int64_t)EM_MAXN + 1;
            const int64_t nm = std::min<int64_t>(nmax, EM_MAXN);
            const size_t smem = (size_t)(12 * nm + 16 + 15) & ~(size_t)15;
            const int thr = nm <= 2048 ? 256 : (nm <= 8192 ? 512 : EM_T);
            cudaFuncSetAttribute(k_event_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, EM_SMEM + 32);
            k_event_merge<<<b->n_inst, thr, smem, S(stream)>>>(*b);
            PP_CHECK_LAUNCH("k_event_merge");
            if (nmax > EM_MAXN) {
                k_event_rank<<<dim3(b->n_inst, 16), 256, 0, S(stream)>>>(*b);
                PP_CHECK_LAUNCH("k_event_rank");
            }
        }
    }
    return PP_OK;
}

int pp_phi(const pp_batch* b, void* stream) {
    if (b->n_inst <= 0) return PP_OK;
    k_phi<<<b->n_inst, 128, 0, S(stream)>>>(*b);
    PP_CHECK_LAUNCH("k_phi");
    return PP_OK;
}

int pp_spp(const pp_batch* b, void* stream) {
    int rc;
    if ((rc = ensure_side_streams())) return rc;
    // phi (cost.py:131-142) depends on the inputs only: it runs on a side stream
    // beside RDO and the DP (only the host reads it), joined before the sweep
    cudaEventRecord(g_side.aux_fork, S(stream));
    cudaStreamWaitEvent(g_side.aux, g_side.aux_fork, 0);
    if ((rc = pp_phi(b, g_side.aux))) return rc;
    cudaEventRecord(g_side.aux_done, g_side.aux);
    if ((rc = pp_rdo(b, stream))) return rc;
    if ((rc = pp_prm(b, stream))) return rc;
    cudaStreamWaitEvent(S(stream), g_side.aux_done, 0);
    if ((rc = pp_pe_sweep(b, stream))) return rc;
    return pp_select(b, stream);
}

int pp_prm_query(const pp_batch* b, int32_t n_query, const int32_t* q_inst, const int32_t* q_l,
                 const int32_t* q_xi, const int32_t* q_r, const int32_t* q_i, int32_t max_xi, double* w,
                 int32_t* frag, int32_t* feasible, void* stream) {
    if (n_query <= 0) return PP_OK;
    if (!b->ws) return fail(PP_EINVAL, "pp_prm_query: pp_batch.ws is NULL (queries read the DP slices)");
    k_query<<<n_query, 32, 0, S(stream)>>>(*b, n_query, q_inst, q_l, q_xi, q_r, q_i, max_xi, w, frag, feasible);
    PP_CHECK_LAUNCH("k_query");
    return PP_OK;
}

int pp_simulate(const pp_batch* ib, const pp_sim_batch* s, void* stream) {
    if (s->n_plan <= 0) return PP_OK;
    if (s->max_N < 1 || s->max_N > PP_MAX_GPUS) return fail(PP_EINVAL, "max_N=%d outside 1..%d", s->max_N, PP_MAX_GPUS);
    const size_t smem = std::max(sim_smem(s->max_N), sizeof(double) * 128);   // + plan_costs / cycle scratch
    cudaFuncSetAttribute(k_sim_plans, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_sim_plans<<<s->n_plan, sim_block(s->max_N), smem, S(stream)>>>(*ib, *s);
    PP_CHECK_LAUNCH("k_sim_plans");
    return PP_OK;
}

int pp_peak_minmax(double* d_out, int32_t iters, int64_t* n_ops, void* stream) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int blocks = sms * 8, threads = 256;
    k_peak_minmax<<<blocks, threads, 0, S(stream)>>>(d_out, iters, 0.5);
    PP_CHECK_LAUNCH("k_peak_minmax");
    *n_ops = (int64_t)blocks * threads * iters * 16;
    return PP_OK;
}

int pp_min_cut(const pp_batch* b, int32_t k, const int32_t* verts, int32_t n, uint8_t* in_a, double* weight,
               void* stream) {
    if (n < 2) return fail(PP_EINVAL, "min cut needs at least 2 vertices");
    const int V = b->max_V;
    const int in_smem = V <= RDO_SMEM_MAX;
    if (!in_smem && !b->ws) return fail(PP_EINVAL, "pp_min_cut: V=%d > %d needs pp_batch.ws", V, RDO_SMEM_MAX);
    const size_t smem = (in_smem ? sizeof(double) * V * V : 0) + rdo_state_bytes(V);
    if (in_smem) {
        cudaFuncSetAttribute(k_min_cut<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_min_cut<true><<<1, 32, smem, S(stream)>>>(*b, k, verts, n, in_a, weight);
    } else {
        cudaFuncSetAttribute(k_min_cut<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_min_cut<false><<<1, 32, smem, S(stream)>>>(*b, k, verts, n, in_a, weight);
    }
    PP_CHECK_LAUNCH("k_min_cut");
    return PP_OK;
}

}  // extern "C"

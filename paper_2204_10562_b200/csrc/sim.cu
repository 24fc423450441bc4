// sim.cu — microbatch scheduler + makespan simulator (scheduler.py:49-238,
// cost.py:162-230), one plan per CTA, one thread per resource.
//
// PE order (scheduler.py:75-106) in closed form: in pass p the block at
// position pos serves microbatch m = p - pos + 1 (1 <= m <= M), positions
// visited in descending order, so each resource serves its backward-side item
// before its forward-side item within a pass.  The heap event loop
// (scheduler.py:121-225) then reduces to the max-plus recurrence
//     start = max(end of the previous item on the resource, end of (m, pos-1))
// and every predecessor (m, pos-1) sits on an ADJACENT resource of the chain
// stage1, chan1, stage2, ..., stageN and completed in pass p-1.  So a pass is
// one step in which each resource lane reads its two neighbours' pass p-1
// completion times from double-buffered shared memory and runs <= 2 items:
//   stage n < N : B_n (pred Y_n, right)   then F_n (pred X_{n-1}, left)
//   stage N     : FB_N (pred X_{N-1}, left)
//   chan n      : Y_n (pred B_{n+1}/FB_N, right) then X_n (pred F_n, left)
// Caller-supplied queues (simulate_with_order) run through k_sim_queues, a
// round-based Kahn sweep that handles arbitrary orders, the forward barrier
// and stall detection.
#include "common.cuh"

namespace pp {

// ---- plan views -------------------------------------------------------------
struct SppPlanView {   // xi-stage plan written by k_backtrack: device ranks are order slices
    const int *ls, *le, *dlo, *dhi, *order;
    const double *minpair = nullptr, *cross = nullptr;   // k_prep's slice tables (optional)
    int V = 0;
    __device__ int stage_ls(int n) const { return ls[n - 1]; }
    __device__ int stage_le(int n) const { return le[n - 1]; }
    __device__ int k(int n) const { return dhi[n - 1] - dlo[n - 1] + 1; }
    __device__ int dev(int n, int a) const { return order[dlo[n - 1] - 1 + a]; }
    // min pairwise bandwidth of stage n's slice / min cross bandwidth between the
    // slices of stages n and n+1 (cost.py:64-80): the exact minima k_prep tabulated
    // over the same device sets (min is order-free, so the bits are the loop's);
    // returns false when the tables are absent
    __device__ bool table_min_pair(int n, double& mp) const {
        if (!minpair) return false;
        mp = minpair[(int64_t)(dlo[n - 1] - 1) * V + (dhi[n - 1] - 1)];
        return true;
    }
    __device__ bool table_min_cross(int n, double& mc) const {
        if (!cross) return false;
        mc = cross[cross_idx(V, dhi[n], dhi[n] - dlo[n] + 1, dhi[n - 1] - dlo[n - 1] + 1)];
        return true;
    }
};

struct ExplicitPlanView {   // caller plan (pp_sim_batch)
    const int *ls, *le, *doff, *devs;
    __device__ int stage_ls(int n) const { return ls[n - 1]; }
    __device__ int stage_le(int n) const { return le[n - 1]; }
    __device__ int k(int n) const { return doff[n] - doff[n - 1]; }
    __device__ int dev(int n, int a) const { return devs[doff[n - 1] + a]; }
    __device__ bool table_min_pair(int, double&) const { return false; }   // arbitrary device sets
    __device__ bool table_min_cross(int, double&) const { return false; }
};

struct InstView {
    int V;
    bool naive;
    const double *fwd, *bwd, *par, *efwd, *ebwd, *bw;
    __device__ InstView(const pp_batch& b, const pp_instance& I)
        : V(I.V), naive(I.flags & PP_SUM_NAIVE), fwd(b.fwd + I.layer_off), bwd(b.bwd + I.layer_off),
          par(b.param + I.layer_off), efwd(b.efwd + I.layer_off), ebwd(b.ebwd + I.layer_off), bw(b.bw + I.bw_off) {}
    __device__ double w(int a, int c) const { return bw[(int64_t)a * V + c]; }
};

__device__ __forceinline__ void bar_sync(int nthr) { asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory"); }

// Per-lane costs: durations (cost.py:205-224), cycle-time term and AllReduce
// (cost.py:83-99, 172-202).  lane = resource index in chain order.
struct LaneCost {
    double dA, dB;      // stage: F (or FB for the last stage) / B ; chan: X / Y
    double cyc;         // per-stage compute or per-channel comm (cost_summary)
    double ar;          // AllReduce time (replicated stages)
    bool has_ar;
    double fs, bs;      // split F / B durations (stage_*_time / k, cost.py:215-218) of ANY stage; 0 on channels
    double mbw;         // min pairwise (stage) / min cross (chan) bandwidth (cost.py:64-80)
};

template <class P>
__device__ LaneCost lane_cost(const P& p, const InstView& I, int N, int lane) {
    LaneCost c{0.0, 0.0, 0.0, 0.0, false, 0.0, 0.0, PP_INF};
    const int n = lane / 2 + 1;
    if ((lane & 1) == 0) {
        const int k = p.k(n), a = p.stage_ls(n), e = p.stage_le(n);
        const double sf = pysum(I.fwd + a - 1, e - a + 1, I.naive) / (double)k;   // cost.py:47
        const double sb = pysum(I.bwd + a - 1, e - a + 1, I.naive) / (double)k;   // cost.py:53
        if (n < N) { c.dA = sf / (double)k; c.dB = sb / (double)k; }             // cost.py:215-218
        else { c.dA = (sf + sb) / (double)k; c.dB = c.dA; }                      // cost.py:219-220
        c.cyc = sf + sb;                                                          // cost.py:56-61
        c.fs = sf / (double)k;
        c.bs = sb / (double)k;
        if (k >= 2) {
            const double total = pysum(I.par + a - 1, e - a + 1, I.naive);
            double mp = PP_INF;
            if (!p.table_min_pair(n, mp))
                for (int x = 0; x < k; ++x)
                    for (int y = x + 1; y < k; ++y) mp = dmin(mp, I.w(p.dev(n, x), p.dev(n, y)));
            c.ar = 2.0 * (double)(k - 1) * total / ((double)k * mp);              // cost.py:99
            c.has_ar = true;
            c.mbw = mp;
        }
    } else {
        const int kl = p.k(n), kr = p.k(n + 1);
        double mc = PP_INF;
        if (!p.table_min_cross(n, mc))
            for (int x = 0; x < kl; ++x)
                for (int y = 0; y < kr; ++y) mc = dmin(mc, I.w(p.dev(n, x), p.dev(n + 1, y)));   // cost.py:74-80
        const double denom = (double)(kl * kr) * mc;                              // cost.py:121-122
        const int edge = p.stage_le(n);
        c.dA = I.efwd[edge - 1] / denom;
        c.dB = I.ebwd[edge - 1] / denom;
        c.cyc = c.dA + c.dB;                                                      // cost.py:194
        c.mbw = mc;
    }
    return c;
}

// Block max-reduce of (cyc, ar) over the R active lanes; returns via smem.
__device__ void reduce_costs(const LaneCost& c, int lane, int R, int nthr, double* red, double* cyc_out,
                             double* ar_out) {
    double cy = (lane < R) ? c.cyc : -PP_INF;
    double ar = (lane < R && c.has_ar) ? c.ar : -PP_INF;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        cy = dmax(cy, __shfl_xor_sync(0xffffffffu, cy, off));
        ar = dmax(ar, __shfl_xor_sync(0xffffffffu, ar, off));
    }
    const int warp = lane >> 5;
    if ((lane & 31) == 0) { red[2 * warp] = cy; red[2 * warp + 1] = ar; }
    bar_sync(nthr);
    if (lane == 0) {
        double a = -PP_INF, b = -PP_INF;
        for (int w = 0; w < nthr / 32; ++w) { a = dmax(a, red[2 * w]); b = dmax(b, red[2 * w + 1]); }
        *cyc_out = a;
        *ar_out = (b == -PP_INF) ? 0.0 : b;   // max(..., default=0.0)  scheduler.py:237
    }
    bar_sync(nthr);
}

// ---- PE sweep (one plan per CTA) --------------------------------------------
// smem: fe[2][R], be[2][R], red[2*32] doubles
template <class P>
__device__ void pe_simulate(const P& p, const InstView& I, int N, int M, int nthr, double* sm, double* o_mk,
                            double* o_bound, double* ev_s, double* ev_e, double* ar_s, double* ar_e) {
    const int R = 2 * N - 1, J = 4 * N - 3;
    const int lane = threadIdx.x;
    double* fe = sm;            // [2][R]
    double* be = sm + 2 * R;    // [2][R]
    double* red = sm + 4 * R;   // [64]
    __shared__ double s_cyc, s_armax;
    LaneCost c{0.0, 0.0, 0.0, 0.0, false, 0.0, 0.0, PP_INF};
    if (lane < R) c = lane_cost(p, I, N, lane);
    reduce_costs(c, lane, R, nthr, red, &s_cyc, &s_armax);
    if (lane == 0) *o_bound = (double)(M + 4 * N - 4) * s_cyc + s_armax;   // scheduler.py:238

    const bool is_stage = (lane & 1) == 0;
    const int n = lane / 2 + 1;
    // positions of this lane's two items (backward-side first within a pass)
    int p_first, p_second;   // p_second = 0 when the lane has one item per pass
    if (is_stage) {
        if (n < N) { p_first = 4 * N - 1 - 2 * n; p_second = 2 * n - 1; }   // B_n, F_n
        else { p_first = 2 * N - 1; p_second = 0; }                       // FB_N
    } else { p_first = 4 * N - 2 - 2 * n; p_second = 2 * n; }              // Y_n, X_n
    // first item's predecessor: right neighbour's backward-side end, except FB_N (left, forward side)
    const bool first_from_left = is_stage && n == N;
    const bool has_left = lane > 0, has_right = lane + 1 < R;
    double rfree = 0.0;
    const int P_total = M + J - 1;
    for (int pass = 1; pass <= P_total; ++pass) {
        const int cur = pass & 1, prv = cur ^ 1;
        if (lane < R) {
            int m = pass - p_first + 1;
            if (m >= 1 && m <= M) {
                double pred;
                if (first_from_left) pred = has_left ? fe[prv * R + lane - 1] : 0.0;
                else pred = has_right ? be[prv * R + lane + 1] : 0.0;
                const double st = dmax(rfree, pred);
                const double en = st + c.dB;   // B / FB / Y
                rfree = en;
                be[cur * R + lane] = en;
                if (ev_s) { const int64_t x = (int64_t)(m - 1) * J + p_first - 1; ev_s[x] = st; ev_e[x] = en; }
            }
            if (p_second) {
                m = pass - p_second + 1;
                if (m >= 1 && m <= M) {
                    const double pred = has_left ? fe[prv * R + lane - 1] : 0.0;
                    const double st = dmax(rfree, pred);
                    const double en = st + c.dA;   // F / X
                    rfree = en;
                    fe[cur * R + lane] = en;
                    if (ev_s) { const int64_t x = (int64_t)(m - 1) * J + p_second - 1; ev_s[x] = st; ev_e[x] = en; }
                }
            }
        }
        bar_sync(nthr);
    }
    // AllReduce windows start at the stage's last compute end (scheduler.py:195-198)
    double arend = -PP_INF;
    if (lane < R && is_stage && c.has_ar) {
        arend = rfree + c.ar;
        if (ar_s) { ar_s[n - 1] = rfree; ar_e[n - 1] = arend; }
    }
    // makespan = max(last B_1 / FB_1 end, AllReduce ends)   (scheduler.py:216-220)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) arend = dmax(arend, __shfl_xor_sync(0xffffffffu, arend, off));
    if ((lane & 31) == 0) red[lane >> 5] = arend;
    if (lane == 0) red[40] = rfree;   // stage1 lane: end of B_1(M) (or FB_1(M))
    bar_sync(nthr);
    if (lane == 0) {
        double mk = red[40];
        for (int w = 0; w < nthr / 32; ++w) mk = dmax(mk, red[w]);
        *o_mk = mk;
    }
}

// One resource's pass of the PE recurrence, branch-free: the B / FB / Y block
// (p1) then the F / X block (p2) of this pass, each applied only while its
// microbatch index is in 1..M (inactive blocks are computed and discarded by a
// select, so the S resources of a lane are straight-line code the compiler
// interleaves — with per-resource branches their chains ran one after another:
// C3 n = 12 sweep ~590 cycles per pass for S = 4).  p1 / p2 far out of range
// disable a block (no F / X block on FB_N; resources past R).  Same fp64
// operations in the same order as pe_simulate when a block is active.
template <bool EV>
__device__ __forceinline__ void pe_pass_slot(int pass, int M, int J, int p1, int p2, bool from_left, double left,
                                             double right, double dA, double dB, double& rf, double& fn, double& bn,
                                             double* ev_s, double* ev_e) {
    const int m1 = pass - p1, m2 = pass - p2;   // microbatch - 1 of each block
    const bool a1 = (unsigned)m1 < (unsigned)M, a2 = (unsigned)m2 < (unsigned)M;
    const double st1 = dmax(rf, from_left ? left : right);
    const double en1 = st1 + dB;                 // B / FB / Y
    const double r1 = a1 ? en1 : rf;
    bn = a1 ? en1 : bn;
    const double st2 = dmax(r1, left);
    const double en2 = st2 + dA;                 // F / X
    rf = a2 ? en2 : r1;
    fn = a2 ? en2 : fn;
    if (EV) {
        if (a1) { const int64_t x = (int64_t)m1 * J + p1 - 1; ev_s[x] = st1; ev_e[x] = en1; }
        if (a2) { const int64_t x = (int64_t)m2 * J + p2 - 1; ev_s[x] = st2; ev_e[x] = en2; }
    }
}
constexpr int PE_OFF = -(1 << 29);   // p1 / p2 of a block that never runs

// ---- PE sweep, one WARP per plan (R = 2N-1 <= 32 S resources) ---------------
// Lane L holds resources q = L*S + s (contiguous blocks): a predecessor on the
// neighbouring resource is in the same lane's registers or one shuffle away, so
// a pass is register work plus two shuffles instead of a shared-memory round
// trip and a CTA barrier.  Same recurrence, same fp64 operations in the same
// order per resource as pe_simulate (bit-identical).
template <int S, bool EV, class P>
__device__ void pe_simulate_warp(const P& p, const InstView& I, int N, int M, double* o_mk, double* o_bound,
                                 double* ev_s, double* ev_e, double* ar_s, double* ar_e) {
    const unsigned FULL = 0xffffffffu;
    const int R = 2 * N - 1, J = 4 * N - 3;
    const int lane = threadIdx.x & 31;
    double dA[S], dB[S], ar[S], fe[S], be[S], rf[S];
    bool has_ar[S], act[S], from_left[S];
    int p1[S], p2[S];
    double cy = -PP_INF, am = -PP_INF;
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const int q = lane * S + s;
        act[s] = q < R;
        LaneCost c{0.0, 0.0, 0.0, 0.0, false, 0.0, 0.0, PP_INF};
        if (act[s]) c = lane_cost(p, I, N, q);
        dA[s] = c.dA; dB[s] = c.dB; ar[s] = c.ar; has_ar[s] = act[s] && c.has_ar;
        if (act[s]) cy = dmax(cy, c.cyc);
        if (has_ar[s]) am = dmax(am, c.ar);
        const bool st = (q & 1) == 0;
        const int n = q / 2 + 1;
        if (st) {
            if (n < N) { p1[s] = 4 * N - 1 - 2 * n; p2[s] = 2 * n - 1; }   // B_n, F_n
            else { p1[s] = 2 * N - 1; p2[s] = PE_OFF; }                  // FB_N (no F / X block)
        } else { p1[s] = 4 * N - 2 - 2 * n; p2[s] = 2 * n; }              // Y_n, X_n
        if (!act[s]) { p1[s] = PE_OFF; p2[s] = PE_OFF; }
        from_left[s] = st && n == N;
        fe[s] = 0.0; be[s] = 0.0; rf[s] = 0.0;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        cy = dmax(cy, __shfl_xor_sync(FULL, cy, off));
        am = dmax(am, __shfl_xor_sync(FULL, am, off));
    }
    if (lane == 0) *o_bound = (double)(M + 4 * N - 4) * cy + (am == -PP_INF ? 0.0 : am);   // scheduler.py:238
    const int P_total = M + J - 1;
    for (int pass = 1; pass <= P_total; ++pass) {
        // neighbours' pass-1 ends: left fe of q-1, right be of q+1
        const double fe_in = __shfl_up_sync(FULL, fe[S - 1], 1);
        const double be_in = __shfl_down_sync(FULL, be[0], 1);
        double fn[S], bn[S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            fn[s] = fe[s]; bn[s] = be[s];
            const int q = lane * S + s;
            const double left = q == 0 ? 0.0 : (s > 0 ? fe[s - 1] : fe_in);
            const double right = q + 1 >= R ? 0.0 : (s + 1 < S ? be[s + 1] : be_in);
            pe_pass_slot<EV>(pass, M, J, p1[s], p2[s], from_left[s], left, right, dA[s], dB[s], rf[s], fn[s], bn[s],
                             ev_s, ev_e);
        }
#pragma unroll
        for (int s = 0; s < S; ++s) { fe[s] = fn[s]; be[s] = bn[s]; }
    }
    // AllReduce windows start at the stage's last compute end (scheduler.py:195-198);
    // makespan = max(last B_1 / FB_1 end, AllReduce ends)   (scheduler.py:216-220)
    double arend = -PP_INF;
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const int q = lane * S + s;
        if (act[s] && (q & 1) == 0 && has_ar[s]) {
            const double e = rf[s] + ar[s];
            arend = dmax(arend, e);
            if (ar_s) { ar_s[q / 2] = rf[s]; ar_e[q / 2] = e; }
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) arend = dmax(arend, __shfl_xor_sync(FULL, arend, off));
    if (lane == 0) *o_mk = dmax(rf[0], arend);
}

// ---- PE sweep, nw WARPS per plan (R = 2N-1 <= 32 nw S): the warp version's
// register blocks, with the two resources at each warp boundary exchanged
// through shared memory (double-buffered by pass parity) and one named barrier
// of the nw warps per pass.  Replaces the one-resource-per-thread CTA sweep
// (pe_simulate) for large N: S independent resources per lane give the pass
// ILP and the barrier spans nw = R / 128 warps instead of R / 32 (C5's
// xi = 256 plan: 1532 passes at ~1.4 k cycles each before).  Same recurrence,
// same fp64 operations in the same order per resource (bit-identical).
// smem: xch[2][2][nw] (fe, be boundary values per pass parity) + red[2 nw]
template <int S, bool EV, class P>
__device__ void pe_simulate_mw(const P& p, const InstView& I, int N, int M, int nw, double* sm, double* o_mk,
                               double* o_bound, double* ev_s, double* ev_e, double* ar_s, double* ar_e) {
    const unsigned FULL = 0xffffffffu;
    const int R = 2 * N - 1, J = 4 * N - 3;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nthr = 32 * nw;
    double* xfe = sm;            // [2][nw]: fe of the warp's last resource
    double* xbe = sm + 2 * nw;   // [2][nw]: be of the warp's first resource
    double* red = sm + 4 * nw;   // [2][nw]
    double dA[S], dB[S], ar[S], fe[S], be[S], rf[S];
    bool has_ar[S], act[S], from_left[S];
    int p1[S], p2[S];
    double cy = -PP_INF, am = -PP_INF;
    const int q0 = (warp * 32 + lane) * S;
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const int q = q0 + s;
        act[s] = q < R;
        LaneCost c{0.0, 0.0, 0.0, 0.0, false, 0.0, 0.0, PP_INF};
        if (act[s]) c = lane_cost(p, I, N, q);
        dA[s] = c.dA; dB[s] = c.dB; ar[s] = c.ar; has_ar[s] = act[s] && c.has_ar;
        if (act[s]) cy = dmax(cy, c.cyc);
        if (has_ar[s]) am = dmax(am, c.ar);
        const bool st = (q & 1) == 0;
        const int n = q / 2 + 1;
        if (st) {
            if (n < N) { p1[s] = 4 * N - 1 - 2 * n; p2[s] = 2 * n - 1; }   // B_n, F_n
            else { p1[s] = 2 * N - 1; p2[s] = PE_OFF; }                  // FB_N (no F / X block)
        } else { p1[s] = 4 * N - 2 - 2 * n; p2[s] = 2 * n; }              // Y_n, X_n
        if (!act[s]) { p1[s] = PE_OFF; p2[s] = PE_OFF; }
        from_left[s] = st && n == N;
        fe[s] = 0.0; be[s] = 0.0; rf[s] = 0.0;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        cy = dmax(cy, __shfl_xor_sync(FULL, cy, off));
        am = dmax(am, __shfl_xor_sync(FULL, am, off));
    }
    if (lane == 0) { red[warp] = cy; red[nw + warp] = am; xfe[warp] = 0.0; xbe[warp] = 0.0; }
    if (nw > 1) bar_sync(nthr);
    if (threadIdx.x == 0) {
        for (int w = 1; w < nw; ++w) { cy = dmax(cy, red[w]); am = dmax(am, red[nw + w]); }
        *o_bound = (double)(M + 4 * N - 4) * cy + (am == -PP_INF ? 0.0 : am);   // scheduler.py:238
    }
    const int P_total = M + J - 1;
    for (int pass = 1; pass <= P_total; ++pass) {
        const int cur = pass & 1, prv = cur ^ 1;
        // neighbours' pass-1 ends: left fe of q-1, right be of q+1 (other warps' via xch)
        double fe_in = __shfl_up_sync(FULL, fe[S - 1], 1);
        double be_in = __shfl_down_sync(FULL, be[0], 1);
        if (lane == 0) fe_in = warp > 0 ? xfe[prv * nw + warp - 1] : 0.0;
        if (lane == 31) be_in = warp + 1 < nw ? xbe[prv * nw + warp + 1] : 0.0;
        double fn[S], bn[S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            fn[s] = fe[s]; bn[s] = be[s];
            const int q = q0 + s;
            const double left = q == 0 ? 0.0 : (s > 0 ? fe[s - 1] : fe_in);
            const double right = q + 1 >= R ? 0.0 : (s + 1 < S ? be[s + 1] : be_in);
            pe_pass_slot<EV>(pass, M, J, p1[s], p2[s], from_left[s], left, right, dA[s], dB[s], rf[s], fn[s], bn[s],
                             ev_s, ev_e);
        }
#pragma unroll
        for (int s = 0; s < S; ++s) { fe[s] = fn[s]; be[s] = bn[s]; }
        if (nw > 1) {
            if (lane == 31) xfe[cur * nw + warp] = fe[S - 1];
            if (lane == 0) xbe[cur * nw + warp] = be[0];
            bar_sync(nthr);
        }
    }
    // AllReduce windows start at the stage's last compute end (scheduler.py:195-198);
    // makespan = max(last B_1 / FB_1 end, AllReduce ends)   (scheduler.py:216-220)
    double arend = -PP_INF;
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const int q = q0 + s;
        if (act[s] && (q & 1) == 0 && has_ar[s]) {
            const double e = rf[s] + ar[s];
            arend = dmax(arend, e);
            if (ar_s) { ar_s[q / 2] = rf[s]; ar_e[q / 2] = e; }
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) arend = dmax(arend, __shfl_xor_sync(FULL, arend, off));
    if (nw > 1) {
        if (lane == 0) red[warp] = arend;
        bar_sync(nthr);
        if (threadIdx.x == 0)
            for (int w = 1; w < nw; ++w) arend = dmax(arend, red[w]);
    }
    if (threadIdx.x == 0) *o_mk = dmax(rf[0], arend);
}
constexpr int PE_MW_S = 4;   // resources per lane of the multi-warp sweep (spp sweeps with V > 64: C5 full
                             // spp sweep 2.7 -> 1.6 ms; 1 per lane measured 2.7 ms)
__host__ __device__ inline int pe_mw_warps(int N) { return (2 * N - 1 + 32 * PE_MW_S - 1) / (32 * PE_MW_S); }

template <class P>
__device__ void pe_simulate_warp_any(const P& p, const InstView& I, int N, int M, double* o_mk, double* o_bound,
                                     double* ev_s, double* ev_e, double* ar_s, double* ar_e) {
    const int R = 2 * N - 1;
    if (ev_s) {
        if (R <= 32) pe_simulate_warp<1, true>(p, I, N, M, o_mk, o_bound, ev_s, ev_e, ar_s, ar_e);
        else if (R <= 64) pe_simulate_warp<2, true>(p, I, N, M, o_mk, o_bound, ev_s, ev_e, ar_s, ar_e);
        else if (R <= 96) pe_simulate_warp<3, true>(p, I, N, M, o_mk, o_bound, ev_s, ev_e, ar_s, ar_e);
        else pe_simulate_warp<4, true>(p, I, N, M, o_mk, o_bound, ev_s, ev_e, ar_s, ar_e);
    } else {
        if (R <= 32) pe_simulate_warp<1, false>(p, I, N, M, o_mk, o_bound, ev_s, ev_e, ar_s, ar_e);
        else if (R <= 64) pe_simulate_warp<2, false>(p, I, N, M, o_mk, o_bound, ev_s, ev_e, ar_s, ar_e);
        else if (R <= 96) pe_simulate_warp<3, false>(p, I, N, M, o_mk, o_bound, ev_s, ev_e, ar_s, ar_e);
        else pe_simulate_warp<4, false>(p, I, N, M, o_mk, o_bound, ev_s, ev_e, ar_s, ar_e);
    }
}

// k_pe_sweep / k_replay with one warp per plan (every N of the batch <= PE_WARP_MAXN)
constexpr int PE_WARP_MAXN = 64;
__global__ void __launch_bounds__(32) k_pe_sweep_w(pp_batch b) {
    const pp_instance I = b.inst[blockIdx.x];
    const int xi = blockIdx.y + 1;
    if (xi > I.V) return;
    const int64_t so = I.sweep_off + xi - 1;
    if (b.sweep_r[so] == 0) {   // infeasible: SweepEntry(makespan=None, bound=None)
        if (threadIdx.x == 0) { b.sweep_mk[so] = PP_INF; b.sweep_bound[so] = PP_INF; }
        return;
    }
    const int64_t st = I.stage_off + (int64_t)xi * (xi - 1) / 2;
    SppPlanView p{b.stage_ls + st, b.stage_le + st, b.stage_dlo + st, b.stage_dhi + st, b.order + I.order_off};
    const WsLayout lay = ws_layout(I.L, I.V);
    p.minpair = b.ws + I.ws_off + lay.minpair; p.cross = b.ws + I.ws_off + lay.cross; p.V = I.V;
    InstView iv(b, I);
    pe_simulate_warp_any(p, iv, xi, I.M, b.sweep_mk + so, b.sweep_bound + so, nullptr, nullptr, nullptr, nullptr);
}

__global__ void __launch_bounds__(32) k_replay_w(pp_batch b) {
    const pp_instance I = b.inst[blockIdx.x];
    const int xi = b.best_xi[blockIdx.x];
    if (xi <= 0) return;
    __shared__ double s_mk, s_bd;
    const int64_t st = I.stage_off + (int64_t)xi * (xi - 1) / 2;
    SppPlanView p{b.stage_ls + st, b.stage_le + st, b.stage_dlo + st, b.stage_dhi + st, b.order + I.order_off};
    const WsLayout lay = ws_layout(I.L, I.V);
    p.minpair = b.ws + I.ws_off + lay.minpair; p.cross = b.ws + I.ws_off + lay.cross; p.V = I.V;
    InstView iv(b, I);
    pe_simulate_warp_any(p, iv, xi, I.M, &s_mk, &s_bd, b.ev_start + I.ev_off, b.ev_end + I.ev_off,
                         b.ar_start + I.ar_off, b.ar_end + I.ar_off);
}

// Resource sort key of block position p in an N-stage plan (scheduler.py:115-118
// via model.py:148-158): compute blocks sort by stage, channels after all
// stages by channel index.
__device__ __forceinline__ int ev_key(int N, int p) {
    if (p & 1) return p <= 2 * N - 1 ? (p + 1) >> 1 : (4 * N - 1 - p) >> 1;
    return (1 << 20) + (p <= 2 * N - 2 ? p >> 1 : (4 * N - 2 - p) >> 1);
}

// The reference's event order of the selected plan's schedule: events sorted by
// (start, resource key, microbatch, position) (scheduler.py:227-231), a strict
// total order.  Each position q is served by one resource in increasing
// microbatch order, so its column start(., q) is non-decreasing in m: the J
// columns are already-sorted runs and ordering the events is a merge.
__device__ __forceinline__ uint64_t ev_tie(int N, int J, int e) {
    const int m = e / J, p = e - m * J + 1;   // m 0-based
    return ((uint64_t)ev_key(N, p) << 43) | ((uint64_t)m << 12) | (uint64_t)p;
}

// k_event_merge: one CTA per instance, start times staged in shared memory, the
// J runs merged pairwise (ceil(log2 J) levels, merge-path split per thread,
// 16-bit event indices ping-ponged in shared memory).  n = M (4N-3) <= EM_MAXN;
// the host sizes shared memory and the block (<= EM_T) from the batch's max_M.
constexpr int EM_T = 1024;
constexpr int EM_SMEM = 216 * 1024;
constexpr int EM_MAXN = EM_SMEM / 12 < 65536 ? EM_SMEM / 12 : 65536;
__global__ void __launch_bounds__(EM_T) k_event_merge(pp_batch b) {
    const pp_instance I = b.inst[blockIdx.x];
    const int N = b.best_xi[blockIdx.x];
    if (N <= 0) return;
    const int M = I.M, J = 4 * N - 3, n = M * J;
    if (n > EM_MAXN) return;   // k_event_rank orders it
    extern __shared__ __align__(16) double em_key[];
    unsigned short* A = reinterpret_cast<unsigned short*>(em_key + n);
    unsigned short* B = A + n;
    const double* st = b.ev_start + I.ev_off;
    const int t = threadIdx.x;
    const int T = blockDim.x;
    for (int k = t; k < n; k += T) {
        em_key[k] = st[k];
        const int q = k / M, m = k - q * M;   // run q = column q+1, in microbatch order
        A[k] = (unsigned short)(m * J + q);
    }
    __syncthreads();
    auto less = [&](int x, int y) {
        const double u = em_key[x], v = em_key[y];
        return u != v ? u < v : ev_tie(N, J, x) < ev_tie(N, J, y);
    };
    const int per = (n + T - 1) / T;
    for (int R = M; R < n; R *= 2) {
        int o = t * per;
        const int oend = min(n, o + per);
        while (o < oend) {
            const int base = o / (2 * R) * (2 * R);
            const int la = min(R, n - base), lb = max(0, min(R, n - base - R));
            const unsigned short* X = A + base;
            const unsigned short* Y = X + la;
            const int d = o - base;
            int lo = max(0, d - lb), hi = min(d, la);   // merge path: X elements among the first d
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (less(X[mid], Y[d - 1 - mid])) lo = mid + 1; else hi = mid;
            }
            int xi = lo, yi = d - lo;
            const int stop = min(oend, base + la + lb);
            // the two heads (index + start) stay in registers: one shared load per output
            int ex = xi < la ? X[xi] : 0, ey = yi < lb ? Y[yi] : 0;
            double kx = em_key[ex], ky = em_key[ey];
            for (; o < stop; ++o) {
                const bool takeX = yi >= lb || (xi < la && (kx != ky ? kx < ky : ev_tie(N, J, ex) < ev_tie(N, J, ey)));
                if (takeX) {
                    B[o] = (unsigned short)ex;
                    if (++xi < la) { ex = X[xi]; kx = em_key[ex]; }
                } else {
                    B[o] = (unsigned short)ey;
                    if (++yi < lb) { ey = Y[yi]; ky = em_key[ey]; }
                }
            }
        }
        __syncthreads();
        unsigned short* T = A; A = B; B = T;
    }
    for (int k = t; k < n; k += T) b.ev_order[I.ev_off + k] = A[k];
}

// k_event_rank: instances too large for k_event_merge.  One thread per event,
// its rank = sum over columns of a binary search for the events below it
// (O(J log M) loads per event); ranks are a permutation.
__global__ void __launch_bounds__(256) k_event_rank(pp_batch b) {
    const pp_instance I = b.inst[blockIdx.x];
    const int N = b.best_xi[blockIdx.x];
    if (N <= 0) return;
    const int M = I.M, J = 4 * N - 3, n = M * J;
    if (n <= EM_MAXN) return;
    const double* st = b.ev_start + I.ev_off;
    for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < n; e += gridDim.y * blockDim.x) {
        const double s = st[e];
        const uint64_t te = ev_tie(N, J, e);
        int rank = 0;
        for (int q = 1; q <= J; ++q) {
            const double* col = st + (q - 1);
            int a = 0, c = M;   // #{m' : (start, tie)(m', q) < (s, te)}: the column is sorted by it
            while (a < c) {
                const int mid = (a + c) >> 1;
                const double v = col[(int64_t)mid * J];
                if (v < s || (v == s && ev_tie(N, J, mid * J + q - 1) < te)) a = mid + 1; else c = mid;
            }
            rank += a;
        }
        b.ev_order[I.ev_off + rank] = e;
    }
}

__host__ __device__ inline int sim_threads(int N) {
    const int R = 2 * N - 1;
    const int t = (R + 31) / 32 * 32;
    return t < 32 ? 32 : t;
}

// Every feasible xi plan of every instance: grid (n_inst, maxV), block 32 pe_mw_warps(maxV).
__global__ void __launch_bounds__(1024) k_pe_sweep(pp_batch b) {
    const pp_instance I = b.inst[blockIdx.x];
    const int xi = blockIdx.y + 1;
    if (xi > I.V) return;
    const int64_t so = I.sweep_off + xi - 1;
    if (b.sweep_r[so] == 0) {   // infeasible: SweepEntry(makespan=None, bound=None)
        if (threadIdx.x == 0) { b.sweep_mk[so] = PP_INF; b.sweep_bound[so] = PP_INF; }
        return;
    }
    const int nw = pe_mw_warps(xi);
    if ((int)threadIdx.x >= 32 * nw) return;
    extern __shared__ double smem_d[];
    const int64_t st = I.stage_off + (int64_t)xi * (xi - 1) / 2;
    SppPlanView p{b.stage_ls + st, b.stage_le + st, b.stage_dlo + st, b.stage_dhi + st, b.order + I.order_off};
    InstView iv(b, I);
    pe_simulate_mw<PE_MW_S, false>(p, iv, xi, I.M, nw, smem_d, b.sweep_mk + so, b.sweep_bound + so, nullptr, nullptr,
                            nullptr, nullptr);
}

// spp selection (planner.py:66-77): first xi with strictly smallest makespan.
__global__ void __launch_bounds__(32) k_select(pp_batch b) {
    const pp_instance I = b.inst[blockIdx.x];
    const int lane = threadIdx.x;
    double best = PP_INF;
    int bx = 0;
    for (int xi = 1 + lane; xi <= I.V; xi += 32) {
        const int64_t so = I.sweep_off + xi - 1;
        if (b.sweep_r[so] == 0) continue;
        const double v = b.sweep_mk[so];
        if (bx == 0 || v < best) { best = v; bx = xi; }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, off);
        const int ox = __shfl_xor_sync(0xffffffffu, bx, off);
        if (ox != 0 && (bx == 0 || ov < best || (ov == best && ox < bx))) { best = ov; bx = ox; }
    }
    if (lane == 0) { b.best_xi[blockIdx.x] = bx; b.best_mk[blockIdx.x] = best; }
}

// Replay the selected plan with event capture: grid n_inst, block 32 pe_mw_warps(maxV).
__global__ void __launch_bounds__(1024) k_replay(pp_batch b) {
    const pp_instance I = b.inst[blockIdx.x];
    const int xi = b.best_xi[blockIdx.x];
    if (xi <= 0) return;
    const int nw = pe_mw_warps(xi);
    if ((int)threadIdx.x >= 32 * nw) return;
    extern __shared__ double smem_d[];
    __shared__ double s_mk, s_bd;
    const int64_t st = I.stage_off + (int64_t)xi * (xi - 1) / 2;
    SppPlanView p{b.stage_ls + st, b.stage_le + st, b.stage_dlo + st, b.stage_dhi + st, b.order + I.order_off};
    InstView iv(b, I);
    pe_simulate_mw<PE_MW_S, true>(p, iv, xi, I.M, nw, smem_d, &s_mk, &s_bd, b.ev_start + I.ev_off, b.ev_end + I.ev_off,
                            b.ar_start + I.ar_off, b.ar_end + I.ar_off);
}

// ---- plan costs (cost_summary, cost.py:172-202; channel_times :162-169;
// block_durations :205-230): per-lane records + workload + Lemma-1 bound.
// workload = max(M*compute_s (+ A_s if replicated), M*(c_fwd+c_bwd)_n); max is
// order-free, so the lane-parallel reduction is the reference's max(w_terms).
__device__ void plan_costs(const LaneCost& c, int lane, int R, int M, int nthr, double* red, double* lane_out,
                           double* o_workload) {
    if (lane < R && lane_out) {
        double* o = lane_out + (int64_t)lane * PP_LANE_COST_FIELDS;
        o[0] = c.dA; o[1] = c.dB; o[2] = c.cyc; o[3] = c.has_ar ? c.ar : 0.0;
        o[4] = c.fs; o[5] = c.bs; o[6] = c.mbw;
    }
    if (!o_workload) return;
    double w = -PP_INF;
    if (lane < R) {
        w = (double)M * c.cyc;
        if (c.has_ar) w = w + c.ar;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) w = dmax(w, __shfl_xor_sync(0xffffffffu, w, off));
    if ((lane & 31) == 0) red[64 + (lane >> 5)] = w;
    bar_sync(nthr);
    if (lane == 0) {
        double a = -PP_INF;
        for (int k = 0; k < nthr / 32; ++k) a = dmax(a, red[64 + k]);
        *o_workload = a;
    }
    bar_sync(nthr);
}

// ---- lockstep cycle schedule (scheduler.py:241-296) ---------------------------
// Cycle c runs position p on microbatch m = c - p + 1 (the wavefront the
// "completed[p-1] > completed[p]" rule produces); a resource runs its chosen
// blocks back to back in ascending position order starting at the cycle
// start t, and the next cycle starts at max(t, every end of this cycle).
// M + 4N - 4 cycles.  red: [2][32] doubles (double-buffered cycle maxima).
__device__ void cycle_simulate(const LaneCost& c, int N, int M, int nthr, double* red, double* ev_s, double* ev_e,
                               double* ar_s, double* ar_e, double* o_mk) {
    const int R = 2 * N - 1, J = 4 * N - 3;
    const int lane = threadIdx.x;
    const bool is_stage = (lane & 1) == 0;
    const int n = lane / 2 + 1;
    int p_lo, p_hi;   // ascending positions; p_hi = 0 when the lane has one block
    if (is_stage) {
        if (n < N) { p_lo = 2 * n - 1; p_hi = 4 * N - 1 - 2 * n; }   // F_n, B_n
        else { p_lo = 2 * N - 1; p_hi = 0; }                        // FB_N
    } else { p_lo = 2 * n; p_hi = 4 * N - 2 - 2 * n; }              // X_n, Y_n
    const int nw = nthr / 32;
    double t = 0.0, last = 0.0;
    const int cycles = M + J - 1;
    for (int cy = 1; cy <= cycles; ++cy) {
        double clock = t;
        if (lane < R) {
            int m = cy - p_lo + 1;
            if (m >= 1 && m <= M) {
                const double st = clock, en = st + c.dA;
                clock = en;
                last = en;
                if (ev_s) { const int64_t x = (int64_t)(m - 1) * J + p_lo - 1; ev_s[x] = st; ev_e[x] = en; }
            }
            m = cy - p_hi + 1;
            if (p_hi && m >= 1 && m <= M) {
                const double st = clock, en = st + c.dB;
                clock = en;
                last = en;
                if (ev_s) { const int64_t x = (int64_t)(m - 1) * J + p_hi - 1; ev_s[x] = st; ev_e[x] = en; }
            }
        }
        double v = clock;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v = dmax(v, __shfl_xor_sync(0xffffffffu, v, off));
        double* buf = red + (cy & 1) * 32;
        if ((lane & 31) == 0) buf[lane >> 5] = v;
        bar_sync(nthr);
        double tn = buf[0];
        for (int k = 1; k < nw; ++k) tn = dmax(tn, buf[k]);
        t = tn;
    }
    // AllReduce at the stage's last compute end; makespan = max(end of B_1(M) / FB_1(M), AR ends)
    double arend = -PP_INF;
    if (lane < R && is_stage && c.has_ar) {
        arend = last + c.ar;
        if (ar_s) { ar_s[n - 1] = last; ar_e[n - 1] = arend; }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) arend = dmax(arend, __shfl_xor_sync(0xffffffffu, arend, off));
    if ((lane & 31) == 0) red[64 + (lane >> 5)] = arend;
    if (lane == 0) red[96] = last;
    bar_sync(nthr);
    if (lane == 0) {
        double mk = red[96];
        for (int k = 0; k < nw; ++k) mk = dmax(mk, red[64 + k]);
        *o_mk = mk;
    }
}

// ---- caller plans -------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_sim_plans(pp_batch b, pp_sim_batch s) {
    const pp_plan P = s.plan[blockIdx.x];
    const pp_instance I = b.inst[P.inst];
    const int N = P.N, M = P.M, R = 2 * N - 1, J = 4 * N - 3;
    const int nthr = sim_threads(N);
    if ((int)threadIdx.x >= nthr) return;
    extern __shared__ double smem_d[];
    ExplicitPlanView pv{s.ls + P.stage_off, s.le + P.stage_off, s.dev_off + P.devoff_off, s.devs};
    InstView iv(b, I);
    double* ev_s = s.ev_start ? s.ev_start + P.ev_off : nullptr;
    double* ev_e = s.ev_end ? s.ev_end + P.ev_off : nullptr;
    if (P.flags & (PP_SIM_CYCLE | PP_SIM_COSTS_ONLY) || s.lane_cost || s.workload) {
        const int lane = threadIdx.x;
        double* red = smem_d;   // [128]
        __shared__ double s_cyc, s_armax;
        LaneCost c{0.0, 0.0, 0.0, 0.0, false, 0.0, 0.0, PP_INF};
        if (lane < R) c = lane_cost(pv, iv, N, lane);
        reduce_costs(c, lane, R, nthr, red, &s_cyc, &s_armax);
        if (lane == 0) s.bound[blockIdx.x] = (double)(M + 4 * N - 4) * s_cyc + s_armax;
        plan_costs(c, lane, R, M, nthr, red, s.lane_cost ? s.lane_cost + P.lane_off * PP_LANE_COST_FIELDS : nullptr,
                   s.workload ? s.workload + blockIdx.x : nullptr);
        if (P.flags & (PP_SIM_CYCLE | PP_SIM_COSTS_ONLY)) {
            const bool cyc = P.flags & PP_SIM_CYCLE;
            if (cyc)
                cycle_simulate(c, N, M, nthr, red, ev_s, ev_e, s.ar_start + P.ar_off, s.ar_end + P.ar_off,
                               s.makespan + blockIdx.x);
            if (lane == 0) {
                s.status[blockIdx.x] = 0;
                s.n_done[blockIdx.x] = cyc ? (int64_t)M * J : 0;
                if (!cyc) s.makespan[blockIdx.x] = 0.0;
                if (s.cycles) s.cycles[blockIdx.x] = cyc ? M + J - 1 : 0;
            }
            for (int r = lane; r < R; r += nthr) s.head[P.lane_off + r] = -1;
            return;
        }
        bar_sync(nthr);
    }
    if (P.flags & PP_SIM_PE_ORDER) {
        // caller plans keep one resource per thread: measured faster than the
        // multi-warp sweep on C5's 256 plans (711 vs 877-931 ns per pass of xi = 256)
        pe_simulate(pv, iv, N, M, nthr, smem_d, s.makespan + blockIdx.x, s.bound + blockIdx.x, ev_s, ev_e,
                    s.ar_start + P.ar_off, s.ar_end + P.ar_off);
        if (threadIdx.x == 0) { s.status[blockIdx.x] = 0; s.n_done[blockIdx.x] = (int64_t)M * J; }
        for (int r = threadIdx.x; r < R; r += nthr) s.head[P.lane_off + r] = -1;
        return;
    }
    // Generic queues: round-based sweep.  comp[(m-1)*J + pos-1] = end time, < 0 = not finished.
    const int lane = threadIdx.x;
    const bool fb = P.flags & PP_SIM_FORWARD_BARRIER;
    double* red = smem_d;   // [64]
    __shared__ double s_cyc, s_armax, s_T;
    __shared__ int s_open;
    __shared__ long long s_prog, s_fwd;
    __shared__ double s_fmax[32];
    LaneCost c{0.0, 0.0, 0.0, 0.0, false, 0.0, 0.0, PP_INF};
    if (lane < R) c = lane_cost(pv, iv, N, lane);
    reduce_costs(c, lane, R, nthr, red, &s_cyc, &s_armax);
    if (lane == 0) s.bound[blockIdx.x] = (double)(M + 4 * N - 4) * s_cyc + s_armax;
    volatile double* comp = s.scratch + P.ev_off;
    for (int64_t x = lane; x < (int64_t)M * J; x += nthr) comp[x] = -1.0;
    const int q0 = (lane < R) ? s.q_off[P.queue_off + lane] : 0;
    const int q1 = (lane < R) ? s.q_off[P.queue_off + lane + 1] : 0;
    const int* items = s.q_items;
    const long long fwd_total = (long long)M * 2 * (N - 1);
    if (lane == 0) { s_open = (!fb || fwd_total == 0) ? 1 : 0; s_T = 0.0; s_fwd = 0; }
    __threadfence_block();
    bar_sync(nthr);
    int head = q0;
    double rfree = 0.0, my_fmax = -PP_INF;
    long long my_fwd = 0;
    for (;;) {
        long long prog = 0;
        const int open = s_open;
        const double T = s_T;
        while (head < q1) {
            const int m = items[2 * head], pos = items[2 * head + 1];
            // forward-side kinds are F (odd pos < 2N-1) and X (even pos < 2N-1); N == 1 has none
            const bool fwd_side = N > 1 && pos < 2 * N - 1;
            if (fb && !fwd_side && !open) break;
            double pred = 0.0;
            if (pos > 1) {
                pred = comp[(int64_t)(m - 1) * J + pos - 2];
                if (pred < 0.0) break;
            }
            double st = dmax(rfree, pred);
            if (fb && !fwd_side) st = dmax(st, T);
            const double en = st + (fwd_side ? c.dA : c.dB);
            rfree = en;
            const int64_t x = (int64_t)(m - 1) * J + pos - 1;
            if (ev_s) { ev_s[x] = st; ev_e[x] = en; }
            __threadfence_block();
            comp[x] = en;
            ++head; ++prog;
            if (fb && fwd_side) { ++my_fwd; my_fmax = dmax(my_fmax, en); }
        }
        // round barrier: progress and forward-completion reductions
        if (lane == 0) s_prog = 0;
        bar_sync(nthr);
        if (prog) atomicAdd((unsigned long long*)&s_prog, (unsigned long long)prog);
        double fm = my_fmax;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) fm = dmax(fm, __shfl_xor_sync(0xffffffffu, fm, off));
        if ((lane & 31) == 0) s_fmax[lane >> 5] = fm;
        if (my_fwd) { atomicAdd((unsigned long long*)&s_fwd, (unsigned long long)my_fwd); my_fwd = 0; }
        bar_sync(nthr);
        bool newly = false;
        if (!s_open && s_fwd == fwd_total) newly = true;
        const long long total_prog = s_prog;
        bar_sync(nthr);
        if (newly) {
            if (lane == 0) {
                double T2 = -PP_INF;
                for (int w = 0; w < nthr / 32; ++w) T2 = dmax(T2, s_fmax[w]);
                s_T = T2;   // barrier opens when the last forward-side item ends (scheduler.py:190-194)
                s_open = 1;
            }
            bar_sync(nthr);
            continue;
        }
        if (total_prog == 0) break;
    }
    // results
    int64_t my_done = (lane < R) ? (int64_t)(head - q0) : 0;
    if (lane < R) s.head[P.lane_off + lane] = (head < q1) ? head - q0 : -1;
    __shared__ unsigned long long s_done;
    if (lane == 0) s_done = 0;
    bar_sync(nthr);
    atomicAdd(&s_done, (unsigned long long)my_done);
    bar_sync(nthr);
    const bool ok = s_done == (unsigned long long)((int64_t)M * J);
    double arend = -PP_INF;
    if (ok && lane < R && (lane & 1) == 0 && c.has_ar) {
        const int n = lane / 2 + 1;
        s.ar_start[P.ar_off + n - 1] = rfree;
        s.ar_end[P.ar_off + n - 1] = rfree + c.ar;
        arend = rfree + c.ar;
    }
    // finish = max over m of end(m, J)
    double fin = -PP_INF;
    if (ok)
        for (int m = 1 + lane; m <= M; m += nthr) fin = dmax(fin, comp[(int64_t)(m - 1) * J + J - 1]);
    double v = dmax(fin, arend);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = dmax(v, __shfl_xor_sync(0xffffffffu, v, off));
    if ((lane & 31) == 0) red[lane >> 5] = v;
    bar_sync(nthr);
    if (lane == 0) {
        double mk = -PP_INF;
        for (int w = 0; w < nthr / 32; ++w) mk = dmax(mk, red[w]);
        s.makespan[blockIdx.x] = ok ? mk : 0.0;
        s.status[blockIdx.x] = ok ? 0 : 1;
        s.n_done[blockIdx.x] = (int64_t)s_done;
    }
}

}  // namespace pp

namespace pp {
// Measurement kernel (bench.py roofline denominator): peak issue rate of the
// fp64 min/max pipe (DMNMX), 8 independent chains per thread, 2 ops per link
// (one max + one min, the same pair the DP spends per factored candidate).
__global__ void __launch_bounds__(256) k_peak_minmax(double* out, int iters, double seed) {
    double x[8];
    const double y = seed + 1e-9 * threadIdx.x;
    const double z = seed * 3.0 + 1e-7 * blockIdx.x;
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = seed * (k + 1);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
            const double a = dmin(dmax(x[k], y), x[k + 1]);
            const double c = dmax(dmin(x[k + 1], z), x[k]);
            x[k] = a;
            x[k + 1] = c;
        }
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.678) out[0] = s;   // never true; keeps the chains alive
}
}  // namespace pp

// dp_persist.cu — the PRM wavefront as ONE persistent, dependency-driven kernel
// (shared-memory path: L <= SR_MAX and V <= SR_MAX).
//
// The per-step launch schedule (prm.cu) puts a grid-wide barrier after every
// expand and every combine: 2(V-1) dependent launches, most of them a partial
// wave.  But only ONE item per step is on the critical path.  Slice i is
// complete once every item (r, i) is done, item (r, i) needs slice j = i - r,
// and the combine of item (r, j + r) is not read until step j + r — so for
// r >= 2 it has r - 1 steps of slack.  The chain is
//     (1, 2) -> (1, 3) -> ... -> (1, V)      (plus the r = 2 items of step j-1)
// and everything else can overlap it.
//
// Tasks (one CTA each, pulled in list order from an atomic queue; a task spins
// on per-instance counters until its inputs are complete, then signals):
//   E1(n, j, g)     expand of the critical target (1, j+1), row group g
//                   (warp per row l', lanes over xi).     waits: slice j of n
//   Eb(n, j, rows)  expand rows for the targets r = 2..V-j.  waits: slice j of n
//   C1(n, j, p)     combine of the critical item (1, j+1) over the l' chunk p
//                   (split-K: exact 64-bit atomicMin into +inf-preset cells).
//                                                          waits: all E1(n, j)
//   Cb(n, j, r, p)  combine of item (r, j + r), part p.  waits: all Eb(n, j)
// List order: for j = 1..V-1: E1(., j), Eb(., j), C1(., j), Cb(., j-1, r asc.).
// Every dependency of a task precedes it in the list, and a task is only
// pulled by a running CTA, so the earliest unfinished task can always run:
// no deadlock, whatever the residency.  Numerics are the per-step kernels'
// device functions unchanged (same fp64 expressions, same min/max sets), so
// every W cell is bit-identical to the launch-per-step path.
#include "common.cuh"

namespace pp {

constexpr int DP_T = 256;      // threads per persistent CTA
constexpr int DP_MAXJ = SR_MAX;
constexpr int DP_R1 = DP_T / 32;   // rows per critical-expand task: one per warp
constexpr int DP_RSPLIT = 4;       // items with r <= DP_RSPLIT are split over l' chunks

__host__ __device__ __forceinline__ int dp_rows_per_task(int j) { return j < 4 ? 8 : (j < 8 ? 4 : (j < 16 ? 2 : 1)); }
// l' chunks (split-K parts) of the combine of item (r, .): an item is read r steps
// after it becomes computable, so the short-slack ones are spread over more CTAs
__host__ __device__ __forceinline__ int dp_kparts(int r) { return r <= 2 ? 8 : (r == 3 ? 4 : (r == 4 ? 2 : 1)); }
__host__ __device__ __forceinline__ int dp_g1(int maxL) { return maxL > 1 ? (maxL - 1 + DP_R1 - 1) / DP_R1 : 1; }

// per-instance counters (ints): [0] queue head (instance 0 only),
// slice[i] at 4 + i (i = 1..V), exp1[j] at 5 + V + j, expb[j] at 5 + 2V + j
struct DpCnt {
    int* c;
    int V;
    __device__ __forceinline__ int* slice(int i) const { return c + 4 + i; }
    __device__ __forceinline__ int* exp1(int j) const { return c + 5 + V + j; }
    __device__ __forceinline__ int* expb(int j) const { return c + 5 + 2 * V + j; }
};
__device__ __forceinline__ DpCnt dp_counters(const pp_batch& b, const pp_instance& I) {
    return DpCnt{reinterpret_cast<int*>(b.ws + I.ws_off + ws_layout(I.L, I.V).dpc), I.V};
}

// Optional per-task timeline (tools/dp_trace.py): 4 x u64 per task id —
// (smid << 32 | kind), fetch time, inputs-ready time, end time (globaltimer ns).
__device__ unsigned long long* g_dp_trace = nullptr;
__device__ int g_dp_trace_cap = 0;

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void dp_wait(const int* cnt, int target, unsigned long long* tr = nullptr) {
    if (threadIdx.x == 0) {
        int ns = 32;
        while (ld_acquire(cnt) < target) {
            __nanosleep(ns);
            ns = ns < 256 ? ns * 2 : 256;
        }
        __threadfence();
        if (tr) tr[2] = gtimer();
    }
    __syncthreads();
}

__device__ __forceinline__ void dp_signal(int* cnt, unsigned long long* tr = nullptr, int kind = 0) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(cnt, 1);
        if (tr) { tr[0] |= (unsigned)kind; tr[3] = gtimer(); }
    }
}

__global__ void __launch_bounds__(128) k_dp_reset(pp_batch b) {
    const pp_instance I = b.inst[blockIdx.x];
    int* c = dp_counters(b, I).c;
    for (int k = threadIdx.x; k < 3 * I.V + 6; k += blockDim.x) c[k] = 0;
}

// Preset W(l, xi, r, j+r) = +inf, xi in [2, j+1], for the split-K items r in
// [r0, r1] and layers [la, lb] (the expand task of those rows does it; the
// combine parts that atomicMin into the cells wait for that task).
__device__ __forceinline__ void dp_preset(const pp_batch& b, const pp_instance& I, int j, int r0, int r1, int la,
                                          int lb) {
    const int L = I.L;
    double* W = b.ws + I.ws_off + ws_layout(L, I.V).W;
    r1 = min(r1, I.V - j);
    if (lb == L - 1) lb = L;   // the task holding the last expand row also takes layer L
    const int nl = lb - la + 1, nr = r1 - r0 + 1;
    if (nl <= 0 || nr <= 0) return;
    for (int e = threadIdx.x; e < nl * nr * j; e += blockDim.x) {
        const int xi = 2 + e % j, q = e / j;
        const int r = r0 + q % nr, l = la + q / nr;
        W[W_idx(L, j + r, l, r, xi)] = PP_INF;
    }
}

// X(l', xi, 1, j+1) = min_{r' <= j-xi+2} max(W_j(l', xi-1, r'), chan(l', r', 1, j+1))
// (partition.py:130-138) for rows l' in [la, lb]: one warp per row, lanes over
// xi, chan(l', r') held by lane (r'-1) % 32 and broadcast by shuffle.
__device__ void expand_r1(const pp_batch& b, const pp_instance& I, int j, int la, int lb, double* chs) {
    const int L = I.L, V = I.V, M = I.M;
    const bool allow = I.flags & PP_ALLOW_REPLICATION;
    const WsLayout lay = ws_layout(L, V);
    double* ws = b.ws + I.ws_off;
    const double* cross = ws + lay.cross;
    double* Xg = ws + lay.X + X_base(L, j + 1, 1);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    constexpr int S = DP_MAXJ / 32, U = 4;
    double* ch = chs + warp * V;   // chan(l', r') of this warp's row, by r' (j < V)
    for (int lp = la + warp; lp <= lb; lp += nw) {
        const double Mp = (double)M * (b.efwd[I.layer_off + lp - 1] + b.ebwd[I.layer_off + lp - 1]);
        const double* Wsrc = ws + lay.W + W_idx(L, j, lp, 1, 1);   // [r'-1][xi'-1], stride j
        const int cls = reinterpret_cast<const int*>(ws + lay.chcls + CHAN_CLS)[lp];
        const double* Tj = ws + lay.chan + (int64_t)max(cls, 0) * tet(V) + chan_step(V, j);
        for (int rp = 1 + lane; rp <= j; rp += 32)   // the class table holds the same quotient
            ch[rp - 1] = cls >= 0 ? Tj[(rp - 1) * (V - j)] : Mp / ((double)(rp * 1) * cross[cross_idx(V, j + 1, 1, rp)]);
        __syncwarp();
        double acc[S];
#pragma unroll
        for (int s = 0; s < S; ++s) acc[s] = PP_INF;
        for (int r0 = 1; r0 <= j; r0 += U) {
            double a[U][S];   // U rows of loads in flight before any use
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int rp = r0 + u;
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    const int xi = 2 + lane + 32 * s;   // reads W_j(l', xi - 1, r')
                    const bool ok = rp <= j && xi <= j + 1 && rp <= j - xi + 2 && W_structural(j, rp, xi - 1, allow);
                    a[u][s] = ok ? Wsrc[(int64_t)(rp - 1) * j + (xi - 2)] : PP_INF;
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const double c = r0 + u <= j ? ch[r0 + u - 1] : PP_INF;
#pragma unroll
                for (int s = 0; s < S; ++s) acc[s] = dmin(acc[s], dmax(a[u][s], c));
            }
        }
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int xi = 2 + lane + 32 * s;
            if (xi <= j + 1) Xg[(int64_t)(lp - 1) * j + (xi - 2)] = acc[s];
        }
        __syncwarp();
    }
}

struct DpSched {
    int n_inst, maxL, maxV, total;
    int g1;                    // critical-expand tasks per instance and step
    int gstart[DP_MAXJ + 1];   // first task of step group j (1..maxV-1), gstart[maxV] = total
    int need[DP_MAXJ + 1];     // slice i complete when its counter reaches need[i]
};

// items r = 2..nr of one step, DP_kparts(r) parts each, instances innermost:
// index o -> (r, part, instance)
__device__ __forceinline__ void dp_cb_decode(int o, int n_inst, int& r, int& p, int& n) {
    r = 2;
    while (r <= DP_RSPLIT && o >= n_inst * dp_kparts(r)) { o -= n_inst * dp_kparts(r); ++r; }
    if (r > DP_RSPLIT) { r += o / n_inst; o %= n_inst; }
    n = o % n_inst;
    p = o / n_inst;
}
__device__ __forceinline__ int dp_cb_count(int n_inst, int nitems) {   // items r = 2..nitems+1
    int c = 0;
    for (int r = 2; r <= nitems + 1; ++r) c += n_inst * dp_kparts(r);
    return c;
}

__device__ __forceinline__ int dp_neb(int maxL, int maxV, int j) {
    const int rows = dp_rows_per_task(j);
    return maxV - j >= 2 ? (maxL - 1 + rows - 1) / rows : 0;
}

__device__ void dp_sched_build(DpSched& s, int n_inst, int maxL, int maxV) {
    s.n_inst = n_inst; s.maxL = maxL; s.maxV = maxV;
    s.g1 = dp_g1(maxL);
    int o = 0;
    for (int j = 1; j < maxV; ++j) {
        s.gstart[j] = o;
        o += n_inst * s.g1;                                          // E1(j)
        o += n_inst * dp_neb(maxL, maxV, j);                         // Eb(j)
        o += n_inst * dp_kparts(1);                                  // C1(j)
        if (j >= 2) o += dp_cb_count(n_inst, maxV - j);              // Cb(j-1), r = 2..
    }
    s.gstart[maxV] = o;
    s.total = o;
    for (int i = 1; i <= maxV; ++i) {
        int nd = 0;
        for (int r = 1; r <= i - 1; ++r) nd += dp_kparts(r);
        s.need[i] = nd;
    }
}

__global__ void __launch_bounds__(DP_T, 2) k_dp_persist(pp_batch b) {
    extern __shared__ __align__(16) double dp_smem[];
    __shared__ DpSched sch;
    __shared__ int s_hist[SR_MAX + 2];
    __shared__ int s_order[1024];
    __shared__ int s_task;
    const int t = threadIdx.x;
    if (t == 0) dp_sched_build(sch, b.n_inst, b.max_L, b.max_V);
    int* head = dp_counters(b, b.inst[0]).c;   // batch-wide queue head: instance 0's counter 0
    __syncthreads();
    const int n_inst = sch.n_inst, maxL = sch.maxL, maxV = sch.maxV;
    for (;;) {
        if (t == 0) s_task = atomicAdd(head, 1);
        __syncthreads();
        const int task = s_task;
        __syncthreads();
        if (task >= sch.total) break;
        unsigned long long* tr = (g_dp_trace && task < g_dp_trace_cap) ? g_dp_trace + 4 * (int64_t)task : nullptr;
        if (tr && t == 0) { unsigned smid; asm("mov.u32 %0, %smid;" : "=r"(smid)); tr[0] = (unsigned long long)smid << 32; tr[1] = gtimer(); tr[2] = 0; }
        int j = 1;
        while (sch.gstart[j + 1] <= task) ++j;
        int o = task - sch.gstart[j];
        // Tasks of an instance smaller than the batch maxima that have no work are
        // skipped, and signal only where a real task of that instance waits.
        const int g1 = sch.g1;
        if (o < n_inst * g1) {   // ---- E1(n, j, g): rows g*8+1 .. g*8+8
            const int n = o % n_inst, g = o / n_inst;
            const pp_instance I = b.inst[n];
            if (j < I.V) {
                const DpCnt c = dp_counters(b, I);
                const int la = 1 + g * DP_R1, lb = min(I.L - 1, (g + 1) * DP_R1);
                if (I.L == 1 && g == 0) dp_preset(b, I, j, 1, 1, 1, 1);
                if (la <= lb) {
                    dp_preset(b, I, j, 1, 1, la, lb);
                    dp_wait(c.slice(j), sch.need[j], tr);
                    expand_r1(b, I, j, la, lb, dp_smem);
                }
                dp_signal(c.exp1(j), tr, 1);
            }
            continue;
        }
        o -= n_inst * g1;
        const int rows = dp_rows_per_task(j);
        const int nEb = dp_neb(maxL, maxV, j);
        if (o < n_inst * nEb) {   // ---- Eb(n, j, row group): targets r = 2..V-j
            const int n = o % n_inst, g = o / n_inst;
            const pp_instance I = b.inst[n];
            if (j <= I.V - 2) {   // else no Cb of (n, j) exists to wait for it
                const DpCnt c = dp_counters(b, I);
                if (I.L == 1 && g == 0) dp_preset(b, I, j, 2, DP_RSPLIT, 1, 1);
                if (1 + g * rows < I.L) {
                    const int l1 = min(I.L - 1, (g + 1) * rows);
                    dp_preset(b, I, j, 2, DP_RSPLIT, 1 + g * rows, l1);
                    dp_wait(c.slice(j), sch.need[j], tr);
                    for (int lp = 1 + g * rows; lp <= l1; ++lp) {
                        expand_row_s(b, I, j, lp, 2, dp_smem);
                        __syncthreads();
                    }
                }
                dp_signal(c.expb(j), tr, 2);   // every row group of the batch maxima signals
            }
            continue;
        }
        o -= n_inst * nEb;
        const int P1 = dp_kparts(1);
        if (o < n_inst * P1) {   // ---- C1(n, j, p): critical combine, l' chunk p
            const int n = o % n_inst, p = o / n_inst;
            const pp_instance I = b.inst[n];
            if (j < I.V) {
                const DpCnt c = dp_counters(b, I);
                dp_wait(c.exp1(j), g1, tr);
                const int per = (maxL - 1 + P1 - 1) / P1;
                const int la = 1 + p * per, lb = (p + 1) * per;
                if (la <= I.L - 1)
                    combine_item_s(b, I, j, 1, 0, 1, dp_smem, s_hist, s_order, false, la, lb, true);
                dp_signal(c.slice(j + 1), tr, 3);
            }
            continue;
        }
        o -= n_inst * P1;
        {   // ---- Cb(n, j-1, r, p)
            const int jb = j - 1;
            int r, p, n;
            dp_cb_decode(o, n_inst, r, p, n);
            const pp_instance I = b.inst[n];
            if (jb < I.V && r <= I.V - jb) {
                const DpCnt c = dp_counters(b, I);
                dp_wait(c.expb(jb), dp_neb(maxL, maxV, jb), tr);
                const int P = dp_kparts(r);
                if (P == 1) {
                    combine_item_s(b, I, jb, r, 0, 1, dp_smem, s_hist, s_order, false);
                } else {
                    const int per = (maxL - 1 + P - 1) / P;
                    const int la = 1 + p * per, lb = (p + 1) * per;
                    if (la <= I.L - 1)
                        combine_item_s(b, I, jb, r, 0, 1, dp_smem, s_hist, s_order, false, la, lb, true);
                }
                dp_signal(c.slice(jb + r), tr, 4);
            }
        }
    }
}

}  // namespace pp

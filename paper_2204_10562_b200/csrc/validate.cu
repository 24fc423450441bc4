// validate.cu — validate_schedule (scheduler.py:303-452) as a batched device
// checker.  The host maps label / resource strings to expected indices and
// formats the messages; every comparison runs here, with the reference's
// tolerance 1e-9 * max(1, |v|...) (scheduler.py:299-300) evaluated in the
// same order.  See include/pipeplan_b200.h for the output encoding.
#include <climits>

#include "common.cuh"

namespace pp {

__device__ __forceinline__ double vtol1(double a) { return 1e-9 * dmax(1.0, fabs(a)); }
__device__ __forceinline__ double vtol2(double a, double b) { return 1e-9 * dmax(dmax(1.0, fabs(a)), fabs(b)); }
__device__ __forceinline__ double vtol3(double a, double b, double c) {
    return 1e-9 * dmax(dmax(dmax(1.0, fabs(a)), fabs(b)), fabs(c));
}

struct ValLayout {   // expected-index arithmetic (scheduler.py:322-338)
    int N, S;        // S = number of stage entries (2N, or 2N-1 when merged)
    bool merged;
    __device__ ValLayout(const pp_validate_args& a)
        : N(a.N), S(2 * a.N - ((a.flags & PP_VAL_MERGED_LAST) ? 1 : 0)), merged(a.flags & PP_VAL_MERGED_LAST) {}
    __device__ int fwd(int n) const { return 2 * (n - 1); }                      // fwd n (or fwdbwd N)
    __device__ int bwd(int n) const { return (merged && n == N) ? 2 * (N - 1) : 2 * (n - 1) + 1; }
    __device__ int cf(int n) const { return S + 2 * (n - 1); }
    __device__ int cb(int n) const { return S + 2 * (n - 1) + 1; }
    // expected duration of index e from the plan's lane records
    __device__ double dur(const double* lc, int e) const {
        if (e < S) {
            const int n = e / 2 + 1;
            const double* r = lc + (int64_t)(2 * (n - 1)) * PP_LANE_COST_FIELDS;
            if (merged && n == N) return r[0];   // FB = stage_compute_time / k
            return (e & 1) ? r[5] : r[4];        // split B / F
        }
        const int n = (e - S) / 2 + 1;
        const double* r = lc + (int64_t)(2 * n - 1) * PP_LANE_COST_FIELDS;
        return ((e - S) & 1) ? r[1] : r[0];
    }
};

__global__ void k_val_init(pp_validate_args a) {
    const int64_t n_slot = (int64_t)a.M * a.n_exp;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n_slot; x += (int64_t)gridDim.x * blockDim.x) {
        a.slot_first[x] = INT_MAX;
        a.slot_last[x] = -1;
        a.slot_count[x] = 0;
    }
}

// phase 1a: slot occupancy (by_key, scheduler.py:316-323) and per-event checks
__global__ void k_val_events(pp_validate_args a) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < a.n_ev; k += (int64_t)gridDim.x * blockDim.x) {
        const int m = a.ev_m[k], e = a.ev_e[k];
        const double s = a.ev_start[k], t = a.ev_end[k];
        uint8_t f = 0;
        if (t < s - vtol2(s, t)) f |= 2;                      // :321-322
        if (e < 0) f |= 4;                                    // :341-342
        else if (m < 1 || m > a.M) f |= 8;                    // :343-344
        else {
            const int64_t x = (int64_t)(m - 1) * a.n_exp + e;
            atomicMin(a.slot_first + x, (int)k);
            atomicMax(a.slot_last + x, (int)k);
            atomicAdd(a.slot_count + x, 1);
        }
        a.ev_flags[k] = f;
    }
}

// phase 1b: duplicates (every event after a slot's first) and the
// missing / resource / duration checks per (m, expected index) (:345-355)
__global__ void k_val_slots(pp_validate_args a) {
    const ValLayout V(a);
    const int64_t n_slot = (int64_t)a.M * a.n_exp;
    const int64_t total = n_slot > a.n_ev ? n_slot : a.n_ev;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
        if (x < a.n_ev) {
            const int m = a.ev_m[x], e = a.ev_e[x];
            if (e >= 0 && m >= 1 && m <= a.M && a.slot_first[(int64_t)(m - 1) * a.n_exp + e] != (int)x)
                a.ev_flags[x] |= 1;
        }
        if (x < n_slot) {
            uint8_t f = 0;
            if (a.slot_count[x] == 0) f = 1;
            else {
                const int k = a.slot_last[x];
                if (!a.ev_res_ok[k]) f |= 2;
                const double d = V.dur(a.lane_cost, (int)(x % a.n_exp));
                const double s = a.ev_start[k], t = a.ev_end[k];
                if (fabs((t - s) - d) > vtol3(d, t, s)) f |= 4;
            }
            a.slot_flags[x] = f;
        }
    }
}

// phase 2a: per-microbatch ordering checks (:376-393) and partials for the
// barrier / AllReduce-ready / makespan reductions.
__global__ void k_val_order(pp_validate_args a) {
    const ValLayout V(a);
    const int N = a.N, M = a.M;
    const int m = blockIdx.x * blockDim.x + threadIdx.x + 1;
    if (m > M) return;
    const int* last = a.slot_last + (int64_t)(m - 1) * a.n_exp;
    auto S_ = [&](int e) { return a.ev_start[last[e]]; };
    auto E_ = [&](int e) { return a.ev_end[last[e]]; };
    double fmax = -PP_INF, bmin = PP_INF;
    for (int n = 1; n < N; ++n) {
        const double* rc = a.lane_cost + (int64_t)(2 * n - 1) * PP_LANE_COST_FIELDS;
        const double cf = rc[0], cb = rc[1];
        const double fe = E_(V.fwd(n)), fs1 = S_(V.fwd(n + 1));
        const double xs = S_(V.cf(n)), xe = E_(V.cf(n));
        const double be1 = E_(V.bwd(n + 1)), bs = S_(V.bwd(n));
        const double ys = S_(V.cb(n)), ye = E_(V.cb(n));
        uint8_t f = 0;
        if (fs1 < fe + cf - vtol2(fe, cf)) f |= 1;
        if (xs < fe - vtol1(fe)) f |= 2;
        if (fs1 < xe - vtol1(xe)) f |= 4;
        if (bs < be1 + cb - vtol2(be1, cb)) f |= 8;
        if (ys < be1 - vtol1(be1)) f |= 16;
        if (bs < ye - vtol1(ye)) f |= 32;
        a.mn_flags[(int64_t)(m - 1) * N + n - 1] = f;
        fmax = dmax(fmax, dmax(fe, xe));
        bmin = dmin(bmin, dmin(bs, ys));
    }
    uint8_t fl = 0;
    if (!V.merged) {
        const double fe = E_(V.fwd(N));
        if (S_(V.bwd(N)) < fe - vtol1(fe)) fl = 64;
    }
    a.mn_flags[(int64_t)(m - 1) * N + N - 1] = fl;
    bmin = dmin(bmin, dmin(S_(V.bwd(N)), S_(V.fwd(N))));   // b_start(m, N), f_start(m, N)
    a.part[m - 1] = fmax;
    a.part[M + m - 1] = bmin;
    a.part[2 * M + m - 1] = E_(V.bwd(1));                  // completion candidate b_end(m, 1)
}

// phase 2b (one CTA): reductions, first-start, AllReduce windows, barrier, makespan
__global__ void __launch_bounds__(256) k_val_final(pp_validate_args a) {
    const ValLayout V(a);
    const int N = a.N, M = a.M, t = threadIdx.x;
    __shared__ double r0[256], r1[256], r2[256];
    double fmax = -PP_INF, bmin = PP_INF, comp = -PP_INF;
    for (int m = t; m < M; m += blockDim.x) {
        fmax = dmax(fmax, a.part[m]);
        bmin = dmin(bmin, a.part[M + m]);
        comp = dmax(comp, a.part[2 * M + m]);
    }
    r0[t] = fmax; r1[t] = bmin; r2[t] = comp;
    __syncthreads();
    // AllReduce checks, one stage per thread (:395-407): ready = max_m b_end(m, s)
    for (int n = 1 + t; n <= N; n += blockDim.x) {
        const double* rs = a.lane_cost + (int64_t)(2 * (n - 1)) * PP_LANE_COST_FIELDS;
        const bool repl = rs[6] != PP_INF;   // min pairwise bandwidth is finite iff k >= 2
        uint8_t f = 0;
        if (repl) {
            if (!a.win_has[n - 1]) f = 1;
            else {
                double ready = -PP_INF;
                for (int m = 1; m <= M; ++m)
                    ready = dmax(ready, a.ev_end[a.slot_last[(int64_t)(m - 1) * a.n_exp + V.bwd(n)]]);
                if (a.win_start[n - 1] < ready - vtol1(ready)) f |= 2;
                const double ar = rs[3];
                if (fabs((a.win_end[n - 1] - a.win_start[n - 1]) - ar) > vtol1(ar)) f |= 4;
            }
        } else if (a.win_has[n - 1]) f = 8;
        a.ar_flags[n - 1] = f;
    }
    if (t != 0) return;
    for (int k = 1; k < (int)blockDim.x; ++k) {
        fmax = dmax(fmax, r0[k]); bmin = dmin(bmin, r1[k]); comp = dmax(comp, r2[k]);
    }
    const double f11 = a.ev_start[a.slot_last[V.fwd(1)]];
    a.stat[0] = fabs(f11) > vtol1(f11);                                        // :372-373
    a.stat[1] = (a.flags & PP_VAL_FORWARD_BARRIER) && N > 1 && bmin < fmax - vtol1(fmax);   // :420-431
    double exp_mk = comp;
    for (int w = 0; w < a.n_win_all; ++w) exp_mk = dmax(exp_mk, a.win_all_end[w]);
    a.stat[2] = fabs(a.makespan - exp_mk) > vtol1(exp_mk);                   // :433-437
    a.scal[0] = exp_mk; a.scal[1] = fmax; a.scal[2] = bmin; a.scal[3] = f11;
}

// phase 2c: per-resource overlap check (:409-417): one CTA per resource lane,
// its events bitonic-sorted by (start, end, event index) in shared memory.
constexpr int VAL_SORT_MAX = 8192;
__global__ void __launch_bounds__(1024) k_val_overlap(pp_validate_args a) {
    const ValLayout V(a);
    const int lane = blockIdx.x, N = a.N, M = a.M;
    const int n = lane / 2 + 1;
    int es[2], ne = 0;
    if ((lane & 1) == 0) {
        es[ne++] = V.fwd(n);
        if (!(V.merged && n == N)) es[ne++] = V.bwd(n);
    } else { es[ne++] = V.cf(n); es[ne++] = V.cb(n); }
    const int cnt = ne * M;
    int P2 = 1;
    while (P2 < cnt) P2 <<= 1;
    extern __shared__ double vsm[];
    double* ks = vsm;              // start
    double* ke = vsm + P2;         // end
    int* ki = (int*)(vsm + 2 * P2);
    for (int j = threadIdx.x; j < P2; j += blockDim.x) {
        if (j < cnt) {
            const int e = es[j / M], m = j % M + 1;
            const int k = a.slot_last[(int64_t)(m - 1) * a.n_exp + e];
            ks[j] = a.ev_start[k]; ke[j] = a.ev_end[k]; ki[j] = k;
        } else { ks[j] = PP_INF; ke[j] = PP_INF; ki[j] = INT_MAX; }
    }
    __syncthreads();
    for (int size = 2; size <= P2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int j = threadIdx.x; j < P2; j += blockDim.x) {
                const int p = j ^ stride;
                if (p > j) {
                    const bool up = (j & size) == 0;
                    const bool gt = ks[j] > ks[p] || (ks[j] == ks[p] && (ke[j] > ke[p] || (ke[j] == ke[p] && ki[j] > ki[p])));
                    if (gt == up) {
                        double t = ks[j]; ks[j] = ks[p]; ks[p] = t;
                        t = ke[j]; ke[j] = ke[p]; ke[p] = t;
                        const int u = ki[j]; ki[j] = ki[p]; ki[p] = u;
                    }
                }
            }
            __syncthreads();
        }
    }
    const int64_t off = a.res_off[lane];
    for (int j = threadIdx.x; j < cnt; j += blockDim.x) {
        a.ov_idx[off + j] = ki[j];
        a.ov_flags[off + j] = (j > 0 && ks[j] < ke[j - 1] - vtol1(ke[j - 1])) ? 1 : 0;
    }
}

// Large-M overlap check (2M > VAL_SORT_MAX): the same (start, end, event index)
// order, bitonic-sorted in global scratch, one launch per (size, stride) pass
// over all lanes at once; then the neighbour check.
__global__ void k_val_ov_fill(pp_validate_args a) {
    const ValLayout V(a);
    const int lane = blockIdx.y, N = a.N, M = a.M;
    const int n = lane / 2 + 1;
    int es[2], ne = 0;
    if ((lane & 1) == 0) {
        es[ne++] = V.fwd(n);
        if (!(V.merged && n == N)) es[ne++] = V.bwd(n);
    } else { es[ne++] = V.cf(n); es[ne++] = V.cb(n); }
    const int64_t cnt = (int64_t)ne * M, P2 = a.sort_cap, base = (int64_t)lane * P2;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < P2; j += (int64_t)gridDim.x * blockDim.x) {
        if (j < cnt) {
            const int e = es[j / M], m = (int)(j % M) + 1;
            const int k = a.slot_last[(int64_t)(m - 1) * a.n_exp + e];
            a.sort_ks[base + j] = a.ev_start[k]; a.sort_ke[base + j] = a.ev_end[k]; a.sort_ki[base + j] = k;
        } else { a.sort_ks[base + j] = PP_INF; a.sort_ke[base + j] = PP_INF; a.sort_ki[base + j] = INT_MAX; }
    }
}
__global__ void k_val_ov_pass(pp_validate_args a, int64_t size, int64_t stride) {
    const int64_t P2 = a.sort_cap, base = (int64_t)blockIdx.y * P2;
    double* ks = a.sort_ks + base;
    double* ke = a.sort_ke + base;
    int32_t* ki = a.sort_ki + base;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < P2; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = j ^ stride;
        if (p > j) {
            const bool up = (j & size) == 0;
            const bool gt = ks[j] > ks[p] || (ks[j] == ks[p] && (ke[j] > ke[p] || (ke[j] == ke[p] && ki[j] > ki[p])));
            if (gt == up) {
                double t = ks[j]; ks[j] = ks[p]; ks[p] = t;
                t = ke[j]; ke[j] = ke[p]; ke[p] = t;
                const int32_t u = ki[j]; ki[j] = ki[p]; ki[p] = u;
            }
        }
    }
}
__global__ void k_val_ov_check(pp_validate_args a) {
    const int lane = blockIdx.y, N = a.N, M = a.M;
    const int ne = ((lane & 1) == 0 && a.flags & 1 && lane / 2 + 1 == N) ? 1 : 2;
    const int64_t cnt = (int64_t)ne * M, base = (int64_t)lane * a.sort_cap, off = a.res_off[lane];
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < cnt; j += (int64_t)gridDim.x * blockDim.x) {
        a.ov_idx[off + j] = a.sort_ki[base + j];
        a.ov_flags[off + j] = (j > 0 && a.sort_ks[base + j] < a.sort_ke[base + j - 1] - vtol1(a.sort_ke[base + j - 1]))
                                  ? 1 : 0;
    }
}

}  // namespace pp

extern "C" int pp_validate_schedule(const pp_validate_args* a, int32_t phase, void* stream) {
    using namespace pp;
    if (a->N < 1 || a->M < 1 || a->N > PP_MAX_GPUS) return fail(PP_EINVAL, "validate: N=%d M=%d", a->N, a->M);
    const int64_t n_slot = (int64_t)a->M * a->n_exp;
    const int sms = num_sms();
    cudaStream_t st = (cudaStream_t)stream;
    if (phase == 1) {
        const int64_t work = n_slot > a->n_ev ? n_slot : a->n_ev;
        const int grid = (int)std::min<int64_t>((work + 255) / 256, (int64_t)sms * 8) + 1;
        k_val_init<<<grid, 256, 0, st>>>(*a);
        PP_CHECK_LAUNCH("k_val_init");
        if (a->n_ev > 0) {
            k_val_events<<<grid, 256, 0, st>>>(*a);
            PP_CHECK_LAUNCH("k_val_events");
        }
        k_val_slots<<<grid, 256, 0, st>>>(*a);
        PP_CHECK_LAUNCH("k_val_slots");
        return PP_OK;
    }
    int64_t P2g = 1;
    while (P2g < 2 * (int64_t)a->M) P2g <<= 1;
    if (2 * a->M > VAL_SORT_MAX && (!a->sort_ks || !a->sort_ke || !a->sort_ki || a->sort_cap < P2g))
        return fail(PP_EINVAL, "validate: %d events per resource need sort scratch of %lld keys per lane", 2 * a->M,
                    (long long)P2g);
    k_val_order<<<(a->M + 127) / 128, 128, 0, st>>>(*a);
    PP_CHECK_LAUNCH("k_val_order");
    k_val_final<<<1, 256, 0, st>>>(*a);
    PP_CHECK_LAUNCH("k_val_final");
    if (2 * a->M > VAL_SORT_MAX) {
        const dim3 g((unsigned)std::min<int64_t>((a->sort_cap + 255) / 256, 1024), 2 * a->N - 1);
        k_val_ov_fill<<<g, 256, 0, st>>>(*a);
        PP_CHECK_LAUNCH("k_val_ov_fill");
        for (int64_t size = 2; size <= a->sort_cap; size <<= 1)
            for (int64_t stride = size >> 1; stride > 0; stride >>= 1) {
                k_val_ov_pass<<<g, 256, 0, st>>>(*a, size, stride);
                PP_CHECK_LAUNCH("k_val_ov_pass");
            }
        k_val_ov_check<<<g, 256, 0, st>>>(*a);
        PP_CHECK_LAUNCH("k_val_ov_check");
        return PP_OK;
    }
    int P2 = 1;
    while (P2 < 2 * a->M) P2 <<= 1;
    const size_t smem = (size_t)P2 * (2 * sizeof(double) + sizeof(int));
    cudaFuncSetAttribute(k_val_overlap, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_val_overlap<<<2 * a->N - 1, 1024, smem, st>>>(*a);
    PP_CHECK_LAUNCH("k_val_overlap");
    return PP_OK;
}

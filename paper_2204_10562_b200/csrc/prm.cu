// prm.cu — DP tables and the PRM dynamic program.
//
// Reference: partition.py:41-162
// (W(l, xi, r, i) recursion), cost.py:64-99 (bandwidth minima, AllReduce).
//
// The DP runs as a wavefront over the device prefix i (W(., ., ., i) needs
// only slices j < i, partition.py:133).  The reference's candidate
//     w(l', r') = max(W(l', xi-1, r', j), chan(l', r'), stage(l'))
// is evaluated in factored form (bit-exact: max/min are exact and monotone):
//   expand(j):  X(l', xi, r, j+r) = min_{r'} max(W_j(l', xi-1, r'), chan(l', r', r, j+r))
//   combine(i): W_i(l, r, xi)     = min_{l'} max(X(l', xi, r, i), stage(l', l, r, i))
// Both are (min, max)-semiring matrix products computed with register
// micro-tiles from shared-memory operand chunks.  Schedule ("diagonal"): step j
// runs expand(j) and then combine for every target (r, j + r) — after step j
// slice j + 1 is complete.  Arg-mins are not stored: the backtrack re-derives
// the reference's first-found (l', r') for the few cells on each chosen path.
#include "common.cuh"

namespace pp {

// W(l, xi, r, i) with the structural +inf rules of partition.py:103-121 applied
// by index (those cells are never materialised by the shared-memory path):
// base cells (r = i) hold a value only at xi = 1; other cells need
// 2 <= xi <= i - r + 1; without replication only r = 1 (or the 1-GPU base).
__device__ __forceinline__ bool W_structural(int i, int r, int xi, bool allow) {
    if (r == i) return xi == 1 && (allow || i == 1);
    return xi >= 2 && xi <= i - r + 1 && (allow || r == 1);
}
__device__ __forceinline__ double W_at(const double* W, int L, int i, int l, int r, int xi, bool allow) {
    return W_structural(i, r, xi, allow) ? W[W_idx(L, i, l, r, xi)] : PP_INF;
}

// ----------------------------------------------------------------------------
// k_prep: per instance tables (partition.py:59-93, cost.py:64-99, cost.py:126-142)
//   prefix[l] = (prefix[l-1] + fwd_l) + bwd_l                     partition.py:62
//   psum[ls][le] = sum(param[ls..le])  (CPython sum)              cost.py:98
//   minpair[lo][hi] = min pairwise bw over order[lo..hi]          cost.py:64-71
//   cross(rp, r, i) = min bw between order[i-r-rp+1..i-r] and order[i-r+1..i]
//                                                                  partition.py:82-93
// grid (n_inst, max(maxL, maxV)); row y handles psum row ls=y+1, minpair row
// lo=y+1 and the cross table of i=y+1.  Row 0 also computes prefix and phi.
// ----------------------------------------------------------------------------
constexpr int PREP_CM_MAX = 64;   // cross table via shared column minima up to this i
__device__ __forceinline__ void prep_body(const pp_batch& b) {
    const pp_instance I = b.inst[blockIdx.x];
    const int L = I.L, V = I.V;
    const bool naive = I.flags & PP_SUM_NAIVE;
    const WsLayout lay = ws_layout(L, V);
    double* ws = b.ws + I.ws_off;
    const double* fwd = b.fwd + I.layer_off;
    const double* bwd = b.bwd + I.layer_off;
    const double* par = b.param + I.layer_off;
    const double* bw = b.bw + I.bw_off;
    const int* order = b.order + I.order_off;
    const int row = blockIdx.y + 1;
    const int t = threadIdx.x;

    if (row == 1 && t == 0) {
        double p = 0.0;
        ws[lay.prefix] = 0.0;
        for (int l = 1; l <= L; ++l) {
            p = p + fwd[l - 1] + bwd[l - 1];
            ws[lay.prefix + l] = p;
        }
        if (L <= SR_MAX && V <= SR_MAX) {   // chan payload classes (bitwise-equal M * (efwd + ebwd))
            double* cv = ws + lay.chcls;
            int* ci = reinterpret_cast<int*>(cv + CHAN_CLS);
            int ncls = 0;
            for (int lp = 1; lp < L; ++lp) {
                const double Mp = (double)I.M * (b.efwd[I.layer_off + lp - 1] + b.ebwd[I.layer_off + lp - 1]);
                int c = -1;
                for (int k = 0; k < ncls; ++k)
                    if (__double_as_longlong(cv[k]) == __double_as_longlong(Mp)) { c = k; break; }
                if (c < 0 && ncls < CHAN_CLS) { cv[ncls] = Mp; c = ncls++; }
                ci[1 + lp - 1] = c;
            }
            // a table only pays off when rows share it: drop single-row classes
            int cnt[CHAN_CLS] = {0, 0, 0, 0}, remap[CHAN_CLS], nk = 0;
            for (int lp = 1; lp < L; ++lp) if (ci[lp] >= 0) ++cnt[ci[lp]];
            for (int k = 0; k < ncls; ++k) {
                remap[k] = cnt[k] >= 2 ? nk : -1;
                if (cnt[k] >= 2) cv[nk++] = cv[k];
            }
            for (int lp = 1; lp < L; ++lp) if (ci[lp] >= 0) ci[lp] = remap[ci[lp]];
            ci[0] = nk;
        }
    }
    // psum row ls = row: running CPython sum over le = ls..L
    if (row <= L && t == 0) {
        PySum s(naive);
        for (int le = row; le <= L; ++le) {
            s.add(par[le - 1]);
            ws[lay.psum + (int64_t)(row - 1) * L + (le - 1)] = s.value();
        }
    }
    if (row > V) return;
    // minpair row lo = row: colmin(hi) = min_{a in [lo, hi-1]} bw(order a, order hi); prefix-min over hi
    __shared__ double s_col[PP_MAX_GPUS];
    for (int hi = row + 1 + t; hi <= V; hi += blockDim.x) {
        double m = PP_INF;
        const double* bwr = bw + (int64_t)order[hi - 1] * V;
        for (int a = row; a < hi; ++a) m = dmin(m, bwr[order[a - 1]]);
        s_col[hi - 1] = m;
    }
    __syncthreads();
    if (t == 0) {
        double m = PP_INF;
        ws[lay.minpair + (int64_t)(row - 1) * V + (row - 1)] = m;
        for (int hi = row + 1; hi <= V; ++hi) {
            m = dmin(m, s_col[hi - 1]);
            ws[lay.minpair + (int64_t)(row - 1) * V + (hi - 1)] = m;
        }
    }
    // cross table for i = row
    const int i = row;
    if (b.max_V <= PREP_CM_MAX) {
        // cm_r(x) = min bandwidth from rank x to the last r ranks (..i): thread per
        // x, incremental in r; then cross(rp, r, i) = min over x in [i-r-rp+1, i-r]
        // of cm_r(x): thread per r, incremental in rp.  Exact minima over the same
        // pairs as the direct loop below.
        extern __shared__ double s_cm[];   // [r-1][x-1], stride max_V (dynamic: max_V^2 doubles)
        const int CM = b.max_V;
        for (int x = 1 + t; x < i; x += blockDim.x) {
            const double* bwr = bw + (int64_t)order[x - 1] * V;
            double m = PP_INF;
            for (int r = 1; r <= i - x; ++r) {
                m = dmin(m, bwr[order[i - r]]);   // rank i - r + 1
                s_cm[(r - 1) * CM + (x - 1)] = m;
            }
        }
        __syncthreads();
        for (int r = 1 + t; r < i; r += blockDim.x) {
            double m = PP_INF;
            for (int rp = 1; rp <= i - r; ++rp) {
                m = dmin(m, s_cm[(r - 1) * CM + (i - r - rp)]);   // x = i - r - rp + 1
                ws[lay.cross + cross_idx(V, i, r, rp)] = m;
            }
        }
        return;
    }
    // thread per r in [1, i-1], sequential over rp
    for (int r = 1 + t; r < i; r += blockDim.x) {
        const int lo = i - r + 1;
        double m = PP_INF;
        for (int rp = 1; rp <= i - r; ++rp) {
            const double* bwr = bw + (int64_t)order[lo - 1 - rp] * V;   // new left device, rank lo - rp
            for (int c = lo; c <= i; ++c) m = dmin(m, bwr[order[c - 1]]);
            ws[lay.cross + cross_idx(V, i, r, rp)] = m;
        }
    }
}
__global__ void __launch_bounds__(128) k_prep(pp_batch b) { prep_body(b); }
__global__ void __launch_bounds__(128) k_prep_p(const pp_batch* __restrict__ bp) {
    const pp_batch b = *bp;
    prep_body(b);
}

// phi (cost.py:126-142): max(p_max * b_max, d_max) / Gamma * (1/b_min - 1/b_max),
// 0 on single-GPU or uniform clusters.  One CTA (128 threads) per instance.
__global__ void __launch_bounds__(128) k_phi(pp_batch b) {
    const pp_instance I = b.inst[blockIdx.x];
    const int L = I.L, V = I.V;
    const double* fwd = b.fwd + I.layer_off;
    const double* bwd = b.bwd + I.layer_off;
    const double* bw = b.bw + I.bw_off;
    const int t = threadIdx.x;
    __shared__ double s_red[2][128];
    double mn = PP_INF, mx = -PP_INF;
    for (int e = t; e < V * V; e += blockDim.x) {
        const int a = e / V, c = e % V;
        if (a < c) { const double x = bw[e]; mn = dmin(mn, x); mx = dmax(mx, x); }
    }
    s_red[0][t] = mn; s_red[1][t] = mx;
    __syncthreads();
    if (t != 0) return;
    for (int k = 1; k < blockDim.x; ++k) { mn = dmin(mn, s_red[0][k]); mx = dmax(mx, s_red[1][k]); }
    double pmax = 0.0, dmax = 0.0;
    PySum g(I.flags & PP_SUM_NAIVE);
    for (int l = 0; l < L; ++l) {
        const double tot = fwd[l] + bwd[l];
        g.add(tot);
        if (l == 0 || tot > pmax) pmax = tot;
    }
    for (int e = 0; e < L - 1; ++e) {
        const double d = b.efwd[I.layer_off + e] + b.ebwd[I.layer_off + e];
        if (e == 0 || d > dmax) dmax = d;
    }
    const double gamma = g.value() / (double)V;   // cost.py:128
    double phi = 0.0;
    if (!(V == 1 || mn == mx)) {
        const double num = (dmax > pmax * mx) ? dmax : pmax * mx;
        phi = num / gamma * (1.0 / mn - 1.0 / mx);
    }
    b.phi[blockIdx.x] = phi;
    if (b.gamma) b.gamma[blockIdx.x] = gamma;
}

// ----------------------------------------------------------------------------
// k_base (once, after k_prep): grid (n_inst, max(L, V)), row y.
//   l = y + 1 <= L : the base row of every slice, W_i(l, r = i, xi) for i = 1..V
//                    (partition.py:117-121: xi = 1 -> M*span(1,l)/i + sync(1,l,1,i), else inf)
//   l' = y in [1, L): T1[r][l'][l] = (M * span(l'+1, l)) / r for r = 1..V-1, l > l'
//                    (partition.py:127; the i-independent half of every stage term)
// ----------------------------------------------------------------------------
__device__ __forceinline__ void base_body(const pp_batch& b, int full_rows) {
    const pp_instance I = b.inst[blockIdx.x];
    const int L = I.L, V = I.V, M = I.M;
    const bool allow = I.flags & PP_ALLOW_REPLICATION;
    const WsLayout lay = ws_layout(L, V);
    double* ws = b.ws + I.ws_off;
    const double* prefix = ws + lay.prefix;
    const double* psum = ws + lay.psum;
    const double* minpair = ws + lay.minpair;
    const int y = blockIdx.y, t = threadIdx.x;
    if (y < L) {
        const int l = y + 1;
        // the chunked path (batch-wide choice) reads whole rows: give it explicit +inf cells
        if (full_rows)
            for (int i = 2; i <= V; ++i) {
                double* row = ws + lay.W + W_base(L, i) + ((int64_t)(l - 1) * i + (i - 1)) * i;
                for (int xi = 2 + t; xi <= i; xi += blockDim.x) row[xi - 1] = PP_INF;
            }
        for (int i = 1; i <= V; ++i) {
            double* row = ws + lay.W + W_base(L, i) + ((int64_t)(l - 1) * i + (i - 1)) * i;
            if (t == 0) {   // only xi = 1 is structural; the rest of the row reads as +inf (W_at)
                double v = PP_INF;
                if (allow || i == 1) {
                    double sync = 0.0;
                    if (i > 1) sync = 2.0 * (double)(i - 1) * psum[l - 1] / ((double)i * minpair[i - 1]);
                    v = (double)M * (prefix[l] - prefix[0]) / (double)i + sync;
                }
                row[0] = v;
            }
        }
    }
    if (L <= SR_MAX && V <= SR_MAX && y + 1 < V) {   // chan tables of step j = y + 1, every class
        const int j = y + 1, nr = V - j;
        const double* cv = ws + lay.chcls;
        const int ncls = reinterpret_cast<const int*>(cv + CHAN_CLS)[0];
        const double* cross = ws + lay.cross;
        for (int c = 0; c < ncls; ++c) {
            double* Tj = ws + lay.chan + (int64_t)c * tet(V) + chan_step(V, j);
            const double Mp = cv[c];
            for (int e = t; e < j * nr; e += blockDim.x) {
                const int rp = 1 + e / nr, r = 1 + e % nr;
                Tj[e] = Mp / ((double)(rp * r) * cross[cross_idx(V, j + r, r, rp)]);   // partition.py:131,137
            }
        }
    }
    if (full_rows && y >= 1 && y < L) {   // T1 feeds the chunked path's S tables only
        const int lp = y, w = L - lp;
        double* T1 = ws + lay.T1;
        for (int e = t; e < (V - 1) * w; e += blockDim.x) {
            const int r = 1 + e / w, l = lp + 1 + e % w;
            T1[stage_idx(L, r, lp, l)] = (double)M * (prefix[l] - prefix[lp]) / (double)r;
        }
    }
}
__global__ void __launch_bounds__(128) k_base(pp_batch b, int full_rows) { base_body(b, full_rows); }
__global__ void __launch_bounds__(128) k_base_p(const pp_batch* __restrict__ bp, int full_rows) {
    const pp_batch b = *bp;
    base_body(b, full_rows);
}

// ----------------------------------------------------------------------------
// Stage-term tables for the shared-memory path.  S(l', l, r, i) depends on the
// item (r, i) only through r and mp = minpair(i-r+1, i) (cost.py:99), so items
// whose last-stage slices have bitwise-equal min-pair bandwidth share one
// table.  k_sdedup: one warp per r assigns every (r, i) the slot of the
// first i' with the same mp (sidx; the slot id is that item's triangular index).
// k_stab: the canonical items' packed triangles
//   row l' (1..L-1): S(l', l) = T1(r, l', l) (+ sync if r > 1), l = l'+1..L.
// ----------------------------------------------------------------------------
__device__ __forceinline__ void sdedup_body(const pp_batch& b) {
    // grid (n_inst, ceil((V-1)/8)), 8 warps: warp w owns width r = 8*y + w + 1.
    // Items (r, i) whose last-stage slices have bitwise-equal min-pair bandwidth
    // share a slot; the slot id is the triangular index of the FIRST such i
    // (sparse ids inside the V(V-1)/2 slot budget, so no cross-r prefix).
    const pp_instance I = b.inst[blockIdx.x];
    const int L = I.L, V = I.V;
    if (L > SR_MAX || V > SR_MAX) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r = (int)blockIdx.y * (blockDim.x >> 5) + warp + 1;
    if (r >= V) return;
    const WsLayout lay = ws_layout(L, V);
    double* ws = b.ws + I.ws_off;
    const double* minpair = ws + lay.minpair;
    int* sidx = reinterpret_cast<int*>(ws + lay.sidx);
    __shared__ double s_mp[8][SR_MAX + 1];
    double* mp = s_mp[warp];
    for (int i = r + 1 + lane; i <= V; i += 32) mp[i] = minpair[(int64_t)(i - r) * V + (i - 1)];
    __syncwarp();
    const int base = (r - 1) * (2 * V - r) / 2 - r - 1;   // slot of (r, i) = base + i
    for (int i = r + 1 + lane; i <= V; i += 32) {
        const double m = mp[i];
        int first = i;
        for (int q = r + 1; q < i; ++q)
            if (mp[q] == m) { first = q; break; }
        sidx[(r - 1) * V + (i - 1)] = base + first;
    }
}
__global__ void __launch_bounds__(256) k_sdedup(pp_batch b) { sdedup_body(b); }
__global__ void __launch_bounds__(256) k_sdedup_p(const pp_batch* __restrict__ bp) {
    const pp_batch b = *bp;
    sdedup_body(b);
}

// Triangle of the canonical item (r, i) of its slot:
//   S(l', l) = (M * span(l'+1, l)) / r (+ ((2 (r-1)) * P(l'+1..l)) / (r * minpair))
// (partition.py:127-129, cost.py:99; the same expression as k_base's T1 + sync),
// filled by `nw` warps starting at warp w0 (one warp for small triangles, the
// whole CTA for large ones), plus its monotonicity flag.
__device__ __forceinline__ void stab_fill(const pp_batch& b, const pp_instance& I, int r, int i, int w0, int nw,
                                          int* s_bad) {
    const int L = I.L, V = I.V, M = I.M;
    const WsLayout lay = ws_layout(L, V);
    double* ws = b.ws + I.ws_off;
    const int slot = reinterpret_cast<const int*>(ws + lay.sidx)[(r - 1) * V + (i - 1)];
    const int lane = threadIdx.x & 31, warp = (threadIdx.x >> 5) - w0;
    const int64_t tri = (int64_t)(L - 1) * L / 2;
    double* out = ws + lay.Stab + (int64_t)slot * tri;
    const double* prefix = ws + lay.prefix;
    const double* psum = ws + lay.psum;
    const double den = (double)r * ws[lay.minpair + (int64_t)(i - r) * V + (i - 1)];
    const uint64_t pol = l2_evict_last_policy();   // re-read by the combine of every step
    const double num = 2.0 * (double)(r - 1);
    // both divisors are fixed for the triangle: reciprocals hoisted (div_fixed, '/' bits)
    const double dr = (double)r, yr = div_recip(dr);
    const bool den_ok = div_fixed_ok(den);
    const double yd = den_ok ? div_recip(den) : 0.0;
    for (int lp = 1 + warp; lp < L; lp += nw) {
        const int off = (lp - 1) * L - (lp - 1) * lp / 2;
        const double pl = prefix[lp];
        for (int l = lp + 1 + lane; l <= L; l += 32) {
            double sv = div_fixed((double)M * (prefix[l] - pl), dr, yr, true);
            if (r > 1) sv += div_fixed(num * psum[(int64_t)lp * L + (l - 1)], den, yd, den_ok);
            st_evict_last(out + off + (l - lp - 1), sv, pol);
        }
    }
    // Is the triangle non-increasing in l' (S(l', l) >= S(l'+1, l) for every l;
    // bit 0) and non-decreasing in l (S(l', l) <= S(l', l+1); bit 1)?  In exact
    // arithmetic it is both (the stage loses layers as l' grows and gains them
    // as l grows); the flags certify it for these rounded values.  Bit 0 lets
    // the combine stop scanning l' early and bisect for the crossing; bit 1
    // lets the bisection of cell l start from cell l-1's crossing.
    if (nw == 1) __syncwarp();
    else __syncthreads();
    bool bad = false, bad_l = false;
    for (int lp = 1 + warp; lp < L; lp += nw) {
        const int o0 = (lp - 1) * L - (lp - 1) * lp / 2, o1 = lp * L - lp * (lp + 1) / 2;
        for (int l = lp + 1 + lane; l <= L; l += 32) {
            if (lp + 1 < L && l >= lp + 2) bad |= !(out[o0 + (l - lp - 1)] >= out[o1 + (l - lp - 2)]);
            if (l < L) bad_l |= !(out[o0 + (l - lp - 1)] <= out[o0 + (l - lp)]);
        }
    }
    bad = __any_sync(0xffffffffu, bad);
    bad_l = __any_sync(0xffffffffu, bad_l);
    const int flags = (bad ? 0 : 1) | (bad_l ? 0 : 2);
    if (nw == 1) {
        if (lane == 0) reinterpret_cast<int*>(ws + lay.smono)[slot] = flags;
        return;
    }
    if (lane == 0 && bad) atomicOr(s_bad, 1);
    if (lane == 0 && bad_l) atomicOr(s_bad, 2);
    __syncthreads();
    if (threadIdx.x == 0) { reinterpret_cast<int*>(ws + lay.smono)[slot] = 3 & ~*s_bad; *s_bad = 0; }
    __syncthreads();
}

// grid (n_inst, maxV - 1): CTA (instance, r).  The warps take i = r+1.. round
// robin and skip non-canonical items (a slot is filled by its first i).  SMALL
// triangles (C4: 496 entries, every item canonical): the warp fills its item at
// once.  BIG ones (C3: 4560 entries, ~2 canonical items per r): the canonical
// items are collected and each is filled by the whole CTA.
template <bool BIG>
__device__ __forceinline__ void stab_body(const pp_batch& b) {
    const pp_instance I = b.inst[blockIdx.x];
    const int r = blockIdx.y + 1;
    const int L = I.L, V = I.V;
    if (L > SR_MAX || V > SR_MAX || r >= V) return;
    __shared__ int s_can[SR_MAX];
    __shared__ int s_nc, s_bad;
    const int* sidx = reinterpret_cast<const int*>(b.ws + I.ws_off + ws_layout(L, V).sidx);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (BIG) {
        if (threadIdx.x == 0) { s_nc = 0; s_bad = 0; }
        __syncthreads();
    }
    for (int i = r + 1 + warp; i <= V; i += nw) {
        const int slot = sidx[(r - 1) * V + (i - 1)];
        bool dup = false;
        for (int q = r + 1 + lane; q < i; q += 32) dup |= sidx[(r - 1) * V + (q - 1)] == slot;
        if (__any_sync(0xffffffffu, dup)) continue;
        if (!BIG) stab_fill(b, I, r, i, warp, 1, &s_bad);
        else if (lane == 0) s_can[atomicAdd(&s_nc, 1)] = i;
    }
    if (!BIG) return;
    __syncthreads();
    const int nc = s_nc;
    for (int c = 0; c < nc; ++c) stab_fill(b, I, r, s_can[c], 0, nw, &s_bad);
}
// big triangles: (maxL - 1) maxL / 2 >= STAB_BIG
constexpr int STAB_BIG = 1024;
__global__ void __launch_bounds__(128) k_stab(pp_batch b) { stab_body<false>(b); }
__global__ void __launch_bounds__(128) k_stab_big(pp_batch b) { stab_body<true>(b); }
__global__ void __launch_bounds__(128) k_stab_p(const pp_batch* __restrict__ bp) {
    const pp_batch b = *bp;
    stab_body<false>(b);
}
__global__ void __launch_bounds__(128) k_stab_big_p(const pp_batch* __restrict__ bp) {
    const pp_batch b = *bp;
    stab_body<true>(b);
}

// Debug timeline of the per-step kernels (tools/step_trace.py): one record of
// 4 x u64 per CTA when g_step_trace is set: (kind << 56 | j << 40 | smid << 32 | block
// linear id), start, end, end of the PDL wait (0 if none) (globaltimer ns).
__device__ unsigned long long* g_step_trace = nullptr;
__device__ int g_step_trace_cap = 0;
__device__ int g_step_trace_n = 0;
__shared__ unsigned long long s_trace_wait;
struct StepTrace {
    unsigned long long t0 = 0;
    __device__ __forceinline__ void begin() {
        if (g_step_trace && threadIdx.x == 0) {
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
            s_trace_wait = 0;
        }
    }
    __device__ __forceinline__ void end(int kind, int j) {
        if (!g_step_trace) return;
        __syncthreads();
        if (threadIdx.x != 0) return;
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        const int k = atomicAdd(&g_step_trace_n, 1);
        if (k >= g_step_trace_cap) return;
        unsigned smid;
        asm("mov.u32 %0, %%smid;" : "=r"(smid));
        const unsigned long long bid = blockIdx.x + (unsigned long long)gridDim.x * (blockIdx.y + (unsigned long long)gridDim.y * blockIdx.z);
        unsigned long long* r = g_step_trace + 4 * (int64_t)k;
        r[0] = ((unsigned long long)kind << 56) | ((unsigned long long)j << 40) | ((unsigned long long)smid << 32) | (bid & 0xffffffffu);
        r[1] = t0; r[2] = t1; r[3] = s_trace_wait;
    }
};

// Programmatic dependent launch (the graph-replayed per-step chain): a kernel
// lets its successor launch as soon as all its CTAs run, and the successor
// stages its producer-independent operands before waiting (no-ops without PDL).
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// where the per-step kernels let their successor launch: 0 = at entry,
// 1 = once the CTA's operands are staged, 2 = after its compute (measured
// best: n = 1 C3 DP 1.42 -> 1.33 ms; early-launched successors only occupy slots)
#ifndef PDL_TRIGGER_AT
#define PDL_TRIGGER_AT 2
#endif
template <int AT>
__device__ __forceinline__ void pdl_trigger_at() {
    if constexpr (AT == PDL_TRIGGER_AT) pdl_trigger();
}
__device__ __forceinline__ void pdl_wait() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (g_step_trace && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(s_trace_wait));
}

// (min, max) micro-kernel: a thread owns a TA x TB register tile and folds one
// K index per step, acc[a][c] = min(acc[a][c], max(p[a], q[c])).
template <int TA, int TB>
__device__ __forceinline__ void mm_step(double (&acc)[TA][TB], const double* prow, const double* qrow) {
    double p[TA], q[TB];
#pragma unroll
    for (int a = 0; a < TA; a += 2) { const double2 v = *reinterpret_cast<const double2*>(prow + a); p[a] = v.x; p[a + 1] = v.y; }
    if constexpr (TB == 1) {
        q[0] = qrow[0];
    } else {
#pragma unroll
        for (int c = 0; c < TB; c += 2) { const double2 v = *reinterpret_cast<const double2*>(qrow + c); q[c] = v.x; q[c + 1] = v.y; }
    }
#pragma unroll
    for (int a = 0; a < TA; ++a)
#pragma unroll
        for (int c = 0; c < TB; ++c) acc[a][c] = dmin(acc[a][c], dmax(p[a], q[c]));
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src) : "memory");
}
// same, with an L2 eviction-priority policy (the stage-term triangles)
__device__ __forceinline__ void cp_async8_hint(double* dst, const double* src, uint64_t pol) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "l"(pol) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }

// TMA 1-D bulk copies (cp.async.bulk) completing on an mbarrier: one thread
// moves a whole contiguous span, no per-element instructions.  Spans are split
// into a 16-byte-aligned body (bulk) and at most one head / tail double (plain
// loads); the shared destination is placed at the same 16-byte phase as the
// source so the body is aligned on both sides.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait0(uint64_t* bar) {   // phase 0 (single-use barrier)
    unsigned ok = 0;
    while (!ok)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(ok) : "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, unsigned parity) {   // reused barrier
    unsigned ok = 0;
    while (!ok)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(double* dst, const double* src, unsigned bytes, uint64_t* bar, uint64_t pol) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}
__device__ __forceinline__ int dphase(const void* p) { return (int)((reinterpret_cast<uintptr_t>(p) >> 3) & 1); }
// dst[e] = src[e] for e in [e0, e1): thread 0 issues the aligned body (arming
// `bar` with its bytes, possibly 0), threads 0/1 copy the head / tail double.
// dst and src must have the same 16-byte phase.
__device__ __forceinline__ void stage_span(double* dst, const double* src, int e0, int e1, uint64_t* bar, uint64_t pol) {
    const int n = e1 - e0;
    const int head = n > 0 ? dphase(src + e0) : 0;
    const int body = max(0, n - head) & ~1;
    const int tail = max(0, n - head - body);
    if (threadIdx.x == 0) {
        mbar_expect_tx(bar, 8u * body);
        if (body) bulk_g2s(dst + e0 + head, src + e0 + head, 8u * body, bar, pol);
        if (head) dst[e0] = src[e0];
    }
    if (threadIdx.x == 1 && tail) dst[e1 - 1] = src[e1 - 1];
}
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

constexpr int KC = 32;   // K chunk staged per __syncthreads
#ifndef EXPAND_TRW
#define EXPAND_TRW 2        // expand register tile 4 xi x 2 r (8 accumulators)
#endif

// ----------------------------------------------------------------------------
// k_expand(j), step j of the wavefront, once slice W_j is final:
//  (a) y < ybase: X(l', xi, r, i = j + r) for every target r (l' = y + 1),
//        X = min_{r' <= j} max(W_j(l', xi-1, r'), chan(l', r', r, i)),
//        chan = (M * payload(l')) / ((r' * r) * cross(r', r, i))   (partition.py:130-138)
//      one CTA per (instance, l', 64 xi x 64 r plane), 4x4 register tiles,
//      K range per tile trimmed to r' <= j - xi + 2 (W_j is inf beyond).
//  (b) y >= ybase: the full stage-term table of step j's combine targets,
//        S[r][l'][l] = T1[r][l'][l] (+ sync(l'+1, l, j+1, j+r) if r > 1), inf for l <= l'
//      (partition.py:127-129, cost.py:99), r = y - ybase + 1.
// ----------------------------------------------------------------------------
constexpr int EX_T = 128, EX_P = 64, EX_S = EX_P + 4;

__global__ void __launch_bounds__(EX_T) k_expand(pp_batch b, int j, int planes_r, int ybase) {
    const pp_instance I = b.inst[blockIdx.x];
    const int L = I.L, V = I.V, M = I.M;
    if (j >= V) return;
    const WsLayout lay = ws_layout(L, V);
    double* ws = b.ws + I.ws_off;
    const int t = threadIdx.x;
    if ((int)blockIdx.y >= ybase) {
        const int r = (int)blockIdx.y - ybase + 1;
        if (blockIdx.z != 0 || r > V - j) return;
        const int i = j + r;
        const double* T1 = ws + lay.T1;
        const double* psum = ws + lay.psum;
        const double den = (double)r * ws[lay.minpair + (int64_t)(i - r) * V + (i - 1)];
    const uint64_t pol = l2_evict_last_policy();   // re-read by the combine of every step
        const double num = 2.0 * (double)(r - 1);
        const bool den_ok = div_fixed_ok(den);
        const double yd = den_ok ? div_recip(den) : 0.0;   // fixed divisor: '/' bits via div_fixed
        double* S = ws + lay.S + stage_idx(L, r, 0, 1);
#pragma unroll 4
        for (int e = t; e < L * L; e += EX_T) {
            const int lp = e / L, l = e - lp * L + 1;
            double s = PP_INF;
            if (lp >= 1 && l > lp) {
                s = T1[stage_idx(L, r, lp, l)];
                if (r > 1) s += div_fixed(num * psum[(int64_t)lp * L + (l - 1)], den, yd, den_ok);
            }
            S[e] = s;
        }
        return;
    }
    const int lp = blockIdx.y + 1;
    if (lp > L - 1) return;
    const int xi0 = 2 + EX_P * (int)(blockIdx.z / planes_r), r0 = 1 + EX_P * (int)(blockIdx.z % planes_r);
    const int nxi = min(EX_P, j + 2 - xi0), nr = min(EX_P, V - j + 1 - r0);
    if (nxi <= 0 || nr <= 0) return;
    const double* Wj = ws + lay.W;
    const double* cross = ws + lay.cross;
    const double Mp = (double)M * (b.efwd[I.layer_off + lp - 1] + b.ebwd[I.layer_off + lp - 1]);   // partition.py:131,137
    __shared__ __align__(16) double As[KC][EX_S];   // [r'][xi - xi0]  W_j(l', xi-1, r')
    __shared__ __align__(16) double Bs[KC][EX_S];   // [r'][r - r0]    chan(l', r', r, j+r)
    const int ntx = (nxi + 3) >> 2, ntr = (nr + 3) >> 2, ntiles = ntx * ntr;
    const int wx = ntx * 4, wr = ntr * 4;
    int tx[2], tr[2], kend[2];
    double acc[2][4][4];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const int id = t + u * EX_T;
        tx[u] = (id < ntiles) ? id % ntx : -1;
        tr[u] = (id < ntiles) ? id / ntx : 0;
        kend[u] = (id < ntiles) ? j - (xi0 + 4 * tx[u]) + 2 : 0;
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[u][a][c] = PP_INF;
    }
    const int kmax = j - xi0 + 2;
    for (int rp0 = 1; rp0 <= kmax; rp0 += KC) {
        const int kc = min(KC, kmax - rp0 + 1);
        for (int e = t; e < kc * wx; e += EX_T) {
            const int rr = e / wx, cc = e - rr * wx;
            As[rr][cc] = (cc < nxi) ? Wj[W_idx(L, j, lp, rp0 + rr, xi0 + cc - 1)] : PP_INF;
        }
        for (int e = t; e < kc * wr; e += EX_T) {
            const int rr = e / wr, cc = e - rr * wr;
            const int rp = rp0 + rr, r = r0 + cc;
            Bs[rr][cc] = (cc < nr) ? Mp / ((double)(rp * r) * cross[cross_idx(V, j + r, r, rp)]) : PP_INF;
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            if (tx[u] < 0) continue;
            const int kk_end = min(kc, kend[u] - rp0 + 1);
            for (int kk = 0; kk < kk_end; ++kk) mm_step<4, 4>(acc[u], &As[kk][4 * tx[u]], &Bs[kk][4 * tr[u]]);
        }
        __syncthreads();
    }
    double* X = ws + lay.X;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        if (tx[u] < 0) continue;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int r = r0 + 4 * tr[u] + c;
            if (r > V - j) continue;
            double* Xr = X + X_base(L, j + r, r) + (int64_t)(lp - 1) * j;
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const int xi = xi0 + 4 * tx[u] + a;
                if (xi <= j + 1) Xr[xi - 2] = acc[u][a][c];
            }
        }
    }
}

// stage(l', l, r, i) = (M * span(l'+1, l)) / r (+ sync(l'+1, l, i-r+1, i) if r > 1)
// partition.py:127-129, cost.py:99 (scalar form, used by the backtrack).
__device__ __forceinline__ double stage_term(int M, int L, int V, const double* prefix, const double* psum,
                                             const double* minpair, int lp, int l, int r, int i) {
    double s = (double)M * (prefix[l] - prefix[lp]) / (double)r;
    if (r > 1) {
        double total = psum[(int64_t)lp * L + (l - 1)];
        s += 2.0 * (double)(r - 1) * total / ((double)r * minpair[(int64_t)(i - r) * V + (i - 1)]);
    }
    return s;
}

// ----------------------------------------------------------------------------
// k_combine_diag(j), step j: every target (r, i = j + r) of slice i,
//   W_i(l, r, xi) = min_{l'} max(S[r][l'][l], X(l', xi, r, i)),  xi in 2..j+1,
// every other cell of the row block is +inf.  All CTAs of a launch share j, so
// their work is uniform.  grid (n_inst, maxV - j, row blocks x xi blocks); the
// K loop streams 32-row chunks of S and X through a cp.async double buffer.
// Register tile TL x TX with TX = 4, 2, 1 for j >= 4, 2..3, 1.
// ----------------------------------------------------------------------------
constexpr int CD_T = 256, CD_L = 64, CD_X = 64, CD_W = 68;
struct CDSmem {
    double X[2][KC][CD_W];   // [l' - lp0][xi - cA]
    double S[2][KC][CD_W];   // [l' - lp0][l - l0]
};
constexpr size_t CD_SMEM = sizeof(CDSmem);

template <int TX>
__device__ void combine_compute(double* Wi, int i, int r, int L, int l0, int nl, int cA, int ncol, int j,
                                const double* __restrict__ X, const double* __restrict__ Srow, CDSmem& sm) {
    constexpr int TL = 16 / TX;
    const int t = threadIdx.x;
    const int ntl = (nl + TL - 1) / TL, ntx = (ncol + TX - 1) / TX, ntiles = ntl * ntx;
    const int wl = ntl * TL, wx = ntx * TX;
    int ti[2], tj[2], kb[2], ke[2];
    double acc[2][TL][TX];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const int id = t + u * CD_T;
        ti[u] = (id < ntiles) ? id / ntx : -1;
        tj[u] = (id < ntiles) ? id % ntx : 0;
        kb[u] = max(1, cA + TX * tj[u] - 1);          // X(l', xi) is inf for l' < xi - 1
        ke[u] = min(L - 1, l0 + TL * ti[u] + TL - 2);  // S(l', l) is inf for l' >= l
#pragma unroll
        for (int a = 0; a < TL; ++a)
#pragma unroll
            for (int c = 0; c < TX; ++c) acc[u][a][c] = PP_INF;
    }
    const int kmin = max(1, cA - 1), kmax = min(L - 1, l0 + nl - 2);
    auto stage = [&](int buf, int lp0) {
        const int kc = min(KC, kmax - lp0 + 1);
        for (int e = t; e < KC * wx; e += CD_T) {
            const int rr = e / wx, cc = e - rr * wx;
            double* d = &sm.X[buf][rr][cc];
            if (rr < kc && cc < ncol) cp_async8(d, X + (int64_t)(lp0 + rr - 1) * j + (cA - 2 + cc));
            else *d = PP_INF;
        }
        for (int e = t; e < KC * wl; e += CD_T) {
            const int rr = e / wl, cc = e - rr * wl;
            double* d = &sm.S[buf][rr][cc];
            if (rr < kc && cc < nl) cp_async8(d, Srow + (int64_t)(lp0 + rr) * L + (l0 - 1 + cc));
            else *d = PP_INF;
        }
        cp_async_commit();
    };
    if (kmin <= kmax) {
        int buf = 0;
        stage(0, kmin);
        for (int lp0 = kmin; lp0 <= kmax; lp0 += KC) {
            if (lp0 + KC <= kmax) { stage(buf ^ 1, lp0 + KC); cp_async_wait<1>(); }
            else cp_async_wait<0>();
            __syncthreads();
            const int kc = min(KC, kmax - lp0 + 1);
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                if (ti[u] < 0) continue;
                const int k0 = max(0, kb[u] - lp0), k1 = min(kc, ke[u] - lp0 + 1);
                for (int kk = k0; kk < k1; ++kk)
                    mm_step<TL, TX>(acc[u], &sm.S[buf][kk][TL * ti[u]], &sm.X[buf][kk][TX * tj[u]]);
            }
            __syncthreads();
            buf ^= 1;
        }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        if (ti[u] < 0) continue;
#pragma unroll
        for (int a = 0; a < TL; ++a) {
            const int l = l0 + TL * ti[u] + a;
            if (l > L || l >= l0 + nl) continue;
            double* row = Wi + ((int64_t)(l - 1) * i + (r - 1)) * i;
#pragma unroll
            for (int c = 0; c < TX; ++c) {
                // only this CTA's DP columns: a padded column past cB is either a
                // structural cell of this plane (the +inf loop writes it) or the
                // next xi plane's first column (its CTA writes it) — never both
                const int xi = cA + TX * tj[u] + c;
                if (xi - cA < ncol) row[xi - 1] = acc[u][a][c];
            }
        }
    }
}

__global__ void __launch_bounds__(CD_T, 2) k_combine_diag(pp_batch b, int j, int planes_x) {
    const pp_instance I = b.inst[blockIdx.x];
    const int L = I.L, V = I.V;
    const int r = blockIdx.y + 1;
    if (j >= V || r > V - j) return;
    const int i = j + r;
    const int l0 = 1 + CD_L * (int)(blockIdx.z / planes_x), x0 = 1 + CD_X * (int)(blockIdx.z % planes_x);
    if (l0 > L || x0 > i) return;
    const int nl = min(CD_L, L - l0 + 1), nx = min(CD_X, i - x0 + 1);
    const bool allow = I.flags & PP_ALLOW_REPLICATION;
    const WsLayout lay = ws_layout(L, V);
    double* ws = b.ws + I.ws_off;
    double* Wi = ws + lay.W + W_base(L, i);
    const int cA = max(x0, 2), cB = min(x0 + nx - 1, j + 1);
    const bool dp_cells = (allow || r == 1) && cA <= cB;   // partition.py:103-104
    const int ncol = dp_cells ? cB - cA + 1 : 0;
    const int TX = ncol >= 4 ? 4 : (ncol >= 2 ? 2 : 1);
    for (int e = threadIdx.x; e < nl * nx; e += CD_T) {   // xi = 1, xi > j + 1, disabled widths
        const int l = l0 + e / nx, xi = x0 + e % nx;
        if (dp_cells && xi >= cA && xi <= cB) continue;
        Wi[((int64_t)(l - 1) * i + (r - 1)) * i + (xi - 1)] = PP_INF;
    }
    if (!dp_cells) return;
    extern __shared__ __align__(16) double cd_smem[];
    CDSmem& sm = *reinterpret_cast<CDSmem*>(cd_smem);
    const double* X = ws + lay.X + X_base(L, i, r);
    const double* Srow = ws + lay.S + stage_idx(L, r, 0, 1);
    if (TX == 4) combine_compute<4>(Wi, i, r, L, l0, nl, cA, ncol, j, X, Srow, sm);
    else if (TX == 2) combine_compute<2>(Wi, i, r, L, l0, nl, cA, ncol, j, X, Srow, sm);
    else combine_compute<1>(Wi, i, r, L, l0, nl, cA, ncol, j, X, Srow, sm);
}

// ----------------------------------------------------------------------------
// Shared-memory-resident fast path (L <= 128 and V <= 128, i.e. C1-C4):
// every work item stages ALL of its operands in shared memory once, crosses a
// single __syncthreads, and then every thread folds its register tiles over
// its own trimmed K range with no further barriers (no barrier stalls, no
// inter-thread imbalance inside a chunk).
// ----------------------------------------------------------------------------

// The (min, max) fold of one 4 xi x TRW r expand tile over r' (lanes sub, sub + ks,
// ...): only the valid cells of A = W_j(l', xi', r') are read, so A's structural
// cells may hold anything (no +inf pass).  Column a (xi = xi0 + a, xi' = xi - 1)
// holds values for r' <= j - xi' + 1 = kend - a (kend = j - xi0 + 2): the bulk
// of the r' range folds every column, the last 3 r' mask the columns whose
// triangle ended.  xi0 = 2: column 0 is xi' = 1, whose only cell is the base
// W_j(l', 1, j) (partition.py:117-121), folded once (min is idempotent, so
// every split-K lane may add it).  With replication (callers check).
template <int TRW>
__device__ __forceinline__ void expand_fold_tri(double (&acc)[4][TRW], const double* A, const double* B, int j,
                                                int nrs, int xi0, const int (&xa)[4], const int (&ra)[TRW], int sub,
                                                int ks) {
    const int kend = j - xi0 + 2;
    const bool base_col = xi0 == 2;
    int rp = 1 + sub;
    for (; rp <= kend - 3; rp += ks) {
        const double* Ar = A + (rp - 1) * j;
        const double* Br = B + (rp - 1) * nrs;
        double p[4], q[TRW];
#pragma unroll
        for (int a = 0; a < 4; ++a) p[a] = Ar[xa[a]];
        if (base_col) p[0] = PP_INF;
#pragma unroll
        for (int c = 0; c < TRW; ++c) q[c] = Br[ra[c]];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int c = 0; c < TRW; ++c) acc[a][c] = dmin(acc[a][c], dmax(p[a], q[c]));
    }
    for (; rp <= kend; rp += ks) {
        const double* Ar = A + (rp - 1) * j;
        const double* Br = B + (rp - 1) * nrs;
        double p[4], q[TRW];
#pragma unroll
        for (int a = 0; a < 4; ++a) p[a] = (rp <= kend - a && !(a == 0 && base_col)) ? Ar[xa[a]] : PP_INF;
#pragma unroll
        for (int c = 0; c < TRW; ++c) q[c] = Br[ra[c]];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int c = 0; c < TRW; ++c) acc[a][c] = dmin(acc[a][c], dmax(p[a], q[c]));
    }
    if (base_col) {
        const double pb = A[(j - 1) * j];
#pragma unroll
        for (int c = 0; c < TRW; ++c) acc[0][c] = dmin(acc[0][c], dmax(pb, B[(j - 1) * nrs + ra[c]]));
    }
}

// expand, step j: one CTA per (instance, l').  smem: A = W_j(l', ., .) block
// [r'][xi'] (j x j, one contiguous copy), B = chan(l', r', r) [r'][r]
// (j x (V-j) exact divisions).  Tiles 4 xi x 4 r; tile K range r' <= j - xi0 + 2.
// Targets r = rfirst..V-j of row l' (rfirst = 2 leaves the r = 1 target to the
// fused critical-path task of the persistent DP).  ex_smem: j * (j + nt) doubles.
__device__ __forceinline__ void expand_row_s(const pp_batch& b, const pp_instance& I, int j, int lp, int rfirst,
                                             double* ex_smem, int rlast = SR_MAX) {
    const int L = I.L, V = I.V, M = I.M;
    const int nr = min(V - j, rlast), nt = nr - rfirst + 1;   // targets r = rfirst..nr
    const int nrow = V - j;                                       // row stride of the chan class table
    if (nt <= 0) return;
    const WsLayout lay = ws_layout(L, V);
    double* ws = b.ws + I.ws_off;
    const double* Wsrc = ws + lay.W + W_idx(L, j, lp, 1, 1);
    const double* cross = ws + lay.cross;
    const double Mp = (double)M * (b.efwd[I.layer_off + lp - 1] + b.ebwd[I.layer_off + lp - 1]);   // partition.py:131,137
    double* A = ex_smem;             // [r'-1][xi'-1], stride j
    double* B = ex_smem + j * j;     // [r'-1][r-rfirst], stride nt
    const int t = threadIdx.x;
    const bool allow = I.flags & PP_ALLOW_REPLICATION;
    const int lane = t & 31;
    const int warp = t >> 5, nw = blockDim.x >> 5;
    // B first: it depends only on tables built before the wavefront, so under
    // PDL it overlaps the previous kernel's tail; A (slice j) after the wait.
    // B[r'-1][r-rfirst] = chan(l', r', r, j + r): copied from the row's payload-class
    // table (same expression, same bits), else divided here
    const int cls = reinterpret_cast<const int*>(ws + lay.chcls + CHAN_CLS)[lp];
    if (cls >= 0) {
        const double* Tj = ws + lay.chan + (int64_t)cls * tet(V) + chan_step(V, j);
        for (int rp = 1 + warp; rp <= j; rp += nw)
            for (int q = lane; q < nt; q += 32) cp_async8(B + (rp - 1) * nt + q, Tj + (rp - 1) * nrow + (q + rfirst - 1));
        cp_async_commit();
    } else {
        cp_async_commit();
        for (int rp = 1 + warp; rp <= j; rp += nw)
            for (int q = lane; q < nt; q += 32) {
                const int r = rfirst + q;
                B[(rp - 1) * nt + q] = Mp / ((double)(rp * r) * cross[cross_idx(V, j + r, r, rp)]);
            }
    }
    pdl_wait();
    // A[r'-1][xi'-1] = W_j(l', xi', r'): materialised cells by cp.async (all in
    // flight at once), structural ones (never written by the DP) as +inf
    for (int rp = 1 + warp; rp <= j; rp += nw)
        for (int xip = 1 + lane; xip <= j; xip += 32) {
            const int e = (rp - 1) * j + (xip - 1);
            if (W_structural(j, rp, xip, allow)) cp_async8(A + e, Wsrc + e);
            else A[e] = PP_INF;
        }
    cp_async_commit();
    __shared__ int64_t s_xb[SR_MAX];   // X_base of target r (the int64 index math once per CTA)
    for (int q = t; q < nt; q += blockDim.x) s_xb[q] = X_base(L, j + rfirst + q, rfirst + q);
    cp_async_wait<0>();
    __syncthreads();
    pdl_trigger_at<1>();
    constexpr int TRW = EXPAND_TRW;   // target columns per register tile (4 xi x TRW r)
    const int ntx = (j + 3) >> 2, ntr = (nt + TRW - 1) / TRW, ntiles = ntx * ntr;
    // split-K when the plane has few tiles: ks consecutive lanes share a tile,
    // fold interleaved r' subsets and min-reduce with shuffles
    int ks = 1;
    while (ks < 8 && ntiles * ks * 2 <= (int)blockDim.x) ks *= 2;
    const int sub = t % ks;
    const unsigned gmask = (ks == 32 ? 0xffffffffu : ((1u << ks) - 1u)) << (lane & ~(ks - 1));
    double* X = ws + lay.X;
    for (int id = t / ks; id < ntiles; id += blockDim.x / ks) {
        const int tx = id % ntx, tr = id / ntx;
        const int xi0 = 2 + 4 * tx, r0 = rfirst + TRW * tr;
        const int kend = j - xi0 + 2;   // W_j(l', xi-1, r') = inf for r' > j - xi + 2
        double acc[4][TRW];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int c = 0; c < TRW; ++c) acc[a][c] = PP_INF;
        // padded columns read in-range garbage-free copies: clamp and mask at the end
        const int xa[4] = {min(xi0 - 1, j) - 1, min(xi0, j) - 1, min(xi0 + 1, j) - 1, min(xi0 + 2, j) - 1};
        int ra[TRW];
#pragma unroll
        for (int c = 0; c < TRW; ++c) ra[c] = min(r0 + c, nr) - rfirst;
        for (int rp = 1 + sub; rp <= kend; rp += ks) {
            const double* Ar = A + (rp - 1) * j;
            const double* Br = B + (rp - 1) * nt;
            double p[4], q[TRW];
#pragma unroll
            for (int a = 0; a < 4; ++a) p[a] = Ar[xa[a]];
#pragma unroll
            for (int c = 0; c < TRW; ++c) q[c] = Br[ra[c]];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int c = 0; c < TRW; ++c) acc[a][c] = dmin(acc[a][c], dmax(p[a], q[c]));
        }
        for (int off = 1; off < ks; off <<= 1)
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int c = 0; c < TRW; ++c) acc[a][c] = dmin(acc[a][c], __shfl_xor_sync(gmask, acc[a][c], off));
        if (sub != 0) continue;
#pragma unroll
        for (int c = 0; c < TRW; ++c) {
            const int r = r0 + c;
            if (r > nr) continue;
            double* Xr = X + s_xb[r - rfirst] + (int64_t)(lp - 1) * j;
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const int xi = xi0 + a;
                if (xi <= j + 1) Xr[xi - 2] = acc[a][c];
            }
        }
    }
}

// expand, step j, for nrows consecutive rows l' that share one chan payload
// class (every row of a transformer stack): the chan block B = chan(cls, r', r)
// is staged ONCE for all rows and the rows' W_j blocks side by side, so the
// block is a (min, max) product of the stacked (row, xi) x r' operand with one
// r' x r operand.  smem: B (j x (V-j)) then nrows A blocks (j x j each).
__device__ __forceinline__ void expand_rows_cls(const pp_batch& b, const pp_instance& I, int j, int lp0, int nrows,
                                                int cls, double* ex_smem) {
    const int L = I.L, V = I.V;
    const int nr = V - j;
    const WsLayout lay = ws_layout(L, V);
    double* ws = b.ws + I.ws_off;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nw = blockDim.x >> 5;
    const bool allow = I.flags & PP_ALLOW_REPLICATION;
    // TMA bulk: the chan block and the rows' W_j blocks (consecutive in W) are
    // each one cp.async.bulk (2 spare doubles of shared memory for the 16-byte
    // phase); the never-written structural cells are set to +inf afterwards
    __shared__ uint64_t s_mbar[2];
    const double* Tj = ws + lay.chan + (int64_t)cls * tet(V) + chan_step(V, j);
    const double* Wsrc = ws + lay.W + W_idx(L, j, lp0, 1, 1);   // rows are consecutive j x j blocks
    double* B = ex_smem + (dphase(ex_smem) ^ dphase(Tj));             // [r'-1][r-1], stride nr
    double* A0 = ex_smem + 1 + j * nr;                                // row k: A0 + k j^2
    A0 += dphase(A0) ^ dphase(Wsrc);
    if (t == 0) { mbar_init(&s_mbar[0]); mbar_init(&s_mbar[1]); }
    __syncthreads();
    stage_span(B, Tj, 0, j * nr, &s_mbar[0], l2_evict_last_policy());
    pdl_wait();
    stage_span(A0, Wsrc, 0, nrows * j * j, &s_mbar[1], l2_evict_normal_policy());
    __shared__ int64_t s_xb[SR_MAX];
    for (int q = t; q < nr; q += blockDim.x) s_xb[q] = X_base(L, j + 1 + q, 1 + q);
    mbar_wait0(&s_mbar[0]);
    mbar_wait0(&s_mbar[1]);
    __syncthreads();   // head / tail copies land (before the +inf pass without replication)
    if (!allow) {      // without replication the valid cells are not a triangle: mask them explicitly
        for (int rp = 1 + warp; rp <= j; rp += nw)
            for (int xip = 1 + lane; xip <= j; xip += 32)
                if (!W_structural(j, rp, xip, allow)) {
                    const int e = (rp - 1) * j + (xip - 1);
                    for (int k = 0; k < nrows; ++k) A0[k * j * j + e] = PP_INF;
                }
        __syncthreads();
    }
    pdl_trigger_at<1>();
    constexpr int TRW = EXPAND_TRW;
    const int ntx = (j + 3) >> 2, ntr = (nr + TRW - 1) / TRW, per_row = ntx * ntr, ntiles = nrows * per_row;
    int ks = 1;
    while (ks < 8 && ntiles * ks * 2 <= (int)blockDim.x) ks *= 2;
    const int sub = t % ks;
    const unsigned gmask = (ks == 32 ? 0xffffffffu : ((1u << ks) - 1u)) << (lane & ~(ks - 1));
    double* X = ws + lay.X;
    for (int id = t / ks; id < ntiles; id += blockDim.x / ks) {
        const int k = id / per_row, rem = id - k * per_row;
        const int tx = rem % ntx, tr = rem / ntx;
        const int xi0 = 2 + 4 * tx, r0 = 1 + TRW * tr;
        const int kend = j - xi0 + 2;
        double acc[4][TRW];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int c = 0; c < TRW; ++c) acc[a][c] = PP_INF;
        const int xa[4] = {min(xi0 - 1, j) - 1, min(xi0, j) - 1, min(xi0 + 1, j) - 1, min(xi0 + 2, j) - 1};
        int ra[TRW];
#pragma unroll
        for (int c = 0; c < TRW; ++c) ra[c] = min(r0 + c, nr) - 1;
        const double* A = A0 + k * j * j;
        if (allow) {
            expand_fold_tri<TRW>(acc, A, B, j, nr, xi0, xa, ra, sub, ks);
        } else {
            for (int rp = 1 + sub; rp <= kend; rp += ks) {
                const double* Ar = A + (rp - 1) * j;
                const double* Br = B + (rp - 1) * nr;
                double p[4], q[TRW];
#pragma unroll
                for (int a = 0; a < 4; ++a) p[a] = Ar[xa[a]];
#pragma unroll
                for (int c = 0; c < TRW; ++c) q[c] = Br[ra[c]];
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int c = 0; c < TRW; ++c) acc[a][c] = dmin(acc[a][c], dmax(p[a], q[c]));
            }
        }
        for (int off = 1; off < ks; off <<= 1)
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int c = 0; c < TRW; ++c) acc[a][c] = dmin(acc[a][c], __shfl_xor_sync(gmask, acc[a][c], off));
        if (sub != 0) continue;
        const int lp = lp0 + k;
#pragma unroll
        for (int c = 0; c < TRW; ++c) {
            const int r = r0 + c;
            if (r > nr) continue;
            double* Xr = X + s_xb[r - 1] + (int64_t)(lp - 1) * j;
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const int xi = xi0 + a;
                if (xi <= j + 1) Xr[xi - 2] = acc[a][c];
            }
        }
    }
}

__global__ void __launch_bounds__(128) k_expand_s(pp_batch b, int j) {
    const pp_instance I = b.inst[blockIdx.x];
    const int lp = blockIdx.y + 1;
    if (j >= I.V || lp > I.L - 1) return;
    extern __shared__ __align__(16) double ex_smem[];
    expand_row_s(b, I, j, lp, 1, ex_smem);
}
// one row l' per CTA (steps with few rows: every SM gets work)
#ifndef EXPAND_MINB
#define EXPAND_MINB 3   // resident 256-thread expand CTAs per SM the register budget targets (80 registers, no spills)
#endif
#ifndef COMBINE_MINB
#define COMBINE_MINB (COMBINE_TL4 == 2 ? 3 : 2)
#endif
__global__ void __launch_bounds__(256, EXPAND_MINB) k_expand_s_p(const pp_batch* __restrict__ bp, int j, int rfirst, int rlast) {
    pdl_trigger_at<0>();
    StepTrace tr;
    tr.begin();
    const pp_batch b = *bp;
    const pp_instance I = b.inst[blockIdx.x];
    const int lp = blockIdx.y + 1;
    if (j >= I.V || lp > I.L - 1) return;
    extern __shared__ __align__(16) double ex_smem[];
    expand_row_s(b, I, j, lp, rfirst, ex_smem, rlast);
    pdl_trigger_at<2>();
    tr.end(1, j);
}
// rb rows per CTA (host: rb * j^2 + j (V-j) doubles of shared memory): rows of one
// payload class share their chan block (expand_rows_cls), others go row by row.
__global__ void __launch_bounds__(256, EXPAND_MINB) k_expand_m_p(const pp_batch* __restrict__ bp, int j, int rb) {
    pdl_trigger_at<0>();
    StepTrace tr;
    tr.begin();
    const pp_batch b = *bp;
    const pp_instance I = b.inst[blockIdx.x];
    const int lp0 = blockIdx.y * rb + 1;
    if (j >= I.V || lp0 > I.L - 1) return;
    extern __shared__ __align__(16) double ex_smem[];
    const int nrows = min(rb, I.L - lp0);
    const int* rcls = reinterpret_cast<const int*>(b.ws + I.ws_off + ws_layout(I.L, I.V).chcls + CHAN_CLS);
    int cls = rcls[lp0];
    for (int k = 1; k < nrows && cls >= 0; ++k)
        if (rcls[lp0 + k] != cls) cls = -1;
    if (cls >= 0) {
        expand_rows_cls(b, I, j, lp0, nrows, cls, ex_smem);
    } else {
        for (int k = 0; k < nrows; ++k) {
            if (k) __syncthreads();   // the previous row's tiles are done with the shared operands
            expand_row_s(b, I, j, lp0 + k, 1, ex_smem);
        }
    }
    pdl_trigger_at<2>();
    tr.end(1, j);
}

// combine, step j: one CTA per (instance, r), target i = j + r.  smem: the
// stage terms of the item as a packed triangle (row l' holds l = l'+1..L,
// S = T1 + sync, T1 from k_base) and X(., ., r, i) (rows l' = 1..L-1, stride j).
// combine reads stage terms straight from global memory for j <= this (0 = always
// stage them in shared memory; j <= 8 measured no better on B200)
constexpr int S_DIRECT_J = 0;
// k_combine_s_p stages with TMA bulk copies (pp_dp_set_bulk / PP_BULK; same bits)
__device__ int g_combine_bulk = 1;
#ifndef COMBINE_TL4
#define COMBINE_TL4 2   // combine register tile 2 l x 4 xi (8 accumulators: 3 CTAs / SM)
#endif
// combine stops scanning l' once no remaining candidate can lower a cell (needs a
// certified monotone stage-term triangle, k_stab); pp_dp_set_early_exit toggles it
__device__ int g_combine_early_exit = 1;

template <int TX, int TL = 16 / TX>
__device__ __forceinline__ int tile_nfast(int L, int l0, int xi0, int lA, int lB) {
    const int kb = max(max(1, xi0 - 1), lA), ke = min(min(L - 1, l0 + TL - 2), lB);
    return max(0, min(ke, l0 - 1) - kb + 1);
}

// One TL x TX tile: fold l' in [kb, ke].  The lane walks its own l' sequence
// (row pointers advance incrementally through the packed triangle), so lanes
// whose tiles have equal trip counts run in lockstep even though they start
// at different l'.
template <int TX, int TL = 16 / TX>
__device__ __forceinline__ void combine_tile_s(const double* Stri, const int* trio, const double* Xs, int L, int j,
                                               int l0, int xi0, int lA, int lB, double (&acc)[TL][TX]) {
#pragma unroll
    for (int a = 0; a < TL; ++a)
#pragma unroll
        for (int c = 0; c < TX; ++c) acc[a][c] = PP_INF;
    int xc[TX];
#pragma unroll
    for (int c = 0; c < TX; ++c) xc[c] = min(xi0 + c, j + 1) - 2;   // clamp padded columns; masked on write
    const int kb = max(max(1, xi0 - 1), lA);   // l' restricted to [lA, lB] (split-K parts)
    const int ke = min(min(L - 1, l0 + TL - 2), lB);
    const int nfast = max(0, min(ke, l0 - 1) - kb + 1);   // l' < l0: every row of the tile has l > l'
    const double* Sr = Stri + trio[kb] + (l0 - kb - 1);  // S(kb, l0)
    const double* Xr = Xs + (kb - 1) * j;
    for (int k = 0; k < nfast; ++k) {
        double p[TL], q[TX];
#pragma unroll
        for (int a = 0; a < TL; ++a) p[a] = Sr[a];
#pragma unroll
        for (int c = 0; c < TX; ++c) q[c] = Xr[xc[c]];
#pragma unroll
        for (int a = 0; a < TL; ++a)
#pragma unroll
            for (int c = 0; c < TX; ++c) acc[a][c] = dmin(acc[a][c], dmax(p[a], q[c]));
        Sr += L - (kb + k) - 1;   // S(l'+1, l0) = S(l', l0) + (L - l' - 1)
        Xr += j;
    }
    for (int lp = max(kb, l0); lp <= ke; ++lp) {   // the tile's diagonal: rows l <= l' are +inf
        const double* Xd = Xs + (lp - 1) * j;
        double q[TX];
#pragma unroll
        for (int c = 0; c < TX; ++c) q[c] = Xd[xc[c]];
#pragma unroll
        for (int a = 0; a < TL; ++a) {
            const int l = l0 + a;
            if (l <= lp || l > L) continue;
            const double pa = Stri[trio[lp] + (l - lp - 1)];
#pragma unroll
            for (int c = 0; c < TX; ++c) acc[a][c] = dmin(acc[a][c], dmax(pa, q[c]));
        }
    }
}

// Same tile, l' descending, for a certified non-increasing S triangle: the
// candidates of row a at l'' < l' are >= S(l'', l0+a) >= S(l', l0+a) = p[a],
// so once p[a] >= max_c acc[a][c] for every row, no remaining l' can lower any
// cell and the fold stops (the min is unchanged, so the bits are too).
template <int TX, int TL = 16 / TX>
__device__ __forceinline__ void combine_tile_s_desc(const double* Stri, const int* trio, const double* Xs, int L,
                                                    int j, int l0, int xi0, int lA, int lB,
                                                    double (&acc)[TL][TX]) {
#pragma unroll
    for (int a = 0; a < TL; ++a)
#pragma unroll
        for (int c = 0; c < TX; ++c) acc[a][c] = PP_INF;
    int xc[TX];
#pragma unroll
    for (int c = 0; c < TX; ++c) xc[c] = min(xi0 + c, j + 1) - 2;
    const int kb = max(max(1, xi0 - 1), lA);
    const int ke = min(min(L - 1, l0 + TL - 2), lB);
    for (int lp = ke; lp >= max(kb, l0); --lp) {   // the tile's diagonal first: rows l <= l' are +inf
        const double* Xd = Xs + (lp - 1) * j;
        double q[TX];
#pragma unroll
        for (int c = 0; c < TX; ++c) q[c] = Xd[xc[c]];
#pragma unroll
        for (int a = 0; a < TL; ++a) {
            const int l = l0 + a;
            if (l <= lp || l > L) continue;
            const double pa = Stri[trio[lp] + (l - lp - 1)];
#pragma unroll
            for (int c = 0; c < TX; ++c) acc[a][c] = dmin(acc[a][c], dmax(pa, q[c]));
        }
    }
    const int hi = min(ke, l0 - 1);
    if (hi < kb) return;
    const double* Sr = Stri + trio[hi] + (l0 - hi - 1);   // S(hi, l0)
    const double* Xr = Xs + (hi - 1) * j;
    const int nrow = min(TL, L - l0 + 1);                 // rows past L hold no cell
    for (int lp = hi; lp >= kb; --lp) {
        double p[TL], q[TX];
#pragma unroll
        for (int a = 0; a < TL; ++a) p[a] = Sr[a];
#pragma unroll
        for (int c = 0; c < TX; ++c) q[c] = Xr[xc[c]];
#pragma unroll
        for (int a = 0; a < TL; ++a)
#pragma unroll
            for (int c = 0; c < TX; ++c) acc[a][c] = dmin(acc[a][c], dmax(p[a], q[c]));
        if (((hi - lp) & 3) == 3) {
            bool done = true;
#pragma unroll
            for (int a = 0; a < TL; ++a) {
                double m = acc[a][0];
#pragma unroll
                for (int c = 1; c < TX; ++c) m = dmax(m, acc[a][c]);
                done &= (a >= nrow) || p[a] >= m;
            }
            if (done) break;
        }
        Sr -= L - lp;   // S(l'-1, l0) = S(l', l0) - (L - l')
        Xr -= j;
    }
}

// One tile folded by ks lanes (split-K inside the CTA, for items with few
// tiles): lane `sub` takes l' = ke - sub, ke - sub - ks, ... (descending), so
// each lane's own remaining candidates only grow in S and a certified-monotone
// triangle lets the lane stop on its own partial minima; the caller
// min-reduces the ks partials with shuffles (min is exact and order-free).
template <int TX, int TL = 16 / TX>
__device__ __forceinline__ void combine_tile_split(const double* Stri, const int* trio, const double* Xs, int L,
                                                   int j, int l0, int xi0, int lA, int lB, int sub, int ks,
                                                   bool mono, double (&acc)[TL][TX]) {
#pragma unroll
    for (int a = 0; a < TL; ++a)
#pragma unroll
        for (int c = 0; c < TX; ++c) acc[a][c] = PP_INF;
    int xc[TX];
#pragma unroll
    for (int c = 0; c < TX; ++c) xc[c] = min(xi0 + c, j + 1) - 2;
    const int kb = max(max(1, xi0 - 1), lA);
    const int ke = min(min(L - 1, l0 + TL - 2), lB);
    const int nrow = min(TL, L - l0 + 1);
    for (int lp = ke - sub; lp >= kb; lp -= ks) {
        const double* Xr = Xs + (lp - 1) * j;
        double q[TX];
#pragma unroll
        for (int c = 0; c < TX; ++c) q[c] = Xr[xc[c]];
        if (lp >= l0) {   // the tile's diagonal: rows l <= l' are +inf
#pragma unroll
            for (int a = 0; a < TL; ++a) {
                const int l = l0 + a;
                if (l <= lp || l > L) continue;
                const double pa = Stri[trio[lp] + (l - lp - 1)];
#pragma unroll
                for (int c = 0; c < TX; ++c) acc[a][c] = dmin(acc[a][c], dmax(pa, q[c]));
            }
            continue;
        }
        const double* Sr = Stri + trio[lp] + (l0 - lp - 1);
        double p[TL];
#pragma unroll
        for (int a = 0; a < TL; ++a) p[a] = Sr[a];
#pragma unroll
        for (int a = 0; a < TL; ++a)
#pragma unroll
            for (int c = 0; c < TX; ++c) acc[a][c] = dmin(acc[a][c], dmax(p[a], q[c]));
        if (mono) {
            bool done = true;
#pragma unroll
            for (int a = 0; a < TL; ++a) {
                double m = acc[a][0];
#pragma unroll
                for (int c = 1; c < TX; ++c) m = dmax(m, acc[a][c]);
                done &= (a >= nrow) || p[a] >= m;
            }
            if (done) break;
        }
    }
}

template <int TX, int TL = 16 / TX>
__device__ __forceinline__ void combine_tiles_s(double* Wi, int i, int r, int L, int j, const double* Stri,
                                                const int* trio, const double* Xs, int* hist, int* order,
                                                int part, int nparts, int lA, int lB, bool atomic, bool mono) {
    const int t = threadIdx.x;
    const int ntl = (L + TL - 1) / TL, ntx = (j + TX - 1) / TX, ntiles = ntl * ntx;
    // the item is split over nparts CTAs: CTA `part` owns the tiles with id = part (mod nparts)
    const int nmine = ntiles > part ? (ntiles - part + nparts - 1) / nparts : 0;
    // order its tiles by trip count (descending) so each warp's lanes run equal-length loops
    for (int k = t; k < L + 2; k += blockDim.x) hist[k] = 0;
    __syncthreads();
    for (int k = t; k < nmine; k += blockDim.x) {
        const int id = part + k * nparts;
        atomicAdd(&hist[L - tile_nfast<TX, TL>(L, 1 + TL * (id / ntx), 2 + TX * (id % ntx), lA, lB)], 1);
    }
    __syncthreads();
    if (t < 32) {   // exclusive prefix over the L + 2 bins: one warp, 5 bins per lane
        const int per = (L + 2 + 31) / 32, b0 = t * per;
        int loc = 0;
        for (int k = b0; k < min(b0 + per, L + 2); ++k) loc += hist[k];
        int inc = loc;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, inc, off);
            if (t >= off) inc += v;
        }
        int o = inc - loc;
        for (int k = b0; k < min(b0 + per, L + 2); ++k) { const int c = hist[k]; hist[k] = o; o += c; }
    }
    __syncthreads();
    for (int k = t; k < nmine; k += blockDim.x) {
        const int id = part + k * nparts;
        order[atomicAdd(&hist[L - tile_nfast<TX, TL>(L, 1 + TL * (id / ntx), 2 + TX * (id % ntx), lA, lB)], 1)] = id;
    }
    __syncthreads();
    // few tiles: ks lanes per tile split its l' range (ks a power of two <= 32)
    int ks = 1;
    while (ks < 32 && nmine * ks * 2 <= (int)blockDim.x) ks *= 2;
    const int lane = t & 31;
    for (int q0 = t; q0 < nmine * ks; q0 += blockDim.x) {
        const int q = q0 / ks, sub = q0 % ks;
        const int id = order[q];
        const int l0 = 1 + TL * (id / ntx), xi0 = 2 + TX * (id % ntx);
        double acc[TL][TX];
        if (ks == 1) {
            if (mono) combine_tile_s_desc<TX, TL>(Stri, trio, Xs, L, j, l0, xi0, lA, lB, acc);
            else combine_tile_s<TX, TL>(Stri, trio, Xs, L, j, l0, xi0, lA, lB, acc);
        } else {
            combine_tile_split<TX, TL>(Stri, trio, Xs, L, j, l0, xi0, lA, lB, sub, ks, mono, acc);
            const unsigned gmask = (ks == 32 ? 0xffffffffu : ((1u << ks) - 1u)) << (lane & ~(ks - 1));
            for (int off = 1; off < ks; off <<= 1)
#pragma unroll
                for (int a = 0; a < TL; ++a)
#pragma unroll
                    for (int c = 0; c < TX; ++c) acc[a][c] = dmin(acc[a][c], __shfl_xor_sync(gmask, acc[a][c], off));
            if (sub != 0) continue;
        }
#pragma unroll
        for (int a = 0; a < TL; ++a) {
            const int l = l0 + a;
            if (l > L) continue;
            double* row = Wi + ((int64_t)(l - 1) * i + (r - 1)) * i;
#pragma unroll
            for (int c = 0; c < TX; ++c) {
                if (xi0 + c > j + 1) continue;
                if (!atomic) { row[xi0 + c - 1] = acc[a][c]; continue; }
                // split-K part: min into a cell preset to +inf.  Non-negative doubles
                // order like their bit patterns, so a 64-bit atomicMin is the exact min.
                if (acc[a][c] < PP_INF)
                    atomicMin(reinterpret_cast<unsigned long long*>(row + xi0 + c - 1),
                              (unsigned long long)__double_as_longlong(acc[a][c]));
            }
        }
    }
}

// One combine work item (r, i = j + r), tiles part (mod nparts).  x_staged: Xs
// already holds X(., ., r, i) (the fused critical-path task computed it).
// smem: trio (L+1)/2+1, Stri (L-1)L/2, Xs (L-1) x j doubles; hist/order scratch.
__device__ __forceinline__ void combine_item_s(const pp_batch& b, const pp_instance& I, int j, int r, int part,
                                               int nparts, double* cs_smem, int* s_hist, int* s_order,
                                               bool x_staged, int lA = 1, int lB = PP_MAX_LAYERS, bool atomic = false,
                                               bool bulk = false) {
    const int L = I.L, V = I.V;
    if (j >= V || r > V - j) return;
    const int i = j + r;
    const bool allow = I.flags & PP_ALLOW_REPLICATION;
    // cells outside xi in [2, j+1] and disabled widths are structural +inf (W_at)
    if (!(allow || r == 1)) return;   // partition.py:103-104
    const WsLayout lay = ws_layout(L, V);
    double* ws = b.ws + I.ws_off;
    double* Wi = ws + lay.W + W_base(L, i);
    const int t = threadIdx.x;
    int* trio = reinterpret_cast<int*>(cs_smem);                 // [L] triangle row offsets
    double* Stri = cs_smem + (L + 1) / 2 + 1;                    // (L-1)L/2
    double* Xs = Stri + (L - 1) * L / 2;                         // (L-1) x j
    for (int lp = 1 + t; lp < L; lp += blockDim.x) trio[lp] = (lp - 1) * L - (lp - 1) * lp / 2;
    // stage X(., ., r, i) and the item's stage-term triangle (its k_stab slot),
    // rows l' in [la, lb] only (a split-K part folds just those), with cp.async:
    // every copy of the CTA is in flight at once
    const int la = max(lA, 1), lb = min(lB, L - 1);
    const double* Sg;
    const int slot = reinterpret_cast<const int*>(ws + lay.sidx)[(r - 1) * V + (i - 1)];
    if (bulk) {
        // TMA bulk path (one call per CTA): the triangle and X spans each one
        // cp.async.bulk; shared bases shifted (1 spare double each) to the
        // 16-byte phase of their global source
        __shared__ uint64_t s_bar[2];
        const int ns = (L - 1) * L / 2;
        Sg = ws + lay.Stab + (int64_t)slot * ns;
        const double* Xg = ws + lay.X + X_base(L, i, r);
        Stri = cs_smem + (L + 1) / 2 + 1;
        Stri += dphase(Stri) ^ dphase(Sg);
        Xs = cs_smem + (L + 1) / 2 + 2 + ns;
        Xs += dphase(Xs) ^ dphase(Xg);
        if (t == 0) { mbar_init(&s_bar[0]); mbar_init(&s_bar[1]); }
        __syncthreads();
        const int s0 = (la - 1) * L - (la - 1) * la / 2, s1 = lb * L - lb * (lb + 1) / 2;
        stage_span(Stri, Sg, s0, s1, &s_bar[0], l2_evict_last_policy());
        pdl_wait();
        stage_span(Xs, Xg, (la - 1) * j, lb * j, &s_bar[1], l2_evict_normal_policy());
        mbar_wait0(&s_bar[0]);
        mbar_wait0(&s_bar[1]);
    } else {
        // the stage-term triangle (built before the wavefront) first: under PDL it
        // overlaps the previous kernel's tail; X (this step's expand) after the wait
        const int ns = (L - 1) * L / 2;
        Sg = ws + lay.Stab + (int64_t)slot * ns;
        const int s0 = (la - 1) * L - (la - 1) * la / 2, s1 = lb * L - lb * (lb + 1) / 2;
        const uint64_t pol = l2_evict_last_policy();
        if (j > S_DIRECT_J)
            for (int e = s0 + t; e < s1; e += blockDim.x) cp_async8_hint(Stri + e, Sg + e, pol);
        cp_async_commit();
        pdl_wait();
        const double* Xg = ws + lay.X + X_base(L, i, r);
        if (!x_staged)
            for (int e = (la - 1) * j + t; e < lb * j; e += blockDim.x) cp_async8(Xs + e, Xg + e);
        cp_async_commit();
        cp_async_wait<0>();
    }
    __syncthreads();
    pdl_trigger_at<1>();
    const double* S = j > S_DIRECT_J ? Stri : Sg;
    const bool mono = g_combine_early_exit && (reinterpret_cast<const int*>(ws + lay.smono)[slot] & 1);
    if (j >= 4) combine_tiles_s<4, COMBINE_TL4>(Wi, i, r, L, j, S, trio, Xs, s_hist, s_order, part, nparts, lA, lB, atomic, mono);
    else if (j >= 2) combine_tiles_s<2, 4 * COMBINE_TL4 / 2>(Wi, i, r, L, j, S, trio, Xs, s_hist, s_order, part, nparts, lA, lB, atomic, mono);
    else combine_tiles_s<1, 8 * COMBINE_TL4 / 2>(Wi, i, r, L, j, S, trio, Xs, s_hist, s_order, part, nparts, lA, lB, atomic, mono);
}

__global__ void __launch_bounds__(256, 2) k_combine_s(pp_batch b, int j) {
    const pp_instance I = b.inst[blockIdx.x];
    extern __shared__ __align__(16) double cs_smem[];
    __shared__ int s_hist[SR_MAX + 2];
    __shared__ int s_order[1024];
    combine_item_s(b, I, j, blockIdx.y + 1, blockIdx.z, gridDim.z, cs_smem, s_hist, s_order, false);
}
__global__ void __launch_bounds__(256, COMBINE_MINB) k_combine_s_p(const pp_batch* __restrict__ bp, int j, int r0) {
    pdl_trigger_at<0>();
    StepTrace tr;
    tr.begin();
    const pp_batch b = *bp;
    const pp_instance I = b.inst[blockIdx.x];
    extern __shared__ __align__(16) double cs_smem[];
    __shared__ int s_hist[SR_MAX + 2];
    __shared__ int s_order[1024];
    combine_item_s(b, I, j, blockIdx.y + r0, blockIdx.z, gridDim.z, cs_smem, s_hist, s_order, false, 1, PP_MAX_LAYERS,
                   false, g_combine_bulk);
    pdl_trigger_at<2>();
    tr.end(2, j);
}

// ----------------------------------------------------------------------------
// Backtrack: re-derive the reference's first-found realizing (l', r') of a
// cell (partition.py:126-141 loop order, strict `best > w`).  The candidate
// values are w(l', r') = max(W_j(l', xi-1, r'), chan(l', r'), stage(l')) and
// min over r' of w(l', .) = max(X(l', xi), stage(l')) exactly, so the
// lexicographically first (l', r') achieving the cell value is: the first
// l' with max(X(l'), stage(l')) == W (X is the stored expansion the DP
// used), then the first r' with w(l', r') == W.  Warp-cooperative.
// ----------------------------------------------------------------------------
__device__ __forceinline__ int warp_first(bool match) {
    const unsigned mask = __ballot_sync(0xffffffffu, match);
    return mask ? __ffs(mask) - 1 : -1;
}

constexpr int WALK_U = 4;
__device__ void dp_walk(const pp_batch& b, const pp_instance& I, int l, int x, int r, int i, double w,
                        int* o_ls, int* o_le, int* o_dlo, int* o_dhi) {
    const int L = I.L, V = I.V, M = I.M;
    const WsLayout lay = ws_layout(L, V);
    const double* ws = b.ws + I.ws_off;
    const double* prefix = ws + lay.prefix;
    const double* psum = ws + lay.psum;
    const double* minpair = ws + lay.minpair;
    const double* cross = ws + lay.cross;
    const double* W = ws + lay.W;
    const bool allow = I.flags & PP_ALLOW_REPLICATION;
    const int lane = threadIdx.x & 31;
    // Shared-memory-path batches hold every stage term in the k_stab triangles and
    // the chan quotients of multi-row payload classes in k_base's tables (the same
    // expressions, so lookups give the bits the divisions would).  The walk does
    // not use them: a table lookup is two dependent global loads (slot / class id,
    // then the entry) where the scalar expression's operands are one independent
    // round, and the walk is a chain of such rounds (C3 n = 1: ~63 stages).
    const bool tables = false;
    const int* sidx = reinterpret_cast<const int*>(ws + lay.sidx);
    const int* rcls = reinterpret_cast<const int*>(ws + lay.chcls + CHAN_CLS);
    const int64_t tri = (int64_t)(L - 1) * L / 2, tcls = (int64_t)tet(V);
    while (x >= 2) {
        const int j = i - r;
        const double* X = ws + lay.X + X_base(L, i, r);
        // slot -1: the batch built no triangle for this item (k_dp_inst2 computes
        // its triangles in shared memory): the scalar stage_term, same expression
        const int slot = tables ? sidx[(r - 1) * V + (i - 1)] : -1;
        const double* St = slot >= 0 ? ws + lay.Stab + (int64_t)slot * tri : nullptr;
        // the candidates of a stage are scanned WALK_U x 32 at a time with all their
        // loads in flight (one memory round trip per chunk instead of per 32)
        int lp = -1;
        for (int base = x - 1; base <= l - 1 && lp < 0; base += 32 * WALK_U) {
            bool match[WALK_U];
#pragma unroll
            for (int u = 0; u < WALK_U; ++u) {
                const int c = base + 32 * u + lane;
                match[u] = false;
                if (c <= l - 1) {
                    const double stc = St ? St[(c - 1) * L - (c - 1) * c / 2 + (l - c - 1)]
                                          : stage_term(M, L, V, prefix, psum, minpair, c, l, r, i);
                    match[u] = dmax(X[(int64_t)(c - 1) * j + (x - 2)], stc) == w;
                }
            }
#pragma unroll
            for (int u = 0; u < WALK_U; ++u) {
                const int f = warp_first(match[u]);
                if (lp < 0 && f >= 0) lp = base + 32 * u + f;
            }
        }
        int rp = -1;
        double w_next = PP_INF;   // W(lp, x-1, rp, j): the next stage's target, from the winning lane
        if (lp > 0) {
            const double st = St ? St[(lp - 1) * L - (lp - 1) * lp / 2 + (l - lp - 1)]
                                 : stage_term(M, L, V, prefix, psum, minpair, lp, l, r, i);
            const double Mp = (double)M * (b.efwd[I.layer_off + lp - 1] + b.ebwd[I.layer_off + lp - 1]);
            const int cls = tables ? rcls[lp] : -1;
            const double* Tj = cls >= 0 ? ws + lay.chan + cls * tcls + chan_step(V, j) : nullptr;
            for (int base = 1; base <= j && rp < 0; base += 32 * WALK_U) {
                bool match[WALK_U];
                double sub[WALK_U];
#pragma unroll
                for (int u = 0; u < WALK_U; ++u) {
                    const int c = base + 32 * u + lane;
                    match[u] = false;
                    sub[u] = PP_INF;
                    if (c <= j) {
                        sub[u] = W_at(W, L, j, lp, c, x - 1, allow);
                        const double chan = Tj ? Tj[(c - 1) * (V - j) + (r - 1)]
                                               : Mp / ((double)(c * r) * cross[cross_idx(V, i, r, c)]);
                        match[u] = dmax(dmax(sub[u], chan), st) == w;
                    }
                }
#pragma unroll
                for (int u = 0; u < WALK_U; ++u) {
                    const int f = warp_first(match[u]);
                    const double sw = __shfl_sync(0xffffffffu, sub[u], f < 0 ? 0 : f);
                    if (rp < 0 && f >= 0) { rp = base + 32 * u + f; w_next = sw; }
                }
            }
        }
        if (rp < 0) {   // cannot happen for a consistent table; leave a detectable hole
            if (lane == 0) { o_ls[x - 1] = 0; o_le[x - 1] = 0; o_dlo[x - 1] = 0; o_dhi[x - 1] = 0; }
            return;
        }
        if (lane == 0) { o_ls[x - 1] = lp + 1; o_le[x - 1] = l; o_dlo[x - 1] = i - r + 1; o_dhi[x - 1] = i; }
        w = w_next;   // == W_at(W, L, j, lp, rp, x - 1, allow)
        l = lp; i = j; r = rp; --x;
    }
    if (lane == 0) { o_ls[0] = 1; o_le[0] = l; o_dlo[0] = 1; o_dhi[0] = i; }
}

// best_partition(xi) for every xi (partition.py:144-162).  grid (n_inst, maxV), block 32.
// one warp: best W(L, xi, r, V) over r and its plan's stages (partition.py:144-162)
__device__ __forceinline__ void backtrack_xi(const pp_batch& b, const pp_instance& I, int xi) {
    const int L = I.L, V = I.V;
    if (xi > V) return;
    const WsLayout lay = ws_layout(L, V);
    const double* W = b.ws + I.ws_off + lay.W;
    const int lane = threadIdx.x & 31;
    double best = PP_INF;
    int br = 0;
    for (int r = 1 + lane; r <= V; r += 32) {
        const double v = (xi <= L) ? W_at(W, L, V, L, r, xi, I.flags & PP_ALLOW_REPLICATION) : PP_INF;
        if (v < best) { best = v; br = r; }   // ascending r per lane: first r on ties
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, off);
        const int orr = __shfl_xor_sync(0xffffffffu, br, off);
        if (ov < best || (ov == best && orr != 0 && (br == 0 || orr < br))) { best = ov; br = orr; }
    }
    const int64_t so = I.sweep_off + xi - 1;
    if (lane == 0) { b.sweep_w[so] = best; b.sweep_r[so] = br; }
    if (br == 0) return;
    const int64_t st = I.stage_off + (int64_t)xi * (xi - 1) / 2;
    dp_walk(b, I, L, xi, br, V, best, b.stage_ls + st, b.stage_le + st, b.stage_dlo + st, b.stage_dhi + st);
}
__device__ __forceinline__ void backtrack_body(const pp_batch& b) {
    const pp_instance I = b.inst[blockIdx.x];
    backtrack_xi(b, I, blockIdx.y + 1);
}
__global__ void __launch_bounds__(32) k_backtrack(pp_batch b) { backtrack_body(b); }
__global__ void __launch_bounds__(32) k_backtrack_p(const pp_batch* __restrict__ bp) {
    const pp_batch b = *bp;
    backtrack_body(b);
}

// PartitionSolver.solve queries (partition.py:95-142).  One warp per query.
__global__ void __launch_bounds__(32) k_query(pp_batch b, int n, const int* qi, const int* ql, const int* qx,
                                              const int* qr, const int* qd, int max_xi, double* w, int* frag,
                                              int* feas) {
    const int q = blockIdx.x;
    if (q >= n) return;
    const pp_instance I = b.inst[qi[q]];
    const int l = ql[q], x = qx[q], r = qr[q], i = qd[q];
    const WsLayout lay = ws_layout(I.L, I.V);
    const double* W = b.ws + I.ws_off + lay.W;
    double v = PP_INF;
    if (x <= i && r <= i) v = W_at(W, I.L, i, l, r, x, I.flags & PP_ALLOW_REPLICATION);
    const int lane = threadIdx.x;
    // Base cells (xi = 1, r = i) are feasible with any value; others iff finite
    // (an infinite candidate never passes `best > w`, partition.py:139).
    const bool f = (x == 1 && r == i && x <= i) ? (v == v && (I.flags & PP_ALLOW_REPLICATION || i == 1)) : (v < PP_INF);
    if (lane == 0) { w[q] = v; feas[q] = f ? 1 : 0; }
    if (!f) return;
    int* fr = frag + (int64_t)q * 4 * max_xi;
    // fragments stored interleaved (ls, le, dlo, dhi) per stage: use strided views
    __shared__ int s_ls[PP_MAX_GPUS], s_le[PP_MAX_GPUS], s_dlo[PP_MAX_GPUS], s_dhi[PP_MAX_GPUS];
    dp_walk(b, I, l, x, r, i, v, s_ls, s_le, s_dlo, s_dhi);
    __syncwarp();
    for (int n2 = lane; n2 < x; n2 += 32) {
        fr[4 * n2 + 0] = s_ls[n2]; fr[4 * n2 + 1] = s_le[n2]; fr[4 * n2 + 2] = s_dlo[n2]; fr[4 * n2 + 3] = s_dhi[n2];
    }
}

}  // namespace pp

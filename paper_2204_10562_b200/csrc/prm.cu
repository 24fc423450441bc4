// prm.cu — device ordering (RDO), DP tables and the PRM dynamic program.
//
// Reference: ordering.py:30-113 (Stoer-Wagner RDO), partition.py:41-162
// (W(l, xi, r, i) recursion), cost.py:64-99 (bandwidth minima, AllReduce).
//
// The DP runs as a wavefront over the device prefix i (W(., ., ., i) needs
// only slices j < i, partition.py:133).  The reference's candidate
//     w(l', r') = max(W(l', xi-1, r', j), chan(l', r'), stage(l'))
// is evaluated in factored form (bit-exact: max/min are exact and monotone):
//   expand(j):  X(l', xi, r, j+r) = min_{r'} max(W_j(l', xi-1, r'), chan(l', r', r, j+r))
//   combine(i): W_i(l, r, xi)     = min_{l'} max(X(l', xi, r, i), stage(l', l, r, i))
// Both are (min, max)-semiring matrix products; each CTA computes a 32x32
// output tile from smem-staged 32x32 operand tiles, 4x2 / 2x4 register
// micro-tiles per thread.  Arg-mins are not stored: the backtrack re-derives
// the reference's first-found (l', r') for the few cells on each chosen path.
#include "common.cuh"

namespace pp {

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
__global__ void __launch_bounds__(128) k_prep(pp_batch b) {
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
    // cross table for i = row: thread per r in [1, i-1], sequential over rp
    const int i = row;
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
}

// ----------------------------------------------------------------------------
// (min, max) micro-kernel shared by expand and combine: a thread owns a 4x4
// register tile of outputs and folds one K index per step,
//     acc[a][c] = min(acc[a][c], max(p[a], q[c])),
// p from a 4-wide slice of the "row" operand and q from the "column" operand,
// both read from shared memory as two LDS.128 each.  Every output's K range
// is trimmed to where its candidates can be finite (the triangular l' < l and
// r' <= j - xi + 2 structure), so padded INF candidates are not evaluated.
// ----------------------------------------------------------------------------
constexpr int KC = 32;   // K chunk staged per __syncthreads

__device__ __forceinline__ void mm_step(double (&acc)[4][4], const double* prow, const double* qrow) {
    const double2 p01 = *reinterpret_cast<const double2*>(prow);
    const double2 p23 = *reinterpret_cast<const double2*>(prow + 2);
    const double2 q01 = *reinterpret_cast<const double2*>(qrow);
    const double2 q23 = *reinterpret_cast<const double2*>(qrow + 2);
    const double p[4] = {p01.x, p01.y, p23.x, p23.y};
    const double q[4] = {q01.x, q01.y, q23.x, q23.y};
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[a][c] = dmin(acc[a][c], dmax(p[a], q[c]));
}

// ----------------------------------------------------------------------------
// k_expand(j): once slice j is final, X(l', xi, r, i = j + r) for every target,
//   X = min_{r' <= j} max(W_j(l', xi-1, r'), chan(l', r', r, i)),
//   chan = (M * payload(l')) / ((r' * r) * cross(r', r, i))   (partition.py:130-138)
// grid (n_inst, maxL-1, planes): one CTA per (instance, l', 64 xi x 64 r plane).
// ----------------------------------------------------------------------------
constexpr int EX_T = 128, EX_P = 64, EX_S = EX_P + 4;

__global__ void __launch_bounds__(EX_T) k_expand(pp_batch b, int j, int planes_r) {
    const pp_instance I = b.inst[blockIdx.x];
    const int L = I.L, V = I.V;
    const int lp = blockIdx.y + 1;
    if (j >= V || lp > L - 1) return;
    const int xi0 = 2 + EX_P * (int)(blockIdx.z / planes_r), r0 = 1 + EX_P * (int)(blockIdx.z % planes_r);
    const int nxi = min(EX_P, j + 2 - xi0), nr = min(EX_P, V - j + 1 - r0);
    if (nxi <= 0 || nr <= 0) return;
    const WsLayout lay = ws_layout(L, V);
    double* ws = b.ws + I.ws_off;
    const double* Wj = ws + lay.W;
    const double* cross = ws + lay.cross;
    const double Mp = (double)I.M * (b.efwd[I.layer_off + lp - 1] + b.ebwd[I.layer_off + lp - 1]);   // partition.py:131,137
    __shared__ __align__(16) double As[KC][EX_S];   // [r'][xi - xi0]  W_j(l', xi-1, r')
    __shared__ __align__(16) double Bs[KC][EX_S];   // [r'][r - r0]    chan(l', r', r, j+r)
    const int t = threadIdx.x;
    const int ntx = (nxi + 3) >> 2, ntr = (nr + 3) >> 2, ntiles = ntx * ntr;
    const int wx = ntx * 4, wr = ntr * 4;
    // up to two 4x4 tiles per thread
    int tx[2], tr[2], kend[2];
    double acc[2][4][4];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const int id = t + u * EX_T;
        tx[u] = (id < ntiles) ? id % ntx : -1;
        tr[u] = (id < ntiles) ? id / ntx : 0;
        // candidates need r' <= j - xi + 2; the tile's smallest xi bounds its K range
        kend[u] = (id < ntiles) ? j - (xi0 + 4 * tx[u]) + 2 : 0;
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[u][a][c] = PP_INF;
    }
    const int kmax = j - xi0 + 2;   // largest r' any output of the plane needs
    for (int rp0 = 1; rp0 <= kmax; rp0 += KC) {
        const int kc = min(KC, kmax - rp0 + 1);
        for (int e = t; e < kc * wx; e += EX_T) {
            const int rr = e / wx, cc = e - rr * wx;
            const int xi = xi0 + cc;
            As[rr][cc] = (cc < nxi) ? Wj[W_idx(L, j, lp, rp0 + rr, xi - 1)] : PP_INF;
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
            for (int kk = 0; kk < kk_end; ++kk) mm_step(acc[u], &As[kk][4 * tx[u]], &Bs[kk][4 * tr[u]]);
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
// partition.py:127-129, cost.py:99.
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
// k_combine(i): slice W_i(l, r, xi) = min_{l'} max(X(l', xi, r, i), stage(l', l, r, i)).
// grid (n_inst, i, planes): one CTA per (instance, r, 128 l x 64 xi plane);
// r = 1 (the largest j) comes first in launch order.
// ----------------------------------------------------------------------------
constexpr int CB_T = 256, CB_L = 128, CB_X = 64;
constexpr size_t CB_SMEM = sizeof(double) * KC * (CB_X + 4 + CB_L + 4);

__global__ void __launch_bounds__(CB_T, 2) k_combine(pp_batch b, int i, int planes_x) {
    const pp_instance I = b.inst[blockIdx.x];
    const int L = I.L, V = I.V, M = I.M;
    const int r = blockIdx.y + 1;
    if (i > V || r > i) return;
    const int l0 = 1 + CB_L * (int)(blockIdx.z / planes_x), x0 = 1 + CB_X * (int)(blockIdx.z % planes_x);
    if (l0 > L || x0 > i) return;
    const int nl = min(CB_L, L - l0 + 1), nx = min(CB_X, i - x0 + 1);
    const bool allow = I.flags & PP_ALLOW_REPLICATION;
    const WsLayout lay = ws_layout(L, V);
    double* ws = b.ws + I.ws_off;
    const double* prefix = ws + lay.prefix;
    const double* psum = ws + lay.psum;
    const double* minpair = ws + lay.minpair;
    double* Wi = ws + lay.W + W_base(L, i);
    const int t = threadIdx.x;
    const int j = i - r;
    // computed columns: xi in [cA, cB]; every other cell of the block is +inf
    const int cA = max(x0, 2), cB = min(x0 + nx - 1, j + 1);
    const bool dp_cells = r < i && (allow || r == 1) && cA <= cB;
    const int ncol = dp_cells ? cB - cA + 1 : 0;
    const int ntx = (ncol + 3) >> 2, ntl = (nl + 3) >> 2, ntiles = dp_cells ? ntx * ntl : 0;
    // fill the cells no tile writes: base row (r == i), xi = 1, xi > j + 1, disabled widths
    for (int e = t; e < nl * nx; e += CB_T) {
        const int l = l0 + e / nx, xi = x0 + e % nx;
        if (dp_cells && xi >= cA && xi < cA + 4 * ntx) continue;
        double v = PP_INF;
        if (r == i && xi == 1 && (allow || i == 1)) {
            // partition.py:117-119: M * span(1, l) / i + sync(1, l, 1, i)
            double sync = 0.0;
            if (i > 1) sync = 2.0 * (double)(i - 1) * psum[l - 1] / ((double)i * minpair[i - 1]);
            v = (double)M * (prefix[l] - prefix[0]) / (double)i + sync;
        }
        Wi[((int64_t)(l - 1) * i + (r - 1)) * i + (xi - 1)] = v;
    }
    if (!dp_cells) return;

    const double* X = ws + lay.X + X_base(L, i, r);
    extern __shared__ __align__(16) double cb_smem[];
    double (*Xs)[CB_X + 4] = reinterpret_cast<double (*)[CB_X + 4]>(cb_smem);              // [l' - lp0][xi - cA]
    double (*Ss)[CB_L + 4] = reinterpret_cast<double (*)[CB_L + 4]>(cb_smem + KC * (CB_X + 4));   // [l' - lp0][l - l0]
    const int wx = ntx * 4, wl = ntl * 4;
    int ti[2], tj[2], kbeg[2], kend[2];
    double acc[2][4][4];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const int id = t + u * CB_T;
        ti[u] = (id < ntiles) ? id / ntx : -1;   // row tile (l)
        tj[u] = (id < ntiles) ? id % ntx : 0;    // column tile (xi)
        // candidates need l' >= xi - 1 (X is +inf below) and l' <= l - 1
        kbeg[u] = max(1, cA + 4 * tj[u] - 1);
        kend[u] = min(L - 1, l0 + 4 * ti[u] + 2);
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[u][a][c] = PP_INF;
    }
    const int kmin = max(1, cA - 1), kmax = min(L - 1, l0 + nl - 2);
    const double mp = minpair[(int64_t)(i - r) * V + (i - 1)];
    for (int lp0 = kmin; lp0 <= kmax; lp0 += KC) {
        const int kc = min(KC, kmax - lp0 + 1);
        for (int e = t; e < kc * wx; e += CB_T) {
            const int rr = e / wx, cc = e - rr * wx;
            Xs[rr][cc] = (cc < ncol) ? X[(int64_t)(lp0 + rr - 1) * j + (cA + cc - 2)] : PP_INF;
        }
        for (int e = t; e < kc * wl; e += CB_T) {
            const int rr = e / wl, cc = e - rr * wl;
            const int lp = lp0 + rr, l = l0 + cc;
            double s = PP_INF;
            if (cc < nl && lp < l) {
                s = (double)M * (prefix[l] - prefix[lp]) / (double)r;
                if (r > 1) s += 2.0 * (double)(r - 1) * psum[(int64_t)lp * L + (l - 1)] / ((double)r * mp);
            }
            Ss[rr][cc] = s;
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            if (ti[u] < 0) continue;
            const int k0 = max(0, kbeg[u] - lp0), k1 = min(kc, kend[u] - lp0 + 1);
            for (int kk = k0; kk < k1; ++kk) mm_step(acc[u], &Ss[kk][4 * ti[u]], &Xs[kk][4 * tj[u]]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        if (ti[u] < 0) continue;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const int l = l0 + 4 * ti[u] + a;
            if (l > L) continue;
            double* row = Wi + ((int64_t)(l - 1) * i + (r - 1)) * i;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int xi = cA + 4 * tj[u] + c;
                if (xi < x0 + nx) row[xi - 1] = acc[u][a][c];
            }
        }
    }
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
    const int lane = threadIdx.x & 31;
    while (x >= 2) {
        const int j = i - r;
        const double* X = ws + lay.X + X_base(L, i, r);
        int lp = -1;
        for (int base = x - 1; base <= l - 1 && lp < 0; base += 32) {
            const int c = base + lane;
            bool match = false;
            if (c <= l - 1)
                match = dmax(X[(int64_t)(c - 1) * j + (x - 2)],
                             stage_term(M, L, V, prefix, psum, minpair, c, l, r, i)) == w;
            const int f = warp_first(match);
            if (f >= 0) lp = base + f;
        }
        int rp = -1;
        if (lp > 0) {
            const double st = stage_term(M, L, V, prefix, psum, minpair, lp, l, r, i);
            const double Mp = (double)M * (b.efwd[I.layer_off + lp - 1] + b.ebwd[I.layer_off + lp - 1]);
            for (int base = 1; base <= j && rp < 0; base += 32) {
                const int c = base + lane;
                bool match = false;
                if (c <= j) {
                    const double sub = W[W_idx(L, j, lp, c, x - 1)];
                    const double chan = Mp / ((double)(c * r) * cross[cross_idx(V, i, r, c)]);
                    match = dmax(dmax(sub, chan), st) == w;
                }
                const int f = warp_first(match);
                if (f >= 0) rp = base + f;
            }
        }
        if (rp < 0) {   // cannot happen for a consistent table; leave a detectable hole
            if (lane == 0) { o_ls[x - 1] = 0; o_le[x - 1] = 0; o_dlo[x - 1] = 0; o_dhi[x - 1] = 0; }
            return;
        }
        if (lane == 0) { o_ls[x - 1] = lp + 1; o_le[x - 1] = l; o_dlo[x - 1] = i - r + 1; o_dhi[x - 1] = i; }
        w = W[W_idx(L, j, lp, rp, x - 1)];
        l = lp; i = j; r = rp; --x;
    }
    if (lane == 0) { o_ls[0] = 1; o_le[0] = l; o_dlo[0] = 1; o_dhi[0] = i; }
}

// best_partition(xi) for every xi (partition.py:144-162).  grid (n_inst, maxV), block 32.
__global__ void __launch_bounds__(32) k_backtrack(pp_batch b) {
    const pp_instance I = b.inst[blockIdx.x];
    const int xi = blockIdx.y + 1;
    const int L = I.L, V = I.V;
    if (xi > V) return;
    const WsLayout lay = ws_layout(L, V);
    const double* W = b.ws + I.ws_off + lay.W;
    const int lane = threadIdx.x;
    double best = PP_INF;
    int br = 0;
    for (int r = 1 + lane; r <= V; r += 32) {
        const double v = (xi <= L) ? W[W_idx(L, V, L, r, xi)] : PP_INF;
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
    if (x <= i && r <= i) v = W[W_idx(I.L, i, l, r, x)];
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

// ----------------------------------------------------------------------------
// RDO (ordering.py:30-113).  One CTA per instance; each warp runs the
// Stoer-Wagner min cut of one vertex group (a node of the recursion tree);
// groups of one recursion level are cut concurrently by different warps.
// A group is identified by its lowest rank `lo`; every vertex stores the lo
// of its current group, so the final rank of vertex v is lo[v].
//
// Inside a cut, vertex k of the group (k = position in the ascending member
// list, so local order == GPU-id order) lives on lane k % 32, register slot
// k / 32: adjacency, supernode and flags never touch memory.  The group's
// weights are a local n x n matrix (shared memory when the instance fits,
// else the instance's global scratch), rebuilt from the cluster for every
// cut as the reference does (ordering.py:50-54).  Arg-max per step: the
// adjacencies are positive doubles, which order like their uint64 bit
// patterns, so the max is two 32-bit __reduce_max_sync (high word, then low
// word among high-word winners) and the reference's smallest-id tie rule
// (ordering.py:66) is a __reduce_min_sync over the tied local indices.
// ----------------------------------------------------------------------------
template <int SLOTS>
__device__ double warp_min_cut_t(double* wl, const double* bw, int V, const int* mem, int n,
                                 unsigned char* side_out) {
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    for (int e = lane; e < n * n; e += 32) {
        const int a = e / n, c = e - a * n;
        wl[e] = (a == c) ? 0.0 : bw[(int64_t)mem[a] * V + mem[c]];
    }
    __syncwarp();
    double adj[SLOTS];
    int grp[SLOTS];
    bool alive[SLOTS], inadj[SLOTS], side[SLOTS];
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
        const int k = lane + 32 * s;
        alive[s] = k < n; grp[s] = k; side[s] = false; inadj[s] = false; adj[s] = 0.0;
    }
    double best_weight = PP_INF;
    for (int n_alive = n; n_alive > 1; --n_alive) {
#pragma unroll
        for (int s = 0; s < SLOTS; ++s) {   // phase starts at the smallest id (ordering.py:61-64)
            const int k = lane + 32 * s;
            inadj[s] = alive[s] && k != 0;
            if (inadj[s]) adj[s] = wl[k];
        }
        int sv = 0, tv = 0;
        double cut = 0.0;
        for (int step = 0; step < n_alive - 1; ++step) {
            unsigned long long bu = 0ull;
            int bk = 0x7fffffff;
#pragma unroll
            for (int s = 0; s < SLOTS; ++s) {
                const unsigned long long u = (unsigned long long)__double_as_longlong(adj[s]);
                if (inadj[s] && u > bu) { bu = u; bk = lane + 32 * s; }
            }
            const unsigned hi = (unsigned)(bu >> 32), lo = (unsigned)bu;
            const unsigned mhi = __reduce_max_sync(FULL, hi);
            const unsigned mlo = __reduce_max_sync(FULL, hi == mhi ? lo : 0u);
            const bool win = bk != 0x7fffffff && hi == mhi && lo == mlo;
            const int nk = (int)__reduce_min_sync(FULL, win ? (unsigned)bk : 0x7fffffffu);
            cut = __longlong_as_double((long long)(((unsigned long long)mhi << 32) | mlo));
            sv = tv; tv = nk;
            const double* row = wl + nk * n;
#pragma unroll
            for (int s = 0; s < SLOTS; ++s) {   // adj[u] += wt(next_v, u)  (ordering.py:69-70)
                const int k = lane + 32 * s;
                if (k == nk) inadj[s] = false;
                if (inadj[s]) adj[s] = adj[s] + row[k];
            }
        }
        if (cut < best_weight) {   // first minimum cut-of-phase (ordering.py:73-75)
            best_weight = cut;
#pragma unroll
            for (int s = 0; s < SLOTS; ++s) side[s] = (grp[s] == tv);
        }
        const int merged = min(sv, tv), other = max(sv, tv);   // ordering.py:77-85
#pragma unroll
        for (int s = 0; s < SLOTS; ++s) {
            const int u = lane + 32 * s;
            if (alive[s] && u != sv && u != tv) {
                const double x = wl[sv * n + u] + wl[tv * n + u];
                wl[merged * n + u] = x;
                wl[u * n + merged] = x;
            }
        }
        __syncwarp();
#pragma unroll
        for (int s = 0; s < SLOTS; ++s) {
            if (grp[s] == other) grp[s] = merged;
            if (lane + 32 * s == other) alive[s] = false;
        }
    }
    // the side holding the smallest id becomes side_a (ordering.py:87-91)
    const bool low = __shfl_sync(FULL, side[0], 0);
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
        const int k = lane + 32 * s;
        if (k < n) side_out[k] = low ? side[s] : !side[s];
    }
    __syncwarp();
    return best_weight;
}

__device__ double warp_min_cut(double* wl, const double* bw, int V, const int* mem, int n, unsigned char* side) {
    if (n <= 32) return warp_min_cut_t<1>(wl, bw, V, mem, n, side);
    if (n <= 64) return warp_min_cut_t<2>(wl, bw, V, mem, n, side);
    if (n <= 128) return warp_min_cut_t<4>(wl, bw, V, mem, n, side);
    if (n <= 256) return warp_min_cut_t<8>(wl, bw, V, mem, n, side);
    return warp_min_cut_t<16>(wl, bw, V, mem, n, side);
}

__global__ void __launch_bounds__(32 * RDO_WARPS) k_rdo(pp_batch b, int w_in_smem) {
    const pp_instance I = b.inst[blockIdx.x];
    if (I.flags & PP_GIVEN_ORDER) return;
    const int V = I.V;
    extern __shared__ double smem_d[];
    char* sm = (char*)smem_d;
    double* W;
    if (w_in_smem) { W = (double*)sm; sm += sizeof(double) * V * V; }
    else W = b.ws + I.ws_off + ws_layout(I.L, V).rdo_w;
    int* lo = (int*)sm;      sm += sizeof(int) * V;
    int* cnt = (int*)sm;     sm += sizeof(int) * V;
    int* first = (int*)sm;   sm += sizeof(int) * V;
    int* glist = (int*)sm;   sm += sizeof(int) * V;
    int* goff = (int*)sm;    sm += sizeof(int) * V;
    int* memall = (int*)sm;  sm += sizeof(int) * V * RDO_WARPS;
    unsigned char* sideall = (unsigned char*)sm;
    const double* bw = b.bw + I.bw_off;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    for (int v = t; v < V; v += blockDim.x) lo[v] = 1;
    __syncthreads();
    __shared__ int s_ngroups;
    for (;;) {
        for (int v = t; v < V; v += blockDim.x) { cnt[v] = 0; first[v] = 0x7fffffff; }
        if (t == 0) s_ngroups = 0;
        __syncthreads();
        for (int v = t; v < V; v += blockDim.x) { atomicAdd(&cnt[lo[v] - 1], 1); atomicMin(&first[lo[v] - 1], v); }
        __syncthreads();
        for (int v = t; v < V; v += blockDim.x) {
            const int g = lo[v];
            if (cnt[g - 1] >= 2 && first[g - 1] == v) glist[atomicAdd(&s_ngroups, 1)] = g;
        }
        __syncthreads();
        const int ng = s_ngroups;
        if (ng == 0) break;
        if (t == 0) {   // disjoint groups: sum of n^2 <= V^2 fits the V x V region
            int o = 0;
            for (int gi = 0; gi < ng; ++gi) { goff[gi] = o; const int c = cnt[glist[gi] - 1]; o += c * c; }
        }
        __syncthreads();
        for (int gi = warp; gi < ng; gi += RDO_WARPS) {
            const int g = glist[gi];
            int* mem = memall + warp * V;
            unsigned char* side = sideall + warp * V;
            int n = 0;
            for (int v0 = 0; v0 < V; v0 += 32) {   // ascending member list
                const int v = v0 + lane;
                const bool in = v < V && lo[v] == g;
                const unsigned m = __ballot_sync(0xffffffffu, in);
                if (in) mem[n + __popc(m & ((1u << lane) - 1))] = v;
                n += __popc(m);
            }
            __syncwarp();
            warp_min_cut(W + goff[gi], bw, V, mem, n, side);
            int na = 0;
            for (int k0 = 0; k0 < n; k0 += 32) {
                const int k = k0 + lane;
                na += __popc(__ballot_sync(0xffffffffu, k < n && side[k]));
            }
            for (int k = lane; k < n; k += 32) lo[mem[k]] = side[k] ? g : g + na;
            __syncwarp();
        }
        __syncthreads();
    }
    int* order = b.order + I.order_off;
    for (int v = t; v < V; v += blockDim.x) order[lo[v] - 1] = v;
}

// global_min_cut on a vertex subset (ordering.py:30-91): one warp.
__global__ void __launch_bounds__(32) k_min_cut(pp_batch b, int k, const int* verts, int n, unsigned char* in_a,
                                                double* weight, int w_in_smem) {
    const pp_instance I = b.inst[k];
    const int V = I.V;
    extern __shared__ double smem_d[];
    char* sm = (char*)smem_d;
    double* W;
    if (w_in_smem) { W = (double*)sm; sm += sizeof(double) * V * V; }
    else W = b.ws + I.ws_off + ws_layout(I.L, V).rdo_w;
    int* mem = (int*)sm;
    for (int q = threadIdx.x; q < n; q += 32) mem[q] = verts[q];
    __syncwarp();
    const double cw = warp_min_cut(W, b.bw + I.bw_off, V, mem, n, in_a);
    if (threadIdx.x == 0) weight[0] = cw;
}

}  // namespace pp

// combine_bis.cu — the combine step as a per-cell crossing search.
//
// Reference: partition.py:123-142 (_solve_uncached), factored as in DESIGN.md
// §2: for the item (r, i = j + r) and column xi,
//     W(l, xi, r, i) = min_{l' in [xi-1, l-1]} max(X(l', xi), S(l', l)),
// X(l', xi) = min_{r'} max(W_j(l', xi-1, r'), chan(l', r', r, i)) (the expand),
// S(l', l) the stage term of layers l'+1..l on the item's last r devices.
//
// When the stage-term triangle is certified non-increasing in l' (k_stab flag
// bit 0) and the X column is non-decreasing in l' (checked here on the
// rounded values), the candidate f(l') = max(X(l'), S(l', l)) is valley-shaped:
// with p* the first l' where X(l') >= S(l', l),
//     l' >= p*:  f = X(l') >= X(p*)          (X rises, and dominates S)
//     l' <  p*:  f = S(l', l) >= S(p*-1, l)  (S falls, and dominates X)
// so the minimum over the whole range is EXACTLY min(X(p*), S(p*-1, l)) — the
// same value, bit for bit, as the exhaustive min (min/max only select).  p* is
// found by a branch-free bisection (ceil(log2(l - xi + 1)) + 1 probes).
// A column that is NOT monotone is handled through its suffix minima
//     g_l(p) = min X(p..l-1),
// non-decreasing in p: a candidate l' is dominated by any later l'' <= l-1 with
// X(l'') <= X(l') (both terms of its max are >= those of l''), so
//     min_{l'} max(X(l'), S(l', l)) = min_p max(g_l(p), S(p, l)),
// again a valley, bisected the same way.  X is non-decreasing between its
// descents d (X(d+1) < X(d)), so g_l(p) = min(X(p), X(d+1) : p <= d <= l-2),
// a value of X bit for bit; the certificate pass records up to CB_DESC
// descents per column (columns with more, or triangles without bit 0, fold
// the candidates: descending with the early exit when bit 0 holds, every l'
// otherwise).  The stored value is all the
// backtrack needs (it re-derives the reference's first-found arg-min).
//
// A CTA owns one item and a group of rows l in [l0, l1]: it stages only what
// those cells read — X rows 1..l1-1 (one TMA bulk copy) and the triangle
// columns S(., l) for its rows, gathered transposed (cp.async) so a cell's
// probes index one contiguous column — and checks the column certificates
// over the staged rows only (all its cells' candidate ranges lie there).
// One thread per cell; a warp's W stores are consecutive xi of one row.
// Small batches split an item over many row groups (the critical item of the
// split chain runs as L/8 CTAs), large ones use one group per item.
#include "common.cuh"

namespace pp {

constexpr int CB_T = 256;    // threads per CTA
constexpr int CB_DESC = 8;   // descents of an X column handled by the suffix-minimum bisection

// S(l', l) in the packed row-major triangle: row l' holds l = l'+1..L
__device__ __forceinline__ int tri_off(int L, int lp, int l) { return (lp - 1) * L - (lp - 1) * lp / 2 + (l - lp - 1); }

// dynamic shared memory of one CTA: X rows (L-1) x j, the group's triangle
// columns (sum of l - 1 over its rows <= min(rg (L-1), L (L-1)/2)), spare
__host__ __device__ __forceinline__ size_t combine_bis_smem_doubles(int L, int j, int rg) {
    const size_t lm = L > 1 ? L - 1 : 0;
    const size_t a = (size_t)rg * lm, b = (size_t)L * lm / 2;
    return lm * j + (a < b ? a : b) + 4;
}

__device__ __forceinline__ void combine_item_bis(const pp_batch& b, const pp_instance& I, int j, int r, int l0,
                                                 int rg, int rb, double* cs_smem) {
    const int L = I.L, V = I.V;
    if (j >= V || r > V - j || l0 > L) return;
    const int i = j + r;
    const bool allow = I.flags & PP_ALLOW_REPLICATION;
    if (!(allow || r == 1)) return;   // partition.py:103-104 (structural +inf, W_at)
    const int l1 = min(L, l0 + rg - 1), nrow = l1 - l0 + 1;
    const WsLayout lay = ws_layout(L, V);
    double* ws = b.ws + I.ws_off;
    double* Wi = ws + lay.W + W_base(L, i);
    const int t = threadIdx.x;
    const int ncol = min(j, L - 1);   // xi = 2..ncol+1 (xi <= L: cells l >= xi exist)
    __shared__ uint64_t s_bar[1];
    const int ns = (L - 1) * L / 2;
    const int slot = reinterpret_cast<const int*>(ws + lay.sidx)[(r - 1) * V + (i - 1)];
    const double* Sg = ws + lay.Stab + (int64_t)slot * ns;
    const double* Xg = ws + lay.X + X_base(L, i, r);
    // the group's triangle columns, packed: S(p, l) = Sc[co(l) + p - 1], p = 1..l-1,
    // co(l) = sum_{l0 <= l' < l} (l' - 1) = ((l-1)(l-2) - (l0-1)(l0-2)) / 2
    double* Sc = cs_smem;
    const int cob = (l0 - 1) * (l0 - 2) / 2 + 1;   // column base: Sc + (l-1)(l-2)/2 - cob, indexed by p
    double* Xs = cs_smem + (l1 * (l1 - 1) / 2 - (l0 - 1) * (l0 - 2) / 2) + 1;
    Xs += dphase(Xs) ^ dphase(Xg);
    const int nx = (min(l1, L) - 1) * j;   // X rows 1..l1-1
    if (t == 0) mbar_init(&s_bar[0]);
    __syncthreads();
    // the triangle was built before the wavefront: it streams in under PDL while
    // the expand drains; X (this step's expand) after the dependency wait
    {
        const uint64_t pol = l2_evict_last_policy();
        const int lane = t & 31, warp = t >> 5, nw = blockDim.x >> 5;
        for (int l = l0 + warp; l <= l1; l += nw) {
            double* col = Sc + ((l - 1) * (l - 2) / 2 - cob);
            for (int p = 1 + lane; p < l; p += 32) cp_async8_hint(col + p, Sg + tri_off(L, p, l), pol);
        }
        cp_async_commit();
    }
    const int sflags = reinterpret_cast<const int*>(ws + lay.smono)[slot];
    // g_combine_early_exit = 0 (pp_dp_set_early_exit): fold every l' (test knob)
    const bool s_dec = (sflags & 1) && g_combine_early_exit, s_inc = (sflags & 2) != 0;
    pdl_wait();
    stage_span(Xs, Xg, 0, nx, &s_bar[0], l2_evict_normal_policy());
    cp_async_wait<0>();
    mbar_wait0(&s_bar[0]);
    __syncthreads();
    pdl_trigger_at<1>();
    // column certificates: the descents d of X(., xi) over the staged rows
    // l' in [xi-1, l1-1] (X(d+1) < X(d)); none = monotone
    __shared__ unsigned char s_desc[SR_MAX][CB_DESC];
    __shared__ unsigned char s_ndesc[SR_MAX];   // 0..CB_DESC, or 255 = more
    {
        const int lane = t & 31, warp = t >> 5, nw = blockDim.x >> 5;
        for (int c = warp; c < ncol; c += nw) {
            const int xi = c + 2;
            int nd = s_dec ? 0 : 255;
            for (int lp0 = xi - 1; lp0 + 1 <= l1 - 1 && nd != 255; lp0 += 32) {
                const int lp = lp0 + lane;
                const bool dsc = lp + 1 <= l1 - 1 && !(Xs[lp * j + c] >= Xs[(lp - 1) * j + c]);
                const unsigned m = __ballot_sync(0xffffffffu, dsc);
                const int k = nd + __popc(m & ((1u << lane) - 1u));
                if (dsc && k < CB_DESC) s_desc[c][k] = (unsigned char)lp;
                nd += __popc(m);
                if (nd > CB_DESC) nd = 255;
            }
            if (lane == 0) s_ndesc[c] = (unsigned char)nd;
        }
    }
    __syncthreads();
    const int64_t ostride = (int64_t)i * i;
    // thread = (column, rb consecutive rows): the first row bisects, later rows of
    // a certified column gallop forward from the previous crossing when the
    // triangle is also non-decreasing in l (p*(l) >= p*(l-1)); rb = 1 for small
    // batches (latency: one cell per thread), 8 for large ones (work)
    const int nrb = (nrow + rb - 1) / rb;
    for (int u = t; u < nrb * ncol; u += blockDim.x) {
        const int c = u % ncol, la = l0 + (u / ncol) * rb, lz = min(l1, la + rb - 1);
        const int xi = c + 2;
        const int nd = s_ndesc[c];
        const bool cert = nd == 0;
        const double* Xc = Xs + c;   // X(l', xi) = Xc[(l'-1) * j]
        int pstar = -1;              // crossing of the previous row (gallop start)
        for (int l = la; l <= lz; ++l) {
            double w = PP_INF;
            if (l >= xi) {
                const int lo = xi - 1, hi = l - 1;
                const double* Sl = Sc + ((l - 1) * (l - 2) / 2 - cob);   // S(l', l) = Sl[l']
                if (cert) {
                    // first p in [lo, hi] with X(p) >= S(p, l) (hi + 1 if none)
                    int base = lo, n = hi - lo + 1;
                    if (s_inc && pstar >= 0) {
                        base = pstar;
                        n = hi - pstar + 1;
                        // gallop: probe pstar, pstar + 1, pstar + 3, ... (1 probe when it stays)
                        for (int step = 1; n > 0; step <<= 1) {
                            const int p = base + step - 1;
                            if (p > hi) break;
                            if (Xc[(p - 1) * j] >= Sl[p]) { n = step - 1; break; }
                            base = p + 1;
                            n = hi - base + 1;
                        }
                    }
                    while (n > 0) {   // branch-free lower bound over [base, base + n)
                        const int half = n >> 1, m = base + half;
                        const bool ge = Xc[(m - 1) * j] >= Sl[m];
                        base = ge ? base : m + 1;
                        n = ge ? half : n - half - 1;
                    }
                    pstar = base;
                    if (base <= hi) w = Xc[(base - 1) * j];
                    if (base > lo) w = dmin(w, Sl[base - 1]);
                } else if (nd != 255) {
                    // the same lower bound on the suffix minima g_l(p) = min(X(p), X(d+1) : p <= d <= l-2)
                    const unsigned char* dl = s_desc[c];
                    auto g = [&](int p) {
                        double v = Xc[(p - 1) * j];
                        for (int k = 0; k < nd; ++k) {
                            const int d = dl[k];
                            if (d >= p && d <= l - 2) v = dmin(v, Xc[d * j]);
                        }
                        return v;
                    };
                    int base = lo, n = hi - lo + 1;
                    while (n > 0) {
                        const int half = n >> 1, m = base + half;
                        const bool ge = g(m) >= Sl[m];
                        base = ge ? base : m + 1;
                        n = ge ? half : n - half - 1;
                    }
                    if (base <= hi) w = g(base);
                    if (base > lo) w = dmin(w, Sl[base - 1]);
                } else if (s_dec) {
                    // descending l': S only grows, stop once it reaches the running min
                    for (int p = hi; p >= lo; --p) {
                        const double sv = Sl[p];
                        if (sv >= w) break;
                        w = dmin(w, dmax(Xc[(p - 1) * j], sv));
                    }
                } else {
                    for (int p = lo; p <= hi; ++p) w = dmin(w, dmax(Xc[(p - 1) * j], Sl[p]));
                }
            }
            Wi[(int64_t)(l - 1) * ostride + (int64_t)(r - 1) * i + (xi - 1)] = w;
        }
    }
}

// one CTA per (instance, item r = r0 + blockIdx.y, rows 1 + rg * blockIdx.z ..), target i = j + r
__global__ void __launch_bounds__(CB_T, 2) k_combine_bis_p(const pp_batch* __restrict__ bp, int j, int r0, int rg,
                                                           int rb) {
    pdl_trigger_at<0>();
    StepTrace tr;
    tr.begin();
    const pp_batch b = *bp;
    const pp_instance I = b.inst[blockIdx.x];
    extern __shared__ __align__(16) double cs_smem[];
    combine_item_bis(b, I, j, blockIdx.y + r0, 1 + rg * (int)blockIdx.z, rg, rb, cs_smem);
    pdl_trigger_at<2>();
    tr.end(2, j);
}

}  // namespace pp

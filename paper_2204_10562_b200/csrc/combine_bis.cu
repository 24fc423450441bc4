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
// found by bisection; when the triangle is also non-decreasing in l (bit 1),
// p*(l) >= p*(l-1) and each cell gallops forward from its predecessor's p*.
// Columns or triangles without the certificate fold every l' (descending with
// the early exit of DESIGN.md §4.3 when bit 0 holds).  The stored value is all
// the backtrack needs (it re-derives the reference's first-found arg-min).
//
// Work per cell drops from (l - xi + 1) candidates to ~2-7 probes; a thread
// owns one column and CB_RB consecutive rows, so the W stores of a warp are
// consecutive xi of one row (coalesced).
#include "common.cuh"

namespace pp {

constexpr int CB_RB = 8;     // rows per thread (one column)
constexpr int CB_T = 256;    // threads per CTA

// S(l', l) in the packed triangle: row l' holds l = l'+1..L
__device__ __forceinline__ int tri_off(int L, int lp, int l) { return (lp - 1) * L - (lp - 1) * lp / 2 + (l - lp - 1); }

__device__ __forceinline__ void combine_item_bis(const pp_batch& b, const pp_instance& I, int j, int r,
                                                 double* cs_smem) {
    const int L = I.L, V = I.V;
    if (j >= V || r > V - j) return;
    const int i = j + r;
    const bool allow = I.flags & PP_ALLOW_REPLICATION;
    if (!(allow || r == 1)) return;   // partition.py:103-104 (structural +inf, W_at)
    const WsLayout lay = ws_layout(L, V);
    double* ws = b.ws + I.ws_off;
    double* Wi = ws + lay.W + W_base(L, i);
    const int t = threadIdx.x;
    const int ncol = min(j, L - 1);   // xi = 2..ncol+1 (xi <= L: cells l >= xi exist)
    __shared__ uint64_t s_bar[2];
    __shared__ unsigned char s_xmono[SR_MAX];
    const int ns = (L - 1) * L / 2;
    const int slot = reinterpret_cast<const int*>(ws + lay.sidx)[(r - 1) * V + (i - 1)];
    const double* Sg = ws + lay.Stab + (int64_t)slot * ns;
    const double* Xg = ws + lay.X + X_base(L, i, r);
    double* Stri = cs_smem;
    Stri += dphase(Stri) ^ dphase(Sg);
    double* Xs = cs_smem + 2 + ns;
    Xs += dphase(Xs) ^ dphase(Xg);
    if (t == 0) { mbar_init(&s_bar[0]); mbar_init(&s_bar[1]); }
    __syncthreads();
    // the triangle was built before the wavefront: it streams in under PDL while
    // the expand drains; X (this step's expand) after the dependency wait
    stage_span(Stri, Sg, 0, ns, &s_bar[0], l2_evict_last_policy());
    pdl_wait();
    stage_span(Xs, Xg, 0, (L - 1) * j, &s_bar[1], l2_evict_normal_policy());
    const int sflags = reinterpret_cast<const int*>(ws + lay.smono)[slot];
    // g_combine_early_exit = 0 (pp_dp_set_early_exit): fold every l' (test knob)
    const bool s_dec = (sflags & 1) && g_combine_early_exit, s_inc = (sflags & 2) != 0;
    mbar_wait0(&s_bar[0]);
    mbar_wait0(&s_bar[1]);
    __syncthreads();
    pdl_trigger_at<1>();
    // column certificates: X(., xi) non-decreasing over l' in [xi-1, L-1]
    {
        const int lane = t & 31, warp = t >> 5, nw = blockDim.x >> 5;
        for (int c = warp; c < ncol; c += nw) {
            const int xi = c + 2;
            bool bad = false;
            for (int lp = xi - 1 + lane; lp + 1 <= L - 1; lp += 32)
                bad |= !(Xs[lp * j + c] >= Xs[(lp - 1) * j + c]);   // rows l' = 1..L-1 at (l'-1)*j
            bad = __any_sync(0xffffffffu, bad);
            if (lane == 0) s_xmono[c] = !bad;
        }
    }
    __syncthreads();
    const int nrb = (L + CB_RB - 1) / CB_RB;
    for (int u = t; u < ncol * nrb; u += blockDim.x) {
        const int c = u % ncol, rb = u / ncol;
        const int xi = c + 2;
        const int l0 = 1 + rb * CB_RB, l1 = min(L, l0 + CB_RB - 1);
        const double* Xc = Xs + c;   // X(l', xi) = Xc[(l'-1) * j]
        double* out = Wi + (int64_t)(r - 1) * i + (xi - 1);   // W(l, xi, r, i) = out[(l-1) * i * i]
        const int64_t ostride = (int64_t)i * i;
        const bool bis = s_dec && s_xmono[c];
        int pstar = -1;   // p* of the previous cell (gallop start), -1 = none
        for (int l = l0; l <= l1; ++l) {
            double w = PP_INF;
            if (l >= xi) {
                const int lo = xi - 1, hi = l - 1;
                if (bis) {
                    // first p in [lo, hi] with X(p) >= S(p, l); hi + 1 if none
                    int a = lo, z = hi + 1;   // invariant: answer in [a, z]
                    if (s_inc && pstar >= 0) {
                        // p*(l) >= p*(l-1): gallop forward from it (1 probe when it stays)
                        a = pstar;
                        for (int step = 1;; step <<= 1) {
                            const int p = a + step - 1;
                            if (p > hi) break;
                            if (Xc[(p - 1) * j] >= Stri[tri_off(L, p, l)]) { z = p; break; }
                            a = p + 1;
                        }
                    }
                    while (a < z) {
                        const int m = (a + z) >> 1;
                        if (Xc[(m - 1) * j] >= Stri[tri_off(L, m, l)]) z = m;
                        else a = m + 1;
                    }
                    pstar = a;
                    if (a <= hi) w = Xc[(a - 1) * j];
                    if (a > lo) w = dmin(w, Stri[tri_off(L, a - 1, l)]);
                } else if (s_dec) {
                    // descending l': S only grows, stop once it reaches the running min
                    for (int p = hi; p >= lo; --p) {
                        const double s = Stri[tri_off(L, p, l)];
                        if (s >= w) break;
                        w = dmin(w, dmax(Xc[(p - 1) * j], s));
                    }
                } else {
                    for (int p = lo; p <= hi; ++p) w = dmin(w, dmax(Xc[(p - 1) * j], Stri[tri_off(L, p, l)]));
                }
            }
            out[(int64_t)(l - 1) * ostride] = w;
        }
    }
}

// one CTA per (instance, item r = r0 + blockIdx.y), target i = j + r
__global__ void __launch_bounds__(CB_T, 2) k_combine_bis_p(const pp_batch* __restrict__ bp, int j, int r0) {
    pdl_trigger_at<0>();
    StepTrace tr;
    tr.begin();
    const pp_batch b = *bp;
    const pp_instance I = b.inst[blockIdx.x];
    extern __shared__ __align__(16) double cs_smem[];
    combine_item_bis(b, I, j, blockIdx.y + r0, cs_smem);
    pdl_trigger_at<2>();
    tr.end(2, j);
}

}  // namespace pp

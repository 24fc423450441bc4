// dp_inst2.cu — the PRM wavefront of ONE small instance inside ONE CTA, with
// every per-step operand built in shared memory (C4: 4096 x (32 layers, 16 GPUs)).
//
// Reference: partition.py:95-142 (PartitionSolver._solve_uncached), factored as
// DESIGN.md §2 (expand X = min_r' max(W_j, chan); combine W = min_l' max(X, S)).
//
// Compared with dp_inst.cu (which stages operands from tables the batch
// kernels k_stab / k_base materialise in global memory), this CTA
//   * computes each step's stage-term triangles S(l', l, r, j + r) itself,
//     straight into shared memory (the expression of k_stab / stage_term, the
//     same bits), so no per-instance triangle table is ever written: k_stab and
//     k_sdedup do not run for these batches (C4: 1.95 GB of triangles per
//     4096 instances no longer go through DRAM; the backtrack computes the few
//     stage terms it needs with the scalar stage_term());
//   * keeps X of the step in shared memory for its own combine (X still goes to
//     global memory once, for the backtrack),
//   * divides by hoisted reciprocals (div_fixed: the bits of '/'): one divisor
//     per chan (r', r) and per stage-term width, ~3 fp64 ops per element, and
//   * walks rows / tiles with incremental indices, none in the (min, max) loops.
// Steps j = 1..V-1 in sequence, two phases each, __syncthreads between:
//   E(j): A = W_j(l', ., .) rows in one TMA bulk copy (structural cells as they
//         are: the fold masks them), B = chan(l', r', r) divided here
//         (partition.py:131-137); tiles 4 xi x 4 r per row; rows whose xi
//         exceed l' + 1 are +inf without a fold (no split fits).
//   C(j): triangles of the items r = 1..V-j (certified non-increasing in l'
//         once per instance); tiles TL x TX per item
//         (prm.cu combine_tile_*), row tiles paired with their mirror.
#include "common.cuh"

namespace pp {

constexpr int DI2_T = 256;

// shared-memory regions (doubles) of one CTA for an (L, V) instance: R1 holds a
// step's A + B (expand) or its items' triangles (combine), XS the step's X
__host__ __device__ __forceinline__ void dp_inst2_regions(int L, int V, int64_t& r1, int64_t& xs) {
    const int64_t lm = L > 1 ? L - 1 : 0, tri = lm * L / 2;
    r1 = 0;
    xs = 0;
    for (int j = 1; j < V; ++j) {
        const int64_t nr = V - j;
        const int64_t e = lm * j * j + lm * j * nr, c = nr * tri;
        r1 = e > r1 ? e : r1;
        r1 = c > r1 ? c : r1;
        xs = lm * j * nr > xs ? lm * j * nr : xs;
    }
}
// prefix (L+1), psum (L x L), minpair (V x V), Mp (L), the step's divisors
// and their reciprocals (chan: V^2/4 + 1 each; stage terms: V each; 1/r), R1, XS,
// then the packed triangle's (l', l) of every offset (2 bytes each)
__host__ __device__ __forceinline__ int64_t dp_inst2_div_doubles(int V) { return 2 * ((int64_t)V * V / 4 + 1) + 3 * V; }
__host__ __device__ __forceinline__ int64_t dp_inst2_smem_doubles(int L, int V) {
    int64_t r1, xs;
    dp_inst2_regions(L, V, r1, xs);
    const int64_t tri = (int64_t)(L > 1 ? L - 1 : 0) * L / 2;
    return (L + 1) + (int64_t)L * L + (int64_t)V * V + L + dp_inst2_div_doubles(V) + 2 + r1 + xs +
           (2 * tri + 7) / 8;
}

// incremental walk of e = t, t + nt, ... as (row, o) with e = row * n + o: one
// division per step instead of one per element
struct Walk2 {
    int row, o, drow, dox, n;
    __device__ __forceinline__ Walk2(int e0, int nt, int n_) : n(n_) {
        row = e0 / n_; o = e0 - row * n_; drow = nt / n_; dox = nt - drow * n_;
    }
    __device__ __forceinline__ void next() {
        row += drow; o += dox;
        if (o >= n) { o -= n; ++row; }
    }
};

// E(j) tiles: TXI columns xi x TRR targets r per thread and row l'; K = r'.
// A holds W_j's rows as copied (structural cells are whatever the workspace
// held): column xi' = xi - 1 of the tile folds only its structural range of r'
// (W_structural: r' <= j - xi' + 1 for xi' >= 2, r' = j alone for xi' = 1;
// r' = 1 only without replication), the common range unmasked and the ragged
// tail under a per-column mask.
template <int TXI, int TRR>
__device__ __forceinline__ void dp_inst2_expand(const double* A, const double* B, double* XS, double* Xg, int L,
                                                int j, int nr, bool allow) {
    const int lm = L - 1, jj = j * j, jn = j * nr;
    // a thread folds column tile tx and its mirror ntx-1-tx: their r' trip counts
    // (j - xi0 + 2 each) sum to a constant, so the lanes of a warp stay in step
    // (only while the step has >= 2 tiles per thread: pairing halves the parallelism)
    const int ntx = (j + TXI - 1) / TXI, ntr = (nr + TRR - 1) / TRR;
    const bool pair = lm * ntx * ntr >= 2 * (int)blockDim.x;
    const int ntx2 = pair ? (ntx + 1) / 2 : ntx, per_row = ntx2 * ntr;
    for (int id = threadIdx.x; id < lm * per_row; id += blockDim.x)
#pragma unroll 1
    for (int half = 0; half < 2; ++half) {
        const int k = id / per_row, rem = id - k * per_row;   // row l' = k + 1
        const int tr = rem / ntx2, px = rem - tr * ntx2;
        const int tx = half ? ntx - 1 - px : px;
        if (half && (!pair || tx == px)) break;
        const int xi0 = 2 + TXI * tx, r0 = 1 + TRR * tr, lp = k + 1;
        double acc[TXI][TRR];
#pragma unroll
        for (int a = 0; a < TXI; ++a)
#pragma unroll
            for (int c = 0; c < TRR; ++c) acc[a][c] = PP_INF;
        if (xi0 - 1 <= lp) {   // else W_j(l', xi', .) = inf for every xi' >= xi0 - 1 > l'
            int xa[TXI], rc[TRR], lo[TXI], span[TXI];
            int kmin = 1 << 30, kmax = 0;
#pragma unroll
            for (int a = 0; a < TXI; ++a) {
                const int xip = xi0 - 1 + a;
                xa[a] = min(xip, j) - 1;
                lo[a] = 1 << 30;
                span[a] = 0;
                if (xip > j) continue;   // padded column (discarded)
                if (xip >= 2) {
                    const int hi = allow ? j - xip + 1 : 1;
                    lo[a] = 1; span[a] = hi - 1;
                    kmin = min(kmin, hi); kmax = max(kmax, hi);
                } else {
                    kmin = 0;
                    if (allow || j == 1) { lo[a] = j; kmax = max(kmax, j); }
                }
            }
            if (kmin > kmax) kmin = kmax;
#pragma unroll
            for (int c = 0; c < TRR; ++c) rc[c] = min(r0 + c, nr) - 1;
            const double* Ar = A + (int64_t)k * jj;
            const double* Br = B + (int64_t)k * jn;
            int rp = 1;
            for (; rp <= kmin; ++rp) {
                double p[TXI], q[TRR];
#pragma unroll
                for (int a = 0; a < TXI; ++a) p[a] = Ar[xa[a]];
#pragma unroll
                for (int c = 0; c < TRR; ++c) q[c] = Br[rc[c]];
#pragma unroll
                for (int a = 0; a < TXI; ++a)
#pragma unroll
                    for (int c = 0; c < TRR; ++c) acc[a][c] = dmin(acc[a][c], dmax(p[a], q[c]));
                Ar += j;
                Br += nr;
            }
            for (; rp <= kmax; ++rp) {
                double p[TXI], q[TRR];
#pragma unroll
                for (int a = 0; a < TXI; ++a) p[a] = (unsigned)(rp - lo[a]) <= (unsigned)span[a] ? Ar[xa[a]] : PP_INF;
#pragma unroll
                for (int c = 0; c < TRR; ++c) q[c] = Br[rc[c]];
#pragma unroll
                for (int a = 0; a < TXI; ++a)
#pragma unroll
                    for (int c = 0; c < TRR; ++c) acc[a][c] = dmin(acc[a][c], dmax(p[a], q[c]));
                Ar += j;
                Br += nr;
            }
        }
#pragma unroll
        for (int c = 0; c < TRR; ++c) {
            const int r = r0 + c;
            if (r > nr) continue;
            double* xs = XS + ((int64_t)(r - 1) * lm + k) * j;
            double* xg = Xg + X_base(L, j + r, r) + (int64_t)k * j;
#pragma unroll
            for (int a = 0; a < TXI; ++a) {
                const int xi = xi0 + a;
                if (xi <= j + 1) { xs[xi - 2] = acc[a][c]; xg[xi - 2] = acc[a][c]; }
            }
        }
    }
}

// C(j) tiles: TL rows x TX columns per thread over every item of the step
// (TX shrinks with j so few-column steps do not fold padded columns)
template <int TX, int TL>
__device__ __forceinline__ void dp_inst2_combine(double* Wg, const double* R1, const double* XS, const int* trio,
                                                 const int* s_mono, int L, int j, int r_hi, int tri) {
    const int lm = L - 1;
    // a thread folds row tile tl and its mirror ntl-1-tl (l' trip counts ~ l0 each:
    // their sum is about constant, so the lanes of a warp stay in step)
    // (only while the step has >= 2 tiles per thread: pairing halves the parallelism)
    const int ntl = (L + TL - 1) / TL, ntx = (j + TX - 1) / TX;
    const bool pair = r_hi * ntl * ntx >= 2 * (int)blockDim.x;
    const int ntl2 = pair ? (ntl + 1) / 2 : ntl, nti = ntl2 * ntx;
    for (int id = threadIdx.x; id < r_hi * nti; id += blockDim.x)
#pragma unroll 1
    for (int half = 0; half < 2; ++half) {
        const int q = id / nti, rem = id - q * nti;
        const int r = q + 1, i = j + r;
        const int pl = rem / ntx, tx = rem - pl * ntx;
        const int tl = half ? ntl - 1 - pl : pl;
        if (half && (!pair || tl == pl)) break;
        const int l0 = 1 + TL * tl, xi0 = 2 + TX * tx;
        const double* Stri = R1 + (int64_t)q * tri;
        const double* Xs = XS + (int64_t)q * lm * j;
        double acc[TL][TX];
        if (s_mono[0]) combine_tile_s_desc<TX, TL>(Stri, trio, Xs, L, j, l0, xi0, 1, L - 1, acc);
        else combine_tile_s<TX, TL>(Stri, trio, Xs, L, j, l0, xi0, 1, L - 1, acc);
        double* Wi = Wg + W_base(L, i);
#pragma unroll
        for (int a = 0; a < TL; ++a) {
            const int l = l0 + a;
            if (l > L) continue;
            double* row = Wi + ((int64_t)(l - 1) * i + (r - 1)) * i;
#pragma unroll
            for (int c = 0; c < TX; ++c)
                if (xi0 + c <= j + 1) row[xi0 + c - 1] = acc[a][c];
        }
    }
}

__global__ void __launch_bounds__(DI2_T, 2) k_dp_inst2(pp_batch b) {
    const pp_instance I = b.inst[blockIdx.x];
    const int L = I.L, V = I.V, M = I.M;
    if (L > SR_MAX || V > SR_MAX || V < 2) return;
    extern __shared__ __align__(16) double d2[];
    __shared__ int trio[SR_MAX];
    __shared__ int s_mono[SR_MAX];
    __shared__ uint64_t s_bar;   // W_j bulk copy of E(j)
    unsigned bar_phase = 0;
    const uint64_t pol = l2_evict_normal_policy();
    if (threadIdx.x == 0) mbar_init(&s_bar);
    const bool allow = I.flags & PP_ALLOW_REPLICATION;
    const WsLayout lay = ws_layout(L, V);
    double* ws = b.ws + I.ws_off;
    const double* cross = ws + lay.cross;
    double* Wg = ws + lay.W;
    double* Xg = ws + lay.X;
    const int t = threadIdx.x, nt = blockDim.x;
    const int lm = L - 1, tri = lm * L / 2;
    double* prefix = d2;
    double* psum = prefix + (L + 1);
    double* minpair = psum + L * L;
    double* Mp = minpair + V * V;
    const int nbd = V * V / 4 + 1;
    double* Bden = Mp + L;          // chan divisors of the step, [r'-1][r-1]
    double* Brec = Bden + nbd;
    double* Sden = Brec + nbd;      // stage-term divisors of the step, [r-1]
    double* Srec = Sden + V;
    double* Trec = Srec + V;        // 1 / r of the step's widths
    double* R1 = d2 + ((Trec + V - d2 + 1) & ~1);   // 16-byte aligned
    int64_t r1n, xsn;
    dp_inst2_regions(L, V, r1n, xsn);
    double* XS = R1 + r1n + 1;                       // 1 spare double: A at W_j's 16-byte phase
    unsigned char* tlp = reinterpret_cast<unsigned char*>(XS + xsn);   // offset o -> l' (then l)
    unsigned char* tl = tlp + tri;
    for (int e = t; e <= L; e += nt) prefix[e] = ws[lay.prefix + e];
    for (int e = t; e < L * L; e += nt) psum[e] = ws[lay.psum + e];
    for (int e = t; e < V * V; e += nt) minpair[e] = ws[lay.minpair + e];
    for (int lp = 1 + t; lp < L; lp += nt) {
        const int o0 = (lp - 1) * L - (lp - 1) * lp / 2;
        trio[lp] = o0;
        Mp[lp] = (double)M * (b.efwd[I.layer_off + lp - 1] + b.ebwd[I.layer_off + lp - 1]);   // partition.py:131,137
        for (int l = lp + 1; l <= L; ++l) { tlp[o0 + l - lp - 1] = (unsigned char)lp; tl[o0 + l - lp - 1] = (unsigned char)l; }
    }
    // no per-instance triangle table exists: the backtrack computes its stage terms
    int* sidx = reinterpret_cast<int*>(ws + lay.sidx);
    for (int e = t; e < V * V; e += nt) sidx[e] = -1;
    if (t == 0) s_mono[0] = g_combine_early_exit;
    __syncthreads();
    // Certificate of every stage-term triangle of the instance at once (DESIGN.md
    // §4.3: S non-increasing in l').  The span half (M * (prefix[l] - prefix[l'])) / r
    // is non-increasing in l' for ANY rounding: prefix is non-decreasing
    // (partition.py:62 adds non-negative times) and fl(-), fl(*), fl(/) by a
    // positive constant and fl(+) are monotone.  So is the sync half
    // (2 (r-1) P(l'+1..l)) / (r * minpair) whenever the packed parameter sums
    // P(l'+1..l) are non-increasing in l', and then so is their rounded sum:
    // one pass over psum decides every item of every step.
    for (int o = t; o < tri; o += nt) {
        const int lp = tlp[o], l = tl[o];
        if (l >= lp + 2 && !(psum[lp * L + (l - 1)] >= psum[(lp + 1) * L + (l - 1)])) s_mono[0] = 0;
    }
    __syncthreads();
    for (int j = 1; j < V; ++j) {
        const int nr = V - j, jj = j * j, jn = j * nr;
        const int r_hi = allow ? nr : 1;   // without replication only r = 1 holds values (partition.py:103-104)
        // the step's divisors: chan (r', r) and stage terms (r), reciprocals hoisted
        for (int o = t; o < jn; o += nt) {
            const int rp = o / nr, q = o - rp * nr, r = q + 1;
            const double d = (double)((rp + 1) * r) * cross[cross_idx(V, j + r, r, rp + 1)];
            Bden[o] = d;
            Brec[o] = div_fixed_ok(d) ? div_recip(d) : 0.0;
        }
        for (int q = t; q < r_hi; q += nt) {
            const int r = q + 1, i = j + r;
            const double d = (double)r * minpair[(i - r) * V + (i - 1)];
            Sden[q] = d;
            Srec[q] = div_fixed_ok(d) ? div_recip(d) : 0.0;
            Trec[q] = div_recip((double)r);
        }
        __syncthreads();
        // ------------------------------------------------------------ E(j)
        if (L > 1) {
            const double* Wj = Wg + W_idx(L, j, 1, 1, 1);   // rows contiguous, j x j each
            double* A = R1 + dphase(Wj);        // [l'-1][r'-1][xi'-1], W_j's 16-byte phase
            double* B = A + (int64_t)lm * jj;   // [l'-1][r'-1][r-1]
            // W_j rows (l' = 1..L-1) in one TMA bulk copy, structural cells as they are
            // (the fold masks them); completes on s_bar while B is divided below
            stage_span(A, Wj, 0, lm * jj, &s_bar, pol);
            {
                Walk2 w(t, nt, jn);
                for (int e = t; e < lm * jn; e += nt, w.next())
                    B[e] = div_fixed(Mp[w.row + 1], Bden[w.o], Brec[w.o], Brec[w.o] != 0.0);
            }
            mbar_wait_parity(&s_bar, bar_phase);
            bar_phase ^= 1;
            __syncthreads();
            // tile shape by the step's column / target counts (no folds of padding)
            if (j == 1) dp_inst2_expand<1, 8>(A, B, XS, Xg, L, j, nr, allow);
            else if (nr <= 2) {
                if (j >= 8) dp_inst2_expand<8, 2>(A, B, XS, Xg, L, j, nr, allow);
                else dp_inst2_expand<4, 2>(A, B, XS, Xg, L, j, nr, allow);
            } else if (j <= 3) dp_inst2_expand<2, 4>(A, B, XS, Xg, L, j, nr, allow);
            else dp_inst2_expand<4, 4>(A, B, XS, Xg, L, j, nr, allow);
            __syncthreads();
        }
        // ------------------------------------------------------------ C(j)
        // stage-term triangles S(l', l) of the items (k_stab / stage_term's expression,
        // cost.py:99, partition.py:127-129), one element per thread:
        //   S(l', l) = (M * span(l'+1, l)) / r + ((2 (r-1)) * P(l'+1..l)) / (r * minpair)
        for (int q = 0; q < r_hi; ++q) {
            const int r = q + 1;
            const double den = Sden[q], rec = Srec[q], tr = Trec[q], dr = (double)r;
            const double c2 = 2.0 * (double)(r - 1);
            const bool ok = rec != 0.0;
            double* Sq = R1 + (int64_t)q * tri;
            for (int o = t; o < tri; o += nt) {
                const int lp = tlp[o], l = tl[o];
                double sv = div_fixed((double)M * (prefix[l] - prefix[lp]), dr, tr, true);
                if (r > 1) sv += div_fixed(c2 * psum[lp * L + (l - 1)], den, rec, ok);
                Sq[o] = sv;
            }
        }
        __syncthreads();
        if (j >= 4) dp_inst2_combine<4, 2>(Wg, R1, XS, trio, s_mono, L, j, r_hi, tri);
        else if (j >= 2) dp_inst2_combine<2, 4>(Wg, R1, XS, trio, s_mono, L, j, r_hi, tri);
        else dp_inst2_combine<1, 8>(Wg, R1, XS, trio, s_mono, L, j, r_hi, tri);
        __syncthreads();   // W_{j+1} complete (its last item, r = 1, was just written) before E(j+1)
    }
}

}  // namespace pp

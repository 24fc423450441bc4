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
//     global memory once, for the backtrack), and
//   * walks rows / tiles with incremental indices: one division pair per staged
//     element, none in the (min, max) loops.
// Steps j = 1..V-1 in sequence, two phases each, __syncthreads between:
//   E(j): A = W_j(l', ., .) rows (structural cells +inf), B = chan(l', r', r)
//         divided here (partition.py:131-137); tiles 4 xi x 4 r per row; rows
//         whose xi exceed l' + 1 are +inf without a fold (no split fits).
//   C(j): triangles of the items r = 1..V-j, certified non-increasing in l'
//          per item; tiles TL x TX per item (prm.cu combine_tile_*).
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
// prefix (L+1), psum (L x L), minpair (V x V), Mp (L), R1, XS, then the packed
// triangle's (l', l) of every offset (2 bytes each)
__host__ __device__ __forceinline__ int64_t dp_inst2_smem_doubles(int L, int V) {
    int64_t r1, xs;
    dp_inst2_regions(L, V, r1, xs);
    const int64_t tri = (int64_t)(L > 1 ? L - 1 : 0) * L / 2;
    return (L + 1) + (int64_t)L * L + (int64_t)V * V + L + r1 + xs + (2 * tri + 7) / 8;
}

// E(j) tiles: TXI columns xi x TRR targets r per thread and row l'; K = r'
template <int TXI, int TRR>
__device__ __forceinline__ void dp_inst2_expand(const double* A, const double* B, double* XS, double* Xg, int L,
                                                int j, int nr) {
    const int lm = L - 1, jj = j * j, jn = j * nr;
    const int ntx = (j + TXI - 1) / TXI, ntr = (nr + TRR - 1) / TRR, per_row = ntx * ntr;
    for (int id = threadIdx.x; id < lm * per_row; id += blockDim.x) {
        const int k = id / per_row, rem = id - k * per_row;   // row l' = k + 1
        const int tr = rem / ntx, tx = rem - tr * ntx;
        const int xi0 = 2 + TXI * tx, r0 = 1 + TRR * tr, lp = k + 1;
        double acc[TXI][TRR];
#pragma unroll
        for (int a = 0; a < TXI; ++a)
#pragma unroll
            for (int c = 0; c < TRR; ++c) acc[a][c] = PP_INF;
        if (xi0 - 1 <= lp) {   // else W_j(l', xi', .) = inf for every xi' >= xi0 - 1 > l'
            const int kend = j - xi0 + 2;   // W_j(l', xi-1, r') = inf for r' > j - xi + 2
            int xa[TXI], rc[TRR];
#pragma unroll
            for (int a = 0; a < TXI; ++a) xa[a] = min(xi0 - 1 + a, j) - 1;
#pragma unroll
            for (int c = 0; c < TRR; ++c) rc[c] = min(r0 + c, nr) - 1;
            const double* Ar = A + (int64_t)k * jj;
            const double* Br = B + (int64_t)k * jn;
            for (int rp = 1; rp <= kend; ++rp) {
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
    const int ntl = (L + TL - 1) / TL, ntx = (j + TX - 1) / TX, nti = ntl * ntx;
    for (int id = threadIdx.x; id < r_hi * nti; id += blockDim.x) {
        const int q = id / nti, rem = id - q * nti;
        const int r = q + 1, i = j + r;
        const int tl = rem / ntx, tx = rem - tl * ntx;
        const int l0 = 1 + TL * tl, xi0 = 2 + TX * tx;
        const double* Stri = R1 + (int64_t)q * tri;
        const double* Xs = XS + (int64_t)q * lm * j;
        double acc[TL][TX];
        if (g_combine_early_exit && s_mono[q]) combine_tile_s_desc<TX, TL>(Stri, trio, Xs, L, j, l0, xi0, 1, L - 1, acc);
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
    double* R1 = Mp + L;
    int64_t r1n, xsn;
    dp_inst2_regions(L, V, r1n, xsn);
    double* XS = R1 + r1n;
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
    __syncthreads();
    // T1(r, l', l) = (M * span(l'+1, l)) / r, the i-independent half of every stage
    // term (k_base's expression), once per instance for r = 1..V-1 (packed
    // triangles, the instance's T1 region; L2-resident while this CTA runs)
    double* T1 = ws + lay.T1;
    for (int e = t; e < (V - 1) * tri; e += nt) {
        int q, o;
        divmod_small(e, tri, 1.0f / (float)tri, q, o);
        const int lp = tlp[o], l = tl[o];
        T1[e] = (double)M * (prefix[l] - prefix[lp]) / (double)(q + 1);
    }
    __syncthreads();
    for (int j = 1; j < V; ++j) {
        const int nr = V - j, jj = j * j;
        // ------------------------------------------------------------ E(j)
        if (L > 1) {
            double* A = R1;                    // [l'-1][r'-1][xi'-1]
            double* B = R1 + (int64_t)lm * jj;  // [l'-1][r'-1][r-1]
            const double* Wj = Wg + W_idx(L, j, 1, 1, 1);   // rows contiguous, j x j each
            const float rj = 1.0f / (float)j;
            for (int e = t; e < lm * jj; e += nt) {
                int row, o, rp, xp;
                divmod_small(e, jj, 1.0f / (float)jj, row, o);
                divmod_small(o, j, rj, rp, xp);
                A[e] = W_structural(j, rp + 1, xp + 1, allow) ? Wj[e] : PP_INF;
            }
            const int jn = j * nr;
            const float rjn = 1.0f / (float)jn, rnr = 1.0f / (float)nr;
            for (int e = t; e < lm * jn; e += nt) {
                int row, o, rp, q;
                divmod_small(e, jn, rjn, row, o);
                divmod_small(o, nr, rnr, rp, q);
                const int r = q + 1;
                B[e] = Mp[row + 1] / ((double)((rp + 1) * r) * cross[cross_idx(V, j + r, r, rp + 1)]);
            }
            __syncthreads();
            // tile shape by the step's column / target counts (no folds of padding)
            if (j == 1) dp_inst2_expand<1, 8>(A, B, XS, Xg, L, j, nr);
            else if (nr <= 2) {
                if (j >= 8) dp_inst2_expand<8, 2>(A, B, XS, Xg, L, j, nr);
                else dp_inst2_expand<4, 2>(A, B, XS, Xg, L, j, nr);
            } else if (j <= 3) dp_inst2_expand<2, 4>(A, B, XS, Xg, L, j, nr);
            else dp_inst2_expand<4, 4>(A, B, XS, Xg, L, j, nr);
            __syncthreads();
        }
        // ------------------------------------------------------------ C(j)
        const int r_hi = allow ? nr : 1;   // without replication only r = 1 holds values (partition.py:103-104)
        // stage-term triangles S(l', l) of the items (k_stab's expression, cost.py:99)
        for (int q = t; q < r_hi; q += nt) s_mono[q] = 1;
        // every (item, l', l) of the step's triangles, one element per thread:
        //   S(l', l) = (M * span(l'+1, l)) / r + ((2 (r-1)) * P(l'+1..l)) / (r * minpair)
        // (k_stab / stage_term's expression, cost.py:99, partition.py:127-129)
        const float rtri = 1.0f / (float)tri;
        for (int e = t; e < r_hi * tri; e += nt) {
            int q, o;
            divmod_small(e, tri, rtri, q, o);
            const int lp = tlp[o], l = tl[o];
            const int r = q + 1, i = j + r;
            double sv = T1[(int64_t)q * tri + o];
            if (r > 1) sv += 2.0 * (double)(r - 1) * psum[lp * L + (l - 1)] / ((double)r * minpair[(i - r) * V + (i - 1)]);
            R1[e] = sv;
        }
        __syncthreads();
        if (g_combine_early_exit)   // certificate: non-increasing in l' (S(l', l) >= S(l'+1, l))
            for (int e = t; e < r_hi * tri; e += nt) {
                int q, o;
                divmod_small(e, tri, rtri, q, o);
                const int lp = tlp[o], l = tl[o];
                if (l >= lp + 2 && !(R1[e] >= R1[(int64_t)q * tri + trio[lp + 1] + (l - lp - 2)])) s_mono[q] = 0;
            }
        __syncthreads();
        if (j >= 4) dp_inst2_combine<4, 2>(Wg, R1, XS, trio, s_mono, L, j, r_hi, tri);
        else if (j >= 2) dp_inst2_combine<2, 4>(Wg, R1, XS, trio, s_mono, L, j, r_hi, tri);
        else dp_inst2_combine<1, 8>(Wg, R1, XS, trio, s_mono, L, j, r_hi, tri);
        __syncthreads();   // W_{j+1} complete (its last item, r = 1, was just written) before E(j+1)
    }
}

}  // namespace pp

// dp_inst.cu — the whole PRM wavefront of ONE instance inside ONE CTA, for
// batches with many more instances than SMs (C4: 4096 x (32 layers, 16 GPUs)).
//
// The per-step schedules parallelise inside an instance; with thousands of
// small instances that is the wrong axis: every step launch is thousands of
// tiny CTAs whose staging, barriers and tails dominate (C4 spent ~7 us per
// instance that way).  Here a CTA walks steps j = 1..V-1 of its instance:
//   expand(j):  rows l' = 1..L-1 in chunks that fit shared memory; per chunk the
//               W_j(l', ., .) blocks and chan(l', ., .) tables are staged once,
//               then every (row, 4 xi x 4 r) tile is one thread;
//   combine(j): items r = 1..V-j in chunks; per chunk the stage-term triangles
//               and X(., ., r, j+r) are staged, then every (item, TL x TX) tile
//               is one thread (certified-monotone triangles stop early).
// The arithmetic is the per-step kernels' device functions, so every W / X
// cell is bit-identical to the other schedules.
#include "common.cuh"

namespace pp {

constexpr int DI_T = 256;

template <int TX, int TL = 16 / TX>
__device__ __forceinline__ void dp_inst_combine(const pp_batch& b, const pp_instance& I, int j, int ra, int rb,
                                                double* smem, int* trio) {
    const int L = I.L, V = I.V;
    const WsLayout lay = ws_layout(L, V);
    double* ws = b.ws + I.ws_off;
    const int tri = (L - 1) * L / 2, per_item = tri + (L - 1) * j;
    const int ntl = (L + TL - 1) / TL, ntx = (j + TX - 1) / TX, nti = ntl * ntx;
    const int nq = rb - ra + 1;
    for (int id = threadIdx.x; id < nq * nti; id += blockDim.x) {
        const int q = id / nti, rem = id % nti;
        const int r = ra + q, i = j + r;
        const int l0 = 1 + TL * (rem / ntx), xi0 = 2 + TX * (rem % ntx);
        const double* Stri = smem + (int64_t)q * per_item;
        const double* Xs = Stri + tri;
        const int slot = reinterpret_cast<const int*>(ws + lay.sidx)[(r - 1) * V + (i - 1)];
        const bool mono = g_combine_early_exit && (reinterpret_cast<const int*>(ws + lay.smono)[slot] & 1);
        double acc[TL][TX];
        if (mono) combine_tile_s_desc<TX, TL>(Stri, trio, Xs, L, j, l0, xi0, 1, L - 1, acc);
        else combine_tile_s<TX, TL>(Stri, trio, Xs, L, j, l0, xi0, 1, L - 1, acc);
        double* Wi = ws + lay.W + W_base(L, i);
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

__global__ void __launch_bounds__(DI_T, 3) k_dp_inst(pp_batch b, int smem_doubles) {
    const pp_instance I = b.inst[blockIdx.x];
    const int L = I.L, V = I.V, M = I.M;
    if (L > SR_MAX || V > SR_MAX) return;
    extern __shared__ __align__(16) double di_smem[];
    __shared__ int trio[SR_MAX];
    const bool allow = I.flags & PP_ALLOW_REPLICATION;
    const WsLayout lay = ws_layout(L, V);
    double* ws = b.ws + I.ws_off;
    const double* cross = ws + lay.cross;
    const int t = threadIdx.x;
    __shared__ double mp_s[SR_MAX];   // M * (edge fwd + bwd bytes) of row l' (partition.py:131,137)
    for (int lp = 1 + t; lp < L; lp += blockDim.x) {
        trio[lp] = (lp - 1) * L - (lp - 1) * lp / 2;
        mp_s[lp] = (double)M * (b.efwd[I.layer_off + lp - 1] + b.ebwd[I.layer_off + lp - 1]);
    }
    __syncthreads();
    for (int j = 1; j < V; ++j) {
        const int nr = V - j;
        // ---------------- expand(j): X(l', xi, r, j + r) for every row and target
        if (L > 1) {
            const int per_row = j * j + j * nr;
            const int R = max(1, min(L - 1, smem_doubles / per_row));
            const int ntx = (j + 3) >> 2, ntr = (nr + 3) >> 2, ntr_tiles = ntx * ntr;
            for (int la = 1; la <= L - 1; la += R) {
                const int nrow = min(R, L - la);
                // A rows W_j(l', ., .) (j x j each, contiguous in W): flat over the chunk
                const double* Wsrc = ws + lay.W + W_idx(L, j, la, 1, 1);
                const float rjj = 1.0f / (float)(j * j), rj = 1.0f / (float)j, rnr = 1.0f / (float)nr;
                for (int e = t; e < nrow * j * j; e += blockDim.x) {
                    int k, o, rp, xip;
                    divmod_small(e, j * j, rjj, k, o);
                    divmod_small(o, j, rj, rp, xip);
                    double* A = di_smem + (int64_t)k * per_row;
                    if (W_structural(j, rp + 1, xip + 1, allow)) cp_async8(A + o, Wsrc + (int64_t)k * j * j + o);
                    else A[o] = PP_INF;
                }
                cp_async_commit();
                // B rows chan(l', r', r, j + r) = Mp(l') / ((r' r) cross(r', r, j + r))
                // (copied from the row's payload-class table when it has one: same bits)
                const int* rcls = reinterpret_cast<const int*>(ws + lay.chcls + CHAN_CLS);
                const double* T0 = ws + lay.chan + chan_step(V, j);
                const int64_t tcls = (int64_t)tet(V);
                const bool any_cls = rcls[0] > 0;
                for (int e = t; e < nrow * j * nr; e += blockDim.x) {
                    int k, o, rp, q;
                    divmod_small(e, j * nr, 1.0f / (float)(j * nr), k, o);
                    const int cls = any_cls ? rcls[la + k] : -1;
                    double* dst = di_smem + (int64_t)k * per_row + j * j + o;
                    if (cls >= 0) { cp_async8(dst, T0 + cls * tcls + o); continue; }
                    divmod_small(o, nr, rnr, rp, q);
                    const int r = 1 + q;
                    *dst = mp_s[la + k] / ((double)((rp + 1) * r) * cross[cross_idx(V, j + r, r, rp + 1)]);
                }
                cp_async_commit();
                cp_async_wait<0>();
                __syncthreads();
                double* X = ws + lay.X;
                for (int id = t; id < nrow * ntr_tiles; id += blockDim.x) {
                    const int k = id / ntr_tiles, rem = id % ntr_tiles;
                    const int tx = rem % ntx, tr = rem / ntx;
                    const int xi0 = 2 + 4 * tx, r0 = 1 + 4 * tr;
                    const int kend = j - xi0 + 2;
                    const double* A = di_smem + (int64_t)k * per_row;
                    const double* B = A + j * j;
                    double acc[4][4];
#pragma unroll
                    for (int a = 0; a < 4; ++a)
#pragma unroll
                        for (int c = 0; c < 4; ++c) acc[a][c] = PP_INF;
                    const int xa[4] = {min(xi0 - 1, j) - 1, min(xi0, j) - 1, min(xi0 + 1, j) - 1, min(xi0 + 2, j) - 1};
                    const int rc[4] = {min(r0, nr) - 1, min(r0 + 1, nr) - 1, min(r0 + 2, nr) - 1, min(r0 + 3, nr) - 1};
                    for (int rp = 1; rp <= kend; ++rp) {
                        const double* Ar = A + (rp - 1) * j;
                        const double* Br = B + (rp - 1) * nr;
                        double p[4], q[4];
#pragma unroll
                        for (int a = 0; a < 4; ++a) { p[a] = Ar[xa[a]]; q[a] = Br[rc[a]]; }
#pragma unroll
                        for (int a = 0; a < 4; ++a)
#pragma unroll
                            for (int c = 0; c < 4; ++c) acc[a][c] = dmin(acc[a][c], dmax(p[a], q[c]));
                    }
                    const int lp = la + k;
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const int r = r0 + c;
                        if (r > nr) continue;
                        double* Xr = X + X_base(L, j + r, r) + (int64_t)(lp - 1) * j;
#pragma unroll
                        for (int a = 0; a < 4; ++a)
                            if (xi0 + a <= j + 1) Xr[xi0 + a - 2] = acc[a][c];
                    }
                }
                __syncthreads();
            }
        }
        // ---------------- combine(j): W(., ., r, j + r) for every target
        const int r_hi = allow ? nr : 1;   // without replication only r = 1 holds values
        const int tri = (L - 1) * L / 2, per_item = tri + (L - 1) * j;
        const int Q = max(1, min(r_hi, smem_doubles / max(per_item, 1)));
        for (int ra = 1; ra <= r_hi; ra += Q) {
            const int rb = min(r_hi, ra + Q - 1);
            for (int q = 0; q <= rb - ra; ++q) {
                const int r = ra + q, i = j + r;
                const int slot = reinterpret_cast<const int*>(ws + lay.sidx)[(r - 1) * V + (i - 1)];
                const double* Sg = ws + lay.Stab + (int64_t)slot * tri;
                const double* Xg = ws + lay.X + X_base(L, i, r);
                double* dst = di_smem + (int64_t)q * per_item;
                for (int e = t; e < tri; e += blockDim.x) cp_async8(dst + e, Sg + e);
                for (int e = t; e < (L - 1) * j; e += blockDim.x) cp_async8(dst + tri + e, Xg + e);
            }
            cp_async_commit();
            cp_async_wait<0>();
            __syncthreads();
            if (j >= 4) dp_inst_combine<4, 2>(b, I, j, ra, rb, di_smem, trio);
            else if (j >= 2) dp_inst_combine<2, 4>(b, I, j, ra, rb, di_smem, trio);
            else dp_inst_combine<1, 8>(b, I, j, ra, rb, di_smem, trio);
            __syncthreads();
        }
    }
}

}  // namespace pp

// rdo.cu — device ordering by recursive minimum cuts (ordering.py:30-113).
#include "common.cuh"

namespace pp {

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
__device__ __forceinline__ double warp_min_cut_t(double* wl, const double* bw, int V, const int* mem, int n,
                                                 unsigned char* side_out) {
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    int mk[SLOTS];   // member ids of this lane's columns
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) mk[s] = lane + 32 * s < n ? mem[lane + 32 * s] : 0;
    for (int a = 0; a < n; ++a) {   // row a: contiguous columns, no index division
        const double* src = bw + (int64_t)mem[a] * V;
#pragma unroll
        for (int s = 0; s < SLOTS; ++s) {
            const int c = lane + 32 * s;
            if (c < n) wl[a * n + c] = (a == c) ? 0.0 : src[mk[s]];
        }
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
    const char* colk[SLOTS];   // this lane's columns: wt(v, k) at colk[s] + v * n8 bytes
    const int n8 = 8 * n;
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) colk[s] = reinterpret_cast<const char*>(wl + lane + 32 * s);
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
            // (ties are the common case on structured clusters: three REDUX beat ballot fast paths)
            const unsigned hi = (unsigned)(bu >> 32), lo = (unsigned)bu;
            const unsigned mhi = __reduce_max_sync(FULL, hi);
            // the lane's candidate while its high word ties the max (bk is the
            // 0x7fffffff sentinel when the lane has none): one select after each REDUX
            const unsigned cand = hi == mhi ? (unsigned)bk : 0x7fffffffu;
            const unsigned mlo = __reduce_max_sync(FULL, hi == mhi ? lo : 0u);
            const int nk = (int)__reduce_min_sync(FULL, lo == mlo ? cand : 0x7fffffffu);
            cut = __longlong_as_double((long long)(((unsigned long long)mhi << 32) | mlo));
            sv = tv; tv = nk;
            const int rowoff = nk * n8;   // bytes: one IMAD from nk to the load address
#pragma unroll
            for (int s = 0; s < SLOTS; ++s) {   // adj[u] += wt(next_v, u)  (ordering.py:69-70)
                const int k = lane + 32 * s;
                // the row entry of every live vertex is loaded (that predicate is known
                // before nk), so the load does not wait for the in-set flag update
                const double x = alive[s] ? *reinterpret_cast<const double*>(colk[s] + rowoff) : 0.0;
                if (k == nk) inadj[s] = false;
                if (inadj[s]) adj[s] = adj[s] + x;
            }
        }
        if (cut < best_weight) {   // first minimum cut-of-phase (ordering.py:73-75)
            best_weight = cut;
#pragma unroll
            for (int s = 0; s < SLOTS; ++s) side[s] = (grp[s] == tv);
        }
        const int merged = min(sv, tv), other = max(sv, tv);   // ordering.py:77-85
        __syncwarp();   // every lane's reads of row nk precede the merge's writes
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

__device__ __forceinline__ double warp_min_cut(double* wl, const double* bw, int V, const int* mem, int n,
                                               unsigned char* side) {
    if (n <= 32) return warp_min_cut_t<1>(wl, bw, V, mem, n, side);
    if (n <= 64) return warp_min_cut_t<2>(wl, bw, V, mem, n, side);
    if (n <= 128) return warp_min_cut_t<4>(wl, bw, V, mem, n, side);
    if (n <= 256) return warp_min_cut_t<8>(wl, bw, V, mem, n, side);
    return warp_min_cut_t<16>(wl, bw, V, mem, n, side);
}

// ----------------------------------------------------------------------------
// Speculative RDO.  The recursion tree of rdo() is a pure function of the
// cluster: node S splits into global_min_cut(S), and global_min_cut(S) depends
// on S alone.  The reference's sequential recursion costs the sum over tree
// nodes of n^2/2 dependent max-adjacency steps (44 k at V = 64) where one cut
// costs only n^2/2.
//
// A round: (1) k_rdo_plan PREDICTS the whole recursion tree of every
// unresolved group with a cheap surrogate; (2) k_rdo_cut computes the EXACT
// global_min_cut of every predicted tree node at once, one warp per node, and
// flags whether it splits the node the predicted way; (3) the next k_rdo_plan
// walks each tree top-down: nodes are accepted while their exact cut matches
// (ranks assigned as rdo() assigns them: side_a the low interval, side_b the
// high one), and a mismatching node's EXACT cut splits it into two new groups
// for the next round; its predicted subtree is dropped.  The prediction only
// decides which cuts are computed in parallel; every accepted node is an exact
// cut of a set the reference recursion reaches, so the order is the
// reference's bit for bit.  Whatever is left after the last round is finished
// by k_rdo (resume).
//
// The surrogate, per tree node S: the cheapest of (a) peeling the GPU of least
// weighted degree inside S (ties -> largest id), and (b) cutting off a
// "block" B ∩ S, where blocks are the connected components of the cluster's
// maximum-bandwidth links (the nodes of a two-tier machine), with cut weight
// sum_{v in B∩S} sum_{u in S\B} bw(u, v) (ties -> the block of largest
// label); (b) only when strictly cheaper.  On the 8 x 8 two-tier C3 cluster
// the real tree is 24 peels, then four node splits, then a peel chain inside
// each node — the surrogate predicts all of it, so one round of cuts settles
// the order and the sequential finisher has nothing left to do.
//
// Tree representation.  A "chain" c is a tree node reached from its parent by
// a block split (or the group's root): its set G_c is peeled k times,
// S_{c,k} = G_c minus its first k peels, and either ends in a singleton or in
// a block split of S_{c,len} into child chains A and B.  Chain ids are
// allocated in DFS preorder inside the group's private range [g-1, g-1+n)
// (g = the group's label = its lowest rank, n = its size; at most n chains),
// so a chain's subtree is the id interval [c, c_end[c]).  Vertex v records
// fg[v] = the deepest chain containing it and pk[v] = its peel index there:
//   v in S_{c,k}  <=>  c <= fg[v] < c_end[c]  and not (fg[v] == c and pk[v] < k).
// Tree node (c, k) is cut item it (the group's items are [g-1, g-1+n-1): a
// binary tree on n leaves has n-1 internal nodes).
// ----------------------------------------------------------------------------
struct RdoState {
    int *lo, *pk, *fg, *blk, *blab, *it_c, *it_k, *it_t, *match, *grp;
    int *c_end, *c_len, *c_a, *c_item0, *c_base, *c_par, *cnt;   // cnt[1] groups, cnt[2] blocks
    unsigned char* sides;                                        // [item][local index]
};
__device__ __forceinline__ RdoState rdo_spec_state(const pp_batch& b, const pp_instance& I) {
    const int V = I.V;
    int* p = (int*)(b.ws + I.ws_off + ws_layout(I.L, V).rdo_st);
    RdoState s;
    int** f[] = {&s.lo, &s.pk, &s.fg, &s.blk, &s.blab, &s.it_c, &s.it_k, &s.it_t, &s.match, &s.grp,
                 &s.c_end, &s.c_len, &s.c_a, &s.c_item0, &s.c_base, &s.c_par};
    for (int q = 0; q < RDO_SPEC_ARRAYS; ++q) *f[q] = p + q * V;
    s.cnt = p + RDO_SPEC_ARRAYS * V;
    s.sides = (unsigned char*)(s.cnt + 4);
    return s;
}

__device__ __forceinline__ bool in_item(const RdoState& st, int c, int k, int v) {
    const int f = st.fg[v];
    return f >= c && f < st.c_end[c] && !(f == c && st.pk[v] < k);
}

// ascending list of {v : pred(v)} into mem (one warp); returns the count
template <class P>
__device__ __forceinline__ int warp_list(int V, int* mem, P pred) {
    const int lane = threadIdx.x & 31;
    int n = 0;
    for (int v0 = 0; v0 < V; v0 += 32) {
        const int v = v0 + lane;
        const bool in = v < V && pred(v);
        const unsigned m = __ballot_sync(0xffffffffu, in);
        if (in) mem[n + __popc(m & ((1u << lane) - 1))] = v;
        n += __popc(m);
    }
    __syncwarp();
    return n;
}

// Blocks (round 0, whole CTA): components of the links of maximum bandwidth,
// by min-label propagation with pointer jumping.  st.blk[v] = compact index of
// v's block when it has >= 2 GPUs and is not the whole cluster, else -1;
// lab / cntb: V ints of shared scratch each.
__device__ void rdo_blocks(const double* bw, int V, const RdoState& st, int* lab, int* cntb) {
    __shared__ unsigned long long s_wmax;
    __shared__ int s_nb;
    const int t = threadIdx.x, nt = blockDim.x;
    if (t == 0) { s_wmax = 0ull; s_nb = 0; }
    __syncthreads();
    unsigned long long m = 0ull;   // positive doubles order like their bit patterns (diagonal: 0)
    for (int e = t; e < V * V; e += nt) m = max(m, (unsigned long long)__double_as_longlong(bw[e] > 0.0 ? bw[e] : 0.0));
    atomicMax(&s_wmax, m);
    for (int v = t; v < V; v += nt) { lab[v] = v; cntb[v] = 0; }
    __syncthreads();
    const double wmax = __longlong_as_double((long long)s_wmax);
    bool more = wmax > 0.0;
    while (more) {
        bool changed = false;
        for (int v = t; v < V; v += nt) {
            int mn = lab[v];
            const double* row = bw + (int64_t)v * V;
            for (int u = 0; u < V; ++u)
                if (u != v && row[u] == wmax) mn = min(mn, lab[u]);
            if (mn < lab[v]) { atomicMin(&lab[v], mn); changed = true; }
        }
        __syncthreads();
        for (int v = t; v < V; v += nt) atomicMin(&lab[v], lab[lab[v]]);
        more = __syncthreads_or(changed);
    }
    for (int v = t; v < V; v += nt) atomicAdd(&cntb[lab[v]], 1);
    __syncthreads();
    for (int v = t; v < V; v += nt)   // compact index of every useful block, kept in cntb[label]
        if (lab[v] == v) cntb[v] = (cntb[v] >= 2 && cntb[v] < V) ? -2 - atomicAdd(&s_nb, 1) : -1;
    __syncthreads();
    for (int v = t; v < V; v += nt) {
        const int c = cntb[lab[v]];
        st.blk[v] = c <= -2 ? -2 - c : -1;
    }
    if (t == 0) st.cnt[2] = s_nb;
    // block labels (smallest GPU of the block) by compact index, for the tie rule
    for (int v = t; v < V; v += nt)
        if (lab[v] == v && cntb[v] <= -2) st.blab[-2 - cntb[v]] = v;
    __syncthreads();
}

// Per-warp shared scratch of k_rdo_plan.
struct RdoWarp {
    int* mem;      // V: ascending member list
    int* stk;      // 3V: prediction stack (accept: member fg / pk / chain peel list)
    double* ext;   // V: per member, weight to S outside its block (-inf: peeled)
    int* bkm;      // V: per member, block index
    int* csr;      // V: members grouped by block (ascending within a block)
    int* boff;     // nb + 1: block offsets into csr
};

// Predicted recursion tree of group g (label g, size n, members fg[v] = V + g - 1
// on entry), one warp.  blab: the nb block labels (shared memory).
template <int SLOTS>
__device__ void warp_predict_tree(const double* bw, int V, const RdoState& st, int g, int n_group, int nb,
                                  const int* blab, const RdoWarp& w) {
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int c_lim = g - 1 + n_group;
    int* mem = w.mem;
    int* stk = w.stk;
    int next_c = g - 1, next_it = g - 1, tmp_next = 1, sp = 1;
    if (lane == 0) { stk[0] = V + g - 1; stk[1] = -1; stk[2] = 0; }
    __syncwarp();
    while (sp > 0) {
        --sp;
        const int tl = stk[3 * sp], par = stk[3 * sp + 1], isA = stk[3 * sp + 2];
        const int c = next_c++;
        if (lane == 0) {
            if (par >= 0 && isA) st.c_a[par] = c;
            st.c_par[c] = par; st.c_end[c] = c + 1; st.c_item0[c] = next_it; st.c_a[c] = -1;
        }
        __syncwarp();
        const int n = warp_list(V, mem, [&](int v) { return st.fg[v] == tl; });
        for (int k = lane; k < n; k += 32) {
            st.fg[mem[k]] = c;
            w.bkm[k] = nb > 0 ? st.blk[mem[k]] : -1;
        }
        __syncwarp();
        // members grouped by block (block q owned by lane q % 32; ascending members
        // within a block).  Blocks are candidates only while they hold >= 2 GPUs of S
        // and not all of it: a set inside one block (a node's peel chain) skips them.
        bool blocks = false;
        if (nb > 0 && n >= 3) {
            for (int q = lane; q <= nb; q += 32) w.boff[q] = 0;
            __syncwarp();
            for (int k0 = 0; k0 < n; k0 += 32) {   // counts, 32 members per pass
                const int k = k0 + lane, bq = k < n ? w.bkm[k] : -1;
                const unsigned m = __match_any_sync(0xffffffffu, bq);
                if (bq >= 0 && lane == __ffs(m) - 1) w.boff[bq + 1] += __popc(m);
                __syncwarp();
            }
            bool elig = false;
            for (int q = lane; q < nb; q += 32) elig |= w.boff[q + 1] >= 2 && w.boff[q + 1] < n;
            blocks = __any_sync(0xffffffffu, elig);
            if (blocks) {
                if (lane == 0)
                    for (int q = 0; q < nb; ++q) w.boff[q + 1] += w.boff[q];
                __syncwarp();
                int* cur = reinterpret_cast<int*>(w.ext);   // fill cursors (ext is free until the steps)
                for (int q = lane; q < nb; q += 32) cur[q] = w.boff[q];
                __syncwarp();
                for (int k0 = 0; k0 < n; k0 += 32) {
                    const int k = k0 + lane, bq = k < n ? w.bkm[k] : -1;
                    const unsigned m = __match_any_sync(0xffffffffu, bq);
                    if (bq >= 0) {
                        w.csr[cur[bq] + __popc(m & ((1u << lane) - 1))] = k;
                    }
                    __syncwarp();
                    if (bq >= 0 && lane == __ffs(m) - 1) cur[bq] += __popc(m);
                    __syncwarp();
                }
            }
        }
        double d[SLOTS], inb[SLOTS];
        int bk[SLOTS];
        bool alive[SLOTS];
#pragma unroll
        for (int s = 0; s < SLOTS; ++s) {
            const int k = lane + 32 * s;
            alive[s] = k < n; d[s] = 0.0; inb[s] = 0.0;
            bk[s] = alive[s] ? w.bkm[k] : -1;
        }
        for (int u = 0; u < n; ++u) {   // bw is symmetric: row mem[u] read lane-contiguously
            const double* row = bw + (int64_t)mem[u] * V;
            const int bu = w.bkm[u];
#pragma unroll
            for (int s = 0; s < SLOTS; ++s) {
                const int k = lane + 32 * s;
                if (k < n && k != u) {
                    const double x = row[mem[k]];
                    d[s] += x;
                    if (bk[s] >= 0 && bk[s] == bu) inb[s] += x;
                }
            }
        }
        int k = 0, n_rem = n;
        bool split = false;
        while (n_rem > 1) {
            // (a) least weighted degree, ties -> largest index: min over (bits, -index)
            unsigned long long bu = ~0ull;
            int bkk = -1;
#pragma unroll
            for (int s = 0; s < SLOTS; ++s) {
                const unsigned long long u = (unsigned long long)__double_as_longlong(d[s] > 0.0 ? d[s] : 0.0);
                if (alive[s] && u <= bu) { bu = u; bkk = lane + 32 * s; }
            }
            const unsigned hi = (unsigned)(bu >> 32), lo = (unsigned)bu;
            const unsigned mhi = __reduce_min_sync(FULL, hi);
            const unsigned mlo = __reduce_min_sync(FULL, hi == mhi ? lo : 0xffffffffu);
            const bool win = bkk >= 0 && hi == mhi && lo == mlo;
            const int t = (int)__reduce_max_sync(FULL, win ? (unsigned)bkk : 0u);
            const double dt = __longlong_as_double((long long)(((unsigned long long)mhi << 32) | mlo));
            // (b) cheapest block B ∩ S with 2 <= |B ∩ S| <= n_rem - 1 (ties -> largest label)
            // A block can only be strictly cheaper than every peel if one of its GPUs
            // sends more weight inside the block than out of it: otherwise
            // cut(B ∩ S) = sum ext(v) >= sum d(v) / 2 >= |B ∩ S| dt / 2 >= dt.
            bool strong = false;
#pragma unroll
            for (int s = 0; s < SLOTS; ++s) strong |= alive[s] && bk[s] >= 0 && 2.0 * inb[s] > d[s];
            int blk_win = -1;
            if (blocks && next_c + sp + 2 <= c_lim && __any_sync(FULL, strong)) {
#pragma unroll
                for (int s = 0; s < SLOTS; ++s) {
                    const int kk = lane + 32 * s;
                    if (kk < n) w.ext[kk] = alive[s] ? d[s] - inb[s] : -PP_INF;
                }
                __syncwarp();
                double bv = PP_INF;
                int bl = -1, bi = -1;
                for (int q = lane; q < nb; q += 32) {
                    double sum = 0.0;
                    int cq = 0;
                    for (int o = w.boff[q]; o < w.boff[q + 1]; ++o) {
                        const double x = w.ext[w.csr[o]];
                        if (x != -PP_INF) { sum += x; ++cq; }
                    }
                    if (cq >= 2 && cq <= n_rem - 1 && (sum < bv || (sum == bv && blab[q] > bl))) {
                        bv = sum; bl = blab[q]; bi = q;
                    }
                }
                for (int off = 1; off < nb && off < 32; off <<= 1) {   // lanes >= nb hold no block
                    const double ov = __shfl_xor_sync(FULL, bv, off);
                    const int ol = __shfl_xor_sync(FULL, bl, off), oi = __shfl_xor_sync(FULL, bi, off);
                    if (ov < bv || (ov == bv && ol > bl)) { bv = ov; bl = ol; bi = oi; }
                }
                bv = __shfl_sync(FULL, bv, 0); bi = __shfl_sync(FULL, bi, 0);
                __syncwarp();
                if (bi >= 0 && bv < dt) blk_win = bi;
            }
            const int item = next_it++;
            if (lane == 0) { st.it_c[item] = c; st.it_k[item] = k; }
            if (blk_win >= 0) {   // block split of S_{c,k}: children A = B ∩ S, B = the rest
                const int tA = V + g - 1 + tmp_next, tB = tA + 1;
                tmp_next += 2;
#pragma unroll
                for (int s = 0; s < SLOTS; ++s)
                    if (alive[s]) st.fg[mem[lane + 32 * s]] = bk[s] == blk_win ? tA : tB;
                if (lane == 0) {
                    st.it_t[item] = -1; st.c_len[c] = k;
                    stk[3 * sp] = tB; stk[3 * sp + 1] = c; stk[3 * sp + 2] = 0;
                    stk[3 * sp + 3] = tA; stk[3 * sp + 4] = c; stk[3 * sp + 5] = 1;
                }
                sp += 2;
                __syncwarp();
                split = true;
                break;
            }
            if (lane == 0) { st.it_t[item] = mem[t]; st.pk[mem[t]] = k; }
            const double* row = bw + (int64_t)mem[t] * V;
            const int btv = w.bkm[t];   // block of t
#pragma unroll
            for (int s = 0; s < SLOTS; ++s) {
                const int kk = lane + 32 * s;
                if (kk == t) alive[s] = false;
                if (alive[s]) {
                    const double x = row[mem[kk]];
                    d[s] -= x;
                    if (bk[s] >= 0 && bk[s] == btv) inb[s] -= x;
                }
            }
            ++k;
            --n_rem;
        }
        if (!split) {
            if (lane == 0) st.c_len[c] = k;
#pragma unroll
            for (int s = 0; s < SLOTS; ++s)
                if (alive[s]) st.pk[mem[lane + 32 * s]] = k;
        }
        __syncwarp();
    }
    // subtree intervals: children follow their parent in preorder
    if (lane == 0)
        for (int c = next_c - 1; c > g - 1; --c) {
            const int p = st.c_par[c];
            if (p >= 0 && st.c_end[c] > st.c_end[p]) st.c_end[p] = st.c_end[c];
        }
    __syncwarp();
}

// MAXS: register slots of the largest group the launch can hold (k_rdo_plan is
// instantiated per batch V class, so small-V batches are not sized for V = 512)
template <int MAXS>
__device__ void warp_predict(const double* bw, int V, const RdoState& st, int g, int n, int nb, const int* blab,
                             const RdoWarp& w) {
    if (MAXS == 1 || n <= 32) warp_predict_tree<1>(bw, V, st, g, n, nb, blab, w);
    else if (MAXS == 2 || n <= 64) warp_predict_tree<(MAXS >= 2 ? 2 : 1)>(bw, V, st, g, n, nb, blab, w);
    else if (MAXS == 4 || n <= 128) warp_predict_tree<(MAXS >= 4 ? 4 : 1)>(bw, V, st, g, n, nb, blab, w);
    else if (MAXS == 8 || n <= 256) warp_predict_tree<(MAXS >= 8 ? 8 : 1)>(bw, V, st, g, n, nb, blab, w);
    else warp_predict_tree<(MAXS >= 16 ? 16 : 1)>(bw, V, st, g, n, nb, blab, w);
}

// ---------------------------------------------------------------------------
// Deduplication: the order is a pure function of the bandwidth
// matrix (ids are sorted, so "smallest id" ties are position ties), and a batch
// often plans one physical cluster for many models / microbatch counts (C3:
// 12 instances, one cluster).  Detected from the data on every call — never
// keyed on the caller's ClusterGraph object: a 64-bit hash of each matrix, then
// the smallest instance with an equal hash AND a bitwise-equal matrix is the
// representative; only representatives run RDO, the others copy its order.
// Representatives via an open-addressing table of 4n slots, four in every
// instance's key record (load <= 1/4, so linear probing stays short):
// k_rdo_hash clears them, k_rdo_insert claims a slot per distinct hash and keeps the smallest
// instance index that hashed there, k_rdo_rep looks its hash up and adopts
// that instance after a bitwise comparison of the two matrices (a hash
// collision just leaves the instance its own representative).  O(1) per
// instance instead of a scan of every earlier instance (C4, 4096 distinct
// clusters: 102 -> ~10 us).
constexpr int RDO_TSLOTS = 4;   // hash-table slots per instance record
struct RdoSlot {
    unsigned long long key;    // claimed hash (0 = empty)
    int tmin, pad;             // smallest instance index with that hash
};
struct RdoKey {
    unsigned long long hash;   // this instance's matrix hash (never 0)
    int rep, pad;
    RdoSlot slot[RDO_TSLOTS];
};
__device__ __forceinline__ RdoKey* rdo_key(const pp_batch& b, const pp_instance& I);
__device__ __forceinline__ RdoSlot* rdo_slot(const pp_batch& b, int s) {
    return &rdo_key(b, b.inst[s / RDO_TSLOTS])->slot[s % RDO_TSLOTS];
}
__device__ __forceinline__ RdoKey* rdo_key(const pp_batch& b, const pp_instance& I) {
    return reinterpret_cast<RdoKey*>(b.ws + I.ws_off + ws_layout(I.L, I.V).rdo_key);
}
__device__ __forceinline__ bool rdo_skip(const pp_batch& b, const pp_instance& I, int k) {
    return (I.flags & PP_GIVEN_ORDER) || rdo_key(b, I)->rep != k;
}
__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
    return x;
}
// one warp per instance: hash (position-mixed sum) of the V x V matrix; rep = self;
// clears the instance's table slot
__global__ void __launch_bounds__(32) k_rdo_hash(pp_batch b, int dedup) {
    const pp_instance I = b.inst[blockIdx.x];
    const int V = I.V;
    const unsigned long long* w = reinterpret_cast<const unsigned long long*>(b.bw + I.bw_off);
    unsigned long long h = 0;
    if (dedup)
        for (int e = threadIdx.x; e < V * V; e += 32) h += mix64(w[e] + 0x9e3779b97f4a7c15ULL * (unsigned long long)(e + 1));
    for (int off = 16; off; off >>= 1) h += __shfl_xor_sync(0xffffffffu, h, off);
    if (threadIdx.x == 0) {
        RdoKey* k = rdo_key(b, I);
        const unsigned long long hk = mix64(h ^ (unsigned long long)V);
        k->hash = hk ? hk : 1ull;
        k->rep = blockIdx.x;
        for (int q = 0; q < RDO_TSLOTS; ++q) { k->slot[q].key = 0ull; k->slot[q].tmin = 0x7fffffff; }
    }
}
// one thread per instance: claim (or find) the slot of its hash, keep the smallest index
__global__ void k_rdo_insert(pp_batch b) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= b.n_inst) return;
    const pp_instance I = b.inst[k];
    if (I.flags & PP_GIVEN_ORDER) return;
    const unsigned long long h = rdo_key(b, I)->hash;
    const int ns = b.n_inst * RDO_TSLOTS;
    int s = (int)(h % (unsigned long long)ns);
    for (int probe = 0; probe < ns; ++probe) {
        RdoSlot* slot = rdo_slot(b, s);
        const unsigned long long prev = atomicCAS(&slot->key, 0ull, h);
        if (prev == 0ull || prev == h) { atomicMin(&slot->tmin, k); return; }
        s = s + 1 == ns ? 0 : s + 1;
    }
}
// one warp per instance: the smallest instance of its hash, if the matrices match bit for bit
__global__ void __launch_bounds__(32) k_rdo_rep(pp_batch b) {
    const int k = blockIdx.x, lane = threadIdx.x;
    const pp_instance I = b.inst[k];
    if (I.flags & PP_GIVEN_ORDER) return;
    const unsigned long long h = rdo_key(b, I)->hash;
    const int ns = b.n_inst * RDO_TSLOTS;
    int s = (int)(h % (unsigned long long)ns), q = k;
    for (int probe = 0; probe < ns; ++probe) {
        const RdoSlot* slot = rdo_slot(b, s);
        if (slot->key == h) { q = slot->tmin; break; }
        if (slot->key == 0ull) break;
        s = s + 1 == ns ? 0 : s + 1;
    }
    if (q == k) return;
    const pp_instance J = b.inst[q];
    if (J.V != I.V) return;
    const int V = I.V;
    const unsigned long long* wk = reinterpret_cast<const unsigned long long*>(b.bw + I.bw_off);
    const unsigned long long* wq = reinterpret_cast<const unsigned long long*>(b.bw + J.bw_off);
    bool diff = false;
    for (int e = lane; e < V * V; e += 32) diff |= wq[e] != wk[e];
    if (!__any_sync(0xffffffffu, diff) && lane == 0) rdo_key(b, I)->rep = q;
}
// duplicates copy their representative's order
__global__ void k_rdo_copy(pp_batch b) {
    const int k = blockIdx.x;
    const pp_instance I = b.inst[k];
    if (I.flags & PP_GIVEN_ORDER) return;
    const int rep = rdo_key(b, I)->rep;
    if (rep == k) return;
    const pp_instance R = b.inst[rep];
    for (int v = threadIdx.x; v < I.V; v += blockDim.x) b.order[I.order_off + v] = b.order[R.order_off + v];
}

// One CTA per instance.  round > 0: accept the previous round's trees;
// predict != 0: predict trees for the unresolved groups (items for k_rdo_cut).
__host__ __device__ inline size_t rdo_plan_smem(int V) {
    const size_t hv = (size_t)(V + 1) / 2;
    // the bandwidth matrix (V <= RDO_SMEM_MAX), ext (V doubles per warp), cnt / first /
    // glist / blab (4V ints), per warp: mem, stk (3V), bkm, csr (V each), boff (hv + 1) ints
    const size_t bwd = V <= RDO_SMEM_MAX ? (size_t)V * V : 0;
    return sizeof(double) * (bwd + RDO_WARPS * (size_t)V) +
           sizeof(int) * (4 * (size_t)V + RDO_WARPS * (6 * (size_t)V + hv + 1));
}

template <int MAXS>
__global__ void __launch_bounds__(32 * RDO_WARPS) k_rdo_plan(pp_batch b, int round, int predict) {
    const pp_instance I = b.inst[blockIdx.x];
    if (rdo_skip(b, I, blockIdx.x)) return;
    const int V = I.V;
    const RdoState st = rdo_spec_state(b, I);
    extern __shared__ __align__(16) double smp[];
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int hv = (V + 1) / 2;
    // the surrogate walks bandwidth rows serially: stage the matrix in shared memory
    const bool bw_smem = V <= RDO_SMEM_MAX;
    double* bws = smp;
    double* sp0 = smp + (bw_smem ? V * V : 0);
    RdoWarp w;
    w.ext = sp0 + warp * V;
    int* cnt = reinterpret_cast<int*>(sp0 + RDO_WARPS * V);
    int* first = cnt + V;
    int* glist = first + V;
    int* blab = glist + V;
    int* wi = blab + V + warp * (6 * V + hv + 1);
    w.mem = wi; w.stk = wi + V; w.bkm = wi + 4 * V; w.csr = wi + 5 * V; w.boff = wi + 6 * V;
    int* mem = w.mem;
    const double* bw = bw_smem ? bws : b.bw + I.bw_off;
    if (bw_smem && (round == 0 || predict)) {
        const double2* src = reinterpret_cast<const double2*>(b.bw + I.bw_off);
        const int n2 = V * V / 2;
        if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
            for (int e = t; e < n2; e += blockDim.x) reinterpret_cast<double2*>(bws)[e] = src[e];
            if ((V * V) & 1) { if (t == 0) bws[V * V - 1] = b.bw[I.bw_off + V * V - 1]; }
        } else {
            for (int e = t; e < V * V; e += blockDim.x) bws[e] = b.bw[I.bw_off + e];
        }
        __syncthreads();
    }
    if (round == 0) {
        for (int v = t; v < V; v += blockDim.x) st.lo[v] = 1;
        rdo_blocks(bw, V, st, cnt, first);
    } else {
        const int ng = st.cnt[1];
        int* fgm = w.stk;           // accept: fg / pk of the chain's members, its peel list
        int* pkm = w.stk + V;
        int* ittm = w.stk + 2 * V;
        for (int gi = warp; gi < ng; gi += RDO_WARPS) {
            const int g = st.grp[gi], c0 = g - 1, cend0 = st.c_end[c0];
            if (lane == 0) st.c_base[c0] = g;
            __syncwarp();
            int skip_until = -1;
            for (int c = c0; c < cend0; ++c) {
                if (c < skip_until) continue;
                const int ce = st.c_end[c];
                const int n = warp_list(V, mem, [&](int v) { const int f = st.fg[v]; return f >= c && f < ce; });
                const int len = st.c_len[c], ca = st.c_a[c];
                const int ni = len + (ca >= 0 ? 1 : 0), it0 = st.c_item0[c];
                for (int q = lane; q < n; q += 32) { fgm[q] = st.fg[mem[q]]; pkm[q] = st.pk[mem[q]]; }
                int k0 = ni;   // first rejected item of the chain
                for (int k = lane; k < ni; k += 32) {
                    ittm[k] = st.it_t[it0 + k];
                    if (!st.match[it0 + k] && k < k0) k0 = k;
                }
                k0 = (int)__reduce_min_sync(0xffffffffu, (unsigned)k0);
                __syncwarp();
                // member q of G_c is in S_{c,j} unless chain c peeled it before j
                auto in_s = [&](int q, int j) { return !(fgm[q] == c && pkm[q] < j); };
                int lo_j = st.c_base[c];
                if (lane == 0) {
                    int hi_j = lo_j + n - 1, ptr = 0;
                    const int np = k0 < len ? k0 : len;
                    for (int j = 0; j < np; ++j) {
                        const int tv = ittm[j];
                        while (!in_s(ptr, j)) ++ptr;   // smallest GPU of S_{c,j}
                        if (mem[ptr] == tv) st.lo[tv] = lo_j++;   // {t} is side_a: lowest rank
                        else st.lo[tv] = hi_j--;                  // {t} is side_b: highest rank
                    }
                    if (k0 == ni) {
                        while (!in_s(ptr, len)) ++ptr;   // smallest GPU of S_{c,len}
                        if (ca >= 0) {   // accepted block split: side_a holds the smallest GPU
                            const int ca_end = st.c_end[ca], cbb = ca_end;   // child B follows A's subtree
                            int na = 0;
                            for (int q = 0; q < n; ++q) na += fgm[q] >= ca && fgm[q] < ca_end;
                            if (fgm[ptr] >= ca && fgm[ptr] < ca_end) { st.c_base[ca] = lo_j; st.c_base[cbb] = lo_j + na; }
                            else { st.c_base[cbb] = lo_j; st.c_base[ca] = lo_j + (hi_j - lo_j + 1 - na); }
                        } else {
                            st.lo[mem[ptr]] = lo_j;   // the chain's last GPU
                        }
                    }
                }
                lo_j = __shfl_sync(0xffffffffu, lo_j, 0);
                if (k0 < ni) {   // the exact cut of S_{c,k0} splits it into two new groups
                    const unsigned char* side = st.sides + (int64_t)(it0 + k0) * V;
                    int na = 0, base = 0;
                    for (int q0 = 0; q0 < n; q0 += 32) {   // local index within S_{c,k0} = rank among its GPUs
                        const int q = q0 + lane;
                        const bool in = q < n && in_s(q, k0);
                        const unsigned m = __ballot_sync(0xffffffffu, in);
                        if (in) na += side[base + __popc(m & ((1u << lane) - 1))];
                        base += __popc(m);
                    }
                    na = (int)__reduce_add_sync(0xffffffffu, (unsigned)na);
                    base = 0;
                    for (int q0 = 0; q0 < n; q0 += 32) {
                        const int q = q0 + lane;
                        const bool in = q < n && in_s(q, k0);
                        const unsigned m = __ballot_sync(0xffffffffu, in);
                        if (in) st.lo[mem[q]] = side[base + __popc(m & ((1u << lane) - 1))] ? lo_j : lo_j + na;
                        base += __popc(m);
                    }
                    skip_until = ce;
                }
                __syncwarp();
            }
        }
    }
    __syncthreads();
    if (!predict) return;
    // unresolved groups: labels held by >= 2 GPUs (first member marks the group)
    const int nb = st.cnt[2];
    for (int v = t; v < V; v += blockDim.x) { cnt[v] = 0; first[v] = 0x7fffffff; st.fg[v] = -1; st.it_c[v] = -1; }
    for (int q = t; q < nb; q += blockDim.x) blab[q] = st.blab[q];
    __syncthreads();
    for (int v = t; v < V; v += blockDim.x) { atomicAdd(&cnt[st.lo[v] - 1], 1); atomicMin(&first[st.lo[v] - 1], v); }
    __syncthreads();
    __shared__ int s_ng;
    if (t == 0) s_ng = 0;
    __syncthreads();
    for (int v = t; v < V; v += blockDim.x) {
        const int g = st.lo[v];
        if (cnt[g - 1] >= 2) st.fg[v] = V + g - 1;   // the tree's root set
        if (cnt[g - 1] >= 2 && first[g - 1] == v) glist[atomicAdd(&s_ng, 1)] = g;
    }
    __syncthreads();
    const int ng = s_ng;
    if (t == 0) st.cnt[1] = ng;
    for (int gi = t; gi < ng; gi += blockDim.x) st.grp[gi] = glist[gi];
    for (int gi = warp; gi < ng; gi += RDO_WARPS) {
        const int g = glist[gi];
        warp_predict<MAXS>(bw, V, st, g, cnt[g - 1], nb, blab, w);
    }
}

// One warp per predicted tree node: exact global_min_cut of S_{c,k}, and
// whether it splits S the predicted way (a singleton {t}, or block child A
// against the rest).
// blockDim = 32 x wpc: warp w of CTA (instance, y) cuts item y * wpc + w, in
// its own slice of `per_warp` bytes of dynamic shared memory (small instances:
// the 32-CTA-per-SM limit, not registers or shared memory, capped the number
// of concurrent cuts at one warp per CTA)
template <bool SMEM>
__global__ void __launch_bounds__(128) k_rdo_cut(pp_batch b, int per_warp) {
    const pp_instance I = b.inst[blockIdx.x];
    if (rdo_skip(b, I, blockIdx.x)) return;
    const int V = I.V;
    // the global-memory variant's per-item scratch (rdo_iw) exists only for
    // V > RDO_SMEM_MAX: a mixed batch runs both variants, each on its instances
    if ((V <= RDO_SMEM_MAX) != SMEM) return;
    const int wpc = blockDim.x >> 5, warp = threadIdx.x >> 5;
    const int item = blockIdx.y * wpc + warp;
    if (item >= V - 1) return;
    const RdoState st = rdo_spec_state(b, I);
    const int c = st.it_c[item];
    if (c < 0) return;
    extern __shared__ double smem_d[];
    char* sm = (char*)smem_d + (size_t)warp * per_warp;
    double* W;
    if constexpr (SMEM) { W = reinterpret_cast<double*>(sm); sm += sizeof(double) * V * V; }
    else W = b.ws + I.ws_off + ws_layout(I.L, V).rdo_iw + (int64_t)item * V * V;
    int* mem = (int*)sm;
    unsigned char* side = (unsigned char*)(mem + V);
    const int lane = threadIdx.x & 31;
    const int k = st.it_k[item], tv = st.it_t[item];
    const int n = warp_list(V, mem, [&](int v) { return in_item(st, c, k, v); });
    warp_min_cut(W, b.bw + I.bw_off, V, mem, n, side);
    bool match;
    if (tv >= 0) {   // predicted peel {t}
        int na = 0, tpos = -1;
        for (int q = lane; q < n; q += 32) {
            na += side[q];
            if (mem[q] == tv) tpos = q;
        }
        na = (int)__reduce_add_sync(0xffffffffu, (unsigned)na);
        tpos = (int)__reduce_max_sync(0xffffffffu, (unsigned)(tpos + 1)) - 1;
        const bool ts = side[tpos];
        match = ts ? na == 1 : na == n - 1;
    } else {         // predicted block split: child A = chains [ca, c_end[ca])
        const int ca = st.c_a[c], ce = st.c_end[ca];
        bool same = true, flip = true;
        for (int q = lane; q < n; q += 32) {
            const int f = st.fg[mem[q]];
            const bool inA = f >= ca && f < ce;
            same &= (side[q] != 0) == inA;
            flip &= (side[q] != 0) != inA;
        }
        match = __all_sync(0xffffffffu, same) || __all_sync(0xffffffffu, flip);
    }
    if (lane == 0) st.match[item] = match ? 1 : 0;
    if (!match)
        for (int q = lane; q < n; q += 32) st.sides[(int64_t)item * V + q] = side[q];
}

// SMEM: the contracted weights live in shared memory (V <= 128); a template
// parameter so the compiler sees the address space and emits LDS/STS.
template <bool SMEM>
__global__ void __launch_bounds__(32 * RDO_WARPS) k_rdo(pp_batch b, int resume) {
    const pp_instance I = b.inst[blockIdx.x];
    if (rdo_skip(b, I, blockIdx.x)) return;
    const int V = I.V;
    extern __shared__ double smem_d[];
    char* sm = (char*)smem_d;
    double* W;
    if constexpr (SMEM) { W = smem_d; sm += sizeof(double) * V * V; }
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
    // resume: start from the groups the speculative rounds left unresolved
    const int* lo_in = resume ? rdo_spec_state(b, I).lo : nullptr;
    for (int v = t; v < V; v += blockDim.x) lo[v] = resume ? lo_in[v] : 1;
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
        // new labels go to `first` (free now) and are copied back after every
        // group of this round is split: warps read lo while others relabel
        for (int v = t; v < V; v += blockDim.x) first[v] = lo[v];
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
            for (int k = lane; k < n; k += 32) first[mem[k]] = side[k] ? g : g + na;
            __syncwarp();
        }
        __syncthreads();
        for (int v = t; v < V; v += blockDim.x) lo[v] = first[v];   // same thread resets first[v] next round
    }
    int* order = b.order + I.order_off;
    for (int v = t; v < V; v += blockDim.x) order[lo[v] - 1] = v;
}

// global_min_cut on a vertex subset (ordering.py:30-91): one warp.
template <bool SMEM>
__global__ void __launch_bounds__(32) k_min_cut(pp_batch b, int k, const int* verts, int n, unsigned char* in_a,
                                                double* weight) {
    const pp_instance I = b.inst[k];
    const int V = I.V;
    extern __shared__ double smem_d[];
    char* sm = (char*)smem_d;
    double* W;
    if constexpr (SMEM) { W = smem_d; sm += sizeof(double) * V * V; }
    else W = b.ws + I.ws_off + ws_layout(I.L, V).rdo_w;
    int* mem = (int*)sm;
    for (int q = threadIdx.x; q < n; q += 32) mem[q] = verts[q];
    __syncwarp();
    const double cw = warp_min_cut(W, b.bw + I.bw_off, V, mem, n, in_a);
    if (threadIdx.x == 0) weight[0] = cw;
}
template __global__ void k_rdo_plan<1>(pp_batch, int, int);
template __global__ void k_rdo_plan<2>(pp_batch, int, int);
template __global__ void k_rdo_plan<4>(pp_batch, int, int);
template __global__ void k_rdo_plan<8>(pp_batch, int, int);
template __global__ void k_rdo_plan<16>(pp_batch, int, int);
template __global__ void k_rdo<true>(pp_batch, int);
template __global__ void k_rdo<false>(pp_batch, int);
template __global__ void k_rdo_cut<true>(pp_batch, int);
template __global__ void k_rdo_cut<false>(pp_batch, int);
template __global__ void k_min_cut<true>(pp_batch, int, const int*, int, unsigned char*, double*);
template __global__ void k_min_cut<false>(pp_batch, int, const int*, int, unsigned char*, double*);

}  // namespace pp

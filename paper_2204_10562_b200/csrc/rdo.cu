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
            // (ties are the common case on structured clusters: three REDUX beat ballot fast paths)
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
// on S alone.  On real topologies the tree is mostly a chain of singleton
// peels (the 8 x 8 two-tier cluster peels 64, 63, ... one GPU at a time), so
// the reference's sequential recursion costs sum_n n^2/2 dependent
// max-adjacency steps (44 k at V = 64) where one cut costs only n^2/2.
//
// A round: (1) k_rdo_plan predicts, for every unresolved group, the whole
// chain S_0 = group, S_{k+1} = S_k \ {t_k} with t_k = the GPU of least
// weighted degree inside S_k (ties -> largest id); (2) k_rdo_cut computes the
// EXACT global_min_cut of every S_k at once, one warp per chain item, and
// flags whether it split off exactly {t_k}; (3) the next k_rdo_plan walks each
// chain: items are accepted while their exact cut matches, each accepted
// singleton takes its rank (side_a -> lowest free rank, side_b -> highest),
// and the first mismatching item's exact cut splits its set into two new
// groups for the next round.  The prediction only decides which cuts are
// computed in parallel; every accepted tree node is an exact cut of the set
// the reference recursion reaches, so the order is the reference's bit for
// bit.  Whatever is left after the last round is finished by k_rdo (resume).
// ----------------------------------------------------------------------------
struct RdoState {
    int *lo, *pk, *it_g, *it_k, *it_t, *match, *grp, *grp_item, *cnt;   // cnt[0] items, cnt[1] groups
    unsigned char* sides;                                              // [item][local index]
};
__device__ __forceinline__ RdoState rdo_spec_state(const pp_batch& b, const pp_instance& I) {
    const int V = I.V;
    int* p = (int*)(b.ws + I.ws_off + ws_layout(I.L, V).rdo_st);
    RdoState s;
    s.lo = p; s.pk = p + V; s.it_g = p + 2 * V; s.it_k = p + 3 * V; s.it_t = p + 4 * V;
    s.match = p + 5 * V; s.grp = p + 6 * V; s.grp_item = p + 7 * V; s.cnt = p + 8 * V;
    s.sides = (unsigned char*)(p + 8 * V + 4);
    return s;
}

// ascending member list of {v : lo[v] == g and pk[v] >= kmin} into mem; returns n (one warp)
__device__ __forceinline__ int warp_members(const int* lo, const int* pk, int V, int g, int kmin, int* mem) {
    const int lane = threadIdx.x & 31;
    int n = 0;
    for (int v0 = 0; v0 < V; v0 += 32) {
        const int v = v0 + lane;
        const bool in = v < V && lo[v] == g && (kmin <= 0 || pk[v] >= kmin);
        const unsigned m = __ballot_sync(0xffffffffu, in);
        if (in) mem[n + __popc(m & ((1u << lane) - 1))] = v;
        n += __popc(m);
    }
    __syncwarp();
    return n;
}

// Predicted peel chain of one group (one warp): pk[mem[k]] = peel index.
template <int SLOTS>
__device__ void warp_predict_chain(const double* bw, int V, const int* mem, int n, int* pk, int* it_t) {
    const int lane = threadIdx.x & 31;
    double d[SLOTS];
    bool alive[SLOTS];
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) { d[s] = 0.0; alive[s] = lane + 32 * s < n; }
    for (int u = 0; u < n; ++u) {   // bw is symmetric: row mem[u] read lane-contiguously
        const double* row = bw + (int64_t)mem[u] * V;
#pragma unroll
        for (int s = 0; s < SLOTS; ++s) {
            const int k = lane + 32 * s;
            if (k < n && k != u) d[s] += row[mem[k]];
        }
    }
    for (int j = 0; j + 1 < n; ++j) {
        // least degree, ties -> largest index: min over (bits, -index)
        unsigned long long bu = ~0ull;
        int bk = -1;
#pragma unroll
        for (int s = 0; s < SLOTS; ++s) {
            const unsigned long long u = (unsigned long long)__double_as_longlong(d[s] > 0.0 ? d[s] : 0.0);
            if (alive[s] && u <= bu) { bu = u; bk = lane + 32 * s; }
        }
        const unsigned hi = (unsigned)(bu >> 32), lo = (unsigned)bu;
        const unsigned mhi = __reduce_min_sync(0xffffffffu, hi);
        const unsigned mlo = __reduce_min_sync(0xffffffffu, hi == mhi ? lo : 0xffffffffu);
        const bool win = bk >= 0 && hi == mhi && lo == mlo;
        const int t = (int)__reduce_max_sync(0xffffffffu, win ? (unsigned)bk : 0u);
        if (lane == 0) { pk[mem[t]] = j; it_t[j] = mem[t]; }
        const double* row = bw + (int64_t)mem[t] * V;
#pragma unroll
        for (int s = 0; s < SLOTS; ++s) {
            const int k = lane + 32 * s;
            if (k == t) alive[s] = false;
            if (alive[s]) d[s] -= row[mem[k]];
        }
    }
#pragma unroll
    for (int s = 0; s < SLOTS; ++s)
        if (alive[s]) pk[mem[lane + 32 * s]] = n - 1;
}

__device__ void warp_predict(const double* bw, int V, const int* mem, int n, int* pk, int* it_t) {
    if (n <= 32) warp_predict_chain<1>(bw, V, mem, n, pk, it_t);
    else if (n <= 64) warp_predict_chain<2>(bw, V, mem, n, pk, it_t);
    else if (n <= 128) warp_predict_chain<4>(bw, V, mem, n, pk, it_t);
    else if (n <= 256) warp_predict_chain<8>(bw, V, mem, n, pk, it_t);
    else warp_predict_chain<16>(bw, V, mem, n, pk, it_t);
}

// ---------------------------------------------------------------------------
// Deduplication: the order is a pure function of the bandwidth
// matrix (ids are sorted, so "smallest id" ties are position ties), and a batch
// often plans one physical cluster for many models / microbatch counts (C3:
// 12 instances, one cluster).  Detected from the data on every call — never
// keyed on the caller's ClusterGraph object: a 64-bit hash of each matrix, then
// the first earlier instance with an equal hash AND a bitwise-equal matrix is
// the representative; only representatives run RDO, the others copy its order.
struct RdoKey { unsigned long long hash; int rep; int pad; };
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
// one warp per instance: hash (position-mixed sum) of the V x V matrix; rep = self
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
        k->hash = mix64(h ^ (unsigned long long)V);
        k->rep = blockIdx.x;
    }
}
// one warp per instance k: the first k' < k with the same V, hash and matrix
// bits (32 candidate hashes per iteration, then a bitwise check of each hit)
__global__ void __launch_bounds__(32) k_rdo_rep(pp_batch b) {
    const int k = blockIdx.x, lane = threadIdx.x;
    const pp_instance I = b.inst[k];
    if (I.flags & PP_GIVEN_ORDER) return;
    const int V = I.V;
    const unsigned long long hk = rdo_key(b, I)->hash;
    const unsigned long long* wk = reinterpret_cast<const unsigned long long*>(b.bw + I.bw_off);
    for (int q0 = 0; q0 < k; q0 += 32) {
        const int q = q0 + lane;
        bool hit = false;
        if (q < k) {
            const pp_instance J = b.inst[q];
            hit = J.V == V && !(J.flags & PP_GIVEN_ORDER) && rdo_key(b, J)->hash == hk;
        }
        unsigned m = __ballot_sync(0xffffffffu, hit);
        while (m) {
            const int qq = q0 + __ffs(m) - 1;
            m &= m - 1;
            const unsigned long long* wq = reinterpret_cast<const unsigned long long*>(b.bw + b.inst[qq].bw_off);
            bool diff = false;
            for (int e = lane; e < V * V; e += 32) diff |= wq[e] != wk[e];
            if (!__any_sync(0xffffffffu, diff)) {
                if (lane == 0) rdo_key(b, I)->rep = qq;
                return;
            }
        }
    }
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

// One CTA per instance.  round > 0: accept the previous round's chains;
// predict != 0: predict chains for the unresolved groups (items for k_rdo_cut).
__global__ void __launch_bounds__(32 * RDO_WARPS) k_rdo_plan(pp_batch b, int round, int predict) {
    const pp_instance I = b.inst[blockIdx.x];
    if (rdo_skip(b, I, blockIdx.x)) return;
    const int V = I.V;
    const RdoState st = rdo_spec_state(b, I);
    extern __shared__ int smi[];
    int* cnt = smi;
    int* first = smi + V;
    int* glist = smi + 2 * V;
    int* memall = smi + 3 * V;   // [RDO_WARPS][V]
    __shared__ int s_ng, s_items;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    int* mem = memall + warp * V;
    if (round == 0) {
        for (int v = t; v < V; v += blockDim.x) st.lo[v] = 1;
    } else {
        const int ng = st.cnt[1];
        for (int gi = warp; gi < ng; gi += RDO_WARPS) {
            const int g = st.grp[gi], it0 = st.grp_item[gi];
            // member lists of other groups change concurrently, but only to labels
            // inside their own rank intervals, never to g
            const int n = warp_members(st.lo, st.pk, V, g, 0, mem);
            int k0 = n - 1;   // first rejected chain item
            for (int k = lane; k < n - 1; k += 32)
                if (!st.match[it0 + k]) { k0 = k; break; }
            k0 = (int)__reduce_min_sync(0xffffffffu, (unsigned)k0);
            int lo_j = g;
            if (lane == 0) {
                int hi_j = g + n - 1, ptr = 0;
                for (int j = 0; j < k0; ++j) {
                    const int tv = st.it_t[it0 + j];
                    while (st.pk[mem[ptr]] < j) ++ptr;   // smallest GPU of S_j
                    if (mem[ptr] == tv) st.lo[tv] = lo_j++;   // {t} is side_a: lowest rank
                    else st.lo[tv] = hi_j--;                  // {t} is side_b: highest rank
                }
            }
            lo_j = __shfl_sync(0xffffffffu, lo_j, 0);
            if (k0 < n - 1) {   // exact cut of S_k0 splits it into two new groups
                const unsigned char* side = st.sides + (int64_t)(it0 + k0) * V;
                int na = 0, base = 0;
                for (int k = lane; k < n - k0; k += 32) na += side[k];
                na = (int)__reduce_add_sync(0xffffffffu, (unsigned)na);
                for (int q0 = 0; q0 < n; q0 += 32) {   // local index within S_k0 = rank among survivors
                    const int q = q0 + lane;
                    const int v = q < n ? mem[q] : 0;
                    const bool in = q < n && st.pk[v] >= k0;
                    const unsigned m = __ballot_sync(0xffffffffu, in);
                    if (in) st.lo[v] = side[base + __popc(m & ((1u << lane) - 1))] ? lo_j : lo_j + na;
                    base += __popc(m);
                }
            } else {
                for (int q = lane; q < n; q += 32)
                    if (st.pk[mem[q]] == n - 1) st.lo[mem[q]] = lo_j;
            }
            __syncwarp();
        }
    }
    __syncthreads();
    if (!predict) return;
    // unresolved groups: labels held by >= 2 GPUs (first member marks the group)
    for (int v = t; v < V; v += blockDim.x) { cnt[v] = 0; first[v] = 0x7fffffff; }
    if (t == 0) s_ng = 0;
    __syncthreads();
    for (int v = t; v < V; v += blockDim.x) { atomicAdd(&cnt[st.lo[v] - 1], 1); atomicMin(&first[st.lo[v] - 1], v); }
    __syncthreads();
    for (int v = t; v < V; v += blockDim.x) {
        const int g = st.lo[v];
        if (cnt[g - 1] >= 2 && first[g - 1] == v) glist[atomicAdd(&s_ng, 1)] = g;
    }
    __syncthreads();
    const int ng = s_ng;
    if (t == 0) {   // groups in label order, items contiguous per group
        for (int a = 1; a < ng; ++a) {
            const int x = glist[a];
            int c = a - 1;
            while (c >= 0 && glist[c] > x) { glist[c + 1] = glist[c]; --c; }
            glist[c + 1] = x;
        }
        int o = 0;
        for (int gi = 0; gi < ng; ++gi) {
            st.grp[gi] = glist[gi];
            st.grp_item[gi] = o;
            o += cnt[glist[gi] - 1] - 1;
        }
        st.cnt[1] = ng;
        s_items = o;
    }
    __syncthreads();
    const double* bw = b.bw + I.bw_off;
    for (int gi = warp; gi < ng; gi += RDO_WARPS) {
        const int g = st.grp[gi], it0 = st.grp_item[gi];
        const int n = warp_members(st.lo, st.pk, V, g, 0, mem);
        warp_predict(bw, V, mem, n, st.pk, st.it_t + it0);
        for (int k = lane; k < n - 1; k += 32) { st.it_g[it0 + k] = g; st.it_k[it0 + k] = k; }
    }
    if (t == 0) st.cnt[0] = s_items;
}

// One warp per predicted chain item: exact global_min_cut of S_k.
template <bool SMEM>
__global__ void __launch_bounds__(32) k_rdo_cut(pp_batch b) {
    const pp_instance I = b.inst[blockIdx.x];
    if (rdo_skip(b, I, blockIdx.x)) return;
    const int V = I.V;
    // the global-memory variant's per-item scratch (rdo_iw) exists only for
    // V > RDO_SMEM_MAX: a mixed batch runs both variants, each on its instances
    if ((V <= RDO_SMEM_MAX) != SMEM) return;
    const RdoState st = rdo_spec_state(b, I);
    const int item = blockIdx.y;
    if (item >= st.cnt[0]) return;
    extern __shared__ double smem_d[];
    char* sm = (char*)smem_d;
    double* W;
    if constexpr (SMEM) { W = smem_d; sm += sizeof(double) * V * V; }
    else W = b.ws + I.ws_off + ws_layout(I.L, V).rdo_iw + (int64_t)item * V * V;
    int* mem = (int*)sm;
    unsigned char* side = (unsigned char*)(mem + V);
    const int lane = threadIdx.x;
    const int g = st.it_g[item], k = st.it_k[item], tv = st.it_t[item];
    const int n = warp_members(st.lo, st.pk, V, g, k, mem);
    warp_min_cut(W, b.bw + I.bw_off, V, mem, n, side);
    int na = 0, tpos = -1;
    for (int q = lane; q < n; q += 32) {
        na += side[q];
        if (mem[q] == tv) tpos = q;
    }
    na = (int)__reduce_add_sync(0xffffffffu, (unsigned)na);
    tpos = (int)__reduce_max_sync(0xffffffffu, (unsigned)(tpos + 1)) - 1;
    const bool ts = side[tpos];
    const bool match = ts ? na == 1 : na == n - 1;
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
template __global__ void k_rdo<true>(pp_batch, int);
template __global__ void k_rdo<false>(pp_batch, int);
template __global__ void k_rdo_cut<true>(pp_batch);
template __global__ void k_rdo_cut<false>(pp_batch);
template __global__ void k_min_cut<true>(pp_batch, int, const int*, int, unsigned char*, double*);
template __global__ void k_min_cut<false>(pp_batch, int, const int*, int, unsigned char*, double*);

}  // namespace pp

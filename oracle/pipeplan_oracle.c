/*
 * oracle/pipeplan_oracle.c
 *
 * TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
 *
 * A plain-C CPU restatement of the reference planning path
 * (/root/reference/pkg/src/pipeplan, "pipeplan" v0.1.0).  It exists only to
 * check the CUDA path: it may be imported, linked or executed only by tests/,
 * __graft_entry__.smoke() (as the checker) and bench.py's cpu_baseline /
 * --impl reference legs.  Nothing in paper_2204_10562_b200/ links it.
 *
 * Parity pinning: the tests/golden/ fixtures were produced by running the live
 * reference (CPython 3.12.3, where float sum() is Neumaier-compensated) via
 * tests/golden/make_golden.py; tests/test_oracle_golden.py checks this file
 * against every fixture bit-for-bit.
 *
 * Restated algorithms (reference file:line):
 *   or_pysum            CPython >= 3.12 builtin sum() over floats, used by
 *                       cost.py:47,53,98,128 (naive mode = CPython <= 3.11)
 *   or_min_cut          ordering.py:30-91   (deterministic Stoer-Wagner)
 *   or_rdo              ordering.py:94-113  (recursive min-cut ordering)
 *   or_prm_new / solve  partition.py:49-142 (W(l, xi, r, i) recursion, evaluated
 *                       bottom-up over xi with the reference's loop order and
 *                       its strict `best > w` first-found tie rule)
 *   or_prm_best         partition.py:144-162
 *   or_pe_queues        scheduler.py:75-106 (pass-order queues)
 *   or_simulate         scheduler.py:121-225 (heap event loop, same heap key)
 *                       + cost.py:205-230 (block durations)
 *   or_lemma1_bound     scheduler.py:234-238 + cost.py:172-202
 *   or_phi              cost.py:126-142
 *   or_spp              planner.py:57-88
 *   or_spp_batch        many or_spp calls on a pthread pool (CPU baseline)
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off; no fast-math).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define OR_INF (1.0 / 0.0)

typedef struct {
    int32_t L, V, M, sum_mode;   /* sum_mode: 1 = Neumaier (CPython >= 3.12), 0 = naive */
    const double *fwd, *bwd, *param;   /* [L] */
    const double *efwd, *ebwd;         /* [L-1] edge l -> l+1 */
    const double *bw;                  /* [V*V] symmetric, sorted-gpu-id index */
} or_inst;

/* ------------------------------------------------------------------------ */
/* CPython builtin sum() over a float iterable with int start 0.            */
/* Python/bltinmodule.c builtin_sum_impl: 0 + x0 on the int fast path, then */
/* the float loop (Neumaier from 3.12), compensation added at the end when  */
/* it is non-zero and finite.                                               */
/* ------------------------------------------------------------------------ */
double or_pysum(const double *x, int64_t n, int32_t mode)
{
    if (n <= 0) return 0.0;
    double f = 0.0 + x[0];
    if (mode == 0) {
        for (int64_t k = 1; k < n; ++k) f = f + x[k];
        return f;
    }
    double c = 0.0;
    for (int64_t k = 1; k < n; ++k) {
        double xi = x[k];
        double t = f + xi;
        if (fabs(f) >= fabs(xi)) c += (f - t) + xi;
        else c += (xi - t) + f;
        f = t;
    }
    if (c != 0.0 && isfinite(c)) f += c;
    return f;
}

/* allocation failure is reported, not dereferenced (the dense DP table is
   ~0.33 GB per 96 x 64 instance; a thread pool of them can exhaust host RAM) */
static void *or_xalloc(void *p, size_t bytes)
{
    if (!p && bytes) {
        fprintf(stderr, "pipeplan_oracle: out of host memory (%zu bytes)\n", bytes);
        abort();
    }
    return p;
}
#define malloc(n) or_xalloc(malloc(n), (size_t)(n))
#define calloc(n, s) or_xalloc(calloc((n), (s)), (size_t)(n) * (size_t)(s))

static inline double pymax2(double a, double b) { return (b > a) ? b : a; }
static inline double pymin2(double a, double b) { return (b < a) ? b : a; }
static inline double BW(const or_inst *I, int a, int b) { return I->bw[(int64_t)a * I->V + b]; }

/* ------------------------------------------------------------------------ */
/* ordering.py:30-91 global_min_cut on the subgraph induced by verts (sorted */
/* ascending indices == ascending GPU ids).  in_a[k] = 1 iff verts[k] lies   */
/* on side_a (the side holding the smallest id).  Returns the cut weight.    */
/* ------------------------------------------------------------------------ */
double or_min_cut(const or_inst *I, const int32_t *verts, int32_t n, uint8_t *in_a)
{
    double *w = (double *)malloc(sizeof(double) * n * n);
    int32_t *grp = (int32_t *)malloc(sizeof(int32_t) * n);
    uint8_t *alive = (uint8_t *)malloc(n);
    uint8_t *best_side = (uint8_t *)calloc(n, 1);
    double *adj = (double *)malloc(sizeof(double) * n);
    uint8_t *in_adj = (uint8_t *)malloc(n);
    for (int a = 0; a < n; ++a) {
        grp[a] = a; alive[a] = 1;
        for (int b = 0; b < n; ++b) w[a * n + b] = (a == b) ? 0.0 : BW(I, verts[a], verts[b]);
    }
    double best_weight = OR_INF;
    int n_alive = n;
    while (n_alive > 1) {
        /* active = sorted(members); start = active[0]  (ordering.py:61-62) */
        int start = -1;
        for (int a = 0; a < n; ++a) if (alive[a]) { start = a; break; }
        int n_adj = 0;
        for (int a = 0; a < n; ++a) {
            in_adj[a] = (alive[a] && a != start);
            if (in_adj[a]) { adj[a] = w[start * n + a]; ++n_adj; }
        }
        int s = start, t = start;
        double cut_of_phase = 0.0;
        while (n_adj > 0) {
            /* next_v = min(adj, key=(-adj[v], v))  (ordering.py:66) */
            int nv = -1;
            for (int a = 0; a < n; ++a) {
                if (!in_adj[a]) continue;
                if (nv < 0 || adj[a] > adj[nv]) nv = a;   /* ascending scan keeps smallest id on ties */
            }
            cut_of_phase = adj[nv];
            in_adj[nv] = 0; --n_adj;
            s = t; t = nv;
            for (int a = 0; a < n; ++a)   /* adj[u] += wt(next_v, u)  (ordering.py:69-70) */
                if (in_adj[a]) adj[a] += w[nv * n + a];
        }
        if (cut_of_phase < best_weight) {   /* ordering.py:73-75 */
            best_weight = cut_of_phase;
            for (int a = 0; a < n; ++a) best_side[a] = (grp[a] == t);
        }
        int merged = s < t ? s : t, other = s < t ? t : s;   /* ordering.py:77-85 */
        for (int u = 0; u < n; ++u) {
            if (!alive[u] || u == s || u == t) continue;
            double v = w[s * n + u] + w[t * n + u];
            w[merged * n + u] = v; w[u * n + merged] = v;
        }
        for (int a = 0; a < n; ++a) if (grp[a] == other) grp[a] = merged;
        alive[other] = 0; --n_alive;
    }
    /* side containing min(verts) == local 0 becomes side_a (ordering.py:87-91) */
    int low_in_side = best_side[0];
    for (int a = 0; a < n; ++a) in_a[a] = low_in_side ? best_side[a] : !best_side[a];
    free(w); free(grp); free(alive); free(best_side); free(adj); free(in_adj);
    return best_weight;
}

static void rdo_rec(const or_inst *I, const int32_t *verts, int32_t n, int32_t rank_low, int32_t *order)
{
    if (n == 1) { order[rank_low - 1] = verts[0]; return; }
    uint8_t *in_a = (uint8_t *)malloc(n);
    or_min_cut(I, verts, n, in_a);
    int32_t *a = (int32_t *)malloc(sizeof(int32_t) * n), *b = (int32_t *)malloc(sizeof(int32_t) * n);
    int na = 0, nb = 0;
    for (int k = 0; k < n; ++k) { if (in_a[k]) a[na++] = verts[k]; else b[nb++] = verts[k]; }
    rdo_rec(I, a, na, rank_low, order);
    rdo_rec(I, b, nb, rank_low + na, order);
    free(in_a); free(a); free(b);
}

/* ordering.py:94-113: order[rank-1] = sorted-id index */
void or_rdo(const or_inst *I, int32_t *order)
{
    int32_t *verts = (int32_t *)malloc(sizeof(int32_t) * I->V);
    for (int k = 0; k < I->V; ++k) verts[k] = k;
    rdo_rec(I, verts, I->V, 1, order);
    free(verts);
}

/* ------------------------------------------------------------------------ */
/* PRM DP  (partition.py:41-162)                                            */
/* ------------------------------------------------------------------------ */
typedef struct {
    const or_inst *I;
    int32_t L, V, M, allow_rep;
    int32_t *order;            /* [V] device order (sorted-id indices) */
    double *prefix;            /* [L+1] partition.py:59-62 */
    double *psum;              /* [L*L] cached sum(param[ls..le]) (cost.py:98) */
    double *minpair;           /* [V*V] min pairwise bw over order[lo..hi] (cost.py:64-71) */
    double *cross;             /* [V*V*V] min cross bw (partition.py:82-93) */
    double *W;                 /* [V][L][V][V] */
    uint8_t *feas;             /* stages is not None */
    int16_t *arg_l, *arg_r;    /* realizing (l_prev, r_prev) */
} or_prm;

#define CELL(P, l, xi, r, i) ((((int64_t)((xi) - 1) * (P)->L + ((l) - 1)) * (P)->V + ((r) - 1)) * (P)->V + ((i) - 1))

static double prm_sync(const or_prm *P, int ls, int le, int lo, int hi)
{
    /* partition.py:70-80 -> cost.py:83-99 */
    int k = hi - lo + 1;
    if (k == 1) return 0.0;
    double total = P->psum[(int64_t)(ls - 1) * P->L + (le - 1)];
    return 2.0 * (double)(k - 1) * total / ((double)k * P->minpair[(lo - 1) * P->V + (hi - 1)]);
}

static double prm_span(const or_prm *P, int lo, int hi) { return P->prefix[hi] - P->prefix[lo - 1]; }

or_prm *or_prm_new(const or_inst *I, const int32_t *order, int32_t allow_rep)
{
    or_prm *P = (or_prm *)calloc(1, sizeof(or_prm));
    int L = I->L, V = I->V, M = I->M;
    P->I = I; P->L = L; P->V = V; P->M = M; P->allow_rep = allow_rep;
    P->order = (int32_t *)malloc(sizeof(int32_t) * V);
    memcpy(P->order, order, sizeof(int32_t) * V);
    P->prefix = (double *)malloc(sizeof(double) * (L + 1));
    P->prefix[0] = 0.0;
    for (int l = 1; l <= L; ++l) P->prefix[l] = P->prefix[l - 1] + I->fwd[l - 1] + I->bwd[l - 1];
    P->psum = (double *)malloc(sizeof(double) * L * L);
    for (int ls = 1; ls <= L; ++ls)
        for (int le = ls; le <= L; ++le)
            P->psum[(int64_t)(ls - 1) * L + (le - 1)] = or_pysum(I->param + ls - 1, le - ls + 1, I->sum_mode);
    P->minpair = (double *)malloc(sizeof(double) * V * V);
    for (int lo = 1; lo <= V; ++lo) {
        double best = OR_INF;
        P->minpair[(lo - 1) * V + (lo - 1)] = best;
        for (int hi = lo + 1; hi <= V; ++hi) {
            for (int a = lo; a < hi; ++a) best = pymin2(best, BW(I, order[a - 1], order[hi - 1]));
            P->minpair[(lo - 1) * V + (hi - 1)] = best;
        }
    }
    /* cross[(rp-1)*V*V + (r-1)*V + (i-1)], valid for rp + r <= i */
    P->cross = (double *)malloc(sizeof(double) * V * V * V);
    for (int i = 1; i <= V; ++i)
        for (int r = 1; r < i; ++r) {
            int lo = i - r + 1;
            double best = OR_INF;
            for (int rp = 1; rp <= i - r; ++rp) {
                int a = lo - 1 - rp + 1;   /* newly added left device (1-based rank) */
                for (int b = lo; b <= i; ++b) best = pymin2(best, BW(I, order[a - 1], order[b - 1]));
                P->cross[((int64_t)(rp - 1) * V + (r - 1)) * V + (i - 1)] = best;
            }
        }
    int64_t ncell = (int64_t)V * L * V * V;
    P->W = (double *)malloc(sizeof(double) * ncell);
    P->feas = (uint8_t *)calloc(ncell, 1);
    P->arg_l = (int16_t *)calloc(ncell, sizeof(int16_t));
    P->arg_r = (int16_t *)calloc(ncell, sizeof(int16_t));
    for (int64_t c = 0; c < ncell; ++c) P->W[c] = OR_INF;

    for (int xi = 1; xi <= V; ++xi) {
        for (int l = 1; l <= L; ++l)
            for (int r = 1; r <= V; ++r)
                for (int i = 1; i <= V; ++i) {
                    int64_t c = CELL(P, l, xi, r, i);
                    if (!allow_rep && r != 1) continue;                 /* partition.py:103-104 */
                    if (l < xi || i < xi) continue;                     /* :115-116 */
                    if (xi == 1 && r == i) {                            /* :117-119 */
                        P->W[c] = (double)M * prm_span(P, 1, l) / (double)i + prm_sync(P, 1, l, 1, i);
                        P->feas[c] = 1;
                        continue;
                    }
                    if (xi == 1 || r == i) continue;                    /* :120-121 */
                    double best = OR_INF;
                    int found = 0, bl = 0, br = 0;
                    int max_rp = allow_rep ? i - r : 1;                 /* :125 */
                    for (int lp = xi - 1; lp <= l - 1; ++lp) {          /* :126 */
                        double stage_w = (double)M * prm_span(P, lp + 1, l) / (double)r;   /* :127 */
                        if (r > 1) stage_w += prm_sync(P, lp + 1, l, i - r + 1, i);       /* :128-129 */
                        double payload = I->efwd[lp - 1] + I->ebwd[lp - 1];               /* :130-131 */
                        for (int rp = 1; rp <= max_rp; ++rp) {          /* :132 */
                            int64_t sc = CELL(P, lp, xi - 1, rp, i - r);
                            if (!P->feas[sc]) continue;                 /* :133-135 */
                            double bw = P->cross[((int64_t)(rp - 1) * V + (r - 1)) * V + (i - 1)];
                            double chan = (double)M * payload / ((double)(rp * r) * bw);       /* :137 */
                            double w = pymax2(pymax2(P->W[sc], chan), stage_w);                /* :138 */
                            if (best > w) { best = w; found = 1; bl = lp; br = rp; }           /* :139-141 */
                        }
                    }
                    if (found) { P->W[c] = best; P->feas[c] = 1; P->arg_l[c] = (int16_t)bl; P->arg_r[c] = (int16_t)br; }
                }
    }
    return P;
}

void or_prm_free(or_prm *P)
{
    if (!P) return;
    free(P->order); free(P->prefix); free(P->psum); free(P->minpair); free(P->cross);
    free(P->W); free(P->feas); free(P->arg_l); free(P->arg_r); free(P);
}

/* Fragments as 4-tuples (layer_start, layer_end, dev_lo, dev_hi) with device
 * ranks 1-based into the order.  Returns 1 feasible / 0 infeasible, -1 bad
 * arguments (partition.py:99-102).  w always written. */
int or_prm_solve(const or_prm *P, int l, int xi, int r, int i, double *w, int32_t *frag)
{
    if (l < 1 || xi < 1 || r < 1 || i < 1) return -1;
    if (l > P->L || i > P->V) return -2;
    if (xi > P->V || r > P->V || r > i) { *w = OR_INF; return 0; }
    int64_t c = CELL(P, l, xi, r, i);
    *w = P->W[c];
    if (!P->feas[c]) return 0;
    /* walk the realizing chain; fragments emitted last-stage first then reversed */
    int cl = l, cx = xi, cr = r, ci = i;
    for (int n = xi; n >= 1; --n) {
        int64_t cc = CELL(P, cl, cx, cr, ci);
        if (cx == 1) {
            frag[4 * (n - 1) + 0] = 1; frag[4 * (n - 1) + 1] = cl;
            frag[4 * (n - 1) + 2] = 1; frag[4 * (n - 1) + 3] = ci;
            break;
        }
        int lp = P->arg_l[cc], rp = P->arg_r[cc];
        frag[4 * (n - 1) + 0] = lp + 1; frag[4 * (n - 1) + 1] = cl;
        frag[4 * (n - 1) + 2] = ci - cr + 1; frag[4 * (n - 1) + 3] = ci;
        cl = lp; ci = ci - cr; cr = rp; cx = cx - 1;
    }
    return 1;
}

double or_prm_W(const or_prm *P, int l, int xi, int r, int i) { return P->W[CELL(P, l, xi, r, i)]; }
int or_prm_feasible(const or_prm *P, int l, int xi, int r, int i) { return P->feas[CELL(P, l, xi, r, i)]; }

/* partition.py:144-162.  Returns 1 with fragments, 0 = (inf, None), -1 bad xi. */
int or_prm_best(const or_prm *P, int xi, double *w, int32_t *frag)
{
    if (xi < 1 || xi > P->V) return -1;
    double best = OR_INF;
    int br = 0;
    for (int r = 1; r <= P->V; ++r) {
        if (!P->allow_rep && r != 1) continue;
        if (xi > P->L) break;
        int64_t c = CELL(P, P->L, xi, r, P->V);
        if (P->feas[c] && best > P->W[c]) { best = P->W[c]; br = r; }
    }
    if (!br) { *w = OR_INF; return 0; }
    return or_prm_solve(P, P->L, xi, br, P->V, w, frag);
}

/* ------------------------------------------------------------------------ */
/* Scheduling  (scheduler.py:49-225, cost.py:205-230)                       */
/* Resources in chain order: index 2n-2 = stage n, 2n-1 = chan n.          */
/* ------------------------------------------------------------------------ */
typedef struct {
    int32_t N;                 /* stages */
    const int32_t *ls, *le;    /* [N] layer intervals (1-based, inclusive) */
    const int32_t *dev_off;    /* [N+1] into devs */
    const int32_t *devs;       /* sorted-id indices */
    int32_t M;
} or_plan;

/* block position -> (resource index, kind) ; kinds: 0 F, 1 X, 2 FB, 3 Y, 4 B */
static void block_info(int N, int pos, int *res, int *kind, int *stage_or_chan)
{
    if (N == 1) { *res = 0; *kind = 2; *stage_or_chan = 1; return; }
    if (pos <= 2 * N - 2) {
        int n = (pos + 1) / 2;
        if (pos & 1) { *res = 2 * n - 2; *kind = 0; } else { *res = 2 * n - 1; *kind = 1; }
        *stage_or_chan = n;
    } else if (pos == 2 * N - 1) {
        *res = 2 * N - 2; *kind = 2; *stage_or_chan = N;
    } else {
        int q = pos - (2 * N - 1);          /* 1.. : Y_{N-1}, B_{N-1}, Y_{N-2}, ... */
        int n = N - (q + 1) / 2;
        if (q & 1) { *res = 2 * n - 1; *kind = 3; } else { *res = 2 * n - 2; *kind = 4; }
        *stage_or_chan = n;
    }
}

static double min_cross(const or_inst *I, const or_plan *p, int n)   /* cost.py:74-80 */
{
    double best = OR_INF;
    for (int a = p->dev_off[n - 1]; a < p->dev_off[n]; ++a)
        for (int b = p->dev_off[n]; b < p->dev_off[n + 1]; ++b)
            best = pymin2(best, BW(I, p->devs[a], p->devs[b]));
    return best;
}

static double min_pair(const or_inst *I, const int32_t *d, int k)   /* cost.py:64-71 */
{
    double best = OR_INF;
    for (int a = 0; a < k; ++a)
        for (int b = a + 1; b < k; ++b) best = pymin2(best, BW(I, d[a], d[b]));
    return best;
}

static double stage_allreduce(const or_inst *I, const or_plan *p, int n)   /* cost.py:83-99 */
{
    int k = p->dev_off[n] - p->dev_off[n - 1];
    if (k == 1) return 0.0;
    double total = or_pysum(I->param + p->ls[n - 1] - 1, p->le[n - 1] - p->ls[n - 1] + 1, I->sum_mode);
    return 2.0 * (double)(k - 1) * total / ((double)k * min_pair(I, p->devs + p->dev_off[n - 1], k));
}

/* cost.py:205-224; dur[pos] for pos 1..J */
static void block_durations(const or_inst *I, const or_plan *p, double *dur)
{
    int N = p->N, J = 4 * N - 3;
    for (int pos = 1; pos <= J; ++pos) {
        int res, kind, sc;
        block_info(N, pos, &res, &kind, &sc);
        if (kind == 0 || kind == 2 || kind == 4) {
            int n = sc, k = p->dev_off[n] - p->dev_off[n - 1];
            int cnt = p->le[n - 1] - p->ls[n - 1] + 1;
            double sf = or_pysum(I->fwd + p->ls[n - 1] - 1, cnt, I->sum_mode) / (double)k;   /* cost.py:47 */
            double sb = or_pysum(I->bwd + p->ls[n - 1] - 1, cnt, I->sum_mode) / (double)k;   /* cost.py:53 */
            if (kind == 0) dur[pos] = sf / (double)k;
            else if (kind == 4) dur[pos] = sb / (double)k;
            else dur[pos] = (sf + sb) / (double)k;                                          /* cost.py:61 */
        } else {
            int n = sc;
            int kl = p->dev_off[n] - p->dev_off[n - 1], kr = p->dev_off[n + 1] - p->dev_off[n];
            double denom = (double)(kl * kr) * min_cross(I, p, n);                            /* cost.py:121-122 */
            int edge = p->le[n - 1];
            dur[pos] = (kind == 1 ? I->efwd[edge - 1] : I->ebwd[edge - 1]) / denom;         /* cost.py:123 */
        }
    }
}

/* scheduler.py:75-106: q_off[2N] (+1) offsets, q_items pairs (m, pos) */
void or_pe_queues(int32_t N, int32_t M, int32_t *q_off, int32_t *q_items)
{
    int J = 4 * N - 3, R = 2 * N - 1;
    /* count per resource, then fill in pass order */
    int32_t *cnt = (int32_t *)calloc(R, sizeof(int32_t));
    for (int pos = 1; pos <= J; ++pos) { int res, kind, sc; block_info(N, pos, &res, &kind, &sc); cnt[res] += M; }
    q_off[0] = 0;
    for (int r = 0; r < R; ++r) q_off[r + 1] = q_off[r] + cnt[r];
    int32_t *fill = (int32_t *)calloc(R, sizeof(int32_t));
    /* pending deques: head/tail counters per position (microbatches enter in order) */
    int32_t *head = (int32_t *)calloc(J + 2, sizeof(int32_t)), *tail = (int32_t *)calloc(J + 2, sizeof(int32_t));
    int32_t **pend = (int32_t **)malloc(sizeof(int32_t *) * (J + 2));
    for (int pos = 1; pos <= J; ++pos) pend[pos] = (int32_t *)malloc(sizeof(int32_t) * M);
    for (int m = 1; m <= M; ++m) pend[1][tail[1]++] = m;
    int64_t remaining = (int64_t)M * J;
    while (remaining) {
        for (int pos = J; pos >= 1; --pos) {
            if (head[pos] == tail[pos]) continue;
            int m = pend[pos][head[pos]++];
            --remaining;
            int res, kind, sc; block_info(N, pos, &res, &kind, &sc);
            int32_t at = q_off[res] + fill[res]++;
            q_items[2 * at] = m; q_items[2 * at + 1] = pos;
            if (pos < J) pend[pos + 1][tail[pos + 1]++] = m;
        }
    }
    for (int pos = 1; pos <= J; ++pos) free(pend[pos]);
    free(pend); free(head); free(tail); free(cnt); free(fill);
}

/* heap entry: (time, cls, resource-name rank, m, pos, start) ordering (scheduler.py:161-164) */
typedef struct { double t; int cls, rrank, m, pos; double start; int res; } hent;

static int hless(const hent *a, const hent *b)
{
    if (a->t != b->t) return a->t < b->t;
    if (a->cls != b->cls) return a->cls < b->cls;
    if (a->rrank != b->rrank) return a->rrank < b->rrank;
    if (a->m != b->m) return a->m < b->m;
    if (a->pos != b->pos) return a->pos < b->pos;
    return a->start < b->start;
}
static void hpush(hent *h, int *n, hent e)
{
    int k = (*n)++;
    h[k] = e;
    while (k > 0) { int p = (k - 1) / 2; if (!hless(&h[k], &h[p])) break; hent t = h[k]; h[k] = h[p]; h[p] = t; k = p; }
}
static hent hpop(hent *h, int *n)
{
    hent top = h[0];
    h[0] = h[--(*n)];
    int k = 0;
    for (;;) {
        int l = 2 * k + 1, r = l + 1, s = k;
        if (l < *n && hless(&h[l], &h[s])) s = l;
        if (r < *n && hless(&h[r], &h[s])) s = r;
        if (s == k) break;
        hent t = h[k]; h[k] = h[s]; h[s] = t; k = s;
    }
    return top;
}

typedef struct {
    int32_t status;            /* 0 ok, 1 stalled */
    int64_t n_done;            /* executions completed */
    int32_t *head_m, *head_pos;/* [R] first unserved queue item per resource (0 if queue drained) */
    int32_t n_events;
    double *ev_start, *ev_end; /* [M*J] in the reference's final sorted order */
    int32_t *ev_m, *ev_pos;
    int32_t n_ar;
    int32_t *ar_stage; double *ar_start, *ar_end;   /* [N] */
    double makespan;
} or_sim_out;

/* rank of each resource name under Python string ordering of "stageN"/"chanN" */
static void resource_name_ranks(int N, int *rank)
{
    int R = 2 * N - 1;
    char (*names)[24] = malloc(sizeof(*names) * R);
    for (int r = 0; r < R; ++r) {
        if ((r & 1) == 0) snprintf(names[r], 24, "stage%d", r / 2 + 1);
        else snprintf(names[r], 24, "chan%d", r / 2 + 1);
    }
    for (int r = 0; r < R; ++r) {
        int k = 0;
        for (int q = 0; q < R; ++q) if (strcmp(names[q], names[r]) < 0) ++k;
        rank[r] = k;
    }
    free(names);
}

typedef struct { double start; int reskey; int m; int64_t seq; int pos; double end; } evrec;
static int ev_cmp(const void *a, const void *b)
{
    const evrec *x = (const evrec *)a, *y = (const evrec *)b;
    if (x->start != y->start) return x->start < y->start ? -1 : 1;
    if (x->reskey != y->reskey) return x->reskey < y->reskey ? -1 : 1;
    if (x->m != y->m) return x->m < y->m ? -1 : 1;
    return x->seq < y->seq ? -1 : (x->seq > y->seq);   /* stable over raw (pop) order */
}

/* scheduler.py:121-225.  Queue items must lie on their own block's resource
 * and 1 <= m <= M, 1 <= pos <= J (checked by the caller). */
int or_simulate(const or_inst *I, const or_plan *p, const int32_t *q_off, const int32_t *q_items,
                int32_t forward_barrier, or_sim_out *out)
{
    int N = p->N, M = p->M, J = 4 * N - 3, R = 2 * N - 1;
    double *dur = (double *)malloc(sizeof(double) * (J + 1));
    block_durations(I, p, dur);
    double *ar_time = (double *)malloc(sizeof(double) * (N + 1));
    uint8_t *has_ar = (uint8_t *)calloc(N + 1, 1);
    for (int n = 1; n <= N; ++n) {
        int k = p->dev_off[n] - p->dev_off[n - 1];
        if (k >= 2) { has_ar[n] = 1; ar_time[n] = stage_allreduce(I, p, n); }
    }
    int *rrank = (int *)malloc(sizeof(int) * R);
    resource_name_ranks(N, rrank);
    int *sorted_res = (int *)malloc(sizeof(int) * R);
    for (int r = 0; r < R; ++r) sorted_res[rrank[r]] = r;

    int32_t *qh = (int32_t *)calloc(R, sizeof(int32_t));
    uint8_t *busy = (uint8_t *)calloc(R, 1);
    int64_t nexec = (int64_t)M * J;
    uint8_t *done = (uint8_t *)calloc(nexec + 1, 1);
    double *dstart = (double *)malloc(sizeof(double) * (nexec + 1));
    double *dend = (double *)malloc(sizeof(double) * (nexec + 1));
    int64_t n_done = 0;
    int32_t *remaining_compute = (int32_t *)calloc(N + 1, sizeof(int32_t));
    for (int n = 1; n <= N; ++n) remaining_compute[n] = q_off[2 * n - 1] - q_off[2 * n - 2];
    double *ar_start = (double *)malloc(sizeof(double) * (N + 1));
    evrec *raw = (evrec *)malloc(sizeof(evrec) * (nexec + 1));
    int64_t n_raw = 0;
    int64_t fwd_left = (int64_t)M * 2 * (N - 1);
    int barrier_open = (!forward_barrier) || fwd_left == 0;
    hent *heap = (hent *)malloc(sizeof(hent) * (R + 1));
    int hn = 0;
#define EXEC(m, pos) (((int64_t)(m) - 1) * J + (pos) - 1)

    /* try_start (scheduler.py:166-178) */
#define TRY_START(res_, t_) do { \
        int rs = (res_); double tt = (t_); \
        if (!busy[rs] && qh[rs] < q_off[rs + 1] - q_off[rs]) { \
            int32_t at = q_off[rs] + qh[rs]; \
            int m = q_items[2 * at], pos = q_items[2 * at + 1]; \
            int bres, bkind, bsc; block_info(N, pos, &bres, &bkind, &bsc); \
            int ok = 1; \
            if (!barrier_open && !(bkind == 0 || bkind == 1)) ok = 0; \
            if (ok && pos > 1 && !done[EXEC(m, pos - 1)]) ok = 0; \
            if (ok) { \
                qh[rs]++; busy[rs] = 1; \
                hent e; e.t = tt + dur[pos]; e.cls = (bkind == 1 || bkind == 3) ? 0 : 1; \
                e.rrank = rrank[rs]; e.m = m; e.pos = pos; e.start = tt; e.res = rs; \
                hpush(heap, &hn, e); \
            } \
        } } while (0)

    for (int k = 0; k < R; ++k) TRY_START(sorted_res[k], 0.0);
    while (hn) {
        hent e = hpop(heap, &hn);
        int bres, bkind, bsc; block_info(N, e.pos, &bres, &bkind, &bsc);
        int64_t x = EXEC(e.m, e.pos);
        if (!done[x]) ++n_done;
        done[x] = 1; dstart[x] = e.start; dend[x] = e.t;
        evrec ev; ev.start = e.start; ev.end = e.t; ev.m = e.m; ev.pos = e.pos; ev.seq = n_raw;
        ev.reskey = (bres & 1) ? (1 << 20) + (bres / 2 + 1) : (bres / 2 + 1);   /* scheduler.py:115-118 */
        raw[n_raw++] = ev;
        busy[e.res] = 0;
        int newly_open = 0;
        if (forward_barrier && !barrier_open && (bkind == 0 || bkind == 1)) {
            if (--fwd_left == 0) { barrier_open = 1; newly_open = 1; }
        }
        if (bkind == 0 || bkind == 2 || bkind == 4) {
            if (--remaining_compute[bsc] == 0 && has_ar[bsc]) ar_start[bsc] = e.t;
        }
        if (newly_open) {
            for (int k = 0; k < R; ++k) TRY_START(sorted_res[k], e.t);
        } else {
            TRY_START(e.res, e.t);
            if (e.pos < J) { int nr, nk, ns; block_info(N, e.pos + 1, &nr, &nk, &ns); TRY_START(nr, e.t); }
        }
    }
#undef TRY_START
    out->n_done = n_done;
    out->n_events = 0; out->n_ar = 0; out->makespan = 0.0;
    int status = 0;
    if (n_done != nexec) {
        status = 1;
        for (int r = 0; r < R; ++r) {
            if (qh[r] < q_off[r + 1] - q_off[r]) {
                int32_t at = q_off[r] + qh[r];
                out->head_m[r] = q_items[2 * at]; out->head_pos[r] = q_items[2 * at + 1];
            } else { out->head_m[r] = 0; out->head_pos[r] = 0; }
        }
    } else {
        double finish = -OR_INF; int first = 1;
        for (int m = 1; m <= M; ++m) {
            double v = dend[EXEC(m, J)];
            if (first || v > finish) { finish = v; first = 0; }
        }
        double mk = finish;
        for (int n = 1; n <= N; ++n) if (has_ar[n]) {
            out->ar_stage[out->n_ar] = n; out->ar_start[out->n_ar] = ar_start[n];
            out->ar_end[out->n_ar] = ar_start[n] + ar_time[n];
            mk = pymax2(mk, out->ar_end[out->n_ar]);
            out->n_ar++;
        }
        out->makespan = mk;
        qsort(raw, n_raw, sizeof(evrec), ev_cmp);
        for (int64_t k = 0; k < n_raw; ++k) {
            out->ev_start[k] = raw[k].start; out->ev_end[k] = raw[k].end;
            out->ev_m[k] = raw[k].m; out->ev_pos[k] = raw[k].pos;
        }
        out->n_events = (int32_t)n_raw;
    }
    out->status = status;
#undef EXEC
    free(dur); free(ar_time); free(has_ar); free(rrank); free(sorted_res); free(qh); free(busy);
    free(done); free(dstart); free(dend); free(remaining_compute); free(ar_start); free(raw); free(heap);
    return status;
}

/* scheduler.py:234-238 -> cost.py:172-202 */
double or_lemma1_bound(const or_inst *I, const or_plan *p)
{
    int N = p->N;
    double cycle = 0.0; int have = 0;
    double ar_max = 0.0; int have_ar = 0;
    for (int n = 1; n <= N; ++n) {
        int k = p->dev_off[n] - p->dev_off[n - 1];
        int cnt = p->le[n - 1] - p->ls[n - 1] + 1;
        double sf = or_pysum(I->fwd + p->ls[n - 1] - 1, cnt, I->sum_mode) / (double)k;
        double sb = or_pysum(I->bwd + p->ls[n - 1] - 1, cnt, I->sum_mode) / (double)k;
        double c = sf + sb;
        if (!have || c > cycle) { cycle = c; have = 1; }
        if (k >= 2) {
            double a = stage_allreduce(I, p, n);
            if (!have_ar || a > ar_max) { ar_max = a; have_ar = 1; }
        }
    }
    for (int n = 1; n < N; ++n) {
        int kl = p->dev_off[n] - p->dev_off[n - 1], kr = p->dev_off[n + 1] - p->dev_off[n];
        double denom = (double)(kl * kr) * min_cross(I, p, n);
        int edge = p->le[n - 1];
        double c = I->efwd[edge - 1] / denom + I->ebwd[edge - 1] / denom;
        if (c > cycle) cycle = c;
    }
    return (double)(p->M + 4 * N - 4) * cycle + ar_max;
}

/* cost.py:126-142 */
double or_phi(const or_inst *I)
{
    int L = I->L, V = I->V;
    double p_max = 0.0, d_max = 0.0;
    double *tot = (double *)malloc(sizeof(double) * L);
    for (int l = 0; l < L; ++l) {
        tot[l] = I->fwd[l] + I->bwd[l];
        if (l == 0 || tot[l] > p_max) p_max = tot[l];
    }
    for (int e = 0; e < L - 1; ++e) {
        double d = I->efwd[e] + I->ebwd[e];
        if (e == 0 || d > d_max) d_max = d;
    }
    double bmin = 0.0, bmax = 0.0; int have = 0;
    for (int a = 0; a < V; ++a)
        for (int b = a + 1; b < V; ++b) {
            double x = BW(I, a, b);
            if (!have) { bmin = bmax = x; have = 1; }
            else { if (x < bmin) bmin = x; if (x > bmax) bmax = x; }
        }
    double g = or_pysum(tot, L, I->sum_mode) / (double)V;
    free(tot);
    if (V == 1 || bmin == bmax) return 0.0;
    return pymax2(p_max * bmax, d_max) / g * (1.0 / bmin - 1.0 / bmax);
}

/* ------------------------------------------------------------------------ */
/* spp  (planner.py:57-88)                                                  */
/* ------------------------------------------------------------------------ */
typedef struct {
    int32_t *order;            /* [V] */
    uint8_t *feasible;         /* [V] */
    double *workload, *makespan, *bound;   /* [V] (makespan/bound undefined if infeasible) */
    int32_t best_xi;
    int32_t *frag;             /* [4V] best plan fragments (ls, le, dev_lo, dev_hi) */
    double best_makespan, phi, theorem_factor;
    or_sim_out sim;            /* best schedule (caller allocates arrays sized for M*(4V-3)) */
} or_spp_out;

static void frag_to_plan(const int32_t *frag, int xi, const int32_t *order, int M,
                         int32_t *ls, int32_t *le, int32_t *dev_off, int32_t *devs, or_plan *p)
{
    dev_off[0] = 0;
    for (int n = 0; n < xi; ++n) {
        ls[n] = frag[4 * n]; le[n] = frag[4 * n + 1];
        int lo = frag[4 * n + 2], hi = frag[4 * n + 3];
        dev_off[n + 1] = dev_off[n] + (hi - lo + 1);
        for (int d = lo; d <= hi; ++d) devs[dev_off[n] + d - lo] = order[d - 1];
    }
    p->N = xi; p->ls = ls; p->le = le; p->dev_off = dev_off; p->devs = devs; p->M = M;
}

int or_spp(const or_inst *I, or_spp_out *out)
{
    int V = I->V, M = I->M;
    or_rdo(I, out->order);
    or_prm *P = or_prm_new(I, out->order, 1);
    int32_t *frag = (int32_t *)malloc(sizeof(int32_t) * 4 * V);
    int32_t *ls = (int32_t *)malloc(sizeof(int32_t) * V), *le = (int32_t *)malloc(sizeof(int32_t) * V);
    int32_t *dev_off = (int32_t *)malloc(sizeof(int32_t) * (V + 1)), *devs = (int32_t *)malloc(sizeof(int32_t) * V);
    int J_max = 4 * V - 3;
    int32_t *q_off = (int32_t *)malloc(sizeof(int32_t) * (2 * V));
    int32_t *q_items = (int32_t *)malloc(sizeof(int32_t) * 2 * (int64_t)M * J_max);
    or_sim_out tmp;
    int64_t cap = (int64_t)M * J_max;
    tmp.head_m = (int32_t *)malloc(sizeof(int32_t) * 2 * V); tmp.head_pos = (int32_t *)malloc(sizeof(int32_t) * 2 * V);
    tmp.ev_start = (double *)malloc(sizeof(double) * cap); tmp.ev_end = (double *)malloc(sizeof(double) * cap);
    tmp.ev_m = (int32_t *)malloc(sizeof(int32_t) * cap); tmp.ev_pos = (int32_t *)malloc(sizeof(int32_t) * cap);
    tmp.ar_stage = (int32_t *)malloc(sizeof(int32_t) * V); tmp.ar_start = (double *)malloc(sizeof(double) * V);
    tmp.ar_end = (double *)malloc(sizeof(double) * V);
    int best_xi = 0;
    double best_mk = 0.0;
    for (int xi = 1; xi <= V; ++xi) {
        double w;
        int ok = or_prm_best(P, xi, &w, frag);
        out->workload[xi - 1] = w;
        out->feasible[xi - 1] = (ok == 1);
        if (ok != 1) { out->makespan[xi - 1] = OR_INF; out->bound[xi - 1] = OR_INF; continue; }
        or_plan plan;
        frag_to_plan(frag, xi, out->order, M, ls, le, dev_off, devs, &plan);
        or_pe_queues(xi, M, q_off, q_items);
        or_simulate(I, &plan, q_off, q_items, 0, &tmp);
        out->makespan[xi - 1] = tmp.makespan;
        out->bound[xi - 1] = or_lemma1_bound(I, &plan);
        if (best_xi == 0 || tmp.makespan < best_mk) {       /* planner.py:76 */
            best_xi = xi; best_mk = tmp.makespan;
            memcpy(out->frag, frag, sizeof(int32_t) * 4 * xi);
            if (out->sim.ev_start) {
                out->sim.status = tmp.status; out->sim.n_done = tmp.n_done;
                out->sim.n_events = tmp.n_events; out->sim.n_ar = tmp.n_ar; out->sim.makespan = tmp.makespan;
                memcpy(out->sim.ev_start, tmp.ev_start, sizeof(double) * tmp.n_events);
                memcpy(out->sim.ev_end, tmp.ev_end, sizeof(double) * tmp.n_events);
                memcpy(out->sim.ev_m, tmp.ev_m, sizeof(int32_t) * tmp.n_events);
                memcpy(out->sim.ev_pos, tmp.ev_pos, sizeof(int32_t) * tmp.n_events);
                memcpy(out->sim.ar_stage, tmp.ar_stage, sizeof(int32_t) * tmp.n_ar);
                memcpy(out->sim.ar_start, tmp.ar_start, sizeof(double) * tmp.n_ar);
                memcpy(out->sim.ar_end, tmp.ar_end, sizeof(double) * tmp.n_ar);
            }
        }
    }
    out->best_xi = best_xi;
    out->best_makespan = best_mk;
    out->phi = or_phi(I);
    out->theorem_factor = (2.0 + (4.0 * V - 4.0) / (double)M) * (1.0 + out->phi);   /* planner.py:52-54,86 */
    free(tmp.head_m); free(tmp.head_pos); free(tmp.ev_start); free(tmp.ev_end); free(tmp.ev_m); free(tmp.ev_pos);
    free(tmp.ar_stage); free(tmp.ar_start); free(tmp.ar_end);
    free(frag); free(ls); free(le); free(dev_off); free(devs); free(q_off); free(q_items);
    or_prm_free(P);
    return best_xi;
}

/* ------------------------------------------------------------------------ */
/* Thread-pool batch driver for the CPU baseline: spp over n instances.     */
/* ------------------------------------------------------------------------ */
typedef struct {
    const or_inst *insts; int n; double *makespan; int32_t *best_xi;
    int next; pthread_mutex_t mu;
} batch_ctx;

static void *batch_worker(void *arg)
{
    batch_ctx *c = (batch_ctx *)arg;
    for (;;) {
        pthread_mutex_lock(&c->mu);
        int k = c->next++;
        pthread_mutex_unlock(&c->mu);
        if (k >= c->n) break;
        const or_inst *I = &c->insts[k];
        int V = I->V;
        or_spp_out o;
        memset(&o, 0, sizeof(o));
        o.order = (int32_t *)malloc(sizeof(int32_t) * V);
        o.feasible = (uint8_t *)malloc(V);
        o.workload = (double *)malloc(sizeof(double) * V);
        o.makespan = (double *)malloc(sizeof(double) * V);
        o.bound = (double *)malloc(sizeof(double) * V);
        o.frag = (int32_t *)malloc(sizeof(int32_t) * 4 * V);
        c->best_xi[k] = or_spp(I, &o);
        c->makespan[k] = o.best_makespan;
        free(o.order); free(o.feasible); free(o.workload); free(o.makespan); free(o.bound); free(o.frag);
    }
    return NULL;
}

int or_spp_batch(int32_t n, const or_inst *insts, double *makespan, int32_t *best_xi, int32_t nthreads)
{
    batch_ctx c;
    c.insts = insts; c.n = n; c.makespan = makespan; c.best_xi = best_xi; c.next = 0;
    pthread_mutex_init(&c.mu, NULL);
    if (nthreads < 1) nthreads = 1;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * nthreads);
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, batch_worker, &c);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(th);
    pthread_mutex_destroy(&c.mu);
    return 0;
}

/* plain simulate_pe (scheduler.py:228-231) over a batch of plans of one
 * instance on a thread pool: the CPU baseline for the C5 simulation config. */
typedef struct {
    const or_inst *I; const or_plan *plans; int n; double *makespan; int next; pthread_mutex_t mu;
} simb_ctx;

static void *simb_worker(void *arg)
{
    simb_ctx *c = (simb_ctx *)arg;
    for (;;) {
        pthread_mutex_lock(&c->mu);
        int k = c->next++;
        pthread_mutex_unlock(&c->mu);
        if (k >= c->n) break;
        const or_plan *p = &c->plans[k];
        int N = p->N, M = p->M, J = 4 * N - 3;
        int64_t cap = (int64_t)M * J;
        int32_t *q_off = (int32_t *)malloc(sizeof(int32_t) * (2 * N));
        int32_t *q_items = (int32_t *)malloc(sizeof(int32_t) * 2 * cap);
        or_pe_queues(N, M, q_off, q_items);
        or_sim_out o;
        o.head_m = (int32_t *)malloc(sizeof(int32_t) * 2 * N); o.head_pos = (int32_t *)malloc(sizeof(int32_t) * 2 * N);
        o.ev_start = (double *)malloc(sizeof(double) * cap); o.ev_end = (double *)malloc(sizeof(double) * cap);
        o.ev_m = (int32_t *)malloc(sizeof(int32_t) * cap); o.ev_pos = (int32_t *)malloc(sizeof(int32_t) * cap);
        o.ar_stage = (int32_t *)malloc(sizeof(int32_t) * N); o.ar_start = (double *)malloc(sizeof(double) * N);
        o.ar_end = (double *)malloc(sizeof(double) * N);
        or_simulate(c->I, p, q_off, q_items, 0, &o);
        c->makespan[k] = o.makespan;
        free(q_off); free(q_items); free(o.head_m); free(o.head_pos); free(o.ev_start); free(o.ev_end);
        free(o.ev_m); free(o.ev_pos); free(o.ar_stage); free(o.ar_start); free(o.ar_end);
    }
    return NULL;
}

int or_simulate_pe_batch(const or_inst *I, int32_t n, const or_plan *plans, double *makespan, int32_t nthreads)
{
    simb_ctx c;
    c.I = I; c.plans = plans; c.n = n; c.makespan = makespan; c.next = 0;
    pthread_mutex_init(&c.mu, NULL);
    if (nthreads < 1) nthreads = 1;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * nthreads);
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, simb_worker, &c);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(th);
    pthread_mutex_destroy(&c.mu);
    return 0;
}

/*
 * CPU ORACLE -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's hot-path algorithms, used as the
 * parity checker by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg (and as the `--impl reference` CPU arm). Nothing in the product path
 * (paper_2410_05534_b200/) links or calls this file.
 *
 * Restated functions (reference = /root/reference/pkg/src/esat/):
 *   oracle_rebuild_batch  egraph.py:93-115  UnionFind.find/union (rank ties -> lower id)
 *                         egraph.py:203-226 EGraph.rebuild (insertion-ordered hashcons scan with
 *                                           the live union-find, first entry survives)
 *                         egraph.py:228-238 _regroup + egraph.py:65-70 node_sort_key order
 *   oracle_ematch_batch   rewrite.py:353-393 _match_param_spec/_match_in_class,
 *                         rewrite.py:396-433 _subst_key dedup + sort (joint_match for 1 pattern)
 *   oracle_joint_batch    rewrite.py:405-433 joint_match for >= 2 source patterns
 *   oracle_extract_batch  extraction.py:121-154 _greedy_fixpoint (Gauss-Seidel passes, cap 4C+8),
 *                         extraction.py:157-166 default node cost, extraction.py:184-242 OCF
 *                         (Alg. 2), extraction.py:67-115 validation/reachability
 *
 * Pinned against the reference itself: the tests/golden fixtures were produced by
 * running the reference (tests/golden/make_golden.py); tests/test_oracle_golden.py
 * checks this file against every vector.
 *
 * Data layout: the packed batch arena of paper_2410_05534_b200/arena.py and
 * include/esat_b200.h (per-leaf bases; CSR offset arrays carry n+1 entries per
 * leaf, so leaf l's offsets start at base[l] + l).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define NONE 0xFFFFFFFFu

enum { X_OK = 0, X_NOT_CONVERGED = 1, X_INFEASIBLE = 2, X_CYCLIC = 3, X_CHILD_NOT_CHOSEN = 4,
       X_ROOT_NOT_CHOSEN = 5, X_NO_ROOT = 6 };

/* ------------------------------------------------------------------------ */
/* union-find (egraph.py:80-115)                                             */

static uint32_t uf_find(uint32_t* parent, uint32_t x) {
    uint32_t r = x;
    while (parent[r] != r) r = parent[r];
    while (parent[x] != r) { uint32_t nx = parent[x]; parent[x] = r; x = nx; }
    return r;
}

static uint32_t uf_union(uint32_t* parent, uint8_t* rank, uint32_t a, uint32_t b) {
    uint32_t ra = uf_find(parent, a), rb = uf_find(parent, b);
    if (ra == rb) return ra;
    if (rank[ra] < rank[rb]) { uint32_t t = ra; ra = rb; rb = t; }
    else if (rank[ra] == rank[rb]) {
        if (rb < ra) { uint32_t t = ra; ra = rb; rb = t; }
        rank[ra]++;
    }
    parent[rb] = ra;
    return ra;
}

/* ------------------------------------------------------------------------ */
/* node-key hash map (canon_map of egraph.py:209)                            */

typedef struct {
    uint32_t* slot;   /* entry index or NONE */
    uint32_t mask;
} kmap;

static uint64_t key_hash(uint32_t sym, const uint32_t* k, uint32_t a) {
    uint64_t h = 0x9E3779B97F4A7C15ull ^ (uint64_t)sym * 0xff51afd7ed558ccdull;
    for (uint32_t i = 0; i < a; i++) {
        h ^= (uint64_t)k[i] + 0x632BE59BD9B4E019ull + (h << 6) + (h >> 2);
        h *= 0xc4ceb9fe1a85ec53ull;
    }
    return h ^ (h >> 29) ^ a;
}

static void kmap_init(kmap* m, uint32_t n) {
    uint32_t cap = 16;
    while (cap < 2 * n + 2) cap <<= 1;
    m->slot = (uint32_t*)malloc(sizeof(uint32_t) * cap);
    memset(m->slot, 0xff, sizeof(uint32_t) * cap);
    m->mask = cap - 1;
}

/* ------------------------------------------------------------------------ */
/* rebuild (egraph.py:203-238)                                               */

typedef struct {
    uint32_t n;
    uint32_t *sym, *koff, *kids, *cid;
    double* cost;
} hclist;

static int rebuild_leaf(uint32_t n0, const uint32_t* sym0, const uint32_t* koff0, const uint32_t* kids0,
                        const uint32_t* cid0, const double* cost0, uint32_t* parent, uint8_t* rank,
                        hclist* out, uint32_t* merges_out) {
    uint32_t K0 = koff0[n0];
    /* working copies; each pass reads `cur` and writes `nxt` (never larger) */
    hclist cur, nxt;
    cur.sym = (uint32_t*)malloc(4 * (n0 + 1)); cur.koff = (uint32_t*)malloc(4 * (n0 + 1));
    cur.kids = (uint32_t*)malloc(4 * (K0 + 1)); cur.cid = (uint32_t*)malloc(4 * (n0 + 1));
    cur.cost = (double*)malloc(8 * (n0 + 1));
    nxt.sym = (uint32_t*)malloc(4 * (n0 + 1)); nxt.koff = (uint32_t*)malloc(4 * (n0 + 1));
    nxt.kids = (uint32_t*)malloc(4 * (K0 + 1)); nxt.cid = (uint32_t*)malloc(4 * (n0 + 1));
    nxt.cost = (double*)malloc(8 * (n0 + 1));
    memcpy(cur.sym, sym0, 4 * n0); memcpy(cur.koff, koff0, 4 * (n0 + 1));
    memcpy(cur.kids, kids0, 4 * K0); memcpy(cur.cid, cid0, 4 * n0); memcpy(cur.cost, cost0, 8 * n0);
    cur.n = n0;
    uint32_t* key = (uint32_t*)malloc(4 * (K0 + 1));
    kmap m;
    kmap_init(&m, n0);
    uint32_t total = 0;
    for (;;) {
        int merged = 0;
        memset(m.slot, 0xff, sizeof(uint32_t) * (m.mask + 1));
        uint32_t ne = 0, nk = 0;
        nxt.koff[0] = 0;
        for (uint32_t i = 0; i < cur.n; i++) {
            uint32_t a = cur.koff[i + 1] - cur.koff[i];
            for (uint32_t j = 0; j < a; j++) key[j] = uf_find(parent, cur.kids[cur.koff[i] + j]);
            uint32_t c = uf_find(parent, cur.cid[i]);
            uint64_t h = key_hash(cur.sym[i], key, a);
            uint32_t s = (uint32_t)h & m.mask, hit = NONE;
            for (;; s = (s + 1) & m.mask) {
                uint32_t e = m.slot[s];
                if (e == NONE) break;
                uint32_t ea = nxt.koff[e + 1] - nxt.koff[e];
                if (nxt.sym[e] == cur.sym[i] && ea == a &&
                    memcmp(nxt.kids + nxt.koff[e], key, 4 * a) == 0) { hit = e; break; }
            }
            if (hit == NONE) {
                m.slot[s] = ne;
                nxt.sym[ne] = cur.sym[i];
                memcpy(nxt.kids + nk, key, 4 * a);
                nk += a;
                nxt.koff[ne + 1] = nk;
                nxt.cid[ne] = c;
                nxt.cost[ne] = cur.cost[i];
                ne++;
            } else if (uf_find(parent, nxt.cid[hit]) != c) {
                nxt.cid[hit] = uf_union(parent, rank, uf_find(parent, nxt.cid[hit]), c);
                merged = 1;
                total++;
            }
        }
        nxt.n = ne;
        for (uint32_t e = 0; e < ne; e++) nxt.cid[e] = uf_find(parent, nxt.cid[e]);
        hclist t = cur; cur = nxt; nxt = t;
        if (!merged) break;
    }
    out->n = cur.n;
    memcpy(out->sym, cur.sym, 4 * cur.n);
    memcpy(out->koff, cur.koff, 4 * (cur.n + 1));
    memcpy(out->kids, cur.kids, 4 * cur.koff[cur.n]);
    memcpy(out->cid, cur.cid, 4 * cur.n);
    memcpy(out->cost, cur.cost, 8 * cur.n);
    *merges_out = total;
    free(cur.sym); free(cur.koff); free(cur.kids); free(cur.cid); free(cur.cost);
    free(nxt.sym); free(nxt.koff); free(nxt.kids); free(nxt.cid); free(nxt.cost);
    free(key); free(m.slot);
    return 0;
}

/* node order inside a class: (rank(name, repr(payload)), children tuple) -- egraph.py:65-70 */
typedef struct {
    const uint32_t* rank_of_sym;
    const hclist* hc;
} sort_ctx;

static int node_cmp(const sort_ctx* sc, uint32_t a, uint32_t b) {
    const hclist* h = sc->hc;
    if (h->cid[a] != h->cid[b]) return h->cid[a] < h->cid[b] ? -1 : 1;
    uint32_t ra = sc->rank_of_sym[h->sym[a]], rb = sc->rank_of_sym[h->sym[b]];
    if (ra != rb) return ra < rb ? -1 : 1;
    uint32_t na = h->koff[a + 1] - h->koff[a], nb = h->koff[b + 1] - h->koff[b];
    const uint32_t *ka = h->kids + h->koff[a], *kb = h->kids + h->koff[b];
    for (uint32_t i = 0; i < na && i < nb; i++)
        if (ka[i] != kb[i]) return ka[i] < kb[i] ? -1 : 1;
    return na < nb ? -1 : (na > nb ? 1 : 0);
}

static void sort_nodes(const sort_ctx* sc, uint32_t* idx, uint32_t n, uint32_t* tmp) {
    /* stable merge sort */
    if (n < 2) return;
    uint32_t h = n / 2;
    sort_nodes(sc, idx, h, tmp);
    sort_nodes(sc, idx + h, n - h, tmp);
    uint32_t i = 0, j = h, k = 0;
    while (i < h && j < n) tmp[k++] = node_cmp(sc, idx[j], idx[i]) < 0 ? idx[j++] : idx[i++];
    while (i < h) tmp[k++] = idx[i++];
    while (j < n) tmp[k++] = idx[j++];
    memcpy(idx, tmp, 4 * n);
}

int oracle_rebuild_batch(uint32_t L, const uint64_t* nb, const uint64_t* kb, const uint64_t* ub,
                         const uint32_t* rank_of_sym,
                         const uint32_t* hc_sym, const uint32_t* hc_koff, const uint32_t* hc_kids,
                         const uint32_t* hc_cid, const double* hc_cost,
                         uint32_t* uf_parent, uint8_t* uf_rank, const uint32_t* root,
                         uint32_t* o_n, uint32_t* o_merges, uint32_t* o_sym, uint32_t* o_koff,
                         uint32_t* o_kids, uint32_t* o_cid, double* o_cost,
                         uint32_t* v_C, uint32_t* v_root, uint32_t* cls_id, uint32_t* cls_off,
                         uint32_t* nd_sym, uint32_t* nd_koff, uint32_t* nd_kpos, double* nd_cost,
                         uint32_t* nd_hc, int n_threads) {
#ifdef _OPENMP
    if (n_threads > 0) omp_set_num_threads(n_threads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (uint32_t l = 0; l < L; l++) {
        uint64_t b = nb[l], k0 = kb[l], u0 = ub[l];
        uint32_t n = (uint32_t)(nb[l + 1] - b), U = (uint32_t)(ub[l + 1] - u0);
        uint32_t* parent = uf_parent + u0;
        uint8_t* rnk = uf_rank + u0;
        hclist out = {0, o_sym + b, o_koff + b + l, o_kids + k0, o_cid + b, o_cost + b};
        rebuild_leaf(n, hc_sym + b, hc_koff + b + l, hc_kids + k0, hc_cid + b, hc_cost + b, parent, rnk,
                     &out, &o_merges[l]);
        o_n[l] = out.n;
        /* regroup -> clean view (classes ascending by id; nodes by node_sort_key) */
        uint32_t ne = out.n;
        uint32_t* idx = (uint32_t*)malloc(4 * (ne + 1));
        uint32_t* tmp = (uint32_t*)malloc(4 * (ne + 1));
        for (uint32_t i = 0; i < ne; i++) idx[i] = i;
        sort_ctx sc = {rank_of_sym, &out};
        sort_nodes(&sc, idx, ne, tmp);
        uint32_t* pos_of = (uint32_t*)malloc(4 * (U + 1));
        for (uint32_t i = 0; i < U; i++) pos_of[i] = NONE;
        uint32_t C = 0;
        uint32_t* cid_l = cls_id + b;
        uint32_t* coff_l = cls_off + b + l;
        for (uint32_t j = 0; j < ne; j++) {
            uint32_t c = out.cid[idx[j]];
            if (pos_of[c] == NONE) { pos_of[c] = C; cid_l[C] = c; coff_l[C] = j; C++; }
        }
        coff_l[C] = ne;
        v_C[l] = C;
        uint32_t* nko = nd_koff + b + l;
        uint32_t kk = 0;
        nko[0] = 0;
        for (uint32_t j = 0; j < ne; j++) {
            uint32_t e = idx[j];
            nd_sym[b + j] = out.sym[e];
            nd_cost[b + j] = out.cost[e];
            nd_hc[b + j] = e;
            for (uint32_t q = out.koff[e]; q < out.koff[e + 1]; q++)
                nd_kpos[k0 + kk++] = pos_of[uf_find(parent, out.kids[q])];
            nko[j + 1] = kk;
        }
        v_root[l] = root[l] == NONE ? NONE : pos_of[uf_find(parent, root[l])];
        free(idx); free(tmp); free(pos_of);
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* e-matching (rewrite.py:353-433)                                            */

typedef struct {
    /* clean view of one leaf */
    uint32_t C;
    const uint32_t *cls_id, *cls_off, *nd_sym, *nd_koff, *nd_kpos;
    /* symbol table */
    const uint32_t *s_name, *s_arity, *s_poff;
    const int32_t* s_par;
    /* pattern program */
    const int32_t* prog;
    int32_t P, V, Q;
    /* state */
    uint32_t vars[64];
    int32_t pv[64];
    uint8_t pv_set[64];
    uint32_t root;
    /* output */
    uint32_t* buf;
    uint64_t n, cap; /* in records */
    uint32_t W;
} mstate;

#define REC(ms, i) ((ms)->prog + 3 + 6 * (i))

static void emit(mstate* ms) {
    if (ms->n == ms->cap) {
        ms->cap = ms->cap ? 2 * ms->cap : 64;
        ms->buf = (uint32_t*)realloc(ms->buf, 4 * ms->cap * ms->W);
    }
    uint32_t* r = ms->buf + ms->n * ms->W;
    r[0] = ms->root;
    for (int v = 0; v < ms->V; v++) r[1 + v] = ms->vars[v];
    for (int q = 0; q < ms->Q; q++) r[1 + ms->V + q] = (uint32_t)ms->pv[q];
    ms->n++;
}

/* goal stack of (pattern node, class position) pairs, solved depth-first */
static void solve(mstate* ms, uint32_t* gp, uint32_t* gc, int top) {
    if (top == 0) { emit(ms); return; }
    top--;
    uint32_t pn = gp[top], cpos = gc[top];
    const int32_t* rec = REC(ms, pn);
    uint32_t cid = ms->cls_id[cpos];
    if (rec[0] == 0) { /* Var */
        int v = rec[1];
        if (ms->vars[v] == NONE) {
            ms->vars[v] = cid;
            solve(ms, gp, gc, top);
            ms->vars[v] = NONE;
        } else if (ms->vars[v] == cid) {
            solve(ms, gp, gc, top);
        }
        gp[top] = pn; gc[top] = cpos; /* keep the caller's stack intact */
        return;
    }
    int32_t name = rec[1], arity = rec[2], nslots = rec[3];
    const int32_t* slots = ms->prog + rec[4];
    const int32_t* kids = ms->prog + rec[5];
    for (uint32_t nd = ms->cls_off[cpos]; nd < ms->cls_off[cpos + 1]; nd++) {
        uint32_t s = ms->nd_sym[nd];
        if ((int32_t)ms->s_name[s] != name || (int32_t)ms->s_arity[s] != arity) continue;
        uint64_t newly = 0; /* pvars bound here */
        int ok = 1;
        if (nslots >= 0) {
            uint32_t np = ms->s_poff[s + 1] - ms->s_poff[s];
            if ((int32_t)np != nslots) continue;
            const int32_t* actual = ms->s_par + ms->s_poff[s];
            for (int j = 0; j < nslots && ok; j++) {
                int32_t sl = slots[j];
                if (sl >= 0) { ok = (sl == actual[j]); }
                else {
                    int q = -sl - 1;
                    if (!ms->pv_set[q]) { ms->pv_set[q] = 1; ms->pv[q] = actual[j]; newly |= 1ull << q; }
                    else ok = (ms->pv[q] == actual[j]);
                }
            }
        }
        if (ok) {
            /* push children in reverse so child 0 is solved first (pre-order binding) */
            for (int j = arity - 1; j >= 0; j--) {
                gp[top + (arity - 1 - j)] = (uint32_t)kids[j];
                gc[top + (arity - 1 - j)] = ms->nd_kpos[ms->nd_koff[nd] + j];
            }
            solve(ms, gp, gc, top + arity);
        }
        for (int q = 0; q < 64; q++) if (newly >> q & 1) ms->pv_set[q] = 0;
    }
    /* restore the goal we consumed (callers re-use the stack) */
    gp[top] = pn; gc[top] = cpos;
}

static int rec_cmp_W;
static int rec_cmp(const void* a, const void* b) {
    const uint32_t *x = (const uint32_t*)a, *y = (const uint32_t*)b;
    for (int i = 0; i < rec_cmp_W; i++) if (x[i] != y[i]) return x[i] < y[i] ? -1 : 1;
    return 0;
}

static int cmpW(const uint32_t* x, const uint32_t* y, uint32_t W) {
    for (uint32_t i = 0; i < W; i++) if (x[i] != y[i]) return x[i] < y[i] ? -1 : 1;
    return 0;
}

static void sort_records(uint32_t* buf, uint64_t n, uint32_t W) {
    /* insertion sort for the tiny per-root lists, merge sort otherwise */
    if (n < 2) return;
    if (n <= 24) {
        uint32_t tmp[256];
        for (uint64_t i = 1; i < n; i++) {
            memcpy(tmp, buf + i * W, 4 * W);
            uint64_t j = i;
            while (j > 0 && cmpW(buf + (j - 1) * W, tmp, W) > 0) { memcpy(buf + j * W, buf + (j - 1) * W, 4 * W); j--; }
            memcpy(buf + j * W, tmp, 4 * W);
        }
        return;
    }
    uint64_t h = n / 2;
    sort_records(buf, h, W);
    sort_records(buf + h * W, n - h, W);
    uint32_t* t = (uint32_t*)malloc(4 * n * W);
    uint64_t i = 0, j = h, k = 0;
    while (i < h && j < n) {
        if (cmpW(buf + j * W, buf + i * W, W) < 0) memcpy(t + (k++) * W, buf + (j++) * W, 4 * W);
        else memcpy(t + (k++) * W, buf + (i++) * W, 4 * W);
    }
    while (i < h) memcpy(t + (k++) * W, buf + (i++) * W, 4 * W);
    while (j < n) memcpy(t + (k++) * W, buf + (j++) * W, 4 * W);
    memcpy(buf, t, 4 * n * W);
    free(t);
}

static uint64_t uniq_records(uint32_t* buf, uint64_t n, uint32_t W) {
    if (n == 0) return 0;
    uint64_t o = 1;
    for (uint64_t i = 1; i < n; i++)
        if (cmpW(buf + (o - 1) * W, buf + i * W, W) != 0) { if (o != i) memcpy(buf + o * W, buf + i * W, 4 * W); o++; }
    return o;
}

/* all matches of one pattern in one leaf, sorted + deduplicated; caller frees *out */
static uint64_t ematch_leaf(mstate* ms, uint32_t** out) {
    uint32_t gp[256], gc[256];
    ms->buf = NULL; ms->n = 0; ms->cap = 0;
    for (int v = 0; v < 64; v++) { ms->vars[v] = NONE; ms->pv_set[v] = 0; }
    uint64_t done = 0;
    for (uint32_t r = 0; r < ms->C; r++) {
        ms->root = ms->cls_id[r];
        gp[0] = 0; gc[0] = r;
        solve(ms, gp, gc, 1);
        /* sort/dedup this root's slice (the root is the leading key: rewrite.py:396-397) */
        uint64_t cnt = ms->n - done;
        sort_records(ms->buf + done * ms->W, cnt, ms->W);
        cnt = uniq_records(ms->buf + done * ms->W, cnt, ms->W);
        ms->n = done + cnt;
        done = ms->n;
    }
    *out = ms->buf;
    return ms->n;
}

static void mstate_init(mstate* ms, uint32_t l, const uint64_t* nb, const uint64_t* kb, const uint32_t* v_C,
                        const uint32_t* cls_id, const uint32_t* cls_off, const uint32_t* nd_sym,
                        const uint32_t* nd_koff, const uint32_t* nd_kpos, const uint32_t* s_name,
                        const uint32_t* s_arity, const uint32_t* s_poff, const int32_t* s_par, const int32_t* prog) {
    uint64_t b = nb[l];
    ms->C = v_C[l];
    ms->cls_id = cls_id + b;
    ms->cls_off = cls_off + b + l;
    /* node indices in cls_off are leaf-relative; shift array bases accordingly */
    ms->nd_sym = nd_sym + b;
    ms->nd_koff = nd_koff + b + l;
    ms->nd_kpos = nd_kpos + kb[l];
    ms->s_name = s_name; ms->s_arity = s_arity; ms->s_poff = s_poff; ms->s_par = s_par;
    ms->prog = prog;
    ms->P = prog[0]; ms->V = prog[1]; ms->Q = prog[2];
    ms->W = 1 + ms->V + ms->Q;
}

/* Single-pattern e-match over every leaf. Output: records of W = 1+V+Q words,
 * leaf l's records at out_words[out_off[l] .. out_off[l+1]) (word offsets).
 * Returns 0, or 3 (capacity) with the required word count in out_off[L]. */
int oracle_ematch_batch(uint32_t L, const uint64_t* nb, const uint64_t* kb, const uint32_t* v_C,
                        const uint32_t* cls_id, const uint32_t* cls_off, const uint32_t* nd_sym,
                        const uint32_t* nd_koff, const uint32_t* nd_kpos,
                        const uint32_t* s_name, const uint32_t* s_arity, const uint32_t* s_poff,
                        const int32_t* s_par, const int32_t* prog,
                        uint64_t cap_words, uint32_t* out_words, uint64_t* out_off, uint32_t* out_count,
                        int n_threads) {
    uint32_t** res = (uint32_t**)calloc(L, sizeof(uint32_t*));
    uint64_t* cnt = (uint64_t*)calloc(L, sizeof(uint64_t));
    uint32_t W = 1 + prog[1] + prog[2];
#ifdef _OPENMP
    if (n_threads > 0) omp_set_num_threads(n_threads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (uint32_t l = 0; l < L; l++) {
        mstate ms;
        mstate_init(&ms, l, nb, kb, v_C, cls_id, cls_off, nd_sym, nd_koff, nd_kpos, s_name, s_arity, s_poff, s_par, prog);
        cnt[l] = ematch_leaf(&ms, &res[l]);
    }
    uint64_t acc = 0;
    for (uint32_t l = 0; l < L; l++) { out_off[l] = acc; out_count[l] = (uint32_t)cnt[l]; acc += cnt[l] * W; }
    out_off[L] = acc;
    int rc = 0;
    if (acc > cap_words) rc = 3;
    else for (uint32_t l = 0; l < L; l++) if (cnt[l]) memcpy(out_words + out_off[l], res[l], 4 * cnt[l] * W);
    for (uint32_t l = 0; l < L; l++) free(res[l]);
    free(res); free(cnt);
    return rc;
}

/* Joint match of S >= 2 source patterns (rewrite.py:405-433) as per-source matching + join.
 * progs: concatenated programs, prog_off[s] = word offset of source s.
 * var_map[vmo[s] + v] = output var slot of source s's var v; same for pvars (pmo).
 * Output record: [S roots][NV vars][NQ pvars], sorted by (roots, vars, pvars) = _subst_key. */
int oracle_joint_batch(uint32_t L, const uint64_t* nb, const uint64_t* kb, const uint32_t* v_C,
                       const uint32_t* cls_id, const uint32_t* cls_off, const uint32_t* nd_sym,
                       const uint32_t* nd_koff, const uint32_t* nd_kpos,
                       const uint32_t* s_name, const uint32_t* s_arity, const uint32_t* s_poff,
                       const int32_t* s_par, uint32_t S, const int32_t* progs, const uint32_t* prog_off,
                       const uint32_t* var_map, const uint32_t* vmo, const uint32_t* pvar_map, const uint32_t* pmo,
                       uint32_t NV, uint32_t NQ,
                       uint64_t cap_words, uint32_t* out_words, uint64_t* out_off, uint32_t* out_count,
                       int n_threads) {
    uint32_t W = S + NV + NQ;
    uint32_t** res = (uint32_t**)calloc(L, sizeof(uint32_t*));
    uint64_t* cnt = (uint64_t*)calloc(L, sizeof(uint64_t));
#ifdef _OPENMP
    if (n_threads > 0) omp_set_num_threads(n_threads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (uint32_t l = 0; l < L; l++) {
        uint32_t* lists[16];
        uint64_t lens[16];
        uint32_t Ws[16];
        int empty = 0;
        for (uint32_t s = 0; s < S; s++) {
            mstate ms;
            mstate_init(&ms, l, nb, kb, v_C, cls_id, cls_off, nd_sym, nd_koff, nd_kpos, s_name, s_arity, s_poff,
                        s_par, progs + prog_off[s]);
            lens[s] = ematch_leaf(&ms, &lists[s]);
            Ws[s] = ms.W;
            if (!lens[s]) empty = 1;
        }
        uint32_t* buf = NULL;
        uint64_t n = 0, cap = 0;
        if (!empty) {
            /* odometer over the S lists with incremental consistency checks */
            uint64_t it[16] = {0};
            uint32_t rec[256];
            uint8_t setv[256], setq[256];
            uint32_t depth = 0;
            memset(setv, 0, sizeof setv); memset(setq, 0, sizeof setq);
            /* iterative DFS */
            it[0] = 0;
            for (;;) {
                if (it[depth] == lens[depth]) {
                    if (depth == 0) break;
                    depth--;
                    it[depth]++;
                    continue;
                }
                /* recompute bindings for levels 0..depth from scratch (S is tiny) */
                memset(setv, 0, NV); memset(setq, 0, NQ);
                int ok = 1;
                for (uint32_t s = 0; s <= depth && ok; s++) {
                    const uint32_t* m = lists[s] + it[s] * Ws[s];
                    const int32_t* pg = progs + prog_off[s];
                    int Vs = pg[1], Qs = pg[2];
                    rec[s] = m[0];
                    for (int v = 0; v < Vs && ok; v++) {
                        uint32_t o = var_map[vmo[s] + v];
                        if (!setv[o]) { setv[o] = 1; rec[S + o] = m[1 + v]; }
                        else ok = rec[S + o] == m[1 + v];
                    }
                    for (int q = 0; q < Qs && ok; q++) {
                        uint32_t o = pvar_map[pmo[s] + q];
                        if (!setq[o]) { setq[o] = 1; rec[S + NV + o] = m[1 + Vs + q]; }
                        else ok = rec[S + NV + o] == m[1 + Vs + q];
                    }
                }
                if (!ok) { it[depth]++; continue; }
                if (depth + 1 == S) {
                    if (n == cap) { cap = cap ? 2 * cap : 256; buf = (uint32_t*)realloc(buf, 4 * cap * W); }
                    memcpy(buf + n * W, rec, 4 * W);
                    n++;
                    it[depth]++;
                } else {
                    depth++;
                    it[depth] = 0;
                }
            }
        }
        sort_records(buf, n, W);
        n = uniq_records(buf, n, W);
        res[l] = buf;
        cnt[l] = n;
        for (uint32_t s = 0; s < S; s++) free(lists[s]);
    }
    uint64_t acc = 0;
    for (uint32_t l = 0; l < L; l++) { out_off[l] = acc; out_count[l] = (uint32_t)cnt[l]; acc += cnt[l] * W; }
    out_off[L] = acc;
    int rc = 0;
    if (acc > cap_words) rc = 3;
    else for (uint32_t l = 0; l < L; l++) if (cnt[l]) memcpy(out_words + out_off[l], res[l], 4 * cnt[l] * W);
    for (uint32_t l = 0; l < L; l++) free(res[l]);
    free(res); free(cnt);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* greedy extraction (extraction.py:121-242)                                 */

typedef struct { uint32_t key; double val; } hent;
typedef struct { hent* e; uint32_t n, cap; } hmap; /* sorted by key */

static void hmap_reserve(hmap* h, uint32_t n) {
    if (n > h->cap) { h->cap = n + 16; h->e = (hent*)realloc(h->e, sizeof(hent) * h->cap); }
}

static int hmap_find(const hmap* h, uint32_t key) {
    int lo = 0, hi = (int)h->n - 1;
    while (lo <= hi) {
        int mid = (lo + hi) >> 1;
        if (h->e[mid].key == key) return mid;
        if (h->e[mid].key < key) lo = mid + 1; else hi = mid - 1;
    }
    return -1;
}

static double pymax(double a, double b) { return b > a ? b : a; } /* Python max(a, b) */

typedef struct {
    uint32_t C;
    const uint32_t *cls_off, *nd_koff, *nd_kpos;
    const double* nd_cost;
    double* cost;
    /* OCF state (ConstituentHistory) */
    hmap* hist;
    uint8_t* present;
    double best_cost;
    hmap best, cand;
    uint32_t prev;
} xstate;

/* ocf_enode_cost (extraction.py:184-226); the node's history is built into xs->cand */
static double ocf_node(xstate* xs, uint32_t nd, uint32_t k) {
    if (xs->prev != k) {
        if (xs->prev != NONE) {
            hmap* dst = &xs->hist[xs->prev];
            hmap_reserve(dst, xs->best.n);
            memcpy(dst->e, xs->best.e, sizeof(hent) * xs->best.n);
            dst->n = xs->best.n;
            xs->present[xs->prev] = 1;
        }
        xs->best_cost = INFINITY;
        xs->best.n = 0;
    }
    xs->prev = k;
    hmap* H = &xs->cand;
    H->n = 0;
    double v = xs->nd_cost[nd];
    hmap merged = {0, 0, 0};
    for (uint32_t q = xs->nd_koff[nd]; q < xs->nd_koff[nd + 1]; q++) {
        uint32_t c = xs->nd_kpos[q];
        if (hmap_find(H, c) >= 0) continue; /* case 1 */
        double cc;
        if (xs->present[c]) { /* case 2 */
            const hmap* hc = &xs->hist[c];
            double m = 0.0;
            hmap_reserve(&merged, H->n + hc->n + 1);
            uint32_t i = 0, j = 0, o = 0;
            while (i < H->n || j < hc->n) {
                if (j == hc->n || (i < H->n && H->e[i].key < hc->e[j].key)) merged.e[o++] = H->e[i++];
                else if (i == H->n || hc->e[j].key < H->e[i].key) merged.e[o++] = hc->e[j++];
                else { m = pymax(m, hc->e[j].val); merged.e[o++] = H->e[i++]; j++; }
            }
            merged.n = o;
            hmap t = *H; *H = merged; merged = t;
            cc = pymax(xs->cost[c] - m, 0.0);
        } else { /* case 3 */
            cc = xs->cost[c];
        }
        /* enode_hist[child] = child_cost (insert or overwrite) */
        int at = hmap_find(H, c);
        if (at >= 0) H->e[at].val = cc;
        else {
            hmap_reserve(H, H->n + 1);
            uint32_t p = H->n;
            while (p > 0 && H->e[p - 1].key > c) { H->e[p] = H->e[p - 1]; p--; }
            H->e[p].key = c; H->e[p].val = cc;
            H->n++;
        }
        v = v + cc;
    }
    free(merged.e);
    if (v < xs->best_cost) {
        hmap t = xs->best; xs->best = xs->cand; xs->cand = t;
        xs->best_cost = v;
    }
    return v;
}

static double default_node(xstate* xs, uint32_t nd) {
    double v = xs->nd_cost[nd];
    for (uint32_t q = xs->nd_koff[nd]; q < xs->nd_koff[nd + 1]; q++) v = v + xs->cost[xs->nd_kpos[q]];
    return v;
}

int oracle_extract_batch(uint32_t L, const uint64_t* nb, const uint64_t* kb, const uint32_t* v_C,
                         const uint32_t* v_root, const uint32_t* cls_id, const uint32_t* cls_off,
                         const uint32_t* nd_koff, const uint32_t* nd_kpos, const double* nd_cost, int method,
                         uint32_t* status, uint32_t* err_class, double* root_cost, double* class_cost,
                         uint32_t* choice, uint8_t* reachable, uint32_t* passes_out, int n_threads) {
#ifdef _OPENMP
    if (n_threads > 0) omp_set_num_threads(n_threads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (uint32_t l = 0; l < L; l++) {
        uint64_t b = nb[l];
        uint32_t C = v_C[l];
        xstate xs;
        memset(&xs, 0, sizeof xs);
        xs.C = C;
        xs.cls_off = cls_off + b + l;
        xs.nd_koff = nd_koff + b + l;
        xs.nd_kpos = nd_kpos + kb[l];
        xs.nd_cost = nd_cost + b;
        xs.cost = class_cost + b;
        uint32_t* ch = choice + b;
        uint8_t* reach = reachable + b;
        for (uint32_t k = 0; k < C; k++) { xs.cost[k] = INFINITY; ch[k] = NONE; reach[k] = 0; }
        if (method == 1) {
            xs.hist = (hmap*)calloc(C + 1, sizeof(hmap));
            xs.present = (uint8_t*)calloc(C + 1, 1);
            xs.prev = NONE;
            xs.best_cost = INFINITY;
        }
        uint64_t cap = 4ull * C + 8;
        uint32_t st = X_NOT_CONVERGED, passes = 0;
        for (uint64_t it = 0; it < cap; it++) {
            int changed = 0;
            passes++;
            for (uint32_t k = 0; k < C; k++) {
                double bv = INFINITY;
                uint32_t bn = NONE;
                for (uint32_t nd = xs.cls_off[k]; nd < xs.cls_off[k + 1]; nd++) {
                    double v = method == 1 ? ocf_node(&xs, nd, k) : default_node(&xs, nd);
                    if (bn == NONE || v < bv) { bv = v; bn = nd; }
                }
                if (bn != NONE && bv < xs.cost[k]) { xs.cost[k] = bv; ch[k] = bn; changed = 1; }
            }
            if (!changed) { st = X_OK; break; }
        }
        passes_out[l] = passes;
        err_class[l] = NONE;
        root_cost[l] = NAN;
        uint32_t root = v_root[l];
        if (st == X_OK && root == NONE) st = X_NO_ROOT;
        if (st == X_OK && !isfinite(xs.cost[root])) st = X_INFEASIBLE;
        if (st == X_OK) {
            root_cost[l] = xs.cost[root];
            /* _reachable_chosen (extraction.py:106-115) */
            uint32_t* stack = (uint32_t*)malloc(4 * (xs.nd_koff[xs.cls_off[C]] + 2));
            uint32_t sp = 0;
            stack[sp++] = root;
            while (sp) {
                uint32_t c = stack[--sp];
                if (reach[c]) continue;
                reach[c] = 1;
                uint32_t nd = ch[c];
                for (uint32_t q = xs.nd_koff[nd]; q < xs.nd_koff[nd + 1]; q++) stack[sp++] = xs.nd_kpos[q];
            }
            free(stack);
            /* validate_extraction (extraction.py:67-87): recursive DFS, children in stored order */
            uint8_t* state = (uint8_t*)calloc(C + 1, 1);
            uint32_t* vs = (uint32_t*)malloc(4 * (C + 2));
            uint32_t* vi = (uint32_t*)malloc(4 * (C + 2));
            uint32_t d = 0;
            vs[0] = root; vi[0] = 0; state[root] = 1;
            d = 1;
            while (d && st == X_OK) {
                uint32_t c = vs[d - 1];
                uint32_t nd = ch[c];
                uint32_t a = xs.nd_koff[nd + 1] - xs.nd_koff[nd];
                if (vi[d - 1] == a) { state[c] = 2; d--; continue; }
                uint32_t kid = xs.nd_kpos[xs.nd_koff[nd] + vi[d - 1]];
                vi[d - 1]++;
                if (state[kid] == 2) continue;
                if (state[kid] == 1) { st = X_CYCLIC; err_class[l] = cls_id[b + kid]; break; }
                if (ch[kid] == NONE) { st = X_CHILD_NOT_CHOSEN; err_class[l] = cls_id[b + kid]; break; }
                state[kid] = 1;
                vs[d] = kid; vi[d] = 0; d++;
            }
            free(state); free(vs); free(vi);
        }
        status[l] = st;
        if (method == 1) {
            for (uint32_t k = 0; k <= C; k++) free(xs.hist[k].e);
            free(xs.hist); free(xs.present); free(xs.best.e); free(xs.cand.e);
        }
    }
    return 0;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

// K11: the apply loop of one MCTS rollout step -- apply_rule (rewrite.py:526-570) on every leaf
// of a rebuilt batch, each leaf with its own rule, writing the leaf's dirty state (the input of
// the next rebuild) in place of the batch's previous input.
//
// Per leaf the reference is strictly sequential: every match of the rule, in the sorted
// joint_match order, sees the adds and unions of the matches before it (hashcons hits, class
// membership for the cycle test, union-find roots). So one thread owns one leaf and replays
// that order exactly; leaves run in parallel. The leaf state lives in the batch arrays:
//   read:  rebuild output hashcons (o_*), working union-find (uf_parent/uf_rank), match lists
//   write: hc_* (insertion-ordered hashcons, new entries appended), uf_*_in, per-leaf counts
// Class membership (EGraph.classes[c].nodes, needed by would_create_cycle, rewrite.py:492-505)
// is a linked list of hashcons entries per class root; union concatenates lists (egraph.py:
// 189-201). class_shape (rewrite.py:286-290) is the shape of the head entry's symbol (tensor
// e-classes are shape-homogeneous). Symbols are looked up by their identity key (apply.py).
#include <cstdio>

#include "esat_internal.cuh"
#include "k_apply_args.cuh"

namespace esat {

namespace {

// debug-build bounds checks (ESAT_DEBUG): report and skip the access instead of faulting
#ifdef ESAT_DEBUG
#define ABAD(cond) ((cond) ? (printf("k_apply leaf %u line %d: %s\n", L.l, __LINE__, #cond), true) : false)
#else
#define ABAD(cond) false
#endif

constexpr int INSTR = 20;
constexpr int MAXI = 24;      // instructions per target
constexpr uint32_t PLAN_CH = 32, PLAN_T = 2;   // matches planned per chunk (one per lane); targets per match
constexpr uint32_t PMAX = 12;                  // instructions per target planned by the planner warp
constexpr uint32_t PW = 3 * PMAX + 1;          // its plan words per target: symbol ids, f64 node costs, flags
constexpr uint32_t PLAN_FAIL = 0xFFFFFFFDu;    // make_symbol fails (or, with PLAN_SLOW, is not interned)
constexpr uint32_t PLAN_SLOW = 1u, PLAN_SHAPE_ERR = 2u, PLAN_SHAPE_MISMATCH = 4u;
constexpr uint32_t NO_SHAPE = 255;
enum Op : int { OP_UNK = 0, OP_INPUT, OP_WEIGHT, OP_EWADD, OP_EWMUL, OP_MATMUL, OP_CONV2D, OP_RELU, OP_TANH,
                OP_SIGMOID, OP_CONCAT, OP_SPLIT, OP_MAXPOOL, OP_TRANSPOSE, OP_NOOP };
constexpr int32_t INT_NONE = (int32_t)0x80000000;

struct Shape {
    uint32_t nd;   // NO_SHAPE: None
    uint32_t d[4];
};

struct Sym {            // a symbol under construction (make_symbol)
    int32_t name;       // name id (-1: never interned)
    uint32_t arity, np;
    uint32_t code[3];   // attribute codes (NO_MATCH_CODE: value absent from the table)
    int32_t ival[3];    // attribute integer values
    Shape shape;
};

struct Leaf {
    const Dev* d;
    const AArgs* a;
    uint32_t l, cap_n, cap_k, cap_u;
    uint32_t n, K, U;                 // live sizes
    uint32_t *sym, *koff, *kids, *cid;
    double* cost;
    uint32_t* parent;
    uint8_t* rank;
    uint32_t *head, *tail, *next, *seen, *stack, *tab;
    uint32_t *pot, *phead, *ptail, *pnext, *eown;   // cycle-test potentials + parent edges (below)
    uint32_t tmask, stamp, lane;
    bool changed, usepot;
};

__device__ __forceinline__ uint32_t find(Leaf& L, uint32_t x) {
    if (ABAD(x >= L.U)) return 0;
    return uf_find(L.parent, x);
}

__device__ Shape sym_shape(const AArgs& a, uint32_t s) {
    Shape sh;
    sh.nd = a.sym_ndim[s];
    for (int i = 0; i < 4; i++) sh.d[i] = a.sym_dims[4 * s + i];
    return sh;
}

__device__ __forceinline__ Shape class_shape(Leaf& L, uint32_t c) {
    const uint32_t e = L.head[find(L, c)];
    Shape sh;
    sh.nd = NO_SHAPE;
    if (e == NONE) return sh;
    if (ABAD(e >= L.n)) return sh;
    return sym_shape(*L.a, L.sym[e]);
}

__device__ __forceinline__ bool shape_eq(const Shape& x, const Shape& y) {
    if (x.nd != y.nd) return false;
    if (x.nd == NO_SHAPE) return true;
    for (uint32_t i = 0; i < x.nd; i++)
        if (x.d[i] != y.d[i]) return false;
    return true;
}

// infer_shape (tensor_ir.py:64-126); false = ShapeError
__device__ bool infer_shape(int op, const Sym& s, const Shape* in, uint32_t nin, Shape& out) {
    if (op == OP_UNK || op == OP_INPUT || op == OP_WEIGHT) return false;
    const uint32_t expect = op == OP_NOOP ? (nin > 1 ? nin : 1u)
                            : (op == OP_RELU || op == OP_TANH || op == OP_SIGMOID || op == OP_SPLIT ||
                               op == OP_MAXPOOL || op == OP_TRANSPOSE)
                                ? 1u : 2u;
    if (nin != expect) return false;
    for (uint32_t i = 0; i < nin; i++) {   // check_shape: 1..4 dims, all >= 1
        if (in[i].nd == NO_SHAPE || in[i].nd < 1 || in[i].nd > 4) return false;
        for (uint32_t j = 0; j < in[i].nd; j++)
            if (in[i].d[j] < 1) return false;
    }
    out.nd = NO_SHAPE;
    switch (op) {
        case OP_EWADD: case OP_EWMUL:
            if (!shape_eq(in[0], in[1])) return false;
            out = in[0];
            return true;
        case OP_MATMUL:
            if (in[0].nd != 2 || in[1].nd != 2 || in[0].d[1] != in[1].d[0]) return false;
            out.nd = 2; out.d[0] = in[0].d[0]; out.d[1] = in[1].d[1];
            return true;
        case OP_CONV2D: {
            if (in[0].nd != 4 || in[1].nd != 4) return false;
            if (in[0].d[1] != in[1].d[1]) return false;
            if (s.ival[0] == INT_NONE || s.ival[1] == INT_NONE) return false;
            const int64_t stride = s.ival[0], pad = s.ival[1];
            if (stride == 0) return false;
            // Python floor division
            auto fdiv = [](int64_t x, int64_t y) { int64_t q = x / y; if ((x % y != 0) && ((x < 0) != (y < 0))) q--; return q; };
            const int64_t oh = fdiv((int64_t)in[0].d[2] + 2 * pad - in[1].d[2], stride) + 1;
            const int64_t ow = fdiv((int64_t)in[0].d[3] + 2 * pad - in[1].d[3], stride) + 1;
            if (oh < 1 || ow < 1) return false;
            out.nd = 4; out.d[0] = in[0].d[0]; out.d[1] = in[1].d[0]; out.d[2] = (uint32_t)oh; out.d[3] = (uint32_t)ow;
            return true;
        }
        case OP_RELU: case OP_TANH: case OP_SIGMOID: case OP_NOOP:
            out = in[0];
            return true;
        case OP_TRANSPOSE:
            if (in[0].nd != 2) return false;
            out.nd = 2; out.d[0] = in[0].d[1]; out.d[1] = in[0].d[0];
            return true;
        case OP_CONCAT: {
            if (s.ival[0] == INT_NONE) return false;
            const int64_t ax = s.ival[0];
            if (in[0].nd != in[1].nd || ax < 0 || ax >= (int64_t)in[0].nd) return false;
            for (uint32_t j = 0; j < in[0].nd; j++)
                if ((int64_t)j != ax && in[0].d[j] != in[1].d[j]) return false;
            out = in[0];
            out.d[ax] = in[0].d[ax] + in[1].d[ax];
            return true;
        }
        case OP_SPLIT: {
            if (s.ival[0] == INT_NONE || s.ival[1] == INT_NONE) return false;
            const int64_t ax = s.ival[0], idx = s.ival[1];
            if (ax < 0 || ax >= (int64_t)in[0].nd) return false;
            if (idx != 0 && idx != 1) return false;
            if (in[0].d[ax] % 2 != 0) return false;
            out = in[0];
            out.d[ax] = in[0].d[ax] / 2;
            return true;
        }
        case OP_MAXPOOL: {
            if (s.ival[0] == INT_NONE || s.ival[1] == INT_NONE) return false;
            const int64_t k = s.ival[0], st = s.ival[1];
            if (in[0].nd != 4 || st == 0) return false;
            auto fdiv = [](int64_t x, int64_t y) { int64_t q = x / y; if ((x % y != 0) && ((x < 0) != (y < 0))) q--; return q; };
            const int64_t oh = fdiv((int64_t)in[0].d[2] - k, st) + 1, ow = fdiv((int64_t)in[0].d[3] - k, st) + 1;
            if (oh < 1 || ow < 1) return false;
            out.nd = 4; out.d[0] = in[0].d[0]; out.d[1] = in[0].d[1]; out.d[2] = (uint32_t)oh; out.d[3] = (uint32_t)ow;
            return true;
        }
        default:
            return false;
    }
}

__device__ __forceinline__ uint32_t fnv(uint32_t h, uint32_t w) {   // word-wise FNV-1a (apply.key_hash)
    return (h ^ w) * 16777619u;
}

// symbol id of s, NONE if it was never interned (apply.py symbol_key_words / key_hash)
__device__ uint32_t sym_lookup(const Dev& d, const AArgs& a, const Sym& s) {
    if (s.name < 0) return NONE;
    for (uint32_t i = 0; i < s.np; i++)
        if (s.code[i] == NO_MATCH_CODE_U) return NONE;
    uint32_t h = 2166136261u;
    h = fnv(h, (uint32_t)s.name); h = fnv(h, s.arity); h = fnv(h, s.np);
    for (uint32_t i = 0; i < s.np; i++) h = fnv(h, s.code[i]);
    h = fnv(h, s.shape.nd);
    if (s.shape.nd != NO_SHAPE)
        for (uint32_t i = 0; i < s.shape.nd; i++) h = fnv(h, s.shape.d[i]);
    for (uint32_t slot = h & a.sym_tmask;; slot = (slot + 1) & a.sym_tmask) {
        const uint32_t c = a.sym_table[slot];
        if (c == NONE) return NONE;
        if (d.sym_name[c] != (uint32_t)s.name || d.sym_arity[c] != s.arity) continue;
        const uint32_t p0 = d.sym_poff[c], pn = d.sym_poff[c + 1] - p0;
        if (pn != s.np) continue;
        bool ok = true;
        for (uint32_t i = 0; i < pn && ok; i++) ok = (uint32_t)d.sym_par[p0 + i] == s.code[i];
        if (!ok) continue;
        const Shape cs = sym_shape(a, c);
        if (!shape_eq(cs, s.shape)) continue;
        return c;
    }
}

// make_symbol (rewrite.py:296-298 / tensor_ir.py:253-265); false = InstantiationError
__device__ bool make_symbol(const AArgs& a, const int32_t* ins, const uint32_t* rec, const Shape* cs, uint32_t nin,
                            Sym& s) {
    s.name = ins[1];
    s.arity = nin;
    s.np = 0;
    s.shape.nd = NO_SHAPE;
    if (a.lang == 0) return true;   // TermLanguage: payload is a function of the name
    const int op = ins[2];
    if (op == OP_UNK || op == OP_INPUT || op == OP_WEIGHT) return false;
    static constexpr int NPARAM[15] = {0, 1, 1, 0, 0, 0, 3, 0, 0, 0, 1, 2, 2, 0, 0};
    const int32_t np = ins[4] < 0 ? 0 : ins[4];
    if (np != NPARAM[op]) return false;
    s.np = (uint32_t)np;
    for (int p = 0; p < np; p++) {
        const int32_t tag = ins[9 + 3 * p], v = ins[10 + 3 * p];
        if (tag == 1) {   // pvar: the code bound by the match
            const uint32_t c = rec[v];
            s.code[p] = c;
            s.ival[p] = c < a.n_values ? a.val_int[c] : INT_NONE;
        } else {
            s.code[p] = tag == 0 ? (uint32_t)v : NO_MATCH_CODE_U;
            s.ival[p] = ins[11 + 3 * p];
        }
    }
    for (uint32_t i = 0; i < nin; i++)
        if (cs[i].nd == NO_SHAPE) return false;   // missing child shape
    return infer_shape(op, s, cs, nin, s.shape);
}

// node_cost (cost_model.py): f64, left-to-right products as in Python
__device__ double node_cost(const AArgs& a, int op, const Sym& s, const Shape* in) {
    if (a.cost_mode == 0) return 1.0;
    const bool leaf = op == OP_INPUT || op == OP_WEIGHT || op == OP_NOOP;
    if (a.cost_mode == 1) return leaf ? 0.0 : 1.0;
    if (leaf) return a.coeff * 0.0;
    double f;
    if (op == OP_MATMUL) {
        f = 2.0 * (double)in[0].d[0];
        f = f * (double)in[0].d[1];
        f = f * (double)in[1].d[1];
    } else if (op == OP_CONV2D) {
        f = 2.0 * (double)s.shape.d[0];
        f = f * (double)in[1].d[1];
        f = f * (double)in[1].d[2];
        f = f * (double)in[1].d[3];
        f = f * (double)s.shape.d[2];
        f = f * (double)s.shape.d[3];
        f = f * (double)in[1].d[0];
    } else {
        unsigned long long p = 1;
        for (uint32_t i = 0; i < s.shape.nd; i++) p *= s.shape.d[i];
        if (op == OP_MAXPOOL) p = p * (unsigned long long)s.ival[0] * (unsigned long long)s.ival[0];
        f = (double)p;
    }
    return a.coeff * f;
}

// hashcons key hash of k_apply's own lookup table (built at staging, probed / extended by the replay):
// a 32-bit multiply-xorshift per child is enough for linear probing at load <= 1/2
__device__ __forceinline__ uint32_t node_hash(uint32_t sym, const uint32_t* k, uint32_t ar) {
    uint32_t h = (sym + 0x7f4a7c15u) * 0x9e3779b1u;
    for (uint32_t i = 0; i < ar; i++) h = ((h ^ (h >> 15)) + k[i]) * 0x85ebca77u;
    return h ^ (h >> 13);
}

// hashcons.get(node): the entry whose stored key equals (sym, kids), NONE if absent
__device__ uint32_t hc_get(Leaf& L, uint32_t sym, const uint32_t* k, uint32_t ar) {
    for (uint32_t s = node_hash(sym, k, ar) & L.tmask;; s = (s + 1) & L.tmask) {
        const uint32_t e = L.tab[s];
        if (e == NONE) return NONE;
        if (ABAD(e >= L.n)) return NONE;
        if (L.sym[e] != sym || L.koff[e + 1] - L.koff[e] != ar) continue;
        bool ok = true;
        for (uint32_t i = 0; i < ar && ok; i++) ok = L.kids[L.koff[e] + i] == k[i];
        if (ok) return e;
    }
}

__device__ void hc_insert(Leaf& L, uint32_t e) {
    const uint32_t ar = L.koff[e + 1] - L.koff[e];
    uint32_t s = node_hash(L.sym[e], L.kids + L.koff[e], ar) & L.tmask;
    while (L.tab[s] != NONE) s = (s + 1) & L.tmask;
    L.tab[s] = e;
}

__device__ __forceinline__ void list_push(Leaf& L, uint32_t c, uint32_t e) {
    L.next[e] = NONE;
    if (L.head[c] == NONE) { L.head[c] = e; L.tail[c] = e; }
    else { L.next[L.tail[c]] = e; L.tail[c] = e; }
}

// would_create_cycle (rewrite.py:492-505): is goal reachable from refs through child edges?
// Warp-cooperative BFS (same reachable set as the reference's DFS): a queue of classes, 32 expanded
// per step, children's roots claimed once per query with an epoch-stamped atomic exchange.
//
// Potential pruning (exact): every class root carries pot with pot[p] >= pot[c] for every child edge
// p -> c between distinct classes, so a class whose pot is below the goal's cannot reach the goal
// and is neither queued nor expanded. Most instantiations reference classes inside the match, below
// the matched class, and are answered without a walk. The invariant is established by a Kahn height
// pass over the rebuilt state (classes in or above a cycle share the top value) and kept by add
// (1 + max over the children) and union (the merged class takes the larger value; ancestors below
// it are raised to it).
__device__ bool reaches(Leaf& L, const uint32_t* refs, uint32_t nrefs, uint32_t goal, bool* overflow,
                        uint32_t* qtail) {
    const uint32_t st = ++L.stamp, cap = L.cap_k + L.cap_n;
    if (ABAD(goal >= L.U)) return false;
    const bool prune = L.usepot;
    const uint32_t pg = prune ? L.pot[goal] : 0u;
    bool found = false;
    if (L.lane == 0) {
        uint32_t qt = 0;
        for (uint32_t i = 0; i < nrefs && !found; i++) {
            const uint32_t c = find(L, refs[i]);
            if (c == goal) found = true;
            else if (L.seen[c] != st && (!prune || L.pot[c] >= pg)) { L.seen[c] = st; L.stack[qt++] = c; }
        }
        *qtail = qt;
    }
    __syncwarp();
    found = __shfl_sync(0xffffffffu, found, 0);
    // the queue length is read by lane 0 and broadcast: a lane that runs ahead into the next round
    // pushes (atomicAdd on *qtail) only after the shuffle, so every lane sees the same length (a
    // per-lane read after the barrier could see another lane's next-round pushes)
    uint32_t qh = 0, qt = __shfl_sync(0xffffffffu, *(volatile uint32_t*)qtail, 0);
    while (!found && qh < qt) {
        const uint32_t idx = qh + L.lane;
        if (idx < qt) {
            const uint32_t c = L.stack[idx];
            if (ABAD(c >= L.U)) continue;
            for (uint32_t e = L.head[c]; e != NONE && !found && !ABAD(e >= L.n); e = L.next[e])
                for (uint32_t q = L.koff[e]; q < L.koff[e + 1]; q++) {
                    const uint32_t r = find(L, L.kids[q]);
                    if (r == goal) { found = true; break; }
                    if (prune && L.pot[r] < pg) continue;
                    if (atomicExch(&L.seen[r], st) != st) {
                        const uint32_t pos = atomicAdd(qtail, 1u);
                        if (pos < cap) L.stack[pos] = r;
                        else *overflow = true;
                    }
                }
        }
        found = __any_sync(0xffffffffu, found);
        __syncwarp();
        qh = qh + 32 < qt ? qh + 32 : qt;
        qt = __shfl_sync(0xffffffffu, *(volatile uint32_t*)qtail, 0);
        if (qt > cap) { qt = cap; }
    }
    __syncwarp();
    return found;
}

// add (egraph.py:175-187); returns the class or NONE on failure (*err set)
__device__ uint32_t add_node(Leaf& L, const Sym& s, int op, const uint32_t* k, const Shape* cs, uint32_t* err) {
    const uint32_t sid = sym_lookup(*L.d, *L.a, s);
    if (sid != NONE) {
        const uint32_t e = hc_get(L, sid, k, s.arity);
        if (e != NONE) return find(L, L.cid[e]);
    }
    if (sid == NONE) { *err = A_NEED_SYMBOL; return NONE; }
    if (L.n + 1 > L.cap_n || L.K + s.arity > L.cap_k || L.U + 1 > L.cap_u) { *err = A_CAPACITY; return NONE; }
    const uint32_t id = L.U++;   // every lane keeps the counters; lane 0 writes the state
    const uint32_t e = L.n++;
    const uint32_t k0 = L.K;
    L.K += s.arity;
    if (L.lane == 0) {
        L.parent[id] = id;
        L.rank[id] = 0;
        L.head[id] = NONE;
        L.seen[id] = 0;
        L.sym[e] = sid;
        for (uint32_t i = 0; i < s.arity; i++) L.kids[k0 + i] = k[i];
        L.koff[e + 1] = L.K;
        L.cid[e] = id;
        L.cost[e] = node_cost(*L.a, op, s, cs);
        hc_insert(L, e);
        list_push(L, id, e);
        if (L.usepot) {   // a new class has no parents: 1 + the highest child potential
            uint32_t pv = 0;
            L.phead[id] = NONE;
            L.ptail[id] = NONE;
            for (uint32_t i = 0; i < s.arity; i++) {
                const uint32_t c = k[i], q = k0 + i;   // children are roots (canonicalised by the caller)
                if (ABAD(c >= L.U) || ABAD(q >= L.cap_k)) continue;
                pv = max(pv, L.pot[c] + 1u);
                L.eown[q] = e;
                L.pnext[q] = NONE;
                if (L.phead[c] == NONE) L.phead[c] = q; else L.pnext[L.ptail[c]] = q;
                L.ptail[c] = q;
            }
            L.pot[id] = pv;
        }
    }
    __syncwarp();
    L.changed = true;
    return id;
}

// raise every ancestor of class w whose potential is below pot[w] to pot[w] (warp-cooperative
// upward walk over the parent-edge lists; each class is raised, and queued, at most once)
__device__ void raise_ancestors(Leaf& L, uint32_t w, uint32_t* qtail) {
    const uint32_t P = L.pot[w], cap = L.cap_k + L.cap_n;
    if (L.lane == 0) { L.stack[0] = w; *qtail = 1; }
    __syncwarp();
    uint32_t qh = 0, qt = 1;
    while (qh < qt) {
        const uint32_t idx = qh + L.lane;
        if (idx < qt) {
            const uint32_t x = L.stack[idx];
            for (uint32_t q = L.phead[x]; q != NONE && !ABAD(x >= L.U); q = L.pnext[q]) {
                if (ABAD(q >= L.K) || ABAD(L.eown[q] >= L.n) || ABAD(L.cid[L.eown[q]] >= L.U)) break;
                const uint32_t p = find(L, L.cid[L.eown[q]]);
                if (p == x || L.pot[p] >= P) continue;
                if (atomicMax(&L.pot[p], P) < P) {
                    const uint32_t pos = atomicAdd(qtail, 1u);
                    if (pos < cap) L.stack[pos] = p;
                }
            }
        }
        __syncwarp();
        qh = qh + 32 < qt ? qh + 32 : qt;
        qt = min(__shfl_sync(0xffffffffu, *(volatile uint32_t*)qtail, 0), cap);
    }
}

// add of an instruction planned in advance: symbol id known (the symbol and its shape depend only on
// class shapes, which no union inside an apply changes -- every union joins classes of one shape),
// node cost from the symbol's shape and attributes
__device__ uint32_t add_node_sid(Leaf& L, uint32_t sid, int op, uint32_t ar, const uint32_t* k, uint32_t* err,
                                 bool known_absent, const uint32_t* pcost) {
    if (!known_absent) {
        const uint32_t e0 = hc_get(L, sid, k, ar);
        if (e0 != NONE) return find(L, L.cid[e0]);
    }
    if (L.n + 1 > L.cap_n || L.K + ar > L.cap_k || L.U + 1 > L.cap_u) { *err = A_CAPACITY; return NONE; }
    double cost;
    if (pcost) {   // priced by the planner warp
        cost = __hiloint2double((int)pcost[1], (int)pcost[0]);
    } else {
        Shape cs[4];   // child class shapes: only the node cost needs them
        for (uint32_t j = 0; j < ar; j++) cs[j] = class_shape(L, k[j]);
        Sym s;
        s.name = 0; s.arity = ar; s.np = 0;
        s.shape = sym_shape(*L.a, sid);
        s.ival[0] = INT_NONE;
        if (op == OP_MAXPOOL) {
            const uint32_t code = (uint32_t)L.d->sym_par[L.d->sym_poff[sid]];
            s.ival[0] = code < L.a->n_values ? L.a->val_int[code] : INT_NONE;
        }
        cost = node_cost(*L.a, op, s, cs);
    }
    const uint32_t id = L.U++;
    const uint32_t e = L.n++;
    const uint32_t k0 = L.K;
    L.K += ar;
    if (L.lane == 0) {
        L.parent[id] = id;
        L.rank[id] = 0;
        L.head[id] = NONE;
        L.seen[id] = 0;
        L.sym[e] = sid;
        for (uint32_t i = 0; i < ar; i++) L.kids[k0 + i] = k[i];
        L.koff[e + 1] = L.K;
        L.cid[e] = id;
        L.cost[e] = cost;
        hc_insert(L, e);
        list_push(L, id, e);
        if (L.usepot) {
            uint32_t pv = 0;
            L.phead[id] = NONE;
            L.ptail[id] = NONE;
            for (uint32_t i = 0; i < ar; i++) {
                const uint32_t c = k[i], q = k0 + i;
                pv = max(pv, L.pot[c] + 1u);
                L.eown[q] = e;
                L.pnext[q] = NONE;
                if (L.phead[c] == NONE) L.phead[c] = q; else L.pnext[L.ptail[c]] = q;
                L.ptail[c] = q;
            }
            L.pot[id] = pv;
        }
    }
    __syncwarp();
    L.changed = true;
    return id;
}

__device__ bool union_classes(Leaf& L, uint32_t a, uint32_t b, uint32_t* qtail) {
    const uint32_t ra = find(L, a), rb = find(L, b);
    __syncwarp();
    if (ra == rb) return false;
    uint32_t win = 0;
    bool raise = false;
    if (L.lane == 0) {
        win = uf_union(L.parent, L.rank, ra, rb);
        const uint32_t lose = win == ra ? rb : ra;
        if (L.head[lose] != NONE) {
            if (L.head[win] == NONE) { L.head[win] = L.head[lose]; L.tail[win] = L.tail[lose]; }
            else { L.next[L.tail[win]] = L.head[lose]; L.tail[win] = L.tail[lose]; }
            L.head[lose] = NONE;
        }
        if (L.usepot) {
            if (L.phead[lose] != NONE) {
                if (L.phead[win] == NONE) { L.phead[win] = L.phead[lose]; L.ptail[win] = L.ptail[lose]; }
                else { L.pnext[L.ptail[win]] = L.phead[lose]; L.ptail[win] = L.ptail[lose]; }
                L.phead[lose] = NONE;
            }
            const uint32_t P = max(L.pot[ra], L.pot[rb]);
            raise = L.pot[ra] != L.pot[rb];   // the lower side's parents may now sit below P
            L.pot[win] = P;
        }
    }
    __syncwarp();
    win = __shfl_sync(0xffffffffu, win, 0);
    raise = __shfl_sync(0xffffffffu, raise, 0);
    if (raise) raise_ancestors(L, win, qtail);
    L.changed = true;
    return true;
}

// One match of the ordered replay (rewrite.py:538-566): per target _target_refs, the cycle test, the
// shape tests, the instantiation and the union. ``plan``: the match's plan (PS words per target,
// flags at FL, node costs at PMAX when COST) or nullptr (full path).
template <uint32_t PS, uint32_t FL, bool COST>
__device__ __forceinline__ void replay_match(Leaf& L, const Dev& d, const AArgs& a, uint32_t rule, const int32_t* rp,
                                             int32_t NT, const uint32_t* rec, const uint32_t* plan, uint32_t& st,
                                             uint32_t& cyc, uint32_t& shp, uint32_t& unions, uint32_t* sh_qtail) {
    for (int32_t t = 0; t < NT && st == A_OK; t++) {
        const int32_t* tp = rp + rp[7 + t];
        const uint32_t ni = (uint32_t)tp[0];
        if (ni > MAXI) { st = A_PROGRAM; break; }
        const uint32_t* pl = plan ? plan + t * PS : nullptr;
        const uint32_t pflags = plan ? pl[FL] : PLAN_SLOW;
        const bool fast = !(pflags & PLAN_SLOW);
        const uint32_t matched = find(L, rec[t]);
        // _target_refs (rewrite.py:463-489): refs set, existing instance class
        uint32_t cid[MAXI];          // class of instruction i (NONE: not existing)
        uint32_t vcls[MAXI];         // root of a var instruction's binding
        uint8_t rmiss[MAXI];         // _target_refs probed instruction i (all children existed) and missed
        uint32_t rbeg[MAXI], rend[MAXI];
        uint32_t refs[64];
        uint32_t nref = 0;
        bool inst_err = false;
        for (uint32_t i = 0; i < ni && !inst_err; i++) {
            const int32_t* ins = tp + 1 + INSTR * i;
            if (ins[0] == 0) {
                const uint32_t c = find(L, rec[ins[1]]);
                cid[i] = c;
                vcls[i] = c;
                rbeg[i] = nref;
                if (nref < 64) refs[nref++] = c;
                rend[i] = nref;
                continue;
            }
            const uint32_t ar = (uint32_t)ins[3];
            uint32_t b0 = nref;
            bool all = true;
            uint32_t kc[4];
            for (uint32_t j = 0; j < ar; j++) {
                const uint32_t ci = (uint32_t)ins[5 + j];
                for (uint32_t r = rbeg[ci]; r < rend[ci]; r++)
                    if (nref < 64) refs[nref++] = refs[r];
                if (cid[ci] == NONE) all = false;
                else kc[j] = cid[ci];
            }
            cid[i] = NONE;
            rmiss[i] = 0;
            if (all) {
                uint32_t sid;
                if (fast) {
                    sid = pl[i];
                    if (sid == PLAN_FAIL) { inst_err = true; break; }
                } else {
                    Shape cs[4];
                    for (uint32_t j = 0; j < ar; j++) cs[j] = class_shape(L, kc[j]);
                    Sym s;
                    if (!make_symbol(a, ins, rec, cs, ar, s)) { inst_err = true; break; }
                    sid = sym_lookup(d, a, s);
                }
                const uint32_t e = sid == NONE ? NONE : hc_get(L, sid, kc, ar);
                if (e != NONE) {
                    const uint32_t c = find(L, L.cid[e]);
                    cid[i] = c;
                    nref = b0;
                    refs[nref++] = c;
                } else {
                    rmiss[i] = 1;
                }
            }
            rbeg[i] = b0;
            rend[i] = nref;
        }
        if (nref >= 64) { st = A_PROGRAM; break; }
        if (inst_err) { shp++; continue; }
        const uint32_t top = ni - 1;
        if (cid[top] != NONE && cid[top] == matched) continue;
        bool ovf = false;
        if (reaches(L, refs + rbeg[top], rend[top] - rbeg[top], matched, &ovf, sh_qtail)) { cyc++; continue; }
        ovf = __any_sync(0xffffffffu, ovf);
        if (ovf) { st = A_CAPACITY; break; }
        // _instance_shape (rewrite.py:508-514) then the matched-class shape test
        if (fast) {
            if (pflags & (PLAN_SHAPE_ERR | PLAN_SHAPE_MISMATCH)) { shp++; continue; }
            uint32_t inst[MAXI];
            uint32_t err = A_OK;
            // every inst[] is a root (a var's find from _target_refs -- adds do not move roots --,
            // a hashcons hit's find, or a new id) and no union happens before the top one
            // an instruction _target_refs found reuses that class (adds never remove a node and
            // move no root); one it probed and missed is still missing unless this target
            // already added a node (two instructions of one target may build the same node)
            bool added = false;
            for (uint32_t i = 0; i < ni && err == A_OK; i++) {
                const int32_t* ins = tp + 1 + INSTR * i;
                if (ins[0] == 0) { inst[i] = vcls[i]; continue; }
                if (cid[i] != NONE) { inst[i] = cid[i]; continue; }
                const uint32_t ar = (uint32_t)ins[3];
                uint32_t kc[4];
                for (uint32_t j = 0; j < ar; j++) kc[j] = inst[ins[5 + j]];
                const uint32_t n0 = L.n;
                inst[i] = add_node_sid(L, pl[i], ins[2], ar, kc, &err, rmiss[i] && !added, COST ? pl + PMAX + 2 * i : nullptr);
                added = added || L.n != n0;
            }
            if (err != A_OK) { st = err; break; }
            if (union_classes(L, inst[top], matched, sh_qtail)) unions++;
            continue;
        }
        Shape sh[MAXI];
        for (uint32_t i = 0; i < ni && !inst_err; i++) {
            const int32_t* ins = tp + 1 + INSTR * i;
            if (ins[0] == 0) { sh[i] = class_shape(L, rec[ins[1]]); continue; }
            const uint32_t ar = (uint32_t)ins[3];
            Shape cs[4];
            for (uint32_t j = 0; j < ar; j++) cs[j] = sh[ins[5 + j]];
            Sym s;
            if (!make_symbol(a, ins, rec, cs, ar, s)) { inst_err = true; break; }
            sh[i] = s.shape;
        }
        if (inst_err) { shp++; continue; }
        const Shape msh = class_shape(L, matched);
        if (sh[top].nd != NO_SHAPE && msh.nd != NO_SHAPE && !shape_eq(sh[top], msh)) { shp++; continue; }
        // _instantiate (rewrite.py:517-523) bottom-up, then union with the matched class
        uint32_t inst[MAXI];
        uint32_t err = A_OK;
        for (uint32_t i = 0; i < ni && err == A_OK; i++) {
            const int32_t* ins = tp + 1 + INSTR * i;
            if (ins[0] == 0) { inst[i] = find(L, rec[ins[1]]); continue; }
            const uint32_t ar = (uint32_t)ins[3];
            uint32_t kc[4];
            Shape cs[4];
            for (uint32_t j = 0; j < ar; j++) { kc[j] = inst[ins[5 + j]]; cs[j] = class_shape(L, kc[j]); }
            Sym s;
            if (!make_symbol(a, ins, rec, cs, ar, s)) { err = A_PROGRAM; break; }   // checked above
            for (uint32_t j = 0; j < ar; j++) kc[j] = find(L, kc[j]);
            inst[i] = add_node(L, s, ins[2], kc, cs, &err);
            if (err == A_NEED_SYMBOL && L.lane == 0) {   // describe the missing symbol for host interning
                uint32_t* ms = a.missing + 16 * (uint64_t)L.l;
                ms[0] = (uint32_t)s.name; ms[1] = s.arity; ms[2] = s.np;
                for (int p = 0; p < 3; p++) { ms[3 + p] = s.code[p]; ms[6 + p] = (uint32_t)s.ival[p]; }
                ms[9] = s.shape.nd;
                for (int p = 0; p < 4; p++) ms[10 + p] = s.shape.d[p];
                ms[14] = (uint32_t)rule; ms[15] = ((uint32_t)t << 8) | i;   // target, instruction
            }
        }
        if (err != A_OK) { st = err; break; }
        if (union_classes(L, inst[top], matched, sh_qtail)) unions++;
    }
}

__device__ __forceinline__ Shape shape_of(const AArgs& a, uint32_t sid) {
    Shape sh;
    sh.nd = NO_SHAPE;
    return sid == NONE ? sh : sym_shape(a, sid);
}

// Plan of one match for the two-warp replay (a lane of the planner warp), per target: for every instruction the symbol
// make_symbol builds and its id (sym_lookup; PLAN_FAIL: make_symbol fails, or not interned with flag
// PLAN_SLOW) and the node cost of an add; flags PLAN_SHAPE_ERR (_instance_shape fails) and
// PLAN_SHAPE_MISMATCH (the matched-class shape test). All of it depends only on class shapes, which
// no union of an apply changes (the shape test admits only same-shape unions; rebuilt classes are
// shape-homogeneous), so the planner reads only what the replay never writes: the symbol tables and
// symc, the symbol of every pre-apply class.
__device__ __noinline__ void plan_match(const Dev& d, const AArgs& a, const int32_t* rp, int32_t NT, const uint32_t* prec,
                           const uint32_t* symc, uint32_t (*pl)[PW]) {
    for (int32_t t = 0; t < NT; t++) {
        const int32_t* tp = rp + rp[7 + t];
        const uint32_t ni = (uint32_t)tp[0];
        uint32_t* p = pl[t];
        uint32_t flags = 0;
        if (ni > PMAX) { p[3 * PMAX] = PLAN_SLOW; continue; }
        Shape shs[PMAX];
        bool bad = false;
        for (uint32_t i = 0; i < ni; i++) {
            const int32_t* ins = tp + 1 + INSTR * i;
            if (ins[0] == 0) { shs[i] = shape_of(a, symc[prec[ins[1]]]); continue; }
            p[i] = PLAN_FAIL;
            if (bad) continue;   // _instance_shape stops at its first failure
            const uint32_t ar = (uint32_t)ins[3];
            Shape cs[4];
            for (uint32_t j = 0; j < ar; j++) cs[j] = shs[ins[5 + j]];
            Sym ps;
            if (!make_symbol(a, ins, prec, cs, ar, ps)) { bad = true; flags |= PLAN_SHAPE_ERR; continue; }
            shs[i] = ps.shape;
            const uint32_t sid = sym_lookup(d, a, ps);
            if (sid == NONE) flags |= PLAN_SLOW;
            p[i] = sid == NONE ? PLAN_FAIL : sid;
            const double c = node_cost(a, ins[2], ps, cs);
            p[PMAX + 2 * i] = (uint32_t)__double2loint(c);
            p[PMAX + 2 * i + 1] = (uint32_t)__double2hiint(c);
        }
        if (!bad) {
            const Shape msh = shape_of(a, symc[prec[t]]);
            if (shs[ni - 1].nd != NO_SHAPE && msh.nd != NO_SHAPE && !shape_eq(shs[ni - 1], msh))
                flags |= PLAN_SHAPE_MISMATCH;
        }
        p[3 * PMAX] = flags;
    }
}

}  // namespace

template <int NW>
__global__ void __launch_bounds__(32 * NW, NW == 1 ? 16 : 1) k_apply(Dev d, AArgs a) {
    // warp 0 stages the rebuilt state into the working arrays, builds the class lists and the lookup
    // table, then replays the matches in order. NW = 1: the lanes plan each chunk of matches before
    // warp 0 replays it; NW = 2 (leaves with many matches): warp 1 plans the next chunk while warp 0
    // replays the current one. A launch handles the leaves whose match count is in [sel_lo, sel_hi).
    const uint32_t l = blockIdx.x, lane = threadIdx.x & 31u, warp = NW == 1 ? 0u : threadIdx.x >> 5;
    if (l >= d.L) return;
    const uint32_t rule = a.leaf_rule[l];
    {
        uint32_t cnt0 = 0;
        if (rule != NONE) {
            const int32_t* rp0 = a.prog + a.rule_off[rule];
            const uint64_t mi = (uint64_t)rp0[1] * d.L + l;
            cnt0 = rp0[0] ? a.j_count[mi] : a.m_count[mi];
        }
        if (cnt0 < a.sel_lo || cnt0 >= a.sel_hi) return;
    }
    uint32_t* rep = a.report + 8 * (uint64_t)l;
    const uint64_t b = d.nb[l], k0 = d.kb[l], u0 = d.ub[l], t0 = d.tb[l];
    Leaf L;
    L.d = &d; L.a = &a; L.l = l;
    L.cap_n = (uint32_t)(d.nb[l + 1] - b);
    L.cap_k = (uint32_t)(d.kb[l + 1] - k0);
    L.cap_u = (uint32_t)(d.ub[l + 1] - u0);
    L.n = d.o_n[l];
    L.U = d.u_reb[l];   // ids of the rebuilt state (an apply never changes the rebuild's outputs)
    L.sym = a.w_sym + b; L.koff = a.w_koff + b + l; L.kids = a.w_kids + k0; L.cid = a.w_cid + b;
    L.cost = a.w_cost + b;
    L.parent = a.w_parent + u0; L.rank = a.w_rank + u0;
    L.head = a.s_head + u0; L.tail = a.s_tail + u0; L.next = a.s_next + b; L.seen = a.s_seen + u0;
    L.stack = a.s_stack + b + k0;
    L.tab = d.s_tc + t0;
    L.pot = a.s_pot + u0; L.phead = a.s_phead + u0; L.ptail = a.s_ptail + u0;
    L.pnext = a.s_pnext + k0; L.eown = a.s_eown + k0;
    L.usepot = !a.no_pot;
    L.tmask = (uint32_t)(d.tb[l + 1] - t0) - 1;
    L.stamp = 0;
    L.changed = false;
    __shared__ uint32_t sh_qtail;
    __shared__ uint32_t sh_plan[NW][PLAN_CH][PLAN_T][NW == 1 ? MAXI + 1 : PW];
    __shared__ uint32_t sh_kahn, sh_stop[2];
    L.lane = lane;
    uint32_t* symc = a.s_pend + u0;   // NW = 2: symbol of every pre-apply class (the planner's shapes)
    if (warp == 0) {
    // the rebuilt state becomes the working state: hashcons entries (canonical keys, classes
    // are roots), union-find, class membership lists, lookup table
    const uint32_t* okoff = d.o_koff + b + l;
    if (lane == 0) L.koff[0] = 0;
    for (uint32_t e = lane; e < L.n; e += 32) {
        L.sym[e] = d.o_sym[b + e];
        L.cid[e] = d.o_cid[b + e];
        L.cost[e] = d.o_cost[b + e];
        L.koff[e + 1] = okoff[e + 1];
    }
    L.K = okoff[L.n];
    for (uint32_t q = lane; q < L.K; q += 32) L.kids[q] = d.o_kids[k0 + q];
    for (uint32_t x = lane; x < L.U; x += 32) {
        L.parent[x] = d.uf_parent[u0 + x];
        L.rank[x] = d.uf_rank[u0 + x];
        L.head[x] = NONE;
        L.seen[x] = 0;
    }
    {   // tables are >= 4 slots and 16-B aligned (esat_batch_create): clear 4 slots per store
        uint4* t4 = reinterpret_cast<uint4*>(L.tab);
        const uint4 none4 = make_uint4(NONE, NONE, NONE, NONE);
        for (uint32_t s = lane; s < (L.tmask + 1) / 4; s += 32) t4[s] = none4;
    }
    __syncwarp();
    for (uint32_t e = lane; e < L.n; e += 32) {
        const uint32_t c = L.cid[e];   // rebuilt classes are union-find roots
        const uint32_t old = atomicExch(&L.head[c], e);
        L.next[e] = old;
        if (old == NONE) L.tail[c] = e;
        const uint32_t ar = L.koff[e + 1] - L.koff[e];
        for (uint32_t s = node_hash(L.sym[e], L.kids + L.koff[e], ar) & L.tmask;; s = (s + 1) & L.tmask)
            if (atomicCAS(&L.tab[s], NONE, e) == NONE) break;
    }
    __syncwarp();
    // from here every lane of warp 0 runs the same sequential replay (identical values in
    // registers); state writes are issued by lane 0 and fenced with __syncwarp, the cycle test uses
    // all lanes
    if (rule != NONE && L.usepot) {
        // cycle-test potentials of the rebuilt state: parent-edge lists (child slots, self-loops left
        // out), then Kahn rounds from the classes without children: pot = height; classes in or
        // above a cycle are never released and share the top value (pot[p] >= pot[c] either way)
        uint32_t* pend = a.s_pend + u0;
        if (lane == 0 && (ABAD(L.U > L.cap_u) || ABAD(L.n > L.cap_n) || ABAD(L.K > L.cap_k))) {}
        for (uint32_t x = lane; x < L.U; x += 32) { L.pot[x] = 0; L.phead[x] = NONE; L.ptail[x] = NONE; pend[x] = 0; }
        __syncwarp();
        for (uint32_t e = lane; e < L.n; e += 32) {
            const uint32_t c = L.cid[e];
            if (ABAD(c >= L.U) || ABAD(L.koff[e + 1] > L.cap_k)) continue;
            for (uint32_t q = L.koff[e]; q < L.koff[e + 1]; q++) {
                L.eown[q] = e;
                const uint32_t k = L.kids[q];   // rebuilt keys are canonical: children are roots
                if (ABAD(k >= L.U)) continue;
                if (k == c) { L.pnext[q] = NONE; continue; }
                atomicAdd(&pend[c], 1u);
                const uint32_t old = atomicExch(&L.phead[k], q);
                L.pnext[q] = old;
                if (old == NONE) L.ptail[k] = q;
            }
        }
        if (lane == 0) sh_kahn = 0;
        __syncwarp();
        for (uint32_t c = lane; c < L.U; c += 32)
            if (L.head[c] != NONE && pend[c] == 0) {
                const uint32_t pos = atomicAdd(&sh_kahn, 1u);
                if (!ABAD(pos >= L.n)) L.stack[pos] = c;
            }
        __syncwarp();
        uint32_t f0 = 0, f1 = __shfl_sync(0xffffffffu, *(volatile uint32_t*)&sh_kahn, 0), round = 0;
        while (f0 < f1) {
            for (uint32_t i = f0 + lane; i < f1; i += 32) {
                const uint32_t c = L.stack[i];
                if (ABAD(c >= L.U)) continue;
                for (uint32_t q = L.phead[c]; q != NONE; q = L.pnext[q]) {
                    if (ABAD(q >= L.K) || ABAD(L.eown[q] >= L.n)) break;
                    const uint32_t pc = L.cid[L.eown[q]];
                    if (ABAD(pc >= L.U)) continue;
                    if (atomicSub(&pend[pc], 1u) == 1u) {
                        L.pot[pc] = round + 1;
                        const uint32_t pos = atomicAdd(&sh_kahn, 1u);
                        if (!ABAD(pos >= L.n)) L.stack[pos] = pc;
                    }
                }
            }
            __syncwarp();
            f0 = f1;
            f1 = __shfl_sync(0xffffffffu, *(volatile uint32_t*)&sh_kahn, 0);
            round++;
        }
        for (uint32_t c = lane; c < L.U; c += 32)
            if (L.head[c] != NONE && pend[c] != 0) L.pot[c] = round + 1;
        __syncwarp();
    }
    if (NW == 2 && rule != NONE)   // (Kahn is done with pend: it becomes symc)
        for (uint32_t x = lane; x < L.U; x += 32) {
            const uint32_t e = L.head[find(L, x)];
            symc[x] = e == NONE ? NONE : L.sym[e];
        }
    }   // warp 0
    __syncthreads();
    uint32_t st = A_OK, found = 0, cyc = 0, shp = 0;
    const uint32_t n_before = L.n;
    uint32_t unions = 0;
    if (rule != NONE && a.node_limit && L.n >= a.node_limit) st = A_NODE_LIMIT;   // rewrite.py:532-537
    if (rule != NONE && st == A_OK) {
        const int32_t* rp = a.prog + a.rule_off[rule];
        const int32_t from_join = rp[0], li = rp[1], W = rp[2], NT = rp[6];
        const uint64_t mi = (uint64_t)li * d.L + l;
        const uint32_t* words = from_join ? a.j_words + a.j_off[mi] : a.m_words + a.m_off[mi];
        const uint32_t cnt = from_join ? a.j_count[mi] : a.m_count[mi];
        found = cnt;
        // Matches are replayed in order in chunks of PLAN_CH. Before a chunk, each lane plans one
        // match: for every target instruction the symbol make_symbol / infer_shape would build and
        // its id (sym_lookup), plus the _instance_shape outcome and the matched-class shape test.
        // These depend only on class shapes, which no union of an apply changes (the shape test
        // admits only same-shape unions; rebuilt classes are shape-homogeneous), so the ordered
        // replay reads them instead of recomputing -- it keeps every state-dependent step (finds,
        // hashcons probes, the cycle test, adds, unions) and the reference's order. A target whose
        // plan hit a symbol the table lacks replays the full path (host interning, below).
        const bool planned = NT <= PLAN_T;
        if constexpr (NW == 1) {
        for (uint32_t m0 = 0; m0 < cnt && st == A_OK; m0 += PLAN_CH) {
          const uint32_t m1 = min(cnt, m0 + PLAN_CH);
          if (planned) {
            __syncwarp();
            if (m0 + lane < m1) {
                const uint32_t* prec = words + (uint64_t)(m0 + lane) * W;
                for (int32_t t = 0; t < NT; t++) {
                    const int32_t* tp = rp + rp[7 + t];
                    const uint32_t ni = (uint32_t)tp[0];
                    uint32_t* pl = sh_plan[0][lane][t];
                    uint32_t flags = 0;
                    if (ni > MAXI) { pl[MAXI] = PLAN_SLOW; continue; }
                    Shape shs[MAXI];
                    bool bad = false;
                    for (uint32_t i = 0; i < ni; i++) {
                        const int32_t* ins = tp + 1 + INSTR * i;
                        if (ins[0] == 0) { shs[i] = class_shape(L, prec[ins[1]]); continue; }
                        pl[i] = PLAN_FAIL;
                        if (bad) continue;   // _instance_shape stops at its first failure
                        const uint32_t ar = (uint32_t)ins[3];
                        Shape cs[4];
                        for (uint32_t j = 0; j < ar; j++) cs[j] = shs[ins[5 + j]];
                        Sym ps;
                        if (!make_symbol(a, ins, prec, cs, ar, ps)) { bad = true; flags |= PLAN_SHAPE_ERR; continue; }
                        shs[i] = ps.shape;
                        const uint32_t sid = sym_lookup(d, a, ps);
                        if (sid == NONE) flags |= PLAN_SLOW;
                        pl[i] = sid == NONE ? PLAN_FAIL : sid;
                    }
                    if (!bad) {
                        const Shape msh = class_shape(L, find(L, prec[t]));
                        if (shs[ni - 1].nd != NO_SHAPE && msh.nd != NO_SHAPE && !shape_eq(shs[ni - 1], msh))
                            flags |= PLAN_SHAPE_MISMATCH;
                    }
                    pl[MAXI] = flags;
                }
            }
            __syncwarp();
          }
          for (uint32_t m = m0; m < m1 && st == A_OK; m++) {
            replay_match<MAXI + 1, MAXI, false>(L, d, a, rule, rp, NT, words + (uint64_t)m * W,
                                                planned ? &sh_plan[0][m - m0][0][0] : nullptr, st, cyc, shp, unions,
                                                &sh_qtail);
          }
        }
        } else {
        // NW = 2: warp 1 plans chunk c+1 (plan_match, with node costs) while warp 0 replays chunk c
        const uint32_t nch = (cnt + PLAN_CH - 1) / PLAN_CH;
        if (warp == 1 && planned && lane < min(cnt, PLAN_CH))
            plan_match(d, a, rp, NT, words + (uint64_t)lane * W, symc, sh_plan[0][lane]);
        __syncthreads();
        for (uint32_t ch = 0; ch < nch; ch++) {
            const uint32_t m0 = ch * PLAN_CH, m1 = min(cnt, m0 + PLAN_CH), buf = ch & 1u;
            if (warp == 1) {
                if (planned && m1 + lane < min(cnt, m1 + PLAN_CH))
                    plan_match(d, a, rp, NT, words + (uint64_t)(m1 + lane) * W, symc, sh_plan[buf ^ 1u][lane]);
            } else {
                for (uint32_t m = m0; m < m1 && st == A_OK; m++)
                    replay_match<PW, 3 * PMAX, true>(L, d, a, rule, rp, NT, words + (uint64_t)m * W,
                                                     planned ? &sh_plan[buf][m - m0][0][0] : nullptr, st, cyc, shp,
                                                     unions, &sh_qtail);
                if (lane == 0) sh_stop[buf] = st;
            }
            __syncthreads();
            if (sh_stop[buf] != A_OK) break;
        }
        }
    }
    if (warp != 0 || lane != 0) return;
    d.n_cnt[l] = L.n;
    d.u_cnt[l] = L.U;
    a.status[l] = st;
    rep[0] = found; rep[1] = L.changed ? 1u : 0u; rep[2] = cyc; rep[3] = shp;
    rep[4] = unions; rep[5] = L.n - n_before; rep[6] = 0; rep[7] = 0;
}

template __global__ void k_apply<1>(Dev, AArgs);
template __global__ void k_apply<2>(Dev, AArgs);

}  // namespace esat

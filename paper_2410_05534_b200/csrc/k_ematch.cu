// K1-K3: batched e-matching (rewrite.py:353-433) and multi-pattern joins.
//
// k_ematch: one CTA per (leaf, pattern). Root classes are split into contiguous per-thread
// chunks so that concatenating thread outputs keeps the reference's order (matches sort
// by root first, rewrite.py:396-397). Each thread runs the backtracking matcher of
// _match_in_class (rewrite.py:371-393) iteratively over the pattern's pre-order: an App
// node scans the e-nodes of its class in node_sort_key order with the name/arity/attribute
// test of _match_param_spec (353-368); a Var binds on first sight and checks equality after.
// Pass 1 counts, a block scan places every thread's raw records in a staging area, pass 2
// writes them, sorts + dedups each root class's slice (rewrite.py:420-433), and a second scan
// compacts the unique records into the output pool. EXISTS mode (is_rule_applicable,
// rewrite.py:579-589) stops at the first match.
//
// k_join: one CTA per (leaf, multi-pattern rule). joint_match threads bindings from source to
// source (rewrite.py:410-419); on device the sources are matched independently (k_ematch) and
// joined on equal shared var/pvar bindings -- the same set. Threads own
// whole groups of source-0 records with equal root; for each combination of root groups of
// the other sources the consistent products form one block with a fixed roots prefix, which is
// sorted locally, so blocks come out in (roots, vars, pvars) = _subst_key order.
#include <cstdio>

#include "k_ematch_args.cuh"

namespace esat {

namespace {

struct Matcher {
    const int32_t* prog;        // shared-memory copy
    int P, V, Q;
    // leaf view
    const uint32_t *cls_id, *cls_off, *nd_sym, *nd_koff, *nd_kpos;
    const uint32_t *s_name, *s_arity, *s_poff;
    const int32_t* s_par;
};

__device__ __forceinline__ const int32_t* rec(const Matcher& m, int i) { return m.prog + 3 + 6 * i; }

// Enumerate all matches rooted at class position r; emit(rec_words) per raw match.
// Returns the number of raw matches (stops after the first when `first_only`).
template <typename Emit>
__device__ uint32_t match_class(const Matcher& m, uint32_t r, bool first_only, Emit emit) {
    uint32_t cls[MAX_PN], choice[MAX_PN], pmask[MAX_PN];
    uint32_t vars[MAX_V];
    int32_t pv[MAX_V];
    uint32_t pset = 0, vbound_here = 0;
    for (int v = 0; v < m.V; v++) vars[v] = NONE;
    uint32_t n = 0;
    cls[0] = r;
    int i = 0;
    bool entering = true;
    while (i >= 0) {
        if (i == m.P) {
            n++;
            emit(m.cls_id[r], vars, pv);
            if (first_only) return n;
            i--;
            entering = false;
            continue;
        }
        const int32_t* pr = rec(m, i);
        if (pr[0] == 0) {  // Var
            const int v = pr[1];
            if (entering) {
                const uint32_t cid = m.cls_id[cls[i]];
                if (vars[v] == NONE) { vars[v] = cid; vbound_here |= 1u << i; i++; continue; }
                if (vars[v] == cid) { vbound_here &= ~(1u << i); i++; continue; }
                i--;
                entering = false;
                continue;
            }
            if (vbound_here >> i & 1u) { vars[v] = NONE; vbound_here &= ~(1u << i); }
            i--;
            continue;
        }
        // App
        const int32_t name = pr[1], arity = pr[2], nslots = pr[3];
        const int32_t* slots = m.prog + pr[4];
        const int32_t* kids = m.prog + pr[5];
        const uint32_t lo = m.cls_off[cls[i]], hi = m.cls_off[cls[i] + 1];
        uint32_t nd;
        if (entering) { nd = lo; pmask[i] = 0; }
        else {
            pset &= ~pmask[i];   // undo attribute bindings made at this node
            pmask[i] = 0;
            nd = choice[i] + 1;
        }
        bool found = false;
        for (; nd < hi; nd++) {
            const uint32_t s = m.nd_sym[nd];
            if ((int32_t)m.s_name[s] != name || (int32_t)m.s_arity[s] != arity) continue;
            if (nslots >= 0) {
                const uint32_t p0 = m.s_poff[s];
                if ((int32_t)(m.s_poff[s + 1] - p0) != nslots) continue;
                uint32_t newly = 0;
                bool ok = true;
                for (int j = 0; j < nslots && ok; j++) {
                    const int32_t sl = slots[j], av = m.s_par[p0 + j];
                    if (sl >= 0) ok = (sl == av);
                    else {
                        const int q = -sl - 1;
                        if (!((pset | newly) >> q & 1u)) { pv[q] = av; newly |= 1u << q; }
                        else ok = (pv[q] == av);
                    }
                }
                if (!ok) continue;
                pset |= newly;
                pmask[i] = newly;
            }
            found = true;
            break;
        }
        if (!found) { i--; entering = false; continue; }
        choice[i] = nd;
        const uint32_t k0 = m.nd_koff[nd];
        for (int j = 0; j < arity; j++) cls[kids[j]] = m.nd_kpos[k0 + j];
        i++;
        entering = true;
    }
    return n;
}


// ---- specialised matcher for patterns of depth <= 2 (all TASO-style sources) -----------------
// Root App whose children are Vars or Apps over Vars only; <= 4 vars, <= 4 pvars, arity <= 3.
// No backtracking stack: an odometer over the e-nodes of the App-children classes, bindings
// held in registers (constant-indexed), re-derived per combination. Same match set as
// match_class (order differs; the per-root sort makes the output identical).
struct Flat2 {
    int32_t ok, name, arity, nslots, V, Q;
    int32_t slots[4];
    int32_t ck[3], cv[3], cname[3], car[3], cns[3];
    int32_t cslots[3][4], gv[3][3];
};

__device__ void decode_flat2(const int32_t* pg, Flat2& f) {
    f.ok = 0;
    const int32_t P = pg[0], V = pg[1], Q = pg[2];
    const int32_t* r0 = pg + 3;
    if (r0[0] != 1 || V > 4 || Q > 4 || r0[2] > 3 || r0[3] > 4) return;
    f.name = r0[1]; f.arity = r0[2]; f.nslots = r0[3]; f.V = V; f.Q = Q;
    for (int i = 0; i < 4; i++) f.slots[i] = i < f.nslots ? pg[r0[4] + i] : 0;
    const int32_t* kids = pg + r0[5];
    for (int j = 0; j < 3; j++) { f.ck[j] = 0; f.cv[j] = 0; f.cname[j] = 0; f.car[j] = 0; f.cns[j] = -1; }
    for (int j = 0; j < f.arity; j++) {
        const int32_t* rc = pg + 3 + 6 * kids[j];
        if (rc[0] == 0) { f.ck[j] = 0; f.cv[j] = rc[1]; continue; }
        if (rc[2] > 3 || rc[3] > 4) return;
        f.ck[j] = 1; f.cname[j] = rc[1]; f.car[j] = rc[2]; f.cns[j] = rc[3];
        for (int i = 0; i < 4; i++) f.cslots[j][i] = i < rc[3] ? pg[rc[4] + i] : 0;
        const int32_t* gk = pg + rc[5];
        for (int g = 0; g < rc[2]; g++) {
            const int32_t* rg = pg + 3 + 6 * gk[g];
            if (rg[0] != 0) return;   // depth > 2
            f.gv[j][g] = rg[1];
        }
    }
    (void)P;
    f.ok = 1;
}

__device__ __forceinline__ bool bind4(uint32_t (&a)[4], uint32_t& set, int idx, uint32_t val) {
    bool ok = true;
#pragma unroll
    for (int i = 0; i < 4; i++)
        if (i == idx) {
            if ((set >> i) & 1u) ok = a[i] == val;
            else { a[i] = val; set |= 1u << i; }
        }
    return ok;
}

__device__ __forceinline__ bool slots_ok(const Matcher& m, uint32_t sym, int32_t nslots, const int32_t* slots,
                                         uint32_t (&pv)[4], uint32_t& pset) {
    if (nslots < 0) return true;
    const uint32_t p0 = m.s_poff[sym];
    if ((int32_t)(m.s_poff[sym + 1] - p0) != nslots) return false;
    for (int j = 0; j < nslots; j++) {
        const int32_t sl = slots[j], av = m.s_par[p0 + j];
        if (sl >= 0) { if (sl != av) return false; }
        else if (!bind4(pv, pset, -sl - 1, (uint32_t)av)) return false;
    }
    return true;
}

template <typename Emit>
__device__ uint32_t match_class_flat2(const Matcher& m, const Flat2& f, uint32_t r, Emit emit) {
    uint32_t n = 0;
    const uint32_t rid = m.cls_id[r];
    for (uint32_t nd = m.cls_off[r]; nd < m.cls_off[r + 1]; nd++) {
        const uint32_t s = m.nd_sym[nd];
        if ((int32_t)m.s_name[s] != f.name || (int32_t)m.s_arity[s] != f.arity) continue;
        uint32_t pv0[4] = {0, 0, 0, 0}, ps0 = 0;
        if (!slots_ok(m, s, f.nslots, f.slots, pv0, ps0)) continue;
        uint32_t kc[3] = {0, 0, 0};
        const uint32_t k0 = m.nd_koff[nd];
#pragma unroll
        for (int j = 0; j < 3; j++)
            if (j < f.arity) kc[j] = m.nd_kpos[k0 + j];
        // child j: a Var binds its class; an App iterates the matching e-nodes of its class.
        // Nested loops with early rejection at each level; bindings copied per level (registers).
        auto child = [&](int j, uint32_t (&vars)[4], uint32_t& vset, uint32_t (&pv)[4], uint32_t& pset,
                         auto&& next) {
            if (j >= f.arity) { next(vars, vset, pv, pset); return; }
            if (!f.ck[j]) {
                uint32_t v2[4] = {vars[0], vars[1], vars[2], vars[3]}, vs2 = vset;
                if (bind4(v2, vs2, f.cv[j], m.cls_id[kc[j]])) next(v2, vs2, pv, pset);
                return;
            }
            for (uint32_t cn = m.cls_off[kc[j]]; cn < m.cls_off[kc[j] + 1]; cn++) {
                const uint32_t cs = m.nd_sym[cn];
                if ((int32_t)m.s_name[cs] != f.cname[j] || (int32_t)m.s_arity[cs] != f.car[j]) continue;
                uint32_t p2[4] = {pv[0], pv[1], pv[2], pv[3]}, ps2 = pset;
                if (!slots_ok(m, cs, f.cns[j], f.cslots[j], p2, ps2)) continue;
                uint32_t v2[4] = {vars[0], vars[1], vars[2], vars[3]}, vs2 = vset;
                const uint32_t g0 = m.nd_koff[cn];
                bool ok = true;
#pragma unroll
                for (int g = 0; g < 3; g++)
                    if (ok && g < f.car[j]) ok = bind4(v2, vs2, f.gv[j][g], m.cls_id[m.nd_kpos[g0 + g]]);
                if (ok) next(v2, vs2, p2, ps2);
            }
        };
        uint32_t vars[4] = {0, 0, 0, 0}, vset = 0;
        auto leafc = [&](uint32_t (&v)[4], uint32_t&, uint32_t (&p)[4], uint32_t&) { n++; emit(rid, v, p); };
        auto lvl2 = [&](uint32_t (&v)[4], uint32_t& vs, uint32_t (&p)[4], uint32_t& ps) { child(2, v, vs, p, ps, leafc); };
        auto lvl1 = [&](uint32_t (&v)[4], uint32_t& vs, uint32_t (&p)[4], uint32_t& ps) { child(1, v, vs, p, ps, lvl2); };
        child(0, vars, vset, pv0, ps0, lvl1);
    }
    return n;
}

__device__ __forceinline__ int cmpw(const uint32_t* a, const uint32_t* b, uint32_t W) {
    for (uint32_t i = 0; i < W; i++)
        if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    return 0;
}

__device__ __forceinline__ void swapw(uint32_t* a, uint32_t* b, uint32_t W) {
    for (uint32_t w = 0; w < W; w++) { const uint32_t t = a[w]; a[w] = b[w]; b[w] = t; }
}

// in-place heapsort of n records of W words (the long slices: O(n log n) instead of insertion's n^2)
__device__ __noinline__ void heap_sort_records(uint32_t* base, uint32_t n, uint32_t W) {
    auto sift = [&](uint32_t root, uint32_t end) {
        while (true) {
            uint32_t c = 2 * root + 1;
            if (c >= end) return;
            if (c + 1 < end && cmpw(base + (uint64_t)c * W, base + (uint64_t)(c + 1) * W, W) < 0) c++;
            if (cmpw(base + (uint64_t)root * W, base + (uint64_t)c * W, W) >= 0) return;
            swapw(base + (uint64_t)root * W, base + (uint64_t)c * W, W);
            root = c;
        }
    };
    for (uint32_t i = n / 2; i-- > 0;) sift(i, n);
    for (uint32_t end = n; end-- > 1;) {
        swapw(base, base + (uint64_t)end * W, W);
        sift(0, end);
    }
}

// sort + unique of n records of W words in place; returns unique count
__device__ uint32_t sort_unique(uint32_t* base, uint32_t n, uint32_t W) {
    uint32_t tmp[MAX_W];
    if (n > 32) heap_sort_records(base, n, W);
    else for (uint32_t i = 1; i < n; i++) {
        for (uint32_t w = 0; w < W; w++) tmp[w] = base[i * W + w];
        uint32_t j = i;
        while (j > 0 && cmpw(base + (j - 1) * W, tmp, W) > 0) {
            for (uint32_t w = 0; w < W; w++) base[j * W + w] = base[(j - 1) * W + w];
            j--;
        }
        for (uint32_t w = 0; w < W; w++) base[j * W + w] = tmp[w];
    }
    if (n == 0) return 0;
    uint32_t o = 1;
    for (uint32_t i = 1; i < n; i++)
        if (cmpw(base + (o - 1) * W, base + i * W, W) != 0) {
            if (o != i)
                for (uint32_t w = 0; w < W; w++) base[o * W + w] = base[i * W + w];
            o++;
        }
    return o;
}

}  // namespace

// optional minimum-CTAs-per-SM bounds for occupancy experiments (an explicit 1 is NOT the default:
// it lets ptxas take 120 registers for k_ematch instead of 80)
#ifdef ESAT_EMATCH_MINB
#define ESAT_EMATCH_LB(T) __launch_bounds__(T, ESAT_EMATCH_MINB)
#else
#define ESAT_EMATCH_LB(T) __launch_bounds__(T)
#endif
#ifdef ESAT_JOIN_MINB
#define ESAT_JOIN_LB(T) __launch_bounds__(T, ESAT_JOIN_MINB)
#else
#define ESAT_JOIN_LB(T) __launch_bounds__(T)
#endif
template <int T>
__global__ void ESAT_EMATCH_LB(T) k_ematch(Dev d, MArgs a) {
    // One CTA per leaf runs every pattern of a chunk of <= 32 call patterns (a call with more runs
    // one launch per chunk; the host passes the chunk's slices of the pattern ids, [pattern][leaf]
    // count / offset rows, per-leaf mask words and scratch). The leaf's clean view (class ids/offsets,
    // node symbols, child CSR) is staged into shared memory with TMA bulk copies when it fits,
    // so the backtracking matcher's dependent loads hit SMEM instead of L2.
    extern __shared__ __align__(16) unsigned char dsm[];
    constexpr uint32_t PROG_WORDS = 1024, SYM_WORDS = 1024;
    __shared__ int32_t sprog[PROG_WORDS];
    __shared__ uint32_t ssym[SYM_WORDS];
    __shared__ uint32_t sh_scan[33];
    __shared__ unsigned long long sh_base;
    __shared__ __align__(8) uint64_t bar;
    constexpr uint32_t MAXP = 32;   // patterns per launch (a call of P patterns runs ceil(P/32) launches)
    __shared__ uint32_t sh_tot[MAXP];
    __shared__ unsigned long long sh_pbase[MAXP];
    const uint32_t l = blockIdx.x, tid = threadIdx.x;
    if (tid < MAXP) sh_tot[tid] = 0;
    const uint32_t L = d.L;
    const uint64_t b = d.nb[l];
    const uint32_t C = d.v_C[l];
    const uint32_t* g_cls_id = d.cls_id + b;
    const uint32_t* g_cls_off = d.cls_off + b + l;
    const uint32_t N = g_cls_off[C];
    const uint32_t* g_nd_sym = d.nd_sym + b;
    const uint32_t* g_nd_koff = d.nd_koff + b + l;
    const uint32_t K = g_nd_koff[N];
    const uint32_t* g_nd_kpos = d.nd_kpos + d.kb[l];
    Matcher m;
    // stage the hot part of the view (class node ranges + node symbols) with TMA bulk copies
    const uint32_t need = staged_bytes_u32(g_cls_off, C + 1) + staged_bytes_u32(g_nd_sym, N);
    m.cls_id = g_cls_id; m.nd_koff = g_nd_koff; m.nd_kpos = g_nd_kpos;
    if (need <= a.smem_bytes) {
        if (tid == 0) mbar_init(&bar, 1);
        __syncthreads();
        unsigned char* cur = dsm;
        uint32_t tx = 0;
        const bool issuer = tid == 0;
        if (issuer) mbar_arrive_expect_tx(&bar, need);
        m.cls_off = stage_u32(g_cls_off, C + 1, &cur, &bar, &tx, issuer);
        m.nd_sym = stage_u32(g_nd_sym, N, &cur, &bar, &tx, issuer);
    } else {
        m.cls_off = g_cls_off; m.nd_sym = g_nd_sym;
    }
    // symbol table (name, arity, attribute CSR) in shared memory when it fits
    const uint32_t ns = d.n_syms, npar = d.sym_poff[ns];
    if (3 * ns + 1 + npar <= SYM_WORDS) {
        for (uint32_t i = tid; i < ns; i += T) { ssym[i] = d.sym_name[i]; ssym[ns + i] = d.sym_arity[i]; }
        for (uint32_t i = tid; i <= ns; i += T) ssym[2 * ns + i] = d.sym_poff[i];
        for (uint32_t i = tid; i < npar; i += T) ssym[3 * ns + 1 + i] = (uint32_t)d.sym_par[i];
        m.s_name = ssym; m.s_arity = ssym + ns; m.s_poff = ssym + 2 * ns;
        m.s_par = reinterpret_cast<const int32_t*>(ssym + 3 * ns + 1);
    } else {
        m.s_name = d.sym_name; m.s_arity = d.sym_arity; m.s_poff = d.sym_poff; m.s_par = d.sym_par;
    }
    // the call's pattern programs: warp 0 reads every pattern's program range at once (a scan gives
    // the shared-memory offsets), then the block copies them word-parallel
    __shared__ uint32_t sp_po[MAXP], sp_pn[MAXP], sp_so[MAXP + 1];
    if (tid < 32) {
        uint32_t po = 0, pn = 0;
        if (tid < a.P) {
            const uint32_t pid = a.pat_ids[tid];
            po = a.prog_off[pid];
            pn = a.prog_off[pid + 1] - po;
        }
        uint32_t inc = pn;
#pragma unroll
        for (uint32_t d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
            if (tid >= d) inc += y;
        }
        if (tid < a.P) { sp_po[tid] = po; sp_pn[tid] = pn; sp_so[tid] = inc - pn; }
        if (tid == 31) sp_so[MAXP] = inc;
    }
    __syncthreads();
    const uint32_t pwords = sp_so[MAXP];
    const bool progs_smem = pwords <= PROG_WORDS;
    if (progs_smem)   // a warp per pattern, its lanes over the program's words
        for (uint32_t pi = tid >> 5; pi < a.P; pi += T / 32)
            for (uint32_t w = tid & 31u; w < sp_pn[pi]; w += 32) sprog[sp_so[pi] + w] = a.prog[sp_po[pi] + w];
    __syncthreads();
    if (need <= a.smem_bytes) mbar_wait(&bar, 0);

    // per-class mask of the operator names present (ids < 32): a pattern whose root operator is
    // absent from a class cannot match there, which prunes most (pattern, class) pairs at once
    uint32_t* cmask = (need <= a.smem_bytes && need + 4 * C + 16 <= a.smem_bytes)
                          ? reinterpret_cast<uint32_t*>(dsm + ((need + 15) & ~15u))
                          : nullptr;
    if (cmask) {
        for (uint32_t k = tid; k < C; k += T) {
            uint32_t mk = 0;
            for (uint32_t nd = m.cls_off[k]; nd < m.cls_off[k + 1]; nd++) {
                const uint32_t nm = m.s_name[m.nd_sym[nd]];
                mk |= nm < 32 ? (1u << nm) : 0xFFFFFFFFu;
            }
            cmask[k] = mk;
        }
        __syncthreads();
    }
    const uint32_t ch = (C + T - 1) / T;
    const uint32_t c_lo = min(C, tid * ch), c_hi = min(C, c_lo + ch);
    auto nothing = [](uint32_t, const uint32_t*, const int32_t*) {};
    // per-pattern program pointers
    auto prog_of = [&](uint32_t pi, uint32_t& poff_smem) -> const int32_t* {
        (void)poff_smem;
        return progs_smem ? sprog + sp_so[pi] : a.prog + sp_po[pi];
    };
    auto set_prog = [&](const int32_t* pg) {
        m.prog = pg;
        m.P = pg[0]; m.V = pg[1]; m.Q = pg[2];
    };
    // root-operator filter bit (0 = no filtering: root is a variable or the name id is large)
    auto root_bit = [&]() -> uint32_t {
        const uint32_t rname = (uint32_t)m.prog[3 + 1];
        return (cmask && m.prog[3] == 1 && rname < 32) ? (1u << rname) : 0u;
    };

    const uint32_t lmask = a.leaf_mask ? a.leaf_mask[l] : 0xFFFFFFFFu;   // patterns this leaf needs
    if (a.mode == 1) {  // existence only (is_rule_applicable, rewrite.py:579-589)
        uint32_t po = 0;
        for (uint32_t pi = 0; pi < a.P; pi++) {
            if (!((lmask >> pi) & 1u)) {
                if (tid == 0) { a.count[(uint64_t)pi * L + l] = 0; a.off[(uint64_t)pi * L + l] = 0; }
                continue;
            }
            set_prog(prog_of(pi, po));
            const uint32_t rbit = root_bit();
            uint32_t any = 0;
            for (uint32_t r = c_lo; r < c_hi && !any; r++)
                if (!rbit || (cmask[r] & rbit)) any = match_class(m, r, true, nothing);
            any = __syncthreads_or(any);
            if (tid == 0) { a.count[(uint64_t)pi * L + l] = any ? 1u : 0u; a.off[(uint64_t)pi * L + l] = 0; }
        }
        return;
    }
    // ---- LIST mode: balanced (pattern, class) work over the flattened index space ----
    // pass 1 counts raw matches of every (pattern, root class) pair into a per-leaf scratch row;
    // a segmented scan turns them into record offsets (pattern-major, class order = the
    // reference's sort order by root); pass 2 writes each pair's records at its offset and
    // sorts + dedups them in place (rewrite.py:420-433).
    __shared__ uint32_t sp_off[MAXP], sp_W[MAXP], sp_rbit[MAXP], sp_dup[MAXP];
    __shared__ Flat2 sp_flat[MAXP];
    __shared__ uint32_t sp_rbase[MAXP + 1];
    __shared__ unsigned long long sp_wbase[MAXP];
    const uint32_t P = a.P;
    if (tid < P) {
        const uint32_t pi = tid;
        sp_off[pi] = progs_smem ? sp_so[pi] : sp_po[pi];
        const int32_t* pg = (progs_smem ? sprog : a.prog) + sp_off[pi];
        sp_W[pi] = 1 + pg[1] + pg[2];
        const uint32_t rname = (uint32_t)pg[3 + 1];
        sp_rbit[pi] = (cmask && pg[3] == 1 && rname < 32) ? (1u << rname) : 0u;
        sp_dup[pi] = 0;
    }
    for (uint32_t pi = tid; pi < P; pi += T) {
        decode_flat2((progs_smem ? sprog + sp_so[pi] : a.prog + sp_po[pi]), sp_flat[pi]);
        if (a.no_flat) sp_flat[pi].ok = 0;
    }
    __syncthreads();
    auto prog_ptr = [&](uint32_t pi) -> const int32_t* { return (progs_smem ? sprog : a.prog) + sp_off[pi]; };
    const uint32_t PC = P * C;
    const float invC = C ? 1.0f / (float)C : 0.0f;
    // i / C for i < P * C (quotient < 32): a float estimate, exact after one correction step
    auto div_c = [&](uint32_t i) -> uint32_t {
        uint32_t q = (uint32_t)((float)i * invC);
        if (q * C > i) q--;
        else if ((q + 1) * C <= i) q++;
        return q;
    };
    uint32_t* pc = a.raw + d.nb[l] * MAXP;   // [P][C] counts -> offsets (C <= n, P <= 32)
    uint32_t* nzl = a.nzl + d.nb[l] * MAXP;  // (pattern, class) pairs with matches (any order)
    __shared__ uint32_t sh_nz, sh_next, sh_next2;
    if (tid == 0) { sh_nz = 0; sh_next = T; sh_next2 = T; }
    __syncthreads();
    // (pattern, class) pairs are handed out dynamically: a thread that drew a heavy pair does not
    // also own a fixed share of the rest
    for (uint32_t i = tid; i < PC; i = atomicAdd(&sh_next, 1u)) {
        const uint32_t pi = div_c(i), r = i - pi * C;
        uint32_t n = 0;
        const uint32_t rb = sp_rbit[pi];
        if (((lmask >> pi) & 1u) && (!rb || (cmask[r] & rb))) {
            if (sp_flat[pi].ok) {
                n = match_class_flat2(m, sp_flat[pi], r, [](uint32_t, const uint32_t (&)[4], const uint32_t (&)[4]) {});
            } else {
                set_prog(prog_ptr(pi));
                n = match_class(m, r, false, nothing);
            }
        }
        pc[i] = n;
        if (n) nzl[atomicAdd(&sh_nz, 1u)] = i;
    }
    __syncthreads();
    // exclusive scan of pc in place: each warp owns a contiguous, 128-aligned share and walks it 128
    // elements at a time (one uint4 per lane, coalesced) with a 4-wide local prefix + shuffle scan;
    // pass A sums, pass B writes prefixes. pc rows start 128-B aligned (leaf base x 32 words).
    {
        constexpr uint32_t NW = T / 32;
        __shared__ uint32_t sh_wsum[NW];
        const uint32_t lane = tid & 31, warp = tid >> 5;
        const uint32_t qw = ((PC + NW - 1) / NW + 127) & ~127u;
        const uint32_t lo = min(PC, warp * qw), hi = min(PC, lo + qw);
        auto load4 = [&](uint32_t i) -> uint4 {   // elements i..i+3, zero past hi
            if (i + 3 < hi) return reinterpret_cast<const uint4*>(pc)[i >> 2];
            uint4 q = make_uint4(0, 0, 0, 0);
            if (i < hi) q.x = pc[i];
            if (i + 1 < hi) q.y = pc[i + 1];
            if (i + 2 < hi) q.z = pc[i + 2];
            return q;
        };
        uint32_t sum = 0;
        for (uint32_t i = lo + 4 * lane; i < hi; i += 128) {
            const uint4 q = load4(i);
            sum += q.x + q.y + q.z + q.w;
        }
        sum = __reduce_add_sync(0xffffffffu, sum);
        if (lane == 0) sh_wsum[warp] = sum;
        __syncthreads();
        uint32_t carry = 0, total = 0;
        for (uint32_t w = 0; w < NW; w++) { if (w < warp) carry += sh_wsum[w]; total += sh_wsum[w]; }
        for (uint32_t b0 = lo; b0 < hi; b0 += 128) {
            const uint32_t i = b0 + 4 * lane;
            const uint4 q = load4(i);
            const uint32_t s0 = q.x, s1 = s0 + q.y, s2 = s1 + q.z, s3 = s2 + q.w;
            uint32_t x = s3;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= (uint32_t)o) x += y;
            }
            const uint32_t ex = carry + x - s3;
            const uint4 r = make_uint4(ex, ex + s0, ex + s1, ex + s2);
            if (i + 3 < hi) {
                reinterpret_cast<uint4*>(pc)[i >> 2] = r;
            } else {
                if (i < hi) pc[i] = r.x;
                if (i + 1 < hi) pc[i + 1] = r.y;
                if (i + 2 < hi) pc[i + 2] = r.z;
            }
            carry += __shfl_sync(0xffffffffu, x, 31);
        }
        __syncthreads();
        if (tid <= P) sp_rbase[tid] = (tid < P && C) ? pc[tid * C] : (tid == P ? total : 0u);
        __syncthreads();
    }
    if (tid == 0) {   // one output allocation for the whole leaf
        unsigned long long words = 0;
        for (uint32_t pi = 0; pi < P; pi++) {
            sp_wbase[pi] = words;
            words += (unsigned long long)(sp_rbase[pi + 1] - sp_rbase[pi]) * sp_W[pi];
        }
        unsigned long long base = atomicAdd(&a.tops[1], words);
        if (base + words > a.out_cap) { atomicOr(a.overflow, 2u); base = ~0ull; }
        sh_base = base;
        for (uint32_t pi = 0; pi < P; pi++) sp_wbase[pi] = base == ~0ull ? ~0ull : base + sp_wbase[pi];
    }
    __syncthreads();
    if (sh_base != ~0ull) {
        const uint32_t grand = sp_rbase[P], nz = sh_nz;
        for (uint32_t j = tid; j < nz; j = atomicAdd(&sh_next2, 1u)) {
            const uint32_t i = nzl[j];
            const uint32_t beg = pc[i], end = (i + 1 < PC) ? pc[i + 1] : grand;
            if (beg == end) continue;
            const uint32_t pi = div_c(i), r = i - pi * C, W = sp_W[pi];
            set_prog(prog_ptr(pi));
            uint32_t* o0 = a.out + sp_wbase[pi] + (uint64_t)(beg - sp_rbase[pi]) * W;
            uint32_t cur = 0;
            if (sp_flat[pi].ok) {
                const Flat2& f = sp_flat[pi];
                match_class_flat2(m, f, r, [&](uint32_t root, const uint32_t (&vars)[4], const uint32_t (&pv)[4]) {
                    uint32_t* o = o0 + (uint64_t)cur * W;
                    o[0] = root;
#pragma unroll
                    for (int v = 0; v < 4; v++) if (v < f.V) o[1 + v] = vars[v];
#pragma unroll
                    for (int q = 0; q < 4; q++) if (q < f.Q) o[1 + f.V + q] = pv[q];
                    cur++;
                });
            } else {
                match_class(m, r, false, [&](uint32_t root, const uint32_t* vars, const int32_t* pv) {
                    uint32_t* o = o0 + (uint64_t)cur * W;
                    o[0] = root;
                    for (int v = 0; v < m.V; v++) o[1 + v] = vars[v];
                    for (int q = 0; q < m.Q; q++) o[1 + m.V + q] = (uint32_t)pv[q];
                    cur++;
                });
            }
            if (cur > 1) {
                const uint32_t u = sort_unique(o0, cur, W);
                if (u != cur) {   // duplicate bindings from different e-nodes: mark the gap
                    for (uint32_t w = u * W; w < cur * W; w++) o0[w] = NONE;
                    atomicOr(&sp_dup[pi], 1u);
                }
            }
        }
    }
    __syncthreads();
    // squeeze out the gaps deduplicated slices left (records whose root word is NONE), block-wide
    // and in order: chunks of T records are read, ranked by a block scan and written back; a
    // record only ever moves left, never into the unread part of the list
    __shared__ uint32_t sp_final[MAXP];
    if (tid < P) sp_final[tid] = sp_rbase[tid + 1] - sp_rbase[tid];
    __syncthreads();
    if (sh_base != ~0ull)
        for (uint32_t pi = 0; pi < P; pi++) {
            if (!sp_dup[pi]) continue;
            const uint32_t W = sp_W[pi], tot = sp_final[pi];
            uint32_t* base = a.out + sp_wbase[pi];
            uint32_t o = 0;
            for (uint32_t c0 = 0; c0 < tot; c0 += T) {
                const uint32_t rr = c0 + tid;
                uint32_t rec[MAX_W];
                const bool keep = rr < tot && base[(uint64_t)rr * W] != NONE;
                if (keep)
                    for (uint32_t w = 0; w < W; w++) rec[w] = base[(uint64_t)rr * W + w];
                uint32_t kt;
                const uint32_t pos = block_exscan(keep ? 1u : 0u, sh_scan, &kt);
                __syncthreads();
                if (keep)
                    for (uint32_t w = 0; w < W; w++) base[(uint64_t)(o + pos) * W + w] = rec[w];
                o += kt;
                __syncthreads();
            }
            if (tid == 0) sp_final[pi] = o;
            __syncthreads();
        }
    if (tid < P) {
        const uint32_t pi = tid;
        const uint64_t oi = (uint64_t)pi * L + l;
        a.count[oi] = sh_base == ~0ull ? 0 : sp_final[pi];
        a.off[oi] = sh_base == ~0ull ? 0 : sp_wbase[pi];
    }
}

// ---------------------------------------------------------------------------------------------
namespace {

struct Src {
    const uint32_t* w;   // records
    uint32_t n, W, V, Q;
    const uint32_t *vmap, *qmap;
};

// Combination of one record per source: consistency on shared vars/pvars; fills out[].
__device__ __forceinline__ bool combine(const Src* src, int S, const uint32_t* idx, uint32_t NV, uint32_t NQ,
                                        uint32_t* out) {
    uint64_t vset = 0, qset = 0;
    for (int s = 0; s < S; s++) {
        const uint32_t* r = src[s].w + (uint64_t)idx[s] * src[s].W;
        out[s] = r[0];
        for (uint32_t v = 0; v < src[s].V; v++) {
            const uint32_t o = src[s].vmap[v];
            if (!(vset >> o & 1ull)) { vset |= 1ull << o; out[S + o] = r[1 + v]; }
            else if (out[S + o] != r[1 + v]) return false;
        }
        for (uint32_t q = 0; q < src[s].Q; q++) {
            const uint32_t o = src[s].qmap[q];
            if (!(qset >> o & 1ull)) { qset |= 1ull << o; out[S + NV + o] = r[1 + src[s].V + q]; }
            else if (out[S + NV + o] != r[1 + src[s].V + q]) return false;
        }
    }
    return true;
}

__device__ __forceinline__ uint32_t group_end(const Src& s, uint32_t i) {
    const uint32_t root = s.w[(uint64_t)i * s.W];
    uint32_t j = i + 1;
    while (j < s.n && s.w[(uint64_t)j * s.W] == root) j++;
    return j;
}

// group_end for a converged warp: 32 records tested per step
__device__ __forceinline__ uint32_t group_end_warp(const Src& s, uint32_t i, uint32_t lane) {
    const uint32_t root = s.w[(uint64_t)i * s.W];
    for (uint32_t j = i + 1;; j += 32) {
        const uint32_t q = j + lane;
        const bool stop = q >= s.n || s.w[(uint64_t)q * s.W] != root;
        const uint32_t m = __ballot_sync(0xffffffffu, stop);
        if (m) return j + __ffs(m) - 1;
    }
}

__device__ __forceinline__ uint32_t group_start_at_or_after(const Src& s, uint32_t p) {
    if (p == 0 || p >= s.n) return p >= s.n ? s.n : 0;
    while (p < s.n && s.w[(uint64_t)p * s.W] == s.w[(uint64_t)(p - 1) * s.W]) p++;
    return p;
}

// Visit every block (source-0 group g0 x root groups of sources 1..S-1); for each block call
// f(block_first_idx[], block_end_idx[]).
template <typename F>
__device__ void for_blocks(const Src* src, int S, uint32_t g0_lo, uint32_t g0_hi, F f) {
    uint32_t lo[MAX_S], hi[MAX_S];
    lo[0] = g0_lo; hi[0] = g0_hi;
    // odometer over groups of sources 1..S-1
    for (int s = 1; s < S; s++) { lo[s] = 0; hi[s] = group_end(src[s], 0); }
    for (;;) {
        f(lo, hi);
        int s = S - 1;
        for (; s >= 1; s--) {
            lo[s] = hi[s];
            if (lo[s] < src[s].n) { hi[s] = group_end(src[s], lo[s]); break; }
            lo[s] = 0;
            hi[s] = group_end(src[s], 0);
        }
        if (s < 1) return;
    }
}

template <typename Emit>
__device__ uint32_t block_products(const Src* src, int S, const uint32_t* lo, const uint32_t* hi, uint32_t NV,
                                   uint32_t NQ, Emit emit) {
    uint32_t idx[MAX_S], rec_[MAX_W];
    for (int s = 0; s < S; s++) idx[s] = lo[s];
    uint32_t n = 0;
    for (;;) {
        if (combine(src, S, idx, NV, NQ, rec_)) { emit(rec_); n++; }
        int s = S - 1;
        for (; s >= 0; s--) {
            if (++idx[s] < hi[s]) break;
            idx[s] = lo[s];
        }
        if (s < 0) return n;
    }
}


constexpr uint32_t JOIN_SMEM_KEYS = 2048;   // source-1 index sorted in shared memory

// Block-wide bitonic sort of n (power of two) u64 keys in shared memory.
__device__ void block_bitonic(unsigned long long* k, uint32_t n) {
    for (uint32_t size = 2; size <= n; size <<= 1)
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            __syncthreads();
            for (uint32_t i = threadIdx.x; i < n / 2; i += blockDim.x) {
                const uint32_t lo = 2 * i - (i & (stride - 1));
                const uint32_t hi = lo + stride;
                const bool up = ((lo & size) == 0);
                const unsigned long long a = k[lo], b = k[hi];
                if ((a > b) == up) { k[lo] = b; k[hi] = a; }
            }
        }
    __syncthreads();
}

__device__ __forceinline__ uint32_t lower_bound_key(const unsigned long long* k, uint32_t n, unsigned long long x) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (k[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// Output plan of a two-source join (shared memory): output word w comes from source src[w]
// at word idx[w]; nchk pairs of (source-0 word, source-1 word) must be equal.
struct JoinPlan {
    uint8_t src[MAX_W], idx[MAX_W];
    uint8_t c0[2 * MAX_V], c1[2 * MAX_V];
    uint32_t nchk, W;
    // source-1 fields the join reads (output words from source 1, consistency checks), staged in
    // SMEM in sorted-index order: record p's field f at s1[p * F + f]
    uint8_t f1[MAX_W + 2 * MAX_V], s1idx[MAX_W], s1chk[2 * MAX_V];
    uint32_t F;
};

__device__ uint8_t plan_slot(JoinPlan& p, uint8_t field) {
    for (uint32_t f = 0; f < p.F; f++)
        if (p.f1[f] == field) return (uint8_t)f;
    p.f1[p.F] = field;
    return (uint8_t)p.F++;
}

// v1: source 1's join variable (its equality with source 0's is guaranteed by the index lookup,
// so it needs no per-product check)
__device__ void make_plan(JoinPlan& p, const Src* s, uint32_t NV, uint32_t NQ, uint32_t v1) {
    p.W = 2 + NV + NQ;
    p.src[0] = 0; p.idx[0] = 0; p.src[1] = 1; p.idx[1] = 0;
    for (uint32_t o = 0; o < NV + NQ; o++) { p.src[2 + o] = 255; p.idx[2 + o] = 0; }
    p.nchk = 0;
    for (uint32_t v = 0; v < s[0].V; v++) { p.src[2 + s[0].vmap[v]] = 0; p.idx[2 + s[0].vmap[v]] = 1 + v; }
    for (uint32_t q = 0; q < s[0].Q; q++) {
        p.src[2 + NV + s[0].qmap[q]] = 0;
        p.idx[2 + NV + s[0].qmap[q]] = 1 + s[0].V + q;
    }
    for (uint32_t v = 0; v < s[1].V; v++) {
        const uint32_t o = 2 + s[1].vmap[v];
        if (p.src[o] == 0) {
            if (v != v1) { p.c0[p.nchk] = p.idx[o]; p.c1[p.nchk] = 1 + v; p.nchk++; }
        } else {
            p.src[o] = 1; p.idx[o] = 1 + v;
        }
    }
    for (uint32_t q = 0; q < s[1].Q; q++) {
        const uint32_t o = 2 + NV + s[1].qmap[q];
        if (p.src[o] == 0) { p.c0[p.nchk] = p.idx[o]; p.c1[p.nchk] = 1 + s[1].V + q; p.nchk++; }
        else { p.src[o] = 1; p.idx[o] = 1 + s[1].V + q; }
    }
    p.F = 0;
    for (uint32_t c = 0; c < p.nchk; c++) p.s1chk[c] = plan_slot(p, p.c1[c]);
    for (uint32_t w = 0; w < p.W; w++) p.s1idx[w] = p.src[w] == 1 ? plan_slot(p, p.idx[w]) : 0;
}

// Products of the source-0 records [g, ge) (one root group) with the source-1 records sharing the
// join variable (runs of the sorted index); consistent pairs are written (out != null) in index
// order. Returns the number of products.
__device__ uint32_t indexed_products(const uint32_t* w0, uint32_t W0, const uint32_t* w1, uint32_t W1,
                                     const JoinPlan& jp, uint32_t g, uint32_t ge, uint32_t v0,
                                     const unsigned long long* keys, uint32_t n1, uint32_t* out) {
    uint32_t n = 0;
    const uint32_t W = jp.W;
    for (uint32_t i = g; i < ge; i++) {
        const uint32_t* m1 = w0 + (uint64_t)i * W0;
        const uint32_t x = m1[1 + v0];
        for (uint32_t p = lower_bound_key(keys, n1, (unsigned long long)x << 32); p < n1 && (uint32_t)(keys[p] >> 32) == x;
             p++) {
            const uint32_t* m2 = w1 + (uint64_t)(uint32_t)keys[p] * W1;
            bool ok = true;
            for (uint32_t c = 0; c < jp.nchk && ok; c++) ok = m1[jp.c0[c]] == m2[jp.c1[c]];
            if (!ok) continue;
            if (out) {
                uint32_t* o = out + (uint64_t)n * W;
                for (uint32_t w = 0; w < W; w++) o[w] = jp.src[w] ? m2[jp.idx[w]] : m1[jp.idx[w]];
            }
            n++;
        }
    }
    return n;
}

}  // namespace

// A root group of several source-0 records yields one sorted run of products per record; the runs
// are merged warp-parallel: each record's final rank = its index in its run + (records below it in
// every other run, by binary search), scattered through a per-warp scratch and copied back.
__device__ __noinline__ void merge_group(uint32_t* gout, uint32_t k, uint32_t cnt, uint32_t W, const uint32_t* runs,
                                         uint32_t* tmp, uint32_t lane) {
    for (uint32_t e = lane; e < cnt; e += 32) {
        uint32_t a = 0;
        while (a + 1 < k && runs[a + 1] <= e) a++;
        const uint32_t* rec = gout + (uint64_t)e * W;
        uint32_t rank = e - runs[a];
        for (uint32_t bb = 0; bb < k; bb++) {
            if (bb == a) continue;
            uint32_t lo = runs[bb], hi = runs[bb + 1];   // first record of run bb not below rec
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (cmpw(gout + (uint64_t)mid * W, rec, W) < 0) lo = mid + 1;
                else hi = mid;
            }
            rank += lo - runs[bb];
        }
        for (uint32_t w = 0; w < W; w++) tmp[rank * W + w] = rec[w];
    }
    __syncwarp();
    for (uint32_t q = lane; q < cnt * W; q += 32) gout[q] = tmp[q];
    __syncwarp();
}

// Products of one source-0 record (fields in m1s) with its staged source-1 run [p0, p1): 32 per
// step, consistent ones compacted by ballot and written as consecutive records from row n.
// WC > 0 fixes the record width at compile time (plan columns and the source-0 values live in
// registers); WC == 0 is the runtime-width path.
template <int WC>
__device__ __forceinline__ uint32_t staged_products(const JoinPlan& jp, const uint32_t* s1, const uint32_t* m1s,
                                                    uint32_t p0, uint32_t p1, uint32_t lane, uint32_t* out,
                                                    uint32_t n) {
    const uint32_t F = jp.F, nchk = jp.nchk, W = WC ? (uint32_t)WC : jp.W;
    constexpr int R = WC ? WC : 1;
    uint32_t v0[R], sl[R];
    bool from1[R];
    if (WC) {
#pragma unroll
        for (int w = 0; w < R; w++) {
            from1[w] = jp.src[w] != 0;
            sl[w] = jp.s1idx[w];
            v0[w] = m1s[jp.idx[w]];
        }
    }
    for (uint32_t base = p0; base < p1; base += 32) {
        const uint32_t p = base + lane;
        bool ok = p < p1;
        const uint32_t* m2 = s1 + (ok ? p : 0u) * F;
        if (nchk)
            for (uint32_t c = 0; c < nchk && ok; c++) ok = m1s[jp.c0[c]] == m2[jp.s1chk[c]];
        const uint32_t mask = __ballot_sync(0xffffffffu, ok);
        if (out && ok) {
            uint32_t* o = out + (uint64_t)(n + __popc(mask & ((1u << lane) - 1u))) * W;
            if (WC) {
#pragma unroll
                for (int w = 0; w < R; w++) o[w] = from1[w] ? m2[sl[w]] : v0[w];
            } else {
                for (uint32_t w = 0; w < W; w++) o[w] = jp.src[w] ? m2[jp.s1idx[w]] : m1s[jp.idx[w]];
            }
        }
        n += __popc(mask);
    }
    return n;
}

// ---- long-list joins (BASELINE config 4's explosion) ---------------------------------------
// Source 1 is sorted by every field it shares with source 0 (the join variable first, then the
// checked variables / attributes, then the record), so a source-0 record's consistent partners are
// exactly one run of the index and its product count is the run length. The preparing CTA writes,
// per source-0 record, the run and the output offset (record order = output order); k_join_big
// then fills the products with a grid of CTAs over source-0 root groups.
__device__ __forceinline__ int tuple_cmp(const uint32_t* ra, const uint32_t* fa, const uint32_t* rb,
                                         const uint32_t* fb, uint32_t nf) {
    for (uint32_t f = 0; f < nf; f++) {
        const uint32_t x = ra[fa[f]], y = rb[fb[f]];
        if (x != y) return x < y ? -1 : 1;
    }
    return 0;
}

template <int T>
__device__ void big_prepare(const JArgs& a, const Src* src, uint32_t NV, uint32_t NQ, uint32_t W, uint32_t v0,
                            uint32_t v1, uint32_t n1p, uint32_t l, uint32_t r, uint32_t L, uint32_t* sh_scan) {
    const uint32_t tid = threadIdx.x, n0 = src[0].n, n1 = src[1].n;
    __shared__ JoinPlan plan;
    __shared__ uint32_t f0[1 + 2 * MAX_V], f1[1 + 2 * MAX_V];
    __shared__ uint32_t sh_nf;
    __shared__ unsigned long long sh_off, sh_base;
    if (tid == 0) {
        make_plan(plan, src, NV, NQ, v1);
        f0[0] = 1 + v0;
        f1[0] = 1 + v1;
        for (uint32_t c = 0; c < plan.nchk; c++) { f0[1 + c] = plan.c0[c]; f1[1 + c] = plan.c1[c]; }
        sh_nf = 1 + plan.nchk;
        const unsigned long long need = (unsigned long long)n1p + 2ull * n0;
        unsigned long long o = atomicAdd(&a.tops[0], need);
        if (o + need > a.gkey_cap) { atomicOr(a.overflow, 4u); o = ~0ull; }
        sh_off = o;
    }
    __syncthreads();
    const uint64_t pi = (uint64_t)r * L + l;
    if (sh_off == ~0ull) {   // no scratch yet: the relaunch after regrowth does the work
        if (tid == 0) { a.count[pi] = 0; a.off[pi] = 0; }
        return;
    }
    unsigned long long* keys = a.gkeys + sh_off;
    unsigned long long* recs = keys + n1p;   // [n0][2]: output record offset, run p0 | p1 << 32
    const uint32_t nf = sh_nf, W1 = src[1].W, W0 = src[0].W;
    const uint32_t *w0 = src[0].w, *w1 = src[1].w;
    for (uint32_t i = tid; i < n1p; i += T) keys[i] = i < n1 ? i : ~0ull;
    __syncthreads();
    // bitonic sort of record indices by (shared fields, index); padding sorts last
    for (uint32_t size = 2; size <= n1p; size <<= 1)
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = tid; i < n1p / 2; i += T) {
                const uint32_t lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
                const bool up = (lo & size) == 0;
                const unsigned long long x = keys[lo], y = keys[hi];
                bool gt;
                if (x == ~0ull || y == ~0ull) gt = x == ~0ull && y != ~0ull;
                else {
                    const int c = tuple_cmp(w1 + x * W1, f1, w1 + y * W1, f1, nf);
                    gt = c > 0 || (c == 0 && x > y);
                }
                if (gt == up) { keys[lo] = y; keys[hi] = x; }
            }
            __syncthreads();
        }
    // per source-0 record: its run of consistent partners, then output offsets by a block scan
    unsigned long long carry = 0;
    for (uint32_t c0 = 0; c0 < n0; c0 += T) {
        const uint32_t i = c0 + tid;
        uint32_t p0 = 0, p1 = 0;
        if (i < n0) {
            const uint32_t* m0 = w0 + (uint64_t)i * W0;
            uint32_t lo = 0, hi = n1;
            while (lo < hi) {   // first partner not below the record's tuple
                const uint32_t mid = (lo + hi) >> 1;
                if (tuple_cmp(w1 + keys[mid] * W1, f1, m0, f0, nf) < 0) lo = mid + 1; else hi = mid;
            }
            p0 = lo;
            hi = n1;
            while (lo < hi) {   // first partner above it
                const uint32_t mid = (lo + hi) >> 1;
                if (tuple_cmp(w1 + keys[mid] * W1, f1, m0, f0, nf) <= 0) lo = mid + 1; else hi = mid;
            }
            p1 = lo;
        }
        uint32_t tot;
        const uint32_t pre = block_exscan(p1 - p0, sh_scan, &tot);
        if (i < n0) {
            recs[2 * (uint64_t)i] = carry + pre;
            recs[2 * (uint64_t)i + 1] = (unsigned long long)p0 | ((unsigned long long)p1 << 32);
        }
        carry += tot;
        __syncthreads();
    }
    if (tid == 0) {
        unsigned long long base = atomicAdd(&a.tops[1], carry * W);
        if (base + carry * W > a.out_cap) { atomicOr(a.overflow, 2u); base = ~0ull; }
        sh_base = base;
        a.count[pi] = base == ~0ull ? 0 : (uint32_t)carry;
        a.off[pi] = base == ~0ull ? 0 : base;
        if (base != ~0ull) {
            a.big[2 * pi] = sh_off;
            a.big[2 * pi + 1] = base;
            atomicAdd(&a.tops[2], 1ull);
        }
    }
}

// Products of the long-list pairs prepared by k_join: grid (L, R, Z), CTA z takes the z-th share of
// source 0's root groups; a warp writes each record's run 32 products at a time at the record's
// offset, then orders groups of several records (their runs are sorted, the group is sorted + deduped).
template <int T>
__global__ void __launch_bounds__(T) k_join_big(uint32_t L, JArgs a) {
    const uint32_t l = blockIdx.x, r = blockIdx.y, z = blockIdx.z, Z = gridDim.z, tid = threadIdx.x;
    const uint64_t pi = (uint64_t)r * L + l;
    if (a.big[2 * pi] == ~0ull) return;
    const uint32_t s0 = a.src_off[r], S = a.src_off[r + 1] - s0;
    if (S != 2) return;
    const uint32_t NV = a.nv[r], NQ = a.nq[r], W = S + NV + NQ;
    Src src[2];
    for (uint32_t s = 0; s < 2; s++) {
        const uint32_t p = a.src[s0 + s];
        const uint64_t mi = (uint64_t)p * L + l;
        src[s].n = a.m_count[mi];
        src[s].w = a.m_words + a.m_off[mi];
        src[s].W = a.m_W[p];
        const uint32_t vo = a.map_off[2 * (s0 + s)], qo = a.map_off[2 * (s0 + s) + 1];
        src[s].V = a.map_off[2 * (s0 + s + 1)] - vo;
        src[s].Q = a.map_off[2 * (s0 + s + 1) + 1] - qo;
        src[s].vmap = a.vmap + vo;
        src[s].qmap = a.qmap + qo;
    }
    uint32_t v0 = NONE, v1 = NONE;
    for (uint32_t b = 0; b < src[1].V && v0 == NONE; b++)
        for (uint32_t a0 = 0; a0 < src[0].V; a0++)
            if (src[0].vmap[a0] == src[1].vmap[b]) { v0 = a0; v1 = b; break; }
    __shared__ JoinPlan plan;
    if (tid == 0) make_plan(plan, src, NV, NQ, v1);
    __syncthreads();
    const uint32_t n0 = src[0].n, n1 = src[1].n;
    uint32_t n1p = 1;
    while (n1p < n1) n1p <<= 1;
    const unsigned long long* keys = a.gkeys + a.big[2 * pi];
    const unsigned long long* recs = keys + n1p;
    uint32_t* out = a.out + a.big[2 * pi + 1];
    const uint32_t *w0 = src[0].w, *w1 = src[1].w;
    const uint32_t W0 = src[0].W, W1 = src[1].W;
    constexpr uint32_t NW = T / 32;
    const uint32_t warp = tid >> 5, lane = tid & 31;
    const uint32_t chz = (n0 + Z - 1) / Z;
    const uint32_t zlo = group_start_at_or_after(src[0], min(n0, z * chz));
    const uint32_t zhi = group_start_at_or_after(src[0], min(n0, (z + 1) * chz));
    const uint32_t chw = (zhi - zlo + NW - 1) / NW;
    const uint32_t wlo = group_start_at_or_after(src[0], min(zhi, zlo + warp * chw));
    const uint32_t whi = group_start_at_or_after(src[0], min(zhi, zlo + (warp + 1) * chw));
    for (uint32_t g = wlo; g < whi;) {
        const uint32_t ge = group_end_warp(src[0], g, lane);
        for (uint32_t i = g; i < ge; i++) {
            const uint32_t* m1 = w0 + (uint64_t)i * W0;
            const unsigned long long o = recs[2 * (uint64_t)i], rr = recs[2 * (uint64_t)i + 1];
            const uint32_t p0 = (uint32_t)rr, p1 = (uint32_t)(rr >> 32);
            for (uint32_t p = p0 + lane; p < p1; p += 32) {
                const uint32_t* m2 = w1 + keys[p] * W1;
                uint32_t* ob = out + (o + (p - p0)) * W;
                for (uint32_t w = 0; w < W; w++) ob[w] = plan.src[w] ? m2[plan.idx[w]] : m1[plan.idx[w]];
            }
        }
        if (ge - g > 1) {   // several source-0 records share the root: order the group's products
            __syncwarp();
            const unsigned long long gb = recs[2 * (uint64_t)g];
            const unsigned long long rr = recs[2 * (uint64_t)(ge - 1) + 1];
            const unsigned long long gend = recs[2 * (uint64_t)(ge - 1)] + ((uint32_t)(rr >> 32) - (uint32_t)rr);
            if (lane == 0) sort_unique(out + gb * W, (uint32_t)(gend - gb), W);
            __syncwarp();
        }
        g = ge;
    }
    (void)v0;
}

template <int T>
__global__ void ESAT_JOIN_LB(T) k_join(uint32_t L, JArgs a) {
    const uint32_t l = blockIdx.x, r = blockIdx.y, tid = threadIdx.x;
    __shared__ uint32_t sh_scan[33];
    __shared__ unsigned long long sh_base;
    const uint32_t s0 = a.src_off[r], S = a.src_off[r + 1] - s0;
    const uint32_t NV = a.nv[r], NQ = a.nq[r], W = S + NV + NQ;
    Src src[MAX_S];
    bool empty = false;
    for (uint32_t s = 0; s < S; s++) {
        const uint32_t p = a.src[s0 + s];
        const uint64_t mi = (uint64_t)p * L + l;
        src[s].n = a.m_count[mi];
        src[s].w = a.m_words + a.m_off[mi];
        src[s].W = a.m_W[p];
        const uint32_t vo = a.map_off[2 * (s0 + s)], qo = a.map_off[2 * (s0 + s) + 1];
        src[s].V = a.map_off[2 * (s0 + s + 1)] - vo;
        src[s].Q = a.map_off[2 * (s0 + s + 1) + 1] - qo;
        src[s].vmap = a.vmap + vo;
        src[s].qmap = a.qmap + qo;
        if (!src[s].n) empty = true;
    }
    // threads own whole root groups of source 0
    uint32_t g_lo = 0, g_hi = 0;
    if (!empty) {
        const uint32_t n0 = src[0].n, ch = (n0 + T - 1) / T;
        g_lo = group_start_at_or_after(src[0], min(n0, tid * ch));
        g_hi = group_start_at_or_after(src[0], min(n0, (tid + 1) * ch));
    }
    // sort-join fast path: two sources sharing a variable -> index source 1 by that variable
    __shared__ unsigned long long sh_keys[JOIN_SMEM_KEYS];
    uint32_t v0 = NONE, v1 = NONE;
    if (S == 2 && !empty)
        for (uint32_t b = 0; b < src[1].V && v0 == NONE; b++)
            for (uint32_t a0 = 0; a0 < src[0].V; a0++)
                if (src[0].vmap[a0] == src[1].vmap[b]) { v0 = a0; v1 = b; break; }
    // long source-1 lists (e-graph explosion): the CTA only prepares an index over every shared
    // field and per-record product runs; k_join_big writes the products with many CTAs
    const bool big = v0 != NONE && src[1].n > JOIN_SMEM_KEYS;
    uint32_t n1p = 0;
    if (v0 != NONE) {
        n1p = 1;
        while (n1p < src[1].n) n1p <<= 1;
    }
    if (big) {
        big_prepare<T>(a, src, NV, NQ, W, v0, v1, n1p, l, r, L, sh_scan);
        return;
    }
    unsigned long long* keys = sh_keys;
    auto key_at = [&](uint32_t p) -> unsigned long long { return sh_keys[p]; };
    const bool indexed = v0 != NONE;
    if (indexed) {
        for (uint32_t i = tid; i < n1p; i += T)
            keys[i] = i < src[1].n ? ((unsigned long long)src[1].w[(uint64_t)i * src[1].W + 1 + v1] << 32) | i
                                   : ~0ull;
        __syncthreads();
        block_bitonic(keys, n1p);
    }
    const uint32_t* w0 = src[0].w;
    const uint32_t* w1 = src[S > 1 ? 1 : 0].w;
    const uint32_t W0 = src[0].W, W1 = src[S > 1 ? 1 : 0].W;
    __shared__ JoinPlan sh_plan;
    if (indexed && tid == 0) make_plan(sh_plan, src, NV, NQ, v1);
    __syncthreads();
    extern __shared__ uint32_t jrun[];
    uint32_t* s1 = jrun + a.run_cap;
    const bool staged = indexed && src[1].n * sh_plan.F <= a.s1_cap;
    if (staged) {   // source-1 fields in sorted-index order: the walk reads SMEM, not scattered global words
        const uint32_t F = sh_plan.F, W1s = src[1].W;
        for (uint32_t e = tid; e < src[1].n * F; e += T) {
            const uint32_t p = e / F, f = e - p * F;
            s1[e] = src[1].w[(uint64_t)(uint32_t)key_at(p) * W1s + sh_plan.f1[f]];
        }
        __syncthreads();
    }
    if (indexed) {
        // ---- warp-cooperative sort-join: a warp owns whole root groups of source 0; the lanes
        // walk the index run of each source-0 record 32 products at a time, compact consistent
        // products with a ballot and write consecutive records (coalesced across the warp). ----
        constexpr uint32_t NW = T / 32;
        __shared__ uint32_t sh_wcnt[NW], sh_wpre[NW];
        const uint32_t warp = tid >> 5, lane = tid & 31;
        const uint32_t n0 = src[0].n, n1 = src[1].n, chw = (n0 + NW - 1) / NW;
        const uint32_t wlo = group_start_at_or_after(src[0], min(n0, warp * chw));
        const uint32_t whi = group_start_at_or_after(src[0], min(n0, (warp + 1) * chw));
        const JoinPlan& jp = sh_plan;
        // run table: for join value x, its run of source-1 records in the sorted index is
        // [run[x] & 0xFFFF, +run[x] >> 16) -- an O(1) lookup instead of two binary searches
        const uint32_t U = a.id_base ? (uint32_t)(a.id_base[l + 1] - a.id_base[l]) : 0u;
        const bool use_run = U > 0 && U <= a.run_cap && n1 <= 0xFFFF;
        if (use_run) {
            for (uint32_t x = tid; x < U; x += T) jrun[x] = 0;
            __syncthreads();
            for (uint32_t q = tid; q < n1; q += T) {
                const uint32_t x = (uint32_t)(key_at(q) >> 32);
                if (q == 0 || (uint32_t)(key_at(q - 1) >> 32) != x) {
                    uint32_t e = q + 1;
                    while (e < n1 && (uint32_t)(key_at(e) >> 32) == x) e++;
                    jrun[x] = q | ((e - q) << 16);
                }
            }
            __syncthreads();
        }
        // source-0 root-group starts as a bitmask (bit i: record i starts a group), built once
        constexpr uint32_t GB_WORDS = 1024;
        __shared__ uint32_t sh_gbits[GB_WORDS];
        const bool gtab = n0 <= 32 * GB_WORDS;
        if (gtab) {
            for (uint32_t i0 = warp * 32; i0 < n0; i0 += T) {
                const uint32_t i = i0 + lane;
                const bool st = i < n0 && (i == 0 || w0[(uint64_t)i * W0] != w0[(uint64_t)(i - 1) * W0]);
                const uint32_t m = __ballot_sync(0xffffffffu, st);
                if (lane == 0) sh_gbits[i0 >> 5] = m;
            }
            __syncthreads();
        }
        auto gend = [&](uint32_t g) -> uint32_t {
            if (!gtab) return group_end_warp(src[0], g, lane);
            uint32_t j = g + 1;
            while (j < n0) {
                const uint32_t bits = sh_gbits[j >> 5] & (0xFFFFFFFFu << (j & 31));
                if (bits) return min(n0, (j & ~31u) + __ffs(bits) - 1);
                j = (j & ~31u) + 32;
            }
            return n0;
        };
        // a root group of several source-0 records yields one sorted run of products per record;
        // the runs are merged warp-parallel: each record's final rank = its index in its run +
        // (records below it in every other run, by binary search), scattered through SMEM
        constexpr uint32_t GS_RUNS = 32;
        __shared__ uint32_t sh_runs[NW][GS_RUNS + 1];
        auto walk = [&](uint32_t* out) -> uint32_t {   // out == nullptr: count only
            uint32_t n = 0;
            for (uint32_t g = wlo; g < whi;) {
                const uint32_t ge = gend(g);
                const uint32_t gstart = n;
                for (uint32_t i = g; i < ge; i++) {
                    if (out && i - g < GS_RUNS && lane == 0) sh_runs[warp][i - g] = n - gstart;
                    // the source-0 record is read with warp-uniform loads (one broadcast each)
                    const uint32_t* m1s = w0 + (uint64_t)i * W0;
                    const uint32_t x = m1s[1 + v0];
                    uint32_t p0, p1;
                    if (use_run) {
                        const uint32_t rr = x < U ? jrun[x] : 0u;
                        p0 = rr & 0xFFFFu;
                        p1 = p0 + (rr >> 16);
                    } else {
                        p0 = lower_bound_key(keys, n1, (unsigned long long)x << 32);
                        p1 = lower_bound_key(keys, n1, ((unsigned long long)x + 1ull) << 32);
                    }
                    if (!out && jp.nchk == 0) { n += p1 - p0; continue; }   // every product is consistent
                    if (staged) {
                        switch (W) {
                            case 5: n = staged_products<5>(jp, s1, m1s, p0, p1, lane, out, n); break;
                            case 8: n = staged_products<8>(jp, s1, m1s, p0, p1, lane, out, n); break;
                            default: n = staged_products<0>(jp, s1, m1s, p0, p1, lane, out, n); break;
                        }
                        continue;
                    }
                    for (uint32_t base = p0; base < p1; base += 32) {
                        const uint32_t p = base + lane;
                        bool ok = p < p1;
                        const uint32_t* m2 = ok ? w1 + (uint64_t)(uint32_t)key_at(p) * W1 : w1;
                        for (uint32_t c = 0; c < jp.nchk && ok; c++) ok = m1s[jp.c0[c]] == m2[jp.c1[c]];
                        const uint32_t mask = __ballot_sync(0xffffffffu, ok);
                        if (out && ok) {
                            uint32_t* o = out + (uint64_t)(n + __popc(mask & ((1u << lane) - 1u))) * W;
                            for (uint32_t w = 0; w < W; w++) o[w] = jp.src[w] ? m2[jp.idx[w]] : m1s[jp.idx[w]];
                        }
                        n += __popc(mask);
                    }
                }
                if (out && ge - g > 1) {   // several source-0 records share the root: order the group
                    __syncwarp();
                    const uint32_t k = ge - g, cnt = n - gstart;
                    if (k <= GS_RUNS && cnt * W <= JOIN_GSORT_WORDS) {
                        if (lane == 0) sh_runs[warp][k] = cnt;
                        __syncwarp();
                        merge_group(out + (uint64_t)gstart * W, k, cnt, W, sh_runs[warp],
                                    a.gsort + (((uint64_t)r * L + l) * NW + warp) * JOIN_GSORT_WORDS, lane);
                    } else {
                        if (lane == 0) sort_unique(out + (uint64_t)gstart * W, cnt, W);
                        __syncwarp();
                    }
                }
                g = ge;
            }
            return n;
        };
        const uint32_t wc = walk(nullptr);
        if (lane == 0) sh_wcnt[warp] = wc;
        __syncthreads();
        if (tid == 0) {
            uint32_t acc = 0;
            for (uint32_t w = 0; w < NW; w++) { sh_wpre[w] = acc; acc += sh_wcnt[w]; }
            unsigned long long base = atomicAdd(&a.tops[1], (unsigned long long)acc * W);
            if (base + (unsigned long long)acc * W > a.out_cap) { atomicOr(a.overflow, 2u); base = ~0ull; }
            sh_base = base;
            a.count[(uint64_t)r * L + l] = acc;
            a.off[(uint64_t)r * L + l] = base == ~0ull ? 0 : base;
        }
        __syncthreads();
        if (sh_base != ~0ull) walk(a.out + sh_base + (uint64_t)sh_wpre[warp] * W);
        return;
    }
    auto count_only = [](const uint32_t*) {};
    uint32_t cnt = 0;
    for (uint32_t g = g_lo; g < g_hi;) {
        const uint32_t ge = group_end(src[0], g);
        for_blocks(src, S, g, ge, [&](const uint32_t* lo, const uint32_t* hi) {
            cnt += block_products(src, S, lo, hi, NV, NQ, count_only);
        });
        g = ge;
    }
    uint32_t tot;
    const uint32_t pre = block_exscan(cnt, sh_scan, &tot);
    if (tid == 0) {
        unsigned long long base = atomicAdd(&a.tops[1], (unsigned long long)tot * W);
        if (base + (unsigned long long)tot * W > a.out_cap) { atomicOr(a.overflow, 2u); base = ~0ull; }
        sh_base = base;
        a.count[(uint64_t)r * L + l] = tot;
        a.off[(uint64_t)r * L + l] = base == ~0ull ? 0 : base;
    }
    __syncthreads();
    if (sh_base == ~0ull) return;
    uint32_t* out = a.out + sh_base + (uint64_t)pre * W;
    uint32_t cur = 0;
    for (uint32_t g = g_lo; g < g_hi;) {
        const uint32_t ge = group_end(src[0], g);
        for_blocks(src, S, g, ge, [&](const uint32_t* lo, const uint32_t* hi) {
            const uint32_t start = cur;
            block_products(src, S, lo, hi, NV, NQ, [&](const uint32_t* rr) {
                for (uint32_t w = 0; w < W; w++) out[(uint64_t)cur * W + w] = rr[w];
                cur++;
            });
            // products of one block share the roots prefix; distinct pairs give distinct keys
            sort_unique(out + (uint64_t)start * W, cur - start, W);
        });
        g = ge;
    }
}

template __global__ void k_ematch<128>(Dev, MArgs);
template __global__ void k_join<128>(uint32_t, JArgs);
template __global__ void k_join_big<128>(uint32_t, JArgs);

}  // namespace esat

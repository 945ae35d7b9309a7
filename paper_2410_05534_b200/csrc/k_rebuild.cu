// K4-K6: batched e-graph rebuild (congruence closure) + regroup into the clean class view.
//
// Reference semantics (egraph.py:203-238): each pass scans the hashcons in insertion order,
// canonicalises every key with the *live* union-find, keeps the first entry per key, and
// unions on a class conflict immediately (so later keys in the same pass see the union).
// Passes repeat until one performs no union. Then _regroup builds classes; iteration order
// of nodes is node_sort_key (egraph.py:65-70).
//
// Device schedule ("first-conflict rounds"), one CTA per leaf:
//   round: (A) keys + class finds for positions >= p0 under the current UF, in parallel;
//          (A2) look up the committed table Tc, else insert into the speculative table Ts
//               keeping the minimum position per key (atomicMin);
//          (B) first occurrence per position; conflict = first occurrence in a different
//              class; p* = min conflict (atomicMin in smem);
//          (C) commit [p0, p*) first occurrences into Tc; one thread performs the exact
//              rank union for p*, Ts is cleared and the next round resumes at p*+1.
//   No conflict => pass done; compact committed entries (block scans) into the new hashcons.
// This reproduces the sequential scan exactly: positions before the first conflict see the
// same UF state the reference saw, and the union is replayed in reference order.
//
// Regroup: per-id histogram -> ascending class ids (block scan) -> scatter -> per-class
// insertion sort by (sym rank, children...) -> clean CSR with children as class positions.
#include "esat_internal.cuh"

namespace esat {

namespace {

struct PassIn {
    const uint32_t *sym, *koff, *kids, *cid;
    const double* cost;
};

__device__ __forceinline__ bool key_eq(const uint32_t* ksym, const uint32_t* kkids, const uint32_t* koff,
                                       uint32_t e, uint32_t i) {
    if (ksym[e] != ksym[i]) return false;
    uint32_t ae = koff[e + 1] - koff[e], ai = koff[i + 1] - koff[i];
    if (ae != ai) return false;
    const uint32_t *ke = kkids + koff[e], *ki = kkids + koff[i];
    for (uint32_t j = 0; j < ai; j++)
        if (ke[j] != ki[j]) return false;
    return true;
}

// node order: (rank(name, repr(payload)), children lexicographic, shorter prefix first)
__device__ __forceinline__ bool node_less(const uint32_t* rank, const uint32_t* sym, const uint32_t* koff,
                                          const uint32_t* kids, uint32_t a, uint32_t b) {
    uint32_t ra = rank[sym[a]], rb = rank[sym[b]];
    if (ra != rb) return ra < rb;
    uint32_t na = koff[a + 1] - koff[a], nb = koff[b + 1] - koff[b];
    const uint32_t *ka = kids + koff[a], *kb = kids + koff[b];
    uint32_t m = na < nb ? na : nb;
    for (uint32_t i = 0; i < m; i++)
        if (ka[i] != kb[i]) return ka[i] < kb[i];
    return na < nb;
}

}  // namespace

template <int T>
__global__ void __launch_bounds__(T) k_rebuild(Dev d) {
    const uint32_t l = blockIdx.x;
    const uint32_t tid = threadIdx.x;
    const uint64_t b = d.nb[l], k0 = d.kb[l], u0 = d.ub[l], t0 = d.tb[l];
    const uint32_t n0 = d.n_cnt ? d.n_cnt[l] : (uint32_t)(d.nb[l + 1] - b);
    const uint32_t U = d.n_cnt ? d.u_cnt[l] : (uint32_t)(d.ub[l + 1] - u0);
    const uint32_t tsz = (uint32_t)(d.tb[l + 1] - t0), tmask = tsz - 1;
    uint32_t* parent = d.uf_parent + u0;
    uint8_t* rank = d.uf_rank + u0;

    uint32_t *ksym = d.s_ksym + b, *kkids = d.s_kkids + k0, *cval = d.s_cval + b, *val = d.s_val + b,
             *first = d.s_first + b;
    uint8_t* flag = d.s_flag + b;
    uint32_t *tc = d.s_tc + t0, *ts = d.s_ts + t0;
    uint32_t *osym = d.o_sym + b, *okoff = d.o_koff + b + l, *okids = d.o_kids + k0, *ocid = d.o_cid + b;
    double* ocost = d.o_cost + b;

    __shared__ uint32_t sh_scan[33];
    __shared__ uint32_t sh_pstar, sh_merges, sh_merged;

    PassIn in{d.hc_sym + b, d.hc_koff + b + l, d.hc_kids + k0, d.hc_cid + b, d.hc_cost + b};
    uint32_t n = n0;
    if (tid == 0) { sh_merges = 0; if (d.u_reb) d.u_reb[l] = U; }
    // the working union-find starts as a copy of the leaf's input (snapshot semantics)
    for (uint32_t x = tid; x < U; x += T) { parent[x] = d.uf_parent_in[u0 + x]; rank[x] = d.uf_rank_in[u0 + x]; }
    __syncthreads();

    for (;;) {  // ---------------- pass (egraph.py:206-225) ----------------
        for (uint32_t s = tid; s < tsz; s += T) { tc[s] = NONE; ts[s] = NONE; }
        if (tid == 0) sh_merged = 0;
        __syncthreads();
        uint32_t p0 = 0;
        for (;;) {  // ------------ round ------------
            // (A) canonical keys and classes under the current union-find
            for (uint32_t i = p0 + tid; i < n; i += T) {
                const uint32_t ko = in.koff[i], a = in.koff[i + 1] - ko;
                ksym[i] = in.sym[i];
                for (uint32_t j = 0; j < a; j++) kkids[ko + j] = uf_find(parent, in.kids[ko + j]);
                cval[i] = uf_find(parent, in.cid[i]);
            }
            if (tid == 0) sh_pstar = n;
            __syncthreads();
            // (A2) committed lookup, else speculative min-position insert
            for (uint32_t i = p0 + tid; i < n; i += T) {
                const uint32_t ko = in.koff[i], a = in.koff[i + 1] - ko;
                const uint32_t h = key_hash(ksym[i], kkids + ko, a);
                uint32_t s = h & tmask, f = NONE;
                for (;; s = (s + 1) & tmask) {
                    uint32_t e = tc[s];
                    if (e == NONE) break;
                    if (key_eq(ksym, kkids, in.koff, e, i)) { f = e; break; }
                }
                first[i] = f;
                if (f != NONE) continue;
                for (s = h & tmask;; s = (s + 1) & tmask) {
                    uint32_t e = ts[s];
                    if (e == NONE) {
                        e = atomicCAS(&ts[s], NONE, i);
                        if (e == NONE) break;
                    }
                    if (key_eq(ksym, kkids, in.koff, e, i)) { atomicMin(&ts[s], i); break; }
                }
            }
            __syncthreads();
            // (B) first occurrences and conflicts
            for (uint32_t i = p0 + tid; i < n; i += T) {
                uint32_t f = first[i];
                if (f == NONE) {
                    const uint32_t ko = in.koff[i], a = in.koff[i + 1] - ko;
                    const uint32_t h = key_hash(ksym[i], kkids + ko, a);
                    for (uint32_t s = h & tmask;; s = (s + 1) & tmask) {
                        uint32_t e = ts[s];
                        if (key_eq(ksym, kkids, in.koff, e, i)) { f = e; break; }
                    }
                    first[i] = f;
                }
                if (f != i) {
                    uint32_t v = f < p0 ? uf_find(parent, val[f]) : cval[f];
                    if (v != cval[i]) atomicMin(&sh_pstar, i);
                }
            }
            __syncthreads();
            const uint32_t pstar = sh_pstar;
            // (C) commit first occurrences in [p0, p*)
            for (uint32_t i = p0 + tid; i < pstar; i += T) {
                if (first[i] == i) {
                    const uint32_t ko = in.koff[i], a = in.koff[i + 1] - ko;
                    const uint32_t h = key_hash(ksym[i], kkids + ko, a);
                    for (uint32_t s = h & tmask;; s = (s + 1) & tmask)
                        if (atomicCAS(&tc[s], NONE, i) == NONE) break;
                    val[i] = cval[i];
                    flag[i] = 1;
                } else {
                    flag[i] = 0;
                }
            }
            __syncthreads();
            if (pstar >= n) break;
            if (tid == 0) {  // exact replay of the reference union (egraph.py:216-221)
                const uint32_t f = first[pstar];
                val[f] = uf_union(parent, rank, uf_find(parent, val[f]), cval[pstar]);
                flag[pstar] = 0;
                sh_merges++;
                sh_merged = 1;
            }
            for (uint32_t s = tid; s < tsz; s += T) ts[s] = NONE;
            p0 = pstar + 1;
            __syncthreads();
        }
        // compaction: hashcons = {key: find(val)} in first-occurrence order (egraph.py:222)
        uint32_t base_e = 0, base_k = 0;
        for (uint32_t c0 = 0; c0 < n; c0 += T) {
            const uint32_t i = c0 + tid;
            const uint32_t f = (i < n) ? flag[i] : 0u;
            const uint32_t a = f ? in.koff[i + 1] - in.koff[i] : 0u;
            uint32_t te, tk;
            const uint32_t pe = block_exscan(f, sh_scan, &te);
            const uint32_t pk = block_exscan(a, sh_scan, &tk);
            if (f) {
                const uint32_t e = base_e + pe, ko = in.koff[i];
                osym[e] = ksym[i];
                okoff[e] = base_k + pk;
                for (uint32_t j = 0; j < a; j++) okids[base_k + pk + j] = kkids[ko + j];
                ocid[e] = uf_find(parent, val[i]);
                ocost[e] = in.cost[i];
            }
            base_e += te;
            base_k += tk;
        }
        if (tid == 0) okoff[base_e] = base_k;
        n = base_e;
        __syncthreads();
        if (!sh_merged) break;
        // another pass over the compacted hashcons: stage it as the next pass's input
        uint32_t *sym2 = d.s_sym2 + b, *koff2 = d.s_koff2 + b + l, *kids2 = d.s_kids2 + k0, *cid2 = d.s_cid2 + b;
        double* cost2 = d.s_cost2 + b;
        for (uint32_t i = tid; i < n; i += T) {
            sym2[i] = osym[i]; cid2[i] = ocid[i]; cost2[i] = ocost[i]; koff2[i] = okoff[i];
        }
        if (tid == 0) koff2[n] = okoff[n];
        for (uint32_t q = tid; q < base_k; q += T) kids2[q] = okids[q];
        in = PassIn{sym2, koff2, kids2, cid2, cost2};
        __syncthreads();
    }

    // ---------------- regroup into the clean view (egraph.py:228-238) ----------------
    uint32_t *cnt = d.s_cnt + u0, *pos_of = d.s_pos + u0, *coff_of = d.s_coff + u0, *perm = d.s_perm + b;
    uint32_t *cls_id = d.cls_id + b, *cls_off = d.cls_off + b + l;
    for (uint32_t x = tid; x < U; x += T) cnt[x] = 0;
    __syncthreads();
    for (uint32_t j = tid; j < n; j += T) atomicAdd(&cnt[ocid[j]], 1u);
    __syncthreads();
    uint32_t base_c = 0, base_n = 0;
    for (uint32_t c0 = 0; c0 < U; c0 += T) {
        const uint32_t x = c0 + tid;
        const uint32_t c = x < U ? cnt[x] : 0u, f = c ? 1u : 0u;
        uint32_t tc_, tn_;
        const uint32_t pc = block_exscan(f, sh_scan, &tc_);
        const uint32_t pn = block_exscan(c, sh_scan, &tn_);
        if (x < U) {
            if (f) {
                const uint32_t p = base_c + pc;
                pos_of[x] = p;
                cls_id[p] = x;
                cls_off[p] = base_n + pn;
                coff_of[x] = base_n + pn;
            } else {
                pos_of[x] = NONE;
            }
        }
        base_c += tc_;
        base_n += tn_;
    }
    const uint32_t C = base_c;
    if (tid == 0) cls_off[C] = n;
    __syncthreads();
    // node_sort_key as a packed key per entry: hi = rank << 32 | (child0 + 1), lo = child1 + 1
    // (0 = absent, so shorter prefixes sort first); more than two children -> the full comparator
    constexpr uint32_t WIDE = 0xFFFFFFFFu;
    uint32_t *key_r = d.s_ksym + b, *key_c0 = d.s_cval + b, *key_c1 = d.s_val + b;
    for (uint32_t j = tid; j < n; j += T) {
        perm[atomicAdd(&coff_of[ocid[j]], 1u)] = j;
        const uint32_t q = okoff[j], a = okoff[j + 1] - q;
        key_r[j] = d.sym_rank[osym[j]];
        key_c0[j] = a > 0 ? okids[q] + 1 : 0u;
        key_c1[j] = a > 2 ? WIDE : (a > 1 ? okids[q + 1] + 1 : 0u);
    }
    __syncthreads();
    for (uint32_t k = tid; k < C; k += T) {  // per-class insertion sort (classes are small)
        const uint32_t lo = cls_off[k], hi = cls_off[k + 1];
        for (uint32_t i = lo + 1; i < hi; i++) {
            const uint32_t v = perm[i];
            const unsigned long long hv = ((unsigned long long)key_r[v] << 32) | key_c0[v];
            const uint32_t lv = key_c1[v];
            uint32_t j = i;
            while (j > lo) {
                const uint32_t u = perm[j - 1];
                const unsigned long long hu = ((unsigned long long)key_r[u] << 32) | key_c0[u];
                bool lt;
                if (hv != hu) lt = hv < hu;
                else if (lv == WIDE || key_c1[u] == WIDE) lt = node_less(d.sym_rank, osym, okoff, okids, v, u);
                else lt = lv < key_c1[u];
                if (!lt) break;
                perm[j] = u;
                j--;
            }
            perm[j] = v;
        }
    }
    __syncthreads();
    uint32_t *nsym = d.nd_sym + b, *nkoff = d.nd_koff + b + l, *nkpos = d.nd_kpos + k0, *nhc = d.nd_hc + b;
    double* ncost = d.nd_cost + b;
    uint32_t base_k = 0;
    for (uint32_t c0 = 0; c0 < n; c0 += T) {
        const uint32_t j = c0 + tid;
        const uint32_t e = j < n ? perm[j] : 0u;
        const uint32_t a = j < n ? okoff[e + 1] - okoff[e] : 0u;
        uint32_t tk;
        const uint32_t pk = block_exscan(a, sh_scan, &tk);
        if (j < n) {
            nsym[j] = osym[e];
            ncost[j] = ocost[e];
            nhc[j] = e;
            nkoff[j] = base_k + pk;
            for (uint32_t q = 0; q < a; q++) nkpos[base_k + pk + q] = pos_of[okids[okoff[e] + q]];
        }
        base_k += tk;
    }
    if (tid == 0) {
        nkoff[n] = base_k;
        d.o_n[l] = n;
        d.o_merges[l] = sh_merges;
        d.v_C[l] = C;
        const uint32_t r = d.root[l];
        d.v_root[l] = r == NONE ? NONE : pos_of[uf_find(parent, r)];
    }
}

template __global__ void k_rebuild<256>(Dev);

}  // namespace esat

// K7-K10: batched greedy extraction -- default cost and the paper's constituent-cost (OCF)
// node cost -- over clean leaf views, one CTA per leaf.
//
// Reference (extraction.py:121-242): passes over classes in ascending canonical id
// (Gauss-Seidel: a class reads this pass's cost of lower classes and last pass's cost of
// the others), nodes in node_sort_key order, first strict minimum wins, class updated only
// on strict improvement, stop after a pass without change (cap 4C+8). OCF (Alg. 2,
// PAPER.md:310-362) threads a ConstituentHistory: each class flushes the history of its
// first strict-min node of the pass; a child's history read by class k is this pass's flush
// for children at lower positions and last pass's flush otherwise (none in pass 0); with a
// single class no flush ever happens.
//
// Device schedule: level(k) = 1 + max level of k's lower-position
// children, so all classes of one level are independent within a pass; a pass is one sweep
// of levels separated by CTA barriers, reading cost_cur for lower positions and the pass-
// start snapshot cost_prev otherwise. Histories are sorted (class position, f64) arrays in a
// per-leaf pool, double-buffered by pass parity; each class materialises only the history
// of its winning node, sized exactly by a read-only cost walk first.
#include "esat_internal.cuh"

namespace esat {

namespace {

struct Hist {
    const uint32_t* key;
    const double* val;
    uint32_t n;
    bool present;
};

__device__ __forceinline__ bool hist_has(const Hist& h, uint32_t key) {
    int lo = 0, hi = (int)h.n - 1;
    while (lo <= hi) {
        int mid = (lo + hi) >> 1;
        uint32_t k = h.key[mid];
        if (k == key) return true;
        if (k < key) lo = mid + 1; else hi = mid - 1;
    }
    return false;
}

__device__ __forceinline__ int hist_find(const uint32_t* key, uint32_t n, uint32_t x) {
    int lo = 0, hi = (int)n - 1;
    while (lo <= hi) {
        int mid = (lo + hi) >> 1;
        uint32_t k = key[mid];
        if (k == x) return mid;
        if (k < x) lo = mid + 1; else hi = mid - 1;
    }
    return -1;
}

struct LeafCtx {
    uint32_t C, k;             // class count, class being evaluated
    int pass;
    const uint32_t *nko, *kpos;
    const double *ncost, *cost, *prev;
    const uint32_t *pk[2];     // pool keys per parity (leaf base applied)
    const double *pv[2];
    const uint32_t *hoff[2], *hlen[2];
};

__device__ __forceinline__ double child_cost(const LeafCtx& c, uint32_t j) {
    return j < c.k ? c.cost[j] : c.prev[j];
}

__device__ __forceinline__ Hist child_hist(const LeafCtx& c, uint32_t j) {
    Hist h{nullptr, nullptr, 0u, false};
    if (c.C == 1) return h;                       // no flush ever happens with one class
    int par;
    if (j < c.k) par = c.pass & 1;                // flushed earlier in this pass
    else if (c.pass == 0) return h;               // not flushed yet
    else par = (c.pass - 1) & 1;                  // last pass's flush
    uint32_t off = c.hoff[par][j];
    h.key = c.pk[par] + off;
    h.val = c.pv[par] + off;
    h.n = c.hlen[par][j];
    h.present = true;
    return h;
}

// Read-only OCF walk for arity <= 2 (extraction.py:205-221): cost and exact history size.
__device__ __forceinline__ double ocf_walk2(const LeafCtx& c, uint32_t nd, uint32_t* size_out,
                                             double* cc1_out, double* cc2_out, bool* skip2_out) {
    const uint32_t q0 = c.nko[nd], a = c.nko[nd + 1] - q0;
    double v = c.ncost[nd];
    uint32_t size = 0;
    *skip2_out = true;
    if (a == 0) { *size_out = 0; return v; }
    const uint32_t c1 = c.kpos[q0];
    const Hist h1 = child_hist(c, c1);
    // case 2 with an empty running history: max_cost = 0 (case 3 when no history)
    const double cc1 = h1.present ? pymax(child_cost(c, c1) - 0.0, 0.0) : child_cost(c, c1);
    v = v + cc1;
    const bool c1_in_h1 = h1.present && hist_has(h1, c1);
    size = h1.n + (c1_in_h1 ? 0u : 1u);
    *cc1_out = cc1;
    if (a == 2) {
        const uint32_t c2 = c.kpos[q0 + 1];
        const bool skip = (c2 == c1) || (h1.present && hist_has(h1, c2));   // case 1
        *skip2_out = skip;
        if (!skip) {
            const Hist h2 = child_hist(c, c2);
            double cc2;
            if (h2.present) {
                double m = 0.0;
                uint32_t ov = 0, i = 0, j = 0;
                while (i < h1.n && j < h2.n) {        // overlap with h1
                    const uint32_t a1 = h1.key[i], a2 = h2.key[j];
                    if (a1 == a2) { m = pymax(m, h2.val[j]); ov++; i++; j++; }
                    else if (a1 < a2) i++;
                    else j++;
                }
                if (!c1_in_h1) {                      // key c1 of the running history
                    const int at = hist_find(h2.key, h2.n, c1);
                    if (at >= 0) { m = pymax(m, h2.val[at]); ov++; }
                }
                cc2 = pymax(child_cost(c, c2) - m, 0.0);
                size += h2.n - ov + (hist_has(h2, c2) ? 0u : 1u);
            } else {
                cc2 = child_cost(c, c2);
                size += 1;
            }
            *cc2_out = cc2;
            v = v + cc2;
        }
    }
    *size_out = size;
    return v;
}

// Materialise the history of an arity <= 2 node into dst (sorted by key).
__device__ void ocf_write2(const LeafCtx& c, uint32_t nd, double cc1, double cc2, bool skip2,
                           uint32_t* dk, double* dv) {
    const uint32_t q0 = c.nko[nd], a = c.nko[nd + 1] - q0;
    if (a == 0) return;
    const uint32_t c1 = c.kpos[q0];
    const Hist h1 = child_hist(c, c1);
    Hist h2{nullptr, nullptr, 0u, false};
    uint32_t c2 = NONE;
    if (a == 2 && !skip2) { c2 = c.kpos[q0 + 1]; h2 = child_hist(c, c2); }
    // union of keys {h1, h2, c1, c2}; value: c1 -> cc1, c2 -> cc2, h1 wins over h2
    uint32_t i = 0, j = 0, o = 0;
    bool d1 = false, d2 = (c2 == NONE);
    for (;;) {
        uint32_t k1 = i < h1.n ? h1.key[i] : NONE;
        uint32_t k2 = j < h2.n ? h2.key[j] : NONE;
        uint32_t ks = d1 ? NONE : c1;
        uint32_t kt = d2 ? NONE : c2;
        uint32_t m = k1;
        if (k2 < m) m = k2;
        if (ks < m) m = ks;
        if (kt < m) m = kt;
        if (m == NONE) break;
        double vv;
        if (m == c1) vv = cc1;
        else if (m == c2) vv = cc2;
        else if (m == k1) vv = h1.val[i];
        else vv = h2.val[j];
        if (m == k1) i++;
        if (m == k2) j++;
        if (m == ks) d1 = true;
        if (m == kt) d2 = true;
        dk[o] = m;
        dv[o] = vv;
        o++;
    }
}

// Generic-arity OCF node (n-ary sink): builds the running history in the pool (current
// parity) child by child, exactly as Alg. 2 mutates enode_hist. Returns the node cost;
// the final history is at (*off_out, *n_out).
__device__ double ocf_generic(const LeafCtx& c, uint32_t nd, uint32_t* top, uint64_t pcap, uint32_t* pk,
                              double* pv, uint32_t* off_out, uint32_t* n_out, uint32_t* over) {
    const uint32_t q0 = c.nko[nd], a = c.nko[nd + 1] - q0;
    double v = c.ncost[nd];
    uint32_t hoff = 0, hn = 0;
    for (uint32_t t = 0; t < a; t++) {
        const uint32_t ck = c.kpos[q0 + t];
        if (hn && hist_find(pk + hoff, hn, ck) >= 0) continue;       // case 1
        const Hist h = child_hist(c, ck);
        double m = 0.0;
        if (h.present) {                                             // overlap max (case 2)
            uint32_t i = 0, j = 0;
            while (i < hn && j < h.n) {
                const uint32_t a1 = pk[hoff + i], a2 = h.key[j];
                if (a1 == a2) { m = pymax(m, h.val[j]); i++; j++; }
                else if (a1 < a2) i++;
                else j++;
            }
        }
        const double cc = h.present ? pymax(child_cost(c, ck) - m, 0.0) : child_cost(c, ck);
        const uint32_t need = hn + h.n + 1;
        const uint32_t noff = atomicAdd(top, need);
        if ((uint64_t)noff + need > pcap) { *over = 1; *off_out = 0; *n_out = 0; return v + cc; }
        uint32_t i = 0, j = 0, o = 0;
        bool dc = false;
        for (;;) {                                                   // keys {H, h, ck}; H wins, ck -> cc
            const uint32_t k1 = i < hn ? pk[hoff + i] : NONE;
            const uint32_t k2 = j < h.n ? h.key[j] : NONE;
            const uint32_t k3 = dc ? NONE : ck;
            uint32_t mk = k1 < k2 ? k1 : k2;
            mk = k3 < mk ? k3 : mk;
            if (mk == NONE) break;
            double vv = (mk == k3) ? cc : (mk == k1 ? pv[hoff + i] : h.val[j]);
            if (mk == k1) i++;
            if (mk == k2) j++;
            if (mk == k3) dc = true;
            pk[noff + o] = mk;
            pv[noff + o] = vv;
            o++;
        }
        hoff = noff;
        hn = o;
        v = v + cc;
    }
    *off_out = hoff;
    *n_out = hn;
    return v;
}

}  // namespace

template <int T>
__global__ void __launch_bounds__(T) k_extract(Dev d, XArgs x) {
    const uint32_t l = blockIdx.x, tid = threadIdx.x;
    const uint64_t b = d.nb[l], k0 = d.kb[l];
    const uint32_t C = d.v_C[l];
    const uint32_t* coff = d.cls_off + b + l;
    LeafCtx c;
    c.C = C;
    c.nko = d.nd_koff + b + l;
    c.kpos = d.nd_kpos + k0;
    c.ncost = d.nd_cost + b;
    double* cost = x.class_cost + b;
    double* prev = x.prev + b;
    c.cost = cost;
    c.prev = prev;
    uint32_t* ch = x.choice + b;
    uint32_t* level = x.level + b;
    uint32_t* order = x.order + b;
    uint32_t* lvcnt = x.lvcnt + b + l;   // C+1 entries
    const bool ocf = x.method == 1;
    uint64_t pb = 0, pcap = 0;
    uint32_t* hoffw[2] = {nullptr, nullptr};
    uint32_t* hlenw[2] = {nullptr, nullptr};
    uint32_t* pkw[2] = {nullptr, nullptr};
    double* pvw[2] = {nullptr, nullptr};
    if (ocf) {
        pb = x.pool_base[l];
        pcap = x.pool_base[l + 1] - pb;
        for (int p = 0; p < 2; p++) {
            pkw[p] = x.pool_key + p * x.pool_stride + pb;
            pvw[p] = x.pool_val + p * x.pool_stride + pb;
            hoffw[p] = x.hoff + p * x.slot_stride + b;
            hlenw[p] = x.hlen + p * x.slot_stride + b;
            c.pk[p] = pkw[p]; c.pv[p] = pvw[p]; c.hoff[p] = hoffw[p]; c.hlen[p] = hlenw[p];
        }
    }

    __shared__ uint32_t sh_scan[33];
    __shared__ uint32_t sh_flag, sh_maxlv, sh_top, sh_over;

    for (uint32_t k = tid; k < C; k += T) {
        cost[k] = __longlong_as_double(0x7ff0000000000000ll);
        prev[k] = cost[k];
        ch[k] = NONE;
        level[k] = 0;
        x.reach[b + k] = 0;
    }
    if (tid == 0) sh_over = 0;
    __syncthreads();
    // ---- K7: wavefront levels over lower-position children ----
    // level[k] = 1 + max level of k's lower-position children. Warp 0 walks the classes in
    // position order 32 at a time: children below the chunk are final; dependencies inside the
    // chunk are resolved by re-evaluating the chunk until no lane changes (chain length + 1 rounds).
    __syncthreads();
    if (tid < 32) {
        uint32_t mx = 0;
        for (uint32_t k0 = 0; k0 < C; k0 += 32) {
            const uint32_t k = k0 + tid;
            uint32_t base = 0;
            if (k < C)
                for (uint32_t nd = coff[k]; nd < coff[k + 1]; nd++)
                    for (uint32_t q = c.nko[nd]; q < c.nko[nd + 1]; q++) {
                        const uint32_t j = c.kpos[q];
                        if (j < k0) { const uint32_t t = level[j] + 1; base = t > base ? t : base; }
                    }
            if (k < C) level[k] = base;
            __syncwarp();
            for (;;) {
                uint32_t lv = base;
                if (k < C)
                    for (uint32_t nd = coff[k]; nd < coff[k + 1]; nd++)
                        for (uint32_t q = c.nko[nd]; q < c.nko[nd + 1]; q++) {
                            const uint32_t j = c.kpos[q];
                            if (j >= k0 && j < k) { const uint32_t t = level[j] + 1; lv = t > lv ? t : lv; }
                        }
                const bool upd = k < C && lv != level[k];
                __syncwarp();
                if (upd) level[k] = lv;
                __syncwarp();
                if (!__any_sync(0xffffffffu, upd)) break;
            }
            const uint32_t lk = k < C ? level[k] : 0u;
            mx = max(mx, __reduce_max_sync(0xffffffffu, lk));
        }
        if (tid == 0) sh_maxlv = mx;
    }
    __syncthreads();
    // counting sort of classes by level
    for (uint32_t k = tid; k <= C; k += T) lvcnt[k] = 0;
    __syncthreads();
    for (uint32_t k = tid; k < C; k += T) atomicAdd(&lvcnt[level[k]], 1u);
    __syncthreads();
    const uint32_t nlv = C ? sh_maxlv + 1 : 0;
    uint32_t base = 0;
    for (uint32_t c0 = 0; c0 <= nlv; c0 += T) {
        const uint32_t i = c0 + tid;
        const uint32_t v = i < nlv ? lvcnt[i] : 0u;
        uint32_t tot;
        const uint32_t p = block_exscan(v, sh_scan, &tot);
        if (i <= nlv) lvcnt[i] = base + p;   // exclusive offsets; lvcnt[nlv] = C
        base += tot;
    }
    __syncthreads();
    for (uint32_t k = tid; k < C; k += T) order[atomicAdd(&lvcnt[level[k]], 1u)] = k;
    __syncthreads();
    // lvcnt[lv] now holds the END of level lv; level lv spans [lv ? lvcnt[lv-1] : 0, lvcnt[lv])

    // ---- K8/K9: Gauss-Seidel passes as level sweeps ----
    const uint64_t cap = 4ull * C + 8;
    uint32_t st = X_NOT_CONVERGED, passes = 0;
    for (uint64_t it = 0; it < cap; it++) {
        const int pass = (int)it;
        c.pass = pass;
        for (uint32_t k = tid; k < C; k += T) prev[k] = cost[k];
        if (tid == 0) { sh_flag = 0; if (pass == 0) sh_top = 0; }
        __syncthreads();
        const int par = pass & 1, ppar = par ^ 1;
        uint8_t* chg_cur = x.chg + par * x.slot_stride + b;
        const uint8_t* chg_prv = x.chg + ppar * x.slot_stride + b;
        for (uint32_t lv = 0; lv < nlv; lv++) {
            const uint32_t lo = lv ? lvcnt[lv - 1] : 0u, hi = lvcnt[lv];
            for (uint32_t idx = lo + tid; idx < hi; idx += T) {
                const uint32_t k = order[idx];
                c.k = k;
                // Dirty skip (exact): the class's inputs are its children's (cost, history) as read
                // under the Gauss-Seidel rule; if none changed since the class's last evaluation its
                // outputs are identical, so only the history slot pointer is carried forward.
                bool need = pass == 0;
                for (uint32_t nd = coff[k]; nd < coff[k + 1] && !need; nd++)
                    for (uint32_t q = c.nko[nd]; q < c.nko[nd + 1]; q++) {
                        const uint32_t j = c.kpos[q];
                        if (j < k ? chg_cur[j] : chg_prv[j]) { need = true; break; }
                    }
                if (!need) {
                    chg_cur[k] = 0;
                    if (ocf && C > 1) { hoffw[par][k] = hoffw[ppar][k]; hlenw[par][k] = hlenw[ppar][k]; }
                    continue;
                }
                double bv = __longlong_as_double(0x7ff0000000000000ll);
                uint32_t bn = NONE;
                bool changed = pass == 0;
                if (!ocf) {
                    for (uint32_t nd = coff[k]; nd < coff[k + 1]; nd++) {
                        double v = c.ncost[nd];
                        for (uint32_t q = c.nko[nd]; q < c.nko[nd + 1]; q++) v = v + child_cost(c, c.kpos[q]);
                        if (bn == NONE || v < bv) { bv = v; bn = nd; }
                    }
                } else {
                    // first strict-min node by ocf_enode_cost; its history is flushed for class k
                    double hb = __longlong_as_double(0x7ff0000000000000ll);
                    uint32_t hn = NONE, hsize = 0, hgoff = 0;
                    double h_cc1 = 0, h_cc2 = 0;
                    bool h_skip2 = true, h_gen = false;
                    for (uint32_t nd = coff[k]; nd < coff[k + 1]; nd++) {
                        double v;
                        if (c.nko[nd + 1] - c.nko[nd] <= 2) {
                            uint32_t size;
                            double cc1 = 0, cc2 = 0;
                            bool skip2;
                            v = ocf_walk2(c, nd, &size, &cc1, &cc2, &skip2);
                            if (v < hb) { hb = v; hn = nd; hsize = size; h_cc1 = cc1; h_cc2 = cc2; h_skip2 = skip2; h_gen = false; }
                        } else {
                            uint32_t goff, gn;
                            v = ocf_generic(c, nd, &sh_top, pcap, pkw[0], pvw[0], &goff, &gn, &sh_over);
                            if (v < hb) { hb = v; hn = nd; hsize = gn; hgoff = goff; h_gen = true; }
                        }
                        if (bn == NONE || v < bv) { bv = v; bn = nd; }
                    }
                    if (C > 1) {
                        uint32_t off = 0;
                        if (hn == NONE || hsize == 0) {
                            hsize = 0;
                        } else if (h_gen) {
                            off = hgoff;
                        } else {
                            off = atomicAdd(&sh_top, hsize);
                            if ((uint64_t)off + hsize > pcap) { sh_over = 1; hsize = 0; off = 0; }
                            else ocf_write2(c, hn, h_cc1, h_cc2, h_skip2, pkw[0] + off, pvw[0] + off);
                        }
                        hoffw[par][k] = off;
                        hlenw[par][k] = hsize;
                        if (!changed) {  // did the flushed history change w.r.t. last pass?
                            const uint32_t o2 = hoffw[ppar][k], n2 = hlenw[ppar][k];
                            if (n2 != hsize) changed = true;
                            for (uint32_t i = 0; i < hsize && !changed; i++)
                                changed = pkw[0][off + i] != pkw[0][o2 + i] ||
                                          __double_as_longlong(pvw[0][off + i]) != __double_as_longlong(pvw[0][o2 + i]);
                        }
                    }
                }
                if (bn != NONE && bv < cost[k]) { cost[k] = bv; ch[k] = bn; sh_flag = 1; changed = true; }
                chg_cur[k] = changed ? 1 : 0;
            }
            __syncthreads();
        }
        passes++;
        const bool any_change = sh_flag != 0;
        __syncthreads();   // everyone has read the flag before thread 0 resets it for the next pass
        if (!any_change) { st = X_OK; break; }
    }
    if (sh_over) st = X_CAPACITY;

    // ---- K10: root check, validation DFS and reachable set (extraction.py:67-115, 149-153) ----
    if (tid == 0) {
        const uint32_t root = d.v_root[l];
        uint32_t err = NONE;
        double rc = __longlong_as_double(0x7ff8000000000000ll);
        if (st == X_OK && root == NONE) st = X_NO_ROOT;
        if (st == X_OK && !(cost[root] < __longlong_as_double(0x7ff0000000000000ll))) st = X_INFEASIBLE;
        if (st == X_OK) {
            rc = cost[root];
            uint8_t* state = x.reach + b;   // 0 unvisited, 1 on stack, 2 done
            uint32_t *vs = x.stk + b, *vi = x.stki + b;
            uint32_t dpt = 1;
            vs[0] = root; vi[0] = 0; state[root] = 1;
            while (dpt) {
                const uint32_t cc = vs[dpt - 1], nd = ch[cc];
                const uint32_t q0 = c.nko[nd], a = c.nko[nd + 1] - q0;
                if (vi[dpt - 1] == a) { state[cc] = 2; dpt--; continue; }
                const uint32_t kid = c.kpos[q0 + vi[dpt - 1]];
                vi[dpt - 1]++;
                if (state[kid] == 2) continue;
                if (state[kid] == 1) { st = X_CYCLIC; err = d.cls_id[b + kid]; break; }
                if (ch[kid] == NONE) { st = X_CHILD_NOT_CHOSEN; err = d.cls_id[b + kid]; break; }
                state[kid] = 1;
                vs[dpt] = kid; vi[dpt] = 0; dpt++;
            }
            if (st == X_OK)
                for (uint32_t k = 0; k < C; k++) state[k] = state[k] == 2 ? 1 : 0;
        }
        x.status[l] = st;
        x.err_class[l] = err;
        x.root_cost[l] = rc;
        x.passes[l] = passes;
    }
}

template __global__ void k_extract<32>(Dev, XArgs);
template __global__ void k_extract<64>(Dev, XArgs);
template __global__ void k_extract<128>(Dev, XArgs);

}  // namespace esat

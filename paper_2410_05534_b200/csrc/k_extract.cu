// K7-K10: batched greedy extraction -- default cost and the paper's constituent-cost (OCF)
// node cost -- over clean leaf views, one CTA (one warp) per leaf.
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
// of levels separated by barriers, reading cost_cur for lower positions and the pass-start
// snapshot cost_prev otherwise. A class whose inputs did not change since its last evaluation
// is skipped (exact dirty skip).
//
// Constituent histories are stored as a dense bitset over class positions (ceil(C/32) words,
// 16-B aligned) plus the f64 contributions in key order. Alg. 2's dictionary operations become
// word operations: membership is a bit test, the overlap of a child's constituents with the
// node's running history is an AND, the inherited (non-overlapping) constituents an OR, and
// values are located by popcount ranks -- no searching, no data-dependent merge walks. Each
// history block also carries, per bitset word, the Python-max of that word's values (from +0.0):
// an overlap that covers a whole word then costs one load instead of one per key (the max of
// Alg. 2's overlap is order-independent: it only ever moves on a strictly greater value).
//
// History block layout (3*NW words): bits[NW] | wmax[NW] (f64).
#include <cstdio>

#include "esat_internal.cuh"

namespace esat {

namespace {

struct Hist {
    const uint32_t* bits;   // NW words (only when present); words outside [4*lo4, 4*hi4) are zero
    const double* wmax;     // NW per-word value maxima (valid inside the occupied range)
    const double* vals;     // n values in key order
    uint32_t n, lo4, hi4;   // value count, occupied uint4-group range
    bool present;
};

struct LeafCtx {
    uint32_t C, k, NW;         // classes, class being evaluated, bitset words (multiple of 4)
    int pass;
    const uint32_t *nko, *kpos;
    const double *ncost, *cost, *prev;
    const uint32_t* pk;        // bitset pool (leaf base applied)
    const double* pv;          // value pool
    const uint32_t *hoff[2], *hvoff[2], *hlen[2], *hrng[2];
};

__device__ __forceinline__ double child_cost(const LeafCtx& c, uint32_t j) {
    return j < c.k ? c.cost[j] : c.prev[j];
}

__device__ __forceinline__ Hist child_hist(const LeafCtx& c, uint32_t j) {
    Hist h{nullptr, nullptr, nullptr, 0u, 0u, 0u, false};
    if (c.C == 1) return h;                       // no flush ever happens with one class
    int par;
    if (j < c.k) par = c.pass & 1;                // flushed earlier in this pass
    else if (c.pass == 0) return h;               // not flushed yet
    else par = (c.pass - 1) & 1;                  // last pass's flush
    h.bits = c.pk + c.hoff[par][j];
    h.wmax = reinterpret_cast<const double*>(h.bits + c.NW);
    h.vals = c.pv + c.hvoff[par][j];
    h.n = c.hlen[par][j];
    const uint32_t rg = c.hrng[par][j];
    h.lo4 = rg & 0xFFFFu;
    h.hi4 = rg >> 16;
    h.present = true;
    return h;
}

__device__ __forceinline__ bool hbit(const Hist& h, uint32_t key) {
    const uint32_t g = key >> 7;
    return h.present && g >= h.lo4 && g < h.hi4 && ((h.bits[key >> 5] >> (key & 31)) & 1u);
}

__device__ __forceinline__ uint4 hword4(const Hist& h, uint32_t w4) {
    return (h.present && w4 >= h.lo4 && w4 < h.hi4) ? reinterpret_cast<const uint4*>(h.bits)[w4]
                                                    : make_uint4(0, 0, 0, 0);
}

__device__ __forceinline__ uint32_t bit_of(uint32_t key, uint32_t w) {
    return (key >> 5) == w ? (1u << (key & 31)) : 0u;
}

// Read-only OCF walk for arity <= 2 (extraction.py:205-221): node cost and exact history size.
__device__ double ocf_walk2(const LeafCtx& c, uint32_t nd, uint32_t* size_out, double* cc1_out, double* cc2_out,
                            bool* skip2_out) {
    const uint32_t q0 = c.nko[nd], a = c.nko[nd + 1] - q0;
    double v = c.ncost[nd];
    *skip2_out = true;
    if (a == 0) { *size_out = 0; return v; }
    const uint32_t c1 = c.kpos[q0];
    const Hist h1 = child_hist(c, c1);
    // case 2 with an empty running history (max_cost = 0), or case 3 without a history
    const double cc1 = h1.present ? pymax(child_cost(c, c1) - 0.0, 0.0) : child_cost(c, c1);
    v = v + cc1;
    uint32_t size = h1.n + (hbit(h1, c1) ? 0u : 1u);
    *cc1_out = cc1;
    if (a == 2) {
        const uint32_t c2 = c.kpos[q0 + 1];
        const bool skip = (c2 == c1) || hbit(h1, c2);   // case 1: already paid for
        *skip2_out = skip;
        if (!skip) {
            const Hist h2 = child_hist(c, c2);
            double cc2;
            if (h2.present) {
                // case 2: overlap of h2's constituents with the running history H1 = h1 + {c1}
                double m = 0.0;
                uint32_t ov = 0, rank2 = 0;
                const uint4* b2v = reinterpret_cast<const uint4*>(h2.bits);
                for (uint32_t w4 = h2.lo4; w4 < h2.hi4; w4++) {
                    const uint4 q2 = b2v[w4];
                    if (!(q2.x | q2.y | q2.z | q2.w)) continue;
                    const uint4 q1 = hword4(h1, w4);
                    const uint32_t w2[4] = {q2.x, q2.y, q2.z, q2.w}, w1[4] = {q1.x, q1.y, q1.z, q1.w};
#pragma unroll
                    for (int t = 0; t < 4; t++) {
                        const uint32_t w = 4 * w4 + t;
                        uint32_t o = w2[t] & (w1[t] | bit_of(c1, w));
                        const uint32_t pc = __popc(w2[t]);
                        if (o == w2[t]) {   // the whole word overlaps: its stored maximum
                            m = pymax(m, h2.wmax[w]);
                            ov += pc;
                        } else {
                            while (o) {
                                const int bpos = __ffs(o) - 1;
                                m = pymax(m, h2.vals[rank2 + __popc(w2[t] & ((1u << bpos) - 1u))]);
                                ov++;
                                o &= o - 1;
                            }
                        }
                        rank2 += pc;
                    }
                }
                cc2 = pymax(child_cost(c, c2) - m, 0.0);
                size += h2.n - ov + (hbit(h2, c2) ? 0u : 1u);
            } else {
                cc2 = child_cost(c, c2);   // case 3
                size += 1;
            }
            *cc2_out = cc2;
            v = v + cc2;
        }
    }
    *size_out = size;
    return v;
}

// Materialise the history of an arity <= 2 node: bitset at ob (NW words), values at ovals.
// Only the occupied uint4-group range is written; it is returned packed as lo4 | hi4 << 16.
__device__ uint32_t ocf_write2(const LeafCtx& c, uint32_t nd, double cc1, double cc2, bool skip2, uint32_t* ob,
                               double* ovals) {
    const uint32_t q0 = c.nko[nd], a = c.nko[nd + 1] - q0;
    uint4* obv = reinterpret_cast<uint4*>(ob);
    double* owm = reinterpret_cast<double*>(ob + c.NW);
    if (a == 0) return 0u;
    const uint32_t c1 = c.kpos[q0];
    const Hist h1 = child_hist(c, c1);
    Hist h2{nullptr, nullptr, nullptr, 0u, 0u, 0u, false};
    uint32_t c2 = NONE;
    if (a == 2 && !skip2) { c2 = c.kpos[q0 + 1]; h2 = child_hist(c, c2); }
    uint32_t lo = c1 >> 7, hi = (c1 >> 7) + 1;
    if (c2 != NONE) { lo = min(lo, c2 >> 7); hi = max(hi, (c2 >> 7) + 1); }
    if (h1.present && h1.hi4 > h1.lo4) { lo = min(lo, h1.lo4); hi = max(hi, h1.hi4); }
    if (h2.present && h2.hi4 > h2.lo4) { lo = min(lo, h2.lo4); hi = max(hi, h2.hi4); }
    // keys {h1, c1, h2, c2}; values: c1 -> cc1, c2 -> cc2, h1 wins over h2 (first writer)
    const double* v1 = h1.vals;
    const double* v2 = h2.vals;
    uint32_t o = 0, rank1 = 0, rank2 = 0;
    for (uint32_t w4 = lo; w4 < hi; w4++) {
        const uint4 q1 = hword4(h1, w4);
        const uint4 q2 = hword4(h2, w4);
        const uint32_t w1[4] = {q1.x, q1.y, q1.z, q1.w}, w2[4] = {q2.x, q2.y, q2.z, q2.w};
        uint32_t wo[4];
#pragma unroll
        for (int t = 0; t < 4; t++) {
            const uint32_t w = 4 * w4 + t;
            const uint32_t sp = bit_of(c1, w) | (c2 != NONE ? bit_of(c2, w) : 0u);
            uint32_t ow = w1[t] | w2[t] | sp;
            wo[t] = ow;
            if (!sp && !(w1[t] & w2[t]) && (!w1[t] || !w2[t])) {
                // word owned by one source and no special key: contiguous value copy
                const uint32_t n1w = __popc(w1[t]), n2w = __popc(w2[t]);
                const double* src = n1w ? v1 + rank1 : v2 + rank2;
                const uint32_t cnt = n1w ? n1w : n2w;
                for (uint32_t i = 0; i < cnt; i++) ovals[o + i] = src[i];
                owm[w] = n1w ? h1.wmax[w] : (n2w ? h2.wmax[w] : 0.0);
                o += cnt;
                rank1 += n1w;
                rank2 += n2w;
                continue;
            }
            double wm = 0.0;
            while (ow) {
                const int bpos = __ffs(ow) - 1;
                const uint32_t key = 32 * w + bpos, below = (1u << bpos) - 1u;
                double val;
                if (key == c1) val = cc1;
                else if (key == c2) val = cc2;
                else if ((w1[t] >> bpos) & 1u) val = v1[rank1 + __popc(w1[t] & below)];
                else val = v2[rank2 + __popc(w2[t] & below)];
                ovals[o++] = val;
                wm = pymax(wm, val);
                ow &= ow - 1;
            }
            owm[w] = wm;
            rank1 += __popc(w1[t]);
            rank2 += __popc(w2[t]);
        }
        obv[w4] = make_uint4(wo[0], wo[1], wo[2], wo[3]);
    }
    return lo | (hi << 16);
}

// Generic-arity OCF node (n-ary sink): the running history is rebuilt in the pool child by
// child, exactly as Alg. 2 mutates enode_hist. Returns the node cost; the final history is at
// (*boff, *voff, *n_out) (boff == NONE for an empty history).
__device__ double ocf_generic(const LeafCtx& c, uint32_t nd, uint32_t* topk, uint32_t* topv, uint64_t capk,
                              uint64_t capv, uint32_t* pk, double* pv, uint32_t* boff, uint32_t* voff,
                              uint32_t* n_out, uint32_t* over) {
    const uint32_t q0 = c.nko[nd], a = c.nko[nd + 1] - q0, NW = c.NW;
    double v = c.ncost[nd];
    uint32_t hb = NONE, hv = 0, hn = 0;   // running history H (none yet)
    for (uint32_t t = 0; t < a; t++) {
        const uint32_t ck = c.kpos[q0 + t];
        if (hb != NONE && ((pk[hb + (ck >> 5)] >> (ck & 31)) & 1u)) continue;   // case 1
        const Hist h = child_hist(c, ck);
        double m = 0.0;
        uint32_t add = 0;
        if (h.present) {
            uint32_t rank = 0;
            for (uint32_t w = 0; w < NW; w++) {
                const uint32_t bw = (w >> 2) >= h.lo4 && (w >> 2) < h.hi4 ? h.bits[w] : 0u;
                const uint32_t Hw = hb != NONE ? pk[hb + w] : 0u;
                uint32_t o = bw & Hw;
                while (o) {
                    const int bpos = __ffs(o) - 1;
                    m = pymax(m, h.vals[rank + __popc(bw & ((1u << bpos) - 1u))]);
                    o &= o - 1;
                }
                add += __popc(bw & ~Hw);
                rank += __popc(bw);
            }
        }
        const double cc = h.present ? pymax(child_cost(c, ck) - m, 0.0) : child_cost(c, ck);
        const bool ck_new = !hbit(h, ck);
        const uint32_t nn = hn + add + (ck_new ? 1u : 0u);
        const uint32_t nb = atomicAdd(topk, 3 * NW), nv = atomicAdd(topv, nn);
        if ((uint64_t)nb + 3 * NW > capk || (uint64_t)nv + nn > capv) {
            atomicOr(over, ((uint64_t)nb + 3 * NW > capk ? 1u : 0u) | ((uint64_t)nv + nn > capv ? 2u : 0u));
            *boff = NONE; *voff = 0; *n_out = 0;
            return v + cc;
        }
        uint32_t o = 0, r0 = 0, r1 = 0;
        for (uint32_t w = 0; w < NW; w++) {
            const uint32_t Hw = hb != NONE ? pk[hb + w] : 0u;
            const uint32_t bw = (h.present && (w >> 2) >= h.lo4 && (w >> 2) < h.hi4) ? h.bits[w] : 0u;
            uint32_t ow = Hw | bw | bit_of(ck, w);
            pk[nb + w] = ow;
            double wm = 0.0;
            while (ow) {
                const int bpos = __ffs(ow) - 1;
                const uint32_t key = 32 * w + bpos, below = (1u << bpos) - 1u;
                double val;
                if (key == ck) val = cc;                                                 // enode_hist[child]
                else if ((Hw >> bpos) & 1u) val = pv[hv + r0 + __popc(Hw & below)];      // H wins (first writer)
                else val = h.vals[r1 + __popc(bw & below)];
                pv[nv + o++] = val;
                wm = pymax(wm, val);
                ow &= ow - 1;
            }
            reinterpret_cast<double*>(pk + nb + NW)[w] = wm;
            r0 += __popc(Hw);
            r1 += __popc(bw);
        }
        hb = nb; hv = nv; hn = nn;
        v = v + cc;
    }
    *boff = hb;
    *voff = hv;
    *n_out = hn;
    return v;
}

}  // namespace

template <int T>
__global__ void __launch_bounds__(T, 1024 / T) k_extract(Dev d, XArgs x) {   // <= 64 regs: 32 resident leaves per SM
    const uint32_t l = blockIdx.x, tid = threadIdx.x;
    const uint64_t b = d.nb[l], k0 = d.kb[l];
    const uint32_t C = d.v_C[l];
    const uint32_t* coff = d.cls_off + b + l;
    LeafCtx c;
    c.C = C;
    c.NW = ((C + 31) / 32 + 3) & ~3u;
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
    uint64_t capk = 0, capv = 0;
    uint32_t* hoffw[2] = {nullptr, nullptr};
    uint32_t* hvoffw[2] = {nullptr, nullptr};
    uint32_t* hlenw[2] = {nullptr, nullptr};
    uint32_t* hrngw[2] = {nullptr, nullptr};
    uint32_t* pkw = nullptr;
    double* pvw = nullptr;
    if (ocf) {
        const uint64_t pbk = x.pool_kbase[l], pbv = x.pool_base[l];
        capk = x.pool_kbase[l + 1] - pbk;
        capv = x.pool_base[l + 1] - pbv;
        pkw = x.pool_key + pbk;
        pvw = x.pool_val + pbv;
        c.pk = pkw;
        c.pv = pvw;
        for (int p = 0; p < 2; p++) {
            hoffw[p] = x.hoff + p * x.slot_stride + b;
            hvoffw[p] = x.hvoff + p * x.slot_stride + b;
            hlenw[p] = x.hlen + p * x.slot_stride + b;
            hrngw[p] = x.hrng + p * x.slot_stride + b;
            c.hoff[p] = hoffw[p]; c.hvoff[p] = hvoffw[p]; c.hlen[p] = hlenw[p]; c.hrng[p] = hrngw[p];
        }
    }

    __shared__ uint32_t sh_scan[33];
    __shared__ uint32_t sh_flag, sh_maxlv, sh_topk, sh_topv, sh_over;

    for (uint32_t k = tid; k < C; k += T) {
        cost[k] = __longlong_as_double(0x7ff0000000000000ll);
        prev[k] = cost[k];
        ch[k] = NONE;
        level[k] = 0;
        x.reach[b + k] = 0;
    }
    if (tid == 0) { sh_over = 0; sh_topk = 0; sh_topv = 0; }
#ifdef ESAT_DEBUG
    long long t_start = clock64(), t_lv = 0, t_sort = 0;
    long long t_pass[8] = {0};
#endif
    __syncthreads();
    // ---- K7: wavefront levels over lower-position children ----
    // level[k] = 1 + max level of k's lower-position children. Warp 0 walks the classes in
    // position order 32 at a time: children below the chunk are final (read from memory); a child
    // inside the chunk is always at a lower lane, so one in-register sweep over the lanes in order
    // (shuffle-broadcast of each lane's finished level) resolves every in-chunk chain exactly.
    if (tid < 32) {
        uint32_t mx = 0;
        for (uint32_t kb0 = 0; kb0 < C; kb0 += 32) {
            const uint32_t k = kb0 + tid;
            uint32_t lv = 0, dep = 0;   // dep: in-chunk children as a lane mask
            if (k < C)
                for (uint32_t nd = coff[k]; nd < coff[k + 1]; nd++)
                    for (uint32_t q = c.nko[nd]; q < c.nko[nd + 1]; q++) {
                        const uint32_t j = c.kpos[q];
                        if (j < kb0) { const uint32_t t = level[j] + 1; lv = t > lv ? t : lv; }
                        else if (j < k) dep |= 1u << (j - kb0);
                    }
#pragma unroll 4
            for (uint32_t i = 0; i < 31; i++) {
                const uint32_t li = __shfl_sync(0xffffffffu, lv, i);
                if ((dep >> i) & 1u) lv = li + 1 > lv ? li + 1 : lv;
            }
            if (k < C) level[k] = lv;
            mx = max(mx, __reduce_max_sync(0xffffffffu, k < C ? lv : 0u));
            __syncwarp();
        }
        if (tid == 0) sh_maxlv = mx;
    }
    __syncthreads();
#ifdef ESAT_DEBUG
    t_lv = clock64();
#endif
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

#ifdef ESAT_DEBUG
    t_sort = clock64();
#endif
    // ---- K8/K9: Gauss-Seidel passes as level sweeps ----
    const uint64_t cap = 4ull * C + 8;
    const uint32_t NW = c.NW;
    uint32_t st = X_NOT_CONVERGED, passes = 0;
    for (uint64_t it = 0; it < cap; it++) {
        const int pass = (int)it;
        c.pass = pass;
        for (uint32_t k = tid; k < C; k += T) prev[k] = cost[k];
        if (tid == 0) sh_flag = 0;
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
                    if (ocf && C > 1) {
                        hoffw[par][k] = hoffw[ppar][k];
                        hvoffw[par][k] = hvoffw[ppar][k];
                        hlenw[par][k] = hlenw[ppar][k];
                        hrngw[par][k] = hrngw[ppar][k];
                    }
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
                    uint32_t hn = NONE, hsize = 0, gb = NONE, gv = 0;
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
                            uint32_t ob, ovf, on;
                            v = ocf_generic(c, nd, &sh_topk, &sh_topv, capk, capv, pkw, pvw, &ob, &ovf, &on, &sh_over);
                            if (v < hb) { hb = v; hn = nd; hsize = on; gb = ob; gv = ovf; h_gen = true; }
                        }
                        if (bn == NONE || v < bv) { bv = v; bn = nd; }
                    }
                    if (C > 1) {
                        uint32_t offk = NONE, offv = 0, rng = 0;
                        if (hn != NONE && h_gen && gb != NONE) {
                            offk = gb; offv = gv; rng = (NW / 4) << 16;
                        } else if (!(hn != NONE && h_gen)) {
                            if (hn == NONE) hsize = 0;
                            offk = atomicAdd(&sh_topk, 3 * NW);
                            offv = atomicAdd(&sh_topv, hsize);
                            if ((uint64_t)offk + 3 * NW > capk || (uint64_t)offv + hsize > capv) {
                                atomicOr(&sh_over, ((uint64_t)offk + 3 * NW > capk ? 1u : 0u) |
                                                   ((uint64_t)offv + hsize > capv ? 2u : 0u));
                                offk = NONE;
                            } else if (hn != NONE) {
                                rng = ocf_write2(c, hn, h_cc1, h_cc2, h_skip2, pkw + offk, pvw + offv);
                            }
                        }
                        if (offk == NONE) { offk = 0; offv = 0; hsize = 0; rng = 0; atomicOr(&sh_over, 4u); }   // status reports it
                        hoffw[par][k] = offk;
                        hvoffw[par][k] = offv;
                        hlenw[par][k] = hsize;
                        hrngw[par][k] = rng;
                        if (!changed) {  // did the flushed history change w.r.t. last pass?
                            const uint32_t ok2 = hoffw[ppar][k], ov2 = hvoffw[ppar][k], n2 = hlenw[ppar][k];
                            const uint32_t r2 = hrngw[ppar][k];
                            if (n2 != hsize) changed = true;
                            // same value count; compare the occupied words of both ranges
                            const uint32_t la = rng & 0xFFFFu, ha = rng >> 16, lb = r2 & 0xFFFFu, hb2 = r2 >> 16;
                            const uint32_t lo = min(la, lb), hi = max(ha, hb2);
                            const uint4* a4 = reinterpret_cast<const uint4*>(pkw + offk);
                            const uint4* b4 = reinterpret_cast<const uint4*>(pkw + ok2);
                            for (uint32_t w4 = lo; w4 < hi && !changed; w4++) {
                                const uint4 p = (w4 >= la && w4 < ha) ? a4[w4] : make_uint4(0, 0, 0, 0);
                                const uint4 q = (w4 >= lb && w4 < hb2) ? b4[w4] : make_uint4(0, 0, 0, 0);
                                changed = p.x != q.x || p.y != q.y || p.z != q.z || p.w != q.w;
                            }
                            for (uint32_t i = 0; i < hsize && !changed; i++)
                                changed = __double_as_longlong(pvw[offv + i]) != __double_as_longlong(pvw[ov2 + i]);
                        }
                    }
                }
                if (bn != NONE && bv < cost[k]) { cost[k] = bv; ch[k] = bn; sh_flag = 1; changed = true; }
                chg_cur[k] = changed ? 1 : 0;
            }
            __syncthreads();
        }
        passes++;
#ifdef ESAT_DEBUG
        if (passes <= 8) t_pass[passes - 1] = clock64();
#endif
        const bool any_change = sh_flag != 0;
        __syncthreads();   // everyone has read the flag before thread 0 resets it for the next pass
        if (!any_change) { st = X_OK; break; }
    }
    if (sh_over) st = X_CAPACITY;

    // ---- K10: root check, validation DFS and reachable set (extraction.py:67-115, 149-153) ----
    // Fast path (warp 0): if every chosen edge reachable from the root points to a lower class
    // position and every reachable class is chosen, the selection is acyclic and the DFS can
    // neither fail nor visit anything else -- the reachable set is then one descending sweep of
    // 32-class chunks (in-chunk parent -> child pushes resolved by a shuffle sweep from the top
    // lane down). Anything else (an upward or self edge, an unchosen child) falls back to the
    // sequential DFS, which reports the reference's error class in the reference's order.
    const uint32_t root = d.v_root[l];
    if (st == X_OK && root == NONE) st = X_NO_ROOT;
    if (st == X_OK && !(cost[root] < __longlong_as_double(0x7ff0000000000000ll))) st = X_INFEASIBLE;
    uint8_t* state = x.reach + b;   // 0 unvisited, 1 on stack, 2 done
    bool fast = false;
    if (st == X_OK && tid < 32) {
        if (tid == 0) state[root] = 2;
        __syncwarp();
        bool bad = false;
        for (int kb0 = (int)((C - 1) & ~31u); kb0 >= 0; kb0 -= 32) {
            const uint32_t k = (uint32_t)kb0 + tid;
            uint32_t r = k < C ? state[k] : 0u, cmask = 0;
            bool up = false;
            uint32_t q0 = 0, q1 = 0;
            if (k < C) {
                const uint32_t nd = ch[k];
                if (nd != NONE) { q0 = c.nko[nd]; q1 = c.nko[nd + 1]; }
            }
            for (uint32_t q = q0; q < q1; q++) {
                const uint32_t j = c.kpos[q];
                if (j >= k) up = true;
                else if (j >= (uint32_t)kb0) cmask |= 1u << (j - kb0);
            }
            for (int i = 31; i >= 0; i--) {
                const uint32_t ri = __shfl_sync(0xffffffffu, r, i), mi = __shfl_sync(0xffffffffu, cmask, i);
                if (ri && ((mi >> tid) & 1u)) r = 2;
            }
            if (r) {
                if (up) bad = true;
                for (uint32_t q = q0; q < q1 && !bad; q++) {
                    const uint32_t j = c.kpos[q];
                    if (ch[j] == NONE) bad = true;
                    else if (j < (uint32_t)kb0) state[j] = 2;
                }
                state[k] = 2;
            }
            __syncwarp();
        }
        fast = !__any_sync(0xffffffffu, bad);
        if (!fast) {
            for (uint32_t k = tid; k < C; k += 32) state[k] = 0;
            __syncwarp();
        }
    }
    if (tid == 0) {
        uint32_t err = NONE;
        double rc = __longlong_as_double(0x7ff8000000000000ll);
        if (st == X_OK) {
            rc = cost[root];
            uint32_t *vs = x.stk + b, *vi = x.stki + b;
            uint32_t dpt = fast ? 0u : 1u;
            if (!fast) { vs[0] = root; vi[0] = 0; state[root] = 1; }
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
        }
#ifdef ESAT_DEBUG
        if (l < 4 || C > 800 && l < 64)
            printf("leaf %u C %u nlv %u passes %u: levels %lld sort %lld pass0 %lld pass1 %lld pass2 %lld k10 %lld cyc\n", l, C,
                   nlv, passes, t_lv - t_start, t_sort - t_lv, t_pass[0] - t_sort, passes > 1 ? t_pass[1] - t_pass[0] : 0ll,
                   passes > 2 ? t_pass[2] - t_pass[1] : 0ll, clock64() - t_pass[passes > 8 ? 7 : passes - 1]);
#endif
        if (st == X_CAPACITY) err = sh_over;   // 1: bitset pool, 2: value pool
        x.status[l] = st;
        x.err_class[l] = err;
        x.root_cost[l] = rc;
        x.passes[l] = passes;
        sh_flag = st;
    }
    __syncthreads();
    if (sh_flag == X_OK) {   // DFS states (2 = visited) -> reachable flags
        uint8_t* state = x.reach + b;
        for (uint32_t k = tid; k < C; k += T) state[k] = state[k] == 2 ? 1 : 0;
    }
}

template __global__ void k_extract<32>(Dev, XArgs);
template __global__ void k_extract<64>(Dev, XArgs);
template __global__ void k_extract<128>(Dev, XArgs);

}  // namespace esat

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
// 16-B aligned). Alg. 2's dictionary operations become word operations: membership is a bit
// test, the overlap of a child's constituents with the node's running history is an AND, the
// inherited (non-overlapping) constituents an OR, and values are located by popcount ranks.
//
// Values are shared at word granularity instead of copied: each bitset word w carries a pointer
// wptr[w] to the f64 values of its keys (key order) in the value pool, and the Python-max of
// those values wmax[w] (folded from +0.0). A merged history whose word w holds exactly one
// source's keys (the later source's keys all shadowed by the earlier one, no new key) reuses
// that source's wptr/wmax; only words that mix sources or hold a new key get fresh values. An
// overlap that covers a whole word costs one wmax load (the max of Alg. 2's overlap is
// order-independent: it only ever moves on a strictly greater value, never on NaN).
//
// History block (4*NW words): bits[NW] | wptr[NW] | wmax[NW] (f64). An empty history is the
// empty word range (no block).
#include <cstdio>

#include "esat_internal.cuh"

namespace esat {

namespace {

struct Hist {
    // block base; words outside [4*lo4, 4*hi4) are zero (not stored). An absent history has
    // lo4 == hi4 == 0, so the range tests below need no separate presence test.
    const uint32_t* bits;
    uint32_t lo4, hi4;      // occupied uint4-group range
    bool present;
};

struct LeafCtx {
    uint32_t C, k, NW;         // classes, class being evaluated, bitset words (multiple of 4)
    int pass;
    const uint32_t *nko, *kpos;
    const double *ncost, *cost, *prev;
    const uint32_t* pk;        // history blocks (leaf base applied)
    const double* pv;          // value pool
    const uint32_t *hoff, *hrng;   // parity p at + p * ss (pointer arithmetic: no local-memory array)
    uint64_t ss;
};

__device__ __forceinline__ double child_cost(const LeafCtx& c, uint32_t j) {
    return j < c.k ? c.cost[j] : c.prev[j];
}

__device__ __forceinline__ Hist child_hist(const LeafCtx& c, uint32_t j) {
    Hist h{nullptr, 0u, 0u, false};
    if (c.C == 1) return h;                       // no flush ever happens with one class
    int par;
    if (j < c.k) par = c.pass & 1;                // flushed earlier in this pass
    else if (c.pass == 0) return h;               // not flushed yet
    else par = (c.pass - 1) & 1;                  // last pass's flush
    const uint64_t at = (uint64_t)par * c.ss + j;
    h.bits = c.pk + c.hoff[at];
    const uint32_t rg = c.hrng[at];
    h.lo4 = rg & 0xFFFFu;
    h.hi4 = rg >> 16;
    h.present = true;
    return h;
}

__device__ __forceinline__ const uint32_t* wptr_of(const LeafCtx& c, const Hist& h) { return h.bits + c.NW; }
__device__ __forceinline__ const double* wmax_of(const LeafCtx& c, const Hist& h) {
    return reinterpret_cast<const double*>(h.bits + 2 * c.NW);
}

__device__ __forceinline__ bool hbit(const Hist& h, uint32_t key) {
    return ((key >> 7) - h.lo4 < h.hi4 - h.lo4) && ((h.bits[key >> 5] >> (key & 31)) & 1u);
}

__device__ __forceinline__ uint4 hword4(const Hist& h, uint32_t w4) {
    return (w4 - h.lo4 < h.hi4 - h.lo4) ? reinterpret_cast<const uint4*>(h.bits)[w4] : make_uint4(0, 0, 0, 0);
}

__device__ __forceinline__ uint32_t hword(const Hist& h, uint32_t w) {
    return ((w >> 2) - h.lo4 < h.hi4 - h.lo4) ? h.bits[w] : 0u;
}

__device__ __forceinline__ uint32_t bit_of(uint32_t key, uint32_t w) {
    return (key >> 5) == w ? (1u << (key & 31)) : 0u;
}

// Python-max over hB's values at the keys hB shares with (hA + {sA}) (extraction.py:205-221,
// PAPER.md Alg. 2 case 2). sA may be NONE.
__device__ double overlap_max(const LeafCtx& c, const Hist& hA, uint32_t sA, const Hist& hB) {
    double m = 0.0;
    const uint4* bB = reinterpret_cast<const uint4*>(hB.bits);
    const uint32_t* pB = wptr_of(c, hB);
    const double* mB = wmax_of(c, hB);
    for (uint32_t w4 = hB.lo4; w4 < hB.hi4; w4++) {
        const uint4 qB = bB[w4];
        if (!(qB.x | qB.y | qB.z | qB.w)) continue;
        const uint4 qA = hword4(hA, w4);
        const uint32_t wB[4] = {qB.x, qB.y, qB.z, qB.w}, wA[4] = {qA.x, qA.y, qA.z, qA.w};
#pragma unroll
        for (int t = 0; t < 4; t++) {
            const uint32_t w = 4 * w4 + t;
            uint32_t o = wB[t] & (wA[t] | bit_of(sA, w));
            if (!o) continue;
            if (o == wB[t]) {   // the whole word overlaps: its stored maximum
                m = pymax(m, mB[w]);
            } else {
                const double* vb = c.pv + pB[w];
                while (o) {
                    const int bpos = __ffs(o) - 1;
                    m = pymax(m, vb[__popc(wB[t] & ((1u << bpos) - 1u))]);
                    o &= o - 1;
                }
            }
        }
    }
    return m;
}

// Value of the merged history at the key of ``bit`` (one set bit of word w): sA's, then sB's
// contribution, then hA's value, then hB's (precedence of Alg. 2's dictionary writes). Branch-free
// -- lanes of a warp merge different words of different classes, and a per-source branch would
// serialise them; the load address falls back to the (valid) pool base for sA / sB keys.
__device__ __forceinline__ double merged_value(uint32_t bit, uint32_t wA, uint32_t wB, const double* va,
                                               const double* vb, uint32_t sAw, uint32_t sBw, double vA, double vB,
                                               const double* pool) {
    const uint32_t below = bit - 1u;
    const bool inA = wA & bit, inB = wB & bit;
    const uint32_t ia = __popc(wA & below), ib = __popc(wB & below);
    const double* base = inA ? va : (inB ? vb : pool);
    const uint32_t idx = inA ? ia : (inB ? ib : 0u);
    double v = base[idx];
    v = (sBw & bit) ? vB : v;
    v = (sAw & bit) ? vA : v;
    return v;
}

// Merged history hA + {sA: vA} + hB + {sB: vB} with precedence sA, sB, hA, hB (first writer of a
// key wins; Alg. 2's enode_hist[child] = cc overrides an inherited value). Writes the block at
// ob and fresh values into the value pool; returns the packed range lo4 | hi4 << 16, or NONE
// when the value pool is exhausted (*over gets bit 2).
//
// With hO present (the class's previous flush), the merge also answers "did the history change?"
// (*chg) and keeps hO's value storage for every word whose keys and values are unchanged, so an
// unchanged history keeps its value pointers from pass to pass and later comparisons against it
// are pointer tests. Without hO, *chg is left alone.
__device__ uint32_t merge_write(const LeafCtx& c, const Hist& hA, uint32_t sA, double vA, const Hist& hB,
                                uint32_t sB, double vB, uint32_t* ob, uint32_t* topv, uint64_t capv, double* pv,
                                uint32_t* over, const Hist& hO, bool* chg) {
    const uint32_t NW = c.NW;
    uint32_t lo = 0xFFFFu, hi = 0;
    if (sA != NONE) { lo = min(lo, sA >> 7); hi = max(hi, (sA >> 7) + 1); }
    if (sB != NONE) { lo = min(lo, sB >> 7); hi = max(hi, (sB >> 7) + 1); }
    if (hA.present && hA.hi4 > hA.lo4) { lo = min(lo, hA.lo4); hi = max(hi, hA.hi4); }
    if (hB.present && hB.hi4 > hB.lo4) { lo = min(lo, hB.lo4); hi = max(hi, hB.hi4); }
    bool dif = false;
    if (hO.present)   // keys of the previous flush outside the new range
        for (uint32_t w = 4 * hO.lo4; w < 4 * hO.hi4 && !dif; w++)
            if ((w < 4 * lo || w >= 4 * hi) && hO.bits[w]) dif = true;
    if (hi <= lo) {
        if (hO.present) *chg = dif;
        return 0u;
    }
    // pass 1: fresh value count (words that mix sources or hold a new key)
    uint32_t fresh = 0;
    for (uint32_t w = 4 * lo; w < 4 * hi; w++) {
        const uint32_t wA = hword(hA, w), wB = hword(hB, w), sp = bit_of(sA, w) | bit_of(sB, w);
        const bool share = !sp && (wA ? !(wB & ~wA) : true);
        if (!share) fresh += __popc(wA | wB | sp);
    }
    const uint32_t base = atomicAdd(topv, fresh);
    if ((uint64_t)base + fresh > capv) { atomicOr(over, 2u); return NONE; }
    // pass 2: bits, word pointers, word maxima, fresh values
    const uint32_t *pA = hA.present ? wptr_of(c, hA) : nullptr, *pB = hB.present ? wptr_of(c, hB) : nullptr;
    const double *mA = hA.present ? wmax_of(c, hA) : nullptr, *mB = hB.present ? wmax_of(c, hB) : nullptr;
    uint32_t* optr = ob + NW;
    double* omax = reinterpret_cast<double*>(ob + 2 * NW);
    const uint32_t* pO = hO.present ? wptr_of(c, hO) : nullptr;
    const double* mO = hO.present ? wmax_of(c, hO) : nullptr;
    uint32_t o = base;
    for (uint32_t w = 4 * lo; w < 4 * hi; w++) {
        const uint32_t wA = hword(hA, w), wB = hword(hB, w), sAw = bit_of(sA, w), sBw = bit_of(sB, w), sp = sAw | sBw;
        uint32_t ow = wA | wB | sp;
        ob[w] = ow;
        // same keys as the previous flush so far? (then its values are the comparison)
        const bool cmp = hO.present && !dif && ow && hword(hO, w) == ow;
        if (hO.present && !dif && hword(hO, w) != ow) dif = true;
        if (!sp && (wA ? !(wB & ~wA) : true)) {   // one source's word (hA's, else hB's, or empty)
            uint32_t sp_ = wA ? pA[w] : (wB ? pB[w] : 0u);
            const double sm = wA ? mA[w] : (wB ? mB[w] : 0.0);
            if (cmp && pO[w] != sp_) {
                const double *x1 = c.pv + sp_, *x2 = c.pv + pO[w];
                bool eq = true;
                for (int i = 0, n = __popc(ow); i < n && eq; i++)
                    eq = __double_as_longlong(x1[i]) == __double_as_longlong(x2[i]);
                if (eq) sp_ = pO[w];   // identical values: keep the previous storage
                else dif = true;
            }
            optr[w] = sp_;
            omax[w] = sm;
            continue;
        }
        const double* va = wA ? c.pv + pA[w] : nullptr;
        const double* vb = wB ? c.pv + pB[w] : nullptr;
        if (cmp) {   // a mixed word with the previous flush's keys: unchanged values keep its storage
            const double* vo = c.pv + pO[w];
            bool eq = true;
            uint32_t m = ow;
            for (int i = 0; m && eq; i++) {
                const uint32_t bit = m & (0u - m);
                const double val = merged_value(bit, wA, wB, va, vb, sAw, sBw, vA, vB, c.pv);
                eq = __double_as_longlong(val) == __double_as_longlong(vo[i]);
                m ^= bit;
            }
            if (eq) { optr[w] = pO[w]; omax[w] = mO[w]; continue; }
            dif = true;
        }
        optr[w] = o;
        double mx = 0.0;
        while (ow) {
            const uint32_t bit = ow & (0u - ow);
            const double val = merged_value(bit, wA, wB, va, vb, sAw, sBw, vA, vB, c.pv);
            pv[o++] = val;
            mx = pymax(mx, val);
            ow ^= bit;
        }
        omax[w] = mx;
    }
    if (hO.present) *chg = dif;
    return lo | (hi << 16);
}

// OCF cost of an arity <= 2 node (extraction.py:205-221), read-only.
__device__ double ocf_walk2(const LeafCtx& c, uint32_t nd, double* cc1_out, double* cc2_out, bool* skip2_out) {
    const uint32_t q0 = c.nko[nd], a = c.nko[nd + 1] - q0;
    double v = c.ncost[nd];
    *skip2_out = true;
    if (a == 0) return v;
    const uint32_t c1 = c.kpos[q0];
    const Hist h1 = child_hist(c, c1);
    // case 2 with an empty running history (max_cost = 0), or case 3 without a history
    const double cc1 = h1.present ? pymax(child_cost(c, c1) - 0.0, 0.0) : child_cost(c, c1);
    v = v + cc1;
    *cc1_out = cc1;
    if (a == 2) {
        const uint32_t c2 = c.kpos[q0 + 1];
        const bool skip = (c2 == c1) || hbit(h1, c2);   // case 1: already paid for
        *skip2_out = skip;
        if (!skip) {
            const Hist h2 = child_hist(c, c2);
            // case 2: overlap of h2's constituents with the running history h1 + {c1}; case 3
            const double cc2 = h2.present ? pymax(child_cost(c, c2) - overlap_max(c, h1, c1, h2), 0.0)
                                          : child_cost(c, c2);
            *cc2_out = cc2;
            v = v + cc2;
        }
    }
    return v;
}

// Generic-arity OCF node (n-ary sink): the running history is rebuilt child by child exactly as
// Alg. 2 mutates enode_hist, each step one merge into a fresh block. Returns the node cost; the
// final history block offset / range go to *boff / *rng (boff NONE on pool exhaustion).
__device__ double ocf_generic(const LeafCtx& c, uint32_t nd, uint32_t* topk, uint32_t* topv, uint64_t capk,
                              uint64_t capv, uint32_t* pk, double* pv, uint32_t* boff, uint32_t* rng,
                              uint32_t* over) {
    const uint32_t q0 = c.nko[nd], a = c.nko[nd + 1] - q0, NW = c.NW;
    double v = c.ncost[nd];
    Hist H{nullptr, 0u, 0u, false};   // running history (none yet)
    uint32_t hb = 0, hr = 0;
    const Hist none{nullptr, 0u, 0u, false};
    for (uint32_t t = 0; t < a; t++) {
        const uint32_t ck = c.kpos[q0 + t];
        if (hbit(H, ck)) continue;   // case 1
        const Hist h = child_hist(c, ck);
        const double cc = h.present ? pymax(child_cost(c, ck) - overlap_max(c, H, NONE, h), 0.0)
                                    : child_cost(c, ck);
        const uint32_t nb = atomicAdd(topk, 4 * NW);
        if ((uint64_t)nb + 4 * NW > capk) { atomicOr(over, 1u); *boff = NONE; *rng = 0; return v + cc; }
        const uint32_t r = merge_write(c, H, ck, cc, h, NONE, 0.0, pk + nb, topv, capv, pv, over, none, nullptr);
        if (r == NONE) { *boff = NONE; *rng = 0; return v + cc; }
        hb = nb; hr = r;
        H.bits = pk + nb; H.lo4 = r & 0xFFFFu; H.hi4 = r >> 16; H.present = true;
        v = v + cc;
    }
    *boff = hb;
    *rng = hr;
    return v;
}

}  // namespace

// Barrier of one leaf's threads: the CTA when it holds one leaf, else the lane group.
template <int G, int T>
__device__ __forceinline__ void gbar(uint32_t gmask) {
    if (G == T) __syncthreads();
    else __syncwarp(gmask);
}

// Exclusive scan over one leaf's threads (G == T: block_exscan; G < 32: shuffles inside the group).
template <int G>
__device__ __forceinline__ uint32_t group_exscan(uint32_t v, uint32_t* smem, uint32_t* total, uint32_t gmask) {
    if (G >= 32) return block_exscan(v, smem, total);
    const uint32_t gl = threadIdx.x % G;
    uint32_t xs = v;
#pragma unroll
    for (int o = 1; o < G; o <<= 1) {
        const uint32_t y = __shfl_up_sync(gmask, xs, o, G);
        if (gl >= (uint32_t)o) xs += y;
    }
    *total = __shfl_sync(gmask, xs, G - 1, G);
    return xs - v;
}

#ifndef ESAT_XG_MINB
#define ESAT_XG_MINB 28
#endif
// G == T: <= 64 registers, 32 resident leaves (warps) per SM. G < 32: the lane groups need more
// registers (<= 72 at 28 CTAs per SM: 56 resident leaves; 80 at 24 measured 1 % slower, 64 at 32 3 %).
template <int T, int G>
__global__ void __launch_bounds__(T, G == T ? 1024 / T : ESAT_XG_MINB) k_extract(Dev d, XArgs x) {
    // G lanes per leaf: G == T is one leaf per CTA (T = 32, 64, 128); G < 32 packs 32/G leaves into
    // one single-warp CTA, each lane group running its leaf independently (its own barriers via
    // __syncwarp(gmask), its own shared flags): the narrow Gauss-Seidel levels of small leaves leave
    // most of a warp idle, so two or four leaves share one warp's issue slots.
    static_assert(G == T || (T == 32 && G < 32 && (32 % G) == 0), "lane groups only inside one warp");
    constexpr uint32_t LPW = T / G;                 // leaves per CTA
    const uint32_t g = G == T ? 0u : threadIdx.x / G;
    const uint32_t tid = G == T ? threadIdx.x : threadIdx.x % G;   // lane within the leaf's group
    const uint32_t gmask = G >= 32 ? 0xffffffffu : (((1u << G) - 1u) << (g * G));
    const uint32_t li = blockIdx.x * LPW + g;
    if (li >= d.L) return;                         // whole group exits together (no CTA-wide barrier below)
    const uint32_t l = x.lorder ? x.lorder[li] : li;
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
    uint32_t* lhn = x.lhn + b;           // flushed node (| skip2 << 31) of each class at its last merge
    double* lcc = x.lcc + 2 * b;         // its two child contributions then
    const bool ocf = x.method == 1;
    uint64_t capk = 0, capv = 0;
    uint32_t* hoffw = nullptr;   // [parity * ss + class]
    uint32_t* hrngw = nullptr;
    const uint64_t ss = x.slot_stride;
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
        hoffw = x.hoff + b;
        hrngw = x.hrng + b;
        c.hoff = hoffw; c.hrng = hrngw; c.ss = ss;
    }

    __shared__ uint32_t sh_scan[33];
    __shared__ uint32_t sh_grp[LPW][8];   // per leaf: flag, max level, bitset top, value top, overflow
    uint32_t* const gv = sh_grp[g];       // one base register; the five scalars are constant offsets
    uint32_t &sh_flag = gv[0], &sh_maxlv = gv[1], &sh_topk = gv[2], &sh_topv = gv[3], &sh_over = gv[4];
#ifdef ESAT_DEBUG
    __shared__ unsigned dbg[2][8];   // per pass: evaluated classes, their nodes, merges, flush reuses, unchanged
    if (tid < 16) dbg[tid / 8][tid % 8] = 0;
#endif

    for (uint32_t k = tid; k < C; k += G) {
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
    gbar<G, T>(gmask);
    // ---- K7: wavefront levels over lower-position children ----
    // level[k] = 1 + max level of k's lower-position children. Warp 0 walks the classes in
    // position order 32 at a time: children below the chunk are final (read from memory); a child
    // inside the chunk is always at a lower lane, so one in-register sweep over the lanes in order
    // (shuffle-broadcast of each lane's finished level) resolves every in-chunk chain exactly.
    constexpr uint32_t CW = G < 32 ? G : 32;       // chunk width of the two in-register sweeps
    if (tid < CW) {
        uint32_t mx = 0;
        for (uint32_t kb0 = 0; kb0 < C; kb0 += CW) {
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
            for (uint32_t i = 0; i < CW - 1; i++) {
                const uint32_t lvi = __shfl_sync(gmask, lv, i, CW);
                if ((dep >> i) & 1u) lv = lvi + 1 > lv ? lvi + 1 : lv;
            }
            if (k < C) level[k] = lv;
            mx = max(mx, __reduce_max_sync(gmask, k < C ? lv : 0u));
            __syncwarp(gmask);
        }
        if (tid == 0) sh_maxlv = mx;
    }
    gbar<G, T>(gmask);
#ifdef ESAT_DEBUG
    t_lv = clock64();
#endif
    // counting sort of classes by level
    for (uint32_t k = tid; k <= C; k += G) lvcnt[k] = 0;
    gbar<G, T>(gmask);
    for (uint32_t k = tid; k < C; k += G) atomicAdd(&lvcnt[level[k]], 1u);
    gbar<G, T>(gmask);
    const uint32_t nlv = C ? sh_maxlv + 1 : 0;
    uint32_t base = 0;
    for (uint32_t c0 = 0; c0 <= nlv; c0 += G) {
        const uint32_t i = c0 + tid;
        const uint32_t v = i < nlv ? lvcnt[i] : 0u;
        uint32_t tot;
        const uint32_t p = group_exscan<G>(v, sh_scan, &tot, gmask);
        if (i <= nlv) lvcnt[i] = base + p;   // exclusive offsets; lvcnt[nlv] = C
        base += tot;
    }
    gbar<G, T>(gmask);
    for (uint32_t k = tid; k < C; k += G) order[atomicAdd(&lvcnt[level[k]], 1u)] = k;
    gbar<G, T>(gmask);
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
        for (uint32_t k = tid; k < C; k += G) prev[k] = cost[k];
        if (tid == 0) sh_flag = 0;
        gbar<G, T>(gmask);
        const int par = pass & 1, ppar = par ^ 1;
        uint8_t* chg_cur = x.chg + par * x.slot_stride + b;
        const uint8_t* chg_prv = x.chg + ppar * x.slot_stride + b;
        for (uint32_t lv = 0; lv < nlv; lv++) {
            const uint32_t lo = lv ? lvcnt[lv - 1] : 0u, hi = lvcnt[lv];
            for (uint32_t idx = lo + tid; idx < hi; idx += G) {
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
                        hoffw[par * ss + k] = hoffw[ppar * ss + k];
                        hrngw[par * ss + k] = hrngw[ppar * ss + k];
                    }
                    continue;
                }
                double bv = __longlong_as_double(0x7ff0000000000000ll);
                uint32_t bn = NONE;
                bool changed = pass == 0, hchg = pass == 0;
#ifdef ESAT_DEBUG
                if (pass < 2) { atomicAdd(&dbg[pass][0], 1u); atomicAdd(&dbg[pass][1], coff[k + 1] - coff[k]); }
#endif
                if (!ocf) {
                    for (uint32_t nd = coff[k]; nd < coff[k + 1]; nd++) {
                        double v = c.ncost[nd];
                        for (uint32_t q = c.nko[nd]; q < c.nko[nd + 1]; q++) v = v + child_cost(c, c.kpos[q]);
                        if (bn == NONE || v < bv) { bv = v; bn = nd; }
                    }
                } else {
                    // first strict-min node by ocf_enode_cost; its history is flushed for class k
                    double hb = __longlong_as_double(0x7ff0000000000000ll);
                    uint32_t hn = NONE, gb = NONE, grng = 0;
                    double h_cc1 = 0, h_cc2 = 0;
                    bool h_skip2 = true, h_gen = false;
                    for (uint32_t nd = coff[k]; nd < coff[k + 1]; nd++) {
                        double v;
                        if (c.nko[nd + 1] - c.nko[nd] <= 2) {
                            double cc1 = 0, cc2 = 0;
                            bool skip2;
                            v = ocf_walk2(c, nd, &cc1, &cc2, &skip2);
                            if (v < hb) { hb = v; hn = nd; h_cc1 = cc1; h_cc2 = cc2; h_skip2 = skip2; h_gen = false; }
                        } else {
                            uint32_t ob, orng;
                            v = ocf_generic(c, nd, &sh_topk, &sh_topv, capk, capv, pkw, pvw, &ob, &orng, &sh_over);
                            if (v < hb) { hb = v; hn = nd; gb = ob; grng = orng; h_gen = true; }
                        }
                        if (bn == NONE || v < bv) { bv = v; bn = nd; }
                    }
                    // Flush reuse (exact): the same flushed node with the same child contributions and
                    // children whose histories did not change (flag bit 1, read under the Gauss-Seidel
                    // rule) merges to the same history -- keep the previous block, no merge, no compare.
                    const uint32_t hkey = hn == NONE ? NONE : (hn | (h_skip2 ? 0x80000000u : 0u));
                    bool same = false;
                    if (C > 1 && pass > 0 && hkey == lhn[k] && !h_gen) {
                        same = true;
                        if (hn != NONE) {
                            for (uint32_t q = c.nko[hn]; q < c.nko[hn + 1] && same; q++) {
                                const uint32_t j = c.kpos[q];
                                same = !((j < k ? chg_cur[j] : chg_prv[j]) & 2u);
                            }
                            same = same && __double_as_longlong(h_cc1) == __double_as_longlong(lcc[2 * k]) &&
                                   __double_as_longlong(h_cc2) == __double_as_longlong(lcc[2 * k + 1]);
                        }
                    }
#ifdef ESAT_DEBUG
                    if (pass < 2) atomicAdd(&dbg[pass][same ? 3 : 2], 1u);
#endif
                    if (same) {
                        hoffw[par * ss + k] = hoffw[ppar * ss + k];
                        hrngw[par * ss + k] = hrngw[ppar * ss + k];
                    } else if (C > 1) {
                        lhn[k] = h_gen ? NONE - 1 : hkey;
                        lcc[2 * k] = h_cc1;
                        lcc[2 * k + 1] = h_cc2;
                        uint32_t offk = 0, rng = 0;
                        bool ok = true, merged = false, mchg = true;
                        if (hn != NONE && h_gen) {
                            ok = gb != NONE;
                            offk = gb; rng = grng;
                        } else if (hn != NONE && c.nko[hn + 1] > c.nko[hn]) {
                            const uint32_t q0 = c.nko[hn], c1 = c.kpos[q0];
                            const bool two = c.nko[hn + 1] - q0 == 2 && !h_skip2;
                            const uint32_t c2 = two ? c.kpos[q0 + 1] : NONE;
                            const Hist h1 = child_hist(c, c1);
                            const Hist h2 = two ? child_hist(c, c2) : Hist{nullptr, 0u, 0u, false};
                            offk = atomicAdd(&sh_topk, 4 * NW);
                            if ((uint64_t)offk + 4 * NW > capk) {
                                atomicOr(&sh_over, 1u);
                                ok = false;
                            } else {
                                Hist hO{nullptr, 0u, 0u, false};
                                if (pass > 0) {
                                    const uint32_t r2 = hrngw[ppar * ss + k];
                                    hO = Hist{pkw + hoffw[ppar * ss + k], r2 & 0xFFFFu, r2 >> 16, true};
                                }
                                rng = merge_write(c, h1, c1, h_cc1, h2, c2, h_cc2, pkw + offk, &sh_topv, capv, pvw,
                                                  &sh_over, hO, &mchg);
                                ok = rng != NONE;
                                merged = pass > 0 && ok;
                            }
                        }   // else: empty history (no node, or a leaf node): the empty range, no block
                        if (!ok) { offk = 0; rng = 0; atomicOr(&sh_over, 4u); }   // status reports it
                        hoffw[par * ss + k] = offk;
                        hrngw[par * ss + k] = rng;
                        hchg = pass == 0;
                        if (merged) hchg = mchg;   // answered by the merge
                        else if (!hchg) {  // did the flushed history change w.r.t. last pass?
                            const uint32_t ok2 = hoffw[ppar * ss + k], r2 = hrngw[ppar * ss + k];
                            const uint32_t la = rng & 0xFFFFu, ha = rng >> 16, lb = r2 & 0xFFFFu, hb2 = r2 >> 16;
                            const uint32_t lo = min(la, lb), hi = max(ha, hb2);
                            const uint32_t* a1 = pkw + offk;
                            const uint32_t* b1 = pkw + ok2;
                            for (uint32_t w = 4 * lo; w < 4 * hi && !hchg; w++) {
                                const uint32_t p = (w >= 4 * la && w < 4 * ha) ? a1[w] : 0u;
                                const uint32_t q = (w >= 4 * lb && w < 4 * hb2) ? b1[w] : 0u;
                                if (p != q) { hchg = true; break; }
                                if (!p) continue;
                                const uint32_t pa = a1[NW + w], pb = b1[NW + w];
                                if (pa == pb) continue;   // shared storage
                                for (uint32_t i = 0; i < (uint32_t)__popc(p); i++)
                                    if (__double_as_longlong(pvw[pa + i]) != __double_as_longlong(pvw[pb + i])) {
                                        hchg = true;
                                        break;
                                    }
                            }
                        }
                    }
                }
                if (bn != NONE && bv < cost[k]) { cost[k] = bv; ch[k] = bn; sh_flag = 1; changed = true; }
                chg_cur[k] = (changed ? 1 : 0) | (hchg ? 2 : 0);   // bit 0 cost, bit 1 history
#ifdef ESAT_DEBUG
                if (pass < 2 && !hchg && !changed) atomicAdd(&dbg[pass][4], 1u);
#endif
            }
            gbar<G, T>(gmask);
        }
        passes++;
#ifdef ESAT_DEBUG
        if (passes <= 8) t_pass[passes - 1] = clock64();
#endif
        const bool any_change = sh_flag != 0;
        gbar<G, T>(gmask);   // everyone has read the flag before thread 0 resets it for the next pass
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
    if (st == X_OK && tid < CW) {
        if (tid == 0) state[root] = 2;
        __syncwarp(gmask);
        bool bad = false;
        for (int kb0 = (int)((C - 1) & ~(CW - 1)); kb0 >= 0; kb0 -= CW) {
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
            for (int i = CW - 1; i >= 0; i--) {
                const uint32_t ri = __shfl_sync(gmask, r, i, CW), mi = __shfl_sync(gmask, cmask, i, CW);
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
            __syncwarp(gmask);
        }
        fast = !__any_sync(gmask, bad);
        if (!fast) {
            for (uint32_t k = tid; k < C; k += CW) state[k] = 0;
            __syncwarp(gmask);
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
        if (l == 0 || l == 5)
            printf("leaf %u dbg p0 %u %u %u %u %u | p1 %u %u %u %u %u\n", l, dbg[0][0], dbg[0][1], dbg[0][2], dbg[0][3],
                   dbg[0][4], dbg[1][0], dbg[1][1], dbg[1][2], dbg[1][3], dbg[1][4]);
#endif
        if (st == X_CAPACITY) err = sh_over;   // 1: bitset pool, 2: value pool
        x.status[l] = st;
        x.err_class[l] = err;
        x.root_cost[l] = rc;
        x.passes[l] = passes;
        x.levels[l] = nlv;
        sh_flag = st;
    }
    gbar<G, T>(gmask);
    if (sh_flag == X_OK) {   // DFS states (2 = visited) -> reachable flags
        uint8_t* state = x.reach + b;
        for (uint32_t k = tid; k < C; k += G) state[k] = state[k] == 2 ? 1 : 0;
    }
}

// Longest-first leaf order for k_extract (one CTA): a leaf's extraction time grows with its class
// count, and a batch of several waves finishes sooner when the largest leaves start first (the
// last wave is then made of small leaves). Counting sort of the leaves by descending class count in
// 256 buckets of 8 classes; order inside a bucket is arbitrary (every leaf's result is independent
// of the order).
__global__ void k_extract_order(Dev d, uint32_t* order) {
    __shared__ uint32_t hist[256];
    __shared__ uint32_t sh_scan[33];
    const uint32_t L = d.L;
    for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (uint32_t l = threadIdx.x; l < L; l += blockDim.x) atomicAdd(&hist[255 - min(d.v_C[l] >> 3, 255u)], 1u);
    __syncthreads();
    uint32_t tot;
    const uint32_t v = threadIdx.x < 256 ? hist[threadIdx.x] : 0u;
    const uint32_t p = block_exscan(v, sh_scan, &tot);
    __syncthreads();
    if (threadIdx.x < 256) hist[threadIdx.x] = p;
    __syncthreads();
    for (uint32_t l = threadIdx.x; l < L; l += blockDim.x)
        order[atomicAdd(&hist[255 - min(d.v_C[l] >> 3, 255u)], 1u)] = l;
}

template __global__ void k_extract<32, 32>(Dev, XArgs);
template __global__ void k_extract<32, 16>(Dev, XArgs);
template __global__ void k_extract<32, 8>(Dev, XArgs);
template __global__ void k_extract<64, 64>(Dev, XArgs);
template __global__ void k_extract<128, 128>(Dev, XArgs);

}  // namespace esat

// Internal device-side definitions shared by the esat_b200 kernels (sm_100a only).
//
// Layout: one *batch* = L leaf e-graphs concatenated (paper_2410_05534_b200/arena.py).
// Leaf l owns node-indexed rows [nb[l], nb[l+1]), kid rows [kb[l], kb[l+1]), id rows
// [ub[l], ub[l+1]); CSR offset arrays store n+1 leaf-relative entries at nb[l] + l.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#ifndef __CUDACC__
#error "CUDA only"
#endif

namespace esat {

constexpr uint32_t NONE = 0xFFFFFFFFu;

// ---- batch view handed to every kernel (by value) ------------------------------
struct Dev {
    uint32_t L;
    const uint64_t *nb, *kb, *ub, *tb;      // node / kid / id / hash-table bases [L+1]
    // dirty hashcons input (egraph.py:138 insertion order) + union-find
    const uint32_t *hc_sym, *hc_koff, *hc_kids, *hc_cid;
    const double* hc_cost;
    const uint32_t* uf_parent_in;     // pristine input union-find (rebuild is a pure function of it)
    const uint8_t* uf_rank_in;
    uint32_t* uf_parent;              // working / output union-find
    uint8_t* uf_rank;
    const uint32_t* root;
    uint32_t *n_cnt, *u_cnt;          // live hashcons entries / ids per leaf (null: the base spans; set after an apply)
    uint32_t* u_reb;                  // ids of the last rebuilt state (written by k_rebuild when non-null)
    // rebuild output: compacted hashcons
    uint32_t *o_n, *o_merges, *o_sym, *o_koff, *o_kids, *o_cid;
    double* o_cost;
    // clean view (input of ematch / extraction)
    uint32_t *v_C, *v_root, *cls_id, *cls_off, *nd_sym, *nd_koff, *nd_kpos, *nd_hc;
    double* nd_cost;
    // rebuild scratch
    uint32_t *s_ksym, *s_kkids, *s_cval, *s_val, *s_first, *s_perm;   // node/kid rows
    uint8_t* s_flag;
    uint32_t *s_sym2, *s_koff2, *s_kids2, *s_cid2;                   // second-pass input copy
    double* s_cost2;
    uint32_t *s_cnt, *s_pos, *s_coff;                                // id rows
    uint32_t *s_tc, *s_ts;                                           // hash tables (tb rows)
    // symbol table
    const uint32_t *sym_name, *sym_arity, *sym_rank, *sym_poff;
    const int32_t* sym_par;
    uint32_t n_syms;
};

// ---- extraction launch arguments (k_extract.cu) ---------------------------------
struct XArgs {
    int method;                 // 0 default, 1 OCF
    uint32_t *status, *err_class, *passes;
    uint32_t* levels;           // [L] Gauss-Seidel levels of each leaf (lane-group choice, esat_extract_shape)
    double *root_cost, *class_cost, *prev;
    uint32_t *choice, *level, *order, *lvcnt, *stk, *stki;
    uint8_t *reach;
    // OCF constituent-history pools, bump-allocated over all passes (unchanged classes keep
    // pointing at earlier histories): bitsets (u32 words) per leaf [pool_kbase[l], pool_kbase[l+1]),
    // contributions (f64) per leaf [pool_base[l], pool_base[l+1])
    const uint64_t* pool_base;
    const uint64_t* pool_kbase;
    uint32_t *pool_key;
    double* pool_val;
    uint32_t *hoff, *hrng;               // [2][node rows] history block offset / occupied range per class position (pass parity)
    uint8_t* chg;                // [2][node rows] class output changed in the pass (dirty skip): bit 0 cost, bit 1 history
    uint32_t* lhn;               // [node rows] flushed node of each class at its last merge (flush reuse)
    double* lcc;                 // [2 x node rows] its child contributions (cc1, cc2)
    uint64_t slot_stride;
    const uint32_t* lorder;      // CTA -> leaf (largest leaves first), or null (identity)
};

enum : uint32_t { X_OK = 0, X_NOT_CONVERGED = 1, X_INFEASIBLE = 2, X_CYCLIC = 3, X_CHILD_NOT_CHOSEN = 4,
                  X_ROOT_NOT_CHOSEN = 5, X_NO_ROOT = 6, X_CAPACITY = 7 };

// ---- small helpers ---------------------------------------------------------------
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

// Path-compressing find. Only called while no union is in flight (unions are issued by
// one thread between barriers), so concurrent compressions all write the same root.
__device__ __forceinline__ uint32_t uf_find(uint32_t* parent, uint32_t x) {
    uint32_t r = x;
    uint32_t p = parent[r];
    while (p != r) { r = p; p = parent[r]; }
    while (true) {
        uint32_t nx = parent[x];
        if (nx == r) break;
        parent[x] = r;
        x = nx;
    }
    return r;
}

// Rank union with ties to the lower id (egraph.py:103-115). Single-thread only.
__device__ __forceinline__ uint32_t uf_union(uint32_t* parent, uint8_t* rank, uint32_t a, uint32_t b) {
    uint32_t ra = uf_find(parent, a), rb = uf_find(parent, b);
    if (ra == rb) return ra;
    if (rank[ra] < rank[rb]) { uint32_t t = ra; ra = rb; rb = t; }
    else if (rank[ra] == rank[rb]) {
        if (rb < ra) { uint32_t t = ra; ra = rb; rb = t; }
        rank[ra] = (uint8_t)(rank[ra] + 1);
    }
    parent[rb] = ra;
    return ra;
}

__device__ __forceinline__ uint64_t mix64(uint64_t h) {
    h ^= h >> 33; h *= 0xff51afd7ed558ccdull; h ^= h >> 33; h *= 0xc4ceb9fe1a85ec53ull; h ^= h >> 33;
    return h;
}

__device__ __forceinline__ uint32_t key_hash(uint32_t sym, const uint32_t* k, uint32_t a) {
    uint64_t h = mix64(0x9E3779B97F4A7C15ull + sym);
    for (uint32_t i = 0; i < a; i++) h = mix64(h ^ (k[i] + 0x632BE59BD9B4E019ull));
    return (uint32_t)(h ^ (h >> 32) ^ a);
}

// CTA-wide exclusive scan of per-thread values (blockDim.x <= 1024). Returns this thread's
// exclusive prefix; *total receives the CTA sum. Uses `smem` (>= 33 words).
__device__ __forceinline__ uint32_t block_exscan(uint32_t v, uint32_t* smem, uint32_t* total) {
    const uint32_t lane = lane_id(), wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (uint32_t)o) x += y;
    }
    __syncthreads();
    if (lane == 31) smem[wid] = x;
    __syncthreads();
    if (wid == 0) {
        uint32_t w = lane < nw ? smem[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= (uint32_t)o) w += y;
        }
        smem[lane] = w;   // inclusive per-warp prefix
    }
    __syncthreads();
    uint32_t warp_base = wid ? smem[wid - 1] : 0u;
    *total = smem[nw - 1];
    __syncthreads();
    return warp_base + x - v;
}

// ---- TMA bulk copies (cp.async.bulk, SASS UBLKCP) global -> shared with an mbarrier ---------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// Stage a u32 array [src, src+n) into 16-B aligned shared memory at *cursor with one bulk copy of
// the enclosing 16-B aligned span; returns the element pointer inside shared memory. Issued by one
// thread; *tx accumulates the bytes the mbarrier must expect. Global buffers carry >= 16 B of
// padding so the rounded-up span never leaves the allocation.
__device__ __forceinline__ const uint32_t* stage_u32(const uint32_t* src, uint32_t n, unsigned char** cursor,
                                                     uint64_t* bar, uint32_t* tx, bool issue) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(src);
    const uintptr_t a0 = a & ~uintptr_t(15), a1 = (a + 4ull * n + 15) & ~uintptr_t(15);
    unsigned char* dst = *cursor;
    const uint32_t bytes = (uint32_t)(a1 - a0);
    if (issue && bytes) bulk_g2s(dst, reinterpret_cast<const void*>(a0), bytes, bar);
    *tx += bytes;
    *cursor = dst + bytes;
    return reinterpret_cast<const uint32_t*>(dst + (a - a0));
}
__device__ __forceinline__ uint32_t staged_bytes_u32(const uint32_t* src, uint32_t n) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(src);
    return (uint32_t)(((a + 4ull * n + 15) & ~uintptr_t(15)) - (a & ~uintptr_t(15)));
}

// Python max(a, b): returns a unless b > a (extraction.py:214, 217).
__device__ __forceinline__ double pymax(double a, double b) { return b > a ? b : a; }

}  // namespace esat

// C ABI of libesat_b200 (declared in include/esat_b200.h): context, batch arena, launches.
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/esat_b200.h"
#include "esat_internal.cuh"

namespace esat {
template <int T> __global__ void k_rebuild(Dev);
template <int T, int G> __global__ void k_extract(Dev, XArgs);
__global__ void k_extract_order(Dev, uint32_t*);
}  // namespace esat
#include "k_ematch_args.cuh"
#include "k_apply_args.cuh"
#include "k_fingerprint_args.cuh"

using namespace esat;

struct esat_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = true;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // side stream: extraction overlaps e-matching (both only read the rebuilt view)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_done = nullptr, ev_s0 = nullptr, ev_s1 = nullptr;
    cudaEvent_t ev_afork = nullptr, ev_ajoin = nullptr;   // esat_apply's two concurrent launches
    bool side_timed = false, side_pending = false, fork_armed = false;
    bool timed = false;
    // max-dynamic-SMEM attributes are per device: tracked per context (one context per device)
    uint32_t ematch_attr = 0;
    uint32_t extract_lanes = 32;   // k_extract lanes per leaf in one-warp CTAs (esat_set_extract_lanes)
    bool join_attr = false;
    char err[512] = {0};
    // symbol table
    uint32_t n_syms = 0;
    uint32_t *sym_name = nullptr, *sym_arity = nullptr, *sym_rank = nullptr, *sym_poff = nullptr;
    int32_t* sym_par = nullptr;
    // patterns
    uint32_t n_pat = 0;
    std::vector<uint32_t> pat_off;
    std::vector<int32_t> pat_words;
    int32_t* d_pat = nullptr;
    uint32_t* d_pat_off = nullptr;
    uint32_t pat_gen = 0, sym_gen = 0;
    // apply loop setup (esat_apply_setup)
    bool apply_ready = false;
    int lang = 0, cost_mode = 0;
    double coeff = 0.0;
    uint32_t a_nsyms = 0, a_tmask = 0, a_nvalues = 0, a_nrules = 0;
    uint8_t* a_ndim = nullptr;
    uint32_t *a_dims = nullptr, *a_table = nullptr, *a_rule_off = nullptr;
    int32_t *a_vint = nullptr, *a_prog = nullptr;
    std::vector<int32_t> a_head;   // per rule: from_join, list index, W
    // fingerprint setup (esat_fingerprint_setup)
    uint32_t f_nsyms = 0;
    uint32_t *f_krank = nullptr, *f_koff = nullptr;
    uint8_t* f_kbytes = nullptr;
};

namespace {

int fail(esat_ctx* c, int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(c->err, sizeof c->err, fmt, ap);
    va_end(ap);
    return code;
}

#define CK(ctx, call)                                                                        \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess)                                                               \
            return fail((ctx), ESAT_E_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

template <typename T>
int dalloc(esat_ctx* c, T** p, size_t n) {
    if (*p) cudaFree(*p);
    *p = nullptr;
    CK(c, cudaMalloc((void**)p, sizeof(T) * (n ? n : 1)));
    return ESAT_OK;
}

}  // namespace

struct esat_batch {
    esat_ctx* ctx = nullptr;
    uint32_t L = 0;
    std::vector<uint64_t> nb, kb, ub, tb;
    uint64_t N = 0, K = 0, U = 0, T = 0;
    bool uploaded = false, rebuilt = false;
    Dev d{};
    XArgs x{};
    // owned device buffers
    std::vector<void*> owned;
    // OCF pool
    double pool_factor = 32.0;   // f64 history entries per e-node
    double pool_kfactor = 0.0;   // history bitsets per e-node (0: derived from pool_factor)
    std::vector<uint64_t> pb, pbk;
    uint64_t pool_total = 0, pool_ktotal = 0;
    uint64_t *d_pb = nullptr, *d_pbk = nullptr;
    uint32_t* pool_key = nullptr;
    double* pool_val = nullptr;
    // e-matching results of the last esat_ematch / esat_join call
    uint32_t m_P = 0, j_R = 0;
    std::vector<uint32_t> m_W, j_W;
    uint32_t *d_pat_ids = nullptr, *d_m_count = nullptr, *d_m_W = nullptr, *d_j_count = nullptr;
    uint64_t *d_m_off = nullptr, *d_j_off = nullptr;
    uint32_t *stage = nullptr, *m_out = nullptr, *j_out = nullptr, *d_over = nullptr;
    uint64_t stage_cap = 0, m_cap = 0, j_cap = 0;
    unsigned long long* j_gkeys = nullptr;   // join index scratch for long source-1 lists
    uint64_t j_gkey_cap = 0;
    uint32_t* j_gsort = nullptr;             // join root-group merge scratch
    uint64_t j_gsort_cap = 0;
    unsigned long long* j_big = nullptr;     // [R][L][2] long-list pair table (k_join -> k_join_big)
    uint64_t j_big_cap = 0;
    bool j_big_seen = false, j_big_launched = false;
    JArgs j_args{};                          // arguments of the last k_join launch (reused by k_join_big)
    unsigned long long* d_tops = nullptr;   // [0] stage, [1] ematch out, [2] join stage, [3] join out
    uint32_t* d_jspec = nullptr;
    uint64_t jspec_cap = 0;
    uint32_t* d_raw = nullptr;
    // optimistic (lazily verified) re-launch of a verified e-match / join call
    uint32_t upload_gen = 0, m_mode = 0, m_Pcap = 0, j_Rcap = 0, m_smem = 0;
    uint32_t j_nsrc = 0, j_nmap_v = 0, j_nmap_q = 0;
    bool m_verified = false, m_pending = false, j_verified = false, j_pending = false;
    bool j_relaunch_needed = false, m_sig_matches_join = false, m_sized = false, j_sized = false;
    std::vector<uint32_t> m_sig, j_sig;
    uint32_t* d_lmask = nullptr;   // per-leaf pattern masks of the last esat_ematch_masked call ([chunk][leaf])
    uint32_t raw_chunks = 0, lmask_chunks = 0;   // pattern chunks (32 patterns each) d_raw / d_lmask hold
    uint32_t* x_order = nullptr;   // k_extract's leaf order (largest first)
    bool lmask_on = false;
    // apply loop: live counts (valid once set by esat_batch_set_counts or an apply) + scratch
    bool counts = false;
    uint32_t *d_ncnt = nullptr, *d_ucnt = nullptr, *d_ureb = nullptr;
    uint32_t *a_rule = nullptr, *a_status = nullptr, *a_report = nullptr, *a_missing = nullptr;
    uint32_t *a_shead = nullptr, *a_stail = nullptr, *a_snext = nullptr, *a_sseen = nullptr, *a_sstack = nullptr;
    uint32_t *a_pot = nullptr, *a_phead = nullptr, *a_ptail = nullptr, *a_pend = nullptr, *a_pnext = nullptr,
             *a_eown = nullptr;
    // fingerprint buffers
    unsigned long long *f_lab0 = nullptr, *f_lab1 = nullptr, *f_tkey = nullptr, *f_fp = nullptr;
    uint32_t *f_rep0 = nullptr, *f_rep1 = nullptr, *f_nord = nullptr, *f_tval = nullptr, *f_cord = nullptr,
             *f_status = nullptr;
    uint8_t* f_lchg = nullptr;
    unsigned long long *f_dec0 = nullptr, *f_dec1 = nullptr;
};

namespace {

// Batch buffers come from the device's stream-ordered memory pool (cudaMallocAsync, release
// threshold raised at context creation): a batch per MCTS call is created and destroyed without
// the device-wide synchronisation and unmapping of cudaMalloc / cudaFree.
static inline void afree(void* p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
}

template <typename T>
int own(esat_batch* b, T** p, size_t n) {
    *p = nullptr;
    // +64 B: TMA bulk copies read 16-B aligned spans that may round past the last element
    CK(b->ctx, cudaMallocAsync((void**)p, sizeof(T) * (n ? n : 1) + 64, b->ctx->stream));
    b->owned.push_back((void*)*p);
    return ESAT_OK;
}

#define OWN(ptr, n)                                         \
    do {                                                    \
        int r_ = own(b, &(ptr), (n));                       \
        if (r_) return r_;                                  \
    } while (0)

void tic(esat_ctx* c) { cudaEventRecord(c->ev0, c->stream); }
void toc(esat_ctx* c) {
    cudaEventRecord(c->ev1, c->stream);
    c->timed = true;
}

int launch_check(esat_ctx* c, const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(c, ESAT_E_CUDA, "%s launch failed: %s", what, cudaGetErrorString(e));
    return ESAT_OK;
}

}  // namespace

extern "C" {

int esat_ctx_create(int device, esat_ctx** out) {
    if (!out) return ESAT_E_ARG;
    esat_ctx* c = new esat_ctx();
    c->device = device;
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreate(&c->ev0);
    if (e == cudaSuccess) e = cudaEventCreate(&c->ev1);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreate(&c->ev_s0);
    if (e == cudaSuccess) e = cudaEventCreate(&c->ev_s1);
    if (e == cudaSuccess) {   // keep freed batch memory in the device pool (stream-ordered reuse)
        cudaMemPool_t pool;
        e = cudaDeviceGetDefaultMemPool(&pool, device);
        uint64_t keep = ~0ull;
        if (e == cudaSuccess) e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    if (e != cudaSuccess) {
        *out = nullptr;
        delete c;
        return ESAT_E_CUDA;
    }
    *out = c;
    return ESAT_OK;
}

int esat_ctx_destroy(esat_ctx* c) {
    if (!c) return ESAT_OK;
    cudaSetDevice(c->device);
    cudaFree(c->sym_name); cudaFree(c->sym_arity); cudaFree(c->sym_rank); cudaFree(c->sym_poff);
    cudaFree(c->sym_par); cudaFree(c->d_pat); cudaFree(c->d_pat_off);
    if (c->side) { cudaStreamSynchronize(c->side); cudaStreamDestroy(c->side); }
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_afork) cudaEventDestroy(c->ev_afork);
    if (c->ev_ajoin) cudaEventDestroy(c->ev_ajoin);
    if (c->ev_done) cudaEventDestroy(c->ev_done);
    if (c->ev_s0) cudaEventDestroy(c->ev_s0);
    if (c->ev_s1) cudaEventDestroy(c->ev_s1);
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    if (c->stream && c->own_stream) cudaStreamDestroy(c->stream);
    delete c;
    return ESAT_OK;
}

const char* esat_last_error(const esat_ctx* c) { return c ? c->err : "null context"; }

int esat_ctx_sync(esat_ctx* c) {
    CK(c, cudaStreamSynchronize(c->stream));
    return ESAT_OK;
}

float esat_last_kernel_ms(const esat_ctx* c) {
    if (!c || !c->timed) return -1.f;
    float ms = -1.f;
    if (cudaEventSynchronize(c->ev1) != cudaSuccess) return -1.f;
    cudaEventElapsedTime(&ms, c->ev0, c->ev1);
    return ms;
}

int esat_symtab_upload(esat_ctx* c, uint32_t n, const uint32_t* name, const uint32_t* arity, const uint32_t* rank,
                       const uint32_t* poff, const int32_t* par) {
    if (!c || (n && (!name || !arity || !rank || !poff))) return ESAT_E_ARG;
    cudaSetDevice(c->device);
    const uint32_t np = n ? poff[n] : 0;
    int r;
    if ((r = dalloc(c, &c->sym_name, n)) || (r = dalloc(c, &c->sym_arity, n)) || (r = dalloc(c, &c->sym_rank, n)) ||
        (r = dalloc(c, &c->sym_poff, n + 1)) || (r = dalloc(c, &c->sym_par, np)))
        return r;
    CK(c, cudaMemcpyAsync(c->sym_name, name, 4ull * n, cudaMemcpyHostToDevice, c->stream));
    CK(c, cudaMemcpyAsync(c->sym_arity, arity, 4ull * n, cudaMemcpyHostToDevice, c->stream));
    CK(c, cudaMemcpyAsync(c->sym_rank, rank, 4ull * n, cudaMemcpyHostToDevice, c->stream));
    CK(c, cudaMemcpyAsync(c->sym_poff, poff, 4ull * (n + 1), cudaMemcpyHostToDevice, c->stream));
    if (np) CK(c, cudaMemcpyAsync(c->sym_par, par, 4ull * np, cudaMemcpyHostToDevice, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    c->n_syms = n;
    c->sym_gen++;
    return ESAT_OK;
}

int esat_patterns_upload(esat_ctx* c, uint32_t n, const uint32_t* off, uint32_t n_words, const int32_t* words) {
    if (!c || (n && (!off || !words))) return ESAT_E_ARG;
    cudaSetDevice(c->device);
    c->pat_off.assign(off, off + n + 1);
    c->pat_words.assign(words, words + n_words);
    int r;
    if ((r = dalloc(c, &c->d_pat, n_words)) || (r = dalloc(c, &c->d_pat_off, n + 1))) return r;
    CK(c, cudaMemcpyAsync(c->d_pat, words, 4ull * n_words, cudaMemcpyHostToDevice, c->stream));
    CK(c, cudaMemcpyAsync(c->d_pat_off, off, 4ull * (n + 1), cudaMemcpyHostToDevice, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    c->n_pat = n;
    c->pat_gen++;
    return ESAT_OK;
}

int esat_batch_create(esat_ctx* c, uint32_t L, const uint64_t* nb, const uint64_t* kb, const uint64_t* ub,
                      esat_batch** out) {
    if (!c || !out || !nb || !kb || !ub) return ESAT_E_ARG;
    cudaSetDevice(c->device);
    esat_batch* b = new esat_batch();
    b->ctx = c;
    b->L = L;
    b->nb.assign(nb, nb + L + 1);
    b->kb.assign(kb, kb + L + 1);
    b->ub.assign(ub, ub + L + 1);
    b->tb.assign(L + 1, 0);
    for (uint32_t l = 0; l < L; l++) {
        uint64_t n = nb[l + 1] - nb[l], t = 4;   // >= 4 slots: every table 16-B aligned (k_apply clears by uint4)
        while (t < 2 * n) t <<= 1;
        b->tb[l + 1] = b->tb[l] + t;
    }
    b->N = nb[L]; b->K = kb[L]; b->U = ub[L]; b->T = b->tb[L];
    const uint64_t N = b->N, K = b->K, U = b->U, T = b->T, NL = N + L;
    Dev& d = b->d;
    d.L = L;
    uint64_t *dnb, *dkb, *dub, *dtb;
    OWN(dnb, L + 1); OWN(dkb, L + 1); OWN(dub, L + 1); OWN(dtb, L + 1);
    CK(c, cudaMemcpy(dnb, nb, 8ull * (L + 1), cudaMemcpyHostToDevice));
    CK(c, cudaMemcpy(dkb, kb, 8ull * (L + 1), cudaMemcpyHostToDevice));
    CK(c, cudaMemcpy(dub, ub, 8ull * (L + 1), cudaMemcpyHostToDevice));
    CK(c, cudaMemcpy(dtb, b->tb.data(), 8ull * (L + 1), cudaMemcpyHostToDevice));
    d.nb = dnb; d.kb = dkb; d.ub = dub; d.tb = dtb;
    uint32_t *hs, *hk, *hkids, *hc, *root;
    double* hcost;
    OWN(hs, N); OWN(hk, NL); OWN(hkids, K); OWN(hc, N); OWN(hcost, N); OWN(root, L);
    d.hc_sym = hs; d.hc_koff = hk; d.hc_kids = hkids; d.hc_cid = hc; d.hc_cost = hcost; d.root = root;
    uint32_t* upi;
    uint8_t* uri;
    OWN(upi, U); OWN(uri, U);
    d.uf_parent_in = upi; d.uf_rank_in = uri;
    OWN(d.uf_parent, U); OWN(d.uf_rank, U);
    OWN(d.o_n, L); OWN(d.o_merges, L); OWN(d.o_sym, N); OWN(d.o_koff, NL); OWN(d.o_kids, K); OWN(d.o_cid, N);
    OWN(d.o_cost, N);
    OWN(d.v_C, L); OWN(d.v_root, L); OWN(d.cls_id, N); OWN(d.cls_off, NL); OWN(d.nd_sym, N); OWN(d.nd_koff, NL);
    OWN(d.nd_kpos, K); OWN(d.nd_hc, N); OWN(d.nd_cost, N);
    OWN(d.s_ksym, N); OWN(d.s_kkids, K); OWN(d.s_cval, N); OWN(d.s_val, N); OWN(d.s_first, N); OWN(d.s_perm, N);
    OWN(d.s_flag, N);
    OWN(d.s_sym2, N); OWN(d.s_koff2, NL); OWN(d.s_kids2, K); OWN(d.s_cid2, N); OWN(d.s_cost2, N);
    OWN(d.s_cnt, U); OWN(d.s_pos, U); OWN(d.s_coff, U);
    OWN(d.s_tc, T); OWN(d.s_ts, T);
    // extraction buffers
    XArgs& x = b->x;
    OWN(x.status, L); OWN(x.err_class, L); OWN(x.passes, L); OWN(x.levels, L); OWN(x.root_cost, L);
    OWN(x.class_cost, N); OWN(x.prev, N); OWN(x.choice, N); OWN(x.level, N); OWN(x.order, N); OWN(x.lvcnt, NL);
    OWN(x.stk, N); OWN(x.stki, N); OWN(x.reach, N);
    OWN(x.hoff, 2 * N); OWN(x.hrng, 2 * N); OWN(x.chg, 2 * N); OWN(x.lhn, N); OWN(x.lcc, 2 * N);
    x.slot_stride = N;
    *out = b;
    return ESAT_OK;
}

int esat_batch_destroy(esat_batch* b) {
    if (!b) return ESAT_OK;
    esat_ctx* c = b->ctx;
    cudaSetDevice(c->device);
    if (c->side) cudaStreamSynchronize(c->side);   // an extraction of this batch may still run there
    cudaStream_t s = c->stream;
    for (void* p : b->owned) afree(p, s);
    afree(b->d_pb, c->stream); afree(b->d_pbk, c->stream); afree(b->pool_key, c->stream); afree(b->pool_val, c->stream);
    afree(b->d_lmask, c->stream);
    afree(b->d_pat_ids, c->stream); afree(b->d_m_count, c->stream); afree(b->d_m_W, c->stream); afree(b->d_j_count, c->stream);
    afree(b->d_m_off, c->stream); afree(b->d_j_off, c->stream); afree(b->stage, c->stream); afree(b->m_out, c->stream); afree(b->j_out, c->stream);
    afree(b->d_over, c->stream); afree(b->j_gkeys, c->stream); afree(b->j_gsort, c->stream); afree(b->j_big, c->stream); afree(b->d_tops, c->stream); afree(b->d_jspec, c->stream); afree(b->d_raw, c->stream);
    delete b;
    return ESAT_OK;
}

int esat_batch_upload(esat_batch* b, const uint32_t* sym, const uint32_t* koff, const uint32_t* kids,
                      const uint32_t* cid, const double* cost, const uint32_t* parent, const uint8_t* rank,
                      const uint32_t* root) {
    if (!b) return ESAT_E_ARG;
    esat_ctx* c = b->ctx;
    cudaSetDevice(c->device);
    cudaStream_t s = c->stream;
    const uint64_t N = b->N, K = b->K, U = b->U, L = b->L;
    CK(c, cudaMemcpyAsync((void*)b->d.hc_sym, sym, 4 * N, cudaMemcpyHostToDevice, s));
    CK(c, cudaMemcpyAsync((void*)b->d.hc_koff, koff, 4 * (N + L), cudaMemcpyHostToDevice, s));
    CK(c, cudaMemcpyAsync((void*)b->d.hc_kids, kids, 4 * K, cudaMemcpyHostToDevice, s));
    CK(c, cudaMemcpyAsync((void*)b->d.hc_cid, cid, 4 * N, cudaMemcpyHostToDevice, s));
    CK(c, cudaMemcpyAsync((void*)b->d.hc_cost, cost, 8 * N, cudaMemcpyHostToDevice, s));
    CK(c, cudaMemcpyAsync((void*)b->d.uf_parent_in, parent, 4 * U, cudaMemcpyHostToDevice, s));
    CK(c, cudaMemcpyAsync((void*)b->d.uf_rank_in, rank, U, cudaMemcpyHostToDevice, s));
    CK(c, cudaMemcpyAsync((void*)b->d.root, root, 4 * L, cudaMemcpyHostToDevice, s));
    b->uploaded = true;
    b->rebuilt = false;
    b->upload_gen++;
    b->counts = false;   // a plain upload fills every arena span (esat_batch_set_counts for headroom)
    b->d.n_cnt = nullptr;
    b->d.u_cnt = nullptr;
    return ESAT_OK;
}

int esat_rebuild(esat_batch* b) {
    if (!b) return ESAT_E_ARG;
    esat_ctx* c = b->ctx;
    if (!b->uploaded) return fail(c, ESAT_E_STATE, "rebuild before upload");
    if (!c->sym_rank) return fail(c, ESAT_E_STATE, "symbol table not uploaded");
    cudaSetDevice(c->device);
    Dev d = b->d;
    d.sym_name = c->sym_name; d.sym_arity = c->sym_arity; d.sym_rank = c->sym_rank; d.sym_poff = c->sym_poff;
    d.sym_par = c->sym_par; d.n_syms = c->n_syms;
    tic(c);
    if (b->L) k_rebuild<256><<<b->L, 256, 0, c->stream>>>(d);
    toc(c);
    int r = launch_check(c, "k_rebuild");
    if (r) return r;
    b->rebuilt = true;
    return ESAT_OK;
}

int esat_batch_set_pool(esat_batch* b, double entries_per_node) {
    if (!b || !(entries_per_node > 0)) return ESAT_E_ARG;
    b->pool_factor = entries_per_node;
    b->pool_kfactor = 0.0;   // the layout is recomputed at the next OCF extraction
    return ESAT_OK;
}

int esat_batch_set_pool2(esat_batch* b, double values_per_node, double bitsets_per_node) {
    if (!b || !(values_per_node > 0) || !(bitsets_per_node > 0)) return ESAT_E_ARG;
    if (b->pool_factor != values_per_node || b->pool_kfactor != bitsets_per_node) {
        b->pool_factor = values_per_node;
        b->pool_kfactor = bitsets_per_node;
    }
    return ESAT_OK;
}

// OCF history pools, laid out per leaf from the live e-node count of the last rebuild (a headroom
// arena's span is far larger than its leaf) and grown, never shrunk, when a layout needs more.
// pool_total / pool_ktotal are the allocated capacities: set only after every allocation and copy
// succeeded, so a failed growth (out of memory) leaves the batch re-allocating on the next call.
static int ensure_pool(esat_batch* b) {
    esat_ctx* c = b->ctx;
    const uint32_t L = b->L;
    // live e-nodes and classes per leaf: a headroom arena (MCTS) reads the last rebuild's sizes; a
    // plain upload (every span is its leaf) bounds the classes by the span
    std::vector<uint32_t> live(L), ncls(L);
    if (b->counts && L) {
        CK(c, cudaMemcpyAsync(live.data(), b->d.o_n, 4ull * L, cudaMemcpyDeviceToHost, c->stream));
        CK(c, cudaMemcpyAsync(ncls.data(), b->d.v_C, 4ull * L, cudaMemcpyDeviceToHost, c->stream));
        CK(c, cudaStreamSynchronize(c->stream));
    } else {
        for (uint32_t l = 0; l < L; l++) live[l] = ncls[l] = (uint32_t)(b->nb[l + 1] - b->nb[l]);
    }
    std::vector<uint64_t> pb(L + 1, 0), pbk(L + 1, 0);
    const double kf = b->pool_kfactor > 0 ? b->pool_kfactor
                                          : (b->pool_factor / 8.0 > 3.0 ? b->pool_factor / 8.0 : 3.0);
    for (uint32_t l = 0; l < L; l++) {
        const uint64_t n = live[l], C = ncls[l];
        const uint64_t nw = ((C + 31) / 32 + 3) & ~3ull;   // bitset words per history (k_extract's NW)
        pb[l + 1] = pb[l] + (uint64_t)(b->pool_factor * (double)n) + 64;
        pbk[l + 1] = pbk[l] + (uint64_t)(kf * (double)C) * 4 * nw + 16 * nw + 64;   // bits|wptr|wmax
    }
    if (b->d_pb && pb == b->pb && pbk == b->pbk && b->pool_total >= pb[L] && b->pool_ktotal >= pbk[L])
        return ESAT_OK;
    if (!b->d_pb) {
        CK(c, cudaMallocAsync((void**)&b->d_pb, 8ull * (L + 1), c->stream));
        CK(c, cudaMallocAsync((void**)&b->d_pbk, 8ull * (L + 1), c->stream));
    }
    if (b->pool_total < pb[L] || b->pool_ktotal < pbk[L]) {
        const uint64_t want = pb[L] > b->pool_total ? pb[L] : b->pool_total;
        const uint64_t kwant = pbk[L] > b->pool_ktotal ? pbk[L] : b->pool_ktotal;
        CK(c, cudaStreamSynchronize(c->stream));
        if (c->side) CK(c, cudaStreamSynchronize(c->side));
        afree(b->pool_key, c->stream); afree(b->pool_val, c->stream);
        b->pool_key = nullptr; b->pool_val = nullptr;
        b->pool_total = 0; b->pool_ktotal = 0;
        CK(c, cudaMallocAsync((void**)&b->pool_key, 4ull * kwant + 64, c->stream));
        CK(c, cudaMallocAsync((void**)&b->pool_val, 8ull * want + 64, c->stream));
        b->pool_total = want;
        b->pool_ktotal = kwant;
    }
    b->pb = pb;
    b->pbk = pbk;
    CK(c, cudaMemcpyAsync(b->d_pb, b->pb.data(), 8ull * (L + 1), cudaMemcpyHostToDevice, c->stream));
    CK(c, cudaMemcpyAsync(b->d_pbk, b->pbk.data(), 8ull * (L + 1), cudaMemcpyHostToDevice, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));   // pb / pbk are host vectors that a later call rewrites
    return ESAT_OK;
}

static int launch_extract(esat_batch* b, int method, cudaStream_t s) {
    esat_ctx* c = b->ctx;
    XArgs x = b->x;
    x.method = method;
    if (method == ESAT_METHOD_OCF) {
        int r = ensure_pool(b);
        if (r) return r;
        x.pool_base = b->d_pb;
        x.pool_kbase = b->d_pbk;
        x.pool_key = b->pool_key;
        x.pool_val = b->pool_val;
    }
    // one warp per leaf keeps a full batch resident (the MCTS case); a batch with fewer leaves than
    // SMs (one huge e-graph, config 4) gives each leaf four warps for its wide levels instead
    static const int xt_env = getenv("ESAT_EXTRACT_THREADS") ? atoi(getenv("ESAT_EXTRACT_THREADS")) : 0;
    const int xt = xt_env ? xt_env : (b->L < 148 ? 128 : 32);
    // more leaves than one wave holds: largest leaves first (k_extract_order)
    static const int xo_env = getenv("ESAT_EXTRACT_ORDER") ? atoi(getenv("ESAT_EXTRACT_ORDER")) : 1;
    x.lorder = nullptr;
    if (xo_env && b->L > 148u * 32u) {
        if (!b->x_order) OWN(b->x_order, b->L);
        k_extract_order<<<1, 1024, 0, s>>>(b->d, b->x_order);
        x.lorder = b->x_order;
    }
    // lanes per leaf in the one-warp CTAs (32: one leaf per warp; 16 / 8: two / four leaves share a
    // warp); ESAT_EXTRACT_LANES overrides the context's setting
    static const int xg_force = getenv("ESAT_EXTRACT_LANES") ? atoi(getenv("ESAT_EXTRACT_LANES")) : 0;
    const int xg_env = xg_force ? xg_force : (int)c->extract_lanes;
    if (b->L) {
        if (xt == 128) k_extract<128, 128><<<b->L, 128, 0, s>>>(b->d, x);
        else if (xt == 64) k_extract<64, 64><<<b->L, 64, 0, s>>>(b->d, x);
        else if (xg_env == 16) k_extract<32, 16><<<(unsigned)((b->L + 1) / 2), 32, 0, s>>>(b->d, x);
        else if (xg_env == 8) k_extract<32, 8><<<(unsigned)((b->L + 3) / 4), 32, 0, s>>>(b->d, x);
        else k_extract<32, 32><<<b->L, 32, 0, s>>>(b->d, x);
    }
    return launch_check(c, "k_extract");
}

int esat_extract(esat_batch* b, int method) {
    if (!b || (method != ESAT_METHOD_DEFAULT && method != ESAT_METHOD_OCF)) return ESAT_E_ARG;
    esat_ctx* c = b->ctx;
    if (!b->rebuilt) return fail(c, ESAT_E_STATE, "extraction requires a rebuilt e-graph");
    cudaSetDevice(c->device);
    tic(c);
    int r = launch_extract(b, method, c->stream);
    toc(c);
    return r;
}

int esat_extract_async(esat_batch* b, int method) {
    if (!b || (method != ESAT_METHOD_DEFAULT && method != ESAT_METHOD_OCF)) return ESAT_E_ARG;
    esat_ctx* c = b->ctx;
    if (!b->rebuilt) return fail(c, ESAT_E_STATE, "extraction requires a rebuilt e-graph");
    cudaSetDevice(c->device);
    if (method == ESAT_METHOD_OCF) {
        int r = ensure_pool(b);   // allocation is synchronous; do it before forking
        if (r) return r;
    }
    if (!c->fork_armed) CK(c, cudaEventRecord(c->ev_fork, c->stream));
    c->fork_armed = false;
    CK(c, cudaStreamWaitEvent(c->side, c->ev_fork, 0));
    CK(c, cudaEventRecord(c->ev_s0, c->side));
    int r = launch_extract(b, method, c->side);
    CK(c, cudaEventRecord(c->ev_s1, c->side));
    CK(c, cudaEventRecord(c->ev_done, c->side));
    c->side_timed = true;
    c->side_pending = true;
    return r;
}

int esat_fork(esat_ctx* c) {
    if (!c) return ESAT_E_ARG;
    CK(c, cudaEventRecord(c->ev_fork, c->stream));
    c->fork_armed = true;
    return ESAT_OK;
}

int esat_wait_async(esat_ctx* c) {
    if (!c) return ESAT_E_ARG;
    if (c->side_pending) {
        CK(c, cudaStreamWaitEvent(c->stream, c->ev_done, 0));
        c->side_pending = false;
    }
    return ESAT_OK;
}

float esat_last_async_ms(const esat_ctx* c) {
    if (!c || !c->side_timed) return -1.f;
    float ms = -1.f;
    if (cudaEventSynchronize(c->ev_s1) != cudaSuccess) return -1.f;
    cudaEventElapsedTime(&ms, c->ev_s0, c->ev_s1);
    return ms;
}

int esat_download_rebuild(esat_batch* b, uint32_t* n_out, uint32_t* merges, uint32_t* sym, uint32_t* koff,
                          uint32_t* kids, uint32_t* cid, double* cost, uint32_t* parent, uint8_t* rank) {
    if (!b) return ESAT_E_ARG;
    esat_ctx* c = b->ctx;
    cudaSetDevice(c->device);
    cudaStream_t s = c->stream;
    const uint64_t N = b->N, K = b->K, U = b->U, L = b->L;
    if (n_out) CK(c, cudaMemcpyAsync(n_out, b->d.o_n, 4 * L, cudaMemcpyDeviceToHost, s));
    if (merges) CK(c, cudaMemcpyAsync(merges, b->d.o_merges, 4 * L, cudaMemcpyDeviceToHost, s));
    if (sym) CK(c, cudaMemcpyAsync(sym, b->d.o_sym, 4 * N, cudaMemcpyDeviceToHost, s));
    if (koff) CK(c, cudaMemcpyAsync(koff, b->d.o_koff, 4 * (N + L), cudaMemcpyDeviceToHost, s));
    if (kids) CK(c, cudaMemcpyAsync(kids, b->d.o_kids, 4 * K, cudaMemcpyDeviceToHost, s));
    if (cid) CK(c, cudaMemcpyAsync(cid, b->d.o_cid, 4 * N, cudaMemcpyDeviceToHost, s));
    if (cost) CK(c, cudaMemcpyAsync(cost, b->d.o_cost, 8 * N, cudaMemcpyDeviceToHost, s));
    if (parent) CK(c, cudaMemcpyAsync(parent, b->d.uf_parent, 4 * U, cudaMemcpyDeviceToHost, s));
    if (rank) CK(c, cudaMemcpyAsync(rank, b->d.uf_rank, U, cudaMemcpyDeviceToHost, s));
    CK(c, cudaStreamSynchronize(s));
    return ESAT_OK;
}

int esat_download_view(esat_batch* b, uint32_t* C, uint32_t* root_pos, uint32_t* cls_id, uint32_t* cls_off,
                       uint32_t* nd_sym, uint32_t* nd_koff, uint32_t* nd_kpos, double* nd_cost, uint32_t* nd_hc) {
    if (!b) return ESAT_E_ARG;
    esat_ctx* c = b->ctx;
    cudaSetDevice(c->device);
    cudaStream_t s = c->stream;
    const uint64_t N = b->N, K = b->K, L = b->L;
    if (C) CK(c, cudaMemcpyAsync(C, b->d.v_C, 4 * L, cudaMemcpyDeviceToHost, s));
    if (root_pos) CK(c, cudaMemcpyAsync(root_pos, b->d.v_root, 4 * L, cudaMemcpyDeviceToHost, s));
    if (cls_id) CK(c, cudaMemcpyAsync(cls_id, b->d.cls_id, 4 * N, cudaMemcpyDeviceToHost, s));
    if (cls_off) CK(c, cudaMemcpyAsync(cls_off, b->d.cls_off, 4 * (N + L), cudaMemcpyDeviceToHost, s));
    if (nd_sym) CK(c, cudaMemcpyAsync(nd_sym, b->d.nd_sym, 4 * N, cudaMemcpyDeviceToHost, s));
    if (nd_koff) CK(c, cudaMemcpyAsync(nd_koff, b->d.nd_koff, 4 * (N + L), cudaMemcpyDeviceToHost, s));
    if (nd_kpos) CK(c, cudaMemcpyAsync(nd_kpos, b->d.nd_kpos, 4 * K, cudaMemcpyDeviceToHost, s));
    if (nd_cost) CK(c, cudaMemcpyAsync(nd_cost, b->d.nd_cost, 8 * N, cudaMemcpyDeviceToHost, s));
    if (nd_hc) CK(c, cudaMemcpyAsync(nd_hc, b->d.nd_hc, 4 * N, cudaMemcpyDeviceToHost, s));
    CK(c, cudaStreamSynchronize(s));
    return ESAT_OK;
}

int esat_download_extract(esat_batch* b, uint32_t* status, uint32_t* err_class, double* root_cost,
                          double* class_cost, uint32_t* choice, uint8_t* reachable, uint32_t* passes) {
    if (!b) return ESAT_E_ARG;
    esat_ctx* c = b->ctx;
    esat_wait_async(c);
    cudaSetDevice(c->device);
    cudaStream_t s = c->stream;
    const uint64_t N = b->N, L = b->L;
    if (status) CK(c, cudaMemcpyAsync(status, b->x.status, 4 * L, cudaMemcpyDeviceToHost, s));
    if (err_class) CK(c, cudaMemcpyAsync(err_class, b->x.err_class, 4 * L, cudaMemcpyDeviceToHost, s));
    if (root_cost) CK(c, cudaMemcpyAsync(root_cost, b->x.root_cost, 8 * L, cudaMemcpyDeviceToHost, s));
    if (class_cost) CK(c, cudaMemcpyAsync(class_cost, b->x.class_cost, 8 * N, cudaMemcpyDeviceToHost, s));
    if (choice) CK(c, cudaMemcpyAsync(choice, b->x.choice, 4 * N, cudaMemcpyDeviceToHost, s));
    if (reachable) CK(c, cudaMemcpyAsync(reachable, b->x.reach, N, cudaMemcpyDeviceToHost, s));
    if (passes) CK(c, cudaMemcpyAsync(passes, b->x.passes, 4 * L, cudaMemcpyDeviceToHost, s));
    CK(c, cudaStreamSynchronize(s));
    return ESAT_OK;
}

int esat_extract_shape(esat_batch* b, uint64_t* classes, uint64_t* levels) {
    if (!b || !classes || !levels) return ESAT_E_ARG;
    esat_ctx* c = b->ctx;
    esat_wait_async(c);
    cudaSetDevice(c->device);
    std::vector<uint32_t> C(b->L), lv(b->L);
    if (b->L) {
        CK(c, cudaMemcpyAsync(C.data(), b->d.v_C, 4 * b->L, cudaMemcpyDeviceToHost, c->stream));
        CK(c, cudaMemcpyAsync(lv.data(), b->x.levels, 4 * b->L, cudaMemcpyDeviceToHost, c->stream));
        CK(c, cudaStreamSynchronize(c->stream));
    }
    uint64_t sc = 0, sl = 0;
    for (uint64_t l = 0; l < b->L; l++) { sc += C[l]; sl += lv[l]; }
    *classes = sc;
    *levels = sl;
    return ESAT_OK;
}

int esat_set_extract_lanes(esat_ctx* c, uint32_t lanes) {
    if (!c || (lanes != 0 && lanes != 8 && lanes != 16 && lanes != 32)) return ESAT_E_ARG;
    c->extract_lanes = lanes ? lanes : 32;
    return ESAT_OK;
}

int esat_ctx_set_stream(esat_ctx* c, void* stream) {
    if (!c) return ESAT_E_ARG;
    if (c->own_stream && c->stream) {
        cudaStreamSynchronize(c->stream);
        cudaStreamDestroy(c->stream);
    }
    c->own_stream = false;
    c->stream = (cudaStream_t)stream;
    return ESAT_OK;
}

int esat_copy_results(esat_batch* b, void* dev_root_cost, void* dev_status) {
    if (!b) return ESAT_E_ARG;
    esat_ctx* c = b->ctx;
    esat_wait_async(c);
    cudaSetDevice(c->device);
    if (dev_root_cost)
        CK(c, cudaMemcpyAsync(dev_root_cost, b->x.root_cost, 8ull * b->L, cudaMemcpyDeviceToDevice, c->stream));
    if (dev_status)
        CK(c, cudaMemcpyAsync(dev_status, b->x.status, 4ull * b->L, cudaMemcpyDeviceToDevice, c->stream));
    return ESAT_OK;
}

int esat_result_device_ptrs(esat_batch* b, void** root_cost, void** status) {
    if (!b) return ESAT_E_ARG;
    if (root_cost) *root_cost = b->x.root_cost;
    if (status) *status = b->x.status;
    return ESAT_OK;
}

}  // extern "C"


// ---- e-matching (k_ematch.cu) ---------------------------------------------------------
namespace {

template <typename T>
int regrow(esat_ctx* c, T** p, uint64_t* cap, uint64_t need) {
    if (*cap >= need && *p) return ESAT_OK;
    uint64_t n = need + need / 4 + 1024;
    afree(*p, c->stream);
    *p = nullptr;
    CK(c, cudaMallocAsync((void**)p, sizeof(T) * n, c->stream));
    *cap = n;
    return ESAT_OK;
}

int ensure_match_meta(esat_batch* b) {
    esat_ctx* c = b->ctx;
    if (!b->d_tops) CK(c, cudaMallocAsync((void**)&b->d_tops, 8 * sizeof(unsigned long long), c->stream));
    if (!b->d_over) CK(c, cudaMallocAsync((void**)&b->d_over, 2 * sizeof(uint32_t), c->stream));
    return ESAT_OK;
}

}  // namespace

extern "C" {

// Launch k_ematch for the call recorded in b (pattern ids / mode already on device).
static int ematch_launch(esat_batch* b) {
    esat_ctx* c = b->ctx;
    const uint64_t L = b->L;
    const uint32_t P = b->m_P;
    int r;
    CK(c, cudaMemsetAsync(b->d_tops, 0, 2 * sizeof(unsigned long long), c->stream));
    CK(c, cudaMemsetAsync(b->d_over, 0, sizeof(uint32_t), c->stream));
    MArgs a{};
    a.prog = c->d_pat; a.prog_off = c->d_pat_off; a.pat_ids = b->d_pat_ids; a.P = P; a.mode = b->m_mode;
    a.stage = b->stage; a.stage_cap = b->stage_cap; a.tops = b->d_tops; a.raw = b->d_raw; a.nzl = b->d_raw + 32ull * (b->N + 1);
    a.out = b->m_out; a.out_cap = b->m_cap; a.count = b->d_m_count; a.off = b->d_m_off; a.overflow = b->d_over;
    Dev d = b->d;
    d.sym_name = c->sym_name; d.sym_arity = c->sym_arity; d.sym_rank = c->sym_rank; d.sym_poff = c->sym_poff;
    d.sym_par = c->sym_par; d.n_syms = c->n_syms;
    a.smem_bytes = b->m_smem;
    a.no_flat = getenv("ESAT_EMATCH_GENERIC") ? 1 : 0;
    a.leaf_mask = b->lmask_on ? b->d_lmask : nullptr;
    const uint32_t cap_bytes = 100 * 1024;
    if (a.smem_bytes > c->ematch_attr) {
        CK(c, cudaFuncSetAttribute(k_ematch<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cap_bytes));
        c->ematch_attr = cap_bytes;
    }
    tic(c);
    // one launch per 32-pattern chunk: the chunk's slices of the call's ids, rows, masks and scratch
    for (uint32_t p0 = 0; L && p0 < P; p0 += 32) {
        const uint32_t ch = p0 / 32;
        MArgs ac = a;
        ac.pat_ids = a.pat_ids + p0;
        ac.P = P - p0 < 32 ? P - p0 : 32;
        ac.count = a.count + (uint64_t)p0 * L;
        ac.off = a.off + (uint64_t)p0 * L;
        ac.raw = a.raw + 64ull * (b->N + 1) * ch;
        ac.nzl = a.nzl + 64ull * (b->N + 1) * ch;
        if (a.leaf_mask) ac.leaf_mask = a.leaf_mask + (uint64_t)ch * L;
        k_ematch<128><<<(unsigned)L, 128, a.smem_bytes, c->stream>>>(d, ac);
    }
    toc(c);
    if ((r = launch_check(c, "k_ematch"))) return r;
    return ESAT_OK;
}

// Synchronous check of the last k_ematch: regrow and relaunch on overflow.
static int ematch_settle(esat_batch* b) {
    esat_ctx* c = b->ctx;
    int r;
    for (int attempt = 0; attempt < 4; attempt++) {
        uint32_t over = 0;
        unsigned long long tops[2];
        CK(c, cudaMemcpyAsync(&over, b->d_over, 4, cudaMemcpyDeviceToHost, c->stream));
        CK(c, cudaMemcpyAsync(tops, b->d_tops, 16, cudaMemcpyDeviceToHost, c->stream));
        CK(c, cudaStreamSynchronize(c->stream));
        if (!over) { b->m_verified = true; b->m_pending = false; return ESAT_OK; }
        if ((r = regrow(c, &b->stage, &b->stage_cap, tops[0]))) return r;
        if ((r = regrow(c, &b->m_out, &b->m_cap, tops[1] > tops[0] ? tops[1] : tops[0]))) return r;
        if ((r = ematch_launch(b))) return r;
    }
    return fail(c, ESAT_E_CAPACITY, "ematch output did not fit after regrowing");
}

static int join_launch(esat_batch* b);
static int join_settle(esat_batch* b);

// Resolve optimistic (unchecked) e-match / join launches: verify capacities, redo on overflow.
// Called before any consumer of the match lists (downloads); a join issued after the e-match is
// relaunched when the e-match had to be redone.
static int verify_matches(esat_batch* b) {
    int r;
    bool redo = false;
    if (b->m_pending) {
        esat_ctx* c = b->ctx;
        uint32_t over = 0;
        CK(c, cudaMemcpyAsync(&over, b->d_over, 4, cudaMemcpyDeviceToHost, c->stream));
        CK(c, cudaStreamSynchronize(c->stream));
        b->m_pending = false;
        if (over) {   // regrow from the recorded totals and relaunch until it fits
            redo = true;
            if ((r = ematch_settle(b))) return r;
        }
    }
    if (b->j_R && (redo || b->j_pending)) {
        if (redo && (r = join_launch(b))) return r;
        if ((r = join_settle(b))) return r;
    }
    b->j_pending = false;
    return ESAT_OK;
}

int esat_ematch(esat_batch* b, uint32_t P, const uint32_t* pat_ids, int mode) {
    return esat_ematch_masked(b, P, pat_ids, mode, nullptr);
}

int esat_ematch_masked(esat_batch* b, uint32_t P, const uint32_t* pat_ids, int mode, const uint32_t* leaf_mask) {
    if (!b || (P && !pat_ids) || (mode != ESAT_MATCH_LIST && mode != ESAT_MATCH_EXISTS)) return ESAT_E_ARG;
    if (P > ESAT_MAX_CALL_PATTERNS)
        return fail(b->ctx, ESAT_E_ARG, "at most %u patterns per esat_ematch call (got %u)", ESAT_MAX_CALL_PATTERNS, P);
    esat_ctx* c = b->ctx;
    if (!b->rebuilt) return fail(c, ESAT_E_STATE, "ematch requires a rebuilt e-graph");
    for (uint32_t i = 0; i < P; i++)
        if (pat_ids[i] >= c->n_pat) return fail(c, ESAT_E_ARG, "pattern id %u out of range", pat_ids[i]);
    cudaSetDevice(c->device);
    const uint64_t L = b->L;
    int r;
    if ((r = ensure_match_meta(b))) return r;
    // Pattern list / programs / symbols unchanged -> no host->device traffic. Capacities are
    // sized by one checked launch per batch; later launches run without a host round-trip and
    // are verified lazily (verify_matches) before any consumer reads the lists.
    std::vector<uint32_t> sig(pat_ids, pat_ids + P);
    sig.push_back((uint32_t)mode);
    sig.push_back(c->pat_gen);
    sig.push_back(c->sym_gen);
    if (sig != b->m_sig) {
        const uint32_t nch = (P + 31) / 32;   // k_ematch runs one CTA per (leaf, 32-pattern chunk)
        if (P > b->m_Pcap) {
            const uint64_t Pc = 32ull * nch;
            afree(b->d_pat_ids, c->stream); afree(b->d_m_count, c->stream); afree(b->d_m_off, c->stream); afree(b->d_m_W, c->stream);
            b->d_pat_ids = nullptr; b->d_m_count = nullptr; b->d_m_off = nullptr; b->d_m_W = nullptr;
            CK(c, cudaMallocAsync((void**)&b->d_pat_ids, 4ull * Pc, c->stream));
            CK(c, cudaMallocAsync((void**)&b->d_m_count, 4ull * Pc * (L ? L : 1), c->stream));
            CK(c, cudaMallocAsync((void**)&b->d_m_off, 8ull * Pc * (L ? L : 1), c->stream));
            CK(c, cudaMallocAsync((void**)&b->d_m_W, 4ull * Pc, c->stream));
            b->m_Pcap = (uint32_t)Pc;
        }
        if (nch > b->raw_chunks) {   // [chunk][leaf][32][C] counts + work lists
            afree(b->d_raw, c->stream);
            b->d_raw = nullptr;
            CK(c, cudaMallocAsync((void**)&b->d_raw, 8ull * (b->N + 1) * 32 * nch + 64, c->stream));
            b->raw_chunks = nch;
        }
        b->m_W.resize(P);
        for (uint32_t i = 0; i < P; i++) {
            const int32_t* pg = c->pat_words.data() + c->pat_off[pat_ids[i]];
            b->m_W[i] = 1 + pg[1] + pg[2];
            if (pg[0] > MAX_PN || pg[1] > MAX_V || pg[2] > MAX_V || (int)b->m_W[i] > MAX_W)
                return fail(c, ESAT_E_ARG, "pattern %u exceeds device limits", pat_ids[i]);
        }
        CK(c, cudaMemcpyAsync(b->d_pat_ids, pat_ids, 4ull * P, cudaMemcpyHostToDevice, c->stream));
        CK(c, cudaMemcpyAsync(b->d_m_W, b->m_W.data(), 4ull * P, cudaMemcpyHostToDevice, c->stream));
        if (!b->stage_cap) {
            if ((r = regrow(c, &b->stage, &b->stage_cap, 4 * b->N + 4096))) return r;
            if ((r = regrow(c, &b->m_out, &b->m_cap, 4 * b->N + 4096))) return r;
        }
        // dynamic SMEM for staging the largest leaf's hot view (bounded; bigger leaves read global)
        uint64_t mx = 0;
        for (uint64_t l = 0; l < L; l++) {
            const uint64_t n = b->nb[l + 1] - b->nb[l];
            const uint64_t bytes = 4 * (2 * n + 1) + 2 * 32 + 4 * n + 32;   // cls_off + nd_sym + class op masks
            mx = bytes > mx ? bytes : mx;
        }
        const uint32_t cap_bytes = 100 * 1024;
        b->m_smem = (uint32_t)(mx < cap_bytes ? mx : cap_bytes);
        if (getenv("ESAT_EMATCH_NOSTAGE")) b->m_smem = 0;
        b->m_sig = sig;
        b->m_sized = false;
    }
    if (leaf_mask) {
        const uint32_t nch = (P + 31) / 32;   // mask words per leaf, chunk-major
        if (nch > b->lmask_chunks) {
            afree(b->d_lmask, c->stream);
            b->d_lmask = nullptr;
            CK(c, cudaMallocAsync((void**)&b->d_lmask, 4ull * nch * (L ? L : 1), c->stream));
            b->lmask_chunks = nch;
        }
        CK(c, cudaMemcpyAsync(b->d_lmask, leaf_mask, 4ull * nch * L, cudaMemcpyHostToDevice, c->stream));
    }
    b->lmask_on = leaf_mask != nullptr;
    b->m_P = P;
    b->m_mode = mode;
    b->j_R = 0;   // a new match call invalidates earlier join results
    b->j_pending = false;
    if ((r = ematch_launch(b))) return r;
    if (mode == ESAT_MATCH_EXISTS) { b->m_pending = false; return ESAT_OK; }
    if (b->m_sized) { b->m_pending = true; return ESAT_OK; }
    if ((r = ematch_settle(b))) return r;
    b->m_pending = false;
    b->m_sized = true;
    return ESAT_OK;
}

// products of the long-list pairs k_join prepared (their table rows are ~0 otherwise)
static int join_big_launch(esat_batch* b) {
    esat_ctx* c = b->ctx;
    const uint64_t L = b->L;
    const uint32_t R = b->j_R;
    constexpr unsigned Z = 512;
    if (L && R) k_join_big<128><<<dim3((unsigned)L, R, Z), 128, 0, c->stream>>>((uint32_t)L, b->j_args);
    b->j_big_launched = true;
    return launch_check(c, "k_join_big");
}

static int join_launch(esat_batch* b) {
    esat_ctx* c = b->ctx;
    const uint64_t L = b->L;
    const uint32_t R = b->j_R, nsrc = b->j_nsrc, nmap_v = b->j_nmap_v, nmap_q = b->j_nmap_q;
    CK(c, cudaMemsetAsync(b->d_tops + 2, 0, 3 * sizeof(unsigned long long), c->stream));
    CK(c, cudaMemsetAsync(b->d_over + 1, 0, sizeof(uint32_t), c->stream));
    const uint32_t* p = b->d_jspec;
    JArgs a{};
    a.R = R;
    a.src_off = p; a.src = p + (R + 1); a.map_off = a.src + nsrc; a.vmap = a.map_off + 2 * (nsrc + 1);
    a.qmap = a.vmap + nmap_v; a.nv = a.qmap + nmap_q; a.nq = a.nv + R;
    a.m_count = b->d_m_count; a.m_off = b->d_m_off; a.m_words = b->m_out; a.m_W = b->d_m_W;
    a.stage = nullptr; a.stage_cap = 0; a.tops = b->d_tops + 2;
    a.out = b->j_out; a.out_cap = b->j_cap; a.count = b->d_j_count; a.off = b->d_j_off; a.overflow = b->d_over + 1;
    {
        const uint64_t need = (uint64_t)R * L * (128 / 32) * JOIN_GSORT_WORDS;
        int rr = regrow(c, &b->j_gsort, &b->j_gsort_cap, need);
        if (rr) return rr;
    }
    a.gsort = b->j_gsort;
    a.gkeys = b->j_gkeys; a.gkey_cap = b->j_gkey_cap;
    {
        int rr = regrow(c, &b->j_big, &b->j_big_cap, 2ull * R * L);
        if (rr) return rr;
        CK(c, cudaMemsetAsync(b->j_big, 0xFF, 16ull * R * L, c->stream));
    }
    a.big = b->j_big;
    // run table in dynamic SMEM: one u32 per class id of the largest leaf (capped)
    uint64_t umax = 0;
    for (uint64_t l = 0; l < L; l++) umax = b->ub[l + 1] - b->ub[l] > umax ? b->ub[l + 1] - b->ub[l] : umax;
    const uint32_t run_cap = (uint32_t)(umax < 16384 ? umax : 16384);
    a.id_base = b->d.ub;
    a.run_cap = run_cap;
    a.s1_cap = JOIN_SMEM_S1;
    if (!c->join_attr) {
        CK(c, cudaFuncSetAttribute(k_join<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   4 * (16384 + JOIN_SMEM_S1)));
        c->join_attr = true;
    }
    tic(c);
    if (L && R)
        k_join<128><<<dim3((unsigned)L, R), 128, 4 * (run_cap + JOIN_SMEM_S1), c->stream>>>((uint32_t)L, a);
    b->j_args = a;
    b->j_big_launched = false;
    int r = launch_check(c, "k_join");
    if (!r && b->j_big_seen) r = join_big_launch(b);   // batches known to hold long source lists
    toc(c);
    b->j_relaunch_needed = true;
    return r;
}

static int join_settle(esat_batch* b) {
    esat_ctx* c = b->ctx;
    int r;
    for (int attempt = 0; attempt < 4; attempt++) {
        uint32_t over = 0;
        unsigned long long tops[3];
        CK(c, cudaMemcpyAsync(&over, b->d_over + 1, 4, cudaMemcpyDeviceToHost, c->stream));
        CK(c, cudaMemcpyAsync(tops, b->d_tops + 2, 24, cudaMemcpyDeviceToHost, c->stream));
        CK(c, cudaStreamSynchronize(c->stream));
        if (!over) {
            if (tops[2] && !b->j_big_launched) {   // long-list pairs were prepared: write them now
                b->j_big_seen = true;
                if ((r = join_big_launch(b))) return r;
            }
            b->j_verified = true;
            b->j_pending = false;
            return ESAT_OK;
        }
        if ((over & 4) && (r = regrow(c, &b->j_gkeys, &b->j_gkey_cap, tops[0]))) return r;
        if ((r = regrow(c, &b->j_out, &b->j_cap, tops[1]))) return r;
        if ((r = join_launch(b))) return r;
    }
    return fail(c, ESAT_E_CAPACITY, "join output did not fit after regrowing");
}

int esat_join(esat_batch* b, uint32_t R, const uint32_t* src_off, const uint32_t* src, const uint32_t* map_off,
              const uint32_t* vmap, const uint32_t* qmap, const uint32_t* nv, const uint32_t* nq) {
    if (!b || (R && (!src_off || !src || !map_off || !nv || !nq))) return ESAT_E_ARG;
    esat_ctx* c = b->ctx;
    if (!b->m_P || b->m_mode != ESAT_MATCH_LIST)
        return fail(c, ESAT_E_STATE, "esat_join needs the source matches of a LIST esat_ematch call");
    cudaSetDevice(c->device);
    const uint64_t L = b->L;
    const uint32_t nsrc = src_off[R];
    std::vector<uint32_t> jW(R);
    for (uint32_t r = 0; r < R; r++) {
        const uint32_t S = src_off[r + 1] - src_off[r];
        if (S < 1 || S > MAX_S) return fail(c, ESAT_E_ARG, "rule %u: %u sources (max %d)", r, S, MAX_S);
        for (uint32_t s = src_off[r]; s < src_off[r + 1]; s++)
            if (src[s] >= b->m_P) return fail(c, ESAT_E_ARG, "join source %u not in the last ematch call", src[s]);
        jW[r] = S + nv[r] + nq[r];
        if (jW[r] > (uint32_t)MAX_W || nv[r] > 64 || nq[r] > 64) return fail(c, ESAT_E_ARG, "rule %u too wide", r);
    }
    const uint32_t nmap_v = map_off[2 * nsrc], nmap_q = map_off[2 * nsrc + 1];
    // spec words: src_off[R+1] src[nsrc] map_off[2*(nsrc+1)] vmap[nmap_v] qmap[nmap_q] nv[R] nq[R]
    std::vector<uint32_t> spec;
    spec.insert(spec.end(), src_off, src_off + R + 1);
    spec.insert(spec.end(), src, src + nsrc);
    spec.insert(spec.end(), map_off, map_off + 2 * (nsrc + 1));
    spec.insert(spec.end(), vmap, vmap + nmap_v);
    spec.insert(spec.end(), qmap, qmap + nmap_q);
    spec.insert(spec.end(), nv, nv + R);
    spec.insert(spec.end(), nq, nq + R);
    int r_;
    if (spec != b->j_sig) {
        if ((r_ = regrow(c, &b->d_jspec, &b->jspec_cap, spec.size()))) return r_;
        CK(c, cudaMemcpyAsync(b->d_jspec, spec.data(), 4 * spec.size(), cudaMemcpyHostToDevice, c->stream));
        if (R > b->j_Rcap) {
            afree(b->d_j_count, c->stream); afree(b->d_j_off, c->stream);
            b->d_j_count = nullptr; b->d_j_off = nullptr;
            CK(c, cudaMallocAsync((void**)&b->d_j_count, 4ull * R * (L ? L : 1), c->stream));
            CK(c, cudaMallocAsync((void**)&b->d_j_off, 8ull * R * (L ? L : 1), c->stream));
            b->j_Rcap = R;
        }
        if (!b->j_cap && (r_ = regrow(c, &b->j_out, &b->j_cap, 4 * b->N + 4096))) return r_;
        b->j_sig = spec;
        b->j_sized = false;
    }
    b->j_W = jW;
    b->j_R = R; b->j_nsrc = nsrc; b->j_nmap_v = nmap_v; b->j_nmap_q = nmap_q;
    if (!b->j_sized) {   // sizing launch: needs settled sources
        b->j_R = 0;
        if ((r_ = verify_matches(b))) return r_;
        b->j_R = R;
        if ((r_ = join_launch(b))) return r_;
        if ((r_ = join_settle(b))) return r_;
        b->j_sized = true;
        b->j_pending = false;
        return ESAT_OK;
    }
    if ((r_ = join_launch(b))) return r_;
    b->j_pending = true;
    return ESAT_OK;
}

int esat_download_counts(esat_batch* b, int from_join, uint32_t* counts) {
    if (!b || !counts) return ESAT_E_ARG;
    esat_ctx* c = b->ctx;
    int rv = verify_matches(b);
    if (rv) return rv;
    cudaSetDevice(c->device);
    const uint64_t n = from_join ? b->j_R : b->m_P;
    if (n * b->L)
        CK(c, cudaMemcpyAsync(counts, from_join ? b->d_j_count : b->d_m_count, 4ull * n * b->L,
                              cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    return ESAT_OK;
}

int esat_download_matches(esat_batch* b, int from_join, uint32_t index, uint32_t* counts, uint64_t* word_off,
                          uint32_t* words, uint64_t words_cap) {
    if (!b || !counts || !word_off) return ESAT_E_ARG;
    esat_ctx* c = b->ctx;
    int rv = verify_matches(b);
    if (rv) return rv;
    const uint32_t n = from_join ? b->j_R : b->m_P;
    if (index >= n) return fail(c, ESAT_E_ARG, "match index %u out of range (%u)", index, n);
    cudaSetDevice(c->device);
    const uint64_t L = b->L;
    const uint32_t W = from_join ? b->j_W[index] : b->m_W[index];
    std::vector<uint64_t> off(L);
    CK(c, cudaMemcpyAsync(counts, (from_join ? b->d_j_count : b->d_m_count) + index * L, 4 * L,
                          cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaMemcpyAsync(off.data(), (from_join ? b->d_j_off : b->d_m_off) + index * L, 8 * L,
                          cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    uint64_t acc = 0;
    for (uint64_t l = 0; l < L; l++) { word_off[l] = acc; acc += (uint64_t)counts[l] * W; }
    word_off[L] = acc;
    if (!words) return ESAT_OK;
    if (words_cap < acc) return fail(c, ESAT_E_CAPACITY, "need %llu words", (unsigned long long)acc);
    const uint32_t* src = from_join ? b->j_out : b->m_out;
    for (uint64_t l = 0; l < L; l++)
        if (counts[l])
            CK(c, cudaMemcpyAsync(words + word_off[l], src + off[l], 4ull * counts[l] * W, cudaMemcpyDeviceToHost,
                                  c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    return ESAT_OK;
}


// ---- apply loop (K11) ----------------------------------------------------------

int esat_apply_setup(esat_ctx* c, int lang, int cost_mode, double coeff, uint32_t n_syms, const uint8_t* sym_ndim,
                     const uint32_t* sym_dims, uint32_t table_size, const uint32_t* sym_table, uint32_t n_values,
                     const int32_t* val_int, uint32_t n_rules, const uint32_t* rule_off, const int32_t* words) {
    if (!c || !sym_ndim || !sym_dims || !sym_table || !rule_off || (n_rules && !words)) return ESAT_E_ARG;
    if (table_size == 0 || (table_size & (table_size - 1))) return fail(c, ESAT_E_ARG, "table size must be a power of 2");
    if (n_syms != c->n_syms) return fail(c, ESAT_E_STATE, "apply symbols (%u) != uploaded symbol table (%u)", n_syms, c->n_syms);
    cudaSetDevice(c->device);
    int r;
    if ((r = dalloc(c, &c->a_ndim, n_syms))) return r;
    if ((r = dalloc(c, &c->a_dims, 4ull * n_syms))) return r;
    if ((r = dalloc(c, &c->a_table, table_size))) return r;
    if ((r = dalloc(c, &c->a_vint, n_values ? n_values : 1))) return r;
    if ((r = dalloc(c, &c->a_rule_off, n_rules + 1))) return r;
    const uint32_t nw = rule_off[n_rules];
    if ((r = dalloc(c, &c->a_prog, nw ? nw : 1))) return r;
    CK(c, cudaMemcpy(c->a_ndim, sym_ndim, n_syms, cudaMemcpyHostToDevice));
    CK(c, cudaMemcpy(c->a_dims, sym_dims, 16ull * n_syms, cudaMemcpyHostToDevice));
    CK(c, cudaMemcpy(c->a_table, sym_table, 4ull * table_size, cudaMemcpyHostToDevice));
    if (n_values) CK(c, cudaMemcpy(c->a_vint, val_int, 4ull * n_values, cudaMemcpyHostToDevice));
    CK(c, cudaMemcpy(c->a_rule_off, rule_off, 4ull * (n_rules + 1), cudaMemcpyHostToDevice));
    if (nw) CK(c, cudaMemcpy(c->a_prog, words, 4ull * nw, cudaMemcpyHostToDevice));
    c->a_head.assign(3ull * n_rules, 0);
    for (uint32_t i = 0; i < n_rules; i++)
        for (int k = 0; k < 3; k++) c->a_head[3 * i + k] = words[rule_off[i] + k];
    c->lang = lang; c->cost_mode = cost_mode; c->coeff = coeff;
    c->a_nsyms = n_syms; c->a_tmask = table_size - 1; c->a_nvalues = n_values; c->a_nrules = n_rules;
    c->apply_ready = true;
    return ESAT_OK;
}

static int ensure_apply_buffers(esat_batch* b) {
    if (b->d_ncnt) return ESAT_OK;
    const uint64_t N = b->N, K = b->K, U = b->U, L = b->L;
    OWN(b->d_ncnt, L); OWN(b->d_ucnt, L); OWN(b->d_ureb, L);
    b->d.u_reb = b->d_ureb;
    OWN(b->a_rule, L); OWN(b->a_status, L); OWN(b->a_report, 8 * L); OWN(b->a_missing, 16 * L);
    OWN(b->a_shead, U); OWN(b->a_stail, U); OWN(b->a_sseen, U); OWN(b->a_snext, N); OWN(b->a_sstack, N + K);
    OWN(b->a_pot, U); OWN(b->a_phead, U); OWN(b->a_ptail, U); OWN(b->a_pend, U); OWN(b->a_pnext, K);
    OWN(b->a_eown, K);
    return ESAT_OK;
}

int esat_batch_set_counts(esat_batch* b, const uint32_t* n_cnt, const uint32_t* u_cnt) {
    if (!b || !n_cnt || !u_cnt) return ESAT_E_ARG;
    esat_ctx* c = b->ctx;
    cudaSetDevice(c->device);
    int r;
    if ((r = ensure_apply_buffers(b))) return r;
    for (uint32_t l = 0; l < b->L; l++)
        if (n_cnt[l] > b->nb[l + 1] - b->nb[l] || u_cnt[l] > b->ub[l + 1] - b->ub[l])
            return fail(c, ESAT_E_ARG, "leaf %u: counts exceed the arena capacity", l);
    CK(c, cudaMemcpyAsync(b->d_ncnt, n_cnt, 4ull * b->L, cudaMemcpyHostToDevice, c->stream));
    CK(c, cudaMemcpyAsync(b->d_ucnt, u_cnt, 4ull * b->L, cudaMemcpyHostToDevice, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    b->counts = true;
    b->d.n_cnt = b->d_ncnt;
    b->d.u_cnt = b->d_ucnt;
    b->rebuilt = false;
    return ESAT_OK;
}

int esat_apply(esat_batch* b, const uint32_t* leaf_rule, uint32_t node_limit) {
    if (!b || !leaf_rule) return ESAT_E_ARG;
    esat_ctx* c = b->ctx;
    if (!c->apply_ready) return fail(c, ESAT_E_STATE, "esat_apply_setup not called");
    if (!b->rebuilt) return fail(c, ESAT_E_STATE, "apply requires a rebuilt e-graph");
    cudaSetDevice(c->device);
    int r;
    if (!b->d_ureb) return fail(c, ESAT_E_STATE, "esat_apply: call esat_batch_set_counts before the rebuild");
    if ((r = verify_matches(b))) return r;
    for (uint32_t l = 0; l < b->L; l++) {
        const uint32_t ru = leaf_rule[l];
        if (ru == 0xFFFFFFFFu) continue;
        if (ru >= c->a_nrules) return fail(c, ESAT_E_ARG, "leaf %u: rule %u out of range", l, ru);
        const int32_t fj = c->a_head[3 * ru], li = c->a_head[3 * ru + 1], W = c->a_head[3 * ru + 2];
        const uint32_t nl = fj ? b->j_R : b->m_P;
        if ((uint32_t)li >= nl) return fail(c, ESAT_E_STATE, "rule %u: match list %d not computed", ru, li);
        if ((uint32_t)W != (fj ? b->j_W[li] : b->m_W[li]))
            return fail(c, ESAT_E_STATE, "rule %u: record width %d differs from the match list's", ru, W);
    }
    CK(c, cudaMemcpyAsync(b->a_rule, leaf_rule, 4ull * b->L, cudaMemcpyHostToDevice, c->stream));
    if (!b->counts) return fail(c, ESAT_E_STATE, "esat_apply: arena without live counts (esat_batch_set_counts)");
    Dev d = b->d;
    d.n_cnt = b->d_ncnt;
    d.u_cnt = b->d_ucnt;
    d.sym_name = c->sym_name; d.sym_arity = c->sym_arity; d.sym_rank = c->sym_rank; d.sym_poff = c->sym_poff;
    d.sym_par = c->sym_par; d.n_syms = c->n_syms;
    AArgs a{};
    a.prog = c->a_prog; a.rule_off = c->a_rule_off; a.leaf_rule = b->a_rule;
    a.sym_ndim = c->a_ndim; a.sym_dims = c->a_dims; a.sym_table = c->a_table; a.sym_tmask = c->a_tmask;
    a.val_int = c->a_vint; a.n_values = c->a_nvalues;
    a.lang = c->lang; a.cost_mode = c->cost_mode; a.coeff = c->coeff; a.node_limit = node_limit;
    a.m_words = b->m_out; a.m_off = b->d_m_off; a.m_count = b->d_m_count;
    a.j_words = b->j_out; a.j_off = b->d_j_off; a.j_count = b->d_j_count;
    a.w_sym = const_cast<uint32_t*>(b->d.hc_sym); a.w_koff = const_cast<uint32_t*>(b->d.hc_koff);
    a.w_kids = const_cast<uint32_t*>(b->d.hc_kids); a.w_cid = const_cast<uint32_t*>(b->d.hc_cid);
    a.w_cost = const_cast<double*>(b->d.hc_cost);
    a.w_parent = const_cast<uint32_t*>(b->d.uf_parent_in); a.w_rank = const_cast<uint8_t*>(b->d.uf_rank_in);
    a.status = b->a_status; a.report = b->a_report; a.missing = b->a_missing;
    a.s_head = b->a_shead; a.s_tail = b->a_stail; a.s_next = b->a_snext; a.s_seen = b->a_sseen;
    a.s_stack = b->a_sstack;
    a.s_pot = b->a_pot; a.s_phead = b->a_phead; a.s_ptail = b->a_ptail; a.s_pend = b->a_pend;
    a.s_pnext = b->a_pnext; a.s_eown = b->a_eown;
    static const int no_pot = getenv("ESAT_APPLY_NO_POT") ? 1 : 0;
    a.no_pot = no_pot;
    // leaves with very many matches (multi-pattern explosions: tens of thousands) get a planner warp
    // beside the replay warp; the rest run one warp each (16 resident leaves per SM) -- the two
    // launches run concurrently. Measured (tools/ap_sweep.sh): a threshold of 256 gains 5 % on the
    // NasRNN rollout step and loses 10 % on ResNeXt's (its many 256..600-match leaves fill the
    // two-warp launch's 4 slots per SM), so only explosions take the two-warp path.
    static const uint32_t heavy = getenv("ESAT_APPLY_HEAVY") ? (uint32_t)atoi(getenv("ESAT_APPLY_HEAVY")) : 2048u;
    if (!c->ev_afork) {
        CK(c, cudaEventCreateWithFlags(&c->ev_afork, cudaEventDisableTiming));
        CK(c, cudaEventCreateWithFlags(&c->ev_ajoin, cudaEventDisableTiming));
    }
    tic(c);
    if (b->L) {
        AArgs ah = a;
        ah.sel_lo = heavy; ah.sel_hi = 0xFFFFFFFFu;
        a.sel_lo = 0; a.sel_hi = heavy;
        CK(c, cudaEventRecord(c->ev_afork, c->stream));
        CK(c, cudaStreamWaitEvent(c->side, c->ev_afork, 0));
        k_apply<2><<<b->L, 64, 0, c->side>>>(d, ah);
        CK(c, cudaEventRecord(c->ev_ajoin, c->side));
        k_apply<1><<<b->L, 32, 0, c->stream>>>(d, a);
        CK(c, cudaStreamWaitEvent(c->stream, c->ev_ajoin, 0));
    }
    toc(c);
    if ((r = launch_check(c, "k_apply"))) return r;
    b->counts = true;
    b->d.n_cnt = b->d_ncnt;
    b->d.u_cnt = b->d_ucnt;
    // the rebuilt view and the rebuild outputs still describe the pre-apply state, so an apply can
    // be retried (after host interning of a missing symbol) until the next esat_rebuild
    b->upload_gen++;
    return ESAT_OK;
}

int esat_download_apply(esat_batch* b, uint32_t* status, uint32_t* report, uint32_t* missing) {
    if (!b) return ESAT_E_ARG;
    esat_ctx* c = b->ctx;
    if (!b->a_status) return fail(c, ESAT_E_STATE, "no apply results");
    cudaSetDevice(c->device);
    cudaStream_t s = c->stream;
    const uint64_t L = b->L;
    if (status) CK(c, cudaMemcpyAsync(status, b->a_status, 4 * L, cudaMemcpyDeviceToHost, s));
    if (report) CK(c, cudaMemcpyAsync(report, b->a_report, 32 * L, cudaMemcpyDeviceToHost, s));
    if (missing) CK(c, cudaMemcpyAsync(missing, b->a_missing, 64 * L, cudaMemcpyDeviceToHost, s));
    CK(c, cudaStreamSynchronize(s));
    return ESAT_OK;
}

int esat_download_state(esat_batch* b, uint32_t* n_cnt, uint32_t* u_cnt, uint32_t* sym, uint32_t* koff,
                        uint32_t* kids, uint32_t* cid, double* cost, uint32_t* parent, uint8_t* rank) {
    if (!b) return ESAT_E_ARG;
    esat_ctx* c = b->ctx;
    cudaSetDevice(c->device);
    cudaStream_t s = c->stream;
    const uint64_t N = b->N, K = b->K, U = b->U, L = b->L;
    if (n_cnt || u_cnt) {
        std::vector<uint32_t> nc(L), uc(L);
        if (b->counts) {
            CK(c, cudaMemcpyAsync(nc.data(), b->d_ncnt, 4 * L, cudaMemcpyDeviceToHost, s));
            CK(c, cudaMemcpyAsync(uc.data(), b->d_ucnt, 4 * L, cudaMemcpyDeviceToHost, s));
            CK(c, cudaStreamSynchronize(s));
        } else {
            for (uint64_t l = 0; l < L; l++) { nc[l] = (uint32_t)(b->nb[l + 1] - b->nb[l]); uc[l] = (uint32_t)(b->ub[l + 1] - b->ub[l]); }
        }
        if (n_cnt) memcpy(n_cnt, nc.data(), 4 * L);
        if (u_cnt) memcpy(u_cnt, uc.data(), 4 * L);
    }
    if (sym) CK(c, cudaMemcpyAsync(sym, b->d.hc_sym, 4 * N, cudaMemcpyDeviceToHost, s));
    if (koff) CK(c, cudaMemcpyAsync(koff, b->d.hc_koff, 4 * (N + L), cudaMemcpyDeviceToHost, s));
    if (kids) CK(c, cudaMemcpyAsync(kids, b->d.hc_kids, 4 * K, cudaMemcpyDeviceToHost, s));
    if (cid) CK(c, cudaMemcpyAsync(cid, b->d.hc_cid, 4 * N, cudaMemcpyDeviceToHost, s));
    if (cost) CK(c, cudaMemcpyAsync(cost, b->d.hc_cost, 8 * N, cudaMemcpyDeviceToHost, s));
    if (parent) CK(c, cudaMemcpyAsync(parent, b->d.uf_parent_in, 4 * U, cudaMemcpyDeviceToHost, s));
    if (rank) CK(c, cudaMemcpyAsync(rank, b->d.uf_rank_in, U, cudaMemcpyDeviceToHost, s));
    CK(c, cudaStreamSynchronize(s));
    return ESAT_OK;
}


// ---- WL fingerprint (K12) --------------------------------------------------------

int esat_fingerprint_setup(esat_ctx* c, uint32_t n_syms, const uint32_t* krank, const uint32_t* key_off,
                           const uint8_t* key_bytes) {
    if (!c || !krank || !key_off || !key_bytes) return ESAT_E_ARG;
    if (n_syms != c->n_syms) return fail(c, ESAT_E_STATE, "fingerprint symbols (%u) != symbol table (%u)", n_syms, c->n_syms);
    cudaSetDevice(c->device);
    int r;
    const uint32_t nb = key_off[n_syms];
    if ((r = dalloc(c, &c->f_krank, n_syms))) return r;
    if ((r = dalloc(c, &c->f_koff, n_syms + 1))) return r;
    if ((r = dalloc(c, &c->f_kbytes, nb + 16))) return r;   // + 16: k_fingerprint reads whole words
    CK(c, cudaMemcpy(c->f_krank, krank, 4ull * n_syms, cudaMemcpyHostToDevice));
    CK(c, cudaMemcpy(c->f_koff, key_off, 4ull * (n_syms + 1), cudaMemcpyHostToDevice));
    if (nb) CK(c, cudaMemcpy(c->f_kbytes, key_bytes, nb, cudaMemcpyHostToDevice));
    c->f_nsyms = n_syms;
    return ESAT_OK;
}

int esat_fingerprint(esat_batch* b) {
    if (!b) return ESAT_E_ARG;
    esat_ctx* c = b->ctx;
    if (!c->f_krank || c->f_nsyms != c->n_syms) return fail(c, ESAT_E_STATE, "esat_fingerprint_setup not called for this symbol table");
    if (!b->rebuilt) return fail(c, ESAT_E_STATE, "fingerprint requires a rebuilt e-graph");
    cudaSetDevice(c->device);
    if (!b->f_lab0) {
        const uint64_t N = b->N, T = b->T, L = b->L;
        OWN(b->f_lab0, N); OWN(b->f_lab1, N); OWN(b->f_rep0, N); OWN(b->f_rep1, N); OWN(b->f_nord, N); OWN(b->f_lchg, N); OWN(b->f_dec0, 4 * N); OWN(b->f_dec1, 4 * N);
        OWN(b->f_tkey, T); OWN(b->f_tval, T); OWN(b->f_cord, T); OWN(b->f_fp, L); OWN(b->f_status, L);
    }
    FArgs a{};
    a.krank = c->f_krank; a.key_off = c->f_koff; a.key_bytes = c->f_kbytes;
    a.lab0 = b->f_lab0; a.lab1 = b->f_lab1; a.rep0 = b->f_rep0; a.rep1 = b->f_rep1; a.nord = b->f_nord; a.lchg = b->f_lchg; a.dec0 = b->f_dec0; a.dec1 = b->f_dec1;
    a.tkey = b->f_tkey; a.tval = b->f_tval; a.cord = b->f_cord; a.fp = b->f_fp; a.status = b->f_status;
    tic(c);
    if (b->L) k_fingerprint<256><<<b->L, 256, 0, c->stream>>>(b->d, a);
    toc(c);
    return launch_check(c, "k_fingerprint");
}

int esat_download_fingerprint(esat_batch* b, uint64_t* fp, uint32_t* status) {
    if (!b) return ESAT_E_ARG;
    esat_ctx* c = b->ctx;
    if (!b->f_fp) return fail(c, ESAT_E_STATE, "no fingerprints computed");
    cudaSetDevice(c->device);
    if (fp) CK(c, cudaMemcpyAsync(fp, b->f_fp, 8ull * b->L, cudaMemcpyDeviceToHost, c->stream));
    if (status) CK(c, cudaMemcpyAsync(status, b->f_status, 4ull * b->L, cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    return ESAT_OK;
}

}  // extern "C"

// ---- device snapshot store (EGraph.snapshot, egraph.py:300-312) -------------------
// An append-only device arena of leaf e-graph states ("slots"): esat_store_save copies the last
// rebuild of batch leaves into new slots (D2D), esat_batch_load_slots fills a batch's input arena
// from slots (D2D) -- an MCTS tree keeps every node's e-graph on the device, and expansions /
// rollouts start from device copies instead of host re-packs. A slot is the leaf's clean
// hashcons (order, symbols, children, classes, costs) + union-find + raw root, the same content
// as the host LeafState (arena.py).
struct esat_store {
    esat_ctx* ctx = nullptr;
    struct Slot { uint64_t on, of, ok, ou; uint32_t n, K, U, root; };
    std::vector<Slot> slots;
    uint64_t capN = 0, capF = 0, capK = 0, capU = 0;   // capacities: nodes, koff entries, kids, ids
    uint32_t *sym = nullptr, *koff = nullptr, *kids = nullptr, *cid = nullptr, *parent = nullptr;
    double* cost = nullptr;
    uint8_t* rank = nullptr;
    uint32_t* d_job = nullptr;   // copy jobs
    uint64_t job_cap = 0;
    uint64_t useN() const { return slots.empty() ? 0 : slots.back().on + slots.back().n; }
    uint64_t useF() const { return slots.empty() ? 0 : slots.back().of + slots.back().n + 1; }
    uint64_t useK() const { return slots.empty() ? 0 : slots.back().ok + slots.back().K; }
    uint64_t useU() const { return slots.empty() ? 0 : slots.back().ou + slots.back().U; }
};

namespace esat {

// job j (16 u32): leaf, slot n, K, U, then node/koff/kid/id offsets on the store side as u64 pairs
struct SlotJob { uint32_t leaf, n, K, U; uint64_t on, of, ok, ou; };

// sizes of the last rebuild of leaves[j]: n, K (= koff[n]), U (rebuilt ids), raw root
__global__ void k_store_sizes(Dev d, const uint32_t* leaves, uint32_t count, uint32_t* out) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= count) return;
    const uint32_t l = leaves[j];
    const uint32_t n = d.o_n[l];
    out[4 * j] = n;
    out[4 * j + 1] = d.o_koff[d.nb[l] + l + n];
    out[4 * j + 2] = d.u_reb ? d.u_reb[l] : (uint32_t)(d.ub[l + 1] - d.ub[l]);
    out[4 * j + 3] = d.root[l];
}

// one CTA per job: batch leaf's rebuild outputs -> store slot (save) or store slot -> batch input
// arena (load)
template <bool SAVE>
__global__ void k_store_copy(Dev d, const SlotJob* jobs, uint32_t* sym, uint32_t* koff, uint32_t* kids,
                             uint32_t* cid, double* cost, uint32_t* parent, uint8_t* rank, uint32_t* in_sym,
                             uint32_t* in_koff, uint32_t* in_kids, uint32_t* in_cid, double* in_cost,
                             uint32_t* in_parent, uint8_t* in_rank) {
    const SlotJob jb = jobs[blockIdx.x];
    const uint32_t l = jb.leaf;
    const uint64_t n0 = d.nb[l], k0 = d.kb[l], u0 = d.ub[l];
    for (uint32_t i = threadIdx.x; i < jb.n; i += blockDim.x) {
        if (SAVE) {
            sym[jb.on + i] = d.o_sym[n0 + i];
            cid[jb.on + i] = d.o_cid[n0 + i];
            cost[jb.on + i] = d.o_cost[n0 + i];
        } else {
            in_sym[n0 + i] = sym[jb.on + i];
            in_cid[n0 + i] = cid[jb.on + i];
            in_cost[n0 + i] = cost[jb.on + i];
        }
    }
    for (uint32_t i = threadIdx.x; i <= jb.n; i += blockDim.x) {
        if (SAVE) koff[jb.of + i] = d.o_koff[n0 + l + i];
        else in_koff[n0 + l + i] = koff[jb.of + i];
    }
    for (uint32_t i = threadIdx.x; i < jb.K; i += blockDim.x) {
        if (SAVE) kids[jb.ok + i] = d.o_kids[k0 + i];
        else in_kids[k0 + i] = kids[jb.ok + i];
    }
    for (uint32_t i = threadIdx.x; i < jb.U; i += blockDim.x) {
        if (SAVE) { parent[jb.ou + i] = d.uf_parent[u0 + i]; rank[jb.ou + i] = d.uf_rank[u0 + i]; }
        else { in_parent[u0 + i] = parent[jb.ou + i]; in_rank[u0 + i] = rank[jb.ou + i]; }
    }
}

}  // namespace esat

namespace {

template <typename T>
int store_grow(esat_store* st, T** p, uint64_t* cap, uint64_t used, uint64_t need) {
    if (need <= *cap && *p) return ESAT_OK;
    esat_ctx* c = st->ctx;
    uint64_t nc = *cap ? *cap : 4096;
    while (nc < need) nc *= 2;
    T* q = nullptr;
    CK(c, cudaMallocAsync((void**)&q, sizeof(T) * nc, c->stream));
    if (*p && used) CK(c, cudaMemcpyAsync(q, *p, sizeof(T) * used, cudaMemcpyDeviceToDevice, c->stream));
    afree(*p, c->stream);
    *p = q;
    *cap = nc;
    return ESAT_OK;
}

int store_reserve(esat_store* st, uint64_t n, uint64_t f, uint64_t k, uint64_t u) {
    int r;
    const uint64_t un = st->useN(), uf = st->useF(), uk = st->useK(), uu = st->useU();
    uint64_t cn = st->capN, cn2 = st->capN, cn3 = st->capN, cu = st->capU;
    if ((r = store_grow(st, &st->sym, &cn, un, un + n)) || (r = store_grow(st, &st->cid, &cn2, un, un + n)) ||
        (r = store_grow(st, &st->cost, &cn3, un, un + n)))
        return r;
    st->capN = cn;
    if ((r = store_grow(st, &st->koff, &st->capF, uf, uf + f))) return r;
    if ((r = store_grow(st, &st->kids, &st->capK, uk, uk + k))) return r;
    uint64_t cu2 = st->capU;
    if ((r = store_grow(st, &st->parent, &cu, uu, uu + u)) || (r = store_grow(st, &st->rank, &cu2, uu, uu + u)))
        return r;
    st->capU = cu;
    return ESAT_OK;
}

int store_jobs(esat_store* st, const std::vector<SlotJob>& jobs) {
    esat_ctx* c = st->ctx;
    const uint64_t words = (sizeof(SlotJob) * jobs.size() + 3) / 4;
    if (words > st->job_cap) {
        afree(st->d_job, c->stream);
        st->d_job = nullptr;
        CK(c, cudaMallocAsync((void**)&st->d_job, 4 * words, c->stream));
        st->job_cap = words;
    }
    CK(c, cudaMemcpyAsync(st->d_job, jobs.data(), sizeof(SlotJob) * jobs.size(), cudaMemcpyHostToDevice, c->stream));
    return ESAT_OK;
}

}  // namespace

extern "C" {

int esat_store_create(esat_ctx* c, esat_store** out) {
    if (!c || !out) return ESAT_E_ARG;
    esat_store* st = new esat_store();
    st->ctx = c;
    *out = st;
    return ESAT_OK;
}

int esat_store_destroy(esat_store* st) {
    if (!st) return ESAT_OK;
    esat_ctx* c = st->ctx;
    cudaSetDevice(c->device);
    afree(st->sym, c->stream); afree(st->koff, c->stream); afree(st->kids, c->stream); afree(st->cid, c->stream);
    afree(st->cost, c->stream); afree(st->parent, c->stream); afree(st->rank, c->stream); afree(st->d_job, c->stream);
    delete st;
    return ESAT_OK;
}

uint32_t esat_store_size(const esat_store* st) { return st ? (uint32_t)st->slots.size() : 0u; }

int esat_store_truncate(esat_store* st, uint32_t count) {
    if (!st || count > st->slots.size()) return ESAT_E_ARG;
    st->slots.resize(count);
    return ESAT_OK;
}

int esat_store_info(const esat_store* st, uint32_t count, const uint32_t* slots, uint32_t* n, uint32_t* K,
                    uint32_t* U, uint32_t* root) {
    if (!st || (count && !slots)) return ESAT_E_ARG;
    for (uint32_t j = 0; j < count; j++) {
        if (slots[j] >= st->slots.size()) return fail(st->ctx, ESAT_E_ARG, "slot %u out of range", slots[j]);
        const esat_store::Slot& s = st->slots[slots[j]];
        if (n) n[j] = s.n;
        if (K) K[j] = s.K;
        if (U) U[j] = s.U;
        if (root) root[j] = s.root;
    }
    return ESAT_OK;
}

int esat_store_save(esat_store* st, esat_batch* b, uint32_t count, const uint32_t* leaves, uint32_t* slots_out) {
    if (!st || !b || b->ctx != st->ctx || (count && (!leaves || !slots_out))) return ESAT_E_ARG;
    esat_ctx* c = st->ctx;
    if (!b->rebuilt) return fail(c, ESAT_E_STATE, "snapshot save requires a rebuilt batch");
    if (!count) return ESAT_OK;
    for (uint32_t j = 0; j < count; j++)
        if (leaves[j] >= b->L) return fail(c, ESAT_E_ARG, "leaf %u out of range", leaves[j]);
    cudaSetDevice(c->device);
    uint32_t *d_leaves = nullptr, *d_sz = nullptr;
    CK(c, cudaMallocAsync((void**)&d_leaves, 4ull * count, c->stream));
    CK(c, cudaMallocAsync((void**)&d_sz, 16ull * count, c->stream));
    CK(c, cudaMemcpyAsync(d_leaves, leaves, 4ull * count, cudaMemcpyHostToDevice, c->stream));
    Dev d = b->d;
    if (!b->counts) d.u_reb = nullptr;
    k_store_sizes<<<(count + 127) / 128, 128, 0, c->stream>>>(d, d_leaves, count, d_sz);
    std::vector<uint32_t> sz(4ull * count);
    CK(c, cudaMemcpyAsync(sz.data(), d_sz, 16ull * count, cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    afree(d_leaves, c->stream);
    afree(d_sz, c->stream);
    uint64_t tn = 0, tk = 0, tu = 0;
    for (uint32_t j = 0; j < count; j++) { tn += sz[4 * j]; tk += sz[4 * j + 1]; tu += sz[4 * j + 2]; }
    int r;
    if ((r = store_reserve(st, tn, tn + count, tk, tu))) return r;
    std::vector<SlotJob> jobs(count);
    for (uint32_t j = 0; j < count; j++) {
        esat_store::Slot s{st->useN(), st->useF(), st->useK(), st->useU(), sz[4 * j], sz[4 * j + 1], sz[4 * j + 2],
                           sz[4 * j + 3]};
        jobs[j] = SlotJob{leaves[j], s.n, s.K, s.U, s.on, s.of, s.ok, s.ou};
        slots_out[j] = (uint32_t)st->slots.size();
        st->slots.push_back(s);
    }
    if ((r = store_jobs(st, jobs))) return r;
    k_store_copy<true><<<count, 256, 0, c->stream>>>(b->d, reinterpret_cast<const SlotJob*>(st->d_job), st->sym,
                                                     st->koff, st->kids, st->cid, st->cost, st->parent, st->rank,
                                                     nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
    return launch_check(c, "k_store_copy");
}

int esat_store_put(esat_store* st, uint32_t n, uint32_t K, uint32_t U, uint32_t root, const uint32_t* sym,
                   const uint32_t* koff, const uint32_t* kids, const uint32_t* cid, const double* cost,
                   const uint32_t* parent, const uint8_t* rank, uint32_t* slot_out) {
    if (!st || !slot_out || !koff || (n && (!sym || !cid || !cost)) || (K && !kids) || (U && (!parent || !rank)))
        return ESAT_E_ARG;
    esat_ctx* c = st->ctx;
    cudaSetDevice(c->device);
    int r;
    if ((r = store_reserve(st, n, n + 1, K, U))) return r;
    esat_store::Slot s{st->useN(), st->useF(), st->useK(), st->useU(), n, K, U, root};
    cudaStream_t q = c->stream;
    if (n) {
        CK(c, cudaMemcpyAsync(st->sym + s.on, sym, 4ull * n, cudaMemcpyHostToDevice, q));
        CK(c, cudaMemcpyAsync(st->cid + s.on, cid, 4ull * n, cudaMemcpyHostToDevice, q));
        CK(c, cudaMemcpyAsync(st->cost + s.on, cost, 8ull * n, cudaMemcpyHostToDevice, q));
    }
    CK(c, cudaMemcpyAsync(st->koff + s.of, koff, 4ull * (n + 1), cudaMemcpyHostToDevice, q));
    if (K) CK(c, cudaMemcpyAsync(st->kids + s.ok, kids, 4ull * K, cudaMemcpyHostToDevice, q));
    if (U) {
        CK(c, cudaMemcpyAsync(st->parent + s.ou, parent, 4ull * U, cudaMemcpyHostToDevice, q));
        CK(c, cudaMemcpyAsync(st->rank + s.ou, rank, U, cudaMemcpyHostToDevice, q));
    }
    CK(c, cudaStreamSynchronize(q));   // the host arrays may be released on return
    *slot_out = (uint32_t)st->slots.size();
    st->slots.push_back(s);
    return ESAT_OK;
}

int esat_store_download(esat_store* st, uint32_t slot, uint32_t* sym, uint32_t* koff, uint32_t* kids, uint32_t* cid,
                        double* cost, uint32_t* parent, uint8_t* rank) {
    if (!st || slot >= st->slots.size()) return ESAT_E_ARG;
    esat_ctx* c = st->ctx;
    cudaSetDevice(c->device);
    const esat_store::Slot& s = st->slots[slot];
    cudaStream_t q = c->stream;
    if (sym && s.n) CK(c, cudaMemcpyAsync(sym, st->sym + s.on, 4ull * s.n, cudaMemcpyDeviceToHost, q));
    if (cid && s.n) CK(c, cudaMemcpyAsync(cid, st->cid + s.on, 4ull * s.n, cudaMemcpyDeviceToHost, q));
    if (cost && s.n) CK(c, cudaMemcpyAsync(cost, st->cost + s.on, 8ull * s.n, cudaMemcpyDeviceToHost, q));
    if (koff) CK(c, cudaMemcpyAsync(koff, st->koff + s.of, 4ull * (s.n + 1), cudaMemcpyDeviceToHost, q));
    if (kids && s.K) CK(c, cudaMemcpyAsync(kids, st->kids + s.ok, 4ull * s.K, cudaMemcpyDeviceToHost, q));
    if (parent && s.U) CK(c, cudaMemcpyAsync(parent, st->parent + s.ou, 4ull * s.U, cudaMemcpyDeviceToHost, q));
    if (rank && s.U) CK(c, cudaMemcpyAsync(rank, st->rank + s.ou, s.U, cudaMemcpyDeviceToHost, q));
    CK(c, cudaStreamSynchronize(q));
    return ESAT_OK;
}

int esat_batch_load_slots(esat_batch* b, esat_store* st, const uint32_t* slots) {
    if (!b || !st || b->ctx != st->ctx || (b->L && !slots)) return ESAT_E_ARG;
    esat_ctx* c = b->ctx;
    cudaSetDevice(c->device);
    std::vector<SlotJob> jobs(b->L);
    std::vector<uint32_t> ncnt(b->L), ucnt(b->L), root(b->L);
    for (uint32_t l = 0; l < b->L; l++) {
        if (slots[l] >= st->slots.size()) return fail(c, ESAT_E_ARG, "slot %u out of range", slots[l]);
        const esat_store::Slot& s = st->slots[slots[l]];
        if (s.n > b->nb[l + 1] - b->nb[l] || s.K > b->kb[l + 1] - b->kb[l] || s.U > b->ub[l + 1] - b->ub[l])
            return fail(c, ESAT_E_ARG, "leaf %u: slot %u exceeds the arena span", l, slots[l]);
        jobs[l] = SlotJob{l, s.n, s.K, s.U, s.on, s.of, s.ok, s.ou};
        ncnt[l] = s.n; ucnt[l] = s.U; root[l] = s.root;
    }
    cudaStream_t q = c->stream;
    const uint64_t N = b->N, K = b->K, U = b->U, L = b->L;
    // unused span entries are zero, as in a host pack (arena.py pack_with_headroom)
    CK(c, cudaMemsetAsync((void*)b->d.hc_sym, 0, 4 * N, q));
    CK(c, cudaMemsetAsync((void*)b->d.hc_koff, 0, 4 * (N + L), q));
    CK(c, cudaMemsetAsync((void*)b->d.hc_kids, 0, 4 * K, q));
    CK(c, cudaMemsetAsync((void*)b->d.hc_cid, 0, 4 * N, q));
    CK(c, cudaMemsetAsync((void*)b->d.hc_cost, 0, 8 * N, q));
    CK(c, cudaMemsetAsync((void*)b->d.uf_parent_in, 0, 4 * U, q));
    CK(c, cudaMemsetAsync((void*)b->d.uf_rank_in, 0, U, q));
    CK(c, cudaMemcpyAsync((void*)b->d.root, root.data(), 4 * L, cudaMemcpyHostToDevice, q));
    int r;
    if (L) {
        if ((r = store_jobs(st, jobs))) return r;
        k_store_copy<false><<<b->L, 256, 0, q>>>(
            b->d, reinterpret_cast<const SlotJob*>(st->d_job), st->sym, st->koff, st->kids, st->cid, st->cost,
            st->parent, st->rank, const_cast<uint32_t*>(b->d.hc_sym), const_cast<uint32_t*>(b->d.hc_koff),
            const_cast<uint32_t*>(b->d.hc_kids), const_cast<uint32_t*>(b->d.hc_cid), const_cast<double*>(b->d.hc_cost),
            const_cast<uint32_t*>(b->d.uf_parent_in), const_cast<uint8_t*>(b->d.uf_rank_in));
        if ((r = launch_check(c, "k_store_copy"))) return r;
    }
    b->uploaded = true;
    b->rebuilt = false;
    b->upload_gen++;
    return esat_batch_set_counts(b, ncnt.data(), ucnt.data());   // synchronises the stream
}

}  // extern "C"

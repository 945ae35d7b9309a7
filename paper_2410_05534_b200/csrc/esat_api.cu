// C ABI of libesat_b200 (declared in include/esat_b200.h): context, batch arena, launches.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../include/esat_b200.h"
#include "esat_internal.cuh"

namespace esat {
template <int T> __global__ void k_rebuild(Dev);
template <int T> __global__ void k_extract(Dev, XArgs);
}  // namespace esat

using namespace esat;

struct esat_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    bool timed = false;
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
    double pool_factor = 8.0;
    std::vector<uint64_t> pb;
    uint64_t pool_total = 0;
    uint64_t* d_pb = nullptr;
    uint32_t* pool_key = nullptr;
    double* pool_val = nullptr;
};

namespace {

template <typename T>
int own(esat_batch* b, T** p, size_t n) {
    *p = nullptr;
    CK(b->ctx, cudaMalloc((void**)p, sizeof(T) * (n ? n : 1)));
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
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    if (c->stream) cudaStreamDestroy(c->stream);
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
        uint64_t n = nb[l + 1] - nb[l], t = 2;
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
    OWN(x.status, L); OWN(x.err_class, L); OWN(x.passes, L); OWN(x.root_cost, L);
    OWN(x.class_cost, N); OWN(x.prev, N); OWN(x.choice, N); OWN(x.level, N); OWN(x.order, N); OWN(x.lvcnt, NL);
    OWN(x.stk, N); OWN(x.stki, N); OWN(x.reach, N);
    OWN(x.hoff, 2 * N); OWN(x.hlen, 2 * N);
    x.slot_stride = N;
    *out = b;
    return ESAT_OK;
}

int esat_batch_destroy(esat_batch* b) {
    if (!b) return ESAT_OK;
    cudaSetDevice(b->ctx->device);
    for (void* p : b->owned) cudaFree(p);
    cudaFree(b->d_pb); cudaFree(b->pool_key); cudaFree(b->pool_val);
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
    CK(c, cudaMemcpyAsync(b->d.uf_parent, parent, 4 * U, cudaMemcpyHostToDevice, s));
    CK(c, cudaMemcpyAsync(b->d.uf_rank, rank, U, cudaMemcpyHostToDevice, s));
    CK(c, cudaMemcpyAsync((void*)b->d.root, root, 4 * L, cudaMemcpyHostToDevice, s));
    b->uploaded = true;
    b->rebuilt = false;
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
    b->pool_total = 0;  // force re-allocation on the next OCF extraction
    return ESAT_OK;
}

static int ensure_pool(esat_batch* b) {
    esat_ctx* c = b->ctx;
    if (b->pool_total) return ESAT_OK;
    b->pb.assign(b->L + 1, 0);
    for (uint32_t l = 0; l < b->L; l++) {
        const uint64_t n = b->nb[l + 1] - b->nb[l];
        b->pb[l + 1] = b->pb[l] + (uint64_t)(b->pool_factor * (double)n) + 64;
    }
    b->pool_total = b->pb[b->L];
    cudaFree(b->d_pb); cudaFree(b->pool_key); cudaFree(b->pool_val);
    b->d_pb = nullptr; b->pool_key = nullptr; b->pool_val = nullptr;
    CK(c, cudaMalloc((void**)&b->d_pb, 8ull * (b->L + 1)));
    CK(c, cudaMemcpy(b->d_pb, b->pb.data(), 8ull * (b->L + 1), cudaMemcpyHostToDevice));
    CK(c, cudaMalloc((void**)&b->pool_key, 2 * 4ull * b->pool_total));
    CK(c, cudaMalloc((void**)&b->pool_val, 2 * 8ull * b->pool_total));
    return ESAT_OK;
}

int esat_extract(esat_batch* b, int method) {
    if (!b || (method != ESAT_METHOD_DEFAULT && method != ESAT_METHOD_OCF)) return ESAT_E_ARG;
    esat_ctx* c = b->ctx;
    if (!b->rebuilt) return fail(c, ESAT_E_STATE, "extraction requires a rebuilt e-graph");
    cudaSetDevice(c->device);
    XArgs x = b->x;
    x.method = method;
    if (method == ESAT_METHOD_OCF) {
        int r = ensure_pool(b);
        if (r) return r;
        x.pool_base = b->d_pb;
        x.pool_key = b->pool_key;
        x.pool_val = b->pool_val;
        x.pool_stride = b->pool_total;
    }
    tic(c);
    if (b->L) k_extract<128><<<b->L, 128, 0, c->stream>>>(b->d, x);
    toc(c);
    return launch_check(c, "k_extract");
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

int esat_result_device_ptrs(esat_batch* b, void** root_cost, void** status) {
    if (!b) return ESAT_E_ARG;
    if (root_cost) *root_cost = b->x.root_cost;
    if (status) *status = b->x.status;
    return ESAT_OK;
}

}  // extern "C"

// ---- e-matching entry points: implemented in k_ematch.cu (weak stubs until linked) ----
extern "C" {
__attribute__((weak)) int esat_ematch(esat_batch* b, uint32_t, const uint32_t*, int) {
    return b ? fail(b->ctx, ESAT_E_STATE, "esat_ematch not built") : ESAT_E_ARG;
}
__attribute__((weak)) int esat_join(esat_batch* b, uint32_t, const uint32_t*, const uint32_t*, const uint32_t*,
                                    const uint32_t*, const uint32_t*, const uint32_t*, const uint32_t*) {
    return b ? fail(b->ctx, ESAT_E_STATE, "esat_join not built") : ESAT_E_ARG;
}
__attribute__((weak)) int esat_download_matches(esat_batch* b, int, uint32_t, uint32_t*, uint64_t*, uint32_t*,
                                                uint64_t) {
    return b ? fail(b->ctx, ESAT_E_STATE, "esat_download_matches not built") : ESAT_E_ARG;
}
}

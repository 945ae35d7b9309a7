// K12: EGraph.fingerprint (egraph.py:247-296) for every leaf of a rebuilt batch -- the
// Weisfeiler-Lehman class refinement whose 64-bit result keys the MCTS extraction cache
// (SURVEY §8(f)2). Bit-exact: labels are BLAKE2b-64 digests (egraph.py:124-129) of the very
// bytes Python's repr() produces for the sorted tuples the reference hashes, so the device
// streams those bytes into its own BLAKE2b instead of building Python objects:
//   label0(c)   = H(repr(sorted(symbol.key() of c's nodes)))
//   label_r(c)  = H(repr(sorted((symbol.key(), (label_{r-1}(child), ...)) for c's nodes)))
// until the induced partition (class -> smallest class id with the same label) repeats, at most
// max(1, C) rounds; then fp = H(repr(sorted(sorted descriptions per class)), repr(root label)).
// symbol.key() is (name, arity, repr(payload)); its repr bytes and its rank among all keys
// (Python tuple order) come from the host (fingerprint.py).
//
// Schedule: one CTA per leaf. Per round a thread owns a class (sorts its node descriptions,
// streams their repr into BLAKE2b); the partition is recomputed with an atomicMin hash table
// keyed by label; the final class order is a CTA bitonic sort with the list comparator, and one
// thread streams the body.
#include "esat_internal.cuh"
#include "k_fingerprint_args.cuh"

namespace esat {

namespace {

__constant__ uint64_t B2B_IV[8] = {0x6a09e667f3bcc908ull, 0xbb67ae8584caa73bull, 0x3c6ef372fe94f82bull,
                                   0xa54ff53a5f1d36f1ull, 0x510e527fade682d1ull, 0x9b05688c2b3e6c1full,
                                   0x1f83d9abfb41bd6bull, 0x5be0cd19137e2179ull};
__device__ __forceinline__ uint64_t rotr(uint64_t x, int n) { return (x >> n) | (x << (64 - n)); }

struct B2b {   // streaming BLAKE2b with an 8-byte digest (hashlib.blake2b(digest_size=8))
    uint64_t h[8];
    // two message blocks as little-endian words: the block being filled (at word `cur`) and at most
    // one full block whose compression is deferred to the caller's next flush() -- lanes of a warp
    // hashing different classes then compress together at the same program point instead of each
    // at its own byte position (SIMT efficiency of the dominant compression)
    uint64_t m[32];
    uint64_t t;       // bytes in the stream up to the end of the last full block
    uint64_t tp;      // counter of the pending block
    uint64_t acc;     // bytes of the word being filled
    uint32_t n;       // bytes in the current block (including acc)
    uint32_t cur;     // 0 or 16: first word of the block being filled
    bool pend;        // the other block is full and not yet compressed

    __device__ void init() {
        for (int i = 0; i < 8; i++) h[i] = B2B_IV[i];
        h[0] ^= 0x01010008ull;
        t = 0;
        n = 0;
        acc = 0;
        cur = 0;
        pend = false;
    }
    __device__ __noinline__ void compress(uint32_t base, uint64_t tt, bool last) {
        // the 12 rounds written out with the BLAKE2b sigma schedule as literals: the message words
        // are read once into registers and every schedule index is a register name (m itself stays
        // addressable for put); one out-of-line copy keeps the kernel's code small
        uint64_t mm[16];
#pragma unroll
        for (int i = 0; i < 16; i++) mm[i] = m[base + i];
        uint64_t v[16];
#pragma unroll
        for (int i = 0; i < 8; i++) { v[i] = h[i]; v[i + 8] = B2B_IV[i]; }
        v[12] ^= tt;
        if (last) v[14] = ~v[14];
#define B2G(a, b, c, d, x, y)                         \
    v[a] = v[a] + v[b] + x; v[d] = rotr(v[d] ^ v[a], 32); \
    v[c] = v[c] + v[d];     v[b] = rotr(v[b] ^ v[c], 24); \
    v[a] = v[a] + v[b] + y; v[d] = rotr(v[d] ^ v[a], 16); \
    v[c] = v[c] + v[d];     v[b] = rotr(v[b] ^ v[c], 63);
#define B2R(s0, s1, s2, s3, s4, s5, s6, s7, s8, s9, s10, s11, s12, s13, s14, s15) \
    B2G(0, 4, 8, 12, mm[s0], mm[s1]) B2G(1, 5, 9, 13, mm[s2], mm[s3])             \
    B2G(2, 6, 10, 14, mm[s4], mm[s5]) B2G(3, 7, 11, 15, mm[s6], mm[s7])           \
    B2G(0, 5, 10, 15, mm[s8], mm[s9]) B2G(1, 6, 11, 12, mm[s10], mm[s11])         \
    B2G(2, 7, 8, 13, mm[s12], mm[s13]) B2G(3, 4, 9, 14, mm[s14], mm[s15])
        B2R(0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15)
        B2R(14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3)
        B2R(11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4)
        B2R(7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8)
        B2R(9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13)
        B2R(2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9)
        B2R(12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11)
        B2R(13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10)
        B2R(6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5)
        B2R(10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0)
        B2R(0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15)
        B2R(14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3)
#undef B2R
#undef B2G
#pragma unroll
        for (int i = 0; i < 8; i++) h[i] ^= v[i] ^ v[i + 8];
    }
    // k (1..8) bytes packed little-endian in v (first byte in the low bits): the stream is filled a
    // word at a time (one shift-or per word, the spill carried into the next word) instead of bytewise
    __device__ __forceinline__ void putw(uint64_t v, uint32_t k) {
        while (k) {
            if (n == 128) {   // a full block is compressed only once more data follows (BLAKE2b rule)
                t += 128;
                if (pend) compress(cur ^ 16, tp, false);   // blocks compress in stream order
                pend = true;
                tp = t;
                cur ^= 16;
                n = 0;
            }
            const uint32_t room = 128 - n, take = k < room ? k : room, sh = n & 7;
            const uint64_t part = take == 8 ? v : (v & ((1ull << (8 * take)) - 1));
            acc |= part << (8 * sh);
            if (sh + take >= 8) {
                m[cur + (n >> 3)] = acc;
                acc = sh ? part >> (8 * (8 - sh)) : 0;
            }
            n += take;
            v = take == 8 ? 0 : v >> (8 * take);
            k -= take;
        }
    }
    __device__ __forceinline__ void put(uint8_t c) { putw(c, 1); }
    // len bytes from s; the buffer is readable (not necessarily meaningful) up to the next 8-byte
    // boundary past s + len + 8, so whole aligned words are read and funnel-shifted
    __device__ void putb(const uint8_t* s, uint32_t len) {
        if (!len) return;
        const uint32_t mis = (uint32_t)((uintptr_t)s & 7);
        const uint64_t* w = (const uint64_t*)(s - mis);
        uint64_t lo = __ldg(w);
        for (uint32_t i = 0; i < len; i += 8) {
            const uint64_t hi = __ldg(++w);
            const uint64_t v = mis ? (lo >> (8 * mis)) | (hi << (8 * (8 - mis))) : lo;
            putw(v, len - i < 8 ? len - i : 8);
            lo = hi;
        }
    }
    // the 8 low decimal digits of r (< 1e8), zero-padded, most significant digit in the low byte
    static __device__ __forceinline__ uint64_t dig8(uint32_t r) {
        uint64_t w = 0;
#pragma unroll
        for (int i = 0; i < 8; i++) { w = (w << 8) | (uint64_t)('0' + r % 10u); r /= 10u; }
        return w;
    }
    __device__ __forceinline__ void putu_head(uint32_t r) {   // r < 1e8 without leading zeros
        uint32_t k = 1;
        for (uint32_t p = 10; k < 8 && r >= p; p *= 10) k++;
        putw(dig8(r) >> (8 * (8 - k)), k);
    }
    __device__ void putu(uint64_t x) {   // decimal repr of a non-negative int, 8 digits per word
        if (x < 100000000ull) { putu_head((uint32_t)x); return; }
        const uint32_t lo = (uint32_t)(x % 100000000ull);
        x /= 100000000ull;
        if (x < 100000000ull) {
            putu_head((uint32_t)x);
        } else {
            putu_head((uint32_t)(x / 100000000ull));
            putw(dig8((uint32_t)(x % 100000000ull)), 8);
        }
        putw(dig8(lo), 8);
    }
    // int.from_bytes(digest, "big"): the digest is h[0] little-endian
    // compresses the deferred full block, if any; call where the lanes of a warp are converged
    __device__ __forceinline__ void flush() {
        if (pend) {
            compress(cur ^ 16, tp, false);
            pend = false;
        }
    }
    __device__ uint64_t final() {
        flush();
        t += n;
        if (n & 7) m[cur + (n >> 3)] = acc;
        for (uint32_t w = (n + 7) >> 3; w < 16; w++) m[cur + w] = 0;
        compress(cur, t, true);
        return __byte_perm((uint32_t)(h[0] >> 32), 0, 0x0123) | ((uint64_t)__byte_perm((uint32_t)h[0], 0, 0x0123) << 32);
    }
};

struct Leaf {
    const Dev* d;
    const FArgs* a;
    uint32_t C;
    const uint32_t *coff, *nko, *kpos, *nsym;
};

// description order of two nodes: (symbol key rank, child labels lexicographic)
__device__ __forceinline__ bool desc_less(const Leaf& L, const unsigned long long* lab, uint32_t x, uint32_t y) {
    const uint32_t sx = L.nsym[x], sy = L.nsym[y];
    const uint32_t rx = L.a->krank[sx], ry = L.a->krank[sy];
    if (rx != ry) return rx < ry;
    const uint32_t qx = L.nko[x], ax = L.nko[x + 1] - qx, qy = L.nko[y], ay = L.nko[y + 1] - qy;
    const uint32_t m = ax < ay ? ax : ay;
    for (uint32_t i = 0; i < m; i++) {
        const uint64_t lx = lab[L.kpos[qx + i]], ly = lab[L.kpos[qy + i]];
        if (lx != ly) return lx < ly;
    }
    return ax < ay;
}

// sorts class c's nodes by description into ord[] (the class's own span of nord); returns the count
__device__ uint32_t sorted_nodes(const Leaf& L, const unsigned long long* lab, uint32_t c, uint32_t* ord, bool with_labels) {
    const uint32_t n0 = L.coff[c], nn = L.coff[c + 1] - n0;
    for (uint32_t i = 0; i < nn; i++) {
        const uint32_t x = n0 + i;
        uint32_t j = i;
        while (j > 0) {
            const uint32_t y = ord[j - 1];
            const bool lt = with_labels ? desc_less(L, lab, x, y) : L.a->krank[L.nsym[x]] < L.a->krank[L.nsym[y]];
            if (!lt) break;
            ord[j] = y;
            j--;
        }
        ord[j] = x;
    }
    return nn;
}

__device__ void put_key(const Leaf& L, B2b& h, uint32_t sym) {
    const uint32_t o = L.a->key_off[sym], e = L.a->key_off[sym + 1];
    h.putb(L.a->key_bytes + o, e - o);
}

// repr((symbol.key(), (label, ...)))
// decimal repr of x as bytes in o[0..2] (first character in the low byte) and its length in o[3]; a
// label is printed once per parent reference but converted once per round
__device__ void store_dec(uint64_t x, unsigned long long* o) {
    uint64_t w[3] = {0, 0, 0};
    uint32_t n = 0;
    auto add = [&](uint64_t v, uint32_t k) {   // k <= 8 bytes, n + k <= 20
        const uint32_t sh = n & 7;
        const uint64_t lo = v << (8 * sh), hi = sh ? v >> (8 * (8 - sh)) : 0;
        if (n < 8) { w[0] |= lo; w[1] |= hi; } else if (n < 16) { w[1] |= lo; w[2] |= hi; } else { w[2] |= lo; }
        n += k;
    };
    auto head = [&](uint32_t r) {
        uint32_t k = 1;
        for (uint32_t p = 10; k < 8 && r >= p; p *= 10) k++;
        add(B2b::dig8(r) >> (8 * (8 - k)), k);
    };
    if (x < 100000000ull) {
        head((uint32_t)x);
    } else {
        const uint32_t lo = (uint32_t)(x % 100000000ull);
        x /= 100000000ull;
        if (x < 100000000ull) {
            head((uint32_t)x);
        } else {
            head((uint32_t)(x / 100000000ull));
            add(B2b::dig8((uint32_t)(x % 100000000ull)), 8);
        }
        add(B2b::dig8(lo), 8);
    }
    o[0] = w[0]; o[1] = w[1]; o[2] = w[2]; o[3] = n;
}

__device__ __forceinline__ void put_dec(B2b& h, const unsigned long long* o) {
    const uint32_t len = (uint32_t)o[3];
    h.putw(o[0], len < 8 ? len : 8);
    if (len > 8) h.putw(o[1], len < 16 ? len - 8 : 8);
    if (len > 16) h.putw(o[2], len - 16);
}

__device__ void put_desc(const Leaf& L, B2b& h, const unsigned long long* dec, uint32_t x) {
    h.put('(');
    put_key(L, h, L.nsym[x]);
    h.putw(0x28202cull, 3);   // ", ("
    const uint32_t q = L.nko[x], ar = L.nko[x + 1] - q;
    for (uint32_t i = 0; i < ar; i++) {
        if (i) h.putw(0x202cull, 2);   // ", "
        put_dec(h, dec + 4ull * L.kpos[q + i]);
    }
    if (ar == 1) h.put(',');
    h.putw(0x2929ull, 2);   // "))"
}

__device__ bool class_less(const Leaf& L, const unsigned long long* lab, const uint32_t* nord, uint32_t a, uint32_t b) {
    const uint32_t na = L.coff[a + 1] - L.coff[a], nb = L.coff[b + 1] - L.coff[b];
    const uint32_t m = na < nb ? na : nb;
    for (uint32_t i = 0; i < m; i++) {
        const uint32_t x = nord[L.coff[a] + i], y = nord[L.coff[b] + i];
        if (desc_less(L, lab, x, y)) return true;
        if (desc_less(L, lab, y, x)) return false;
    }
    return na < nb;
}

}  // namespace

template <int T>
__global__ void __launch_bounds__(T, 1024 / T) k_fingerprint(Dev d, FArgs a) {
    const uint32_t l = blockIdx.x, tid = threadIdx.x;
    const uint64_t b = d.nb[l], t0 = d.tb[l];
    Leaf L;
    L.d = &d; L.a = &a;
    L.C = d.v_C[l];
    L.coff = d.cls_off + b + l;
    L.nko = d.nd_koff + b + l;
    L.kpos = d.nd_kpos + d.kb[l];
    L.nsym = d.nd_sym + b;
    const uint32_t C = L.C;
    unsigned long long* lab[2] = {a.lab0 + b, a.lab1 + b};
    uint32_t* rep[2] = {a.rep0 + b, a.rep1 + b};
    uint32_t* nord = a.nord + b;
    uint8_t* lchg = a.lchg + b;
    unsigned long long* dec[2] = {a.dec0 + 4 * b, a.dec1 + 4 * b};
    const uint32_t tsz = (uint32_t)(d.tb[l + 1] - t0), tmask = tsz - 1;
    unsigned long long* tkey = a.tkey + t0;
    uint32_t* tval = a.tval + t0;
    __shared__ uint32_t sh_bad, sh_changed, sh_next;
    if (tid == 0) { sh_bad = 0; sh_next = T; }
    __syncthreads();
    // round 0: labels from the sorted symbol keys
    for (uint32_t c = tid; c < C; c += T) {
        uint32_t* ord = nord + L.coff[c];
        const uint32_t nn = sorted_nodes(L, nullptr, c, ord, false);
        B2b h;
        h.init();
        h.put('[');
        for (uint32_t i = 0; i < nn; i++) {
            if (i) h.putw(0x202cull, 2);   // ", "
            put_key(L, h, L.nsym[ord[i]]);
            h.flush();
        }
        h.put(']');
        h.put(0x1f);
        lab[0][c] = h.final();
        store_dec(lab[0][c], dec[0] + 4ull * c);
        rep[0][c] = NONE;
    }
    __syncthreads();
    int cur = 0;
    const uint32_t rounds = C > 1 ? C : 1;
    for (uint32_t it = 0; it < rounds && !sh_bad; it++) {
        const unsigned long long* lc = lab[cur];
        unsigned long long* ln = lab[cur ^ 1];
        // classes handed out dynamically, so a few big ones no longer stall the end-of-round barrier
        for (uint32_t c = tid; c < C; c = atomicAdd(&sh_next, 1u)) {
            // From the second refinement on, a class none of whose children changed label in the last
            // round hashes exactly the bytes it hashed then, so its label carries over.
            if (it > 0) {
                bool dirty = false;
                for (uint32_t nd = L.coff[c]; nd < L.coff[c + 1] && !dirty; nd++)
                    for (uint32_t q = L.nko[nd]; q < L.nko[nd + 1]; q++)
                        if (lchg[L.kpos[q]]) { dirty = true; break; }
                if (!dirty) {
                    ln[c] = lc[c];
                    for (int w = 0; w < 4; w++) dec[cur ^ 1][4ull * c + w] = dec[cur][4ull * c + w];
                    continue;
                }
            }
            uint32_t* ord = nord + L.coff[c];
            const uint32_t nn = sorted_nodes(L, lc, c, ord, true);
            B2b h;
            h.init();
            h.put('[');
            for (uint32_t i = 0; i < nn; i++) {
                if (i) h.putw(0x202cull, 2);   // ", "
                put_desc(L, h, dec[cur], ord[i]);
                h.flush();
            }
            h.put(']');
            h.put(0x1f);
            ln[c] = h.final();
            store_dec(ln[c], dec[cur ^ 1] + 4ull * c);
        }
        for (uint32_t s = tid; s < tsz; s += T) { tkey[s] = ~0ull; tval[s] = NONE; }
        if (tid == 0) sh_changed = 0;
        __syncthreads();
        // partition: every class -> smallest class position (= smallest id) with its label
        for (uint32_t c = tid; c < C; c += T) {
            const unsigned long long key = ln[c];
            lchg[c] = key != lc[c];
            uint32_t s = (uint32_t)(mix64(key) & tmask);
            while (true) {
                const unsigned long long prev = atomicCAS(&tkey[s], ~0ull, key);
                if (prev == ~0ull || prev == key) break;
                s = (s + 1) & tmask;
            }
            atomicMin(&tval[s], c);
        }
        __syncthreads();
        uint32_t* rp = rep[cur ^ 1];
        const uint32_t* rq = rep[cur];
        for (uint32_t c = tid; c < C; c += T) {
            const unsigned long long key = ln[c];
            uint32_t s = (uint32_t)(mix64(key) & tmask);
            while (tkey[s] != key) s = (s + 1) & tmask;
            rp[c] = tval[s];
            if (it == 0 || rp[c] != rq[c]) sh_changed = 1;   // the first partition never matches None
        }
        __syncthreads();
        cur ^= 1;
        const bool stop = !sh_changed;
        if (tid == 0) sh_next = T;
        __syncthreads();
        if (stop) break;
    }
    if (sh_bad) {
        if (tid == 0) { a.status[l] = 1; a.fp[l] = 0; }
        return;
    }
    // body: classes sorted by their sorted descriptions (final labels)
    const unsigned long long* lf = lab[cur];
    for (uint32_t c = tid; c < C; c += T) sorted_nodes(L, lf, c, nord + L.coff[c], true);
    uint32_t P = 1;
    while (P < C) P <<= 1;
    uint32_t* cord = a.cord + t0;   // tb rows: >= 2n >= P
    for (uint32_t i = tid; i < P; i += T) cord[i] = i < C ? i : NONE;
    __syncthreads();
    for (uint32_t k = 2; k <= P; k <<= 1)
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = tid; i < P; i += T) {
                const uint32_t p = i ^ j;
                if (p <= i) continue;
                const uint32_t x = cord[i], y = cord[p];
                const bool up = (i & k) == 0;
                // NONE (padding) sorts last
                const bool gt = x == NONE ? y != NONE : (y != NONE && class_less(L, lf, nord, y, x));
                if (gt == up) { cord[i] = y; cord[p] = x; }
            }
            __syncthreads();
        }
    if (tid == 0) {
        B2b h;
        h.init();
        h.put('[');
        for (uint32_t i = 0; i < C; i++) {
            const uint32_t c = cord[i];
            if (i) h.putw(0x202cull, 2);   // ", "
            h.put('[');
            for (uint32_t q = L.coff[c]; q < L.coff[c + 1]; q++) {
                if (q != L.coff[c]) h.putw(0x202cull, 2);   // ", "
                put_desc(L, h, dec[cur], nord[q]);
            }
            h.put(']');
        }
        h.put(']');
        h.put(0x1f);
        const uint32_t rp = d.v_root[l];
        if (rp == NONE) h.putw(0x656e6f4eull, 4);   // "None"
        else h.putu(lf[rp]);
        h.put(0x1f);
        a.fp[l] = h.final();
        a.status[l] = 0;
    }
}

template __global__ void k_fingerprint<256>(Dev, FArgs);

}  // namespace esat

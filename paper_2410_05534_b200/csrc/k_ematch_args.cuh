// Launch arguments of k_ematch / k_join (k_ematch.cu), shared with esat_api.cu.
#pragma once
#include "esat_internal.cuh"

namespace esat {

constexpr int MAX_PN = 16;   // pattern nodes (larger patterns are rejected with ESAT_E_ARG)
constexpr int MAX_V = 8;     // vars / pvars per pattern
constexpr int MAX_W = 24;    // words per record
constexpr int MAX_S = 4;     // sources per multi-pattern rule

struct MArgs {
    const int32_t* prog;        // all pattern programs
    const uint32_t* prog_off;   // [n_patterns_total + 1]
    const uint32_t* pat_ids;    // patterns of this call [P]
    uint32_t P;
    int mode;                   // 0 list, 1 exists
    uint32_t* stage;
    uint64_t stage_cap;
    unsigned long long* tops;   // [0] stage top, [1] out top (words)
    uint32_t* out;
    uint64_t out_cap;
    uint32_t* count;            // [P][L] (this launch's chunk of the call's rows)
    uint64_t* off;              // [P][L] word offsets into out
    uint32_t* overflow;
    uint32_t smem_bytes;        // dynamic shared memory for staging one leaf's view
    uint32_t* raw;              // [L][32][T] per-thread raw match counts (count -> fill placement)
    uint32_t* nzl;              // [L][32][C] (pattern, class) pairs with matches (pass-2 work list)
    int no_flat;                // 1: always use the generic backtracking matcher
    const uint32_t* leaf_mask;  // [L] bit p: match chunk-pattern p on this leaf (nullptr: all)
};

struct JArgs {
    uint32_t R;
    const uint32_t *src_off, *src, *map_off, *vmap, *qmap, *nv, *nq;
    // single-pattern inputs (from the last k_ematch call)
    const uint32_t* m_count;
    const uint64_t* m_off;
    const uint32_t* m_words;
    const uint32_t* m_W;        // words per record of call-pattern p
    uint32_t* stage;
    uint64_t stage_cap;
    unsigned long long* tops;
    uint32_t* out;
    uint64_t out_cap;
    uint32_t* count;            // [R][L]
    uint64_t* off;
    uint32_t* overflow;
    const uint64_t* id_base;    // per-leaf id bases (run-table size)
    uint32_t run_cap;           // dynamic SMEM run-table entries
    uint32_t s1_cap;            // dynamic SMEM words for the staged source-1 fields (after the run table)
    uint32_t* gsort;            // [R][L][warps][JOIN_GSORT_WORDS] root-group merge scratch
    unsigned long long* gkeys;  // global index scratch for source-1 lists beyond the SMEM index
    uint64_t gkey_cap;          //   (bump-allocated through tops[0]; overflow bit 4 -> regrow)
    unsigned long long* big;    // [R][L][2] long-list pairs: scratch offsets of (index, record table); ~0 = none
};

#ifndef ESAT_JOIN_S1
#define ESAT_JOIN_S1 2048
#endif
constexpr uint32_t JOIN_SMEM_S1 = ESAT_JOIN_S1;   // SMEM words for staged source-1 join fields (2048: 7 CTAs per SM; 4096 measured 11-15 % slower joins, 1024 unstages NasRNN)
constexpr uint32_t JOIN_GSORT_WORDS = 1024; // per-warp words for merging a root group's product runs

template <int T> __global__ void k_ematch(Dev, MArgs);
template <int T> __global__ void k_join(uint32_t, JArgs);
template <int T> __global__ void k_join_big(uint32_t, JArgs);

}  // namespace esat

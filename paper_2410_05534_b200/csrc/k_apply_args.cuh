// Launch arguments of k_apply (K11, the device apply loop).
#pragma once
#include <cstdint>

namespace esat {

constexpr uint32_t NO_MATCH_CODE_U = 0x3FFFFFFFu;   // symtab.NO_MATCH_CODE

enum : uint32_t { A_OK = 0, A_NODE_LIMIT = 1, A_NEED_SYMBOL = 2, A_CAPACITY = 3, A_PROGRAM = 4 };

struct AArgs {
    // rule target programs (apply.py) and the rule each leaf applies (NONE: none)
    const int32_t* prog;
    const uint32_t* rule_off;
    const uint32_t* leaf_rule;
    // symbols: shapes, identity-key hash table, attribute integer values by code
    const uint8_t* sym_ndim;
    const uint32_t* sym_dims;     // [n_syms][4]
    const uint32_t* sym_table;
    uint32_t sym_tmask;
    const int32_t* val_int;
    uint32_t n_values;
    int lang;                      // 0 TermLanguage, 1 TensorLanguage
    int cost_mode;                 // 0 term (1.0), 1 unit, 2 analytic
    double coeff;
    uint32_t node_limit;
    // match lists of the last e-match / join calls
    const uint32_t* m_words;
    const uint64_t* m_off;
    const uint32_t* m_count;
    const uint32_t* j_words;
    const uint64_t* j_off;
    const uint32_t* j_count;
    // outputs: the leaf's dirty state (batch input arrays) + report
    uint32_t *w_sym, *w_koff, *w_kids, *w_cid;
    double* w_cost;
    uint32_t* w_parent;
    uint8_t* w_rank;
    uint32_t *status, *report, *missing;   // report [L][4]: matches_found, changed, cycles, shapes
    // scratch
    uint32_t *s_head, *s_tail, *s_next, *s_seen, *s_stack;
    // cycle-test potentials: pot[U], parent-edge lists phead/ptail[U] over child slots pnext/eown[K],
    // Kahn pending counts pend[U]
    uint32_t *s_pot, *s_phead, *s_ptail, *s_pend, *s_pnext, *s_eown;
    uint32_t sel_lo, sel_hi;   // the launch handles leaves whose rule has a match count in [sel_lo, sel_hi)
    int no_pot;   // 1: plain BFS without potential pruning (env ESAT_APPLY_NO_POT; for measurement)
};

template <int NW>
__global__ void k_apply(Dev d, AArgs a);

}  // namespace esat

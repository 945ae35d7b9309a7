/*
 * esat_b200 -- C ABI of the B200-native (sm_100a) hot path of the MCTS-guided
 * equality-saturation optimizer (arXiv 2410.05534; reference = /root/reference/pkg/src/esat).
 *
 * The reference's boundary for this path is a pure-Python function-level API (no plugin
 * registry or FFI exists). Each entry point below replaces one reference
 * function, batched over many e-graph "leaves" (MCTS leaves / rollout states):
 *
 *   esat_rebuild       <- EGraph.rebuild                 egraph.py:203-238 (+ _regroup)
 *   esat_ematch        <- ematch / joint_match (1 source) rewrite.py:400-433
 *   esat_ematch(EXISTS)<- is_rule_applicable             rewrite.py:579-589
 *   esat_join          <- joint_match (>= 2 sources)      rewrite.py:405-433
 *   esat_extract       <- extract_default_greedy          extraction.py:157-166
 *                         extract_ocf_greedy              extraction.py:229-242
 *                         (+ validate_extraction / _reachable_chosen, extraction.py:67-115)
 *   esat_batch_upload  <- EGraph.snapshot into device slots (egraph.py:300-312)
 *   esat_store_save / esat_batch_load_slots <- EGraph.snapshot kept on the device (D2D)
 *
 * Plain C types only. All functions return ESAT_OK (0) or an ESAT_E_* code; the message
 * is available from esat_last_error(ctx). Threading: one host thread per context (the
 * reference's single-writer contract, egraph.py:133); a context owns one CUDA stream.
 *
 * ---------------------------------------------------------------------------------------
 * Batch arena (host upload format; paper_2410_05534_b200/arena.py):
 *   L leaves; per-leaf bases node_base/kid_base/id_base (uint64, L+1 entries each).
 *   hc_sym  u32[N]   interned symbol per hashcons entry (insertion order = reference order)
 *   hc_koff u32[N+L] CSR child offsets, n+1 leaf-relative entries per leaf at node_base[l]+l
 *   hc_kids u32[K]   child class ids as stored in the entry key
 *   hc_cid  u32[N]   class id stored for the entry
 *   hc_cost f64[N]   operator cost of the node (cost model)
 *   uf_parent u32[U], uf_rank u8[U]   union-find (egraph.py:80-115)
 *   root    u32[L]   raw root id per leaf (0xFFFFFFFF = none)
 *
 * Clean view (written by esat_rebuild, read by ematch/extract), per leaf:
 *   C classes with ascending canonical ids cls_id[C]; cls_off[C+1] node ranges; nodes in
 *   node_sort_key order (egraph.py:65-70) with nd_sym, nd_cost, nd_koff (CSR) and nd_kpos
 *   (children as class POSITIONS); nd_hc maps a view node to its new hashcons entry.
 *
 * Symbol table: name id, arity, rank (order of (name, repr(payload))), attribute codes
 *   (order-preserving ints: ints numerically then strings) -- paper_2410_05534_b200/symtab.py.
 *
 * Pattern program (int32, paper_2410_05534_b200/patterns.py compile_pattern):
 *   [P, V, Q] then P records of 6 words {kind(0 var/1 app), ident(var idx | name id),
 *   arity, nslots(-1 = no attribute spec), slot_off, child_off} (offsets from the program
 *   start), then attribute slots (>=0 literal code, <0 pvar -(q+1)), then child indices.
 *   Var/pvar indices follow sorted names. A match record is W = 1+V+Q u32 words
 *   [root class id][var class ids][pvar codes], sorted ascending and unique per leaf
 *   (rewrite.py:396-397, 420-433).
 */
#ifndef ESAT_B200_H
#define ESAT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ESAT_OK 0
#define ESAT_E_ARG 1          /* bad argument -> ValueError / StructuralError            */
#define ESAT_E_CUDA 2         /* CUDA runtime failure                                    */
#define ESAT_E_CAPACITY 3     /* output/pool capacity exceeded -> grow and retry         */
#define ESAT_E_STATE 4        /* call out of order (e.g. ematch before rebuild): the
                                 reference's "requires a rebuilt e-graph" StructuralError */

/* per-leaf extraction status (esat_extract) -> exception mapping in extraction.py */
#define ESAT_X_OK 0
#define ESAT_X_NOT_CONVERGED 1     /* ExtractionError("greedy extraction failed to converge") */
#define ESAT_X_INFEASIBLE 2        /* InfeasibleExtraction("root e-class has no finite-cost program") */
#define ESAT_X_CYCLIC 3            /* ExtractionError("cyclic selection through e-class %u") */
#define ESAT_X_CHILD_NOT_CHOSEN 4  /* ExtractionError("child e-class %u required but not chosen") */
#define ESAT_X_ROOT_NOT_CHOSEN 5   /* ExtractionError("root e-class not chosen") */
#define ESAT_X_NO_ROOT 6           /* StructuralError("e-graph has no root") */
#define ESAT_X_CAPACITY 7          /* OCF history pool too small: grow and retry; err_class holds the
                                      overflow mask (1: bitset pool, 2: value pool) */

#define ESAT_METHOD_DEFAULT 0
#define ESAT_METHOD_OCF 1

#define ESAT_MATCH_LIST 0
#define ESAT_MATCH_EXISTS 1

typedef struct esat_ctx esat_ctx;
typedef struct esat_batch esat_batch;

/* context: one per GPU per process */
int esat_ctx_create(int device, esat_ctx** out);
int esat_ctx_destroy(esat_ctx* ctx);
const char* esat_last_error(const esat_ctx* ctx);
int esat_ctx_sync(esat_ctx* ctx);

/* symbol table (replaces Symbol interning; egraph.py:34-70, rewrite.py:275-277) */
int esat_symtab_upload(esat_ctx* ctx, uint32_t n_syms, const uint32_t* name_id, const uint32_t* arity,
                       const uint32_t* rank, const uint32_t* param_off, const int32_t* param_codes);

/* pattern programs (compiled from rewrite.py:43-65 patterns) */
int esat_patterns_upload(esat_ctx* ctx, uint32_t n_patterns, const uint32_t* prog_off,
                         uint32_t n_words, const int32_t* prog_words);

/* batches: device-resident leaf arenas */
int esat_batch_create(esat_ctx* ctx, uint32_t n_leaves, const uint64_t* node_base, const uint64_t* kid_base,
                      const uint64_t* id_base, esat_batch** out);
int esat_batch_destroy(esat_batch* b);
int esat_batch_upload(esat_batch* b, const uint32_t* hc_sym, const uint32_t* hc_koff, const uint32_t* hc_kids,
                      const uint32_t* hc_cid, const double* hc_cost, const uint32_t* uf_parent,
                      const uint8_t* uf_rank, const uint32_t* root);

/* EGraph.rebuild over every leaf; per-leaf merge counts stay on device (download below) */
int esat_rebuild(esat_batch* b);

/* e-match patterns[0..n) over every leaf (mode LIST or EXISTS); n <= ESAT_MAX_CALL_PATTERNS
 * (one k_ematch launch per 32-pattern chunk) */
#define ESAT_MAX_CALL_PATTERNS 1024u
int esat_ematch(esat_batch* b, uint32_t n_patterns, const uint32_t* pattern_ids, int mode);
/* the same, with per-leaf pattern masks: ceil(n/32) words per leaf, chunk-major -- bit p of
 * leaf_mask[c * n_leaves + l] selects call-pattern 32c+p on leaf l (0: the leaf is not matched, its
 * counts are 0). An MCTS rollout step matches only the sources of the rule each leaf applies
 * (SPEC.md:603-611); joins of unmatched sources are empty. */
int esat_ematch_masked(esat_batch* b, uint32_t n_patterns, const uint32_t* pattern_ids, int mode,
                       const uint32_t* leaf_mask);
/* joint_match of multi-pattern rules over the LIST results of their source patterns.
 * rule r: n_src[r] sources (pattern ids src[src_off[r]..]); var_map/pvar_map give the output
 * slot of each source var/pvar (sorted combined names); out record = [S roots][NV][NQ]. */
int esat_join(esat_batch* b, uint32_t n_rules, const uint32_t* src_off, const uint32_t* src,
              const uint32_t* map_off, const uint32_t* var_map, const uint32_t* pvar_map,
              const uint32_t* n_vars, const uint32_t* n_pvars);

/* greedy extraction (method DEFAULT or OCF) over every leaf; OCF constituent histories live in a
 * per-leaf pool of entries_per_node * n entries per pass parity (ESAT_X_CAPACITY -> grow, retry) */
int esat_batch_set_pool(esat_batch* b, double entries_per_node);
/* separate sizing of the f64 contribution pool and the bitset pool (ceil(C/32) words per history) */
int esat_batch_set_pool2(esat_batch* b, double values_per_node, double bitsets_per_node);
int esat_extract(esat_batch* b, int method);
/* the same on the context's side stream: extraction only reads the rebuilt view, so it overlaps
 * esat_ematch / esat_join on the main stream; esat_wait_async joins it back (downloads and
 * esat_copy_results join implicitly) */
int esat_extract_async(esat_batch* b, int method);
/* mark the current point of the main stream as the side stream's start (so work issued on the
 * main stream after esat_fork overlaps a later esat_extract_async) */
int esat_fork(esat_ctx* ctx);
int esat_wait_async(esat_ctx* ctx);
float esat_last_async_ms(const esat_ctx* ctx);

/* downloads (host buffers sized from the batch bases) */
int esat_download_rebuild(esat_batch* b, uint32_t* n_out, uint32_t* merges, uint32_t* hc_sym, uint32_t* hc_koff,
                          uint32_t* hc_kids, uint32_t* hc_cid, double* hc_cost, uint32_t* uf_parent, uint8_t* uf_rank);
int esat_download_view(esat_batch* b, uint32_t* C, uint32_t* root_pos, uint32_t* cls_id, uint32_t* cls_off,
                       uint32_t* nd_sym, uint32_t* nd_koff, uint32_t* nd_kpos, double* nd_cost, uint32_t* nd_hc);
/* match results of the i-th pattern (ematch) or rule (join) of the LAST call: per-leaf
 * counts[L] and word offsets[L+1] (into words); words may be NULL to query sizes. */
int esat_download_matches(esat_batch* b, int from_join, uint32_t index, uint32_t* counts, uint64_t* word_off,
                          uint32_t* words, uint64_t words_cap);
/* counts[n][L] of every pattern (ematch) or rule (join) of the last call in one copy: match counts
 * in LIST mode, 0/1 existence in EXISTS mode (is_rule_applicable of every source at once) */
int esat_download_counts(esat_batch* b, int from_join, uint32_t* counts);
int esat_download_extract(esat_batch* b, uint32_t* status, uint32_t* err_class, double* root_cost,
                          double* class_cost, uint32_t* choice, uint8_t* reachable, uint32_t* passes);
/* shape of the last extraction: total e-classes and total Gauss-Seidel levels over the batch's
 * leaves (mean level width = classes / levels; the host picks the lane-group width from it) */
int esat_extract_shape(esat_batch* b, uint64_t* classes, uint64_t* levels);
/* k_extract lanes per leaf in one-warp CTAs for every later extraction on this context: 32 (one
 * leaf per warp), 16 or 8 (two / four leaves share a warp: narrow levels); 0 = 32. Results are
 * identical for every width. */
int esat_set_extract_lanes(esat_ctx* ctx, uint32_t lanes);

/* run all work of this context on a caller-owned CUDA stream (e.g. torch's current stream) */
int esat_ctx_set_stream(esat_ctx* ctx, void* cuda_stream);
/* device-to-device copy of per-leaf root costs (f64[L]) and statuses (u32[L]) into caller
 * buffers on the context stream -- feeds the NCCL all-gather of MCTS leaf results */
int esat_copy_results(esat_batch* b, void* dev_root_cost, void* dev_status);
/* device pointers of per-leaf summary results (for fused collectives over NCCL) */
int esat_result_device_ptrs(esat_batch* b, void** root_cost, void** status);

/* timing of the last compute call on the context stream, in milliseconds (CUDA events) */
float esat_last_kernel_ms(const esat_ctx* ctx);

/* ---- apply loop: apply_rule on every leaf of a rebuilt batch ----------------
 * Replaces rewrite.py:526-570 (apply_rule: _target_refs 460-489, would_create_cycle 492-505,
 * _instance_shape 508-514, _instantiate 517-523, EGraph.add/union egraph.py:175-201) and the
 * language hooks make_symbol (rewrite.py:296-298, tensor_ir.py:253-265) / infer_shape
 * (tensor_ir.py:64-126). Status per leaf: */
#define ESAT_A_OK 0
#define ESAT_A_NODE_LIMIT 1     /* StructuralError: node limit not above the node count (rewrite.py:532-537) */
#define ESAT_A_NEED_SYMBOL 2    /* a new operator symbol must be interned on the host, then retry */
#define ESAT_A_CAPACITY 3       /* the leaf's arena headroom is exhausted: re-pack with more, retry */
#define ESAT_A_PROGRAM 4        /* target program beyond device limits */

/* symbol identities (paper_2410_05534_b200/apply.py): per-symbol shape (ndim 255 = none, dims
 * [n][4]), open-addressing key table (power-of-2 size), attribute integer values by code, the
 * language (0 term, 1 tensor), cost model (0 term, 1 unit, 2 analytic x coeff) and the rule
 * target programs (offsets [n_rules+1] into words) */
int esat_apply_setup(esat_ctx* ctx, int lang, int cost_mode, double coeff, uint32_t n_syms, const uint8_t* sym_ndim,
                     const uint32_t* sym_dims, uint32_t table_size, const uint32_t* sym_table, uint32_t n_values,
                     const int32_t* val_int, uint32_t n_rules, const uint32_t* rule_off, const int32_t* words);
/* live entry / id counts of an arena uploaded with headroom (spans larger than the leaves) */
int esat_batch_set_counts(esat_batch* b, const uint32_t* n_cnt, const uint32_t* u_cnt);
/* apply rule leaf_rule[l] (0xFFFFFFFF: none) to every leaf, using the match lists of the last
 * esat_ematch / esat_join calls; the leaf's dirty state replaces the batch input (next: esat_rebuild) */
int esat_apply(esat_batch* b, const uint32_t* leaf_rule, uint32_t node_limit);
/* status[L], report[L][8] = {matches_found, changed, cycles_filtered, shape_filtered (ApplyReport,
 * rewrite.py:440-448), unions performed, e-nodes added, 0, 0}, missing[L][16] = descriptor of a
 * symbol to intern */
int esat_download_apply(esat_batch* b, uint32_t* status, uint32_t* report, uint32_t* missing);
/* ---- WL fingerprint: EGraph.fingerprint (egraph.py:247-296) per rebuilt leaf ----
 * krank[s] = rank of symbol s's key (name, arity, repr(payload)) in Python tuple order,
 * key_bytes[key_off[s]:key_off[s+1]] = repr(key) (UTF-8) (paper_2410_05534_b200/fingerprint.py) */
int esat_fingerprint_setup(esat_ctx* ctx, uint32_t n_syms, const uint32_t* krank, const uint32_t* key_off,
                           const uint8_t* key_bytes);
int esat_fingerprint(esat_batch* b);
/* fp[L] = the reference's 64-bit fingerprint; status[L] 0 ok */
int esat_download_fingerprint(esat_batch* b, uint64_t* fp, uint32_t* status);
/* the batch input (dirty) arena with live counts: hashcons + union-find, spans as created */
int esat_download_state(esat_batch* b, uint32_t* n_cnt, uint32_t* u_cnt, uint32_t* sym, uint32_t* koff,
                        uint32_t* kids, uint32_t* cid, double* cost, uint32_t* parent, uint8_t* rank);

/* ---- device snapshot store: EGraph.snapshot (egraph.py:300-312) as D2D copies into slots ---- */
typedef struct esat_store esat_store;
int esat_store_create(esat_ctx* ctx, esat_store** out);
int esat_store_destroy(esat_store* st);
/* number of slots; slots are append-only, esat_store_truncate drops the newest */
uint32_t esat_store_size(const esat_store* st);
int esat_store_truncate(esat_store* st, uint32_t count);
/* copy the last rebuild of batch leaves[0..count) (clean hashcons + union-find + raw root) into
 * new slots (device to device); their ids go to slots_out */
int esat_store_save(esat_store* st, esat_batch* b, uint32_t count, const uint32_t* leaves, uint32_t* slots_out);
/* one host leaf state (the batch-arena format of one leaf, koff with n+1 entries) into a new slot */
int esat_store_put(esat_store* st, uint32_t n, uint32_t K, uint32_t U, uint32_t root, const uint32_t* sym,
                   const uint32_t* koff, const uint32_t* kids, const uint32_t* cid, const double* cost,
                   const uint32_t* parent, const uint8_t* rank, uint32_t* slot_out);
/* sizes of slots: hashcons entries, child slots, union-find ids, raw root (any pointer may be NULL) */
int esat_store_info(const esat_store* st, uint32_t count, const uint32_t* slots, uint32_t* n, uint32_t* K,
                    uint32_t* U, uint32_t* root);
int esat_store_download(esat_store* st, uint32_t slot, uint32_t* sym, uint32_t* koff, uint32_t* kids, uint32_t* cid,
                        double* cost, uint32_t* parent, uint8_t* rank);
/* fill the input arena of b (leaf l's spans must hold slot slots[l]) from the store, device to
 * device, and set the live counts (as esat_batch_upload + esat_batch_set_counts) */
int esat_batch_load_slots(esat_batch* b, esat_store* st, const uint32_t* slots);

#ifdef __cplusplus
}
#endif
#endif /* ESAT_B200_H */

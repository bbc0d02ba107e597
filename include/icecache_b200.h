/* icecache_b200.h -- C ABI of the B200-native IceCache decode hot path.
 *
 * The reference (arXiv 2604.10539, /root/reference/pkg/src/icecache) exposes
 * this path as a Python/NumPy API; there is no FFI in the reference.  Each
 * entry point below replaces the reference call named beside it, batched over
 * T independent DCI trees (one per (sequence, layer, kv head)):
 *
 *   icb_build            dci_indexing                 dci.py:479-568
 *   icb_query            DciTree.query + find_page_index + gqa_union
 *                                                     dci.py:318-364, pagestore.py:111-113,
 *                                                     attention.py:96-103, engine.py:436-447
 *   icb_insert           DciTree.insert / _grow_top   dci.py:385-449
 *   icb_alloc_resident_pages  TierStore.allocate_page (sink / window)
 *                                                     pagestore.py:138-149, engine.py:263-276
 *   icb_rotate_window    Engine._rotate_layer         engine.py:516-534
 *   icb_append_window    window append                engine.py:426-429
 *   icb_sparse_attention sparse_attention + TierStore.backload/evict_unselected
 *                                                     attention.py:77-93, pagestore.py:169-215,
 *                                                     engine.py:449-475
 *   icb_dense_attention  full_attention (skip layers) attention.py:55-74, engine.py:418-422
 *   icb_export_tree / icb_tree_info  host mirror for structure checks (DciTree fields,
 *                                                     check_invariants dci.py:453-476)
 *
 * All array arguments marked "dev" are device pointers (plain CUDA memory);
 * "host" arguments are host memory.  `stream` is a cudaStream_t (NULL = legacy
 * default stream).  Every call returns ICB_OK or an error code; the message is
 * available from icb_last_error().  Errors map to the reference exceptions
 * (errors.py:8-40): ICB_E_INPUT -> InputError, ICB_E_CONFIG -> ConfigError,
 * ICB_E_CONSISTENCY -> ConsistencyError, ICB_E_DEGENERATE -> DegenerateQueryError.
 */
#ifndef ICECACHE_B200_H
#define ICECACHE_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ICB_OK 0
#define ICB_E_INPUT 1
#define ICB_E_CONFIG 2
#define ICB_E_CONSISTENCY 3
#define ICB_E_CUDA 4
#define ICB_E_CAPACITY 5
#define ICB_E_POLICY 6
#define ICB_E_DEGENERATE 7

#define ICB_KV_F32 0
#define ICB_KV_BF16 1

#define ICB_ROLE_SINK 1
#define ICB_ROLE_WINDOW 2
#define ICB_ROLE_INDEXED 3

#define ICB_SENTINEL_LEVEL (-1)

typedef struct icb_forest icb_forest;

typedef struct {
  int32_t n_trees;     /* T */
  int32_t dim;         /* key dim d (<= 128) */
  int32_t dim_v;       /* value dim d' (<= 128) */
  int32_t page_size;   /* s (2..32) */
  int32_t kv_dtype;    /* ICB_KV_F32 | ICB_KV_BF16: storage of page K/V */
  int32_t tok_cap;     /* token ids must be < tok_cap (rows are indexed by token id) */
  int32_t node_cap;    /* nodes per tree */
  int32_t page_cap;    /* page ids per tree */
  int32_t member_cap;  /* member-pool entries per tree */
  int32_t own_cap;     /* owned-node list entries per tree */
  int32_t dirs_cap;    /* cached P-DCI direction sets per tree */
  double promotion_ratio; /* r */
  /* KV offload (BASELINE config 3; TierStore, pagestore.py:117-215): when
   * kv_host != 0 all page K/V live in pinned, device-mapped host memory and
   * each fused decode step (icb_query_attend / icb_step_attend) gathers the
   * pages it attends -- sink, window and selected -- into a per-tree HBM pool
   * of pool_pages slots (pages already resident are kept, the rest are
   * evicted).  pool_pages must cover sink + window + the largest selection. */
  int32_t kv_host;
  int32_t pool_pages;
} icb_forest_config;

const char *icb_last_error(void);
int icb_version(void);

int icb_forest_create(const icb_forest_config *cfg, icb_forest **out);
int icb_forest_destroy(icb_forest *f);

/* Seed each tree's level stream: SeedSequence(entropy words).spawn_key=(0,)
 * (dci.py:180-183).  host: trees[n], words[n][stride], n_words[n]. */
int icb_seed_trees(icb_forest *f, const int32_t *trees, int32_t n, const uint32_t *words,
                   int32_t stride, const int32_t *n_words);

/* Allocate `count` resident pinned pages of `role` per tree and fill them in
 * token order with `n_tokens` entries (tokens dev [n][n_tokens], keys dev
 * [n][n_tokens][dim], values dev [n][n_tokens][dim_v]).  Sink pages are
 * recorded as the tree's sink list, window pages appended to its window ring. */
int icb_alloc_resident_pages(icb_forest *f, const int32_t *trees, int32_t n, int32_t role,
                             int32_t count, int32_t n_tokens, const int32_t *tokens,
                             const float *keys, const float *values, void *stream);

/* Batch build of n trees over n_points (token, key) pairs each.  trees dev[n];
 * tokens dev [n][n_points]; keys dev [n][n_points][dim] fp32; values dev or
 * NULL; scales dev [n] fp64 or NULL (derive KeyScale.from_keys). */
int icb_build(icb_forest *f, const int32_t *trees, int32_t n, int32_t n_points,
              const int32_t *tokens, const float *keys, const float *values,
              const double *scales, void *stream);

/* Multi-level search for G query heads per tree plus the GQA page union.
 * queries dev [n][G][dim] raw queries (lifted in-kernel, geometry.py:89-98),
 * or, with lifted_input=1, [n][G][dim+1] already-lifted vectors.
 * out_ids dev [n][G][k_out] ranked by (d2, id); out_counts dev [n][G];
 * out_pages dev [n][pages_cap] ascending unique page ids (may be NULL);
 * out_npages dev [n].  distance/queries counters accumulate in the trees. */
int icb_query(icb_forest *f, const int32_t *trees, int32_t n, int32_t G, const float *queries,
              int32_t lifted_input, int32_t k, int64_t beam, int64_t visit_cap,
              int32_t target_level, int32_t *out_ids, int32_t k_out, int32_t *out_counts,
              int32_t *out_pages, int32_t pages_cap, int32_t *out_npages, void *stream);

/* The decode step's selection and attention in one launch: icb_query
 * (SENTINEL target, raw queries) followed, in the same CTA, by
 * icb_sparse_attention over the tree's sink, window and selected pages
 * (engine.py:436-475: page_select per head, gqa_union, backload,
 * sparse_attention, evict_unselected).  attn_out dev [n][G][dim_v];
 * attn_stats dev [n][5] or NULL (the residency counters of
 * icb_sparse_attention). */
int icb_query_attend(icb_forest *f, const int32_t *trees, int32_t n, int32_t G, const float *queries,
                     int32_t k, int64_t beam, int64_t visit_cap, int32_t *out_ids, int32_t k_out,
                     int32_t *out_counts, int32_t *out_pages, int32_t pages_cap, int32_t *out_npages,
                     float *attn_out, int64_t *attn_stats, int32_t scalar_bytes, void *stream);

/* One whole decode step of a stage of indexed trees in one launch
 * (Engine.decode_step, engine.py:412-475, with _rotate_layer, :516-534):
 * each tree's CTA first rotates its oldest window page into the tree when
 * `rotate` (as icb_rotate_window; rot_stats dev [n][2] or NULL), then appends
 * the decode token (as icb_append_window_dev: token_dev, win_keys dev
 * [n][dim], win_values dev [n][dim_v]), then runs icb_query_attend.  Results
 * are identical to those four calls in sequence; the step's slowest rotation
 * no longer holds back every tree's search. */
int icb_step_attend(icb_forest *f, const int32_t *trees, int32_t n, int32_t G, const float *queries,
                    int32_t k, int64_t beam, int64_t visit_cap, int32_t *out_ids, int32_t k_out,
                    int32_t *out_counts, int32_t *out_pages, int32_t pages_cap, int32_t *out_npages,
                    float *attn_out, int64_t *attn_stats, int32_t scalar_bytes, int32_t rotate,
                    int64_t *rot_stats, const int32_t *token_dev, const float *win_keys,
                    const float *win_values, void *stream);

/* Sequential inserts of m points per tree (trees in parallel).  levels dev
 * [n][m] or NULL (draw from the tree's stream); out_levels dev or NULL. */
int icb_insert(icb_forest *f, const int32_t *trees, int32_t n, int32_t m, const int32_t *tokens,
               const float *keys, const float *values, const int32_t *levels,
               int32_t *out_levels, void *stream);

/* Engine._rotate_layer: offload the oldest window page, insert its entries,
 * release it, allocate a fresh window page.  stats dev [n][2] += (bytes, 1). */
int icb_rotate_window(icb_forest *f, const int32_t *trees, int32_t n, int32_t scalar_bytes,
                      int64_t *stats, void *stream);

/* Append one token to the first non-full window page of each tree.
 * keys dev [n][dim], values dev [n][dim_v]. */
int icb_append_window(icb_forest *f, const int32_t *trees, int32_t n, int32_t token,
                      const float *keys, const float *values, void *stream);

/* Sparse attention of G query heads per tree over sink, window and the
 * selected pages (pages dev [n][pages_cap], npages dev [n]); out dev
 * [n][G][dim_v] fp32.  stats dev [n][5] (accumulated): pages_selected,
 * tokens_loaded, pages_loaded, bytes_moved, transactions.  Residency
 * (hot = selected U pinned) is updated per tree.  splits: split-K factor
 * (0 = auto). */
int icb_sparse_attention(icb_forest *f, const int32_t *trees, int32_t n, int32_t G,
                         const float *queries, const int32_t *pages, int32_t pages_cap,
                         const int32_t *npages, float *out, int64_t *stats,
                         int32_t scalar_bytes, int32_t splits, void *stream);

/* Dense decode attention (skip layers / fallback): n heads-groups, G query
 * heads each, over n_tokens contiguous K/V rows.  k dev [n][ld][ceil4(dim)],
 * v dev [n][ld][ceil4(dim_v)] (kv_dtype; rows padded to 4 elements, as
 * icb_dense_append writes them), q dev [n][G][dim], out dev [n][G][dim_v].
 * Logits are scaled by 1/sqrt(dim) (attention.py:70, d = q.size). */
int icb_dense_attention(int32_t n, int32_t G, int32_t dim, int32_t dim_v, int32_t kv_dtype,
                        const float *q, const void *k, const void *v, int64_t ld,
                        int32_t n_tokens, float *out, int32_t splits, void *stream);

/* Evaluation support (engine.py:536-566): mask dev [n][tok_cap] uint8 set to 1
 * for every token of tree trees[b]'s sink, window and selected pages (the
 * attended set of sparse_attention), 0 elsewhere. */
int icb_attended_mask(icb_forest *f, const int32_t *trees, int32_t n, const int32_t *pages, int32_t pages_cap,
                      const int32_t *npages, uint8_t *mask, void *stream);

/* DciTree.pdci_query (dci.py:282-298): the k nearest members of one node to
 * a lifted query (q_lifted dev [dim + 1]), ranked by (d2, id); P-DCI visit
 * list of visit_cap members for nodes above EXHAUSTIVE_NODE_LIMIT that the cap
 * does not cover.  out_ids dev [>= min(k, node size)], out_count dev [1]. */
int icb_node_query(icb_forest *f, int32_t tree, int32_t node, const float *q_lifted, int32_t k,
                   int64_t visit_cap, int32_t *out_ids, int32_t *out_count, void *stream);

/* Selection reuse (engine.py:321-363, select_with_reuse): for tree trees[b]
 * (a non-anchor layer) the page list of the token lists that query output
 * row src_rows[b] holds (src_ids [rows][G][k_stride], src_counts [rows][G],
 * as written by icb_query), mapped through trees[b]'s own page table:
 * sorted unique page ids (find_page_index, pagestore.py:111-113). */
int icb_pages_from_tokens(icb_forest *f, const int32_t *trees, int32_t n, const int32_t *src_rows,
                          const int32_t *src_ids, const int32_t *src_counts, int32_t G, int32_t k_stride,
                          int32_t *out_pages, int32_t pages_cap, int32_t *out_npages, void *stream);

/* CUDA-graph variants: the decode position is read from device memory
 * (token_dev[0] = the token being decoded), so one captured decode step
 * replays for every position.  icb_append_window_dev is icb_append_window
 * (engine.py:425-428); icb_dense_attention_dev attends rows
 * [0, token_dev[0] + 1) (engine.py:418-422); icb_dense_append writes the
 * step's K/V row of each skip-layer plane at row token_dev[0] (the K/V
 * mirror append, engine.py:414-416). */
int icb_append_window_dev(icb_forest *f, const int32_t *trees, int32_t n, const int32_t *token_dev,
                          const float *keys, const float *values, void *stream);
int icb_dense_attention_dev(int32_t n, int32_t G, int32_t dim, int32_t dim_v, int32_t kv_dtype,
                            const float *q, const void *k, const void *v, int64_t ld,
                            const int32_t *token_dev, float *out, int32_t splits, void *stream);
int icb_dense_append(int32_t n, int32_t dim, int32_t dim_v, int32_t kv_dtype, const float *k,
                     const float *v, void *dense_k, void *dense_v, int64_t ld,
                     const int32_t *token_dev, void *stream);

/* Reference-shaped attention outputs (AttentionOutput.weights,
 * attention.py:26-93).  The decode hot path computes only value_out; these
 * serve the API around it.
 *
 * icb_exact_attention: full_attention (attention.py:55-74) of one query over
 * n_rows key/value rows, all fp64: logits k.q / sqrt(dim), max-subtracted
 * softmax, weights @ V.  q dev [dim], k dev [n_rows][dim], v dev
 * [n_rows][dim_v] (double); weights dev [n_rows], out dev [dim_v] (double).
 *
 * icb_attention_weights: for each tree trees[b] and query head g, the tokens
 * of its attended set in entry order -- sink pages, window pages, selected
 * pages (pages dev [n][pages_cap], npages dev [n]) each in append order
 * (engine.py:454-461) -- and their softmax weights, logits in fp64 from the
 * stored K (kv dtype) and the fp32 query (q dev [n][G][dim]).  out_tokens dev
 * [n][cap] int32, out_weights dev [n][G][cap] double, out_count dev [n]
 * (attended tokens; entries past cap are dropped).
 *
 * icb_dense_weights: the same over dense planes (skip layers / fallback,
 * engine.py:418-422): rows [0, n_tokens) of k dev [n][ld][ceil4(dim)];
 * out_weights dev [n][G][n_tokens]. */
int icb_exact_attention(int32_t n_rows, int32_t dim, int32_t dim_v, const double *q, const double *k,
                        const double *v, double *weights, double *out, void *stream);
int icb_attention_weights(icb_forest *f, const int32_t *trees, int32_t n, int32_t G, const float *queries,
                          const int32_t *pages, int32_t pages_cap, const int32_t *npages,
                          int32_t *out_tokens, double *out_weights, int32_t cap, int32_t *out_count,
                          void *stream);
int icb_dense_weights(int32_t n, int32_t G, int32_t dim, int32_t kv_dtype, const float *q, const void *k,
                      int64_t ld, int32_t n_tokens, double *out_weights, void *stream);

/* Per-tree summary (host out[16]): levels, top_node, n_nodes, next_page,
 * n_points, err, n_window, n_sink, query_count, distance_evals, scale_clamps,
 * member_top, own_top, n_dirs, 0, 0.  Synchronizes the device. */
int icb_tree_info(icb_forest *f, int32_t tree, int64_t *out);

/* Copy one tree's arrays to host buffers (any may be NULL).  Sizes: node
 * arrays node_cap, members member_cap, page arrays page_cap (page_tok
 * page_cap*s), token arrays tok_cap, own_list own_cap.  win/sink: 8 each. */
int icb_export_tree(icb_forest *f, int32_t tree, int32_t *node_level, int32_t *node_parent,
                    int32_t *node_owner, int32_t *node_off, int32_t *node_size,
                    int32_t *node_lastpage, int32_t *members, int32_t *page_fill,
                    int8_t *page_role, int32_t *page_tok, int32_t *tok2page, int8_t *level,
                    int32_t *own_base, int32_t *own_list, float *lift, float *tail,
                    int32_t *win, int32_t *sink);

/* Read page K/V back (host float, converted from the storage dtype):
 * keys [count][s][dim], values [count][s][dim_v] for page ids pages[count]. */
int icb_read_pages(icb_forest *f, int32_t tree, const int32_t *pages, int32_t count, float *keys,
                   float *values);

/* Sticky device error bits of every tree (host out[n_trees]); clear=1 resets
 * them.  Synchronizes the device. */
int icb_errors(icb_forest *f, int32_t *out, int32_t clear);
/* Clear a tree's sticky device error bits (after the host reported them). */
int icb_clear_errors(icb_forest *f, int32_t tree);
/* KeyScale.c of a built tree (host out). */
int icb_read_meta_c(icb_forest *f, int32_t tree, double *c);
/* KeyScale c of an empty tree that grows by inserts only (DciTree(dim, scale,
 * ...), dci.py:164-176; geometry.py:47-56).  A build sets c itself. */
int icb_set_scale(icb_forest *f, int32_t tree, double c);
/* KV offload: out host [n_trees][2] = bytes gathered host -> HBM pool so far,
 * pages resident in the pool now (ICB_E_CONFIG when kv_host = 0). */
int icb_pool_stats(icb_forest *f, int64_t *out);
/* Host-side restatement check: n PCG64 doubles of SeedSequence(words, spawn). */
int icb_host_pcg_doubles(const uint32_t *words, int32_t n_words, const uint32_t *spawn,
                         int32_t n_spawn, int32_t n, double *out);
/* The same stream after a jump of `skip` draws (the LCG jump the device level
 * draw uses to split the stream across threads). */
int icb_host_pcg_jump_doubles(const uint32_t *words, int32_t n_words, const uint32_t *spawn,
                              int32_t n_spawn, int64_t skip, int32_t n, double *out);

#ifdef __cplusplus
}
#endif
#endif

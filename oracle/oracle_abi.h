/*
 * oracle_abi.h — TEST INFRASTRUCTURE ONLY.
 *
 * One C interface implemented twice, so the parity tests can run the same
 * case through either CPU checker:
 *   - oracle/annkit_oracle.c  : our plain-C restatement of the reference
 *                               algorithms (built to oracle/liboracle.so);
 *   - oracle/ref_shim.cpp     : a thin extern "C" wrapper around the
 *                               UNMODIFIED reference library, compiled from
 *                               /root/reference/proj/src where it lies
 *                               (built to oracle/_ref/libannkit_ref.so).
 *
 * Nothing in the product path (paper_1609_07228_b200/) links or loads either
 * library; only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
 * leg do, and only as the checker / the timed CPU reference arm.
 *
 * Handles are opaque.  Status codes: 0 ok, 1 invalid_argument,
 * 2 out_of_range, 5 anything else; ora_last_error() has the message.
 */
#ifndef ANNKIT_ORACLE_ABI_H
#define ANNKIT_ORACLE_ABI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* ora_last_error(void);
const char* ora_impl_name(void);

/* dataset.hpp:28-37 VectorSet; dataset.cpp:201-214 gen_synthetic */
void* ora_vs_create(const float* data, uint32_t n, uint32_t dim);
void ora_vs_free(void* vs);
void ora_gen_synthetic(uint32_t n, uint32_t dim, uint64_t seed, float* out);
/* the BASELINE configs' Gaussian mixture (restatement of annk_gen_mixture; not a reference function) */
void ora_gen_mixture(uint32_t n, uint32_t dim, uint32_t n_centers, float center_lo, float center_hi, float sd,
                     float clip_lo, float clip_hi, int round_to_int, uint64_t seed, uint32_t stream_id,
                     uint32_t workers, float* out);
float ora_l2_sq(const float* a, const float* b, uint32_t dim);
uint64_t ora_mix64(uint64_t x);
uint64_t ora_substream(uint64_t seed, uint64_t id);
/* first `count` outputs of std::mt19937_64(seed) */
void ora_mt19937_64(uint64_t seed, uint32_t count, uint64_t* out);

/* eval.cpp:33-80 brute_force_knn / brute_force_graph (dists optional) */
int ora_brute_force(void* base, void* queries, uint32_t k, uint32_t workers, uint32_t* ids,
                    float* dists, uint64_t* dist_comps);

/* kd_forest.cpp:245-264 build_forest, exported per tree */
void* ora_forest_build(void* vs, uint32_t n_trees, uint32_t leaf_cap, uint64_t seed,
                       uint32_t workers, int* status);
void ora_forest_free(void* f);
uint32_t ora_forest_num_trees(void* f);
uint32_t ora_forest_num_nodes(void* f, uint32_t t);
/* arrays sized num_nodes (node fields) and n (point_index) */
void ora_forest_export(void* f, uint32_t t, uint32_t* split_dim, float* split_val,
                       uint32_t* left, uint32_t* right, uint32_t* depth, uint8_t* even,
                       uint32_t* point_index, uint32_t* root_and_leaves /* [root, leaf_count] */);
/* Builds a forest from exported arrays (node arrays concatenated over trees). */
void* ora_forest_import(uint32_t n, uint32_t dim, uint32_t leaf_cap, uint64_t seed,
                        uint32_t n_trees, const uint32_t* node_counts, const uint32_t* roots,
                        const uint32_t* split_dim, const float* split_val, const uint32_t* left,
                        const uint32_t* right, const uint32_t* depth, const uint8_t* even,
                        const uint32_t* point_index);
/* kd_forest.cpp:266-305 */
int ora_search_leaves(void* f, uint32_t t, const float* q, uint32_t qlen, uint32_t n_leaves,
                      uint32_t* out, uint32_t* n_out);
int ora_descend_from(void* f, uint32_t t, const float* q, uint32_t qlen, uint32_t node,
                     uint32_t* out);

/* graph_build.hpp:17-30 RefineState */
void* ora_init_graph(void* vs, void* f, uint32_t k, uint32_t conquer_depth, uint32_t pool_cap,
                     uint32_t sample_cap, uint64_t seed, uint32_t workers, int* status);
void* ora_init_random(void* vs, uint32_t k, uint32_t pool_cap, uint32_t sample_cap,
                      uint64_t seed, uint32_t workers, int* status);
/* pools given as n rows of pool_cap slots, sizes[i] valid entries each */
void* ora_state_import(uint32_t n, uint32_t k, uint32_t pool_cap, uint32_t sample_cap,
                       uint64_t seed, uint32_t iteration, uint64_t dist_comps,
                       const uint32_t* sizes, const uint32_t* ids, const float* dists,
                       const uint8_t* flags);
void ora_state_free(void* s);
/* meta = [iteration, dist_comps, last_changes] */
void ora_state_export(void* s, uint32_t* sizes, uint32_t* ids, float* dists, uint8_t* flags,
                      uint64_t* meta);
/* which: 0 g_new, 1 g_old, 2 g_rnew, 3 g_rold.  offsets has n+1 entries;
 * data may be NULL (offsets only). */
void ora_state_lists(void* s, int which, uint32_t* offsets, uint32_t* data);
uint64_t ora_nn_descent_iteration(void* s, void* vs, uint32_t workers);
uint64_t ora_nn_expansion_iteration(void* s, void* vs, uint32_t workers);
void ora_rebuild_sample_lists(void* s);
/* shard-mode protocol (test-only; see annkit_oracle.c) */
void ora_shard_sample(void* s, uint32_t lo, uint32_t hi, uint32_t* fnew, uint32_t* cnew, uint32_t* fold,
                      uint32_t* cold, uint64_t* thr);
void ora_shard_union(void* s, const uint32_t* fnew, const uint32_t* cnew, const uint32_t* fold,
                     const uint32_t* cold);
uint64_t ora_shard_join(void* s, void* vs, uint32_t lo, uint32_t hi, const uint64_t* thr, uint64_t* n_offers);
void ora_shard_offers_get(uint32_t* tgt, uint64_t* key, uint32_t* src);
uint64_t ora_shard_replay(void* s, const uint32_t* tgt, const uint64_t* key, const uint32_t* src, size_t m);
void ora_shard_finish(void* s, uint64_t changes);
void ora_union_reverse_lists(void* s);
int ora_refine_nn_descent(void* s, void* vs, uint32_t max_iters, uint32_t workers,
                          double min_change_rate);
int ora_finalize(void* s, void* vs, uint32_t k, uint32_t* ids, float* dists);
double ora_pool_topk_accuracy(void* s, const uint32_t* gt_ids, uint32_t gt_n, uint32_t gt_k);

/* graph_build.cpp:395-461 build_graph.  strategy: 0 efanna, 1 random-descent,
 * 2 nn-expansion, 3 brute-force, 4 init-only.  log rows: [iteration, seconds,
 * dist_comps, changes, accuracy], up to max_iters+1 rows.
 * summary = [init_s, refine_s, dist_comps, early_stopped]. */
int ora_build_graph(void* vs, void* f, uint32_t k, uint32_t conquer_depth, uint32_t pool_cap,
                    uint32_t sample_cap, uint32_t max_iters, int strategy, uint64_t seed,
                    uint32_t workers, double min_change_rate, const uint32_t* gt_ids,
                    uint32_t gt_k, uint32_t* out_ids, float* out_dists, double* log_rows,
                    uint32_t* n_log, double* summary);

/* search.cpp:121-236.  One call searches every query (per-query seed =
 * substream(seed, qi) as recall_curve does).  stats per query:
 * [dist_comps, leaves_visited, graph_hops, seed_points].  ids/dists are
 * nq*k_return.  time_us (nullable) gets the per-query StopWatch time. */
int ora_search(void* base, void* f, const uint32_t* graph_ids, const float* graph_dists,
               uint32_t graph_n, uint32_t graph_k, void* queries, uint32_t k_return,
               uint32_t pool_size, uint32_t expansion, uint32_t iters, uint32_t n_trees_used,
               uint32_t random_seed_count, uint64_t seed, int random_init, uint32_t workers,
               uint32_t* out_ids, float* out_dists, uint64_t* stats, double* time_us);

#ifdef __cplusplus
}
#endif

#endif

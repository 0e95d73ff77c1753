/*
 * annkit_b200.h — the drop-in C-ABI for EFANNA's data-parallel hot paths on
 * NVIDIA B200 (sm_100a).
 *
 * The reference ("annkit", /root/reference/proj) exposes its hot path as a
 * C++ library API (free functions over value types, proj/include/annkit/ headers);
 * it has no plugin registry or FFI.  This header is the thin C layer that the
 * reference-shaped host API (paper_1609_07228_b200/api.py, and any C++/ctypes
 * caller) binds: plain pointers and sizes, no torch types, opaque handles for
 * device-resident objects.  Each entry point names the reference interface it
 * replaces.
 *
 * Conventions
 *   - Every function returns an annk_status; annk_last_error() (thread-local)
 *     carries the message.  ANNK_INVALID_ARGUMENT / ANNK_OUT_OF_RANGE map to
 *     the reference's std::invalid_argument / std::out_of_range.
 *   - Host buffers are borrowed for the duration of the call.  Calls are
 *     synchronous: on return, outputs are in the caller's buffers.
 *   - Results are bit-identical to the reference at workers = 1 (distances are
 *     the reference's sequential fp32 l2_sq; ties ordered by id).
 *   - There is no CPU fallback: without a usable sm_100 device every compute
 *     entry point fails with ANNK_CUDA_ERROR.
 */
#ifndef ANNKIT_B200_H
#define ANNKIT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    ANNK_OK = 0,
    ANNK_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument */
    ANNK_OUT_OF_RANGE = 2,     /* reference: std::out_of_range     */
    ANNK_CUDA_ERROR = 3,
    ANNK_OUT_OF_MEMORY = 4,
    ANNK_INTERNAL = 5
} annk_status;

typedef struct annk_dataset annk_dataset;   /* VectorSet       dataset.hpp:28-37      */
typedef struct annk_forest annk_forest;     /* KdForest        kd_forest.hpp:47-53    */
typedef struct annk_state annk_state;       /* RefineState     graph_build.hpp:17-30  */
typedef struct annk_searcher annk_searcher; /* GraphSearcher   search.hpp:43-76       */

/* ---------------------------------------------------------------- runtime */
const char* annk_last_error(void);
const char* annk_version(void);
/* Selects the CUDA device for subsequent calls from this process (default 0). */
int annk_set_device(int device);
/* The library's CUDA stream (cudaStream_t as an integer) — for event timing. */
uint64_t annk_stream(void);
/* Number of kernels this library has launched since load. */
uint64_t annk_launch_count(void);
int annk_synchronize(void);
/* Per-kernel CUDA-event timing on the library stream (no reference
 * counterpart; the reference only has StopWatch wall time, util.hpp:21-31).
 * report writes "kernel_name launches total_ms" lines. */
int annk_profile_enable(int on);
int annk_profile_reset(void);
int annk_profile_report(char* buf, uint64_t cap);

/* ---------------------------------------------------------------- dataset */
/* Uploads an n x dim row-major fp32 matrix (VectorSet::data).  Values must be
 * finite (load_fvecs dataset.cpp:123-126 rejects the rest). */
int annk_dataset_create(const float* host, uint32_t n, uint32_t dim, annk_dataset** out);
int annk_dataset_destroy(annk_dataset* ds);
int annk_dataset_shape(const annk_dataset* ds, uint32_t* n, uint32_t* dim);
/* [n, dim, exact_u8_path (0/1), bytes per row the kernels gather].  The u8
 * path is taken when every value is an integer in [0,255] and dim*255^2 < 2^24:
 * then the reference's fp32 l2_sq is exact and |a|^2+|b|^2-2a.b in int32 equals it. */
int annk_dataset_info(const annk_dataset* ds, uint32_t* out4);

/* dataset.hpp:67-77 distances, computed on the device with the reference's
 * sequential fp32 chain (bit-identical): l2_sq of two host vectors; dist_sq
 * of m id pairs (a[j], b[j]) of a set; dist_sq_q of a host query against m
 * ids.  Ids past the set: ANNK_OUT_OF_RANGE (dataset.cpp:218,225). */
int annk_l2_sq(const float* a, const float* b, uint32_t dim, float* out);
int annk_dist_sq(const annk_dataset* ds, const uint32_t* a, const uint32_t* b, uint32_t m, float* out);
int annk_dist_sq_q(const annk_dataset* ds, const float* q, uint32_t dim, const uint32_t* b, uint32_t m,
                   float* out);
/* dataset.cpp:201-214 gen_synthetic — host helper, same bytes as the reference. */
int annk_gen_synthetic(uint32_t n, uint32_t dim, uint64_t seed, float* out);
/* Seeded Gaussian-mixture generator for the BASELINE configs (no reference
 * counterpart).  round_to_int != 0 rounds to
 * integers (SIFT-like); values are clipped to [lo, hi].  stream 1 = base,
 * 2 = queries; centers always come from stream 0. */
int annk_gen_mixture(uint32_t n, uint32_t dim, uint32_t n_centers, float center_lo,
                     float center_hi, float sd, float clip_lo, float clip_hi, int round_to_int,
                     uint64_t seed, uint32_t stream_id, float* out);

/* ------------------------------------------------------------ exact kNN */
/* eval.cpp:33-61 brute_force_knn and eval.cpp:63-80 brute_force_graph.
 * queries == NULL selects self mode (row i excludes i; k <= n-1), else query
 * mode (k <= n).  out_ids: nq*k; out_dists nullable; dist_comps (nullable) is
 * incremented like the reference's counter. */
int annk_brute_force_knn(const annk_dataset* base, const annk_dataset* queries, uint32_t k,
                         uint32_t* out_ids, float* out_dists, uint64_t* dist_comps);
/* Same on a subset of rows (self mode): rows[0..n_rows) selects which base
 * rows act as queries (used to score accuracy on a seeded sample). */
int annk_brute_force_rows(const annk_dataset* base, const uint32_t* rows, uint32_t n_rows,
                          uint32_t k, uint32_t* out_ids, float* out_dists);
/* Measurement only (no reference counterpart): (256-query block, 64-row base
 * tile) pairs of the last exact-kNN run on the tcgen05 u8 kernel -- all of
 * them, and the ones its MMA passes visited (fewer when the pruned scan dropped
 * cells that provably hold no neighbour; the result is the same).  Synchronises. */
int annk_bf_last_scan(uint64_t* tiles_total, uint64_t* tiles_visited, int* pruned);
/* Measurement only: the dense tcgen05 kind::i8 rate of this GPU in tera-ops/s
 * (u8 multiply-add = 2 ops), one CTA per SM issuing `groups` M=128 x N=256 x K=128
 * MMA groups on shared-memory operands -- the exact-kNN roofline's denominator. */
int annk_measure_i8_peak(uint32_t groups, double* tera_ops);
/* eval.cpp:129-155 accuracy_vs_k: for each k' in k_list, the fraction of graph
 * edges (n x k ids) whose target lies in the exact k'-NN of the source (exact
 * self-mode truth at max k' computed on the device). out: n_k doubles. */
int annk_accuracy_vs_k(const annk_dataset* vs, const uint32_t* graph_ids, uint32_t n, uint32_t k,
                       const uint32_t* k_list, uint32_t n_k, double* out);

/* ---------------------------------------------------------------- forest */
/* kd_forest.cpp:245-264 build_forest — bit-identical trees (same split_dim,
 * split_val, point_index, node numbering) for the same seed. */
int annk_forest_build(const annk_dataset* ds, uint32_t n_trees, uint32_t leaf_cap, uint64_t seed,
                      annk_forest** out);
int annk_forest_destroy(annk_forest* f);
/* counts[0..3] = n_trees, n, dim, leaf_cap; *seed */
int annk_forest_info(const annk_forest* f, uint32_t* counts, uint64_t* seed);
/* per tree: [num_nodes, root, leaf_count, max_depth] */
int annk_forest_tree_info(const annk_forest* f, uint32_t t, uint32_t* info);
/* KdTree fields (kd_forest.hpp:18-42); node arrays sized num_nodes, point_index n. */
int annk_forest_export(const annk_forest* f, uint32_t t, uint32_t* split_dim, float* split_val,
                       uint32_t* left, uint32_t* right, uint32_t* depth, uint8_t* even_split,
                       uint32_t* point_index);
/* Inverse of export (e.g. a forest loaded from an AKF1 file, kd_forest.cpp:332-372). */
int annk_forest_import(uint32_t n, uint32_t dim, uint32_t leaf_cap, uint64_t seed,
                       uint32_t n_trees, const uint32_t* node_counts, const uint32_t* roots,
                       const uint32_t* split_dim, const float* split_val, const uint32_t* left,
                       const uint32_t* right, const uint32_t* depth, const uint8_t* even_split,
                       const uint32_t* point_index, annk_forest** out);
/* kd_forest.cpp:276-305 search_leaves for a batch of queries on tree t:
 * out is nq * n_leaves (unused slots = 0xffffffff), out_counts nq. */
int annk_search_leaves(const annk_forest* f, uint32_t t, const float* queries, uint32_t nq,
                       uint32_t dim, uint32_t n_leaves, uint32_t* out, uint32_t* out_counts);
/* kd_forest.cpp:266-274 descend_from, batched: start[i] -> out[i]. */
int annk_descend_from(const annk_forest* f, uint32_t t, const float* queries, uint32_t nq,
                      uint32_t dim, const uint32_t* start, uint32_t* out);

/* ------------------------------------------------------- graph building */
/* graph_build.cpp:230-292 init_graph. */
int annk_init_graph(const annk_dataset* ds, const annk_forest* f, uint32_t k,
                    uint32_t conquer_depth, uint32_t pool_cap, uint32_t sample_cap, uint64_t seed,
                    annk_state** out);
/* graph_build.cpp:294-326 init_random (the random-descent baseline's start):
 * per point min(pool_cap, n-1) distinct ids drawn from
 * mt19937_64(substream(seed, i)) (all other points when pool_cap >= n-1). */
int annk_init_random(const annk_dataset* ds, uint32_t k, uint32_t pool_cap, uint32_t sample_cap,
                     uint64_t seed, annk_state** out);
/* A RefineState from host pools (n rows of pool_cap slots, sizes[i] used). */
int annk_state_import(uint32_t n, uint32_t k, uint32_t pool_cap, uint32_t sample_cap,
                      uint64_t seed, uint32_t iteration, uint64_t dist_comps,
                      const uint32_t* sizes, const uint32_t* ids, const float* dists,
                      const uint8_t* flags, annk_state** out);
int annk_state_destroy(annk_state* s);
/* meta = [n, k, pool_cap, sample_cap, seed, iteration, dist_comps, last_changes] */
int annk_state_meta(const annk_state* s, uint64_t* meta);
/* Pools to host (ids/dists/flags are n*pool_cap; slots >= sizes[i] unspecified). */
int annk_state_export(const annk_state* s, uint32_t* sizes, uint32_t* ids, float* dists,
                      uint8_t* flags);
/* Adjacency lists of the last sampling step (which: 0 g_new, 1 g_old, 2 g_rnew,
 * 3 g_rold), CSR: offsets n+1 (always), data nullable. */
int annk_state_lists(const annk_state* s, int which, uint32_t* offsets, uint32_t* data);
/* graph_build.cpp:105-162 detail::nn_descent_iteration.  *changes receives
 * the reference's single-worker count: offers its pools accept in its
 * sequential order (point ascending, then pair order), including entries a
 * later offer of the same round evicts again. */
int annk_nn_descent_iteration(annk_state* s, const annk_dataset* ds, uint64_t* changes);
/* graph_build.cpp:164-207 detail::nn_expansion_iteration (the paper's NN-expansion
 * baseline): unchecked pool entries are expanded against the round-start pools.
 * `checked` is bit 1 of the state's flag bytes (annk_state_export). */
int annk_nn_expansion_iteration(annk_state* s, const annk_dataset* ds, uint64_t* changes);
/* graph_build.cpp:59-86 and :88-103 (the two halves of the sampling step). */
int annk_rebuild_sample_lists(annk_state* s);
int annk_union_reverse_lists(annk_state* s);
/* graph_build.cpp:328-335 refine_nn_descent; *iters_run may be NULL. */
int annk_refine_nn_descent(annk_state* s, const annk_dataset* ds, uint32_t max_iters,
                           double min_change_rate, uint32_t* iters_run);
/* graph_build.cpp:346-373 finalize: ids/dists are n*k. */
int annk_finalize(annk_state* s, const annk_dataset* ds, uint32_t k, uint32_t* ids, float* dists);
/* The last round of a build and finalize in one call (graph_build.cpp:105-162
 * followed by :346-373): identical pools, *changes, dist_comps and rows to
 * annk_nn_descent_iteration + annk_finalize.  The replay runs in ascending
 * target chunks, and each chunk's finalized rows travel to ids/dists (host
 * or device, n*k) on a second stream while the next chunk replays.
 * *round_dist_comps (nullable) receives dist_comps after the round, before
 * finalize's fill-up of sparse pools (the reference logs that value). */
int annk_nn_descent_iteration_finalize(annk_state* s, const annk_dataset* ds, uint32_t k, uint32_t* ids,
                                       float* dists, uint64_t* changes, uint64_t* round_dist_comps);
/* graph_build.cpp:209-226 detail::pool_topk_accuracy.  rows == NULL scores all
 * n rows against gt (n x gt_k); otherwise gt row r belongs to point rows[r]. */
int annk_pool_topk_accuracy(const annk_state* s, const uint32_t* gt_ids, uint32_t gt_rows,
                            uint32_t gt_k, const uint32_t* rows, double* acc);
/* Sum over points of |g_new|+|g_old| for the last sampling step (the join's
 * row-gather count; used for the roofline). */
int annk_state_join_rows(const annk_state* s, uint64_t* rows);
/* Last round's device counters: [join_rows, accepted offers, spilled offers,
 * per-point offer slots]. */
int annk_state_stats(const annk_state* s, uint64_t* out4);

/* ----------------------------------------------------- shard mode (multi-GPU)
 * one process per GPU, pools sharded by point.  A state owns the
 * points [lo, hi): init, sampling, the join (as the visiting point i), the
 * merge (as the target) and finalize touch only those.  One NN-descent round
 * over G ranks (the driver is paper_1609_07228_b200/sharded.py):
 *   annk_shard_sample        forward lists + tails of the owned points
 *   all-gather               annk_state_rows(FNEW, CNEW, FOLD, COLD, THR) rows
 *   annk_shard_union         reverse lists from all forward lists, union
 *                            (graph_build.cpp:88-103; same RNG streams on every rank)
 *   annk_shard_join          local join of owned points; offers to any target,
 *                            each tagged with its source point
 *   all-to-all               annk_shard_offers_count/pack per destination range,
 *                            annk_shard_offers_add on the receiver
 *   annk_shard_merge         the owned pools replay their offers in the
 *                            reference's order (source point ascending, then
 *                            the source's pair order; graph_build.cpp:129-156)
 * The pools, flags and `changes` equal the single-GPU ones and the reference's.
 * A round too large for one join launch runs in global source ranges, in
 * ascending order: annk_shard_join_range + exchange + annk_shard_merge_piece
 * per range, then annk_shard_finish_round.  Buffers passed to the row / offer
 * calls may be host or device pointers (UVA copies). */
#define ANNK_ROWS_FNEW 0 /* n x sample_cap u32: sampled new ids (pool order) */
#define ANNK_ROWS_CNEW 1 /* n u32 */
#define ANNK_ROWS_FOLD 2 /* n x pool_cap u32: sampled old ids */
#define ANNK_ROWS_COLD 3 /* n u32 */
#define ANNK_ROWS_THR 4  /* n u64: start-of-round pool tail keys */
/* init_graph for the points [lo, hi) only (the rest stay empty). */
int annk_init_graph_shard(const annk_dataset* ds, const annk_forest* f, uint32_t k,
                          uint32_t conquer_depth, uint32_t pool_cap, uint32_t sample_cap, uint64_t seed,
                          uint32_t lo, uint32_t hi, annk_state** out);
int annk_state_set_shard(annk_state* s, uint32_t lo, uint32_t hi);
/* Copies rows [lo, hi) of a per-point buffer out of (put = 0) or into (put = 1) the state. */
int annk_state_rows(annk_state* s, int which, int put, uint32_t lo, uint32_t hi, void* buf);
int annk_shard_sample(annk_state* s);
int annk_shard_union(annk_state* s);
int annk_shard_join(annk_state* s, const annk_dataset* ds, uint64_t* comps);
/* Join of the owned sources in [ilo, ihi).  *ok = 0 when the range's offers
 * exceed one launch (nothing is kept; *offers reports how many there were). */
int annk_shard_join_range(annk_state* s, const annk_dataset* ds, uint32_t ilo, uint32_t ihi, uint64_t* comps,
                          uint64_t* offers, uint32_t* ok);
/* Offers held for targets [lo, hi): total count; then pack them target-major
 * (counts: hi - lo u32, keys: total u64, srcs: total u32 source points). */
int annk_shard_offers_count(annk_state* s, uint32_t lo, uint32_t hi, uint64_t* total);
int annk_shard_offers_pack(annk_state* s, uint32_t lo, uint32_t hi, uint32_t* counts, uint64_t* keys,
                           uint32_t* srcs);
/* Adds received offers for owned targets [lo, hi) (same packed layout). */
int annk_shard_offers_add(annk_state* s, uint32_t lo, uint32_t hi, const uint32_t* counts,
                          const uint64_t* keys, const uint32_t* srcs);
int annk_shard_merge(annk_state* s, uint64_t* changes);
/* Pieces of a round joined in source ranges: replay one piece's offers, then
 * close the round (the changes returned by finish are the round's total). */
int annk_shard_merge_piece(annk_state* s, uint64_t* changes);
int annk_shard_finish_round(annk_state* s, uint64_t* changes);

/* --------------------------------------------------------------- search */
/* search.cpp:23-35 GraphSearcher(base, forest, graph): validates the graph
 * and uploads it (n x graph_k ids). forest may be NULL (random init only). */
int annk_searcher_create(const annk_dataset* base, const annk_forest* f, const uint32_t* graph_ids,
                         uint32_t graph_n, uint32_t graph_k, annk_searcher** out);
int annk_searcher_destroy(annk_searcher* s);
typedef struct {
    uint32_t k_return;          /* SearchParams (search.hpp:13-21) */
    uint32_t pool_size;
    uint32_t expansion;
    uint32_t iters;
    uint32_t n_trees_used;
    uint32_t random_seed_count;
    uint64_t seed;
    int32_t random_init;        /* 1 = search_random_init (search.cpp:156-180) with per-query seed
                                   substream(seed, qi); 2 = the same with `seed` used as given */
} annk_search_params;
/* search.cpp:121-154 GraphSearcher::search for a batch of queries (host
 * nq x dim).  Per-query seed = substream(params.seed, qi) as in recall_curve
 * (search.cpp:208).  out_ids/out_dists nq*k_return; stats (nullable) nq*4 =
 * [dist_comps, leaves_visited, graph_hops, seed_points] (SearchStats). */
int annk_search(annk_searcher* s, const float* queries, uint32_t nq, uint32_t dim,
                const annk_search_params* params, uint32_t* out_ids, float* out_dists,
                uint64_t* stats);
/* Same with the queries already on the device (a dataset handle). */
int annk_search_dataset(annk_searcher* s, const annk_dataset* queries,
                        const annk_search_params* params, uint32_t* out_ids, float* out_dists,
                        uint64_t* stats);

#ifdef __cplusplus
}
#endif

#endif

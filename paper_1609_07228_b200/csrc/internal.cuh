// internal.cuh — device-resident object layouts shared by the kernels.
#pragma once

#include <memory>
#include <new>
#include <string>
#include <vector>

#include "common.cuh"

// Tree node as the kernels see it: 16 bytes, one sector per descent hop.
// (Reference KdNode, kd_forest.hpp:18-27; depth and even_split live in
// side arrays because descents never read them.)
struct __align__(16) KdNodeDev {  // one 128-bit load per descent step
    uint32_t split_dim;  // annk::kLeaf => leaf
    float split_val;
    uint32_t left;   // internal: left child; leaf: range start in point_index
    uint32_t right;  // internal: right child; leaf: range end
};

struct annk_dataset {
    uint32_t n = 0, dim = 0, ld = 0;  // ld = padded row stride (floats), multiple of 4
    annk::DevBuf<float> data;         // n x ld, zero padded
    // Exact u8 datapath: when every value is an integer in [0,255] and
    // dim * 255^2 < 2^24, the reference's sequential fp32 l2_sq never rounds,
    // so ||a||^2 + ||b||^2 - 2 a.b in int32 (dp4a) is bit-identical to it.
    bool u8 = false;
    uint32_t ld8 = 0;                 // bytes per u8 row, multiple of 16
    annk::DevBuf<uint8_t> data8;      // n x ld8, zero padded
    annk::DevBuf<int32_t> norms8;     // n squared norms
};

void make_u8(annk_dataset* ds);  // runtime.cu: enables the u8 path when exact

// Integer-exact squared distance of two u8 rows (ld8 bytes, 16-byte aligned):
// na + nb - 2 * dot, dot by dp4a on 4-byte lanes.
__device__ __forceinline__ float l2_u8(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b,
                                       uint32_t ld8, int32_t na, int32_t nb) {
    uint32_t dot = 0;  // unsigned overload: bytes are 0..255
    for (uint32_t i = 0; i < ld8; i += 16) {
        const uint4 x = *reinterpret_cast<const uint4*>(a + i);
        const uint4 y = *reinterpret_cast<const uint4*>(b + i);
        dot = __dp4a(x.x, y.x, dot);
        dot = __dp4a(x.y, y.y, dot);
        dot = __dp4a(x.z, y.z, dot);
        dot = __dp4a(x.w, y.w, dot);
    }
    return float(na + nb - 2 * int32_t(dot));
}

struct TreeDev {
    annk::DevBuf<KdNodeDev> nodes;
    annk::DevBuf<uint32_t> depth;
    annk::DevBuf<uint8_t> even;
    annk::DevBuf<uint32_t> pidx;    // point_index permutation (n)
    annk::DevBuf<uint32_t> parent;  // lazily built (init_graph)
    annk::DevBuf<uint32_t> owner;   // lazily built: leaf owning each point
    annk::DevBuf<uint32_t> sib_off;   // lazily built: per-leaf sibling lists (CSR)
    annk::DevBuf<uint32_t> sib_list;
    uint32_t num_nodes = 0, root = 0, leaf_count = 0, max_depth = 0;
};

// Plain view passed to kernels that walk several trees.
struct TreeView {
    const KdNodeDev* nodes;
    const uint32_t* depth;
    const uint32_t* pidx;
    const uint32_t* parent;
    const uint32_t* owner;
    const uint32_t* sib_off;   // per node: start of its sibling list (leaves only)
    const uint32_t* sib_list;  // leaf ancestors' siblings, nearest level first
    uint32_t root, num_nodes, leaf_count, max_depth;
};

struct annk_forest {
    uint32_t n_trees = 0, n = 0, dim = 0, leaf_cap = 0;
    uint64_t seed = 0;
    std::vector<TreeDev> trees;
    annk::DevBuf<TreeView> views;  // device copy of per-tree views
    bool links_ready = false;
};

struct annk_state {
    uint32_t n = 0, k = 0, P = 0, S = 0;
    uint64_t seed = 0;
    uint32_t iteration = 0;
    uint64_t dist_comps = 0, last_changes = 0;
    annk::DevBuf<uint64_t> keys;   // n x P ascending; kEmptyKey beyond size
    annk::DevBuf<uint8_t> flags;   // n x P flag_new
    annk::DevBuf<uint32_t> sizes;  // n
    // sampling-step scratch, reused across iterations
    annk::DevBuf<uint32_t> fnew, fold, cnew, cold;  // forward lists, pool order (n x S, n x P)
    annk::DevBuf<uint32_t> rn_cnt, ro_cnt, rn_off, ro_off, rn_cur, ro_cur, rn_data, ro_data;
    annk::DevBuf<uint32_t> gnew, gold, gncnt, gocnt;  // unioned lists, sorted (n x 2S, n x (P+S))
    annk::DevBuf<uint64_t> thr;                       // start-of-round pool tail per point
    annk::DevBuf<uint32_t> ocnt;                      // join offer counts
    annk::DevBuf<uint64_t> obuf;                      // n x offer_cap offer keys
    annk::DevBuf<uint32_t> osrc;                      // n x offer_cap source point of each offer
    annk::DevBuf<uint32_t> ov_tgt;                    // spill list: target ids
    annk::DevBuf<uint64_t> ov_key;                    // spill list: offer keys
    annk::DevBuf<uint32_t> ov_src;                    // spill list: source points
    annk::DevBuf<uint32_t> order;                     // point visit order (tree-0 leaf order) for L2 locality
    uint32_t ov_cap = 0;
    int stage = 0;  // 0 none, 1 after rebuild_sample_lists, 2 after union_reverse_lists
    bool counts_fused = false;  // the last do_sample also counted the reverse lists (unsharded)
    uint64_t join_rows = 0;
    uint32_t offer_cap = 0;
    uint64_t last_offers = 0, last_spilled = 0;
    // join -> merge hand-off (offers stay on device between the phases)
    annk::DevBuf<uint32_t> ov_count;   // spill list fill (1)
    annk::DevBuf<uint32_t> ov_off;     // per-target start in the target-sorted spill list (n + 1)
    uint32_t spilled = 0;
    bool spill_sorted = false;
    uint64_t pending_comps = 0;
    annk::DevBuf<uint32_t> rp_big;        // replay: targets deferred to the global-scratch pass
    annk::DevBuf<uint64_t> rp_runkey;     // replay scratch (grow-only): runs of the deferred targets
    annk::DevBuf<uint32_t> rp_pstart, rp_seqoff;
    uint64_t piece_changes = 0, piece_comps = 0;  // shard mode: a round joined in source ranges
    uint32_t join_pieces = 1;  // visit-list pieces per round (> 1 once a round overflowed one join launch)
    // shard mode (multi-GPU): this state owns points [lo, hi); init / sample /
    // join / merge / finalize touch only those, lists and thresholds of the
    // other points arrive through annk_state_rows
    uint32_t lo = 0, hi = 0;
    bool sharded = false;
    annk::DevBuf<uint32_t> order_own;  // visit order restricted to [lo, hi)
    annk::DevBuf<uint32_t> pack_cnt, pack_off;
    uint32_t pack_lo = 0, pack_hi = 0;
};

struct annk_searcher {
    const annk_dataset* base = nullptr;
    const annk_forest* forest = nullptr;
    uint32_t gn = 0, gk = 0;
    annk::DevBuf<uint32_t> graph;  // gn x gk
    annk::DevBuf<uint32_t> bitmap;  // search visited bitmaps (slots x words), all-zero between launches
};

namespace annk {
void set_error(const std::string& m);

// Runs f at the C-ABI boundary: exceptions become status codes + message.
template <class F>
int abi(F&& f) {
    try {
        f();
        return kOk;
    } catch (const Error& e) {
        set_error(e.what());
        return e.code;
    } catch (const std::bad_alloc&) {
        set_error("host allocation failed");
        return kOutOfMemory;
    } catch (const std::exception& e) {
        set_error(e.what());
        return kInternal;
    }
}

// parent / owner / sibling tables of every tree (init's divide-and-conquer
// walk); rebuilt on request, as the reference's init_graph rebuilds its
// equivalents on every call (graph_build.cpp:238-257)
void forest_ensure_links(annk_forest* f, bool rebuild = false);
void forest_upload_views(annk_forest* f);
// exact top-k helper used by brute force and accuracy scoring
void brute_force_device(const annk_dataset* base, const float* qdata, uint32_t q_ld, uint32_t nq,
                        const uint32_t* self_rows, uint32_t k, uint64_t* out_keys);
// merge `splits` sorted k-lists per query (nq x splits x k keys) into the final k
// (the lists need not be sorted; out_stride: keys between consecutive queries' output rows, 0 = k;
// first_sorted: list 0 is sorted and the others hold their keys first, so a query whose other
// lists are empty is copied)
void merge_split_lists(const uint64_t* part, uint32_t nq, uint32_t splits, uint32_t k, uint64_t* out_keys,
                       uint32_t out_stride = 0, bool first_sorted = false);
// exact kNN on tcgen05 (brute_force_tc.cu); false when the shape is not supported
bool brute_force_tc(const annk_dataset* base, uint32_t nq, const uint32_t* self_ids, uint32_t k,
                    uint64_t* out_keys, const uint8_t* q8, const int32_t* qnorm);
void brute_force_tc_last_scan(uint64_t* total, uint64_t* visited, int* pruned);
// exact kNN of fp32 rows: tcgen05 bf16x3 candidates + exact re-rank (brute_force_f32_tc.cu)
bool brute_force_tc_f32(const annk_dataset* base, const float* qdata, uint32_t nq, const uint32_t* self_ids,
                        uint32_t k, uint64_t* out_keys);
// the exact CUDA-core kernel for fp32 rows (brute_force.cu)
void brute_force_f32_tiles(const annk_dataset* base, const float* qdata, uint32_t nq, const uint32_t* self_ids,
                           uint32_t k, uint64_t* out_keys);
extern uint32_t g_bf_f32_overflow;
}  // namespace annk

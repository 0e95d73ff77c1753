// join.cuh — host interface of the NN-descent local join and the exact-order
// pool replay (join.cu).  Used by graph_build.cu's round driver.
#pragma once

#include "internal.cuh"

namespace annk {

// One join launch over the visit list, restricted to sources in [ilo, ihi).
// Offers land in the state's slots (obuf/osrc) or spill list (ov_*), each
// tagged with its source point.  Returns false when the launch produced more
// offers than one launch may hold (counters[1] >= limit); pools are untouched.
struct JoinCounters {
    unsigned long long comps = 0, offers = 0;
    uint32_t spilled = 0;
};
void join_launch(annk_state* s, const annk_dataset* ds, const uint32_t* order, uint32_t n_visit, uint32_t ilo,
                 uint32_t ihi, uint32_t ov_abort, JoinCounters* out);

// Groups the spill list by target (stable) so every target's offers are
// slots[0, min(cnt, cap)) followed by its spill segment.
void group_spills(annk_state* s);

// Replays the offers of targets [lo, hi) into their pools in the reference's
// sequential order (source point ascending, then the source's pair order),
// NeighborPool::insert semantics; returns the accepted inserts (`changes`).
uint64_t replay_offers(annk_state* s, uint32_t lo, uint32_t hi);

}  // namespace annk

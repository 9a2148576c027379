// feature.cuh — launch interface of the D-channel feature kernels (fp32, HBM-bound).
#pragma once
#include "tk_common.cuh"

namespace tk {

constexpr int kMaxPeers = 8;

struct GatherParams {
    int64_t n_pixels;
    int k;                 // record slots per pixel
    const int32_t* index;  // P x k
    const double* weight;  // P x k
    const uint8_t* count;  // P
    const float* feat;     // N x D
    int d;
    float* out;            // P x D
    int width, height;     // image shape (0: plain pixel order)
    // Fused gather + all-gather over peer memory: n_peers > 0 stores every output row slice into
    // peers[r] + px * peer_stride + peer_off for every rank r (its own HBM and, over NVLink, the
    // other ranks'); out is then unused.  D % 4 == 0 and peer_off % 4 == 0.
    int n_peers = 0;
    int peer_stride = 0, peer_off = 0;
    float* peers[kMaxPeers] = {};
};

struct ListGatherParams {
    int64_t n_pixels;
    const int32_t* offsets;  // P + 1
    const int32_t* src;
    const double* w;
    const float* feat;
    int d;
    float* out;
};

struct SlotKeyParams {
    int64_t n_slots;       // P x k
    int k;
    int64_t n_gaussians;
    const int32_t* index;
    const double* weight;
    const uint8_t* count;
    uint32_t* keys;        // unused (kept for layout stability)
    uint32_t* vals;        // unused
    float* wnorm;          // renormalised slot weight (render.cpp:324-329)
    int32_t* zero2 = nullptr;  // two counters zeroed on the way (launch_slot_index)
};

struct FeatBwdParams {
    int64_t n_gaussians;
    int k;
    int d;
    const int32_t* seg;    // N + 1 record offsets per Gaussian
    const uint32_t* slots; // records sorted by (Gaussian, slot)
    const float* wnorm;
    const float* grad;     // P x D
    float* out;            // N x D
};

// Gaussians with more than kLongSeg records (a near-camera Gaussian in the Top-K of most pixels
// owns one record per pixel) are not summed by one warp.  Their slot-sorted records (pixel order)
// are cut at kBands pixel-row band boundaries and into items of at most kLongItem records; each
// item is summed into its own partial row, and a Gaussian's partial rows (numbered in record
// order) are added in that order by a fixed two-level tree (groups of kCombineGroup rows, then
// the group sums), so the result never depends on execution order: deterministic.
// The items are listed band-major and a persistent grid of warps walks the list in order, one
// warp per (item, 128-channel column block), so the items in flight cover a narrow band of image
// rows and the dF rows that the long Gaussians of a pixel share are re-read from L2, not HBM.
// (Round 2 before this: kLongSeg-record items, all in flight at once, one warp per item over all
// D channels and a serial per-Gaussian combine -- 1.2 ms of a 1.7 ms feature backward at config 1,
// K = 16, DRAM-bound on dF re-reads.)
#ifndef TK_LONG_SEG
#define TK_LONG_SEG 1024
#endif
constexpr int kLongSeg = TK_LONG_SEG;
#ifndef TK_LONG_ITEM
#define TK_LONG_ITEM 128
#endif
constexpr int kLongItem = TK_LONG_ITEM;
constexpr int kBands = 32;  // one lane per band in the plan kernels
constexpr int kCombineGroup = 32;
// counters: [0] items (= partial rows), [1] long Gaussians, [2] level-1 rows, then per band:
// item counts, fill cursors, exclusive offsets
constexpr int kPlanBandCnt = 3, kPlanBandFill = kPlanBandCnt + kBands, kPlanBandOff = kPlanBandFill + kBands;
constexpr int kPlanCounters = kPlanBandOff + kBands;  // + 1: k_long_count's done counter
struct LongPlan {
    int4* items;        // {g, first record, end record, partial row}, band-major
    int4* longs;        // {g, first partial row, partial rows, first level-1 row}
    int32_t* counters;  // kPlanCounters
    int2* l1_map;       // level-1 row -> {long Gaussian, group}
    float* partial;     // cap_items x D
    float* l1;          // cap_l1 x D
    int64_t cap_items, cap_l1;
    const int32_t* queue;   // launch_slot_index's queue: long segments at its back
    const int32_t* qcount;  // number of queued long segments (device)
    const uint32_t* slots;  // records sorted by (Gaussian, slot): record -> slot
    int k, width, band_rows;
};
// capacity of the item list for m valid records among n Gaussians (each long Gaussian adds at
// most one partial item per band) and of the level-1 rows
inline int64_t long_plan_longs(int64_t m, int64_t n) { return m / kLongSeg < n ? m / kLongSeg : n; }
inline int64_t long_plan_capacity(int64_t m, int64_t n) { return m / kLongItem + long_plan_longs(m, n) * kBands + 1; }
inline int64_t long_plan_l1_capacity(int64_t m, int64_t n) {
    return long_plan_capacity(m, n) / kCombineGroup + long_plan_longs(m, n) + 1;
}

void launch_feature_gather(const GatherParams& p, cudaStream_t st);
void launch_list_gather(const ListGatherParams& p, cudaStream_t st);
// Inverted index of the records: a stable radix sort of (Gaussian id, slot) over the P x k slots.
// seg (n+1) becomes the segment offsets, *sorted_vals the valid slot ids grouped by Gaussian,
// ascending within each segment (one of vals / vals_alt).  queue: n + 2 int32 (long-segment queue
// at its back, counters at [n], [n+1]).  radix_scratch: radix_scratch_bytes(n_slots).
void launch_slot_index(const SlotKeyParams& p, int64_t n_gaussians, int32_t* seg, int32_t* queue, uint32_t* keys,
                       uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt, const uint32_t** sorted_vals,
                       void* radix_scratch, int32_t* plan_counters, cudaStream_t st);
// the long-segment queue left by launch_slot_index: entries queue[n - 1 - i] for i < queue[n + 1]
void launch_long_plan(const int32_t* seg, int64_t n, const LongPlan& plan, cudaStream_t st);
// backward_feature's reduction; long segments through plan (band-major items + two-level combine)
void launch_feature_bwd(const FeatBwdParams& p, const LongPlan& plan, cudaStream_t st);
// *first = smallest slot whose index >= n (device u64, preset to ~0)
void launch_first_stale(const int32_t* index, int64_t n_slots, int64_t n, unsigned long long* first,
                        cudaStream_t st);
// interleave [G][P][ds] shard slices into [P][G*ds]
void launch_interleave(const float* in, int64_t n_pixels, int ds, int g, float* out, cudaStream_t st);

}  // namespace tk

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

// Gaussians with more than kLongSeg records (a Gaussian filling the view owns one record per
// pixel) are not summed by one warp: their records are cut into kLongSeg chunks summed by
// separate warps into `partial`, then combined in chunk order (deterministic).  The plan is
// built on the device from the long-segment queue of launch_slot_index.
constexpr int kLongSeg = 1024;
struct LongPlan {
    int4* items;        // {g, chunk, slot in partial, -}
    int4* longs;        // {g, first partial slot, chunks, -}
    int32_t* counters;  // [0] items, [1] long Gaussians
    float* partial;     // cap_items x D
    int64_t cap_items;
    const int32_t* queue;   // launch_slot_index's cursor scratch: long queue at its back
    const int32_t* qcount;  // number of queued long segments (device)
};
// capacity of the chunk list for m valid records among n Gaussians
inline int64_t long_plan_capacity(int64_t m, int64_t n) {
    return m / kLongSeg + (m / kLongSeg < n ? m / kLongSeg : n) + 1;
}

void launch_feature_gather(const GatherParams& p, cudaStream_t st);
void launch_list_gather(const ListGatherParams& p, cudaStream_t st);
// Inverted index of the records by counting: cnt_seg (n+1) becomes the segment offsets, recs /
// sorted hold the valid slot ids grouped by Gaussian (sorted: ascending within each segment).
// cursor: n + 2 int32 of scratch.
void launch_slot_index(const SlotKeyParams& p, int64_t n_gaussians, int32_t* cnt_seg, int32_t* cursor, uint32_t* recs,
                       uint32_t* sorted, int64_t* total, void* scan_scratch, cudaStream_t st);
// the long-segment queue left in cursor by launch_slot_index: entries cursor[n - 1 - i] for
// i < cursor[n + 1]
void launch_long_plan(const int32_t* seg, int64_t n, const LongPlan& plan, cudaStream_t st);
// backward_feature's reduction; long segments through plan (chunks + ordered combine)
void launch_feature_bwd(const FeatBwdParams& p, const LongPlan& plan, cudaStream_t st);
// *first = smallest slot whose index >= n (device u64, preset to ~0)
void launch_first_stale(const int32_t* index, int64_t n_slots, int64_t n, unsigned long long* first,
                        cudaStream_t st);
// interleave [G][P][ds] shard slices into [P][G*ds]
void launch_interleave(const float* in, int64_t n_pixels, int ds, int g, float* out, cudaStream_t st);

}  // namespace tk

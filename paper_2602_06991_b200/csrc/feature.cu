// feature.cu — K5 Top-K feature gather, K6 full-blend gather, K7 feature backward, K10 stale
// check.  fp32 features, HBM-bound: one warp per output row, 128-bit loads of the K selected
// D-channel rows (read-only path) and 128-bit streaming stores of the output row.
#include "feature.cuh"

#include <algorithm>
#include <cstdlib>

#include "sort.cuh"
#include "tile_stage.cuh"
#include "tk_common.cuh"

namespace tk {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ float4 fma4(float a, float4 x, float4 acc) {
    acc.x = fmaf(a, x.x, acc.x);
    acc.y = fmaf(a, x.y, acc.y);
    acc.z = fmaf(a, x.z, acc.z);
    acc.w = fmaf(a, x.w, acc.w);
    return acc;
}

__device__ __forceinline__ float4 ldg4(const float4* p) { return __ldg(p); }

// Store float4 q of pixel px's output row: to p.out, or (fused all-gather) into every rank's
// full-width buffer at this rank's channel offset -- local HBM or a peer's over NVLink.
__device__ __forceinline__ void store_out4(const GatherParams& p, int64_t px, int q, float4 v) {
    if (p.n_peers == 0) {
        __stcs(reinterpret_cast<float4*>(p.out + px * p.d) + q, v);
        return;
    }
    for (int r = 0; r < p.n_peers; ++r)
        __stcs(reinterpret_cast<float4*>(p.peers[r] + px * p.peer_stride + p.peer_off) + q, v);
}

// Pixel of virtual index v when the image is walked in 16x16 tiles (neighbouring pixels share
// most of their Top-K Gaussians, so tile order keeps those feature rows L2-resident).
__device__ __forceinline__ int64_t tiled_pixel(int64_t v, int width, int height, int tiles_x, bool* valid) {
    const int64_t t = v >> 8;
    const int l = static_cast<int>(v & 255);
    const int x = static_cast<int>(t % tiles_x) * 16 + (l & 15), y = static_cast<int>(t / tiles_x) * 16 + (l >> 4);
    *valid = x < width && y < height;
    return static_cast<int64_t>(y) * width + x;
}

// render_feature (render.cpp:319-334) for D % 4 == 0: one warp per pixel, two pixels in flight
// per warp (all 2*K*D/128 row loads issued before the FMAs), pixels visited in tile order,
// 128-bit read-only loads of the selected rows and 128-bit streaming stores of the output row.
__global__ void __launch_bounds__(kThreads) k_gather_tiled(GatherParams p) {
    pdl_prologue();
    const int lane = threadIdx.x & 31;
    const int64_t nw = static_cast<int64_t>(gridDim.x) * kWarps;
    const int D = p.d, d4 = D >> 2;
    const int tiles_x = (p.width + 15) / 16, tiles_y = (p.height + 15) / 16;
    const int64_t nv = static_cast<int64_t>(tiles_x) * tiles_y * 256;
    for (int64_t v0 = ((static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5) * 2; v0 < nv; v0 += nw * 2) {
        int64_t px[2];
        int c[2], id[2];
        float wn[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            bool valid;
            px[u] = tiled_pixel(v0 + u, p.width, p.height, tiles_x, &valid);
            // the record slots load alongside the count (one memory round trip, not two)
            int idl = 0;
            double wdl = 0.0;
            if (valid && lane < p.k) {
                idl = p.index[px[u] * p.k + lane];
                wdl = p.weight[px[u] * p.k + lane];
            }
            c[u] = valid ? p.count[px[u]] : 0;
            const double wd = lane < c[u] ? wdl : 0.0;
            id[u] = lane < c[u] ? idl : 0;
            double sum = 0.0;
            for (int j = 0; j < c[u]; ++j) sum += __shfl_sync(0xffffffffu, wd, j);
            wn[u] = lane < c[u] ? static_cast<float>(wd / sum) : 0.0f;
            c[u] = valid ? c[u] : -1;  // -1: outside the image, nothing to write
        }
        const int cmax = max(c[0], c[1]);
        for (int base = 0; base < d4; base += 128) {
            float4 acc[2][4];
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
                for (int m = 0; m < 4; ++m) acc[u][m] = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int j = 0; j < cmax; ++j) {
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int g = __shfl_sync(0xffffffffu, id[u], j);
                    const float wj = __shfl_sync(0xffffffffu, wn[u], j);
                    if (j < c[u]) {
                        const float4* row = reinterpret_cast<const float4*>(p.feat + static_cast<int64_t>(g) * D);
#pragma unroll
                        for (int m = 0; m < 4; ++m) {
                            const int q = base + m * 32 + lane;
                            if (q < d4) acc[u][m] = fma4(wj, ldg4(row + q), acc[u][m]);
                        }
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                if (c[u] < 0) continue;
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    const int q = base + m * 32 + lane;
                    if (q < d4) store_out4(p, px[u], q, acc[u][m]);
                }
            }
        }
    }
    if (p.n_peers > 0) __threadfence_system();  // peer stores complete before the rank barrier
}

// render_feature (render.cpp:319-334) over tile-staged rows (tile_stage.cuh): one CTA per
// 16 x 16 pixel tile (persistent over tiles), then warp w writes pixels 32w..32w+31 (lane =
// channel quad), each record's row read from shared memory or, unstaged, from global memory.
// F is bit-identical to k_gather_tiled's (same weights, same slot-order FMAs per channel).
constexpr int kGSide = kStageSide, kGPix = kStagePix;

// Is channel quad q (lane's quad m of the pass) inside the row?  MODE 2: always; MODE 1: the
// pass's valid quad groups (warp-uniform); MODE 0: per lane.
template <int MODE>
__device__ __forceinline__ bool quad_ok(int q, int m, int d4, int mq) {
    return MODE == 2 ? true : (MODE == 1 ? m < mq : q < d4);
}

// MODE 2 ("full"): D % 512 == 0 and no peers (the common case) -- no per-quad bounds checks, plain
// streaming stores; MODE 1: D % 128 == 0 and no peers -- warp-uniform bounds per pass (D = 768);
// MODE 0: generic.  The arithmetic is identical in all three.
// stores; the arithmetic is identical.
template <int KMAX, int MODE>
__global__ void __launch_bounds__(kGPix, 2) k_gather_staged(GatherParams p, int rows) {
    pdl_prologue();
    extern __shared__ __align__(128) unsigned char gsm[];
    const int D = p.d, d4 = D >> 2;
    const StageSmem sm = stage_layout<KMAX>(gsm, rows, D);
    const float* srow = sm.srow;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tiles_x = (p.width + kGSide - 1) / kGSide, tiles_y = (p.height + kGSide - 1) / kGSide;
    stage_init(sm);
    unsigned phase = 0;
    for (int tile = blockIdx.x; tile < tiles_x * tiles_y; tile += gridDim.x) {
        const int tx0 = (tile % tiles_x) * kGSide, ty0 = (tile / tiles_x) * kGSide;
        const int x = tx0 + (tid % kGSide), y = ty0 + tid / kGSide;
        const bool in = x < p.width && y < p.height;
        const int64_t px = static_cast<int64_t>(y) * p.width + x;
        const StagedPixel<KMAX> sp =
            stage_tile<KMAX>(sm, rows, D, p.feat, p.index, p.weight, p.k, px, in ? p.count[px] : -1, phase);
        const int c = sp.c;
        int slot[KMAX];
        float wn[KMAX];
#pragma unroll
        for (int j = 0; j < KMAX; ++j) {
            slot[j] = sp.slot[j];
            wn[j] = sp.wn[j];
        }
        // warp w: the tile's pixels 32w .. 32w + 31, two at a time
        for (int i = 0; i < 32; i += 2) {
            int ci[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) ci[u] = __shfl_sync(0xffffffffu, c, i + u);
            for (int base = 0; base < d4; base += 128) {
                const int mq = (d4 - base) >> 5;  // MODE 1: quads groups valid in this pass
                float4 acc[2][4];
#pragma unroll
                for (int u = 0; u < 2; ++u)
#pragma unroll
                    for (int m = 0; m < 4; ++m) acc[u][m] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int j = 0; j < KMAX; ++j) {
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int sj = __shfl_sync(0xffffffffu, slot[j], i + u);
                        const float wj = __shfl_sync(0xffffffffu, wn[j], i + u);
                        if (j < ci[u] && sj >= 0) {  // staged row (shared memory)
                            const float4* row = reinterpret_cast<const float4*>(srow + static_cast<size_t>(sj) * D);
#pragma unroll
                            for (int m = 0; m < 4; ++m) {
                                const int q = base + m * 32 + lane;
                                if (quad_ok<MODE>(q, m, d4, mq)) acc[u][m] = fma4(wj, row[q], acc[u][m]);
                            }
                        } else if (j < ci[u]) {  // beyond the staged set: global (L2)
                            const float4* row = reinterpret_cast<const float4*>(p.feat + static_cast<int64_t>(-1 - sj) * D);
#pragma unroll
                            for (int m = 0; m < 4; ++m) {
                                const int q = base + m * 32 + lane;
                                if (quad_ok<MODE>(q, m, d4, mq)) acc[u][m] = fma4(wj, ldg4(row + q), acc[u][m]);
                            }
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    if (ci[u] < 0) continue;
                    const int t = warp * 32 + i + u;
                    const int64_t pxo = static_cast<int64_t>(ty0 + t / kGSide) * p.width + tx0 + (t % kGSide);
#pragma unroll
                    for (int m = 0; m < 4; ++m) {
                        const int q = base + m * 32 + lane;
                        if (MODE >= 1) {
                            if (quad_ok<MODE>(q, m, d4, mq)) __stcs(reinterpret_cast<float4*>(p.out + pxo * p.d) + q, acc[u][m]);
                        } else if (q < d4) store_out4(p, pxo, q, acc[u][m]);
                    }
                }
            }
        }
        __syncthreads();  // the staged rows and the hash are reused by the next tile
    }
    if (p.n_peers > 0) __threadfence_system();  // peer stores complete before the rank barrier
}

// render_feature (render.cpp:319-334): F[p] = sum_j (w_j / sum_w) f[idx_j], sum in slot order.
template <bool VEC>
__global__ void __launch_bounds__(kThreads) k_gather(GatherParams p) {
    pdl_prologue();
    const int lane = threadIdx.x & 31;
    const int64_t nw = static_cast<int64_t>(gridDim.x) * kWarps;
    const int D = p.d;
    for (int64_t px = (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5; px < p.n_pixels; px += nw) {
        const int c = p.count[px];
        int id = 0;
        double wd = 0.0;
        if (lane < c) {
            id = p.index[px * p.k + lane];
            wd = p.weight[px * p.k + lane];
        }
        double sum = 0.0;
        for (int j = 0; j < c; ++j) sum += __shfl_sync(0xffffffffu, wd, j);
        const float wn = lane < c ? static_cast<float>(wd / sum) : 0.0f;
        if (VEC) {
            const int d4 = D >> 2;
            float4* orow = reinterpret_cast<float4*>(p.out + px * D);
            for (int base = 0; base < d4; base += 128) {
                float4 acc[4];
#pragma unroll
                for (int m = 0; m < 4; ++m) acc[m] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 2
                for (int j = 0; j < c; ++j) {
                    const int g = __shfl_sync(0xffffffffu, id, j);
                    const float wj = __shfl_sync(0xffffffffu, wn, j);
                    const float4* row = reinterpret_cast<const float4*>(p.feat + static_cast<int64_t>(g) * D);
#pragma unroll
                    for (int m = 0; m < 4; ++m) {
                        const int q = base + m * 32 + lane;
                        if (q < d4) acc[m] = fma4(wj, ldg4(row + q), acc[m]);
                    }
                }
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    const int q = base + m * 32 + lane;
                    if (q < d4) __stcs(orow + q, acc[m]);
                }
            }
        } else {
            float* orow = p.out + px * D;
            for (int base = 0; base < D; base += 128) {
                float acc[4] = {0.f, 0.f, 0.f, 0.f};
                for (int j = 0; j < c; ++j) {
                    const int g = __shfl_sync(0xffffffffu, id, j);
                    const float wj = __shfl_sync(0xffffffffu, wn, j);
                    const float* row = p.feat + static_cast<int64_t>(g) * D;
#pragma unroll
                    for (int m = 0; m < 4; ++m) {
                        const int q = base + m * 32 + lane;
                        if (q < D) acc[m] = fmaf(wj, __ldg(row + q), acc[m]);
                    }
                }
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    const int q = base + m * 32 + lane;
                    if (q < D) __stcs(orow + q, acc[m]);
                }
            }
        }
    }
}

// feature_pass_full_blend (render.cpp:277-280): F[p] = sum_i w_i f_i over the contributor list.
template <bool VEC>
__global__ void __launch_bounds__(kThreads) k_list_gather(ListGatherParams p) {
    pdl_prologue();
    const int lane = threadIdx.x & 31;
    const int64_t nw = static_cast<int64_t>(gridDim.x) * kWarps;
    const int D = p.d;
    for (int64_t px = (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5; px < p.n_pixels; px += nw) {
        const int r0 = p.offsets[px], r1 = p.offsets[px + 1];
        const int step = VEC ? 128 : 128;
        const int dd = VEC ? D >> 2 : D;
        for (int base = 0; base < dd; base += step) {
            float4 acc4[4];
            float acc1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int m = 0; m < 4; ++m) acc4[m] = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int r = r0; r < r1; r += 32) {
                const int nr = min(32, r1 - r);
                int sid = 0;
                float sw = 0.f;
                if (lane < nr) {
                    sid = p.src[r + lane];
                    sw = static_cast<float>(p.w[r + lane]);
                }
                for (int j = 0; j < nr; ++j) {
                    const int g = __shfl_sync(0xffffffffu, sid, j);
                    const float wj = __shfl_sync(0xffffffffu, sw, j);
                    if (VEC) {
                        const float4* row = reinterpret_cast<const float4*>(p.feat + static_cast<int64_t>(g) * D);
#pragma unroll
                        for (int m = 0; m < 4; ++m) {
                            const int q = base + m * 32 + lane;
                            if (q < dd) acc4[m] = fma4(wj, ldg4(row + q), acc4[m]);
                        }
                    } else {
                        const float* row = p.feat + static_cast<int64_t>(g) * D;
#pragma unroll
                        for (int m = 0; m < 4; ++m) {
                            const int q = base + m * 32 + lane;
                            if (q < dd) acc1[m] = fmaf(wj, __ldg(row + q), acc1[m]);
                        }
                    }
                }
            }
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const int q = base + m * 32 + lane;
                if (q < dd) {
                    if (VEC) __stcs(reinterpret_cast<float4*>(p.out + px * D) + q, acc4[m]);
                    else __stcs(p.out + px * D + q, acc1[m]);
                }
            }
        }
    }
}

// Inverted index (Gaussian -> record slots) by a stable radix sort: key = Gaussian id of the slot
// (n for an empty slot: it sorts past every segment), value = slot id.  Slots enter in ascending
// order and the LSD sort is stable, so every Gaussian's records come out in slot (pixel, j) order
// -- the fixed reduction order of backward_feature -- with no atomics and no per-segment sort, at a
// cost independent of how many records one Gaussian owns (a near-camera Gaussian in the Top-K of
// every pixel: one segment of P records).  The renormalised slot weight is computed on the way.
__global__ void k_slot_keys(SlotKeyParams p, uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    pdl_prologue();
    const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p.zero2 && s < 2) p.zero2[s] = 0;
    if (s >= p.n_slots) return;
    const int64_t px = s / p.k;
    const int j = static_cast<int>(s - px * p.k);
    const int c = p.count[px];
    const int32_t id = p.index[s];
    float wn = 0.0f;
    uint32_t key = static_cast<uint32_t>(p.n_gaussians);
    if (j < c && id >= 0) {
        key = static_cast<uint32_t>(id);
        double sum = 0.0;                                    // backward.cpp:303-304, slot order
        for (int jj = 0; jj < c; ++jj) sum += p.weight[px * p.k + jj];
        wn = static_cast<float>(p.weight[s] / sum);
    }
    p.wnorm[s] = wn;
    keys[s] = key;
    vals[s] = static_cast<uint32_t>(s);
}

// Segments longer than kLongSeg go to the chunked path: queued at the back of `queue`
// (queue[n - 1 - i], i < counts[1]); the queue order is irrelevant (each segment is summed by its
// own chunks and combined in chunk order).
__global__ void k_long_queue(const int32_t* __restrict__ seg, int64_t n, int32_t* __restrict__ queue,
                             int32_t* __restrict__ counts, int32_t* __restrict__ plan_counters) {
    pdl_prologue();
    if (plan_counters && blockIdx.x == 0)  // the long plan's counters start at zero (no memset)
        for (int i = threadIdx.x; i < kPlanCounters + 1; i += blockDim.x) plan_counters[i] = 0;
    for (int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < n;
         g += static_cast<int64_t>(gridDim.x) * blockDim.x)
        if (seg[g + 1] - seg[g] > kLongSeg) queue[n - 1 - atomicAdd(counts + 1, 1)] = static_cast<int32_t>(g);
}

// Inverted index (Gaussian -> record slots) by counting: count, scan, fill, then sort every
// segment by slot so the reduction order never depends on the atomic fill order.
// Sum of w_j * dF[px_j] over records [r0, r1) of a segment for the channel pass at `base`
// (acc4: 4 float4 per lane when VEC, acc1: 4 floats otherwise), records in slot order.
template <bool VEC, int MODE = 0>
__device__ __forceinline__ void accum_records(const FeatBwdParams& p, int r0, int r1, int base, int lane,
                                              float4 (&acc4)[4], float (&acc1)[4]) {
    const int D = p.d;
    const int dd = VEC ? D >> 2 : D;
    for (int r = r0; r < r1; r += 32) {
        const int nr = min(32, r1 - r);
        int64_t spx = 0;
        float sw = 0.f;
        if (lane < nr) {
            const uint32_t s = p.slots[r + lane];
            spx = static_cast<int64_t>(s / static_cast<uint32_t>(p.k));
            sw = p.wnorm[s];
        }
#pragma unroll 2
        for (int j = 0; j < nr; ++j) {
            const int64_t pxj = __shfl_sync(0xffffffffu, spx, j);
            float wj = __shfl_sync(0xffffffffu, sw, j);
            if (!isfinite(wj)) {
                // Zero-weight records: the reference skips pixels whose gradient row is all zero
                // (backward.cpp:296-302), so 0/0 only propagates for live rows.
                bool any = false;
                for (int q = lane; q < D; q += 32) any |= p.grad[pxj * D + q] != 0.0f;
                if (!__any_sync(0xffffffffu, any)) continue;
            }
            if (VEC) {
                const float4* row = reinterpret_cast<const float4*>(p.grad + pxj * D);
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    const int q = base + m * 32 + lane;
                    if (quad_ok<MODE>(q, m, dd, (dd - base) >> 5)) acc4[m] = fma4(wj, ldg4(row + q), acc4[m]);
                }
            } else {
                const float* row = p.grad + pxj * D;
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    const int q = base + m * 32 + lane;
                    if (q < dd) acc1[m] = fmaf(wj, __ldg(row + q), acc1[m]);
                }
            }
        }
    }
}

template <bool VEC, int MODE = 0>
__device__ __forceinline__ void store_pass(float* dst, int dd, int base, int lane, const float4 (&acc4)[4],
                                           const float (&acc1)[4]) {
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        const int q = base + m * 32 + lane;
        if (quad_ok<(VEC ? MODE : 0)>(q, m, dd, (dd - base) >> 5)) {
            if (VEC) __stcs(reinterpret_cast<float4*>(dst) + q, acc4[m]);
            else __stcs(dst + q, acc1[m]);
        }
    }
}

// backward_feature (backward.cpp:288-319) as a deterministic segmented reduction: one warp per
// Gaussian sums its records in (pixel, slot) order and writes the dense row once (segments
// longer than kLongSeg are left to the chunk / combine kernels).
// MODE (quad_ok): 2 = VEC with D % 512 == 0, 0 = generic (the D % 128 mode measured no gain here:
// 3.576 against 3.564 ms at config 5)
template <bool VEC, int MODE>
__global__ void __launch_bounds__(kThreads) k_feat_bwd(FeatBwdParams p) {
    pdl_prologue();
    const int lane = threadIdx.x & 31;
    const int64_t nw = static_cast<int64_t>(gridDim.x) * kWarps;
    const int dd = VEC ? p.d >> 2 : p.d;
    for (int64_t g = (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5; g < p.n_gaussians; g += nw) {
        const int r0 = p.seg[g], r1 = p.seg[g + 1];
        if (r1 - r0 > kLongSeg) continue;
        for (int base = 0; base < dd; base += 128) {
            float4 acc4[4];
            float acc1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int m = 0; m < 4; ++m) acc4[m] = make_float4(0.f, 0.f, 0.f, 0.f);
            accum_records<VEC, MODE>(p, r0, r1, base, lane, acc4, acc1);
            store_pass<VEC, MODE>(p.out + g * p.d, dd, base, lane, acc4, acc1);
        }
    }
}

// ---- long segments: band-major plan (feature.cuh)
__device__ __forceinline__ int record_row(const LongPlan& pl, int r) {
    return static_cast<int>((pl.slots[r] / static_cast<uint32_t>(pl.k)) / static_cast<uint32_t>(pl.width));
}

// Lane b's band of records [lo, hi) within [r0, r1): records ascend in slot (pixel) order, so
// band b starts at the first record on pixel row >= b * band_rows.
__device__ __forceinline__ void band_range(const LongPlan& pl, int r0, int r1, int lane, int& lo, int& hi) {
    int a = r0, b = r1;
    if (lane > 0) {
        const int row0 = lane * pl.band_rows;
        while (a < b) {
            const int mid = (a + b) >> 1;
            if (record_row(pl, mid) < row0) a = mid + 1;
            else b = mid;
        }
    }
    lo = a;
    hi = __shfl_down_sync(0xffffffffu, lo, 1);
    if (lane == kBands - 1) hi = r1;
}

// One warp per queued long segment: its items per band, its partial rows (numbered in record
// order), its level-1 groups.
__global__ void __launch_bounds__(kThreads) k_long_count(const int32_t* __restrict__ seg, int64_t n, LongPlan pl) {
    pdl_prologue();
    const int lane = threadIdx.x & 31;
    const int64_t nw = static_cast<int64_t>(gridDim.x) * kWarps;
    const int nq = *pl.qcount;
    for (int64_t i = (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5; i < nq; i += nw) {
        const int g = pl.queue[n - 1 - i];
        const int r0 = seg[g], r1 = seg[g + 1];
        if (r1 - r0 <= kLongSeg) continue;
        int lo, hi;
        band_range(pl, r0, r1, lane, lo, hi);
        const int nb = (hi - lo + kLongItem - 1) / kLongItem;
        const int ng = static_cast<int>(__reduce_add_sync(0xffffffffu, static_cast<unsigned>(nb)));
        const int ngrp = (ng + kCombineGroup - 1) / kCombineGroup;
        int base = 0, li = 0, l1 = 0;
        if (lane == 0) {
            base = atomicAdd(&pl.counters[0], ng);
            li = atomicAdd(&pl.counters[1], 1);
            l1 = atomicAdd(&pl.counters[2], ngrp);
            pl.longs[li] = make_int4(g, base, ng, l1);
        }
        li = __shfl_sync(0xffffffffu, li, 0);
        l1 = __shfl_sync(0xffffffffu, l1, 0);
        for (int q = lane; q < ngrp; q += 32) pl.l1_map[l1 + q] = make_int2(li, q);
        if (nb > 0) atomicAdd(&pl.counters[kPlanBandCnt + lane], nb);
    }
    // the last block to finish turns the band counts into the bands' offsets in the item list
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&pl.counters[kPlanCounters], 1) == static_cast<int>(gridDim.x) - 1;
    __syncthreads();
    if (last && threadIdx.x < 32) {
        __threadfence();
        const int v = atomicAdd(&pl.counters[kPlanBandCnt + lane], 0);  // L2 value
        int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += u;
        }
        pl.counters[kPlanBandOff + lane] = x - v;
    }
}

// One warp per long Gaussian: its items into the band-major list (the order within a band is
// the atomics' order and irrelevant: every item owns its partial row).
__global__ void __launch_bounds__(kThreads) k_long_fill(const int32_t* __restrict__ seg, LongPlan pl) {
    pdl_prologue();
    const int lane = threadIdx.x & 31;
    const int64_t nw = static_cast<int64_t>(gridDim.x) * kWarps;
    const int nl = pl.counters[1];
    for (int64_t li = (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5; li < nl; li += nw) {
        const int4 lg = pl.longs[li];
        const int g = lg.x;
        int lo, hi;
        band_range(pl, seg[g], seg[g + 1], lane, lo, hi);
        const int nb = (hi - lo + kLongItem - 1) / kLongItem;
        int local = nb;  // exclusive scan over the bands: first partial row of this band
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, local, o);
            if (lane >= o) local += u;
        }
        local -= nb;
        if (nb > 0) {
            const int pos = pl.counters[kPlanBandOff + lane] + atomicAdd(&pl.counters[kPlanBandFill + lane], nb);
            for (int c = 0; c < nb; ++c)
                pl.items[pos + c] = make_int4(g, lo + c * kLongItem, min(hi, lo + (c + 1) * kLongItem), lg.y + local + c);
        }
    }
}

// Column helpers of the long-segment kernels: VEC = float4 columns, else float columns.
template <bool VEC> struct Col;
template <> struct Col<true> {
    using T = float4;
    static __device__ __forceinline__ T zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
    static __device__ __forceinline__ T ld(const float* row, int q) { return __ldg(reinterpret_cast<const float4*>(row) + q); }
    static __device__ __forceinline__ T ldcs(const float* row, int q) { return __ldcs(reinterpret_cast<const float4*>(row) + q); }
    static __device__ __forceinline__ void st(float* row, int q, T v) { reinterpret_cast<float4*>(row)[q] = v; }
    static __device__ __forceinline__ T fma(float w, T x, T a) { return fma4(w, x, a); }
    static __device__ __forceinline__ T add(T a, T b) { return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w); }
};
template <> struct Col<false> {
    using T = float;
    static __device__ __forceinline__ T zero() { return 0.f; }
    static __device__ __forceinline__ T ld(const float* row, int q) { return __ldg(row + q); }
    static __device__ __forceinline__ T ldcs(const float* row, int q) { return __ldcs(row + q); }
    static __device__ __forceinline__ void st(float* row, int q, T v) { row[q] = v; }
    static __device__ __forceinline__ T fma(float w, T x, T a) { return fmaf(w, x, a); }
    static __device__ __forceinline__ T add(T a, T b) { return a + b; }
};

// Persistent warps over the band-major (item, 32-column block) list: the item's records summed
// in slot order into its partial row (per channel: acc = fma(w_j, dF_j, acc), j ascending, as in
// accum_records), eight record rows in flight per lane.
template <bool VEC>
#ifndef TK_ITEMS_MINB
#define TK_ITEMS_MINB 3
#endif
#ifndef TK_ITEMS_DEPTH
#define TK_ITEMS_DEPTH 8
#endif
__global__ void __launch_bounds__(kThreads, TK_ITEMS_MINB) k_feat_bwd_items(FeatBwdParams p, LongPlan plan) {
    pdl_prologue();
    using C = Col<VEC>;
    const int lane = threadIdx.x & 31;
    const int64_t nw = static_cast<int64_t>(gridDim.x) * kWarps;
    const int D = p.d;
    const int dd = VEC ? D >> 2 : D;
    const int parts = (dd + 31) >> 5;
    const int64_t ntask = static_cast<int64_t>(plan.counters[0]) * parts;
    for (int64_t t = (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5; t < ntask; t += nw) {
        const int it = static_cast<int>(t / parts);
        const int q = static_cast<int>(t - static_cast<int64_t>(it) * parts) * 32 + lane;
        const bool on = q < dd;
        const int4 item = plan.items[it];
        typename C::T acc = C::zero();
        for (int r = item.y; r < item.z; r += 32) {
            const int nr = min(32, item.z - r);
            int64_t spx = 0;
            float sw = 0.f;
            if (lane < nr) {
                const uint32_t s = p.slots[r + lane];
                spx = static_cast<int64_t>(s / static_cast<uint32_t>(p.k));
                sw = p.wnorm[s];
            }
            if (!__any_sync(0xffffffffu, lane < nr && !isfinite(sw))) {
                int j = 0;
                for (; j + TK_ITEMS_DEPTH <= nr; j += TK_ITEMS_DEPTH) {
                    typename C::T v[TK_ITEMS_DEPTH];
                    float w[TK_ITEMS_DEPTH];
#pragma unroll
                    for (int u = 0; u < TK_ITEMS_DEPTH; ++u) {
                        const int64_t px = __shfl_sync(0xffffffffu, spx, j + u);
                        w[u] = __shfl_sync(0xffffffffu, sw, j + u);
                        v[u] = on ? C::ld(p.grad + px * D, q) : C::zero();
                    }
#pragma unroll
                    for (int u = 0; u < TK_ITEMS_DEPTH; ++u) acc = C::fma(w[u], v[u], acc);
                }
                for (; j < nr; ++j) {
                    const int64_t px = __shfl_sync(0xffffffffu, spx, j);
                    const float wj = __shfl_sync(0xffffffffu, sw, j);
                    if (on) acc = C::fma(wj, C::ld(p.grad + px * D, q), acc);
                }
            } else {
                for (int j = 0; j < nr; ++j) {
                    const int64_t pxj = __shfl_sync(0xffffffffu, spx, j);
                    const float wj = __shfl_sync(0xffffffffu, sw, j);
                    if (!isfinite(wj)) {  // as accum_records: only live gradient rows propagate 0/0
                        bool any = false;
                        for (int c = lane; c < D; c += 32) any |= p.grad[pxj * D + c] != 0.0f;
                        if (!__any_sync(0xffffffffu, any)) continue;
                    }
                    if (on) acc = C::fma(wj, C::ld(p.grad + pxj * D, q), acc);
                }
            }
        }
        if (on) C::st(plan.partial + static_cast<int64_t>(item.w) * D, q, acc);
    }
}

// Level 1 of the combine: each group of kCombineGroup consecutive partial rows of a long
// Gaussian added in row order (all loads of the group issued before the adds).
template <bool VEC>
__global__ void __launch_bounds__(kThreads) k_long_combine1(FeatBwdParams p, LongPlan plan) {
    pdl_prologue();
    using C = Col<VEC>;
    const int lane = threadIdx.x & 31;
    const int64_t nw = static_cast<int64_t>(gridDim.x) * kWarps;
    const int D = p.d;
    const int dd = VEC ? D >> 2 : D;
    const int parts = (dd + 31) >> 5;
    const int64_t ntask = static_cast<int64_t>(plan.counters[2]) * parts;
    for (int64_t t = (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5; t < ntask; t += nw) {
        const int r = static_cast<int>(t / parts);
        const int q = static_cast<int>(t - static_cast<int64_t>(r) * parts) * 32 + lane;
        if (q >= dd) continue;
        const int2 m = plan.l1_map[r];
        const int4 lg = plan.longs[m.x];
        const int c0 = m.y * kCombineGroup, c1 = min(lg.z, c0 + kCombineGroup);
        const float* base = plan.partial + static_cast<int64_t>(lg.y) * D;
        typename C::T acc = C::zero();
        int c = c0;
        for (; c + 8 <= c1; c += 8) {
            typename C::T v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = C::ldcs(base + static_cast<int64_t>(c + u) * D, q);
#pragma unroll
            for (int u = 0; u < 8; ++u) acc = C::add(acc, v[u]);
        }
        for (; c < c1; ++c) acc = C::add(acc, C::ldcs(base + static_cast<int64_t>(c) * D, q));
        C::st(plan.l1 + static_cast<int64_t>(r) * D, q, acc);
    }
}

// Level 2: a long Gaussian's group sums added in group order, the dense row written once.
template <bool VEC>
__global__ void __launch_bounds__(kThreads) k_long_combine2(FeatBwdParams p, LongPlan plan) {
    pdl_prologue();
    using C = Col<VEC>;
    const int lane = threadIdx.x & 31;
    const int64_t nw = static_cast<int64_t>(gridDim.x) * kWarps;
    const int D = p.d;
    const int dd = VEC ? D >> 2 : D;
    const int parts = (dd + 31) >> 5;
    const int64_t ntask = static_cast<int64_t>(plan.counters[1]) * parts;
    for (int64_t t = (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5; t < ntask; t += nw) {
        const int li = static_cast<int>(t / parts);
        const int q = static_cast<int>(t - static_cast<int64_t>(li) * parts) * 32 + lane;
        if (q >= dd) continue;
        const int4 lg = plan.longs[li];
        const int ngrp = (lg.z + kCombineGroup - 1) / kCombineGroup;
        const float* base = plan.l1 + static_cast<int64_t>(lg.w) * D;
        typename C::T acc = C::zero();
        int c = 0;
        for (; c + 8 <= ngrp; c += 8) {
            typename C::T v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = C::ldcs(base + static_cast<int64_t>(c + u) * D, q);
#pragma unroll
            for (int u = 0; u < 8; ++u) acc = C::add(acc, v[u]);
        }
        for (; c < ngrp; ++c) acc = C::add(acc, C::ldcs(base + static_cast<int64_t>(c) * D, q));
        C::st(p.out + static_cast<int64_t>(lg.x) * D, q, acc);
    }
}

// First slot (in slot order) whose index is >= n: the reference throws on it (render.cpp:305-311).
__global__ void k_first_stale(const int32_t* __restrict__ index, int64_t n_slots, int64_t n,
                              unsigned long long* __restrict__ first) {
    pdl_prologue();
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n_slots;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        if (index[i] >= n) atomicMin(first, static_cast<unsigned long long>(i));
}

__global__ void k_interleave(const float* __restrict__ in, int64_t n_pixels, int ds, int g, float* __restrict__ out) {
    pdl_prologue();
    const int64_t total = n_pixels * g * ds;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t px = i / (static_cast<int64_t>(g) * ds);
        const int64_t rem = i - px * g * ds;
        const int r = static_cast<int>(rem / ds), c = static_cast<int>(rem - static_cast<int64_t>(r) * ds);
        out[i] = in[(static_cast<int64_t>(r) * n_pixels + px) * ds + c];
    }
}

inline unsigned warp_grid(int64_t rows) {
    const int64_t blocks = (rows + kWarps - 1) / kWarps;
    const int64_t cap = 148LL * 32;
    return static_cast<unsigned>(blocks < cap ? (blocks > 0 ? blocks : 1) : cap);
}

// One warp per row with no grid-stride cap.  Observed on this driver and B200 (not guaranteed by
// CUDA): blocks are dispatched roughly in index order, so the warps in flight cover a narrow
// window of rows (k_feat_bwd: the <= K Gaussians that read a pixel's dF row are then closer in
// time; 0.745 -> 0.729 ms against the capped persistent grid, warp_grid, kept as the fallback if
// a later measurement regresses).  Correctness never depends on the order.
inline unsigned warp_grid_all(int64_t rows) {
    return static_cast<unsigned>(std::max<int64_t>(1, (rows + kWarps - 1) / kWarps));
}

inline bool vec_ok(const void* a, const void* b, int d) {
    return (d % 4) == 0 && (reinterpret_cast<uintptr_t>(a) % 16) == 0 && (reinterpret_cast<uintptr_t>(b) % 16) == 0;
}

}  // namespace

// Shared memory of k_gather_staged: staged rows + hash (keys, slots) + row ids + counters/barrier
// (TK_GATHER_SMEM_KB overrides, experiments).
size_t staged_smem() {
    static const size_t b = [] {
        const char* e = std::getenv("TK_GATHER_SMEM_KB");
        const int kb = e ? std::atoi(e) : 0;
        return static_cast<size_t>(kb >= 24 && kb <= 224 ? kb : 112) * 1024;
    }();
    return b;
}

template <int KMAX, int MODE>
void launch_gather_staged_impl(const GatherParams& p, int rows, size_t budget, cudaStream_t st) {
    static FuncAttrCache attr;
    set_func_attr(attr, reinterpret_cast<const void*>(k_gather_staged<KMAX, MODE>),
                  cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(budget));
    const size_t smem = stage_smem_bytes<KMAX>(rows, p.d);
    const int tiles = ((p.width + kGSide - 1) / kGSide) * ((p.height + kGSide - 1) / kGSide);
    const int per_sm = static_cast<int>(std::max<size_t>(1, (227 * 1024) / (smem + 1024)));
    launch_k<false>(k_gather_staged<KMAX, MODE>, std::min(tiles, 148 * per_sm), kGPix, smem, st, p, rows);
}

template <int KMAX>
bool launch_gather_staged(const GatherParams& p, cudaStream_t st) {
    const size_t budget = staged_smem();
    const int rows = stage_rows<KMAX>(budget, p.d);
    if (rows < 8) return false;
    if (p.n_peers == 0 && p.d % 512 == 0) launch_gather_staged_impl<KMAX, 2>(p, rows, budget, st);
    else if (p.n_peers == 0 && p.d % 128 == 0) launch_gather_staged_impl<KMAX, 1>(p, rows, budget, st);
    else launch_gather_staged_impl<KMAX, 0>(p, rows, budget, st);
    return true;
}

bool gather_staged_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("TK_GATHER_STAGED");
        return !(e && e[0] == '0');
    }();
    return on;
}

void launch_feature_gather(const GatherParams& p, cudaStream_t st) {
    if (p.n_pixels <= 0 || p.d <= 0) return;
    const bool img = p.width > 0 && static_cast<int64_t>(p.width) * p.height == p.n_pixels;
    if (vec_ok(p.feat, p.out, p.d) && img && gather_staged_enabled() && p.k <= 8 &&
        (p.k <= 3 ? launch_gather_staged<3>(p, st) : p.k <= 4 ? launch_gather_staged<4>(p, st) : launch_gather_staged<8>(p, st))) {
        dbg_launch("k_gather_staged", st);
        return;
    }
    if (vec_ok(p.feat, p.out, p.d) && img)
        launch_k<false>(k_gather_tiled, warp_grid((p.n_pixels + 1) / 2), kThreads, 0, st, p);
    else if (vec_ok(p.feat, p.out, p.d)) launch_k<false>(k_gather<true>, warp_grid(p.n_pixels), kThreads, 0, st, p);
    else launch_k<false>(k_gather<false>, warp_grid(p.n_pixels), kThreads, 0, st, p);
    dbg_launch("k_gather", st);
}

void launch_list_gather(const ListGatherParams& p, cudaStream_t st) {
    if (p.n_pixels <= 0 || p.d <= 0) return;
    if (vec_ok(p.feat, p.out, p.d)) launch_k<false>(k_list_gather<true>, warp_grid(p.n_pixels), kThreads, 0, st, p);
    else launch_k<false>(k_list_gather<false>, warp_grid(p.n_pixels), kThreads, 0, st, p);
    dbg_launch("k_list_gather", st);
}

void launch_slot_index(const SlotKeyParams& p, int64_t n_gaussians, int32_t* seg, int32_t* queue, uint32_t* keys,
                       uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt, const uint32_t** sorted_vals,
                       void* radix_scratch, int32_t* plan_counters, cudaStream_t st) {
    int32_t* counts = queue + n_gaussians;  // [0] unused, [1] long segments
    *sorted_vals = vals;
    if (p.n_slots <= 0 || n_gaussians <= 0) {
        cudaMemsetAsync(counts, 0, 2 * sizeof(int32_t), st);
        if (p.n_slots <= 0) cudaMemsetAsync(seg, 0, (n_gaussians + 1) * sizeof(int32_t), st);
        if (plan_counters) cudaMemsetAsync(plan_counters, 0, (kPlanCounters + 1) * sizeof(int32_t), st);
        if (p.n_slots <= 0) return;
    }
    SlotKeyParams q = p;
    q.zero2 = n_gaussians > 0 ? counts : nullptr;  // k_slot_keys zeroes the queue counters
    launch_k(k_slot_keys, static_cast<unsigned>((p.n_slots + 255) / 256), 256, 0, st, q, keys, vals);
    dbg_launch("k_slot_keys", st);
    int bits = 0;
    while (bits < 32 && (static_cast<uint64_t>(n_gaussians) >> bits) != 0) ++bits;  // keys in [0, n]
    bool alt = false;
    if (p.n_slots > 1 && bits > 0)
        radix_sort_pairs_u32(keys, vals, keys_alt, vals_alt, p.n_slots, 0, bits, radix_scratch, st, &alt);
    *sorted_vals = alt ? vals_alt : vals;
    segment_offsets_u32(alt ? keys_alt : keys, p.n_slots, seg, n_gaussians, st);
    if (n_gaussians > 0) {
        const unsigned g1 = static_cast<unsigned>(std::min<int64_t>((n_gaussians + 255) / 256, 148 * 16));
        launch_k(k_long_queue, g1, 256, 0, st, seg, n_gaussians, queue, counts, plan_counters);
        dbg_launch("k_long_queue", st);
    }
}

void launch_long_plan(const int32_t* seg, int64_t n, const LongPlan& plan, cudaStream_t st) {
    // counters zeroed by k_long_queue (launch_slot_index)
    if (n <= 0) return;
    launch_k(k_long_count, 148 * 2, kThreads, 0, st, seg, n, plan);
    dbg_launch("k_long_count", st);
    launch_k(k_long_fill, 148 * 2, kThreads, 0, st, seg, plan);
    dbg_launch("k_long_fill", st);
}

void launch_feature_bwd(const FeatBwdParams& p, const LongPlan& plan, cudaStream_t st) {
    if (p.n_gaussians <= 0 || p.d <= 0) return;
    const bool vec = vec_ok(p.grad, p.out, p.d) && (reinterpret_cast<uintptr_t>(plan.partial) % 16) == 0 &&
                     (reinterpret_cast<uintptr_t>(plan.l1) % 16) == 0;
    if (vec && p.d % 512 == 0) launch_k<false>(k_feat_bwd<true, 2>, warp_grid_all(p.n_gaussians), kThreads, 0, st, p);
    else if (vec) launch_k<false>(k_feat_bwd<true, 0>, warp_grid_all(p.n_gaussians), kThreads, 0, st, p);
    else launch_k<false>(k_feat_bwd<false, 0>, warp_grid_all(p.n_gaussians), kThreads, 0, st, p);
    dbg_launch("k_feat_bwd", st);
    // persistent grids: the band-major item list is walked in order by every resident warp
    if (vec) launch_k<false>(k_feat_bwd_items<true>, 148 * 6, kThreads, 0, st, p, plan);
    else launch_k<false>(k_feat_bwd_items<false>, 148 * 6, kThreads, 0, st, p, plan);
    dbg_launch("k_feat_bwd_items", st);
    if (vec) launch_k<false>(k_long_combine1<true>, 148 * 4, kThreads, 0, st, p, plan);
    else launch_k<false>(k_long_combine1<false>, 148 * 4, kThreads, 0, st, p, plan);
    dbg_launch("k_long_combine1", st);
    if (vec) launch_k<false>(k_long_combine2<true>, 148 * 2, kThreads, 0, st, p, plan);
    else launch_k<false>(k_long_combine2<false>, 148 * 2, kThreads, 0, st, p, plan);
    dbg_launch("k_long_combine2", st);
}

void launch_first_stale(const int32_t* index, int64_t n_slots, int64_t n, unsigned long long* first,
                        cudaStream_t st) {
    if (n_slots > 0) launch_k<false>(k_first_stale, 296, 256, 0, st, index, n_slots, n, first);
    dbg_launch("k_first_stale", st);
}

void launch_interleave(const float* in, int64_t n_pixels, int ds, int g, float* out, cudaStream_t st) {
    if (n_pixels > 0) launch_k<false>(k_interleave, 148 * 8, 256, 0, st, in, n_pixels, ds, g, out);
    dbg_launch("k_interleave", st);
}

}  // namespace tk

// tile_stage.cuh — shared-memory staging of the feature rows a 16 x 16 pixel tile reads through its
// Top-K records (render.cpp:319-334 gathers; losses.cpp:92-118 feature loss).
//
// One CTA of 256 threads per tile, thread t = pixel t.  Each thread loads its pixel's records and
// normalised weights (w_j / sum_w in fp64, slot order, rounded to fp32 like the unstaged gathers),
// inserts the ids into a shared hash table with reference counts, and the ids read by two or more
// records get a staged row: up to `rows` of them are bulk-copied (TMA, one cp.async.bulk per row)
// into shared memory.  A pixel's records then name a staged row (slot >= 0) or, for ids read once
// or beyond the staged set, the global row (slot = -1 - id).  Neighbouring pixels share many of
// their K rows, so part of the P*K row reads through L2 become one read per distinct
// (tile, Gaussian); sums over the rows keep the slot order, so results are bit-identical.
#pragma once
#include "tk_common.cuh"

namespace tk {

constexpr int kStageSide = 16, kStagePix = kStageSide * kStageSide;

__host__ __device__ constexpr int pow2_ceil(int v) { return v <= 1 ? 1 : 2 * pow2_ceil((v + 1) / 2); }

template <int KMAX>
__host__ __device__ constexpr int stage_hash_size() {
    return 2 * kStagePix * pow2_ceil(KMAX);  // power of two, load factor <= 1/2
}

struct StageSmem {
    uint64_t* bar;  // bulk-copy barrier
    int* ucount;    // ids given a staged slot
    float* srow;    // [rows][D]
    int* hkey;      // [hash] id or -1
    int* hslot;     // [hash] reference count, then staged slot (rows = not staged)
    int* row_id;    // [rows]
};

template <int KMAX>
inline size_t stage_smem_bytes(int rows, int d) {
    return 128 + static_cast<size_t>(rows) * d * 4 + static_cast<size_t>(stage_hash_size<KMAX>()) * 8 +
           static_cast<size_t>(rows) * 4;
}

// Largest row count whose layout fits in `budget` bytes (at most every record distinct).
template <int KMAX>
inline int stage_rows(size_t budget, int d) {
    const size_t fixed = 128 + static_cast<size_t>(stage_hash_size<KMAX>()) * 8;
    if (budget <= fixed) return 0;
    const size_t r = (budget - fixed) / (static_cast<size_t>(d) * 4 + 4);
    return static_cast<int>(r < static_cast<size_t>(kStagePix * KMAX) ? r : kStagePix * KMAX);
}

template <int KMAX>
__device__ __forceinline__ StageSmem stage_layout(unsigned char* gsm, int rows, int d) {
    StageSmem s;
    s.bar = reinterpret_cast<uint64_t*>(gsm);
    s.ucount = reinterpret_cast<int*>(gsm + 8);
    s.srow = reinterpret_cast<float*>(gsm + 128);
    s.hkey = reinterpret_cast<int*>(gsm + 128 + static_cast<size_t>(rows) * d * 4);
    s.hslot = s.hkey + stage_hash_size<KMAX>();
    s.row_id = s.hslot + stage_hash_size<KMAX>();
    return s;
}

__device__ __forceinline__ void stage_init(const StageSmem& s) {
    if (threadIdx.x == 0) {
        mbar_init(s.bar, 1);
        fence_mbar_init();
    }
}

// This thread's pixel after staging: record count (-1 outside the image), staged slot or
// -1 - id per record, normalised fp32 weights.
template <int KMAX>
struct StagedPixel {
    int c;
    int slot[KMAX];
    float wn[KMAX];
};

// Stage one tile.  px: this thread's pixel (ignored when c < 0); c: its record count, or -1
// (outside the image) / 0 (no records used).  Every thread of the CTA must call it; on return
// the staged rows are visible to the whole CTA.  The caller synchronises the CTA before staging
// the next tile (the rows and the hash are reused).
template <int KMAX>
__device__ __forceinline__ StagedPixel<KMAX> stage_tile(const StageSmem& s, int rows, int d, const float* feat,
                                                        const int32_t* index, const double* weight, int k,
                                                        int64_t px, int c, unsigned& phase) {
    constexpr int kHash = stage_hash_size<KMAX>();
    const int tid = threadIdx.x;
    for (int h = tid; h < kHash; h += kStagePix) {
        s.hkey[h] = -1;
        s.hslot[h] = 0;
    }
    if (tid == 0) s.ucount[0] = 0;
    __syncthreads();
    StagedPixel<KMAX> o;
    o.c = c;
    int gid[KMAX], hpos[KMAX];
    double wd[KMAX];
    double sum = 0.0;
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
        gid[j] = 0;
        wd[j] = 0.0;
        if (j < c) {
            gid[j] = index[px * k + j];
            wd[j] = weight[px * k + j];
            sum += wd[j];
        }
    }
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
        o.wn[j] = j < c ? static_cast<float>(wd[j] / sum) : 0.0f;
        hpos[j] = 0;
        if (j < c) {
            unsigned h = (static_cast<unsigned>(gid[j]) * 2654435761u) & (kHash - 1);
            while (true) {
                const int old = atomicCAS(&s.hkey[h], -1, gid[j]);
                if (old == -1 || old == gid[j]) break;
                h = (h + 1) & (kHash - 1);
            }
            atomicAdd(&s.hslot[h], 1);
            hpos[j] = static_cast<int>(h);
        }
    }
    __syncthreads();
    // number the ids read by two or more records (a row read once gains nothing from staging)
    for (int h = tid; h < kHash; h += kStagePix) {
        const int g = s.hkey[h];
        if (g >= 0) {
            const int sl = s.hslot[h] >= 2 ? atomicAdd(s.ucount, 1) : rows;
            s.hslot[h] = sl < rows ? sl : rows;
            if (sl < rows) s.row_id[sl] = g;
        }
    }
    __syncthreads();
    const int staged = min(s.ucount[0], rows);
    if (staged > 0) {
        if (tid == 0) mbar_arrive_expect_tx(s.bar, static_cast<unsigned>(staged) * d * 4);
        for (int r = tid; r < staged; r += kStagePix)
            bulk_g2s(s.srow + static_cast<size_t>(r) * d, feat + static_cast<int64_t>(s.row_id[r]) * d, d * 4, s.bar);
    }
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
        const int sl = j < c ? s.hslot[hpos[j]] : 0;
        o.slot[j] = sl < rows ? sl : -1 - gid[j];
    }
    if (staged > 0) {
        mbar_wait(s.bar, phase);
        phase ^= 1u;
    }
    return o;
}

}  // namespace tk

// sort.cu — exclusive scan and stable LSD radix sort (8-bit digits), written for sm_100a.
//
// The reference sorts with std::sort on (z, src) (render.cpp:108-111) and fills tile lists with
// a serial counting pass (render.cpp:134-153).  On the GPU both become stable radix sorts:
// the depth sort on the fp64 bit pattern of z (positive doubles order like their bits) with
// values pre-ordered by src, and the tile binning on tile id with values pre-ordered by depth
// rank.  Stability reproduces the reference's tie rules exactly.
#include "sort.cuh"

#include <algorithm>

namespace tk {

size_t align_bytes(size_t b) { return (b + 255) / 256 * 256; }

namespace {

constexpr int SCAN_THREADS = 512;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

__device__ __forceinline__ int64_t warp_incl_scan(int64_t v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
    }
    return v;
}

// Block-wide exclusive scan of one int64 per thread; returns exclusive prefix, *block_total.
template <int NT>
__device__ int64_t block_excl_scan(int64_t v, int64_t* block_total) {
    __shared__ int64_t warp_sums[NT / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t incl = warp_incl_scan(v);
    if (lane == 31) warp_sums[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        int64_t s = lane < NT / 32 ? warp_sums[lane] : 0;
        s = warp_incl_scan(s);
        if (lane < NT / 32) warp_sums[lane] = s;
    }
    __syncthreads();
    const int64_t warp_off = warp > 0 ? warp_sums[warp - 1] : 0;
    *block_total = warp_sums[NT / 32 - 1];
    __syncthreads();
    return warp_off + incl - v;
}

__global__ void __launch_bounds__(SCAN_THREADS) k_scan_reduce(const int32_t* __restrict__ in, int64_t n,
                                                              int64_t* __restrict__ bsum) {
    const int64_t base = static_cast<int64_t>(blockIdx.x) * SCAN_TILE;
    int64_t s = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        const int64_t idx = base + static_cast<int64_t>(i) * SCAN_THREADS + threadIdx.x;
        if (idx < n) s += in[idx];
    }
    int64_t tot;
    block_excl_scan<SCAN_THREADS>(s, &tot);
    if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) k_scan_blocks(int64_t* __restrict__ bsum, int64_t nb,
                                                       int64_t* __restrict__ total) {
    int64_t carry = 0;
    for (int64_t base = 0; base < nb; base += 1024) {
        const int64_t idx = base + threadIdx.x;
        const int64_t v = idx < nb ? bsum[idx] : 0;
        int64_t tot;
        const int64_t ex = block_excl_scan<1024>(v, &tot);
        if (idx < nb) bsum[idx] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) *total = carry;
}

__global__ void __launch_bounds__(SCAN_THREADS) k_scan_apply(const int32_t* __restrict__ in, int32_t* __restrict__ out,
                                                             int64_t n, const int64_t* __restrict__ bsum) {
    const int64_t base = static_cast<int64_t>(blockIdx.x) * SCAN_TILE + static_cast<int64_t>(threadIdx.x) * SCAN_ITEMS;
    int32_t v[SCAN_ITEMS];
    int64_t s = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        v[i] = base + i < n ? in[base + i] : 0;
        s += v[i];
    }
    int64_t tot;
    int64_t run = bsum[blockIdx.x] + block_excl_scan<SCAN_THREADS>(s, &tot);
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        if (base + i < n) out[base + i] = static_cast<int32_t>(run);
        run += v[i];
    }
}

constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_ROUNDS = 16;
constexpr int RS_TILE = RS_THREADS * RS_ROUNDS;
constexpr int RS_RADIX = 256;

template <typename K>
__global__ void __launch_bounds__(RS_THREADS) k_rs_hist(const K* __restrict__ keys, int64_t n, int shift,
                                                        int32_t* __restrict__ hist, int nb) {
    __shared__ int32_t cnt[RS_RADIX];
    cnt[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = static_cast<int64_t>(blockIdx.x) * RS_TILE;
#pragma unroll 4
    for (int r = 0; r < RS_ROUNDS; ++r) {
        const int64_t idx = base + r * RS_THREADS + threadIdx.x;
        if (idx < n) atomicAdd(&cnt[static_cast<unsigned>(keys[idx] >> shift) & 0xffu], 1);
    }
    __syncthreads();
    hist[static_cast<int64_t>(threadIdx.x) * nb + blockIdx.x] = cnt[threadIdx.x];
}

template <typename K>
__global__ void __launch_bounds__(RS_THREADS) k_rs_scatter(const K* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                           K* __restrict__ kout, uint32_t* __restrict__ vout,
                                                           int64_t n, int shift, const int32_t* __restrict__ offs,
                                                           int nb) {
    __shared__ int32_t base[RS_RADIX];
    __shared__ int32_t wc[RS_WARPS][RS_RADIX + 1];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    base[tid] = offs[static_cast<int64_t>(tid) * nb + blockIdx.x];
#pragma unroll
    for (int w = 0; w < RS_WARPS; ++w) wc[w][tid] = 0;
    const unsigned lt = (1u << lane) - 1u;
    const int64_t tile0 = static_cast<int64_t>(blockIdx.x) * RS_TILE;
    __syncthreads();
    for (int r = 0; r < RS_ROUNDS; ++r) {
        const int64_t idx = tile0 + r * RS_THREADS + tid;
        const bool valid = idx < n;
        K key = 0;
        uint32_t val = 0;
        unsigned digit = RS_RADIX;  // invalid lanes group together and are never written
        if (valid) {
            key = kin[idx];
            val = vin[idx];
            digit = static_cast<unsigned>(key >> shift) & 0xffu;
        }
        const unsigned peers = __match_any_sync(0xffffffffu, digit);
        const int rank = __popc(peers & lt);
        const bool leader = rank == 0;
        if (leader && valid) wc[warp][digit] = __popc(peers);
        __syncthreads();
        {  // thread d: exclusive prefix over warps of digit d, then advance the running base
            int32_t run = base[tid];
#pragma unroll
            for (int w = 0; w < RS_WARPS; ++w) {
                const int32_t c = wc[w][tid];
                wc[w][tid] = run;
                run += c;
            }
            base[tid] = run;
        }
        __syncthreads();
        if (valid) {
            const int32_t pos = wc[warp][digit] + rank;
            kout[pos] = key;
            vout[pos] = val;
        }
        __syncthreads();
#pragma unroll
        for (int w = 0; w < RS_WARPS; ++w) wc[w][tid] = 0;
        __syncthreads();
        if (tile0 + (r + 1) * RS_THREADS >= n) break;  // uniform across the block
    }
}

template <typename K>
void radix_sort_impl(K* keys, uint32_t* vals, K* keys_alt, uint32_t* vals_alt, int64_t n, int begin_bit,
                     int end_bit, void* scratch, cudaStream_t st, bool* result_in_alt, int64_t* launches) {
    *result_in_alt = false;
    if (n <= 0 || end_bit <= begin_bit) return;
    const int nb = static_cast<int>((n + RS_TILE - 1) / RS_TILE);
    const int64_t hn = static_cast<int64_t>(RS_RADIX) * nb;
    char* sp = static_cast<char*>(scratch);
    int32_t* hist = reinterpret_cast<int32_t*>(sp);
    sp += align_bytes(hn * sizeof(int32_t));
    int64_t* total = reinterpret_cast<int64_t*>(sp);
    sp += 256;
    void* scan_scratch = sp;
    K* kin = keys;
    uint32_t* vin = vals;
    K* kout = keys_alt;
    uint32_t* vout = vals_alt;
    bool in_alt = false;
    for (int shift = begin_bit; shift < end_bit; shift += 8) {
        k_rs_hist<K><<<nb, RS_THREADS, 0, st>>>(kin, n, shift, hist, nb);
        scan_exclusive(hist, hist, hn, total, scan_scratch, st, launches);
        k_rs_scatter<K><<<nb, RS_THREADS, 0, st>>>(kin, vin, kout, vout, n, shift, hist, nb);
        *launches += 2;
        std::swap(kin, kout);
        std::swap(vin, vout);
        in_alt = !in_alt;
    }
    *result_in_alt = in_alt;
}

__global__ void k_segment_offsets(const uint32_t* __restrict__ keys, int64_t n, int32_t* __restrict__ offsets,
                                  int64_t nseg) {
    const int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (g > nseg) return;
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (static_cast<int64_t>(keys[mid]) < g) lo = mid + 1;
        else hi = mid;
    }
    offsets[g] = static_cast<int32_t>(lo);
}

}  // namespace

size_t scan_scratch_bytes(int64_t n) {
    const int64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
    return align_bytes(static_cast<size_t>(nb + 1) * sizeof(int64_t));
}

void scan_exclusive(const int32_t* in, int32_t* out, int64_t n, int64_t* total, void* scratch, cudaStream_t st,
                    int64_t* launches) {
    const int64_t nb = std::max<int64_t>(1, (n + SCAN_TILE - 1) / SCAN_TILE);
    int64_t* bsum = static_cast<int64_t*>(scratch);
    k_scan_reduce<<<static_cast<unsigned>(nb), SCAN_THREADS, 0, st>>>(in, n, bsum);
    k_scan_blocks<<<1, 1024, 0, st>>>(bsum, nb, total);
    k_scan_apply<<<static_cast<unsigned>(nb), SCAN_THREADS, 0, st>>>(in, out, n, bsum);
    *launches += 3;
}

size_t radix_scratch_bytes(int64_t n) {
    const int64_t nb = (n + RS_TILE - 1) / RS_TILE + 1;
    const int64_t hn = static_cast<int64_t>(RS_RADIX) * nb;
    return align_bytes(hn * sizeof(int32_t)) + 256 + scan_scratch_bytes(hn);
}

void radix_sort_pairs_u64(uint64_t* keys, uint32_t* vals, uint64_t* keys_alt, uint32_t* vals_alt, int64_t n,
                          int begin_bit, int end_bit, void* scratch, cudaStream_t st, bool* result_in_alt,
                          int64_t* launches) {
    radix_sort_impl<uint64_t>(keys, vals, keys_alt, vals_alt, n, begin_bit, end_bit, scratch, st, result_in_alt,
                              launches);
}

void radix_sort_pairs_u32(uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt, int64_t n,
                          int begin_bit, int end_bit, void* scratch, cudaStream_t st, bool* result_in_alt,
                          int64_t* launches) {
    radix_sort_impl<uint32_t>(keys, vals, keys_alt, vals_alt, n, begin_bit, end_bit, scratch, st, result_in_alt,
                              launches);
}

void segment_offsets_u32(const uint32_t* keys, int64_t n, int32_t* offsets, int64_t n_segments, cudaStream_t st,
                         int64_t* launches) {
    const int64_t total = n_segments + 1;
    k_segment_offsets<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(keys, n, offsets, n_segments);
    *launches += 1;
}

}  // namespace tk

// sort.cu — exclusive scan and stable LSD radix sort (8-bit digits), written for sm_100a.
//
// The reference sorts with std::sort on (z, src) (render.cpp:108-111) and fills tile lists with
// a serial counting pass (render.cpp:134-153).  On the GPU both become stable radix sorts:
// the depth sort on the fp64 bit pattern of z (positive doubles order like their bits) with
// values pre-ordered by src, and the tile binning on tile id with values pre-ordered by depth
// rank.  Stability reproduces the reference's tie rules exactly.
#include "sort.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "tk_common.cuh"

namespace tk {

size_t align_bytes(size_t b) { return (b + 255) / 256 * 256; }

namespace {
thread_local int64_t t_launches = 0;  // kernels launched by this host thread (dbg_launch after each)
}

int64_t launch_count() { return t_launches; }

bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("TK_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

void dbg_launch(const char* name, cudaStream_t st) {
    ++t_launches;
    static const int on = [] {
        const char* e = std::getenv("TK_SYNC_CHECK");
        return e && e[0] == '1' ? 1 : 0;
    }();
    if (!on) return;
    cudaError_t e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) std::fprintf(stderr, "[tk] kernel %s failed: %s\n", name, cudaGetErrorString(e));
}

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

// Single-pass scan with decoupled look-back: each block publishes its aggregate, then its
// inclusive prefix once the predecessor's prefix is known (status word: 2-bit flag | 62-bit sum).
// Block order comes from a ticket so a block only ever waits on blocks already running.
constexpr unsigned long long kFlagAgg = 1ull << 62, kFlagPrefix = 2ull << 62, kValMask = (1ull << 62) - 1;

__global__ void __launch_bounds__(SCAN_THREADS) k_scan_lookback(const int32_t* __restrict__ in,
                                                                int32_t* __restrict__ out, int64_t n,
                                                                unsigned long long* __restrict__ status,
                                                                int* __restrict__ ticket, int64_t* __restrict__ total,
                                                                int nb) {
    pdl_prologue();
    __shared__ int bid_s;
    __shared__ int64_t excl_s;
    if (threadIdx.x == 0) bid_s = atomicAdd(ticket, 1);
    __syncthreads();
    const int bid = bid_s;
    const int64_t base = static_cast<int64_t>(bid) * SCAN_TILE + static_cast<int64_t>(threadIdx.x) * SCAN_ITEMS;
    int32_t v[SCAN_ITEMS];
    int64_t s = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        v[i] = base + i < n ? in[base + i] : 0;
        s += v[i];
    }
    int64_t tot;
    const int64_t local = block_excl_scan<SCAN_THREADS>(s, &tot);
    if (threadIdx.x < 32) {  // warp 0: publish, then look back 32 predecessors at a time
        const int lane = threadIdx.x;
        volatile unsigned long long* vs = status;
        int64_t excl = 0;
        if (bid == 0) {
            if (lane == 0) vs[0] = kFlagPrefix | static_cast<unsigned long long>(tot);
        } else {
            if (lane == 0) {
                vs[bid] = kFlagAgg | static_cast<unsigned long long>(tot);
                __threadfence();
            }
            __syncwarp();
            for (int p = bid - 1;; p -= 32) {
                const int q = p - lane;
                unsigned long long w = q >= 0 ? vs[q] : (2ull << 62);  // before block 0: prefix 0
                while (__any_sync(0xffffffffu, (w & ~kValMask) == 0))
                    if ((w & ~kValMask) == 0) w = vs[q];
                const unsigned pm = __ballot_sync(0xffffffffu, (w & ~kValMask) == kFlagPrefix);
                const int first = pm ? __ffs(pm) - 1 : 32;  // closest predecessor holding a prefix
                int64_t val = lane <= first ? static_cast<int64_t>(w & kValMask) : 0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
                excl += val;
                if (pm) break;
            }
            if (lane == 0) {
                __threadfence();
                vs[bid] = kFlagPrefix | static_cast<unsigned long long>(excl + tot);
            }
        }
        if (lane == 0) {
            excl_s = excl;
            if (bid == nb - 1) *total = excl + tot;
        }
    }
    __syncthreads();
    int64_t run = excl_s + local;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        if (base + i < n) out[base + i] = static_cast<int32_t>(run);
        run += v[i];
    }
}

// Whole scan in one launch for small inputs (radix histograms, tile counts).
constexpr int64_t kSmallScan = 1024 * 64;
__global__ void __launch_bounds__(1024) k_scan_single(const int32_t* __restrict__ in, int32_t* __restrict__ out,
                                                      int64_t n, int64_t* __restrict__ total) {
    pdl_prologue();
    const int64_t per = (n + 1023) / 1024;
    const int64_t b = static_cast<int64_t>(threadIdx.x) * per;
    const int64_t e = b + per < n ? b + per : n;
    int64_t s = 0;
    for (int64_t i = b; i < e; ++i) s += in[i];
    int64_t tot;
    int64_t run = block_excl_scan<1024>(s, &tot);
    for (int64_t i = b; i < e; ++i) {
        const int32_t v = in[i];
        out[i] = static_cast<int32_t>(run);
        run += v;
    }
    if (threadIdx.x == 0) *total = tot;
}

// TK_RADIX_LEGACY=1: per-pass histogram + scan + scatter instead of onesweep (A/B, tests).
bool legacy_radix() {
    static const bool on = [] {
        const char* e = std::getenv("TK_RADIX_LEGACY");
        return e && e[0] == '1';
    }();
    return on;
}

constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_ROUNDS = 8;
constexpr int RS_TILE = RS_THREADS * RS_ROUNDS;
constexpr int RS_RADIX = 256;

// Per-block digit histogram.  Warp-aggregated (match_any) so runs of equal digits -- tile ids,
// Gaussian ids -- cost one shared atomic per distinct digit per warp.
template <typename K>
__global__ void __launch_bounds__(RS_THREADS) k_rs_hist(const K* __restrict__ keys, int64_t n, int shift,
                                                        int32_t* __restrict__ hist, int nb) {
    pdl_prologue();
    __shared__ int32_t cnt[RS_RADIX];
    cnt[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = static_cast<int64_t>(blockIdx.x) * RS_TILE;
    const unsigned lane = threadIdx.x & 31;
#pragma unroll 4
    for (int r = 0; r < RS_ROUNDS; ++r) {
        const int64_t idx = base + r * RS_THREADS + threadIdx.x;
        const unsigned d = idx < n ? static_cast<unsigned>(keys[idx] >> shift) & 0xffu : RS_RADIX;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        if (d < RS_RADIX && lane == static_cast<unsigned>(__ffs(peers) - 1)) atomicAdd(&cnt[d], __popc(peers));
    }
    __syncthreads();
    hist[static_cast<int64_t>(threadIdx.x) * nb + blockIdx.x] = cnt[threadIdx.x];
}

// Stable scatter.  Each warp owns a contiguous 256-key slice of the block's 2048-key tile and
// ranks its keys round by round (match_any) against a warp-private digit counter row, so the
// ranking needs no block barrier; one block scan over (digit, warp) counts then gives every
// key's position in the digit-sorted tile, which is staged in shared memory and written out with
// consecutive threads on consecutive addresses of each digit's global run.
//
// ONESWEEP = true: the pass needs no per-block histogram.  Blocks take tiles in ticket order,
// publish their per-digit counts in a status word per (tile, digit) and look back over the
// predecessors' words (decoupled look-back, one thread per digit) for the digit's offset; the
// digit's global start comes from the all-pass histogram of k_rs_ghist.
constexpr uint32_t kOsAgg = 1u << 30, kOsPrefix = 2u << 30, kOsMask = kOsAgg - 1;

struct OnesweepArgs {
    const int32_t* gcount;  // [256] digit totals of this pass
    uint32_t* status;       // [nb][256] (flag | value), zeroed
    int* ticket;            // zeroed
};

template <typename K, bool ONESWEEP>
__global__ void __launch_bounds__(RS_THREADS) k_rs_scatter(const K* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                           K* __restrict__ kout, uint32_t* __restrict__ vout,
                                                           int64_t n, int shift, const int32_t* __restrict__ offs,
                                                           int nb, OnesweepArgs os) {
    pdl_prologue();
    __shared__ int32_t gbase[RS_RADIX];
    __shared__ int32_t lstart[RS_RADIX];
    __shared__ int32_t wc[RS_WARPS][RS_RADIX];  // per-warp digit counts, then per-(warp, digit) offsets
    __shared__ K skey[RS_TILE];
    __shared__ uint32_t sval[RS_TILE];
    __shared__ int32_t wsum[RS_WARPS];
    __shared__ int32_t gsum[RS_WARPS];
    __shared__ int bid_s;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned lt = (1u << lane) - 1u;
    if (ONESWEEP) {
        if (tid == 0) bid_s = atomicAdd(os.ticket, 1);
    } else {
        gbase[tid] = offs[static_cast<int64_t>(tid) * nb + blockIdx.x];
    }
#pragma unroll
    for (int w = 0; w < RS_WARPS; ++w) wc[w][tid] = 0;
    __syncthreads();
    const int bid = ONESWEEP ? bid_s : static_cast<int>(blockIdx.x);
    const int64_t tile0 = static_cast<int64_t>(bid) * RS_TILE;
    const int tile_n = static_cast<int>(n - tile0 < RS_TILE ? n - tile0 : RS_TILE);
    constexpr int kSlice = RS_TILE / RS_WARPS;  // 256 keys per warp
    K key[RS_ROUNDS];
    uint32_t val[RS_ROUNDS];
    unsigned dig[RS_ROUNDS];
    int pos[RS_ROUNDS];
#pragma unroll
    for (int r = 0; r < RS_ROUNDS; ++r) {
        const int li = warp * kSlice + r * 32 + lane;
        dig[r] = RS_RADIX;
        if (li < tile_n) {
            key[r] = kin[tile0 + li];
            val[r] = vin[tile0 + li];
            dig[r] = static_cast<unsigned>(key[r] >> shift) & 0xffu;
        }
        const unsigned d = dig[r];
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const int rank = __popc(peers & lt);
        pos[r] = (d < RS_RADIX ? wc[warp][d] : 0) + rank;  // rank among this warp's keys of digit d
        __syncwarp();
        if (d < RS_RADIX && rank == 0) wc[warp][d] += __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    {  // thread = digit: counts over warps, exclusive over digits (lstart), then per-warp offsets
        int32_t tot = 0;
#pragma unroll
        for (int w = 0; w < RS_WARPS; ++w) tot += wc[w][tid];
        int incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        int woff = 0;
        for (int w = 0; w < warp; ++w) woff += wsum[w];
        const int32_t start = woff + incl - tot;
        lstart[tid] = start;
        int32_t acc = start;
#pragma unroll
        for (int w = 0; w < RS_WARPS; ++w) {
            const int32_t c = wc[w][tid];
            wc[w][tid] = acc;
            acc += c;
        }
        if (ONESWEEP) {
            // publish this tile's count of digit tid, then look back for the earlier tiles' total
            volatile uint32_t* st = os.status;
            const int64_t me = static_cast<int64_t>(bid) * RS_RADIX + tid;
            uint32_t excl = 0;
            if (bid == 0) {
                st[me] = kOsPrefix | static_cast<uint32_t>(tot);
            } else {
                st[me] = kOsAgg | static_cast<uint32_t>(tot);
                // eight predecessors' words per round go out together; consumed in order up to
                // the nearest one holding a prefix (block 0 always does)
                constexpr int kLB = 8;
                bool done = false;
                for (int64_t q = me - RS_RADIX; !done; q -= kLB * RS_RADIX) {
                    uint32_t w[kLB];
#pragma unroll
                    for (int j = 0; j < kLB; ++j) w[j] = q - j * RS_RADIX >= 0 ? st[q - j * RS_RADIX] : uint32_t{kOsPrefix};
#pragma unroll
                    for (int j = 0; j < kLB; ++j) {
                        if (done) break;
                        while ((w[j] & ~kOsMask) == 0) w[j] = st[q - j * RS_RADIX];
                        excl += w[j] & kOsMask;
                        done = (w[j] & kOsPrefix) != 0;
                    }
                }
                st[me] = kOsPrefix | (excl + static_cast<uint32_t>(tot));
            }
            // the digit's global start: exclusive scan of the pass histogram over digits
            const int32_t gc = os.gcount[tid];
            int ginc = gc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int u = __shfl_up_sync(0xffffffffu, ginc, o);
                if (lane >= o) ginc += u;
            }
            if (lane == 31) gsum[warp] = ginc;
            __syncthreads();
            int goff = 0;
            for (int w = 0; w < warp; ++w) goff += gsum[w];
            gbase[tid] = goff + ginc - gc + static_cast<int32_t>(excl);
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < RS_ROUNDS; ++r) {
        const unsigned d = dig[r];
        if (d < RS_RADIX) {
            const int lpos = wc[warp][d] + pos[r];
            skey[lpos] = key[r];
            sval[lpos] = val[r];
        }
    }
    __syncthreads();
    for (int j = tid; j < tile_n; j += RS_THREADS) {
        const K kj = skey[j];
        const unsigned d = static_cast<unsigned>(kj >> shift) & 0xffu;
        const int32_t gpos = gbase[d] + (j - lstart[d]);
        kout[gpos] = kj;
        vout[gpos] = sval[j];
    }
}

// Digit totals of every pass at once (the histograms are order independent): counts[p][d].
template <typename K>
__global__ void __launch_bounds__(RS_THREADS) k_rs_ghist(const K* __restrict__ keys, int64_t n, int begin_bit,
                                                         int npass, int32_t* __restrict__ counts) {
    pdl_prologue();
    __shared__ int32_t cnt[8][RS_RADIX];
    for (int p = 0; p < 8; ++p) cnt[p][threadIdx.x] = 0;
    __syncthreads();
    const unsigned lane = threadIdx.x & 31;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * RS_THREADS + threadIdx.x; i - threadIdx.x < n;
         i += static_cast<int64_t>(gridDim.x) * RS_THREADS) {
        const bool in = i < n;
        const K k = in ? keys[i] : K(0);
        for (int p = 0; p < npass; ++p) {
            const unsigned d = in ? static_cast<unsigned>(k >> (begin_bit + 8 * p)) & 0xffu : RS_RADIX;
            const unsigned peers = __match_any_sync(0xffffffffu, d);
            if (d < RS_RADIX && lane == static_cast<unsigned>(__ffs(peers) - 1)) atomicAdd(&cnt[p][d], __popc(peers));
        }
    }
    __syncthreads();
    for (int p = 0; p < npass; ++p)
        if (cnt[p][threadIdx.x]) atomicAdd(&counts[p * RS_RADIX + threadIdx.x], cnt[p][threadIdx.x]);
}

template <typename K>
void radix_sort_impl(K* keys, uint32_t* vals, K* keys_alt, uint32_t* vals_alt, int64_t n, int begin_bit,
                     int end_bit, void* scratch, cudaStream_t st, bool* result_in_alt) {
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
    const int npass = (end_bit - begin_bit + 7) / 8;
    if (n < (1LL << 30) && npass <= 8 && !legacy_radix()) {
        // onesweep: one all-pass histogram, then one look-back scatter per pass
        char* op = static_cast<char*>(scratch);
        int32_t* gcount = reinterpret_cast<int32_t*>(op);
        int* tickets = reinterpret_cast<int*>(op + 8 * RS_RADIX * sizeof(int32_t));
        uint32_t* status = reinterpret_cast<uint32_t*>(op + align_bytes(8 * RS_RADIX * sizeof(int32_t) + 8 * sizeof(int)));
        const size_t status_words = static_cast<size_t>(nb) * RS_RADIX;
        cudaMemsetAsync(scratch, 0,
                        align_bytes(8 * RS_RADIX * sizeof(int32_t) + 8 * sizeof(int)) +
                            npass * status_words * sizeof(uint32_t),
                        st);
        const int hblocks = static_cast<int>(std::min<int64_t>(nb, 148 * 4));
        launch_k(k_rs_ghist<K>, hblocks, RS_THREADS, 0, st, kin, n, begin_bit, npass, gcount);
        dbg_launch("k_rs_ghist", st);
        for (int p = 0; p < npass; ++p) {
            const OnesweepArgs os{gcount + p * RS_RADIX, status + p * status_words, tickets + p};
            launch_k(k_rs_scatter<K, true>, nb, RS_THREADS, 0, st, kin, vin, kout, vout, n, begin_bit + 8 * p, nullptr, nb,
                                                             os);
            dbg_launch("k_rs_onesweep", st);
            std::swap(kin, kout);
            std::swap(vin, vout);
            in_alt = !in_alt;
        }
        *result_in_alt = in_alt;
        return;
    }
    for (int shift = begin_bit; shift < end_bit; shift += 8) {
        launch_k(k_rs_hist<K>, nb, RS_THREADS, 0, st, kin, n, shift, hist, nb);
        dbg_launch("k_rs_hist", st);
        scan_exclusive(hist, hist, hn, total, scan_scratch, st);
        launch_k(k_rs_scatter<K, false>, nb, RS_THREADS, 0, st, kin, vin, kout, vout, n, shift, hist, nb, OnesweepArgs{});
        dbg_launch("k_rs_scatter", st);
        std::swap(kin, kout);
        std::swap(vin, vout);
        in_alt = !in_alt;
    }
    *result_in_alt = in_alt;
}

// Finish a radix sort that only ordered key bits >= lo_bit: sort each run of equal high bits by
// (full key, value).  Runs longer than 64 set *overflow (the caller redoes a full sort).
__global__ void k_fixup_runs(uint64_t* __restrict__ keys, uint32_t* __restrict__ vals, int64_t n, int lo_bit,
                             int32_t* __restrict__ overflow) {
    pdl_prologue();
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t c = keys[i] >> lo_bit;
    if (i > 0 && (keys[i - 1] >> lo_bit) == c) return;
    int64_t j = i + 1;
    while (j < n && (keys[j] >> lo_bit) == c) {
        ++j;
        if (j - i > 64) {
            *overflow = 1;
            return;
        }
    }
    for (int64_t a = i + 1; a < j; ++a) {  // insertion sort by (key, val)
        const uint64_t k = keys[a];
        const uint32_t v = vals[a];
        int64_t b = a - 1;
        while (b >= i && (keys[b] > k || (keys[b] == k && vals[b] > v))) {
            keys[b + 1] = keys[b];
            vals[b + 1] = vals[b];
            --b;
        }
        keys[b + 1] = k;
        vals[b + 1] = v;
    }
}

__global__ void k_segment_offsets(const uint32_t* __restrict__ keys, int64_t n, int32_t* __restrict__ offsets,
                                  int64_t nseg) {
    pdl_prologue();
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

// Small device -> host-mapped copies (scalars, loss values): stores from a kernel travel over the
// bus without a copy engine, so they never queue behind large asynchronous DMA transfers.
__global__ void k_copy_words(const unsigned long long* __restrict__ src, unsigned long long* __restrict__ dst, int n) {
    pdl_prologue();
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

}  // namespace

// fp64 FMA throughput probe (8 independent chains per thread): the denominator of the fp64
// roofline the bench reports for the geometric sweeps.
__global__ void k_dfma_probe(double* out, int iters, double a, double b) {
    pdl_prologue();
    double x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3 + j;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, b);
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j];
    if (s == 12345.678) out[0] = s;
}

double measure_fp64_fma_rate(cudaStream_t st) {
    double* out = nullptr;
    if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) return 0.0;
    const int blocks = 148 * 8, threads = 256, iters = 1 << 13;
    launch_k<false>(k_dfma_probe, blocks, threads, 0, st, out, 16, 0.999, 1e-3);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0, st);
        launch_k<false>(k_dfma_probe, blocks, threads, 0, st, out, iters, 0.999, 1e-3);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    return static_cast<double>(blocks) * threads * iters * 8 / (best / 1e3);
}

void copy_words_to_mapped(void* dst_mapped, const void* src, int words, cudaStream_t st) {
    if (words <= 0) return;
    launch_k(k_copy_words, 1, 32, 0, st, static_cast<const unsigned long long*>(src),
                                   static_cast<unsigned long long*>(dst_mapped), words);
    dbg_launch("k_copy_words", st);
}

size_t scan_scratch_bytes(int64_t n) {
    const int64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
    return align_bytes(static_cast<size_t>(nb + 2) * sizeof(int64_t));
}

void scan_exclusive(const int32_t* in, int32_t* out, int64_t n, int64_t* total, void* scratch, cudaStream_t st) {
    if (n <= kSmallScan) {
        launch_k(k_scan_single, 1, 1024, 0, st, in, out, n, total);
        dbg_launch("k_scan_single", st);
        return;
    }
    // single pass: a block reads its whole tile before writing it, so in-place is safe
    const int64_t nb = std::max<int64_t>(1, (n + SCAN_TILE - 1) / SCAN_TILE);
    unsigned long long* status = static_cast<unsigned long long*>(scratch);
    int* ticket = reinterpret_cast<int*>(status + nb);
    cudaMemsetAsync(status, 0, (nb + 1) * sizeof(unsigned long long), st);
    launch_k(k_scan_lookback, static_cast<unsigned>(nb), SCAN_THREADS, 0, st, in, out, n, status, ticket, total,
                                                                      static_cast<int>(nb));
    dbg_launch("k_scan_lookback", st);
}

size_t radix_scratch_bytes(int64_t n) {
    const int64_t nb = (n + RS_TILE - 1) / RS_TILE + 1;
    const int64_t hn = static_cast<int64_t>(RS_RADIX) * nb;
    const size_t legacy = align_bytes(hn * sizeof(int32_t)) + 256 + scan_scratch_bytes(hn);
    const size_t onesweep = align_bytes(8 * RS_RADIX * sizeof(int32_t) + 8 * sizeof(int)) + 8 * hn * sizeof(uint32_t);
    return std::max(legacy, onesweep);
}

void radix_sort_pairs_u64(uint64_t* keys, uint32_t* vals, uint64_t* keys_alt, uint32_t* vals_alt, int64_t n,
                          int begin_bit, int end_bit, void* scratch, cudaStream_t st, bool* result_in_alt) {
    radix_sort_impl<uint64_t>(keys, vals, keys_alt, vals_alt, n, begin_bit, end_bit, scratch, st, result_in_alt);
}

void radix_sort_pairs_u32(uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt, int64_t n,
                          int begin_bit, int end_bit, void* scratch, cudaStream_t st, bool* result_in_alt) {
    radix_sort_impl<uint32_t>(keys, vals, keys_alt, vals_alt, n, begin_bit, end_bit, scratch, st, result_in_alt);
}

void fixup_runs_u64(uint64_t* keys, uint32_t* vals, int64_t n, int lo_bit, int32_t* overflow, cudaStream_t st) {
    if (n <= 1 || lo_bit <= 0) return;
    launch_k(k_fixup_runs, static_cast<unsigned>((n + 255) / 256), 256, 0, st, keys, vals, n, lo_bit, overflow);
    dbg_launch("k_fixup_runs", st);
}

void segment_offsets_u32(const uint32_t* keys, int64_t n, int32_t* offsets, int64_t n_segments, cudaStream_t st) {
    const int64_t total = n_segments + 1;
    launch_k(k_segment_offsets, static_cast<unsigned>((total + 255) / 256), 256, 0, st, keys, n, offsets, n_segments);
    dbg_launch("k_segment_offsets", st);
}

}  // namespace tk

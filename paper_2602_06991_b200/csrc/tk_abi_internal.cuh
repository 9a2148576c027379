// tk_abi_internal.cuh — shared state of the C-ABI translation units (tk_abi.cu: context,
// scene, frame entry points; tk_abi_map.cu: mapping iteration and structural edits;
// tk_abi_io.cu: checkpoints and queries).  Internal: included by those three files only.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <utility>
#include <vector>

#include "feature.cuh"
#include "geometric.cuh"
#include "mapedit.cuh"
#include "mapping.cuh"
#include "prepare.cuh"
#include "sort.cuh"
#include "tk_common.cuh"
#include "tk_render.h"

namespace tkabi {

inline thread_local std::string g_err;

struct TkError {
    tk_status st;
    std::string msg;
};

[[noreturn]] inline void fail(tk_status st, const std::string& msg) { throw TkError{st, msg}; }

#define CK(call)                                                                               \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess)                                                                 \
            fail(e_ == cudaErrorMemoryAllocation ? TK_ERR_OOM : TK_ERR_CUDA,                   \
                 std::string(#call) + ": " + cudaGetErrorString(e_));                          \
    } while (0)

#define CK_LAUNCH(ctx)                                                                         \
    do {                                                                                       \
        cudaError_t e_ = cudaGetLastError();                                                   \
        if (e_ != cudaSuccess) fail(TK_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e_)); \
    } while (0)

// Device memory pool (tk_abi.cu): freed blocks are cached per device and handed back to
// later allocations of up to their size (a block serves requests of at least half its size), so
// the map edits that regrow or compact GB-sized arrays (insert_gaussians, prune_map) and the
// capacity growth of the frame buffers do not pay cudaMalloc / cudaFree on every call.  A free
// synchronises the device first (as cudaFree does), so a cached block is never reused while a
// kernel on another stream still reads it.  On cudaMalloc failure the cache is returned to the
// driver and the allocation retried; the cache is emptied when the last context is destroyed.
void* pool_alloc(size_t bytes, size_t* got);
void pool_free(void* p, size_t bytes);
void pool_trim();

// Owning device allocation (move-only; returned to the pool on destruction or release()).
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) {
        o.p = nullptr;
        o.bytes = 0;
    }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p;
            bytes = o.bytes;
            o.p = nullptr;
            o.bytes = 0;
        }
        return *this;
    }
    ~DevBuf() { release(); }
    void release() {
        if (p) pool_free(p, bytes);
        p = nullptr;
        bytes = 0;
    }
};

template <class T>
T* ensure(DevBuf& b, size_t count) {
    const size_t need = std::max<size_t>(count, 1) * sizeof(T);
    if (b.bytes < need) {
        b.release();
        b.p = pool_alloc(tk::align_bytes(need + need / 8), &b.bytes);
    }
    return static_cast<T*>(b.p);
}

template <class T>
T* ptr(const DevBuf& b) {
    return static_cast<T*>(b.p);
}

struct PrepKey {
    double pose[7];
    double fx, fy, cx, cy, near_plane, far_plane, dilation;
    int width, height, tile_size;
    uint64_t scene_version;
    bool operator==(const PrepKey& o) const { return std::memcmp(this, &o, sizeof(PrepKey)) == 0; }
};

struct FwdKey {
    PrepKey prep;
    double tfloor, alpha_clamp, bg[3];
    bool operator==(const FwdKey& o) const { return std::memcmp(this, &o, sizeof(FwdKey)) == 0; }
};

// NCCL entry points, resolved at tk_comm_init time so the library loads without NCCL.
struct NcclApi {
    void* handle = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    bool load() {
        if (handle) return true;
        handle = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!handle) handle = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!handle) return false;
        GetUniqueId = reinterpret_cast<decltype(GetUniqueId)>(dlsym(handle, "ncclGetUniqueId"));
        CommInitRank = reinterpret_cast<decltype(CommInitRank)>(dlsym(handle, "ncclCommInitRank"));
        AllGather = reinterpret_cast<decltype(AllGather)>(dlsym(handle, "ncclAllGather"));
        AllReduce = reinterpret_cast<decltype(AllReduce)>(dlsym(handle, "ncclAllReduce"));
        CommDestroy = reinterpret_cast<decltype(CommDestroy)>(dlsym(handle, "ncclCommDestroy"));
        GetErrorString = reinterpret_cast<decltype(GetErrorString)>(dlsym(handle, "ncclGetErrorString"));
        return GetUniqueId && CommInitRank && AllGather && AllReduce && CommDestroy && GetErrorString;
    }
};
inline NcclApi g_nccl;

#define NK(call)                                                                               \
    do {                                                                                       \
        ncclResult_t r_ = (call);                                                              \
        if (r_ != ncclSuccess) fail(TK_ERR_NCCL, std::string(#call) + ": " + g_nccl.GetErrorString(r_)); \
    } while (0)

// CUDA-event phase timer on the context stream (tk_profile_*).
struct Profiler {
    bool on = false;
    std::vector<cudaEvent_t> pool;
    struct Rec {
        int phase;
        cudaEvent_t a, b;
    };
    std::vector<Rec> pending;
    double ms[TK_NUM_PHASES] = {};
    int64_t cnt[TK_NUM_PHASES] = {};
    cudaEvent_t get() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        return e;
    }
    void drain() {
        for (const Rec& r : pending) {
            float t = 0.f;
            CK(cudaEventSynchronize(r.b));
            CK(cudaEventElapsedTime(&t, r.a, r.b));
            ms[r.phase] += t;
            cnt[r.phase] += 1;
            pool.push_back(r.a);
            pool.push_back(r.b);
        }
        pending.clear();
    }
    ~Profiler() {
        for (const Rec& r : pending) {
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
        }
        for (cudaEvent_t e : pool) cudaEventDestroy(e);
    }
};

// One keyframe of SceneMap::keyframes, device-resident (ground-truth images + pose).
// The last kernel that reads a device input buffer: an asynchronous upload into the buffer waits
// for it alone rather than for all compute issued so far.
struct ReaderEvent {
    cudaEvent_t ev = nullptr;
    bool pending = false;
    void record(cudaStream_t st) {
        CK(cudaEventRecord(ev, st));
        pending = true;
    }
};

struct Keyframe {
    tk_pose pose{};
    int w = 0, h = 0, d = 0;
    bool has_feature = false;
    int64_t depth_n = 0;  // pixels with valid ground-truth depth (losses.cpp:68-71)
    DevBuf color, depth, feature, valid;
    void release() {
        color.release();
        depth.release();
        feature.release();
        valid.release();
    }
};

}  // namespace tkabi

using namespace tkabi;  // internal header: the ABI units use these names unqualified

struct tk_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;                    // main stream (tk_get_stream)
    cudaStream_t s_feat = nullptr, s_geo = nullptr;  // side streams: feature path, geometry backward
    cudaStream_t cur = nullptr;                       // stream the current call enqueues on
    cudaEvent_t ev_main = nullptr, ev_feat = nullptr, ev_geo = nullptr;
    // TK_HOST_ASYNC copies: host->device on s_in, device->host on s_out (both copy engines busy at
    // once); ev_cmp orders them after the compute issued so far, ev_in / ev_out order compute after them
    cudaStream_t s_in = nullptr, s_out = nullptr;
    cudaEvent_t ev_cmp = nullptr, ev_in = nullptr, ev_out[5] = {};
    bool out_pending[5] = {};
    // pose twists of asynchronous backward_geometric calls: a ring of host-mapped slots, copied
    // into the callers' structs at tk_synchronize
    static constexpr int kTwistSlots = 64;
    double* h_twist = nullptr;
    double* h_twist_dev = nullptr;
    std::vector<std::pair<double*, int>> twist_pending;
    int twist_next = 0;
    bool feat_pending = false, geo_pending = false;
    Profiler prof;
    // scene mirror
    int64_t n = 0;
    int32_t d = 0;
    uint64_t generation = 0;
    uint64_t scene_version = 0;
    bool has_scene = false, has_features = false;
    DevBuf mean, log_scale, rotation, opacity_logit, color, feature;
    // TK_HOST_ASYNC uploads are double-buffered: the next scene lands in the back set (which only
    // waits for the compute that read it, ev_scene_free) while the front set is still in use
    DevBuf mean_b, log_scale_b, rotation_b, opacity_logit_b, color_b, feature_b;
    cudaEvent_t ev_scene_free = nullptr;
    bool scene_free_pending = false;
    // last readers of the asynchronous upstream-gradient inputs (feature backward; geometry sweep)
    ReaderEvent fgrad_reader, ggrad_reader;
    // projection, per Gaussian
    DevBuf pmx, pmy, pixx, pixy, piyy, pz, pop, rect, valid, ntiles, pos;
    DevBuf dkeys, dvals, dkeys_alt, dvals_alt, ntiles_sorted, pair_off;
    DevBuf tkeys, tvals, tkeys_alt, tvals_alt, tile_offsets, padded_cnt, padded_start;
    DevBuf te;  // chunk-major tile entries (tk::EntryChunk)
    DevBuf wl, wl_count;  // per-warp culled entry lists (forward -> backward)
    DevBuf entry_pair;    // padded tile-entry position -> pair emission index (fixed-order merge)
    DevBuf emit_big;      // depth ranks whose tile rectangles are emitted by whole warps
    int64_t padded_cap = 0;
    DevBuf scratch, scratch_feat, dscal;
    int64_t* hscal = nullptr;      // host-mapped mirror of dscal (written by k_copy_words)
    int64_t* hscal_dev = nullptr;  //   its device address
    // prepared scene
    bool prepared = false;
    PrepKey prep_key{};
    int64_t n_vis = 0, n_pairs = 0;
    int tiles_x = 0, tiles_y = 0;
    const uint32_t* order = nullptr;
    const uint32_t* tile_keys_sorted = nullptr;
    const uint32_t* tile_vals_sorted = nullptr;
    // forward outputs / records
    DevBuf o_color, o_depth, o_alpha, o_index, o_weight, o_count, o_contrib, aux_t, aux_n;
    bool has_records = false;
    int rec_w = 0, rec_h = 0, rec_k = 0;
    uint64_t rec_generation = 0;
    int64_t rec_map_size = 0;
    bool aux_valid = false;
    FwdKey aux_key{};
    // external records staging
    DevBuf x_index, x_weight, x_count;
    // feature
    DevBuf f_out, f_grad_in, f_grad_out, s_keys, s_vals, s_keys_alt, s_vals_alt, s_queue, s_wnorm, s_seg;
    int64_t fout_pixels = 0;
    // geometric backward
    bool geom_atomic = false;  // TK_GEOM_BWD_ATOMIC=1: fp64 atomicAdd flush (non-deterministic)
    DevBuf g_part, g_flag, g_big;  // per-(entry, warp block) MidGrad partials, written flags, big ranks
    DevBuf g_color_in, g_depth_in, mid, twist, twist_part, twist_out, gg_mean, gg_ls, gg_rot, gg_op, gg_col;
    // full blend
    DevBuf l_count, l_off, l_src, l_w;
    // mapping iteration: keyframes, optimiser state (per group m / v), statistics, loss scratch
    std::vector<Keyframe> kfs;
    bool opt_ready = false;
    int64_t opt_n = 0, stat_n = -1;
    int32_t opt_d = 0;
    int64_t step_geo = 0, step_feat = 0;
    DevBuf am[5], av[5], fm, fv, stat_count, stat_maxc;
    DevBuf ssim_rows, ssim_win, l_gc, l_gd, l_partial, l_values, l_fscale, l_signs;
    double* hvals = nullptr;  // host-mapped {map, geo, feat} of the last optimize_step
    double* hvals_dev = nullptr;
    bool has_values = false;
    // segment_by_query scratch (kept across calls: no allocation on the query path)
    DevBuf q_feat, q_emb, q_labels, q_best, q_acc, q_nacc, q_part;
    DevBuf lp_items, lp_longs, lp_counters, lp_partial, lp_l1, lp_l1map;  // long-segment plan
    // lazy feature Adam: steps applied per row, every step's constants (host + device, 1-based);
    // feat_stale: some rows lag the step count (replayed by flush_features before features are read)
    DevBuf f_last, f_tab, f_active, f_active_n, f_active_grad;
    std::vector<tk::AdamStepParams> f_tab_host;
    bool feat_stale = false;
    DevBuf row_ss;                                        // D-sharded partial row norms
    // geometry split: this context sweeps band `band` of `band_n` (tk_geometry_band)
    int band = 0, band_n = 1;
    // multi-GPU
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0, d_total = 0;
    DevBuf gather_buf;
    // fused render_feature + all-gather over peer memory: every rank's full-width output buffer
    float* peer_ptrs[tk::kMaxPeers] = {};
    int peer_n = 0, peer_rank = 0, peer_dtotal = 0;
    int64_t peer_pixels = 0;
    bool peer_ipc = false;  // peer_ptrs[r != peer_rank] opened from CUDA IPC handles (tk_comm_p2p_setup)
    DevBuf peer_own, peer_word;
};

namespace tkabi {

struct PhaseScope {
    tk_ctx* c;
    int phase;
    cudaEvent_t a = nullptr;
    PhaseScope(tk_ctx* ctx, int ph) : c(ctx), phase(ph) {
        if (c->prof.on) {
            a = c->prof.get();
            CK(cudaEventRecord(a, c->cur));
        }
    }
    ~PhaseScope() {
        if (a) {
            cudaEvent_t b = c->prof.get();
            cudaEventRecord(b, c->cur);
            c->prof.pending.push_back({phase, a, b});
        }
    }
};

inline tk_status guard_status(const TkError& e) {
    g_err = e.msg;
    return e.st;
}

template <class F>
tk_status guarded(F&& f) {
    try {
        f();
        g_err.clear();
        return TK_OK;
    } catch (const TkError& e) {
        return guard_status(e);
    } catch (const std::exception& e) {
        g_err = e.what();
        return TK_ERR_STATE;
    }
}

// Asynchronous device->host copies are tagged by the buffers they read, so only the compute that
// overwrites those buffers waits for them (kOutMisc: waited at the start of every call).
enum OutTag { kOutMisc = 0, kOutRec = 1, kOutF = 2, kOutDF = 3, kOutGG = 4 };

struct Records {
    int w = 0, h = 0, k = 0;
    const int32_t* index = nullptr;
    const double* weight = nullptr;
    const uint8_t* count = nullptr;
};

struct SlotIndex {
    const int32_t* seg;
    const uint32_t* slots;
    const float* wnorm;
    tk::LongPlan plan;  // chunks of the segments longer than tk::kLongSeg
};

// helpers defined in tk_abi.cu
void copy_in(void* dst, const void* src, size_t bytes, int mem, tk_ctx* c, const ReaderEvent* reader = nullptr);
void copy_out(void* dst, const void* src, size_t bytes, int mem, tk_ctx* c, int tag = kOutMisc);
void sync(tk_ctx* c);
void wait_out(tk_ctx* c, int tag);
void wait_async_out(tk_ctx* c);
void on_main(tk_ctx* c);
void main_done(tk_ctx* c);
void on_side(tk_ctx* c, bool feat);
void side_done(tk_ctx* c, bool feat);
int bits_for(uint64_t max_value);
void check_frame(const tk_camera* cam, const tk_settings* s);
tk::Frame make_frame(tk_ctx* c, const tk_camera* cam, const tk_settings* s);
PrepKey make_prep_key(tk_ctx* c, const tk_pose* pose, const tk_camera* cam, const tk_settings* s);
FwdKey make_fwd_key(const PrepKey& pk, const tk_settings* s);
tk::TileEntries tile_entries(tk_ctx* c);
void ensure_scratch(tk_ctx* c, int64_t n, bool feat = false);
void prepare(tk_ctx* c, const tk_pose* pose, const tk_camera* cam, const tk_settings* s);
void forward(tk_ctx* c, const tk_camera* cam, const tk_settings* s, bool records);
std::string stale_message(const char* fn, int32_t idx, int64_t n);
Records resolve_records(tk_ctx* c, const tk_topk_view* v, const char* fn);
SlotIndex build_slot_index(tk_ctx* c, const Records& r);
double* geom_sweep(tk_ctx* c, const tk::Frame& f, const double* gc, const double* gd);
tk::ChainParams chain_params(tk_ctx* c, const tk_pose* pose, const tk_camera* cam, const tk_settings* s,
                             const double* mid);
void scene_changed(tk_ctx* c);
void release_peers(tk_ctx* c);
// Bring every row of the lazily optimised features up to the current feature step (no-op unless
// a lazy step left rows behind).  Called before anything reads or replaces features or moments.
void flush_features(tk_ctx* c);
void require_features(tk_ctx* c);

}  // namespace tkabi

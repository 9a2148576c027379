// tk_abi.cu — the C ABI (include/tk_render.h): context, device-resident scene mirror, and the
// host orchestration of the sm_100a kernels for each reference entry point.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "feature.cuh"
#include "geometric.cuh"
#include "mapedit.cuh"
#include "mapping.cuh"
#include "prepare.cuh"
#include "sort.cuh"
#include "tk_common.cuh"
#include "tk_render.h"

namespace {

thread_local std::string g_err;

struct TkError {
    tk_status st;
    std::string msg;
};

[[noreturn]] void fail(tk_status st, const std::string& msg) { throw TkError{st, msg}; }

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

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
};

template <class T>
T* ensure(DevBuf& b, size_t count) {
    const size_t need = std::max<size_t>(count, 1) * sizeof(T);
    if (b.bytes < need) {
        b.release();
        const size_t alloc = tk::align_bytes(need + need / 8);
        CK(cudaMalloc(&b.p, alloc));
        b.bytes = alloc;
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
NcclApi g_nccl;

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

}  // namespace

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
    int64_t launches = 0;
    Profiler prof;
    // scene mirror
    int64_t n = 0;
    int32_t d = 0;
    uint64_t generation = 0;
    uint64_t scene_version = 0;
    bool has_scene = false, has_features = false;
    DevBuf mean, log_scale, rotation, opacity_logit, color, feature;
    // projection, per Gaussian
    DevBuf pmx, pmy, pixx, pixy, piyy, pz, pop, rect, valid, ntiles, pos;
    DevBuf dkeys, dvals, dkeys_alt, dvals_alt, ntiles_sorted, pair_off;
    DevBuf tkeys, tvals, tkeys_alt, tvals_alt, tile_offsets, padded_cnt, padded_start;
    DevBuf te;  // chunk-major tile entries (tk::EntryChunk)
    DevBuf wl, wl_count;  // per-warp culled entry lists (forward -> backward)
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
    DevBuf f_out, f_grad_in, f_grad_out, s_keys, s_vals, s_keys_alt, s_vals_alt, s_wnorm, s_seg;
    int64_t fout_pixels = 0;
    // geometric backward
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
    DevBuf lp_items, lp_longs, lp_counters, lp_partial;  // long-segment chunk plan
    DevBuf row_ss;                                        // D-sharded partial row norms
    // multi-GPU
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0, d_total = 0;
    DevBuf gather_buf;
};

namespace {

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

tk_status guard_status(const TkError& e) {
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

// Host <-> device copies made inside an API call (timed as TK_PHASE_COPY when profiling).
void copy_in(void* dst, const void* src, size_t bytes, int mem, tk_ctx* c) {
    if (bytes == 0) return;
    if (mem == TK_HOST_ASYNC) {  // after the compute issued so far (it may still read dst), before what follows
        CK(cudaEventRecord(c->ev_cmp, c->cur));
        CK(cudaStreamWaitEvent(c->s_in, c->ev_cmp, 0));
        if (c->out_pending[0]) CK(cudaStreamWaitEvent(c->s_in, c->ev_out[0], 0));  // untagged reads (misc)
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->s_in));
        CK(cudaEventRecord(c->ev_in, c->s_in));
        CK(cudaStreamWaitEvent(c->cur, c->ev_in, 0));
        return;
    }
    PhaseScope phase(c, TK_PHASE_COPY);
    CK(cudaMemcpyAsync(dst, src, bytes, mem == TK_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                       c->cur));
}

// Asynchronous device->host copies are tagged by the buffers they read, so only the compute that
// overwrites those buffers waits for them (kOutMisc: waited at the start of every call).
enum OutTag { kOutMisc = 0, kOutRec = 1, kOutF = 2, kOutDF = 3, kOutGG = 4 };

void copy_out(void* dst, const void* src, size_t bytes, int mem, tk_ctx* c, int tag = kOutMisc) {
    if (bytes == 0 || dst == nullptr) return;
    if (mem == TK_HOST_ASYNC) {  // after the compute that produced src; its overwriters wait for it
        CK(cudaEventRecord(c->ev_cmp, c->cur));
        CK(cudaStreamWaitEvent(c->s_out, c->ev_cmp, 0));
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->s_out));
        CK(cudaEventRecord(c->ev_out[tag], c->s_out));
        c->out_pending[tag] = true;
        return;
    }
    PhaseScope phase(c, TK_PHASE_COPY);
    CK(cudaMemcpyAsync(dst, src, bytes, mem == TK_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                       c->cur));
}

void sync(tk_ctx* c) { CK(cudaStreamSynchronize(c->cur)); }

// Stream discipline.  The main stream owns everything that (re)writes the scene mirror, the
// PreparedScene and the forward records; the feature calls run on s_feat and the geometry
// backward on s_geo, each ordered after the main stream's latest work (ev_main), so the
// HBM-bound feature kernels and the fp64-bound geometry backward overlap.  Main-stream work
// first waits for outstanding side-stream work that still reads those buffers.
// Compute issued from here on may overwrite the buffers an asynchronous device->host copy of
// this tag still reads: order it after that copy.
void wait_out(tk_ctx* c, int tag) {
    if (c->out_pending[tag]) {
        CK(cudaStreamWaitEvent(c->cur, c->ev_out[tag], 0));
        if (c->cur != c->stream) CK(cudaStreamWaitEvent(c->stream, c->ev_out[tag], 0));
        c->out_pending[tag] = false;
    }
}
void wait_async_out(tk_ctx* c) { wait_out(c, kOutMisc); }

void on_main(tk_ctx* c) {
    c->cur = c->stream;
    wait_async_out(c);
    if (c->feat_pending) {
        CK(cudaStreamWaitEvent(c->stream, c->ev_feat, 0));
        c->feat_pending = false;
    }
    if (c->geo_pending) {
        CK(cudaStreamWaitEvent(c->stream, c->ev_geo, 0));
        c->geo_pending = false;
    }
}
void main_done(tk_ctx* c) { CK(cudaEventRecord(c->ev_main, c->stream)); }
void on_side(tk_ctx* c, bool feat) {
    c->cur = feat ? c->s_feat : c->s_geo;
    CK(cudaStreamWaitEvent(c->cur, c->ev_main, 0));
    wait_async_out(c);
}
void side_done(tk_ctx* c, bool feat) {
    CK(cudaEventRecord(feat ? c->ev_feat : c->ev_geo, c->cur));
    if (feat) c->feat_pending = true;
    else c->geo_pending = true;
}

int bits_for(uint64_t max_value) {  // bits needed to represent values in [0, max_value]
    int b = 0;
    while (b < 64 && (max_value >> b) != 0) ++b;
    return b;
}

void check_frame(const tk_camera* cam, const tk_settings* s) {
    if (!cam || !s) fail(TK_ERR_BAD_ARG, "null camera or settings");
    if (cam->width <= 0 || cam->height <= 0) fail(TK_ERR_BAD_ARG, "camera width/height must be positive");
    if (s->tile_size <= 0) fail(TK_ERR_BAD_ARG, "tile_size must be positive");
    if (s->top_k < 0) fail(TK_ERR_BAD_ARG, "top_k must be >= 0");
}

tk::Frame make_frame(tk_ctx* c, const tk_camera* cam, const tk_settings* s) {
    tk::Frame f{};
    f.width = cam->width;
    f.height = cam->height;
    f.tile_size = s->tile_size;
    f.tiles_x = (cam->width + s->tile_size - 1) / s->tile_size;   // render.cpp:122-123
    f.tiles_y = (cam->height + s->tile_size - 1) / s->tile_size;
    f.k = std::min(s->top_k, tk::kMaxTopK);                        // render.cpp:161
    f.tfloor = s->transmittance_floor;
    f.alpha_clamp = s->alpha_clamp;
    for (int i = 0; i < 3; ++i) f.bg[i] = s->background[i];
    (void)c;
    return f;
}

PrepKey make_prep_key(tk_ctx* c, const tk_pose* pose, const tk_camera* cam, const tk_settings* s) {
    PrepKey k;
    std::memset(&k, 0, sizeof(k));
    const double pv[7] = {pose->qw, pose->qx, pose->qy, pose->qz, pose->tx, pose->ty, pose->tz};
    std::memcpy(k.pose, pv, sizeof(pv));
    k.fx = cam->fx;
    k.fy = cam->fy;
    k.cx = cam->cx;
    k.cy = cam->cy;
    k.near_plane = cam->near_plane;
    k.far_plane = cam->far_plane;
    k.dilation = s->cov2d_dilation;
    k.width = cam->width;
    k.height = cam->height;
    k.tile_size = s->tile_size;
    k.scene_version = c->scene_version;
    return k;
}

FwdKey make_fwd_key(const PrepKey& pk, const tk_settings* s) {
    FwdKey k;
    std::memset(&k, 0, sizeof(k));
    k.prep = pk;
    k.tfloor = s->transmittance_floor;
    k.alpha_clamp = s->alpha_clamp;
    for (int i = 0; i < 3; ++i) k.bg[i] = s->background[i];
    return k;
}

tk::TileEntries tile_entries(tk_ctx* c) {
    tk::TileEntries t;
    t.chunks = ptr<tk::EntryChunk>(c->te);
    return t;
}

void ensure_scratch(tk_ctx* c, int64_t n, bool feat = false) {
    const size_t need = std::max(tk::radix_scratch_bytes(n), tk::scan_scratch_bytes(n + 1));
    ensure<char>(feat ? c->scratch_feat : c->scratch, need);
}

// prepare_scene (render.cpp:73-156) on the device; cached on (pose, camera, settings, scene).
void prepare(tk_ctx* c, const tk_pose* pose, const tk_camera* cam, const tk_settings* s) {
    if (!c->has_scene) fail(TK_ERR_STATE, "no scene uploaded (tk_scene_upload)");
    const PrepKey key = make_prep_key(c, pose, cam, s);
    if (c->prepared && c->prep_key == key) return;
    c->prepared = false;
    c->aux_valid = false;
    PhaseScope phase(c, TK_PHASE_PREPARE);
    const int64_t n = c->n;
    cudaStream_t st = c->cur;
    const tk::Frame f = make_frame(c, cam, s);
    const int n_tiles = f.tiles_x * f.tiles_y;
    c->tiles_x = f.tiles_x;
    c->tiles_y = f.tiles_y;
    int64_t* dscal = ensure<int64_t>(c->dscal, 16);
    ensure_scratch(c, std::max<int64_t>(n, n_tiles + 1));

    tk::ProjectParams pp{};
    pp.n = n;
    pp.mean = ptr<double>(c->mean);
    pp.log_scale = ptr<double>(c->log_scale);
    pp.rotation = ptr<double>(c->rotation);
    pp.opacity_logit = ptr<double>(c->opacity_logit);
    const double pv[7] = {pose->qw, pose->qx, pose->qy, pose->qz, pose->tx, pose->ty, pose->tz};
    std::memcpy(pp.pose, pv, sizeof(pv));
    pp.fx = cam->fx;
    pp.fy = cam->fy;
    pp.cx = cam->cx;
    pp.cy = cam->cy;
    pp.near_plane = cam->near_plane;
    pp.far_plane = cam->far_plane;
    pp.dilation = s->cov2d_dilation;
    pp.tile_size = s->tile_size;
    pp.tiles_x = f.tiles_x;
    pp.tiles_y = f.tiles_y;
    pp.mx = ensure<double>(c->pmx, n);
    pp.my = ensure<double>(c->pmy, n);
    pp.ixx = ensure<double>(c->pixx, n);
    pp.ixy = ensure<double>(c->pixy, n);
    pp.iyy = ensure<double>(c->piyy, n);
    pp.z = ensure<double>(c->pz, n);
    pp.opacity = ensure<double>(c->pop, n);
    pp.rect = ensure<int4>(c->rect, n);
    pp.valid = ensure<int32_t>(c->valid, n);
    pp.ntiles = ensure<int32_t>(c->ntiles, n);
    pp.key_min = reinterpret_cast<uint64_t*>(dscal + 1);
    pp.key_max = reinterpret_cast<uint64_t*>(dscal + 2);
    CK(cudaMemsetAsync(dscal + 1, 0xff, sizeof(int64_t), st));
    CK(cudaMemsetAsync(dscal + 2, 0, sizeof(int64_t), st));
    tk::launch_project(pp, st);
    c->launches += n > 0;
    CK_LAUNCH(c);

    int32_t* pos = ensure<int32_t>(c->pos, n);
    tk::scan_exclusive(pp.valid, pos, n, dscal + 0, c->scratch.p, st, &c->launches);
    uint64_t* dkeys = ensure<uint64_t>(c->dkeys, n);
    uint32_t* dvals = ensure<uint32_t>(c->dvals, n);
    uint64_t* dkeys_alt = ensure<uint64_t>(c->dkeys_alt, n);
    uint32_t* dvals_alt = ensure<uint32_t>(c->dvals_alt, n);
    tk::launch_compact(pp.valid, pos, pp.z, n, pp.key_min, dkeys, dvals, st);
    c->launches += n > 0;
    CK_LAUNCH(c);
    tk::copy_words_to_mapped(c->hscal_dev, dscal, 3, st);
    sync(c);
    const int64_t n_vis = n > 0 ? c->hscal[0] : 0;
    const uint64_t kmin = static_cast<uint64_t>(c->hscal[1]), kmax = static_cast<uint64_t>(c->hscal[2]);
    c->n_vis = n_vis;

    // Depth sort (render.cpp:108-111): stable LSD radix over the top 24 bits in which the visible
    // fp64 depth keys differ (values start in src order), then every run of equal high bits is
    // ordered by (full key, src).  A run longer than 64 keys triggers a full-width sort instead.
    const int hb = n_vis > 1 ? bits_for(kmax - kmin) : 0;
    int32_t* nts = ensure<int32_t>(c->ntiles_sorted, n_vis);
    int32_t* poff = ensure<int32_t>(c->pair_off, n_vis);
    auto depth_sort = [&](int lo_bit) {
        bool alt = false;
        CK(cudaMemsetAsync(dscal + 7, 0, sizeof(int64_t), st));
        if (n_vis > 1) {
            tk::radix_sort_pairs_u64(dkeys, dvals, dkeys_alt, dvals_alt, n_vis, lo_bit, hb, c->scratch.p, st, &alt,
                                     &c->launches);
            tk::fixup_runs_u64(alt ? dkeys_alt : dkeys, alt ? dvals_alt : dvals, n_vis, lo_bit,
                               reinterpret_cast<int32_t*>(dscal + 7), st, &c->launches);
            CK_LAUNCH(c);
        }
        c->order = alt ? dvals_alt : dvals;
        tk::launch_sorted_ntiles(c->order, n_vis, pp.ntiles, nts, st);
        c->launches += n_vis > 0;
        tk::scan_exclusive(nts, poff, n_vis, dscal + 3, c->scratch.p, st, &c->launches);
        tk::copy_words_to_mapped(c->hscal_dev + 3, dscal + 3, 5, st);
        sync(c);
    };
    const int lo = hb > 24 ? hb - 24 : 0;
    depth_sort(lo);
    if (lo > 0 && c->hscal[7] != 0) {  // pathological run of near-equal depths: sort every bit
        tk::launch_compact(pp.valid, pos, pp.z, n, pp.key_min, dkeys, dvals, st);
        depth_sort(0);
    }
    const int64_t n_pairs = n_vis > 0 ? c->hscal[3] : 0;
    if (n_pairs > INT32_MAX) fail(TK_ERR_BAD_ARG, "tile list exceeds 2^31 entries");
    c->n_pairs = n_pairs;

    uint32_t* tkeys = ensure<uint32_t>(c->tkeys, n_pairs);
    uint32_t* tvals = ensure<uint32_t>(c->tvals, n_pairs);
    uint32_t* tkeys_alt = ensure<uint32_t>(c->tkeys_alt, n_pairs);
    uint32_t* tvals_alt = ensure<uint32_t>(c->tvals_alt, n_pairs);
    tk::launch_emit_pairs(c->order, n_vis, pp.rect, nts, poff, f.tiles_x, tkeys, tvals, st);
    c->launches += n_vis > 0;
    ensure_scratch(c, std::max<int64_t>(n_pairs, n_tiles + 1));
    bool talt = false;
    const int tbits = bits_for(static_cast<uint64_t>(n_tiles - 1));
    if (n_pairs > 1 && tbits > 0) {
        tk::radix_sort_pairs_u32(tkeys, tvals, tkeys_alt, tvals_alt, n_pairs, 0, tbits, c->scratch.p, st, &talt,
                                 &c->launches);
    }
    c->tile_keys_sorted = talt ? tkeys_alt : tkeys;
    c->tile_vals_sorted = talt ? tvals_alt : tvals;
    int32_t* toff = ensure<int32_t>(c->tile_offsets, n_tiles + 1);
    tk::segment_offsets_u32(c->tile_keys_sorted, n_pairs, toff, n_tiles, st, &c->launches);
    int32_t* pcnt = ensure<int32_t>(c->padded_cnt, n_tiles + 1);
    int32_t* pstart = ensure<int32_t>(c->padded_start, n_tiles + 1);
    tk::launch_padded_counts(toff, n_tiles, pcnt, st);
    c->launches += 1;
    tk::scan_exclusive(pcnt, pstart, n_tiles + 1, dscal + 4, c->scratch.p, st, &c->launches);
    const int64_t padded_cap = n_pairs + static_cast<int64_t>(tk::kEntryAlign) * n_tiles + 128;
    ensure<tk::EntryChunk>(c->te, padded_cap / tk::kChunk + 1);
    ensure<int32_t>(c->wl, padded_cap * tk::geom_blocks_per_tile(s->tile_size));
    tk::MaterializeParams mp{};
    mp.n_pairs = n_pairs;
    mp.tile_keys = c->tile_keys_sorted;
    mp.tile_vals = c->tile_vals_sorted;
    mp.tile_offsets = toff;
    mp.padded_start = pstart;
    mp.order = c->order;
    mp.mx = pp.mx;
    mp.my = pp.my;
    mp.ixx = pp.ixx;
    mp.ixy = pp.ixy;
    mp.iyy = pp.iyy;
    mp.z = pp.z;
    mp.opacity = pp.opacity;
    mp.color = ptr<double>(c->color);
    mp.out = tile_entries(c);
    tk::launch_materialize(mp, st);
    c->launches += n_pairs > 0;
    CK_LAUNCH(c);
    c->prepared = true;
    c->prep_key = key;
}


// geometric_pass (render.cpp:158-240).  Record/colour outputs are optional (null = skip);
// the per-pixel aux (final T, entries visited) is always written for the backward.
void forward(tk_ctx* c, const tk_camera* cam, const tk_settings* s, bool records) {
    const tk::Frame f = make_frame(c, cam, s);
    const int64_t P = static_cast<int64_t>(f.width) * f.height;
    const int k = f.k;
    cudaStream_t st = c->cur;
    tk::GeomFwdParams gp{};
    gp.f = f;
    gp.te = tile_entries(c);
    gp.tile_offsets = ptr<int32_t>(c->tile_offsets);
    gp.padded_start = ptr<int32_t>(c->padded_start);
    gp.aux.t_final = ensure<double>(c->aux_t, P);
    gp.aux.n_iter = ensure<int32_t>(c->aux_n, P);
    gp.aux.wl = ptr<int32_t>(c->wl);
    gp.aux.wl_count = ensure<int32_t>(c->wl_count, tk::geom_blocks(f));
    gp.pair_count = reinterpret_cast<unsigned long long*>(ensure<int64_t>(c->dscal, 16) + 13);  // tk_pair_count
    if (records) {
        wait_out(c, kOutRec);
        gp.color = ensure<double>(c->o_color, P * 3);
        gp.depth = ensure<double>(c->o_depth, P);
        gp.alpha = ensure<double>(c->o_alpha, P);
        gp.topk_index = ensure<int32_t>(c->o_index, P * std::max(k, 1));
        gp.topk_weight = ensure<double>(c->o_weight, P * std::max(k, 1));
        gp.topk_count = ensure<uint8_t>(c->o_count, P);
        gp.contrib = ensure<unsigned long long>(c->o_contrib, c->n);
        CK(cudaMemsetAsync(gp.contrib, 0, std::max<int64_t>(c->n, 1) * sizeof(double), st));
    }
    const int nblk = tk::geom_blocks(f);
    {
        PhaseScope phase(c, TK_PHASE_GEOM_FWD);
        tk::launch_geom_fwd(tk::kGeomForward, gp, nblk, st);
    }
    c->launches += 1;
    CK_LAUNCH(c);
    if (records) {
        c->has_records = true;
        c->rec_w = f.width;
        c->rec_h = f.height;
        c->rec_k = k;
        c->rec_generation = c->generation;
        c->rec_map_size = c->n;
    }
}

std::string stale_message(const char* fn, int32_t idx, int64_t n) {
    return std::string(fn) + ": top-k record references gaussian " + std::to_string(idx) + " but the map holds " +
           std::to_string(n) + " (stale snapshot)";
}

struct Records {
    int w = 0, h = 0, k = 0;
    const int32_t* index = nullptr;
    const double* weight = nullptr;
    const uint8_t* count = nullptr;
};

// Resolve a TopKGrid argument to device pointers, with the reference's stale-index check
// (render.cpp:305-311, backward.cpp:278-283) done before any work.
Records resolve_records(tk_ctx* c, const tk_topk_view* v, const char* fn) {
    Records r;
    const int64_t n = c->n;
    cudaStream_t st = c->cur;
    if (!v) {
        if (!c->has_records) fail(TK_ERR_STATE, std::string(fn) + ": no records (call tk_render_geometric first)");
        r.w = c->rec_w;
        r.h = c->rec_h;
        r.k = c->rec_k;
        r.index = ptr<int32_t>(c->o_index);
        r.weight = ptr<double>(c->o_weight);
        r.count = ptr<uint8_t>(c->o_count);
        if (c->rec_map_size <= n) return r;  // indices < rec_map_size <= n by construction
    } else {
        if (v->width < 0 || v->height < 0 || v->k < 0) fail(TK_ERR_BAD_ARG, "negative TopKGrid shape");
        r.w = v->width;
        r.h = v->height;
        r.k = v->k;
        const int64_t slots = static_cast<int64_t>(r.w) * r.h * r.k;
        const int64_t P = static_cast<int64_t>(r.w) * r.h;
        if (v->mem == TK_HOST) {
            for (int64_t q = 0; q < slots; ++q)
                if (v->index[q] >= n) fail(TK_ERR_STALE_INDEX, stale_message(fn, v->index[q], n));
            int32_t* di = ensure<int32_t>(c->x_index, slots);
            double* dw = ensure<double>(c->x_weight, slots);
            uint8_t* dc = ensure<uint8_t>(c->x_count, P);
            copy_in(di, v->index, slots * sizeof(int32_t), TK_HOST, c);
            copy_in(dw, v->weight, slots * sizeof(double), TK_HOST, c);
            copy_in(dc, v->count, P, TK_HOST, c);
            r.index = di;
            r.weight = dw;
            r.count = dc;
            return r;
        }
        r.index = v->index;
        r.weight = v->weight;
        r.count = v->count;
    }
    // device-side check: first offending slot in slot order
    const int64_t slots = static_cast<int64_t>(r.w) * r.h * r.k;
    int64_t* dscal = ensure<int64_t>(c->dscal, 16);
    CK(cudaMemsetAsync(dscal + 5, 0xff, sizeof(int64_t), st));
    tk::launch_first_stale(r.index, slots, n, reinterpret_cast<unsigned long long*>(dscal + 5), st);
    c->launches += slots > 0;
    tk::copy_words_to_mapped(c->hscal_dev + 5, dscal + 5, 1, st);
    sync(c);
    const uint64_t first = static_cast<uint64_t>(c->hscal[5]);
    if (first != ~0ull) {
        int32_t idx = 0;
        CK(cudaMemcpy(&idx, r.index + first, sizeof(int32_t), cudaMemcpyDeviceToHost));
        fail(TK_ERR_STALE_INDEX, stale_message(fn, idx, n));
    }
    return r;
}

struct SlotIndex {
    const int32_t* seg;
    const uint32_t* slots;
    const float* wnorm;
    tk::LongPlan plan;  // chunks of the segments longer than tk::kLongSeg
};

// Inverted (Gaussian -> record slots) index of a TopKGrid, ascending slot order per Gaussian.
SlotIndex build_slot_index(tk_ctx* c, const Records& r) {
    const int64_t slots = static_cast<int64_t>(r.w) * r.h * r.k;
    const int64_t n = c->n;
    uint32_t* recs = ensure<uint32_t>(c->s_keys, slots);
    uint32_t* svals = ensure<uint32_t>(c->s_vals, slots);
    int32_t* cursor = ensure<int32_t>(c->s_keys_alt, n + 2);
    float* wn = ensure<float>(c->s_wnorm, slots);
    int32_t* seg = ensure<int32_t>(c->s_seg, n + 1);
    ensure_scratch(c, std::max<int64_t>(slots, n + 1), true);
    PhaseScope phase(c, TK_PHASE_FBWD_INDEX);
    tk::SlotKeyParams sk{slots, r.k, n, r.index, r.weight, r.count, nullptr, nullptr, wn};
    int64_t* dscal = ensure<int64_t>(c->dscal, 16);
    tk::launch_slot_index(sk, n, seg, cursor, recs, svals, dscal + 8, c->scratch_feat.p, c->cur, &c->launches);
    tk::LongPlan plan{};
    plan.cap_items = tk::long_plan_capacity(slots, n);
    plan.items = ensure<int4>(c->lp_items, plan.cap_items);
    plan.longs = ensure<int4>(c->lp_longs, plan.cap_items);
    plan.counters = ensure<int32_t>(c->lp_counters, 2);
    plan.partial = ensure<float>(c->lp_partial, plan.cap_items * std::max(c->d, 1));
    plan.queue = cursor;
    plan.qcount = cursor + n + 1;
    tk::launch_long_plan(seg, n, plan, c->cur);
    c->launches += 1;
    return SlotIndex{seg, svals, wn, plan};
}

// The backward sweep of backward_geometric (backward.cpp:106-188) into the per-Gaussian
// projected-space gradients (n x 10), on the forward state of this context.
double* geom_sweep(tk_ctx* c, const tk::Frame& f, const double* gc, const double* gd) {
    const int64_t n = c->n;
    double* mid = ensure<double>(c->mid, n * 10);
    CK(cudaMemsetAsync(mid, 0, std::max<int64_t>(n, 1) * 10 * sizeof(double), c->cur));
    tk::GeomBwdParams bp{};
    bp.f = f;
    bp.te = tile_entries(c);
    bp.tile_offsets = ptr<int32_t>(c->tile_offsets);
    bp.padded_start = ptr<int32_t>(c->padded_start);
    bp.aux.t_final = ptr<double>(c->aux_t);
    bp.aux.n_iter = ptr<int32_t>(c->aux_n);
    bp.aux.wl = ptr<int32_t>(c->wl);
    bp.aux.wl_count = ptr<int32_t>(c->wl_count);
    bp.grad_color = gc;
    bp.grad_depth = gd;
    bp.mid = mid;
    {
        PhaseScope phase(c, TK_PHASE_GEOM_BWD);
        tk::launch_geom_bwd(bp, tk::geom_blocks(f), c->cur);
    }
    c->launches += 1;
    CK_LAUNCH(c);
    return mid;
}

tk::ChainParams chain_params(tk_ctx* c, const tk_pose* pose, const tk_camera* cam, const tk_settings* s,
                             const double* mid) {
    tk::ChainParams cp{};
    cp.n = c->n;
    cp.mid = mid;
    cp.mean = ptr<double>(c->mean);
    cp.log_scale = ptr<double>(c->log_scale);
    cp.rotation = ptr<double>(c->rotation);
    cp.opacity_logit = ptr<double>(c->opacity_logit);
    const double pv[7] = {pose->qw, pose->qx, pose->qy, pose->qz, pose->tx, pose->ty, pose->tz};
    std::memcpy(cp.pose, pv, sizeof(pv));
    cp.fx = cam->fx;
    cp.fy = cam->fy;
    cp.dilation = s->cov2d_dilation;
    return cp;
}

// Grow a device array to new_count elements keeping the first old_count (structural edits).
template <class T>
T* grow_keep(tk_ctx* c, DevBuf& b, int64_t old_count, int64_t new_count, bool zero_tail) {
    const size_t need = static_cast<size_t>(std::max<int64_t>(new_count, 1)) * sizeof(T);
    if (b.bytes < need) {
        DevBuf nb;
        const size_t alloc = tk::align_bytes(need + need / 8);
        CK(cudaMalloc(&nb.p, alloc));
        nb.bytes = alloc;
        if (old_count > 0 && b.p)
            CK(cudaMemcpyAsync(nb.p, b.p, old_count * sizeof(T), cudaMemcpyDeviceToDevice, c->cur));
        CK(cudaStreamSynchronize(c->cur));
        b.release();
        b = nb;
    }
    if (zero_tail && new_count > old_count)
        CK(cudaMemsetAsync(ptr<T>(b) + old_count, 0, (new_count - old_count) * sizeof(T), c->cur));
    return ptr<T>(b);
}

// Keep the rows flagged in keep (n rows of `width` elements) in order, into a fresh buffer.
template <class T>
void compact_rows(tk_ctx* c, DevBuf& b, int64_t n, int width, int64_t n_keep, const int32_t* keep,
                  const int32_t* pos) {
    if (!b.p || width <= 0) return;
    DevBuf nb;
    ensure<T>(nb, std::max<int64_t>(n_keep, 1) * width);
    if (sizeof(T) == 8)
        tk::launch_compact_f64(reinterpret_cast<const double*>(b.p), static_cast<double*>(nb.p), keep, pos, n, width,
                               c->cur);
    else
        tk::launch_compact_f32(reinterpret_cast<const float*>(b.p), static_cast<float*>(nb.p), keep, pos, n, width,
                               c->cur);
    c->launches += n > 0;
    CK_LAUNCH(c);
    CK(cudaStreamSynchronize(c->cur));
    b.release();
    b = nb;
}

// prune_map's candidate draw (mapper.cpp:80-139), host side: candidates have topk_count <=
// threshold; ceil(keep_ratio * candidates) survive, drawn without replacement proportionally to
// max_contribution with std::mt19937_64(seed), uniformly once the mass is exhausted.
std::vector<int32_t> prune_select(const std::vector<int32_t>& counts, const std::vector<double>& maxc,
                                  double keep_ratio, uint64_t seed, int32_t threshold) {
    std::vector<int32_t> cand;
    for (size_t i = 0; i < counts.size(); ++i)
        if (counts[i] <= threshold) cand.push_back(static_cast<int32_t>(i));
    std::vector<int32_t> removed;
    if (cand.empty()) return removed;
    std::vector<double> score(cand.size());
    double total = 0.0;
    for (size_t i = 0; i < cand.size(); ++i) {
        score[i] = maxc[cand[i]];
        total += score[i];
    }
    if (!(total > 0.0)) return removed;  // survival weights undefined: keep every candidate
    const size_t keep = static_cast<size_t>(std::ceil(keep_ratio * static_cast<double>(cand.size())));
    if (keep >= cand.size()) return removed;
    std::mt19937_64 rng(seed);
    std::vector<uint8_t> kept(cand.size(), 0);
    std::vector<size_t> pool(cand.size());
    for (size_t i = 0; i < pool.size(); ++i) pool[i] = i;
    double mass = total;
    for (size_t draw = 0; draw < keep; ++draw) {
        size_t pick = 0;
        if (mass > 0.0) {
            const double u = static_cast<double>(rng() >> 11) * 0x1.0p-53 * mass;  // canonical_unit * mass
            double acc = 0.0;
            pick = pool.size() - 1;
            for (size_t q = 0; q < pool.size(); ++q) {
                acc += score[pool[q]];
                if (u < acc) {
                    pick = q;
                    break;
                }
            }
        } else {
            pick = static_cast<size_t>(rng() % pool.size());
        }
        const size_t chosen = pool[pick];
        kept[chosen] = 1;
        mass -= score[chosen];
        if (mass < 0.0) mass = 0.0;
        pool.erase(pool.begin() + static_cast<std::ptrdiff_t>(pick));
    }
    for (size_t i = 0; i < cand.size(); ++i)
        if (!kept[i]) removed.push_back(cand[i]);
    return removed;
}

void scene_changed(tk_ctx* c) {
    c->scene_version += 1;
    c->prepared = false;
    c->aux_valid = false;
}

void require_features(tk_ctx* c) {
    if (!c->has_scene) fail(TK_ERR_STATE, "no scene uploaded (tk_scene_upload)");
    if (!c->has_features) fail(TK_ERR_STATE, "scene has no features uploaded");
}

}  // namespace

// =========================================================================================
extern "C" {

void tk_default_settings(tk_settings* s) {  // render.hpp:14-21
    s->top_k = 3;
    s->tile_size = 16;
    s->transmittance_floor = 1e-4;
    s->background[0] = s->background[1] = s->background[2] = 0.0;
    s->cov2d_dilation = 0.3;
    s->alpha_clamp = 0.999;
}

const char* tk_last_error(void) { return g_err.c_str(); }
int32_t tk_abi_version(void) { return TK_ABI_VERSION; }

tk_status tk_create(int32_t device, tk_ctx** out) {
    return guarded([&] {
        if (!out) fail(TK_ERR_BAD_ARG, "null out");
        *out = nullptr;
        int count = 0;
        CK(cudaGetDeviceCount(&count));
        if (device < 0 || device >= count) fail(TK_ERR_BAD_ARG, "device index out of range");
        CK(cudaSetDevice(device));
        tk_ctx* c = new tk_ctx;
        c->device = device;
        cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
        // The HBM-bound feature chain (short dependent launches) gets the highest priority so its
        // blocks are scheduled as soon as the long fp64 geometry-backward grid frees SM slots.
        int prio_lo = 0, prio_hi = 0;
        cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
        // Side streams only with TK_OVERLAP=1: on B200 the fp64 geometry backward and the feature
        // kernels each fill the SMs' register files, so overlapping them measured no gain; the
        // default aliases every stream to the main one (per-kernel times stay unambiguous).
        const char* overlap = std::getenv("TK_OVERLAP");
        if (!(overlap && overlap[0] == '1')) {
            if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->s_feat, cudaStreamNonBlocking);
            if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->s_geo, cudaStreamNonBlocking);
            if (e == cudaSuccess) {  // alias the side streams to the main stream
                cudaStreamDestroy(c->s_feat);
                cudaStreamDestroy(c->s_geo);
                c->s_feat = c->s_geo = c->stream;
            }
        } else {
            if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&c->s_feat, cudaStreamNonBlocking, prio_hi);
            if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&c->s_geo, cudaStreamNonBlocking, prio_lo);
        }
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_main, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_feat, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_geo, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->s_in, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->s_out, cudaStreamNonBlocking);
        for (cudaEvent_t* ev : {&c->ev_cmp, &c->ev_in, &c->ev_out[0], &c->ev_out[1], &c->ev_out[2], &c->ev_out[3],
                                &c->ev_out[4]})
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
        if (e == cudaSuccess)
            e = cudaHostAlloc(reinterpret_cast<void**>(&c->h_twist), tk_ctx::kTwistSlots * 8 * sizeof(double),
                              cudaHostAllocMapped);
        if (e == cudaSuccess) e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->h_twist_dev), c->h_twist, 0);
        if (e == cudaSuccess) e = cudaHostAlloc(reinterpret_cast<void**>(&c->hvals), 4 * sizeof(double), cudaHostAllocMapped);
        if (e == cudaSuccess) e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->hvals_dev), c->hvals, 0);
        c->cur = c->stream;
        if (e == cudaSuccess) e = cudaHostAlloc(reinterpret_cast<void**>(&c->hscal), 16 * sizeof(int64_t), cudaHostAllocMapped);
        if (e == cudaSuccess) e = cudaMalloc(&c->dscal.p, 16 * sizeof(int64_t));
        if (e == cudaSuccess) {
            c->dscal.bytes = 16 * sizeof(int64_t);
            e = cudaMemset(c->dscal.p, 0, 16 * sizeof(int64_t));
        }
        if (e == cudaSuccess) e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->hscal_dev), c->hscal, 0);
        if (e != cudaSuccess) {
            delete c;
            fail(TK_ERR_CUDA, std::string("tk_create: ") + cudaGetErrorString(e));
        }
        *out = c;
    });
}

tk_status tk_destroy(tk_ctx* c) {
    if (!c) return TK_OK;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    if (c->s_feat) cudaStreamSynchronize(c->s_feat);
    if (c->s_geo) cudaStreamSynchronize(c->s_geo);
    if (c->s_in) cudaStreamSynchronize(c->s_in);
    if (c->s_out) cudaStreamSynchronize(c->s_out);
    DevBuf* all[] = {&c->mean, &c->log_scale, &c->rotation, &c->opacity_logit, &c->color, &c->feature, &c->pmx,
                     &c->pmy, &c->pixx, &c->pixy, &c->piyy, &c->pz, &c->pop, &c->rect, &c->valid, &c->ntiles,
                     &c->pos, &c->dkeys, &c->dvals, &c->dkeys_alt, &c->dvals_alt, &c->ntiles_sorted, &c->pair_off,
                     &c->tkeys, &c->tvals, &c->tkeys_alt, &c->tvals_alt, &c->tile_offsets, &c->padded_cnt,
                     &c->padded_start, &c->scratch, &c->scratch_feat, &c->dscal, &c->o_color, &c->o_depth, &c->o_alpha, &c->o_index,
                     &c->o_weight, &c->o_count, &c->o_contrib, &c->aux_t, &c->aux_n, &c->x_index, &c->x_weight,
                     &c->x_count, &c->f_out, &c->f_grad_in, &c->f_grad_out, &c->s_keys, &c->s_vals,
                     &c->s_keys_alt, &c->s_vals_alt, &c->s_wnorm, &c->s_seg, &c->g_color_in, &c->g_depth_in,
                     &c->mid, &c->twist, &c->twist_part, &c->twist_out, &c->gg_mean, &c->gg_ls, &c->gg_rot,
                     &c->gg_op, &c->gg_col, &c->l_count, &c->l_off, &c->l_src, &c->l_w, &c->gather_buf,
                     &c->wl, &c->wl_count};
    for (DevBuf* b : all) b->release();
    c->te.release();
    for (Keyframe& k : c->kfs) k.release();
    for (int g = 0; g < 5; ++g) {
        c->am[g].release();
        c->av[g].release();
    }
    DevBuf* mapping[] = {&c->fm, &c->fv, &c->stat_count, &c->stat_maxc, &c->ssim_rows, &c->ssim_win, &c->l_gc,
                         &c->l_gd, &c->l_partial, &c->l_values, &c->l_fscale, &c->l_signs, &c->q_feat,
                         &c->q_emb, &c->q_labels, &c->q_best, &c->q_acc, &c->q_nacc, &c->q_part,
                         &c->lp_items, &c->lp_longs, &c->lp_counters, &c->lp_partial, &c->row_ss};
    for (DevBuf* b : mapping) b->release();
    if (c->hvals) cudaFreeHost(c->hvals);
    if (c->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(c->comm);
    if (c->hscal) cudaFreeHost(c->hscal);
    if (c->stream) cudaStreamDestroy(c->stream);
    if (c->s_feat && c->s_feat != c->stream) cudaStreamDestroy(c->s_feat);
    if (c->s_geo && c->s_geo != c->stream) cudaStreamDestroy(c->s_geo);
    for (cudaEvent_t e : {c->ev_main, c->ev_feat, c->ev_geo, c->ev_cmp, c->ev_in, c->ev_out[0], c->ev_out[1],
                          c->ev_out[2], c->ev_out[3], c->ev_out[4]})
        if (e) cudaEventDestroy(e);
    if (c->h_twist) cudaFreeHost(c->h_twist);
    if (c->s_in) cudaStreamDestroy(c->s_in);
    if (c->s_out) cudaStreamDestroy(c->s_out);
    delete c;
    return TK_OK;
}

tk_status tk_synchronize(tk_ctx* c) {
    return guarded([&] {
        CK(cudaSetDevice(c->device));
        CK(cudaStreamSynchronize(c->s_feat));
        CK(cudaStreamSynchronize(c->s_geo));
        CK(cudaStreamSynchronize(c->stream));
        CK(cudaStreamSynchronize(c->s_in));
        CK(cudaStreamSynchronize(c->s_out));
        for (bool& b : c->out_pending) b = false;
        for (const auto& t : c->twist_pending) std::memcpy(t.first, c->h_twist + 8 * t.second, 6 * sizeof(double));
        c->twist_pending.clear();
    });
}

tk_status tk_join(tk_ctx* c) {
    return guarded([&] {
        CK(cudaSetDevice(c->device));
        on_main(c);
        // the copy streams too: the main stream then follows every asynchronous host copy
        CK(cudaEventRecord(c->ev_in, c->s_in));
        CK(cudaStreamWaitEvent(c->stream, c->ev_in, 0));
        CK(cudaEventRecord(c->ev_out[kOutMisc], c->s_out));
        CK(cudaStreamWaitEvent(c->stream, c->ev_out[kOutMisc], 0));
        main_done(c);
    });
}

void* tk_get_stream(tk_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }
int64_t tk_kernel_launches(tk_ctx* c) { return c ? c->launches : 0; }

tk_status tk_host_alloc(size_t bytes, void** out) {
    return guarded([&] { CK(cudaHostAlloc(out, std::max<size_t>(bytes, 1), cudaHostAllocDefault)); });
}
tk_status tk_host_free(void* p) {
    return guarded([&] {
        if (p) CK(cudaFreeHost(p));
    });
}

tk_status tk_scene_upload(tk_ctx* c, const tk_scene_view* s, int32_t mem) {
    return guarded([&] {
        if (!c || !s) fail(TK_ERR_BAD_ARG, "null argument");
        if (s->n < 0 || s->d < 0) fail(TK_ERR_BAD_ARG, "negative scene size");
        if (s->n > INT32_MAX - 1) fail(TK_ERR_BAD_ARG, "scene larger than 2^31-1 Gaussians");
        CK(cudaSetDevice(c->device));
        on_main(c);
        cudaStream_t st = c->cur;
        const int64_t n = s->n;
        if (!s->feature && c->has_features && (n != c->n || s->d != c->d))
            fail(TK_ERR_BAD_ARG, "feature == NULL requires unchanged n and d");
        copy_in(ensure<double>(c->mean, n * 3), s->mean, n * 3 * sizeof(double), mem, c);
        copy_in(ensure<double>(c->log_scale, n * 3), s->log_scale, n * 3 * sizeof(double), mem, c);
        copy_in(ensure<double>(c->rotation, n * 4), s->rotation, n * 4 * sizeof(double), mem, c);
        copy_in(ensure<double>(c->opacity_logit, n), s->opacity_logit, n * sizeof(double), mem, c);
        copy_in(ensure<double>(c->color, n * 3), s->color, n * 3 * sizeof(double), mem, c);
        if (s->feature) {
            copy_in(ensure<float>(c->feature, n * std::max(s->d, 1)), s->feature,
                    static_cast<size_t>(n) * s->d * sizeof(float), mem, c);
            c->has_features = true;
        }
        c->n = n;
        c->d = s->d;
        c->generation = s->generation;
        c->scene_version += 1;
        c->has_scene = true;
        c->prepared = false;
        c->aux_valid = false;
        main_done(c);
    });
}

tk_status tk_device_view_get(tk_ctx* c, tk_device_view* v) {
    return guarded([&] {
        std::memset(v, 0, sizeof(*v));
        v->color = ptr<double>(c->o_color);
        v->depth = ptr<double>(c->o_depth);
        v->alpha = ptr<double>(c->o_alpha);
        v->topk_index = ptr<int32_t>(c->o_index);
        v->topk_weight = ptr<double>(c->o_weight);
        v->topk_count = ptr<uint8_t>(c->o_count);
        v->contributions = ptr<double>(c->o_contrib);
        v->feature_out = ptr<float>(c->f_out);
        v->feature_grad = ptr<float>(c->f_grad_out);
        const int64_t P = static_cast<int64_t>(c->rec_w) * c->rec_h;
        v->grad_feature_in = ensure<float>(c->f_grad_in, std::max<int64_t>(P, 1) * std::max(c->d, 1));
        v->mean = ptr<double>(c->mean);
        v->feature = ptr<float>(c->feature);
        v->n = c->n;
        v->d = c->d;
        v->width = c->rec_w;
        v->height = c->rec_h;
        v->k = c->rec_k;
    });
}

tk_status tk_prepare_scene(tk_ctx* c, const tk_pose* pose, const tk_camera* cam, const tk_settings* s,
                           int64_t* n_entries, int64_t* n_tile_entries, int32_t* tiles_x, int32_t* tiles_y) {
    return guarded([&] {
        check_frame(cam, s);
        CK(cudaSetDevice(c->device));
        on_main(c);
        prepare(c, pose, cam, s);
        if (n_entries) *n_entries = c->n_vis;
        if (n_tile_entries) *n_tile_entries = c->n_pairs;
        if (tiles_x) *tiles_x = c->tiles_x;
        if (tiles_y) *tiles_y = c->tiles_y;
        main_done(c);
    });
}

tk_status tk_prepared_export(tk_ctx* c, double* entries7, int32_t* src, int32_t* tile_offsets,
                             int32_t* tile_entries_out) {
    return guarded([&] {
        if (!c->prepared) fail(TK_ERR_STATE, "no prepared scene");
        CK(cudaSetDevice(c->device));
        on_main(c);
        cudaStream_t st = c->cur;
        const int64_t nv = c->n_vis;
        DevBuf e7, s7;
        double* de = ensure<double>(e7, nv * 7);
        int32_t* ds = ensure<int32_t>(s7, nv);
        tk::launch_export_entries(c->order, nv, ptr<double>(c->pmx), ptr<double>(c->pmy), ptr<double>(c->pixx),
                                  ptr<double>(c->pixy), ptr<double>(c->piyy), ptr<double>(c->pz),
                                  ptr<double>(c->pop), de, ds, st);
        CK_LAUNCH(c);
        copy_out(entries7, de, nv * 7 * sizeof(double), TK_HOST, c);
        copy_out(src, ds, nv * sizeof(int32_t), TK_HOST, c);
        copy_out(tile_offsets, ptr<int32_t>(c->tile_offsets),
                 (static_cast<int64_t>(c->tiles_x) * c->tiles_y + 1) * sizeof(int32_t), TK_HOST, c);
        copy_out(tile_entries_out, c->tile_vals_sorted, c->n_pairs * sizeof(int32_t), TK_HOST, c);
        sync(c);
        e7.release();
        s7.release();
        main_done(c);
    });
}

tk_status tk_render_geometric(tk_ctx* c, const tk_pose* pose, const tk_camera* cam, const tk_settings* s,
                              tk_geom_out* out) {
    return guarded([&] {
        check_frame(cam, s);
        CK(cudaSetDevice(c->device));
        on_main(c);
        prepare(c, pose, cam, s);
        forward(c, cam, s, true);
        c->aux_valid = true;
        c->aux_key = make_fwd_key(c->prep_key, s);
        if (out) {
            const int64_t P = static_cast<int64_t>(cam->width) * cam->height;
            const int64_t k = c->rec_k;
            cudaStream_t st = c->cur;
            copy_out(out->color, c->o_color.p, P * 3 * sizeof(double), out->mem, c, kOutRec);
            copy_out(out->depth, c->o_depth.p, P * sizeof(double), out->mem, c, kOutRec);
            copy_out(out->alpha, c->o_alpha.p, P * sizeof(double), out->mem, c, kOutRec);
            copy_out(out->topk_index, c->o_index.p, P * k * sizeof(int32_t), out->mem, c, kOutRec);
            copy_out(out->topk_weight, c->o_weight.p, P * k * sizeof(double), out->mem, c, kOutRec);
            copy_out(out->topk_count, c->o_count.p, P, out->mem, c, kOutRec);
            copy_out(out->contributions, c->o_contrib.p, c->n * sizeof(double), out->mem, c, kOutRec);
            out->generation = c->generation;
            out->map_size = c->n;
            if (out->mem == TK_HOST) sync(c);
        }
        main_done(c);
    });
}

tk_status tk_render_feature(tk_ctx* c, const tk_topk_view* topk, float* out, int32_t out_mem) {
    return guarded([&] {
        CK(cudaSetDevice(c->device));
        on_side(c, true);
        require_features(c);
        const Records r = resolve_records(c, topk, "render_feature");
        if (r.k > tk::kMaxTopK) fail(TK_ERR_BAD_ARG, "TopKGrid k exceeds 32");
        const int64_t P = static_cast<int64_t>(r.w) * r.h;
        wait_out(c, kOutF);
        float* dst = (out && out_mem == TK_DEVICE) ? out : ensure<float>(c->f_out, P * std::max(c->d, 1));
        tk::GatherParams gp{P, r.k, r.index, r.weight, r.count, ptr<float>(c->feature), c->d, dst, r.w, r.h};
        {
            PhaseScope phase(c, TK_PHASE_GATHER);
            tk::launch_feature_gather(gp, c->cur);
        }
        c->launches += P > 0;
        CK_LAUNCH(c);
        c->fout_pixels = P;
        if (out && out_mem != TK_DEVICE) {
            copy_out(out, dst, static_cast<size_t>(P) * c->d * sizeof(float), out_mem, c, kOutF);
            if (out_mem == TK_HOST) sync(c);
        }
        side_done(c, true);
    });
}

tk_status tk_backward_feature(tk_ctx* c, const tk_topk_view* topk, const float* grad, int32_t grad_mem, float* out,
                              int32_t out_mem) {
    return guarded([&] {
        CK(cudaSetDevice(c->device));
        on_side(c, true);
        require_features(c);
        const Records r = resolve_records(c, topk, "backward_feature");
        if (r.k > tk::kMaxTopK) fail(TK_ERR_BAD_ARG, "TopKGrid k exceeds 32");
        cudaStream_t st = c->cur;
        const int64_t P = static_cast<int64_t>(r.w) * r.h;
        const int64_t slots = P * r.k;
        const int64_t n = c->n;
        const float* g = grad;
        if (!grad) {
            if (grad_mem != TK_DEVICE) fail(TK_ERR_BAD_ARG, "null grad_feature");
            g = ensure<float>(c->f_grad_in, P * std::max(c->d, 1));
        } else if (grad_mem != TK_DEVICE) {
            float* dg = ensure<float>(c->f_grad_in, P * std::max(c->d, 1));
            copy_in(dg, grad, static_cast<size_t>(P) * c->d * sizeof(float), grad_mem, c);
            g = dg;
        }
        const SlotIndex si = build_slot_index(c, r);
        wait_out(c, kOutDF);
        float* dst = (out && out_mem == TK_DEVICE) ? out : ensure<float>(c->f_grad_out, n * std::max(c->d, 1));
        tk::FeatBwdParams fp{n, r.k, c->d, si.seg, si.slots, si.wnorm, g, dst};
        {
            PhaseScope phase(c, TK_PHASE_FBWD);
            tk::launch_feature_bwd(fp, si.plan, st);
        }
        c->launches += n > 0 ? 3 : 0;
        CK_LAUNCH(c);
        if (out && out_mem != TK_DEVICE) {
            copy_out(out, dst, static_cast<size_t>(n) * c->d * sizeof(float), out_mem, c, kOutDF);
            if (out_mem == TK_HOST) sync(c);
        }
        side_done(c, true);
    });
}

tk_status tk_render_feature_full_blend(tk_ctx* c, const tk_pose* pose, const tk_camera* cam, const tk_settings* s,
                                       float* out, int32_t out_mem) {
    return guarded([&] {
        check_frame(cam, s);
        CK(cudaSetDevice(c->device));
        on_main(c);
        require_features(c);
        prepare(c, pose, cam, s);
        cudaStream_t st = c->cur;
        const tk::Frame f = make_frame(c, cam, s);
        const int64_t P = static_cast<int64_t>(f.width) * f.height;
        tk::GeomFwdParams gp{};
        gp.f = f;
        gp.te = tile_entries(c);
        gp.tile_offsets = ptr<int32_t>(c->tile_offsets);
        gp.padded_start = ptr<int32_t>(c->padded_start);
            gp.list_count = ensure<int32_t>(c->l_count, P + 1);
        int32_t* off = ensure<int32_t>(c->l_off, P + 1);
        CK(cudaMemsetAsync(gp.list_count + P, 0, sizeof(int32_t), st));
        const int nblk = tk::geom_blocks(f);
        tk::launch_geom_fwd(tk::kGeomCount, gp, nblk, st);
        ensure_scratch(c, P + 1);
        int64_t* dscal = ensure<int64_t>(c->dscal, 16);
        tk::scan_exclusive(gp.list_count, off, P + 1, dscal + 6, c->scratch.p, st, &c->launches);
        tk::copy_words_to_mapped(c->hscal_dev + 6, dscal + 6, 1, st);
        sync(c);
        const int64_t total = c->hscal[6];
        if (total > INT32_MAX) fail(TK_ERR_BAD_ARG, "contributor lists exceed 2^31 entries");
        gp.list_offsets = off;
        gp.list_src = ensure<int32_t>(c->l_src, total);
        gp.list_w = ensure<double>(c->l_w, total);
        tk::launch_geom_fwd(tk::kGeomList, gp, nblk, st);
        float* dst = (out && out_mem == TK_DEVICE) ? out : ensure<float>(c->f_out, P * std::max(c->d, 1));
        tk::ListGatherParams lp{P, off, gp.list_src, gp.list_w, ptr<float>(c->feature), c->d, dst};
        tk::launch_list_gather(lp, st);
        c->launches += 3;
        CK_LAUNCH(c);
        if (out && out_mem == TK_HOST) {
            copy_out(out, dst, static_cast<size_t>(P) * c->d * sizeof(float), TK_HOST, c);
            sync(c);
        }
        main_done(c);
    });
}

tk_status tk_backward_geometric(tk_ctx* c, const tk_pose* pose, const tk_camera* cam, const tk_settings* s,
                                const double* grad_color, const double* grad_depth, int32_t grad_mem,
                                tk_geom_grads* out) {
    return guarded([&] {
        check_frame(cam, s);
        if (!grad_color) fail(TK_ERR_BAD_ARG, "null grad_color");
        CK(cudaSetDevice(c->device));
        // backward.cpp:75 recomputes prepare_scene; it is reused when the forward of this context
        // ran on the same inputs, and only then does the call stay off the main stream.
        const FwdKey fk = make_fwd_key(make_prep_key(c, pose, cam, s), s);
        if (!(c->prepared && c->aux_valid && c->aux_key == fk)) {
            on_main(c);
            prepare(c, pose, cam, s);
            forward(c, cam, s, false);
            c->aux_valid = true;
            c->aux_key = fk;
            main_done(c);
        }
        on_side(c, false);  // the sweep overlaps the feature path (s_feat)
        cudaStream_t st = c->cur;
        const tk::Frame f = make_frame(c, cam, s);
        const int64_t P = static_cast<int64_t>(f.width) * f.height;
        const int64_t n = c->n;
        const double* gc = grad_color;
        const double* gd = grad_depth;
        if (grad_mem != TK_DEVICE) {
            double* dgc = ensure<double>(c->g_color_in, P * 3);
            copy_in(dgc, grad_color, P * 3 * sizeof(double), grad_mem, c);
            gc = dgc;
            if (grad_depth) {
                double* dgd = ensure<double>(c->g_depth_in, P);
                copy_in(dgd, grad_depth, P * sizeof(double), grad_mem, c);
                gd = dgd;
            }
        }
        double* mid = geom_sweep(c, f, gc, gd);
        const bool dev_out = out && out->mem == TK_DEVICE;
        wait_out(c, kOutGG);
        tk::ChainParams cp = chain_params(c, pose, cam, s, mid);
        cp.g_mean = dev_out && out->mean ? out->mean : ensure<double>(c->gg_mean, n * 3);
        cp.g_log_scale = dev_out && out->log_scale ? out->log_scale : ensure<double>(c->gg_ls, n * 3);
        cp.g_rotation = dev_out && out->rotation ? out->rotation : ensure<double>(c->gg_rot, n * 4);
        cp.g_opacity_logit = dev_out && out->opacity_logit ? out->opacity_logit : ensure<double>(c->gg_op, n);
        cp.g_color = dev_out && out->color ? out->color : ensure<double>(c->gg_col, n * 3);
        cp.twist = ensure<double>(c->twist, (n + 127) / 128 * 6);
        double* tpart = ensure<double>(c->twist_part, 148 * 6);
        double* tout = ensure<double>(c->twist_out, 6);
        {
            PhaseScope phase(c, TK_PHASE_CHAIN);
            tk::launch_chain(cp, st);
            tk::launch_twist_reduce(cp.twist, n, tpart, tout, st);
        }
        c->launches += 2;
        CK_LAUNCH(c);
        if (out) {
            if (out->mem != TK_DEVICE) {
                copy_out(out->mean, cp.g_mean, n * 3 * sizeof(double), out->mem, c, kOutGG);
                copy_out(out->log_scale, cp.g_log_scale, n * 3 * sizeof(double), out->mem, c, kOutGG);
                copy_out(out->rotation, cp.g_rotation, n * 4 * sizeof(double), out->mem, c, kOutGG);
                copy_out(out->opacity_logit, cp.g_opacity_logit, n * sizeof(double), out->mem, c, kOutGG);
                copy_out(out->color, cp.g_color, n * 3 * sizeof(double), out->mem, c, kOutGG);
            }
            if (out->mem == TK_HOST_ASYNC) {  // the twist lands in the struct at tk_synchronize
                if (static_cast<int>(c->twist_pending.size()) == tk_ctx::kTwistSlots) {  // ring full: drain it
                    sync(c);
                    for (const auto& t : c->twist_pending)
                        std::memcpy(t.first, c->h_twist + 8 * t.second, 6 * sizeof(double));
                    c->twist_pending.clear();
                }
                const int slot = c->twist_next;
                c->twist_next = (c->twist_next + 1) % tk_ctx::kTwistSlots;
                // 48 bytes stored by a kernel: not queued behind the large copies of s_out
                tk::copy_words_to_mapped(c->h_twist_dev + 8 * slot, tout, 6, c->cur);
                c->twist_pending.emplace_back(out->pose_twist, slot);
            } else {
                copy_out(out->pose_twist, tout, 6 * sizeof(double), TK_HOST, c);
                sync(c);
            }
        }
        side_done(c, false);
    });
}

tk_status tk_fp64_rate(tk_ctx* c, double* fma_per_s) {
    return guarded([&] {
        CK(cudaSetDevice(c->device));
        CK(cudaStreamSynchronize(c->stream));
        *fma_per_s = tk::measure_fp64_fma_rate(c->stream);
        CK_LAUNCH(c);
    });
}

tk_status tk_pair_count(tk_ctx* c, int64_t* pairs, int32_t reset) {
    return guarded([&] {
        CK(cudaSetDevice(c->device));
        int64_t* dscal = ensure<int64_t>(c->dscal, 16);
        CK(cudaStreamSynchronize(c->stream));
        tk::copy_words_to_mapped(c->hscal_dev + 13, dscal + 13, 1, c->stream);
        CK(cudaStreamSynchronize(c->stream));
        if (pairs) *pairs = c->hscal[13];
        if (reset) CK(cudaMemsetAsync(dscal + 13, 0, sizeof(int64_t), c->stream));
    });
}

tk_status tk_invalidate(tk_ctx* c) {
    return guarded([&] {
        c->prepared = false;
        c->aux_valid = false;
    });
}

tk_status tk_profile_enable(tk_ctx* c, int32_t on) {
    return guarded([&] { c->prof.on = on != 0; });
}

tk_status tk_profile_read(tk_ctx* c, double* ms, int64_t* counts, int32_t reset) {
    return guarded([&] {
        CK(cudaSetDevice(c->device));
        c->prof.drain();
        for (int i = 0; i < TK_NUM_PHASES; ++i) {
            if (ms) ms[i] = c->prof.ms[i];
            if (counts) counts[i] = c->prof.cnt[i];
            if (reset) {
                c->prof.ms[i] = 0.0;
                c->prof.cnt[i] = 0;
            }
        }
    });
}

tk_status tk_comm_unique_id(uint8_t id[128]) {
    return guarded([&] {
        if (!g_nccl.load()) fail(TK_ERR_NCCL, "libnccl.so.2 not found");
        ncclUniqueId uid;
        NK(g_nccl.GetUniqueId(&uid));
        static_assert(sizeof(uid) == 128, "ncclUniqueId size");
        std::memcpy(id, &uid, 128);
    });
}

tk_status tk_comm_init(tk_ctx* c, const uint8_t id[128], int32_t nranks, int32_t rank, int32_t d_total) {
    return guarded([&] {
        if (!g_nccl.load()) fail(TK_ERR_NCCL, "libnccl.so.2 not found");
        if (nranks < 1 || rank < 0 || rank >= nranks) fail(TK_ERR_BAD_ARG, "bad rank / nranks");
        CK(cudaSetDevice(c->device));
        ncclUniqueId uid;
        std::memcpy(&uid, id, 128);
        NK(g_nccl.CommInitRank(&c->comm, nranks, uid, rank));
        c->nranks = nranks;
        c->rank = rank;
        c->d_total = d_total;
    });
}

tk_status tk_allgather_feature(tk_ctx* c, float* out, int32_t out_mem) {
    return guarded([&] {
        if (!c->comm) fail(TK_ERR_STATE, "tk_comm_init not called");
        if (c->d * c->nranks != c->d_total) fail(TK_ERR_BAD_ARG, "d_total must equal nranks * d_shard");
        CK(cudaSetDevice(c->device));
        on_side(c, true);
        cudaStream_t st = c->cur;
        const int64_t P = c->fout_pixels;
        const size_t slice = static_cast<size_t>(P) * c->d;
        float* gath = ensure<float>(c->gather_buf, slice * c->nranks);
        NK(g_nccl.AllGather(c->f_out.p, gath, slice, ncclFloat32, c->comm, st));
        float* dst = out && out_mem == TK_DEVICE ? out : nullptr;
        DevBuf tmp;
        if (!dst) dst = ensure<float>(tmp, slice * c->nranks);
        tk::launch_interleave(gath, P, c->d, c->nranks, dst, st);
        c->launches += 1;
        CK_LAUNCH(c);
        if (out && out_mem == TK_HOST) copy_out(out, dst, slice * c->nranks * sizeof(float), TK_HOST, c);
        sync(c);
        tmp.release();
        side_done(c, true);
    });
}

tk_status tk_allreduce_sum_f64(tk_ctx* c, double* values, int32_t count) {
    return guarded([&] {
        if (!c->comm) fail(TK_ERR_STATE, "tk_comm_init not called");
        CK(cudaSetDevice(c->device));
        on_main(c);
        DevBuf tmp;
        double* d = ensure<double>(tmp, count);
        copy_in(d, values, count * sizeof(double), TK_HOST, c);
        NK(g_nccl.AllReduce(d, d, count, ncclFloat64, ncclSum, c->comm, c->cur));
        copy_out(values, d, count * sizeof(double), TK_HOST, c);
        sync(c);
        tmp.release();
        main_done(c);
    });
}

// ------------------------------------------------------------------ mapping iteration
void tk_default_mapper_config(tk_mapper_config* cfg) {
    cfg->lambda_geo = 1.0;  // losses.hpp:9-21
    cfg->lambda_feat = 1.0;
    cfg->lambda1 = 0.2;
    cfg->lambda2 = 1.0;
    cfg->color_secondary = 0;
    cfg->feature_update_period = 5;  // mapper.hpp:16
    cfg->l1_deadband = 0.0;
    cfg->lr_mean = 2e-3;  // optimizer.hpp:15-22
    cfg->lr_log_scale = 5e-3;
    cfg->lr_rotation = 1e-3;
    cfg->lr_opacity = 5e-2;
    cfg->lr_color = 2e-2;
    cfg->lr_feature = 1e-2;
    cfg->beta1 = 0.9;  // optimizer.hpp:9-13
    cfg->beta2 = 0.999;
    cfg->eps = 1e-8;
    cfg->min_log_scale = -10.0;  // mapper.hpp:31-32
    cfg->max_log_scale = 1.0;
}

tk_status tk_keyframe_set(tk_ctx* c, int32_t slot, const tk_pose* pose, const tk_frame_view* fr) {
    return guarded([&] {
        if (!c || !pose || !fr) fail(TK_ERR_BAD_ARG, "null argument");
        if (slot < 0 || slot > (1 << 20)) fail(TK_ERR_BAD_ARG, "keyframe slot out of range");
        if (fr->width <= 0 || fr->height <= 0 || fr->d < 0) fail(TK_ERR_BAD_ARG, "bad frame shape");
        if (!fr->color || !fr->depth) fail(TK_ERR_BAD_ARG, "frame needs color and depth");
        if (fr->d > 0 && !fr->feature) fail(TK_ERR_BAD_ARG, "frame feature is NULL but d > 0");
        CK(cudaSetDevice(c->device));
        on_main(c);
        if (static_cast<size_t>(slot) >= c->kfs.size()) c->kfs.resize(slot + 1);
        Keyframe& k = c->kfs[slot];
        k.pose = *pose;
        k.w = fr->width;
        k.h = fr->height;
        k.d = fr->d;
        k.has_feature = fr->d > 0;
        const int64_t P = static_cast<int64_t>(k.w) * k.h;
        float* col = ensure<float>(k.color, P * 3);
        float* dep = ensure<float>(k.depth, P);
        copy_in(col, fr->color, P * 3 * sizeof(float), fr->mem, c);
        copy_in(dep, fr->depth, P * sizeof(float), fr->mem, c);
        float* feat = nullptr;
        if (k.has_feature) {
            feat = ensure<float>(k.feature, P * k.d);
            copy_in(feat, fr->feature, static_cast<size_t>(P) * k.d * sizeof(float), fr->mem, c);
        }
        uint8_t* valid = ensure<uint8_t>(k.valid, P);
        int64_t* dscal = ensure<int64_t>(c->dscal, 16);
        tk::launch_gt_valid(feat, P, k.d, valid, dscal + 9, dep, c->cur);
        c->launches += 1;
        CK_LAUNCH(c);
        if (c->comm)  // D-sharded: a pixel's keyframe row is valid if any shard's channels are non-zero
            NK(g_nccl.AllReduce(valid, valid, static_cast<size_t>(P), ncclUint8, ncclMax, c->comm, c->cur));
        tk::copy_words_to_mapped(c->hscal_dev + 9, dscal + 9, 1, c->cur);
        sync(c);
        k.depth_n = c->hscal[9];
        main_done(c);
    });
}

tk_status tk_optimizer_reset(tk_ctx* c, int32_t reset_stats) {
    return guarded([&] {
        if (!c) fail(TK_ERR_BAD_ARG, "null context");
        if (!c->has_scene) fail(TK_ERR_STATE, "no scene uploaded (tk_scene_upload)");
        CK(cudaSetDevice(c->device));
        on_main(c);
        const int64_t n = c->n;
        const int dims[5] = {3, 3, 4, 1, 3};
        for (int g = 0; g < 5; ++g) {
            CK(cudaMemsetAsync(ensure<double>(c->am[g], n * dims[g]), 0, std::max<int64_t>(n, 1) * dims[g] * 8, c->cur));
            CK(cudaMemsetAsync(ensure<double>(c->av[g], n * dims[g]), 0, std::max<int64_t>(n, 1) * dims[g] * 8, c->cur));
        }
        const int64_t nd = n * std::max(c->d, 1);
        CK(cudaMemsetAsync(ensure<float>(c->fm, nd), 0, std::max<int64_t>(nd, 1) * 4, c->cur));
        CK(cudaMemsetAsync(ensure<float>(c->fv, nd), 0, std::max<int64_t>(nd, 1) * 4, c->cur));
        if (reset_stats || c->stat_n != n) {
            CK(cudaMemsetAsync(ensure<int32_t>(c->stat_count, n), 0, std::max<int64_t>(n, 1) * 4, c->cur));
            CK(cudaMemsetAsync(ensure<double>(c->stat_maxc, n), 0, std::max<int64_t>(n, 1) * 8, c->cur));
            c->stat_n = n;
        }
        c->step_geo = c->step_feat = 0;
        c->opt_ready = true;
        c->opt_n = n;
        c->opt_d = c->d;
        main_done(c);
    });
}

tk_status tk_optimize_step(tk_ctx* c, const tk_mapper_config* cfg, const tk_camera* cam, const tk_settings* s,
                           int32_t slot, int64_t iteration, double* values_out, int32_t* feature_step_out) {
    return guarded([&] {
        check_frame(cam, s);
        if (!cfg) fail(TK_ERR_BAD_ARG, "null mapper config");
        if (slot < 0 || static_cast<size_t>(slot) >= c->kfs.size() || c->kfs[slot].w == 0)
            fail(TK_ERR_BAD_ARG, "optimize_step: no keyframe in that slot");
        if (cfg->feature_update_period <= 0) fail(TK_ERR_BAD_ARG, "feature_update_period must be positive");
        if (!c->has_scene) fail(TK_ERR_STATE, "no scene uploaded (tk_scene_upload)");
        if (!c->opt_ready || c->opt_n != c->n || c->opt_d != c->d || c->stat_n != c->n)
            fail(TK_ERR_STATE, "optimizer state does not match the scene (tk_optimizer_reset)");
        const Keyframe& kf = c->kfs[slot];
        if (kf.w != cam->width || kf.h != cam->height)
            fail(TK_ERR_BAD_ARG, "compute_losses: render/frame shape mismatch");
        const bool feature_step = (iteration % cfg->feature_update_period) == 0;  // mapper.cpp:171
        const bool sharded = c->comm != nullptr;  // D-sharded mapping (features: this rank's slice)
        const bool use_ssim = cfg->lambda1 != 0.0 && cfg->color_secondary == 0;
        if (use_ssim && (cam->width < tk::kSsimWin || cam->height < tk::kSsimWin))
            fail(TK_ERR_BAD_ARG, "ssim: image smaller than the 11x11 window");
        if (feature_step) {
            if (c->d <= 0 || !c->has_features)
                fail(TK_ERR_BAD_ARG, "compute_losses: feature loss requested but render has no feature image");
            if (kf.d != c->d) fail(TK_ERR_BAD_ARG, "compute_losses: feature shape mismatch");
        }
        CK(cudaSetDevice(c->device));
        on_main(c);
        cudaStream_t st = c->cur;
        // render_geometric on the keyframe pose (mapper.cpp:173)
        prepare(c, &kf.pose, cam, s);
        forward(c, cam, s, true);
        const tk::Frame f = make_frame(c, cam, s);
        const int64_t P = static_cast<int64_t>(f.width) * f.height;
        const int64_t n = c->n;
        const int d = c->d;
        double* gc = ensure<double>(c->l_gc, P * 3);
        double* gd = ensure<double>(c->l_gd, P);
        double* partial = ensure<double>(c->l_partial, tk::kLossBlocks * tk::kLossSlots);
        double* values = ensure<double>(c->l_values, 4);
        float* fscale = ensure<float>(c->l_fscale, 1);
        const int wpp = (d + 15) / 16;
        uint32_t* signs = feature_step ? ensure<uint32_t>(c->l_signs, P * std::max(wpp, 1)) : nullptr;
        {
            PhaseScope phase(c, TK_PHASE_LOSS);
            CK(cudaMemsetAsync(partial, 0, tk::kLossBlocks * tk::kLossSlots * sizeof(double), st));
            tk::launch_topk_stats(ptr<int32_t>(c->o_index), ptr<uint8_t>(c->o_count), P, f.k,
                                  ptr<int32_t>(c->stat_count), st);
            c->launches += 1;
            // compute_losses (mapper.cpp:176, losses.cpp:22-133)
            tk::ColorLossParams lp{};
            lp.w = f.width;
            lp.h = f.height;
            lp.color = ptr<double>(c->o_color);
            lp.depth = ptr<double>(c->o_depth);
            lp.gt_color = ptr<float>(kf.color);
            lp.gt_depth = ptr<float>(kf.depth);
            lp.lambda_geo = cfg->lambda_geo;
            lp.lambda1 = cfg->lambda1;
            lp.lambda2 = cfg->lambda2;
            lp.deadband = cfg->l1_deadband;
            lp.use_ssim = use_ssim ? 1 : 0;
            lp.use_depth = (kf.depth_n > 0 && cfg->lambda2 != 0.0) ? 1 : 0;
            lp.inv_color_n = 1.0 / (static_cast<double>(f.width) * f.height * 3.0);
            lp.inv_depth_n = kf.depth_n > 0 ? 1.0 / static_cast<double>(kf.depth_n) : 0.0;
            {
                const int ow = f.width - tk::kSsimWin + 1, oh = f.height - tk::kSsimWin + 1;
                const size_t count = use_ssim ? static_cast<size_t>(ow) * oh * 3 : 1;  // ssim.cpp:119-123
                lp.inv_count = 1.0 / static_cast<double>(count);
                double sum = 0.0;  // gaussian_kernel(), ssim.cpp:18-28
                for (int i = 0; i < tk::kSsimWin; ++i) {
                    const double dd = i - tk::kSsimWin / 2;
                    lp.kern[i] = std::exp(-0.5 * dd * dd / (1.5 * 1.5));
                    sum += lp.kern[i];
                }
                for (double& v : lp.kern) v /= sum;
                if (use_ssim) {
                    lp.win = ensure<double>(c->ssim_win, 15LL * oh * ow);
                }
            }
            lp.grad_color = gc;
            lp.grad_depth = gd;
            lp.partial = partial;
            tk::launch_color_loss(lp, st, &c->launches);
            if (feature_step) {
                tk::FeatLossParams fl{};
                fl.width = f.width;
                fl.height = f.height;
                fl.k = f.k;
                fl.d = d;
                fl.index = ptr<int32_t>(c->o_index);
                fl.weight = ptr<double>(c->o_weight);
                fl.count = ptr<uint8_t>(c->o_count);
                fl.feat = ptr<float>(c->feature);
                fl.gt = ptr<float>(kf.feature);
                fl.gt_valid = ptr<uint8_t>(kf.valid);
                fl.signs = signs;
                fl.partial = partial;
                tk::launch_feature_loss(fl, st);
                c->launches += 1;
            }
            if (sharded)  // feature partials differ per shard; colour / depth rows are replicas
                NK(g_nccl.AllReduce(partial, partial, tk::kLossBlocks * tk::kLossSlots, ncclFloat64, ncclSum, c->comm,
                                    st));
            tk::FinalizeParams fp{};
            fp.partial = partial;
            fp.nparts = tk::kLossBlocks;
            fp.replicas = sharded ? static_cast<double>(c->nranks) : 1.0;
            fp.lambda_geo = cfg->lambda_geo;
            fp.lambda_feat = cfg->lambda_feat;
            fp.lambda1 = cfg->lambda1;
            fp.lambda2 = cfg->lambda2;
            fp.use_ssim = lp.use_ssim;
            fp.secondary_l1 = (cfg->lambda1 != 0.0 && cfg->color_secondary != 0) ? 1 : 0;
            fp.use_depth = lp.use_depth;
            fp.feature_step = feature_step ? 1 : 0;
            fp.d = sharded ? c->d_total : d;  // losses.cpp:106: mean over every channel
            fp.inv_color_n = lp.inv_color_n;
            fp.inv_depth_n = lp.inv_depth_n;
            fp.inv_count = lp.inv_count;
            fp.values = values;
            fp.feat_scale = fscale;
            tk::launch_loss_finalize(fp, st);
            c->launches += 1;
            CK_LAUNCH(c);
        }
        tk::copy_words_to_mapped(c->hvals_dev, values, 3, st);
        c->has_values = true;
        // backward_geometric (mapper.cpp:179-180) on this forward
        double* mid = geom_sweep(c, f, gc, gd);
        if (sharded)  // replicas stay bit-identical: one all-reduced geometry gradient on every shard
            NK(g_nccl.AllReduce(mid, mid, static_cast<size_t>(n) * 10, ncclFloat64, ncclSum, c->comm, st));
        {
            PhaseScope phase(c, TK_PHASE_ADAM);
            // geometry groups (mapper.cpp:183-236): five adam_step calls, one step counter each
            c->step_geo += 1;
            tk::GeoAdamParams ga{};
            ga.mean = ptr<double>(c->mean);
            ga.log_scale = ptr<double>(c->log_scale);
            ga.rotation = ptr<double>(c->rotation);
            ga.opacity_logit = ptr<double>(c->opacity_logit);
            ga.color = ptr<double>(c->color);
            for (int g = 0; g < 5; ++g) {
                ga.m[g] = ptr<double>(c->am[g]);
                ga.v[g] = ptr<double>(c->av[g]);
            }
            ga.lr[0] = cfg->lr_mean;
            ga.lr[1] = cfg->lr_log_scale;
            ga.lr[2] = cfg->lr_rotation;
            ga.lr[3] = cfg->lr_opacity;
            ga.lr[4] = cfg->lr_color;
            ga.beta1 = cfg->beta1;
            ga.beta2 = cfg->beta2;
            ga.eps = cfg->eps;
            ga.bc1 = 1.0 - std::pow(cfg->beta1, static_cast<double>(c->step_geo));  // optimizer.cpp:52-53
            ga.bc2 = 1.0 - std::pow(cfg->beta2, static_cast<double>(c->step_geo));
            ga.min_log_scale = cfg->min_log_scale;
            ga.max_log_scale = cfg->max_log_scale;
            ga.contrib = ptr<unsigned long long>(c->o_contrib);
            ga.max_contrib = ptr<double>(c->stat_maxc);
            tk::ChainParams cp = chain_params(c, &kf.pose, cam, s, mid);
            cp.mid_scale = sharded ? 1.0 / c->nranks : 1.0;
            cp.g_mean = ensure<double>(c->gg_mean, n * 3);
            cp.g_log_scale = ensure<double>(c->gg_ls, n * 3);
            cp.g_rotation = ensure<double>(c->gg_rot, n * 4);
            cp.g_opacity_logit = ensure<double>(c->gg_op, n);
            cp.g_color = ensure<double>(c->gg_col, n * 3);
            cp.twist = nullptr;
            tk::launch_chain(cp, st);
            ga.g[0] = cp.g_mean;
            ga.g[1] = cp.g_log_scale;
            ga.g[2] = cp.g_rotation;
            ga.g[3] = cp.g_opacity_logit;
            ga.g[4] = cp.g_color;
            tk::launch_geo_adam(ga, n, st);
            c->launches += n > 0 ? 2 : 0;
            CK_LAUNCH(c);
            if (feature_step && d > 0) {  // mapper.cpp:239-252
                c->step_feat += 1;
                Records r;
                r.w = f.width;
                r.h = f.height;
                r.k = f.k;
                r.index = ptr<int32_t>(c->o_index);
                r.weight = ptr<double>(c->o_weight);
                r.count = ptr<uint8_t>(c->o_count);
                const SlotIndex si = build_slot_index(c, r);
                tk::FeatAdamParams fa{};
                fa.n = n;
                fa.k = f.k;
                fa.d = d;
                fa.seg = si.seg;
                fa.slots = si.slots;
                fa.wnorm = si.wnorm;
                fa.signs = signs;
                fa.scale = fscale;
                fa.feat = ptr<float>(c->feature);
                fa.m = ptr<float>(c->fm);
                fa.v = ptr<float>(c->fv);
                fa.lr = static_cast<float>(cfg->lr_feature);
                fa.beta1 = static_cast<float>(cfg->beta1);
                fa.beta2 = static_cast<float>(cfg->beta2);
                fa.eps = static_cast<float>(cfg->eps);
                fa.one_m_beta1 = static_cast<float>(1.0 - cfg->beta1);
                fa.one_m_beta2 = static_cast<float>(1.0 - cfg->beta2);
                fa.inv_bc1 = static_cast<float>(1.0 / (1.0 - std::pow(cfg->beta1, static_cast<double>(c->step_feat))));
                fa.inv_bc2 = static_cast<float>(1.0 / (1.0 - std::pow(cfg->beta2, static_cast<double>(c->step_feat))));
                fa.plan = si.plan;
                if (sharded) fa.row_ss = ensure<float>(c->row_ss, n);
                tk::launch_feature_adam(fa, st);
                c->launches += n > 0 ? 3 : 0;
                if (sharded) {  // mapper.cpp:249: the norm of the whole row, over every shard
                    NK(g_nccl.AllReduce(fa.row_ss, fa.row_ss, static_cast<size_t>(n), ncclFloat32, ncclSum, c->comm,
                                        st));
                    tk::launch_feature_renorm(ptr<float>(c->feature), fa.row_ss, n, d, st);
                    c->launches += 1;
                }
                CK_LAUNCH(c);
            }
        }
        // the scene changed: the next render re-projects (records keep the pre-step snapshot)
        c->scene_version += 1;
        c->prepared = false;
        c->aux_valid = false;
        if (feature_step_out) *feature_step_out = feature_step ? 1 : 0;
        if (values_out) {
            sync(c);
            std::memcpy(values_out, c->hvals, 3 * sizeof(double));
        }
        main_done(c);
    });
}

tk_status tk_loss_values(tk_ctx* c, double values[3]) {
    return guarded([&] {
        if (!c->has_values) fail(TK_ERR_STATE, "no optimize_step has run");
        CK(cudaSetDevice(c->device));
        CK(cudaStreamSynchronize(c->stream));
        std::memcpy(values, c->hvals, 3 * sizeof(double));
    });
}

tk_status tk_scene_download(tk_ctx* c, const tk_scene_out* o) {
    return guarded([&] {
        if (!c || !o) fail(TK_ERR_BAD_ARG, "null argument");
        if (!c->has_scene) fail(TK_ERR_STATE, "no scene uploaded (tk_scene_upload)");
        if ((o->topk_count || o->max_contribution) && c->stat_n != c->n)
            fail(TK_ERR_STATE, "no selection statistics for this scene (tk_optimizer_reset)");
        CK(cudaSetDevice(c->device));
        on_main(c);
        const int64_t n = c->n;
        copy_out(o->mean, c->mean.p, n * 3 * sizeof(double), o->mem, c);
        copy_out(o->log_scale, c->log_scale.p, n * 3 * sizeof(double), o->mem, c);
        copy_out(o->rotation, c->rotation.p, n * 4 * sizeof(double), o->mem, c);
        copy_out(o->opacity_logit, c->opacity_logit.p, n * sizeof(double), o->mem, c);
        copy_out(o->color, c->color.p, n * 3 * sizeof(double), o->mem, c);
        if (o->feature && c->has_features)
            copy_out(o->feature, c->feature.p, static_cast<size_t>(n) * c->d * sizeof(float), o->mem, c);
        copy_out(o->topk_count, c->stat_count.p, n * sizeof(int32_t), o->mem, c);
        copy_out(o->max_contribution, c->stat_maxc.p, n * sizeof(double), o->mem, c);
        if (o->mem == TK_HOST) sync(c);
        main_done(c);
    });
}

// ------------------------------------------------------------------ structural edits
tk_status tk_scene_info(tk_ctx* c, int64_t* n, int32_t* d, uint64_t* generation) {
    return guarded([&] {
        if (!c) fail(TK_ERR_BAD_ARG, "null context");
        if (n) *n = c->n;
        if (d) *d = c->d;
        if (generation) *generation = c->generation;
    });
}

tk_status tk_insert_gaussians(tk_ctx* c, const tk_source_view* src, double tau, const tk_pose* w2c,
                              int32_t* inserted) {
    return guarded([&] {
        if (!c || !src || !w2c) fail(TK_ERR_BAD_ARG, "null argument");
        if (src->n < 0 || src->d < 0) fail(TK_ERR_BAD_ARG, "negative source size");
        if (src->n > 0 && (!src->position || !src->color || !src->spacing || !src->distance))
            fail(TK_ERR_BAD_ARG, "insert_gaussians: position, color, spacing and distance are required");
        if (!c->has_scene) fail(TK_ERR_STATE, "no scene uploaded (tk_scene_upload)");
        CK(cudaSetDevice(c->device));
        on_main(c);
        cudaStream_t st = c->cur;
        const int64_t ns = src->n;
        if (inserted) *inserted = 0;
        if (ns == 0) {
            main_done(c);
            return;
        }
        DevBuf bpos, bcol, bsp, bdist, bfeat, bflag, bflag32, bslot;
        auto dev_in = [&](DevBuf& b, const void* p, size_t bytes) -> const void* {
            if (src->mem == TK_DEVICE) return p;
            ensure<char>(b, bytes);
            copy_in(b.p, p, bytes, TK_HOST, c);
            return b.p;
        };
        const double* pos = static_cast<const double*>(dev_in(bpos, src->position, ns * 3 * sizeof(double)));
        const double* col = static_cast<const double*>(dev_in(bcol, src->color, ns * 3 * sizeof(double)));
        const double* sp = static_cast<const double*>(dev_in(bsp, src->spacing, ns * sizeof(double)));
        const double* dist = static_cast<const double*>(dev_in(bdist, src->distance, ns * sizeof(double)));
        const float* feat = (src->feature && src->d > 0)
                                ? static_cast<const float*>(dev_in(bfeat, src->feature, ns * src->d * sizeof(float)))
                                : nullptr;
        uint8_t* flag = ensure<uint8_t>(bflag, ns);
        int32_t* flag32 = ensure<int32_t>(bflag32, ns);
        int32_t* slot = ensure<int32_t>(bslot, ns);
        tk::launch_insert_flags(dist, ns, tau, flag, flag32, st);
        ensure_scratch(c, ns + 1);
        int64_t* dscal = ensure<int64_t>(c->dscal, 16);
        tk::scan_exclusive(flag32, slot, ns, dscal + 10, c->scratch.p, st, &c->launches);
        tk::copy_words_to_mapped(c->hscal_dev + 10, dscal + 10, 1, st);
        sync(c);
        const int64_t total = c->hscal[10];
        c->launches += 1;
        if (total > 0) {
            if (c->d == 0 && feat && (c->n == 0 || !c->has_features)) c->d = src->d;  // mapper.cpp:40-41
            const int64_t n0 = c->n, n1 = n0 + total;
            const int d = c->d;
            tk::InsertParams ip{};
            ip.n_src = ns;
            ip.base = n0;
            ip.position = pos;
            ip.color = col;
            ip.feature = feat;
            ip.d_src = src->d;
            ip.spacing = sp;
            ip.slot = slot;
            ip.flag = flag;
            // se3_inverse (pose.cpp:14-19) and its normalised rotation (mapper.cpp:25-26)
            const double qi[4] = {w2c->qw, -w2c->qx, -w2c->qy, -w2c->qz};
            const double t[3] = {w2c->tx, w2c->ty, w2c->tz};
            double ti[3];
            tk::quat_rotate_eigen(qi, t, ti);
            const double qn = std::sqrt(((qi[0] * qi[0] + qi[1] * qi[1]) + qi[2] * qi[2]) + qi[3] * qi[3]);
            for (int a = 0; a < 4; ++a) {
                ip.qi[a] = qi[a];
                ip.rot[a] = qi[a] / qn;
            }
            for (int a = 0; a < 3; ++a) ip.ti[a] = -ti[a];
            ip.opacity_logit = std::log(0.5 / (1.0 - 0.5));                     // logit(0.5)
            ip.d = d;
            ip.mean = grow_keep<double>(c, c->mean, n0 * 3, n1 * 3, false);
            ip.log_scale = grow_keep<double>(c, c->log_scale, n0 * 3, n1 * 3, false);
            ip.rotation = grow_keep<double>(c, c->rotation, n0 * 4, n1 * 4, false);
            ip.opacity = grow_keep<double>(c, c->opacity_logit, n0, n1, false);
            ip.color_out = grow_keep<double>(c, c->color, n0 * 3, n1 * 3, false);
            if (d > 0) {
                ip.feat = grow_keep<float>(c, c->feature, c->has_features ? n0 * d : 0, n1 * d, false);
                c->has_features = true;
            }
            tk::launch_insert_fill(ip, st);
            c->launches += 1;
            CK_LAUNCH(c);
            if (c->opt_ready && c->opt_n == n0) {  // OptimizerState::extend (optimizer.cpp:29-36)
                const int dims[5] = {3, 3, 4, 1, 3};
                for (int g = 0; g < 5; ++g) {
                    grow_keep<double>(c, c->am[g], n0 * dims[g], n1 * dims[g], true);
                    grow_keep<double>(c, c->av[g], n0 * dims[g], n1 * dims[g], true);
                }
                grow_keep<float>(c, c->fm, n0 * c->opt_d, n1 * d, true);
                grow_keep<float>(c, c->fv, n0 * c->opt_d, n1 * d, true);
                if (c->opt_d != d) {  // the feature group is sized now (mapper.cpp:54)
                    CK(cudaMemsetAsync(c->fm.p, 0, n1 * d * sizeof(float), st));
                    CK(cudaMemsetAsync(c->fv.p, 0, n1 * d * sizeof(float), st));
                }
                c->opt_n = n1;
                c->opt_d = d;
            }
            if (c->stat_n == n0) {
                grow_keep<int32_t>(c, c->stat_count, n0, n1, true);
                grow_keep<double>(c, c->stat_maxc, n0, n1, true);
                c->stat_n = n1;
            }
            c->n = n1;
            c->generation += 1;                                                 // mapper.cpp:56
            scene_changed(c);
            if (inserted) *inserted = static_cast<int32_t>(total);
        }
        sync(c);
        for (DevBuf* b : {&bpos, &bcol, &bsp, &bdist, &bfeat, &bflag, &bflag32, &bslot}) b->release();
        main_done(c);
    });
}

tk_status tk_prune_map(tk_ctx* c, double keep_ratio, uint64_t seed, int32_t threshold, int32_t* removed_out,
                       int64_t* n_removed) {
    return guarded([&] {
        if (!c) fail(TK_ERR_BAD_ARG, "null context");
        if (!c->has_scene) fail(TK_ERR_STATE, "no scene uploaded (tk_scene_upload)");
        if (c->stat_n != c->n) fail(TK_ERR_STATE, "no selection statistics for this scene (tk_optimizer_reset)");
        CK(cudaSetDevice(c->device));
        on_main(c);
        cudaStream_t st = c->cur;
        const int64_t n = c->n;
        std::vector<int32_t> counts(n);
        std::vector<double> maxc(n);
        copy_out(counts.data(), c->stat_count.p, n * sizeof(int32_t), TK_HOST, c);
        copy_out(maxc.data(), c->stat_maxc.p, n * sizeof(double), TK_HOST, c);
        sync(c);
        const std::vector<int32_t> removed = prune_select(counts, maxc, keep_ratio, seed, threshold);
        const int64_t nr = static_cast<int64_t>(removed.size());
        if (nr > 0) {  // mapper.cpp:141-154 + OptimizerState::compact
            DevBuf brem, bkeep, bpos;
            int32_t* drem = ensure<int32_t>(brem, nr);
            copy_in(drem, removed.data(), nr * sizeof(int32_t), TK_HOST, c);
            int32_t* keep = ensure<int32_t>(bkeep, n);
            int32_t* pos = ensure<int32_t>(bpos, n);
            tk::launch_keep_flags(drem, nr, n, keep, st);
            ensure_scratch(c, n + 1);
            int64_t* dscal = ensure<int64_t>(c->dscal, 16);
            tk::scan_exclusive(keep, pos, n, dscal + 11, c->scratch.p, st, &c->launches);
            c->launches += 2;
            const int64_t nk = n - nr;
            compact_rows<double>(c, c->mean, n, 3, nk, keep, pos);
            compact_rows<double>(c, c->log_scale, n, 3, nk, keep, pos);
            compact_rows<double>(c, c->rotation, n, 4, nk, keep, pos);
            compact_rows<double>(c, c->opacity_logit, n, 1, nk, keep, pos);
            compact_rows<double>(c, c->color, n, 3, nk, keep, pos);
            if (c->has_features && c->d > 0) compact_rows<float>(c, c->feature, n, c->d, nk, keep, pos);
            if (c->opt_ready && c->opt_n == n) {
                const int dims[5] = {3, 3, 4, 1, 3};
                for (int g = 0; g < 5; ++g) {
                    compact_rows<double>(c, c->am[g], n, dims[g], nk, keep, pos);
                    compact_rows<double>(c, c->av[g], n, dims[g], nk, keep, pos);
                }
                if (c->opt_d > 0) {
                    compact_rows<float>(c, c->fm, n, c->opt_d, nk, keep, pos);
                    compact_rows<float>(c, c->fv, n, c->opt_d, nk, keep, pos);
                }
                c->opt_n = nk;
            }
            sync(c);
            for (DevBuf* b : {&brem, &bkeep, &bpos}) b->release();
            c->n = nk;
            c->generation += 1;                                                 // mapper.cpp:153
            scene_changed(c);
        }
        // the statistics window restarts at every prune (mapper.cpp:156-159)
        CK(cudaMemsetAsync(c->stat_count.p, 0, std::max<int64_t>(c->n, 1) * sizeof(int32_t), st));
        CK(cudaMemsetAsync(c->stat_maxc.p, 0, std::max<int64_t>(c->n, 1) * sizeof(double), st));
        c->stat_n = c->n;
        if (removed_out && nr) std::memcpy(removed_out, removed.data(), nr * sizeof(int32_t));
        if (n_removed) *n_removed = nr;
        main_done(c);
    });
}

// ------------------------------------------------------------------ checkpoint / query
namespace {
constexpr char kSplfMagic[4] = {'S', 'P', 'L', 'F'};
constexpr uint32_t kSplfVersion = 1;

tk::SplfView splf_view(tk_ctx* c) {
    tk::SplfView v{};
    v.n = c->n;
    v.d = c->d;
    v.mean = ptr<double>(c->mean);
    v.log_scale = ptr<double>(c->log_scale);
    v.rotation = ptr<double>(c->rotation);
    v.opacity_logit = ptr<double>(c->opacity_logit);
    v.color = ptr<double>(c->color);
    v.feature = ptr<float>(c->feature);
    return v;
}
}  // namespace

tk_status tk_checkpoint_save(tk_ctx* c, const char* path) {
    return guarded([&] {
        if (!c || !path) fail(TK_ERR_BAD_ARG, "null argument");
        if (!c->has_scene) fail(TK_ERR_STATE, "no scene uploaded (tk_scene_upload)");
        if (c->d > 0 && !c->has_features) fail(TK_ERR_STATE, "scene has no features uploaded");
        CK(cudaSetDevice(c->device));
        on_main(c);
        const int64_t n = c->n;
        const int64_t W = 14 + c->d;
        DevBuf rec;
        float* drec = ensure<float>(rec, n * W);
        tk::launch_splf_pack(splf_view(c), drec, c->cur);
        c->launches += n > 0;
        CK_LAUNCH(c);
        const size_t body = static_cast<size_t>(n) * W * sizeof(float);
        char* host = nullptr;
        CK(cudaHostAlloc(reinterpret_cast<void**>(&host), 20 + body, cudaHostAllocDefault));
        std::memcpy(host, kSplfMagic, 4);                                        // checkpoint.cpp:42-45
        const uint32_t ver = kSplfVersion, dim = static_cast<uint32_t>(c->d);
        const uint64_t cnt = static_cast<uint64_t>(n);
        std::memcpy(host + 4, &ver, 4);
        std::memcpy(host + 8, &dim, 4);
        std::memcpy(host + 12, &cnt, 8);
        copy_out(host + 20, drec, body, TK_HOST, c);
        sync(c);
        rec.release();
        FILE* f = std::fopen(path, "wb");
        if (!f) {
            cudaFreeHost(host);
            fail(TK_ERR_BAD_ARG, std::string("checkpoint: cannot open ") + path + " for writing");
        }
        const size_t wrote = std::fwrite(host, 1, 20 + body, f);
        const int closed = std::fclose(f);
        cudaFreeHost(host);
        if (wrote != 20 + body || closed != 0) fail(TK_ERR_BAD_ARG, std::string("checkpoint: write failed for ") + path);
        main_done(c);
    });
}

tk_status tk_checkpoint_load(tk_ctx* c, const char* path) {
    return guarded([&] {
        if (!c || !path) fail(TK_ERR_BAD_ARG, "null argument");
        FILE* f = std::fopen(path, "rb");
        if (!f) fail(TK_ERR_BAD_ARG, std::string("checkpoint: cannot open ") + path);
        char hdr[20];
        const size_t got = std::fread(hdr, 1, 20, f);
        if (got < 4 || std::memcmp(hdr, kSplfMagic, 4) != 0) {
            std::fclose(f);
            fail(TK_ERR_BAD_ARG, std::string("checkpoint: bad magic in ") + path);
        }
        uint32_t ver = 0, dim = 0;
        uint64_t cnt = 0;
        if (got >= 8) std::memcpy(&ver, hdr + 4, 4);
        if (got >= 8 && ver != kSplfVersion) {
            std::fclose(f);
            fail(TK_ERR_BAD_ARG, "checkpoint: unsupported version " + std::to_string(ver) + " in " + path);
        }
        if (got < 20) {
            std::fclose(f);
            fail(TK_ERR_BAD_ARG, std::string("checkpoint: truncated file ") + path);
        }
        std::memcpy(&dim, hdr + 8, 4);
        std::memcpy(&cnt, hdr + 12, 8);
        if (cnt > static_cast<uint64_t>(INT32_MAX - 1)) {
            std::fclose(f);
            fail(TK_ERR_BAD_ARG, std::string("checkpoint: count too large in ") + path);
        }
        const int64_t n = static_cast<int64_t>(cnt);
        const int64_t W = 14 + static_cast<int64_t>(dim);
        const size_t body = static_cast<size_t>(n) * W * sizeof(float);
        char* host = nullptr;
        if (cudaHostAlloc(reinterpret_cast<void**>(&host), std::max<size_t>(body, 1), cudaHostAllocDefault) != cudaSuccess) {
            std::fclose(f);
            fail(TK_ERR_OOM, "checkpoint: pinned staging allocation failed");
        }
        const size_t rb = std::fread(host, 1, body, f);
        std::fclose(f);
        if (rb != body) {
            cudaFreeHost(host);
            fail(TK_ERR_BAD_ARG, std::string("checkpoint: truncated file ") + path);
        }
        CK(cudaSetDevice(c->device));
        on_main(c);
        DevBuf rec;
        float* drec = ensure<float>(rec, n * W);
        copy_in(drec, host, body, TK_HOST, c);
        ensure<double>(c->mean, n * 3);
        ensure<double>(c->log_scale, n * 3);
        ensure<double>(c->rotation, n * 4);
        ensure<double>(c->opacity_logit, n);
        ensure<double>(c->color, n * 3);
        ensure<float>(c->feature, n * std::max<int64_t>(dim, 1));
        c->n = n;
        c->d = static_cast<int32_t>(dim);
        tk::launch_splf_unpack(drec, splf_view(c), c->cur);
        c->launches += n > 0;
        CK_LAUNCH(c);
        sync(c);
        rec.release();
        cudaFreeHost(host);
        c->generation = 0;  // a loaded SceneMap starts at generation 0 (scene_map.hpp)
        c->has_scene = true;
        c->has_features = true;
        c->opt_ready = false;
        c->stat_n = -1;
        scene_changed(c);
        main_done(c);
    });
}

tk_status tk_segment_by_query(tk_ctx* c, const float* feature, int64_t n_pixels, int32_t d_feature,
                              int32_t feature_mem, const double* embeddings, int32_t classes, uint8_t* labels,
                              int32_t labels_mem) {
    return guarded([&] {
        if (!c || !embeddings || !labels) fail(TK_ERR_BAD_ARG, "null argument");
        if (classes <= 0 || classes > 255) fail(TK_ERR_BAD_ARG, "segment_by_query: classes must be in [1, 255]");
        CK(cudaSetDevice(c->device));
        on_side(c, true);
        cudaStream_t st = c->cur;
        // the context's own F under D-sharding is a channel slice: score it and all-reduce
        const bool sharded = !feature && c->comm && c->nranks > 1;
        const int d = feature ? d_feature : c->d, d_total = sharded ? c->d_total : d;
        if (d <= 0) fail(TK_ERR_BAD_ARG, "segment_by_query: embedding dimension mismatch");
        const int64_t P = feature ? n_pixels : c->fout_pixels;
        const float* F = feature;
        DevBuf &bf = c->q_feat, &be = c->q_emb, &bl = c->q_labels, &bb = c->q_best, &bacc = c->q_acc, &bn = c->q_nacc,
               &bpart = c->q_part;
        if (!F) {
            if (!c->f_out.p || c->fout_pixels <= 0) fail(TK_ERR_STATE, "segment_by_query: no rendered feature image");
            F = ptr<float>(c->f_out);
        } else if (feature_mem == TK_HOST) {
            float* df = ensure<float>(bf, P * d);
            copy_in(df, feature, static_cast<size_t>(P) * d * sizeof(float), TK_HOST, c);
            F = df;
        }
        double* de = ensure<double>(be, static_cast<int64_t>(classes) * d_total);
        copy_in(de, embeddings, static_cast<size_t>(classes) * d_total * sizeof(double), TK_HOST, c);
        uint8_t* dl = (labels_mem == TK_DEVICE) ? labels : ensure<uint8_t>(bl, P);
        tk::QueryParams q{};
        q.n_pixels = P;
        q.d = d;
        q.c0 = sharded ? c->rank * d : 0;
        q.d_total = d_total;
        q.classes = classes;
        q.feat = F;
        q.emb = de;
        q.labels = dl;
        q.best = ensure<double>(bb, P);
        if (tk::segment_query_chunk(d, classes) < d) {
            q.acc = ensure<double>(bacc, P * classes);
            q.nacc = ensure<double>(bn, P);
        }
        if (sharded) {  // per-rank partial dots over its channel slice, all-reduced (sum) with NCCL
            double* part = ensure<double>(bpart, P * (classes + 1));
            q.partial = part;
            q.norm2 = part + P * classes;
            tk::launch_segment_query(q, st);
            NK(g_nccl.AllReduce(part, part, static_cast<size_t>(P) * (classes + 1), ncclFloat64, ncclSum, c->comm, st));
            tk::launch_query_argmax(part, part + P * classes, P, classes, dl, st);
            c->launches += 2;
        } else {
            tk::launch_segment_query(q, st);
            c->launches += 1;
        }
        CK_LAUNCH(c);
        if (labels_mem == TK_HOST) {
            copy_out(labels, dl, P, TK_HOST, c);
            sync(c);
        }
        side_done(c, true);
    });
}

}  // extern "C"

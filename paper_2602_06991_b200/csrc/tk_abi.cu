// tk_abi.cu — the C ABI (include/tk_render.h): context, device-resident scene mirror, and the
// host orchestration of the sm_100a kernels for each reference frame entry point.  The mapping
// iteration lives in tk_abi_map.cu, checkpoints and queries in tk_abi_io.cu.
#include "tk_abi_internal.cuh"

#include <map>
#include <mutex>

namespace tkabi {

// ---------------------------------------------------------------- device memory pool
namespace {
std::mutex g_pool_mu;
std::map<int, std::multimap<size_t, void*>> g_pool;  // device -> cached blocks by size
int g_live_ctx = 0;
}  // namespace

void* pool_alloc(size_t bytes, size_t* got) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        auto& m = g_pool[dev];
        auto it = m.lower_bound(bytes);
        if (it != m.end() && it->first / 2 <= bytes) {
            void* p = it->second;
            *got = it->first;
            m.erase(it);
            return p;
        }
    }
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        pool_trim();
        e = cudaMalloc(&p, bytes);
    }
    CK(e);
    *got = bytes;
    return p;
}

void pool_free(void* p, size_t bytes) {
    if (!p) return;
    // the block's own device (the current device may be another context's)
    cudaPointerAttributes at{};
    int cur = 0;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess || cudaGetDevice(&cur) != cudaSuccess) {
        cudaGetLastError();
        cudaFree(p);
        return;
    }
    const int dev = at.device;
    if (dev != cur) cudaSetDevice(dev);
    const bool ok = cudaDeviceSynchronize() == cudaSuccess;
    if (!ok) cudaFree(p);  // a faulted context: hand the block back directly
    if (dev != cur) cudaSetDevice(cur);
    if (!ok) return;
    std::lock_guard<std::mutex> lk(g_pool_mu);
    g_pool[dev].emplace(bytes, p);
}

void pool_trim() {
    int cur = 0;
    cudaGetDevice(&cur);
    std::lock_guard<std::mutex> lk(g_pool_mu);
    for (auto& [dev, m] : g_pool) {
        if (m.empty()) continue;
        cudaSetDevice(dev);
        cudaDeviceSynchronize();
        for (auto& kv : m) cudaFree(kv.second);
        m.clear();
    }
    cudaSetDevice(cur);
}


// Host <-> device copies made inside an API call (timed as TK_PHASE_COPY when profiling).
// TK_HOST_ASYNC: the copy runs on s_in after the compute that may still read dst -- all compute
// issued so far, or, when the caller knows dst's last reader, only `reader` (`has_reader` false:
// dst has not been read yet) -- and the compute that follows waits for it.
void copy_in(void* dst, const void* src, size_t bytes, int mem, tk_ctx* c, const ReaderEvent* reader) {
    if (bytes == 0) return;
    if (mem == TK_HOST_ASYNC) {
        if (!reader) {
            CK(cudaEventRecord(c->ev_cmp, c->cur));
            CK(cudaStreamWaitEvent(c->s_in, c->ev_cmp, 0));
        } else if (reader->pending) {
            CK(cudaStreamWaitEvent(c->s_in, reader->ev, 0));
        }
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


void copy_out(void* dst, const void* src, size_t bytes, int mem, tk_ctx* c, int tag) {
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
    f.tile_begin = 0;
    f.tile_end = f.tiles_x * f.tiles_y;
    (void)c;
    return f;
}

// Geometry split (tk_geometry_band): the sweeps cover tile rows [band * rows_b, (band + 1) * rows_b),
// rows_b = ceil(tiles_y / bands); the pixels of a band are one contiguous run of `band_pixels`
// pixels (the last band padded), so the per-pixel records all-gather as equal NCCL chunks.
int64_t band_pixels(const tk::Frame& f, int bands) {
    const int rows_b = (f.tiles_y + bands - 1) / bands;
    return static_cast<int64_t>(rows_b) * f.tile_size * f.width;
}
void apply_band(tk_ctx* c, tk::Frame& f) {
    if (c->band_n <= 1) return;
    const int rows_b = (f.tiles_y + c->band_n - 1) / c->band_n;
    const int ty0 = std::min(f.tiles_y, c->band * rows_b), ty1 = std::min(f.tiles_y, ty0 + rows_b);
    f.tile_begin = ty0 * f.tiles_x;
    f.tile_end = ty1 * f.tiles_x;
}
// all ranks of tk_comm take part: records are all-gathered and MidGrad sum-reduced
bool band_collective(const tk_ctx* c) { return c->band_n > 1 && c->comm && c->nranks == c->band_n; }

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

void ensure_scratch(tk_ctx* c, int64_t n, bool feat) {
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
    CK_LAUNCH(c);

    int32_t* pos = ensure<int32_t>(c->pos, n);
    tk::scan_exclusive(pp.valid, pos, n, dscal + 0, c->scratch.p, st);
    uint64_t* dkeys = ensure<uint64_t>(c->dkeys, n);
    uint32_t* dvals = ensure<uint32_t>(c->dvals, n);
    uint64_t* dkeys_alt = ensure<uint64_t>(c->dkeys_alt, n);
    uint32_t* dvals_alt = ensure<uint32_t>(c->dvals_alt, n);
    tk::launch_compact(pp.valid, pos, pp.z, n, pp.key_min, dkeys, dvals, st);
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
            tk::radix_sort_pairs_u64(dkeys, dvals, dkeys_alt, dvals_alt, n_vis, lo_bit, hb, c->scratch.p, st, &alt);
            tk::fixup_runs_u64(alt ? dkeys_alt : dkeys, alt ? dvals_alt : dvals, n_vis, lo_bit,
                               reinterpret_cast<int32_t*>(dscal + 7), st);
            CK_LAUNCH(c);
        }
        c->order = alt ? dvals_alt : dvals;
        tk::launch_sorted_ntiles(c->order, n_vis, pp.ntiles, nts, st);
        tk::scan_exclusive(nts, poff, n_vis, dscal + 3, c->scratch.p, st);
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
    tk::launch_emit_pairs(c->order, n_vis, pp.rect, nts, poff, f.tiles_x, tkeys, tvals,
                          ensure<int32_t>(c->emit_big, std::max<int64_t>(n_vis, 1)),
                          reinterpret_cast<int32_t*>(dscal + 14), st);  // emit queue count
    ensure_scratch(c, std::max<int64_t>(n_pairs, n_tiles + 1));
    bool talt = false;
    const int tbits = bits_for(static_cast<uint64_t>(n_tiles - 1));
    if (n_pairs > 1 && tbits > 0) {
        tk::radix_sort_pairs_u32(tkeys, tvals, tkeys_alt, tvals_alt, n_pairs, 0, tbits, c->scratch.p, st, &talt);
    }
    c->tile_keys_sorted = talt ? tkeys_alt : tkeys;
    c->tile_vals_sorted = talt ? tvals_alt : tvals;
    int32_t* toff = ensure<int32_t>(c->tile_offsets, n_tiles + 1);
    tk::segment_offsets_u32(c->tile_keys_sorted, n_pairs, toff, n_tiles, st);
    int32_t* pcnt = ensure<int32_t>(c->padded_cnt, n_tiles + 1);
    int32_t* pstart = ensure<int32_t>(c->padded_start, n_tiles + 1);
    tk::launch_padded_counts(toff, n_tiles, pcnt, st);
    tk::scan_exclusive(pcnt, pstart, n_tiles + 1, dscal + 4, c->scratch.p, st);
    const int64_t padded_cap = n_pairs + static_cast<int64_t>(tk::kEntryAlign) * n_tiles + 128;
    ensure<tk::EntryChunk>(c->te, padded_cap / tk::kChunk + 1);
    ensure<int32_t>(c->wl, padded_cap * tk::geom_blocks_per_tile(s->tile_size));
    c->padded_cap = padded_cap;
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
    mp.rect = pp.rect;
    mp.pair_off = poff;
    mp.tiles_x = f.tiles_x;
    mp.entry_pair = ensure<int32_t>(c->entry_pair, padded_cap);
    tk::launch_materialize(mp, st);
    CK_LAUNCH(c);
    c->prepared = true;
    c->prep_key = key;
}


// geometric_pass (render.cpp:158-240).  Record/colour outputs are optional (null = skip);
// the per-pixel aux (final T, entries visited) is always written for the backward.
void forward(tk_ctx* c, const tk_camera* cam, const tk_settings* s, bool records) {
    tk::Frame f = make_frame(c, cam, s);
    apply_band(c, f);
    const bool gather = band_collective(c) && records;
    // record buffers hold whole bands when they are all-gathered (the last band padded)
    const int64_t P = gather ? band_pixels(f, c->band_n) * c->band_n : static_cast<int64_t>(f.width) * f.height;
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
    CK_LAUNCH(c);
    if (gather) {  // every rank swept its band: assemble the whole frame's records on every rank
        const int64_t bp = band_pixels(f, c->band_n);
        const int64_t off = bp * c->rank;
        const size_t kk = static_cast<size_t>(std::max(k, 1));
        NK(g_nccl.AllGather(gp.topk_index + off * kk, gp.topk_index, bp * kk, ncclInt32, c->comm, st));
        NK(g_nccl.AllGather(gp.topk_weight + off * kk, gp.topk_weight, bp * kk, ncclFloat64, c->comm, st));
        NK(g_nccl.AllGather(gp.topk_count + off, gp.topk_count, bp, ncclUint8, c->comm, st));
        NK(g_nccl.AllGather(gp.color + off * 3, gp.color, bp * 3, ncclFloat64, c->comm, st));
        NK(g_nccl.AllGather(gp.depth + off, gp.depth, bp, ncclFloat64, c->comm, st));
        NK(g_nccl.AllGather(gp.alpha + off, gp.alpha, bp, ncclFloat64, c->comm, st));
        // peak weights: positive doubles order like their bit patterns (render.cpp:212's max)
        NK(g_nccl.AllReduce(gp.contrib, gp.contrib, static_cast<size_t>(c->n), ncclUint64, ncclMax, c->comm, st));
    }
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


// Inverted (Gaussian -> record slots) index of a TopKGrid, ascending slot order per Gaussian.
SlotIndex build_slot_index(tk_ctx* c, const Records& r) {
    const int64_t slots = static_cast<int64_t>(r.w) * r.h * r.k;
    const int64_t n = c->n;
    uint32_t* keys = ensure<uint32_t>(c->s_keys, slots);
    uint32_t* vals = ensure<uint32_t>(c->s_vals, slots);
    uint32_t* keys_alt = ensure<uint32_t>(c->s_keys_alt, slots);
    uint32_t* vals_alt = ensure<uint32_t>(c->s_vals_alt, slots);
    int32_t* queue = ensure<int32_t>(c->s_queue, n + 2);
    float* wn = ensure<float>(c->s_wnorm, slots);
    int32_t* seg = ensure<int32_t>(c->s_seg, n + 1);
    ensure_scratch(c, std::max<int64_t>(slots, n + 1), true);
    PhaseScope phase(c, TK_PHASE_FBWD_INDEX);
    tk::SlotKeyParams sk{slots, r.k, n, r.index, r.weight, r.count, nullptr, nullptr, wn};
    const uint32_t* sorted = nullptr;
    int32_t* plan_counters = ensure<int32_t>(c->lp_counters, tk::kPlanCounters + 1);
    tk::launch_slot_index(sk, n, seg, queue, keys, vals, keys_alt, vals_alt, &sorted, c->scratch_feat.p, plan_counters,
                          c->cur);
    tk::LongPlan plan{};
    plan.cap_items = tk::long_plan_capacity(slots, n);
    plan.cap_l1 = tk::long_plan_l1_capacity(slots, n);
    plan.items = ensure<int4>(c->lp_items, plan.cap_items);
    plan.longs = ensure<int4>(c->lp_longs, tk::long_plan_longs(slots, n) + 1);
    plan.counters = plan_counters;
    plan.l1_map = ensure<int2>(c->lp_l1map, plan.cap_l1);
    plan.partial = ensure<float>(c->lp_partial, plan.cap_items * std::max(c->d, 1));
    plan.l1 = ensure<float>(c->lp_l1, plan.cap_l1 * std::max(c->d, 1));
    plan.queue = queue;
    plan.qcount = queue + n + 1;
    plan.slots = sorted;
    plan.k = r.k;
    plan.width = std::max(r.w, 1);
    plan.band_rows = std::max(1, (r.h + tk::kBands - 1) / tk::kBands);
    tk::launch_long_plan(seg, n, plan, c->cur);
    return SlotIndex{seg, sorted, wn, plan};
}

// The backward sweep of backward_geometric (backward.cpp:106-188) into the per-Gaussian
// projected-space gradients (n x 10), on the forward state of this context.
double* geom_sweep(tk_ctx* c, const tk::Frame& f0, const double* gc, const double* gd) {
    tk::Frame f = f0;
    apply_band(c, f);
    const int64_t n = c->n;
    double* mid = ensure<double>(c->mid, n * 10);
    if (c->geom_atomic) CK(cudaMemsetAsync(mid, 0, std::max<int64_t>(n, 1) * 10 * sizeof(double), c->cur));
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
    bp.nsub = tk::geom_blocks_per_tile(f.tile_size);
    if (!c->geom_atomic) {
        const int64_t slots = std::max<int64_t>(c->n_pairs, 1) * bp.nsub;
        bp.part = ensure<double>(c->g_part, slots * 10);
        // flags + the queue counters behind them, zeroed in one memset
        const int64_t fbytes = tk::align_up(slots, 16);
        bp.part_flag = ensure<uint8_t>(c->g_flag, fbytes + 16);
        bp.entry_pair = ptr<int32_t>(c->entry_pair);
        CK(cudaMemsetAsync(bp.part_flag, 0, fbytes + 16, c->cur));
    }
    {
        PhaseScope phase(c, TK_PHASE_GEOM_BWD);
        tk::launch_geom_bwd(bp, tk::geom_blocks(f), c->cur);
        if (!c->geom_atomic) {
            tk::MidReduceParams mr{};
            mr.nv = c->n_vis;
            mr.order = c->order;
            mr.ntiles_sorted = ptr<int32_t>(c->ntiles_sorted);
            mr.pair_off = ptr<int32_t>(c->pair_off);
            mr.part = bp.part;
            mr.part_flag = bp.part_flag;
            mr.nsub = bp.nsub;
            mr.mid = mid;
            mr.big_list = ensure<int32_t>(c->g_big, std::max<int64_t>(c->n_vis, 1));
            mr.big_count = reinterpret_cast<int32_t*>(
                bp.part_flag + tk::align_up(std::max<int64_t>(c->n_pairs, 1) * bp.nsub, 16));
            tk::launch_mid_reduce(mr, c->cur);
        }
    }
    CK_LAUNCH(c);
    if (band_collective(c)) {  // each rank merged its band's partials: sum them over the ranks
        if (c->geom_atomic) fail(TK_ERR_STATE, "the geometry split needs the deterministic merge");
        NK(g_nccl.AllReduce(mid, mid, static_cast<size_t>(c->n_vis) * 10, ncclFloat64, ncclSum, c->comm, c->cur));
    }
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
    if (!c->geom_atomic) {  // geom_sweep's fixed-order merge leaves mid by depth rank
        cp.order = c->order;
        cp.ntiles_sorted = ptr<int32_t>(c->ntiles_sorted);
        cp.nv = c->n_vis;
    }
    return cp;
}
void flush_features(tk_ctx* c) {
    if (!c->feat_stale) return;
    c->feat_stale = false;
    if (!c->opt_ready || c->opt_n != c->n || c->opt_d != c->d || !c->f_last.p) return;
    tk::FeatAdamParams fa{};
    fa.n = c->n;
    fa.d = c->d;
    fa.feat = ptr<float>(c->feature);
    fa.m = ptr<float>(c->fm);
    fa.v = ptr<float>(c->fv);
    fa.last = ptr<int32_t>(c->f_last);
    fa.tab = ptr<tk::AdamStepParams>(c->f_tab);
    tk::launch_feature_catchup(fa, static_cast<int>(c->step_feat), false, c->cur);
    CK_LAUNCH(c);
}

// Drop the fused all-gather's peer buffers (IPC mappings closed, own buffer freed).
void release_peers(tk_ctx* c) {
    if (c->peer_ipc)
        for (int r = 0; r < c->peer_n; ++r)
            if (r != c->peer_rank && c->peer_ptrs[r]) cudaIpcCloseMemHandle(c->peer_ptrs[r]);
    c->peer_own.release();
    for (float*& q : c->peer_ptrs) q = nullptr;
    c->peer_n = 0;
    c->peer_ipc = false;
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

}  // namespace tkabi

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
        {
            std::lock_guard<std::mutex> lk(g_pool_mu);
            ++g_live_ctx;
        }
        c->device = device;
        cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
        // The HBM-bound feature chain (short dependent launches) gets the highest priority so its
        // blocks are scheduled as soon as the long fp64 geometry-backward grid frees SM slots.
        int prio_lo = 0, prio_hi = 0;
        cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
        // Side streams only with TK_OVERLAP=1: on B200 the fp64 geometry backward and the feature
        // kernels each fill the SMs' register files, so overlapping them measured no gain; the
        // default aliases every stream to the main one (per-kernel times stay unambiguous).
        const char* gat = std::getenv("TK_GEOM_BWD_ATOMIC");
        c->geom_atomic = gat && gat[0] == '1';
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
                                &c->ev_out[4], &c->ev_scene_free, &c->fgrad_reader.ev, &c->ggrad_reader.ev})
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
            {
                std::lock_guard<std::mutex> lk(g_pool_mu);
                --g_live_ctx;
            }
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
    // device buffers (DevBuf members, keyframes) are freed by their destructors in `delete c`
    if (c->hvals) cudaFreeHost(c->hvals);
    release_peers(c);
    if (c->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(c->comm);
    if (c->hscal) cudaFreeHost(c->hscal);
    if (c->stream) cudaStreamDestroy(c->stream);
    if (c->s_feat && c->s_feat != c->stream) cudaStreamDestroy(c->s_feat);
    if (c->s_geo && c->s_geo != c->stream) cudaStreamDestroy(c->s_geo);
    for (cudaEvent_t e : {c->ev_main, c->ev_feat, c->ev_geo, c->ev_cmp, c->ev_in, c->ev_out[0], c->ev_out[1],
                          c->ev_out[2], c->ev_out[3], c->ev_out[4], c->ev_scene_free, c->fgrad_reader.ev,
                          c->ggrad_reader.ev})
        if (e) cudaEventDestroy(e);
    if (c->h_twist) cudaFreeHost(c->h_twist);
    if (c->s_in) cudaStreamDestroy(c->s_in);
    if (c->s_out) cudaStreamDestroy(c->s_out);
    delete c;
    bool last = false;
    {
        std::lock_guard<std::mutex> lk(tkabi::g_pool_mu);
        last = --g_live_ctx <= 0;
        if (last) g_live_ctx = 0;
    }
    if (last) pool_trim();
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
int64_t tk_kernel_launches(tk_ctx* c) { return c ? tk::launch_count() : 0; }

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
        flush_features(c);  // lazily optimised feature rows must be current
        cudaStream_t st = c->cur;
        const int64_t n = s->n;
        if (!s->feature && c->has_features && (n != c->n || s->d != c->d))
            fail(TK_ERR_BAD_ARG, "feature == NULL requires unchanged n and d");
        if (mem == TK_HOST_ASYNC) {
            // Double buffer: the copies fill the back set, waiting only for the compute that read
            // it (issued before the previous upload) -- not for the frame still running on the
            // front set -- then the sets swap; compute issued from here on waits for the copies.
            if (c->scene_free_pending) CK(cudaStreamWaitEvent(c->s_in, c->ev_scene_free, 0));
            if (c->out_pending[0]) CK(cudaStreamWaitEvent(c->s_in, c->ev_out[0], 0));
            auto up = [&](void* dst, const void* src, size_t bytes) {
                if (bytes) CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->s_in));
            };
            up(ensure<double>(c->mean_b, n * 3), s->mean, n * 3 * sizeof(double));
            up(ensure<double>(c->log_scale_b, n * 3), s->log_scale, n * 3 * sizeof(double));
            up(ensure<double>(c->rotation_b, n * 4), s->rotation, n * 4 * sizeof(double));
            up(ensure<double>(c->opacity_logit_b, n), s->opacity_logit, n * sizeof(double));
            up(ensure<double>(c->color_b, n * 3), s->color, n * 3 * sizeof(double));
            if (s->feature)
                up(ensure<float>(c->feature_b, n * std::max(s->d, 1)), s->feature,
                   static_cast<size_t>(n) * s->d * sizeof(float));
            CK(cudaEventRecord(c->ev_in, c->s_in));
            CK(cudaEventRecord(c->ev_scene_free, st));  // the outgoing front set: read by compute so far
            c->scene_free_pending = true;
            CK(cudaStreamWaitEvent(st, c->ev_in, 0));
            std::swap(c->mean, c->mean_b);
            std::swap(c->log_scale, c->log_scale_b);
            std::swap(c->rotation, c->rotation_b);
            std::swap(c->opacity_logit, c->opacity_logit_b);
            std::swap(c->color, c->color_b);
            if (s->feature) {
                std::swap(c->feature, c->feature_b);
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
            return;
        }
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

tk_status tk_scene_upload_features(tk_ctx* c, int64_t n, int32_t d, const float* feature, int32_t mem) {
    return guarded([&] {
        if (!c || (!feature && n * d > 0)) fail(TK_ERR_BAD_ARG, "null argument");
        if (!c->has_scene || n != c->n || d != c->d)
            fail(TK_ERR_BAD_ARG, "tk_scene_upload_features: n and d must match the resident geometry");
        CK(cudaSetDevice(c->device));
        on_main(c);
        flush_features(c);  // pending lazy rows would otherwise overwrite the new values
        if (mem == TK_HOST_ASYNC) mem = TK_HOST;
        copy_in(ensure<float>(c->feature, n * std::max(d, 1)), feature, static_cast<size_t>(n) * d * sizeof(float), mem,
                c);
        c->has_features = true;  // geometry, the PreparedScene and the forward state stay valid
        main_done(c);
    });
}

tk_status tk_device_view_get(tk_ctx* c, tk_device_view* v) {
    return guarded([&] {
        std::memset(v, 0, sizeof(*v));
        if (c->feat_stale) {  // the view exposes the feature rows: bring them up to date
            CK(cudaSetDevice(c->device));
            on_main(c);
            flush_features(c);
            main_done(c);
        }
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
        flush_features(c);  // lazily optimised feature rows must be current
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
        // backward.cpp:273-321 reads the map's size and feature_dim only, never feature values
        if (!c->has_scene) fail(TK_ERR_STATE, "no scene uploaded (tk_scene_upload)");
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
            copy_in(dg, grad, static_cast<size_t>(P) * c->d * sizeof(float), grad_mem, c, &c->fgrad_reader);
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
        CK_LAUNCH(c);
        c->fgrad_reader.record(st);  // the next asynchronous grad_feature upload waits only for this
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
        flush_features(c);  // lazily optimised feature rows must be current
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
        tk::scan_exclusive(gp.list_count, off, P + 1, dscal + 6, c->scratch.p, st);
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
            copy_in(dgc, grad_color, P * 3 * sizeof(double), grad_mem, c, &c->ggrad_reader);
            gc = dgc;
            if (grad_depth) {
                double* dgd = ensure<double>(c->g_depth_in, P);
                copy_in(dgd, grad_depth, P * sizeof(double), grad_mem, c, &c->ggrad_reader);
                gd = dgd;
            }
        }
        double* mid = geom_sweep(c, f, gc, gd);
        c->ggrad_reader.record(c->cur);  // the next asynchronous grad upload waits only for the sweep
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
            tk::launch_twist_reduce(cp.twist, tk::chain_items(cp), tpart, tout, st);
        }
        CK_LAUNCH(c);
        if (out) {
            if (out->mem != TK_DEVICE) {
                copy_out(out->mean, cp.g_mean, n * 3 * sizeof(double), out->mem, c, kOutGG);
                copy_out(out->log_scale, cp.g_log_scale, n * 3 * sizeof(double), out->mem, c, kOutGG);
                copy_out(out->rotation, cp.g_rotation, n * 4 * sizeof(double), out->mem, c, kOutGG);
                copy_out(out->opacity_logit, cp.g_opacity_logit, n * sizeof(double), out->mem, c, kOutGG);
                copy_out(out->color, cp.g_color, n * 3 * sizeof(double), out->mem, c, kOutGG);
            }
            if (out->mem == TK_HOST_ASYNC || out->mem == TK_DEVICE) {  // the twist lands at tk_synchronize
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
        CK_LAUNCH(c);
        if (out && out_mem == TK_HOST) copy_out(out, dst, slice * c->nranks * sizeof(float), TK_HOST, c);
        sync(c);
        tmp.release();
        side_done(c, true);
    });
}

tk_status tk_comm_set_peers(tk_ctx* c, int32_t rank, int32_t nranks, int32_t d_total, float* const* buffers,
                            int64_t n_pixels) {
    return guarded([&] {
        if (!c || !buffers) fail(TK_ERR_BAD_ARG, "null argument");
        if (nranks < 1 || nranks > tk::kMaxPeers || rank < 0 || rank >= nranks)
            fail(TK_ERR_BAD_ARG, "bad rank / nranks (1 <= nranks <= 8)");
        if (d_total <= 0 || d_total % nranks || (d_total / nranks) % 4 || n_pixels < 0)
            fail(TK_ERR_BAD_ARG, "d_total must split into nranks slices of a multiple of 4 channels");
        for (int r = 0; r < nranks; ++r)
            if (!buffers[r]) fail(TK_ERR_BAD_ARG, "null peer buffer");
        CK(cudaSetDevice(c->device));
        release_peers(c);
        for (int r = 0; r < nranks; ++r) c->peer_ptrs[r] = buffers[r];
        c->peer_n = nranks;
        c->peer_rank = rank;
        c->peer_dtotal = d_total;
        c->peer_pixels = n_pixels;
    });
}

tk_status tk_comm_p2p_setup(tk_ctx* c, int64_t n_pixels) {
    return guarded([&] {
        if (!c) fail(TK_ERR_BAD_ARG, "null context");
        if (!c->comm) fail(TK_ERR_STATE, "tk_comm_init not called");
        if (c->nranks > tk::kMaxPeers) fail(TK_ERR_BAD_ARG, "fused all-gather supports up to 8 ranks");
        if (c->d_total % c->nranks || (c->d_total / c->nranks) % 4)
            fail(TK_ERR_BAD_ARG, "d_total must split into nranks slices of a multiple of 4 channels");
        CK(cudaSetDevice(c->device));
        on_main(c);
        sync(c);
        release_peers(c);
        // every rank's IPC handle to every rank (NCCL all-gather of the 64-byte handles).  A rank
        // that cannot export its buffer still joins the all-gather (with a zero handle), so every
        // rank sees the failure and returns the same error instead of hanging in the collective.
        cudaIpcMemHandle_t mine;
        std::memset(&mine, 0, sizeof(mine));
        float* own = nullptr;
        std::string export_error;
        try {
            own = ensure<float>(c->peer_own, static_cast<size_t>(std::max<int64_t>(n_pixels, 1)) * c->d_total);
            CK(cudaIpcGetMemHandle(&mine, own));
        } catch (const TkError& e) {
            export_error = e.msg;
            std::memset(&mine, 0, sizeof(mine));
        }
        static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
        DevBuf hb;
        uint8_t* dh = ensure<uint8_t>(hb, 64 * (c->nranks + 1));
        CK(cudaMemcpyAsync(dh + 64 * c->nranks, &mine, 64, cudaMemcpyHostToDevice, c->cur));
        NK(g_nccl.AllGather(dh + 64 * c->nranks, dh, 64, ncclUint8, c->comm, c->cur));
        std::vector<cudaIpcMemHandle_t> all(c->nranks);
        CK(cudaMemcpyAsync(all.data(), dh, 64 * c->nranks, cudaMemcpyDeviceToHost, c->cur));
        sync(c);
        hb.release();
        static const cudaIpcMemHandle_t zero{};
        for (int r = 0; r < c->nranks; ++r)
            if (std::memcmp(&all[r], &zero, sizeof(zero)) == 0) {
                c->peer_own.release();
                fail(TK_ERR_CUDA, "tk_comm_p2p_setup: rank " + std::to_string(r) + " could not export its buffer" +
                                      (export_error.empty() ? std::string() : " (" + export_error + ")"));
            }
        c->peer_ipc = true;
        // the barrier word (tk_render_feature_gathered), initialised once; a max-reduce keeps it 0
        CK(cudaMemsetAsync(ensure<int32_t>(c->peer_word, 1), 0, sizeof(int32_t), c->cur));
        c->peer_n = c->nranks;
        c->peer_rank = c->rank;
        c->peer_dtotal = c->d_total;
        c->peer_pixels = n_pixels;
        for (int r = 0; r < c->nranks; ++r) {
            if (r == c->rank) {
                c->peer_ptrs[r] = own;
                continue;
            }
            void* q = nullptr;
            CK(cudaIpcOpenMemHandle(&q, all[r], cudaIpcMemLazyEnablePeerAccess));
            c->peer_ptrs[r] = static_cast<float*>(q);
        }
        main_done(c);
    });
}

tk_status tk_render_feature_gathered(tk_ctx* c, const tk_topk_view* topk, float* out, int32_t out_mem) {
    return guarded([&] {
        if (!c) fail(TK_ERR_BAD_ARG, "null context");
        if (c->peer_n == 0) fail(TK_ERR_STATE, "no peer buffers (tk_comm_p2p_setup or tk_comm_set_peers)");
        CK(cudaSetDevice(c->device));
        on_side(c, true);
        flush_features(c);  // lazily optimised feature rows must be current
        require_features(c);
        if (c->d * c->peer_n != c->peer_dtotal) fail(TK_ERR_BAD_ARG, "d_total must equal nranks * d_shard");
        const Records r = resolve_records(c, topk, "render_feature");
        if (r.k > tk::kMaxTopK) fail(TK_ERR_BAD_ARG, "TopKGrid k exceeds 32");
        const int64_t P = static_cast<int64_t>(r.w) * r.h;
        if (P > c->peer_pixels) fail(TK_ERR_BAD_ARG, "frame larger than the registered peer buffers");
        if (reinterpret_cast<uintptr_t>(ptr<float>(c->feature)) % 16) fail(TK_ERR_BAD_ARG, "feature rows misaligned");
        wait_out(c, kOutF);
        tk::GatherParams gp{P, r.k, r.index, r.weight, r.count, ptr<float>(c->feature), c->d, nullptr, r.w, r.h};
        if (c->comm && c->peer_ipc) {
            // Stream-ordered rank barrier BEFORE the peer stores: every rank's stream has passed
            // everything it enqueued before this call -- its reads of the previous frame's
            // gathered buffer included -- so this frame's stores cannot overwrite a map a peer is
            // still reading (write-after-read across ranks).  Readers on other streams must be
            // ordered before the next call by the caller (tk_comm_gathered_buffer contract).
            NK(g_nccl.AllReduce(ptr<int32_t>(c->peer_word), ptr<int32_t>(c->peer_word), 1, ncclInt32, ncclMax,
                                c->comm, c->cur));
        }
        gp.n_peers = c->peer_n;
        gp.peer_stride = c->peer_dtotal;
        gp.peer_off = c->peer_rank * c->d;
        for (int q = 0; q < c->peer_n; ++q) gp.peers[q] = c->peer_ptrs[q];
        {
            PhaseScope phase(c, TK_PHASE_GATHER);
            tk::launch_feature_gather(gp, c->cur);
        }
        CK_LAUNCH(c);
        if (c->comm && c->peer_ipc) {  // stream-ordered rank barrier: every peer's slice has landed
            NK(g_nccl.AllReduce(ptr<int32_t>(c->peer_word), ptr<int32_t>(c->peer_word), 1, ncclInt32, ncclMax,
                                c->comm, c->cur));
        }
        if (out) {
            const size_t bytes = static_cast<size_t>(P) * c->peer_dtotal * sizeof(float);
            copy_out(out, c->peer_ptrs[c->peer_rank], bytes, out_mem == TK_DEVICE ? TK_DEVICE : out_mem, c, kOutF);
            if (out_mem == TK_HOST) sync(c);
        }
        side_done(c, true);
    });
}

tk_status tk_geometry_band(tk_ctx* c, int32_t band, int32_t nbands) {
    return guarded([&] {
        if (!c) fail(TK_ERR_BAD_ARG, "null context");
        if (nbands < 1 || band < 0 || band >= nbands) fail(TK_ERR_BAD_ARG, "band must be in [0, nbands)");
        if (c->comm && nbands > 1 && (nbands != c->nranks || band != c->rank))
            fail(TK_ERR_BAD_ARG, "under tk_comm the geometry split needs nbands == nranks and band == rank");
        if (nbands > 1 && c->geom_atomic) fail(TK_ERR_STATE, "the geometry split needs the deterministic merge");
        c->band = band;
        c->band_n = nbands;
        c->prepared = false;  // the forward state of another band is no use
        c->aux_valid = false;
    });
}

tk_status tk_comm_gathered_buffer(tk_ctx* c, float** buffer) {
    return guarded([&] {
        if (!c || !buffer) fail(TK_ERR_BAD_ARG, "null argument");
        if (c->peer_n == 0) fail(TK_ERR_STATE, "no peer buffers");
        *buffer = c->peer_ptrs[c->peer_rank];
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

}  // extern "C"

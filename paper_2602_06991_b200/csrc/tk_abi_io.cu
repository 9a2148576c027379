// tk_abi_io.cu — the C ABI of the map formats and queries: SPLF checkpoints and
// segment_by_query.
#include "tk_abi_internal.cuh"

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

extern "C" {

// ------------------------------------------------------------------ FEAT feature frames
// read_feature_bin / write_feature_bin (synth/dataset.cpp:48-76): "FEAT", uint32 h, w, d, then
// h * w * d fp32 in HWC order -- the keyframe's feature image, streamed through pinned memory.
namespace {
constexpr char kFeatMagic[4] = {'F', 'E', 'A', 'T'};
}

tk_status tk_keyframe_load_features(tk_ctx* c, int32_t slot, const char* path) {
    return guarded([&] {
        if (!c || !path) fail(TK_ERR_BAD_ARG, "null argument");
        if (slot < 0 || static_cast<size_t>(slot) >= c->kfs.size() || c->kfs[slot].w == 0)
            fail(TK_ERR_BAD_ARG, "keyframe_load_features: no keyframe in that slot");
        std::FILE* fp = std::fopen(path, "rb");
        if (!fp) fail(TK_ERR_BAD_ARG, std::string("dataset: cannot open ") + path);
        struct Closer {
            std::FILE* f;
            ~Closer() { std::fclose(f); }
        } closer{fp};
        char magic[4];
        uint32_t hdr[3];
        if (std::fread(magic, 1, 4, fp) != 4 || std::memcmp(magic, kFeatMagic, 4) != 0)
            fail(TK_ERR_BAD_ARG, std::string("dataset: bad magic in ") + path);
        if (std::fread(hdr, 4, 3, fp) != 3) fail(TK_ERR_BAD_ARG, std::string("dataset: truncated header in ") + path);
        Keyframe& k = c->kfs[slot];
        const uint32_t h = hdr[0], w = hdr[1], d = hdr[2];
        if (static_cast<int>(h) != k.h || static_cast<int>(w) != k.w)
            fail(TK_ERR_BAD_ARG, "keyframe_load_features: feature image shape differs from the keyframe");
        const int64_t P = static_cast<int64_t>(w) * h;
        const size_t bytes = static_cast<size_t>(P) * d * sizeof(float);
        CK(cudaSetDevice(c->device));
        on_main(c);
        float* host = nullptr;
        CK(cudaHostAlloc(reinterpret_cast<void**>(&host), std::max<size_t>(bytes, 4), cudaHostAllocDefault));
        struct HostFree {
            float* p;
            ~HostFree() { cudaFreeHost(p); }
        } hf{host};
        if (std::fread(host, 1, bytes, fp) != bytes) fail(TK_ERR_BAD_ARG, std::string("dataset: truncated data in ") + path);
        k.d = static_cast<int>(d);
        k.has_feature = d > 0;
        float* feat = d > 0 ? ensure<float>(k.feature, static_cast<size_t>(P) * d) : nullptr;
        if (d > 0) copy_in(feat, host, bytes, TK_HOST, c);
        uint8_t* valid = ensure<uint8_t>(k.valid, P);
        int64_t* dscal = ensure<int64_t>(c->dscal, 16);
        tk::launch_gt_valid(feat, P, k.d, valid, dscal + 9, ptr<float>(k.depth), c->cur);
        CK_LAUNCH(c);
        if (c->comm) NK(g_nccl.AllReduce(valid, valid, static_cast<size_t>(P), ncclUint8, ncclMax, c->comm, c->cur));
        tk::copy_words_to_mapped(c->hscal_dev + 9, dscal + 9, 1, c->cur);
        sync(c);
        k.depth_n = c->hscal[9];
        main_done(c);
    });
}

tk_status tk_keyframe_save_features(tk_ctx* c, int32_t slot, const char* path) {
    return guarded([&] {
        if (!c || !path) fail(TK_ERR_BAD_ARG, "null argument");
        if (slot < 0 || static_cast<size_t>(slot) >= c->kfs.size() || c->kfs[slot].w == 0)
            fail(TK_ERR_BAD_ARG, "keyframe_save_features: no keyframe in that slot");
        const Keyframe& k = c->kfs[slot];
        const int64_t P = static_cast<int64_t>(k.w) * k.h;
        const size_t bytes = static_cast<size_t>(P) * (k.has_feature ? k.d : 0) * sizeof(float);
        CK(cudaSetDevice(c->device));
        on_main(c);
        float* host = nullptr;
        CK(cudaHostAlloc(reinterpret_cast<void**>(&host), std::max<size_t>(bytes, 4), cudaHostAllocDefault));
        struct HostFree {
            float* p;
            ~HostFree() { cudaFreeHost(p); }
        } hf{host};
        if (bytes) copy_out(host, ptr<float>(k.feature), bytes, TK_HOST, c);
        sync(c);
        std::FILE* fp = std::fopen(path, "wb");
        if (!fp) fail(TK_ERR_BAD_ARG, std::string("dataset: cannot open ") + path + " for writing");
        const uint32_t hdr[3] = {static_cast<uint32_t>(k.h), static_cast<uint32_t>(k.w),
                                 static_cast<uint32_t>(k.has_feature ? k.d : 0)};
        const bool ok = std::fwrite(kFeatMagic, 1, 4, fp) == 4 && std::fwrite(hdr, 4, 3, fp) == 3 &&
                        std::fwrite(host, 1, bytes, fp) == bytes;
        const bool closed = std::fclose(fp) == 0;
        if (!ok || !closed) fail(TK_ERR_BAD_ARG, std::string("dataset: write failed for ") + path);
        main_done(c);
    });
}

tk_status tk_checkpoint_save(tk_ctx* c, const char* path) {
    return guarded([&] {
        if (!c || !path) fail(TK_ERR_BAD_ARG, "null argument");
        if (!c->has_scene) fail(TK_ERR_STATE, "no scene uploaded (tk_scene_upload)");
        if (c->d > 0 && !c->has_features) fail(TK_ERR_STATE, "scene has no features uploaded");
        CK(cudaSetDevice(c->device));
        on_main(c);
        flush_features(c);  // lazily optimised feature rows must be current
        const int64_t n = c->n;
        const int64_t W = 14 + c->d;
        DevBuf rec;
        float* drec = ensure<float>(rec, n * W);
        tk::launch_splf_pack(splf_view(c), drec, c->cur);
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
        flush_features(c);  // lazily optimised feature rows must be current
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
        } else {
            tk::launch_segment_query(q, st);
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

// fslam_raster.hpp — C++ mirror of the reference renderer API over the C ABI (tk_render.h).
//
// Drop-in for proj/include/fslam/raster/render.hpp + backward.hpp: the same type names, field
// names, defaults and function signatures (Eigen replaced by small POD vectors), the same
// pure-function semantics (every call sees the map as passed) and the same error behaviour (a
// stale Top-K record throws std::runtime_error with the reference's message).  All work runs in
// libtkrender.so on the GPU; there is no CPU fallback.
//
// Reference interface -> this header
//   render.hpp:14-21   RenderSettings            render.hpp:27-44  TopKGrid
//   render.hpp:46-55   RenderOutput              render.hpp:60-71  render_geometric /
//   render.hpp:84-92   raster_detail::PreparedScene                 render_feature /
//   backward.hpp:15-22 GeomGrads                                    render_feature_full_blend
//   backward.hpp:27-34 backward_geometric / backward_feature
//   core/types.hpp     CameraIntrinsics, Gaussian3D   core/image.hpp Image<T>   core/pose.hpp Pose
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "tk_render.h"

namespace tk {
namespace fslam {

struct Vec3 {
    double x = 0, y = 0, z = 0;
};
struct Quat {  // (w, x, y, z)
    double w = 1, x = 0, y = 0, z = 0;
};

inline double logistic(double x) { return 1.0 / (1.0 + std::exp(-x)); }  // types.hpp:12
inline double logit(double p) { return std::log(p / (1.0 - p)); }

struct CameraIntrinsics {  // types.hpp:15-21
    double fx = 0, fy = 0;
    double cx = 0, cy = 0;
    int width = 0, height = 0;
    double near_plane = 0.05;
    double far_plane = 100.0;
};

struct Pose {  // pose.hpp:11-19 (world-to-camera)
    Quat rotation;
    Vec3 translation;
    static Pose identity() { return {}; }
};

struct Gaussian3D {  // types.hpp:25-44
    Vec3 mean;
    Vec3 log_scale;
    Quat rotation;
    double opacity_logit = 0.0;
    Vec3 color;
    std::vector<double> feature;  // unit L2 norm
    int topk_count = 0;
    double max_contribution = 0.0;
    double opacity() const { return logistic(opacity_logit); }
};

struct SceneMap {  // scene_map.hpp:16-27
    std::vector<Gaussian3D> gaussians;
    std::uint64_t generation = 0;
    int feature_dim = 0;
    // Not in the reference: edit counters for the device mirror's UploadPolicy::kVersioned.  A
    // caller that edits parameters in place (optimize_step's Adam, mapper.cpp:183-252) bumps
    // geometry_version / feature_version; structural edits bump generation as in the reference.
    std::uint64_t geometry_version = 0;
    std::uint64_t feature_version = 0;
    std::size_t size() const { return gaussians.size(); }
    bool empty() const { return gaussians.empty(); }
};

template <typename T>
struct Image {  // image.hpp:10-34, H x W x C, channel fastest
    int width = 0, height = 0, channels = 1;
    std::vector<T> data;
    Image() = default;
    Image(int w, int h, int c, T fill = T{})
        : width(w), height(h), channels(c), data(static_cast<std::size_t>(w) * h * c, fill) {}
    bool empty() const { return data.empty(); }
    std::size_t pixel_count() const { return static_cast<std::size_t>(width) * height; }
    std::size_t offset(int x, int y, int c = 0) const {
        return (static_cast<std::size_t>(y) * width + x) * channels + c;
    }
    T& at(int x, int y, int c = 0) { return data[offset(x, y, c)]; }
    const T& at(int x, int y, int c = 0) const { return data[offset(x, y, c)]; }
};
using ImageD = Image<double>;
using ImageF = Image<float>;

struct RenderSettings {  // render.hpp:14-21
    int top_k = 3;
    double transmittance_floor = 1e-4;
    Vec3 background;
    int tile_size = 16;
    double cov2d_dilation = 0.3;
    double alpha_clamp = 0.999;
};

inline constexpr int kMaxTopK = 32;  // render.hpp:23

struct TopKGrid {  // render.hpp:27-44
    int width = 0, height = 0, k = 0;
    std::vector<std::int32_t> index;
    std::vector<double> weight;
    std::vector<std::uint8_t> count;
    // Not in the reference: set by Renderer::render_geometric to name the records the context
    // still holds on the device, so render_feature / backward_feature on this grid skip the
    // host -> device copy of index / weight / count.  Records are treated as the immutable value
    // outputs they are in the reference; a grid built or edited by hand must keep device_token 0.
    std::uint64_t device_token = 0;
    TopKGrid() = default;
    TopKGrid(int w, int h, int kk)
        : width(w), height(h), k(kk), index(static_cast<std::size_t>(w) * h * kk, -1),
          weight(static_cast<std::size_t>(w) * h * kk, 0.0), count(static_cast<std::size_t>(w) * h, 0) {}
    std::size_t slot(int x, int y, int j) const { return (static_cast<std::size_t>(y) * width + x) * k + j; }
    std::size_t pixel(int x, int y) const { return static_cast<std::size_t>(y) * width + x; }
};

struct RenderOutput {  // render.hpp:46-55
    ImageD color, depth, alpha, feature;
    TopKGrid topk;
    std::vector<double> contributions;
    std::uint64_t generation = 0;
    std::size_t map_size = 0;
};

struct GeomGrads {  // backward.hpp:15-22; rotation gradient order (w, x, y, z)
    std::vector<Vec3> mean, log_scale;
    std::vector<Quat> rotation;
    std::vector<double> opacity_logit;
    std::vector<Vec3> color;
    double pose_twist[6] = {0, 0, 0, 0, 0, 0};
};

namespace raster_detail {
struct ProjEntry {  // render.hpp:75-81
    double mx, my, ixx, ixy, iyy, z, opacity;
    std::int32_t src;
};
struct PreparedScene {  // render.hpp:84-92
    std::vector<ProjEntry> entries;
    std::vector<std::int32_t> tile_offsets;
    std::vector<std::int32_t> tile_entries;
    int tiles_x = 0, tiles_y = 0, width = 0, height = 0;
    std::uint64_t generation = 0;
    std::size_t map_size = 0;
};
inline constexpr double kLogWeightCutoff = -27.631021115928547;  // render.hpp:97
}  // namespace raster_detail

namespace detail {
inline void check(tk_status s) {
    if (s != TK_OK) throw std::runtime_error(tk_last_error());
}
inline tk_pose to_c(const Pose& p) {
    return {p.rotation.w, p.rotation.x, p.rotation.y, p.rotation.z,
            p.translation.x, p.translation.y, p.translation.z};
}
inline tk_camera to_c(const CameraIntrinsics& c) {
    return {c.fx, c.fy, c.cx, c.cy, c.width, c.height, c.near_plane, c.far_plane};
}
inline tk_settings to_c(const RenderSettings& s) {
    tk_settings o;
    o.top_k = s.top_k;
    o.tile_size = s.tile_size;
    o.transmittance_floor = s.transmittance_floor;
    o.background[0] = s.background.x;
    o.background[1] = s.background.y;
    o.background[2] = s.background.z;
    o.cov2d_dilation = s.cov2d_dilation;
    o.alpha_clamp = s.alpha_clamp;
    return o;
}
}  // namespace detail

// Upload policy of the device mirror.
//   kAlways    (default): the reference's pure semantics -- every entry point copies the parts of the
//              map it reads (geometry for prepare / render_geometric / backward_geometric, features
//              for render_feature, both for the full blend; backward_feature reads only the map's
//              size and feature_dim), so in-place edits between calls are always seen.
//   kVersioned: a part is copied only when (generation, size, feature_dim, its version counter)
//              differs from the copy on the device (the mirror keyed by
//              SceneMap::generation plus explicit dirty counters).  The caller bumps
//              SceneMap::geometry_version / feature_version after in-place edits.
enum class UploadPolicy { kAlways, kVersioned };

// One device context with a resident copy of the last map it was given.  Host staging is pinned
// (tk_host_alloc) and packed by several threads for large maps.
class Renderer {
public:
    explicit Renderer(int device = 0, UploadPolicy policy = UploadPolicy::kAlways) : policy_(policy) {
        detail::check(tk_create(device, &ctx_));
    }
    ~Renderer() {
        tk_destroy(ctx_);
        for (auto& b : pinned_) tk_host_free(b.p);
    }
    Renderer(const Renderer&) = delete;
    Renderer& operator=(const Renderer&) = delete;
    tk_ctx* context() const { return ctx_; }
    void set_policy(UploadPolicy p) { policy_ = p; }
    // bytes copied host -> device for the map so far (geometry, features) -- the boundary's cost
    std::uint64_t geometry_bytes_uploaded() const { return geo_bytes_; }
    std::uint64_t feature_bytes_uploaded() const { return feat_bytes_; }
    void invalidate() { geo_key_.valid = feat_key_.valid = false; }

    // Whole map (geometry + features), as before: kept for callers that want one explicit upload.
    void upload(const SceneMap& m) {
        sync_geometry(m, true);
        sync_features(m, true);
    }

    // The geometry half: SoA fp64 mean / log_scale / rotation / opacity_logit / color.
    void sync_geometry(const SceneMap& m, bool force = false) {
        const std::size_t n = m.size();
        const int d = m.feature_dim;
        const Key key{m.generation, n, d, m.geometry_version, true};
        if (!force && policy_ == UploadPolicy::kVersioned && key == geo_key_) return;
        double* mean = stage<double>(0, n * 3);
        double* ls = stage<double>(1, n * 3);
        double* rot = stage<double>(2, n * 4);
        double* op = stage<double>(3, n);
        double* col = stage<double>(4, n * 3);
        parallel_rows(n, n * 14, [&](std::size_t i0, std::size_t i1) {
            for (std::size_t i = i0; i < i1; ++i) {
                const Gaussian3D& g = m.gaussians[i];
                mean[i * 3 + 0] = g.mean.x;
                mean[i * 3 + 1] = g.mean.y;
                mean[i * 3 + 2] = g.mean.z;
                ls[i * 3 + 0] = g.log_scale.x;
                ls[i * 3 + 1] = g.log_scale.y;
                ls[i * 3 + 2] = g.log_scale.z;
                rot[i * 4 + 0] = g.rotation.w;
                rot[i * 4 + 1] = g.rotation.x;
                rot[i * 4 + 2] = g.rotation.y;
                rot[i * 4 + 3] = g.rotation.z;
                op[i] = g.opacity_logit;
                col[i * 3 + 0] = g.color.x;
                col[i * 3 + 1] = g.color.y;
                col[i * 3 + 2] = g.color.z;
            }
        });
        // a new size or feature_dim invalidates the resident features: ship them in the same call
        const bool reshape = !dev_shape_valid_ || dev_n_ != n || dev_d_ != d;
        const float* feat = nullptr;
        if (reshape) {
            feat = pack_features(m);
            feat_key_ = Key{m.generation, n, d, m.feature_version, true};
            feat_bytes_ += n * static_cast<std::uint64_t>(d) * sizeof(float);
        }
        tk_scene_view v{static_cast<int64_t>(n), d, mean, ls, rot, op, col, feat, m.generation};
        detail::check(tk_scene_upload(ctx_, &v, TK_HOST));
        geo_bytes_ += n * 14 * sizeof(double);
        geo_key_ = key;
        dev_shape_valid_ = true;
        dev_n_ = n;
        dev_d_ = d;
    }

    // The feature half: fp32 rows N x D (the reference's unit-norm fp64 features, rounded once).
    void sync_features(const SceneMap& m, bool force = false) {
        const std::size_t n = m.size();
        const int d = m.feature_dim;
        if (!dev_shape_valid_ || dev_n_ != n || dev_d_ != d) {
            sync_geometry(m, true);  // ships the features with the new shape
            return;
        }
        const Key key{m.generation, n, d, m.feature_version, true};
        if (!force && policy_ == UploadPolicy::kVersioned && key == feat_key_) return;
        const float* feat = pack_features(m);
        detail::check(tk_scene_upload_features(ctx_, static_cast<int64_t>(n), d, feat, TK_HOST));
        feat_bytes_ += n * static_cast<std::uint64_t>(d) * sizeof(float);
        feat_key_ = key;
    }

    // Only the map's size and feature_dim on the device (backward_feature).
    void sync_shape(const SceneMap& m) {
        if (!dev_shape_valid_ || dev_n_ != m.size() || dev_d_ != m.feature_dim) sync_geometry(m, true);
    }

    raster_detail::PreparedScene prepare_scene(const SceneMap& m, const Pose& pose, const CameraIntrinsics& cam,
                                               const RenderSettings& s) {
        sync_geometry(m);
        const tk_pose p = detail::to_c(pose);
        const tk_camera c = detail::to_c(cam);
        const tk_settings st = detail::to_c(s);
        int64_t ne = 0, nt = 0;
        int32_t tx = 0, ty = 0;
        detail::check(tk_prepare_scene(ctx_, &p, &c, &st, &ne, &nt, &tx, &ty));
        std::vector<double> e7(static_cast<std::size_t>(ne) * 7);
        std::vector<int32_t> src(static_cast<std::size_t>(ne));
        raster_detail::PreparedScene out;
        out.tile_offsets.resize(static_cast<std::size_t>(tx) * ty + 1);
        out.tile_entries.resize(static_cast<std::size_t>(nt));
        detail::check(tk_prepared_export(ctx_, e7.data(), src.data(), out.tile_offsets.data(), out.tile_entries.data()));
        out.entries.resize(static_cast<std::size_t>(ne));
        for (int64_t q = 0; q < ne; ++q)
            out.entries[q] = {e7[q * 7 + 0], e7[q * 7 + 1], e7[q * 7 + 2], e7[q * 7 + 3],
                              e7[q * 7 + 4], e7[q * 7 + 5], e7[q * 7 + 6], src[q]};
        out.tiles_x = tx;
        out.tiles_y = ty;
        out.width = cam.width;
        out.height = cam.height;
        out.generation = m.generation;
        out.map_size = m.size();
        return out;
    }

    RenderOutput render_geometric(const SceneMap& m, const Pose& pose, const CameraIntrinsics& cam,
                                  const RenderSettings& s) {  // render.cpp:293-299
        sync_geometry(m);
        const int w = cam.width, h = cam.height, k = std::min(std::max(s.top_k, 0), kMaxTopK);
        RenderOutput out;
        out.color = ImageD(w, h, 3);
        out.depth = ImageD(w, h, 1);
        out.alpha = ImageD(w, h, 1);
        out.topk = TopKGrid(w, h, k);
        out.contributions.assign(m.size(), 0.0);
        tk_geom_out g{TK_HOST, out.color.data.data(), out.depth.data.data(), out.alpha.data.data(),
                      out.topk.index.data(), out.topk.weight.data(), out.topk.count.data(),
                      out.contributions.data(), 0, 0};
        const tk_pose p = detail::to_c(pose);
        const tk_camera c = detail::to_c(cam);
        const tk_settings st = detail::to_c(s);
        detail::check(tk_render_geometric(ctx_, &p, &c, &st, &g));
        out.generation = g.generation;
        out.map_size = static_cast<std::size_t>(g.map_size);
        out.topk.device_token = records_token_ = ++token_seq_;  // the context now holds these records
        return out;
    }

    ImageD render_feature(const SceneMap& m, const TopKGrid& t) {  // render.cpp:301-337
        sync_features(m);
        const std::size_t nf = static_cast<std::size_t>(t.width) * t.height * m.feature_dim;
        float* f = stage<float>(7, nf);  // pinned: the read-back runs at the full PCIe rate
        tk_topk_view v{t.width, t.height, t.k, t.index.data(), t.weight.data(), t.count.data(), TK_HOST};
        detail::check(tk_render_feature(ctx_, resident(t) ? nullptr : &v, f, TK_HOST));
        ImageD out(t.width, t.height, m.feature_dim);
        widen(f, nf, out.data);
        return out;
    }

    ImageD render_feature_full_blend(const SceneMap& m, const Pose& pose, const CameraIntrinsics& cam,
                                     const RenderSettings& s) {  // render.cpp:339-343
        sync_geometry(m);
        sync_features(m);
        const std::size_t nf = static_cast<std::size_t>(cam.width) * cam.height * m.feature_dim;
        float* f = stage<float>(7, nf);
        const tk_pose p = detail::to_c(pose);
        const tk_camera c = detail::to_c(cam);
        const tk_settings st = detail::to_c(s);
        detail::check(tk_render_feature_full_blend(ctx_, &p, &c, &st, f, TK_HOST));
        ImageD out(cam.width, cam.height, m.feature_dim);
        widen(f, nf, out.data);
        return out;
    }

    std::vector<double> backward_feature(const SceneMap& m, const TopKGrid& t,
                                         const ImageD& grad_feature) {  // backward.cpp:273-321
        sync_shape(m);
        float* g = stage<float>(6, grad_feature.data.size());
        const double* gs = grad_feature.data.data();
        parallel_rows(grad_feature.data.size(), grad_feature.data.size(), [&](std::size_t i0, std::size_t i1) {
            for (std::size_t i = i0; i < i1; ++i) g[i] = static_cast<float>(gs[i]);
        });
        const std::size_t no = m.size() * static_cast<std::size_t>(m.feature_dim);
        float* o = stage<float>(8, no);
        tk_topk_view v{t.width, t.height, t.k, t.index.data(), t.weight.data(), t.count.data(), TK_HOST};
        detail::check(tk_backward_feature(ctx_, resident(t) ? nullptr : &v, g, TK_HOST, o, TK_HOST));
        std::vector<double> out(no);
        widen(o, no, out);
        return out;
    }

    GeomGrads backward_geometric(const SceneMap& m, const Pose& pose, const CameraIntrinsics& cam,
                                 const RenderSettings& s, const ImageD& grad_color,
                                 const ImageD& grad_depth) {  // backward.cpp:72-271
        sync_geometry(m);
        const std::size_t n = m.size();
        double* gm = stage<double>(9, n * 3);
        double* gl = stage<double>(10, n * 3);
        double* gr = stage<double>(11, n * 4);
        double* go = stage<double>(12, n);
        double* gc = stage<double>(13, n * 3);
        tk_geom_grads out{TK_HOST, gm, gl, gr, go, gc, {0, 0, 0, 0, 0, 0}};
        const tk_pose p = detail::to_c(pose);
        const tk_camera c = detail::to_c(cam);
        const tk_settings st = detail::to_c(s);
        detail::check(tk_backward_geometric(ctx_, &p, &c, &st, grad_color.data.data(),
                                            grad_depth.empty() ? nullptr : grad_depth.data.data(), TK_HOST, &out));
        GeomGrads g;
        g.mean.resize(n);
        g.log_scale.resize(n);
        g.rotation.resize(n);
        g.opacity_logit.assign(go, go + n);
        g.color.resize(n);
        parallel_rows(n, n * 14, [&](std::size_t i0, std::size_t i1) {
            for (std::size_t i = i0; i < i1; ++i) {
                g.mean[i] = {gm[i * 3], gm[i * 3 + 1], gm[i * 3 + 2]};
                g.log_scale[i] = {gl[i * 3], gl[i * 3 + 1], gl[i * 3 + 2]};
                g.rotation[i] = {gr[i * 4], gr[i * 4 + 1], gr[i * 4 + 2], gr[i * 4 + 3]};
                g.color[i] = {gc[i * 3], gc[i * 3 + 1], gc[i * 3 + 2]};
            }
        });
        for (int a = 0; a < 6; ++a) g.pose_twist[a] = out.pose_twist[a];
        return g;
    }

private:
    struct Key {
        std::uint64_t generation = 0;
        std::size_t n = 0;
        int d = 0;
        std::uint64_t version = 0;
        bool valid = false;
        bool operator==(const Key& o) const {
            return valid && o.valid && generation == o.generation && n == o.n && d == o.d && version == o.version;
        }
    };
    struct Pinned {
        void* p = nullptr;
        std::size_t bytes = 0;
    };

    template <class T>
    T* stage(int slot, std::size_t count) {  // pinned staging buffer `slot`, grown on demand
        if (pinned_.size() <= static_cast<std::size_t>(slot)) pinned_.resize(slot + 1);
        Pinned& b = pinned_[slot];
        const std::size_t need = std::max<std::size_t>(count, 1) * sizeof(T);
        if (b.bytes < need) {
            if (b.p) tk_host_free(b.p);
            b.p = nullptr;
            b.bytes = 0;
            detail::check(tk_host_alloc(need, &b.p));
            b.bytes = need;
        }
        return static_cast<T*>(b.p);
    }

    const float* pack_features(const SceneMap& m) {
        const std::size_t n = m.size();
        const int d = m.feature_dim;
        float* f = stage<float>(5, n * static_cast<std::size_t>(d));
        parallel_rows(n, n * static_cast<std::size_t>(d), [&](std::size_t i0, std::size_t i1) {
            for (std::size_t i = i0; i < i1; ++i) {
                const std::vector<double>& src = m.gaussians[i].feature;
                const int c1 = std::min<int>(d, static_cast<int>(src.size()));
                float* row = f + i * static_cast<std::size_t>(d);
                for (int c = 0; c < c1; ++c) row[c] = static_cast<float>(src[c]);
                for (int c = c1; c < d; ++c) row[c] = 0.0f;
            }
        });
        return f;
    }

    // rows [0, n) split over the host's threads when the copy is large (>= 4M elements)
    template <class F>
    static void parallel_rows(std::size_t n, std::size_t elems, F&& fn) {
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        const unsigned t = elems < (std::size_t(1) << 22) ? 1u : std::min<unsigned>(hw, 32u);
        if (t <= 1 || n < t) {
            fn(std::size_t(0), n);
            return;
        }
        std::vector<std::thread> pool;
        const std::size_t step = (n + t - 1) / t;
        for (unsigned k = 0; k < t; ++k) {
            const std::size_t i0 = std::min(n, k * step), i1 = std::min(n, i0 + step);
            if (i0 < i1) pool.emplace_back([&fn, i0, i1] { fn(i0, i1); });
        }
        for (auto& th : pool) th.join();
    }

    static void widen(const float* f, std::size_t n, std::vector<double>& d) {  // fp32 results -> fp64 API
        parallel_rows(n, n, [&](std::size_t i0, std::size_t i1) {
            for (std::size_t i = i0; i < i1; ++i) d[i] = f[i];
        });
    }

    bool resident(const TopKGrid& t) const { return t.device_token != 0 && t.device_token == records_token_; }

    tk_ctx* ctx_ = nullptr;
    UploadPolicy policy_ = UploadPolicy::kAlways;
    std::vector<Pinned> pinned_;
    Key geo_key_, feat_key_;
    bool dev_shape_valid_ = false;
    std::size_t dev_n_ = 0;
    int dev_d_ = 0;
    std::uint64_t geo_bytes_ = 0, feat_bytes_ = 0;
    std::uint64_t records_token_ = 0, token_seq_ = 0;
};

// Free functions with the reference signatures, on a per-thread default context (device 0).
inline Renderer& default_renderer() {
    thread_local std::unique_ptr<Renderer> r;
    if (!r) r = std::make_unique<Renderer>(0);
    return *r;
}
inline RenderOutput render_geometric(const SceneMap& m, const Pose& p, const CameraIntrinsics& c,
                                     const RenderSettings& s) {
    return default_renderer().render_geometric(m, p, c, s);
}
inline ImageD render_feature(const SceneMap& m, const TopKGrid& t) { return default_renderer().render_feature(m, t); }
inline ImageD render_feature_full_blend(const SceneMap& m, const Pose& p, const CameraIntrinsics& c,
                                       const RenderSettings& s) {
    return default_renderer().render_feature_full_blend(m, p, c, s);
}
inline std::vector<double> backward_feature(const SceneMap& m, const TopKGrid& t, const ImageD& g) {
    return default_renderer().backward_feature(m, t, g);
}
inline GeomGrads backward_geometric(const SceneMap& m, const Pose& p, const CameraIntrinsics& c,
                                    const RenderSettings& s, const ImageD& gc, const ImageD& gd) {
    return default_renderer().backward_geometric(m, p, c, s, gc, gd);
}
namespace raster_detail {
inline PreparedScene prepare_scene(const SceneMap& m, const Pose& p, const CameraIntrinsics& c,
                                   const RenderSettings& s) {
    return default_renderer().prepare_scene(m, p, c, s);
}
}  // namespace raster_detail

}  // namespace fslam
}  // namespace tk

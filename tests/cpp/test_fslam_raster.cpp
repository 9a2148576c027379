// test_fslam_raster.cpp — the reference's raster tests (proj/tests/test_raster.cpp,
// test_backward.cpp) written against the C++ mirror include/tk/fslam_raster.hpp, plus parity with
// the CPU oracle (oracle/include/oracle.h; test infrastructure) through the same C++ types.
// Built and run by tests/test_cpp_api.py on a GPU box.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "oracle.h"
#include "tk/fslam_raster.hpp"
#include "tk_synth.h"

using namespace tk::fslam;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                                  \
    do {                                                                             \
        ++g_checks;                                                                  \
        if (!(cond)) {                                                               \
            ++g_fail;                                                                \
            std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);              \
        }                                                                            \
    } while (0)
#define CHECK_NEAR(a, b, tol) CHECK(std::fabs((a) - (b)) <= (tol))

static CameraIntrinsics centered_camera(int side, double focal) {  // test_raster.cpp:17-25
    CameraIntrinsics c;
    c.width = c.height = side;
    c.fx = c.fy = focal;
    c.cx = c.cy = static_cast<double>(side / 2);
    c.near_plane = 0.05;
    c.far_plane = 50.0;
    return c;
}

static CameraIntrinsics test_camera(int w, int h) {  // testutil.hpp:55-65
    CameraIntrinsics c;
    c.width = w;
    c.height = h;
    c.fx = c.fy = 0.9 * w;
    c.cx = 0.5 * (w - 1);
    c.cy = 0.5 * (h - 1);
    c.near_plane = 0.05;
    c.far_plane = 50.0;
    return c;
}

// flat_gaussian (test_raster.cpp:27-37).  The reference KATs use log_scale 1.0, which the
// reference's own projection cull (projection.cpp:19-20) removes; -2.0 keeps the centre answers.
static Gaussian3D flat_gaussian(Vec3 mean, double opacity, Vec3 color, double ls, int d = 2) {
    Gaussian3D g;
    g.mean = mean;
    g.log_scale = {ls, ls, ls};
    g.opacity_logit = logit(opacity);
    g.color = color;
    g.feature.assign(d, 0.0);
    g.feature[0] = 1.0;
    return g;
}

static SceneMap random_scene(int n, int d, uint64_t seed) {  // testutil.hpp:31-53
    std::vector<double> mean(n * 3), ls(n * 3), rot(n * 4), op(n), col(n * 3), feat(static_cast<size_t>(n) * d);
    tk_synth_arrays a{n, d, mean.data(), ls.data(), rot.data(), op.data(), col.data(), feat.data()};
    tk_synth_random_scene(n, d, seed, 0.8, 6.0, &a);
    SceneMap m;
    m.feature_dim = d;
    for (int i = 0; i < n; ++i) {
        Gaussian3D g;
        g.mean = {mean[i * 3], mean[i * 3 + 1], mean[i * 3 + 2]};
        g.log_scale = {ls[i * 3], ls[i * 3 + 1], ls[i * 3 + 2]};
        g.rotation = {rot[i * 4], rot[i * 4 + 1], rot[i * 4 + 2], rot[i * 4 + 3]};
        g.opacity_logit = op[i];
        g.color = {col[i * 3], col[i * 3 + 1], col[i * 3 + 2]};
        g.feature.assign(feat.begin() + static_cast<long>(i) * d, feat.begin() + static_cast<long>(i + 1) * d);
        m.gaussians.push_back(g);
    }
    return m;
}

// The same map in the oracle's C ABI.
struct OracleMap {
    orc_map* h = nullptr;
    explicit OracleMap(const SceneMap& m) {
        const size_t n = m.size();
        const int d = m.feature_dim;
        std::vector<double> mean(n * 3), ls(n * 3), rot(n * 4), op(n), col(n * 3), feat(n * d);
        for (size_t i = 0; i < n; ++i) {
            const Gaussian3D& g = m.gaussians[i];
            mean[i * 3] = g.mean.x; mean[i * 3 + 1] = g.mean.y; mean[i * 3 + 2] = g.mean.z;
            ls[i * 3] = g.log_scale.x; ls[i * 3 + 1] = g.log_scale.y; ls[i * 3 + 2] = g.log_scale.z;
            rot[i * 4] = g.rotation.w; rot[i * 4 + 1] = g.rotation.x; rot[i * 4 + 2] = g.rotation.y;
            rot[i * 4 + 3] = g.rotation.z;
            op[i] = g.opacity_logit;
            col[i * 3] = g.color.x; col[i * 3 + 1] = g.color.y; col[i * 3 + 2] = g.color.z;
            for (int c = 0; c < d; ++c) feat[i * d + c] = g.feature[c];
        }
        h = orc_map_create(static_cast<int64_t>(n), d, mean.data(), ls.data(), rot.data(), op.data(), col.data(),
                           feat.data(), m.generation);
    }
    ~OracleMap() { orc_map_free(h); }
};

static orc_settings orc(const RenderSettings& s) {
    orc_settings o;
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

int main() {
    Renderer r(0);
    {  // empty map renders the background (test_raster.cpp:41-58)
        SceneMap m;
        m.feature_dim = 2;
        RenderSettings s;
        s.background = {0.2, 0.4, 0.6};
        const RenderOutput o = r.render_geometric(m, Pose::identity(), centered_camera(32, 40.0), s);
        CHECK_NEAR(o.color.at(5, 7, 0), 0.2, 1e-15);
        CHECK_NEAR(o.color.at(31, 31, 2), 0.6, 1e-15);
        CHECK(o.depth.at(3, 3) == 0.0 && o.alpha.at(3, 3) == 0.0 && o.topk.count[o.topk.pixel(3, 3)] == 0);
    }
    {  // single gaussian blends one term (test_raster.cpp:60-77)
        SceneMap m;
        m.feature_dim = 2;
        m.gaussians.push_back(flat_gaussian({0, 0, 2}, 0.5, {1, 0, 0}, -2.0));
        const RenderOutput o = r.render_geometric(m, Pose::identity(), centered_camera(33, 16.0), RenderSettings{});
        CHECK_NEAR(o.color.at(16, 16, 0), 0.5, 1e-12);
        CHECK_NEAR(o.depth.at(16, 16), 1.0, 1e-12);
        CHECK_NEAR(o.alpha.at(16, 16), 0.5, 1e-12);
        CHECK_NEAR(o.contributions[0], 0.5, 1e-12);
    }
    {  // two on-axis gaussians (test_raster.cpp:79-100)
        SceneMap m;
        m.feature_dim = 2;
        m.gaussians.push_back(flat_gaussian({0, 0, 1}, 0.6, {1, 0, 0}, -2.0));
        m.gaussians.push_back(flat_gaussian({0, 0, 2}, 0.8, {0, 1, 0}, -2.0));
        RenderSettings s;
        s.transmittance_floor = 0.0;
        const RenderOutput o = r.render_geometric(m, Pose::identity(), centered_camera(33, 16.0), s);
        CHECK_NEAR(o.color.at(16, 16, 0), 0.6, 1e-9);
        CHECK_NEAR(o.color.at(16, 16, 1), 0.32, 1e-9);
        CHECK_NEAR(o.depth.at(16, 16), 1.24, 1e-9);
    }
    {  // renormalisation KAT + stale index (test_raster.cpp:208-253)
        SceneMap m;
        m.feature_dim = 3;
        m.gaussians.push_back(flat_gaussian({0, 0, 1}, 0.5, {1, 0, 0}, -2.0, 3));
        m.gaussians.push_back(flat_gaussian({0, 0, 2}, 0.5, {0, 1, 0}, -2.0, 3));
        m.gaussians[1].feature = {0, 1, 0};
        TopKGrid grid(1, 1, 2);
        grid.count[0] = 2;
        grid.index = {0, 1};
        grid.weight = {0.3, 0.1};
        const ImageD f = r.render_feature(m, grid);
        CHECK_NEAR(f.at(0, 0, 0), 0.75, 1e-6);
        CHECK_NEAR(f.at(0, 0, 1), 0.25, 1e-6);
        TopKGrid stale(1, 1, 1);
        stale.count[0] = 1;
        stale.index[0] = 5;
        stale.weight[0] = 0.5;
        bool threw = false;
        try {
            r.render_feature(m, stale);
        } catch (const std::runtime_error& e) {
            threw = std::string(e.what()) ==
                    "render_feature: top-k record references gaussian 5 but the map holds 2 (stale snapshot)";
        }
        CHECK(threw);
    }
    {  // tiled GPU render == oracle render (indices exact), tile-size independence
        const SceneMap m = random_scene(400, 8, 3);
        const CameraIntrinsics cam = test_camera(64, 48);
        RenderSettings s;
        s.background = {0.1, 0.2, 0.3};
        const RenderOutput a = r.render_geometric(m, Pose::identity(), cam, s);
        RenderSettings s8 = s;
        s8.tile_size = 8;
        const RenderOutput b = r.render_geometric(m, Pose::identity(), cam, s8);
        CHECK(a.topk.index == b.topk.index);
        CHECK(std::memcmp(a.color.data.data(), b.color.data.data(), a.color.data.size() * 8) == 0);
        OracleMap om(m);
        const size_t P = 64 * 48;
        std::vector<double> color(P * 3), depth(P), alpha(P), weight(P * 3), contrib(m.size());
        std::vector<int32_t> index(P * 3);
        std::vector<uint8_t> count(P);
        const tk_pose p = tk::fslam::detail::to_c(Pose::identity());
        const orc_pose op{p.qw, p.qx, p.qy, p.qz, p.tx, p.ty, p.tz};
        const orc_camera oc{cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height, cam.near_plane, cam.far_plane};
        const orc_settings os = orc(s);
        orc_render_geometric(om.h, &op, &oc, &os, color.data(), depth.data(), alpha.data(), index.data(), weight.data(),
                             count.data(), contrib.data());
        CHECK(a.topk.index == index);
        CHECK(a.topk.count == count);
        double err = 0.0;
        for (size_t i = 0; i < color.size(); ++i) err = std::max(err, std::fabs(color[i] - a.color.data[i]));
        CHECK(err < 1e-9);
        // feature forward / backward vs the oracle
        const ImageD f = r.render_feature(m, a.topk);
        std::vector<double> fo(P * 8);
        orc_render_feature(om.h, 64, 48, 3, index.data(), weight.data(), count.data(), fo.data());
        double ferr = 0.0;
        for (size_t i = 0; i < fo.size(); ++i) ferr = std::max(ferr, std::fabs(fo[i] - f.data[i]));
        CHECK(ferr < 1e-5);
        ImageD gf(64, 48, 8);
        for (size_t i = 0; i < gf.data.size(); ++i) gf.data[i] = std::sin(0.37 * static_cast<double>(i));
        const std::vector<double> df = r.backward_feature(m, a.topk, gf);
        std::vector<double> dfo(m.size() * 8);
        orc_backward_feature(om.h, 64, 48, 3, index.data(), weight.data(), count.data(), gf.data.data(), dfo.data());
        double berr = 0.0;
        for (size_t i = 0; i < dfo.size(); ++i) berr = std::max(berr, std::fabs(dfo[i] - df[i]));
        CHECK(berr < 1e-4);
    }
    {  // backward: zero upstream gradients give zero (test_backward.cpp:104-120)
        const SceneMap m = random_scene(10, 3, 4);
        const CameraIntrinsics cam = test_camera(16, 16);
        RenderSettings s;
        s.transmittance_floor = 0.0;
        const GeomGrads g = r.backward_geometric(m, Pose::identity(), cam, s, ImageD(16, 16, 3), ImageD(16, 16, 1));
        double mx = 0.0;
        for (const Vec3& v : g.mean) mx = std::max(mx, std::fabs(v.x) + std::fabs(v.y) + std::fabs(v.z));
        CHECK(mx == 0.0);
        CHECK(g.pose_twist[0] == 0.0 && g.pose_twist[5] == 0.0);
    }
    {  // device mirror: resident records, per-part uploads, the versioned policy
        SceneMap m = random_scene(400, 8, 3);
        const CameraIntrinsics cam = test_camera(64, 48);
        RenderSettings s;
        const RenderOutput a = r.render_geometric(m, Pose::identity(), cam, s);
        CHECK(a.topk.device_token != 0);
        TopKGrid host = a.topk;
        host.device_token = 0;  // forces the host -> device copy of the records
        const ImageD f_res = r.render_feature(m, a.topk), f_host = r.render_feature(m, host);
        CHECK(f_res.data == f_host.data);
        ImageD gf(64, 48, 8);
        for (size_t i = 0; i < gf.data.size(); ++i) gf.data[i] = std::cos(0.11 * static_cast<double>(i));
        CHECK(r.backward_feature(m, a.topk, gf) == r.backward_feature(m, host, gf));
        // kAlways sees an in-place edit; kVersioned sees it once the caller bumps the counter
        Renderer rv(0, UploadPolicy::kVersioned);
        const RenderOutput v0 = rv.render_geometric(m, Pose::identity(), cam, s);
        const ImageD fv0 = rv.render_feature(m, v0.topk);
        const uint64_t geo0 = rv.geometry_bytes_uploaded(), feat0 = rv.feature_bytes_uploaded();
        rv.backward_geometric(m, Pose::identity(), cam, s, ImageD(64, 48, 3, 0.5), ImageD(64, 48, 1, 0.25));
        rv.render_feature(m, v0.topk);
        CHECK(rv.geometry_bytes_uploaded() == geo0 && rv.feature_bytes_uploaded() == feat0);  // nothing re-sent
        for (auto& g : m.gaussians) g.feature[0] = -g.feature[0];
        CHECK(r.render_feature(m, a.topk).data != f_res.data);    // kAlways: the edit is seen
        CHECK(rv.render_feature(m, v0.topk).data == fv0.data);    // kVersioned, no bump: resident copy
        m.feature_version += 1;
        CHECK(rv.render_feature(m, v0.topk).data == r.render_feature(m, a.topk).data);
        CHECK(rv.feature_bytes_uploaded() > feat0 && rv.geometry_bytes_uploaded() == geo0);
        m.gaussians[7].mean.x += 0.05;
        m.geometry_version += 1;
        const RenderOutput v1 = rv.render_geometric(m, Pose::identity(), cam, s);
        const RenderOutput a1 = r.render_geometric(m, Pose::identity(), cam, s);
        CHECK(v1.topk.index == a1.topk.index && v1.color.data == a1.color.data);
        CHECK(rv.geometry_bytes_uploaded() > geo0);
        m.gaussians.pop_back();  // structural edit: size change ships both halves
        m.generation += 1;
        const RenderOutput v2 = rv.render_geometric(m, Pose::identity(), cam, s);
        const RenderOutput a2 = r.render_geometric(m, Pose::identity(), cam, s);
        CHECK(v2.topk.index == a2.topk.index && rv.render_feature(m, v2.topk).data == r.render_feature(m, a2.topk).data);
    }
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}

// dropin_mapping.cpp — the drop-in boundary measured the way a reference caller uses it: the
// renderer-call sequence of optimize_step (proj/src/map/mapper.cpp:173-245) at BASELINE config 3
// through the C++ mirror include/tk/fslam_raster.hpp, on the reference's own AoS SceneMap
// (Gaussian3D with a heap std::vector<double> feature per Gaussian) and fp64 Image<double> API.
//
// Per iteration (feature_update_period 5, mapper.hpp:16):
//   render_geometric(map, pose, cam, s)                               mapper.cpp:173
//   render.feature = render_feature(map, render.topk)   feature steps mapper.cpp:174
//   backward_geometric(map, pose, cam, s, grad_color, grad_depth)    mapper.cpp:179-180
//   backward_feature(map, render.topk, grad_feature)    feature steps mapper.cpp:240
// The reference computes the losses and the Adam steps on the host between these calls; they are
// not part of the renderer boundary and are left out here: the upstream gradients are fixed
// seeded images (as in bench.py), and the in-place Adam edits are represented by bumping
// SceneMap::geometry_version every iteration and feature_version after every feature step (what
// a caller using UploadPolicy::kVersioned does).  The device-side mapping iteration that also runs
// losses and Adam on the GPU is tk_optimize_step (bench.py "mapping").
//
// Prints one JSON object per upload policy: iterations/s, and the bytes that crossed PCIe per
// iteration by category.
//   g++ -O2 -std=c++17 -pthread -I include -I scenegen/include scripts/dropin_mapping.cpp \
//       -L paper_2602_06991_b200/lib -ltkrender -L scenegen/lib -ltk_synth -o dropin_mapping
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tk/fslam_raster.hpp"
#include "tk_synth.h"

using namespace tk::fslam;

int main(int argc, char** argv) {
    const int64_t N = argc > 1 ? std::atoll(argv[1]) : 1000000;
    const int W = argc > 2 ? std::atoi(argv[2]) : 1200, H = argc > 3 ? std::atoi(argv[3]) : 680;
    const int D = argc > 4 ? std::atoi(argv[4]) : 512;
    const int iters = argc > 5 ? std::atoi(argv[5]) : 10;
    const int period = 5;

    // the bench recipe scene (fslam_main.cpp:167-196), features seeded unit rows
    tk_synth_spec spec;
    tk_synth_default_spec(&spec);
    spec.seed = 7;
    spec.spacing = std::sqrt(70.0 / static_cast<double>(N));
    spec.feature_dim = D > 4 ? D : 4;
    spec.classes = 4;
    const int64_t total = tk_synth_build_scene(&spec, nullptr, nullptr);
    std::vector<double> mean(total * 3), ls(total * 3), rot(total * 4), op(total), col(total * 3);
    tk_synth_arrays a{total, spec.feature_dim, mean.data(), ls.data(), rot.data(), op.data(), col.data(), nullptr};
    tk_synth_build_scene(&spec, &a, nullptr);
    const int64_t n = total < N ? total : N;
    std::vector<double> feat(static_cast<size_t>(n) * D);
    tk_synth_unit_features(n, D, 7, nullptr, feat.data());
    SceneMap map;
    map.feature_dim = D;
    map.gaussians.resize(n);
    for (int64_t i = 0; i < n; ++i) {
        Gaussian3D& g = map.gaussians[i];
        g.mean = {mean[i * 3], mean[i * 3 + 1], mean[i * 3 + 2]};
        g.log_scale = {ls[i * 3], ls[i * 3 + 1], ls[i * 3 + 2]};
        g.rotation = {rot[i * 4], rot[i * 4 + 1], rot[i * 4 + 2], rot[i * 4 + 3]};
        g.opacity_logit = op[i];
        g.color = {col[i * 3], col[i * 3 + 1], col[i * 3 + 2]};
        g.feature.assign(feat.begin() + i * D, feat.begin() + (i + 1) * D);
    }
    feat.clear();
    feat.shrink_to_fit();
    double pv[8 * 7];
    tk_synth_trajectory(0, 8, &spec, pv);
    Pose pose;
    pose.rotation = {pv[0], pv[1], pv[2], pv[3]};
    pose.translation = {pv[4], pv[5], pv[6]};
    CameraIntrinsics cam;
    cam.fx = cam.fy = 0.9 * W;
    cam.cx = 0.5 * (W - 1);
    cam.cy = 0.5 * (H - 1);
    cam.width = W;
    cam.height = H;
    cam.far_plane = 20.0;
    RenderSettings s;
    ImageD gc(W, H, 3), gd(W, H, 1), gf(W, H, D);
    tk_synth_uniform_fill(static_cast<int64_t>(gc.data.size()), 12, -1.0, 1.0, gc.data.data());
    tk_synth_uniform_fill(static_cast<int64_t>(gd.data.size()), 13, -1.0, 1.0, gd.data.data());
    {
        std::vector<float> tmp(gf.data.size());
        tk_synth_hash_fill_f32(static_cast<int64_t>(tmp.size()), 11, -1.f, 1.f, tmp.data());
        for (size_t i = 0; i < tmp.size(); ++i) gf.data[i] = tmp[i];
    }
    const double P = static_cast<double>(W) * H;

    std::printf("[");
    for (int pol = 0; pol < 2; ++pol) {
        const UploadPolicy policy = pol == 0 ? UploadPolicy::kAlways : UploadPolicy::kVersioned;
        Renderer r(0, policy);
        double call_s[4] = {0, 0, 0, 0};  // render_geometric, render_feature, backward_geometric, backward_feature
        auto timed = [&](int k, auto&& fn) {
            const auto a = std::chrono::steady_clock::now();
            fn();
            call_s[k] += std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count();
        };
        auto iteration = [&](int it) {
            const bool feature_step = it % period == 0;
            RenderOutput render;
            timed(0, [&] { render = r.render_geometric(map, pose, cam, s); });
            if (feature_step) timed(1, [&] { render.feature = r.render_feature(map, render.topk); });
            timed(2, [&] { const GeomGrads g = r.backward_geometric(map, pose, cam, s, gc, gd); });
            map.geometry_version += 1;  // Adam on the five geometry groups (mapper.cpp:183-236)
            if (feature_step) {
                timed(3, [&] { const std::vector<double> fg = r.backward_feature(map, render.topk, gf); });
                map.feature_version += 1;  // feature Adam + renormalise (mapper.cpp:239-252)
            }
        };
        iteration(0);  // warm-up: allocations, first upload of both halves
        for (double& v : call_s) v = 0.0;
        const uint64_t geo0 = r.geometry_bytes_uploaded(), feat0 = r.feature_bytes_uploaded();
        const auto t0 = std::chrono::steady_clock::now();
        for (int it = 1; it <= iters; ++it) iteration(it);
        const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        const double geo = static_cast<double>(r.geometry_bytes_uploaded() - geo0) / iters;
        const double fe = static_cast<double>(r.feature_bytes_uploaded() - feat0) / iters;
        const double fsteps = static_cast<double>(iters / period) / iters;  // feature steps among 1..iters
        // host <-> device bytes of the call outputs / inputs besides the map (per iteration):
        // render_geometric out: colour/depth/alpha fp64, records, contributions; render_feature out
        // (fp32 F); backward_geometric in: dC, dD fp64, out: 14 fp64 per Gaussian; backward_feature
        // in: dF fp32, out: dense N x D fp32.  Records stay resident (TopKGrid::device_token).
        const double io = P * 5 * 8 + P * 3 * 12 + P + n * 8.0 + P * 4 * 8 + n * 14 * 8.0 +
                          fsteps * (P * D * 4.0 + P * D * 4.0 + n * D * 4.0);
        std::printf("%s{\"policy\": \"%s\", \"iterations_per_s\": %.4f, \"ms_per_iteration\": %.3f, \"iterations\": %d, "
                    "\"feature_update_period\": %d, \"geometry_upload_bytes_per_iteration\": %.0f, "
                    "\"feature_upload_bytes_per_iteration\": %.0f, \"other_transfer_bytes_per_iteration\": %.0f, "
                    "\"ms_per_call_type_per_iteration\": {\"render_geometric\": %.2f, \"render_feature\": %.2f, "
                    "\"backward_geometric\": %.2f, \"backward_feature\": %.2f}}",
                    pol ? ", " : "", pol == 0 ? "always" : "versioned", iters / sec, 1000.0 * sec / iters, iters, period,
                    geo, fe, io, 1000.0 * call_s[0] / iters, 1000.0 * call_s[1] / iters, 1000.0 * call_s[2] / iters,
                    1000.0 * call_s[3] / iters);
    }
    std::printf("]\n");
    return 0;
}

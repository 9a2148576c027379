// oracle.cpp — CPU fp64 restatement of the reference raster path.
//
// TEST INFRASTRUCTURE ONLY (see oracle/include/oracle.h).  Every function cites the
// reference file:line it restates (paths relative to /root/reference/proj).  Small dense
// products that the reference evaluates through Eigen are written out with a fixed
// left-to-right summation order; the GPU path follows the same order so that the discrete
// decisions (visibility, sort keys, tile ranges, cutoffs, Top-K) agree bit for bit.
#include "oracle.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

thread_local std::string g_err;

inline int max_threads() {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
inline int thread_id() {
#ifdef _OPENMP
    return omp_get_thread_num();
#else
    return 0;
#endif
}

// ---------------------------------------------------------------- core types
constexpr int kMaxTopK = 32;                                   // render.hpp:23
constexpr double kLogWeightCutoff = -27.631021115928547;       // render.hpp:97

struct Gaussian {                      // Gaussian3D, types.hpp:25-44
    double mean[3];
    double log_scale[3];
    double rot[4];                     // (w, x, y, z)
    double opacity_logit;
    double color[3];
    std::vector<double> feature;       // heap VectorXd per Gaussian (types.hpp:31)
    int topk_count = 0;                // selection statistics (types.hpp:34-35)
    double max_contribution = 0.0;
};

}  // namespace

struct orc_map {                       // SceneMap, scene_map.hpp:16-27
    std::vector<Gaussian> gaussians;
    uint64_t generation = 0;
    int feature_dim = 0;
    size_t size() const { return gaussians.size(); }
};

namespace {

inline double logistic(double x) { return 1.0 / (1.0 + std::exp(-x)); }  // types.hpp:12

// Quaternion -> rotation matrix, Eigen's Quaternion::toRotationMatrix form (pose.hpp:16).
void quat_to_matrix(double w, double x, double y, double z, double r[3][3]) {
    const double tx = 2.0 * x, ty = 2.0 * y, tz = 2.0 * z;
    const double twx = tx * w, twy = ty * w, twz = tz * w;
    const double txx = tx * x, txy = ty * x, txz = tz * x;
    const double tyy = ty * y, tyz = tz * y, tzz = tz * z;
    r[0][0] = 1.0 - (tyy + tzz);
    r[0][1] = txy - twz;
    r[0][2] = txz + twy;
    r[1][0] = txy + twz;
    r[1][1] = 1.0 - (txx + tzz);
    r[1][2] = tyz - twx;
    r[2][0] = txz - twy;
    r[2][1] = tyz + twx;
    r[2][2] = 1.0 - (txx + tyy);
}

// q.normalized() (types.hpp:40): coefficients divided by sqrt of the squared norm.
void quat_normalized(const double q[4], double out[4]) {
    const double n2 = ((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3];
    const double n = std::sqrt(n2);
    for (int i = 0; i < 4; ++i) out[i] = q[i] / n;
}

// Gaussian3D::covariance (types.hpp:39-43): R diag(exp(2 ls)) R^T.
void covariance(const Gaussian& g, double sig[3][3], double r_out[3][3] = nullptr,
                double s2_out[3] = nullptr) {
    double q[4];
    quat_normalized(g.rot, q);
    double r[3][3];
    quat_to_matrix(q[0], q[1], q[2], q[3], r);
    double s2[3];
    for (int k = 0; k < 3; ++k) s2[k] = std::exp(2.0 * g.log_scale[k]);
    double m[3][3];
    for (int i = 0; i < 3; ++i)
        for (int k = 0; k < 3; ++k) m[i][k] = r[i][k] * s2[k];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) sig[i][j] = (m[i][0] * r[j][0] + m[i][1] * r[j][1]) + m[i][2] * r[j][2];
    if (r_out) std::memcpy(r_out, r, sizeof(r));
    if (s2_out) std::memcpy(s2_out, s2, sizeof(s2));
}

struct Projected {                     // Projected2D, projection.hpp:10-15
    double mx = 0, my = 0;
    double c00 = 0, c01 = 0, c10 = 0, c11 = 0;
    double depth = 0;
    bool visible = false;
};

// project_gaussian, projection.cpp:7-35.
Projected project_gaussian(const Gaussian& g, const orc_pose& pose, const orc_camera& cam,
                           double dilation) {
    Projected out;
    double w[3][3];
    quat_to_matrix(pose.qw, pose.qx, pose.qy, pose.qz, w);
    const double t[3] = {pose.tx, pose.ty, pose.tz};
    double p[3];
    for (int i = 0; i < 3; ++i)
        p[i] = ((w[i][0] * g.mean[0] + w[i][1] * g.mean[1]) + w[i][2] * g.mean[2]) + t[i];
    const double z = p[2];
    if (!(z > cam.near_plane && z < cam.far_plane)) return out;                  // :14
    const double max_ls = std::max(std::max(g.log_scale[0], g.log_scale[1]), g.log_scale[2]);
    const double max_extent = 3.0 * std::exp(max_ls);                            // :19
    if (z <= max_extent) return out;                                             // :20
    out.depth = z;
    out.mx = cam.fx * p[0] / z + cam.cx;                                         // :23
    out.my = cam.fy * p[1] / z + cam.cy;
    const double j[2][3] = {{cam.fx / z, 0.0, -cam.fx * p[0] / (z * z)},        // :25-27
                            {0.0, cam.fy / z, -cam.fy * p[1] / (z * z)}};
    double a[2][3];                                                              // :29  A = J W
    for (int i = 0; i < 2; ++i)
        for (int c = 0; c < 3; ++c) a[i][c] = (j[i][0] * w[0][c] + j[i][1] * w[1][c]) + j[i][2] * w[2][c];
    double sig[3][3];
    covariance(g, sig);
    double b[2][3];                                                              // (A Sigma)
    for (int i = 0; i < 2; ++i)
        for (int c = 0; c < 3; ++c) b[i][c] = (a[i][0] * sig[0][c] + a[i][1] * sig[1][c]) + a[i][2] * sig[2][c];
    double cv[2][2];                                                             // (A Sigma) A^T
    for (int i = 0; i < 2; ++i)
        for (int c = 0; c < 2; ++c) cv[i][c] = (b[i][0] * a[c][0] + b[i][1] * a[c][1]) + b[i][2] * a[c][2];
    cv[0][0] += dilation;                                                        // :31-32
    cv[1][1] += dilation;
    out.c00 = cv[0][0];
    out.c01 = cv[0][1];
    out.c10 = cv[1][0];
    out.c11 = cv[1][1];
    out.visible = true;
    return out;
}

inline double max_eigenvalue(double a, double b, double c) {  // render.cpp:35-39
    const double mid = 0.5 * (a + c);
    const double dif = 0.5 * (a - c);
    return mid + std::sqrt(dif * dif + b * b);
}

struct ProjEntry {                     // raster_detail::ProjEntry, render.hpp:75-81
    double mx, my, ixx, ixy, iyy, z, opacity;
    int32_t src;
};

struct TopKBuffer {                    // render.cpp:41-69
    double w[kMaxTopK];
    int32_t idx[kMaxTopK];
    int n = 0;
    // Front-to-back order: only a strictly larger weight displaces (ties keep the closer one).
    void insert(double weight, int32_t index, int k) {
        int j;
        if (n < k) {
            j = n++;
        } else if (weight > w[k - 1]) {
            j = k - 1;
        } else {
            return;
        }
        while (j > 0 && w[j - 1] < weight) {
            w[j] = w[j - 1];
            idx[j] = idx[j - 1];
            --j;
        }
        w[j] = weight;
        idx[j] = index;
    }
};

}  // namespace

struct orc_prep {                      // PreparedScene, render.hpp:84-92
    std::vector<ProjEntry> entries;
    std::vector<int32_t> tile_offsets;
    std::vector<int32_t> tile_entries;
    int tiles_x = 0, tiles_y = 0, width = 0, height = 0;
    uint64_t generation = 0;
    size_t map_size = 0;
};

namespace {

// prepare_scene, render.cpp:73-156.
void prepare_scene(const orc_map& map, const orc_pose& pose, const orc_camera& cam,
                   const orc_settings& s, orc_prep& prep) {
    prep.width = cam.width;
    prep.height = cam.height;
    prep.generation = map.generation;
    prep.map_size = map.size();
    const int n = static_cast<int>(map.size());
    std::vector<ProjEntry> proj(n);
    std::vector<double> radius(n, -1.0);

#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i) {
        const Projected p = project_gaussian(map.gaussians[i], pose, cam, s.cov2d_dilation);
        if (!p.visible) continue;
        const double a = p.c00, b = p.c01, c = p.c11;
        const double det = a * c - b * b;
        if (!(det > 0.0) || !std::isfinite(det)) continue;       // :90-91
        ProjEntry& e = proj[i];
        e.mx = p.mx;
        e.my = p.my;
        e.ixx = c / det;
        e.ixy = -b / det;
        e.iyy = a / det;
        e.z = p.depth;
        e.opacity = logistic(map.gaussians[i].opacity_logit);
        e.src = i;
        radius[i] = std::sqrt(-2.0 * kLogWeightCutoff * max_eigenvalue(a, b, c));  // :101
    }

    std::vector<int32_t> order;
    order.reserve(n);
    for (int i = 0; i < n; ++i)
        if (radius[i] >= 0.0) order.push_back(i);
    std::sort(order.begin(), order.end(), [&](int32_t l, int32_t r) {    // :108-111
        if (proj[l].z != proj[r].z) return proj[l].z < proj[r].z;
        return l < r;
    });
    prep.entries.clear();
    prep.entries.reserve(order.size());
    std::vector<double> rad_sorted;
    rad_sorted.reserve(order.size());
    for (int32_t i : order) {
        prep.entries.push_back(proj[i]);
        rad_sorted.push_back(radius[i]);
    }

    const int ts = s.tile_size;
    prep.tiles_x = (cam.width + ts - 1) / ts;
    prep.tiles_y = (cam.height + ts - 1) / ts;
    const int n_tiles = prep.tiles_x * prep.tiles_y;
    auto tile_range = [&](const ProjEntry& e, double r, int& tx0, int& tx1, int& ty0, int& ty1) {
        tx0 = std::max(0, static_cast<int>(std::floor((e.mx - r) / ts)));          // :126-132
        tx1 = std::min(prep.tiles_x - 1, static_cast<int>(std::floor((e.mx + r) / ts)));
        ty0 = std::max(0, static_cast<int>(std::floor((e.my - r) / ts)));
        ty1 = std::min(prep.tiles_y - 1, static_cast<int>(std::floor((e.my + r) / ts)));
        return tx0 <= tx1 && ty0 <= ty1;
    };
    std::vector<int32_t> counts(n_tiles, 0);
    for (size_t q = 0; q < prep.entries.size(); ++q) {
        int tx0, tx1, ty0, ty1;
        if (!tile_range(prep.entries[q], rad_sorted[q], tx0, tx1, ty0, ty1)) continue;
        for (int ty = ty0; ty <= ty1; ++ty)
            for (int tx = tx0; tx <= tx1; ++tx) ++counts[ty * prep.tiles_x + tx];
    }
    prep.tile_offsets.assign(n_tiles + 1, 0);
    for (int t = 0; t < n_tiles; ++t) prep.tile_offsets[t + 1] = prep.tile_offsets[t] + counts[t];
    prep.tile_entries.assign(prep.tile_offsets.back(), 0);
    std::vector<int32_t> cursor(prep.tile_offsets.begin(), prep.tile_offsets.end() - 1);
    for (size_t q = 0; q < prep.entries.size(); ++q) {
        int tx0, tx1, ty0, ty1;
        if (!tile_range(prep.entries[q], rad_sorted[q], tx0, tx1, ty0, ty1)) continue;
        for (int ty = ty0; ty <= ty1; ++ty)
            for (int tx = tx0; tx <= tx1; ++tx)
                prep.tile_entries[cursor[ty * prep.tiles_x + tx]++] = static_cast<int32_t>(q);
    }
}

struct GeomOut {
    double* color;
    double* depth;
    double* alpha;
    int32_t* index;
    double* weight;
    uint8_t* count;
    double* contributions;
};

// geometric_pass, render.cpp:158-240.
void geometric_pass(const orc_prep& prep, const orc_map& map, const orc_settings& s, GeomOut o) {
    const int w = prep.width, h = prep.height;
    const int k = std::min(s.top_k, kMaxTopK);
    const size_t P = static_cast<size_t>(w) * h;
    if (o.color) std::fill(o.color, o.color + P * 3, 0.0);
    if (o.depth) std::fill(o.depth, o.depth + P, 0.0);
    if (o.alpha) std::fill(o.alpha, o.alpha + P, 0.0);
    if (o.index) std::fill(o.index, o.index + P * k, -1);
    if (o.weight) std::fill(o.weight, o.weight + P * k, 0.0);
    if (o.count) std::fill(o.count, o.count + P, 0);
    std::vector<double> contributions(prep.map_size, 0.0);

    const int n_threads = max_threads();
    std::vector<std::vector<double>> contrib(n_threads);
    const int ts = s.tile_size;
    const int n_tiles = prep.tiles_x * prep.tiles_y;

#pragma omp parallel
    {
        std::vector<double>& local = contrib[thread_id()];
        local.assign(prep.map_size, 0.0);
#pragma omp for schedule(static)
        for (int t = 0; t < n_tiles; ++t) {
            const int tx = t % prep.tiles_x, ty = t / prep.tiles_x;
            const int x0 = tx * ts, x1 = std::min(w, x0 + ts);
            const int y0 = ty * ts, y1 = std::min(h, y0 + ts);
            const int32_t* list = prep.tile_entries.data() + prep.tile_offsets[t];
            const int list_n = prep.tile_offsets[t + 1] - prep.tile_offsets[t];
            for (int y = y0; y < y1; ++y) {
                for (int x = x0; x < x1; ++x) {
                    double T = 1.0;
                    double acc_r = 0, acc_g = 0, acc_b = 0, acc_d = 0, acc_w = 0;
                    TopKBuffer buf;
                    for (int li = 0; li < list_n; ++li) {
                        const ProjEntry& e = prep.entries[list[li]];
                        const double dx = x - e.mx, dy = y - e.my;
                        const double power = -0.5 * (e.ixx * dx * dx + e.iyy * dy * dy) - e.ixy * dx * dy;
                        if (power < kLogWeightCutoff) continue;                       // :200
                        double alpha = e.opacity * std::exp(power);
                        if (alpha > s.alpha_clamp) alpha = s.alpha_clamp;             // :202
                        const double weight = alpha * T;
                        if (weight > 0.0) {
                            const double* col = map.gaussians[e.src].color;
                            acc_r += weight * col[0];
                            acc_g += weight * col[1];
                            acc_b += weight * col[2];
                            acc_d += weight * e.z;
                            acc_w += weight;
                            buf.insert(weight, e.src, k);
                            if (weight > local[e.src]) local[e.src] = weight;
                        }
                        T *= 1.0 - alpha;
                        if (T < s.transmittance_floor) break;                         // :215
                    }
                    const size_t px = static_cast<size_t>(y) * w + x;
                    if (o.color) {
                        o.color[px * 3 + 0] = acc_r + T * s.background[0];
                        o.color[px * 3 + 1] = acc_g + T * s.background[1];
                        o.color[px * 3 + 2] = acc_b + T * s.background[2];
                    }
                    if (o.depth) o.depth[px] = acc_d;
                    if (o.alpha) o.alpha[px] = acc_w;
                    if (o.count) o.count[px] = static_cast<uint8_t>(buf.n);
                    for (int j = 0; j < buf.n; ++j) {
                        if (o.index) o.index[px * k + j] = buf.idx[j];
                        if (o.weight) o.weight[px * k + j] = buf.w[j];
                    }
                }
            }
        }
    }
    for (int t = 0; t < n_threads; ++t) {                                              // :235-239
        if (contrib[t].empty()) continue;
        for (size_t i = 0; i < prep.map_size; ++i)
            if (contrib[t][i] > contributions[i]) contributions[i] = contrib[t][i];
    }
    if (o.contributions) std::copy(contributions.begin(), contributions.end(), o.contributions);
}

// feature_pass_full_blend, render.cpp:242-289.
void feature_pass_full_blend(const orc_prep& prep, const orc_map& map, const orc_settings& s,
                             double* out) {
    const int w = prep.width, h = prep.height;
    const int d = map.feature_dim;
    std::fill(out, out + static_cast<size_t>(w) * h * d, 0.0);
    std::vector<double> feat(prep.map_size * static_cast<size_t>(d));                  // :249-251
    for (size_t i = 0; i < prep.map_size; ++i)
        for (int c = 0; c < d; ++c) feat[i * d + c] = map.gaussians[i].feature[c];
    const int ts = s.tile_size;
    const int n_tiles = prep.tiles_x * prep.tiles_y;
#pragma omp parallel for schedule(static)
    for (int t = 0; t < n_tiles; ++t) {
        const int tx = t % prep.tiles_x, ty = t / prep.tiles_x;
        const int x0 = tx * ts, x1 = std::min(w, x0 + ts);
        const int y0 = ty * ts, y1 = std::min(h, y0 + ts);
        const int32_t* list = prep.tile_entries.data() + prep.tile_offsets[t];
        const int list_n = prep.tile_offsets[t + 1] - prep.tile_offsets[t];
        for (int y = y0; y < y1; ++y)
            for (int x = x0; x < x1; ++x) {
                double T = 1.0;
                double* px = out + (static_cast<size_t>(y) * w + x) * d;
                for (int li = 0; li < list_n; ++li) {
                    const ProjEntry& e = prep.entries[list[li]];
                    const double dx = x - e.mx, dy = y - e.my;
                    const double power = -0.5 * (e.ixx * dx * dx + e.iyy * dy * dy) - e.ixy * dx * dy;
                    if (power < kLogWeightCutoff) continue;
                    double alpha = e.opacity * std::exp(power);
                    if (alpha > s.alpha_clamp) alpha = s.alpha_clamp;
                    const double weight = alpha * T;
                    if (weight > 0.0) {
                        const double* f = feat.data() + static_cast<size_t>(e.src) * d;
                        for (int c = 0; c < d; ++c) px[c] += weight * f[c];
                    }
                    T *= 1.0 - alpha;
                    if (T < s.transmittance_floor) break;
                }
            }
    }
}

bool check_stale(const char* fn, const int32_t* index, size_t n_slots, int32_t n) {
    for (size_t q = 0; q < n_slots; ++q) {                                             // render.cpp:305-311
        if (index[q] >= n) {
            g_err = std::string(fn) + ": top-k record references gaussian " + std::to_string(index[q]) +
                    " but the map holds " + std::to_string(n) + " (stale snapshot)";
            return false;
        }
    }
    return true;
}

// render_feature, render.cpp:301-337.
int render_feature(const orc_map& map, int w, int h, int k, const int32_t* index, const double* weight,
                   const uint8_t* count, double* out) {
    const int d = map.feature_dim;
    const int32_t n = static_cast<int32_t>(map.size());
    if (!check_stale("render_feature", index, static_cast<size_t>(w) * h * k, n)) return 1;
    std::vector<double> feat(static_cast<size_t>(n) * d);                              // :313-315
    for (int32_t i = 0; i < n; ++i)
        for (int c = 0; c < d; ++c) feat[static_cast<size_t>(i) * d + c] = map.gaussians[i].feature[c];
    std::fill(out, out + static_cast<size_t>(w) * h * d, 0.0);
#pragma omp parallel for schedule(static)
    for (int y = 0; y < h; ++y) {
        for (int x = 0; x < w; ++x) {
            const size_t px = static_cast<size_t>(y) * w + x;
            const int cnt = count[px];
            if (cnt == 0) continue;
            double sum = 0.0;
            for (int j = 0; j < cnt; ++j) sum += weight[px * k + j];
            double* o = out + px * d;
            for (int j = 0; j < cnt; ++j) {
                const size_t sl = px * k + j;
                const double wn = weight[sl] / sum;
                const double* f = feat.data() + static_cast<size_t>(index[sl]) * d;
                for (int c = 0; c < d; ++c) o[c] += wn * f[c];
            }
        }
    }
    return 0;
}

// backward_feature, backward.cpp:273-321.
int backward_feature(const orc_map& map, int w, int h, int k, const int32_t* index, const double* weight,
                     const uint8_t* count, const double* grad, double* out, int threads = 0) {
    const int d = map.feature_dim;
    const int32_t n = static_cast<int32_t>(map.size());
    if (!check_stale("backward_feature", index, static_cast<size_t>(w) * h * k, n)) return 1;
    const int n_threads = threads > 0 ? threads : max_threads();
    std::vector<std::vector<double>> partials(n_threads);
#pragma omp parallel num_threads(n_threads)
    {
        std::vector<double>& local = partials[thread_id()];
        local.assign(static_cast<size_t>(n) * d, 0.0);
#pragma omp for schedule(static)
        for (int y = 0; y < h; ++y) {
            for (int x = 0; x < w; ++x) {
                const size_t px = static_cast<size_t>(y) * w + x;
                const int cnt = count[px];
                if (cnt == 0) continue;
                const double* gf = grad + px * d;
                bool any = false;
                for (int c = 0; c < d; ++c)
                    if (gf[c] != 0.0) { any = true; break; }
                if (!any) continue;
                double sum = 0.0;
                for (int j = 0; j < cnt; ++j) sum += weight[px * k + j];
                for (int j = 0; j < cnt; ++j) {
                    const size_t sl = px * k + j;
                    const double wn = weight[sl] / sum;
                    double* dst = local.data() + static_cast<size_t>(index[sl]) * d;
                    for (int c = 0; c < d; ++c) dst[c] += wn * gf[c];
                }
            }
        }
    }
    const size_t total = static_cast<size_t>(n) * d;
    std::fill(out, out + total, 0.0);
    for (int t = 0; t < n_threads; ++t) {                                              // :315-319
        if (partials[t].empty()) continue;
        for (size_t i = 0; i < total; ++i) out[i] += partials[t][i];
    }
    return 0;
}

struct MidGrad {                       // backward.cpp:36-42
    double mx = 0, my = 0, ixx = 0, ixy = 0, iyy = 0, z = 0, opacity = 0, cr = 0, cg = 0, cb = 0;
};
struct PixContrib {                    // backward.cpp:44-51
    int32_t entry;
    double alpha, weight, t_before, gexp;
    bool clamped;
};

// d(R)/d(q_k) for unit q = (w,x,y,z), backward.cpp:54-68.
void rotation_jacobians(const double q[4], double dr[4][3][3]) {
    const double w = q[0], x = q[1], y = q[2], z = q[3];
    const double m0[3][3] = {{0, -2 * z, 2 * y}, {2 * z, 0, -2 * x}, {-2 * y, 2 * x, 0}};
    const double m1[3][3] = {{0, 2 * y, 2 * z}, {2 * y, -4 * x, -2 * w}, {2 * z, 2 * w, -4 * x}};
    const double m2[3][3] = {{-4 * y, 2 * x, 2 * w}, {2 * x, 0, 2 * z}, {-2 * w, 2 * z, -4 * y}};
    const double m3[3][3] = {{-4 * z, -2 * w, 2 * x}, {2 * w, -4 * z, 2 * y}, {2 * x, 2 * y, 0}};
    std::memcpy(dr[0], m0, sizeof(m0));
    std::memcpy(dr[1], m1, sizeof(m1));
    std::memcpy(dr[2], m2, sizeof(m2));
    std::memcpy(dr[3], m3, sizeof(m3));
}

struct GeomGradsOut {
    double* mean;
    double* log_scale;
    double* rotation;
    double* opacity_logit;
    double* color;
    double* twist;
};

// backward_geometric, backward.cpp:72-271.
void backward_geometric(const orc_map& map, const orc_pose& pose, const orc_camera& cam,
                        const orc_settings& s, const double* grad_color, const double* grad_depth,
                        GeomGradsOut out) {
    orc_prep prep;
    prepare_scene(map, pose, cam, s, prep);                                            // :75
    const size_t n = map.size();
    const int n_threads = max_threads();
    std::vector<std::vector<MidGrad>> partials(n_threads);
    const int ts = s.tile_size;
    const int n_tiles = prep.tiles_x * prep.tiles_y;
    const int w = prep.width, h = prep.height;

#pragma omp parallel
    {
        std::vector<MidGrad>& mid = partials[thread_id()];
        mid.assign(n, MidGrad{});
        std::vector<PixContrib> stack;
#pragma omp for schedule(static)
        for (int t = 0; t < n_tiles; ++t) {
            const int tx = t % prep.tiles_x, ty = t / prep.tiles_x;
            const int x0 = tx * ts, x1 = std::min(w, x0 + ts);
            const int y0 = ty * ts, y1 = std::min(h, y0 + ts);
            const int32_t* list = prep.tile_entries.data() + prep.tile_offsets[t];
            const int list_n = prep.tile_offsets[t + 1] - prep.tile_offsets[t];
            for (int y = y0; y < y1; ++y) {
                for (int x = x0; x < x1; ++x) {
                    const size_t px = static_cast<size_t>(y) * w + x;
                    const double gc[3] = {grad_color[px * 3 + 0], grad_color[px * 3 + 1], grad_color[px * 3 + 2]};
                    const double gd = grad_depth ? grad_depth[px] : 0.0;
                    if (gc[0] == 0.0 && gc[1] == 0.0 && gc[2] == 0.0 && gd == 0.0) continue;  // :102-105
                    stack.clear();
                    double T = 1.0;
                    for (int li = 0; li < list_n; ++li) {                              // :107-124
                        const ProjEntry& e = prep.entries[list[li]];
                        const double dx = x - e.mx, dy = y - e.my;
                        const double power = -0.5 * (e.ixx * dx * dx + e.iyy * dy * dy) - e.ixy * dx * dy;
                        if (power < kLogWeightCutoff) continue;
                        const double gexp = std::exp(power);
                        double alpha = e.opacity * gexp;
                        const bool clamped = alpha > s.alpha_clamp;
                        if (clamped) alpha = s.alpha_clamp;
                        stack.push_back({list[li], alpha, alpha * T, T, gexp, clamped});
                        T *= 1.0 - alpha;
                        if (T < s.transmittance_floor) break;
                    }
                    double suffix_c[3] = {T * s.background[0], T * s.background[1], T * s.background[2]};
                    double suffix_d = 0.0;
                    for (size_t si = stack.size(); si-- > 0;) {                        // :130-160
                        const PixContrib& pc = stack[si];
                        const ProjEntry& e = prep.entries[pc.entry];
                        MidGrad& g = mid[e.src];
                        const double* col = map.gaussians[e.src].color;
                        g.cr += gc[0] * pc.weight;
                        g.cg += gc[1] * pc.weight;
                        g.cb += gc[2] * pc.weight;
                        g.z += gd * pc.weight;
                        const double one_minus = 1.0 - pc.alpha;
                        const double gc_col = (gc[0] * col[0] + gc[1] * col[1]) + gc[2] * col[2];
                        const double gc_suf = (gc[0] * suffix_c[0] + gc[1] * suffix_c[1]) + gc[2] * suffix_c[2];
                        const double d_alpha = pc.t_before * (gc_col + gd * e.z) - (gc_suf + gd * suffix_d) / one_minus;
                        suffix_c[0] += pc.weight * col[0];
                        suffix_c[1] += pc.weight * col[1];
                        suffix_c[2] += pc.weight * col[2];
                        suffix_d += pc.weight * e.z;
                        if (pc.clamped) continue;
                        g.opacity += d_alpha * pc.gexp;
                        const double d_power = d_alpha * pc.alpha;
                        const double dx = x - e.mx, dy = y - e.my;
                        g.mx += d_power * (e.ixx * dx + e.ixy * dy);
                        g.my += d_power * (e.ixy * dx + e.iyy * dy);
                        g.ixx += d_power * (-0.5 * dx * dx);
                        g.ixy += d_power * (-dx * dy);
                        g.iyy += d_power * (-0.5 * dy * dy);
                    }
                }
            }
        }
    }

    std::vector<MidGrad> mid(n);                                                       // :166-178
    for (int t = 0; t < n_threads; ++t) {
        if (partials[t].empty()) continue;
        for (size_t i = 0; i < n; ++i) {
            MidGrad& a = mid[i];
            const MidGrad& b = partials[t][i];
            a.mx += b.mx; a.my += b.my;
            a.ixx += b.ixx; a.ixy += b.ixy; a.iyy += b.iyy;
            a.z += b.z; a.opacity += b.opacity;
            a.cr += b.cr; a.cg += b.cg; a.cb += b.cb;
        }
    }

    std::fill(out.mean, out.mean + n * 3, 0.0);
    std::fill(out.log_scale, out.log_scale + n * 3, 0.0);
    std::fill(out.rotation, out.rotation + n * 4, 0.0);
    std::fill(out.opacity_logit, out.opacity_logit + n, 0.0);
    std::fill(out.color, out.color + n * 3, 0.0);
    double wm[3][3];
    quat_to_matrix(pose.qw, pose.qx, pose.qy, pose.qz, wm);
    const double tr[3] = {pose.tx, pose.ty, pose.tz};
    std::vector<double> twist(n * 6, 0.0);

#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < static_cast<int64_t>(n); ++i) {                             // :190-267
        const MidGrad& g = mid[i];
        const bool touched = g.mx != 0 || g.my != 0 || g.ixx != 0 || g.ixy != 0 || g.iyy != 0 ||
                             g.z != 0 || g.opacity != 0 || g.cr != 0 || g.cg != 0 || g.cb != 0;
        if (!touched) continue;
        const Gaussian& gs = map.gaussians[i];
        out.color[i * 3 + 0] = g.cr;
        out.color[i * 3 + 1] = g.cg;
        out.color[i * 3 + 2] = g.cb;
        const double op = logistic(gs.opacity_logit);
        out.opacity_logit[i] = g.opacity * op * (1.0 - op);

        double p[3];
        for (int r = 0; r < 3; ++r) p[r] = ((wm[r][0] * gs.mean[0] + wm[r][1] * gs.mean[1]) + wm[r][2] * gs.mean[2]) + tr[r];
        const double z = p[2];
        const double inv_z = 1.0 / z, inv_z2 = inv_z * inv_z;
        const double j[2][3] = {{cam.fx * inv_z, 0.0, -cam.fx * p[0] * inv_z2},
                                {0.0, cam.fy * inv_z, -cam.fy * p[1] * inv_z2}};
        double a[2][3];
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 3; ++c) a[r][c] = (j[r][0] * wm[0][c] + j[r][1] * wm[1][c]) + j[r][2] * wm[2][c];
        double q[4];
        quat_normalized(gs.rot, q);
        double rr[3][3], s2[3], sigma[3][3];
        covariance(gs, sigma, rr, s2);
        double as[2][3];
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 3; ++c) as[r][c] = (a[r][0] * sigma[0][c] + a[r][1] * sigma[1][c]) + a[r][2] * sigma[2][c];
        double cv[2][2];
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 2; ++c) cv[r][c] = (as[r][0] * a[c][0] + as[r][1] * a[c][1]) + as[r][2] * a[c][2];
        cv[0][0] += s.cov2d_dilation;
        cv[1][1] += s.cov2d_dilation;
        // Matrix2d::inverse(): adjugate times the reciprocal determinant.
        const double invdet = 1.0 / (cv[0][0] * cv[1][1] - cv[1][0] * cv[0][1]);
        const double inv[2][2] = {{cv[1][1] * invdet, -cv[0][1] * invdet}, {-cv[1][0] * invdet, cv[0][0] * invdet}};
        const double ginv[2][2] = {{g.ixx, 0.5 * g.ixy}, {0.5 * g.ixy, g.iyy}};
        double t1[2][2], gcov[2][2];
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 2; ++c) t1[r][c] = inv[r][0] * ginv[0][c] + inv[r][1] * ginv[1][c];
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 2; ++c) gcov[r][c] = -(t1[r][0] * inv[0][c] + t1[r][1] * inv[1][c]);
        // g_sigma = A^T gcov A ; g_a = 2 gcov A Sigma ; g_j = g_a W^T ; g_w = J^T g_a
        double ga_tmp[2][3];  // gcov A
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 3; ++c) ga_tmp[r][c] = gcov[r][0] * a[0][c] + gcov[r][1] * a[1][c];
        double gsig[3][3];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) gsig[r][c] = a[0][r] * ga_tmp[0][c] + a[1][r] * ga_tmp[1][c];
        double g_a[2][3];
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 3; ++c)
                g_a[r][c] = 2.0 * ((ga_tmp[r][0] * sigma[0][c] + ga_tmp[r][1] * sigma[1][c]) + ga_tmp[r][2] * sigma[2][c]);
        double g_j[2][3];
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 3; ++c) g_j[r][c] = (g_a[r][0] * wm[c][0] + g_a[r][1] * wm[c][1]) + g_a[r][2] * wm[c][2];
        double g_w[3][3];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) g_w[r][c] = j[0][r] * g_a[0][c] + j[1][r] * g_a[1][c];
        double gp[3];                                                                   // :235-240
        gp[0] = g.mx * cam.fx * inv_z + g_j[0][2] * (-cam.fx * inv_z2);
        gp[1] = g.my * cam.fy * inv_z + g_j[1][2] * (-cam.fy * inv_z2);
        gp[2] = g.mx * (-cam.fx * p[0] * inv_z2) + g.my * (-cam.fy * p[1] * inv_z2) + g.z +
                g_j[0][0] * (-cam.fx * inv_z2) + g_j[0][2] * (2.0 * cam.fx * p[0] * inv_z2 * inv_z) +
                g_j[1][1] * (-cam.fy * inv_z2) + g_j[1][2] * (2.0 * cam.fy * p[1] * inv_z2 * inv_z);
        for (int r = 0; r < 3; ++r)                                                     // :242 W^T gp
            out.mean[i * 3 + r] = (wm[0][r] * gp[0] + wm[1][r] * gp[1]) + wm[2][r] * gp[2];
        // log-scale: 2 s2_k (R^T gsig R)_kk  (:245-246)
        for (int kk = 0; kk < 3; ++kk) {
            double acc = 0.0;
            for (int r = 0; r < 3; ++r) {
                double row = 0.0;
                for (int c = 0; c < 3; ++c) row += gsig[r][c] * rr[c][kk];
                acc += rr[r][kk] * row;
            }
            out.log_scale[i * 3 + kk] = 2.0 * s2[kk] * acc;
        }
        // rotation: g_r = 2 gsig R diag(s2); g_qhat_k = <g_r, dR/dq_k>; normalisation (:249-256)
        double g_r[3][3];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c)
                g_r[r][c] = 2.0 * ((gsig[r][0] * rr[0][c] + gsig[r][1] * rr[1][c]) + gsig[r][2] * rr[2][c]) * s2[c];
        double dr[4][3][3];
        rotation_jacobians(q, dr);
        double gq[4];
        for (int kk = 0; kk < 4; ++kk) {
            double acc = 0.0;
            for (int c = 0; c < 3; ++c)
                for (int r = 0; r < 3; ++r) acc += g_r[r][c] * dr[kk][r][c];
            gq[kk] = acc;
        }
        const double qdot = ((q[0] * gq[0] + q[1] * gq[1]) + q[2] * gq[2]) + q[3] * gq[3];
        const double qn = std::sqrt(((gs.rot[0] * gs.rot[0] + gs.rot[1] * gs.rot[1]) + gs.rot[2] * gs.rot[2]) + gs.rot[3] * gs.rot[3]);
        for (int kk = 0; kk < 4; ++kk) out.rotation[i * 4 + kk] = (gq[kk] - q[kk] * qdot) / qn;
        // pose twist (:259-266)
        double* tw = &twist[i * 6];
        tw[0] = gp[0];
        tw[1] = gp[1];
        tw[2] = gp[2];
        tw[3] = p[1] * gp[2] - p[2] * gp[1];
        tw[4] = p[2] * gp[0] - p[0] * gp[2];
        tw[5] = p[0] * gp[1] - p[1] * gp[0];
        double gwwt[3][3];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) gwwt[r][c] = (g_w[r][0] * wm[c][0] + g_w[r][1] * wm[c][1]) + g_w[r][2] * wm[c][2];
        tw[3] += gwwt[2][1] - gwwt[1][2];
        tw[4] += gwwt[0][2] - gwwt[2][0];
        tw[5] += gwwt[1][0] - gwwt[0][1];
    }
    for (int a = 0; a < 6; ++a) out.twist[a] = 0.0;
    for (size_t i = 0; i < n; ++i)                                                     // :269
        for (int a = 0; a < 6; ++a) out.twist[a] += twist[i * 6 + a];
}

}  // namespace

// ======================================================================== C ABI

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

int orc_max_threads(void) { return max_threads(); }
void orc_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

orc_map* orc_map_create(int64_t n, int32_t d, const double* mean, const double* log_scale,
                        const double* rotation, const double* opacity_logit, const double* color,
                        const double* feature, uint64_t generation) {
    orc_map* m = new orc_map;
    m->generation = generation;
    m->feature_dim = d;
    m->gaussians.resize(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
        Gaussian& g = m->gaussians[i];
        for (int c = 0; c < 3; ++c) {
            g.mean[c] = mean[i * 3 + c];
            g.log_scale[c] = log_scale[i * 3 + c];
            g.color[c] = color[i * 3 + c];
        }
        for (int c = 0; c < 4; ++c) g.rot[c] = rotation[i * 4 + c];
        g.opacity_logit = opacity_logit[i];
        g.feature.assign(feature ? feature + i * d : nullptr, feature ? feature + (i + 1) * d : nullptr);
        if (!feature) g.feature.assign(d, 0.0);
    }
    return m;
}

void orc_map_free(orc_map* m) { delete m; }

int orc_project_gaussian(const orc_map* m, int64_t i, const orc_pose* pose, const orc_camera* cam,
                         double dilation, double* out7) {
    const Projected p = project_gaussian(m->gaussians[i], *pose, *cam, dilation);
    out7[0] = p.mx; out7[1] = p.my;
    out7[2] = p.c00; out7[3] = p.c01; out7[4] = p.c10; out7[5] = p.c11;
    out7[6] = p.depth;
    return p.visible ? 1 : 0;
}

orc_prep* orc_prepare_scene(const orc_map* m, const orc_pose* pose, const orc_camera* cam,
                            const orc_settings* s) {
    orc_prep* p = new orc_prep;
    prepare_scene(*m, *pose, *cam, *s, *p);
    return p;
}

void orc_prep_sizes(const orc_prep* p, int64_t* n_entries, int64_t* n_tile_entries, int32_t* tiles_x,
                    int32_t* tiles_y) {
    *n_entries = static_cast<int64_t>(p->entries.size());
    *n_tile_entries = static_cast<int64_t>(p->tile_entries.size());
    *tiles_x = p->tiles_x;
    *tiles_y = p->tiles_y;
}

void orc_prep_export(const orc_prep* p, double* entries7, int32_t* src, int32_t* tile_offsets,
                     int32_t* tile_entries) {
    for (size_t q = 0; q < p->entries.size(); ++q) {
        const ProjEntry& e = p->entries[q];
        double* o = entries7 + q * 7;
        o[0] = e.mx; o[1] = e.my; o[2] = e.ixx; o[3] = e.ixy; o[4] = e.iyy; o[5] = e.z; o[6] = e.opacity;
        src[q] = e.src;
    }
    std::copy(p->tile_offsets.begin(), p->tile_offsets.end(), tile_offsets);
    std::copy(p->tile_entries.begin(), p->tile_entries.end(), tile_entries);
}

void orc_prep_free(orc_prep* p) { delete p; }

int orc_geometric_pass(const orc_prep* p, const orc_map* m, const orc_settings* s, double* color,
                       double* depth, double* alpha, int32_t* topk_index, double* topk_weight,
                       uint8_t* topk_count, double* contributions) {
    geometric_pass(*p, *m, *s, GeomOut{color, depth, alpha, topk_index, topk_weight, topk_count, contributions});
    return 0;
}

int orc_render_geometric(const orc_map* m, const orc_pose* pose, const orc_camera* cam,
                         const orc_settings* s, double* color, double* depth, double* alpha,
                         int32_t* topk_index, double* topk_weight, uint8_t* topk_count,
                         double* contributions) {
    orc_prep p;
    prepare_scene(*m, *pose, *cam, *s, p);
    geometric_pass(p, *m, *s, GeomOut{color, depth, alpha, topk_index, topk_weight, topk_count, contributions});
    return 0;
}

int orc_render_feature(const orc_map* m, int32_t width, int32_t height, int32_t k,
                       const int32_t* topk_index, const double* topk_weight, const uint8_t* topk_count,
                       double* out_feature) {
    return render_feature(*m, width, height, k, topk_index, topk_weight, topk_count, out_feature);
}

int orc_render_feature_full_blend(const orc_map* m, const orc_pose* pose, const orc_camera* cam,
                                  const orc_settings* s, double* out_feature) {
    orc_prep p;
    prepare_scene(*m, *pose, *cam, *s, p);
    feature_pass_full_blend(p, *m, *s, out_feature);
    return 0;
}

int orc_backward_feature(const orc_map* m, int32_t width, int32_t height, int32_t k,
                         const int32_t* topk_index, const double* topk_weight, const uint8_t* topk_count,
                         const double* grad_feature, double* out) {
    return backward_feature(*m, width, height, k, topk_index, topk_weight, topk_count, grad_feature, out);
}

int orc_backward_geometric(const orc_map* m, const orc_pose* pose, const orc_camera* cam,
                           const orc_settings* s, const double* grad_color, const double* grad_depth,
                           double* g_mean, double* g_log_scale, double* g_rotation,
                           double* g_opacity_logit, double* g_color, double* pose_twist) {
    backward_geometric(*m, *pose, *cam, *s, grad_color, grad_depth,
                       GeomGradsOut{g_mean, g_log_scale, g_rotation, g_opacity_logit, g_color, pose_twist});
    return 0;
}

// render_reference, reference.cpp:22-121 (serial, no tiles, Eigen inverse, stable depth sort,
// independent full-sort Top-K selection).
int orc_render_reference(const orc_map* m, const orc_pose* pose, const orc_camera* cam,
                         const orc_settings* s, double* color, double* depth, double* alpha,
                         double* transmittance, double* feature_blend, int32_t* topk_index,
                         double* topk_weight, uint8_t* topk_count, double* contributions,
                         int64_t* record_offsets, int32_t* rec_index, double* rec_weight,
                         int64_t* n_records) {
    const orc_map& map = *m;
    const int w = cam->width, h = cam->height;
    const int k = std::min(s->top_k, kMaxTopK);
    const int d = map.feature_dim;
    const size_t P = static_cast<size_t>(w) * h;
    struct RefProj { double mx, my, i00, i01, i10, i11, z, opacity; int32_t src; };
    std::vector<RefProj> proj;
    for (size_t i = 0; i < map.size(); ++i) {
        const Projected p = project_gaussian(map.gaussians[i], *pose, *cam, s->cov2d_dilation);
        if (!p.visible) continue;
        const double det = p.c00 * p.c11 - p.c10 * p.c01;                  // Matrix2d::determinant
        if (!(det > 0.0) || !std::isfinite(det)) continue;
        const double invdet = 1.0 / det;                                     // Matrix2d::inverse
        proj.push_back({p.mx, p.my, p.c11 * invdet, -p.c01 * invdet, -p.c10 * invdet, p.c00 * invdet,
                        p.depth, logistic(map.gaussians[i].opacity_logit), static_cast<int32_t>(i)});
    }
    std::stable_sort(proj.begin(), proj.end(), [](const RefProj& a, const RefProj& b) { return a.z < b.z; });
    std::vector<double> contrib(map.size(), 0.0);
    if (feature_blend) std::fill(feature_blend, feature_blend + P * d, 0.0);
    if (topk_index) std::fill(topk_index, topk_index + P * k, -1);
    if (topk_weight) std::fill(topk_weight, topk_weight + P * k, 0.0);
    std::vector<std::pair<int32_t, double>> hits;
    std::vector<int> sel;
    int64_t rec_total = 0;
    for (int y = 0; y < h; ++y) {
        for (int x = 0; x < w; ++x) {
            const size_t px = static_cast<size_t>(y) * w + x;
            double T = 1.0;
            double acc[3] = {0, 0, 0};
            double acc_d = 0.0, acc_w = 0.0;
            hits.clear();
            for (size_t pi = 0; pi < proj.size(); ++pi) {
                const RefProj& e = proj[pi];
                const double dx = x - e.mx, dy = y - e.my;
                // -0.5 * diff.dot(inv_cov * diff)   (reference.cpp:64)
                const double v0 = e.i00 * dx + e.i01 * dy;
                const double v1 = e.i10 * dx + e.i11 * dy;
                const double power = -0.5 * (dx * v0 + dy * v1);
                if (power < kLogWeightCutoff) continue;
                double a = e.opacity * std::exp(power);
                if (a > s->alpha_clamp) a = s->alpha_clamp;
                const double wgt = a * T;
                if (wgt > 0.0) {
                    const double* col = map.gaussians[e.src].color;
                    acc[0] += wgt * col[0];
                    acc[1] += wgt * col[1];
                    acc[2] += wgt * col[2];
                    acc_d += wgt * e.z;
                    acc_w += wgt;
                    hits.emplace_back(static_cast<int32_t>(pi), wgt);
                    if (feature_blend) {
                        double* o = feature_blend + px * d;
                        const std::vector<double>& f = map.gaussians[e.src].feature;
                        for (int c = 0; c < d; ++c) o[c] += wgt * f[c];
                    }
                    if (wgt > contrib[e.src]) contrib[e.src] = wgt;
                }
                T *= 1.0 - a;
                if (T < s->transmittance_floor) break;
            }
            if (color) {
                color[px * 3 + 0] = acc[0] + T * s->background[0];
                color[px * 3 + 1] = acc[1] + T * s->background[1];
                color[px * 3 + 2] = acc[2] + T * s->background[2];
            }
            if (depth) depth[px] = acc_d;
            if (alpha) alpha[px] = acc_w;
            if (transmittance) transmittance[px] = T;
            sel.resize(hits.size());
            for (size_t i = 0; i < sel.size(); ++i) sel[i] = static_cast<int>(i);
            std::sort(sel.begin(), sel.end(), [&](int a, int b) {
                if (hits[a].second != hits[b].second) return hits[a].second > hits[b].second;
                const RefProj& pa = proj[hits[a].first];
                const RefProj& pb = proj[hits[b].first];
                if (pa.z != pb.z) return pa.z < pb.z;
                return pa.src < pb.src;
            });
            const int cnt = std::min<int>(k, static_cast<int>(sel.size()));
            if (topk_count) topk_count[px] = static_cast<uint8_t>(cnt);
            for (int j = 0; j < cnt; ++j) {
                if (topk_index) topk_index[px * k + j] = proj[hits[sel[j]].first].src;
                if (topk_weight) topk_weight[px * k + j] = hits[sel[j]].second;
            }
            if (record_offsets) record_offsets[px] = rec_total;
            if (rec_index) {
                for (size_t r = 0; r < hits.size(); ++r) {
                    rec_index[rec_total + r] = proj[hits[r].first].src;
                    rec_weight[rec_total + r] = hits[r].second;
                }
            }
            rec_total += static_cast<int64_t>(hits.size());
        }
    }
    if (record_offsets) record_offsets[P] = rec_total;
    if (n_records) *n_records = rec_total;
    if (contributions) std::copy(contrib.begin(), contrib.end(), contributions);
    return 0;
}

int orc_time_frame(const orc_map* m, const orc_pose* pose, const orc_camera* cam, const orc_settings* s,
                   const double* grad_feature, const double* grad_color, const double* grad_depth,
                   int reps, int feature_threads, double* times) {
    using Clock = std::chrono::steady_clock;
    auto secs = [](Clock::time_point a, Clock::time_point b) {
        return std::chrono::duration<double>(b - a).count();
    };
    const int w = cam->width, h = cam->height;
    const int k = std::min(s->top_k, kMaxTopK);
    const size_t P = static_cast<size_t>(w) * h;
    const size_t n = m->size();
    const int d = m->feature_dim;
    std::vector<double> color(P * 3), depth(P), alpha(P), weight(P * k), contrib(n);
    std::vector<int32_t> index(P * k);
    std::vector<uint8_t> count(P);
    std::vector<double> feat(P * d), dfeat(n * static_cast<size_t>(d));
    std::vector<double> gm(n * 3), gl(n * 3), gr(n * 4), go(n), gcl(n * 3);
    double twist[6];
    for (int i = 0; i < 6; ++i) times[i] = 1e300;
    for (int r = 0; r < reps; ++r) {
        const auto t0 = Clock::now();
        orc_prep prep;
        prepare_scene(*m, *pose, *cam, *s, prep);
        const auto t1 = Clock::now();
        geometric_pass(prep, *m, *s, GeomOut{color.data(), depth.data(), alpha.data(), index.data(),
                                             weight.data(), count.data(), contrib.data()});
        const auto t2 = Clock::now();
        render_feature(*m, w, h, k, index.data(), weight.data(), count.data(), feat.data());
        const auto t3 = Clock::now();
        backward_feature(*m, w, h, k, index.data(), weight.data(), count.data(), grad_feature, dfeat.data(),
                         feature_threads);
        const auto t4 = Clock::now();
        backward_geometric(*m, *pose, *cam, *s, grad_color, grad_depth,
                           GeomGradsOut{gm.data(), gl.data(), gr.data(), go.data(), gcl.data(), twist});
        const auto t5 = Clock::now();
        times[0] = std::min(times[0], secs(t0, t1));
        times[1] = std::min(times[1], secs(t1, t2));
        times[2] = std::min(times[2], secs(t2, t3));
        times[3] = std::min(times[3], secs(t3, t4));
        times[4] = std::min(times[4], secs(t4, t5));
        times[5] = std::min(times[5], secs(t0, t5));
    }
    return max_threads();
}

}  // extern "C"

// Mapping iteration (losses, SSIM, Adam, optimize_step): map/losses.cpp, core/ssim.cpp,
// map/optimizer.cpp, map/mapper.cpp.
#include "oracle_mapping.inc"

// synth.cpp — synthetic scene / trajectory / feature generators (see include/tk_synth.h).
// Restates the reference generators so inputs are identical for GPU and CPU runs.
#include "tk_synth.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

inline double uniform(std::mt19937_64& rng, double lo, double hi) {  // testutil.hpp:16-19
    const double u = static_cast<double>(rng() >> 11) * 0x1.0p-53;
    return lo + u * (hi - lo);
}

struct V3 {
    double x, y, z;
};
inline V3 operator+(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 operator-(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 operator*(double s, V3 a) { return {s * a.x, s * a.y, s * a.z}; }
inline V3 operator-(V3 a) { return {-a.x, -a.y, -a.z}; }
inline double dot(V3 a, V3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
inline V3 cross(V3 a, V3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
inline double norm(V3 a) { return std::sqrt(dot(a, a)); }
inline V3 normalized(V3 a) {
    const double n = norm(a);
    return {a.x / n, a.y / n, a.z / n};
}

struct Quat {
    double w, x, y, z;
};

Quat quat_normalized(Quat q) {
    const double n = std::sqrt(((q.w * q.w + q.x * q.x) + q.y * q.y) + q.z * q.z);
    return {q.w / n, q.x / n, q.y / n, q.z / n};
}

// Quaternion * vector (Eigen _transformVector).
V3 rotate(Quat q, V3 v) {
    const V3 qv{q.x, q.y, q.z};
    V3 uv = cross(qv, v);
    uv = uv + uv;
    return v + q.w * uv + cross(qv, uv);
}

// Quaternion::FromTwoVectors(a, b) (Eigen setFromTwoVectors).  The antiparallel branch picks
// the x axis, a valid null-space direction of [a; b] for a = +z (SVD axis in the reference).
Quat from_two_vectors(V3 a, V3 b) {
    const V3 v0 = normalized(a), v1 = normalized(b);
    double c = dot(v1, v0);
    if (c < -1.0 + 1e-12) {
        c = std::max(c, -1.0);
        V3 axis{1.0, 0.0, 0.0};
        if (std::abs(v0.x) > 0.9) axis = {0.0, 1.0, 0.0};
        axis = normalized(cross(v0, cross(axis, v0)));  // orthogonal to v0
        const double w2 = (1.0 + c) * 0.5;
        const double sv = std::sqrt(1.0 - w2);
        return {std::sqrt(w2), axis.x * sv, axis.y * sv, axis.z * sv};
    }
    const V3 axis = cross(v0, v1);
    const double s = std::sqrt((1.0 + c) * 2.0);
    const double invs = 1.0 / s;
    return {s * 0.5, axis.x * invs, axis.y * invs, axis.z * invs};
}

// Quaternion(Matrix3d) (Eigen quaternionbase_assign_impl).
Quat from_matrix(const double m[3][3]) {
    Quat q{};
    double t = (m[0][0] + m[1][1]) + m[2][2];
    if (t > 0.0) {
        t = std::sqrt(t + 1.0);
        q.w = 0.5 * t;
        t = 0.5 / t;
        q.x = (m[2][1] - m[1][2]) * t;
        q.y = (m[0][2] - m[2][0]) * t;
        q.z = (m[1][0] - m[0][1]) * t;
    } else {
        int i = 0;
        if (m[1][1] > m[0][0]) i = 1;
        if (m[2][2] > m[i][i]) i = 2;
        const int j = (i + 1) % 3, k = (j + 1) % 3;
        t = std::sqrt(m[i][i] - m[j][j] - m[k][k] + 1.0);
        double c[3];
        c[i] = 0.5 * t;
        t = 0.5 / t;
        q.w = (m[k][j] - m[j][k]) * t;
        c[j] = (m[j][i] + m[i][j]) * t;
        c[k] = (m[k][i] + m[i][k]) * t;
        q.x = c[0];
        q.y = c[1];
        q.z = c[2];
    }
    return q;
}

struct Surface {  // scene.cpp:19-27
    V3 origin, u_axis, v_axis;
    double u_len, v_len;
    V3 normal;
    int class_id;
    V3 color;
};

V3 palette(int class_id) {  // scene.cpp:31-37
    static const V3 table[] = {
        {0.85, 0.35, 0.25}, {0.30, 0.65, 0.85}, {0.80, 0.75, 0.40}, {0.40, 0.80, 0.45},
        {0.70, 0.45, 0.80}, {0.90, 0.60, 0.30}, {0.35, 0.80, 0.75}, {0.60, 0.60, 0.60},
    };
    return table[class_id % 8];
}

struct G {
    V3 mean, ls;
    Quat rot;
    double logit;
    V3 color;
    int cls;
};

void tile_surface(const Surface& s, const tk_synth_spec& spec, std::mt19937_64& rng,
                  std::vector<G>& out) {  // scene.cpp:39-69
    const int nu = std::max(1, static_cast<int>(std::round(s.u_len / spec.spacing)));
    const int nv = std::max(1, static_cast<int>(std::round(s.v_len / spec.spacing)));
    const double du = s.u_len / nu, dv = s.v_len / nv;
    const Quat rot = from_two_vectors({0, 0, 1}, s.normal);
    const double tangent = 0.6 * spec.spacing, normal_s = 0.05 * spec.spacing;
    const V3 ls{std::log(tangent), std::log(tangent), std::log(normal_s)};
    const double logit = std::log(spec.opacity / (1.0 - spec.opacity));
    for (int i = 0; i < nu; ++i)
        for (int j = 0; j < nv; ++j) {
            const double ju = uniform(rng, -spec.jitter, spec.jitter) * du;
            const double jv = uniform(rng, -spec.jitter, spec.jitter) * dv;
            G g;
            g.mean = s.origin + ((i + 0.5) * du) * s.u_axis + ((j + 0.5) * dv) * s.v_axis + ju * s.u_axis +
                     jv * s.v_axis;
            g.ls = ls;
            g.rot = rot;
            g.logit = logit;
            g.color = s.color;
            g.cls = s.class_id;
            out.push_back(g);
        }
}

std::vector<G> build(const tk_synth_spec& spec) {  // scene.cpp:73-144
    const auto cls = [&](int kind) { return std::min(kind, spec.classes - 1); };
    const V3 lo{spec.room_min[0], spec.room_min[1], spec.room_min[2]};
    const V3 hi{spec.room_max[0], spec.room_max[1], spec.room_max[2]};
    const V3 ext = hi - lo;
    const V3 X{1, 0, 0}, Y{0, 1, 0}, Z{0, 0, 1};
    std::vector<Surface> surfaces;
    surfaces.push_back({lo, X, Y, ext.x, ext.y, Z, cls(0), palette(cls(0))});
    surfaces.push_back({{lo.x, lo.y, hi.z}, X, Y, ext.x, ext.y, -Z, cls(1), palette(cls(1))});
    surfaces.push_back({{lo.x, lo.y, lo.z}, X, Z, ext.x, ext.z, Y, cls(2), palette(cls(2))});
    surfaces.push_back({{lo.x, hi.y, lo.z}, X, Z, ext.x, ext.z, -Y, cls(2), 0.85 * palette(cls(2))});
    surfaces.push_back({{lo.x, lo.y, lo.z}, Y, Z, ext.y, ext.z, X, cls(2), 0.7 * palette(cls(2))});
    surfaces.push_back({{hi.x, lo.y, lo.z}, Y, Z, ext.y, ext.z, -X, cls(2), 0.55 * palette(cls(2))});
    std::mt19937_64 rng(spec.seed);
    for (int b = 0; b < spec.boxes; ++b) {
        const double sx = uniform(rng, 0.18, 0.38) * ext.x;
        const double sy = uniform(rng, 0.18, 0.38) * ext.y;
        const double sz = uniform(rng, 0.25, 0.55) * ext.z;
        const double ang = 2.0 * M_PI * (b + uniform(rng, 0.0, 0.6)) / std::max(1, spec.boxes);
        const double rad = uniform(rng, 0.45, 0.8) * 0.5 * std::min(ext.x, ext.y);
        const double cx = std::clamp(0.5 * (lo.x + hi.x) + rad * std::cos(ang), lo.x + 0.2 * ext.x, hi.x - 0.2 * ext.x);
        const double cy = std::clamp(0.5 * (lo.y + hi.y) + rad * std::sin(ang), lo.y + 0.2 * ext.y, hi.y - 0.2 * ext.y);
        const V3 bl{cx - 0.5 * sx, cy - 0.5 * sy, lo.z};
        const V3 bh{cx + 0.5 * sx, cy + 0.5 * sy, lo.z + sz};
        const int c = cls(3);
        const V3 col = (1.0 - 0.25 * b) * palette(c);
        surfaces.push_back({{bl.x, bl.y, bh.z}, X, Y, sx, sy, Z, c, col});
        surfaces.push_back({{bl.x, bl.y, bl.z}, X, Z, sx, sz, -Y, c, col});
        surfaces.push_back({{bl.x, bh.y, bl.z}, X, Z, sx, sz, Y, c, col});
        surfaces.push_back({{bl.x, bl.y, bl.z}, Y, Z, sy, sz, -X, c, col});
        surfaces.push_back({{bh.x, bl.y, bl.z}, Y, Z, sy, sz, X, c, col});
    }
    std::vector<G> out;
    for (const Surface& s : surfaces) tile_surface(s, spec, rng, out);
    return out;
}

void look_at(V3 eye, V3 target, double* pose7) {  // scene.cpp:148-165
    const V3 forward = normalized(target - eye);
    V3 up{0, 0, 1};
    if (std::abs(dot(forward, up)) > 0.999) up = {0, 1, 0};
    const V3 right = normalized(cross(forward, up));
    const V3 down = normalized(cross(forward, right));
    // world-to-camera rotation = (cam_to_world)^T, whose rows are right, down, forward.
    const double m[3][3] = {{right.x, right.y, right.z}, {down.x, down.y, down.z}, {forward.x, forward.y, forward.z}};
    const Quat q = quat_normalized(from_matrix(m));
    const V3 t = -rotate(q, eye);
    pose7[0] = q.w; pose7[1] = q.x; pose7[2] = q.y; pose7[3] = q.z;
    pose7[4] = t.x; pose7[5] = t.y; pose7[6] = t.z;
}

inline uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

}  // namespace

extern "C" {

void tk_synth_default_spec(tk_synth_spec* s) {  // scene.hpp:13-23
    s->room_min[0] = -2.0; s->room_min[1] = -2.0; s->room_min[2] = 0.0;
    s->room_max[0] = 2.0; s->room_max[1] = 2.0; s->room_max[2] = 2.5;
    s->classes = 4;
    s->feature_dim = 16;
    s->spacing = 0.05;
    s->jitter = 0.2;
    s->opacity = 0.95;
    s->boxes = 3;
    s->seed = 1;
}

void tk_synth_random_scene(int32_t count, int32_t d, uint64_t seed, double zmin, double zmax,
                           tk_synth_arrays* o) {  // testutil.hpp:31-53
    std::mt19937_64 rng(seed);
    for (int i = 0; i < count; ++i) {
        const double z = uniform(rng, zmin, zmax);
        const double mx = uniform(rng, -0.45, 0.45) * z;
        const double my = uniform(rng, -0.45, 0.45) * z;
        o->mean[i * 3 + 0] = mx; o->mean[i * 3 + 1] = my; o->mean[i * 3 + 2] = z;
        for (int c = 0; c < 3; ++c) o->log_scale[i * 3 + c] = uniform(rng, -3.2, -1.6);
        // Eigen::Quaterniond(w, x, y, z) is a function call: argument evaluation order is
        // unspecified and GCC (the reference's compiler) evaluates right to left.
        Quat q;
        q.z = uniform(rng, -1, 1);
        q.y = uniform(rng, -1, 1);
        q.x = uniform(rng, -1, 1);
        q.w = uniform(rng, -1, 1);
        q = quat_normalized(q);
        o->rotation[i * 4 + 0] = q.w; o->rotation[i * 4 + 1] = q.x;
        o->rotation[i * 4 + 2] = q.y; o->rotation[i * 4 + 3] = q.z;
        o->opacity_logit[i] = uniform(rng, -1.5, 2.2);
        for (int c = 0; c < 3; ++c) o->color[i * 3 + c] = uniform(rng, 0.05, 0.95);
        std::vector<double> f(d);
        for (int c = 0; c < d; ++c) f[c] = uniform(rng, -1, 1);
        double n2 = 0.0;
        for (int c = 0; c < d; ++c) n2 += f[c] * f[c];
        const double nrm = std::sqrt(n2);
        if (o->feature)
            for (int c = 0; c < d; ++c) o->feature[static_cast<int64_t>(i) * d + c] = nrm > 0 ? f[c] / nrm : f[c];
    }
}

int64_t tk_synth_build_scene(const tk_synth_spec* spec, tk_synth_arrays* o, uint8_t* class_ids) {
    if (spec->feature_dim < spec->classes) return -1;  // scene.cpp:74-77
    const std::vector<G> gs = build(*spec);
    const int64_t n = static_cast<int64_t>(gs.size());
    if (!o) return n;
    const int64_t m = std::min<int64_t>(n, o->n > 0 ? o->n : n);  // truncate (fslam_main.cpp:193)
    for (int64_t i = 0; i < m; ++i) {
        const G& g = gs[i];
        o->mean[i * 3 + 0] = g.mean.x; o->mean[i * 3 + 1] = g.mean.y; o->mean[i * 3 + 2] = g.mean.z;
        o->log_scale[i * 3 + 0] = g.ls.x; o->log_scale[i * 3 + 1] = g.ls.y; o->log_scale[i * 3 + 2] = g.ls.z;
        o->rotation[i * 4 + 0] = g.rot.w; o->rotation[i * 4 + 1] = g.rot.x;
        o->rotation[i * 4 + 2] = g.rot.y; o->rotation[i * 4 + 3] = g.rot.z;
        o->opacity_logit[i] = g.logit;
        o->color[i * 3 + 0] = g.color.x; o->color[i * 3 + 1] = g.color.y; o->color[i * 3 + 2] = g.color.z;
        if (class_ids) class_ids[i] = static_cast<uint8_t>(g.cls);
        if (o->feature) {
            double* f = o->feature + i * o->d;
            std::fill(f, f + o->d, 0.0);
            if (g.cls < o->d) f[g.cls] = 1.0;
        }
    }
    return m;
}

int tk_synth_trajectory(int32_t kind, int32_t n, const tk_synth_spec* spec, double* poses) {
    if (n < 2) return -1;  // scene.cpp:170
    const V3 lo{spec->room_min[0], spec->room_min[1], spec->room_min[2]};
    const V3 hi{spec->room_max[0], spec->room_max[1], spec->room_max[2]};
    const V3 center = 0.5 * (lo + hi);
    const V3 ext = hi - lo;
    if (kind == 0) {  // orbit, scene.cpp:177-193
        const double radius = 0.3 * std::min(ext.x, ext.y);
        const V3 eye_base{center.x, center.y, lo.z + 0.72 * ext.z};
        const V3 target{center.x, center.y, lo.z + 0.25 * ext.z};
        for (int i = 0; i < n; ++i) {
            const double az = 2.0 * M_PI * i / n;
            const V3 off{radius * std::cos(az), radius * std::sin(az), 0.0};
            look_at(eye_base + off, target - 2.2 * off, poses + 7 * i);
        }
        return 0;
    }
    // lawnmower, scene.cpp:195-229
    const double inset = 0.3;
    const double x0 = lo.x + inset * ext.x, x1 = hi.x - inset * ext.x;
    const double y0 = lo.y + inset * ext.y, y1 = hi.y - inset * ext.y;
    const double z = center.z + 0.1 * ext.z;
    const double rows[3] = {y0, 0.5 * (y0 + y1), y1};
    std::vector<V3> wp;
    for (int r = 0; r < 3; ++r) {
        const bool fwd = (r % 2) == 0;
        wp.push_back({fwd ? x0 : x1, rows[r], z});
        wp.push_back({fwd ? x1 : x0, rows[r], z});
    }
    std::vector<double> cum{0.0};
    for (size_t i = 1; i < wp.size(); ++i) cum.push_back(cum.back() + norm(wp[i] - wp[i - 1]));
    const double total = cum.back();
    double att[7];
    look_at({0, 0, 0}, normalized(V3{1.0, 0.0, -0.55}), att);
    const Quat q{att[0], att[1], att[2], att[3]};
    for (int i = 0; i < n; ++i) {
        const double s = total * i / (n - 1);
        size_t seg = 1;
        while (seg + 1 < cum.size() && cum[seg] < s) ++seg;
        const double t = (s - cum[seg - 1]) / std::max(1e-12, cum[seg] - cum[seg - 1]);
        const V3 eye = (1.0 - t) * wp[seg - 1] + t * wp[seg];
        const V3 tr = -rotate(q, eye);
        double* p = poses + 7 * i;
        p[0] = q.w; p[1] = q.x; p[2] = q.y; p[3] = q.z;
        p[4] = tr.x; p[5] = tr.y; p[6] = tr.z;
    }
    return 0;
}

void tk_synth_unit_features(int64_t n, int32_t d, uint64_t seed, float* out_f32, double* out_f64) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        std::vector<double> f(d);
        double n2 = 0.0;
        for (int c = 0; c < d; ++c) {
            const uint64_t r = splitmix64(seed * 0x100000001B3ull ^ (static_cast<uint64_t>(i) * d + c));
            f[c] = -1.0 + 2.0 * (static_cast<double>(r >> 11) * 0x1.0p-53);
            n2 += f[c] * f[c];
        }
        const double inv = 1.0 / std::sqrt(n2);
        for (int c = 0; c < d; ++c) {
            const double v = f[c] * inv;
            if (out_f32) out_f32[i * d + c] = static_cast<float>(v);
            if (out_f64) out_f64[i * d + c] = v;
        }
    }
}

void tk_synth_uniform_fill(int64_t count, uint64_t seed, double lo, double hi, double* out) {
    std::mt19937_64 rng(seed);
    for (int64_t i = 0; i < count; ++i) out[i] = uniform(rng, lo, hi);
}

void tk_synth_hash_fill_f32(int64_t count, uint64_t seed, float lo, float hi, float* out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < count; ++i) {
        const uint64_t r = splitmix64(seed * 0x9E3779B97F4A7C15ull ^ static_cast<uint64_t>(i));
        out[i] = lo + static_cast<float>(static_cast<double>(r >> 40) * 0x1.0p-24) * (hi - lo);
    }
}

}  // extern "C"

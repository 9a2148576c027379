/*
 * tk_synth.h — synthetic inputs for the Top-K feature-render path (host C++, no CUDA).
 *
 * These are the reference's scene generators, restated so that benchmarks and parity tests
 * can build identical inputs for the GPU path and the CPU oracle:
 *   tk_synth_random_scene  <- testutil::random_scene   (proj/tests/testutil.hpp:31-53)
 *   tk_synth_build_scene   <- build_synthetic_scene    (proj/src/synth/scene.cpp:73-144)
 *   tk_synth_trajectory    <- generate_trajectory      (proj/src/synth/scene.cpp:169-230)
 *   tk_synth_unit_features <- seeded random unit rows (replaces the one-hot
 *                              class embeddings of scene.cpp:81-82 so gathers are non-trivial)
 * All randomness is std::mt19937_64 with uniform = (rng() >> 11) * 2^-53 (testutil.hpp:16-19),
 * except tk_synth_unit_features, which uses a counter-based splitmix64 stream so 1M x 512 rows
 * can be generated in parallel.
 */
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Gaussian SoA arrays (the layout tk_scene_upload consumes). */
typedef struct {
    int64_t n;
    int32_t d;
    double* mean;          /* n x 3 */
    double* log_scale;     /* n x 3 */
    double* rotation;      /* n x 4, (w, x, y, z) */
    double* opacity_logit; /* n */
    double* color;         /* n x 3 */
    double* feature;       /* n x d, may be NULL */
} tk_synth_arrays;

/* SceneSpec (proj/include/fslam/synth/scene.hpp:13-23). */
typedef struct {
    double room_min[3];
    double room_max[3];
    int32_t classes;
    int32_t feature_dim;
    double spacing;
    double jitter;
    double opacity;
    int32_t boxes;
    uint64_t seed;
} tk_synth_spec;

void tk_synth_default_spec(tk_synth_spec* spec);

/* testutil::random_scene(count, feature_dim, seed, depth_min, depth_max); arrays preallocated. */
void tk_synth_random_scene(int32_t count, int32_t feature_dim, uint64_t seed, double depth_min,
                           double depth_max, tk_synth_arrays* out);

/* build_synthetic_scene: call with out == NULL to get the Gaussian count; then with arrays of
 * that size.  class_ids (n bytes) may be NULL.  Features are the one-hot class embeddings
 * (scene.cpp:81-82) when out->feature != NULL.  Returns the count, or -1 on a bad spec. */
int64_t tk_synth_build_scene(const tk_synth_spec* spec, tk_synth_arrays* out, uint8_t* class_ids);

/* generate_trajectory: kind 0 = orbit, 1 = lawnmower. poses: n x 7 (qw,qx,qy,qz,tx,ty,tz). */
int tk_synth_trajectory(int32_t kind, int32_t n, const tk_synth_spec* spec, double* poses);

/* Row-normalised U(-1,1) features, n x d, float or double output (one of them non-NULL). */
void tk_synth_unit_features(int64_t n, int32_t d, uint64_t seed, float* out_f32, double* out_f64);

/* Seeded U(lo,hi) fill (mt19937_64, testutil uniform) for upstream-gradient images. */
void tk_synth_uniform_fill(int64_t count, uint64_t seed, double lo, double hi, double* out);

/* Counter-based (splitmix64, OpenMP) U(lo,hi) fill of fp32 images too large for a serial
 * generator (the P x D upstream feature gradient of the benchmark). */
void tk_synth_hash_fill_f32(int64_t count, uint64_t seed, float lo, float hi, float* out);

#ifdef __cplusplus
}
#endif

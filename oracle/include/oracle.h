/*
 * oracle.h — C ABI of the CPU fp64 restatement of the reference renderer.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the
 * B200 path and the CPU baseline of bench.py.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it.  The product library (paper_2602_06991_b200/) never links,
 * imports or calls anything under oracle/.
 *
 * It restates, function by function, the reference's raster path
 * (/root/reference/proj, read-only, cannot be built here: Eigen3, libpng,
 * doctest and CLI11 are absent — see DESIGN.md "Oracle"):
 *   core/types.hpp:12-44, core/pose.hpp:16, core/projection.cpp:7-35,
 *   raster/render.cpp:34-343, raster/backward.cpp:35-321,
 *   raster/reference.cpp:22-121.
 * Bit-level pinning: the reference runs its small fixed-size products through
 * Eigen (not vendored, version unpinned); this restatement fixes one
 * summation order (left to right) and is compiled with -ffp-contract=off and
 * no -march, like the reference build (proj/CMakeLists.txt:7-9).  It is pinned
 * to the reference's own known-answer tests at their stated tolerances
 * (tests/test_oracle_kats.py).
 */
#pragma once
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same field layout as tk_camera / tk_pose / tk_settings in include/tk_render.h. */
typedef struct {
    double fx, fy, cx, cy;
    int32_t width, height;
    double near_plane, far_plane;
} orc_camera; /* CameraIntrinsics, types.hpp:15-21 */

typedef struct {
    double qw, qx, qy, qz; /* world-to-camera rotation (not normalised on use, pose.hpp:16) */
    double tx, ty, tz;
} orc_pose; /* Pose, pose.hpp:11-19 */

typedef struct {
    int32_t top_k;
    int32_t tile_size;
    double transmittance_floor;
    double background[3];
    double cov2d_dilation;
    double alpha_clamp;
} orc_settings; /* RenderSettings, render.hpp:14-21 */

typedef struct orc_map orc_map;   /* SceneMap (AoS + per-Gaussian heap feature) */
typedef struct orc_prep orc_prep; /* raster_detail::PreparedScene */

const char* orc_last_error(void);

/* Map: SoA inputs are copied into the reference's AoS layout. features: n*d doubles. */
orc_map* orc_map_create(int64_t n, int32_t d, const double* mean, const double* log_scale,
                        const double* rotation_wxyz, const double* opacity_logit,
                        const double* color, const double* feature, uint64_t generation);
void orc_map_free(orc_map* m);

/* project_gaussian (projection.cpp:7-35). out7 = mx,my,c00,c01,c10,c11,depth. returns visible. */
int orc_project_gaussian(const orc_map* m, int64_t i, const orc_pose* pose, const orc_camera* cam,
                         double dilation, double* out7);

/* prepare_scene (render.cpp:73-156) */
orc_prep* orc_prepare_scene(const orc_map* m, const orc_pose* pose, const orc_camera* cam,
                            const orc_settings* s);
void orc_prep_sizes(const orc_prep* p, int64_t* n_entries, int64_t* n_tile_entries,
                    int32_t* tiles_x, int32_t* tiles_y);
/* entries7: n_entries x {mx,my,ixx,ixy,iyy,z,opacity}; src: n_entries; tile_offsets: tiles+1 */
void orc_prep_export(const orc_prep* p, double* entries7, int32_t* src, int32_t* tile_offsets,
                     int32_t* tile_entries);
void orc_prep_free(orc_prep* p);

/* geometric_pass (render.cpp:158-240) on a prepared scene. Any output may be NULL. */
int orc_geometric_pass(const orc_prep* p, const orc_map* m, const orc_settings* s, double* color,
                       double* depth, double* alpha, int32_t* topk_index, double* topk_weight,
                       uint8_t* topk_count, double* contributions);

/* render_geometric (render.cpp:293-299) */
int orc_render_geometric(const orc_map* m, const orc_pose* pose, const orc_camera* cam,
                         const orc_settings* s, double* color, double* depth, double* alpha,
                         int32_t* topk_index, double* topk_weight, uint8_t* topk_count,
                         double* contributions);

/* render_feature (render.cpp:301-337). returns 0 ok, 1 stale index (message in orc_last_error). */
int orc_render_feature(const orc_map* m, int32_t width, int32_t height, int32_t k,
                       const int32_t* topk_index, const double* topk_weight,
                       const uint8_t* topk_count, double* out_feature);

/* render_feature_full_blend (render.cpp:242-289, 339-343) */
int orc_render_feature_full_blend(const orc_map* m, const orc_pose* pose, const orc_camera* cam,
                                  const orc_settings* s, double* out_feature);

/* backward_feature (backward.cpp:273-321). out: n*d dense. */
int orc_backward_feature(const orc_map* m, int32_t width, int32_t height, int32_t k,
                         const int32_t* topk_index, const double* topk_weight,
                         const uint8_t* topk_count, const double* grad_feature, double* out);

/* backward_geometric (backward.cpp:72-271). grad_depth may be NULL (empty image). */
int orc_backward_geometric(const orc_map* m, const orc_pose* pose, const orc_camera* cam,
                           const orc_settings* s, const double* grad_color,
                           const double* grad_depth, double* g_mean, double* g_log_scale,
                           double* g_rotation, double* g_opacity_logit, double* g_color,
                           double* pose_twist);

/* render_reference (reference.cpp:22-121). feature_blend (P*d) and the per-pixel contributor
 * records are produced only when the pointers are non-NULL.  records: flattened, with
 * record_offsets[P+1]; call first with rec_index=NULL to get the total count in *n_records. */
int orc_render_reference(const orc_map* m, const orc_pose* pose, const orc_camera* cam,
                         const orc_settings* s, double* color, double* depth, double* alpha,
                         double* transmittance, double* feature_blend, int32_t* topk_index,
                         double* topk_weight, uint8_t* topk_count, double* contributions,
                         int64_t* record_offsets, int32_t* rec_index, double* rec_weight,
                         int64_t* n_records);

/* Timing harness for the CPU baseline (fslam_main.cpp:28-36 time_call: best of reps,
 * steady_clock).  Times each reference function separately on the given inputs and writes
 * seconds into times[6] = {prepare_scene, geometric_pass, render_feature, backward_feature,
 * backward_geometric, frame_total}.  grad_* are the upstream gradients.  Returns threads used. */
int orc_time_frame(const orc_map* m, const orc_pose* pose, const orc_camera* cam,
                   const orc_settings* s, const double* grad_feature, const double* grad_color,
                   const double* grad_depth, int reps, int feature_threads, double* times);

int orc_max_threads(void);
void orc_set_threads(int n);

/* ---- one mapping iteration (map/losses.cpp, core/ssim.cpp, map/optimizer.cpp, map/mapper.cpp) ----
 * Same field layout as tk_mapper_config in include/tk_render.h.  Flattens MapperConfig's
 * LossWeights (losses.hpp:9-21), GroupLearningRates / AdamParams (optimizer.hpp:9-23),
 * Schedule::feature_update_period (mapper.hpp:16) and the log-scale clamps (mapper.hpp:31-32). */
typedef struct {
    double lambda_geo, lambda_feat, lambda1, lambda2;
    int32_t color_secondary;        /* 0 = D-SSIM, 1 = duplicated L1 (ColorSecondaryTerm) */
    int32_t feature_update_period;
    double l1_deadband;
    double lr_mean, lr_log_scale, lr_rotation, lr_opacity, lr_color, lr_feature;
    double beta1, beta2, eps;
    double min_log_scale, max_log_scale;
} orc_mapper_config;

typedef struct orc_opt orc_opt; /* OptimizerState (optimizer.hpp:25-53) */
orc_opt* orc_opt_create(int64_t n, int32_t d);
void orc_opt_free(orc_opt* o);

/* ssim_with_grad (ssim.cpp:110-158); images h x w x c, channel fastest. */
double orc_ssim_with_grad(int32_t w, int32_t h, int32_t c, const double* a, const double* b, double* grad);

/* compute_losses (losses.cpp:22-133). values[3] = {map, geo, feat}; grad_feature may be NULL. */
int orc_compute_losses(int32_t w, int32_t h, int32_t d, const double* color, const double* depth,
                       const uint8_t* topk_count, const double* feature, const float* gt_color,
                       const float* gt_depth, const float* gt_feature, const orc_mapper_config* cfg,
                       int32_t include_feature, double* values, double* grad_color, double* grad_depth,
                       double* grad_feature);

/* optimize_step (mapper.cpp:162-255) on a caller-chosen keyframe, without the prune branch.
 * Updates the map and optimizer state in place; values[3] as above. */
int orc_optimize_step(orc_map* m, orc_opt* o, const orc_mapper_config* cfg, const orc_camera* cam,
                      const orc_settings* s, const orc_pose* kf_pose, const float* gt_color,
                      const float* gt_depth, const float* gt_feature, int64_t iteration, double* values,
                      int32_t* feature_step);

/* update_contribution_stats (mapper.cpp:62-78); 1 = generation / size mismatch (orc_last_error). */
int orc_update_contribution_stats(orc_map* m, uint64_t generation, int64_t map_size, int32_t w, int32_t h,
                                  int32_t k, const int32_t* index, const uint8_t* count,
                                  const double* contributions);

/* insert_gaussians (mapper.cpp:19-60): SoA source points (feature n x d_src or NULL). */
int orc_insert_gaussians(orc_map* m, orc_opt* o, int64_t n_src, const double* position, const double* color,
                         const double* feature, int32_t d_src, const double* spacing, const double* distance,
                         double tau, const orc_pose* world_to_camera);
/* prune_map (mapper.cpp:80-160) + OptimizerState::compact; returns the number removed. */
int64_t orc_prune_map(orc_map* m, orc_opt* o, double keep_ratio, uint64_t seed, int32_t threshold,
                      int32_t* removed_out);
int orc_checkpoint_save(const orc_map* m, const char* path);      /* checkpoint.cpp:39-63 */
orc_map* orc_checkpoint_load(const char* path);                    /* checkpoint.cpp:65-98 */
void orc_segment_by_query(int32_t w, int32_t h, int32_t d, const double* feature, int32_t classes,
                          const double* emb, uint8_t* out);           /* metrics.cpp:66-94 */
int64_t orc_map_size(const orc_map* m);
double* orc_opt_moments(orc_opt* o, int32_t group, int32_t which, int64_t* count);
uint64_t orc_map_generation(const orc_map* m);
int32_t orc_map_feature_dim(const orc_map* m);
void orc_map_set_stats(orc_map* m, const int32_t* topk_count, const double* max_contribution);

/* Map parameters and selection statistics back out in SoA form (any pointer may be NULL). */
void orc_map_export(const orc_map* m, double* mean, double* log_scale, double* rotation,
                    double* opacity_logit, double* color, double* feature, int32_t* topk_count,
                    double* max_contribution);

#ifdef __cplusplus
}
#endif

// mapedit.cuh — structural edits of the device-resident map: insert_gaussians (mapper.cpp:19-60)
// and the row compaction behind prune_map / OptimizerState::compact (mapper.cpp:141-154,
// optimizer.cpp:9-27).
#pragma once
#include "tk_common.cuh"

namespace tk {

struct InsertParams {
    int64_t n_src;
    int64_t base;            // index of the first inserted Gaussian (map size before)
    const double* position;  // n_src x 3, camera frame
    const double* color;     // n_src x 3
    const float* feature;    // n_src x d_src or null
    int d_src;
    const double* spacing;   // n_src
    const int32_t* slot;     // exclusive scan of the insert flags
    const uint8_t* flag;     // distance >= tau
    double qi[4];            // cam-to-world rotation conj(q) (not normalised: Pose::apply)
    double ti[3];            // cam-to-world translation
    double rot[4];           // normalised conj(q) (mapper.cpp:26)
    double opacity_logit;    // logit(0.5)
    int d;                   // map feature dim
    double* mean;
    double* log_scale;
    double* rotation;
    double* opacity;
    double* color_out;
    float* feat;
};

// flag[i] = distance[i] >= tau (mapper.cpp:30)
void launch_insert_flags(const double* distance, int64_t n, double tau, uint8_t* flag, int32_t* flag_i32,
                         cudaStream_t st);
void launch_insert_fill(const InsertParams& p, cudaStream_t st);

// keep[i] = 0 for every i in removed[0..n_removed) (ascending or not), else 1
void launch_keep_flags(const int32_t* removed, int64_t n_removed, int64_t n, int32_t* keep, cudaStream_t st);
// dst[pos[r]*width + c] = src[r*width + c] for every kept row r (element-parallel)
void launch_compact_f64(const double* src, double* dst, const int32_t* keep, const int32_t* pos, int64_t n,
                        int width, cudaStream_t st);
void launch_compact_f32(const float* src, float* dst, const int32_t* keep, const int32_t* pos, int64_t n, int width,
                        cudaStream_t st);

// Quaternion * vector as Eigen::Quaternion::_transformVector: uv = 2 (q.vec x v); v + w uv + q.vec x uv
__host__ __device__ inline void quat_rotate_eigen(const double q[4], const double v[3], double out[3]) {
    const double qx = q[1], qy = q[2], qz = q[3];
    double uv[3] = {qy * v[2] - qz * v[1], qz * v[0] - qx * v[2], qx * v[1] - qy * v[0]};
    for (int a = 0; a < 3; ++a) uv[a] += uv[a];
    const double c[3] = {qy * uv[2] - qz * uv[1], qz * uv[0] - qx * uv[2], qx * uv[1] - qy * uv[0]};
    for (int a = 0; a < 3; ++a) out[a] = (v[a] + q[0] * uv[a]) + c[a];
}

}  // namespace tk

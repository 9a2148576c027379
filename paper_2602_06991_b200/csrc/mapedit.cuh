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

// SoA view of the resident map for the SPLF checkpoint pack / unpack (checkpoint.cpp:39-98).
struct SplfView {
    int64_t n;
    int d;
    double* mean;
    double* log_scale;
    double* rotation;
    double* opacity_logit;
    double* color;
    float* feature;
};
void launch_splf_pack(const SplfView& v, float* rec, cudaStream_t st);      // rec: n x (14 + d) f32
void launch_splf_unpack(const float* rec, const SplfView& v, cudaStream_t st);

// segment_by_query (eval/metrics.cpp:66-94) over a rendered H x W x D feature image.
struct QueryParams {
    int64_t n_pixels;
    int d;              // channels held here (a shard [c0, c0 + d) of d_total under tk_comm)
    int c0, d_total;
    int classes;
    const float* feat;  // n_pixels x d
    const double* emb;  // classes x d_total (row-major, device)
    uint8_t* labels;    // n_pixels (255 = kInvalidLabel)
    double* best;       // n_pixels scratch
    double* partial;    // non-null: write per-class partial dots (n_pixels x classes) instead
    double* norm2;      //   and the partial squared norms (n_pixels)
    double* acc;        // n_pixels x classes running dots (only when D spans several chunks)
    double* nacc;       // n_pixels running squared norms (idem)
};
// channels per shared-memory pass (the whole D when classes x D x 8 B fits in 160 KB)
int segment_query_chunk(int d, int classes);
void launch_segment_query(const QueryParams& p, cudaStream_t st);
void launch_query_argmax(const double* scores, const double* norm2, int64_t n, int classes, uint8_t* labels,
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

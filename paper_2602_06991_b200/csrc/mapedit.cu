// mapedit.cu — insertion and compaction kernels for the device-resident map (rare, structural
// edits: once per keyframe / every prune_period iterations).  --fmad=false: the inserted means
// follow Pose::apply's Eigen rotation formula operation by operation, like the oracle.
#include "mapedit.cuh"

namespace tk {

namespace {

__global__ void k_insert_flags(const double* __restrict__ distance, int64_t n, double tau, uint8_t* __restrict__ flag,
                               int32_t* __restrict__ flag_i32) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const bool f = !(distance[i] < tau);  // mapper.cpp:30 skips distance < tau only
        flag[i] = f ? 1 : 0;
        flag_i32[i] = f ? 1 : 0;
    }
}

// One warp per source point: geometry on lane 0, the feature row (normalised in fp64) across lanes.
__global__ void __launch_bounds__(256) k_insert_fill(InsertParams p) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = static_cast<int64_t>(gridDim.x) * (blockDim.x / 32);
    for (int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < p.n_src; i += nw) {
        if (!p.flag[i]) continue;
        const int64_t g = p.base + p.slot[i];
        if (lane == 0) {
            double pc[3];
            quat_rotate_eigen(p.qi, p.position + i * 3, pc);                   // cam_to_world.apply
            for (int a = 0; a < 3; ++a) p.mean[g * 3 + a] = pc[a] + p.ti[a];
            const double sc = fmax(1e-6, 0.5 * p.spacing[i]);                 // mapper.cpp:35-36
            const double ls = log(sc);
            for (int a = 0; a < 3; ++a) p.log_scale[g * 3 + a] = ls;
            for (int a = 0; a < 4; ++a) p.rotation[g * 4 + a] = p.rot[a];
            p.opacity[g] = p.opacity_logit;
            for (int a = 0; a < 3; ++a) p.color_out[g * 3 + a] = p.color[i * 3 + a];
        }
        if (p.d > 0) {                                                         // mapper.cpp:42-49
            const bool same = p.feature && p.d_src == p.d;
            double n2 = 0.0;
            if (same)
                for (int c = lane; c < p.d; c += 32) {
                    const double v = p.feature[i * p.d + c];
                    n2 += v * v;
                }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) n2 += __shfl_xor_sync(0xffffffffu, n2, o);
            const double nrm = sqrt(n2);
            const bool use = same && nrm > 1e-9;
            const double cst = 1.0 / sqrt(static_cast<double>(p.d));
            for (int c = lane; c < p.d; c += 32)
                p.feat[g * p.d + c] = static_cast<float>(use ? static_cast<double>(p.feature[i * p.d + c]) / nrm : cst);
        }
    }
}

__global__ void k_fill_one(int32_t* __restrict__ v, int64_t n) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        v[i] = 1;
}

__global__ void k_keep_flags(const int32_t* __restrict__ removed, int64_t n_removed, int64_t n,
                             int32_t* __restrict__ keep) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n_removed;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t r = removed[i];
        if (r >= 0 && r < n) keep[r] = 0;
    }
}

template <class T>
__global__ void k_compact(const T* __restrict__ src, T* __restrict__ dst, const int32_t* __restrict__ keep,
                          const int32_t* __restrict__ pos, int64_t n, int width) {
    const int64_t total = n * width;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = e / width;
        if (keep[r]) dst[static_cast<int64_t>(pos[r]) * width + (e - r * width)] = src[e];
    }
}

inline unsigned grid_for(int64_t items) {
    const int64_t b = (items + 255) / 256;
    return static_cast<unsigned>(b < 1 ? 1 : (b < 148 * 32 ? b : 148 * 32));
}

}  // namespace

void launch_insert_flags(const double* distance, int64_t n, double tau, uint8_t* flag, int32_t* flag_i32,
                         cudaStream_t st) {
    if (n <= 0) return;
    k_insert_flags<<<grid_for(n), 256, 0, st>>>(distance, n, tau, flag, flag_i32);
    dbg_launch("k_insert_flags", st);
}

void launch_insert_fill(const InsertParams& p, cudaStream_t st) {
    if (p.n_src <= 0) return;
    k_insert_fill<<<grid_for(p.n_src * 32), 256, 0, st>>>(p);
    dbg_launch("k_insert_fill", st);
}

void launch_keep_flags(const int32_t* removed, int64_t n_removed, int64_t n, int32_t* keep, cudaStream_t st) {
    if (n <= 0) return;
    k_fill_one<<<grid_for(n), 256, 0, st>>>(keep, n);  // keep = 1, then 0 at the removed rows
    dbg_launch("k_fill_one", st);
    if (n_removed > 0) k_keep_flags<<<grid_for(n_removed), 256, 0, st>>>(removed, n_removed, n, keep);
    dbg_launch("k_keep_flags", st);
}

void launch_compact_f64(const double* src, double* dst, const int32_t* keep, const int32_t* pos, int64_t n,
                        int width, cudaStream_t st) {
    if (n <= 0 || width <= 0) return;
    k_compact<double><<<grid_for(n * width), 256, 0, st>>>(src, dst, keep, pos, n, width);
    dbg_launch("k_compact_f64", st);
}

void launch_compact_f32(const float* src, float* dst, const int32_t* keep, const int32_t* pos, int64_t n, int width,
                        cudaStream_t st) {
    if (n <= 0 || width <= 0) return;
    k_compact<float><<<grid_for(n * width), 256, 0, st>>>(src, dst, keep, pos, n, width);
    dbg_launch("k_compact_f32", st);
}

}  // namespace tk

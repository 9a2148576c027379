// mapedit.cu — insertion and compaction kernels for the device-resident map (rare, structural
// edits: once per keyframe / every prune_period iterations).  --fmad=false: the inserted means
// follow Pose::apply's Eigen rotation formula operation by operation, like the oracle.
#include "mapedit.cuh"

#include <algorithm>

namespace tk {

namespace {

__global__ void k_insert_flags(const double* __restrict__ distance, int64_t n, double tau, uint8_t* __restrict__ flag,
                               int32_t* __restrict__ flag_i32) {
    pdl_prologue();
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const bool f = !(distance[i] < tau);  // mapper.cpp:30 skips distance < tau only
        flag[i] = f ? 1 : 0;
        flag_i32[i] = f ? 1 : 0;
    }
}

// One warp per source point: geometry on lane 0, the feature row (normalised in fp64) across lanes.
__global__ void __launch_bounds__(256) k_insert_fill(InsertParams p) {
    pdl_prologue();
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
    pdl_prologue();
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        v[i] = 1;
}

__global__ void k_keep_flags(const int32_t* __restrict__ removed, int64_t n_removed, int64_t n,
                             int32_t* __restrict__ keep) {
    pdl_prologue();
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n_removed;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t r = removed[i];
        if (r >= 0 && r < n) keep[r] = 0;
    }
}

template <class T>
__global__ void k_compact(const T* __restrict__ src, T* __restrict__ dst, const int32_t* __restrict__ keep,
                          const int32_t* __restrict__ pos, int64_t n, int width) {
    pdl_prologue();
    const int64_t total = n * width;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = e / width;
        if (keep[r]) dst[static_cast<int64_t>(pos[r]) * width + (e - r * width)] = src[e];
    }
}

// SPLF record (checkpoint.cpp:41-55): f32 mean[3], log_scale[3], quat w,x,y,z, opacity_logit,
// color[3], feature[D]; element-parallel over the n x (14 + D) record array.
__global__ void k_splf_pack(SplfView v, float* __restrict__ rec) {
    pdl_prologue();
    const int W = 14 + v.d;
    const int64_t total = v.n * W;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = e / W;
        const int c = static_cast<int>(e - r * W);
        float x;
        if (c < 3) x = static_cast<float>(v.mean[r * 3 + c]);
        else if (c < 6) x = static_cast<float>(v.log_scale[r * 3 + c - 3]);
        else if (c < 10) x = static_cast<float>(v.rotation[r * 4 + c - 6]);
        else if (c == 10) x = static_cast<float>(v.opacity_logit[r]);
        else if (c < 14) x = static_cast<float>(v.color[r * 3 + c - 11]);
        else x = v.feature[r * v.d + c - 14];
        rec[e] = x;
    }
}

__global__ void k_splf_unpack(const float* __restrict__ rec, SplfView v) {
    pdl_prologue();
    const int W = 14 + v.d;
    const int64_t total = v.n * W;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = e / W;
        const int c = static_cast<int>(e - r * W);
        const float x = rec[e];
        if (c < 3) v.mean[r * 3 + c] = x;
        else if (c < 6) v.log_scale[r * 3 + c - 3] = x;
        else if (c < 10) v.rotation[r * 4 + c - 6] = x;
        else if (c == 10) v.opacity_logit[r] = x;
        else if (c < 14) v.color[r * 3 + c - 11] = x;
        else v.feature[r * v.d + c - 14] = x;
    }
}

// segment_by_query (metrics.cpp:66-94): lane = class, kQP pixels per warp at a time (independent
// dot chains); each pixel's feature row is broadcast channel by channel from registers, the
// embeddings are staged transposed in shared memory (fp64; one chunk of channels per pass, the
// whole D when it fits) and one shared-memory read serves the warp's kQP pixels.  Dots and squared
// norms accumulate in channel order without contraction (the reference's summation); the first
// maximum wins.  Multi-chunk passes carry the running sums through p.acc / p.nacc.
constexpr int kQP = 4;
__device__ __forceinline__ void query_finish(const QueryParams& p, int64_t px, int cb, int cls, int lane,
                                             double dot, double norm2, bool last) {
    const int C = p.classes;
    if (!last) {
        if (cls < C) p.acc[px * C + cls] = dot;
        if (lane == 0 && cb + 32 >= C) p.nacc[px] = norm2;
        return;
    }
    if (p.partial) {
        if (cls < C) p.partial[px * C + cls] = dot;
        if (lane == 0 && cb == 0) p.norm2[px] = norm2;
        return;
    }
    double best = cls < C ? dot : -1e300;  // argmax: first maximum wins (strict >)
    int arg = cls < C ? cls : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
        if (ob > best || (ob == best && oa < arg)) {
            best = ob;
            arg = oa;
        }
    }
    if (lane == 0) {
        if (cb == 0) {
            p.best[px] = best;
            p.labels[px] = norm2 < 1e-12 ? 255 : static_cast<uint8_t>(arg);
        } else if (norm2 >= 1e-12 && best > p.best[px]) {
            p.best[px] = best;
            p.labels[px] = static_cast<uint8_t>(arg);
        }
    }
}

__global__ void __launch_bounds__(512) k_segment_query(QueryParams p, int chunk) {
    pdl_prologue();
    extern __shared__ double et[];  // [chunk][classes]
    const int lane = threadIdx.x & 31;
    const int warps = blockDim.x >> 5;
    const int C = p.classes, D = p.d;
    for (int c0 = 0; c0 < D; c0 += chunk) {
        const int cn = min(chunk, D - c0);
        const bool first = c0 == 0, last = c0 + cn >= D;
        __syncthreads();
        for (int e = threadIdx.x; e < cn * C; e += blockDim.x) {
            const int ci = e / C, k = e - ci * C;
            et[ci * C + k] = p.emb[static_cast<int64_t>(k) * p.d_total + p.c0 + c0 + ci];
        }
        __syncthreads();
        for (int64_t px0 = (static_cast<int64_t>(blockIdx.x) * warps + (threadIdx.x >> 5)) * kQP; px0 < p.n_pixels;
             px0 += static_cast<int64_t>(gridDim.x) * warps * kQP) {
            for (int cb = 0; cb < C; cb += 32) {
                const int cls = cb + lane;
                const int clsr = cls < C ? cls : C - 1;  // clamped read index (result discarded)
                double dot[kQP], nrm[kQP];
                int64_t px[kQP];
#pragma unroll
                for (int u = 0; u < kQP; ++u) {
                    px[u] = min(px0 + u, p.n_pixels - 1);
                    dot[u] = (!first && cls < C) ? p.acc[px[u] * C + cls] : 0.0;
                    nrm[u] = first ? 0.0 : p.nacc[px[u]];
                }
                int cc = 0;
                for (; cc + 32 <= cn; cc += 32) {
                    double fv[kQP];
#pragma unroll
                    for (int u = 0; u < kQP; ++u) fv[u] = static_cast<double>(p.feat[px[u] * D + c0 + cc + lane]);
#pragma unroll 8
                    for (int j = 0; j < 32; ++j) {
                        const double e = et[(cc + j) * C + clsr];
#pragma unroll
                        for (int u = 0; u < kQP; ++u) {
                            const double f = __shfl_sync(0xffffffffu, fv[u], j);
                            nrm[u] += f * f;
                            dot[u] += e * f;
                        }
                    }
                }
                if (cc < cn) {  // channel tail (D % 32)
                    const int m = cn - cc;
                    double fv[kQP];
#pragma unroll
                    for (int u = 0; u < kQP; ++u)
                        fv[u] = lane < m ? static_cast<double>(p.feat[px[u] * D + c0 + cc + lane]) : 0.0;
                    for (int j = 0; j < m; ++j) {
                        const double e = et[(cc + j) * C + clsr];
#pragma unroll
                        for (int u = 0; u < kQP; ++u) {
                            const double f = __shfl_sync(0xffffffffu, fv[u], j);
                            nrm[u] += f * f;
                            dot[u] += e * f;
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < kQP; ++u)
                    if (px0 + u < p.n_pixels) query_finish(p, px0 + u, cb, cls, lane, dot[u], nrm[u], last);
            }
        }
    }
}

// Argmax over the all-reduced partial scores of the D-sharded path.
__global__ void k_query_argmax(const double* __restrict__ scores, const double* __restrict__ norm2, int64_t n,
                               int C, uint8_t* __restrict__ labels) {
    pdl_prologue();
    for (int64_t px = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; px < n;
         px += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (norm2[px] < 1e-12) {
            labels[px] = 255;
            continue;
        }
        int best = 0;
        double bd = -1e300;
        for (int k = 0; k < C; ++k)
            if (scores[px * C + k] > bd) {
                bd = scores[px * C + k];
                best = k;
            }
        labels[px] = static_cast<uint8_t>(best);
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
    launch_k<false>(k_insert_flags, grid_for(n), 256, 0, st, distance, n, tau, flag, flag_i32);
    dbg_launch("k_insert_flags", st);
}

void launch_insert_fill(const InsertParams& p, cudaStream_t st) {
    if (p.n_src <= 0) return;
    launch_k<false>(k_insert_fill, grid_for(p.n_src * 32), 256, 0, st, p);
    dbg_launch("k_insert_fill", st);
}

void launch_keep_flags(const int32_t* removed, int64_t n_removed, int64_t n, int32_t* keep, cudaStream_t st) {
    if (n <= 0) return;
    launch_k<false>(k_fill_one, grid_for(n), 256, 0, st, keep, n);  // keep = 1, then 0 at the removed rows
    dbg_launch("k_fill_one", st);
    if (n_removed > 0) launch_k<false>(k_keep_flags, grid_for(n_removed), 256, 0, st, removed, n_removed, n, keep);
    dbg_launch("k_keep_flags", st);
}

void launch_compact_f64(const double* src, double* dst, const int32_t* keep, const int32_t* pos, int64_t n,
                        int width, cudaStream_t st) {
    if (n <= 0 || width <= 0) return;
    launch_k<false>(k_compact<double>, grid_for(n * width), 256, 0, st, src, dst, keep, pos, n, width);
    dbg_launch("k_compact_f64", st);
}

void launch_splf_pack(const SplfView& v, float* rec, cudaStream_t st) {
    if (v.n <= 0) return;
    launch_k<false>(k_splf_pack, grid_for(v.n * (14 + v.d)), 256, 0, st, v, rec);
    dbg_launch("k_splf_pack", st);
}

void launch_splf_unpack(const float* rec, const SplfView& v, cudaStream_t st) {
    if (v.n <= 0) return;
    launch_k<false>(k_splf_unpack, grid_for(v.n * (14 + v.d)), 256, 0, st, rec, v);
    dbg_launch("k_splf_unpack", st);
}

int segment_query_chunk(int d, int classes) {
    const int fit = static_cast<int>((160 * 1024) / (sizeof(double) * (classes > 0 ? classes : 1)));
    int chunk = fit >= d ? d : (fit / 32) * 32;
    return chunk < 32 ? 32 : chunk;
}

void launch_segment_query(const QueryParams& p, cudaStream_t st) {
    if (p.n_pixels <= 0 || p.d <= 0) return;
    const int chunk = segment_query_chunk(p.d, p.classes);
    const size_t smem = static_cast<size_t>(chunk) * p.classes * sizeof(double);
    static FuncAttrCache attr;
    if (smem > 48 * 1024)
        set_func_attr(attr, reinterpret_cast<const void*>(k_segment_query), cudaFuncAttributeMaxDynamicSharedMemorySize,
                      static_cast<int>(smem), true);
    const int64_t per_sm = std::max<int64_t>(1, (227 * 1024) / static_cast<int64_t>(smem + 1024));
    const int64_t blocks = std::min<int64_t>((p.n_pixels + 16 * kQP - 1) / (16 * kQP), 148 * std::min<int64_t>(per_sm, 4));
    launch_k<false>(k_segment_query, static_cast<unsigned>(blocks), 512, smem, st, p, chunk);
    dbg_launch("k_segment_query", st);
}

void launch_query_argmax(const double* scores, const double* norm2, int64_t n, int classes, uint8_t* labels,
                         cudaStream_t st) {
    if (n <= 0) return;
    launch_k<false>(k_query_argmax, grid_for(n), 256, 0, st, scores, norm2, n, classes, labels);
    dbg_launch("k_query_argmax", st);
}

void launch_compact_f32(const float* src, float* dst, const int32_t* keep, const int32_t* pos, int64_t n, int width,
                        cudaStream_t st) {
    if (n <= 0 || width <= 0) return;
    launch_k<false>(k_compact<float>, grid_for(n * width), 256, 0, st, src, dst, keep, pos, n, width);
    dbg_launch("k_compact_f32", st);
}

}  // namespace tk

// mapping.cu — the per-iteration loss and optimiser kernels of one mapping step
// (map/mapper.cpp:162-255).  Compiled with --fmad=false: the colour/depth L1 and the D-SSIM
// gradient follow ssim.cpp / losses.cpp operation by operation, so grad_color is bit-identical
// to the fp64 oracle; the feature kernels use explicit fmaf (fp32, stated tolerance).
//
// Data per step (config 3: 1200x680, D = 512, 1M Gaussians):
//   colour loss + SSIM: fp64 image maps, ~40 B/pixel/channel of map traffic (L2-resident tiles);
//   feature loss: reads the K selected feature rows (as render_feature) and the keyframe's
//     D-channel row, writes 2 sign bits per channel instead of the fp32 dL/dF image;
//   feature Adam: per Gaussian reads the sign words of its records, then f, m, v (fp32) once.
#include "mapping.cuh"

#include <algorithm>
#include <cstdlib>

#include "tile_stage.cuh"
#include "feature.cuh"
#include "sort.cuh"

namespace tk {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr double kC1 = 0.01 * 0.01;  // ssim.cpp:15-16
constexpr double kC2 = 0.03 * 0.03;
constexpr int kHalo = kSsimWin - 1;

__device__ __forceinline__ double sgn(double v) { return v > 0.0 ? 1.0 : (v < 0.0 ? -1.0 : 0.0); }

// Deterministic block sum of NV doubles (fixed shuffle tree, then warps in order).
template <int NV, int NW = kWarps>
__device__ __forceinline__ void block_sum_store(double (&v)[NV], double* __restrict__ dst) {
    __shared__ double sh[NV][NW];
#pragma unroll
    for (int a = 0; a < NV; ++a)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[a] += __shfl_xor_sync(0xffffffffu, v[a], o);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0)
#pragma unroll
        for (int a = 0; a < NV; ++a) sh[a][warp] = v[a];
    __syncthreads();
    if (threadIdx.x < NV) {
        double s = 0.0;
        for (int w = 0; w < NW; ++w) s += sh[threadIdx.x][w];
        dst[threadIdx.x] = s;
    }
}

// ---------------------------------------------------------------- keyframe preprocessing
__global__ void __launch_bounds__(kThreads) k_gt_valid(const float* __restrict__ gt, int64_t pixels, int d,
                                                       uint8_t* __restrict__ valid, const float* __restrict__ gt_depth,
                                                       unsigned long long* __restrict__ depth_n) {
    pdl_prologue();
    const int lane = threadIdx.x & 31;
    const int64_t nw = static_cast<int64_t>(gridDim.x) * kWarps;
    unsigned long long cnt = 0;
    for (int64_t px = (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5; px < pixels; px += nw) {
        bool any = false;
        if (gt)
            for (int c = lane; c < d; c += 32) any |= gt[px * d + c] != 0.0f;  // losses.cpp:98-100
        any = __any_sync(0xffffffffu, any);
        if (lane == 0) {
            valid[px] = any ? 1 : 0;
            cnt += gt_depth[px] > 0.0f ? 1 : 0;                              // losses.cpp:68-71
        }
    }
    if (lane == 0 && cnt) atomicAdd(depth_n, cnt);
}

// ---------------------------------------------------------------- colour / depth / SSIM
// Window statistics of ssim_with_grad (ssim.cpp:31-50 convolve_valid, then :128-145) for a
// 32 x 8 tile of windows of one channel: the (8+10) x (32+10) input patch of a and b is staged
// in shared memory, the row pass goes to shared memory, the column pass runs per window.  Sums
// run in the reference's tap order, so every statistic is bit-identical to the oracle's.
constexpr int kSW = 32, kSH = 8;
constexpr int kPW = kSW + kHalo, kPH = kSH + kHalo;

__global__ void __launch_bounds__(kThreads) k_ssim_stats(ColorLossParams p) {
    pdl_prologue();
    __shared__ double pa[kPH][kPW], pb[kPH][kPW];
    __shared__ double hs[5][kPH][kSW];
    const int ow = p.w - kHalo, oh = p.h - kHalo;
    const int64_t plane_w = static_cast<int64_t>(oh) * ow;
    const int tx = (ow + kSW - 1) / kSW, ty = (oh + kSH - 1) / kSH;
    const int ntiles = 3 * tx * ty;
    double v[1] = {0.0};
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int c = tile / (tx * ty);
        const int t2 = tile - c * tx * ty;
        const int wx0 = (t2 % tx) * kSW, wy0 = (t2 / tx) * kSH;
        __syncthreads();
        for (int e = threadIdx.x; e < kPH * kPW; e += kThreads) {
            const int ey = e / kPW, ex = e - ey * kPW;
            const int x = wx0 + ex, y = wy0 + ey;
            double va = 0.0, vb = 0.0;
            if (x < p.w && y < p.h) {
                const int64_t q = (static_cast<int64_t>(y) * p.w + x) * 3 + c;
                va = p.color[q];
                vb = static_cast<double>(p.gt_color[q]);
            }
            pa[ey][ex] = va;
            pb[ey][ex] = vb;
        }
        __syncthreads();
        for (int e = threadIdx.x; e < kPH * kSW; e += kThreads) {  // row pass (ssim.cpp:36-41)
            const int ey = e / kSW, ex = e - ey * kSW;
            double sa = 0.0, sb = 0.0, saa = 0.0, sbb = 0.0, sab = 0.0;
#pragma unroll
            for (int i = 0; i < kSsimWin; ++i) {
                const double va = pa[ey][ex + i], vb = pb[ey][ex + i], kw = p.kern[i];
                sa += kw * va;
                sb += kw * vb;
                saa += kw * (va * va);
                sbb += kw * (vb * vb);
                sab += kw * (va * vb);
            }
            hs[0][ey][ex] = sa;
            hs[1][ey][ex] = sb;
            hs[2][ey][ex] = saa;
            hs[3][ey][ex] = sbb;
            hs[4][ey][ex] = sab;
        }
        __syncthreads();
        const int lx = threadIdx.x % kSW, ly = threadIdx.x / kSW;
        const int wx = wx0 + lx, wy = wy0 + ly;
        if (wx >= ow || wy >= oh) continue;
        double st[5];
#pragma unroll
        for (int m = 0; m < 5; ++m) {  // column pass (ssim.cpp:42-48)
            double acc = 0.0;
#pragma unroll
            for (int i = 0; i < kSsimWin; ++i) acc += p.kern[i] * hs[m][ly + i][lx];
            st[m] = acc;
        }
        const double mu_a = st[0], mu_b = st[1];
        const double var_a = st[2] - mu_a * mu_a;
        const double var_b = st[3] - mu_b * mu_b;
        const double cov = st[4] - mu_a * mu_b;
        const double a1 = 2.0 * mu_a * mu_b + kC1;
        const double a2 = 2.0 * cov + kC2;
        const double b1 = mu_a * mu_a + mu_b * mu_b + kC1;
        const double b2 = var_a + var_b + kC2;
        v[0] += (a1 * a2) / (b1 * b2);
        const double d_mu = 2.0 * (mu_b * a2 * b1 - mu_a * a1 * a2) / (b1 * b1 * b2);
        const double d_var = -a1 * a2 / (b1 * b2 * b2);
        const double d_cov = 2.0 * a1 / (b1 * b2);
        double* o = p.win + c * plane_w + static_cast<int64_t>(wy) * ow + wx;
        o[0] = mu_a;
        o[3 * plane_w] = mu_b;
        o[6 * plane_w] = d_mu;
        o[9 * plane_w] = d_var * 2.0;  // the reference's (d_var * 2.0), exact
        o[12 * plane_w] = d_cov;
    }
    block_sum_store<1>(v, p.partial + blockIdx.x * kLossSlots + kSsimSum);
}

// Per pixel: colour L1 (losses.cpp:36-46), the D-SSIM gradient gathered over every window that
// covers the pixel in the reference's (wy, wx) accumulation order (ssim.cpp:147-154), the
// colour-gradient mix (losses.cpp:50-58), depth L1 (losses.cpp:64-80) and the lambda folds
// (losses.cpp:128-130).  Each thread owns a 1 x 4 pixel column of a 16 x 64 tile, so one
// shared-memory window read serves up to four pixels; (inv_count * wgt) comes from a 11 x 11
// table computed like the reference's product.
#ifndef TK_CL_KCR
#define TK_CL_KCR 4
#endif
constexpr int kCX = 16, kCR = TK_CL_KCR, kCY = (kThreads / kCX) * kCR;
constexpr int kCWX = kCX + kHalo, kCWY = kCY + kHalo;
// weight table rows ky = -(kCR-1) .. kHalo+kCR-1: rows outside 0..kHalo hold zeros, so taps of a
// window that does not cover the pixel add +-0 (no branch; sums unchanged bit for bit)
constexpr int kTwRows = kSsimWin + 2 * (kCR - 1);
constexpr size_t kColorSmem = (5 * kCWY * kCWX + kTwRows * kSsimWin) * sizeof(double);

__global__ void __launch_bounds__(kThreads) k_color_loss(ColorLossParams p) {
    pdl_prologue();
    extern __shared__ double smem[];
    double* sw = smem;                        // [5][kCWY][kCWX]
    double* tw = smem + 5 * kCWY * kCWX;      // [kTwRows][11] inv_count * (kern[ky] * kern[kx]), zero rows around
    const int ow = p.w - kHalo, oh = p.h - kHalo;
    const int64_t plane_w = static_cast<int64_t>(oh > 0 ? oh : 0) * (ow > 0 ? ow : 0);
    const int tx = (p.w + kCX - 1) / kCX, ty = (p.h + kCY - 1) / kCY;
    const int lx = threadIdx.x % kCX, lr = threadIdx.x / kCX;
    const double scale = -0.5 * p.lambda1;
    const double fold_d = p.lambda_geo * p.lambda2;
    for (int e = threadIdx.x; e < kTwRows * kSsimWin; e += kThreads) {
        const int ky = e / kSsimWin - (kCR - 1), kx = e % kSsimWin;
        tw[e] = ky >= 0 && ky <= kHalo ? p.inv_count * (p.kern[ky] * p.kern[kx]) : 0.0;
    }
    double v[2] = {0.0, 0.0};
    for (int tile = blockIdx.x; tile < tx * ty; tile += gridDim.x) {
        const int x0 = (tile % tx) * kCX, y0 = (tile / tx) * kCY;
        const int x = x0 + lx, ys = y0 + lr * kCR;
        double g[3][kCR];
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int j = 0; j < kCR; ++j) g[c][j] = 0.0;
        if (p.use_ssim) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                __syncthreads();
                // windows outside the valid range are staged as zeros: their term is
                // tw * (0 + 0 * (a - 0) + 0 * (b - 0)) = +0, which leaves every sum bit-identical
                // (a sum starting at +0 is never -0), so the gather below needs no bounds tests
                for (int e = threadIdx.x; e < kCWY * kCWX; e += kThreads) {
                    const int ey = e / kCWX, ex = e - ey * kCWX;
                    const int wy = y0 - kHalo + ey, wx = x0 - kHalo + ex;
                    const bool ok = wy >= 0 && wy < oh && wx >= 0 && wx < ow;
                    const double* src = p.win + c * plane_w + static_cast<int64_t>(ok ? wy : 0) * ow + (ok ? wx : 0);
#pragma unroll
                    for (int m = 0; m < 5; ++m) sw[(m * kCWY + ey) * kCWX + ex] = ok ? src[m * 3 * plane_w] : 0.0;
                }
                __syncthreads();
                if (x >= p.w) continue;
                double av[kCR], bv[kCR];
#pragma unroll
                for (int j = 0; j < kCR; ++j) {
                    const int y = min(ys + j, p.h - 1);
                    const int64_t q = (static_cast<int64_t>(y) * p.w + x) * 3 + c;
                    av[j] = p.color[q];
                    bv[j] = static_cast<double>(p.gt_color[q]);
                }
                for (int wy = ys - kHalo; wy <= ys + kCR - 1; ++wy) {
                    const int ey = wy - (y0 - kHalo);
#pragma unroll
                    for (int kx = kHalo; kx >= 0; --kx) {  // wx = x - kx ascending
                        const int ex = lx + kHalo - kx;
                        const double* wp = sw + ey * kCWX + ex;
                        const double mu_a = wp[0], mu_b = wp[kCWY * kCWX], d_mu = wp[2 * kCWY * kCWX];
                        const double dv2 = wp[3 * kCWY * kCWX], d_cov = wp[4 * kCWY * kCWX];
#pragma unroll
                        for (int j = 0; j < kCR; ++j) {
                            const int ky = ys + j - wy;
                            g[c][j] += tw[(ky + kCR - 1) * kSsimWin + kx] * (d_mu + dv2 * (av[j] - mu_a) + d_cov * (bv[j] - mu_b));
                        }
                    }
                }
            }
        }
        if (x >= p.w) continue;
#pragma unroll
        for (int j = 0; j < kCR; ++j) {
            const int y = ys + j;
            if (y >= p.h) break;
            const int64_t px = static_cast<int64_t>(y) * p.w + x;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const double diff = p.color[px * 3 + c] - static_cast<double>(p.gt_color[px * 3 + c]);
                v[0] += fmax(fabs(diff) - p.deadband, 0.0);
                double gc = (fabs(diff) > p.deadband ? sgn(diff) : 0.0) * p.inv_color_n;
                if (p.use_ssim) gc = (1.0 - p.lambda1) * gc + scale * g[c][j];
                p.grad_color[px * 3 + c] = gc * p.lambda_geo;
            }
            double gd = 0.0;
            if (p.use_depth) {
                const float t = p.gt_depth[px];
                if (t > 0.0f) {
                    const double diff = p.depth[px] - static_cast<double>(t);
                    v[1] += fmax(fabs(diff) - p.deadband, 0.0);
                    gd = (fabs(diff) > p.deadband ? sgn(diff) : 0.0) * p.inv_depth_n;
                }
            }
            p.grad_depth[px] = gd * fold_d;
        }
    }
    block_sum_store<2>(v, p.partial + blockIdx.x * kLossSlots + kL1Color);
}

// ---------------------------------------------------------------- feature loss
__device__ __forceinline__ float4 fma4(float a, float4 x, float4 acc) {
    acc.x = fmaf(a, x.x, acc.x);
    acc.y = fmaf(a, x.y, acc.y);
    acc.z = fmaf(a, x.z, acc.z);
    acc.w = fmaf(a, x.w, acc.w);
    return acc;
}

__device__ __forceinline__ uint32_t sign_bits(float d) { return (d > 0.0f ? 1u : 0u) | (d < 0.0f ? 2u : 0u); }

__device__ __forceinline__ int64_t tiled_pixel(int64_t v, int width, int height, int tiles_x, bool* valid) {
    const int64_t t = v >> 8;
    const int l = static_cast<int>(v & 255);
    const int x = static_cast<int>(t % tiles_x) * 16 + (l & 15), y = static_cast<int>(t / tiles_x) * 16 + (l >> 4);
    *valid = x < width && y < height;
    return static_cast<int64_t>(y) * width + x;
}

// k_feature_loss_vec over tile-staged rows (tile_stage.cuh): one CTA per 16 x 16 tile; a pixel
// uses its records only when live (count > 0 and a non-zero keyframe row, losses.cpp:98-104);
// warp w then computes pixels 32w..32w+31 two at a time, keyframe rows loaded first, the
// rendered rows from shared memory (or global for unstaged ids), and stores sign(F - GT) as
// 2-bit codes plus the |F - GT| and live-pixel partial sums.  The rendered row, the signs and
// the live count are those of k_feature_loss_vec; the |F - GT| sum differs only in fp64
// summation order.
template <int KMAX, bool FULL>
__global__ void __launch_bounds__(kStagePix, 2) k_feature_loss_staged(FeatLossParams p, int rows) {
    pdl_prologue();
    extern __shared__ __align__(128) unsigned char gsm[];
    const int D = p.d, d4 = D >> 2, wpp = (D + 15) >> 4;
    const StageSmem sm = stage_layout<KMAX>(gsm, rows, D);
    const float* srow = sm.srow;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tiles_x = (p.width + kStageSide - 1) / kStageSide, tiles_y = (p.height + kStageSide - 1) / kStageSide;
    stage_init(sm);
    unsigned phase = 0;
    double v[2] = {0.0, 0.0};
    for (int tile = blockIdx.x; tile < tiles_x * tiles_y; tile += gridDim.x) {
        const int tx0 = (tile % tiles_x) * kStageSide, ty0 = (tile / tiles_x) * kStageSide;
        const int x = tx0 + (tid % kStageSide), y = ty0 + tid / kStageSide;
        const bool in = x < p.width && y < p.height;
        const int64_t px = static_cast<int64_t>(y) * p.width + x;
        const int cnt = in ? p.count[px] : 0;
        const bool live = cnt > 0 && p.gt_valid[px];
        if (live) v[1] += 1.0;
        const StagedPixel<KMAX> sp =
            stage_tile<KMAX>(sm, rows, D, p.feat, p.index, p.weight, p.k, px, in ? (live ? cnt : 0) : -1, phase);
        for (int i = 0; i < 32; i += 2) {
            int ci[2];
            int64_t pxo[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                ci[u] = __shfl_sync(0xffffffffu, sp.c, i + u);
                const int t = warp * 32 + i + u;
                pxo[u] = static_cast<int64_t>(ty0 + t / kStageSide) * p.width + tx0 + (t % kStageSide);
            }
            for (int base = 0; base < d4; base += 128) {
                float4 gt[2][4], acc[2][4];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const float4* grow = reinterpret_cast<const float4*>(p.gt + pxo[u] * D);
#pragma unroll
                    for (int m = 0; m < 4; ++m) {
                        const int q = base + m * 32 + lane;
                        gt[u][m] = (ci[u] > 0 && (FULL || q < d4)) ? __ldcs(grow + q) : make_float4(0.f, 0.f, 0.f, 0.f);
                        acc[u][m] = make_float4(0.f, 0.f, 0.f, 0.f);
                    }
                }
#pragma unroll
                for (int j = 0; j < KMAX; ++j) {
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int sj = __shfl_sync(0xffffffffu, sp.slot[j], i + u);
                        const float wj = __shfl_sync(0xffffffffu, sp.wn[j], i + u);
                        if (j < ci[u] && sj >= 0) {
                            const float4* row = reinterpret_cast<const float4*>(srow + static_cast<size_t>(sj) * D);
#pragma unroll
                            for (int m = 0; m < 4; ++m) {
                                const int q = base + m * 32 + lane;
                                if ((FULL || q < d4)) acc[u][m] = fma4(wj, row[q], acc[u][m]);
                            }
                        } else if (j < ci[u]) {
                            const float4* row = reinterpret_cast<const float4*>(p.feat + static_cast<int64_t>(-1 - sj) * D);
#pragma unroll
                            for (int m = 0; m < 4; ++m) {
                                const int q = base + m * 32 + lane;
                                if ((FULL || q < d4)) acc[u][m] = fma4(wj, __ldg(row + q), acc[u][m]);
                            }
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    if (ci[u] < 0) continue;
                    uint32_t* srw = p.signs + pxo[u] * wpp;
                    float sabs = 0.0f;
#pragma unroll
                    for (int m = 0; m < 4; ++m) {
                        const int q = base + m * 32 + lane;
                        uint32_t byte = 0;
                        if (ci[u] > 0 && (FULL || q < d4)) {
                            const float4 t = gt[u][m];
                            const float dx = acc[u][m].x - t.x, dy = acc[u][m].y - t.y;
                            const float dz = acc[u][m].z - t.z, dw = acc[u][m].w - t.w;
                            sabs += (fabsf(dx) + fabsf(dy)) + (fabsf(dz) + fabsf(dw));
                            byte = sign_bits(dx) | (sign_bits(dy) << 2) | (sign_bits(dz) << 4) | (sign_bits(dw) << 6);
                        }
                        uint32_t word = byte << (8 * (lane & 3));
                        word |= __shfl_xor_sync(0xffffffffu, word, 1);
                        word |= __shfl_xor_sync(0xffffffffu, word, 2);
                        if ((lane & 3) == 0 && (FULL || q < d4)) srw[q >> 2] = word;
                    }
                    v[0] += static_cast<double>(sabs);
                }
            }
        }
        __syncthreads();  // the staged rows and the hash are reused by the next tile
    }
    block_sum_store<2, kStagePix / 32>(v, p.partial + blockIdx.x * kLossSlots + kFeatAbs);
}

// render_feature (render.cpp:319-334) fused with the masked feature L1 (losses.cpp:92-118):
// the rendered row never leaves registers; per channel only sign(F - GT) is stored (the
// gradient is lambda_feat * sign / (feat_n * D), with the scalar applied in the Adam kernel).
// D % 4 == 0: two pixels per warp in 16x16 tile order, 128-bit loads.
__global__ void __launch_bounds__(kThreads) k_feature_loss_vec(FeatLossParams p) {
    pdl_prologue();
    const int lane = threadIdx.x & 31;
    const int64_t nw = static_cast<int64_t>(gridDim.x) * kWarps;
    const int D = p.d, d4 = D >> 2, wpp = (D + 15) >> 4;
    const int tiles_x = (p.width + 15) / 16, tiles_y = (p.height + 15) / 16;
    const int64_t nv = static_cast<int64_t>(tiles_x) * tiles_y * 256;
    double v[2] = {0.0, 0.0};
    for (int64_t v0 = ((static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5) * 2; v0 < nv; v0 += nw * 2) {
        int64_t px[2];
        int c[2], id[2];
        float wn[2];
        bool in[2];
        float4 gt[2][4];
        // keyframe rows first: they do not depend on the records, so their loads overlap the
        // record loads and the Top-K row gather (a pixel without records wastes its first pass)
        auto load_gt = [&](int base, bool first) {
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const float4* grow = reinterpret_cast<const float4*>(p.gt + px[u] * D);
                const bool want = first ? in[u] : c[u] > 0;
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    const int q = base + m * 32 + lane;
                    gt[u][m] = (want && q < d4) ? __ldcs(grow + q) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
        };
#pragma unroll
        for (int u = 0; u < 2; ++u) px[u] = tiled_pixel(v0 + u, p.width, p.height, tiles_x, &in[u]);
        load_gt(0, true);
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            // the record slots load alongside count / mask (one memory round trip, not two)
            int idl = 0;
            double wdl = 0.0;
            if (in[u] && lane < p.k) {
                idl = p.index[px[u] * p.k + lane];
                wdl = p.weight[px[u] * p.k + lane];
            }
            const int cnt = in[u] ? p.count[px[u]] : 0;
            const bool live = cnt > 0 && p.gt_valid[px[u]];
            c[u] = live ? cnt : 0;
            const double wd = lane < c[u] ? wdl : 0.0;
            id[u] = lane < c[u] ? idl : 0;
            double sum = 0.0;
            for (int j = 0; j < c[u]; ++j) sum += __shfl_sync(0xffffffffu, wd, j);
            wn[u] = lane < c[u] ? static_cast<float>(wd / sum) : 0.0f;
            if (lane == 0 && live) v[1] += 1.0;
        }
        const int cmax = max(c[0], c[1]);
        for (int base = 0; base < d4; base += 128) {
            if (base > 0) load_gt(base, false);
            float4 acc[2][4];
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
                for (int m = 0; m < 4; ++m) acc[u][m] = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int j = 0; j < cmax; ++j) {
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int g = __shfl_sync(0xffffffffu, id[u], j);
                    const float wj = __shfl_sync(0xffffffffu, wn[u], j);
                    if (j < c[u]) {
                        const float4* row = reinterpret_cast<const float4*>(p.feat + static_cast<int64_t>(g) * D);
#pragma unroll
                        for (int m = 0; m < 4; ++m) {
                            const int q = base + m * 32 + lane;
                            if (q < d4) acc[u][m] = fma4(wj, __ldg(row + q), acc[u][m]);
                        }
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                if (!in[u]) continue;
                uint32_t* srow = p.signs + px[u] * wpp;
                float sabs = 0.0f;
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    const int q = base + m * 32 + lane;
                    uint32_t byte = 0;
                    if (c[u] > 0 && q < d4) {
                        const float4 t = gt[u][m];
                        const float dx = acc[u][m].x - t.x, dy = acc[u][m].y - t.y;
                        const float dz = acc[u][m].z - t.z, dw = acc[u][m].w - t.w;
                        sabs += (fabsf(dx) + fabsf(dy)) + (fabsf(dz) + fabsf(dw));
                        byte = sign_bits(dx) | (sign_bits(dy) << 2) | (sign_bits(dz) << 4) | (sign_bits(dw) << 6);
                    }
                    uint32_t word = byte << (8 * (lane & 3));
                    word |= __shfl_xor_sync(0xffffffffu, word, 1);
                    word |= __shfl_xor_sync(0xffffffffu, word, 2);
                    if ((lane & 3) == 0 && q < d4) srow[q >> 2] = word;
                }
                v[0] += static_cast<double>(sabs);
            }
        }
    }
    block_sum_store<2>(v, p.partial + blockIdx.x * kLossSlots + kFeatAbs);
}

// Any D: one pixel per warp, scalar channels.
__global__ void __launch_bounds__(kThreads) k_feature_loss_scalar(FeatLossParams p) {
    pdl_prologue();
    const int lane = threadIdx.x & 31;
    const int64_t nw = static_cast<int64_t>(gridDim.x) * kWarps;
    const int D = p.d, wpp = (D + 15) >> 4;
    const int64_t P = static_cast<int64_t>(p.width) * p.height;
    double v[2] = {0.0, 0.0};
    for (int64_t px = (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5; px < P; px += nw) {
        const int cnt = p.count[px];
        const bool live = cnt > 0 && p.gt_valid[px];
        const int c = live ? cnt : 0;
        int id = 0;
        double wd = 0.0;
        if (lane < c) {
            id = p.index[px * p.k + lane];
            wd = p.weight[px * p.k + lane];
        }
        double sum = 0.0;
        for (int j = 0; j < c; ++j) sum += __shfl_sync(0xffffffffu, wd, j);
        const float wn = lane < c ? static_cast<float>(wd / sum) : 0.0f;
        if (lane == 0 && live) v[1] += 1.0;
        for (int base = 0; base < D; base += 32) {
            const int q = base + lane;
            float acc = 0.0f;
            for (int j = 0; j < c; ++j) {
                const int g = __shfl_sync(0xffffffffu, id, j);
                const float wj = __shfl_sync(0xffffffffu, wn, j);
                if (q < D) acc = fmaf(wj, __ldg(p.feat + static_cast<int64_t>(g) * D + q), acc);
            }
            uint32_t bits = 0;
            if (c > 0 && q < D) {
                const float dq = acc - p.gt[px * D + q];
                v[0] += static_cast<double>(fabsf(dq));
                bits = sign_bits(dq);
            }
            uint32_t word = bits << (2 * (lane & 15));
#pragma unroll
            for (int o = 1; o < 16; o <<= 1) word |= __shfl_xor_sync(0xffffffffu, word, o);
            if ((lane & 15) == 0 && q < D) p.signs[px * wpp + (q >> 4)] = word;
        }
    }
    block_sum_store<2>(v, p.partial + blockIdx.x * kLossSlots + kFeatAbs);
}

// Loss values (losses.cpp:84-126) from the per-block partials, summed in a fixed order.
__global__ void __launch_bounds__(kThreads) k_loss_finalize(FinalizeParams p) {
    pdl_prologue();
    __shared__ double tot[kLossSlots];
    for (int s = 0; s < kLossSlots; ++s) {
        double v[1] = {0.0};
        for (int b = threadIdx.x; b < p.nparts; b += kThreads) v[0] += p.partial[b * kLossSlots + s];
        block_sum_store<1>(v, &tot[s]);
        __syncthreads();
    }
    if (threadIdx.x != 0) return;
    if (p.replicas != 1.0) {  // colour / depth / SSIM / feat_n are identical on every shard
        tot[kL1Color] /= p.replicas;
        tot[kL1Depth] /= p.replicas;
        tot[kSsimSum] /= p.replicas;
        tot[kFeatCount] /= p.replicas;
    }
    const double l1_color = tot[kL1Color] * p.inv_color_n;
    double secondary = 0.0;
    if (p.use_ssim) secondary = 0.5 * (1.0 - tot[kSsimSum] * p.inv_count);
    else if (p.secondary_l1) secondary = l1_color;
    const double l1_depth = p.use_depth ? tot[kL1Depth] * p.inv_depth_n : 0.0;
    const double geo = (1.0 - p.lambda1) * l1_color + p.lambda1 * secondary + p.lambda2 * l1_depth;
    double feat = 0.0;
    float fscale = 0.0f;
    if (p.feature_step && tot[kFeatCount] > 0.0) {
        const double inv = 1.0 / (tot[kFeatCount] * p.d);
        feat = tot[kFeatAbs] * inv;
        fscale = static_cast<float>(p.lambda_feat * inv);
    }
    const double lf = p.feature_step ? p.lambda_feat : 0.0;
    p.values[0] = p.lambda_geo * geo + lf * feat;
    p.values[1] = geo;
    p.values[2] = feat;
    if (p.feat_scale) *p.feat_scale = fscale;
}

// update_contribution_stats (mapper.cpp:68-73): Top-K selection counts (integer atomics).
__global__ void k_topk_stats(const int32_t* __restrict__ index, const uint8_t* __restrict__ count, int64_t pixels,
                             int k, int32_t* __restrict__ topk_count) {
    pdl_prologue();
    for (int64_t px = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; px < pixels;
         px += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int c = count[px];
        for (int j = 0; j < c; ++j) atomicAdd(topk_count + index[px * k + j], 1);
    }
}

// ---------------------------------------------------------------- feature backward + Adam
// w * sign for the 2-bit code at bit `sh` (01 = +1, 10 = -1, 00 = 0): selects, no conversions.
__device__ __forceinline__ float signed_w(uint32_t bits, int sh, float w) {
    float t = (bits >> sh) & 1u ? w : 0.0f;
    return (bits >> (sh + 1)) & 1u ? -w : t;
}

// adam_step (optimizer.cpp:57-61) in fp32 with the bias corrections as host reciprocals and a
// reciprocal-sqrt / fast-divide epilogue (the fp32 feature path's stated tolerance).
__device__ __forceinline__ float adam1(float g, float& m, float& v, float f, const AdamStepParams& p) {
    m = fmaf(p.beta1, m, p.one_m_beta1 * g);
    v = fmaf(p.beta2, v, p.one_m_beta2 * g * g);
    const float mhat = m * p.inv_bc1, vhat = v * p.inv_bc2;
    const float den = vhat * rsqrtf(fmaxf(vhat, 1e-30f)) + p.eps;
    return f - __fdividef(p.lr * mhat, den);
}

// One Adam step of a channel quad (gradient a * scale) and its squared-norm contribution: the one
// code path of the eager step and of k_feature_catchup's replay, so both round alike.
__device__ __forceinline__ float adam_quad(float4& f, float4& mm, float4& vv, float4 a, float scale,
                                           const AdamStepParams& s) {
    f.x = adam1(a.x * scale, mm.x, vv.x, f.x, s);
    f.y = adam1(a.y * scale, mm.y, vv.y, f.y, s);
    f.z = adam1(a.z * scale, mm.z, vv.z, f.z, s);
    f.w = adam1(a.w * scale, mm.w, vv.w, f.w, s);
    return f.x * f.x + f.y * f.y + f.z * f.z + f.w * f.w;
}

__device__ __forceinline__ float4 scale4(float4 f, float inv) {
    f.x *= inv;
    f.y *= inv;
    f.z *= inv;
    f.w *= inv;
    return f;
}

__device__ __forceinline__ float warp_sum(float s) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

#ifndef SIGN_GROUP
#define SIGN_GROUP 2
#endif
// Sum over records [r0, r1) of w_j * sign(F - F_gt)[px_j] for the channel pass at `base`
// (4 float4 per lane), records in slot order.
template <int GROUP = SIGN_GROUP>
__device__ __forceinline__ void accum_signs(const FeatAdamParams& p, int r0, int r1, int base, int lane, float scale,
                                            float4 (&acc)[4]) {
    const int d4 = p.d >> 2, wpp = (p.d + 15) >> 4;
    const uint32_t* __restrict__ signs = p.signs;
    for (int r = r0; r < r1; r += 32) {
        const int nr = min(32, r1 - r);
        int64_t spx = 0;
        float sw = 0.f;
        if (lane < nr) {
            const uint32_t s = p.slots[r + lane];
            spx = static_cast<int64_t>(s / static_cast<uint32_t>(p.k));
            sw = p.wnorm[s];
        }
        // kGroup records' sign words are loaded before any is summed (the loads overlap); the
        // sums still run record by record, so the result is that of the sequential sweep
        constexpr int kGroup = GROUP;
        for (int j = 0; j < nr; j += kGroup) {
            const uint32_t* srow[kGroup];
            float wj[kGroup];
            uint32_t bw[kGroup][4];
#pragma unroll
            for (int t = 0; t < kGroup; ++t) {
                srow[t] = signs + __shfl_sync(0xffffffffu, spx, j + t) * wpp;
                wj[t] = __shfl_sync(0xffffffffu, sw, j + t);
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    const int q = base + m * 32 + lane;
                    bw[t][m] = (j + t < nr && q < d4) ? __ldg(srow[t] + (q >> 2)) >> (8 * (q & 3)) : 0u;
                }
            }
#pragma unroll
            for (int t = 0; t < kGroup; ++t) {
                if (j + t >= nr) break;
                if (!isfinite(wj[t])) {  // backward.cpp:296-302: all-zero gradient rows are skipped
                    bool any = false;
                    for (int q = lane; q < wpp; q += 32) any |= srow[t][q] != 0u;
                    if (!__any_sync(0xffffffffu, any) || scale == 0.0f) continue;
                }
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    acc[m].x += signed_w(bw[t][m], 0, wj[t]);
                    acc[m].y += signed_w(bw[t][m], 2, wj[t]);
                    acc[m].z += signed_w(bw[t][m], 4, wj[t]);
                    acc[m].w += signed_w(bw[t][m], 6, wj[t]);
                }
            }
        }
    }
}

// backward_feature (backward.cpp:288-319) over the sign image, fused with the feature Adam
// step and the renormalisation of mapper.cpp:239-252.  One warp per Gaussian (all N: Adam
// moves every row through its moments); records summed in (pixel, slot) order.  LONG = false:
// every Gaussian with <= kLongSeg records; LONG = true: the long Gaussians of the plan, whose
// chunk partials (k_feature_adam_chunks) are added in chunk order.
template <bool LONG, bool LAZY>
__global__ void __launch_bounds__(kThreads) k_feature_adam_vec(FeatAdamParams p, LongPlan plan) {
    pdl_prologue();
    const int lane = threadIdx.x & 31;
    const int64_t nw = static_cast<int64_t>(gridDim.x) * kWarps;
    const int64_t warp_id = (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
    const int D = p.d, d4 = D >> 2;
    const float scale = *p.scale;
    // One row: Adam over its channel quads (gradient = sign sums of its records, or the long
    // plan's chunk partials), then the renormalisation (mapper.cpp:249).
    auto process_row = [&](int64_t g, int r0, int r1, int4 lg, bool loaded, float4 (&fk)[4], float4 (&mk)[4],
                           float4 (&vk)[4]) {
        float4* __restrict__ frow = reinterpret_cast<float4*>(p.feat + g * D);
        float4* __restrict__ mrow = reinterpret_cast<float4*>(p.m + g * D);
        float4* __restrict__ vrow = reinterpret_cast<float4*>(p.v + g * D);
        auto load_pass = [&](int base) {
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const int q = base + m * 32 + lane;
                if (q < d4) {
                    fk[m] = __ldcs(frow + q);
                    mk[m] = __ldcs(mrow + q);
                    vk[m] = __ldcs(vrow + q);
                }
            }
        };
        if (!loaded) load_pass(0);
        if (p.last && lane == 0) p.last[g] = p.cur;
        float ss = 0.0f;
        for (int base = 0; base < d4; base += 128) {
            if (base > 0) load_pass(base);
            float4 acc[4];
#pragma unroll
            for (int m = 0; m < 4; ++m) acc[m] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (!LONG) {
                accum_signs(p, r0, r1, base, lane, scale, acc);
            } else {
                for (int c = 0; c < lg.z; ++c) {
                    const float4* part = reinterpret_cast<const float4*>(plan.partial + static_cast<int64_t>(lg.y + c) * D);
#pragma unroll
                    for (int m = 0; m < 4; ++m) {
                        const int q = base + m * 32 + lane;
                        if (q < d4) {
                            const float4 t = part[q];
                            acc[m].x += t.x;
                            acc[m].y += t.y;
                            acc[m].z += t.z;
                            acc[m].w += t.w;
                        }
                    }
                }
            }
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const int q = base + m * 32 + lane;
                if (q >= d4) continue;
                float4 f = fk[m], mm = mk[m], vv = vk[m];
                ss += adam_quad(f, mm, vv, acc[m], scale, p.st);
                __stcs(mrow + q, mm);
                __stcs(vrow + q, vv);
                fk[m] = f;
                if (d4 > 128) frow[q] = f;
            }
        }
        const float ssum = warp_sum(ss);
        if (p.row_ss) {  // D-sharded: the norm needs every shard's channels (k_feature_renorm)
            if (lane == 0) p.row_ss[g] = ssum;
            if (d4 <= 128)
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    const int q = m * 32 + lane;
                    if (q < d4) __stcs(frow + q, fk[m]);
                }
            return;
        }
        const bool renorm = ssum > 1e-24f;  // norm > 1e-12 (mapper.cpp:249)
        const float inv = renorm ? rsqrtf(ssum) : 1.0f;
        if (d4 <= 128) {
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const int q = m * 32 + lane;
                if (q < d4) __stcs(frow + q, renorm ? scale4(fk[m], inv) : fk[m]);
            }
        } else if (renorm) {
            for (int q = lane; q < d4; q += 32) {
                float4 f = frow[q];
                f.x *= inv;
                f.y *= inv;
                f.z *= inv;
                f.w *= inv;
                frow[q] = f;
            }
        }
    };
    float4 fk[4], mk[4], vk[4];
    if (LONG) {
        for (int64_t wi = warp_id; wi < plan.counters[1]; wi += nw) {
            const int4 lg = plan.longs[wi];
            process_row(lg.x, p.seg[lg.x], p.seg[lg.x + 1], lg, false, fk, mk, vk);
        }
    } else if (LAZY) {
        // only the rows with records (the active list): their sign sums were gathered by
        // k_active_grad into p.grad, so the Adam pass is a plain stream (no record sweep here)
        const int na = *p.n_active;
        for (int64_t wi = warp_id; wi < na; wi += nw) {
            const int64_t g = p.active[wi];
            const int r0 = p.seg[g], r1 = p.seg[g + 1];
            if (r1 - r0 > kLongSeg) continue;
            float4* __restrict__ frow = reinterpret_cast<float4*>(p.feat + g * D);
            float4* __restrict__ mrow = reinterpret_cast<float4*>(p.m + g * D);
            float4* __restrict__ vrow = reinterpret_cast<float4*>(p.v + g * D);
            const float4* __restrict__ grow = reinterpret_cast<const float4*>(p.grad + wi * D);
            float4 acc[4];
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const int q = m * 32 + lane;
                if (q < d4) {
                    fk[m] = __ldcs(frow + q);
                    mk[m] = __ldcs(mrow + q);
                    vk[m] = __ldcs(vrow + q);
                    acc[m] = __ldcs(grow + q);
                }
            }
            if (lane == 0) p.last[g] = p.cur;
            float ss = 0.0f;
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const int q = m * 32 + lane;
                if (q >= d4) continue;
                ss += adam_quad(fk[m], mk[m], vk[m], acc[m], scale, p.st);
                __stcs(mrow + q, mk[m]);
                __stcs(vrow + q, vk[m]);
            }
            const float ssum = warp_sum(ss);
            const bool renorm = ssum > 1e-24f;  // norm > 1e-12 (mapper.cpp:249)
            const float inv = renorm ? rsqrtf(ssum) : 1.0f;
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const int q = m * 32 + lane;
                if (q < d4) __stcs(frow + q, renorm ? scale4(fk[m], inv) : fk[m]);
            }
        }
    } else {
        for (int64_t g = warp_id; g < p.n; g += nw) {
            float4* __restrict__ frow = reinterpret_cast<float4*>(p.feat + g * D);
            float4* __restrict__ mrow = reinterpret_cast<float4*>(p.m + g * D);
            float4* __restrict__ vrow = reinterpret_cast<float4*>(p.v + g * D);
            // the row's parameter / moment loads go out first: they overlap the segment bounds and
            // the record sweep (a skipped long row only wastes its first pass of loads)
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const int q = m * 32 + lane;
                if (q < d4) {
                    fk[m] = __ldcs(frow + q);
                    mk[m] = __ldcs(mrow + q);
                    vk[m] = __ldcs(vrow + q);
                }
            }
            const int r0 = p.seg[g], r1 = p.seg[g + 1];
            if (r1 - r0 > kLongSeg) continue;
            process_row(g, r0, r1, make_int4(0, 0, 0, 0), true, fk, mk, vk);
        }
    }
}

// Lazy step, phase 1: the sign sums of every active row with at most kLongSeg records, in slot
// order (accum_signs, the eager kernel's sweep), into p.grad[active position].  Only the sums are
// held per lane, so twice the warps of the Adam kernel are resident to hide the sweep's latency.
__global__ void __launch_bounds__(kThreads) k_active_grad(FeatAdamParams p) {
    pdl_prologue();
    const int lane = threadIdx.x & 31;
    const int64_t nw = static_cast<int64_t>(gridDim.x) * kWarps;
    const int D = p.d, d4 = D >> 2;
    const float scale = *p.scale;
    const int na = *p.n_active;
    for (int64_t wi = (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5; wi < na; wi += nw) {
        const int64_t g = p.active[wi];
        const int r0 = p.seg[g], r1 = p.seg[g + 1];
        if (r1 - r0 > kLongSeg) continue;
        float4 acc[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) acc[m] = make_float4(0.f, 0.f, 0.f, 0.f);
        accum_signs(p, r0, r1, 0, lane, scale, acc);
        float4* __restrict__ grow = reinterpret_cast<float4*>(p.grad + wi * D);
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const int q = m * 32 + lane;
            if (q < d4) grow[q] = acc[m];
        }
    }
}

// Replay of the zero-gradient feature steps a lazy step skipped (rows without records): steps
// last[g] + 1 .. target of every stale row (ONLY_ACTIVE: of the rows with records in p.seg, before
// a step reads them), each with its own constants tab[t], the row held in registers throughout.
// Step by step it runs the eager kernel's arithmetic for a row with no records (gradient +0,
// adam_quad, warp_sum, renormalisation), so the result is bit-identical to having run every step
// eagerly.  D % 4 == 0 and D <= 512 (one register pass per row).
template <bool ONLY_ACTIVE>
__global__ void __launch_bounds__(kThreads) k_feature_catchup(FeatAdamParams p, int target) {
    pdl_prologue();
    const int lane = threadIdx.x & 31;
    const int64_t nw = static_cast<int64_t>(gridDim.x) * kWarps;
    const int D = p.d, d4 = D >> 2;
    const int64_t warp_id = (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
    const int64_t count = ONLY_ACTIVE ? *p.n_active : (p.n + 31) / 32;
    for (int64_t wi = warp_id; wi < count; wi += nw) {
      // ONLY_ACTIVE: one active row per warp visit; else 32 consecutive rows tested together
      const int64_t g0 = ONLY_ACTIVE ? 0 : wi * 32;
      const int64_t gl = ONLY_ACTIVE ? (lane == 0 ? p.active[wi] : -1) : g0 + lane;
      int from_l = target;
      if (gl >= 0 && gl < p.n) from_l = p.last[gl];
      unsigned stale = __ballot_sync(0xffffffffu, from_l < target);
      while (stale) {
        const int l = __ffs(stale) - 1;
        stale &= stale - 1;
        const int64_t g = ONLY_ACTIVE ? __shfl_sync(0xffffffffu, gl, l) : g0 + l;
        const int from = __shfl_sync(0xffffffffu, from_l, l);
        float4* __restrict__ frow = reinterpret_cast<float4*>(p.feat + g * D);
        float4* __restrict__ mrow = reinterpret_cast<float4*>(p.m + g * D);
        float4* __restrict__ vrow = reinterpret_cast<float4*>(p.v + g * D);
        float4 fk[4], mk[4], vk[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const int q = m * 32 + lane;
            if (q < d4) {
                fk[m] = __ldcs(frow + q);
                mk[m] = __ldcs(mrow + q);
                vk[m] = __ldcs(vrow + q);
            }
        }
        const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int t = from + 1; t <= target; ++t) {
            const AdamStepParams st = p.tab[t];
            float ss = 0.0f;
#pragma unroll
            for (int m = 0; m < 4; ++m)
                if (m * 32 + lane < d4) ss += adam_quad(fk[m], mk[m], vk[m], zero, 0.0f, st);
            const float ssum = warp_sum(ss);
            const bool renorm = ssum > 1e-24f;
            const float inv = renorm ? rsqrtf(ssum) : 1.0f;
            if (renorm)
#pragma unroll
                for (int m = 0; m < 4; ++m) fk[m] = scale4(fk[m], inv);
        }
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const int q = m * 32 + lane;
            if (q < d4) {
                __stcs(frow + q, fk[m]);
                __stcs(mrow + q, mk[m]);
                __stcs(vrow + q, vk[m]);
            }
        }
        if (lane == 0) p.last[g] = target;
      }
    }
}

__global__ void k_active_rows(const int32_t* __restrict__ seg, int64_t n, int32_t* __restrict__ active,
                              int32_t* __restrict__ n_active) {
    pdl_prologue();
    const int lane = threadIdx.x & 31;
    for (int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g - lane < n;
         g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const bool a = g < n && seg[g + 1] > seg[g];
        const unsigned m = __ballot_sync(0xffffffffu, a);
        int base = 0;
        if (lane == 0 && m) base = atomicAdd(n_active, __popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (a) active[base + __popc(m & ((1u << lane) - 1u))] = static_cast<int32_t>(g);
    }
}

__global__ void k_fill_i32(int32_t* __restrict__ a, int64_t n, int32_t value) {
    pdl_prologue();
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        a[i] = value;
}

// One warp per chunk of a long segment: its sign sums into the plan's partial rows.
__global__ void __launch_bounds__(kThreads) k_feature_adam_chunks(FeatAdamParams p, LongPlan plan) {
    pdl_prologue();
    const int lane = threadIdx.x & 31;
    const int64_t nw = static_cast<int64_t>(gridDim.x) * kWarps;
    const int D = p.d, d4 = D >> 2;
    const float scale = *p.scale;
    const int ni = plan.counters[0];
    for (int64_t it = (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5; it < ni; it += nw) {
        const int4 item = plan.items[it];
        const int r0 = item.y, r1 = item.z;
        for (int base = 0; base < d4; base += 128) {
            float4 acc[4];
#pragma unroll
            for (int m = 0; m < 4; ++m) acc[m] = make_float4(0.f, 0.f, 0.f, 0.f);
            accum_signs(p, r0, r1, base, lane, scale, acc);
            float4* dst = reinterpret_cast<float4*>(plan.partial + static_cast<int64_t>(item.w) * D);
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const int q = base + m * 32 + lane;
                if (q < d4) dst[q] = acc[m];
            }
        }
    }
}

__global__ void __launch_bounds__(kThreads) k_feature_adam_scalar(FeatAdamParams p) {
    pdl_prologue();
    const int lane = threadIdx.x & 31;
    const int64_t nw = static_cast<int64_t>(gridDim.x) * kWarps;
    const int D = p.d, wpp = (D + 15) >> 4;
    const float scale = *p.scale;
    for (int64_t g = (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5; g < p.n; g += nw) {
        const int r0 = p.seg[g], r1 = p.seg[g + 1];
        if (p.last && lane == 0) p.last[g] = p.cur;
        float* frow = p.feat + g * D;
        float ss = 0.0f;
        for (int base = 0; base < D; base += 32) {
            const int q = base + lane;
            float acc = 0.0f;
            for (int r = r0; r < r1; ++r) {
                const uint32_t s = p.slots[r];
                const int64_t pxj = static_cast<int64_t>(s / static_cast<uint32_t>(p.k));
                const float wj = p.wnorm[s];
                const uint32_t* srow = p.signs + pxj * wpp;
                if (!isfinite(wj)) {
                    bool any = false;
                    for (int t = lane; t < wpp; t += 32) any |= srow[t] != 0u;
                    if (!__any_sync(0xffffffffu, any) || scale == 0.0f) continue;
                }
                if (q < D) acc += signed_w(srow[q >> 4], 2 * (q & 15), wj);
            }
            if (q < D) {
                float mm = p.m[g * D + q], vv = p.v[g * D + q];
                const float f = adam1(acc * scale, mm, vv, frow[q], p.st);
                p.m[g * D + q] = mm;
                p.v[g * D + q] = vv;
                frow[q] = f;
                ss += f * f;
            }
        }
        const float ssum = warp_sum(ss);
        if (p.row_ss) {  // D-sharded: k_feature_renorm scales once the norms are all-reduced
            if (lane == 0) p.row_ss[g] = ssum;
            continue;
        }
        const float norm = sqrtf(ssum);
        if (norm > 1e-12f)
            for (int q = lane; q < D; q += 32) frow[q] /= norm;
    }
}

__global__ void k_feature_renorm(float* __restrict__ feat, const float* __restrict__ ss, int64_t n, int d) {
    pdl_prologue();
    const int64_t total = n * d;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const float s2 = ss[e / d];
        if (s2 > 1e-24f) feat[e] *= rsqrtf(s2);
    }
}

inline unsigned capped_grid(int64_t items, int per_block, int64_t cap) {
    const int64_t b = (items + per_block - 1) / per_block;
    return static_cast<unsigned>(b < 1 ? 1 : (b < cap ? b : cap));
}

}  // namespace

void launch_gt_valid(const float* gt, int64_t pixels, int d, uint8_t* valid, int64_t* depth_n_out,
                     const float* gt_depth, cudaStream_t st) {
    cudaMemsetAsync(depth_n_out, 0, sizeof(int64_t), st);
    if (pixels <= 0) return;
    launch_k<false>(k_gt_valid, capped_grid(pixels, kWarps, 148 * 16), kThreads, 0, st, 
        gt, pixels, d, valid, gt_depth, reinterpret_cast<unsigned long long*>(depth_n_out));
    dbg_launch("k_gt_valid", st);
}

void launch_color_loss(const ColorLossParams& p, cudaStream_t st) {
    const int64_t P = static_cast<int64_t>(p.w) * p.h;
    if (P <= 0) return;
    if (p.use_ssim) {
        const int ow = p.w - kHalo, oh = p.h - kHalo;
        const int64_t tiles = 3LL * ((ow + kSW - 1) / kSW) * ((oh + kSH - 1) / kSH);
        launch_k<false>(k_ssim_stats, capped_grid(tiles, 1, kLossBlocks), kThreads, 0, st, p);
        dbg_launch("k_ssim_stats", st);
    }
    static FuncAttrCache attr;
    set_func_attr(attr, reinterpret_cast<const void*>(k_color_loss), cudaFuncAttributeMaxDynamicSharedMemorySize,
                  static_cast<int>(kColorSmem));
    const int64_t tiles = static_cast<int64_t>((p.w + kCX - 1) / kCX) * ((p.h + kCY - 1) / kCY);
    launch_k<false>(k_color_loss, capped_grid(tiles, 1, kLossBlocks), kThreads, kColorSmem, st, p);
    dbg_launch("k_color_loss", st);
}

template <int KMAX>
bool launch_feature_loss_staged(const FeatLossParams& p, cudaStream_t st) {
    constexpr size_t kBudget = 112 * 1024;
    const int rows = stage_rows<KMAX>(kBudget, p.d);
    if (rows < 8) return false;
    const int tiles = ((p.width + kStageSide - 1) / kStageSide) * ((p.height + kStageSide - 1) / kStageSide);
    const int grid = std::min(std::min(tiles, 148 * 2), kLossBlocks);
    if (p.d % 512 == 0) {  // no per-quad bounds checks (identical arithmetic)
        static FuncAttrCache attr;
        set_func_attr(attr, reinterpret_cast<const void*>(k_feature_loss_staged<KMAX, true>),
                      cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kBudget));
        launch_k<false>(k_feature_loss_staged<KMAX, true>, grid, kStagePix, stage_smem_bytes<KMAX>(rows, p.d), st, p,
                        rows);
    } else {
        static FuncAttrCache attr;
        set_func_attr(attr, reinterpret_cast<const void*>(k_feature_loss_staged<KMAX, false>),
                      cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kBudget));
        launch_k<false>(k_feature_loss_staged<KMAX, false>, grid, kStagePix, stage_smem_bytes<KMAX>(rows, p.d), st, p,
                        rows);
    }
    return true;
}

bool loss_staged_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("TK_LOSS_STAGED");
        return !(e && e[0] == '0');
    }();
    return on;
}

void launch_feature_loss(const FeatLossParams& p, cudaStream_t st) {
    const int64_t P = static_cast<int64_t>(p.width) * p.height;
    if (P <= 0 || p.d <= 0) return;
    const bool vec = (p.d % 4) == 0 && (reinterpret_cast<uintptr_t>(p.feat) % 16) == 0 &&
                     (reinterpret_cast<uintptr_t>(p.gt) % 16) == 0;
    if (vec && loss_staged_enabled() && p.k <= 8 &&
        (p.k <= 3 ? launch_feature_loss_staged<3>(p, st) : p.k <= 4 ? launch_feature_loss_staged<4>(p, st) : launch_feature_loss_staged<8>(p, st))) {
        dbg_launch("k_feature_loss_staged", st);
        return;
    }
    if (vec) launch_k<false>(k_feature_loss_vec, capped_grid((P + 1) / 2, kWarps, kLossBlocks), kThreads, 0, st, p);
    else launch_k<false>(k_feature_loss_scalar, capped_grid(P, kWarps, kLossBlocks), kThreads, 0, st, p);
    dbg_launch("k_feature_loss", st);
}

void launch_loss_finalize(const FinalizeParams& p, cudaStream_t st) {
    launch_k<false>(k_loss_finalize, 1, kThreads, 0, st, p);
    dbg_launch("k_loss_finalize", st);
}

void launch_topk_stats(const int32_t* index, const uint8_t* count, int64_t pixels, int k, int32_t* topk_count,
                       cudaStream_t st) {
    if (pixels <= 0 || k <= 0) return;
    launch_k<false>(k_topk_stats, capped_grid(pixels, 256, 148 * 8), 256, 0, st, index, count, pixels, k, topk_count);
    dbg_launch("k_topk_stats", st);
}

void launch_feature_renorm(float* feat, const float* ss, int64_t n, int d, cudaStream_t st) {
    if (n <= 0 || d <= 0) return;
    launch_k<false>(k_feature_renorm, capped_grid(n * d, 256, 148 * 32), 256, 0, st, feat, ss, n, d);
    dbg_launch("k_feature_renorm", st);
}

void launch_feature_adam(const FeatAdamParams& p, cudaStream_t st) {
    if (p.n <= 0 || p.d <= 0) return;
    const bool vec = (p.d % 4) == 0 && (reinterpret_cast<uintptr_t>(p.feat) % 16) == 0 &&
                     (reinterpret_cast<uintptr_t>(p.m) % 16) == 0 && (reinterpret_cast<uintptr_t>(p.v) % 16) == 0;
    if (vec) {
        if (p.lazy) {
            launch_k<false>(k_active_grad, 148 * 32, kThreads, 0, st, p);
            dbg_launch("k_active_grad", st);
            launch_k<false>(k_feature_adam_vec<false, true>, 148 * 16, kThreads, 0, st, p, p.plan);
        } else {
            launch_k<false>(k_feature_adam_vec<false, false>, capped_grid(p.n, kWarps, 148 * 32), kThreads, 0, st, p, p.plan);
        }
        dbg_launch("k_feature_adam_vec", st);
        launch_k<false>(k_feature_adam_chunks, 148 * 8, kThreads, 0, st, p, p.plan);
        dbg_launch("k_feature_adam_chunks", st);
        launch_k<false>(k_feature_adam_vec<true, false>, 148 * 4, kThreads, 0, st, p, p.plan);
        dbg_launch("k_feature_adam_vec<long>", st);
    } else {
        launch_k<false>(k_feature_adam_scalar, capped_grid(p.n, kWarps, 148 * 32), kThreads, 0, st, p);
        dbg_launch("k_feature_adam_scalar", st);
    }
}

bool feature_adam_lazy_ok(const FeatAdamParams& p) {
    return p.d > 0 && (p.d % 4) == 0 && p.d <= 512 && !p.row_ss && p.last && p.tab && p.active && p.n_active &&
           p.grad && p.cap_active > 0 &&
           (reinterpret_cast<uintptr_t>(p.feat) % 16) == 0 && (reinterpret_cast<uintptr_t>(p.m) % 16) == 0 &&
           (reinterpret_cast<uintptr_t>(p.v) % 16) == 0;
}

void launch_feature_catchup(const FeatAdamParams& p, int target, bool only_active, cudaStream_t st) {
    if (p.n <= 0 || p.d <= 0 || target <= 0) return;
    const unsigned grid = capped_grid(p.n, kWarps, 148 * 32);
    if (only_active) launch_k<false>(k_feature_catchup<true>, grid, kThreads, 0, st, p, target);
    else launch_k<false>(k_feature_catchup<false>, grid, kThreads, 0, st, p, target);
    dbg_launch("k_feature_catchup", st);
}

void launch_active_rows(const int32_t* seg, int64_t n, int32_t* active, int32_t* n_active, cudaStream_t st) {
    cudaMemsetAsync(n_active, 0, sizeof(int32_t), st);
    if (n <= 0) return;
    launch_k<false>(k_active_rows, capped_grid(n, 256, 148 * 8), 256, 0, st, seg, n, active, n_active);
    dbg_launch("k_active_rows", st);
}

void launch_fill_i32(int32_t* a, int64_t n, int32_t value, cudaStream_t st) {
    if (n <= 0) return;
    launch_k<false>(k_fill_i32, capped_grid(n, 256, 148 * 8), 256, 0, st, a, n, value);
    dbg_launch("k_fill_i32", st);
}

}  // namespace tk

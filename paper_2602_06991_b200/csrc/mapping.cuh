// mapping.cuh — launch interface of the mapping-iteration kernels (map/losses.cpp, core/ssim.cpp,
// map/optimizer.cpp, map/mapper.cpp): colour/depth L1 + D-SSIM with their gradients, the fused
// Top-K gather + masked feature L1, the fused feature backward + Adam + renormalise, selection
// statistics and the deterministic loss reduction.
#pragma once
#include "feature.cuh"
#include "tk_common.cuh"

namespace tk {

constexpr int kSsimWin = 11;

// Partial-sum slots written per block by the loss kernels (summed by k_loss_finalize).
enum LossSlot { kL1Color = 0, kL1Depth = 1, kSsimSum = 2, kFeatAbs = 3, kFeatCount = 4, kLossSlots = 5 };
constexpr int kLossBlocks = 148 * 4;  // partial-sum rows (grid of every loss kernel is capped to this)

struct ColorLossParams {
    int w, h;
    const double* color;     // rendered, H x W x 3
    const double* depth;     // rendered, H x W
    const float* gt_color;   // keyframe, H x W x 3
    const float* gt_depth;   // keyframe, H x W
    double lambda_geo, lambda1, lambda2, deadband;
    int use_ssim;            // lambda1 != 0 and the secondary term is D-SSIM
    int use_depth;           // depth_n > 0 and lambda2 != 0
    double inv_color_n, inv_depth_n, inv_count;
    double kern[kSsimWin];   // gaussian_kernel() of ssim.cpp:18-28 (host-computed)
    double* win;             // 5 x 3 x OH x OW  per window: mu_a, mu_b, d_mu, 2 d_var, d_cov
    double* grad_color;      // H x W x 3 (final, lambda_geo folded)
    double* grad_depth;      // H x W
    double* partial;         // kLossBlocks x kLossSlots
};

struct FeatLossParams {
    int width, height, k, d;
    const int32_t* index;
    const double* weight;
    const uint8_t* count;
    const float* feat;       // N x D scene features
    const float* gt;         // H x W x D keyframe features
    const uint8_t* gt_valid; // H x W: any non-zero channel in the keyframe row
    uint32_t* signs;         // H x W x ceil(D/16): 2 bits per channel (01 = +1, 10 = -1)
    double* partial;
};

struct FinalizeParams {
    const double* partial;
    int nparts;
    double replicas = 1.0;   // partial rows summed over this many D-shards (replicated slots / replicas)
    double lambda_geo, lambda_feat, lambda1, lambda2;
    int use_ssim, secondary_l1, use_depth, feature_step, d;
    double inv_color_n, inv_depth_n, inv_count;
    double* values;          // map, geo, feat
    float* feat_scale;       // lambda_feat / (feat_n * d), or 0
};

// Constants of one feature Adam step (optimizer.cpp:49-63 in fp32; bias corrections as host reciprocals).
struct AdamStepParams {
    float lr, beta1, beta2, one_m_beta1, one_m_beta2, eps, inv_bc1, inv_bc2;
};

struct FeatAdamParams {
    int64_t n;
    int k, d;
    const int32_t* seg;      // N + 1
    const uint32_t* slots;   // records sorted by (Gaussian, slot)
    const float* wnorm;
    const uint32_t* signs;
    const float* scale;      // device scalar from k_loss_finalize
    float* feat;             // N x D, updated in place
    float* m;
    float* v;
    AdamStepParams st;       // this step's constants
    LongPlan plan;           // segments longer than kLongSeg: chunk partials + ordered combine
    float* row_ss = nullptr; // D-sharded: per-Gaussian partial squared norms out, rows left unscaled
    // Feature steps applied per row (last[g] = cur for every row a step processes).  lazy != 0:
    // rows without records are skipped; their zero-gradient steps are replayed from tab[] (step
    // t's constants, 1-based) by k_feature_catchup before anything reads them.
    int32_t* last = nullptr;
    int cur = 0;
    int lazy = 0;
    const AdamStepParams* tab = nullptr;
    const int32_t* active = nullptr;    // lazy: the rows with records (any order), *n_active of them
    const int32_t* n_active = nullptr;
    float* grad = nullptr;              // lazy: [cap_active][D] sign sums of the active rows (scratch)
    int64_t cap_active = 0;
};

// active[0 .. *n_active) = the rows g with seg[g + 1] > seg[g] (unordered)
void launch_active_rows(const int32_t* seg, int64_t n, int32_t* active, int32_t* n_active, cudaStream_t st);

// Whether the feature Adam of this shape can run lazily (vector path, one register pass per row).
bool feature_adam_lazy_ok(const FeatAdamParams& p);
// Replay the skipped zero-gradient steps up to `target` of rows with last[g] < target -- every row
// (only_active = false) or the rows of p.active (true).
void launch_feature_catchup(const FeatAdamParams& p, int target, bool only_active, cudaStream_t st);
// last[0..n) = value
void launch_fill_i32(int32_t* a, int64_t n, int32_t value, cudaStream_t st);

// D-sharded renormalisation: f /= sqrt(ss[g]) when sqrt(ss[g]) > 1e-12 (ss all-reduced over shards)
void launch_feature_renorm(float* feat, const float* ss, int64_t n, int d, cudaStream_t st);

void launch_gt_valid(const float* gt, int64_t pixels, int d, uint8_t* valid, int64_t* depth_n_out,
                     const float* gt_depth, cudaStream_t st);
void launch_color_loss(const ColorLossParams& p, cudaStream_t st);
void launch_feature_loss(const FeatLossParams& p, cudaStream_t st);
void launch_loss_finalize(const FinalizeParams& p, cudaStream_t st);
void launch_topk_stats(const int32_t* index, const uint8_t* count, int64_t pixels, int k, int32_t* topk_count,
                       cudaStream_t st);
void launch_feature_adam(const FeatAdamParams& p, cudaStream_t st);

}  // namespace tk

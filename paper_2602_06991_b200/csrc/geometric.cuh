// geometric.cuh — launch interface of the geometric forward / backward kernels (fp64).
#pragma once
#include "tk_common.cuh"

namespace tk {

enum GeomMode { kGeomForward = 0, kGeomCount = 1, kGeomList = 2 };

struct GeomFwdParams {
    Frame f;
    TileEntries te;
    const int32_t* tile_offsets;  // CSR over tiles (reference tile_offsets)
    const int32_t* padded_start;  // start of each tile in the padded tile-ordered arrays
    // kGeomForward outputs (any may be null except aux)
    double* color;
    double* depth;
    double* alpha;
    int32_t* topk_index;
    double* topk_weight;
    uint8_t* topk_count;
    unsigned long long* contrib;  // n, fp64 bit patterns (max of positive doubles)
    PixelAux aux;
    // kGeomCount / kGeomList (full blend)
    int32_t* list_count;
    const int32_t* list_offsets;
    int32_t* list_src;
    double* list_w;
    unsigned long long* pair_count;  // += pixel-entry pairs blended (power >= cutoff, pixel live), or null
};

struct GeomBwdParams {
    Frame f;
    TileEntries te;
    const int32_t* tile_offsets;
    const int32_t* padded_start;
    PixelAux aux;              // from the forward
    const double* grad_color;  // P x 3
    const double* grad_depth;  // P or null
    // Deterministic flush (default): each warp writes its per-entry MidGrad partial to its own
    // slot (tile pair in emission order x warp block, so each Gaussian's slots are contiguous)
    // and flags it; k_mid_* sum every Gaussian's slots in a fixed order.  part == null: fp64
    // atomicAdd into mid (TK_GEOM_BWD_ATOMIC=1).
    double* mid;               // n x 10: mx,my,ixx,ixy,iyy,z,opacity,cr,cg,cb (atomic mode)
    double* part;              // pairs x nsub x 10 partials, or null
    uint8_t* part_flag;        // pairs x nsub: 1 = partial written this sweep (zeroed first)
    const int32_t* entry_pair; // padded entry position -> pair emission index (k_materialize)
    int nsub;                  // warp blocks per tile
};

// Fixed-order per-Gaussian sum of the backward's slot partials (backward.cpp:166-178 merges its
// per-thread partials in thread order; here: the Gaussian's tile pairs in emission order -- tile
// rows, then columns, as render.cpp:146-153 emits them -- and the warp blocks of each tile in
// block order).  Bit-deterministic run to run.
struct MidReduceParams {
    int64_t nv;                   // depth-sorted visible Gaussians
    const uint32_t* order;        // depth rank -> Gaussian id
    const int32_t* ntiles_sorted; // tile pairs per depth rank
    const int32_t* pair_off;      // first pair (emission index) per depth rank
    const double* part;           // pairs x nsub x 10
    const uint8_t* part_flag;     // pairs x nsub
    int nsub;
    double* mid;                  // nv x 10 by depth rank, written for every rank with tile pairs
    int32_t* big_list;            // nv: medium ranks from the front, huge ranks from the back
    int32_t* big_count;           // [medium, huge], zeroed beforehand
};

struct ChainParams {
    int64_t n;
    const double* mid;
    const double* mean;
    const double* log_scale;
    const double* rotation;
    const double* opacity_logit;
    double pose[7];
    double fx, fy, dilation;
    double* g_mean;
    double* g_log_scale;
    double* g_rotation;
    double* g_opacity_logit;
    double* g_color;
    double* twist;  // ceil(items / 128) x 6 block partials, or null (mapping: no pose gradient)
    double mid_scale = 1.0;  // applied to mid (1 / ranks after a D-sharded all-reduce)
    // Rank mode (the deterministic merge): mid is indexed by depth rank, written for every rank
    // with tile pairs; the chain runs over those ranks only and the outputs are zero-filled first.
    const uint32_t* order = nullptr;       // depth rank -> Gaussian id (null: mid by Gaussian id)
    const int32_t* ntiles_sorted = nullptr;
    int64_t nv = 0;
};
// number of per-block twist partials the chain writes (k_twist_final's input)
__host__ __device__ inline int64_t chain_items(const ChainParams& p) { return p.order ? p.nv : p.n; }

// In-place Adam over the five geometry groups (optimizer.hpp:25-53 layout: one m / v array per
// group, strided like the parameters).  Group order: mean, log_scale, rotation, opacity, color.
struct GeoAdamParams {
    double* mean;
    double* log_scale;
    double* rotation;
    double* opacity_logit;
    double* color;
    const double* g[5];  // gradients (k_chain outputs)
    double* m[5];
    double* v[5];
    double lr[5];
    double beta1, beta2, eps, bc1, bc2;
    double min_log_scale, max_log_scale;
    const unsigned long long* contrib;  // forward peak weights (fp64 bits), or null
    double* max_contrib;
};

// number of one-warp CTAs covering the frame's swept tiles [tile_begin, tile_end)
int geom_blocks(const Frame& f);
int geom_blocks_per_tile(int tile_size);
void launch_geom_fwd(int mode, const GeomFwdParams& p, int n_blocks, cudaStream_t st);
void launch_geom_bwd(const GeomBwdParams& p, int n_blocks, cudaStream_t st);
void launch_mid_reduce(const MidReduceParams& p, cudaStream_t st);
void launch_chain(const ChainParams& p, cudaStream_t st);
// Adam + clamps + renormalisation + peak statistic over every Gaussian (thread per Gaussian)
void launch_geo_adam(const GeoAdamParams& a, int64_t n, cudaStream_t st);
// deterministic sum of k_chain's per-block twist partials -> out[6] (device); items = chain_items()
void launch_twist_reduce(const double* twist, int64_t items, double* partial, double* out, cudaStream_t st);

}  // namespace tk

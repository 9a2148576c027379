// prepare.cuh — launch interface of the projection / depth-sort / tile-binning kernels.
#pragma once
#include "tk_common.cuh"

namespace tk {

struct ProjectParams {
    int64_t n;
    const double* mean;
    const double* log_scale;
    const double* rotation;
    const double* opacity_logit;
    double pose[7];  // qw,qx,qy,qz,tx,ty,tz
    double fx, fy, cx, cy, near_plane, far_plane, dilation;
    int tile_size, tiles_x, tiles_y;
    // outputs, indexed by Gaussian
    double *mx, *my, *ixx, *ixy, *iyy, *z, *opacity;
    int4* rect;
    int32_t* valid;
    int32_t* ntiles;
    uint64_t* key_min;  // device scalars, preset to ~0 / 0
    uint64_t* key_max;
};

struct MaterializeParams {
    int64_t n_pairs;
    const uint32_t* tile_keys;   // tile id per pair (sorted)
    const uint32_t* tile_vals;   // depth rank per pair
    const int32_t* tile_offsets; // CSR (tiles + 1)
    const int32_t* padded_start; // padded CSR start per tile
    const uint32_t* order;       // depth rank -> Gaussian id
    const double *mx, *my, *ixx, *ixy, *iyy, *z, *opacity, *color;
    TileEntries out;
    // emission index of every materialised entry (k_emit_pairs order: depth rank s's tiles at
    // pair_off[s] + local, row-major in its rectangle): entry_pair[padded position]; null = not needed
    const int4* rect;
    const int32_t* pair_off;
    int tiles_x;
    int32_t* entry_pair;
};

void launch_project(const ProjectParams& p, cudaStream_t st);
void launch_compact(const int32_t* valid, const int32_t* pos, const double* z, int64_t n, const uint64_t* key_min,
                    uint64_t* keys, uint32_t* vals, cudaStream_t st);
void launch_sorted_ntiles(const uint32_t* order, int64_t nv, const int32_t* ntiles, int32_t* ntiles_sorted,
                          cudaStream_t st);
// big: nv int32 scratch, nbig: one device int32 (ranks spanning many tiles, emitted by warps)
void launch_emit_pairs(const uint32_t* order, int64_t nv, const int4* rect, const int32_t* ntiles_sorted,
                       const int32_t* pair_off, int tiles_x, uint32_t* tkeys, uint32_t* tvals, int32_t* big,
                       int32_t* nbig, cudaStream_t st);
void launch_padded_counts(const int32_t* tile_offsets, int n_tiles, int32_t* padded, cudaStream_t st);
void launch_materialize(const MaterializeParams& p, cudaStream_t st);
void launch_export_entries(const uint32_t* order, int64_t nv, const double* mx, const double* my, const double* ixx,
                           const double* ixy, const double* iyy, const double* z, const double* opacity,
                           double* out7, int32_t* src, cudaStream_t st);

}  // namespace tk

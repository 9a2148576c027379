// prepare.cu — K1-K3: fp64 EWA projection, depth sort and tile binning (prepare_scene).
//
// Compiled with --fmad=false: every product and sum below is rounded exactly like the CPU
// restatement (oracle/src/oracle.cpp) of project_gaussian (projection.cpp:7-35) and
// prepare_scene (render.cpp:73-156), so the visible set, the depth keys, the radii and the tile
// ranges — every discrete decision of the PreparedScene — agree bit for bit.
#include "prepare.cuh"
#include "sort.cuh"

namespace tk {

namespace {

__device__ __forceinline__ void quat_to_matrix(double w, double x, double y, double z, double r[3][3]) {
    const double tx = 2.0 * x, ty = 2.0 * y, tz = 2.0 * z;
    const double twx = tx * w, twy = ty * w, twz = tz * w;
    const double txx = tx * x, txy = ty * x, txz = tz * x;
    const double tyy = ty * y, tyz = tz * y, tzz = tz * z;
    r[0][0] = 1.0 - (tyy + tzz);
    r[0][1] = txy - twz;
    r[0][2] = txz + twy;
    r[1][0] = txy + twz;
    r[1][1] = 1.0 - (txx + tzz);
    r[1][2] = tyz - twx;
    r[2][0] = txz - twy;
    r[2][1] = tyz + twx;
    r[2][2] = 1.0 - (txx + tyy);
}

// Projection of Gaussian i; writes the ProjEntry fields, radius and tile rectangle.
#ifndef TK_PROJECT_MINB
#define TK_PROJECT_MINB 4  // 64 registers, 4 resident blocks: 70 -> 49 us (3 blocks: 54 us)
#endif
__global__ void __launch_bounds__(256, TK_PROJECT_MINB) k_project(ProjectParams p) {
    pdl_prologue();
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    bool ok = false;
    uint64_t key = 0;
    if (i < p.n) {
        int32_t ntiles = 0;
        double w[3][3];
        quat_to_matrix(p.pose[0], p.pose[1], p.pose[2], p.pose[3], w);
        const double m0 = p.mean[i * 3 + 0], m1 = p.mean[i * 3 + 1], m2 = p.mean[i * 3 + 2];
        double pc[3];
#pragma unroll
        for (int r = 0; r < 3; ++r) pc[r] = ((w[r][0] * m0 + w[r][1] * m1) + w[r][2] * m2) + p.pose[4 + r];
        const double z = pc[2];
        const double ls0 = p.log_scale[i * 3 + 0], ls1 = p.log_scale[i * 3 + 1], ls2 = p.log_scale[i * 3 + 2];
        if (z > p.near_plane && z < p.far_plane) {                                    // projection.cpp:14
            const double max_extent = 3.0 * exp(fmax(fmax(ls0, ls1), ls2));          // :19
            if (!(z <= max_extent)) {                                                 // :20
                const double mx = p.fx * pc[0] / z + p.cx;                           // :23
                const double my = p.fy * pc[1] / z + p.cy;
                const double j00 = p.fx / z, j02 = -p.fx * pc[0] / (z * z);          // :25-27
                const double j11 = p.fy / z, j12 = -p.fy * pc[1] / (z * z);
                const double jm[2][3] = {{j00, 0.0, j02}, {0.0, j11, j12}};
                double a[2][3];
#pragma unroll
                for (int r = 0; r < 2; ++r)
#pragma unroll
                    for (int c = 0; c < 3; ++c) a[r][c] = (jm[r][0] * w[0][c] + jm[r][1] * w[1][c]) + jm[r][2] * w[2][c];
                // covariance (types.hpp:39-43): R(q/|q|) diag(exp(2 ls)) R^T
                const double q0 = p.rotation[i * 4 + 0], q1 = p.rotation[i * 4 + 1];
                const double q2 = p.rotation[i * 4 + 2], q3 = p.rotation[i * 4 + 3];
                const double qn = sqrt(((q0 * q0 + q1 * q1) + q2 * q2) + q3 * q3);
                double rr[3][3];
                quat_to_matrix(q0 / qn, q1 / qn, q2 / qn, q3 / qn, rr);
                const double s2[3] = {exp(2.0 * ls0), exp(2.0 * ls1), exp(2.0 * ls2)};
                double sig[3][3];
#pragma unroll
                for (int r = 0; r < 3; ++r)
#pragma unroll
                    for (int c = 0; c < 3; ++c)
                        sig[r][c] = ((rr[r][0] * s2[0]) * rr[c][0] + (rr[r][1] * s2[1]) * rr[c][1]) +
                                    (rr[r][2] * s2[2]) * rr[c][2];
                double b[2][3];
#pragma unroll
                for (int r = 0; r < 2; ++r)
#pragma unroll
                    for (int c = 0; c < 3; ++c) b[r][c] = (a[r][0] * sig[0][c] + a[r][1] * sig[1][c]) + a[r][2] * sig[2][c];
                const double c00 = ((b[0][0] * a[0][0] + b[0][1] * a[0][1]) + b[0][2] * a[0][2]) + p.dilation;
                const double c01 = (b[0][0] * a[1][0] + b[0][1] * a[1][1]) + b[0][2] * a[1][2];
                const double c11 = ((b[1][0] * a[1][0] + b[1][1] * a[1][1]) + b[1][2] * a[1][2]) + p.dilation;
                const double det = c00 * c11 - c01 * c01;                             // render.cpp:90
                if (det > 0.0 && isfinite(det)) {                                     // :91
                    const double mid = 0.5 * (c00 + c11), dif = 0.5 * (c00 - c11);    // :35-39
                    const double lmax = mid + sqrt(dif * dif + c01 * c01);
                    const double radius = sqrt(-2.0 * kLogWeightCutoff * lmax);       // :101
                    p.mx[i] = mx;
                    p.my[i] = my;
                    p.ixx[i] = c11 / det;                                             // :95-97
                    p.ixy[i] = -c01 / det;
                    p.iyy[i] = c00 / det;
                    p.z[i] = z;
                    p.opacity[i] = 1.0 / (1.0 + exp(-p.opacity_logit[i]));            // types.hpp:12
                    const double ts = static_cast<double>(p.tile_size);               // :126-132
                    const int tx0 = max(0, x86_double_to_int(floor((mx - radius) / ts)));
                    const int tx1 = min(p.tiles_x - 1, x86_double_to_int(floor((mx + radius) / ts)));
                    const int ty0 = max(0, x86_double_to_int(floor((my - radius) / ts)));
                    const int ty1 = min(p.tiles_y - 1, x86_double_to_int(floor((my + radius) / ts)));
                    if (tx0 <= tx1 && ty0 <= ty1) {
                        const int64_t cnt = static_cast<int64_t>(tx1 - tx0 + 1) * (ty1 - ty0 + 1);
                        ntiles = cnt > INT32_MAX ? INT32_MAX : static_cast<int32_t>(cnt);
                    }
                    p.rect[i] = make_int4(tx0, tx1, ty0, ty1);
                    ok = true;
                    key = static_cast<uint64_t>(__double_as_longlong(z));
                }
            }
        }
        p.valid[i] = ok ? 1 : 0;
        p.ntiles[i] = ntiles;
    }
    // key range of the visible set -> number of radix passes (one block-level reduction).
    __shared__ unsigned long long smin, smax;
    if (threadIdx.x == 0) {
        smin = ~0ull;
        smax = 0ull;
    }
    __syncthreads();
    {
        unsigned long long lo = ok ? key : ~0ull, hi = ok ? key : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long a = __shfl_xor_sync(0xffffffffu, lo, o);
            const unsigned long long b = __shfl_xor_sync(0xffffffffu, hi, o);
            lo = a < lo ? a : lo;
            hi = b > hi ? b : hi;
        }
        if ((threadIdx.x & 31) == 0 && hi >= lo) {
            atomicMin(&smin, lo);
            atomicMax(&smax, hi);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0 && smax >= smin) {
        atomicMin(reinterpret_cast<unsigned long long*>(p.key_min), smin);
        atomicMax(reinterpret_cast<unsigned long long*>(p.key_max), smax);
    }
}

// Sort keys: fp64 bit pattern of z minus the smallest visible one (positive doubles order like
// their bits, so this is monotone and packs the key range into the low bits).
__global__ void k_compact(const int32_t* __restrict__ valid, const int32_t* __restrict__ pos,
                          const double* __restrict__ z, int64_t n, const uint64_t* __restrict__ key_min,
                          uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    pdl_prologue();
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n || !valid[i]) return;
    const int32_t q = pos[i];
    keys[q] = static_cast<uint64_t>(__double_as_longlong(z[i])) - *key_min;
    vals[q] = static_cast<uint32_t>(i);
}

__global__ void k_sorted_ntiles(const uint32_t* __restrict__ order, int64_t nv, const int32_t* __restrict__ ntiles,
                                int32_t* __restrict__ ntiles_sorted) {
    pdl_prologue();
    const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (s >= nv) return;
    ntiles_sorted[s] = ntiles[order[s]];
}

// One thread per sorted entry: emit (tile, depth rank) pairs in rank order (render.cpp:146-153).
// An entry spanning more than kEmitThread tiles (a near-camera Gaussian can cover the whole
// image) is queued for k_emit_big, which writes its rectangle with a whole warp; the pair
// positions depend only on pair_off and the tile's place in the rectangle, not on who writes.
constexpr int kEmitThread = 64;

__device__ __forceinline__ void emit_pair(const int4& r, int32_t o0, int local, uint32_t s, int tiles_x,
                                          uint32_t* tkeys, uint32_t* tvals) {
    const int w = r.y - r.x + 1;
    const int ty = r.z + local / w, tx = r.x + local % w;
    tkeys[o0 + local] = static_cast<uint32_t>(ty * tiles_x + tx);
    tvals[o0 + local] = s;
}

__global__ void k_emit_pairs(const uint32_t* __restrict__ order, int64_t nv, const int4* __restrict__ rect,
                             const int32_t* __restrict__ ntiles_sorted, const int32_t* __restrict__ pair_off,
                             int tiles_x, uint32_t* __restrict__ tkeys, uint32_t* __restrict__ tvals,
                             int32_t* __restrict__ big, int32_t* __restrict__ nbig) {
    pdl_prologue();
    const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (s >= nv) return;
    const int nt = ntiles_sorted[s];
    if (nt == 0) return;
    if (nt > kEmitThread) {
        big[atomicAdd(nbig, 1)] = static_cast<int32_t>(s);
        return;
    }
    const int4 r = rect[order[s]];
    int32_t o = pair_off[s];
    for (int ty = r.z; ty <= r.w; ++ty)
        for (int tx = r.x; tx <= r.y; ++tx) {
            tkeys[o] = static_cast<uint32_t>(ty * tiles_x + tx);
            tvals[o] = static_cast<uint32_t>(s);
            ++o;
        }
}

__global__ void __launch_bounds__(256) k_emit_big(const uint32_t* __restrict__ order, const int4* __restrict__ rect,
                                                  const int32_t* __restrict__ ntiles_sorted,
                                                  const int32_t* __restrict__ pair_off, int tiles_x,
                                                  uint32_t* __restrict__ tkeys, uint32_t* __restrict__ tvals,
                                                  const int32_t* __restrict__ big, const int32_t* __restrict__ nbig) {
    pdl_prologue();
    const int lane = threadIdx.x & 31;
    const int nb = *nbig;
    for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nb; w += (gridDim.x * blockDim.x) >> 5) {
        const uint32_t s = static_cast<uint32_t>(big[w]);
        const int4 r = rect[order[s]];
        const int nt = ntiles_sorted[s];
        const int32_t o0 = pair_off[s];
        for (int local = lane; local < nt; local += 32) emit_pair(r, o0, local, s, tiles_x, tkeys, tvals);
    }
}

__global__ void k_padded_counts(const int32_t* __restrict__ tile_offsets, int n_tiles, int32_t* __restrict__ padded) {
    pdl_prologue();
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t > n_tiles) return;
    padded[t] = t < n_tiles ? static_cast<int32_t>(align_up(tile_offsets[t + 1] - tile_offsets[t], kEntryAlign)) : 0;
}

// Tile-ordered SoA copy of the entries (plus colours) into the padded layout.
__global__ void k_materialize(MaterializeParams p) {
    pdl_prologue();
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= p.n_pairs) return;
    const uint32_t t = p.tile_keys[j];
    const uint32_t s = p.tile_vals[j];
    const int64_t dst = static_cast<int64_t>(p.padded_start[t]) + (j - p.tile_offsets[t]);
    const uint32_t i = p.order[s];
    EntryChunk& ch = p.out.chunks[dst / kChunk];
    const int l = static_cast<int>(dst % kChunk);
    ch.f[0][l] = p.mx[i];
    ch.f[1][l] = p.my[i];
    ch.f[2][l] = p.ixx[i];
    ch.f[3][l] = p.ixy[i];
    ch.f[4][l] = p.iyy[i];
    ch.f[5][l] = p.z[i];
    ch.f[6][l] = p.opacity[i];
    ch.f[7][l] = p.color[i * 3 + 0];
    ch.f[8][l] = p.color[i * 3 + 1];
    ch.f[9][l] = p.color[i * 3 + 2];
    ch.src[l] = static_cast<int32_t>(i);
    if (p.entry_pair) {
        const int4 r = p.rect[i];
        const int tx = static_cast<int>(t % static_cast<uint32_t>(p.tiles_x)), ty = static_cast<int>(t / static_cast<uint32_t>(p.tiles_x));
        p.entry_pair[dst] = p.pair_off[s] + (ty - r.z) * (r.y - r.x + 1) + (tx - r.x);
    }
    // Bounding box of {d : -0.5 d^T A d >= cutoff}, A = (ixx, ixy; ixy, iyy): |d_x| <= sqrt(R Sxx)
    // with R = -2 cutoff and S = A^-1.  Inflated (1e-6 relative + 1e-3 px) so that rounding can
    // never cull an entry that contributes to a pixel of the block (culling only skips work).
    const double ixx = p.ixx[i], ixy = p.ixy[i], iyy = p.iyy[i];
    const double det = ixx * iyy - ixy * ixy;
    const double r2 = -2.0 * kLogWeightCutoff;
    const double hx = sqrt(r2 * (iyy / det)), hy = sqrt(r2 * (ixx / det));
    ch.hx[l] = det > 0.0 ? static_cast<float>(hx * (1.0 + 1e-6) + 1e-3) : 3.0e38f;
    ch.hy[l] = det > 0.0 ? static_cast<float>(hy * (1.0 + 1e-6) + 1e-3) : 3.0e38f;
}

__global__ void k_export_entries(const uint32_t* __restrict__ order, int64_t nv, const double* __restrict__ mx,
                                 const double* __restrict__ my, const double* __restrict__ ixx,
                                 const double* __restrict__ ixy, const double* __restrict__ iyy,
                                 const double* __restrict__ z, const double* __restrict__ opacity,
                                 double* __restrict__ out7, int32_t* __restrict__ src) {
    pdl_prologue();
    const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (s >= nv) return;
    const uint32_t i = order[s];
    double* o = out7 + s * 7;
    o[0] = mx[i];
    o[1] = my[i];
    o[2] = ixx[i];
    o[3] = ixy[i];
    o[4] = iyy[i];
    o[5] = z[i];
    o[6] = opacity[i];
    src[s] = static_cast<int32_t>(i);
}

inline unsigned blocks_for(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

}  // namespace

void launch_project(const ProjectParams& p, cudaStream_t st) {
    if (p.n > 0) launch_k(k_project, blocks_for(p.n, 256), 256, 0, st, p);
    dbg_launch("k_project", st);
}

void launch_compact(const int32_t* valid, const int32_t* pos, const double* z, int64_t n, const uint64_t* key_min,
                    uint64_t* keys, uint32_t* vals, cudaStream_t st) {
    if (n > 0) launch_k(k_compact, blocks_for(n, 256), 256, 0, st, valid, pos, z, n, key_min, keys, vals);
    dbg_launch("k_compact", st);
}

void launch_sorted_ntiles(const uint32_t* order, int64_t nv, const int32_t* ntiles, int32_t* ntiles_sorted,
                          cudaStream_t st) {
    if (nv > 0) launch_k(k_sorted_ntiles, blocks_for(nv, 256), 256, 0, st, order, nv, ntiles, ntiles_sorted);
    dbg_launch("k_sorted_ntiles", st);
}

void launch_emit_pairs(const uint32_t* order, int64_t nv, const int4* rect, const int32_t* ntiles_sorted,
                       const int32_t* pair_off, int tiles_x, uint32_t* tkeys, uint32_t* tvals, int32_t* big,
                       int32_t* nbig, cudaStream_t st) {
    if (nv > 0) {
        cudaMemsetAsync(nbig, 0, sizeof(int32_t), st);
        launch_k(k_emit_pairs, blocks_for(nv, 128), 128, 0, st, order, nv, rect, ntiles_sorted, pair_off, tiles_x, tkeys,
                                                          tvals, big, nbig);
        dbg_launch("k_emit_pairs", st);
        launch_k(k_emit_big, 148 * 2, 256, 0, st, order, rect, ntiles_sorted, pair_off, tiles_x, tkeys, tvals, big, nbig);
        dbg_launch("k_emit_big", st);
    }
}

void launch_padded_counts(const int32_t* tile_offsets, int n_tiles, int32_t* padded, cudaStream_t st) {
    launch_k(k_padded_counts, blocks_for(n_tiles + 1, 256), 256, 0, st, tile_offsets, n_tiles, padded);
    dbg_launch("k_padded_counts", st);
}

void launch_materialize(const MaterializeParams& p, cudaStream_t st) {
    if (p.n_pairs > 0) launch_k(k_materialize, blocks_for(p.n_pairs, 256), 256, 0, st, p);
    dbg_launch("k_materialize", st);
}

void launch_export_entries(const uint32_t* order, int64_t nv, const double* mx, const double* my, const double* ixx,
                           const double* ixy, const double* iyy, const double* z, const double* opacity,
                           double* out7, int32_t* src, cudaStream_t st) {
    if (nv > 0) {
        launch_k(k_export_entries, blocks_for(nv, 256), 256, 0, st, order, nv, mx, my, ixx, ixy, iyy, z, opacity, out7,
                                                              src);
        dbg_launch("k_export_entries", st);
    }
}

}  // namespace tk

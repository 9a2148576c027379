/*
 * tk_render.h — C ABI of the B200-native Top-K feature-render path (libtkrender.so).
 *
 * Drop-in boundary for the reference renderer API (proj/include/fslam/raster/render.hpp,
 * backward.hpp).  Plain pointers and sizes only; every call is enqueued on the context's CUDA
 * stream and returns a status.  On error the status is non-zero and tk_last_error() holds the
 * message; the C++ mirror (include/tk/fslam_raster.hpp) rethrows it as std::runtime_error
 * with the reference's message text.
 *
 * Entry point                      replaces (reference, /root/reference/proj/...)
 * ------------------------------   -----------------------------------------------------------
 * tk_scene_upload                  SceneMap / Gaussian3D buffers (map/scene_map.hpp:16-27,
 *                                  core/types.hpp:25-44) -> device-resident SoA mirror
 * tk_prepare_scene                 raster_detail::prepare_scene   (raster/render.hpp:99-100)
 * tk_prepared_export               raster_detail::PreparedScene    (raster/render.hpp:84-92)
 * tk_render_geometric              render_geometric               (raster/render.hpp:60-61)
 * tk_render_feature                render_feature                 (raster/render.hpp:66)
 * tk_render_feature_full_blend     render_feature_full_blend      (raster/render.hpp:70-71)
 * tk_backward_feature              backward_feature               (raster/backward.hpp:33-34)
 * tk_backward_geometric            backward_geometric             (raster/backward.hpp:27-29)
 * tk_comm_* / tk_allgather_feature multi-GPU D-sharding (no reference counterpart)
 * tk_keyframe_set                  SceneMap::keyframes entry (map/scene_map.hpp, Keyframe)
 * tk_optimizer_reset               OptimizerState (map/optimizer.hpp:25-53), zeroed
 * tk_optimize_step                 optimize_step without pruning (map/mapper.hpp:72-73,
 *                                  mapper.cpp:162-255): compute_losses (losses.hpp:42-43),
 *                                  adam_step (optimizer.hpp:58-59), update_contribution_stats
 * tk_scene_download                SceneMap parameters + Gaussian3D statistics back to the host
 * tk_insert_gaussians              insert_gaussians (map/mapper.hpp:41-43, mapper.cpp:19-60)
 * tk_prune_map                     prune_map + OptimizerState::compact (mapper.hpp:53-54,
 *                                  mapper.cpp:80-160, optimizer.cpp:9-47)
 * tk_checkpoint_save / _load       save_checkpoint / load_checkpoint, SPLF v1 (map/checkpoint.hpp:9-14)
 * tk_segment_by_query              segment_by_query (eval/metrics.hpp, metrics.cpp:66-94)
 *
 * Memory spaces: every buffer argument is tagged TK_HOST or TK_DEVICE.  Host buffers are
 * copied in/out inside the call (pinned memory from tk_host_alloc is fastest); device buffers
 * are used in place.  Device results that the caller did not ask to receive stay resident in
 * the context and can be read with tk_device_view().
 */
#pragma once
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TK_ABI_VERSION 1

typedef enum {
    TK_OK = 0,
    TK_ERR_STALE_INDEX = 1, /* render.cpp:307-310, backward.cpp:279-282 */
    TK_ERR_BAD_ARG = 2,     /* shape / argument mismatch */
    TK_ERR_CUDA = 3,
    TK_ERR_NCCL = 4,
    TK_ERR_OOM = 5,
    TK_ERR_STATE = 6 /* e.g. no scene uploaded, no records rendered */
} tk_status;

/* TK_HOST_ASYNC: pinned host memory copied on the context's own copy streams (host->device and
 * device->host run concurrently on the two copy engines); the call returns without waiting, the
 * host buffer must stay untouched until tk_synchronize().  Asynchronous scene uploads are
 * double-buffered (the next scene streams in while the current frame still computes on the
 * previous one; device views from tk_device_view_get refer to the scene current at the call), and
 * asynchronous upstream-gradient uploads wait only for the previous call that read their buffer. */
enum { TK_HOST = 0, TK_DEVICE = 1, TK_HOST_ASYNC = 2 };

typedef struct tk_ctx tk_ctx;

typedef struct { /* CameraIntrinsics, core/types.hpp:15-21 */
    double fx, fy, cx, cy;
    int32_t width, height;
    double near_plane, far_plane;
} tk_camera;

typedef struct { /* Pose (world-to-camera), core/pose.hpp:11-19; quaternion used unnormalised */
    double qw, qx, qy, qz;
    double tx, ty, tz;
} tk_pose;

typedef struct { /* RenderSettings, raster/render.hpp:14-21 */
    int32_t top_k;
    int32_t tile_size;
    double transmittance_floor;
    double background[3];
    double cov2d_dilation;
    double alpha_clamp;
} tk_settings;

typedef struct { /* Gaussian SoA view; rotation is (w,x,y,z) */
    int64_t n;
    int32_t d;              /* feature channels held by this context (a shard under tk_comm) */
    const double* mean;     /* n x 3 */
    const double* log_scale;/* n x 3 */
    const double* rotation; /* n x 4 */
    const double* opacity_logit; /* n */
    const double* color;    /* n x 3 */
    const float* feature;   /* n x d, fp32; NULL keeps the resident features (n, d unchanged) */
    uint64_t generation;    /* SceneMap::generation (scene_map.hpp:16) */
} tk_scene_view;

typedef struct { /* TopKGrid, raster/render.hpp:27-44 (slot = (y*W+x)*k + j) */
    int32_t width, height, k;
    const int32_t* index;  /* W*H*k, -1 unused */
    const double* weight;  /* W*H*k */
    const uint8_t* count;  /* W*H */
    int32_t mem;           /* TK_HOST / TK_DEVICE */
} tk_topk_view;

typedef struct { /* RenderOutput, raster/render.hpp:46-55; NULL pointers are skipped */
    int32_t mem;
    double* color;         /* H*W*3 */
    double* depth;         /* H*W */
    double* alpha;         /* H*W, sum of weights (render.cpp:222) */
    int32_t* topk_index;   /* H*W*k */
    double* topk_weight;   /* H*W*k */
    uint8_t* topk_count;   /* H*W */
    double* contributions; /* n */
    uint64_t generation;   /* out: stamped (render.cpp:167-168) */
    int64_t map_size;      /* out */
} tk_geom_out;

typedef struct { /* GeomGrads, raster/backward.hpp:15-22; NULL pointers are skipped */
    int32_t mem;
    double* mean;          /* n x 3 */
    double* log_scale;     /* n x 3 */
    double* rotation;      /* n x 4 (w,x,y,z) */
    double* opacity_logit; /* n */
    double* color;         /* n x 3 */
    double pose_twist[6];  /* out: [nu, omega]; with TK_HOST_ASYNC or TK_DEVICE written at
                            * tk_synchronize (the struct must stay alive until then), so a
                            * device-resident frame never waits on the host */
} tk_geom_grads;

typedef struct { /* resident device buffers of the last calls (read-only views) */
    const double* color;
    const double* depth;
    const double* alpha;
    const int32_t* topk_index;
    const double* topk_weight;
    const uint8_t* topk_count;
    const double* contributions;
    const float* feature_out;   /* render_feature result, H*W*d */
    const float* feature_grad;  /* backward_feature result, n*d */
    float* grad_feature_in;     /* staging buffer for dL/dF, H*W*d (writable) */
    const double* mean;         /* scene mirror */
    float* feature;             /* scene features, n*d (writable: in-place optimiser updates) */
    int64_t n;
    int32_t d, width, height, k;
} tk_device_view;

void tk_default_settings(tk_settings* s);
const char* tk_last_error(void);
int32_t tk_abi_version(void);

tk_status tk_create(int32_t device, tk_ctx** out);
tk_status tk_destroy(tk_ctx* ctx);
tk_status tk_synchronize(tk_ctx* ctx);
/* The context runs the feature calls and the geometry backward on two side streams so they
 * overlap, and TK_HOST_ASYNC copies on two copy streams; tk_join orders the main stream
 * (tk_get_stream) after all of them, device-side. */
tk_status tk_join(tk_ctx* ctx);
void* tk_get_stream(tk_ctx* ctx); /* cudaStream_t of the main stream */

tk_status tk_host_alloc(size_t bytes, void** out); /* pinned host memory */
tk_status tk_host_free(void* p);

tk_status tk_scene_upload(tk_ctx* ctx, const tk_scene_view* scene, int32_t mem);
/* Replace the resident features only (n, d must match the resident geometry); the geometry, the
 * prepared scene and the forward records stay valid.  For drop-in callers whose map changed only
 * in its features (mapper.cpp:239-252, the feature Adam step). */
tk_status tk_scene_upload_features(tk_ctx* ctx, int64_t n, int32_t d, const float* feature, int32_t mem);
tk_status tk_device_view_get(tk_ctx* ctx, tk_device_view* out);

tk_status tk_prepare_scene(tk_ctx* ctx, const tk_pose* pose, const tk_camera* cam,
                           const tk_settings* s, int64_t* n_entries, int64_t* n_tile_entries,
                           int32_t* tiles_x, int32_t* tiles_y);
/* host outputs: entries7 = n_entries x {mx,my,ixx,ixy,iyy,z,opacity}, src, tile_offsets
 * (tiles+1), tile_entries (n_tile_entries) — the PreparedScene of the last prepare. */
tk_status tk_prepared_export(tk_ctx* ctx, double* entries7, int32_t* src, int32_t* tile_offsets,
                             int32_t* tile_entries);

tk_status tk_render_geometric(tk_ctx* ctx, const tk_pose* pose, const tk_camera* cam,
                              const tk_settings* s, tk_geom_out* out);
/* topk == NULL: the records of the last tk_render_geometric on this context. */
tk_status tk_render_feature(tk_ctx* ctx, const tk_topk_view* topk, float* out, int32_t out_mem);
tk_status tk_render_feature_full_blend(tk_ctx* ctx, const tk_pose* pose, const tk_camera* cam,
                                       const tk_settings* s, float* out, int32_t out_mem);
/* grad_feature: H*W*d fp32 (NULL + TK_DEVICE: the context's grad_feature_in buffer). out: n*d */
tk_status tk_backward_feature(tk_ctx* ctx, const tk_topk_view* topk, const float* grad_feature,
                              int32_t grad_mem, float* out, int32_t out_mem);
/* grad_color H*W*3, grad_depth H*W (may be NULL = empty image, backward.cpp:104) */
tk_status tk_backward_geometric(tk_ctx* ctx, const tk_pose* pose, const tk_camera* cam,
                                const tk_settings* s, const double* grad_color,
                                const double* grad_depth, int32_t grad_mem, tk_geom_grads* out);

/* Multi-GPU feature-dimension sharding (one process per GPU, NCCL over NVLink). */
tk_status tk_comm_unique_id(uint8_t id[128]);
tk_status tk_comm_init(tk_ctx* ctx, const uint8_t id[128], int32_t nranks, int32_t rank,
                       int32_t d_total);
/* All-gather of every rank's [H*W][d_shard] slice of the last render_feature into the full
 * H*W*d_total HWC map (channel-interleaved), on every rank. */
tk_status tk_allgather_feature(tk_ctx* ctx, float* out, int32_t out_mem);
tk_status tk_allreduce_sum_f64(tk_ctx* ctx, double* values, int32_t count); /* host values */
/* Fused render_feature + all-gather over peer memory (NVLink P2P stores, no NCCL data path):
 * each rank gathers its d_shard channels and stores every output row slice straight into every
 * rank's full [H*W][d_total] buffer at channel offset rank * d_shard, then (under tk_comm) a
 * stream-ordered NCCL all-reduce of one word acts as the rank barrier, after which the calling
 * rank's buffer holds the full HWC map -- the tk_allgather_feature result without the gather
 * buffer or the interleave pass.  Peer buffers come from tk_comm_p2p_setup (collective: each rank
 * allocates n_pixels * d_total floats and the CUDA IPC handles are exchanged over NCCL; call again,
 * on every rank, for a larger frame) or, for ranks driven from one process, from
 * tk_comm_set_peers (every rank's device buffer in rank order; the caller orders the ranks'
 * streams: there is no barrier).  d_shard % 4 == 0, nranks <= 8.  out: NULL or a copy of the
 * calling rank's full map (TK_HOST / TK_DEVICE / TK_HOST_ASYNC); tk_comm_gathered_buffer returns
 * the buffer itself. */
tk_status tk_comm_p2p_setup(tk_ctx* ctx, int64_t n_pixels);
tk_status tk_comm_set_peers(tk_ctx* ctx, int32_t rank, int32_t nranks, int32_t d_total,
                            float* const* buffers, int64_t n_pixels);
tk_status tk_render_feature_gathered(tk_ctx* ctx, const tk_topk_view* topk, float* out,
                                     int32_t out_mem);
tk_status tk_comm_gathered_buffer(tk_ctx* ctx, float** buffer);

/* Geometry split across ranks (the Amdahl term of the D-sharded frame): the geometric forward and
 * backward sweeps cover only band `band` of `nbands` bands of whole tile rows (rows_b =
 * ceil(tiles_y / nbands)).  Under tk_comm with nranks == nbands and band == rank, tk_render_geometric
 * all-gathers the per-pixel records, colour, depth and alpha of every band (NCCL, equal band-sized
 * chunks) and max-reduces the peak contributions, and tk_backward_geometric sum-reduces the merged
 * per-Gaussian projected gradients (N_vis x 10 fp64) before the chain rule, so every rank ends with
 * the whole frame's outputs; the sum over bands is fixed for a fixed nbands (NCCL reduction order),
 * not bit-identical to the unsplit sweep.  Without tk_comm the context sweeps its band only (band
 * outputs valid, the rest stale): single-process simulation of the split.  nbands = 1 restores the
 * whole-image sweeps.  Not supported by tk_optimize_step. */
tk_status tk_geometry_band(tk_ctx* ctx, int32_t band, int32_t nbands);

/* ---- one mapping iteration on the device (map/mapper.cpp:162-255) ---- */
typedef struct { /* MapperConfig knobs of one iteration; same layout as the oracle's orc_mapper_config */
    double lambda_geo, lambda_feat, lambda1, lambda2; /* LossWeights, losses.hpp:9-21 */
    int32_t color_secondary;        /* 0 = D-SSIM, 1 = duplicated L1 (ColorSecondaryTerm) */
    int32_t feature_update_period;  /* Schedule, mapper.hpp:16 */
    double l1_deadband;
    double lr_mean, lr_log_scale, lr_rotation, lr_opacity, lr_color, lr_feature; /* optimizer.hpp:15-22 */
    double beta1, beta2, eps;       /* AdamParams, optimizer.hpp:9-13 */
    double min_log_scale, max_log_scale; /* mapper.hpp:31-32 */
} tk_mapper_config;

typedef struct { /* Frame (ground truth of one keyframe): fp32 images, HWC */
    int32_t width, height, d;
    const float* color;   /* H*W*3 */
    const float* depth;   /* H*W; <= 0 marks invalid depth */
    const float* feature; /* H*W*d, or NULL (then d must be 0) */
    int32_t mem;
} tk_frame_view;

typedef struct { /* SceneMap parameters + statistics out; NULL pointers are skipped */
    int32_t mem;
    double* mean;             /* n x 3 */
    double* log_scale;        /* n x 3 */
    double* rotation;         /* n x 4 */
    double* opacity_logit;    /* n */
    double* color;            /* n x 3 */
    float* feature;           /* n x d */
    int32_t* topk_count;      /* n, Gaussian3D::topk_count */
    double* max_contribution; /* n, Gaussian3D::max_contribution */
} tk_scene_out;

void tk_default_mapper_config(tk_mapper_config* cfg); /* the reference's defaults */
/* Store keyframe `slot` (0-based; slots grow on demand) device-resident: pose + frame. */
tk_status tk_keyframe_set(tk_ctx* ctx, int32_t slot, const tk_pose* pose, const tk_frame_view* frame);
/* Zero the Adam state of every group for the resident scene (n, d) and, when reset_stats,
 * the selection statistics (topk_count, max_contribution). */
tk_status tk_optimizer_reset(tk_ctx* ctx, int32_t reset_stats);
/* Under tk_comm (D-sharded: every rank holds d = d_total / nranks feature channels and the same
 * geometry) the step is the D-sharded mapping iteration: keyframe feature masks, the loss
 * partials, the geometry gradients and the feature row norms are all-reduced with NCCL, so the
 * geometry replicas stay bit-identical and each rank updates its channel slice.
 * One optimisation step on keyframe `slot` (the caller samples it; mapper.cpp:167-168):
 * render, losses, backward, Adam per group (features on iteration % feature_update_period
 * == 0), renormalisation, statistics.  values_out (host, may be NULL = stay on the device,
 * no synchronisation) receives {map, geo, feat} (LossValues, losses.hpp:23-27). */
tk_status tk_optimize_step(tk_ctx* ctx, const tk_mapper_config* cfg, const tk_camera* cam,
                           const tk_settings* s, int32_t slot, int64_t iteration, double* values_out,
                           int32_t* feature_step_out);
/* The feature Adam of tk_optimize_step is lazy (TK_LAZY_ADAM=0 for eager): a feature step updates
 * only the rows the frame's records reach; every other row's zero-gradient steps are replayed,
 * bit-identically to the eager step, right before anything reads feature rows (the feature
 * renders, tk_scene_download, structural edits, checkpoints, tk_device_view_get) or the next step
 * that reaches them.  tk_optimizer_flush brings every row up to date now (asynchronous). */
tk_status tk_optimizer_flush(tk_ctx* ctx);
/* Loss values of the last tk_optimize_step (synchronises). */
tk_status tk_loss_values(tk_ctx* ctx, double values[3]);
tk_status tk_scene_download(tk_ctx* ctx, const tk_scene_out* out);

/* ---- structural edits of the resident map (generation bumps, optimiser state in lockstep) ---- */
typedef struct { /* SourcePoint batch (track/gicp.hpp:18-25), SoA */
    int64_t n;
    int32_t d;               /* feature channels of the source points (0: none) */
    const double* position;  /* n x 3, camera frame */
    const double* color;     /* n x 3 */
    const float* feature;    /* n x d, or NULL */
    const double* spacing;   /* n: local sample spacing (scene units) */
    const double* distance;  /* n: correspondence distance to the map (inf: none) */
    int32_t mem;
} tk_source_view;

tk_status tk_scene_info(tk_ctx* ctx, int64_t* n, int32_t* d, uint64_t* generation);
/* Inserts one Gaussian per source point with distance >= tau (mapper.cpp:29-52), extends the
 * optimiser state and statistics with zeros and bumps the generation when any is inserted. */
tk_status tk_insert_gaussians(tk_ctx* ctx, const tk_source_view* src, double tau_insert,
                              const tk_pose* world_to_camera, int32_t* inserted);
/* Two-stage prune on the context's statistics: the draw runs on the host exactly as
 * mapper.cpp:85-139 (std::mt19937_64(seed)); the map, features and every optimiser group are
 * compacted in lockstep on the device; statistics restart at zero.  removed_out (host, capacity
 * n, may be NULL) receives the removed indices in ascending order. */
tk_status tk_prune_map(tk_ctx* ctx, double keep_ratio, uint64_t seed, int32_t topk_count_threshold,
                       int32_t* removed_out, int64_t* n_removed);
/* The candidate draw of prune_map alone (mapper.cpp:80-139), on host statistics; no context, no
 * GPU.  Same removed indices as the reference's sequential scan, bit for bit, in O(C log C)
 * (Fenwick pool with an exact rounding-bounded fallback).  removed_out: capacity n. */
tk_status tk_prune_draw(const int32_t* topk_count, const double* max_contribution, int64_t n, double keep_ratio,
                        uint64_t seed, int32_t topk_count_threshold, int32_t* removed_out, int64_t* n_removed);

/* FEAT feature frames (synth/dataset.cpp:48-76: "FEAT", uint32 h, w, d, then h*w*d fp32 HWC):
 * load replaces keyframe `slot`'s feature image (same h x w as the keyframe; its row-validity mask
 * is recomputed) straight from the file; save writes it.  Errors carry the reference's messages
 * ("dataset: cannot open <path>", "dataset: bad magic in <path>", "dataset: truncated header in
 * <path>", "dataset: truncated data in <path>", "dataset: write failed for <path>"). */
tk_status tk_keyframe_load_features(tk_ctx* ctx, int32_t slot, const char* path);
tk_status tk_keyframe_save_features(tk_ctx* ctx, int32_t slot, const char* path);

/* SPLF v1 checkpoint (checkpoint.cpp:39-98): little-endian "SPLF", u32 version, u32 D, u64 N, then
 * per Gaussian f32 mean[3], log_scale[3], quat w,x,y,z, opacity_logit, color[3], feature[D].
 * Packed / unpacked on the device; load replaces the resident map (generation 0, optimiser state
 * and statistics invalidated).  Errors carry the reference's messages. */
tk_status tk_checkpoint_save(tk_ctx* ctx, const char* path);
tk_status tk_checkpoint_load(tk_ctx* ctx, const char* path);

/* segment_by_query (metrics.cpp:66-94): per pixel the argmax over classes of embedding . F
 * (first maximum wins; squared norm < 1e-12 -> 255).  feature: n_pixels x d fp32 (NULL: the last
 * tk_render_feature result, d and n_pixels then come from the context); embeddings: host,
 * classes x d fp64 row-major (classes x d_total for the context's sharded F).  fp64 dots in
 * channel order (bit-identical to the reference on the same F).  Under tk_comm with nranks > 1
 * each rank scores its channel slice and the partial dots are all-reduced (sum) with NCCL. */
tk_status tk_segment_by_query(tk_ctx* ctx, const float* feature, int64_t n_pixels, int32_t d,
                              int32_t feature_mem, const double* embeddings, int32_t classes,
                              uint8_t* labels, int32_t labels_mem);

/* Drop the cached PreparedScene / forward state: the next call re-projects, re-sorts and
 * re-bins (the reference recomputes prepare_scene in every call, render.cpp:295). */
tk_status tk_invalidate(tk_ctx* ctx);

/* Pixel-entry pairs the geometric forward blended (power >= cutoff, pixel not saturated) since
 * the last reset -- the work unit of the fp64-bound sweeps (synchronises). */
tk_status tk_pair_count(tk_ctx* ctx, int64_t* pairs, int32_t reset);

/* Measured fp64 FMA instructions per second of the context's device (a ~30 ms probe): the
 * denominator of the fp64 roofline of the geometric sweeps. */
tk_status tk_fp64_rate(tk_ctx* ctx, double* fma_per_s);

/* Profiling: number of kernels the library has launched from the calling host thread (every
 * launch site counts itself; take differences around a region to count that region's kernels). */
int64_t tk_kernel_launches(tk_ctx* ctx);

/* Per-phase device time (CUDA events on the context stream).  Phases: */
enum {
    TK_PHASE_PREPARE = 0,      /* projection + depth sort + tile binning + materialise */
    TK_PHASE_GEOM_FWD = 1,     /* geometric pass (alpha blend + Top-K) */
    TK_PHASE_GATHER = 2,       /* Top-K feature gather */
    TK_PHASE_FBWD_INDEX = 3,   /* feature backward: slot keys + radix sort + segments */
    TK_PHASE_FBWD = 4,         /* feature backward: segmented reduction kernel */
    TK_PHASE_GEOM_BWD = 5,     /* geometric backward sweep */
    TK_PHASE_CHAIN = 6,        /* per-Gaussian chain rule + twist reduction */
    TK_PHASE_FULL_BLEND = 7,   /* full-blend feature pass */
    TK_PHASE_ALLGATHER = 8,    /* NCCL all-gather + interleave */
    TK_PHASE_COPY = 9,         /* host <-> device copies made inside calls */
    TK_PHASE_LOSS = 10,        /* compute_losses: colour/depth L1, D-SSIM, fused feature L1 */
    TK_PHASE_ADAM = 11,        /* chain rule + geometry Adam, feature backward + Adam */
    TK_NUM_PHASES = 12
};
tk_status tk_profile_enable(tk_ctx* ctx, int32_t on);
/* ms[TK_NUM_PHASES], counts[TK_NUM_PHASES] accumulated since the last reset (synchronises). */
tk_status tk_profile_read(tk_ctx* ctx, double* ms, int64_t* counts, int32_t reset);

#ifdef __cplusplus
}
#endif

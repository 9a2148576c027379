"""Python mirror of the reference renderer API over the C ABI (include/tk_render.h).

Same function names, argument meaning and error behaviour as
proj/include/fslam/raster/render.hpp and backward.hpp: renders are pure functions of
(map, pose, camera, settings); a stale Top-K record raises RuntimeError with the reference's
message.  Everything executes in libtkrender.so on the GPU — there is no CPU fallback.

A :class:`Renderer` owns one device context; the module-level functions use a lazily created
default renderer on device 0.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .types import (CameraIntrinsics, Frame, GeomGrads, LossValues, MapperConfig, Pose, PreparedScene,
                    RenderOutput, RenderSettings, SceneMap, TopKGrid, K_MAX_TOP_K)


def _c(a: np.ndarray | None, dtype) -> np.ndarray | None:
    if a is None:
        return None
    return np.ascontiguousarray(a, dtype=dtype)


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data


def to_pose(p: Pose) -> N.tk_pose:
    q, t = p.rotation, p.translation
    return N.tk_pose(q[0], q[1], q[2], q[3], t[0], t[1], t[2])


def to_camera(c: CameraIntrinsics) -> N.tk_camera:
    return N.tk_camera(c.fx, c.fy, c.cx, c.cy, c.width, c.height, c.near_plane, c.far_plane)


def to_settings(s: RenderSettings) -> N.tk_settings:
    out = N.tk_settings()
    out.top_k = s.top_k
    out.tile_size = s.tile_size
    out.transmittance_floor = s.transmittance_floor
    out.background[:] = tuple(s.background)
    out.cov2d_dilation = s.cov2d_dilation
    out.alpha_clamp = s.alpha_clamp
    return out


def to_mapper_config(cfg: MapperConfig) -> N.tk_mapper_config:
    out = N.tk_mapper_config()
    for name, _ in N.tk_mapper_config._fields_:
        setattr(out, name, getattr(cfg, name))
    return out


class Renderer:
    """One CUDA context (tk_ctx) with a device-resident mirror of the last uploaded map."""

    def __init__(self, device: int = 0):
        self.lib = N.render_lib()
        h = C.c_void_p()
        N.check(self.lib.tk_create(device, C.byref(h)))
        self.ctx = h
        self._scene_token = None

    def close(self) -> None:
        if self.ctx:
            self.lib.tk_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- scene mirror
    def upload(self, m: SceneMap, force: bool = False) -> None:
        """Copy the map into the device mirror (SoA fp64 geometry, fp32 features)."""
        arrays = (_c(m.mean, np.float64), _c(m.log_scale, np.float64), _c(m.rotation, np.float64),
                  _c(m.opacity_logit, np.float64), _c(m.color, np.float64))
        feat = None if m.feature is None else _c(m.feature, np.float32)
        d = m.feature_dim if feat is None else int(feat.shape[1]) if feat.ndim == 2 else m.feature_dim
        view = N.tk_scene_view(m.size(), d, *(_p(a) for a in arrays), _p(feat), m.generation)
        N.check(self.lib.tk_scene_upload(self.ctx, C.byref(view), N.TK_HOST))
        self._keep = (arrays, feat)
        self._scene_token = None

    def _sync_scene(self, m: SceneMap) -> None:
        # The reference takes the map by const reference on every call; the drop-in re-uploads
        # it on every call so in-place edits are always seen.
        self.upload(m)

    def geometry_band(self, band: int, nbands: int) -> None:
        """Sweep only band `band` of `nbands` bands of tile rows (tk_geometry_band)."""
        N.check(self.lib.tk_geometry_band(self.ctx, band, nbands))

    def launches(self) -> int:
        return int(self.lib.tk_kernel_launches(self.ctx))

    def synchronize(self) -> None:
        N.check(self.lib.tk_synchronize(self.ctx))

    # ---------------------------------------------------------------- entry points
    def prepare_scene(self, m: SceneMap, pose: Pose, cam: CameraIntrinsics, s: RenderSettings) -> PreparedScene:
        """raster_detail::prepare_scene (render.cpp:73-156)."""
        self._sync_scene(m)
        ne, nt = C.c_int64(), C.c_int64()
        tx, ty = C.c_int32(), C.c_int32()
        N.check(self.lib.tk_prepare_scene(self.ctx, C.byref(to_pose(pose)), C.byref(to_camera(cam)),
                                          C.byref(to_settings(s)), C.byref(ne), C.byref(nt), C.byref(tx),
                                          C.byref(ty)))
        e7 = np.zeros((ne.value, 7))
        src = np.zeros(ne.value, np.int32)
        toff = np.zeros(tx.value * ty.value + 1, np.int32)
        tent = np.zeros(nt.value, np.int32)
        N.check(self.lib.tk_prepared_export(self.ctx, _p(e7), _p(src), _p(toff), _p(tent)))
        return PreparedScene(e7, src, toff, tent, tx.value, ty.value, cam.width, cam.height, m.generation, m.size())

    def render_geometric(self, m: SceneMap, pose: Pose, cam: CameraIntrinsics, s: RenderSettings) -> RenderOutput:
        """render_geometric (render.cpp:293-299)."""
        self._sync_scene(m)
        w, h = cam.width, cam.height
        k = max(0, min(s.top_k, K_MAX_TOP_K))
        color = np.zeros((h, w, 3))
        depth = np.zeros((h, w))
        alpha = np.zeros((h, w))
        index = np.zeros(w * h * k, np.int32)
        weight = np.zeros(w * h * k)
        count = np.zeros(w * h, np.uint8)
        contrib = np.zeros(m.size())
        out = N.tk_geom_out(N.TK_HOST, _p(color), _p(depth), _p(alpha), _p(index), _p(weight), _p(count),
                            _p(contrib), 0, 0)
        N.check(self.lib.tk_render_geometric(self.ctx, C.byref(to_pose(pose)), C.byref(to_camera(cam)),
                                             C.byref(to_settings(s)), C.byref(out)))
        return RenderOutput(color=color, depth=depth, alpha=alpha, topk=TopKGrid(w, h, k, index, weight, count),
                            contributions=contrib, generation=out.generation, map_size=out.map_size)

    @staticmethod
    def _topk_view(t: TopKGrid):
        idx = _c(t.index, np.int32)
        wt = _c(t.weight, np.float64)
        cnt = _c(t.count, np.uint8)
        return N.tk_topk_view(t.width, t.height, t.k, _p(idx), _p(wt), _p(cnt), N.TK_HOST), (idx, wt, cnt)

    def render_feature(self, m: SceneMap, topk: TopKGrid) -> np.ndarray:
        """render_feature (render.cpp:301-337): H x W x D (fp32)."""
        self._sync_scene(m)
        view, keep = self._topk_view(topk)
        out = np.zeros((topk.height, topk.width, m.feature_dim), np.float32)
        N.check(self.lib.tk_render_feature(self.ctx, C.byref(view), _p(out), N.TK_HOST))
        return out

    def comm_set_peers(self, rank: int, nranks: int, d_total: int, buffers: list[int], n_pixels: int) -> None:
        """Register every rank's full-width output buffer (device pointers, rank order) for the
        fused render + all-gather of ranks driven from one process (tk_comm_set_peers)."""
        arr = (C.c_void_p * len(buffers))(*buffers)
        N.check(self.lib.tk_comm_set_peers(self.ctx, rank, nranks, d_total, arr, n_pixels))

    def render_feature_gathered(self, m: SceneMap, topk: TopKGrid | None = None) -> None:
        """render_feature of this rank's channel slice stored into every rank's full-width buffer
        (tk_render_feature_gathered; topk None = this context's own records)."""
        self._sync_scene(m)
        if topk is None:
            N.check(self.lib.tk_render_feature_gathered(self.ctx, None, None, N.TK_HOST))
            return
        view, keep = self._topk_view(topk)
        N.check(self.lib.tk_render_feature_gathered(self.ctx, C.byref(view), None, N.TK_HOST))

    def render_feature_full_blend(self, m: SceneMap, pose: Pose, cam: CameraIntrinsics,
                                  s: RenderSettings) -> np.ndarray:
        """render_feature_full_blend (render.cpp:339-343)."""
        self._sync_scene(m)
        out = np.zeros((cam.height, cam.width, m.feature_dim), np.float32)
        N.check(self.lib.tk_render_feature_full_blend(self.ctx, C.byref(to_pose(pose)), C.byref(to_camera(cam)),
                                                      C.byref(to_settings(s)), _p(out), N.TK_HOST))
        return out

    def backward_feature(self, m: SceneMap, topk: TopKGrid, grad_feature: np.ndarray) -> np.ndarray:
        """backward_feature (backward.cpp:273-321): flat N x D."""
        self._sync_scene(m)
        view, keep = self._topk_view(topk)
        g = _c(grad_feature, np.float32)
        if g.size != topk.width * topk.height * m.feature_dim:
            raise ValueError("backward_feature: grad_feature shape does not match the grid")
        out = np.zeros(m.size() * m.feature_dim, np.float32)
        N.check(self.lib.tk_backward_feature(self.ctx, C.byref(view), _p(g), N.TK_HOST, _p(out), N.TK_HOST))
        return out

    def backward_geometric(self, m: SceneMap, pose: Pose, cam: CameraIntrinsics, s: RenderSettings,
                           grad_color: np.ndarray, grad_depth: np.ndarray | None) -> GeomGrads:
        """backward_geometric (backward.cpp:72-271)."""
        self._sync_scene(m)
        n = m.size()
        gc = _c(grad_color, np.float64)
        gd = None if grad_depth is None or np.size(grad_depth) == 0 else _c(grad_depth, np.float64)
        if gc.size != cam.width * cam.height * 3:
            raise ValueError("backward_geometric: grad_color shape does not match the camera")
        g = GeomGrads(np.zeros((n, 3)), np.zeros((n, 3)), np.zeros((n, 4)), np.zeros(n), np.zeros((n, 3)),
                      np.zeros(6))
        out = N.tk_geom_grads(N.TK_HOST, _p(g.mean), _p(g.log_scale), _p(g.rotation), _p(g.opacity_logit),
                              _p(g.color))
        N.check(self.lib.tk_backward_geometric(self.ctx, C.byref(to_pose(pose)), C.byref(to_camera(cam)),
                                               C.byref(to_settings(s)), _p(gc), _p(gd), N.TK_HOST, C.byref(out)))
        g.pose_twist[:] = list(out.pose_twist)
        return g

    # ---------------------------------------------------------------- mapping iteration
    def keyframe_set(self, slot: int, pose: Pose, frame: Frame) -> None:
        """Store a keyframe (SceneMap::keyframes entry) device-resident."""
        col = _c(frame.color, np.float32)
        dep = _c(frame.depth, np.float32)
        feat = None if frame.feature is None else _c(frame.feature, np.float32)
        h, w = dep.shape[:2]
        d = 0 if feat is None else int(feat.shape[-1])
        if col.size != w * h * 3 or (feat is not None and feat.size != w * h * d):
            raise ValueError("keyframe_set: frame images disagree in shape")
        view = N.tk_frame_view(w, h, d, _p(col), _p(dep), _p(feat), N.TK_HOST)
        N.check(self.lib.tk_keyframe_set(self.ctx, slot, C.byref(to_pose(pose)), C.byref(view)))

    def keyframe_load_features(self, slot: int, path: str) -> None:
        """Replace keyframe `slot`'s feature image from a FEAT file (dataset.cpp:63-76)."""
        N.check(self.lib.tk_keyframe_load_features(self.ctx, slot, str(path).encode()))

    def keyframe_save_features(self, slot: int, path: str) -> None:
        """Write keyframe `slot`'s feature image as a FEAT file (dataset.cpp:48-61)."""
        N.check(self.lib.tk_keyframe_save_features(self.ctx, slot, str(path).encode()))

    def optimizer_reset(self, reset_stats: bool = True) -> None:
        """A zeroed OptimizerState (optimizer.hpp:25-53) for the resident map."""
        N.check(self.lib.tk_optimizer_reset(self.ctx, int(reset_stats)))

    def optimize_step(self, cfg: MapperConfig, cam: CameraIntrinsics, s: RenderSettings, slot: int,
                      iteration: int, fetch: bool = True) -> tuple[LossValues | None, bool]:
        """optimize_step on keyframe `slot` (mapper.cpp:162-255 without pruning).  With fetch=False the
        loss values stay on the device (no synchronisation); read them with loss_values()."""
        vals = (C.c_double * 3)()
        fs = C.c_int32()
        N.check(self.lib.tk_optimize_step(self.ctx, C.byref(to_mapper_config(cfg)), C.byref(to_camera(cam)),
                                          C.byref(to_settings(s)), slot, iteration,
                                          vals if fetch else None, C.byref(fs)))
        return (LossValues(vals[0], vals[1], vals[2]) if fetch else None), bool(fs.value)

    def loss_values(self) -> LossValues:
        vals = (C.c_double * 3)()
        N.check(self.lib.tk_loss_values(self.ctx, vals))
        return LossValues(vals[0], vals[1], vals[2])

    def scene_download(self, n: int, d: int, stats: bool = True) -> dict:
        """The resident map's parameters and (stats=True) selection statistics."""
        o = dict(mean=np.zeros((n, 3)), log_scale=np.zeros((n, 3)), rotation=np.zeros((n, 4)),
                 opacity_logit=np.zeros(n), color=np.zeros((n, 3)), feature=np.zeros((n, d), np.float32))
        if stats:
            o.update(topk_count=np.zeros(n, np.int32), max_contribution=np.zeros(n))
        out = N.tk_scene_out(N.TK_HOST, *[_p(o.get(x)) for x in ("mean", "log_scale", "rotation", "opacity_logit",
                                                                  "color", "feature", "topk_count",
                                                                  "max_contribution")])
        N.check(self.lib.tk_scene_download(self.ctx, C.byref(out)))
        return o


    def scene_info(self) -> tuple[int, int, int]:
        n, d, g = C.c_int64(), C.c_int32(), C.c_uint64()
        N.check(self.lib.tk_scene_info(self.ctx, C.byref(n), C.byref(d), C.byref(g)))
        return n.value, d.value, g.value

    def insert_gaussians(self, position, color, feature, spacing, distance, tau: float, world_to_camera: Pose) -> int:
        """insert_gaussians (mapper.cpp:19-60) on the resident map; returns the number inserted."""
        pos = _c(position, np.float64).reshape(-1, 3)
        n = pos.shape[0]
        col = _c(color, np.float64).reshape(n, 3)
        feat = None if feature is None else _c(feature, np.float32).reshape(n, -1)
        d = 0 if feat is None else feat.shape[1]
        sp = _c(spacing, np.float64).reshape(n)
        dist = _c(distance, np.float64).reshape(n)
        view = N.tk_source_view(n, d, _p(pos), _p(col), _p(feat), _p(sp), _p(dist), N.TK_HOST)
        out = C.c_int32()
        N.check(self.lib.tk_insert_gaussians(self.ctx, C.byref(view), tau, C.byref(to_pose(world_to_camera)),
                                             C.byref(out)))
        return out.value

    def prune_map(self, keep_ratio: float, seed: int, threshold: int) -> np.ndarray:
        """prune_map (mapper.cpp:80-160); returns the removed indices (ascending)."""
        n = self.scene_info()[0]
        out = np.zeros(max(n, 1), np.int32)
        k = C.c_int64()
        N.check(self.lib.tk_prune_map(self.ctx, keep_ratio, seed & ((1 << 64) - 1), threshold, _p(out), C.byref(k)))
        return out[:k.value].copy()


    # ---------------------------------------------------------------- checkpoint / query
    def checkpoint_save(self, path: str) -> None:
        """save_checkpoint (checkpoint.cpp:39-63) of the resident map (SPLF v1)."""
        N.check(self.lib.tk_checkpoint_save(self.ctx, path.encode()))

    def checkpoint_load(self, path: str) -> tuple[int, int]:
        """load_checkpoint (checkpoint.cpp:65-98) straight into the device SoA; returns (n, d)."""
        N.check(self.lib.tk_checkpoint_load(self.ctx, path.encode()))
        n, d, _ = self.scene_info()
        return n, d

    def segment_by_query(self, feature: np.ndarray | None, embeddings: np.ndarray,
                         shape: tuple[int, int] | None = None) -> np.ndarray:
        """segment_by_query (metrics.cpp:66-94): H x W uint8 labels (255 = invalid).  feature None:
        the last render_feature output of this context (shape = (H, W) then)."""
        emb = _c(embeddings, np.float64)
        if feature is None:
            h, w = shape
            f, n, d, mem = None, h * w, 0, N.TK_DEVICE
        else:
            f = _c(feature, np.float32)
            h, w, d = f.shape
            n, mem = h * w, N.TK_HOST
        if feature is not None and emb.shape[1] != d:
            raise RuntimeError("segment_by_query: embedding dimension mismatch")
        out = np.zeros((h, w), np.uint8)
        N.check(self.lib.tk_segment_by_query(self.ctx, _p(f), n, d, mem, _p(emb), emb.shape[0], _p(out), N.TK_HOST))
        return out


class MT19937_64:
    """std::mt19937_64 (the reference mapper's keyframe sampler, mapper.cpp:167)."""

    _MASK = (1 << 64) - 1

    def __init__(self, seed: int = 5489):
        self.mt = [0] * 312
        self.mt[0] = seed & self._MASK
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & self._MASK
        self.idx = 312

    def _twist(self) -> None:
        mt = self.mt
        for i in range(312):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= 312:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEB880000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & self._MASK


class Mapper:
    """The mapping loop of map/mapper.cpp over a device-resident map: keyframes live in HBM, each
    optimize_step samples one with ``rng() % len(keyframes)`` (mapper.cpp:167), runs render,
    losses, backward and Adam on the GPU and prunes on schedule (mapper.cpp:256-260)."""

    def __init__(self, renderer: Renderer, m: SceneMap, cfg: MapperConfig, cam: CameraIntrinsics,
                 settings: RenderSettings | None = None):
        self.r, self.cfg, self.cam = renderer, cfg, cam
        self.settings = settings or RenderSettings()
        self.n, self.d = m.size(), m.feature_dim
        renderer.upload(m)
        renderer.optimizer_reset(True)
        self.n_keyframes = 0

    def add_keyframe(self, pose: Pose, frame: Frame) -> int:
        self.r.keyframe_set(self.n_keyframes, pose, frame)
        self.n_keyframes += 1
        return self.n_keyframes - 1

    def optimize_step(self, iteration: int, rng: MT19937_64, fetch: bool = True):
        if self.n_keyframes == 0:
            raise RuntimeError("optimize_step: no keyframes")
        slot = rng() % self.n_keyframes
        vals, fstep = self.r.optimize_step(self.cfg, self.cam, self.settings, slot, iteration, fetch)
        pruned = 0
        c = self.cfg
        if c.pruning and c.prune_period > 0 and iteration > 0 and iteration % c.prune_period == 0:
            pruned = len(self.r.prune_map(c.prune_keep_ratio, rng(), c.topk_count_threshold))
            self.n, self.d, _ = self.r.scene_info()
        return dict(iteration=iteration, losses=vals, feature_step=fstep, keyframe=slot, pruned=pruned,
                    gaussian_count=self.n)

    def insert(self, position, color, feature, spacing, distance, world_to_camera: Pose) -> int:
        """insert_gaussians with the config's tau_insert; the optimiser state extends in lockstep."""
        k = self.r.insert_gaussians(position, color, feature, spacing, distance, self.cfg.tau_insert,
                                    world_to_camera)
        self.n, self.d, _ = self.r.scene_info()
        return k

    def export(self) -> dict:
        return self.r.scene_download(self.n, self.d)


_default: Renderer | None = None


def default_renderer() -> Renderer:
    global _default
    if _default is None:
        _default = Renderer(0)
    return _default


def prepare_scene(m, pose, cam, s):
    return default_renderer().prepare_scene(m, pose, cam, s)


def render_geometric(m, pose, cam, s):
    return default_renderer().render_geometric(m, pose, cam, s)


def render_feature(m, topk):
    return default_renderer().render_feature(m, topk)


def render_feature_full_blend(m, pose, cam, s):
    return default_renderer().render_feature_full_blend(m, pose, cam, s)


def backward_feature(m, topk, grad_feature):
    return default_renderer().backward_feature(m, topk, grad_feature)


def backward_geometric(m, pose, cam, s, grad_color, grad_depth):
    return default_renderer().backward_geometric(m, pose, cam, s, grad_color, grad_depth)

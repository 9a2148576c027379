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
from .types import (CameraIntrinsics, GeomGrads, Pose, PreparedScene, RenderOutput, RenderSettings, SceneMap,
                    TopKGrid, K_MAX_TOP_K)


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

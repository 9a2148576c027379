"""ctypes wrapper of the CPU oracle (oracle/include/oracle.h).

TEST INFRASTRUCTURE ONLY: the checker the GPU path is compared against, never the product.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_LIB = os.path.join(ORACLE_DIR, "_build", "liboracle.so")


class orc_camera(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32), ("near_plane", C.c_double), ("far_plane", C.c_double)]


class orc_pose(C.Structure):
    _fields_ = [("qw", C.c_double), ("qx", C.c_double), ("qy", C.c_double), ("qz", C.c_double),
                ("tx", C.c_double), ("ty", C.c_double), ("tz", C.c_double)]


class orc_settings(C.Structure):
    _fields_ = [("top_k", C.c_int32), ("tile_size", C.c_int32), ("transmittance_floor", C.c_double),
                ("background", C.c_double * 3), ("cov2d_dilation", C.c_double), ("alpha_clamp", C.c_double)]


_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)
    return ORACLE_LIB


def lib():
    global _lib
    if _lib is None:
        srcs = [os.path.join(ORACLE_DIR, "src", f) for f in ("oracle.cpp", "oracle_mapping.inc")]
        srcs.append(os.path.join(ORACLE_DIR, "include", "oracle.h"))
        if not os.path.exists(ORACLE_LIB) or any(
                os.path.exists(f) and os.path.getmtime(f) > os.path.getmtime(ORACLE_LIB) for f in srcs):
            build()
        L = C.CDLL(ORACLE_LIB)
        vp = C.c_void_p
        L.orc_last_error.restype = C.c_char_p
        L.orc_map_create.restype = vp
        L.orc_map_create.argtypes = [C.c_int64, C.c_int32, vp, vp, vp, vp, vp, vp, C.c_uint64]
        L.orc_map_free.argtypes = [vp]
        L.orc_project_gaussian.argtypes = [vp, C.c_int64, vp, vp, C.c_double, vp]
        L.orc_prepare_scene.restype = vp
        L.orc_prepare_scene.argtypes = [vp, vp, vp, vp]
        L.orc_prep_sizes.argtypes = [vp, vp, vp, vp, vp]
        L.orc_prep_export.argtypes = [vp, vp, vp, vp, vp]
        L.orc_prep_free.argtypes = [vp]
        L.orc_geometric_pass.argtypes = [vp] * 10
        L.orc_render_geometric.argtypes = [vp] * 11
        L.orc_render_feature.argtypes = [vp, C.c_int32, C.c_int32, C.c_int32, vp, vp, vp, vp]
        L.orc_render_feature_full_blend.argtypes = [vp] * 5
        L.orc_backward_feature.argtypes = [vp, C.c_int32, C.c_int32, C.c_int32, vp, vp, vp, vp, vp]
        L.orc_backward_geometric.argtypes = [vp] * 12
        L.orc_render_reference.argtypes = [vp] * 17
        L.orc_time_frame.argtypes = [vp, vp, vp, vp, vp, vp, vp, C.c_int, C.c_int, vp]
        L.orc_max_threads.restype = C.c_int
        L.orc_set_threads.argtypes = [C.c_int]
        L.orc_opt_create.restype = vp
        L.orc_opt_create.argtypes = [C.c_int64, C.c_int32]
        L.orc_opt_free.argtypes = [vp]
        L.orc_ssim_with_grad.restype = C.c_double
        L.orc_ssim_with_grad.argtypes = [C.c_int32, C.c_int32, C.c_int32, vp, vp, vp]
        L.orc_compute_losses.argtypes = [C.c_int32, C.c_int32, C.c_int32] + [vp] * 8 + [C.c_int32] + [vp] * 4
        L.orc_optimize_step.argtypes = [vp] * 9 + [C.c_int64, vp, vp]
        L.orc_map_export.argtypes = [vp] * 9
        L.orc_insert_gaussians.restype = C.c_int
        L.orc_insert_gaussians.argtypes = [vp, vp, C.c_int64, vp, vp, vp, C.c_int32, vp, vp, C.c_double, vp]
        L.orc_prune_map.restype = C.c_int64
        L.orc_prune_map.argtypes = [vp, vp, C.c_double, C.c_uint64, C.c_int32, vp]
        L.orc_map_size.restype = C.c_int64
        L.orc_map_size.argtypes = [vp]
        L.orc_map_generation.restype = C.c_uint64
        L.orc_map_generation.argtypes = [vp]
        L.orc_map_feature_dim.restype = C.c_int32
        L.orc_map_feature_dim.argtypes = [vp]
        L.orc_map_set_stats.argtypes = [vp, vp, vp]
        L.orc_opt_moments.restype = C.POINTER(C.c_double)
        L.orc_opt_moments.argtypes = [vp, C.c_int32, C.c_int32, C.POINTER(C.c_int64)]
        L.orc_checkpoint_save.restype = C.c_int
        L.orc_checkpoint_save.argtypes = [vp, C.c_char_p]
        L.orc_checkpoint_load.restype = vp
        L.orc_checkpoint_load.argtypes = [C.c_char_p]
        L.orc_segment_by_query.argtypes = [C.c_int32, C.c_int32, C.c_int32, vp, C.c_int32, vp, vp]
        L.orc_update_contribution_stats.argtypes = [vp, C.c_uint64, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                                                    vp, vp, vp]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def pose_c(p):
    q, t = p.rotation, p.translation
    return orc_pose(q[0], q[1], q[2], q[3], t[0], t[1], t[2])


def cam_c(c):
    return orc_camera(c.fx, c.fy, c.cx, c.cy, c.width, c.height, c.near_plane, c.far_plane)


def settings_c(s):
    o = orc_settings()
    o.top_k, o.tile_size, o.transmittance_floor = s.top_k, s.tile_size, s.transmittance_floor
    o.background[:] = tuple(s.background)
    o.cov2d_dilation, o.alpha_clamp = s.cov2d_dilation, s.alpha_clamp
    return o


class OracleMap:
    """SceneMap in the oracle's AoS layout (fp64 features)."""

    def __init__(self, m):
        self.n, self.d = m.size(), m.feature_dim
        arrs = [np.ascontiguousarray(a, np.float64) for a in (m.mean, m.log_scale, m.rotation, m.opacity_logit,
                                                              m.color)]
        feat = None if m.feature is None else np.ascontiguousarray(m.feature, np.float64)
        self.h = lib().orc_map_create(self.n, self.d, *[_p(a) for a in arrs], _p(feat), m.generation)

    def __del__(self):
        try:
            lib().orc_map_free(self.h)
        except Exception:
            pass


def render_geometric(m, pose, cam, s):
    om = OracleMap(m)
    W, H = cam.width, cam.height
    k = min(s.top_k, 32)
    out = dict(color=np.zeros((H, W, 3)), depth=np.zeros((H, W)), alpha=np.zeros((H, W)),
               index=np.zeros(W * H * k, np.int32), weight=np.zeros(W * H * k), count=np.zeros(W * H, np.uint8),
               contributions=np.zeros(m.size()))
    lib().orc_render_geometric(om.h, C.byref(pose_c(pose)), C.byref(cam_c(cam)), C.byref(settings_c(s)),
                               *[_p(out[x]) for x in ("color", "depth", "alpha", "index", "weight", "count",
                                                      "contributions")])
    out["k"] = k
    return out


def prepare_scene(m, pose, cam, s):
    om = OracleMap(m)
    L = lib()
    h = L.orc_prepare_scene(om.h, C.byref(pose_c(pose)), C.byref(cam_c(cam)), C.byref(settings_c(s)))
    ne, nt, tx, ty = C.c_int64(), C.c_int64(), C.c_int32(), C.c_int32()
    L.orc_prep_sizes(h, C.byref(ne), C.byref(nt), C.byref(tx), C.byref(ty))
    e7 = np.zeros((ne.value, 7))
    src = np.zeros(ne.value, np.int32)
    toff = np.zeros(tx.value * ty.value + 1, np.int32)
    tent = np.zeros(nt.value, np.int32)
    L.orc_prep_export(h, _p(e7), _p(src), _p(toff), _p(tent))
    L.orc_prep_free(h)
    return dict(entries=e7, src=src, tile_offsets=toff, tile_entries=tent, tiles_x=tx.value, tiles_y=ty.value)


def project_gaussian(m, i, pose, cam, dilation=0.3):
    om = OracleMap(m)
    out = np.zeros(7)
    vis = lib().orc_project_gaussian(om.h, i, C.byref(pose_c(pose)), C.byref(cam_c(cam)), C.c_double(dilation),
                                     _p(out))
    return bool(vis), out


class StaleIndex(RuntimeError):
    pass


def render_feature(m, w, h, k, index, weight, count):
    om = OracleMap(m)
    out = np.zeros((h, w, m.feature_dim))
    rc = lib().orc_render_feature(om.h, w, h, k, _p(np.ascontiguousarray(index, np.int32)),
                                  _p(np.ascontiguousarray(weight, np.float64)),
                                  _p(np.ascontiguousarray(count, np.uint8)), _p(out))
    if rc:
        raise StaleIndex(lib().orc_last_error().decode())
    return out


def render_feature_full_blend(m, pose, cam, s):
    om = OracleMap(m)
    out = np.zeros((cam.height, cam.width, m.feature_dim))
    lib().orc_render_feature_full_blend(om.h, C.byref(pose_c(pose)), C.byref(cam_c(cam)), C.byref(settings_c(s)),
                                        _p(out))
    return out


def backward_feature(m, w, h, k, index, weight, count, grad):
    om = OracleMap(m)
    out = np.zeros(m.size() * m.feature_dim)
    g = np.ascontiguousarray(grad, np.float64)
    rc = lib().orc_backward_feature(om.h, w, h, k, _p(np.ascontiguousarray(index, np.int32)),
                                    _p(np.ascontiguousarray(weight, np.float64)),
                                    _p(np.ascontiguousarray(count, np.uint8)), _p(g), _p(out))
    if rc:
        raise StaleIndex(lib().orc_last_error().decode())
    return out


def _mem_available_gb() -> float:
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable"):
                return int(line.split()[1]) / 2**20
    except OSError:
        pass
    return 16.0


def backward_feature_slices(m, w, h, k, index, weight, count, grad, width=64):
    """backward_feature (backward.cpp:273-321) one channel slice at a time: the op never mixes
    channels (each channel of dF scatters into the same channel of df), so the oracle run on a map
    holding channels [c0, c1) and on grad[..., c0:c1] is exactly that slice of the full result.
    Keeps the oracle's per-thread N x width fp64 partials (backward.cpp:290-291) within host RAM
    at configs 3 and 5.  Yields (c0, c1, df_slice[n, c1 - c0])."""
    from paper_2602_06991_b200.types import SceneMap
    n, d = m.size(), m.feature_dim
    L = lib()
    cores = L.orc_max_threads()
    per_thread_gb = n * width * 8 / 2**30
    threads = max(1, min(cores, int((_mem_available_gb() * 0.5 - 2 * per_thread_gb) / max(per_thread_gb, 1e-9))))
    L.orc_set_threads(threads)
    try:
        idx = np.ascontiguousarray(index, np.int32)
        wt = np.ascontiguousarray(weight, np.float64)
        cnt = np.ascontiguousarray(count, np.uint8)
        g3 = grad.reshape(h, w, d)
        for c0 in range(0, d, width):
            c1 = min(d, c0 + width)
            ms = SceneMap(m.mean, m.log_scale, m.rotation, m.opacity_logit, m.color,
                          np.ascontiguousarray(m.feature[:, c0:c1]), m.generation, c1 - c0)
            yield c0, c1, backward_feature(ms, w, h, k, idx, wt, cnt,
                                           np.ascontiguousarray(g3[..., c0:c1], np.float64)).reshape(n, c1 - c0)
    finally:
        L.orc_set_threads(cores)


def backward_geometric(m, pose, cam, s, grad_color, grad_depth):
    om = OracleMap(m)
    n = m.size()
    g = dict(mean=np.zeros((n, 3)), log_scale=np.zeros((n, 3)), rotation=np.zeros((n, 4)),
             opacity_logit=np.zeros(n), color=np.zeros((n, 3)), pose_twist=np.zeros(6))
    gc = np.ascontiguousarray(grad_color, np.float64)
    gd = None if grad_depth is None else np.ascontiguousarray(grad_depth, np.float64)
    lib().orc_backward_geometric(om.h, C.byref(pose_c(pose)), C.byref(cam_c(cam)), C.byref(settings_c(s)), _p(gc),
                                 _p(gd), *[_p(g[x]) for x in ("mean", "log_scale", "rotation", "opacity_logit",
                                                              "color", "pose_twist")])
    return g


def render_reference(m, pose, cam, s, with_features=False, keep_records=False):
    om = OracleMap(m)
    W, H = cam.width, cam.height
    P = W * H
    k = min(s.top_k, 32)
    o = dict(color=np.zeros((H, W, 3)), depth=np.zeros((H, W)), alpha=np.zeros((H, W)),
             transmittance=np.zeros((H, W)), feature_blend=np.zeros((H, W, m.feature_dim)) if with_features else None,
             index=np.zeros(P * k, np.int32), weight=np.zeros(P * k), count=np.zeros(P, np.uint8),
             contributions=np.zeros(m.size()))
    nrec = C.c_int64()
    L = lib()
    args = [om.h, C.byref(pose_c(pose)), C.byref(cam_c(cam)), C.byref(settings_c(s))]
    outs = [_p(o[x]) for x in ("color", "depth", "alpha", "transmittance", "feature_blend", "index", "weight",
                               "count", "contributions")]
    if keep_records:
        L.orc_render_reference(*args, *[None] * 9, None, None, None, C.byref(nrec))
        offs = np.zeros(P + 1, np.int64)
        ri = np.zeros(nrec.value, np.int32)
        rw = np.zeros(nrec.value)
        L.orc_render_reference(*args, *outs, _p(offs), _p(ri), _p(rw), C.byref(nrec))
        o["records"] = [list(zip(ri[offs[p]:offs[p + 1]], rw[offs[p]:offs[p + 1]])) for p in range(P)]
    else:
        L.orc_render_reference(*args, *outs, None, None, None, C.byref(nrec))
    o["k"] = k
    return o


class orc_mapper_config(C.Structure):
    _fields_ = [("lambda_geo", C.c_double), ("lambda_feat", C.c_double), ("lambda1", C.c_double),
                ("lambda2", C.c_double), ("color_secondary", C.c_int32), ("feature_update_period", C.c_int32),
                ("l1_deadband", C.c_double), ("lr_mean", C.c_double), ("lr_log_scale", C.c_double),
                ("lr_rotation", C.c_double), ("lr_opacity", C.c_double), ("lr_color", C.c_double),
                ("lr_feature", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
                ("min_log_scale", C.c_double), ("max_log_scale", C.c_double)]


def mapper_config_c(cfg):
    o = orc_mapper_config()
    for name, _ in orc_mapper_config._fields_:
        setattr(o, name, getattr(cfg, name))
    return o


def ssim_with_grad(a, b):
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    h, w, c = a.shape
    g = np.zeros_like(a)
    return lib().orc_ssim_with_grad(w, h, c, _p(a), _p(b), _p(g)), g


def compute_losses(color, depth, count, feature, gt_color, gt_depth, gt_feature, cfg, include_feature):
    """compute_losses (losses.cpp:22-133) -> (values{map,geo,feat}, grad_color, grad_depth, grad_feature)."""
    h, w = depth.shape
    d = 0 if gt_feature is None else gt_feature.shape[-1]
    vals = np.zeros(3)
    gc, gd = np.zeros((h, w, 3)), np.zeros((h, w))
    gf = np.zeros((h, w, d)) if include_feature else None
    f = None if feature is None else np.ascontiguousarray(feature, np.float64)
    gtf = None if gt_feature is None else np.ascontiguousarray(gt_feature, np.float32)
    lib().orc_compute_losses(w, h, d, _p(np.ascontiguousarray(color, np.float64)),
                             _p(np.ascontiguousarray(depth, np.float64)), _p(np.ascontiguousarray(count, np.uint8)),
                             _p(f), _p(np.ascontiguousarray(gt_color, np.float32)),
                             _p(np.ascontiguousarray(gt_depth, np.float32)), _p(gtf),
                             C.byref(mapper_config_c(cfg)), int(include_feature), _p(vals), _p(gc), _p(gd), _p(gf))
    return dict(map=vals[0], geo=vals[1], feat=vals[2]), gc, gd, gf


class OracleMapper:
    """SceneMap + OptimizerState driven through optimize_step (mapper.cpp:162-255, no pruning)."""

    def __init__(self, m, cfg):
        self.map = OracleMap(m)
        self.n, self.d = self.map.n, self.map.d
        self.opt = lib().orc_opt_create(self.n, self.d)
        self.cfg = mapper_config_c(cfg)

    def __del__(self):
        try:
            lib().orc_opt_free(self.opt)
        except Exception:
            pass

    def step(self, pose, cam, s, gt_color, gt_depth, gt_feature, iteration):
        vals = np.zeros(3)
        fs = C.c_int32()
        gtf = None if gt_feature is None else np.ascontiguousarray(gt_feature, np.float32)
        lib().orc_optimize_step(self.map.h, self.opt, C.byref(self.cfg), C.byref(cam_c(cam)), C.byref(settings_c(s)),
                                C.byref(pose_c(pose)), _p(np.ascontiguousarray(gt_color, np.float32)),
                                _p(np.ascontiguousarray(gt_depth, np.float32)), _p(gtf), int(iteration), _p(vals),
                                C.byref(fs))
        return dict(map=vals[0], geo=vals[1], feat=vals[2]), bool(fs.value)

    def update_contribution_stats(self, generation, map_size, w, h, k, index, count, contributions):
        rc = lib().orc_update_contribution_stats(self.map.h, generation, map_size, w, h, k,
                                                 _p(np.ascontiguousarray(index, np.int32)),
                                                 _p(np.ascontiguousarray(count, np.uint8)),
                                                 _p(np.ascontiguousarray(contributions, np.float64)))
        if rc:
            raise RuntimeError(lib().orc_last_error().decode())

    def size(self):
        return int(lib().orc_map_size(self.map.h))

    def generation(self):
        return int(lib().orc_map_generation(self.map.h))

    def set_stats(self, topk_count, max_contribution):
        lib().orc_map_set_stats(self.map.h, _p(np.ascontiguousarray(topk_count, np.int32)),
                                _p(np.ascontiguousarray(max_contribution, np.float64)))

    def moments(self, group, which=0):
        cnt = C.c_int64()
        ptr = lib().orc_opt_moments(self.opt, group, which, C.byref(cnt))
        return np.ctypeslib.as_array(ptr, shape=(cnt.value,)) if cnt.value else np.zeros(0)

    def insert(self, position, color, feature, spacing, distance, tau, pose):
        """insert_gaussians (mapper.cpp:19-60); returns the number inserted."""
        pos = np.ascontiguousarray(position, np.float64)
        f = None if feature is None else np.ascontiguousarray(feature, np.float64)
        d_src = 0 if f is None else f.shape[1]
        n = lib().orc_insert_gaussians(self.map.h, self.opt, pos.shape[0], _p(pos),
                                       _p(np.ascontiguousarray(color, np.float64)), _p(f), d_src,
                                       _p(np.ascontiguousarray(spacing, np.float64)),
                                       _p(np.ascontiguousarray(distance, np.float64)), tau, C.byref(pose_c(pose)))
        self.n = self.size()
        self.d = int(lib().orc_map_feature_dim(self.map.h))
        return n

    def prune(self, keep_ratio, seed, threshold):
        """prune_map (mapper.cpp:80-160); returns the removed indices."""
        out = np.zeros(max(1, self.size()), np.int32)
        k = lib().orc_prune_map(self.map.h, self.opt, keep_ratio, seed, threshold, _p(out))
        self.n = self.size()
        return out[:k].copy()

    def export(self):
        n, d = self.size(), self.d
        o = dict(mean=np.zeros((n, 3)), log_scale=np.zeros((n, 3)), rotation=np.zeros((n, 4)),
                 opacity_logit=np.zeros(n), color=np.zeros((n, 3)), feature=np.zeros((n, d)),
                 topk_count=np.zeros(n, np.int32), max_contribution=np.zeros(n))
        lib().orc_map_export(self.map.h, *[_p(o[x]) for x in ("mean", "log_scale", "rotation", "opacity_logit",
                                                              "color", "feature", "topk_count", "max_contribution")])
        return o


def checkpoint_save(m, path):
    om = OracleMap(m)
    if lib().orc_checkpoint_save(om.h, path.encode()):
        raise RuntimeError(lib().orc_last_error().decode())


def checkpoint_load(path):
    """load_checkpoint -> dict of SoA arrays (fp64) + feature_dim."""
    h = lib().orc_checkpoint_load(path.encode())
    if not h:
        raise RuntimeError(lib().orc_last_error().decode())
    n = int(lib().orc_map_size(h))
    d = int(lib().orc_map_feature_dim(h))
    o = dict(mean=np.zeros((n, 3)), log_scale=np.zeros((n, 3)), rotation=np.zeros((n, 4)),
             opacity_logit=np.zeros(n), color=np.zeros((n, 3)), feature=np.zeros((n, d)))
    lib().orc_map_export(h, *[_p(o[x]) for x in ("mean", "log_scale", "rotation", "opacity_logit", "color",
                                                 "feature")], None, None)
    lib().orc_map_free(h)
    o["feature_dim"] = d
    return o


def segment_by_query(feature, emb):
    f = np.ascontiguousarray(feature, np.float64)
    e = np.ascontiguousarray(emb, np.float64)
    h, w, d = f.shape
    out = np.zeros((h, w), np.uint8)
    lib().orc_segment_by_query(w, h, d, _p(f), e.shape[0], _p(e), _p(out))
    return out

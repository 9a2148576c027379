"""Synthetic inputs: the reference's generators (testutil.hpp, scene.cpp) restated in host C++
(scenegen/csrc/synth.cpp, scenegen/include/tk_synth.h) so the GPU path and the oracle see identical
inputs.  Input synthesis for the tests and the bench; the product library never loads it."""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from paper_2602_06991_b200.types import CameraIntrinsics, Pose, SceneMap

from . import _lib as N


def _arrays(n: int, d: int, with_features: bool):
    a = {
        "mean": np.zeros((n, 3)), "log_scale": np.zeros((n, 3)), "rotation": np.zeros((n, 4)),
        "opacity_logit": np.zeros(n), "color": np.zeros((n, 3)),
        "feature": np.zeros((n, d)) if with_features else None,
    }
    v = N.tk_synth_arrays(n, d, *(a[k].ctypes.data if a[k] is not None else None
                                  for k in ("mean", "log_scale", "rotation", "opacity_logit", "color", "feature")))
    return a, v


def random_scene(count: int, feature_dim: int, seed: int, depth_min: float = 0.8,
                 depth_max: float = 6.0) -> SceneMap:
    """testutil::random_scene (proj/tests/testutil.hpp:31-53)."""
    a, v = _arrays(count, feature_dim, True)
    N.synth_lib().tk_synth_random_scene(count, feature_dim, seed, depth_min, depth_max, C.byref(v))
    return SceneMap(feature_dim=feature_dim, **a)


def test_camera(width: int, height: int, focal: float = 0.0) -> CameraIntrinsics:
    """testutil::test_camera (proj/tests/testutil.hpp:55-65)."""
    f = focal if focal > 0.0 else 0.9 * width
    return CameraIntrinsics(fx=f, fy=f, cx=0.5 * (width - 1), cy=0.5 * (height - 1), width=width, height=height,
                            near_plane=0.05, far_plane=50.0)


def default_spec(**kw) -> N.tk_synth_spec:
    s = N.tk_synth_spec()
    N.synth_lib().tk_synth_default_spec(C.byref(s))
    for k, val in kw.items():
        if k in ("room_min", "room_max"):
            getattr(s, k)[:] = val
        else:
            setattr(s, k, val)
    return s


def build_synthetic_scene(spec: N.tk_synth_spec, truncate: int | None = None):
    """build_synthetic_scene (proj/src/synth/scene.cpp:73-144); returns (SceneMap, class_ids)."""
    lib = N.synth_lib()
    n = lib.tk_synth_build_scene(C.byref(spec), None, None)
    if n < 0:
        raise ValueError("build_synthetic_scene: feature_dim must be >= classes")
    m = n if truncate is None else min(n, truncate)
    a, v = _arrays(m, spec.feature_dim, True)
    cls = np.zeros(m, dtype=np.uint8)
    lib.tk_synth_build_scene(C.byref(spec), C.byref(v), cls.ctypes.data)
    return SceneMap(feature_dim=spec.feature_dim, **a), cls


def generate_trajectory(kind: str, n: int, spec: N.tk_synth_spec) -> list[Pose]:
    """generate_trajectory (proj/src/synth/scene.cpp:169-230); kind 'orbit' or 'lawnmower'."""
    out = np.zeros((n, 7))
    if N.synth_lib().tk_synth_trajectory(0 if kind == "orbit" else 1, n, C.byref(spec), out.ctypes.data) != 0:
        raise ValueError("generate_trajectory: need at least 2 poses")
    return [Pose(rotation=tuple(r[:4]), translation=tuple(r[4:])) for r in out]


def unit_features(n: int, d: int, seed: int, dtype=np.float32) -> np.ndarray:
    """Seeded random unit rows (SURVEY.md §8(d) replacement for the one-hot embeddings)."""
    out = np.empty((n, d), dtype=dtype)
    if dtype == np.float32:
        N.synth_lib().tk_synth_unit_features(n, d, seed, out.ctypes.data, None)
    else:
        N.synth_lib().tk_synth_unit_features(n, d, seed, None, out.ctypes.data)
    return out


def uniform_image(shape, seed: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """Seeded U(lo, hi) image (test_backward.cpp:96-100 random_image)."""
    out = np.empty(int(np.prod(shape)))
    N.synth_lib().tk_synth_uniform_fill(out.size, seed, lo, hi, out.ctypes.data)
    return out.reshape(shape)


def bench_scene(n_gaussians: int, width: int, height: int, d: int, seed: int = 7, feature_seed: int = 7):
    """The reference bench recipe (fslam_main.cpp:167-196): SceneSpec{seed, spacing=sqrt(70/N)},
    truncated to N, camera fx=fy=0.9W, far 20, pose = orbit(8)[0]; features are seeded unit rows."""
    spec = default_spec(seed=seed, spacing=math.sqrt(70.0 / max(1, n_gaussians)), feature_dim=max(d, 4),
                        classes=4)
    scene, cls = build_synthetic_scene(spec, truncate=n_gaussians)
    scene.class_ids = cls  # for render_ground_truth (scene.cpp:232-276)
    scene.feature = None
    scene.feature_dim = d
    cam = CameraIntrinsics(fx=0.9 * width, fy=0.9 * width, cx=0.5 * (width - 1), cy=0.5 * (height - 1),
                           width=width, height=height, near_plane=0.05, far_plane=20.0)
    pose = generate_trajectory("orbit", 8, spec)[0]
    return scene, cam, pose, spec


def render_ground_truth(renderer, scene, class_ids: np.ndarray, embeddings: np.ndarray, poses, cam) -> list:
    """render_ground_truth (proj/src/synth/scene.cpp:232-276): a K = 1 render of the scene per pose
    (on the GPU, through `renderer`); colour clamped to [0, 1]; depth, label and the label's class
    embedding only where alpha > 0.5 and a Top-1 record exists (label 255 elsewhere).  Returns
    [(Frame, label image)]."""
    from paper_2602_06991_b200.types import Frame, RenderSettings
    s = RenderSettings(top_k=1, transmittance_floor=1e-4, background=(0.0, 0.0, 0.0))
    emb = np.ascontiguousarray(embeddings, np.float32)
    out = []
    for pose in poses:
        r = renderer.render_geometric(scene, pose, cam, s)
        h, w = cam.height, cam.width
        covered = (r.alpha > 0.5) & (r.topk.count.reshape(h, w) > 0)
        top = r.topk.index.reshape(h, w)
        label = np.full((h, w), 255, np.uint8)
        label[covered] = class_ids[top[covered]]
        feat = np.zeros((h, w, emb.shape[1]), np.float32)
        feat[covered] = emb[label[covered]]
        frame = Frame(color=np.clip(r.color, 0.0, 1.0).astype(np.float32),
                      depth=np.where(covered, r.depth, 0.0).astype(np.float32), feature=feat)
        out.append((frame, label))
    return out

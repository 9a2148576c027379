"""Host-side mirror of the reference renderer's value types (no Eigen, numpy arrays).

Field names and defaults follow the reference headers so code written against
proj/include/fslam/{core,raster,map} reads the same.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

K_MAX_TOP_K = 32                          # render.hpp:23
K_LOG_WEIGHT_CUTOFF = -27.631021115928547  # render.hpp:97


@dataclass
class CameraIntrinsics:  # core/types.hpp:15-21
    fx: float = 0.0
    fy: float = 0.0
    cx: float = 0.0
    cy: float = 0.0
    width: int = 0
    height: int = 0
    near_plane: float = 0.05
    far_plane: float = 100.0


@dataclass
class Pose:  # core/pose.hpp:11-19, world-to-camera; rotation quaternion (w, x, y, z)
    rotation: tuple = (1.0, 0.0, 0.0, 0.0)
    translation: tuple = (0.0, 0.0, 0.0)

    @staticmethod
    def identity() -> "Pose":
        return Pose()


@dataclass
class RenderSettings:  # raster/render.hpp:14-21
    top_k: int = 3
    transmittance_floor: float = 1e-4
    background: tuple = (0.0, 0.0, 0.0)
    tile_size: int = 16
    cov2d_dilation: float = 0.3
    alpha_clamp: float = 0.999


@dataclass
class SceneMap:  # map/scene_map.hpp:16-27 as SoA arrays; rotation (w,x,y,z); feature (n, d)
    mean: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    log_scale: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    rotation: np.ndarray = field(default_factory=lambda: np.zeros((0, 4)))
    opacity_logit: np.ndarray = field(default_factory=lambda: np.zeros(0))
    color: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    feature: np.ndarray | None = None
    generation: int = 0
    feature_dim: int = 0

    def size(self) -> int:
        return int(self.mean.shape[0])

    def __len__(self) -> int:
        return self.size()

    def copy(self) -> "SceneMap":
        return SceneMap(self.mean.copy(), self.log_scale.copy(), self.rotation.copy(), self.opacity_logit.copy(),
                        self.color.copy(), None if self.feature is None else self.feature.copy(), self.generation,
                        self.feature_dim)


@dataclass
class TopKGrid:  # raster/render.hpp:27-44; slot = (y*W + x)*k + j
    width: int = 0
    height: int = 0
    k: int = 0
    index: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    weight: np.ndarray = field(default_factory=lambda: np.zeros(0))
    count: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))

    @staticmethod
    def empty(w: int, h: int, k: int) -> "TopKGrid":
        return TopKGrid(w, h, k, np.full(w * h * k, -1, np.int32), np.zeros(w * h * k), np.zeros(w * h, np.uint8))

    def slot(self, x: int, y: int, j: int) -> int:
        return (y * self.width + x) * self.k + j

    def pixel(self, x: int, y: int) -> int:
        return y * self.width + x


@dataclass
class RenderOutput:  # raster/render.hpp:46-55; images are H x W x C
    color: np.ndarray | None = None
    depth: np.ndarray | None = None
    alpha: np.ndarray | None = None
    feature: np.ndarray | None = None
    topk: TopKGrid | None = None
    contributions: np.ndarray | None = None
    generation: int = 0
    map_size: int = 0


@dataclass
class GeomGrads:  # raster/backward.hpp:15-22
    mean: np.ndarray
    log_scale: np.ndarray
    rotation: np.ndarray
    opacity_logit: np.ndarray
    color: np.ndarray
    pose_twist: np.ndarray


@dataclass
class PreparedScene:  # raster/render.hpp:84-92 (entries as n x 7: mx,my,ixx,ixy,iyy,z,opacity)
    entries: np.ndarray
    src: np.ndarray
    tile_offsets: np.ndarray
    tile_entries: np.ndarray
    tiles_x: int
    tiles_y: int
    width: int
    height: int
    generation: int
    map_size: int


@dataclass
class Frame:  # map/scene_map.hpp Keyframe::frame: color H x W x 3, depth H x W, feature H x W x d (fp32)
    color: np.ndarray
    depth: np.ndarray
    feature: np.ndarray | None = None


@dataclass
class MapperConfig:
    """The mapping-iteration knobs of MapperConfig (map/mapper.hpp:23-35) flattened: LossWeights
    (losses.hpp:9-21), GroupLearningRates and AdamParams (optimizer.hpp:9-23),
    Schedule::feature_update_period (mapper.hpp:16) and the log-scale clamps (mapper.hpp:31-32)."""
    lambda_geo: float = 1.0
    lambda_feat: float = 1.0
    lambda1: float = 0.2
    lambda2: float = 1.0
    color_secondary: int = 0  # 0 = D-SSIM (kDssim), 1 = duplicated L1 (kL1Duplicate)
    feature_update_period: int = 5
    l1_deadband: float = 0.0
    lr_mean: float = 2e-3
    lr_log_scale: float = 5e-3
    lr_rotation: float = 1e-3
    lr_opacity: float = 5e-2
    lr_color: float = 2e-2
    lr_feature: float = 1e-2
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    min_log_scale: float = -10.0
    max_log_scale: float = 1.0
    # host-side schedule of optimize_step / insert_gaussians (mapper.hpp:14-35)
    prune_period: int = 500
    prune_keep_ratio: float = 0.5
    topk_count_threshold: int = 0
    pruning: bool = True
    tau_insert: float = 0.05


@dataclass
class LossValues:  # map/losses.hpp:23-27
    map: float = 0.0
    geo: float = 0.0
    feat: float = 0.0

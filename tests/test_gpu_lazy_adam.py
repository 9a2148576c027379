"""Lazy feature Adam (tk_optimize_step updates only the rows a frame's records reach; the other rows'
zero-gradient steps are replayed by k_feature_catchup before anything reads them) against the
eager step (TK_LAZY_ADAM=0, read once per process, hence the subprocesses): a mapping run over three
keyframes with different visible sets, a feature render of the resident map in the middle, a prune
and a final download must be bit-identical (geometry frozen: its backward sums with atomics)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import ctypes as C, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
sys.path.insert(0, sys.argv[1] + "/tests")
from _se3 import axis_angle
from paper_2602_06991_b200 import _native as N, api
import scenegen as synth
from paper_2602_06991_b200.api import to_camera, to_pose, to_settings
from paper_2602_06991_b200.types import Frame, MapperConfig, Pose, RenderSettings

D = int(sys.argv[3])
m = synth.random_scene(3000, D, 4)
truth = m.copy()
rng = np.random.default_rng(5)
truth.mean = truth.mean + rng.normal(0, 0.03, truth.mean.shape)
cam = synth.test_camera(96, 72)
s = RenderSettings()
poses = [Pose(), Pose(axis_angle(0.25, (0, 1, 0)), (0.3, 0.0, 0.1)), Pose(axis_angle(-0.3, (1, 0.2, 0)), (-0.2, 0.1, 0.0))]
gr = api.Renderer(0)
frames = []
for i, p in enumerate(poses):
    g = gr.render_geometric(truth, p, cam, s)
    feat = rng.normal(0, 1, (72, 96, D)).astype(np.float32)
    feat[g.alpha < 0.3] = 0.0
    frames.append(Frame(color=g.color.astype(np.float32), depth=g.depth.astype(np.float32), feature=feat))
gr.close()
r = api.Renderer(0)
r.upload(m)
r.optimizer_reset(True)
for i, (p, fr) in enumerate(zip(poses, frames)):
    r.keyframe_set(i, p, fr)
# geometry learning rates 0: the geometry backward sums with atomics (not bit-reproducible run to
# run), so a frozen geometry keeps the records -- and with them the feature path -- comparable bitwise
cfg = MapperConfig(feature_update_period=int(sys.argv[4]), lr_feature=5e-2, lr_mean=0.0, lr_log_scale=0.0,
                   lr_rotation=0.0, lr_opacity=0.0, lr_color=0.0)
out = {}
for it in range(1, 16):
    r.optimize_step(cfg, cam, s, it % 3, it)
    if it == 7:  # a feature render of the resident (partly stale) map
        gout = N.tk_geom_out(N.TK_DEVICE, None, None, None, None, None, None, None, 0, 0)
        N.check(r.lib.tk_render_geometric(r.ctx, C.byref(to_pose(poses[1])), C.byref(to_camera(cam)),
                                          C.byref(to_settings(s)), C.byref(gout)))
        F = np.zeros((72, 96, D), np.float32)
        N.check(r.lib.tk_render_feature(r.ctx, None, F.ctypes.data, N.TK_HOST))
        out["F7"] = F
    if it == 10:
        out["removed"] = r.prune_map(0.6, 1234, 2)
    if it == 12:  # new Gaussians enter with fresh moments at the current feature step
        rs = np.random.default_rng(9)
        npts = 200
        pos = np.c_[rs.uniform(-1, 1, npts), rs.uniform(-0.7, 0.7, npts), rs.uniform(2, 5, npts)]
        out["inserted"] = np.array([r.insert_gaussians(pos, rs.uniform(0, 1, (npts, 3)),
                                                       rs.normal(0, 1, (npts, D)).astype(np.float32),
                                                       np.full(npts, 0.05), np.full(npts, 1.0), 0.05, Pose())])
n, d, _ = r.scene_info()
for k, v in r.scene_download(n, d).items():
    out[k] = v
r.close()
np.savez(sys.argv[2], **out)
"""


@pytest.mark.parametrize("d,period", [(32, 1), (64, 2), (512, 1)])
def test_lazy_feature_adam_bit_identical_to_eager(tmp_path, d, period):
    res = {}
    for lazy in ("1", "0"):
        path = tmp_path / f"run_{lazy}.npz"
        env = dict(os.environ, TK_LAZY_ADAM=lazy)
        subprocess.run([sys.executable, "-c", CHILD, ROOT, str(path), str(d), str(period)], check=True, env=env,
                       timeout=600)
        res[lazy] = np.load(path)
    a, b = res["1"], res["0"]
    assert sorted(a.files) == sorted(b.files)
    for k in a.files:
        assert np.array_equal(a[k], b[k]), k

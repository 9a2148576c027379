"""Context lifecycle: tk_destroy frees every device buffer a context allocated (frames, feature
path, mapping state, staged gathers), so repeated create / use / destroy leaves device memory where
it started."""
import numpy as np
import pytest
import torch

from paper_2602_06991_b200 import api
import scenegen as synth
from paper_2602_06991_b200.types import Frame, MapperConfig, Pose, RenderSettings

pytestmark = pytest.mark.gpu


def use_context(m, cam):
    r = api.Renderer(0)
    try:
        s = RenderSettings()
        g = r.render_geometric(m, Pose(), cam, s)
        F = r.render_feature(m, g.topk)
        r.backward_feature(m, g.topk, np.ones_like(F))
        r.backward_geometric(m, Pose(), cam, s, np.ones((cam.height, cam.width, 3)), np.ones((cam.height, cam.width)))
        r.upload(m)
        r.optimizer_reset(True)
        r.keyframe_set(0, Pose(), Frame(color=g.color.astype(np.float32), depth=g.depth.astype(np.float32), feature=F))
        r.optimize_step(MapperConfig(feature_update_period=1), cam, s, 0, 1)
        r.synchronize()
    finally:
        r.close()


def test_destroy_releases_device_memory():
    m = synth.random_scene(20000, 64, 3)
    cam = synth.test_camera(320, 240)
    use_context(m, cam)  # first use: module loads, allocator warm-up
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    for _ in range(8):
        use_context(m, cam)
    torch.cuda.synchronize()
    free1, _ = torch.cuda.mem_get_info()
    assert free0 - free1 < 64 << 20, f"{(free0 - free1) >> 20} MiB not returned"

"""Parity at BASELINE.json's configs 1 and 2 (100k Gaussians, 640 x 480, D = 512, the bench recipe
scene and orbit pose; config 2 sweeps K over 1/4/8/16, forward + backward): every entry point of the
path against the CPU oracle at full size, under the contract of test_gpu_parity.py."""
import numpy as np
import pytest

import _oracle as O
from paper_2602_06991_b200 import api
import scenegen as synth
from paper_2602_06991_b200.types import RenderSettings

pytestmark = pytest.mark.gpu

N_G, W, H, D = 100_000, 640, 480, 512


@pytest.fixture(scope="module")
def scene():
    m, cam, pose, _ = synth.bench_scene(N_G, W, H, D)
    m.feature = synth.unit_features(m.size(), D, 7)
    r = api.Renderer(0)
    yield r, m, cam, pose
    r.close()


@pytest.mark.parametrize("k", [3, 1, 4, 8, 16])
def test_c1_c2_forward_backward_match_oracle(scene, k):
    r, m, cam, pose = scene
    s = RenderSettings(top_k=k)
    g = r.render_geometric(m, pose, cam, s)
    o = O.render_geometric(m, pose, cam, s)
    assert (g.topk.count == o["count"]).all() and (g.topk.index == o["index"]).all()
    np.testing.assert_allclose(g.topk.weight, o["weight"], rtol=1e-9, atol=0)
    for f in ("color", "depth", "alpha"):
        np.testing.assert_allclose(getattr(g, f), o[f], rtol=0, atol=1e-9)
    F = r.render_feature(m, g.topk)
    fo = O.render_feature(m, W, H, k, g.topk.index, g.topk.weight, g.topk.count)
    assert (np.abs(F.astype(np.float64) - fo) <= 1e-5 * np.maximum(1.0, np.abs(fo))).all()
    G = synth.uniform_image((H, W, D), 11).astype(np.float32)
    df = r.backward_feature(m, g.topk, G)
    dfo = O.backward_feature(m, W, H, k, g.topk.index, g.topk.weight, g.topk.count, G.astype(np.float64))
    assert (np.abs(df.astype(np.float64) - dfo) <= 2e-5 * np.maximum(1.0, np.abs(dfo))).all()
    gc = synth.uniform_image((H, W, 3), 12)
    gd = synth.uniform_image((H, W), 13)
    gg = r.backward_geometric(m, pose, cam, s, gc, gd)
    go = O.backward_geometric(m, pose, cam, s, gc, gd)
    for f in ("mean", "log_scale", "rotation", "opacity_logit", "color"):
        a, b = getattr(gg, f), go[f]
        scale = max(1e-12, np.abs(b).max())
        np.testing.assert_array_less(np.abs(a - b), 1e-4 * np.maximum(np.abs(b), 1e-2 * scale) + 1e-12)


def test_c1_full_blend_matches_oracle(scene):
    """render_feature_full_blend (render.cpp:242-289, 339-343: every contributor, no
    renormalisation) at full config-1 size against the oracle."""
    r, m, cam, pose = scene
    s = RenderSettings()
    f = r.render_feature_full_blend(m, pose, cam, s)
    o = O.render_feature_full_blend(m, pose, cam, s)
    assert (np.abs(f.astype(np.float64) - o) <= 2e-5 * np.maximum(1.0, np.abs(o))).all()


def test_c1_backward_geometric_bit_deterministic(scene):
    r, m, cam, pose = scene
    s = RenderSettings(top_k=3)
    gc = synth.uniform_image((H, W, 3), 12)
    gd = synth.uniform_image((H, W), 13)
    a = r.backward_geometric(m, pose, cam, s, gc, gd)
    b = r.backward_geometric(m, pose, cam, s, gc, gd)
    for f in ("mean", "log_scale", "rotation", "opacity_logit", "color", "pose_twist"):
        assert getattr(a, f).tobytes() == getattr(b, f).tobytes(), f

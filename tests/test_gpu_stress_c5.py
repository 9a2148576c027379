"""Parity at BASELINE.json's config 5 (the stress render: 4M Gaussians, 1920 x 1080, D = 768, K = 3,
the bench recipe scene and orbit pose), forward and backward: the GPU prepare_scene, geometric pass,
feature gather, feature backward (element-wise, 64-channel oracle slices) and geometry backward
against the CPU oracle, with the contract of test_gpu_parity.py (records and tile lists exact)."""
import numpy as np
import pytest

import _oracle as O
from paper_2602_06991_b200 import api
import scenegen as synth
from paper_2602_06991_b200.types import RenderSettings

pytestmark = pytest.mark.gpu

N_G, W, H, D, K = 4_000_000, 1920, 1080, 768, 3


@pytest.fixture(scope="module")
def c5():
    m, cam, pose, _ = synth.bench_scene(N_G, W, H, D)
    m.feature = synth.unit_features(m.size(), D, 7)
    r = api.Renderer(0)
    yield r, m, cam, pose
    r.close()


def test_c5_geometric_prepare_and_gather_match_oracle(c5):
    r, m, cam, pose = c5
    s = RenderSettings(top_k=K)
    g = r.render_geometric(m, pose, cam, s)
    o = O.render_geometric(m, pose, cam, s)
    assert (g.topk.count == o["count"]).all() and (g.topk.index == o["index"]).all()
    np.testing.assert_allclose(g.topk.weight, o["weight"], rtol=1e-9, atol=0)
    for f in ("color", "depth", "alpha"):
        np.testing.assert_allclose(getattr(g, f), o[f], rtol=0, atol=1e-9)
    np.testing.assert_allclose(g.contributions, o["contributions"], rtol=1e-9, atol=0)
    del o
    p = r.prepare_scene(m, pose, cam, s)
    po = O.prepare_scene(m, pose, cam, s)
    assert (p.src == po["src"]).all() and (p.tile_offsets == po["tile_offsets"]).all()
    assert (p.tile_entries == po["tile_entries"]).all()
    del p, po
    F = r.render_feature(m, g.topk)
    fo = O.render_feature(m, W, H, K, g.topk.index, g.topk.weight, g.topk.count)
    assert (np.abs(F.astype(np.float64) - fo) <= 1e-5 * np.maximum(1.0, np.abs(fo))).all()


def test_c5_backward_feature_matches_oracle(c5):
    r, m, cam, pose = c5
    g = r.render_geometric(m, pose, cam, RenderSettings(top_k=K))
    G = synth.uniform_image((H, W, D), 11).astype(np.float32)
    df = r.backward_feature(m, g.topk, G).reshape(m.size(), D)
    for c0, c1, o in O.backward_feature_slices(m, W, H, K, g.topk.index, g.topk.weight, g.topk.count, G):
        a = df[:, c0:c1].astype(np.float64)
        bad = np.abs(a - o) > 2e-5 * np.maximum(1.0, np.abs(o))
        assert not bad.any(), (c0, c1, int(bad.sum()))
        assert np.array_equal((a == 0).all(axis=1), (o == 0).all(axis=1)), (c0, c1)


def test_c5_backward_geometric_matches_oracle_and_is_deterministic(c5):
    r, m, cam, pose = c5
    s = RenderSettings(top_k=K)
    gc = synth.uniform_image((H, W, 3), 12)
    gd = synth.uniform_image((H, W), 13)
    g = r.backward_geometric(m, pose, cam, s, gc, gd)
    o = O.backward_geometric(m, pose, cam, s, gc, gd)
    for f in ("mean", "log_scale", "rotation", "opacity_logit", "color"):
        a, b = getattr(g, f), o[f]
        scale = max(1e-12, np.abs(b).max())
        np.testing.assert_array_less(np.abs(a - b), 1e-4 * np.maximum(np.abs(b), 1e-2 * scale) + 1e-12)
        za, zb = (a.reshape(len(a), -1) == 0).all(axis=1), (b.reshape(len(b), -1) == 0).all(axis=1)
        assert (za == zb).all(), f
    scale = max(1e-12, np.abs(o["pose_twist"]).max())
    np.testing.assert_array_less(np.abs(g.pose_twist - o["pose_twist"]),
                                 1e-4 * np.maximum(np.abs(o["pose_twist"]), 1e-2 * scale) + 1e-12)
    del o
    again = r.backward_geometric(m, pose, cam, s, gc, gd)
    for f in ("mean", "log_scale", "rotation", "opacity_logit", "color", "pose_twist"):
        assert getattr(g, f).tobytes() == getattr(again, f).tobytes(), f

"""render_ground_truth (scene.cpp:232-276) through the GPU renderer against the same assembly over
the oracle's K = 1 render: labels, features and depth exactly equal, colour within fp32 rounding."""
import numpy as np
import pytest

import _oracle as O
from paper_2602_06991_b200 import api
import scenegen as synth
from paper_2602_06991_b200.types import RenderSettings

pytestmark = pytest.mark.gpu


def test_render_ground_truth_matches_oracle_assembly():
    scene, cam, pose, spec = synth.bench_scene(20000, 160, 120, 16)
    emb = synth.unit_features(4, 16, 99)
    r = api.Renderer(0)
    try:
        (frame, label), = synth.render_ground_truth(r, scene, scene.class_ids, emb, [pose], cam)
    finally:
        r.close()
    o = O.render_geometric(scene, pose, cam, RenderSettings(top_k=1, transmittance_floor=1e-4))
    covered = (o["alpha"] > 0.5) & (o["count"].reshape(120, 160) > 0)
    want_label = np.full((120, 160), 255, np.uint8)
    want_label[covered] = scene.class_ids[o["index"].reshape(120, 160)[covered]]
    assert covered.mean() > 0.2
    assert (label == want_label).all()
    want_feat = np.zeros((120, 160, 16), np.float32)
    want_feat[covered] = emb[want_label[covered]]
    assert (frame.feature == want_feat).all()
    np.testing.assert_allclose(frame.depth, np.where(covered, o["depth"], 0.0).astype(np.float32), rtol=1e-6, atol=0)
    np.testing.assert_allclose(frame.color, np.clip(o["color"], 0, 1).astype(np.float32), rtol=0, atol=1e-6)

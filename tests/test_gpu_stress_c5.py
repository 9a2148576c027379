"""Parity at BASELINE.json's config 5 (the stress render: 4M Gaussians, 1920 x 1080, D = 768, K = 3,
the bench recipe scene and orbit pose): the GPU prepare_scene, geometric pass and feature gather
against the CPU oracle, with the contract of test_gpu_parity.py (records and tile lists exact)."""
import numpy as np
import pytest

import _oracle as O
from paper_2602_06991_b200 import api, synth
from paper_2602_06991_b200.types import RenderSettings

pytestmark = pytest.mark.gpu

N_G, W, H, D, K = 4_000_000, 1920, 1080, 768, 3


def test_c5_geometric_prepare_and_gather_match_oracle():
    m, cam, pose, _ = synth.bench_scene(N_G, W, H, D)
    m.feature = synth.unit_features(m.size(), D, 7)
    r = api.Renderer(0)
    try:
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
    finally:
        r.close()

"""FEAT feature frames into device keyframes (tk_keyframe_load_features / _save_features): loading
the file gives the same mapping step as passing the image to tk_keyframe_set; saving writes the
reference's bytes; errors carry the reference's messages."""
import numpy as np
import pytest

from paper_2602_06991_b200 import _native as N
from paper_2602_06991_b200 import api, dataset
import scenegen as synth
from paper_2602_06991_b200.types import Frame, MapperConfig, Pose, RenderSettings

pytestmark = pytest.mark.gpu


def test_feat_file_keyframe_equals_in_memory(tmp_path):
    m = synth.random_scene(800, 16, 2)
    cam = synth.test_camera(64, 48)
    s = RenderSettings()
    gr = api.Renderer(0)
    g = gr.render_geometric(m, Pose(), cam, s)
    gr.close()
    feat = np.random.default_rng(1).normal(size=(48, 64, 16)).astype(np.float32)
    feat[g.alpha < 0.3] = 0.0
    frame = Frame(color=g.color.astype(np.float32), depth=g.depth.astype(np.float32), feature=feat)
    path = tmp_path / "000003.feat"
    dataset.write_feature_bin(str(path), feat)
    cfg = MapperConfig(feature_update_period=1)
    results = []
    for via_file in (False, True):
        r = api.Renderer(0)
        try:
            mm = m.copy()
            mm.mean = mm.mean + 0.01
            r.upload(mm)
            r.optimizer_reset(True)
            if via_file:  # the keyframe's colour/depth first, then the features from the FEAT file
                r.keyframe_set(0, Pose(), Frame(color=frame.color, depth=frame.depth,
                                                feature=np.zeros_like(feat)))
                r.keyframe_load_features(0, str(path))
                out = tmp_path / "saved.feat"
                r.keyframe_save_features(0, str(out))
                assert out.read_bytes() == path.read_bytes()
            else:
                r.keyframe_set(0, Pose(), frame)
            v, _ = r.optimize_step(cfg, cam, s, 0, 1)
            results.append((v, r.scene_download(mm.size(), 16)["feature"]))
        finally:
            r.close()
    (va, fa), (vb, fb) = results
    assert va.feat == vb.feat and va.geo == vb.geo and np.array_equal(fa, fb)


def test_feat_file_errors(tmp_path):
    r = api.Renderer(0)
    try:
        z = np.zeros((8, 8, 3), np.float32)
        r.keyframe_set(0, Pose(), Frame(color=z, depth=z[..., 0].copy(), feature=np.zeros((8, 8, 4), np.float32)))
        assert r.lib.tk_keyframe_load_features(r.ctx, 0, str(tmp_path / "none.feat").encode()) == N.TK_ERR_BAD_ARG
        assert b"dataset: cannot open" in r.lib.tk_last_error()
        bad = tmp_path / "bad.feat"
        bad.write_bytes(b"NOPE" + bytes(12))
        assert r.lib.tk_keyframe_load_features(r.ctx, 0, str(bad).encode()) == N.TK_ERR_BAD_ARG
        assert b"dataset: bad magic in" in r.lib.tk_last_error()
        wrong = tmp_path / "wrong.feat"
        dataset.write_feature_bin(str(wrong), np.zeros((4, 8, 4), np.float32))
        assert r.lib.tk_keyframe_load_features(r.ctx, 0, str(wrong).encode()) == N.TK_ERR_BAD_ARG
        assert r.lib.tk_keyframe_load_features(r.ctx, 3, str(wrong).encode()) == N.TK_ERR_BAD_ARG
        trunc = tmp_path / "trunc.feat"
        trunc.write_bytes(wrong.read_bytes()[:40])
        dataset.write_feature_bin(str(wrong), np.zeros((8, 8, 4), np.float32))
        trunc.write_bytes(wrong.read_bytes()[:40])
        assert r.lib.tk_keyframe_load_features(r.ctx, 0, str(trunc).encode()) == N.TK_ERR_BAD_ARG
        assert b"dataset: truncated data in" in r.lib.tk_last_error()
    finally:
        r.close()

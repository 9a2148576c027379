"""GPU parity of the SPLF checkpoint path (tk_checkpoint_save / _load, checkpoint.cpp:39-98) and of
segment_by_query (tk_segment_by_query, metrics.cpp:66-94) against the oracle.

Contract: checkpoint files byte-identical to the oracle's save of the same map; a device load
exports exactly the oracle's load (fp32 -> fp64 is exact); labels exactly equal to the oracle on
the same fp32 feature image (fp64 dots in channel order on both sides).
"""
import numpy as np
import pytest

import _oracle as O
from paper_2602_06991_b200 import api
import scenegen as synth
from paper_2602_06991_b200.types import Pose, RenderSettings

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def R():
    r = api.Renderer(0)
    yield r
    r.close()


@pytest.mark.parametrize("n,d", [(25, 8), (3000, 64), (10, 0)])
def test_checkpoint_save_matches_oracle_bytes(R, tmp_path, n, d):
    m = synth.random_scene(n, max(d, 1), 5)
    m.feature = np.zeros((n, 0)) if d == 0 else m.feature.astype(np.float32).astype(np.float64)
    m.feature_dim = d
    R.upload(m)
    pg, po = str(tmp_path / "gpu.bin"), str(tmp_path / "oracle.bin")
    R.checkpoint_save(pg)
    O.checkpoint_save(m, po)
    assert open(pg, "rb").read() == open(po, "rb").read()


def test_checkpoint_load_round_trip(R, tmp_path):
    m = synth.random_scene(500, 16, 8)
    p1, p2 = str(tmp_path / "a.bin"), str(tmp_path / "b.bin")
    O.checkpoint_save(m, p1)
    assert R.checkpoint_load(p1) == (500, 16)
    assert R.scene_info()[2] == 0
    o = O.checkpoint_load(p1)
    out = R.scene_download(500, 16, stats=False)
    for key in ("mean", "log_scale", "rotation", "opacity_logit", "color"):
        assert (out[key] == o[key]).all(), key
    assert (out["feature"].astype(np.float64) == o["feature"]).all()
    R.checkpoint_save(p2)
    assert open(p1, "rb").read() == open(p2, "rb").read()


def test_checkpoint_errors_carry_reference_messages(R, tmp_path):
    with pytest.raises(RuntimeError, match="checkpoint: cannot open"):
        R.checkpoint_load(str(tmp_path / "missing.bin"))
    m = synth.random_scene(20, 4, 1)
    p = str(tmp_path / "a.bin")
    O.checkpoint_save(m, p)
    raw = open(p, "rb").read()
    short = str(tmp_path / "short.bin")
    open(short, "wb").write(raw[:40])
    with pytest.raises(RuntimeError, match="checkpoint: truncated file .*short.bin"):
        R.checkpoint_load(short)
    bad = str(tmp_path / "bad.bin")
    open(bad, "wb").write(b"XXXX" + raw[4:])
    with pytest.raises(RuntimeError, match="checkpoint: bad magic"):
        R.checkpoint_load(bad)
    ver = str(tmp_path / "ver.bin")
    open(ver, "wb").write(raw[:4] + (7).to_bytes(4, "little") + raw[8:])
    with pytest.raises(RuntimeError, match="checkpoint: unsupported version 7"):
        R.checkpoint_load(ver)


@pytest.mark.parametrize("h,w,d,classes", [(40, 50, 16, 4), (33, 47, 512, 20), (16, 20, 96, 70), (24, 24, 600, 40)])
def test_segment_by_query_matches_oracle(R, h, w, d, classes):
    rng = np.random.default_rng(d + classes)
    feat = rng.normal(size=(h, w, d)).astype(np.float32)
    feat[rng.uniform(size=(h, w)) < 0.1] = 0.0          # invalid pixels
    feat[0, 0] = 1e-8                                     # norm2 below 1e-12 -> invalid
    emb = rng.normal(size=(classes, d))
    emb[1] = emb[0]                                       # tie: the first maximum wins
    got = R.segment_by_query(feat, emb)
    want = O.segment_by_query(feat.astype(np.float64), emb)
    assert (got == want).all()
    assert got[0, 0] == 255


def test_segment_by_query_on_rendered_features(R):
    m = synth.random_scene(400, 32, 3)
    cam = synth.test_camera(64, 48)
    out = R.render_geometric(m, Pose(), cam, RenderSettings())
    F = R.render_feature(m, out.topk)
    emb = np.random.default_rng(1).normal(size=(12, 32))
    got = R.segment_by_query(None, emb, shape=(48, 64))  # the context's resident F
    want = O.segment_by_query(F.astype(np.float64), emb)
    assert (got == want).all()

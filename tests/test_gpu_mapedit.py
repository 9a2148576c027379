"""GPU parity of the structural map edits (tk_insert_gaussians, tk_prune_map) against the oracle's
insert_gaussians / prune_map (mapper.cpp:19-60, 80-160), including the optimiser state moving in
lockstep (checked through the optimisation steps that follow, which read every moment).

Contract: removed indices, sizes, generations and topk_count exactly equal; inserted means / scales
/ rotations abs <= 1e-12; features abs <= 1e-6 (fp32 storage); after edits the next optimize_step
matches as in test_gpu_mapping.py.
"""
import numpy as np
import pytest

import _oracle as O
from _se3 import axis_angle
from paper_2602_06991_b200 import api
import scenegen as synth
from paper_2602_06991_b200.types import Frame, MapperConfig, Pose, RenderSettings, SceneMap

pytestmark = pytest.mark.gpu
INF = float("inf")


@pytest.fixture(scope="module")
def R():
    r = api.Renderer(0)
    yield r
    r.close()


def empty_map(d):
    return SceneMap(mean=np.zeros((0, 3)), log_scale=np.zeros((0, 3)), rotation=np.zeros((0, 4)),
                    opacity_logit=np.zeros(0), color=np.zeros((0, 3)), feature=np.zeros((0, d)), feature_dim=d)


def sources(n, d, seed, z0=1.5):
    rng = np.random.default_rng(seed)
    pos = np.c_[rng.uniform(-0.6, 0.6, (n, 2)), rng.uniform(z0, z0 + 1.5, n)]
    col = rng.uniform(0, 1, (n, 3))
    feat = rng.normal(size=(n, d)).astype(np.float32)
    feat[:3] = 0.0  # zero rows take the constant 1/sqrt(d) feature (mapper.cpp:46-48)
    sp = rng.uniform(0.01, 0.08, n)
    dist = np.where(rng.uniform(size=n) < 0.3, 0.01, INF)
    return pos, col, feat, sp, dist


def compare_maps(R, om, feat_tol=1e-6, geo_tol=1e-12):
    n, d, gen = R.scene_info()
    assert n == om.size() and gen == om.generation()
    o = om.export()
    g = R.scene_download(n, d)
    for key in ("mean", "log_scale", "rotation", "opacity_logit", "color"):
        np.testing.assert_allclose(g[key], o[key], rtol=0, atol=geo_tol, err_msg=key)
    np.testing.assert_allclose(g["feature"], o["feature"], rtol=0, atol=feat_tol, err_msg="feature")
    assert (g["topk_count"] == o["topk_count"]).all()
    np.testing.assert_allclose(g["max_contribution"], o["max_contribution"], rtol=1e-9, atol=0)


@pytest.mark.parametrize("pose", [Pose(), Pose(axis_angle(0.3, (0.2, 1.0, 0.1)), (0.2, -0.1, 0.4))],
                         ids=["identity", "posed"])
def test_insert_matches_oracle(R, pose):
    d = 8
    pos, col, feat, sp, dist = sources(200, d, 3)
    om = O.OracleMapper(empty_map(0), MapperConfig())
    R.upload(empty_map(0))
    R.optimizer_reset(True)
    k_o = om.insert(pos, col, feat.astype(np.float64), sp, dist, 0.05, pose)
    k_g = R.insert_gaussians(pos, col, feat, sp, dist, 0.05, pose)
    assert k_g == k_o > 0
    compare_maps(R, om)
    # a second batch without features: constant features (feature size != map dim)
    pos2, col2, _, sp2, dist2 = sources(50, d, 4)
    assert R.insert_gaussians(pos2, col2, None, sp2, dist2, 0.05, pose) == \
        om.insert(pos2, col2, None, sp2, dist2, 0.05, pose)
    compare_maps(R, om)


def keyframe_for(m, cam, pose, seed):
    rng = np.random.default_rng(seed)
    truth = m.copy()
    truth.mean = truth.mean + rng.normal(0, 0.02, truth.mean.shape)
    gt = O.render_geometric(truth, pose, cam, RenderSettings())
    feat = rng.normal(0, 1, (cam.height, cam.width, m.feature_dim)).astype(np.float32)
    feat[gt["alpha"] < 0.3] = 0.0
    return Frame(color=gt["color"].astype(np.float32), depth=gt["depth"].astype(np.float32), feature=feat)


@pytest.mark.parametrize("keep,thr", [(0.5, 0), (0.3, 2), (0.9, 1)])
def test_prune_after_steps_matches_oracle(R, keep, thr):
    m = synth.random_scene(400, 8, 21)
    cam = synth.test_camera(64, 48)
    s = RenderSettings()
    cfg = MapperConfig(feature_update_period=2)
    frame = keyframe_for(m, cam, Pose(), 5)
    om = O.OracleMapper(m, cfg)
    R.upload(m)
    R.optimizer_reset(True)
    R.keyframe_set(0, Pose(), frame)
    for it in (1, 2, 3):
        om.step(Pose(), cam, s, frame.color, frame.depth, frame.feature, it)
        R.optimize_step(cfg, cam, s, 0, it)
    rem_o = om.prune(keep, 1234 + thr, thr)
    rem_g = R.prune_map(keep, 1234 + thr, thr)
    assert rem_o.size > 0 and (rem_g == rem_o).all()
    compare_maps(R, om, feat_tol=2e-5, geo_tol=1e-10)
    # the moments moved with their Gaussians: the next steps (which read every moment) still match
    for it in (4, 5):
        ov, _ = om.step(Pose(), cam, s, frame.color, frame.depth, frame.feature, it)
        gv, _ = R.optimize_step(cfg, cam, s, 0, it)
        assert gv.geo == pytest.approx(ov["geo"], rel=1e-10)
    compare_maps(R, om, feat_tol=2e-5, geo_tol=1e-10)


def test_prune_without_candidates_resets_statistics(R):
    m = synth.random_scene(100, 4, 2)
    cam = synth.test_camera(32, 24)
    cfg = MapperConfig()
    R.upload(m)
    R.optimizer_reset(True)
    R.keyframe_set(0, Pose(), keyframe_for(m, cam, Pose(), 1))
    R.optimize_step(cfg, cam, RenderSettings(), 0, 1)
    removed = R.prune_map(0.5, 7, -1)  # threshold -1: no candidates
    assert removed.size == 0
    g = R.scene_download(100, 4)
    assert (g["topk_count"] == 0).all() and (g["max_contribution"] == 0).all()
    assert R.scene_info()[2] == m.generation


def test_mapper_loop_with_insert_and_prune_matches_oracle(R):
    """A short SLAM-style mapping run: insert, optimise with the reference's rng draws, prune on
    schedule (prune_period 3), insert again, optimise (mapper.cpp:162-265 with insertion)."""
    d = 6
    cam = synth.test_camera(48, 40)
    s = RenderSettings()
    cfg = MapperConfig(feature_update_period=2, prune_period=3, prune_keep_ratio=0.5, topk_count_threshold=1)
    pos, col, feat, sp, dist = sources(300, d, 7)
    seed_map = synth.random_scene(300, d, 9)
    frame = keyframe_for(seed_map, cam, Pose(), 2)
    om = O.OracleMapper(empty_map(0), cfg)
    mp = api.Mapper(R, empty_map(0), cfg, cam, s)
    assert mp.insert(pos, col, feat, sp, dist, Pose()) == om.insert(pos, col, feat.astype(np.float64), sp, dist,
                                                                    cfg.tau_insert, Pose())
    mp.add_keyframe(Pose(), frame)
    rng_g, rng_o = api.MT19937_64(42), api.MT19937_64(42)
    for it in range(1, 8):
        rec = mp.optimize_step(it, rng_g)
        rng_o()  # keyframe draw (one keyframe)
        ov, _ = om.step(Pose(), cam, s, frame.color, frame.depth, frame.feature, it)
        assert rec["losses"].geo == pytest.approx(ov["geo"], rel=1e-10)
        if it % cfg.prune_period == 0:
            removed = om.prune(cfg.prune_keep_ratio, rng_o(), cfg.topk_count_threshold)
            assert rec["pruned"] == removed.size
        if it == 4:
            p2, c2, f2, s2, d2 = sources(60, d, 11)
            assert mp.insert(p2, c2, f2, s2, d2, Pose()) == om.insert(p2, c2, f2.astype(np.float64), s2, d2,
                                                                      cfg.tau_insert, Pose())
    compare_maps(R, om, feat_tol=3e-5, geo_tol=1e-10)

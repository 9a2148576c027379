"""Pin the mapping-iteration oracle (oracle/src/oracle_mapping.inc) to the reference's own tests.

Restates, at the reference's tolerances, proj/tests/test_core.cpp:187-240 (SSIM), and
proj/tests/test_mapper.cpp:124-158 (contribution statistics), :270-311 (loss mix) and
:313-415 (the single-Gaussian optimize_step problem: schedule, period one, fit).  CPU only.
"""
import math

import numpy as np
import pytest

import _oracle as O
import scenegen as synth
from paper_2602_06991_b200.types import MapperConfig, Pose, RenderSettings, SceneMap


def logit(p):
    return math.log(p / (1.0 - p))


def ssim_value(a, b):
    return O.ssim_with_grad(a, b)[0]


def test_ssim_basics_and_fd_gradient():  # test_core.cpp:187-240
    rng = np.random.default_rng(9)
    a = rng.uniform(0, 1, (16, 16, 1))
    b = rng.uniform(0, 1, (16, 16, 1))
    assert ssim_value(a, a) == pytest.approx(1.0, rel=1e-12)
    assert ssim_value(a, 1.0 - a) < 0.0
    base, grad = O.ssim_with_grad(a, b)
    direction = rng.uniform(-1, 1, a.shape)
    analytic = float((grad * direction).sum())
    h = 1e-6
    fd = (ssim_value(a + h * direction, b) - ssim_value(a - h * direction, b)) / (2 * h)
    assert abs(analytic - fd) / max(abs(fd), 1e-9) < 1e-6
    for idx in (8 * 16 + 8, 5 * 16 + 9):
        y, x = divmod(idx, 16)
        hp = 1e-5
        ap, am = a.copy(), a.copy()
        ap[y, x, 0] += hp
        am[y, x, 0] -= hp
        fd1 = (ssim_value(ap, b) - ssim_value(am, b)) / (2 * hp)
        assert abs(grad[y, x, 0] - fd1) / max(abs(fd1), 1e-3) < 1e-4


def test_ssim_multichannel_mean_over_channels():  # ssim.cpp:90-108: mean over every channel's windows
    rng = np.random.default_rng(3)
    a = rng.uniform(0, 1, (14, 17, 3))
    b = rng.uniform(0, 1, (14, 17, 3))
    per = [ssim_value(a[..., c:c + 1], b[..., c:c + 1]) for c in range(3)]
    assert ssim_value(a, b) == pytest.approx(np.mean(per), rel=1e-12)


def stats_map(n, d=2):  # test_mapper.cpp:67-80
    return SceneMap(mean=np.array([[i, 0, 1] for i in range(n)], float), log_scale=np.zeros((n, 3)),
                    rotation=np.tile([1.0, 0, 0, 0], (n, 1)), opacity_logit=np.zeros(n), color=np.zeros((n, 3)),
                    feature=np.eye(n, d), feature_dim=d)


def test_contribution_statistics_accumulate():  # test_mapper.cpp:124-158
    m = stats_map(3)
    om = O.OracleMapper(m, MapperConfig())
    w, h, k = 4, 3, 2
    index = np.zeros(w * h * k, np.int32)
    count = np.ones(w * h, np.uint8)
    count[0] = 2
    index[1] = 1
    om.update_contribution_stats(0, 3, w, h, k, index, count, np.array([0.4, 0.25, 0.0]))
    e = om.export()
    assert list(e["topk_count"]) == [12, 1, 0]
    assert e["max_contribution"][0] == 0.4 and e["max_contribution"][2] == 0.0
    om.update_contribution_stats(0, 3, w, h, k, index, count, np.array([0.7, 0.1, 0.0]))
    e = om.export()
    assert e["topk_count"][0] == 24
    assert e["max_contribution"][0] == 0.7 and e["max_contribution"][1] == 0.25
    with pytest.raises(RuntimeError, match="does not match map generation"):
        om.update_contribution_stats(99, 3, w, h, k, index, count, np.zeros(3))


@pytest.fixture(scope="module")
def loss_setup():  # test_mapper.cpp:270-281
    cam = synth.test_camera(16, 16)
    m = synth.random_scene(5, 4, 3)
    r = O.render_geometric(m, Pose(), cam, RenderSettings())
    gt_color = r["color"].astype(np.float32)
    gt_depth = r["depth"].astype(np.float32)
    gt_feature = np.zeros((16, 16, 4), np.float32)
    return r, gt_color, gt_depth, gt_feature


def test_identical_render_gives_zero_loss(loss_setup):
    r, gc, gd, gf = loss_setup
    v, *_ = O.compute_losses(r["color"], r["depth"], r["count"], None, gc, gd, gf, MapperConfig(), False)
    assert v["geo"] < 1e-7 and v["map"] < 1e-7


def test_uniform_color_offset_plain_l1(loss_setup):
    r, gc, gd, gf = loss_setup
    cfg = MapperConfig(lambda1=0.0, lambda2=0.0, lambda_feat=0.0)
    v, *_ = O.compute_losses(r["color"] + 0.1, r["depth"], r["count"], None, gc, gd, gf, cfg, False)
    assert v["map"] == pytest.approx(0.1, rel=1e-6)


def test_invalid_depth_pixels_carry_no_depth_loss(loss_setup):
    r, gc, gd, gf = loss_setup
    v, _, g_depth, _ = O.compute_losses(r["color"], r["depth"] + 123.0, r["count"], None, gc, np.zeros_like(gd), gf,
                                        MapperConfig(lambda1=0.0), False)
    assert v["geo"] < 1e-7 and (g_depth == 0).all()


def test_feature_term_masks_uncovered_and_invalid_pixels():  # losses.cpp:88-118
    rng = np.random.default_rng(5)
    h, w, d = 12, 13, 3
    feat = rng.normal(size=(h, w, d))
    gt = rng.normal(size=(h, w, d)).astype(np.float32)
    gt[:3] = 0.0
    count = rng.integers(0, 3, (h, w)).astype(np.uint8)
    cfg = MapperConfig(lambda_feat=0.7)
    v, _, _, gf = O.compute_losses(np.zeros((h, w, 3)), np.zeros((h, w)), count, feat, np.zeros((h, w, 3), np.float32),
                                   np.zeros((h, w), np.float32), gt, cfg, True)
    mask = (count > 0) & (np.abs(gt).sum(-1) > 0)
    diff = feat - gt.astype(np.float64)
    assert v["feat"] == pytest.approx(np.abs(diff[mask]).sum() / (mask.sum() * d), rel=1e-12)
    assert v["map"] == pytest.approx(1.0 * v["geo"] + 0.7 * v["feat"], rel=1e-12)
    assert (gf[~mask] == 0).all()
    assert np.allclose(gf[mask], 0.7 * np.sign(diff[mask]) / (mask.sum() * d), rtol=0, atol=0)


def single_gaussian_problem():  # test_mapper.cpp:313-357
    cam = synth.test_camera(24, 24)
    s = RenderSettings(transmittance_floor=0.0)
    truth = SceneMap(mean=np.array([[0.05, -0.03, 1.5]]), log_scale=np.full((1, 3), math.log(0.12)),
                     rotation=np.array([[1.0, 0, 0, 0]]), opacity_logit=np.array([logit(0.8)]),
                     color=np.array([[0.8, 0.3, 0.2]]), feature=np.array([[1.0, 0.0]]), feature_dim=2)
    gt = O.render_geometric(truth, Pose(), cam, s)
    gt_color = gt["color"].astype(np.float32)
    gt_depth = gt["depth"].astype(np.float32)
    gt_feature = np.zeros((24, 24, 2), np.float32)
    gt_feature[gt["alpha"] > 0.3, 0] = 1.0
    start = SceneMap(mean=truth.mean + [0.06, -0.04, 0.08], log_scale=truth.log_scale.copy(),
                     rotation=truth.rotation.copy(), opacity_logit=np.array([logit(0.5)]),
                     color=np.array([[0.5, 0.5, 0.5]]), feature=np.array([[0.0, 1.0]]), feature_dim=2)
    return start, cam, s, gt_color, gt_depth, gt_feature


def test_hybrid_schedule_touches_features_only_on_period():  # test_mapper.cpp:360-376
    start, cam, s, gc, gd, gf = single_gaussian_problem()
    om = O.OracleMapper(start, MapperConfig(feature_update_period=5))
    for it in range(1, 13):
        before = om.export()["feature"].copy()
        v, fstep = om.step(Pose(), cam, s, gc, gd, gf, it)
        changed = np.linalg.norm(om.export()["feature"] - before) > 0
        assert fstep == (it % 5 == 0) and changed == fstep
        if not fstep:
            assert v["feat"] == 0.0


def test_every_step_carries_feature_term_with_period_one():  # test_mapper.cpp:378-391
    start, cam, s, gc, gd, gf = single_gaussian_problem()
    om = O.OracleMapper(start, MapperConfig(feature_update_period=1))
    for it in range(1, 6):
        v, fstep = om.step(Pose(), cam, s, gc, gd, gf, it)
        assert fstep and v["feat"] > 0.0


def test_single_gaussian_fits_its_keyframe():  # test_mapper.cpp:393-415
    start, cam, s, gc, gd, gf = single_gaussian_problem()
    om = O.OracleMapper(start, MapperConfig(feature_update_period=1))
    first = last = None
    for it in range(1, 201):
        v, _ = om.step(Pose(), cam, s, gc, gd, gf, it)
        first = v["geo"] if first is None else first
        last = v["geo"]
    assert last < first / 10.0
    e = om.export()
    assert e["feature"][0, 0] > 0.9
    assert abs(np.linalg.norm(e["feature"][0]) - 1.0) < 1e-6
    assert np.linalg.norm(e["rotation"][0]) == pytest.approx(1.0, rel=1e-9)
    assert e["color"].max() <= 1.0 and e["color"].min() >= 0.0


# ---- insertion and pruning (test_mapper.cpp:84-122, 160-268, 417-441)
INF = float("inf")


def simple_sources(n, d):  # test_mapper.cpp:17-27
    pos = np.array([[0.1 * i, 0.0, 1.0 + 0.1 * i] for i in range(n)])
    col = np.full((n, 3), 0.5)
    feat = np.zeros((n, d))
    feat[np.arange(n), np.arange(n) % d] = 1.0
    return pos, col, feat, np.full(n, 0.05)


def empty_mapper(d=0):
    m = SceneMap(mean=np.zeros((0, 3)), log_scale=np.zeros((0, 3)), rotation=np.zeros((0, 4)),
                 opacity_logit=np.zeros(0), color=np.zeros((0, 3)), feature=np.zeros((0, d)), feature_dim=d)
    return O.OracleMapper(m, MapperConfig())


def test_insertion_keeps_only_far_enough_points():
    pos, col, feat, sp = simple_sources(3, 4)
    om = empty_mapper()
    assert om.insert(pos, col, feat, sp, [0.01, 0.02, 0.03], 0.05, Pose()) == 0
    assert om.size() == 0 and om.generation() == 0
    om = empty_mapper()
    assert om.insert(pos, col, feat, sp, [INF] * 3, 0.05, Pose()) == 3
    assert om.size() == 3 and om.generation() == 1 and om.moments(0).size == 9
    e = om.export()
    assert np.allclose(1.0 / (1.0 + np.exp(-e["opacity_logit"])), 0.5)
    assert np.all(np.abs(np.linalg.norm(e["feature"], axis=1) - 1.0) < 1e-9)
    om = empty_mapper()
    assert om.insert(pos, col, feat, sp, [0.01, 0.2, 0.07], 0.05, Pose()) == 2
    e = om.export()
    assert np.linalg.norm(e["mean"][0] - pos[1]) < 1e-12 and np.linalg.norm(e["mean"][1] - pos[2]) < 1e-12
    om = empty_mapper()
    p1, c1, f1, s1 = simple_sources(1, 4)
    assert om.insert(p1, c1, f1, s1, [INF], 0.05, Pose(translation=np.array([-1.0, 0.0, 0.0]))) == 1
    assert np.linalg.norm(om.export()["mean"][0] - [1.0, 0.0, 1.0]) < 1e-12


def prune_case(counts, maxc, keep, seed, thr=0):
    om = O.OracleMapper(stats_map(len(counts)), MapperConfig())
    om.set_stats(counts, maxc)
    return om, om.prune(keep, seed, thr)


def test_prune_keeps_non_candidates_untouched():
    om, removed = prune_case([1, 2, 3, 4], [0.1, 0.2, 0.3, 0.4], 0.5, 7)
    e = om.export()
    assert removed.size == 0 and om.size() == 4
    assert (e["topk_count"] == 0).all() and (e["max_contribution"] == 0).all()
    om, removed = prune_case([0, 0, 5], [0.0, 0.0, 0.9], 0.5, 7)
    assert removed.size == 0 and om.size() == 3
    for seed in range(50):
        om, removed = prune_case([5, 0, 3, 0], [0.1, 0.2, 0.3, 0.4], 0.5, seed)
        assert set(removed.tolist()) <= {1, 3} and om.size() == 4 - removed.size
        assert om.moments(0).size == 3 * om.size()


def survival_oracle(scores, keep):  # test_mapper.cpp:32-65, the exact draw-tree marginals
    n = len(scores)
    marg = np.zeros(n)
    stack = [(list(range(n)), 1.0, keep)]
    while stack:
        pool, prob, left = stack.pop()
        if left == 0:
            continue
        mass = sum(scores[i] for i in pool)
        for p, idx in enumerate(pool):
            pick = scores[idx] / mass if mass > 0 else 1.0 / len(pool)
            if pick <= 0:
                continue
            marg[idx] += prob * pick
            stack.append((pool[:p] + pool[p + 1:], prob * pick, left - 1))
    return marg


@pytest.mark.parametrize("scores,trials,seed0,tol", [([0.25] * 4, 4000, 1000, 0.03),
                                                     ([0.9, 0.1, 0.05, 0.0], 6000, 9000, 0.02),
                                                     ([0.9, 0.0, 0.0, 0.0], 6000, 40000, 0.025)])
def test_prune_survival_frequencies_match_draw_tree(scores, trials, seed0, tol):  # test_mapper.cpp:199-268
    marg = survival_oracle(scores, 2)
    survived = np.zeros(4)
    for t in range(trials):
        om, removed = prune_case([0, 0, 0, 0], scores, 0.5, seed0 + t)
        alive = np.ones(4, bool)
        alive[removed] = False
        survived += alive
    assert np.all(np.abs(survived / trials - marg) < tol)


def test_optimizer_state_in_lockstep_through_insert_and_prune():  # test_mapper.cpp:417-441
    pos, col, feat, sp = simple_sources(6, 4)
    om = empty_mapper()
    om.insert(pos, col, feat, sp, [INF] * 6, 0.05, Pose())
    om.set_stats([3 if i % 2 == 0 else 0 for i in range(6)], [0.1 * (i + 1) for i in range(6)])
    mom = om.moments(0)
    for i in range(6):
        mom[i * 3] = 100.0 + i
    removed = om.prune(0.5, 5, 0)
    assert removed.size == 1 and om.moments(0).size == 3 * om.size()
    e = om.export()
    mom = om.moments(0)
    for i in range(om.size()):
        tag = int(round(mom[i * 3] - 100.0))
        assert np.linalg.norm(e["mean"][i] - pos[tag]) < 1e-12


# ---- SPLF checkpoint (test_mapper.cpp:443-468) and segment_by_query (test_eval.cpp:65-113)
def test_checkpoint_round_trips_bit_exactly(tmp_path):
    m = synth.random_scene(25, 8, 5)
    p1, p2 = str(tmp_path / "a.bin"), str(tmp_path / "b.bin")
    O.checkpoint_save(m, p1)
    loaded = O.checkpoint_load(p1)
    assert loaded["mean"].shape[0] == 25 and loaded["feature_dim"] == 8
    m2 = SceneMap(mean=loaded["mean"], log_scale=loaded["log_scale"], rotation=loaded["rotation"],
                  opacity_logit=loaded["opacity_logit"], color=loaded["color"], feature=loaded["feature"],
                  feature_dim=8)
    O.checkpoint_save(m2, p2)
    b1, b2 = open(p1, "rb").read(), open(p2, "rb").read()
    assert b1 == b2 and len(b1) == 20 + 25 * (14 + 8) * 4
    with pytest.raises(RuntimeError, match="cannot open"):
        O.checkpoint_load(str(tmp_path / "missing.bin"))
    p3 = str(tmp_path / "short.bin")
    open(p3, "wb").write(b1[:40])
    with pytest.raises(RuntimeError, match="truncated file .*short.bin"):
        O.checkpoint_load(p3)


def test_segmentation_by_query_kats():  # test_eval.cpp:65-90
    emb = np.eye(4, 8)
    feat = np.zeros((10, 10, 8))
    feat[:, :5, 0] = 1.0
    feat[:, 5:, 1] = 1.0
    pred = O.segment_by_query(feat, emb)
    assert (pred[:, :5] == 0).all() and (pred[:, 5:] == 1).all()
    feat[0, 0] = 0.0
    assert O.segment_by_query(feat, emb)[0, 0] == 255


def test_random_unit_features_split_evenly():  # test_eval.cpp:93-113 (smaller)
    rng = np.random.default_rng(123)
    v = rng.uniform(-1, 1, (100, 1000, 16))
    v /= np.linalg.norm(v, axis=-1, keepdims=True)
    pred = O.segment_by_query(v, np.eye(4, 16))
    frac = np.bincount(pred.ravel(), minlength=4)[:4] / pred.size
    assert np.all(np.abs(frac - 0.25) < 0.01)

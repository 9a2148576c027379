"""Parity at BASELINE.json's full config-3 size (1M Gaussians, 1200 x 680, D = 512, K = 3, the bench
recipe scene and orbit pose): the GPU path against the CPU oracle where the oracle finishes in
seconds (prepare / geometric pass / feature gather / geometry backward), and size-independent
properties where it would not (tile-size independence, weight conservation, Top-K ordering,
linearity and the forward/backward adjoint of the feature path, run-to-run bit-determinism).
Tolerances as in test_gpu_parity.py."""
import numpy as np
import pytest

import _oracle as O
from paper_2602_06991_b200 import api
import scenegen as synth
from paper_2602_06991_b200.types import RenderSettings

pytestmark = pytest.mark.gpu

N_G, W, H, D, K = 1_000_000, 1200, 680, 512, 3


@pytest.fixture(scope="module")
def full():
    m, cam, pose, _ = synth.bench_scene(N_G, W, H, D)
    m.feature = synth.unit_features(m.size(), D, 7)
    r = api.Renderer(0)
    yield r, m, cam, pose
    r.close()


def test_fullsize_geometric_and_prepare_match_oracle(full):
    r, m, cam, pose = full
    s = RenderSettings(top_k=K)
    g = r.render_geometric(m, pose, cam, s)
    o = O.render_geometric(m, pose, cam, s)
    assert (g.topk.count == o["count"]).all() and (g.topk.index == o["index"]).all()
    np.testing.assert_allclose(g.topk.weight, o["weight"], rtol=1e-9, atol=0)
    for f in ("color", "depth", "alpha"):
        np.testing.assert_allclose(getattr(g, f), o[f], rtol=0, atol=1e-9)
    np.testing.assert_allclose(g.contributions, o["contributions"], rtol=1e-9, atol=0)
    p = r.prepare_scene(m, pose, cam, s)
    po = O.prepare_scene(m, pose, cam, s)
    assert (p.src == po["src"]).all() and (p.tile_offsets == po["tile_offsets"]).all()
    assert (p.tile_entries == po["tile_entries"]).all()


def test_fullsize_tile_size_independent_and_conserving(full):
    r, m, cam, pose = full
    ref = r.render_geometric(m, pose, cam, RenderSettings(top_k=K))
    for tile in (8, 32):
        g = r.render_geometric(m, pose, cam, RenderSettings(top_k=K, tile_size=tile))
        assert (g.topk.index == ref.topk.index).all() and (g.topk.count == ref.topk.count).all()
        assert np.array_equal(g.topk.weight, ref.topk.weight) and np.array_equal(g.color, ref.color)
        assert np.array_equal(g.depth, ref.depth) and np.array_equal(g.alpha, ref.alpha)
    again = r.render_geometric(m, pose, cam, RenderSettings(top_k=K))
    assert np.array_equal(again.color, ref.color) and (again.topk.index == ref.topk.index).all()
    # sum of weights + final transmittance = 1 (T recovered from two backgrounds)
    b = r.render_geometric(m, pose, cam, RenderSettings(top_k=K, background=(1.0, 1.0, 1.0)))
    T = b.color[..., 0] - ref.color[..., 0]
    np.testing.assert_allclose(ref.alpha + T, 1.0, atol=1e-9)
    # Top-K records: valid distinct ids, weights non-increasing, count <= K
    idx = ref.topk.index.reshape(H * W, K)
    wt = ref.topk.weight.reshape(H * W, K)
    cnt = ref.topk.count.astype(np.int64)
    assert cnt.max() <= K
    live = np.arange(K)[None, :] < cnt[:, None]
    assert ((idx >= 0) & (idx < m.size()))[live].all() and (idx[~live] == -1).all()
    assert (np.diff(np.where(live, wt, -np.inf), axis=1)[live[:, 1:]] <= 0).all()
    assert (idx[:, 0] != idx[:, 1])[cnt >= 2].all() and (idx[:, 1] != idx[:, 2])[cnt >= 3].all()


def test_fullsize_feature_matches_oracle_linear_and_adjoint(full):
    r, m, cam, pose = full
    g = r.render_geometric(m, pose, cam, RenderSettings(top_k=K))
    F = r.render_feature(m, g.topk)
    fo = O.render_feature(m, W, H, K, g.topk.index, g.topk.weight, g.topk.count)
    err = np.abs(F.astype(np.float64) - fo)
    assert (err <= 1e-5 * np.maximum(1.0, np.abs(fo))).all()
    del fo, err
    m2 = m.copy()
    m2.feature = (m.feature.astype(np.float32) * 2).astype(np.float32)
    assert np.array_equal(r.render_feature(m2, g.topk), 2 * F)  # exact: scaling by 2 commutes
    G = synth.uniform_image((H, W, D), 11).astype(np.float32)
    df = r.backward_feature(m, g.topk, G)
    assert np.array_equal(r.backward_feature(m, g.topk, G), df)  # bit-deterministic
    lhs = float(np.dot(F.astype(np.float64).ravel(), G.astype(np.float64).ravel()))
    rhs = float(np.dot(m.feature.astype(np.float32).astype(np.float64).ravel(), df.astype(np.float64)))
    assert lhs == pytest.approx(rhs, rel=1e-4, abs=1e-2)


def test_fullsize_backward_geometric_matches_oracle(full):
    r, m, cam, pose = full
    s = RenderSettings(top_k=K)
    gc = synth.uniform_image((H, W, 3), 12)
    gd = synth.uniform_image((H, W), 13)
    g = r.backward_geometric(m, pose, cam, s, gc, gd)
    o = O.backward_geometric(m, pose, cam, s, gc, gd)
    for f in ("mean", "log_scale", "rotation", "opacity_logit", "color"):
        a, b = getattr(g, f), o[f]
        scale = max(1e-12, np.abs(b).max())
        np.testing.assert_array_less(np.abs(a - b), 1e-4 * np.maximum(np.abs(b), 1e-2 * scale) + 1e-12)
        # the untouched set (Gaussians with no gradient at all) is the same; single components may
        # cancel to exactly 0 in one summation order and to a rounding residue in the other
        za, zb = (a.reshape(len(a), -1) == 0).all(axis=1), (b.reshape(len(b), -1) == 0).all(axis=1)
        assert (za == zb).all(), f
    scale = max(1e-12, np.abs(o["pose_twist"]).max())
    np.testing.assert_array_less(np.abs(g.pose_twist - o["pose_twist"]),
                                 1e-4 * np.maximum(np.abs(o["pose_twist"]), 1e-2 * scale) + 1e-12)


def test_fullsize_mapping_iterations_match_oracle(full):
    """Two tk_optimize_step iterations (a feature step and a geometry step) on the config-3 map
    against the oracle's optimize_step: the bench's mapping workload (ground-truth keyframe of the
    recipe scene, perturbed map), tolerances of tests/test_gpu_mapping.py."""
    from paper_2602_06991_b200.types import MapperConfig
    r, m, cam, pose = full
    emb = synth.unit_features(4, D, 99)
    gt, _ = synth.render_ground_truth(r, m, m.class_ids, emb, [pose], cam)[0]
    rng = np.random.default_rng(17)
    spacing = float(np.median(np.exp(m.log_scale[:, 0]))) * 2.0
    mp = m.copy()
    mp.mean = m.mean + rng.normal(0.0, 0.3 * spacing, m.mean.shape)
    mp.color = np.clip(m.color + rng.normal(0.0, 0.05, m.color.shape), 0.0, 1.0)
    cfg = MapperConfig()
    s = RenderSettings(top_k=K)
    om = O.OracleMapper(mp, cfg)
    r.upload(mp)
    r.optimizer_reset(True)
    r.keyframe_set(0, pose, gt)
    for it in (5, 6):
        ov, ofs = om.step(pose, cam, s, gt.color, gt.depth, gt.feature, it)
        gv, gfs = r.optimize_step(cfg, cam, s, 0, it)
        assert gfs == ofs
        assert gv.geo == pytest.approx(ov["geo"], rel=1e-10), it
        assert gv.feat == pytest.approx(ov["feat"], rel=1e-5, abs=1e-12), it
    o = om.export()
    g = r.scene_download(mp.size(), D)
    for key in ("mean", "log_scale", "rotation", "opacity_logit", "color"):
        np.testing.assert_allclose(g[key], o[key], rtol=0, atol=1e-10, err_msg=key)
    # features: 2e-5 everywhere except where the feature L1's sign(F - F_gt) ties below fp32
    # resolution (fp32 F on the GPU, fp64 in the oracle): a flipped sign moves that channel's Adam
    # step by at most 2 * lr_feature.  At this size a few dozen of the 5.1e8 channels do.
    dev = np.abs(g["feature"].astype(np.float64) - o["feature"])
    bad = dev > 2e-5
    assert bad.sum() <= 1e-6 * dev.size, f"{bad.sum()} channels beyond 2e-5"
    assert dev.max() <= 2 * cfg.lr_feature + 2e-5
    assert (g["topk_count"] == o["topk_count"]).all()
    np.testing.assert_allclose(g["max_contribution"], o["max_contribution"], rtol=1e-9, atol=0)


def test_fullsize_backward_feature_matches_oracle_elementwise(full):
    """backward_feature at config 3 element by element against the oracle, run one 64-channel
    slice at a time (the op never mixes channels, so each slice is exact) to keep the oracle's
    per-thread N x D fp64 partials within host RAM."""
    r, m, cam, pose = full
    g = r.render_geometric(m, pose, cam, RenderSettings(top_k=K))
    G = synth.uniform_image((H, W, D), 11).astype(np.float32)
    df = r.backward_feature(m, g.topk, G).reshape(m.size(), D)
    for c0, c1, o in O.backward_feature_slices(m, W, H, K, g.topk.index, g.topk.weight, g.topk.count, G):
        a = df[:, c0:c1].astype(np.float64)
        bad = np.abs(a - o) > 2e-5 * np.maximum(1.0, np.abs(o))
        assert not bad.any(), (c0, c1, int(bad.sum()))
        # rows no record references are exactly zero on both sides (dense N x D, backward.cpp:315)
        assert np.array_equal((a == 0).all(axis=1), (o == 0).all(axis=1)), (c0, c1)


GEOM_FIELDS = ("mean", "log_scale", "rotation", "opacity_logit", "color", "pose_twist")


def test_fullsize_backward_geometric_bit_deterministic(full):
    """backward_geometric twice on fresh forwards (the drop-in re-uploads and re-prepares on every
    call): every gradient byte-identical (the reference merges its per-thread partials in a fixed
    order, backward.cpp:166-178; the GPU sums each Gaussian's slot partials in a fixed order)."""
    r, m, cam, pose = full
    s = RenderSettings(top_k=K)
    gc = synth.uniform_image((H, W, 3), 12)
    gd = synth.uniform_image((H, W), 13)
    a = r.backward_geometric(m, pose, cam, s, gc, gd)
    for _ in range(2):
        b = r.backward_geometric(m, pose, cam, s, gc, gd)
        for f in GEOM_FIELDS:
            assert getattr(a, f).tobytes() == getattr(b, f).tobytes(), f


def test_fullsize_mapping_run_bit_deterministic(full):
    """Ten tk_optimize_step iterations (features every 5th step) from the same start, twice: the
    optimised map, its Adam-driven geometry and the selection statistics are byte-identical."""
    from paper_2602_06991_b200.types import MapperConfig
    r, m, cam, pose = full
    emb = synth.unit_features(4, D, 99)
    gt, _ = synth.render_ground_truth(r, m, m.class_ids, emb, [pose], cam)[0]
    rng = np.random.default_rng(23)
    spacing = float(np.median(np.exp(m.log_scale[:, 0]))) * 2.0
    mp = m.copy()
    mp.mean = m.mean + rng.normal(0.0, 0.3 * spacing, m.mean.shape)
    cfg = MapperConfig()
    s = RenderSettings(top_k=K)
    runs = []
    for _ in range(2):
        r.upload(mp)
        r.optimizer_reset(True)
        r.keyframe_set(0, pose, gt)
        losses = [r.optimize_step(cfg, cam, s, 0, it)[0] for it in range(10)]
        runs.append((r.scene_download(mp.size(), D), [(v.map, v.geo, v.feat) for v in losses]))
    (a, la), (b, lb) = runs
    assert la == lb
    for key in a:
        assert a[key].tobytes() == b[key].tobytes(), key

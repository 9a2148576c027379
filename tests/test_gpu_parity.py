"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle.

Contract:
  * PreparedScene order and CSR: exactly equal.
  * topk.count and topk.index: exactly equal.
  * colour / depth / alpha: abs <= 1e-9 (fp64 on both sides; only exp() differs by <= 1 ulp).
  * Top-K weights and contributions: rel <= 1e-9.
  * F and df (fp32 features on the GPU vs fp64 oracle): abs <= 1e-5 * max(1, |x|).
  * geometry grads: rel <= 1e-4 (floor 1e-6 * max|g|, the reference's FD tolerance).
"""
import numpy as np
import pytest

import _oracle as O
from _se3 import axis_angle
from paper_2602_06991_b200 import api
import scenegen as synth
from paper_2602_06991_b200.types import CameraIntrinsics, Pose, RenderSettings, SceneMap, TopKGrid

pytestmark = pytest.mark.gpu

FEAT_TOL = 1e-5


@pytest.fixture(scope="module")
def R():
    r = api.Renderer(0)
    yield r
    r.close()


def assert_geom_equal(g, o, w_rtol=1e-9, img_atol=1e-9):
    assert (g.topk.count == o["count"]).all(), "top-k counts differ"
    assert (g.topk.index == o["index"]).all(), "top-k indices differ"
    np.testing.assert_allclose(g.topk.weight, o["weight"], rtol=w_rtol, atol=0)
    np.testing.assert_allclose(g.color, o["color"], rtol=0, atol=img_atol)
    np.testing.assert_allclose(g.depth, o["depth"], rtol=0, atol=img_atol)
    np.testing.assert_allclose(g.alpha, o["alpha"], rtol=0, atol=img_atol)
    np.testing.assert_allclose(g.contributions, o["contributions"], rtol=w_rtol, atol=0)


def feat_close(a, b, tol=FEAT_TOL):
    np.testing.assert_array_less(np.abs(np.asarray(a, np.float64) - b), tol * np.maximum(1.0, np.abs(b)) + 1e-30)


def aniso_scene():
    """Needle- and sheet-like Gaussians at random orientations: their cutoff ellipses fill little
    of their bounding boxes, so the exact ellipse-vs-block cull decides many block corners."""
    m = synth.random_scene(400, 8, 23)
    ls = m.log_scale.copy()
    ls[:, 0] += 1.5
    ls[:, 1] -= 2.5
    m.log_scale = ls
    return m


SCENES = [
    ("random300_seed1", lambda: synth.random_scene(300, 8, 1), lambda: synth.test_camera(64, 48), Pose()),
    ("random250_seed17", lambda: synth.random_scene(250, 8, 17), lambda: synth.test_camera(64, 64),
     Pose(axis_angle(0.2, (0, 1, 0)), (0.05, -0.02, 0.1))),
    ("aniso400_seed23", aniso_scene, lambda: synth.test_camera(96, 80), Pose(axis_angle(0.3, (1, 0, 0)), (0, 0, 0))),
    ("random2000_seed5", lambda: synth.random_scene(2000, 16, 5), lambda: synth.test_camera(160, 120), Pose()),
]


@pytest.mark.parametrize("name,mk,cam,pose", SCENES, ids=[s[0] for s in SCENES])
@pytest.mark.parametrize("tile", [16, 8, 32])
def test_prepared_scene_exact(R, name, mk, cam, pose, tile):
    m, c = mk(), cam()
    s = RenderSettings(tile_size=tile)
    g = R.prepare_scene(m, pose, c, s)
    o = O.prepare_scene(m, pose, c, s)
    assert (g.src == o["src"]).all(), "depth order differs"
    assert (g.tile_offsets == o["tile_offsets"]).all(), "tile CSR offsets differ"
    assert (g.tile_entries == o["tile_entries"]).all(), "tile lists differ"
    # mean2d and depth are bit-identical (mul/add/div only); the inverse covariance and opacity
    # go through exp() (CUDA libdevice vs glibc), which may differ in the last ulp
    assert (g.entries[:, [0, 1, 5]] == o["entries"][:, [0, 1, 5]]).all()
    np.testing.assert_allclose(g.entries[:, [2, 3, 4, 6]], o["entries"][:, [2, 3, 4, 6]], rtol=1e-13)


@pytest.mark.parametrize("name,mk,cam,pose", SCENES, ids=[s[0] for s in SCENES])
@pytest.mark.parametrize("k", [1, 3, 4, 8, 16, 32])
def test_render_geometric_matches_oracle(R, name, mk, cam, pose, k):
    m, c = mk(), cam()
    s = RenderSettings(top_k=k, background=(0.1, 0.2, 0.3))
    assert_geom_equal(R.render_geometric(m, pose, c, s), O.render_geometric(m, pose, c, s))


@pytest.mark.parametrize("floor", [0.0, 1e-4, 5e-2])
def test_render_geometric_floor_variants(R, floor):
    m, c = synth.random_scene(400, 4, 9), synth.test_camera(48, 48)
    s = RenderSettings(transmittance_floor=floor)
    assert_geom_equal(R.render_geometric(m, Pose(), c, s), O.render_geometric(m, Pose(), c, s))


def test_tile_size_independent_and_deterministic(R):  # test_raster.cpp:285-305
    m, c = synth.random_scene(250, 4, 17), synth.test_camera(64, 64)
    a = R.render_geometric(m, Pose(), c, RenderSettings())
    b = R.render_geometric(m, Pose(), c, RenderSettings())
    d = R.render_geometric(m, Pose(), c, RenderSettings(tile_size=8))
    e = R.render_geometric(m, Pose(), c, RenderSettings(tile_size=13))
    for x in (b, d, e):
        assert a.color.tobytes() == x.color.tobytes() and a.depth.tobytes() == x.depth.tobytes()
        assert (a.topk.index == x.topk.index).all() and (a.contributions == x.contributions).all()


def test_empty_map_and_degenerate(R):  # test_raster.cpp:41-58, 307-319
    empty = SceneMap(feature=np.zeros((0, 2)), feature_dim=2)
    cam = CameraIntrinsics(fx=40, fy=40, cx=16, cy=16, width=32, height=32, near_plane=0.05, far_plane=50)
    o = R.render_geometric(empty, Pose(), cam, RenderSettings(background=(0.2, 0.4, 0.6)))
    assert np.allclose(o.color, [0.2, 0.4, 0.6]) and (o.depth == 0).all() and (o.topk.count == 0).all()
    deg = SceneMap(mean=np.array([[0, 0, 1.0]]), log_scale=np.full((1, 3), 400.0), rotation=np.array([[1.0, 0, 0, 0]]),
                   opacity_logit=np.zeros(1), color=np.ones((1, 3)), feature=np.ones((1, 2)), feature_dim=2)
    cam16 = CameraIntrinsics(fx=10, fy=10, cx=8, cy=8, width=16, height=16, near_plane=0.05, far_plane=50)
    assert R.render_geometric(deg, Pose(), cam16, RenderSettings(cov2d_dilation=0.0)).alpha[8, 8] == 0.0


def test_single_and_two_gaussian_kats(R):  # test_raster.cpp:60-100 (log_scale -2: see oracle KATs)
    def flat(gs):
        n = len(gs)
        return SceneMap(mean=np.array([g[0] for g in gs], float), log_scale=np.full((n, 3), -2.0),
                        rotation=np.tile([1.0, 0, 0, 0], (n, 1)),
                        opacity_logit=np.array([np.log(g[1] / (1 - g[1])) for g in gs]),
                        color=np.array([g[2] for g in gs], float), feature=np.ones((n, 2)), feature_dim=2)
    cam = CameraIntrinsics(fx=16, fy=16, cx=16, cy=16, width=33, height=33, near_plane=0.05, far_plane=50)
    o = R.render_geometric(flat([((0, 0, 2), 0.5, (1, 0, 0))]), Pose(), cam, RenderSettings())
    assert o.color[16, 16, 0] == pytest.approx(0.5, rel=1e-12) and o.depth[16, 16] == pytest.approx(1.0, rel=1e-12)
    assert o.contributions[0] == pytest.approx(0.5, rel=1e-12)
    two = flat([((0, 0, 1), 0.6, (1, 0, 0)), ((0, 0, 2), 0.8, (0, 1, 0))])
    o = R.render_geometric(two, Pose(), cam, RenderSettings(transmittance_floor=0.0))
    assert o.color[16, 16, 0] == pytest.approx(0.6, rel=1e-9) and o.color[16, 16, 1] == pytest.approx(0.32, rel=1e-9)
    assert o.depth[16, 16] == pytest.approx(1.24, rel=1e-9)


@pytest.mark.parametrize("d", [3, 4, 16, 512, 1000, 1030])
@pytest.mark.parametrize("k", [1, 3, 16])
def test_render_feature_matches_oracle(R, d, k):
    m, c = synth.random_scene(600, d, 21), synth.test_camera(64, 48)
    s = RenderSettings(top_k=k)
    g = R.render_geometric(m, Pose(), c, s)
    f = R.render_feature(m, g.topk)
    o = O.render_feature(m, c.width, c.height, g.topk.k, g.topk.index, g.topk.weight, g.topk.count)
    assert f.shape == o.shape
    feat_close(f, o)


def test_render_feature_renormalisation_kat(R):  # test_raster.cpp:208-241
    m = SceneMap(mean=np.array([[0, 0, 1.0], [0, 0, 2.0]]), log_scale=np.full((2, 3), -2.0),
                 rotation=np.tile([1.0, 0, 0, 0], (2, 1)), opacity_logit=np.zeros(2), color=np.zeros((2, 3)),
                 feature=np.array([[1.0, 0, 0], [0, 1.0, 0]]), feature_dim=3)
    f = R.render_feature(m, TopKGrid(1, 1, 2, np.array([0, 1], np.int32), np.array([0.3, 0.1]), np.array([2], np.uint8)))
    assert f[0, 0, 0] == pytest.approx(0.75, rel=1e-6) and f[0, 0, 1] == pytest.approx(0.25, rel=1e-6)
    assert f[0, 0, 2] == 0.0
    f1 = R.render_feature(m, TopKGrid(1, 1, 1, np.array([1], np.int32), np.array([0.123]), np.array([1], np.uint8)))
    assert f1[0, 0, 1] == 1.0
    f0 = R.render_feature(m, TopKGrid.empty(1, 1, 2))
    assert (f0 == 0).all()


def test_stale_index_raises_reference_message(R):  # test_raster.cpp:243-253, test_backward.cpp:201-205
    m = synth.random_scene(3, 4, 6)
    grid = TopKGrid(1, 1, 1, np.array([5], np.int32), np.array([0.5]), np.array([1], np.uint8))
    with pytest.raises(RuntimeError, match=r"^render_feature: top-k record references gaussian 5 but the map "
                                           r"holds 3 \(stale snapshot\)$"):
        R.render_feature(m, grid)
    with pytest.raises(RuntimeError, match=r"^backward_feature: top-k record references gaussian 5"):
        R.backward_feature(m, grid, np.ones((1, 1, 4)))


def test_stale_device_records_after_map_shrinks(R):
    big = synth.random_scene(400, 4, 3)
    c = synth.test_camera(48, 48)
    R.render_geometric(big, Pose(), c, RenderSettings())
    import ctypes as C
    from paper_2602_06991_b200 import _native as N
    small = big.copy()
    for f in ("mean", "log_scale", "rotation", "opacity_logit", "color", "feature"):
        setattr(small, f, getattr(small, f)[:10].copy())
    R.upload(small)
    out = np.zeros((48, 48, 4), np.float32)
    st = R.lib.tk_render_feature(R.ctx, None, out.ctypes.data, N.TK_HOST)
    assert st == N.TK_ERR_STALE_INDEX
    assert b"stale snapshot" in R.lib.tk_last_error()


@pytest.mark.parametrize("d", [4, 64, 512, 1000, 1030])
@pytest.mark.parametrize("k", [1, 3, 8])
def test_backward_feature_matches_oracle(R, d, k):
    m, c = synth.random_scene(500, d, 33), synth.test_camera(48, 40)
    s = RenderSettings(top_k=k)
    g = R.render_geometric(m, Pose(), c, s)
    gf = synth.uniform_image((c.height, c.width, d), 11).astype(np.float32)
    gf[5, :, :] = 0.0  # zero rows are skipped by the reference
    b = R.backward_feature(m, g.topk, gf)
    o = O.backward_feature(m, c.width, c.height, g.topk.k, g.topk.index, g.topk.weight, g.topk.count,
                           gf.astype(np.float64))
    feat_close(b, o, 2e-5)


def test_backward_feature_passthrough(R):  # test_backward.cpp:181-206
    m = synth.random_scene(3, 4, 6)
    grid = TopKGrid(1, 1, 1, np.array([2], np.int32), np.array([0.4]), np.array([1], np.uint8))
    assert (R.backward_feature(m, grid, np.zeros((1, 1, 4))) == 0).all()
    g = np.zeros((1, 1, 4))
    g[0, 0, 0], g[0, 0, 3] = 0.7, -0.2
    out = R.backward_feature(m, grid, g)
    assert out[8] == pytest.approx(0.7) and out[11] == pytest.approx(-0.2) and out[0] == 0.0


def test_feature_forward_backward_adjoint(R):
    """<F, G> == <f, dL/df> for the linear map f -> F (size-independent property)."""
    m, c = synth.random_scene(3000, 32, 8), synth.test_camera(128, 96)
    g = R.render_geometric(m, Pose(), c, RenderSettings(top_k=4))
    F = R.render_feature(m, g.topk).astype(np.float64)
    G = synth.uniform_image(F.shape, 4).astype(np.float32)
    df = R.backward_feature(m, g.topk, G).astype(np.float64)
    lhs = float((F * G).sum())
    rhs = float((m.feature.astype(np.float32).astype(np.float64).reshape(-1) * df).sum())
    assert lhs == pytest.approx(rhs, rel=1e-4, abs=1e-3)


def geom_close(a, b, rtol=1e-4):
    scale = max(1e-12, np.abs(b).max())
    np.testing.assert_array_less(np.abs(a - b), rtol * np.maximum(np.abs(b), 1e-2 * scale) + 1e-12)


@pytest.mark.parametrize("name,mk,cam,pose", SCENES, ids=[s[0] for s in SCENES])
@pytest.mark.parametrize("floor", [0.0, 1e-4])
def test_backward_geometric_matches_oracle(R, name, mk, cam, pose, floor):
    m, c = mk(), cam()
    s = RenderSettings(transmittance_floor=floor, background=(0.3, 0.1, 0.2))
    gc = synth.uniform_image((c.height, c.width, 3), 12)
    gd = synth.uniform_image((c.height, c.width), 13)
    g = R.backward_geometric(m, pose, c, s, gc, gd)
    o = O.backward_geometric(m, pose, c, s, gc, gd)
    for f in ("mean", "log_scale", "rotation", "opacity_logit", "color"):
        geom_close(getattr(g, f), o[f])
        assert ((getattr(g, f) == 0) == (o[f] == 0)).all(), f"untouched set differs for {f}"
    geom_close(g.pose_twist, o["pose_twist"])


def test_backward_geometric_after_forward_reuses_and_matches(R):
    m, c = synth.random_scene(800, 4, 44), synth.test_camera(96, 72)
    s = RenderSettings()
    gc = synth.uniform_image((72, 96, 3), 12)
    gd = synth.uniform_image((72, 96), 13)
    R.render_geometric(m, Pose(), c, s)
    g1 = R.backward_geometric(m, Pose(), c, s, gc, gd)
    g2 = R.backward_geometric(m, Pose(), c, s, gc, None)
    o1 = O.backward_geometric(m, Pose(), c, s, gc, gd)
    o2 = O.backward_geometric(m, Pose(), c, s, gc, None)
    geom_close(g1.mean, o1["mean"])
    geom_close(g2.mean, o2["mean"])


def test_backward_geometric_zero_grads(R):  # test_backward.cpp:104-120
    m, c = synth.random_scene(10, 3, 4), synth.test_camera(16, 16)
    g = R.backward_geometric(m, Pose(), c, RenderSettings(transmittance_floor=0.0), np.zeros((16, 16, 3)),
                             np.zeros((16, 16)))
    for f in ("mean", "log_scale", "rotation", "opacity_logit", "color", "pose_twist"):
        assert (getattr(g, f) == 0).all()


@pytest.mark.parametrize("d", [5, 64])
def test_full_blend_matches_oracle(R, d):
    m, c = synth.random_scene(400, d, 31), synth.test_camera(48, 40)
    s = RenderSettings()
    f = R.render_feature_full_blend(m, Pose(), c, s)
    o = O.render_feature_full_blend(m, Pose(), c, s)
    feat_close(f, o)


def test_bench_recipe_scene_parity(R):
    """Config-1 recipe (bench scene, orbit pose) at reduced size: indices exact vs the oracle."""
    m, cam, pose, _ = synth.bench_scene(20000, 160, 120, 32)
    m.feature = synth.unit_features(m.size(), 32, 7)
    s = RenderSettings()
    g = R.render_geometric(m, pose, cam, s)
    o = O.render_geometric(m, pose, cam, s)
    assert_geom_equal(g, o)
    p = R.prepare_scene(m, pose, cam, s)
    po = O.prepare_scene(m, pose, cam, s)
    assert (p.tile_entries == po["tile_entries"]).all() and (p.src == po["src"]).all()


def test_nccl_single_rank_allgather_equals_render(R):
    """tk_comm_* with one rank: the all-gather + interleave path returns the rendered map."""
    import ctypes as C
    from paper_2602_06991_b200 import _native as N
    m, c = synth.random_scene(500, 16, 2), synth.test_camera(48, 32)
    g = R.render_geometric(m, Pose(), c, RenderSettings())
    f = R.render_feature(m, g.topk)
    uid = (C.c_uint8 * 128)()
    N.check(R.lib.tk_comm_unique_id(uid))
    N.check(R.lib.tk_comm_init(R.ctx, uid, 1, 0, 16))
    N.check(R.lib.tk_render_feature(R.ctx, None, None, N.TK_DEVICE))
    full = np.zeros((32, 48, 16), np.float32)
    N.check(R.lib.tk_allgather_feature(R.ctx, full.ctypes.data, N.TK_HOST))
    assert (full == f).all()


def test_backward_feature_bit_deterministic(R):
    m, c = synth.random_scene(2000, 64, 12), synth.test_camera(96, 64)
    g = R.render_geometric(m, Pose(), c, RenderSettings(top_k=4))
    gf = synth.uniform_image((64, 96, 64), 3).astype(np.float32)
    a = R.backward_feature(m, g.topk, gf)
    b = R.backward_feature(m, g.topk, gf)
    assert a.tobytes() == b.tobytes()


@pytest.mark.parametrize("w,h", [(64, 48), (160, 120)])
def test_backward_feature_huge_segments(R, w, h):
    """A Gaussian filling the view owns one Top-K record per pixel: segments beyond the block sort
    tile (8192 records at 160x120) take the tiled bitonic + merge-by-rank path."""
    m = synth.random_scene(300, 16, 4)
    m.mean[1:, 2] += 3.0          # everything else behind the big one
    m.mean[0] = (0.0, 0.0, 0.95)  # in front; z > 3 exp(max log_scale) keeps it past the cull
    m.log_scale[0] = (-1.25, -1.25, -1.25)
    m.opacity_logit[0] = -2.0
    cam = synth.test_camera(w, h)
    g = R.render_geometric(m, Pose(), cam, RenderSettings(top_k=4))
    counts = np.bincount(g.topk.index[g.topk.index >= 0], minlength=m.size())
    assert counts.max() > (8192 if w * h > 8192 else 100)
    gf = synth.uniform_image((h, w, 16), 5).astype(np.float32)
    a = R.backward_feature(m, g.topk, gf)
    b = R.backward_feature(m, g.topk, gf)
    assert a.tobytes() == b.tobytes()
    o = O.backward_feature(m, w, h, 4, g.topk.index, g.topk.weight, g.topk.count, gf.astype(np.float64))
    feat_close(a, o, 2e-5)


@pytest.mark.parametrize("tile", [8, 13, 32, 64])
def test_backward_geometric_tile_sizes_match_oracle(R, tile):
    """The fixed-order merge at 1, 4, 16 and 64 warp blocks per tile (tile sizes 8, 13, 32, 64): slot
    indexing (pair x warp block) and the merge tiers match the oracle, and the result is the same
    byte for byte when repeated."""
    m, c = synth.random_scene(900, 4, 71), synth.test_camera(100, 76)
    s = RenderSettings(tile_size=tile, background=(0.2, 0.1, 0.0))
    gc = synth.uniform_image((c.height, c.width, 3), 21)
    gd = synth.uniform_image((c.height, c.width), 22)
    g = R.backward_geometric(m, Pose(), c, s, gc, gd)
    o = O.backward_geometric(m, Pose(), c, s, gc, gd)
    for f in ("mean", "log_scale", "rotation", "opacity_logit", "color"):
        geom_close(getattr(g, f), o[f])
    geom_close(g.pose_twist, o["pose_twist"])
    again = R.backward_geometric(m, Pose(), c, s, gc, gd)
    for f in ("mean", "log_scale", "rotation", "opacity_logit", "color", "pose_twist"):
        assert getattr(g, f).tobytes() == getattr(again, f).tobytes(), f


def test_features_only_upload_keeps_geometry_state(R):
    """tk_scene_upload_features replaces the features only (the prepared scene and the forward
    records stay valid): the gather then reads the new rows; n / d mismatches are rejected."""
    import ctypes as C
    from paper_2602_06991_b200 import _native as N
    m, c = synth.random_scene(300, 8, 5), synth.test_camera(48, 40)
    s = RenderSettings()
    g = R.render_geometric(m, Pose(), c, s)
    m2 = m.copy()
    m2.feature = (m.feature.astype(np.float32) * -0.5).astype(np.float32)
    feat = np.ascontiguousarray(m2.feature, np.float32)
    N.check(R.lib.tk_scene_upload_features(R.ctx, m.size(), 8, feat.ctypes.data, N.TK_HOST))
    out = np.zeros((40, 48, 8), np.float32)
    N.check(R.lib.tk_render_feature(R.ctx, None, out.ctypes.data, N.TK_HOST))  # resident records
    ref = O.render_feature(m2, 48, 40, 3, g.topk.index, g.topk.weight, g.topk.count)
    feat_close(out, ref)
    with pytest.raises(N.TkError):
        N.check(R.lib.tk_scene_upload_features(R.ctx, m.size() + 1, 8, feat.ctypes.data, N.TK_HOST))
    with pytest.raises(N.TkError):
        N.check(R.lib.tk_scene_upload_features(R.ctx, m.size(), 4, feat.ctypes.data, N.TK_HOST))

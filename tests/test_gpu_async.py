"""TK_HOST_ASYNC: host buffers copied on the context's copy streams must give exactly the results
of the synchronous path once tk_synchronize returns, across back-to-back frames whose uploads and
read-backs overlap (the bench e2e pattern), including the pose twist delivered at synchronize."""
import ctypes as C

import numpy as np
import pytest

from paper_2602_06991_b200 import _native as N
from paper_2602_06991_b200 import api
import scenegen as synth
from paper_2602_06991_b200.api import to_camera, to_pose, to_settings
from paper_2602_06991_b200.types import Pose, RenderSettings

pytestmark = pytest.mark.gpu


def pinned(lib, shape, dtype, keep):
    nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
    p = C.c_void_p()
    N.check(lib.tk_host_alloc(nbytes, C.byref(p)))
    keep.append(p)
    return np.ctypeslib.as_array(C.cast(p, C.POINTER(np.ctypeslib.as_ctypes_type(dtype))), shape=shape)


def run_frame(R, scenes, cam, s, grads, mem, keep):
    """Frames over several scenes through the C ABI; returns the host outputs of each frame."""
    lib = R.lib
    P = cam.width * cam.height
    k = s.top_k
    results = []
    cp, cc, cs = to_pose(Pose()), to_camera(cam), to_settings(s)
    for m, (gF, gC, gD) in zip(scenes, grads):
        n, d = m.size(), m.feature_dim
        geo = [pinned(lib, a.shape, np.float64, keep) for a in (m.mean, m.log_scale, m.rotation, m.opacity_logit,
                                                                m.color)]
        for dst, a in zip(geo, (m.mean, m.log_scale, m.rotation, m.opacity_logit, m.color)):
            dst[...] = a
        feat = pinned(lib, (n, d), np.float32, keep)
        feat[...] = m.feature
        o = dict(color=pinned(lib, (P * 3,), np.float64, keep), index=pinned(lib, (P * k,), np.int32, keep),
                 F=pinned(lib, (P * d,), np.float32, keep), df=pinned(lib, (n * d,), np.float32, keep),
                 gmean=pinned(lib, (n * 3,), np.float64, keep))
        view = N.tk_scene_view(n, d, *(a.ctypes.data for a in geo), feat.ctypes.data, 0)
        N.check(lib.tk_invalidate(R.ctx))
        N.check(lib.tk_scene_upload(R.ctx, C.byref(view), mem))
        gout = N.tk_geom_out(mem, o["color"].ctypes.data, None, None, o["index"].ctypes.data, None, None, None, 0, 0)
        N.check(lib.tk_render_geometric(R.ctx, C.byref(cp), C.byref(cc), C.byref(cs), C.byref(gout)))
        N.check(lib.tk_render_feature(R.ctx, None, C.c_void_p(o["F"].ctypes.data), mem))
        N.check(lib.tk_backward_feature(R.ctx, None, C.c_void_p(gF.ctypes.data), mem, C.c_void_p(o["df"].ctypes.data),
                                        mem))
        gg = N.tk_geom_grads(mem, o["gmean"].ctypes.data, None, None, None, None)
        N.check(lib.tk_backward_geometric(R.ctx, C.byref(cp), C.byref(cc), C.byref(cs), C.c_void_p(gC.ctypes.data),
                                          C.c_void_p(gD.ctypes.data), mem, C.byref(gg)))
        results.append((o, gg))
    N.check(lib.tk_synchronize(R.ctx))
    return [({k2: v.copy() for k2, v in o.items()}, np.array(list(gg.pose_twist))) for o, gg in results]


def test_async_host_buffers_match_synchronous():
    R = api.Renderer(0)
    keep = []
    try:
        cam = synth.test_camera(96, 64)
        s = RenderSettings(top_k=3)
        scenes = [synth.random_scene(1500, 32, seed) for seed in (1, 2, 3)]
        grads = []
        for i in range(3):
            gF = pinned(R.lib, (64 * 96 * 32,), np.float32, keep)
            gF[...] = synth.uniform_image((64, 96, 32), 10 + i).astype(np.float32).ravel()
            gC = pinned(R.lib, (64 * 96 * 3,), np.float64, keep)
            gC[...] = synth.uniform_image((64, 96, 3), 20 + i).ravel()
            gD = pinned(R.lib, (64 * 96,), np.float64, keep)
            gD[...] = synth.uniform_image((64, 96), 30 + i).ravel()
            grads.append((gF, gC, gD))
        sync = run_frame(R, scenes, cam, s, grads, N.TK_HOST, keep)
        asyn = run_frame(R, scenes, cam, s, grads, N.TK_HOST_ASYNC, keep)
        for (os_, ts), (oa, ta) in zip(sync, asyn):
            assert (os_["index"] == oa["index"]).all()
            assert (os_["color"] == oa["color"]).all()
            assert (os_["F"] == oa["F"]).all()
            assert (os_["df"] == oa["df"]).all()  # feature backward is bit-deterministic
            np.testing.assert_allclose(oa["gmean"], os_["gmean"], rtol=1e-9, atol=1e-14)
            np.testing.assert_allclose(ta, ts, rtol=1e-9, atol=1e-12)
            assert np.abs(ta).sum() > 0
    finally:
        for p in keep:
            R.lib.tk_host_free(p)
        R.close()


def test_async_double_buffered_upload_keeps_features_and_frames():
    """TK_HOST_ASYNC scene uploads are double-buffered: a geometry-only async upload (feature NULL)
    keeps the current features, and back-to-back frames on alternating buffers all match the
    synchronous path (no frame sees another frame's scene)."""
    cam = synth.test_camera(80, 56)
    s = RenderSettings(top_k=3)
    a = synth.random_scene(1200, 16, 11)
    b = synth.random_scene(1200, 16, 12)
    hybrid = b.copy()
    hybrid.feature = a.feature.copy()  # b's geometry with a's features

    def frame_sync(m):
        R = api.Renderer(0)
        try:
            g = R.render_geometric(m, Pose(), cam, s)
            return g.topk.index.copy(), R.render_feature(m, g.topk)
        finally:
            R.close()

    plan = [(a, True, a), (b, False, hybrid), (b, True, b), (a, True, a), (a, False, a)]
    want = [frame_sync(w) for _, _, w in plan]
    R = api.Renderer(0)
    keep = []
    try:
        lib = R.lib
        cp, cc, cs = to_pose(Pose()), to_camera(cam), to_settings(s)
        P = cam.width * cam.height
        outs = []
        for m, with_feat, _ in plan:
            arrays = (m.mean, m.log_scale, m.rotation, m.opacity_logit, m.color)
            geo = [pinned(lib, x.shape, np.float64, keep) for x in arrays]
            for dst, x in zip(geo, arrays):
                dst[...] = x
            feat = None
            if with_feat:
                feat = pinned(lib, (m.size(), 16), np.float32, keep)
                feat[...] = m.feature
            view = N.tk_scene_view(m.size(), 16, *(x.ctypes.data for x in geo),
                                   feat.ctypes.data if feat is not None else None, 0)
            N.check(lib.tk_scene_upload(R.ctx, C.byref(view), N.TK_HOST_ASYNC))
            idx = pinned(lib, (P * 3,), np.int32, keep)
            F = pinned(lib, (P * 16,), np.float32, keep)
            gout = N.tk_geom_out(N.TK_HOST_ASYNC, None, None, None, idx.ctypes.data, None, None, None, 0, 0)
            N.check(lib.tk_render_geometric(R.ctx, C.byref(cp), C.byref(cc), C.byref(cs), C.byref(gout)))
            N.check(lib.tk_render_feature(R.ctx, None, C.c_void_p(F.ctypes.data), N.TK_HOST_ASYNC))
            outs.append((idx, F))
        N.check(lib.tk_synchronize(R.ctx))
        for i, ((idx, F), (widx, wF)) in enumerate(zip(outs, want)):
            assert (idx == widx.ravel()).all(), i
            assert np.array_equal(F.reshape(wF.shape), wF), i
    finally:
        for p in keep:
            R.lib.tk_host_free(p)
        R.close()

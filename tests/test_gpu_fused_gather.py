"""Fused render_feature + all-gather over peer memory (tk_render_feature_gathered, SURVEY.md
§8(e)): each rank stores its channel slice of every output row straight into every rank's
full-width buffer.  Ranks are simulated from one process with tk_comm_set_peers and run one after
the other (no rank waits on another): every buffer must then equal the unsharded render_feature
bit for bit, since each channel's weighted sum is the same computation whatever the shard."""
import ctypes as C

import numpy as np
import pytest
import torch

from paper_2602_06991_b200 import _native as N
from paper_2602_06991_b200 import api, dist
import scenegen as synth
from paper_2602_06991_b200.types import Pose, RenderSettings

pytestmark = pytest.mark.gpu


def shard(m, world, rank):
    s = m.copy()
    s.feature = dist.shard_features(m.feature, world, rank)
    s.feature_dim = s.feature.shape[1]
    return s


@pytest.mark.parametrize("world,d,k,shape", [(1, 32, 3, (96, 64)), (2, 64, 3, (96, 64)), (4, 128, 4, (80, 72)),
                                             (8, 512, 3, (64, 48)), (2, 64, 8, (50, 40))])
def test_fused_gather_equals_unsharded(world, d, k, shape):
    w, h = shape
    m = synth.random_scene(900, d, 7)
    cam = synth.test_camera(w, h)
    s = RenderSettings(top_k=k)
    full = api.Renderer(0)
    try:
        g = full.render_geometric(m, Pose(), cam, s)
        F = full.render_feature(m, g.topk)
    finally:
        full.close()
    P = w * h
    bufs = [torch.full((P * d,), float("nan"), device="cuda") for _ in range(world)]
    ptrs = [b.data_ptr() for b in bufs]
    for r in range(world):
        R = api.Renderer(0)
        try:
            sm = shard(m, world, r)
            R.comm_set_peers(r, world, d, ptrs, P)
            R.render_geometric(sm, Pose(), cam, s)  # identical records on every rank
            R.render_feature_gathered(sm)
            R.synchronize()
        finally:
            R.close()
    torch.cuda.synchronize()
    for b in bufs:
        assert np.array_equal(b.cpu().numpy().reshape(h, w, d), F)


def test_fused_gather_host_copy_and_errors():
    m = synth.random_scene(300, 16, 3)
    cam = synth.test_camera(48, 32)
    s = RenderSettings()
    R = api.Renderer(0)
    try:
        g = R.render_geometric(m, Pose(), cam, s)
        F = R.render_feature(m, g.topk)
        lib = R.lib
        # no peers registered
        assert lib.tk_render_feature_gathered(R.ctx, None, None, N.TK_HOST) == N.TK_ERR_STATE
        buf = torch.zeros(48 * 32 * 16, device="cuda")
        arr = (C.c_void_p * 1)(buf.data_ptr())
        assert lib.tk_comm_set_peers(R.ctx, 0, 9, 16, arr, 48 * 32) == N.TK_ERR_BAD_ARG   # > 8 ranks
        assert lib.tk_comm_set_peers(R.ctx, 1, 1, 16, arr, 48 * 32) == N.TK_ERR_BAD_ARG   # rank >= nranks
        assert lib.tk_comm_set_peers(R.ctx, 0, 1, 18, arr, 48 * 32) == N.TK_ERR_BAD_ARG   # slice % 4
        N.check(lib.tk_comm_set_peers(R.ctx, 0, 1, 32, arr, 48 * 32))
        assert lib.tk_render_feature_gathered(R.ctx, None, None, N.TK_HOST) == N.TK_ERR_BAD_ARG  # d_total
        N.check(lib.tk_comm_set_peers(R.ctx, 0, 1, 16, arr, 100))
        assert lib.tk_render_feature_gathered(R.ctx, None, None, N.TK_HOST) == N.TK_ERR_BAD_ARG  # too small
        N.check(lib.tk_comm_set_peers(R.ctx, 0, 1, 16, arr, 48 * 32))
        out = np.zeros((32, 48, 16), np.float32)
        N.check(lib.tk_render_feature_gathered(R.ctx, None, out.ctypes.data, N.TK_HOST))
        assert np.array_equal(out, F)
        p = C.c_void_p()
        N.check(lib.tk_comm_gathered_buffer(R.ctx, C.byref(p)))
        assert p.value == buf.data_ptr()
        assert np.array_equal(buf.cpu().numpy().reshape(32, 48, 16), F)
    finally:
        R.close()


def test_p2p_setup_single_rank_nccl():
    """tk_comm_p2p_setup over a one-rank NCCL communicator: the IPC-handle exchange, the buffer
    registration and the NCCL rank barrier of tk_render_feature_gathered; re-setup for a larger frame."""
    m = synth.random_scene(500, 32, 9)
    s = RenderSettings()
    R = api.Renderer(0)
    try:
        lib = R.lib
        uid = (C.c_uint8 * 128)()
        N.check(lib.tk_comm_unique_id(uid))
        N.check(lib.tk_comm_init(R.ctx, uid, 1, 0, 32))
        for w, h in [(40, 30), (72, 56)]:
            cam = synth.test_camera(w, h)
            g = R.render_geometric(m, Pose(), cam, s)
            F = R.render_feature(m, g.topk)
            N.check(lib.tk_comm_p2p_setup(R.ctx, w * h))
            out = np.zeros((h, w, 32), np.float32)
            N.check(lib.tk_render_feature_gathered(R.ctx, None, out.ctypes.data, N.TK_HOST))
            assert np.array_equal(out, F)
    finally:
        R.close()

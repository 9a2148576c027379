"""Multi-rank host logic of the D-sharded path on CPU: world_size 2, gloo, 127.0.0.1.

Each rank gathers its channel slice of the Top-K feature map (host statement of the gather), the
slices are all-gathered over gloo and interleaved exactly as tk_allgather_feature does on the
device, and the result must equal the unsharded gather bit for bit (channels never mix).  The
unique-id broadcast and max-over-ranks timing helpers used by bench.py are exercised too.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2602_06991_b200 import dist as tkdist

import _dist_ref as dref


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _records(P=48, N=40, K=3, seed=0):
    rng = np.random.default_rng(seed)
    count = rng.integers(0, K + 1, size=P).astype(np.uint8)
    index = np.full(P * K, -1, np.int32)
    weight = np.zeros(P * K)
    for p in range(P):
        c = int(count[p])
        index[p * K:p * K + c] = rng.choice(N, size=c, replace=False)
        weight[p * K:p * K + c] = np.sort(rng.uniform(0.01, 1.0, size=c))[::-1]
    feat = rng.standard_normal((N, 12))
    return feat, index, weight, count, K


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        feat, index, weight, count, K = _records()
        mine = tkdist.shard_features(feat, world, rank)
        part = dref.gather_reference(mine, index, weight, count, K)
        parts = [torch.zeros_like(torch.from_numpy(part)) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(part))
        full = tkdist.interleave([p.numpy() for p in parts])
        ref = dref.gather_reference(feat, index, weight, count, K)
        uid = tkdist.broadcast_bytes(dist, bytes(range(128)) if rank == 0 else None, 128)
        tmax = tkdist.max_over_ranks(dist, 1.0 + rank)
        q.put((rank, bool(np.array_equal(full, ref)), uid == bytes(range(128)), tmax))
    finally:
        dist.destroy_process_group()


def _feature_step_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        feat, index, weight, count, K = _records(P=60, N=40, K=3, seed=3)
        rng = np.random.default_rng(7)
        P, D = count.shape[0], feat.shape[1]
        F = rng.standard_normal((P, D))
        gt = rng.standard_normal((P, D))
        gt[::7] = 0.0                      # invalid keyframe rows
        gt[3, : D // 2] = 0.0              # valid only through the other shard's channels
        m0 = rng.standard_normal((feat.shape[0], D)) * 1e-3
        v0 = np.abs(rng.standard_normal((feat.shape[0], D))) * 1e-6
        args = dict(k=K, lam=1.0, lr=1e-2, beta1=0.9, beta2=0.999, eps=1e-8, step=3, d_total=D)

        def amax(x):
            t = torch.from_numpy(np.ascontiguousarray(x))
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return t.numpy()

        def asum(x):
            t = torch.from_numpy(np.ascontiguousarray(x))
            dist.all_reduce(t)
            return t.numpy()

        c0, c1 = tkdist.shard_range(D, world, rank)
        fs, ms, vs, l1 = dref.feature_step_shard(F[:, c0:c1], gt[:, c0:c1], count, index, weight,
                                                   feat=feat[:, c0:c1], m=m0[:, c0:c1], v=v0[:, c0:c1],
                                                   allreduce_max=amax, allreduce_sum=asum, **args)
        parts = [torch.zeros_like(torch.from_numpy(np.ascontiguousarray(fs))) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(np.ascontiguousarray(fs)))
        full_f = np.concatenate([p.numpy() for p in parts], axis=1)
        ref_f, _, _, ref_l1 = dref.feature_step_shard(F, gt, count, index, weight, feat=feat, m=m0, v=v0,
                                                        allreduce_max=lambda x: x, allreduce_sum=lambda x: x, **args)
        q.put((rank, float(np.abs(full_f - ref_f).max()), abs(l1 - ref_l1)))
    finally:
        dist.destroy_process_group()


def test_sharded_feature_step_equals_unsharded():
    """The D-sharded mapping step's exchanges (mask max, |F-F_gt| sum, row-norm sum) reproduce the
    unsharded feature L1 + backward + Adam + renormalisation (world 2, gloo)."""
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_feature_step_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, dmax, dl1 in res:
        assert dmax < 1e-12 and dl1 < 1e-12, (rank, dmax, dl1)


def test_shard_range():
    assert tkdist.shard_range(512, 8, 3) == (192, 256)
    assert tkdist.shard_range(768, 2, 1) == (384, 768)
    with pytest.raises(ValueError):
        tkdist.shard_range(10, 3, 0)


def test_two_rank_feature_shard_allgather_matches_full_render():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, equal, uid_ok, tmax in res:
        assert equal, f"rank {rank}: sharded gather != full gather"
        assert uid_ok
        assert tmax == 2.0


def _band_worker(rank, world, port, q):
    """The geometry split's data flow with the CPU oracle as the per-rank compute: rank r owns the
    pixel rows of its band; records are all-gathered (equal band chunks, the last padded), the
    peak contributions max-reduced, and the geometry gradients of the band-masked upstream
    gradients sum-reduced -- the whole frame's outputs on every rank."""
    import torch
    import torch.distributed as dist

    import _oracle as O
    import scenegen as synth
    from paper_2602_06991_b200.types import Pose, RenderSettings
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = synth.random_scene(120, 4, 9)
        cam = synth.test_camera(40, 36)
        s = RenderSettings(top_k=3, tile_size=8, background=(0.1, 0.2, 0.3))
        W, H, K = cam.width, cam.height, 3
        full = O.render_geometric(m, Pose(), cam, s)
        y0, y1 = tkdist.band_rows(H, s.tile_size, world, rank)
        bp = tkdist.band_rows(H, s.tile_size, world, 0)[1] * W  # pixels per band chunk (padded)
        # this rank's band of records, padded to the chunk
        idx = np.full(bp * K, -1, np.int32)
        idx[:(y1 - y0) * W * K] = full["index"][y0 * W * K:y1 * W * K]
        parts = [torch.zeros(bp * K, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(idx))
        gathered = np.concatenate([p.numpy() for p in parts])[:W * H * K]
        contrib = torch.from_numpy(np.ascontiguousarray(full["contributions"]))
        dist.all_reduce(contrib, op=dist.ReduceOp.MAX)
        gc = synth.uniform_image((H, W, 3), 12)
        gd = synth.uniform_image((H, W), 13)
        mask = np.zeros((H, W))
        mask[y0:y1] = 1.0
        g = O.backward_geometric(m, Pose(), cam, s, gc * mask[..., None], gd * mask)
        mine = torch.from_numpy(np.concatenate([g[f].ravel() for f in ("mean", "log_scale", "rotation",
                                                                        "opacity_logit", "color", "pose_twist")]))
        dist.all_reduce(mine)
        ref = O.backward_geometric(m, Pose(), cam, s, gc, gd)
        refv = np.concatenate([ref[f].ravel() for f in ("mean", "log_scale", "rotation", "opacity_logit", "color",
                                                        "pose_twist")])
        err = float(np.max(np.abs(mine.numpy() - refv) / (np.abs(refv) + 1e-9 * np.abs(refv).max() + 1e-300)))
        q.put((rank, bool(np.array_equal(gathered, full["index"])),
               bool(np.array_equal(contrib.numpy(), full["contributions"])), err))
    finally:
        dist.destroy_process_group()


def test_geometry_split_band_flow_matches_whole_frame():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_band_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, rec_ok, contrib_ok, err in res:
        assert rec_ok and contrib_ok and err < 1e-9, (rank, rec_ok, contrib_ok, err)


def test_band_rows_cover_the_image():
    for H, ts, G in [(680, 16, 8), (480, 16, 3), (36, 8, 2), (10, 32, 4)]:
        rows = [tkdist.band_rows(H, ts, G, b) for b in range(G)]
        assert rows[0][0] == 0 and rows[-1][1] == H
        assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))

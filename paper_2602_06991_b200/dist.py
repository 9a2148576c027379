"""Host-side logic of the feature-dimension sharding.

Every rank holds channels [c0, c1) of every Gaussian's feature and a replica of the geometry; the
integer Top-K records are recomputed identically on every rank (deterministic fp64 path), each rank
gathers / scatters only its slice, and tk_allgather_feature (NCCL) all-gathers the [P][D/G] slices
into the HWC [P][D] map.  This module holds the rank bookkeeping shared by bench.py and the tests;
the device side is in paper_2602_06991_b200/csrc/tk_abi.cu (tk_comm_*, k_interleave).
"""
from __future__ import annotations

import numpy as np


def shard_range(d_total: int, world: int, rank: int) -> tuple[int, int]:
    """Channel slice of `rank`; NCCL all-gather needs equal slices, so D must divide evenly."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    if d_total % world:
        raise ValueError(f"feature dim {d_total} does not split evenly over {world} ranks")
    ds = d_total // world
    return rank * ds, (rank + 1) * ds


def shard_features(features: np.ndarray, world: int, rank: int) -> np.ndarray:
    c0, c1 = shard_range(features.shape[1], world, rank)
    return np.ascontiguousarray(features[:, c0:c1])


def interleave(slices: list[np.ndarray]) -> np.ndarray:
    """[G] x [P][ds] -> [P][G*ds]: the host statement of the device k_interleave after NCCL."""
    return np.concatenate([np.asarray(s) for s in slices], axis=1)


def gather_reference(features: np.ndarray, index: np.ndarray, weight: np.ndarray, count: np.ndarray,
                     k: int) -> np.ndarray:
    """Top-K feature gather on the host (render.cpp:319-334) for small sharding tests."""
    P = count.shape[0]
    out = np.zeros((P, features.shape[1]))
    for p in range(P):
        c = int(count[p])
        if c == 0:
            continue
        w = weight[p * k:p * k + c]
        s = w.sum()
        for j in range(c):
            out[p] += (w[j] / s) * features[index[p * k + j]]
    return out


def broadcast_bytes(dist, payload: bytes | None, nbytes: int, src: int = 0) -> bytes:
    """Broadcast a fixed-size byte string (the NCCL unique id) over an initialised process group."""
    import torch
    t = torch.zeros(nbytes, dtype=torch.uint8)
    if dist.get_rank() == src:
        t[:] = torch.tensor(list(payload), dtype=torch.uint8)
    dist.broadcast(t, src)
    return bytes(t.tolist())


def max_over_ranks(dist, value: float) -> float:
    """Max of a scalar over ranks (the bench's timing rule: slowest rank defines the step)."""
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def feature_step_shard(F, gt, count, index, weight, k, feat, m, v, lam, lr, beta1, beta2, eps, step, d_total,
                       allreduce_max, allreduce_sum):
    """Host statement of the D-sharded feature half of one mapping iteration (tk_optimize_step
    under tk_comm): masked feature L1 (losses.cpp:92-118) on this rank's channel slice, the
    feature backward (backward.cpp:288-319), Adam (optimizer.cpp:49-63) and the row
    renormalisation (mapper.cpp:249) -- with the three exchanges the device path makes: the
    keyframe-row validity mask (max), the |F - F_gt| sum (sum) and the row squared norms (sum).
    F, gt: [P][ds] this rank's channels; feat, m, v: [N][ds].  Returns (feat, m, v, l1_feat)."""
    P = count.shape[0]
    valid = allreduce_max((np.abs(gt) > 0).any(axis=1).astype(np.float64)) > 0
    live = (count > 0) & valid
    feat_n = int(live.sum())
    diff = np.where(live[:, None], F - gt, 0.0)
    abs_sum = allreduce_sum(np.array([np.abs(diff).sum()]))[0]
    inv = 1.0 / (feat_n * d_total) if feat_n else 0.0
    g = np.zeros_like(feat)
    sign = np.sign(diff)
    for p in range(P):
        c = int(count[p])
        if c == 0 or not live[p]:
            continue
        w = weight[p * k:p * k + c]
        s = w.sum()
        for j in range(c):
            g[index[p * k + j]] += (w[j] / s) * sign[p] * (lam * inv)
    m = beta1 * m + (1.0 - beta1) * g
    v = beta2 * v + (1.0 - beta2) * g * g
    f = feat - lr * (m / (1.0 - beta1 ** step)) / (np.sqrt(v / (1.0 - beta2 ** step)) + eps)
    ss = allreduce_sum((f * f).sum(axis=1))
    norm = np.sqrt(ss)
    f = np.where(norm[:, None] > 1e-12, f / np.where(norm > 0, norm, 1.0)[:, None], f)
    return f, m, v, abs_sum * inv

"""Host restatements of the D-sharded data flow (TEST INFRASTRUCTURE ONLY: the checker for the
device path of paper_2602_06991_b200/dist.py + tk_comm_*, never the product)."""
from __future__ import annotations

import numpy as np


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

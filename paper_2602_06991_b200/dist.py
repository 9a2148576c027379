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


def band_rows(height: int, tile_size: int, nbands: int, band: int) -> tuple[int, int]:
    """Pixel rows [y0, y1) swept by `band` under the geometry split (tk_geometry_band): whole tile
    rows, rows_b = ceil(tiles_y / nbands) per band, the last band possibly shorter or empty."""
    tiles_y = (height + tile_size - 1) // tile_size
    rows_b = (tiles_y + nbands - 1) // nbands
    ty0 = min(tiles_y, band * rows_b)
    ty1 = min(tiles_y, ty0 + rows_b)
    return min(height, ty0 * tile_size), min(height, ty1 * tile_size)


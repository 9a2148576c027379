"""Records-per-Gaussian histogram of backward_feature's inverted index (bench recipe scene).

    python scripts/seg_hist.py [n_gaussians width height k]     (GPU; default config 3, K = 3)

Prints the distinct Gaussians, the record count, and how many records sit in segments longer
than 64 / 128 / 256 / 512 / 1024 (the kLongSeg candidates of feature.cuh).
"""
import sys

import numpy as np

import scenegen as synth
from paper_2602_06991_b200.api import Renderer
from paper_2602_06991_b200.types import RenderSettings


def main():
    n, w, h, k = (int(a) for a in (sys.argv[1:5] if len(sys.argv) >= 5 else (1_000_000, 1200, 680, 3)))
    scene, cam, pose, _ = synth.bench_scene(n, w, h, 4)
    r = Renderer(0)
    out = r.render_geometric(scene, pose, cam, RenderSettings(top_k=k))
    idx = out.topk.index.reshape(-1, k)
    cnt = out.topk.count.astype(np.int64)
    valid = np.arange(k)[None, :] < cnt[:, None]
    ids = idx[valid]
    seg = np.bincount(ids, minlength=scene.size())
    nz = seg[seg > 0]
    print(f"n {scene.size()} pixels {w * h} K {k} records {ids.size} distinct {nz.size} "
          f"mean {nz.mean():.1f} max {nz.max()}")
    q = np.percentile(nz, [50, 90, 99, 99.9])
    print("percentiles 50/90/99/99.9:", " ".join(f"{v:.0f}" for v in q))
    for t in (64, 128, 256, 512, 1024):
        long = nz[nz > t]
        print(f"> {t:5d}: {long.size:7d} segments, {long.sum():9d} records ({long.sum() / ids.size:.3f})")


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Run mapping iterations (tk_optimize_step) on the config-3 map for ncu.

  python scripts/map_profile.py [--iters 10] [--config c3]

Iterations 1..iters on one keyframe (feature steps at multiples of 5); prints per-phase times from
the CUDA-event profiler.  Under ncu, pair with --launch-skip to capture the later iterations.
"""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import CONFIGS  # noqa: E402
from paper_2602_06991_b200 import _native as N  # noqa: E402
import scenegen as synth
from paper_2602_06991_b200.api import to_camera, to_pose, to_settings  # noqa: E402
from paper_2602_06991_b200.types import RenderSettings  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--config", default="c3")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    lib, slib = N.render_lib(), synth.N.synth_lib()
    n, W, H, D, K = cfg["n"], cfg["w"], cfg["h"], cfg["d"], cfg["k"]
    P = W * H
    scene, cam, pose, spec = synth.bench_scene(n, W, H, D)
    feat = synth.unit_features(scene.size(), D, 7)
    h = C.c_void_p()
    N.check(lib.tk_create(0, C.byref(h)))
    ctx = h
    geo = [np.ascontiguousarray(a, np.float64) for a in (scene.mean, scene.log_scale, scene.rotation,
                                                          scene.opacity_logit, scene.color)]
    view = N.tk_scene_view(scene.size(), D, *(a.ctypes.data for a in geo), feat.ctypes.data, scene.generation)
    N.check(lib.tk_scene_upload(ctx, C.byref(view), N.TK_HOST))
    col = np.empty(P * 3, np.float32)
    dep = np.empty(P, np.float32)
    gtf = np.empty(P * D, np.float32)
    slib.tk_synth_hash_fill_f32(col.size, 21, 0.0, 1.0, col.ctypes.data)
    slib.tk_synth_hash_fill_f32(dep.size, 22, 0.5, 4.0, dep.ctypes.data)
    slib.tk_synth_hash_fill_f32(gtf.size, 23, -1.0, 1.0, gtf.ctypes.data)
    frame = N.tk_frame_view(W, H, D, col.ctypes.data, dep.ctypes.data, gtf.ctypes.data, N.TK_HOST)
    mc = N.tk_mapper_config()
    lib.tk_default_mapper_config(C.byref(mc))
    N.check(lib.tk_optimizer_reset(ctx, 1))
    N.check(lib.tk_keyframe_set(ctx, 0, C.byref(to_pose(pose)), C.byref(frame)))
    ccam, cset = to_camera(cam), to_settings(RenderSettings(top_k=K))
    N.check(lib.tk_profile_enable(ctx, 1))
    for it in range(1, args.iters + 1):
        vals = (C.c_double * 3)()
        N.check(lib.tk_optimize_step(ctx, C.byref(mc), C.byref(ccam), C.byref(cset), 0, it, vals, None))
        print(f"iter {it}: map {vals[0]:.6f} geo {vals[1]:.6f} feat {vals[2]:.6f}")
    ph_ms = (C.c_double * len(N.PHASES))()
    ph_cnt = (C.c_int64 * len(N.PHASES))()
    N.check(lib.tk_profile_read(ctx, ph_ms, ph_cnt, 1))
    print(json.dumps({nm: [ph_ms[i] / args.iters, int(ph_cnt[i])] for i, nm in enumerate(N.PHASES) if ph_cnt[i]}))
    lib.tk_destroy(ctx)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Device timeline of mapping iterations (or frames) from CUPTI through torch.profiler.

  python scripts/timeline.py [--mode map|frame] [--iters 6] [--out gpurun_out/timeline.txt]

Prints, for the last iteration, every kernel / memcpy / memset on the device in start order with
its duration and the idle gap before it, then totals (busy, idle, largest gaps).  The numbers
are wall-clock on the device (no replay), so gaps from host synchronisation are visible.
"""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import CONFIGS  # noqa: E402
from paper_2602_06991_b200 import _native as N  # noqa: E402
import scenegen as synth
from paper_2602_06991_b200.api import to_camera, to_pose, to_settings  # noqa: E402
from paper_2602_06991_b200.types import Pose, RenderSettings  # noqa: E402


def setup(cfg):
    lib, slib = N.render_lib(), synth.N.synth_lib()
    n, W, H, D, K = cfg["n"], cfg["w"], cfg["h"], cfg["d"], cfg["k"]
    scene, cam, pose, _ = synth.bench_scene(n, W, H, D)
    feat = synth.unit_features(scene.size(), D, 7)
    h = C.c_void_p()
    N.check(lib.tk_create(0, C.byref(h)))
    geo = [np.ascontiguousarray(a, np.float64) for a in (scene.mean, scene.log_scale, scene.rotation,
                                                          scene.opacity_logit, scene.color)]
    view = N.tk_scene_view(scene.size(), D, *(a.ctypes.data for a in geo), feat.ctypes.data, scene.generation)
    N.check(lib.tk_scene_upload(h, C.byref(view), N.TK_HOST))
    return lib, slib, h, scene, cam, pose, (W, H, D, K), (geo, feat)


def e2e_step(lib, ctx, scene, keep, pose, ccam, cset, P, D, K):
    """bench.py's e2e step: pinned host scene and upstream grads in, host outputs back (TK_HOST_ASYNC)."""
    geo, feat = keep
    n = scene.size()
    hold = []

    def pinned(n_el, dt):
        t = torch.empty(n_el, dtype=dt, pin_memory=True)
        hold.append(t)
        return t

    g_pin = [pinned(a.size, torch.float64) for a in geo]
    for t, a in zip(g_pin, geo):
        t.numpy()[...] = a.ravel()
    f_pin = pinned(feat.size, torch.float32)
    f_pin.numpy()[...] = feat.ravel()
    gF, gC, gD = pinned(P * D, torch.float32), pinned(P * 3, torch.float64), pinned(P, torch.float64)
    for t in (gF, gC, gD):
        t.uniform_()
    o = {nm: pinned(sz, dt) for nm, sz, dt in [
        ("color", P * 3, torch.float64), ("depth", P, torch.float64), ("alpha", P, torch.float64),
        ("index", P * K, torch.int32), ("weight", P * K, torch.float64), ("count", P, torch.uint8),
        ("contrib", n, torch.float64), ("F", P * D, torch.float32), ("df", n * D, torch.float32),
        ("gmean", n * 3, torch.float64), ("gls", n * 3, torch.float64), ("grot", n * 4, torch.float64),
        ("gop", n, torch.float64), ("gcol", n * 3, torch.float64)]}
    view = N.tk_scene_view(n, D, *(t.data_ptr() for t in g_pin), f_pin.data_ptr(), 0)
    A = N.TK_HOST_ASYNC
    gout = N.tk_geom_out(A, *(o[x].data_ptr() for x in ("color", "depth", "alpha", "index", "weight", "count",
                                                         "contrib")), 0, 0)
    gg = N.tk_geom_grads(A, *(o[x].data_ptr() for x in ("gmean", "gls", "grot", "gop", "gcol")))
    cp = to_pose(pose)

    def step(it):
        _ = hold
        N.check(lib.tk_invalidate(ctx))
        N.check(lib.tk_scene_upload(ctx, C.byref(view), A))
        N.check(lib.tk_render_geometric(ctx, C.byref(cp), C.byref(ccam), C.byref(cset), C.byref(gout)))
        N.check(lib.tk_render_feature(ctx, None, C.c_void_p(o["F"].data_ptr()), A))
        N.check(lib.tk_backward_feature(ctx, None, C.c_void_p(gF.data_ptr()), A, C.c_void_p(o["df"].data_ptr()), A))
        N.check(lib.tk_backward_geometric(ctx, C.byref(cp), C.byref(ccam), C.byref(cset), C.c_void_p(gC.data_ptr()),
                                          C.c_void_p(gD.data_ptr()), A, C.byref(gg)))
        if it % 5 == 4:
            N.check(lib.tk_synchronize(ctx))
    return step


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="map", choices=["map", "frame", "e2e"])
    ap.add_argument("--iters", type=int, default=6)
    ap.add_argument("--config", default="c3")
    ap.add_argument("--out", default="gpurun_out/timeline.txt")
    args = ap.parse_args()
    lib, slib, ctx, scene, cam, pose, (W, H, D, K), keep = setup(CONFIGS[args.config])
    P = W * H
    ccam, cset = to_camera(cam), to_settings(RenderSettings(top_k=K))
    if args.mode == "map":
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

        def step(it):
            vals = (C.c_double * 3)()
            N.check(lib.tk_optimize_step(ctx, C.byref(mc), C.byref(ccam), C.byref(cset), 0, it, vals, None))
    elif args.mode == "e2e":
        step = e2e_step(lib, ctx, scene, keep, pose, ccam, cset, P, D, K)
    else:
        cp = to_pose(pose)
        gF = torch.rand(P * D, device="cuda", dtype=torch.float32)
        gC = torch.rand(P * 3, device="cuda", dtype=torch.float64)
        gD = torch.rand(P, device="cuda", dtype=torch.float64)
        fo = torch.empty(P * D, device="cuda", dtype=torch.float32)
        dfo = torch.empty(scene.size() * D, device="cuda", dtype=torch.float32)

        def step(it):
            N.check(lib.tk_invalidate(ctx))
            gout = N.tk_geom_out(N.TK_DEVICE, None, None, None, None, None, None, None, 0, 0)
            N.check(lib.tk_render_geometric(ctx, C.byref(cp), C.byref(ccam), C.byref(cset), C.byref(gout)))
            N.check(lib.tk_render_feature(ctx, None, C.c_void_p(fo.data_ptr()), N.TK_DEVICE))
            N.check(lib.tk_backward_feature(ctx, None, C.c_void_p(gF.data_ptr()), N.TK_DEVICE,
                                            C.c_void_p(dfo.data_ptr()), N.TK_DEVICE))
            gg = N.tk_geom_grads(N.TK_DEVICE, None, None, None, None, None)
            N.check(lib.tk_backward_geometric(ctx, C.byref(cp), C.byref(ccam), C.byref(cset),
                                              C.c_void_p(gC.data_ptr()), C.c_void_p(gD.data_ptr()), N.TK_DEVICE,
                                              C.byref(gg)))
            N.check(lib.tk_synchronize(ctx))

    for it in range(1, args.iters):
        step(it)
    torch.cuda.synchronize()
    marks = []
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for it in range(args.iters, args.iters + 5):
            marks.append(len(marks))
            step(it)
        torch.cuda.synchronize()
    tmp = "/tmp/tk_trace.json"
    prof.export_chrome_trace(tmp)
    ev = [e for e in json.load(open(tmp))["traceEvents"]
          if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
    ev.sort(key=lambda e: e["ts"])
    # split into iterations at the project kernel (start of every prepare)
    starts = [i for i, e in enumerate(ev) if "k_project" in e["name"]]
    lo, hi = (starts[-2], starts[-1]) if len(starts) >= 2 else (0, len(ev))
    if args.mode == "map" and len(starts) >= 5:
        lo, hi = starts[-1], len(ev)  # last iteration: a feature step when iters+4 is a multiple of 5
    if args.mode == "e2e":
        lo, hi = 0, len(ev)
    seg = ev[lo:hi]
    lines = []
    t0 = seg[0]["ts"]
    prev_end = t0
    busy = 0.0
    gaps = []
    for e in seg:
        gap = e["ts"] - prev_end
        gaps.append((gap, e["name"][:60]))
        lines.append(f"{e['ts'] - t0:9.1f} {e['dur']:8.1f} gap {gap:7.1f}  s{e['args'].get('stream')} {e['name'][:90]}")
        busy += e["dur"]
        prev_end = max(prev_end, e["ts"] + e["dur"])
    span = prev_end - t0
    streams = {}
    for e in seg:
        streams.setdefault((e["args"].get("stream"), e["cat"]), []).append(e["dur"])
    for (sid, cat), d in sorted(streams.items(), key=lambda x: str(x[0])):
        lines.append(f"stream {sid} {cat}: {len(d)} ops, busy {sum(d):.1f} us of {span:.1f}")
    gaps.sort(reverse=True)
    lines.append(f"span {span:.1f} us, busy (sum of durations) {busy:.1f} us, {len(seg)} device ops")
    lines.append("largest gaps: " + "; ".join(f"{g:.1f} before {n}" for g, n in gaps[:8]))
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    open(args.out, "w").write("\n".join(lines) + "\n")
    print("\n".join(ln for ln in lines if ln.startswith(("span", "stream", "largest"))))
    lib.tk_destroy(ctx)


if __name__ == "__main__":
    main()

"""Timeline of the e2e frame step (TK_HOST_ASYNC): host time per call and main-stream event times."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS  # noqa: E402
from paper_2602_06991_b200 import _native as N, synth  # noqa: E402
from paper_2602_06991_b200.api import to_camera, to_pose, to_settings  # noqa: E402
from paper_2602_06991_b200.types import RenderSettings  # noqa: E402

cfg = CONFIGS["c3"]
lib, slib = N.render_lib(), N.synth_lib()
n, W, H, D, K = cfg["n"], cfg["w"], cfg["h"], cfg["d"], cfg["k"]
P = W * H
scene, cam, pose, spec = synth.bench_scene(n, W, H, D)
feat = synth.unit_features(scene.size(), D, 7)
n = scene.size()
h = C.c_void_p()
N.check(lib.tk_create(0, C.byref(h)))
ctx = h


def pin(a):
    t = torch.empty(a.size, dtype={np.float64: torch.float64, np.float32: torch.float32}[a.dtype.type], pin_memory=True)
    t.numpy()[...] = a.ravel()
    return t


geo = [pin(np.ascontiguousarray(a, np.float64)) for a in (scene.mean, scene.log_scale, scene.rotation,
                                                           scene.opacity_logit, scene.color)]
fp = pin(np.ascontiguousarray(feat, np.float32))
gF = pin(np.random.default_rng(1).uniform(-1, 1, P * D).astype(np.float32))
gC = pin(np.random.default_rng(2).uniform(-1, 1, P * 3))
gD = pin(np.random.default_rng(3).uniform(-1, 1, P))
outs = {k: torch.empty(sz, dtype=dt, pin_memory=True) for k, sz, dt in [
    ("color", P * 3, torch.float64), ("depth", P, torch.float64), ("alpha", P, torch.float64),
    ("index", P * K, torch.int32), ("weight", P * K, torch.float64), ("count", P, torch.uint8),
    ("contrib", n, torch.float64), ("F", P * D, torch.float32), ("df", n * D, torch.float32),
    ("gmean", n * 3, torch.float64), ("gls", n * 3, torch.float64), ("grot", n * 4, torch.float64),
    ("gop", n, torch.float64), ("gcol", n * 3, torch.float64)]}
A = N.TK_HOST_ASYNC
view = N.tk_scene_view(n, D, *(t.data_ptr() for t in geo), fp.data_ptr(), 0)
gout = N.tk_geom_out(A, *(outs[x].data_ptr() for x in ("color", "depth", "alpha", "index", "weight", "count",
                                                       "contrib")), 0, 0)
gg = N.tk_geom_grads(A, *(outs[x].data_ptr() for x in ("gmean", "gls", "grot", "gop", "gcol")))
cp, cc, cs = to_pose(pose), to_camera(cam), to_settings(RenderSettings(top_k=K))
stream = torch.cuda.ExternalStream(lib.tk_get_stream(ctx))
calls = [("invalidate", lambda: lib.tk_invalidate(ctx)),
         ("scene_upload", lambda: lib.tk_scene_upload(ctx, C.byref(view), A)),
         ("render_geometric", lambda: lib.tk_render_geometric(ctx, C.byref(cp), C.byref(cc), C.byref(cs), C.byref(gout))),
         ("render_feature", lambda: lib.tk_render_feature(ctx, None, C.c_void_p(outs["F"].data_ptr()), A)),
         ("backward_feature", lambda: lib.tk_backward_feature(ctx, None, C.c_void_p(gF.data_ptr()), A,
                                                              C.c_void_p(outs["df"].data_ptr()), A)),
         ("backward_geometric", lambda: lib.tk_backward_geometric(ctx, C.byref(cp), C.byref(cc), C.byref(cs),
                                                                  C.c_void_p(gC.data_ptr()), C.c_void_p(gD.data_ptr()),
                                                                  A, C.byref(gg)))]
for _ in range(2):
    for _, f in calls:
        N.check(f())
N.check(lib.tk_synchronize(ctx))
t0 = time.time()
e0 = torch.cuda.Event(enable_timing=True)
e0.record(stream)
rec = []
for step in range(3):
    for name, f in calls:
        th = time.time()
        N.check(f())
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        rec.append((step, name, (time.time() - th) * 1e3, time.time() - t0, ev))
N.check(lib.tk_join(ctx))
ee = torch.cuda.Event(enable_timing=True)
ee.record(stream)
N.check(lib.tk_synchronize(ctx))
print(f"total {e0.elapsed_time(ee):.1f} ms for 3 steps")
for step, name, hms, hat, ev in rec:
    print(f"step {step} {name:20s} host {hms:7.2f} ms  host_at {hat * 1e3:8.1f}  main_at {e0.elapsed_time(ev):8.1f}")

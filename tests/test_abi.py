"""CPU checks of the drop-in boundary: the C-ABI libraries build, load without a GPU and
export every symbol their headers declare (no compute calls here)."""
import ctypes as C
import os
import re

import pytest

from paper_2602_06991_b200 import _native as N
from scenegen import _lib as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER_DIRS = {"tk_render.h": os.path.join(ROOT, "include"), "tk_synth.h": os.path.join(ROOT, "scenegen", "include")}


def declared(header):
    txt = open(os.path.join(HEADER_DIRS[header], header)).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(tk_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2602_06991_b200 import build
    build.build()
    S.build()


@pytest.mark.parametrize("header,path", [("tk_render.h", N.RENDER_LIB), ("tk_synth.h", S.SYNTH_LIB)])
def test_library_exports_every_declared_symbol(header, path):
    lib = C.CDLL(path)
    names = declared(header)
    assert names, header
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_ctypes_bindings_cover_header():
    assert sorted(n for n, _, _ in N.RENDER_SYMBOLS) == declared("tk_render.h")
    assert sorted(n for n, _, _ in S.SYNTH_SYMBOLS) == declared("tk_synth.h")


def test_struct_layouts_match_header(tmp_path):
    """ctypes mirrors must match the C compiler's layout of every POD struct in the headers."""
    structs = {"tk_camera": N.tk_camera, "tk_pose": N.tk_pose, "tk_settings": N.tk_settings,
               "tk_scene_view": N.tk_scene_view, "tk_topk_view": N.tk_topk_view, "tk_geom_out": N.tk_geom_out,
               "tk_geom_grads": N.tk_geom_grads, "tk_device_view": N.tk_device_view,
               "tk_synth_arrays": S.tk_synth_arrays, "tk_synth_spec": S.tk_synth_spec,
               "tk_mapper_config": N.tk_mapper_config, "tk_frame_view": N.tk_frame_view,
               "tk_scene_out": N.tk_scene_out, "tk_source_view": N.tk_source_view}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "tk_render.h"', '#include "tk_synth.h"',
             "int main(void) {"]
    for name, cls in structs.items():
        lines.append(f'printf("{name} %zu\\n", sizeof({name}));')
        for fname, _ in cls._fields_:
            lines.append(f'printf("{name}.{fname} %zu\\n", offsetof({name}, {fname}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    import subprocess
    subprocess.run(["gcc", "-I" + os.path.join(ROOT, "include"), "-I" + HEADER_DIRS["tk_synth.h"], str(src), "-o", str(exe)], check=True)
    got = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True).stdout.splitlines())
    for name, cls in structs.items():
        assert int(got[name]) == C.sizeof(cls), name
        for fname, _ in cls._fields_:
            assert int(got[f"{name}.{fname}"]) == getattr(cls, fname).offset, (name, fname)


def test_default_settings_match_reference():  # render.hpp:14-21
    s = N.tk_settings()
    N.render_lib().tk_default_settings(C.byref(s))
    assert (s.top_k, s.tile_size, s.transmittance_floor, tuple(s.background), s.cov2d_dilation, s.alpha_clamp) == \
        (3, 16, 1e-4, (0.0, 0.0, 0.0), 0.3, 0.999)


def test_default_mapper_config_matches_reference_and_oracle_layout(tmp_path):
    """tk_default_mapper_config == MapperConfig() (losses.hpp, optimizer.hpp, mapper.hpp defaults),
    and tk_mapper_config has the oracle's orc_mapper_config layout field by field."""
    from paper_2602_06991_b200.types import MapperConfig
    import _oracle as O
    cfg = N.tk_mapper_config()
    N.render_lib().tk_default_mapper_config(C.byref(cfg))
    ref = MapperConfig()
    for name, _ in N.tk_mapper_config._fields_:
        assert getattr(cfg, name) == getattr(ref, name), name
    assert [f for f, _ in O.orc_mapper_config._fields_] == [f for f, _ in N.tk_mapper_config._fields_]
    assert C.sizeof(O.orc_mapper_config) == C.sizeof(N.tk_mapper_config)


def test_mt19937_64_matches_the_standard():  # [rand.predef]: 10000th output of default-seeded engine
    from paper_2602_06991_b200.api import MT19937_64
    r = MT19937_64()
    for _ in range(9999):
        r()
    assert r() == 9981545732273789042


def test_create_without_gpu_fails_cleanly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    st = N.render_lib().tk_create(0, C.byref(h))
    assert st != N.TK_OK and not h.value
    assert N.render_lib().tk_last_error()


def test_synth_generators_are_deterministic():
    import scenegen as synth
    a = synth.random_scene(50, 8, 3)
    b = synth.random_scene(50, 8, 3)
    assert (a.mean == b.mean).all() and (a.feature == b.feature).all()
    spec = synth.default_spec(seed=7, spacing=0.2)
    s1, c1 = synth.build_synthetic_scene(spec)
    s2, c2 = synth.build_synthetic_scene(spec)
    assert s1.size() > 0 and (s1.mean == s2.mean).all() and (c1 == c2).all()
    poses = synth.generate_trajectory("orbit", 8, spec)
    assert len(poses) == 8
    f = synth.unit_features(100, 16, 7)
    import numpy as np
    assert np.allclose(np.linalg.norm(f, axis=1), 1.0, atol=1e-6)

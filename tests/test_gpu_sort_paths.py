"""Both radix-sort paths of prepare_scene (onesweep look-back passes and the per-pass histogram +
scan + scatter kept for n >= 2^30 / TK_RADIX_LEGACY=1) give the oracle's PreparedScene exactly,
on a scene large enough for hundreds of sort tiles per pass (long look-back chains)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import _oracle as O
from paper_2602_06991_b200 import api
import scenegen as synth
from paper_2602_06991_b200.types import RenderSettings

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2602_06991_b200 import api
import scenegen as synth
from paper_2602_06991_b200.types import RenderSettings
m, cam, pose, _ = synth.bench_scene(int(sys.argv[3]), 320, 240, 4)
p = api.Renderer(0).prepare_scene(m, pose, cam, RenderSettings())
np.savez(sys.argv[2], e7=p.entries, src=p.src, toff=p.tile_offsets, tent=p.tile_entries)
"""


@pytest.mark.parametrize("n", [150000, 700000])
def test_prepare_onesweep_and_legacy_match_oracle(tmp_path, n):
    m, cam, pose, _ = synth.bench_scene(n, 320, 240, 4)
    s = RenderSettings()
    r = api.Renderer(0)
    try:
        p = r.prepare_scene(m, pose, cam, s)
    finally:
        r.close()
    o = O.prepare_scene(m, pose, cam, s)
    assert (p.src == o["src"]).all() and (p.tile_offsets == o["tile_offsets"]).all()
    assert (p.tile_entries == o["tile_entries"]).all()
    out = tmp_path / "legacy.npz"
    env = dict(os.environ, TK_RADIX_LEGACY="1")
    subprocess.run([sys.executable, "-c", CHILD, ROOT, str(out), str(n)], check=True, env=env, timeout=600)
    q = np.load(out)
    assert (q["src"] == p.src).all() and (q["toff"] == p.tile_offsets).all() and (q["tent"] == p.tile_entries).all()
    assert (q["e7"] == p.entries).all()

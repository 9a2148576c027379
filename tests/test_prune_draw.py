"""prune_map's candidate draw (mapper.cpp:80-139) through tk_prune_draw (host code of the C ABI,
no GPU): the Fenwick draw with its exact rounding-bounded fallback must remove exactly the indices
the reference's sequential scan removes (the oracle's orc_prune_map restates that loop verbatim),
over score distributions that stress ties, zeros, wide magnitudes, the uniform phase after the
mass is exhausted and the "u past the pool's running sum" fallback."""
import ctypes as C
import zlib

import numpy as np
import pytest

import _oracle as O
import scenegen as synth
from paper_2602_06991_b200 import _native as N
from paper_2602_06991_b200.types import MapperConfig


def draw(counts, maxc, keep_ratio, seed, threshold):
    lib = N.render_lib()
    n = counts.size
    out = np.zeros(max(1, n), np.int32)
    nr = C.c_int64()
    N.check(lib.tk_prune_draw(counts.ctypes.data, maxc.ctypes.data, n, keep_ratio, seed, threshold,
                              out.ctypes.data, C.byref(nr)))
    return out[:nr.value].copy()


def oracle_draw(counts, maxc, keep_ratio, seed, threshold):
    m = synth.random_scene(counts.size, 1, 3)
    om = O.OracleMapper(m, MapperConfig())
    om.set_stats(counts, maxc)
    return om.prune(keep_ratio, seed, threshold)


def scores(kind, n, rng):
    if kind == "uniform":
        return rng.random(n)
    if kind == "ties":
        return rng.choice([0.1, 0.2, 0.30000000000000004, 1e-3], n)
    if kind == "zeros":
        return np.where(rng.random(n) < 0.5, 0.0, rng.random(n))
    if kind == "magnitudes":
        return 10.0 ** rng.uniform(-15, 0, n)
    if kind == "few":  # mass exhausted after a handful of draws: uniform phase
        s = np.zeros(n)
        s[rng.choice(n, 7, replace=False)] = rng.random(7)
        return s
    if kind == "dominant":  # one huge score and a sea of tiny ones: running sums far from exact
        s = 10.0 ** rng.uniform(-17, -13, n)
        s[n // 3] = 1.0
        return s
    raise ValueError(kind)


@pytest.mark.parametrize("kind", ["uniform", "ties", "zeros", "magnitudes", "few", "dominant"])
@pytest.mark.parametrize("keep", [0.5, 0.1, 0.97])
def test_prune_draw_matches_reference_scan(kind, keep):
    rng = np.random.default_rng(zlib.crc32(f"{kind}-{keep}".encode()))  # reproducible across processes
    n = 6000
    counts = rng.integers(0, 3, n).astype(np.int32)
    maxc = scores(kind, n, rng)
    for seed, thr in ((11, 0), (12, 1), (13, 5)):
        got = draw(counts, maxc, keep, seed, thr)
        ref = oracle_draw(counts, maxc, keep, seed, thr)
        assert np.array_equal(got, ref), (kind, keep, seed, thr, got.size, ref.size)


def test_prune_draw_edge_cases():
    z = np.zeros(10, np.int32)
    assert draw(z, np.zeros(10), 0.5, 1, 0).size == 0          # zero mass: keep everyone
    assert draw(z + 5, np.ones(10), 0.5, 1, 0).size == 0      # no candidates
    assert draw(z, np.ones(10), 1.0, 1, 0).size == 0          # keep every candidate
    assert draw(np.zeros(0, np.int32), np.zeros(0), 0.5, 1, 0).size == 0
    c = np.zeros(9, np.int32)
    s = np.array([0.5, -0.25, 0.0, 1.0, 0.0, 2.0, 0.1, 0.0, 3.0])  # negative score: the verbatim loop
    assert np.array_equal(draw(c, s, 0.4, 5, 0), oracle_draw(c, s, 0.4, 5, 0))


def test_prune_draw_config3_scale_is_fast():
    """A million candidates (config 3's map): the reference's O(C^2) scan would take hours."""
    import time
    rng = np.random.default_rng(1)
    n = 1_000_000
    counts = np.zeros(n, np.int32)
    maxc = np.where(rng.random(n) < 0.3, rng.random(n), 0.0)
    t0 = time.time()
    removed = draw(counts, maxc, 0.5, 7, 0)
    assert time.time() - t0 < 30.0
    assert removed.size == n - int(np.ceil(0.5 * n)) and np.all(np.diff(removed) > 0)


@pytest.mark.parametrize("scale", ["1e6", "1e14"])
def test_prune_draw_exact_fallback_path(monkeypatch, scale):
    """A widened rounding bound sends many (1e6) or all (1e14) weighted draws through the exact
    fallback scan: still the reference's picks."""
    monkeypatch.setenv("TK_PRUNE_BOUND_SCALE", scale)
    rng = np.random.default_rng(5)
    n = 3000
    counts = np.zeros(n, np.int32)
    for kind in ("uniform", "magnitudes", "dominant", "zeros"):
        maxc = scores(kind, n, rng)
        assert np.array_equal(draw(counts, maxc, 0.5, 9, 0), oracle_draw(counts, maxc, 0.5, 9, 0)), kind

"""The C++ mirror (include/tk/fslam_raster.hpp): compiles on CPU; its reference-style tests run
on the GPU against the CUDA library and the CPU oracle."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2602_06991_b200", "lib")
SYNTH = os.path.join(ROOT, "scenegen")
SRC = os.path.join(ROOT, "tests", "cpp", "test_fslam_raster.cpp")


def _compile(out, syntax_only=False):
    import _oracle
    from scenegen import _lib as S
    _oracle.build()
    S.build()
    cmd = ["g++", "-std=c++17", "-O1", "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(ROOT, "oracle", "include"),
           "-I" + os.path.join(SYNTH, "include"),
           "-I/usr/local/cuda/include", SRC]
    if syntax_only:
        cmd += ["-fsyntax-only"]
    else:
        cmd += ["-o", out, "-L" + LIB, "-ltkrender", "-L" + os.path.join(SYNTH, "lib"), "-ltk_synth",
                "-L" + os.path.join(ROOT, "oracle", "_build"), "-loracle", "-Wl,-rpath," + LIB,
                "-Wl,-rpath," + os.path.join(SYNTH, "lib"), "-Wl,-rpath," + os.path.join(ROOT, "oracle", "_build")]
    subprocess.run(cmd, check=True)


def test_cpp_mirror_compiles():
    _compile(None, syntax_only=True)


@pytest.mark.gpu
def test_cpp_mirror_reference_tests(tmp_path):
    exe = str(tmp_path / "test_fslam_raster")
    _compile(exe)
    res = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(res.stdout)
    assert res.returncode == 0, res.stdout + res.stderr

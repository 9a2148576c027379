"""ctypes binding of scenegen/include/tk_synth.h (libtk_synth.so): the reference's synthetic-input
generators restated in host C++ (testutil.hpp, scene.cpp).  Input synthesis shared by the tests and
both bench arms -- not part of the product library (paper_2602_06991_b200/)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc", "synth.cpp")
HEADER = os.path.join(HERE, "include", "tk_synth.h")
SYNTH_LIB = os.path.join(HERE, "lib", "libtk_synth.so")


class tk_synth_arrays(C.Structure):
    _fields_ = [("n", C.c_int64), ("d", C.c_int32), ("mean", C.c_void_p), ("log_scale", C.c_void_p),
                ("rotation", C.c_void_p), ("opacity_logit", C.c_void_p), ("color", C.c_void_p),
                ("feature", C.c_void_p)]


class tk_synth_spec(C.Structure):
    _fields_ = [("room_min", C.c_double * 3), ("room_max", C.c_double * 3), ("classes", C.c_int32),
                ("feature_dim", C.c_int32), ("spacing", C.c_double), ("jitter", C.c_double),
                ("opacity", C.c_double), ("boxes", C.c_int32), ("seed", C.c_uint64)]


SYNTH_SYMBOLS = [
    ("tk_synth_default_spec", None, [C.POINTER(tk_synth_spec)]),
    ("tk_synth_random_scene", None, [C.c_int32, C.c_int32, C.c_uint64, C.c_double, C.c_double,
                                     C.POINTER(tk_synth_arrays)]),
    ("tk_synth_build_scene", C.c_int64, [C.POINTER(tk_synth_spec), C.POINTER(tk_synth_arrays), C.c_void_p]),
    ("tk_synth_trajectory", C.c_int, [C.c_int32, C.c_int32, C.POINTER(tk_synth_spec), C.c_void_p]),
    ("tk_synth_unit_features", None, [C.c_int64, C.c_int32, C.c_uint64, C.c_void_p, C.c_void_p]),
    ("tk_synth_uniform_fill", None, [C.c_int64, C.c_uint64, C.c_double, C.c_double, C.c_void_p]),
    ("tk_synth_hash_fill_f32", None, [C.c_int64, C.c_uint64, C.c_float, C.c_float, C.c_void_p]),
]

_synth = None


def build(force: bool = False) -> str:
    os.makedirs(os.path.dirname(SYNTH_LIB), exist_ok=True)
    if force or not os.path.exists(SYNTH_LIB) or any(
            os.path.getmtime(f) > os.path.getmtime(SYNTH_LIB) for f in (SRC, HEADER)):
        subprocess.run(["g++", "-O3", "-std=c++17", "-fopenmp", "-fPIC", "-shared", "-I" + os.path.dirname(HEADER),
                        SRC, "-o", SYNTH_LIB], check=True)
    return SYNTH_LIB


def synth_lib():
    global _synth
    if _synth is None:
        if not os.path.exists(SYNTH_LIB):
            raise ImportError(f"{SYNTH_LIB} missing: build it with `python -m scenegen._lib`")
        lib = C.CDLL(SYNTH_LIB)
        for name, res, args in SYNTH_SYMBOLS:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _synth = lib
    return _synth


if __name__ == "__main__":
    print(build(force=True))

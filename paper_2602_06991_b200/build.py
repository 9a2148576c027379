"""Build the native libraries in-tree (nvcc / g++ only; no torch extension machinery).

  lib/libtkrender.so   sm_100a CUDA kernels + the C ABI of include/tk_render.h

The geometry TUs (prepare.cu, geometric.cu) and the loss / optimiser TU (mapping.cu) are compiled with --fmad=false so their fp64
arithmetic rounds like the reference's x86-64 build (no FMA contraction); the feature TU is
fp32 and keeps FMA.  Run:  python -m paper_2602_06991_b200.build
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "lib")
BUILD = os.path.join(ROOT, "build", "native")
INCLUDE = os.path.join(ROOT, "include")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
              "--expt-relaxed-constexpr", "-I" + INCLUDE, "-I" + CSRC]

CUDA_UNITS = [
    ("sort.cu", []),
    ("prepare.cu", ["--fmad=false"]),
    ("geometric.cu", ["--fmad=false"]),
    ("feature.cu", []),
    ("mapping.cu", ["--fmad=false"]),
    ("mapedit.cu", ["--fmad=false"]),
    ("tk_abi.cu", []),
    ("tk_abi_map.cu", []),
    ("tk_abi_io.cu", []),
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _run(cmd: list[str], log) -> None:
    res = subprocess.run(cmd, capture_output=True, text=True)
    log.write(" ".join(cmd) + "\n" + res.stdout + res.stderr + "\n")
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd[:3])} ...")


def _stale(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build(force: bool = False, verbose: bool = False, variant: str | None = None,
          defines: list[str] | None = None) -> dict[str, str]:
    """Compile libtkrender.so.  variant/defines: an A/B build with extra -D flags into
    lib/<variant>/libtkrender.so (loaded through TK_RENDER_LIB; scripts/ab_libs.sh)."""
    global LIB, BUILD
    if variant:
        lib0, build0 = LIB, BUILD
        LIB, BUILD = os.path.join(lib0, variant), os.path.join(build0 + "_" + variant)
        try:
            return _build(force, verbose, ["-D" + d for d in (defines or [])])
        finally:
            LIB, BUILD = lib0, build0
    return _build(force, verbose, [])


def _build(force: bool, verbose: bool, extra_flags: list[str]) -> dict[str, str]:
    os.makedirs(LIB, exist_ok=True)
    os.makedirs(BUILD, exist_ok=True)
    nvcc = _nvcc()
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers += [os.path.join(INCLUDE, f) for f in os.listdir(INCLUDE) if f.endswith(".h")]
    out = {}
    with open(os.path.join(BUILD, "build.log"), "w") as log:
        objs = []
        for src, extra in CUDA_UNITS:
            s = os.path.join(CSRC, src)
            o = os.path.join(BUILD, src.replace(".cu", ".o"))
            if force or _stale(o, [s] + headers):
                _run([nvcc, *ARCH, *NVCC_FLAGS, *extra, *extra_flags, "-c", s, "-o", o], log)
            objs.append(o)
        so = os.path.join(LIB, "libtkrender.so")
        if force or _stale(so, objs):
            _run([nvcc, *ARCH, "-shared", "-Xcompiler", "-fPIC", *objs, "-o", so, "-ldl"], log)
        out["tkrender"] = so
    if verbose:
        print(open(os.path.join(BUILD, "build.log")).read())
    return out


if __name__ == "__main__":
    # python -m paper_2602_06991_b200.build [--force] [-v] [--variant NAME -DFOO ...]
    args = sys.argv[1:]
    var = args[args.index("--variant") + 1] if "--variant" in args else None
    defs = [a[2:] for a in args if a.startswith("-D")]
    print(build(force="--force" in args, verbose="-v" in args, variant=var, defines=defs))

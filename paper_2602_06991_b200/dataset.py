"""FEAT feature-frame files (synth/dataset.cpp:48-76) on the host: "FEAT", uint32 height, width,
channels (little endian), then height * width * channels fp32 in HWC order.  The device path reads
them straight into a keyframe (tk_keyframe_load_features / Renderer.keyframe_load_features)."""
from __future__ import annotations

import struct

import numpy as np

MAGIC = b"FEAT"


def write_feature_bin(path: str, image: np.ndarray) -> None:
    """write_feature_bin (dataset.cpp:48-61): image is H x W x D."""
    img = np.ascontiguousarray(image, np.float32)
    if img.ndim != 3:
        raise ValueError("feature image must be H x W x D")
    h, w, d = img.shape
    try:
        with open(path, "wb") as f:
            f.write(MAGIC + struct.pack("<III", h, w, d) + img.tobytes())
    except OSError as e:
        raise RuntimeError(f"dataset: cannot open {path} for writing") from e


def read_feature_bin(path: str) -> np.ndarray:
    """read_feature_bin (dataset.cpp:63-76), with the reference's error messages."""
    try:
        raw = open(path, "rb").read()
    except OSError as e:
        raise RuntimeError(f"dataset: cannot open {path}") from e
    if raw[:4] != MAGIC:
        raise RuntimeError(f"dataset: bad magic in {path}")
    if len(raw) < 16:
        raise RuntimeError(f"dataset: truncated header in {path}")
    h, w, d = struct.unpack("<III", raw[4:16])
    n = h * w * d * 4
    if len(raw) < 16 + n:
        raise RuntimeError(f"dataset: truncated data in {path}")
    return np.frombuffer(raw[16:16 + n], np.float32).reshape(h, w, d).copy()

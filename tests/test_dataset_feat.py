"""FEAT feature-frame format (synth/dataset.cpp:48-76) on the host: byte layout, round trip and the
reference's error messages."""
import struct

import numpy as np
import pytest

from paper_2602_06991_b200 import dataset


def test_feat_layout_and_round_trip(tmp_path):
    img = np.random.default_rng(3).normal(size=(5, 7, 3)).astype(np.float32)
    p = tmp_path / "000000.feat"
    dataset.write_feature_bin(str(p), img)
    raw = p.read_bytes()
    assert raw[:4] == b"FEAT" and struct.unpack("<III", raw[4:16]) == (5, 7, 3)
    assert raw[16:] == img.tobytes() and len(raw) == 16 + img.size * 4
    assert np.array_equal(dataset.read_feature_bin(str(p)), img)


def test_feat_errors(tmp_path):
    with pytest.raises(RuntimeError, match="dataset: cannot open"):
        dataset.read_feature_bin(str(tmp_path / "missing.feat"))
    bad = tmp_path / "bad.feat"
    bad.write_bytes(b"FEAX" + bytes(12))
    with pytest.raises(RuntimeError, match="dataset: bad magic in"):
        dataset.read_feature_bin(str(bad))
    short = tmp_path / "short.feat"
    short.write_bytes(b"FEAT" + bytes(6))
    with pytest.raises(RuntimeError, match="dataset: truncated header in"):
        dataset.read_feature_bin(str(short))
    trunc = tmp_path / "trunc.feat"
    trunc.write_bytes(b"FEAT" + struct.pack("<III", 2, 2, 2) + bytes(20))
    with pytest.raises(RuntimeError, match="dataset: truncated data in"):
        dataset.read_feature_bin(str(trunc))

"""Reader for the reference's TMAS fixture format (tensorio.py:18-59), test helper."""

from __future__ import annotations

import json
import struct
from pathlib import Path

import numpy as np

_HEADER = struct.Struct("<4sHHQQ8x")
_DT = {0: np.dtype("uint8"), 1: np.dtype("<f4"), 2: np.dtype("<u2")}
GOLDEN = Path(__file__).resolve().parent


def read_tensor(path) -> np.ndarray:
    raw = Path(path).read_bytes()
    magic, tag, version, rows, cols = _HEADER.unpack_from(raw)
    assert magic == b"TMAS" and version == 1, path
    dt = _DT[tag]
    body = raw[_HEADER.size:]
    assert len(body) == rows * cols * dt.itemsize, path
    return np.frombuffer(body, dtype=dt).reshape(rows, cols).copy()


def load_case(name: str) -> dict:
    d = GOLDEN / name
    meta = json.loads((d / "case.json").read_text())
    case = dict(meta)
    case["a_codes"] = read_tensor(d / "a_codes.bin")
    case["a_scales"] = read_tensor(d / "a_scales.bin")
    b = read_tensor(d / "b_codes.bin")
    sb = read_tensor(d / "b_scales.bin")
    if "b_shape" in meta:
        b = b.reshape(meta["b_shape"])
        sb = sb.reshape(meta["sb_shape"])
    case["b_codes"] = b
    case["b_scales"] = sb
    case["c_golden"] = read_tensor(d / "c_golden.bin")
    return case


CASES = ["residual253", "c1", "k640", "ktail", "k1664", "perexpert", "perexpert_t"]

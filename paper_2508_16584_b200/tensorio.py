"""TMAS tensor files and golden-fixture exchange.

The reference's flat binary format (tensorio.py:1-59): a 32-byte little-endian
header -- magic ``TMAS``, uint16 dtype tag, uint16 version 1, uint64 rows,
uint64 cols, 8 reserved bytes -- then the row-major payload.  Tags: 0 = uint8
(FP8 codes), 1 = float32 (scales), 2 = uint16 (bf16 output bits).

``read_tensor`` / ``write_tensor`` keep the reference's names, numpy types and
InvalidInput errors, byte for byte (tests/test_tensorio.py replays the files the
reference wrote).  ``load_tensor`` / ``save_tensor`` move a file straight
between disk and HBM through a pinned staging buffer, so large configs' operands
never take a pageable numpy detour.  ``write_fixture`` / ``read_fixture`` use the
directory layout of the reference's make_golden_fixture.py:39-50 (five .bin
files plus a key=value config.txt), extended with ``b_shape`` for per-expert B.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from .errors import ConfigError, InvalidInput

MAGIC = b"TMAS"
VERSION = 1
_HEADER = struct.Struct("<4sHHQQ8x")
HEADER_BYTES = _HEADER.size  # 32

_TAG_FOR_DTYPE = {np.dtype("uint8"): 0, np.dtype("<f4"): 1, np.dtype("<u2"): 2}
_DTYPE_FOR_TAG = {v: k for k, v in _TAG_FOR_DTYPE.items()}
# torch dtypes a device tensor may carry for each tag (the first one is what load_tensor returns)
_TORCH_FOR_TAG = {0: (torch.uint8, torch.float8_e4m3fn, torch.int8), 1: (torch.float32,),
                  2: (torch.uint16, torch.bfloat16, torch.int16, torch.float16)}


def write_tensor(path, arr: np.ndarray) -> None:
    """tensorio.py:30-40: 2-D uint8 / float32 / uint16 array -> TMAS file."""
    arr = np.ascontiguousarray(arr)
    if arr.ndim != 2:
        raise InvalidInput(f"only 2-D tensors are serialized, got ndim={arr.ndim}")
    dt = arr.dtype.newbyteorder("<")
    if dt not in _TAG_FOR_DTYPE:
        raise InvalidInput(f"unsupported dtype {arr.dtype}")
    with open(path, "wb") as f:
        f.write(_HEADER.pack(MAGIC, _TAG_FOR_DTYPE[dt], VERSION, arr.shape[0], arr.shape[1]))
        f.write(arr.astype(dt, copy=False).tobytes())


def _parse_header(path, raw: bytes, size: int):
    """tensorio.py:44-58 checks, in the same order: header, magic, version, tag, payload size."""
    if len(raw) < HEADER_BYTES:
        raise InvalidInput(f"{path}: truncated header")
    magic, tag, version, rows, cols = _HEADER.unpack_from(raw)
    if magic != MAGIC:
        raise InvalidInput(f"{path}: bad magic {magic!r}")
    if version != VERSION:
        raise InvalidInput(f"{path}: unsupported version {version}")
    if tag not in _DTYPE_FOR_TAG:
        raise InvalidInput(f"{path}: unknown dtype tag {tag}")
    need = rows * cols * _DTYPE_FOR_TAG[tag].itemsize
    if size - HEADER_BYTES != need:
        raise InvalidInput(f"{path}: payload is {size - HEADER_BYTES} bytes, expected {need}")
    return tag, rows, cols


def read_tensor(path) -> np.ndarray:
    """tensorio.py:43-59: TMAS file -> a fresh 2-D numpy array."""
    raw = Path(path).read_bytes()
    tag, rows, cols = _parse_header(path, raw, len(raw))
    return np.frombuffer(raw, dtype=_DTYPE_FOR_TAG[tag], offset=HEADER_BYTES).reshape(rows, cols).copy()


def load_tensor(path, device="cuda", *, dtype: torch.dtype | None = None) -> torch.Tensor:
    """TMAS file -> 2-D tensor on ``device``, read into pinned memory and copied stream-ordered.

    ``dtype`` reinterprets the payload (same element size): e.g. torch.float8_e4m3fn for
    codes or torch.bfloat16 for output bits.  Default: uint8 / float32 / uint16 by tag.
    """
    path = Path(path)
    with open(path, "rb") as f:
        head = f.read(HEADER_BYTES)
        tag, rows, cols = _parse_header(path, head, path.stat().st_size)
        want = _TORCH_FOR_TAG[tag][0] if dtype is None else dtype
        if want not in _TORCH_FOR_TAG[tag]:
            raise InvalidInput(f"{path}: tag {tag} payload cannot be viewed as {want}")
        nbytes = rows * cols * _DTYPE_FOR_TAG[tag].itemsize
        dev = torch.device(device)
        host = torch.empty(nbytes, dtype=torch.uint8, pin_memory=dev.type == "cuda")
        if nbytes and f.readinto(memoryview(host.numpy())) != nbytes:
            raise InvalidInput(f"{path}: short read")
    return host.to(dev, non_blocking=True).view(want).view(rows, cols)


def save_tensor(path, t: torch.Tensor) -> None:
    """2-D tensor (any device) -> TMAS file; the tag follows the element type (see _TORCH_FOR_TAG)."""
    if t.dim() != 2:
        raise InvalidInput(f"only 2-D tensors are serialized, got ndim={t.dim()}")
    tag = next((g for g, dts in _TORCH_FOR_TAG.items() if t.dtype in dts), None)
    if tag is None:
        raise InvalidInput(f"unsupported dtype {t.dtype}")
    rows, cols = t.shape
    flat = t.contiguous().view(-1).view(torch.uint8)
    host = torch.empty(flat.numel(), dtype=torch.uint8, pin_memory=t.is_cuda)
    host.copy_(flat)  # synchronous D2H: the bytes are on the host before the write
    with open(path, "wb") as f:
        f.write(_HEADER.pack(MAGIC, tag, VERSION, rows, cols))
        f.write(memoryview(host.numpy()))


# --------------------------------------------------------------------------------------------
# golden fixtures (make_golden_fixture.py:39-50)

FIXTURE_FILES = ("a_codes.bin", "a_scales.bin", "b_codes.bin", "b_scales.bin", "c_golden.bin")


@dataclass
class Fixture:
    """One golden case: operands, the expected bf16 bits and the problem shape."""

    a_codes: np.ndarray         # u8 [M, K]
    a_scales: np.ndarray        # f32 [M, kb]
    b_codes: np.ndarray         # u8 [K, N] shared, or [G, K, N] / [G, N, K] per expert
    b_scales: np.ndarray        # f32 [kb, nb] or [G, kb, nb] / [G, nb, kb]
    c_golden: np.ndarray        # u16 [M, N]
    n: int
    k: int
    group_sizes: tuple[int, ...]
    seed: int = 0
    b_layout: str = "kn"        # "kn" (reference) or "nk" (K-major, dgrad)


def parse_config_file(path) -> dict[str, str]:
    """cli.py:70-84: ``key = value`` lines, ``#`` comments; ConfigError on a malformed line."""
    out: dict[str, str] = {}
    try:
        text = Path(path).read_text()
    except OSError as e:
        raise ConfigError(f"cannot read config {path}: {e}") from e
    for ln, line in enumerate(text.splitlines(), 1):
        line = line.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise ConfigError(f"{path}:{ln}: expected key=value, got {line!r}")
        key, val = line.split("=", 1)
        out[key.strip()] = val.strip()
    return out


def _ints(cfg: dict[str, str], key: str) -> tuple[int, ...]:
    try:
        return tuple(int(x) for x in cfg[key].split(",") if x.strip())
    except (KeyError, ValueError) as e:
        raise ConfigError(f"config key {key!r} missing or not a comma list of ints") from e


def write_fixture(out_dir, fx: Fixture, *, comment: str = "golden case") -> None:
    """Write the reference's fixture layout; per-expert B is stored as its 2-D [G*K, N] view."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    b, sb = np.asarray(fx.b_codes), np.asarray(fx.b_scales)
    write_tensor(out / "a_codes.bin", fx.a_codes)
    write_tensor(out / "a_scales.bin", fx.a_scales)
    write_tensor(out / "b_codes.bin", b.reshape(-1, b.shape[-1]))
    write_tensor(out / "b_scales.bin", sb.reshape(-1, sb.shape[-1]))
    write_tensor(out / "c_golden.bin", fx.c_golden)
    lines = [f"# {comment}", f"n = {fx.n}", f"k = {fx.k}",
             f"group_sizes = {','.join(str(g) for g in fx.group_sizes)}", f"seed = {fx.seed}"]
    if b.ndim == 3:
        lines += [f"b_layout = {fx.b_layout}", f"b_shape = {','.join(map(str, b.shape))}",
                  f"sb_shape = {','.join(map(str, sb.shape))}"]
    (out / "config.txt").write_text("\n".join(lines) + "\n")


def read_fixture(in_dir) -> Fixture:
    """Read a fixture directory written by write_fixture or by make_golden_fixture.py."""
    d = Path(in_dir)
    cfg = parse_config_file(d / "config.txt")
    (n,), (k,) = _ints(cfg, "n"), _ints(cfg, "k")
    arrs = {name[:-4]: read_tensor(d / name) for name in FIXTURE_FILES}
    b, sb = arrs["b_codes"], arrs["b_scales"]
    if "b_shape" in cfg:
        b = b.reshape(_ints(cfg, "b_shape"))
        sb = sb.reshape(_ints(cfg, "sb_shape"))
    gs = _ints(cfg, "group_sizes")
    fx = Fixture(a_codes=arrs["a_codes"], a_scales=arrs["a_scales"], b_codes=b, b_scales=sb,
                 c_golden=arrs["c_golden"], n=n, k=k, group_sizes=gs, seed=int(cfg.get("seed", 0)),
                 b_layout=cfg.get("b_layout", "kn"))
    m = sum(gs)
    if fx.a_codes.shape != (m, k) or fx.c_golden.shape != (m, n):
        raise InvalidInput(f"{d}: A {fx.a_codes.shape} / C {fx.c_golden.shape} do not match M={m}, N={n}, K={k}")
    return fx

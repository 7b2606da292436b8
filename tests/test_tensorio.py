"""TMAS files and fixture exchange (paper_2508_16584_b200/tensorio.py).

The byte-level pin: every .bin under tests/golden/ was written by the
reference's own write_tensor (tests/golden/make_golden.py), so reading each and
writing it back must reproduce the file byte for byte.  The rest follows the
reference's test_tensorio.py (round trip, 32-byte header, rejects) plus the
device loader and the fixture directory round trip.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2508_16584_b200 import tensorio as tio
from paper_2508_16584_b200.errors import ConfigError, InvalidInput
from tmas import CASES, GOLDEN, load_case

BINS = ["a_codes.bin", "a_scales.bin", "b_codes.bin", "b_scales.bin", "c_golden.bin"]


@pytest.mark.parametrize("name", CASES)
def test_reference_written_files_round_trip_byte_for_byte(name, tmp_path):
    for f in BINS:
        src = GOLDEN / name / f
        arr = tio.read_tensor(src)
        tio.write_tensor(tmp_path / f, arr)
        assert (tmp_path / f).read_bytes() == src.read_bytes(), (name, f)


@pytest.mark.parametrize("dtype", [np.uint8, np.float32, np.uint16])
def test_round_trip(tmp_path, dtype):
    arr = np.random.default_rng(0).integers(0, 200, size=(7, 13)).astype(dtype)
    tio.write_tensor(tmp_path / "t.bin", arr)
    back = tio.read_tensor(tmp_path / "t.bin")
    assert back.dtype == np.dtype(dtype) and np.array_equal(back, arr)


def test_header_is_32_bytes_little_endian(tmp_path):
    tio.write_tensor(tmp_path / "t.bin", np.zeros((3, 5), dtype=np.uint8))
    raw = (tmp_path / "t.bin").read_bytes()
    assert raw[:4] == tio.MAGIC and len(raw) == 32 + 15
    assert int.from_bytes(raw[8:16], "little") == 3 and int.from_bytes(raw[16:24], "little") == 5


def test_rejects_bad_inputs(tmp_path):
    p = tmp_path / "t.bin"
    with pytest.raises(InvalidInput):
        tio.write_tensor(p, np.zeros(4, dtype=np.uint8))
    with pytest.raises(InvalidInput):
        tio.write_tensor(p, np.zeros((2, 2), dtype=np.int64))
    tio.write_tensor(p, np.zeros((2, 2), dtype=np.float32))
    good = p.read_bytes()
    bad = {"magic.bin": b"XXXX" + good[4:], "short.bin": good[:10], "trunc.bin": good[:-4],
           "version.bin": good[:6] + b"\x02\x00" + good[8:], "tag.bin": good[:4] + b"\x07\x00" + good[6:]}
    for name, raw in bad.items():
        (tmp_path / name).write_bytes(raw)
        with pytest.raises(InvalidInput):
            tio.read_tensor(tmp_path / name)
        with pytest.raises(InvalidInput):
            tio.load_tensor(tmp_path / name, "cpu")


def test_load_and_save_tensor_host_device_path(tmp_path):
    """load_tensor/save_tensor on the CPU device: same bytes, dtype views by tag."""
    src = GOLDEN / "c1" / "c_golden.bin"
    t = tio.load_tensor(src, "cpu")
    assert t.dtype == torch.uint16 and np.array_equal(t.numpy(), tio.read_tensor(src))
    tb = tio.load_tensor(src, "cpu", dtype=torch.bfloat16)
    assert tb.dtype == torch.bfloat16
    tio.save_tensor(tmp_path / "c.bin", tb)
    assert (tmp_path / "c.bin").read_bytes() == src.read_bytes()
    codes = tio.load_tensor(GOLDEN / "c1" / "a_codes.bin", "cpu", dtype=torch.float8_e4m3fn)
    tio.save_tensor(tmp_path / "a.bin", codes)
    assert (tmp_path / "a.bin").read_bytes() == (GOLDEN / "c1" / "a_codes.bin").read_bytes()
    with pytest.raises(InvalidInput):
        tio.load_tensor(src, "cpu", dtype=torch.float32)  # tag 2 is 2-byte
    with pytest.raises(InvalidInput):
        tio.save_tensor(tmp_path / "x.bin", torch.zeros(3, dtype=torch.float32))
    with pytest.raises(InvalidInput):
        tio.save_tensor(tmp_path / "x.bin", torch.zeros((2, 2), dtype=torch.int64))


@pytest.mark.parametrize("name", ["residual253", "perexpert", "perexpert_t"])
def test_fixture_directory_round_trip(name, tmp_path):
    c = load_case(name)
    layout = "nk" if c.get("b_layout") == "expert_nk" else "kn"
    fx = tio.Fixture(a_codes=c["a_codes"], a_scales=c["a_scales"], b_codes=c["b_codes"], b_scales=c["b_scales"],
                     c_golden=c["c_golden"], n=c["n"], k=c["k"], group_sizes=tuple(c["group_sizes"]),
                     seed=c["seed"], b_layout=layout)
    tio.write_fixture(tmp_path / name, fx)
    for f in BINS:  # the operand files are the reference's bytes
        assert (tmp_path / name / f).read_bytes() == (GOLDEN / name / f).read_bytes(), f
    back = tio.read_fixture(tmp_path / name)
    assert (back.n, back.k, back.group_sizes, back.seed, back.b_layout) == (fx.n, fx.k, fx.group_sizes, fx.seed, layout)
    for f in ("a_codes", "a_scales", "b_codes", "b_scales", "c_golden"):
        assert np.array_equal(getattr(back, f), getattr(fx, f)), f


def test_reads_the_reference_fixture_config_format(tmp_path):
    """make_golden_fixture.py:45-50 writes a commented key=value config.txt with one group."""
    d = tmp_path / "residual253"
    d.mkdir()
    for f in BINS:
        (d / f).write_bytes((GOLDEN / "residual253" / f).read_bytes())
    (d / "config.txt").write_text("# canonical residual-store case: one group of 253 rows\n"
                                  "n = 128\nk = 128\ngroup_sizes = 253\nseed = 0\n")
    fx = tio.read_fixture(d)
    assert fx.group_sizes == (253,) and fx.a_codes.shape == (253, 128) and fx.b_codes.shape == (128, 128)
    (d / "config.txt").write_text("n = 128\nk 128\n")
    with pytest.raises(ConfigError):
        tio.read_fixture(d)
    (d / "config.txt").write_text("n = 128\nk = 128\ngroup_sizes = 250\n")
    with pytest.raises(InvalidInput):
        tio.read_fixture(d)

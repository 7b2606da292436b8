"""Fixture replay on the GPU: TMAS files -> HBM (tensorio.load_tensor) -> grouped GEMM -> TMAS file.

The written output is compared with the reference-written c_golden.bin under
helpers.REL_TOL (the add order inside a k-block differs from the reference).
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2508_16584_b200 as tg
from helpers import assert_parity
from tmas import CASES, GOLDEN, load_case

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", CASES)
def test_replay_fixture_from_files(name, tmp_path):
    case = load_case(name)
    d = GOLDEN / name
    layout = "nk" if case.get("b_layout") == "expert_nk" else "kn"
    a = tg.load_tensor(d / "a_codes.bin", "cuda", dtype=torch.float8_e4m3fn)
    sa = tg.load_tensor(d / "a_scales.bin", "cuda")
    b = tg.load_tensor(d / "b_codes.bin", "cuda", dtype=torch.float8_e4m3fn)
    sb = tg.load_tensor(d / "b_scales.bin", "cuda")
    if "b_shape" in case:
        b = b.view(*case["b_shape"])
        sb = sb.view(*case["sb_shape"])
    gs = torch.tensor(case["group_sizes"], dtype=torch.int32, device="cuda")
    c = tg.grouped_gemm_fp8(a, sa, b, sb, gs, b_layout=layout)
    m = sum(case["group_sizes"])
    tg.save_tensor(tmp_path / "c_adaptive.bin", c[:m])
    got = tg.read_tensor(tmp_path / "c_adaptive.bin")
    assert got.dtype == np.uint16 and got.shape == case["c_golden"].shape
    assert_parity(got, case["c_golden"], label=name)

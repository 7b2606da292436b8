#!/usr/bin/env python3
"""Regenerate the golden fixtures under tests/golden/ from the REFERENCE itself.

This script is test infrastructure. It imports the read-only reference package
``tma_sim`` (path from ``$TMA_SIM_REF``, default ``/root/reference/pkg/src``)
and runs its own ``run_adaptive`` / ``run_padded_baseline``
(``engine.py:184-343`` / ``:346-402``) on fixed seeded cases.  It writes the
operands and the expected bf16 output bits in the reference's own ``TMAS``
tensor file format (``tensorio.py:18-59``).  The GPU box never runs this
script: ``/root/reference`` does not exist there.  Only its outputs, committed
in this directory, travel.

Cases (each a directory with a_codes/a_scales/b_codes/b_scales/c_golden .bin
plus case.json):

* residual253  -- the reference's canonical fixture
                  (``scripts/make_golden_fixture.py:31-50``).  The sha256 values
                  are pinned in SURVEY.md Appendix A and re-checked here.
* c1           -- BASELINE.json configs[0]: M_g = {1, 67, 128, 255}, N=256, K=512.
* k640         -- K=640 gives 20-byte scale rows, so the over-fetch has
                  row_prev != 0 (``prefetch.py:50-72``).  N=192 adds a narrow tail
                  column tile.
* ktail        -- K=208 leaves an 80-wide tail k-block; it includes an empty group.
* k1664        -- K=1664 (13 scale columns, ``test_acceptance.py:168``).
* perexpert    -- a per-expert B [G,K,N].  The reference supports only a shared B
                  (``engine.py:137``).  The golden is a loop of single-group
                  reference calls, one per expert.
* perexpert_t  -- the same with B stored K-major [G,N,K] (dgrad layout).  Only the
                  storage differs; the math is identical.

plans.json pins the host planners.  It holds format_plan strings, DescriptorPool
selections, plan_prefetch windows, account() reports and generate_group_sizes
draws, all computed by the reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

import numpy as np

REF = os.environ.get("TMA_SIM_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from tma_sim.cli import golden_case, random_operands  # noqa: E402
from tma_sim.descriptors import format_plan, plan_group_stores, plan_two_phase, pool_heights  # noqa: E402
from tma_sim.engine import (  # noqa: E402
    GroupedOperands,
    ProblemConfig,
    run_adaptive,
    run_padded_baseline,
    verify_bitwise,
)
from tma_sim.fp8 import Fp8Tensor  # noqa: E402
from tma_sim.prefetch import plan_prefetch  # noqa: E402
from tma_sim.tensorio import write_tensor  # noqa: E402
from tma_sim.workload import account, generate_group_sizes  # noqa: E402

OUT = Path(__file__).resolve().parent

SURVEY_SHA256 = {
    "a_codes.bin": "f1ee649821c385c950ea8a44ebf88acfeabfbbebd2d87ce9f80c842caec21d40",
    "a_scales.bin": "4ea4eb308de7c5919780939f7be88c5e04c833b9cc1523be5e113c2de151273f",
    "b_codes.bin": "2e0c0943f8e234cdf17f684a0bcf17a159766436d8273939988c458376e4933c",
    "b_scales.bin": "761ec4e0a7e023d0892eb83aed9cf8892cb2dc5166e7d80626c55033e5d10d88",
    "c_golden.bin": "65f249eaa68a96b04c6fc6c11171b956e157da7d3046ec9be881863024ffec75",
}


def _write_case(name, config, operands, c_bits, extra=None, b3=None, sb3=None):
    d = OUT / name
    d.mkdir(parents=True, exist_ok=True)
    write_tensor(d / "a_codes.bin", operands.a_codes.codes)
    write_tensor(d / "a_scales.bin", operands.a_scales)
    if b3 is None:
        write_tensor(d / "b_codes.bin", operands.b_codes.codes)
        write_tensor(d / "b_scales.bin", operands.b_scales)
    else:
        # per-expert: stack experts along rows, shapes recorded in case.json
        write_tensor(d / "b_codes.bin", b3.reshape(-1, b3.shape[-1]))
        write_tensor(d / "b_scales.bin", sb3.reshape(-1, sb3.shape[-1]))
    write_tensor(d / "c_golden.bin", c_bits)
    meta = {
        "n": config.n,
        "k": config.k,
        "group_sizes": list(config.group_sizes),
        "block_m": config.block_m,
        "block_n": config.block_n,
        "plan": format_plan(plan_group_stores(config.group_sizes, config.block_m)),
    }
    if extra:
        meta.update(extra)
    (d / "case.json").write_text(json.dumps(meta, indent=1) + "\n")


def _shared_case(name, n, k, sizes, seed):
    config = ProblemConfig(n=n, k=k, group_sizes=tuple(sizes))
    ops = random_operands(config, seed)
    run = run_adaptive(config, ops)
    base = run_padded_baseline(config, ops)
    assert verify_bitwise(run.c_bits, base).equal
    _write_case(name, config, ops, run.c_bits, {"seed": seed, "b_layout": "shared_kn"})
    return config, ops, run.c_bits


def _per_expert_case(name, n, k, sizes, seed, kmajor=False):
    """Per-expert oracle: one single-group reference call per expert."""
    cfg_all = ProblemConfig(n=n, k=k, group_sizes=tuple(sizes))
    ops_all = random_operands(cfg_all, seed)  # A and S_A for all rows
    offs = cfg_all.row_offsets()
    kb, nb = cfg_all.k_blocks, cfg_all.n_scale_blocks
    b3 = np.empty((len(sizes), k, n), dtype=np.uint8)
    sb3 = np.empty((len(sizes), kb, nb), dtype=np.float32)
    c = np.zeros((cfg_all.m_total, n), dtype=np.uint16)
    for g, rows in enumerate(sizes):
        # each expert draws its own B from a distinct seed
        cfg_b = ProblemConfig(n=n, k=k, group_sizes=(1,))
        ops_b = random_operands(cfg_b, seed * 1000 + 17 + g)
        b3[g] = ops_b.b_codes.codes
        sb3[g] = ops_b.b_scales
        if rows == 0:
            continue
        cfg_g = ProblemConfig(n=n, k=k, group_sizes=(rows,))
        off = offs[g]
        ops_g = GroupedOperands(
            Fp8Tensor(ops_all.a_codes.codes[off : off + rows]),
            np.ascontiguousarray(ops_all.a_scales[off : off + rows]),
            Fp8Tensor(b3[g]),
            sb3[g],
        )
        c[off : off + rows] = run_adaptive(cfg_g, ops_g).c_bits
    extra = {"seed": seed, "b_layout": "expert_nk" if kmajor else "expert_kn"}
    if kmajor:
        b3s = np.ascontiguousarray(np.transpose(b3, (0, 2, 1)))  # [G, N, K]
        sb3s = np.ascontiguousarray(np.transpose(sb3, (0, 2, 1)))  # [G, nb, kb]
    else:
        b3s, sb3s = b3, sb3
    extra["b_shape"] = list(b3s.shape)
    extra["sb_shape"] = list(sb3s.shape)
    _write_case(name, cfg_all, ops_all, c, extra, b3=b3s, sb3=sb3s)


def main() -> int:
    # 1. the reference's canonical fixture, byte for byte
    config, ops = golden_case(0)
    run = run_adaptive(config, ops)
    assert verify_bitwise(run.c_bits, run_padded_baseline(config, ops)).equal
    _write_case("residual253", config, ops, run.c_bits, {"seed": 0, "b_layout": "shared_kn"})
    for fname, want in SURVEY_SHA256.items():
        got = hashlib.sha256((OUT / "residual253" / fname).read_bytes()).hexdigest()
        if got != want:
            raise SystemExit(f"residual253/{fname}: sha256 {got} != pinned {want}")

    _shared_case("c1", 256, 512, (1, 67, 128, 255), 0)
    _shared_case("k640", 192, 640, (5, 130, 37, 0, 200), 7)
    _shared_case("ktail", 64, 208, (3, 0, 129), 11)
    _shared_case("k1664", 128, 1664, (77, 130), 13)
    _per_expert_case("perexpert", 128, 384, (70, 0, 131, 128), 5)
    _per_expert_case("perexpert_t", 256, 256, (200, 1, 64), 6, kmajor=True)

    # host-planner pins
    plans = {}
    plans["format_plan"] = {
        "253": format_plan(plan_group_stores((253,), 128)),
        "253,256,0,40": format_plan(plan_group_stores((253, 256, 0, 40), 128)),
        "1,67,128,255": format_plan(plan_group_stores((1, 67, 128, 255), 128)),
    }
    plans["two_phase_128"] = []
    for rows in range(0, 513):
        p = plan_two_phase(rows, 128)
        plans["two_phase_128"].append(
            None
            if p is None
            else [p.residual_rows, p.desc_rows, p.phase_a.smem_row, p.phase_a.gmem_row,
                  p.phase_b.smem_row, p.phase_b.gmem_row]
        )
    plans["pool_heights"] = {str(b): pool_heights(b) for b in (1, 2, 64, 128, 256)}
    pre = []
    for rb in (4, 8, 16, 20, 48, 52, 64, 96, 128, 224, 256):
        for row in (0, 1, 2, 3, 5, 7, 13, 127, 128, 253, 1000, 4097):
            w = plan_prefetch(row * rb, rb, 128)
            pre.append([rb, row, w.start_addr, w.row_prev, w.row_next, w.total_rows])
    plans["prefetch"] = pre
    acc = []
    for sizes, n, k in (
        ((1, 67, 128, 255), 256, 512),
        ((253, 256, 1, 0), 256, 128),
        ((5, 130, 37, 0, 200), 192, 640),
    ):
        r = account(sizes, n, k)
        acc.append([list(sizes), n, k, r.m_total, r.padded_rows, r.bytes_actual, r.bytes_padded,
                    r.saving_pct, r.eliminated_traffic_bytes, r.residual_store_ops])
    plans["account"] = acc
    gen = []
    for m, g, s in ((32768, 32, 0), (8192, 32, 5000), (65536, 4, 3), (100, 8, 1), (5, 8, 2)):
        gen.append([m, g, s, [int(x) for x in generate_group_sizes(m, g, s)]])
    plans["generate_group_sizes"] = gen
    (OUT / "plans.json").write_text(json.dumps(plans) + "\n")
    print(f"wrote golden fixtures under {OUT}")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())

"""Host planners: the reference's descriptor-pool, two-phase and prefetch API.

These functions have the same names, arguments and errors as the reference's
planning layer (descriptors.py, prefetch.py, workload.py).  The arithmetic runs
in libtagg.so (csrc/tagg_plan.cpp), the same geometry the kernel applies on
the device.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from ._lib import lib
from .errors import raise_for_status

GUARD_ROWS = 16  # prefetch.py:19


def _i64(arr):
    a = np.ascontiguousarray(np.asarray(arr, dtype=np.int64))
    return a, a.ctypes.data_as(ctypes.c_void_p)


def pool_heights(block_rows: int) -> list[int]:
    """descriptors.py:31-35"""
    out = np.zeros(64, dtype=np.int64)
    n = lib().tagg_pool_heights(int(block_rows), out.ctypes.data_as(ctypes.c_void_p), 64)
    if n < 0:
        raise_for_status(n, "pool_heights")
    return [int(x) for x in out[:n]]


@dataclass(frozen=True)
class DescriptorPool:
    """descriptors.py:38-54.  ``entries`` maps box height -> height.  The device
    pool holds one CUtensorMap per height (built per launch in tagg_gemm.cu)."""

    block_rows: int
    entries: dict

    def __len__(self) -> int:
        return len(self.entries)

    def select(self, residual_rows: int) -> int:
        h = lib().tagg_pool_select(int(residual_rows), int(self.block_rows))
        if h < 0:
            raise_for_status(int(h), "DescriptorPool.select")
        return int(h)


def build_pool(block_rows: int) -> DescriptorPool:
    """descriptors.py:57-69 (host view of the kernel's store pool)."""
    return DescriptorPool(block_rows, {h: h for h in pool_heights(block_rows)})


@dataclass(frozen=True)
class StorePhase:
    smem_row: int
    gmem_row: int


@dataclass(frozen=True)
class TwoPhasePlan:
    """descriptors.py:78-92"""

    residual_rows: int
    desc_rows: int
    phase_a: StorePhase
    phase_b: StorePhase

    @property
    def overlap_rows(self) -> int:
        return 2 * self.desc_rows - self.residual_rows

    def covered_gmem_rows(self) -> range:
        return range(self.phase_a.gmem_row, self.phase_b.gmem_row + self.desc_rows)


@dataclass(frozen=True)
class GroupStorePlan:
    """descriptors.py:109-114"""

    group: int
    rows: int
    full_tiles: int
    residual: TwoPhasePlan | None


def plan_group_stores(group_sizes, block_rows: int) -> list[GroupStorePlan]:
    """descriptors.py:117-129"""
    sizes, ptr = _i64(group_sizes)
    out = np.zeros((max(len(sizes), 1), 9), dtype=np.int64)
    rc = lib().tagg_plan_group_stores(ptr, len(sizes), int(block_rows), out.ctypes.data_as(ctypes.c_void_p))
    raise_for_status(rc, "plan_group_stores")
    plans = []
    for g in range(len(sizes)):
        _, rows, full, res, d, asm, agm, bsm, bgm = (int(x) for x in out[g])
        two = None if res == 0 else TwoPhasePlan(res, d, StorePhase(asm, agm), StorePhase(bsm, bgm))
        plans.append(GroupStorePlan(g, rows, full, two))
    return plans


def plan_two_phase(rows: int, block_rows: int) -> TwoPhasePlan | None:
    """descriptors.py:95-106"""
    return plan_group_stores([rows], block_rows)[0].residual


def format_plan(plans) -> str:
    """descriptors.py:132-150 (identical text)."""
    lines = []
    for p in plans:
        if p.residual is None:
            lines.append(f"group {p.group}: full={p.full_tiles} res=0")
            continue
        r = p.residual
        d = r.desc_rows
        a, b = r.phase_a, r.phase_b
        lines.append(
            f"group {p.group}: full={p.full_tiles} res={r.residual_rows} desc={d} "
            f"A:[{a.smem_row}..{a.smem_row + d - 1}]->[{a.gmem_row}..{a.gmem_row + d - 1}] "
            f"B:[{b.smem_row}..{b.smem_row + d - 1}]->[{b.gmem_row}..{b.gmem_row + d - 1}]"
        )
    return "\n".join(lines)


def scale_row_bytes(k: int) -> int:
    """prefetch.py:22-24"""
    return 4 * (-(-int(k) // 128))


def window_rows(block_rows: int) -> int:
    """prefetch.py:27-28"""
    return int(block_rows) + GUARD_ROWS


@dataclass(frozen=True)
class PrefetchWindow:
    """prefetch.py:31-47"""

    start_addr: int
    row_prev: int
    row_next: int
    total_rows: int
    row_bytes: int

    @property
    def window_bytes(self) -> int:
        return self.total_rows * self.row_bytes

    @property
    def valid_row_offset(self) -> int:
        return self.row_prev


def plan_prefetch(tile_start_addr: int, row_bytes: int, block_rows: int) -> PrefetchWindow:
    """prefetch.py:50-72"""
    if row_bytes <= 0:
        raise ValueError("row_bytes must be positive")
    out = np.zeros(4, dtype=np.int64)
    rc = lib().tagg_plan_prefetch(int(tile_start_addr), int(row_bytes), int(block_rows),
                                  out.ctypes.data_as(ctypes.c_void_p))
    raise_for_status(rc, "plan_prefetch")
    return PrefetchWindow(int(out[0]), int(out[1]), int(out[2]), int(out[3]), int(row_bytes))


def pad_rows(group_sizes, block_rows: int = 128) -> int:
    """workload.py:59-65"""
    sizes, ptr = _i64(group_sizes)
    return int(lib().tagg_pad_rows(ptr, len(sizes), int(block_rows)))


def row_payload_bytes(n: int, k: int) -> int:
    """workload.py:68-70"""
    return int(k) + scale_row_bytes(k) + 2 * int(n)


@dataclass(frozen=True)
class TrafficReport:
    """workload.py:73-81"""

    m_total: int
    padded_rows: int
    bytes_actual: int
    bytes_padded: int
    saving_pct: float
    eliminated_traffic_bytes: int
    residual_store_ops: int


def account(group_sizes, n: int, k: int, block_rows: int = 128, block_cols: int = 128) -> TrafficReport:
    """workload.py:84-111: the analytic "memory saved" metric."""
    sizes = [int(g) for g in group_sizes]
    m_total = sum(sizes)
    padded = pad_rows(sizes, block_rows)
    per_row = row_payload_bytes(n, k)
    actual = m_total * per_row
    padded_b = (m_total + padded) * per_row
    saving = 0.0 if padded_b == 0 else 1.0 - actual / padded_b
    n_tiles = -(-int(n) // block_cols)
    return TrafficReport(
        m_total=m_total,
        padded_rows=padded,
        bytes_actual=actual,
        bytes_padded=padded_b,
        saving_pct=100.0 * saving,
        eliminated_traffic_bytes=2 * padded * (int(k) + scale_row_bytes(k)),
        residual_store_ops=2 * n_tiles * sum(1 for g in sizes if g % block_rows != 0),
    )


def generate_group_sizes(m_total: int, groups: int, seed: int, *, max_attempts: int = 64) -> np.ndarray:
    """workload.py:30-56 (paper Appendix C.1 group-size generator)."""
    from .errors import InvalidInput

    if groups < 1:
        raise InvalidInput(f"groups must be >= 1, got {groups}")
    if m_total < 0:
        raise InvalidInput(f"m_total must be >= 0, got {m_total}")
    if m_total == 0:
        return np.zeros(groups, dtype=np.int64)
    hi = 2 * (m_total // groups)
    if hi == 0:
        sizes = np.zeros(groups, dtype=np.int64)
        sizes[-1] = m_total
        return sizes
    for attempt in range(max_attempts):
        rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence((seed, attempt))))
        v = rng.integers(0, hi, size=groups, endpoint=True).astype(np.int64)
        total = int(v.sum())
        if total == 0:
            continue
        v = np.floor((m_total / total) * v).astype(np.int64)
        v[-1] += m_total - int(v.sum())
        return v
    raise InvalidInput(f"no non-zero draw in {max_attempts} attempts (seed={seed})")

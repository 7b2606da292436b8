"""CPU ORACLE for the host planners (test infrastructure, never the product path).

Pure-Python restatement of the reference's planning layer.  It pins the
product's C++ planner (``tagg_plan_*`` in libtagg.so) and the kernel's
debug tile map bit for bit.  Every function cites the reference line it
restates (paths relative to /root/reference/pkg/src/tma_sim/).
"""

from __future__ import annotations

import math

import numpy as np

GUARD_ROWS = 16          # prefetch.py:19
GLOBAL_ALIGNMENT = 16    # memory.py:27
PAD_BLOCK_ROWS = 128     # workload.py:27


def floor_pow2(n: int) -> int:
    """descriptors.py:27-28"""
    return 1 << (n.bit_length() - 1)


def pool_heights(block_rows: int) -> list[int]:
    """descriptors.py:31-35"""
    if block_rows < 1 or block_rows & (block_rows - 1):
        raise ValueError(f"block_rows must be a power of two, got {block_rows}")
    return [1 << i for i in range(block_rows.bit_length())]


def pool_select(residual_rows: int, block_rows: int) -> int:
    """DescriptorPool.select, descriptors.py:48-54 (returns the box height)."""
    if residual_rows < 1 or residual_rows > block_rows:
        raise ValueError(f"residual_rows {residual_rows} outside [1, {block_rows}]")
    return floor_pow2(residual_rows)


def plan_two_phase(rows: int, block_rows: int):
    """descriptors.py:95-106 -> (res, d, a_smem, a_gmem, b_smem, b_gmem) or None."""
    res = rows % block_rows
    if res == 0:
        return None
    d = floor_pow2(res)
    return (res, d, 0, rows - res, res - d, rows - d)


def plan_group_stores(group_sizes, block_rows: int):
    """descriptors.py:117-129 -> list of (group, rows, full_tiles, two_phase|None)."""
    return [(g, int(r), int(r) // block_rows, plan_two_phase(int(r), block_rows))
            for g, r in enumerate(group_sizes)]


def format_plan(plans) -> str:
    """descriptors.py:132-150"""
    lines = []
    for g, _rows, full, res in plans:
        if res is None:
            lines.append(f"group {g}: full={full} res=0")
            continue
        r, d, asm, agm, bsm, bgm = res
        lines.append(
            f"group {g}: full={full} res={r} desc={d} "
            f"A:[{asm}..{asm + d - 1}]->[{agm}..{agm + d - 1}] "
            f"B:[{bsm}..{bsm + d - 1}]->[{bgm}..{bgm + d - 1}]"
        )
    return "\n".join(lines)


def kernel_tile_map(group_sizes, n: int, tile: str = "pair_n256", c_row_offsets=None, num_pairs=None, raster=8):
    """The store geometry the B200 kernel uses, stated with the reference planner.

    Every stored piece follows plan_two_phase (descriptors.py:72-106) for its block
    height.  For the 1-CTA and 256x128 pair tiles that is exactly the reference tile
    loop (tile_map, block_m = 128).  The default 256x256 pair tile computes a group's
    last pair tile with at most 128 valid rows as a HALF tile (one tcgen05.mma M=128
    per K step, 64 rows per CTA), and each CTA stores its 64-row piece with the
    reference plan at block_rows = 64: a full piece is one 64-row store, a residual
    piece the two-phase store.  Tail balancing (num_pairs = the launch's CTA pairs,
    tagg_launch_clusters): when T mod num_pairs <= num_pairs / 2 for T scheduled
    tiles, the last T mod num_pairs tiles in schedule order each run as two half
    tiles of 128 rows (64-row pieces again).  The mapping of rows to groups (which C
    rows each piece writes, never a row past M_g) is the reference's in every case.
    Records: (g, m_tile, n0, a_row0, valid, d, phaseA_gmem_row, phaseB_smem_row,
    phaseB_gmem_row), m_tile = the reference's 128-row tile index.
    """
    if tile != "pair_n256":
        return tile_map(group_sizes, n, c_row_offsets=c_row_offsets)
    sizes = [int(x) for x in group_sizes]
    offs, coffs, o = [], [], 0
    for g, rows in enumerate(sizes):
        offs.append(o)
        coffs.append(o if c_row_offsets is None else int(c_row_offsets[g]))
        o += rows
    ntn = -(-n // 256)
    # the kernel's static schedule (decode_tile): groups in order, inside a group
    # super-rows of `raster` pair m-tiles (tagg_raster_tiles) with n-tiles outer
    sched = []
    for g, rows in enumerate(sizes):
        pt = -(-rows // 256)
        for local in range(pt * ntn):
            sr = local // (raster * ntn)
            h = min(raster, pt - sr * raster)
            loc = local - sr * raster * ntn
            sched.append((g, sr * raster + loc % h, (loc // h) * 256))
    T = len(sched)
    x = 0
    if num_pairs:
        tail = T % num_pairs
        x = tail if (tail and 2 * tail <= num_pairs) else 0

    def piece(g, mt, n0, r0, v):
        d = 1 << (v.bit_length() - 1)
        for c in (n0, n0 + 128):
            if c < n:
                recs.append((g, mt, c, offs[g] + r0, v, d, coffs[g] + r0, v - d, coffs[g] + r0 + v - d))

    recs = []
    for idx, (g, pm, n0) in enumerate(sched):
        rows, base = sizes[g], 256 * pm
        if idx >= T - x:  # tail balancing: two half tiles of 128 rows
            for sub in range(2):
                for j in range(2):
                    r0 = base + 128 * sub + 64 * j
                    v = min(64, rows - r0)
                    if v > 0:
                        piece(g, 2 * pm + sub, n0, r0, v)
        elif rows - base <= 128:  # half tile: two 64-row pieces
            for j in range(2):
                r0 = base + 64 * j
                v = min(64, rows - r0)
                if v > 0:
                    piece(g, 2 * pm, n0, r0, v)
        else:
            for t in (2 * pm, 2 * pm + 1):
                r0 = 128 * t
                v = min(128, rows - r0)
                piece(g, t, n0, r0, v)
    return recs


def scale_row_bytes(k: int) -> int:
    """prefetch.py:22-24"""
    return 4 * (-(-k // 128))


def plan_prefetch(tile_start_addr: int, row_bytes: int, block_rows: int):
    """prefetch.py:50-72 -> (start_addr, row_prev, row_next, total_rows)."""
    if row_bytes <= 0:
        raise ValueError("row_bytes must be positive")
    for r in range(GUARD_ROWS):
        start = tile_start_addr - r * row_bytes
        if start % GLOBAL_ALIGNMENT == 0:
            total = block_rows + GUARD_ROWS
            return (start, r, total - r, total)
    raise ValueError("NoAlignedSolution")


def tile_map(group_sizes, n: int, block_m: int = 128, block_n: int = 128, c_row_offsets=None):
    """The tile -> (group, row) mapping of the reference tile loop (engine.py:269-335).

    One record per (group, m-tile, n-tile):
    (g, m_tile, n0, a_row0, valid, d, phaseA_gmem_row, phaseB_smem_row, phaseB_gmem_row).
    Full tiles carry d = block_m and identical phase rows (one store of height
    block_m at the tile's first row, engine.py:318-322).  Residual tiles carry the
    two-phase plan (engine.py:323-335).  Gmem rows are absolute rows of C.  They
    equal the A row plus any caller-supplied output-row offset per group.
    """
    recs = []
    off = 0
    for g, rows in enumerate(group_sizes):
        rows = int(rows)
        coff = off if c_row_offsets is None else int(c_row_offsets[g])
        full = rows // block_m
        res = plan_two_phase(rows, block_m)
        mt_count = full + (1 if res else 0)
        for t in range(mt_count):
            is_res = res is not None and t == full
            for n0 in range(0, n, block_n):
                if not is_res:
                    r0 = t * block_m
                    recs.append((g, t, n0, off + r0, block_m, block_m, coff + r0, 0, coff + r0))
                else:
                    r, d, _asm, agm, bsm, bgm = res
                    recs.append((g, t, n0, off + t * block_m, r, d, coff + agm, bsm, coff + bgm))
        off += rows
    return recs


def pad_rows(group_sizes, block_rows: int = PAD_BLOCK_ROWS) -> int:
    """workload.py:59-65"""
    return sum(-(-int(g) // block_rows) * block_rows - int(g) for g in group_sizes)


def row_payload_bytes(n: int, k: int) -> int:
    """workload.py:68-70"""
    return k + scale_row_bytes(k) + 2 * n


def account(group_sizes, n: int, k: int, block_rows: int = PAD_BLOCK_ROWS, block_cols: int = 128):
    """workload.py:84-111 -> dict with the TrafficReport fields."""
    sizes = [int(g) for g in group_sizes]
    m_total = sum(sizes)
    padded = pad_rows(sizes, block_rows)
    per_row = row_payload_bytes(n, k)
    bytes_actual = m_total * per_row
    bytes_padded = (m_total + padded) * per_row
    saving = 0.0 if bytes_padded == 0 else 1.0 - bytes_actual / bytes_padded
    return dict(
        m_total=m_total,
        padded_rows=padded,
        bytes_actual=bytes_actual,
        bytes_padded=bytes_padded,
        saving_pct=100.0 * saving,
        eliminated_traffic_bytes=2 * padded * (k + scale_row_bytes(k)),
        residual_store_ops=2 * (-(-n // block_cols)) * sum(1 for g in sizes if g % block_rows),
    )


def generate_group_sizes(m_total: int, groups: int, seed: int, max_attempts: int = 64):
    """workload.py:30-56 (paper Appendix C.1 generator)."""
    if groups < 1 or m_total < 0:
        raise ValueError("bad arguments")
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
    raise ValueError("no non-zero draw")


def n_tiles(n: int, block_n: int = 128):
    """engine.py:117-120"""
    return [(c, min(block_n, n - c)) for c in range(0, n, block_n)]


def k_blocks(k: int) -> int:
    """fp8.py:128-129"""
    return math.ceil(k / 128)

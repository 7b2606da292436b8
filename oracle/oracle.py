"""CPU ORACLE entry points (test infrastructure, never the product path).

ctypes front end for liboracle.so (oracle/tagg_oracle.c), the C restatement
of the reference's grouped FP8 GEMM (engine.py:346-402 semantics).  Only
tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import this
module, and only as the checker or the timed CPU baseline.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "liboracle.so"
_lib = None


def build() -> Path:
    """Compile the oracle with its Makefile (gcc)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(LIB_PATH))
        L.tagg_oracle_grouped_gemm.restype = ctypes.c_int
        L.tagg_oracle_grouped_gemm.argtypes = [
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
        ]
        L.tagg_oracle_wgrad.restype = ctypes.c_int
        L.tagg_oracle_wgrad.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_void_p, ctypes.c_int]
        L.tagg_oracle_bf16_from_f32.restype = ctypes.c_uint16
        L.tagg_oracle_bf16_from_f32.argtypes = [ctypes.c_float]
        L.tagg_oracle_decode.restype = ctypes.c_float
        L.tagg_oracle_decode.argtypes = [ctypes.c_uint8]
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def grouped_gemm(a_codes, a_scales, b_codes, b_scales, group_sizes, *, b_layout="kn",
                 c_row_offsets=None, c_rows=None, n_range=None, threads=None, out=None):
    """C bits (uint16) of the reference semantics.

    b_codes: [K,N] shared (reference layout) or [G,K,N] per expert ("kn"), or
    [G,N,K] per expert when b_layout == "nk" (dgrad / K-major).  b_scales:
    [kb,nb] / [G,kb,nb] ("kn") or [G,nb,kb] ("nk").
    """
    a_codes = np.ascontiguousarray(a_codes, dtype=np.uint8)
    a_scales = np.ascontiguousarray(a_scales, dtype=np.float32)
    b_codes = np.ascontiguousarray(b_codes, dtype=np.uint8)
    b_scales = np.ascontiguousarray(b_scales, dtype=np.float32)
    sizes = np.ascontiguousarray(np.asarray(group_sizes, dtype=np.int64))
    G = len(sizes)
    M, K = a_codes.shape
    if b_layout == "kn":
        N = b_codes.shape[-1]
        shared = b_codes.ndim == 2
        b_es = 0 if shared else K * N
        kb, nb = b_scales.shape[-2], b_scales.shape[-1]
        sb_es = 0 if shared else kb * nb
        sb_kb, sb_nb, kmajor = nb, 1, 0
    elif b_layout == "nk":
        N = b_codes.shape[-2]
        b_es = N * K
        nb, kb = b_scales.shape[-2], b_scales.shape[-1]
        sb_es = nb * kb
        sb_kb, sb_nb, kmajor = 1, kb, 1
    else:
        raise ValueError(b_layout)
    offs = None
    if c_row_offsets is not None:
        offs = np.ascontiguousarray(np.asarray(c_row_offsets, dtype=np.int64))
    rows = c_rows if c_rows is not None else M
    if out is None:
        out = np.zeros((rows, N), dtype=np.uint16)
    n0, n1 = (0, N) if n_range is None else n_range
    nthr = threads or 1
    rc = lib().tagg_oracle_grouped_gemm(
        _ptr(a_codes), _ptr(a_scales), _ptr(b_codes), b_es, kmajor, _ptr(b_scales), sb_es,
        sb_kb, sb_nb, _ptr(sizes), G, N, K, _ptr(out),
        _ptr(offs) if offs is not None else None, out.shape[1], n0, n1, nthr)
    if rc != 0:
        raise ValueError(f"oracle rejected arguments (rc={rc})")
    return out


def host_threads() -> int:
    return len(os.sched_getaffinity(0))


def wgrad(x_codes, x_scales, dy_codes, dy_scales, group_sizes, *, threads=None):
    """dW bits [G, K, N] (uint16) of the weight gradient X_g^T dY_g (tagg_oracle_wgrad).

    x_codes [M, K], dy_codes [M, N]; x_scales [TB, K], dy_scales [TB, N]: one row per
    (group, 128-token block), blocks numbered group by group.
    """
    x_codes = np.ascontiguousarray(x_codes, dtype=np.uint8)
    dy_codes = np.ascontiguousarray(dy_codes, dtype=np.uint8)
    x_scales = np.ascontiguousarray(x_scales, dtype=np.float32)
    dy_scales = np.ascontiguousarray(dy_scales, dtype=np.float32)
    sizes = np.ascontiguousarray(np.asarray(group_sizes, dtype=np.int64))
    G = len(sizes)
    K, N = x_codes.shape[1], dy_codes.shape[1]
    out = np.zeros((G, K, N), dtype=np.uint16)
    rc = lib().tagg_oracle_wgrad(_ptr(x_codes), _ptr(x_scales), _ptr(dy_codes), _ptr(dy_scales), _ptr(sizes),
                                 G, K, N, _ptr(out), threads or 1)
    if rc != 0:
        raise ValueError(f"oracle rejected arguments (rc={rc})")
    return out

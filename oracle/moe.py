"""CPU ORACLE for the MoE FFN steps around the GEMM (test infrastructure only).

numpy float32 restatements of csrc/tagg_moe.cu:
* swiglu(h_bits): v = fl(fl(g / fl(1 + exp(-g))) * u) per element, g = gate, u = up (the
  first and second halves of each bf16 row).  The kernel uses the fast exp and division
  (a few ulp), so tests compare the quantized result with a tolerance.
* combine(c_bits, dest, w): acc = fl(acc + fl(w * c)) in k order, then bf16 RNE -- the
  same operation order as the kernel, so the result is bit-exact.
The quantizer applied to v is fp8.quantize_row_tiles (fp8.py:132-151).
"""

from __future__ import annotations

import numpy as np

from .fp8 import bf16_bits_to_f32


def swiglu(h_bits: np.ndarray) -> np.ndarray:
    h = bf16_bits_to_f32(h_bits)
    i = h.shape[1] // 2
    g, u = h[:, :i], h[:, i:2 * i]
    with np.errstate(over="ignore"):
        den = (np.float32(1.0) + np.exp(-g)).astype(np.float32)
    return ((g / den).astype(np.float32) * u).astype(np.float32)


def bf16_rne(x: np.ndarray) -> np.ndarray:
    """engine.py:46-50: (u + 0x7FFF + ((u >> 16) & 1)) >> 16."""
    u = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


def combine(c_bits: np.ndarray, dest: np.ndarray, w: np.ndarray) -> np.ndarray:
    c = bf16_bits_to_f32(c_bits)
    t, topk = w.shape
    acc = np.zeros((t, c.shape[1]), np.float32)
    for k in range(topk):
        rows = c[dest.reshape(t, topk)[:, k]]
        acc = (acc + (w[:, k:k + 1].astype(np.float32) * rows).astype(np.float32)).astype(np.float32)
    return bf16_rne(acc)


def swiglu_backward(h_bits: np.ndarray, dh_bits: np.ndarray) -> np.ndarray:
    """d[g | u] in float32 from gate|up rows and dL/d(silu(g) * u) (tagg_moe.cu K9)."""
    h = bf16_bits_to_f32(h_bits).astype(np.float64)
    dh = bf16_bits_to_f32(dh_bits).astype(np.float64)
    i = h.shape[1] // 2
    g, u = h[:, :i], h[:, i:2 * i]
    with np.errstate(over="ignore"):
        sig = 1.0 / (1.0 + np.exp(-g))
    return np.concatenate([dh * u * sig * (1 + g * (1 - sig)), dh * g * sig], axis=1).astype(np.float32)

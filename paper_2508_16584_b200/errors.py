"""Exception hierarchy of the reference (errors.py:6-76), same names and bases.

C-ABI status codes (include/tagg.h) map onto these classes in
``raise_for_status``.  A caller catching the reference's exceptions catches ours
the same way.
"""

from __future__ import annotations


class SimError(Exception):
    """Base class (errors.py:6)."""


class InvalidInput(SimError):
    """errors.py:10"""


class ConfigError(SimError):
    """errors.py:14"""


class InvalidBlockM(ConfigError):
    """errors.py:18"""


class InvalidBlockN(ConfigError):
    """errors.py:22"""


class AlignmentError(SimError):
    """errors.py:30-40: a global start address violates the 16-byte rule."""


class BoundsError(SimError):
    """errors.py:43-57"""


class ResOutOfRange(SimError):
    """errors.py:60"""


class NoAlignedSolution(SimError):
    """errors.py:64-68"""


class ShapeMismatch(SimError):
    """errors.py:71"""


class Unsupported(SimError):
    """Shape exceeds this build's on-chip budget (no reference counterpart)."""


class CudaError(SimError):
    """CUDA runtime/driver failure inside the native library."""


_CODES = {
    -1: ConfigError,
    -2: InvalidBlockM,
    -3: InvalidBlockN,
    -4: ShapeMismatch,
    -5: AlignmentError,
    -6: NoAlignedSolution,
    -7: ResOutOfRange,
    -8: Unsupported,
    -9: CudaError,
}


def raise_for_status(code: int, what: str) -> None:
    if code == 0:
        return
    cls = _CODES.get(int(code), SimError)
    raise cls(f"{what}: {cls.__name__} (status {code})")

"""Error hierarchy of the drop-in boundary.

Mirrors the reference's ``localmap.errors`` names (pkg/src/localmap/errors.py:4-37) so
callers that catch ``LocalMapError`` subclasses keep working. The C ABI never throws:
every entry point returns an ``lm_status`` code (include/lm_b200.h) and the Python
facade maps it back onto these classes in ``_lib.check``.
"""

from __future__ import annotations


class LocalMapError(Exception):
    """Root of every error this package raises (errors.py:4)."""


class DegenerateGeometryError(LocalMapError):
    """Zero baseline, point at infinity and similar ill-posed geometry (errors.py:8)."""


class InvalidArgumentError(LocalMapError):
    """A caller broke the operation contract (errors.py:12)."""


class InvalidStateError(LocalMapError):
    """Entity in the wrong lifecycle state, e.g. dead keyframe (errors.py:16)."""


class SlotConflictError(InvalidStateError):
    """Keypoint slot already bound to another map point (errors.py:20)."""


class StoreCapacityError(InvalidStateError):
    """A pre-allocated device arena is full (errors.py:24)."""


class DeviceError(LocalMapError):
    """CUDA runtime failure or a missing native library. Never swallowed."""

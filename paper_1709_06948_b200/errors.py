"""Exception types, mirroring the reference's hot-path errors (errors.py:6-44)."""

from __future__ import annotations


class VoxmiError(Exception):
    """Base class for package-specific errors (errors.py:6)."""


class OutOfBoundsError(VoxmiError):
    """A point falls outside the representable voxel index range (errors.py:35)."""


class EmptyOverlapError(VoxmiError):
    """The occupied bounds do not intersect at the probed pose (errors.py:39)."""


class NoOverlapError(VoxmiError):
    """No probed pose produced any overlap (errors.py:43)."""

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


class FormatError(VoxmiError):
    """A file does not conform to its declared format (errors.py:9-27): the
    path, the reason, and the line or byte offset of the offending record."""

    def __init__(self, path, reason: str, line: int | None = None,
                 byte_offset: int | None = None):
        self.path = str(path)
        self.reason = reason
        self.line = line
        self.byte_offset = byte_offset
        loc = f", line {line}" if line is not None else (
            f", byte {byte_offset}" if byte_offset is not None else "")
        super().__init__(f"{self.path}{loc}: {reason}")

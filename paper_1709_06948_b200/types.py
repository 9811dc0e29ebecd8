"""Value types of the hot path, mirroring the reference's dataclasses.

FeatureKind / GridSpec (voxel.py:33-62), FeatureMap (voxel.py:129-164),
BinningSpec / JointHistogram / MIResult (mi.py:40-108), AlignmentConfig
(align.py:47-67, without the Nelder-Mead simplex, which is out of scope).
Objects of the reference package itself are accepted wherever these are
(duck-typed on the same field names), so a voxmi caller can hand its own
FeatureMap / GridSpec / BinningSpec straight to this package.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field

import numpy as np

NO_OVERLAP_SENTINEL = -1e300  # mi.py:34
DEFAULT_BIN_COUNT = 32        # mi.py:36
KEY_INDEX_MIN = -(1 << 20)    # voxel.py:26
KEY_INDEX_MAX = (1 << 20) - 1  # voxel.py:27


class FeatureKind(enum.Enum):
    """Per-voxel scalar feature (voxel.py:33-46)."""

    VARZ = "varz"
    COUNT = "count"

    @classmethod
    def from_name(cls, name: str) -> "FeatureKind":
        try:
            return cls(name.strip().lower())
        except ValueError:
            raise ValueError(
                f"unknown feature kind {name!r}; expected 'varz' or 'count'") from None

    @property
    def code(self) -> int:
        return 0 if self is FeatureKind.VARZ else 1


DEFAULT_UPPER_CLAMP = {FeatureKind.VARZ: 2.0, FeatureKind.COUNT: 64.0}  # mi.py:37


def as_kind(kind) -> FeatureKind:
    """Accept this package's FeatureKind, the reference's, or a name."""
    if isinstance(kind, FeatureKind):
        return kind
    if isinstance(kind, str):
        return FeatureKind.from_name(kind)
    value = getattr(kind, "value", None)
    if isinstance(value, str):
        return FeatureKind.from_name(value)
    raise ValueError(f"not a feature kind: {kind!r}")


@dataclass(frozen=True)
class GridSpec:
    """Cubic voxel grid: origin (3 floats, m) and edge length (voxel.py:49-62)."""

    origin: np.ndarray = field(default_factory=lambda: np.zeros(3))
    resolution: float = 1.0

    def __post_init__(self):
        origin = np.asarray(self.origin, dtype=np.float64)
        if origin.shape != (3,) or not np.isfinite(origin).all():
            raise ValueError(f"grid origin must be 3 finite floats, got {self.origin}")
        object.__setattr__(self, "origin", origin)
        if not (np.isfinite(self.resolution) and self.resolution > 0):
            raise ValueError(f"grid resolution must be > 0, got {self.resolution}")


@dataclass(frozen=True)
class BinningSpec:
    """Linear binning with bin 0 reserved for no-feature (mi.py:40-59)."""

    kind: FeatureKind
    bin_count: int = DEFAULT_BIN_COUNT
    upper_clamp: float = 0.0

    def __post_init__(self):
        object.__setattr__(self, "kind", as_kind(self.kind))
        if self.bin_count < 2:
            raise ValueError(f"bin_count must be >= 2, got {self.bin_count}")
        if self.upper_clamp == 0.0:
            object.__setattr__(self, "upper_clamp", DEFAULT_UPPER_CLAMP[self.kind])
        if not self.upper_clamp > 0:
            raise ValueError(f"upper_clamp must be > 0, got {self.upper_clamp}")


@dataclass(frozen=True)
class FeatureMap:
    """Occupied voxels of one scan: sorted packed keys, features, (2, 3) bounds
    (voxel.py:129-164)."""

    kind: FeatureKind
    keys: np.ndarray
    values: np.ndarray
    bounds: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "kind", as_kind(self.kind))
        if self.keys.shape != self.values.shape:
            raise ValueError("keys and values must have matching shapes")
        if self.values.size and (not np.isfinite(self.values).all() or (self.values < 0).any()):
            raise ValueError("features must be finite and >= 0")

    def __len__(self) -> int:
        return self.keys.shape[0]


@dataclass(frozen=True)
class JointHistogram:
    """(B+1)^2 joint counts, row = scan A bin, column = scan B bin (mi.py:82-98)."""

    counts: np.ndarray
    total: int
    spec: BinningSpec

    def row_marginal(self) -> np.ndarray:
        return self.counts.sum(axis=1)

    def col_marginal(self) -> np.ndarray:
        return self.counts.sum(axis=0)


@dataclass(frozen=True)
class MIResult:
    """Entropy breakdown in nats (mi.py:101-108)."""

    mi: float
    h_x: float
    h_y: float
    h_xy: float


@dataclass(frozen=True)
class AlignmentConfig:
    """Feature, grid, binning and phi switch of one run (align.py:47-67).

    The reference's Nelder-Mead ``simplex`` field is accepted and ignored:
    the serial optimizer is outside this package's scope.
    """

    feature: FeatureKind = FeatureKind.VARZ
    grid: GridSpec = field(default_factory=GridSpec)
    binning: BinningSpec | None = None
    phi_enabled: bool = True
    simplex: object = None

    def __post_init__(self):
        feature = as_kind(self.feature)
        object.__setattr__(self, "feature", feature)
        binning = self.binning
        if binning is None:
            binning = BinningSpec(kind=feature)
        elif as_kind(binning.kind) is not feature:
            raise ValueError(f"binning kind {binning.kind} does not match feature {feature}")
        object.__setattr__(self, "binning", binning)

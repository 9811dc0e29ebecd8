"""B200-native batched MI pose evaluation (arXiv 1709.06948 hot path).

Drop-in for the reference `voxmi` package's hot path -- ``mi_objective``
(mi.py:194-219) and its callers -- with the work done by hand-written sm_100a
kernels behind a C ABI (include/vmi.h, libvmi.so).  See DESIGN.md.
"""

from .api import (SWEEP_AXES, SearchResult, clear_cache, compute_feature_map, engine_for,
                  grid_search, grid_search_sharded, joint_histogram_at, mi_at, mi_objective,
                  mi_objective_batch, sweep_axis)
from .align import AlignmentReport, align, align_batch
from .engine import MIEngine, entropy_exact, mutual_information_exact
from .optim import OptimResult, SimplexConfig, nelder_mead_maximize_batched
from .errors import EmptyOverlapError, NoOverlapError, OutOfBoundsError, VoxmiError
from .geometry import (EulerPose, PointCloud, as_pose_array, euler_to_transform, normalized,
                       transform_to_euler, validate_transform)
from .types import (DEFAULT_BIN_COUNT, DEFAULT_UPPER_CLAMP, KEY_INDEX_MAX, KEY_INDEX_MIN,
                    NO_OVERLAP_SENTINEL, AlignmentConfig, BinningSpec, FeatureKind, FeatureMap,
                    GridSpec, JointHistogram, MIResult)
from ._lib import VmiError, poses_to_mats
from .scan_io import load_kitti_bin, save_kitti_bin

__all__ = [
    "AlignmentReport", "align", "align_batch", "OptimResult", "SimplexConfig", "nelder_mead_maximize_batched",
    "normalized", "transform_to_euler", "validate_transform",
    "SWEEP_AXES", "SearchResult", "clear_cache", "compute_feature_map", "engine_for",
    "grid_search", "grid_search_sharded", "joint_histogram_at", "mi_at", "mi_objective",
    "mi_objective_batch",
    "sweep_axis", "MIEngine", "entropy_exact", "mutual_information_exact", "EmptyOverlapError",
    "NoOverlapError", "OutOfBoundsError", "VoxmiError", "EulerPose", "PointCloud",
    "as_pose_array", "euler_to_transform", "DEFAULT_BIN_COUNT", "DEFAULT_UPPER_CLAMP",
    "KEY_INDEX_MAX", "KEY_INDEX_MIN", "NO_OVERLAP_SENTINEL", "AlignmentConfig", "BinningSpec",
    "FeatureKind", "FeatureMap", "GridSpec", "JointHistogram", "MIResult", "VmiError",
    "poses_to_mats", "load_kitti_bin", "save_kitti_bin",
]

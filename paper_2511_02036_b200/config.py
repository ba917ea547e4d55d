"""Stage parameters of the hot path, same fields and defaults as the reference.

Cited from pkg/src/localmap/config.py: GateConfig 13-19, MatchConfig 22-30, FuseConfig
33-44, CullConfig 63-72 (only the recent-point fields are used here), StoreConfig 75-82,
MapConfig 85-90. ``chunk_size`` fields are accepted for signature compatibility; the
device grid does not chunk by them.
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass
class GateConfig:
    cos_parallax_max: float = 0.9998
    chi2_mono: float = 5.991
    scale_ratio_slack: float = 1.5


@dataclass
class MatchConfig:
    match_max_distance: int = 50
    chi2_epi: float = 3.84
    level_window: int = 1
    neighbor_count: int = 10
    chunk_size: int = 256


@dataclass
class FuseConfig:
    match_max_distance: int = 50
    fuse_radius: float = 3.0
    min_view_cos: float = 0.5
    dist_band_slack: float = 1.5
    level_window: int = 1
    n1: int = 20
    n2: int = 5
    chunk_size: int = 512


@dataclass
class CullConfig:
    found_ratio_min: float = 0.25
    probation_kfs: int = 3
    min_obs_graduate: int = 3
    redundancy_ratio: float = 0.9
    min_redundant_observers: int = 3
    scale_tolerance_levels: int = 0


@dataclass
class StoreConfig:
    """Ledger sizes (config.py:75-82) plus the device arena capacities."""

    keypoint_record_bytes: int = 16
    descriptor_bytes: int = 32
    map_point_record_bytes: int = 100
    capacity: int = 4096
    # device arenas (this package only)
    max_keyframes: int = 4096  # = capacity; <= LM_MAX_KF_SLOTS (8192)
    max_keypoints: int = 1 << 21
    max_points: int = 1 << 20
    obs_pool_entries: int = 1 << 24
    max_keypoints_per_kf: int = 8192


@dataclass
class MapConfig:
    min_obs_keep: int = 2
    min_covis_weight: int = 1
